"""ctypes binding of include/fdsweep_b200.h with the reference's names and
error classes (proj/include/fdsweep/types.hpp:14-36).

Complex arrays cross the C-ABI as interleaved float64 pairs (``fds_c64``), the
layout of std::complex<double>. Host layouts follow the reference:
samples ``values[j, k]`` (per-frequency AoS, types.hpp:40-45), residues
``residues[k, m]`` (vecfit.hpp:21-30), time series ``values[k, n]``.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIB_NAME = "libfdsweep_b200.so"


def library_path() -> Path:
    # FDSWEEP_LIB_VARIANT=jitter selects the race-stress build (same code with
    # timing perturbation at the synchronisation points; tests only)
    if os.environ.get("FDSWEEP_LIB_VARIANT") == "jitter":
        return HERE / _LIB_NAME.replace(".so", "_jitter.so")
    return HERE / _LIB_NAME


class Error(RuntimeError):
    """Base of the toolkit errors (types.hpp:14-17)."""


class ValidationError(Error):
    pass


class NumericError(Error):
    pass


class IoError(Error):
    pass


class ConvergenceError(Error):
    pass


class CudaError(Error):
    """The device path failed; there is no CPU fallback."""


_ERRS = {1: ValidationError, 2: NumericError, 3: IoError, 4: ConvergenceError, 5: CudaError}


class _C64(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class BemDesc(ctypes.Structure):
    _fields_ = [
        ("n_vertices", ctypes.c_int),
        ("vertices", ctypes.c_void_p),
        ("n_elements", ctypes.c_int),
        ("triangles", ctypes.c_void_p),
        ("shear_modulus", ctypes.c_double),
        ("poisson_ratio", ctypes.c_double),
        ("density", ctypes.c_double),
        ("traction", ctypes.c_void_p),
        ("n_channels", ctypes.c_int),
        ("channels", ctypes.c_void_p),
        ("max_batch", ctypes.c_int),
    ]


class AfsConfigC(ctypes.Structure):
    _fields_ = [
        ("initial_count", ctypes.c_int),
        ("alpha_high", ctypes.c_double),
        ("alpha_low", ctypes.c_double),
        ("e1_threshold", ctypes.c_double),
        ("e2_threshold", ctypes.c_double),
        ("validation_steps", ctypes.c_int),
        ("n_orf", ctypes.c_int),
        ("orf_indices", ctypes.c_void_p),
        ("n_test", ctypes.c_int),
        ("test_indices", ctypes.c_void_p),
        ("omega_max", ctypes.c_double),
        ("eta", ctypes.c_double),
        ("period", ctypes.c_double),
        ("grid_points", ctypes.c_int),
        ("time_points", ctypes.c_int),
        ("max_iterations", ctypes.c_int),
        ("seed", ctypes.c_uint64),
        ("n_relocations", ctypes.c_int),
    ]


class AfsSummaryC(ctypes.Structure):
    _fields_ = [("n_c", ctypes.c_int), ("converged", ctypes.c_int), ("solver_calls", ctypes.c_int),
                ("n_history", ctypes.c_int), ("order", ctypes.c_int), ("n_orf", ctypes.c_int),
                ("orf_indices", ctypes.c_int * 8)]


SYSTEM_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, _C64, ctypes.c_void_p)

_lib = None


def lib():
    """Loads the CUDA library; raises CudaError when it is missing (no fallback)."""
    global _lib
    if _lib is None:
        p = library_path()
        if not p.exists():
            raise CudaError(f"{p} is missing: build it with `make -C paper_1511_04355_b200` "
                            "(or __graft_entry__.build()); there is no CPU fallback")
        _lib = ctypes.CDLL(str(p))
        _lib.fds_last_error.restype = ctypes.c_char_p
        _lib.fds_version.restype = ctypes.c_char_p
        _lib.fds_kernel_launches.restype = ctypes.c_int64
    return _lib


def _check(rc: int):
    if rc != 0:
        cls = _ERRS.get(rc, Error)
        raise cls(lib().fds_last_error().decode())


def _cz(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def version() -> str:
    return lib().fds_version().decode()


def profile_enable(on: bool = True):
    """Per-kernel-class device timings (CUDA events) and algorithmic work, as bench.py reads them."""
    _check(lib().fds_profile_enable(1 if on else 0))


def profile_read(kind: int):
    """(launch count, total ms, total algorithmic work) of one profiler class (csrc/common.cuh kProf*)."""
    c, ms, wk = ctypes.c_int(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(lib().fds_profile_read(kind, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    return c.value, ms.value, wk.value


def redzone_check() -> dict:
    """Debug (fds_debug_redzone_check): with FDSWEEP_REDZONE set before the library loads, compares the
    guard zones around every device allocation of the library; `overwritten_bytes` must be 0."""
    on, bad, chk, live = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
    _check(lib().fds_debug_redzone_check(ctypes.byref(on), ctypes.byref(bad), ctypes.byref(chk), ctypes.byref(live)))
    return {"enabled": bool(on.value), "overwritten_bytes": bad.value, "checks": chk.value, "live": live.value}


def kernel_launches() -> int:
    return int(lib().fds_kernel_launches())


def zgesv_batch(A, rhs):
    """x[b] = A[b]^{-1} rhs[b] on the GPU (A: (B, n, n) complex; rhs: (B, n))."""
    A = np.asarray(A, np.complex128)
    if A.ndim == 2:
        A = A[None]
    rhs = np.asarray(rhs, np.complex128).reshape(A.shape[0], A.shape[1])
    B, n, _ = A.shape
    Acm = np.ascontiguousarray(np.transpose(A, (0, 2, 1)))  # column-major per matrix
    r = np.ascontiguousarray(rhs)
    x = np.zeros_like(r)
    _check(lib().fds_zgesv_batch(n, B, _p(Acm), _p(r), _p(x)))
    return x


# ---------------------------------------------------------------- BEM system
@dataclass
class SystemDescriptor:
    channel_count: int
    channel_labels: list
    band_hint: float | None = None


class BemSystem:
    """FrequencySystem (systems.hpp:34-42) backed by the GPU collocation BEM.

    ``evaluate(s)`` returns the displacement at the channel DOFs (element-major
    u[3e + {x,y,z}]) for the Laplace parameter s; ``evaluate_batch`` solves B
    frequencies as independent batched systems.
    """

    def __init__(self, vertices, triangles, traction, mu=1.0, nu=0.25, rho=1.0, channels=None,
                 max_batch=0):
        self._v = np.ascontiguousarray(vertices, np.float64)
        self._t = np.ascontiguousarray(triangles, np.int32)
        self._tr = np.ascontiguousarray(traction, np.float64)
        self._ch = None if channels is None else np.ascontiguousarray(channels, np.int32)
        d = BemDesc(self._v.shape[0], _p(self._v), self._t.shape[0], _p(self._t), float(mu), float(nu),
                    float(rho), _p(self._tr), 0 if self._ch is None else len(self._ch), _p(self._ch),
                    int(max_batch))
        h = ctypes.c_void_p()
        _check(lib().fds_bem_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self.unknowns = 3 * self._t.shape[0]
        k = lib().fds_bem_channels(self._h)
        labels = [f"u{d}" for d in (range(self.unknowns) if self._ch is None else self._ch)]
        self._desc = SystemDescriptor(k, labels)

    def descriptor(self) -> SystemDescriptor:
        return self._desc

    @property
    def handle(self):
        return self._h

    def evaluate(self, s) -> np.ndarray:
        return self.evaluate_batch([s])[0]

    def evaluate_batch(self, s) -> np.ndarray:
        s = _cz(np.atleast_1d(s))
        out = np.zeros((len(s), self._desc.channel_count), np.complex128)
        _check(lib().fds_bem_evaluate_batch(self._h, _p(s), len(s), _p(out)))
        return out

    def evaluate_batch_device(self, s):
        """Device-resident result; returns the raw device pointer (bench use)."""
        s = _cz(np.atleast_1d(s))
        ptr = ctypes.c_void_p()
        _check(lib().fds_bem_evaluate_batch_device(self._h, _p(s), len(s), ctypes.byref(ptr)))
        return ptr.value

    def assemble(self, s):
        n = self.unknowns
        A = np.zeros((n, n), np.complex128, order="F")
        b = np.zeros(n, np.complex128)
        _check(lib().fds_bem_assemble_host(self._h, _C64(float(np.real(s)), float(np.imag(s))), _p(A), _p(b)))
        return A, b

    def assemble_entries(self, s, rows, cols, with_rhs=False):
        """A(s)[rows[i], cols[i]] assembled on the device (and b(s) if with_rhs)."""
        r = np.ascontiguousarray(rows, np.int32)
        c = np.ascontiguousarray(cols, np.int32)
        out = np.zeros(len(r), np.complex128)
        b = np.zeros(self.unknowns, np.complex128) if with_rhs else None
        _check(lib().fds_bem_assemble_entries(self._h, _C64(float(np.real(s)), float(np.imag(s))), len(r), _p(r),
                                              _p(c), _p(out), _p(b)))
        return (out, b) if with_rhs else out

    def residual(self, s, u):
        """Device backward-error norms of a full solution u: dict(res, a_inf, u, b)."""
        u = _cz(u)
        if u.shape != (self.unknowns,):
            raise ValidationError("residual: u must hold every unknown")
        nr = np.zeros(4)
        _check(lib().fds_bem_residual(self._h, _C64(float(np.real(s)), float(np.imag(s))), _p(u), _p(nr)))
        return dict(res=nr[0], a_inf=nr[1], u=nr[2], b=nr[3])

    def last_timing(self):
        a, l_, s, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        _check(lib().fds_bem_last_timing(self._h, ctypes.byref(a), ctypes.byref(l_), ctypes.byref(s),
                                         ctypes.byref(n)))
        return dict(assembly_ms=a.value, lu_ms=l_.value, solve_ms=s.value, launches=n.value)

    def cumulative_timing(self, reset=False):
        """Stage times summed over every solve since create / the last reset."""
        out = np.zeros(4)
        _check(lib().fds_bem_cumulative_timing(self._h, _p(out), int(bool(reset))))
        return dict(assembly_ms=out[0], lu_ms=out[1], solve_ms=out[2], frequencies=int(out[3]))

    def set_solver(self, kind: str = "lu", tol: float = 1e-12, restart: int = 60, max_iter: int = 1000):
        """'lu' (batched LU, default) or 'gmres' (restarted GMRES, all frequencies
        in lockstep, right block-Jacobi, stop at ||b - A u|| <= tol ||b||; a
        frequency that misses tol within max_iter is solved by LU instead)."""
        k = {"lu": 0, "gmres": 1}[kind]
        _check(lib().fds_bem_set_solver(self._h, k, ctypes.c_double(tol), int(restart), int(max_iter)))

    def last_gmres(self):
        it, res, fb = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        _check(lib().fds_bem_last_gmres(self._h, ctypes.byref(it), ctypes.byref(res), ctypes.byref(fb)))
        return dict(iterations=it.value, rel_residual=res.value, lu_fallbacks=fb.value)

    def close(self):
        if getattr(self, "_h", None):
            lib().fds_bem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- vector fitting
@dataclass
class RationalModel:
    """vecfit.hpp:21-30: poles (M,), residues (K, M), channel_labels."""

    poles: np.ndarray
    residues: np.ndarray
    channel_labels: list = field(default_factory=list)

    def order(self):
        return len(self.poles)

    def channel_count(self):
        return self.residues.shape[0]


def relocate_poles(s, values, poles):
    """vecfit.cpp:188-354 -> (new_poles, per_channel_rms, movement)"""
    s, v, p = _cz(s), _cz(values), _cz(poles)
    J, K = v.shape
    out = np.zeros(len(p), np.complex128)
    rms = np.zeros(K)
    mv = ctypes.c_double()
    _check(lib().fds_vf_relocate(J, K, _p(s), _p(v), len(p), _p(p), _p(out), _p(rms), ctypes.byref(mv)))
    return out, rms, mv.value


def identify_residues(s, values, poles):
    """vecfit.cpp:356-408 for every column of values (J, K) -> (residues (K, M), rms (K,))"""
    s, p = _cz(s), _cz(poles)
    v = _cz(values)
    if v.ndim == 1:
        v = v[:, None]
    J, K = v.shape
    res = np.zeros((K, len(p)), np.complex128)
    rms = np.zeros(K)
    _check(lib().fds_vf_identify_residues(J, K, _p(s), _p(v), len(p), _p(p), _p(res), _p(rms)))
    return res, rms


def vector_fit(s, values, orf, order, n_relocations=3, channel_labels=None):
    """vecfit.cpp:410-488 -> (RationalModel, report dict)"""
    s, v = _cz(s), _cz(values)
    J, K = v.shape
    orf = np.ascontiguousarray(orf, np.int32)
    poles = np.zeros(order, np.complex128)
    res = np.zeros((K, order), np.complex128)
    ri = np.zeros(2, np.int32)
    rd = np.zeros(1)
    rms = np.zeros(K)
    rrms = np.zeros(max(len(orf), 1))
    _check(lib().fds_vector_fit(J, K, _p(s), _p(v), len(orf), _p(orf), int(order), int(n_relocations),
                                _p(poles), _p(res), _p(ri), _p(rd), _p(rms), _p(rrms)))
    labels = list(channel_labels) if channel_labels else [f"ch{k}" for k in range(K)]
    rep = dict(iterations=int(ri[0]), unstable=int(ri[1]), movement=float(rd[0]), rms=rms,
               reloc_rms=rrms[: len(orf)])
    return RationalModel(poles, res, labels), rep


def eval_model(model: RationalModel, s):
    s = _cz(np.atleast_1d(s))
    p, r = _cz(model.poles), _cz(model.residues)
    out = np.zeros((len(s), r.shape[0]), np.complex128)
    _check(lib().fds_eval_model(len(p), _p(p), r.shape[0], _p(r), len(s), _p(s), _p(out)))
    return out


def fit_error_evf(model: RationalModel, channel, s, values):
    """vecfit.cpp:511-526 on the device: E_vf of one channel; values (J, K)."""
    p, r = _cz(model.poles), _cz(np.atleast_2d(model.residues))
    s, v = _cz(np.atleast_1d(s)), _cz(np.atleast_2d(values))
    out = ctypes.c_double()
    _check(lib().fds_fit_error_evf(len(p), _p(p), r.shape[0], _p(r), int(channel), len(s), _p(s), _p(v),
                                   ctypes.byref(out)))
    return out.value


def channel_errors(high: RationalModel, low: RationalModel, grid):
    g = _cz(grid)
    ph, rh, pl, rl = _cz(high.poles), _cz(high.residues), _cz(low.poles), _cz(low.residues)
    out = np.zeros(rh.shape[0])
    _check(lib().fds_channel_errors(len(ph), _p(ph), _p(rh), len(pl), _p(pl), _p(rl), rh.shape[0], len(g),
                                    _p(g), _p(out)))
    return out


def select_new_frequency(high: RationalModel, low: RationalModel, grid, existing, orf_positions, radius):
    g, ex = _cz(grid), _cz(existing)
    op = np.ascontiguousarray(orf_positions, np.int32)
    ph, rh, pl, rl = _cz(high.poles), _cz(high.residues), _cz(low.poles), _cz(low.residues)
    out = np.zeros(1, np.complex128)
    _check(lib().fds_select_new_frequency(len(ph), _p(ph), _p(rh), len(pl), _p(pl), _p(rl), rh.shape[0], len(g),
                                          _p(g), len(ex), _p(ex), len(op), _p(op), ctypes.c_double(radius),
                                          _p(out)))
    return complex(out[0])


# ---------------------------------------------------------------- laplace
def fsm_invert(period, Ns, eta, half_spectra, hanning=True):
    """laplace.cpp:89-125: half (K, Ns/2+1) -> (K, Ns)"""
    h = _cz(np.atleast_2d(half_spectra))
    out = np.zeros((h.shape[0], Ns))
    _check(lib().fds_fsm_invert(ctypes.c_double(period), int(Ns), ctypes.c_double(eta), h.shape[0], _p(h),
                                int(bool(hanning)), _p(out)))
    return out


def rational_invert(model: RationalModel, t):
    """laplace.cpp:127-164 -> (K, T)"""
    t = np.ascontiguousarray(t, np.float64)
    p, r = _cz(model.poles), _cz(np.atleast_2d(model.residues))
    out = np.zeros((r.shape[0], len(t)))
    _check(lib().fds_rational_invert(len(p), _p(p), r.shape[0], _p(r), len(t), _p(t), _p(out)))
    return out


# ---------------------------------------------------------------- AFS
def _afs_cfg(cfg: dict, keep: list):
    orf = np.ascontiguousarray(cfg.get("orf_indices", []), np.int32)
    test = np.ascontiguousarray(cfg.get("test_indices", []), np.int32)
    keep += [orf, test]
    return AfsConfigC(int(cfg.get("initial_count", 16)), float(cfg.get("alpha_high", 2.0)),
                      float(cfg.get("alpha_low", 2.3)), float(cfg.get("e1_threshold", 1e-4)),
                      float(cfg.get("e2_threshold", 2e-3)), int(cfg.get("validation_steps", 3)), len(orf),
                      _p(orf) if len(orf) else None, len(test), _p(test) if len(test) else None,
                      float(cfg["omega_max"]), float(cfg["eta"]), float(cfg["period"]),
                      int(cfg.get("grid_points", 4096)), int(cfg.get("time_points", 512)),
                      int(cfg.get("max_iterations", 500)), int(cfg.get("seed", 0)),
                      int(cfg.get("n_relocations", 3)))


def run_afs(system, cap=1024, **cfg):
    """afs.cpp:226-396. ``system`` is a BemSystem or any object with
    ``descriptor().channel_count`` and ``evaluate(s)`` (called back from C++)."""
    keep = []
    c = _afs_cfg(cfg, keep)
    K = system.descriptor().channel_count
    ss = np.zeros(cap, np.complex128)
    vals = np.zeros((cap, K), np.complex128)
    hist = np.zeros((cap, 8))
    poles = np.zeros(cap, np.complex128)
    res = np.zeros(K * cap, np.complex128)
    summ = AfsSummaryC()

    def partial():
        n = summ.n_c
        return dict(samples=ss[:n].copy(), values=vals[:n].copy(), n_c=n, solver_calls=summ.solver_calls,
                    history=hist[: summ.n_history].copy(), orf=list(summ.orf_indices[: min(summ.n_orf, 8)]))

    def check(rc):
        try:
            _check(rc)
        except Error as e:  # the iterations completed before the reference algorithm failed
            e.partial = partial()
            raise

    if isinstance(system, BemSystem):
        check(lib().fds_run_afs_bem(system.handle, ctypes.byref(c), cap, _p(ss), _p(vals), _p(hist), _p(poles),
                                     _p(res), ctypes.byref(summ)))
    else:
        err = []

        def cb(user, s, out):
            try:
                v = np.asarray(system.evaluate(complex(s.re, s.im)), np.complex128)
                ctypes.memmove(out, v.ctypes.data, v.nbytes)
                return 0
            except Exception as e:  # pragma: no cover - propagated below
                err.append(e)
                return 1

        fn = SYSTEM_FN(cb)
        rc = lib().fds_run_afs_callback(fn, None, K, ctypes.byref(c), cap, _p(ss), _p(vals), _p(hist), _p(poles),
                                        _p(res), ctypes.byref(summ))
        if err:
            raise err[0]
        check(rc)
    n, M = summ.n_c, summ.order
    return dict(samples=ss[:n].copy(), values=vals[:n].copy(), n_c=n, converged=bool(summ.converged),
                solver_calls=summ.solver_calls, history=hist[: summ.n_history].copy(), poles=poles[:M].copy(),
                residues=res[: K * M].reshape(K, M).copy(), orf=list(summ.orf_indices[: min(summ.n_orf, 8)]))


def damping_eta(kappa, period):
    """laplace.cpp:62-65 (host arithmetic)."""
    if not period > 0:
        raise ValidationError("damping_eta: period must be positive")
    return kappa * math.log(10.0) / period
