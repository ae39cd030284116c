"""ORACLE — test infrastructure only.

ctypes binding of ``oracle/_ref/libfdsweep_oracle.so`` (the CPU checker: the
reference's own afs.cpp/systems.cpp/io.cpp + the restated vecfit/laplace + the
new BEM oracle). Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module; the
product package never does.

Complex arrays cross the boundary as interleaved float64 pairs, exactly the
layout of ``std::complex<double>`` (proj/include/fdsweep/types.hpp:10).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libfdsweep_oracle.so"

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double


class OracleError(RuntimeError):
    """Carries the reference error class name (types.hpp:14-36)."""

    CLASSES = {1: "ValidationError", 2: "NumericError", 3: "IoError", 4: "ConvergenceError", 9: "Error"}

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = self.CLASSES.get(code, "Error")
        super().__init__(f"{self.kind}: {msg}")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` (or __graft_entry__.build())")
        _lib = ctypes.CDLL(str(LIB_PATH))
        _lib.orc_last_error.restype = ctypes.c_char_p
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


def _c(a):
    """complex array -> contiguous interleaved float64 view"""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def call(name, *args):
    f = getattr(lib(), name)
    conv = []
    for a in args:
        if isinstance(a, np.ndarray):
            conv.append(_ptr(a))
        elif isinstance(a, float):
            conv.append(_D(a))
        elif isinstance(a, bool):
            conv.append(_I(int(a)))
        elif isinstance(a, int):
            conv.append(_I(a))
        elif isinstance(a, bytes):
            conv.append(ctypes.c_char_p(a))
        else:
            conv.append(a)
    _check(f(*conv))


# ----------------------------------------------------------------- vecfit
def initial_poles(omega_max, order):
    out = np.zeros(order, np.complex128)
    call("orc_initial_poles", float(omega_max), int(order), out)
    return out


def is_conjugate_closed(poles, tol=1e-9):
    p = _c(poles)
    out = np.zeros(1, np.int32)
    call("orc_is_conjugate_closed", len(p), p, float(tol), out)
    return bool(out[0])


def canonical_poles(poles):
    p = _c(poles)
    out = np.zeros_like(p)
    call("orc_canonical_poles", len(p), p, out)
    return out


def relocate_poles(s, vals, poles):
    """s: (J,), vals: (J, K), poles: (M,) -> (new_poles, per_channel_rms, movement)"""
    s, vals, poles = _c(s), _c(vals), _c(poles)
    J, K = vals.shape
    out = np.zeros(len(poles), np.complex128)
    rms = np.zeros(K)
    mv = np.zeros(1)
    call("orc_relocate_poles", J, K, s, vals, len(poles), poles, out, rms, mv)
    return out, rms, float(mv[0])


def last_relocation():
    """Stacked sigma system (rows x M), its rhs and the companion matrix H (or None)
    of the last relocate_poles call (oracle test hook, vecfit.cpp:281,324)."""
    r, c, hh = (np.zeros(1, np.int32) for _ in range(3))
    call("orc_last_relocation_dims", r, c, hh)
    rows, M = int(r[0]), int(c[0])
    A = np.zeros((rows, M), order="F")
    b = np.zeros(rows)
    H = np.zeros((M, M), order="F")
    call("orc_last_relocation", A, b, H)
    return A, b, (H if hh[0] else None)


def colpivqr(A, b=None):
    """The oracle's ColPivHouseholderQR: dict(rdiag, perm, rank, nonzero_pivots, maxpivot, x)."""
    A = np.asfortranarray(A, np.float64)
    m, n = A.shape
    bb = np.zeros(m) if b is None else np.ascontiguousarray(b, np.float64)
    rd = np.zeros(min(m, n))
    perm = np.zeros(n, np.int32)
    rank, npv = np.zeros(1, np.int32), np.zeros(1, np.int32)
    mp = np.zeros(1)
    x = np.zeros(n)
    call("orc_colpivqr", m, n, A, bb, rd, perm, rank, npv, mp, x)
    return dict(rdiag=rd, perm=perm, rank=int(rank[0]), nonzero_pivots=int(npv[0]), maxpivot=float(mp[0]), x=x)


def real_eigenvalues(H):
    H = np.asfortranarray(H, np.float64)
    ev = np.zeros(H.shape[0], np.complex128)
    call("orc_real_eigenvalues", H.shape[0], H, ev)
    return ev


def identify_residues(s, vals, poles):
    s, vals, poles = _c(s), _c(vals), _c(poles)
    out = np.zeros(len(poles), np.complex128)
    rms = np.zeros(1)
    call("orc_identify_residues", len(s), s, vals, len(poles), poles, out, rms)
    return out, float(rms[0])


def identify_residues_many(s, vals, poles, threads=1):
    """identify_residues per channel (vals (J, K)) on `threads` OpenMP threads -> (K, M)."""
    s, vals, poles = _c(s), _c(vals), _c(poles)
    J, K = vals.shape
    out = np.zeros((K, len(poles)), np.complex128)
    call("orc_identify_residues_many", J, K, s, vals, len(poles), poles, int(threads), out)
    return out


def vector_fit(s, vals, orf, order, n_reloc=3):
    """Returns dict(poles, residues (K, M), iterations, movement, unstable, rms, reloc_rms)."""
    s, vals = _c(s), _c(vals)
    J, K = vals.shape
    orf = np.ascontiguousarray(orf, dtype=np.int32)
    poles = np.zeros(order, np.complex128)
    res = np.zeros((K, order), np.complex128)
    it = np.zeros(1, np.int32)
    mv = np.zeros(1)
    un = np.zeros(1, np.int32)
    rms = np.zeros(K)
    rrms = np.zeros(len(orf))
    call("orc_vector_fit", J, K, s, vals, len(orf), orf, int(order), int(n_reloc), poles, res, it, mv, un, rms, rrms)
    return dict(poles=poles, residues=res, iterations=int(it[0]), movement=float(mv[0]),
                unstable=int(un[0]), rms=rms, reloc_rms=rrms)


def eval_model(poles, residues, s):
    poles, residues = _c(poles), _c(np.atleast_2d(residues))
    out = np.zeros(residues.shape[0], np.complex128)
    call("orc_eval_model", len(poles), poles, residues.shape[0], residues, float(np.real(s)), float(np.imag(s)), out)
    return out


def fit_error_evf(poles, residues, ch, s, vals):
    poles, residues, s, vals = _c(poles), _c(np.atleast_2d(residues)), _c(s), _c(vals)
    out = np.zeros(1)
    call("orc_fit_error_evf", len(poles), poles, residues.shape[0], residues, int(ch), len(s), s, vals, out)
    return float(out[0])


# ----------------------------------------------------------------- laplace
def damping_eta(kappa, T):
    out = np.zeros(1)
    call("orc_damping_eta", float(kappa), float(T), out)
    return float(out[0])


def hanning_window(k, ns):
    out = np.zeros(1)
    call("orc_hanning_window", int(k), int(ns), out)
    return float(out[0])


def conjugate_fill(half):
    h = _c(half)
    out = np.zeros(2 * (len(h) - 1), np.complex128)
    call("orc_conjugate_fill", len(h), h, out)
    return out


def fsm_grid(T, ns):
    dw, dt, wm = np.zeros(1), np.zeros(1), np.zeros(1)
    nc = np.zeros(1, np.int32)
    call("orc_fsm_grid", float(T), int(ns), dw, dt, wm, nc)
    return float(dw[0]), float(dt[0]), float(wm[0]), int(nc[0])


def fsm_invert(T, ns, eta, half, hanning=True):
    """half: (K, Ns/2+1) -> (K, Ns)"""
    half = _c(np.atleast_2d(half))
    out = np.zeros((half.shape[0], ns))
    call("orc_fsm_invert", float(T), int(ns), float(eta), half.shape[0], half, bool(hanning), out)
    return out


def rational_invert(poles, residues, t):
    poles, residues = _c(poles), _c(np.atleast_2d(residues))
    t = np.ascontiguousarray(t, dtype=np.float64)
    out = np.zeros((residues.shape[0], len(t)))
    call("orc_rational_invert", len(poles), poles, residues.shape[0], residues, len(t), t, out)
    return out


# ----------------------------------------------------------------- afs
def initial_frequencies(j0, eta, omega_max):
    out = np.zeros(j0, np.complex128)
    call("orc_initial_frequencies", int(j0), float(eta), float(omega_max), out)
    return out


def fit_orders(J, ah=2.0, al=2.3):
    mh, ml = np.zeros(1, np.int32), np.zeros(1, np.int32)
    call("orc_fit_orders", int(J), float(ah), float(al), mh, ml)
    return int(mh[0]), int(ml[0])


def channel_errors(ph, rh, pl, rl, grid):
    ph, rh, pl, rl, grid = _c(ph), _c(np.atleast_2d(rh)), _c(pl), _c(np.atleast_2d(rl)), _c(grid)
    out = np.zeros(rh.shape[0])
    call("orc_channel_errors", len(ph), ph, len(pl), pl, rh.shape[0], rh, rl, len(grid), grid, out)
    return out


def select_new_frequency(ph, rh, pl, rl, grid, existing, orf_pos, radius):
    ph, rh, pl, rl, grid, ex = _c(ph), _c(np.atleast_2d(rh)), _c(pl), _c(np.atleast_2d(rl)), _c(grid), _c(existing)
    op = np.ascontiguousarray(orf_pos, dtype=np.int32)
    out = np.zeros(1, np.complex128)
    call("orc_select_new_frequency", len(ph), ph, len(pl), pl, rh.shape[0], rh, rl, len(grid), grid,
         len(ex), ex, len(op), op, float(radius), out)
    return complex(out[0])


def error_e1(t, cur, prev):
    t = np.ascontiguousarray(t, np.float64)
    cur, prev = np.ascontiguousarray(cur, np.float64), np.ascontiguousarray(prev, np.float64)
    out = np.zeros(1)
    call("orc_error_e1", cur.shape[0], len(t), t, cur, prev, out)
    return float(out[0])


class System:
    """A reference FrequencySystem (systems.cpp factory) or the BEM oracle system."""

    def __init__(self, handle):
        self.h = ctypes.c_void_p(handle)

    @classmethod
    def from_json(cls, text: str):
        h = ctypes.c_void_p()
        call("orc_system_from_json", text.encode(), ctypes.byref(h))
        return cls(h.value)

    @classmethod
    def bem(cls, bem: "Bem", dofs):
        d = np.ascontiguousarray(dofs, np.int32)
        h = ctypes.c_void_p()
        call("orc_system_bem", bem.h, len(d), d, ctypes.byref(h))
        s = cls(h.value)
        s._keep = bem
        return s

    @classmethod
    def callback(cls, channels, fn):
        """A system whose evaluate(s) returns fn(s) (a length-`channels` complex
        vector): lets the reference run_afs run on responses computed elsewhere."""
        proto = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                 ctypes.POINTER(ctypes.c_double))

        def tramp(_ctx, sr, si, out):
            try:
                v = np.ascontiguousarray(fn(complex(sr, si)), np.complex128)
                ctypes.memmove(out, v.ctypes.data, 16 * channels)
                return 0
            except Exception:  # noqa: BLE001 - reported as a NumericError by the oracle
                return 1

        cb = proto(tramp)
        h = ctypes.c_void_p()
        call("orc_system_callback", int(channels), cb, None, ctypes.byref(h))
        s = cls(h.value)
        s._keep = cb
        return s

    @property
    def channels(self):
        return lib().orc_system_channels(self.h)

    def evaluate(self, s):
        out = np.zeros(self.channels, np.complex128)
        call("orc_system_evaluate", self.h, float(np.real(s)), float(np.imag(s)), out)
        return out

    def __del__(self):
        try:
            lib().orc_system_destroy(self.h)
        except Exception:
            pass


def run_afs(system: System, *, omega_max, eta, period, orf=(), test=(), initial_count=16,
            alpha_high=2.0, alpha_low=2.3, e1_threshold=1e-4, e2_threshold=2e-3,
            validation_steps=3, grid_points=4096, time_points=512, max_iterations=500, seed=0,
            n_relocations=3, cap=1024):
    """Runs the REFERENCE run_afs (proj/src/afs.cpp:226-396) on the oracle VF."""
    cd = np.array([alpha_high, alpha_low, e1_threshold, e2_threshold, omega_max, eta, period], np.float64)
    ci = np.array([initial_count, validation_steps, grid_points, time_points, max_iterations, seed,
                   n_relocations], np.int32)
    orf = np.ascontiguousarray(orf, np.int32)
    test = np.ascontiguousarray(test, np.int32)
    ss = np.zeros(cap, np.complex128)
    nc, conv, calls, nh, order, norf = (np.zeros(1, np.int32) for _ in range(6))
    hist = np.zeros((cap, 8))
    poles = np.zeros(cap, np.complex128)
    orf_used = np.zeros(max(system.channels, 8), np.int32)
    res = np.zeros((system.channels, cap), np.complex128)
    try:
        call("orc_run_afs", system.h, cd, ci, len(orf), orf, len(test), test, cap, ss, nc, conv, calls, hist,
             nh, poles, order, orf_used, norf, res)
    except OracleError as e:  # samples solved before the reference threw (on_sample, afs.cpp:296)
        e.partial = dict(samples=ss[: int(nc[0])].copy(), n_c=int(nc[0]), solver_calls=int(calls[0]))
        raise
    n = int(nc[0])
    M = int(order[0])
    resid = np.ascontiguousarray(res.reshape(-1)[: system.channels * M].reshape(system.channels, M))
    return dict(samples=ss[:n].copy(), n_c=n, converged=bool(conv[0]), solver_calls=int(calls[0]),
                history=hist[: int(nh[0])].copy(), poles=poles[:M].copy(), residues=resid,
                orf=orf_used[: int(norf[0])].copy())


# ----------------------------------------------------------------- BEM
class Bem:
    def __init__(self, vertices, triangles, traction, mu=1.0, nu=0.25, rho=1.0):
        v = np.ascontiguousarray(vertices, np.float64)
        t = np.ascontiguousarray(triangles, np.int32)
        tr = np.ascontiguousarray(traction, np.float64)
        h = ctypes.c_void_p()
        call("orc_bem_create", v.shape[0], v, t.shape[0], t, float(mu), float(nu), float(rho), tr, ctypes.byref(h))
        self.h = h
        self.n = 3 * t.shape[0]

    def assemble(self, s):
        A = np.zeros((self.n, self.n), np.complex128, order="F")
        b = np.zeros(self.n, np.complex128)
        call("orc_bem_assemble", self.h, float(np.real(s)), float(np.imag(s)), A, b)
        return A, b

    def solve(self, s):
        u = np.zeros(self.n, np.complex128)
        call("orc_bem_solve", self.h, float(np.real(s)), float(np.imag(s)), u)
        return u

    def solve_openblas(self, s, openblas_path):
        u = np.zeros(self.n, np.complex128)
        t = np.zeros(2)
        call("orc_bem_solve_openblas", self.h, str(openblas_path).encode(), float(np.real(s)), float(np.imag(s)), u, t)
        return u, t

    def entries(self, s, rows, cols):
        """A(s)[rows[i], cols[i]] (same arithmetic as assemble; full-size spot checks)."""
        r = np.ascontiguousarray(rows, np.int32)
        c = np.ascontiguousarray(cols, np.int32)
        out = np.zeros(len(r), np.complex128)
        call("orc_bem_entries", self.h, float(np.real(s)), float(np.imag(s)), len(r), r, c, out)
        return out

    def rhs_rows(self, s, rows):
        r = np.ascontiguousarray(rows, np.int32)
        out = np.zeros(len(r), np.complex128)
        call("orc_bem_rhs_rows", self.h, float(np.real(s)), float(np.imag(s)), len(r), r, out)
        return out

    def self_block(self, e, s):
        U = np.zeros(9, np.complex128)
        T = np.zeros(9, np.complex128)
        call("orc_bem_self_block", self.h, int(e), float(np.real(s)), float(np.imag(s)), U, T)
        return U.reshape(3, 3), T.reshape(3, 3)

    def __del__(self):
        try:
            lib().orc_bem_destroy(self.h)
        except Exception:
            pass


def kernel_ut(rv, n, s, mu=1.0, nu=0.25, rho=1.0):
    rv = np.ascontiguousarray(rv, np.float64)
    n = np.ascontiguousarray(n, np.float64)
    U = np.zeros(9, np.complex128)
    T = np.zeros(9, np.complex128)
    call("orc_kernel_ut", float(mu), float(nu), float(rho), rv, n, float(np.real(s)), float(np.imag(s)), U, T)
    return U.reshape(3, 3), T.reshape(3, 3)


def kernel_abcd(z, mu=1.0, nu=0.25, rho=1.0):
    out = np.zeros(4, np.complex128)
    call("orc_kernel_abcd", float(mu), float(nu), float(rho), float(np.real(z)), float(np.imag(z)), out)
    return out


def lu_solve(A, b):
    A = np.asfortranarray(A, np.complex128)
    b = _c(b)
    x = np.zeros_like(b)
    call("orc_lu_solve", len(b), A, b, x)
    return x


def openblas_path():
    import glob
    import scipy

    cands = glob.glob(os.path.join(os.path.dirname(scipy.__file__), "..", "scipy.libs", "libscipy_openblas*.so"))
    return os.path.abspath(cands[0]) if cands else None
