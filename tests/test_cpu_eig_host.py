"""CPU test of the product's host eigenvalue step (relocate_poles' companion
matrix, vecfit.cpp:324; paper_1511_04355_b200/csrc/eig_host.cpp) against LAPACK
dgeev (numpy), without a GPU: the translation unit is compiled on its own with
g++ into a temporary shared object. It must find every eigenvalue to ~1e-13 of
||H||, return real eigenvalues with an exactly zero imaginary part and complex
ones as adjacent exact conjugate pairs (+Im first) — the properties the pole
split of vecfit.cpp:328-350 relies on."""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_1511_04355_b200" / "csrc"

WRAP = r'''
#include "eig_host.h"
extern "C" int eig_host_eigenvalues(int n, const double* a, double* out) {
    std::vector<std::complex<double>> ev;
    if (!fdsb::eig::eigenvalues(n, a, ev)) return 1;
    for (int i = 0; i < n; ++i) { out[2 * i] = ev[i].real(); out[2 * i + 1] = ev[i].imag(); }
    return 0;
}
'''


@pytest.fixture(scope="module")
def eig(tmp_path_factory):
    d = tmp_path_factory.mktemp("eig")
    (d / "wrap.cpp").write_text(WRAP)
    so = d / "libeig.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-I{CSRC}", str(d / "wrap.cpp"),
                    str(CSRC / "eig_host.cpp"), "-o", str(so)], check=True)
    lib = ctypes.CDLL(str(so))

    def run(H):
        Hf = np.asfortranarray(H, np.float64)
        n = Hf.shape[0]
        out = np.zeros(2 * n)
        rc = lib.eig_host_eigenvalues(n, Hf.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        return out[0::2] + 1j * out[1::2]

    return run


def _companion(rng, n):
    """blockdiag(poles) - b c^T as relocate_poles builds it (vecfit.cpp:297-324)."""
    H = np.zeros((n, n))
    bv = np.zeros(n)
    m = 0
    while m < n:
        if m + 1 < n and rng.random() < 0.8:
            a = -rng.random() + 1j * 40 * rng.random()
            H[m:m + 2, m:m + 2] = [[a.real, a.imag], [-a.imag, a.real]]
            bv[m] = 2.0
            m += 2
        else:
            H[m, m] = -rng.random()
            bv[m] = 1.0
            m += 1
    return H - np.outer(bv, rng.normal(size=n))


@pytest.mark.parametrize("kind", ["random", "companion", "graded", "symmetric"])
def test_host_eigenvalues_match_lapack(eig, kind):
    rng = np.random.default_rng({"random": 1, "companion": 2, "graded": 3, "symmetric": 4}[kind])
    for _ in range(150):
        n = int(rng.integers(1, 72))
        if kind == "random":
            H = rng.normal(size=(n, n))
        elif kind == "companion":
            H = _companion(rng, n)
        elif kind == "graded":
            H = np.triu(rng.normal(size=(n, n)), -1) * np.logspace(0, -8, n)[None, :]
        else:
            H = rng.normal(size=(n, n))
            H = H + H.T
        ev = eig(H)
        lap = np.linalg.eigvals(H)
        sc = max(np.linalg.norm(H, 2), 1e-300)
        for w in lap:
            assert np.min(np.abs(ev - w)) <= 1e-12 * sc
        if kind == "symmetric":
            assert np.all(ev.imag == 0.0)
        assert np.sum(ev.imag > 0) == np.sum(ev.imag < 0)
        i = 0
        while i < n:  # conjugate pairs adjacent, +Im first, exactly conjugate
            if ev[i].imag != 0.0:
                assert ev[i].imag > 0 and ev[i + 1] == np.conj(ev[i])
                i += 2
            else:
                i += 1


def test_host_eigenvalues_exact_real_split(eig):
    """Exactly real spectra (upper triangular, diagonal, 1x1) come back with
    zero imaginary parts and the diagonal values unchanged."""
    rng = np.random.default_rng(9)
    for n in (1, 2, 5, 30):
        d = -rng.random(n) * 10
        H = np.diag(d) + np.triu(rng.normal(size=(n, n)), 1)
        ev = eig(H)
        assert np.all(ev.imag == 0.0)
        np.testing.assert_allclose(np.sort(ev.real), np.sort(d), rtol=1e-12)
