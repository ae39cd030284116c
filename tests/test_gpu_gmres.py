"""GMRES solver path of the BEM handle: same solutions as
the LU path / CPU oracle within the solution tolerance (1e-9 rel. L2), true
residual at or below tol, bit-identical repeated solves, convergence errors."""
import math

import numpy as np
import pytest

import paper_1511_04355_b200 as P
import pyoracle as O
from paper_1511_04355_b200 import mesh

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("level,load", [(1, "pressure"), (2, "random")])
def test_gmres_matches_oracle(level, load):
    V, F = mesh.icosphere(level)
    tr = mesh.pressure_traction(V, F) if load == "pressure" else mesh.random_traction(F.shape[0], seed=1)
    s = 0.25 + 1j * 2 * math.pi / 20.0 * np.array([0, 3, 17, 60])
    g = P.BemSystem(V, F, tr)
    g.set_solver("gmres", tol=1e-13)
    u = g.evaluate_batch(s)
    st = g.last_gmres()
    assert st["rel_residual"] <= 1e-13 and st["iterations"] > 0
    orc = O.Bem(V, F, tr)
    for b, sv in enumerate(s):
        assert rel(u[b], orc.solve(sv)) < 1e-9
    assert np.array_equal(u, g.evaluate_batch(s))  # deterministic


def test_gmres_vs_lu_full_size_cfg2():
    V, F = mesh.icosphere(3)
    tr = mesh.random_traction(F.shape[0], seed=0)
    s = 0.25 + 1j * np.array([0.0, 5.0, 40.0])
    a = P.BemSystem(V, F, tr)
    ul = a.evaluate_batch(s)
    a.set_solver("gmres", tol=1e-13)
    ug = a.evaluate_batch(s)
    assert rel(ug, ul) < 1e-10


def test_gmres_stagnation_falls_back_to_lu():
    """A frequency whose GMRES misses tol within max_iter is solved by LU: the
    batch still returns the LU solution for it (to rounding: the fallback factors
    with another LU schedule)."""
    V, F = mesh.icosphere(2)
    g = P.BemSystem(V, F, mesh.pressure_traction(V, F))
    s = np.array([0.25 + 3j, 0.25 + 7j])
    ul = g.evaluate_batch(s)
    g.set_solver("gmres", tol=1e-15, restart=2, max_iter=3)
    ug = g.evaluate_batch(s)
    assert g.last_gmres()["lu_fallbacks"] == 2
    assert np.linalg.norm(ug - ul) / np.linalg.norm(ul) < 1e-13  # rounding: other LU schedule
    with pytest.raises(P.ValidationError):
        g.set_solver("gmres", tol=-1.0)
