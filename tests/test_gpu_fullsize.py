"""Parity at BASELINE.json's full sizes (configs 2, 4, 5) through the C-ABI.

Where the CPU oracle can finish in seconds it is compared directly (cfg2
frequencies, cfg5 DOF subsets); at N = 15360 the size-independent property is
the backward error of the solve against the device-assembled system.
"""
import math

import numpy as np
import pytest

import paper_1511_04355_b200 as P
import pyoracle as O
from paper_1511_04355_b200 import mesh

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_cfg2_batch_matches_oracle_on_sampled_frequencies():
    V, F = mesh.icosphere(3)
    tr = mesh.pressure_traction(V, F)
    s = 0.25 + 1j * (2 * math.pi / 20.0) * np.arange(129)
    gpu = P.BemSystem(V, F, tr)
    u = gpu.evaluate_batch(s)
    u2 = gpu.evaluate_batch(s)
    assert np.array_equal(u, u2)  # bit-identical repeated 129-frequency batch
    orc = O.Bem(V, F, tr)
    ob = O.openblas_path()
    for b in (0, 1, 64, 128):
        uo, _ = orc.solve_openblas(s[b], ob)
        assert rel_l2(u[b], uo) < 1e-9


def test_cfg4_backward_error_n15360():
    V, F = mesh.icosphere(4)
    tr = mesh.random_traction(F.shape[0], seed=0)
    gpu = P.BemSystem(V, F, tr, max_batch=1)
    s = complex(0.25, 2 * math.pi / 20.0 * 7)
    A, b = gpu.assemble(s)
    u = gpu.evaluate(s)
    r = A @ u - b
    assert np.linalg.norm(r) / (np.linalg.norm(A, ord=np.inf) * np.linalg.norm(u) + np.linalg.norm(b)) < 1e-13
    assert np.linalg.norm(r) / np.linalg.norm(b) < 1e-10


def test_cfg5_vf_and_reconstruction_subset_parity():
    rng = np.random.default_rng(0)
    D, J, pairs = 300_000, 40, 24
    heads = -(0.01 + 0.49 * rng.random(pairs)) + 1j * 40.0 * rng.random(pairs)
    poles = np.stack([heads, heads.conj()], 1).reshape(-1)
    wmax = 1.2 * heads.imag.max()
    T = math.pi * 512 / wmax
    eta = 3 * math.log(10) / T
    s = eta + 1j * wmax * (1 - np.cos(np.arange(J) * math.pi / (2 * (J - 1))))
    rh = rng.normal(size=(D, pairs)) + 1j * rng.normal(size=(D, pairs))
    res = np.stack([rh, rh.conj()], 2).reshape(D, -1)
    vals = (1.0 / (s[:, None] - poles[None, :])) @ res.T
    vals += 1e-3 * (rng.normal(size=vals.shape) + 1j * rng.normal(size=vals.shape))
    model, rep = P.vector_fit(s, vals[:, :5], [0, 1, 2, 3, 4], 48, 3)
    o = O.vector_fit(s, vals[:, :5], [0, 1, 2, 3, 4], 48, 3)
    worst = max(min(abs(g - w) / abs(w) for g in model.poles) for w in o["poles"])
    assert worst < 1e-6
    R, _ = P.identify_residues(s, vals, model.poles)  # all 300k DOFs on the GPU
    # 3000 DOFs spread over the whole set against the oracle (per-DOF rel-L2)
    sub = np.sort(rng.choice(D, 3000, replace=False))
    ro = O.identify_residues_many(s, vals[:, sub], model.poles, threads=8)
    err = np.linalg.norm(R[sub] - ro, axis=1) / np.linalg.norm(ro, axis=1)
    print(f"cfg5 residues, 3000 DOFs: max rel-L2 {err.max():.2e}")
    assert err.max() < 1e-9
    t = np.arange(512) * T / 512
    h = P.rational_invert(P.RationalModel(model.poles, R[sub]), t)
    ho = O.rational_invert(model.poles, R[sub], t)
    assert rel_l2(h, ho) < 1e-10
    sk = eta + 1j * (2 * math.pi / T) * np.arange(257)
    half = (1.0 / (sk[:, None] - poles[None, :])) @ res[sub].T  # (257, 3000)
    f = P.fsm_invert(T, 512, eta, half.T.copy())
    fo = O.fsm_invert(T, 512, eta, half.T.copy())
    assert rel_l2(f, fo) < 1e-10
