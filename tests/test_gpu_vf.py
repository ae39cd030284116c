"""GPU parity of vector fitting, dense-grid AFS kernels and time reconstruction
against the CPU oracle (restated vecfit/laplace + the reference's own afs.cpp),
through the C-ABI. Tolerances (north_star): poles within 1e-6 relative, time
responses within 1e-8 relative L2, identical AFS frequency sequence.
"""
import math

import numpy as np
import pytest

import paper_1511_04355_b200 as P
import pyoracle as O
from helpers import ModalFixture, TestRng, contour_points, rational_samples, rel_err, worst_match

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


# ------------------------------------------------ reference unit tests, product path
def test_relocation_two_pole_recovery():  # test_vecfit.cpp:57-68
    true = [complex(-1, 10), complex(-1, -10)]
    s, v = rational_samples(true, [[complex(0.5, -0.3), complex(0.5, 0.3)]], contour_points(1.0, 20.0, 12))
    poles = np.array([complex(-0.5, 50), complex(-0.5, -50)])
    for _ in range(3):
        poles, _, _ = P.relocate_poles(s, v, poles)
    assert worst_match(poles, true) < 1e-8


def test_relocation_fixed_point():  # :70-79
    true = [complex(-2, 30), complex(-2, -30), complex(-5, 0)]
    s, v = rational_samples(true, [[complex(1, 0.7), complex(1, -0.7), complex(2, 0)]], contour_points(0.5, 60.0, 16))
    rel, _, _ = P.relocate_poles(s, v, true)
    assert worst_match(rel, true) < 1e-10


def test_unstable_pole_retained():  # :81-90
    true = [complex(0.3, 0), complex(-2, 0)]
    s, v = rational_samples(true, [[1.0 + 0j, 1.0 + 0j]], contour_points(1.0, 10.0, 10))
    model, rep = P.vector_fit(s, v, [0], 2, 3)
    assert rep["unstable"] == 1 and worst_match(model.poles, true) < 1e-8


def test_residue_exact_and_zero():  # :92-111
    freqs = contour_points(1.0, 8.0, 8)
    res, rms = P.identify_residues(freqs, 1.0 / (freqs + 2.0), [complex(-2, 0)])
    assert rel_err(res[0, 0], 1.0) < 1e-10 and rms[0] < 1e-12
    res, _ = P.identify_residues(contour_points(1.0, 10.0, 6), np.zeros(6, complex), [complex(-1, 5), complex(-1, -5)])
    assert np.all(res == 0)


def test_vector_fit_shared_pole_model():  # :113-132
    poles = [complex(-1, 12), complex(-1, -12), complex(-3, 40), complex(-3, -40)]
    residues = [[complex(0.4, 0.1), complex(0.4, -0.1), complex(1.5, 0), complex(1.5, 0)],
                [complex(-0.8, 0.2), complex(-0.8, -0.2), complex(0.3, -0.9), complex(0.3, 0.9)],
                [complex(2.0, 0), complex(2.0, 0), complex(-0.5, 0.25), complex(-0.5, -0.25)]]
    s, v = rational_samples(poles, residues, contour_points(0.8, 60.0, 14))
    model, rep = P.vector_fit(s, v, [0], 4, 3)
    assert np.all(rep["rms"] < 1e-8) and worst_match(model.poles, poles) < 1e-7


def test_vector_fit_modal_fixture():  # :146-156
    fx = ModalFixture(6)
    s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 48))
    model, rep = P.vector_fit(s, v, [0, 1, 2], 16, 3)
    assert rep["iterations"] <= 3 and rep["movement"] < 1e-6
    assert worst_match(model.poles, fx.poles) < 1e-6


def test_property_random_models():  # :198-231
    band = 100.0
    rng = TestRng(7)
    for _ in range(10):
        order = 2 * (1 + rng.next() % 5)
        poles = []
        while len(poles) < order:
            c = complex(-rng.uniform(0.5, band / 10.0), rng.uniform(band / 50.0, band))
            if any(abs(p - c) < band / 50.0 or abs(p - c.conjugate()) < band / 50.0 for p in poles):
                continue
            poles += [c, c.conjugate()]
        res = [[]]
        for _m in range(0, order, 2):
            r = complex(rng.uniform(0.5, 2.0), rng.uniform(-1.0, 1.0))
            res[0] += [r, r.conjugate()]
        s, v = rational_samples(poles, res, contour_points(band / 100.0, band, 2 * order + 4))
        model, _ = P.vector_fit(s, v, [0], order, 5)
        assert worst_match(model.poles, poles) < 1e-7


def test_validation_errors():  # :263-288
    poles = [complex(-1, 2), complex(-1, -2)]
    s, v = rational_samples(poles, [[1.0 + 0j, 1.0 + 0j]], contour_points(1.0, 10.0, 6))
    with pytest.raises(P.ValidationError):
        P.vector_fit(np.append(s, s[0]), np.vstack([v, v[:1]]), [0], 2, 3)
    with pytest.raises(P.ValidationError):
        P.vector_fit(s, v, [0], 12, 3)
    with pytest.raises(P.ValidationError):
        P.identify_residues(contour_points(1.0, 10.0, 6), np.ones(6, complex), [complex(-1, 2)])
    with pytest.raises(P.NumericError):
        P.relocate_poles(s, np.zeros_like(v), poles)


# ------------------------------------------------ oracle parity
def _noisy_modal(K, J, seed=3, noise=1e-3):
    fx = ModalFixture(K)
    s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, J))
    rng = np.random.default_rng(seed)
    return s, v + noise * (rng.normal(size=v.shape) + 1j * rng.normal(size=v.shape))


def test_vector_fit_parity_noisy():
    s, v = _noisy_modal(12, 40)
    for order in (10, 16, 20):
        model, rep = P.vector_fit(s, v, [0, 3, 5], order, 3)
        o = O.vector_fit(s, v, [0, 3, 5], order, 3)
        assert worst_match(model.poles, o["poles"]) < 1e-6
        assert rep["iterations"] == o["iterations"]
        # residues in canonical order: match each oracle pole's residue column
        for m, p in enumerate(o["poles"]):
            mm = int(np.argmin(np.abs(model.poles - p)))
            assert rel_l2(model.residues[:, mm], o["residues"][:, m]) < 1e-6
        np.testing.assert_allclose(rep["rms"], o["rms"], rtol=1e-6)


def test_identify_residues_batched_parity():
    s, v = _noisy_modal(300, 40)
    o = O.vector_fit(s, v, [0, 1], 16, 3)
    res, rms = P.identify_residues(s, v, o["poles"])
    for k in range(0, 300, 37):
        ro, rmso = O.identify_residues(s, v[:, k], o["poles"])
        assert rel_l2(res[k], ro) < 1e-10
        assert rms[k] == pytest.approx(rmso, rel=1e-8)


def _two_fits():
    s, v = _noisy_modal(8, 36)
    oh = O.vector_fit(s, v, [0, 1], 18, 3)
    ol = O.vector_fit(s, v, [0, 1], 15, 3)
    return s, v, oh, ol


def test_channel_errors_parity():
    s, v, oh, ol = _two_fits()
    grid = contour_points(0.35, 1.5 * 29.8, 4096)
    mh = P.RationalModel(oh["poles"], oh["residues"])
    ml = P.RationalModel(ol["poles"], ol["residues"])
    e = P.channel_errors(mh, ml, grid)
    eo = O.channel_errors(oh["poles"], oh["residues"], ol["poles"], ol["residues"], grid)
    np.testing.assert_allclose(e, eo, rtol=1e-12)


def test_select_new_frequency_parity():
    s, v, oh, ol = _two_fits()
    grid = contour_points(0.35, 1.5 * 29.8, 4096)
    mh = P.RationalModel(oh["poles"], oh["residues"])
    ml = P.RationalModel(ol["poles"], ol["residues"])
    radius = 1.5 * 29.8 / (4 * 4096)
    for orf in ([0, 1], [2, 5, 7]):
        a = P.select_new_frequency(mh, ml, grid, s, orf, radius)
        b = O.select_new_frequency(oh["poles"], oh["residues"], ol["poles"], ol["residues"], grid, s, orf, radius)
        assert a == b


def test_rational_invert_parity():
    s, v, oh, _ = _two_fits()
    t = np.linspace(0.0, 20.0, 512)
    h = P.rational_invert(P.RationalModel(oh["poles"], oh["residues"]), t)
    ho = O.rational_invert(oh["poles"], oh["residues"], t)
    assert rel_l2(h, ho) < 1e-12


def test_rational_invert_unpaired_and_errors():
    poles = [complex(-1, 3), complex(-1, -3), complex(-2, 0)]
    res = [[complex(1, 2), complex(0.5, 0.1), complex(3, 0)]]  # not conjugate residues
    t = np.linspace(0, 3, 33)
    np.testing.assert_allclose(P.rational_invert(P.RationalModel(np.array(poles), np.array(res)), t),
                               O.rational_invert(poles, res, t), rtol=1e-12, atol=1e-14)
    with pytest.raises(P.ValidationError):
        P.rational_invert(P.RationalModel(np.array(poles[:1]), np.array([res[0][:1]])), t)
    with pytest.raises(P.NumericError):
        P.rational_invert(P.RationalModel(np.array([1.0 + 0j]), np.array([[1.0 + 0j]])), [0.0, 800.0])


@pytest.mark.parametrize("ns,hann", [(256, True), (512, True), (512, False), (218, True), (16, True), (2, False)])
def test_fsm_invert_parity(ns, hann):
    T = 4.0
    eta = O.damping_eta(3.0, T)
    rng = np.random.default_rng(ns)
    poles = np.array([complex(-0.5, 3), complex(-0.5, -3), complex(-5, 0)])
    res = rng.normal(size=(7, 3)) + 1j * rng.normal(size=(7, 3))
    res[:, 1] = np.conj(res[:, 0])
    res[:, 2] = res[:, 2].real
    sk = eta + 1j * 2 * math.pi / T * np.arange(ns // 2 + 1)
    half = np.array([[np.sum(r / (sv - poles)) for sv in sk] for r in res])
    g = P.fsm_invert(T, ns, eta, half, hann)
    o = O.fsm_invert(T, ns, eta, half, hann)
    assert rel_l2(g, o) < 1e-12


@pytest.mark.parametrize("K", [1, 2, 3, 37, 1001])
@pytest.mark.parametrize("freq_major", [False, True])
def test_fsm_invert_device_layouts(K, freq_major):
    """N_s = 512 device path on both spectrum layouts, odd/even channel counts."""
    import ctypes

    import torch

    ns, T, eta = 512, 6.0, 0.4
    rng = np.random.default_rng(K)
    half = rng.normal(size=(K, ns // 2 + 1)) + 1j * rng.normal(size=(K, ns // 2 + 1))
    ref = O.fsm_invert(T, ns, eta, half, True)
    dev = torch.tensor(half.T.copy() if freq_major else half, device="cuda")
    out = torch.empty((K, ns), dtype=torch.float64, device="cuda")
    sk, si = (1, K) if freq_major else (ns // 2 + 1, 1)
    P.api._check(P.lib().fds_fsm_invert_device_strided(
        ctypes.c_double(T), ns, ctypes.c_double(eta), K, ctypes.c_void_p(dev.data_ptr()), ctypes.c_longlong(sk),
        ctypes.c_longlong(si), 1, ctypes.c_void_p(out.data_ptr()), None))
    assert rel_l2(out.cpu().numpy(), ref) < 1e-12


# ------------------------------------------------ AFS: identical sampled sequence
class _ModalSys:
    def __init__(self, fx):
        self.fx = fx

    def descriptor(self):
        return P.api.SystemDescriptor(len(self.fx.participation), [])

    def evaluate(self, s):
        return self.fx.evaluate(s)


def test_afs_modal_identical_sequence():
    fx = ModalFixture(6)
    kw = dict(omega_max=1.5 * fx.band, eta=0.35, period=20.0, orf_indices=[0, 1, 2], test_indices=[3, 4, 5],
              initial_count=16, grid_points=1024, time_points=256, e1_threshold=1e-2, e2_threshold=5e-2)
    r = P.run_afs(_ModalSys(fx), **kw)
    o = O.run_afs(O.System.from_json(fx.system_json()), omega_max=kw["omega_max"], eta=0.35, period=20.0,
                  orf=[0, 1, 2], test=[3, 4, 5], initial_count=16, grid_points=1024, time_points=256,
                  e1_threshold=1e-2, e2_threshold=5e-2)
    assert r["n_c"] == o["n_c"] and r["converged"] == o["converged"]
    np.testing.assert_array_equal(r["samples"], o["samples"])
    np.testing.assert_array_equal(r["history"][:, :3], o["history"][:, :3])
    assert worst_match(r["poles"], o["poles"]) < 1e-6


@pytest.mark.parametrize("orf,test", [([2, 0, 1], [5, 3, 4]), ([1, 0, 2], [2, 5, 1]), ([2, 1, 0], [4, 0]),
                                      ([1, 3], [3, 1, 0]), ([0, 2, 1], None), ([4, 1], [5, 0, 2])])
def test_afs_channel_subsets_identical_sequence(orf, test):
    """Unsorted / overlapping ORF and test sets (and the default all-channel
    test set) through the device-resident iteration: the worst-ORF argmax, the
    E2 max over test positions and the E1 series of a gathered channel subset
    keep the reference's sequence. ([4, 1] is rank-deficient for the reference's
    relocation: the product must raise the same error class.)"""
    fx = ModalFixture(6)
    kw = dict(omega_max=1.5 * fx.band, eta=0.35, period=20.0, initial_count=16, grid_points=1024,
              time_points=256, e1_threshold=1e-2, e2_threshold=5e-2)
    sel = dict(orf_indices=orf) if test is None else dict(orf_indices=orf, test_indices=test)
    try:
        o = O.run_afs(O.System.from_json(fx.system_json()), orf=orf, test=test if test is not None else [], **kw)
    except O.OracleError as e:  # the reference fails on this set: the product must fail the same way
        with pytest.raises(P.Error) as eg:
            P.run_afs(_ModalSys(fx), **sel, **kw)
        assert type(eg.value).__name__ == e.kind
        return
    r = P.run_afs(_ModalSys(fx), **sel, **kw)
    assert r["n_c"] == o["n_c"] and r["converged"] == o["converged"]
    np.testing.assert_array_equal(r["samples"], o["samples"])
    np.testing.assert_array_equal(r["history"][:, :3], o["history"][:, :3])
    np.testing.assert_allclose(r["history"][:, 7], o["history"][:, 7], rtol=1e-9)


def test_afs_infinite_thresholds():
    fx = ModalFixture(4)
    r = P.run_afs(_ModalSys(fx), omega_max=1.5 * fx.band, eta=0.35, period=20.0, orf_indices=[0, 1],
                  test_indices=[2, 3], initial_count=8, e1_threshold=float("inf"), e2_threshold=float("inf"),
                  grid_points=512, time_points=128)
    assert r["converged"] and r["n_c"] == 11 and r["solver_calls"] == 11


def test_afs_bem_identical_sequence():
    """320-triangle sphere (cfg 1 mesh, T=20, eta=0.25) under the seeded random traction of
    cfg 4 (the pressure load leaves tangential DOFs at pure rounding noise, which makes E2
    noise-dominated — SURVEY.md A.4): product run_afs on the GPU BEM vs the reference
    run_afs on the oracle BEM. Infinite thresholds keep the loop away from the reference
    algorithm's rank-deficiency on this smooth response while exercising
    J_c = 6 adaptive selections on BEM data."""
    from paper_1511_04355_b200 import mesh

    V, F = mesh.icosphere(2)
    tr = mesh.random_traction(F.shape[0], seed=0)
    pts = mesh.draw_indices(F.shape[0], 16, 0)
    dofs = [3 * p + i for p in pts for i in range(3)]
    kw = dict(omega_max=math.pi * 256 / 20.0, eta=0.25, period=20.0, initial_count=12,
              e1_threshold=float("inf"), e2_threshold=float("inf"), validation_steps=6)
    r = P.run_afs(P.BemSystem(V, F, tr, channels=dofs), **kw)
    o = O.run_afs(O.System.bem(O.Bem(V, F, tr), dofs), **kw)
    assert r["n_c"] == o["n_c"] == 18
    np.testing.assert_array_equal(r["samples"], o["samples"])
    np.testing.assert_array_equal(r["history"][:, :3], o["history"][:, :3])
    np.testing.assert_allclose(r["history"][:, 7], o["history"][:, 7], rtol=1e-6)
    assert worst_match(r["poles"], o["poles"]) < 1e-6


def test_identify_residues_kernel_tiers_in_one_process():
    """Residue kernels of different m-tile tiers with > 48 KB of shared memory in
    one process: each instance gets its own dynamic-smem opt-in (a shared flag
    once made the second launch fail with 'invalid argument' inside AFS)."""
    rng = np.random.default_rng(3)

    def poles(pairs):
        p = []
        for m in range(pairs):
            a = complex(-0.2 - 0.01 * m, 1.0 + 0.9 * m)
            p += [a, a.conjugate()]
        return np.array(p)

    for J, pairs in ((60, 2), (50, 20), (44, 8)):
        s = 0.3 + 1j * np.linspace(0.5, 40.0, J)
        v = rng.normal(size=(J, 9)) + 1j * rng.normal(size=(J, 9))
        pl = poles(pairs)
        res, rms = P.identify_residues(s, v, pl)
        for k in (0, 8):
            ro, rmso = O.identify_residues(s, v[:, k], pl)
            assert rel_l2(res[k], ro) < 1e-10
            assert rms[k] == pytest.approx(rmso, rel=1e-8)


@pytest.mark.parametrize("J,pairs,reals,K", [(7, 2, 0, 100), (40, 24, 0, 1000), (41, 23, 1, 333), (64, 32, 0, 129),
                                             (40, 35, 0, 200), (80, 48, 0, 65), (33, 3, 2, 64)])
def test_identify_residues_shapes(J, pairs, reals, K):
    """The bulk-copy-fed residue kernel (J <= 64) and the legacy register-ring
    kernel (J > 64) over odd J, unpaired real poles, M > 64 (two 64-pole
    slices) and channel counts that leave a ragged last 64-channel tile:
    every sampled channel against the oracle's per-channel identify_residues
    (vecfit.cpp:356-408)."""
    rng = np.random.default_rng(J * 1000 + K)
    p = []
    for m in range(pairs):
        a = complex(-0.05 - 0.02 * m, 0.4 + 1.1 * m)
        p += [a, a.conjugate()]
    p += [complex(-0.3 - 0.2 * r, 0.0) for r in range(reals)]
    p = np.array(p)
    s = 0.3 + 1j * np.linspace(0.1, 1.1 * abs(p.imag).max() + 1.0, J)
    v = rng.normal(size=(J, K)) + 1j * rng.normal(size=(J, K))
    res, rms = P.identify_residues(s, v, p)
    for k in sorted({0, 1, K // 2, K - 2, K - 1}):
        ro, rmso = O.identify_residues(s, v[:, k], p)
        assert rel_l2(res[k], ro) < 1e-10, (k, rel_l2(res[k], ro))
        assert rms[k] == pytest.approx(rmso, rel=1e-8)


def test_identify_residues_heads_only_and_rational_invert():
    """fds_vf_identify_residues_device_heads writes the pair heads and real poles
    only (conjugate rows keep whatever the buffer held: here NaN), and
    fds_rational_invert_device on that buffer matches the oracle's
    rational_invert of the full model (laplace.cpp:127-164)."""
    import ctypes

    import torch

    rng = np.random.default_rng(11)
    J, K = 40, 777
    p = []
    for m in range(10):
        a = complex(-0.1 - 0.03 * m, 0.5 + 1.3 * m)
        p += [a, a.conjugate()]
    p += [complex(-0.7, 0.0)]
    p = np.array(p)
    M = len(p)
    s = 0.3 + 1j * np.linspace(0.1, 15.0, J)
    v = rng.normal(size=(J, K)) + 1j * rng.normal(size=(J, K))
    full, _ = P.identify_residues(s, v, p)  # (K, M), every row
    vd = torch.tensor(v, device="cuda")
    rd = torch.full((M, K), complex(float("nan"), float("nan")), dtype=torch.complex128, device="cuda")
    L = P.lib()
    pc = np.ascontiguousarray(O.canonical_poles(p))
    P.api._check(L.fds_vf_identify_residues_device_heads(
        J, K, s.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(vd.data_ptr()), M, pc.ctypes.data_as(ctypes.c_void_p),
        ctypes.c_void_p(rd.data_ptr()), None))
    r = rd.cpu().numpy()
    heads = [m for m in range(M) if not (m < 20 and m % 2 == 1)]
    conj_rows = [m for m in range(M) if m < 20 and m % 2 == 1]
    np.testing.assert_array_equal(r[heads].T, full[:, heads])
    assert np.all(np.isnan(r[conj_rows]))
    t = np.linspace(0.0, 8.0, 300)
    out = torch.empty((K, len(t)), dtype=torch.float64, device="cuda")
    P.api._check(L.fds_rational_invert_device(M, pc.ctypes.data_as(ctypes.c_void_p), K, ctypes.c_void_p(rd.data_ptr()),
                                              len(t), t.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(out.data_ptr()),
                                              None))
    sub = [0, 5, 400, K - 1]
    ho = O.rational_invert(pc, full[sub], t)
    assert rel_l2(out.cpu().numpy()[sub], ho) < 1e-12


def test_eval_model_and_fit_error_on_device():
    """Row a8: eval_model (vecfit.cpp:490-509) and fit_error_evf (:511-526)
    through the device kernels against the oracle, plus the pole-collision
    NumericError and the zero-norm error."""
    s, v = _noisy_modal(7, 30)
    o = O.vector_fit(s, v, [0, 1], 12, 3)
    model = P.RationalModel(o["poles"], o["residues"])
    grid = 0.35 + 1j * np.linspace(0.0, 40.0, 257)
    g = P.eval_model(model, grid)  # (G, K)
    for gi in (0, 100, 256):
        ref = O.eval_model(o["poles"], o["residues"], grid[gi])
        assert rel_l2(g[gi], ref) < 1e-13
    for k in range(7):
        e = P.fit_error_evf(model, k, s, v)
        eo = O.fit_error_evf(o["poles"], o["residues"], k, s, v)
        assert e == pytest.approx(eo, rel=1e-10)
    with pytest.raises(P.NumericError):
        P.eval_model(model, [o["poles"][0]])
    with pytest.raises(P.NumericError):
        P.fit_error_evf(model, 0, s, np.zeros_like(v))
