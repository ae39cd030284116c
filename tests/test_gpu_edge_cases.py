"""Edge cases of the device path against the reference semantics (the oracle):
the same error class for the same invalid input, and empty / minimal / ragged
inputs that the reference accepts (vecfit.cpp:410-488, laplace.cpp:89-164,
afs.cpp:59-84 validation)."""
import math

import numpy as np
import pytest

import paper_1511_04355_b200 as P
import pyoracle as O

pytestmark = pytest.mark.gpu

KIND = {P.ValidationError: "ValidationError", P.NumericError: "NumericError", P.ConvergenceError: "ConvergenceError"}


def same_error(gpu_call, oracle_call):
    with pytest.raises(P.Error) as eg:
        gpu_call()
    with pytest.raises(O.OracleError) as eo:
        oracle_call()
    assert KIND.get(type(eg.value)) == eo.value.kind, (eg.value, eo.value)


def contour(J, eta=0.3, wmax=30.0):
    return eta + 1j * wmax * (1 - np.cos(np.arange(J) * math.pi / (2 * (J - 1))))


def model_values(s, poles, res):
    return np.array([[np.sum(r / (sv - poles)) for r in res] for sv in s])


POLES = np.array([complex(-0.5, 4), complex(-0.5, -4), complex(-2, 0)])
RES = np.array([[1 + 2j, 1 - 2j, 0.5], [0.3 - 1j, 0.3 + 1j, -2.0]])


@pytest.mark.parametrize("case", ["order_too_high", "empty_orf", "orf_out_of_range", "zero_relocations",
                                  "duplicate_frequency"])
def test_vector_fit_errors_match_reference(case):
    s = contour(10)
    v = model_values(s, POLES, RES)
    orf, order, nrel = [0, 1], 4, 3
    if case == "order_too_high":
        order = 20
    elif case == "empty_orf":
        orf = []
    elif case == "orf_out_of_range":
        orf = [0, 5]
    elif case == "zero_relocations":
        nrel = 0
    elif case == "duplicate_frequency":
        s = s.copy()
        s[3] = s[2]
    same_error(lambda: P.vector_fit(s, v, orf, order, nrel), lambda: O.vector_fit(s, v, orf, order, nrel))


def test_identify_residues_pole_collision_matches_reference():
    s = contour(8)
    v = model_values(s, POLES, RES)
    poles = POLES.copy()
    poles[2] = s[4]  # a sample frequency on a pole: basis division by zero
    same_error(lambda: P.identify_residues(s, v, poles), lambda: O.identify_residues(s, v[:, 0], poles))


def test_minimal_sample_count_fit():
    """J = order/2 + 1 samples, one channel: still solvable, same poles as the oracle."""
    s = contour(4)
    v = model_values(s, POLES[:2], RES[:1, :2])
    m, _ = P.vector_fit(s, v, [0], 2, 3)
    o = O.vector_fit(s, v, [0], 2, 3)
    for p in o["poles"]:
        assert np.min(np.abs(m.poles - p)) / abs(p) < 1e-6


def test_fsm_and_rational_invert_empty_and_single():
    T, ns, eta = 4.0, 16, 0.5
    assert P.fsm_invert(T, ns, eta, np.zeros((0, ns // 2 + 1), complex)).shape == (0, ns)
    half = np.ones((1, ns // 2 + 1), complex)
    np.testing.assert_allclose(P.fsm_invert(T, ns, eta, half), O.fsm_invert(T, ns, eta, half), rtol=0, atol=1e-13)
    model = P.RationalModel(POLES, RES)
    t1 = np.array([0.7])
    np.testing.assert_allclose(P.rational_invert(model, t1), O.rational_invert(POLES, RES, t1), rtol=1e-13)
    same_error(lambda: P.rational_invert(model, np.array([1.0, 0.5])),
               lambda: O.rational_invert(POLES, RES, np.array([1.0, 0.5])))
    same_error(lambda: P.fsm_invert(T, 15, eta, np.ones((1, 8), complex)),
               lambda: O.fsm_invert(T, 15, eta, np.ones((1, 8), complex)))


@pytest.mark.parametrize("bad", [dict(initial_count=3), dict(alpha_high=2.5, alpha_low=2.3),
                                 dict(e1_threshold=0.0), dict(validation_steps=-1), dict(grid_points=1),
                                 dict(time_points=1), dict(max_iterations=0), dict(n_relocations=0),
                                 dict(orf=[0, 0]), dict(test=[7])])
def test_afs_config_errors_match_reference(bad):
    from helpers import ModalFixture

    fx = ModalFixture(6)
    base = dict(omega_max=1.5 * 29.8, eta=0.35, period=20.0, grid_points=256, time_points=128)
    cfg = {**base, **bad}

    class Sys:
        def descriptor(self):
            return P.api.SystemDescriptor(6, [])

        def evaluate(self, s):
            return fx.evaluate(s)

    gcfg = {("orf_indices" if k == "orf" else "test_indices" if k == "test" else k): v for k, v in cfg.items()}
    same_error(lambda: P.run_afs(Sys(), **gcfg), lambda: O.run_afs(O.System.from_json(fx.system_json()), **cfg))
