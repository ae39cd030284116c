"""Pins the CPU oracle's vector fitting to the reference's own unit tests.

Each test restates one TEST_CASE of proj/tests/test_vecfit.cpp (line numbers
cited) with the same data, calls and tolerances, against the oracle
(oracle/_ref/libfdsweep_oracle.so). These are the golden pins of the oracle
(SURVEY.md §4, §8c): the Eigen-backed reference cannot be built here.
"""
import numpy as np
import pytest

import pyoracle as O
from helpers import ModalFixture, TestRng, contour_points, rational_samples, rel_err, worst_match


def test_initial_poles_single_pair():  # test_vecfit.cpp:35-40
    p = O.initial_poles(100.0, 2)
    assert len(p) == 2
    assert p[0] == complex(-1.0, 100.0) and p[1] == complex(-1.0, -100.0)


def test_initial_poles_equally_spaced():  # :42-48
    p = O.initial_poles(100.0, 4)
    assert p[0] == complex(-0.5, 50.0) and p[2] == complex(-1.0, 100.0)
    assert O.is_conjugate_closed(p)


def test_initial_poles_odd_order():  # :50-55
    p = O.initial_poles(200.0, 5)
    assert len(p) == 5 and p[4] == complex(-2.0, 0.0)
    assert O.is_conjugate_closed(p)


def test_relocation_two_pole_recovery():  # :57-68
    true = [complex(-1, 10), complex(-1, -10)]
    s, v = rational_samples(true, [[complex(0.5, -0.3), complex(0.5, 0.3)]], contour_points(1.0, 20.0, 12))
    poles = np.array([complex(-0.5, 50), complex(-0.5, -50)])
    for _ in range(3):
        poles, _, _ = O.relocate_poles(s, v, poles)
    assert worst_match(poles, true) < 1e-8
    assert O.is_conjugate_closed(poles)


def test_relocation_exact_poles_fixed_point():  # :70-79
    true = [complex(-2, 30), complex(-2, -30), complex(-5, 0)]
    s, v = rational_samples(true, [[complex(1, 0.7), complex(1, -0.7), complex(2, 0)]], contour_points(0.5, 60.0, 16))
    rel, _, _ = O.relocate_poles(s, v, true)
    assert worst_match(rel, true) < 1e-10


def test_relocation_keeps_unstable():  # :81-90
    true = [complex(0.3, 0), complex(-2, 0)]
    s, v = rational_samples(true, [[1.0 + 0j, 1.0 + 0j]], contour_points(1.0, 10.0, 10))
    r = O.vector_fit(s, v, [0], 2, 3)
    assert r["unstable"] == 1
    assert worst_match(r["poles"], true) < 1e-8


def test_residue_identification_exact():  # :92-102
    freqs = contour_points(1.0, 8.0, 8)
    vals = 1.0 / (freqs + 2.0)
    res, rms = O.identify_residues(freqs, vals, [complex(-2, 0)])
    assert rel_err(res[0], 1.0) < 1e-10
    assert rms < 1e-12


def test_residue_identification_zero_data():  # :104-111
    freqs = contour_points(1.0, 10.0, 6)
    res, _ = O.identify_residues(freqs, np.zeros(6, complex), [complex(-1, 5), complex(-1, -5)])
    assert np.all(np.abs(res) == 0.0)


def test_vector_fit_one_orf_three_channels():  # :113-132
    poles = [complex(-1, 12), complex(-1, -12), complex(-3, 40), complex(-3, -40)]
    residues = [[complex(0.4, 0.1), complex(0.4, -0.1), complex(1.5, 0), complex(1.5, 0)],
                [complex(-0.8, 0.2), complex(-0.8, -0.2), complex(0.3, -0.9), complex(0.3, 0.9)],
                [complex(2.0, 0), complex(2.0, 0), complex(-0.5, 0.25), complex(-0.5, -0.25)]]
    s, v = rational_samples(poles, residues, contour_points(0.8, 60.0, 14))
    r = O.vector_fit(s, v, [0], 4, 3)
    assert r["residues"].shape[0] == 3
    assert np.all(r["rms"] < 1e-8)
    assert worst_match(r["poles"], poles) < 1e-7
    assert O.is_conjugate_closed(r["poles"])
    assert np.all(np.isfinite(r["residues"]))


def test_vector_fit_exact_recovery_half_count():  # :134-144
    poles = [complex(-0.5, 8), complex(-0.5, -8), complex(-2, 25), complex(-2, -25)]
    residues = [[complex(1, -0.4), complex(1, 0.4), complex(0.7, 0), complex(0.7, 0)]]
    s, v = rational_samples(poles, residues, contour_points(0.5, 40.0, 8))
    r = O.vector_fit(s, v, [0], 4, 4)
    assert worst_match(r["poles"], poles) < 1e-8
    assert worst_match(r["residues"][0], residues[0]) < 1e-8


def test_vector_fit_modal_fixture():  # :146-156
    fx = ModalFixture(6)
    s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 48))
    r = O.vector_fit(s, v, [0, 1, 2], 16, 3)
    assert r["iterations"] <= 3
    assert r["movement"] < 1e-6
    assert worst_match(r["poles"], fx.poles) < 1e-6


def test_model_evaluation_basics():  # :158-175
    poles, res = [complex(-2, 0)], [[1.0 + 0j]]
    assert O.eval_model(poles, res, 0j)[0] == complex(0.5, 0)
    s = complex(0.3, 4.0)
    assert rel_err(O.eval_model(poles, res, s.conjugate())[0], O.eval_model(poles, res, s)[0].conjugate()) < 1e-15
    assert rel_err(O.eval_model(poles, [[2.0 + 0j]], s)[0], 2.0 * O.eval_model(poles, res, s)[0]) < 1e-15
    with pytest.raises(O.OracleError) as e:
        O.eval_model(poles, res, complex(-2, 0))
    assert e.value.kind == "NumericError"


def test_fit_error_evf():  # :177-196
    poles, res = [complex(-2, 0)], [[1.0 + 0j]]
    s, v = rational_samples(poles, res, contour_points(1.0, 10.0, 6))
    assert O.fit_error_evf(poles, res, 0, s, v) == 0.0
    assert O.fit_error_evf(poles, [[0j]], 0, s, v) == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(O.OracleError) as e:
        O.fit_error_evf(poles, res, 0, s, np.zeros_like(v))
    assert e.value.kind == "NumericError"


def test_property_well_separated_models():  # :198-231
    band = 100.0
    rng = TestRng(7)
    for _trial in range(10):
        order = 2 * (1 + rng.next() % 5)
        poles = []
        while len(poles) < order:
            cand = complex(-rng.uniform(0.5, band / 10.0), rng.uniform(band / 50.0, band))
            if any(abs(p - cand) < band / 50.0 or abs(p - cand.conjugate()) < band / 50.0 for p in poles):
                continue
            poles += [cand, cand.conjugate()]
        residues = [[]]
        for _m in range(0, order, 2):
            r = complex(rng.uniform(0.5, 2.0), rng.uniform(-1.0, 1.0))
            residues[0] += [r, r.conjugate()]
        s, v = rational_samples(poles, residues, contour_points(band / 100.0, band, 2 * order + 4))
        r = O.vector_fit(s, v, [0], order, 5)
        assert worst_match(r["poles"], poles) < 1e-7
        assert O.is_conjugate_closed(r["poles"])


@pytest.mark.xfail(strict=True, reason=(
    "reference test_vecfit.cpp:233-246 as written: after 6 relocations the poles still move "
    "by 1.3e-5, so the residue RMS exceeds the relocation RMS by 1.7e-5 relative (> 1e-6). "
    "An independent numpy/LAPACK restatement reproduces the identical pole trajectory to 1e-11 "
    "(tests/test_oracle_crosscheck.py), so this pins a property the algorithm does not have "
    "at n_relocations=6; the converged form is asserted below."))
def test_residue_rms_never_lags_relocation():  # :233-246
    _rms_lag_check(6)


def test_residue_rms_never_lags_relocation_converged():  # :233-246 at convergence
    _rms_lag_check(12)


def _rms_lag_check(n_reloc):
    fx = ModalFixture(4)
    s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 40))
    r = O.vector_fit(s, v, [0, 1], 12, n_reloc)
    assert len(r["reloc_rms"]) == 2
    for k in range(2):
        assert r["rms"][k] <= r["reloc_rms"][k] * (1 + 1e-6) + 1e-15


@pytest.mark.xfail(strict=True, raises=O.OracleError, reason=(
    "reference test_vecfit.cpp:248-261 as written sweeps the order to J/2 = 32 on exactly "
    "16-pole modal data: from order 18 the sigma least-squares system is exactly rank-deficient "
    "(two |R_ii| ~ 5e-16 vs Eigen's threshold min(m,n)*eps*max|R_kk| ~ 4e-15), so "
    "relocate_poles must throw NumericError (vecfit.cpp:282-284); the sweep up to the true "
    "order is asserted below."))
def test_raising_order_does_not_degrade():  # :248-261
    _order_sweep(32)


def test_raising_order_does_not_degrade_to_true_order():  # :248-261, M <= 16
    _order_sweep(16)


def _order_sweep(max_order):
    fx = ModalFixture(3)
    s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 64))
    prev = -1.0
    for order in range(4, max_order + 1, 2):
        r = O.vector_fit(s, v, [0], order, 3)
        evf = O.fit_error_evf(r["poles"], r["residues"], 0, s, v)
        if prev >= 0:
            assert evf <= 1.1 * prev + 1e-12
        prev = evf


class TestValidationFailures:  # :263-288
    def setup_method(self):
        poles = [complex(-1, 2), complex(-1, -2)]
        self.s, self.v = rational_samples(poles, [[1.0 + 0j, 1.0 + 0j]], contour_points(1.0, 10.0, 6))
        self.poles = poles

    def test_duplicate_frequencies(self):
        s = np.append(self.s, self.s[0])
        v = np.vstack([self.v, self.v[:1]])
        with pytest.raises(O.OracleError) as e:
            O.vector_fit(s, v, [0], 2, 3)
        assert e.value.kind == "ValidationError"

    def test_order_too_high(self):
        with pytest.raises(O.OracleError) as e:
            O.vector_fit(self.s, self.v, [0], 12, 3)
        assert e.value.kind == "ValidationError"

    def test_non_closed_poles(self):
        with pytest.raises(O.OracleError) as e:
            O.identify_residues(contour_points(1.0, 10.0, 6), np.ones(6, complex), [complex(-1, 2)])
        assert e.value.kind == "ValidationError"

    def test_zero_data_relocation(self):
        with pytest.raises(O.OracleError) as e:
            O.relocate_poles(self.s, np.zeros_like(self.v), self.poles)
        assert e.value.kind == "NumericError"
