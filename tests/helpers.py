"""Shared test fixtures — a Python restatement of the reference's
proj/tests/test_helpers.hpp (TestRng xorshift64 :20-38, rational_sum /
rational_samples :41-65, contour_points :74-80, mode_partial_fractions :85-95,
ModalFixture :97-136, make_rod_layout :145-157). Independent of every code
path under test: responses are summed term by term from known poles/residues.
"""
import math

import numpy as np

MASK = (1 << 64) - 1


class TestRng:
    """xorshift64 seeded with seed ^ 0x9e3779b97f4a7c15 (test_helpers.hpp:20-38)."""

    __test__ = False

    def __init__(self, seed):
        self.state = (seed ^ 0x9E3779B97F4A7C15) & MASK
        if self.state == 0:
            self.state = 1

    def next(self):
        s = self.state
        s ^= (s << 13) & MASK
        s ^= s >> 7
        s ^= (s << 17) & MASK
        self.state = s & MASK
        return self.state

    def uniform(self, lo, hi):
        u = (self.next() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u

    def normal(self):
        """Box–Muller on two uniforms (pinned generator for seeded loads)."""
        u1 = self.uniform(0.0, 1.0)
        u2 = self.uniform(0.0, 1.0)
        u1 = max(u1, 2.0 ** -60)
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def rational_sum(poles, residues, s):
    acc = 0j
    for p, r in zip(poles, residues):
        acc += r / (s - p)
    return acc


def rational_samples(poles, residues, freqs):
    """-> (s (J,), values (J, K))"""
    vals = np.array([[rational_sum(poles, row, s) for row in residues] for s in freqs], np.complex128)
    return np.array(freqs, np.complex128), vals


def contour_points(eta, omega_max, count):
    return np.array([complex(eta, omega_max * j / (count - 1)) for j in range(count)])


def mode_partial_fractions(omega, zeta, phi):
    damped = omega * math.sqrt(1.0 - zeta * zeta)
    p = complex(-zeta * omega, damped)
    r = phi / (2j * damped)
    return [p, p.conjugate()], [r, r.conjugate()]


class ModalFixture:
    def __init__(self, channels=10):
        self.omega = [2.1, 2.7, 5.3, 8.9, 13.1, 13.7, 21.4, 29.8]
        self.zeta = [0.01, 0.02, 0.015, 0.01, 0.03, 0.025, 0.02, 0.05]
        rng = TestRng(42)
        self.participation = []
        for _ in range(channels):
            row = []
            for _n in range(len(self.omega)):
                phi = rng.uniform(0.2, 2.0)
                if rng.next() % 2 == 0:
                    phi = -phi
                row.append(phi)
            self.participation.append(row)
        self.poles = []
        self.residues = [[] for _ in range(channels)]
        for k in range(channels):
            for n in range(len(self.omega)):
                p, r = mode_partial_fractions(self.omega[n], self.zeta[n], self.participation[k][n])
                self.residues[k] += r
                if k == 0:
                    self.poles += p
        self.band = max(self.omega)

    def system_json(self):
        import json

        part = {f"ch{k}": row for k, row in enumerate(self.participation)}
        return json.dumps({"type": "modal", "omega": self.omega, "zeta": self.zeta, "participation": part})

    def evaluate(self, s):
        den = [s * s + 2 * z * w * s + w * w for w, z in zip(self.omega, self.zeta)]
        return np.array([sum(phi / d for phi, d in zip(row, den)) for row in self.participation])

    def samples(self, freqs):
        return np.array(freqs), np.array([self.evaluate(s) for s in freqs])


def rel_err(got, want):
    return abs(got - want) / max(abs(want), 1e-300)


def worst_match(got, want):
    """Each wanted value against its nearest candidate (test_vecfit.cpp:22-31)."""
    worst = 0.0
    for w in want:
        best = min(rel_err(g, w) for g in got)
        worst = max(worst, best)
    return worst
