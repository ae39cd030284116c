"""Synthetic BEM meshes and loads for the BASELINE.json configurations.

Deterministic host-side generators (numpy, no randomness outside the pinned
xorshift64 generator of proj/src/afs.cpp:31-37 / tests/test_helpers.hpp:20-38):

* ``icosphere(level)`` — unit sphere, recursive 4-way midpoint subdivision of an
  icosahedron projected to the sphere; levels 2/3/4 give 320/1280/5120
  triangles (configs 1/2/4).
* ``cube_cavity(n)`` — unit cube [0,1]^3, n x n squares per face, each split
  into two right triangles along the (i,j)->(i+1,j+1) diagonal (config 3:
  n = 32 -> 12288 triangles).

Triangles are ordered so that the geometric normal (v1-v0) x (v2-v0) is the
OUTWARD normal of the elastic domain, i.e. it points INTO the cavity. The BEM
(host C-ABI ``fds_bem_create`` and the CPU oracle alike) takes that normal as n(y).
"""
from __future__ import annotations

import math

import numpy as np

MASK = (1 << 64) - 1


def _icosahedron():
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    v /= np.linalg.norm(v, axis=1)[:, None]
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    return v, f


def icosphere(level: int, radius: float = 1.0):
    """-> (vertices (nv,3) float64, triangles (ne,3) int32); normals point to the centre."""
    v, f = _icosahedron()
    verts = [tuple(x) for x in v]
    for _ in range(level):
        cache = {}
        nf = []

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                p = np.add(verts[a], verts[b]) * 0.5
                p = p / np.linalg.norm(p)
                cache[key] = len(verts)
                verts.append(tuple(p))
            return cache[key]

        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        f = np.array(nf, dtype=np.int64)
    V = np.array(verts, dtype=np.float64) * radius
    # icosahedron faces are counter-clockwise seen from outside (normal outward);
    # flip to point into the cavity (domain-outward for the exterior problem).
    F = f[:, [0, 2, 1]].astype(np.int32)
    return V, F


def cube_cavity(n: int):
    """Unit cube cavity surface, 12 n^2 triangles, normals pointing into the cube."""
    verts = {}
    vl = []

    def vid(p):
        key = tuple(int(round(c * n)) for c in p)
        if key not in verts:
            verts[key] = len(vl)
            vl.append(tuple(c / n for c in key))
        return verts[key]

    tris = []
    # each face: fixed axis a at value 0 or 1; (u,v) the two other axes in right-handed order
    for a in range(3):
        u, w = (a + 1) % 3, (a + 2) % 3
        for side in (0, 1):
            for i in range(n):
                for j in range(n):
                    def P(ii, jj):
                        p = [0.0, 0.0, 0.0]
                        p[a] = float(side)
                        p[u] = ii / n
                        p[w] = jj / n
                        return vid(p)
                    p00, p10, p11, p01 = P(i, j), P(i + 1, j), P(i + 1, j + 1), P(i, j + 1)
                    # (u x w) = +e_a: ccw in (u,w) has normal +e_a.
                    t1, t2 = [p00, p10, p11], [p00, p11, p01]
                    # into the cube: side 0 needs +e_a, side 1 needs -e_a
                    if side == 1:
                        t1, t2 = t1[::-1], t2[::-1]
                    tris += [t1, t2]
    return np.array(vl, dtype=np.float64), np.array(tris, dtype=np.int32)


def element_geometry(V, F):
    """-> centroids (ne,3), unit normals (ne,3), areas (ne,)"""
    p0, p1, p2 = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    c = (p0 + p1 + p2) / 3.0
    nn = np.cross(p1 - p0, p2 - p0)
    tw = np.linalg.norm(nn, axis=1)
    return c, nn / tw[:, None], 0.5 * tw


def pressure_traction(V, F, p0: float = 1.0):
    """Cavity pressure p0 (x Heaviside 1/s): traction on the solid t = -p0 n (n into the cavity)."""
    _, n, _ = element_geometry(V, F)
    return np.ascontiguousarray(-p0 * n)


class XorShift64:
    """The reference's generator (proj/src/afs.cpp:31-37): state = seed ^ 0x9e3779b97f4a7c15."""

    def __init__(self, seed: int):
        self.state = (seed ^ 0x9E3779B97F4A7C15) & MASK
        if self.state == 0:
            self.state = 1

    def next(self) -> int:
        s = self.state
        s ^= (s << 13) & MASK
        s ^= s >> 7
        s ^= (s << 17) & MASK
        self.state = s & MASK
        return self.state

    def uniform(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53

    def normal(self) -> float:
        u1 = max(self.uniform(), 2.0 ** -60)
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def random_traction(ne: int, seed: int = 0):
    """Config 4: per-element i.i.d. N(0,1) 3-vectors, xorshift64 + Box–Muller, seed 0."""
    g = XorShift64(seed)
    return np.array([[g.normal() for _ in range(3)] for _ in range(ne)], dtype=np.float64)


def draw_indices(n: int, k: int, seed: int):
    """proj/src/afs.cpp:28-46 (sorted partial Fisher–Yates with xorshift64)."""
    pool = list(range(n))
    g = XorShift64(seed)
    out = []
    for i in range(k):
        j = i + g.next() % (n - i)
        pool[i], pool[j] = pool[j], pool[i]
        out.append(pool[i])
    return sorted(out)


def sphere_radial_analytic(s, a=1.0, mu=1.0, nu=0.25, rho=1.0, p0=1.0):
    """Spherical cavity under Heaviside pressure: U_r(a, s)."""
    lam = 2 * mu * nu / (1 - 2 * nu)
    cp = math.sqrt((lam + 2 * mu) / rho)
    k = s / cp
    return (p0 / s) * a * (1 + k * a) / ((lam + 2 * mu) * k * k * a * a + 4 * mu * (1 + k * a))
