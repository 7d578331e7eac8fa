"""Synthetic input meshes of the benchmark configurations.

``kuhn`` is the reference's own tg::generate_grid (mesh.cpp:96-169, through
libtgk's bit-identical host generator).  ``unstructured_tri`` builds the C4
operator-learning mesh: a 2D unstructured triangulation of the unit square
with scrambled numbering, so the assembly sees no grid structure:

  * (n+1)^2 points of the uniform grid, interior points jittered by
    U[-0.15h, 0.15h] per coordinate (seed 42) — every triangle keeps a
    positive area (the worst-case doubled area is 0.4h^2);
  * one random diagonal per cell (seed 43): E = 2n^2, nnz = N + 2*edges;
  * random node and element permutations (seed 44);
  * counter-clockwise orientation (positive Jacobian, batch.cpp:98-101).

Random numbers are std::mt19937_64 draws mapped as u = (x >> 11) * 2^-53, the
reference tests' uniform() (acceptance.cpp:47), so a C++ caller can rebuild
the same mesh.
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (seeded with one 64-bit integer)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def next(self):
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK

    def uniform(self, n):
        """n draws of (x >> 11) * 2^-53 in [0, 1)."""
        return np.array([(self.next() >> 11) for _ in range(n)], dtype=np.float64) * (2.0 ** -53)


def _permutation(rng: MT19937_64, n):
    """Fisher-Yates with j = floor(u * (i + 1))."""
    p = np.arange(n, dtype=np.int64)
    u = rng.uniform(max(0, n - 1))
    for t, i in enumerate(range(n - 1, 0, -1)):
        j = int(u[t] * (i + 1))
        p[i], p[j] = p[j], p[i]
    return p


def unstructured_tri(n=256, jitter=0.15, seeds=(42, 43, 44)):
    """C4 mesh: returns (nodes N x 2 float64, elements E x 3 int64)."""
    h = 1.0 / n
    i, j = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="xy")
    x = (i.reshape(-1) * h).astype(np.float64)
    y = (j.reshape(-1) * h).astype(np.float64)
    interior = (i.reshape(-1) > 0) & (i.reshape(-1) < n) & (j.reshape(-1) > 0) & (j.reshape(-1) < n)
    ni = int(interior.sum())
    u = MT19937_64(seeds[0]).uniform(2 * ni).reshape(ni, 2)
    x[interior] += (2.0 * u[:, 0] - 1.0) * jitter * h
    y[interior] += (2.0 * u[:, 1] - 1.0) * jitter * h
    nodes = np.stack([x, y], axis=1)
    ci, cj = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    n00 = (cj * (n + 1) + ci).reshape(-1)
    n10, n01, n11 = n00 + 1, n00 + (n + 1), n00 + (n + 2)
    diag = MT19937_64(seeds[1]).uniform(n * n) < 0.5
    t1 = np.where(diag[:, None], np.stack([n00, n10, n11], 1), np.stack([n00, n10, n01], 1))
    t2 = np.where(diag[:, None], np.stack([n00, n11, n01], 1), np.stack([n10, n11, n01], 1))
    elems = np.stack([t1, t2], axis=1).reshape(-1, 3).astype(np.int64)
    rng = MT19937_64(seeds[2])
    pn = _permutation(rng, nodes.shape[0])        # new node id -> old node id
    pe = _permutation(rng, elems.shape[0])        # new element id -> old element id
    inv = np.empty_like(pn)
    inv[pn] = np.arange(pn.size)
    nodes = nodes[pn]
    elems = inv[elems[pe]]
    # counter-clockwise orientation
    p0, p1, p2 = nodes[elems[:, 0]], nodes[elems[:, 1]], nodes[elems[:, 2]]
    area2 = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])
    neg = area2 < 0
    elems[neg, 1], elems[neg, 2] = elems[neg, 2].copy(), elems[neg, 1].copy()
    return np.ascontiguousarray(nodes), np.ascontiguousarray(elems)


def kuhn(kind, divisions, extents=None):
    """tg::generate_grid (mesh.cpp:96-169), bit-identical."""
    from . import tgfem
    m = tgfem.generate_grid(kind, extents or [1.0] * len(divisions), list(divisions))
    return m.nodes, m.elements


def batch_fields(B, E, seed0=1000, lo=0.5):
    """Operator-learning coefficient batch: rho[b, e] = lo + U[0,1) (numpy PCG64, seed seed0 + b)."""
    out = np.empty((B, E))
    for b in range(B):
        out[b] = lo + np.random.default_rng(seed0 + b).random(E)
    return out
