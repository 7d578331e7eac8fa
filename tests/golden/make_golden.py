"""Generates tests/golden/*.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists and
`make -C oracle ref` produced oracle/_ref/libtgref.so):

    python tests/golden/make_golden.py

The fixtures pin the oracle restatement and the GPU path to the reference's
own known-answer tests:
  ref_triangle.npz   reference triangle K, F, M (test_batch.cpp:72-91, acceptance.cpp:136-161)
  tri3_1x1.npz       1x1 TRI3 grid load [2/6,1/6,1/6,2/6] (test_routing.cpp:139-154)
  mesh_*.npz         small grids: mesh arrays, full routing (pattern, segment maps),
                     assembled K/F/M for several coefficient kinds, elasticity,
                     gradient products and the adjoint gather inputs/outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402


def u01(rng, n):
    """acceptance.cpp:47 uniform(): (rng() >> 11) * 2^-53 of a mt19937_64 stream."""
    return np.array([(rng() >> 11) * 2.0 ** -53 for _ in range(n)])


class MT64:
    """std::mt19937_64 (for the seeded inputs the reference's tests use)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                self.mt[k] = v
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & 0xFFFFFFFFFFFFFFFF


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print(name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def ref_triangle():
    m = ref.Mesh.from_arrays("tri3", [[0, 0], [1, 0], [0, 1]], [[0, 1, 2]])
    r = ref.Routing(m, 1)
    K, F, M = ref.assemble(m, r, sources=[1.0], with_mass=True)
    K1, F1, _ = ref.assemble(m, r, sources=[1.0])
    save("ref_triangle.npz", nodes=m.nodes, elements=m.elements, offsets=r.offsets, cols=r.cols,
         K_deg2=K, F_deg2=F, M=M, K=K1, F=F1)


def tri3_1x1():
    m = ref.Mesh.grid("tri3", [1.0, 1.0], [1, 1])
    r = ref.Routing(m, 1)
    K, F, _ = ref.assemble(m, r, sources=[1.0])
    save("tri3_1x1.npz", nodes=m.nodes, elements=m.elements, K=K, F=F)


def small_mesh(tag, kind, ext, div, seed):
    m = ref.Mesh.grid(kind, ext, div)
    r = ref.Routing(m, 1)
    rng = MT64(seed)
    rho = 0.5 + u01(rng, m.E)
    nodal = 0.5 + u01(rng, m.N)
    src = u01(rng, m.E) - 0.5
    out = dict(nodes=m.nodes, elements=m.elements, boundary=m.boundary_nodes,
               content_hash=np.uint64(m.content_hash()), offsets=r.offsets, cols=r.cols,
               vec_offsets=r.vec_offsets, vec_slots=r.vec_slots, mat_offsets=r.mat_offsets,
               mat_slots=r.mat_slots, rho=rho, nodal=nodal, src=src)
    out["K_const"], out["F_const"], _ = ref.assemble(m, r, sources=[1.0])
    out["K_rho"], out["F_rho"], out["M_rho"] = ref.assemble(m, r, diffusion=("element", rho),
                                                            sources=[("element", src)], with_mass=True)
    out["K_nodal"], out["F_nodal"], _ = ref.assemble(m, r, diffusion=("nodal", nodal),
                                                     sources=[("nodal", nodal)])
    out["K_mass"], _, _ = ref.assemble(m, r, problem="mass", diffusion=("element", rho))
    # elasticity (E=1, nu=0.3 -> lambda, mu of lame_from_young, batch.cpp:353-357)
    d = m.dim
    nu = 0.3
    lam = 1.0 * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    rv = ref.Routing(m, d)
    out["v_offsets"], out["v_cols"] = rv.offsets, rv.cols
    out["v_mat_offsets"], out["v_mat_slots"] = rv.mat_offsets, rv.mat_slots
    out["lam"], out["mu"] = np.float64(lam), np.float64(mu)
    out["K_elast"], out["F_elast"], _ = ref.assemble(m, rv, problem="elasticity", lam=lam, mu=mu,
                                                     sources=[1.0] * d)
    # adjoint inputs/outputs: gradient_products + unit-coefficient local stiffness
    lam_v = u01(rng, m.N) - 0.5
    U = u01(rng, m.N) - 0.5
    out["adj_lambda"], out["adj_U"] = lam_v, U
    out["dK"], out["dF"] = r.gradient_products(lam_v, U)
    out["K0_local"] = ref.local(m, 1, 0, np.ones(m.E))
    save(f"mesh_{tag}.npz", **out)


def allen_cahn(tag, kind, ext, div, seed, eps):
    """AllenCahnStepper Newton re-assembly (timestep.cpp:144-178) through the reference code."""
    m = ref.Mesh.grid(kind, ext, div)
    r = ref.Routing(m, 1)
    u = 2.0 * u01(MT64(seed), m.N) - 1.0
    T, F = ref.allen_cahn(m, r, u, eps)
    save(f"allen_cahn_{tag}.npz", nodes=m.nodes, elements=m.elements, u=u, eps=np.float64(eps), T=T, F=F)


if __name__ == "__main__":
    ref_triangle()
    tri3_1x1()
    small_mesh("tri3_3x3", "tri3", [1.0, 1.0], [3, 3], 11)
    small_mesh("tri3_7x5", "tri3", [1.0, 0.5], [7, 5], 12)
    small_mesh("tet4_2x2x2", "tet4", [1.0, 1.0, 1.0], [2, 2, 2], 13)
    small_mesh("tet4_3x2x4", "tet4", [1.3, 0.7, 1.1], [3, 2, 4], 14)
    allen_cahn("tri3_7x5", "tri3", [1.0, 0.5], [7, 5], 21, 0.8)
    allen_cahn("tet4_3x2x4", "tet4", [1.3, 0.7, 1.1], [3, 2, 4], 22, 0.35)
