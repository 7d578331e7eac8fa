"""CPU: pin the oracle restatement (oracle/tg_oracle.c) to the reference.

1. against the golden fixtures generated from the unmodified reference
   (tests/golden/make_golden.py) — always;
2. against the reference library itself (oracle/_ref/libtgref.so) on seeded
   random grids, mirroring acceptance.cpp:72-132 — when it is loadable.
"""
import glob
import os

import numpy as np
import pytest

from oracle import port
from tests._util import MT64, assert_bitwise

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def test_reference_triangle_known_answers():
    g = load("ref_triangle.npz")
    r = port.Routing(3, port.dofmap("tri3", g["elements"], 1))
    K, F, _ = port.assemble("tri3", g["nodes"], g["elements"], r, sources=[1.0])
    # test_batch.cpp:72-91: K = [[1,-.5,-.5],[-.5,.5,0],[-.5,0,.5]], F = 1/6
    dense = np.zeros((3, 3))
    for i in range(3):
        for t in range(r.offsets[i], r.offsets[i + 1]):
            dense[i, r.cols[t]] = K[t]
    np.testing.assert_allclose(dense, [[1, -.5, -.5], [-.5, .5, 0], [-.5, 0, .5]], atol=1e-14)
    np.testing.assert_allclose(F, [1 / 6] * 3, atol=1e-14)
    assert_bitwise(K, g["K"], "K")
    assert_bitwise(F, g["F"], "F")
    K2, F2, M = port.assemble("tri3", g["nodes"], g["elements"], r, sources=[1.0], with_mass=True)
    Md = np.zeros((3, 3))
    for i in range(3):
        for t in range(r.offsets[i], r.offsets[i + 1]):
            Md[i, r.cols[t]] = M[t]
    np.testing.assert_allclose(Md, np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]]) / 24, atol=1e-14)
    assert_bitwise(M, g["M"], "M")
    assert_bitwise(K2, g["K_deg2"], "K deg2")
    assert_bitwise(F2, g["F_deg2"], "F deg2")


def test_tri3_1x1_load():
    g = load("tri3_1x1.npz")
    nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [1, 1])
    assert np.array_equal(nodes, g["nodes"]) and np.array_equal(elems, g["elements"])
    r = port.Routing(4, port.dofmap("tri3", elems, 1))
    K, F, _ = port.assemble("tri3", nodes, elems, r, sources=[1.0])
    np.testing.assert_allclose(F, [2 / 6, 1 / 6, 1 / 6, 2 / 6], rtol=1e-15)  # test_routing.cpp:147-150
    assert_bitwise(F, g["F"])
    assert_bitwise(K, g["K"])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "mesh_*.npz"))))
def test_small_mesh_golden(path):
    g = dict(np.load(path))
    kind = "tet4" if g["nodes"].shape[1] == 3 else "tri3"
    nodes, elems = g["nodes"], g["elements"]
    assert port.content_hash(kind, nodes, elems) == int(g["content_hash"])
    N = nodes.shape[0]
    r = port.Routing(N, port.dofmap(kind, elems, 1))
    for key in ["offsets", "cols", "vec_offsets", "vec_slots", "mat_offsets", "mat_slots"]:
        assert np.array_equal(getattr(r, key), g[key]), key
    K, F, _ = port.assemble(kind, nodes, elems, r, sources=[1.0])
    assert_bitwise(K, g["K_const"], "K const")
    assert_bitwise(F, g["F_const"], "F const")
    K, F, M = port.assemble(kind, nodes, elems, r, diffusion=("element", g["rho"]),
                            sources=[("element", g["src"])], with_mass=True)
    assert_bitwise(K, g["K_rho"], "K rho")
    assert_bitwise(F, g["F_rho"], "F rho")
    assert_bitwise(M, g["M_rho"], "M rho")
    K, F, _ = port.assemble(kind, nodes, elems, r, diffusion=("nodal", g["nodal"]),
                            sources=[("nodal", g["nodal"])])
    assert_bitwise(K, g["K_nodal"], "K nodal")
    assert_bitwise(F, g["F_nodal"], "F nodal")
    K, _, _ = port.assemble(kind, nodes, elems, r, problem="mass", diffusion=("element", g["rho"]))
    assert_bitwise(K, g["K_mass"], "K mass")
    d = nodes.shape[1]
    rv = port.Routing(N * d, port.dofmap(kind, elems, d))
    assert np.array_equal(rv.offsets, g["v_offsets"]) and np.array_equal(rv.cols, g["v_cols"])
    assert np.array_equal(rv.mat_offsets, g["v_mat_offsets"])
    assert np.array_equal(rv.mat_slots, g["v_mat_slots"])
    K, F, _ = port.assemble(kind, nodes, elems, rv, problem="elasticity", lam=float(g["lam"]),
                            mu=float(g["mu"]), sources=[1.0] * d)
    assert_bitwise(K, g["K_elast"], "K elasticity")
    assert_bitwise(F, g["F_elast"], "F elasticity")
    dK, dF = r.gradient_products(g["adj_lambda"], g["adj_U"])
    assert_bitwise(dK, g["dK"], "dK")
    assert_bitwise(dF, g["dF"], "dF")
    K0 = port.local(kind, nodes, elems, 1, port.DIFFUSION, np.ones(elems.shape[0]))
    assert_bitwise(K0, g["K0_local"], "K0 local")
    # adjoint gather (tg_main.cpp:846-850) vs the pattern-generic chain rule (acceptance.cpp:372-377)
    dm = port.dofmap(kind, elems, 1)
    fused = port.adjoint_gather(dm, K0, g["adj_lambda"], g["adj_U"])
    generic = r.adjoint_generic(K0, g["dK"])
    np.testing.assert_allclose(fused, generic, rtol=1e-12, atol=1e-15)
    direct = np.einsum("ea,eab,eb->e", g["adj_lambda"][dm], K0, g["adj_U"][dm])
    np.testing.assert_allclose(fused, direct, rtol=1e-12, atol=1e-15)


def _ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library oracle/_ref/libtgref.so not built here")
    return ref


def test_random_grids_vs_reference():
    """acceptance.cpp:72-132 style: seeded random grids, port == reference bitwise."""
    ref = _ref()
    rng = MT64(2024)
    for trial in range(24):
        kind = ["tri3", "tet4"][trial % 2]
        d = port.element_dim(kind)
        div, ext = [], []
        for c in range(d):
            div.append(1 + rng() % (12 if d == 2 else 5))
            ext.append(0.5 + 1.5 * rng.uniform(1)[0])
        m = ref.Mesh.grid(kind, ext, div)
        nodes, elems = port.generate_grid(kind, ext, div)
        assert np.array_equal(nodes, m.nodes) and np.array_equal(elems, m.elements)
        comps = 1 if trial % 4 < 2 else d
        rr = ref.Routing(m, comps)
        pr = port.Routing(rr.N, port.dofmap(kind, elems, comps))
        for key in ["offsets", "cols", "mat_offsets", "mat_slots", "vec_offsets", "vec_slots"]:
            assert np.array_equal(getattr(pr, key), getattr(rr, key)), (trial, key)
        if comps == 1:
            rho = 0.5 + rng.uniform(m.E)
            src = rng.uniform(m.E) - 0.5
            kw = dict(diffusion=("element", rho), sources=[("element", src)], with_mass=True)
        else:
            kw = dict(problem="elasticity", lam=0.5 + rng.uniform(1)[0], mu=0.3 + rng.uniform(1)[0],
                      sources=[0.25, -1.0, 2.0][:d])
        a = ref.assemble(m, rr, **kw)
        b = port.assemble(kind, nodes, elems, pr, **kw)
        for x, y in zip(a, b):
            if x is not None:
                assert_bitwise(y, x, f"trial {trial}")


def test_reference_errors():
    with pytest.raises(port.OracleError, match="divisions"):
        port.generate_grid("tri3", [1, 1], [0, 2])
    nodes = np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 0.0]])  # clockwise: det < 0
    with pytest.raises(port.OracleError, match="element 0 has non-positive Jacobian"):
        port.local("tri3", nodes, np.array([[0, 1, 2]]), 1, port.DIFFUSION, np.ones(1))


def _simp_case():
    nodes, elems = port.generate_grid("tet4", [1.0, 0.8, 1.2], [3, 2, 3])
    E = elems.shape[0]
    rng = np.random.default_rng(12)
    lam = np.full(E, 0.5769230769230769)
    mu = np.full(E, 0.38461538461538464)
    K0 = port.local("tet4", nodes, elems, 1, port.ELASTICITY, lam, mu)
    U = rng.standard_normal(nodes.shape[0] * 3)
    rho = 0.05 + 0.95 * rng.random(E)
    return nodes, elems, K0, U, rho


@pytest.mark.parametrize("p", [3.0, 2.5])
def test_simp_sensitivity_restatement_vs_reference(p):
    """port.simp_sensitivity against the unmodified reference library's
    simp_sensitivity (adjoint.cpp:101-125), bitwise, on TET4 elasticity DoFs."""
    ref = _ref()
    nodes, elems, K0, U, rho = _simp_case()
    dm = port.dofmap("tet4", elems, 3)
    got = port.simp_sensitivity(dm, rho, p, 1e-9, 1.0, K0, U)
    rm = ref.Mesh.from_arrays("tet4", nodes, elems)
    rr = ref.Routing(rm, 3)
    assert_bitwise(got, rr.simp_sensitivity(rho, p, 1e-9, 1.0, K0, U), f"simp_sensitivity p={p}")
