"""GPU parity: the CUDA path through the C ABI vs the oracle restatement and the
golden fixtures from the reference.  Bar: bit-exact for pattern/slot map/index
work; CSR values bit-exact in the exact arithmetic mode (stronger than the
north-star's 1e-12 scaled tolerance, which the fast mode is held to)."""
import glob
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import port  # noqa: E402
from tests._util import MT64, assert_bitwise, assert_scaled_close  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GOLDEN = sorted(glob.glob(os.path.join(GOLD, "mesh_*.npz")))


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_05052_b200 import engine
    return engine


def kind_of(nodes):
    return "tet4" if nodes.shape[1] == 3 else "tri3"


def np_(t):
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------ routing
@pytest.mark.parametrize("path", GOLDEN)
def test_routing_bit_exact_golden(eng, path):
    g = dict(np.load(path))
    kind = kind_of(g["nodes"])
    m = eng.DeviceMesh(kind, g["nodes"], g["elements"])
    r = eng.Routing(m, 1, segments=True)
    h = r.host_arrays()
    for key in ["offsets", "cols", "vec_offsets", "vec_slots", "mat_offsets", "mat_slots"]:
        assert np.array_equal(h[key], g[key]), key
    # slot_of is the inverse of mat_slots
    inv = np.empty(h["mat_slots"].size, np.int64)
    inv[h["mat_slots"].astype(np.int64)] = np.repeat(np.arange(r.nnz), np.diff(h["mat_offsets"].astype(np.int64)))
    assert np.array_equal(h["slot_of"].astype(np.int64), inv)
    d = g["nodes"].shape[1]
    rv = eng.Routing(m, d, segments=True)
    hv = rv.host_arrays()
    assert np.array_equal(hv["offsets"], g["v_offsets"]) and np.array_equal(hv["cols"], g["v_cols"])
    assert np.array_equal(hv["mat_offsets"], g["v_mat_offsets"])
    assert np.array_equal(hv["mat_slots"], g["v_mat_slots"])


@pytest.mark.parametrize("kind,div", [("tri3", [64, 45]), ("tet4", [14, 9, 11]), ("tet4", [30, 30, 30])])
def test_routing_bit_exact_vs_oracle(eng, kind, div):
    ext = [1.0] * len(div)
    nodes, elems = port.generate_grid(kind, ext, div)
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1, segments=True)
    h = r.host_arrays()
    pr = port.Routing(nodes.shape[0], port.dofmap(kind, elems, 1))
    for key in ["offsets", "cols", "vec_offsets", "vec_slots", "mat_offsets", "mat_slots"]:
        assert np.array_equal(h[key], getattr(pr, key)), key
    assert np.array_equal(h["slot_of"].astype(np.int64), pr.slot_of())


def test_routing_permuted_unstructured(eng):
    """Random node/element permutation (C4-style input): pattern still bit-exact."""
    rng = np.random.default_rng(44)
    nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [40, 40])
    pn = rng.permutation(nodes.shape[0])
    inv = np.argsort(pn)
    nodes = nodes[pn]
    elems = inv[elems][rng.permutation(elems.shape[0])]
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1, segments=True)
    h = r.host_arrays()
    pr = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
    for key in ["offsets", "cols", "vec_slots", "mat_offsets", "mat_slots"]:
        assert np.array_equal(h[key], getattr(pr, key)), key


# ------------------------------------------------------------------ stage I
@pytest.mark.parametrize("kind,div", [("tri3", [9, 7]), ("tet4", [4, 3, 5])])
@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_local_tensors_bit_exact(eng, kind, div, degree):
    rng = np.random.default_rng(degree)
    nodes, elems = port.generate_grid(kind, [1.0, 0.8, 1.3][: len(div)], div)
    nodes = nodes + 0.01 * rng.random(nodes.shape)  # non-uniform elements
    m = eng.DeviceMesh(kind, nodes, elems)
    E = elems.shape[0]
    Q = port.tables(kind, degree)["Q"]
    d = nodes.shape[1]
    c = 0.5 + rng.random(E * Q)
    c2 = 0.5 + rng.random(E * Q)
    cv = rng.random(E * Q * d) - 0.5
    assert_bitwise(np_(eng.local_stiffness_diffusion(m, degree, c)),
                   port.local(kind, nodes, elems, degree, port.DIFFUSION, c), "diffusion")
    assert_bitwise(np_(eng.local_mass(m, degree, c)),
                   port.local(kind, nodes, elems, degree, port.MASS, c), "mass")
    assert_bitwise(np_(eng.local_load(m, degree, c)),
                   port.local(kind, nodes, elems, degree, port.LOAD, c), "load")
    assert_bitwise(np_(eng.local_load_vector(m, degree, cv)),
                   port.local(kind, nodes, elems, degree, port.LOAD_VECTOR, cv), "load_vector")
    assert_bitwise(np_(eng.local_stiffness_elasticity(m, degree, c, c2)),
                   port.local(kind, nodes, elems, degree, port.ELASTICITY, c, c2), "elasticity")
    geo = eng.geometry(m, degree)
    ref = port.geometry(kind, nodes, elems, degree)
    for key in ["jac", "det", "jac_invT", "qpts", "grads"]:
        assert_bitwise(np_(geo[key]), ref[key], key)
    nodal = rng.random(nodes.shape[0])
    f = port.Field(2, 0.0, nodal.ctypes.data, nodal.size)
    ev = np.zeros(E * Q)
    port.lib().tgo_evaluate(port.KINDS[kind], nodes.ctypes.data, np.ascontiguousarray(elems).ctypes.data,
                            E, nodes.shape[0], degree, port.C.byref(f), ev.ctypes.data)
    assert_bitwise(np_(eng.evaluate_field(m, degree, ("nodal", nodal))), ev, "nodal evaluate")


# ------------------------------------------------------------------ stage II + fused
@pytest.mark.parametrize("path", GOLDEN)
def test_reduce_and_fused_assemble_golden(eng, path):
    g = dict(np.load(path))
    kind = kind_of(g["nodes"])
    m = eng.DeviceMesh(kind, g["nodes"], g["elements"])
    r = eng.Routing(m, 1, segments=True)
    K, F, _ = eng.assemble(m, r, sources=[1.0])
    assert_bitwise(np_(K), g["K_const"], "K const")
    assert_bitwise(np_(F), g["F_const"], "F const")
    K, F, M = eng.assemble(m, r, diffusion=("element", g["rho"]), sources=[("element", g["src"])],
                           with_mass=True)
    assert_bitwise(np_(K), g["K_rho"], "K rho")
    assert_bitwise(np_(F), g["F_rho"], "F rho")
    assert_bitwise(np_(M), g["M_rho"], "M rho")
    K, F, _ = eng.assemble(m, r, diffusion=("nodal", g["nodal"]), sources=[("nodal", g["nodal"])])
    assert_bitwise(np_(K), g["K_nodal"], "K nodal")
    assert_bitwise(np_(F), g["F_nodal"], "F nodal")
    K, F, _ = eng.assemble(m, r, kind="mass", diffusion=("element", g["rho"]))
    assert_bitwise(np_(K), g["K_mass"], "K mass")
    assert not np_(F).any()
    # materialised Stage II on the reference's own local tensors
    K0 = g["K0_local"]
    assert_bitwise(np_(eng.reduce_matrix(r, K0)), port.Routing(r.N, port.dofmap(kind, g["elements"], 1)).reduce_matrix(K0))
    # elasticity
    d = g["nodes"].shape[1]
    rv = eng.Routing(m, d)
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=float(g["lam"]), mu=float(g["mu"]),
                           sources=[1.0] * d)
    assert_bitwise(np_(K), g["K_elast"], "K elasticity")
    assert_bitwise(np_(F), g["F_elast"], "F elasticity")


@pytest.mark.parametrize("kind,div", [("tri3", [120, 97]), ("tet4", [23, 17, 19]), ("tet4", [32, 32, 32])])
def test_fused_assemble_bit_exact_vs_oracle(eng, kind, div):
    rng = MT64(2024)
    nodes, elems = port.generate_grid(kind, [1.0, 1.2, 0.9][: len(div)], div)
    E, Nn = elems.shape[0], nodes.shape[0]
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(Nn, port.dofmap(kind, elems, 1))
    rho = 0.5 + np.random.default_rng(1).random(E)
    for kw in [dict(sources=[1.0]),
               dict(diffusion=("element", rho), sources=[1.0], with_mass=True),
               dict(diffusion=2.5, sources=[("element", rho)], with_mass=True)]:
        K, F, M = eng.assemble(m, r, **kw)
        Kr, Fr, Mr = port.assemble(kind, nodes, elems, pr, **kw)
        assert_bitwise(np_(K), Kr, f"K {kw.keys()}")
        assert_bitwise(np_(F), Fr, "F")
        if Mr is not None:
            assert_bitwise(np_(M), Mr, "M")
    del rng


def test_assemble_host_entry_matches_device(eng):
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [10, 8, 6])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    rho = 0.5 + np.random.default_rng(3).random(elems.shape[0])
    Kd, Fd, Md = eng.assemble(m, r, diffusion=("element", rho), sources=[1.0], with_mass=True)
    Kh, Fh, Mh = eng.assemble_host(m, r, diffusion=("element", rho), sources=[1.0], with_mass=True)
    assert_bitwise(Kh, np_(Kd))
    assert_bitwise(Fh, np_(Fd))
    assert_bitwise(Mh, np_(Md))


def test_run_to_run_determinism(eng):
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [20, 20, 20])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    a = [np_(x) for x in eng.assemble(m, r, sources=[1.0], with_mass=True)]
    for _ in range(3):
        b = [np_(x) for x in eng.assemble(m, r, sources=[1.0], with_mass=True)]
        for x, y in zip(a, b):
            assert_bitwise(x, y)


def test_elasticity_vs_oracle(eng):
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [6, 5, 7])
    m = eng.DeviceMesh("tet4", nodes, elems)
    rv = eng.Routing(m, 3)
    pr = port.Routing(nodes.shape[0] * 3, port.dofmap("tet4", elems, 3))
    lam = 0.5 + np.random.default_rng(5).random(elems.shape[0])
    kw = dict(kind="elasticity", lam=("element", lam), mu=0.384615, sources=[1.0, -2.0, 0.5])
    K, F, _ = eng.assemble(m, rv, **kw)
    kw2 = dict(kw)
    kw2["problem"] = kw2.pop("kind")
    Kr, Fr, _ = port.assemble("tet4", nodes, elems, pr, **kw2)
    assert_bitwise(np_(K), Kr)
    assert_bitwise(np_(F), Fr)
    # 2D plane stress
    nodes, elems = port.generate_grid("tri3", [2.0, 1.0], [12, 7])
    m = eng.DeviceMesh("tri3", nodes, elems)
    rv = eng.Routing(m, 2)
    pr = port.Routing(nodes.shape[0] * 2, port.dofmap("tri3", elems, 2))
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=1.2, mu=0.8, plane_stress=True, sources=[0.0, -1.0])
    Kr, Fr, _ = port.assemble("tri3", nodes, elems, pr, problem="elasticity", lam=1.2, mu=0.8,
                              plane_stress=True, sources=[0.0, -1.0])
    assert_bitwise(np_(K), Kr)
    assert_bitwise(np_(F), Fr)


# ------------------------------------------------------------------ batched + adjoint
def test_batched_equals_single_field(eng):
    nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [30, 30])
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
    rng = np.random.default_rng(1000)
    B = 5
    rho = 0.5 + rng.random((B, elems.shape[0]))
    K, F = eng.assemble_batched(m, r, rho, source=1.0)
    for b in range(B):
        Kr, Fr, _ = port.assemble("tri3", nodes, elems, pr, diffusion=("element", rho[b]), sources=[1.0])
        assert_bitwise(np_(K[b]), Kr, f"field {b}")
        if b == 0:
            assert_bitwise(np_(F), Fr)


@pytest.mark.parametrize("path", GOLDEN)
def test_gradient_products_and_adjoint_golden(eng, path):
    g = dict(np.load(path))
    kind = kind_of(g["nodes"])
    m = eng.DeviceMesh(kind, g["nodes"], g["elements"])
    r = eng.Routing(m, 1)
    dK, dF = eng.gradient_products(r, g["adj_lambda"], g["adj_U"])
    assert_bitwise(np_(dK[0]), g["dK"])
    assert_bitwise(np_(dF[0]), g["dF"])
    dm = port.dofmap(kind, g["elements"], 1)
    want = port.adjoint_gather(dm, g["K0_local"], g["adj_lambda"], g["adj_U"])
    got = eng.adjoint_gather(m, r, g["adj_lambda"], g["adj_U"], degree=1)
    assert_bitwise(np_(got[0]), want)


def test_batched_adjoint_vs_oracle(eng):
    nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [24, 20])
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1)
    Nn, E = nodes.shape[0], elems.shape[0]
    rng = np.random.default_rng(2000)
    B = 19  # not a multiple of the per-block field count
    lam = rng.random((B, Nn)) - 0.5
    U = rng.random((B, Nn)) - 0.5
    got = np_(eng.adjoint_gather(m, r, lam, U, degree=1))
    dm = port.dofmap("tri3", elems, 1)
    K0 = port.local("tri3", nodes, elems, 1, port.DIFFUSION, np.ones(E))
    for b in range(B):
        assert_bitwise(got[b], port.adjoint_gather(dm, K0, lam[b], U[b]), f"field {b}")


@pytest.mark.parametrize("kind,degree,env", [
    ("tri3", 2, {}), ("tet4", 1, {}), ("tet4", 2, {"TGK_ADJ_FPB": "3"}),
    ("tri3", 1, {"TGK_ADJ_FLAT": "1"}), ("tet4", 2, {"TGK_ADJ_FLAT": "1"}),
    ("unstructured", 1, {"TGK_ADJ_FPB": "1"}),
])
def test_adjoint_paths_vs_oracle(eng, monkeypatch, kind, degree, env):
    """Grouped (default) and flat transpose gathers, bit-exact per field."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if kind == "unstructured":
        from paper_2602_05052_b200 import meshgen
        kind = "tri3"
        nodes, elems = meshgen.unstructured_tri(40)
    elif kind == "tri3":
        nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [33, 29])
    else:
        nodes, elems = port.generate_grid("tet4", [1.0] * 3, [7, 6, 8])
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1)
    Nn, E = nodes.shape[0], elems.shape[0]
    rng = np.random.default_rng(2100)
    B = 7
    lam = rng.random((B, Nn)) - 0.5
    U = rng.random((B, Nn)) - 0.5
    got = np_(eng.adjoint_gather(m, r, lam, U, degree=degree))
    dm = port.dofmap(kind, elems, 1)
    K0 = port.local(kind, nodes, elems, degree, port.DIFFUSION, np.ones(E * port.tables(kind, degree)["Q"]))
    for b in range(B):
        assert_bitwise(got[b], port.adjoint_gather(dm, K0, lam[b], U[b]), f"field {b}")


# ------------------------------------------------------------------ errors
def test_errors(eng):
    from paper_2602_05052_b200 import InputError
    nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [4, 4])
    bad = elems.copy()
    bad[[5, 9]] = bad[[5, 9]][:, [0, 2, 1]]  # flip two elements: smallest index reported
    m = eng.DeviceMesh("tri3", nodes, bad)
    r = eng.Routing(m, 1)
    with pytest.raises(InputError, match="element 5 has non-positive Jacobian determinant"):
        eng.assemble(m, r, sources=[1.0])
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1)
    with pytest.raises(InputError, match="per-element coefficient"):
        eng.assemble(m, r, diffusion=("element", np.ones(3)))
    with pytest.raises(InputError, match="component count"):
        eng.assemble(m, r, kind="elasticity")
    rv = eng.Routing(m, 2)
    with pytest.raises(InputError, match="mu > 0"):
        eng.assemble(m, rv, kind="elasticity", mu=0.0)
    with pytest.raises(InputError, match="one component per dimension"):
        eng.assemble(m, rv, kind="elasticity", sources=[1.0])
    with pytest.raises(InputError, match="only supported for scalar"):
        eng.assemble(m, rv, kind="elasticity", with_mass=True)


# ------------------------------------------------------------------ drop-in module
def test_tgfem_dropin_matches_reference_smoke(eng):
    """proj/tests/test_python_smoke.py:18-26 against our module."""
    from paper_2602_05052_b200 import tgfem
    mesh = tgfem.generate_grid("tri3", [1.0, 1.0], [3, 3])
    local = tgfem.local_stiffness(mesh)
    assert local.shape == (18, 3, 3)
    g = dict(np.load(os.path.join(GOLD, "mesh_tri3_3x3.npz")))
    assert_bitwise(local, g["K0_local"])
    reduced = tgfem.reduce_matrix(mesh, local)
    oracle = tgfem.scatter_add_oracle(mesh, local)
    assert (reduced["values"] == oracle["values"]).all()
    assert (reduced["cols"] == g["cols"]).all() and (reduced["offsets"] == g["offsets"]).all()
    assert_bitwise(reduced["values"], g["K_const"])
    rho = g["rho"]
    lk = tgfem.local_stiffness(mesh, rho)
    assert_bitwise(lk, port.local("tri3", mesh.nodes, mesh.elements, 1, port.DIFFUSION, rho))


# ------------------------------------------------------------------ full-size properties (C2)
def test_c2_size_properties(eng):
    """TET4 Kuhn 100^3 (6M tets): size-independent invariants of the fused output."""
    from paper_2602_05052_b200 import tgfem
    mesh = tgfem.generate_grid("tet4", [1.0, 1.0, 1.0], [100, 100, 100])
    m = eng.DeviceMesh("tet4", mesh.nodes, mesh.elements)
    r = eng.Routing(m, 1)
    assert r.nnz == 15210901 and r.N == 1030301
    K, F, M = eng.assemble(m, r, sources=[1.0], with_mass=True)
    h = r.host_arrays(slot_of=False)
    rows = np.repeat(np.arange(r.N), np.diff(h["offsets"]))
    Kn, Fn, Mn = np_(K), np_(F), np_(M)
    # stiffness annihilates constants; mass sums to the volume; load sums to volume * f
    rowsum = np.bincount(rows, weights=Kn, minlength=r.N)
    assert np.abs(rowsum).max() <= 1e-12 * np.abs(Kn).max()
    assert abs(Mn.sum() - 1.0) < 1e-10
    assert abs(Fn.sum() - 1.0) < 1e-10
    # stiffness is bitwise symmetric (K_e symmetric, same fold order)
    perm = np.lexsort((rows, h["cols"]))  # (col,row) order = transpose
    assert_bitwise(Kn[perm], Kn[np.lexsort((h["cols"], rows))])


@pytest.mark.parametrize("scale", [2.0 ** -30, 1e-15, 3.0e12])
def test_division_paths_bit_exact(eng, scale):
    """Certified meshes use the Markstein division, uncertified ones (tiny or huge
    coordinates) IEEE division; both must reproduce the reference bit for bit."""
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [7, 6, 5])
    nodes = nodes * scale + 0.37 * scale
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    rho = 0.5 + np.random.default_rng(9).random(elems.shape[0])
    K, F, M = eng.assemble(m, r, diffusion=("element", rho), sources=[1.0], with_mass=True)
    Kr, Fr, Mr = port.assemble("tet4", nodes, elems, pr, diffusion=("element", rho), sources=[1.0],
                               with_mass=True)
    assert_bitwise(np_(K), Kr)
    assert_bitwise(np_(F), Fr)
    assert_bitwise(np_(M), Mr)
