"""GPU parity of the fast mode (TGK_MODE_FAST, csrc/fast.cu + csrc/plan_fast.cpp).

The north star's contract: CSR pattern bit-exact (the fast
mode shares the routing), values within |dv| <= 1e-12 |v_ref| + 1e-14 max|v_ref|
against the reference (oracle restatement or the unmodified reference library
oracle/_ref/libtgref.so), and run-to-run bitwise determinism.

Reference semantics: tg::assemble (proj/src/physics.cpp:10-75) with the local
kernels of proj/src/batch.cpp:156-289 and reduce_matrix/reduce_vector
(proj/src/routing.cpp:87-132).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import port  # noqa: E402
from tests._util import assert_bitwise, assert_scaled_close  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_05052_b200 import engine
    return engine


def np_(t):
    return t.detach().cpu().numpy()


def permuted(nodes, elems, seed):
    rng = np.random.default_rng(seed)
    pn = rng.permutation(nodes.shape[0])
    inv = np.argsort(pn)
    return nodes[pn], inv[elems][rng.permutation(elems.shape[0])]


def meshes():
    from paper_2602_05052_b200 import meshgen
    yield "tri3-grid", "tri3", *port.generate_grid("tri3", [1.0, 1.3], [83, 61])
    yield "tet4-grid", "tet4", *port.generate_grid("tet4", [1.0, 0.8, 1.1], [19, 14, 17])
    yield "tri3-unstructured", "tri3", *meshgen.unstructured_tri(64)
    yield "tet4-permuted", "tet4", *permuted(*port.generate_grid("tet4", [1.0, 1.0, 1.0], [11, 9, 10]), 5)


CASES = [
    ("K+F", dict(sources=[1.0])),
    ("K", dict()),
    ("K+M+F", dict(sources=[1.0], with_mass=True)),
    ("K(2.5)+M", dict(diffusion=2.5, with_mass=True)),
    ("elem K+F(elem)+M", "elem"),
    ("nodal K+F(nodal)", "nodal"),
    ("nodal K+F(const)+M", "nodal-m"),
    ("mass(const)", dict(problem="mass", diffusion=1.7)),
    ("mass(elem)", "mass-elem"),
    ("mass(nodal) -> exact kernel", "mass-nodal"),
]


def _kw(case, E, Nn):
    rng = np.random.default_rng(7)
    rho, nod = 0.5 + rng.random(E), 0.5 + rng.random(Nn)
    if isinstance(case, dict):
        return dict(case)
    return {
        "elem": dict(diffusion=("element", rho), sources=[("element", rho)], with_mass=True),
        "nodal": dict(diffusion=("nodal", nod), sources=[("nodal", nod)]),
        "nodal-m": dict(diffusion=("nodal", nod), sources=[2.0], with_mass=True),
        "mass-elem": dict(problem="mass", diffusion=("element", rho)),
        "mass-nodal": dict(problem="mass", diffusion=("nodal", nod)),
    }[case]


@pytest.mark.parametrize("name,kind,nodes,elems", list(meshes()), ids=[m[0] for m in meshes()])
def test_fast_within_tolerance_vs_oracle(eng, name, kind, nodes, elems):
    E, Nn = elems.shape[0], nodes.shape[0]
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(Nn, port.dofmap(kind, elems, 1))
    for label, case in CASES:
        kw = _kw(case, E, Nn)
        problem = kw.pop("problem", "poisson")
        K, F, M = eng.assemble(m, r, kind=problem, mode="fast", **kw)
        Kr, Fr, Mr = port.assemble(kind, nodes, elems, pr, problem=problem, **kw)
        assert_scaled_close(np_(K), Kr, what=f"{name} {label} K")
        assert_scaled_close(np_(F), Fr, what=f"{name} {label} F")
        if Mr is not None and problem != "mass":
            assert_scaled_close(np_(M), Mr, what=f"{name} {label} M")
        # deterministic: a second run is bitwise identical
        K2, F2, M2 = eng.assemble(m, r, kind=problem, mode="fast", **kw)
        assert_bitwise(np_(K2), np_(K), f"{name} {label} K rerun")
        assert_bitwise(np_(F2), np_(F), f"{name} {label} F rerun")


@pytest.mark.parametrize("R", ["32", "64", "128", "200"])
@pytest.mark.parametrize("kind,div", [("tet4", [23, 19, 21]), ("tri3", [150, 131])])
def test_fast_rows_per_block(eng, monkeypatch, R, kind, div):
    """Every rows-per-block choice of the fast plan (TGK_FAST_R) meets the tolerance."""
    monkeypatch.setenv("TGK_FAST_R", R)
    nodes, elems = port.generate_grid(kind, [1.0, 1.1, 0.9][: len(div)], div)
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap(kind, elems, 1))
    for kw in [dict(sources=[1.0]), dict(sources=[1.0], with_mass=True)]:
        K, F, M = eng.assemble(m, r, mode="fast", **kw)
        Kr, Fr, Mr = port.assemble(kind, nodes, elems, pr, **kw)
        assert_scaled_close(np_(K), Kr, what=f"R={R} K")
        assert_scaled_close(np_(F), Fr, what=f"R={R} F")
        if Mr is not None:
            assert_scaled_close(np_(M), Mr, what=f"R={R} M")


def test_fast_c1_full_size(eng):
    nodes, elems = port.generate_grid("tri3", [1.0, 1.0], [256, 256])
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
    K, F, _ = eng.assemble(m, r, mode="fast", sources=[1.0])
    Kr, Fr, _ = port.assemble("tri3", nodes, elems, pr, sources=[1.0])
    assert_scaled_close(np_(K), Kr, what="C1 K")
    assert_scaled_close(np_(F), Fr, what="C1 F")


@pytest.mark.slow
def test_fast_c2_c2a_full_size_vs_reference_library(eng):
    """C2 (K+M+F) and C2a (K+F) on the 6M-tet Kuhn cube in fast mode against the
    unmodified reference library's tg::assemble (oracle/_ref/libtgref.so)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref/libtgref.so not built")
    ref.set_threads(0)
    rm = ref.Mesh.grid("tet4", [1.0, 1.0, 1.0], [100, 100, 100])
    rr = ref.Routing(rm, 1)
    m = eng.DeviceMesh("tet4", *port.generate_grid("tet4", [1.0] * 3, [100] * 3))
    r = eng.Routing(m, 1)
    for kw in [dict(sources=[1.0], with_mass=True), dict(sources=[1.0])]:
        K, F, M = eng.assemble(m, r, mode="fast", **kw)
        Kr, Fr, Mr = ref.assemble(rm, rr, **kw)
        assert_scaled_close(np_(K), Kr, what=f"K {sorted(kw)}")
        assert_scaled_close(np_(F), Fr, what=f"F {sorted(kw)}")
        if Mr is not None:
            assert_scaled_close(np_(M), Mr, what="M")
        K2, _, _ = eng.assemble(m, r, mode="fast", **kw)
        assert torch.equal(K.view(torch.int64), K2.view(torch.int64))


def test_fast_restricted_rows_and_elements(eng):
    """Owned-row partitions (halo mode) and element-range slabs (exchange mode)
    in fast mode: the owned rows agree with the exact kernel within tolerance and
    the rows outside are left untouched."""
    from paper_2602_05052_b200 import _native as N
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [12, 10, 14])
    m = eng.DeviceMesh("tet4", nodes, elems)
    Nn, E = nodes.shape[0], elems.shape[0]
    for setter, lo, hi in [("tgk_routing_set_owned_rows", Nn // 3, 2 * Nn // 3),
                           ("tgk_routing_set_element_range", E // 4, 3 * E // 4)]:
        r = eng.Routing(m, 1)
        N.check(getattr(N.lib(), setter)(r._h, lo, hi))
        out = []
        for mode in ["exact", "fast"]:
            K = torch.full((r.nnz,), 7.0, dtype=torch.float64, device="cuda")
            F = torch.full((r.N,), 7.0, dtype=torch.float64, device="cuda")
            M = torch.full((r.nnz,), 7.0, dtype=torch.float64, device="cuda")
            eng.assemble(m, r, sources=[1.0], with_mass=True, mode=mode, out=(K, F, M))
            out.append((np_(K), np_(F), np_(M)))
        for a, b, what in zip(out[0], out[1], "KFM"):
            untouched = a == 7.0
            assert np.array_equal(untouched, b == 7.0), f"{setter} {what}: written set differs"
            assert_scaled_close(b[~untouched], a[~untouched], what=f"{setter} {what}")


def test_fast_errors(eng):
    """The smallest inverted element is reported with the reference's message (batch.cpp:124-126)."""
    from paper_2602_05052_b200 import InputError
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [4, 4, 4])
    bad = elems.copy()
    bad[[5, 9]] = bad[[5, 9]][:, [1, 0, 2, 3]]  # inverted elements 5 and 9
    m = eng.DeviceMesh("tet4", nodes, bad)
    r = eng.Routing(m, 1)
    with pytest.raises(InputError, match="element 5 has non-positive Jacobian determinant"):
        eng.assemble(m, r, sources=[1.0], mode="fast")


@pytest.mark.parametrize("kind,mesh,kw", [
    ("tet4", "grid", dict(sources=[1.0, 1.0, 1.0])),
    ("tet4", "permuted", dict(sources=[0.5, -1.0, 2.0])),
    ("tet4", "grid", dict()),
    ("tri3", "grid", dict(sources=[1.0, -0.5])),
    ("tri3", "unstructured", dict(plane_stress=True, sources=[1.0, 1.0])),
], ids=["tet-grid-f", "tet-permuted-f", "tet-grid-nof", "tri-grid-f", "tri-unstructured-planestress"])
def test_fast_elasticity_vs_oracle(eng, kind, mesh, kw):
    """Fast-mode vector elasticity (k_fast_elast): 3x3 / 2x2 blocks on the
    scalar fast plan, within the scaled tolerance of local_stiffness_elasticity
    + reduce_matrix (batch.cpp:183-248, routing.cpp:109-132)."""
    from paper_2602_05052_b200 import meshgen
    if mesh == "unstructured":
        nodes, elems = meshgen.unstructured_tri(40)
    elif mesh == "permuted":
        nodes, elems = permuted(*port.generate_grid("tet4", [1.0, 1.2, 0.8], [8, 7, 9]), 3)
    else:
        nodes, elems = port.generate_grid(kind, [1.0, 1.1, 0.9][: 3 if kind == "tet4" else 2],
                                          [9, 8, 7] if kind == "tet4" else [31, 27])
    d = 3 if kind == "tet4" else 2
    m = eng.DeviceMesh(kind, nodes, elems)
    rv = eng.Routing(m, d)
    prv = port.Routing(nodes.shape[0] * d, port.dofmap(kind, elems, d))
    lam, mu = 0.5769230769230769, 0.38461538461538464
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=lam, mu=mu, mode="fast", **kw)
    Kr, Fr, _ = port.assemble(kind, nodes, elems, prv, problem="elasticity", lam=lam, mu=mu, **kw)
    assert_scaled_close(np_(K), Kr, what="elasticity K")
    assert_scaled_close(np_(F), Fr, what="elasticity F")
    K2, F2, _ = eng.assemble(m, rv, kind="elasticity", lam=lam, mu=mu, mode="fast", **kw)
    assert_bitwise(np_(K2), np_(K), "elasticity rerun")


def test_fast_elasticity_c3_30(eng):
    """C3's fast kernel on a 30^3 Kuhn cube (162k tets, 3 DoF/node)."""
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [30, 30, 30])
    m = eng.DeviceMesh("tet4", nodes, elems)
    rv = eng.Routing(m, 3)
    pr = port.Routing(nodes.shape[0] * 3, port.dofmap("tet4", elems, 3))
    lam, mu = 0.5769230769230769, 0.38461538461538464
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=lam, mu=mu, sources=[1.0, 1.0, 1.0], mode="fast")
    Kr, Fr, _ = port.assemble("tet4", nodes, elems, pr, problem="elasticity", lam=lam, mu=mu,
                              sources=[1.0, 1.0, 1.0])
    assert_scaled_close(np_(K), Kr, what="C3 K")
    assert_scaled_close(np_(F), Fr, what="C3 F")


def _elast_fields(kind, E, variant):
    rng = np.random.default_rng(11)
    lam_e = ("element", 0.3 + rng.random(E))
    mu_e = ("element", 0.2 + rng.random(E))
    d = 3 if kind == "tet4" else 2
    f_e = [("element", rng.standard_normal(E)) for _ in range(d)]
    return {
        "lam+mu elem, F elem": dict(lam=lam_e, mu=mu_e, sources=f_e),
        "lam elem, mu const, F mixed": dict(lam=lam_e, mu=0.4, sources=[1.0] + f_e[1:]),
        "lam const, mu elem, F const": dict(lam=0.6, mu=mu_e, sources=[0.5] * d),
        "lam+mu elem, no F": dict(lam=lam_e, mu=mu_e),
    }[variant]


@pytest.mark.parametrize("variant", ["lam+mu elem, F elem", "lam elem, mu const, F mixed",
                                     "lam const, mu elem, F const", "lam+mu elem, no F"])
@pytest.mark.parametrize("kind,mesh,ps", [("tet4", "permuted", False), ("tri3", "unstructured", True),
                                          ("tri3", "grid", False)])
def test_fast_elasticity_element_fields(eng, kind, mesh, ps, variant):
    """k_fast_elast with per-element Lame parameters (plane-stress transform per
    element, batch.cpp:359-361) and per-element body force, vs the oracle
    (batch.cpp:183-269) within the SURVEY.md 8(c) tolerance; deterministic."""
    from paper_2602_05052_b200 import meshgen
    if mesh == "unstructured":
        nodes, elems = meshgen.unstructured_tri(40)
    elif mesh == "permuted":
        nodes, elems = permuted(*port.generate_grid("tet4", [1.0, 1.2, 0.8], [8, 7, 9]), 3)
    else:
        nodes, elems = port.generate_grid("tri3", [1.0, 1.1], [31, 27])
    d = 3 if kind == "tet4" else 2
    kw = _elast_fields(kind, elems.shape[0], variant)
    m = eng.DeviceMesh(kind, nodes, elems)
    rv = eng.Routing(m, d)
    prv = port.Routing(nodes.shape[0] * d, port.dofmap(kind, elems, d))
    K, F, _ = eng.assemble(m, rv, kind="elasticity", plane_stress=ps, mode="fast", **kw)
    Kr, Fr, _ = port.assemble(kind, nodes, elems, prv, problem="elasticity", plane_stress=ps, **kw)
    assert_scaled_close(np_(K), Kr, what="elasticity K")
    assert_scaled_close(np_(F), Fr, what="elasticity F")
    K2, F2, _ = eng.assemble(m, rv, kind="elasticity", plane_stress=ps, mode="fast", **kw)
    assert_bitwise(np_(K2), np_(K), "rerun K")
    assert_bitwise(np_(F2), np_(F), "rerun F")


def test_fast_elasticity_element_errors(eng):
    """mu <= 0 in a per-element field -> 'elasticity requires mu > 0' (batch.cpp:194-195);
    an inverted element is reported first (batch_geometry runs before the Lame check)."""
    from paper_2602_05052_b200._native import InputError
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [4, 4, 4])
    E = elems.shape[0]
    mu = np.full(E, 0.4)
    mu[17] = 0.0
    m = eng.DeviceMesh("tet4", nodes, elems)
    rv = eng.Routing(m, 3)
    with pytest.raises(InputError, match="mu > 0"):
        eng.assemble(m, rv, kind="elasticity", lam=0.5, mu=("element", mu), mode="fast")
    bad = elems.copy()
    bad[[5, 9]] = bad[[5, 9]][:, [1, 0, 2, 3]]
    mb = eng.DeviceMesh("tet4", nodes, bad)
    rb = eng.Routing(mb, 3)
    with pytest.raises(InputError, match="element 5 has non-positive Jacobian determinant"):
        eng.assemble(mb, rb, kind="elasticity", lam=0.5, mu=("element", mu), mode="fast")


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("problem", ["poisson K+M+F", "mass", "elasticity"])
def test_fields_batched(eng, mode, problem):
    """tgk_assemble_fields_batched_d: batch member b equals the single-field
    assembly with the slots set to row b (bitwise: same kernels), and the
    oracle (exact: bitwise; fast: scaled tolerance)."""
    from paper_2602_05052_b200 import meshgen
    rng = np.random.default_rng(3)
    B = 3
    if problem == "elasticity":
        kind = "tet4"
        nodes, elems = permuted(*port.generate_grid("tet4", [1.0, 1.0, 1.0], [6, 7, 5]), 2)
        d, E = 3, elems.shape[0]
        fields = {"lam": 0.3 + rng.random((B, E)), "mu": 0.2 + rng.random((B, E)),
                  "source1": rng.standard_normal((B, E))}
        base = dict(kind="elasticity", lam=1.0, mu=1.0, sources=[1.0, 0.0, -1.0])
    else:
        kind = "tri3"
        nodes, elems = meshgen.unstructured_tri(48)
        d, E = 1, elems.shape[0]
        fields = {"diffusion": 0.5 + rng.random((B, E))}
        base = dict(kind="mass") if problem == "mass" else dict(kind="poisson", sources=[1.0], with_mass=True)
        if problem != "mass":
            fields["source0"] = rng.standard_normal((B, E))
    m = eng.DeviceMesh(kind, nodes, elems)
    rv = eng.Routing(m, d)
    prv = port.Routing(nodes.shape[0] * d, port.dofmap(kind, elems, d))
    K, F, M = eng.assemble_fields_batched(m, rv, {k: torch.from_numpy(v) for k, v in fields.items()},
                                          mode=mode, **base)
    assert K.shape == (B, rv.nnz) and F.shape == (B, rv.N)
    assert (M is not None) == (problem == "poisson K+M+F")
    for b in range(B):
        kw = dict(base)
        srcs = list(kw.pop("sources", ()))
        kwb = {}
        for slot, v in fields.items():
            if slot.startswith("source"):
                srcs[int(slot[-1])] = ("element", v[b])
            else:
                kwb[slot] = ("element", v[b])
                kw.pop(slot, None)
        Kb, Fb, Mb = eng.assemble(m, rv, sources=srcs, mode=mode, **kw, **kwb)
        assert_bitwise(np_(K[b]), np_(Kb), f"member {b} K")
        assert_bitwise(np_(F[b]), np_(Fb), f"member {b} F")
        if M is not None:
            assert_bitwise(np_(M[b]), np_(Mb), f"member {b} M")
        pk = dict(kw)
        pk["problem"] = pk.pop("kind")
        Kr, Fr, Mr = port.assemble(kind, nodes, elems, prv, sources=srcs, **pk, **kwb)
        check = assert_bitwise if mode == "exact" else (lambda a, b_, w: assert_scaled_close(a, b_, what=w))
        check(np_(Kb), Kr, f"member {b} K vs oracle")
        check(np_(Fb), Fr, f"member {b} F vs oracle")
        if M is not None:
            check(np_(Mb), Mr, f"member {b} M vs oracle")


def test_assemble_batched_fast_mode(eng):
    """tgk_assemble_batched_d accepts TGK_MODE_FAST and runs the batched exact
    kernels (their bit-identical results meet the fast contract; the fast
    batched variants measured slower, profiles/r02_fast_experiments.txt)."""
    from paper_2602_05052_b200 import meshgen
    nodes, elems = meshgen.unstructured_tri(48)
    rho = 1e-3 + np.random.default_rng(4).random((13, elems.shape[0]))
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1)
    rt = torch.from_numpy(rho)
    K, F = eng.assemble_batched(m, r, rt, source=1.0, mode="fast")
    Kx, Fx = eng.assemble_batched(m, r, rt, source=1.0, mode="exact")
    assert_bitwise(np_(K), np_(Kx), "K")
    assert_bitwise(np_(F), np_(Fx), "F")


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_isolated_nodes_and_tiny_meshes(eng, mode):
    """Edge cases the reference accepts: nodes referenced by no element (empty
    CSR rows, F_i = 0), a single element, and a mesh whose rows fit one block."""
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [3, 2, 2])
    extra = np.array([[5.0, 5.0, 5.0], [6.0, 5.0, 5.0]])
    nodes2 = np.vstack([nodes[:7], extra, nodes[7:]])  # two isolated nodes in the middle of the numbering
    remap = np.where(np.arange(nodes.shape[0]) >= 7, np.arange(nodes.shape[0]) + 2, np.arange(nodes.shape[0]))
    elems2 = remap[elems]
    one_n = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    one_e = np.array([[0, 1, 2, 3]])
    for nn, ee in [(nodes2, elems2), (one_n, one_e)]:
        m = eng.DeviceMesh("tet4", nn, ee)
        r = eng.Routing(m, 1)
        pr = port.Routing(nn.shape[0], port.dofmap("tet4", ee, 1))
        for kw in [dict(sources=[1.0]), dict(sources=[2.0], with_mass=True)]:
            K, F, M = eng.assemble(m, r, mode=mode, **kw)
            Kr, Fr, Mr = port.assemble("tet4", nn, ee, pr, **kw)
            pairs = [(K, Kr, "K"), (F, Fr, "F")] + ([(M, Mr, "M")] if kw.get("with_mass") else [])
            for g, w, what in pairs:
                if mode == "exact":
                    assert_bitwise(np_(g), w, what)
                else:
                    assert_scaled_close(np_(g), w, what=what)


def test_fast_elasticity_isolated_nodes(eng):
    """Fast elasticity with two nodes referenced by no element: empty vector rows
    and zero loads there, the rest within the tolerance of the oracle."""
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [3, 2, 2])
    extra = np.array([[5.0, 5.0, 5.0], [6.0, 5.0, 5.0]])
    nn = np.vstack([nodes[:7], extra, nodes[7:]])
    remap = np.where(np.arange(nodes.shape[0]) >= 7, np.arange(nodes.shape[0]) + 2, np.arange(nodes.shape[0]))
    ee = remap[elems]
    m = eng.DeviceMesh("tet4", nn, ee)
    rv = eng.Routing(m, 3)
    pr = port.Routing(nn.shape[0] * 3, port.dofmap("tet4", ee, 3))
    kw = dict(lam=0.5769230769230769, mu=0.38461538461538464, sources=[1.0, 0.5, -1.0])
    K, F, _ = eng.assemble(m, rv, kind="elasticity", mode="fast", **kw)
    Kr, Fr, _ = port.assemble("tet4", nn, ee, pr, problem="elasticity", **kw)
    assert_scaled_close(np_(K), Kr, what="K")
    assert_scaled_close(np_(F), Fr, what="F")


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_fields_batched_reports_inverted_element(eng, mode):
    """tgk_assemble_fields_batched_d reads the members' status words back once:
    an inverted element is still reported like a per-field loop would."""
    from paper_2602_05052_b200 import InputError
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [3, 3, 3])
    bad = elems.copy()
    bad[[5, 9]] = bad[[5, 9]][:, [1, 0, 2, 3]]
    m = eng.DeviceMesh("tet4", nodes, bad)
    r = eng.Routing(m, 1)
    rho = torch.from_numpy(0.5 + np.random.default_rng(1).random((4, bad.shape[0])))
    with pytest.raises(InputError, match="element 5 has non-positive Jacobian determinant"):
        eng.assemble_fields_batched(m, r, {"diffusion": rho}, sources=[1.0], mode=mode)
