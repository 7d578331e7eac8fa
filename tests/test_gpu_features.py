"""GPU: multi-GPU slab assembly (emulated on one device), the batched C4 kernel
on the unstructured mesh, and the interface-combine kernel — through the C ABI,
checked against the CPU oracle."""
import ctypes as C

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


@pytest.mark.parametrize("mode,with_mass", [("exchange", False), ("exchange", True), ("halo", True)])
def test_slabs_on_one_gpu_match_single_gpu(eng, mode, with_mass):
    """Every rank of a 3-slab partition run in turn on one GPU; the NCCL P2P is
    replaced by a device copy, the interface sum is libtgk's combine kernel."""
    from paper_2602_05052_b200 import _native as N
    from paper_2602_05052_b200 import dist as D
    L = N.lib()
    div, world = (5, 4, 3), 3
    parts = []
    for rank in range(world):
        s = D.slab(div, rank, world, mode)
        nodes, elems = D.slab_mesh(s)
        m = eng.DeviceMesh("tet4", nodes, elems)
        r = eng.Routing(m, 1)
        N.check(L.tgk_routing_set_owned_rows(r._h, s.own_lo, s.calc_hi))
        if mode == "exchange":
            N.check(L.tgk_routing_set_element_range(r._h, s.elem_lo, s.elem_hi))
        K, F, M = eng.assemble(m, r, sources=[1.0], with_mass=with_mass)
        rp = r.host_arrays(slot_of=False, segments=False)["offsets"]
        parts.append((s, rp, K, F, M, (m, r)))
    if mode == "exchange":
        for rank in range(1, world):
            s, rp, K, F, M, _ = parts[rank]
            sl, rpl, Kl, Fl, Ml, _ = parts[rank - 1]
            lo, hi = s.bottom_rows
            tl, th = sl.top_rows
            for a, al in [(K, Kl)] + ([(M, Ml)] if with_mass else []):
                D.gpu_combine(al[int(rpl[tl]):int(rpl[th])].clone(), a[int(rp[lo]):int(rp[hi])])
            D.gpu_combine(Fl[tl:th].clone(), F[lo:hi])
    torch.cuda.synchronize()
    nodes, elems = port.generate_grid("tet4", [1.0] * 3, [5, 4, 3 * world])
    pr = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    Kr, Fr, Mr = port.assemble("tet4", nodes, elems, pr, sources=[1.0], with_mass=with_mass)
    for s, rp, K, F, M, _ in parts:
        g0, g1 = s.node_offset + s.own_lo, s.node_offset + s.own_hi
        assert np.array_equal(rp[s.own_lo:s.own_hi + 1] - rp[s.own_lo], pr.offsets[g0:g1 + 1] - pr.offsets[g0])
        got = {"K": np_(K)[rp[s.own_lo]:rp[s.own_hi]], "F": np_(F)[s.own_lo:s.own_hi]}
        want = {"K": Kr[pr.offsets[g0]:pr.offsets[g1]], "F": Fr[g0:g1]}
        if with_mass:
            got["M"] = np_(M)[rp[s.own_lo]:rp[s.own_hi]]
            want["M"] = Mr[pr.offsets[g0]:pr.offsets[g1]]
        for key in got:
            if mode == "halo" or s.rank == 0:
                assert_bitwise(got[key], want[key], f"rank {s.rank} {key}")
            else:
                nif = s.layer if key == "F" else int(rp[s.own_lo + s.layer] - rp[s.own_lo])
                assert_scaled_close(got[key][:nif], want[key][:nif], what=f"rank {s.rank} interface {key}")
                assert_bitwise(got[key][nif:], want[key][nif:], f"rank {s.rank} interior {key}")


def test_batched_c4_mesh_bit_exact(eng):
    from paper_2602_05052_b200 import meshgen
    nodes, elems = meshgen.unstructured_tri(40)
    m = eng.DeviceMesh("tri3", nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
    B = 7
    rho = meshgen.batch_fields(B, elems.shape[0])
    K, F = eng.assemble_batched(m, r, rho, source=1.0)
    torch.cuda.synchronize()
    for b in range(B):
        Kr, Fr, _ = port.assemble("tri3", nodes, elems, pr, diffusion=("element", rho[b]), sources=[1.0])
        assert_bitwise(np_(K[b]), Kr, f"field {b}")
        if b == 0:
            assert_bitwise(np_(F), Fr, "F")


def test_batched_tet4_bit_exact(eng):
    nodes, elems = port.generate_grid("tet4", [1.0] * 3, [6, 5, 4])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    rho = 0.5 + np.random.default_rng(5).random((3, elems.shape[0]))
    K, F = eng.assemble_batched(m, r, rho, source=1.0)
    for b in range(3):
        Kr, Fr, _ = port.assemble("tet4", nodes, elems, pr, diffusion=("element", rho[b]), sources=[1.0])
        assert_bitwise(np_(K[b]), Kr, f"field {b}")


@pytest.mark.parametrize("kind,env", [
    ("tri3", {"TGK_BATCHED_CHUNKED": "1"}),             # row-block chunked kernel
    ("tri3", {"TGK_ENTRY_R": "8", "TGK_ENTRY_FPB": "3"}),
    ("tri3", {"TGK_ENTRY_R": "256", "TGK_ENTRY_SORT": "1"}),  # several entries / halo elements per thread
    ("tri3", {"TGK_ENTRY_SYM": "1", "TGK_ENTRY_MAXC": "0", "TGK_ENTRY_STCS": "1", "TGK_ENTRY_SORT": "2"}),
    ("tri3", {"TGK_ENTRY_SYM": "1", "TGK_ENTRY_R": "16"}),
    ("tet4", {"TGK_ENTRY_R": "64"}),
    ("tet4", {"TGK_ENTRY_R": "4", "TGK_ENTRY_FPB": "1"}),
])
def test_batched_paths_bit_exact(eng, monkeypatch, kind, env):
    """Entry-owned kernel (default), its plan parameters, and the chunked
    kernel all equal the per-field reference assemble bit for bit."""
    from paper_2602_05052_b200 import meshgen
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if kind == "tri3":
        nodes, elems = meshgen.unstructured_tri(48)
    else:
        nodes, elems = port.generate_grid("tet4", [1.0] * 3, [7, 5, 6])
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1)
    pr = port.Routing(nodes.shape[0], port.dofmap(kind, elems, 1))
    B = 5
    rho = meshgen.batch_fields(B, elems.shape[0])
    K, F = eng.assemble_batched(m, r, rho, source=1.0)
    torch.cuda.synchronize()
    for b in range(B):
        Kr, Fr, _ = port.assemble(kind, nodes, elems, pr, diffusion=("element", rho[b]), sources=[1.0])
        assert_bitwise(np_(K[b]), Kr, f"field {b}")
        if b == 0:
            assert_bitwise(np_(F), Fr, "F")


def test_interface_combine_kernel(eng):
    from paper_2602_05052_b200 import dist as D
    rng = np.random.default_rng(9)
    a, b = rng.random(10007), rng.random(10007)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    D.gpu_combine(ta, tb)
    assert_bitwise(np_(tb), a + b)


@pytest.mark.parametrize("kind,div,comps", [("tri3", [9, 7], 1), ("tet4", [4, 3, 5], 1), ("tet4", [3, 3, 2], 3)])
def test_routing_cache_round_trip_with_reference(eng, tmp_path, kind, div, comps):
    """save_routing / load_routing (routing.cpp:194-234): our file is byte-identical to
    the reference's, the reference's file loads into a routing that assembles identically,
    and a hash mismatch is a cache miss (the reference returns false)."""
    from oracle import ref
    nodes, elems = port.generate_grid(kind, [1.0] * len(div), div)
    h = port.content_hash(kind, nodes, elems)
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, comps, segments=True)
    ours = tmp_path / "ours.bin"
    r.save(h, ours)
    if ref.available():
        rm = ref.Mesh.from_arrays(kind, nodes, elems)
        theirs = tmp_path / "ref.bin"
        ref.Routing(rm, comps).save(h, theirs)
        assert ours.read_bytes() == theirs.read_bytes()
    r2 = eng.Routing.load(m, h, ours, components=comps)
    assert r2 is not None
    a, b = r.host_arrays(), r2.host_arrays()
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    kw = dict(kind="elasticity", lam=0.6, mu=0.4, sources=[1.0] * 3) if comps == 3 else dict(sources=[1.0])
    K1, F1, _ = eng.assemble(m, r, **kw)
    K2, F2, _ = eng.assemble(m, r2, **kw)
    assert_bitwise(np_(K1), np_(K2), "K")
    assert_bitwise(np_(F1), np_(F2), "F")
    assert eng.Routing.load(m, h ^ 1, ours, components=comps) is None
    assert eng.Routing.load(m, h, tmp_path / "missing.bin", components=comps) is None


def test_spmv_and_condense_match_reference(eng):
    """SparseOperator::apply and condense / restrict_to_free / expand (sparse.cpp:18-31,
    solver.cpp:20-103) on the device, bit-identical to the reference library."""
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library (oracle/_ref) not built")
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [7, 6, 5])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    rho = 0.5 + np.random.default_rng(3).random(elems.shape[0])
    K, F, M = eng.assemble(m, r, diffusion=("element", rho), sources=[1.0], with_mass=True)
    rm = ref.Mesh.from_arrays("tet4", nodes, elems)
    rr = ref.Routing(rm, 1)
    x = np.random.default_rng(4).random(nodes.shape[0]) - 0.5
    assert_bitwise(np_(eng.spmv(r, K, x)), ref.spmv(rr, np_(K), x), "spmv")
    bnd = rm.boundary_nodes
    rng = np.random.default_rng(5)
    dofs = np.concatenate([bnd, bnd[:7]])              # duplicates: the last value wins
    vals = rng.random(dofs.size)
    c = eng.Condensed(r, K, F, dofs, vals)
    got = c.arrays()
    want = ref.condense(rr, np_(K), np_(F), dofs, vals)
    for key in want:
        if want[key].dtype == np.float64:
            assert_bitwise(got[key], want[key], key)
        else:
            assert np.array_equal(got[key], want[key]), key
    Mff = np_(c.restrict_to_free(M))
    want_M = ref.condense(rr, np_(M), np_(F), dofs, vals)["values"]
    assert_bitwise(Mff, want_M, "restrict_to_free")
    uf = rng.random(c.n_free)
    u = np_(c.expand(uf))
    full = np.zeros(nodes.shape[0])
    full[want["free_dofs"]] = uf
    full[want["fixed_dofs"]] = want["prescribed"]
    assert_bitwise(u, full, "expand")
    with pytest.raises(eng.N.InputError, match="out of range"):
        eng.Condensed(r, K, F, [nodes.shape[0]], [1.0])


def test_device_poisson_solve_matches_reference_bicgstab(eng):
    """assemble -> condense -> BiCGSTAB -> expand on the device (solver.cpp:34-292) vs the
    reference's bicgstab on the same condensed system: converged, same solution to
    solver tolerance (dot products are parallel reductions, not the serial fold)."""
    from oracle import ref
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [12, 10, 9])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    rho = 0.5 + np.random.default_rng(8).random(elems.shape[0])
    K, F, _ = eng.assemble(m, r, diffusion=("element", rho), sources=[1.0])
    from paper_2602_05052_b200 import tgfem
    bnd = tgfem.Mesh("tet4", nodes, elems).boundary_nodes
    c = eng.Condensed(r, K, F, bnd, np.zeros(bnd.size))
    u, rep = eng.solve_condensed(c, tol_rel=1e-12)
    assert rep["converged"] and rep["rel_residual"] <= 1e-12
    a = c.arrays()
    # residual of the full system on the free rows: K u - F == 0 there
    Ku = np_(eng.spmv(r, K, u))
    res = (Ku - np_(F))[a["free_dofs"]]
    assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(np_(F)[a["free_dofs"]])
    assert np.all(np_(u)[a["fixed_dofs"]] == 0.0)
    if ref.available():
        xr, rr = ref.bicgstab(a["offsets"], a["cols"], a["values"], a["F_f"], tol_rel=1e-12)
        assert rr["converged"]
        uf = np_(u)[a["free_dofs"]]
        assert np.max(np.abs(uf - xr)) <= 1e-9 * np.max(np.abs(xr))
        assert abs(rep["iterations"] - rr["iterations"]) <= max(3, rr["iterations"] // 5)


def test_tgfem_solve_poisson_device(eng):
    """module.cpp:133-157 drop-in: residual of the full system on free rows, zero on the
    boundary, and agreement with a direct sparse solve (scipy) of the same system."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    from paper_2602_05052_b200 import tgfem
    mesh = tgfem.generate_grid("tri3", [1.0, 1.0], [40, 30])
    rho = 0.5 + np.random.default_rng(2).random(mesh.element_count())
    out = tgfem.solve_poisson(mesh, rho, 1.0)
    u = out["u"]
    assert out["rel_residual"] <= 1e-10
    r = port.Routing(mesh.node_count(), port.dofmap("tri3", mesh.elements, 1))
    K, F, _ = port.assemble("tri3", mesh.nodes, mesh.elements, r, diffusion=("element", rho), sources=[1.0])
    A = sp.csr_matrix((K, r.cols, r.offsets), shape=(mesh.node_count(),) * 2)
    b = mesh.boundary_nodes
    free = np.setdiff1d(np.arange(mesh.node_count()), b)
    ref_u = np.zeros(mesh.node_count())
    ref_u[free] = spla.spsolve(A[free][:, free].tocsc(), F[free])
    assert np.all(u[b] == 0.0)
    assert np.max(np.abs(u - ref_u)) <= 1e-8 * np.max(np.abs(ref_u))


@pytest.mark.parametrize("kind,div,kw", [
    ("tri3", [40, 33], dict(sources=[1.0])),
    ("tet4", [11, 9, 8], dict(sources=[1.0], with_mass=True)),
    ("tet4", [9, 8, 7], dict(diffusion="element", sources=["nodal"])),
    ("tri3", [25, 20], dict(kind="mass", diffusion="nodal")),
])
def test_fp32_mode_within_tolerance(eng, kind, div, kw):
    """tgk_assemble_f32_d vs the fp64 reference: |dv| <= 1e-5 |v| + 1e-7 max|v|."""
    nodes, elems = port.generate_grid(kind, [1.0] * len(div), div)
    rng = np.random.default_rng(11)
    fields = {"element": ("element", 0.5 + rng.random(elems.shape[0])),
              "nodal": ("nodal", 0.5 + rng.random(nodes.shape[0]))}
    kw = {k: ([fields.get(x, x) for x in v] if isinstance(v, list) else fields.get(v, v)) for k, v in kw.items()}
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1)
    K32, F32, M32 = eng.assemble(m, r, dtype=torch.float32, **kw)
    assert K32.dtype == torch.float32
    pr = port.Routing(nodes.shape[0], port.dofmap(kind, elems, 1))
    pkw = dict(kw)
    if pkw.pop("kind", None) == "mass":
        pkw["problem"] = "mass"
    Kr, Fr, Mr = port.assemble(kind, nodes, elems, pr, **pkw)
    assert_scaled_close(np_(K32).astype(np.float64), Kr, rel=1e-5, floor=1e-7, what="K fp32")
    if kw.get("sources"):
        assert_scaled_close(np_(F32).astype(np.float64), Fr, rel=1e-5, floor=1e-7, what="F fp32")
    if kw.get("with_mass"):
        assert_scaled_close(np_(M32).astype(np.float64), Mr, rel=1e-5, floor=1e-7, what="M fp32")


@pytest.mark.parametrize("p", [3.0, 2.5])
def test_simp_sensitivity_gpu(eng, p):
    """tgk_simp_sensitivity_d (adjoint.cpp:101-125) on TET4 elasticity DoFs (k = 12)
    and scalar TRI3 DoFs (k = 3) vs the restatement: bitwise for the standard
    penalty p = 3, within 1e-15 relative (device pow) otherwise; a DoF map
    entry out of range is an InputError."""
    from paper_2602_05052_b200 import InputError
    nodes, elems = port.generate_grid("tet4", [1.0, 0.8, 1.2], [5, 4, 6])
    E = elems.shape[0]
    rng = np.random.default_rng(12)
    K0 = port.local("tet4", nodes, elems, 1, port.ELASTICITY, np.full(E, 0.5769230769230769),
                    np.full(E, 0.38461538461538464))
    U = rng.standard_normal(nodes.shape[0] * 3)
    rho = 0.05 + 0.95 * rng.random(E)
    dm = port.dofmap("tet4", elems, 3)
    got = eng.simp_sensitivity(dm, rho, p, 1e-9, 1.0, K0, U).cpu().numpy()
    want = port.simp_sensitivity(dm, rho, p, 1e-9, 1.0, K0, U)
    if p == 3.0:
        assert_bitwise(got, want, "simp_sensitivity k=12")
    else:
        np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)
    tn, te = port.generate_grid("tri3", [1.0, 1.0], [9, 7])
    K2 = port.local("tri3", tn, te, 1, port.DIFFUSION, np.ones(te.shape[0]))
    U2 = rng.standard_normal(tn.shape[0])
    r2 = 0.05 + 0.95 * rng.random(te.shape[0])
    d2 = port.dofmap("tri3", te, 1)
    g2 = eng.simp_sensitivity(d2, r2, 3.0, 1e-9, 1.0, K2, U2).cpu().numpy()
    assert_bitwise(g2, port.simp_sensitivity(d2, r2, 3.0, 1e-9, 1.0, K2, U2), "simp_sensitivity k=3")
    bad = dm.copy()
    bad[4, 7] = U.size + 3
    with pytest.raises(InputError, match="element 4 maps a DoF outside"):
        eng.simp_sensitivity(bad, rho, p, 1e-9, 1.0, K0, U)
