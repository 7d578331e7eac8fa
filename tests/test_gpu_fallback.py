"""Meshes beyond the fused plan layouts still assemble.

The reference builds routing for any connectivity (proj/src/routing.cpp:12-85)
and folds segments of any length (routing.cpp:117-124).  Here: fans whose hub
node has 50-80 neighbours — past the per-thread routing row builder (64), the
fast plan's row limit (62) and the exact row-block plan's (32) — go through
the long-row routing builder and the materialised Stage I + II fallback, and
must match the reference library bit for bit (exact mode) or within the
SURVEY.md 8(c) tolerance (fast mode)."""
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


def fan_tri(n):
    """Hub node 0 and a ring of n nodes; triangles (0, i, i+1), counter-clockwise."""
    t = 2 * np.pi * np.arange(n) / n
    nodes = np.vstack([[0.0, 0.0], np.stack([np.cos(t), np.sin(t)], 1)])
    elems = np.array([[0, 1 + i, 1 + (i + 1) % n] for i in range(n)], dtype=np.int64)
    return nodes, elems


def bicone_tet(n, layers=2):
    """Tets around the axis A-B: (A, B, r_i, r_i+1) with a ring of n nodes, plus
    an outer layer so ring nodes are ordinary; hubs A and B have n + 1 neighbours."""
    t = 2 * np.pi * np.arange(n) / n
    ring = np.stack([np.cos(t), np.sin(t), np.zeros(n)], 1)
    outer = np.stack([2 * np.cos(t), 2 * np.sin(t), np.zeros(n)], 1)
    nodes = np.vstack([[0.0, 0.0, -1.0], [0.0, 0.0, 1.0], ring, outer])
    el = []
    for i in range(n):
        j = (i + 1) % n
        el.append([0, 1, 2 + i, 2 + j])
        if layers > 1:  # wedge between the ring and the outer ring, split into tets touching B
            el.append([1, 2 + i, 2 + n + i, 2 + n + j])
            el.append([1, 2 + i, 2 + n + j, 2 + j])
    elems = np.array(el, dtype=np.int64)
    # orient every tet positively (the reference rejects det <= 0)
    X = nodes[elems]
    det = np.einsum("ij,ij->i", X[:, 1] - X[:, 0], np.cross(X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]))
    flip = det < 0
    elems[flip] = elems[flip][:, [0, 1, 3, 2]]
    return nodes, elems


CASES = [dict(sources=[1.0]), dict(sources=[1.0], with_mass=True),
         dict(diffusion=("element", None), sources=[("element", None)], with_mass=True)]


def _kw(kw, E):
    kw = dict(kw)
    rho = 0.5 + np.random.default_rng(9).random(E)
    if isinstance(kw.get("diffusion"), tuple):
        kw["diffusion"] = ("element", rho)
        kw["sources"] = [("element", rho)]
    return kw


@pytest.mark.parametrize("name,kind,mesh", [("tri3 fan 80", "tri3", fan_tri(80)),
                                            ("tet4 bicone 48", "tet4", bicone_tet(48)),
                                            ("tet4 bicone 70", "tet4", bicone_tet(70))],
                         ids=["tri-fan80", "tet-bicone48", "tet-bicone70"])
def test_high_valence_meshes_vs_reference(eng, name, kind, mesh):
    from oracle import ref
    nodes, elems = mesh
    E, Nn = elems.shape[0], nodes.shape[0]
    m = eng.DeviceMesh(kind, nodes, elems)
    r = eng.Routing(m, 1, segments=True)
    pr = port.Routing(Nn, port.dofmap(kind, elems, 1))
    h = r.host_arrays()
    assert int(np.diff(h["offsets"]).max()) > 32, "the hub row must exceed the row-block plan"
    for key in ["offsets", "cols", "vec_slots", "mat_offsets", "mat_slots"]:
        assert np.array_equal(h[key], getattr(pr, key)), f"{name}: routing {key}"
    assert np.array_equal(h["slot_of"].astype(np.int64), pr.slot_of())
    use_ref = ref.available()
    if use_ref:
        rm = ref.Mesh.from_arrays(kind, nodes, elems)
        rr = ref.Routing(rm, 1)
    for kw in CASES:
        kw = _kw(kw, E)
        want = ref.assemble(rm, rr, **kw) if use_ref else port.assemble(kind, nodes, elems, pr, **kw)
        for mode in ["exact", "fast"]:
            K, F, M = eng.assemble(m, r, mode=mode, **kw)
            got = [np_(K), np_(F)] + ([np_(M)] if kw.get("with_mass") else [])
            for g, w, what in zip(got, want, "KFM"):
                if mode == "exact":
                    assert_bitwise(g, w, f"{name} {mode} {what} {sorted(kw)}")
                else:
                    assert_scaled_close(g, w, what=f"{name} {mode} {what} {sorted(kw)}")


def test_high_valence_elasticity_and_batched(eng):
    """Elasticity (materialised fallback) and the batched entry point on a fan."""
    nodes, elems = bicone_tet(40)
    E, Nn = elems.shape[0], nodes.shape[0]
    m = eng.DeviceMesh("tet4", nodes, elems)
    rv = eng.Routing(m, 3)
    prv = port.Routing(Nn * 3, port.dofmap("tet4", elems, 3))
    lam, mu = 0.5769230769230769, 0.38461538461538464
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=lam, mu=mu, sources=[1.0, 0.5, 0.25])
    Kr, Fr, _ = port.assemble("tet4", nodes, elems, prv, problem="elasticity", lam=lam, mu=mu,
                              sources=[1.0, 0.5, 0.25])
    assert_bitwise(np_(K), Kr, "elasticity K")
    assert_bitwise(np_(F), Fr, "elasticity F")
    r = eng.Routing(m, 1)
    pr = port.Routing(Nn, port.dofmap("tet4", elems, 1))
    rho = np.stack([0.5 + np.random.default_rng(50 + b).random(E) for b in range(3)])
    Kb, Fb = eng.assemble_batched(m, r, rho, source=1.0)
    for b in range(3):
        Kr, Fr, _ = port.assemble("tet4", nodes, elems, pr, diffusion=("element", rho[b]), sources=[1.0])
        assert_bitwise(np_(Kb[b]), Kr, f"batched field {b}")
        if b == 0:
            assert_bitwise(np_(Fb), Fr, "batched F")


def test_connectivity_change_marks_routings_stale(eng):
    """tgk_mesh_upload with DIFFERENT connectivity invalidates routings built
    before; identical connectivity (the e2e path) does not."""
    from paper_2602_05052_b200 import InputError
    from paper_2602_05052_b200 import _native as N
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [3, 3, 3])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    L = N.lib()
    n64 = np.ascontiguousarray(nodes)
    e64 = np.ascontiguousarray(elems, dtype=np.int64)
    N.check(L.tgk_mesh_upload(m._h, n64.ctypes.data, e64.ctypes.data, None))
    K1, _, _ = eng.assemble(m, r, sources=[1.0])  # same connectivity: still valid
    e2 = e64.copy()
    e2[[0, 1]] = e2[[1, 0]]
    N.check(L.tgk_mesh_upload(m._h, None, e2.ctypes.data, None))
    with pytest.raises(InputError, match="earlier connectivity"):
        eng.assemble(m, r, sources=[1.0])
    r2 = eng.Routing(m, 1)
    K2, _, _ = eng.assemble(m, r2, sources=[1.0])
    pr = port.Routing(nodes.shape[0], port.dofmap("tet4", e2, 1))
    Kr, _, _ = port.assemble("tet4", nodes, e2, pr, sources=[1.0])
    assert_bitwise(np_(K2), Kr, "rebuilt routing")


@pytest.mark.parametrize("kind,mesh", [("tri3", "unstructured"), ("tet4", "bicone")], ids=["tri-unstructured", "tet-bicone"])
def test_scatter_add_oracle_independent_vs_reference(eng, kind, mesh):
    """tgk_scatter_add (the reference's scatter_add_oracle, routing.cpp:134-175,
    by a global key sort independent of the routing build) against the
    reference library: pattern and values bit-identical, with and without F."""
    from oracle import ref
    from paper_2602_05052_b200 import _native as N
    from paper_2602_05052_b200 import meshgen, tgfem
    import ctypes as C
    if not ref.available():
        pytest.skip("reference library not built")
    nodes, elems = meshgen.unstructured_tri(24) if mesh == "unstructured" else bicone_tet(70)
    k = elems.shape[1]
    rng = np.random.default_rng(3)
    lk = rng.standard_normal((elems.shape[0], k, k))
    lf = rng.standard_normal((elems.shape[0], k))
    rm = ref.Mesh.from_arrays(kind, nodes, elems)
    rr = ref.Routing(rm, 1)
    offs, cols, vals, F = rr.scatter_add(lk, lf)
    m = eng.DeviceMesh(kind, nodes, elems)
    nnz = C.c_int64()
    L = N.lib()
    N.check(L.tgk_scatter_add(m._h, lk.ctypes.data, None, C.byref(nnz), None, None, None, None))
    assert nnz.value == cols.size
    o2, c2, v2, F2 = (np.zeros(offs.size, np.int64), np.zeros(cols.size, np.int64), np.zeros(cols.size),
                      np.zeros(F.size))
    N.check(L.tgk_scatter_add(m._h, lk.ctypes.data, lf.ctypes.data, C.byref(nnz), o2.ctypes.data,
                              c2.ctypes.data, v2.ctypes.data, F2.ctypes.data))
    assert np.array_equal(o2, offs) and np.array_equal(c2, cols)
    assert_bitwise(v2, vals, "scatter K")
    assert_bitwise(F2, F, "scatter F")
    tm = tgfem.Mesh(kind, nodes, elems)
    d = tgfem.scatter_add_oracle(tm, lk)
    assert_bitwise(d["values"], vals, "tgfem.scatter_add_oracle")


def test_fast_elasticity_long_rows(eng):
    """Fast-mode elasticity on a bicone whose hub rows have 49 entries (copy-out
    runs of 9 x 49 values, diagonal blocks from the zero row sums over 48
    off-diagonal blocks) vs the oracle within the SURVEY.md 8(c) tolerance."""
    nodes, elems = bicone_tet(48)
    m = eng.DeviceMesh("tet4", nodes, elems)
    rv = eng.Routing(m, 3)
    pr = port.Routing(nodes.shape[0] * 3, port.dofmap("tet4", elems, 3))
    lam, mu = 0.5769230769230769, 0.38461538461538464
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=lam, mu=mu, sources=[1.0, -1.0, 0.5], mode="fast")
    Kr, Fr, _ = port.assemble("tet4", nodes, elems, pr, problem="elasticity", lam=lam, mu=mu,
                              sources=[1.0, -1.0, 0.5])
    assert_scaled_close(np_(K), Kr, what="K")
    assert_scaled_close(np_(F), Fr, what="F")


def test_async_upload_checks(eng):
    """tgk_mesh_upload_async (the pipelined e2e path): identical connectivity
    passes tgk_mesh_upload_check and assembles like the oracle; an out-of-range
    node id is reported by the check (status 2) and never reaches the kernels;
    changed connectivity marks the routings stale at the check."""
    from paper_2602_05052_b200 import InputError
    from paper_2602_05052_b200 import _native as N
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [3, 3, 3])
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    L = N.lib()
    n64 = np.ascontiguousarray(nodes * 1.5)
    e64 = np.ascontiguousarray(elems, dtype=np.int64)
    N.check(L.tgk_mesh_upload_async(m._h, n64.ctypes.data, e64.ctypes.data, None))
    K, F, _ = eng.assemble(m, r, sources=[1.0], mode="fast")
    N.check(L.tgk_mesh_upload_check(m._h))
    pr = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    Kr, Fr, _ = port.assemble("tet4", n64, elems, pr, sources=[1.0])
    assert_scaled_close(np_(K), Kr, what="K after async upload")
    bad = e64.copy()
    bad[7, 2] = nodes.shape[0] + 5
    N.check(L.tgk_mesh_upload_async(m._h, None, bad.ctypes.data, None))
    with pytest.raises(InputError, match="element 7 references a node outside"):
        N.check(L.tgk_mesh_upload_check(m._h))
    N.check(L.tgk_mesh_upload(m._h, None, e64.ctypes.data, None))  # restore (blocking path)
    e2 = e64.copy()
    e2[[0, 1]] = e2[[1, 0]]
    N.check(L.tgk_mesh_upload_async(m._h, None, e2.ctypes.data, None))
    N.check(L.tgk_mesh_upload_check(m._h))
    with pytest.raises(InputError, match="earlier connectivity"):
        eng.assemble(m, r, sources=[1.0])
