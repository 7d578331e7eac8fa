"""The C++ drop-in (adapter/physics_gpu.cpp) through the reference's own API.

oracle/_ref/libtgref_gpu.so is the unmodified reference library with its
tg::assemble replaced by the adapter (oracle/Makefile `refgpu`); its ctypes
shim builds ProblemSpec / Mesh / DofMap / RoutingMatrices / CoefficientField
objects exactly as reference code does.  Every result must be bit-identical to
the CPU library's tg::assemble (proj/src/physics.cpp:10-75), K and M must carry
the routing's own pattern pointer (routing.cpp:114; consumers check it at
timestep.cpp:140 and adjoint.cpp:73), and QUAD4 meshes (not P1) must still
assemble through the renamed CPU implementation."""
import os

import numpy as np
import pytest

from tests._util import assert_bitwise, assert_scaled_close

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_adapter_library_built_and_exports_assemble():
    """CPU-side: the drop-in library links libtgk and exports tg::assemble and the renamed CPU path."""
    from oracle import ref, ref_gpu
    if not ref.available():
        pytest.skip("reference library not built")
    assert ref_gpu.available(), "oracle/_ref/libtgref_gpu.so missing or not loadable"
    import subprocess
    syms = subprocess.run(["nm", "-D", ref_gpu.LIB_PATH], capture_output=True, text=True).stdout
    assert "_ZN2tg8assembleERKNS_11ProblemSpecERKNS_4MeshERKNS_6DofMapERKNS_15RoutingMatricesEb" in syms
    assert "_ZN2tg12assemble_cpuERKNS_11ProblemSpecERKNS_4MeshERKNS_6DofMapERKNS_15RoutingMatricesEb" in syms
    assert " U tgk_assemble" in syms
    assert "_ZN2tg20simp_sensitivity_cpuERKSt6vectorIdSaIdEEdddS4_RKNS_4MeshERKNS_6DofMapES4_" in syms
    assert " U tgk_simp_sensitivity_d" in syms


torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def libs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ref, ref_gpu
    if not (ref.available() and ref_gpu.available()):
        pytest.skip("reference libraries not built")
    ref.set_threads(0)
    ref_gpu.set_threads(0)
    return ref, ref_gpu


def _pair(libs, kind, nodes=None, elems=None, divs=None, comps=1):
    ref, gpu = libs
    out = []
    for L in (ref, gpu):
        m = L.Mesh.grid(kind, [1.0] * len(divs), divs) if divs else L.Mesh.from_arrays(kind, nodes, elems)
        out.append((m, L.Routing(m, comps)))
    return out


def _cases(E, Nn, dim):
    rng = np.random.default_rng(5)
    rho, nod = 0.5 + rng.random(E), 0.5 + rng.random(Nn)
    c = [dict(sources=[1.0]),
         dict(sources=[1.0], with_mass=True),
         dict(diffusion=("element", rho), sources=[("element", rho)], with_mass=True),
         dict(diffusion=("nodal", nod), sources=[("nodal", nod)]),
         dict(sources=[("checkerboard", 3)]),
         dict(problem="mass", diffusion=("element", rho), with_mass=True)]
    if dim == 2:
        c.append(dict(diffusion=("multisine", (3, 1.0)), sources=[("checkerboard", 2)], with_mass=True))
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("kind,divs", [("tet4", [7, 6, 5]), ("tri3", [23, 17])])
def test_dropin_bitwise_and_pattern_identity(libs, kind, divs):
    ref, gpu = libs
    (mc, rc), (mg, rg) = _pair(libs, kind, divs=divs)
    E, Nn = mc.E, mc.N
    for kw in _cases(E, Nn, len(divs)):
        want = ref.assemble(mc, rc, **kw)
        got = gpu.assemble(mg, rg, **kw)
        assert gpu.last_pattern_shared() == 1, f"{kw}: K/M not on the routing's pattern pointer"
        for g, w, what in zip(got, want, "KFM"):
            if w is None:
                continue
            assert_bitwise(g, w, f"{kind} {what} {sorted(kw)}")


@pytest.mark.gpu
def test_dropin_elasticity_unstructured_and_fan(libs):
    ref, gpu = libs
    from paper_2602_05052_b200 import meshgen
    from tests.test_gpu_fallback import bicone_tet
    lam, mu = 0.5769230769230769, 0.38461538461538464
    for kind, nodes, elems, comps, kw in [
            ("tri3", *meshgen.unstructured_tri(32), 2, dict(problem="elasticity", lam=lam, mu=mu, plane_stress=True,
                                                           sources=[1.0, -0.5])),
            ("tet4", *port_grid("tet4", [4, 3, 5]), 3, dict(problem="elasticity", lam=lam, mu=mu,
                                                          sources=[1.0, 1.0, 1.0])),
            ("tet4", *bicone_tet(70), 1, dict(sources=[1.0], with_mass=True)),
            ("tri3", *meshgen.unstructured_tri(32), 1, dict(diffusion=("multisine", (4, 1.5)), sources=[1.0]))]:
        (mc, rc), (mg, rg) = _pair(libs, kind, nodes, elems, comps=comps)
        want = ref.assemble(mc, rc, **kw)
        got = gpu.assemble(mg, rg, **kw)
        assert gpu.last_pattern_shared() == 1
        for g, w, what in zip(got, want, "KFM"):
            if w is not None:
                assert_bitwise(g, w, f"{kind} {what} {sorted(kw)}")


def port_grid(kind, divs):
    from oracle import port
    return port.generate_grid(kind, [1.0] * len(divs), divs)


@pytest.mark.gpu
def test_dropin_quad4_delegates_to_cpu_and_fast_mode(libs, monkeypatch):
    ref, gpu = libs
    (mc, rc), (mg, rg) = _pair(libs, "quad4", divs=[6, 5])
    want = ref.assemble(mc, rc, sources=[1.0], with_mass=True)
    got = gpu.assemble(mg, rg, sources=[1.0], with_mass=True)
    for g, w, what in zip(got, want, "KFM"):
        assert_bitwise(g, w, f"quad4 {what}")
    monkeypatch.setenv("TG_GPU_ASSEMBLE_MODE", "fast")
    (mc, rc), (mg, rg) = _pair(libs, "tet4", divs=[9, 8, 7])
    want = ref.assemble(mc, rc, sources=[1.0], with_mass=True)
    got = gpu.assemble(mg, rg, sources=[1.0], with_mass=True)
    assert gpu.last_pattern_shared() == 1
    for g, w, what in zip(got, want, "KFM"):
        assert_scaled_close(g, w, what=f"fast {what}")


@pytest.mark.gpu
def test_dropin_errors_match_reference(libs):
    ref, gpu = libs
    (mc, rc), (mg, rg) = _pair(libs, "tri3", divs=[4, 4])
    for L, m, r in [(ref, mc, rc), (gpu, mg, rg)]:
        with pytest.raises(L.RefError, match="per-element coefficient: expected"):
            L.assemble(m, r, diffusion=("element", np.ones(3)))
        with pytest.raises(L.RefError, match="component count"):
            L.assemble(m, r, problem="elasticity")


@pytest.mark.gpu
@pytest.mark.parametrize("kind,comps,divs", [("tet4", 3, [4, 3, 5]), ("quad4", 2, [12, 7]), ("tri3", 1, [9, 8])])
def test_dropin_simp_sensitivity_bitwise(libs, kind, comps, divs):
    """tg::simp_sensitivity through adapter/adjoint_gpu.cpp (the reference's own
    Mesh / DofMap types) vs the CPU library: bitwise for p = 3 — including the
    QUAD4 vector-elasticity DoFs of the reference's topology optimisation."""
    (mr, rr), (mg, rg) = _pair(libs, kind, divs=divs, comps=comps)
    E, kd = rr.E, rr.k  # elements, local DoFs per element
    rng = np.random.default_rng(21)
    K0 = rng.standard_normal((E, kd, kd))
    K0 = K0 + K0.transpose(0, 2, 1)
    U = rng.standard_normal(rr.N)
    rho = 0.05 + 0.95 * rng.random(E)
    want = rr.simp_sensitivity(rho, 3.0, 1e-9, 1.0, K0, U)
    got = rg.simp_sensitivity(rho, 3.0, 1e-9, 1.0, K0, U)
    assert_bitwise(got, want, f"{kind} simp_sensitivity")

