"""Size-independent properties at the BASELINE.json sizes (the
reference's own property checks — acceptance.cpp:245-265 global rigid modes,
test_physics.cpp:72-85 mass sum = volume — and the zero row sums of P1
stiffness), in both arithmetic modes:

* C2 (TET4 100^3, K+M+F): K 1 = 0, sum(M) = |Omega| = 1, sum(F) = f |Omega|;
* C3 (TET4 100^3 elasticity): the six rigid-body modes in the kernel of K
  (|K r|_inf <= 1e-10 max|K| max|r|, the reference's acceptance bound), and
  sum of each load component = f_c |Omega|.
The products run on the device (tgk_spmv_d)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import port  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_05052_b200 import engine
    return engine


@pytest.fixture(scope="module")
def cube():
    return port.generate_grid("tet4", [1.0, 1.0, 1.0], [100, 100, 100])


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_c2_row_sums_mass_and_load(eng, cube, mode):
    nodes, elems = cube
    m = eng.DeviceMesh("tet4", nodes, elems)
    r = eng.Routing(m, 1)
    K, F, M = eng.assemble(m, r, sources=[1.0], with_mass=True, mode=mode)
    ones = torch.ones(r.N, dtype=torch.float64, device=K.device)
    k1 = eng.spmv(r, K, ones)
    assert float(k1.abs().max()) <= 1e-12 * float(K.abs().max()) * 16, "K 1 != 0"
    assert abs(float(M.sum()) - 1.0) <= 1e-12, f"sum(M) = {float(M.sum())!r}"
    assert abs(float(F.sum()) - 1.0) <= 1e-12, f"sum(F) = {float(F.sum())!r}"


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_c3_rigid_modes_and_load(eng, cube, mode):
    nodes, elems = cube
    m = eng.DeviceMesh("tet4", nodes, elems)
    rv = eng.Routing(m, 3)
    f = [1.0, -0.5, 0.25]
    K, F, _ = eng.assemble(m, rv, kind="elasticity", lam=0.5769230769230769, mu=0.38461538461538464,
                           sources=f, mode=mode)
    X = torch.from_numpy(nodes).to(K.device)
    n = X.shape[0]
    modes = []
    for c in range(3):  # translations
        u = torch.zeros(n, 3, dtype=torch.float64, device=K.device)
        u[:, c] = 1.0
        modes.append(u)
    for a, b in [(0, 1), (1, 2), (0, 2)]:  # infinitesimal rotations in the (a, b) plane
        u = torch.zeros(n, 3, dtype=torch.float64, device=K.device)
        u[:, a] = -X[:, b]
        u[:, b] = X[:, a]
        modes.append(u)
    kmax = float(K.abs().max())
    for i, u in enumerate(modes):
        ku = eng.spmv(rv, K, u.reshape(-1))
        assert float(ku.abs().max()) <= 1e-10 * kmax * float(u.abs().max()), f"rigid mode {i}"
    Fc = F.reshape(n, 3).sum(0).cpu().numpy()
    np.testing.assert_allclose(Fc, f, rtol=1e-12, atol=1e-14)
