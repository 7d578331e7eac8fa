"""Allen-Cahn Newton re-assembly (AllenCahnStepper::step, timestep.cpp:144-178;
SURVEY.md 8(f) rank 1): tangent mass T and reaction load F for a nodal state.

CPU: the golden fixtures (generated from the reference's own code path through
oracle/ref_shim.cpp) agree with a restatement on the oracle port
(interpolate_nodal + the reaction formulas of batch.cpp:314-351 in numpy, then
the port's local_mass / local_load and ascending-slot reduce).
GPU: tgk_allen_cahn_d (one fused pass) is bit-identical to the fixtures and to
the reference library on a larger grid.
"""
import glob
import os

import numpy as np
import pytest

from oracle import port, ref
from tests._util import assert_bitwise

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIXTURES = sorted(glob.glob(os.path.join(GOLD, "allen_cahn_*.npz")))


def restated(kind, nodes, elems, u, eps):
    """batch.cpp:314-351 on the oracle port (numpy float64 ops are exact IEEE, no FMA)."""
    k = elems.shape[1]
    deg = port.default_degree(kind, 1)
    tb = port.tables(kind, deg)
    B = tb["B"]  # Q x k
    Q = B.shape[0]
    v = np.zeros((elems.shape[0], Q))
    for q in range(Q):  # interpolate_nodal: s = 0; s += B[a] * u[conn[a]]
        s = np.zeros(elems.shape[0])
        for a in range(k):
            s = s + B[q, a] * u[elems[:, a]]
        v[:, q] = s
    e2 = eps * eps
    tang = -e2 * (3.0 * v * v - 1.0)
    react = -e2 * v * (v * v - 1.0)
    r = port.Routing(nodes.shape[0], port.dofmap(kind, elems, 1))
    T = r.reduce_matrix(port.local(kind, nodes, elems, deg, port.MASS, tang.reshape(-1)).reshape(-1))
    F = r.reduce_vector(port.local(kind, nodes, elems, deg, port.LOAD, react.reshape(-1)).reshape(-1))
    return T, F


@pytest.mark.parametrize("path", FIXTURES)
def test_restatement_matches_reference_fixture(path):
    g = dict(np.load(path))
    kind = "tet4" if g["nodes"].shape[1] == 3 else "tri3"
    T, F = restated(kind, g["nodes"], g["elements"], g["u"], float(g["eps"]))
    assert_bitwise(T, g["T"], "T")
    assert_bitwise(F, g["F"], "F")


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES)
def test_gpu_allen_cahn_golden(path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_05052_b200 import engine
    g = dict(np.load(path))
    kind = "tet4" if g["nodes"].shape[1] == 3 else "tri3"
    m = engine.DeviceMesh(kind, g["nodes"], g["elements"])
    r = engine.Routing(m, 1)
    T, F = engine.allen_cahn(m, r, g["u"], float(g["eps"]))
    assert_bitwise(T.cpu().numpy(), g["T"], "T")
    assert_bitwise(F.cpu().numpy(), g["F"], "F")


@pytest.mark.gpu
def test_gpu_allen_cahn_vs_reference_library():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_05052_b200 import engine
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [13, 11, 9])
    u = 2.0 * np.random.default_rng(5).random(nodes.shape[0]) - 1.0
    m = engine.DeviceMesh("tet4", nodes, elems)
    r = engine.Routing(m, 1)
    T, F = engine.allen_cahn(m, r, u, 0.3)
    if ref.available():
        rm = ref.Mesh.from_arrays("tet4", nodes, elems)
        Tr, Fr = ref.allen_cahn(rm, ref.Routing(rm, 1), u, 0.3)
    else:
        Tr, Fr = restated("tet4", nodes, elems, u, 0.3)
    assert_bitwise(T.cpu().numpy(), Tr, "T")
    assert_bitwise(F.cpu().numpy(), Fr, "F")
