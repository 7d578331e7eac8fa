"""The pybind11 module `_tgfem` (paper_2602_05052_b200/bindings/module.cpp):
the reference's compiled Python module (proj/bindings/module.cpp:54-196) over
the C ABI.  Its checks follow the reference's own Python smoke test
(proj/tests/test_python_smoke.py: grid, local_stiffness + reduce_matrix vs
scatter_add_oracle, solve_poisson, compliance, errors), plus parity of the
computed arrays with the oracle.  CPU: the module loads, exports the
reference's names, runs the host helpers and fails loudly on compute calls;
GPU: the compute path."""
import importlib
import os
import sys

import numpy as np
import pytest

from oracle import port
from tests._util import assert_bitwise

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_05052_b200", "lib")
NAMES = ["InputError", "Mesh", "NumericalError", "compliance", "generate_grid", "load_gmsh", "local_stiffness",
         "reduce_matrix", "scatter_add_oracle", "set_thread_count", "solve_poisson", "topopt_cantilever", "write_gmsh"]


@pytest.fixture(scope="module")
def tg():
    from paper_2602_05052_b200 import build
    build.build_module()
    sys.path.insert(0, LIB)
    try:
        yield importlib.import_module("_tgfem")
    finally:
        sys.path.remove(LIB)


def _has_gpu():
    from paper_2602_05052_b200 import _native
    return _native.lib().tgk_device_count() > 0


def test_module_exports_reference_names(tg):
    for n in NAMES:
        assert hasattr(tg, n), n


def test_grid_and_errors_host(tg):
    mesh = tg.generate_grid("quad4", [1.0, 1.0], [4, 4])
    assert mesh.node_count() == 25 and mesh.element_count() == 16
    assert mesh.nodes.shape == (25, 2) and mesh.elements.shape == (16, 4)
    assert len(mesh.boundary_nodes) == 16
    nodes, elems = port.generate_grid("tet4", [1.0, 2.0, 0.5], [3, 4, 2])
    m3 = tg.generate_grid("tet4", [1.0, 2.0, 0.5], [3, 4, 2])
    assert_bitwise(m3.nodes, nodes, "nodes")
    assert np.array_equal(m3.elements, elems)
    assert m3.kind == "tet4" and m3.dim == 3
    with pytest.raises(tg.InputError, match="unknown element kind: hex8"):
        tg.generate_grid("hex8", [1.0, 1.0], [2, 2])
    assert tg.compliance([4.0], [2.0]) == 8.0
    with pytest.raises(NotImplementedError):
        tg.topopt_cantilever()


def test_compute_fails_loudly_without_gpu(tg):
    if _has_gpu():
        pytest.skip("GPU present")
    mesh = tg.generate_grid("tri3", [1.0, 1.0], [3, 3])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        tg.local_stiffness(mesh)


@pytest.mark.gpu
def test_smoke_semantics_on_gpu(tg):
    """The reference smoke test's assertions, and bitwise parity with the oracle."""
    mesh = tg.generate_grid("tri3", [1.0, 1.0], [3, 3])
    local = tg.local_stiffness(mesh)
    assert local.shape == (18, 3, 3)
    reduced = tg.reduce_matrix(mesh, local)
    oracle = tg.scatter_add_oracle(mesh, local)
    for key in ("values", "cols", "offsets"):
        assert (reduced[key] == oracle[key]).all(), key
    # parity with the oracle restatement (local_stiffness_diffusion + reduce_matrix)
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [5, 4, 6])
    m3 = tg.generate_grid("tet4", [1.0, 1.0, 1.0], [5, 4, 6])
    rho = 0.5 + np.random.default_rng(2).random(elems.shape[0])
    loc = tg.local_stiffness(m3, rho)
    want = port.local("tet4", nodes, elems, 1, port.DIFFUSION, rho)
    assert_bitwise(loc, want, "local_stiffness")
    red = tg.reduce_matrix(m3, loc)
    pr = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    assert np.array_equal(red["offsets"], pr.offsets) and np.array_equal(red["cols"], pr.cols)
    assert_bitwise(red["values"], pr.reduce_matrix(want.reshape(-1)), "reduce_matrix")
    res = tg.solve_poisson(tg.generate_grid("tri3", [1.0, 1.0], [8, 8]))
    assert res["rel_residual"] < 1e-9
    u = res["u"]
    assert len(u) == 81 and max(u) > 0.0
    m8 = tg.generate_grid("tri3", [1.0, 1.0], [8, 8])
    for n in m8.boundary_nodes:
        assert u[n] == 0.0
    with pytest.raises(tg.InputError):
        tg.local_stiffness(mesh, np.ones(3))
