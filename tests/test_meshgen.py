"""CPU: the C4 unstructured input mesh (paper_2602_05052_b200/meshgen.py) is a
valid reference mesh with the SURVEY.md 8(d) sizes, deterministic, and its RNG
is std::mt19937_64."""
import numpy as np

from oracle import port, ref
from paper_2602_05052_b200 import meshgen
from tests._util import MT64


def test_mt19937_64_matches_std():
    a, b = MT64(42), meshgen.MT19937_64(42)
    assert all(a() == b.next() for _ in range(2000))


def test_c4_mesh_sizes_and_validity():
    nodes, elems = meshgen.unstructured_tri(256)
    assert nodes.shape == (257 * 257, 2) and elems.shape == (2 * 256 * 256, 3)
    r = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
    assert r.nnz == 460289  # N + 2 * edges
    p = nodes[elems]
    area2 = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 2, 0] - p[:, 0, 0]) * (p[:, 1, 1] - p[:, 0, 1])
    assert area2.min() > 0.3 / 256 ** 2  # CCW, worst case 0.4 h^2
    assert np.isclose(area2.sum() / 2, 1.0)
    if ref.available():
        ref.Mesh.from_arrays("tri3", nodes, elems, validate=True)  # Mesh::validate (mesh.cpp:56-77)


def test_c4_mesh_deterministic_and_scrambled():
    n1, e1 = meshgen.unstructured_tri(24)
    n2, e2 = meshgen.unstructured_tri(24)
    assert np.array_equal(n1, n2) and np.array_equal(e1, e2)
    # numbering carries no grid structure: consecutive elements are not neighbours
    shared = np.mean([len(set(e1[i]) & set(e1[i + 1])) > 0 for i in range(len(e1) - 1)])
    assert shared < 0.2
