"""CPU: MSH 4.1 ingest/export parity with the reference (gmsh_io.cpp:64-250),
the input half of SURVEY.md 8(c)'s identical-input rule for unstructured meshes
(C4): our writer is byte-identical to tg::write_gmsh and our reader returns the
same arrays as tg::load_gmsh (tag re-packing, boundary groups, validation)."""
import os

import numpy as np
import pytest

from oracle import ref
from paper_2602_05052_b200 import meshgen, tgfem

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference library (oracle/_ref) not built")


def test_writer_byte_identical_and_round_trip(tmp_path):
    nodes, elems = meshgen.unstructured_tri(20)
    ours, theirs = tmp_path / "ours.msh", tmp_path / "ref.msh"
    tgfem.write_gmsh(tgfem.Mesh("tri3", nodes, elems), ours)
    ref.Mesh.from_arrays("tri3", nodes, elems).write_gmsh(theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    m = tgfem.load_gmsh(ours)
    r = ref.Mesh.load_gmsh(ours)
    assert np.array_equal(m.nodes, r.nodes) and np.array_equal(m.nodes, nodes)
    assert np.array_equal(m.elements, r.elements) and np.array_equal(m.elements, elems)
    assert np.array_equal(m.boundary_nodes, r.boundary_nodes)


def test_tet4_round_trip(tmp_path):
    nodes, elems = meshgen.kuhn("tet4", [3, 4, 2])
    p = tmp_path / "t.msh"
    tgfem.write_gmsh(tgfem.Mesh("tet4", nodes, elems), p)
    r = ref.Mesh.load_gmsh(p)
    assert np.array_equal(r.nodes, nodes) and np.array_equal(r.elements, elems)


def test_reader_repacks_tags_and_reads_boundary_groups(tmp_path):
    text = """$MeshFormat
4.1 0 8
$EndMeshFormat
$Entities
junk
$EndEntities
$Nodes
2 4 3 12
1 7 0 2
12
3
1.0 0.0 0.0
0.0 0.0 0.0
1 9 0 2
5
8
0.0 1.0 0.0
1.0 1.0 0.0
$EndNodes
$Elements
2 3 1 3
2 1 2 2
1 3 12 8
2 3 8 5
1 4 1 1
3 12 3
$EndElements
"""
    p = tmp_path / "x.msh"
    p.write_text(text)
    m = tgfem.load_gmsh(p)
    r = ref.Mesh.load_gmsh(p)
    assert np.array_equal(m.nodes, r.nodes)
    assert np.array_equal(m.elements, r.elements)
    assert np.array_equal(m.boundary_nodes, r.boundary_nodes)
    assert m.boundary_tags == {"4": [0, 3]}


@pytest.mark.parametrize("body,msg", [
    ("$Nodes\n0 0 0 0\n$EndNodes\n", "no $MeshFormat"),
    ("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n", "unsupported mesh format"),
    ("$MeshFormat\n4.1 0 8\n$EndMeshFormat\n", "no $Nodes"),
])
def test_reader_errors_mirror_reference(tmp_path, body, msg):
    p = tmp_path / "bad.msh"
    p.write_text(body)
    with pytest.raises(tgfem.InputError, match=msg.replace("$", r"\$")):
        tgfem.load_gmsh(p)
    with pytest.raises(ref.RefError, match=msg.replace("$", r"\$")):
        ref.Mesh.load_gmsh(p)
