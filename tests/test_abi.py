"""CPU: the C-ABI library loads, exports every symbol include/tgk.h declares,
and its host helpers match the reference; compute entry points fail loudly
(no CPU fallback) when no GPU is present."""
import os
import re

import numpy as np
import pytest

from paper_2602_05052_b200 import _native as N
from paper_2602_05052_b200 import tgfem
from oracle import port
from tests._util import assert_bitwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_functions():
    src = open(os.path.join(ROOT, "include", "tgk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tgk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers the header exactly
    assert sorted(N.EXPORTS) == names


def test_library_has_sm100a_code():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", ["mesh_tri3_3x3.npz", "mesh_tet4_3x2x4.npz", "mesh_tri3_7x5.npz"])
def test_host_helpers_match_reference(name):
    g = dict(np.load(os.path.join(GOLD, name)))
    kind = "tet4" if g["nodes"].shape[1] == 3 else "tri3"
    d = g["nodes"].shape[1]
    # recover the grid arguments from the golden node array
    ext = g["nodes"].max(axis=0)
    div = [len(np.unique(g["nodes"][:, c])) - 1 for c in range(d)]
    m = tgfem.generate_grid(kind, list(ext), div)
    assert np.array_equal(m.nodes, g["nodes"]) and np.array_equal(m.elements, g["elements"])
    assert m.content_hash() == int(g["content_hash"])
    assert np.array_equal(m.boundary_nodes, g["boundary"])
    m.validate()


def test_tables_match_oracle():
    import ctypes as C
    for kind in ["tri3", "tet4"]:
        for deg in range(1, 5):
            t = port.tables(kind, deg)
            Q = C.c_int()
            k, d = port.element_nodes(kind), port.element_dim(kind)
            pts, w, B, G = np.zeros(33), np.zeros(11), np.zeros(44), np.zeros(132)
            N.check(N.lib().tgk_tables(N.KINDS[kind], deg, C.byref(Q), pts.ctypes.data,
                                       w.ctypes.data, B.ctypes.data, G.ctypes.data))
            q = Q.value
            assert q == t["Q"]
            assert_bitwise(w[:q], t["weights"])
            assert_bitwise(B[: q * k], t["B"])
            assert_bitwise(G[: q * k * d], t["G"])


def test_host_errors_mirror_reference():
    with pytest.raises(N.InputError, match="divisions must be >= 1"):
        tgfem.generate_grid("tri3", [1.0, 1.0], [0, 3])
    with pytest.raises(N.InputError, match="unknown element kind"):
        tgfem.generate_grid("hex8", [1.0, 1.0], [2, 2])
    m = tgfem.Mesh("tri3", [[0, 0], [0, 1], [1, 0]], [[0, 1, 2]])
    with pytest.raises(N.InputError, match="non-positive orientation"):
        m.validate()
    m = tgfem.Mesh("tri3", [[0, 0], [1, 0], [0, 1]], [[0, 1, 1]])
    with pytest.raises(N.InputError, match="repeats node"):
        m.validate()
    assert tgfem.compliance([4.0], [2.0]) == 8.0


def test_no_cpu_fallback_without_gpu():
    if N.lib().tgk_device_count() > 0:
        pytest.skip("GPU present")
    m = tgfem.generate_grid("tri3", [1.0, 1.0], [2, 2])
    with pytest.raises(N.CudaError, match="no usable CUDA device"):
        tgfem.local_stiffness(m)
