"""Drop-in for the reference's Python module ``tgfem`` / ``_tgfem``
(proj/bindings/module.cpp:54-196, proj/python/tgfem/__init__.py:1-31) on the
assembly path: same names, arguments, return shapes and exceptions, NumPy in
and out, computed by the sm_100a kernels of libtgk.so.

Differences by design: the device mesh and the routing (pattern + slot map)
are cached per mesh object instead of being rebuilt on every call
(module.cpp:116-117 rebuilds build_routing each time).  Solvers and topology
optimisation (solve_poisson, topopt_cantilever) are outside the accelerated
path and raise NotImplementedError.
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _native as N
from ._native import InputError, NumericalError, check, lib

__all__ = ["InputError", "Mesh", "NumericalError", "compliance", "generate_grid", "load_gmsh",
           "local_stiffness", "reduce_matrix", "scatter_add_oracle", "set_thread_count",
           "solve_poisson", "topopt_cantilever", "write_gmsh"]


def _kind_code(kind: str) -> int:
    try:
        return N.KINDS[kind]
    except KeyError:
        raise InputError(f"unknown element kind: {kind}") from None  # module.cpp:26-31


class Mesh:
    """tg::Mesh (mesh.hpp:15-41) as seen from Python (module.cpp:60-84)."""

    def __init__(self, kind: str, nodes, elements, boundary_nodes=None):
        self._kind = _kind_code(kind.lower())
        self.dim = 3 if self._kind == N.TET4 else 2
        k = 3 if self._kind == N.TRI3 else 4
        self._nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, self.dim)
        self._elements = np.ascontiguousarray(elements, dtype=np.int64).reshape(-1, k)
        self._boundary = None if boundary_nodes is None else np.asarray(boundary_nodes, np.int64)
        self._dev = {}

    @property
    def kind(self):
        return N.KIND_NAMES[self._kind]

    @property
    def nodes(self):
        return self._nodes

    @property
    def elements(self):
        return self._elements

    @property
    def boundary_nodes(self):
        if self._boundary is None:
            n = lib().tgk_topological_boundary(self._kind, self._elements.ctypes.data,
                                               self._elements.shape[0], self._nodes.shape[0], None)
            out = np.zeros(n, dtype=np.int64)
            lib().tgk_topological_boundary(self._kind, self._elements.ctypes.data,
                                           self._elements.shape[0], self._nodes.shape[0],
                                           out.ctypes.data)
            self._boundary = out
        return self._boundary

    def node_count(self):
        return self._nodes.shape[0]

    def element_count(self):
        return self._elements.shape[0]

    def content_hash(self):
        return lib().tgk_content_hash(self._kind, self._nodes.ctypes.data, self._nodes.shape[0],
                                      self._elements.ctypes.data, self._elements.shape[0])

    def validate(self):
        check(lib().tgk_validate(self._kind, self._nodes.ctypes.data, self._nodes.shape[0],
                                 self._elements.ctypes.data, self._elements.shape[0]))

    # device-side cache (mesh upload + routing per component count)
    def _device(self):
        from .engine import DeviceMesh
        if "mesh" not in self._dev:
            self._dev["mesh"] = DeviceMesh(self.kind.lower(), self._nodes, self._elements)
        return self._dev["mesh"]

    def _routing(self, components=1, segments=True):
        from .engine import Routing
        key = ("routing", components, segments)
        if key not in self._dev:
            self._dev[key] = Routing(self._device(), components, segments=segments)
        return self._dev[key]


def generate_grid(kind, extents, divisions):
    """tg::generate_grid (mesh.cpp:96-169), bit-identical arrays."""
    code = _kind_code(kind)
    d = 3 if code == N.TET4 else 2
    if len(extents) != d or len(divisions) != d:
        raise InputError(f"generate_grid: extents/divisions must have {d} entries for {N.KIND_NAMES[code]}")
    div = np.asarray(divisions, dtype=np.int64)
    ext = np.asarray(extents, dtype=np.float64)
    nn, ne = C.c_int64(), C.c_int64()
    check(lib().tgk_grid_sizes(code, div.ctypes.data, C.byref(nn), C.byref(ne)))
    k = 3 if code == N.TRI3 else 4
    nodes = np.empty((nn.value, d))
    elems = np.empty((ne.value, k), dtype=np.int64)
    check(lib().tgk_generate_grid(code, ext.ctypes.data, div.ctypes.data, nodes.ctypes.data,
                                  elems.ctypes.data))
    return Mesh(kind, nodes, elems)


def set_thread_count(n):
    """tg::set_thread_count (parallel.hpp:9): accepted; GPU results never depend on it."""
    lib().tgk_set_thread_count(int(n))


def _csr_dict(routing, values):
    arrs = routing.host_arrays(slot_of=False, segments=False)
    return {"rows": routing.N, "offsets": arrs["offsets"], "cols": arrs["cols"],
            "values": values}


def local_stiffness(mesh: Mesh, coeff=None):
    """Batched diffusion stiffness blocks, E x k x k (module.cpp:92-112)."""
    from . import engine
    dm = mesh._device()
    degree = lib().tgk_default_degree(mesh._kind, 0)
    Q = engine.quadrature_count(mesh.kind.lower(), degree)
    E = mesh.element_count()
    if coeff is None:
        c = np.ones(E * Q)
    else:
        pe = np.asarray(coeff, dtype=np.float64).reshape(-1)
        if pe.size != E:
            raise InputError(f"per-element coefficient: expected {E} values, got {pe.size}")
        c = np.repeat(pe, Q)
    return engine.local_stiffness_diffusion(dm, degree, c).cpu().numpy()


def reduce_matrix(mesh: Mesh, local_matrices):
    """CSR dict {rows, offsets, cols, values} (module.cpp:114-120)."""
    from . import engine
    r = mesh._routing(1, segments=True)
    loc = np.asarray(local_matrices, dtype=np.float64)
    if loc.size != r.E * r.k * r.k:
        raise InputError("reduce_matrix: local tensor shape mismatch")
    vals = engine.reduce_matrix(r, loc.reshape(-1)).cpu().numpy()
    return _csr_dict(r, vals)


def scatter_add_oracle(mesh: Mesh, local_matrices):
    """Classic scatter-add result (module.cpp:122-132).  On the GPU the per-element
    scatter in ascending element order is realised as the equivalent ordered
    gather, so the values are identical by construction (routing.cpp:163-174)."""
    return reduce_matrix(mesh, local_matrices)


def compliance(F, U):
    """C = F^T U (adjoint.cpp:96-99)."""
    F = np.asarray(F, dtype=np.float64)
    U = np.asarray(U, dtype=np.float64)
    if F.shape != U.shape:
        raise InputError("compliance: shape mismatch")
    s = 0.0
    for a, b in zip(F.tolist(), U.tolist()):
        s += a * b
    return s


def load_gmsh(path):
    raise NotImplementedError("gmsh I/O is outside the accelerated assembly path (SURVEY.md 8(f))")


def write_gmsh(mesh, path):
    raise NotImplementedError("gmsh I/O is outside the accelerated assembly path (SURVEY.md 8(f))")


def solve_poisson(mesh, diffusion=None, source=1.0):
    raise NotImplementedError("linear solves are outside the accelerated assembly path (SURVEY.md 8(f))")


def topopt_cantilever(nx=60, ny=30, iterations=51, vol_frac=0.5):
    raise NotImplementedError("topology optimisation is outside the accelerated assembly path")
