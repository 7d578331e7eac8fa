"""Drop-in for the reference's Python module ``tgfem`` / ``_tgfem``
(proj/bindings/module.cpp:54-196, proj/python/tgfem/__init__.py:1-31) on the
assembly path: same names, arguments, return shapes and exceptions, NumPy in
and out, computed by the sm_100a kernels of libtgk.so.

Differences by design: the device mesh and the routing (pattern + slot map)
are cached per mesh object instead of being rebuilt on every call
(module.cpp:116-117 rebuilds build_routing each time).  solve_poisson runs on
the device (condensation + BiCGSTAB); topology optimisation (topopt_cantilever)
is outside the accelerated path and raises NotImplementedError.
"""
from __future__ import annotations

import ctypes as C

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
        # private copies, exposed read-only: the device mesh / routing cached in
        # _dev stay consistent with them (the reference returns copies, module.cpp:63-75)
        self._nodes = np.array(nodes, dtype=np.float64).reshape(-1, self.dim)
        self._elements = np.array(elements, dtype=np.int64).reshape(-1, k)
        self._nodes.setflags(write=False)
        self._elements.setflags(write=False)
        self._boundary = None if boundary_nodes is None else np.asarray(boundary_nodes, np.int64)
        self.boundary_tags = {}  # gmsh entity tag -> sorted node ids (mesh.hpp boundary_tags)
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
    """Classic scatter-add result (module.cpp:122-132): its own pattern and a
    per-element scatter in element order (routing.cpp:134-175), computed on the
    GPU by an algorithm independent of the routing build (tgk_scatter_add: one
    stable radix sort of all (row, col) contribution keys, run sums in slot order)."""
    loc = np.ascontiguousarray(local_matrices, dtype=np.float64)
    k = mesh.elements.shape[1]
    if loc.size != mesh.element_count() * k * k:
        raise InputError("scatter_add_oracle: local tensor shape mismatch")
    dm = mesh._device()
    nnz = C.c_int64()
    check(lib().tgk_scatter_add(dm._h, loc.ctypes.data, None, C.byref(nnz), None, None, None, None))
    n = mesh.node_count()
    offsets = np.zeros(n + 1, np.int64)
    cols = np.zeros(nnz.value, np.int64)
    values = np.zeros(nnz.value)
    check(lib().tgk_scatter_add(dm._h, loc.ctypes.data, None, C.byref(nnz), offsets.ctypes.data, cols.ctypes.data,
                                values.ctypes.data, None))
    return {"rows": n, "offsets": offsets, "cols": cols, "values": values}


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


_GMSH_DIM = {1: 1, 2: 2, 3: 2, 4: 3, 15: 0}      # gmsh_io.cpp kind_dim
_GMSH_NODES = {1: 2, 2: 3, 3: 4, 4: 4, 15: 1}    # gmsh_io.cpp kind_nodes
_GMSH_KIND = {2: "tri3", 3: "quad4", 4: "tet4"}


def load_gmsh(path):
    """tg::load_gmsh (gmsh_io.cpp:64-221): MSH 4.x ASCII; node tags re-packed to
    0-based indices in ascending tag order, one volume element kind, lower-
    dimensional elements become boundary tag groups; Mesh::validate at the end.
    The input-side half of SURVEY.md 8(c)'s identical-input rule."""
    try:
        f = open(path)
    except OSError:
        raise InputError(f"cannot open mesh file: {path}") from None
    lines = []
    with f:
        for raw in f:
            ln = raw.rstrip("\n")
            if ln.endswith("\r"):
                ln = ln[:-1]
            if ln:
                lines.append(ln)
    pos = 0

    def nxt(what):
        nonlocal pos
        if pos >= len(lines):
            raise InputError(f"{path}:{pos}: unexpected end of file in {what}")
        pos += 1
        return lines[pos - 1]

    nodes_by_tag, raw_elems, saw_format = {}, [], False
    while pos < len(lines):
        ln = nxt("file")
        if not ln.startswith("$"):
            continue
        section = ln[1:]
        if section == "MeshFormat":
            head = nxt("$MeshFormat").split()
            try:
                version, binary = float(head[0]), int(head[1])
            except (IndexError, ValueError):
                raise InputError(f"{path}: unsupported mesh format (need MSH 4.x ASCII)") from None
            if version < 4.0 or version >= 5.0 or binary != 0:
                raise InputError(f"{path}: unsupported mesh format (need MSH 4.x ASCII)")
            saw_format = True
            if nxt("$MeshFormat") != "$EndMeshFormat":
                raise InputError(f"{path}: missing $EndMeshFormat")
        elif section == "Nodes":
            nb = int(nxt("$Nodes").split()[0])
            for _ in range(nb):
                _, _, _, count = (int(x) for x in nxt("$Nodes").split()[:4])
                tags = [int(nxt("node tags").split()[0]) for _ in range(count)]
                for t in tags:
                    xs = nxt("node coordinates").split()
                    nodes_by_tag[t] = (float(xs[0]), float(xs[1]), float(xs[2]))
            if nxt("$Nodes") != "$EndNodes":
                raise InputError(f"{path}: missing $EndNodes")
        elif section == "Elements":
            nb = int(nxt("$Elements").split()[0])
            for _ in range(nb):
                _, etag, etype, count = (int(x) for x in nxt("$Elements").split()[:4])
                nn = _GMSH_NODES.get(etype)
                if nn is None:
                    raise InputError(f"{path}: unsupported element type {etype}")
                for _ in range(count):
                    parts = nxt("element list").split()
                    if len(parts) < 1 + nn:
                        raise InputError(f"{path}: malformed element connectivity")
                    raw_elems.append((etype, etag, [int(x) for x in parts[1:1 + nn]]))
            if nxt("$Elements") != "$EndElements":
                raise InputError(f"{path}: missing $EndElements")
        else:  # skip unknown sections ($Entities, $PhysicalNames, ...)
            end = "$End" + section
            while nxt(end) != end:
                pass
    if not saw_format:
        raise InputError(f"{path}: not a Gmsh MSH file (no $MeshFormat)")
    if not nodes_by_tag:
        raise InputError(f"{path}: no $Nodes section")
    if not raw_elems:
        raise InputError(f"{path}: no $Elements section")
    vol_dim = max(_GMSH_DIM[t] for t, _, _ in raw_elems)
    vol_types = {t for t, _, _ in raw_elems if _GMSH_DIM[t] == vol_dim}
    if len(vol_types) > 1:
        a, b = sorted(vol_types)[:2]
        raise InputError(f"{path}: mixed volume element kinds (types {a} and {b})")
    vol_type = vol_types.pop()
    if vol_type not in _GMSH_KIND:
        raise InputError(f"{path}: no supported volume elements (TRI3/QUAD4/TET4)")
    tags = sorted(nodes_by_tag)
    index_of = {t: i for i, t in enumerate(tags)}
    nodes = np.array([nodes_by_tag[t][:vol_dim] for t in tags], dtype=np.float64)
    elems, groups, bnodes = [], {}, set()
    for etype, etag, conn in raw_elems:
        try:
            ids = [index_of[t] for t in conn]
        except KeyError as exc:
            raise InputError(f"{path}: element references unknown node tag {exc.args[0]}") from None
        if _GMSH_DIM[etype] == vol_dim:
            elems.append(ids)
        else:
            groups.setdefault(str(etag), []).extend(ids)
            bnodes.update(ids)
    mesh = Mesh(_GMSH_KIND[vol_type], nodes, np.array(elems, dtype=np.int64),
                boundary_nodes=sorted(bnodes) if bnodes else None)
    mesh.boundary_tags = {k: sorted(set(v)) for k, v in sorted(groups.items())}
    mesh.validate()
    return mesh


def _fmt17(x):
    """std::ostream << double at precision(17) (default floatfield) == printf %.17g."""
    return "%.17g" % x


def write_gmsh(mesh, path):
    """tg::write_gmsh (gmsh_io.cpp:223-250): MSH 4.1 ASCII, one node and one element block,
    tags 1..N / 1..E; byte-identical to the reference writer."""
    try:
        out = open(path, "w")
    except OSError:
        raise InputError(f"cannot open file for writing: {path}") from None
    nodes, elems = mesh.nodes, mesh.elements
    N, E = nodes.shape[0], elems.shape[0]
    gtype = {"TRI3": 2, "QUAD4": 3, "TET4": 4}[mesh.kind]
    dim = mesh.dim
    w = ["$MeshFormat\n4.1 0 8\n$EndMeshFormat\n", f"$Nodes\n1 {N} 1 {N}\n", f"{dim} 1 0 {N}\n"]
    w.extend(f"{i + 1}\n" for i in range(N))
    for i in range(N):
        x = nodes[i]
        z = x[2] if dim == 3 else 0.0
        w.append(f"{_fmt17(x[0])} {_fmt17(x[1])} {_fmt17(z)}\n")
    w.append("$EndNodes\n")
    w.append(f"$Elements\n1 {E} 1 {E}\n{dim} 1 {gtype} {E}\n")
    for e in range(E):
        w.append(str(e + 1) + "".join(f" {int(v) + 1}" for v in elems[e]) + "\n")
    w.append("$EndElements\n")
    with out:
        out.write("".join(w))


def solve_poisson(mesh, diffusion=None, source=1.0):
    """Homogeneous-Dirichlet Poisson solve (module.cpp:133-157) on the GPU: fused
    assembly, condensation of the boundary nodes (solver.cpp:34-85) and Jacobi
    BiCGSTAB (solver.cpp:105-227); returns {u, iterations, rel_residual}.
    Difference by design: the reference's dense LU for <= 2000 free DoFs
    (solver.cpp:274-281) is not ported; BiCGSTAB is used at every size."""
    from . import engine
    dm = mesh._device()
    r = mesh._routing(1, segments=False)
    coef = 1.0 if diffusion is None else ("element", np.asarray(diffusion, dtype=np.float64))
    K, F, _ = engine.assemble(dm, r, diffusion=coef, sources=[float(source)])
    b = mesh.boundary_nodes
    cond = engine.Condensed(r, K, F, b, np.zeros(b.size))
    if cond.n_free == 0:
        return {"u": cond.expand(np.zeros(0)).cpu().numpy(), "iterations": 0, "rel_residual": 0.0}
    u, rep = engine.solve_condensed(cond)
    if not rep["converged"]:
        raise NumericalError(f"linear solve did not converge: rel_residual = {rep['rel_residual']} "
                             f"after {rep['iterations']} iterations")
    return {"u": u.cpu().numpy(), "iterations": rep["iterations"], "rel_residual": rep["rel_residual"]}


def topopt_cantilever(nx=60, ny=30, iterations=51, vol_frac=0.5):
    raise NotImplementedError("topology optimisation is outside the accelerated assembly path")
