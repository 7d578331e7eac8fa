"""TEST INFRASTRUCTURE ONLY — ctypes binding of the unmodified reference library.

oracle/_ref/libtgref.so is every /root/reference/proj/src/*.cpp compiled in
place by oracle/Makefile plus oracle/ref_shim.cpp (extern "C" forwarders).  On
the GPU box /root/reference is absent but the prebuilt .so travels with the
snapshot; ``available()`` reports whether it can be loaded.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .port import Field, field, KINDS, PROBLEMS, element_dim, element_nodes

_HERE = os.path.dirname(os.path.abspath(__file__))
# oracle/ref_gpu.py loads this module a second time with the GPU drop-in library
LIB_PATH = os.environ.get("_TGREF_LIB_OVERRIDE") or os.path.join(_HERE, "_ref", "libtgref.so")

_lib = None


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def available():
    try:
        lib()
        return True
    except OSError:
        return False


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.tgr_last_error.restype = C.c_char_p
        L.tgr_set_threads.argtypes = [C.c_int]
        L.tgr_mesh_grid.argtypes = [C.c_int, P, P, C.POINTER(P)]
        L.tgr_mesh_arrays.argtypes = [C.c_int, P, C.c_int64, P, C.c_int64, C.c_int, C.POINTER(P)]
        L.tgr_mesh_load_gmsh.argtypes = [C.c_char_p, C.POINTER(P)]
        L.tgr_mesh_write_gmsh.argtypes = [P, C.c_char_p]
        L.tgr_mesh_free.argtypes = [P]
        L.tgr_mesh_sizes.argtypes = [P, P, P, P, P, P]
        L.tgr_mesh_copy.argtypes = [P, P, P, P]
        L.tgr_mesh_hash.restype = C.c_uint64
        L.tgr_mesh_hash.argtypes = [P]
        L.tgr_routing.argtypes = [P, C.c_int, C.POINTER(P)]
        L.tgr_routing_free.argtypes = [P]
        L.tgr_routing_sizes.argtypes = [P, P, P, P, P]
        L.tgr_routing_copy.argtypes = [P] * 8
        L.tgr_routing_save.argtypes = [P, C.c_uint64, C.c_char_p]
        L.tgr_quadrature.argtypes = [C.c_int, C.c_int, P, P, P, P, P]
        L.tgr_geometry.argtypes = [P, C.c_int, P, P, P, P, P]
        L.tgr_local.argtypes = [P, C.c_int, C.c_int, P, P, P]
        L.tgr_reduce_matrix.argtypes = [P, P, P]
        L.tgr_reduce_vector.argtypes = [P, P, P]
        L.tgr_scatter_add.argtypes = [P] * 8
        L.tgr_assemble.argtypes = [P, P, C.c_int, P, P, P, C.c_int, C.c_int, P, C.c_int, P, P, P, P]
        L.tgr_last_pattern_shared.restype = C.c_int
        L.tgr_gradient_products.argtypes = [P] * 5
        L.tgr_simp_sensitivity.argtypes = [P, P, P, C.c_double, C.c_double, C.c_double, P, P, P]
        L.tgr_allen_cahn.argtypes = [P, P, P, C.c_double, P, P]
        L.tgr_condense.argtypes = [P, P, P, C.c_int64] + [P] * 12
        L.tgr_spmv.argtypes = [P] * 4
        L.tgr_bicgstab.argtypes = [C.c_int64, P, P, P, P, P, C.c_double, C.c_double, C.c_int64, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().tgr_last_error().decode())


def last_pattern_shared():
    """1 if the last assemble() returned K (and M) on the routing's own pattern pointer."""
    return lib().tgr_last_pattern_shared()


def set_threads(n):
    lib().tgr_set_threads(int(n))


def thread_count():
    return lib().tgr_thread_count()


class Mesh:
    def __init__(self, handle):
        self._h = handle
        n, e, b, d, k = (C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(), C.c_int())
        lib().tgr_mesh_sizes(handle, C.byref(n), C.byref(e), C.byref(b), C.byref(d), C.byref(k))
        self.N, self.E, self.dim, self.k = n.value, e.value, d.value, k.value
        self.kind = {2: "tri3" if self.k == 3 else "quad4", 3: "tet4"}[self.dim]
        self.nodes = np.zeros((self.N, self.dim))
        self.elements = np.zeros((self.E, self.k), dtype=np.int64)
        self.boundary_nodes = np.zeros(b.value, dtype=np.int64)
        lib().tgr_mesh_copy(handle, _p(self.nodes), _p(self.elements), _p(self.boundary_nodes))

    @classmethod
    def grid(cls, kind, extents, divisions):
        h = C.c_void_p()
        ext = np.asarray(extents, dtype=np.float64)
        div = np.asarray(divisions, dtype=np.int64)
        _check(lib().tgr_mesh_grid(KINDS[kind], _p(ext), _p(div), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, kind, nodes, elements, validate=True):
        h = C.c_void_p()
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        elements = np.ascontiguousarray(elements, dtype=np.int64)
        _check(lib().tgr_mesh_arrays(KINDS[kind], _p(nodes), nodes.shape[0], _p(elements),
                                     elements.shape[0], int(validate), C.byref(h)))
        return cls(h.value)

    @classmethod
    def load_gmsh(cls, path):
        h = C.c_void_p()
        _check(lib().tgr_mesh_load_gmsh(str(path).encode(), C.byref(h)))
        return cls(h.value)

    def write_gmsh(self, path):
        _check(lib().tgr_mesh_write_gmsh(self._h, str(path).encode()))

    def content_hash(self):
        return lib().tgr_mesh_hash(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().tgr_mesh_free(self._h)
            self._h = None


class Routing:
    """build_dofmap + build_routing of the reference."""

    def __init__(self, mesh: Mesh, comps=1):
        h = C.c_void_p()
        _check(lib().tgr_routing(mesh._h, comps, C.byref(h)))
        self._h = h.value
        self.mesh = mesh
        N, E, k, nnz = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        lib().tgr_routing_sizes(self._h, C.byref(N), C.byref(E), C.byref(k), C.byref(nnz))
        self.N, self.E, self.k, self.nnz = N.value, E.value, k.value, nnz.value
        self.offsets = np.zeros(self.N + 1, dtype=np.int64)
        self.cols = np.zeros(self.nnz, dtype=np.int64)
        self.vec_offsets = np.zeros(self.N + 1, dtype=np.uint32)
        self.vec_slots = np.zeros(self.E * self.k, dtype=np.uint32)
        self.mat_offsets = np.zeros(self.nnz + 1, dtype=np.uint32)
        self.mat_slots = np.zeros(self.E * self.k * self.k, dtype=np.uint32)
        self.dofmap = np.zeros((self.E, self.k), dtype=np.int64)
        lib().tgr_routing_copy(self._h, _p(self.offsets), _p(self.cols), _p(self.vec_offsets),
                               _p(self.vec_slots), _p(self.mat_offsets), _p(self.mat_slots),
                               _p(self.dofmap))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().tgr_routing_free(self._h)
            self._h = None

    def slot_of(self):
        out = np.empty(self.E * self.k * self.k, dtype=np.int64)
        seg = np.repeat(np.arange(self.nnz, dtype=np.int64), np.diff(self.mat_offsets.astype(np.int64)))
        out[self.mat_slots.astype(np.int64)] = seg
        return out

    def save(self, hash_, path):
        _check(lib().tgr_routing_save(self._h, hash_, str(path).encode()))

    def reduce_matrix(self, local_m):
        local_m = np.ascontiguousarray(local_m, dtype=np.float64)
        out = np.zeros(self.nnz)
        _check(lib().tgr_reduce_matrix(self._h, _p(local_m), _p(out)))
        return out

    def reduce_vector(self, local_v):
        local_v = np.ascontiguousarray(local_v, dtype=np.float64)
        out = np.zeros(self.N)
        _check(lib().tgr_reduce_vector(self._h, _p(local_v), _p(out)))
        return out

    def scatter_add(self, localK, localF):
        offs = np.zeros(self.N + 1, dtype=np.int64)
        cols = np.zeros(self.nnz, dtype=np.int64)
        vals = np.zeros(self.nnz)
        F = np.zeros(self.N)
        lk = None if localK is None else np.ascontiguousarray(localK, dtype=np.float64)
        lf = None if localF is None else np.ascontiguousarray(localF, dtype=np.float64)
        _check(lib().tgr_scatter_add(self.mesh._h, self._h, _p(lk), _p(lf), _p(offs), _p(cols),
                                     _p(vals), _p(F)))
        return offs, cols, vals, F

    def gradient_products(self, lam, U):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        U = np.ascontiguousarray(U, dtype=np.float64)
        dK = np.zeros(self.nnz)
        dF = np.zeros(self.N)
        _check(lib().tgr_gradient_products(self._h, _p(lam), _p(U), _p(dK), _p(dF)))
        return dK, dF

    def simp_sensitivity(self, rho, p, E_min, E_max, K0, U):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        K0 = np.ascontiguousarray(K0, dtype=np.float64)
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.zeros(self.E)
        _check(lib().tgr_simp_sensitivity(self.mesh._h, self._h, _p(rho), p, E_min, E_max,
                                          _p(K0), _p(U), _p(out)))
        return out


def quadrature(kind, degree):
    Q = C.c_int()
    k, d = element_nodes(kind), element_dim(kind)
    pts, w, B, G = np.zeros(33), np.zeros(11), np.zeros(44), np.zeros(132)
    _check(lib().tgr_quadrature(KINDS[kind], degree, C.byref(Q), _p(pts), _p(w), _p(B), _p(G)))
    q = Q.value
    return dict(Q=q, points=pts[: q * d].reshape(q, d), weights=w[:q],
                B=B[: q * k].reshape(q, k), G=G[: q * k * d].reshape(q, k, d))


def geometry(mesh: Mesh, degree):
    Q = quadrature(mesh.kind, degree)["Q"]
    E, d, k = mesh.E, mesh.dim, mesh.k
    out = dict(jac=np.zeros((E, Q, d, d)), det=np.zeros((E, Q)), jac_invT=np.zeros((E, Q, d, d)),
               qpts=np.zeros((E, Q, d)), grads=np.zeros((E, Q, k, d)))
    _check(lib().tgr_geometry(mesh._h, degree, _p(out["jac"]), _p(out["det"]), _p(out["jac_invT"]),
                              _p(out["qpts"]), _p(out["grads"])))
    return out


def local(mesh: Mesh, degree, what, c1, c2=None):
    E, kg, d = mesh.E, mesh.k, mesh.dim
    shape = {0: (E, kg, kg), 1: (E, kg * d, kg * d), 2: (E, kg, kg), 3: (E, kg), 4: (E, kg * d)}[what]
    out = np.zeros(shape)
    c1 = np.ascontiguousarray(c1, dtype=np.float64)
    c2 = None if c2 is None else np.ascontiguousarray(c2, dtype=np.float64)
    _check(lib().tgr_local(mesh._h, degree, what, _p(c1), _p(c2), _p(out)))
    return out


def allen_cahn(mesh: Mesh, routing: Routing, u, eps):
    """AllenCahnStepper re-assembly (timestep.cpp:144-178): (T values, reaction load F)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    T = np.zeros(routing.nnz)
    F = np.zeros(routing.N)
    _check(lib().tgr_allen_cahn(mesh._h, routing._h, _p(u), C.c_double(eps), _p(T), _p(F)))
    return T, F


def condense(routing: Routing, K, F, dofs, values):
    """condense (solver.cpp:34-85): dict of free_dofs, fixed_dofs, prescribed, offsets, cols, values, F_f."""
    dofs = np.ascontiguousarray(dofs, dtype=np.int64)
    values = np.ascontiguousarray(values, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    F = np.ascontiguousarray(F, dtype=np.float64)
    N, nnz = routing.N, routing.nnz
    nf, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
    buf = dict(free_dofs=np.zeros(N, np.int64), fixed_dofs=np.zeros(N, np.int64), prescribed=np.zeros(N),
               offsets=np.zeros(N + 1, np.int64), cols=np.zeros(nnz, np.int64), values=np.zeros(nnz), F_f=np.zeros(N))
    _check(lib().tgr_condense(routing._h, _p(K), _p(F), dofs.size, _p(dofs), _p(values), C.byref(nf), C.byref(nc),
                              C.byref(nz), *[_p(buf[k]) for k in ["free_dofs", "fixed_dofs", "prescribed", "offsets",
                                                                 "cols", "values", "F_f"]]))
    n, c, z = nf.value, nc.value, nz.value
    return dict(free_dofs=buf["free_dofs"][:n], fixed_dofs=buf["fixed_dofs"][:c], prescribed=buf["prescribed"][:c],
                offsets=buf["offsets"][:n + 1], cols=buf["cols"][:z], values=buf["values"][:z], F_f=buf["F_f"][:n])


def bicgstab(offsets, cols, values, b, tol_rel=1e-10, tol_abs=1e-10, max_iter=10000):
    """bicgstab (solver.cpp:105-227) from a zero initial guess: (x, report)."""
    n = len(offsets) - 1
    x = np.zeros(n)
    it, rel, conv = C.c_int64(), C.c_double(), C.c_int()
    _check(lib().tgr_bicgstab(n, _p(np.ascontiguousarray(offsets, np.int64)), _p(np.ascontiguousarray(cols, np.int64)),
                              _p(np.ascontiguousarray(values, np.float64)), _p(np.ascontiguousarray(b, np.float64)),
                              _p(x), tol_rel, tol_abs, max_iter, C.byref(it), C.byref(rel), C.byref(conv)))
    return x, {"iterations": it.value, "rel_residual": rel.value, "converged": bool(conv.value)}


def spmv(routing: Routing, values, x):
    """SparseOperator::apply (sparse.cpp:18-31)."""
    y = np.zeros(routing.N)
    _check(lib().tgr_spmv(routing._h, _p(np.ascontiguousarray(values, dtype=np.float64)),
                          _p(np.ascontiguousarray(x, dtype=np.float64)), _p(y)))
    return y


def assemble(mesh: Mesh, routing: Routing, problem="poisson", diffusion=1.0, lam=1.0, mu=1.0,
             plane_stress=False, sources=(), with_mass=False, timing=False):
    """tg::assemble (physics.cpp:10-75).  Returns (K, F, M|None[, seconds])."""
    keep = []
    fd, a = field(diffusion); keep.append(a)
    fl, a = field(lam); keep.append(a)
    fm, a = field(mu); keep.append(a)
    srcs = (Field * max(1, len(sources)))()
    for i, s in enumerate(sources):
        f, a = field(s)
        keep.append(a)
        srcs[i] = f
    K = np.zeros(routing.nnz)
    F = np.zeros(routing.N)
    M = np.zeros(routing.nnz) if with_mass else None
    secs = C.c_double()
    _check(lib().tgr_assemble(mesh._h, routing._h, PROBLEMS[problem], C.byref(fd), C.byref(fl),
                              C.byref(fm), int(plane_stress), len(sources), srcs, int(with_mass),
                              _p(K), _p(F), _p(M), C.byref(secs)))
    if timing:
        return K, F, M, secs.value
    return K, F, M
