"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/tg_oracle.c (the C restatement).

Mirrors the reference's Python-visible behaviour closely enough for parity tests:
int64 connectivity, fp64 everything, InputError on bad input.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libtgoracle.so")

KINDS = {"tri3": 0, "quad4": 1, "tet4": 2}
DIFFUSION, ELASTICITY, MASS, LOAD, LOAD_VECTOR = range(5)


class OracleError(RuntimeError):
    pass


class Field(C.Structure):
    _fields_ = [("type", C.c_int), ("value", C.c_double), ("data", C.c_void_p), ("n", C.c_int64)]


def field(spec):
    """spec: float (constant) | ('element', array) | ('nodal', array);
    reference library only: ('checkerboard', frequency) | ('multisine', (K, r)) —
    the reference's Analytic fields checkerboard_source / multi_sine_field."""
    if spec is None:
        return None, None
    if isinstance(spec, (int, float)):
        return Field(0, float(spec), None, 0), None
    kind, arr = spec
    if kind == "checkerboard":
        return Field(3, float(arr), None, 0), None
    if kind == "multisine":
        return Field(4, float(arr[1]), None, int(arr[0])), None
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    t = {"element": 1, "nodal": 2}[kind]
    return Field(t, 0.0, arr.ctypes.data, arr.size), arr


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OracleError(f"{LIB_PATH} missing: run `make -C oracle port`")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.tgo_last_error.restype = C.c_char_p
        L.tgo_routing_build.restype = P
        L.tgo_routing_build.argtypes = [C.c_int64, C.c_int64, C.c_int, P]
        L.tgo_routing_free.argtypes = [P]
        L.tgo_routing_nnz.restype = C.c_int64
        L.tgo_routing_nnz.argtypes = [P]
        L.tgo_routing_copy.argtypes = [P] * 7
        L.tgo_reduce_vector.argtypes = [P] * 3
        L.tgo_reduce_matrix.argtypes = [P] * 3
        L.tgo_scatter_add.argtypes = [P] * 6
        L.tgo_gradient_products.argtypes = [P] * 5
        L.tgo_adjoint_gather.argtypes = [C.c_int64, C.c_int, P, P, P, P, P]
        L.tgo_adjoint_generic.argtypes = [P] * 5
        L.tgo_grid_sizes.argtypes = [C.c_int, P, P, P]
        L.tgo_generate_grid.argtypes = [C.c_int, P, P, P, P]
        L.tgo_content_hash.restype = C.c_uint64
        L.tgo_content_hash.argtypes = [C.c_int, P, C.c_int64, P, C.c_int64]
        L.tgo_dofmap.argtypes = [C.c_int, P, C.c_int64, C.c_int, P]
        L.tgo_tables.argtypes = [C.c_int, C.c_int, P, P, P, P, P]
        L.tgo_geometry.argtypes = [C.c_int, P, P, C.c_int64, C.c_int, P, P, P, P, P, P]
        L.tgo_local.argtypes = [C.c_int, P, P, C.c_int64, C.c_int, C.c_int, P, P, P, P]
        L.tgo_evaluate.argtypes = [C.c_int, P, P, C.c_int64, C.c_int64, C.c_int, P, P]
        L.tgo_assemble.argtypes = [C.c_int, P, C.c_int64, P, C.c_int64, P, C.c_int, P, P, P,
                                   C.c_int, C.c_int, P, C.c_int, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _check(rc):
    if rc != 0:
        raise OracleError(lib().tgo_last_error().decode())


def element_dim(kind):
    return 3 if kind == "tet4" else 2


def element_nodes(kind):
    return 3 if kind == "tri3" else 4


def default_degree(kind, mass):
    return lib().tgo_default_degree(KINDS[kind], int(mass))


def tables(kind, degree):
    Q = C.c_int()
    k, d = element_nodes(kind), element_dim(kind)
    pts = np.zeros(11 * 3)
    w = np.zeros(11)
    B = np.zeros(11 * 4)
    G = np.zeros(11 * 12)
    _check(lib().tgo_tables(KINDS[kind], degree, C.byref(Q), _p(pts), _p(w), _p(B), _p(G)))
    q = Q.value
    return dict(Q=q, points=pts[: q * d].reshape(q, d), weights=w[:q],
                B=B[: q * k].reshape(q, k), G=G[: q * k * d].reshape(q, k, d))


def generate_grid(kind, extents, divisions):
    div = np.asarray(divisions, dtype=np.int64)
    ext = np.asarray(extents, dtype=np.float64)
    n, e = C.c_int64(), C.c_int64()
    lib().tgo_grid_sizes(KINDS[kind], _p(div), C.byref(n), C.byref(e))
    d, k = element_dim(kind), element_nodes(kind)
    nodes = np.zeros((n.value, d))
    elems = np.zeros((e.value, k), dtype=np.int64)
    _check(lib().tgo_generate_grid(KINDS[kind], _p(ext), _p(div), _p(nodes), _p(elems)))
    return nodes, elems


def content_hash(kind, nodes, elems):
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    return lib().tgo_content_hash(KINDS[kind], _p(nodes), nodes.shape[0], _p(elems), elems.shape[0])


def dofmap(kind, elems, comps):
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    k = element_nodes(kind) * comps
    out = np.zeros((elems.shape[0], k), dtype=np.int64)
    lib().tgo_dofmap(KINDS[kind], _p(elems), elems.shape[0], comps, _p(out))
    return out


def geometry(kind, nodes, elems, degree):
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    E = elems.shape[0]
    Q = tables(kind, degree)["Q"]
    d, k = element_dim(kind), element_nodes(kind)
    out = dict(jac=np.zeros((E, Q, d, d)), det=np.zeros((E, Q)), jac_invT=np.zeros((E, Q, d, d)),
               qpts=np.zeros((E, Q, d)), grads=np.zeros((E, Q, k, d)))
    bad = C.c_int64(-1)
    _check(lib().tgo_geometry(KINDS[kind], _p(nodes), _p(elems), E, degree, _p(out["jac"]),
                              _p(out["det"]), _p(out["jac_invT"]), _p(out["qpts"]),
                              _p(out["grads"]), C.byref(bad)))
    return out


def local(kind, nodes, elems, degree, what, c1, c2=None):
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    E = elems.shape[0]
    kg, d = element_nodes(kind), element_dim(kind)
    if what in (DIFFUSION, MASS):
        shape = (E, kg, kg)
    elif what == ELASTICITY:
        shape = (E, kg * d, kg * d)
    elif what == LOAD:
        shape = (E, kg)
    else:
        shape = (E, kg * d)
    out = np.zeros(shape)
    Q = tables(kind, degree)["Q"]
    c1 = np.ascontiguousarray(c1, dtype=np.float64)
    c2 = None if c2 is None else np.ascontiguousarray(c2, dtype=np.float64)
    per_point = d if what == LOAD_VECTOR else 1  # vector source: d components per point
    for c in (c1, c2):  # per quadrature point (E x Q [x d]); the restatement does not bounds-check
        if c is not None and c.size != E * Q * per_point:
            raise ValueError(f"local: coefficient has {c.size} values, expected {E * Q * per_point}")
    bad = C.c_int64(-1)
    _check(lib().tgo_local(KINDS[kind], _p(nodes), _p(elems), E, degree, what, _p(c1), _p(c2),
                           _p(out), C.byref(bad)))
    return out


class Routing:
    """build_routing (routing.cpp:12-85) restated."""

    def __init__(self, N, dofmap_arr):
        dm = np.ascontiguousarray(dofmap_arr, dtype=np.int64)
        self.E, self.k = dm.shape
        self.N = int(N)
        self.dofmap = dm
        self._h = lib().tgo_routing_build(self.N, self.E, self.k, _p(dm))
        if not self._h:
            raise OracleError(lib().tgo_last_error().decode())
        self.nnz = lib().tgo_routing_nnz(self._h)
        self.offsets = np.zeros(self.N + 1, dtype=np.int64)
        self.cols = np.zeros(self.nnz, dtype=np.int64)
        self.vec_offsets = np.zeros(self.N + 1, dtype=np.uint32)
        self.vec_slots = np.zeros(self.E * self.k, dtype=np.uint32)
        self.mat_offsets = np.zeros(self.nnz + 1, dtype=np.uint32)
        self.mat_slots = np.zeros(self.E * self.k * self.k, dtype=np.uint32)
        lib().tgo_routing_copy(self._h, _p(self.offsets), _p(self.cols), _p(self.vec_offsets),
                               _p(self.vec_slots), _p(self.mat_offsets), _p(self.mat_slots))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().tgo_routing_free(self._h)
            self._h = None

    def slot_of(self):
        """Element-to-CSR-slot map: inverse of mat_slots (slot_of[u] = t)."""
        out = np.empty(self.E * self.k * self.k, dtype=np.int64)
        seg = np.repeat(np.arange(self.nnz, dtype=np.int64), np.diff(self.mat_offsets.astype(np.int64)))
        out[self.mat_slots.astype(np.int64)] = seg
        return out

    def reduce_matrix(self, local_m):
        local_m = np.ascontiguousarray(local_m, dtype=np.float64)
        out = np.zeros(self.nnz)
        lib().tgo_reduce_matrix(self._h, _p(local_m), _p(out))
        return out

    def reduce_vector(self, local_v):
        local_v = np.ascontiguousarray(local_v, dtype=np.float64)
        out = np.zeros(self.N)
        lib().tgo_reduce_vector(self._h, _p(local_v), _p(out))
        return out

    def scatter_add(self, localK, localF):
        vals = np.zeros(self.nnz)
        F = np.zeros(self.N)
        lk = None if localK is None else np.ascontiguousarray(localK, dtype=np.float64)
        lf = None if localF is None else np.ascontiguousarray(localF, dtype=np.float64)
        lib().tgo_scatter_add(self._h, _p(self.dofmap), _p(lk), _p(lf), _p(vals), _p(F))
        return vals, F

    def gradient_products(self, lam, U):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        U = np.ascontiguousarray(U, dtype=np.float64)
        dK = np.zeros(self.nnz)
        dF = np.zeros(self.N)
        lib().tgo_gradient_products(self._h, _p(lam), _p(U), _p(dK), _p(dF))
        return dK, dF

    def adjoint_generic(self, K0, dK):
        K0 = np.ascontiguousarray(K0, dtype=np.float64)
        dK = np.ascontiguousarray(dK, dtype=np.float64)
        out = np.zeros(self.E)
        lib().tgo_adjoint_generic(self._h, _p(self.dofmap), _p(K0), _p(dK), _p(out))
        return out


def adjoint_gather(dofmap_arr, K0, lam, U):
    dm = np.ascontiguousarray(dofmap_arr, dtype=np.int64)
    E, k = dm.shape
    K0 = np.ascontiguousarray(K0, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros(E)
    lib().tgo_adjoint_gather(E, k, _p(dm), _p(K0), _p(lam), _p(U), _p(out))
    return out


PROBLEMS = {"poisson": 0, "elasticity": 1, "mass": 2}


def assemble(kind, nodes, elems, routing, problem="poisson", diffusion=1.0, lam=1.0, mu=1.0,
             plane_stress=False, sources=(), with_mass=False):
    """assemble (physics.cpp:10-75) restated.  Returns (K_values, F, M_values|None)."""
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int64)
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
    _check(lib().tgo_assemble(KINDS[kind], _p(nodes), nodes.shape[0], _p(elems), elems.shape[0],
                              routing._h, PROBLEMS[problem], C.byref(fd), C.byref(fl), C.byref(fm),
                              int(plane_stress), len(sources), srcs, int(with_mass), _p(K), _p(F),
                              _p(M)))
    return K, F, M


def simp_sensitivity(dofmap_arr, rho, p, E_min, E_max, K0, U):
    """simp_sensitivity (adjoint.cpp:101-125) restated (pure Python floats, the
    reference's operation order; small sizes only)."""
    dm = np.asarray(dofmap_arr, dtype=np.int64)
    E, k = dm.shape
    K0 = np.asarray(K0, dtype=np.float64).reshape(E, k, k)
    out = np.zeros(E)
    for e in range(E):
        ue = [float(U[g]) for g in dm[e]]
        quad = 0.0
        for a in range(k):
            row = 0.0
            for b in range(k):
                row += float(K0[e, a, b]) * ue[b]
            quad += ue[a] * row
        out[e] = -p * float(rho[e]) ** (p - 1.0) * (E_max - E_min) * quad
    return out
