"""Device-resident API over libtgk.so, with torch tensors as the buffers.

PyTorch supplies CUDA memory and streams only; every computation runs in the
hand-written sm_100a kernels of libtgk.so.  Names follow the reference's C++
API (tg::assemble, build_routing, reduce_matrix, gradient_products, ...).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from ._native import check, lib

_DEV = torch.device("cuda")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _cuda_f64(x, n=None):
    t = torch.as_tensor(x, dtype=torch.float64, device=_DEV).contiguous()
    if n is not None and t.numel() != n:
        raise N.InputError(f"expected {n} values, got {t.numel()}")
    return t


def field(spec, keep):
    """float | ('element', values) | ('nodal', values) -> (Field, keepalive list)."""
    if spec is None:
        return N.Field(N.FIELD_CONSTANT, 1.0, None, 0)
    if isinstance(spec, (int, float)):
        return N.Field(N.FIELD_CONSTANT, float(spec), None, 0)
    kind, vals = spec
    t = _cuda_f64(vals).reshape(-1)
    keep.append(t)
    ftype = {"element": N.FIELD_ELEMENT, "nodal": N.FIELD_NODAL}[kind]
    return N.Field(ftype, 0.0, C.c_void_p(t.data_ptr()), t.numel())


class DeviceMesh:
    """A tg::Mesh resident on the GPU (fp64 node-major coordinates, int32 connectivity)."""

    def __init__(self, kind, nodes, elements):
        self.kind = kind.lower() if isinstance(kind, str) else N.KIND_NAMES[kind].lower()
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        elements = np.ascontiguousarray(elements, dtype=np.int64)
        self.N, self.dim = nodes.shape
        self.E, self.k = elements.shape
        h = C.c_void_p()
        check(lib().tgk_mesh_create(N.KINDS[self.kind], nodes.ctypes.data, self.N,
                                    elements.ctypes.data, self.E, C.byref(h)))
        self._h = h
        self._keep = None

    @classmethod
    def from_device(cls, kind, nodes: torch.Tensor, conn: torch.Tensor):
        """Wrap device tensors (float64 N x d, int32 E x k) without copying."""
        self = cls.__new__(cls)
        self.kind = kind
        nodes = nodes.contiguous()
        conn = conn.to(torch.int32).contiguous()
        self.N, self.dim = nodes.shape
        self.E, self.k = conn.shape
        h = C.c_void_p()
        check(lib().tgk_mesh_create_d(N.KINDS[kind], nodes.data_ptr(), self.N, conn.data_ptr(),
                                      self.E, C.byref(h)))
        self._h = h
        self._keep = (nodes, conn)
        return self

    def upload(self, nodes=None, elements=None, stream=None):
        """Host -> device copy of new coordinates / connectivity (same sizes)."""
        np_n = None if nodes is None else np.ascontiguousarray(nodes, dtype=np.float64)
        np_e = None if elements is None else np.ascontiguousarray(elements, dtype=np.int64)
        check(lib().tgk_mesh_upload(self._h, None if np_n is None else np_n.ctypes.data,
                                    None if np_e is None else np_e.ctypes.data, _stream(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tgk_mesh_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self._h = None


class Routing:
    """build_dofmap + build_routing on the GPU (routing.cpp:12-85), bit-identical."""

    def __init__(self, mesh: DeviceMesh, components=1, segments=False, stream=None):
        self.mesh = mesh
        h = C.c_void_p()
        check(lib().tgk_routing_build(mesh._h, int(components), N.ROUTING_SEGMENTS if segments else 0,
                                      _stream(stream), C.byref(h)))
        self._h = h
        v = N.RoutingView()
        check(lib().tgk_routing_get_view(h, C.byref(v)))
        self.N, self.E, self.nnz, self.k = v.N, v.E, v.nnz, v.k
        self.components = v.components
        self.has_segments = bool(v.mat_offsets)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tgk_routing_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    def host_arrays(self, slot_of=True, segments=None):
        """Reference-layout arrays copied to host numpy (RoutingMatrices + CsrPattern)."""
        segments = self.has_segments if segments is None else segments
        Ek = self.E * self.k
        out = dict(offsets=np.zeros(self.N + 1, np.int64), cols=np.zeros(self.nnz, np.int64))
        want_slot = slot_of and self.components == 1
        if want_slot:
            out["slot_of"] = np.zeros(Ek * self.k, np.uint32)
        if segments:
            out.update(vec_offsets=np.zeros(self.N + 1, np.uint32), vec_slots=np.zeros(Ek, np.uint32),
                       mat_offsets=np.zeros(self.nnz + 1, np.uint32),
                       mat_slots=np.zeros(Ek * self.k, np.uint32))
        g = lambda k: out[k].ctypes.data if k in out else None  # noqa: E731
        check(lib().tgk_routing_copy(self._h, g("offsets"), g("cols"), g("slot_of"), g("vec_offsets"),
                                     g("vec_slots"), g("mat_offsets"), g("mat_slots")))
        return out

    def save(self, mesh_hash, path):
        """save_routing (routing.cpp:194-209): the reference's "tg-rout2" cache file."""
        check(lib().tgk_routing_save(self._h, C.c_uint64(mesh_hash), str(path).encode()))

    @classmethod
    def load(cls, mesh: DeviceMesh, mesh_hash, path, components=1, stream=None):
        """load_routing (routing.cpp:211-234): a Routing, or None on a cache miss."""
        h, hit = C.c_void_p(), C.c_int(0)
        check(lib().tgk_routing_load(mesh._h, int(components), C.c_uint64(mesh_hash), str(path).encode(),
                                     _stream(stream), C.byref(hit), C.byref(h)))
        if not hit.value:
            return None
        self = cls.__new__(cls)
        self.mesh = mesh
        self._h = h
        v = N.RoutingView()
        check(lib().tgk_routing_get_view(h, C.byref(v)))
        self.N, self.E, self.nnz, self.k = v.N, v.E, v.nnz, v.k
        self.components = v.components
        self.has_segments = bool(v.mat_offsets)
        return self


MODES = {"exact": 0, "fast": 1}


def make_problem(kind="poisson", diffusion=1.0, lam=1.0, mu=1.0, plane_stress=False, sources=(),
                 with_mass=False, keep=None, mode="exact"):
    keep = [] if keep is None else keep
    p = N.Problem()
    p.kind = {"poisson": N.POISSON, "elasticity": N.ELASTICITY, "mass": N.MASS}[kind]
    p.diffusion = field(diffusion, keep)
    p.lam = field(lam, keep)
    p.mu = field(mu, keep)
    p.plane_stress = int(bool(plane_stress))
    p.n_source = len(sources)
    for i, s in enumerate(sources):
        p.source[i] = field(s, keep)
    p.with_mass = int(bool(with_mass))
    p.mode = MODES[mode]
    return p, keep


def assemble(mesh: DeviceMesh, routing: Routing, kind="poisson", diffusion=1.0, lam=1.0, mu=1.0,
             plane_stress=False, sources=(), with_mass=False, dtype=torch.float64, out=None, stream=None,
             mode="exact"):
    """tg::assemble (physics.cpp:10-75) on the GPU.  Returns (K values, F, M values | None).
    mode="exact": bit-identical to the reference; mode="fast": within the 1e-12
    scaled tolerance of SURVEY.md 8(c), deterministic (TGK_MODE_FAST).
    dtype=torch.float32 runs the fp32 variant (tgk_assemble_f32_d, scalar problems).
    A Mass problem returns no M (physics.cpp:25-31 returns before with_mass)."""
    if kind == "mass":
        with_mass = False
    p, keep = make_problem(kind, diffusion, lam, mu, plane_stress, sources, with_mass, mode=mode)
    if out is None:
        K = torch.empty(routing.nnz, dtype=dtype, device=_DEV)
        F = torch.empty(routing.N, dtype=dtype, device=_DEV)
        M = torch.empty(routing.nnz, dtype=dtype, device=_DEV) if with_mass else None
    else:
        K, F, M = out
    if dtype == torch.float32:
        check(lib().tgk_assemble_f32_d(C.byref(p), mesh._h, routing._h, _ptr(K), _ptr(F), _ptr(M), None,
                                       _stream(stream)))
    else:
        check(lib().tgk_assemble_d(C.byref(p), mesh._h, routing._h, _ptr(K), _ptr(F), _ptr(M), _stream(stream)))
    del keep
    return K, F, M


def assemble_host(mesh: DeviceMesh, routing: Routing, kind="poisson", diffusion=1.0, lam=1.0,
                  mu=1.0, plane_stress=False, sources=(), with_mass=False, out=None, mode="exact"):
    """Same as assemble() through the host-buffer C-ABI entry (copies inside the call)."""
    keep = []
    if kind == "mass":
        with_mass = False

    def hfield(spec):
        if spec is None or isinstance(spec, (int, float)):
            return N.Field(N.FIELD_CONSTANT, 1.0 if spec is None else float(spec), None, 0)
        kind_, vals = spec
        a = np.ascontiguousarray(vals, dtype=np.float64).reshape(-1)
        keep.append(a)
        return N.Field({"element": N.FIELD_ELEMENT, "nodal": N.FIELD_NODAL}[kind_], 0.0,
                       a.ctypes.data, a.size)

    p = N.Problem()
    p.kind = {"poisson": N.POISSON, "elasticity": N.ELASTICITY, "mass": N.MASS}[kind]
    p.diffusion, p.lam, p.mu = hfield(diffusion), hfield(lam), hfield(mu)
    p.plane_stress = int(bool(plane_stress))
    p.n_source = len(sources)
    for i, s in enumerate(sources):
        p.source[i] = hfield(s)
    p.with_mass = int(bool(with_mass))
    p.mode = MODES[mode]
    if out is None:
        K = np.empty(routing.nnz)
        F = np.empty(routing.N)
        M = np.empty(routing.nnz) if with_mass else None
    else:
        K, F, M = out
    check(lib().tgk_assemble(C.byref(p), mesh._h, routing._h, K.ctypes.data, F.ctypes.data,
                             None if M is None else M.ctypes.data))
    return K, F, M


# ---------------------------------------------------------------- Stage I / II, materialised
def quadrature_count(kind, degree):
    Q = C.c_int()
    check(lib().tgk_tables(N.KINDS[kind], degree, C.byref(Q), None, None, None, None))
    return Q.value


def geometry(mesh: DeviceMesh, degree, stream=None):
    """batch_geometry + push_forward (batch.cpp:56-154): dict of E x Q x ... tensors."""
    Q = quadrature_count(mesh.kind, degree)
    E, d, k = mesh.E, mesh.dim, mesh.k
    z = lambda *s: torch.empty(*s, dtype=torch.float64, device=_DEV)  # noqa: E731
    out = dict(jac=z(E, Q, d, d), det=z(E, Q), jac_invT=z(E, Q, d, d), qpts=z(E, Q, d),
               grads=z(E, Q, k, d))
    check(lib().tgk_geometry_d(mesh._h, degree, _ptr(out["jac"]), _ptr(out["det"]),
                               _ptr(out["jac_invT"]), _ptr(out["qpts"]), _ptr(out["grads"]),
                               _stream(stream)))
    return out


def _table(x, mesh, degree, per=1):
    Q = quadrature_count(mesh.kind, degree)
    return _cuda_f64(x, mesh.E * Q * per)


def local_stiffness_diffusion(mesh, degree, coeff_eq, stream=None):
    c = _table(coeff_eq, mesh, degree)
    out = torch.empty(mesh.E, mesh.k, mesh.k, dtype=torch.float64, device=_DEV)
    check(lib().tgk_local_stiffness_diffusion_d(mesh._h, degree, _ptr(c), _ptr(out), _stream(stream)))
    return out


def local_stiffness_elasticity(mesh, degree, lam_eq, mu_eq, stream=None):
    lam = _table(lam_eq, mesh, degree)
    mu = _table(mu_eq, mesh, degree)
    kk = mesh.k * mesh.dim
    out = torch.empty(mesh.E, kk, kk, dtype=torch.float64, device=_DEV)
    check(lib().tgk_local_stiffness_elasticity_d(mesh._h, degree, _ptr(lam), _ptr(mu), _ptr(out),
                                                 _stream(stream)))
    return out


def local_mass(mesh, degree, coeff_eq, stream=None):
    c = _table(coeff_eq, mesh, degree)
    out = torch.empty(mesh.E, mesh.k, mesh.k, dtype=torch.float64, device=_DEV)
    check(lib().tgk_local_mass_d(mesh._h, degree, _ptr(c), _ptr(out), _stream(stream)))
    return out


def local_load(mesh, degree, source_eq, stream=None):
    s = _table(source_eq, mesh, degree)
    out = torch.empty(mesh.E, mesh.k, dtype=torch.float64, device=_DEV)
    check(lib().tgk_local_load_d(mesh._h, degree, _ptr(s), _ptr(out), _stream(stream)))
    return out


def local_load_vector(mesh, degree, source_eqc, stream=None):
    s = _table(source_eqc, mesh, degree, per=mesh.dim)
    out = torch.empty(mesh.E, mesh.k * mesh.dim, dtype=torch.float64, device=_DEV)
    check(lib().tgk_local_load_vector_d(mesh._h, degree, _ptr(s), _ptr(out), _stream(stream)))
    return out


def evaluate_field(mesh, degree, spec, stream=None):
    keep = []
    f = field(spec, keep)
    Q = quadrature_count(mesh.kind, degree)
    out = torch.empty(mesh.E, Q, dtype=torch.float64, device=_DEV)
    check(lib().tgk_evaluate_field_d(mesh._h, degree, C.byref(f), _ptr(out), _stream(stream)))
    return out


def reduce_matrix(routing: Routing, local, stream=None):
    loc = _cuda_f64(local, routing.E * routing.k * routing.k)
    out = torch.empty(routing.nnz, dtype=torch.float64, device=_DEV)
    check(lib().tgk_reduce_matrix_d(routing._h, _ptr(loc), _ptr(out), _stream(stream)))
    return out


def reduce_vector(routing: Routing, local, stream=None):
    loc = _cuda_f64(local, routing.E * routing.k)
    out = torch.empty(routing.N, dtype=torch.float64, device=_DEV)
    check(lib().tgk_reduce_vector_d(routing._h, _ptr(loc), _ptr(out), _stream(stream)))
    return out


# ---------------------------------------------------------------- batched + adjoint
def assemble_batched(mesh, routing, rho, source=1.0, with_load=True, stream=None, mode="exact"):
    """B per-element coefficient fields (B x E) -> K values (B x nnz) [+ one F (N)]."""
    rho = _cuda_f64(rho).reshape(-1, mesh.E)
    B = rho.shape[0]
    K = torch.empty(B, routing.nnz, dtype=torch.float64, device=_DEV)
    F = torch.empty(routing.N, dtype=torch.float64, device=_DEV) if with_load else None
    check(lib().tgk_assemble_batched_d(mesh._h, routing._h, B, _ptr(rho), float(source), _ptr(K),
                                       _ptr(F), MODES[mode], _stream(stream)))
    return K, F


def assemble_fields_batched(mesh, routing, fields, kind="poisson", diffusion=1.0, lam=1.0, mu=1.0,
                            plane_stress=False, sources=(), with_mass=False, with_load=True, stream=None,
                            mode="exact"):
    """Batched assembly over coefficient fields for any problem kind
    (tgk_assemble_fields_batched_d): `fields` maps a slot ("diffusion", "lam",
    "mu", "source0".."source2") to a B x E per-element tensor; member b is the
    problem with those slots set to row b.  Returns K (B x nnz), F (B x N | None),
    M (B x nnz | None), stacked member-major."""
    if kind == "mass":
        with_mass = False
    p, keep = make_problem(kind, diffusion, lam, mu, plane_stress, sources, with_mass, mode=mode)
    rows = {k: _cuda_f64(v).reshape(-1, mesh.E) for k, v in fields.items()}
    Bs = {v.shape[0] for v in rows.values()}
    if len(Bs) != 1:
        raise ValueError("every batched field needs the same batch size")
    B = Bs.pop()
    fb = (N.FieldBatch * max(1, len(rows)))()
    for i, (slot, v) in enumerate(rows.items()):
        fb[i] = N.FieldBatch(N.SLOTS[slot], v.data_ptr(), mesh.E)
    K = torch.empty(B, routing.nnz, dtype=torch.float64, device=_DEV)
    F = torch.empty(B, routing.N, dtype=torch.float64, device=_DEV) if with_load else None
    M = torch.empty(B, routing.nnz, dtype=torch.float64, device=_DEV) if with_mass else None
    check(lib().tgk_assemble_fields_batched_d(C.byref(p), mesh._h, routing._h, B, fb, len(rows), _ptr(K),
                                              _ptr(F), _ptr(M), _stream(stream)))
    del keep, rows
    return K, F, M


def simp_sensitivity(dof_map, rho, p, E_min, E_max, unit_stiffness, U, stream=None):
    """simp_sensitivity (adjoint.cpp:101-125) on the GPU: dof_map E x k (the
    DofMap's element-to-DoF array), unit_stiffness E x k x k, U (n_dofs)."""
    dm = torch.as_tensor(np.ascontiguousarray(dof_map, dtype=np.int64)).to(_DEV)
    E, k = dm.shape
    rho = _cuda_f64(rho, E)
    K0 = _cuda_f64(unit_stiffness, E * k * k)
    U = _cuda_f64(U)
    out = torch.empty(E, dtype=torch.float64, device=_DEV)
    check(lib().tgk_simp_sensitivity_d(E, k, _ptr(dm), _ptr(rho), float(p), float(E_min), float(E_max), _ptr(K0),
                                       _ptr(U), U.numel(), _ptr(out), _stream(stream)))
    return out


def gradient_products(routing, lam, U, stream=None):
    """gradient_products (adjoint.cpp:68-82), batched: lam, U (B x N) -> dK (B x nnz), dF (B x N)."""
    lam = _cuda_f64(lam).reshape(-1, routing.N)
    U = _cuda_f64(U).reshape(-1, routing.N)
    B = lam.shape[0]
    dK = torch.empty(B, routing.nnz, dtype=torch.float64, device=_DEV)
    dF = torch.empty(B, routing.N, dtype=torch.float64, device=_DEV)
    check(lib().tgk_gradient_products_d(routing._h, B, _ptr(lam), _ptr(U), _ptr(dK), _ptr(dF),
                                        _stream(stream)))
    return dK, dF


def adjoint_gather(mesh, routing, lam, U, degree=1, stream=None):
    """dGamma/drho[b,e] = lambda_e^T K0_e U_e (tg_main.cpp:846-850), K0 recomputed in registers."""
    lam = _cuda_f64(lam).reshape(-1, routing.N)
    U = _cuda_f64(U).reshape(-1, routing.N)
    B = lam.shape[0]
    out = torch.empty(B, mesh.E, dtype=torch.float64, device=_DEV)
    check(lib().tgk_adjoint_gather_d(mesh._h, routing._h, B, _ptr(lam), _ptr(U), _ptr(out),
                                     int(degree), _stream(stream)))
    return out


def allen_cahn(mesh, routing, u, eps, with_load=True, stream=None):
    """AllenCahnStepper Newton re-assembly (timestep.cpp:144-178), fused: tangent-mass values T
    (nnz) and reaction load F (N) for the nodal state u."""
    u = _cuda_f64(u, routing.N)
    T = torch.empty(routing.nnz, dtype=torch.float64, device=_DEV)
    F = torch.empty(routing.N, dtype=torch.float64, device=_DEV) if with_load else None
    check(lib().tgk_allen_cahn_d(mesh._h, routing._h, _ptr(u), float(eps), _ptr(T), _ptr(F), _stream(stream)))
    return T, F


# ---------------------------------------------------------------- consumers of the CSR
def _csr_device(routing):
    if not hasattr(routing, "_csr_dev"):
        h = routing.host_arrays(slot_of=False, segments=False)
        routing._csr_dev = (torch.from_numpy(h["offsets"]).to(_DEV), torch.from_numpy(h["cols"]).to(_DEV))
    return routing._csr_dev


def spmv(routing, values, x, stream=None):
    """SparseOperator::apply (sparse.cpp:18-31) on the routing's pattern."""
    off, cols = _csr_device(routing)
    x = _cuda_f64(x, routing.N)
    y = torch.empty(routing.N, dtype=torch.float64, device=_DEV)
    check(lib().tgk_spmv_d(routing.N, _ptr(off), _ptr(cols), _ptr(values), _ptr(x), _ptr(y), _stream(stream)))
    return y


class Condensed:
    """condense (solver.cpp:34-85) on the device: K_ff pattern and values, F_f, free /
    constrained DoFs and prescribed values, held by a libtgk handle."""

    def __init__(self, routing, K, F, dofs, values, stream=None):
        off, cols = _csr_device(routing)
        d = torch.as_tensor(np.asarray(dofs, dtype=np.int64)).to(_DEV)
        v = _cuda_f64(values, d.numel())
        h = C.c_void_p()
        check(lib().tgk_condense_d(routing.N, _ptr(off), _ptr(cols), _ptr(K), _ptr(F), d.numel(), _ptr(d), _ptr(v),
                                   _stream(stream), C.byref(h)))
        self._h, self._routing = h, routing
        nf, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().tgk_condensed_info(h, C.byref(nf), C.byref(nc), C.byref(nz), *([None] * 8)))
        self.n_free, self.n_fixed, self.nnz_ff = nf.value, nc.value, nz.value

    def arrays(self):
        """Host copies: free_dofs, fixed_dofs, prescribed, offsets, cols, values, F_f."""
        out = dict(free_dofs=np.empty(self.n_free, np.int64), fixed_dofs=np.empty(self.n_fixed, np.int64),
                   prescribed=np.empty(self.n_fixed), offsets=np.empty(self.n_free + 1, np.int64),
                   cols=np.empty(self.nnz_ff, np.int64), values=np.empty(self.nnz_ff), F_f=np.empty(self.n_free))
        check(lib().tgk_condensed_copy(self._h, *[out[k].ctypes.data for k in
                                                  ["free_dofs", "fixed_dofs", "prescribed", "offsets", "cols",
                                                   "values", "F_f"]]))
        return out

    def restrict_to_free(self, A, stream=None):
        """restrict_to_free (solver.cpp:87-103) of another operator on the routing's pattern."""
        off, cols = _csr_device(self._routing)
        out = torch.empty(self.nnz_ff, dtype=torch.float64, device=_DEV)
        check(lib().tgk_restrict_to_free_d(self._h, _ptr(off), _ptr(cols), _ptr(A), _ptr(out), _stream(stream)))
        return out

    def expand(self, u_free, stream=None):
        """CondensedSystem::expand (solver.cpp:20-26)."""
        u_free = _cuda_f64(u_free, self.n_free)
        u = torch.empty(self._routing.N, dtype=torch.float64, device=_DEV)
        check(lib().tgk_expand_d(self._h, _ptr(u_free), _ptr(u), _stream(stream)))
        return u

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tgk_condensed_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None


def bicgstab(offsets, cols, values, b, x0=None, tol_rel=1e-10, tol_abs=1e-10, max_iter=10000, stream=None):
    """bicgstab (solver.cpp:105-227) on a device CSR (offsets, cols, values: torch CUDA tensors).
    Returns (x, report dict) like tg::SolveReport."""
    n = offsets.numel() - 1
    b = _cuda_f64(b, n)
    x = torch.zeros(n, dtype=torch.float64, device=_DEV) if x0 is None else _cuda_f64(x0, n).clone()
    it, rel, conv = C.c_int64(), C.c_double(), C.c_int()
    check(lib().tgk_bicgstab_d(n, _ptr(offsets), _ptr(cols), _ptr(values), _ptr(b), _ptr(x), float(tol_rel),
                               float(tol_abs), int(max_iter), C.byref(it), C.byref(rel), C.byref(conv),
                               _stream(stream)))
    return x, {"iterations": it.value, "rel_residual": rel.value, "converged": bool(conv.value)}


def solve_condensed(cond, tol_rel=1e-10, tol_abs=1e-10, max_iter=10000, stream=None):
    """Solve K_ff u_f = F_f on the device and expand with the prescribed values
    (solve_condensed solver.cpp:268-292, BiCGSTAB path; the reference switches to a
    dense LU below 2000 free DoFs, which is not ported)."""
    off = torch.empty(cond.n_free + 1, dtype=torch.int64, device=_DEV)
    cols = torch.empty(cond.nnz_ff, dtype=torch.int64, device=_DEV)
    vals = torch.empty(cond.nnz_ff, dtype=torch.float64, device=_DEV)
    F_f = torch.empty(cond.n_free, dtype=torch.float64, device=_DEV)
    ptrs = [C.c_void_p() for _ in range(7)]
    check(lib().tgk_condensed_info(cond._h, None, None, None, *[C.byref(p) for p in ptrs]))
    for t, pp, n, es in [(off, ptrs[3], cond.n_free + 1, 8), (cols, ptrs[4], cond.nnz_ff, 8),
                         (vals, ptrs[5], cond.nnz_ff, 8), (F_f, ptrs[6], cond.n_free, 8)]:
        if n:
            _copy_d2d(t, pp.value, n * es)
    u_f, rep = bicgstab(off, cols, vals, F_f, tol_rel=tol_rel, tol_abs=tol_abs, max_iter=max_iter, stream=stream)
    return cond.expand(u_f, stream=stream), rep


def _copy_d2d(dst, src_ptr, nbytes, stream=None):
    check(lib().tgk_copy_d2d(_ptr(dst), C.c_void_p(src_ptr), C.c_int64(nbytes), _stream(stream)))
