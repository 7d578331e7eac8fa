// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (the `tg::` sources
// under /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libtgref.so).  It exists so that Python tests, the golden-vector
// generator and `bench.py --impl reference` can drive the reference's own code
// path through ctypes.  Every entry point forwards to the reference function
// named in its comment; nothing here re-implements reference arithmetic.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "tg/adjoint.hpp"
#include "tg/batch.hpp"
#include "tg/coefficient.hpp"
#include "tg/dofmap.hpp"
#include "tg/errors.hpp"
#include "tg/gmsh_io.hpp"
#include "tg/mesh.hpp"
#include "tg/parallel.hpp"
#include "tg/physics.hpp"
#include "tg/reference.hpp"
#include "tg/routing.hpp"
#include "tg/solver.hpp"
#include "tg/sparse.hpp"

using namespace tg;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const InputError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

ElementKind kind_of(int k) {
    switch (k) {
        case 0: return ElementKind::TRI3;
        case 1: return ElementKind::QUAD4;
        case 2: return ElementKind::TET4;
    }
    throw InputError("unknown element kind code " + std::to_string(k));
}

struct RefRouting {
    DofMap dofmap;
    RoutingMatrices routing;
};

}  // namespace

extern "C" {

typedef struct {
    int type;          // 0 constant, 1 per-element, 2 nodal
    double value;      // constant value
    const double* data;
    std::int64_t n;
} tgr_field;

const char* tgr_last_error(void) { return g_err.c_str(); }

void tgr_set_threads(int n) { set_thread_count(n); }          // parallel.cpp:14
int tgr_thread_count(void) { return thread_count(); }         // parallel.cpp:16

// ---------------------------------------------------------------- mesh
// generate_grid (mesh.cpp:96-169)
int tgr_mesh_grid(int kind, const double* ext, const std::int64_t* div, void** out) {
    return guarded([&] {
        const int d = element_dim(kind_of(kind));
        std::vector<double> e(ext, ext + d);
        std::vector<std::int64_t> v(div, div + d);
        *out = new Mesh(generate_grid(kind_of(kind), e, v));
    });
}

// Mesh from arrays + Mesh::validate (mesh.cpp:56-77); boundary via topological_boundary.
int tgr_mesh_arrays(int kind, const double* nodes, std::int64_t n_nodes, const std::int64_t* elems,
                    std::int64_t n_elems, int validate, void** out) {
    return guarded([&] {
        auto m = std::make_unique<Mesh>();
        m->kind = kind_of(kind);
        m->dim = element_dim(m->kind);
        m->nodes.assign(nodes, nodes + n_nodes * m->dim);
        m->elements.assign(elems, elems + n_elems * element_nodes(m->kind));
        if (validate) {
            m->boundary_nodes = topological_boundary(*m);
            m->validate();
        }
        *out = m.release();
    });
}

int tgr_mesh_load_gmsh(const char* path, void** out) {  // gmsh_io.cpp:64-221
    return guarded([&] { *out = new Mesh(load_gmsh(path)); });
}

int tgr_mesh_write_gmsh(void* mesh, const char* path) {  // gmsh_io.cpp:223-250
    return guarded([&] { write_gmsh(*static_cast<Mesh*>(mesh), path); });
}

void tgr_mesh_free(void* m) { delete static_cast<Mesh*>(m); }

void tgr_mesh_sizes(void* mp, std::int64_t* n_nodes, std::int64_t* n_elems, std::int64_t* n_bnd,
                    int* dim, int* k) {
    const auto& m = *static_cast<Mesh*>(mp);
    *n_nodes = m.node_count();
    *n_elems = m.element_count();
    *n_bnd = static_cast<std::int64_t>(m.boundary_nodes.size());
    *dim = m.dim;
    *k = element_nodes(m.kind);
}

void tgr_mesh_copy(void* mp, double* nodes, std::int64_t* elems, std::int64_t* bnd) {
    const auto& m = *static_cast<Mesh*>(mp);
    if (nodes) std::memcpy(nodes, m.nodes.data(), m.nodes.size() * sizeof(double));
    if (elems) std::memcpy(elems, m.elements.data(), m.elements.size() * sizeof(std::int64_t));
    if (bnd)
        std::memcpy(bnd, m.boundary_nodes.data(), m.boundary_nodes.size() * sizeof(std::int64_t));
}

std::uint64_t tgr_mesh_hash(void* mp) { return static_cast<Mesh*>(mp)->content_hash(); }

// ---------------------------------------------------------------- routing
// build_dofmap (dofmap.cpp:9-25) + build_routing (routing.cpp:12-85)
int tgr_routing(void* mp, int comps, void** out) {
    return guarded([&] {
        auto r = std::make_unique<RefRouting>();
        r->dofmap = build_dofmap(*static_cast<Mesh*>(mp), comps);
        r->routing = build_routing(*static_cast<Mesh*>(mp), r->dofmap);
        *out = r.release();
    });
}

void tgr_routing_free(void* r) { delete static_cast<RefRouting*>(r); }

void tgr_routing_sizes(void* rp, std::int64_t* N, std::int64_t* E, std::int64_t* k,
                       std::int64_t* nnz) {
    const auto& r = static_cast<RefRouting*>(rp)->routing;
    *N = r.N;
    *E = r.E;
    *k = r.k;
    *nnz = r.nnz();
}

void tgr_routing_copy(void* rp, std::int64_t* offsets, std::int64_t* cols, std::uint32_t* vec_off,
                      std::uint32_t* vec_slots, std::uint32_t* mat_off, std::uint32_t* mat_slots,
                      std::int64_t* dofmap) {
    const auto& rr = *static_cast<RefRouting*>(rp);
    const auto& r = rr.routing;
    auto cp = [](auto* dst, const auto& v) {
        if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(offsets, r.pattern->offsets);
    cp(cols, r.pattern->cols);
    cp(vec_off, r.vec_offsets);
    cp(vec_slots, r.vec_slots);
    cp(mat_off, r.mat_offsets);
    cp(mat_slots, r.mat_slots);
    cp(dofmap, rr.dofmap.map);
}

// save_routing / load_routing (routing.cpp:194-234)
int tgr_routing_save(void* rp, std::uint64_t hash, const char* path) {
    return guarded([&] { save_routing(static_cast<RefRouting*>(rp)->routing, hash, path); });
}

// ---------------------------------------------------------------- stage I
int tgr_quadrature(int kind, int degree, int* Q, double* points, double* weights, double* B,
                   double* G) {  // reference_tables (reference.cpp:223-239)
    return guarded([&] {
        const auto t = reference_tables(kind_of(kind), degree);
        *Q = t.rule.Q;
        if (points) std::memcpy(points, t.rule.points.data(), t.rule.points.size() * 8);
        if (weights) std::memcpy(weights, t.rule.weights.data(), t.rule.weights.size() * 8);
        if (B) std::memcpy(B, t.B.data(), t.B.size() * 8);
        if (G) std::memcpy(G, t.G.data(), t.G.size() * 8);
    });
}

int tgr_default_degree(int kind, int mass) {
    return mass ? default_mass_degree(kind_of(kind)) : default_stiffness_degree(kind_of(kind));
}

// batch_geometry (batch.cpp:56-128) + push_forward (batch.cpp:130-154)
int tgr_geometry(void* mp, int degree, double* jac, double* det, double* jac_invT, double* qpts,
                 double* grads) {
    return guarded([&] {
        const auto& m = *static_cast<Mesh*>(mp);
        const auto t = reference_tables(m.kind, degree);
        const auto g = batch_geometry(m, t);
        if (jac) std::memcpy(jac, g.jac.data(), g.jac.size() * 8);
        if (det) std::memcpy(det, g.det.data(), g.det.size() * 8);
        if (jac_invT) std::memcpy(jac_invT, g.jac_invT.data(), g.jac_invT.size() * 8);
        if (qpts) std::memcpy(qpts, g.phys_qpoints.data(), g.phys_qpoints.size() * 8);
        if (grads) {
            const auto pg = push_forward(g, t);
            std::memcpy(grads, pg.G.data(), pg.G.size() * 8);
        }
    });
}

// what: 0 local_stiffness_diffusion (batch.cpp:156-181), c1 = coeff E x Q
//       1 local_stiffness_elasticity (batch.cpp:183-248), c1 = lambda, c2 = mu (E x Q)
//       2 local_mass (batch.cpp:250-269), c1 = coeff
//       3 local_load (batch.cpp:271-289), c1 = source E x Q
//       4 local_load_vector (batch.cpp:291-312), c1 = source E x Q x d
int tgr_local(void* mp, int degree, int what, const double* c1, const double* c2, double* out) {
    return guarded([&] {
        const auto& m = *static_cast<Mesh*>(mp);
        const auto t = reference_tables(m.kind, degree);
        const auto g = batch_geometry(m, t);
        const std::size_t nq = static_cast<std::size_t>(g.E) * g.Q;
        std::vector<double> res;
        if (what == 0 || what == 1) {
            const auto pg = push_forward(g, t);
            if (what == 0) {
                res = local_stiffness_diffusion(g, pg, std::vector<double>(c1, c1 + nq), t);
            } else {
                res = local_stiffness_elasticity(g, pg, std::vector<double>(c1, c1 + nq),
                                                 std::vector<double>(c2, c2 + nq), t);
            }
        } else if (what == 2) {
            res = local_mass(g, std::vector<double>(c1, c1 + nq), t);
        } else if (what == 3) {
            res = local_load(g, std::vector<double>(c1, c1 + nq), t);
        } else if (what == 4) {
            res = local_load_vector(g, std::vector<double>(c1, c1 + nq * g.d), t);
        } else {
            throw InputError("tgr_local: unknown kernel");
        }
        std::memcpy(out, res.data(), res.size() * 8);
    });
}

// Allen-Cahn Newton re-assembly exactly as AllenCahnStepper does it
// (timestep.cpp:118-135 tables/geometry at the mass degree, :144-146 reaction
// load, :177-178 tangent): T = reduce_matrix(local_mass(reaction_tangent_coefficient(u))),
// F = reduce_vector(local_reaction_load(u)).
int tgr_allen_cahn(void* mp, void* rp, const double* u, double eps, double* T, double* F) {
    return guarded([&] {
        const auto& m = *static_cast<Mesh*>(mp);
        const auto& r = static_cast<RefRouting*>(rp)->routing;
        const auto t = reference_tables(m.kind, default_mass_degree(m.kind));
        const auto g = batch_geometry(m, t);
        const std::vector<double> un(u, u + m.node_count());
        const auto tc = reaction_tangent_coefficient(g, m, un, eps, t);    // batch.cpp:344-351
        const auto Tm = reduce_matrix(r, local_mass(g, tc, t));
        const auto Fv = reduce_vector(r, local_reaction_load(g, m, un, eps, t));  // batch.cpp:335-342
        std::memcpy(T, Tm.values.data(), Tm.values.size() * 8);
        std::memcpy(F, Fv.data(), Fv.size() * 8);
    });
}

// condense (solver.cpp:34-85) of a K on the routing's pattern; outputs sized by
// the caller: free/fixed lists and F_f (N), K_ff offsets (N+1), cols/values (nnz).
int tgr_condense(void* rp, const double* K, const double* F, std::int64_t nd, const std::int64_t* dofs,
                 const double* vals, std::int64_t* n_free, std::int64_t* n_fixed, std::int64_t* nnz_ff,
                 std::int64_t* free_dofs, std::int64_t* fixed_dofs, double* prescribed, std::int64_t* offsets,
                 std::int64_t* cols, double* values, double* F_f) {
    return guarded([&] {
        const auto& r = static_cast<RefRouting*>(rp)->routing;
        SparseOperator Kop;
        Kop.pattern = r.pattern;
        Kop.values.assign(K, K + r.nnz());
        const auto sys = condense(Kop, std::vector<double>(F, F + r.N), std::vector<std::int64_t>(dofs, dofs + nd),
                                  std::vector<double>(vals, vals + nd));
        *n_free = static_cast<std::int64_t>(sys.free_dofs.size());
        *n_fixed = static_cast<std::int64_t>(sys.constrained_dofs.size());
        *nnz_ff = static_cast<std::int64_t>(sys.K_ff.values.size());
        std::memcpy(free_dofs, sys.free_dofs.data(), sys.free_dofs.size() * 8);
        std::memcpy(fixed_dofs, sys.constrained_dofs.data(), sys.constrained_dofs.size() * 8);
        std::memcpy(prescribed, sys.prescribed.data(), sys.prescribed.size() * 8);
        std::memcpy(offsets, sys.K_ff.pattern->offsets.data(), sys.K_ff.pattern->offsets.size() * 8);
        std::memcpy(cols, sys.K_ff.pattern->cols.data(), sys.K_ff.pattern->cols.size() * 8);
        std::memcpy(values, sys.K_ff.values.data(), sys.K_ff.values.size() * 8);
        std::memcpy(F_f, sys.F_f.data(), sys.F_f.size() * 8);
    });
}

// bicgstab (solver.cpp:105-227) on a CSR given as arrays
int tgr_bicgstab(std::int64_t n, const std::int64_t* off, const std::int64_t* cols, const double* vals,
                 const double* b, double* x, double tol_rel, double tol_abs, std::int64_t max_iter,
                 std::int64_t* iters, double* rel, int* conv) {
    return guarded([&] {
        auto pat = std::make_shared<CsrPattern>();
        pat->rows = n;
        pat->offsets.assign(off, off + n + 1);
        pat->cols.assign(cols, cols + off[n]);
        SparseOperator A;
        A.pattern = pat;
        A.values.assign(vals, vals + off[n]);
        std::vector<double> xv(x, x + n);
        SolverConfig cfg;
        cfg.tol_rel = tol_rel;
        cfg.tol_abs = tol_abs;
        cfg.max_iter = max_iter;
        const auto rep = bicgstab(A, std::vector<double>(b, b + n), xv, cfg);
        std::memcpy(x, xv.data(), n * 8);
        *iters = rep.iterations;
        *rel = rep.rel_residual;
        *conv = rep.converged ? 1 : 0;
    });
}

// SparseOperator::apply (sparse.cpp:18-31) on the routing's pattern
int tgr_spmv(void* rp, const double* vals, const double* x, double* y) {
    return guarded([&] {
        const auto& r = static_cast<RefRouting*>(rp)->routing;
        SparseOperator A;
        A.pattern = r.pattern;
        A.values.assign(vals, vals + r.nnz());
        const auto out = A.apply(std::vector<double>(x, x + r.N));
        std::memcpy(y, out.data(), out.size() * 8);
    });
}

// ---------------------------------------------------------------- stage II
int tgr_reduce_matrix(void* rp, const double* local, double* values) {  // routing.cpp:109-125
    return guarded([&] {
        const auto& r = static_cast<RefRouting*>(rp)->routing;
        const std::size_t n = static_cast<std::size_t>(r.E) * r.k * r.k;
        const auto K = reduce_matrix(r, std::vector<double>(local, local + n));
        std::memcpy(values, K.values.data(), K.values.size() * 8);
    });
}

int tgr_reduce_vector(void* rp, const double* local, double* F) {  // routing.cpp:87-100
    return guarded([&] {
        const auto& r = static_cast<RefRouting*>(rp)->routing;
        const std::size_t n = static_cast<std::size_t>(r.E) * r.k;
        const auto v = reduce_vector(r, std::vector<double>(local, local + n));
        std::memcpy(F, v.data(), v.size() * 8);
    });
}

// scatter_add_oracle (routing.cpp:134-175). Pattern sizes equal the routing's.
int tgr_scatter_add(void* mp, void* rp, const double* localK, const double* localF,
                    std::int64_t* offsets, std::int64_t* cols, double* values, double* F) {
    return guarded([&] {
        const auto& rr = *static_cast<RefRouting*>(rp);
        const auto& r = rr.routing;
        const std::size_t nk = static_cast<std::size_t>(r.E) * r.k;
        SparseOperator K;
        std::vector<double> Fv;
        scatter_add_oracle(*static_cast<Mesh*>(mp), rr.dofmap,
                           localK ? std::vector<double>(localK, localK + nk * r.k)
                                  : std::vector<double>{},
                           localF ? std::vector<double>(localF, localF + nk) : std::vector<double>{},
                           K, Fv);
        if (offsets) std::memcpy(offsets, K.pattern->offsets.data(), K.pattern->offsets.size() * 8);
        if (cols) std::memcpy(cols, K.pattern->cols.data(), K.pattern->cols.size() * 8);
        if (values && localK) std::memcpy(values, K.values.data(), K.values.size() * 8);
        if (F && localF) std::memcpy(F, Fv.data(), Fv.size() * 8);
    });
}

// ---------------------------------------------------------------- assemble
namespace {
CoefficientField field_of(const tgr_field& f) {
    switch (f.type) {
        case 0: return CoefficientField::constant(f.value);
        case 1: return CoefficientField::per_element(std::vector<double>(f.data, f.data + f.n));
        case 2: return CoefficientField::nodal(std::vector<double>(f.data, f.data + f.n));
        // the reference's own Analytic fields (physics.cpp:77-107)
        case 3: return checkerboard_source(static_cast<int>(f.value));
        case 4: return multi_sine_field(static_cast<int>(f.n), f.value, 7);
    }
    throw InputError("unknown field type");
}
thread_local int g_pattern_shared = -1;
}  // namespace

// 1 if the last tgr_assemble returned K (and M) on the routing's own pattern
// pointer (routing.cpp:114; checked by timestep.cpp:140, adjoint.cpp:73), else 0.
int tgr_last_pattern_shared() { return g_pattern_shared; }

// assemble (physics.cpp:10-75).  problem: 0 Poisson, 1 elasticity, 2 mass.
// seconds: steady_clock duration of the assemble() call alone.
int tgr_assemble(void* mp, void* rp, int problem, const tgr_field* diffusion,
                 const tgr_field* lambda, const tgr_field* mu, int plane_stress, int n_source,
                 const tgr_field* sources, int with_mass, double* K, double* F, double* M,
                 double* seconds) {
    return guarded([&] {
        const auto& m = *static_cast<Mesh*>(mp);
        const auto& rr = *static_cast<RefRouting*>(rp);
        ProblemSpec ps;
        ps.kind = problem == 0   ? ProblemKind::PoissonDiffusion
                  : problem == 1 ? ProblemKind::LinearElasticity
                                 : ProblemKind::Mass;
        if (diffusion) ps.diffusion = field_of(*diffusion);
        if (lambda) ps.lambda = field_of(*lambda);
        if (mu) ps.mu = field_of(*mu);
        ps.plane_stress = plane_stress != 0;
        for (int s = 0; s < n_source; ++s) ps.source.push_back(field_of(sources[s]));
        const auto t0 = std::chrono::steady_clock::now();
        const auto sys = assemble(ps, m, rr.dofmap, rr.routing, with_mass != 0);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        g_pattern_shared = sys.K.pattern.get() == rr.routing.pattern.get() &&
                           (!sys.M || sys.M->pattern.get() == rr.routing.pattern.get()) && sys.K.symmetric &&
                           (!sys.M || sys.M->symmetric);
        if (K) std::memcpy(K, sys.K.values.data(), sys.K.values.size() * 8);
        if (F) std::memcpy(F, sys.F.data(), sys.F.size() * 8);
        if (M && sys.M) std::memcpy(M, sys.M->values.data(), sys.M->values.size() * 8);
    });
}

// gradient_products (adjoint.cpp:68-82) on the routing's pattern.
int tgr_gradient_products(void* rp, const double* lambda, const double* U, double* dK,
                          double* dF) {
    return guarded([&] {
        const auto& r = static_cast<RefRouting*>(rp)->routing;
        SparseOperator K;
        K.pattern = r.pattern;
        K.values.assign(static_cast<std::size_t>(r.nnz()), 0.0);
        const std::size_t N = static_cast<std::size_t>(r.N);
        const auto g = gradient_products(K, std::vector<double>(lambda, lambda + N),
                                         std::vector<double>(U, U + N));
        std::memcpy(dK, g.dK.values.data(), g.dK.values.size() * 8);
        if (dF) std::memcpy(dF, g.dF.data(), g.dF.size() * 8);
    });
}

// simp_sensitivity (adjoint.cpp:101-125): -p rho^{p-1} (Emax-Emin) u_e^T K0_e u_e
int tgr_simp_sensitivity(void* mp, void* rp, const double* rho, double p, double E_min,
                         double E_max, const double* K0, const double* U, double* out) {
    return guarded([&] {
        const auto& m = *static_cast<Mesh*>(mp);
        const auto& rr = *static_cast<RefRouting*>(rp);
        const std::size_t E = static_cast<std::size_t>(m.element_count());
        const std::size_t k = static_cast<std::size_t>(rr.dofmap.k);
        const auto s = simp_sensitivity(std::vector<double>(rho, rho + E), p, E_min, E_max,
                                        std::vector<double>(K0, K0 + E * k * k), m, rr.dofmap,
                                        std::vector<double>(U, U + rr.dofmap.N));
        std::memcpy(out, s.data(), E * 8);
    });
}

}  // extern "C"
