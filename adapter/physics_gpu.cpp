// GPU drop-in for tg::assemble (proj/include/tg/physics.hpp:55-56,
// proj/src/physics.cpp:10-75): the reference's C++ assembly API, unchanged
// signature and semantics, computed by libtgk through its C ABI (include/tgk.h).
//
// Compiled against the UNMODIFIED reference headers (-I proj/include).  A
// maintainer links this object in place of physics.cpp's assemble (either by
// deleting that function from physics.cpp, or — as oracle/Makefile does for the
// tests — by renaming the reference symbol to tg::assemble_cpu with objcopy, in
// which case QUAD4 meshes, which libtgk does not assemble, are delegated to it).
//
// Contract kept from the reference:
//  - same checks and exception types / messages (InputError, NumericalError);
//  - K.pattern = M.pattern = routing.pattern — the SAME shared_ptr, which
//    consumers compare by identity (timestep.cpp:59,140; adjoint.cpp:73);
//  - symmetric = true; F all-zero without a source; no M for ProblemKind::Mass
//    (physics.cpp:25-31 returns before the with_mass branch); AllenCahnReaction
//    assembles like PoissonDiffusion (physics.cpp:33-34);
//  - the caller's RoutingMatrices are used as given (uploaded once per routing
//    and cached by its pattern pointer), never rebuilt;
//  - bit-identical values (TGK_MODE_EXACT, the default); TG_GPU_ASSEMBLE_MODE=fast
//    selects TGK_MODE_FAST (within 1e-12 scaled tolerance, deterministic).
// Coefficient fields are converted through the public interface only:
// constant -> TGK_FIELD_CONSTANT; any other field is evaluated by the caller's
// own CoefficientField::evaluate (coefficient.cpp:34-55, Analytic included, with
// the quadrature-point images computed on the GPU by tgk_geometry_d) and passed
// as TGK_FIELD_ELEMENT when every element's row is constant (per-element
// fields: the fused kernels), else as the E x Q table TGK_FIELD_QUAD.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "tg/batch.hpp"
#include "tg/errors.hpp"
#include "tg/physics.hpp"
#include "tg/reference.hpp"
#include "tgk.h"

namespace tg {

// The reference implementation under another name, when the integrator kept
// it (oracle/Makefile renames physics.cpp's symbol); used for QUAD4 only.
__attribute__((weak)) AssembledSystem assemble_cpu(const ProblemSpec&, const Mesh&, const DofMap&,
                                                   const RoutingMatrices&, bool);

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = tgk_last_error();
    if (rc == TGK_ERR_INPUT) throw InputError(msg);
    if (rc == TGK_ERR_NUMERICAL) throw NumericalError(msg);
    throw std::runtime_error("libtgk: " + msg);
}

void check(int rc) {
    if (rc != TGK_OK) raise(rc);
}

// Device mesh + routing for one (routing pattern, mesh arrays) pair.  The
// routing is uploaded once; coordinates and connectivity are re-uploaded on
// every call (the caller may have moved nodes in place between calls).
struct DeviceState {
    const CsrPattern* pattern = nullptr;
    const std::int64_t* elements = nullptr;
    std::int64_t E = 0, N = 0;
    int comps = 0;
    tgk_mesh* mesh = nullptr;
    tgk_routing* routing = nullptr;
    double* d_qpts = nullptr;  // quadrature-point images (non-constant fields)
    int qpts_degree = -1;
    ~DeviceState() {
        if (routing) tgk_routing_destroy(routing);
        if (mesh) tgk_mesh_destroy(mesh);
        if (d_qpts) tgk_free_d(d_qpts);
    }
};

std::mutex g_mu;
std::vector<std::unique_ptr<DeviceState>> g_cache;  // most recent last; a few entries

DeviceState& device_state(const Mesh& mesh, const RoutingMatrices& routing, int comps) {
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        DeviceState& s = **it;
        if (s.pattern == routing.pattern.get() && s.elements == mesh.elements.data() &&
            s.E == mesh.element_count() && s.N == mesh.node_count() && s.comps == comps) {
            check(tgk_mesh_upload(s.mesh, mesh.nodes.data(), mesh.elements.data(), nullptr));
            return s;
        }
    }
    auto s = std::make_unique<DeviceState>();
    s->pattern = routing.pattern.get();
    s->elements = mesh.elements.data();
    s->E = mesh.element_count();
    s->N = mesh.node_count();
    s->comps = comps;
    const int kind = static_cast<int>(mesh.kind);  // tg::ElementKind codes == TGK_TRI3 / TGK_QUAD4 / TGK_TET4
    check(tgk_mesh_create(kind, mesh.nodes.data(), s->N, mesh.elements.data(), s->E, &s->mesh));
    const CsrPattern& p = *routing.pattern;
    check(tgk_routing_create_host(s->mesh, comps, routing.N, routing.E, routing.k, p.nnz(), p.offsets.data(),
                                  p.cols.data(), routing.vec_offsets.data(), routing.vec_slots.data(),
                                  routing.mat_offsets.data(), routing.mat_slots.data(), nullptr, &s->routing));
    if (g_cache.size() >= 4) g_cache.erase(g_cache.begin());
    g_cache.push_back(std::move(s));
    return *g_cache.back();
}

// A CoefficientField as a tgk_field; `keep` owns the host arrays.
tgk_field to_field(const CoefficientField& f, const Mesh& mesh, int degree, DeviceState& ds,
                   std::vector<std::vector<double>>& keep) {
    if (f.is_constant()) return tgk_field{TGK_FIELD_CONSTANT, f.constant_value(), nullptr, 0};
    const ReferenceTables tables = reference_tables(mesh.kind, degree);
    GeometryBatch geom;
    geom.E = mesh.element_count();
    geom.Q = static_cast<int>(tables.B.size() / element_nodes(mesh.kind));
    geom.k_geom = element_nodes(mesh.kind);
    geom.d = mesh.dim;
    // quadrature-point images (batch.cpp:76-128), bit-identical to batch_geometry's
    const std::size_t nq = static_cast<std::size_t>(geom.E) * geom.Q;
    if (ds.qpts_degree != degree) {
        if (!ds.d_qpts) check(tgk_alloc_d(reinterpret_cast<void**>(&ds.d_qpts), sizeof(double) * 3 * nq + 8));
        check(tgk_geometry_d(ds.mesh, degree, nullptr, nullptr, nullptr, ds.d_qpts, nullptr, nullptr));
        ds.qpts_degree = degree;
    }
    geom.phys_qpoints.resize(nq * geom.d);
    check(tgk_copy_d2h(geom.phys_qpoints.data(), ds.d_qpts, sizeof(double) * nq * geom.d));
    std::vector<double> tab = f.evaluate(mesh, tables, geom);
    bool per_element = true;
    for (std::size_t e = 0; e < static_cast<std::size_t>(geom.E) && per_element; ++e)
        for (int q = 1; q < geom.Q; ++q)
            if (std::memcmp(&tab[e * geom.Q + q], &tab[e * geom.Q], sizeof(double)) != 0) {
                per_element = false;
                break;
            }
    if (per_element) {
        std::vector<double> v(static_cast<std::size_t>(geom.E));
        for (std::size_t e = 0; e < v.size(); ++e) v[e] = tab[e * geom.Q];
        keep.push_back(std::move(v));
        return tgk_field{TGK_FIELD_ELEMENT, 0.0, keep.back().data(), geom.E};
    }
    keep.push_back(std::move(tab));
    return tgk_field{TGK_FIELD_QUAD, 0.0, keep.back().data(), static_cast<std::int64_t>(nq)};
}

}  // namespace

AssembledSystem assemble(const ProblemSpec& problem, const Mesh& mesh, const DofMap& dofmap,
                         const RoutingMatrices& routing, bool with_mass) {
    const int d = mesh.dim;
    const int comps = problem.components(d);
    if (dofmap.components != comps)
        throw InputError("assemble: dofmap component count does not match problem kind");
    if (mesh.kind == ElementKind::QUAD4) {
        if (&assemble_cpu != nullptr) return assemble_cpu(problem, mesh, dofmap, routing, with_mass);
        throw InputError("GPU assemble: P1 TRI3 / TET4 meshes only (QUAD4 needs the reference's CPU path)");
    }
    if (!routing.pattern) throw InputError("assemble: routing has no pattern");
    if (tgk_device_count() <= 0) throw std::runtime_error("GPU assemble: no usable CUDA device (no CPU fallback)");
    std::lock_guard<std::mutex> lock(g_mu);
    DeviceState& ds = device_state(mesh, routing, comps);
    const bool needs_high_degree =
        !problem.diffusion.is_constant() || problem.kind == ProblemKind::Mass || with_mass;
    const int degree = needs_high_degree ? default_mass_degree(mesh.kind) : default_stiffness_degree(mesh.kind);
    std::vector<std::vector<double>> keep;
    tgk_problem p{};
    p.kind = problem.kind == ProblemKind::LinearElasticity ? TGK_ELASTICITY
             : problem.kind == ProblemKind::Mass           ? TGK_MASS
                                                           : TGK_POISSON;  // AllenCahnReaction: physics.cpp:33-34
    p.diffusion = to_field(problem.diffusion, mesh, degree, ds, keep);
    p.lambda = tgk_field{TGK_FIELD_CONSTANT, 1.0, nullptr, 0};
    p.mu = tgk_field{TGK_FIELD_CONSTANT, 1.0, nullptr, 0};
    if (p.kind == TGK_ELASTICITY) {
        p.lambda = to_field(problem.lambda, mesh, degree, ds, keep);
        p.mu = to_field(problem.mu, mesh, degree, ds, keep);
        p.plane_stress = problem.plane_stress ? 1 : 0;
        if (!problem.source.empty() && static_cast<int>(problem.source.size()) != d)
            throw InputError("elasticity body force needs one component per dimension");
        p.n_source = problem.source.empty() ? 0 : d;
    } else if (p.kind == TGK_POISSON) {
        p.n_source = problem.source.empty() ? 0 : 1;  // physics.cpp:39: source.front()
    }
    for (int s = 0; s < p.n_source; ++s) p.source[s] = to_field(problem.source[s], mesh, degree, ds, keep);
    const bool mass_out = with_mass && p.kind != TGK_MASS;
    if (with_mass && comps != 1) throw InputError("mass matrix assembly only supported for scalar fields");
    p.with_mass = mass_out ? 1 : 0;
    const char* mode = std::getenv("TG_GPU_ASSEMBLE_MODE");
    p.mode = mode && std::string(mode) == "fast" ? TGK_MODE_FAST : TGK_MODE_EXACT;

    AssembledSystem out;
    out.K.pattern = routing.pattern;
    out.K.values.resize(static_cast<std::size_t>(routing.pattern->nnz()));
    out.K.symmetric = true;
    out.F.assign(static_cast<std::size_t>(routing.N), 0.0);
    std::vector<double> Mv;
    if (mass_out) Mv.resize(out.K.values.size());
    check(tgk_assemble(&p, ds.mesh, ds.routing, out.K.values.data(), out.F.data(), mass_out ? Mv.data() : nullptr));
    if (mass_out) {
        SparseOperator M;
        M.pattern = routing.pattern;
        M.values = std::move(Mv);
        M.symmetric = true;
        out.M = std::move(M);
    }
    return out;
}

}  // namespace tg
