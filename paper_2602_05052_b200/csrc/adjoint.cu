// Adjoint pieces (adjoint.cpp:68-82 and the per-element chain rule of
// acceptance.cpp:357-378 / tg_main.cpp:840-856), batched operator-learning
// assembly, and the vector (elasticity) assembly path.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);
int fused_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K,
                          double* F, double* M, cudaStream_t st, unsigned long long* d_bad);
int batched_entries(const tgk_mesh* m, tgk_routing* r, int64_t B, const double* rho, double source, double* K,
                    double* F, cudaStream_t st, unsigned long long* d_bad);
int batched_fused(const tgk_mesh* m, tgk_routing* r, int64_t B, const double* rho, double source, double* K,
                  double* F, cudaStream_t st, unsigned long long* d_bad);
int local_elasticity_nocheck(const tgk_mesh* m, int degree, const double* lam, const double* mu, double* out,
                             cudaStream_t st);
int routing_scratch(tgk_routing* r, int slot, size_t n, double** out);

namespace {

// gradient_products: dK[b,t] = lambda_b[i] * U_b[cols[t]] for t in row i; dF = -lambda
__global__ void k_gradient_products(const int64_t* row_ptr, const int64_t* cols, int64_t N,
                                    int64_t nnz, int64_t B, const double* lam, const double* U,
                                    double* dK, double* dF) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nnz) {
        int64_t lo = 0, hi = N;  // row of t: last i with row_ptr[i] <= t
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (row_ptr[mid] <= t) lo = mid; else hi = mid;
        }
        const int64_t j = cols[t];
        for (int64_t b = 0; b < B; ++b) dK[b * nnz + t] = lam[b * N + lo] * U[b * N + j];
    }
    if (dF && t < N)
        for (int64_t b = 0; b < B; ++b) dF[b * N + t] = -lam[b * N + t];
}

// Fused transpose gather: out[b,e] = sum_{a,c} (lambda_b[g_a] * K0_e[a,c]) * U_b[g_c]
// (tg_main.cpp:846-850 order), K0_e = local_stiffness_diffusion with unit
// coefficient at quadrature degree DEG, recomputed in registers.
template <int KIND, int DEG, int FPB>
__global__ void __launch_bounds__(128) k_adjoint_gather(const double* nodes, const int32_t* conn,
                                                        int64_t E, int64_t N, int64_t B,
                                                        const double* lam, const double* U,
                                                        double* out, unsigned long long* bad) {
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    using R = Rule<KIND, DEG>;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t g[k];
    double X[k][d];
#pragma unroll
    for (int a = 0; a < k; ++a) g[a] = __ldg(conn + e * k + a);
#pragma unroll
    for (int a = 0; a < k; ++a)
#pragma unroll
        for (int c = 0; c < d; ++c) X[a][c] = __ldg(nodes + int64_t(g[a]) * d + c);
    double det, G[k][d];
    if (!simplex_geometry<KIND>(X, det, G)) {
        atomicMin(bad, static_cast<unsigned long long>(e));
        return;
    }
    double K0[k][k];
#pragma unroll
    for (int a = 0; a < k; ++a)
#pragma unroll
        for (int c = a; c < k; ++c) {
            const double dot = gdot<KIND>(G, a, c);
            double v = (R::w(0) * det * 1.0) * dot;
#pragma unroll
            for (int q = 1; q < Q; ++q) v += (R::w(q) * det * 1.0) * dot;
            K0[a][c] = v;
            K0[c][a] = v;
        }
    const int64_t b0 = int64_t(blockIdx.y) * FPB;
#pragma unroll 1
    for (int f = 0; f < FPB; ++f) {
        const int64_t b = b0 + f;
        if (b >= B) break;
        const double* lb = lam + b * N;
        const double* ub = U + b * N;
        double la[k], uc[k];
#pragma unroll
        for (int a = 0; a < k; ++a) {
            la[a] = __ldg(lb + g[a]);
            uc[a] = __ldg(ub + g[a]);
        }
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int c = 0; c < k; ++c) s += la[a] * K0[a][c] * uc[c];
        out[b * E + e] = s;
    }
}

// Grouped transpose gather (plan_entries.cpp build_group_plan): a block
// takes one group of G spatially compact elements (one per thread) and FPB
// fields.  K0_e stays in registers across the fields; per field the group's
// lambda_b / U_b node values are gathered once into shared memory (double
// buffered, the next field's loads in flight while this one is summed), so
// each node value is read from L2 once per group instead of once per
// incident element.  Same per-element expression as k_adjoint_gather.
constexpr int kGroupThreads = 256;

struct GroupArgs {
    const double* nodes;
    const int32_t* conn;
    int64_t E, N, B, fpb;
    const double* lam;
    const double* U;
    double* out;
    GroupPlanDev pl;
    unsigned long long* bad;
};

template <int KIND, int DEG, int NPT>
__global__ void __launch_bounds__(kGroupThreads) k_adjoint_groups(GroupArgs p) {
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q, T = kGroupThreads;
    using R = Rule<KIND, DEG>;
    extern __shared__ __align__(16) double2 sv[];  // [2 buffers][max_nodes] of (lambda, U)
    const int MN = p.pl.max_nodes;
    const int tid = threadIdx.x;
    const int64_t g = blockIdx.x;
    const int64_t q0 = p.pl.grp_off[g];
    const int ne = static_cast<int>(p.pl.grp_off[g + 1] - q0);
    const int64_t n0 = p.pl.node_off[g];
    const int nn = static_cast<int>(p.pl.node_off[g + 1] - n0);
    const bool has_e = tid < ne;
    const uint32_t e = has_e ? __ldg(p.pl.elems + q0 + tid) : 0u;
    const uint64_t lc = has_e ? __ldg(reinterpret_cast<const unsigned long long*>(p.pl.lconn) + q0 + tid) : 0ull;
    uint32_t gid[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) gid[j] = tid + j * T < nn ? __ldg(p.pl.gnodes + n0 + tid + j * T) : 0u;
    const int64_t b0 = int64_t(blockIdx.y) * p.fpb;
    const int64_t b1 = b0 + p.fpb < p.B ? b0 + p.fpb : p.B;
    double rl[NPT], ru[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        rl[j] = tid + j * T < nn ? __ldg(p.lam + b0 * p.N + gid[j]) : 0.0;
        ru[j] = tid + j * T < nn ? __ldg(p.U + b0 * p.N + gid[j]) : 0.0;
    }
    double K0[k][k];
    bool ok = false;
    if (has_e) {
        double X[k][d];
#pragma unroll
        for (int a = 0; a < k; ++a) {
            const int64_t gn = __ldg(p.conn + int64_t(e) * k + a);
#pragma unroll
            for (int c = 0; c < d; ++c) X[a][c] = __ldg(p.nodes + gn * d + c);
        }
        double det, G[k][d];
        ok = simplex_geometry<KIND>(X, det, G);
        if (!ok) atomicMin(p.bad, static_cast<unsigned long long>(e));
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int c = a; c < k; ++c) {
                const double dot = ok ? gdot<KIND>(G, a, c) : 0.0;
                double v = (R::w(0) * det * 1.0) * dot;
#pragma unroll
                for (int q = 1; q < Q; ++q) v += (R::w(q) * det * 1.0) * dot;
                K0[a][c] = v;
                K0[c][a] = v;
            }
    }
    int li[k];
#pragma unroll
    for (int a = 0; a < k; ++a) li[a] = static_cast<int>((lc >> (16 * a)) & 0xffff);
    int buf = 0;
    for (int64_t b = b0; b < b1; ++b, buf ^= 1) {
        double2* slu = sv + size_t(buf) * MN;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
            if (tid + j * T < nn) slu[tid + j * T] = make_double2(rl[j], ru[j]);
        if (b + 1 < b1) {
#pragma unroll
            for (int j = 0; j < NPT; ++j)
                if (tid + j * T < nn) {
                    rl[j] = __ldg(p.lam + (b + 1) * p.N + gid[j]);
                    ru[j] = __ldg(p.U + (b + 1) * p.N + gid[j]);
                }
        }
        __syncthreads();
        if (ok) {
            double la[k], uc[k];
#pragma unroll
            for (int a = 0; a < k; ++a) {  // one 16-byte load per node
                const double2 lu = slu[li[a]];
                la[a] = lu.x;
                uc[a] = lu.y;
            }
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int c = 0; c < k; ++c) s += la[a] * K0[a][c] * uc[c];
            p.out[b * p.E + e] = s;
        }
    }
}

template <int KIND, int DEG>
int launch_adjoint_groups(const GroupArgs& a, int npt, cudaStream_t st) {
    const size_t smem = sizeof(double) * 4 * size_t(a.pl.max_nodes);
    const dim3 grid(static_cast<unsigned>(a.pl.n_groups), static_cast<unsigned>((a.B + a.fpb - 1) / a.fpb));
    auto go = [&](auto kern) -> int {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (a.pl.n_groups > 0) kern<<<grid, kGroupThreads, smem, st>>>(a);
        KERNEL_CHECK("adjoint_groups");
        return TGK_OK;
    };
    if (npt == 1) return go(k_adjoint_groups<KIND, DEG, 1>);
    if (npt == 2) return go(k_adjoint_groups<KIND, DEG, 2>);
    return go(k_adjoint_groups<KIND, DEG, 4>);
}

// plane-stress lambda (batch.cpp:359-361) in place, and the mu > 0 check
__global__ void k_plane_stress(double* lam, const double* mu, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) lam[i] = 2.0 * lam[i] * mu[i] / (lam[i] + 2.0 * mu[i]);
}

__global__ void k_min_value(const double* v, int64_t n, unsigned long long* flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && v[i] <= 0.0) atomicMin(flag, 0ull);
}

__global__ void k_interleave(const double* comp, int64_t n, int d, int c, double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i * d + c] = comp[i];
}

}  // namespace

// Elasticity (physics.cpp:45-66) through the materialised stage kernels:
// evaluate -> local_stiffness_elasticity -> reduce_matrix, and the vector
// load -> reduce_vector.  Bit-identical to the reference.
int elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K,
                        double* F, cudaStream_t st) {
    const int d = m->d;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT;
    const int degree = high ? 2 : 1;
    int Q = 0;
    TGK_TRY(tgk_tables(m->kind, degree, &Q, nullptr, nullptr, nullptr, nullptr));
    const int64_t nq = m->E * Q;
    const int kk = m->k * d;
    double *lam, *mu, *local, *src, *comp;  // cached on the routing: no per-call cudaMalloc of E*kk*kk doubles
    TGK_TRY(routing_scratch(r, 0, nq, &lam));
    TGK_TRY(routing_scratch(r, 1, nq, &mu));
    TGK_TRY(routing_scratch(r, 2, size_t(m->E) * kk * kk, &local));
    TGK_TRY(tgk_evaluate_field_d(m, degree, &pr->lambda, lam, st));
    TGK_TRY(tgk_evaluate_field_d(m, degree, &pr->mu, mu, st));
    if (d == 2 && pr->plane_stress) {
        k_plane_stress<<<grid_for(nq, 256), 256, 0, st>>>(lam, mu, nq);
        KERNEL_CHECK("plane_stress");
    }
    {
        DevBuf<unsigned long long> flag;
        TGK_TRY(flag.alloc(1));
        CUDA_TRY(cudaMemsetAsync(flag.p, 0xff, sizeof(unsigned long long), st));
        k_min_value<<<grid_for(nq, 256), 256, 0, st>>>(mu, nq, flag.p);
        KERNEL_CHECK("mu_check");
        unsigned long long h = ULLONG_MAX;
        CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (h != ULLONG_MAX) return set_error(TGK_ERR_INPUT, "elasticity requires mu > 0");
    }
    TGK_TRY(local_elasticity_nocheck(m, degree, lam, mu, local, st));
    TGK_TRY(tgk_reduce_matrix_d(r, local, K, st));
    if (F) {
        if (pr->n_source > 0) {
            TGK_TRY(routing_scratch(r, 3, size_t(nq) * d, &src));
            TGK_TRY(routing_scratch(r, 4, nq, &comp));
            for (int c = 0; c < d; ++c) {
                TGK_TRY(tgk_evaluate_field_d(m, degree, &pr->source[c], comp, st));
                k_interleave<<<grid_for(nq, 256), 256, 0, st>>>(comp, nq, d, c, src);
                KERNEL_CHECK("interleave");
            }
            TGK_TRY(tgk_local_load_vector_d(m, degree, src, local, st));
            TGK_TRY(tgk_reduce_vector_d(r, local, F, st));
        } else {
            CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
        }
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return TGK_OK;
}

int ensure_scalar_segments(tgk_routing* r, cudaStream_t st);

// Scalar assembly (physics.cpp:10-75) through the materialised Stage I + II
// drop-ins: evaluate -> local_stiffness_diffusion / local_mass -> reduce_matrix,
// local_load -> reduce_vector.  Bit-identical to the reference for any mesh
// connectivity: the fallback of the fused kernels when a mesh exceeds their
// plan layouts (rows longer than 32 entries, halos beyond the block tables;
// fused.cu), so nothing the reference assembles is rejected.  Builds the
// routing's segment maps on first use; partitioned routings are not supported
// on this path.
int materialised_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                                 double* M, cudaStream_t st, unsigned long long* d_bad) {
    if (r->own_hi >= 0 || r->elem_hi >= 0)
        return set_error(TGK_ERR_INPUT, "assemble: this mesh exceeds the fused plan layout and the materialised "
                                        "fallback does not support row / element partitions");
    const bool is_mass = pr->kind == TGK_MASS;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT || is_mass || pr->with_mass;
    const int degree = high ? 2 : 1;  // default_mass_degree / default_stiffness_degree (physics.cpp:18-21)
    const bool has_f = !is_mass && pr->n_source > 0;
    TGK_TRY(ensure_scalar_segments(r, st));
    int Q = 0;
    TGK_TRY(tgk_tables(m->kind, degree, &Q, nullptr, nullptr, nullptr, nullptr));
    const int64_t nq = m->E * Q;
    double *coef, *local;
    TGK_TRY(routing_scratch(r, 0, nq, &coef));
    TGK_TRY(routing_scratch(r, 2, size_t(m->E) * m->k * m->k, &local));
    if (d_bad) CUDA_TRY(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), st));
    TGK_TRY(tgk_evaluate_field_d(m, degree, &pr->diffusion, coef, st));
    if (is_mass) TGK_TRY(tgk_local_mass_d(m, degree, coef, local, st));
    else TGK_TRY(tgk_local_stiffness_diffusion_d(m, degree, coef, local, st));
    TGK_TRY(tgk_reduce_matrix_d(r, local, K, st));
    if (pr->with_mass && !is_mass && M) {
        const tgk_field ones{TGK_FIELD_CONSTANT, 1.0, nullptr, 0};
        TGK_TRY(tgk_evaluate_field_d(m, degree, &ones, coef, st));
        TGK_TRY(tgk_local_mass_d(m, degree, coef, local, st));
        TGK_TRY(tgk_reduce_matrix_d(r, local, M, st));
    }
    if (F) {
        if (has_f) {
            TGK_TRY(tgk_evaluate_field_d(m, degree, &pr->source[0], coef, st));
            TGK_TRY(tgk_local_load_d(m, degree, coef, local, st));
            TGK_TRY(tgk_reduce_vector_d(r, local, F, st));
        } else {
            CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
        }
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return TGK_OK;
}

}  // namespace tgk

namespace tgk {
namespace {

// simp_sensitivity (adjoint.cpp:101-125), one thread per element in the
// reference's operation order: u_e gathered through the DoF map, row_a =
// left fold over b of K0_e[a][b] u_e[b], quad = left fold over a of u_e[a]
// row_a, sens = ((-p * rho^(p-1)) * (E_max - E_min)) * quad.  rho^(p-1) as
// rho * rho for the standard penalty p = 3 (correctly rounded like std::pow),
// else pow.  Out-of-range DoF indices are reported, never dereferenced.
template <int K>
__global__ void k_simp_sensitivity(int64_t E, int kr, const int64_t* __restrict__ map, const double* __restrict__ rho,
                                   double p, double E_min, double E_max, const double* __restrict__ K0,
                                   const double* __restrict__ U, int64_t n_dofs, double* __restrict__ sens,
                                   unsigned long long* bad) {
    const int k = K > 0 ? K : kr;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        double ue[K > 0 ? K : 32];
        bool ok = true;
        for (int a = 0; a < k; ++a) {
            const int64_t g = __ldg(map + e * k + a);
            ok = ok && g >= 0 && g < n_dofs;
            ue[a] = (g >= 0 && g < n_dofs) ? __ldg(U + g) : 0.0;
        }
        if (!ok) atomicMin(bad, static_cast<unsigned long long>(e));
        const double* Ke = K0 + e * k * k;
        double quad = 0.0;
        for (int a = 0; a < k; ++a) {
            double row = 0.0;
            for (int b = 0; b < k; ++b) row += __ldg(Ke + a * k + b) * ue[b];
            quad += ue[a] * row;
        }
        const double r = __ldg(rho + e);
        const double pw = p == 3.0 ? r * r : pow(r, p - 1.0);
        sens[e] = -p * pw * (E_max - E_min) * quad;
    }
}

}  // namespace
}  // namespace tgk

extern "C" {

int tgk_gradient_products_d(const tgk_routing* r, int64_t B, const double* lam, const double* U,
                            double* dK, double* dF, void* stream) {
    using namespace tgk;
    if (!r) return set_error(TGK_ERR_INPUT, "gradient_products: null routing");
    TGK_TRY(ensure_device());
    const int64_t n = std::max(r->nnz, r->N);
    k_gradient_products<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
        r->row_ptr, r->col_idx, r->N, r->nnz, B, lam, U, dK, dF);
    KERNEL_CHECK("gradient_products");
    return TGK_OK;
}

int tgk_adjoint_gather_d(const tgk_mesh* m, const tgk_routing* r, int64_t B, const double* lam,
                         const double* U, double* out, int degree, void* stream) {
    using namespace tgk;
    if (!m || !r) return set_error(TGK_ERR_INPUT, "adjoint_gather: null argument");
    if (r->components != 1) return set_error(TGK_ERR_INPUT, "adjoint_gather: scalar routing required");
    TGK_TRY(check_routing_fresh(m, r));
    TGK_TRY(ensure_device());
    cudaStream_t st = as_stream(stream);
    unsigned long long* badp = nullptr;  // the routing's persistent status words
    TGK_TRY(routing_flags(const_cast<tgk_routing*>(r), &badp));
    CUDA_TRY(cudaMemsetAsync(badp, 0xff, sizeof(unsigned long long), st));
    if (m->kind != TGK_TET4 && m->kind != TGK_TRI3) return set_error(TGK_ERR_INPUT, "adjoint_gather: TRI3/TET4 only");
    if (degree != 1 && degree != 2) return set_error(TGK_ERR_INPUT, "adjoint_gather: degree must be 1 or 2");
    if (B <= 0) return TGK_OK;
    if (!getenv("TGK_ADJ_FLAT")) {
        const GroupPlanDev* pl = nullptr;
        TGK_TRY(ensure_group_plan(const_cast<tgk_routing*>(r), kGroupThreads, &pl));
        const int npt = (pl->max_nodes + kGroupThreads - 1) / kGroupThreads;
        if (npt <= 4) {
            GroupArgs a{};
            a.nodes = m->nodes;
            a.conn = m->conn;
            a.E = m->E;
            a.N = m->N;
            a.B = B;
            a.fpb = 16;
            if (const char* e = getenv("TGK_ADJ_FPB")) a.fpb = std::max(1, atoi(e));
            a.lam = lam;
            a.U = U;
            a.out = out;
            a.pl = *pl;
            a.bad = badp;
            const int np = npt <= 1 ? 1 : npt <= 2 ? 2 : 4;
            if (m->kind == TGK_TET4)
                TGK_TRY((degree == 1 ? launch_adjoint_groups<TGK_TET4, 1>(a, np, st)
                                     : launch_adjoint_groups<TGK_TET4, 2>(a, np, st)));
            else
                TGK_TRY((degree == 1 ? launch_adjoint_groups<TGK_TRI3, 1>(a, np, st)
                                     : launch_adjoint_groups<TGK_TRI3, 2>(a, np, st)));
            return check_bad(badp, st);
        }
    }
    constexpr int FPB = 8;
    const dim3 grid(grid_for(m->E, 128), static_cast<unsigned>((B + FPB - 1) / FPB));
    if (m->kind == TGK_TET4) {
        if (degree == 1) k_adjoint_gather<TGK_TET4, 1, FPB><<<grid, 128, 0, st>>>(m->nodes, m->conn, m->E, m->N, B, lam, U, out, badp);
        else k_adjoint_gather<TGK_TET4, 2, FPB><<<grid, 128, 0, st>>>(m->nodes, m->conn, m->E, m->N, B, lam, U, out, badp);
    } else {
        if (degree == 1) k_adjoint_gather<TGK_TRI3, 1, FPB><<<grid, 128, 0, st>>>(m->nodes, m->conn, m->E, m->N, B, lam, U, out, badp);
        else k_adjoint_gather<TGK_TRI3, 2, FPB><<<grid, 128, 0, st>>>(m->nodes, m->conn, m->E, m->N, B, lam, U, out, badp);
    }
    KERNEL_CHECK("adjoint_gather");
    return check_bad(badp, st);
}

// One batched launch (batched.cu: halo geometry cached per block, all fields
// folded through the same plan); one fused launch per field when the block
// working set does not fit shared memory.
int tgk_assemble_batched_d(const tgk_mesh* m, const tgk_routing* r, int64_t B, const double* rho,
                           double source, double* K, double* F, int mode, void* stream) {
    using namespace tgk;
    if (!m || !r) return set_error(TGK_ERR_INPUT, "assemble_batched: null argument");
    if (mode != TGK_MODE_EXACT && mode != TGK_MODE_FAST)
        return set_error(TGK_ERR_INPUT, "assemble_batched: unknown arithmetic mode");
    if (r->components != 1) return set_error(TGK_ERR_INPUT, "assemble_batched: scalar routing required");
    TGK_TRY(check_routing_fresh(m, r));
    if (B < 0) return set_error(TGK_ERR_INPUT, "assemble_batched: negative batch");
    TGK_TRY(ensure_device());
    cudaStream_t st = as_stream(stream);
    unsigned long long* badp = nullptr;  // the routing's persistent status words
    TGK_TRY(routing_flags(const_cast<tgk_routing*>(r), &badp));
    CUDA_TRY(cudaMemsetAsync(badp, 0xff, sizeof(unsigned long long), st));
    if (B == 0) return TGK_OK;
    // TGK_MODE_FAST takes the same kernels: their bit-identical results meet
    // the fast contract, and the fast-mode variants measured slower on C4
    // (profiles/r02_fast_experiments.txt)
    if (!getenv("TGK_BATCHED_LOOP") && !getenv("TGK_BATCHED_CHUNKED")) {
        const int rc = batched_entries(m, const_cast<tgk_routing*>(r), B, rho, source, K, F, st, badp);
        if (rc == TGK_OK) return check_bad(badp, st);
        if (rc != TGK_ERR_INPUT) return rc;
    }
    if (!getenv("TGK_BATCHED_LOOP")) {
        const int rc = batched_fused(m, const_cast<tgk_routing*>(r), B, rho, source, K, F, st, badp);
        if (rc == TGK_OK) return check_bad(badp, st);
        if (rc != TGK_ERR_INPUT) return rc;
    }
    for (int64_t b = 0; b < B; ++b) {
        tgk_problem p{};
        p.kind = TGK_POISSON;
        p.diffusion = tgk_field{TGK_FIELD_ELEMENT, 0.0, rho + b * m->E, m->E};
        p.n_source = (F && b == 0) ? 1 : 0;
        p.source[0] = tgk_field{TGK_FIELD_CONSTANT, source, nullptr, 0};
        TGK_TRY(fused_scalar_assemble(&p, m, const_cast<tgk_routing*>(r), K + b * r->nnz,
                                      b == 0 ? F : nullptr, nullptr, st, badp));
        if (b + 1 == B || (b & 63) == 63) TGK_TRY(check_bad(badp, st));
    }
    return TGK_OK;
}

int tgk_simp_sensitivity_d(int64_t E, int k, const int64_t* d_map, const double* d_rho, double p, double E_min,
                           double E_max, const double* d_unit_stiffness, const double* d_U, int64_t n_dofs,
                           double* d_sens, void* stream) {
    using namespace tgk;
    if (E < 0 || k <= 0 || k > 32 || n_dofs < 0 ||
        (E > 0 && (!d_map || !d_rho || !d_unit_stiffness || !d_U || !d_sens)))
        return set_error(TGK_ERR_INPUT, "simp_sensitivity: shape mismatch");  // adjoint.cpp:107-110
    TGK_TRY(ensure_device());
    if (E == 0) return TGK_OK;
    cudaStream_t st = as_stream(stream);
    DevBuf<unsigned long long> bad;
    TGK_TRY(bad.alloc(1));
    CUDA_TRY(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    const unsigned G = grid_for(E, 128);
    auto go = [&](auto kern) {
        kern<<<G, 128, 0, st>>>(E, k, d_map, d_rho, p, E_min, E_max, d_unit_stiffness, d_U, n_dofs, d_sens, bad.p);
    };
    switch (k) {
        case 3: go(k_simp_sensitivity<3>); break;
        case 4: go(k_simp_sensitivity<4>); break;
        case 6: go(k_simp_sensitivity<6>); break;
        case 8: go(k_simp_sensitivity<8>); break;
        case 12: go(k_simp_sensitivity<12>); break;
        default: go(k_simp_sensitivity<0>); break;
    }
    KERNEL_CHECK("simp_sensitivity");
    unsigned long long h = ULLONG_MAX;
    CUDA_TRY(cudaMemcpyAsync(&h, bad.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (h != ULLONG_MAX)
        return set_error(TGK_ERR_INPUT, "simp_sensitivity: element " + std::to_string(h) + " maps a DoF outside [0," +
                                            std::to_string(n_dofs) + ")");
    return TGK_OK;
}

}  // extern "C"
