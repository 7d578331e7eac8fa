// Fused P1 Map+Reduce assembly (tg::assemble, physics.cpp:10-75) for scalar
// problems: stiffness (or coefficient mass), optional unit mass M and load F,
// straight from mesh + coefficients to CSR values, with no local tensor ever
// written to HBM and no atomics.
//
// Decomposition ("row blocks", see tgk_internal.hpp / plan.cpp): CUDA block b
// owns <= 256 CSR rows (mesh nodes, compact in space via a Morton ordering)
// and walks every element incident to them — its halo — in ascending element
// id, 256 elements per chunk:
//   phase A  one thread per halo element: gather coordinates, exact geometry
//            and local K_e/M_e/F_e into shared memory;
//   phase B  one thread per owned row: fold that row's records of this chunk
//            (ascending element) into shared-memory accumulators.
// Each CSR value is therefore the left fold, from +0.0, of its contributions
// in ascending element order — the reference reduction's order
// (routing.cpp:117-124) — so with the exact element arithmetic of
// element.cuh the output is bit-identical to the CPU reference.
// Elements on a block boundary are recomputed by every block they touch
// (halo recompute); the plan records the factor.
#include <cub/block/block_scan.cuh>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);

namespace {

struct FieldDev {
    int type;
    double value;
    const double* data;
};

struct FusedArgs {
    const double* nodes;
    const int32_t* conn;
    const int64_t* row_ptr;
    const int64_t* row_off;
    const uint32_t* rows;
    const int64_t* halo_off;
    const uint32_t* halo;
    const int64_t* chunk_off;
    const int64_t* chunk_rec_off;
    const uint8_t* chunk_cnt;
    const uint32_t* recs;
    FieldDev coef;
    FieldDev src;
    double* K;
    double* M;
    double* F;
    int lmax;
    unsigned long long* bad;
};

// KTYPE 0: diffusion stiffness, 1: coefficient mass (ProblemKind::Mass)
template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F>
struct FusedCfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    static constexpr int nK = KTYPE == 0 ? k * (k + 1) / 2 : k * k;
    static constexpr int offM = nK;
    static constexpr int nM = HAS_M ? k * k : 0;
    static constexpr int offF = nK + nM;
    static constexpr int nF = HAS_F ? k : 0;
    static constexpr int raw = nK + nM + nF;
    static constexpr int stride = raw % 2 == 0 ? raw + 1 : raw;  // odd: spreads smem banks
    static constexpr int nmat = 1 + (HAS_M ? 1 : 0);
    static size_t smem_bytes(int lmax) {
        return sizeof(double) * (size_t(kChunk) * stride + size_t(kRowsPerBlock) * lmax * nmat +
                                 (HAS_F ? kRowsPerBlock : 0));
    }
};

__device__ __forceinline__ double field_at_elem(const FieldDev& f, int64_t e) {
    return f.type == TGK_FIELD_ELEMENT ? __ldg(f.data + e) : f.value;
}

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F>
__global__ void __launch_bounds__(256) k_fused_scalar(FusedArgs p) {
    using C = FusedCfg<KIND, DEG, KTYPE, HAS_M, HAS_F>;
    using R = Rule<KIND, DEG>;
    constexpr int k = C::k, d = C::d, Q = C::Q;
    extern __shared__ double smem[];
    double* ke = smem;                                         // kChunk x stride
    double* accK = ke + kChunk * C::stride;                    // lmax x kRowsPerBlock
    double* accM = accK + kRowsPerBlock * p.lmax;              // (HAS_M)
    double* accF = accK + kRowsPerBlock * p.lmax * C::nmat;    // (HAS_F)
    using Scan = cub::BlockScan<int, 256>;
    __shared__ typename Scan::TempStorage scan_tmp;

    const int tid = threadIdx.x;
    const int64_t blk = blockIdx.x;
    const int64_t r0 = p.row_off[blk];
    const int nr = static_cast<int>(p.row_off[blk + 1] - r0);
    const int64_t h0 = p.halo_off[blk];
    const int64_t nh = p.halo_off[blk + 1] - h0;
    const int64_t c0 = p.chunk_off[blk];
    const int nch = static_cast<int>(p.chunk_off[blk + 1] - c0);

    for (int i = tid; i < kRowsPerBlock * p.lmax * C::nmat; i += 256) accK[i] = 0.0;
    if (HAS_F) accF[tid] = 0.0;

    for (int c = 0; c < nch; ++c) {
        // ---------------- phase A: one halo element per thread
        const int64_t h = int64_t(c) * kChunk + tid;
        if (h < nh) {
            const int64_t e = p.halo[h0 + h];
            double X[k][d];
            int32_t nid[k];
#pragma unroll
            for (int a = 0; a < k; ++a) nid[a] = __ldg(p.conn + e * k + a);
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int cc = 0; cc < d; ++cc) X[a][cc] = __ldg(p.nodes + int64_t(nid[a]) * d + cc);
            double det;
            double G[k][d];
            double* out = ke + tid * C::stride;
            if (!simplex_geometry<KIND>(X, det, G)) {
                atomicMin(p.bad, static_cast<unsigned long long>(e));
                for (int i = 0; i < C::raw; ++i) out[i] = 0.0;
            } else {
                // coefficient at the quadrature points: scale_q = w_q * det * c_q
                double sc[Q];
                if (p.coef.type == TGK_FIELD_NODAL) {
                    double u[k];
#pragma unroll
                    for (int a = 0; a < k; ++a) u[a] = __ldg(p.coef.data + nid[a]);
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        double v = basis<KIND, DEG>(q, 0) * u[0];
#pragma unroll
                        for (int a = 1; a < k; ++a) v += basis<KIND, DEG>(q, a) * u[a];
                        sc[q] = R::w(q) * det * v;
                    }
                } else {
                    const double cv = field_at_elem(p.coef, e);
#pragma unroll
                    for (int q = 0; q < Q; ++q) sc[q] = R::w(q) * det * cv;
                }
                if constexpr (KTYPE == 0) {
                    // local_stiffness_diffusion (batch.cpp:168-177)
#pragma unroll
                    for (int a = 0; a < k; ++a)
#pragma unroll
                        for (int b = a; b < k; ++b) {
                            const double dot = gdot<KIND>(G, a, b);
                            double v = sc[0] * dot;
#pragma unroll
                            for (int q = 1; q < Q; ++q) v += sc[q] * dot;
                            out[sym_idx<k>(a, b)] = v;
                        }
                } else {
                    // local_mass with the coefficient (batch.cpp:259-265)
#pragma unroll
                    for (int a = 0; a < k; ++a)
#pragma unroll
                        for (int b = 0; b < k; ++b) {
                            double v = sc[0] * basis<KIND, DEG>(0, a) * basis<KIND, DEG>(0, b);
#pragma unroll
                            for (int q = 1; q < Q; ++q)
                                v += sc[q] * basis<KIND, DEG>(q, a) * basis<KIND, DEG>(q, b);
                            out[a * k + b] = v;
                        }
                }
                if constexpr (HAS_M) {
                    // with_mass: local_mass with ones (physics.cpp:70-71); w*det*1.0 == w*det
#pragma unroll
                    for (int a = 0; a < k; ++a)
#pragma unroll
                        for (int b = 0; b < k; ++b) {
                            double v = R::w(0) * det * basis<KIND, DEG>(0, a) * basis<KIND, DEG>(0, b);
#pragma unroll
                            for (int q = 1; q < Q; ++q)
                                v += R::w(q) * det * basis<KIND, DEG>(q, a) * basis<KIND, DEG>(q, b);
                            out[C::offM + a * k + b] = v;
                        }
                }
                if constexpr (HAS_F) {
                    // local_load (batch.cpp:280-286)
                    double sf[Q];
                    if (p.src.type == TGK_FIELD_NODAL) {
                        double u[k];
#pragma unroll
                        for (int a = 0; a < k; ++a) u[a] = __ldg(p.src.data + nid[a]);
#pragma unroll
                        for (int q = 0; q < Q; ++q) {
                            double v = basis<KIND, DEG>(q, 0) * u[0];
#pragma unroll
                            for (int a = 1; a < k; ++a) v += basis<KIND, DEG>(q, a) * u[a];
                            sf[q] = R::w(q) * det * v;
                        }
                    } else {
                        const double fv = field_at_elem(p.src, e);
#pragma unroll
                        for (int q = 0; q < Q; ++q) sf[q] = R::w(q) * det * fv;
                    }
#pragma unroll
                    for (int a = 0; a < k; ++a) {
                        double v = sf[0] * basis<KIND, DEG>(0, a);
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += sf[q] * basis<KIND, DEG>(q, a);
                        out[C::offF + a] = v;
                    }
                }
            }
        }
        // record offsets of this chunk: exclusive scan of the per-row counts
        const int64_t cg = c0 + c;
        const int cnt = tid < nr ? p.chunk_cnt[cg * kRowsPerBlock + tid] : 0;
        int off;
        Scan(scan_tmp).ExclusiveSum(cnt, off);
        __syncthreads();
        // ---------------- phase B: one owned row per thread, ascending element
        if (cnt > 0) {
            const uint32_t* rr = p.recs + p.chunk_rec_off[cg] + off;
            for (int j = 0; j < cnt; ++j) {
                const uint32_t rec = __ldg(rr + j);
                const int hl = rec & 0xff;
                const int a = (rec >> 8) & 3;
                const double* src = ke + hl * C::stride;
#pragma unroll
                for (int b = 0; b < k; ++b) {
                    const int pos = (rec >> (10 + 5 * b)) & 31;
                    const int ix = KTYPE == 0 ? sym_idx<k>(a, b) : a * k + b;
                    accK[pos * kRowsPerBlock + tid] += src[ix];
                    if constexpr (HAS_M) accM[pos * kRowsPerBlock + tid] += src[C::offM + a * k + b];
                }
                if constexpr (HAS_F) accF[tid] += src[C::offF + a];
            }
        }
        __syncthreads();
    }
    // ---------------- epilogue: owned rows -> CSR values / F
    if (tid < nr) {
        const int64_t row = p.rows[r0 + tid];
        const int64_t rp = p.row_ptr[row];
        const int len = static_cast<int>(p.row_ptr[row + 1] - rp);
        for (int q = 0; q < len; ++q) p.K[rp + q] = accK[q * kRowsPerBlock + tid];
        if constexpr (HAS_M)
            for (int q = 0; q < len; ++q) p.M[rp + q] = accM[q * kRowsPerBlock + tid];
        if constexpr (HAS_F) p.F[row] = accF[tid];
    }
}

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F>
int launch_fused(const FusedArgs& a, int64_t n_blocks, cudaStream_t st) {
    using C = FusedCfg<KIND, DEG, KTYPE, HAS_M, HAS_F>;
    auto kern = k_fused_scalar<KIND, DEG, KTYPE, HAS_M, HAS_F>;
    const size_t smem = C::smem_bytes(a.lmax);
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<static_cast<unsigned>(n_blocks), 256, smem, st>>>(a);
    KERNEL_CHECK("fused_scalar");
    return TGK_OK;
}

template <int KIND, int DEG>
int dispatch_flags(int ktype, bool m, bool f, const FusedArgs& a, int64_t nb, cudaStream_t st) {
    if (ktype == 1) return launch_fused<KIND, DEG, 1, false, false>(a, nb, st);
    if (m && f) return launch_fused<KIND, DEG, 0, true, true>(a, nb, st);
    if (m) return launch_fused<KIND, DEG, 0, true, false>(a, nb, st);
    if (f) return launch_fused<KIND, DEG, 0, false, true>(a, nb, st);
    return launch_fused<KIND, DEG, 0, false, false>(a, nb, st);
}

}  // namespace

int ensure_plan(tgk_routing* r);

// Scalar fused assembly on device buffers.  Returns after the bad-element check.
int fused_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K,
                          double* F, double* M, cudaStream_t st, unsigned long long* d_bad) {
    TGK_TRY(ensure_plan(r));
    const PlanDev& pl = r->plan;
    const bool is_mass = pr->kind == TGK_MASS;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT || is_mass || pr->with_mass;
    const int degree = high ? 2 : 1;  // default_mass_degree / default_stiffness_degree for P1
    const bool has_f = !is_mass && pr->n_source > 0;
    const bool has_m = pr->with_mass != 0;
    FusedArgs a{};
    a.nodes = m->nodes;
    a.conn = m->conn;
    a.row_ptr = r->row_ptr;
    a.row_off = pl.row_off;
    a.rows = pl.rows;
    a.halo_off = pl.halo_off;
    a.halo = pl.halo;
    a.chunk_off = pl.chunk_off;
    a.chunk_rec_off = pl.chunk_rec_off;
    a.chunk_cnt = pl.chunk_cnt;
    a.recs = pl.recs;
    a.coef = FieldDev{pr->diffusion.type, pr->diffusion.value, pr->diffusion.data};
    if (has_f) a.src = FieldDev{pr->source[0].type, pr->source[0].value, pr->source[0].data};
    a.K = K;
    a.M = M;
    a.F = F;
    a.lmax = pl.lmax;
    DevBuf<unsigned long long> bad;
    if (!d_bad) TGK_TRY(bad.alloc(1));
    a.bad = d_bad ? d_bad : bad.p;
    CUDA_TRY(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), st));
    if (!has_f && F) CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
    const int ktype = is_mass ? 1 : 0;
    if (m->kind == TGK_TET4) {
        if (degree == 1) TGK_TRY((dispatch_flags<TGK_TET4, 1>(ktype, has_m, has_f, a, pl.n_blocks, st)));
        else TGK_TRY((dispatch_flags<TGK_TET4, 2>(ktype, has_m, has_f, a, pl.n_blocks, st)));
    } else {
        if (degree == 1) TGK_TRY((dispatch_flags<TGK_TRI3, 1>(ktype, has_m, has_f, a, pl.n_blocks, st)));
        else TGK_TRY((dispatch_flags<TGK_TRI3, 2>(ktype, has_m, has_f, a, pl.n_blocks, st)));
    }
    if (!d_bad) return check_bad(bad.p, st);
    return TGK_OK;  // asynchronous: the caller inspects *d_bad
}

}  // namespace tgk
