// Fused P1 Map+Reduce assembly, v4 ("row blocks with update rounds"), for
// scalar problems (tg::assemble, physics.cpp:10-75): stiffness (or
// coefficient mass), optional unit mass M and load F, straight from mesh +
// coefficients to CSR values.  No local tensor is written to HBM or staged in
// shared memory, and there are no atomics.
//
// CUDA block b owns up to R CSR rows (Morton-compact mesh nodes) and walks
// the elements incident to them (its halo, plan4.cpp) in chunks of T, one
// element per thread:
//   prologue  the block's node table (coordinates of every node its halo
//             touches; owned rows first) arrives by cp.async together with
//             the first chunks' block-local connectivity and update records;
//   compute   each thread evaluates its element's local K_e / M_e / F_e in
//             registers with the reference's exact operation order
//             (element.cuh);
//   update    for every owned node a of the element, the thread adds row a
//             of the local tensors into the block's shared-memory row
//             accumulators.  Two elements of a chunk that touch the same row
//             do so in different plan-computed rounds (separated by
//             __syncthreads), in ascending element order, so every CSR value
//             is the left fold from +0.0 of its contributions in ascending
//             element order — the reference reduction (routing.cpp:117-124).
//   epilogue  the accumulators are written to the CSR values row by row.
// Boundary elements are recomputed by every block they touch (halo recompute).
#include <cstdio>
#include <vector>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);
int mesh_division_safe(tgk_mesh* m, cudaStream_t st, bool* safe);

namespace {

struct Field4 {
    int type;
    double value;
    const double* data;
};

struct Fused4Args {
    const double* nodes;
    const int64_t* row_off;
    const uint32_t* rows;
    const int64_t* rows_rp;
    const int64_t* bnode_off;
    const uint32_t* bnodes;
    const int64_t* halo_off;
    const uint32_t* halo;
    const uint64_t* hconn;
    const int64_t* chunk_off;
    const int64_t* chunk_rec;
    const uint32_t* chunk_meta;
    const uint16_t* chunk_wbase;
    const uint32_t* recs;
    Field4 coef, src;
    double* K;
    double* M;
    double* F;
    int lmax;        // max CSR row length
    int S;           // accumulator stride (odd, >= R)
    int max_recs;    // largest record segment of a chunk (multiple of 4)
    int max_bnodes;  // largest block node table (even)
    int max_chunks;  // largest chunk count of a block
    unsigned long long* bad;
};

#ifndef TGK4_RING
#define TGK4_RING 3
#endif
constexpr int kRing4 = TGK4_RING;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// c(x_q) for a constant / per-element / nodal field (coefficient.cpp:34-55,
// interpolate_nodal batch.cpp:321-330)
template <int KIND, int DEG>
__device__ __forceinline__ double field4_q(int type, double value, const double* u, int q) {
    constexpr int k = P1<KIND>::k;
    if (type == TGK_FIELD_NODAL) {
        double v = basis<KIND, DEG>(q, 0) * u[0];
#pragma unroll
        for (int a = 1; a < k; ++a) v += basis<KIND, DEG>(q, a) * u[a];
        return v;
    }
    return type == TGK_FIELD_ELEMENT ? u[0] : value;
}

template <int KIND, int T>
struct Smem4 {
    static constexpr int d = P1<KIND>::d;
    // byte offsets inside the dynamic shared memory (all 16-byte aligned)
    size_t accK, accM, accF, nt, ntc, nts, hc, rc, wb, cr, cm, total;
    __host__ __device__ Smem4(int lmax, int S, bool has_m, bool has_f, bool nodal_c, bool nodal_s, int max_bnodes,
                              int max_recs, int max_chunks) {
        auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
        size_t o = 0;
        accK = o; o = al(o + sizeof(double) * size_t(lmax) * S);
        accM = o; o = al(o + (has_m ? sizeof(double) * size_t(lmax) * S : 0));
        accF = o; o = al(o + (has_f ? sizeof(double) * size_t(S) : 0));
        nt = o; o = al(o + sizeof(double) * size_t(max_bnodes) * d);
        ntc = o; o = al(o + (nodal_c ? sizeof(double) * size_t(max_bnodes) : 0));
        nts = o; o = al(o + (nodal_s ? sizeof(double) * size_t(max_bnodes) : 0));
        hc = o; o = al(o + sizeof(uint64_t) * size_t(T) * kRing4);
        rc = o; o = al(o + sizeof(uint32_t) * size_t(max_recs) * kRing4);
        wb = o; o = al(o + sizeof(uint16_t) * 8 * kRing4);
        cr = o; o = al(o + sizeof(int64_t) * size_t(max_chunks + 1));
        cm = o; o = al(o + sizeof(uint32_t) * size_t(max_chunks));
        total = o;
    }
};

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int T, bool FDIV>
__global__ void __launch_bounds__(T, T == 256 ? 2 : 4) k_fused4(Fused4Args p) {
    using Rl = Rule<KIND, DEG>;
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rl::Q;
    extern __shared__ __align__(16) unsigned char smem4[];
    const bool nodal_c = p.coef.type == TGK_FIELD_NODAL;
    const bool nodal_s = HAS_F && p.src.type == TGK_FIELD_NODAL;
    const Smem4<KIND, T> L(p.lmax, p.S, HAS_M, HAS_F, nodal_c, nodal_s, p.max_bnodes, p.max_recs, p.max_chunks);
    double* accK = reinterpret_cast<double*>(smem4 + L.accK);
    double* accM = reinterpret_cast<double*>(smem4 + L.accM);
    double* accF = reinterpret_cast<double*>(smem4 + L.accF);
    double* nt = reinterpret_cast<double*>(smem4 + L.nt);
    double* ntc = reinterpret_cast<double*>(smem4 + L.ntc);
    double* nts = reinterpret_cast<double*>(smem4 + L.nts);
    uint64_t* hc_s = reinterpret_cast<uint64_t*>(smem4 + L.hc);
    uint32_t* rc_s = reinterpret_cast<uint32_t*>(smem4 + L.rc);
    uint16_t* wb_s = reinterpret_cast<uint16_t*>(smem4 + L.wb);
    int64_t* cr_s = reinterpret_cast<int64_t*>(smem4 + L.cr);
    uint32_t* cm_s = reinterpret_cast<uint32_t*>(smem4 + L.cm);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t blk = blockIdx.x;
    const int64_t r0 = p.row_off[blk];
    const int nr = static_cast<int>(p.row_off[blk + 1] - r0);
    const int64_t h0 = p.halo_off[blk];
    const int64_t nh = p.halo_off[blk + 1] - h0;
    const int64_t c0 = p.chunk_off[blk];
    const int nch = static_cast<int>(p.chunk_off[blk + 1] - c0);
    const int64_t n0 = p.bnode_off[blk];
    const int nbn = static_cast<int>(p.bnode_off[blk + 1] - n0);

    for (int i = tid; i <= nch; i += T) cr_s[i] = p.chunk_rec[c0 + i];
    for (int i = tid; i < nch; i += T) cm_s[i] = p.chunk_meta[c0 + i];
    // zero the accumulators (+0.0: the reference fold's start, routing.cpp:119)
    for (int i = tid; i < p.lmax * p.S; i += T) {
        accK[i] = 0.0;
        if constexpr (HAS_M) accM[i] = 0.0;
    }
    if constexpr (HAS_F)
        for (int i = tid; i < p.S; i += T) accF[i] = 0.0;
    // node table (coordinates [+ nodal coefficient / source]) by cp.async
    for (int i = tid; i < nbn; i += T) {
        const int64_t g = p.bnodes[n0 + i];
#pragma unroll
        for (int c = 0; c < d; ++c) cp_async8(nt + i * d + c, p.nodes + g * d + c);
        if (nodal_c) cp_async8(ntc + i, p.coef.data + g);
        if (nodal_s) cp_async8(nts + i, p.src.data + g);
    }
    cp_async_commit();
    __syncthreads();  // chunk table visible

    // stage chunk c's connectivity, records and warp bases into ring slot c % kRing4
    auto stage = [&](int c) {
        if (c < nch) {
            const int sl = c % kRing4;
            const int64_t hb = h0 + int64_t(c) * T;
            const int64_t rem = nh - int64_t(c) * T;
            const int ne = rem < T ? static_cast<int>(rem) : T;
            uint64_t* hdst = hc_s + sl * T;
            if (tid < ne) cp_async8(hdst + tid, p.hconn + hb + tid);
            const int64_t rb = cr_s[c];
            const int nrec4 = static_cast<int>((cr_s[c + 1] - rb) >> 2);
            uint32_t* rdst = rc_s + sl * p.max_recs;
            for (int i = tid; i < nrec4; i += T) cp_async16(rdst + 4 * i, p.recs + rb + 4 * i);
            if (tid == 0) cp_async16(wb_s + sl * 8, p.chunk_wbase + (c0 + c) * 8);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int c = 0; c < kRing4 - 1; ++c) stage(c);

    for (int c = 0; c < nch; ++c) {
        cp_async_wait<kRing4 - 2>();  // chunk c (and the node table) landed
        __syncthreads();              // ... and is visible; chunk c-1's updates are complete
        stage(c + kRing4 - 1);        // into the slot chunk c-1 released
        const int sl = c % kRing4;
        const int64_t h = int64_t(c) * T + tid;
        const bool valid = h < nh;
        int ln[4] = {0, 0, 0, 0};
        unsigned mask = 0;
        double Kv[k][k], Mv[HAS_M ? k : 1][HAS_M ? k : 1], Fv[HAS_F ? k : 1];
        if (valid) {
            const uint64_t hcv = hc_s[sl * T + tid];
#pragma unroll
            for (int a = 0; a < k; ++a) {
                ln[a] = static_cast<int>((hcv >> (16 * a)) & 0xffff);
                if (ln[a] < nr) mask |= 1u << a;
            }
            double X[k][d], cu[k], fu[k];
#pragma unroll
            for (int a = 0; a < k; ++a) {
#pragma unroll
                for (int cc = 0; cc < d; ++cc) X[a][cc] = nt[ln[a] * d + cc];
                cu[a] = nodal_c ? ntc[ln[a]] : 0.0;
                fu[a] = nodal_s ? nts[ln[a]] : 0.0;
            }
            const bool elem_c = p.coef.type == TGK_FIELD_ELEMENT;
            const bool elem_s = HAS_F && p.src.type == TGK_FIELD_ELEMENT;
            if (elem_c || elem_s) {
                const int64_t e = p.halo[h0 + h];
                if (elem_c) cu[0] = __ldg(p.coef.data + e);
                if (elem_s) fu[0] = __ldg(p.src.data + e);
            }
            double det, G[k][d];
            if (!simplex_geometry<KIND, FDIV>(X, det, G)) {
                atomicMin(p.bad, static_cast<unsigned long long>(p.halo[h0 + h]));
                det = 0.0;
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int cc = 0; cc < d; ++cc) G[a][cc] = 0.0;
            }
            double sc[Q];  // w_q * det * c_q  (batch.cpp:169 / :261)
#pragma unroll
            for (int q = 0; q < Q; ++q) sc[q] = Rl::w(q) * det * field4_q<KIND, DEG>(p.coef.type, p.coef.value, cu, q);
            if constexpr (KTYPE == 0) {
                // local_stiffness_diffusion (batch.cpp:168-177); K_e symmetric bitwise
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int b = a; b < k; ++b) {
                        const double dot = gdot<KIND>(G, a, b);
                        double v = sc[0] * dot;
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += sc[q] * dot;
                        Kv[a][b] = v;
                        Kv[b][a] = v;
                    }
            } else {
                // local_mass with the coefficient (batch.cpp:259-265)
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int b = 0; b < k; ++b) {
                        double v = sc[0] * basis<KIND, DEG>(0, a) * basis<KIND, DEG>(0, b);
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += sc[q] * basis<KIND, DEG>(q, a) * basis<KIND, DEG>(q, b);
                        Kv[a][b] = v;
                    }
            }
            if constexpr (HAS_M) {
                // with_mass: local_mass with ones (physics.cpp:70-71); w*det*1.0 == w*det
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int b = 0; b < k; ++b) {
                        double v = Rl::w(0) * det * basis<KIND, DEG>(0, a) * basis<KIND, DEG>(0, b);
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += Rl::w(q) * det * basis<KIND, DEG>(q, a) * basis<KIND, DEG>(q, b);
                        Mv[a][b] = v;
                    }
            }
            if constexpr (HAS_F) {
                // local_load (batch.cpp:280-286)
                double sf[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) sf[q] = Rl::w(q) * det * field4_q<KIND, DEG>(p.src.type, p.src.value, fu, q);
#pragma unroll
                for (int a = 0; a < k; ++a) {
                    double v = sf[0] * basis<KIND, DEG>(0, a);
#pragma unroll
                    for (int q = 1; q < Q; ++q) v += sf[q] * basis<KIND, DEG>(q, a);
                    Fv[a] = v;
                }
            }
        }
        // this thread's update records: one per owned local node, in a order,
        // at (warp base + exclusive warp prefix of the owned counts)
        const int cnt = __popc(mask);
        int x = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        const uint32_t* rs = rc_s + sl * p.max_recs + wb_s[sl * 8 + warp] + (x - cnt);
        uint32_t rec[4] = {0, 0, 0, 0};
        {
            int j = 0;
#pragma unroll
            for (int a = 0; a < k; ++a)
                if (mask & (1u << a)) rec[a] = rs[j++];
        }
        const int nrounds = static_cast<int>(cm_s[c]);
        for (int r = 0; r < nrounds; ++r) {
            if (r > 0) __syncthreads();
#pragma unroll
            for (int a = 0; a < k; ++a) {
                if ((mask & (1u << a)) && static_cast<int>((rec[a] >> 24) & 31) == r) {
                    const int row = ln[a];
                    int pos[k];
                    double ok[k], om[HAS_M ? k : 1];
#pragma unroll
                    for (int b = 0; b < k; ++b) {
                        pos[b] = static_cast<int>((rec[a] >> (5 * b)) & 31) * p.S + row;
                        ok[b] = accK[pos[b]];
                        if constexpr (HAS_M) om[b] = accM[pos[b]];
                    }
                    double of = 0.0;
                    if constexpr (HAS_F) of = accF[row];
#pragma unroll
                    for (int b = 0; b < k; ++b) {
                        accK[pos[b]] = ok[b] + Kv[a][b];
                        if constexpr (HAS_M) accM[pos[b]] = om[b] + Mv[a][b];
                    }
                    if constexpr (HAS_F) accF[row] = of + Fv[a];
                }
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    // epilogue: owned rows -> CSR values; one warp store per row (contiguous run)
    constexpr int W = T / 32;
    for (int rb = warp * 32; rb < nr; rb += W * 32) {
        const int64_t my = rb + lane < nr ? p.rows_rp[r0 + rb + lane] : 0;
        const int nn = nr - rb < 32 ? nr - rb : 32;
        for (int i = 0; i < nn; ++i) {
            const long long pk = __shfl_sync(0xffffffffu, static_cast<long long>(my), i);
            const int64_t rp = pk & ((int64_t(1) << 56) - 1);
            const int len = static_cast<int>(pk >> 56);
            if (lane < len) {
                p.K[rp + lane] = accK[lane * p.S + rb + i];
                if constexpr (HAS_M) p.M[rp + lane] = accM[lane * p.S + rb + i];
            }
        }
    }
    if constexpr (HAS_F)
        for (int i = tid; i < nr; i += T) p.F[p.rows[r0 + i]] = accF[i];
}

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int T, bool FDIV>
int launch4(const Fused4Args& a, int64_t n_blocks, cudaStream_t st) {
    auto kern = k_fused4<KIND, DEG, KTYPE, HAS_M, HAS_F, T, FDIV>;
    const Smem4<KIND, T> L(a.lmax, a.S, HAS_M, HAS_F, a.coef.type == TGK_FIELD_NODAL,
                           HAS_F && a.src.type == TGK_FIELD_NODAL, a.max_bnodes, a.max_recs, a.max_chunks);
    if (L.total > 227 * 1024)
        return set_error(TGK_ERR_INPUT, "fused assembly: block working set exceeds shared memory (" +
                                            std::to_string(L.total) + " B)");
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    if (n_blocks > 0) kern<<<static_cast<unsigned>(n_blocks), T, L.total, st>>>(a);
    KERNEL_CHECK("fused4");
    return TGK_OK;
}

template <int KIND, int DEG, int T, bool FDIV>
int dispatch4_t(int ktype, bool m, bool f, const Fused4Args& a, int64_t nb, cudaStream_t st) {
    if (ktype == 1) return launch4<KIND, DEG, 1, false, false, T, FDIV>(a, nb, st);
    if (m && f) return launch4<KIND, DEG, 0, true, true, T, FDIV>(a, nb, st);
    if (m) return launch4<KIND, DEG, 0, true, false, T, FDIV>(a, nb, st);
    if (f) return launch4<KIND, DEG, 0, false, true, T, FDIV>(a, nb, st);
    return launch4<KIND, DEG, 0, false, false, T, FDIV>(a, nb, st);
}

template <int KIND, int DEG>
int dispatch4(int ktype, bool m, bool f, const Fused4Args& a, int64_t nb, int T, bool fdiv, cudaStream_t st) {
    if (T == 256)
        return fdiv ? dispatch4_t<KIND, DEG, 256, true>(ktype, m, f, a, nb, st)
                    : dispatch4_t<KIND, DEG, 256, false>(ktype, m, f, a, nb, st);
    return fdiv ? dispatch4_t<KIND, DEG, 128, true>(ktype, m, f, a, nb, st)
                : dispatch4_t<KIND, DEG, 128, false>(ktype, m, f, a, nb, st);
}

}  // namespace

// Block shape of the v4 kernel: R rows per block, T threads (= elements per chunk).
void fused4_shape(const tgk_problem* pr, int* R, int* T) {
    *R = 256;
    *T = 128;
    (void)pr;
    if (const char* e = getenv("TGK4_R")) *R = atoi(e);
    if (const char* e = getenv("TGK4_T")) *T = atoi(e) == 256 ? 256 : 128;
}

int fused4_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                           double* M, cudaStream_t st, unsigned long long* d_bad) {
    int R, T;
    fused4_shape(pr, &R, &T);
    const PlanDev4* pl = nullptr;
    TGK_TRY(ensure_plan4(r, R, T, &pl));
    const bool is_mass = pr->kind == TGK_MASS;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT || is_mass || pr->with_mass;
    const int degree = high ? 2 : 1;  // default_mass_degree / default_stiffness_degree for P1
    const bool has_f = !is_mass && pr->n_source > 0;
    const bool has_m = pr->with_mass != 0;
    Fused4Args a{};
    a.nodes = m->nodes;
    a.row_off = pl->row_off;
    a.rows = pl->rows;
    a.rows_rp = pl->rows_rp;
    a.bnode_off = pl->bnode_off;
    a.bnodes = pl->bnodes;
    a.halo_off = pl->halo_off;
    a.halo = pl->halo;
    a.hconn = pl->hconn;
    a.chunk_off = pl->chunk_off;
    a.chunk_rec = pl->chunk_rec;
    a.chunk_meta = pl->chunk_meta;
    a.chunk_wbase = pl->chunk_wbase;
    a.recs = pl->recs;
    a.coef = Field4{pr->diffusion.type, pr->diffusion.value, pr->diffusion.data};
    a.src = Field4{TGK_FIELD_CONSTANT, 0.0, nullptr};
    if (has_f) a.src = Field4{pr->source[0].type, pr->source[0].value, pr->source[0].data};
    a.K = K;
    a.M = M;
    a.F = F;
    a.lmax = pl->lmax > 0 ? pl->lmax : 1;
    a.S = pl->R | 1;
    a.max_recs = pl->max_chunk_recs > 0 ? pl->max_chunk_recs : 4;
    a.max_bnodes = pl->max_bnodes + (pl->max_bnodes & 1);
    a.max_chunks = pl->max_block_chunks;
    DevBuf<unsigned long long> bad;
    if (!d_bad) TGK_TRY(bad.alloc(1));
    a.bad = d_bad ? d_bad : bad.p;
    CUDA_TRY(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), st));
    if (!has_f && F) CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
    const int ktype = is_mass ? 1 : 0;
    bool fdiv = false;
    TGK_TRY(mesh_division_safe(const_cast<tgk_mesh*>(m), st, &fdiv));
    if (getenv("TGK_IEEE_DIV")) fdiv = false;
    if (m->kind == TGK_TET4) {
        if (degree == 1) TGK_TRY((dispatch4<TGK_TET4, 1>(ktype, has_m, has_f, a, pl->n_blocks, T, fdiv, st)));
        else TGK_TRY((dispatch4<TGK_TET4, 2>(ktype, has_m, has_f, a, pl->n_blocks, T, fdiv, st)));
    } else {
        if (degree == 1) TGK_TRY((dispatch4<TGK_TRI3, 1>(ktype, has_m, has_f, a, pl->n_blocks, T, fdiv, st)));
        else TGK_TRY((dispatch4<TGK_TRI3, 2>(ktype, has_m, has_f, a, pl->n_blocks, T, fdiv, st)));
    }
    if (!d_bad) return check_bad(bad.p, st);
    return TGK_OK;
}

}  // namespace tgk
