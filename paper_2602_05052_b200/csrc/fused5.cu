// Fused P1 Map+Reduce assembly, v5, for scalar problems (tg::assemble,
// physics.cpp:10-75): stiffness (or coefficient mass), optional unit mass M
// and load F, from mesh + coefficients straight to CSR values — no local
// tensor in HBM, no atomics, bit-identical to the reference.
//
// Decomposition as v3 (fused.cu): CUDA block b owns R CSR rows (Morton-compact
// mesh nodes) and recomputes the elements incident to them (its halo) in
// level order, R elements per chunk:
//   prologue  block node table (coordinates [+ nodal fields]) by cp.async;
//   phase A   one thread per element: exact local K_e / M_e / F_e
//             (element.cuh) into shared memory, rows "rotated" (diagonal
//             first, pack_rec order);
//   phase B   one thread per WORK ITEM = an owned row with records in this
//             chunk (plan5.cpp; items sorted by record count so warps are
//             balanced and idle rows cost nothing): the row's diagonal, mass
//             diagonal and load are read into registers, its records folded
//             in ascending element order (off-diagonals as shared-memory
//             read-modify-writes), then written back;
//   epilogue  one warp per row stores the row's CSR run contiguously.
// Every CSR value is thus the left fold from +0.0 of its contributions in
// ascending element order — the reference's Reduce (routing.cpp:117-124).
#include <cstdio>
#include <vector>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);
int mesh_division_safe(tgk_mesh* m, cudaStream_t st, bool* safe);

namespace {

struct Field5 {
    int type;
    double value;
    const double* data;
};

struct Fused5Args {
    const double* nodes;
    const int64_t* row_off;
    const uint32_t* rows;
    const int64_t* rows_rp;
    const int64_t* halo_off;
    const uint32_t* halo;
    const int64_t* bnode_off;
    const uint32_t* bnodes;
    const uint16_t* halo_lconn;
    const int64_t* chunk_off;
    const int64_t* chunk_rec;
    const int64_t* chunk_item;
    const uint32_t* chunk_nitems;
    const uint32_t* items;
    const uint32_t* recs;
    Field5 coef, src;
    double* K;
    double* M;
    double* F;
    int lmax, S, max_recs, max_items, max_bnodes, max_chunks;
    unsigned long long* bad;
};

#ifndef TGK5_RING
#define TGK5_RING 3
#endif
constexpr int kRing5 = TGK5_RING;

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

// Slot of K_e[a][b] within the rotated row a: 0 for the diagonal, then the
// other local nodes ascending (pack_rec order).
__host__ __device__ constexpr int rot5(int a, int b) { return b == a ? 0 : (b < a ? b + 1 : b); }

template <int KIND, int DEG>
__device__ __forceinline__ double field5_q(int type, double value, const double* u, int q) {
    constexpr int k = P1<KIND>::k;
    if (type == TGK_FIELD_NODAL) {  // interpolate_nodal (batch.cpp:321-330)
        double v = basis<KIND, DEG>(q, 0) * u[0];
#pragma unroll
        for (int a = 1; a < k; ++a) v += basis<KIND, DEG>(q, a) * u[a];
        return v;
    }
    return type == TGK_FIELD_ELEMENT ? u[0] : value;
}

// Per-element tensor layout in shared memory (doubles): K rows 4x4 rotated,
// then M rows (HAS_M), then F (HAS_F); stride = 2 x odd (conflict-free
// 128-bit accesses by lanes with consecutive elements).
template <bool HAS_M, bool HAS_F>
struct KeLayout {
    static constexpr int offK = 0, offM = 16, offF = 16 + (HAS_M ? 16 : 0);
    static constexpr int raw = offF + (HAS_F ? 4 : 0);
    static constexpr int stride = (raw / 2) % 2 == 1 ? raw : raw + 2;
};

struct Smem5 {
    size_t ke, accK, accM, accF, nt, ntc, nts, lc, rc, it, cr, ci, cn, total;
    __host__ __device__ Smem5(int R, int d, int ke_stride, int lmax, int S, bool has_m, bool has_f, bool nodal_c,
                              bool nodal_s, int max_bnodes, int max_recs, int max_items, int max_chunks) {
        auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
        size_t o = 0;
        ke = o; o = al(o + sizeof(double) * size_t(R) * ke_stride);
        accK = o; o = al(o + sizeof(double) * size_t(lmax) * S);
        accM = o; o = al(o + (has_m ? sizeof(double) * size_t(lmax) * S : 0));
        accF = o; o = al(o + (has_f ? sizeof(double) * size_t(R) : 0));
        nt = o; o = al(o + sizeof(double) * size_t(max_bnodes) * d);
        ntc = o; o = al(o + (nodal_c ? sizeof(double) * size_t(max_bnodes) : 0));
        nts = o; o = al(o + (nodal_s ? sizeof(double) * size_t(max_bnodes) : 0));
        lc = o; o = al(o + sizeof(uint64_t) * size_t(R) * kRing5);
        rc = o; o = al(o + sizeof(uint32_t) * size_t(max_recs) * kRing5);
        it = o; o = al(o + sizeof(uint32_t) * size_t(max_items) * kRing5);
        cr = o; o = al(o + sizeof(int64_t) * size_t(max_chunks + 1));
        ci = o; o = al(o + sizeof(int64_t) * size_t(max_chunks + 1));
        cn = o; o = al(o + sizeof(uint32_t) * size_t(max_chunks + 1));
        total = o;
    }
};

// Phase A body: the reference's local kernels for one element into `out`.
template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, bool FDIV>
__device__ __forceinline__ void element5(const Fused5Args& p, const double* nt, const double* ntc,
                                         const double* nts, const ushort4 ln, int64_t h_global, double* out) {
    using Lk = KeLayout<HAS_M, HAS_F>;
    using Rl = Rule<KIND, DEG>;
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rl::Q;
    const int ids[4] = {ln.x, ln.y, ln.z, ln.w};
    double X[k][d], cu[k], fu[k];
#pragma unroll
    for (int a = 0; a < k; ++a) {
#pragma unroll
        for (int c = 0; c < d; ++c) X[a][c] = nt[ids[a] * d + c];
        cu[a] = p.coef.type == TGK_FIELD_NODAL ? ntc[ids[a]] : 0.0;
        fu[a] = (HAS_F && p.src.type == TGK_FIELD_NODAL) ? nts[ids[a]] : 0.0;
    }
    if (p.coef.type == TGK_FIELD_ELEMENT || (HAS_F && p.src.type == TGK_FIELD_ELEMENT)) {
        const int64_t e = p.halo[h_global];
        if (p.coef.type == TGK_FIELD_ELEMENT) cu[0] = __ldg(p.coef.data + e);
        if (HAS_F && p.src.type == TGK_FIELD_ELEMENT) fu[0] = __ldg(p.src.data + e);
    }
    double det, G[k][d];
    if (!simplex_geometry<KIND, FDIV>(X, det, G)) {
        atomicMin(p.bad, static_cast<unsigned long long>(p.halo[h_global]));
#pragma unroll
        for (int i = 0; i < Lk::raw; ++i) out[i] = 0.0;
        return;
    }
    double sc[Q];  // w_q * det * c_q  (batch.cpp:169 / :261)
#pragma unroll
    for (int q = 0; q < Q; ++q) sc[q] = Rl::w(q) * det * field5_q<KIND, DEG>(p.coef.type, p.coef.value, cu, q);
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
                out[Lk::offK + a * 4 + rot5(a, b)] = v;
                out[Lk::offK + b * 4 + rot5(b, a)] = v;
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
                out[Lk::offK + a * 4 + rot5(a, b)] = v;
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
                out[Lk::offM + a * 4 + rot5(a, b)] = v;
            }
    }
    if constexpr (HAS_F) {
        // local_load (batch.cpp:280-286)
        double sf[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) sf[q] = Rl::w(q) * det * field5_q<KIND, DEG>(p.src.type, p.src.value, fu, q);
#pragma unroll
        for (int a = 0; a < k; ++a) {
            double v = sf[0] * basis<KIND, DEG>(0, a);
#pragma unroll
            for (int q = 1; q < Q; ++q) v += sf[q] * basis<KIND, DEG>(q, a);
            out[Lk::offF + a] = v;
        }
    }
}

template <int R>
constexpr int minb5() { return R == 256 ? 2 : (R == 128 ? 4 : 8); }

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int R, bool FDIV>
__global__ void __launch_bounds__(R, minb5<R>()) k_fused5(Fused5Args p) {
    using Lk = KeLayout<HAS_M, HAS_F>;
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
    extern __shared__ __align__(16) unsigned char smem5[];
    const bool nodal_c = p.coef.type == TGK_FIELD_NODAL;
    const bool nodal_s = HAS_F && p.src.type == TGK_FIELD_NODAL;
    const Smem5 L(R, d, Lk::stride, p.lmax, p.S, HAS_M, HAS_F, nodal_c, nodal_s, p.max_bnodes, p.max_recs,
                  p.max_items, p.max_chunks);
    double* ke = reinterpret_cast<double*>(smem5 + L.ke);
    double* accK = reinterpret_cast<double*>(smem5 + L.accK);
    double* accM = reinterpret_cast<double*>(smem5 + L.accM);
    double* accF = reinterpret_cast<double*>(smem5 + L.accF);
    double* nt = reinterpret_cast<double*>(smem5 + L.nt);
    double* ntc = reinterpret_cast<double*>(smem5 + L.ntc);
    double* nts = reinterpret_cast<double*>(smem5 + L.nts);
    ushort4* lc_s = reinterpret_cast<ushort4*>(smem5 + L.lc);
    uint32_t* rc_s = reinterpret_cast<uint32_t*>(smem5 + L.rc);
    uint32_t* it_s = reinterpret_cast<uint32_t*>(smem5 + L.it);
    int64_t* cr_s = reinterpret_cast<int64_t*>(smem5 + L.cr);
    int64_t* ci_s = reinterpret_cast<int64_t*>(smem5 + L.ci);
    uint32_t* cn_s = reinterpret_cast<uint32_t*>(smem5 + L.cn);

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

    for (int i = tid; i <= nch; i += R) {
        cr_s[i] = p.chunk_rec[c0 + i];
        ci_s[i] = p.chunk_item[c0 + i];
        if (i < nch) cn_s[i] = p.chunk_nitems[c0 + i];
    }
    // node table by cp.async (one commit group, completed with chunk 0)
    for (int i = tid; i < nbn; i += R) {
        const int64_t g = p.bnodes[n0 + i];
#pragma unroll
        for (int c = 0; c < d; ++c) cp_async8(nt + i * d + c, p.nodes + g * d + c);
        if (nodal_c) cp_async8(ntc + i, p.coef.data + g);
        if (nodal_s) cp_async8(nts + i, p.src.data + g);
    }
    cp_async_commit();
    // accumulators start at +0.0 (the reference fold's start, routing.cpp:119)
    for (int i = tid; i < p.lmax * p.S; i += R) {
        accK[i] = 0.0;
        if constexpr (HAS_M) accM[i] = 0.0;
    }
    if constexpr (HAS_F) accF[tid] = 0.0;
    __syncthreads();  // chunk tables visible

    auto stage = [&](int c) {
        if (c < nch) {
            const int sl = c % kRing5;
            const int64_t hb = h0 + int64_t(c) * R;
            const int64_t rem = nh - int64_t(c) * R;
            const int ne = rem < R ? static_cast<int>(rem) : R;
            if (tid < ne) cp_async8(lc_s + sl * R + tid, p.halo_lconn + (hb + tid) * 4);
            const int64_t rb = cr_s[c];
            const int nrec4 = static_cast<int>((cr_s[c + 1] - rb) >> 2);
            uint32_t* rdst = rc_s + sl * p.max_recs;
            for (int i = tid; i < nrec4; i += R) cp_async16(rdst + 4 * i, p.recs + rb + 4 * i);
            const int64_t ib = ci_s[c];
            const int nit4 = static_cast<int>((ci_s[c + 1] - ib) >> 2);
            uint32_t* idst = it_s + sl * p.max_items;
            for (int i = tid; i < nit4; i += R) cp_async16(idst + 4 * i, p.items + ib + 4 * i);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int c = 0; c < kRing5 - 1; ++c) stage(c);

    for (int c = 0; c < nch; ++c) {
        cp_async_wait<kRing5 - 2>();  // chunk c (and the node table) landed
        __syncthreads();              // visible; phase B(c-1) done with ke and its ring slot
        stage(c + kRing5 - 1);
        const int sl = c % kRing5;
        // ---------------- phase A: this thread's element of chunk c
        const int64_t h = int64_t(c) * R + tid;
        if (h < nh)
            element5<KIND, DEG, KTYPE, HAS_M, HAS_F, FDIV>(p, nt, ntc, nts, lc_s[sl * R + tid], h0 + h,
                                                           ke + tid * Lk::stride);
        __syncthreads();
        // ---------------- phase B: work item tid folds its row's records of chunk c
        if (tid < static_cast<int>(cn_s[c])) {
            const uint32_t item = it_s[sl * p.max_items + tid];
            const int lr = item & 0xff;
            const int cnt = (item >> 8) & 0xff;
            const uint32_t* rs = rc_s + sl * p.max_recs + (item >> 16);
            uint32_t rec = rs[0];
            const int dpos = ((rec >> 25) & 31) * p.S + lr;
            double dK = accK[dpos], dM = 0.0, dF = 0.0;
            if constexpr (HAS_M) dM = accM[dpos];
            if constexpr (HAS_F) dF = accF[lr];
            for (int j = 0; j < cnt; ++j) {
                const uint32_t rec_n = j + 1 < cnt ? rs[j + 1] : rec;
                const int hl = rec & 0xff;
                const int a = (rec >> 8) & 3;
                const double* src = ke + hl * Lk::stride + a * 4;
                const double2 k01 = *reinterpret_cast<const double2*>(src + Lk::offK);
                const double2 k23 = *reinterpret_cast<const double2*>(src + Lk::offK + 2);
                double2 m01 = make_double2(0.0, 0.0), m23 = m01;
                if constexpr (HAS_M) {
                    m01 = *reinterpret_cast<const double2*>(src + Lk::offM);
                    m23 = *reinterpret_cast<const double2*>(src + Lk::offM + 2);
                }
                double fv = 0.0;
                if constexpr (HAS_F) fv = ke[hl * Lk::stride + Lk::offF + a];
                const double kv[4] = {k01.x, k01.y, k23.x, k23.y};
                const double mv[4] = {m01.x, m01.y, m23.x, m23.y};
                // the k-1 positions of one record are distinct columns: load all, add, store all
                int pos[k - 1];
                double ak[k - 1], am[k - 1];
#pragma unroll
                for (int j2 = 0; j2 < k - 1; ++j2) {
                    pos[j2] = ((rec >> (10 + 5 * j2)) & 31) * p.S + lr;
                    ak[j2] = accK[pos[j2]];
                    if constexpr (HAS_M) am[j2] = accM[pos[j2]];
                }
#pragma unroll
                for (int j2 = 0; j2 < k - 1; ++j2) {
                    accK[pos[j2]] = ak[j2] + kv[j2 + 1];
                    if constexpr (HAS_M) accM[pos[j2]] = am[j2] + mv[j2 + 1];
                }
                dK += kv[0];
                if constexpr (HAS_M) dM += mv[0];
                if constexpr (HAS_F) dF += fv;
                rec = rec_n;
            }
            accK[dpos] = dK;
            if constexpr (HAS_M) accM[dpos] = dM;
            if constexpr (HAS_F) accF[lr] = dF;
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    // ---------------- epilogue: one warp per row, contiguous CSR runs
    constexpr int W = R / 32;
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
        if (tid < nr) p.F[p.rows[r0 + tid]] = accF[tid];
}

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int R, bool FDIV>
int launch5(const Fused5Args& a, int64_t n_blocks, cudaStream_t st) {
    using Lk = KeLayout<HAS_M, HAS_F>;
    auto kern = k_fused5<KIND, DEG, KTYPE, HAS_M, HAS_F, R, FDIV>;
    const Smem5 L(R, P1<KIND>::d, Lk::stride, a.lmax, a.S, HAS_M, HAS_F, a.coef.type == TGK_FIELD_NODAL,
                  HAS_F && a.src.type == TGK_FIELD_NODAL, a.max_bnodes, a.max_recs, a.max_items, a.max_chunks);
    if (L.total > 227 * 1024)
        return set_error(TGK_ERR_INPUT, "fused assembly: block working set exceeds shared memory (" +
                                            std::to_string(L.total) + " B)");
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    if (n_blocks > 0) kern<<<static_cast<unsigned>(n_blocks), R, L.total, st>>>(a);
    KERNEL_CHECK("fused5");
    return TGK_OK;
}

template <int KIND, int DEG, int R, bool FDIV>
int dispatch5_r(int ktype, bool m, bool f, const Fused5Args& a, int64_t nb, cudaStream_t st) {
    if (ktype == 1) return launch5<KIND, DEG, 1, false, false, R, FDIV>(a, nb, st);
    if (m && f) return launch5<KIND, DEG, 0, true, true, R, FDIV>(a, nb, st);
    if (m) return launch5<KIND, DEG, 0, true, false, R, FDIV>(a, nb, st);
    if (f) return launch5<KIND, DEG, 0, false, true, R, FDIV>(a, nb, st);
    return launch5<KIND, DEG, 0, false, false, R, FDIV>(a, nb, st);
}

template <int KIND, int DEG>
int dispatch5(int ktype, bool m, bool f, const Fused5Args& a, int64_t nb, int R, bool fdiv, cudaStream_t st) {
    if (R == 256)
        return fdiv ? dispatch5_r<KIND, DEG, 256, true>(ktype, m, f, a, nb, st)
                    : dispatch5_r<KIND, DEG, 256, false>(ktype, m, f, a, nb, st);
    if (R == 64)
        return fdiv ? dispatch5_r<KIND, DEG, 64, true>(ktype, m, f, a, nb, st)
                    : dispatch5_r<KIND, DEG, 64, false>(ktype, m, f, a, nb, st);
    return fdiv ? dispatch5_r<KIND, DEG, 128, true>(ktype, m, f, a, nb, st)
                : dispatch5_r<KIND, DEG, 128, false>(ktype, m, f, a, nb, st);
}

}  // namespace

int fused5_rows_per_block(const tgk_problem* pr) {
    (void)pr;
    if (const char* e = getenv("TGK5_R")) {
        const int r = atoi(e);
        return r == 64 || r == 256 ? r : 128;
    }
    return 128;
}

int fused5_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                           double* M, cudaStream_t st, unsigned long long* d_bad) {
    const int R = fused5_rows_per_block(pr);
    const PlanDev5* pl = nullptr;
    TGK_TRY(ensure_plan5(r, R, &pl));
    const bool is_mass = pr->kind == TGK_MASS;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT || is_mass || pr->with_mass;
    const int degree = high ? 2 : 1;  // default_mass_degree / default_stiffness_degree for P1
    const bool has_f = !is_mass && pr->n_source > 0;
    const bool has_m = pr->with_mass != 0;
    Fused5Args a{};
    a.nodes = m->nodes;
    a.row_off = pl->row_off;
    a.rows = pl->rows;
    a.rows_rp = pl->rows_rp;
    a.halo_off = pl->halo_off;
    a.halo = pl->halo;
    a.bnode_off = pl->bnode_off;
    a.bnodes = pl->bnodes;
    a.halo_lconn = pl->halo_lconn;
    a.chunk_off = pl->chunk_off;
    a.chunk_rec = pl->chunk_rec;
    a.chunk_item = pl->chunk_item;
    a.chunk_nitems = pl->chunk_nitems;
    a.items = pl->items;
    a.recs = pl->recs;
    a.coef = Field5{pr->diffusion.type, pr->diffusion.value, pr->diffusion.data};
    a.src = Field5{TGK_FIELD_CONSTANT, 0.0, nullptr};
    if (has_f) a.src = Field5{pr->source[0].type, pr->source[0].value, pr->source[0].data};
    a.K = K;
    a.M = M;
    a.F = F;
    a.lmax = pl->lmax > 0 ? pl->lmax : 1;
    a.S = pl->R | 1;
    a.max_recs = pl->max_chunk_recs > 0 ? pl->max_chunk_recs : 4;
    a.max_items = pl->max_chunk_items > 0 ? pl->max_chunk_items : 4;
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
        if (degree == 1) TGK_TRY((dispatch5<TGK_TET4, 1>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, st)));
        else TGK_TRY((dispatch5<TGK_TET4, 2>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, st)));
    } else {
        if (degree == 1) TGK_TRY((dispatch5<TGK_TRI3, 1>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, st)));
        else TGK_TRY((dispatch5<TGK_TRI3, 2>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, st)));
    }
    if (!d_bad) return check_bad(bad.p, st);
    return TGK_OK;
}

}  // namespace tgk
