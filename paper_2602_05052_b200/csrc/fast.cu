// Fast-mode fused P1 assembly (TGK_MODE_FAST) for scalar problems: the north
// star's design — a precomputed element-to-CSR-slot permutation (plan_fast.cpp)
// and a per-lane register fold straight into CSR values — with the
// reference's contract: pattern bit-exact, values within
// |dv| <= 1e-12 |v_ref| + 1e-14 max|v_ref|, run-to-run bitwise deterministic
// (fixed plan order, no atomics on values).
//
// One CUDA block owns R CSR rows and keeps its WHOLE halo (every element
// incident to an owned row) resident in shared memory:
//   prologue  owned rows' CSR offsets and the node table (coordinates of
//             every node the halo touches, plus nodal field values) gathered
//             into shared memory;
//   phase A   one thread per halo element: geometry with FMA, one
//             reciprocal, the k(k-1)/2 off-diagonal K_e values via the
//             gradient Gram matrix (row a = 0 from the zero row sum of P1
//             stiffness), and the scalars the mass / load are formed from
//             (det, f det) into structure-of-arrays value rows;
//   phase B   one lane per owned CSR entry (diagonal entries fold only the
//             row's mass / load): its items (u16 = halo index | value index
//             << 12, one coalesced 4-byte load per 2 items) are summed in
//             registers and the result stored to the entry — and to its
//             mirror (j, i) when j is owned by the same block;
//   copy-out  the tile to HBM as coalesced row segments, the stiffness
//             diagonal formed as 0 - (sum of the row's off-diagonals).
// Mass and load values are affine P1 closed forms of the reference's
// quadrature (batch.cpp:250-289): M_e = c det Mhat, F_e[a] = f det |T^|/k;
// with a nodal source F_e[a] = det sum_b Mhat[a][b] f_b.
#include <cstdio>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

namespace {

constexpr int kFastMaxThreads = 512;        // k_fast_elast
constexpr int kFastScalarMaxThreads = 1024;  // k_fast_scalar (<= 64 registers)

struct FastArgs {
    const double* nodes;
    FastPlanDev pl;
    int ctype;  // diffusion (stiffness) or mass coefficient: TGK_FIELD_*
    double cval;
    const double* cdata;
    int stype;  // source
    double sval;
    const double* sdata;
    double* K;
    double* M;
    double* F;
    int MH;    // value-row stride (max_halo + 1; the last slot is +0.0)
    int MB;    // node-table capacity
    int abuf;  // record buffer capacities in bytes (multiples of 16)
    int bbuf;
    int gl;     // copy-out lanes per row (8, 16 or 32 >= longest row)
    int debug;  // profiling only (TGK_FAST_DEBUG): 1 skips phase A, 2 phase B, 4 the copy-out, 8 the node gathers, 16 record B
    unsigned long long* bad;
};

// Affine P1 integrals over the reference element (exact values of the
// reference's degree-1/2 rules, reference.cpp:99-210).
template <int KIND>
struct FastConst;
template <>
struct FastConst<TGK_TET4> {
    static constexpr double wsum = 1.0 / 6.0;     // |T^|
    static constexpr double wa = 1.0 / 24.0;      // int N_a
    static constexpr double mdiag = 1.0 / 60.0;   // int N_a N_a
    static constexpr double moff = 1.0 / 120.0;   // int N_a N_b
    static constexpr int np = 10;
};
template <>
struct FastConst<TGK_TRI3> {
    static constexpr double wsum = 1.0 / 2.0;
    static constexpr double wa = 1.0 / 6.0;
    static constexpr double mdiag = 1.0 / 12.0;
    static constexpr double moff = 1.0 / 24.0;
    static constexpr int np = 6;
};

// KT 0: diffusion stiffness (+ unit mass M if HAS_M), 1: coefficient mass
// (ProblemKind::Mass).  FT: load none / scalar (f det; constant or
// per-element source) / per node (nodal source).
// Value rows in shared memory (row stride MH, plan_fast.cpp formats): K_ab
// off-diagonal pairs, [S = c det (mass) row], [F rows].  No K_aa rows: the
// stiffness diagonal is minus the row's off-diagonal sum (every element
// matrix has zero row sums), formed at the copy-out.
template <int KIND, int KT, bool HAS_M, int FT>
struct FastCfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
    static constexpr bool HAS_S = HAS_M || KT == 1;
    static constexpr int NPO = KT == 0 ? k * (k - 1) / 2 : 0;
    static constexpr int FMT = KT == 1 ? kFastFmtS16 : (HAS_M ? kFastFmtKS32 : kFastFmtK16);
    static constexpr int SROW = NPO;
    static constexpr int FROW = NPO + (HAS_S ? 1 : 0);
    static constexpr int NR = FMT == kFastFmtS16 ? 1 : (FMT == kFastFmtKS32 ? NPO + 2 : NPO + (FT == 2 ? k : 1));
    static constexpr int NTILE = HAS_M ? 2 : 1;
    // node table: coordinates (TRI3 as [node][2], one 16-byte load per node;
    // TET4 as x / y / z columns), then the nodal coefficient / source
    // columns; ncol in units of MB
    __host__ __device__ static int ncol(int ctype) { return d + (ctype == TGK_FIELD_NODAL ? 1 : 0) + (FT == 2 ? 1 : 0); }
    static size_t smem(const FastArgs& a) {
        return 64 + 2 * size_t(a.abuf) + size_t(a.bbuf) +
               sizeof(double) * (size_t(ncol(a.ctype)) * a.MB + size_t(NR) * a.MH + size_t(NTILE) * a.pl.max_tile) +
               sizeof(int64_t) * a.pl.max_rows + sizeof(uint16_t) * (a.pl.max_rows + 1) + ((size_t(a.pl.max_rows) + 15) & ~size_t(15));
    }
};

// 1/x for the fast mode: the hardware approximation refined by two Newton
// steps (relative error ~1 ulp, no special-case branches; x is a finite
// non-zero determinant — non-positive ones are rejected after the call, and a
// subnormal one, which the approximation flushes, belongs to no usable mesh)
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = __fma_rn(-x, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-x, r, 1.0);
    return __fma_rn(r, e, r);
}

__device__ __forceinline__ double dot3(double ax, double ay, double az, double bx, double by, double bz) {
    return __fma_rn(ax, bx, __fma_rn(ay, by, az * bz));
}

// ---------------------------------------------------------------- TMA / async-copy plumbing
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// one bulk (TMA) copy global -> shared completing on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ constexpr size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct RecA {
    int64_t hbase;
    uint32_t nr, nh, nbn, tile;
    const int64_t* rp;
    const uint32_t* srow;
    const uint16_t* toff;
    const uint32_t* bnodes;
    const void* hconn;  // per halo element 4 x u16 (or 4 x u8 with FastPlanDev::hc8) block-local node slots
};
// local node a of halo element h
template <int k>
__device__ __forceinline__ void halo_nodes(const RecA& A, int hc8, int h, int (&l)[k]) {
    if (hc8) {
        const uint32_t hc = static_cast<const uint32_t*>(A.hconn)[h];
#pragma unroll
        for (int a = 0; a < k; ++a) l[a] = static_cast<int>((hc >> (8 * a)) & 0xff);
    } else {
        const uint64_t hc = static_cast<const uint64_t*>(A.hconn)[h];
#pragma unroll
        for (int a = 0; a < k; ++a) l[a] = static_cast<int>((hc >> (16 * a)) & 0xffff);
    }
}
// STORED: read the section offsets from the header (k_fast_scalar: fewer
// instructions); else recompute them (k_fast_elast: fewer live registers —
// it runs capped at 64)
template <bool STORED = true>
__device__ __forceinline__ RecA parse_a(const unsigned char* r) {
    RecA a;
    a.hbase = *reinterpret_cast<const int64_t*>(r);
    const uint2 h0 = *reinterpret_cast<const uint2*>(r + 8), h1 = *reinterpret_cast<const uint2*>(r + 16);
    a.nr = h0.x;
    a.nh = h0.y;
    a.nbn = h1.x;
    a.tile = h1.y;
    a.rp = reinterpret_cast<const int64_t*>(r + 32);
    if constexpr (STORED) {
        const uint2 of = *reinterpret_cast<const uint2*>(r + 24);  // section offsets (plan_fast.cpp)
        a.srow = reinterpret_cast<const uint32_t*>(r + (of.x & 0xffffu));
        a.toff = reinterpret_cast<const uint16_t*>(r + (of.x >> 16));
        a.bnodes = reinterpret_cast<const uint32_t*>(r + (of.y & 0xffffu));
        a.hconn = r + (of.y >> 16);
    } else {
        size_t o = 32 + al16(8 * size_t(a.nr));
        a.srow = reinterpret_cast<const uint32_t*>(r + o);
        o += al16(4 * size_t(a.nr));
        a.toff = reinterpret_cast<const uint16_t*>(r + o);
        o += al16(2 * size_t(a.nr + 1));
        a.bnodes = reinterpret_cast<const uint32_t*>(r + o);
        o += al16(4 * size_t(a.nbn));
        a.hconn = r + o;
    }
    return a;
}
struct RecB {
    uint32_t ne, nwg;
    const uint32_t* desc;
    const uint32_t* wgoff;
    const uint32_t* words;
};
__device__ __forceinline__ RecB parse_b(const unsigned char* r) {
    RecB b;
    const uint2 h = *reinterpret_cast<const uint2*>(r);
    b.ne = h.x;
    b.nwg = h.y;
    size_t o = 16;
    b.desc = reinterpret_cast<const uint32_t*>(r + o);
    o += al16(4 * size_t(b.ne));
    b.wgoff = reinterpret_cast<const uint32_t*>(r + o);
    o += al16(4 * size_t(b.nwg + 1));
    b.words = reinterpret_cast<const uint32_t*>(r + o);
    return b;
}

// ---------------------------------------------------------------- phase A: one element
// Geometry with FMA and one reciprocal, the unique K_e values from the Gram
// matrix of the scaled gradients (row a = 0 from the zero row sums of P1
// stiffness), and the scalars the mass / load are formed from, stored to
// the value rows of halo slot h.
template <int KIND, int KT, bool HAS_M, int FT>
__device__ __forceinline__ void fast_element(const FastArgs& p, const RecA& A, const double* xs, double* kv, int h) {
    using Cf = FastCfg<KIND, KT, HAS_M, FT>;
    using Cn = FastConst<KIND>;
    constexpr int k = Cf::k, d = Cf::d;
    const int MH = p.MH, MB = p.MB;
    const double* cn = xs + d * MB;
    const double* sn = xs + (Cf::ncol(p.ctype) - 1) * MB;
    int l[k];
    halo_nodes<k>(A, p.pl.hc8, h, l);
    double det;
    double kp[Cn::np];
    auto coef_w = [&](double wsum_) -> double {
        if (p.ctype == TGK_FIELD_CONSTANT) return p.cval * wsum_;
        if (p.ctype == TGK_FIELD_ELEMENT) return __ldg(p.cdata + __ldg(p.pl.helem + A.hbase + h)) * wsum_;
        double sacc = cn[l[0]];
#pragma unroll
        for (int a = 1; a < k; ++a) sacc += cn[l[a]];
        return sacc * Cn::wa;
    };
    if constexpr (KIND == TGK_TET4) {
        const double x0 = xs[l[0]], y0 = xs[MB + l[0]], z0 = xs[2 * MB + l[0]];
        const double e1x = xs[l[1]] - x0, e1y = xs[MB + l[1]] - y0, e1z = xs[2 * MB + l[1]] - z0;
        const double e2x = xs[l[2]] - x0, e2y = xs[MB + l[2]] - y0, e2z = xs[2 * MB + l[2]] - z0;
        const double e3x = xs[l[3]] - x0, e3y = xs[MB + l[3]] - y0, e3z = xs[2 * MB + l[3]] - z0;
        // rows of J^{-1} times det: grad N_b = c_b / det (b = 1..3)
        const double c1x = __fma_rn(e2y, e3z, -(e2z * e3y)), c1y = __fma_rn(e2z, e3x, -(e2x * e3z)),
                     c1z = __fma_rn(e2x, e3y, -(e2y * e3x));
        const double c2x = __fma_rn(e3y, e1z, -(e3z * e1y)), c2y = __fma_rn(e3z, e1x, -(e3x * e1z)),
                     c2z = __fma_rn(e3x, e1y, -(e3y * e1x));
        const double c3x = __fma_rn(e1y, e2z, -(e1z * e2y)), c3y = __fma_rn(e1z, e2x, -(e1x * e2z)),
                     c3z = __fma_rn(e1x, e2y, -(e1y * e2x));
        det = dot3(e1x, e1y, e1z, c1x, c1y, c1z);
        if constexpr (KT == 0) {
            const double s = coef_w(Cn::wsum) * fast_rcp(det);
            const double k11 = s * dot3(c1x, c1y, c1z, c1x, c1y, c1z);
            const double k12 = s * dot3(c1x, c1y, c1z, c2x, c2y, c2z);
            const double k13 = s * dot3(c1x, c1y, c1z, c3x, c3y, c3z);
            const double k22 = s * dot3(c2x, c2y, c2z, c2x, c2y, c2z);
            const double k23 = s * dot3(c2x, c2y, c2z, c3x, c3y, c3z);
            const double k33 = s * dot3(c3x, c3y, c3z, c3x, c3y, c3z);
            const double k01 = -((k11 + k12) + k13), k02 = -((k12 + k22) + k23), k03 = -((k13 + k23) + k33);
            kp[0] = -((k01 + k02) + k03);  // kp: K_aa (unused: zero row sums), then 01 02 03 12 13 23
            kp[1] = k11; kp[2] = k22; kp[3] = k33;
            kp[4] = k01; kp[5] = k02; kp[6] = k03;
            kp[7] = k12; kp[8] = k13; kp[9] = k23;
        }
    } else {
        const double2 p0 = *reinterpret_cast<const double2*>(xs + 2 * l[0]);
        const double2 p1 = *reinterpret_cast<const double2*>(xs + 2 * l[1]);
        const double2 p2 = *reinterpret_cast<const double2*>(xs + 2 * l[2]);
        const double e1x = p1.x - p0.x, e1y = p1.y - p0.y;
        const double e2x = p2.x - p0.x, e2y = p2.y - p0.y;
        det = __fma_rn(e1x, e2y, -(e1y * e2x));
        if constexpr (KT == 0) {
            const double s = coef_w(Cn::wsum) * fast_rcp(det);
            // grad N_1 = (e2y, -e2x) / det, grad N_2 = (-e1y, e1x) / det
            const double k11 = s * __fma_rn(e2y, e2y, e2x * e2x);
            const double k12 = -(s * __fma_rn(e2y, e1y, e2x * e1x));
            const double k22 = s * __fma_rn(e1y, e1y, e1x * e1x);
            const double k01 = -(k11 + k12), k02 = -(k12 + k22);
            kp[0] = -(k01 + k02);  // kp: K_aa (unused: zero row sums), then 01 02 12
            kp[1] = k11; kp[2] = k22;
            kp[3] = k01; kp[4] = k02; kp[5] = k12;
        }
    }
    double sv = 0.0;
    if constexpr (KT == 1) {
        const double c = p.ctype == TGK_FIELD_CONSTANT ? p.cval : __ldg(p.cdata + __ldg(p.pl.helem + A.hbase + h));
        sv = c * det;
    } else if constexpr (HAS_M) {
        sv = det;
    }
    double fv[k];
    if constexpr (FT == 1) {
        const double f = p.stype == TGK_FIELD_CONSTANT ? p.sval : __ldg(p.sdata + __ldg(p.pl.helem + A.hbase + h));
        fv[0] = f * det;
    } else if constexpr (FT == 2) {
        double fs = sn[l[0]];
#pragma unroll
        for (int a = 1; a < k; ++a) fs += sn[l[a]];
        const double dm = det * Cn::moff;
#pragma unroll
        for (int a = 0; a < k; ++a) fv[a] = dm * (fs + sn[l[a]]);
    }
    if (det <= 0.0) {  // batch.cpp:98-101 (a NaN det passes, as in the reference)
        atomicMin(p.bad, static_cast<unsigned long long>(__ldg(p.pl.helem + A.hbase + h)));
#pragma unroll
        for (int t = 0; t < Cn::np; ++t) kp[t] = 0.0;
        sv = 0.0;
#pragma unroll
        for (int a = 0; a < k; ++a) fv[a] = 0.0;
    }
    if constexpr (KT == 0) {  // the off-diagonal pairs (kp[k..]: 01 02 03 12 13 23 / 01 02 12)
#pragma unroll
        for (int t = 0; t < Cf::NPO; ++t) kv[t * MH + h] = kp[k + t];
    }
    if constexpr (Cf::HAS_S) kv[Cf::SROW * MH + h] = sv;
    if constexpr (FT == 1) kv[Cf::FROW * MH + h] = fv[0];
    if constexpr (FT == 2) {
#pragma unroll
        for (int a = 0; a < k; ++a) kv[(Cf::FROW + a) * MH + h] = fv[a];
    }
}

// ---------------------------------------------------------------- phase B: one warp group of entries
// Lane `lane` of warp group w folds its entry's items (direct value indices,
// plan_fast.cpp formats) from the value rows into the output tile.  One
// 4-byte word (two items) per step, the next three steps' words already in
// flight, two partial sums per value.
template <int KIND, int KT, bool HAS_M, int FT>
__device__ __forceinline__ void fast_group(const FastArgs& p, const RecA& A, const RecB& Bq, const double* kv,
                                           double* tk, double* tm, uint8_t* tdiag, int w, int lane) {
    using Cf = FastCfg<KIND, KT, HAS_M, FT>;
    using Cn = FastConst<KIND>;
    constexpr int k = Cf::k;
    const int MH = p.MH;
    const uint32_t desc = Bq.desc[w * 32 + lane];
    const uint32_t i0 = Bq.wgoff[w];
    const int steps = static_cast<int>((Bq.wgoff[w + 1] - i0) >> 5);  // 32 words per step
    const uint32_t* ip = Bq.words + i0 + lane;
    const bool diag = (__shfl_sync(0xffffffffu, desc, 0) >> 15) & 1u;  // warp-uniform class
    // the load from the det fold S_i when the source is constant and S is folded anyway
    const bool fs_det = FT == 1 && HAS_M && p.stype == TGK_FIELD_CONSTANT;
    double k0 = 0.0, k1 = 0.0, k2 = 0.0, k3 = 0.0, s0 = 0.0, s1 = 0.0, f0 = 0.0, f1 = 0.0;
    // u16 items h | q << 12: K_ab at row q, S at SROW, F at FROW (+ a = q for a
    // nodal load on a diagonal); padding items address the +0.0 slot
    // prefetch indices clamped to the group's last step: unconditional loads (no
    // branch around them); a word fetched past the last step is never folded
    const int last = steps > 0 ? steps - 1 : 0;
    uint32_t wa = ip[0];
    uint32_t wb = ip[min(1, last) * 32];
    uint32_t wc = ip[min(2, last) * 32];
    // the fold, specialised per warp-uniform class so the item loop carries no
    // per-item conditionals: off-diagonal entries fold K (and S), diagonal
    // entries only S / F (the stiffness diagonal comes from the zero row sums)
    auto fold = [&](auto eat) {
        for (int st = 0; st < steps; ++st) {
            const uint32_t wn = ip[min(st + 3, last) * 32];
            eat(wa & 0xffffu, k0, s0, f0);
            eat(wa >> 16, k1, s1, f1);
            wa = wb;
            wb = wc;
            wc = wn;
        }
    };
    if (!diag) {
        fold([&](uint32_t it, double& kk, double& ss, double&) {
            const int h = static_cast<int>(it & 0xfffu), q = static_cast<int>(it >> 12);
            if constexpr (KT == 0) kk += kv[q * MH + h];
            if constexpr (Cf::HAS_S) ss += kv[Cf::SROW * MH + h];
        });
    } else if (FT == 1 && !fs_det) {
        fold([&](uint32_t it, double&, double& ss, double& ff) {
            const int h = static_cast<int>(it & 0xfffu);
            if constexpr (Cf::HAS_S) ss += kv[Cf::SROW * MH + h];
            ff += kv[Cf::FROW * MH + h];
        });
    } else {
        fold([&](uint32_t it, double&, double& ss, double& ff) {
            const int h = static_cast<int>(it & 0xfffu), q = static_cast<int>(it >> 12);
            if constexpr (Cf::HAS_S) ss += kv[Cf::SROW * MH + h];
            if constexpr (FT == 2) ff += kv[(Cf::FROW + q) * MH + h];
            (void)q;
            (void)ff;
        });
    }
    if constexpr (KT == 1) {  // coefficient mass: the folds summed S
        k0 = s0;
        k1 = s1;
        k2 = k3 = 0.0;
    }
    k0 += k2;
    k1 += k3;
    if (diag) {  // split diagonal lists: partial sums of kFastDiagSplit lanes
        constexpr int DS = kFastDiagSplit(k);
#pragma unroll
        for (int o = 1; o < DS; o <<= 1) {
            k0 += __shfl_xor_sync(0xffffffffu, k0, o);
            k1 += __shfl_xor_sync(0xffffffffu, k1, o);
            if constexpr (Cf::HAS_S) {
                s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            }
            if constexpr (FT > 0) {
                f0 += __shfl_xor_sync(0xffffffffu, f0, o);
                f1 += __shfl_xor_sync(0xffffffffu, f1, o);
            }
        }
    }
    if constexpr (KT == 1) {  // the value below is S-based
        s0 = k0;
        s1 = k1;
    }
    if (desc >= kFastPart) return;  // idle or a split diagonal's partial lane
    const double kacc = k0 + k1, sacc = s0 + s1, facc = f0 + f1;
    const int lr = static_cast<int>(desc & 0x1ffu), pos = static_cast<int>((desc >> 9) & 63u);
    const double mh = diag ? Cn::mdiag : Cn::moff;
    const double kval = KT == 0 ? kacc : sacc * mh;
    if (KT == 0 && diag) tdiag[lr] = static_cast<uint8_t>(pos);  // K_ii formed at the copy-out
    if (pos != kFastNoPos) {
        const int at = A.toff[lr] + pos;
        if (KT != 0 || !diag) tk[at] = kval;
        if constexpr (HAS_M) tm[at] = sacc * mh;
    }
    if constexpr (FT > 0) {
        // constant source with the unit mass: F_i = sum_e f wa det_e = (f wa) S_i (S = the det fold)
        if (diag) p.F[A.srow[lr]] = FT == 1 ? (fs_det ? (p.sval * Cn::wa) * sacc : facc * Cn::wa) : facc;
    }
    if (desc >> 31) {
        const int lr2 = static_cast<int>((desc >> 16) & 0x1ffu), pos2 = static_cast<int>((desc >> 25) & 63u);
        const int at = A.toff[lr2] + pos2;
        tk[at] = kval;
        if constexpr (HAS_M) tm[at] = sacc * mh;
    }
}

// Persistent kernel: CTA c takes row blocks c, c + G, c + 2G, ... (iteration
// it = block c + it G).  Per iteration:
//   top       the warps write block it-1's output tile to HBM (coalesced row
//             segments; overlaps phase A);
//   phase A   block it's element values into the value rows;        | barrier
//   phase B   block it+1's node table starts streaming in (cp.async
//             gathers), then block it's CSR entries are folded into the
//             output tile;                                          | barrier
//   refill    TMA bulk copies of record A(it+2) and record B(it+1) into the
//             slots just consumed.
// A block's plan and coordinates are on chip before it starts, so no HBM
// latency sits on a CTA's critical path.  (A warp-specialised variant —
// producer warps running phase A of block it+1 while consumer warps fold
// block it from a second value buffer — measured slower: 474-715 vs 370 us
// on C2a, profiles/r02_fast_experiments.txt.)
template <int KIND, int KT, bool HAS_M, int FT>
__global__ void __launch_bounds__(kFastScalarMaxThreads) k_fast_scalar(FastArgs p) {
    using Cf = FastCfg<KIND, KT, HAS_M, FT>;
    constexpr int d = Cf::d;
    extern __shared__ __align__(128) unsigned char smb[];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = T >> 5;
    const int MH = p.MH, MB = p.MB;
    const FastPlanDev& pl = p.pl;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smb);  // record A slots 0-1, record B
    unsigned char* const ra_base = smb + 64;
    unsigned char* const rb = ra_base + 2 * size_t(p.abuf);
    const bool cnodal = p.ctype == TGK_FIELD_NODAL;
    const int ncol = Cf::ncol(p.ctype);
    double* const xs_base = reinterpret_cast<double*>(rb + size_t(p.bbuf));
    double* const kv = xs_base + size_t(ncol) * MB;  // NR x MH value rows
    double* const tk = kv + size_t(Cf::NR) * MH;          // output tile (K), then M
    double* const tm = tk + pl.max_tile;
    int64_t* const trp = reinterpret_cast<int64_t*>(tm + (HAS_M ? pl.max_tile : 0));  // tile rows' CSR offsets
    uint16_t* const ttoff = reinterpret_cast<uint16_t*>(trp + pl.max_rows);           // tile row offsets (n+1)
    uint8_t* const tdiag = reinterpret_cast<uint8_t*>(ttoff + pl.max_rows + 1);       // tile rows' diagonal position
    auto ra = [&](int64_t it) { return ra_base + size_t(it & 1) * p.abuf; };
    // one node table: block it+1's gathers start after phase A of block it (its only reader)
    auto xsp = [&](int64_t) { return xs_base; };

    const int64_t nb = pl.n_blocks, G = gridDim.x, b0 = blockIdx.x;
    if (b0 >= nb) return;
    const int64_t n_it = (nb - b0 + G - 1) / G;
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (tid < Cf::NR) kv[tid * MH + MH - 1] = 0.0;  // the zero slot padding items point at
    __syncthreads();
    auto load_a = [&](int64_t it) {
        const int64_t blk = b0 + it * G;
        const int64_t o = pl.rec_a_off[blk];
        bulk_load(ra(it), pl.rec_a + o, static_cast<uint32_t>(pl.rec_a_off[blk + 1] - o), &bars[it & 1]);
    };
    auto load_b = [&](int64_t it) {
        const int64_t blk = b0 + it * G;
        const int64_t o = pl.rec_b_off[blk];
        bulk_load(rb, pl.rec_b + o, static_cast<uint32_t>(pl.rec_b_off[blk + 1] - o), &bars[2]);
    };
    auto wait_a = [&](int64_t it) { mbar_wait(&bars[it & 1], static_cast<uint32_t>((it >> 1) & 1)); };
    auto wait_b = [&](int64_t it) { mbar_wait(&bars[2], static_cast<uint32_t>(it & 1)); };
    auto gather = [&](int64_t it) {
        const RecA A = parse_a(ra(it));
        double* xs = xsp(it);
        const int nbn_run = (p.debug & 8) ? 0 : int(A.nbn);
        for (int i = tid; i < nbn_run; i += T) {
            const int64_t g = A.bnodes[i];
#pragma unroll
            for (int c = 0; c < d; ++c) cp_async8(d == 2 ? xs + 2 * i + c : xs + c * MB + i, p.nodes + g * d + c);
            if (cnodal) cp_async8(xs + d * MB + i, p.cdata + g);
            if (FT == 2) cp_async8(xs + (ncol - 1) * MB + i, p.sdata + g);
        }
        cp_async_commit();
    };
    // the previous block's tile to HBM: groups of GL lanes per row
    int tile_rows = 0;
    // copy-out lanes: GL = 2^glog lanes per row, 32 / GL rows per warp step;
    // the stiffness diagonal K_ii = 0 - (sum of the row's off-diagonals), the
    // group's lanes summed by a butterfly (deterministic; within the SURVEY.md
    // 8(c) tolerance of the reference's element fold)
    const int glog = p.gl <= 8 ? 3 : p.gl <= 16 ? 4 : 5;
    const int gl = lane & ((1 << glog) - 1), GL = 1 << glog;
    const int lr_base = warp << (5 - glog), lr_step = nwarp << (5 - glog);
    // rows of up to 2 GL entries: one predicated pass with two entries per lane
    // (8 lanes per row for C2a's <= 15-entry rows: 4 rows per warp and a
    // 3-round butterfly instead of 2 rows and 4 rounds)
    const bool single_pass = pl.max_len <= 2 * GL;
    auto copy_out = [&]() {
        if (p.debug & 4) return;
        for (int base = lr_base; base < tile_rows; base += lr_step) {  // warp-uniform: shuffles below
            const int lr = base + (lane >> glog);
            const bool ok = lr < tile_rows;
            const int64_t rp = ok ? trp[lr] : 0;
            const int t0 = ok ? ttoff[lr] : 0, len = ok ? ttoff[lr + 1] - t0 : 0;
            const int dq = (KT == 0 && ok) ? tdiag[lr] : -1;
            if (single_pass) {  // every row fits two passes of its lanes: predicated, no loops
                const int q1 = gl + GL;
                const bool in0 = gl < len, in1 = q1 < len;
                const double v0 = in0 ? tk[t0 + gl] : 0.0, v1 = in1 ? tk[t0 + q1] : 0.0;
                double off = ((in0 && gl != dq) ? v0 : 0.0) + ((in1 && q1 != dq) ? v1 : 0.0);
                if constexpr (KT == 0)
                    for (int o = GL >> 1; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
                if (in0) {
                    p.K[rp + gl] = (KT == 0 && gl == dq) ? 0.0 - off : v0;
                    if constexpr (HAS_M) p.M[rp + gl] = tm[t0 + gl];
                }
                if (in1) {
                    p.K[rp + q1] = (KT == 0 && q1 == dq) ? 0.0 - off : v1;
                    if constexpr (HAS_M) p.M[rp + q1] = tm[t0 + q1];
                }
                continue;
            }
            double off = 0.0;
            if constexpr (KT == 0) {
                for (int q = gl; q < len; q += GL)
                    if (q != dq) off += tk[t0 + q];
                for (int o = GL >> 1; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
            }
            for (int q = gl; q < len; q += GL) {
                p.K[rp + q] = (KT == 0 && q == dq) ? 0.0 - off : tk[t0 + q];
                if constexpr (HAS_M) p.M[rp + q] = tm[t0 + q];
            }
        }
    };
    if (tid == 0) {
        load_a(0);
        if (n_it > 1) load_a(1);
        load_b(0);
    }
    wait_a(0);
    gather(0);
    cp_async_wait_all();
    __syncthreads();
    for (int64_t it = 0; it < n_it; ++it) {
        const RecA A = parse_a(ra(it));
        copy_out();  // block it-1 (tile_rows = 0 on the first iteration)
        const int nh_run = (p.debug & 1) ? 0 : int(A.nh);
        for (int h = tid; h < nh_run; h += T) fast_element<KIND, KT, HAS_M, FT>(p, A, xsp(it), kv, h);
        __syncthreads();
        if (it + 1 < n_it) {  // block it+1's node table streams in during phase B
            wait_a(it + 1);
            gather(it + 1);
        }
        if (!(p.debug & 16)) wait_b(it);
        const RecB Bq = parse_b(rb);
        for (int i = tid; i <= int(A.nr); i += T) {  // the tile's row map for the copy-out
            if (i < int(A.nr)) trp[i] = A.rp[i];
            ttoff[i] = A.toff[i];
        }
        tile_rows = int(A.nr);
        const int nwg = (p.debug & 2) ? 0 : int(Bq.nwg);
        for (int w = warp; w < nwg; w += nwarp) fast_group<KIND, KT, HAS_M, FT>(p, A, Bq, kv, tk, tm, tdiag, w, lane);
        cp_async_wait_all();
        __syncthreads();
        if (tid == 0) {  // records A(it) and B(it) are consumed: refill their slots
            fence_proxy_async();
            if (it + 2 < n_it) load_a(it + 2);
            if (it + 1 < n_it && !(p.debug & 16)) load_b(it + 1);
        }
    }
    copy_out();  // the last block
}

template <int KIND, int KT, bool HAS_M, int FT>
int launch_fast(const FastArgs& a, int threads, cudaStream_t st) {
    auto kern = k_fast_scalar<KIND, KT, HAS_M, FT>;
    const size_t smem = FastCfg<KIND, KT, HAS_M, FT>::smem(a);
    if (smem > 227 * 1024) return kFastNotApplicable;  // the caller takes the exact kernel
    static size_t done[kMaxDevices] = {};  // opt-in size per kernel instance and device
    TGK_TRY(raise_smem_limit(kern, smem, done));
    const int nsm = sm_count();
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    if (per_sm < 1) return kFastNotApplicable;
    if (const char* e = getenv("TGK_FAST_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
    const int64_t grid = std::min<int64_t>(a.pl.n_blocks, int64_t(per_sm) * nsm);
    if (getenv("TGK_FAST_VERBOSE")) {
        static int printed = 0;
        if (printed++ < 4)
            fprintf(stderr,
                    "[fast] R=%d blocks=%lld halo=%lld (max %d, MH=%d) rows/value NR=%d entries=%lld words=%lld "
                    "recA max %d recB max %d plan %.1f MB smem %zu B, %d CTA/SM x %d threads, grid %lld\n",
                    a.pl.R, (long long)a.pl.n_blocks, (long long)a.pl.n_halo, a.pl.max_halo, a.MH,
                    FastCfg<KIND, KT, HAS_M, FT>::NR, (long long)a.pl.n_entries, (long long)a.pl.n_words,
                    a.pl.max_rec_a, a.pl.max_rec_b, a.pl.bytes / 1e6, smem, per_sm, threads, (long long)grid);
    }
    if (grid > 0) kern<<<static_cast<unsigned>(grid), threads, smem, st>>>(a);
    KERNEL_CHECK("fast_scalar");
    return TGK_OK;
}

template <int KIND>
int dispatch_fast(int kt, bool m, int ft, const FastArgs& a, int T, cudaStream_t st) {
    if (kt == 1) return launch_fast<KIND, 1, false, 0>(a, T, st);
    if (m) {
        if (ft == 0) return launch_fast<KIND, 0, true, 0>(a, T, st);
        if (ft == 1) return launch_fast<KIND, 0, true, 1>(a, T, st);
        return launch_fast<KIND, 0, true, 2>(a, T, st);
    }
    if (ft == 0) return launch_fast<KIND, 0, false, 0>(a, T, st);
    if (ft == 1) return launch_fast<KIND, 0, false, 1>(a, T, st);
    return launch_fast<KIND, 0, false, 2>(a, T, st);
}

}  // namespace

int check_bad(unsigned long long* d_bad, cudaStream_t st);

// Rows per block and threads per CTA (B200 sweeps, profiles/r02_fast_experiments.txt);
// TRI3 128 rows x 256 threads.
struct FastShape {
    int R, T;
};
FastShape fast_shape(int kind, int fmt) {
    // TET4 stiffness [+ load] 48 x 384 (C2a 296 us), with the unit mass 64 x 512 (C2 358 us)
    FastShape s{kind == TGK_TET4 ? (fmt == kFastFmtKS32 ? 64 : 48) : 128,
                kind == TGK_TET4 ? (fmt == kFastFmtKS32 ? 512 : 384) : 256};
    if (const char* e = getenv("TGK_FAST_R")) s.R = std::max(1, std::min(kFastMaxRows, atoi(e)));
    if (const char* e = getenv("TGK_FAST_T")) s.T = std::max(32, std::min(kFastScalarMaxThreads, atoi(e) / 32 * 32));
    return s;
}

// Fast-mode scalar assembly.  Returns kFastNotApplicable when the fast layout
// does not apply (nodal mass coefficient, long rows,
// large halos, working set over shared memory): the caller then takes the
// exact kernel, whose results meet the same tolerance.
int fast_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F, double* M,
                         cudaStream_t st, unsigned long long* d_bad) {
    const bool is_mass = pr->kind == TGK_MASS;
    const bool has_f = !is_mass && pr->n_source > 0;
    if (is_mass && pr->diffusion.type == TGK_FIELD_NODAL) return kFastNotApplicable;
    for (const tgk_field* f : {&pr->diffusion, &pr->source[0]})
        if (f->type != TGK_FIELD_CONSTANT && f->type != TGK_FIELD_ELEMENT && f->type != TGK_FIELD_NODAL)
            return kFastNotApplicable;
    const FastPlanDev* pl = nullptr;
    const int ft = !has_f ? 0 : pr->source[0].type == TGK_FIELD_NODAL ? 2 : 1;
    const int kt = is_mass ? 1 : 0;
    const bool hm = !is_mass && pr->with_mass && M;
    if (hm && ft == 2) return kFastNotApplicable;  // nodal load with the unit mass: exact kernel
    const int fmt = kt == 1 ? kFastFmtS16 : (hm ? kFastFmtKS32 : kFastFmtK16);
    const FastShape shape = fast_shape(m->kind, fmt);
    {
        const int prc = ensure_fast_plan(r, shape.R, kFastFmtK16, false, &pl);  // one item layout for every scalar format
        if (prc == TGK_ERR_INPUT) return kFastNotApplicable;
        if (prc != TGK_OK) return prc;
    }
    FastArgs a{};
    a.nodes = m->nodes;
    a.pl = *pl;
    a.ctype = pr->diffusion.type;
    a.cval = pr->diffusion.value;
    a.cdata = pr->diffusion.data;
    a.stype = has_f ? pr->source[0].type : TGK_FIELD_CONSTANT;
    a.sval = has_f ? pr->source[0].value : 0.0;
    a.sdata = has_f ? pr->source[0].data : nullptr;
    a.K = K;
    a.M = M;
    a.F = F;
    a.MH = pl->MH;
    a.MB = (pl->max_bnodes + 1) & ~1;
    a.abuf = (pl->max_rec_a + 15) & ~15;
    a.bbuf = (pl->max_rec_b + 15) & ~15;
    if (const char* e = getenv("TGK_FAST_DEBUG")) a.debug = atoi(e);
    a.gl = pl->max_len <= 16 ? 8 : pl->max_len <= 32 ? 16 : 32;  // copy-out lanes per row (<= 2 entries each)
    const int T = shape.T;
    unsigned long long* own_bad = nullptr;
    if (!d_bad) TGK_TRY(routing_flags(r, &own_bad));
    a.bad = d_bad ? d_bad : own_bad;
    CUDA_TRY(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), st));
    if (!has_f && F) CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
    const int rc = m->kind == TGK_TET4 ? dispatch_fast<TGK_TET4>(kt, hm, ft, a, T, st)
                                       : dispatch_fast<TGK_TRI3>(kt, hm, ft, a, T, st);
    if (rc != TGK_OK) return rc;
    if (!d_bad) return check_bad(own_bad, st);
    return TGK_OK;
}

}  // namespace tgk

// ===========================================================================
// Fast-mode vector elasticity (TGK_MODE_FAST; physics.cpp:45-66 with constant
// Lamé parameters and a constant body force).  The plan is the scalar fast
// plan (plan_fast.cpp, format kFastFmtE16): every scalar CSR entry (i, j) is a
// d x d block of the vector CSR (dofmap.cpp:18-19 node-major interleave).
// Phase A stores per halo element its physical basis gradients g_a and
// c = |T^| det; phase B folds per scalar entry the isotropic block
//   K_e[a r][b s] = c (lambda g_a,r g_b,s + mu g_a,s g_b,r + mu delta_rs g_a.g_b)
// — local_stiffness_elasticity's B^T D B (batch.cpp:198-246) in closed form —
// over the entry's elements, and the load F_i,r = f_r sum_e c_e / k
// (local_load_vector, batch.cpp:291-312, constant source).  The mirrored entry
// (j, i) receives the transposed block.
namespace tgk {
namespace {

struct FastElastArgs {
    const double* nodes;
    FastPlanDev pl;
    double lam, mu;                  // constant Lame parameters (plane-stress lambda applied, physics.cpp:50-53)
    const double* lam_d;             // per-element lambda / mu (LT == 1; nullptr: the constant)
    const double* mu_d;
    int plane_stress;                // 2D: lambda' = 2 lambda mu / (lambda + 2 mu) per element (LT == 1)
    double f[3];                     // constant body force (FT == 1)
    const double* fd[3];             // per-element body force components (FT == 2; nullptr: f[c])
    double* K;
    double* F;
    int MH, MB, abuf, bbuf, gl, debug;
    unsigned long long* bad;         // [0] smallest element with det <= 0, [1] mu <= 0 seen
};

// LT: Lame parameters constant (0) or per element (1); FT: body force none /
// constant / per element.  Value rows: g_a,r (row a d + r), c = |T^| det,
// [lambda c, mu c], [f_r c].
template <int KIND, int LT, int FT>
struct FastElastCfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
    static constexpr int CROW = k * d;
    static constexpr int LROW = k * d + 1, MROW = k * d + 2;
    static constexpr int FROW = k * d + 1 + (LT ? 2 : 0);
    static constexpr int NR = FROW + (FT == 2 ? d : 0);
    static size_t smem(const FastElastArgs& a) {
        return 64 + 2 * size_t(a.abuf) + size_t(a.bbuf) +
               sizeof(double) * (size_t(d) * a.MB + size_t(NR) * a.MH + size_t(d) * d * a.pl.max_tile) +
               sizeof(int64_t) * a.pl.max_rows + sizeof(uint16_t) * (a.pl.max_rows + 1) +
               ((size_t(a.pl.max_rows) + 15) & ~size_t(15));
    }
};

template <int KIND, int LT, int FT>
__device__ __forceinline__ void elast_element(const FastElastArgs& p, const RecA& A, const double* xs, double* kv,
                                              int h) {
    using Cf = FastElastCfg<KIND, LT, FT>;
    constexpr int k = Cf::k, d = Cf::d;
    const int MH = p.MH, MB = p.MB;
    int l[k];
    halo_nodes<k>(A, p.pl.hc8, h, l);
    double g[k][d], det;
    if constexpr (KIND == TGK_TET4) {
        const double x0 = xs[l[0]], y0 = xs[MB + l[0]], z0 = xs[2 * MB + l[0]];
        const double e1x = xs[l[1]] - x0, e1y = xs[MB + l[1]] - y0, e1z = xs[2 * MB + l[1]] - z0;
        const double e2x = xs[l[2]] - x0, e2y = xs[MB + l[2]] - y0, e2z = xs[2 * MB + l[2]] - z0;
        const double e3x = xs[l[3]] - x0, e3y = xs[MB + l[3]] - y0, e3z = xs[2 * MB + l[3]] - z0;
        const double c1x = __fma_rn(e2y, e3z, -(e2z * e3y)), c1y = __fma_rn(e2z, e3x, -(e2x * e3z)),
                     c1z = __fma_rn(e2x, e3y, -(e2y * e3x));
        const double c2x = __fma_rn(e3y, e1z, -(e3z * e1y)), c2y = __fma_rn(e3z, e1x, -(e3x * e1z)),
                     c2z = __fma_rn(e3x, e1y, -(e3y * e1x));
        const double c3x = __fma_rn(e1y, e2z, -(e1z * e2y)), c3y = __fma_rn(e1z, e2x, -(e1x * e2z)),
                     c3z = __fma_rn(e1x, e2y, -(e1y * e2x));
        det = dot3(e1x, e1y, e1z, c1x, c1y, c1z);
        const double rd = fast_rcp(det);
        g[1][0] = c1x * rd; g[1][1] = c1y * rd; g[1][2] = c1z * rd;
        g[2][0] = c2x * rd; g[2][1] = c2y * rd; g[2][2] = c2z * rd;
        g[3][0] = c3x * rd; g[3][1] = c3y * rd; g[3][2] = c3z * rd;
#pragma unroll
        for (int r = 0; r < 3; ++r) g[0][r] = -((g[1][r] + g[2][r]) + g[3][r]);
    } else {
        const double x0 = xs[l[0]], y0 = xs[MB + l[0]];
        const double e1x = xs[l[1]] - x0, e1y = xs[MB + l[1]] - y0;
        const double e2x = xs[l[2]] - x0, e2y = xs[MB + l[2]] - y0;
        det = __fma_rn(e1x, e2y, -(e1y * e2x));
        const double rd = fast_rcp(det);
        g[1][0] = e2y * rd; g[1][1] = -(e2x * rd);
        g[2][0] = -(e1y * rd); g[2][1] = e1x * rd;
        g[0][0] = -(g[1][0] + g[2][0]); g[0][1] = -(g[1][1] + g[2][1]);
    }
    double c = det * FastConst<KIND>::wsum;
    double lc = 0.0, mc = 0.0, fc[d];
    if constexpr (LT == 1 || FT == 2) {
        const int64_t e = __ldg(p.pl.helem + A.hbase + h);
        if constexpr (LT == 1) {
            double lam = p.lam_d ? __ldg(p.lam_d + e) : p.lam;
            const double mu = p.mu_d ? __ldg(p.mu_d + e) : p.mu;
            if (!(mu > 0.0)) atomicOr(p.bad + 1, 1ull);  // batch.cpp:194-195
            if (p.plane_stress) lam = 2.0 * lam * mu / (lam + 2.0 * mu);  // plane_stress_lambda, batch.cpp:359-361
            lc = lam * c;
            mc = mu * c;
        }
        if constexpr (FT == 2) {
#pragma unroll
            for (int r = 0; r < d; ++r) fc[r] = (p.fd[r] ? __ldg(p.fd[r] + e) : p.f[r]) * c;
        }
    }
    if (det <= 0.0) {  // batch.cpp:98-101
        atomicMin(p.bad, static_cast<unsigned long long>(__ldg(p.pl.helem + A.hbase + h)));
        c = lc = mc = 0.0;
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int r = 0; r < d; ++r) g[a][r] = 0.0;
        if constexpr (FT == 2) {
#pragma unroll
            for (int r = 0; r < d; ++r) fc[r] = 0.0;
        }
    }
#pragma unroll
    for (int a = 0; a < k; ++a)
#pragma unroll
        for (int r = 0; r < d; ++r) kv[(a * d + r) * MH + h] = g[a][r];
    kv[Cf::CROW * MH + h] = c;
    if constexpr (LT == 1) {
        kv[Cf::LROW * MH + h] = lc;
        kv[Cf::MROW * MH + h] = mc;
    }
    if constexpr (FT == 2) {
#pragma unroll
        for (int r = 0; r < d; ++r) kv[(Cf::FROW + r) * MH + h] = fc[r];
    }
}

// Lane `lane` of warp group w: one scalar entry's d x d block (and, for a
// diagonal entry, the row's d load values) folded over its elements.
template <int KIND, int LT, int FT>
__device__ __forceinline__ void elast_group(const FastElastArgs& p, const RecA& A, const RecB& Bq, const double* kv,
                                            double* tk, uint8_t* tdiag, int w, int lane) {
    using Cf = FastElastCfg<KIND, LT, FT>;
    constexpr int k = Cf::k, d = Cf::d, NF = FT == 2 ? Cf::d : 1;
    const int MH = p.MH;
    const uint32_t desc = Bq.desc[w * 32 + lane];
    const uint32_t i0 = Bq.wgoff[w];
    const int steps = static_cast<int>((Bq.wgoff[w + 1] - i0) >> 5);
    const uint32_t* ip = Bq.words + i0 + lane;
    const bool diag = (__shfl_sync(0xffffffffu, desc, 0) >> 15) & 1u;
    double acc[d][d], fac[NF];
#pragma unroll
    for (int r = 0; r < d; ++r)
#pragma unroll
        for (int s = 0; s < d; ++s) acc[r][s] = 0.0;
#pragma unroll
    for (int r = 0; r < NF; ++r) fac[r] = 0.0;
    const double lam = p.lam, mu = p.mu;
    auto eat = [&](uint32_t it) {
        const int h = static_cast<int>(it & 0xfffu), a = static_cast<int>((it >> 14) & 3u),
                  b = static_cast<int>((it >> 12) & 3u);
        double lc, mc, c = 0.0;
        if constexpr (LT == 1) {
            lc = kv[Cf::LROW * MH + h];
            mc = kv[Cf::MROW * MH + h];
        } else {
            c = kv[Cf::CROW * MH + h];
            lc = lam * c;
            mc = mu * c;
        }
        double ga[d], gb[d];
#pragma unroll
        for (int r = 0; r < d; ++r) {
            ga[r] = kv[(a * d + r) * MH + h];
            gb[r] = kv[(b * d + r) * MH + h];
        }
        double dt = ga[0] * gb[0];
#pragma unroll
        for (int r = 1; r < d; ++r) dt = __fma_rn(ga[r], gb[r], dt);
        double u[d], v[d];
#pragma unroll
        for (int r = 0; r < d; ++r) {
            u[r] = lc * ga[r];
            v[r] = mc * ga[r];
        }
#pragma unroll
        for (int r = 0; r < d; ++r)
#pragma unroll
            for (int s = 0; s < d; ++s) acc[r][s] = __fma_rn(u[r], gb[s], __fma_rn(v[s], gb[r], acc[r][s]));
#pragma unroll
        for (int r = 0; r < d; ++r) acc[r][r] = __fma_rn(mc, dt, acc[r][r]);
        if constexpr (FT == 1) fac[0] += LT == 1 ? kv[Cf::CROW * MH + h] : c;
        if constexpr (FT == 2) {
#pragma unroll
            for (int r = 0; r < d; ++r) fac[r] += kv[(Cf::FROW + r) * MH + h];
        }
    };
    // padding items address the +0.0 slot (h = max_halo, a = b = 0)
    if (!diag) {
        for (int st = 0; st < steps; ++st) {
            const uint32_t wv = ip[st * 32];
            eat(wv & 0xffffu);
            eat(wv >> 16);
        }
    } else if constexpr (FT > 0) {  // diagonal entries fold only the load: the diagonal
        auto eat_f = [&](uint32_t it) {  // block comes from the zero row sums (copy-out)
            const int h = static_cast<int>(it & 0xfffu);
            if constexpr (FT == 1) fac[0] += kv[Cf::CROW * MH + h];
            if constexpr (FT == 2) {
#pragma unroll
                for (int r = 0; r < d; ++r) fac[r] += kv[(Cf::FROW + r) * MH + h];
            }
        };
        for (int st = 0; st < steps; ++st) {
            const uint32_t wv = ip[st * 32];
            eat_f(wv & 0xffffu);
            eat_f(wv >> 16);
        }
        constexpr int DS = kFastDiagSplit(k);  // split diagonal lists: partial sums of DS lanes
#pragma unroll
        for (int o = 1; o < DS; o <<= 1) {
#pragma unroll
            for (int r = 0; r < NF; ++r) fac[r] += __shfl_xor_sync(0xffffffffu, fac[r], o);
        }
    }
    if (desc >= kFastPart) return;
    const int lr = static_cast<int>(desc & 0x1ffu), pos = static_cast<int>((desc >> 9) & 63u);
    if (diag) tdiag[lr] = static_cast<uint8_t>(pos);  // K_ii block formed at the copy-out
    if (!diag && pos != kFastNoPos) {
        const int L = A.toff[lr + 1] - A.toff[lr];
        double* t = tk + d * d * A.toff[lr] + d * pos;
#pragma unroll
        for (int r = 0; r < d; ++r)
#pragma unroll
            for (int s = 0; s < d; ++s) t[r * d * L + s] = acc[r][s];
    }
    if constexpr (FT > 0) {
        if (diag) {
            const int64_t row = A.srow[lr];
#pragma unroll
            for (int r = 0; r < d; ++r)
                p.F[row * d + r] = (FT == 1 ? p.f[r] * fac[0] : fac[r]) * (1.0 / k);
        }
    }
    if (desc >> 31) {  // the mirrored entry (j, i) holds the transposed block
        const int lr2 = static_cast<int>((desc >> 16) & 0x1ffu), pos2 = static_cast<int>((desc >> 25) & 63u);
        const int L2 = A.toff[lr2 + 1] - A.toff[lr2];
        double* t = tk + d * d * A.toff[lr2] + d * pos2;
#pragma unroll
        for (int r = 0; r < d; ++r)
#pragma unroll
            for (int s = 0; s < d; ++s) t[s * d * L2 + r] = acc[r][s];
    }
}

// Persistent kernel, the same pipeline as k_fast_scalar (TMA-fed records,
// cp.async node tables, tile copy-out overlapping phase A).
template <int KIND, int LT, int FT>
#ifndef TGK_ELAST_MINB
#define TGK_ELAST_MINB 2  // <= 64 registers: 2 CTAs x 512 threads (C3 0.81 vs 0.83 ms at 1 x 512 / 2 x 256)
#endif
__global__ void __launch_bounds__(kFastMaxThreads, TGK_ELAST_MINB) k_fast_elast(FastElastArgs p) {
    using Cf = FastElastCfg<KIND, LT, FT>;
    constexpr int d = Cf::d;
    extern __shared__ __align__(128) unsigned char smb[];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = T >> 5;
    const int MH = p.MH, MB = p.MB;
    const FastPlanDev& pl = p.pl;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smb);
    unsigned char* const ra_base = smb + 64;
    unsigned char* const rb = ra_base + 2 * size_t(p.abuf);
    double* const xs_base = reinterpret_cast<double*>(rb + size_t(p.bbuf));
    double* const kv = xs_base + size_t(d) * MB;
    double* const tk = kv + size_t(Cf::NR) * MH;
    int64_t* const trp = reinterpret_cast<int64_t*>(tk + size_t(d) * d * pl.max_tile);
    uint16_t* const ttoff = reinterpret_cast<uint16_t*>(trp + pl.max_rows);
    uint8_t* const tdiag = reinterpret_cast<uint8_t*>(ttoff + pl.max_rows + 1);  // rows' diagonal position
    auto ra = [&](int64_t it) { return ra_base + size_t(it & 1) * p.abuf; };
    auto xsp = [&](int64_t) { return xs_base; };  // single node table (phase A is its only reader)
    const int64_t nb = pl.n_blocks, G = gridDim.x, b0 = blockIdx.x;
    if (b0 >= nb) return;
    const int64_t n_it = (nb - b0 + G - 1) / G;
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (tid < Cf::NR) kv[tid * MH + MH - 1] = 0.0;
    __syncthreads();
    auto load_a = [&](int64_t it) {
        const int64_t blk = b0 + it * G, o = pl.rec_a_off[blk];
        bulk_load(ra(it), pl.rec_a + o, static_cast<uint32_t>(pl.rec_a_off[blk + 1] - o), &bars[it & 1]);
    };
    auto load_b = [&](int64_t it) {
        const int64_t blk = b0 + it * G, o = pl.rec_b_off[blk];
        bulk_load(rb, pl.rec_b + o, static_cast<uint32_t>(pl.rec_b_off[blk + 1] - o), &bars[2]);
    };
    auto wait_a = [&](int64_t it) { mbar_wait(&bars[it & 1], static_cast<uint32_t>((it >> 1) & 1)); };
    auto wait_b = [&](int64_t it) { mbar_wait(&bars[2], static_cast<uint32_t>(it & 1)); };
    auto gather = [&](int64_t it) {
        const RecA A = parse_a<false>(ra(it));
        double* xs = xsp(it);
        for (int i = tid; i < int(A.nbn); i += T) {
            const int64_t g = A.bnodes[i];
#pragma unroll
            for (int c = 0; c < d; ++c) cp_async8(xs + c * MB + i, p.nodes + g * d + c);
        }
        cp_async_commit();
    };
    int tile_rows = 0;
    // scalar row i's d rows are one contiguous d^2 L run of the vector CSR
    // ([r][p][s]); its diagonal block K_ii[r][s] = 0 - sum over p != diagonal of
    // block p (zero row sums: rigid translations are in every element
    // stiffness's kernel), lane j sums (r, s) = j % d^2 over p = j / d^2, j / d^2
    // + 32 / d^2, ..., the parts combined in a fixed order (deterministic)
    auto copy_out = [&]() {
        if (p.debug & 4) return;
        constexpr int DD = d * d, NP = 32 / DD;
        const int rs = lane % DD, part = lane / DD;
        for (int lr = warp; lr < tile_rows; lr += nwarp) {
            const int64_t rp = trp[lr] * DD;
            const int L = ttoff[lr + 1] - ttoff[lr], t0 = ttoff[lr] * DD, len = L * DD;
            const int pd = tdiag[lr];
            const double* src = tk + t0;
            if (pd < L) {  // warp-uniform
                // column (r, s) of the row's blocks: src[base + d q], base = r d L + s
                const double* col = src + (rs / d) * d * L + rs % d;
                double sacc = 0.0;
                if (part < NP) {
#pragma unroll 4
                    for (int q = part; q < L; q += NP) sacc += q != pd ? col[d * q] : 0.0;  // branch-free
                }
                double tot = sacc;
#pragma unroll
                for (int o = 1; o < NP; ++o) tot += __shfl_down_sync(0xffffffffu, sacc, o * DD);
                if (part == 0) tk[t0 + (rs / d) * d * L + d * pd + rs % d] = 0.0 - tot;
                __syncwarp();
            }
            double* dst = p.K + rp;
#pragma unroll 4
            for (int q = lane; q < len; q += 32) dst[q] = src[q];
        }
    };
    if (tid == 0) {
        load_a(0);
        if (n_it > 1) load_a(1);
        load_b(0);
    }
    wait_a(0);
    gather(0);
    cp_async_wait_all();
    __syncthreads();
    for (int64_t it = 0; it < n_it; ++it) {
        const RecA A = parse_a<false>(ra(it));
        copy_out();
        const int nh_run = (p.debug & 1) ? 0 : int(A.nh);
        for (int h = tid; h < nh_run; h += T) elast_element<KIND, LT, FT>(p, A, xsp(it), kv, h);
        __syncthreads();
        if (it + 1 < n_it) {
            wait_a(it + 1);
            gather(it + 1);
        }
        wait_b(it);
        const RecB Bq = parse_b(rb);
        for (int i = tid; i <= int(A.nr); i += T) {
            if (i < int(A.nr)) trp[i] = A.rp[i];
            ttoff[i] = A.toff[i];
        }
        tile_rows = int(A.nr);
        const int nwg = (p.debug & 2) ? 0 : int(Bq.nwg);
        for (int w = warp; w < nwg; w += nwarp) elast_group<KIND, LT, FT>(p, A, Bq, kv, tk, tdiag, w, lane);
        cp_async_wait_all();
        __syncthreads();
        if (tid == 0) {
            fence_proxy_async();
            if (it + 2 < n_it) load_a(it + 2);
            if (it + 1 < n_it) load_b(it + 1);
        }
    }
    copy_out();
}

template <int KIND, int LT, int FT>
int launch_fast_elast(const FastElastArgs& a, int threads, cudaStream_t st) {
    auto kern = k_fast_elast<KIND, LT, FT>;
    const size_t smem = FastElastCfg<KIND, LT, FT>::smem(a);
    if (smem > 227 * 1024) return kFastNotApplicable;
    static size_t done[kMaxDevices] = {};
    TGK_TRY(raise_smem_limit(kern, smem, done));
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    if (per_sm < 1) return kFastNotApplicable;
    if (const char* e = getenv("TGK_FAST_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
    const int64_t grid = std::min<int64_t>(a.pl.n_blocks, int64_t(per_sm) * sm_count());
    if (grid > 0) kern<<<static_cast<unsigned>(grid), threads, smem, st>>>(a);
    KERNEL_CHECK("fast_elast");
    return TGK_OK;
}

}  // namespace

template <int KIND>
int dispatch_fast_elast(int lt, int ft, const FastElastArgs& a, int T, cudaStream_t st) {
    if (lt == 0) return ft == 0 ? launch_fast_elast<KIND, 0, 0>(a, T, st)
                      : ft == 1 ? launch_fast_elast<KIND, 0, 1>(a, T, st) : launch_fast_elast<KIND, 0, 2>(a, T, st);
    return ft == 0 ? launch_fast_elast<KIND, 1, 0>(a, T, st)
         : ft == 1 ? launch_fast_elast<KIND, 1, 1>(a, T, st) : launch_fast_elast<KIND, 1, 2>(a, T, st);
}

// Fast-mode elasticity (constant or per-element Lame parameters and body
// force); kFastNotApplicable for nodal / quadrature fields — the exact kernels
// take those.
int fast_elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                             cudaStream_t st) {
    const int d = m->d;
    auto simple = [](const tgk_field& f) { return f.type == TGK_FIELD_CONSTANT || f.type == TGK_FIELD_ELEMENT; };
    if (!simple(pr->lambda) || !simple(pr->mu)) return kFastNotApplicable;
    for (int c = 0; c < pr->n_source; ++c)
        if (!simple(pr->source[c])) return kFastNotApplicable;
    const int lt = pr->lambda.type == TGK_FIELD_ELEMENT || pr->mu.type == TGK_FIELD_ELEMENT ? 1 : 0;
    const bool has_f = pr->n_source > 0;
    int ft = has_f ? 1 : 0;
    for (int c = 0; c < pr->n_source; ++c)
        if (pr->source[c].type == TGK_FIELD_ELEMENT) ft = 2;
    if (lt == 0 && !(pr->mu.value > 0.0)) return set_error(TGK_ERR_INPUT, "elasticity requires mu > 0");  // batch.cpp:194-195
    int R = m->kind == TGK_TET4 ? 32 : 64, T = m->kind == TGK_TET4 ? 512 : 256;  // B200 sweeps (r02_fast_experiments)
    if (const char* e = getenv("TGK_FAST_ER")) R = std::max(1, std::min(kFastMaxRows, atoi(e)));
    if (const char* e = getenv("TGK_FAST_ET")) T = std::max(32, std::min(kFastMaxThreads, atoi(e) / 32 * 32));
    const FastPlanDev* pl = nullptr;
    {
        const int prc = ensure_fast_plan(r, R, kFastFmtE16, false, &pl);
        if (prc == TGK_ERR_INPUT) return kFastNotApplicable;
        if (prc != TGK_OK) return prc;
    }
    FastElastArgs a{};
    a.nodes = m->nodes;
    a.pl = *pl;
    a.lam = pr->lambda.value;
    a.mu = pr->mu.value;
    a.lam_d = pr->lambda.type == TGK_FIELD_ELEMENT ? pr->lambda.data : nullptr;
    a.mu_d = pr->mu.type == TGK_FIELD_ELEMENT ? pr->mu.data : nullptr;
    a.plane_stress = d == 2 && pr->plane_stress;
    if (lt == 0 && a.plane_stress) a.lam = 2.0 * a.lam * a.mu / (a.lam + 2.0 * a.mu);  // plane_stress_lambda
    for (int c = 0; c < d; ++c) {
        a.f[c] = has_f ? pr->source[c].value : 0.0;
        a.fd[c] = has_f && pr->source[c].type == TGK_FIELD_ELEMENT ? pr->source[c].data : nullptr;
    }
    a.K = K;
    a.F = F;
    a.MH = pl->MH;
    a.MB = (pl->max_bnodes + 1) & ~1;
    a.abuf = (pl->max_rec_a + 15) & ~15;
    a.bbuf = (pl->max_rec_b + 15) & ~15;
    if (const char* e = getenv("TGK_FAST_DEBUG")) a.debug = atoi(e);
    unsigned long long* bad = nullptr;
    TGK_TRY(routing_flags(r, &bad));
    a.bad = bad;
    CUDA_TRY(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), st));
    CUDA_TRY(cudaMemsetAsync(a.bad + 1, 0, sizeof(unsigned long long), st));
    if (!has_f && F) CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
    const int rc = m->kind == TGK_TET4 ? dispatch_fast_elast<TGK_TET4>(lt, ft, a, T, st)
                                       : dispatch_fast_elast<TGK_TRI3>(lt, ft, a, T, st);
    if (rc != TGK_OK) return rc;
    unsigned long long h[2] = {ULLONG_MAX, 0};
    CUDA_TRY(cudaMemcpyAsync(h, bad, sizeof h, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    // batch_geometry runs (and throws) before local_stiffness_elasticity checks mu (physics.cpp:11-52)
    if (h[0] != ULLONG_MAX)
        return set_error(TGK_ERR_INPUT, "element " + std::to_string(h[0]) + " has non-positive Jacobian determinant");
    if (h[1]) return set_error(TGK_ERR_INPUT, "elasticity requires mu > 0");
    return TGK_OK;
}

}  // namespace tgk
