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
//             reciprocal, the k(k+1)/2 unique K_e values via the gradient
//             Gram matrix (row a = 0 from the zero row sum of P1 stiffness),
//             and the scalars the mass / load are formed from (det, f det)
//             into structure-of-arrays value rows;
//   phase B   one lane per owned CSR entry (diagonal entries also fold the
//             row's load): its items (u16 = halo index | value index << 12,
//             one coalesced 8-byte load per 4 items) are summed in registers
//             and the result stored to the entry — and to its mirror (j, i)
//             when j is owned by the same block.
// Mass and load values are affine P1 closed forms of the reference's
// quadrature (batch.cpp:250-289): M_e = c det Mhat, F_e[a] = f det |T^|/k;
// with a nodal source F_e[a] = det sum_b Mhat[a][b] f_b.
#include <cstdio>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

namespace {

constexpr int kFastMaxThreads = 512;

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
template <int KIND, int KT, bool HAS_M, int FT>
struct FastCfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
    static constexpr bool HAS_S = HAS_M || KT == 1;
    static constexpr int NP = KT == 0 ? FastConst<KIND>::np : 0;
    static constexpr int SROW = NP;
    static constexpr int FROW = NP + (HAS_S ? 1 : 0);
    static constexpr int NR = FROW + (FT == 1 ? 1 : FT == 2 ? k : 0);
    static constexpr int NTILE = HAS_M ? 2 : 1;
    __host__ __device__ static int ncol(int ctype) { return d + (ctype == TGK_FIELD_NODAL ? 1 : 0) + (FT == 2 ? 1 : 0); }
    static size_t smem(const FastArgs& a) {
        return 64 + 2 * size_t(a.abuf) + size_t(a.bbuf) + sizeof(double) * (2 * size_t(ncol(a.ctype)) * a.MB +
                                                                             size_t(NR) * a.MH + size_t(NTILE) * a.pl.max_tile);
    }
};

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
    const uint64_t* hconn;
};
__device__ __forceinline__ RecA parse_a(const unsigned char* r) {
    RecA a;
    a.hbase = *reinterpret_cast<const int64_t*>(r);
    const uint2 h0 = *reinterpret_cast<const uint2*>(r + 8), h1 = *reinterpret_cast<const uint2*>(r + 16);
    a.nr = h0.x;
    a.nh = h0.y;
    a.nbn = h1.x;
    a.tile = h1.y;
    size_t o = 32;
    a.rp = reinterpret_cast<const int64_t*>(r + o);
    o += al16(8 * size_t(a.nr));
    a.srow = reinterpret_cast<const uint32_t*>(r + o);
    o += al16(4 * size_t(a.nr));
    a.toff = reinterpret_cast<const uint16_t*>(r + o);
    o += al16(2 * size_t(a.nr + 1));
    a.bnodes = reinterpret_cast<const uint32_t*>(r + o);
    o += al16(4 * size_t(a.nbn));
    a.hconn = reinterpret_cast<const uint64_t*>(r + o);
    return a;
}
struct RecB {
    uint32_t ne, nwg;
    const uint32_t* desc;
    const uint32_t* wgoff;
    const uint16_t* items;
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
    b.items = reinterpret_cast<const uint16_t*>(r + o);
    return b;
}

// Persistent kernel: CTA c takes row blocks c, c + G, c + 2G, ...  While
// block b is computed, record A of block b+G (TMA) and then its node table
// (cp.async gathers) and record B (TMA) stream into the spare buffers, so a
// block's plan and coordinates are on chip before it starts.
template <int KIND, int KT, bool HAS_M, int FT>
__global__ void __launch_bounds__(kFastMaxThreads) k_fast_scalar(FastArgs p) {
    using Cf = FastCfg<KIND, KT, HAS_M, FT>;
    using Cn = FastConst<KIND>;
    constexpr int k = Cf::k, d = Cf::d;
    extern __shared__ __align__(128) unsigned char smb[];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = T >> 5;
    const int MH = p.MH, MB = p.MB;
    const FastPlanDev& pl = p.pl;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smb);  // record A slot 0 / 1, record B
    unsigned char* const ra0 = smb + 64;
    unsigned char* const ra1 = smb + 64 + p.abuf;
    unsigned char* rb = smb + 64 + 2 * p.abuf;
    const bool cnodal = p.ctype == TGK_FIELD_NODAL;
    const int ncol = Cf::ncol(p.ctype);
    double* const xs0 = reinterpret_cast<double*>(rb + p.bbuf);
    double* const xs1 = xs0 + size_t(ncol) * MB;
    double* kv = xs1 + size_t(ncol) * MB;  // NR x MH value rows
    double* tk = kv + size_t(Cf::NR) * MH;    // output tile (K), then M
    double* tm = tk + pl.max_tile;

    const int64_t nb = pl.n_blocks, G = gridDim.x;
    int64_t b = blockIdx.x;
    if (b >= nb) return;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
    }
    if (tid < Cf::NR) kv[tid * MH + MH - 1] = 0.0;  // the zero slot padding items point at
    __syncthreads();
    auto load_a = [&](int64_t blk, int slot) {
        const int64_t o = pl.rec_a_off[blk];
        bulk_load(slot ? ra1 : ra0, pl.rec_a + o, static_cast<uint32_t>(pl.rec_a_off[blk + 1] - o), &bars[slot]);
    };
    auto load_b = [&](int64_t blk) {
        const int64_t o = pl.rec_b_off[blk];
        bulk_load(rb, pl.rec_b + o, static_cast<uint32_t>(pl.rec_b_off[blk + 1] - o), &bars[2]);
    };
    auto gather = [&](const RecA& A, double* xs) {
        for (int i = tid; i < int(A.nbn); i += T) {
            const int64_t g = A.bnodes[i];
#pragma unroll
            for (int c = 0; c < d; ++c) cp_async8(xs + c * MB + i, p.nodes + g * d + c);
            if (cnodal) cp_async8(xs + d * MB + i, p.cdata + g);
            if (FT == 2) cp_async8(xs + (ncol - 1) * MB + i, p.sdata + g);
        }
        cp_async_commit();
    };
    if (tid == 0) {
        load_a(b, 0);
        load_b(b);
    }
    mbar_wait(&bars[0], 0);
    uint32_t phs = 0b01u, phb = 0;  // bit s: parity record-A slot s completes with next
    gather(parse_a(ra0), xs0);
    cp_async_wait_all();
    __syncthreads();
    int slot = 0;
    for (;;) {
        const int64_t bn = b + G;
        const RecA A = parse_a(slot ? ra1 : ra0);
        const double* xs = slot ? xs1 : xs0;
        const double* cn = xs + d * MB;
        const double* sn = xs + (ncol - 1) * MB;
        if (tid == 0 && bn < nb) {
            fence_proxy_async();
            load_a(bn, slot ^ 1);
        }
        // ---------------- phase A: element values
        for (int h = tid; h < int(A.nh); h += T) {
            const uint64_t hc = A.hconn[h];
            int l[k];
#pragma unroll
            for (int a = 0; a < k; ++a) l[a] = static_cast<int>((hc >> (16 * a)) & 0xffff);
            double det;
            double kp[Cn::np];
            auto coef_w = [&](double wsum_) -> double {
                if (p.ctype == TGK_FIELD_CONSTANT) return p.cval * wsum_;
                if (p.ctype == TGK_FIELD_ELEMENT) return __ldg(p.cdata + __ldg(pl.helem + A.hbase + h)) * wsum_;
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
                    const double s = coef_w(Cn::wsum) * __drcp_rn(det);
                    const double k11 = s * dot3(c1x, c1y, c1z, c1x, c1y, c1z);
                    const double k12 = s * dot3(c1x, c1y, c1z, c2x, c2y, c2z);
                    const double k13 = s * dot3(c1x, c1y, c1z, c3x, c3y, c3z);
                    const double k22 = s * dot3(c2x, c2y, c2z, c2x, c2y, c2z);
                    const double k23 = s * dot3(c2x, c2y, c2z, c3x, c3y, c3z);
                    const double k33 = s * dot3(c3x, c3y, c3z, c3x, c3y, c3z);
                    // row a = 0 from the zero row sums of P1 stiffness (grad N_0 = -sum_b grad N_b)
                    const double k01 = -((k11 + k12) + k13), k02 = -((k12 + k22) + k23), k03 = -((k13 + k23) + k33);
                    kp[0] = -((k01 + k02) + k03);
                    kp[1] = k01; kp[2] = k02; kp[3] = k03;
                    kp[4] = k11; kp[5] = k12; kp[6] = k13;
                    kp[7] = k22; kp[8] = k23; kp[9] = k33;
                }
            } else {
                const double x0 = xs[l[0]], y0 = xs[MB + l[0]];
                const double e1x = xs[l[1]] - x0, e1y = xs[MB + l[1]] - y0;
                const double e2x = xs[l[2]] - x0, e2y = xs[MB + l[2]] - y0;
                det = __fma_rn(e1x, e2y, -(e1y * e2x));
                if constexpr (KT == 0) {
                    const double s = coef_w(Cn::wsum) * __drcp_rn(det);
                    // grad N_1 = (e2y, -e2x) / det, grad N_2 = (-e1y, e1x) / det
                    const double k11 = s * __fma_rn(e2y, e2y, e2x * e2x);
                    const double k12 = -(s * __fma_rn(e2y, e1y, e2x * e1x));
                    const double k22 = s * __fma_rn(e1y, e1y, e1x * e1x);
                    const double k01 = -(k11 + k12), k02 = -(k12 + k22);
                    kp[0] = -(k01 + k02);
                    kp[1] = k01; kp[2] = k02;
                    kp[3] = k11; kp[4] = k12; kp[5] = k22;
                }
            }
            double sv = 0.0;
            if constexpr (KT == 1) {
                const double c =
                    p.ctype == TGK_FIELD_CONSTANT ? p.cval : __ldg(p.cdata + __ldg(pl.helem + A.hbase + h));
                sv = c * det;
            } else if constexpr (HAS_M) {
                sv = det;
            }
            double fv[k];
            if constexpr (FT == 1) {
                const double f =
                    p.stype == TGK_FIELD_CONSTANT ? p.sval : __ldg(p.sdata + __ldg(pl.helem + A.hbase + h));
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
                atomicMin(p.bad, static_cast<unsigned long long>(__ldg(pl.helem + A.hbase + h)));
#pragma unroll
                for (int t = 0; t < Cn::np; ++t) kp[t] = 0.0;
                sv = 0.0;
#pragma unroll
                for (int a = 0; a < k; ++a) fv[a] = 0.0;
            }
            if constexpr (KT == 0) {
#pragma unroll
                for (int t = 0; t < Cn::np; ++t) kv[t * MH + h] = kp[t];
            }
            if constexpr (Cf::HAS_S) kv[Cf::SROW * MH + h] = sv;
            if constexpr (FT == 1) kv[Cf::FROW * MH + h] = fv[0];
            if constexpr (FT == 2) {
#pragma unroll
                for (int a = 0; a < k; ++a) kv[(Cf::FROW + a) * MH + h] = fv[a];
            }
        }
        __syncthreads();
        // next block's node table streams in during phase B
        if (bn < nb) {
            mbar_wait(&bars[slot ^ 1], (phs >> (slot ^ 1)) & 1u);
            phs ^= 1u << (slot ^ 1);
            gather(parse_a(slot ? ra0 : ra1), slot ? xs0 : xs1);
        }
        mbar_wait(&bars[2], phb);
        phb ^= 1;
        const RecB Bq = parse_b(rb);
        // ---------------- phase B: one lane per CSR entry, register folds into the output tile
        for (int s = tid; s < int(Bq.ne); s += T) {
            const uint32_t desc = Bq.desc[s];
            const int w = s >> 5;
            const uint32_t i0 = Bq.wgoff[w];
            const int steps = static_cast<int>((Bq.wgoff[w + 1] - i0) >> 7);
            const uint2* ip = reinterpret_cast<const uint2*>(Bq.items + i0) + lane;
            const bool diag = (__shfl_sync(0xffffffffu, desc, 0) >> 15) & 1u;  // warp-uniform class
            double kacc = 0.0, sacc = 0.0, facc = 0.0;
            if (diag) {
                for (int st = 0; st < steps; ++st) {
                    const uint2 wv = ip[st * 32];
                    const uint32_t its[4] = {wv.x & 0xffffu, wv.x >> 16, wv.y & 0xffffu, wv.y >> 16};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int h = static_cast<int>(its[j] & 0xfffu), a = static_cast<int>(its[j] >> 12);
                        if constexpr (KT == 0) kacc += kv[(a * k - ((a * (a - 1)) >> 1)) * MH + h];
                        if constexpr (Cf::HAS_S) sacc += kv[Cf::SROW * MH + h];
                        if constexpr (FT == 1) facc += kv[Cf::FROW * MH + h];
                        if constexpr (FT == 2) facc += kv[(Cf::FROW + a) * MH + h];
                    }
                }
            } else {
                for (int st = 0; st < steps; ++st) {
                    const uint2 wv = ip[st * 32];
                    const uint32_t its[4] = {wv.x & 0xffffu, wv.x >> 16, wv.y & 0xffffu, wv.y >> 16};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int h = static_cast<int>(its[j] & 0xfffu), q = static_cast<int>(its[j] >> 12);
                        if constexpr (KT == 0) kacc += kv[q * MH + h];
                        if constexpr (Cf::HAS_S) sacc += kv[Cf::SROW * MH + h];
                    }
                }
            }
            if (desc == kFastIdle) continue;
            const int lr = static_cast<int>(desc & 0x1ffu), pos = static_cast<int>((desc >> 9) & 63u);
            const double mh = diag ? Cn::mdiag : Cn::moff;
            const double kval = KT == 0 ? kacc : sacc * mh;
            if (pos != kFastNoPos) {
                const int at = A.toff[lr] + pos;
                tk[at] = kval;
                if constexpr (HAS_M) tm[at] = sacc * mh;
            }
            if constexpr (FT > 0) {
                if (diag) p.F[A.srow[lr]] = FT == 1 ? facc * Cn::wa : facc;
            }
            if (desc >> 31) {
                const int lr2 = static_cast<int>((desc >> 16) & 0x1ffu), pos2 = static_cast<int>((desc >> 25) & 63u);
                const int at = A.toff[lr2] + pos2;
                tk[at] = kval;
                if constexpr (HAS_M) tm[at] = sacc * mh;
            }
        }
        __syncthreads();
        if (tid == 0 && bn < nb) {
            fence_proxy_async();
            load_b(bn);
        }
        // ---------------- coalesced copy-out: one warp per owned row
        for (int lr = warp; lr < int(A.nr); lr += nwarp) {
            const int64_t rp = A.rp[lr];
            const int t0 = A.toff[lr], len = A.toff[lr + 1] - t0;
            for (int q = lane; q < len; q += 32) {
                p.K[rp + q] = tk[t0 + q];
                if constexpr (HAS_M) p.M[rp + q] = tm[t0 + q];
            }
        }
        if (bn >= nb) break;
        cp_async_wait_all();
        __syncthreads();
        b = bn;
        slot ^= 1;
    }
}

template <int KIND, int KT, bool HAS_M, int FT>
int launch_fast(const FastArgs& a, int threads, cudaStream_t st) {
    auto kern = k_fast_scalar<KIND, KT, HAS_M, FT>;
    const size_t smem = FastCfg<KIND, KT, HAS_M, FT>::smem(a);
    if (smem > 227 * 1024) return kFastNotApplicable;  // the caller takes the exact kernel
    // opt-in size per kernel instance and device (a process may drive several GPUs)
    static size_t done[64] = {};
    static int sms[64] = {};
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= 64 || done[dev] < smem) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        if (dev < 64) done[dev] = smem;
    }
    int nsm = dev < 64 ? sms[dev] : 0;
    if (nsm == 0) {
        CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        if (dev < 64) sms[dev] = nsm;
    }
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    if (per_sm < 1) return kFastNotApplicable;
    if (const char* e = getenv("TGK_FAST_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
    const int64_t grid = std::min<int64_t>(a.pl.n_blocks, int64_t(per_sm) * nsm);
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

int fast_rows_per_block(int kind) {
    if (const char* e = getenv("TGK_FAST_R")) return std::max(1, std::min(kFastMaxRows, atoi(e)));
    return kind == TGK_TET4 ? 64 : 128;
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
    {
        const int prc = ensure_fast_plan(r, fast_rows_per_block(m->kind), &pl);
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
    a.MH = pl->max_halo + 1;
    a.MB = (pl->max_bnodes + 1) & ~1;
    a.abuf = (pl->max_rec_a + 15) & ~15;
    a.bbuf = (pl->max_rec_b + 15) & ~15;
    int T = 256;
    if (const char* e = getenv("TGK_FAST_T")) T = std::max(32, std::min(kFastMaxThreads, atoi(e) / 32 * 32));
    unsigned long long* own_bad = nullptr;
    if (!d_bad) TGK_TRY(routing_flags(r, &own_bad));
    a.bad = d_bad ? d_bad : own_bad;
    CUDA_TRY(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), st));
    if (!has_f && F) CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(double) * r->N, st));
    const int ft = !has_f ? 0 : a.stype == TGK_FIELD_NODAL ? 2 : 1;
    const int kt = is_mass ? 1 : 0;
    const bool hm = !is_mass && pr->with_mass && M;
    const int rc = m->kind == TGK_TET4 ? dispatch_fast<TGK_TET4>(kt, hm, ft, a, T, st)
                                       : dispatch_fast<TGK_TRI3>(kt, hm, ft, a, T, st);
    if (rc != TGK_OK) return rc;
    if (!d_bad) return check_bad(own_bad, st);
    return TGK_OK;
}

}  // namespace tgk
