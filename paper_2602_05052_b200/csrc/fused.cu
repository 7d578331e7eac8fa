// Fused P1 Map+Reduce assembly (tg::assemble, physics.cpp:10-75) for scalar
// problems: stiffness (or coefficient mass), optional unit mass M and load F,
// straight from mesh + coefficients to CSR values, with no local tensor ever
// written to HBM and no atomics.
//
// Decomposition ("row blocks", see tgk_internal.hpp / plan.cpp): CUDA block b
// owns R CSR rows (mesh nodes, compact in space via a Morton ordering) and
// walks every element incident to them — its halo, ordered by level in the
// per-row ascending-element chains (plan.cpp) — R elements per chunk:
//   prologue  the block's node table (coordinates of every node its halo
//             touches) is gathered once into shared memory;
//   phase A   one thread per halo element: exact geometry and local
//             K_e / M_e / F_e from the node table into shared memory;
//   phase B   one thread per owned row: fold that row's records of the chunk
//             (ascending element) — diagonal and load in registers, the
//             off-diagonal entries in shared-memory accumulators.
// The next chunk's block-local connectivity and records arrive by cp.async
// while the current chunk is computed.  Each CSR value is the left fold, from
// +0.0, of its contributions in ascending element order — the reference
// reduction's order (routing.cpp:117-124) — so with the exact element
// arithmetic of element.cuh the output is bit-identical to the CPU reference.
// Elements on a block boundary are recomputed by every block they touch
// (halo recompute; the plan statistics report the factor).
#include <cstdio>
#include <vector>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

#ifndef TGK_MINB
#define TGK_MINB(R) ((R) == 256 ? 2 : ((R) == 128 ? 4 : 8))
#endif

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);
int mesh_division_safe(tgk_mesh* m, cudaStream_t st, bool* safe);

namespace {

struct FieldDev {
    int type;
    double value;
    const double* data;
};

struct FusedArgs {
    const double* nodes;
    const int64_t* row_ptr;
    const int64_t* row_off;
    const uint32_t* rows;
    const int64_t* rows_rp;
    const int64_t* halo_off;
    const uint32_t* halo;
    const int64_t* bnode_off;
    const uint32_t* bnodes;
    const uint16_t* halo_lconn;
    const int64_t* chunk_off;
    const int64_t* chunk_rec_off;
    const uint16_t* chunk_row_off;
    const uint32_t* recs;
    FieldDev coef;
    FieldDev src;
    void* K;  // T* (double, or float in the fp32 mode)
    void* M;
    void* F;
    int lmax;
    int max_recs;
    int max_bnodes;
    int ntcols;  // doubles per node-table entry: 3 coordinates [+ nodal coefficient] [+ nodal source]
    int max_chunks;  // most halo chunks of one block (dynamic chunk-offset table)
    int debug;  // profiling only (TGK_FUSED_DEBUG): 1 skips phase B, 2 skips phase A math
    long long* trace;  // profiling only (TGK_FUSED_TRACE): per block 8 clock64 stamps
    unsigned long long* bad;
};

constexpr int kMaxChunks = 255;  // halo chunks per block (plan-enforced)
#ifndef TGK_RING
#define TGK_RING 2
#endif
#ifndef TGK_R_BIG
#define TGK_R_BIG 256
#endif
constexpr int kRing = TGK_RING;  // cp.async ring slots: chunk c+kRing-1 is requested while c is computed

// Slot of K_e[a][b] within the rotated shared-memory row a: 0 for the
// diagonal, then the other local nodes in ascending order (see pack_rec).
__host__ __device__ constexpr int rot(int a, int b) { return b == a ? 0 : (b < a ? b + 1 : b); }

// KTYPE 0: diffusion stiffness, 1: coefficient mass (ProblemKind::Mass);
// T: double (exact mode) or float (fp32 mode)
template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int R, typename T = double, bool FCONST = false>
struct FusedCfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    // local tensors in shared memory: rotated rows of 4 values (16-byte aligned).
    // MDET: the unit mass M_e depends on the element only through det, so
    // phase A stores det and phase B forms each record's M row from it with
    // the reference's expression (a smaller block working set: more resident
    // blocks for C2)
    static constexpr bool MDET = HAS_M && KTYPE == 0;
    // FDET: with MDET and a constant source the load F_e[a] is formed from det
    // in the fold as well (same expression as phase A's local_load)
    static constexpr bool FDET = FCONST && KTYPE == 0 && HAS_F;
    static constexpr bool DETSLOT = MDET || FDET;  // det stored at offM
    static constexpr int KIND_ = KIND, DEG_ = DEG;
    static constexpr int offK = 0;
    static constexpr int offM = 4 * k;
    static constexpr int offF = offM + (DETSLOT ? 2 : (HAS_M ? 4 * k : 0));
    static constexpr int raw = offF + (HAS_F && !FDET ? 4 : 0);
    // stride = (16-byte vector) x odd: conflict-free 128-bit accesses across lanes
    static constexpr int VEC = 16 / int(sizeof(T));
    static constexpr int stride = ((raw + VEC - 1) / VEC) % 2 == 1 ? (raw + VEC - 1) / VEC * VEC
                                                                   : (raw + VEC - 1) / VEC * VEC + VEC;
    static constexpr int nmat = 1 + (HAS_M ? 1 : 0);
    // node table: coordinates, d doubles per node (odd 8-byte-word stride for
    // d = 3: random node gathers spread over all bank pairs), then the nodal
    // coefficient and nodal source as separate arrays (used only when nodal)
    static constexpr int NV = 3;      // TRI3 pads to 3 as well (odd stride)
    // doubles per node in the table: the coordinates, then the nodal
    // coefficient / source columns only when those fields are nodal (FusedArgs::ntcols)
    static size_t smem_bytes(int lmax, int max_recs, int max_bnodes, int ntcols, int max_chunks) {
        return sizeof(T) * (size_t(R) * stride + size_t(R) * lmax * nmat + size_t(max_bnodes) * ntcols) +
               kRing * (sizeof(uint32_t) * size_t(max_recs) + sizeof(uint16_t) * size_t(row_off_stride(R)) +
                        sizeof(uint16_t) * 4 * size_t(R)) +
               sizeof(int64_t) * size_t(max_chunks + 1);
    }
};

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

// Four consecutive values of a 16-byte aligned shared-memory row.
__device__ __forceinline__ void load4(const double* src, double (&v)[4]) {
    const double2 a = *reinterpret_cast<const double2*>(src);
    const double2 b = *reinterpret_cast<const double2*>(src + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void load4(const float* src, float (&v)[4]) {
    const float4 a = *reinterpret_cast<const float4*>(src);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}

// Row a of the unit-coefficient local mass from det, rotated like the record
// ([M_aa, M_ab for b != a ascending]): local_mass with ones (physics.cpp:70-71,
// batch.cpp:259-265), M_e[a][b] = sum_q ((w_q det) N_a(q)) N_b(q) in the
// reference's order — identical to phase A's expression (element_values).
// N_a(q) for a runtime local node a (selects, no divergence).
template <int KIND, int DEG, typename T>
__device__ __forceinline__ void basis_row(int a, T (&na)[Rule<KIND, DEG>::Q]) {
    constexpr int k = P1<KIND>::k, Q = Rule<KIND, DEG>::Q;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        T v = T(basis<KIND, DEG>(q, 0));
#pragma unroll
        for (int c = 1; c < k; ++c) v = a == c ? T(basis<KIND, DEG>(q, c)) : v;
        na[q] = v;
    }
}

template <int KIND, int DEG, typename T>
__device__ __forceinline__ void mass_row(T det, int a, T (&mv)[4], T (&na)[Rule<KIND, DEG>::Q]) {
    using Rl = Rule<KIND, DEG>;
    constexpr int k = P1<KIND>::k, Q = Rl::Q;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        T v = T(basis<KIND, DEG>(q, 0));
#pragma unroll
        for (int c = 1; c < k; ++c) v = a == c ? T(basis<KIND, DEG>(q, c)) : v;
        na[q] = v;
    }
#pragma unroll
    for (int j = 0; j < k; ++j) {
        // rotated column: j = 0 is a itself, j >= 1 is local node j-1 (below a) or j
        const bool lower = j - 1 < a;
        T v = T(0);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const T nb = j == 0 ? na[q]
                                : (lower ? T(basis<KIND, DEG>(q, j > 0 ? j - 1 : 0)) : T(basis<KIND, DEG>(q, j < k ? j : 0)));
            const T term = T(Rl::w(q)) * det * na[q] * nb;
            v = q == 0 ? term : v + term;
        }
        mv[j] = v;
    }
}

// One record's rotated local tensor row (K, M) and F_e[a] from shared memory.
template <typename T, bool HAS_M, bool HAS_F>
struct RowVals {
    T kv[4];
    T mv[HAS_M ? 4 : 1];
    T f;
    template <class C>
    __device__ __forceinline__ void load(const T* ke, uint32_t rec, T fval) {
        const int hl = rec & 0xff;
        const int a = (rec >> 8) & 3;
        const T* src = ke + hl * C::stride + a * 4;
        load4(src + C::offK, kv);
        if constexpr (C::DETSLOT) {
            using Rl = Rule<C::KIND_, C::DEG_>;
            const T det = ke[hl * C::stride + C::offM];
            T na[Rl::Q];
            if constexpr (C::MDET) {
                mass_row<C::KIND_, C::DEG_, T>(det, a, mv, na);
            } else {
                basis_row<C::KIND_, C::DEG_, T>(a, na);
            }
            if constexpr (C::FDET) {  // local_load with a constant source (batch.cpp:280-286)
                T v = T(0);
#pragma unroll
                for (int q = 0; q < Rl::Q; ++q) {
                    const T term = (T(Rl::w(q)) * det * fval) * na[q];
                    v = q == 0 ? term : v + term;
                }
                f = v;
            }
        }
        if constexpr (HAS_M && !C::MDET) {
            T m4[4];
            load4(src + C::offM, m4);
#pragma unroll
            for (int i = 0; i < 4; ++i) mv[i] = m4[i];
        }
        if constexpr (HAS_F && !C::FDET) f = ke[hl * C::stride + C::offF + a];
    }
};

// Internal field types of the Allen-Cahn Newton re-assembly (tgk_allen_cahn_d):
// nodal state u interpolated at q, then the reaction tangent coefficient
// -e2 (3 v^2 - 1) (batch.cpp:344-351) or the reaction source -e2 v (v^2 - 1)
// (batch.cpp:335-342), e2 = eps^2 with eps in FieldDev::value.
constexpr int kFieldAcTangent = 100, kFieldAcReaction = 101;
__host__ __device__ inline bool nodal_like(int type) {
    return type == TGK_FIELD_NODAL || type == kFieldAcTangent || type == kFieldAcReaction;
}

// c(x_q) for a constant / per-element / nodal field (coefficient.cpp:34-55,
// interpolate_nodal batch.cpp:321-330)
template <int KIND, int DEG, typename T = double>
__device__ __forceinline__ T field_q(const FieldDev& f, const T* u, int q) {
    constexpr int k = P1<KIND>::k;
    if (nodal_like(f.type)) {
        T v = T(basis<KIND, DEG>(q, 0)) * u[0];
#pragma unroll
        for (int a = 1; a < k; ++a) v += T(basis<KIND, DEG>(q, a)) * u[a];
        if (f.type == kFieldAcTangent) {
            const T e2 = T(f.value) * T(f.value);
            return -e2 * (T(3) * v * v - T(1));
        }
        if (f.type == kFieldAcReaction) {
            const T e2 = T(f.value) * T(f.value);
            return -e2 * v * (v * v - T(1));
        }
        return v;
    }
    return f.type == TGK_FIELD_ELEMENT ? u[0] : T(f.value);
}

// Where phase A puts an element's values: rotated rows per element (v3) or
// structure-of-arrays rows over the chunk (entry kernel).
template <class C, typename T>
struct RotSink {
    T* out;
    __device__ __forceinline__ void Ksym(int a, int b, int, T v) {
        out[C::offK + a * 4 + rot(a, b)] = v;
        out[C::offK + b * 4 + rot(b, a)] = v;
    }
    __device__ __forceinline__ void K(int a, int b, T v) { out[C::offK + a * 4 + rot(a, b)] = v; }
    static constexpr bool kMDet = C::MDET;   // M_e formed from det in the fold: skip it here
    static constexpr bool kDet = C::DETSLOT;  // store det
    __device__ __forceinline__ void M(int a, int b, T v) {
        if constexpr (!C::MDET) out[C::offM + a * 4 + rot(a, b)] = v;
    }
    __device__ __forceinline__ void Det(T v) {
        if constexpr (C::DETSLOT) out[C::offM] = v;
    }
    __device__ __forceinline__ void F(int a, T v) {
        if constexpr (!C::FDET) out[C::offF + a] = v;
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < C::raw; ++i) out[i] = T(0);
    }
};

// Phase A body: the reference's local kernels for one element into `sink`.
// nt: the block's node table; ln: block-local node ids.  NTB: node-table
// capacity (the nodal coefficient / source columns start at NTB * NV).
template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, bool FDIV, typename T, class Sink>
__device__ __forceinline__ void element_values(const FieldDev& coef, const FieldDev& src, const uint32_t* halo,
                                               unsigned long long* bad, int NTB, const T* nt, const ushort4 ln,
                                               int64_t h_global, Sink& sink) {
    using Rl = Rule<KIND, DEG>;
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rl::Q, NV = 3;
    const int ids[4] = {ln.x, ln.y, ln.z, ln.w};
    T X[k][d];
    T cu[k], fu[k];
#pragma unroll
    for (int a = 0; a < k; ++a)
#pragma unroll
        for (int c = 0; c < d; ++c) X[a][c] = nt[ids[a] * NV + c];
    if (nodal_like(coef.type)) {
        const T* cs = nt + NTB * NV;
#pragma unroll
        for (int a = 0; a < k; ++a) cu[a] = cs[ids[a]];
    }
    if (HAS_F && nodal_like(src.type)) {
        const T* ss = nt + NTB * (NV + (nodal_like(coef.type) ? 1 : 0));
#pragma unroll
        for (int a = 0; a < k; ++a) fu[a] = ss[ids[a]];
    }
    if (coef.type == TGK_FIELD_ELEMENT || (HAS_F && src.type == TGK_FIELD_ELEMENT)) {
        const int64_t e = halo[h_global];
        if (coef.type == TGK_FIELD_ELEMENT) cu[0] = T(__ldg(coef.data + e));
        if (HAS_F && src.type == TGK_FIELD_ELEMENT) fu[0] = T(__ldg(src.data + e));
    }
    T det, G[k][d];
    if (!simplex_geometry<KIND, FDIV, T>(X, det, G)) {
        atomicMin(bad, static_cast<unsigned long long>(halo[h_global]));
        sink.zero();
        return;
    }
    T sc[Q];  // w_q * det * c_q  (batch.cpp:169 / :261)
#pragma unroll
    for (int q = 0; q < Q; ++q) sc[q] = T(Rl::w(q)) * det * field_q<KIND, DEG, T>(coef, cu, q);
    if constexpr (KTYPE == 0) {
        // local_stiffness_diffusion (batch.cpp:168-177); K_e symmetric bitwise
        int t = 0;
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int b = a; b < k; ++b) {
                const T dot = gdot<KIND, T>(G, a, b);
                T v = sc[0] * dot;
#pragma unroll
                for (int q = 1; q < Q; ++q) v += sc[q] * dot;
                sink.Ksym(a, b, t++, v);
            }
    } else {
        // local_mass with the coefficient (batch.cpp:259-265)
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int b = 0; b < k; ++b) {
                T v = sc[0] * T(basis<KIND, DEG>(0, a)) * T(basis<KIND, DEG>(0, b));
#pragma unroll
                for (int q = 1; q < Q; ++q) v += sc[q] * T(basis<KIND, DEG>(q, a)) * T(basis<KIND, DEG>(q, b));
                sink.K(a, b, v);
            }
    }
    if constexpr (Sink::kDet) sink.Det(det);
    if constexpr (HAS_M && !Sink::kMDet) {
        // with_mass: local_mass with ones (physics.cpp:70-71); w*det*1.0 == w*det
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int b = 0; b < k; ++b) {
                T v = T(Rl::w(0)) * det * T(basis<KIND, DEG>(0, a)) * T(basis<KIND, DEG>(0, b));
#pragma unroll
                for (int q = 1; q < Q; ++q)
                    v += T(Rl::w(q)) * det * T(basis<KIND, DEG>(q, a)) * T(basis<KIND, DEG>(q, b));
                sink.M(a, b, v);
            }
    }
    if constexpr (HAS_F) {
        // local_load (batch.cpp:280-286)
        T sf[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) sf[q] = T(Rl::w(q)) * det * field_q<KIND, DEG, T>(src, fu, q);
#pragma unroll
        for (int a = 0; a < k; ++a) {
            T v = sf[0] * T(basis<KIND, DEG>(0, a));
#pragma unroll
            for (int q = 1; q < Q; ++q) v += sf[q] * T(basis<KIND, DEG>(q, a));
            sink.F(a, v);
        }
    }
}

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int R, bool FDIV, typename T, bool FCONST = false>
__global__ void __launch_bounds__(R, TGK_MINB(R)) k_fused_scalar(FusedArgs p) {
    using C = FusedCfg<KIND, DEG, KTYPE, HAS_M, HAS_F, R, T, FCONST>;
    constexpr int k = C::k, d = C::d, NV = C::NV;
    constexpr int ROS = R + 8;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* ke = reinterpret_cast<T*>(smem_raw);                          // R x stride
    T* accK = ke + R * C::stride;                                    // lmax x R
    T* accM = accK + R * p.lmax;                                     // (HAS_M)
    T* nt = accK + R * p.lmax * C::nmat;                             // max_bnodes x ntcols
    uint32_t* rec_s = reinterpret_cast<uint32_t*>(nt + p.max_bnodes * p.ntcols);  // kRing x max_recs
    uint16_t* ro_s = reinterpret_cast<uint16_t*>(rec_s + kRing * p.max_recs);  // kRing x ROS
    ushort4* lc_s = reinterpret_cast<ushort4*>(ro_s + kRing * ROS);           // kRing x R
    int64_t* cro_s = reinterpret_cast<int64_t*>(lc_s + kRing * R);           // this block's chunk record offsets

    const int tid = threadIdx.x;
    const int64_t blk = blockIdx.x;
    long long t_start = 0, t_pro = 0, t_a = 0, t_b = 0, t_loop = 0;
    if (p.trace && tid == 0) t_start = clock64();
    const int64_t r0 = p.row_off[blk];
    const int nr = static_cast<int>(p.row_off[blk + 1] - r0);
    const int64_t h0 = p.halo_off[blk];
    const int64_t nh = p.halo_off[blk + 1] - h0;
    const int64_t c0 = p.chunk_off[blk];
    const int nch = static_cast<int>(p.chunk_off[blk + 1] - c0);

    // stage chunk c's block-local connectivity, records and row offsets into
    // ring slot c % kRing; always commits a group (possibly empty) so that the
    // wait below can use a fixed depth
    auto stage = [&](int c) {
        if (c < nch) {
            const int sl = c % kRing;
            const int64_t cg = c0 + c;
            const int64_t rb = cro_s[c];
            const int nrec4 = static_cast<int>((cro_s[c + 1] - rb) >> 2);
            uint32_t* rdst = rec_s + sl * p.max_recs;
            for (int i = tid; i < nrec4; i += R) cp_async16(rdst + 4 * i, p.recs + rb + 4 * i);
            uint16_t* odst = ro_s + sl * ROS;
            const uint16_t* osrc = p.chunk_row_off + cg * ROS;
            for (int i = tid; i < ROS / 8; i += R) cp_async16(odst + 8 * i, osrc + 8 * i);
            const int64_t hb = h0 + int64_t(c) * R;
            const int64_t rem = nh - int64_t(c) * R;
            const int ne = rem < R ? static_cast<int>(rem) : R;
            if (tid < ne) cp_async8(lc_s + sl * R + tid, p.halo_lconn + (hb + tid) * 4);
        }
        cp_async_commit();
    };

    // this thread's owned row: id, CSR offset and length (used by the epilogue)
    int64_t my_row = 0, my_rp = 0;
    int my_len = 0;
    if (tid < nr) {
        my_row = p.rows[r0 + tid];
        const int64_t packed = p.rows_rp[r0 + tid];  // CSR offset | length << 56 (plan.cpp)
        my_rp = packed & ((int64_t(1) << 56) - 1);
        my_len = static_cast<int>(packed >> 56);
    }
    for (int i = tid; i <= nch; i += R) cro_s[i] = p.chunk_rec_off[c0 + i];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kRing - 1; ++c) stage(c);
    // node table: coordinates (+ nodal coefficient / source) of every node of the
    // halo; all index loads first, then all coordinate loads (one round trip each)
    {
        const int64_t n0 = p.bnode_off[blk];
        const int nbn = static_cast<int>(p.bnode_off[blk + 1] - n0);
        constexpr int NPT = 4;  // nodes per thread per batch
        for (int base = 0; base < nbn; base += NPT * R) {
            int64_t g[NPT];
#pragma unroll
            for (int u = 0; u < NPT; ++u) {
                const int i = base + u * R + tid;
                g[u] = i < nbn ? static_cast<int64_t>(p.bnodes[n0 + i]) : -1;
            }
#pragma unroll
            for (int u = 0; u < NPT; ++u) {
                const int i = base + u * R + tid;
                if (g[u] < 0) continue;
                T* dst = nt + i * NV;
#pragma unroll
                for (int c = 0; c < d; ++c) dst[c] = T(__ldg(p.nodes + g[u] * d + c));
                if (nodal_like(p.coef.type)) nt[p.max_bnodes * NV + i] = T(__ldg(p.coef.data + g[u]));
                if constexpr (HAS_F)
                    if (nodal_like(p.src.type))
                        nt[p.max_bnodes * (NV + (nodal_like(p.coef.type) ? 1 : 0)) + i] = T(__ldg(p.src.data + g[u]));
            }
        }
    }
    for (int i = tid; i < R * p.lmax * C::nmat; i += R) accK[i] = T(0);
    T dK = T(0), dM = T(0), dF = T(0);  // diagonal K, M and the load F of the owned row
    int diag_pos = 0;

    long long t_mark = 0;
    for (int c = 0; c < nch; ++c) {
        cp_async_wait<kRing - 2>();  // chunk c landed (later chunks may be in flight)
        __syncthreads();  // chunk c visible; node table ready; phase B(c-1) done
        if (p.trace && tid == 0) {
            const long long t = clock64();
            if (c == 0) t_pro = t - t_start; else t_b += t - t_mark;
            t_mark = t;
        }
        stage(c + kRing - 1);  // into the slot phase B(c-1) just released
        // ---------------- phase A: this thread's element of chunk c
        const int64_t h = int64_t(c) * R + tid;
        if (h < nh) {
            T* out = ke + tid * C::stride;
            if (p.debug & 2) {
                for (int i = 0; i < C::raw; ++i) out[i] = nt[0];
            } else {
                RotSink<C, T> sink{out};
                element_values<KIND, DEG, KTYPE, HAS_M, HAS_F, FDIV, T>(p.coef, p.src, p.halo, p.bad, p.max_bnodes, nt,
                                                                       lc_s[(c % kRing) * R + tid], h0 + h, sink);
            }
        }
        __syncthreads();
        if (p.trace && tid == 0) {
            const long long t = clock64();
            t_a += t - t_mark;
            t_mark = t;
        }
        // ---------------- phase B: owned row tid folds its records of chunk c.
        // The diagonal entry (the element's node that IS this row) and F live in
        // registers; the off-diagonal entries are shared-memory read-modify-writes.
        // The next record and its local tensor row are loaded before the
        // current record's stores.
        if (tid < nr && !(p.debug & 1)) {
            const uint16_t* ro = ro_s + (c % kRing) * ROS;
            const uint32_t* rs = rec_s + (c % kRing) * p.max_recs;
            int j = ro[tid];
            const int j1 = ro[tid + 1];
            if (j < j1) {
                uint32_t rec = rs[j];
                RowVals<T, HAS_M, HAS_F> v;
                v.template load<C>(ke, rec, T(p.src.value));
                for (; j < j1; ++j) {
                    const uint32_t rec_n = j + 1 < j1 ? rs[j + 1] : rec;
                    RowVals<T, HAS_M, HAS_F> vn;
                    vn.template load<C>(ke, rec_n, T(p.src.value));
                    // the k-1 positions of one record are distinct columns: load all,
                    // add, store all (no false read-after-write serialisation)
                    int pos[k - 1];
                    T ak[k - 1], am[k - 1];
#pragma unroll
                    for (int j2 = 0; j2 < k - 1; ++j2) {
                        pos[j2] = ((rec >> (10 + 5 * j2)) & 31) * R + tid;
                        ak[j2] = accK[pos[j2]];
                        if constexpr (HAS_M) am[j2] = accM[pos[j2]];
                    }
#pragma unroll
                    for (int j2 = 0; j2 < k - 1; ++j2) {
                        accK[pos[j2]] = ak[j2] + v.kv[j2 + 1];
                        if constexpr (HAS_M) accM[pos[j2]] = am[j2] + v.mv[j2 + 1];
                    }
                    dK += v.kv[0];
                    if constexpr (HAS_M) dM += v.mv[0];
                    if constexpr (HAS_F) dF += v.f;
                    diag_pos = (rec >> 25) & 31;
                    rec = rec_n;
                    v = vn;
                }
            }
        }
    }
    __syncthreads();
    if (p.trace && tid == 0) {
        const long long t = clock64();
        t_b += t - t_mark;
        t_loop = t;
    }
    // ---------------- epilogue: owned rows -> CSR values, one store per position
    // (lane = row: conflict-free shared-memory reads; L2 merges the row runs)
    if (tid < nr) {
        accK[diag_pos * R + tid] = dK;
        if constexpr (HAS_M) accM[diag_pos * R + tid] = dM;
        T* Ko = static_cast<T*>(p.K);
        T* Mo = static_cast<T*>(p.M);
        for (int q = 0; q < my_len; ++q) {
            Ko[my_rp + q] = accK[q * R + tid];
            if constexpr (HAS_M) Mo[my_rp + q] = accM[q * R + tid];
        }
    }
    if (HAS_F && tid < nr) static_cast<T*>(p.F)[my_row] = dF;
    if (p.trace && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long* tr = p.trace + blk * 8;
        tr[0] = t_start; tr[1] = t_pro; tr[2] = t_a; tr[3] = t_b; tr[4] = clock64() - t_loop;
        tr[5] = smid; tr[6] = nch; tr[7] = clock64();
    }
}

template <int KIND, int DEG, int KTYPE, bool HAS_M, bool HAS_F, int R, bool FDIV, typename T, bool FCONST = false>
int launch_fused(const FusedArgs& a, int64_t n_blocks, cudaStream_t st) {
    using C = FusedCfg<KIND, DEG, KTYPE, HAS_M, HAS_F, R, T, FCONST>;
    auto kern = k_fused_scalar<KIND, DEG, KTYPE, HAS_M, HAS_F, R, FDIV, T, FCONST>;
    const size_t smem = C::smem_bytes(a.lmax, a.max_recs, a.max_bnodes, a.ntcols, a.max_chunks);
    // raise the instance's dynamic shared-memory limit only when it grows, per
    // device (small meshes are launch-overhead bound)
    static size_t smem_set[kMaxDevices] = {};
    TGK_TRY(raise_smem_limit(kern, smem, smem_set));
    if (n_blocks > 0) kern<<<static_cast<unsigned>(n_blocks), R, smem, st>>>(a);
    KERNEL_CHECK("fused_scalar");
    return TGK_OK;
}

template <int KIND, int DEG, int R, bool FDIV, typename T>
int dispatch_r(int ktype, bool m, bool f, const FusedArgs& a, int64_t nb, cudaStream_t st) {
    if (ktype == 1) return f ? launch_fused<KIND, DEG, 1, false, true, R, FDIV, T>(a, nb, st)
                             : launch_fused<KIND, DEG, 1, false, false, R, FDIV, T>(a, nb, st);
    if (m && f)
        return a.src.type == TGK_FIELD_CONSTANT ? launch_fused<KIND, DEG, 0, true, true, R, FDIV, T, true>(a, nb, st)
                                                : launch_fused<KIND, DEG, 0, true, true, R, FDIV, T>(a, nb, st);
    if (m) return launch_fused<KIND, DEG, 0, true, false, R, FDIV, T>(a, nb, st);
    if (f)
        return a.src.type == TGK_FIELD_CONSTANT ? launch_fused<KIND, DEG, 0, false, true, R, FDIV, T, true>(a, nb, st)
                                                : launch_fused<KIND, DEG, 0, false, true, R, FDIV, T>(a, nb, st);
    return launch_fused<KIND, DEG, 0, false, false, R, FDIV, T>(a, nb, st);
}

// Rows per block R, value type (fp64 / fp32) and FDIV (Markstein division on
// meshes certified division-safe, fp64 only) select the kernel instance.
template <int KIND, int DEG>
int dispatch_flags(int ktype, bool m, bool f, const FusedArgs& a, int64_t nb, int R, bool fdiv, bool f32,
                   cudaStream_t st) {
    if (f32) {
        if (R == 64) return dispatch_r<KIND, DEG, 64, false, float>(ktype, m, f, a, nb, st);
        return dispatch_r<KIND, DEG, 128, false, float>(ktype, m, f, a, nb, st);
    }
    if (R == 128)
        return fdiv ? dispatch_r<KIND, DEG, 128, true, double>(ktype, m, f, a, nb, st)
                    : dispatch_r<KIND, DEG, 128, false, double>(ktype, m, f, a, nb, st);
    if (R == 64)
        return fdiv ? dispatch_r<KIND, DEG, 64, true, double>(ktype, m, f, a, nb, st)
                    : dispatch_r<KIND, DEG, 64, false, double>(ktype, m, f, a, nb, st);
    return fdiv ? dispatch_r<KIND, DEG, TGK_R_BIG, true, double>(ktype, m, f, a, nb, st)
                : dispatch_r<KIND, DEG, TGK_R_BIG, false, double>(ktype, m, f, a, nb, st);
}

}  // namespace

int fused_rows_per_block(const tgk_problem* pr, int64_t n_rows) {
    if (const char* env = getenv("TGK_FUSED_R")) {
        const int r = atoi(env);
        return r == 64 || r == 128 ? r : TGK_R_BIG;
    }
    // measured on B200 (profiles/r01_fused_experiments.txt): 128 rows per block
    // for K+F, 64 for K+M+F (C2: 797 vs 850 us with the mass and load formed
    // from det in the fold), and 64 when 128-row blocks would not fill the GPU
    // once (C1: 16.0 -> 13.4 us)
    if (pr->with_mass) return 64;
    const int sms = sm_count();
    return n_rows < int64_t(128) * 4 * sms ? 64 : 128;
}

// Fused scalar assembly core: ktype 0 (diffusion stiffness) / 1 (coefficient
// mass), quadrature degree, optional unit mass M and load F.
static int fused_core(const tgk_mesh* m, tgk_routing* r, int R, int ktype, int degree, bool has_m, bool has_f,
                      FieldDev coef, FieldDev src, void* K, void* F, void* M, cudaStream_t st,
                      unsigned long long* d_bad, bool f32 = false) {
    if (f32 && R != 64) R = 128;  // the fp32 instances exist for 64 and 128 rows per block
    const PlanDev* pl = nullptr;
    TGK_TRY(ensure_plan(r, R, &pl));
    FusedArgs a{};
    a.nodes = m->nodes;
    a.row_ptr = r->row_ptr;
    a.row_off = pl->row_off;
    a.rows = pl->rows;
    a.rows_rp = pl->rows_rp;
    a.halo_off = pl->halo_off;
    a.halo = pl->halo;
    a.bnode_off = pl->bnode_off;
    a.bnodes = pl->bnodes;
    a.halo_lconn = pl->halo_lconn;
    a.chunk_off = pl->chunk_off;
    a.chunk_rec_off = pl->chunk_rec_off;
    a.chunk_row_off = pl->chunk_row_off;
    a.recs = pl->recs;
    a.coef = coef;
    a.src = has_f ? src : FieldDev{TGK_FIELD_CONSTANT, 0.0, nullptr};
    a.K = K;
    a.M = M;
    a.F = F;
    a.lmax = pl->lmax;
    a.max_recs = pl->max_chunk_recs > 0 ? pl->max_chunk_recs : 4;
    a.max_bnodes = (pl->max_bnodes + 3) & ~3;  // node table ends 16-byte aligned for fp32 and fp64
    a.max_chunks = pl->max_block_chunks;
    a.ntcols = 3 + (nodal_like(a.coef.type) ? 1 : 0) + (has_f && nodal_like(a.src.type) ? 1 : 0);
    if (const char* dbg = getenv("TGK_FUSED_DEBUG")) a.debug = atoi(dbg);
    DevBuf<long long> trace;
    const char* trace_path = getenv("TGK_FUSED_TRACE");
    if (trace_path) {
        TGK_TRY(trace.alloc(pl->n_blocks * 8));
        a.trace = trace.p;
    }
    unsigned long long* own_bad = nullptr;
    if (!d_bad) TGK_TRY(routing_flags(r, &own_bad));
    a.bad = d_bad ? d_bad : own_bad;
    CUDA_TRY(cudaMemsetAsync(a.bad, 0xff, sizeof(unsigned long long), st));
    if (!has_f && F) CUDA_TRY(cudaMemsetAsync(F, 0, (f32 ? sizeof(float) : sizeof(double)) * r->N, st));
    bool fdiv = false;
    TGK_TRY(mesh_division_safe(const_cast<tgk_mesh*>(m), st, &fdiv));
    if (getenv("TGK_IEEE_DIV")) fdiv = false;
    if (m->kind == TGK_TET4) {
        if (degree == 1) TGK_TRY((dispatch_flags<TGK_TET4, 1>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, f32, st)));
        else TGK_TRY((dispatch_flags<TGK_TET4, 2>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, f32, st)));
    } else {
        if (degree == 1) TGK_TRY((dispatch_flags<TGK_TRI3, 1>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, f32, st)));
        else TGK_TRY((dispatch_flags<TGK_TRI3, 2>(ktype, has_m, has_f, a, pl->n_blocks, R, fdiv, f32, st)));
    }
    if (trace_path) {
        std::vector<long long> h(pl->n_blocks * 8);
        CUDA_TRY(cudaMemcpyAsync(h.data(), trace.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (FILE* f = fopen(trace_path, "wb")) {
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
    }
    if (!d_bad) return check_bad(own_bad, st);
    return TGK_OK;  // asynchronous: the caller inspects *d_bad
}

// Scalar fused assembly on device buffers.  With d_bad == nullptr it checks
// the bad-element flag (synchronising); otherwise it is fully asynchronous.
int materialised_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                                 double* M, cudaStream_t st, unsigned long long* d_bad);

int fused_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K,
                          double* F, double* M, cudaStream_t st, unsigned long long* d_bad) {
    const bool is_mass = pr->kind == TGK_MASS;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT || is_mass || pr->with_mass;
    const int degree = high ? 2 : 1;  // default_mass_degree / default_stiffness_degree for P1
    const bool has_f = !is_mass && pr->n_source > 0;
    const FieldDev coef{pr->diffusion.type, pr->diffusion.value, pr->diffusion.data};
    const FieldDev src = has_f ? FieldDev{pr->source[0].type, pr->source[0].value, pr->source[0].data}
                               : FieldDev{TGK_FIELD_CONSTANT, 0.0, nullptr};
    const int64_t n_rows = r->own_hi < 0 ? r->N : r->own_hi - r->own_lo;
    const int R = fused_rows_per_block(pr, n_rows);
    {
        // the row-block plan's layout limits (rows of <= 32 entries, <= 255 halo
        // chunks and <= 65535 nodes per block): any other mesh takes the
        // materialised Stage I + II path, bit-identical as well
        const PlanDev* pl = nullptr;
        const int prc = r->lmax > kMaxRowLen ? TGK_ERR_INPUT : ensure_plan(r, R, &pl);
        if (prc == TGK_ERR_INPUT) return materialised_scalar_assemble(pr, m, r, K, F, M, st, d_bad);
        if (prc != TGK_OK) return prc;
    }
    return fused_core(m, r, R, is_mass ? 1 : 0, degree, pr->with_mass != 0, has_f, coef, src, K, F, M, st, d_bad);
}

// fp32 mode (tgk_assemble_f32_d): the same fused kernel in single precision,
// fp32 CSR values; held to |dv| <= 1e-5 |v_ref| + 1e-7 max|v_ref| against the
// fp64 reference.
int fused_scalar_assemble_f32(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, float* K, float* F,
                              float* M, cudaStream_t st, unsigned long long* d_bad) {
    const bool is_mass = pr->kind == TGK_MASS;
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT || is_mass || pr->with_mass;
    const bool has_f = !is_mass && pr->n_source > 0;
    const FieldDev coef{pr->diffusion.type, pr->diffusion.value, pr->diffusion.data};
    const FieldDev src = has_f ? FieldDev{pr->source[0].type, pr->source[0].value, pr->source[0].data}
                               : FieldDev{TGK_FIELD_CONSTANT, 0.0, nullptr};
    const int64_t n_rows = r->own_hi < 0 ? r->N : r->own_hi - r->own_lo;
    return fused_core(m, r, fused_rows_per_block(pr, n_rows), is_mass ? 1 : 0, high ? 2 : 1, pr->with_mass != 0, has_f,
                      coef, src, K, F, M, st, d_bad, true);
}

// Allen-Cahn Newton re-assembly (AllenCahnStepper::step, timestep.cpp:144-178)
// in one fused pass at the mass degree: T = reduce_matrix(local_mass(
// reaction_tangent_coefficient(u))) and F = reduce_vector(local_reaction_load(u)).
int fused_allen_cahn(const tgk_mesh* m, tgk_routing* r, const double* u, double eps, double* T, double* F,
                     cudaStream_t st) {
    const FieldDev tang{kFieldAcTangent, eps, u}, react{kFieldAcReaction, eps, u};
    return fused_core(m, r, 128, 1, 2, false, F != nullptr, tang, react, T, F, nullptr, st, nullptr);
}

}  // namespace tgk
