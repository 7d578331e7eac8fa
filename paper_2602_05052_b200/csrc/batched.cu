// Batched operator-learning assembly (BASELINE.json configs[3], "C4"): B
// per-element coefficient fields rho_b on one mesh -> B stiffness matrices on
// one CSR pattern (+ one load vector), i.e. B x (CoefficientField::per_element
// evaluate + local_stiffness_diffusion + reduce_matrix) of the reference
// (coefficient.cpp:34-55, batch.cpp:156-181, routing.cpp:109-132), fused.
//
// Same row-block plan as the scalar fused kernel (plan.cpp), but the geometry
// of the whole block halo is computed ONCE and kept in shared memory (det and
// the k(k+1)/2 gradient dot products per element; small for 2D meshes), then
// for every field b the block re-runs only the cheap part: sc_q = w_q*det*rho_b
// and K_e = sum_q sc_q*(G_a.G_b) in the reference's operation order (phase A),
// and the ascending-element row fold (phase B) — bit-identical to B calls of
// the reference assemble.  Output K is field-major (B x nnz).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);

namespace {

struct BatchedArgs {
    const double* nodes;
    const double* rho;  // B x E
    int64_t E, nnz, B;
    double source;
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
    double* K;  // B x nnz
    double* F;  // N (may be null)
    int lmax, max_halo, max_bnodes, max_block_recs, max_block_chunks;
    int64_t fields_per_block;  // blockIdx.y selects a group of fields (fills the GPU for few row blocks)
    unsigned long long* bad;
};

__host__ __device__ constexpr int brot(int a, int b) { return b == a ? 0 : (b < a ? b + 1 : b); }

template <int KIND>
struct BCfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
    static constexpr int ND = k * (k + 1) / 2;  // unique gradient dot products
    static constexpr int NG = ND + 1;           // + det
    static constexpr int raw = 4 * k + 4;  // k rotated K rows of 4 doubles, then F
    static constexpr int stride = (raw / 2) % 2 == 1 ? raw : raw + 2;  // 2 x odd: conflict-free lanes
    static size_t smem(int R, int lmax, int max_halo, int max_bnodes, int max_block_recs, int max_block_chunks) {
        auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
        size_t o = 0;
        o = al(o + sizeof(double) * size_t(max_halo) * NG);            // geometry cache
        o = al(o + sizeof(double) * size_t(R) * stride);               // ke
        o = al(o + sizeof(double) * size_t(R) * lmax);                 // acc
        o = al(o + sizeof(double) * size_t(max_bnodes) * d);           // node table
        o = al(o + sizeof(uint32_t) * size_t(max_halo));               // halo element ids
        o = al(o + sizeof(uint32_t) * size_t(max_block_recs));         // records of all chunks
        o = al(o + sizeof(uint16_t) * size_t(max_block_chunks) * (R + 8));  // row offsets of all chunks
        o = al(o + sizeof(int64_t) * size_t(max_block_chunks + 1));    // chunk record offsets
        return o;
    }
};

template <int KIND, int DEG, int R>
__global__ void __launch_bounds__(R) k_batched(BatchedArgs p) {
    using C = BCfg<KIND>;
    using Rl = Rule<KIND, DEG>;
    constexpr int k = C::k, d = C::d, Q = Rl::Q, NG = C::NG, ROS = R + 8;
    extern __shared__ __align__(16) unsigned char smb[];
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t o = 0;
    double* geo = reinterpret_cast<double*>(smb + o); o = al(o + sizeof(double) * size_t(p.max_halo) * NG);
    double* ke = reinterpret_cast<double*>(smb + o); o = al(o + sizeof(double) * size_t(R) * C::stride);
    double* acc = reinterpret_cast<double*>(smb + o); o = al(o + sizeof(double) * size_t(R) * p.lmax);
    double* nt = reinterpret_cast<double*>(smb + o); o = al(o + sizeof(double) * size_t(p.max_bnodes) * d);
    uint32_t* hid = reinterpret_cast<uint32_t*>(smb + o); o = al(o + sizeof(uint32_t) * size_t(p.max_halo));
    uint32_t* rec_s = reinterpret_cast<uint32_t*>(smb + o); o = al(o + sizeof(uint32_t) * size_t(p.max_block_recs));
    uint16_t* ro_s = reinterpret_cast<uint16_t*>(smb + o); o = al(o + sizeof(uint16_t) * size_t(p.max_block_chunks) * ROS);
    int64_t* cro = reinterpret_cast<int64_t*>(smb + o);

    const int tid = threadIdx.x;
    const int64_t blk = blockIdx.x;
    const int64_t r0 = p.row_off[blk];
    const int nr = static_cast<int>(p.row_off[blk + 1] - r0);
    const int64_t h0 = p.halo_off[blk];
    const int nh = static_cast<int>(p.halo_off[blk + 1] - h0);
    const int64_t c0 = p.chunk_off[blk];
    const int nch = static_cast<int>(p.chunk_off[blk + 1] - c0);
    const int64_t n0 = p.bnode_off[blk];
    const int nbn = static_cast<int>(p.bnode_off[blk + 1] - n0);

    // ---------------- prologue: node table, halo ids, records, row offsets
    for (int i = tid; i <= nch; i += R) cro[i] = p.chunk_rec_off[c0 + i] - p.chunk_rec_off[c0];
    for (int i = tid; i < nbn; i += R) {
        const int64_t g = p.bnodes[n0 + i];
#pragma unroll
        for (int c = 0; c < d; ++c) nt[i * d + c] = __ldg(p.nodes + g * d + c);
    }
    for (int i = tid; i < nh; i += R) hid[i] = p.halo[h0 + i];
    {
        const int64_t rb = p.chunk_rec_off[c0];
        const int nrec = static_cast<int>(p.chunk_rec_off[c0 + nch] - rb);
        for (int i = tid; i < nrec; i += R) rec_s[i] = p.recs[rb + i];
        for (int i = tid; i < nch * ROS; i += R) ro_s[i] = p.chunk_row_off[c0 * ROS + i];
    }
    __syncthreads();
    // ---------------- geometry of the whole halo, once (batch.cpp:76-154)
    for (int h = tid; h < nh; h += R) {
        const ushort4 ln = *reinterpret_cast<const ushort4*>(p.halo_lconn + (h0 + h) * 4);
        const int ids[4] = {ln.x, ln.y, ln.z, ln.w};
        double X[k][d];
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int c = 0; c < d; ++c) X[a][c] = nt[ids[a] * d + c];
        double det, G[k][d];
        if (!simplex_geometry<KIND, false>(X, det, G)) {
            atomicMin(p.bad, static_cast<unsigned long long>(hid[h]));
            det = 0.0;
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int c = 0; c < d; ++c) G[a][c] = 0.0;
        }
        double* g = geo + h * NG;
        g[0] = det;
        int t = 1;
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int b = a; b < k; ++b) g[t++] = gdot<KIND>(G, a, b);
    }
    // ---------------- one pass per field
    const int64_t bf0 = int64_t(blockIdx.y) * p.fields_per_block;
    const int64_t bf1 = bf0 + p.fields_per_block < p.B ? bf0 + p.fields_per_block : p.B;
    for (int64_t b = bf0; b < bf1; ++b) {
        const double* rho_b = p.rho + b * p.E;
        const bool with_f = b == 0 && p.F != nullptr;
        for (int i = tid; i < R * p.lmax; i += R) acc[i] = 0.0;
        double dK = 0.0, dF = 0.0;
        int diag_pos = 0;
        for (int c = 0; c < nch; ++c) {
            __syncthreads();  // geometry ready / previous phase B done with ke
            const int h = c * R + tid;
            if (h < nh) {
                // phase A: local_stiffness_diffusion with c_q = rho_b[e] (batch.cpp:168-177)
                const double* g = geo + h * NG;
                const double det = g[0];
                const double rho = __ldg(rho_b + hid[h]);
                double sc[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) sc[q] = Rl::w(q) * det * rho;
                double* out = ke + tid * C::stride;
                int t = 1;
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int bb = a; bb < k; ++bb) {
                        const double dot = g[t++];
                        double v = sc[0] * dot;
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += sc[q] * dot;
                        out[a * 4 + brot(a, bb)] = v;
                        out[bb * 4 + brot(bb, a)] = v;
                    }
                if (with_f) {
                    // local_load with a constant source (batch.cpp:280-286)
#pragma unroll
                    for (int a = 0; a < k; ++a) {
                        double v = (Rl::w(0) * det * p.source) * basis<KIND, DEG>(0, a);
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += (Rl::w(q) * det * p.source) * basis<KIND, DEG>(q, a);
                        out[4 * k + a] = v;
                    }
                }
            }
            __syncthreads();
            // phase B: owned row tid folds its records of chunk c, ascending element
            if (tid < nr) {
                const uint16_t* ro = ro_s + c * ROS;
                const uint32_t* rs = rec_s + cro[c];
                for (int j = ro[tid]; j < ro[tid + 1]; ++j) {
                    const uint32_t rec = rs[j];
                    const int hl = rec & 0xff;
                    const int a = (rec >> 8) & 3;
                    const double* src = ke + hl * C::stride + a * 4;
                    int pos[k - 1];
                    double ak[k - 1];
#pragma unroll
                    for (int j2 = 0; j2 < k - 1; ++j2) {
                        pos[j2] = ((rec >> (10 + 5 * j2)) & 31) * R + tid;
                        ak[j2] = acc[pos[j2]];
                    }
#pragma unroll
                    for (int j2 = 0; j2 < k - 1; ++j2) acc[pos[j2]] = ak[j2] + src[j2 + 1];
                    dK += src[0];
                    if (with_f) dF += ke[hl * C::stride + 4 * k + a];
                    diag_pos = (rec >> 25) & 31;
                }
            }
        }
        __syncthreads();
        // epilogue: this field's rows -> K_b
        if (tid < nr) {
            const int64_t packed = p.rows_rp[r0 + tid];
            const int64_t rp = packed & ((int64_t(1) << 56) - 1);
            const int len = static_cast<int>(packed >> 56);
            acc[diag_pos * R + tid] = dK;
            double* Kb = p.K + b * p.nnz + rp;
            for (int q = 0; q < len; ++q) Kb[q] = acc[q * R + tid];
            if (with_f) p.F[p.rows[r0 + tid]] = dF;
        }
    }
}

template <int KIND, int DEG, int R>
int launch_batched(const BatchedArgs& a, int64_t nb, cudaStream_t st) {
    auto kern = k_batched<KIND, DEG, R>;
    const size_t smem = BCfg<KIND>::smem(R, a.lmax, a.max_halo, a.max_bnodes, a.max_block_recs, a.max_block_chunks);
    if (smem > 227 * 1024) return TGK_ERR_INPUT;  // caller falls back to one fused launch per field
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 grid(static_cast<unsigned>(nb), static_cast<unsigned>((a.B + a.fields_per_block - 1) / a.fields_per_block));
    if (nb > 0) kern<<<grid, R, smem, st>>>(a);
    KERNEL_CHECK("batched");
    return TGK_OK;
}

// ---------------------------------------------------------------------------
// Entry-owned batched kernel (plan_entries.cpp).  A block owns R rows and its
// whole halo; thread t owns halo elements t, t+T, ... and CSR entries t, t+T,
// ...  Prologue: the geometry of its halo elements (det + the k(k+1)/2
// gradient dot products) into registers, once, and for field 0 the load
// vector.  Then FPI fields per iteration: each thread writes its halo
// elements' k(k+1)/2 local stiffness values per field (sc_q = w_q*det*rho_b,
// K_e[a][b] = sum_q sc_q*(G_a.G_b) in the reference's order,
// batch.cpp:168-177) to a double-buffered shared array, one barrier, and
// folds each of its entries' contribution lists in a register from +0.0 in
// ascending element order (routing.cpp:117-124) and streams the values out.
// MAXC > 0: the contribution lists (shared-memory offsets) live in registers,
// padded with the offset of a +0.0 slot (adding +0.0 to a sum that started at
// +0.0 never changes it: the sum is never -0.0); MAXC = 0: they are read from
// shared memory.  The next fields' coefficients are prefetched.
constexpr int kEntryThreads = 256;
constexpr int kEntryFPI = 2;  // fields per barrier

struct EntryArgs {
    const double* nodes;
    const double* rho;  // B x E
    int64_t E, nnz, B;
    double source;
    EntryPlanDev pl;
    double* K;  // B x nnz
    double* F;  // N (may be null)
    int64_t fields_per_block;
    int streaming_stores;  // st.global.cs (evict-first) for K
    unsigned long long* bad;
};

template <int KIND>
struct ECfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d, ND = k * (k + 1) / 2;
    __host__ __device__ static int fstride(int MH) { return ND * MH + 2; }  // one field's values + the +0.0 slot (even)
    static size_t smem(const EntryPlanDev& pl, bool lists_in_smem) {
        auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
        const size_t vals = size_t(2 * kEntryFPI) * fstride(pl.max_halo);
        size_t o = al(sizeof(double) * std::max(vals, size_t(pl.max_bnodes) * d));  // values | node table
        if (lists_in_smem) o = al(o + sizeof(uint32_t) * size_t(pl.max_contrib));
        return o;
    }
};

template <int KIND, int DEG, int EPT, int HPT, int MAXC>
__global__ void __launch_bounds__(kEntryThreads) k_batched_entries(EntryArgs p) {
    using Rl = Rule<KIND, DEG>;
    using Cf = ECfg<KIND>;
    constexpr int k = Cf::k, d = Cf::d, Q = Rl::Q, ND = Cf::ND, T = kEntryThreads, FPI = kEntryFPI;
    extern __shared__ __align__(16) unsigned char smb[];
    const EntryPlanDev& pl = p.pl;
    const int MH = pl.max_halo;
    const int FS = Cf::fstride(MH);
    double* kb = reinterpret_cast<double*>(smb);
    double* nt = kb;  // node table, prologue only
    uint32_t* cs_s = reinterpret_cast<uint32_t*>(
        smb + ((sizeof(double) * (size_t(2 * FPI) * FS > size_t(pl.max_bnodes) * d ? size_t(2 * FPI) * FS
                                                                              : size_t(pl.max_bnodes) * d) +
               15) &
              ~size_t(15)));

    const int tid = threadIdx.x;
    const int64_t blk = blockIdx.x;
    const int64_t r0 = pl.row_off[blk];
    const int nr = static_cast<int>(pl.row_off[blk + 1] - r0);
    const int64_t h0 = pl.halo_off[blk];
    const int nh = static_cast<int>(pl.halo_off[blk + 1] - h0);
    const int64_t n0 = pl.bnode_off[blk];
    const int nbn = static_cast<int>(pl.bnode_off[blk + 1] - n0);
    const int64_t e0 = pl.ent_off[blk];
    const int ne = static_cast<int>(pl.ent_off[blk + 1] - e0);
    const int64_t c0 = pl.contrib_off[blk];

    if (MAXC == 0) {
        const int ncs = static_cast<int>(pl.contrib_off[blk + 1] - c0);
        for (int i = tid; i < ncs; i += T) cs_s[i] = __ldg(pl.contrib + c0 + i);
    }
    for (int i = tid; i < nbn; i += T) {
        const int64_t g = pl.bnodes[n0 + i];
#pragma unroll
        for (int c = 0; c < d; ++c) nt[i * d + c] = __ldg(p.nodes + g * d + c);
    }
    uint32_t eid[HPT];
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh) {
        const int h = tid + hh * T;
        eid[hh] = h < nh ? __ldg(pl.halo + h0 + h) : 0u;
    }
    const int64_t bf0 = int64_t(blockIdx.y) * p.fields_per_block;
    const int64_t bf1 = bf0 + p.fields_per_block < p.B ? bf0 + p.fields_per_block : p.B;
    double rn[HPT][FPI];
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh)
#pragma unroll
        for (int f = 0; f < FPI; ++f)
            rn[hh][f] = (tid + hh * T < nh && bf0 + f < bf1) ? __ldg(p.rho + (bf0 + f) * p.E + eid[hh]) : 0.0;
    // my entries: CSR positions and contribution lists
    const uint32_t zslot = uint32_t(ND * MH);  // +0.0 slot of a field's values
    int64_t epos[EPT], epos2[EPT];
    uint32_t cb[EPT], ce[EPT];
    uint32_t cl[EPT][MAXC > 0 ? MAXC : 1];
    int wl[EPT];  // warp-uniform longest list
    {
        const uint32_t* coff = pl.coff + e0 + blk;
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            const int e = tid + j * T;
            epos[j] = e < ne ? __ldg(pl.epos + e0 + e) : 0;
            epos2[j] = e < ne ? __ldg(pl.epos2 + e0 + e) : -1;
            cb[j] = e < ne ? __ldg(coff + e) : 0u;
            ce[j] = e < ne ? __ldg(coff + e + 1) : 0u;
            wl[j] = static_cast<int>(__reduce_max_sync(0xffffffffu, ce[j] - cb[j]));
            if (MAXC > 0) {
#pragma unroll
                for (int c = 0; c < (MAXC > 0 ? MAXC : 1); ++c)
                    cl[j][c] = cb[j] + c < ce[j] ? __ldg(pl.contrib + c0 + cb[j] + c) : zslot;
            }
        }
    }
    __syncthreads();
    // ---------------- halo geometry, once (batch.cpp:76-154)
    double gd[HPT][ND], gdet[HPT];
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh) {
        const int h = tid + hh * T;
        gdet[hh] = 0.0;
#pragma unroll
        for (int t = 0; t < ND; ++t) gd[hh][t] = 0.0;
        if (h < nh) {
            const uint64_t hc = __ldg(reinterpret_cast<const unsigned long long*>(pl.hconn) + h0 + h);
            double X[k][d];
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int c = 0; c < d; ++c) X[a][c] = nt[int((hc >> (16 * a)) & 0xffff) * d + c];
            double det, G[k][d];
            if (!simplex_geometry<KIND, false>(X, det, G)) {
                atomicMin(p.bad, static_cast<unsigned long long>(eid[hh]));
                det = 0.0;
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int c = 0; c < d; ++c) G[a][c] = 0.0;
            }
            gdet[hh] = det;
            int t = 0;
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int b = a; b < k; ++b) gd[hh][t++] = gdot<KIND>(G, a, b);
        }
    }
    __syncthreads();  // node table (aliasing the value buffers) no longer read
    for (int i = tid; i < 2 * FPI; i += T) kb[i * FS + zslot] = 0.0;
    if (bf0 == 0 && p.F != nullptr) {
        // local_load with a constant source (batch.cpp:280-286) into the second
        // buffer set (first used by iteration 1), then the ascending-element row fold
        double* fe = kb + FPI * FS;
#pragma unroll
        for (int hh = 0; hh < HPT; ++hh) {
            const int h = tid + hh * T;
            if (h < nh) {
                const double det = gdet[hh];
#pragma unroll
                for (int a = 0; a < k; ++a) {
                    double v = (Rl::w(0) * det * p.source) * basis<KIND, DEG>(0, a);
#pragma unroll
                    for (int q = 1; q < Q; ++q) v += (Rl::w(q) * det * p.source) * basis<KIND, DEG>(q, a);
                    fe[a * MH + h] = v;
                }
            }
        }
        __syncthreads();
        const int64_t f0 = pl.fcontrib_off[blk];
        const uint32_t* fcoff = pl.fcoff + r0 + blk;
        for (int i = tid; i < nr; i += T) {
            double v = 0.0;
            for (uint32_t c = __ldg(fcoff + i); c < __ldg(fcoff + i + 1); ++c) v += fe[__ldg(pl.fcontrib + f0 + c)];
            p.F[pl.rows[r0 + i]] = v;
        }
    }
    // ---------------- FPI fields per iteration
    int set = 0;
    for (int64_t b = bf0; b < bf1; b += FPI, set ^= 1) {
        double* kv = kb + set * FPI * FS;
#pragma unroll
        for (int hh = 0; hh < HPT; ++hh) {
            const int h = tid + hh * T;
            if (h < nh) {
#pragma unroll
                for (int f = 0; f < FPI; ++f) {
                    const double rho = rn[hh][f];
                    if (b + FPI + f < bf1) rn[hh][f] = __ldg(p.rho + (b + FPI + f) * p.E + eid[hh]);
                    double sc[Q];
#pragma unroll
                    for (int q = 0; q < Q; ++q) sc[q] = Rl::w(q) * gdet[hh] * rho;
#pragma unroll
                    for (int t = 0; t < ND; ++t) {
                        const double dot = gd[hh][t];
                        double v = sc[0] * dot;
#pragma unroll
                        for (int q = 1; q < Q; ++q) v += sc[q] * dot;
                        kv[f * FS + t * MH + h] = v;
                    }
                }
            }
        }
        __syncthreads();
        const int nf = bf1 - b < FPI ? static_cast<int>(bf1 - b) : FPI;
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            if (j * T >= ne) break;  // block-uniform
            double v[FPI];
#pragma unroll
            for (int f = 0; f < FPI; ++f) v[f] = 0.0;
            if (MAXC > 0) {
#pragma unroll
                for (int c = 0; c < (MAXC > 0 ? MAXC : 1); ++c) {
                    if (c < wl[j]) {  // warp-uniform
#pragma unroll
                        for (int f = 0; f < FPI; ++f) v[f] += kv[f * FS + cl[j][c]];
                    }
                }
            } else {
                for (uint32_t c = cb[j]; c < ce[j]; ++c) {
                    const uint32_t u = cs_s[c];
#pragma unroll
                    for (int f = 0; f < FPI; ++f) v[f] += kv[f * FS + u];
                }
            }
            if (tid + j * T < ne) {
#pragma unroll
                for (int f = 0; f < FPI; ++f)
                    if (f < nf) {
                        double* Kb = p.K + (b + f) * p.nnz;
                        if (p.streaming_stores) {
                            __stcs(Kb + epos[j], v[f]);
                            if (epos2[j] >= 0) __stcs(Kb + epos2[j], v[f]);
                        } else {
                            Kb[epos[j]] = v[f];
                            if (epos2[j] >= 0) Kb[epos2[j]] = v[f];
                        }
                    }
            }
        }
    }
}

template <int KIND, int EPT, int HPT, int MAXC>
int launch_entries(const EntryArgs& a, int64_t groups, cudaStream_t st) {
    auto kern = k_batched_entries<KIND, 2, EPT, HPT, MAXC>;
    const size_t smem = ECfg<KIND>::smem(a.pl, MAXC == 0);
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 grid(static_cast<unsigned>(a.pl.n_blocks), static_cast<unsigned>(groups));
    if (a.pl.n_blocks > 0) kern<<<grid, kEntryThreads, smem, st>>>(a);
    KERNEL_CHECK("batched_entries");
    return TGK_OK;
}

template <int KIND, int MAXC>
int launch_entries_eh(const EntryArgs& a, int ept, int hpt, int64_t groups, cudaStream_t st) {
    if (hpt == 1) {
        if (ept == 1) return launch_entries<KIND, 1, 1, MAXC>(a, groups, st);
        if (ept == 2) return launch_entries<KIND, 2, 1, MAXC>(a, groups, st);
        return launch_entries<KIND, 4, 1, MAXC>(a, groups, st);
    }
    if (ept == 1) return launch_entries<KIND, 1, 2, MAXC>(a, groups, st);
    if (ept == 2) return launch_entries<KIND, 2, 2, MAXC>(a, groups, st);
    return launch_entries<KIND, 4, 2, MAXC>(a, groups, st);
}

int pow2_at_least(int x) {
    int v = 1;
    while (v < x) v <<= 1;
    return v;
}

}  // namespace

// Returns TGK_ERR_INPUT without launching (and without setting an error
// message) when the block working set does not fit shared memory.
int batched_fused(const tgk_mesh* m, tgk_routing* r, int64_t B, const double* rho, double source, double* K,
                  double* F, cudaStream_t st, unsigned long long* d_bad) {
    constexpr int R = 64;
    const PlanDev* pl = nullptr;
    TGK_TRY(ensure_plan(r, R, &pl));
    BatchedArgs a{};
    a.nodes = m->nodes;
    a.rho = rho;
    a.E = m->E;
    a.nnz = r->nnz;
    a.B = B;
    a.source = source;
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
    a.K = K;
    a.F = F;
    a.lmax = pl->lmax;
    a.max_halo = pl->max_block_halo;
    a.max_bnodes = pl->max_bnodes;
    a.max_block_recs = pl->max_block_recs;
    a.max_block_chunks = pl->max_block_chunks;
    a.bad = d_bad;
    // field groups: about 16 resident blocks' worth of work per SM in total
    const int64_t groups = std::max<int64_t>(1, std::min<int64_t>(B, (148 * 16 + pl->n_blocks - 1) / std::max<int64_t>(1, pl->n_blocks)));
    a.fields_per_block = (B + groups - 1) / groups;
    if (const char* e = getenv("TGK_BATCHED_FPB")) a.fields_per_block = std::max(1, atoi(e));
    if (m->kind == TGK_TRI3) return launch_batched<TGK_TRI3, 2, R>(a, pl->n_blocks, st);
    return launch_batched<TGK_TET4, 2, R>(a, pl->n_blocks, st);
}

// Entry-owned batched kernel.  Returns TGK_ERR_INPUT without launching (and
// without an error message) when it does not apply: element-range slabs, or
// no rows-per-block choice whose block working set fits.
int batched_entries(const tgk_mesh* m, tgk_routing* r, int64_t B, const double* rho, double source, double* K,
                    double* F, cudaStream_t st, unsigned long long* d_bad) {
    const tgk_routing* s = r->scalar ? r->scalar : r;
    if (s->elem_hi >= 0) return TGK_ERR_INPUT;
    int R0 = m->kind == TGK_TRI3 ? 64 : 16;
    if (const char* e = getenv("TGK_ENTRY_R")) R0 = std::max(1, atoi(e));
    int maxc_cap = 16;  // register-resident contribution lists up to this length
    if (const char* e = getenv("TGK_ENTRY_MAXC")) maxc_cap = atoi(e);
    const EntryPlanDev* pl = nullptr;
    int ept = 0, hpt = 0, maxc = 0;
    size_t smem = 0;
    for (int R = R0; R >= 4; R /= 2) {
        TGK_TRY(ensure_entry_plan(r, R, &pl));
        ept = pow2_at_least((pl->max_entries + kEntryThreads - 1) / kEntryThreads);
        hpt = pow2_at_least((pl->max_halo + kEntryThreads - 1) / kEntryThreads);
        maxc = pl->max_clen <= 8 && maxc_cap >= 8 ? 8 : pl->max_clen <= 16 && maxc_cap >= 16 ? 16 : 0;
        smem = m->kind == TGK_TRI3 ? ECfg<TGK_TRI3>::smem(*pl, maxc == 0) : ECfg<TGK_TET4>::smem(*pl, maxc == 0);
        if (ept <= 4 && hpt <= 2 && smem <= 200 * 1024) break;
        pl = nullptr;
    }
    if (!pl) return TGK_ERR_INPUT;
    EntryArgs a{};
    a.nodes = m->nodes;
    a.rho = rho;
    a.E = m->E;
    a.nnz = r->nnz;
    a.B = B;
    a.source = source;
    a.pl = *pl;
    a.K = K;
    a.F = F;
    a.bad = d_bad;
    a.streaming_stores = 0;
    if (const char* e = getenv("TGK_ENTRY_STCS")) a.streaming_stores = atoi(e);
    // fields per block: few enough that the blocks in flight at any time work
    // on a handful of fields (their coefficient vectors stay in L2 for the
    // random per-element gathers), enough to amortise the prologue
    int64_t fpb = 8;
    if (const char* e = getenv("TGK_ENTRY_FPB")) fpb = std::max(1, atoi(e));
    a.fields_per_block = std::min<int64_t>(B, fpb);
    a.fields_per_block += a.fields_per_block % kEntryFPI;  // whole iterations
    const int64_t groups = (B + a.fields_per_block - 1) / a.fields_per_block;
    if (m->kind == TGK_TRI3) {
        if (maxc == 8) return launch_entries_eh<TGK_TRI3, 8>(a, ept, hpt, groups, st);
        if (maxc == 16) return launch_entries_eh<TGK_TRI3, 16>(a, ept, hpt, groups, st);
        return launch_entries_eh<TGK_TRI3, 0>(a, ept, hpt, groups, st);
    }
    if (maxc == 8) return launch_entries_eh<TGK_TET4, 8>(a, ept, hpt, groups, st);
    if (maxc == 16) return launch_entries_eh<TGK_TET4, 16>(a, ept, hpt, groups, st);
    return launch_entries_eh<TGK_TET4, 0>(a, ept, hpt, groups, st);
}

}  // namespace tgk
