// Fused P1 linear-elasticity assembly (tg::assemble LinearElasticity branch,
// physics.cpp:45-66): K (3x3 / 2x2 blocks on the node-major interleaved DoF
// numbering, dofmap.cpp:18-19) and the body-force load F, straight from mesh +
// Lame fields to CSR values, bit-identical to the reference.
//
// Same row-block plan as the scalar fused kernel (plan.cpp, built on the
// SCALAR routing): CUDA block b owns R mesh nodes = R*d DoF rows and walks the
// elements incident to them in level order, R per chunk.
//   phase A  one thread per element: exact geometry (det, G, batch.cpp:76-154)
//            and the quadrature values of lambda, mu (plane-stress corrected)
//            and the body force into shared memory;
//   phase B  one thread per owned node row: for each record (element e, local
//            node a) in ascending element order it forms the d x (k d) block
//            rows of local_stiffness_elasticity (batch.cpp:198-246) for node a
//            — only the structural nonzeros of B and D*B, which is exact (a
//            skipped term is +-0.0 added to a sum that starts at +0.0) — and
//            folds them into the row's accumulators: the diagonal d x d block
//            and the load in registers, the off-diagonal blocks in shared
//            memory (lane = row: conflict-free);
//   epilogue each node's d DoF rows are one contiguous run of d*d*len values
//            of the vector CSR (slot_v(d i + c, d j + c') = d^2 rp_s[i] +
//            d c len_s(i) + d (t_s - rp_s[i]) + c'), written by one warp.
#include <climits>
#include <cstdlib>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

int check_bad(unsigned long long* d_bad, cudaStream_t st);

namespace {

struct FieldE {
    int type;
    double value;
    const double* data;
};

struct ElastArgs {
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
    const int64_t* chunk_rec_off;
    const uint16_t* chunk_row_off;
    const uint32_t* recs;
    FieldE lam, mu, src[3];
    int n_src, plane_stress;
    double* K;
    double* F;
    int lmax, S, max_recs, max_bnodes, max_chunks, ntcols;
    unsigned long long* bad;     // [0] first bad element, [1] mu <= 0 flag
};

constexpr int kRingE = 3;

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// gradient component carried by Voigt row i for displacement component c, -1 if structurally zero
// (batch.cpp:205-227)
template <int D>
__host__ __device__ constexpr int vcomp(int i, int c) {
    if (D == 3) {
        return i == 0 ? (c == 0 ? 0 : -1)
             : i == 1 ? (c == 1 ? 1 : -1)
             : i == 2 ? (c == 2 ? 2 : -1)
             : i == 3 ? (c == 0 ? 1 : (c == 1 ? 0 : -1))
             : i == 4 ? (c == 1 ? 2 : (c == 2 ? 1 : -1))
             : (c == 0 ? 2 : (c == 2 ? 0 : -1));
    }
    return i == 0 ? (c == 0 ? 0 : -1) : i == 1 ? (c == 1 ? 1 : -1) : (c == 0 ? 1 : (c == 1 ? 0 : -1));
}

template <int KIND, int DEG>
struct ECfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    // per element in shared memory: G (k x d), det, lambda_q, mu_q, f_qc
    static constexpr int offG = 0, offDet = k * d, offLam = offDet + 1, offMu = offLam + Q, offF = offMu + Q;
    static constexpr int raw = offF + Q * d;
    static constexpr int stride = raw % 2 == 0 ? ((raw / 2) % 2 == 1 ? raw : raw + 2) : raw;  // odd or 2 x odd
};

template <int KIND, int DEG>
__device__ __forceinline__ double fieldE_q(const FieldE& f, const double* nod, int64_t e, int q) {
    constexpr int k = P1<KIND>::k;
    if (f.type == TGK_FIELD_NODAL) {  // interpolate_nodal (batch.cpp:321-330)
        double v = basis<KIND, DEG>(q, 0) * nod[0];
#pragma unroll
        for (int a = 1; a < k; ++a) v += basis<KIND, DEG>(q, a) * nod[a];
        return v;
    }
    return f.type == TGK_FIELD_ELEMENT ? __ldg(f.data + e) : f.value;
}

// ---------------------------------------------------------------------------
// Exact fused elasticity: the block rows of K_e are computed by one thread per
// RECORD (all lanes busy), then folded.
// Per chunk of C halo elements:
//   phase A   one thread per element: geometry + quadrature values;
//   phase B1  one thread per record (element e, owned node a): block row a of
//             local_stiffness_elasticity (batch.cpp:198-246, structural
//             nonzeros only, per-value quadrature fold in the reference order)
//             and F_e[a] into a record buffer, blocks rotated like the record
//             (diagonal block first, then the other nodes ascending);
//   phase B2  one thread per (owned node row, block entry (c, c')) — warp
//             c*d + c', lane = row: folds entry (c, c') of each of its
//             records' blocks in ascending element order, the diagonal block
//             entry and F_c (c' = 0) in registers, the others into shared
//             accumulators [pos][c][c'][row].
template <int D, int R>
constexpr int elast2_threads() { return (R * D * D + 31) / 32 * 32; }

template <int KIND, int DEG>
struct E2Cfg {
    static constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
    static constexpr int RS = k * d * d + d;                  // record buffer doubles: k blocks + F
    static constexpr int RSP = RS % 2 == 1 ? RS : RS + 1;     // odd stride: spread banks
};

template <int KIND, int DEG, int R>
__global__ void __launch_bounds__(elast2_threads<P1<KIND>::d, R>(), R <= 16 ? 3 : 2) k_fused_elast2(ElastArgs p) {
    using C = ECfg<KIND, DEG>;
    using C2 = E2Cfg<KIND, DEG>;
    using Rl = Rule<KIND, DEG>;
    constexpr int k = C::k, d = C::d, Q = C::Q, ns = d == 2 ? 3 : 6;
    constexpr int T = elast2_threads<d, R>(), ROS = R + 8, RSP = C2::RSP;
    const int CH = p.S;  // halo elements per chunk (plan C)
    extern __shared__ __align__(16) unsigned char sme[];
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t o = 0;
    double* ke = reinterpret_cast<double*>(sme + o); o = al(o + sizeof(double) * size_t(CH) * C::stride);
    double* rb = reinterpret_cast<double*>(sme + o); o = al(o + sizeof(double) * size_t(p.max_recs) * RSP);
    double* acc = reinterpret_cast<double*>(sme + o); o = al(o + sizeof(double) * size_t(p.lmax) * d * d * R);
    double* nt = reinterpret_cast<double*>(sme + o); o = al(o + sizeof(double) * size_t(p.max_bnodes) * p.ntcols);
    uint32_t* rec_s = reinterpret_cast<uint32_t*>(sme + o); o = al(o + sizeof(uint32_t) * kRingE * size_t(p.max_recs));
    uint16_t* ro_s = reinterpret_cast<uint16_t*>(sme + o); o = al(o + sizeof(uint16_t) * kRingE * ROS);
    ushort4* lc_s = reinterpret_cast<ushort4*>(sme + o); o = al(o + sizeof(ushort4) * kRingE * size_t(CH));
    int64_t* cro = reinterpret_cast<int64_t*>(sme + o);

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

    for (int i = tid; i <= nch; i += T) cro[i] = p.chunk_rec_off[c0 + i];
    for (int i = tid; i < nbn; i += T) {
        const int64_t g = p.bnodes[n0 + i];
#pragma unroll
        for (int c = 0; c < d; ++c) cpa8(nt + i * p.ntcols + c, p.nodes + g * d + c);
        int col = d;
        if (p.lam.type == TGK_FIELD_NODAL) cpa8(nt + i * p.ntcols + col++, p.lam.data + g);
        if (p.mu.type == TGK_FIELD_NODAL) cpa8(nt + i * p.ntcols + col++, p.mu.data + g);
        for (int c = 0; c < p.n_src; ++c)
            if (p.src[c].type == TGK_FIELD_NODAL) cpa8(nt + i * p.ntcols + col++, p.src[c].data + g);
    }
    cpa_commit();
    for (int i = tid; i < p.lmax * d * d * R; i += T) acc[i] = 0.0;
    __syncthreads();

    auto stage = [&](int c) {
        if (c < nch) {
            const int sl = c % kRingE;
            const int64_t cg = c0 + c;
            const int64_t rbeg = cro[c];
            const int nrec4 = static_cast<int>((cro[c + 1] - rbeg) >> 2);
            uint32_t* rdst = rec_s + sl * p.max_recs;
            for (int i = tid; i < nrec4; i += T) cpa16(rdst + 4 * i, p.recs + rbeg + 4 * i);
            uint16_t* odst = ro_s + sl * ROS;
            for (int i = tid; i < ROS / 8; i += T) cpa16(odst + 8 * i, p.chunk_row_off + cg * ROS + 8 * i);
            const int64_t hb = h0 + int64_t(c) * CH;
            const int64_t rem = nh - int64_t(c) * CH;
            const int ne = rem < CH ? static_cast<int>(rem) : CH;
            for (int i = tid; i < ne; i += T) cpa8(lc_s + sl * CH + i, p.halo_lconn + (hb + i) * 4);
        }
        cpa_commit();
    };
#pragma unroll
    for (int c = 0; c < kRingE - 1; ++c) stage(c);

    // B2 role: thread (block entry (c, c'), owned row) = (tid / R, tid % R)
    const int fw = tid / R, frow = tid % R;  // block entry (c, c') = fw, owned row
    const bool folder = fw < d * d && frow < nr;
    const int fc = folder ? fw / d : 0, fcp = folder ? fw % d : 0;
    double dK = 0.0, dF = 0.0;
    int diag_pos = 0;

    for (int c = 0; c < nch; ++c) {
        cpa_wait<kRingE - 2>();
        __syncthreads();
        stage(c + kRingE - 1);
        const int sl = c % kRingE;
        // ---------------- phase A: geometry and quadrature values, one thread per element
        const int64_t rem = nh - int64_t(c) * CH;
        const int ne = rem < CH ? static_cast<int>(rem) : CH;
        for (int t = tid; t < ne; t += T) {
            const int64_t h = int64_t(c) * CH + t;
            const ushort4 ln = lc_s[sl * CH + t];
            const int ids[4] = {ln.x, ln.y, ln.z, ln.w};
            double X[k][d];
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int cc = 0; cc < d; ++cc) X[a][cc] = nt[ids[a] * p.ntcols + cc];
            double* out = ke + t * C::stride;
            double det, G[k][d];
            const int64_t e = p.halo[h0 + h];
            if (!simplex_geometry<KIND, false>(X, det, G)) {
                atomicMin(p.bad, static_cast<unsigned long long>(e));
                det = 0.0;
#pragma unroll
                for (int a = 0; a < k; ++a)
#pragma unroll
                    for (int cc = 0; cc < d; ++cc) G[a][cc] = 0.0;
            }
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int cc = 0; cc < d; ++cc) out[C::offG + a * d + cc] = G[a][cc];
            out[C::offDet] = det;
            int col = d;
            double nl[k], nm[k];
            if (p.lam.type == TGK_FIELD_NODAL) {
#pragma unroll
                for (int a = 0; a < k; ++a) nl[a] = nt[ids[a] * p.ntcols + col];
                ++col;
            }
            if (p.mu.type == TGK_FIELD_NODAL) {
#pragma unroll
                for (int a = 0; a < k; ++a) nm[a] = nt[ids[a] * p.ntcols + col];
                ++col;
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                double lam = fieldE_q<KIND, DEG>(p.lam, nl, e, q);
                const double mu = fieldE_q<KIND, DEG>(p.mu, nm, e, q);
                if (mu <= 0.0) atomicMin(p.bad + 1, 0ull);  // batch.cpp:194-195
                if (d == 2 && p.plane_stress) lam = 2.0 * lam * mu / (lam + 2.0 * mu);  // batch.cpp:359-361
                out[C::offLam + q] = lam;
                out[C::offMu + q] = mu;
            }
            for (int cc = 0; cc < d; ++cc) {
                double ns_[k];
                const bool nodal = cc < p.n_src && p.src[cc].type == TGK_FIELD_NODAL;
                if (nodal) {
#pragma unroll
                    for (int a = 0; a < k; ++a) ns_[a] = nt[ids[a] * p.ntcols + col];
                    ++col;
                }
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    out[C::offF + q * d + cc] = cc < p.n_src ? fieldE_q<KIND, DEG>(p.src[cc], ns_, e, q) : 0.0;
            }
        }
        __syncthreads();
        // ---------------- phase B1: block row a of each record, one thread per record
        const uint16_t* ro = ro_s + sl * ROS;
        const uint32_t* rs = rec_s + sl * p.max_recs;
        const int nrec = ro[R];
        for (int j = tid; j < nrec; j += T) {
            const uint32_t rec = rs[j];
            const int hl = rec & 0xff;
            const int a = (rec >> 8) & 3;
            const double* el = ke + hl * C::stride;
            double G[k][d];
#pragma unroll
            for (int b = 0; b < k; ++b)
#pragma unroll
                for (int cc = 0; cc < d; ++cc) G[b][cc] = el[C::offG + b * d + cc];
            double Ga[d];
#pragma unroll
            for (int cc = 0; cc < d; ++cc)
                Ga[cc] = a == 0 ? G[0][cc] : a == 1 ? G[1][cc] : a == 2 ? G[2][cc] : G[k - 1][cc];
            const double det = el[C::offDet];
            double lq[Q], tmq[Q], muq[Q], scq[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                lq[q] = el[C::offLam + q];
                muq[q] = el[C::offMu + q];
                tmq[q] = 2.0 * muq[q];
                scq[q] = Rl::w(q) * det;
            }
            double* out = rb + size_t(j) * RSP;
#pragma unroll
            for (int b = 0; b < k; ++b) {
                const int blkslot = b == a ? 0 : (b < a ? b + 1 : b);  // rotated: diagonal block first
#pragma unroll
                for (int cp = 0; cp < d; ++cp) {
                    const double g = G[b][cp];
                    const double tr = 0.0 + g;  // batch.cpp:231-232
#pragma unroll
                    for (int cc = 0; cc < d; ++cc) {
                        double kv = 0.0;
#pragma unroll
                        for (int q = 0; q < Q; ++q) {
                            double s = 0.0;
#pragma unroll
                            for (int i = 0; i < ns; ++i) {
                                const int ga = vcomp<d>(i, cc);
                                if (ga < 0) continue;
                                double DB;
                                if (i < d) {
                                    DB = i == cp ? lq[q] * tr + tmq[q] * g : lq[q] * tr + tmq[q] * 0.0;
                                } else {
                                    const int gb = vcomp<d>(i, cp);
                                    if (gb < 0) continue;
                                    DB = muq[q] * G[b][gb];
                                }
                                s += Ga[ga] * DB;
                            }
                            kv += scq[q] * s;
                        }
                        out[blkslot * d * d + cc * d + cp] = kv;
                    }
                }
            }
            // local_load_vector (batch.cpp:303-308)
#pragma unroll
            for (int cc = 0; cc < d; ++cc) {
                double fa = 0.0;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const double sB = scq[q] * (a == 0 ? basis<KIND, DEG>(q, 0) : a == 1 ? basis<KIND, DEG>(q, 1)
                                                : a == 2 ? basis<KIND, DEG>(q, 2) : basis<KIND, DEG>(q, k - 1));
                    fa += sB * el[C::offF + q * d + cc];
                }
                out[k * d * d + cc] = fa;
            }
        }
        __syncthreads();
        // ---------------- phase B2: fold, thread = (block entry (c, c'), owned row)
        if (folder) {
            for (int j = ro[frow]; j < ro[frow + 1]; ++j) {
                const uint32_t rec = rs[j];
                const double* src = rb + size_t(j) * RSP + fc * d + fcp;
                dK += src[0];
                int pos[k - 1];
                double old[k - 1];
#pragma unroll
                for (int jj = 0; jj < k - 1; ++jj) {
                    pos[jj] = (rec >> (10 + 5 * jj)) & 31;
                    old[jj] = acc[((size_t(pos[jj]) * d + fc) * d + fcp) * R + frow];
                }
#pragma unroll
                for (int jj = 0; jj < k - 1; ++jj)
                    acc[((size_t(pos[jj]) * d + fc) * d + fcp) * R + frow] = old[jj] + src[(jj + 1) * d * d];
                if (fcp == 0) dF += rb[size_t(j) * RSP + k * d * d + fc];
                diag_pos = (rec >> 25) & 31;
            }
        }
    }
    cpa_wait<0>();
    __syncthreads();
    if (folder) {
        acc[((size_t(diag_pos) * d + fc) * d + fcp) * R + frow] = dK;
        if (fcp == 0) p.F[int64_t(p.rows[r0 + frow]) * d + fc] = dF;
    }
    __syncthreads();
    // epilogue: node r's d DoF rows = d*d*len contiguous values [d^2 rp, d^2 (rp + len)); a warp per node
    for (int i = warp; i < nr; i += T / 32) {
        const int64_t pk = p.rows_rp[r0 + i];
        const int64_t rp = pk & ((int64_t(1) << 56) - 1);
        const int len = static_cast<int>(pk >> 56);
        double* dst = p.K + rp * d * d;
        const int dl = d * len;
        for (int v = lane; v < d * dl; v += 32) {
            const int cc = v >= dl ? (v >= 2 * dl ? 2 : 1) : 0, rem2 = v - cc * dl;
            const int pos = rem2 / d, cp = rem2 - pos * d;
            dst[v] = acc[((size_t(pos) * d + cc) * d + cp) * R + i];
        }
    }
}

template <int KIND, int DEG, int R>
size_t elast2_smem(const ElastArgs& a) {
    using C = ECfg<KIND, DEG>;
    constexpr int d = C::d;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t o = 0;
    o = al(o + sizeof(double) * size_t(a.S) * C::stride);
    o = al(o + sizeof(double) * size_t(a.max_recs) * E2Cfg<KIND, DEG>::RSP);
    o = al(o + sizeof(double) * size_t(a.lmax) * d * d * R);
    o = al(o + sizeof(double) * size_t(a.max_bnodes) * a.ntcols);
    o = al(o + sizeof(uint32_t) * kRingE * size_t(a.max_recs));
    o = al(o + sizeof(uint16_t) * kRingE * (R + 8));
    o = al(o + sizeof(ushort4) * kRingE * size_t(a.S));
    o += sizeof(int64_t) * (a.max_chunks + 2);
    return o;
}

template <int KIND, int DEG, int R>
int launch_elast2(const ElastArgs& a, int64_t nb, cudaStream_t st) {
    auto kern = k_fused_elast2<KIND, DEG, R>;
    const size_t smem = elast2_smem<KIND, DEG, R>(a);
    if (smem > 227 * 1024)
        return set_error(TGK_ERR_INPUT, "fused elasticity: block working set exceeds shared memory (" +
                                            std::to_string(smem) + " B)");
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (nb > 0) kern<<<static_cast<unsigned>(nb), elast2_threads<P1<KIND>::d, R>(), smem, st>>>(a);
    KERNEL_CHECK("fused_elast2");
    return TGK_OK;
}

}  // namespace

// Fused elasticity on device buffers (r: the vector routing; its scalar part carries the plan).
int elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                        cudaStream_t st);

int fused_elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                              cudaStream_t st) {
    int C2 = 48, R2 = 16;  // v2 chunk size and rows per block (measured: C3 6.65 ms at 64, 5.65 ms at 48)
    if (const char* e = getenv("TGK_ELAST_C")) C2 = atoi(e);
    if (const char* e = getenv("TGK_ELAST_R")) R2 = atoi(e) == 32 ? 32 : 16;
    const PlanDev* pl = nullptr;
    {
        // the row-block plan's layout limits (fused.cu): other meshes take the
        // materialised Stage I + II path (elasticity_assemble), bit-identical too
        const tgk_routing* s = r->scalar ? r->scalar : r;
        const int prc = s->lmax > kMaxRowLen ? TGK_ERR_INPUT : ensure_plan(r, R2, &pl, C2);
        if (prc == TGK_ERR_INPUT) return elasticity_assemble(pr, m, r, K, F, st);
        if (prc != TGK_OK) return prc;
    }
    const bool high = pr->diffusion.type != TGK_FIELD_CONSTANT;  // physics.cpp:18-21
    const int d = m->d;
    ElastArgs a{};
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
    a.chunk_rec_off = pl->chunk_rec_off;
    a.chunk_row_off = pl->chunk_row_off;
    a.recs = pl->recs;
    a.lam = FieldE{pr->lambda.type, pr->lambda.value, pr->lambda.data};
    a.mu = FieldE{pr->mu.type, pr->mu.value, pr->mu.data};
    a.n_src = pr->n_source > 0 ? d : 0;
    for (int c = 0; c < a.n_src; ++c) a.src[c] = FieldE{pr->source[c].type, pr->source[c].value, pr->source[c].data};
    a.plane_stress = pr->plane_stress;
    a.K = K;
    a.F = F;
    a.lmax = pl->lmax > 0 ? pl->lmax : 1;
    a.S = C2;  // chunk size
    a.max_recs = pl->max_chunk_recs > 0 ? pl->max_chunk_recs : 4;
    a.max_bnodes = pl->max_bnodes + (pl->max_bnodes & 1);
    a.max_chunks = pl->max_block_chunks;
    a.ntcols = d + (a.lam.type == TGK_FIELD_NODAL) + (a.mu.type == TGK_FIELD_NODAL);
    for (int c = 0; c < a.n_src; ++c) a.ntcols += a.src[c].type == TGK_FIELD_NODAL;
    unsigned long long* badp = nullptr;  // the routing's persistent status words
    TGK_TRY(routing_flags(r, &badp));
    CUDA_TRY(cudaMemsetAsync(badp, 0xff, 2 * sizeof(unsigned long long), st));
    a.bad = badp;
    if (R2 == 16) {
        if (m->kind == TGK_TET4)
            TGK_TRY((high ? launch_elast2<TGK_TET4, 2, 16>(a, pl->n_blocks, st) : launch_elast2<TGK_TET4, 1, 16>(a, pl->n_blocks, st)));
        else
            TGK_TRY((high ? launch_elast2<TGK_TRI3, 2, 16>(a, pl->n_blocks, st) : launch_elast2<TGK_TRI3, 1, 16>(a, pl->n_blocks, st)));
    } else {
        if (m->kind == TGK_TET4)
            TGK_TRY((high ? launch_elast2<TGK_TET4, 2, 32>(a, pl->n_blocks, st) : launch_elast2<TGK_TET4, 1, 32>(a, pl->n_blocks, st)));
        else
            TGK_TRY((high ? launch_elast2<TGK_TRI3, 2, 32>(a, pl->n_blocks, st) : launch_elast2<TGK_TRI3, 1, 32>(a, pl->n_blocks, st)));
    }
    unsigned long long h[2] = {ULLONG_MAX, ULLONG_MAX};
    CUDA_TRY(cudaMemcpyAsync(h, badp, sizeof h, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    // batch_geometry runs (and throws) before local_stiffness_elasticity checks mu (physics.cpp:11-52)
    if (h[0] != ULLONG_MAX)
        return set_error(TGK_ERR_INPUT, "element " + std::to_string(h[0]) + " has non-positive Jacobian determinant");
    if (h[1] != ULLONG_MAX) return set_error(TGK_ERR_INPUT, "elasticity requires mu > 0");
    return TGK_OK;
}

}  // namespace tgk
