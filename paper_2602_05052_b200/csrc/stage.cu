// Materialised Stage I (Map) and Stage II (Reduce) kernels: the drop-in for
// the reference's public batch.hpp / routing.hpp functions that hand whole
// E x ... arrays across the API (batch.cpp:56-312, routing.cpp:87-125).  The
// fused path (fused.cu) never materialises these; they exist for API parity
// and for the parity tests of each stage.
//
// Arithmetic follows the reference literally (FMA disabled), one thread per
// element (Map) or per output (Reduce, ascending-slot left fold).
#include <algorithm>
#include <climits>

#include "cuda_util.cuh"
#include "element.cuh"
#include "tgk_internal.hpp"

namespace tgk {

__device__ __forceinline__ void flag_bad(unsigned long long* bad, int64_t e) {
    atomicMin(bad, static_cast<unsigned long long>(e));
}

// Host-side bad-element check after a kernel (batch.cpp:124-126 message).
int check_bad(unsigned long long* d_bad, cudaStream_t st) {
    unsigned long long h = ULLONG_MAX;
    CUDA_TRY(cudaMemcpyAsync(&h, d_bad, sizeof h, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (h != ULLONG_MAX)
        return set_error(TGK_ERR_INPUT, "element " + std::to_string(h) +
                                            " has non-positive Jacobian determinant");
    return TGK_OK;
}

namespace {

template <int KIND>
__device__ __forceinline__ void load_element(const double* nodes, const int32_t* conn, int64_t e,
                                             double (&X)[P1<KIND>::k][P1<KIND>::d]) {
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d;
#pragma unroll
    for (int a = 0; a < k; ++a) {
        const int64_t n = conn[e * k + a];
#pragma unroll
        for (int c = 0; c < d; ++c) X[a][c] = nodes[n * d + c];
    }
}

// batch_geometry + push_forward, literal reference sequence (batch.cpp:76-152)
template <int KIND, int DEG>
__global__ void k_geometry(const double* nodes, const int32_t* conn, int64_t E, double* jac,
                           double* det_out, double* jinv, double* qpts, double* grads,
                           unsigned long long* bad) {
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    double X[k][d];
    load_element<KIND>(nodes, conn, e, X);
    // reference gradients Ghat (reference.cpp:59-71)
    auto ghat = [](int a, int j) -> double { return a == 0 ? -1.0 : (j == a - 1 ? 1.0 : 0.0); };
    double J[d * d];
#pragma unroll
    for (int i = 0; i < d * d; ++i) J[i] = 0.0;
#pragma unroll
    for (int a = 0; a < k; ++a)
#pragma unroll
        for (int i = 0; i < d; ++i)
#pragma unroll
            for (int j = 0; j < d; ++j) J[i * d + j] += X[a][i] * ghat(a, j);
    double det;
    double T[d * d];
    if constexpr (d == 2) {
        det = J[0] * J[3] - J[1] * J[2];
        T[0] = J[3] / det; T[1] = -J[2] / det; T[2] = -J[1] / det; T[3] = J[0] / det;
    } else {
        det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
              J[2] * (J[3] * J[7] - J[4] * J[6]);
        const double c00 = J[4] * J[8] - J[5] * J[7];
        const double c01 = J[5] * J[6] - J[3] * J[8];
        const double c02 = J[3] * J[7] - J[4] * J[6];
        const double c10 = J[2] * J[7] - J[1] * J[8];
        const double c11 = J[0] * J[8] - J[2] * J[6];
        const double c12 = J[1] * J[6] - J[0] * J[7];
        const double c20 = J[1] * J[5] - J[2] * J[4];
        const double c21 = J[2] * J[3] - J[0] * J[5];
        const double c22 = J[0] * J[4] - J[1] * J[3];
        T[0] = c00 / det; T[1] = c01 / det; T[2] = c02 / det;
        T[3] = c10 / det; T[4] = c11 / det; T[5] = c12 / det;
        T[6] = c20 / det; T[7] = c21 / det; T[8] = c22 / det;
    }
    if (det <= 0.0) flag_bad(bad, e);
    double G[k * d];
#pragma unroll
    for (int a = 0; a < k; ++a)
#pragma unroll
        for (int i = 0; i < d; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < d; ++j) s += T[i * d + j] * ghat(a, j);
            G[a * d + i] = s;
        }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int64_t eq = e * Q + q;
        if (jac)
            for (int i = 0; i < d * d; ++i) jac[eq * d * d + i] = J[i];
        if (det_out) det_out[eq] = det;
        if (jinv)
            for (int i = 0; i < d * d; ++i) jinv[eq * d * d + i] = T[i];
        if (qpts)
#pragma unroll
            for (int c = 0; c < d; ++c) {
                double x = 0.0;
#pragma unroll
                for (int a = 0; a < k; ++a) x += basis<KIND, DEG>(q, a) * X[a][c];
                qpts[eq * d + c] = x;
            }
        if (grads)
            for (int i = 0; i < k * d; ++i) grads[eq * k * d + i] = G[i];
    }
}

// local kernels (batch.cpp:156-312); `what` as tgk_local_* entry points
enum { L_DIFF = 0, L_ELAST = 1, L_MASS = 2, L_LOAD = 3, L_LOADV = 4 };

template <int KIND, int DEG, int WHAT>
__global__ void k_local(const double* nodes, const int32_t* conn, int64_t E, const double* c1,
                        const double* c2, double* out, unsigned long long* bad) {
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    using R = Rule<KIND, DEG>;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    double X[k][d];
    load_element<KIND>(nodes, conn, e, X);
    double det;
    double G[k][d];
    if (!simplex_geometry<KIND>(X, det, G)) {
        flag_bad(bad, e);
        return;
    }
    if constexpr (WHAT == L_DIFF) {
        double Ke[k * k];
#pragma unroll
        for (int i = 0; i < k * k; ++i) Ke[i] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const double scale = R::w(q) * det * c1[e * Q + q];
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int b = 0; b < k; ++b) Ke[a * k + b] += scale * gdot<KIND>(G, a, b);
        }
        for (int i = 0; i < k * k; ++i) out[e * k * k + i] = Ke[i];
    } else if constexpr (WHAT == L_MASS) {
        double Me[k * k];
#pragma unroll
        for (int i = 0; i < k * k; ++i) Me[i] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const double scale = R::w(q) * det * c1[e * Q + q];
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int b = 0; b < k; ++b)
                    Me[a * k + b] += scale * basis<KIND, DEG>(q, a) * basis<KIND, DEG>(q, b);
        }
        for (int i = 0; i < k * k; ++i) out[e * k * k + i] = Me[i];
    } else if constexpr (WHAT == L_LOAD) {
        double Fe[k];
#pragma unroll
        for (int a = 0; a < k; ++a) Fe[a] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const double scale = R::w(q) * det * c1[e * Q + q];
#pragma unroll
            for (int a = 0; a < k; ++a) Fe[a] += scale * basis<KIND, DEG>(q, a);
        }
        for (int a = 0; a < k; ++a) out[e * k + a] = Fe[a];
    } else if constexpr (WHAT == L_LOADV) {
        double Fe[k * d];
#pragma unroll
        for (int a = 0; a < k * d; ++a) Fe[a] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const double scale = R::w(q) * det;
#pragma unroll
            for (int a = 0; a < k; ++a)
#pragma unroll
                for (int c = 0; c < d; ++c)
                    Fe[a * d + c] += scale * basis<KIND, DEG>(q, a) * c1[(e * Q + q) * d + c];
        }
        for (int a = 0; a < k * d; ++a) out[e * k * d + a] = Fe[a];
    } else {  // L_ELAST: batch.cpp:198-246, literal (B and DB with their zeros)
        constexpr int kk = k * d, ns = d == 2 ? 3 : 6;
        double* Ke = out + e * kk * kk;
        for (int i = 0; i < kk * kk; ++i) Ke[i] = 0.0;
        for (int q = 0; q < Q; ++q) {
            double B[ns * kk], DB[ns * kk];
            for (int i = 0; i < ns * kk; ++i) B[i] = 0.0;
            if constexpr (d == 2) {
                for (int a = 0; a < k; ++a) {
                    const double gx = G[a][0], gy = G[a][1];
                    B[0 * kk + a * 2 + 0] = gx;
                    B[1 * kk + a * 2 + 1] = gy;
                    B[2 * kk + a * 2 + 0] = gy;
                    B[2 * kk + a * 2 + 1] = gx;
                }
            } else {
                for (int a = 0; a < k; ++a) {
                    const double gx = G[a][0], gy = G[a][1], gz = G[a][2];
                    B[0 * kk + a * 3 + 0] = gx;
                    B[1 * kk + a * 3 + 1] = gy;
                    B[2 * kk + a * 3 + 2] = gz;
                    B[3 * kk + a * 3 + 0] = gy;
                    B[3 * kk + a * 3 + 1] = gx;
                    B[4 * kk + a * 3 + 1] = gz;
                    B[4 * kk + a * 3 + 2] = gy;
                    B[5 * kk + a * 3 + 0] = gz;
                    B[5 * kk + a * 3 + 2] = gx;
                }
            }
            const double lam = c1[e * Q + q], mu = c2[e * Q + q];
            for (int col = 0; col < kk; ++col) {
                double tr = 0.0;
                for (int i = 0; i < d; ++i) tr += B[i * kk + col];
                for (int i = 0; i < d; ++i) DB[i * kk + col] = lam * tr + 2.0 * mu * B[i * kk + col];
                for (int i = d; i < ns; ++i) DB[i * kk + col] = mu * B[i * kk + col];
            }
            const double scale = R::w(q) * det;
            for (int a = 0; a < kk; ++a)
                for (int b = 0; b < kk; ++b) {
                    double s = 0.0;
                    for (int i = 0; i < ns; ++i) s += B[i * kk + a] * DB[i * kk + b];
                    Ke[a * kk + b] += scale * s;
                }
        }
    }
}


// ------------------------------------------------------------------ elasticity local kernel
// local_stiffness_elasticity (batch.cpp:183-248) with the reference's
// operation order but only over the STRUCTURAL nonzeros of the Voigt B and
// D*B (batch.cpp:205-236): every skipped term is a product with an exact
// structural zero (+-0.0), and adding +-0.0 to a partial sum that starts at
// +0.0 never changes it, so all values are bit-identical to the literal loop.
// Warp per 32 elements; each row of K_e is staged in shared memory and written
// by the warp as contiguous runs (coalesced element-major output).
template <int D>
__host__ __device__ constexpr int bcomp(int i, int c) {
    // gradient component carried by B[i][a*D + c] (Voigt row i), -1 if structurally zero
    if (D == 3) {
        return i == 0 ? (c == 0 ? 0 : -1)
             : i == 1 ? (c == 1 ? 1 : -1)
             : i == 2 ? (c == 2 ? 2 : -1)
             : i == 3 ? (c == 0 ? 1 : (c == 1 ? 0 : -1))   // gamma_xy
             : i == 4 ? (c == 1 ? 2 : (c == 2 ? 1 : -1))   // gamma_yz
             : (c == 0 ? 2 : (c == 2 ? 0 : -1));           // gamma_xz
    }
    return i == 0 ? (c == 0 ? 0 : -1) : i == 1 ? (c == 1 ? 1 : -1) : (c == 0 ? 1 : (c == 1 ? 0 : -1));
}

template <int KIND, int DEG>
__global__ void __launch_bounds__(32) k_local_elasticity(const double* nodes, const int32_t* conn, int64_t E,
                                                         const double* lam_eq, const double* mu_eq, double* out,
                                                         unsigned long long* bad) {
    constexpr int k = P1<KIND>::k, d = P1<KIND>::d, Q = Rule<KIND, DEG>::Q;
    constexpr int kk = k * d, ns = d == 2 ? 3 : 6;
    using R = Rule<KIND, DEG>;
    __shared__ double tile[32 * (kk + 1)];
    const int lane = threadIdx.x;
    const int64_t e0 = int64_t(blockIdx.x) * 32;
    const int64_t e = e0 + lane;
    const bool valid = e < E;
    double G[k][d];
    double det = 0.0;
    bool ok = false;
    if (valid) {
        double X[k][d];
        load_element<KIND>(nodes, conn, e, X);
        ok = simplex_geometry<KIND>(X, det, G);
        if (!ok) flag_bad(bad, e);
    }
    if (!ok) {
#pragma unroll
        for (int a = 0; a < k; ++a)
#pragma unroll
            for (int c = 0; c < d; ++c) G[a][c] = 0.0;
    }
    const int nvalid = E - e0 < 32 ? static_cast<int>(E - e0) : 32;
#pragma unroll
    for (int ar = 0; ar < kk; ++ar) {
        const int a = ar / d, c = ar % d;  // compile-time after unrolling
        double row[kk];
#pragma unroll
        for (int j = 0; j < kk; ++j) row[j] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const double lam = valid ? lam_eq[e * Q + q] : 0.0;
            const double mu = valid ? mu_eq[e * Q + q] : 1.0;
            const double two_mu = 2.0 * mu;
            const double scale = R::w(q) * det;
#pragma unroll
            for (int b = 0; b < k; ++b)
#pragma unroll
                for (int cp = 0; cp < d; ++cp) {
                    const double g = G[b][cp];
                    const double tr = 0.0 + g;  // the column's only normal entry (batch.cpp:232)
                    double s = 0.0;
#pragma unroll
                    for (int i = 0; i < ns; ++i) {
                        const int ga = bcomp<d>(i, c);
                        if (ga < 0) continue;  // B[i][a*d+c] structurally zero
                        const double Ba = G[a][ga];
                        double DB;
                        if (i < d) {
                            DB = i == cp ? lam * tr + two_mu * g : lam * tr + two_mu * 0.0;  // batch.cpp:233
                        } else {
                            const int gb = bcomp<d>(i, cp);
                            if (gb < 0) continue;  // mu * 0.0 (batch.cpp:234)
                            DB = mu * G[b][gb];
                        }
                        s += Ba * DB;
                    }
                    row[b * d + cp] += scale * s;  // batch.cpp:240-242
                }
        }
#pragma unroll
        for (int j = 0; j < kk; ++j) tile[lane * (kk + 1) + j] = row[j];
        __syncwarp();
        // coalesced store of row ar of the warp's (up to) 32 elements
        for (int f = lane; f < nvalid * kk; f += 32) {
            const int el = f / kk, col = f % kk;
            out[(e0 + el) * kk * kk + ar * kk + col] = tile[el * (kk + 1) + col];
        }
        __syncwarp();
    }
}

// CoefficientField::evaluate (coefficient.cpp:34-55) -> E x Q
template <int KIND, int DEG>
__global__ void k_evaluate(const int32_t* conn, int64_t E, int type, double value,
                           const double* data, double* out) {
    constexpr int k = P1<KIND>::k, Q = Rule<KIND, DEG>::Q;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        double v;
        if (type == TGK_FIELD_CONSTANT) {
            v = value;
        } else if (type == TGK_FIELD_ELEMENT) {
            v = data[e];
        } else {  // interpolate_nodal (batch.cpp:321-330)
            v = 0.0;
#pragma unroll
            for (int a = 0; a < k; ++a) v += basis<KIND, DEG>(q, a) * data[conn[e * k + a]];
        }
        out[e * Q + q] = v;
    }
}

// reduce_matrix / reduce_vector (routing.cpp:92-99, 117-124)
// (left fold from +0.0 in ascending slot order; the gathers of up to four
// contributions are issued before their adds, so each thread keeps four
// independent loads in flight instead of a dependent chain.  Staging a
// block's whole slot range in shared memory first measured slower: 44.0 vs
// 39.7 us on the RM workload.)
constexpr int kSegThreads = 256;
__global__ void k_segment_reduce(const uint32_t* __restrict__ off, const uint32_t* __restrict__ slots, int64_t n,
                                 const double* __restrict__ local, double* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t u1 = __ldg(off + t + 1);
    uint32_t u = __ldg(off + t);
    double s = 0.0;
    for (; u + 4 <= u1; u += 4) {
        const uint32_t a0 = __ldg(slots + u), a1 = __ldg(slots + u + 1), a2 = __ldg(slots + u + 2),
                       a3 = __ldg(slots + u + 3);
        const double v0 = __ldg(local + a0), v1 = __ldg(local + a1), v2 = __ldg(local + a2), v3 = __ldg(local + a3);
        s += v0;
        s += v1;
        s += v2;
        s += v3;
    }
    if (u + 2 <= u1) {
        const uint32_t a0 = __ldg(slots + u), a1 = __ldg(slots + u + 1);
        const double v0 = __ldg(local + a0), v1 = __ldg(local + a1);
        s += v0;
        s += v1;
        u += 2;
    }
    if (u < u1) s += __ldg(local + __ldg(slots + u));
    out[t] = s;
}

template <int KIND, template <int, int> class Launch, class... Args>
int dispatch_degree(int degree, Args... args) {
    switch (degree) {
        case 1: return Launch<KIND, 1>::run(args...);
        case 2: return Launch<KIND, 2>::run(args...);
        case 3: return Launch<KIND, 3>::run(args...);
        case 4: return Launch<KIND, 4>::run(args...);
    }
    return set_error(TGK_ERR_INPUT, "quadrature degree " + std::to_string(degree) +
                                        " unsupported; supported degrees: 1,2,3,4");
}

template <int KIND, int DEG>
struct GeomLaunch {
    static int run(const tgk_mesh* m, double* jac, double* det, double* jinv, double* qp,
                   double* gr, unsigned long long* bad, cudaStream_t st) {
        k_geometry<KIND, DEG><<<grid_for(m->E, 128), 128, 0, st>>>(m->nodes, m->conn, m->E, jac, det,
                                                                  jinv, qp, gr, bad);
        KERNEL_CHECK("geometry");
        return TGK_OK;
    }
};

template <int WHAT>
struct LocalOf {
    template <int KIND, int DEG>
    struct L {
        static int run(const tgk_mesh* m, const double* c1, const double* c2, double* out,
                       unsigned long long* bad, cudaStream_t st) {
            if constexpr (WHAT == L_ELAST) {
                k_local_elasticity<KIND, DEG><<<grid_for(m->E, 32), 32, 0, st>>>(m->nodes, m->conn, m->E, c1, c2,
                                                                                  out, bad);
                KERNEL_CHECK("local_elasticity");
                return TGK_OK;
            }
            k_local<KIND, DEG, WHAT><<<grid_for(m->E, 128), 128, 0, st>>>(m->nodes, m->conn, m->E,
                                                                         c1, c2, out, bad);
            KERNEL_CHECK("local");
            return TGK_OK;
        }
    };
};

template <int KIND, int DEG>
struct EvalLaunch {
    static int run(const tgk_mesh* m, const tgk_field* f, double* out, cudaStream_t st) {
        k_evaluate<KIND, DEG><<<grid_for(m->E, 256), 256, 0, st>>>(m->conn, m->E, f->type, f->value,
                                                                  f->data, out);
        KERNEL_CHECK("evaluate");
        return TGK_OK;
    }
};

int check_mesh(const tgk_mesh* m) {
    if (!m) return set_error(TGK_ERR_INPUT, "null mesh");
    if (m->kind != TGK_TRI3 && m->kind != TGK_TET4)
        return set_error(TGK_ERR_INPUT, "P1 kernels support TRI3 and TET4 meshes only");
    return ensure_device();
}

template <int WHAT>
int run_local(const tgk_mesh* m, int degree, const double* c1, const double* c2, double* out,
              void* stream) {
    TGK_TRY(check_mesh(m));
    cudaStream_t st = as_stream(stream);
    DevBuf<unsigned long long> bad;
    TGK_TRY(bad.alloc(1));
    CUDA_TRY(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    if (m->kind == TGK_TET4)
        TGK_TRY((dispatch_degree<TGK_TET4, LocalOf<WHAT>::template L>(degree, m, c1, c2, out, bad.p, st)));
    else
        TGK_TRY((dispatch_degree<TGK_TRI3, LocalOf<WHAT>::template L>(degree, m, c1, c2, out, bad.p, st)));
    return check_bad(bad.p, st);
}

// int64 -> int32 connectivity with the range check of mesh.cpp:61-64; also
// records whether any entry differs from the previous contents (`changed`).
__device__ __forceinline__ int32_t narrow_one(int64_t v, int64_t i, int64_t n_nodes, unsigned long long* bad) {
    const bool out = v < 0 || v >= n_nodes;
    if (out) atomicMin(bad, static_cast<unsigned long long>(i));
    return out ? 0 : static_cast<int32_t>(v);  // never an out-of-range node id on the device
}

// int64 -> int32 connectivity with the range check (mesh.cpp:61-64) and change
// detection; 16-byte loads / stores, four entries per thread and iteration,
// no data-dependent branch in the streaming loop
__global__ void k_narrow(const int64_t* __restrict__ src, int64_t n, int64_t n_nodes, int32_t* __restrict__ dst,
                         unsigned long long* bad, unsigned long long* changed, int vec) {
    unsigned diff = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n4 = vec ? n / 4 : 0;
    for (int64_t q = t0; q < n4; q += stride) {
        const longlong2 a = reinterpret_cast<const longlong2*>(src)[2 * q];
        const longlong2 b = reinterpret_cast<const longlong2*>(src)[2 * q + 1];
        const int4 old = reinterpret_cast<const int4*>(dst)[q];
        int4 w;
        w.x = narrow_one(a.x, 4 * q, n_nodes, bad);
        w.y = narrow_one(a.y, 4 * q + 1, n_nodes, bad);
        w.z = narrow_one(b.x, 4 * q + 2, n_nodes, bad);
        w.w = narrow_one(b.y, 4 * q + 3, n_nodes, bad);
        diff |= unsigned(w.x != old.x) | unsigned(w.y != old.y) | unsigned(w.z != old.z) | unsigned(w.w != old.w);
        reinterpret_cast<int4*>(dst)[q] = w;
    }
    for (int64_t i = 4 * n4 + t0; i < n; i += stride) {
        const int32_t w = narrow_one(src[i], i, n_nodes, bad);
        diff |= unsigned(dst[i] != w);
        dst[i] = w;
    }
    if (__any_sync(0xffffffffu, diff != 0) && (threadIdx.x & 31) == 0) atomicOr(changed, 1ull);
}

}  // namespace

// local_stiffness_elasticity without the host-side mu check (the caller checked mu on the device)
int local_elasticity_nocheck(const tgk_mesh* m, int degree, const double* lam, const double* mu, double* out,
                             cudaStream_t st) {
    return run_local<L_ELAST>(m, degree, lam, mu, out, st);
}

// Cached device scratch of a routing handle (slot < 6, grows on demand).
int routing_scratch(tgk_routing* r, int slot, size_t n, double** out) {
    if (r->scr_n[slot] < n) {
        if (r->scr[slot]) cudaFree(r->scr[slot]);
        r->scr[slot] = nullptr;
        r->scr_n[slot] = 0;
        CUDA_TRY(cudaMalloc(&r->scr[slot], sizeof(double) * std::max<size_t>(1, n)));
        r->scr_n[slot] = n;
    }
    *out = r->scr[slot];
    return TGK_OK;
}

// Division-safety certificate of a mesh (element.cuh ExactDiv): every
// coordinate is 0 or has 2^-40 <= |x| <= 2^40.
__global__ void k_coord_range(const double* x, int64_t n, unsigned* bad) {
    unsigned b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double a = fabs(x[i]);
        b |= (a != 0.0 && (a < 0x1p-40 || a > 0x1p40)) ? 1u : 0u;  // NaN/inf: > fails, < fails...
        b |= (a != a || a == __longlong_as_double(0x7ff0000000000000ll)) ? 1u : 0u;
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// Persistent per-mesh flag words (device + pinned host), allocated on first use.
// [0] coordinate certification, [1] / [2] first bad entry / changed of the
// blocking upload, [3] / [4] the same accumulated by asynchronous uploads
// until tgk_mesh_upload_check
int mesh_flags(tgk_mesh* m) {
    if (!m->d_flags) {
        CUDA_TRY(cudaMalloc(&m->d_flags, 5 * sizeof(unsigned long long)));
        const unsigned long long init[5] = {0, ULLONG_MAX, 0, ULLONG_MAX, 0};
        CUDA_TRY(cudaMemcpy(m->d_flags, init, sizeof init, cudaMemcpyHostToDevice));
    }
    if (!m->h_flags) CUDA_TRY(cudaMallocHost(&m->h_flags, 5 * sizeof(unsigned long long)));
    return TGK_OK;
}

int narrow_connectivity_async(tgk_mesh* m, const int64_t* src, int64_t n, int64_t n_nodes, int32_t* dst,
                              cudaStream_t st) {
    TGK_TRY(mesh_flags(m));
    const int vec = (reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0) ? 1 : 0;
    k_narrow<<<std::min<unsigned>(grid_for(n / 4 + 1, 256), 148 * 16), 256, 0, st>>>(src, n, n_nodes, dst,
                                                                                    m->d_flags + 3, m->d_flags + 4, vec);
    KERNEL_CHECK("narrow_connectivity");
    return TGK_OK;
}

// Waits for the device, reads and resets the asynchronous upload flags.
int mesh_async_flags(tgk_mesh* m, int64_t* bad, bool* changed) {
    *bad = -1;
    *changed = false;
    if (!m->d_flags) return TGK_OK;
    CUDA_TRY(cudaDeviceSynchronize());
    unsigned long long h[2] = {ULLONG_MAX, 0};
    CUDA_TRY(cudaMemcpy(h, m->d_flags + 3, sizeof h, cudaMemcpyDeviceToHost));
    const unsigned long long init[2] = {ULLONG_MAX, 0};
    CUDA_TRY(cudaMemcpy(m->d_flags + 3, init, sizeof init, cudaMemcpyHostToDevice));
    *bad = h[0] == ULLONG_MAX ? -1 : static_cast<int64_t>(h[0]);
    *changed = h[1] != 0;
    return TGK_OK;
}

int mesh_division_safe(tgk_mesh* m, cudaStream_t st, bool* safe) {
    if (m->div_safe < 0) {
        TGK_TRY(mesh_flags(m));
        unsigned* flag = reinterpret_cast<unsigned*>(m->d_flags);
        CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(unsigned), st));
        const int64_t n = m->N * m->d;
        k_coord_range<<<std::min<unsigned>(grid_for(n, 256), 148 * 8), 256, 0, st>>>(m->nodes, n, flag);
        KERNEL_CHECK("coord_range");
        CUDA_TRY(cudaMemcpyAsync(m->h_flags, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        m->div_safe = *reinterpret_cast<unsigned*>(m->h_flags) == 0 ? 1 : 0;
    }
    *safe = m->div_safe == 1;
    return TGK_OK;
}

int narrow_connectivity(tgk_mesh* m, const int64_t* src, int64_t n, int64_t n_nodes, int32_t* dst, int64_t* bad,
                        cudaStream_t st) {
    TGK_TRY(mesh_flags(m));
    unsigned long long* flag = m->d_flags + 1;  // [1] first bad entry, [2] changed
    CUDA_TRY(cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), st));
    CUDA_TRY(cudaMemsetAsync(flag + 1, 0, sizeof(unsigned long long), st));
    const int vec = (reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0) ? 1 : 0;
    k_narrow<<<std::min<unsigned>(grid_for(n / 4 + 1, 256), 148 * 16), 256, 0, st>>>(src, n, n_nodes, dst, flag,
                                                                                    flag + 1, vec);
    KERNEL_CHECK("narrow_connectivity");
    CUDA_TRY(cudaMemcpyAsync(m->h_flags + 1, flag, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const unsigned long long h = m->h_flags[1];
    *bad = h == ULLONG_MAX ? -1 : static_cast<int64_t>(h);
    if (m->h_flags[2]) ++m->conn_version;  // routings built before refuse to assemble (check_routing_fresh)
    return TGK_OK;
}

}  // namespace tgk

extern "C" {

int tgk_geometry_d(const tgk_mesh* m, int degree, double* d_jac, double* d_det,
                   double* d_jac_invT, double* d_qpts, double* d_grads, void* stream) {
    using namespace tgk;
    TGK_TRY(check_mesh(m));
    cudaStream_t st = as_stream(stream);
    DevBuf<unsigned long long> bad;
    TGK_TRY(bad.alloc(1));
    CUDA_TRY(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    if (m->kind == TGK_TET4)
        TGK_TRY((dispatch_degree<TGK_TET4, GeomLaunch>(degree, m, d_jac, d_det, d_jac_invT, d_qpts,
                                                       d_grads, bad.p, st)));
    else
        TGK_TRY((dispatch_degree<TGK_TRI3, GeomLaunch>(degree, m, d_jac, d_det, d_jac_invT, d_qpts,
                                                       d_grads, bad.p, st)));
    return check_bad(bad.p, st);
}

int tgk_local_stiffness_diffusion_d(const tgk_mesh* m, int degree, const double* c, double* out,
                                    void* stream) {
    return tgk::run_local<tgk::L_DIFF>(m, degree, c, nullptr, out, stream);
}

int tgk_local_stiffness_elasticity_d(const tgk_mesh* m, int degree, const double* lam,
                                     const double* mu, double* out, void* stream) {
    using namespace tgk;
    TGK_TRY(check_mesh(m));
    // batch.cpp:194-195: mu <= 0 anywhere is an input error
    const int64_t n = m->E * (m->kind == TGK_TET4 ? (degree == 1 ? 1 : degree == 2 ? 4 : degree == 3 ? 5 : 11)
                                                   : (degree == 1 ? 1 : degree == 2 ? 3 : degree == 3 ? 4 : 6));
    std::vector<double> h(n);
    CUDA_TRY(cudaMemcpy(h.data(), mu, n * sizeof(double), cudaMemcpyDeviceToHost));
    for (double v : h)
        if (v <= 0.0) return set_error(TGK_ERR_INPUT, "elasticity requires mu > 0");
    return run_local<L_ELAST>(m, degree, lam, mu, out, stream);
}

int tgk_local_mass_d(const tgk_mesh* m, int degree, const double* c, double* out, void* stream) {
    return tgk::run_local<tgk::L_MASS>(m, degree, c, nullptr, out, stream);
}

int tgk_local_load_d(const tgk_mesh* m, int degree, const double* src, double* out, void* stream) {
    return tgk::run_local<tgk::L_LOAD>(m, degree, src, nullptr, out, stream);
}

int tgk_local_load_vector_d(const tgk_mesh* m, int degree, const double* src, double* out,
                            void* stream) {
    return tgk::run_local<tgk::L_LOADV>(m, degree, src, nullptr, out, stream);
}

int tgk_evaluate_field_d(const tgk_mesh* m, int degree, const tgk_field* f, double* out,
                         void* stream) {
    using namespace tgk;
    TGK_TRY(check_mesh(m));
    if (!f) return set_error(TGK_ERR_INPUT, "null field");
    if (f->type == TGK_FIELD_ELEMENT && f->n != m->E)
        return set_error(TGK_ERR_INPUT, "per-element coefficient: expected " + std::to_string(m->E) +
                                            " values, got " + std::to_string(f->n));
    if (f->type == TGK_FIELD_NODAL && f->n != m->N)
        return set_error(TGK_ERR_INPUT, "nodal field: expected " + std::to_string(m->N) +
                                            " values, got " + std::to_string(f->n));
    cudaStream_t st = as_stream(stream);
    if (f->type == TGK_FIELD_QUAD) {  // already at the quadrature points: E x Q copy
        int Q = 0;
        TGK_TRY(tgk_tables(m->kind, degree, &Q, nullptr, nullptr, nullptr, nullptr));
        if (f->n != m->E * Q)
            return set_error(TGK_ERR_INPUT, "quadrature table: expected E x Q = " + std::to_string(m->E * Q) +
                                                " values, got " + std::to_string(f->n));
        CUDA_TRY(cudaMemcpyAsync(out, f->data, sizeof(double) * f->n, cudaMemcpyDeviceToDevice, st));
        return TGK_OK;
    }
    if (m->kind == TGK_TET4)
        TGK_TRY((dispatch_degree<TGK_TET4, EvalLaunch>(degree, m, f, out, st)));
    else
        TGK_TRY((dispatch_degree<TGK_TRI3, EvalLaunch>(degree, m, f, out, st)));
    return TGK_OK;
}

int tgk_reduce_matrix_d(const tgk_routing* r, const double* local, double* values, void* stream) {
    using namespace tgk;
    if (!r || !r->mat_offsets)
        return set_error(TGK_ERR_INPUT, "reduce_matrix: routing built without TGK_ROUTING_SEGMENTS");
    TGK_TRY(ensure_device());
    k_segment_reduce<<<grid_for(r->nnz, kSegThreads), kSegThreads, 0, as_stream(stream)>>>(
        r->mat_offsets, r->mat_slots, r->nnz, local, values);
    KERNEL_CHECK("reduce_matrix");
    return TGK_OK;
}

int tgk_reduce_vector_d(const tgk_routing* r, const double* local, double* F, void* stream) {
    using namespace tgk;
    if (!r || !r->vec_offsets)
        return set_error(TGK_ERR_INPUT, "reduce_vector: routing built without TGK_ROUTING_SEGMENTS");
    TGK_TRY(ensure_device());
    k_segment_reduce<<<grid_for(r->N, kSegThreads), kSegThreads, 0, as_stream(stream)>>>(r->vec_offsets, r->vec_slots,
                                                                                       r->N, local, F);
    KERNEL_CHECK("reduce_vector");
    return TGK_OK;
}

}  // extern "C"

namespace tgk {
namespace {
// Interface-row sum of the multi-GPU exchange: values = lower + values
// (lower: the partial fold of the rank below = elements with smaller ids).
__global__ void k_interface_combine(const double* lower, double* values, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        values[i] = lower[i] + values[i];
}
}  // namespace
}  // namespace tgk

extern "C" int tgk_interface_combine_d(const double* d_lower, double* d_values, int64_t n, void* stream) {
    using namespace tgk;
    if (n < 0 || (n > 0 && (!d_lower || !d_values))) return set_error(TGK_ERR_INPUT, "interface_combine: bad arguments");
    TGK_TRY(ensure_device());
    if (n == 0) return TGK_OK;
    k_interface_combine<<<std::min<unsigned>(grid_for(n, 256), 148 * 8), 256, 0, as_stream(stream)>>>(d_lower, d_values, n);
    KERNEL_CHECK("interface_combine");
    return TGK_OK;
}
