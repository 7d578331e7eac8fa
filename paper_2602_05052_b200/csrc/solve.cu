// The first consumers of the assembled CSR, kept on the device (SURVEY.md
// 8(f) ranks 2-3): SparseOperator::apply (sparse.cpp:18-31), Dirichlet
// condensation condense (solver.cpp:34-85) with restrict_to_free
// (solver.cpp:87-103) and CondensedSystem::expand (solver.cpp:20-26).
// Every output value is produced by one thread in the reference's order (a
// row's products summed from +0.0 in column order; the condensed right-hand
// side corrected by the fixed columns in column order), so results are
// bit-identical to the reference.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>

#include "cuda_util.cuh"
#include "tgk_internal.hpp"

struct tgk_condensed {
    int64_t full_size = 0, n_free = 0, n_fixed = 0, nnz_ff = 0;
    int64_t* free_dofs = nullptr;   // n_free, ascending
    int64_t* fixed_dofs = nullptr;  // n_fixed, ascending
    double* prescribed = nullptr;   // n_fixed
    int64_t* offsets = nullptr;     // n_free + 1 (K_ff pattern)
    int64_t* cols = nullptr;        // nnz_ff
    double* values = nullptr;       // nnz_ff
    double* F_f = nullptr;          // n_free
    unsigned char* fixed = nullptr; // full_size
    double* g = nullptr;            // full_size prescribed values (0 on free DoFs)
    ~tgk_condensed() {
        for (void* p : {(void*)free_dofs, (void*)fixed_dofs, (void*)prescribed, (void*)offsets, (void*)cols,
                        (void*)values, (void*)F_f, (void*)fixed, (void*)g})
            if (p) cudaFree(p);
    }
};

namespace tgk {
namespace {

// y = A x, one row per thread (sparse.cpp:23-29)
__global__ void k_spmv(int64_t rows, const int64_t* off, const int64_t* cols, const double* vals, const double* x,
                       double* y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t t = off[i]; t < off[i + 1]; ++t) s += vals[t] * x[cols[t]];
        y[i] = s;
    }
}

// last occurrence wins (solver.cpp:42-47 assigns in list order)
__global__ void k_mark_last(const int64_t* dofs, int64_t n, int64_t N, unsigned long long* win, int* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = dofs[i];
        if (d < 0 || d >= N) {
            atomicExch(bad, 1);
            continue;
        }
        atomicMax(win + d, static_cast<unsigned long long>(i + 1));
    }
}

__global__ void k_fix(const unsigned long long* win, const double* vals, int64_t N, unsigned char* fixed, double* g,
                      int64_t* is_free, int64_t* is_fixed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long w = win[i];
        fixed[i] = w ? 1 : 0;
        g[i] = w ? vals[w - 1] : 0.0;
        is_free[i] = w ? 0 : 1;
        is_fixed[i] = w ? 1 : 0;
    }
}

__global__ void k_lists(int64_t N, const unsigned char* fixed, const double* g, const int64_t* free_index,
                        const int64_t* fixed_index, int64_t* free_dofs, int64_t* fixed_dofs, double* prescribed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (fixed[i]) {
            fixed_dofs[fixed_index[i]] = i;
            prescribed[fixed_index[i]] = g[i];
        } else {
            free_dofs[free_index[i]] = i;
        }
    }
}

__global__ void k_count_free(int64_t n_free, const int64_t* free_dofs, const int64_t* off, const int64_t* cols,
                             const unsigned char* fixed, int64_t* cnt) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_free; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = free_dofs[f];
        int64_t c = 0;
        for (int64_t t = off[i]; t < off[i + 1]; ++t) c += fixed[cols[t]] ? 0 : 1;
        cnt[f] = c;
    }
}

// condense (solver.cpp:65-81): free columns re-indexed, F_f = F_i - sum K_ij g_j over fixed j
__global__ void k_fill(int64_t n_free, const int64_t* free_dofs, const int64_t* off, const int64_t* cols,
                       const double* K, const double* F, const unsigned char* fixed, const double* g,
                       const int64_t* free_index, const int64_t* off_ff, int64_t* cols_ff, double* vals_ff,
                       double* F_f) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_free; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = free_dofs[f];
        double rhs = F[i];
        int64_t o = off_ff[f];
        for (int64_t t = off[i]; t < off[i + 1]; ++t) {
            const int64_t j = cols[t];
            if (fixed[j]) {
                rhs -= K[t] * g[j];
            } else {
                cols_ff[o] = free_index[j];
                vals_ff[o] = K[t];
                ++o;
            }
        }
        F_f[f] = rhs;
    }
}

// restrict_to_free (solver.cpp:96-99)
__global__ void k_restrict(int64_t n_free, const int64_t* free_dofs, const int64_t* off, const int64_t* cols,
                           const double* A, const unsigned char* fixed, const int64_t* off_ff, double* out) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_free; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = free_dofs[f];
        int64_t o = off_ff[f];
        for (int64_t t = off[i]; t < off[i + 1]; ++t)
            if (!fixed[cols[t]]) out[o++] = A[t];
    }
}

// CondensedSystem::expand (solver.cpp:20-26)
__global__ void k_expand(int64_t n_free, const int64_t* free_dofs, const double* u_free, int64_t n_fixed,
                         const int64_t* fixed_dofs, const double* prescribed, double* u) {
    const int64_t n = n_free > n_fixed ? n_free : n_fixed;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n_free) u[free_dofs[i]] = u_free[i];
        if (i < n_fixed) u[fixed_dofs[i]] = prescribed[i];
    }
}


// ------------------------------------------------------------------ BiCGSTAB (solver.cpp:105-227)
constexpr int kDotBlocks = 296, kDotThreads = 256;

// Deterministic dot product: fixed grid, fixed per-thread ranges, fixed tree
// orders (the reference uses a serial left fold, solver.cpp:11-16; results
// agree to rounding, run-to-run bitwise reproducible here).
__global__ void k_dot_partial(const double* a, const double* b, int64_t n, double* part) {
    __shared__ double sh[kDotThreads];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kDotThreads + threadIdx.x; i < n; i += (int64_t)kDotBlocks * kDotThreads)
        s += a[i] * b[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kDotThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
// two dot products in one pass (a.b, c.d), each with k_dot_partial's exact
// partition and tree order (bitwise equal to two separate calls)
__global__ void k_dot2_partial(const double* a, const double* b, const double* c, const double* d, int64_t n,
                               double* part) {
    __shared__ double sh[2][kDotThreads];
    double s0 = 0.0, s1 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kDotThreads + threadIdx.x; i < n; i += (int64_t)kDotBlocks * kDotThreads) {
        s0 += a[i] * b[i];
        s1 += c[i] * d[i];
    }
    sh[0][threadIdx.x] = s0;
    sh[1][threadIdx.x] = s1;
    __syncthreads();
    for (int w = kDotThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sh[0][threadIdx.x] += sh[0][threadIdx.x + w];
            sh[1][threadIdx.x] += sh[1][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0][0];
        part[kDotBlocks + blockIdx.x] = sh[1][0];
    }
}
__global__ void k_dot_final(const double* part, double* out) {
    __shared__ double sh[512];
    sh[threadIdx.x] = threadIdx.x < kDotBlocks ? part[threadIdx.x] : 0.0;
    __syncthreads();
    for (int w = 256; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// SparseOperator::diagonal (sparse.cpp:50-57) -> 1 / d; flags a zero diagonal
__global__ void k_inv_diag(int64_t n, const int64_t* off, const int64_t* cols, const double* vals, double* inv,
                           int* zero) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        int64_t lo = off[i], hi = off[i + 1];
        while (lo < hi) {  // CsrPattern::find (sparse.cpp:10-16)
            const int64_t mid = (lo + hi) >> 1;
            if (cols[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo < off[i + 1] && cols[lo] == i) d = vals[lo];
        if (d == 0.0) atomicExch(zero, 1);
        inv[i] = 1.0 / d;
    }
}

// r = b - A x (+ non-finite flag)
__global__ void k_residual(int64_t n, const int64_t* off, const int64_t* cols, const double* vals, const double* x,
                           const double* b, double* r, int* nonfinite) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t t = off[i]; t < off[i + 1]; ++t) s += vals[t] * x[cols[t]];
        const double v = b[i] - s;
        if (!isfinite(v)) atomicExch(nonfinite, 1);
        r[i] = v;
    }
}

// p = r + beta (p - omega v); phat = inv_diag p
// BiCGSTAB with device-resident scalars (one host synchronisation per
// iteration): the scalars live in sc[], the iteration's exit state in *state
// (0 running, 1 converged at s, 2 breakdown before the iteration counts,
// 3 omega breakdown, 4 non-finite residual); every kernel after an exit is a
// no-op, so the host learns the outcome from one read-back at the end.
enum { S_RHO, S_ALPHA, S_OMEGA, S_BETA, S_RHONEW, S_RTV, S_SS, S_TT, S_TS, S_RR, S_RES, S_SNORM, S_COUNT };

__global__ void k_it_begin(double* sc, int* state, double eps) {  // rho_new, beta (solver.cpp:150-158)
    if (*state) return;
    const double rn = sc[S_RHONEW];
    if (!isfinite(rn) || fabs(rn) < eps) {
        *state = 2;
        return;
    }
    sc[S_BETA] = (rn / sc[S_RHO]) * (sc[S_ALPHA] / sc[S_OMEGA]);
    sc[S_RHO] = rn;
}
__global__ void k_it_alpha(double* sc, int* state) {
    if (*state) return;
    const double alpha = sc[S_RHO] / sc[S_RTV];
    if (!isfinite(alpha)) *state = 2;
    else sc[S_ALPHA] = alpha;
}
__global__ void k_it_s(double* sc, int* state, double tol) {
    if (*state) return;
    const double sn = sqrt(sc[S_SS]);
    sc[S_SNORM] = sn;
    if (sn <= tol) *state = 1;
}
__global__ void k_it_omega(double* sc, int* state, double eps) {
    if (*state) return;
    const double tt = sc[S_TT], omega = sc[S_TS] / tt;
    if (!isfinite(omega) || tt < eps) *state = 3;
    else sc[S_OMEGA] = omega;
}
__global__ void k_it_end(double* sc, int* state) {
    if (*state) return;
    const double res = sqrt(sc[S_RR]);
    sc[S_RES] = res;
    if (!isfinite(res)) *state = 4;
}
__global__ void k_bicg_p(int64_t n, const double* r, const double* v, const double* inv, const double* sc,
                         const int* state, double* p, double* phat) {
    if (*state) return;
    const double beta = sc[S_BETA], omega = sc[S_OMEGA];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double pi = r[i] + beta * (p[i] - omega * v[i]);
        p[i] = pi;
        phat[i] = inv[i] * pi;
    }
}
__global__ void k_bicg_s(int64_t n, const double* r, const double* v, const double* sc, const int* state, double* s) {
    if (*state) return;
    const double alpha = sc[S_ALPHA];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s[i] = r[i] - alpha * v[i];
}
__global__ void k_scale(int64_t n, const double* inv, const double* x, const int* state, double* y) {
    if (state && *state) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = inv[i] * x[i];
}
// x += alpha phat (+ omega shat); r = s - omega t.  stage 1 (after the s
// check): only on state 1; stage 2 (after omega): full update on state 0,
// x += alpha phat on state 3.
__global__ void k_bicg_x(int64_t n, const double* sc, const int* state, int stage, const double* phat,
                         const double* shat, const double* s, const double* t, double* x, double* r) {
    const int st = *state;
    const bool half = stage == 1 ? st == 1 : st == 3;
    const bool full = stage == 2 && st == 0;
    if (!half && !full) return;
    const double alpha = sc[S_ALPHA], omega = sc[S_OMEGA];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (full) {
            x[i] += alpha * phat[i] + omega * shat[i];
            r[i] = s[i] - omega * t[i];
        } else {
            x[i] += alpha * phat[i];
        }
    }
}

int exclusive_scan(const int64_t* in, int64_t* out, int64_t n, cudaStream_t st) {
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st));
    DevBuf<unsigned char> t;
    TGK_TRY(t.alloc(std::max<size_t>(tmp, 1)));
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, st));
    return TGK_OK;
}

unsigned grid_n(int64_t n) { return std::min<unsigned>(grid_for(n, 256), 148 * 16); }

}  // namespace
}  // namespace tgk

extern "C" {

int tgk_spmv_d(int64_t rows, const int64_t* d_offsets, const int64_t* d_cols, const double* d_values,
               const double* d_x, double* d_y, void* stream) {
    using namespace tgk;
    if (rows < 0 || (rows > 0 && (!d_offsets || !d_cols || !d_values || !d_x || !d_y)))
        return set_error(TGK_ERR_INPUT, "sparse apply: bad arguments");
    TGK_TRY(ensure_device());
    if (rows == 0) return TGK_OK;
    k_spmv<<<grid_n(rows), 256, 0, as_stream(stream)>>>(rows, d_offsets, d_cols, d_values, d_x, d_y);
    KERNEL_CHECK("spmv");
    return TGK_OK;
}

int tgk_condense_d(int64_t N, const int64_t* d_offsets, const int64_t* d_cols, const double* d_K, const double* d_F,
                   int64_t n_dirichlet, const int64_t* d_dofs, const double* d_values, void* stream,
                   tgk_condensed** out) {
    using namespace tgk;
    if (!out || N < 0 || (N > 0 && (!d_offsets || !d_cols || !d_K || !d_F)) ||
        (n_dirichlet > 0 && (!d_dofs || !d_values)))
        return set_error(TGK_ERR_INPUT, "condense: bad arguments");
    TGK_TRY(ensure_device());
    cudaStream_t st = as_stream(stream);
    auto c = new tgk_condensed();
    c->full_size = N;
    auto fail = [&](int rc) {
        delete c;
        return rc;
    };
    DevBuf<unsigned long long> win;
    DevBuf<int> bad;
    DevBuf<int64_t> is_free, is_fixed, free_index, fixed_index, cnt;
    int rc = win.alloc(std::max<int64_t>(N, 1));
    if (!rc) rc = bad.alloc(1);
    if (!rc) rc = is_free.alloc(N + 1);
    if (!rc) rc = is_fixed.alloc(N + 1);
    if (!rc) rc = free_index.alloc(N + 1);
    if (!rc) rc = fixed_index.alloc(N + 1);
    if (rc) return fail(rc);
    auto cu = [&](cudaError_t e, const char* what) { return e == cudaSuccess ? TGK_OK : cuda_fail(e, what); };
    if ((rc = cu(cudaMalloc(&c->fixed, std::max<int64_t>(N, 1)), "cudaMalloc")) ||
        (rc = cu(cudaMalloc(&c->g, sizeof(double) * std::max<int64_t>(N, 1)), "cudaMalloc")))
        return fail(rc);
    if ((rc = cu(cudaMemsetAsync(win.p, 0, sizeof(unsigned long long) * std::max<int64_t>(N, 1), st), "memset")) ||
        (rc = cu(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "memset")) ||
        (rc = cu(cudaMemsetAsync(is_free.p + N, 0, sizeof(int64_t), st), "memset")) ||
        (rc = cu(cudaMemsetAsync(is_fixed.p + N, 0, sizeof(int64_t), st), "memset")))
        return fail(rc);
    if (n_dirichlet > 0) k_mark_last<<<grid_n(n_dirichlet), 256, 0, st>>>(d_dofs, n_dirichlet, N, win.p, bad.p);
    if (N > 0) k_fix<<<grid_n(N), 256, 0, st>>>(win.p, d_values, N, c->fixed, c->g, is_free.p, is_fixed.p);
    if ((rc = cu(cudaGetLastError(), "launch condense"))) return fail(rc);
    int hbad = 0;
    if ((rc = cu(cudaMemcpyAsync(&hbad, bad.p, sizeof hbad, cudaMemcpyDeviceToHost, st), "memcpy")) ||
        (rc = cu(cudaStreamSynchronize(st), "sync")))
        return fail(rc);
    if (hbad) return fail(set_error(TGK_ERR_INPUT, "condense: dirichlet dof out of range"));
    if ((rc = exclusive_scan(is_free.p, free_index.p, N + 1, st)) || (rc = exclusive_scan(is_fixed.p, fixed_index.p, N + 1, st)))
        return fail(rc);
    if ((rc = cu(cudaMemcpyAsync(&c->n_free, free_index.p + N, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "memcpy")) ||
        (rc = cu(cudaMemcpyAsync(&c->n_fixed, fixed_index.p + N, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "memcpy")) ||
        (rc = cu(cudaStreamSynchronize(st), "sync")))
        return fail(rc);
    const int64_t nf = c->n_free, nc = c->n_fixed;
    if ((rc = cu(cudaMalloc(&c->free_dofs, sizeof(int64_t) * std::max<int64_t>(nf, 1)), "cudaMalloc")) ||
        (rc = cu(cudaMalloc(&c->fixed_dofs, sizeof(int64_t) * std::max<int64_t>(nc, 1)), "cudaMalloc")) ||
        (rc = cu(cudaMalloc(&c->prescribed, sizeof(double) * std::max<int64_t>(nc, 1)), "cudaMalloc")) ||
        (rc = cu(cudaMalloc(&c->offsets, sizeof(int64_t) * (nf + 1)), "cudaMalloc")) ||
        (rc = cu(cudaMalloc(&c->F_f, sizeof(double) * std::max<int64_t>(nf, 1)), "cudaMalloc")))
        return fail(rc);
    if (N > 0)
        k_lists<<<grid_n(N), 256, 0, st>>>(N, c->fixed, c->g, free_index.p, fixed_index.p, c->free_dofs, c->fixed_dofs,
                                          c->prescribed);
    if ((rc = cnt.alloc(nf + 1))) return fail(rc);
    if ((rc = cu(cudaMemsetAsync(cnt.p + nf, 0, sizeof(int64_t), st), "memset"))) return fail(rc);
    if (nf > 0) k_count_free<<<grid_n(nf), 256, 0, st>>>(nf, c->free_dofs, d_offsets, d_cols, c->fixed, cnt.p);
    if ((rc = cu(cudaGetLastError(), "launch condense"))) return fail(rc);
    if ((rc = exclusive_scan(cnt.p, c->offsets, nf + 1, st))) return fail(rc);
    if ((rc = cu(cudaMemcpyAsync(&c->nnz_ff, c->offsets + nf, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "memcpy")) ||
        (rc = cu(cudaStreamSynchronize(st), "sync")))
        return fail(rc);
    if ((rc = cu(cudaMalloc(&c->cols, sizeof(int64_t) * std::max<int64_t>(c->nnz_ff, 1)), "cudaMalloc")) ||
        (rc = cu(cudaMalloc(&c->values, sizeof(double) * std::max<int64_t>(c->nnz_ff, 1)), "cudaMalloc")))
        return fail(rc);
    if (nf > 0)
        k_fill<<<grid_n(nf), 256, 0, st>>>(nf, c->free_dofs, d_offsets, d_cols, d_K, d_F, c->fixed, c->g, free_index.p,
                                          c->offsets, c->cols, c->values, c->F_f);
    if ((rc = cu(cudaGetLastError(), "launch condense")) || (rc = cu(cudaStreamSynchronize(st), "sync"))) return fail(rc);
    *out = c;
    return TGK_OK;
}

int tgk_condensed_info(const tgk_condensed* c, int64_t* n_free, int64_t* n_fixed, int64_t* nnz_ff,
                       const int64_t** d_free_dofs, const int64_t** d_fixed_dofs, const double** d_prescribed,
                       const int64_t** d_offsets, const int64_t** d_cols, const double** d_values,
                       const double** d_F_f) {
    if (!c) return tgk::set_error(TGK_ERR_INPUT, "condensed: null handle");
    if (n_free) *n_free = c->n_free;
    if (n_fixed) *n_fixed = c->n_fixed;
    if (nnz_ff) *nnz_ff = c->nnz_ff;
    if (d_free_dofs) *d_free_dofs = c->free_dofs;
    if (d_fixed_dofs) *d_fixed_dofs = c->fixed_dofs;
    if (d_prescribed) *d_prescribed = c->prescribed;
    if (d_offsets) *d_offsets = c->offsets;
    if (d_cols) *d_cols = c->cols;
    if (d_values) *d_values = c->values;
    if (d_F_f) *d_F_f = c->F_f;
    return TGK_OK;
}

int tgk_restrict_to_free_d(const tgk_condensed* c, const int64_t* d_offsets, const int64_t* d_cols, const double* d_A,
                           double* d_out, void* stream) {
    using namespace tgk;
    if (!c || (c->n_free > 0 && (!d_offsets || !d_cols || !d_A || !d_out)))
        return set_error(TGK_ERR_INPUT, "restrict_to_free: bad arguments");
    TGK_TRY(ensure_device());
    if (c->n_free == 0) return TGK_OK;
    k_restrict<<<grid_n(c->n_free), 256, 0, as_stream(stream)>>>(c->n_free, c->free_dofs, d_offsets, d_cols, d_A,
                                                                 c->fixed, c->offsets, d_out);
    KERNEL_CHECK("restrict_to_free");
    return TGK_OK;
}

int tgk_expand_d(const tgk_condensed* c, const double* d_u_free, double* d_u, void* stream) {
    using namespace tgk;
    if (!c || !d_u || (c->n_free > 0 && !d_u_free)) return set_error(TGK_ERR_INPUT, "expand: bad arguments");
    TGK_TRY(ensure_device());
    cudaStream_t st = as_stream(stream);
    CUDA_TRY(cudaMemsetAsync(d_u, 0, sizeof(double) * c->full_size, st));
    const int64_t n = std::max(c->n_free, c->n_fixed);
    if (n > 0)
        k_expand<<<grid_n(n), 256, 0, st>>>(c->n_free, c->free_dofs, d_u_free, c->n_fixed, c->fixed_dofs,
                                            c->prescribed, d_u);
    KERNEL_CHECK("expand");
    return TGK_OK;
}

int tgk_condensed_copy(const tgk_condensed* c, int64_t* free_dofs, int64_t* fixed_dofs, double* prescribed,
                       int64_t* offsets, int64_t* cols, double* values, double* F_f) {
    using namespace tgk;
    if (!c) return set_error(TGK_ERR_INPUT, "condensed: null handle");
    auto cp = [](void* dst, const void* src, size_t bytes) -> int {
        if (dst && bytes) CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        return TGK_OK;
    };
    TGK_TRY(cp(free_dofs, c->free_dofs, sizeof(int64_t) * c->n_free));
    TGK_TRY(cp(fixed_dofs, c->fixed_dofs, sizeof(int64_t) * c->n_fixed));
    TGK_TRY(cp(prescribed, c->prescribed, sizeof(double) * c->n_fixed));
    TGK_TRY(cp(offsets, c->offsets, sizeof(int64_t) * (c->n_free + 1)));
    TGK_TRY(cp(cols, c->cols, sizeof(int64_t) * c->nnz_ff));
    TGK_TRY(cp(values, c->values, sizeof(double) * c->nnz_ff));
    TGK_TRY(cp(F_f, c->F_f, sizeof(double) * c->n_free));
    return TGK_OK;
}


// Jacobi-preconditioned BiCGSTAB with restarts, divergence rollback and the
// best-iterate fallback of the reference (solver.cpp:105-227), on device CSR.
int tgk_bicgstab_d(int64_t n, const int64_t* d_offsets, const int64_t* d_cols, const double* d_values,
                   const double* d_b, double* d_x, double tol_rel, double tol_abs, int64_t max_iter,
                   int64_t* iterations, double* rel_residual, int* converged, void* stream) {
    using namespace tgk;
    if (n < 0 || (n > 0 && (!d_offsets || !d_cols || !d_values || !d_b || !d_x)))
        return set_error(TGK_ERR_INPUT, "bicgstab: bad arguments");
    TGK_TRY(ensure_device());
    // the iteration body is replayed as one CUDA graph: capture needs a real
    // stream, so the legacy default stream is replaced by a blocking stream
    // (implicitly ordered after the caller's legacy-stream work)
    cudaStream_t st = as_stream(stream);
    cudaStream_t own = nullptr;
    if (!st) {
        CUDA_TRY(cudaStreamCreate(&own));
        st = own;
    }
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            if (s) cudaStreamDestroy(s);
        }
    } stream_guard{own};
    int64_t iters = 0;
    if (iterations) *iterations = 0;
    if (rel_residual) *rel_residual = 0.0;
    if (converged) *converged = 0;
    if (n == 0) {
        if (converged) *converged = 1;
        return TGK_OK;
    }
    DevBuf<double> r, p, v, phat, shat, s, t, rt, inv, best_x, part, scal, sc;
    DevBuf<int> flag, state;
    for (DevBuf<double>* b : {&r, &p, &v, &phat, &shat, &s, &t, &rt, &inv, &best_x}) TGK_TRY(b->alloc(n));
    TGK_TRY(part.alloc(2 * kDotBlocks));
    TGK_TRY(scal.alloc(2));
    TGK_TRY(sc.alloc(S_COUNT));
    struct PinnedBuf {  // read-back of the scalars + state (pinned: capturable copies)
        double* p = nullptr;
        ~PinnedBuf() {
            if (p) cudaFreeHost(p);
        }
    } hbuf;
    CUDA_TRY(cudaMallocHost(&hbuf.p, sizeof(double) * (S_COUNT + 1)));
    struct GraphGuard {
        cudaGraphExec_t e = nullptr;
        ~GraphGuard() {
            if (e) cudaGraphExecDestroy(e);
        }
    } graph_guard;
    cudaGraphExec_t& graph_exec = graph_guard.e;
    bool graph_tried = false;
    TGK_TRY(flag.alloc(1));
    TGK_TRY(state.alloc(1));
    const unsigned G = grid_n(n);
    auto dot = [&](const double* a, const double* b, double* out) -> int {
        k_dot_partial<<<kDotBlocks, kDotThreads, 0, st>>>(a, b, n, part.p);
        k_dot_final<<<1, 512, 0, st>>>(part.p, scal.p);
        CUDA_TRY(cudaMemcpyAsync(out, scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        return TGK_OK;
    };
    // device-side dot products into the scalar slots (no host synchronisation)
    auto dot_d = [&](const double* a, const double* b, int slot) {
        k_dot_partial<<<kDotBlocks, kDotThreads, 0, st>>>(a, b, n, part.p);
        k_dot_final<<<1, 512, 0, st>>>(part.p, sc.p + slot);
    };
    auto dot2_d = [&](const double* a, const double* b, const double* c, const double* d, int slot0, int slot1) {
        k_dot2_partial<<<kDotBlocks, kDotThreads, 0, st>>>(a, b, c, d, n, part.p);
        k_dot_final<<<1, 512, 0, st>>>(part.p, sc.p + slot0);
        k_dot_final<<<1, 512, 0, st>>>(part.p + kDotBlocks, sc.p + slot1);
    };
    auto nrm = [&](const double* a, double* out) -> int {
        TGK_TRY(dot(a, a, out));
        *out = std::sqrt(*out);
        return TGK_OK;
    };
    auto residual = [&](double* out_r, bool* finite) -> int {  // out_r = b - A x
        CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
        k_residual<<<G, 256, 0, st>>>(n, d_offsets, d_cols, d_values, d_x, d_b, out_r, flag.p);
        int h = 0;
        CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        *finite = h == 0;
        return TGK_OK;
    };
    double norm_b = 0.0;
    TGK_TRY(nrm(d_b, &norm_b));
    if (norm_b == 0.0) {  // solver.cpp:113-117
        CUDA_TRY(cudaMemsetAsync(d_x, 0, sizeof(double) * n, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (converged) *converged = 1;
        return TGK_OK;
    }
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    k_inv_diag<<<G, 256, 0, st>>>(n, d_offsets, d_cols, d_values, inv.p, flag.p);
    int zero = 0;
    CUDA_TRY(cudaMemcpyAsync(&zero, flag.p, sizeof zero, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (zero) return set_error(TGK_ERR_NUMERICAL, "Jacobi preconditioner: zero diagonal entry");
    const double tol = tol_rel * norm_b, eps_bd = 1e-300;
    const int max_restarts = 8;
    CUDA_TRY(cudaMemcpyAsync(best_x.p, d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    double best_res = 1e300;
    for (int pass = 0; pass <= max_restarts && iters < max_iter; ++pass) {
        bool finite = true;
        TGK_TRY(residual(r.p, &finite));
        if (!finite) {  // diverged iterate: roll back to the best one (solver.cpp:140-145)
            CUDA_TRY(cudaMemcpyAsync(d_x, best_x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            TGK_TRY(residual(r.p, &finite));
        }
        double res = 0.0;
        TGK_TRY(nrm(r.p, &res));
        if (res < best_res) {
            best_res = res;
            CUDA_TRY(cudaMemcpyAsync(best_x.p, d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        }
        if (res <= tol) break;
        CUDA_TRY(cudaMemcpyAsync(rt.p, r.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemsetAsync(p.p, 0, sizeof(double) * n, st));
        CUDA_TRY(cudaMemsetAsync(v.p, 0, sizeof(double) * n, st));
        {  // rho = alpha = omega = 1, rho_new = rt . r (solver.cpp:146-150)
            const double init[3] = {1.0, 1.0, 1.0};
            CUDA_TRY(cudaMemcpyAsync(sc.p + S_RHO, init, sizeof init, cudaMemcpyHostToDevice, st));
            dot_d(rt.p, r.p, S_RHONEW);
        }
        const double eps_rho = eps_bd * norm_b * norm_b;
        auto launch_iteration = [&]() -> int {
            CUDA_TRY(cudaMemsetAsync(state.p, 0, sizeof(int), st));
            k_it_begin<<<1, 1, 0, st>>>(sc.p, state.p, eps_rho);
            k_bicg_p<<<G, 256, 0, st>>>(n, r.p, v.p, inv.p, sc.p, state.p, p.p, phat.p);
            k_spmv<<<G, 256, 0, st>>>(n, d_offsets, d_cols, d_values, phat.p, v.p);
            dot_d(rt.p, v.p, S_RTV);
            k_it_alpha<<<1, 1, 0, st>>>(sc.p, state.p);
            k_bicg_s<<<G, 256, 0, st>>>(n, r.p, v.p, sc.p, state.p, s.p);
            dot_d(s.p, s.p, S_SS);
            k_it_s<<<1, 1, 0, st>>>(sc.p, state.p, tol);
            k_bicg_x<<<G, 256, 0, st>>>(n, sc.p, state.p, 1, phat.p, nullptr, nullptr, nullptr, d_x, nullptr);
            k_scale<<<G, 256, 0, st>>>(n, inv.p, s.p, state.p, shat.p);
            k_spmv<<<G, 256, 0, st>>>(n, d_offsets, d_cols, d_values, shat.p, t.p);
            dot2_d(t.p, t.p, t.p, s.p, S_TT, S_TS);
            k_it_omega<<<1, 1, 0, st>>>(sc.p, state.p, eps_bd);
            k_bicg_x<<<G, 256, 0, st>>>(n, sc.p, state.p, 2, phat.p, shat.p, s.p, t.p, d_x, r.p);
            // ||r|| and the next iteration's rho = rt . r in one pass
            dot2_d(r.p, r.p, rt.p, r.p, S_RR, S_RHONEW);
            k_it_end<<<1, 1, 0, st>>>(sc.p, state.p);
            CUDA_TRY(cudaMemcpyAsync(hbuf.p, sc.p, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(hbuf.p + S_COUNT, state.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            return TGK_OK;
        };
        // one graph for the whole iteration (17 launches + 2 read-backs): captured
        // once per solve, replayed per iteration; direct launches if capture fails
        if (!graph_tried) {
            graph_tried = true;
            if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                (void)launch_iteration();
                cudaGraph_t g = nullptr;
                if (cudaStreamEndCapture(st, &g) == cudaSuccess && g) {
                    if (cudaGraphInstantiate(&graph_exec, g, 0) != cudaSuccess) graph_exec = nullptr;
                    cudaGraphDestroy(g);
                }
            }
            cudaGetLastError();  // a failed capture leaves the direct path
        }
        while (res > tol && iters < max_iter) {
            if (graph_exec) CUDA_TRY(cudaGraphLaunch(graph_exec, st));
            else TGK_TRY(launch_iteration());
            CUDA_TRY(cudaStreamSynchronize(st));  // the iteration's one host synchronisation
            const double* hs = hbuf.p;
            int hstate = 0;
            std::memcpy(&hstate, hbuf.p + S_COUNT, sizeof hstate);
            if (hstate == 2) break;  // rho or alpha breakdown: the iteration does not count
            ++iters;
            if (hstate == 1) {  // ||s|| <= tol: x += alpha phat done
                res = hs[S_SNORM];
                break;
            }
            if (hstate == 3) break;  // omega breakdown: x += alpha phat done
            res = hs[S_RES];
            if (hstate == 4) break;
        }
        KERNEL_CHECK("bicgstab");
    }
    // report the true residual, roll back to the best iterate if worse (solver.cpp:210-218)
    bool finite = true;
    TGK_TRY(residual(r.p, &finite));
    double fin = 0.0;
    TGK_TRY(nrm(r.p, &fin));
    if (!finite || fin > best_res) {
        CUDA_TRY(cudaMemcpyAsync(d_x, best_x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        TGK_TRY(residual(r.p, &finite));
        TGK_TRY(nrm(r.p, &fin));
    }
    if (iterations) *iterations = iters;
    if (rel_residual) *rel_residual = fin / norm_b;
    if (converged) *converged = (fin / norm_b <= tol_rel || fin <= tol_abs) ? 1 : 0;
    return TGK_OK;
}

int tgk_copy_d2d(void* dst, const void* src, int64_t nbytes, void* stream) {
    using namespace tgk;
    if (nbytes < 0 || (nbytes > 0 && (!dst || !src))) return set_error(TGK_ERR_INPUT, "copy_d2d: bad arguments");
    if (nbytes) CUDA_TRY(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
    return TGK_OK;
}

void tgk_condensed_destroy(tgk_condensed* c) { delete c; }

// Device memory plumbing for host-language callers without the CUDA runtime
// headers (the C++ adapter, ctypes).
int tgk_alloc_d(void** p, int64_t nbytes) {
    using namespace tgk;
    if (!p || nbytes < 0) return set_error(TGK_ERR_INPUT, "alloc_d: bad arguments");
    TGK_TRY(ensure_device());
    *p = nullptr;
    CUDA_TRY(cudaMalloc(p, nbytes > 0 ? size_t(nbytes) : 1));
    return TGK_OK;
}

int tgk_free_d(void* p) {
    if (p) cudaFree(p);
    return TGK_OK;
}

int tgk_copy_d2h(void* dst, const void* src, int64_t nbytes) {
    using namespace tgk;
    if (nbytes < 0 || (nbytes > 0 && (!dst || !src))) return set_error(TGK_ERR_INPUT, "copy_d2h: bad arguments");
    if (nbytes) CUDA_TRY(cudaMemcpy(dst, src, nbytes, cudaMemcpyDeviceToHost));
    return TGK_OK;
}

int tgk_copy_h2d(void* dst, const void* src, int64_t nbytes) {
    using namespace tgk;
    if (nbytes < 0 || (nbytes > 0 && (!dst || !src))) return set_error(TGK_ERR_INPUT, "copy_h2d: bad arguments");
    if (nbytes) CUDA_TRY(cudaMemcpy(dst, src, nbytes, cudaMemcpyHostToDevice));
    return TGK_OK;
}

}  // extern "C"
