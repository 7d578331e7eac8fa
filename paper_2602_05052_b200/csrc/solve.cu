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

void tgk_condensed_destroy(tgk_condensed* c) { delete c; }

}  // extern "C"
