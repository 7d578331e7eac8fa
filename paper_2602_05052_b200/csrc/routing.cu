// GPU routing build: the CSR pattern, the element-to-CSR-slot map and the
// reference's segment maps, bit-identical to build_routing
// (/root/reference/proj/src/routing.cpp:12-85).
//
//  1. incidence counts per DoF (integer atomics: order-free, deterministic)
//  2. vec_offsets = exclusive scan; vec_slots = stable radix sort of the
//     (dof, slot) pairs keyed by dof  -> ascending slot within each DoF,
//     exactly routing.cpp:47-62
//  3. one thread per row builds the sorted unique neighbour list from its
//     incident elements (the same set as sort+unique of all (g_a,g_b) pairs,
//     routing.cpp:17-36) — count pass, scan, fill pass
//  4. slot_of[(e*k+a)*k+b] = find(g_a, g_b) by binary search (sparse.cpp:10-16)
//  5. optional reference segment maps mat_offsets/mat_slots: per-row threads
//     walk their incidences in ascending slot order (routing.cpp:64-83)
// Vector (components = d) patterns are derived from the scalar one: DoF
// numbering is node-major interleaved (dofmap.cpp:18-19), so row (i,c) holds
// columns {d*j + c' : j in row i}.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "cuda_util.cuh"
#include "tgk_internal.hpp"

namespace tgk {
namespace {

constexpr int kMaxRow = 64;  // scalar row-length limit of the per-thread row builder

__global__ void k_count_incidence(const int32_t* conn, int64_t Ek, uint32_t* cnt) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < Ek;
         s += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[conn[s]], 1u);
}

__global__ void k_iota_keys(const int32_t* conn, int64_t Ek, uint32_t* keys, uint32_t* vals) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < Ek;
         s += (int64_t)gridDim.x * blockDim.x) {
        keys[s] = static_cast<uint32_t>(conn[s]);
        vals[s] = static_cast<uint32_t>(s);
    }
}

// sorted-unique insertion into a small per-thread list
__device__ __forceinline__ int insert_unique(int32_t* list, int len, int32_t v) {
    int p = len;
    while (p > 0 && list[p - 1] > v) --p;
    if (p > 0 && list[p - 1] == v) return len;
    for (int q = len; q > p; --q) list[q] = list[q - 1];
    list[p] = v;
    return len + 1;
}

template <bool FILL>
__global__ void k_row_pattern(const int32_t* conn, int k, int64_t N, const uint32_t* vec_off,
                              const uint32_t* vec_slots, int64_t* row_len, const int64_t* row_ptr,
                              int64_t* cols, int* overflow) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int32_t list[kMaxRow];
    int len = 0;
    for (uint32_t s = vec_off[i]; s < vec_off[i + 1]; ++s) {
        const int64_t e = vec_slots[s] / k;
        for (int b = 0; b < k; ++b) {
            len = insert_unique(list, len, conn[e * k + b]);
            if (len >= kMaxRow) {  // long row: built by k_row_long (global scratch list)
                if (!FILL) {
                    row_len[i] = -1;
                    atomicExch(overflow, 1);
                }
                return;
            }
        }
    }
    if (!FILL) {
        row_len[i] = len;
    } else {
        int64_t* out = cols + row_ptr[i];
        for (int p = 0; p < len; ++p) out[p] = list[p];
    }
}

// Rows with kMaxRow or more neighbours (fans, high-valence nodes of
// unstructured meshes): one thread per such row builds the sorted unique list
// in a global scratch segment bounded by its incidences x k.
__global__ void k_row_long(const int32_t* conn, int k, const uint32_t* vec_off, const uint32_t* vec_slots,
                           const int64_t* rows, const int64_t* scr_off, int64_t n_long, int32_t* scr,
                           int64_t* row_len) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_long) return;
    const int64_t i = rows[t];
    int32_t* list = scr + scr_off[t];
    int64_t len = 0;
    for (uint32_t s = vec_off[i]; s < vec_off[i + 1]; ++s) {
        const int64_t e = vec_slots[s] / k;
        for (int b = 0; b < k; ++b) {
            const int32_t v = conn[e * k + b];
            int64_t p = len;
            while (p > 0 && list[p - 1] > v) --p;
            if (p > 0 && list[p - 1] == v) continue;
            for (int64_t q = len; q > p; --q) list[q] = list[q - 1];
            list[p] = v;
            ++len;
        }
    }
    row_len[i] = len;
}

__global__ void k_row_long_fill(const int64_t* rows, const int64_t* scr_off, int64_t n_long, const int32_t* scr,
                                const int64_t* row_ptr, int64_t* cols) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_long) return;
    const int64_t i = rows[t];
    for (int64_t p = 0; p < row_ptr[i + 1] - row_ptr[i]; ++p) cols[row_ptr[i] + p] = scr[scr_off[t] + p];
}

__device__ __forceinline__ int64_t find_col(const int64_t* cols, int64_t lo, int64_t hi, int64_t j) {
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (cols[mid] < j) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_slot_of(const int32_t* conn, int k, int64_t E, const int64_t* row_ptr,
                          const int64_t* cols, uint32_t* slot_of) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // s = e*k + a
    if (s >= E * k) return;
    const int64_t e = s / k;
    const int64_t row = conn[s];
    const int64_t lo = row_ptr[row], hi = row_ptr[row + 1];
    for (int b = 0; b < k; ++b)
        slot_of[s * k + b] = static_cast<uint32_t>(find_col(cols, lo, hi, conn[e * k + b]));
}

// mat segment counts, per scalar row (routing.cpp:65-71)
__global__ void k_mat_count(int k, int64_t N, const uint32_t* vec_off, const uint32_t* vec_slots,
                            const int64_t* row_ptr, const uint32_t* slot_of, uint32_t* count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    for (uint32_t s = vec_off[i]; s < vec_off[i + 1]; ++s) {
        const uint64_t slot = vec_slots[s];
        for (int b = 0; b < k; ++b) count[slot_of[slot * k + b]] += 1;  // row-private: no race
    }
}

// mat_slots fill (routing.cpp:72-83): ascending slot within each nonzero
// (rows longer than kMaxRow keep their cursors in the global scratch gcur, nnz entries)
__global__ void k_mat_fill(int k, int64_t N, const uint32_t* vec_off, const uint32_t* vec_slots,
                           const int64_t* row_ptr, const uint32_t* slot_of,
                           const uint32_t* mat_off, uint32_t* mat_slots, uint32_t* gcur) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t rp = row_ptr[i];
    const int len = static_cast<int>(row_ptr[i + 1] - rp);
    uint32_t lcur[kMaxRow];
    uint32_t* cur = len > kMaxRow ? gcur + rp : lcur;
    for (int p = 0; p < len; ++p) cur[p] = mat_off[rp + p];
    for (uint32_t s = vec_off[i]; s < vec_off[i + 1]; ++s) {
        const uint64_t slot = vec_slots[s];
        for (int b = 0; b < k; ++b) {
            const int p = static_cast<int>(slot_of[slot * k + b] - rp);
            mat_slots[cur[p]++] = static_cast<uint32_t>(slot * k + b);
        }
    }
}

// ---- vector (components = c) routing derived from the scalar routing
__global__ void k_vec_pattern(int c, int64_t N, const int64_t* rp_s, const int64_t* cols_s,
                              int64_t* rp_v, int64_t* cols_v) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // r = i*c + ci
    if (r >= N * c) return;
    const int64_t i = r / c, ci = r % c;
    const int64_t len = rp_s[i + 1] - rp_s[i];
    const int64_t start = (int64_t)c * c * rp_s[i] + ci * c * len;
    rp_v[r] = start;
    if (r == N * c - 1) rp_v[N * c] = (int64_t)c * c * rp_s[N];
    for (int64_t p = 0; p < len; ++p)
        for (int cj = 0; cj < c; ++cj) cols_v[start + c * p + cj] = c * cols_s[rp_s[i] + p] + cj;
}

__global__ void k_vec_segments(int c, int k, int64_t N, const uint32_t* vo_s, const uint32_t* vs_s,
                               uint32_t* vo_v, uint32_t* vs_v) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= N * c) return;
    const int64_t i = r / c, ci = r % c;
    const uint32_t cnt = vo_s[i + 1] - vo_s[i];
    const uint32_t start = c * vo_s[i] + ci * cnt;
    vo_v[r] = start;
    if (r == N * c - 1) vo_v[N * c] = c * vo_s[N];
    const int kv = k * c;
    for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t s = vs_s[vo_s[i] + q];
        const uint32_t e = s / k, a = s % k;
        vs_v[start + q] = e * kv + a * c + ci;
    }
}

__global__ void k_vec_mat_count(int c, int64_t nnz_s, const int64_t* rp_s, int64_t N,
                                const uint32_t* count_s, const int64_t* rp_v, uint32_t* count_v) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= N * c) return;
    const int64_t i = r / c;
    const int64_t len = rp_s[i + 1] - rp_s[i];
    for (int64_t p = 0; p < len; ++p)
        for (int cj = 0; cj < c; ++cj) count_v[rp_v[r] + c * p + cj] = count_s[rp_s[i] + p];
}

__global__ void k_vec_mat_fill(int c, int k, int64_t N, const uint32_t* vo_s, const uint32_t* vs_s,
                               const int64_t* rp_s, const uint32_t* slot_of_s,
                               const int64_t* rp_v, const uint32_t* mat_off_v,
                               uint32_t* mat_slots_v, uint32_t* gcur) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= N * c) return;
    const int64_t i = r / c, ci = r % c;
    const int64_t len = rp_s[i + 1] - rp_s[i];
    uint32_t lcur[kMaxRow * 3];
    uint32_t* cur = len * c > kMaxRow * 3 ? gcur + rp_v[r] : lcur;
    for (int64_t q = 0; q < len * c; ++q) cur[q] = mat_off_v[rp_v[r] + q];
    const uint32_t kv = k * c;
    for (uint32_t s_ix = vo_s[i]; s_ix < vo_s[i + 1]; ++s_ix) {
        const uint64_t s = vs_s[s_ix];
        const uint32_t e = static_cast<uint32_t>(s / k), a = static_cast<uint32_t>(s % k);
        for (int b = 0; b < k; ++b) {
            const int64_t p = slot_of_s[s * k + b] - rp_s[i];
            for (int cj = 0; cj < c; ++cj) {
                const uint32_t u = (e * kv + a * c + ci) * kv + b * c + cj;
                mat_slots_v[cur[c * p + cj]++] = u;
            }
        }
    }
}

template <class T>
int exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t st) {
    size_t tmp_bytes = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, n, st));
    DevBuf<unsigned char> tmp;
    TGK_TRY(tmp.alloc(tmp_bytes + 1));
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, in, out, n, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return TGK_OK;
}

int build_scalar(const tgk_mesh* m, int flags, cudaStream_t st, tgk_routing* r) {
    const int k = m->k;
    const int64_t N = m->N, E = m->E, Ek = E * k;
    r->N = N;
    r->E = E;
    r->k = k;
    r->components = 1;
    const unsigned B = 256;
    // 1-2: incidence CSR (vec_offsets / vec_slots)
    DevBuf<uint32_t> cnt, vo, vs, keys_in, keys_out, vals_in;
    TGK_TRY(cnt.alloc(N + 1));
    TGK_TRY(vo.alloc(N + 1));
    TGK_TRY(vs.alloc(Ek));
    CUDA_TRY(cudaMemsetAsync(cnt.p, 0, (N + 1) * sizeof(uint32_t), st));
    k_count_incidence<<<grid_for(Ek, B), B, 0, st>>>(m->conn, Ek, cnt.p);
    KERNEL_CHECK("count_incidence");
    TGK_TRY(exclusive_scan<uint32_t>(cnt.p, vo.p, N + 1, st));
    TGK_TRY(keys_in.alloc(Ek));
    TGK_TRY(keys_out.alloc(Ek));
    TGK_TRY(vals_in.alloc(Ek));
    k_iota_keys<<<grid_for(Ek, B), B, 0, st>>>(m->conn, Ek, keys_in.p, vals_in.p);
    KERNEL_CHECK("iota_keys");
    {
        int end_bit = 1;
        while ((int64_t(1) << end_bit) < N) ++end_bit;
        size_t tmp_bytes = 0;
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in.p, keys_out.p,
                                                 vals_in.p, vs.p, Ek, 0, end_bit, st));
        DevBuf<unsigned char> tmp;
        TGK_TRY(tmp.alloc(tmp_bytes + 1));
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys_in.p, keys_out.p,
                                                 vals_in.p, vs.p, Ek, 0, end_bit, st));
    }
    keys_in.reset();
    keys_out.reset();
    vals_in.reset();
    // 3: pattern
    DevBuf<int64_t> row_len, rp;
    DevBuf<int> overflow;
    TGK_TRY(row_len.alloc(N + 1));
    TGK_TRY(rp.alloc(N + 1));
    TGK_TRY(overflow.alloc(1));
    CUDA_TRY(cudaMemsetAsync(overflow.p, 0, sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(row_len.p + N, 0, sizeof(int64_t), st));
    k_row_pattern<false><<<grid_for(N, 128), 128, 0, st>>>(m->conn, k, N, vo.p, vs.p, row_len.p,
                                                          nullptr, nullptr, overflow.p);
    KERNEL_CHECK("row_pattern");
    int ovf = 0;
    CUDA_TRY(cudaMemcpyAsync(&ovf, overflow.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    DevBuf<int64_t> long_rows, long_off;
    DevBuf<int32_t> long_scr;
    int64_t n_long = 0;
    {
        std::vector<int64_t> h_len(N);
        CUDA_TRY(cudaMemcpy(h_len.data(), row_len.p, N * sizeof(int64_t), cudaMemcpyDeviceToHost));
        if (ovf) {  // rows of kMaxRow+ neighbours: global-scratch builder
            std::vector<uint32_t> h_vo(N + 1);
            CUDA_TRY(cudaMemcpy(h_vo.data(), vo.p, (N + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            std::vector<int64_t> lr, lo{0};
            for (int64_t i = 0; i < N; ++i)
                if (h_len[i] < 0) {
                    lr.push_back(i);
                    lo.push_back(lo.back() + int64_t(h_vo[i + 1] - h_vo[i]) * k);
                }
            n_long = static_cast<int64_t>(lr.size());
            TGK_TRY(long_rows.alloc(n_long));
            TGK_TRY(long_off.alloc(n_long + 1));
            TGK_TRY(long_scr.alloc(std::max<int64_t>(1, lo.back())));
            CUDA_TRY(cudaMemcpy(long_rows.p, lr.data(), n_long * sizeof(int64_t), cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(long_off.p, lo.data(), (n_long + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
            k_row_long<<<grid_for(n_long, 64), 64, 0, st>>>(m->conn, k, vo.p, vs.p, long_rows.p, long_off.p, n_long,
                                                            long_scr.p, row_len.p);
            KERNEL_CHECK("row_long");
            CUDA_TRY(cudaMemcpy(h_len.data(), row_len.p, N * sizeof(int64_t), cudaMemcpyDeviceToHost));
        }
        // row length max (for the fused plans) and row_ptr
        int64_t lmax = 0;
        for (auto v : h_len) lmax = v > lmax ? v : lmax;
        r->lmax = static_cast<int>(lmax);
    }
    TGK_TRY(exclusive_scan<int64_t>(row_len.p, rp.p, N + 1, st));
    int64_t nnz = 0;
    CUDA_TRY(cudaMemcpy(&nnz, rp.p + N, sizeof(int64_t), cudaMemcpyDeviceToHost));
    r->nnz = nnz;
    DevBuf<int64_t> cols;
    TGK_TRY(cols.alloc(nnz));
    k_row_pattern<true><<<grid_for(N, 128), 128, 0, st>>>(m->conn, k, N, vo.p, vs.p, nullptr, rp.p,
                                                         cols.p, overflow.p);
    KERNEL_CHECK("row_pattern_fill");
    if (n_long > 0) {
        k_row_long_fill<<<grid_for(n_long, 64), 64, 0, st>>>(long_rows.p, long_off.p, n_long, long_scr.p, rp.p, cols.p);
        KERNEL_CHECK("row_long_fill");
    }
    // 4: element-to-slot map
    DevBuf<uint32_t> slot;
    TGK_TRY(slot.alloc(Ek * k));
    k_slot_of<<<grid_for(Ek, B), B, 0, st>>>(m->conn, k, E, rp.p, cols.p, slot.p);
    KERNEL_CHECK("slot_of");
    // 5: reference segment maps
    if (flags & TGK_ROUTING_SEGMENTS) {
        if (E * k * static_cast<int64_t>(k) > static_cast<int64_t>(UINT32_MAX))
            return set_error(TGK_ERR_INPUT, "build_routing: mesh exceeds 2^32-1 local matrix slots");
        DevBuf<uint32_t> mcount, mo, ms;
        TGK_TRY(mcount.alloc(nnz + 1));
        TGK_TRY(mo.alloc(nnz + 1));
        TGK_TRY(ms.alloc(Ek * k));
        CUDA_TRY(cudaMemsetAsync(mcount.p, 0, (nnz + 1) * sizeof(uint32_t), st));
        k_mat_count<<<grid_for(N, 128), 128, 0, st>>>(k, N, vo.p, vs.p, rp.p, slot.p, mcount.p);
        KERNEL_CHECK("mat_count");
        TGK_TRY(exclusive_scan<uint32_t>(mcount.p, mo.p, nnz + 1, st));
        DevBuf<uint32_t> gcur;
        if (r->lmax > kMaxRow) TGK_TRY(gcur.alloc(nnz));
        k_mat_fill<<<grid_for(N, 128), 128, 0, st>>>(k, N, vo.p, vs.p, rp.p, slot.p, mo.p, ms.p, gcur.p);
        KERNEL_CHECK("mat_fill");
        CUDA_TRY(cudaStreamSynchronize(st));
        r->mat_offsets = mo.release();
        r->mat_slots = ms.release();
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    r->vec_offsets = vo.release();
    r->vec_slots = vs.release();
    r->row_ptr = rp.release();
    r->col_idx = cols.release();
    r->slot_of = slot.release();
    r->scalar = r;
    return TGK_OK;
}

int build_vector(const tgk_mesh* m, int c, int flags, cudaStream_t st, tgk_routing* s,
                 tgk_routing* r) {
    const int k = m->k;
    const int64_t N = m->N, E = m->E;
    r->N = N * c;
    r->E = E;
    r->k = k * c;
    r->components = c;
    r->lmax = s->lmax;
    r->nnz = s->nnz * c * c;
    DevBuf<int64_t> rp, cols;
    TGK_TRY(rp.alloc(N * c + 1));
    TGK_TRY(cols.alloc(r->nnz));
    k_vec_pattern<<<grid_for(N * c, 128), 128, 0, st>>>(c, N, s->row_ptr, s->col_idx, rp.p, cols.p);
    KERNEL_CHECK("vec_pattern");
    if (flags & TGK_ROUTING_SEGMENTS) {
        if (E * static_cast<int64_t>(r->k) * r->k > static_cast<int64_t>(UINT32_MAX))
            return set_error(TGK_ERR_INPUT, "build_routing: mesh exceeds 2^32-1 local matrix slots");
        DevBuf<uint32_t> vo, vs, mcount_s, mcount, mo, ms;
        TGK_TRY(vo.alloc(N * c + 1));
        TGK_TRY(vs.alloc(E * r->k));
        k_vec_segments<<<grid_for(N * c, 128), 128, 0, st>>>(c, k, N, s->vec_offsets, s->vec_slots,
                                                            vo.p, vs.p);
        KERNEL_CHECK("vec_segments");
        TGK_TRY(mcount_s.alloc(s->nnz + 1));
        CUDA_TRY(cudaMemsetAsync(mcount_s.p, 0, (s->nnz + 1) * sizeof(uint32_t), st));
        k_mat_count<<<grid_for(N, 128), 128, 0, st>>>(k, N, s->vec_offsets, s->vec_slots, s->row_ptr,
                                                     s->slot_of, mcount_s.p);
        KERNEL_CHECK("mat_count");
        TGK_TRY(mcount.alloc(r->nnz + 1));
        CUDA_TRY(cudaMemsetAsync(mcount.p + r->nnz, 0, sizeof(uint32_t), st));
        k_vec_mat_count<<<grid_for(N * c, 128), 128, 0, st>>>(c, s->nnz, s->row_ptr, N, mcount_s.p,
                                                             rp.p, mcount.p);
        KERNEL_CHECK("vec_mat_count");
        TGK_TRY(mo.alloc(r->nnz + 1));
        TGK_TRY(exclusive_scan<uint32_t>(mcount.p, mo.p, r->nnz + 1, st));
        TGK_TRY(ms.alloc(E * static_cast<int64_t>(r->k) * r->k));
        DevBuf<uint32_t> gcur;
        if (s->lmax * c > kMaxRow * 3) TGK_TRY(gcur.alloc(r->nnz));
        k_vec_mat_fill<<<grid_for(N * c, 128), 128, 0, st>>>(c, k, N, s->vec_offsets, s->vec_slots,
                                                            s->row_ptr, s->slot_of, rp.p, mo.p,
                                                            ms.p, gcur.p);
        KERNEL_CHECK("vec_mat_fill");
        CUDA_TRY(cudaStreamSynchronize(st));
        r->vec_offsets = vo.release();
        r->vec_slots = vs.release();
        r->mat_offsets = mo.release();
        r->mat_slots = ms.release();
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    r->row_ptr = rp.release();
    r->col_idx = cols.release();
    r->scalar = s;
    return TGK_OK;
}

}  // namespace

// The reference segment maps (mat_offsets / mat_slots, routing.cpp:64-83) of a
// scalar routing built without TGK_ROUTING_SEGMENTS, on demand (the
// materialised Stage II fallback of the fused kernels needs them).
int check_routing_fresh(const tgk_mesh* m, const tgk_routing* r) {
    if (r->mesh == m && r->mesh_version != m->conn_version)
        return set_error(TGK_ERR_INPUT, "routing was built for an earlier connectivity of this mesh "
                                        "(tgk_mesh_upload changed it): destroy and rebuild the routing");
    return TGK_OK;
}

int ensure_scalar_segments(tgk_routing* r, cudaStream_t st) {
    if (r->mat_offsets) return TGK_OK;
    if (r->components != 1) return set_error(TGK_ERR_INPUT, "segment maps: scalar routing expected");
    const int k = r->k;
    const int64_t N = r->N, E = r->E, nnz = r->nnz;
    if (E * k * static_cast<int64_t>(k) > static_cast<int64_t>(UINT32_MAX))
        return set_error(TGK_ERR_INPUT, "build_routing: mesh exceeds 2^32-1 local matrix slots");
    DevBuf<uint32_t> mcount, mo, ms, gcur;
    TGK_TRY(mcount.alloc(nnz + 1));
    TGK_TRY(mo.alloc(nnz + 1));
    TGK_TRY(ms.alloc(E * k * k));
    CUDA_TRY(cudaMemsetAsync(mcount.p, 0, (nnz + 1) * sizeof(uint32_t), st));
    k_mat_count<<<grid_for(N, 128), 128, 0, st>>>(k, N, r->vec_offsets, r->vec_slots, r->row_ptr, r->slot_of,
                                                 mcount.p);
    KERNEL_CHECK("mat_count");
    TGK_TRY(exclusive_scan<uint32_t>(mcount.p, mo.p, nnz + 1, st));
    if (r->lmax > kMaxRow) TGK_TRY(gcur.alloc(nnz));
    k_mat_fill<<<grid_for(N, 128), 128, 0, st>>>(k, N, r->vec_offsets, r->vec_slots, r->row_ptr, r->slot_of, mo.p,
                                                ms.p, gcur.p);
    KERNEL_CHECK("mat_fill");
    CUDA_TRY(cudaStreamSynchronize(st));
    r->mat_offsets = mo.release();
    r->mat_slots = ms.release();
    return TGK_OK;
}

}  // namespace tgk

tgk_routing::~tgk_routing() {
    for (void* p : {(void*)row_ptr, (void*)col_idx, (void*)slot_of, (void*)vec_offsets,
                    (void*)vec_slots, (void*)mat_offsets, (void*)mat_slots, (void*)scratch_K,
                    (void*)scratch_F, (void*)scratch_M})
        if (p) cudaFree(p);
    for (auto& pl : plan) pl.release();
    entry_plan.release();
    group_plan.release();
    if (flags) cudaFree(flags);
    for (auto& fp : fast_plan) fp.release();
    fast_plan_used = nullptr;
    for (double* p : scr)
        if (p) cudaFree(p);
    if (scalar && scalar != this) delete scalar;
}


namespace tgk {

// Device routing from host arrays in the reference layout (the cache loader
// and tgk_routing_create_host): pattern + segment maps uploaded, the
// element-to-slot map inverted from mat_slots, the scalar routing of vector
// problems rebuilt on the GPU.
int routing_from_arrays(const tgk_mesh* m, int components, int64_t N, int64_t E, int k, int64_t nnz,
                        const int64_t* off, const int64_t* cols, const uint32_t* vo, const uint32_t* vs,
                        const uint32_t* mo, const uint32_t* ms, cudaStream_t st, int* hit, tgk_routing** out) {
    TGK_TRY(ensure_device());
    const size_t Ek = static_cast<size_t>(E) * k;
    auto* r = new tgk_routing();
    r->mesh = m;
    r->mesh_version = m->conn_version;
    r->N = N;
    r->E = E;
    r->k = k;
    r->nnz = nnz;
    r->components = components;
    int64_t lmax = 0;
    for (int64_t i = 0; i < N; ++i) lmax = std::max<int64_t>(lmax, off[i + 1] - off[i]);
    r->lmax = static_cast<int>(components == 1 ? lmax : lmax / components);
    auto up = [](auto*& dst, const auto* src, size_t n) -> int {
        using T = typename std::remove_const<typename std::remove_pointer<decltype(src)>::type>::type;
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&dst), std::max<size_t>(1, n) * sizeof(T)));
        if (n) CUDA_TRY(cudaMemcpy(dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
        return TGK_OK;
    };
    int rc = TGK_OK;
    if (!rc) rc = up(r->row_ptr, off, size_t(N + 1));
    if (!rc) rc = up(r->col_idx, cols, size_t(nnz));
    if (!rc) rc = up(r->vec_offsets, vo, size_t(N + 1));
    if (!rc) rc = up(r->vec_slots, vs, Ek);
    if (!rc) rc = up(r->mat_offsets, mo, size_t(nnz + 1));
    if (!rc) rc = up(r->mat_slots, ms, Ek * k);
    if (!rc && components == 1) {
        // element-to-slot map = inverse of the segment map (slot_of[mat_slots[u]] = t)
        std::vector<uint32_t> slot(Ek * k);
        for (int64_t t = 0; t < nnz; ++t)
            for (uint32_t u = mo[t]; u < mo[t + 1]; ++u) slot[ms[u]] = static_cast<uint32_t>(t);
        rc = up(r->slot_of, slot.data(), slot.size());
        r->scalar = r;
    } else if (!rc) {
        // the fused kernels run on the node-level (scalar) routing: rebuild it on the GPU
        auto* s = new tgk_routing();
        s->mesh = m;
        s->mesh_version = m->conn_version;
        rc = build_scalar(m, 0, st, s);
        if (rc) delete s;
        else r->scalar = s;
    }
    if (rc) {
        if (r->scalar == r) r->scalar = nullptr;
        delete r;
        return rc;
    }
    *hit = 1;
    *out = r;
    return TGK_OK;
}

}  // namespace tgk

extern "C" {

int tgk_routing_build(const tgk_mesh* m, int components, int flags, void* stream,
                      tgk_routing** out) {
    using namespace tgk;
    if (!m || !out) return set_error(TGK_ERR_INPUT, "tgk_routing_build: null argument");
    TGK_TRY(ensure_device());
    if (m->kind == TGK_QUAD4)
        return set_error(TGK_ERR_INPUT, "tgk_routing_build: QUAD4 is not a P1 element (TRI3/TET4 only)");
    if (components != 1 && components != m->d)
        return set_error(TGK_ERR_INPUT, "components per node must be 1 or the mesh dimension");
    cudaStream_t st = as_stream(stream);
    auto* s = new tgk_routing();
    s->mesh = m;
    s->mesh_version = m->conn_version;
    int rc = build_scalar(m, components == 1 ? flags : 0, st, s);
    if (rc != TGK_OK) {
        delete s;
        return rc;
    }
    if (components == 1) {
        *out = s;
        return TGK_OK;
    }
    auto* v = new tgk_routing();
    v->mesh = m;
    v->mesh_version = m->conn_version;
    rc = build_vector(m, components, flags | TGK_ROUTING_SEGMENTS, st, s, v);
    if (rc != TGK_OK) {
        v->scalar = s;
        delete v;
        return rc;
    }
    *out = v;
    return TGK_OK;
}

void tgk_routing_destroy(tgk_routing* r) { delete r; }

int tgk_routing_get_view(const tgk_routing* r, tgk_routing_view* v) {
    if (!r || !v) return tgk::set_error(TGK_ERR_INPUT, "tgk_routing_get_view: null argument");
    v->N = r->N;
    v->E = r->E;
    v->nnz = r->nnz;
    v->k = r->k;
    v->components = r->components;
    v->row_ptr = r->row_ptr;
    v->col_idx = r->col_idx;
    v->slot_of = r->components == 1 ? r->slot_of : nullptr;
    v->vec_offsets = r->vec_offsets;
    v->vec_slots = r->vec_slots;
    v->mat_offsets = r->mat_offsets;
    v->mat_slots = r->mat_slots;
    return TGK_OK;
}

// load_routing (routing.cpp:211-234): the reference's "tg-rout2" cache file ->
// a device routing.  *hit = 0 (and TGK_OK) on a missing file, wrong magic,
// mesh-hash mismatch, size mismatch with the mesh or a short read — the cases
// in which the reference returns false and the caller rebuilds.
int tgk_routing_load(const tgk_mesh* m, int components, uint64_t mesh_hash, const char* path, void* stream,
                     int* hit, tgk_routing** out) {
    using namespace tgk;
    if (!m || !path || !hit || !out) return set_error(TGK_ERR_INPUT, "tgk_routing_load: null argument");
    *hit = 0;
    *out = nullptr;
    if (components != 1 && components != m->d)
        return set_error(TGK_ERR_INPUT, "components per node must be 1 or the mesh dimension");
    FILE* f = std::fopen(path, "rb");
    if (!f) return TGK_OK;
    int64_t h[6];
    auto rd = [f](void* dst, size_t bytes) { return std::fread(dst, 1, bytes, f) == bytes; };
    if (!rd(h, sizeof h) || static_cast<uint64_t>(h[0]) != 0x74672d726f757432ull ||
        static_cast<uint64_t>(h[1]) != mesh_hash || h[2] != m->N * components || h[3] != m->E ||
        h[4] != m->k * components) {
        std::fclose(f);
        return TGK_OK;
    }
    const int64_t N = h[2], E = h[3], nnz = h[5];
    const int k = static_cast<int>(h[4]);
    const size_t Ek = static_cast<size_t>(E) * k;
    std::vector<int64_t> off(N + 1), cols(nnz);
    std::vector<uint32_t> vo(N + 1), vs(Ek), mo(nnz + 1), ms(Ek * k);
    const bool ok = rd(off.data(), off.size() * 8) && rd(cols.data(), cols.size() * 8) && rd(vo.data(), vo.size() * 4) &&
                    rd(vs.data(), vs.size() * 4) && rd(mo.data(), mo.size() * 4) && rd(ms.data(), ms.size() * 4);
    std::fclose(f);
    if (!ok) return TGK_OK;
    return tgk::routing_from_arrays(m, components, N, E, k, nnz, off.data(), cols.data(), vo.data(), vs.data(),
                                    mo.data(), ms.data(), as_stream(stream), hit, out);
}

// Device routing from a caller's RoutingMatrices host arrays (routing.hpp:16-32):
// the caller's pattern and segment maps are uploaded as given, no rebuild.
int tgk_routing_create_host(const tgk_mesh* m, int components, int64_t N, int64_t E, int k, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx, const uint32_t* vec_offsets,
                            const uint32_t* vec_slots, const uint32_t* mat_offsets, const uint32_t* mat_slots,
                            void* stream, tgk_routing** out) {
    using namespace tgk;
    if (!m || !out || !row_ptr || !col_idx || !vec_offsets || !vec_slots || !mat_offsets || !mat_slots)
        return set_error(TGK_ERR_INPUT, "tgk_routing_create_host: null argument");
    if (components != 1 && components != m->d)
        return set_error(TGK_ERR_INPUT, "components per node must be 1 or the mesh dimension");
    if (N != m->N * components || E != m->E || k != m->k * components)
        return set_error(TGK_ERR_INPUT, "tgk_routing_create_host: routing sizes do not match the mesh");
    if (row_ptr[N] != nnz || int64_t(vec_offsets[N]) != E * k || int64_t(mat_offsets[nnz]) != E * k * k)
        return set_error(TGK_ERR_INPUT, "tgk_routing_create_host: inconsistent routing arrays");
    int hit = 0;
    return routing_from_arrays(m, components, N, E, k, nnz, row_ptr, col_idx, vec_offsets, vec_slots, mat_offsets,
                               mat_slots, as_stream(stream), &hit, out);
}

int tgk_routing_copy(const tgk_routing* r, int64_t* row_ptr, int64_t* col_idx, uint32_t* slot_of,
                     uint32_t* vec_offsets, uint32_t* vec_slots, uint32_t* mat_offsets,
                     uint32_t* mat_slots) {
    using namespace tgk;
    auto cp = [](void* dst, const void* src, size_t bytes) -> int {
        if (!dst) return TGK_OK;
        if (!src) return set_error(TGK_ERR_INPUT, "tgk_routing_copy: array not built (use TGK_ROUTING_SEGMENTS)");
        CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        return TGK_OK;
    };
    const size_t Ek = static_cast<size_t>(r->E) * r->k;
    TGK_TRY(cp(row_ptr, r->row_ptr, (r->N + 1) * sizeof(int64_t)));
    TGK_TRY(cp(col_idx, r->col_idx, r->nnz * sizeof(int64_t)));
    TGK_TRY(cp(slot_of, r->components == 1 ? r->slot_of : nullptr, Ek * r->k * sizeof(uint32_t)));
    TGK_TRY(cp(vec_offsets, r->vec_offsets, (r->N + 1) * sizeof(uint32_t)));
    TGK_TRY(cp(vec_slots, r->vec_slots, Ek * sizeof(uint32_t)));
    TGK_TRY(cp(mat_offsets, r->mat_offsets, (r->nnz + 1) * sizeof(uint32_t)));
    TGK_TRY(cp(mat_slots, r->mat_slots, Ek * r->k * sizeof(uint32_t)));
    return TGK_OK;
}

}  // extern "C"
