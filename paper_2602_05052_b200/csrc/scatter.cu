// The reference's independent correctness baseline scatter_add_oracle
// (routing.cpp:134-175) on the GPU, by a different algorithm than the
// routing build (routing.cu): every local contribution (e, a, b) becomes a
// (row, col) key with its flattened slot as payload; one stable radix sort
// groups equal (row, col) pairs in ascending slot order (= the reference's
// per-element scatter order, elements ascending), the distinct keys are the
// pattern (its per-row sort + unique, :143-158) and each run is summed from
// +0.0 in that order (:162-168) — bit-identical to the reference.  The load
// vector is the same over node keys.  Setup-style code (temporary buffers);
// used by tgfem.scatter_add_oracle.
#include <cub/cub.cuh>

#include <vector>

#include "cuda_util.cuh"
#include "tgk_internal.hpp"

namespace tgk {
namespace {

__global__ void k_pair_keys(const int32_t* conn, int64_t E, int k, uint64_t* keys, uint32_t* slots) {
    const int64_t n = E * k * k;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = s / (k * k), ab = s % (k * k), a = ab / k, b = ab % k;
        keys[s] = (uint64_t(uint32_t(conn[e * k + a])) << 32) | uint32_t(conn[e * k + b]);
        slots[s] = static_cast<uint32_t>(s);
    }
}

__global__ void k_node_keys(const int32_t* conn, int64_t Ek, uint64_t* keys, uint32_t* slots) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < Ek; s += (int64_t)gridDim.x * blockDim.x) {
        keys[s] = uint32_t(conn[s]);
        slots[s] = static_cast<uint32_t>(s);
    }
}

// one thread per run: values[t] = left fold from +0.0 of local[slot] over the run
__global__ void k_run_sum(const uint32_t* slots, const uint32_t* run_start, const uint32_t* run_len, int64_t n_runs,
                          const double* local, double* out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_runs; t += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        const uint32_t s0 = run_start[t], s1 = s0 + run_len[t];
        for (uint32_t u = s0; u < s1; ++u) v += local[slots[u]];
        out[t] = v;
    }
}

__global__ void k_pattern_from_keys(const uint64_t* ukeys, int64_t nnz, int64_t N, int64_t* offsets, int64_t* cols) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = int64_t(ukeys[t] >> 32);
        cols[t] = int64_t(ukeys[t] & 0xffffffffu);
        const int64_t prev = t == 0 ? -1 : int64_t(ukeys[t - 1] >> 32);
        for (int64_t i = prev + 1; i <= row; ++i) offsets[i] = t;  // rows prev+1 .. row start here
        if (t == nnz - 1)
            for (int64_t i = row + 1; i <= N; ++i) offsets[i] = nnz;
    }
}

// Sort (key, slot) pairs stably by key and run-length encode: sorted slots,
// run starts and lengths, distinct keys.
int sort_runs(DevBuf<uint64_t>& keys, DevBuf<uint32_t>& slots, int64_t n, int key_bits, cudaStream_t st,
              DevBuf<uint64_t>& ukeys, DevBuf<uint32_t>& sorted_slots, DevBuf<uint32_t>& run_start,
              DevBuf<uint32_t>& run_len, int64_t* n_runs) {
    DevBuf<uint64_t> keys_out;
    TGK_TRY(keys_out.alloc(n));
    TGK_TRY(sorted_slots.alloc(n));
    size_t tmp_bytes = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_out.p, slots.p, sorted_slots.p, n, 0,
                                             key_bits, st));
    DevBuf<unsigned char> tmp;
    TGK_TRY(tmp.alloc(tmp_bytes + 1));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys_out.p, slots.p, sorted_slots.p, n, 0,
                                             key_bits, st));
    TGK_TRY(ukeys.alloc(n));
    TGK_TRY(run_len.alloc(n));
    DevBuf<int64_t> d_runs;
    TGK_TRY(d_runs.alloc(1));
    tmp_bytes = 0;
    CUDA_TRY(cub::DeviceRunLengthEncode::Encode(nullptr, tmp_bytes, keys_out.p, ukeys.p, run_len.p, d_runs.p, n, st));
    TGK_TRY(tmp.alloc(tmp_bytes + 1));
    CUDA_TRY(cub::DeviceRunLengthEncode::Encode(tmp.p, tmp_bytes, keys_out.p, ukeys.p, run_len.p, d_runs.p, n, st));
    CUDA_TRY(cudaMemcpyAsync(n_runs, d_runs.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    TGK_TRY(run_start.alloc(*n_runs + 1));
    tmp_bytes = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, run_len.p, run_start.p, *n_runs, st));
    TGK_TRY(tmp.alloc(tmp_bytes + 1));
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, run_len.p, run_start.p, *n_runs, st));
    return TGK_OK;
}

}  // namespace
}  // namespace tgk

extern "C" int tgk_scatter_add(const tgk_mesh* m, const double* local_matrices, const double* local_vectors,
                               int64_t* nnz, int64_t* offsets, int64_t* cols, double* values, double* F) {
    using namespace tgk;
    if (!m || !nnz) return set_error(TGK_ERR_INPUT, "scatter_add: null argument");
    TGK_TRY(ensure_device());
    const int k = m->k;
    const int64_t E = m->E, N = m->N, n = E * k * k;
    if (n > int64_t(UINT32_MAX)) return set_error(TGK_ERR_INPUT, "scatter_add: more than 2^32-1 local slots");
    cudaStream_t st = nullptr;
    int nbits = 1;
    while ((int64_t(1) << nbits) < N) ++nbits;
    {
        DevBuf<uint64_t> keys, ukeys;
        DevBuf<uint32_t> slots, sorted, rs, rl;
        TGK_TRY(keys.alloc(n));
        TGK_TRY(slots.alloc(n));
        k_pair_keys<<<grid_for(n, 256), 256, 0, st>>>(m->conn, E, k, keys.p, slots.p);
        KERNEL_CHECK("pair_keys");
        int64_t runs = 0;
        TGK_TRY(sort_runs(keys, slots, n, 32 + nbits, st, ukeys, sorted, rs, rl, &runs));
        *nnz = runs;
        if (offsets || cols) {
            DevBuf<int64_t> d_off, d_cols;
            TGK_TRY(d_off.alloc(N + 1));
            TGK_TRY(d_cols.alloc(runs));
            CUDA_TRY(cudaMemsetAsync(d_off.p, 0, sizeof(int64_t) * (N + 1), st));
            k_pattern_from_keys<<<grid_for(runs, 256), 256, 0, st>>>(ukeys.p, runs, N, d_off.p, d_cols.p);
            KERNEL_CHECK("pattern_from_keys");
            if (offsets) CUDA_TRY(cudaMemcpy(offsets, d_off.p, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost));
            if (cols) CUDA_TRY(cudaMemcpy(cols, d_cols.p, sizeof(int64_t) * runs, cudaMemcpyDeviceToHost));
        }
        if (values && local_matrices) {
            DevBuf<double> d_local, d_vals;
            TGK_TRY(d_local.alloc(n));
            TGK_TRY(d_vals.alloc(runs));
            CUDA_TRY(cudaMemcpy(d_local.p, local_matrices, sizeof(double) * n, cudaMemcpyHostToDevice));
            k_run_sum<<<grid_for(runs, 256), 256, 0, st>>>(sorted.p, rs.p, rl.p, runs, d_local.p, d_vals.p);
            KERNEL_CHECK("run_sum");
            CUDA_TRY(cudaMemcpy(values, d_vals.p, sizeof(double) * runs, cudaMemcpyDeviceToHost));
        } else if (values) {
            std::vector<double> z(static_cast<size_t>(runs), 0.0);
            std::copy(z.begin(), z.end(), values);
        }
    }
    if (F) {
        std::vector<double> f(static_cast<size_t>(N), 0.0);
        if (local_vectors) {  // F[g_a] += Fe[a], elements ascending (:169-172)
            const int64_t Ek = E * k;
            DevBuf<uint64_t> keys, ukeys;
            DevBuf<uint32_t> slots, sorted, rs, rl;
            TGK_TRY(keys.alloc(Ek));
            TGK_TRY(slots.alloc(Ek));
            k_node_keys<<<grid_for(Ek, 256), 256, 0, st>>>(m->conn, Ek, keys.p, slots.p);
            KERNEL_CHECK("node_keys");
            int64_t runs = 0;
            TGK_TRY(sort_runs(keys, slots, Ek, nbits, st, ukeys, sorted, rs, rl, &runs));
            DevBuf<double> d_lv, d_f;
            TGK_TRY(d_lv.alloc(Ek));
            TGK_TRY(d_f.alloc(runs));
            CUDA_TRY(cudaMemcpy(d_lv.p, local_vectors, sizeof(double) * Ek, cudaMemcpyHostToDevice));
            k_run_sum<<<grid_for(runs, 256), 256, 0, st>>>(sorted.p, rs.p, rl.p, runs, d_lv.p, d_f.p);
            KERNEL_CHECK("run_sum");
            std::vector<uint64_t> hk(static_cast<size_t>(runs));
            std::vector<double> hv(static_cast<size_t>(runs));
            CUDA_TRY(cudaMemcpy(hk.data(), ukeys.p, sizeof(uint64_t) * runs, cudaMemcpyDeviceToHost));
            CUDA_TRY(cudaMemcpy(hv.data(), d_f.p, sizeof(double) * runs, cudaMemcpyDeviceToHost));
            for (int64_t t = 0; t < runs; ++t) f[hk[t]] = hv[t];  // nodes without elements stay +0.0
        }
        std::copy(f.begin(), f.end(), F);
    }
    return TGK_OK;
}
