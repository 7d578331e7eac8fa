// CUDA plumbing shared by the .cu translation units of libtgk.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "tgk_internal.hpp"

namespace tgk {

inline int cuda_fail(cudaError_t e, const char* what) {
    return set_error(TGK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(call)                                            \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::tgk::cuda_fail(_e, #call); \
    } while (0)

#define KERNEL_CHECK(name)                                               \
    do {                                                                 \
        cudaError_t _e = cudaGetLastError();                             \
        if (_e != cudaSuccess) return ::tgk::cuda_fail(_e, "launch " name); \
    } while (0)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Owning device buffer for temporaries.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    int alloc(size_t count) {
        reset();
        n = count;
        if (count == 0) return TGK_OK;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess) {
            p = nullptr;
            return cuda_fail(e, "cudaMalloc");
        }
        return TGK_OK;
    }
    T* release() {
        T* r = p;
        p = nullptr;
        n = 0;
        return r;
    }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

inline int ensure_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return set_error(TGK_ERR_CUDA, "no usable CUDA device (libtgk has no CPU fallback)");
    return TGK_OK;
}

inline unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    return static_cast<unsigned>(g);
}

// Per-device caches (a process may drive several GPUs): the SM count, and a
// kernel instance's raised dynamic shared-memory limit (`done` is the call
// site's static array of kMaxDevices sizes).
constexpr int kMaxDevices = 64;
inline int sm_count() {
    static int n[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev >= kMaxDevices) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }
    if (n[dev] == 0) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
    return n[dev] > 0 ? n[dev] : 148;
}
template <class Kern>
int raise_smem_limit(Kern kern, size_t smem, size_t* done) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < kMaxDevices && done[dev] >= smem) return TGK_OK;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (dev < kMaxDevices) done[dev] = smem;
    return TGK_OK;
}

// Device-side first-bad-element reporter (smallest index wins: deterministic).
struct BadElem {
    unsigned long long* flag;  // init to ~0ull
};

}  // namespace tgk
