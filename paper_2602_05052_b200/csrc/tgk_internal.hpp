// Internal declarations shared by the host (C++) and device (CUDA) halves of
// libtgk.so.  Not part of the public ABI (see include/tgk.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tgk.h"

#ifdef __CUDACC__
#define TGK_HD __host__ __device__
#else
#define TGK_HD
#endif

namespace tgk {

// ----------------------------------------------------------------- errors
int set_error(int code, const std::string& msg);
const std::string& last_error();

#define TGK_TRY(expr)                   \
    do {                                \
        int _rc = (expr);               \
        if (_rc != TGK_OK) return _rc;  \
    } while (0)

inline int element_dim(int kind) { return kind == TGK_TET4 ? 3 : 2; }
inline int element_nodes(int kind) { return kind == TGK_TRI3 ? 3 : 4; }

// ----------------------------------------------------------------- fused plan
// Row-block ("node block") plan for the fused Map+Reduce kernel.  Each CUDA
// block owns a set of CSR rows (mesh nodes) and recomputes every element
// incident to them ("halo"), in ascending element order, in chunks of
// kChunk elements.  For every owned row the incidences (element, local node
// a, CSR positions of the element's nodes within the row) are stored per
// chunk as packed 32-bit records, grouped by row, ascending element within
// a row — so each CSR value is folded in ascending element order, the
// reference's order (routing.cpp:117-124).
constexpr int kRowsPerBlock = 256;  // owned rows per CUDA block (= threads)
constexpr int kChunk = 256;         // halo elements per chunk (= threads)
constexpr int kMaxRowLen = 32;      // CSR row length limit of the packed record (5-bit positions)

struct PlanHost {
    int64_t n_blocks = 0;
    int lmax = 0;                        // max CSR row length
    std::vector<int64_t> row_off;        // n_blocks+1 into rows
    std::vector<uint32_t> rows;          // owned node ids, ascending within a block
    std::vector<int64_t> halo_off;       // n_blocks+1 into halo
    std::vector<uint32_t> halo;          // incident element ids, ascending within a block
    std::vector<int64_t> chunk_off;      // per block: first chunk index (n_blocks+1)
    std::vector<int64_t> chunk_rec_off;  // per chunk: first record (total_chunks+1)
    std::vector<uint8_t> chunk_cnt;      // per chunk x kRowsPerBlock: records of that row in the chunk
    std::vector<uint32_t> recs;          // packed records
};

struct PlanDev {
    int64_t n_blocks = 0;
    int lmax = 0;
    int64_t* row_off = nullptr;
    uint32_t* rows = nullptr;
    int64_t* halo_off = nullptr;
    uint32_t* halo = nullptr;
    int64_t* chunk_off = nullptr;
    int64_t* chunk_rec_off = nullptr;
    uint8_t* chunk_cnt = nullptr;
    uint32_t* recs = nullptr;
    int64_t bytes = 0;
    int64_t n_halo = 0, n_records = 0;
};

// record layout: bits 0-7 element index within the chunk, 8-9 local node a,
// 10+5b.. CSR position of local node b's column within the row.
TGK_HD inline uint32_t pack_rec(int hl, int a, const int* pos, int k) {
    uint32_t r = uint32_t(hl) | (uint32_t(a) << 8);
    for (int b = 0; b < k; ++b) r |= uint32_t(pos[b]) << (10 + 5 * b);
    return r;
}

// Builds the plan on the host from the scalar routing (row_ptr, vec segment
// map = node->incidence CSR in ascending slot order, slot_of).
int build_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn,
               const int64_t* row_ptr, const uint32_t* vec_offsets, const uint32_t* vec_slots,
               const uint32_t* slot_of, int64_t row_lo, int64_t row_hi, PlanHost& out);

}  // namespace tgk

// ----------------------------------------------------------------- handles
struct tgk_mesh {
    int kind = TGK_TET4;
    int d = 3, k = 4;
    int64_t N = 0, E = 0;
    double* nodes = nullptr;  // device, N x d
    int32_t* conn = nullptr;  // device, E x k
    int64_t* staging = nullptr;  // device int64 connectivity staging for host uploads
    bool owned = false;
};

struct tgk_routing {
    int64_t N = 0, E = 0, nnz = 0;  // DoF-level
    int k = 0, components = 1;
    int lmax = 0;                    // max scalar row length
    const tgk_mesh* mesh = nullptr;
    int64_t* row_ptr = nullptr;
    int64_t* col_idx = nullptr;
    uint32_t* slot_of = nullptr;     // scalar routing only
    uint32_t* vec_offsets = nullptr;
    uint32_t* vec_slots = nullptr;
    uint32_t* mat_offsets = nullptr;
    uint32_t* mat_slots = nullptr;
    // scalar (node-level) routing used by vector problems and the fused plan
    tgk_routing* scalar = nullptr;   // == this for components == 1
    tgk::PlanDev plan;
    bool has_plan = false;
    int64_t own_lo = 0, own_hi = -1;  // owned scalar row range (-1: all rows)
    double* scratch_K = nullptr;     // device output buffers of the host-buffer entry point
    double* scratch_F = nullptr;
    double* scratch_M = nullptr;
    ~tgk_routing();
};
