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
// block owns R CSR rows (mesh nodes, compact in space) and recomputes every
// element incident to them ("halo"), in ascending element order, in chunks of
// R elements (one per thread).  For every owned row the incidences (element,
// local node a, CSR positions of the element's nodes within the row) are
// stored per chunk as packed 32-bit records, grouped by row, ascending element
// within a row — so each CSR value is folded in ascending element order, the
// reference's order (routing.cpp:117-124).
constexpr int kMaxRowLen = 32;  // CSR row length limit of the packed record (5-bit positions)
constexpr int kPlanSlots = 3;   // plans cached per routing, keyed by (rows per block, chunk size)

struct PlanHost {
    int R = 256;                         // rows per block
    int C = 256;                         // halo elements per chunk (= threads per block)
    int64_t n_blocks = 0;
    int lmax = 0;                        // max CSR row length
    int max_chunk_recs = 0;              // largest record segment of one chunk (padded)
    std::vector<int64_t> row_off;        // n_blocks+1 into rows
    std::vector<uint32_t> rows;          // owned node ids, ascending within a block
    std::vector<int64_t> rows_rp;        // per owned row: row_ptr[row] | row length << 56
    std::vector<int64_t> halo_off;       // n_blocks+1 into halo
    std::vector<uint32_t> halo;          // incident element ids, level-ordered within a block
    int max_bnodes = 0;                  // largest block node table
    std::vector<int64_t> bnode_off;      // n_blocks+1 into bnodes
    std::vector<uint32_t> bnodes;        // per block: sorted unique nodes of its halo elements
    std::vector<uint16_t> halo_lconn;    // 4 block-local node indices per halo element (TRI3: 4th = 0)
    std::vector<int64_t> chunk_off;      // per block: first chunk index (n_blocks+1)
    std::vector<int64_t> chunk_rec_off;  // per chunk: first record (multiple of 4), total+1
    std::vector<uint16_t> chunk_row_off; // per chunk: R+8 u16 row offsets into its records
    std::vector<uint32_t> recs;          // packed records (chunk segments padded to 16 B)
};

struct PlanDev {
    int R = 0, C = 0;
    int64_t n_blocks = 0;
    int lmax = 0;
    int max_chunk_recs = 0;
    int64_t* row_off = nullptr;
    uint32_t* rows = nullptr;
    int64_t* rows_rp = nullptr;
    int64_t* halo_off = nullptr;
    uint32_t* halo = nullptr;
    int max_bnodes = 0;
    int64_t* bnode_off = nullptr;
    uint32_t* bnodes = nullptr;
    uint16_t* halo_lconn = nullptr;
    int64_t* chunk_off = nullptr;
    int64_t* chunk_rec_off = nullptr;
    uint16_t* chunk_row_off = nullptr;
    uint32_t* recs = nullptr;
    int64_t bytes = 0;
    int64_t n_halo = 0, n_records = 0;
    int max_block_halo = 0, max_block_recs = 0, max_block_chunks = 0;  // per-block maxima (batched kernel)
    void release();
};

inline int row_off_stride(int R) { return R + 8; }  // u16 entries per chunk (16-byte multiple)

// record layout: bits 0-7 element index within the chunk, 8-9 local node a
// (the element's node that is this row), 10-14 / 15-19 / 20-24 CSR positions
// (within the row) of the element's OTHER nodes b != a in ascending b,
// 25-29 the row's diagonal position.  The fused kernel stores each local
// tensor row a "rotated" to match: [K_aa, K_ab for b != a ascending].
TGK_HD inline uint32_t pack_rec(int hl, int a, const int* pos, int k) {
    uint32_t r = uint32_t(hl) | (uint32_t(a) << 8);
    int j = 0;
    for (int b = 0; b < k; ++b)
        if (b != a) r |= uint32_t(pos[b]) << (10 + 5 * j++);
    return r | (uint32_t(pos[a]) << 25);
}

std::vector<uint32_t> order_block_halo(int k, const int32_t* conn, const uint32_t* rows, int64_t nrows,
                                       const uint32_t* vec_offsets, const uint32_t* vec_slots, int64_t elem_lo,
                                       int64_t elem_hi, int C);
std::vector<uint32_t> morton_order(int kind, int64_t N, const double* nodes, int64_t row_lo, int64_t row_hi);

// Builds the plan on the host from the scalar routing (row_ptr, vec segment
// map = node->incidence CSR in ascending slot order, slot_of) for the owned
// row range [row_lo, row_hi) with R rows per block.
int build_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn,
               const int64_t* row_ptr, const uint32_t* vec_offsets, const uint32_t* vec_slots,
               const uint32_t* slot_of, int64_t row_lo, int64_t row_hi, int64_t elem_lo, int64_t elem_hi, int R,
               int C, PlanHost& out);

// Entry plan of the batched kernel (plan_entries.cpp, batched.cu): blocks of
// R owned rows with their whole halo; per owned CSR entry the list of its
// contributions (halo element | dot-product index << 16, ascending element)
// so a thread folds the entry in a register.  Per-entry offsets (coff) and
// per-row load offsets (fcoff) are block-relative and stored n+1 per block
// (block b's segment starts at ent_off[b] + b, resp. row_off[b] + b).
struct EntryPlanHost {
    int R = 64;
    int64_t n_blocks = 0;
    int max_halo = 0, max_bnodes = 0, max_contrib = 0, max_fcontrib = 0, max_entries = 0, max_clen = 0;
    std::vector<int64_t> row_off, halo_off, bnode_off, ent_off, contrib_off, fcontrib_off;
    std::vector<uint32_t> rows, halo, bnodes, contrib, fcontrib, coff, fcoff;
    std::vector<uint64_t> hconn;  // 4 x u16 block-local node indices per halo element
    std::vector<int64_t> epos;    // CSR position of each folded entry
    std::vector<int64_t> epos2;   // mirrored position (j, i) stored with the same value, or -1
};

struct EntryPlanDev {
    int R = 0;
    int64_t n_blocks = 0;
    int max_halo = 0, max_bnodes = 0, max_contrib = 0, max_fcontrib = 0, max_entries = 0, max_clen = 0;
    const int64_t *row_off = nullptr, *halo_off = nullptr, *bnode_off = nullptr, *ent_off = nullptr,
                  *contrib_off = nullptr, *fcontrib_off = nullptr, *epos = nullptr, *epos2 = nullptr;
    const uint32_t *rows = nullptr, *halo = nullptr, *bnodes = nullptr, *contrib = nullptr, *fcontrib = nullptr,
                   *coff = nullptr, *fcoff = nullptr;
    const uint64_t* hconn = nullptr;
    void* blob = nullptr;  // one device allocation holding every array
    int64_t bytes = 0;
    void release();
};

// Element-group plan of the adjoint transpose gather (plan_entries.cpp,
// adjoint.cu): elements in Morton order of their centroids, cut into groups
// of G; per group the element ids, the sorted unique nodes and each element's
// group-local node indices (4 x u16).  A block stages the group's lambda_b /
// U_b values once per field instead of gathering them once per element.
struct GroupPlanHost {
    int G = 256;
    int64_t n_groups = 0;
    int max_nodes = 0;
    std::vector<int64_t> grp_off, node_off;
    std::vector<uint32_t> elems, gnodes;
    std::vector<uint64_t> lconn;
};

struct GroupPlanDev {
    int G = 0;
    int64_t n_groups = 0;
    int max_nodes = 0;
    const int64_t *grp_off = nullptr, *node_off = nullptr;
    const uint32_t *elems = nullptr, *gnodes = nullptr;
    const uint64_t* lconn = nullptr;
    void* blob = nullptr;
    int64_t bytes = 0;
    void release();
};

int build_group_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn, int G,
                     GroupPlanHost& P);

// Fast-mode plan (plan_fast.cpp, fast.cu k_fast_scalar): blocks of R owned
// rows with their whole halo resident in shared memory; per owned CSR entry
// its element-to-slot list (u16 items = halo index | value index << 12),
// folded in a register by one lane.  Entry descriptor (u32): bits 0-8 local
// row, 9-14 position in the row (63: none), 15 diagonal entry (also the row's
// load), 16-24 / 25-30 local row / position of the mirrored entry (j, i),
// 31 mirrored.  kFastIdle marks a padding slot.
constexpr int kFastMaxRows = 511;
constexpr int kFastMaxRowLen = 62;
constexpr int kFastNoPos = 63;
constexpr int kFastMaxHalo = 4095;
constexpr uint32_t kFastIdle = 0xffffffffu;
constexpr uint32_t kFastPart = 0xfffffffeu;  // lanes 1.. of a split diagonal entry
TGK_HD constexpr int kFastDiagSplit(int k) { return k == 4 ? 4 : 2; }
constexpr int kFastNotApplicable = -100;  // fast_scalar_assemble: take the exact kernel
struct FastPlanHost {
    int R = 64;
    int64_t n_blocks = 0;
    int max_halo = 0, max_bnodes = 0, max_rows = 0;
    std::vector<int64_t> row_off, halo_off, bnode_off, ent_off, item_off;  // n_blocks+1 each (ent_off: multiples of 32)
    std::vector<uint32_t> rows, helem, bnodes, desc;
    std::vector<uint64_t> hconn;     // 4 x u16 block-local node indices per halo element
    std::vector<uint32_t> list_off;  // per block, per entry: item offsets (block-relative), n+1 per block
    std::vector<uint16_t> items;     // generic items: halo index | (a * 4 + b) << 12 (row node a, column node b)
};

// value-row formats of the fast kernel (plan_fast.cpp ensure_fast_plan)
constexpr int kFastFmtK16 = 0;   // stiffness [+ load]
constexpr int kFastFmtKS32 = 1;  // stiffness + unit mass [+ scalar load]
constexpr int kFastFmtS16 = 2;   // coefficient mass
constexpr int kFastFmtE16 = 3;   // vector elasticity (3 x 3 / 2 x 2 blocks per scalar entry)
constexpr int kFastPlanSlots = 3;

// Device form: two byte records per block, each one TMA bulk copy into shared
// memory (fast.cu).  Record A (prologue + phase A): header {int64 halo base,
// u32 rows, halo, nodes, tile}, per row int64 CSR offset, u32 row id, u16 tile
// offset (n+1), u32 node table, u64 block-local connectivity.  Record B
// (phase B): header {u32 entries, warp groups}, u32 descriptors, u32 warp-group
// word offsets (n+1), the item words.  Sections 16-byte aligned.
struct FastPlanDev {
    int R = 0, fmt = -1, MH = 0;
    bool fnodal = false;
    int64_t n_blocks = 0;
    int max_halo = 0, max_bnodes = 0, max_rows = 0, max_tile = 0, max_len = 0;
    int max_rec_a = 0, max_rec_b = 0;  // bytes
    int hc8 = 0;                       // block-local connectivity as 4 x u8 (every node table <= 255), else 4 x u16
    int64_t n_halo = 0, n_items = 0, n_words = 0, n_entries = 0;
    int64_t row_lo = -1, row_hi = -1, elem_lo = -1, elem_hi = -1;  // the ranges it was built for
    const int64_t *rec_a_off = nullptr, *rec_b_off = nullptr;       // n_blocks+1 byte offsets
    const unsigned char *rec_a = nullptr, *rec_b = nullptr;
    const uint32_t* helem = nullptr;  // halo element ids (per-element fields, bad-element report)
    void* blob = nullptr;
    int64_t bytes = 0;
    void release();
};
int fast_value_rows(int k, int fmt, bool fnodal);

// Returns TGK_ERR_INPUT WITHOUT an error message when the fast layout does not
// apply (row longer than kFastMaxRowLen, halo larger than kFastMaxHalo):
// the caller then takes the exact kernel.
int build_fast_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn,
                    const int64_t* row_ptr, const uint32_t* vec_offsets, const uint32_t* vec_slots,
                    const uint32_t* slot_of, int64_t row_lo, int64_t row_hi, int64_t elem_lo, int64_t elem_hi,
                    int R, FastPlanHost& P);

int build_entry_plan(int kind, int64_t N, const double* nodes, const int32_t* conn, const int64_t* row_ptr,
                     const uint32_t* vec_offsets, const uint32_t* vec_slots, const uint32_t* slot_of,
                     int64_t row_lo, int64_t row_hi, int R, EntryPlanHost& P);

}  // namespace tgk

// ----------------------------------------------------------------- handles
struct tgk_mesh {
    int kind = TGK_TET4;
    int d = 3, k = 4;
    int64_t N = 0, E = 0;
    double* nodes = nullptr;     // device, N x d
    int32_t* conn = nullptr;     // device, E x k
    int64_t* staging = nullptr;  // device int64 connectivity staging for host uploads
    int div_safe = -1;           // coordinates certified for Markstein division (-1 unknown)
    uint64_t conn_version = 0;   // bumped whenever an upload changes the connectivity
    bool owned = false;
    // persistent validation scratch (no per-call cudaMalloc / cudaFree, which
    // would serialise the device): 2 device flags, 2 pinned host words
    unsigned long long* d_flags = nullptr;
    unsigned long long* h_flags = nullptr;
};

struct tgk_routing {
    int64_t N = 0, E = 0, nnz = 0;  // DoF-level
    int k = 0, components = 1;
    int lmax = 0;                    // max scalar row length
    const tgk_mesh* mesh = nullptr;
    uint64_t mesh_version = 0;       // the mesh's conn_version the routing was built for
    int64_t* row_ptr = nullptr;
    int64_t* col_idx = nullptr;
    uint32_t* slot_of = nullptr;     // scalar routing only
    uint32_t* vec_offsets = nullptr;
    uint32_t* vec_slots = nullptr;
    uint32_t* mat_offsets = nullptr;
    uint32_t* mat_slots = nullptr;
    // scalar (node-level) routing used by vector problems and the fused plan
    tgk_routing* scalar = nullptr;   // == this for components == 1
    tgk::PlanDev plan[tgk::kPlanSlots];
    tgk::EntryPlanDev entry_plan;    // batched kernel plan (built on first batched call)
    tgk::GroupPlanDev group_plan;    // adjoint gather plan (built on first adjoint call)
    tgk::FastPlanDev fast_plan[tgk::kFastPlanSlots];  // fast-mode plans (TGK_MODE_FAST), per R / format / ranges
    int fast_plan_next = 0;
    const tgk::FastPlanDev* fast_plan_used = nullptr;  // the plan of the latest fast-mode assembly
    int64_t own_lo = 0, own_hi = -1;  // owned scalar row range (-1: all rows)
    int64_t elem_lo = 0, elem_hi = -1;  // elements taking part in the fused assembly (-1: all)
    double* scr[6] = {};             // cached device scratch (materialised elasticity path)
    size_t scr_n[6] = {};
    unsigned long long* flags = nullptr;  // persistent device status words (4), see routing_flags
    double* scratch_K = nullptr;     // device output buffers of the host-buffer entry point
    double* scratch_F = nullptr;
    double* scratch_M = nullptr;
    ~tgk_routing();
};

namespace tgk {
// Build (once per R) and upload the fused plan of the routing's scalar part.
int ensure_plan(tgk_routing* r, int R, const PlanDev** out, int C = 0);  // C = 0: chunk size R
int ensure_entry_plan(tgk_routing* r, int R, const EntryPlanDev** out);
// The routing's 4 persistent device status words (allocated once: no per-call
// cudaMalloc / cudaFree, which would serialise the device).  A routing handle
// is used by one stream at a time.
int routing_flags(tgk_routing* r, unsigned long long** out);
int ensure_group_plan(tgk_routing* r, int G, const GroupPlanDev** out);
// Fast-mode plan for R rows per block over the routing's owned rows / element
// range; TGK_ERR_INPUT without a message when the fast layout does not apply.
int ensure_fast_plan(tgk_routing* r, int R, int fmt, bool fnodal, const FastPlanDev** out);
// status 2 when the mesh's connectivity changed (tgk_mesh_upload) after the
// routing was built from it: its pattern, slot map and plans are stale
int check_routing_fresh(const tgk_mesh* m, const tgk_routing* r);
struct ScalarRoutingHost {
    std::vector<double> nodes;
    std::vector<int32_t> conn;
    std::vector<int64_t> row_ptr;
    std::vector<uint32_t> vo, vs, slot;
};
int fetch_scalar_routing(const tgk_routing* r, ScalarRoutingHost& h);
}
