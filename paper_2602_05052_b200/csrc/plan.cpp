// Host construction of the fused-assembly row-block plan (see tgk_internal.hpp).
//
// Inputs are the scalar routing arrays (bit-identical to the reference's
// build_routing): row_ptr (CsrPattern::offsets), the node incidence CSR
// vec_offsets/vec_slots (ascending slot e*k+a per node, routing.cpp:47-62) and
// the element-to-slot map slot_of.  Steps:
//  1. order nodes along a Morton curve of their coordinates and cut the order
//     into blocks of kRowsPerBlock nodes (compact in space => small halos);
//  2. per block, the halo = unique elements incident to its nodes, ordered by
//     level in the per-row precedence chains (see below), then id;
//  3. per block and halo chunk, one packed record per (owned row, incident
//     element): element index within the chunk, local node a, and the CSR
//     position (t - row_ptr[row]) of each of the element's nodes in the row.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

#include "tgk_internal.hpp"

namespace tgk {

namespace {

uint64_t spread3(uint64_t x) {  // 21 bits -> every third bit
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

uint64_t spread2(uint64_t x) {  // 32 bits -> every second bit
    x &= 0xffffffffull;
    x = (x | x << 16) & 0x0000ffff0000ffffull;
    x = (x | x << 8) & 0x00ff00ff00ff00ffull;
    x = (x | x << 4) & 0x0f0f0f0f0f0f0f0full;
    x = (x | x << 2) & 0x3333333333333333ull;
    x = (x | x << 1) & 0x5555555555555555ull;
    return x;
}

}  // namespace

// Owned rows [row_lo, row_hi) in Morton order of their coordinates.
std::vector<uint32_t> morton_order(int kind, int64_t N, const double* nodes, int64_t row_lo, int64_t row_hi) {
    const int d = element_dim(kind);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t i = 0; i < N; ++i)
        for (int c = 0; c < d; ++c) {
            lo[c] = std::min(lo[c], nodes[i * d + c]);
            hi[c] = std::max(hi[c], nodes[i * d + c]);
        }
    double span = 0;
    for (int c = 0; c < d; ++c) span = std::max(span, hi[c] - lo[c]);
    if (!(span > 0)) span = 1.0;
    const double scale = (d == 3 ? double((1u << 21) - 1) : double(0xffffffffu)) / span;
    std::vector<std::pair<uint64_t, uint32_t>> key;
    key.reserve(static_cast<size_t>(row_hi - row_lo));
    for (int64_t i = row_lo; i < row_hi; ++i) {
        uint64_t m = 0;
        for (int c = 0; c < d; ++c) {
            const uint64_t q = static_cast<uint64_t>((nodes[i * d + c] - lo[c]) * scale);
            m |= (d == 3 ? spread3(q) : spread2(q)) << c;
        }
        key.push_back({m, static_cast<uint32_t>(i)});
    }
    std::sort(key.begin(), key.end());
    std::vector<uint32_t> out(key.size());
    for (size_t i = 0; i < key.size(); ++i) out[i] = key[i].second;
    return out;
}

// The halo of a row block (every element incident to one of its rows, inside
// [elem_lo, elem_hi)) in fold-compatible order.  Level schedule: every owned
// row's elements must be folded in ascending id, i.e. they form a chain;
// level(e) = longest chain ending at e.  Ordering the halo by (level, id) keeps
// each row's elements ascending across and within chunks of C while giving
// every row at most one element per level -> balanced folds.  Within a chunk
// the order is free (every consumer folds by element id): each chunk is
// ordered by the element's first node so the lanes of a warp gather nearby
// node-table entries (TGK_CHUNK_SORT=0 disables).
std::vector<uint32_t> order_block_halo(int k, const int32_t* conn, const uint32_t* rows, int64_t nrows,
                                       const uint32_t* vec_offsets, const uint32_t* vec_slots, int64_t elem_lo,
                                       int64_t elem_hi, int C) {
    auto in_range = [elem_lo, elem_hi](uint32_t e) { return int64_t(e) >= elem_lo && int64_t(e) < elem_hi; };
    std::vector<uint32_t> tmp;
    for (int64_t i = 0; i < nrows; ++i) {
        const uint32_t row = rows[i];
        for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s)
            if (in_range(vec_slots[s] / k)) tmp.push_back(vec_slots[s] / k);
    }
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    const int64_t nh = static_cast<int64_t>(tmp.size());
    std::vector<int> level(nh, 0);
    {
        std::vector<std::pair<uint32_t, uint32_t>> edges;  // (next, pred) as halo indices
        for (int64_t i = 0; i < nrows; ++i) {
            const uint32_t row = rows[i];
            int64_t prev = -1;
            for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s) {
                const uint32_t e = vec_slots[s] / k;
                if (!in_range(e)) continue;
                const int64_t hix = std::lower_bound(tmp.begin(), tmp.end(), e) - tmp.begin();
                if (prev >= 0) edges.push_back({static_cast<uint32_t>(hix), static_cast<uint32_t>(prev)});
                prev = hix;
            }
        }
        std::sort(edges.begin(), edges.end());  // by target: a topological order
        for (const auto& ed : edges) level[ed.first] = std::max(level[ed.first], level[ed.second] + 1);
    }
    std::vector<std::pair<int, uint32_t>> order(nh);
    for (int64_t h = 0; h < nh; ++h) order[h] = {level[h], tmp[h]};
    std::sort(order.begin(), order.end());
    static const bool chunk_sort = !(getenv("TGK_CHUNK_SORT") && atoi(getenv("TGK_CHUNK_SORT")) == 0);
    if (chunk_sort)
        for (int64_t c0 = 0; c0 < nh; c0 += C) {
            const int64_t c1 = std::min<int64_t>(nh, c0 + C);
            std::sort(order.begin() + c0, order.begin() + c1, [&](const auto& x, const auto& y) {
                const int32_t nx = conn[int64_t(x.second) * k], ny = conn[int64_t(y.second) * k];
                return nx != ny ? nx < ny : x.second < y.second;
            });
        }
    std::vector<uint32_t> out(nh);
    for (int64_t h = 0; h < nh; ++h) out[h] = order[h].second;
    return out;
}

int build_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn,
               const int64_t* row_ptr, const uint32_t* vec_offsets, const uint32_t* vec_slots,
               const uint32_t* slot_of, int64_t row_lo, int64_t row_hi, int64_t elem_lo, int64_t elem_hi, int R,
               int C, PlanHost& P) {
    // elements outside [elem_lo, elem_hi) take no part (multi-GPU slabs that
    // exchange interface partial sums instead of recomputing the halo)
    auto in_range = [elem_lo, elem_hi](uint32_t e) { return int64_t(e) >= elem_lo && int64_t(e) < elem_hi; };
    const int d = element_dim(kind), k = element_nodes(kind);
    (void)E;
    // R rows per block, chunks of C halo elements (C threads; R = C x rows per thread)
    if (R != 16 && R != 32 && R != 64 && R != 128 && R != 256)
        return set_error(TGK_ERR_INPUT, "fused plan: R must be 16, 32, 64, 128 or 256");
    if (C < 16 || C > 256 || C % 16)
        return set_error(TGK_ERR_INPUT, "fused plan: chunk size must be a multiple of 16 in [16, 256]");
    P.R = R;
    P.C = C;
    // --- 1. Morton order of the owned nodes
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t i = 0; i < N; ++i)
        for (int c = 0; c < d; ++c) {
            lo[c] = std::min(lo[c], nodes[i * d + c]);
            hi[c] = std::max(hi[c], nodes[i * d + c]);
        }
    const double span = [&] {
        double s = 0;
        for (int c = 0; c < d; ++c) s = std::max(s, hi[c] - lo[c]);
        return s > 0 ? s : 1.0;
    }();
    const double scale = (d == 3 ? double((1u << 21) - 1) : double(0xffffffffu)) / span;
    std::vector<std::pair<uint64_t, uint32_t>> key;
    key.reserve(static_cast<size_t>(row_hi - row_lo));
    for (int64_t i = row_lo; i < row_hi; ++i) {
        uint64_t m = 0;
        for (int c = 0; c < d; ++c) {
            const uint64_t q = static_cast<uint64_t>((nodes[i * d + c] - lo[c]) * scale);
            m |= (d == 3 ? spread3(q) : spread2(q)) << c;
        }
        key.push_back({m, static_cast<uint32_t>(i)});
    }
    const int64_t n_owned = static_cast<int64_t>(key.size());
    std::sort(key.begin(), key.end());

    int lmax = 0;
    for (int64_t i = 0; i < N; ++i) lmax = std::max<int>(lmax, static_cast<int>(row_ptr[i + 1] - row_ptr[i]));
    if (lmax > kMaxRowLen)
        return set_error(TGK_ERR_INPUT, "fused plan: CSR row longer than " +
                                            std::to_string(kMaxRowLen) + " entries");
    P.lmax = lmax;
    const int64_t nb = (n_owned + R - 1) / R;
    P.n_blocks = nb;
    P.row_off.resize(nb + 1);
    P.rows.resize(n_owned);
    for (int64_t b = 0; b <= nb; ++b) P.row_off[b] = std::min<int64_t>(b * R, n_owned);
    for (int64_t b = 0; b < nb; ++b) {
        for (int64_t i = P.row_off[b]; i < P.row_off[b + 1]; ++i) P.rows[i] = key[i].second;
        std::sort(P.rows.begin() + P.row_off[b], P.rows.begin() + P.row_off[b + 1]);
    }
    key.clear();
    key.shrink_to_fit();
    P.rows_rp.resize(n_owned + 1);
    for (int64_t i = 0; i < n_owned; ++i)  // CSR offset | row length << 56
        P.rows_rp[i] = row_ptr[P.rows[i]] | ((row_ptr[P.rows[i] + 1] - row_ptr[P.rows[i]]) << 56);
    P.rows_rp[n_owned] = 0;

    // --- 2/3. halos and records, blocks in parallel
    const int ros = row_off_stride(R);
    struct BlockOut {
        std::vector<uint32_t> halo;
        std::vector<uint16_t> row_off;  // nch x ros
        std::vector<uint32_t> recs;     // chunk segments, each padded to a multiple of 4
        std::vector<int64_t> chunk_sizes;
    };
    std::vector<BlockOut> out(nb);
    auto work = [&](int64_t b_begin, int64_t b_end) {
        for (int64_t b = b_begin; b < b_end; ++b) {
            BlockOut& o = out[b];
            const int64_t rs = P.row_off[b], re = P.row_off[b + 1];
            o.halo = order_block_halo(k, conn, P.rows.data() + rs, re - rs, vec_offsets, vec_slots, elem_lo, elem_hi, C);
            const int64_t nh = static_cast<int64_t>(o.halo.size());
            std::vector<std::pair<uint32_t, uint32_t>> where(nh);  // (element, position)
            for (int64_t h = 0; h < nh; ++h) where[h] = {o.halo[h], static_cast<uint32_t>(h)};
            std::sort(where.begin(), where.end());
            const int64_t nch = (nh + C - 1) / C;
            // records grouped chunk-major, then row, ascending element within a row
            std::vector<std::vector<uint32_t>> per_chunk(nch);
            std::vector<std::vector<uint16_t>> cnt(nch, std::vector<uint16_t>(R, 0));
            for (int64_t i = rs; i < re; ++i) {
                const int lr = static_cast<int>(i - rs);
                const uint32_t row = P.rows[i];
                const int64_t rp = row_ptr[row];
                for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s) {
                    const uint32_t slot = vec_slots[s];
                    const uint32_t e = slot / k;
                    if (!in_range(e)) continue;
                    const int a = static_cast<int>(slot % k);
                    const int64_t hpos =
                        std::lower_bound(where.begin(), where.end(), std::make_pair(e, 0u))->second;
                    const int64_t ch = hpos / C;
                    int pos[4] = {0, 0, 0, 0};
                    for (int bb = 0; bb < k; ++bb)
                        pos[bb] = static_cast<int>(slot_of[static_cast<int64_t>(slot) * k + bb] - rp);
                    per_chunk[ch].push_back(pack_rec(static_cast<int>(hpos % C), a, pos, k));
                    ++cnt[ch][lr];
                }
            }
            o.chunk_sizes.resize(nch);
            o.row_off.assign(nch * ros, 0);
            for (int64_t ch = 0; ch < nch; ++ch) {
                // per_chunk[ch] was appended row by row in ascending row order: already grouped
                uint16_t acc = 0;
                for (int lr = 0; lr < R; ++lr) {
                    o.row_off[ch * ros + lr] = acc;
                    acc = static_cast<uint16_t>(acc + cnt[ch][lr]);
                }
                for (int j = R; j < ros; ++j) o.row_off[ch * ros + j] = acc;
                auto& v = per_chunk[ch];
                while (v.size() % 4) v.push_back(0);
                o.chunk_sizes[ch] = static_cast<int64_t>(v.size());
                o.recs.insert(o.recs.end(), v.begin(), v.end());
            }
        }
    };
    const int nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    {
        std::vector<std::thread> pool;
        const int64_t per = (nb + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            const int64_t b0 = t * per, b1 = std::min(nb, b0 + per);
            if (b0 < b1) pool.emplace_back(work, b0, b1);
        }
        for (auto& th : pool) th.join();
    }
    // --- concatenate
    P.halo_off.assign(nb + 1, 0);
    P.chunk_off.assign(nb + 1, 0);
    for (int64_t b = 0; b < nb; ++b) {
        P.halo_off[b + 1] = P.halo_off[b] + static_cast<int64_t>(out[b].halo.size());
        P.chunk_off[b + 1] = P.chunk_off[b] + static_cast<int64_t>(out[b].chunk_sizes.size());
    }
    const int64_t total_chunks = P.chunk_off[nb];
    for (int64_t b = 0; b < nb; ++b)
        if (P.chunk_off[b + 1] - P.chunk_off[b] > 255)
            return set_error(TGK_ERR_INPUT, "fused plan: a row block needs more than 255 halo chunks");
    P.halo.resize(P.halo_off[nb]);
    P.halo_lconn.assign(P.halo.size() * 4, 0);
    P.chunk_row_off.resize(total_chunks * ros);
    P.chunk_rec_off.assign(total_chunks + 1, 0);
    int64_t nrec = 0;
    int maxrec = 0;
    for (int64_t b = 0; b < nb; ++b) {
        std::copy(out[b].halo.begin(), out[b].halo.end(), P.halo.begin() + P.halo_off[b]);
        std::copy(out[b].row_off.begin(), out[b].row_off.end(), P.chunk_row_off.begin() + P.chunk_off[b] * ros);
        for (size_t ch = 0; ch < out[b].chunk_sizes.size(); ++ch) {
            P.chunk_rec_off[P.chunk_off[b] + ch] = nrec;
            nrec += out[b].chunk_sizes[ch];
            maxrec = std::max<int>(maxrec, static_cast<int>(out[b].chunk_sizes[ch]));
        }
    }
    P.chunk_rec_off[total_chunks] = nrec;
    P.max_chunk_recs = maxrec;
    P.recs.resize(nrec);
    for (int64_t b = 0; b < nb; ++b)
        std::copy(out[b].recs.begin(), out[b].recs.end(), P.recs.begin() + P.chunk_rec_off[P.chunk_off[b]]);
    // block node tables (the halo's nodes, staged in shared memory by the
    // kernel) and block-local connectivity
    P.bnode_off.assign(nb + 1, 0);
    std::vector<std::vector<uint32_t>> bn(nb);
    auto node_work = [&](int64_t b_begin, int64_t b_end) {
        for (int64_t b = b_begin; b < b_end; ++b) {
            auto& v = bn[b];
            for (int64_t h = P.halo_off[b]; h < P.halo_off[b + 1]; ++h)
                for (int a = 0; a < k; ++a) v.push_back(static_cast<uint32_t>(conn[static_cast<int64_t>(P.halo[h]) * k + a]));
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            for (int64_t h = P.halo_off[b]; h < P.halo_off[b + 1]; ++h)
                for (int a = 0; a < k; ++a) {
                    const uint32_t g = static_cast<uint32_t>(conn[static_cast<int64_t>(P.halo[h]) * k + a]);
                    P.halo_lconn[h * 4 + a] = static_cast<uint16_t>(std::lower_bound(v.begin(), v.end(), g) - v.begin());
                }
        }
    };
    {
        std::vector<std::thread> pool;
        const int64_t per = (nb + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            const int64_t b0 = t * per, b1 = std::min(nb, b0 + per);
            if (b0 < b1) pool.emplace_back(node_work, b0, b1);
        }
        for (auto& th : pool) th.join();
    }
    int maxbn = 0;
    for (int64_t b = 0; b < nb; ++b) {
        P.bnode_off[b + 1] = P.bnode_off[b] + static_cast<int64_t>(bn[b].size());
        maxbn = std::max<int>(maxbn, static_cast<int>(bn[b].size()));
    }
    if (maxbn > 65535) return set_error(TGK_ERR_INPUT, "fused plan: block node table exceeds 65535 nodes");
    P.max_bnodes = maxbn;
    P.bnodes.resize(P.bnode_off[nb]);
    for (int64_t b = 0; b < nb; ++b) std::copy(bn[b].begin(), bn[b].end(), P.bnodes.begin() + P.bnode_off[b]);
    return TGK_OK;
}

}  // namespace tgk
