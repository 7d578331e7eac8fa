// Host construction of the v5 fused-assembly plan (fused5.cu).
//
// Same decomposition as v3 (plan.cpp): blocks of R owned rows (Morton-compact
// mesh nodes), each block's halo (elements incident to its rows) ordered by
// level in the per-row ascending element chains, a block node table and
// 4 x u16 block-local connectivity per halo element, chunks of R halo
// elements.  New in v5: per chunk, only the owned rows that have records in it
// ("active rows") become WORK ITEMS (local row, first record, record count),
// sorted by record count, descending, so the threads of a warp fold similar
// numbers of records and inactive rows cost nothing.  Records are grouped by
// work item, ascending element within an item: every CSR value is folded in
// ascending element order, the reference's order (routing.cpp:117-124).
//
// Inputs are the scalar routing arrays, bit-identical to build_routing
// (routing.cpp:12-85): row_ptr, the node incidence CSR vec_offsets/vec_slots
// (ascending slot e*k+a per node, routing.cpp:47-62) and slot_of.
#include <algorithm>
#include <thread>

#include "tgk_internal.hpp"

namespace tgk {

std::vector<uint32_t> morton_order(int kind, int64_t N, const double* nodes, int64_t row_lo, int64_t row_hi);

int build_plan5(int kind, int64_t N, const double* nodes, const int32_t* conn, const int64_t* row_ptr,
                const uint32_t* vec_offsets, const uint32_t* vec_slots, const uint32_t* slot_of,
                int64_t row_lo, int64_t row_hi, int R, Plan5Host& P) {
    const int k = element_nodes(kind);
    if (R != 64 && R != 128 && R != 256) return set_error(TGK_ERR_INPUT, "fused plan: R must be 64, 128 or 256");
    P = Plan5Host{};
    P.R = R;
    const std::vector<uint32_t> order = morton_order(kind, N, nodes, row_lo, row_hi);
    const int64_t n_owned = static_cast<int64_t>(order.size());
    int lmax = 0;
    for (int64_t i = 0; i < N; ++i) lmax = std::max<int>(lmax, static_cast<int>(row_ptr[i + 1] - row_ptr[i]));
    if (lmax > kMaxRowLen)
        return set_error(TGK_ERR_INPUT, "fused plan: CSR row longer than " + std::to_string(kMaxRowLen) + " entries");
    P.lmax = lmax;
    const int64_t nb = (n_owned + R - 1) / R;
    P.n_blocks = nb;
    P.row_off.resize(nb + 1);
    P.rows.resize(n_owned);
    for (int64_t b = 0; b <= nb; ++b) P.row_off[b] = std::min<int64_t>(b * R, n_owned);
    for (int64_t b = 0; b < nb; ++b) {
        std::copy(order.begin() + P.row_off[b], order.begin() + P.row_off[b + 1], P.rows.begin() + P.row_off[b]);
        std::sort(P.rows.begin() + P.row_off[b], P.rows.begin() + P.row_off[b + 1]);
    }
    P.rows_rp.resize(n_owned + 1);
    for (int64_t i = 0; i < n_owned; ++i)  // CSR offset | row length << 56
        P.rows_rp[i] = row_ptr[P.rows[i]] | ((row_ptr[P.rows[i] + 1] - row_ptr[P.rows[i]]) << 56);
    P.rows_rp[n_owned] = 0;

    struct BlockOut {
        std::vector<uint32_t> halo, bnodes, items, recs;
        std::vector<uint16_t> lconn;
        std::vector<int64_t> chunk_nrec, chunk_nitem;  // padded counts per chunk
        int err = 0;
        std::string msg;
    };
    std::vector<BlockOut> out(nb);
    auto work = [&](int64_t b_begin, int64_t b_end) {
        std::vector<uint32_t> tmp;
        std::vector<std::pair<uint32_t, uint32_t>> edges;
        for (int64_t b = b_begin; b < b_end; ++b) {
            BlockOut& o = out[b];
            const int64_t rs = P.row_off[b], re = P.row_off[b + 1];
            const int nr = static_cast<int>(re - rs);
            const uint32_t* rows = P.rows.data() + rs;
            // halo + levels (longest chain ending at each element)
            tmp.clear();
            for (int i = 0; i < nr; ++i)
                for (uint32_t s = vec_offsets[rows[i]]; s < vec_offsets[rows[i] + 1]; ++s) tmp.push_back(vec_slots[s] / k);
            std::sort(tmp.begin(), tmp.end());
            tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
            const int64_t nh = static_cast<int64_t>(tmp.size());
            std::vector<int> level(nh, 0);
            edges.clear();
            for (int i = 0; i < nr; ++i) {
                int64_t prev = -1;
                for (uint32_t s = vec_offsets[rows[i]]; s < vec_offsets[rows[i] + 1]; ++s) {
                    const int64_t hix = std::lower_bound(tmp.begin(), tmp.end(), vec_slots[s] / k) - tmp.begin();
                    if (prev >= 0) edges.push_back({static_cast<uint32_t>(hix), static_cast<uint32_t>(prev)});
                    prev = hix;
                }
            }
            std::sort(edges.begin(), edges.end());
            for (const auto& ed : edges) level[ed.first] = std::max(level[ed.first], level[ed.second] + 1);
            std::vector<std::pair<int, uint32_t>> ord(nh);
            for (int64_t h = 0; h < nh; ++h) ord[h] = {level[h], tmp[h]};
            std::sort(ord.begin(), ord.end());
            o.halo.resize(nh);
            std::vector<std::pair<uint32_t, uint32_t>> where(nh);  // (element, halo position)
            for (int64_t h = 0; h < nh; ++h) {
                o.halo[h] = ord[h].second;
                where[h] = {ord[h].second, static_cast<uint32_t>(h)};
            }
            std::sort(where.begin(), where.end());
            // node table and block-local connectivity
            for (int64_t h = 0; h < nh; ++h)
                for (int a = 0; a < k; ++a) o.bnodes.push_back(static_cast<uint32_t>(conn[int64_t(o.halo[h]) * k + a]));
            std::sort(o.bnodes.begin(), o.bnodes.end());
            o.bnodes.erase(std::unique(o.bnodes.begin(), o.bnodes.end()), o.bnodes.end());
            if (o.bnodes.size() > 65535) {
                o.err = 1;
                o.msg = "fused plan: block node table exceeds 65535 nodes";
                return;
            }
            o.lconn.assign(nh * 4, 0);
            for (int64_t h = 0; h < nh; ++h)
                for (int a = 0; a < k; ++a) {
                    const uint32_t g = static_cast<uint32_t>(conn[int64_t(o.halo[h]) * k + a]);
                    o.lconn[h * 4 + a] = static_cast<uint16_t>(std::lower_bound(o.bnodes.begin(), o.bnodes.end(), g) - o.bnodes.begin());
                }
            // records per (chunk, row), ascending element within a row
            const int64_t nch = (nh + R - 1) / R;
            std::vector<std::vector<std::vector<uint32_t>>> per(nch, std::vector<std::vector<uint32_t>>(nr));
            for (int i = 0; i < nr; ++i) {
                const uint32_t row = rows[i];
                const int64_t rp = row_ptr[row];
                for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s) {
                    const uint32_t slot = vec_slots[s];
                    const uint32_t e = slot / k;
                    const int a = static_cast<int>(slot % k);
                    const int64_t hpos = std::lower_bound(where.begin(), where.end(), std::make_pair(e, 0u))->second;
                    int pos[4] = {0, 0, 0, 0};
                    for (int bb = 0; bb < k; ++bb) pos[bb] = static_cast<int>(slot_of[int64_t(slot) * k + bb] - rp);
                    per[hpos / R][i].push_back(pack_rec(static_cast<int>(hpos % R), a, pos, k));
                }
            }
            for (int64_t ch = 0; ch < nch; ++ch) {
                std::vector<int> act;
                for (int i = 0; i < nr; ++i)
                    if (!per[ch][i].empty()) act.push_back(i);
                std::stable_sort(act.begin(), act.end(),
                                 [&](int x, int y) { return per[ch][x].size() > per[ch][y].size(); });
                std::vector<uint32_t> recs, items;
                for (int i : act) {
                    const auto& v = per[ch][i];
                    if (recs.size() > 65535 || v.size() > 255) {
                        o.err = 1;
                        o.msg = "fused plan: chunk record segment too large";
                        return;
                    }
                    items.push_back(static_cast<uint32_t>(i) | (static_cast<uint32_t>(v.size()) << 8) |
                                    (static_cast<uint32_t>(recs.size()) << 16));
                    recs.insert(recs.end(), v.begin(), v.end());
                }
                const int64_t nit = static_cast<int64_t>(items.size());
                while (items.size() % 4) items.push_back(0);
                while (recs.size() % 4) recs.push_back(0);
                o.chunk_nitem.push_back(nit);
                o.chunk_nrec.push_back(static_cast<int64_t>(recs.size()));
                o.items.insert(o.items.end(), items.begin(), items.end());
                o.recs.insert(o.recs.end(), recs.begin(), recs.end());
            }
        }
    };
    const int nthreads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    {
        std::vector<std::thread> pool;
        const int64_t per = (nb + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            const int64_t b0 = t * per, b1 = std::min(nb, b0 + per);
            if (b0 < b1) pool.emplace_back(work, b0, b1);
        }
        for (auto& th : pool) th.join();
    }
    for (int64_t b = 0; b < nb; ++b)
        if (out[b].err) return set_error(TGK_ERR_INPUT, out[b].msg);
    // concatenate
    P.halo_off.assign(nb + 1, 0);
    P.bnode_off.assign(nb + 1, 0);
    P.chunk_off.assign(nb + 1, 0);
    for (int64_t b = 0; b < nb; ++b) {
        P.halo_off[b + 1] = P.halo_off[b] + static_cast<int64_t>(out[b].halo.size());
        P.bnode_off[b + 1] = P.bnode_off[b] + static_cast<int64_t>(out[b].bnodes.size());
        P.chunk_off[b + 1] = P.chunk_off[b] + static_cast<int64_t>(out[b].chunk_nrec.size());
        P.max_bnodes = std::max<int>(P.max_bnodes, static_cast<int>(out[b].bnodes.size()));
        P.max_block_chunks = std::max<int>(P.max_block_chunks, static_cast<int>(out[b].chunk_nrec.size()));
    }
    const int64_t nchunks = P.chunk_off[nb];
    P.halo.resize(P.halo_off[nb]);
    P.halo_lconn.resize(P.halo_off[nb] * 4);
    P.bnodes.resize(P.bnode_off[nb]);
    P.chunk_rec.assign(nchunks + 1, 0);
    P.chunk_item.assign(nchunks + 1, 0);
    P.chunk_nitems.assign(nchunks, 0);
    int64_t nrec = 0, nitem = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const BlockOut& o = out[b];
        std::copy(o.halo.begin(), o.halo.end(), P.halo.begin() + P.halo_off[b]);
        std::copy(o.lconn.begin(), o.lconn.end(), P.halo_lconn.begin() + P.halo_off[b] * 4);
        std::copy(o.bnodes.begin(), o.bnodes.end(), P.bnodes.begin() + P.bnode_off[b]);
        int64_t io = 0;
        for (size_t c = 0; c < o.chunk_nrec.size(); ++c) {
            const int64_t gc = P.chunk_off[b] + static_cast<int64_t>(c);
            P.chunk_rec[gc] = nrec;
            P.chunk_item[gc] = nitem;
            P.chunk_nitems[gc] = static_cast<uint32_t>(o.chunk_nitem[c]);
            const int64_t nit_pad = (o.chunk_nitem[c] + 3) / 4 * 4;
            P.max_chunk_recs = std::max<int>(P.max_chunk_recs, static_cast<int>(o.chunk_nrec[c]));
            P.max_chunk_items = std::max<int>(P.max_chunk_items, static_cast<int>(nit_pad));
            nrec += o.chunk_nrec[c];
            nitem += nit_pad;
            io += nit_pad;
        }
        (void)io;
    }
    P.chunk_rec[nchunks] = nrec;
    P.chunk_item[nchunks] = nitem;
    P.recs.resize(nrec);
    P.items.resize(nitem);
    for (int64_t b = 0; b < nb; ++b) {
        if (!out[b].recs.empty())
            std::copy(out[b].recs.begin(), out[b].recs.end(), P.recs.begin() + P.chunk_rec[P.chunk_off[b]]);
        if (!out[b].items.empty())
            std::copy(out[b].items.begin(), out[b].items.end(), P.items.begin() + P.chunk_item[P.chunk_off[b]]);
    }
    return TGK_OK;
}

}  // namespace tgk
