// Host construction of the v4 fused-assembly plan ("row blocks with update
// rounds", see tgk_internal.hpp Plan4Host and fused4.cu).
//
// Inputs are the scalar routing arrays, bit-identical to the reference's
// build_routing (routing.cpp:12-85): row_ptr (CsrPattern::offsets), the node
// incidence CSR vec_offsets/vec_slots (ascending slot e*k+a per node,
// routing.cpp:47-62) and the element-to-slot map slot_of.
//
// Per block of R owned rows (Morton-compact, ascending ids):
//  1. halo  = every element incident to an owned row, ordered by (level, id)
//     where level(e) = longest chain ending at e in the per-row ascending
//     element chains.  Every row meets its elements in ascending id order.
//  2. node table = owned rows first (block-local ids 0..nr-1 == local row),
//     then the halo's other nodes ascending; hconn = the 4 block-local node
//     ids of each halo element.
//  3. chunks of T consecutive halo elements (one per thread); within a chunk
//     the r-th element (in halo order) touching an owned row updates it in
//     update round r, so each CSR value is folded in ascending element order
//     — the reference reduction's order (routing.cpp:117-124).
//  4. one 32-bit record per (halo element, owned local node a): the CSR
//     positions (within row a) of the element's k nodes and the round.
#include <algorithm>
#include <numeric>
#include <thread>

#include "tgk_internal.hpp"

namespace tgk {

std::vector<uint32_t> morton_order(int kind, int64_t N, const double* nodes, int64_t row_lo, int64_t row_hi);

int build_plan4(int kind, int64_t N, const double* nodes, const int32_t* conn, const int64_t* row_ptr,
                const uint32_t* vec_offsets, const uint32_t* vec_slots, const uint32_t* slot_of,
                int64_t row_lo, int64_t row_hi, int R, int T, Plan4Host& P) {
    const int k = element_nodes(kind);
    if (R < 32 || R > 1024 || T < 32 || T > 256 || T % 32)
        return set_error(TGK_ERR_INPUT, "fused plan: unsupported block shape");
    P = Plan4Host{};
    P.R = R;
    P.T = T;
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

    const int W = T / 32;
    struct BlockOut {
        std::vector<uint32_t> halo, bnodes, recs;
        std::vector<uint64_t> hconn;
        std::vector<int64_t> chunk_nrec;   // padded record count per chunk
        std::vector<uint32_t> chunk_meta;  // rounds per chunk
        std::vector<uint16_t> wbase;       // W per chunk, padded to 8
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
            auto local_row = [&](uint32_t g) -> int {  // owned local row of global node g, or -1
                const uint32_t* p = std::lower_bound(rows, rows + nr, g);
                return (p != rows + nr && *p == g) ? static_cast<int>(p - rows) : -1;
            };
            // 1. halo + levels
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
            std::sort(edges.begin(), edges.end());  // targets ascending == ids ascending: topological
            for (const auto& ed : edges) level[ed.first] = std::max(level[ed.first], level[ed.second] + 1);
            std::vector<std::pair<int, uint32_t>> ord(nh);
            for (int64_t h = 0; h < nh; ++h) ord[h] = {level[h], tmp[h]};
            std::sort(ord.begin(), ord.end());
            o.halo.resize(nh);
            for (int64_t h = 0; h < nh; ++h) o.halo[h] = ord[h].second;
            // 2. node table: owned rows, then the other halo nodes ascending
            std::vector<uint32_t> others;
            for (int64_t h = 0; h < nh; ++h)
                for (int a = 0; a < k; ++a) {
                    const uint32_t g = static_cast<uint32_t>(conn[static_cast<int64_t>(o.halo[h]) * k + a]);
                    if (local_row(g) < 0) others.push_back(g);
                }
            std::sort(others.begin(), others.end());
            others.erase(std::unique(others.begin(), others.end()), others.end());
            o.bnodes.assign(rows, rows + nr);
            o.bnodes.insert(o.bnodes.end(), others.begin(), others.end());
            if (o.bnodes.size() > 65535) {
                o.err = 1;
                o.msg = "fused plan: block node table exceeds 65535 nodes";
                return;
            }
            o.hconn.resize(nh);
            // 3./4. chunks, rounds, records
            std::vector<uint8_t> cnt(nr, 0);
            std::vector<int> touched;
            int64_t h = 0;
            while (h < nh) {
                const int64_t c0 = h;
                int rounds = 0;
                std::vector<uint32_t> crec;
                std::vector<uint16_t> wb(8, 0);
                touched.clear();
                for (; h < nh && h - c0 < T; ++h) {
                    const int64_t e = o.halo[h];
                    const int lane = static_cast<int>(h - c0);
                    if (lane % 32 == 0) wb[lane / 32] = static_cast<uint16_t>(crec.size());
                    uint64_t hc = 0;
                    for (int a = 0; a < k; ++a) {
                        const uint32_t g = static_cast<uint32_t>(conn[e * k + a]);
                        const int lr = local_row(g);
                        const uint32_t ln = lr >= 0 ? static_cast<uint32_t>(lr)
                                                    : static_cast<uint32_t>(nr + (std::lower_bound(others.begin(), others.end(), g) - others.begin()));
                        hc |= static_cast<uint64_t>(ln) << (16 * a);
                        if (lr < 0) continue;
                        const int rd = cnt[lr];
                        if (rd >= 31) {
                            o.err = 1;
                            o.msg = "fused plan: more than 31 update rounds in a chunk";
                            return;
                        }
                        if (cnt[lr]++ == 0) touched.push_back(lr);
                        rounds = std::max(rounds, rd + 1);
                        const int64_t rp = row_ptr[g];
                        uint32_t rec = static_cast<uint32_t>(rd) << 24;
                        for (int bb = 0; bb < k; ++bb)
                            rec |= static_cast<uint32_t>(slot_of[(e * k + a) * k + bb] - rp) << (5 * bb);
                        crec.push_back(rec);
                    }
                    o.hconn[h] = hc;
                }
                for (int lr : touched) cnt[lr] = 0;
                while (crec.size() % 4) crec.push_back(0);
                o.chunk_nrec.push_back(static_cast<int64_t>(crec.size()));
                o.chunk_meta.push_back(static_cast<uint32_t>(rounds));
                o.wbase.insert(o.wbase.end(), wb.begin(), wb.end());
                o.recs.insert(o.recs.end(), crec.begin(), crec.end());
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
    (void)W;
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
        if (P.chunk_off[b + 1] - P.chunk_off[b] > kMaxChunks4)
            return set_error(TGK_ERR_INPUT, "fused plan: a row block needs more than " + std::to_string(kMaxChunks4) + " chunks");
        P.max_bnodes = std::max<int>(P.max_bnodes, static_cast<int>(out[b].bnodes.size()));
    }
    const int64_t nchunks = P.chunk_off[nb];
    P.halo.resize(P.halo_off[nb]);
    P.hconn.resize(P.halo_off[nb]);
    P.bnodes.resize(P.bnode_off[nb]);
    P.chunk_rec.assign(nchunks + 1, 0);
    P.chunk_meta.resize(nchunks);
    P.chunk_wbase.resize(nchunks * 8);
    int64_t nrec = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const BlockOut& o = out[b];
        std::copy(o.halo.begin(), o.halo.end(), P.halo.begin() + P.halo_off[b]);
        std::copy(o.hconn.begin(), o.hconn.end(), P.hconn.begin() + P.halo_off[b]);
        std::copy(o.bnodes.begin(), o.bnodes.end(), P.bnodes.begin() + P.bnode_off[b]);
        std::copy(o.wbase.begin(), o.wbase.end(), P.chunk_wbase.begin() + P.chunk_off[b] * 8);
        for (size_t c = 0; c < o.chunk_nrec.size(); ++c) {
            const int64_t gc = P.chunk_off[b] + static_cast<int64_t>(c);
            P.chunk_rec[gc] = nrec;
            P.chunk_meta[gc] = o.chunk_meta[c];
            P.max_rounds = std::max<int>(P.max_rounds, static_cast<int>(o.chunk_meta[c]));
            P.max_chunk_recs = std::max<int>(P.max_chunk_recs, static_cast<int>(o.chunk_nrec[c]));
            nrec += o.chunk_nrec[c];
        }
    }
    P.chunk_rec[nchunks] = nrec;
    P.recs.resize(nrec);
    for (int64_t b = 0; b < nb; ++b)
        if (!out[b].recs.empty())
            std::copy(out[b].recs.begin(), out[b].recs.end(), P.recs.begin() + P.chunk_rec[P.chunk_off[b]]);
    return TGK_OK;
}

}  // namespace tgk
