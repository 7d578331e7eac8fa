// Host construction of the ENTRY plan of the batched kernel (batched.cu,
// k_batched_entries): blocks of R owned rows (Morton-compact mesh nodes, as
// plan.cpp), each block's whole halo (elements incident to its rows, ascending
// id) and block node table, and for every owned CSR entry (row i, column j)
// its contribution list — the halo elements containing both nodes, ascending
// element id, each with the index of the gradient dot product G_a.G_b that
// forms its K_e[a][b] — so one thread can fold the entry in a register in the
// reference's order (routing.cpp:117-124).  Same for each owned row's load
// F_i (contributions (element, a)).
//
// Inputs are the scalar routing arrays, bit-identical to build_routing
// (routing.cpp:12-85): row_ptr, the node incidence CSR vec_offsets/vec_slots
// (ascending slot e*k+a per node) and slot_of.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

#include "tgk_internal.hpp"

namespace tgk {

std::vector<uint32_t> morton_order(int kind, int64_t N, const double* nodes, int64_t row_lo, int64_t row_hi);

namespace {
constexpr int sym_pair(int k, int a, int b) {  // index of (min, max) in the packed upper triangle
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo * k - lo * (lo - 1) / 2 + (hi - lo);
}
}  // namespace

int build_entry_plan(int kind, int64_t N, const double* nodes, const int32_t* conn, const int64_t* row_ptr,
                     const uint32_t* vec_offsets, const uint32_t* vec_slots, const uint32_t* slot_of,
                     int64_t row_lo, int64_t row_hi, int R, EntryPlanHost& P) {
    const int k = element_nodes(kind);
    P = EntryPlanHost{};
    P.R = R;
    if (R < 1 || R > 1024) return set_error(TGK_ERR_INPUT, "entry plan: rows per block out of range");
    // order of a block's entries over the threads: 0 (default) row-major, 1 by
    // contribution count (longest first), 2 diagonal entries first, then the
    // off-diagonal ones row-major.  Row-major measured fastest on C4 (its
    // contiguous stores outweigh the idle lanes of mixed-length warps).
    const char* es = getenv("TGK_ENTRY_SORT");
    const int entry_order = es ? atoi(es) : 0;
    // TGK_ENTRY_SYM=1: an off-diagonal entry (i, j) with both rows in the
    // block is folded once and stored to (i, j) and (j, i) — both folds run
    // over the same elements in the same order with K_e[a][b] == K_e[b][a]
    // bitwise.  A third fewer loads but scattered mirror stores: slower on C4.
    const char* sy = getenv("TGK_ENTRY_SYM");
    const bool symmetric = sy && atoi(sy) != 0;
    const std::vector<uint32_t> order = morton_order(kind, N, nodes, row_lo, row_hi);
    const int64_t n_owned = static_cast<int64_t>(order.size());
    const int64_t nb = (n_owned + R - 1) / R;
    P.n_blocks = nb;
    struct BlockOut {
        std::vector<uint32_t> rows, halo, bnodes, contrib, fcontrib, coff, fcoff;  // coff/fcoff: n+1
        std::vector<uint64_t> hconn;
        std::vector<int64_t> epos, epos2;
        int max_clen = 0;
        int err = 0;
        std::string msg;
    };
    std::vector<BlockOut> out(nb);
    auto work = [&](int64_t b0, int64_t b1) {
        for (int64_t b = b0; b < b1; ++b) {
            BlockOut& o = out[b];
            const int64_t rs = b * R, re = std::min<int64_t>(n_owned, rs + R);
            o.rows.assign(order.begin() + rs, order.begin() + re);
            std::sort(o.rows.begin(), o.rows.end());
            for (uint32_t row : o.rows)
                for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s) o.halo.push_back(vec_slots[s] / k);
            std::sort(o.halo.begin(), o.halo.end());
            o.halo.erase(std::unique(o.halo.begin(), o.halo.end()), o.halo.end());
            for (uint32_t e : o.halo)
                for (int a = 0; a < k; ++a) o.bnodes.push_back(static_cast<uint32_t>(conn[int64_t(e) * k + a]));
            std::sort(o.bnodes.begin(), o.bnodes.end());
            o.bnodes.erase(std::unique(o.bnodes.begin(), o.bnodes.end()), o.bnodes.end());
            if (o.halo.size() > 65535 || o.bnodes.size() > 65535) {
                o.err = 1;
                o.msg = "entry plan: block halo or node table exceeds 65535";
                return;
            }
            for (uint32_t e : o.halo) {
                uint64_t hc = 0;
                for (int a = 0; a < k; ++a) {
                    const uint32_t g = static_cast<uint32_t>(conn[int64_t(e) * k + a]);
                    hc |= uint64_t(std::lower_bound(o.bnodes.begin(), o.bnodes.end(), g) - o.bnodes.begin()) << (16 * a);
                }
                o.hconn.push_back(hc);
            }
            // per owned row: its entries' contribution lists and its load contributions
            std::vector<std::vector<uint32_t>> lists;
            std::vector<int64_t> lpos, lpos2;
            std::vector<char> ldiag;
            o.fcoff.push_back(0);
            auto owned = [&o](uint32_t j) { return std::binary_search(o.rows.begin(), o.rows.end(), j); };
            for (uint32_t row : o.rows) {
                const int64_t rp = row_ptr[row];
                const int len = static_cast<int>(row_ptr[row + 1] - rp);
                std::vector<std::vector<uint32_t>> ent(len);
                std::vector<int64_t> mirror(len, -1);  // CSR position of (j, row) when folded here too
                std::vector<char> skip(len, 0), col_is_row(len, 0);
                for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s) {  // ascending element
                    const uint32_t slot = vec_slots[s];
                    const uint32_t e = slot / k;
                    const int a = static_cast<int>(slot % k);
                    const uint32_t h = static_cast<uint32_t>(std::lower_bound(o.halo.begin(), o.halo.end(), e) - o.halo.begin());
                    for (int bb = 0; bb < k; ++bb) {
                        const int64_t p = int64_t(slot_of[int64_t(slot) * k + bb]) - rp;
                        ent[p].push_back(h | (uint32_t(sym_pair(k, a, bb)) << 16));
                        const uint32_t j = static_cast<uint32_t>(conn[int64_t(e) * k + bb]);
                        col_is_row[p] = j == row;
                        if (symmetric && j != row && owned(j)) {
                            if (j < row) skip[p] = 1;  // folded by row j's entry (j, row)
                            else mirror[p] = slot_of[(int64_t(e) * k + bb) * k + a];
                        }
                    }
                    o.fcontrib.push_back(h | (uint32_t(a) << 16));
                }
                o.fcoff.push_back(static_cast<uint32_t>(o.fcontrib.size()));
                for (int p = 0; p < len; ++p) {
                    if (skip[p]) continue;
                    lists.push_back(std::move(ent[p]));
                    lpos.push_back(rp + p);
                    lpos2.push_back(mirror[p]);
                    ldiag.push_back(col_is_row[p]);
                }
            }
            std::vector<uint32_t> perm(lists.size());
            std::iota(perm.begin(), perm.end(), 0u);
            if (entry_order == 1)
                std::stable_sort(perm.begin(), perm.end(),
                                 [&](uint32_t x, uint32_t y) { return lists[x].size() > lists[y].size(); });
            else if (entry_order == 2)
                std::stable_partition(perm.begin(), perm.end(), [&](uint32_t x) { return ldiag[x] != 0; });
            o.coff.push_back(0);
            for (const auto& l : lists) o.max_clen = std::max<int>(o.max_clen, static_cast<int>(l.size()));
            for (uint32_t x : perm) {
                o.contrib.insert(o.contrib.end(), lists[x].begin(), lists[x].end());
                o.coff.push_back(static_cast<uint32_t>(o.contrib.size()));
                o.epos.push_back(lpos[x]);
                o.epos2.push_back(lpos2[x]);
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
    for (const auto& o : out)
        if (o.err) return set_error(TGK_ERR_INPUT, o.msg);
    auto cat = [&](auto member, auto& off, auto& dst) {
        off.assign(nb + 1, 0);
        for (int64_t b = 0; b < nb; ++b) off[b + 1] = off[b] + static_cast<int64_t>((out[b].*member).size());
        dst.resize(off[nb]);
        for (int64_t b = 0; b < nb; ++b) {
            const auto& v = out[b].*member;
            std::copy(v.begin(), v.end(), dst.begin() + off[b]);
        }
    };
    cat(&BlockOut::rows, P.row_off, P.rows);
    cat(&BlockOut::halo, P.halo_off, P.halo);
    std::vector<int64_t> dummy;
    cat(&BlockOut::hconn, dummy, P.hconn);
    cat(&BlockOut::bnodes, P.bnode_off, P.bnodes);
    cat(&BlockOut::epos, P.ent_off, P.epos);
    cat(&BlockOut::epos2, dummy, P.epos2);
    cat(&BlockOut::contrib, P.contrib_off, P.contrib);
    cat(&BlockOut::fcontrib, P.fcontrib_off, P.fcontrib);
    // per-entry / per-row offsets are block-relative (u32), n+1 per block
    P.coff.clear();
    P.fcoff.clear();
    for (int64_t b = 0; b < nb; ++b) {
        P.coff.insert(P.coff.end(), out[b].coff.begin(), out[b].coff.end());
        P.fcoff.insert(P.fcoff.end(), out[b].fcoff.begin(), out[b].fcoff.end());
        P.max_halo = std::max<int>(P.max_halo, static_cast<int>(out[b].halo.size()));
        P.max_bnodes = std::max<int>(P.max_bnodes, static_cast<int>(out[b].bnodes.size()));
        P.max_contrib = std::max<int>(P.max_contrib, static_cast<int>(out[b].contrib.size()));
        P.max_fcontrib = std::max<int>(P.max_fcontrib, static_cast<int>(out[b].fcontrib.size()));
        P.max_entries = std::max<int>(P.max_entries, static_cast<int>(out[b].epos.size()));
        P.max_clen = std::max(P.max_clen, out[b].max_clen);
    }
    // the kernel keeps the per-element values structure-of-arrays, [index][halo
    // element] with a row stride of max_halo (rounded to even): pre-resolve
    // (h, index) to the shared-memory offset
    P.max_halo = (P.max_halo + 1) & ~1;
    for (auto* v : {&P.contrib, &P.fcontrib})
        for (uint32_t& u : *v) u = (u >> 16) * uint32_t(P.max_halo) + (u & 0xffffu);
    return TGK_OK;
}

int build_group_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn, int G,
                     GroupPlanHost& P) {
    const int k = element_nodes(kind), d = element_dim(kind);
    P = GroupPlanHost{};
    P.G = G;
    if (G < 32 || G > 1024) return set_error(TGK_ERR_INPUT, "group plan: group size out of range");
    std::vector<double> cen(size_t(E) * d, 0.0);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a)
            for (int c = 0; c < d; ++c) cen[e * d + c] += nodes[int64_t(conn[e * k + a]) * d + c];
    const std::vector<uint32_t> order = morton_order(kind, E, cen.data(), 0, E);
    const int64_t ng = (E + G - 1) / G;
    P.n_groups = ng;
    P.grp_off.resize(ng + 1);
    P.node_off.assign(ng + 1, 0);
    P.elems.resize(E);
    P.lconn.resize(E);
    std::vector<std::vector<uint32_t>> gn(ng);
    auto work = [&](int64_t g0, int64_t g1) {
        for (int64_t g = g0; g < g1; ++g) {
            const int64_t lo = g * G, hi = std::min<int64_t>(E, lo + G);
            std::vector<uint32_t> el(order.begin() + lo, order.begin() + hi);
            std::sort(el.begin(), el.end());  // ascending ids: the output stores of a warp share sectors more often
            std::vector<uint32_t>& nd = gn[g];
            for (uint32_t e : el)
                for (int a = 0; a < k; ++a) nd.push_back(static_cast<uint32_t>(conn[int64_t(e) * k + a]));
            std::sort(nd.begin(), nd.end());
            nd.erase(std::unique(nd.begin(), nd.end()), nd.end());
            for (int64_t i = lo; i < hi; ++i) {
                const uint32_t e = el[i - lo];
                P.elems[i] = e;
                uint64_t lc = 0;
                for (int a = 0; a < k; ++a) {
                    const uint32_t n = static_cast<uint32_t>(conn[int64_t(e) * k + a]);
                    lc |= uint64_t(std::lower_bound(nd.begin(), nd.end(), n) - nd.begin()) << (16 * a);
                }
                P.lconn[i] = lc;
            }
        }
    };
    const int nthreads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    {
        std::vector<std::thread> pool;
        const int64_t per = (ng + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            const int64_t g0 = t * per, g1 = std::min(ng, g0 + per);
            if (g0 < g1) pool.emplace_back(work, g0, g1);
        }
        for (auto& th : pool) th.join();
    }
    for (int64_t g = 0; g <= ng; ++g) P.grp_off[g] = std::min<int64_t>(E, g * G);
    for (int64_t g = 0; g < ng; ++g) {
        P.node_off[g + 1] = P.node_off[g] + static_cast<int64_t>(gn[g].size());
        P.max_nodes = std::max<int>(P.max_nodes, static_cast<int>(gn[g].size()));
    }
    P.gnodes.reserve(P.node_off[ng]);
    for (const auto& v : gn) P.gnodes.insert(P.gnodes.end(), v.begin(), v.end());
    return TGK_OK;
}


}  // namespace tgk

