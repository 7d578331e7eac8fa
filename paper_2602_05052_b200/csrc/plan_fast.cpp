// Host construction of the fast-mode plan (TGK_MODE_FAST, fast.cu).
//
// The plan is the north star's "precomputed element-to-CSR-slot permutation":
// for every CSR entry a CUDA block owns, the list of (halo element, local
// pair) whose local value lands on it — exactly the segments of the
// reference's mat_offsets/mat_slots (routing.cpp:64-84), re-expressed against
// the block's shared-memory element values.  Layout:
//
//  - owned rows in Morton order of their coordinates, cut into blocks of R
//    rows (compact in space => small halos);
//  - per block its halo (every element incident to an owned row, ascending
//    id), the halo's block-local connectivity (4 x u16) and its node table;
//  - per block its entries: one per owned row ("diagonal": the diagonal value
//    and the row's load) and one per off-diagonal CSR entry; an entry (i, j)
//    whose column j is an owned row of the same block is folded once and
//    stored to (i, j) and (j, i) (K, M symmetric: both folds would run over
//    the same elements with K_e[a][b] == K_e[b][a]).  Entries are sorted by
//    list length (warps of uniform work), each class padded to whole warps;
//  - per warp of 32 entries the items, u16 = halo index | value index << 12,
//    interleaved [step][lane][4] so every step is one coalesced 8-byte load
//    per lane.  Short lists are padded with the block's zero slot.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <thread>

#include "tgk_internal.hpp"

namespace tgk {

namespace {

constexpr int kSymTet[4][4] = {{0, 1, 2, 3}, {1, 4, 5, 6}, {2, 5, 7, 8}, {3, 6, 8, 9}};
constexpr int kSymTri[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};

inline int sym_pair_k(int k, int a, int b) { return k == 4 ? kSymTet[a][b] : kSymTri[a][b]; }

}  // namespace

int build_fast_plan(int kind, int64_t N, int64_t E, const double* nodes, const int32_t* conn,
                    const int64_t* row_ptr, const uint32_t* vec_offsets, const uint32_t* vec_slots,
                    const uint32_t* slot_of, int64_t row_lo, int64_t row_hi, int64_t elem_lo, int64_t elem_hi,
                    int R, FastPlanHost& P) {
    const int k = element_nodes(kind);
    (void)E;
    P = FastPlanHost{};
    P.R = R;
    if (R < 1 || R > kFastMaxRows) return set_error(TGK_ERR_INPUT, "fast plan: rows per block out of range");
    auto in_range = [elem_lo, elem_hi](uint32_t e) { return int64_t(e) >= elem_lo && int64_t(e) < elem_hi; };
    for (int64_t i = row_lo; i < row_hi; ++i)
        if (row_ptr[i + 1] - row_ptr[i] > kFastMaxRowLen) return TGK_ERR_INPUT;  // not applicable (no message)
    const std::vector<uint32_t> order = morton_order(kind, N, nodes, row_lo, row_hi);
    const int64_t n_owned = static_cast<int64_t>(order.size());
    const int64_t nb = (n_owned + R - 1) / R;
    P.n_blocks = nb;
    struct BlockOut {
        std::vector<uint32_t> rows, helem, bnodes, desc;
        std::vector<uint64_t> hconn;
        std::vector<uint16_t> items;
        std::vector<int64_t> wg_items;  // items per warp group (u16 units)
        bool fail = false;
    };
    std::vector<BlockOut> out(nb);
    auto work = [&](int64_t b0, int64_t b1) {
        std::vector<std::vector<uint16_t>> lists;
        for (int64_t b = b0; b < b1; ++b) {
            BlockOut& o = out[b];
            const int64_t rs = b * R, re = std::min<int64_t>(n_owned, rs + R);
            o.rows.assign(order.begin() + rs, order.begin() + re);
            std::sort(o.rows.begin(), o.rows.end());
            for (uint32_t row : o.rows)
                for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s)
                    if (in_range(vec_slots[s] / k)) o.helem.push_back(vec_slots[s] / k);
            std::sort(o.helem.begin(), o.helem.end());
            o.helem.erase(std::unique(o.helem.begin(), o.helem.end()), o.helem.end());
            for (uint32_t e : o.helem)
                for (int a = 0; a < k; ++a) o.bnodes.push_back(static_cast<uint32_t>(conn[int64_t(e) * k + a]));
            std::sort(o.bnodes.begin(), o.bnodes.end());
            o.bnodes.erase(std::unique(o.bnodes.begin(), o.bnodes.end()), o.bnodes.end());
            if (o.helem.size() > size_t(kFastMaxHalo) || o.bnodes.size() > 65535) {
                o.fail = true;
                return;
            }
            for (uint32_t e : o.helem) {
                uint64_t hc = 0;
                for (int a = 0; a < k; ++a) {
                    const uint32_t g = static_cast<uint32_t>(conn[int64_t(e) * k + a]);
                    hc |= uint64_t(std::lower_bound(o.bnodes.begin(), o.bnodes.end(), g) - o.bnodes.begin()) << (16 * a);
                }
                o.hconn.push_back(hc);
            }
            auto local_row = [&o](uint32_t j) -> int {
                auto it = std::lower_bound(o.rows.begin(), o.rows.end(), j);
                return it != o.rows.end() && *it == j ? static_cast<int>(it - o.rows.begin()) : -1;
            };
            auto halo_index = [&o](uint32_t e) {
                return static_cast<uint16_t>(std::lower_bound(o.helem.begin(), o.helem.end(), e) - o.helem.begin());
            };
            // entries: (class, steps, lr, p) sort key + desc + list
            struct Ent {
                int cls, steps, lr, p;
                uint32_t desc;
                int list;
            };
            std::vector<Ent> ents;
            lists.clear();
            for (int lr = 0; lr < static_cast<int>(o.rows.size()); ++lr) {
                const uint32_t row = o.rows[lr];
                const int64_t rp = row_ptr[row];
                const int len = static_cast<int>(row_ptr[row + 1] - rp);
                std::vector<int> col(len, -1);         // owned local row of the column, or -1
                std::vector<int> pos2(len, -1);        // position of `row` within that row
                std::vector<std::vector<uint16_t>> ent(len);
                std::vector<uint16_t> diag;
                int pdiag = kFastNoPos;
                for (uint32_t s = vec_offsets[row]; s < vec_offsets[row + 1]; ++s) {  // ascending element
                    const uint32_t slot = vec_slots[s];
                    const uint32_t e = slot / k;
                    const int a = static_cast<int>(slot % k);
                    const bool use = in_range(e);
                    const uint16_t h = use ? halo_index(e) : 0;
                    for (int bb = 0; bb < k; ++bb) {
                        const int p = static_cast<int>(int64_t(slot_of[int64_t(slot) * k + bb]) - rp);
                        const uint32_t j = static_cast<uint32_t>(conn[int64_t(e) * k + bb]);
                        if (bb == a) {
                            pdiag = p;
                            continue;
                        }
                        const int lj = local_row(j);
                        if (lj >= 0) {
                            col[p] = lj;
                            pos2[p] = static_cast<int>(int64_t(slot_of[(int64_t(e) * k + bb) * k + a]) - row_ptr[j]);
                        }
                        if (use) ent[p].push_back(static_cast<uint16_t>(h | (sym_pair_k(k, a, bb) << 12)));
                    }
                    if (use) diag.push_back(static_cast<uint16_t>(h | (a << 12)));
                }
                // the row's diagonal entry (also its load value)
                lists.push_back(std::move(diag));
                ents.push_back({0, 0, lr, pdiag, uint32_t(lr) | (uint32_t(pdiag) << 9) | (1u << 15),
                                static_cast<int>(lists.size()) - 1});
                for (int p = 0; p < len; ++p) {
                    if (p == pdiag) continue;
                    uint32_t d = uint32_t(lr) | (uint32_t(p) << 9);
                    if (col[p] >= 0) {
                        if (o.rows[col[p]] < row) continue;  // folded by (j, row), stored mirrored
                        d |= (uint32_t(col[p]) << 16) | (uint32_t(pos2[p]) << 25) | (1u << 31);
                    }
                    lists.push_back(std::move(ent[p]));
                    ents.push_back({1, 0, lr, p, d, static_cast<int>(lists.size()) - 1});
                }
            }
            for (auto& en : ents) en.steps = (static_cast<int>(lists[en.list].size()) + 3) / 4;
            std::stable_sort(ents.begin(), ents.end(), [](const Ent& x, const Ent& y) {
                if (x.cls != y.cls) return x.cls < y.cls;
                if (x.steps != y.steps) return x.steps > y.steps;
                if (x.lr != y.lr) return x.lr < y.lr;
                return x.p < y.p;
            });
            const uint16_t zero_item = static_cast<uint16_t>(kFastMaxHalo);  // the zero slot, value index 0
            for (int cls = 0; cls < 2; ++cls) {
                std::vector<const Ent*> c;
                for (const auto& en : ents)
                    if (en.cls == cls) c.push_back(&en);
                for (size_t w0 = 0; w0 < c.size(); w0 += 32) {
                    int steps = 0;
                    for (size_t l = w0; l < std::min(c.size(), w0 + 32); ++l) steps = std::max(steps, c[l]->steps);
                    const size_t base = o.items.size();
                    o.items.resize(base + size_t(steps) * 32 * 4, zero_item);
                    for (int lane = 0; lane < 32; ++lane) {
                        const size_t l = w0 + lane;
                        if (l >= c.size()) {
                            o.desc.push_back(kFastIdle);
                            continue;
                        }
                        o.desc.push_back(c[l]->desc);
                        const auto& li = lists[c[l]->list];
                        for (size_t t = 0; t < li.size(); ++t)
                            o.items[base + (t / 4) * 128 + lane * 4 + (t % 4)] = li[t];
                    }
                    o.wg_items.push_back(int64_t(steps) * 128);
                }
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
        if (o.fail) return TGK_ERR_INPUT;  // not applicable (no message): the exact kernel takes it
    auto cat = [&](auto member, std::vector<int64_t>* off, auto& dst) {
        if (off) off->assign(nb + 1, 0);
        size_t total = 0;
        for (int64_t b = 0; b < nb; ++b) {
            if (off) (*off)[b] = static_cast<int64_t>(total);
            total += (out[b].*member).size();
        }
        if (off) (*off)[nb] = static_cast<int64_t>(total);
        dst.resize(total);
        size_t at = 0;
        for (int64_t b = 0; b < nb; ++b) {
            const auto& v = out[b].*member;
            std::copy(v.begin(), v.end(), dst.begin() + at);
            at += v.size();
        }
    };
    cat(&BlockOut::rows, &P.row_off, P.rows);
    cat(&BlockOut::helem, &P.halo_off, P.helem);
    cat(&BlockOut::hconn, nullptr, P.hconn);
    cat(&BlockOut::bnodes, &P.bnode_off, P.bnodes);
    cat(&BlockOut::desc, &P.ent_off, P.desc);
    cat(&BlockOut::items, nullptr, P.items);
    // warp-group item offsets (u16 units), one per 32 entry slots, +1
    P.wg_item.assign(P.desc.size() / 32 + 1, 0);
    {
        size_t g = 0;
        int64_t acc = 0;
        for (int64_t b = 0; b < nb; ++b)
            for (int64_t n : out[b].wg_items) {
                P.wg_item[g++] = acc;
                acc += n;
            }
        P.wg_item[g] = acc;
    }
    for (int64_t b = 0; b < nb; ++b) {
        P.max_halo = std::max<int>(P.max_halo, static_cast<int>(out[b].helem.size()));
        P.max_bnodes = std::max<int>(P.max_bnodes, static_cast<int>(out[b].bnodes.size()));
        P.max_rows = std::max<int>(P.max_rows, static_cast<int>(out[b].rows.size()));
    }
    // padding items point at the zero slot, halo index max_halo of every value row
    for (uint16_t& it : P.items)
        if ((it & 0xfff) == kFastMaxHalo) it = static_cast<uint16_t>((it & 0xf000) | P.max_halo);
    return TGK_OK;
}

}  // namespace tgk

// ---------------------------------------------------------------------------
// Upload (one device allocation, 16-byte aligned segments), cached on the
// scalar routing per (R, owned rows, element range).
#include <cuda_runtime.h>

namespace tgk {

void FastPlanDev::release() {
    if (blob) cudaFree(blob);
    *this = FastPlanDev{};
}

int ensure_fast_plan(tgk_routing* rr, int R, const FastPlanDev** out) {
    tgk_routing* r = rr->scalar ? rr->scalar : rr;
    FastPlanDev& D = r->fast_plan;
    const int64_t lo = r->own_hi < 0 ? 0 : r->own_lo, hi = r->own_hi < 0 ? r->N : r->own_hi;
    const int64_t elo = r->elem_hi < 0 ? 0 : r->elem_lo, ehi = r->elem_hi < 0 ? r->E : r->elem_hi;
    if (D.blob && D.R == R && D.row_lo == lo && D.row_hi == hi && D.elem_lo == elo && D.elem_hi == ehi) {
        *out = &D;
        return TGK_OK;
    }
    D.release();
    const tgk_mesh* m = r->mesh;
    ScalarRoutingHost h;
    TGK_TRY(fetch_scalar_routing(r, h));
    FastPlanHost P;
    const int rc = build_fast_plan(m->kind, m->N, m->E, h.nodes.data(), h.conn.data(), h.row_ptr.data(), h.vo.data(),
                                   h.vs.data(), h.slot.data(), lo, hi, elo, ehi, R, P);
    if (rc != TGK_OK) return rc;
    // ---- per-block records (layout: tgk_internal.hpp FastPlanDev; fast.cu FastRecA/B)
    auto al16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    const int64_t nb = P.n_blocks;
    std::vector<int64_t> a_off(nb + 1, 0), b_off(nb + 1, 0);
    int max_a = 0, max_b = 0, max_tile = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const size_t nr = size_t(P.row_off[b + 1] - P.row_off[b]), nh = size_t(P.halo_off[b + 1] - P.halo_off[b]),
                     nbn = size_t(P.bnode_off[b + 1] - P.bnode_off[b]), ne = size_t(P.ent_off[b + 1] - P.ent_off[b]);
        const size_t nwg = ne / 32;
        const int64_t g0 = P.ent_off[b] / 32;
        const size_t ni = size_t(P.wg_item[g0 + nwg] - P.wg_item[g0]);
        const size_t sa = 32 + al16(8 * nr) + al16(4 * nr) + al16(2 * (nr + 1)) + al16(4 * nbn) + al16(8 * nh);
        const size_t sb = 16 + al16(4 * ne) + al16(4 * (nwg + 1)) + al16(2 * ni);
        a_off[b + 1] = a_off[b] + int64_t(sa);
        b_off[b + 1] = b_off[b] + int64_t(sb);
        max_a = std::max<int>(max_a, int(sa));
        max_b = std::max<int>(max_b, int(sb));
    }
    std::vector<unsigned char> ra(size_t(a_off[nb])), rb(size_t(b_off[nb]));
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t r0 = P.row_off[b], h0 = P.halo_off[b], n0 = P.bnode_off[b], e0 = P.ent_off[b];
        const uint32_t nr = uint32_t(P.row_off[b + 1] - r0), nh = uint32_t(P.halo_off[b + 1] - h0),
                       nbn = uint32_t(P.bnode_off[b + 1] - n0), ne = uint32_t(P.ent_off[b + 1] - e0);
        unsigned char* pa = ra.data() + a_off[b];
        std::vector<uint16_t> toff(nr + 1, 0);
        for (uint32_t i = 0; i < nr; ++i) {
            const uint32_t row = P.rows[r0 + i];
            toff[i + 1] = uint16_t(toff[i] + (h.row_ptr[row + 1] - h.row_ptr[row]));
        }
        max_tile = std::max<int>(max_tile, toff[nr]);
        const uint32_t hdr[4] = {nr, nh, nbn, toff[nr]};
        std::memcpy(pa, &h0, 8);
        std::memcpy(pa + 8, hdr, 16);
        size_t o = 32;
        for (uint32_t i = 0; i < nr; ++i) {
            const int64_t rp = h.row_ptr[P.rows[r0 + i]];
            std::memcpy(pa + o + 8 * i, &rp, 8);
        }
        o += al16(8 * size_t(nr));
        std::memcpy(pa + o, P.rows.data() + r0, 4 * size_t(nr));
        o += al16(4 * size_t(nr));
        std::memcpy(pa + o, toff.data(), 2 * size_t(nr + 1));
        o += al16(2 * size_t(nr + 1));
        std::memcpy(pa + o, P.bnodes.data() + n0, 4 * size_t(nbn));
        o += al16(4 * size_t(nbn));
        std::memcpy(pa + o, P.hconn.data() + h0, 8 * size_t(nh));
        unsigned char* pb = rb.data() + b_off[b];
        const uint32_t nwg = ne / 32;
        const int64_t g0 = e0 / 32;
        const uint32_t hb[2] = {ne, nwg};
        std::memcpy(pb, hb, 8);
        o = 16;
        std::memcpy(pb + o, P.desc.data() + e0, 4 * size_t(ne));
        o += al16(4 * size_t(ne));
        for (uint32_t w = 0; w <= nwg; ++w) {
            const uint32_t rel = uint32_t(P.wg_item[g0 + w] - P.wg_item[g0]);
            std::memcpy(pb + o + 4 * w, &rel, 4);
        }
        o += al16(4 * size_t(nwg + 1));
        std::memcpy(pb + o, P.items.data() + P.wg_item[g0], 2 * size_t(P.wg_item[g0 + nwg] - P.wg_item[g0]));
    }
    size_t total = 0;
    auto reserve = [&total](size_t bytes) {
        const size_t at = total;
        total += (bytes + 15) & ~size_t(15);
        return at;
    };
    const size_t o_ao = reserve(8 * a_off.size()), o_bo = reserve(8 * b_off.size()), o_ra = reserve(ra.size()),
                 o_rb = reserve(rb.size()), o_he = reserve(4 * P.helem.size());
    std::vector<unsigned char> img(std::max<size_t>(total, 16));
    std::memcpy(img.data() + o_ao, a_off.data(), 8 * a_off.size());
    std::memcpy(img.data() + o_bo, b_off.data(), 8 * b_off.size());
    if (!ra.empty()) std::memcpy(img.data() + o_ra, ra.data(), ra.size());
    if (!rb.empty()) std::memcpy(img.data() + o_rb, rb.data(), rb.size());
    if (!P.helem.empty()) std::memcpy(img.data() + o_he, P.helem.data(), 4 * P.helem.size());
    void* blob = nullptr;
    cudaError_t ce = cudaMalloc(&blob, img.size());
    if (ce != cudaSuccess) return set_error(TGK_ERR_CUDA, std::string("fast plan: cudaMalloc: ") + cudaGetErrorString(ce));
    ce = cudaMemcpy(blob, img.data(), img.size(), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        cudaFree(blob);
        return set_error(TGK_ERR_CUDA, std::string("fast plan upload: ") + cudaGetErrorString(ce));
    }
    auto* base = static_cast<unsigned char*>(blob);
    D.blob = blob;
    D.bytes = static_cast<int64_t>(img.size());
    D.R = R;
    D.n_blocks = P.n_blocks;
    D.max_halo = P.max_halo;
    D.max_bnodes = P.max_bnodes;
    D.max_rows = P.max_rows;
    D.max_tile = max_tile;
    D.max_rec_a = max_a;
    D.max_rec_b = max_b;
    D.n_halo = static_cast<int64_t>(P.helem.size());
    D.n_items = static_cast<int64_t>(P.items.size());
    D.n_entries = static_cast<int64_t>(P.desc.size());
    D.row_lo = lo;
    D.row_hi = hi;
    D.elem_lo = elo;
    D.elem_hi = ehi;
    D.rec_a_off = reinterpret_cast<const int64_t*>(base + o_ao);
    D.rec_b_off = reinterpret_cast<const int64_t*>(base + o_bo);
    D.rec_a = base + o_ra;
    D.rec_b = base + o_rb;
    D.helem = reinterpret_cast<const uint32_t*>(base + o_he);
    *out = &D;
    return TGK_OK;
}

}  // namespace tgk
