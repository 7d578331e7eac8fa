// Host construction of the fast-mode plan (TGK_MODE_FAST, fast.cu).
//
// The plan is the north star's "precomputed element-to-CSR-slot permutation":
// for every CSR entry a CUDA block owns, the list of (halo element, local
// pair) whose local value lands on it — exactly the segments of the
// reference's mat_offsets/mat_slots (routing.cpp:64-84), re-expressed as
// shared-memory addresses of the block's element values.  Layout:
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
//  - per warp of 32 entries the items, interleaved [step][lane][4 bytes] so
//    every step is one coalesced 4-byte load per lane (two u16 items).  Items are direct
//    indices of the values in the block's shared-memory value rows (format
//    below); short lists are padded with the zero slot.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <thread>

#include <cuda_runtime.h>

#include "tgk_internal.hpp"

namespace tgk {

namespace {

constexpr int kSymTet[4][4] = {{0, 1, 2, 3}, {1, 4, 5, 6}, {2, 5, 7, 8}, {3, 6, 8, 9}};
constexpr int kSymTri[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};

inline int sym_pair_k(int k, int a, int b) { return k == 4 ? kSymTet[a][b] : kSymTri[a][b]; }

// value row of a packed pair (sym index): K_aa rows 0..k-1, then the
// off-diagonal pairs in sym order (tet: 01 02 03 12 13 23; tri: 01 02 12)
inline int pair_row(int k, int q) {
    if (k == 4) {
        static const int r[10] = {0, 4, 5, 6, 1, 7, 8, 2, 9, 3};
        return r[q];
    }
    static const int r[6] = {0, 3, 4, 1, 5, 2};
    return r[q];
}

// value row of an off-diagonal pair in the fast kernel (fast.cu FastCfg): the
// K_aa rows are not stored — the diagonal comes from the zero row sums of the
// assembled stiffness (k_fast_scalar copy-out)
inline int offdiag_row(int k, int q) { return pair_row(k, q) - k; }

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
        std::vector<uint32_t> list_off;  // per entry, n+1 (block-relative)
        std::vector<uint16_t> items;     // generic items: halo index | (a * 4 + b) << 12 (row node a, column node b)
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
            struct Ent {
                int cls, len, lr, p;
                uint32_t desc;
                int list;
            };
            std::vector<Ent> ents;
            lists.clear();
            for (int lr = 0; lr < static_cast<int>(o.rows.size()); ++lr) {
                const uint32_t row = o.rows[lr];
                const int64_t rp = row_ptr[row];
                const int len = static_cast<int>(row_ptr[row + 1] - rp);
                std::vector<int> col(len, -1);   // owned local row of the column, or -1
                std::vector<int> pos2(len, -1);  // position of `row` within that row
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
                        if (use) ent[p].push_back(static_cast<uint16_t>(h | ((a * 4 + bb) << 12)));
                    }
                    if (use) diag.push_back(static_cast<uint16_t>(h | ((a * 4 + a) << 12)));
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
            for (auto& en : ents) en.len = static_cast<int>(lists[en.list].size());
            std::stable_sort(ents.begin(), ents.end(), [](const Ent& x, const Ent& y) {
                if (x.cls != y.cls) return x.cls < y.cls;
                if (x.len != y.len) return x.len > y.len;
                if (x.lr != y.lr) return x.lr < y.lr;
                return x.p < y.p;
            });
            o.list_off.push_back(0);
            const int dsplit = kFastDiagSplit(k);
            for (int cls = 0; cls < 2; ++cls) {
                size_t n = 0;
                for (const auto& en : ents) {
                    if (en.cls != cls) continue;
                    const auto& li = lists[en.list];
                    // a diagonal entry's list (the row's incident elements, ~24 in 3D)
                    // is split over dsplit consecutive lanes, summed by shuffles:
                    // balanced warps instead of a few long folds
                    const int parts = cls == 0 ? dsplit : 1;
                    const size_t chunk = (li.size() + parts - 1) / parts;
                    for (int q = 0; q < parts; ++q) {
                        o.desc.push_back(q == 0 ? en.desc : kFastPart);
                        const size_t t0 = std::min(li.size(), q * chunk), t1 = std::min(li.size(), t0 + chunk);
                        o.items.insert(o.items.end(), li.begin() + t0, li.begin() + t1);
                        o.list_off.push_back(static_cast<uint32_t>(o.items.size()));
                        ++n;
                    }
                }
                for (; n % 32; ++n) {  // whole warps per class
                    o.desc.push_back(kFastIdle);
                    o.list_off.push_back(static_cast<uint32_t>(o.items.size()));
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
    cat(&BlockOut::items, &P.item_off, P.items);
    P.list_off.clear();
    for (int64_t b = 0; b < nb; ++b) {  // block-relative, n+1 per block
        P.list_off.insert(P.list_off.end(), out[b].list_off.begin(), out[b].list_off.end());
        P.max_halo = std::max<int>(P.max_halo, static_cast<int>(out[b].helem.size()));
        P.max_bnodes = std::max<int>(P.max_bnodes, static_cast<int>(out[b].bnodes.size()));
        P.max_rows = std::max<int>(P.max_rows, static_cast<int>(out[b].rows.size()));
    }
    return TGK_OK;
}

// ---------------------------------------------------------------------------
// Upload: two byte records per block (layout in tgk_internal.hpp FastPlanDev)
// with the items resolved for the value-row formats (fast.cu FastCfg):
//   scalar formats (kFastFmtK16 stiffness [+ load], kFastFmtKS32 + unit mass,
//                kFastFmtS16 coefficient mass) share one item layout, u16 =
//                h | row << 12: an off-diagonal item names the K_ab value row
//                (0 .. k(k-1)/2 - 1), a diagonal item the local node a (the
//                kernel forms the S / F indices from h and a).  The stiffness
//                diagonal is not folded: it is minus the row's off-diagonal
//                sum (zero row sums of P1 stiffness), formed at the copy-out;
//   kFastFmtE16  vector elasticity (fast.cu k_fast_elast): items u16 = the
//                generic h | (a * 4 + b) << 12, the kernel reads the scaled
//                gradients of nodes a, b of halo element h.
// MH = max halo + 1: index MH - 1 of every row is the +0.0 padding slot.
void FastPlanDev::release() {
    if (blob) cudaFree(blob);
    *this = FastPlanDev{};
}

int fast_value_rows(int k, int fmt, bool fnodal) {
    const int npo = k * (k - 1) / 2;  // off-diagonal pairs (fast.cu FastCfg::NPO)
    if (fmt == kFastFmtS16) return 1;
    if (fmt == kFastFmtE16) return 1;  // items carry (h, a, b), not value indices
    if (fmt == kFastFmtKS32) return npo + 2;
    return npo + (fnodal ? k : 1);
}

int ensure_fast_plan(tgk_routing* rr, int R, int fmt, bool fnodal, const FastPlanDev** out) {
    tgk_routing* r = rr->scalar ? rr->scalar : rr;
    const int64_t lo = r->own_hi < 0 ? 0 : r->own_lo, hi = r->own_hi < 0 ? r->N : r->own_hi;
    const int64_t elo = r->elem_hi < 0 ? 0 : r->elem_lo, ehi = r->elem_hi < 0 ? r->E : r->elem_hi;
    for (auto& D : r->fast_plan)
        if (D.blob && D.R == R && D.fmt == fmt && D.fnodal == fnodal && D.row_lo == lo && D.row_hi == hi &&
            D.elem_lo == elo && D.elem_hi == ehi) {
            *out = r->fast_plan_used = &D;
            return TGK_OK;
        }
    FastPlanDev* slot = nullptr;
    for (auto& D : r->fast_plan)
        if (!D.blob) {
            slot = &D;
            break;
        }
    if (!slot) slot = &r->fast_plan[r->fast_plan_next++ % kFastPlanSlots];  // evict round-robin
    slot->release();
    FastPlanDev& D = *slot;
    const tgk_mesh* m = r->mesh;
    const int k = m->k;
    ScalarRoutingHost h;
    TGK_TRY(fetch_scalar_routing(r, h));
    FastPlanHost P;
    const int rc = build_fast_plan(m->kind, m->N, m->E, h.nodes.data(), h.conn.data(), h.row_ptr.data(), h.vo.data(),
                                   h.vs.data(), h.slot.data(), lo, hi, elo, ehi, R, P);
    if (rc != TGK_OK) return rc;
    const int MH = P.max_halo + 1;
    const int NP = k * (k + 1) / 2;
    const uint32_t zero = uint32_t(MH - 1);  // padding item: halo slot max_halo (+0.0), row 0
    // generic item -> resolved index / word
    // scalar formats: u16 = h | (value row of K_ab) << 12 — off-diagonal pairs
    // their row (k..NP-1), diagonals a (row a = K_aa); the kernel forms the
    // S / F indices from h (and a) itself.  Elasticity: the generic item.
    (void)NP;
    (void)zero;
    auto off_item = [&](uint16_t g) -> uint32_t {
        if (fmt == kFastFmtE16) return g;  // elasticity: the kernel reads g_a, g_b of element h
        const uint32_t hh = g & 0xfffu, a = (g >> 12) >> 2, b = (g >> 12) & 3u;
        return hh | (uint32_t(offdiag_row(k, sym_pair_k(k, int(a), int(b)))) << 12);
    };
    auto diag_item = [&](uint16_t g) -> uint32_t {
        if (fmt == kFastFmtE16) return g;
        return (g & 0xfffu) | (uint32_t((g >> 12) >> 2) << 12);
    };
    auto al16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    const int64_t nb = P.n_blocks;
    // block-local connectivity bytes per halo element: 4 x u8 when every block's
    // node table fits 255 entries (halves the largest part of record A)
    const int hc8 = P.max_bnodes <= 255 ? 1 : 0;
    const size_t hcb = hc8 ? 4 : 8;
    std::vector<int64_t> a_off(nb + 1, 0), b_off(nb + 1, 0);
    std::vector<std::vector<unsigned char>> recb(nb);
    int max_a = 0, max_b = 0, max_tile = 0, max_len = 0;
    int64_t n_words = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const size_t nr = size_t(P.row_off[b + 1] - P.row_off[b]), nh = size_t(P.halo_off[b + 1] - P.halo_off[b]),
                     nbn = size_t(P.bnode_off[b + 1] - P.bnode_off[b]);
        const size_t sa = 32 + al16(8 * nr) + al16(4 * nr) + al16(2 * (nr + 1)) + al16(4 * nbn) + al16(hcb * nh);
        a_off[b + 1] = a_off[b] + int64_t(sa);
        max_a = std::max<int>(max_a, int(sa));
        // record B: header, descriptors, warp-group word offsets, words
        const int64_t e0 = P.ent_off[b];
        const uint32_t ne = uint32_t(P.ent_off[b + 1] - e0), nwg = ne / 32;
        const uint32_t* loff = P.list_off.data() + e0 + b;  // block-relative, n+1
        const uint16_t* gi = P.items.data() + P.item_off[b];
        std::vector<uint32_t> wgoff(nwg + 1, 0), words;
        for (uint32_t w = 0; w < nwg; ++w) {
            const bool diag = (P.desc[e0 + w * 32] >> 15) & 1u;  // lane 0 is never idle
            // u16 items, 2 per 4-byte word, one word per lane per step
            // ([step][lane]: each step one coalesced 128-byte warp load)
            int steps = 0;
            for (int l = 0; l < 32; ++l) {
                const int n = int(loff[w * 32 + l + 1] - loff[w * 32 + l]);
                steps = std::max(steps, (n + 1) / 2);
            }
            const size_t base = words.size();
            words.resize(base + size_t(steps) * 32, zero | (zero << 16));
            for (int l = 0; l < 32; ++l) {
                const uint32_t i0 = loff[w * 32 + l], i1 = loff[w * 32 + l + 1];
                for (uint32_t t = 0; t < i1 - i0; ++t) {
                    const uint32_t v = diag ? diag_item(gi[i0 + t]) : off_item(gi[i0 + t]);
                    uint32_t& wd = words[base + size_t(t / 2) * 32 + size_t(l)];
                    wd = (t % 2) ? ((wd & 0xffffu) | (v << 16)) : ((wd & 0xffff0000u) | v);
                }
            }
            wgoff[w + 1] = uint32_t(words.size());
        }
        const size_t sb = 16 + al16(4 * size_t(ne)) + al16(4 * size_t(nwg + 1)) + al16(4 * words.size());
        auto& rbv = recb[b];
        rbv.assign(sb, 0);
        const uint32_t hb[2] = {ne, nwg};
        std::memcpy(rbv.data(), hb, 8);
        size_t o = 16;
        std::memcpy(rbv.data() + o, P.desc.data() + e0, 4 * size_t(ne));
        o += al16(4 * size_t(ne));
        std::memcpy(rbv.data() + o, wgoff.data(), 4 * size_t(nwg + 1));
        o += al16(4 * size_t(nwg + 1));
        if (!words.empty()) std::memcpy(rbv.data() + o, words.data(), 4 * words.size());
        n_words += int64_t(words.size());
        b_off[b + 1] = b_off[b] + int64_t(sb);
        max_b = std::max<int>(max_b, int(sb));
    }
    std::vector<unsigned char> ra(size_t(a_off[nb])), rb(size_t(b_off[nb]));
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t r0 = P.row_off[b], h0 = P.halo_off[b], n0 = P.bnode_off[b];
        const uint32_t nr = uint32_t(P.row_off[b + 1] - r0), nh = uint32_t(P.halo_off[b + 1] - h0),
                       nbn = uint32_t(P.bnode_off[b + 1] - n0);
        unsigned char* pa = ra.data() + a_off[b];
        std::vector<uint16_t> toff(nr + 1, 0);
        for (uint32_t i = 0; i < nr; ++i) {
            const uint32_t row = P.rows[r0 + i];
            toff[i + 1] = uint16_t(toff[i] + (h.row_ptr[row + 1] - h.row_ptr[row]));
            max_len = std::max<int>(max_len, int(h.row_ptr[row + 1] - h.row_ptr[row]));
        }
        max_tile = std::max<int>(max_tile, toff[nr]);
        const uint32_t hdr[4] = {nr, nh, nbn, toff[nr]};
        std::memcpy(pa, &h0, 8);
        std::memcpy(pa + 8, hdr, 16);
        {  // byte offsets of srow / toff / bnodes / hconn (the kernels read them, no arithmetic)
            const size_t o_srow = 32 + al16(8 * size_t(nr)), o_toff = o_srow + al16(4 * size_t(nr)),
                         o_bn = o_toff + al16(2 * size_t(nr + 1)), o_hc = o_bn + al16(4 * size_t(nbn));
            const uint16_t offs[4] = {uint16_t(o_srow), uint16_t(o_toff), uint16_t(o_bn), uint16_t(o_hc)};
            std::memcpy(pa + 24, offs, 8);
        }
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
        if (hc8) {
            for (uint32_t i = 0; i < nh; ++i) {
                const uint64_t hc = P.hconn[h0 + i];
                const uint32_t c8 = uint32_t(hc & 0xff) | uint32_t((hc >> 16) & 0xff) << 8 |
                                    uint32_t((hc >> 32) & 0xff) << 16 | uint32_t((hc >> 48) & 0xff) << 24;
                std::memcpy(pa + o + 4 * size_t(i), &c8, 4);
            }
        } else {
            std::memcpy(pa + o, P.hconn.data() + h0, 8 * size_t(nh));
        }
        std::memcpy(rb.data() + b_off[b], recb[b].data(), recb[b].size());
    }
    recb.clear();
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
    D.fmt = fmt;
    D.fnodal = fnodal;
    D.MH = MH;
    D.n_blocks = P.n_blocks;
    D.max_halo = P.max_halo;
    D.max_bnodes = P.max_bnodes;
    D.max_rows = P.max_rows;
    D.max_tile = max_tile;
    D.max_len = max_len;
    D.max_rec_a = max_a;
    D.max_rec_b = max_b;
    D.hc8 = hc8;
    D.n_halo = static_cast<int64_t>(P.helem.size());
    D.n_items = static_cast<int64_t>(P.items.size());
    D.n_words = n_words;
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
    *out = r->fast_plan_used = &D;
    return TGK_OK;
}

}  // namespace tgk

extern "C" int tgk_routing_fast_plan_info(const tgk_routing* rr, int* rows_per_block, int64_t* n_blocks, int64_t* n_halo,
                                          int64_t* n_entries, int64_t* n_words, int64_t* bytes) {
    if (!rr) return tgk::set_error(TGK_ERR_INPUT, "null routing");
    const tgk_routing* r = rr->scalar ? rr->scalar : rr;
    const tgk::FastPlanDev* D = r->fast_plan_used;
    if (!D || !D->blob) return tgk::set_error(TGK_ERR_INPUT, "no fast-mode assembly on this routing yet");
    if (rows_per_block) *rows_per_block = D->R;
    if (n_blocks) *n_blocks = D->n_blocks;
    if (n_halo) *n_halo = D->n_halo;
    if (n_entries) *n_entries = D->n_entries;
    if (n_words) *n_words = D->n_words;
    if (bytes) *bytes = D->bytes;
    return TGK_OK;
}

namespace tgk {

}  // namespace tgk
