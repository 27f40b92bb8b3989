// Host-native dual tree traversal for the defmm plan (C-ABI: include/defmm_b200.h).
//
// Restates the reference's recursive DTT (traversal.py:320-348; blank_dtt
// traversal.py:182-200 visits the same HF pairs) as a level-synchronous,
// TARGET-MAJOR sweep.  All visited pairs are same-level and the sons of a
// non-admissible non-leaf pair (t, s) are visited pairwise, so the candidate
// sources of every son of t are the sons of t's "near list" (in near-list
// order: the reference's depth-first order restricted to one target).  Per pair:
//   M2L  if gap^2 >= g2min[level]   (exact: the reference MAC is an up-set in
//        the integer gap^2; plan.py derives the threshold from the reference's
//        own FP64 expression, traversal.py:100-113)
//   P2P  else if t or s is a leaf   (traversal.py:336-343)
//   recurse otherwise               (traversal.py:345-348).
// The HF key (nearest direction, directions.py:78-89) of a translation is
// looked up in dense per-level tables over [-R, R]^3 computed by plan.py with
// the reference's exact numpy semantics.
//
// Outputs, all in one pass:
//  * M2L events in ROW order: rows = distinct (target, key), ordered by
//    (level, target, key); events of a row in traversal order.
//  * parent-pair blocks for the blocked M2L kernel: group = (level, key,
//    target parent P), holding the rows of P's children with that key;
//    block = (group, source parent Q) with per-child source events, the
//    translation of each child offset and the 64-bit (a, b) pair mask.
//    Groups are ordered (level, key, P); blocks of a group in first-use order
//    of Q along P's near list.
//  * P2P events (t, s) in traversal order.
//
// Each level is processed in parallel over chunks of target parents (all
// sons of a parent share one candidate list) and merged in chunk order, so
// the output does not depend on the thread count.  Sorting is by counting
// (keys: the level's direction range; blocks: Q's rank in P's near list).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "../../include/defmm_b200.h"

struct defmm_dtt_level {
    std::vector<int32_t> ev_s, ev_trans;          // events
    std::vector<int64_t> row_end;                 // global end event of each row
    std::vector<int32_t> row_t, row_key;
    std::vector<int64_t> grp_rows;                // 8 per group, global row id or -1
    std::vector<int32_t> grp_p, grp_key;
    std::vector<int64_t> grp_end;                 // global end block of each group
    std::vector<int64_t> blk_src;                 // 8 per block, global event id or -1
    std::vector<int32_t> blk_trans;               // 27 per block, dense translation id or -1
    std::vector<int64_t> blk_mask;
    std::vector<int32_t> p_t, p_s;                // near field
};

struct defmm_dtt {
    std::vector<defmm_dtt_level> lev;  // outputs per level (no regrowth copies)
    int64_t n_ev = 0, n_row = 0, n_grp = 0, n_blk = 0, n_pp = 0;
    std::vector<int64_t> trans_dense;  // used dense table entries, ascending (= compact id order)
    int nthr = 1;
};

namespace {

struct Tree {
    const int64_t* level_off;  // depth + 2 entries
    int32_t depth;
    const int64_t* coords;
    const int64_t* first_son;
    const int64_t* n_sons;
    const int64_t* parent;
};

struct Ev {       // one M2L event of a son of the current target parent
    int32_t key;  // level-local key (0 at LF levels)
    int32_t qr;   // rank of the source parent in the target parent's near list
    int32_t a, b, d;
    int32_t trans;
    int32_t s;
    int64_t ev;   // chunk-local event id
    int64_t row;  // chunk-local row id
};

struct Grp {
    int32_t key, p;
    int64_t rows[8];
    int64_t b0, b1;  // chunk-local block range
};

struct Chunk {  // everything one chunk of target parents produces
    std::vector<int32_t> ev_s, ev_trans;
    std::vector<int32_t> row_t, row_key;
    std::vector<int64_t> row_cnt;
    std::vector<Grp> grp;
    std::vector<int64_t> blk_src;
    std::vector<int32_t> blk_trans;
    std::vector<int64_t> blk_mask;
    std::vector<int32_t> p_t, p_s;
    std::vector<int64_t> near_s;
    int status = 0;
    void clear() {
        ev_s.clear(); ev_trans.clear(); row_t.clear(); row_key.clear(); row_cnt.clear(); grp.clear();
        blk_src.clear(); blk_trans.clear(); blk_mask.clear(); p_t.clear(); p_s.clear(); near_s.clear();
        status = 0;
    }
};

inline int octant(const int64_t* c, const int64_t* cp) {
    return (int)((c[0] - 2 * cp[0]) * 4 + (c[1] - 2 * cp[1]) * 2 + (c[2] - 2 * cp[2]));
}

int n_threads() {
    const char* e = std::getenv("DEFMM_PLAN_THREADS");
    int n = e ? std::atoi(e) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(n, 64));
}

// run fn(chunk index) for every chunk on a small thread pool
template <class F>
void parallel_chunks(int64_t nchunks, int nthr, F&& fn) {
    if (nthr <= 1 || nchunks <= 1) {
        for (int64_t c = 0; c < nchunks; ++c) fn(c);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    const int nt = (int)std::min<int64_t>(nthr, nchunks);
    for (int i = 0; i < nt; ++i)
        pool.emplace_back([&]() {
            for (int64_t c; (c = next.fetch_add(1)) < nchunks;) fn(c);
        });
    for (auto& th : pool) th.join();
}

// split [0, n) into contiguous chunks of roughly equal weight
std::vector<int64_t> split_by_weight(const std::vector<int64_t>& wcum, int64_t target_chunks) {
    const int64_t n = (int64_t)wcum.size() - 1;
    std::vector<int64_t> cut{0};
    const int64_t tot = wcum[n];
    const int64_t per = std::max<int64_t>(1, tot / std::max<int64_t>(1, target_chunks));
    int64_t next = per;
    for (int64_t i = 1; i < n; ++i)
        if (wcum[i] >= next) {
            cut.push_back(i);
            next = wcum[i] + per;
        }
    cut.push_back(n);
    if (n == 0) cut.assign({0, 0});
    return cut;
}

}  // namespace

extern "C" int defmm_dtt_build(const int64_t* t_level_off, int32_t t_depth, const int64_t* t_coords,
                               const int64_t* t_first_son, const int64_t* t_nsons, const int64_t* t_parent,
                               const int64_t* s_level_off, int32_t s_depth, const int64_t* s_coords,
                               const int64_t* s_first_son, const int64_t* s_nsons, const int64_t* s_parent,
                               int32_t depth, const int64_t* g2min, const int32_t* R, const int64_t* tab_off,
                               const int32_t* key_tab, defmm_dtt** out) {
    if (!out || !t_level_off || !s_level_off || !g2min || !R || !tab_off || !key_tab || depth < 0) return -1;
    *out = nullptr;
    defmm_dtt* d = new (std::nothrow) defmm_dtt();
    if (!d) return -2;
    const Tree T{t_level_off, t_depth, t_coords, t_first_son, t_nsons, t_parent};
    const Tree S{s_level_off, s_depth, s_coords, s_first_son, s_nsons, s_parent};
    const int nthr = n_threads();
    int status = 0;
    try {
        // candidates of the sons of target parent p (level l-1):
        // cand/cqr[cptr[p - off(l-1)] .. cptr[p - off(l-1) + 1]), cqr = rank of
        // the candidate's source parent in p's near list; cqn = near-list size
        std::vector<int64_t> cand{S.level_off[0]}, cptr{0, 1};
        std::vector<int32_t> cqr{0};
        std::vector<int64_t> cqn{1};
        std::vector<Chunk> chunks;
        std::vector<int32_t> near_c;   // per target of the level: chunk, range in its near_s
        std::vector<int64_t> near_b, near_e;
        for (int lev = 0; lev <= depth; ++lev) {
            if (lev > T.depth || lev > S.depth) break;
            auto tL = std::chrono::steady_clock::now();
            const int64_t t0 = T.level_off[lev], t1 = T.level_off[lev + 1];
            const int64_t g2m = g2min[lev];
            const int64_t r = R[lev];
            const int64_t w = 2 * r + 1;
            const int64_t toff = tab_off[lev];
            // level-local key range (HF levels); LF levels have the single key -1
            int32_t kmin = INT32_MAX, kmax = -1;
            for (int64_t i = tab_off[lev]; i < tab_off[lev + 1]; ++i)
                if (key_tab[i] >= 0) {
                    kmin = std::min(kmin, key_tab[i]);
                    kmax = std::max(kmax, key_tab[i]);
                }
            const bool hf = kmax >= 0;
            const int32_t kbase = hf ? kmin : -1;
            const int32_t nkey = hf ? kmax - kmin + 1 : 1;

            // target parents of this level (level 0: one virtual parent, the root target)
            const int64_t p0 = lev ? T.level_off[lev - 1] : 0, p1 = lev ? T.level_off[lev] : 1;
            const int64_t np_ = p1 - p0;
            std::vector<int64_t> wcum(np_ + 1, 0);
            for (int64_t i = 0; i < np_; ++i) {
                const int64_t ns = lev ? T.n_sons[p0 + i] : 1;
                wcum[i + 1] = wcum[i] + (cptr[i + 1] - cptr[i]) * ns + 1;
            }
            const std::vector<int64_t> cut = split_by_weight(wcum, (int64_t)nthr * 8);
            const int64_t nch = (int64_t)cut.size() - 1;
            if ((int64_t)chunks.size() < nch) chunks.resize(nch);
            near_c.assign(t1 - t0, 0);
            near_b.assign(t1 - t0, 0);
            near_e.assign(t1 - t0, 0);

            parallel_chunks(nch, nthr, [&](int64_t c) {
                Chunk& o = chunks[c];
                o.clear();
                std::vector<Ev> tev, stage, tmp;
                std::vector<int64_t> hist(hf ? nkey + 1 : 1);
                std::vector<int64_t> slot;
                auto count_sort = [&](std::vector<Ev>& v) {  // stable by key
                    if (!hf || v.size() < 2) return;
                    std::fill(hist.begin(), hist.end(), 0);
                    for (const Ev& e : v) ++hist[e.key + 1];
                    for (int32_t k = 0; k < nkey; ++k) hist[k + 1] += hist[k];
                    tmp.resize(v.size());
                    for (const Ev& e : v) tmp[hist[e.key]++] = e;
                    v.swap(tmp);
                };
                for (int64_t pi = cut[c]; pi < cut[c + 1] && !o.status; ++pi) {
                    const int64_t p = p0 + pi;
                    const int64_t la = cptr[pi], lb = cptr[pi + 1];
                    int64_t tb, te;
                    if (lev == 0) {
                        tb = t0;
                        te = t1;
                    } else {
                        if (T.n_sons[p] == 0) continue;
                        tb = T.first_son[p];
                        te = tb + T.n_sons[p];
                    }
                    stage.clear();
                    for (int64_t t = tb; t < te; ++t) {
                        const int a = lev ? octant(T.coords + 3 * t, T.coords + 3 * p) : 0;
                        tev.clear();
                        near_c[t - t0] = (int32_t)c;
                        near_b[t - t0] = (int64_t)o.near_s.size();
                        const int64_t* ct = T.coords + 3 * t;
                        const bool t_leaf = T.n_sons[t] == 0;
                        for (int64_t k = la; k < lb; ++k) {
                            const int64_t s = cand[k];
                            const int64_t* cs = S.coords + 3 * s;
                            const int64_t d0 = ct[0] - cs[0], d1 = ct[1] - cs[1], d2 = ct[2] - cs[2];
                            const int64_t g0 = std::max<int64_t>((d0 < 0 ? -d0 : d0) - 1, 0);
                            const int64_t g1 = std::max<int64_t>((d1 < 0 ? -d1 : d1) - 1, 0);
                            const int64_t g2 = std::max<int64_t>((d2 < 0 ? -d2 : d2) - 1, 0);
                            if (g0 * g0 + g1 * g1 + g2 * g2 >= g2m) {
                                if (lev == 0 || d0 < -r || d0 > r || d1 < -r || d1 > r || d2 < -r || d2 > r) {
                                    // outside the key table / an M2L between roots (no parent pair)
                                    o.status = lev == 0 ? -5 : -4;
                                    return;
                                }
                                const int64_t idx = toff + ((d0 + r) * w + (d1 + r)) * w + (d2 + r);
                                const int b = octant(cs, S.coords + 3 * S.parent[s]);
                                Ev e;
                                e.key = hf ? key_tab[idx] - kbase : 0;
                                e.qr = cqr[k];
                                e.a = a;
                                e.b = b;
                                e.d = ((((a >> 2) & 1) - ((b >> 2) & 1)) + 1) * 9 +
                                      ((((a >> 1) & 1) - ((b >> 1) & 1)) + 1) * 3 + ((a & 1) - (b & 1)) + 1;
                                e.trans = (int32_t)idx;
                                e.s = (int32_t)s;
                                tev.push_back(e);
                            } else if (t_leaf || S.n_sons[s] == 0) {
                                o.p_t.push_back((int32_t)t);
                                o.p_s.push_back((int32_t)s);
                            } else {
                                o.near_s.push_back(s);
                            }
                        }
                        near_e[t - t0] = (int64_t)o.near_s.size();
                        // rows = (t, key), events of a row in candidate order
                        count_sort(tev);
                        for (size_t i = 0; i < tev.size(); ++i) {
                            Ev& e = tev[i];
                            if (i == 0 || e.key != tev[i - 1].key) {
                                o.row_t.push_back((int32_t)t);
                                o.row_key.push_back(hf ? e.key + kbase : -1);
                                o.row_cnt.push_back(0);
                            }
                            ++o.row_cnt.back();
                            e.row = (int64_t)o.row_t.size() - 1;
                            e.ev = (int64_t)o.ev_s.size();
                            o.ev_s.push_back(e.s);
                            o.ev_trans.push_back(e.trans);
                            stage.push_back(e);
                        }
                    }
                    // parent-pair blocks of p: group per key, block per source parent
                    count_sort(stage);
                    if (slot.size() < (size_t)cqn[pi]) slot.assign(cqn[pi], -1);
                    size_t i = 0;
                    while (i < stage.size()) {
                        Grp g;
                        g.key = stage[i].key;
                        g.p = (int32_t)p;
                        for (int k = 0; k < 8; ++k) g.rows[k] = -1;
                        g.b0 = (int64_t)o.blk_mask.size();
                        size_t j = i;
                        for (; j < stage.size() && stage[j].key == g.key; ++j) {
                            const Ev& e = stage[j];
                            int64_t blk = slot[e.qr];
                            if (blk < 0) {
                                blk = slot[e.qr] = (int64_t)o.blk_mask.size();
                                o.blk_mask.push_back(0);
                                o.blk_src.insert(o.blk_src.end(), 8, -1);
                                o.blk_trans.insert(o.blk_trans.end(), 27, -1);
                            }
                            g.rows[e.a] = e.row;
                            o.blk_src[8 * blk + e.b] = e.ev;
                            o.blk_trans[27 * blk + e.d] = e.trans;
                            o.blk_mask[blk] |= (int64_t)((uint64_t)1 << (8 * e.a + e.b));
                        }
                        for (size_t k = i; k < j; ++k) slot[stage[k].qr] = -1;
                        g.b1 = (int64_t)o.blk_mask.size();
                        o.grp.push_back(g);
                        i = j;
                    }
                }
            });
            auto tA = std::chrono::steady_clock::now();
            for (int64_t c = 0; c < nch; ++c)
                if (chunks[c].status) status = chunks[c].status;
            if (status) break;

            // ---- ordered merge (chunk order; copies run in parallel) ------------
            struct Off { int64_t ev, row, grp, blk, pp; };
            std::vector<Off> off(nch + 1, Off{0, 0, 0, 0, 0});
            d->lev.emplace_back();
            defmm_dtt_level& L = d->lev.back();
            off[0] = Off{d->n_ev, d->n_row, 0, 0, 0};
            for (int64_t c = 0; c < nch; ++c) {
                const Chunk& o = chunks[c];
                off[c + 1] = Off{off[c].ev + (int64_t)o.ev_s.size(), off[c].row + (int64_t)o.row_t.size(),
                                 off[c].grp + (int64_t)o.grp.size(), off[c].blk + (int64_t)o.blk_mask.size(),
                                 off[c].pp + (int64_t)o.p_t.size()};
            }
            const int64_t ng = off[nch].grp, nb = off[nch].blk;
            const int64_t lev_ev = off[nch].ev - d->n_ev, lev_row = off[nch].row - d->n_row;
            L.ev_s.resize(lev_ev);
            L.ev_trans.resize(lev_ev);
            L.row_t.resize(lev_row);
            L.row_key.resize(lev_row);
            L.row_end.resize(lev_row);
            L.p_t.resize(off[nch].pp);
            L.p_s.resize(off[nch].pp);
            std::vector<Grp> lgrp(ng);
            std::vector<int64_t> lsrc(8 * nb);
            std::vector<int32_t> ltr(27 * nb);
            std::vector<int64_t> lmask(nb);
            parallel_chunks(nch, nthr, [&](int64_t c) {
                const Chunk& o = chunks[c];
                const Off& f = off[c];
                const int64_t le = f.ev - d->n_ev, lr = f.row - d->n_row;
                std::copy(o.ev_s.begin(), o.ev_s.end(), L.ev_s.begin() + le);
                std::copy(o.ev_trans.begin(), o.ev_trans.end(), L.ev_trans.begin() + le);
                std::copy(o.row_t.begin(), o.row_t.end(), L.row_t.begin() + lr);
                std::copy(o.row_key.begin(), o.row_key.end(), L.row_key.begin() + lr);
                int64_t e = f.ev;
                for (size_t i = 0; i < o.row_cnt.size(); ++i) L.row_end[lr + i] = (e += o.row_cnt[i]);
                std::copy(o.p_t.begin(), o.p_t.end(), L.p_t.begin() + f.pp);
                std::copy(o.p_s.begin(), o.p_s.end(), L.p_s.begin() + f.pp);
                for (size_t i = 0; i < o.grp.size(); ++i) {
                    Grp g = o.grp[i];
                    for (int k = 0; k < 8; ++k)
                        if (g.rows[k] >= 0) g.rows[k] += f.row;
                    g.b0 += f.blk;
                    g.b1 += f.blk;
                    lgrp[f.grp + i] = g;
                }
                for (size_t i = 0; i < o.blk_src.size(); ++i)
                    lsrc[8 * f.blk + i] = o.blk_src[i] >= 0 ? o.blk_src[i] + f.ev : -1;
                std::copy(o.blk_trans.begin(), o.blk_trans.end(), ltr.begin() + 27 * f.blk);
                std::copy(o.blk_mask.begin(), o.blk_mask.end(), lmask.begin() + f.blk);
            });
            // groups of this level in (key, P) order (merged in P order):
            // stable counting sort by key, then gather the blocks
            std::vector<int64_t> gorder(ng);
            {
                std::vector<int64_t> h(nkey + 1, 0);
                for (const Grp& g : lgrp) ++h[g.key + 1];
                for (int32_t k = 0; k < nkey; ++k) h[k + 1] += h[k];
                for (int64_t i = 0; i < ng; ++i) gorder[h[lgrp[i].key]++] = i;
            }
            const int64_t b_base = d->n_blk;
            std::vector<int64_t> nbo(ng + 1, 0);  // new block offset per ordered group
            for (int64_t i = 0; i < ng; ++i) nbo[i + 1] = nbo[i] + (lgrp[gorder[i]].b1 - lgrp[gorder[i]].b0);
            L.grp_rows.resize(8 * ng);
            L.grp_p.resize(ng);
            L.grp_key.resize(ng);
            L.grp_end.resize(ng);
            L.blk_src.resize(8 * nb);
            L.blk_trans.resize(27 * nb);
            L.blk_mask.resize(nb);
            std::vector<int64_t> gw(ng + 1);
            for (int64_t i = 0; i <= ng; ++i) gw[i] = nbo[i] + i;
            const std::vector<int64_t> gcut = split_by_weight(gw, (int64_t)nthr * 4);
            parallel_chunks((int64_t)gcut.size() - 1, nthr, [&](int64_t c) {
                for (int64_t i = gcut[c]; i < gcut[c + 1]; ++i) {
                    const Grp& g = lgrp[gorder[i]];
                    const int64_t bo = nbo[i];
                    std::copy(g.rows, g.rows + 8, L.grp_rows.begin() + 8 * i);
                    L.grp_p[i] = g.p;
                    L.grp_key[i] = hf ? g.key + kbase : -1;
                    L.grp_end[i] = b_base + nbo[i + 1];
                    std::copy(lsrc.begin() + 8 * g.b0, lsrc.begin() + 8 * g.b1, L.blk_src.begin() + 8 * bo);
                    std::copy(ltr.begin() + 27 * g.b0, ltr.begin() + 27 * g.b1, L.blk_trans.begin() + 27 * bo);
                    std::copy(lmask.begin() + g.b0, lmask.begin() + g.b1, L.blk_mask.begin() + bo);
                }
            });
            d->n_ev += lev_ev;
            d->n_row += lev_row;
            d->n_grp += ng;
            d->n_blk += nb;
            d->n_pp += off[nch].pp;
            auto tB = std::chrono::steady_clock::now();
            if (std::getenv("DEFMM_PLAN_DEBUG"))
                std::fprintf(stderr, "lev %d: classify %.3f s merge %.3f s ev %zu\n", lev,
                             std::chrono::duration<double>(tA - tL).count(), std::chrono::duration<double>(tB - tA).count(),
                             (size_t)d->n_ev);
            if (lev == depth) break;

            // ---- next level's candidates: sons of near(t) for every target t --
            const int64_t nt = t1 - t0;
            std::vector<int64_t> ncptr(nt + 1, 0), ncqn(nt, 0);
            for (int64_t i = 0; i < nt; ++i) {
                const Chunk& o = chunks[near_c[i]];
                int64_t n = 0;
                for (int64_t k = near_b[i]; k < near_e[i]; ++k) n += S.n_sons[o.near_s[k]];
                ncptr[i + 1] = ncptr[i] + n;
                ncqn[i] = near_e[i] - near_b[i];
            }
            std::vector<int64_t> ncand(ncptr[nt]);
            std::vector<int32_t> ncqr(ncptr[nt]);
            std::vector<int64_t> tw(nt + 1);
            for (int64_t i = 0; i <= nt; ++i) tw[i] = ncptr[i] + i;
            const std::vector<int64_t> tcut = split_by_weight(tw, (int64_t)nthr * 4);
            parallel_chunks((int64_t)tcut.size() - 1, nthr, [&](int64_t c) {
                for (int64_t i = tcut[c]; i < tcut[c + 1]; ++i) {
                    const Chunk& o = chunks[near_c[i]];
                    int64_t pos = ncptr[i];
                    for (int64_t k = near_b[i]; k < near_e[i]; ++k) {
                        const int64_t s = o.near_s[k];
                        for (int64_t son = S.first_son[s]; son < S.first_son[s] + S.n_sons[s]; ++son) {
                            ncand[pos] = son;
                            ncqr[pos] = (int32_t)(k - near_b[i]);
                            ++pos;
                        }
                    }
                }
            });
            cand.swap(ncand);
            cqr.swap(ncqr);
            cptr.swap(ncptr);
            cqn.swap(ncqn);
        }
        // ---- translation ids: dense table index -> rank among the used entries
        if (!status) {
            const int64_t ntab = tab_off[depth + 1];
            std::vector<uint8_t> used(ntab, 0);
            for (const auto& L : d->lev)
                for (int32_t v : L.ev_trans) used[v] = 1;
            std::vector<int32_t> remap(ntab, -1);
            for (int64_t i = 0; i < ntab; ++i)
                if (used[i]) {
                    remap[i] = (int32_t)d->trans_dense.size();
                    d->trans_dense.push_back(i);
                }
            for (auto& L : d->lev) {
                const int64_t n = (int64_t)L.ev_trans.size(), per = n / (4 * nthr) + 1;
                parallel_chunks((n + per - 1) / per, nthr, [&](int64_t c) {
                    for (int64_t i = c * per; i < std::min(n, (c + 1) * per); ++i) L.ev_trans[i] = remap[L.ev_trans[i]];
                });
                for (int32_t& v : L.blk_trans)
                    if (v >= 0) v = remap[v];
            }
        }
        d->nthr = nthr;
    } catch (...) {
        delete d;
        return -2;
    }
    if (status) {
        delete d;
        return status;
    }
    *out = d;
    return 0;
}

extern "C" int defmm_dtt_sizes(const defmm_dtt* d, int64_t* sizes) {
    if (!d || !sizes) return -1;
    sizes[0] = d->n_ev;
    sizes[1] = d->n_row;
    sizes[2] = d->n_grp;
    sizes[3] = d->n_blk;
    sizes[4] = d->n_pp;
    sizes[5] = (int64_t)d->trans_dense.size();
    return 0;
}

namespace {
template <class T>
T* put(T* dst, const std::vector<T>& v) {
    if (!dst) return nullptr;
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
    return dst + v.size();
}
template <class T>
T* fill(T* dst, size_t n, T v) {
    if (!dst) return nullptr;
    std::fill(dst, dst + n, v);
    return dst + n;
}
}  // namespace

extern "C" int defmm_dtt_fetch(const defmm_dtt* d, int32_t* ev_s, int32_t* ev_trans, int64_t* row_ptr,
                               int32_t* row_t, int32_t* row_key, int32_t* row_lev, int64_t* grp_rows,
                               int32_t* grp_p, int32_t* grp_key, int32_t* grp_lev, int64_t* grp_ptr,
                               int64_t* blk_src, int32_t* blk_trans, int64_t* blk_mask, int32_t* p_t,
                               int32_t* p_s) {
    if (!d) return -1;
    if (row_ptr) *row_ptr++ = 0;
    if (grp_ptr) *grp_ptr++ = 0;
    for (size_t l = 0; l < d->lev.size(); ++l) {
        const defmm_dtt_level& L = d->lev[l];
        ev_s = put(ev_s, L.ev_s);
        ev_trans = put(ev_trans, L.ev_trans);
        row_ptr = put(row_ptr, L.row_end);
        row_t = put(row_t, L.row_t);
        row_key = put(row_key, L.row_key);
        row_lev = fill(row_lev, L.row_t.size(), (int32_t)l);
        grp_rows = put(grp_rows, L.grp_rows);
        grp_p = put(grp_p, L.grp_p);
        grp_key = put(grp_key, L.grp_key);
        grp_lev = fill(grp_lev, L.grp_p.size(), (int32_t)l);
        grp_ptr = put(grp_ptr, L.grp_end);
        blk_src = put(blk_src, L.blk_src);
        blk_trans = put(blk_trans, L.blk_trans);
        blk_mask = put(blk_mask, L.blk_mask);
        p_t = put(p_t, L.p_t);
        p_s = put(p_s, L.p_s);
    }
    return 0;
}

extern "C" int defmm_dtt_translations(const defmm_dtt* d, int64_t* dense_ids) {
    if (!d) return -1;
    put(dense_ids, d->trans_dense);
    return 0;
}

extern "C" int defmm_dtt_source_hats(const defmm_dtt* d, const int64_t* m_dense, const int64_t* base,
                                     const int64_t* nd, const int64_t* s_level_off, const int32_t* key_base,
                                     int64_t n_mult, int32_t* src_hat, int64_t* hat_slot, int64_t* n_hat) {
    if (!d || !m_dense || !base || !nd || !s_level_off || !key_base || !src_hat || !hat_slot || !n_hat) return -1;
    // pass 1: multipole slot of every event's (source cell, key)
    std::atomic<int> bad{0};
    int64_t e_off = 0;
    for (size_t l = 0; l < d->lev.size(); ++l) {
        const defmm_dtt_level& L = d->lev[l];
        const int64_t nr = (int64_t)L.row_t.size(), per = nr / (4 * d->nthr) + 1;
        const int64_t e0 = e_off;
        parallel_chunks((nr + per - 1) / per, d->nthr, [&](int64_t c) {
            const int64_t r0 = c * per, r1 = std::min(nr, (c + 1) * per);
            int64_t e = r0 ? L.row_end[r0 - 1] : e0;
            for (int64_t r = r0; r < r1; ++r) {
                const int64_t loc = L.row_key[r] >= 0 ? L.row_key[r] - key_base[l] : 0;
                for (; e < L.row_end[r]; ++e) {
                    const int64_t sl = m_dense[base[l] + (L.ev_s[e - e0] - s_level_off[l]) * nd[l] + loc];
                    if (sl < 0 || sl >= n_mult) bad.store(1);
                    src_hat[e] = (int32_t)sl;
                }
            }
        });
        e_off += (int64_t)L.ev_s.size();
    }
    if (bad.load()) return -6;  // an M2L source without its expansion (blank-pass inconsistency)
    // pass 2: spectra = used multipole slots, ascending
    std::vector<int32_t> rank(n_mult, -1);
    for (int64_t e = 0; e < e_off; ++e) rank[src_hat[e]] = 0;
    int64_t k = 0;
    for (int64_t i = 0; i < n_mult; ++i)
        if (rank[i] == 0) {
            rank[i] = (int32_t)k;
            hat_slot[k++] = i;
        }
    *n_hat = k;
    const int64_t per = e_off / (4 * d->nthr) + 1;
    parallel_chunks((e_off + per - 1) / per, d->nthr, [&](int64_t c) {
        for (int64_t e = c * per; e < std::min(e_off, (c + 1) * per); ++e) src_hat[e] = rank[src_hat[e]];
    });
    return 0;
}

extern "C" void defmm_dtt_free(defmm_dtt* d) { delete d; }
