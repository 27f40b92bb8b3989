// Host builder of the frequency-sliced tile M2L lists (K7 v11; C-ABI in
// include/defmm_b200.h: defmm_m2l_tiles).  Rows of one level and key, in
// (grandparent, parent, cell) = Morton order, are packed greedily parent by
// parent into tiles whose operand union (distinct source spectra + distinct
// derived symbols) stays within max_ops; a parent group that alone exceeds
// max_ops is packed row by row, and a row that alone exceeds it overflows to
// the row kernel.  Inside a tile, K consecutive siblings form a group whose
// events are merged per source spectrum (ascending source id, rows in order):
// the entry order of the sibling-group kernel, so the per-row sums are
// formed in the same order.  Operand counting uses per-operand stamps, O(events).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <tuple>
#include <vector>

#include "../../include/defmm_b200.h"

namespace {

struct Stamps {
    std::vector<int64_t> tile_s, tile_y, run_s, run_y;
    std::vector<int32_t> loc_s, loc_y;
    Stamps(int64_t n_hat, int64_t n_trans)
        : tile_s(n_hat, -1), tile_y(n_trans, -1), run_s(n_hat, -1), run_y(n_trans, -1), loc_s(n_hat, 0),
          loc_y(n_trans, 0) {}
};

}  // namespace

extern "C" int defmm_m2l_tiles(int64_t n_ids, const int64_t* ids, const int64_t* row_slot, const int64_t* row_ptr,
                               const int32_t* ent, const int64_t* l_cell, const int64_t* l_dir, const int64_t* level,
                               const int64_t* parent, int64_t n_hat, int64_t n_trans, int32_t K, int32_t max_ops,
                               int32_t max_ev, int64_t* out_ids, int64_t* tile_op_ptr, int32_t* ops, int64_t* tile_grp_ptr,
                               int32_t* grp_row, int64_t* grp_ent_ptr, uint16_t* ent_out, int64_t* overflow,
                               int64_t* counts) {
    if (n_ids < 0 || K < 1 || K > 7 || max_ops < 1 || max_ops > 65535 || max_ev < 1) return -1;
    const int ES = 8;
    // rows sorted by (level, key, grandparent, parent, cell)
    struct R {
        int64_t lev, key, gp, par, cell, id;
    };
    std::vector<R> rs((size_t)n_ids);
    for (int64_t i = 0; i < n_ids; ++i) {
        const int64_t r = ids[i];
        const int64_t c = l_cell[row_slot[r]];
        const int64_t p = parent[c];
        rs[(size_t)i] = {level[c], l_dir[row_slot[r]], p >= 0 ? parent[p] : -1, p, c, r};
    }
    std::sort(rs.begin(), rs.end(), [](const R& a, const R& b) {
        return std::tie(a.lev, a.key, a.gp, a.par, a.cell) < std::tie(b.lev, b.key, b.gp, b.par, b.cell);
    });
    Stamps st(n_hat, n_trans);
    int64_t n_tiles = 0, n_rows = 0, n_ops = 0, n_groups = 0, n_ent = 0, n_over = 0, run_id = 0;
    tile_op_ptr[0] = 0;
    tile_grp_ptr[0] = 0;
    grp_ent_ptr[0] = 0;
    // operands of rows [a, b) not yet in tile `tile`: count (deduplicated within the run)
    auto new_ops = [&](int64_t a, int64_t b, int64_t tile) {
        const int64_t run = run_id++;
        int64_t c = 0;
        for (int64_t i = a; i < b; ++i) {
            const int64_t r = rs[(size_t)i].id;
            for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
                const int32_t s = ent[2 * e], y = ent[2 * e + 1];
                if (st.tile_s[s] != tile && st.run_s[s] != run) {
                    st.run_s[s] = run;
                    ++c;
                }
                if (st.tile_y[y] != tile && st.run_y[y] != run) {
                    st.run_y[y] = run;
                    ++c;
                }
            }
        }
        return c;
    };
    auto events = [&](int64_t a, int64_t b) {
        int64_t c = 0;
        for (int64_t i = a; i < b; ++i) c += row_ptr[rs[(size_t)i].id + 1] - row_ptr[rs[(size_t)i].id];
        return c;
    };
    // current tile: rows [t0, t1) of rs, operand count, event count
    int64_t t0 = 0, t1 = 0, t_ops = 0, t_ev = 0;
    std::vector<std::tuple<int64_t, int, int64_t, int32_t>> ev;  // (source, k, row-in-group slot, local symbol)
    auto close_tile = [&]() {
        if (t1 == t0) return;
        const int64_t tile = n_tiles;
        // tile-local operand ids: sources (ascending), then symbols (ascending)
        std::vector<int32_t> src, sym;
        for (int64_t i = t0; i < t1; ++i) {
            const int64_t r = rs[(size_t)i].id;
            for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
                src.push_back(ent[2 * e]);
                sym.push_back(ent[2 * e + 1]);
            }
        }
        std::sort(src.begin(), src.end());
        src.erase(std::unique(src.begin(), src.end()), src.end());
        std::sort(sym.begin(), sym.end());
        sym.erase(std::unique(sym.begin(), sym.end()), sym.end());
        for (size_t j = 0; j < src.size(); ++j) {
            st.loc_s[src[j]] = (int32_t)j;
            ops[n_ops + (int64_t)j] = src[j];
        }
        for (size_t j = 0; j < sym.size(); ++j) {
            st.loc_y[sym[j]] = (int32_t)(src.size() + j);
            ops[n_ops + (int64_t)src.size() + (int64_t)j] = -1 - sym[j];
        }
        n_ops += (int64_t)(src.size() + sym.size());
        tile_op_ptr[tile + 1] = n_ops;
        // sibling groups of K rows, entries merged per source
        int64_t i = t0;
        while (i < t1) {
            int64_t j = i;
            while (j < t1 && j - i < K && rs[(size_t)j].par == rs[(size_t)i].par) ++j;
            const int64_t g = n_groups++;
            ev.clear();
            for (int k = 0; k < K; ++k) {
                if (i + k < j) {
                    out_ids[n_rows] = rs[(size_t)(i + k)].id;
                    grp_row[g * K + k] = (int32_t)n_rows++;
                    const int64_t r = rs[(size_t)(i + k)].id;
                    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e)
                        ev.emplace_back(ent[2 * e], k, 0, st.loc_y[ent[2 * e + 1]]);
                } else {
                    grp_row[g * K + k] = -1;
                }
            }
            std::sort(ev.begin(), ev.end(),
                      [](const auto& a, const auto& b) { return std::tie(std::get<0>(a), std::get<1>(a)) <
                                                                std::tie(std::get<0>(b), std::get<1>(b)); });
            for (size_t a = 0; a < ev.size();) {
                size_t b = a;
                uint16_t* o = ent_out + n_ent * ES;
                for (int c = 0; c < ES; ++c) o[c] = c <= K ? 0xFFFF : 0;
                o[0] = (uint16_t)st.loc_s[std::get<0>(ev[a])];
                while (b < ev.size() && std::get<0>(ev[b]) == std::get<0>(ev[a])) {
                    o[1 + std::get<1>(ev[b])] = (uint16_t)std::get<3>(ev[b]);
                    ++b;
                }
                ++n_ent;
                a = b;
            }
            grp_ent_ptr[g + 1] = n_ent;
            i = j;
        }
        tile_grp_ptr[tile + 1] = n_groups;
        ++n_tiles;
        t0 = t1;
        t_ops = 0;
        t_ev = 0;
    };
    auto commit = [&](int64_t a, int64_t b) {  // rows [a, b) join the current tile (stamps set)
        for (int64_t i = a; i < b; ++i) {
            const int64_t r = rs[(size_t)i].id;
            for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
                st.tile_s[ent[2 * e]] = n_tiles;
                st.tile_y[ent[2 * e + 1]] = n_tiles;
            }
        }
    };
    auto same_lk = [&](int64_t a, int64_t b) { return rs[(size_t)a].lev == rs[(size_t)b].lev && rs[(size_t)a].key == rs[(size_t)b].key; };
    int64_t i = 0;
    const int64_t n = n_ids;
    // pass 1: decide tiles over rs, moving overflow rows out (kept = rs without them)
    {
        std::vector<R> tmp;
        tmp.reserve((size_t)n);
        for (int64_t a = 0; a < n; ++a) {
            const int64_t r = rs[(size_t)a].id;
            // a row whose own operands exceed max_ops overflows
            const int64_t c = new_ops(a, a + 1, -2);
            if (c > max_ops || events(a, a + 1) > max_ev)
                overflow[n_over++] = r;
            else
                tmp.push_back(rs[(size_t)a]);
        }
        rs.swap(tmp);
    }
    const int64_t m = (int64_t)rs.size();
    while (i < m) {
        // the next parent run [i, j)
        int64_t j = i + 1;
        while (j < m && rs[(size_t)j].par == rs[(size_t)i].par && same_lk(i, j)) ++j;
        if (t1 > t0 && !same_lk(t0, i)) close_tile();
        const int64_t add = new_ops(i, j, n_tiles), add_ev = events(i, j);
        if (t_ops + add <= max_ops && t_ev + add_ev <= max_ev) {
            commit(i, j);
            t_ops += add;
            t_ev += add_ev;
            t1 = j;
            i = j;
            continue;
        }
        if (t1 > t0) {  // the run does not fit: close the tile and retry the run in a fresh one
            close_tile();
            continue;
        }
        // a parent run larger than a tile alone: row by row
        for (int64_t a = i; a < j; ++a) {
            const int64_t c = new_ops(a, a + 1, n_tiles), ce = events(a, a + 1);
            if ((t_ops + c > max_ops || t_ev + ce > max_ev) && t1 > t0) close_tile();
            const int64_t c2 = t1 > t0 ? c : new_ops(a, a + 1, n_tiles);
            commit(a, a + 1);
            t_ops += c2;
            t_ev += ce;
            t1 = a + 1;
        }
        i = j;
    }
    close_tile();
    counts[0] = n_tiles;
    counts[1] = n_rows;
    counts[2] = n_ops;
    counts[3] = n_groups;
    counts[4] = n_ent;
    counts[5] = n_over;
    return 0;
}
