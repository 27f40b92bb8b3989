// Host-native tiling of the M2L rows for the shared-memory tile kernel
// (K7 v6, defmm_m2l_tile_*; C-ABI: include/defmm_b200.h).
//
// A tile is a run of consecutive rows (callers order them (level, key,
// Morton target)) whose source spectra and derived symbols, as a UNION, fit
// the kernel's shared-memory budget of u_max operand slices.  Morton-adjacent
// rows with the same key share most of their sources and (shifted by one
// cell) most of their translations, so the union is 4-8x smaller than the
// rows' 2 * events operand loads (cfg2: SURVEY §8(d) list shapes, measured
// in profiles/r01_summary_v5.md).  The kernel stages the union once per
// frequency slice and reads every event's operands from shared memory.
//
// Greedy, one pass, O(events): a row joins the open tile if the union grows
// to at most u_max operands and the tile has fewer than k_max rows; otherwise
// the tile is closed and the row opens the next one (also when the tile would
// exceed e_max events, the kernel's shared-memory event buffer).  A row whose
// own operands exceed u_max (or events e_max) is not tiled (the caller runs
// it on the row kernel).
#include <cstdint>
#include <vector>

#include "../../include/defmm_b200.h"

extern "C" int defmm_m2l_tiles(int64_t n_order, const int64_t* order, const int64_t* row_ptr, const int32_t* ent,
                               int64_t n_hat, int64_t n_trans, int32_t u_max, int32_t k_max, int32_t e_max,
                               int64_t* tile_ptr,
                               int64_t* tile_rows, int64_t* op_ptr, int32_t* ops, int64_t* ev_ptr, uint32_t* ev,
                               int64_t* counts) {
    if (u_max <= 0 || u_max > 65535 || k_max <= 0 || e_max <= 0) return -1;
    // stamps: which tile an operand was last added to, and its local index
    std::vector<int64_t> s_tile(n_hat, -1), t_tile(n_trans, -1);
    std::vector<int32_t> s_loc(n_hat, 0), t_loc(n_trans, 0);
    std::vector<int64_t> s_trial(n_hat, -1), t_trial(n_trans, -1);
    int64_t n_tiles = 0, n_rows = 0, n_ops = 0, n_ev = 0, n_untiled = 0;
    int64_t tile = -1;  // open tile id
    int32_t tile_u = 0, tile_k = 0;
    int64_t tile_e = 0;
    tile_ptr[0] = 0;
    op_ptr[0] = 0;
    ev_ptr[0] = 0;
    auto close_tile = [&]() {
        if (tile >= 0 && tile_k > 0) {
            ++n_tiles;
            tile_ptr[n_tiles] = n_rows;
            op_ptr[n_tiles] = n_ops;
        }
        tile_u = 0;
        tile_k = 0;
        tile_e = 0;
    };
    for (int64_t i = 0; i < n_order; ++i) {
        const int64_t r = order[i];
        const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
        // operands of the row alone, and those not yet in the open tile
        int32_t own = 0, fresh = 0;
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t s = ent[2 * e], t = ent[2 * e + 1];
            if (s_trial[s] != i) {
                s_trial[s] = i;
                ++own;
                if (s_tile[s] != tile || tile < 0) ++fresh;
            }
            if (t_trial[t] != i) {
                t_trial[t] = i;
                ++own;
                if (t_tile[t] != tile || tile < 0) ++fresh;
            }
        }
        if (own > u_max || e1 - e0 > e_max) {  // too long for any tile
            ++n_untiled;
            continue;
        }
        if (tile < 0 || tile_k >= k_max || tile_u + fresh > u_max || tile_e + (e1 - e0) > e_max) {
            close_tile();
            tile = n_tiles;  // id of the tile being filled
        }
        // add the row
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t s = ent[2 * e], t = ent[2 * e + 1];
            if (s_tile[s] != tile) {
                s_tile[s] = tile;
                s_loc[s] = tile_u++;
                ops[n_ops++] = s;
            }
            if (t_tile[t] != tile) {
                t_tile[t] = tile;
                t_loc[t] = tile_u++;
                ops[n_ops++] = -1 - t;
            }
            ev[n_ev++] = (uint32_t)s_loc[s] | ((uint32_t)t_loc[t] << 16);
        }
        tile_e += e1 - e0;
        tile_rows[n_rows++] = r;
        ev_ptr[n_rows] = n_ev;
        ++tile_k;
    }
    close_tile();
    counts[0] = n_tiles;
    counts[1] = n_rows;
    counts[2] = n_ops;
    counts[3] = n_ev;
    counts[4] = n_untiled;
    return 0;
}
