// Host-side octree build for the defmm B200 path (C-ABI: include/defmm_b200.h).
//
// Restates tree.py:132-213: a cell with more than ncrit particles (and level
// below the depth cap) is split by a STABLE partition of its particle slice on
// the octant code 4*(x >= cx) + 2*(y >= cy) + (z >= cz), the centre being
// (lower + coords*beta) + 0.5*beta in FP64 (tree.py:165-166, geometry.py:71-72).
// Sons are created in octant order, empty octants skipped; the recursion is
// depth first, so cells come out in the reference's creation order.  Compiled
// with -ffp-contract=off so every comparison sees the reference's exact doubles.
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/defmm_b200.h"

struct defmm_tree {
    std::vector<int64_t> perm;
    std::vector<double> pts;
    std::vector<int32_t> level;
    std::vector<int64_t> coords, start, stop, parent;
};

namespace {

// Recursion depth is bounded by the depth cap (default 30), so plain recursion
// reproduces the reference's creation order directly.
struct Rec {
    defmm_tree* t;
    double lower[3];
    double side;
    int32_t ncrit, cap;
    std::vector<double> tmp_pts;
    std::vector<int64_t> tmp_perm;
    std::vector<uint8_t> oct;

    int64_t make(int32_t lev, int64_t c0, int64_t c1, int64_t c2, int64_t a, int64_t b, int64_t par) {
        t->level.push_back(lev);
        t->coords.push_back(c0);
        t->coords.push_back(c1);
        t->coords.push_back(c2);
        t->start.push_back(a);
        t->stop.push_back(b);
        t->parent.push_back(par);
        return (int64_t)t->level.size() - 1;
    }

    void split(int64_t c) {
        const int64_t a = t->start[c], b = t->stop[c];
        const int32_t lev = t->level[c];
        if (b - a <= ncrit || lev >= cap) return;
        const double beta = side / (double)(int64_t(1) << lev);
        double ctr[3];
        for (int k = 0; k < 3; ++k) {
            const double alpha = lower[k] + (double)t->coords[3 * c + k] * beta;
            ctr[k] = alpha + 0.5 * beta;
        }
        int64_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        double* p = t->pts.data();
        for (int64_t i = a; i < b; ++i) {
            const int o = ((p[3 * i] >= ctr[0]) ? 4 : 0) | ((p[3 * i + 1] >= ctr[1]) ? 2 : 0) |
                          ((p[3 * i + 2] >= ctr[2]) ? 1 : 0);
            oct[i] = (uint8_t)o;
            ++cnt[o];
        }
        int64_t off[9];
        off[0] = 0;
        for (int o = 0; o < 8; ++o) off[o + 1] = off[o] + cnt[o];
        int64_t pos[8];
        for (int o = 0; o < 8; ++o) pos[o] = off[o];
        for (int64_t i = a; i < b; ++i) {  // stable counting sort on the octant
            const int64_t d = pos[oct[i]]++;
            std::memcpy(&tmp_pts[3 * d], &p[3 * i], 3 * sizeof(double));
            tmp_perm[d] = t->perm[i];
        }
        std::memcpy(&p[3 * a], tmp_pts.data(), 3 * (b - a) * sizeof(double));
        std::memcpy(&t->perm[a], tmp_perm.data(), (b - a) * sizeof(int64_t));
        const int64_t c0 = t->coords[3 * c], c1 = t->coords[3 * c + 1], c2 = t->coords[3 * c + 2];
        for (int o = 0; o < 8; ++o) {
            if (cnt[o] == 0) continue;
            const int64_t s = make(lev + 1, 2 * c0 + ((o >> 2) & 1), 2 * c1 + ((o >> 1) & 1),
                                   2 * c2 + (o & 1), a + off[o], a + off[o + 1], c);
            split(s);
        }
    }
};

}  // namespace

extern "C" int defmm_tree_build(const double* pts, int64_t n, const double lower[3], double side,
                                int32_t ncrit, int32_t depth_cap, defmm_tree** out) {
    if (!pts || !out || n <= 0 || ncrit < 1 || depth_cap < 0 || !(side > 0)) return -1;
    defmm_tree* t = new (std::nothrow) defmm_tree();
    if (!t) return -2;
    try {
        t->perm.resize(n);
        for (int64_t i = 0; i < n; ++i) t->perm[i] = i;
        t->pts.assign(pts, pts + 3 * n);
        Rec r;
        r.t = t;
        for (int k = 0; k < 3; ++k) r.lower[k] = lower[k];
        r.side = side;
        r.ncrit = ncrit;
        r.cap = depth_cap;
        r.tmp_pts.resize(3 * n);
        r.tmp_perm.resize(n);
        r.oct.resize(n);
        const int64_t root = r.make(0, 0, 0, 0, 0, n, -1);
        r.split(root);
    } catch (...) {
        delete t;
        return -2;
    }
    *out = t;
    return 0;
}

extern "C" int64_t defmm_tree_ncells(const defmm_tree* t) { return t ? (int64_t)t->level.size() : -1; }

extern "C" int defmm_tree_fetch(const defmm_tree* t, int64_t* perm, double* sorted_pts, int32_t* level,
                                int64_t* coords, int64_t* start, int64_t* stop, int64_t* parent) {
    if (!t) return -1;
    const size_t n = t->perm.size(), m = t->level.size();
    if (perm) std::memcpy(perm, t->perm.data(), n * sizeof(int64_t));
    if (sorted_pts) std::memcpy(sorted_pts, t->pts.data(), 3 * n * sizeof(double));
    if (level) std::memcpy(level, t->level.data(), m * sizeof(int32_t));
    if (coords) std::memcpy(coords, t->coords.data(), 3 * m * sizeof(int64_t));
    if (start) std::memcpy(start, t->start.data(), m * sizeof(int64_t));
    if (stop) std::memcpy(stop, t->stop.data(), m * sizeof(int64_t));
    if (parent) std::memcpy(parent, t->parent.data(), m * sizeof(int64_t));
    return 0;
}

extern "C" void defmm_tree_free(defmm_tree* t) { delete t; }
