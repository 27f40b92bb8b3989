// Device-side plan construction: the octant path of
// every particle and the pair classification of the level-synchronous dual
// tree traversal.  Host orchestration (sorts, scans, compaction) lives in
// paper_2202_04894_b200/gpu_build.py on torch device tensors; these kernels
// hold the decisions that must be bit-identical to the reference:
//  * tree.py:165-166 / geometry.py:71-72: centre = (lower + coords * beta) +
//    0.5 * beta in FP64 with every product and sum rounded separately
//    (__dmul_rn / __dadd_rn, never fused), test p >= centre;
//  * traversal.py:100-113 as the integer gap^2 threshold per level, the
//    nearest-direction key from the dense per-level table (plan.py).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../include/defmm_b200.h"

namespace {

int report_pg(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

// keys[i] = the particle's octant path to depth D, 3 bits per level (level 0's
// octant in the highest bits): o = 4 (x >= cx) + 2 (y >= cy) + (z >= cz)
__global__ void __launch_bounds__(256) tree_keys_kernel(int64_t n, const double* __restrict__ pts, double lx,
                                                        double ly, double lz, double side, int depth,
                                                        int64_t* __restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    int64_t c0 = 0, c1 = 0, c2 = 0, key = 0;
    double beta = side;  // side / 2^level: exact halving
    for (int l = 0; l < depth; ++l) {
        const double h = __dmul_rn(0.5, beta);
        const double cx = __dadd_rn(__dadd_rn(lx, __dmul_rn((double)c0, beta)), h);
        const double cy = __dadd_rn(__dadd_rn(ly, __dmul_rn((double)c1, beta)), h);
        const double cz = __dadd_rn(__dadd_rn(lz, __dmul_rn((double)c2, beta)), h);
        const int b0 = x >= cx, b1 = y >= cy, b2 = z >= cz;
        c0 = 2 * c0 + b0;
        c1 = 2 * c1 + b1;
        c2 = 2 * c2 + b2;
        key = (key << 3) | (int64_t)(4 * b0 + 2 * b1 + b2);
        beta = h;
    }
    keys[i] = key;
}

// One candidate pair (t, s) of same-level cells: kind = 0 M2L (gap^2 >= g2min),
// 1 P2P (else, a leaf on either side), 2 expand (sons x sons).  For M2L pairs
// key = key_tab[tab_off + dense(t - s)] (level-local direction, -1 at LF levels
// when the table holds -1) and dense = the table index (the translation id);
// status is set to 1 when a translation falls outside [-R, R]^3.
__global__ void __launch_bounds__(256) dtt_classify_kernel(
    int64_t n, const int64_t* __restrict__ pt, const int64_t* __restrict__ ps, const int64_t* __restrict__ tco,
    const int64_t* __restrict__ sco, const int64_t* __restrict__ t_nsons, const int64_t* __restrict__ s_nsons,
    int64_t g2min, int32_t R, int64_t tab_off, const int32_t* __restrict__ key_tab, int8_t* __restrict__ kind,
    int32_t* __restrict__ key, int64_t* __restrict__ dense, int64_t* __restrict__ nexp, int32_t* status) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t t = pt[i], s = ps[i];
    int64_t d[3], g2 = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d[k] = tco[3 * t + k] - sco[3 * s + k];
        const int64_t a = (d[k] < 0 ? -d[k] : d[k]) - 1;  // cells apart along the axis
        if (a > 0) g2 += a * a;
    }
    int8_t kd;
    int32_t ky = -1;
    int64_t dn = -1, ne = 0;
    if (g2 >= g2min) {
        kd = 0;
        if (d[0] < -R || d[0] > R || d[1] < -R || d[1] > R || d[2] < -R || d[2] > R) {
            *status = 1;
        } else {
            const int64_t w = 2 * (int64_t)R + 1;
            dn = tab_off + ((d[0] + R) * w + (d[1] + R)) * w + (d[2] + R);
            ky = key_tab[dn];
        }
    } else if (t_nsons[t] == 0 || s_nsons[s] == 0) {
        kd = 1;
    } else {
        kd = 2;
        ne = t_nsons[t] * s_nsons[s];
    }
    kind[i] = kd;
    key[i] = ky;
    dense[i] = dn;
    nexp[i] = ne;
}

}  // namespace

extern "C" {

int defmm_tree_keys(int64_t n, const double* pts, const double lower[3], double side, int32_t depth,
                    int64_t* keys, void* stream) {
    if (n <= 0) return 0;
    if (depth < 0 || depth > 21) return -1;
    const int64_t blocks = (n + 255) / 256;
    if (blocks >= ((int64_t)1 << 31)) return -1;
    tree_keys_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, pts, lower[0], lower[1], lower[2], side,
                                                                        depth, keys);
    return report_pg(cudaGetLastError());
}

int defmm_dtt_classify(int64_t n, const int64_t* pair_t, const int64_t* pair_s, const int64_t* t_coords,
                       const int64_t* s_coords, const int64_t* t_nsons, const int64_t* s_nsons, int64_t g2min,
                       int32_t R, int64_t tab_off, const int32_t* key_tab, int8_t* kind, int32_t* key,
                       int64_t* dense, int64_t* nexp, int32_t* status, void* stream) {
    if (n <= 0) return 0;
    const int64_t blocks = (n + 255) / 256;
    if (blocks >= ((int64_t)1 << 31)) return -1;
    dtt_classify_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        n, pair_t, pair_s, t_coords, s_coords, t_nsons, s_nsons, g2min, R, tab_off, key_tab, kind, key, dense, nexp,
        status);
    return report_pg(cudaGetLastError());
}

}  // extern "C"
