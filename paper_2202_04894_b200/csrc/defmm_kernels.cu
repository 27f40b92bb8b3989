// B200 (sm_100a) kernels of the defmm FMM matvec, behind the C-ABI declared
// in include/defmm_b200.h.  Every operator is templated on the storage real
// type R (double -> "c128", float -> "c64") and on the interpolation order L.
//
// Design notes (DESIGN.md has the roofline of each kernel):
//  * every kernel owns its outputs -- one CTA or warp per output object
//    (expansion slot, M2L row, target leaf) -- so there are no atomics and
//    reruns are bitwise deterministic (test_traversal.py:224-231's contract);
//  * plane-wave modulations are applied in CELL-RELATIVE form
//    (e^{i kappa <xi - y, u>} factorised per axis), equal to the reference's
//    absolute-coordinate products (interpolation.py:104-137,
//    traversal.py:245-280, 362-391) in exact arithmetic and keeping every
//    phase small -- which is what makes the FP32 (c64) path accurate;
//  * the modulated M2M/L2L Kronecker factor C[k][j] = A[k][j] e^{i th (2x_k -
//    bit - x_j)} is split as diag(e^{i th 2x_k}) A diag(e^{-i th (bit+x_j)}):
//    real Lagrange factors (the reference's "t+s+r" strategy,
//    interpolation.py:194-200) between two diagonal phase scalings;
//  * the Fourier-domain M2L streams per-translation ("derived") symbols that
//    are materialised once per plan from the canonical ones through the
//    closed form of the cube-group frequency permutation (fourier.py:123-196).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "../../include/defmm_b200.h"

namespace {

thread_local char g_last_error[256] = "";

int report(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return 0;
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
    return (int)e;
}

// ---------------------------------------------------------------------------
// complex helpers (V = double2 | float2)

template <typename R>
struct Cx;
template <>
struct Cx<double> {
    using t = double2;
};
template <>
struct Cx<float> {
    using t = float2;
};
template <typename R>
using cx = typename Cx<R>::t;

template <typename V>
__device__ __forceinline__ V cz() {
    V v;
    v.x = 0;
    v.y = 0;
    return v;
}
template <typename V, typename S>
__device__ __forceinline__ V cmk(S re, S im) {
    V v;
    v.x = re;
    v.y = im;
    return v;
}
template <typename V>
__device__ __forceinline__ V cmul(V a, V b) {
    return cmk<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// c + a*b
template <typename V>
__device__ __forceinline__ V cfma(V a, V b, V c) {
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
    return c;
}
// c + s*a, s real
template <typename V, typename S>
__device__ __forceinline__ V crfma(S s, V a, V c) {
    c.x = fma(s, a.x, c.x);
    c.y = fma(s, a.y, c.y);
    return c;
}
template <typename V>
__device__ __forceinline__ V cadd(V a, V b) {
    return cmk<V>(a.x + b.x, a.y + b.y);
}
template <typename V, typename S>
__device__ __forceinline__ V cscale(V a, S s) {
    return cmk<V>(a.x * s, a.y * s);
}
template <typename V>
__device__ __forceinline__ V cconj(V a) {
    return cmk<V>(a.x, -a.y);
}
__device__ __forceinline__ double2 cexpi(double ph) {
    double s, c;
    sincos(ph, &s, &c);
    return make_double2(c, s);
}
__device__ __forceinline__ float2 cexpi(float ph) {
    float s, c;
    sincosf(ph, &s, &c);
    return make_float2(c, s);
}
__device__ __forceinline__ double2 to_d(double2 v) { return v; }
__device__ __forceinline__ double2 to_d(float2 v) { return make_double2(v.x, v.y); }
template <typename V>
__device__ __forceinline__ V from_d(double2 v);
template <>
__device__ __forceinline__ double2 from_d<double2>(double2 v) {
    return v;
}
template <>
__device__ __forceinline__ float2 from_d<float2>(double2 v) {
    return make_float2((float)v.x, (float)v.y);
}

// Equispaced nodes x_j = j/(L-1) (interpolation.py:51-56) and the Lagrange
// cardinal functions S_k(x) = prod_{j != k} (x - x_j)/(x_k - x_j) (:59-69).
template <int L, typename R>
__device__ __forceinline__ R node(int j) {
    return (R)j / (R)(L - 1);
}
// S_k(x) = w_k prod_{j != k} (x - x_j) with the barycentric weights
// w_k = 1 / prod_{j != k} (x_k - x_j) = (L-1)^(L-1) (-1)^(L-1-k) / (k! (L-1-k)!)
// as compile-time constants and the products shared through prefix / suffix
// products: 4 L multiplications per evaluation.  (The reference's form divides
// L (L-1) times per evaluation, interpolation.py:59-69 -- a third of the P2M and
// L2P instructions were those divisions; the values agree to rounding.)
template <int L>
struct LagrangeWeights {
    double w[L];
    constexpr LagrangeWeights() : w{} {
        for (int k = 0; k < L; ++k) {
            double num = 1.0, den = 1.0;
            for (int j = 0; j < L - 1; ++j) num *= (double)(L - 1);
            for (int j = 0; j < L; ++j)
                if (j != k) den *= (double)(k - j);
            w[k] = num / den;
        }
    }
};
template <int L, typename R>
__device__ __forceinline__ void lagrange(R x, R* S) {
    constexpr LagrangeWeights<L> lw{};
    R dl[L], suf[L];
#pragma unroll
    for (int j = 0; j < L; ++j) dl[j] = x - node<L, R>(j);
    suf[L - 1] = (R)1;
#pragma unroll
    for (int k = L - 2; k >= 0; --k) suf[k] = suf[k + 1] * dl[k + 1];
    R pre = (R)1;
#pragma unroll
    for (int k = 0; k < L; ++k) {
        S[k] = pre * suf[k] * (R)lw.w[k];
        pre = pre * dl[k];
    }
}

template <int L>
__host__ __device__ constexpr int cube() { return L * L * L; }
template <int L>
__host__ __device__ constexpr int pad() { return 2 * L - 1; }
template <int L>
__host__ __device__ constexpr int per_lane() { return (cube<L>() + 31) / 32; }
// stride (in complex entries) of one P^3 spectrum in HBM: padded to an even
// count for complex64 so two entries form one aligned 16-B vector load
template <typename R, int L>
__host__ __device__ constexpr int spec_stride() {
    return sizeof(R) == 4 ? (pad<L>() * pad<L>() * pad<L>() + 1) / 2 * 2 : pad<L>() * pad<L>() * pad<L>();
}

// M2M/L2L factor tables A_bit[k][j] = S_k((bit + x_j)/2), bit in {0,1}
// (interpolation.py:140-148), computed once per CTA in shared memory.
template <int L, typename R>
__device__ __forceinline__ void make_factor_tables(R* A) {
    for (int t = threadIdx.x; t < 2 * L * L; t += blockDim.x) {
        const int bit = t / (L * L), k = (t / L) % L, j = t % L;
        const double x = ((double)bit + node<L, double>(j)) / 2.0;
        double v = 1.0;  // S_k(x), evaluated directly (no runtime-indexed local array)
        for (int m = 0; m < L; ++m)
            if (m != k) v = v * (x - node<L, double>(m)) / (node<L, double>(k) - node<L, double>(m));
        A[t] = (R)v;
    }
}

// tw[k] = e^{-2 pi i k / P}
template <int P, typename V>
__device__ __forceinline__ void make_twiddles(V* tw) {
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)k / (double)P, &s, &c);
        tw[k] = from_d<V>(make_double2(c, -s));
    }
}

// twm[f * L + x] = e^{-2 pi i (f x mod P) / P}, f < P, x < L: the pruned DFT
// factors, so the inner loops index without a modulo (M2F was ALU-bound on it)
// e^{-2 pi i k / P} for every P = 2L-1 (L = 2..8), filled once by the
// launchers (cudaMemcpyToSymbol); kernels build their P x L matrix from it
__constant__ double2 c_tw[8][15];
__constant__ float2 c_twf[8][15];  // the same, rounded to float (complex64 M2F v2)
// A_0[k][j] = S_k(x_j / 2) of every order (row L-1, entry k L + j), filled with
// c_tw; A_1 is its mirror image, A_1[k][j] = A_0[L-1-k][L-1-j] (the nodes are
// symmetric about 1/2), so the fiber kernels below need this table only
__constant__ double c_a0[8][64];
__constant__ float c_a0f[8][64];

// ---------------------------------------------------------------------------
// Spectral layout.  Every P^3 spectrum (multipole spectra, symbols, local
// accumulators) is stored in ORBIT ORDER: the natural frequency indices
// j = f0 P^2 + f1 P + f2 grouped by their orbit under the 48-element cube group
// acting on (f0, f1, f2) mod P (fourier.py:90-101 / rotated_index below), the
// orbits packed first-fit-decreasing into SLICES of <= SLICE_W positions (each
// slice closed under every rotation).  g_forder[L-1][pos] =
// natural index at a position, g_finv the inverse.  All orbits but the zero
// frequency have even size and the zero orbit sits in the last slice, so
// every other slice starts at an even position (16-B vector loads for c64).
// The Hadamard product is
// order-agnostic, the kernels that touch natural indices (M2F, symbols, F2L,
// rotations) go through these tables.
constexpr int SLICE_W = 128;  // positions per slice: 4 per lane
constexpr int MAX_SLICES = 40;
constexpr int MAX_P3 = 15 * 15 * 15;
__device__ int16_t g_forder[8][MAX_P3];
__device__ int16_t g_finv[8][MAX_P3];

template <int L>
__device__ __forceinline__ int forder(int pos) {
    return g_forder[L - 1][pos];
}
template <int L>
__device__ __forceinline__ int finv(int j) {
    return g_finv[L - 1][j];
}

template <int L, typename V>
__device__ __forceinline__ void make_twiddle_matrix(V* twm) {
    constexpr int P = 2 * L - 1;
    for (int t = threadIdx.x; t < P * L; t += blockDim.x) {
        const int f = t / L, x = t - (t / L) * L;
        twm[t] = from_d<V>(c_tw[L - 1][(f * x) % P]);
    }
}

// ---------------------------------------------------------------------------
// K2: P2M.  One CTA per (leaf, key).  Per particle and axis the modulated 1D
// weights W_a = S_a(xh) e^{i kappa beta u (x_a - xh)} are staged in shared
// memory; the L^3 output entries are tensor sums over the particles.

// threads per CTA: the L^3 entries, at most 128 -- at L <= 4 a 64-thread CTA
// leaves no lane idle in the entry loop and doubles the leaves in flight per SM
// (the kernel is bound by the latency of its dependent cell / particle loads)
template <int L>
__host__ __device__ constexpr int p2m_threads() {
    return cube<L>() <= 64 ? 64 : 128;
}

template <typename R, int L>
__global__ void __launch_bounds__(p2m_threads<L>()) p2m_kernel(
    int64_t n, const int32_t* __restrict__ cell, const int32_t* __restrict__ dir,
    const int64_t* __restrict__ out_slot, const int64_t* __restrict__ cstart,
    const int64_t* __restrict__ cstop, const double* __restrict__ calpha,
    const int32_t* __restrict__ clevel, const double* __restrict__ lbeta,
    const double* __restrict__ dirs, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, const cx<R>* __restrict__ q, double kappa, cx<R>* __restrict__ mult) {
    using V = cx<R>;
    constexpr int L3 = cube<L>();
    constexpr int NT = p2m_threads<L>();
    constexpr int PER = (L3 + NT - 1) / NT;
    constexpr int CH = 32;
    __shared__ V W[3][CH][L];
    const int64_t i = blockIdx.x;
    const int c = cell[i];
    const int d = dir[i];
    const double beta = lbeta[clevel[c]];
    const double ibeta = 1.0 / beta;  // one division per CTA, not one per particle and axis
    double al[3];
    R ku[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        al[k] = calpha[3 * c + k];
        ku[k] = (R)(d >= 0 ? kappa * beta * dirs[3 * d + k] : 0.0);
    }
    const int64_t s0 = cstart[c], s1 = cstop[c];
    // e^{i ku (x_k - xh)} = e^{i ku x_k} e^{-i ku xh}: the node factors once per
    // CTA, one sincos per particle and axis (HF keys only; LF: ku = 0)
    __shared__ V T[3][L];
    if (threadIdx.x < 3 * L) {
        const int ax = threadIdx.x / L, k = threadIdx.x % L;
        T[ax][k] = d >= 0 ? cexpi(ku[ax] * node<L, R>(k)) : cmk<V>((R)1, (R)0);
    }
    V acc[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) acc[m] = cz<V>();
    for (int64_t base = s0; base < s1; base += CH) {
        const int cnt = (int)((s1 - base) < CH ? (s1 - base) : CH);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * 3; t += NT) {
            const int p = t / 3, ax = t - 3 * (t / 3);
            const double* pp = ax == 0 ? px : (ax == 1 ? py : pz);
            const R xh = (R)((pp[base + p] - al[ax]) * ibeta);
            R S[L];
            lagrange<L, R>(xh, S);
            V qq = ax == 0 ? q[base + p] : cmk<V>((R)1, (R)0);
            if (d >= 0) qq = cmul(qq, cexpi(-ku[ax] * xh));
#pragma unroll
            for (int k = 0; k < L; ++k) W[ax][p][k] = cmul(qq, cscale(T[ax][k], S[k]));
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int r = threadIdx.x + m * NT;
            if (r < L3) {
                const int a = r / (L * L), b = (r / L) % L, cc = r % L;
                V s = acc[m];
                for (int p = 0; p < cnt; ++p) s = cfma(cmul(W[0][p][a], W[1][p][b]), W[2][p][cc], s);
                acc[m] = s;
            }
        }
    }
    const int64_t o = out_slot[i] * L3;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int r = threadIdx.x + m * NT;
        if (r < L3) mult[o + r] = acc[m];
    }
}

// ---------------------------------------------------------------------------
// K4/K5: M2M and L2L, one WARP per output slot (8 warps per CTA), the three
// real mode products in per-warp shared memory with __syncwarp only.

constexpr int NODAL_WARPS = 8;
#ifndef DEFMM_NODAL_MINB
#define DEFMM_NODAL_MINB 4  // <= 64 registers: 4 CTAs/SM (L5: M2M -12..-32%, L2L -13..-29%)
#endif

// One mode product along `axis` of an L^3 tile (C order) with the real factor
// A_bit: TRANSPOSE=false -> out k, in j, coefficient A[bit][k][j] (M2M);
// TRANSPOSE=true -> out j, in k, coefficient A[bit][k][j] (L2L).
template <int L, typename R, bool TRANSPOSE>
__device__ __forceinline__ cx<R> mode_product(const R* A, int bit, int axis, const cx<R>* x, int r) {
    using V = cx<R>;
    const int i0 = r / (L * L), i1 = (r / L) % L, i2 = r % L;
    const int o = axis == 0 ? i0 : (axis == 1 ? i1 : i2);
    const int stride = axis == 0 ? L * L : (axis == 1 ? L : 1);
    const int base = r - o * stride;
    const R* Ab = A + bit * L * L;
    V v = cz<V>();
#pragma unroll
    for (int t = 0; t < L; ++t) {
        const R a = TRANSPOSE ? Ab[t * L + o] : Ab[o * L + t];
        v = crfma(a, x[base + t * stride], v);
    }
    return v;
}

// the nodal buffers of one warp: 2 L^3 complex + 9 L complex of separable
// plane-wave phase tables (dynamic shared memory), then the factor tables
template <typename R, int L>
__host__ __device__ constexpr int nodal_smem_bytes() {
    return NODAL_WARPS * (2 * cube<L>() + 9 * L) * (int)sizeof(cx<R>) + 2 * L * L * (int)sizeof(R);
}

template <typename R, int L>
__global__ void __launch_bounds__(32 * NODAL_WARPS, DEFMM_NODAL_MINB) m2m_kernel(
    int64_t n, const int64_t* __restrict__ out_slot, const int32_t* __restrict__ dir,
    const int64_t* __restrict__ son_slot, double son_beta, const double* __restrict__ dirs, double kappa,
    cx<R>* __restrict__ mult) {
    using V = cx<R>;
    constexpr int L3 = cube<L>(), E = per_lane<L>();
    extern __shared__ unsigned char smraw[];
    V* bufs = reinterpret_cast<V*>(smraw);
    V* tabs = bufs + NODAL_WARPS * 2 * L3;
    R* A = reinterpret_cast<R*>(tabs + NODAL_WARPS * 9 * L);
    make_factor_tables<L, R>(A);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * NODAL_WARPS + w;
    if (i >= n) return;
    const int d = dir[i];
    R ku[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ku[k] = (R)(d >= 0 ? kappa * son_beta * dirs[3 * d + k] : 0.0);
    V* X = bufs + w * 2 * L3;
    V* T = X + L3;
    // separable phases (HF keys): son side Q[ax][bit][j] = e^{-i ku_ax (bit + x_j)},
    // father side F[ax][k] = e^{i 2 ku_ax x_k} -- 9 L sincos per slot instead of
    // 9 L^3 (one per element and son)
    V* Q = tabs + w * 9 * L;
    V* F = Q + 6 * L;
    if (d >= 0) {
        for (int t = lane; t < 9 * L; t += 32) {
            if (t < 6 * L) {
                const int ax = t / (2 * L), bit = (t / L) & 1, j = t % L;
                Q[t] = cexpi(-ku[ax] * ((R)bit + node<L, R>(j)));
            } else {
                const int ax = (t - 6 * L) / L, k = t % L;
                F[ax * L + k] = cexpi(2 * ku[ax] * node<L, R>(k));
            }
        }
    }
    V acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = cz<V>();
    // runtime son loop (measured faster than unrolling the octants or
    // prefetching all son expansions: code size / registers)
    for (int o = 0; o < 8; ++o) {
        const int64_t ss = son_slot[8 * i + o];
        if (ss < 0) continue;  // warp-uniform
        const int b0 = (o >> 2) & 1, b1 = (o >> 1) & 1, b2 = o & 1;
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) {
                const int j0 = r / (L * L), j1 = (r / L) % L, j2 = r % L;
                const V m = mult[ss * L3 + r];
                // son-side phase e^{-i th (bit + x_j)} (conj plane wave on the son grid)
                X[r] = d >= 0 ? cmul(cmul(m, Q[(0 + b0) * L + j0]), cmul(Q[(2 + b1) * L + j1], Q[(4 + b2) * L + j2]))
                              : m;
            }
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) T[r] = mode_product<L, R, false>(A, b0, 0, X, r);
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) X[r] = mode_product<L, R, false>(A, b1, 1, T, r);
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) acc[e] = cadd(acc[e], mode_product<L, R, false>(A, b2, 2, X, r));
        }
    }
    const int64_t ob = out_slot[i] * L3;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        if (r < L3) {
            const int k0 = r / (L * L), k1 = (r / L) % L, k2 = r % L;
            // father-side phase e^{i th 2 x_k}
            mult[ob + r] = d >= 0 ? cmul(cmul(acc[e], F[k0]), cmul(F[L + k1], F[2 * L + k2])) : acc[e];
        }
    }
}

// K4/K5 v2: the mode products with one FIBER per lane.  A lane loads the L
// entries of its fiber once, forms the L outputs with the interpolation factors
// as constant-bank operands (c_a0) and writes them back in place: L loads +
// L stores per 2 L^2 FFMA instead of two shared loads per FFMA pair (v1 issues
// as many LDS as FFMA).  The bit-1 factor matrix is the mirror image of the
// bit-0 one, so a lane whose son sits in the upper half walks its fiber
// backwards with the same constants -- which lets the lanes of one warp work on
// the tiles of TWO sons at once (2 L^2 fibers per pass: all 32 lanes at L = 4).
template <int L, typename R>
__device__ __forceinline__ R a0c(int k, int j) {
    if constexpr (sizeof(R) == 4) {
        return c_a0f[L - 1][k * L + j];
    } else {
        return c_a0[L - 1][k * L + j];
    }
}

// Position of entry r = (i0, i1, i2) in a v2 tile.  At L = 4 the 16-entry planes
// of the 64-entry tile alias in shared memory (4-way bank conflicts of the fiber
// accesses along two of the three axes), so the tile is XOR-swizzled:
// (i0, i1, i2) -> 16 i0 + 4 (i1 ^ i0) + (i2 ^ i0) = r ^ 5 (r >> 4); every fiber
// access of 16 lanes then touches 16 different 8-byte banks.
template <int L>
__device__ __forceinline__ int tile_pos(int r) {
    if constexpr (L == 4) {
        return r ^ (5 * (r >> 4));
    } else {
        return r;
    }
}

// in-place product of fiber f (of L^2) of an L^3 tile along AXIS with A_bit
// (TRANSPOSE=false: out k, in j, A[k][j], M2M) or its transpose (L2L)
template <int L, typename R, bool TRANSPOSE, int AXIS>
__device__ __forceinline__ void fiber_product(cx<R>* tile, int f, int bit) {
    using V = cx<R>;
    V x[L];
    if constexpr (L == 4) {
        // swizzled tile: entry t of the (mirrored) fiber sits at (C t) ^ lb -- the
        // fields of the index are 2-bit wide, so the mirror t -> 3 - t = t ^ 3 and
        // the swizzle commute with the multiplication by C
        constexpr int C = AXIS == 0 ? 21 : (AXIS == 1 ? 4 : 1);
        const int hi = f >> 2, lo = f & 3, m = bit ? 3 : 0;
        const int lb = AXIS == 0 ? (f ^ (21 * m))
                                 : (AXIS == 1 ? ((4 * m) ^ (20 * hi + (lo ^ hi)))
                                              : (m ^ (16 * hi + 4 * (lo ^ hi) + hi)));
#pragma unroll
        for (int j = 0; j < L; ++j) x[j] = tile[(C * j) ^ lb];
#pragma unroll
        for (int k = 0; k < L; ++k) {
            V v = cz<V>();
#pragma unroll
            for (int j = 0; j < L; ++j) v = crfma(TRANSPOSE ? a0c<L, R>(j, k) : a0c<L, R>(k, j), x[j], v);
            tile[(C * k) ^ lb] = v;
        }
    } else {
        constexpr int stride = AXIS == 0 ? L * L : (AXIS == 1 ? L : 1);
        const int base = AXIS == 0 ? f : (AXIS == 1 ? (f / L) * (L * L) + f % L : f * L);
        V* p = tile + base + (bit ? (L - 1) * stride : 0);
        const int sg = bit ? -stride : stride;
#pragma unroll
        for (int j = 0; j < L; ++j) x[j] = p[j * sg];
#pragma unroll
        for (int k = 0; k < L; ++k) {
            V v = cz<V>();
#pragma unroll
            for (int j = 0; j < L; ++j) v = crfma(TRANSPOSE ? a0c<L, R>(j, k) : a0c<L, R>(k, j), x[j], v);
            p[k * sg] = v;
        }
    }
}

// the three products of the (up to) two tiles at `tiles`, `tiles + L^3`; oa, ob
// = octants of the tiles' sons (ob < 0: one tile)
template <int L, typename R, bool TRANSPOSE>
__device__ __forceinline__ void fiber_products(cx<R>* tiles, int oa, int ob, int lane) {
    constexpr int L2 = L * L, L3 = L * L * L, NP = (2 * L2 + 31) / 32;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int id = p * 32 + lane, t = id >= L2;
        if (id < 2 * L2 && (!t || ob >= 0))
            fiber_product<L, R, TRANSPOSE, 0>(tiles + t * L3, id - t * L2, ((t ? ob : oa) >> 2) & 1);
    }
    __syncwarp();
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int id = p * 32 + lane, t = id >= L2;
        if (id < 2 * L2 && (!t || ob >= 0))
            fiber_product<L, R, TRANSPOSE, 1>(tiles + t * L3, id - t * L2, ((t ? ob : oa) >> 1) & 1);
    }
    __syncwarp();
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int id = p * 32 + lane, t = id >= L2;
        if (id < 2 * L2 && (!t || ob >= 0))
            fiber_product<L, R, TRANSPOSE, 2>(tiles + t * L3, id - t * L2, (t ? ob : oa) & 1);
    }
    __syncwarp();
}

template <typename R, int L>
__host__ __device__ constexpr int nodal2_smem_bytes() {
    return NODAL_WARPS * (2 * cube<L>() + 9 * L) * (int)sizeof(cx<R>);
}
// a fiber (L entries) and the per-lane accumulators (L^3 / 32 entries) live in
// registers: the 64-register cap of DEFMM_NODAL_MINB spills from L = 6 (L = 5 in FP64)
template <typename R, int L>
__host__ __device__ constexpr int nodal2_minb() {
    return (sizeof(R) == 4 ? L <= 5 : L <= 4) ? DEFMM_NODAL_MINB : ((sizeof(R) == 8 && L >= 7) ? 1 : 2);
}

template <typename R, int L>
__global__ void __launch_bounds__(32 * NODAL_WARPS, nodal2_minb<R, L>()) m2m_fiber_kernel(
    int64_t n, const int64_t* __restrict__ out_slot, const int32_t* __restrict__ dir,
    const int64_t* __restrict__ son_slot, double son_beta, const double* __restrict__ dirs, double kappa,
    cx<R>* __restrict__ mult) {
    using V = cx<R>;
    constexpr int L3 = cube<L>(), E = per_lane<L>();
    extern __shared__ unsigned char smraw[];
    V* bufs = reinterpret_cast<V*>(smraw);
    V* tabs = bufs + NODAL_WARPS * 2 * L3;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * NODAL_WARPS + w;
    if (i >= n) return;
    const int d = dir[i];
    R ku[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ku[k] = (R)(d >= 0 ? kappa * son_beta * dirs[3 * d + k] : 0.0);
    V* X = bufs + w * 2 * L3;  // the tiles of two sons
    V* Q = tabs + w * 9 * L;   // separable phases, as in m2m_kernel
    V* F = Q + 6 * L;
    if (d >= 0) {
        for (int t = lane; t < 9 * L; t += 32) {
            if (t < 6 * L) {
                const int ax = t / (2 * L), bit = (t / L) & 1, j = t % L;
                Q[t] = cexpi(-ku[ax] * ((R)bit + node<L, R>(j)));
            } else {
                const int ax = (t - 6 * L) / L, k = t % L;
                F[ax * L + k] = cexpi(2 * ku[ax] * node<L, R>(k));
            }
        }
    }
    V acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = cz<V>();
    int oa = -1;
    int64_t sa = 0;
    for (int o = 0; o <= 8; ++o) {  // present sons, two at a time (o == 8: an unpaired last one)
        const int64_t sb = o < 8 ? son_slot[8 * i + o] : -1;
        if (o < 8 && sb < 0) continue;  // warp-uniform
        if (o < 8 && oa < 0) {
            oa = o;
            sa = sb;
            continue;
        }
        if (oa < 0) break;
        const int ob = o < 8 ? o : -1;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (t == 1 && ob < 0) break;
            const int os = t ? ob : oa;
            const int64_t ss = t ? sb : sa;
            const int b0 = (os >> 2) & 1, b1 = (os >> 1) & 1, b2 = os & 1;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int r = lane + 32 * e;
                if (r < L3) {
                    const int j0 = r / (L * L), j1 = (r / L) % L, j2 = r % L;
                    const V m = mult[ss * L3 + r];
                    X[t * L3 + tile_pos<L>(r)] = d >= 0 ? cmul(cmul(m, Q[(0 + b0) * L + j0]),
                                                               cmul(Q[(2 + b1) * L + j1], Q[(4 + b2) * L + j2]))
                                                        : m;
                }
            }
        }
        __syncwarp();
        fiber_products<L, R, false>(X, oa, ob, lane);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) {
                acc[e] = cadd(acc[e], X[tile_pos<L>(r)]);
                if (ob >= 0) acc[e] = cadd(acc[e], X[L3 + tile_pos<L>(r)]);
            }
        }
        oa = -1;
    }
    const int64_t obase = out_slot[i] * L3;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        if (r < L3) {
            const int k0 = r / (L * L), k1 = (r / L) % L, k2 = r % L;
            mult[obase + r] = d >= 0 ? cmul(cmul(acc[e], F[k0]), cmul(F[L + k1], F[2 * L + k2])) : acc[e];
        }
    }
}

template <typename R, int L>
__global__ void __launch_bounds__(32 * NODAL_WARPS, DEFMM_NODAL_MINB) l2l_kernel(
    int64_t n, const int64_t* __restrict__ out_slot, const int8_t* __restrict__ octant,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_slot,
    const int32_t* __restrict__ src_dir, double son_beta, const double* __restrict__ dirs, double kappa,
    cx<R>* __restrict__ local) {
    using V = cx<R>;
    constexpr int L3 = cube<L>(), E = per_lane<L>();
    extern __shared__ unsigned char smraw[];
    V* bufs = reinterpret_cast<V*>(smraw);
    V* tabs = bufs + NODAL_WARPS * 2 * L3;
    R* A = reinterpret_cast<R*>(tabs + NODAL_WARPS * 9 * L);
    make_factor_tables<L, R>(A);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * NODAL_WARPS + w;
    if (i >= n) return;
    // separable phases per source (HF keys): father side G[ax][k] =
    // e^{-i 2 ku_ax x_k}, son side H[ax][j] = e^{i ku_ax (bit_ax + x_j)}
    V* G = tabs + w * 9 * L;
    V* H = G + 3 * L;
    const int o = octant[i];
    const int b0 = (o >> 2) & 1, b1 = (o >> 1) & 1, b2 = o & 1;
    V* X = bufs + w * 2 * L3;
    V* T = X + L3;
    const int64_t ob = out_slot[i] * L3;
    V acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        acc[e] = r < L3 ? local[ob + r] : cz<V>();
    }
    const int64_t s0 = ptr[i], s1 = ptr[i + 1];
    V nxt[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        nxt[e] = (s0 < s1 && r < L3) ? local[src_slot[s0] * L3 + r] : cz<V>();
    }
    for (int64_t s = s0; s < s1; ++s) {
        const int d = src_dir[s];
        V cur[E];
#pragma unroll
        for (int e = 0; e < E; ++e) cur[e] = nxt[e];
        if (s + 1 < s1) {  // next source in flight during this one's transform
            const int64_t nb = src_slot[s + 1] * L3;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int r = lane + 32 * e;
                if (r < L3) nxt[e] = local[nb + r];
            }
        }
        R ku[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) ku[k] = (R)(d >= 0 ? kappa * son_beta * dirs[3 * d + k] : 0.0);
        __syncwarp();
        if (d >= 0) {
            for (int t = lane; t < 6 * L; t += 32) {
                const int ax = (t % (3 * L)) / L, k = t % L;
                const int bit = ax == 0 ? b0 : (ax == 1 ? b1 : b2);
                if (t < 3 * L) G[t] = cexpi(-2 * ku[ax] * node<L, R>(k));
                else H[t - 3 * L] = cexpi(ku[ax] * ((R)bit + node<L, R>(k)));
            }
            __syncwarp();
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) {
                const int k0 = r / (L * L), k1 = (r / L) % L, k2 = r % L;
                // father-side phase e^{-i th 2 x_k} (conj plane wave on the father grid)
                X[r] = d >= 0 ? cmul(cmul(cur[e], G[k0]), cmul(G[L + k1], G[2 * L + k2])) : cur[e];
            }
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) T[r] = mode_product<L, R, true>(A, b0, 0, X, r);
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) X[r] = mode_product<L, R, true>(A, b1, 1, T, r);
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) {
                const V y = mode_product<L, R, true>(A, b2, 2, X, r);
                const int j0 = r / (L * L), j1 = (r / L) % L, j2 = r % L;
                // son-side phase e^{i th (bit + x_j)}
                acc[e] = cadd(acc[e], d >= 0 ? cmul(cmul(y, H[j0]), cmul(H[L + j1], H[2 * L + j2])) : y);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        if (r < L3) local[ob + r] = acc[e];
    }
}

// K5 v2: L2L with fiber mode products (see m2m_fiber_kernel): the father locals
// of TWO sources of the output slot are transformed at once (one tile each; they
// share the son's octant), each with its own separable phase tables.
template <typename R, int L>
__host__ __device__ constexpr int l2l2_smem_bytes() {
    return NODAL_WARPS * (2 * cube<L>() + 12 * L) * (int)sizeof(cx<R>);
}
// every (type, order) runs the v2 kernels; FP64 at L >= 7 (2 x 16 accumulators and
// a fiber per lane) with one CTA per SM and the full register budget (nodal2_minb):
// cfg5 L8 downward pass 8.2 -> 5.3 ms against v1
template <typename R, int L>
__host__ __device__ constexpr bool nodal2_ok() {
    return true;
}

template <typename R, int L>
__global__ void __launch_bounds__(32 * NODAL_WARPS, nodal2_minb<R, L>()) l2l_fiber_kernel(
    int64_t n, const int64_t* __restrict__ out_slot, const int8_t* __restrict__ octant,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_slot,
    const int32_t* __restrict__ src_dir, double son_beta, const double* __restrict__ dirs, double kappa,
    cx<R>* __restrict__ local) {
    using V = cx<R>;
    constexpr int L3 = cube<L>(), E = per_lane<L>();
    extern __shared__ unsigned char smraw[];
    V* bufs = reinterpret_cast<V*>(smraw);
    V* tabs = bufs + NODAL_WARPS * 2 * L3;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * NODAL_WARPS + w;
    if (i >= n) return;
    // per tile t: father side G_t[ax][k] = e^{-i 2 ku_ax x_k}, son side
    // H_t[ax][j] = e^{i ku_ax (bit_ax + x_j)} at tabs + t 6L (+ 3L)
    V* GH = tabs + w * 12 * L;
    const int o = octant[i];
    const int b0 = (o >> 2) & 1, b1 = (o >> 1) & 1, b2 = o & 1;
    V* X = bufs + w * 2 * L3;
    const int64_t ob = out_slot[i] * L3;
    V acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        acc[e] = r < L3 ? local[ob + r] : cz<V>();
    }
    const int64_t s0 = ptr[i], s1 = ptr[i + 1];
    for (int64_t s = s0; s < s1; s += 2) {
        const bool two = s + 1 < s1;  // warp-uniform
        const int dA = src_dir[s], dB = two ? src_dir[s + 1] : -1;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int d = t ? dB : dA;
            if (d < 0) continue;
            R ku[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) ku[k] = (R)(kappa * son_beta * dirs[3 * d + k]);
            for (int q = lane; q < 6 * L; q += 32) {
                const int ax = (q % (3 * L)) / L, k = q % L;
                const int bit = ax == 0 ? b0 : (ax == 1 ? b1 : b2);
                GH[t * 6 * L + q] = q < 3 * L ? cexpi(-2 * ku[ax] * node<L, R>(k))
                                              : cexpi(ku[ax] * ((R)bit + node<L, R>(k)));
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (t == 1 && !two) break;
            const int d = t ? dB : dA;
            const int64_t sb = src_slot[s + t] * L3;
            const V* G = GH + t * 6 * L;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int r = lane + 32 * e;
                if (r < L3) {
                    const int k0 = r / (L * L), k1 = (r / L) % L, k2 = r % L;
                    const V c = local[sb + r];
                    // father-side phase e^{-i th 2 x_k} (conj plane wave on the father grid)
                    X[t * L3 + tile_pos<L>(r)] = d >= 0 ? cmul(cmul(c, G[k0]), cmul(G[L + k1], G[2 * L + k2])) : c;
                }
            }
        }
        __syncwarp();
        fiber_products<L, R, true>(X, o, two ? o : -1, lane);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (t == 1 && !two) break;
            const int d = t ? dB : dA;
            const V* H = GH + t * 6 * L + 3 * L;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int r = lane + 32 * e;
                if (r < L3) {
                    const V y = X[t * L3 + tile_pos<L>(r)];
                    const int j0 = r / (L * L), j1 = (r / L) % L, j2 = r % L;
                    // son-side phase e^{i th (bit + x_j)}
                    acc[e] = cadd(acc[e], d >= 0 ? cmul(cmul(y, H[j0]), cmul(H[L + j1], H[2 * L + j2])) : y);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int r = lane + 32 * e;
        if (r < L3) local[ob + r] = acc[e];
    }
}

// ---------------------------------------------------------------------------
// K6 M2F: L^3 corner of a zero P^3 grid -> unitary forward DFT
// (fourier.py:67-72), pruned per axis; one WARP per expansion.

constexpr int M2F_WARPS = 4;

template <typename R, int L>
__global__ void __launch_bounds__(32 * M2F_WARPS) m2f_kernel(int64_t n, const int64_t* __restrict__ src_slot,
                                                             const cx<R>* __restrict__ mult,
                                                             cx<R>* __restrict__ hat) {
    using V = cx<R>;
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int WS = L3 + L * L * P + L * P * P;
    extern __shared__ unsigned char smraw[];
    V* tw = reinterpret_cast<V*>(smraw);  // twiddle matrix P x L
    make_twiddle_matrix<L, V>(tw);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * M2F_WARPS + w;
    if (i >= n) return;
    V* X = tw + P * L + w * WS;  // L^3
    V* Y1 = X + L3;          // [a][b][f2]
    V* Y2 = Y1 + L * L * P;  // [a][f1][f2]
    const int64_t s = src_slot[i] * L3;
    for (int r = lane; r < L3; r += 32) X[r] = mult[s + r];
    __syncwarp();
    for (int t = lane; t < L * L * P; t += 32) {
        const int ab = t / P, f2 = t % P;
        V v = cz<V>();
#pragma unroll
        for (int c = 0; c < L; ++c) v = cfma(X[ab * L + c], tw[f2 * L + c], v);
        Y1[t] = v;
    }
    __syncwarp();
    for (int t = lane; t < L * P * P; t += 32) {
        const int a = t / (P * P), f1 = (t / P) % P, f2 = t % P;
        V v = cz<V>();
#pragma unroll
        for (int b = 0; b < L; ++b) v = cfma(Y1[(a * L + b) * P + f2], tw[f1 * L + b], v);
        Y2[t] = v;
    }
    __syncwarp();
    const R scale = (R)(1.0 / (P * sqrt((double)P)));
    constexpr int SS = spec_stride<R, L>();
    V* out = hat + i * (int64_t)SS;
    for (int t = lane; t < SS; t += 32) {
        V v = cz<V>();
        if (t < P3) {
            const int j = forder<L>(t);  // orbit-ordered position -> natural frequency
            const int f0 = j / (P * P), f12 = j % (P * P);
#pragma unroll
            for (int a = 0; a < L; ++a) v = cfma(Y2[a * P * P + f12], tw[f0 * L + a], v);
        }
        out[t] = cscale(v, scale);  // the pad entry (c64) is written as 0
    }
}

// K6 v2 M2F (small orders): the same pruned transform with one 1D DFT ROW per
// lane -- a lane loads its row's L inputs once and produces its P outputs with
// the twiddles as compile-time constant-bank operands (c_tw), instead of one
// output per lane re-reading L inputs and L twiddles from shared memory (v1 was
// L1/shared-throughput bound at 94%, 25% of the HBM roofline, r01_summary_v6).
// The natural-order spectrum is assembled in shared memory and written out
// coalesced in orbit order.
// When the P^3 staging buffer would take a warp past 12 KB of shared memory
// (c64 L >= 6, c128 L >= 5) the last stage writes the spectrum straight to
// global memory in orbit order (scattered within the expansion's own
// spectrum) instead: twice the warps per SM, shared memory being the
// occupancy limit (c128 L5 1946 -> 1327 us, c64 L6 717 -> 666 us; c64 L5 is
// faster staged: 897 vs 992 us)
template <typename R, int L>
__host__ __device__ constexpr bool m2f2_direct() {
    constexpr int P = 2 * L - 1;
    return (L * L * L + L * L * P + L * P * P + P * P * P) * (int)sizeof(cx<R>) > 12 * 1024;
}
template <typename R, int L>
__host__ __device__ constexpr int m2f2_warp_elems() {
    constexpr int P = 2 * L - 1;
    return L * L * L + L * L * P + L * P * P + (m2f2_direct<R, L>() ? 0 : P * P * P);
}
template <typename R, int L>
__host__ __device__ constexpr bool m2f2_fits() {
    return m2f2_warp_elems<R, L>() * (int)sizeof(cx<R>) <= 24 * 1024;
}

template <int L, typename V>
__device__ __forceinline__ V twc(int f, int c) {  // e^{-2 pi i f c / P} (compile-time f, c)
    constexpr int P = 2 * L - 1;
    if constexpr (sizeof(V) == 8) {
        return c_twf[L - 1][(f * c) % P];
    } else {
        return c_tw[L - 1][(f * c) % P];
    }
}

// A warp transforms M2F_HPW consecutive expansions and loads the next one's
// entries into registers while it works on the current one: with one expansion
// per warp the kernel waited on that load (long-scoreboard stalls at 15 warps
// per issue, 25% issue utilisation, ncu on cfg2 L6).  Measured: L4 c64 87 -> 75 us
// (cfg2), L5 c64 881 -> 710 us (cfg3); the direct-store variant (c64 L >= 6,
// c128 L >= 5) lost 4% to the longer tail and keeps one expansion per warp.
template <typename R, int L>
__host__ __device__ constexpr int m2f2_hpw() {
    return m2f2_direct<R, L>() ? 1 : 4;
}

template <typename R, int L>
__global__ void __launch_bounds__(32 * M2F_WARPS) m2f2_kernel(int64_t n, const int64_t* __restrict__ src_slot,
                                                              const cx<R>* __restrict__ mult,
                                                              cx<R>* __restrict__ hat) {
    using V = cx<R>;
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P, PP = P * P, E = per_lane<L>();
    extern __shared__ unsigned char smraw[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int M2F_HPW = m2f2_hpw<R, L>();
    const int64_t i0 = ((int64_t)blockIdx.x * M2F_WARPS + w) * M2F_HPW;
    if (i0 >= n) return;
    V* X = reinterpret_cast<V*>(smraw) + w * m2f2_warp_elems<R, L>();
    V* Y1 = X + L3;          // [a][b][f2]
    V* Y2 = Y1 + L * L * P;  // [a][f1][f2]
    V* Z = Y2 + L * PP;      // [f0][f1][f2] natural order
    V nxt[E];
    {
        const int64_t s = src_slot[i0] * L3;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            nxt[e] = r < L3 ? mult[s + r] : cz<V>();
        }
    }
    for (int h = 0; h < M2F_HPW; ++h) {
        const int64_t i = i0 + h;
        if (i >= n) break;
        __syncwarp();  // the previous expansion's readers of the buffers are done
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < L3) X[r] = nxt[e];
        }
        if (h + 1 < M2F_HPW && i + 1 < n) {
            const int64_t s = src_slot[i + 1] * L3;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int r = lane + 32 * e;
                if (r < L3) nxt[e] = mult[s + r];
            }
        }
        __syncwarp();
        for (int row = lane; row < L * L; row += 32) {  // axis 2: c -> f2
            V x[L];
#pragma unroll
            for (int c = 0; c < L; ++c) x[c] = X[row * L + c];
#pragma unroll
            for (int f = 0; f < P; ++f) {
                V v = cz<V>();
#pragma unroll
                for (int c = 0; c < L; ++c) v = cfma(x[c], twc<L, V>(f, c), v);
                Y1[row * P + f] = v;
            }
        }
        __syncwarp();
        for (int row = lane; row < L * P; row += 32) {  // axis 1: b -> f1; row = (a, f2)
            const int a = row / P, f2 = row % P;
            V y[L];
#pragma unroll
            for (int b = 0; b < L; ++b) y[b] = Y1[(a * L + b) * P + f2];
#pragma unroll
            for (int f = 0; f < P; ++f) {
                V v = cz<V>();
#pragma unroll
                for (int b = 0; b < L; ++b) v = cfma(y[b], twc<L, V>(f, b), v);
                Y2[(a * P + f) * P + f2] = v;
            }
        }
        __syncwarp();
        const R scale = (R)(1.0 / (P * sqrt((double)P)));
        for (int row = lane; row < PP; row += 32) {  // axis 0: a -> f0; row = (f1, f2)
            V z[L];
#pragma unroll
            for (int a = 0; a < L; ++a) z[a] = Y2[a * PP + row];
#pragma unroll
            for (int f = 0; f < P; ++f) {
                V v = cz<V>();
#pragma unroll
                for (int a = 0; a < L; ++a) v = cfma(z[a], twc<L, V>(f, a), v);
                if constexpr (m2f2_direct<R, L>()) {
                    hat[i * (int64_t)spec_stride<R, L>() + finv<L>(f * PP + row)] = cscale(v, scale);
                } else {
                    Z[f * PP + row] = cscale(v, scale);
                }
            }
        }
        constexpr int SS = spec_stride<R, L>();
        V* out = hat + i * (int64_t)SS;
        if constexpr (m2f2_direct<R, L>()) {
            if (lane == 0 && SS > P3) out[P3] = cz<V>();  // pad entry (c64)
        } else {
            __syncwarp();
            for (int t = lane; t < SS; t += 32) out[t] = t < P3 ? Z[forder<L>(t)] : cz<V>();  // pad entry (c64) = 0
        }
    }
}

// K9 symbols: kernel column G(beta (t + z)) on the difference grid (wrap
// order) and its unnormalised forward DFT (fourier.py:156-183), in FP64,
// stored as R.
template <typename R, int L>
__global__ void __launch_bounds__(256) symbols_kernel(int64_t n, const int32_t* __restrict__ tvec,
                                                      const double* __restrict__ beta, double kappa,
                                                      cx<R>* __restrict__ sym) {
    constexpr int P = pad<L>(), P3 = P * P * P;
    extern __shared__ unsigned char smraw[];
    double2* tw = reinterpret_cast<double2*>(smraw);
    double2* A = tw + P;
    double2* B = A + P3;
    const int64_t i = blockIdx.x;
    make_twiddles<P, double2>(tw);
    const double h = 1.0 / (L - 1);
    const double b = beta[i];
    const double inv4pi = 1.0 / (4.0 * 3.141592653589793);
    for (int t = threadIdx.x; t < P3; t += blockDim.x) {
        const int k0 = t / (P * P), k1 = (t / P) % P, k2 = t % P;
        const double zx = tvec[3 * i + 0] + (k0 < L ? k0 : k0 - P) * h;
        const double zy = tvec[3 * i + 1] + (k1 < L ? k1 : k1 - P) * h;
        const double zz = tvec[3 * i + 2] + (k2 < L ? k2 : k2 - P) * h;
        const double r = b * sqrt(zx * zx + zy * zy + zz * zz);
        A[t] = cscale(cexpi(kappa * r), inv4pi / r);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < P3; t += blockDim.x) {
        const int row = t / P, f = t % P;
        double2 v = make_double2(0.0, 0.0);
        for (int k = 0; k < P; ++k) v = cfma(A[row * P + k], tw[(f * k) % P], v);
        B[t] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < P3; t += blockDim.x) {
        const int a = t / (P * P), f = (t / P) % P, c = t % P;
        double2 v = make_double2(0.0, 0.0);
        for (int k = 0; k < P; ++k) v = cfma(B[(a * P + k) * P + c], tw[(f * k) % P], v);
        A[t] = v;
    }
    __syncthreads();
    constexpr int SS = spec_stride<R, L>();
    cx<R>* out = sym + i * (int64_t)SS;
    for (int t = threadIdx.x; t < SS; t += blockDim.x) {
        double2 v = make_double2(0.0, 0.0);
        if (t < P3) {
            const int j = forder<L>(t);
            const int f = j / (P * P), bc = j % (P * P);
            for (int k = 0; k < P; ++k) v = cfma(A[k * P * P + bc], tw[(f * k) % P], v);
        }
        out[t] = from_d<cx<R>>(v);
    }
}

// itertools.permutations(range(3)) order (fourier.py:94)
__constant__ int8_t c_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

// flat index of the canonical entry feeding frequency j under rotation rid:
// mapped[perm[a]] = (sign[a] f[a]) mod P  (fourier.py:123-143)
template <int P>
__device__ __forceinline__ int rotated_index(int j, int rid) {
    const int f[3] = {j / (P * P), (j / P) % P, j % P};
    const int wt[3] = {P * P, P, 1};
    const int pi = rid >> 3;
    int idx = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int ng = (rid >> (2 - a)) & 1;
        idx += wt[c_perm[pi][a]] * (ng ? (f[a] ? P - f[a] : 0) : f[a]);
    }
    return idx;
}

// K9b: derived symbols D_t[j] = D_canon[rotated_index(j, rid)] (permute_symbol,
// fourier.py:186-196), materialised once per plan so the M2L streams them with
// coalesced loads (the in-loop gather made v1 L1-bound, profiles/r01_summary_v1.md).
template <typename R, int L>
__global__ void __launch_bounds__(256) expand_symbols_kernel(int64_t n, const int32_t* __restrict__ canon,
                                                             const int8_t* __restrict__ rid,
                                                             const cx<R>* __restrict__ symc,
                                                             cx<R>* __restrict__ symd) {
    constexpr int P = pad<L>(), P3 = P * P * P;
    const int64_t i = blockIdx.x;
    const int r = rid[i];
    constexpr int SS = spec_stride<R, L>();
    const cx<R>* src = symc + (int64_t)canon[i] * SS;
    cx<R>* dst = symd + i * SS;
    for (int t = threadIdx.x; t < SS; t += blockDim.x)
        dst[t] = t < P3 ? src[finv<L>(rotated_index<P>(forder<L>(t), r))] : cz<cx<R>>();
}

// ---------------------------------------------------------------------------
// K7+K8: Hadamard M2L + fused F2L.

template <int L>
__host__ __device__ constexpr int m2l_threads() {
    return L <= 3 ? 128 : L == 4 ? 352 : L == 5 ? 256 : L == 6 ? 448 : L == 7 ? 320 : 384;
}
// complex64: one thread per PAIR of frequencies (16-B loads)
template <int L>
__host__ __device__ constexpr int m2l_threads_c64() {
    return L <= 2 ? 32 : L == 3 ? 64 : L == 4 ? 192 : L == 5 ? 384 : L == 6 ? 352 : L == 7 ? 384 : 576;
}
template <typename R, int L>
__host__ __device__ constexpr int m2l_block() {
    return sizeof(R) == 4 ? m2l_threads_c64<L>() : m2l_threads<L>();
}

// pruned inverse DFT of one accumulated spectrum X (P^3, smem) into an L^3
// nodal vector (fourier.py:74-80): contract f0 -> a, f1 -> b, f2 -> c;
// tw = the P x L twiddle matrix (make_twiddle_matrix), conjugated here.
// ROWS = true: one 1D row per thread with constant-bank twiddles (standalone
// f2l_rows_kernel: 80 -> 60 us on cfg2); the fused F2L of the M2L row kernel
// keeps the per-output form (the row variant's registers cost the row
// kernel's occupancy: 1.65 -> 1.70 ms)
template <int L, typename V, bool ROWS = false>
__device__ __forceinline__ void f2l_row(const V* tw, V* X, V* Z1, V* out, int nt) {
    constexpr int P = pad<L>(), L3 = cube<L>();
    if constexpr (ROWS && P <= 9) {
        // one 1D inverse-DFT ROW per thread: P inputs loaded once, L outputs
        // with the twiddles as compile-time constant-bank operands (the
        // per-output variant re-read P inputs and P twiddles from shared memory)
        constexpr int PP = P * P;
        for (int row = threadIdx.x; row < PP; row += nt) {  // axis 0: f0 -> a; row = (f1, f2)
            V x[P];
#pragma unroll
            for (int f = 0; f < P; ++f) x[f] = X[f * PP + row];
#pragma unroll
            for (int a = 0; a < L; ++a) {
                V v = cz<V>();
#pragma unroll
                for (int f = 0; f < P; ++f) v = cfma(x[f], cconj(c_tw[L - 1][(f * a) % P]), v);
                Z1[a * PP + row] = v;
            }
        }
        __syncthreads();
        for (int row = threadIdx.x; row < L * P; row += nt) {  // axis 1: f1 -> b; row = (a, f2)
            const int a = row / P, f2 = row % P;
            V y[P];
#pragma unroll
            for (int f = 0; f < P; ++f) y[f] = Z1[(a * P + f) * P + f2];
#pragma unroll
            for (int b = 0; b < L; ++b) {
                V v = cz<V>();
#pragma unroll
                for (int f = 0; f < P; ++f) v = cfma(y[f], cconj(c_tw[L - 1][(f * b) % P]), v);
                X[(a * L + b) * P + f2] = v;
            }
        }
        __syncthreads();
        const double scale = 1.0 / (P * sqrt((double)P));
        for (int row = threadIdx.x; row < L * L; row += nt) {  // axis 2: f2 -> c; row = (a, b)
            V z[P];
#pragma unroll
            for (int f = 0; f < P; ++f) z[f] = X[row * P + f];
#pragma unroll
            for (int c = 0; c < L; ++c) {
                V v = cz<V>();
#pragma unroll
                for (int f = 0; f < P; ++f) v = cfma(z[f], cconj(c_tw[L - 1][(f * c) % P]), v);
                out[row * L + c] = cscale(v, scale);
            }
        }
    } else {
        for (int t = threadIdx.x; t < L * P * P; t += nt) {
            const int a = t / (P * P), f12 = t % (P * P);
            V v = cz<V>();
#pragma unroll
            for (int f0 = 0; f0 < P; ++f0) v = cfma(X[f0 * P * P + f12], cconj(tw[f0 * L + a]), v);
            Z1[t] = v;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < L * L * P; t += nt) {
            const int a = t / (L * P), b = (t / P) % L, f2 = t % P;
            V v = cz<V>();
#pragma unroll
            for (int f1 = 0; f1 < P; ++f1) v = cfma(Z1[(a * P + f1) * P + f2], cconj(tw[f1 * L + b]), v);
            X[t] = v;
        }
        __syncthreads();
        const double scale = 1.0 / (P * sqrt((double)P));
        for (int t = threadIdx.x; t < L3; t += nt) {
            const int ab = t / L, c = t % L;
            V v = cz<V>();
#pragma unroll
            for (int f2 = 0; f2 < P; ++f2) v = cfma(X[ab * P + f2], cconj(tw[f2 * L + c]), v);
            out[t] = cscale(v, scale);
        }
    }
}

// Product M2L: one CTA per target row (= local slot with >= 1 M2L source),
// entries {source spectrum, derived symbol} streamed coalesced, two entries
// in flight per iteration, accumulation and F2L in FP64 for both storage types.
template <typename R, int L>
__global__ void __launch_bounds__(m2l_block<R, L>()) m2l_rows_kernel(
    int64_t nrows, const int64_t* __restrict__ row_slot, const int64_t* __restrict__ row_ptr,
    const int2* __restrict__ ent, const cx<R>* __restrict__ hat, const cx<R>* __restrict__ symd,
    cx<R>* __restrict__ local) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int SS = spec_stride<R, L>();
    constexpr int NT = m2l_block<R, L>();
    constexpr bool VEC = sizeof(R) == 4;     // complex64: two frequencies per thread
    constexpr int W = VEC ? 2 : 1;           // complex entries per load
    constexpr int PER = (SS / W + NT - 1) / NT;
    extern __shared__ unsigned char smraw[];
    double2* tw = reinterpret_cast<double2*>(smraw);
    double2* X = tw + P * L;
    double2* Z1 = X + P3 + 1;
    double2* O = Z1 + L * P * P;
    const int64_t row = blockIdx.x;
    make_twiddle_matrix<L, double2>(tw);
    // two independent entries in flight per iteration (4 was measured slower:
    // registers -> occupancy).  Products and the two partial sums are formed in
    // the storage precision (c64: FP32 -- converting every operand to FP64 made
    // the F2F unit the bottleneck, profiles/r01_summary_v2.md); the partial
    // sums are combined and transformed (F2L) in FP64.
    using V = cx<R>;
    V acc[2][PER][W];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int m = 0; m < PER; ++m)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[u][m][w] = cz<V>();
    const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
    for (int64_t e = e0; e < e1; e += 2) {
        const bool two = e + 1 < e1;
        const int2 a = ent[e];
        const int2 b = two ? ent[e + 1] : a;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int jv = threadIdx.x + m * NT;  // vector index
            if (jv * W < SS) {
                if constexpr (VEC) {
                    const float4 sa = __ldg(reinterpret_cast<const float4*>(hat + (int64_t)a.x * SS) + jv);
                    const float4 da = __ldg(reinterpret_cast<const float4*>(symd + (int64_t)a.y * SS) + jv);
                    const float4 sb = __ldg(reinterpret_cast<const float4*>(hat + (int64_t)b.x * SS) + jv);
                    const float4 db = __ldg(reinterpret_cast<const float4*>(symd + (int64_t)b.y * SS) + jv);
                    acc[0][m][0] = cfma(make_float2(da.x, da.y), make_float2(sa.x, sa.y), acc[0][m][0]);
                    acc[0][m][1] = cfma(make_float2(da.z, da.w), make_float2(sa.z, sa.w), acc[0][m][1]);
                    if (two) {
                        acc[1][m][0] = cfma(make_float2(db.x, db.y), make_float2(sb.x, sb.y), acc[1][m][0]);
                        acc[1][m][1] = cfma(make_float2(db.z, db.w), make_float2(sb.z, sb.w), acc[1][m][1]);
                    }
                } else {
                    const V sa = __ldg(hat + (int64_t)a.x * SS + jv);
                    const V da = __ldg(symd + (int64_t)a.y * SS + jv);
                    const V sb = __ldg(hat + (int64_t)b.x * SS + jv);
                    const V db = __ldg(symd + (int64_t)b.y * SS + jv);
                    acc[0][m][0] = cfma(da, sa, acc[0][m][0]);
                    if (two) acc[1][m][0] = cfma(db, sb, acc[1][m][0]);
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int jv = threadIdx.x + m * NT;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const int j = jv * W + w;
            if (j < P3) X[forder<L>(j)] = cadd(to_d(acc[0][m][w]), to_d(acc[1][m][w]));
        }
    }
    __syncthreads();
    f2l_row<L, double2>(tw, X, Z1, O, NT);
    __syncthreads();
    cx<R>* out = local + row_slot[row] * L3;
    for (int t = threadIdx.x; t < L3; t += NT) out[t] = from_d<cx<R>>(O[t]);
}

// ---------------------------------------------------------------------------
// K7 v8: sibling-group M2L (pair / quartet).  One CTA per group of K = 2 or 4
// sibling rows (same level, key and target parent; fewer when the sibling set
// runs out).  The group's events are merged per source spectrum: entry
// {s, symbol of row 0 or -1, ..., symbol of row K-1 or -1} (padded to 4 / 8
// ints), so a source several rows read is loaded once -- 1.6 (K = 2) / ~1.4
// (K = 4) operand loads per event instead of the row kernel's 2 on surface
// data, with the row kernel's streaming structure and register budget (the
// row kernel is bound by the L1/shared data path: only register reuse takes
// bytes off it).  F2L of the group's rows in shared memory, one after another.
#ifndef DEFMM_PAIR_REGS
#define DEFMM_PAIR_REGS 56
#endif
template <int K>
struct GroupEnt;
template <>
struct GroupEnt<2> {
    int4 a;  // {s, t0, t1, 0}
};
template <>
struct GroupEnt<3> {
    int4 a;  // {s, t0, t1, t2}
};
template <>
struct GroupEnt<4> {
    int4 a, b;  // {s, t0, t1, t2}, {t3, 0, 0, 0}
};
template <int K>
__device__ __forceinline__ GroupEnt<K> load_gent(const int* ent, int64_t e) {
    GroupEnt<K> g;
    g.a = __ldg(reinterpret_cast<const int4*>(ent) + (K <= 3 ? e : 2 * e));
    if constexpr (K == 4) g.b = __ldg(reinterpret_cast<const int4*>(ent) + 2 * e + 1);
    return g;
}
template <int K>
__device__ __forceinline__ int gent_src(const GroupEnt<K>& g) { return g.a.x; }
template <int K>
__device__ __forceinline__ int gent_sym(const GroupEnt<K>& g, int k) {
    if constexpr (K == 2) {
        return k == 0 ? g.a.y : g.a.z;
    } else if constexpr (K == 3) {
        return k == 0 ? g.a.y : k == 1 ? g.a.z : g.a.w;
    } else {
        return k == 0 ? g.a.y : k == 1 ? g.a.z : k == 2 ? g.a.w : g.b.x;
    }
}

#ifndef DEFMM_TRIPLE_REGS
#define DEFMM_TRIPLE_REGS 56
#endif
#ifndef DEFMM_QUARTET_REGS
#define DEFMM_QUARTET_REGS 56
#endif
template <typename R, int L, int K>
__host__ __device__ constexpr int group_min_blocks() {  // register cap per K, at most 32 CTAs/SM
    constexpr int regs = K == 2 ? DEFMM_PAIR_REGS : K == 3 ? DEFMM_TRIPLE_REGS : DEFMM_QUARTET_REGS;
    return 65536 / (m2l_block<R, L>() * regs) < 32 ? 65536 / (m2l_block<R, L>() * regs) : 32;
}
template <typename R, int L, int K>
__global__ void __launch_bounds__(m2l_block<R, L>(), group_min_blocks<R, L, K>())
    m2l_group_kernel(int64_t ngroups, const int64_t* __restrict__ grp_slot, const int64_t* __restrict__ grp_ptr,
                     const int* __restrict__ ent, const cx<R>* __restrict__ hat, const cx<R>* __restrict__ symd,
                     cx<R>* __restrict__ local) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int SS = spec_stride<R, L>();
    constexpr int NT = m2l_block<R, L>();
    constexpr bool VEC = sizeof(R) == 4;
    constexpr int W = VEC ? 2 : 1;
    constexpr int PER = (SS / W + NT - 1) / NT;
#ifndef DEFMM_PAIR_UNROLL
#define DEFMM_PAIR_UNROLL 3
#endif
#ifndef DEFMM_QUARTET_UNROLL
#define DEFMM_QUARTET_UNROLL 1
#endif
    constexpr int UNROLL = K == 2 ? DEFMM_PAIR_UNROLL : K == 3 ? 2 : DEFMM_QUARTET_UNROLL;  // entries in flight
    using V = cx<R>;
    using VT = std::conditional_t<VEC, float4, double2>;
    extern __shared__ unsigned char smraw[];
    double2* tw = reinterpret_cast<double2*>(smraw);
    double2* X = tw + P * L;
    double2* Z1 = X + P3 + 1;
    double2* O = Z1;  // Z1 is dead after the second axis: 6 CTAs fit a 64 KB carveout
    const int64_t g = blockIdx.x;
    make_twiddle_matrix<L, double2>(tw);
    const VT* hv = reinterpret_cast<const VT*>(hat);
    const VT* dv = reinterpret_cast<const VT*>(symd);
    constexpr int NV = SS / W;
    V acc[K][PER][W];
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
        for (int m = 0; m < PER; ++m)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[u][m][w] = cz<V>();
    auto fma_v = [](V (&a)[W], const VT& d, const VT& x) {
        if constexpr (VEC) {
            a[0] = cfma(make_float2(d.x, d.y), make_float2(x.x, x.y), a[0]);
            a[W - 1] = cfma(make_float2(d.z, d.w), make_float2(x.z, x.w), a[W - 1]);
        } else {
            a[0] = cfma(d, x, a[0]);
        }
    };
    const int64_t e0 = grp_ptr[g], e1 = grp_ptr[g + 1];
    for (int64_t e = e0; e < e1; e += UNROLL) {
        GroupEnt<K> en[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            if (e + u < e1) {
                en[u] = load_gent<K>(ent, e + u);
            } else {  // no-op entry: every symbol absent
                en[u] = load_gent<K>(ent, e);
                en[u].a.y = en[u].a.z = -1;
                if constexpr (K >= 3) en[u].a.w = -1;
                if constexpr (K == 4) en[u].b.x = -1;
            }
        }
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int jv = threadIdx.x + m * NT;
            if (jv < NV) {
                VT sv[UNROLL], dk[UNROLL][K];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    sv[u] = __ldg(hv + (int64_t)gent_src<K>(en[u]) * NV + jv);
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const int t = gent_sym<K>(en[u], k);
                        dk[u][k] = t >= 0 ? __ldg(dv + (int64_t)t * NV + jv) : VT{};
                    }
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u)
#pragma unroll
                    for (int k = 0; k < K; ++k) fma_v(acc[k][m], dk[u][k], sv[u]);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < K; ++u) {
        const int64_t slot = grp_slot[K * g + u];
        if (slot < 0) break;  // uniform; rows fill the group from the front
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int jv = threadIdx.x + m * NT;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const int j = jv * W + w;
                if (jv < NV && j < P3) X[forder<L>(j)] = to_d(acc[u][m][w]);
            }
        }
        __syncthreads();
        f2l_row<L, double2>(tw, X, Z1, O, NT);
        __syncthreads();
        cx<R>* out = local + slot * L3;
        for (int t = threadIdx.x; t < L3; t += NT) out[t] = from_d<cx<R>>(O[t]);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K7 v13: staged M2L.  The sibling-group kernel above moves ~1.3 spectra
// L2 -> SM per event (one symbol per event, a source per ~3 events) and is
// bound by that fabric (profiles/r02/summary_v2.md).  A derived symbol depends
// only on (level, key, t - s): the target parents of one (level, key) that lie
// next to each other read the SAME symbols for the same parent-relative source
// offset u = s - 2 parent.  So here a CTA owns NW = 8 neighbouring "warp
// units" (a target parent's <= K = 4 sibling rows each, same level and key)
// and one spectral slice of <= 32 16-B vectors; its classes (distinct u) are
// packed into stages of <= ns_cap symbol slices, which a producer warp copies
// ONCE per CTA into a shared-memory ring (cp.async.bulk, complete_tx on the
// stage's "full" mbarrier).  Each consumer warp walks its own entries of the
// stage -- {source spectrum, ring slot of row k's symbol or 0xff} -- with the
// source slice prefetched PF entries ahead into registers (LDG) and the
// symbols read from the ring (LDS.128), then releases the stage through its
// "empty" mbarrier.  No CTA-wide barrier in the loop.  The accumulated slices
// go to lhat; f2l_rows_kernel applies the inverse DFT.
__device__ __forceinline__ uint32_t sm32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sm32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sm32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n" ::"r"(sm32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     sm32(dst)),
                 "l"(src), "r"(bytes), "r"(sm32(b))
                 : "memory");
}

// (c0, c1) += a * (b0, b1): one packed FP32 FMA (FFMA2) with a scalar multiplier
__device__ __forceinline__ void ffma2(float& c0, float& c1, float a, float b0, float b1) {
    float2 av = make_float2(a, a), bv = make_float2(b0, b1), cv = make_float2(c0, c1);
    uint64_t ua = *reinterpret_cast<uint64_t*>(&av), ub = *reinterpret_cast<uint64_t*>(&bv);
    uint64_t uc = *reinterpret_cast<uint64_t*>(&cv);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(uc) : "l"(ua), "l"(ub));
    cv = *reinterpret_cast<float2*>(&uc);
    c0 = cv.x;
    c1 = cv.y;
}
__device__ __forceinline__ void ffma2(double&, double&, double, double, double) {}  // c128: not used

#ifndef DEFMM_STAGE_MINB
#define DEFMM_STAGE_MINB 3
#endif
constexpr int STG_NW = 8;     // consumer warps (warp units) per CTA
constexpr int STG_K = 4;      // rows per warp unit
constexpr int STG_MAXDEPTH = 8;  // ring stages (runtime depth <= this)
constexpr int STG_PF = 4;     // source slices in flight per warp (the loop is unrolled 4-way)

template <typename R, int L>
struct StageCfg {
    static constexpr int W = sizeof(R) == 4 ? 2 : 1;              // complex entries per 16-B vector
    static constexpr int NV = spec_stride<R, L>() / W;            // vectors per spectrum
    static constexpr int NSLICE = (NV + 31) / 32;                 // spectral slices (grid.y role)
    static constexpr int SW = (NV + NSLICE - 1) / NSLICE;         // vectors (= lanes) per slice
    static constexpr int SB = SW * 16;                            // bytes per ring slot
};

// ring buffer b: slots [0, ns_cap) filled by the producer, slot ns_cap = zeros
// (the entries name it for an absent row, so the loop has no branch per row)
template <typename R, int L>
__global__ void __launch_bounds__(32 * (STG_NW + 1), DEFMM_STAGE_MINB)
    m2l_stage_kernel(int ns_cap, int depth, const int* __restrict__ cta_stage, const int* __restrict__ cta_went,
                     const int* __restrict__ stage_slot_ptr, const int* __restrict__ slot_sym,
                     const int* __restrict__ stage_wend, const int2* __restrict__ ent,
                     const int* __restrict__ cta_rows, const cx<R>* __restrict__ hat,
                     const cx<R>* __restrict__ symd, cx<R>* __restrict__ lhat) {
    using C = StageCfg<R, L>;
    constexpr bool VEC = sizeof(R) == 4;
    using VT = std::conditional_t<VEC, float4, double2>;
    constexpr int NV = C::NV, SW = C::SW, SB = C::SB, NW = STG_NW, K = STG_K, PF = STG_PF;
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
    uint64_t* empty = full + STG_MAXDEPTH;
    unsigned char* ring = smraw + 128;  // [depth][ns_cap + 1][SB]
    const uint32_t bufb = (uint32_t)(ns_cap + 1) * SB;
    const int cta = blockIdx.x / C::NSLICE, slice = blockIdx.x % C::NSLICE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int v0 = slice * SW;
    const int nvec = min(SW, NV - v0);  // vectors of this slice (> 0)
    if (threadIdx.x == 0) {
        for (int s = 0; s < depth; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int t = threadIdx.x; t < depth * (SB / 16); t += blockDim.x)  // the zero slots
        reinterpret_cast<float4*>(ring + (size_t)(t / (SB / 16)) * bufb + (size_t)ns_cap * SB)[t % (SB / 16)] =
            make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    const int st0 = cta_stage[cta], nst = cta_stage[cta + 1] - st0;
    if (warp == NW) {  // producer warp: one bulk copy per symbol slice
        const unsigned char* sb = reinterpret_cast<const unsigned char*>(symd) + (size_t)v0 * 16;
        const uint32_t bytes = (uint32_t)nvec * 16u;
        int p0 = stage_slot_ptr[st0];
        int p1 = nst > 0 ? stage_slot_ptr[st0 + 1] : p0;
        // the next stage's symbol ids are fetched before waiting for its buffer
        int id0 = p0 + lane < p1 ? __ldg(slot_sym + p0 + lane) : 0;
        int id1 = p0 + lane + 32 < p1 ? __ldg(slot_sym + p0 + lane + 32) : 0;
        int buf = 0, round = 0;
        for (int i = 0; i < nst; ++i) {
            const int q1 = i + 1 < nst ? stage_slot_ptr[st0 + i + 2] : p1;
            const int n0 = p1 + lane < q1 ? __ldg(slot_sym + p1 + lane) : 0;
            const int n1 = p1 + lane + 32 < q1 ? __ldg(slot_sym + p1 + lane + 32) : 0;
            if (round > 0) mbar_wait(&empty[buf], (uint32_t)((round - 1) & 1));
            if (lane == 0) mbar_expect_tx(&full[buf], (uint32_t)(p1 - p0) * bytes);
            __syncwarp();
            unsigned char* dst = ring + (size_t)buf * bufb;
            if (p0 + lane < p1) bulk_g2s(dst + (size_t)lane * SB, sb + (size_t)id0 * (NV * 16), bytes, &full[buf]);
            if (p0 + lane + 32 < p1)
                bulk_g2s(dst + (size_t)(lane + 32) * SB, sb + (size_t)id1 * (NV * 16), bytes, &full[buf]);
            for (int j = p0 + lane + 64; j < p1; j += 32)  // ns_cap > 64
                bulk_g2s(dst + (size_t)(j - p0) * SB, sb + (size_t)__ldg(slot_sym + j) * (NV * 16), bytes, &full[buf]);
            p0 = p1;
            p1 = q1;
            id0 = n0;
            id1 = n1;
            if (++buf == depth) {
                buf = 0;
                ++round;
            }
        }
        return;
    }
    // lanes past the slice repeat its last vector (no predicates in the loop)
    const int lc = min(lane, nvec - 1);
    const VT* hv = reinterpret_cast<const VT*>(hat) + v0 + lc;
    // complex64: two packed accumulators per (row, frequency), P += s.re * (d.re, d.im) and
    // Q += s.im * (d.re, d.im) -- one FFMA2 each with the source part as the scalar
    // operand; sum = (P.x - Q.y, P.y + Q.x) at the end.  complex128: plain FP64 FMAs.
    constexpr int NA = VEC ? 8 : 2;
    R acc[K][NA];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < NA; ++c) acc[k][c] = 0;
    const int cw = cta * NW + warp;
    int i = cta_went[cw];
    // stage ends of this warp: stage_wend[st0 NW + warp nst + s]
    const int* wend = stage_wend + (size_t)st0 * NW + (size_t)warp * nst;
    const int e_total = nst > 0 ? wend[nst - 1] : i;
    // entries in chunks of 32 (one per lane) advancing by 32 - PF, so entry j and the
    // prefetched j + PF are both in the current chunk; broadcast by shuffles
    constexpr int CH = 32 - PF;
    int cbase = i;
    int2 cur = __ldg(ent + cbase + lane), nxt = __ldg(ent + cbase + CH + lane);
    VT srcq[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {  // entries past e_total are other warps' (or padding): valid sources
        const int sid = __shfl_sync(0xffffffffu, cur.x, u);
        srcq[u] = __ldg(hv + (size_t)sid * NV);
    }
    int buf = 0, round = 0, phase = 0;
    int nxt_end = nst > 0 ? wend[0] : i;
    const uint32_t ring32 = sm32(ring) + (uint32_t)lc * 16u;
    for (int st = 0; st < nst; ++st) {
        const int end = nxt_end;  // the next stage's end is requested a stage ahead
        nxt_end = st + 1 < nst ? __ldg(wend + st + 1) : e_total;
        mbar_wait(&full[buf], (uint32_t)(round & 1));
        const uint32_t rb = ring32 + (uint32_t)buf * bufb;
        // one entry, source in ring register U (static index); the next source of that
        // register (entry i + PF) is requested once the entry's products are issued
#define DEFMM_STAGE_BODY(U)                                                                          \
    {                                                                                                \
        const int j = i - cbase;                                                                     \
        const uint32_t slots = (uint32_t)__shfl_sync(0xffffffffu, cur.y, j);                         \
        const int sidn = __shfl_sync(0xffffffffu, cur.x, j + PF);                                    \
        const VT s = srcq[U];                                                                        \
        _Pragma("unroll") for (int k = 0; k < K; ++k) {                                              \
            const uint32_t addr = __byte_perm(slots, 0u, 0x4440u + k) * (uint32_t)SB + rb;           \
            if constexpr (VEC) {                                                                     \
                float4 d;                                                                            \
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"                              \
                             : "=f"(d.x), "=f"(d.y), "=f"(d.z), "=f"(d.w)                            \
                             : "r"(addr));                                                           \
                ffma2(acc[k][0], acc[k][1], s.x, d.x, d.y);                                          \
                ffma2(acc[k][2], acc[k][3], s.y, d.x, d.y);                                          \
                ffma2(acc[k][4], acc[k][5], s.z, d.z, d.w);                                          \
                ffma2(acc[k][6], acc[k][7], s.w, d.z, d.w);                                          \
            } else {                                                                                 \
                double2 d;                                                                           \
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(d.x), "=d"(d.y) : "r"(addr)); \
                acc[k][0] = fma(d.x, s.x, acc[k][0]);                                                \
                acc[k][0] = fma(-d.y, s.y, acc[k][0]);                                               \
                acc[k][1] = fma(d.x, s.y, acc[k][1]);                                                \
                acc[k][1] = fma(d.y, s.x, acc[k][1]);                                                \
            }                                                                                        \
        }                                                                                            \
        srcq[U] = __ldg(hv + (size_t)sidn * NV); /* after the last use of s: lands in place */      \
        ++i;                                                                                         \
    }
        while (i < end) {
            if (i - cbase >= CH) {  // next chunk of entries (every 28th entry)
                cur = nxt;
                cbase += CH;
                nxt = __ldg(ent + cbase + CH + lane);
            }
            const int lim = min(end, cbase + CH);
            // enter the 4-way unrolled sequence at the ring position of entry i
            if (phase == 1) goto stage_l1;
            if (phase == 2) goto stage_l2;
            if (phase == 3) goto stage_l3;
        stage_l0:
            if (i >= lim) { phase = 0; goto stage_done; }
            DEFMM_STAGE_BODY(0)
        stage_l1:
            if (i >= lim) { phase = 1; goto stage_done; }
            DEFMM_STAGE_BODY(1)
        stage_l2:
            if (i >= lim) { phase = 2; goto stage_done; }
            DEFMM_STAGE_BODY(2)
        stage_l3:
            if (i >= lim) { phase = 3; goto stage_done; }
            DEFMM_STAGE_BODY(3)
            goto stage_l0;
        stage_done:;
        }
#undef DEFMM_STAGE_BODY
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);
        if (++buf == depth) {
            buf = 0;
            ++round;
        }
    }
    if (lane < nvec) {
        VT* lv = reinterpret_cast<VT*>(lhat) + v0 + lane;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int row = cta_rows[(size_t)cw * K + k];
            if (row >= 0) {
                if constexpr (VEC) {
                    lv[(size_t)row * NV] = make_float4(acc[k][0] - acc[k][3], acc[k][1] + acc[k][2],
                                                       acc[k][4] - acc[k][7], acc[k][5] + acc[k][6]);
                } else {
                    lv[(size_t)row * NV] = make_double2(acc[k][0], acc[k][1]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K7 v3: parent-pair blocked M2L.  A CTA owns a group = (target parent P,
// key) with up to 8 target rows (its children a); a block = (group, source
// parent Q) holds up to 8 source spectra (children b) and, per child offset
// delta = a - b in [-1,1]^3, the derived symbol of translation
// 2 (P - Q) + delta.  Every (a, b) pair with its bit in the block mask is one
// M2L event.  The pair -> (symbol, spectrum, accumulator) indices are
// compile-time constants after unrolling over delta and b, so each loaded
// spectrum/symbol is reused for all pairs of the block from registers.
// Accumulated spectra go to lhat (row-major, stride SS); f2l_rows_kernel
// then applies the pruned inverse DFT.

// bit 8a+b of every (a, b) pair with a - b = delta(d)
__host__ __device__ constexpr uint64_t pairs_of(int d) {
    uint64_t m = 0;
    for (int b = 0; b < 8; ++b) {
        const int a0 = ((b >> 2) & 1) + d / 9 - 1, a1 = ((b >> 1) & 1) + (d / 3) % 3 - 1, a2 = (b & 1) + d % 3 - 1;
        if (a0 >= 0 && a0 <= 1 && a1 >= 0 && a1 <= 1 && a2 >= 0 && a2 <= 1)
            m |= (uint64_t)1 << (8 * (a0 * 4 + a1 * 2 + a2) + b);
    }
    return m;
}
__host__ __device__ constexpr int pair_a(int d, int b) {
    const int a0 = ((b >> 2) & 1) + d / 9 - 1, a1 = ((b >> 1) & 1) + (d / 3) % 3 - 1, a2 = (b & 1) + d % 3 - 1;
    return (a0 >= 0 && a0 <= 1 && a1 >= 0 && a1 <= 1 && a2 >= 0 && a2 <= 1) ? a0 * 4 + a1 * 2 + a2 : -1;
}

template <typename R, int L>
__host__ __device__ constexpr int m2lb_threads() {
    return m2l_threads<L>();  // one complex entry per thread and load
}

template <typename R>
struct Vec2;  // two complex entries (c64) / one (c128) per thread-load
template <>
struct Vec2<float> {  // one complex64 per load: 2-wide float4 needed 200 registers
    using t = float2;
    static constexpr int W = 1;
};
template <>
struct Vec2<double> {
    using t = double2;
    static constexpr int W = 1;
};

__device__ __forceinline__ void vfma(double2 (&acc)[1], const double2& d, const double2& s) {
    acc[0] = cfma(d, s, acc[0]);
}
__device__ __forceinline__ void vfma(float2 (&acc)[1], const float2& d, const float2& s) {
    acc[0] = cfma(d, s, acc[0]);
}

// Planar block (surface data): every pair (a, b) has a_p == b_p == v for one
// axis p -- 4 x 4 in-plane pairs, 9 in-plane offsets: 4 spectra + 9 symbols
// serve up to 16 events with no predicated-off pair.  i, j = in-plane child
// index (2 bits), octant = embed(i, p, v).
__host__ __device__ constexpr int embed2(int i, int p, int v) {
    // in-plane bits (hi, lo) go to the two remaining axes in increasing order
    return p == 0 ? (v << 2) | i : p == 1 ? (((i >> 1) & 1) << 2) | (v << 1) | (i & 1) : (i << 1) | v;
}
__host__ __device__ constexpr int delta_index3(int a, int b) {
    return ((((a >> 2) & 1) - ((b >> 2) & 1)) + 1) * 9 + ((((a >> 1) & 1) - ((b >> 1) & 1)) + 1) * 3 +
           (((a & 1) - (b & 1)) + 1);
}

template <int PP, int PV, typename VT, typename V, int W>
__device__ __forceinline__ void planar_block(uint64_t mask, const int32_t* bs, const int32_t* bt, const VT* hv,
                                             const VT* dv, int64_t NV, int jv, bool act, V (&acc)[8][W]) {
    VT S[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int sidx = __ldg(bs + embed2(i, PP, PV));
        S[i] = (sidx >= 0 && act) ? __ldg(hv + (int64_t)sidx * NV + jv) : VT{};
    }
    // in-plane offsets (du, dv) in [-1,1]^2 -> 9 symbols
    VT D[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) {
        // representative pair with this in-plane offset
        const int du = e / 3 - 1, dw = e % 3 - 1;
        const int ia = ((du > 0) << 1) | (dw > 0), ib = ((du < 0) << 1) | (dw < 0);
        const int d = delta_index3(embed2(ia, PP, PV), embed2(ib, PP, PV));
        const int tidx = __ldg(bt + d);
        D[e] = (tidx >= 0 && act) ? __ldg(dv + (int64_t)tidx * NV + jv) : VT{};
    }
#pragma unroll
    for (int ia = 0; ia < 4; ++ia)
#pragma unroll
        for (int ib = 0; ib < 4; ++ib) {
            const int a = embed2(ia, PP, PV), b = embed2(ib, PP, PV);
            const int e = (((ia >> 1) & 1) - ((ib >> 1) & 1) + 1) * 3 + ((ia & 1) - (ib & 1) + 1);
            if ((mask >> (8 * a + b)) & 1) vfma(acc[a], D[e], S[ib]);
        }
}

#ifndef DEFMM_M2LB_MINBLOCKS
#define DEFMM_M2LB_MINBLOCKS 2
#endif
template <typename R, int L>
__global__ void __launch_bounds__(m2lb_threads<R, L>(), DEFMM_M2LB_MINBLOCKS) m2l_blocked_kernel(
    int64_t ngroups, const int64_t* __restrict__ grp_ptr, const int64_t* __restrict__ grp_rows,
    const int32_t* __restrict__ blk_src, const int32_t* __restrict__ blk_trans,
    const int64_t* __restrict__ blk_mask, const int8_t* __restrict__ blk_kind, const cx<R>* __restrict__ hat,
    const cx<R>* __restrict__ symd, cx<R>* __restrict__ lhat) {
    using VT = typename Vec2<R>::t;
    using V = cx<R>;
    constexpr int W = Vec2<R>::W;
    constexpr int SS = spec_stride<R, L>();
    constexpr int NV = SS / W;
    constexpr int NT = m2lb_threads<R, L>();
    constexpr int PER = (NV + NT - 1) / NT;
    const int64_t g = blockIdx.x;
    const int64_t b0 = grp_ptr[g], b1 = grp_ptr[g + 1];
    const VT* hv = reinterpret_cast<const VT*>(hat);
    const VT* dv = reinterpret_cast<const VT*>(symd);
    for (int m = 0; m < PER; ++m) {
        const int jv = threadIdx.x + m * NT;
        const bool act = jv < NV;
        V acc[8][W];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[a][w] = cz<V>();
        for (int64_t blk = b0; blk < b1; ++blk) {
            const uint64_t mask = (uint64_t)__ldg(blk_mask + blk);
            const int32_t* bs = blk_src + 8 * blk;
            const int32_t* bt = blk_trans + 27 * blk;
            const int kind = blk_kind ? __ldg(blk_kind + blk) : -1;  // warp-uniform
            if (kind >= 0) {
                switch (kind) {
                    case 0: planar_block<0, 0>(mask, bs, bt, hv, dv, NV, jv, act, acc); break;
                    case 1: planar_block<0, 1>(mask, bs, bt, hv, dv, NV, jv, act, acc); break;
                    case 2: planar_block<1, 0>(mask, bs, bt, hv, dv, NV, jv, act, acc); break;
                    case 3: planar_block<1, 1>(mask, bs, bt, hv, dv, NV, jv, act, acc); break;
                    case 4: planar_block<2, 0>(mask, bs, bt, hv, dv, NV, jv, act, acc); break;
                    default: planar_block<2, 1>(mask, bs, bt, hv, dv, NV, jv, act, acc); break;
                }
                continue;
            }
            VT S[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int sidx = __ldg(bs + b);
                S[b] = (sidx >= 0 && act) ? __ldg(hv + (int64_t)sidx * NV + jv) : VT{};
            }
            // branch-free body (one basic block): the scheduler can then issue
            // every symbol load of the block before the FMAs that consume them
            // (a per-delta `continue` serialised their latencies)
            VT D[27];
#pragma unroll
            for (int d = 0; d < 27; ++d) {
                const int tidx = __ldg(bt + d);
                D[d] = ((mask & pairs_of(d)) != 0 && act) ? __ldg(dv + (int64_t)max(tidx, 0) * NV + jv) : VT{};
            }
#pragma unroll
            for (int d = 0; d < 27; ++d) {
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const int a = pair_a(d, b);  // compile-time after unrolling
                    if (a >= 0 && ((mask >> (8 * a + b)) & 1)) vfma(acc[a], D[d], S[b]);
                }
            }
        }
        if (act) {
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int64_t row = grp_rows[8 * g + a];
                if (row >= 0) {
#pragma unroll
                    for (int w = 0; w < W; ++w) lhat[row * SS + (int64_t)jv * W + w] = acc[a][w];
                }
            }
        }
    }
}

// pruned inverse DFT of accumulated spectra (fourier.py:74-80), one CTA per row:
// local[row_slot[r]] = F2L(lhat[r]); FP64 transform for both storage types
template <typename R, int L>
__global__ void __launch_bounds__(128) f2l_rows_kernel(int64_t nrows, const int64_t* __restrict__ row_slot,
                                                       const cx<R>* __restrict__ lhat, cx<R>* __restrict__ local) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int SS = spec_stride<R, L>();
    extern __shared__ unsigned char smraw[];
    double2* tw = reinterpret_cast<double2*>(smraw);
    double2* X = tw + P * L;
    double2* Z1 = X + P3 + 1;
    double2* O = Z1 + L * P * P;
    const int64_t r = blockIdx.x;
    make_twiddle_matrix<L, double2>(tw);
    const cx<R>* src = lhat + r * SS;
    for (int j = threadIdx.x; j < P3; j += blockDim.x) X[forder<L>(j)] = to_d(src[j]);
    __syncthreads();
    f2l_row<L, double2, true>(tw, X, Z1, O, blockDim.x);
    __syncthreads();
    cx<R>* out = local + row_slot[r] * L3;
    for (int t = threadIdx.x; t < L3; t += blockDim.x) out[t] = from_d<cx<R>>(O[t]);
}

// Reference M2L (v1, c128): canonical symbols gathered in the inner loop.
// Kept as an independent operator for the parity tests.
template <int L>
__global__ void __launch_bounds__(m2l_threads<L>()) m2l_canon_kernel(
    int64_t nrows, const int64_t* __restrict__ row_slot, const int64_t* __restrict__ row_ptr,
    const int32_t* __restrict__ e_src, const int32_t* __restrict__ e_sym,
    const int8_t* __restrict__ e_rid, const double2* __restrict__ hat,
    const double2* __restrict__ sym, double2* __restrict__ local) {
    constexpr int P = pad<L>(), P3 = P * P * P;
    constexpr int NT = m2l_threads<L>();
    constexpr int PER = (P3 + NT - 1) / NT;
    extern __shared__ unsigned char smraw[];
    double2* tw = reinterpret_cast<double2*>(smraw);
    double2* X = tw + P * L;
    double2* Z1 = X + P3;
    const int64_t row = blockIdx.x;
    make_twiddle_matrix<L, double2>(tw);
    double2 acc[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) acc[m] = make_double2(0.0, 0.0);
    for (int64_t e = row_ptr[row]; e < row_ptr[row + 1]; ++e) {
        const double2* S = hat + (int64_t)e_src[e] * P3;
        const double2* D = sym + (int64_t)e_sym[e] * P3;
        const int rid = e_rid[e];
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int j = threadIdx.x + m * NT;
            if (j < P3) acc[m] = cfma(__ldg(D + finv<L>(rotated_index<P>(forder<L>(j), rid))), __ldg(S + j), acc[m]);
        }
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int j = threadIdx.x + m * NT;
        if (j < P3) X[forder<L>(j)] = acc[m];
    }
    __syncthreads();
    f2l_row<L, double2>(tw, X, Z1, local + row_slot[row] * cube<L>(), NT);
}

// ---------------------------------------------------------------------------
// K3: L2P + near-field add + un-permute.  One CTA per target leaf, one thread
// per particle; L2P(x) = sum_abc loc[abc] conj(W0_a W1_b W2_c) with the same
// per-axis weights as P2M.  Output accumulated in FP64.

template <typename R, int L>
__global__ void __launch_bounds__(64, sizeof(R) == 4 ? 16 : 8) l2p_kernel(
    int64_t n, const int32_t* __restrict__ leaf_cell, const int64_t* __restrict__ slot_lo,
    const int64_t* __restrict__ slot_hi, const int32_t* __restrict__ slot_dir,
    const int64_t* __restrict__ cstart, const int64_t* __restrict__ cstop,
    const double* __restrict__ calpha, const int32_t* __restrict__ clevel,
    const double* __restrict__ lbeta, const double* __restrict__ dirs, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, double kappa,
    const cx<R>* __restrict__ local, const cx<R>* __restrict__ near, const int64_t* __restrict__ perm,
    cx<R>* __restrict__ out) {
    using V = cx<R>;
    constexpr int L3 = cube<L>();
    constexpr int NT = 64;
    __shared__ V loc[L3];
    __shared__ V T[3][L];
    const int64_t i = blockIdx.x;
    const int c = leaf_cell[i];
    const double beta = lbeta[clevel[c]];
    const double ibeta = 1.0 / beta;
    const double al[3] = {calpha[3 * c], calpha[3 * c + 1], calpha[3 * c + 2]};
    const int64_t s0 = cstart[c], s1 = cstop[c];
    const int64_t k0 = slot_lo[i], k1 = slot_hi[i];
    for (int64_t base = s0; base < s1; base += NT) {
        const int64_t p = base + threadIdx.x;
        const bool valid = p < s1;
        R xh[3] = {0, 0, 0};
        if (valid) {
            xh[0] = (R)((px[p] - al[0]) * ibeta);
            xh[1] = (R)((py[p] - al[1]) * ibeta);
            xh[2] = (R)((pz[p] - al[2]) * ibeta);
        }
        R S[3][L];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) lagrange<L, R>(xh[ax], S[ax]);
        double2 acc = valid ? to_d(near[p]) : make_double2(0.0, 0.0);
        for (int64_t s = k0; s < k1; ++s) {
            const int d = slot_dir[s];
            __syncthreads();
            for (int r = threadIdx.x; r < L3; r += NT) loc[r] = local[s * L3 + r];
            // e^{i ku (xh - x_k)} = e^{i ku xh} e^{-i ku x_k}: node factors once
            // per slot, one sincos per particle and axis (HF keys only)
            if (threadIdx.x < 3 * L) {
                const int ax = threadIdx.x / L, k = threadIdx.x % L;
                const R ku = (R)(d >= 0 ? kappa * beta * dirs[3 * d + ax] : 0.0);
                T[ax][k] = d >= 0 ? cexpi(-ku * node<L, R>(k)) : cmk<V>((R)1, (R)0);
            }
            __syncthreads();
            V W[3][L];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                V e = cmk<V>((R)1, (R)0);
                if (d >= 0) e = cexpi((R)(kappa * beta * dirs[3 * d + ax]) * xh[ax]);  // uniform branch
#pragma unroll
                for (int k = 0; k < L; ++k) W[ax][k] = cscale(cmul(e, T[ax][k]), S[ax][k]);
            }
            V va = cz<V>();
#pragma unroll
            for (int a = 0; a < L; ++a) {
                V vb = cz<V>();
#pragma unroll
                for (int b = 0; b < L; ++b) {
                    V vc = cz<V>();
#pragma unroll
                    for (int cc = 0; cc < L; ++cc) vc = cfma(loc[(a * L + b) * L + cc], W[2][cc], vc);
                    vb = cfma(vc, W[1][b], vb);
                }
                va = cfma(vb, W[0][a], va);
            }
            acc = cadd(acc, to_d(va));
        }
        if (valid) out[perm[p]] = from_d<V>(acc);
    }
}

// ---------------------------------------------------------------------------
// K1: P2P.  One CTA per target leaf; `split` threads per target share the
// sources (fixed-order shuffle reduction); source runs staged in shared
// memory.  Coordinate differences in FP64 (cell-relative accuracy for the
// FP32 path, SURVEY §7 hard part 6), kernel arithmetic in R, sums in FP64.

constexpr int P2P_NT = 128;
constexpr int P2P_TILE = 256;

__device__ __forceinline__ double2 helm_pair(double dx, double dy, double dz, double2 qs, double kpi,
                                             double tol) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double rinv = rsqrt(r2);  // r2 = 0 -> inf -> r = NaN -> masked below
    const double r = r2 * rinv;
    const bool ok = r >= tol;       // kernel.py:40-43 singularity suppression
    double s, c;
    sincospi(kpi * (ok ? r : 0.0), &s, &c);
    const double g = ok ? rinv * (1.0 / (4.0 * 3.141592653589793)) : 0.0;
    const double gr = g * c, gi = g * s;
    return make_double2(gr * qs.x - gi * qs.y, gr * qs.y + gi * qs.x);
}

// P2P-specific FP64 transcendental pieces.  The CUDA library rsqrt/sincospi
// cost ~128 issued instructions per pair in the P2P loop (64-bit polynomial
// constants rematerialised with UMOV pairs, special-case branches): with the
// coefficients in constant memory (DFMA reads them as c[][] operands) and no
// special cases (r2 = 0 is masked by the r >= tol test) the loop is bound by
// the FP64 pipe instead of instruction issue.
// sin(pi y) / y and cos(pi y) on |y| <= 1/4: Taylor coefficients (error
// < 2.3e-16 absolute, checked against libm), rounded to double.
__constant__ double c_sinpi[8] = {3.141592653589793, -5.16771278004997, 2.5501640398773455,
                                  -0.5992645293207921, 0.08214588661112823, -0.0073704309457143504,
                                  0.00046630280576761255, -2.1915353447830217e-05};
__constant__ double c_cospi[9] = {1.0, -4.934802200544679, 4.0587121264167685, -1.3352627688545895,
                                  0.2353306303588932, -0.02580689139001406, 0.0019295743094039231,
                                  -0.0001046381049248457, 4.303069587032947e-06};

// sin(pi x), cos(pi x) for 0 <= x < 2^50: x = y + n/2 with n = rint(2x) by the
// 1.5 * 2^52 trick (y exact, |y| <= 1/4), quadrant n mod 4.
__device__ __forceinline__ void sincospi_p2p(double x, double& s, double& c) {
    const double magic = 6755399441055744.0;
    const double t = fma(x, 2.0, magic);
    const int q = __double2loint(t);
    const double y = fma(t - magic, -0.5, x);
    const double y2 = y * y;
    double ps = c_sinpi[7];
#pragma unroll
    for (int k = 6; k >= 0; --k) ps = fma(ps, y2, c_sinpi[k]);
    double pc = c_cospi[8];
#pragma unroll
    for (int k = 7; k >= 0; --k) pc = fma(pc, y2, c_cospi[k]);
    const double sy = ps * y;
    const double ss = (q & 1) ? pc : sy, cc = (q & 1) ? sy : pc;
    // quadrant signs by XOR on the sign bit (a negation would be a DADD on the FP64 pipe,
    // the bound of this kernel, plus two selects)
    s = __hiloint2double(__double2hiint(ss) ^ ((q & 2) << 30), __double2loint(ss));
    c = __hiloint2double(__double2hiint(cc) ^ (((q + 1) & 2) << 30), __double2loint(cc));
}

// 1/sqrt(x): hardware approximation + one third-order Newton step
// (relative error O(d^3) from the ~2^-22 seed); x = 0 -> NaN (masked).
__device__ __forceinline__ double rsqrt_p2p(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);  // 1 - x y^2
    return fma(y * e, fma(0.375, e, 0.5), y);
}

__device__ __forceinline__ double2 helm_pair_p2p(double dx, double dy, double dz, double2 qs, double kpi,
                                                 double tol) {
    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const double rinv = rsqrt_p2p(r2);
    const double r = r2 * rinv;
    const bool ok = r >= tol;  // kernel.py:40-43 singularity suppression (NaN at r2 = 0 -> false)
    double s, c;
    sincospi_p2p(kpi * (ok ? r : 0.0), s, c);
    const double g = ok ? rinv : 0.0;  // 1/(4 pi) is folded into the staged charges
    const double gr = g * c, gi = g * s;
    return make_double2(gr * qs.x - gi * qs.y, gr * qs.y + gi * qs.x);
}

// Work items: a target leaf's flattened source list (its merged runs) is cut
// into pieces [f0, f1) of bounded size so that the few coarse leaves next to
// huge source cells (cfg3: up to 1.6 M sources) do not serialise the kernel.
// item_out < 0: the item is the leaf's only one and writes near[] directly;
// otherwise it writes nt partial sums at partial[item_out + (t - t0)],
// combined in fixed order by p2p_reduce_kernel.
struct P2PItems {
    const int32_t* leaf;
    const int64_t* f0;
    const int64_t* f1;
    const int64_t* out;
};

// One work item = targets [t0, t1) of a leaf against the sources [f0, f1) of
// its flattened run list (runs e in [e0, e1)).  Threads take a PAIR of
// targets each (every staged source feeds two pair evaluations from
// registers); when the leaf has fewer than P2P_NT pairs, `parts` =
// P2P_NT / pairs threads share a pair's sources (every parts-th source) and
// are reduced through shared memory in fixed part order (deterministic).
// Sources are staged in PACKED tiles of up to P2P_TILE (a tile may span
// several runs: cfg3/cfg5 leaves have 14-18 short runs), double-buffered: the
// next tile's global loads are issued before the current tile is consumed
// and stored after it, one barrier per tile.  The run table is staged in
// windows of P2P_MAXRUNS runs.
//   tgt(t) -> TS        target state (coordinates) of target t
//   load(g) -> Src      staged form of source g
//   pair(TS, Src, A&)   accumulate one pair
//   store(t, A)         write the item's result for target t
constexpr int P2P_MAXRUNS = 128;
constexpr int P2P_PER = P2P_TILE / P2P_NT;  // staged sources per thread and tile

template <typename Src, typename A, typename TGT, typename LOAD, typename PAIR, typename STORE>
__device__ __forceinline__ void p2p_item(int64_t t0, int64_t t1, int64_t e0, int64_t e1, int64_t f0, int64_t f1,
                                         const int64_t* __restrict__ src_lo, const int64_t* __restrict__ src_hi,
                                         Src (*tiles)[P2P_TILE], A (*red)[P2P_NT], int64_t* rlo, int64_t* rpre,
                                         TGT&& tgt, LOAD&& load, PAIR&& pair, STORE&& store) {
    const int64_t np_all = (t1 - t0 + 1) / 2;
    const int np = (int)(np_all < P2P_NT ? np_all : P2P_NT);
    const int parts = P2P_NT / np;
    const int pi = threadIdx.x % np, part = threadIdx.x / np;
    for (int64_t pb = 0; pb < np_all; pb += np) {
        const int64_t ta = t0 + 2 * (pb + pi), tb = ta + 1;
        const bool va = part < parts && ta < t1, vb = va && tb < t1;
        const auto TA = tgt(va ? ta : t0);
        const auto TB = tgt(vb ? tb : (va ? ta : t0));
        A acca{}, accb{};
        int64_t base = 0;  // flattened offset of the first run of the window
        for (int64_t w0 = e0; w0 < e1 && base < f1; w0 += P2P_MAXRUNS) {
            const int nr = (int)((e1 - w0) < P2P_MAXRUNS ? (e1 - w0) : P2P_MAXRUNS);
            __syncthreads();
            for (int k = threadIdx.x; k < nr; k += P2P_NT) {
                rlo[k] = src_lo[w0 + k];
                rpre[k + 1] = src_hi[w0 + k] - src_lo[w0 + k];
            }
            __syncthreads();
            if (threadIdx.x == 0) {  // inclusive prefix of the run lengths (<= 128 adds)
                int64_t acc = base;
                rpre[0] = base;
                for (int k = 1; k <= nr; ++k) {
                    acc += rpre[k];
                    rpre[k] = acc;
                }
            }
            __syncthreads();
            const int64_t wend = rpre[nr];
            const int64_t lo = f0 > base ? f0 : base, hi = f1 < wend ? f1 : wend;
            auto fetch = [&](int64_t fb, int cnt, Src (&v)[P2P_PER]) {
#pragma unroll
                for (int j = 0; j < P2P_PER; ++j) {
                    const int k = threadIdx.x + j * P2P_NT;
                    if (k < cnt) {
                        const int64_t g = fb + k;
                        int r = 0, top = nr;  // last run with rpre[r] <= g
                        while (top - r > 1) {
                            const int mid = (r + top) >> 1;
                            if (rpre[mid] <= g) r = mid; else top = mid;
                        }
                        v[j] = load(rlo[r] + (g - rpre[r]));
                    }
                }
            };
            auto put = [&](int buf, int cnt, const Src (&v)[P2P_PER]) {
#pragma unroll
                for (int j = 0; j < P2P_PER; ++j) {
                    const int k = threadIdx.x + j * P2P_NT;
                    if (k < cnt) tiles[buf][k] = v[j];
                }
            };
            if (lo < hi) {
                Src v[P2P_PER];
                int cnt = (int)((hi - lo) < P2P_TILE ? (hi - lo) : P2P_TILE);
                fetch(lo, cnt, v);
                put(0, cnt, v);
                __syncthreads();
                int buf = 0;
                for (int64_t fb = lo; fb < hi; fb += P2P_TILE) {
                    const int64_t fn = fb + P2P_TILE;
                    const int cn = fn < hi ? (int)((hi - fn) < P2P_TILE ? (hi - fn) : P2P_TILE) : 0;
                    if (cn) fetch(fn, cn, v);  // in flight while the current tile is consumed
                    if (va) {
                        const Src* tl = tiles[buf];
#pragma unroll 2
                        for (int k = part; k < cnt; k += parts) {
                            const Src sk = tl[k];
                            pair(TA, sk, acca);
                            pair(TB, sk, accb);
                        }
                    }
                    if (cn) put(buf ^ 1, cn, v);
                    __syncthreads();
                    buf ^= 1;
                    cnt = cn;
                }
            }
            base = wend;
        }
        red[0][threadIdx.x] = acca;
        red[1][threadIdx.x] = accb;
        __syncthreads();
        if (part == 0 && va) {
            A a = red[0][pi], b = red[1][pi];
            for (int q = 1; q < parts; ++q) {
                a = a + red[0][pi + q * np];
                b = b + red[1][pi + q * np];
            }
            store(ta, a);
            if (vb) store(tb, b);
        }
        __syncthreads();
    }
}

struct P2PAcc64 {  // FP64 complex partial sum
    double re, im;
    __device__ P2PAcc64 operator+(const P2PAcc64& o) const { return {re + o.re, im + o.im}; }
};
struct P2PAcc32 {
    float re, im;
    __device__ P2PAcc32 operator+(const P2PAcc32& o) const { return {re + o.re, im + o.im}; }
};
struct P2PSrc64 {  // source position + charge / (4 pi)
    double x, y, z;
    double2 q;
};
struct P2PTgt64 {
    double x, y, z;
};

#ifndef DEFMM_P2P_MINB64
#define DEFMM_P2P_MINB64 4
#endif
#ifndef DEFMM_P2P_MINB32
#define DEFMM_P2P_MINB32 8
#endif
template <typename R>
__global__ void __launch_bounds__(P2P_NT, DEFMM_P2P_MINB64) p2p_kernel(
    int64_t n, P2PItems it, const int64_t* __restrict__ tgt_lo, const int64_t* __restrict__ tgt_hi,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_lo,
    const int64_t* __restrict__ src_hi, const double* __restrict__ tx,
    const double* __restrict__ ty, const double* __restrict__ tz, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, const cx<R>* __restrict__ q,
    double kappa, double tol, cx<R>* __restrict__ near, cx<R>* __restrict__ partial) {
    using V = cx<R>;
    __shared__ P2PSrc64 tiles[2][P2P_TILE];
    __shared__ P2PAcc64 red[2][P2P_NT];
    __shared__ int64_t rlo[P2P_MAXRUNS], rpre[P2P_MAXRUNS + 1];
    const double inv4pi = 1.0 / (4.0 * 3.141592653589793);
    const double kpi = kappa / 3.141592653589793;
    for (int64_t item = blockIdx.x; item < n; item += gridDim.x) {
        const int leaf = it.leaf[item];
        const int64_t f0 = it.f0[item], f1 = it.f1[item], ob = it.out[item];
        const int64_t t0 = tgt_lo[leaf], t1 = tgt_hi[leaf];
        p2p_item(
            t0, t1, ptr[leaf], ptr[leaf + 1], f0, f1, src_lo, src_hi, tiles, red, rlo, rpre,
            [&](int64_t t) { return P2PTgt64{tx[t], ty[t], tz[t]}; },
            [&](int64_t g) {
                const double2 qq = to_d(q[g]);
                return P2PSrc64{px[g], py[g], pz[g], make_double2(qq.x * inv4pi, qq.y * inv4pi)};
            },
            [&](const P2PTgt64& t, const P2PSrc64& s, P2PAcc64& a) {
                const double2 g = helm_pair_p2p(t.x - s.x, t.y - s.y, t.z - s.z, s.q, kpi, tol);
                a.re += g.x;
                a.im += g.y;
            },
            [&](int64_t t, const P2PAcc64& a) {
                const V v = from_d<V>(make_double2(a.re, a.im));
                if (ob < 0) near[t] = v;
                else partial[ob + (t - t0)] = v;
            });
    }
}

// near[t] = sum_m partial[base + m * nt + (t - t0)] for the split leaves
template <typename R>
__global__ void __launch_bounds__(128) p2p_reduce_kernel(int64_t n, const int32_t* __restrict__ leaf,
                                                         const int64_t* __restrict__ base,
                                                         const int32_t* __restrict__ nitems,
                                                         const int64_t* __restrict__ tgt_lo,
                                                         const int64_t* __restrict__ tgt_hi,
                                                         const cx<R>* __restrict__ partial,
                                                         cx<R>* __restrict__ near) {
    const int64_t i = blockIdx.x;
    const int l = leaf[i];
    const int64_t t0 = tgt_lo[l], nt = tgt_hi[l] - t0;
    const int k = nitems[i];
    for (int64_t x = threadIdx.x; x < nt; x += blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
        for (int m = 0; m < k; ++m) acc = cadd(acc, to_d(partial[base[i] + m * nt + x]));
        near[t0 + x] = from_d<cx<R>>(acc);
    }
}

// complex64 near field in TARGET-RELATIVE coordinates: every item stages its
// sources as FP32 offsets from a reference point c of its target leaf (the
// leaf's first target), formed in FP64 before rounding, and its targets the
// same way (SURVEY §7 hard part 6: cell-relative coordinates).
//   HILO = false: one float per offset, dx = x'_t - x'_s is one FADD; the
//     offset rounding (2^-25 |x_s - c|) bounds the near-field floor at a few
//     1e-7 -- enough for L <= 5, whose c64 bar is >= ~1e-5.
//   HILO = true: hi/lo float pairs per offset, dx = (x'h_t - x'h_s) +
//     (x'l_t - x'l_s) (three FADDs) -- float rounding of dx itself, needed by
//     the L >= 6 bar (cfg2 L6: 3.1e-6).
// Charges are staged pre-scaled by 1/(4 pi).  e^{i kappa r} via the reduction
// of u = kappa r / (2 pi) to [-1/2, 1/2] and the hardware sin/cos (abs. error
// < 4e-7 on [-pi, pi]); FP32 partial sums per thread, combined with a
// fixed-order shuffle.
__device__ __forceinline__ float rsqrt_approx(float x) {  // MUFU.RSQ without denormal fix-ups
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <bool HILO>
struct P2PF32Src;
template <>
struct P2PF32Src<false> {  // (x', y', z', q.re / 4 pi), q.im / 4 pi
    float4 a;
    float qi;
};
template <>
struct P2PF32Src<true> {  // hi (x, y, z, q.re / 4 pi), lo (x, y, z, q.im / 4 pi)
    float4 a, b;
};

// target offsets: hi in x[0..2], lo in x[3..5] (HILO only)
template <bool HILO>
__device__ __forceinline__ void pair_f32(const float (&t)[6], const P2PF32Src<HILO>& s, float k2pi, float ftol,
                                         float& ar, float& ai) {
    float dx, dy, dz, qr, qi;
    if constexpr (HILO) {
        dx = (t[0] - s.a.x) + (t[3] - s.b.x);
        dy = (t[1] - s.a.y) + (t[4] - s.b.y);
        dz = (t[2] - s.a.z) + (t[5] - s.b.z);
        qr = s.a.w;
        qi = s.b.w;
    } else {
        dx = t[0] - s.a.x;
        dy = t[1] - s.a.y;
        dz = t[2] - s.a.z;
        qr = s.a.w;
        qi = s.qi;
    }
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float rinv = rsqrt_approx(r2);  // r2 = 0 -> inf -> r = NaN -> masked
    const float r = r2 * rinv;
    const bool ok = r >= ftol;
    float u = k2pi * (ok ? r : 0.0f);
    // u - rint(u) by the 1.5 * 2^23 round-to-nearest trick: two FADDs on the
    // FMA pipe instead of FRND on the XU pipe; exact for |u| < 2^22 (the
    // near-field kappa r / 2 pi is far below)
    u -= __fsub_rn(__fadd_rn(u, 12582912.0f), 12582912.0f);
    float sn, cs;
    __sincosf(6.283185307179586f * u, &sn, &cs);
    const float g = ok ? rinv : 0.0f;
    const float gr = g * cs, gi = g * sn;
    ar = fmaf(gr, qr, fmaf(-gi, qi, ar));
    ai = fmaf(gr, qi, fmaf(gi, qr, ai));
}

template <bool HILO>
__device__ __forceinline__ void rel_f32(double x, double c, float& hi, float& lo) {
    const double d = x - c;
    hi = __double2float_rn(d);
    lo = HILO ? __double2float_rn(d - (double)hi) : 0.0f;
}

template <bool HILO>
struct P2PTgt32 {
    float t[6];  // offsets: hi x, y, z, then lo x, y, z (HILO)
};

template <bool HILO>
__global__ void __launch_bounds__(P2P_NT, DEFMM_P2P_MINB32) p2p_f32_kernel(
    int64_t n, P2PItems it, const int64_t* __restrict__ tgt_lo, const int64_t* __restrict__ tgt_hi,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_lo,
    const int64_t* __restrict__ src_hi, const double* __restrict__ tx,
    const double* __restrict__ ty, const double* __restrict__ tz, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, const float2* __restrict__ q,
    double kappa, double tol, float2* __restrict__ near, float2* __restrict__ partial) {
    __shared__ P2PF32Src<HILO> tiles[2][P2P_TILE];
    __shared__ P2PAcc32 red[2][P2P_NT];
    __shared__ int64_t rlo[P2P_MAXRUNS], rpre[P2P_MAXRUNS + 1];
    const float k2pi = (float)(kappa / (2.0 * 3.141592653589793));
    const float ftol = (float)tol;
    const float inv4pi = (float)(1.0 / (4.0 * 3.141592653589793));
    for (int64_t item = blockIdx.x; item < n; item += gridDim.x) {
        const int leaf = it.leaf[item];
        const int64_t f0 = it.f0[item], f1 = it.f1[item], ob = it.out[item];
        const int64_t t0 = tgt_lo[leaf], t1 = tgt_hi[leaf];
        const double cx = tx[t0], cy = ty[t0], cz = tz[t0];  // reference point of the item
        p2p_item(
            t0, t1, ptr[leaf], ptr[leaf + 1], f0, f1, src_lo, src_hi, tiles, red, rlo, rpre,
            [&](int64_t t) {
                P2PTgt32<HILO> T;
                rel_f32<HILO>(tx[t], cx, T.t[0], T.t[3]);
                rel_f32<HILO>(ty[t], cy, T.t[1], T.t[4]);
                rel_f32<HILO>(tz[t], cz, T.t[2], T.t[5]);
                return T;
            },
            [&](int64_t g) {
                const float2 qq = q[g];
                P2PF32Src<HILO> v;
                float lx, ly, lz;
                rel_f32<HILO>(px[g], cx, v.a.x, lx);
                rel_f32<HILO>(py[g], cy, v.a.y, ly);
                rel_f32<HILO>(pz[g], cz, v.a.z, lz);
                v.a.w = qq.x * inv4pi;
                if constexpr (HILO) {
                    v.b = make_float4(lx, ly, lz, qq.y * inv4pi);
                } else {
                    v.qi = qq.y * inv4pi;
                }
                return v;
            },
            [&](const P2PTgt32<HILO>& T, const P2PF32Src<HILO>& s, P2PAcc32& a) {
                pair_f32<HILO>(T.t, s, k2pi, ftol, a.re, a.im);
            },
            [&](int64_t t, const P2PAcc32& a) {
                const float2 v = make_float2(a.re, a.im);
                if (ob < 0) near[t] = v;
                else partial[ob + (t - t0)] = v;
            });
    }
}

// ---------------------------------------------------------------------------
// K1 v2: MUTUAL P2P (single-tree plans).  G(|x_t - x_s|) is symmetric, and in
// single-tree mode the near-field relation is too: s is in the source list of
// t's leaf iff t is in the list of s's leaf.  An item here is a target leaf A
// against a piece of its source list CLIPPED to particles >= A's first one:
// first A itself (evaluated one-directionally, every ordered pair), then the
// leaves after A in Morton order, for which every evaluated G feeds BOTH the
// row sum of its target (registers, as in K1) and the column sum of its
// source, G q_t.  Column sums are accumulated in per-warp shared-memory copies
// (plain read-add-write: the threads of a warp visit distinct sources at every
// step -- thread pi starts at source pi of its part and rotates), merged in
// fixed warp order after every tile and written to partial[]; p2p_gather then
// sums, for every particle, the row partials of its own leaf's items and the
// column partials of the items that listed it, in list order (no atomics:
// reruns are bitwise identical).  Half the kernel evaluations of K1.
constexpr int P2P_WARPS = P2P_NT / 32;

template <typename Src, typename TILES, typename A, typename TGT, typename MUTE, typename LOAD, typename PAIR,
          typename STORE>
__device__ __forceinline__ void p2p_item_mut(int64_t t0, int64_t t1, int64_t e0, int64_t e1, int64_t f0, int64_t f1,
                                             const int64_t* __restrict__ src_lo,
                                             const int64_t* __restrict__ src_hi, TILES& tiles,
                                             A (*col)[P2P_TILE], A (*red)[P2P_NT], int64_t* rlo, int64_t* rpre,
                                             TGT&& tgt, MUTE&& mute, LOAD&& load, PAIR&& pair, STORE&& store_row,
                                             A* __restrict__ colout) {
    const int64_t np_all = (t1 - t0 + 1) / 2;  // <= P2P_NT (checked by the host)
    const int np = (int)np_all;
    const int parts = P2P_NT / np;
    const int pi = threadIdx.x % np, part = threadIdx.x / np;
    const int warp = threadIdx.x >> 5;
    const int64_t ta = t0 + 2 * pi, tb = ta + 1;
    const bool va = part < parts && ta < t1, vb = va && tb < t1;
    const auto TA = tgt(va ? ta : t0);
    auto TB = tgt(vb ? tb : (va ? ta : t0));
    if (!vb) mute(TB);  // an absent second target adds nothing to the column sums
    A acca{}, accb{};
    int64_t base = 0;  // flattened offset of the first run of the window (col[][] is all zero here)
    for (int64_t w0 = e0; w0 < e1 && base < f1; w0 += P2P_MAXRUNS) {
        const int nr = (int)((e1 - w0) < P2P_MAXRUNS ? (e1 - w0) : P2P_MAXRUNS);
        __syncthreads();
        for (int k = threadIdx.x; k < nr; k += P2P_NT) {
            rlo[k] = src_lo[w0 + k];
            rpre[k + 1] = src_hi[w0 + k] - src_lo[w0 + k];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t acc = base;
            rpre[0] = base;
            for (int k = 1; k <= nr; ++k) {
                acc += rpre[k];
                rpre[k] = acc;
            }
        }
        __syncthreads();
        const int64_t wend = rpre[nr];
        const int64_t lo = f0 > base ? f0 : base, hi = f1 < wend ? f1 : wend;
        auto fetch = [&](int64_t fb, int cnt, Src (&v)[P2P_PER]) {
#pragma unroll
            for (int j = 0; j < P2P_PER; ++j) {
                const int k = threadIdx.x + j * P2P_NT;
                if (k < cnt) {
                    const int64_t g = fb + k;
                    int r = 0, top = nr;  // last run with rpre[r] <= g
                    while (top - r > 1) {
                        const int mid = (r + top) >> 1;
                        if (rpre[mid] <= g) r = mid; else top = mid;
                    }
                    v[j] = load(rlo[r] + (g - rpre[r]));
                }
            }
        };
        auto put = [&](int buf, int cnt, const Src (&v)[P2P_PER]) {
#pragma unroll
            for (int j = 0; j < P2P_PER; ++j) {
                const int k = threadIdx.x + j * P2P_NT;
                if (k < cnt) tiles.put(buf, k, v[j]);
            }
        };
        if (lo < hi) {
            Src v[P2P_PER];
            int cnt = (int)((hi - lo) < P2P_TILE ? (hi - lo) : P2P_TILE);
            fetch(lo, cnt, v);
            put(0, cnt, v);
            __syncthreads();
            int buf = 0;
            for (int64_t fb = lo; fb < hi; fb += P2P_TILE) {
                const int64_t fn = fb + P2P_TILE;
                const int cn = fn < hi ? (int)((hi - fn) < P2P_TILE ? (hi - fn) : P2P_TILE) : 0;
                if (cn) fetch(fn, cn, v);  // in flight while the current tile is consumed
                if (va) {
                    A* cw = col[warp];
                    // part p owns the block [p B, (p + 1) B) of the tile's sources; thread pi
                    // starts at the pi-th of them and rotates over M >= np positions, so the
                    // threads of a warp touch distinct, consecutive sources at every step
                    // (conflict-free reads of the SoA tile and of the column sums)
                    const int B = (cnt + parts - 1) / parts;
                    const int k0 = part * B;
                    const int mp = cnt > k0 ? (cnt - k0 < B ? cnt - k0 : B) : 0;
                    if (mp >= np) {
                        // every position is a source: two of them per step with separate row
                        // sums (four independent kernel evaluations in flight per thread)
                        int idx = pi;
                        int jj = 0;
                        A a2{}, b2{};
                        for (; jj + 2 <= mp; jj += 2) {
                            const int i0 = idx, i1 = idx + 1 == mp ? 0 : idx + 1;
                            idx = i1 + 1 == mp ? 0 : i1 + 1;
                            const Src s0 = tiles.get(buf, k0 + i0), s1 = tiles.get(buf, k0 + i1);
                            A c0{}, c1{};
                            pair(TA, s0, acca, c0);
                            pair(TA, s1, a2, c1);
                            pair(TB, s0, accb, c0);
                            pair(TB, s1, b2, c1);
                            cw[k0 + i0] = cw[k0 + i0] + c0;
                            cw[k0 + i1] = cw[k0 + i1] + c1;
                        }
                        if (jj < mp) {
                            const Src s0 = tiles.get(buf, k0 + idx);
                            A c0{};
                            pair(TA, s0, acca, c0);
                            pair(TB, s0, accb, c0);
                            cw[k0 + idx] = cw[k0 + idx] + c0;
                        }
                        acca = acca + a2;
                        accb = accb + b2;
                    } else {  // fewer sources than target pairs: idle positions keep the threads apart
                        int idx = pi;
                        for (int jj = 0; jj < np; ++jj) {
                            if (idx < mp) {
                                const Src sk = tiles.get(buf, k0 + idx);
                                A cv{};
                                pair(TA, sk, acca, cv);
                                pair(TB, sk, accb, cv);
                                cw[k0 + idx] = cw[k0 + idx] + cv;
                            }
                            if (++idx == np) idx = 0;
                        }
                    }
                }
                if (cn) put(buf ^ 1, cn, v);
                __syncthreads();
                // column sums of the tile: warp copies merged in fixed order, then cleared
                for (int k = threadIdx.x; k < cnt; k += P2P_NT) {
                    A sum = col[0][k];
                    col[0][k] = A{};
#pragma unroll
                    for (int w = 1; w < P2P_WARPS; ++w) {
                        sum = sum + col[w][k];
                        col[w][k] = A{};
                    }
                    colout[(fb - f0) + k] = sum;
                }
                __syncthreads();
                buf ^= 1;
                cnt = cn;
            }
        }
        base = wend;
    }
    red[0][threadIdx.x] = acca;
    red[1][threadIdx.x] = accb;
    __syncthreads();
    if (part == 0 && va) {
        A a = red[0][pi], b = red[1][pi];
        for (int q = 1; q < parts; ++q) {
            a = a + red[0][pi + q * np];
            b = b + red[1][pi + q * np];
        }
        store_row(ta, a);
        if (vb) store_row(tb, b);
    }
    __syncthreads();
}

// source tiles of the mutual kernels in SoA form (lanes read consecutive sources)
struct P2PTiles64 {
    double x[2][P2P_TILE], y[2][P2P_TILE], z[2][P2P_TILE];
    double2 q[2][P2P_TILE];
    __device__ __forceinline__ void put(int b, int k, const P2PSrc64& s) {
        x[b][k] = s.x;
        y[b][k] = s.y;
        z[b][k] = s.z;
        q[b][k] = s.q;
    }
    __device__ __forceinline__ P2PSrc64 get(int b, int k) const { return P2PSrc64{x[b][k], y[b][k], z[b][k], q[b][k]}; }
};

struct P2PTgt64q {  // target position + its charge / (4 pi)
    double x, y, z;
    double2 q;
};

// G(r) feeds the row sum (source charge) and the column sum (target charge)
__device__ __forceinline__ void helm_pair_mut(double dx, double dy, double dz, double2 qs, double2 qt, double kpi,
                                              double tol, P2PAcc64& row, P2PAcc64& colv) {
    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
    const double rinv = rsqrt_p2p(r2);
    const double r = r2 * rinv;
    const bool ok = r >= tol;  // kernel.py:40-43 (NaN at r2 = 0 -> false)
    double s, c;
    sincospi_p2p(kpi * (ok ? r : 0.0), s, c);
    const double g = ok ? rinv : 0.0;
    const double gr = g * c, gi = g * s;
    row.re = fma(gr, qs.x, fma(-gi, qs.y, row.re));
    row.im = fma(gr, qs.y, fma(gi, qs.x, row.im));
    colv.re = fma(gr, qt.x, fma(-gi, qt.y, colv.re));
    colv.im = fma(gr, qt.y, fma(gi, qt.x, colv.im));
}

struct P2PMutItems {
    const int32_t* leaf;
    const int64_t* f0;
    const int64_t* f1;
    const int64_t* row;  // partial[] offset of the item's nt row sums
    const int64_t* col;  // partial[] offset of its f1 - f0 column sums
};

#ifndef DEFMM_P2P_MUT_MINB64
#define DEFMM_P2P_MUT_MINB64 4
#endif
template <typename R>
__global__ void __launch_bounds__(P2P_NT, DEFMM_P2P_MUT_MINB64) p2p_mut_kernel(
    int64_t n, P2PMutItems it, const int64_t* __restrict__ tgt_lo, const int64_t* __restrict__ tgt_hi,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_lo,
    const int64_t* __restrict__ src_hi, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, const cx<R>* __restrict__ q, double kappa, double tol,
    double2* __restrict__ partial) {
    __shared__ P2PTiles64 tiles;
    __shared__ P2PAcc64 col[P2P_WARPS][P2P_TILE];
    __shared__ P2PAcc64 red[2][P2P_NT];
    __shared__ int64_t rlo[P2P_MAXRUNS], rpre[P2P_MAXRUNS + 1];
    const double inv4pi = 1.0 / (4.0 * 3.141592653589793);
    const double kpi = kappa / 3.141592653589793;
    for (int k = threadIdx.x; k < P2P_WARPS * P2P_TILE; k += P2P_NT) col[0][k] = P2PAcc64{};  // kept zero by the flushes
    for (int64_t item = blockIdx.x; item < n; item += gridDim.x) {
        const int leaf = it.leaf[item];
        const int64_t f0 = it.f0[item], f1 = it.f1[item], rb = it.row[item];
        const int64_t t0 = tgt_lo[leaf], t1 = tgt_hi[leaf];
        p2p_item_mut<P2PSrc64>(
            t0, t1, ptr[leaf], ptr[leaf + 1], f0, f1, src_lo, src_hi, tiles, col, red, rlo, rpre,
            [&](int64_t t) {
                const double2 qq = to_d(q[t]);
                return P2PTgt64q{px[t], py[t], pz[t], make_double2(qq.x * inv4pi, qq.y * inv4pi)};
            },
            [](P2PTgt64q& T) { T.q = make_double2(0.0, 0.0); },
            [&](int64_t g) {
                const double2 qq = to_d(q[g]);
                return P2PSrc64{px[g], py[g], pz[g], make_double2(qq.x * inv4pi, qq.y * inv4pi)};
            },
            [&](const P2PTgt64q& t, const P2PSrc64& s, P2PAcc64& a, P2PAcc64& cv) {
                helm_pair_mut(t.x - s.x, t.y - s.y, t.z - s.z, s.q, t.q, kpi, tol, a, cv);
            },
            [&](int64_t t, const P2PAcc64& a) { partial[rb + (t - t0)] = make_double2(a.re, a.im); },
            reinterpret_cast<P2PAcc64*>(partial + it.col[item]));
    }
}

template <bool HILO>
struct P2PTiles32;
template <>
struct P2PTiles32<false> {
    float4 a[2][P2P_TILE];
    float qi[2][P2P_TILE];
    __device__ __forceinline__ void put(int b, int k, const P2PF32Src<false>& s) {
        a[b][k] = s.a;
        qi[b][k] = s.qi;
    }
    __device__ __forceinline__ P2PF32Src<false> get(int b, int k) const {
        P2PF32Src<false> s;
        s.a = a[b][k];
        s.qi = qi[b][k];
        return s;
    }
};
template <>
struct P2PTiles32<true> {
    float4 a[2][P2P_TILE], bb[2][P2P_TILE];
    __device__ __forceinline__ void put(int b, int k, const P2PF32Src<true>& s) {
        a[b][k] = s.a;
        bb[b][k] = s.b;
    }
    __device__ __forceinline__ P2PF32Src<true> get(int b, int k) const {
        P2PF32Src<true> s;
        s.a = a[b][k];
        s.b = bb[b][k];
        return s;
    }
};

template <bool HILO>
struct P2PTgt32q {
    float t[6];  // offsets: hi x, y, z, then lo x, y, z (HILO)
    float qr, qi;  // charge / (4 pi)
};

template <bool HILO>
__device__ __forceinline__ void pair_f32_mut(const P2PTgt32q<HILO>& T, const P2PF32Src<HILO>& s, float k2pi,
                                             float ftol, P2PAcc32& row, P2PAcc32& colv) {
    float dx, dy, dz, qr, qi;
    if constexpr (HILO) {
        dx = (T.t[0] - s.a.x) + (T.t[3] - s.b.x);
        dy = (T.t[1] - s.a.y) + (T.t[4] - s.b.y);
        dz = (T.t[2] - s.a.z) + (T.t[5] - s.b.z);
        qr = s.a.w;
        qi = s.b.w;
    } else {
        dx = T.t[0] - s.a.x;
        dy = T.t[1] - s.a.y;
        dz = T.t[2] - s.a.z;
        qr = s.a.w;
        qi = s.qi;
    }
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float rinv = rsqrt_approx(r2);  // r2 = 0 -> inf -> r = NaN -> masked
    const float r = r2 * rinv;
    const bool ok = r >= ftol;
    float u = k2pi * (ok ? r : 0.0f);
    u -= __fsub_rn(__fadd_rn(u, 12582912.0f), 12582912.0f);
    float sn, cs;
    __sincosf(6.283185307179586f * u, &sn, &cs);
    const float g = ok ? rinv : 0.0f;
    const float gr = g * cs, gi = g * sn;
    row.re = fmaf(gr, qr, fmaf(-gi, qi, row.re));
    row.im = fmaf(gr, qi, fmaf(gi, qr, row.im));
    colv.re = fmaf(gr, T.qr, fmaf(-gi, T.qi, colv.re));
    colv.im = fmaf(gr, T.qi, fmaf(gi, T.qr, colv.im));
}

template <bool HILO>
__global__ void __launch_bounds__(P2P_NT, DEFMM_P2P_MINB32) p2p_mut_f32_kernel(
    int64_t n, P2PMutItems it, const int64_t* __restrict__ tgt_lo, const int64_t* __restrict__ tgt_hi,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_lo,
    const int64_t* __restrict__ src_hi, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, const float2* __restrict__ q, double kappa, double tol,
    float2* __restrict__ partial) {
    __shared__ P2PTiles32<HILO> tiles;
    __shared__ P2PAcc32 col[P2P_WARPS][P2P_TILE];
    __shared__ P2PAcc32 red[2][P2P_NT];
    __shared__ int64_t rlo[P2P_MAXRUNS], rpre[P2P_MAXRUNS + 1];
    const float k2pi = (float)(kappa / (2.0 * 3.141592653589793));
    const float ftol = (float)tol;
    const float inv4pi = (float)(1.0 / (4.0 * 3.141592653589793));
    for (int k = threadIdx.x; k < P2P_WARPS * P2P_TILE; k += P2P_NT) col[0][k] = P2PAcc32{};  // kept zero by the flushes
    for (int64_t item = blockIdx.x; item < n; item += gridDim.x) {
        const int leaf = it.leaf[item];
        const int64_t f0 = it.f0[item], f1 = it.f1[item], rb = it.row[item];
        const int64_t t0 = tgt_lo[leaf], t1 = tgt_hi[leaf];
        const double cx = px[t0], cy = py[t0], cz = pz[t0];  // reference point of the item
        p2p_item_mut<P2PF32Src<HILO>>(
            t0, t1, ptr[leaf], ptr[leaf + 1], f0, f1, src_lo, src_hi, tiles, col, red, rlo, rpre,
            [&](int64_t t) {
                P2PTgt32q<HILO> T;
                rel_f32<HILO>(px[t], cx, T.t[0], T.t[3]);
                rel_f32<HILO>(py[t], cy, T.t[1], T.t[4]);
                rel_f32<HILO>(pz[t], cz, T.t[2], T.t[5]);
                const float2 qq = q[t];
                T.qr = qq.x * inv4pi;
                T.qi = qq.y * inv4pi;
                return T;
            },
            [](P2PTgt32q<HILO>& T) { T.qr = T.qi = 0.0f; },
            [&](int64_t g) {
                const float2 qq = q[g];
                P2PF32Src<HILO> v;
                float lx, ly, lz;
                rel_f32<HILO>(px[g], cx, v.a.x, lx);
                rel_f32<HILO>(py[g], cy, v.a.y, ly);
                rel_f32<HILO>(pz[g], cz, v.a.z, lz);
                v.a.w = qq.x * inv4pi;
                if constexpr (HILO) {
                    v.b = make_float4(lx, ly, lz, qq.y * inv4pi);
                } else {
                    v.qi = qq.y * inv4pi;
                }
                return v;
            },
            [&](const P2PTgt32q<HILO>& T, const P2PF32Src<HILO>& s, P2PAcc32& a, P2PAcc32& cv) {
                pair_f32_mut<HILO>(T, s, k2pi, ftol, a, cv);
            },
            [&](int64_t t, const P2PAcc32& a) { partial[rb + (t - t0)] = make_float2(a.re, a.im); },
            reinterpret_cast<P2PAcc32*>(partial + it.col[item]));
    }
}

// Gather task j (leaf l = task_leaf[j]): out[x] = sum over its contributor
// segments c in [cptr[j], cptr[j+1]) (in list order) of partial[cbase[c] + x],
// xlo[c] <= x < xhi[c]; out = near + tgt_lo[l] when task_out[j] < 0, else
// partial + task_out[j] (a pre-sum row read by a later pass).  FP64 sums.
template <typename R>
__global__ void __launch_bounds__(64) p2p_gather_kernel(int64_t n, const int32_t* __restrict__ task_leaf,
                                                        const int64_t* __restrict__ task_out,
                                                        const int64_t* __restrict__ tgt_lo,
                                                        const int64_t* __restrict__ tgt_hi,
                                                        const int64_t* __restrict__ cptr,
                                                        const int64_t* __restrict__ cbase,
                                                        const int32_t* __restrict__ cxlo,
                                                        const int32_t* __restrict__ cxhi, cx<R>* partial,
                                                        cx<R>* __restrict__ near) {
    const int64_t j = blockIdx.x;
    const int l = task_leaf[j];
    const int64_t t0 = tgt_lo[l];
    const int nt = (int)(tgt_hi[l] - t0);
    const int64_t ob = task_out[j];
    cx<R>* out = ob < 0 ? near + t0 : partial + ob;
    const int64_t c0 = cptr[j], c1 = cptr[j + 1];
    for (int x = threadIdx.x; x < nt; x += blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t c = c0; c < c1; ++c) {
            if (x >= __ldg(cxlo + c) && x < __ldg(cxhi + c)) acc = cadd(acc, to_d(partial[__ldg(cbase + c) + x]));
        }
        out[x] = from_d<cx<R>>(acc);
    }
}

// K10: direct sum (FP64).  Sources are split over blockIdx.y so that a few
// thousand check targets still fill the GPU; partial sums land in
// part[blockIdx.y][target] and are reduced in a fixed order by direct_reduce.
constexpr int DIRECT_SPLIT = 64;

__global__ void __launch_bounds__(128) direct_kernel(
    int64_t nt, const double* __restrict__ tx, const double* __restrict__ ty,
    const double* __restrict__ tz, int64_t ns, const double* __restrict__ sx,
    const double* __restrict__ sy, const double* __restrict__ sz, const double2* __restrict__ q,
    double kappa, double tol, double2* __restrict__ part) {
    __shared__ double ax[256], ay[256], az[256];
    __shared__ double2 aq[256];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = t < nt;
    const double x = valid ? tx[t] : 0.0, y = valid ? ty[t] : 0.0, z = valid ? tz[t] : 0.0;
    const double kpi = kappa / 3.141592653589793;
    const int64_t chunk = (ns + gridDim.y - 1) / gridDim.y;
    const int64_t lo = blockIdx.y * chunk, hi = (lo + chunk) < ns ? lo + chunk : ns;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t sb = lo; sb < hi; sb += 256) {
        const int cnt = (int)((hi - sb) < 256 ? (hi - sb) : 256);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
            ax[k] = sx[sb + k];
            ay[k] = sy[sb + k];
            az[k] = sz[sb + k];
            aq[k] = q[sb + k];
        }
        __syncthreads();
        if (valid)
            for (int k = 0; k < cnt; ++k) {
                const double2 g = helm_pair(x - ax[k], y - ay[k], z - az[k], aq[k], kpi, tol);
                acc.x += g.x;
                acc.y += g.y;
            }
    }
    if (valid) part[blockIdx.y * nt + t] = acc;
}

__global__ void direct_reduce(int64_t nt, int nsplit, const double2* __restrict__ part,
                              double2* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < nsplit; ++k) acc = cadd(acc, part[k * nt + t]);
    out[t] = acc;
}

// ---------------------------------------------------------------------------
// launch helpers

struct HostLayout {
    int P3 = 0, nslices = 0;
    std::vector<int16_t> forder, finv;
    std::vector<int32_t> start;
};

// orbit-ordered spectral layout of order L (see g_forder): orbits keyed by the
// sorted per-axis |frequency| (min(f, P - f)), enumerated in key order,
// packed first-fit-decreasing into slices of <= SLICE_W positions
HostLayout make_layout(int L) {
    HostLayout H;
    const int P = 2 * L - 1, P3 = P * P * P;
    H.P3 = P3;
    std::vector<std::vector<int>> orbits;
    std::vector<int> key_of(P3);
    const int A = P / 2 + 1;
    std::vector<int> orbit_of_key(A * A * A, -1);
    for (int j = 0; j < P3; ++j) {
        int a[3] = {j / (P * P), (j / P) % P, j % P};
        for (int& x : a) x = std::min(x, P - x);
        std::sort(a, a + 3);
        key_of[j] = (a[0] * A + a[1]) * A + a[2];
    }
    for (int k = 0; k < A * A * A; ++k)
        for (int j = 0; j < P3; ++j)
            if (key_of[j] == k) {
                if (orbit_of_key[k] < 0) {
                    orbit_of_key[k] = (int)orbits.size();
                    orbits.emplace_back();
                }
                orbits[orbit_of_key[k]].push_back(j);
            }
    // orbit 0 = the zero frequency (key 0): packed last, alone at the end
    std::vector<int> order;
    for (size_t i = 1; i < orbits.size(); ++i) order.push_back((int)i);
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return orbits[x].size() > orbits[y].size(); });
    std::vector<std::vector<int>> bins;
    std::vector<int> fill;
    for (int o : order) {
        const int sz = (int)orbits[o].size();
        size_t b = 0;
        while (b < bins.size() && fill[b] + sz > SLICE_W) ++b;
        if (b == bins.size()) {
            bins.emplace_back();
            fill.push_back(0);
        }
        bins[b].push_back(o);
        fill[b] += sz;
    }
    // the zero orbit goes into the least-filled bin, which is moved last
    size_t zb = 0;
    for (size_t b = 1; b < bins.size(); ++b)
        if (fill[b] < fill[zb]) zb = b;
    if (bins.empty() || fill[zb] + 1 > SLICE_W) {
        bins.emplace_back();
        fill.push_back(0);
        zb = bins.size() - 1;
    }
    bins[zb].push_back(0);
    fill[zb] += 1;
    std::rotate(bins.begin() + zb, bins.begin() + zb + 1, bins.end());
    H.nslices = (int)bins.size();
    H.forder.resize(P3);
    H.finv.resize(P3);
    H.start.assign(1, 0);
    int pos = 0;
    for (const auto& b : bins) {
        for (int o : b)
            for (int j : orbits[o]) H.forder[pos++] = (int16_t)j;
        H.start.push_back(pos);
    }
    for (int t = 0; t < P3; ++t) H.finv[H.forder[t]] = (int16_t)t;
    return H;
}

const HostLayout& layout_of(int L) {
    static HostLayout cache[9];
    static bool made[9] = {};
    if (!made[L]) {
        cache[L] = make_layout(L);
        made[L] = true;
    }
    return cache[L];
}

// device tables (spectral layout, twiddles) are per device: filled once per
// device the process launches on (keyed by the current device)
int ensure_twiddles() {
    constexpr int MAX_DEV = 64;
    static bool done[MAX_DEV] = {};
    int dev = 0;
    if (int rc = report(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
    if (dev < 0 || dev >= MAX_DEV) return report(cudaErrorInvalidDevice, "ensure_twiddles: device index");
    if (done[dev]) return 0;
    for (int L = 2; L <= 8; ++L) {
        const HostLayout& H = layout_of(L);
        if (H.nslices > MAX_SLICES) return report(cudaErrorInvalidValue, "spectral layout: too many slices");
        const size_t o = (size_t)(L - 1);
        int rc = report(cudaMemcpyToSymbol(g_forder, H.forder.data(), H.P3 * sizeof(int16_t),
                                           o * MAX_P3 * sizeof(int16_t)), "cudaMemcpyToSymbol(g_forder)");
        if (!rc)
            rc = report(cudaMemcpyToSymbol(g_finv, H.finv.data(), H.P3 * sizeof(int16_t),
                                           o * MAX_P3 * sizeof(int16_t)), "cudaMemcpyToSymbol(g_finv)");
        if (rc) return rc;
    }
    double2 h[8][15] = {};
    for (int L = 2; L <= 8; ++L) {
        const int P = 2 * L - 1;
        for (int k = 0; k < P; ++k) {
            const double a = 2.0 * 3.14159265358979323846 * (double)k / (double)P;
            h[L - 1][k] = make_double2(cos(a), -sin(a));
        }
    }
    int rc = report(cudaMemcpyToSymbol(c_tw, h, sizeof(h)), "cudaMemcpyToSymbol(c_tw)");
    if (rc == 0) {  // the bit-0 interpolation factors, the arithmetic of make_factor_tables
        static double a0[8][64];
        static float a0f[8][64];
        for (int L = 2; L <= 8; ++L)
            for (int k = 0; k < L; ++k)
                for (int j = 0; j < L; ++j) {
                    const double x = (0.0 + (double)j / (double)(L - 1)) / 2.0;
                    double v = 1.0;
                    for (int m = 0; m < L; ++m)
                        if (m != k)
                            v = v * (x - (double)m / (double)(L - 1)) /
                                ((double)k / (double)(L - 1) - (double)m / (double)(L - 1));
                    a0[L - 1][k * L + j] = v;
                    a0f[L - 1][k * L + j] = (float)v;
                }
        rc = report(cudaMemcpyToSymbol(c_a0, a0, sizeof(a0)), "cudaMemcpyToSymbol(c_a0)");
        if (rc == 0) rc = report(cudaMemcpyToSymbol(c_a0f, a0f, sizeof(a0f)), "cudaMemcpyToSymbol(c_a0f)");
    }
    if (rc == 0) {
        float2 hf[8][15] = {};
        for (int l = 0; l < 8; ++l)
            for (int k = 0; k < 15; ++k) hf[l][k] = make_float2((float)h[l][k].x, (float)h[l][k].y);
        rc = report(cudaMemcpyToSymbol(c_twf, hf, sizeof(hf)), "cudaMemcpyToSymbol(c_twf)");
    }
    if (rc == 0) done[dev] = true;
    return rc;
}

template <typename K>
int set_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return 0;
    return report(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                  "cudaFuncSetAttribute");
}

inline bool grid_ok(int64_t n) { return n > 0 && n < ((int64_t)1 << 31); }
// DEFMM_CARVEOUT=<percent>: one preferred L1/shared carveout for every kernel
// (kernels with different carveouts cannot share an SM, which serialises the
// P2P stream against the far-field stream)
inline int carveout_pct() {
    static const int pct = [] {
        const char* e = getenv("DEFMM_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    return pct;
}
template <typename K>
inline int carve(K* k) {
    if (carveout_pct() >= 0)
        cudaFuncSetAttribute((const void*)k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct());
    return 0;
}
inline unsigned blocks_of(int64_t n, int per) { return (unsigned)((n + per - 1) / per); }

#define DEFMM_DISPATCH_L(L, ...)                              \
    switch (L) {                                              \
        case 2: { constexpr int LL = 2; __VA_ARGS__; } break; \
        case 3: { constexpr int LL = 3; __VA_ARGS__; } break; \
        case 4: { constexpr int LL = 4; __VA_ARGS__; } break; \
        case 5: { constexpr int LL = 5; __VA_ARGS__; } break; \
        case 6: { constexpr int LL = 6; __VA_ARGS__; } break; \
        case 7: { constexpr int LL = 7; __VA_ARGS__; } break; \
        case 8: { constexpr int LL = 8; __VA_ARGS__; } break; \
        default: return -3;                                   \
    }

template <typename R>
int launch_p2m(int32_t L, int64_t n, const int32_t* cell, const int32_t* dir, const int64_t* out_slot,
               const int64_t* cell_start, const int64_t* cell_stop, const double* cell_alpha,
               const int32_t* cell_level, const double* level_beta, const double* dirs, const double* px,
               const double* py, const double* pz, const void* q, double kappa, void* mult, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (carve(p2m_kernel<R, LL>), p2m_kernel<R, LL><<<(unsigned)n, p2m_threads<LL>(), 0, s>>>(
                            n, cell, dir, out_slot, cell_start, cell_stop, cell_alpha, cell_level, level_beta,
                            dirs, px, py, pz, (const cx<R>*)q, kappa, (cx<R>*)mult)));
    return report(cudaGetLastError(), "p2m");
}

// DEFMM_NODAL=elem keeps the v1 M2M/L2L kernels (one output entry per lane)
inline bool nodal_fiber() {
    static const bool on = [] {
        const char* e = getenv("DEFMM_NODAL");
        return !(e && strcmp(e, "elem") == 0);
    }();
    return on;
}

template <typename R>
int launch_m2m(int32_t L, int64_t n, const int64_t* out_slot, const int32_t* dir, const int64_t* son_slot,
               double son_beta, const double* dirs, double kappa, void* mult, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    if (nodal_fiber()) {
        if (int rc0 = ensure_twiddles()) return rc0;
        bool launched = false;
        DEFMM_DISPATCH_L(L, {
            if constexpr (nodal2_ok<R, LL>()) {
                const size_t bytes = nodal2_smem_bytes<R, LL>();
                int rc = set_smem(m2m_fiber_kernel<R, LL>, bytes);
                if (rc) return rc;
                carve(m2m_fiber_kernel<R, LL>);
                m2m_fiber_kernel<R, LL><<<blocks_of(n, NODAL_WARPS), 32 * NODAL_WARPS, bytes, s>>>(
                    n, out_slot, dir, son_slot, son_beta, dirs, kappa, (cx<R>*)mult);
                launched = true;
            }
        });
        if (launched) return report(cudaGetLastError(), "m2m");
    }
    DEFMM_DISPATCH_L(L, {
        const size_t bytes = nodal_smem_bytes<R, LL>();
        int rc = set_smem(m2m_kernel<R, LL>, bytes);
        if (rc) return rc;
        carve(m2m_kernel<R, LL>);
        m2m_kernel<R, LL><<<blocks_of(n, NODAL_WARPS), 32 * NODAL_WARPS, bytes, s>>>(
            n, out_slot, dir, son_slot, son_beta, dirs, kappa, (cx<R>*)mult);
    });
    return report(cudaGetLastError(), "m2m");
}

template <typename R>
int launch_l2l(int32_t L, int64_t n, const int64_t* out_slot, const int8_t* octant, const int64_t* ptr,
               const int64_t* src_slot, const int32_t* src_dir, double son_beta, const double* dirs,
               double kappa, void* local, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    if (nodal_fiber()) {
        if (int rc0 = ensure_twiddles()) return rc0;
        bool launched = false;
        DEFMM_DISPATCH_L(L, {
            if constexpr (nodal2_ok<R, LL>()) {
                const size_t bytes = l2l2_smem_bytes<R, LL>();
                int rc = set_smem(l2l_fiber_kernel<R, LL>, bytes);
                if (rc) return rc;
                carve(l2l_fiber_kernel<R, LL>);
                l2l_fiber_kernel<R, LL><<<blocks_of(n, NODAL_WARPS), 32 * NODAL_WARPS, bytes, s>>>(
                    n, out_slot, octant, ptr, src_slot, src_dir, son_beta, dirs, kappa, (cx<R>*)local);
                launched = true;
            }
        });
        if (launched) return report(cudaGetLastError(), "l2l");
    }
    DEFMM_DISPATCH_L(L, {
        const size_t bytes = nodal_smem_bytes<R, LL>();
        int rc = set_smem(l2l_kernel<R, LL>, bytes);
        if (rc) return rc;
        carve(l2l_kernel<R, LL>);
        l2l_kernel<R, LL><<<blocks_of(n, NODAL_WARPS), 32 * NODAL_WARPS, bytes, s>>>(
            n, out_slot, octant, ptr, src_slot, src_dir, son_beta, dirs, kappa, (cx<R>*)local);
    });
    return report(cudaGetLastError(), "l2l");
}

template <typename R>
int launch_m2f(int32_t L, int64_t n, const int64_t* src_slot, const void* mult, void* hat, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        if constexpr (m2f2_fits<R, LL>()) {
            if (int rc1 = ensure_twiddles()) return rc1;
            const size_t bytes = sizeof(cx<R>) * M2F_WARPS * m2f2_warp_elems<R, LL>();
            int rc = set_smem(m2f2_kernel<R, LL>, bytes);
            if (rc) return rc;
            carve(m2f2_kernel<R, LL>);
            m2f2_kernel<R, LL><<<blocks_of(n, M2F_WARPS * m2f2_hpw<R, LL>()), 32 * M2F_WARPS, bytes, s>>>(
                n, src_slot, (const cx<R>*)mult, (cx<R>*)hat);
        } else {
            const size_t bytes = sizeof(cx<R>) * (P * LL + M2F_WARPS * (LL * LL * LL + LL * LL * P + LL * P * P));
            int rc = set_smem(m2f_kernel<R, LL>, bytes);
            if (rc) return rc;
            carve(m2f_kernel<R, LL>);
            m2f_kernel<R, LL><<<blocks_of(n, M2F_WARPS), 32 * M2F_WARPS, bytes, s>>>(
                n, src_slot, (const cx<R>*)mult, (cx<R>*)hat);
        }
    });
    return report(cudaGetLastError(), "m2f");
}

template <typename R>
int launch_symbols(int32_t L, int64_t n, const int32_t* tvec, const double* beta, double kappa, void* sym,
                   void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P + 2 * P * P * P);
        int rc = set_smem(symbols_kernel<R, LL>, bytes);
        if (rc) return rc;
        symbols_kernel<R, LL><<<(unsigned)n, 256, bytes, s>>>(n, tvec, beta, kappa, (cx<R>*)sym);
    });
    return report(cudaGetLastError(), "symbols");
}

template <typename R>
int launch_expand(int32_t L, int64_t n, const int32_t* canon, const int8_t* rid, const void* symc, void* symd,
                  void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (expand_symbols_kernel<R, LL><<<(unsigned)n, 256, 0, s>>>(
                            n, canon, rid, (const cx<R>*)symc, (cx<R>*)symd)));
    return report(cudaGetLastError(), "expand_symbols");
}

template <typename R>
int launch_m2l_rows(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                    const int32_t* entries, const void* hat, const void* symd, void* local, void* stream) {
    if (nrows == 0) return 0;
    if (!grid_ok(nrows)) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P * LL + P * P * P + 1 + LL * P * P + LL * LL * LL);
        int rc = set_smem(m2l_rows_kernel<R, LL>, bytes);
        if (rc) return rc;
        carve(m2l_rows_kernel<R, LL>);
        m2l_rows_kernel<R, LL><<<(unsigned)nrows, m2l_block<R, LL>(), bytes, s>>>(
            nrows, row_slot, row_ptr, (const int2*)entries, (const cx<R>*)hat, (const cx<R>*)symd,
            (cx<R>*)local);
    });
    return report(cudaGetLastError(), "m2l_rows");
}

template <typename R>
int launch_m2l_group(int32_t L, int32_t K, int64_t ngroups, const int64_t* grp_slot, const int64_t* grp_ptr,
                     const int32_t* ent, const void* hat, const void* symd, void* local, void* stream) {
    if (ngroups == 0) return 0;
    if (!grid_ok(ngroups) || K < 2 || K > 4) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
#define DEFMM_GROUP_LAUNCH(KK)                                                                              \
    {                                                                                                       \
        int rc = set_smem(m2l_group_kernel<R, LL, KK>, bytes);                                              \
        if (rc) return rc;                                                                                  \
        carve(m2l_group_kernel<R, LL, KK>);                                                                 \
        m2l_group_kernel<R, LL, KK><<<(unsigned)ngroups, m2l_block<R, LL>(), bytes, s>>>(                   \
            ngroups, grp_slot, grp_ptr, ent, (const cx<R>*)hat, (const cx<R>*)symd, (cx<R>*)local);         \
    }
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P * LL + P * P * P + 1 + LL * P * P);  // O aliases Z1
        if (K == 2) DEFMM_GROUP_LAUNCH(2) else if (K == 3) DEFMM_GROUP_LAUNCH(3) else DEFMM_GROUP_LAUNCH(4)
    });
#undef DEFMM_GROUP_LAUNCH
    return report(cudaGetLastError(), "m2l_group");
}

template <typename R>
int launch_m2l_stage(int32_t L, int64_t ncta, int32_t ns_cap, int32_t depth, const int32_t* cta_stage,
                     const int32_t* cta_went, const int32_t* stage_slot_ptr, const int32_t* slot_sym,
                     const int32_t* stage_wend, const int32_t* entries, const int32_t* cta_rows, const void* hat,
                     const void* symd, void* lhat, void* stream) {
    if (ncta == 0) return 0;
    if (ns_cap < 8 || ns_cap > 254 || depth < 2 || depth > STG_MAXDEPTH) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        using C = StageCfg<R, LL>;
        if (!grid_ok(ncta * C::NSLICE)) return -1;
        const size_t bytes = 128 + (size_t)depth * (ns_cap + 1) * C::SB;
        if (bytes > 227 * 1024) return -1;
        int rc = set_smem(m2l_stage_kernel<R, LL>, bytes);
        if (rc) return rc;
        m2l_stage_kernel<R, LL><<<(unsigned)(ncta * C::NSLICE), 32 * (STG_NW + 1), bytes, s>>>(
            ns_cap, depth, cta_stage, cta_went, stage_slot_ptr, slot_sym, stage_wend, (const int2*)entries,
            cta_rows, (const cx<R>*)hat, (const cx<R>*)symd, (cx<R>*)lhat);
    });
    return report(cudaGetLastError(), "m2l_stage");
}

template <typename R>
int launch_m2l_blocked(int32_t L, int64_t ngroups, const int64_t* grp_ptr, const int64_t* grp_rows,
                       const int32_t* blk_src, const int32_t* blk_trans, const int64_t* blk_mask,
                       const int8_t* blk_kind, const void* hat, const void* symd, void* lhat, void* stream) {
    if (ngroups == 0) return 0;
    if (!grid_ok(ngroups)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (carve(m2l_blocked_kernel<R, LL>), m2l_blocked_kernel<R, LL><<<(unsigned)ngroups, m2lb_threads<R, LL>(), 0, s>>>(
                            ngroups, grp_ptr, grp_rows, blk_src, blk_trans, blk_mask, blk_kind,
                            (const cx<R>*)hat, (const cx<R>*)symd, (cx<R>*)lhat)));
    return report(cudaGetLastError(), "m2l_blocked");
}

template <typename R>
int launch_f2l_rows(int32_t L, int64_t nrows, const int64_t* row_slot, const void* lhat, void* local,
                    void* stream) {
    if (nrows == 0) return 0;
    if (!grid_ok(nrows)) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P * LL + P * P * P + 1 + LL * P * P + LL * LL * LL);
        int rc = set_smem(f2l_rows_kernel<R, LL>, bytes);
        if (rc) return rc;
        carve(f2l_rows_kernel<R, LL>);
        f2l_rows_kernel<R, LL><<<(unsigned)nrows, 128, bytes, s>>>(nrows, row_slot, (const cx<R>*)lhat,
                                                                   (cx<R>*)local);
    });
    return report(cudaGetLastError(), "f2l_rows");
}

template <typename R>
int launch_l2p(int32_t L, int64_t n, const int32_t* leaf_cell, const int64_t* slot_lo, const int64_t* slot_hi,
               const int32_t* slot_dir, const int64_t* cell_start, const int64_t* cell_stop,
               const double* cell_alpha, const int32_t* cell_level, const double* level_beta, const double* dirs,
               const double* px, const double* py, const double* pz, double kappa, const void* local,
               const void* near, const int64_t* perm, void* out, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (carve(l2p_kernel<R, LL>), l2p_kernel<R, LL><<<(unsigned)n, 64, 0, s>>>(
                            n, leaf_cell, slot_lo, slot_hi, slot_dir, cell_start, cell_stop, cell_alpha,
                            cell_level, level_beta, dirs, px, py, pz, kappa, (const cx<R>*)local,
                            (const cx<R>*)near, perm, (cx<R>*)out)));
    return report(cudaGetLastError(), "l2p");
}

template <typename R>
int launch_p2p(int64_t n_items, const int32_t* item_leaf, const int64_t* item_f0, const int64_t* item_f1,
               const int64_t* item_out, const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* ptr,
               const int64_t* src_lo, const int64_t* src_hi, const double* tx, const double* ty, const double* tz,
               const double* sx, const double* sy, const double* sz, const void* q, double kappa, double tol,
               void* near, void* partial, int64_t n_split, const int32_t* split_leaf, const int64_t* split_base,
               const int32_t* split_n, int32_t grid, int32_t hilo, void* stream) {
    if (n_items == 0) return 0;
    if (!grid_ok(n_items)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    const P2PItems it{item_leaf, item_f0, item_f1, item_out};
    // grid > 0: a persistent grid striding over the items (leaves SM room for
    // the concurrently running far-field kernels); 0: one CTA per item
    const unsigned ng = (unsigned)(grid > 0 && grid < n_items ? grid : n_items);
    if constexpr (sizeof(R) == 4) {
        if (hilo) {
            carve(p2p_f32_kernel<true>);
            p2p_f32_kernel<true><<<ng, P2P_NT, 0, s>>>(n_items, it, tgt_lo, tgt_hi, ptr, src_lo, src_hi, tx, ty,
                                                       tz, sx, sy, sz, (const float2*)q, kappa, tol,
                                                       (float2*)near, (float2*)partial);
        } else {
            carve(p2p_f32_kernel<false>);
            p2p_f32_kernel<false><<<ng, P2P_NT, 0, s>>>(n_items, it, tgt_lo, tgt_hi, ptr, src_lo, src_hi, tx, ty,
                                                        tz, sx, sy, sz, (const float2*)q, kappa, tol,
                                                        (float2*)near, (float2*)partial);
        }
    } else {
        carve(p2p_kernel<R>);
        p2p_kernel<R><<<ng, P2P_NT, 0, s>>>(n_items, it, tgt_lo, tgt_hi, ptr, src_lo, src_hi, tx,
                                                           ty, tz, sx, sy, sz, (const cx<R>*)q, kappa, tol,
                                                           (cx<R>*)near, (cx<R>*)partial);
    }
    if (n_split > 0) {
        if (!grid_ok(n_split)) return -1;
        carve(p2p_reduce_kernel<R>);
        p2p_reduce_kernel<R><<<(unsigned)n_split, 128, 0, s>>>(n_split, split_leaf, split_base, split_n, tgt_lo,
                                                                tgt_hi, (const cx<R>*)partial, (cx<R>*)near);
    }
    return report(cudaGetLastError(), "p2p");
}

template <typename R>
int launch_p2p_mutual(int64_t n_items, const int32_t* item_leaf, const int64_t* item_f0, const int64_t* item_f1,
                      const int64_t* item_row, const int64_t* item_col, const int64_t* tgt_lo,
                      const int64_t* tgt_hi, const int64_t* ptr, const int64_t* src_lo, const int64_t* src_hi,
                      const double* px, const double* py, const double* pz, const void* q, double kappa,
                      double tol, void* partial, int32_t grid, int32_t hilo, void* stream) {
    if (n_items == 0) return 0;
    if (!grid_ok(n_items)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    const P2PMutItems it{item_leaf, item_f0, item_f1, item_row, item_col};
    const unsigned ng = (unsigned)(grid > 0 && grid < n_items ? grid : n_items);
    if constexpr (sizeof(R) == 4) {
        if (hilo) {
            carve(p2p_mut_f32_kernel<true>);
            p2p_mut_f32_kernel<true><<<ng, P2P_NT, 0, s>>>(n_items, it, tgt_lo, tgt_hi, ptr, src_lo, src_hi, px, py,
                                                           pz, (const float2*)q, kappa, tol, (float2*)partial);
        } else {
            carve(p2p_mut_f32_kernel<false>);
            p2p_mut_f32_kernel<false><<<ng, P2P_NT, 0, s>>>(n_items, it, tgt_lo, tgt_hi, ptr, src_lo, src_hi, px,
                                                            py, pz, (const float2*)q, kappa, tol, (float2*)partial);
        }
    } else {
        carve(p2p_mut_kernel<R>);
        p2p_mut_kernel<R><<<ng, P2P_NT, 0, s>>>(n_items, it, tgt_lo, tgt_hi, ptr, src_lo, src_hi, px, py, pz,
                                                (const cx<R>*)q, kappa, tol, (double2*)partial);
    }
    return report(cudaGetLastError(), "p2p_mutual");
}

template <typename R>
int launch_p2p_gather(int64_t n, const int32_t* task_leaf, const int64_t* task_out, const int64_t* tgt_lo,
                      const int64_t* tgt_hi, const int64_t* cptr, const int64_t* cbase, const int32_t* cxlo,
                      const int32_t* cxhi, void* partial, void* near, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    carve(p2p_gather_kernel<R>);
    p2p_gather_kernel<R><<<(unsigned)n, 64, 0, (cudaStream_t)stream>>>(n, task_leaf, task_out, tgt_lo, tgt_hi, cptr,
                                                                      cbase, cxlo, cxhi, (cx<R>*)partial,
                                                                      (cx<R>*)near);
    return report(cudaGetLastError(), "p2p_gather");
}

}  // namespace

extern "C" {

int defmm_abi_version(void) { return DEFMM_ABI_VERSION; }

int defmm_spectral_layout(int32_t L, int32_t* forder, int32_t* slice_start, int32_t* nslices) {
    if (L < 2 || L > 8) return -1;
    const HostLayout& H = layout_of(L);
    if (nslices) *nslices = H.nslices;
    if (forder)
        for (int t = 0; t < H.P3; ++t) forder[t] = H.forder[t];
    if (slice_start)
        for (int t = 0; t <= H.nslices; ++t) slice_start[t] = H.start[t];
    return 0;
}
const char* defmm_last_error(void) { return g_last_error; }

#define DEFMM_EXPORT_TYPED(SUFFIX, R)                                                                               \
    int defmm_p2m_##SUFFIX(int32_t L, int64_t n, const int32_t* cell, const int32_t* dir, const int64_t* out_slot,  \
                           const int64_t* cell_start, const int64_t* cell_stop, const double* cell_alpha,          \
                           const int32_t* cell_level, const double* level_beta, const double* dirs,                \
                           const double* px, const double* py, const double* pz, const void* q, double kappa,      \
                           void* mult, void* stream) {                                                             \
        return launch_p2m<R>(L, n, cell, dir, out_slot, cell_start, cell_stop, cell_alpha, cell_level,             \
                             level_beta, dirs, px, py, pz, q, kappa, mult, stream);                                \
    }                                                                                                               \
    int defmm_m2m_##SUFFIX(int32_t L, int64_t n, const int64_t* out_slot, const int32_t* dir,                       \
                           const int64_t* son_slot, double son_beta, const double* dirs, double kappa, void* mult,  \
                           void* stream) {                                                                         \
        return launch_m2m<R>(L, n, out_slot, dir, son_slot, son_beta, dirs, kappa, mult, stream);                  \
    }                                                                                                               \
    int defmm_m2f_##SUFFIX(int32_t L, int64_t n, const int64_t* src_slot, const void* mult, void* hat,              \
                           void* stream) {                                                                         \
        return launch_m2f<R>(L, n, src_slot, mult, hat, stream);                                                   \
    }                                                                                                               \
    int defmm_symbols_##SUFFIX(int32_t L, int64_t n, const int32_t* tvec, const double* beta, double kappa,         \
                               void* sym, void* stream) {                                                          \
        return launch_symbols<R>(L, n, tvec, beta, kappa, sym, stream);                                            \
    }                                                                                                               \
    int defmm_expand_symbols_##SUFFIX(int32_t L, int64_t n, const int32_t* canon, const int8_t* rid,                \
                                      const void* sym_canon, void* sym_derived, void* stream) {                    \
        return launch_expand<R>(L, n, canon, rid, sym_canon, sym_derived, stream);                                 \
    }                                                                                                               \
    int defmm_m2l_rows_##SUFFIX(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,          \
                                const int32_t* entries, const void* hat, const void* sym_derived, void* local,     \
                                void* stream) {                                                                    \
        return launch_m2l_rows<R>(L, nrows, row_slot, row_ptr, entries, hat, sym_derived, local, stream);          \
    }                                                                                                               \
    int defmm_m2l_group_##SUFFIX(int32_t L, int32_t K, int64_t ngroups, const int64_t* grp_slot,                  \
                                 const int64_t* grp_ptr, const int32_t* entries, const void* hat,                 \
                                 const void* sym_derived, void* local, void* stream) {                            \
        return launch_m2l_group<R>(L, K, ngroups, grp_slot, grp_ptr, entries, hat, sym_derived, local, stream);   \
    }                                                                                                               \
    int defmm_m2l_stage_##SUFFIX(int32_t L, int64_t ncta, int32_t ns_cap, int32_t depth,                           \
                                 const int32_t* cta_stage, const int32_t* cta_went,                               \
                                 const int32_t* stage_slot_ptr, const int32_t* slot_sym,                          \
                                 const int32_t* stage_wend, const int32_t* entries, const int32_t* cta_rows,      \
                                 const void* hat, const void* sym_derived, void* lhat, void* stream) {            \
        return launch_m2l_stage<R>(L, ncta, ns_cap, depth, cta_stage, cta_went, stage_slot_ptr, slot_sym,         \
                                   stage_wend, entries, cta_rows, hat, sym_derived, lhat, stream);                \
    }                                                                                                               \
    int defmm_m2l_blocked_##SUFFIX(int32_t L, int64_t ngroups, const int64_t* grp_ptr, const int64_t* grp_rows,     \
                                   const int32_t* blk_src, const int32_t* blk_trans, const int64_t* blk_mask,     \
                                   const int8_t* blk_kind, const void* hat, const void* sym_derived, void* lhat,  \
                                   void* stream) {                                                                \
        return launch_m2l_blocked<R>(L, ngroups, grp_ptr, grp_rows, blk_src, blk_trans, blk_mask, blk_kind, hat,   \
                                     sym_derived, lhat, stream);                                                  \
    }                                                                                                               \
    int defmm_f2l_rows_##SUFFIX(int32_t L, int64_t nrows, const int64_t* row_slot, const void* lhat, void* local,   \
                                void* stream) {                                                                    \
        return launch_f2l_rows<R>(L, nrows, row_slot, lhat, local, stream);                                        \
    }                                                                                                               \
    int defmm_l2l_##SUFFIX(int32_t L, int64_t n, const int64_t* out_slot, const int8_t* octant,                     \
                           const int64_t* ptr, const int64_t* src_slot, const int32_t* src_dir, double son_beta,   \
                           const double* dirs, double kappa, void* local, void* stream) {                          \
        return launch_l2l<R>(L, n, out_slot, octant, ptr, src_slot, src_dir, son_beta, dirs, kappa, local,         \
                             stream);                                                                              \
    }                                                                                                               \
    int defmm_l2p_##SUFFIX(int32_t L, int64_t n, const int32_t* leaf_cell, const int64_t* slot_lo,                  \
                           const int64_t* slot_hi, const int32_t* slot_dir, const int64_t* cell_start,             \
                           const int64_t* cell_stop, const double* cell_alpha, const int32_t* cell_level,          \
                           const double* level_beta, const double* dirs, const double* px, const double* py,       \
                           const double* pz, double kappa, const void* local, const void* near,                    \
                           const int64_t* perm, void* out, void* stream) {                                         \
        return launch_l2p<R>(L, n, leaf_cell, slot_lo, slot_hi, slot_dir, cell_start, cell_stop, cell_alpha,       \
                             cell_level, level_beta, dirs, px, py, pz, kappa, local, near, perm, out, stream);     \
    }                                                                                                               \
    int defmm_p2p_mutual_##SUFFIX(int64_t n_items, const int32_t* item_leaf, const int64_t* item_f0,              \
                                  const int64_t* item_f1, const int64_t* item_row, const int64_t* item_col,       \
                                  const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* ptr,               \
                                  const int64_t* src_lo, const int64_t* src_hi, const double* px,                 \
                                  const double* py, const double* pz, const void* q, double kappa, double tol,    \
                                  void* partial, int32_t grid, int32_t hilo, void* stream) {                      \
        return launch_p2p_mutual<R>(n_items, item_leaf, item_f0, item_f1, item_row, item_col, tgt_lo, tgt_hi,      \
                                    ptr, src_lo, src_hi, px, py, pz, q, kappa, tol, partial, grid, hilo, stream); \
    }                                                                                                               \
    int defmm_p2p_gather_##SUFFIX(int64_t n, const int32_t* task_leaf, const int64_t* task_out,                     \
                                  const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* cptr,              \
                                  const int64_t* cbase, const int32_t* cxlo, const int32_t* cxhi, void* partial,  \
                                  void* near, void* stream) {                                                     \
        return launch_p2p_gather<R>(n, task_leaf, task_out, tgt_lo, tgt_hi, cptr, cbase, cxlo, cxhi, partial,      \
                                    near, stream);                                                                \
    }                                                                                                               \
    int defmm_p2p_##SUFFIX(int64_t n_items, const int32_t* item_leaf, const int64_t* item_f0,                    \
                           const int64_t* item_f1, const int64_t* item_out, const int64_t* tgt_lo,                \
                           const int64_t* tgt_hi, const int64_t* ptr, const int64_t* src_lo,                      \
                           const int64_t* src_hi, const double* tx, const double* ty, const double* tz,           \
                           const double* sx, const double* sy, const double* sz, const void* q, double kappa,     \
                           double tol, void* near, void* partial, int64_t n_split, const int32_t* split_leaf,     \
                           const int64_t* split_base, const int32_t* split_n, int32_t grid, int32_t hilo,         \
                           void* stream) {                                                                        \
        return launch_p2p<R>(n_items, item_leaf, item_f0, item_f1, item_out, tgt_lo, tgt_hi, ptr, src_lo, src_hi,  \
                             tx, ty, tz, sx, sy, sz, q, kappa, tol, near, partial, n_split, split_leaf,           \
                             split_base, split_n, grid, hilo, stream);                                            \
    }

DEFMM_EXPORT_TYPED(c128, double)
DEFMM_EXPORT_TYPED(c64, float)

int defmm_m2l_canon_c128(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                         const int32_t* e_src, const int32_t* e_sym, const int8_t* e_rid, const void* hat,
                         const void* sym, void* local, void* stream) {
    if (nrows == 0) return 0;
    if (!grid_ok(nrows)) return -1;
    if (int rc0 = ensure_twiddles()) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P * LL + P * P * P + LL * P * P);
        int rc = set_smem(m2l_canon_kernel<LL>, bytes);
        if (rc) return rc;
        m2l_canon_kernel<LL><<<(unsigned)nrows, m2l_threads<LL>(), bytes, s>>>(
            nrows, row_slot, row_ptr, e_src, e_sym, e_rid, (const double2*)hat, (const double2*)sym,
            (double2*)local);
    });
    return report(cudaGetLastError(), "m2l_canon");
}

int defmm_spectrum_stride(int32_t L, int32_t c64) {
    int v = -3;
    if (c64) {
        DEFMM_DISPATCH_L(L, v = spec_stride<float, LL>());
    } else {
        DEFMM_DISPATCH_L(L, v = spec_stride<double, LL>());
    }
    return v;
}

int64_t defmm_direct_workspace_bytes(int64_t nt) { return (int64_t)DIRECT_SPLIT * nt * (int64_t)sizeof(double2); }

int defmm_direct_c128(int64_t nt, const double* tx, const double* ty, const double* tz, int64_t ns,
                      const double* sx, const double* sy, const double* sz, const void* q, double kappa,
                      double tol, void* workspace, void* out, void* stream) {
    if (nt == 0) return 0;
    const int64_t blocks = (nt + 127) / 128;
    if (!grid_ok(blocks)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    const int split = ns >= (int64_t)DIRECT_SPLIT * 256 ? DIRECT_SPLIT : 1;
    double2* part = (double2*)workspace;
    direct_kernel<<<dim3((unsigned)blocks, split), 128, 0, s>>>(nt, tx, ty, tz, ns, sx, sy, sz,
                                                                (const double2*)q, kappa, tol, part);
    direct_reduce<<<(unsigned)blocks, 128, 0, s>>>(nt, split, part, (double2*)out);
    return report(cudaGetLastError(), "direct");
}

}  // extern "C"
