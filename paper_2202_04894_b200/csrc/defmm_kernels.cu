// B200 (sm_100a) kernels of the defmm FMM matvec, behind the C-ABI declared
// in include/defmm_b200.h.  complex128 path (double2 interleaved complex).
//
// Design notes (see DESIGN.md for the roofline of each kernel):
//  * every kernel owns its outputs -- one CTA per output object (expansion
//    slot, M2L row, target leaf) -- so there are no atomics and reruns are
//    bitwise deterministic (test_traversal.py:224-231's contract);
//  * all plane-wave modulations are applied in CELL-RELATIVE form
//    (e^{i kappa <xi - y, u>} factorised per axis), which equals the
//    reference's absolute-coordinate products (interpolation.py:104-137,
//    traversal.py:245-280, 362-391) in exact arithmetic and keeps phases small;
//  * the Fourier-domain M2L gathers canonical symbols through the closed form
//    of the cube-group frequency permutation (fourier.py:123-143) instead of
//    materialising one P^3 spectrum per translation.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../include/defmm_b200.h"

namespace {

thread_local char g_last_error[256] = "";

int report(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return 0;
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
    return (int)e;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// c + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
    return c;
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cexpi(double ph) {
    double s, c;
    sincos(ph, &s, &c);
    return make_double2(c, s);
}

// Predicated 16-B read-only load that the compiler cannot sink below later
// code: keeps all loads of an M2L run in flight together.
__device__ __forceinline__ double2 ldg_pred(const double2* p, bool pred) {
    double2 v;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tmov.f64 %0, 0d0000000000000000;\n\t"
        "mov.f64 %1, 0d0000000000000000;\n\t@q ld.global.nc.v2.f64 {%0, %1}, [%2];\n\t}"
        : "=d"(v.x), "=d"(v.y)
        : "l"(p), "r"((int)pred));
    return v;
}

// Equispaced nodes x_j = j/(L-1) (interpolation.py:51-56) and the Lagrange
// cardinal functions S_k(x) = prod_{j != k} (x - x_j)/(x_k - x_j) (:59-69).
template <int L>
__device__ __forceinline__ double node(int j) {
    return (double)j / (double)(L - 1);
}
template <int L>
__device__ __forceinline__ void lagrange(double x, double* S) {
#pragma unroll
    for (int k = 0; k < L; ++k) {
        double v = 1.0;
#pragma unroll
        for (int j = 0; j < L; ++j)
            if (j != k) v = v * (x - node<L>(j)) / (node<L>(k) - node<L>(j));
        S[k] = v;
    }
}

template <int L>
__host__ __device__ constexpr int cube() { return L * L * L; }
template <int L>
__host__ __device__ constexpr int pad() { return 2 * L - 1; }
__host__ __device__ constexpr int round32(int x) { return (x + 31) / 32 * 32; }

// threads per CTA for the L^3-shaped operators (one thread per nodal entry)
template <int L>
__host__ __device__ constexpr int nodal_threads() { return round32(cube<L>()) < 64 ? 64 : round32(cube<L>()); }

// ---------------------------------------------------------------------------
// K2: P2M.  One CTA per (leaf, key).  Per particle and axis the modulated 1D
// weights W_a = S_a(xh) e^{i kappa beta u (x_a - xh)} are staged in shared
// memory; the L^3 output entries are then tensor sums over the particles.

template <int L>
__global__ void __launch_bounds__(128) p2m_kernel(
    int64_t n, const int32_t* __restrict__ cell, const int32_t* __restrict__ dir,
    const int64_t* __restrict__ out_slot, const int64_t* __restrict__ cstart,
    const int64_t* __restrict__ cstop, const double* __restrict__ calpha,
    const int32_t* __restrict__ clevel, const double* __restrict__ lbeta,
    const double* __restrict__ dirs, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, const double2* __restrict__ q, double kappa,
    double2* __restrict__ mult) {
    constexpr int L3 = cube<L>();
    constexpr int NT = 128;
    constexpr int PER = (L3 + NT - 1) / NT;
    constexpr int CH = 32;
    __shared__ double2 W[3][CH][L];
    const int64_t i = blockIdx.x;
    const int c = cell[i];
    const int d = dir[i];
    const double beta = lbeta[clevel[c]];
    double al[3], ku[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        al[k] = calpha[3 * c + k];
        ku[k] = d >= 0 ? kappa * beta * dirs[3 * d + k] : 0.0;
    }
    const int64_t s0 = cstart[c], s1 = cstop[c];
    double2 acc[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) acc[m] = make_double2(0.0, 0.0);
    for (int64_t base = s0; base < s1; base += CH) {
        const int cnt = (int)((s1 - base) < (int64_t)(CH) ? (s1 - base) : (int64_t)(CH));
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * 3; t += NT) {
            const int p = t / 3, ax = t - 3 * (t / 3);
            const double* pp = ax == 0 ? px : (ax == 1 ? py : pz);
            const double xh = (pp[base + p] - al[ax]) / beta;
            double S[L];
            lagrange<L>(xh, S);
            const double2 qq = ax == 0 ? q[base + p] : make_double2(1.0, 0.0);
#pragma unroll
            for (int k = 0; k < L; ++k) {
                const double2 w = cscale(cexpi(ku[ax] * (node<L>(k) - xh)), S[k]);
                W[ax][p][k] = cmul(qq, w);
            }
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int r = threadIdx.x + m * NT;
            if (r < L3) {
                const int a = r / (L * L), b = (r / L) % L, cc = r % L;
                double2 s = acc[m];
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
// K4/K5: M2M and L2L.  The modulated Kronecker factor of one son octant is
// C_ax[k][j] = A_bit[k][j] e^{i kappa v_ax beta_s (2 x_k - bit - x_j)}, with
// A_bit[k][j] = S_k((bit + x_j)/2) (interpolation.py:140-148); L2L uses
// C'_ax[j][k] = conj(C_ax[k][j]) (interpolation.py:151-154 + the conjugate
// modulation of traversal.py:362-391).  Three mode products in shared memory.

template <int L>
__device__ __forceinline__ void build_factors(double2 (*C)[L][L], int oct, const double ku[3],
                                              bool transpose_conj) {
    for (int t = threadIdx.x; t < 3 * L * L; t += blockDim.x) {
        const int ax = t / (L * L), k = (t / L) % L, j = t % L;  // C[ax][k][j]
        const int bit = (oct >> (2 - ax)) & 1;
        double S[L];
        // A_bit[k][j] = S_k((bit + x_j)/2) ; for the transpose use (k <-> j)
        const int kk = transpose_conj ? j : k;  // father node index
        const int jj = transpose_conj ? k : j;  // son node index
        lagrange<L>(((double)bit + node<L>(jj)) / 2.0, S);
        const double ph = ku[ax] * (2.0 * node<L>(kk) - (double)bit - node<L>(jj));
        double2 w = cscale(cexpi(ph), S[kk]);
        if (transpose_conj) w = cconj(w);
        C[ax][k][j] = w;
    }
}

// y = (C0 (x) C1 (x) C2) x for one L^3 tile; x and tmp in shared memory; the
// result for entry r = threadIdx.x (< L^3) is returned.
template <int L>
__device__ __forceinline__ double2 kron3_apply(const double2 (*C)[L][L], double2* x, double2* tmp) {
    constexpr int L3 = cube<L>();
    const int r = threadIdx.x;
    const int a = r / (L * L), b = (r / L) % L, c = r % L;
    double2 v = make_double2(0.0, 0.0);
    if (r < L3) {
#pragma unroll
        for (int j = 0; j < L; ++j) v = cfma(C[0][a][j], x[(j * L + b) * L + c], v);
    }
    __syncthreads();
    if (r < L3) tmp[r] = v;
    __syncthreads();
    v = make_double2(0.0, 0.0);
    if (r < L3) {
#pragma unroll
        for (int j = 0; j < L; ++j) v = cfma(C[1][b][j], tmp[(a * L + j) * L + c], v);
    }
    __syncthreads();
    if (r < L3) x[r] = v;
    __syncthreads();
    v = make_double2(0.0, 0.0);
    if (r < L3) {
#pragma unroll
        for (int j = 0; j < L; ++j) v = cfma(C[2][c][j], x[(a * L + b) * L + j], v);
    }
    return v;
}

template <int L>
__global__ void __launch_bounds__(nodal_threads<L>()) m2m_kernel(
    int64_t n, const int64_t* __restrict__ out_slot, const int32_t* __restrict__ dir,
    const int64_t* __restrict__ son_slot, double son_beta, const double* __restrict__ dirs,
    double kappa, double2* __restrict__ mult) {
    constexpr int L3 = cube<L>();
    __shared__ double2 C[3][L][L];
    __shared__ double2 X[L3], T[L3];
    const int64_t i = blockIdx.x;
    const int d = dir[i];
    double ku[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ku[k] = d >= 0 ? kappa * son_beta * dirs[3 * d + k] : 0.0;
    double2 acc = make_double2(0.0, 0.0);
    for (int o = 0; o < 8; ++o) {
        const int64_t ss = son_slot[8 * i + o];
        if (ss < 0) continue;
        __syncthreads();
        if (threadIdx.x < L3) X[threadIdx.x] = mult[ss * L3 + threadIdx.x];
        build_factors<L>(C, o, ku, false);
        __syncthreads();
        acc = cadd(acc, kron3_apply<L>(C, X, T));
    }
    if (threadIdx.x < L3) mult[out_slot[i] * L3 + threadIdx.x] = acc;
}

template <int L>
__global__ void __launch_bounds__(nodal_threads<L>()) l2l_kernel(
    int64_t n, const int64_t* __restrict__ out_slot, const int8_t* __restrict__ octant,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_slot,
    const int32_t* __restrict__ src_dir, double son_beta, const double* __restrict__ dirs,
    double kappa, double2* __restrict__ local) {
    constexpr int L3 = cube<L>();
    __shared__ double2 C[3][L][L];
    __shared__ double2 X[L3], T[L3];
    const int64_t i = blockIdx.x;
    const int oct = octant[i];
    const int64_t o = out_slot[i] * L3;
    double2 acc = make_double2(0.0, 0.0);
    if (threadIdx.x < L3) acc = local[o + threadIdx.x];
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
        const int d = src_dir[e];
        double ku[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) ku[k] = d >= 0 ? kappa * son_beta * dirs[3 * d + k] : 0.0;
        __syncthreads();
        if (threadIdx.x < L3) X[threadIdx.x] = local[src_slot[e] * L3 + threadIdx.x];
        build_factors<L>(C, oct, ku, true);
        __syncthreads();
        acc = cadd(acc, kron3_apply<L>(C, X, T));
    }
    if (threadIdx.x < L3) local[o + threadIdx.x] = acc;
}

// ---------------------------------------------------------------------------
// Pruned odd-size 3D DFTs.  tw[k] = e^{-2 pi i k / P}.

template <int P>
__device__ __forceinline__ void make_twiddles(double2* tw) {
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)k / (double)P, &s, &c);
        tw[k] = make_double2(c, -s);
    }
}

// K6 M2F: L^3 corner of a zero P^3 grid -> unitary forward DFT (fourier.py:67-72).
template <int L>
__global__ void __launch_bounds__(128) m2f_kernel(int64_t n, const int64_t* __restrict__ src_slot,
                                                  const double2* __restrict__ mult,
                                                  double2* __restrict__ hat) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    extern __shared__ double2 sm[];
    double2* tw = sm;                 // P
    double2* X = tw + P;              // L^3
    double2* Y1 = X + L3;             // L*L*P   [a][b][f2]
    double2* Y2 = Y1 + L * L * P;     // L*P*P   [a][f1][f2]
    const int64_t i = blockIdx.x;
    make_twiddles<P>(tw);
    const int64_t s = src_slot[i] * L3;
    for (int r = threadIdx.x; r < L3; r += blockDim.x) X[r] = mult[s + r];
    __syncthreads();
    for (int t = threadIdx.x; t < L * L * P; t += blockDim.x) {
        const int ab = t / P, f2 = t % P;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < L; ++c) v = cfma(X[ab * L + c], tw[(f2 * c) % P], v);
        Y1[t] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < L * P * P; t += blockDim.x) {
        const int a = t / (P * P), f1 = (t / P) % P, f2 = t % P;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < L; ++b) v = cfma(Y1[(a * L + b) * P + f2], tw[(f1 * b) % P], v);
        Y2[t] = v;
    }
    __syncthreads();
    const double scale = 1.0 / (P * sqrt((double)P));
    double2* out = hat + i * (int64_t)P3;
    for (int t = threadIdx.x; t < P3; t += blockDim.x) {
        const int f0 = t / (P * P), f12 = t % (P * P);
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int a = 0; a < L; ++a) v = cfma(Y2[a * P * P + f12], tw[(f0 * a) % P], v);
        out[t] = cscale(v, scale);
    }
}

// K9 symbols: kernel column on the difference grid (wrap order) and its
// unnormalised forward DFT (fourier.py:156-183).
template <int L>
__global__ void __launch_bounds__(256) symbols_kernel(int64_t n, const int32_t* __restrict__ tvec,
                                                      const double* __restrict__ beta, double kappa,
                                                      double2* __restrict__ sym) {
    constexpr int P = pad<L>(), P3 = P * P * P;
    extern __shared__ double2 sm[];
    double2* tw = sm;
    double2* A = tw + P;
    double2* B = A + P3;
    const int64_t i = blockIdx.x;
    make_twiddles<P>(tw);
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
    // axis 2, then 1, then 0 (full DFTs)
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
    double2* out = sym + i * (int64_t)P3;
    for (int t = threadIdx.x; t < P3; t += blockDim.x) {
        const int f = t / (P * P), bc = t % (P * P);
        double2 v = make_double2(0.0, 0.0);
        for (int k = 0; k < P; ++k) v = cfma(A[k * P * P + bc], tw[(f * k) % P], v);
        out[t] = v;
    }
}

// ---------------------------------------------------------------------------
// K7+K8: Hadamard M2L over a target-major CSR row, then the pruned inverse
// DFT (F2L) of the accumulated spectrum, written once to the local slot.

// itertools.permutations(range(3)) order (fourier.py:94)
__constant__ int8_t c_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

template <int L>
__host__ __device__ constexpr int m2l_threads() {
    return L <= 3 ? 128 : L == 4 ? 352 : L == 5 ? 256 : L == 6 ? 448 : L == 7 ? 320 : 384;
}

template <int L>
__global__ void __launch_bounds__(m2l_threads<L>()) m2l_kernel(
    int64_t nrows, const int64_t* __restrict__ row_slot, const int64_t* __restrict__ row_ptr,
    const int32_t* __restrict__ e_src, const int32_t* __restrict__ e_sym,
    const int8_t* __restrict__ e_rid, const double2* __restrict__ hat,
    const double2* __restrict__ sym, double2* __restrict__ local) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int NT = m2l_threads<L>();
    constexpr int PER = (P3 + NT - 1) / NT;
    extern __shared__ double2 sm[];
    double2* tw = sm;             // P
    double2* X = tw + P;          // P^3
    double2* Z1 = X + P3;         // L*P*P
    const int64_t row = blockIdx.x;
    make_twiddles<P>(tw);
    int f[PER][3];
    double2 acc[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int j = threadIdx.x + m * NT;
        f[m][0] = j / (P * P);
        f[m][1] = (j / P) % P;
        f[m][2] = j % P;
        acc[m] = make_double2(0.0, 0.0);
    }
    const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
    for (int64_t e = e0; e < e1; ++e) {
        const int64_t src = e_src[e];
        const int64_t sy = e_sym[e];
        const int rid = e_rid[e];
        const int pi = rid >> 3;
        int w[3], ng[3];
        const int wt[3] = {P * P, P, 1};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            w[a] = wt[c_perm[pi][a]];
            ng[a] = (rid >> (2 - a)) & 1;
        }
        const double2* S = hat + src * P3;
        const double2* D = sym + sy * P3;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int j = threadIdx.x + m * NT;
            if (j < P3) {
                int idx = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int fa = f[m][a];
                    const int v = ng[a] ? (fa ? P - fa : 0) : fa;
                    idx += w[a] * v;
                }
                acc[m] = cfma(__ldg(D + idx), __ldg(S + j), acc[m]);
            }
        }
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int j = threadIdx.x + m * NT;
        if (j < P3) X[j] = acc[m];
    }
    __syncthreads();
    // inverse, pruned: contract f0 -> a (L*P*P outputs) ...
    for (int t = threadIdx.x; t < L * P * P; t += NT) {
        const int a = t / (P * P), f12 = t % (P * P);
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int f0 = 0; f0 < P; ++f0) v = cfma(X[f0 * P * P + f12], cconj(tw[(f0 * a) % P]), v);
        Z1[t] = v;
    }
    __syncthreads();
    // ... f1 -> b (L*L*P outputs, into X) ...
    for (int t = threadIdx.x; t < L * L * P; t += NT) {
        const int a = t / (L * P), b = (t / P) % L, f2 = t % P;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int f1 = 0; f1 < P; ++f1) v = cfma(Z1[(a * P + f1) * P + f2], cconj(tw[(f1 * b) % P]), v);
        X[t] = v;
    }
    __syncthreads();
    // ... f2 -> c (L^3 outputs), scaled by P^{-3/2}
    const double scale = 1.0 / (P * sqrt((double)P));
    double2* out = local + row_slot[row] * L3;
    for (int t = threadIdx.x; t < L3; t += NT) {
        const int ab = t / L, c = t % L;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) v = cfma(X[ab * P + f2], cconj(tw[(f2 * c) % P]), v);
        out[t] = cscale(v, scale);
    }
}

// Derived symbols: D_t[j] = D_canon[perm_rid(j)] materialised once per plan so
// that the M2L inner loop streams them with coalesced 16-B loads (the v1
// in-loop gather cost ~20 L1 wavefronts per warp and event, see
// profiles/r01_summary_v1.md).
template <int L>
__global__ void __launch_bounds__(256) expand_symbols_kernel(int64_t n, const int32_t* __restrict__ canon,
                                                             const int8_t* __restrict__ rid,
                                                             const double2* __restrict__ symc,
                                                             double2* __restrict__ symd) {
    constexpr int P = pad<L>(), P3 = P * P * P;
    const int64_t i = blockIdx.x;
    const int r = rid[i];
    const int pi = r >> 3;
    const int wt[3] = {P * P, P, 1};
    int w[3], ng[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        w[a] = wt[c_perm[pi][a]];
        ng[a] = (r >> (2 - a)) & 1;
    }
    const double2* src = symc + (int64_t)canon[i] * P3;
    double2* dst = symd + i * P3;
    for (int j = threadIdx.x; j < P3; j += blockDim.x) {
        const int f[3] = {j / (P * P), (j / P) % P, j % P};
        int idx = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) idx += w[a] * (ng[a] ? (f[a] ? P - f[a] : 0) : f[a]);
        dst[j] = src[idx];
    }
}

// M2L v2: one CTA per group of <= G target rows that share a parent cell and a
// key (siblings), entries sorted by source so each source spectrum is loaded
// once per group into registers; derived symbols streamed coalesced; G
// register accumulators; F2L epilogue per row.  Entry = {src hat index,
// translation id | a << 29} (a = row index inside the group).
template <int L>
__host__ __device__ constexpr int m2l_group_size() { return L <= 5 ? 8 : (L == 6 ? 4 : 2); }

template <int L>
__device__ __forceinline__ void f2l_row(const double2* tw, double2* X, double2* Z1, double2* out) {
    constexpr int P = pad<L>(), L3 = cube<L>();
    const int NT = blockDim.x;
    for (int t = threadIdx.x; t < L * P * P; t += NT) {
        const int a = t / (P * P), f12 = t % (P * P);
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int f0 = 0; f0 < P; ++f0) v = cfma(X[f0 * P * P + f12], cconj(tw[(f0 * a) % P]), v);
        Z1[t] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < L * L * P; t += NT) {
        const int a = t / (L * P), b = (t / P) % L, f2 = t % P;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int f1 = 0; f1 < P; ++f1) v = cfma(Z1[(a * P + f1) * P + f2], cconj(tw[(f1 * b) % P]), v);
        X[t] = v;
    }
    __syncthreads();
    const double scale = 1.0 / (P * sqrt((double)P));
    for (int t = threadIdx.x; t < L3; t += NT) {
        const int ab = t / L, c = t % L;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int f2 = 0; f2 < P; ++f2) v = cfma(X[ab * P + f2], cconj(tw[(f2 * c) % P]), v);
        out[t] = cscale(v, scale);
    }
}

// M2L v1b: one CTA per target row (high occupancy), derived symbols streamed
// coalesced; two entries in flight per iteration.
template <int L>
__global__ void __launch_bounds__(m2l_threads<L>()) m2l_rows_kernel(
    int64_t nrows, const int64_t* __restrict__ row_slot, const int64_t* __restrict__ row_ptr,
    const int2* __restrict__ ent, const double2* __restrict__ hat, const double2* __restrict__ symd,
    double2* __restrict__ local) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int NT = m2l_threads<L>();
    constexpr int PER = (P3 + NT - 1) / NT;
    extern __shared__ double2 sm[];
    double2* tw = sm;
    double2* X = tw + P;
    double2* Z1 = X + P3;
    const int64_t row = blockIdx.x;
    make_twiddles<P>(tw);
    double2 acc[PER], acc2[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) acc[m] = acc2[m] = make_double2(0.0, 0.0);
    const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
    int64_t e = e0;
    for (; e + 2 <= e1; e += 2) {
        const int2 a = ent[e], b = ent[e + 1];
        const double2* Sa = hat + (int64_t)a.x * P3;
        const double2* Da = symd + (int64_t)a.y * P3;
        const double2* Sb = hat + (int64_t)b.x * P3;
        const double2* Db = symd + (int64_t)b.y * P3;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int j = threadIdx.x + m * NT;
            if (j < P3) {
                const double2 sa = __ldg(Sa + j), da = __ldg(Da + j), sb = __ldg(Sb + j), db = __ldg(Db + j);
                acc[m] = cfma(da, sa, acc[m]);
                acc2[m] = cfma(db, sb, acc2[m]);
            }
        }
    }
    if (e < e1) {
        const int2 a = ent[e];
        const double2* Sa = hat + (int64_t)a.x * P3;
        const double2* Da = symd + (int64_t)a.y * P3;
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int j = threadIdx.x + m * NT;
            if (j < P3) acc[m] = cfma(__ldg(Da + j), __ldg(Sa + j), acc[m]);
        }
    }
#pragma unroll
    for (int m = 0; m < PER; ++m) {
        const int j = threadIdx.x + m * NT;
        if (j < P3) X[j] = cadd(acc[m], acc2[m]);
    }
    __syncthreads();
    f2l_row<L>(tw, X, Z1, local + row_slot[row] * L3);
}

// Run record of the grouped M2L: {source spectrum index, target mask, G
// derived-symbol ids (one per row of the group; unused where the mask bit is 0)}.
template <int L>
__host__ __device__ constexpr int m2l_run_words() { return m2l_group_size<L>() + 2; }

template <int L>
__global__ void __launch_bounds__(m2l_threads<L>()) m2l_grouped_kernel(
    int64_t ngroups, const int64_t* __restrict__ grp_rows, const int64_t* __restrict__ grp_ptr,
    const int32_t* __restrict__ runs, const double2* __restrict__ hat, const double2* __restrict__ symd,
    double2* __restrict__ local) {
    constexpr int P = pad<L>(), L3 = cube<L>(), P3 = P * P * P;
    constexpr int NT = m2l_threads<L>();
    constexpr int PER = (P3 + NT - 1) / NT;
    constexpr int G = m2l_group_size<L>();
    constexpr int W = m2l_run_words<L>();
    constexpr int CHUNK = 128;  // run records staged in shared memory per pass
    extern __shared__ double2 sm[];
    double2* tw = sm;
    double2* X = tw + P;
    double2* Z1 = X + P3;
    int32_t* rec = reinterpret_cast<int32_t*>(Z1 + L * P * P);  // CHUNK * W ints
    const int64_t g = blockIdx.x;
    make_twiddles<P>(tw);
    double2 acc[G][PER];
#pragma unroll
    for (int k = 0; k < G; ++k)
#pragma unroll
        for (int m = 0; m < PER; ++m) acc[k][m] = make_double2(0.0, 0.0);
    const int64_t r0 = grp_ptr[g], r1 = grp_ptr[g + 1];
    for (int64_t cb = r0; cb < r1; cb += CHUNK) {
        const int n = (int)((r1 - cb) < CHUNK ? (r1 - cb) : CHUNK);
        __syncthreads();
        for (int t = threadIdx.x; t < n * W; t += NT) rec[t] = runs[cb * W + t];
        __syncthreads();
        double2 S[PER], Sn[PER];
        {
            const double2* Sp = hat + (int64_t)rec[0] * P3;
#pragma unroll
            for (int m = 0; m < PER; ++m) {
                const int j = threadIdx.x + m * NT;
                S[m] = j < P3 ? __ldg(Sp + j) : make_double2(0.0, 0.0);
            }
        }
        for (int r = 0; r < n; ++r) {
            const int32_t* rr = rec + r * W;
            const unsigned mask = (unsigned)rr[1];
            // prefetch the next source spectrum
            // all symbol loads of this run + the next source in flight together
            double2 D[G][PER];
#pragma unroll
            for (int k = 0; k < G; ++k) {
                const double2* Dp = symd + (int64_t)rr[2 + k] * P3;
#pragma unroll
                for (int m = 0; m < PER; ++m) {
                    const int j = threadIdx.x + m * NT;
                    D[k][m] = ldg_pred(Dp + j, ((mask >> k) & 1) && j < P3);
                }
            }
            {
                const bool more = r + 1 < n;
                const double2* Sp = hat + (int64_t)(more ? rr[W] : 0) * P3;
#pragma unroll
                for (int m = 0; m < PER; ++m) {
                    const int j = threadIdx.x + m * NT;
                    Sn[m] = ldg_pred(Sp + j, more && j < P3);
                }
            }
            // register fence: every D load above is issued before any FMA below
#pragma unroll
            for (int k = 0; k < G; ++k)
#pragma unroll
                for (int m = 0; m < PER; ++m) asm volatile("" : "+d"(D[k][m].x), "+d"(D[k][m].y));
#pragma unroll
            for (int k = 0; k < G; ++k) {
                if ((mask >> k) & 1) {
#pragma unroll
                    for (int m = 0; m < PER; ++m) acc[k][m] = cfma(D[k][m], S[m], acc[k][m]);
                }
            }
#pragma unroll
            for (int m = 0; m < PER; ++m) S[m] = Sn[m];
        }
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
        const int64_t row = grp_rows[g * G + k];
        if (row < 0) break;
        __syncthreads();
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int j = threadIdx.x + m * NT;
            if (j < P3) X[j] = acc[k][m];
        }
        __syncthreads();
        f2l_row<L>(tw, X, Z1, local + row * L3);
    }
}

// ---------------------------------------------------------------------------
// K3: L2P + near-field add + un-permute.  One CTA per target leaf, one thread
// per particle; L2P(x) = sum_abc loc[abc] conj(W0_a W1_b W2_c) with the same
// per-axis weights as P2M.

template <int L>
__global__ void __launch_bounds__(64) l2p_kernel(
    int64_t n, const int32_t* __restrict__ leaf_cell, const int64_t* __restrict__ slot_lo,
    const int64_t* __restrict__ slot_hi, const int32_t* __restrict__ slot_dir,
    const int64_t* __restrict__ cstart, const int64_t* __restrict__ cstop,
    const double* __restrict__ calpha, const int32_t* __restrict__ clevel,
    const double* __restrict__ lbeta, const double* __restrict__ dirs, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, double kappa,
    const double2* __restrict__ local, const double2* __restrict__ near,
    const int64_t* __restrict__ perm, double2* __restrict__ out) {
    constexpr int L3 = cube<L>();
    constexpr int NT = 64;
    __shared__ double2 loc[L3];
    const int64_t i = blockIdx.x;
    const int c = leaf_cell[i];
    const double beta = lbeta[clevel[c]];
    const double al[3] = {calpha[3 * c], calpha[3 * c + 1], calpha[3 * c + 2]};
    const int64_t s0 = cstart[c], s1 = cstop[c];
    const int64_t k0 = slot_lo[i], k1 = slot_hi[i];
    for (int64_t base = s0; base < s1; base += NT) {
        const int64_t p = base + threadIdx.x;
        const bool valid = p < s1;
        double xh[3] = {0.0, 0.0, 0.0};
        if (valid) {
            xh[0] = (px[p] - al[0]) / beta;
            xh[1] = (py[p] - al[1]) / beta;
            xh[2] = (pz[p] - al[2]) / beta;
        }
        double S[3][L];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) lagrange<L>(xh[ax], S[ax]);
        double2 acc = valid ? near[p] : make_double2(0.0, 0.0);
        for (int64_t s = k0; s < k1; ++s) {
            const int d = slot_dir[s];
            __syncthreads();
            for (int r = threadIdx.x; r < L3; r += NT) loc[r] = local[s * L3 + r];
            __syncthreads();
            double2 W[3][L];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                const double ku = d >= 0 ? kappa * beta * dirs[3 * d + ax] : 0.0;
#pragma unroll
                for (int k = 0; k < L; ++k)
                    W[ax][k] = cscale(cexpi(ku * (xh[ax] - node<L>(k))), S[ax][k]);
            }
            double2 va = make_double2(0.0, 0.0);
#pragma unroll
            for (int a = 0; a < L; ++a) {
                double2 vb = make_double2(0.0, 0.0);
#pragma unroll
                for (int b = 0; b < L; ++b) {
                    double2 vc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int cc = 0; cc < L; ++cc) vc = cfma(loc[(a * L + b) * L + cc], W[2][cc], vc);
                    vb = cfma(vc, W[1][b], vb);
                }
                va = cfma(vb, W[0][a], va);
            }
            acc = cadd(acc, va);
        }
        if (valid) out[perm[p]] = acc;
    }
}

// ---------------------------------------------------------------------------
// K1: P2P.  One CTA per target leaf; `split` threads per target share the
// sources (fixed-order shuffle reduction); source runs staged in shared memory.

constexpr int P2P_NT = 128;
constexpr int P2P_TILE = 256;

__device__ __forceinline__ double2 helm_pair(double dx, double dy, double dz, double2 qs, double kpi,
                                             double tol) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double rinv = rsqrt(r2);  // r2 = 0 -> inf -> r = NaN -> masked below
    const double r = r2 * rinv;
    const bool ok = r >= tol;     // kernel.py:40-43 singularity suppression
    double s, c;
    sincospi(kpi * (ok ? r : 0.0), &s, &c);
    const double g = ok ? rinv * (1.0 / (4.0 * 3.141592653589793)) : 0.0;
    const double gr = g * c, gi = g * s;
    return make_double2(gr * qs.x - gi * qs.y, gr * qs.y + gi * qs.x);
}

__global__ void __launch_bounds__(P2P_NT) p2p_kernel(
    int64_t n, const int64_t* __restrict__ tgt_lo, const int64_t* __restrict__ tgt_hi,
    const int64_t* __restrict__ ptr, const int64_t* __restrict__ src_lo,
    const int64_t* __restrict__ src_hi, const double* __restrict__ tx,
    const double* __restrict__ ty, const double* __restrict__ tz, const double* __restrict__ px,
    const double* __restrict__ py, const double* __restrict__ pz, const double2* __restrict__ q,
    double kappa, double tol, double2* __restrict__ near) {
    __shared__ double sx[P2P_TILE], sy[P2P_TILE], sz[P2P_TILE];
    __shared__ double2 sq[P2P_TILE];
    const int64_t i = blockIdx.x;
    const int64_t t0 = tgt_lo[i], t1 = tgt_hi[i];
    const int64_t nt = t1 - t0;
    const int split = nt <= 16 ? 8 : nt <= 32 ? 4 : nt <= 64 ? 2 : 1;
    const int per_pass = P2P_NT / split;
    const double kpi = kappa / 3.141592653589793;
    const int64_t e0 = ptr[i], e1 = ptr[i + 1];
    for (int64_t tb = t0; tb < t1; tb += per_pass) {
        const int64_t t = tb + threadIdx.x / split;
        const int part = threadIdx.x % split;
        const bool valid = t < t1;
        const double xt = valid ? tx[t] : 0.0, yt = valid ? ty[t] : 0.0, zt = valid ? tz[t] : 0.0;
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t e = e0; e < e1; ++e) {
            const int64_t a = src_lo[e], b = src_hi[e];
            for (int64_t sb = a; sb < b; sb += P2P_TILE) {
                const int cnt = (int)((b - sb) < (int64_t)(P2P_TILE) ? (b - sb) : (int64_t)(P2P_TILE));
                __syncthreads();
                for (int k = threadIdx.x; k < cnt; k += P2P_NT) {
                    sx[k] = px[sb + k];
                    sy[k] = py[sb + k];
                    sz[k] = pz[sb + k];
                    sq[k] = q[sb + k];
                }
                __syncthreads();
                if (valid) {
                    for (int k = part; k < cnt; k += split) {
                        const double2 g = helm_pair(xt - sx[k], yt - sy[k], zt - sz[k], sq[k], kpi, tol);
                        acc.x += g.x;
                        acc.y += g.y;
                    }
                }
            }
        }
        for (int off = 1; off < split; off <<= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
        }
        if (valid && part == 0) near[t] = acc;
    }
}

// K10: direct sum, one thread per target, all sources tiled through smem.
__global__ void __launch_bounds__(128) direct_kernel(
    int64_t nt, const double* __restrict__ tx, const double* __restrict__ ty,
    const double* __restrict__ tz, int64_t ns, const double* __restrict__ sx,
    const double* __restrict__ sy, const double* __restrict__ sz, const double2* __restrict__ q,
    double kappa, double tol, double2* __restrict__ out) {
    __shared__ double ax[256], ay[256], az[256];
    __shared__ double2 aq[256];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = t < nt;
    const double x = valid ? tx[t] : 0.0, y = valid ? ty[t] : 0.0, z = valid ? tz[t] : 0.0;
    const double kpi = kappa / 3.141592653589793;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t sb = 0; sb < ns; sb += 256) {
        const int cnt = (int)((ns - sb) < (int64_t)(256) ? (ns - sb) : (int64_t)(256));
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
    if (valid) out[t] = acc;
}

// ---------------------------------------------------------------------------
// launch helpers

template <typename K>
int set_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return 0;
    return report(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                  "cudaFuncSetAttribute");
}

inline int grid_ok(int64_t n) { return n > 0 && n < (int64_t)1 << 31; }

#define DEFMM_DISPATCH_L(L, ...)           \
    switch (L) {                           \
        case 2: { constexpr int LL = 2; __VA_ARGS__; } break; \
        case 3: { constexpr int LL = 3; __VA_ARGS__; } break; \
        case 4: { constexpr int LL = 4; __VA_ARGS__; } break; \
        case 5: { constexpr int LL = 5; __VA_ARGS__; } break; \
        case 6: { constexpr int LL = 6; __VA_ARGS__; } break; \
        case 7: { constexpr int LL = 7; __VA_ARGS__; } break; \
        case 8: { constexpr int LL = 8; __VA_ARGS__; } break; \
        default: return -3;                \
    }

}  // namespace

extern "C" {

int defmm_abi_version(void) { return DEFMM_ABI_VERSION; }
const char* defmm_last_error(void) { return g_last_error; }

int defmm_p2m_c128(int32_t L, int64_t n, const int32_t* cell, const int32_t* dir, const int64_t* out_slot,
                   const int64_t* cell_start, const int64_t* cell_stop, const double* cell_alpha,
                   const int32_t* cell_level, const double* level_beta, const double* dirs,
                   const double* px, const double* py, const double* pz, const void* q, double kappa,
                   void* mult, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (p2m_kernel<LL><<<(unsigned)n, 128, 0, s>>>(
                            n, cell, dir, out_slot, cell_start, cell_stop, cell_alpha, cell_level,
                            level_beta, dirs, px, py, pz, (const double2*)q, kappa, (double2*)mult)));
    return report(cudaGetLastError(), "p2m");
}

int defmm_m2m_c128(int32_t L, int64_t n, const int64_t* out_slot, const int32_t* dir, const int64_t* son_slot,
                   double son_beta, const double* dirs, double kappa, void* mult, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (m2m_kernel<LL><<<(unsigned)n, nodal_threads<LL>(), 0, s>>>(
                            n, out_slot, dir, son_slot, son_beta, dirs, kappa, (double2*)mult)));
    return report(cudaGetLastError(), "m2m");
}

int defmm_l2l_c128(int32_t L, int64_t n, const int64_t* out_slot, const int8_t* octant, const int64_t* ptr,
                   const int64_t* src_slot, const int32_t* src_dir, double son_beta, const double* dirs,
                   double kappa, void* local, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (l2l_kernel<LL><<<(unsigned)n, nodal_threads<LL>(), 0, s>>>(
                            n, out_slot, octant, ptr, src_slot, src_dir, son_beta, dirs, kappa,
                            (double2*)local)));
    return report(cudaGetLastError(), "l2l");
}

int defmm_m2f_c128(int32_t L, int64_t n, const int64_t* src_slot, const void* mult, void* hat, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P + LL * LL * LL + LL * LL * P + LL * P * P);
        int rc = set_smem(m2f_kernel<LL>, bytes);
        if (rc) return rc;
        m2f_kernel<LL><<<(unsigned)n, 128, bytes, s>>>(n, src_slot, (const double2*)mult, (double2*)hat);
    });
    return report(cudaGetLastError(), "m2f");
}

int defmm_symbols_c128(int32_t L, int64_t n, const int32_t* tvec, const double* beta, double kappa, void* sym,
                       void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P + 2 * P * P * P);
        int rc = set_smem(symbols_kernel<LL>, bytes);
        if (rc) return rc;
        symbols_kernel<LL><<<(unsigned)n, 256, bytes, s>>>(n, tvec, beta, kappa, (double2*)sym);
    });
    return report(cudaGetLastError(), "symbols");
}

int defmm_m2l_c128(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                   const int32_t* e_src, const int32_t* e_sym, const int8_t* e_rid, const void* hat,
                   const void* sym, void* local, void* stream) {
    if (nrows == 0) return 0;
    if (!grid_ok(nrows)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P + P * P * P + LL * P * P);
        int rc = set_smem(m2l_kernel<LL>, bytes);
        if (rc) return rc;
        m2l_kernel<LL><<<(unsigned)nrows, m2l_threads<LL>(), bytes, s>>>(
            nrows, row_slot, row_ptr, e_src, e_sym, e_rid, (const double2*)hat, (const double2*)sym,
            (double2*)local);
    });
    return report(cudaGetLastError(), "m2l");
}

int defmm_expand_symbols_c128(int32_t L, int64_t n, const int32_t* canon, const int8_t* rid, const void* sym_canon,
                               void* sym_derived, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (expand_symbols_kernel<LL><<<(unsigned)n, 256, 0, s>>>(
                            n, canon, rid, (const double2*)sym_canon, (double2*)sym_derived)));
    return report(cudaGetLastError(), "expand_symbols");
}

int defmm_m2l_group_size(int32_t L) {
    int g = -3;
    DEFMM_DISPATCH_L(L, g = m2l_group_size<LL>());
    return g;
}

int defmm_m2l_grouped_c128(int32_t L, int64_t ngroups, const int64_t* grp_rows, const int64_t* grp_ptr,
                           const int32_t* runs, const void* hat, const void* sym_derived, void* local,
                           void* stream) {
    if (ngroups == 0) return 0;
    if (!grid_ok(ngroups)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P + P * P * P + LL * P * P) + sizeof(int32_t) * 128 * m2l_run_words<LL>();
        int rc = set_smem(m2l_grouped_kernel<LL>, bytes);
        if (rc) return rc;
        m2l_grouped_kernel<LL><<<(unsigned)ngroups, m2l_threads<LL>(), bytes, s>>>(
            ngroups, grp_rows, grp_ptr, runs, (const double2*)hat, (const double2*)sym_derived, (double2*)local);
    });
    return report(cudaGetLastError(), "m2l_grouped");
}

int defmm_m2l_rows_c128(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                        const int32_t* entries, const void* hat, const void* sym_derived, void* local,
                        void* stream) {
    if (nrows == 0) return 0;
    if (!grid_ok(nrows)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, {
        constexpr int P = 2 * LL - 1;
        const size_t bytes = sizeof(double2) * (P + P * P * P + LL * P * P);
        int rc = set_smem(m2l_rows_kernel<LL>, bytes);
        if (rc) return rc;
        m2l_rows_kernel<LL><<<(unsigned)nrows, m2l_threads<LL>(), bytes, s>>>(
            nrows, row_slot, row_ptr, (const int2*)entries, (const double2*)hat, (const double2*)sym_derived,
            (double2*)local);
    });
    return report(cudaGetLastError(), "m2l_rows");
}

int defmm_l2p_c128(int32_t L, int64_t n, const int32_t* leaf_cell, const int64_t* slot_lo, const int64_t* slot_hi,
                   const int32_t* slot_dir, const int64_t* cell_start, const int64_t* cell_stop,
                   const double* cell_alpha, const int32_t* cell_level, const double* level_beta,
                   const double* dirs, const double* px, const double* py, const double* pz, double kappa,
                   const void* local, const void* near, const int64_t* perm, void* out, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    DEFMM_DISPATCH_L(L, (l2p_kernel<LL><<<(unsigned)n, 64, 0, s>>>(
                            n, leaf_cell, slot_lo, slot_hi, slot_dir, cell_start, cell_stop, cell_alpha,
                            cell_level, level_beta, dirs, px, py, pz, kappa, (const double2*)local,
                            (const double2*)near, perm, (double2*)out)));
    return report(cudaGetLastError(), "l2p");
}

int defmm_p2p_c128(int64_t n, const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* ptr,
                   const int64_t* src_lo, const int64_t* src_hi, const double* tx, const double* ty,
                   const double* tz, const double* sx, const double* sy, const double* sz, const void* q,
                   double kappa, double tol, void* near, void* stream) {
    if (n == 0) return 0;
    if (!grid_ok(n)) return -1;
    p2p_kernel<<<(unsigned)n, P2P_NT, 0, (cudaStream_t)stream>>>(n, tgt_lo, tgt_hi, ptr, src_lo, src_hi, tx, ty,
                                                                 tz, sx, sy, sz, (const double2*)q, kappa,
                                                                 tol, (double2*)near);
    return report(cudaGetLastError(), "p2p");
}

int defmm_direct_c128(int64_t nt, const double* tx, const double* ty, const double* tz, int64_t ns,
                      const double* sx, const double* sy, const double* sz, const void* q, double kappa,
                      double tol, void* out, void* stream) {
    if (nt == 0) return 0;
    const int64_t blocks = (nt + 127) / 128;
    if (!grid_ok(blocks)) return -1;
    direct_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(nt, tx, ty, tz, ns, sx, sy, sz,
                                                                      (const double2*)q, kappa, tol,
                                                                      (double2*)out);
    return report(cudaGetLastError(), "direct");
}

}  // extern "C"
