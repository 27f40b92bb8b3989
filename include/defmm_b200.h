/*
 * defmm_b200.h -- C-ABI of the B200-native defmm FMM matvec (libdefmm_b200.so).
 *
 * The reference (helmfmm, a pure-Python/numpy package) has no FFI layer: its
 * boundary is the Python API.  These entry points are the
 * native operators underneath that API; each one replaces the reference
 * function named in its comment.  Conventions:
 *   - all array pointers are DEVICE pointers owned by the caller (torch
 *     tensors on the host side), except the defmm_tree_* calls (HOST memory);
 *   - complex arrays are interleaved (re, im) pairs: double2 for "c128";
 *   - `stream` is a cudaStream_t passed as void*; nothing synchronises, nothing
 *     allocates device memory, every call is re-entrant per stream;
 *   - return value 0 = success, > 0 = a cudaError_t, < 0 = invalid argument.
 * Orders 2 <= L <= 8 are compiled (P = 2L-1).
 */
#ifndef DEFMM_B200_H
#define DEFMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DEFMM_ABI_VERSION 1

int defmm_abi_version(void);
/* last CUDA error string seen by the library (thread-local), for messages */
const char* defmm_last_error(void);

/* ---- host: octree build -------------------------------------------------
 * Replaces tree.py:132-213 (build_tree's recursive stable octant split with
 * FP64 `p >= centre` tests, centre = (lower + coords*beta) + 0.5*beta).
 * pts: n x 3 row-major doubles.  Output cells come in creation (DFS) order. */
typedef struct defmm_tree defmm_tree;
int defmm_tree_build(const double* pts, int64_t n, const double lower[3], double side,
                     int32_t ncrit, int32_t depth_cap, defmm_tree** out);
int64_t defmm_tree_ncells(const defmm_tree* t);
/* perm[n]: sorted -> input index; sorted_pts[n*3]; per cell: level, coords[3],
 * start, stop, parent (-1 for the root) */
int defmm_tree_fetch(const defmm_tree* t, int64_t* perm, double* sorted_pts, int32_t* level,
                     int64_t* coords, int64_t* start, int64_t* stop, int64_t* parent);
void defmm_tree_free(defmm_tree* t);

/* ---- device operators (complex128) --------------------------------------
 * Shared geometry arrays: cell_alpha[ncell*3] lower corners, cell_level[ncell],
 * level_beta[depth+1] side lengths, cell_start/stop particle ranges (sorted
 * order), dirs[ndir*3] unit directions (global ids; -1 = low frequency),
 * particles px/py/pz (sorted order), q (double2). */

/* K2 P2M -- interpolation.py:109-124 via traversal.py:224-236.
 * For i < n: mult[out_slot[i]] = P2M(cell[i], direction dir[i]). */
int defmm_p2m_c128(int32_t L, int64_t n, const int32_t* cell, const int32_t* dir,
                   const int64_t* out_slot, const int64_t* cell_start, const int64_t* cell_stop,
                   const double* cell_alpha, const int32_t* cell_level, const double* level_beta,
                   const double* dirs, const double* px, const double* py, const double* pz,
                   const void* q, double kappa, void* mult, void* stream);

/* K4 M2M -- traversal.py:239-280 + interpolation.py:140-200.
 * For i < n: mult[out_slot[i]] = sum over octants o with son_slot[8i+o] >= 0
 * of (C0 (x) C1 (x) C2) mult[son_slot[8i+o]], C the modulated per-axis factors
 * (dir[i] < 0: plain Lagrange factors).  son_beta = side of the son level. */
int defmm_m2m_c128(int32_t L, int64_t n, const int64_t* out_slot, const int32_t* dir,
                   const int64_t* son_slot, double son_beta, const double* dirs, double kappa,
                   void* mult, void* stream);

/* K6 M2F -- fourier.py:67-72 (pad L^3 -> P^3 corner, fftn / P^1.5).
 * For i < n: hat[i] = M2F(mult[src_slot[i]]). */
int defmm_m2f_c128(int32_t L, int64_t n, const int64_t* src_slot, const void* mult, void* hat,
                   void* stream);

/* K9 symbols -- fourier.py:156-183 (unnormalised fftn of G(beta (t + z))).
 * For i < n: sym[i] = symbol(t = tvec[3i..3i+2], beta[i]). */
int defmm_symbols_c128(int32_t L, int64_t n, const int32_t* tvec, const double* beta,
                       double kappa, void* sym, void* stream);

/* K7+K8 Hadamard M2L + fused F2L -- traversal.py:320-342 (m2l_hadamard,
 * fourier.py:83-87) and traversal.py:405-414 (f2l, fourier.py:74-80).
 * For row r < nrows: local[row_slot[r]] = F2L( sum_{e in [row_ptr[r], row_ptr[r+1])}
 *   Dperm(sym[e_sym[e]], e_rid[e]) (*) hat[e_src[e]] ), Dperm = canonical symbol
 * gathered through the 48-element cube-group frequency map (fourier.py:123-143). */
int defmm_m2l_c128(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                   const int32_t* e_src, const int32_t* e_sym, const int8_t* e_rid,
                   const void* hat, const void* sym, void* local, void* stream);

/* K9b derived symbols -- fourier.py:186-196 (permute_symbol) materialised:
 * sym_derived[i] = sym_canon[canon[i]] gathered through rotation rid[i]. */
int defmm_expand_symbols_c128(int32_t L, int64_t n, const int32_t* canon, const int8_t* rid,
                              const void* sym_canon, void* sym_derived, void* stream);

/* rows per M2L group compiled for order L (8, 4 or 2) */
int defmm_m2l_group_size(int32_t L);

/* K7+K8 v2 (product path): grouped Hadamard M2L + fused F2L.  Group g owns
 * the target rows grp_rows[G*g .. G*g+G) (-1 padded, G = defmm_m2l_group_size),
 * siblings sharing a parent cell and a key.  Its runs [grp_ptr[g], grp_ptr[g+1])
 * are records of G+2 int32: {source spectrum index, row mask, derived-symbol
 * index for each row of the mask}, one per distinct source.
 * local[grp_rows[..]] = F2L(sum D (*) hat). */
int defmm_m2l_grouped_c128(int32_t L, int64_t ngroups, const int64_t* grp_rows,
                           const int64_t* grp_ptr, const int32_t* runs, const void* hat,
                           const void* sym_derived, void* local, void* stream);

/* K7+K8 v1b: row-major Hadamard M2L over derived symbols + fused F2L.  Row r
 * (target slot row_slot[r]) owns entries [row_ptr[r], row_ptr[r+1]), int32
 * pairs {source spectrum index, derived-symbol index}. */
int defmm_m2l_rows_c128(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                        const int32_t* entries, const void* hat, const void* sym_derived,
                        void* local, void* stream);

/* K5 L2L -- traversal.py:355-391 in gather form.
 * For i < n: local[out_slot[i]] += sum_{e in [ptr[i], ptr[i+1])}
 *   (C'0 (x) C'1 (x) C'2) local[src_slot[e]], C' the transposed/conjugate-
 * modulated factors of direction src_dir[e] for son octant octant[i]. */
int defmm_l2l_c128(int32_t L, int64_t n, const int64_t* out_slot, const int8_t* octant,
                   const int64_t* ptr, const int64_t* src_slot, const int32_t* src_dir,
                   double son_beta, const double* dirs, double kappa, void* local, void* stream);

/* K3 L2P + un-permute -- interpolation.py:127-137 via traversal.py:394-402,
 * tree.py:224-228.  For leaf i < n: for p in [cell_start, cell_stop):
 *   out[perm[p]] = near[p] + sum_{s in [slot_lo[i], slot_hi[i])} L2P(local[s], slot_dir[s]). */
int defmm_l2p_c128(int32_t L, int64_t n, const int32_t* leaf_cell, const int64_t* slot_lo,
                   const int64_t* slot_hi, const int32_t* slot_dir, const int64_t* cell_start,
                   const int64_t* cell_stop, const double* cell_alpha, const int32_t* cell_level,
                   const double* level_beta, const double* dirs, const double* px,
                   const double* py, const double* pz, double kappa, const void* local,
                   const void* near, const int64_t* perm, void* out, void* stream);

/* K1 P2P -- traversal.py:303-317 + kernel.py:37-55.  For target leaf i < n:
 * near[p] = sum over source ranges [src_lo[e], src_hi[e]), e in [ptr[i], ptr[i+1]),
 * of G(|x_p - y_s|) q_s for p in [tgt_lo[i], tgt_hi[i]); G = 0 for r < tol.
 * Targets t*, sources s* (the same arrays in single-tree mode). */
int defmm_p2p_c128(int64_t n, const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* ptr,
                   const int64_t* src_lo, const int64_t* src_hi, const double* tx,
                   const double* ty, const double* tz, const double* sx, const double* sy,
                   const double* sz, const void* q, double kappa, double tol, void* near,
                   void* stream);

/* K10 direct sum -- kernel.py:58-75: out[i] = sum_s G(|t_i - y_s|) q_s. */
int defmm_direct_c128(int64_t nt, const double* tx, const double* ty, const double* tz,
                      int64_t ns, const double* sx, const double* sy, const double* sz,
                      const void* q, double kappa, double tol, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DEFMM_B200_H */
