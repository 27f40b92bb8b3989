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

/* ---- host: dual tree traversal (plan lists) ------------------------------
 * Replaces the reference's recursive DTT (traversal.py:320-348, whose HF pair
 * set equals blank_dtt traversal.py:182-200) for one (target, source) tree
 * pair on a common grid.  Trees are level-major arrays (HOST memory):
 * level_off[depth+2], coords[ncell*3], first_son, n_sons, parent.  Per level l:
 * M2L iff gap^2 >= g2min[l] (the reference MAC, traversal.py:100-113, as an
 * exact integer threshold); key = key_tab[tab_off[l] + dense(t_vec)] with
 * dense(t) = ((t0+R)(2R+1) + t1+R)(2R+1) + t2+R over |t|_inf <= R[l]
 * (nearest direction, directions.py:78-89; -1 at LF levels); P2P iff either
 * cell is a leaf (traversal.py:336-343); else recurse into sons x sons.
 * Returns -4 when a translation falls outside its level's key table. */
typedef struct defmm_dtt defmm_dtt;
int defmm_dtt_build(const int64_t* t_level_off, int32_t t_depth, const int64_t* t_coords,
                    const int64_t* t_first_son, const int64_t* t_nsons, const int64_t* t_parent,
                    const int64_t* s_level_off, int32_t s_depth, const int64_t* s_coords,
                    const int64_t* s_first_son, const int64_t* s_nsons, const int64_t* s_parent,
                    int32_t depth, const int64_t* g2min, const int32_t* R, const int64_t* tab_off,
                    const int32_t* key_tab, defmm_dtt** out);
/* sizes[6] = {M2L events, rows, groups, blocks, P2P events, translations} */
int defmm_dtt_sizes(const defmm_dtt* d, int64_t* sizes);
/* rows = distinct (target, key) in (level, target, key) order, row_ptr[rows+1]
 * over the events (ev_s source cell, ev_trans translation id); groups =
 * (level, key, target parent) with grp_rows[8*g + octant] = row id or -1 and
 * grp_ptr[groups+1] over the blocks; block = (group, source parent) with
 * blk_src[8*b + octant] = event id or -1, blk_trans[27*b + child offset] =
 * translation id or -1, blk_mask bit 8a+b = pair (a, b) is an event.
 * Translation ids (ev_trans, blk_trans) rank the distinct (level, t_vec) in
 * dense-table order; defmm_dtt_translations lists their dense indices.
 * P2P events (p_t, p_s).  Any pointer may be NULL (not copied). */
int defmm_dtt_fetch(const defmm_dtt* d, int32_t* ev_s, int32_t* ev_trans, int64_t* row_ptr,
                    int32_t* row_t, int32_t* row_key, int32_t* row_lev, int64_t* grp_rows,
                    int32_t* grp_p, int32_t* grp_key, int32_t* grp_lev, int64_t* grp_ptr,
                    int64_t* blk_src, int32_t* blk_trans, int64_t* blk_mask, int32_t* p_t,
                    int32_t* p_s);
int defmm_dtt_translations(const defmm_dtt* d, int64_t* dense_ids);
/* Spectrum index of every M2L event's source expansion (the M2F list,
 * fourier.py:67-72 applied once per used multipole): slot = m_dense[base[l] +
 * (ev_s - s_level_off[l]) * nd[l] + loc], loc = row key - key_base[l] (0 at LF
 * levels); hat_slot[0..*n_hat) = the used slots ascending (capacity n_mult),
 * src_hat[event] = rank of its slot.  -6 if an event has no source expansion. */
int defmm_dtt_source_hats(const defmm_dtt* d, const int64_t* m_dense, const int64_t* base, const int64_t* nd,
                          const int64_t* s_level_off, const int32_t* key_base, int64_t n_mult,
                          int32_t* src_hat, int64_t* hat_slot, int64_t* n_hat);
void defmm_dtt_free(defmm_dtt* d);

/* ---- device: plan construction -----------------------
 * defmm_tree_keys -- tree.py:132-213's octant decisions per particle: keys[i] =
 * the octant path of pts[i] (n x 3 row-major doubles, DEVICE) to `depth` <= 21
 * levels, 3 bits per level, level 0 in the highest bits; octant = 4 (x >= cx) +
 * 2 (y >= cy) + (z >= cz), centre = (lower + coords * beta) + 0.5 * beta with
 * every FP64 product and sum rounded separately (bit-identical to tree.py:165-166,
 * geometry.py:71-72).  lower[3] is HOST memory.
 * defmm_dtt_classify -- one level of the dual tree traversal (traversal.py:320-348)
 * over n candidate pairs (pair_t[i], pair_s[i]) of same-level cells (all arrays
 * DEVICE): kind[i] = 0 M2L (integer gap^2 >= g2min, the reference MAC as in
 * defmm_dtt_build), 1 P2P (else, either cell a leaf), 2 expand (nexp[i] = sons x
 * sons pairs); for M2L pairs dense[i] = tab_off + dense(t - s) over |t|_inf <= R and
 * key[i] = key_tab[dense[i]]; *status = 1 if a translation leaves the table. */
int defmm_tree_keys(int64_t n, const double* pts, const double lower[3], double side, int32_t depth,
                    int64_t* keys, void* stream);
int defmm_dtt_classify(int64_t n, const int64_t* pair_t, const int64_t* pair_s, const int64_t* t_coords,
                       const int64_t* s_coords, const int64_t* t_nsons, const int64_t* s_nsons, int64_t g2min,
                       int32_t R, int64_t tab_off, const int32_t* key_tab, int8_t* kind, int32_t* key,
                       int64_t* dense, int64_t* nexp, int32_t* status, void* stream);

/* ---- host: stage packing of the staged M2L (K7 v13) --------------------------
 * Classes c < ncls (ordered; cls_cta[c] non-decreasing) read the symbols
 * cls_sym[cls_ptr[c] .. cls_ptr[c+1]) (ids < n_sym_ids).  Greedy, in order: a
 * class joins the current stage of its CTA while the stage's DISTINCT symbols
 * stay <= ns_cap, else it opens the next one.  cls_stage_rel[c] = stage index
 * within the CTA.  -2 if a class alone exceeds ns_cap. */
int defmm_stage_pack(int64_t ncls, const int64_t* cls_cta, const int64_t* cls_ptr, const int64_t* cls_sym,
                     int64_t n_sym_ids, int32_t ns_cap, int64_t* cls_stage_rel);

/* ---- FMA peak probe (measurement only) --------------------------------------
 * Launches 4 x SMs CTAs of 256 threads, each thread running 8 independent FMA
 * chains for iters x 16 steps: flops = 2 * 8 * 16 * iters * threads.  fp64
 * selects double.  out: one element, written only to keep the chains live. */
int defmm_fma_peak(int32_t fp64, int64_t iters, void* out, void* stream);

/* ---- L2 -> SM streaming probe (measurement only) ---------------------------
 * ctas_per_sm x SMs CTAs of 512 threads read the n_vec 16-B vectors of buf
 * (an L2-resident buffer) iters times with L2-only cached 128-bit loads:
 * bytes moved L2 -> SM = 16 * n_vec * iters (rounded up to whole passes of
 * 4 x grid vectors).  out: one float, written only to keep the loads live. */
int defmm_l2_stream(const void* buf, int64_t n_vec, int32_t iters, int32_t ctas_per_sm, void* out, void* stream);

/* ---- device operators ------------------------------------------------------
 * Every operator exists as *_c128 (complex arrays are double2 = interleaved
 * FP64 re/im, exactly the reference's complex128; all arithmetic FP64) and
 * *_c64 (float2 storage).  What the c64 operators compute in: cell-relative
 * coordinates (x - alpha)/beta and target-relative P2P differences are formed
 * in FP64 and rounded once (hi/lo float pairs in the P2P at L >= 6); the
 * P2M/M2M/L2L tensor sums, the M2F, the Hadamard M2L products and per-row
 * sums, and the P2P pair terms and per-target sums are FP32; the F2L inverse
 * transform, the L2P sum and the near + far combine are FP64.
 * Shared geometry arrays: cell_alpha[ncell*3] lower corners, cell_level[ncell],
 * level_beta[depth+1] side lengths, cell_start/stop particle ranges (sorted
 * order), dirs[ndir*3] unit directions (global ids; -1 = low frequency),
 * particles px/py/pz (FP64, sorted order), q charges.
 *
 * K2 P2M -- interpolation.py:109-124 via traversal.py:224-236.
 *   for i < n: mult[out_slot[i]] = P2M(cell[i], direction dir[i])
 * K4 M2M -- traversal.py:239-280 + interpolation.py:140-200.
 *   for i < n: mult[out_slot[i]] = sum over octants o with son_slot[8i+o] >= 0 of
 *   (C0 (x) C1 (x) C2) mult[son_slot[8i+o]], C the modulated per-axis factors of
 *   direction dir[i] (< 0: plain Lagrange factors); son_beta = son-level side.
 * K6 M2F -- fourier.py:67-72 (pad L^3 -> P^3 corner, fftn / P^1.5).
 *   for i < n: hat[i] = M2F(mult[src_slot[i]])
 * K9 symbols -- fourier.py:156-183 (unnormalised fftn of G(beta (t + z))).
 *   for i < n: sym[i] = symbol(t = tvec[3i..3i+2], beta[i]) (computed in FP64)
 * K9b derived symbols -- fourier.py:186-196 (permute_symbol) materialised:
 *   sym_derived[i] = sym_canon[canon[i]] gathered through rotation rid[i]
 * K7+K8 Hadamard M2L + fused F2L -- traversal.py:320-342 (m2l_hadamard,
 *   fourier.py:83-87) and traversal.py:405-414 (f2l, fourier.py:74-80).
 *   Row r (target slot row_slot[r]) owns entries [row_ptr[r], row_ptr[r+1]),
 *   int32 pairs {source spectrum index, derived-symbol index}:
 *   local[row_slot[r]] = F2L(sum_e sym_derived[e.sym] (*) hat[e.src])
 * K7 v3 blocked M2L (product path) -- the same sums grouped in parent-pair blocks:
 *   group g = (target parent, key) owns rows grp_rows[8g+a] (row index into lhat,
 *   -1 absent) and blocks [grp_ptr[g], grp_ptr[g+1]); block k = (source parent)
 *   holds spectra blk_src[8k+b] (-1 absent), derived symbols blk_trans[27k+d]
 *   for child offset d = (a-b)+(1,1,1) in base 3, and blk_mask[k] with bit 8a+b
 *   set for every M2L event (a, b); blk_kind[k] (or NULL = all general) = -1 for a
 *   general block, 2p+v for a PLANAR block whose pairs all have a_p = b_p = v
 *   (surface data: 4x4 in-plane pairs, no predicated-off pair).  lhat[row] = sum D (*) hat  (stride
 *   defmm_spectrum_stride);  then K8 f2l_rows: local[row_slot[r]] = F2L(lhat[r]).
 *   K7 v8 sibling-group variant (m2l_group, K = 2, 3 or 4 rows): CTA g = rows
 *   grp_slot[K g + k] (local slots; trailing -1 when the group is short);
 *   entry e in [grp_ptr[g], grp_ptr[g+1]) = entries[S e .. S e + K] (S = 4 for
 *   K = 2, 8 for K = 4) = {source spectrum, derived symbol for row k or -1
 *   (k < K), 0 padding}; local[slot] = F2L(sum) -- the row kernel's sums,
 *   merged per source.
 *   K7 v13 staged variant (m2l_stage): CTA c = 8 "warp units" (a target parent's <= 4
 *   sibling rows each, same level and key, neighbouring parents) x one spectral slice of
 *   <= 32 16-B vectors (grid = ncta x slices of the order).  Its stages
 *   [cta_stage[c], cta_stage[c+1]) hold the derived symbols slot_sym[stage_slot_ptr[s] ..
 *   stage_slot_ptr[s+1]) (<= ns_cap per stage), copied once per CTA into a shared-memory
 *   ring of `depth` stages (2..8; depth x (ns_cap+1) slices must fit 227 KB);
 *   warp unit w of CTA c owns the entries [cta_went[8c+w], ...) = int32 pairs {source
 *   spectrum, 4 bytes: shared-memory slot of row k's symbol, ns_cap = none}, those of stage s
 *   ending at stage_wend[8 cta_stage[c] + w n_c + (s - cta_stage[c])], n_c = the CTA's stage count
 *   (the entry array is readable 64 entries past its end);
 *   lhat[cta_rows[4(8c+w)+k]] = sum (row index, -1 absent); then K8 f2l_rows.
 * K5 L2L -- traversal.py:355-391 in gather form.
 *   for i < n: local[out_slot[i]] += sum_{e in [ptr[i], ptr[i+1])}
 *   (C'0 (x) C'1 (x) C'2) local[src_slot[e]], C' the transposed/conjugate-
 *   modulated factors of direction src_dir[e] for son octant octant[i].
 * K3 L2P + un-permute -- interpolation.py:127-137 via traversal.py:394-402,
 *   tree.py:224-228.  For leaf i < n, p in [cell_start, cell_stop):
 *   out[perm[p]] = near[p] + sum_{s in [slot_lo[i], slot_hi[i])} L2P(local[s], slot_dir[s]).
 * K1 P2P -- traversal.py:303-317 + kernel.py:37-55.  Target leaf l owns the merged
 *   source runs [src_lo[e], src_hi[e]), e in [ptr[l], ptr[l+1]); their concatenation
 *   is cut into work items i < n_items = (item_leaf[i], flattened range
 *   [item_f0[i], item_f1[i])).  For p in [tgt_lo[l], tgt_hi[l]) an item computes
 *   sum_s G(|x_p - y_s|) q_s (G = 0 for r < tol) into near[p] when
 *   item_out[i] < 0 (the leaf's only item), else into
 *   partial[item_out[i] + p - tgt_lo[l]]; the n_split split leaves are then
 *   reduced in item order: near[p] = sum_{m < split_n} partial[split_base + m*nt + ...].
 *   Targets t*, sources s* (the same arrays in single-tree mode).  grid > 0 launches
 *   a persistent grid of `grid` CTAs striding over the items (so the P2P leaves SM
 *   room for the far-field kernels running concurrently on another stream);
 *   grid = 0 launches one CTA per item.  Results do not depend on grid.  hilo
 *   (c64 only): 1 = hi/lo float pairs of the target-relative coordinates
 *   (accuracy for L >= 6), 0 = single floats (cheaper; L <= 5).
 * K1 v2 mutual P2P (single-tree plans: targets == sources) -- the same sums with every
 *   G(|x_t - x_s|) evaluated once for the pair (t, s), s after t's leaf: leaf l's source
 *   runs are clipped to particles >= tgt_lo[l] (its own particles first, evaluated
 *   one-directionally); item i = (item_leaf[i], flattened range [item_f0[i], item_f1[i]))
 *   writes its nt row sums to partial[item_row[i] ..] and, for every listed source, the
 *   column sum  sum_t G q_t  to partial[item_col[i] + (f - item_f0[i])].  p2p_gather task
 *   j (leaf l = task_leaf[j]) then forms out[x] = sum_c partial[cbase[c] + x] over its
 *   contributor segments c in [cptr[j], cptr[j+1]) with cxlo[c] <= x < cxhi[c], in list
 *   order (the row partials of the leaf's items, the column partials of the items that
 *   listed it); out = near + tgt_lo[l] if task_out[j] < 0, else partial + task_out[j] (very
 *   long lists are pre-summed in chunks by earlier gather launches).
 *   Leaves must hold <= 256 particles.  No atomics: reruns are bitwise identical.
 */
#define DEFMM_DECLARE_TYPED(SUFFIX)                                                              \
    int defmm_p2m_##SUFFIX(int32_t L, int64_t n, const int32_t* cell, const int32_t* dir,        \
                           const int64_t* out_slot, const int64_t* cell_start,                  \
                           const int64_t* cell_stop, const double* cell_alpha,                  \
                           const int32_t* cell_level, const double* level_beta,                 \
                           const double* dirs, const double* px, const double* py,              \
                           const double* pz, const void* q, double kappa, void* mult,           \
                           void* stream);                                                       \
    int defmm_m2m_##SUFFIX(int32_t L, int64_t n, const int64_t* out_slot, const int32_t* dir,    \
                           const int64_t* son_slot, double son_beta, const double* dirs,        \
                           double kappa, void* mult, void* stream);                             \
    int defmm_m2f_##SUFFIX(int32_t L, int64_t n, const int64_t* src_slot, const void* mult,      \
                           void* hat, void* stream);                                            \
    int defmm_symbols_##SUFFIX(int32_t L, int64_t n, const int32_t* tvec, const double* beta,    \
                               double kappa, void* sym, void* stream);                          \
    int defmm_expand_symbols_##SUFFIX(int32_t L, int64_t n, const int32_t* canon,                \
                                      const int8_t* rid, const void* sym_canon,                 \
                                      void* sym_derived, void* stream);                         \
    int defmm_m2l_rows_##SUFFIX(int32_t L, int64_t nrows, const int64_t* row_slot,               \
                                const int64_t* row_ptr, const int32_t* entries,                 \
                                const void* hat, const void* sym_derived, void* local,          \
                                void* stream);                                                  \
    int defmm_m2l_group_##SUFFIX(int32_t L, int32_t K, int64_t ngroups, const int64_t* grp_slot,  \
                                 const int64_t* grp_ptr, const int32_t* entries, const void* hat, \
                                 const void* sym_derived, void* local, void* stream);             \
    int defmm_m2l_stage_##SUFFIX(int32_t L, int64_t ncta, int32_t ns_cap, int32_t depth,             \
                                 const int32_t* cta_stage,                                          \
                                 const int32_t* cta_went, const int32_t* stage_slot_ptr,            \
                                 const int32_t* slot_sym, const int32_t* stage_wend,                \
                                 const int32_t* entries, const int32_t* cta_rows, const void* hat,  \
                                 const void* sym_derived, void* lhat, void* stream);                \
    int defmm_m2l_blocked_##SUFFIX(int32_t L, int64_t ngroups, const int64_t* grp_ptr,           \
                                   const int64_t* grp_rows, const int32_t* blk_src,             \
                                   const int32_t* blk_trans, const int64_t* blk_mask,           \
                                   const int8_t* blk_kind, const void* hat,                     \
                                   const void* sym_derived, void* lhat, void* stream);          \
    int defmm_f2l_rows_##SUFFIX(int32_t L, int64_t nrows, const int64_t* row_slot,               \
                                const void* lhat, void* local, void* stream);                   \
    int defmm_l2l_##SUFFIX(int32_t L, int64_t n, const int64_t* out_slot, const int8_t* octant,  \
                           const int64_t* ptr, const int64_t* src_slot, const int32_t* src_dir, \
                           double son_beta, const double* dirs, double kappa, void* local,      \
                           void* stream);                                                       \
    int defmm_l2p_##SUFFIX(int32_t L, int64_t n, const int32_t* leaf_cell,                       \
                           const int64_t* slot_lo, const int64_t* slot_hi,                      \
                           const int32_t* slot_dir, const int64_t* cell_start,                  \
                           const int64_t* cell_stop, const double* cell_alpha,                  \
                           const int32_t* cell_level, const double* level_beta,                 \
                           const double* dirs, const double* px, const double* py,              \
                           const double* pz, double kappa, const void* local, const void* near, \
                           const int64_t* perm, void* out, void* stream);                       \
    int defmm_p2p_mutual_##SUFFIX(int64_t n_items, const int32_t* item_leaf, const int64_t* item_f0, \
                                  const int64_t* item_f1, const int64_t* item_row,                   \
                                  const int64_t* item_col, const int64_t* tgt_lo,                    \
                                  const int64_t* tgt_hi, const int64_t* ptr, const int64_t* src_lo,  \
                                  const int64_t* src_hi, const double* px, const double* py,         \
                                  const double* pz, const void* q, double kappa, double tol,         \
                                  void* partial, int32_t grid, int32_t hilo, void* stream);          \
    int defmm_p2p_gather_##SUFFIX(int64_t n, const int32_t* task_leaf, const int64_t* task_out,      \
                                  const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* cptr, \
                                  const int64_t* cbase, const int32_t* cxlo, const int32_t* cxhi,    \
                                  void* partial, void* near, void* stream);                          \
    int defmm_p2p_##SUFFIX(int64_t n_items, const int32_t* item_leaf, const int64_t* item_f0,    \
                           const int64_t* item_f1, const int64_t* item_out,                     \
                           const int64_t* tgt_lo, const int64_t* tgt_hi, const int64_t* ptr,    \
                           const int64_t* src_lo, const int64_t* src_hi, const double* tx,      \
                           const double* ty, const double* tz, const double* sx,                \
                           const double* sy, const double* sz, const void* q, double kappa,     \
                           double tol, void* near, void* partial, int64_t n_split,              \
                           const int32_t* split_leaf, const int64_t* split_base,                \
                           const int32_t* split_n, int32_t grid, int32_t hilo,                  \
                           void* stream);

/* expands to: defmm_p2m_c128 defmm_m2m_c128 defmm_m2f_c128 defmm_symbols_c128
 * defmm_expand_symbols_c128 defmm_m2l_rows_c128 defmm_m2l_group_c128 defmm_m2l_stage_c128 defmm_m2l_blocked_c128
 * defmm_f2l_rows_c128 defmm_l2l_c128 defmm_l2p_c128 defmm_p2p_c128 defmm_p2p_mutual_c128
 * defmm_p2p_gather_c128 */
DEFMM_DECLARE_TYPED(c128)
/* expands to: defmm_p2m_c64 defmm_m2m_c64 defmm_m2f_c64 defmm_symbols_c64
 * defmm_expand_symbols_c64 defmm_m2l_rows_c64 defmm_m2l_group_c64 defmm_m2l_stage_c64 defmm_m2l_blocked_c64
 * defmm_f2l_rows_c64 defmm_l2l_c64 defmm_l2p_c64 defmm_p2p_c64 defmm_p2p_mutual_c64
 * defmm_p2p_gather_c64 */
DEFMM_DECLARE_TYPED(c64)

/* Spectral layout of order L (HOST call, no device needed): every spectrum is
 * stored in orbit order, forder[pos] = natural frequency f0 P^2 + f1 P + f2 at
 * storage position pos < P^3; slices [slice_start[k], slice_start[k+1]),
 * k < *nslices, are unions of cube-group orbits of <= 128 positions. */
int defmm_spectral_layout(int32_t L, int32_t* forder, int32_t* slice_start, int32_t* nslices);

/* K7 reference variant (c128): canonical symbols gathered through the closed-
 * form rotation inside the loop (e_sym canonical id, e_rid rotation id). */
int defmm_m2l_canon_c128(int32_t L, int64_t nrows, const int64_t* row_slot, const int64_t* row_ptr,
                         const int32_t* e_src, const int32_t* e_sym, const int8_t* e_rid,
                         const void* hat, const void* sym, void* local, void* stream);

/* Entries between consecutive P^3 spectra (hat, sym, sym_derived): P^3 for
 * c128, P^3 rounded up to even for c64 (aligned 16-B vector loads; the pad
 * entry is written as 0). */
int defmm_spectrum_stride(int32_t L, int32_t c64);

/* K10 direct sum -- kernel.py:58-75: out[i] = sum_s G(|t_i - y_s|) q_s (FP64).
 * workspace: defmm_direct_workspace_bytes(nt) bytes of device memory. */
int64_t defmm_direct_workspace_bytes(int64_t nt);
int defmm_direct_c128(int64_t nt, const double* tx, const double* ty, const double* tz,
                      int64_t ns, const double* sx, const double* sy, const double* sz,
                      const void* q, double kappa, double tol, void* workspace, void* out,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DEFMM_B200_H */
