/*
 * particula_b200.h -- C ABI of the B200-native LJ short-range MD hot path.
 *
 * Drop-in boundary for the reference package `particula` (arXiv 2109.09056
 * proxy, /root/reference/pkg/src/particula).  The reference has no FFI of its
 * own: its "interface" is the set of Python module functions listed below.
 * Each entry point here replaces the numpy body of one of them; the Python
 * package `paper_2109_09056_b200` keeps the reference's names, argument
 * meanings and exceptions and calls these functions through ctypes.
 *
 * Conventions
 *   - every pointer argument named d_* is DEVICE memory owned by the caller
 *     (torch tensors); the library never allocates or frees caller memory;
 *   - `stream` is a cudaStream_t passed as void*; all calls are asynchronous
 *     on that stream unless stated otherwise;
 *   - return value: PC_OK or a negative status; pc_last_error() holds the
 *     message (thread-local).  The Python shim maps PC_ERR_VALUE -> ValueError,
 *     PC_ERR_RUNTIME -> RuntimeError, PC_ERR_OVERLAP -> FloatingPointError
 *     (ref neighbors.py:107-118, decomp.py:138-140, md.py:118-119);
 *   - positions are FP64 (x, y, z, tag) quadruples ("pos4", 32 B per particle,
 *     one DRAM sector per gather); `tag` is an int64 stored bit-for-bit in the
 *     4th slot (global id in MD, caller index in the list API).
 */
#ifndef PARTICULA_B200_H
#define PARTICULA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PC_OK 0
#define PC_ERR_VALUE (-1)     /* ValueError            */
#define PC_ERR_RUNTIME (-2)   /* RuntimeError          */
#define PC_ERR_OVERLAP (-3)   /* FloatingPointError    */
#define PC_ERR_CUDA (-4)      /* CUDA launch / runtime */
#define PC_ERR_CAPACITY (-5)  /* output capacity too small; caller grows + retries */

/* Periodic box, ref geometry.py:10-58.  mi_thresh[a] = smallest d > 0 with
 * fl(d / length[a]) > 0.5 (the division-free, bit-exact form of
 * d - L*round(d/L) for |d| < L); +inf on non-periodic axes. */
typedef struct pc_box {
  double low[3];
  double high[3];
  double length[3];
  double mi_thresh[3];
  int32_t periodic[3];
  int32_t ndim;
} pc_box;

/* Linked-cell grid: cell = clamp(floor((x - low) / width), 0, nc - 1) per
 * axis, row-major flat id.  Ref binning.py:58-73 (width = cell_size) and
 * neighbors.py:56-60 (width = L / nc). */
typedef struct pc_grid {
  double low[3];
  double high[3];
  double width[3];
  int32_t nc[3];
  int32_t ncells;
  int32_t ndim;       /* coordinates per position actually used (1..3) */
  int32_t pad;
} pc_grid;

/* LJ parameters, ref md.py:89-126. */
typedef struct pc_lj {
  double epsilon;
  double sigma;
  double cutoff2;      /* cutoff*cutoff evaluated in FP64 on the host */
  double overlap2;     /* (1e-10*sigma)^2 : FloatingPointError below */
} pc_lj;

/* ---- library ---------------------------------------------------------- */
const char* pc_last_error(void);
int pc_version(void);
/* Kernels launched through this library since load (bench evidence). */
int64_t pc_launch_count(void);
int pc_device_sync(void* stream);

/* ---- particle storage (ref aosoa.py) ----------------------------------- */
/* AoSoA element move: element (i, w) of `src` goes to element (map[i], w) of
 * `dst`.  Word w of particle i lives at byte
 *   struct_bytes*(i/V) + word_base[w] + (i%V)*8,
 * word_base[w] = field byte offset + 8*V*component (ref aosoa.py:63-67).
 * Replaces the per-field copy_out/copy_in of ref binning.py:90-101. */
int pc_aosoa_permute(const void* d_src, void* d_dst, const int64_t* d_map,
                     int64_t n, int32_t V, int64_t struct_bytes,
                     const int64_t* d_word_base, int32_t nwords, void* stream);

/* dst[k] = src[order[k]] for rows of row_bytes (4 or a multiple of 8). */
int pc_gather_rows(const void* d_src, void* d_dst, const int32_t* d_order,
                   int64_t n, int32_t row_bytes, void* stream);
/* dst[order[k]] = src[k] (row_bytes 4 or a multiple of 8). */
int pc_scatter_rows(const void* d_src, void* d_dst, const int32_t* d_order,
                    int64_t n, int32_t row_bytes, void* stream);
/* One AoSoA field <-> dense (n, ncomp) 8-byte words (copy_out / copy_in of
 * ref aosoa.py:124-142). */
int pc_aosoa_field(void* d_buf, int64_t n, int32_t V, int64_t struct_bytes,
                   int64_t field_off, int32_t ncomp, void* d_dense, int32_t to_dense,
                   void* stream);

/* ---- binning (ref binning.py:49-101) ------------------------------------ */
/* Per-particle flat cell id and warp-aggregated atomic cell counts
 * (ref binning.py:58-73,83 and neighbors.py:56-65).  d_cell_count must be
 * zeroed by the caller.  check_inside != 0 raises the ValueError of
 * binning.py:68-69 through d_flag (bit 0). */
int pc_bin_count(const double* d_x, int64_t n, int32_t x_stride,
                 const pc_grid* grid, int32_t check_inside, int32_t* d_cell_of,
                 int64_t* d_axis_idx /* (n, ndim) per-axis cells or NULL */,
                 int32_t* d_cell_count, int32_t* d_flag, void* stream);
/* pc_bin_count of planar x | y | z positions (3-D, no axis indices, no
 * inside check): the MD engine bins straight from its staging copy. */
int pc_bin_count_planar(const double* d_planar, int64_t planar_stride, int64_t n,
                        const pc_grid* grid, int32_t* d_cell_of, int32_t* d_cell_count,
                        int32_t* d_flag, void* stream);

/* Digit "cells" of int64 keys for the LSD passes of bin_by_key
 * (ref binning.py:49-55): cell = ((key[perm[i]] - kmin) >> shift) & mask. */
int pc_key_digits(const int64_t* d_keys, const int32_t* d_perm, int64_t n, int64_t kmin,
                  int32_t shift, int64_t mask, int32_t* d_cell_of, int32_t* d_cell_count,
                  void* stream);

/* Permutation.is_bijection (ref binning.py:26-33): d_flag bit0 = out of range,
 * bit1 = duplicate.  d_seen (n int32) zeroed by the caller. */
int pc_check_bijection(const int64_t* d_map, int64_t n, int32_t* d_seen, int32_t* d_flag,
                       void* stream);

/* Exclusive prefix sum of n int32 counts into n+1 entries (last = total);
 * the _i64 variant widens to int64 (CSR offsets, ref neighbors.py:125-128).
 * d_tmp must hold pc_scan_tmp_bytes(n) bytes. */
int pc_scan_i32(const int32_t* d_in, int32_t* d_out, int64_t n,
                void* d_tmp, int64_t tmp_bytes, void* stream);
int pc_scan_i32_i64(const int32_t* d_in, int64_t* d_out, int64_t n,
                    void* d_tmp, int64_t tmp_bytes, void* stream);
int64_t pc_scan_tmp_bytes(int64_t n);

/* Stable partition of n keys in [0, nbins), nbins <= 256 (grouping by owner
 * rank, ref decomp.py:97-99; key digits of bin_by_key, ref binning.py:49-55).
 * pc_partition_hist writes hist[b * C + c] = count of key b in chunk c of
 * 1024 elements (C = pc_partition_chunks(n)); the caller scans it
 * (pc_scan_i32: off, nbins * C + 1 entries; bin b starts at off[b * C]);
 * pc_partition_place writes order[dst] = src, equal keys in ascending src.
 * O(n) at any bin occupancy (pc_bin_place is for small linked cells). */
int64_t pc_partition_chunks(int64_t n);
int pc_partition_hist(const int32_t* d_keys, int64_t n, int32_t nbins, int32_t* d_hist,
                      void* stream);
int pc_partition_place(const int32_t* d_keys, int64_t n, int32_t nbins, const int32_t* d_off,
                       int32_t* d_order, void* stream);

/* Stable counting-sort placement: order[dst] = src with equal cells kept in
 * ascending src order (ref binning.py:49-55 argsort(kind="stable")).
 * d_cell_fill (ncells) must be zeroed by the caller. */
int pc_bin_place(const int32_t* d_cell_of, int64_t n, const int32_t* d_cell_start,
                 int32_t ncells, int32_t* d_cell_fill, int32_t* d_order_tmp,
                 int32_t* d_order, void* stream);
/* pc_bin_place without the within-cell stabilisation (order inside a cell
 * arbitrary): for callers that re-sort every cell anyway (pc_cell_zsort,
 * which ranks by (z, particle index)). */
int pc_bin_place_unstable(const int32_t* d_cell_of, int64_t n, const int32_t* d_cell_start,
                          int32_t* d_cell_fill, int32_t* d_order, void* stream);

/* map[order[k]] = k  (Permutation.map of ref binning.py:13-33). */
int pc_invert_order(const int32_t* d_order, int64_t n, int64_t* d_map,
                    void* stream);

/* ---- neighbor lists (ref neighbors.py:49-134) ---------------------------- */
/* Build from cell-sorted pos4 (d_pos_sorted[k] = particle order[k]) and the
 * cell offsets of `grid` (ncells+1).  Predicate: min-image r^2 < cutoff2 with
 * r^2 = (dx*dx + dz*dz) + dy*dy in FP64, no FMA (bit-exact to the reference).
 * half != 0 keeps only tag_j > tag_i (neighbors.py:121-122).
 *   mode PC_NBR_COUNT : write d_count[k] only
 *   mode PC_NBR_CSR   : write row k at d_offsets[k] into d_index
 *   mode PC_NBR_ELL   : transposed ELL, entry (k, s) at d_index[s*ell_stride+k],
 *                       s < ell_width; overflow -> d_flag bit 1 (counts still exact)
 * out_tags != 0 writes tag_j (caller index space), else the sorted index j.
 * Rows are emitted in ascending sorted index order. */
#define PC_NBR_COUNT 0
#define PC_NBR_CSR 1
#define PC_NBR_ELL 2
#define PC_NBR_SELL 3   /* SELL-32x4: ell_width = entries/row (mult. of 4),
                           ell_stride = dummy row index used for padding */
int pc_nbr_build(const double* d_pos_sorted, int32_t n, const int32_t* d_cell_start,
                 const pc_grid* grid, const pc_box* box, double cutoff2,
                 int32_t half, int32_t mode, int32_t out_tags,
                 int32_t* d_count, const int64_t* d_offsets, int32_t* d_index,
                 int64_t ell_stride, int32_t ell_width, int32_t* d_flag,
                 void* stream,
                 const double* d_posb /* binning positions (NULL: d_pos_sorted) */,
                 const pc_box* box_exact /* min-image box of the predicate (NULL: box) */);

/* MD hot-path build into the SELL-32x4 layout the force kernel reads: entry
 * k of row a at int word ((a>>5)*(width/4) + k/4)*128 + (a&31)*4 + k%4,
 * partial quads padded with `dummy` (a row whose position is NaN).  Uses the
 * shared-memory staged kernel (FP32 prefilter with a bounded band, exact FP64
 * predicate inside it: bit-identical sets) when every periodic axis has >= 3
 * cells, else the per-particle kernel.  d_flag bit 1: a row exceeded width
 * (counts exact, caller grows and rebuilds); bit 4: staging capacity
 * exceeded (caller rebuilds with pc_nbr_build).  *h_used_staged reports the
 * kernel chosen.  Decomposed domains bin owned+ghost particles by d_posb
 * (ghosts shifted by their periodic image into the local frame) on a local
 * grid/box while the FP64 predicate uses the raw positions and the global
 * box_exact, exactly the reference's ghost convention (md.py:181-188). */
int pc_nbr_build_sell(const double* d_pos_sorted, int32_t n, const int32_t* d_cell_start,
                      const pc_grid* grid, const pc_box* box, double cutoff2,
                      int32_t width, int32_t dummy, int32_t* d_count, int32_t* d_index,
                      int32_t* d_flag, int32_t* h_used_staged, void* stream,
                      const double* d_posb, const pc_box* box_exact,
                      int32_t half /* keep one entry per unordered pair (Newton 3) */);

/* ---- device neighbor traversal consumers (pc_traverse.cu) ----------------- */
/* Built on include/particula_b200_traverse.cuh (for_each_neighbor /
 * for_each_neighbor2 as device functors, ref neighbors.py:137-154) over a CSR
 * list (int64 offsets, int32 index), rows [begin, end), team != 0: one warp
 * per row.  d_x (n, 3) f64; the minimum image on box's periodic axes.
 * coordination: d_out[i] += #{stored j : |x_j - x_i|^2 < r_inner^2};
 * angle_sum (full list): d_out[i] += sum over stored pairs j before k of
 * cos(angle j-i-k).  d_out (n) zeroed by the caller. */
int pc_traverse_coordination(const double* d_x, const pc_box* box, const int64_t* d_offsets,
                             const int32_t* d_index, int32_t n, int32_t begin, int32_t end,
                             double r_inner, int32_t team, double* d_out, void* stream);
int pc_traverse_angle_sum(const double* d_x, const pc_box* box, const int64_t* d_offsets,
                          const int32_t* d_index, int32_t n, int32_t begin, int32_t end,
                          int32_t team, double* d_out, void* stream);

/* ---- Ewald real-space pass (pc_longrange.cu) ------------------------------ */
/* Replaces ref longrange.py:47-72 (_real_space) over a pair list (the half
 * Verlet list of longrange.spme, longrange.py:142-146, expanded to (i, j)):
 * dx = x[j] - x[i] with the exact minimum image on periodic axes, r^2 in the
 * einsum order, pairs with r^2 < r_cut^2 contribute E = q_i q_j erfc(alpha r)/r
 * and f[j] += s dx, f[i] -= s dx, s = q_i q_j (erfc(alpha r)/r^2 +
 * 2 alpha/sqrt(pi) exp(-(alpha r)^2)/r)/r (FP64 atomics; d_f (n, 3) zeroed by
 * the caller).  d_epart gets pc_ewald_real_blocks(npairs) energy partials;
 * d_flag bit 4: a selected pair with r < 1e-10 (ValueError in the ref). */
int64_t pc_ewald_real_blocks(int64_t npairs);
/* Row index of every CSR entry (ref VerletList.pairs, neighbors.py:39-46):
 * d_pi[k] = i for k in [offsets[i], offsets[i+1]). */
int pc_csr_pairs(const int64_t* d_offsets, int32_t n, int32_t* d_pi, void* stream);
int pc_ewald_real_pairs(const double* d_x, const double* d_q, const int32_t* d_pi,
                        const int32_t* d_pj, int64_t npairs, const pc_box* box, double alpha,
                        double r_cut, double* d_f, double* d_epart, int32_t* d_flag,
                        void* stream);

/* ---- deterministic mode ------------------------------------ */
/* pc_sell_sort_by_tag: order every row of a SELL list (pc_nbr_build_sell) by
 * the neighbours' global ids (int64 tags in d_pos4 .w), so each atom's pair
 * terms accumulate in one order under any decomposition (rows > 256 entries
 * set flag bit 2).  pc_lj_force_sell_atoms: pc_lj_force_sell writing one
 * (KE, PE, px, py, pz) row per atom to d_atom (n_rows x 5) instead of per-warp
 * partials; the caller scatters owned rows by global id and reduces them in
 * id order (pc_scatter_rows + pc_reduce_partials): energy series bitwise
 * equal for any rank grid (ref test_acceptance.py:79-92, criterion 3). */
int pc_sell_sort_by_tag(const double* d_pos4, int32_t n, const int32_t* d_count,
                        int32_t* d_index, int32_t width, int32_t* d_flag, void* stream);
int pc_lj_force_sell_atoms(const double* d_pos, const double* d_planar, int64_t planar_stride,
                           int32_t n_rows, const int32_t* d_count, const int32_t* d_index,
                           int32_t width, const pc_box* box, const pc_lj* lj, double mi_guard,
                           double* d_f3, int64_t f_stride, double* d_v, int64_t v_stride,
                           double dtm, double mass, double* d_atom, int32_t* d_flag,
                           void* stream);

/* ---- tile-staged MD hot path (pc_tile.cu) -------------------------------- */
/* MD-engine replacement of ref neighbors.py:49-97 (Verlet build) +
 * md.py:99-126 (forces) + md.py:251-257 (final half kick) for a 3-D box with
 * >= 3 cells of `grid` per axis.  A tile = 2x2 columns x 4 z-cells of `grid`;
 * its neighbourhood (4x4 columns x 6 cells = cell-sorted index runs) is
 * staged in shared memory by TMA bulk copies; lists hold 16-bit slots into
 * that staging area, grouped per row-warp of 32 home rows in bank-conflict-
 * free "rounds" (layout: pc_tile.cu header).  Positions are the planar FP64
 * arrays x|y|z at d_planar with stride planar_stride (a multiple of 16
 * elements, >= n + 1).
 *
 * pc_tile_count: number of tiles.  pc_tile_rows: d_rw[tile] = row-warps of
 * the tile (max(1, ceil(home rows / 32)): a tile without rows keeps one empty
 * row-warp); the caller scans them into d_rw0
 * (ntiles + 1 entries; total row-warps RW = d_rw0[ntiles]) and provides
 * d_plan (ntiles * pc_tile_plan_ints() int32), d_rowidx (RW * 32 int32),
 * d_rounds (RW int32), d_partial (RW * 5 doubles) and d_list (RW * q8 * 512
 * bytes). */
int32_t pc_tile_count(const pc_grid* grid);
/* Per-cell z-sort of a cell-sorted order (ref-transparent: the reference
 * sums forces and energies in global-id order, md.py:7-11): cell c holds
 * d_order[cs[c] .. cs[c+1]); d_out lists the same particles ranked by
 * (z of d_pos4 row, position in the cell).  The tile path relies on it:
 * staged columns and home rows become z-sorted runs. */
int pc_cell_zsort(const double* d_z, int64_t z_stride, const int32_t* d_cell_start,
                  int32_t ncells, const int32_t* d_order, int32_t* d_out, void* stream);
int32_t pc_tile_plan_ints(void);
int32_t pc_tile_stage_cap(void);
int pc_tile_rows(const int32_t* d_cell_start, const pc_grid* grid, int32_t* d_rw,
                 void* stream);
/* As pc_tile_rows for a decomposed domain (ref decomp.py:143-260: owned rows
 * + ghost rows in one local array): d_skip[i] != 0 marks ghost i; only the
 * owned home particles are rows (pc_tile_build_domain numbers them the same
 * way), so no row-warp runs ghost lanes. */
int pc_tile_rows_domain(const int32_t* d_cell_start, const pc_grid* grid, const int32_t* d_skip,
                        int32_t* d_rw, void* stream);
/* Verlet build at cutoff2 (the reference's FP64 predicate behind an FP32
 * band prefilter) + round scheduling.  d_flag (3 int32, zeroed by the
 * caller): [0] bit 1 = a row-warp needs more than 8*q8 rounds ([2] = the
 * largest; >= 2^20: a row exceeds 112 entries), bit 4 = a neighbourhood
 * exceeds pc_tile_stage_cap() slots ([1] = the largest).  The caller grows
 * q8 and rebuilds, or falls back to pc_nbr_build_sell. */
int pc_tile_build(const double* d_planar, int64_t planar_stride, const int32_t* d_cell_start,
                  const pc_grid* grid, const pc_box* box, double cutoff2, int32_t q8,
                  const int32_t* d_rw0, int32_t* d_plan, int32_t* d_rowidx, int32_t* d_rounds,
                  void* d_list, int32_t* d_flag, void* stream);
/* pc_tile_build for a decomposed domain (owned + ghost rows, ref
 * md.py:176-188): cells, tiles and the FP32 prefilter use d_bplanar (ghosts
 * shifted by their periodic image into the local frame; grid/box = the local
 * grid and box), the exact FP64 predicate uses the raw positions d_planar and
 * the global box_exact (the reference's ghost convention), and particles i
 * with d_skip[i] != 0 (ghosts) are never rows (no list, no force entry; the
 * rows of a tile are its owned home particles, d_rw0 from
 * pc_tile_rows_domain with the same d_skip).  NULL d_bplanar / box_exact /
 * d_skip: pc_tile_build.  d_tile_ghost (nullable, one int per tile): 1 when
 * the tile's staged neighbourhood holds a ghost row (d_skip), else 0 -- the
 * interior / boundary split of pc_tile_force. */
int pc_tile_build_domain(const double* d_planar, int64_t planar_stride,
                         const int32_t* d_cell_start, const pc_grid* grid, const pc_box* box,
                         double cutoff2, int32_t q8, const int32_t* d_rw0, int32_t* d_plan,
                         int32_t* d_rowidx, int32_t* d_rounds, void* d_list, int32_t* d_flag,
                         void* stream, const double* d_bplanar, const pc_box* box_exact,
                         const int32_t* d_skip, int32_t* d_tile_ghost);
/* pc_tile_build_domain with the round order of pc_tile_order applied inside
 * the build (order_kind 1: residue round-robin, each row-warp's list read
 * back from L2 right after it is written -- the same lists as pc_tile_build +
 * pc_tile_order(kind 1), without the separate pass over HBM; 0: the build's
 * order).  d_skip / d_bplanar / box_exact / d_tile_ghost nullable as in
 * pc_tile_build_domain. */
int pc_tile_build_ordered(const double* d_planar, int64_t planar_stride,
                          const int32_t* d_cell_start, const pc_grid* grid, const pc_box* box,
                          double cutoff2, int32_t q8, const int32_t* d_rw0, int32_t* d_plan,
                          int32_t* d_rowidx, int32_t* d_rounds, void* d_list, int32_t* d_flag,
                          void* stream, const double* d_bplanar, const pc_box* box_exact,
                          const int32_t* d_skip, int32_t* d_tile_ghost, int32_t order_kind);
/* Reorder the rounds of every row-warp (after pc_tile_build, same list):
 * residue round-robin per row so that the 16 lanes of a half-warp read 16
 * distinct shared-memory bank pairs in most rounds.  rw_bound >= the total
 * row-warps, which the kernel reads from d_rw_total (= d_rw0[ntiles]).
 * kind: 0 = keep the build's ascending order, 1 = residue round-robin,
 * 2 = class-major rotated to the lane's residue. */
int pc_tile_order(int32_t rw_bound, const int32_t* d_rw_total, const int32_t* d_rounds,
                  void* d_list, int32_t q8, int32_t kind, void* stream);
/* LJ force over the tile lists: exact FP64 r^2 < rc^2 re-test in the
 * reference's rounding order (minimum image on rows within mi_guard of a
 * periodic face), FP32 LJ magnitude, FP64 accumulation; writes f (planar,
 * f_stride), applies the final half kick v += dtm*f when d_v != NULL and
 * writes (KE, PE, px, py, pz) partials, pc_tile_force_partials(ntiles) of
 * them (one per warp of the persistent grid).  Overlap
 * (r^2 < overlap2) sets d_flag bit 2.  With d_planar_next != NULL the next
 * step's integrate block (v' = v + dtm_next f, x' = wrap(x + dt v'), ref
 * md.py:219-231) is fused into the epilogue and written to d_planar_next /
 * d_v_next (same strides); d_planar and d_v keep this step's state.
 * d_virial (nullable): the pair virial W = sum over pairs of r.F, one
 * partial per warp in column 0 of a zero-initialised (partials, 5) array
 * (reduce with pc_reduce_partials).  The reference has no virial; this is
 * the north-star "FP64 energy/virial reduction" (BASELINE.json).
 * d_tiles / d_trange (nullable): run only the tiles d_tiles[trange[0] ..
 * trange[1]) (device-side bounds; ntiles stays the launch bound) -- the
 * interior / boundary passes that overlap a decomposed domain's ghost
 * refresh (ref md.py:192-200); each pass writes its own partial rows. */
int pc_tile_force(const double* d_planar, int64_t planar_stride, int32_t ntiles,
                  const int32_t* d_plan, const int32_t* d_rowidx, const int32_t* d_rounds,
                  const void* d_list, int32_t q8, const pc_box* box, const pc_lj* lj,
                  double mi_guard, double* d_f3, int64_t f_stride, double* d_v, int64_t v_stride,
                  double dtm, double mass, double* d_partial, int32_t* d_flag,
                  double* d_planar_next, double* d_v_next, double dtm_next, double dt,
                  double* d_virial, const int32_t* d_tiles, const int32_t* d_trange,
                  void* stream);
int32_t pc_tile_force_partials(int32_t ntiles);
/* pos4 x, y, z <- planar rows [0, n) (tags untouched). */
int pc_pos_from_planar(const double* d_planar, int64_t planar_stride, int32_t n, double* d_pos4,
                       void* stream);
/* Tile lists -> per-row particle indices: d_count[row], d_table[row*width+k]
 * (rows = cell-sorted particle indices; inspection / parity tests). */
int pc_tile_decode(int32_t ntiles, const int32_t* d_plan, const int32_t* d_rowidx,
                   const int32_t* d_rounds, const void* d_list, int32_t q8, int32_t width,
                   int32_t* d_count, int32_t* d_table, void* stream);

/* CSR -> dense (n, width) int64 table, -1 padded (ref neighbors.py:130-134). */
int pc_csr_to_dense(const int64_t* d_offsets, int32_t n, const int32_t* d_index,
                    int32_t width, int64_t* d_table, void* stream);

/* Sort every CSR row ascending (int32 values), warp per row. */
int pc_sort_rows(const int64_t* d_offsets, int32_t n, int32_t* d_index,
                 void* stream);

/* ---- LJ force (ref md.py:89-126) ----------------------------------------- */
/* Force on rows [0, n_rows) from a neighbor list over pos4 (rows index the
 * same pos4 array; neighbor values index it too).  FP64 min-image and exact
 * cutoff test, FP32 LJ magnitude, FP64 force accumulation (exactly
 * antisymmetric pair forces), FP64 energy partials.
 * Layout: ell_stride > 0 -> transposed ELL (d_index[s*ell_stride + i]);
 *         else CSR via d_offsets.
 * Outputs (any may be NULL):
 *   d_f3      : double[3][f_stride] planar force
 *   d_f64     : double (n_rows, 3) row-major force (API path)
 *   d_pe      : double per-row energy, each pair booked on the smaller tag
 *   d_v       : double[3][v_stride] planar velocity, fused final half kick
 *               v += dtm*f (ref md.py:251-257) when non-NULL
 *   d_partial : double[5*gridDim] per-block (KE after kick, PE, px, py, pz)
 * Overlap (r^2 < overlap2) sets d_flag bit 2 (FloatingPointError). */
int pc_lj_force(const double* d_pos, int32_t n_rows, const int32_t* d_count,
                const int64_t* d_offsets, const int32_t* d_index,
                int64_t ell_stride, const pc_box* box, const pc_lj* lj,
                double* d_f3, int64_t f_stride, double* d_f64, double* d_pe,
                double* d_v, int64_t v_stride, double dtm, double mass,
                double* d_partial, int32_t* d_flag, void* stream);
int32_t pc_lj_force_blocks(int32_t n_rows);

/* MD hot-path force over the SELL-32x4 list of pc_nbr_build_sell: per row one
 * 128-bit index load per 4 neighbors (software-pipelined) and 4 independent
 * 256-bit pos4 gathers in flight.  Minimum image is applied only on axes where
 * the row particle lies within `mi_guard` of a periodic face: for a Verlet
 * list whose pairs stay closer than mi_guard this is bit-identical to applying
 * it everywhere (pass +inf to always apply it).  FP64 pair arithmetic and
 * accumulation, fused final half kick (d_v may be NULL), per-WARP partials
 * (pc_lj_force_sell_partials(n) rows of KE after kick, PE with each pair
 * booked half on either side, px, py, pz). */
int32_t pc_lj_force_sell_partials(int32_t n_rows);
int pc_lj_force_sell(const double* d_pos, const double* d_planar /* x|y|z planar copy or
                     NULL: gathers then read 24 B as three 64-bit loads */,
                     int64_t planar_stride, int32_t n_rows, const int32_t* d_count,
                     const int32_t* d_index, int32_t width, const pc_box* box,
                     const pc_lj* lj, double mi_guard, double* d_f3, int64_t f_stride,
                     double* d_v, int64_t v_stride, double dtm, double mass,
                     double* d_partial, int32_t* d_flag, void* stream);

/* Half list over the SELL layout of pc_nbr_build_sell(half=1): each pair once,
 * f_i += F in registers, f_j -= F by FP64 atomics (not bitwise deterministic);
 * d_f3 zeroed by the caller, final kick by pc_kick.  Partials: per warp, PE
 * only (full pair energy once). */
int pc_lj_force_sell_half(const double* d_pos, int32_t n_rows, const int32_t* d_count,
                          const int32_t* d_index, int32_t width, const pc_box* box,
                          const pc_lj* lj, double mi_guard, double* d_f3, int64_t f_stride,
                          double* d_partial, int32_t* d_flag, void* stream);

/* Half-list Newton-3 variant: rows hold j > i only; f_j -= F via FP64
 * atomics (not bitwise deterministic).  d_f3 must be zeroed by the caller. */
int pc_lj_force_half(const double* d_pos, int32_t n_rows, const int32_t* d_count,
                     const int32_t* d_index, int64_t ell_stride,
                     const pc_box* box, const pc_lj* lj, double* d_f3,
                     int64_t f_stride, double* d_pe_total, int32_t* d_flag,
                     void* stream);

/* ---- integrate (ref md.py:219-257, geometry.py:40-49) --------------------- */
/* v += dtm*f; x += dt*v; x = wrap(x) on rows [0,n) -- numpy rounding order. */
int pc_kick_drift_wrap(double* d_pos, double* d_v, int64_t v_stride,
                       const double* d_f3, int64_t f_stride, int32_t n,
                       double dtm, double dt, const pc_box* box,
                       double* d_planar /* optional x|y|z planar copy, or NULL */,
                       int64_t planar_stride, void* stream);
/* The decomposed engine's rebuild permutation: rows k of d_pos4_out,
 * d_bin4_out (local-frame positions), d_v_out (planar, v_stride) and
 * d_ghost_out <- rows d_order[k]; and the planar x | y | z copies of the new
 * pos4 / bin4 rows into d_planar / d_bplanar (planar_stride). */
int pc_domain_permute(const int32_t* d_order, int32_t n, const double* d_pos4,
                      double* d_pos4_out, const double* d_bin4, double* d_bin4_out,
                      const double* d_v, double* d_v_out, int64_t v_stride,
                      const int32_t* d_ghost, int32_t* d_ghost_out, double* d_planar,
                      double* d_bplanar, int64_t planar_stride, void* stream);
/* Rebuild permutation in one pass: row k of d_pos4_out (x, y, z from the
 * planar d_planar, the id from d_pos4 .w), of d_v_out (planar velocities,
 * stride v_stride) and of the planar d_planar_out <- row d_order[k]. */
int pc_md_permute(const int32_t* d_order, int32_t n, const double* d_planar,
                  int64_t planar_stride, const double* d_pos4, double* d_pos4_out,
                  const double* d_v, double* d_v_out, int64_t v_stride, double* d_planar_out,
                  void* stream);
/* planar[a*stride + i] = pos4[i].a for a = x, y, z. */
int pc_pos_planar(const double* d_pos, int32_t n, double* d_planar, int64_t planar_stride,
                  void* stream);
/* v += dtm*f, plus the per-block diagnostic partials (KE, 0, px, py, pz). */
int pc_kick(double* d_v, int64_t v_stride, const double* d_f3, int64_t f_stride,
            int32_t n, double dtm, double mass, double* d_partial, void* stream);

/* Box.wrap / Box.min_image in place on (rows, d) FP64 arrays
 * (ref geometry.py:40-49, :51-58). */
int pc_box_wrap(double* d_x, int64_t rows, int32_t d, const pc_box* box, void* stream);
int pc_box_min_image(double* d_x, int64_t rows, int32_t d, const pc_box* box, void* stream);

/* lj_pair (ref md.py:89-96) in FP64: e[n], f[n][3] for dx[n][3], r2[n]. */
int pc_lj_pair(const double* d_dx, const double* d_r2, int64_t n, double eps, double sigma,
               double* d_e, double* d_f, void* stream);

/* ---- domain decomposition (ref decomp.py) -------------------------------- */
/* Owning rank of each (n, d) position: ravel(min(floor((x-low)/block), dims-1))
 * with `fabric` describing the rank grid (width = block lengths, nc = dims);
 * outside the global box -> d_flag bit 0 (ref decomp.py:58-66). */
int pc_owner_of(const double* d_x, int64_t n, int32_t d, const pc_grid* fabric,
                int32_t* d_owner, int32_t* d_flag, void* stream);
/* pc_owner_of over a decomposed domain's owned + ghost rows (the migrate's
 * first step, ref decomp.py:86-88 drops ghosts): rows with d_skip[i] != 0
 * get owner skip_owner (an out-of-range key the partition drops) and are not
 * checked -- their positions are not maintained between refreshes. */
int pc_owner_of_domain(const double* d_x, int64_t n, int32_t d, const pc_grid* fabric,
                       const int32_t* d_skip, int32_t skip_owner, int32_t* d_owner,
                       int32_t* d_flag, void* stream);
/* Wrapped position outside the box on a non-periodic axis -> d_flag bit 3
 * (ref decomp.py:92-96). */
int pc_check_nonperiodic(const double* d_x, int64_t n, int32_t d, const pc_box* box,
                         int32_t* d_flag, void* stream);
/* Reverse halo of the half-list (Newton-3) decomposed engine (ref
 * decomp.py:263-300, halo_scatter): pc_halo_force_pack copies the planar
 * forces of rows d_rows[k] (ghosts, source-rank order) into d_buf (m x 3)
 * and clears them; pc_halo_force_add adds d_buf (m x 3) onto rows d_rows[k]
 * (owners, in export order) with FP64 atomics -- a particle exported as
 * several images appears several times. */
int pc_halo_force_pack(double* d_f3, int64_t f_stride, const int32_t* d_rows, int64_t m,
                       double* d_buf, void* stream);
int pc_halo_force_add(double* d_f3, int64_t f_stride, const int32_t* d_rows, int64_t m,
                      const double* d_buf, void* stream);
/* Fused halo selection for the decomposed MD engine (same export set and
 * (slot, particle index) order as pc_halo_plan + scan + pc_compact, ref
 * decomp.py:143-228), reading pos4 rows (x, y, z, id bits) directly:
 * pc_halo_select_count writes d_hist[slot * C + c] = exported particles of
 * slot `slot` in chunk c (C = pc_halo_select_chunks(n)); after an exclusive
 * scan of d_hist (pc_scan_i32 -> d_off, slot s starts at d_off[s * C]),
 * pc_halo_select_place writes d_out_idx[k] (particle index) and the ghost
 * row d_out_rows[k] = (x, y, z, id bits, shift of the winning image).
 * h_in_lo / h_in_hi (nullable, 3 doubles each, d = 3): an interior box of
 * the source block -- the block shrunk by the halo width and a relative
 * margin -- whose particles are farther than the width from every other
 * block and skip the image tests (same export set). */
int64_t pc_halo_select_chunks(int64_t n);
int pc_halo_select_count(const double* d_pos4, int64_t n, int32_t d, int32_t n_off,
                         const int32_t* h_slot, const double* h_shift, const double* h_lo,
                         const double* h_hi, int32_t n_slots, double w2, int32_t* d_hist,
                         void* stream, const double* h_in_lo, const double* h_in_hi);
int pc_halo_select_place(const double* d_pos4, int64_t n, int32_t d, int32_t n_off,
                         const int32_t* h_slot, const double* h_shift, const double* h_lo,
                         const double* h_hi, int32_t n_slots, double w2, const int32_t* d_off,
                         int32_t* d_out_idx, double* d_out_rows, void* stream,
                         const double* h_in_lo, const double* h_in_hi);
/* Halo export planning for one source rank (ref decomp.py:143-228): n_off
 * candidate images in product order (host arrays: destination slot, shift,
 * destination box lo/hi, each d wide); per particle and slot the best image
 * (strict <, first wins) is exported iff its squared distance to the box is
 * < w2.  Writes d_flags[slot*n + i] (int32 0/1) and d_best_off (int8). */
int pc_halo_plan(const double* d_x, int64_t n, int32_t d, int32_t n_off, const int32_t* h_slot,
                 const double* h_shift, const double* h_lo, const double* h_hi,
                 int32_t n_slots, double w2, int32_t* d_flags, int8_t* d_best_off,
                 void* stream);
/* Stable compaction: out_idx[pos[i]] = i (and its offset code) where flag[i]. */
int pc_compact(const int32_t* d_flag, const int32_t* d_pos, int64_t n, int32_t* d_out_idx,
               const int8_t* d_best_off, int8_t* d_out_off, void* stream);
/* dst[k] = src[idx[k]] (+ shift[k]) over rows of w doubles (ghost staging,
 * ref decomp.py:243-246). */
int pc_gather_shift(const double* d_src, const int32_t* d_idx, int64_t m, int32_t w,
                    const double* d_shift, double* d_dst, void* stream);
/* Per-step halo refresh: buf[k] = pos4[rows[k]].xyz (pack; _planar: from
 * the planar x|y|z copy) and pos4[rows[k]].xyz = buf[k] (+ planar copy; NULL
 * d_pos: planar only) (unpack), buf (m, 3) f64. */
int pc_halo_pack(const double* d_pos, const int32_t* d_rows, int64_t m, double* d_buf,
                 void* stream);
int pc_halo_pack_planar(const double* d_planar, int64_t planar_stride, const int32_t* d_rows,
                        int64_t m, double* d_buf, void* stream);
int pc_halo_unpack(const double* d_buf, const int32_t* d_rows, int64_t m, double* d_pos,
                   double* d_planar, int64_t planar_stride, void* stream);
/* Peer-memory halo exchange between processes (CUDA IPC over NVLink): the
 * per-step refresh / reverse all-to-all of ref decomp.py:231-260 / 263-300
 * (the exchange `_step` of md.py:192-200 runs every step) without NCCL.
 * A window = [2 parities x cap rows x width f64][arrive: world i64][ack:
 * world i64]; step k uses parity k & 1.  _window_alloc: cudaMalloc (zeroed)
 * + the IPC handle (pc_p2p_handle_bytes() bytes) into h_handle; _open /
 * _close map / unmap a peer's window.  _put: rows [src0, src0 + count) of
 * d_send to each destination window's parity block at row dst0 (table of
 * pc_p2p_dest_bytes()-byte entries {window, src0, count, dst0} in device
 * memory); _signal: flags[me] = value in each window of such a table
 * (flag_off in doubles from the window base); _wait: until the own
 * window's flags[ranks[t]] >= target (spin limit -> *d_err = 1). */
int pc_p2p_window_bytes(int64_t cap_rows, int32_t width, int32_t world, int64_t* bytes);
int pc_p2p_window_alloc(int64_t cap_rows, int32_t width, int32_t world, void** d_window,
                        void* h_handle);
int pc_p2p_window_free(void* d_window);
int32_t pc_p2p_handle_bytes(void);
int32_t pc_p2p_dest_bytes(void);
int pc_p2p_open(const void* h_handle, void** d_peer);
int pc_p2p_close(void* d_peer);
int pc_p2p_put(const double* d_send, const void* d_dests, int32_t n_dst, int64_t max_rows,
               int32_t width, int64_t cap_rows, int32_t parity, void* stream);
int pc_p2p_signal(const void* d_dests, int32_t n_dst, int64_t flag_off, int32_t me,
                  int64_t value, void* stream);
/* The refresh's pack fused into the put: exported row
 * d_rows[src0 + k] of the planar x|y|z positions straight into each
 * destination window (width 3), no send buffer. */
int pc_p2p_pack_put(const double* d_planar, int64_t planar_stride, const int32_t* d_rows,
                    const void* d_dests, int32_t n_dst, int64_t max_rows, int64_t cap_rows,
                    int32_t parity, void* stream);
int pc_p2p_wait(const void* d_window, int64_t flag_off, const int32_t* d_ranks, int32_t n,
                int64_t target, int32_t* d_err, int64_t spin_limit, void* stream);
/* dst[idx[k]] += src[k] over rows of w doubles, idx distinct per call
 * (one destination's ghost block of ref decomp.py:281-289). */
int pc_scatter_add(double* d_dst, const int32_t* d_idx, int64_t m, int32_t w,
                   const double* d_src, void* stream);

/* Exact, order-independent column sums of (n x w) FP64 rows (w <= 8; rows
 * with d_skip[i] != 0 left out; |values| < 2^50, bits below 2^-90
 * truncated): pc_exact_sum ADDS each column's integer part and three 30-bit
 * fraction limbs into d_limbs (w x 4 int64, zeroed by the caller; integer
 * sums, so limbs of disjoint row sets -- threads, ranks, devices -- simply
 * add); pc_exact_finish converts the limbs into w doubles.  The
 * deterministic mode's energies (ref md.py:261-277). */
int pc_exact_sum(const double* d_rows, int64_t n, int32_t w, const int32_t* d_skip,
                 int64_t* d_limbs, void* stream);
int pc_exact_finish(const int64_t* d_limbs, int32_t w, double* d_out, void* stream);
/* Sum per-block partials (nblocks x 5) into out[5] in a fixed order. */
int pc_reduce_partials(const double* d_partial, int32_t nblocks, double* d_out,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PARTICULA_B200_H */
