// Verlet neighbor lists from cell-sorted positions (ref neighbors.py:49-134).
//
// One thread per (sorted) particle sweeps its deduplicated 27-cell stencil;
// after the counting sort every stencil cell is a contiguous index range, so
// candidate positions stream through L1/L2 as 256-bit pos4 loads.  The pair
// predicate is the reference's FP64 one, bit for bit: min-image
// (geometry.py:51-58), r^2 = (dx^2 + dz^2) + dy^2 without FMA
// (neighbors.py:92, numpy einsum order), strict r^2 < cutoff^2 (:93).
#include "pc_common.cuh"

namespace pc {

template <int MODE>
__global__ void __launch_bounds__(128)
nbr_build_kernel(const double* __restrict__ pos, int n, const int* __restrict__ cell_start,
                 pc_grid g, pc_box b, double cutoff2, int half, int out_tags,
                 int* __restrict__ count, const int64_t* __restrict__ offsets,
                 int* __restrict__ index, int64_t ell_stride, int ell_width,
                 int* __restrict__ flag, const double* __restrict__ posb, pc_box e) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 pi = ld_pos4(pos + 4 * (int64_t)i);
  const double4 bi = ld_pos4(posb + 4 * (int64_t)i);
  const int64_t ti = tag_of(pi.w);
  int sx[3], sy[3], sz[3];
  int nx = axis_stencil(cell_coord(bi.x, g.low[0], g.width[0], g.nc[0]), g.nc[0],
                        b.periodic[0], sx);
  int ny = axis_stencil(cell_coord(bi.y, g.low[1], g.width[1], g.nc[1]), g.nc[1],
                        b.periodic[1], sy);
  int nz = axis_stencil(cell_coord(bi.z, g.low[2], g.width[2], g.nc[2]), g.nc[2],
                        b.periodic[2], sz);
  int64_t row = 0;
  if (MODE == PC_NBR_CSR) row = offsets[i];
  int cnt = 0;
  for (int a = 0; a < nx; ++a) {
    for (int c = 0; c < ny; ++c) {
      const int base_cell = (sx[a] * g.nc[1] + sy[c]) * g.nc[2];
      // merge z-cells that are adjacent in memory into one index range
      int k = 0;
      while (k < nz) {
        int z0 = sz[k];
        int z1 = z0;
        while (k + 1 < nz && sz[k + 1] == z1 + 1) { ++k; ++z1; }
        ++k;
        const int jb = cell_start[base_cell + z0];
        const int je = cell_start[base_cell + z1 + 1];
        for (int j = jb; j < je; ++j) {
          if (j == i) continue;
          const double4 pj = ld_pos4(pos + 4 * (int64_t)j);
          const double dx = min_image(__dsub_rn(pj.x, pi.x), e.length[0], e.mi_thresh[0]);
          const double dy = min_image(__dsub_rn(pj.y, pi.y), e.length[1], e.mi_thresh[1]);
          const double dz = min_image(__dsub_rn(pj.z, pi.z), e.length[2], e.mi_thresh[2]);
          if (r2_exact(dx, dy, dz) < cutoff2) {
            const int64_t tj = tag_of(pj.w);
            if (half && !(tj > ti)) continue;
            if (posb != pos) {
              // decomposed domain: accept only the ghost image adjacent to i in
              // the local frame (another image of the same particle is ~L away)
              const double4 bj = ld_pos4(posb + 4 * (int64_t)j);
              const double lim = sqrt(cutoff2) * (1.0 + 1e-9);
              if ((!b.periodic[0] && fabs(bj.x - bi.x) > lim) ||
                  (!b.periodic[1] && fabs(bj.y - bi.y) > lim) ||
                  (!b.periodic[2] && fabs(bj.z - bi.z) > lim))
                continue;
            }
            if (MODE != PC_NBR_COUNT) {
              const int v = out_tags ? (int)tj : j;
              if (MODE == PC_NBR_CSR) {
                index[row + cnt] = v;
              } else if (MODE == PC_NBR_ELL) {
                if (cnt < ell_width) index[(int64_t)cnt * ell_stride + i] = v;
              } else if (cnt < ell_width) {
                index[sell_word(i, cnt, ell_width >> 2)] = v;
              }
            }
            ++cnt;
          }
        }
      }
    }
  }
  count[i] = cnt;
  if (MODE == PC_NBR_SELL) {
    // pad the last quad with the dummy row (NaN position, never interacts)
    for (int k = cnt; k < ell_width && (k & 3); ++k)
      index[sell_word(i, k, ell_width >> 2)] = (int)ell_stride;
  }
  if ((MODE == PC_NBR_ELL || MODE == PC_NBR_SELL) && cnt > ell_width)
    atomicOr(flag, kFlagOverflow);
}

// ---- staged build (MD hot path) -------------------------------------------
// One CTA per (x, y) column segment of kSegCells home cells.  The 9 stencil
// columns' cells z0-1 .. z1 are staged once into shared memory as FP32
// coordinates relative to the segment centre (periodic image applied per
// staged cell) plus the particle index, so each home particle scans its 27
// stencil cells as 9 contiguous shared-memory ranges.  FP32 r^2 decides
// every candidate outside a rigorously bounded band around cutoff^2; inside
// the band the reference's FP64 predicate is evaluated on the global FP64
// positions, so the result is bit-identical to pc_nbr_build / the reference.
// Requires >= 3 cells on every periodic axis (else the v1 kernel is used).
constexpr int kSegCells = 4;
constexpr int kStageCells = kSegCells + 2;
constexpr int kBuildThreads = 128;

struct StagedParams {
  double cutoff2;
  float lo2, hi2;      // FP32 band: r2f < lo2 -> hit, r2f >= hi2 -> miss
  int Q;               // quads per SELL slice
  int dummy;           // padding row index
  int max_stage;       // staged-candidate capacity (float4 entries)
  int nseg;            // z segments per column
  int half;            // keep only j > i (sorted row index): Newton-3 half list
};

__device__ __forceinline__ bool exact_pair(const double* pos, int a, int j, const pc_box& b,
                                           double cutoff2) {
  const double4 pa = ld_pos4(pos + 4 * (int64_t)a);
  const double4 pj = ld_pos4(pos + 4 * (int64_t)j);
  const double dx = min_image(__dsub_rn(pj.x, pa.x), b.length[0], b.mi_thresh[0]);
  const double dy = min_image(__dsub_rn(pj.y, pa.y), b.length[1], b.mi_thresh[1]);
  const double dz = min_image(__dsub_rn(pj.z, pa.z), b.length[2], b.mi_thresh[2]);
  return r2_exact(dx, dy, dz) < cutoff2;
}

template <int MODE>
__global__ void __launch_bounds__(kBuildThreads)
nbr_build_staged_kernel(const double* __restrict__ pos, int n, const int* __restrict__ cell_start,
                        pc_grid g, pc_box b, StagedParams p, int* __restrict__ count,
                        int* __restrict__ index, int* __restrict__ flag,
                        const double* __restrict__ posb, pc_box e) {
  extern __shared__ float4 stage[];
  __shared__ int cell_off[9][kStageCells + 1];   // staged offset of each cell per column
  __shared__ int cell_src[9][kStageCells];       // first global index of each staged cell
  __shared__ double cell_shift[9][kStageCells][3];
  __shared__ int total;

  const int col = blockIdx.x / p.nseg;
  const int seg = blockIdx.x - col * p.nseg;
  const int cx = col / g.nc[1], cy = col - (col / g.nc[1]) * g.nc[1];
  const int z0 = seg * kSegCells;
  const int z1 = min(z0 + kSegCells, g.nc[2]);
  const int nz = z1 - z0 + 2;                    // staged cells per column
  const double ox = g.low[0] + (cx + 0.5) * g.width[0];
  const double oy = g.low[1] + (cy + 0.5) * g.width[1];
  const double oz = g.low[2] + 0.5 * (z0 + z1) * g.width[2];

  // per (column, staged cell): source range and periodic shift
  if (threadIdx.x < 9 * kStageCells) {
    const int c = threadIdx.x / kStageCells, k = threadIdx.x - c * kStageCells;
    int xs = cx + c / 3 - 1, ys = cy + c % 3 - 1, zs = z0 - 1 + k;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    bool ok = k < nz;
    if (xs < 0) { if (b.periodic[0]) { xs += g.nc[0]; sx = -b.length[0]; } else ok = false; }
    if (xs >= g.nc[0]) { if (b.periodic[0]) { xs -= g.nc[0]; sx = b.length[0]; } else ok = false; }
    if (ys < 0) { if (b.periodic[1]) { ys += g.nc[1]; sy = -b.length[1]; } else ok = false; }
    if (ys >= g.nc[1]) { if (b.periodic[1]) { ys -= g.nc[1]; sy = b.length[1]; } else ok = false; }
    if (zs < 0) { if (b.periodic[2]) { zs += g.nc[2]; sz = -b.length[2]; } else ok = false; }
    if (zs >= g.nc[2]) { if (b.periodic[2]) { zs -= g.nc[2]; sz = b.length[2]; } else ok = false; }
    int cnt = 0, src = 0;
    if (ok) {
      const int cell = (xs * g.nc[1] + ys) * g.nc[2] + zs;
      src = cell_start[cell];
      cnt = cell_start[cell + 1] - src;
    }
    cell_src[c][k] = src;
    cell_off[c][k + 1] = cnt;   // counts for now, scanned below
    cell_shift[c][k][0] = sx;
    cell_shift[c][k][1] = sy;
    cell_shift[c][k][2] = sz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int c = 0; c < 9; ++c) {
      cell_off[c][0] = run;
      for (int k = 0; k < kStageCells; ++k) {
        run += cell_off[c][k + 1];
        cell_off[c][k + 1] = run;
      }
    }
    total = run;
  }
  __syncthreads();
  if (total > p.max_stage) {           // dense region: caller falls back to v1
    if (threadIdx.x == 0) atomicOr(flag, kFlagStage);
    return;
  }
  // stage: FP32 coordinates relative to the segment centre, image applied
  for (int c = 0; c < 9; ++c) {
    for (int k = 0; k < nz; ++k) {
      const int m = cell_off[c][k + 1] - cell_off[c][k];
      const int src = cell_src[c][k];
      const int dst = cell_off[c][k];
      const double sx = cell_shift[c][k][0], sy = cell_shift[c][k][1], sz = cell_shift[c][k][2];
      for (int t = threadIdx.x; t < m; t += blockDim.x) {
        const double4 q = ld_pos4(posb + 4 * (int64_t)(src + t));
        float4 s;
        s.x = (float)(q.x + sx - ox);
        s.y = (float)(q.y + sy - oy);
        s.z = (float)(q.z + sz - oz);
        s.w = __int_as_float(src + t);
        stage[dst + t] = s;
      }
    }
  }
  __syncthreads();

  // Sweep: warp w owns home cell k = w + 1 (staged position; window = staged
  // cells k-1..k+1 of every column, 9 contiguous smem ranges shared by all of
  // the cell's particles).  Lanes are the cell's particles (chunks of 32);
  // every candidate is one broadcast LDS.128 for the whole warp, so the loop
  // bounds are warp-uniform.  Hits collect in a 4-entry register queue that
  // is flushed as one 128-bit SELL store per quad.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Q = p.Q;
  for (int k = warp + 1; k <= z1 - z0; k += kBuildThreads / 32) {
    const int hs = cell_off[4][k];                 // staged slot of the first home particle
    const int hn = cell_off[4][k + 1] - hs;
    for (int h0 = 0; h0 < hn; h0 += 32) {
      const bool act = h0 + lane < hn;
      const float4 me = act ? stage[hs + h0 + lane] : make_float4(1e30f, 1e30f, 1e30f, 0.f);
      const int a = act ? __float_as_int(me.w) : -1;
      int4* row = reinterpret_cast<int4*>(index) + (int64_t)(a >> 5) * Q * 32 + (a & 31);
      int cnt = 0;
      int b0 = p.dummy, b1 = p.dummy, b2 = p.dummy, b3 = p.dummy;
      for (int c = 0; c < 9; ++c) {
        const int s0 = cell_off[c][k - 1], s1 = cell_off[c][k + 2];
#pragma unroll 2
        for (int s = s0; s < s1; ++s) {
          const float4 q = stage[s];
          const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
          const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
          if (r2 < p.hi2) {
            const int j = __float_as_int(q.w);
            if ((p.half ? j > a : j != a) &&
                (r2 < p.lo2 || exact_pair(pos, a, j, e, p.cutoff2))) {
              if (MODE == PC_NBR_SELL) {
                b0 = b1; b1 = b2; b2 = b3; b3 = j;
                if ((cnt & 3) == 3 && cnt < 4 * Q) row[(cnt >> 2) * 32] = make_int4(b0, b1, b2, b3);
              }
              ++cnt;
            }
          }
        }
      }
      if (act) {
        if (MODE == PC_NBR_SELL) {
          const int r = cnt & 3;          // open quad: the last r entries, dummy padded
          if (r && cnt < 4 * Q) {
            int4 v = make_int4(p.dummy, p.dummy, p.dummy, p.dummy);
            if (r == 1) v.x = b3;
            if (r == 2) { v.x = b2; v.y = b3; }
            if (r == 3) { v.x = b1; v.y = b2; v.z = b3; }
            row[(cnt >> 2) * 32] = v;
          }
          if (cnt > 4 * Q) atomicOr(flag, kFlagOverflow);
        }
        count[a] = cnt;
      }
    }
  }
}

// Warp per row: ascending order by rank counting (values in a row are
// distinct particle indices).  Rows up to kSortSmem entries are staged in
// shared memory; longer rows (only at pathological densities) fall back to a
// single-lane insertion sort in place.
constexpr int kSortWarps = 8;
constexpr int kSortSmem = 512;

__global__ void __launch_bounds__(kSortWarps * 32)
sort_rows_kernel(const int64_t* __restrict__ offsets, int n, int* __restrict__ index) {
  __shared__ int buf[kSortWarps][kSortSmem];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int row = blockIdx.x * kSortWarps + wid;
  if (row >= n) return;
  int64_t b = offsets[row];
  int m = (int)(offsets[row + 1] - b);
  if (m <= 1) return;
  if (m <= kSortSmem) {
    for (int k = lane; k < m; k += 32) buf[wid][k] = index[b + k];
    __syncwarp();
    for (int k = lane; k < m; k += 32) {
      int v = buf[wid][k];
      int rank = 0;
      for (int t = 0; t < m; ++t) rank += (buf[wid][t] < v);
      index[b + rank] = v;
    }
    return;
  }
  // long rows (pathological densities): single-lane insertion sort
  if (lane == 0) {
    for (int k = 1; k < m; ++k) {
      int v = index[b + k];
      int t = k - 1;
      while (t >= 0 && index[b + t] > v) { index[b + t + 1] = index[b + t]; --t; }
      index[b + t + 1] = v;
    }
  }
}

}  // namespace pc

using namespace pc;

extern "C" {

int pc_nbr_build(const double* d_pos_sorted, int32_t n, const int32_t* d_cell_start,
                 const pc_grid* grid, const pc_box* box, double cutoff2, int32_t half,
                 int32_t mode, int32_t out_tags, int32_t* d_count, const int64_t* d_offsets,
                 int32_t* d_index, int64_t ell_stride, int32_t ell_width, int32_t* d_flag,
                 void* stream, const double* d_posb, const pc_box* box_exact) {
  if (n <= 0) return PC_OK;
  const double* posb = d_posb ? d_posb : d_pos_sorted;
  const pc_box ebox = box_exact ? *box_exact : *box;
  if (mode == PC_NBR_CSR && d_offsets == nullptr) {
    set_error("pc_nbr_build: CSR mode needs offsets");
    return PC_ERR_VALUE;
  }
  if (mode == PC_NBR_ELL && (ell_stride < n || ell_width < 0)) {
    set_error("pc_nbr_build: bad ELL geometry");
    return PC_ERR_VALUE;
  }
  cudaStream_t s = as_stream(stream);
  unsigned blocks = (unsigned)((n + 127) / 128);
  switch (mode) {
    case PC_NBR_COUNT:
      nbr_build_kernel<PC_NBR_COUNT><<<blocks, 128, 0, s>>>(
          d_pos_sorted, n, d_cell_start, *grid, *box, cutoff2, half, out_tags, d_count,
          d_offsets, d_index, ell_stride, ell_width, d_flag, posb, ebox);
      break;
    case PC_NBR_CSR:
      nbr_build_kernel<PC_NBR_CSR><<<blocks, 128, 0, s>>>(
          d_pos_sorted, n, d_cell_start, *grid, *box, cutoff2, half, out_tags, d_count,
          d_offsets, d_index, ell_stride, ell_width, d_flag, posb, ebox);
      break;
    case PC_NBR_ELL:
      nbr_build_kernel<PC_NBR_ELL><<<blocks, 128, 0, s>>>(
          d_pos_sorted, n, d_cell_start, *grid, *box, cutoff2, half, out_tags, d_count,
          d_offsets, d_index, ell_stride, ell_width, d_flag, posb, ebox);
      break;
    case PC_NBR_SELL:
      if (ell_width % 4) {
        set_error("pc_nbr_build: SELL width must be a multiple of 4");
        return PC_ERR_VALUE;
      }
      nbr_build_kernel<PC_NBR_SELL><<<blocks, 128, 0, s>>>(
          d_pos_sorted, n, d_cell_start, *grid, *box, cutoff2, half, out_tags, d_count,
          d_offsets, d_index, ell_stride, ell_width, d_flag, posb, ebox);
      break;
    default:
      set_error("pc_nbr_build: unknown mode %d", mode);
      return PC_ERR_VALUE;
  }
  return check_launch("pc_nbr_build");
}

int pc_sort_rows(const int64_t* d_offsets, int32_t n, int32_t* d_index, void* stream) {
  if (n <= 0) return PC_OK;
  unsigned blocks = (unsigned)((n + kSortWarps - 1) / kSortWarps);
  sort_rows_kernel<<<blocks, kSortWarps * 32, 0, as_stream(stream)>>>(d_offsets, n, d_index);
  return check_launch("pc_sort_rows");
}

}  // extern "C"

namespace pc {
static int g_stage_bytes = 0;
}

// Deterministic mode: order every SELL row by the neighbours'
// global ids (the tag in pos4.w), so a row's pair terms are accumulated in
// the same order under any decomposition or cell order.  Warp per row: tags
// into shared memory, rank = number of smaller tags (ids in a row are
// distinct), scatter back.
constexpr int kSortRowCap = 256;

__global__ void __launch_bounds__(256)
sell_sort_by_tag_kernel(const double* __restrict__ pos, int n, const int* __restrict__ count,
                        int* __restrict__ nbr, int Q, int* __restrict__ flag) {
  __shared__ long long tag[8][kSortRowCap];
  __shared__ int idx[8][kSortRowCap];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + w;
  if (i >= n) return;
  const int m = count[i];
  if (m > kSortRowCap) {
    if (lane == 0) atomicOr(flag, kFlagOverflow);
    return;
  }
  for (int e = lane; e < m; e += 32) {
    const int j = nbr[sell_word(i, e, Q)];
    idx[w][e] = j;
    tag[w][e] = tag_of(pos[4 * (int64_t)j + 3]);
  }
  __syncwarp();
  for (int e = lane; e < m; e += 32) {
    const long long t = tag[w][e];
    int r = 0;
    for (int u = 0; u < m; ++u) r += tag[w][u] < t;
    nbr[sell_word(i, r, Q)] = idx[w][e];
  }
}

extern "C" int pc_sell_sort_by_tag(const double* d_pos, int32_t n, const int32_t* d_count,
                                   int32_t* d_index, int32_t width, int32_t* d_flag,
                                   void* stream) {
  using namespace pc;
  if (n <= 0) return PC_OK;
  if (width % 4) {
    set_error("pc_sell_sort_by_tag: width must be a multiple of 4");
    return PC_ERR_VALUE;
  }
  sell_sort_by_tag_kernel<<<(n + 7) / 8, 256, 0, as_stream(stream)>>>(d_pos, n, d_count, d_index,
                                                                    width / 4, d_flag);
  return check_launch("pc_sell_sort_by_tag");
}

extern "C" int pc_nbr_build_sell(const double* d_pos_sorted, int32_t n,
                                 const int32_t* d_cell_start, const pc_grid* grid,
                                 const pc_box* box, double cutoff2, int32_t width,
                                 int32_t dummy, int32_t* d_count, int32_t* d_index,
                                 int32_t* d_flag, int32_t* h_used_staged, void* stream,
                                 const double* d_posb, const pc_box* box_exact,
                                 int32_t half) {
  using namespace pc;
  if (n <= 0) return PC_OK;
  if (width % 4 || width <= 0) {
    set_error("pc_nbr_build_sell: width must be a positive multiple of 4");
    return PC_ERR_VALUE;
  }
  cudaStream_t s = as_stream(stream);
  bool staged = grid->ndim == 3;
  for (int a = 0; a < 3; ++a) staged &= !(box->periodic[a] && grid->nc[a] < 3);
  if (h_used_staged) *h_used_staged = staged ? 1 : 0;
  if (!staged) {
    // half: the per-particle kernel compares tags (global ids) -- also one
    // entry per unordered pair
    return pc_nbr_build(d_pos_sorted, n, d_cell_start, grid, box, cutoff2, half, PC_NBR_SELL,
                        0, d_count, nullptr, d_index, dummy, width, d_flag, stream, d_posb,
                        box_exact);
  }
  // FP32 prefilter band (see header comment of nbr_build_staged_kernel)
  double U = 0.0;
  const double wz = grid->width[2] * (kSegCells / 2.0 + 1.0);
  U = fmax(fmax(1.5 * grid->width[0], 1.5 * grid->width[1]), wz);
  const double rc = sqrt(cutoff2);
  const double e23 = ldexp(1.0, -23), e24 = ldexp(1.0, -24);
  const double err = 2.0 * sqrt(3.0) * rc * (e23 * U + e24 * rc) + 3.0 * e24 * cutoff2;
  const double margin = 8.0 * err + 1e-12 * cutoff2;
  StagedParams p;
  p.cutoff2 = cutoff2;
  p.lo2 = nextafterf((float)(cutoff2 - margin), -INFINITY);
  p.hi2 = nextafterf((float)(cutoff2 + margin), INFINITY);
  p.Q = width / 4;
  p.dummy = dummy;
  const int stage_bytes = 32 * 1024;
  p.max_stage = stage_bytes / (int)sizeof(float4);
  p.nseg = (grid->nc[2] + kSegCells - 1) / kSegCells;
  p.half = half;
  if (g_stage_bytes < stage_bytes) {
    cudaFuncSetAttribute(nbr_build_staged_kernel<PC_NBR_SELL>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, stage_bytes);
    g_stage_bytes = stage_bytes;
  }
  const int64_t blocks = (int64_t)grid->nc[0] * grid->nc[1] * p.nseg;
  nbr_build_staged_kernel<PC_NBR_SELL><<<(unsigned)blocks, kBuildThreads, stage_bytes, s>>>(
      d_pos_sorted, n, d_cell_start, *grid, *box, p, d_count, d_index, d_flag,
      d_posb ? d_posb : d_pos_sorted, box_exact ? *box_exact : *box);
  return check_launch("pc_nbr_build_sell");
}
