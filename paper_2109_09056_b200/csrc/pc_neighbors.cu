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
                 int* __restrict__ flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 pi = ld_pos4(pos + 4 * (int64_t)i);
  const int64_t ti = tag_of(pi.w);
  int sx[3], sy[3], sz[3];
  int nx = axis_stencil(cell_coord(pi.x, g.low[0], g.width[0], g.nc[0]), g.nc[0],
                        b.periodic[0], sx);
  int ny = axis_stencil(cell_coord(pi.y, g.low[1], g.width[1], g.nc[1]), g.nc[1],
                        b.periodic[1], sy);
  int nz = axis_stencil(cell_coord(pi.z, g.low[2], g.width[2], g.nc[2]), g.nc[2],
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
          const double dx = min_image(__dsub_rn(pj.x, pi.x), b.length[0], b.mi_thresh[0]);
          const double dy = min_image(__dsub_rn(pj.y, pi.y), b.length[1], b.mi_thresh[1]);
          const double dz = min_image(__dsub_rn(pj.z, pi.z), b.length[2], b.mi_thresh[2]);
          if (r2_exact(dx, dy, dz) < cutoff2) {
            const int64_t tj = tag_of(pj.w);
            if (half && !(tj > ti)) continue;
            if (MODE != PC_NBR_COUNT) {
              const int v = out_tags ? (int)tj : j;
              if (MODE == PC_NBR_CSR) {
                index[row + cnt] = v;
              } else if (cnt < ell_width) {
                index[(int64_t)cnt * ell_stride + i] = v;
              }
            }
            ++cnt;
          }
        }
      }
    }
  }
  count[i] = cnt;
  if (MODE == PC_NBR_ELL && cnt > ell_width) atomicOr(flag, kFlagOverflow);
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
                 void* stream) {
  if (n <= 0) return PC_OK;
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
          d_offsets, d_index, ell_stride, ell_width, d_flag);
      break;
    case PC_NBR_CSR:
      nbr_build_kernel<PC_NBR_CSR><<<blocks, 128, 0, s>>>(
          d_pos_sorted, n, d_cell_start, *grid, *box, cutoff2, half, out_tags, d_count,
          d_offsets, d_index, ell_stride, ell_width, d_flag);
      break;
    case PC_NBR_ELL:
      nbr_build_kernel<PC_NBR_ELL><<<blocks, 128, 0, s>>>(
          d_pos_sorted, n, d_cell_start, *grid, *box, cutoff2, half, out_tags, d_count,
          d_offsets, d_index, ell_stride, ell_width, d_flag);
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
