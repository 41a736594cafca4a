// Linked-cell binning: cell assignment + warp-aggregated counts, device
// prefix scan, stable counting-sort placement, permutation helpers.
// Replaces ref binning.py:49-101 and the sort inside neighbors.py:56-66.
#include "pc_common.cuh"

namespace pc {

// ---- K1: cell id + count -------------------------------------------------
__global__ void __launch_bounds__(256)
bin_count_kernel(const double* __restrict__ x, int64_t n, int x_stride, int64_t a_stride,
                 pc_grid g, int check_inside, int* __restrict__ cell_of,
                 int64_t* __restrict__ axis_idx, int* __restrict__ cell_count,
                 int* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int cell = -1;
  if (i < n) {
    const double* p = x + i * x_stride;
    int c[3] = {0, 0, 0};
    bool outside = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {     // unrolled: no local copy of g (was a 112-B stack frame)
      if (a >= g.ndim) break;
      double v = p[a * a_stride];
      outside |= (v < g.low[a]) || (v > g.high[a]);
      c[a] = cell_coord(v, g.low[a], g.width[a], g.nc[a]);
      if (axis_idx) axis_idx[i * g.ndim + a] = c[a];
    }
    if (check_inside && outside) atomicOr(flag, kFlagOutside);
    cell = (c[0] * g.nc[1] + c[1]) * g.nc[2] + c[2];
    cell_of[i] = cell;
  }
  // warp-aggregated atomics: consecutive particles mostly share a cell
  unsigned peers = __match_any_sync(0xffffffffu, cell);
  int leader = __ffs(peers) - 1;
  if (cell >= 0 && (int)(threadIdx.x & 31) == leader)
    atomicAdd(cell_count + cell, __popc(peers));
}

// Integer keys -> digit "cells" for the LSD passes of bin_by_key.
__global__ void __launch_bounds__(256)
key_digit_kernel(const int64_t* __restrict__ keys, const int* __restrict__ perm, int64_t n,
                 int64_t kmin, int shift, int64_t mask, int* __restrict__ cell_of,
                 int* __restrict__ cell_count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int cell = -1;
  if (i < n) {
    int64_t k = keys[perm ? perm[i] : i];
    uint64_t u = (uint64_t)k - (uint64_t)kmin;
    cell = (int)((u >> shift) & (uint64_t)mask);
    cell_of[i] = cell;
  }
  unsigned peers = __match_any_sync(0xffffffffu, cell);
  int leader = __ffs(peers) - 1;
  if (cell >= 0 && (int)(threadIdx.x & 31) == leader) atomicAdd(cell_count + cell, __popc(peers));
}

// Permutation.is_bijection (ref binning.py:26-33): range + duplicate check.
__global__ void bijection_kernel(const int64_t* __restrict__ map, int64_t n,
                                 int* __restrict__ seen, int* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t d = map[i];
  if (d < 0 || d >= n) {
    atomicOr(flag, 1);
    return;
  }
  if (atomicAdd(seen + d, 1) != 0) atomicOr(flag, 2);
}

// ---- K2: exclusive scan (tile reduce -> recursive scan of sums -> apply) --
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem_warp, T& total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) smem_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : T(0);
    T si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T t = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += t;
    }
    smem_warp[lane] = si - s;
    if (lane == 31) smem_warp[32] = si;
  }
  __syncthreads();
  total = smem_warp[32];
  T r = inc - v + smem_warp[wid];
  __syncthreads();
  return r;
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kScanThreads)
scan_tiles_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t n,
                  Tout* __restrict__ tile_sums) {
  __shared__ Tout warp_sums[33];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  Tout v[kScanItems];
  Tout local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < n) ? (Tout)in[base + k] : Tout(0);
    local += v[k];
  }
  Tout total;
  Tout run = block_exclusive_scan<Tout>(local, warp_sums, total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

template <typename Tout>
__global__ void scan_add_kernel(Tout* __restrict__ out, int64_t n,
                                const Tout* __restrict__ tile_offsets) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_offsets[i / kScanTile];
}

template <typename Tout>
__global__ void scan_total_kernel(const Tout* __restrict__ tile_offsets, int64_t ntiles,
                                  const Tout* __restrict__ tile_sums, Tout* __restrict__ out,
                                  int64_t n) {
  out[n] = tile_offsets[ntiles - 1] + tile_sums[ntiles - 1];
}

static int64_t scan_tmp_elems(int64_t n) {
  // per level: tile sums + scanned tile offsets
  int64_t total = 0;
  while (true) {
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles < 1) tiles = 1;
    total += 2 * tiles + 1;
    if (tiles == 1) break;
    n = tiles;
  }
  return total;
}

// out has n+1 entries; tmp holds scan_tmp_elems(n) Tout values.
template <typename Tin, typename Tout>
static int scan_impl(const Tin* in, Tout* out, int64_t n, Tout* tmp, cudaStream_t s) {
  if (n == 0) {
    cudaMemsetAsync(out, 0, sizeof(Tout), s);
    return check_launch("scan(empty)", 0);
  }
  int64_t tiles = (n + kScanTile - 1) / kScanTile;
  Tout* sums = tmp;
  Tout* offs = tmp + tiles;
  scan_tiles_kernel<Tin, Tout><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, sums);
  int launched = 2;
  if (tiles == 1) {
    cudaMemsetAsync(offs, 0, sizeof(Tout), s);
  } else {
    int rc = scan_impl<Tout, Tout>(sums, offs, tiles, tmp + 2 * tiles + 1, s);
    if (rc) return rc;
    scan_add_kernel<Tout><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, offs);
    launched = 3;
  }
  scan_total_kernel<Tout><<<1, 1, 0, s>>>(offs, tiles, sums, out, n);
  return check_launch("scan", launched);
}

// ---- K3: stable placement -----------------------------------------------
__global__ void bin_place_kernel(const int* __restrict__ cell_of, int64_t n,
                                 const int* __restrict__ cell_start,
                                 int* __restrict__ cell_fill, int* __restrict__ order_tmp) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int cell = i < n ? cell_of[i] : -1;
  // warp-aggregated slot reservation, ranks within the warp by lane order
  unsigned peers = __match_any_sync(0xffffffffu, cell);
  int lane = threadIdx.x & 31;
  int leader = __ffs(peers) - 1;
  int base = 0;
  if (cell >= 0 && lane == leader) base = atomicAdd(cell_fill + cell, __popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (cell >= 0) {
    int rank = __popc(peers & ((1u << lane) - 1u));
    order_tmp[cell_start[cell] + base + rank] = (int)i;
  }
}

// Warp per cell: atomics made the in-cell order arbitrary; restore the stable
// (ascending source index) order by rank counting.  Source indices in a cell
// are distinct, so rank = #smaller is a bijection onto the segment.
__global__ void __launch_bounds__(256)
bin_stabilize_kernel(const int* __restrict__ cell_start, int ncells,
                     const int* __restrict__ order_tmp, int* __restrict__ order) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= ncells) return;
  int b = cell_start[warp], e = cell_start[warp + 1];
  int m = e - b;
  if (m == 0) return;
  if (m <= 32) {
    int v = lane < m ? order_tmp[b + lane] : 0x7fffffff;
    int rank = 0;
    for (int t = 0; t < m; ++t) {
      int u = __shfl_sync(0xffffffffu, v, t);
      rank += (u < v);
    }
    if (lane < m) order[b + rank] = v;
    return;
  }
  for (int k = lane; k < m; k += 32) {
    int v = order_tmp[b + k];
    int rank = 0;
    for (int t = 0; t < m; ++t) rank += (order_tmp[b + t] < v);
    order[b + rank] = v;
  }
}

__global__ void invert_order_kernel(const int* __restrict__ order, int64_t n,
                                    int64_t* __restrict__ map) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) map[order[k]] = k;
}

// ---- row gather / AoSoA permute ------------------------------------------
__global__ void gather_rows16_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                     const int* __restrict__ order, int64_t n, int vecs) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t k = t / vecs;
  int c = (int)(t - k * vecs);
  if (k < n) dst[k * vecs + c] = src[(int64_t)order[k] * vecs + c];
}

__global__ void gather_rows4_kernel(const int* __restrict__ src, int* __restrict__ dst,
                                    const int* __restrict__ order, int64_t n) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = src[order[k]];
}

__global__ void gather_rows8_kernel(const int64_t* __restrict__ src, int64_t* __restrict__ dst,
                                    const int* __restrict__ order, int64_t n, int words) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t k = t / words;
  int c = (int)(t - k * words);
  if (k < n) dst[k * words + c] = src[(int64_t)order[k] * words + c];
}

__global__ void scatter_rows8_kernel(const int64_t* __restrict__ src, int64_t* __restrict__ dst,
                                     const int* __restrict__ order, int64_t n, int words) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t k = t / words;
  int c = (int)(t - k * words);
  if (k < n) dst[(int64_t)order[k] * words + c] = src[k * words + c];
}

__global__ void scatter_rows4_kernel(const int* __restrict__ src, int* __restrict__ dst,
                                     const int* __restrict__ order, int64_t n) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[order[k]] = src[k];
}

// AoSoA field <-> dense (n, ncomp) copy (ref aosoa.py:124-142).
__global__ void aosoa_field_kernel(uint8_t* __restrict__ buf, int64_t n, int V,
                                   int64_t struct_bytes, int64_t field_off, int ncomp,
                                   int64_t* __restrict__ dense, int to_dense) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = t / ncomp;
  int c = (int)(t - i * ncomp);
  if (i >= n) return;
  int64_t off = struct_bytes * (i / V) + field_off + ((int64_t)c * V + (i % V)) * 8;
  int64_t* p = reinterpret_cast<int64_t*>(buf + off);
  if (to_dense) dense[t] = *p;
  else *p = dense[t];
}

__global__ void csr_to_dense_kernel(const int64_t* __restrict__ offsets, int n,
                                    const int* __restrict__ index, int width,
                                    int64_t* __restrict__ table) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = t / (width > 0 ? width : 1);
  int s = (int)(t - i * width);
  if (width == 0 || i >= n) return;
  int64_t b = offsets[i], m = offsets[i + 1] - b;
  table[t] = s < m ? (int64_t)index[b + s] : -1;
}

__global__ void aosoa_permute_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                     const int64_t* __restrict__ map, int64_t n, int V,
                                     int64_t struct_bytes, const int64_t* __restrict__ word_base,
                                     int nwords) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = t / nwords;
  int w = (int)(t - i * nwords);
  if (i >= n) return;
  int64_t d = map[i];
  int64_t so = struct_bytes * (i / V) + word_base[w] + (i % V) * 8;
  int64_t dof = struct_bytes * (d / V) + word_base[w] + (d % V) * 8;
  *reinterpret_cast<int64_t*>(dst + dof) = *reinterpret_cast<const int64_t*>(src + so);
}

}  // namespace pc

using namespace pc;

extern "C" {

int pc_bin_count(const double* d_x, int64_t n, int32_t x_stride, const pc_grid* grid,
                 int32_t check_inside, int32_t* d_cell_of, int64_t* d_axis_idx,
                 int32_t* d_cell_count, int32_t* d_flag, void* stream) {
  if (n <= 0) return PC_OK;
  if (grid->ndim < 1 || grid->ndim > 3 || x_stride < grid->ndim) {
    set_error("pc_bin_count: bad ndim/x_stride");
    return PC_ERR_VALUE;
  }
  unsigned blocks = (unsigned)((n + 255) / 256);
  bin_count_kernel<<<blocks, 256, 0, as_stream(stream)>>>(d_x, n, x_stride, 1, *grid,
                                                          check_inside, d_cell_of, d_axis_idx,
                                                          d_cell_count, d_flag);
  return check_launch("pc_bin_count");
}

int pc_bin_count_planar(const double* d_planar, int64_t planar_stride, int64_t n,
                        const pc_grid* grid, int32_t* d_cell_of, int32_t* d_cell_count,
                        int32_t* d_flag, void* stream) {
  if (n <= 0) return PC_OK;
  if (grid->ndim != 3) {
    set_error("pc_bin_count_planar: 3-D only");
    return PC_ERR_VALUE;
  }
  unsigned blocks = (unsigned)((n + 255) / 256);
  bin_count_kernel<<<blocks, 256, 0, as_stream(stream)>>>(d_planar, n, 1, planar_stride, *grid,
                                                          0, d_cell_of, nullptr, d_cell_count,
                                                          d_flag);
  return check_launch("pc_bin_count_planar");
}

int pc_key_digits(const int64_t* d_keys, const int32_t* d_perm, int64_t n, int64_t kmin,
                  int32_t shift, int64_t mask, int32_t* d_cell_of, int32_t* d_cell_count,
                  void* stream) {
  if (n <= 0) return PC_OK;
  key_digit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_keys, d_perm, n, kmin, shift, mask, d_cell_of, d_cell_count);
  return check_launch("pc_key_digits");
}

int pc_check_bijection(const int64_t* d_map, int64_t n, int32_t* d_seen, int32_t* d_flag,
                       void* stream) {
  if (n <= 0) return PC_OK;
  bijection_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(d_map, n, d_seen,
                                                                               d_flag);
  return check_launch("pc_check_bijection");
}

int pc_scatter_rows(const void* d_src, void* d_dst, const int32_t* d_order, int64_t n,
                    int32_t row_bytes, void* stream) {
  if (n <= 0) return PC_OK;
  cudaStream_t s = as_stream(stream);
  if (row_bytes == 4) {
    scatter_rows4_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        (const int*)d_src, (int*)d_dst, d_order, n);
  } else if (row_bytes % 8 == 0) {
    int words = row_bytes / 8;
    int64_t tot = n * words;
    scatter_rows8_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
        (const int64_t*)d_src, (int64_t*)d_dst, d_order, n, words);
  } else {
    set_error("pc_scatter_rows: row_bytes must be 4 or a multiple of 8");
    return PC_ERR_VALUE;
  }
  return check_launch("pc_scatter_rows");
}

int pc_aosoa_field(void* d_buf, int64_t n, int32_t V, int64_t struct_bytes, int64_t field_off,
                   int32_t ncomp, void* d_dense, int32_t to_dense, void* stream) {
  int64_t tot = n * ncomp;
  if (tot <= 0) return PC_OK;
  aosoa_field_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, as_stream(stream)>>>(
      (uint8_t*)d_buf, n, V, struct_bytes, field_off, ncomp, (int64_t*)d_dense, to_dense);
  return check_launch("pc_aosoa_field");
}

int pc_csr_to_dense(const int64_t* d_offsets, int32_t n, const int32_t* d_index, int32_t width,
                    int64_t* d_table, void* stream) {
  int64_t tot = (int64_t)n * width;
  if (tot <= 0) return PC_OK;
  csr_to_dense_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_offsets, n, d_index, width, d_table);
  return check_launch("pc_csr_to_dense");
}

// ---- stable partition into few bins (<= 256) ------------------------------
// The atomic placement + per-cell stabilisation above is built for linked
// cells of ~20 particles (rank counting is O(m^2) per cell).  Grouping by
// owner rank (ref decomp.py:97-99) or by a key digit puts up to n elements in
// one bin, so these use a chunked stable partition instead: per 1024-element
// chunk a histogram (bin-major hist[b * nchunks + c]), one exclusive scan
// (pc_scan_i32: off = global start of chunk c's elements of bin b), then each
// element's rank among equal keys of its chunk in index order (MATCH.ANY in
// the warp + per-warp prefix per bin).  O(n), deterministic, stable.
constexpr int kPartChunk = 1024;
constexpr int kPartMaxBins = 256;

__global__ void __launch_bounds__(kPartChunk)
partition_hist_kernel(const int* __restrict__ keys, int64_t n, int nbins, int nchunks,
                      int* __restrict__ hist) {
  __shared__ int h[kPartMaxBins];
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kPartChunk + threadIdx.x;
  if (i < n) {
    const int k = keys[i];
    if ((unsigned)k < (unsigned)nbins) atomicAdd(&h[k], 1);     // (out of range: dropped)
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    hist[(int64_t)b * nchunks + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(kPartChunk)
partition_place_kernel(const int* __restrict__ keys, int64_t n, int nbins, int nchunks,
                       const int* __restrict__ off, int* __restrict__ order) {
  __shared__ int wc[kPartChunk / 32][kPartMaxBins];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = lane; b < nbins; b += 32) wc[warp][b] = 0;
  const int64_t i = (int64_t)blockIdx.x * kPartChunk + threadIdx.x;
  const int kraw = i < n ? keys[i] : -1;
  const int key = (unsigned)kraw < (unsigned)nbins ? kraw : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  __syncwarp();
  if (key >= 0 && rank == 0) wc[warp][key] = __popc(peers);
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {    // prefix over warps
    int run = 0;
    for (int w = 0; w < kPartChunk / 32; ++w) {
      const int v = wc[w][b];
      wc[w][b] = run;
      run += v;
    }
  }
  __syncthreads();
  if (key >= 0)
    order[off[(int64_t)key * nchunks + blockIdx.x] + wc[warp][key] + rank] = (int)i;
}

int64_t pc_partition_chunks(int64_t n) { return n > 0 ? (n + kPartChunk - 1) / kPartChunk : 0; }

int pc_partition_hist(const int32_t* d_keys, int64_t n, int32_t nbins, int32_t* d_hist,
                      void* stream) {
  if (nbins <= 0 || nbins > kPartMaxBins) {
    set_error("pc_partition_hist: nbins must be in [1, %d]", kPartMaxBins);
    return PC_ERR_VALUE;
  }
  if (n <= 0) return PC_OK;
  const int64_t nch = pc_partition_chunks(n);
  partition_hist_kernel<<<(unsigned)nch, kPartChunk, 0, as_stream(stream)>>>(
      d_keys, n, nbins, (int)nch, d_hist);
  return check_launch("pc_partition_hist");
}

int pc_partition_place(const int32_t* d_keys, int64_t n, int32_t nbins, const int32_t* d_off,
                       int32_t* d_order, void* stream) {
  if (nbins <= 0 || nbins > kPartMaxBins) {
    set_error("pc_partition_place: nbins must be in [1, %d]", kPartMaxBins);
    return PC_ERR_VALUE;
  }
  if (n <= 0) return PC_OK;
  const int64_t nch = pc_partition_chunks(n);
  partition_place_kernel<<<(unsigned)nch, kPartChunk, 0, as_stream(stream)>>>(
      d_keys, n, nbins, (int)nch, d_off, d_order);
  return check_launch("pc_partition_place");
}

int64_t pc_scan_tmp_bytes(int64_t n) { return scan_tmp_elems(n) * (int64_t)sizeof(int64_t); }

int pc_scan_i32(const int32_t* d_in, int32_t* d_out, int64_t n, void* d_tmp,
                int64_t tmp_bytes, void* stream) {
  if (tmp_bytes < pc_scan_tmp_bytes(n)) {
    set_error("pc_scan_i32: scratch too small");
    return PC_ERR_VALUE;
  }
  return scan_impl<int, int>(d_in, d_out, n, reinterpret_cast<int*>(d_tmp), as_stream(stream));
}

int pc_scan_i32_i64(const int32_t* d_in, int64_t* d_out, int64_t n, void* d_tmp,
                    int64_t tmp_bytes, void* stream) {
  if (tmp_bytes < pc_scan_tmp_bytes(n)) {
    set_error("pc_scan_i32_i64: scratch too small");
    return PC_ERR_VALUE;
  }
  return scan_impl<int, int64_t>(d_in, d_out, n, reinterpret_cast<int64_t*>(d_tmp),
                                 as_stream(stream));
}

int pc_bin_place(const int32_t* d_cell_of, int64_t n, const int32_t* d_cell_start,
                 int32_t ncells, int32_t* d_cell_fill, int32_t* d_order_tmp, int32_t* d_order,
                 void* stream) {
  if (n <= 0) return PC_OK;
  cudaStream_t s = as_stream(stream);
  bin_place_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d_cell_of, n, d_cell_start,
                                                               d_cell_fill, d_order_tmp);
  unsigned wblocks = (unsigned)(((int64_t)ncells * 32 + 255) / 256);
  bin_stabilize_kernel<<<wblocks, 256, 0, s>>>(d_cell_start, ncells, d_order_tmp, d_order);
  return check_launch("pc_bin_place", 2);
}

int pc_bin_place_unstable(const int32_t* d_cell_of, int64_t n, const int32_t* d_cell_start,
                          int32_t* d_cell_fill, int32_t* d_order, void* stream) {
  if (n <= 0) return PC_OK;
  bin_place_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_cell_of, n, d_cell_start, d_cell_fill, d_order);
  return check_launch("pc_bin_place_unstable");
}

int pc_invert_order(const int32_t* d_order, int64_t n, int64_t* d_map, void* stream) {
  if (n <= 0) return PC_OK;
  invert_order_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(d_order, n,
                                                                                  d_map);
  return check_launch("pc_invert_order");
}

int pc_gather_rows(const void* d_src, void* d_dst, const int32_t* d_order, int64_t n,
                   int32_t row_bytes, void* stream) {
  if (n <= 0) return PC_OK;
  cudaStream_t s = as_stream(stream);
  if (row_bytes == 4) {
    gather_rows4_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        (const int*)d_src, (int*)d_dst, d_order, n);
    return check_launch("pc_gather_rows");
  }
  if (row_bytes % 8) {
    set_error("pc_gather_rows: row_bytes must be 4 or a multiple of 8");
    return PC_ERR_VALUE;
  }
  bool al16 = (row_bytes % 16 == 0) && ((uintptr_t)d_src % 16 == 0) && ((uintptr_t)d_dst % 16 == 0);
  if (al16) {
    int vecs = row_bytes / 16;
    int64_t tot = n * vecs;
    gather_rows16_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
        (const int4*)d_src, (int4*)d_dst, d_order, n, vecs);
  } else {
    int words = row_bytes / 8;
    int64_t tot = n * words;
    gather_rows8_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
        (const int64_t*)d_src, (int64_t*)d_dst, d_order, n, words);
  }
  return check_launch("pc_gather_rows");
}

int pc_aosoa_permute(const void* d_src, void* d_dst, const int64_t* d_map, int64_t n, int32_t V,
                     int64_t struct_bytes, const int64_t* d_word_base, int32_t nwords,
                     void* stream) {
  if (n <= 0 || nwords <= 0) return PC_OK;
  int64_t tot = n * nwords;
  aosoa_permute_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, as_stream(stream)>>>(
      (const uint8_t*)d_src, (uint8_t*)d_dst, d_map, n, V, struct_bytes, d_word_base, nwords);
  return check_launch("pc_aosoa_permute");
}

}  // extern "C"
