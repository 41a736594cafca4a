/* Device-side neighbor traversal over the CSR Verlet list of pc_nbr_build /
 * neighbors.build_verlet (int64 offsets[n + 1], int32 index[]): the B200
 * counterpart of the reference's for_each_neighbor / for_each_neighbor2
 * (ref neighbors.py:137-154), as device functors -- Cabana's
 * "neighbor parallel loops" for pair and three-body kernels.
 *
 *   pc_traverse::for_each_neighbor(list, begin, end, f, policy, stream)
 *       f(i, j) once per stored entry of rows [begin, end)
 *   pc_traverse::for_each_neighbor2(list, begin, end, f, policy, stream)
 *       f(i, j, k) once per pair of stored entries j before k of row i
 *       (full lists only, as the reference requires)
 *
 * Policies: Serial -- one thread per row, entries in stored order (the
 * reference's order within a row); Team -- one warp per row, the lanes
 * stride over the row's entries (or its (a, b) pairs), for long rows.  Rows
 * run concurrently in both: a functor that accumulates across rows must use
 * atomics or write per-row outputs.  Header-only CUDA C++ (sm_100a); include
 * from your own .cu and launch on your stream. */
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pc_traverse {

struct CsrList {
  const int64_t* offsets;   // n + 1
  const int32_t* index;     // offsets[n] entries
  int32_t n;
};

enum class Policy { Serial, Team };

namespace detail {

template <class F>
__global__ void pairs_serial(CsrList l, int begin, int end, F f) {
  const int i = begin + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= end) return;
  for (int64_t e = l.offsets[i]; e < l.offsets[i + 1]; ++e) f(i, (int)l.index[e]);
}

template <class F>
__global__ void pairs_team(CsrList l, int begin, int end, F f) {
  const int i = begin + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= end) return;
  for (int64_t e = l.offsets[i] + lane; e < l.offsets[i + 1]; e += 32) f(i, (int)l.index[e]);
}

template <class F>
__global__ void triplets_serial(CsrList l, int begin, int end, F f) {
  const int i = begin + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= end) return;
  const int64_t b = l.offsets[i], e = l.offsets[i + 1];
  for (int64_t a = b; a < e; ++a) {
    const int j = (int)l.index[a];
    for (int64_t c = a + 1; c < e; ++c) f(i, j, (int)l.index[c]);
  }
}

// (a, c) pairs of a row with m entries, a < c, enumerated by p in
// [0, m(m-1)/2): a is the largest with a * (2m - a - 1) / 2 <= p
__device__ __forceinline__ void unrank_pair(int64_t p, int64_t m, int64_t& a, int64_t& c) {
  const double mm = 2.0 * (double)m - 1.0;
  int64_t t = (int64_t)floor((mm - sqrt(mm * mm - 8.0 * (double)p)) * 0.5);
  if (t < 0) t = 0;
  while (t > 0 && t * (2 * m - t - 1) / 2 > p) --t;
  while ((t + 1) * (2 * m - t - 2) / 2 <= p) ++t;
  a = t;
  c = p - t * (2 * m - t - 1) / 2 + t + 1;
}

template <class F>
__global__ void triplets_team(CsrList l, int begin, int end, F f) {
  const int i = begin + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= end) return;
  const int64_t b = l.offsets[i], m = l.offsets[i + 1] - b;
  const int64_t np = m * (m - 1) / 2;
  for (int64_t p = lane; p < np; p += 32) {
    int64_t a, c;
    unrank_pair(p, m, a, c);
    f(i, (int)l.index[b + a], (int)l.index[b + c]);
  }
}

inline unsigned blocks_for(int64_t threads, int per_block) {
  return (unsigned)((threads + per_block - 1) / per_block);
}

}  // namespace detail

template <class F>
cudaError_t for_each_neighbor(const CsrList& l, int begin, int end, F f,
                              Policy policy = Policy::Serial, cudaStream_t s = 0) {
  if (begin < 0) begin = 0;
  if (end > l.n) end = l.n;
  if (end <= begin) return cudaSuccess;
  const int rows = end - begin;
  if (policy == Policy::Serial)
    detail::pairs_serial<<<detail::blocks_for(rows, 256), 256, 0, s>>>(l, begin, end, f);
  else
    detail::pairs_team<<<detail::blocks_for((int64_t)rows * 32, 256), 256, 0, s>>>(l, begin, end,
                                                                                  f);
  return cudaGetLastError();
}

template <class F>
cudaError_t for_each_neighbor2(const CsrList& l, int begin, int end, F f,
                               Policy policy = Policy::Serial, cudaStream_t s = 0) {
  if (begin < 0) begin = 0;
  if (end > l.n) end = l.n;
  if (end <= begin) return cudaSuccess;
  const int rows = end - begin;
  if (policy == Policy::Serial)
    detail::triplets_serial<<<detail::blocks_for(rows, 256), 256, 0, s>>>(l, begin, end, f);
  else
    detail::triplets_team<<<detail::blocks_for((int64_t)rows * 32, 256), 256, 0, s>>>(l, begin,
                                                                                     end, f);
  return cudaGetLastError();
}

}  // namespace pc_traverse
