// Velocity-Verlet integrate blocks of ref md.py:219-257 with the periodic
// wrap of geometry.py:40-49, in numpy's rounding order (no FMA contraction).
#include "pc_common.cuh"

namespace pc {

constexpr int kIntThreads = 256;

__global__ void __launch_bounds__(kIntThreads)
kick_drift_wrap_kernel(double* __restrict__ pos, double* __restrict__ v, int64_t vs,
                       const double* __restrict__ f, int64_t fs, int n, double dtm, double dt,
                       pc_box b, double* __restrict__ planar, int64_t ps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* p = pos + 4 * (int64_t)i;
  double x[3] = {p[0], p[1], p[2]};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double va = __dadd_rn(v[a * vs + i], __dmul_rn(dtm, f[a * fs + i]));
    v[a * vs + i] = va;
    double xa = __dadd_rn(x[a], __dmul_rn(dt, va));
    if (b.periodic[a]) xa = wrap_axis(xa, b.low[a], b.high[a], b.length[a]);
    x[a] = xa;
  }
  p[0] = x[0];
  p[1] = x[1];
  p[2] = x[2];
  if (planar) {
    planar[i] = x[0];
    planar[ps + i] = x[1];
    planar[2 * ps + i] = x[2];
  }
}

__global__ void pos_planar_kernel(const double* __restrict__ pos, int n,
                                  double* __restrict__ planar, int64_t ps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = ld_pos4(pos + 4 * (int64_t)i);
  planar[i] = p.x;
  planar[ps + i] = p.y;
  planar[2 * ps + i] = p.z;
}

// Rebuild permutation in one pass (ref md.py:169-188 sort + the planar copy):
// dst row k <- src row order[k]: x, y, z from the current planar positions,
// the id from pos4 .w, the planar velocities; writes the new pos4 rows and
// the new planar positions (a different buffer than the source).
// The decomposed engine's rebuild permutation in one pass: pos4, the
// local-frame binpos4, planar velocities and ghost flags by order[k], plus
// the planar x | y | z copies of both position arrays.
__global__ void domain_permute_kernel(const int* __restrict__ order, int n,
                                      const double* __restrict__ pos4,
                                      double* __restrict__ pos4_out,
                                      const double* __restrict__ bin4,
                                      double* __restrict__ bin4_out,
                                      const double* __restrict__ v, double* __restrict__ v_out,
                                      int64_t vs, const int* __restrict__ ghost,
                                      int* __restrict__ ghost_out, double* __restrict__ pl,
                                      double* __restrict__ bpl, int64_t ps) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int j = order[k];
  const double4 p = ld_pos4(pos4 + 4 * (int64_t)j);
  const double4 q = ld_pos4(bin4 + 4 * (int64_t)j);
  reinterpret_cast<double4*>(pos4_out)[k] = p;
  reinterpret_cast<double4*>(bin4_out)[k] = q;
  pl[k] = p.x;
  pl[ps + k] = p.y;
  pl[2 * ps + k] = p.z;
  bpl[k] = q.x;
  bpl[ps + k] = q.y;
  bpl[2 * ps + k] = q.z;
  v_out[k] = v[j];
  v_out[vs + k] = v[vs + j];
  v_out[2 * vs + k] = v[2 * vs + j];
  ghost_out[k] = ghost[j];
}

__global__ void md_permute_kernel(const int* __restrict__ order, int n,
                                  const double* __restrict__ pl, int64_t ps,
                                  const double* __restrict__ pos4, double* __restrict__ pos4_out,
                                  const double* __restrict__ v, double* __restrict__ v_out,
                                  int64_t vs, double* __restrict__ pl_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int j = order[k];
  const double x = pl[j], y = pl[ps + j], z = pl[2 * ps + j];
  const double w = pos4[4 * (int64_t)j + 3];
  reinterpret_cast<double4*>(pos4_out)[k] = make_double4(x, y, z, w);
  pl_out[k] = x;
  pl_out[ps + k] = y;
  pl_out[2 * ps + k] = z;
  v_out[k] = v[j];
  v_out[vs + k] = v[vs + j];
  v_out[2 * vs + k] = v[2 * vs + j];
}

__global__ void __launch_bounds__(kIntThreads)
kick_kernel(double* __restrict__ v, int64_t vs, const double* __restrict__ f, int64_t fs, int n,
            double dtm, double mass, double* __restrict__ partial) {
  __shared__ double red[kIntThreads / 32][5];
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double ke = 0.0, px = 0.0, py = 0.0, pz = 0.0;
  if (i < n) {
    double vx = __dadd_rn(v[i], __dmul_rn(dtm, f[i]));
    double vy = __dadd_rn(v[vs + i], __dmul_rn(dtm, f[fs + i]));
    double vz = __dadd_rn(v[2 * vs + i], __dmul_rn(dtm, f[2 * fs + i]));
    v[i] = vx;
    v[vs + i] = vy;
    v[2 * vs + i] = vz;
    ke = __dmul_rn(0.5 * mass, r2_exact(vx, vy, vz));
    px = mass * vx;
    py = mass * vy;
    pz = mass * vz;
  }
  if (!partial) return;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  ke = warp_sum(ke);
  px = warp_sum(px);
  py = warp_sum(py);
  pz = warp_sum(pz);
  if (lane == 0) {
    red[wid][0] = ke; red[wid][1] = 0.0; red[wid][2] = px; red[wid][3] = py; red[wid][4] = pz;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double s = 0.0;
    for (int w = 0; w < kIntThreads / 32; ++w) s += red[w][threadIdx.x];
    partial[blockIdx.x * 5 + threadIdx.x] = s;
  }
}

// Fixed-order reduction of block partials: deterministic for a given grid.
__global__ void __launch_bounds__(1024)
reduce_partials_kernel(const double* __restrict__ partial, int nblocks, double* __restrict__ out) {
  __shared__ double red[32][5];
  double s[5] = {0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < 5; ++k) s[k] += partial[b * 5 + k];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double v = warp_sum(s[k]);
    if (lane == 0) red[wid][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][threadIdx.x];
    out[threadIdx.x] = t;
  }
}

// ---- exact, order-independent sums (deterministic mode) --------------------
// Each FP64 value v (|v| < 2^50) is split exactly into an integer part and
// three 30-bit fraction limbs: |v| = i + (f1 2^60 + f2 2^30 + f3) 2^-90 - r,
// 0 <= r < 2^-90 (the bits below 2^-90 are truncated), limbs signed as v.  Limb sums are
// integer additions, so any partition of the atoms over threads, blocks,
// ranks or devices gives the same limb totals: the energies of a
// decomposed run equal the single-domain ones bit for bit (ref md.py:7-11,
// 261-277: "sums in global-id order" -- here the order does not matter at
// all), and ranks combine 4 x width int64 instead of one row per atom.
constexpr int kExactLimbs = 4;
constexpr int kExactMaxW = 8;

__device__ __forceinline__ void exact_split(double v, long long* l) {
  // split |v| (a - floor(a) is exact for a >= 0; for a small negative v,
  // v - floor(v) = v + 1 would round) and give the limbs v's sign: limbs may
  // be negative, exact_finish_kernel's floor-division carries normalise them
  const double a = fabs(v);
  const double hi = floor(a);
  double f = (a - hi) * 1073741824.0;            // exact: a - floor(a), * 2^30
  const double f1 = floor(f);
  f = (f - f1) * 1073741824.0;
  const double f2 = floor(f);
  f = (f - f2) * 1073741824.0;
  const double f3 = floor(f);
  const long long s = v < 0.0 ? -1 : 1;
  l[0] = s * (long long)hi;
  l[1] = s * (long long)f1;
  l[2] = s * (long long)f2;
  l[3] = s * (long long)f3;
}

__global__ void exact_sum_kernel(const double* __restrict__ rows, int64_t n, int w,
                                 const int* __restrict__ skip, long long* __restrict__ limbs) {
  long long acc[kExactMaxW][kExactLimbs];
#pragma unroll
  for (int c = 0; c < kExactMaxW; ++c)
#pragma unroll
    for (int q = 0; q < kExactLimbs; ++q) acc[c][q] = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (skip && skip[i]) continue;
#pragma unroll
    for (int c = 0; c < kExactMaxW; ++c) {
      if (c >= w) break;
      long long l[kExactLimbs];
      exact_split(rows[i * w + c], l);
#pragma unroll
      for (int q = 0; q < kExactLimbs; ++q) acc[c][q] += l[q];
    }
  }
#pragma unroll
  for (int c = 0; c < kExactMaxW; ++c) {
    if (c >= w) break;
#pragma unroll
    for (int q = 0; q < kExactLimbs; ++q) {
      long long v = acc[c][q];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0 && v)
        atomicAdd(reinterpret_cast<unsigned long long*>(limbs + c * kExactLimbs + q),
                  (unsigned long long)v);
    }
  }
}

// limbs -> doubles: carry-normalise the fraction limbs into [0, 2^30), then
// i + F 2^-90 with F = (f1 2^60 + f2 2^30 + f3) (deterministic rounding)
__global__ void exact_finish_kernel(const long long* __restrict__ limbs, int w,
                                    double* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= w) return;
  const long long M = 1LL << 30;
  long long i = limbs[c * 4], f1 = limbs[c * 4 + 1], f2 = limbs[c * 4 + 2], f3 = limbs[c * 4 + 3];
  long long k = f3 >> 30; f3 -= k * M; f2 += k;        // arithmetic shifts: floor division
  k = f2 >> 30; f2 -= k * M; f1 += k;
  k = f1 >> 30; f1 -= k * M; i += k;
  const double frac = ((double)f1 * 1073741824.0 + (double)f2) * 1073741824.0 + (double)f3;
  out[c] = (double)i + frac * 8.077935669463161e-28;     // 2^-90
}

// Box.wrap / Box.min_image on (rows, d) arrays (ref geometry.py:40-58).
__global__ void box_wrap_kernel(double* __restrict__ x, int64_t rows, int d, pc_box b) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * d) return;
  int a = (int)(t % d);
  if (b.periodic[a]) x[t] = wrap_axis(x[t], b.low[a], b.high[a], b.length[a]);
}

__global__ void box_min_image_kernel(double* __restrict__ x, int64_t rows, int d, pc_box b) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * d) return;
  int a = (int)(t % d);
  if (b.periodic[a]) {
    double v = x[t];
    double L = b.length[a];
    // literal form: general |v| (no |v| < L precondition here)
    x[t] = __dsub_rn(v, __dmul_rn(L, rint(__ddiv_rn(v, L))));
  }
}

// lj_pair of ref md.py:89-96 in FP64, same operation order.
__global__ void lj_pair_kernel(const double* __restrict__ dx, const double* __restrict__ r2,
                               int64_t n, double eps, double sigma, double* __restrict__ e,
                               double* __restrict__ f) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q = r2[i];
  double sr2 = __ddiv_rn(__dmul_rn(sigma, sigma), q);
  double sr6 = __dmul_rn(__dmul_rn(sr2, sr2), sr2);
  double sr12 = __dmul_rn(sr6, sr6);
  e[i] = __dmul_rn(__dmul_rn(4.0, eps), __dsub_rn(sr12, sr6));
  double fm = __ddiv_rn(__dmul_rn(__dmul_rn(24.0, eps), __dsub_rn(__dmul_rn(2.0, sr12), sr6)), q);
#pragma unroll
  for (int a = 0; a < 3; ++a) f[3 * i + a] = __dmul_rn(-fm, dx[3 * i + a]);
}

}  // namespace pc

using namespace pc;

extern "C" {

int pc_kick_drift_wrap(double* d_pos, double* d_v, int64_t v_stride, const double* d_f3,
                       int64_t f_stride, int32_t n, double dtm, double dt, const pc_box* box,
                       double* d_planar, int64_t planar_stride, void* stream) {
  if (n <= 0) return PC_OK;
  kick_drift_wrap_kernel<<<(n + kIntThreads - 1) / kIntThreads, kIntThreads, 0,
                           as_stream(stream)>>>(d_pos, d_v, v_stride, d_f3, f_stride, n, dtm, dt,
                                                *box, d_planar, planar_stride);
  return check_launch("pc_kick_drift_wrap");
}

int pc_domain_permute(const int32_t* d_order, int32_t n, const double* d_pos4,
                      double* d_pos4_out, const double* d_bin4, double* d_bin4_out,
                      const double* d_v, double* d_v_out, int64_t v_stride,
                      const int32_t* d_ghost, int32_t* d_ghost_out, double* d_planar,
                      double* d_bplanar, int64_t planar_stride, void* stream) {
  if (n <= 0) return PC_OK;
  domain_permute_kernel<<<(n + kIntThreads - 1) / kIntThreads, kIntThreads, 0,
                          as_stream(stream)>>>(d_order, n, d_pos4, d_pos4_out, d_bin4,
                                               d_bin4_out, d_v, d_v_out, v_stride, d_ghost,
                                               d_ghost_out, d_planar, d_bplanar, planar_stride);
  return check_launch("pc_domain_permute");
}

int pc_md_permute(const int32_t* d_order, int32_t n, const double* d_planar,
                  int64_t planar_stride, const double* d_pos4, double* d_pos4_out,
                  const double* d_v, double* d_v_out, int64_t v_stride, double* d_planar_out,
                  void* stream) {
  if (n <= 0) return PC_OK;
  if (d_planar == d_planar_out) {
    set_error("pc_md_permute: the planar source and destination must differ");
    return PC_ERR_VALUE;
  }
  md_permute_kernel<<<(n + kIntThreads - 1) / kIntThreads, kIntThreads, 0, as_stream(stream)>>>(
      d_order, n, d_planar, planar_stride, d_pos4, d_pos4_out, d_v, d_v_out, v_stride,
      d_planar_out);
  return check_launch("pc_md_permute");
}

int pc_pos_planar(const double* d_pos, int32_t n, double* d_planar, int64_t planar_stride,
                  void* stream) {
  if (n <= 0) return PC_OK;
  pos_planar_kernel<<<(n + kIntThreads - 1) / kIntThreads, kIntThreads, 0, as_stream(stream)>>>(
      d_pos, n, d_planar, planar_stride);
  return check_launch("pc_pos_planar");
}

int pc_kick(double* d_v, int64_t v_stride, const double* d_f3, int64_t f_stride, int32_t n,
            double dtm, double mass, double* d_partial, void* stream) {
  if (n <= 0) n = 0;
  int blocks = n == 0 ? 1 : (n + kIntThreads - 1) / kIntThreads;
  kick_kernel<<<blocks, kIntThreads, 0, as_stream(stream)>>>(d_v, v_stride, d_f3, f_stride, n,
                                                             dtm, mass, d_partial);
  return check_launch("pc_kick");
}

int pc_box_wrap(double* d_x, int64_t rows, int32_t d, const pc_box* box, void* stream) {
  int64_t t = rows * d;
  if (t <= 0) return PC_OK;
  box_wrap_kernel<<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(d_x, rows, d, *box);
  return check_launch("pc_box_wrap");
}

int pc_box_min_image(double* d_x, int64_t rows, int32_t d, const pc_box* box, void* stream) {
  int64_t t = rows * d;
  if (t <= 0) return PC_OK;
  box_min_image_kernel<<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(d_x, rows, d,
                                                                                   *box);
  return check_launch("pc_box_min_image");
}

int pc_lj_pair(const double* d_dx, const double* d_r2, int64_t n, double eps, double sigma,
               double* d_e, double* d_f, void* stream) {
  if (n <= 0) return PC_OK;
  lj_pair_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(d_dx, d_r2, n, eps,
                                                                             sigma, d_e, d_f);
  return check_launch("pc_lj_pair");
}

int pc_exact_sum(const double* d_rows, int64_t n, int32_t w, const int32_t* d_skip,
                 int64_t* d_limbs, void* stream) {
  if (w < 1 || w > kExactMaxW) {
    set_error("pc_exact_sum: width must be in [1, %d]", kExactMaxW);
    return PC_ERR_VALUE;
  }
  if (n <= 0) return PC_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  exact_sum_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      d_rows, n, w, d_skip, reinterpret_cast<long long*>(d_limbs));
  return check_launch("pc_exact_sum");
}

int pc_exact_finish(const int64_t* d_limbs, int32_t w, double* d_out, void* stream) {
  if (w < 1 || w > kExactMaxW) {
    set_error("pc_exact_finish: width must be in [1, %d]", kExactMaxW);
    return PC_ERR_VALUE;
  }
  exact_finish_kernel<<<1, 32, 0, as_stream(stream)>>>(
      reinterpret_cast<const long long*>(d_limbs), w, d_out);
  return check_launch("pc_exact_finish");
}

int pc_reduce_partials(const double* d_partial, int32_t nblocks, double* d_out, void* stream) {
  reduce_partials_kernel<<<1, 1024, 0, as_stream(stream)>>>(d_partial, nblocks, d_out);
  return check_launch("pc_reduce_partials");
}

}  // extern "C"
