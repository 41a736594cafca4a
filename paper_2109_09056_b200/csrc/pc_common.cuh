// Shared device helpers for the particula B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/particula_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "particula_b200 targets sm_100a (B200) only"
#endif

namespace pc {

// ---- host-side error plumbing ---------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what, int launches = 1);
void note_launch(int k);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kFlagOutside = 1;   // ValueError: position outside box
constexpr int kFlagOverflow = 2;  // neighbor row exceeded ELL width
constexpr int kFlagOverlap = 4;   // FloatingPointError: r^2 < overlap^2
constexpr int kFlagNonPeriodic = 8;
constexpr int kFlagStage = 16;     // staged build: neighborhood exceeded smem

// ---- device helpers ------------------------------------------------------
// 256-bit read-only gather of one pos4 (x, y, z, tag): one DRAM sector.
__device__ __forceinline__ double4 ld_pos4(const double* p) {
  double4 r;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ int64_t tag_of(double w) { return __double_as_longlong(w); }

// Exact d - L*round_half_even(d/L) (ref geometry.py:51-58).  For |d| < L the
// rounded quotient is -1, 0 or 1 and the threshold test `|d| >= T` (T from
// the host, pc_box.mi_thresh) decides it without a division; fl(|d| - L) with
// the sign of -d equals fl(d -/+ L) because round-to-nearest is symmetric.
// |d| >= L (unwrapped input) falls back to the literal division formula.
__device__ __forceinline__ double min_image(double d, double L, double T) {
  double a = fabs(d);
  if (a >= T) {
    if (a < L) return copysign(__dsub_rn(a, L), -d);
    return __dsub_rn(d, __dmul_rn(L, rint(__ddiv_rn(d, L))));
  }
  return d;
}

// Branch-free minimum image for wrapped coordinates (|d| < L): the fast form
// of pc::min_image without its |d| >= L division fallback.
__device__ __forceinline__ double min_image_wrapped(double d, double L, double T) {
  const double a = fabs(d);
  const double t = copysign(__dsub_rn(a, L), -d);
  return a >= T ? t : d;
}

// ---- periodic wrap of ref geometry.py:40-49 (numpy rounding) --------------
// numpy float mod (npy_divmod): fmod, then shift a nonzero remainder whose
// sign differs from the divisor's; zero takes the divisor's sign.
__device__ __forceinline__ double np_mod(double a, double L) {
  double m = fmod(a, L);
  if (m != 0.0) {
    if ((L < 0.0) != (m < 0.0)) m = __dadd_rn(m, L);
  } else {
    m = copysign(0.0, L);
  }
  return m;
}

__device__ __forceinline__ double wrap_axis(double x, double low, double high, double L) {
  double w = __dadd_rn(low, np_mod(__dsub_rn(x, low), L));
  return w >= high ? low : w;
}

// The same for a particle that moved less than one box length out of
// [low, high) (every MD step): fmod(a, L) is a for a in [0, L) and the exact
// a - L (Sterbenz) for a in [L, 2L); a in (-L, 0) takes numpy's +L fix.
__device__ __forceinline__ double wrap_axis_near(double x, double low, double high, double L) {
  const double a = __dsub_rn(x, low);
  if (!(a > -L && a < 2.0 * L)) return wrap_axis(x, low, high, L);
  const double m = a >= L ? __dsub_rn(a, L) : (a < 0.0 ? __dadd_rn(a, L) : a);
  const double w = __dadd_rn(low, m == 0.0 ? 0.0 : m);
  return w >= high ? low : w;
}

// numpy einsum order on this build: (x*x + z*z) + y*y, no FMA.
__device__ __forceinline__ double r2_exact(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
}

__device__ __forceinline__ int cell_coord(double x, double low, double width, int nc) {
  // floor((x - low) / width), clamped to [0, nc-1]; IEEE division as numpy
  double q = floor(__ddiv_rn(__dsub_rn(x, low), width));
  int c = q < 0.0 ? 0 : (q >= (double)nc ? nc - 1 : (int)q);
  return c;
}

// Distinct neighbor-cell coordinates along one axis, ascending (ref
// neighbors.py:76-89 dedups stencil cells through a set and visits them in
// sorted flat-id order; row-major flat ids make per-axis ascending order the
// same thing).  Returns the count (1..3).
__device__ __forceinline__ int axis_stencil(int c, int nc, int periodic, int out[3]) {
  int k = 0;
  int cand[3] = {c - 1, c, c + 1};
  for (int t = 0; t < 3; ++t) {
    int v = cand[t];
    if (periodic) {
      v = ((v % nc) + nc) % nc;
    } else if (v < 0 || v >= nc) {
      continue;
    }
    bool dup = false;
    for (int u = 0; u < k; ++u) dup |= (out[u] == v);
    if (!dup) out[k++] = v;
  }
  // sort ascending (k <= 3)
  for (int i = 1; i < k; ++i) {
    int v = out[i];
    int j = i - 1;
    while (j >= 0 && out[j] > v) { out[j + 1] = out[j]; --j; }
    out[j + 1] = v;
  }
  return k;
}

// SELL-32x4 neighbor layout: rows grouped in slices of 32 consecutive rows;
// each slice owns Q quads; entry k of row a lives at int word
//   ((a>>5)*Q + (k>>2))*128 + (a&31)*4 + (k&3)
// so one 128-bit load returns 4 consecutive neighbors of one row and a warp's
// load of quad q is 512 contiguous bytes.
__device__ __forceinline__ int64_t sell_word(int a, int k, int Q) {
  return ((int64_t)(a >> 5) * Q + (k >> 2)) * 128 + (a & 31) * 4 + (k & 3);
}

// FP64 -> FP32 by truncation through the bit pattern (integer pipe, no F2F);
// valid for finite values in the FP32 normal range (r^2 of interacting pairs).
__device__ __forceinline__ float d2f_bits(double v) {
  const unsigned hi = (unsigned)__double2hiint(v);
  const unsigned lo = (unsigned)__double2loint(v);
  const unsigned e = (hi >> 20) & 0x7FFu;
  const unsigned f = (hi & 0x80000000u) | ((e - 896u) << 23) | ((hi & 0xFFFFFu) << 3) | (lo >> 29);
  return __uint_as_float(f);
}

// FP32 -> FP64 exactly through the bit pattern (normal numbers and zero).
__device__ __forceinline__ double f2d_bits(float v) {
  const unsigned b = __float_as_uint(v);
  const unsigned mag = b & 0x7FFFFFFFu;
  const unsigned hi = mag ? ((b & 0x80000000u) | (((mag >> 23) + 896u) << 20) |
                             ((b & 0x7FFFFFu) >> 3))
                          : (b & 0x80000000u);
  const unsigned lo = b << 29;
  return __hiloint2double((int)hi, (int)lo);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace pc
