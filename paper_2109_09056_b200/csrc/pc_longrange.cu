// Ewald real-space pass (sm_100a): the erfc-screened Coulomb pair sum of
// ref longrange.py:47-72 over a half Verlet list -- the only consumer of
// build_verlet besides the MD driver (longrange.spme, longrange.py:142-146).
//
// One thread per (i, j) pair (any pair list: the half list's CSR expanded, or
// caller-given arrays), FP64 throughout: displacement and exact minimum image
// as the reference (`dx - L*round(dx/L)`, pc::min_image), r^2 in numpy's
// einsum order, the strict r^2 < r_cut^2 selection, r = sqrt(r^2), and the
// reference's expression order for the energy and the radial magnitude.
// erfc/exp are CUDA's double-precision functions (a few ulp, not scipy's
// bits): parity is ~1e-15 relative per pair, 1e-12 on sums (tested).  Both
// sides accumulate with FP64 atomics; the energy goes to per-block partials.
#include "pc_common.cuh"

namespace pc {

constexpr int kEwaldThreads = 256;

__global__ void __launch_bounds__(kEwaldThreads)
ewald_real_pairs_kernel(const double* __restrict__ x, const double* __restrict__ q,
                        const int* __restrict__ pi, const int* __restrict__ pj, int64_t npairs,
                        pc_box b, double alpha, double rc2, double* __restrict__ f,
                        double* __restrict__ epart, int* __restrict__ flag) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  if (k < npairs) {
    const int i = pi[k], j = pj[k];
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      d[a] = __dsub_rn(x[3 * (int64_t)j + a], x[3 * (int64_t)i + a]);
      if (b.periodic[a]) d[a] = min_image(d[a], b.length[a], b.mi_thresh[a]);
    }
    const double r2 = r2_exact(d[0], d[1], d[2]);
    if (r2 < rc2) {
      const double r = __dsqrt_rn(r2);
      if (r < 1e-10) atomicOr(flag, kFlagOverlap);
      const double qq = __dmul_rn(q[i], q[j]);
      const double ar = __dmul_rn(alpha, r);
      const double er = erfc(ar);
      e = __ddiv_rn(__dmul_rn(qq, er), r);                       // qq * erfc / r
      // qq * (erfc/r2 + 2*alpha/sqrt(pi) * exp(-(alpha r)^2) / r)
      const double c = __ddiv_rn(__dmul_rn(2.0, alpha), 1.7724538509055159);
      const double g = __ddiv_rn(__dmul_rn(c, exp(-__dmul_rn(ar, ar))), r);
      const double mag = __dmul_rn(qq, __dadd_rn(__ddiv_rn(er, r2), g));
      const double s = __ddiv_rn(mag, r);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double fv = __dmul_rn(s, d[a]);
        atomicAdd(f + 3 * (int64_t)j + a, fv);
        atomicAdd(f + 3 * (int64_t)i + a, -fv);
      }
    }
  }
  // block energy partial (fixed tree order)
  __shared__ double red[kEwaldThreads / 32];
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kEwaldThreads / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) epart[blockIdx.x] = v;
  }
}

// pair i of every CSR entry: pi[k] = i for k in [off[i], off[i+1])
__global__ void csr_pairs_kernel(const int64_t* __restrict__ off, int n, int* __restrict__ pi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t k = off[i]; k < off[i + 1]; ++k) pi[k] = i;
}

}  // namespace pc

extern "C" {


using namespace pc;

int pc_csr_pairs(const int64_t* d_offsets, int32_t n, int32_t* d_pi, void* stream) {
  if (n <= 0) return PC_OK;
  csr_pairs_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(d_offsets, n, d_pi);
  return check_launch("pc_csr_pairs");
}

int64_t pc_ewald_real_blocks(int64_t npairs) {
  return npairs > 0 ? (npairs + kEwaldThreads - 1) / kEwaldThreads : 0;
}

int pc_ewald_real_pairs(const double* d_x, const double* d_q, const int32_t* d_pi,
                        const int32_t* d_pj, int64_t npairs, const pc_box* box, double alpha,
                        double r_cut, double* d_f, double* d_epart, int32_t* d_flag,
                        void* stream) {
  if (!(alpha > 0.0) || !(r_cut > 0.0)) {
    set_error("pc_ewald_real_pairs: alpha and r_cut must be positive");
    return PC_ERR_VALUE;
  }
  if (npairs <= 0) return PC_OK;
  const int64_t blocks = pc_ewald_real_blocks(npairs);
  ewald_real_pairs_kernel<<<(unsigned)blocks, kEwaldThreads, 0, as_stream(stream)>>>(
      d_x, d_q, d_pi, d_pj, npairs, *box, alpha, r_cut * r_cut, d_f, d_epart,
      d_flag);
  return check_launch("pc_ewald_real_pairs");
}

}  // extern "C"
