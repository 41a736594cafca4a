// Lennard-Jones force over a Verlet list (ref md.py:89-126).
//
// Thread per row.  Each candidate j is gathered as one 256-bit pos4 load; the
// displacement, minimum image and the exact-cutoff re-filter run in FP64 with
// the reference's rounding order, so the set of interacting pairs is the
// reference's set bit for bit.  The LJ magnitude (rcp, sr6, fmag) is FP32;
// the force is accumulated in FP64 as f += fmag*dx on the FP64 displacement,
// so pair forces stay exactly antisymmetric and total momentum is conserved
// to FP64 rounding (ref test: |P| < 1e-9).  Energies are booked on the
// smaller tag (md.py:123-125) in FP32 per row and reduced in FP64.
// The final half kick v += dtm*f (md.py:251-257) and the KE/PE/momentum
// block partials are fused into the epilogue.
#include "pc_common.cuh"

namespace pc {

constexpr int kForceThreads = 256;

struct LJConst {
  double cutoff2, overlap2;
  float sig2, eps4, eps2, eps24;
  double sig2d, eps2d, eps24d;
};

__device__ __forceinline__ void block_partials(double v0, double v1, double v2, double v3,
                                               double v4, double* __restrict__ out) {
  __shared__ double red[kForceThreads / 32][5];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v0 = warp_sum(v0);
  v1 = warp_sum(v1);
  v2 = warp_sum(v2);
  v3 = warp_sum(v3);
  v4 = warp_sum(v4);
  if (lane == 0) {
    red[wid][0] = v0; red[wid][1] = v1; red[wid][2] = v2; red[wid][3] = v3; red[wid][4] = v4;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double s = 0.0;
    for (int w = 0; w < kForceThreads / 32; ++w) s += red[w][threadIdx.x];
    out[blockIdx.x * 5 + threadIdx.x] = s;
  }
}

template <bool ELL>
__global__ void __launch_bounds__(kForceThreads)
lj_force_kernel(const double* __restrict__ pos, int n_rows, const int* __restrict__ count,
                const int64_t* __restrict__ offsets, const int* __restrict__ index,
                int64_t ell_stride, pc_box b, LJConst c, double* __restrict__ f3,
                int64_t f_stride, double* __restrict__ f64, double* __restrict__ pe,
                double* __restrict__ v, int64_t v_stride, double dtm, double mass,
                double* __restrict__ partial, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n_rows;
  double fx = 0.0, fy = 0.0, fz = 0.0;
  float ei = 0.f;
  bool overlap = false;
  if (live) {
    const double4 pi = ld_pos4(pos + 4 * (int64_t)i);
    const int64_t ti = tag_of(pi.w);
    const int m = count[i];
    const int* __restrict__ row = ELL ? index + i : index + offsets[i];
    const int64_t step = ELL ? ell_stride : 1;
#pragma unroll 4
    for (int k = 0; k < m; ++k) {
      const int j = __ldg(row + (int64_t)k * step);
      const double4 pj = ld_pos4(pos + 4 * (int64_t)j);
      const double dx = min_image(__dsub_rn(pj.x, pi.x), b.length[0], b.mi_thresh[0]);
      const double dy = min_image(__dsub_rn(pj.y, pi.y), b.length[1], b.mi_thresh[1]);
      const double dz = min_image(__dsub_rn(pj.z, pi.z), b.length[2], b.mi_thresh[2]);
      const double r2 = r2_exact(dx, dy, dz);
      if (r2 < c.cutoff2) {
        overlap |= (r2 < c.overlap2);
        const float inv = __frcp_rn((float)r2);
        const float sr2 = c.sig2 * inv;
        const float sr6 = sr2 * sr2 * sr2;
        const double fmag = (double)(c.eps24 * sr6 * (2.f * sr6 - 1.f) * inv);
        fx = fma(-fmag, dx, fx);
        fy = fma(-fmag, dy, fy);
        fz = fma(-fmag, dz, fz);
        if (tag_of(pj.w) > ti) ei += c.eps4 * sr6 * (sr6 - 1.f);
      }
    }
    if (overlap) atomicOr(flag, kFlagOverlap);
    if (f3) {
      f3[i] = fx;
      f3[f_stride + i] = fy;
      f3[2 * f_stride + i] = fz;
    }
    if (f64) {
      f64[3 * (int64_t)i + 0] = fx;
      f64[3 * (int64_t)i + 1] = fy;
      f64[3 * (int64_t)i + 2] = fz;
    }
    if (pe) pe[i] = (double)ei;
  }
  if (partial == nullptr && v == nullptr) return;
  double ke = 0.0, px = 0.0, py = 0.0, pz = 0.0;
  if (live && v) {
    // numpy: v[:o] += dtm * f[:o]  -> t = dtm*f (rounded), v = v + t (rounded)
    double vx = __dadd_rn(v[i], __dmul_rn(dtm, fx));
    double vy = __dadd_rn(v[v_stride + i], __dmul_rn(dtm, fy));
    double vz = __dadd_rn(v[2 * v_stride + i], __dmul_rn(dtm, fz));
    v[i] = vx;
    v[v_stride + i] = vy;
    v[2 * v_stride + i] = vz;
    ke = __dmul_rn(0.5 * mass, r2_exact(vx, vy, vz));
    px = mass * vx;
    py = mass * vy;
    pz = mass * vz;
  }
  if (partial) block_partials(ke, live ? (double)ei : 0.0, px, py, pz, partial);
}

// Half list (Newton's third law): each unordered pair once, f_j -= F through
// FP64 atomics.  Energies summed per warp into one FP64 accumulator.
__global__ void __launch_bounds__(kForceThreads)
lj_force_half_kernel(const double* __restrict__ pos, int n_rows, const int* __restrict__ count,
                     const int* __restrict__ index, int64_t ell_stride, pc_box b, LJConst c,
                     double* __restrict__ f3, int64_t f_stride, double* __restrict__ pe_total,
                     int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double fx = 0.0, fy = 0.0, fz = 0.0;
  float ei = 0.f;
  if (i < n_rows) {
    const double4 pi = ld_pos4(pos + 4 * (int64_t)i);
    const int m = count[i];
    bool overlap = false;
#pragma unroll 2
    for (int k = 0; k < m; ++k) {
      const int j = __ldg(index + (int64_t)k * ell_stride + i);
      const double4 pj = ld_pos4(pos + 4 * (int64_t)j);
      const double dx = min_image(__dsub_rn(pj.x, pi.x), b.length[0], b.mi_thresh[0]);
      const double dy = min_image(__dsub_rn(pj.y, pi.y), b.length[1], b.mi_thresh[1]);
      const double dz = min_image(__dsub_rn(pj.z, pi.z), b.length[2], b.mi_thresh[2]);
      const double r2 = r2_exact(dx, dy, dz);
      if (r2 < c.cutoff2) {
        overlap |= (r2 < c.overlap2);
        const float inv = __frcp_rn((float)r2);
        const float sr2 = c.sig2 * inv;
        const float sr6 = sr2 * sr2 * sr2;
        const double fmag = (double)(c.eps24 * sr6 * (2.f * sr6 - 1.f) * inv);
        const double gx = fmag * dx, gy = fmag * dy, gz = fmag * dz;
        fx -= gx;
        fy -= gy;
        fz -= gz;
        atomicAdd(f3 + j, gx);
        atomicAdd(f3 + f_stride + j, gy);
        atomicAdd(f3 + 2 * f_stride + j, gz);
        ei += c.eps4 * sr6 * (sr6 - 1.f);
      }
    }
    if (overlap) atomicOr(flag, kFlagOverlap);
    atomicAdd(f3 + i, fx);
    atomicAdd(f3 + f_stride + i, fy);
    atomicAdd(f3 + 2 * f_stride + i, fz);
  }
  if (pe_total) {
    double e = warp_sum((double)ei);
    if ((threadIdx.x & 31) == 0) atomicAdd(pe_total, e);
  }
}

// ---- MD hot path: SELL-32x4 list ------------------------------------------
// One pair: FP64 displacement (minimum image only where the row particle is
// near a periodic face, see pc_lj_force_sell), exact FP64 cutoff test, FP64
// LJ magnitude and accumulation; energy booked half on each side of the pair.
//

// The pair magnitude is evaluated in FP64 from an approximate reciprocal
// (MUFU.RCP64H, ~2^-22) refined by one Newton step (~2^-44): no FP32<->FP64
// conversions, ~11 DFMA-pipe ops, error far below the 1e-5 force tolerance.
// Force/energy prefactors (24 eps, 2 eps) are applied once per row.
template <bool MI>
__device__ __forceinline__ void sell_pair(const double4& pj, const double4& pi, bool nx, bool ny,
                                          bool nz, const pc_box& b, const LJConst& c, double& fx,
                                          double& fy, double& fz, double& pe, bool& overlap) {
  double dx = __dsub_rn(pj.x, pi.x);
  double dy = __dsub_rn(pj.y, pi.y);
  double dz = __dsub_rn(pj.z, pi.z);
  if (MI) {
    if (nx) dx = min_image_wrapped(dx, b.length[0], b.mi_thresh[0]);
    if (ny) dy = min_image_wrapped(dy, b.length[1], b.mi_thresh[1]);
    if (nz) dz = min_image_wrapped(dz, b.length[2], b.mi_thresh[2]);
  }
  const double r2 = r2_exact(dx, dy, dz);
  if (r2 < c.cutoff2) {
    overlap |= (r2 < c.overlap2);
    double inv;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(r2));
    inv = fma(inv, fma(-r2, inv, 1.0), inv);
    const double sr2 = c.sig2d * inv;
    const double sr6 = sr2 * sr2 * sr2;
    const double fm = fma(2.0 * sr6, sr6, -sr6) * inv;      // (2 sr12 - sr6) / r2
    fx = fma(-fm, dx, fx);
    fy = fma(-fm, dy, fy);
    fz = fma(-fm, dz, fz);
    pe = fma(sr6, sr6, pe - sr6);                            // sr12 - sr6
  }
}

// Gather of one candidate: pos4 (one 256-bit load) or planar x/y/z arrays
// (three 64-bit loads; 24 B instead of 32 B per candidate and 8-B items, so
// a warp's 32 scattered requests touch fewer L1 lines and wavefronts).
template <bool PLANAR>
__device__ __forceinline__ double4 gather(const double* __restrict__ pos,
                                          const double* __restrict__ pl, int64_t ps, int j) {
  if (PLANAR) {
    double4 r;
    r.x = __ldg(pl + j);
    r.y = __ldg(pl + ps + j);
    r.z = __ldg(pl + 2 * ps + j);
    r.w = 0.0;
    return r;
  }
  return ld_pos4(pos + 4 * (int64_t)j);
}

// Software-pipelined row sweep over the planar positions: while quad q is
// computed, the positions of quad q+1 and the indices of quad q+2 are in
// flight (lanes past their own row length gather the NaN dummy row).
template <bool MI>
__device__ __forceinline__ void sell_row_pipe(const double* __restrict__ pl, int64_t ps,
                                              int dummy, const int4* __restrict__ row, int mq,
                                              int qmax, const double4& pi, bool nx, bool ny,
                                              bool nz, const pc_box& b, const LJConst& c,
                                              double& fx, double& fy, double& fz, double& pe,
                                              bool& overlap) {
  const int4 d4 = make_int4(dummy, dummy, dummy, dummy);
  int4 i1 = mq > 0 ? __ldg(row) : d4;
  int4 i2 = mq > 1 ? __ldg(row + 32) : d4;
  double4 c0 = gather<true>(nullptr, pl, ps, i1.x), c1 = gather<true>(nullptr, pl, ps, i1.y);
  double4 c2 = gather<true>(nullptr, pl, ps, i1.z), c3 = gather<true>(nullptr, pl, ps, i1.w);
  for (int q = 0; q < qmax; ++q) {
    const int4 i3 = q + 2 < mq ? __ldg(row + (int64_t)(q + 2) * 32) : d4;
    const double4 n0 = gather<true>(nullptr, pl, ps, i2.x);
    const double4 n1 = gather<true>(nullptr, pl, ps, i2.y);
    const double4 n2 = gather<true>(nullptr, pl, ps, i2.z);
    const double4 n3 = gather<true>(nullptr, pl, ps, i2.w);
    if (q < mq) {
      sell_pair<MI>(c0, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
      sell_pair<MI>(c1, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
      sell_pair<MI>(c2, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
      sell_pair<MI>(c3, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
    }
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    i2 = i3;
  }
}

template <bool MI, bool PLANAR>
__device__ __forceinline__ void sell_row(const double* __restrict__ pos,
                                         const double* __restrict__ pl, int64_t ps,
                                         const int4* __restrict__ row, int mq, int qmax,
                                         const double4& pi, bool nx, bool ny, bool nz,
                                         const pc_box& b, const LJConst& c, double& fx,
                                         double& fy, double& fz, double& pe, bool& overlap) {
  if (PLANAR) {
    sell_row_pipe<MI>(pl, ps, (int)(ps - 1), row, mq, qmax, pi, nx, ny, nz, b, c, fx, fy, fz,
                      pe, overlap);
    return;
  }
  int4 nxt = make_int4(0, 0, 0, 0);
  if (mq > 0) nxt = __ldg(row);
  for (int q = 0; q < qmax; ++q) {
    const int4 cur = nxt;
    if (q + 1 < mq) nxt = __ldg(row + (int64_t)(q + 1) * 32);
    if (q < mq) {
      const double4 p0 = gather<PLANAR>(pos, pl, ps, cur.x);
      const double4 p1 = gather<PLANAR>(pos, pl, ps, cur.y);
      const double4 p2 = gather<PLANAR>(pos, pl, ps, cur.z);
      const double4 p3 = gather<PLANAR>(pos, pl, ps, cur.w);
      sell_pair<MI>(p0, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
      sell_pair<MI>(p1, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
      sell_pair<MI>(p2, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
      sell_pair<MI>(p3, pi, nx, ny, nz, b, c, fx, fy, fz, pe, overlap);
    }
  }
}

template <bool PLANAR, bool ATOM = false>
__global__ void __launch_bounds__(kForceThreads, PLANAR ? 2 : 3)
lj_force_sell_kernel(const double* __restrict__ pos, const double* __restrict__ pl, int64_t ps,
                     int n_rows, const int* __restrict__ count,
                     const int4* __restrict__ nbr, int Q, pc_box b, LJConst c, double guard,
                     double* __restrict__ f3, int64_t f_stride, double* __restrict__ v,
                     int64_t v_stride, double dtm, double mass, double* __restrict__ partial,
                     int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool live = i < n_rows;
  double4 pi = make_double4(0.0, 0.0, 0.0, 0.0);
  int m = 0;
  if (live) {
    pi = ld_pos4(pos + 4 * (int64_t)i);
    m = count[i];
  }
  const int mq = (m + 3) >> 2;
  const int qmax = __reduce_max_sync(0xffffffffu, mq);
  const bool nx = b.periodic[0] && (pi.x - b.low[0] < guard || b.high[0] - pi.x <= guard);
  const bool ny = b.periodic[1] && (pi.y - b.low[1] < guard || b.high[1] - pi.y <= guard);
  const bool nz = b.periodic[2] && (pi.z - b.low[2] < guard || b.high[2] - pi.z <= guard);
  const int4* row = nbr + (int64_t)(i >> 5) * Q * 32 + lane;
  double fx = 0.0, fy = 0.0, fz = 0.0, pe = 0.0;
  bool overlap = false;
  if (__any_sync(0xffffffffu, live && (nx || ny || nz)))
    sell_row<true, PLANAR>(pos, pl, ps, row, mq, qmax, pi, nx, ny, nz, b, c, fx, fy, fz, pe,
                           overlap);
  else
    sell_row<false, PLANAR>(pos, pl, ps, row, mq, qmax, pi, nx, ny, nz, b, c, fx, fy, fz, pe,
                            overlap);
  if (overlap) atomicOr(flag, kFlagOverlap);
  fx *= c.eps24d;
  fy *= c.eps24d;
  fz *= c.eps24d;
  pe *= c.eps2d;
  double ke = 0.0, px = 0.0, py = 0.0, pz = 0.0;
  if (live) {
    f3[i] = fx;
    f3[f_stride + i] = fy;
    f3[2 * f_stride + i] = fz;
    if (v) {
      const double vx = __dadd_rn(v[i], __dmul_rn(dtm, fx));
      const double vy = __dadd_rn(v[v_stride + i], __dmul_rn(dtm, fy));
      const double vz = __dadd_rn(v[2 * v_stride + i], __dmul_rn(dtm, fz));
      v[i] = vx;
      v[v_stride + i] = vy;
      v[2 * v_stride + i] = vz;
      ke = __dmul_rn(0.5 * mass, r2_exact(vx, vy, vz));
      px = mass * vx;
      py = mass * vy;
      pz = mass * vz;
    }
  }
  if (ATOM) {
    // deterministic mode: one (KE, PE, px, py, pz) row per atom, reduced by
    // the caller in global-id order
    if (live) {
      double* o = partial + (int64_t)i * 5;
      o[0] = ke; o[1] = pe; o[2] = px; o[3] = py; o[4] = pz;
    }
  } else if (partial) {
    // per-warp partials: no block barrier, so fast warps retire early
    ke = warp_sum(ke);
    pe = warp_sum(pe);
    px = warp_sum(px);
    py = warp_sum(py);
    pz = warp_sum(pz);
    if (lane == 0) {
      double* o = partial + (int64_t)(i >> 5) * 5;
      o[0] = ke; o[1] = pe; o[2] = px; o[3] = py; o[4] = pz;
    }
  }
}

// Half list over the SELL layout (Newton's third law, ref md.py has no half
// path: the reference force for a half list is the full-list force).  Each
// stored pair is evaluated once; the row accumulates +F in registers and the
// neighbour receives -F through FP64 atomics (RED.E.ADD.F64), so f must be
// zeroed before and the final kick runs as a separate pc_kick.  PE partials
// book each pair's full energy once.
__global__ void __launch_bounds__(kForceThreads, 3)
lj_force_sell_half_kernel(const double* __restrict__ pos, int n_rows,
                          const int* __restrict__ count, const int4* __restrict__ nbr, int Q,
                          pc_box b, LJConst c, double guard, double* __restrict__ f3,
                          int64_t fs, double* __restrict__ partial, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool live = i < n_rows;
  double4 pi = make_double4(0.0, 0.0, 0.0, 0.0);
  int m = 0;
  if (live) {
    pi = ld_pos4(pos + 4 * (int64_t)i);
    m = count[i];
  }
  const bool nx = b.periodic[0] && (pi.x - b.low[0] < guard || b.high[0] - pi.x <= guard);
  const bool ny = b.periodic[1] && (pi.y - b.low[1] < guard || b.high[1] - pi.y <= guard);
  const bool nz = b.periodic[2] && (pi.z - b.low[2] < guard || b.high[2] - pi.z <= guard);
  const int4* row = nbr + (int64_t)(i >> 5) * Q * 32 + lane;
  double fx = 0.0, fy = 0.0, fz = 0.0, pe = 0.0;
  bool overlap = false;
  const int mq = (m + 3) >> 2;
  int4 nxt = make_int4(0, 0, 0, 0);
  if (mq > 0) nxt = __ldg(row);
  for (int q = 0; q < mq; ++q) {
    const int4 cur = nxt;
    if (q + 1 < mq) nxt = __ldg(row + (int64_t)(q + 1) * 32);
    const int js[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = js[u];
      const double4 pj = ld_pos4(pos + 4 * (int64_t)j);
      double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
      if (nx) dx = min_image_wrapped(dx, b.length[0], b.mi_thresh[0]);
      if (ny) dy = min_image_wrapped(dy, b.length[1], b.mi_thresh[1]);
      if (nz) dz = min_image_wrapped(dz, b.length[2], b.mi_thresh[2]);
      const double r2 = r2_exact(dx, dy, dz);
      if (r2 < c.cutoff2) {
        overlap |= (r2 < c.overlap2);
        double inv;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(r2));
        inv = fma(inv, fma(-r2, inv, 1.0), inv);
        const double sr2 = c.sig2d * inv;
        const double sr6 = sr2 * sr2 * sr2;
        const double fm = c.eps24d * fma(2.0 * sr6, sr6, -sr6) * inv;
        const double gx = fm * dx, gy = fm * dy, gz = fm * dz;
        fx -= gx;
        fy -= gy;
        fz -= gz;
        atomicAdd(f3 + j, gx);
        atomicAdd(f3 + fs + j, gy);
        atomicAdd(f3 + 2 * fs + j, gz);
        pe = fma(sr6, sr6, pe - sr6);
      }
    }
  }
  if (overlap) atomicOr(flag, kFlagOverlap);
  if (live) {
    atomicAdd(f3 + i, fx);
    atomicAdd(f3 + fs + i, fy);
    atomicAdd(f3 + 2 * fs + i, fz);
  }
  if (partial) {
    pe = warp_sum(pe * 2.0 * c.eps2d);                       // 4 eps (sr12 - sr6)
    if (lane == 0) {
      double* o = partial + (int64_t)(i >> 5) * 5;
      o[0] = 0.0; o[1] = pe; o[2] = 0.0; o[3] = 0.0; o[4] = 0.0;
    }
  }
}

static LJConst make_const(const pc_lj* lj) {
  LJConst c;
  c.cutoff2 = lj->cutoff2;
  c.overlap2 = lj->overlap2;
  c.sig2 = (float)(lj->sigma * lj->sigma);
  c.eps4 = (float)(4.0 * lj->epsilon);
  c.eps2 = (float)(2.0 * lj->epsilon);
  c.eps24 = (float)(24.0 * lj->epsilon);
  c.sig2d = lj->sigma * lj->sigma;
  c.eps2d = 2.0 * lj->epsilon;
  c.eps24d = 24.0 * lj->epsilon;
  return c;
}

}  // namespace pc

using namespace pc;

extern "C" {

int32_t pc_lj_force_blocks(int32_t n_rows) {
  return n_rows <= 0 ? 1 : (n_rows + kForceThreads - 1) / kForceThreads;
}

int32_t pc_lj_force_sell_partials(int32_t n_rows) {
  return pc_lj_force_blocks(n_rows) * (kForceThreads / 32);
}

int pc_lj_force(const double* d_pos, int32_t n_rows, const int32_t* d_count,
                const int64_t* d_offsets, const int32_t* d_index, int64_t ell_stride,
                const pc_box* box, const pc_lj* lj, double* d_f3, int64_t f_stride,
                double* d_f64, double* d_pe, double* d_v, int64_t v_stride, double dtm,
                double mass, double* d_partial, int32_t* d_flag, void* stream) {
  if (n_rows < 0) {
    set_error("pc_lj_force: negative row count");
    return PC_ERR_VALUE;
  }
  if (ell_stride <= 0 && d_offsets == nullptr && n_rows > 0) {
    set_error("pc_lj_force: CSR layout needs offsets");
    return PC_ERR_VALUE;
  }
  LJConst c = make_const(lj);
  unsigned blocks = (unsigned)pc_lj_force_blocks(n_rows);
  cudaStream_t s = as_stream(stream);
  if (ell_stride > 0)
    lj_force_kernel<true><<<blocks, kForceThreads, 0, s>>>(
        d_pos, n_rows, d_count, d_offsets, d_index, ell_stride, *box, c, d_f3, f_stride, d_f64,
        d_pe, d_v, v_stride, dtm, mass, d_partial, d_flag);
  else
    lj_force_kernel<false><<<blocks, kForceThreads, 0, s>>>(
        d_pos, n_rows, d_count, d_offsets, d_index, ell_stride, *box, c, d_f3, f_stride, d_f64,
        d_pe, d_v, v_stride, dtm, mass, d_partial, d_flag);
  return check_launch("pc_lj_force");
}

int pc_lj_force_sell(const double* d_pos, const double* d_planar, int64_t planar_stride,
                     int32_t n_rows, const int32_t* d_count,
                     const int32_t* d_index, int32_t width, const pc_box* box, const pc_lj* lj,
                     double mi_guard, double* d_f3, int64_t f_stride, double* d_v,
                     int64_t v_stride, double dtm, double mass, double* d_partial,
                     int32_t* d_flag, void* stream) {
  if (n_rows < 0 || width % 4) {
    set_error("pc_lj_force_sell: bad rows/width");
    return PC_ERR_VALUE;
  }
  LJConst c = make_const(lj);
  unsigned blocks = (unsigned)pc_lj_force_blocks(n_rows);
  if (d_planar)
    lj_force_sell_kernel<true><<<blocks, kForceThreads, 0, as_stream(stream)>>>(
        d_pos, d_planar, planar_stride, n_rows, d_count, reinterpret_cast<const int4*>(d_index),
        width / 4, *box, c, mi_guard, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial,
        d_flag);
  else
    lj_force_sell_kernel<false><<<blocks, kForceThreads, 0, as_stream(stream)>>>(
        d_pos, d_planar, planar_stride, n_rows, d_count, reinterpret_cast<const int4*>(d_index),
        width / 4, *box, c, mi_guard, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial,
        d_flag);
  return check_launch("pc_lj_force_sell");
}

int pc_lj_force_sell_atoms(const double* d_pos, const double* d_planar, int64_t planar_stride,
                           int32_t n_rows, const int32_t* d_count, const int32_t* d_index,
                           int32_t width, const pc_box* box, const pc_lj* lj, double mi_guard,
                           double* d_f3, int64_t f_stride, double* d_v, int64_t v_stride,
                           double dtm, double mass, double* d_atom, int32_t* d_flag,
                           void* stream) {
  if (n_rows < 0 || width % 4 || !d_atom || !d_planar) {
    set_error("pc_lj_force_sell_atoms: bad rows/width or missing planar/atom arrays");
    return PC_ERR_VALUE;
  }
  LJConst c = make_const(lj);
  unsigned blocks = (unsigned)pc_lj_force_blocks(n_rows);
  lj_force_sell_kernel<true, true><<<blocks, kForceThreads, 0, as_stream(stream)>>>(
      d_pos, d_planar, planar_stride, n_rows, d_count, reinterpret_cast<const int4*>(d_index),
      width / 4, *box, c, mi_guard, d_f3, f_stride, d_v, v_stride, dtm, mass, d_atom, d_flag);
  return check_launch("pc_lj_force_sell_atoms");
}

int pc_lj_force_sell_half(const double* d_pos, int32_t n_rows, const int32_t* d_count,
                          const int32_t* d_index, int32_t width, const pc_box* box,
                          const pc_lj* lj, double mi_guard, double* d_f3, int64_t f_stride,
                          double* d_partial, int32_t* d_flag, void* stream) {
  if (n_rows < 0 || width % 4) {
    set_error("pc_lj_force_sell_half: bad rows/width");
    return PC_ERR_VALUE;
  }
  LJConst c = make_const(lj);
  unsigned blocks = (unsigned)pc_lj_force_blocks(n_rows);
  lj_force_sell_half_kernel<<<blocks, kForceThreads, 0, as_stream(stream)>>>(
      d_pos, n_rows, d_count, reinterpret_cast<const int4*>(d_index), width / 4, *box, c,
      mi_guard, d_f3, f_stride, d_partial, d_flag);
  return check_launch("pc_lj_force_sell_half");
}

int pc_lj_force_half(const double* d_pos, int32_t n_rows, const int32_t* d_count,
                     const int32_t* d_index, int64_t ell_stride, const pc_box* box,
                     const pc_lj* lj, double* d_f3, int64_t f_stride, double* d_pe_total,
                     int32_t* d_flag, void* stream) {
  if (n_rows <= 0) return PC_OK;
  LJConst c = make_const(lj);
  unsigned blocks = (unsigned)pc_lj_force_blocks(n_rows);
  lj_force_half_kernel<<<blocks, kForceThreads, 0, as_stream(stream)>>>(
      d_pos, n_rows, d_count, d_index, ell_stride, *box, c, d_f3, f_stride, d_pe_total, d_flag);
  return check_launch("pc_lj_force_half");
}

}  // extern "C"
