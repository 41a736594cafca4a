// Tile-staged MD hot path: Verlet build into 16-bit slot lists and the LJ
// force kernel that resolves those slots in shared memory.
//
// Why: with one thread per particle the 75 neighbour gathers of a warp hit
// ~24 distinct 32-B sectors per load instruction and saturate the L1 data
// pipe (profiles/r01: 80 % of peak, 270 us per 1M-atom force pass).  A tile
// (one column segment of kTileZ cells, pc_tile.cuh) stages the FP64
// positions of its 27-cell neighbourhood once per step into shared memory
// (planar x/y/z, 8-B words), and its rows store 2-byte slots into that
// staging area instead of 4-byte particle indices: the index stream from HBM
// halves and the gathers become LDS.64.
//
// Exactness is unchanged: the build's pair test is the reference's FP64
// predicate (FP32 prefilter with the rigorous band of pc_nbr_build_sell),
// and the force kernel's cutoff test is exact FP64 inside a band around rc^2
// decided in FP32 elsewhere.  The LJ magnitude is FP32 (F2F conversions run
// at full rate on B200, measured), accumulation FP64 (exact antisymmetry).
#include "pc_tile.cuh"

namespace pc {

constexpr int kTileThreads = 32 * kTileZ;  // build: one warp per home cell
constexpr int kForceTileThreads = 96;   // force: ~78 home rows per tile (kTileZ = 4)

struct TileBuildParams {
  double cutoff2;
  float lo2, hi2;
  int Q;            // quads (4 slots) per row
  int max_stage;    // staged particles capacity
};

struct TileForceParams {
  double cutoff2, overlap2;
  float lo2f, hi2f;    // FP32 band around cutoff^2 for the exact decision
  float sig2, eps24, eps2;
  double guard;        // min image only within this distance of a global face
  int Q;
  int max_stage;
};

// home rows per tile -> 32-row slices -> slice offsets (scan done on host side)
__global__ void tile_slices_kernel(const int* __restrict__ cell_start, pc_grid g, int ntiles,
                                   int* __restrict__ slices) {
  int tile = blockIdx.x * blockDim.x + threadIdx.x;
  if (tile >= ntiles) return;
  int cx, cy, z0, z1;
  tile_coords(tile, g, cx, cy, z0, z1);
  const int base = (cx * g.nc[1] + cy) * g.nc[2];
  const int nh = cell_start[base + z1] - cell_start[base + z0];
  slices[tile] = (nh + 31) >> 5;
}

// staged slot -> (column, cell) by binary search over the cumulative offsets
__device__ __forceinline__ void slot_cell(const TileTable& t, int s, int& c, int& k) {
  int lo = 0, hi = kTileCols * kTileCells - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    const int cm = mid / kTileCells, km = mid - cm * kTileCells;
    if (t.off[cm][km] <= s) lo = mid; else hi = mid - 1;
  }
  c = lo / kTileCells;
  k = lo - c * kTileCells;
}

__global__ void __launch_bounds__(kTileThreads)
tile_build_kernel(const double* __restrict__ pos, const double* __restrict__ posb,
                  const int* __restrict__ cell_start, pc_grid g, pc_box b, pc_box e,
                  TileBuildParams p, const int* __restrict__ slice0, int* __restrict__ count,
                  uint16_t* __restrict__ list, int* __restrict__ flag) {
  extern __shared__ float4 stage[];
  __shared__ TileTable t;
  tile_table(blockIdx.x, g, b, cell_start, t);
  if (t.total + 1 > p.max_stage) {       // +1: the dummy padding slot
    if (threadIdx.x == 0) {
      atomicOr(flag, kFlagStage);
      atomicMax(flag + 1, t.total + 1);  // capacity the caller must provide
    }
    return;
  }
  int cx, cy, z0, z1;
  tile_coords(blockIdx.x, g, cx, cy, z0, z1);
  const double ox = g.low[0] + (cx + 0.5) * g.width[0];
  const double oy = g.low[1] + (cy + 0.5) * g.width[1];
  const double oz = g.low[2] + 0.5 * (z0 + z1) * g.width[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // stage: warp per cell, lanes over its (contiguous) particles
  for (int e = warp; e < kTileCols * kTileCells; e += kTileThreads / 32) {
    const int c = e / kTileCells, k = e - c * kTileCells;
    const int m = t.off[c][k + 1] - t.off[c][k];
    const int src = t.src[c][k], dst = t.off[c][k];
    const double sx = t.shift[c][k][0], sy = t.shift[c][k][1], sz = t.shift[c][k][2];
    for (int q = lane; q < m; q += 32) {
      const double4 r = ld_pos4(posb + 4 * (int64_t)(src + q));
      float4 v;
      v.x = (float)(r.x + sx - ox);
      v.y = (float)(r.y + sy - oy);
      v.z = (float)(r.z + sz - oz);
      v.w = __int_as_float(src + q);
      stage[dst + q] = v;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  const int Q = p.Q;
  const int64_t tile_base = (int64_t)slice0[blockIdx.x] * Q * 128;
  for (int k = warp + 1; k <= t.nzh; k += kTileThreads / 32) {
    const int hs = t.off[4][k];
    const int hn = t.off[4][k + 1] - hs;
    for (int h = 0; h < hn; ++h) {
      const float4 me = stage[hs + h];
      const int a = __float_as_int(me.w);
      const int u = a - t.home_first;                      // row within the tile
      uint16_t* row = list + tile_base + (int64_t)(u >> 5) * Q * 128 + (u & 31) * 4;
      int cnt = 0;
      for (int c = 0; c < kTileCols; ++c) {
        const int s0 = t.off[c][k - 1], s1 = t.off[c][k + 2];
        for (int s = s0 + lane; s - lane < s1; s += 32) {
          bool hit = false;
          if (s < s1) {
            const float4 q = stage[s];
            const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
            const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            const int j = __float_as_int(q.w);
            if (r2 < p.hi2 && j != a) {
              if (r2 < p.lo2) {
                hit = true;
              } else {
                const double4 pa = ld_pos4(pos + 4 * (int64_t)a);
                const double4 pj = ld_pos4(pos + 4 * (int64_t)j);
                const double ex = min_image(__dsub_rn(pj.x, pa.x), e.length[0], e.mi_thresh[0]);
                const double ey = min_image(__dsub_rn(pj.y, pa.y), e.length[1], e.mi_thresh[1]);
                const double ez = min_image(__dsub_rn(pj.z, pa.z), e.length[2], e.mi_thresh[2]);
                hit = r2_exact(ex, ey, ez) < p.cutoff2;
              }
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, hit);
          if (hit) {
            const int kk = cnt + __popc(m & lt);
            if (kk < 4 * Q) row[(kk >> 2) * 128 + (kk & 3)] = (uint16_t)s;
          }
          cnt += __popc(m);
        }
      }
      // pad the open quad with the dummy slot t.total (a NaN row in the force
      // kernel's staging area: never interacts)
      const int kp = cnt + lane;
      if (lane < 4 && (kp & 3) && (kp >> 2) == (cnt >> 2) && kp < 4 * Q)
        row[(kp >> 2) * 128 + (kp & 3)] = (uint16_t)t.total;
      if (lane == 0) {
        count[a] = cnt;
        if (cnt > 4 * Q) atomicOr(flag, kFlagOverflow);
      }
    }
  }
}

// ---- TMA / mbarrier helpers ----------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, UBLKCP); completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// One candidate slot: FP64 displacement from the staged pos4 row (LDS.128 +
// LDS.64), minimum image on near-face axes, the reference's exact FP64 r^2
// and cutoff test, FP32 LJ magnitude, FP64 accumulation.
template <bool MI>
__device__ __forceinline__ void tile_pair(const double4* __restrict__ st, int s, double xi,
                                          double yi, double zi, bool nx, bool ny, bool nz,
                                          const pc_box& gb, const TileForceParams& p,
                                          double& fx, double& fy, double& fz, double& pe,
                                          bool& overlap) {
  const double2 xy = *reinterpret_cast<const double2*>(st + s);
  const double zz = reinterpret_cast<const double*>(st + s)[2];
  double dx = __dsub_rn(xy.x, xi);
  double dy = __dsub_rn(xy.y, yi);
  double dz = __dsub_rn(zz, zi);
  if (MI) {
    if (nx) { const double a = fabs(dx); if (a >= gb.mi_thresh[0]) dx = copysign(__dsub_rn(a, gb.length[0]), -dx); }
    if (ny) { const double a = fabs(dy); if (a >= gb.mi_thresh[1]) dy = copysign(__dsub_rn(a, gb.length[1]), -dy); }
    if (nz) { const double a = fabs(dz); if (a >= gb.mi_thresh[2]) dz = copysign(__dsub_rn(a, gb.length[2]), -dz); }
  }
  const double r2 = r2_exact(dx, dy, dz);
  if (r2 < p.cutoff2) {
    overlap |= r2 < p.overlap2;
    const float inv = rcp_approx((float)r2);
    const float sr2 = p.sig2 * inv;
    const float sr6 = sr2 * sr2 * sr2;
    const double fm = (double)(sr6 * (2.f * sr6 - 1.f) * inv);
    fx = fma(-fm, dx, fx);
    fy = fma(-fm, dy, fy);
    fz = fma(-fm, dz, fz);
    pe += (double)(sr6 * (sr6 - 1.f));
  }
}

template <bool MI>
__device__ __forceinline__ void tile_row(const double4* st, const ushort4* __restrict__ row,
                                         int mq, double xi, double yi, double zi, bool nx,
                                         bool ny, bool nz, const pc_box& gb,
                                         const TileForceParams& p, double& fx, double& fy,
                                         double& fz, double& pe, bool& overlap) {
  ushort4 nxt = make_ushort4(0, 0, 0, 0);
  if (mq > 0) nxt = __ldg(row);
  for (int q = 0; q < mq; ++q) {
    const ushort4 cur = nxt;
    if (q + 1 < mq) nxt = __ldg(row + (int64_t)(q + 1) * 32);
    tile_pair<MI>(st, cur.x, xi, yi, zi, nx, ny, nz, gb, p, fx, fy, fz, pe, overlap);
    tile_pair<MI>(st, cur.y, xi, yi, zi, nx, ny, nz, gb, p, fx, fy, fz, pe, overlap);
    tile_pair<MI>(st, cur.z, xi, yi, zi, nx, ny, nz, gb, p, fx, fy, fz, pe, overlap);
    tile_pair<MI>(st, cur.w, xi, yi, zi, nx, ny, nz, gb, p, fx, fy, fz, pe, overlap);
  }
}

// One CTA per tile.  Thread 0 stages the tile's neighbourhood with TMA bulk
// copies of contiguous pos4 runs (one per z-run of each stencil column) into
// shared memory, completing on an mbarrier; slot t.total is set to NaN (the
// build pads rows with it).  Then one thread per home row sweeps its slot list.
__global__ void __launch_bounds__(kForceTileThreads)
tile_force_kernel(const double* __restrict__ pos, const int* __restrict__ cell_start,
                  pc_grid g, pc_box b, pc_box gb, TileForceParams p,
                  const int* __restrict__ slice0, const int* __restrict__ count,
                  const uint16_t* __restrict__ list, double* __restrict__ f3, int64_t fs,
                  double* __restrict__ v, int64_t vs, double dtm, double mass,
                  double* __restrict__ partial, int* __restrict__ flag) {
  extern __shared__ __align__(128) double4 st[];
  __shared__ TileTable t;
  __shared__ __align__(8) uint64_t bar;
  tile_table(blockIdx.x, g, b, cell_start, t);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double ke = 0.0, pet = 0.0, px = 0.0, py = 0.0, pz = 0.0;
  if (t.total + 1 > p.max_stage) {
    if (threadIdx.x == 0) atomicOr(flag, kFlagStage);
  } else {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (uint32_t)t.total * 32u);
      for (int c = 0; c < kTileCols; ++c) {
        int k = 0;
        while (k < kTileCells) {
          const int src = t.src[c][k];
          int end = src + (t.off[c][k + 1] - t.off[c][k]);
          const int dst = t.off[c][k];
          int k2 = k + 1;
          while (k2 < kTileCells && t.src[c][k2] == end) {   // contiguous in memory
            end += t.off[c][k2 + 1] - t.off[c][k2];
            ++k2;
          }
          if (end > src)
            bulk_g2s(st + dst, pos + 4 * (int64_t)src, (uint32_t)(end - src) * 32u, &bar);
          k = k2;
        }
      }
      st[t.total] = make_double4(__longlong_as_double(0x7ff8000000000000ll),
                                 __longlong_as_double(0x7ff8000000000000ll),
                                 __longlong_as_double(0x7ff8000000000000ll), 0.0);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    const int Q = p.Q;
    const int64_t tile_base = (int64_t)slice0[blockIdx.x] * Q * 32;       // in ushort4
    const int hs0 = t.off[4][1];
    bool overlap = false;
    for (int u = threadIdx.x; u < t.nhome; u += blockDim.x) {
      const int a = t.home_first + u;
      const double4 me = st[hs0 + u];
      const double xi = me.x, yi = me.y, zi = me.z;
      const int m = count[a];
      const bool nx = gb.periodic[0] && (xi - gb.low[0] < p.guard || gb.high[0] - xi <= p.guard);
      const bool ny = gb.periodic[1] && (yi - gb.low[1] < p.guard || gb.high[1] - yi <= p.guard);
      const bool nz = gb.periodic[2] && (zi - gb.low[2] < p.guard || gb.high[2] - zi <= p.guard);
      const ushort4* row = reinterpret_cast<const ushort4*>(list) + tile_base +
                           (int64_t)(u >> 5) * Q * 32 + (u & 31);
      double fx = 0.0, fy = 0.0, fz = 0.0, pe = 0.0;
      const int mq = (m + 3) >> 2;
      if (__any_sync(__activemask(), nx || ny || nz))
        tile_row<true>(st, row, mq, xi, yi, zi, nx, ny, nz, gb, p, fx, fy, fz, pe, overlap);
      else
        tile_row<false>(st, row, mq, xi, yi, zi, nx, ny, nz, gb, p, fx, fy, fz, pe, overlap);
      fx *= (double)p.eps24;
      fy *= (double)p.eps24;
      fz *= (double)p.eps24;
      f3[a] = fx;
      f3[fs + a] = fy;
      f3[2 * fs + a] = fz;
      pet += pe * (double)p.eps2;
      if (v) {
        const double vx = __dadd_rn(v[a], __dmul_rn(dtm, fx));
        const double vy = __dadd_rn(v[vs + a], __dmul_rn(dtm, fy));
        const double vz = __dadd_rn(v[2 * vs + a], __dmul_rn(dtm, fz));
        v[a] = vx;
        v[vs + a] = vy;
        v[2 * vs + a] = vz;
        ke += __dmul_rn(0.5 * mass, r2_exact(vx, vy, vz));
        px += mass * vx;
        py += mass * vy;
        pz += mass * vz;
      }
    }
    if (overlap) atomicOr(flag, kFlagOverlap);
  }
  if (partial) {
    ke = warp_sum(ke);
    pet = warp_sum(pet);
    px = warp_sum(px);
    py = warp_sum(py);
    pz = warp_sum(pz);
    if (lane == 0) {
      double* o = partial + ((int64_t)blockIdx.x * (kForceTileThreads / 32) + warp) * 5;
      o[0] = ke; o[1] = pet; o[2] = px; o[3] = py; o[4] = pz;
    }
  }
}

static double band_margin(const pc_grid& g, double cutoff2) {
  const double U = fmax(fmax(1.5 * g.width[0], 1.5 * g.width[1]), (kTileZ / 2.0 + 1.0) * g.width[2]);
  const double rc = sqrt(cutoff2);
  const double e23 = ldexp(1.0, -23), e24 = ldexp(1.0, -24);
  const double err = 2.0 * sqrt(3.0) * rc * (e23 * U + e24 * rc) + 3.0 * e24 * cutoff2;
  return 8.0 * err + 1e-12 * cutoff2;
}

static int g_build_smem = 0, g_force_smem = 0;

}  // namespace pc

using namespace pc;

extern "C" {

int32_t pc_tile_count(const pc_grid* grid) {
  return grid->nc[0] * grid->nc[1] * ((grid->nc[2] + kTileZ - 1) / kTileZ);
}

int pc_tile_slices(const int32_t* d_cell_start, const pc_grid* grid, int32_t* d_slices,
                   void* stream) {
  const int nt = pc_tile_count(grid);
  tile_slices_kernel<<<(nt + 255) / 256, 256, 0, as_stream(stream)>>>(d_cell_start, *grid, nt,
                                                                      d_slices);
  return check_launch("pc_tile_slices");
}

int pc_tile_build(const double* d_pos, const double* d_posb, const int32_t* d_cell_start,
                  const pc_grid* grid, const pc_box* box_local, const pc_box* box_exact,
                  double cutoff2, int32_t width, int32_t max_stage, const int32_t* d_slice0,
                  int32_t* d_count, uint16_t* d_list, int32_t* d_flag, void* stream) {
  if (width % 4 || width <= 0 || max_stage > 65535) {
    set_error("pc_tile_build: width must be a positive multiple of 4, max_stage <= 65535");
    return PC_ERR_VALUE;
  }
  for (int a = 0; a < 3; ++a)
    if (box_local->periodic[a] && grid->nc[a] < 3) {
      set_error("pc_tile_build: periodic axis with fewer than 3 cells");
      return PC_ERR_VALUE;
    }
  TileBuildParams p;
  const double margin = band_margin(*grid, cutoff2);
  p.cutoff2 = cutoff2;
  p.lo2 = nextafterf((float)(cutoff2 - margin), -INFINITY);
  p.hi2 = nextafterf((float)(cutoff2 + margin), INFINITY);
  p.Q = width / 4;
  p.max_stage = max_stage;
  const int smem = max_stage * (int)sizeof(float4);
  if (smem > g_build_smem) {
    cudaFuncSetAttribute(tile_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    g_build_smem = smem;
  }
  const int nt = pc_tile_count(grid);
  tile_build_kernel<<<nt, kTileThreads, smem, as_stream(stream)>>>(
      d_pos, d_posb ? d_posb : d_pos, d_cell_start, *grid, *box_local,
      box_exact ? *box_exact : *box_local, p, d_slice0, d_count, d_list, d_flag);
  return check_launch("pc_tile_build");
}

int32_t pc_tile_force_partials(const pc_grid* grid) {
  return pc_tile_count(grid) * (kForceTileThreads / 32);
}

int pc_tile_force(const double* d_pos, const int32_t* d_cell_start,
                  const pc_grid* grid, const pc_box* box_local, const pc_box* box_global,
                  const pc_lj* lj, double mi_guard, int32_t width, int32_t max_stage,
                  const int32_t* d_slice0, const int32_t* d_count, const uint16_t* d_list,
                  double* d_f3, int64_t f_stride, double* d_v, int64_t v_stride, double dtm,
                  double mass, double* d_partial, int32_t* d_flag, void* stream) {
  TileForceParams p;
  p.cutoff2 = lj->cutoff2;
  p.overlap2 = lj->overlap2;
  // FP32 r^2 from FP32-rounded FP64 displacements: relative error < 4 ulp
  p.lo2f = nextafterf((float)(lj->cutoff2 * (1.0 - 1e-5)), -INFINITY);
  p.hi2f = nextafterf((float)(lj->cutoff2 * (1.0 + 1e-5)), INFINITY);
  p.sig2 = (float)(lj->sigma * lj->sigma);
  p.eps24 = (float)(24.0 * lj->epsilon);
  p.eps2 = (float)(2.0 * lj->epsilon);
  p.guard = mi_guard;
  p.Q = width / 4;
  p.max_stage = max_stage;
  const int smem = max_stage * (int)sizeof(double4);
  if (smem > g_force_smem) {
    cudaFuncSetAttribute(tile_force_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    g_force_smem = smem;
  }
  const int nt = pc_tile_count(grid);
  tile_force_kernel<<<nt, kForceTileThreads, smem, as_stream(stream)>>>(
      d_pos, d_cell_start, *grid, *box_local, *box_global, p, d_slice0,
      d_count, d_list, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial, d_flag);
  return check_launch("pc_tile_force");
}

}  // extern "C"
