// Tile-staged MD hot path (sm_100a): Verlet build into per-warp "round"
// lists of 16-bit shared-memory slots, and the LJ force kernel that resolves
// those slots against an FP64 neighbourhood staged by the TMA engine.
//
// Why (profiles/r01, profiles/r01b): with one thread per particle gathering
// its neighbours from global memory, a warp's 32 scattered 32-B requests
// touch ~21 distinct 128-B L1 lines per load instruction; the L1 tag/data
// pipe serves about one line per cycle, which alone costs ~180 us of the
// 282 us force pass at 1M atoms.  Here a CTA owns a tile of 2x2 columns x
// kTZ cells of the linked-cell grid; the FP64 x|y|z of its 4x4 x (kTZ+2)
// cell neighbourhood (~1900 particles, ~45 KB) is copied into shared memory
// by cp.async.bulk (one bulk copy per contiguous index run and coordinate,
// completing on an mbarrier), and every candidate becomes three LDS.64.
//
// Tile geometry (tile_setup, shared by the build, the force kernel and the
// host decoder): staged column sc = sxo*4 + syo (sxo, syo in 0..3 map to grid
// columns x0-1+sxo, y0-1+syo, periodic wrap); each staged column contributes
// three "segments" -- the z-cell below the grid (periodic wrap, z0 == 0), the
// in-range cells, the z-cell above the grid (wrap) -- each a contiguous run of
// the cell-sorted particle arrays.  A segment is copied from its even-aligned
// start (16-B TMA alignment), so slot = seg_dst + (index - seg_src).  In the
// force kernel's staging ring a tile's allocation starts with 16 dummy slots
// (1e30 positions, one per LDS.64 bank pair) used as padding, so list
// entries are byte offsets (slot + 16) * 8, dummies i * 8 (kSlotBias).
//
// List layout: home rows of a tile are numbered column by column and grouped
// in row-warps of 32.  Row-warp rw (global numbering rw0[tile] + w) holds
// rounds[rw] rounds; in round r lane l reads slot
//   list16[((rw*Q8 + r/8)*32 + l)*8 + r%8]
// i.e. one 128-bit load gives a lane its next 8 slots and a warp's load is 512
// contiguous bytes.  Every round is a row's neighbour or a dummy.
//
// Exactness: the build decides each candidate with FP32 coordinates relative
// to the tile centre outside a rigorously bounded band around cutoff^2 and
// with the reference's FP64 predicate inside it (same bound as
// pc_nbr_build_sell); the force kernel re-tests r^2 < rc^2 in FP64 with the
// reference's rounding order (pc_common.cuh r2_exact) on raw positions, with
// the exact threshold minimum image on rows near a periodic face.  The LJ
// magnitude is FP32 (r^2 narrowed by integer bit operations: FP64->FP32 F2F
// issues at ~8 lanes/clk/SM on B200, measured, scripts/micro/pipes2.cu),
// the force is accumulated in FP64 as f += fm*dx so pair terms are exactly
// antisymmetric (momentum conserved to FP64 rounding).
#include <stdlib.h>
#include <string.h>

#include "pc_common.cuh"

namespace pc {

constexpr int kBX = 2, kBY = 2, kTZ = 4;
constexpr int kSX = kBX + 2, kSY = kBY + 2, kSZ = kTZ + 2;
constexpr int kSCols = kSX * kSY;
constexpr int kSegs = kSCols * 3;
constexpr int kNDummy = 16;
constexpr uint32_t kSlotBias = 16;   // list byte offset of staged slot s: (s + 16) * 8
#ifndef PC_FORCE_SLEEP
#define PC_FORCE_SLEEP 64
#endif
#ifndef PC_FORCE_WARPS
#define PC_FORCE_WARPS 32
#endif
constexpr int kForceWarps = PC_FORCE_WARPS;
constexpr int kBuildWarps = 10;
constexpr int kHitCap = 112;
// force-kernel staging capacity (slots) and per-coordinate stride in shared
// memory: compile-time so every LDS is [slot*8 + immediate]
constexpr int kStageCap = 2304;

struct TileSetup {
  int seg_src[kSegs];          // even-aligned first index of the copied run
  int seg_len[kSegs];          // copied elements (even, 0 = empty)
  int seg_dst[kSegs];          // first slot
  float seg_shift[kSegs][3];   // periodic image (build prefilter only; exact multiples of L in FP64 below)
  int cell_lo[kSCols][kSZ];    // slot range of each staged cell (build only)
  int cell_hi[kSCols][kSZ];
  int home_start[kBX * kBY];   // first particle of each home column's z-range
  int home_pre[kBX * kBY + 1]; // tile-row offset of each home column
  int home_cell0[kBX * kBY];   // cell_start index of the first home cell of the column
  int S, H, bx, by, bz, z0;
  double ox, oy, oz;           // tile centre (build prefilter origin)
};

struct TileDims {
  int ntx, nty, ntz, ntiles;
};

__host__ __device__ inline TileDims tile_dims(const pc_grid& g) {
  TileDims d;
  d.ntx = (g.nc[0] + kBX - 1) / kBX;
  d.nty = (g.nc[1] + kBY - 1) / kBY;
  d.ntz = (g.nc[2] + kTZ - 1) / kTZ;
  d.ntiles = d.ntx * d.nty * d.ntz;
  return d;
}

// Fill T for `tile`.  All threads call it (contains barriers).  CELLS: also
// the per-cell slot table used by the build.
template <bool CELLS>
__device__ void tile_setup(int tile, const pc_grid& g, const pc_box& b,
                           const int* __restrict__ cs, TileSetup& T) {
  const TileDims d = tile_dims(g);
  const int tz = tile % d.ntz;
  const int t2 = tile / d.ntz;
  const int ty = t2 % d.nty, tx = t2 / d.nty;
  const int x0 = tx * kBX, y0 = ty * kBY, z0 = tz * kTZ;
  const int bx = min(kBX, g.nc[0] - x0), by = min(kBY, g.nc[1] - y0), bz = min(kTZ, g.nc[2] - z0);
  const int nx = g.nc[0], ny = g.nc[1], nz = g.nc[2];
  for (int e = threadIdx.x; e < kSegs; e += blockDim.x) {
    const int col = e / 3, part = e - col * 3;
    const int sxo = col / kSY, syo = col - sxo * kSY;
    int gx = x0 - 1 + sxo, gy = y0 - 1 + syo;
    bool ok = sxo <= bx + 1 && syo <= by + 1;
    float shx = 0.f, shy = 0.f, shz = 0.f;
    if (gx < 0) { if (b.periodic[0]) { gx += nx; shx = -1.f; } else ok = false; }
    if (gx >= nx) { if (b.periodic[0]) { gx -= nx; shx = 1.f; } else ok = false; }
    if (gy < 0) { if (b.periodic[1]) { gy += ny; shy = -1.f; } else ok = false; }
    if (gy >= ny) { if (b.periodic[1]) { gy -= ny; shy = 1.f; } else ok = false; }
    const int zlo = z0 - 1, zhi = z0 + bz;      // staged z-cells, inclusive
    int za = 0, zb = -1;
    if (part == 0) {
      if (zlo < 0 && b.periodic[2]) { za = zb = nz - 1; shz = -1.f; }
    } else if (part == 1) {
      za = max(zlo, 0);
      zb = min(zhi, nz - 1);
    } else {
      if (zhi >= nz && b.periodic[2]) { za = zb = 0; shz = 1.f; }
    }
    int src = 0, len = 0;
    if (ok && zb >= za) {
      const int base = (gx * ny + gy) * nz;
      const int first = cs[base + za], end = cs[base + zb + 1];
      if (end > first) {
        src = first & ~1;
        len = ((end + 1) & ~1) - src;
      }
    }
    T.seg_src[e] = src;
    T.seg_len[e] = len;
    T.seg_shift[e][0] = shx;
    T.seg_shift[e][1] = shy;
    T.seg_shift[e][2] = shz;
  }
  if (threadIdx.x < kBX * kBY) {
    const int c = threadIdx.x, hx = c / kBY, hy = c - hx * kBY;
    int st = 0, cnt = 0, c0 = 0;
    if (hx < bx && hy < by) {
      c0 = ((x0 + hx) * ny + (y0 + hy)) * nz + z0;
      st = cs[c0];
      cnt = cs[c0 + bz] - st;
    }
    T.home_start[c] = st;
    T.home_cell0[c] = c0;
    T.home_pre[c + 1] = cnt;     // scanned below
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int carry = 0;
    for (int base = 0; base < kSegs; base += 32) {
      const int e = base + lane;
      const int v = e < kSegs ? T.seg_len[e] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (e < kSegs) T.seg_dst[e] = carry + inc - v;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      T.S = carry;
      T.home_pre[0] = 0;
      for (int c = 0; c < kBX * kBY; ++c) T.home_pre[c + 1] += T.home_pre[c];
      T.H = T.home_pre[kBX * kBY];
      T.bx = bx;
      T.by = by;
      T.bz = bz;
      T.z0 = z0;
      T.ox = g.low[0] + (x0 + 0.5 * bx) * g.width[0];
      T.oy = g.low[1] + (y0 + 0.5 * by) * g.width[1];
      T.oz = g.low[2] + (z0 + 0.5 * bz) * g.width[2];
    }
  }
  if (CELLS) {
    __syncthreads();
    for (int e = threadIdx.x; e < kSCols * kSZ; e += blockDim.x) {
      const int col = e / kSZ, k = e - col * kSZ;
      int lo = 0, hi = 0;
      if (k <= bz + 1) {
        const int part = (k == 0 && z0 == 0) ? 0 : ((k == bz + 1 && z0 + bz == nz) ? 2 : 1);
        const int seg = col * 3 + part;
        if (T.seg_len[seg] > 0) {
          const int sxo = col / kSY, syo = col - sxo * kSY;
          const int gx = (x0 - 1 + sxo + nx) % nx, gy = (y0 - 1 + syo + ny) % ny;
          const int gz = (z0 - 1 + k + nz) % nz;
          const int cell = (gx * ny + gy) * nz + gz;
          lo = T.seg_dst[seg] + (cs[cell] - T.seg_src[seg]);
          hi = lo + (cs[cell + 1] - cs[cell]);
        }
      }
      T.cell_lo[col][k] = lo;
      T.cell_hi[col][k] = hi;
    }
  }
  __syncthreads();
}

// tile row u -> particle index (and home column)
__device__ __forceinline__ int home_row(const TileSetup& T, int u, int& c) {
  c = 0;
#pragma unroll
  for (int k = 1; k < kBX * kBY; ++k) c += (u >= T.home_pre[k]) ? 1 : 0;
  return T.home_start[c] + (u - T.home_pre[c]);
}

// per tile: row-warps = ceil(home rows / 32)
__global__ void tile_rows_kernel(const int* __restrict__ cs, pc_grid g, int* __restrict__ rw) {
  const TileDims d = tile_dims(g);
  const int tile = blockIdx.x * blockDim.x + threadIdx.x;
  if (tile >= d.ntiles) return;
  const int tz = tile % d.ntz, t2 = tile / d.ntz;
  const int ty = t2 % d.nty, tx = t2 / d.nty;
  const int x0 = tx * kBX, y0 = ty * kBY, z0 = tz * kTZ;
  const int bx = min(kBX, g.nc[0] - x0), by = min(kBY, g.nc[1] - y0), bz = min(kTZ, g.nc[2] - z0);
  int h = 0;
  for (int hx = 0; hx < bx; ++hx)
    for (int hy = 0; hy < by; ++hy) {
      const int c0 = ((x0 + hx) * g.nc[1] + (y0 + hy)) * g.nc[2] + z0;
      h += cs[c0 + bz] - cs[c0];
    }
  rw[tile] = (h + 31) >> 5;
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

// streaming 128-bit load of list words (read once per step: no L1 allocation)
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---- per-tile plan (written by the build, read by the force kernel) --------
// ints: [0] non-empty segments m, [1] staged slots S, [2] row-warps, [3] rw0,
// then m x (src, len, dst).
constexpr int kPlanInts = 4 + 3 * kSegs;

// ---- build ------------------------------------------------------------------
struct TileBuildParams {
  double cutoff2;
  float lo2, hi2;      // FP32 band: r2f < lo2 -> hit, r2f >= hi2 -> miss, else exact FP64
  int Q8;              // list capacity per row-warp, in 8-round groups
  int max_stage;       // staged slots capacity (multiple of 16); dummies follow
  int64_t ps;          // planar stride
};

__device__ __forceinline__ bool exact_pair_pl(const double* __restrict__ pl, int64_t ps, int a,
                                              int j, const pc_box& b, double cutoff2) {
  const double dx = min_image(__dsub_rn(pl[j], pl[a]), b.length[0], b.mi_thresh[0]);
  const double dy = min_image(__dsub_rn(pl[ps + j], pl[ps + a]), b.length[1], b.mi_thresh[1]);
  const double dz =
      min_image(__dsub_rn(pl[2 * ps + j], pl[2 * ps + a]), b.length[2], b.mi_thresh[2]);
  return r2_exact(dx, dy, dz) < cutoff2;
}

// Rounds of a row-warp: entry k of every row in round k (the build's
// ascending sweep order; pc_tile_order reorders them), padded with dummies.
// Encoding (kSlotBias): staged slot s -> byte offset (s + 16) * 8 from the
// tile's allocation start; i * 8 (i < 16) is one of the tile's 16 dummy slots
// (1e30 positions in front of the staged slots, one per LDS.64 bank pair).
__device__ __forceinline__ int plain_rows(const uint16_t* __restrict__ hits, int cnt, int lane,
                                          uint4* __restrict__ out, int cap_rounds) {
  const int R = __reduce_max_sync(0xffffffffu, cnt);
  const uint32_t d = (uint32_t)((lane & 15) * 8);
  for (int r8 = 0; r8 < R && r8 + 8 <= cap_rounds; r8 += 8) {
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int r = r8 + 2 * h;
      const uint32_t lo = r < cnt ? ((uint32_t)hits[r * 32] + kSlotBias) * 8u : d;
      const uint32_t hi = r + 1 < cnt ? ((uint32_t)hits[(r + 1) * 32] + kSlotBias) * 8u : d;
      w[h] = lo | (hi << 16);
    }
    out[(r8 >> 3) * 32] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  return R;
}

// particle index of staged slot s
__device__ __forceinline__ int slot_index(const TileSetup& T, int s) {
  int e = 0;
  while (e < kSegs - 1 && !(T.seg_len[e] > 0 && s >= T.seg_dst[e] && s < T.seg_dst[e] + T.seg_len[e]))
    ++e;
  return T.seg_src[e] + (s - T.seg_dst[e]);
}

// Build.  Particles are z-sorted inside every cell (pc_cell_zsort at the
// rebuild), so each staged column -- cells in z order, each cell z-sorted --
// is one z-sorted run of slots, and the home rows of a column are z-sorted
// too.  The FP32 staged copy (x, y, z relative to the tile centre, periodic
// image applied) sits in slot order.  One warp handles one row at a time:
// lanes 0..8 bound its 9 stencil columns to the z-window |dz| < h, h^2 =
// hi2 - (lateral distance to the column)^2 (binary search in the stencil's
// first and last cell), then all 32 lanes sweep the windows' candidates in
// parallel and compact the hits with a ballot into the row's hit list
// (ascending slots).  Candidates outside the FP32 band decide in FP32;
// inside it the reference's FP64 predicate decides (exact).

__global__ void __launch_bounds__(kBuildWarps * 32, 2)
tile_build_kernel(const double* __restrict__ pl, const int* __restrict__ cs, pc_grid g, pc_box b,
                  TileBuildParams p, const int* __restrict__ rw0, int* __restrict__ plan,
                  int* __restrict__ rowidx, int* __restrict__ rounds, uint4* __restrict__ list,
                  int* __restrict__ flag, const double* __restrict__ bpl, pc_box e,
                  const int* __restrict__ skip) {
  extern __shared__ float4 cz[];                 // staged FP32 copy | per-warp hit rows
  __shared__ TileSetup T;
  uint16_t* hits_all = reinterpret_cast<uint16_t*>(cz + p.max_stage);
  tile_setup<true>(blockIdx.x, g, b, cs, T);
  if (T.S > p.max_stage) {
    // flag it; leave an empty plan so that a speculatively launched force
    // pass stays in bounds (the caller discards it and falls back)
    if (threadIdx.x == 0) {
      atomicOr(flag, kFlagStage);
      atomicMax(flag + 1, T.S);
      int* pg = plan + (int64_t)blockIdx.x * kPlanInts;
      pg[0] = 0;
      pg[1] = 0;
      pg[2] = 0;
      pg[3] = rw0[blockIdx.x];
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nrw = (T.H + 31) >> 5;
  const int bz = T.bz;
  if (warp == 0) {                       // compacted plan of this tile
    int* pg = plan + (int64_t)blockIdx.x * kPlanInts;
    int base = 0;
    for (int e0 = 0; e0 < kSegs; e0 += 32) {
      const int e = e0 + lane;
      const bool ne = e < kSegs && T.seg_len[e] > 0;
      const unsigned bal = __ballot_sync(0xffffffffu, ne);
      if (ne) {
        const int k = base + __popc(bal & ((1u << lane) - 1u));
        pg[4 + 3 * k] = T.seg_src[e];
        pg[5 + 3 * k] = T.seg_len[e];
        pg[6 + 3 * k] = T.seg_dst[e];
      }
      base += __popc(bal);
    }
    if (lane == 0) {
      pg[0] = base;
      pg[1] = T.S;
      pg[2] = nrw;
      pg[3] = rw0[blockIdx.x];
    }
  }
  const int64_t ps = p.ps;
  for (int e = 0; e < kSegs; ++e) {      // stage: slot order
    const int len = T.seg_len[e];
    if (len == 0) continue;
    const int src = T.seg_src[e], dst = T.seg_dst[e];
    const double sx = (double)T.seg_shift[e][0] * b.length[0] - T.ox;
    const double sy = (double)T.seg_shift[e][1] * b.length[1] - T.oy;
    const double sz = (double)T.seg_shift[e][2] * b.length[2] - T.oz;
    for (int t = threadIdx.x; t < len; t += blockDim.x) {
      const int j = src + t;
      float4 q;
      q.x = (float)(bpl[j] + sx);
      q.y = (float)(bpl[ps + j] + sy);
      q.z = (float)(bpl[2 * ps + j] + sz);
      q.w = 0.f;
      cz[dst + t] = q;
    }
  }
  __syncthreads();

  uint16_t* hits = hits_all + warp * kHitCap * 32 + lane;     // [k][lane]
  for (int w = warp; w < nrw; w += kBuildWarps) {
    const int u = w * 32 + lane;
    const bool act = u < T.H;
    int cnt = 0, a = -1, pos = -1, nband = 0;
    if (act) {
      int ho = 0;                                // hit-list word offset (k * 32)
      const int hlast = (kHitCap - 1) * 32;
      float mx = 0.f;
      int c = 0;
#pragma unroll
      for (int q = 1; q < kBX * kBY; ++q) c += (u >= T.home_pre[q]) ? 1 : 0;
      const int hx = c / kBY, hy = c - hx * kBY;
      const int hcol = (hx + 1) * kSY + (hy + 1);
      pos = T.cell_lo[hcol][1] + (u - T.home_pre[c]);
      int k = 1;
      for (int kk = 2; kk <= bz; ++kk) k += (pos >= T.cell_lo[hcol][kk]) ? 1 : 0;
      a = slot_index(T, pos);
      const float4 me = cz[pos];
      // rows flagged in `skip` (ghosts of a decomposed domain) keep an empty
      // list: zero force, and they are never a row of the force pass's pairs
      const bool scan = !(skip && skip[a]);
      // every stencil column is swept over the same z-window |dz| < h,
      // h = sqrt(hi2) (lateral pruning would only shorten some lanes'
      // windows; the warp runs the longest anyway)
      const float h = sqrtf(p.hi2) * 1.0001f + 1e-4f;
      const float zlo = me.z - h, zhi = me.z + h;
#pragma unroll 1
      for (int cc = 0; cc < (scan ? 9 : 0); ++cc) {
        const int col = (hx + cc / 3) * kSY + (hy + cc % 3);
        // [lo, e1) in cell k-1 (suffix), cell k, [b3, hi) in cell k+1 (prefix)
        int lo = T.cell_lo[col][k - 1], h1 = T.cell_hi[col][k - 1];
        while (lo < h1) {
          const int mid = (lo + h1) >> 1;
          if (cz[mid].z < zlo) lo = mid + 1; else h1 = mid;
        }
        const int e1 = T.cell_hi[col][k - 1];
        const int b2 = T.cell_lo[col][k], e2 = T.cell_hi[col][k];
        const int b3 = T.cell_lo[col][k + 1];
        int hi = b3, h3 = T.cell_hi[col][k + 1];
        while (hi < h3) {
          const int mid = (hi + h3) >> 1;
          if (cz[mid].z <= zhi) hi = mid + 1; else h3 = mid;
        }
        // the three pieces are one run unless a periodic z wrap splits them;
        // the row's own slot splits its own column's run
        const bool one = (e1 == b2) && (e2 == b3);
        for (int piece = 0; piece < (one ? 2 : 4); ++piece) {
          int s0, s1;
          if (one) {
            s0 = piece == 0 ? lo : max(lo, pos + 1);
            s1 = piece == 0 ? min(hi, pos) : hi;
          } else {
            s0 = piece == 0 ? lo : (piece == 1 ? b2 : (piece == 2 ? max(b2, pos + 1) : b3));
            s1 = piece == 0 ? e1 : (piece == 1 ? min(e2, pos) : (piece == 2 ? e2 : hi));
          }
          // four candidates per step: independent tests, then stores at the
          // running hit offset (a non-hit's store is overwritten by the next
          // hit); one short dependency chain per step instead of per candidate
          int i = s0;
          for (; i + 4 <= s1; i += 4) {
            bool h[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float4 q = cz[i + u];
              const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
              const float rr = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
              h[u] = rr < p.hi2;
              mx = fmaxf(mx, h[u] ? rr : 0.f);
            }
            const int o1 = ho + (h[0] ? 32 : 0);
            const int o2 = o1 + (h[1] ? 32 : 0);
            const int o3 = o2 + (h[2] ? 32 : 0);
            hits[ho] = (uint16_t)i;
            hits[min(o1, hlast)] = (uint16_t)(i + 1);
            hits[min(o2, hlast)] = (uint16_t)(i + 2);
            hits[min(o3, hlast)] = (uint16_t)(i + 3);
            ho = min(o3 + (h[3] ? 32 : 0), hlast);
          }
          for (; i < s1; ++i) {
            const float4 q = cz[i];
            const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
            const float rr = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            hits[ho] = (uint16_t)i;
            const bool hit = rr < p.hi2;
            mx = fmaxf(mx, hit ? rr : 0.f);
            ho = min(ho + (hit ? 32 : 0), hlast);
          }
        }
      }
      cnt = ho >> 5;
      if (cnt >= kHitCap - 1) cnt = kHitCap;        // (possible) overflow
      nband = mx >= p.lo2 ? 1 : 0;
    }
    // hits inside the FP32 band: the reference's FP64 predicate decides (rare)
    if (__any_sync(0xffffffffu, nband > 0)) {
      if (nband > 0 && cnt < kHitCap) {
        const float4 me = cz[pos];
        int m = 0;
        for (int t = 0; t < cnt; ++t) {
          const int v = hits[t * 32];
          const float4 q = cz[v];
          const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
          const float rr = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
          const bool keep =
              rr < p.lo2 || exact_pair_pl(pl, ps, a, slot_index(T, v), e, p.cutoff2);
          if (keep) hits[m++ * 32] = (uint16_t)v;
        }
        cnt = m;
      }
    }
    const int rw = rw0[blockIdx.x] + w;
    rowidx[(int64_t)rw * 32 + lane] = a;
    const int cmax = __reduce_max_sync(0xffffffffu, cnt);
    if (cmax >= kHitCap) {        // (the unconditional hit store clobbers entry kHitCap-1)
      if (lane == 0) {
        atomicOr(flag, kFlagOverflow);
        atomicMax(flag + 2, 1 << 20);
        rounds[rw] = 0;           // keep a speculative force pass in bounds
      }
      __syncwarp();
      continue;
    }
    __syncwarp();
    const int cap = 8 * p.Q8;
    uint4* lout = list + (int64_t)rw * p.Q8 * 32 + lane;
    const int R = plain_rows(hits, cnt, lane, lout, cap);
    if (lane == 0) {
      rounds[rw] = ((R + 7) & ~7) > cap ? 0 : R;
      if (((R + 7) & ~7) > cap) {
        atomicOr(flag, kFlagOverflow);
        atomicMax(flag + 2, R);
      }
    }
    __syncwarp();
  }
}

__global__ void pos_from_planar_kernel(const double* __restrict__ pl, int64_t ps, int n,
                                       double* __restrict__ pos4) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pos4[4 * (int64_t)i] = pl[i];
  pos4[4 * (int64_t)i + 1] = pl[ps + i];
  pos4[4 * (int64_t)i + 2] = pl[2 * ps + i];
}

// Per-cell z-sort of a cell-sorted order: cell c = order[cs[c] .. cs[c+1]);
// out = the same particles ranked by (z, position in the cell).  Warp per
// cell; z read from the unsorted pos4 rows.
__global__ void __launch_bounds__(256)
cell_zsort_kernel(const double* __restrict__ pos4, const int* __restrict__ cs, int ncells,
                  const int* __restrict__ order, int* __restrict__ out) {
  const int cell = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (cell >= ncells) return;
  const int s0 = cs[cell], m = cs[cell + 1] - s0;
  for (int t0 = 0; t0 < m; t0 += 32) {
    const int t = t0 + lane;
    const int src = t < m ? order[s0 + t] : 0;
    const double z = t < m ? pos4[4 * (int64_t)src + 2] : 0.0;
    int rk = 0;
    for (int u0 = 0; u0 < m; u0 += 32) {
      const int uu = u0 + lane;
      const double zu_l = uu < m ? pos4[4 * (int64_t)order[s0 + uu] + 2] : 0.0;
      const int lim = min(32, m - u0);
      for (int v = 0; v < lim; ++v) {
        const double zu = __shfl_sync(0xffffffffu, zu_l, v);
        rk += (zu < z || (zu == z && u0 + v < t)) ? 1 : 0;
      }
    }
    if (t < m) out[s0 + rk] = src;
  }
}

// ---- force ------------------------------------------------------------------
// Persistent kernel: one CTA of kForceWarps warps per SM walks its tiles
// (blockIdx.x + k*gridDim.x) through a shared-memory staging RING.  Row-warps
// of all its tiles form one queue (item i -> tile k by the prefix of row-warp
// counts); a warp takes the next item, prefetches the row's list / position /
// index words, waits until tile k is staged and sweeps the rounds.
//
// The ring is three equal planes (x | y | z, kRingSlots doubles each, so a
// slot's y and z are immediate offsets from its x).  Tile k occupies S_k + 16
// contiguous slots -- 16 dummies (1e30) then its staged slots -- allocated in
// tile order, wrapping to the ring start when the tail does not fit, and
// released in tile order once all its row-warps are done.  Sizing exactly
// (instead of fixed 2320-slot buffers) keeps ~4.7 tiles in flight: a tile is
// held from its first row-warp's start to its last one's end, about
// 1 + warps/row-warps-per-tile = 4.2 tiles at 32 warps, and warps waited
// ~15 % of the time with 4 fixed buffers (profiles/r01d).  The warp
// releasing a tile issues the TMA bulk copies of as many next tiles as fit,
// under a shared-memory lock; per-tile mbarriers live in a ring of kRing
// (parity from k).
constexpr int kRing = 8;            // tiles in flight at most (mbarriers, per-tile state)
constexpr int kRingSlots = 9600;    // slots per plane: 3 x 9600 x 8 B = 225 KB

struct TileForceParams {
  double cutoff2, overlap2;
  float sig2;
  double eps24d, eps2d;
  double guard;        // minimum image only within this distance of a periodic face
  int Q8;
  int64_t ps;
};

struct ForceShared {
  uint64_t bar[kRing];
  int base[kRing];           // first slot of tile k's allocation (k % kRing)
  int end_v[kRing];          // virtual end of the allocation (-1: none)
  int done[kRing];           // finished row-warps of tile k
  int fin[kRing];            // tile k finished (all row-warps)
  volatile int ready[kRing]; // k once tile k's copies are issued (k % kRing), else older
  int issued;                // tiles 0..issued-1 have ring space
  int released;              // tiles 0..released-1 released, in order
  int head_v, tail_v;        // virtual ring positions (slots, monotonic)
  int lock;
  int next_item;
  int K;                     // tiles of this CTA
  int items;                 // row-warps of this CTA
};

// FP64 -> FP32 by truncation in two integer instructions (SHF.L.W + IADD):
// the funnel shift moves exponent bits 8..0 and 23 mantissa bits into place,
// +0x40000000 rebiases the 9-bit exponent field modulo 512 (1023 - 127 = 896
// = 384 mod 512, -384 = 128 mod 512).  Exact for positive v with FP32-normal
// magnitude (an interacting pair's r^2); anything else is garbage, which the
// caller replaces by a select.
__device__ __forceinline__ float d2f_fast(double v) {
  const unsigned hi = (unsigned)__double2hiint(v);
  const unsigned lo = (unsigned)__double2loint(v);
  return __uint_as_float(__funnelshift_l(lo, hi, 3) + 0x40000000u);
}

// One round: `off` is the byte offset of the slot in a coordinate array.
template <bool MI, bool UNIT_SIGMA>
__device__ __forceinline__ void tile_pair(const char* __restrict__ st, uint32_t off, double xi,
                                          double yi, double zi, bool nx, bool ny, bool nz,
                                          const pc_box& b, const TileForceParams& p, double& fx,
                                          double& fy, double& fz, float& pe, bool& overlap) {
  const double* q = reinterpret_cast<const double*>(st + off);
  double dx = __dsub_rn(q[0], xi);
  double dy = __dsub_rn(q[kRingSlots], yi);
  double dz = __dsub_rn(q[2 * kRingSlots], zi);
  if (MI) {
    // staged coordinates are wrapped into the box: |d| < L, so the exact
    // threshold form needs no division fallback (dummies: 1e30 stays huge)
    if (nx) dx = min_image_wrapped(dx, b.length[0], b.mi_thresh[0]);
    if (ny) dy = min_image_wrapped(dy, b.length[1], b.mi_thresh[1]);
    if (nz) dz = min_image_wrapped(dz, b.length[2], b.mi_thresh[2]);
  }
  const double r2 = r2_exact(dx, dy, dz);
  const bool inter = r2 < p.cutoff2;
  overlap |= r2 < p.overlap2;
  // branch-free: a non-interacting lane evaluates the pair at r^2 = 1e30
  // (all terms underflow to exactly 0; 0 * dx = 0 for the finite dummies)
  const float r2f = inter ? d2f_fast(r2) : 1e30f;
  const float inv = rcp_approx(r2f);
  const float sr2 = UNIT_SIGMA ? inv : p.sig2 * inv;
  const float sr6 = sr2 * sr2 * sr2;
  const float fm = (sr6 * inv) * fmaf(2.0f, sr6, -1.0f);     // (2 sr12 - sr6) / r2
  pe += fmaf(sr6, sr6, -sr6);                                  // sr12 - sr6
  const double fmd = (double)fm;
  fx = fma(-fmd, dx, fx);
  fy = fma(-fmd, dy, fy);
  fz = fma(-fmd, dz, fz);
}

template <bool MI, bool UNIT_SIGMA>
__device__ __forceinline__ void tile_row(const char* __restrict__ st,
                                         const uint4* __restrict__ lp, uint4 first, int R,
                                         double xi, double yi, double zi, bool nx, bool ny,
                                         bool nz, const pc_box& b, const TileForceParams& p,
                                         double& fx, double& fy, double& fz, float& pe,
                                         bool& overlap) {
  const int G = R >> 3;           // full 8-round groups
  const int tail = R & 7;         // rounds of the open group (padded with dummies: skipped)
  uint4 nxt = first;
  for (int gi = 0; gi < G; ++gi) {
    const uint4 q = nxt;
    if (gi + 1 < G || tail) nxt = ld_stream(lp + (gi + 1) * 32);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      tile_pair<MI, UNIT_SIGMA>(st, w[h] & 0xFFFFu, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz,
                                pe, overlap);
      tile_pair<MI, UNIT_SIGMA>(st, w[h] >> 16, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, pe,
                                overlap);
    }
  }
  // open group: pairs in twos (warp-uniform count)
  for (int j = 0; j < tail; j += 2) {
    const uint32_t w = (j >> 1) == 0 ? nxt.x : ((j >> 1) == 1 ? nxt.y : ((j >> 1) == 2 ? nxt.z : nxt.w));
    tile_pair<MI, UNIT_SIGMA>(st, w & 0xFFFFu, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, pe,
                              overlap);
    if (j + 1 < tail)
      tile_pair<MI, UNIT_SIGMA>(st, w >> 16, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, pe,
                                overlap);
  }
}

// Lane 0, ring lock held: allocate ring space for as many next tiles as fit
// (in tile order); returns the first tile allocated, F.issued is one past the
// last.  `sz` = staged slots per tile (0: no rows, nothing to stage).
__device__ __forceinline__ int ring_alloc(ForceShared& F, const int* __restrict__ sz) {
  const int k0 = F.issued;
  for (;;) {
    // release finished tiles in order first (tiles without rows finish at
    // allocation: a run of them must not fill the window of kRing)
    while (F.released < F.issued && F.fin[F.released & (kRing - 1)]) {
      const int e = F.end_v[F.released & (kRing - 1)];
      if (e >= 0) F.tail_v = e;
      F.released += 1;
    }
    const int k = F.issued;
    if (k >= F.K || k - F.released >= kRing) break;
    const int q = k & (kRing - 1);
    const int S = sz[k];
    if (S > 0) {
      const int A = S + (int)kSlotBias;          // even: segments are even-aligned
      int h = F.head_v;
      const int pos = h % kRingSlots;
      if (pos + A > kRingSlots) h += kRingSlots - pos;      // wrap: skip the ring tail
      if (h + A - F.tail_v > kRingSlots) break;            // no room yet
      F.base[q] = h % kRingSlots;
      F.head_v = h + A;
      F.end_v[q] = h + A;
      F.fin[q] = 0;
    } else {
      F.base[q] = 0;
      F.end_v[q] = -1;
      F.fin[q] = 1;                               // no rows: never waited on
    }
    F.done[q] = 0;
    F.issued = k + 1;
  }
  return k0;
}

// Whole warp: issue the TMA copies of tiles [k0, k1) (space allocated) and
// publish each as ready.
__device__ void ring_stage(ForceShared& F, double* __restrict__ ring, int k0, int k1,
                           const int* __restrict__ plan, const double* __restrict__ pl,
                           int64_t ps, int lane) {
  for (int k = k0; k < k1; ++k) {
    const int q = k & (kRing - 1);
    const int tile = blockIdx.x + k * gridDim.x;
    const int* gp = plan + (int64_t)tile * kPlanInts;
    const bool rows = F.end_v[q] >= 0;
    const int m = rows ? gp[0] : 0, S = rows ? gp[1] : 0;
    if (lane == 0) mbar_expect_tx(&F.bar[q], (uint32_t)S * 24u);   // S = 0: plain arrive
    __syncwarp();
    if (rows) {
      double* st = ring + F.base[q];
      if (lane < kNDummy)
#pragma unroll
        for (int a = 0; a < 3; ++a) st[a * kRingSlots + lane] = 1e30;
      for (int e = lane; e < m; e += 32) {
        const int src = gp[4 + 3 * e], len = gp[5 + 3 * e];
        const int dst = gp[6 + 3 * e] + (int)kSlotBias;
#pragma unroll
        for (int a = 0; a < 3; ++a)
          bulk_g2s(st + a * kRingSlots + dst, pl + a * ps + src, (uint32_t)len * 8u, &F.bar[q]);
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      F.ready[q] = k;
    }
  }
  __syncwarp();
}

// Whole warp: tile k finished -- release finished tiles in order, allocate
// and stage the next ones (copies issued outside the lock).
__device__ void ring_release(ForceShared& F, double* __restrict__ ring, int k,
                             const int* __restrict__ plan, const int* __restrict__ sz,
                             const double* __restrict__ pl, int64_t ps, int lane) {
  int k0 = 0, k1 = 0;
  if (lane == 0) {
    while (atomicCAS(&F.lock, 0, 1) != 0) __nanosleep(32);
    __threadfence_block();
    F.fin[k & (kRing - 1)] = 1;
    k0 = ring_alloc(F, sz);
    k1 = F.issued;
    __threadfence_block();
    atomicExch(&F.lock, 0);
  }
  k0 = __shfl_sync(0xffffffffu, k0, 0);
  k1 = __shfl_sync(0xffffffffu, k1, 0);
  __threadfence_block();
  ring_stage(F, ring, k0, k1, plan, pl, ps, lane);
}

template <bool UNIT_SIGMA>
__global__ void __launch_bounds__(kForceWarps * 32, 1)
tile_force_kernel(const double* __restrict__ pl, TileForceParams p, int ntiles,
                  const int* __restrict__ plan, const int* __restrict__ rowidx,
                  const int* __restrict__ rounds, const uint4* __restrict__ list, pc_box b,
                  double* __restrict__ f3, int64_t fs, double* __restrict__ v, int64_t vs,
                  double dtm, double mass, double* __restrict__ partial, int* __restrict__ flag,
                  double* __restrict__ x_next, double* __restrict__ v_next,
                  double dtm_next, double dt, int* __restrict__ scratch) {
  extern __shared__ double dyn[];
  double* ring = dyn;                                              // x | y | z planes
  __shared__ ForceShared F;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  // item prefix (K + 1) and first row-warp (K) per tile of this CTA: global
  // scratch (L1-resident), so the whole shared memory is staging ring
  const int Kmax = (ntiles + (int)gridDim.x - 1) / (int)gridDim.x;   // same stride for all CTAs
  int* pre = scratch + (int64_t)blockIdx.x * (3 * Kmax + 1);
  int* rwbk = pre + K + 1;
  int* sz = rwbk + K;                                                 // staged slots per tile
  if (warp == 0) {
    // row-warp prefix over this CTA's tiles
    int carry = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int k = k0 + lane;
      const int* gpk = plan + (int64_t)(blockIdx.x + k * gridDim.x) * kPlanInts;
      const int c = k < K ? gpk[2] : 0;
      if (k < K) {
        rwbk[k] = gpk[3];
        sz[k] = c > 0 ? gpk[1] : 0;
      }
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (k < K) pre[k] = carry + inc - c;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      pre[K] = carry;
      F.items = carry;
      F.K = K;
      F.next_item = 0;
      F.issued = 0;
      F.released = 0;
      F.head_v = 0;
      F.tail_v = 0;
      F.lock = 0;
      for (int q = 0; q < kRing; ++q) {
        mbar_init(&F.bar[q], 1);
        F.ready[q] = -1;
      }
    }
    __syncwarp();
    __threadfence_block();
    int k1 = 0;
    if (lane == 0) {                                      // no other warp runs yet
      ring_alloc(F, sz);
      k1 = F.issued;
    }
    k1 = __shfl_sync(0xffffffffu, k1, 0);
    __threadfence_block();
    ring_stage(F, ring, 0, k1, plan, pl, p.ps, lane);
  }
  __threadfence_block();
  __syncthreads();
  const int items = F.items;
  double ake = 0.0, ape = 0.0, apx = 0.0, apy = 0.0, apz = 0.0;   // this lane's rows

  for (;;) {
    int i = 0;
    if (lane == 0) i = atomicAdd(&F.next_item, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= items) break;
    // tile sequence index of item i (pre is ascending; K is small)
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int k = lo;
    const int rw = rwbk[k] + (i - pre[k]);
    // prefetch everything that does not depend on the staged tile
    const int a = rowidx[(int64_t)rw * 32 + lane];
    const int R = rounds[rw];
    const uint4* lp = list + (int64_t)rw * p.Q8 * 32 + lane;
    const uint4 first = R > 0 ? ld_stream(lp) : make_uint4(0u, 0u, 0u, 0u);
    const bool act = a >= 0;
    double xi = 0.0, yi = 0.0, zi = 0.0;
    if (act) {
      xi = pl[a];
      yi = pl[p.ps + a];
      zi = pl[2 * p.ps + a];
    }
    // tile k: wait until its copies are issued (tile order), then complete
    const int q = k & (kRing - 1);
    while (F.ready[q] != k) __nanosleep(PC_FORCE_SLEEP);
    __threadfence_block();
    mbar_wait(&F.bar[q], (uint32_t)((k / kRing) & 1));
    const char* st = reinterpret_cast<const char*>(ring + F.base[q]);

    const bool nx = act && b.periodic[0] && (xi - b.low[0] < p.guard || b.high[0] - xi <= p.guard);
    const bool ny = act && b.periodic[1] && (yi - b.low[1] < p.guard || b.high[1] - yi <= p.guard);
    const bool nz = act && b.periodic[2] && (zi - b.low[2] < p.guard || b.high[2] - zi <= p.guard);
    double fx = 0.0, fy = 0.0, fz = 0.0;
    float pe = 0.f;
    bool overlap = false;
    if (__any_sync(0xffffffffu, nx || ny || nz))
      tile_row<true, UNIT_SIGMA>(st, lp, first, R, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, pe,
                                 overlap);
    else
      tile_row<false, UNIT_SIGMA>(st, lp, first, R, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, pe,
                                  overlap);
    // the tile's last row-warp releases it (in tile order) and refills the ring
    int last = 0;
    if (lane == 0) last = atomicAdd(&F.done[q], 1) + 1 == pre[k + 1] - pre[k];
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) ring_release(F, ring, k, plan, sz, pl, p.ps, lane);
    if (overlap) atomicOr(flag, kFlagOverlap);
    double ke = 0.0, px = 0.0, py = 0.0, pz = 0.0, ped = 0.0;
    if (act) {
      fx *= p.eps24d;
      fy *= p.eps24d;
      fz *= p.eps24d;
      ped = (double)pe * p.eps2d;
      f3[a] = fx;
      f3[fs + a] = fy;
      f3[2 * fs + a] = fz;
      if (v) {
        // numpy: v[:o] += dtm * f[:o]  (ref md.py:251-257), no contraction
        const double vx = __dadd_rn(v[a], __dmul_rn(dtm, fx));
        const double vy = __dadd_rn(v[vs + a], __dmul_rn(dtm, fy));
        const double vz = __dadd_rn(v[2 * vs + a], __dmul_rn(dtm, fz));
        v[a] = vx;
        v[vs + a] = vy;
        v[2 * vs + a] = vz;
        ke = __dmul_rn(0.5 * mass, r2_exact(vx, vy, vz));
        px = mass * vx;
        py = mass * vy;
        pz = mass * vz;
        if (x_next) {
          // next step's integrate block (ref md.py:219-231) fused: it uses
          // this force, so v' = v + dtm f, x' = wrap(x + dt v') are final
          // now; written to the alternate buffers (neighbour tiles still
          // stage x of this step)
          const double ux = __dadd_rn(vx, __dmul_rn(dtm_next, fx));
          const double uy = __dadd_rn(vy, __dmul_rn(dtm_next, fy));
          const double uz = __dadd_rn(vz, __dmul_rn(dtm_next, fz));
          double nx_ = __dadd_rn(xi, __dmul_rn(dt, ux));
          double ny_ = __dadd_rn(yi, __dmul_rn(dt, uy));
          double nz_ = __dadd_rn(zi, __dmul_rn(dt, uz));
          if (b.periodic[0]) nx_ = wrap_axis_near(nx_, b.low[0], b.high[0], b.length[0]);
          if (b.periodic[1]) ny_ = wrap_axis_near(ny_, b.low[1], b.high[1], b.length[1]);
          if (b.periodic[2]) nz_ = wrap_axis_near(nz_, b.low[2], b.high[2], b.length[2]);
          v_next[a] = ux;
          v_next[vs + a] = uy;
          v_next[2 * vs + a] = uz;
          x_next[a] = nx_;
          x_next[p.ps + a] = ny_;
          x_next[2 * p.ps + a] = nz_;
        }
      }
    }
    ake += ke;
    ape += ped;
    apx += px;
    apy += py;
    apz += pz;
  }
  // one (KE, PE, px, py, pz) partial per warp of the grid
  if (partial) {
    ake = warp_sum(ake);
    ape = warp_sum(ape);
    apx = warp_sum(apx);
    apy = warp_sum(apy);
    apz = warp_sum(apz);
    if (lane == 0) {
      double* o = partial + ((int64_t)blockIdx.x * kForceWarps + warp) * 5;
      o[0] = ake; o[1] = ape; o[2] = apx; o[3] = apy; o[4] = apz;
    }
  }
}

// ---- list reorder: residue round-robin rounds (after the build) ------------
// One warp per row-warp.  Reads the plain (ascending) list, reorders every
// lane's row in shared memory -- class-major scatter by bank-pair residue,
// then round-robin emission: in round r lane l prefers residue (l + r) % 16,
// falling back to the next non-empty residue (rotate + ffs over a 16-bit
// mask) -- and writes it back in place.  The 16 lanes of a half-warp then
// prefer 16 distinct residues in every round: 1.6 LDS.64 passes per
// half-warp instead of 2.5 (simulated), force pass -14 % (measured).
constexpr int kOrdWarps = 8;
constexpr int kOrdSmem = kOrdWarps * (kHitCap * 32 * 2 + 16 * 32 * 4);

// RR = false: class-major with the start rotated to the lane's residue (the
// cheaper variant, simulated 1.9 passes per half-warp).  Per-class state
// lives in a per-lane shared table st[c][lane] (conflict-free: bank = lane).
template <bool RR>
__global__ void __launch_bounds__(kOrdWarps * 32, 3)
tile_order_kernel(uint4* __restrict__ list, const int* __restrict__ rounds,
                  const int* __restrict__ rw_total, int Q8) {
  extern __shared__ __align__(16) unsigned char osm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = blockIdx.x * kOrdWarps + warp;
  if (rw >= *rw_total) return;
  uint32_t* st = reinterpret_cast<uint32_t*>(osm) + warp * 16 * 32 + lane;   // [c][lane]
  uint16_t* Bm = reinterpret_cast<uint16_t*>(osm + kOrdWarps * 16 * 32 * 4) +
                 warp * kHitCap * 32 + lane;                                  // [k][lane]
  const int R = rounds[rw];
  if (R <= 0 || R > kHitCap) return;
  uint4* lp = list + (int64_t)rw * Q8 * 32 + lane;
  const uint32_t dmin = kSlotBias * 8u;                 // real entries: v >= dmin
  const int G = (R + 7) >> 3;
#pragma unroll
  for (int c = 0; c < 16; ++c) st[c * 32] = 0u;
  int cnt = 0;                                          // real entries precede padding
  for (int g = 0; g < G; ++g) {                         // per-class counts
    const uint4 q = lp[g * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      if (g * 8 + t < R && v >= dmin) {
        uint32_t* sc = st + ((v >> 3) & 15) * 32;
        *sc += 1u;
        ++cnt;
      }
    }
  }
  // exclusive prefix -> st[c] = start | start << 16 (next | begin); end = next start
  uint32_t run = 0u;
  int s0 = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint32_t n = st[c * 32];
    if (!RR && c == (lane & 15)) s0 = (int)run;
    st[c * 32] = run | ((run + n) << 16);               // next | end
    run += n;
  }
  unsigned ne = 0u;
  for (int g = 0; g < G; ++g) {                         // class-major scatter -> smem
    const uint4 q = lp[g * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      if (g * 8 + t < cnt) {
        const int c = (v >> 3) & 15;
        uint32_t* sc = st + c * 32;
        const uint32_t e = *sc;
        *sc = e + 1u;
        int pos = (int)(e & 0xFFFFu);
        if (RR) ne |= 1u << c;
        else { pos -= s0; if (pos < 0) pos += cnt; }
        Bm[pos * 32] = (uint16_t)v;
      }
    }
  }
  if (RR) {                                             // rewind next to begin
    uint32_t beg = 0u;                                  // begin(c) = end(c - 1)
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint32_t end = st[c * 32] >> 16;
      st[c * 32] = beg | (end << 16);
      beg = end;
    }
  }
  for (int g = 0; g < G; ++g) {                         // emit 8 rounds per uint4
    uint32_t o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int r = g * 8 + t;
      uint32_t v;
      if (r < cnt) {
        int pos = r;
        if (RR) {
          // in round r lane l prefers residue (l + r) % 16, else the next
          // non-empty one
          const int pref = (lane + r) & 15;
          const unsigned rot = ((ne >> pref) | (ne << (16 - pref))) & 0xFFFFu;
          const int c = (pref + __ffs(rot) - 1) & 15;
          uint32_t* sc = st + c * 32;
          const uint32_t e = *sc;
          pos = (int)(e & 0xFFFFu);
          *sc = e + 1u;
          if ((uint32_t)pos + 1u == (e >> 16)) ne &= ~(1u << c);
        }
        v = Bm[pos * 32];
      } else {
        v = (uint32_t)((lane + r) & 15) * 8u;
      }
      o[t >> 1] |= (t & 1) ? (v << 16) : v;
    }
    lp[g * 32] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ---- decode: tile lists -> per-row dense table of particle indices ---------
__global__ void __launch_bounds__(256)
tile_decode_kernel(const int* __restrict__ plan, int Q8, int max_stage,
                   const int* __restrict__ rowidx, const int* __restrict__ rounds,
                   const uint4* __restrict__ list, int width, int* __restrict__ count,
                   int* __restrict__ table) {
  __shared__ int pg[kPlanInts];
  const int* gp = plan + (int64_t)blockIdx.x * kPlanInts;
  for (int i = threadIdx.x; i < kPlanInts; i += blockDim.x) pg[i] = gp[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = pg[0], nrw = pg[2];
  for (int w = warp; w < nrw; w += blockDim.x / 32) {
    const int rw = pg[3] + w;
    const int a = rowidx[(int64_t)rw * 32 + lane];
    if (a < 0) continue;
    const int R = rounds[rw];
    const uint16_t* lp = reinterpret_cast<const uint16_t*>(list + (int64_t)rw * Q8 * 32 + lane);
    int cnt = 0;
    for (int r = 0; r < R; ++r) {
      const int s = (lp[(r >> 3) * 32 * 8 + (r & 7)] >> 3) - (int)kSlotBias;
      if (s < 0) continue;                    // dummy
      int e = 0;
      while (e < m - 1 && !(s >= pg[6 + 3 * e] && s < pg[6 + 3 * e] + pg[5 + 3 * e])) ++e;
      const int j = pg[4 + 3 * e] + (s - pg[6 + 3 * e]);
      if (cnt < width) table[(int64_t)a * width + cnt] = j;
      ++cnt;
    }
    count[a] = cnt;
  }
}

}  // namespace pc

using namespace pc;

namespace {
int g_build_smem = 0, g_force_smem = 0;
}

extern "C" {

int32_t pc_tile_count(const pc_grid* grid) { return tile_dims(*grid).ntiles; }

static int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int32_t pc_tile_force_partials(int32_t ntiles) {
  const int grid = ntiles < sm_count() ? ntiles : sm_count();
  return (grid > 0 ? grid : 1) * kForceWarps;
}
int32_t pc_tile_plan_ints(void) { return kPlanInts; }
int32_t pc_tile_stage_cap(void) { return kStageCap; }

int pc_pos_from_planar(const double* d_planar, int64_t planar_stride, int32_t n, double* d_pos4,
                       void* stream) {
  if (n <= 0) return PC_OK;
  pos_from_planar_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(d_planar, planar_stride,
                                                                         n, d_pos4);
  return check_launch("pc_pos_from_planar");
}

int pc_cell_zsort(const double* d_pos4, const int32_t* d_cell_start, int32_t ncells,
                  const int32_t* d_order, int32_t* d_out, void* stream) {
  if (ncells <= 0) return PC_OK;
  cell_zsort_kernel<<<(ncells + 7) / 8, 256, 0, as_stream(stream)>>>(d_pos4, d_cell_start, ncells,
                                                                     d_order, d_out);
  return check_launch("pc_cell_zsort");
}

int pc_tile_rows(const int32_t* d_cell_start, const pc_grid* grid, int32_t* d_rw, void* stream) {
  const int nt = tile_dims(*grid).ntiles;
  if (nt <= 0) return PC_OK;
  tile_rows_kernel<<<(nt + 127) / 128, 128, 0, as_stream(stream)>>>(d_cell_start, *grid, d_rw);
  return check_launch("pc_tile_rows");
}

int pc_tile_build(const double* d_planar, int64_t planar_stride, const int32_t* d_cell_start,
                  const pc_grid* grid, const pc_box* box, double cutoff2, int32_t q8,
                  const int32_t* d_rw0, int32_t* d_plan, int32_t* d_rowidx, int32_t* d_rounds,
                  void* d_list, int32_t* d_flag, void* stream) {
  return pc_tile_build_domain(d_planar, planar_stride, d_cell_start, grid, box, cutoff2, q8,
                              d_rw0, d_plan, d_rowidx, d_rounds, d_list, d_flag, stream,
                              nullptr, nullptr, nullptr);
}

int pc_tile_build_domain(const double* d_planar, int64_t planar_stride,
                         const int32_t* d_cell_start, const pc_grid* grid, const pc_box* box,
                         double cutoff2, int32_t q8, const int32_t* d_rw0, int32_t* d_plan,
                         int32_t* d_rowidx, int32_t* d_rounds, void* d_list, int32_t* d_flag,
                         void* stream, const double* d_bplanar, const pc_box* box_exact,
                         const int32_t* d_skip) {
  if (q8 <= 0 || planar_stride % 16) {
    set_error("pc_tile_build: bad list capacity or planar stride");
    return PC_ERR_VALUE;
  }
  for (int a = 0; a < 3; ++a)
    if (grid->nc[a] < 3 || grid->ndim != 3) {
      set_error("pc_tile_build: needs >= 3 cells per axis in 3-D");
      return PC_ERR_VALUE;
    }
  // FP32 prefilter band (same bound as pc_nbr_build_sell): |coordinate
  // relative to the tile centre| <= U
  const double U = fmax(fmax((kBX / 2.0 + 1.0) * grid->width[0], (kBY / 2.0 + 1.0) * grid->width[1]),
                        (kTZ / 2.0 + 1.0) * grid->width[2]);
  const double rc = sqrt(cutoff2);
  const double e23 = ldexp(1.0, -23), e24 = ldexp(1.0, -24);
  const double err = 2.0 * sqrt(3.0) * rc * (e23 * U + e24 * rc) + 3.0 * e24 * cutoff2;
  const double margin = 8.0 * err + 1e-12 * cutoff2;
  TileBuildParams p;
  p.cutoff2 = cutoff2;
  p.lo2 = nextafterf((float)(cutoff2 - margin), -INFINITY);
  p.hi2 = nextafterf((float)(cutoff2 + margin), INFINITY);
  p.Q8 = q8;
  p.max_stage = kStageCap;
  p.ps = planar_stride;
  const int smem = kStageCap * (int)sizeof(float4) +
                   kBuildWarps * 32 * kHitCap * (int)sizeof(uint16_t);
  if (smem > g_build_smem) {
    if (cudaFuncSetAttribute(tile_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess) {
      set_error("pc_tile_build: %d B of shared memory not available", smem);
      return PC_ERR_CAPACITY;
    }
    g_build_smem = smem;
  }
  const int nt = tile_dims(*grid).ntiles;
  tile_build_kernel<<<nt, kBuildWarps * 32, smem, as_stream(stream)>>>(
      d_planar, d_cell_start, *grid, *box, p, d_rw0, d_plan, d_rowidx, d_rounds,
      reinterpret_cast<uint4*>(d_list), d_flag, d_bplanar ? d_bplanar : d_planar,
      box_exact ? *box_exact : *box, d_skip);
  return check_launch("pc_tile_build");
}

int pc_tile_force(const double* d_planar, int64_t planar_stride, int32_t ntiles,
                  const int32_t* d_plan, const int32_t* d_rowidx, const int32_t* d_rounds,
                  const void* d_list, int32_t q8, const pc_box* box, const pc_lj* lj,
                  double mi_guard, double* d_f3, int64_t f_stride, double* d_v, int64_t v_stride,
                  double dtm, double mass, double* d_partial, int32_t* d_flag,
                  double* d_planar_next, double* d_v_next, double dtm_next, double dt,
                  void* stream) {
  if (d_planar_next && !d_v) {
    set_error("pc_tile_force: the fused integrate needs the velocities");
    return PC_ERR_VALUE;
  }
  if (q8 <= 0 || planar_stride % 16) {
    set_error("pc_tile_force: bad list capacity or planar stride");
    return PC_ERR_VALUE;
  }
  if (ntiles <= 0) return PC_OK;
  TileForceParams p;
  p.cutoff2 = lj->cutoff2;
  p.overlap2 = lj->overlap2;
  p.sig2 = (float)(lj->sigma * lj->sigma);
  p.eps24d = 24.0 * lj->epsilon;
  p.eps2d = 2.0 * lj->epsilon;
  p.guard = mi_guard;
  p.Q8 = q8;
  p.ps = planar_stride;
  const int sms = sm_count();
  const int grid = ntiles < sms ? ntiles : sms;
  const int K = (ntiles + grid - 1) / grid;
  // the staging ring in dynamic smem; the CTAs' item prefixes in scratch
  static int smem_max = 0;
  if (smem_max == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem_max <= 0) smem_max = 227 * 1024;
  }
  const int static_bytes = 2048;                           // ForceShared + reserve
  const int smem = 3 * kRingSlots * (int)sizeof(double);
  if (smem + static_bytes > smem_max) {
    set_error("pc_tile_force: the staging ring does not fit in shared memory");
    return PC_ERR_CAPACITY;
  }
  static int* scratch = nullptr;
  static int64_t scratch_n = 0;
  const int64_t need = (int64_t)grid * (3 * K + 1);
  if (need > scratch_n) {
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    scratch_n = 0;
    if (cudaMalloc(&scratch, need * sizeof(int)) != cudaSuccess) {
      set_error("pc_tile_force: scratch allocation of %lld ints failed", (long long)need);
      return PC_ERR_CAPACITY;
    }
    scratch_n = need;
  }
  const bool unit = lj->sigma == 1.0;
  if (smem > g_force_smem) {
    cudaError_t e1 = cudaFuncSetAttribute(tile_force_kernel<true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaError_t e2 = cudaFuncSetAttribute(tile_force_kernel<false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      set_error("pc_tile_force: %d B of shared memory not available", smem);
      return PC_ERR_CAPACITY;
    }
    g_force_smem = smem;
  }
  if (unit)
    tile_force_kernel<true><<<grid, kForceWarps * 32, smem, as_stream(stream)>>>(
        d_planar, p, ntiles, d_plan, d_rowidx, d_rounds, reinterpret_cast<const uint4*>(d_list),
        *box, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial, d_flag, d_planar_next,
        d_v_next, dtm_next, dt, scratch);
  else
    tile_force_kernel<false><<<grid, kForceWarps * 32, smem, as_stream(stream)>>>(
        d_planar, p, ntiles, d_plan, d_rowidx, d_rounds, reinterpret_cast<const uint4*>(d_list),
        *box, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial, d_flag, d_planar_next,
        d_v_next, dtm_next, dt, scratch);
  return check_launch("pc_tile_force");
}

int pc_tile_order(int32_t rw_bound, const int32_t* d_rw_total, const int32_t* d_rounds,
                  void* d_list, int32_t q8, int32_t kind, void* stream) {
  if (rw_bound <= 0 || kind == 0) return PC_OK;
  static int set = 0;
  const int smem = kOrdSmem;
  if (!set) {
    if (cudaFuncSetAttribute(tile_order_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(tile_order_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
      set_error("pc_tile_order: %d B of shared memory not available", smem);
      return PC_ERR_CAPACITY;
    }
    set = 1;
  }
  const int grid = (rw_bound + kOrdWarps - 1) / kOrdWarps;
  uint4* l = reinterpret_cast<uint4*>(d_list);
  if (kind == 1)
    tile_order_kernel<true><<<grid, kOrdWarps * 32, smem, as_stream(stream)>>>(
        l, d_rounds, d_rw_total, q8);
  else
    tile_order_kernel<false><<<grid, kOrdWarps * 32, smem, as_stream(stream)>>>(
        l, d_rounds, d_rw_total, q8);
  return check_launch("pc_tile_order");
}

int pc_tile_decode(int32_t ntiles, const int32_t* d_plan, const int32_t* d_rowidx,
                   const int32_t* d_rounds, const void* d_list, int32_t q8, int32_t width,
                   int32_t* d_count, int32_t* d_table, void* stream) {
  if (ntiles <= 0) return PC_OK;
  tile_decode_kernel<<<ntiles, 256, 0, as_stream(stream)>>>(
      d_plan, q8, kStageCap, d_rowidx, d_rounds, reinterpret_cast<const uint4*>(d_list), width,
      d_count, d_table);
  return check_launch("pc_tile_decode");
}

}  // extern "C"
