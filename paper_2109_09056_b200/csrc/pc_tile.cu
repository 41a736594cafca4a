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
// start (16-B TMA alignment), so slot = seg_dst + (index - seg_src).  Slots
// [max_stage, max_stage + 16) hold NaN positions ("dummies", one per
// LDS.64 bank pair) used as padding: a NaN r^2 fails the cutoff test.
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
#ifndef PC_FORCE_SLEEP
#define PC_FORCE_SLEEP 256      // tile-wait poll interval (ns): 64 -> 256 frees ~0.5 % at C3 (profiles/r02g)
#endif
#ifndef PC_FORCE_WARPS
#define PC_FORCE_WARPS 32
#endif
constexpr int kForceWarps = PC_FORCE_WARPS;
#ifndef PC_FORCE_VIRIAL
#define PC_FORCE_VIRIAL 1       // rows sum u = 2 sr12 - sr6 and sr6: energy + pair virial
#endif
#ifndef PC_FORCE_MIU
#define PC_FORCE_MIU 1          // warp-uniform minimum-image axis flags (C3 force 1034 vs 1056 us, C2 169 vs 173 us, profiles/r02ah)
#endif
#ifndef PC_FORCE_PFDIST
#define PC_FORCE_PFDIST 2       // list groups ahead of the one in use that are L2-prefetched (3 / 4 / 6: 1063 / 1067 / 1070 vs 1052 us at C3, profiles/r02x)
#endif
#ifndef PC_FORCE_HALFU
#define PC_FORCE_HALFU 1        // accumulate u / 2 and fm / 2 (bit-identical results, one instruction less per pair pair)
#endif
#ifndef PC_FORCE_PREFETCH
#define PC_FORCE_PREFETCH 1     // L2 prefetch of list groups two ahead + epilogue velocities
#endif
#ifndef PC_BUILD_WARPS
#define PC_BUILD_WARPS 10       // build warps per CTA (2 CTAs per SM); 8 / 6: build +23 / +36 % (profiles/r02ad)
#endif
constexpr int kBuildWarps = PC_BUILD_WARPS;
#ifndef PC_HIT_CAP
#define PC_HIT_CAP 112          // build hit rows per lane (the row's list capacity)
#endif
constexpr int kHitCap = PC_HIT_CAP;
constexpr int kHitSlack = 3;   // spare rows per hit column (unclamped 4-candidate stores)
// force-kernel staging capacity (slots) and per-coordinate stride in shared
// memory: compile-time so every LDS is [slot*8 + immediate]
constexpr int kStageCap = 2304;
constexpr int kStageStride = kStageCap + 16;

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

// per tile: row-warps = ceil(home rows / 32); with `skip` (a decomposed
// domain's ghost flags) only the owned home rows are rows.  One warp per tile
// (the owned count is a ballot sweep over the tile's ~300 home particles).
__global__ void tile_rows_kernel(const int* __restrict__ cs, pc_grid g, int* __restrict__ rw,
                                 const int* __restrict__ skip) {
  const TileDims d = tile_dims(g);
  const int tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (tile >= d.ntiles) return;
  const int tz = tile % d.ntz, t2 = tile / d.ntz;
  const int ty = t2 % d.nty, tx = t2 / d.nty;
  const int x0 = tx * kBX, y0 = ty * kBY, z0 = tz * kTZ;
  const int bx = min(kBX, g.nc[0] - x0), by = min(kBY, g.nc[1] - y0), bz = min(kTZ, g.nc[2] - z0);
  int h = 0;
  for (int hx = 0; hx < bx; ++hx)
    for (int hy = 0; hy < by; ++hy) {
      const int c0 = ((x0 + hx) * g.nc[1] + (y0 + hy)) * g.nc[2] + z0;
      const int j0 = cs[c0], j1 = cs[c0 + bz];
      if (skip) {
        for (int j = j0; j < j1; j += 32)
          h += __popc(__ballot_sync(0xffffffffu, j + lane < j1 && !skip[j + lane]));
      } else {
        h += j1 - j0;
      }
    }
  // at least one row-warp per tile: a tile without home rows still gets an
  // (empty) item, so the force kernel's warp that takes it releases the
  // staging buffer the tile was loaded into (nothing else would)
  if (lane == 0) rw[tile] = max(1, (h + 31) >> 5);
}

// ---- TMA / mbarrier helpers ----------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

#ifndef PC_BUILD_JOINTSEARCH
#define PC_BUILD_JOINTSEARCH 1   // a column window's two bisections in one loop (C3 build + order 5.25 vs 5.35 ms, profiles/r02ap)
#endif
#ifndef PC_BUILD_MASKTAIL
#define PC_BUILD_MASKTAIL 1   // a piece's last 1-3 candidates as one masked 4-candidate step (build + order -0.3 %, profiles/r02ak)
#endif
#ifndef PC_STS_CLOBBER
#define PC_STS_CLOBBER 0   // 1: "memory" clobber on the hit stores (no measurable difference, profiles/r02w)
#endif
// Hit-list store of the build sweeps.  Without a "memory" clobber the
// compiler may issue the next step's staging loads before this step's hit
// stores (different arrays); every sweep ends with compiler_fence() before
// the hit list is read back.
__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
#if PC_STS_CLOBBER
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
#else
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v));
#endif
}
__device__ __forceinline__ void compiler_fence() { asm volatile("" ::: "memory"); }

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

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- two pairs per call: the FP32 LJ magnitude as packed f32x2 ------------
// sm_100 issues FADD2/FMUL2/FFMA2 (two FP32 lanes per thread, one issue
// slot): the seven FP32 instructions of a pair's LJ magnitude become 3.5 per
// pair.  Same per-element rounding as the scalar form (fma.rn / mul.rn on
// each half); the row's u and sr6 sums are kept as two partial sums.
typedef unsigned long long f32x2_t;
__device__ __forceinline__ f32x2_t pk2(float a, float b) {
  f32x2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(f32x2_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2_t mul2(f32x2_t a, f32x2_t b) {
  f32x2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2_t add2(f32x2_t a, f32x2_t b) {
  f32x2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2_t fma2(f32x2_t a, f32x2_t b, f32x2_t c) {
  f32x2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
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
  int sched;           // 1: bank-conflict-free round schedule, 0: ascending order
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

// Residue-group resolution of one proposal pass (see schedule_rows): lanes
// of the same half-warp proposing slots of equal residue form a group (one
// MATCH.ANY); the lowest critical lane of the group, else its lowest lane,
// wins, and so does every lane proposing the winner's slot.
__device__ __forceinline__ bool resolve(bool has, int s, unsigned crit, int half, int lane,
                                        unsigned& taken) {
  const unsigned FULL = 0xffffffffu;
  const int r = s & 15;
  const unsigned g = __match_any_sync(FULL, has ? (unsigned)((half << 4) | r)
                                                : (unsigned)(32 + lane));
  const unsigned gc = g & crit;
  const int wl = __ffs(gc ? gc : g) - 1;
  const int ws = __shfl_sync(FULL, s, wl);
  const unsigned all = __reduce_or_sync(FULL, has ? (1u << ((half << 4) + r)) : 0u);
  taken |= (all >> (half << 4)) & 0xFFFFu;
  return has && s == ws;
}

// Bank-conflict-free round schedule of one row-warp.  Every lane holds its
// row's slots in sweep order (hits[k*32]); in each round each lane takes one
// entry so that within a half-warp (one LDS.64 pass of 16 lanes; measured,
// scripts/micro/lds_banks.cu: conflicts across the two halves are free) all
// lanes read distinct bank pairs (slot % 16) or the very same slot
// (broadcast).  Two passes per round: every lane proposes its next entry;
// per residue the lowest "critical" lane (remaining entries >= the warp's
// maximum - 1: it bounds the round count), else the lowest lane, wins,
// together with every lane proposing the winner's slot; losers then propose
// the first entry of their next three whose residue is still free.  Lanes
// left unassigned read a NaN-free dummy of a free residue.  Simulated on LJ
// tiles: 1.08x the rounds of the longest row; measured 2.0 LDS wavefronts
// per LDS.64 (unscheduled sweep order: 4.9).  The 4-entry window lives in two
// registers of packed u16 (entry removal = two PRMTs).  Emits slot*8 (the
// byte offset of the slot in one coordinate array).
__device__ __forceinline__ int schedule_rows(const uint16_t* __restrict__ hits, int cnt,
                                             int lane, int dummy0, uint4* __restrict__ out,
                                             int cap_rounds, bool two_pass) {
  const unsigned FULL = 0xffffffffu;
  const int half = lane >> 4;
  auto ld = [&](int k) -> uint32_t { return k < cnt ? (uint32_t)hits[k * 32] : 0xFFFFu; };
  uint32_t w01 = ld(0) | (ld(1) << 16), w23 = ld(2) | (ld(3) << 16);
  int ptr = 4;
  int rem = cnt;
  int R = 0;
  uint32_t b0 = 0u, b1 = 0u, b2 = 0u, b3 = 0u;     // 8 x u16 shift register
  for (;;) {
    const int maxrem = __reduce_max_sync(FULL, rem);
    if (maxrem == 0) break;
    const unsigned crit = __ballot_sync(FULL, rem > 0 && rem >= maxrem - 1);
    unsigned taken = 0u;
    const int e0 = (int)(w01 & 0xFFFFu);
    int pi = -1, outs = -1;
    if (resolve(rem > 0, e0, crit, half, lane, taken)) {
      pi = 0;
      outs = e0;
    }
    if (two_pass && __any_sync(FULL, pi < 0 && rem > 1)) {
      const int e1 = (int)(w01 >> 16), e2 = (int)(w23 & 0xFFFFu), e3 = (int)(w23 >> 16);
      int q = -1, qs = 0;
      if (pi < 0) {
        if (e3 != 0xFFFF && !((taken >> (e3 & 15)) & 1u)) { q = 3; qs = e3; }
        if (e2 != 0xFFFF && !((taken >> (e2 & 15)) & 1u)) { q = 2; qs = e2; }
        if (e1 != 0xFFFF && !((taken >> (e1 & 15)) & 1u)) { q = 1; qs = e1; }
      }
      if (resolve(q >= 0, qs, crit, half, lane, taken)) {
        pi = q;
        outs = qs;
      }
    }
    if (pi >= 0) {       // drop entry pi, append the next hit
      const uint32_t nx = ld(ptr);
      ++ptr;
      --rem;
      const uint32_t n01 = pi == 0 ? __byte_perm(w01, w23, 0x5432)
                                   : (pi == 1 ? __byte_perm(w01, w23, 0x5410) : w01);
      w23 = __byte_perm(w23, nx, pi == 3 ? 0x5410 : 0x5432);
      w01 = n01;
    } else {
      outs = dummy0 + (__ffs(~taken & 0xFFFFu) - 1);
    }
    b0 = __funnelshift_r(b0, b1, 16);
    b1 = __funnelshift_r(b1, b2, 16);
    b2 = __funnelshift_r(b2, b3, 16);
    b3 = (b3 >> 16) | ((uint32_t)(outs * 8) << 16);
    ++R;
    if ((R & 7) == 0 && R <= cap_rounds) out[((R >> 3) - 1) * 32] = make_uint4(b0, b1, b2, b3);
  }
  if (R & 7) {     // pad the open group with conflict-free dummies
    const uint32_t d = (uint32_t)((dummy0 + (lane & 15)) * 8);
    for (int r = R; r & 7; ++r) {
      b0 = __funnelshift_r(b0, b1, 16);
      b1 = __funnelshift_r(b1, b2, 16);
      b2 = __funnelshift_r(b2, b3, 16);
      b3 = (b3 >> 16) | (d << 16);
    }
    if (((R + 7) & ~7) <= cap_rounds) out[(R >> 3) * 32] = make_uint4(b0, b1, b2, b3);
  }
  return R;
}

// ---- residue round-robin row order (default) --------------------------------
// Lane-local bank-conflict avoidance (no cross-lane coordination).  The
// entries of a row are bucketed by bank-pair residue (slot % 16) and emitted
// round-robin: in round r the lane prefers residue (lane + r) % 16 -- the 16
// lanes of a half-warp prefer 16 distinct residues in every round -- and
// falls back to the next non-empty residue.  Simulated on LJ tiles: 1.6
// LDS.64 passes per half-warp instead of 2.5 for the ascending order, at the
// same round count; measured: force pass -14 %.  Cost: the row's class-major
// order is scattered into its own list column (global, L2-resident), then
// read back in round-robin order (rotate + ffs over the mask of non-empty
// residues, byte counters packed in two 64-bit words), then written out.
__device__ __forceinline__ int rr_rows(uint16_t* __restrict__ hits, int cnt, int lane,
                                       int dummy0, uint4* __restrict__ out, int cap_rounds) {
  uint16_t* col = reinterpret_cast<uint16_t*>(out);     // slot k at (k >> 3) * 256 + (k & 7)
  const unsigned long long B = 0x0101010101010101ull;
  unsigned long long clo = 0ull, chi = 0ull;            // per-class counts (bytes)
  for (int k = 0; k < cnt; ++k) {
    const int c = hits[k * 32] & 15;
    const unsigned long long inc = 1ull << ((c & 7) * 8);
    if (c < 8) clo += inc; else chi += inc;
  }
  const unsigned long long ilo = clo * B;               // inclusive byte prefix (< 256)
  const unsigned long long slo = ilo - clo;
  const unsigned long long shi = chi * B - chi + (ilo >> 56) * B;
  unsigned long long rlo = slo, rhi = shi;
  for (int k = 0; k < cnt; ++k) {                       // class-major scatter
    const uint32_t v = hits[k * 32];
    const int c = v & 15, sh = (c & 7) * 8;
    const unsigned long long inc = 1ull << sh;
    int pos;
    if (c < 8) { pos = (int)((rlo >> sh) & 0xFFull); rlo += inc; }
    else       { pos = (int)((rhi >> sh) & 0xFFull); rhi += inc; }
    col[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)(v * 8u);
  }
  const unsigned long long nz = ((clo | (clo >> 1) | (clo >> 2) | (clo >> 3) | (clo >> 4) |
                                  (clo >> 5) | (clo >> 6) | (clo >> 7)) & B);
  const unsigned long long nzh = ((chi | (chi >> 1) | (chi >> 2) | (chi >> 3) | (chi >> 4) |
                                   (chi >> 5) | (chi >> 6) | (chi >> 7)) & B);
  // byte-wise "non-zero" flags -> 16-bit mask (bit c = class c non-empty)
  unsigned ne = (unsigned)(((nz * 0x0102040810204080ull) >> 56) & 0xFFull) |
                ((unsigned)(((nzh * 0x0102040810204080ull) >> 56) & 0xFFull) << 8);
  unsigned long long plo = slo, phi = shi, qlo = clo, qhi = chi;
  for (int r0 = 0; r0 < cnt; r0 += 8) {                 // round-robin emission
    // 8 rounds: positions from the register state first, then 8 independent
    // loads of the class-major copy (L2 round trips overlap)
    int pos[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int pref = (lane + r0 + u) & 15;
      const unsigned rot = ((ne >> pref) | (ne << (16 - pref))) & 0xFFFFu;
      const int c = (pref + __ffs(rot) - 1) & 15, sh = (c & 7) * 8;
      const unsigned long long inc = 1ull << sh;
      unsigned left;
      if (c < 8) {
        pos[u] = (int)((plo >> sh) & 0xFFull);
        plo += inc;
        qlo -= inc;
        left = (unsigned)((qlo >> sh) & 0xFFull);
      } else {
        pos[u] = (int)((phi >> sh) & 0xFFull);
        phi += inc;
        qhi -= inc;
        left = (unsigned)((qhi >> sh) & 0xFFull);
      }
      if (left == 0u) ne &= ~(1u << c);
      if (r0 + u >= cnt) pos[u] = 0;      // past the row: any valid address
      if (ne == 0u) ne = 1u;              // (exhausted: keep ffs defined)
    }
    uint16_t vals[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) vals[u] = col[(pos[u] >> 3) * 256 + (pos[u] & 7)];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (r0 + u < cnt) hits[(r0 + u) * 32] = vals[u];
  }
  const int R = __reduce_max_sync(0xffffffffu, cnt);
  for (int r8 = 0; r8 < R && r8 + 8 <= cap_rounds; r8 += 8) {
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int r = r8 + 2 * h;
      const uint32_t lo = r < cnt ? (uint32_t)hits[r * 32]
                                  : (uint32_t)(dummy0 + ((lane + r) & 15)) * 8u;
      const uint32_t hi = r + 1 < cnt ? (uint32_t)hits[(r + 1) * 32]
                                      : (uint32_t)(dummy0 + ((lane + r + 1) & 15)) * 8u;
      w[h] = lo | (hi << 16);
    }
    out[(r8 >> 3) * 32] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  return R;
}

// Cheaper variant (default): class-major order with the residue classes
// visited in a lane-rotated order (lane l starts at residue l % 16).  The
// row's entries are scattered straight into their final list positions (one
// pass over the hits; per-class running counts as packed bytes).  Simulated:
// 2.0 LDS.64 passes per half-warp (round-robin: 1.6, ascending: 2.5).
__device__ __forceinline__ int cm_rows(const uint16_t* __restrict__ hits, int cnt, int lane,
                                       int dummy0, uint4* __restrict__ out, int cap_rounds) {
  uint16_t* col = reinterpret_cast<uint16_t*>(out);     // slot k at (k >> 3) * 256 + (k & 7)
  const unsigned long long B = 0x0101010101010101ull;
  unsigned long long clo = 0ull, chi = 0ull;            // per-class counts (bytes)
  for (int k = 0; k < cnt; ++k) {
    const int c = hits[k * 32] & 15;
    const unsigned long long inc = 1ull << ((c & 7) * 8);
    if (c < 8) clo += inc; else chi += inc;
  }
  const unsigned long long ilo = clo * B;
  unsigned long long rlo = ilo - clo;                   // exclusive prefix = class starts
  unsigned long long rhi = chi * B - chi + (ilo >> 56) * B;
  const int l0 = lane & 15;
  const int s0 = (int)(((l0 < 8 ? rlo : rhi) >> ((l0 & 7) * 8)) & 0xFFull);
  for (int k = 0; k < cnt; ++k) {
    const uint32_t v = hits[k * 32];
    const int c = v & 15, sh = (c & 7) * 8;
    const unsigned long long inc = 1ull << sh;
    int pos;
    if (c < 8) { pos = (int)((rlo >> sh) & 0xFFull); rlo += inc; }
    else       { pos = (int)((rhi >> sh) & 0xFFull); rhi += inc; }
    pos -= s0;                                          // rotate: class l0 first
    if (pos < 0) pos += cnt;
    col[(pos >> 3) * 256 + (pos & 7)] = (uint16_t)(v * 8u);
  }
  const int R = __reduce_max_sync(0xffffffffu, cnt);
  for (int r = cnt; r < ((R + 7) & ~7) && r < cap_rounds; ++r)
    col[(r >> 3) * 256 + (r & 7)] = (uint16_t)((dummy0 + ((lane + r) & 15)) * 8);
  return R;
}

// Unscheduled rounds: entry k of every row in round k (sweep order), padded
// with dummies -- the cheap alternative to schedule_rows (PC_TILE_NOSCHED).
__device__ __forceinline__ int plain_rows(const uint16_t* __restrict__ hits, int cnt, int lane,
                                          int dummy0, uint4* __restrict__ out, int cap_rounds) {
  const int R = __reduce_max_sync(0xffffffffu, cnt);
  const uint32_t d = (uint32_t)((dummy0 + (lane & 15)) * 8);
  for (int r8 = 0; r8 < R && r8 + 8 <= cap_rounds; r8 += 8) {
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int r = r8 + 2 * h;
      const uint32_t lo = r < cnt ? (uint32_t)hits[r * 32] * 8u : d;
      const uint32_t hi = r + 1 < cnt ? (uint32_t)hits[(r + 1) * 32] * 8u : d;
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

// Decomposed domain (`skip` = ghost flags): the tile's rows are its OWNED
// home particles only, numbered in (home column, z) order -- ghost rows carry
// no list, and a row-warp mixing owned and ghost lanes would run its ghost
// lanes idle in the build, the order pass and every force pass.  Lane L of
// row-warp w gets the (32 w + L)-th owned home slot (-1: none) and its home
// column; one ballot scan of the home slots per row-warp.
__device__ __forceinline__ int owned_row_slot(const TileSetup& T, const int* __restrict__ skip,
                                              int w, int lane, int& col) {
  const int target = 32 * w + lane;
  int base = 0, mine = -1;
  col = 0;
  for (int c = 0; c < kBX * kBY; ++c) {
    const int hx = c / kBY, hy = c - hx * kBY;
    if (hx >= T.bx || hy >= T.by) continue;
    const int hcol = (hx + 1) * kSY + (hy + 1);
    const int s0 = T.cell_lo[hcol][1], s1 = T.cell_hi[hcol][T.bz];
    const int e = hcol * 3 + 1;                  // home cells: the in-range segment
    const int off = T.seg_src[e] - T.seg_dst[e];
    for (int s = s0; s < s1 && base < 32 * w + 32; s += 32) {
      const int sl = s + lane;
      const bool own = sl < s1 && !skip[off + sl];
      const unsigned bal = __ballot_sync(0xffffffffu, own);
      const int n = target - base;
      const bool in = n >= 0 && n < __popc(bal);
      const int src = in ? (int)__fns(bal, 0, n + 1) : 0;
      const int got = __shfl_sync(0xffffffffu, sl, src);
      if (in) {
        mine = got;
        col = c;
      }
      base += __popc(bal);
    }
  }
  return mine;
}

// Residue round-robin order of one row-warp's list, in place (the lane's own
// column of uint4 groups at lp; the list was just written by this warp, so it
// is read back from L2): the algorithm of tile_order_kernel<true> below with
// a u16 per-class state (next | end << 8, positions <= kHitCap < 256).
// st: this warp's [16][32] u16 table + lane; Bm: >= kHitCap + 1 rows of
// [k][32] u16 + lane (the build's hit buffer, free once the list is out).
__device__ __forceinline__ void rr_order_rowwarp(uint4* __restrict__ lp, int R,
                                                 uint16_t* __restrict__ st,
                                                 uint16_t* __restrict__ Bm, int lane,
                                                 int dummy0) {
  const uint32_t dmin = (uint32_t)dummy0 * 8u;
  const int G = (R + 7) >> 3;
#pragma unroll
  for (int c = 0; c < 16; ++c) st[c * 32] = 0;
  int cnt = 0;                                          // real entries precede padding
  uint4 qn = lp[0];
  for (int g = 0; g < G; ++g) {                         // per-class counts
    const uint4 q = qn;
    if (g + 1 < G) qn = lp[(g + 1) * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      const uint32_t real = v < dmin ? 1u : 0u;
      st[((v >> 3) & 15) * 32] += (uint16_t)real;
      cnt += (int)real;
    }
  }
  uint32_t run = 0u;
#pragma unroll
  for (int c = 0; c < 16; ++c) {                        // next | end << 8
    const uint32_t n = st[c * 32];
    st[c * 32] = (uint16_t)(run | ((run + n) << 8));
    run += n;
  }
  unsigned ne = 0u;
  qn = lp[0];
  for (int g = 0; g < G; ++g) {                         // class-major scatter -> Bm
    const uint4 q = qn;
    if (g + 1 < G) qn = lp[(g + 1) * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      const bool real = v < dmin;
      const int c = (v >> 3) & 15;
      const uint32_t e = st[c * 32];
      st[c * 32] = (uint16_t)(e + (real ? 1u : 0u));
      ne |= real ? 1u << c : 0u;
      Bm[(real ? (int)(e & 0xFFu) : kHitCap) * 32] = (uint16_t)v;
    }
  }
  uint32_t beg = 0u;                                    // rewind next to begin(c) = end(c - 1)
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint32_t end = (uint32_t)st[c * 32] >> 8;
    st[c * 32] = (uint16_t)(beg | (end << 8));
    beg = end;
  }
  for (int g = 0; g < G; ++g) {                         // emit 8 rounds per uint4
    uint32_t o[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int r = g * 8 + t;
      const bool real = r < cnt;
      const int pref = (lane + r) & 15;
      const unsigned rot = ((ne >> pref) | (ne << (16 - pref))) & 0xFFFFu;
      const int c = (pref + __ffs(rot) - 1) & 15;
      const uint32_t e = st[c * 32];
      const int pos = (int)(e & 0xFFu);
      st[c * 32] = (uint16_t)(e + (real ? 1u : 0u));
      if (real && (uint32_t)pos + 1u == (e >> 8)) ne &= ~(1u << c);
      const uint32_t vb = Bm[(real ? pos : kHitCap) * 32];
      const uint32_t v = real ? vb : (uint32_t)(dummy0 + ((lane + r) & 15)) * 8u;
      o[t >> 1] |= (t & 1) ? (v << 16) : v;
    }
    lp[g * 32] = make_uint4(o[0], o[1], o[2], o[3]);
  }
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

// ORD: the residue round-robin order of every row-warp is applied right
// after its list is written (rr_order_rowwarp, list read back from L2),
// instead of a separate pc_tile_order pass over HBM; nine warps (the
// per-warp class table needs the shared memory of the tenth).
__host__ __device__ constexpr int build_warps(bool ord) { return ord ? 9 : kBuildWarps; }

template <bool ORD>
__global__ void __launch_bounds__(build_warps(ORD) * 32, 2)
tile_build_kernel(const double* __restrict__ pl, const int* __restrict__ cs, pc_grid g, pc_box b,
                  TileBuildParams p, const int* __restrict__ rw0, int* __restrict__ plan,
                  int* __restrict__ rowidx, int* __restrict__ rounds, uint4* __restrict__ list,
                  int* __restrict__ flag, const double* __restrict__ bpl, pc_box e,
                  const int* __restrict__ skip, int* __restrict__ tile_ghost) {
  extern __shared__ float4 cz[];                 // staged FP32 copy | per-warp hit rows
  __shared__ TileSetup T;
  uint16_t* hits_all = reinterpret_cast<uint16_t*>(cz + p.max_stage);
  tile_setup<true>(blockIdx.x, g, b, cs, T);
  if (T.S > p.max_stage) {
    // flag it; leave an empty plan so that a speculatively launched force
    // pass stays in bounds (the caller discards it and falls back).  The
    // tile keeps ONE empty row-warp (no rows, zero rounds): the force
    // kernel's warp that takes it releases the staging buffer the tile was
    // loaded into -- a tile without items would hold its buffer forever and
    // stall every later tile of the CTA (tile_rows_kernel reserves >= 1
    // row-warp per tile, so rw0[tile] is this tile's own)
    const int r0 = rw0[blockIdx.x];
    if (threadIdx.x < 32) rowidx[(int64_t)r0 * 32 + threadIdx.x] = -1;
    if (threadIdx.x == 0) {
      atomicOr(flag, kFlagStage);
      atomicMax(flag + 1, T.S);
      int* pg = plan + (int64_t)blockIdx.x * kPlanInts;
      pg[0] = 0;
      pg[1] = 0;
      pg[2] = 1;
      pg[3] = r0;
      rounds[r0] = 0;
      if (tile_ghost) tile_ghost[blockIdx.x] = 1;
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // as tile_rows_kernel (owned home rows only when `skip` is given)
  const int nrw = skip ? rw0[blockIdx.x + 1] - rw0[blockIdx.x] : max(1, (T.H + 31) >> 5);
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
  int ghost_seen = 0;        // a ghost row among the staged particles (tile_ghost)
  // stage: slot order, one warp per segment (a segment is ~40 particles:
  // all threads walking every segment left 7 of 8 idle)
  for (int e = threadIdx.x >> 5; e < kSegs; e += build_warps(ORD)) {
    const int len = T.seg_len[e];
    if (len == 0) continue;
    const int src = T.seg_src[e], dst = T.seg_dst[e];
    const double sx = (double)T.seg_shift[e][0] * b.length[0] - T.ox;
    const double sy = (double)T.seg_shift[e][1] * b.length[1] - T.oy;
    const double sz = (double)T.seg_shift[e][2] * b.length[2] - T.oz;
    for (int t = threadIdx.x & 31; t < len; t += 32) {
      const int j = src + t;
      float4 q;
      q.x = (float)(bpl[j] + sx);
      q.y = (float)(bpl[ps + j] + sy);
      q.z = (float)(bpl[2 * ps + j] + sz);
      q.w = 0.f;
      cz[dst + t] = q;
      if (tile_ghost && skip) ghost_seen |= skip[j];
    }
  }
  // interior tiles (no ghost in the staged neighbourhood) do not read ghost
  // positions: their force pass may run while the ghost refresh is in flight
  ghost_seen = __syncthreads_or(ghost_seen);
  if (tile_ghost && threadIdx.x == 0) tile_ghost[blockIdx.x] = ghost_seen ? 1 : 0;

  uint16_t* hits = hits_all + warp * (kHitCap + kHitSlack) * 32 + lane;   // [k][lane]
  for (int w = warp; w < nrw; w += build_warps(ORD)) {
    const int u = w * 32 + lane;
    int ocol = 0;
    const int opos = skip ? owned_row_slot(T, skip, w, lane, ocol) : -1;
    const bool act = skip ? opos >= 0 : u < T.H;
    int cnt = 0, a = -1, pos = -1, nband = 0;
    if (act) {
      // hit list: entry k of this lane's row at shared byte address hbase + 64 k
      const uint32_t hbase = smem_u32(hits);
      const uint32_t hend = hbase + (uint32_t)(kHitCap - 1) * 64u;
      uint32_t ha = hbase;
      float mx = 0.f;
      int c = 0;
#pragma unroll
      for (int q = 1; q < kBX * kBY; ++q) c += (u >= T.home_pre[q]) ? 1 : 0;
      if (skip) c = ocol;
      const int hx = c / kBY, hy = c - hx * kBY;
      const int hcol = (hx + 1) * kSY + (hy + 1);
      pos = skip ? opos : T.cell_lo[hcol][1] + (u - T.home_pre[c]);
      int k = 1;
      for (int kk = 2; kk <= bz; ++kk) k += (pos >= T.cell_lo[hcol][kk]) ? 1 : 0;
      a = slot_index(T, pos);
      const float4 me = cz[pos];
      // (with `skip`, ghosts of a decomposed domain are never rows)
      const bool scan = true;
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
        const int e1 = T.cell_hi[col][k - 1];
        const int b2 = T.cell_lo[col][k], e2 = T.cell_hi[col][k];
        const int b3 = T.cell_lo[col][k + 1];
        int hi = b3, h3 = T.cell_hi[col][k + 1];
#if PC_BUILD_JOINTSEARCH
        // both bisections in one loop: two independent load chains in flight
        while (lo < h1 || hi < h3) {
          const int m1 = (lo + h1) >> 1, m3 = (hi + h3) >> 1;
          const float z1 = lo < h1 ? cz[m1].z : 0.f;
          const float z3 = hi < h3 ? cz[m3].z : 0.f;
          if (lo < h1) {
            if (z1 < zlo) lo = m1 + 1; else h1 = m1;
          }
          if (hi < h3) {
            if (z3 <= zhi) hi = m3 + 1; else h3 = m3;
          }
        }
#else
        while (lo < h1) {
          const int mid = (lo + h1) >> 1;
          if (cz[mid].z < zlo) lo = mid + 1; else h1 = mid;
        }
        while (hi < h3) {
          const int mid = (hi + h3) >> 1;
          if (cz[mid].z <= zhi) hi = mid + 1; else h3 = mid;
        }
#endif
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
            // absolute shared addresses; one clamp per step (the column's
            // kHitSlack spare rows take o1..o3 past the last row)
            const uint32_t o1 = ha + (h[0] ? 64u : 0u);
            const uint32_t o2 = o1 + (h[1] ? 64u : 0u);
            const uint32_t o3 = o2 + (h[2] ? 64u : 0u);
            st_shared_u16(ha, (uint16_t)i);
            st_shared_u16(o1, (uint16_t)(i + 1));
            st_shared_u16(o2, (uint16_t)(i + 2));
            st_shared_u16(o3, (uint16_t)(i + 3));
            ha = min(o3 + (h[3] ? 64u : 0u), hend);
          }
#if PC_BUILD_MASKTAIL
          if (i < s1) {
            // the last 1-3 candidates as one masked step (independent
            // tests instead of a chain of single ones; slots past s1 are read
            // -- staged neighbours or the hit rows behind the staging area --
            // and masked out)
            bool h[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float4 q = cz[i + u];
              const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
              const float rr = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
              h[u] = rr < p.hi2 && i + u < s1;
              mx = fmaxf(mx, h[u] ? rr : 0.f);
            }
            const uint32_t o1 = ha + (h[0] ? 64u : 0u);
            const uint32_t o2 = o1 + (h[1] ? 64u : 0u);
            const uint32_t o3 = o2 + (h[2] ? 64u : 0u);
            st_shared_u16(ha, (uint16_t)i);
            st_shared_u16(o1, (uint16_t)(i + 1));
            st_shared_u16(o2, (uint16_t)(i + 2));
            st_shared_u16(o3, (uint16_t)(i + 3));
            ha = min(o3 + (h[3] ? 64u : 0u), hend);
          }
#else
          for (; i < s1; ++i) {
            const float4 q = cz[i];
            const float dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
            const float rr = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            st_shared_u16(ha, (uint16_t)i);
            const bool hit = rr < p.hi2;
            mx = fmaxf(mx, hit ? rr : 0.f);
            ha = min(ha + (hit ? 64u : 0u), hend);
          }
#endif
        }
      }
      compiler_fence();
      cnt = (int)((ha - hbase) >> 6);
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
    const int R = p.sched == 0   ? cm_rows(hits, cnt, lane, p.max_stage, lout, cap)
                  : p.sched == 4 ? rr_rows(hits, cnt, lane, p.max_stage, lout, cap)
                  : p.sched == 3 ? plain_rows(hits, cnt, lane, p.max_stage, lout, cap)
                                 : schedule_rows(hits, cnt, lane, p.max_stage, lout, cap,
                                                 p.sched == 1);
    if (lane == 0) {
      rounds[rw] = ((R + 7) & ~7) > cap ? 0 : R;
      if (((R + 7) & ~7) > cap) {
        atomicOr(flag, kFlagOverflow);
        atomicMax(flag + 2, R);
      }
    }
    __syncwarp();
    if (ORD && R > 0 && ((R + 7) & ~7) <= cap) {
      uint16_t* st = reinterpret_cast<uint16_t*>(
                         hits_all + build_warps(ORD) * (kHitCap + kHitSlack) * 32) +
                     warp * 16 * 32 + lane;
      rr_order_rowwarp(lout, R, st, hits, lane, p.max_stage);
      __syncwarp();
    }
  }
}

// (Build variants with per-lane spherical z-windows -- a flat piece sweep and
// a column-lockstep sweep over planar FP32 copies with packed tests, and a
// per-column z index -- were measured in r02q-r02t and removed: none beat
// tile_build_kernel, profiles/r02t; source in git 4ae9a62.)

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
cell_zsort_kernel(const double* __restrict__ zp, int64_t zs, const int* __restrict__ cs,
                  int ncells, const int* __restrict__ order, int* __restrict__ out) {
  const int cell = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (cell >= ncells) return;
  const int s0 = cs[cell], m = cs[cell + 1] - s0;
  for (int t0 = 0; t0 < m; t0 += 32) {
    const int t = t0 + lane;
    const int src = t < m ? order[s0 + t] : 0;
    const double z = t < m ? zp[zs * src] : 0.0;
    // rank by (z, particle index): independent of the input order inside
    // the cell, so the placement before it need not be stable
    int rk = 0;
    for (int u0 = 0; u0 < m; u0 += 32) {
      const int uu = u0 + lane;
      const int su_l = uu < m ? order[s0 + uu] : 0;
      const double zu_l = uu < m ? zp[zs * su_l] : 0.0;
      const int lim = min(32, m - u0);
      for (int v = 0; v < lim; ++v) {
        const double zu = __shfl_sync(0xffffffffu, zu_l, v);
        const int su = __shfl_sync(0xffffffffu, su_l, v);
        rk += (zu < z || (zu == z && su < src)) ? 1 : 0;
      }
    }
    if (t < m) out[s0 + rk] = src;
  }
}

// ---- force ------------------------------------------------------------------
// Persistent kernel: one CTA of kForceWarps warps per SM walks its tiles
// (blockIdx.x + k*gridDim.x) through a ring of kNBuf shared-memory staging
// buffers.  Row-warps of all its tiles form one queue (item i -> tile k by
// the prefix of row-warp counts); a warp takes the next item, prefetches the
// row's list / position / index words, waits on the buffer's mbarrier and
// sweeps the rounds.  The warp finishing a tile's last row-warp frees its
// buffer and immediately issues the TMA bulk copies of the next unloaded
// tile into it, so staging overlaps the compute of the tiles in flight and
// no warp idles at a tile boundary.
constexpr int kNBuf = 4;       // max staging buffers (runtime: as many as fit)
extern __shared__ __align__(16) double pc_force_dyn[];

struct TileForceParams {
  double cutoff2, overlap2;
  float sig2;
  double eps24d, eps2d;
  double guard;        // minimum image only within this distance of a periodic face
  int Q8;
  int64_t ps;
};

// (Measured and removed: per-tile mbarrier waits instead of the
// buffer poll, claiming items one ahead, L2 prefetch of the next items' list
// heads, a second list group in registers, per-buffer code paths.)
struct ForceShared {
  uint64_t bar[kNBuf];
  volatile int seq[kNBuf];   // tile sequence index held by each buffer (-1: none)
  int par[kNBuf];            // mbarrier parity of the current use
  int uses[kNBuf];
  int done[kNBuf];           // finished row-warps of the current tile
  int next_item;
  int loaded;                // tickets: next tile sequence index to load
  int K;                     // tiles of this CTA
  int items;                 // row-warps of this CTA
  const int* tiles;          // tile subset (nullptr: all tiles)
  int t0;                    // first entry of the subset in `tiles`
};

// tile of this CTA's sequence index k (all tiles, or a subset list)
__device__ __forceinline__ int tile_at(const int* __restrict__ tiles, int t0, int k) {
  const int s = (int)blockIdx.x + k * (int)gridDim.x;
  return tiles ? tiles[t0 + s] : s;
}

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
                                          double& fy, double& fz, float& su, float& s6,
                                          bool& overlap) {
  const double* q = reinterpret_cast<const double*>(st + off);
  double dx = __dsub_rn(q[0], xi);
  double dy = __dsub_rn(q[kStageStride], yi);
  double dz = __dsub_rn(q[2 * kStageStride], zi);
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
  // u = 2 sr12 - sr6 = r F(r) / 24 eps: the pair virial; fm = u / r^2; the
  // pair energy sr12 - sr6 = (u - sr6) / 2 -- so the row keeps two sums,
  // sum u (virial) and sum sr6, at the cost the single energy sum had
#if PC_FORCE_VIRIAL
  const float u = sr6 * fmaf(2.0f, sr6, -1.0f);
  const float fm = u * inv;
  su += u;
  s6 += sr6;
#else     // energy only (r01 form): su holds 2 sum (sr12 - sr6), s6 stays 0
  const float fm = (sr6 * inv) * fmaf(2.0f, sr6, -1.0f);
  su += 2.0f * fmaf(sr6, sr6, -sr6);
#endif
  const double fmd = (double)fm;
  fx = fma(-fmd, dx, fx);
  fy = fma(-fmd, dy, fy);
  fz = fma(-fmd, dz, fz);
}

// FP64 half of a pair: displacement (minimum image near periodic faces),
// exact r^2 and cutoff test; returns the narrowed r^2 of an interacting pair,
// else 1e30 (the FP32 terms then vanish exactly)
template <bool MI>
__device__ __forceinline__ float pair_geom(const char* __restrict__ st, uint32_t off, double xi,
                                           double yi, double zi, bool nx, bool ny, bool nz,
                                           const pc_box& b, const TileForceParams& p, double& dx,
                                           double& dy, double& dz, bool& overlap) {
  const double* q = reinterpret_cast<const double*>(st + off);
  dx = __dsub_rn(q[0], xi);
  dy = __dsub_rn(q[kStageStride], yi);
  dz = __dsub_rn(q[2 * kStageStride], zi);
  if (MI) {
    if (nx) dx = min_image_wrapped(dx, b.length[0], b.mi_thresh[0]);
    if (ny) dy = min_image_wrapped(dy, b.length[1], b.mi_thresh[1]);
    if (nz) dz = min_image_wrapped(dz, b.length[2], b.mi_thresh[2]);
  }
  const double r2 = r2_exact(dx, dy, dz);
  overlap |= r2 < p.overlap2;
  return r2 < p.cutoff2 ? d2f_fast(r2) : 1e30f;
}

template <bool MI, bool UNIT_SIGMA>
__device__ __forceinline__ void tile_pair2(const char* __restrict__ st, uint32_t w, double xi,
                                           double yi, double zi, bool nx, bool ny, bool nz,
                                           const pc_box& b, const TileForceParams& p,
                                           double& fx, double& fy, double& fz, f32x2_t& su2,
                                           f32x2_t& s62, bool& overlap) {
  double dxa, dya, dza, dxb, dyb, dzb;
  const float ra = pair_geom<MI>(st, w & 0xFFFFu, xi, yi, zi, nx, ny, nz, b, p, dxa, dya, dza,
                                 overlap);
  const float rb = pair_geom<MI>(st, w >> 16, xi, yi, zi, nx, ny, nz, b, p, dxb, dyb, dzb,
                                 overlap);
  const f32x2_t inv = pk2(rcp_approx(ra), rcp_approx(rb));
  const f32x2_t sr2 = UNIT_SIGMA ? inv : mul2(pk2(p.sig2, p.sig2), inv);
  const f32x2_t sr6 = mul2(mul2(sr2, sr2), sr2);
#if PC_FORCE_HALFU
  // h = u / 2 = sr6 (sr6 - 1/2), fm / 2 = h / r^2: the halves of the r01
  // terms bit for bit (fl(2 sr6 - 1) = 2 fl(sr6 - 1/2); scaling by 2 is
  // exact), one FADD2 with an immediate instead of a materialised 2.0 and an
  // FFMA2; tile_row2 doubles the row's sums and force (exact)
  const f32x2_t u = mul2(sr6, add2(sr6, pk2(-0.5f, -0.5f)));
#else
  // u = 2 sr12 - sr6 = sr6 (2 sr6 - 1) (pair virial); fm = u / r^2
  const f32x2_t u = mul2(sr6, fma2(pk2(2.0f, 2.0f), sr6, pk2(-1.0f, -1.0f)));
#endif
  const f32x2_t fm = mul2(u, inv);
  su2 = add2(su2, u);
  s62 = add2(s62, sr6);
  float fa, fb;
  upk2(fm, fa, fb);
  const double fda = (double)fa, fdb = (double)fb;
  fx = fma(-fda, dxa, fx);
  fy = fma(-fda, dya, fy);
  fz = fma(-fda, dza, fz);
  fx = fma(-fdb, dxb, fx);
  fy = fma(-fdb, dyb, fy);
  fz = fma(-fdb, dzb, fz);
}

#ifndef PC_FORCE_PACKED
#define PC_FORCE_PACKED 1       // FP32 LJ terms of two pairs as f32x2 (FFMA2/FMUL2/FADD2)
#endif

template <bool MI, bool UNIT_SIGMA, int B>
__device__ __forceinline__ void tile_row2(const char* __restrict__ st_rt,
                                          const uint4* __restrict__ lp, uint4 first, int R,
                                          double xi, double yi, double zi, bool nx, bool ny,
                                          bool nz, const pc_box& b, const TileForceParams& p,
                                          double& fx, double& fy, double& fz, float& su,
                                          float& s6, bool& overlap) {
  const char* __restrict__ st =
      B >= 0 ? reinterpret_cast<const char*>(pc_force_dyn) + (size_t)B * 3 * kStageStride * 8
             : st_rt;
  const int G = R >> 3;
  const int tail = R & 7;
  f32x2_t su2 = 0ull, s62 = 0ull;   // (+0.0f, +0.0f)
  uint4 nxt = first;
  for (int gi = 0; gi < G; ++gi) {
    const uint4 q = nxt;
    if (gi + 1 < G || tail) nxt = ld_stream(lp + (gi + 1) * 32);
    if (PC_FORCE_PREFETCH && gi + PC_FORCE_PFDIST < G) prefetch_l2(lp + (gi + PC_FORCE_PFDIST) * 32);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int h = 0; h < 4; ++h)
      tile_pair2<MI, UNIT_SIGMA>(st, w[h], xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, su2, s62,
                                 overlap);
  }
  // open group: pairs in twos (an odd tail's partner is a padding dummy:
  // far and NaN-free, it adds exactly 0)
  for (int j = 0; j < tail; j += 2) {
    const uint32_t w = (j >> 1) == 0 ? nxt.x : ((j >> 1) == 1 ? nxt.y : ((j >> 1) == 2 ? nxt.z : nxt.w));
    tile_pair2<MI, UNIT_SIGMA>(st, w, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, su2, s62,
                               overlap);
  }
  float a0, a1, c0, c1;
  upk2(su2, a0, a1);
  upk2(s62, c0, c1);
  su = a0 + a1;
  s6 = c0 + c1;
#if PC_FORCE_HALFU
  su *= 2.0f;
  fx *= 2.0;
  fy *= 2.0;
  fz *= 2.0;
#endif
}

template <bool MI, bool UNIT_SIGMA, int B>
__device__ __forceinline__ void tile_row(const char* __restrict__ st_rt,
                                         const uint4* __restrict__ lp, uint4 first, int R,
                                         double xi, double yi, double zi, bool nx, bool ny,
                                         bool nz, const pc_box& b, const TileForceParams& p,
                                         double& fx, double& fy, double& fz, float& su,
                                         float& s6, bool& overlap) {
  // B >= 0: buffer B at a compile-time offset of the dynamic shared window
  const char* __restrict__ st =
      B >= 0 ? reinterpret_cast<const char*>(pc_force_dyn) + (size_t)B * 3 * kStageStride * 8
             : st_rt;
  const int G = R >> 3;           // full 8-round groups
  const int tail = R & 7;         // rounds of the open group (padded with dummies: skipped)
  uint4 nxt = first;
  for (int gi = 0; gi < G; ++gi) {
    const uint4 q = nxt;
    if (gi + 1 < G || tail) nxt = ld_stream(lp + (gi + 1) * 32);
    // the group after next into L2 (no register: the list streams from HBM
    // at ~1 us latency, one group of compute ahead is not always enough)
    if (PC_FORCE_PREFETCH && gi + PC_FORCE_PFDIST < G) prefetch_l2(lp + (gi + PC_FORCE_PFDIST) * 32);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      tile_pair<MI, UNIT_SIGMA>(st, w[h] & 0xFFFFu, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz,
                                su, s6, overlap);
      tile_pair<MI, UNIT_SIGMA>(st, w[h] >> 16, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, su,
                                s6, overlap);
    }
  }
  // open group: pairs in twos (warp-uniform count)
  for (int j = 0; j < tail; j += 2) {
    const uint32_t w = (j >> 1) == 0 ? nxt.x : ((j >> 1) == 1 ? nxt.y : ((j >> 1) == 2 ? nxt.z : nxt.w));
    tile_pair<MI, UNIT_SIGMA>(st, w & 0xFFFFu, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, su,
                              s6, overlap);
    if (j + 1 < tail)
      tile_pair<MI, UNIT_SIGMA>(st, w >> 16, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, su, s6,
                                overlap);
  }
}

// whole warp: stage tile sequence k of this CTA into buffer b
__device__ __forceinline__ void force_load(ForceShared& F, double* __restrict__ stage, int b,
                                           int k, const int* __restrict__ plan,
                                           const double* __restrict__ pl, int64_t ps, int lane,
                                           const uint4* __restrict__ list,
                                           const int* __restrict__ rowidx, int Q8) {
  const int tile = tile_at(F.tiles, F.t0, k);
  const int* gp = plan + (int64_t)tile * kPlanInts;
  const int m = gp[0], S = gp[1];
  double* st = stage + (int64_t)b * 3 * kStageStride;
  uint64_t* bar = &F.bar[b];
  if (lane == 0) {
    F.done[b] = 0;
    F.par[b] = F.uses[b] & 1;
    F.uses[b] += 1;
    mbar_expect_tx(bar, (uint32_t)S * 24u);
  }
  __syncwarp();
  for (int e = lane; e < m; e += 32) {
    const int src = gp[4 + 3 * e], len = gp[5 + 3 * e], dst = gp[6 + 3 * e];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      bulk_g2s(st + a * kStageStride + dst, pl + a * ps + src, (uint32_t)len * 8u, bar);
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    F.seq[b] = k;
  }
}

template <bool UNIT_SIGMA>
__global__ void __launch_bounds__(kForceWarps * 32, 1)
tile_force_kernel(const double* __restrict__ pl, TileForceParams p, int ntiles,
                  const int* __restrict__ plan, const int* __restrict__ rowidx,
                  const int* __restrict__ rounds, const uint4* __restrict__ list, pc_box b,
                  double* __restrict__ f3, int64_t fs, double* __restrict__ v, int64_t vs,
                  double dtm, double mass, double* __restrict__ partial, int* __restrict__ flag,
                  int nbuf, double* __restrict__ x_next, double* __restrict__ v_next,
                  double dtm_next, double dt, double* __restrict__ virial,
                  const int* __restrict__ tiles, const int* __restrict__ trange) {
  double* dyn = pc_force_dyn;
  double* stage = dyn;                                             // nbuf x (x|y|z)
  __shared__ ForceShared F;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // all tiles, or the subset tiles[trange[0] .. trange[1]) (interior /
  // boundary passes of a decomposed domain; `ntiles` is then the bound the
  // grid and the shared memory were sized for)
  int t0 = 0, nt = ntiles;
  if (tiles) {
    t0 = trange[0];
    nt = trange[1] - t0;
  }
  const int K = max(0, (nt - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x);
  int* pre = reinterpret_cast<int*>(dyn + nbuf * 3 * kStageStride);    // K + 1 item prefix
  int* rwbk = pre + K + 1;                                              // first row-warp per k
  if (warp == 0) {
    // row-warp prefix over this CTA's tiles
    int carry = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int k = k0 + lane;
      const int* gpk = plan + (int64_t)(k < K ? tile_at(tiles, t0, k) : 0) * kPlanInts;
      const int c = k < K ? gpk[2] : 0;
      if (k < K) rwbk[k] = gpk[3];
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
      F.tiles = tiles;
      F.t0 = t0;
      F.next_item = 0;
      for (int q = 0; q < kNBuf; ++q) {
        F.seq[q] = -1;
        F.uses[q] = 0;
        mbar_init(&F.bar[q], 1);
      }
      F.loaded = min(K, nbuf);
    }
    __syncwarp();
    for (int q = 0; q < min(K, nbuf); ++q) force_load(F, stage, q, q, plan, pl, p.ps, lane, list, rowidx, p.Q8);
  } else if (warp == 1) {
    for (int q = 0; q < nbuf; ++q)
      if (lane < kNDummy)
        for (int a = 0; a < 3; ++a) stage[(q * 3 + a) * kStageStride + kStageCap + lane] = 1e30;
  }
  __syncthreads();
  const int items = F.items;
  double ake = 0.0, ape = 0.0, apx = 0.0, apy = 0.0, apz = 0.0;   // this lane's rows
  double avir = 0.0;

  // tile sequence index and global row-warp of item i (pre is ascending; K is small)
  auto locate = [&](int i, int& k) -> int {
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= i) lo = mid; else hi = mid - 1;
    }
    k = lo;
    return rwbk[lo] + (i - pre[lo]);
  };
  for (;;) {
    int i = 0;
    if (lane == 0) i = atomicAdd(&F.next_item, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= items) break;
    int k;
    const int rw = locate(i, k);
    const int a = rowidx[(int64_t)rw * 32 + lane];
    // prefetch everything that does not depend on the staged tile
    const int R = rounds[rw];
    const uint4* lp = list + (int64_t)rw * p.Q8 * 32 + lane;
    const uint4 first = R > 0 ? ld_stream(lp) : make_uint4(0u, 0u, 0u, 0u);
    const bool act = a >= 0;
    double xi = 0.0, yi = 0.0, zi = 0.0;
    if (act) {
      xi = pl[a];
      yi = pl[p.ps + a];
      zi = pl[2 * p.ps + a];
      if (PC_FORCE_PREFETCH && v) {  // the epilogue's velocities: into L2 now, read after the rounds
        prefetch_l2(v + a);
        prefetch_l2(v + vs + a);
        prefetch_l2(v + 2 * vs + a);
      }
    }
    // buffer holding tile k (loaded in ticket order; spin until published)
    int bsel = -1;
    for (;;) {
#pragma unroll
      for (int q = 0; q < kNBuf; ++q)
        if (F.seq[q] == k) bsel = q;
      if (bsel >= 0) break;
      __nanosleep(PC_FORCE_SLEEP);
    }
    __threadfence_block();
    mbar_wait(&F.bar[bsel], (uint32_t)F.par[bsel]);
    const char* st = reinterpret_cast<const char*>(stage + (int64_t)bsel * 3 * kStageStride);

#if PC_FORCE_MIU
    const bool nx = __any_sync(0xffffffffu, act && b.periodic[0] &&
                               (xi - b.low[0] < p.guard || b.high[0] - xi <= p.guard));
    const bool ny = __any_sync(0xffffffffu, act && b.periodic[1] &&
                               (yi - b.low[1] < p.guard || b.high[1] - yi <= p.guard));
#else
    const bool nx = act && b.periodic[0] && (xi - b.low[0] < p.guard || b.high[0] - xi <= p.guard);
    const bool ny = act && b.periodic[1] && (yi - b.low[1] < p.guard || b.high[1] - yi <= p.guard);
#endif
#if PC_FORCE_MIU
    // warp-uniform axis flags: the minimum image is exact for every pair of a
    // staged (wrapped) neighbourhood, so lanes away from the face may take it
    // too, and the per-axis branches of the minimum-image body stay uniform
    const bool nz = __any_sync(0xffffffffu, act && b.periodic[2] &&
                               (zi - b.low[2] < p.guard || b.high[2] - zi <= p.guard));
#else
    const bool nz = act && b.periodic[2] && (zi - b.low[2] < p.guard || b.high[2] - zi <= p.guard);
#endif
    double fx = 0.0, fy = 0.0, fz = 0.0;
    float su = 0.f, s6 = 0.f;
    bool overlap = false;
    const bool mi = __any_sync(0xffffffffu, nx || ny || nz);
#if PC_FORCE_PACKED
#define PC_ROWFN tile_row2
#else
#define PC_ROWFN tile_row
#endif
#define PC_ROW(BB)                                                                            \
  if (mi)                                                                                     \
    PC_ROWFN<true, UNIT_SIGMA, BB>(st, lp, first, R, xi, yi, zi, nx, ny, nz, b, p, fx, fy, fz, \
                                   su, s6, overlap);                                          \
  else                                                                                        \
    PC_ROWFN<false, UNIT_SIGMA, BB>(st, lp, first, R, xi, yi, zi, nx, ny, nz, b, p, fx, fy,   \
                                    fz, su, s6, overlap);
    PC_ROW(-1)
#undef PC_ROW
    // release the buffer when this was the tile's last row-warp; refill it
    int last = 0;
    if (lane == 0) last = atomicAdd(&F.done[bsel], 1) + 1 == pre[k + 1] - pre[k];
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      int kn = 0;
      if (lane == 0) {
        F.seq[bsel] = -1;
        kn = atomicAdd(&F.loaded, 1);
      }
      kn = __shfl_sync(0xffffffffu, kn, 0);
      if (kn < K) force_load(F, stage, bsel, kn, plan, pl, p.ps, lane, list, rowidx, p.Q8);
    }
    if (overlap) atomicOr(flag, kFlagOverlap);
    double ke = 0.0, px = 0.0, py = 0.0, pz = 0.0, ped = 0.0;
    if (act) {
      fx *= p.eps24d;
      fy *= p.eps24d;
      fz *= p.eps24d;
      // row energy 2 eps (sum sr12 - sr6) = eps (sum u - sum sr6); row
      // virial sum_j r.F / 2 = 12 eps sum u (both halves of each pair)
      ped = ((double)su - (double)s6) * p.eps2d * 0.5;
      avir += (double)su * p.eps24d * 0.5;
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
  if (virial) {
    avir = warp_sum(avir);
    // column 0 of a (partials, 5) zero-initialised array: pc_reduce_partials sums it
    if (lane == 0) virial[((int64_t)blockIdx.x * kForceWarps + warp) * 5] = avir;
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
#ifndef PC_ORDER_PREFETCH
#define PC_ORDER_PREFETCH 1
#endif
constexpr int kOrdSmem = kOrdWarps * ((kHitCap + 1) * 32 * 2 + 16 * 32 * 4);

// Residue round-robin order, r02 rewrite (PC_TILE_ORDER_IMPL=1 keeps the r01
// kernel below): the same rounds bit for bit, fewer instructions per entry.
// Groups of eight rounds that hold only real entries in every lane (below
// the warp's shortest row) take paths without the real / padding selects;
// the non-empty-class mask is derived from the counts and kept doubled
// (bits c and c + 16), so the preferred rotation is one shift.
__global__ void __launch_bounds__(kOrdWarps * 32, 3)
tile_order_rr_kernel(uint4* __restrict__ list, const int* __restrict__ rounds,
                     const int* __restrict__ rw_total, int Q8, int dummy0) {
  extern __shared__ __align__(16) unsigned char osm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = blockIdx.x * kOrdWarps + warp;
  if (rw >= *rw_total) return;
  uint32_t* st = reinterpret_cast<uint32_t*>(osm) + warp * 16 * 32 + lane;   // [c][lane]
  uint16_t* Bm = reinterpret_cast<uint16_t*>(osm + kOrdWarps * 16 * 32 * 4) +
                 warp * (kHitCap + 1) * 32 + lane;    // [k][lane], row kHitCap: dump
  const int R = rounds[rw];
  if (R <= 0 || R > kHitCap) return;
  uint4* lp = list + (int64_t)rw * Q8 * 32 + lane;
  const uint32_t dmin = (uint32_t)dummy0 * 8u;
  const int G = (R + 7) >> 3;
#pragma unroll
  for (int c = 0; c < 16; ++c) st[c * 32] = 0u;
  int cnt = 0;                                          // real entries precede padding
  // the first read of the list comes from HBM: two groups in flight
  uint4 qn = lp[0], qn2 = G > 1 ? lp[32] : make_uint4(0u, 0u, 0u, 0u);
  for (int g = 0; g < G; ++g) {                         // per-class counts
    const uint4 q = qn;
    qn = qn2;
    if (g + 2 < G) qn2 = lp[(g + 2) * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      const uint32_t real = v < dmin ? 1u : 0u;
      st[((v >> 3) & 15) * 32] += real;
      cnt += (int)real;
    }
  }
  const int gfull = __reduce_min_sync(0xffffffffu, cnt) >> 3;   // groups real in every lane
  uint32_t run = 0u, ne = 0u;
#pragma unroll
  for (int c = 0; c < 16; ++c) {                        // next | end << 16
    const uint32_t n = st[c * 32];
    st[c * 32] = run | ((run + n) << 16);
    ne |= n ? (1u << c) : 0u;
    run += n;
  }
  qn = lp[0];
  for (int g = 0; g < G; ++g) {                         // class-major scatter -> Bm
    const uint4 q = qn;
    if (g + 1 < G) qn = lp[(g + 1) * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    if (g < gfull) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
        uint32_t* sc = st + ((v >> 3) & 15) * 32;
        const uint32_t e = *sc;
        *sc = e + 1u;
        Bm[(e & 0xFFFFu) * 32] = (uint16_t)v;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
        const bool real = v < dmin;
        uint32_t* sc = st + ((v >> 3) & 15) * 32;
        const uint32_t e = *sc;
        *sc = e + (real ? 1u : 0u);
        Bm[(real ? (int)(e & 0xFFFFu) : kHitCap) * 32] = (uint16_t)v;
      }
    }
  }
  uint32_t beg = 0u;                                    // rewind next to begin(c) = end(c - 1)
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint32_t end = st[c * 32] >> 16;
    st[c * 32] = beg | (end << 16);
    beg = end;
  }
  uint32_t ne2 = ne | (ne << 16);                       // doubled: rotation = one shift
  for (int g = 0; g < G; ++g) {                         // emit 8 rounds per uint4
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    const int base = lane + g * 8;
    if (g < gfull) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        // in round r lane l prefers residue (l + r) % 16, else the next
        // non-empty one
        const int pref = (base + t) & 15;
        const int c = (pref + __ffs(ne2 >> pref) - 1) & 15;
        uint32_t* sc = st + c * 32;
        const uint32_t e = *sc;
        const uint32_t pos = e & 0xFFFFu;
        *sc = e + 1u;
        if (pos + 1u == (e >> 16)) ne2 &= ~(0x10001u << c);
        const uint32_t v = Bm[pos * 32];
        o[t >> 1] |= (t & 1) ? (v << 16) : v;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int r = g * 8 + t;
        const bool real = r < cnt;
        const int pref = (base + t) & 15;
        const int c = (pref + __ffs(ne2 >> pref) - 1) & 15;
        uint32_t* sc = st + c * 32;
        const uint32_t e = *sc;
        const uint32_t pos = e & 0xFFFFu;
        *sc = e + (real ? 1u : 0u);
        if (real && pos + 1u == (e >> 16)) ne2 &= ~(0x10001u << c);
        const uint32_t vb = Bm[(real ? (int)pos : kHitCap) * 32];
        const uint32_t v = real ? vb : (uint32_t)(dummy0 + ((lane + r) & 15)) * 8u;
        o[t >> 1] |= (t & 1) ? (v << 16) : v;
      }
    }
    lp[g * 32] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// RR = false: class-major with the start rotated to the lane's residue (the
// cheaper variant, simulated 1.9 passes per half-warp).  Per-class state
// lives in a per-lane shared table st[c][lane] (conflict-free: bank = lane).
template <bool RR>
__global__ void __launch_bounds__(kOrdWarps * 32, 3)
tile_order_kernel(uint4* __restrict__ list, const int* __restrict__ rounds,
                  const int* __restrict__ rw_total, int Q8, int dummy0) {
  extern __shared__ __align__(16) unsigned char osm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = blockIdx.x * kOrdWarps + warp;
  if (rw >= *rw_total) return;
  uint32_t* st = reinterpret_cast<uint32_t*>(osm) + warp * 16 * 32 + lane;   // [c][lane]
  uint16_t* Bm = reinterpret_cast<uint16_t*>(osm + kOrdWarps * 16 * 32 * 4) +
                 warp * (kHitCap + 1) * 32 + lane;    // [k][lane], row kHitCap: dump
  const int R = rounds[rw];
  if (R <= 0 || R > kHitCap) return;
  uint4* lp = list + (int64_t)rw * Q8 * 32 + lane;
  const uint32_t dmin = (uint32_t)dummy0 * 8u;
  const int G = (R + 7) >> 3;
#pragma unroll
  for (int c = 0; c < 16; ++c) st[c * 32] = 0u;
  int cnt = 0;                                          // real entries precede padding
  // list groups are loaded one ahead in both passes (the first use of each
  // group stalled on its load: ~26 % of the kernel's stall samples, r02c)
  uint4 qn = lp[0];
  for (int g = 0; g < G; ++g) {                         // per-class counts
    const uint4 q = PC_ORDER_PREFETCH ? qn : lp[g * 32];
    if (PC_ORDER_PREFETCH && g + 1 < G) qn = lp[(g + 1) * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      // branch-free: a padding entry (v >= dmin; the groups past R are
      // padding too) adds 0 to its residue's count
      const uint32_t real = v < dmin ? 1u : 0u;
      uint32_t* sc = st + ((v >> 3) & 15) * 32;
      *sc += real;
      cnt += (int)real;
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
  qn = lp[0];
  for (int g = 0; g < G; ++g) {                         // class-major scatter -> smem
    const uint4 q = PC_ORDER_PREFETCH ? qn : lp[g * 32];
    if (PC_ORDER_PREFETCH && g + 1 < G) qn = lp[(g + 1) * 32];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t v = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
      // branch-free: padding entries leave the state and land in the dump row
      const bool real = v < dmin;
      const int c = (v >> 3) & 15;
      uint32_t* sc = st + c * 32;
      const uint32_t e = *sc;
      *sc = e + (real ? 1u : 0u);
      int pos = (int)(e & 0xFFFFu);
      if (RR) ne |= real ? 1u << c : 0u;
      else { pos -= s0; if (pos < 0) pos += cnt; }
      Bm[(real ? pos : kHitCap) * 32] = (uint16_t)v;
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
      const bool real = r < cnt;
      int pos = r;
      if (RR) {
        // in round r lane l prefers residue (l + r) % 16, else the next
        // non-empty one (branch-free: past cnt the state is left unchanged)
        const int pref = (lane + r) & 15;
        const unsigned rot = ((ne >> pref) | (ne << (16 - pref))) & 0xFFFFu;
        const int c = (pref + __ffs(rot) - 1) & 15;
        uint32_t* sc = st + c * 32;
        const uint32_t e = *sc;
        pos = (int)(e & 0xFFFFu);
        *sc = e + (real ? 1u : 0u);
        if (real && (uint32_t)pos + 1u == (e >> 16)) ne &= ~(1u << c);
      }
      const uint32_t vb = Bm[(real ? pos : kHitCap) * 32];
      const uint32_t v = real ? vb : (uint32_t)(dummy0 + ((lane + r) & 15)) * 8u;
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
      const int s = lp[(r >> 3) * 32 * 8 + (r & 7)] >> 3;
      if (s >= max_stage) continue;
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

int pc_cell_zsort(const double* d_z, int64_t z_stride, const int32_t* d_cell_start,
                  int32_t ncells, const int32_t* d_order, int32_t* d_out, void* stream) {
  if (ncells <= 0) return PC_OK;
  cell_zsort_kernel<<<(ncells + 7) / 8, 256, 0, as_stream(stream)>>>(d_z, z_stride, d_cell_start,
                                                                     ncells, d_order, d_out);
  return check_launch("pc_cell_zsort");
}

int pc_tile_rows(const int32_t* d_cell_start, const pc_grid* grid, int32_t* d_rw, void* stream) {
  return pc_tile_rows_domain(d_cell_start, grid, nullptr, d_rw, stream);
}

int pc_tile_rows_domain(const int32_t* d_cell_start, const pc_grid* grid, const int32_t* d_skip,
                        int32_t* d_rw, void* stream) {
  const int nt = tile_dims(*grid).ntiles;
  if (nt <= 0) return PC_OK;
  tile_rows_kernel<<<(nt + 7) / 8, 256, 0, as_stream(stream)>>>(d_cell_start, *grid, d_rw,
                                                                 d_skip);
  return check_launch("pc_tile_rows_domain");
}

int pc_tile_build(const double* d_planar, int64_t planar_stride, const int32_t* d_cell_start,
                  const pc_grid* grid, const pc_box* box, double cutoff2, int32_t q8,
                  const int32_t* d_rw0, int32_t* d_plan, int32_t* d_rowidx, int32_t* d_rounds,
                  void* d_list, int32_t* d_flag, void* stream) {
  return pc_tile_build_domain(d_planar, planar_stride, d_cell_start, grid, box, cutoff2, q8,
                              d_rw0, d_plan, d_rowidx, d_rounds, d_list, d_flag, stream,
                              nullptr, nullptr, nullptr, nullptr);
}

int pc_tile_build_domain(const double* d_planar, int64_t planar_stride,
                         const int32_t* d_cell_start, const pc_grid* grid, const pc_box* box,
                         double cutoff2, int32_t q8, const int32_t* d_rw0, int32_t* d_plan,
                         int32_t* d_rowidx, int32_t* d_rounds, void* d_list, int32_t* d_flag,
                         void* stream, const double* d_bplanar, const pc_box* box_exact,
                         const int32_t* d_skip, int32_t* d_tile_ghost) {
  return pc_tile_build_ordered(d_planar, planar_stride, d_cell_start, grid, box, cutoff2, q8,
                               d_rw0, d_plan, d_rowidx, d_rounds, d_list, d_flag, stream,
                               d_bplanar, box_exact, d_skip, d_tile_ghost, 0);
}

int pc_tile_build_ordered(const double* d_planar, int64_t planar_stride,
                          const int32_t* d_cell_start, const pc_grid* grid, const pc_box* box,
                          double cutoff2, int32_t q8, const int32_t* d_rw0, int32_t* d_plan,
                          int32_t* d_rowidx, int32_t* d_rounds, void* d_list, int32_t* d_flag,
                          void* stream, const double* d_bplanar, const pc_box* box_exact,
                          const int32_t* d_skip, int32_t* d_tile_ghost, int32_t order_kind) {
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
  p.sched = getenv("PC_TILE_SCHED") ? atoi(getenv("PC_TILE_SCHED")) : 3;
  p.ps = planar_stride;
  const int nt = tile_dims(*grid).ntiles;
  {
    // order_kind 1: the residue round-robin order fused into the build
    // (tile_build_kernel<true>); 0: the build's ascending order
    const bool ord = order_kind == 1;
    const int bw = build_warps(ord);
    const int smem = kStageCap * (int)sizeof(float4) +
                     bw * 32 * (kHitCap + kHitSlack) * (int)sizeof(uint16_t) +
                     (ord ? bw * 16 * 32 * (int)sizeof(uint16_t) : 0);
    if (smem > g_build_smem) {
      if (cudaFuncSetAttribute(tile_build_kernel<false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
          cudaFuncSetAttribute(tile_build_kernel<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        set_error("pc_tile_build: %d B of shared memory not available", smem);
        return PC_ERR_CAPACITY;
      }
      g_build_smem = smem;
    }
    auto kern = ord ? tile_build_kernel<true> : tile_build_kernel<false>;
    kern<<<nt, bw * 32, smem, as_stream(stream)>>>(
        d_planar, d_cell_start, *grid, *box, p, d_rw0, d_plan, d_rowidx, d_rounds,
        reinterpret_cast<uint4*>(d_list), d_flag, d_bplanar ? d_bplanar : d_planar,
        box_exact ? *box_exact : *box, d_skip, d_tile_ghost);
    return check_launch("pc_tile_build");
  }
}

int pc_tile_force(const double* d_planar, int64_t planar_stride, int32_t ntiles,
                  const int32_t* d_plan, const int32_t* d_rowidx, const int32_t* d_rounds,
                  const void* d_list, int32_t q8, const pc_box* box, const pc_lj* lj,
                  double mi_guard, double* d_f3, int64_t f_stride, double* d_v, int64_t v_stride,
                  double dtm, double mass, double* d_partial, int32_t* d_flag,
                  double* d_planar_next, double* d_v_next, double dtm_next, double dt,
                  double* d_virial, const int32_t* d_tiles, const int32_t* d_trange,
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
  // as many staging buffers as fit next to the item prefix (2..kNBuf)
  static int smem_max = 0;
  if (smem_max == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem_max <= 0) smem_max = 227 * 1024;
  }
  const int buf_bytes = 3 * kStageStride * (int)sizeof(double);
  const int pre_bytes = (2 * K + 1) * (int)sizeof(int);
  const int static_bytes = (int)sizeof(ForceShared) + 256;
  int nbuf = kNBuf;
  while (nbuf > 2 && nbuf * buf_bytes + pre_bytes + static_bytes > smem_max) --nbuf;
  const int smem = nbuf * buf_bytes + pre_bytes + K * (int)sizeof(int);
  if (smem + static_bytes > smem_max) {
    set_error("pc_tile_force: %d tiles per CTA do not fit in shared memory", K);
    return PC_ERR_CAPACITY;
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
        *box, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial, d_flag, nbuf, d_planar_next,
        d_v_next, dtm_next, dt, d_virial, d_tiles, d_trange);
  else
    tile_force_kernel<false><<<grid, kForceWarps * 32, smem, as_stream(stream)>>>(
        d_planar, p, ntiles, d_plan, d_rowidx, d_rounds, reinterpret_cast<const uint4*>(d_list),
        *box, d_f3, f_stride, d_v, v_stride, dtm, mass, d_partial, d_flag, nbuf, d_planar_next,
        d_v_next, dtm_next, dt, d_virial, d_tiles, d_trange);
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
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(tile_order_rr_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
      set_error("pc_tile_order: %d B of shared memory not available", smem);
      return PC_ERR_CAPACITY;
    }
    set = 1;
  }
  const int grid = (rw_bound + kOrdWarps - 1) / kOrdWarps;
  uint4* l = reinterpret_cast<uint4*>(d_list);
  static const int impl = getenv("PC_TILE_ORDER_IMPL") ? atoi(getenv("PC_TILE_ORDER_IMPL")) : 2;
  if (kind == 1 && impl == 2)
    tile_order_rr_kernel<<<grid, kOrdWarps * 32, smem, as_stream(stream)>>>(
        l, d_rounds, d_rw_total, q8, kStageCap);
  else if (kind == 1)
    tile_order_kernel<true><<<grid, kOrdWarps * 32, smem, as_stream(stream)>>>(
        l, d_rounds, d_rw_total, q8, kStageCap);
  else
    tile_order_kernel<false><<<grid, kOrdWarps * 32, smem, as_stream(stream)>>>(
        l, d_rounds, d_rw_total, q8, kStageCap);
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
