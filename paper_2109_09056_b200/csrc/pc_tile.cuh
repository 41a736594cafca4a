// Tile geometry shared by the tile Verlet build and the tile force kernel.
//
// A tile is a segment of kTileZ consecutive cells along z in one (x, y)
// column of the linked-cell grid; its home particles are one contiguous index
// range after the cell sort.  Its staged neighbourhood is the 9 stencil
// columns x (kTileZ + 2) cells (z0-1 .. z1), enumerated column by column and
// cell by cell; a particle's position in that enumeration is its "slot".
// Both kernels derive the identical slot numbering from cell_start, so the
// build can store 16-bit slots and the force kernel can resolve them in
// shared memory.
#pragma once

#include "pc_common.cuh"

namespace pc {

constexpr int kTileZ = 4;
constexpr int kTileCells = kTileZ + 2;
constexpr int kTileCols = 9;

struct TileTable {
  int off[kTileCols][kTileCells + 1];   // staged offset of each cell, [c][k+1] = end
  int src[kTileCols][kTileCells];       // first global index of each staged cell
  double shift[kTileCols][kTileCells][3];
  int total;
  int home_first;                       // global index of the first home particle
  int nhome;
  int nzh;                              // home cells in this tile
};

__device__ __forceinline__ void tile_coords(int tile, const pc_grid& g, int& cx, int& cy,
                                            int& z0, int& z1) {
  const int nseg = (g.nc[2] + kTileZ - 1) / kTileZ;
  const int col = tile / nseg;
  const int seg = tile - col * nseg;
  cx = col / g.nc[1];
  cy = col - cx * g.nc[1];
  z0 = seg * kTileZ;
  z1 = min(z0 + kTileZ, g.nc[2]);
}

// Fill `t` (shared) for tile `tile`; call with all threads, contains barriers.
__device__ void tile_table(int tile, const pc_grid& g, const pc_box& b,
                           const int* __restrict__ cell_start, TileTable& t) {
  int cx, cy, z0, z1;
  tile_coords(tile, g, cx, cy, z0, z1);
  const int nz = z1 - z0 + 2;
  for (int e = threadIdx.x; e < kTileCols * kTileCells; e += blockDim.x) {
    const int c = e / kTileCells, k = e - c * kTileCells;
    int xs = cx + c / 3 - 1, ys = cy + c % 3 - 1, zs = z0 - 1 + k;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    bool ok = k < nz;
    if (xs < 0) { if (b.periodic[0]) { xs += g.nc[0]; sx = -b.length[0]; } else ok = false; }
    if (xs >= g.nc[0]) { if (b.periodic[0]) { xs -= g.nc[0]; sx = b.length[0]; } else ok = false; }
    if (ys < 0) { if (b.periodic[1]) { ys += g.nc[1]; sy = -b.length[1]; } else ok = false; }
    if (ys >= g.nc[1]) { if (b.periodic[1]) { ys -= g.nc[1]; sy = b.length[1]; } else ok = false; }
    if (zs < 0) { if (b.periodic[2]) { zs += g.nc[2]; sz = -b.length[2]; } else ok = false; }
    if (zs >= g.nc[2]) { if (b.periodic[2]) { zs -= g.nc[2]; sz = b.length[2]; } else ok = false; }
    int cnt = 0, src = 0;
    if (ok) {
      const int cell = (xs * g.nc[1] + ys) * g.nc[2] + zs;
      src = cell_start[cell];
      cnt = cell_start[cell + 1] - src;
    }
    t.src[c][k] = src;
    t.off[c][k + 1] = cnt;
    t.shift[c][k][0] = sx;
    t.shift[c][k][1] = sy;
    t.shift[c][k][2] = sz;
  }
  __syncthreads();
  if (threadIdx.x < 32) {   // warp scan over the 90 cell counts in enumeration order
    const int lane = threadIdx.x;
    int carry = 0;
    for (int base = 0; base < kTileCols * kTileCells; base += 32) {
      const int e = base + lane;
      const int c = e / kTileCells, k = e - c * kTileCells;
      const int v = e < kTileCols * kTileCells ? t.off[c][k + 1] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (e < kTileCols * kTileCells) {
        t.off[c][k + 1] = carry + inc;       // end of cell e
        if (k == 0) t.off[c][0] = carry + inc - v;
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      t.total = carry;
      t.home_first = t.src[4][1];
      t.nzh = z1 - z0;
      t.nhome = t.off[4][z1 - z0 + 1] - t.off[4][1];
    }
  }
  __syncthreads();
}

}  // namespace pc
