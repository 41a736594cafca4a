// Spatial decomposition kernels: ownership, halo export planning, shifted
// ghost staging and the reverse (scatter-add) halo.  Replace the numpy bodies
// of ref decomp.py:58-66 (owner_of), :115-228 (build_halo), :231-260
// (halo_gather staging) and :263-300 (halo_scatter).
#include "pc_common.cuh"

namespace pc {

constexpr int kMaxSlots = 26;

// One candidate image of a source rank's particles (ref decomp.py:164-194):
// destination slot, periodic shift and destination box.
struct HaloOffset {
  int slot;            // index of the destination among this rank's distinct dests
  double shift[3];
  double lo[3], hi[3];
};

struct HaloTable {
  int n_off;                       // offsets in product order (<= 26)
  int n_slots;                     // distinct destinations
  int d;                           // dimensionality
  int has_in;                      // in_lo / in_hi valid
  double w2;
  // interior box (selection only): a particle strictly inside it is farther
  // than the halo width from every other block, so it exports nothing
  double in_lo[3], in_hi[3];
  HaloOffset off[kMaxSlots];
};

// owner = ravel(min(floor((x - low) / bl), dims - 1)); outside the global
// box -> flag bit 0 (ValueError, ref decomp.py:62-63).
__global__ void owner_kernel(const double* __restrict__ x, int64_t n, int d, pc_grid g,
                             int* __restrict__ owner, int* __restrict__ flag,
                             const int* __restrict__ skip, int skip_owner) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (skip && skip[i]) {        // a ghost row: dropped by the migrate, no check
    owner[i] = skip_owner;
    return;
  }
  int c[3] = {0, 0, 0};
  bool outside = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {       // unrolled: no local copy of g
    if (a >= d) break;
    const double v = x[i * d + a];
    outside |= (v < g.low[a]) || (v > g.high[a]);
    double q = floor(__ddiv_rn(__dsub_rn(v, g.low[a]), g.width[a]));
    int ci = (int)q;
    if (q >= (double)g.nc[a]) ci = g.nc[a] - 1;
    if (!(q >= 0.0)) ci = 0;            // outside (flagged): keep the owner a valid rank
    c[a] = ci;
  }
  if (outside) atomicOr(flag, kFlagOutside);
  owner[i] = (c[0] * g.nc[1] + c[1]) * g.nc[2] + c[2];
}

// Non-periodic axis: wrapped position outside [low, high] -> flag bit 3
// (ref decomp.py:92-96).
__global__ void nonperiodic_check_kernel(const double* __restrict__ x, int64_t n, int d,
                                         pc_box b, int* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a >= d) break;
    if (b.periodic[a]) continue;
    const double v = x[i * d + a];
    if (v < b.low[a] || v > b.high[a]) atomicOr(flag, kFlagNonPeriodic);
  }
}

// Squared distance of x + shift to the closed box, einsum order (x^2+z^2)+y^2
// for d = 3 (ref decomp.py:115-120).
__device__ __forceinline__ double dist2_box(const double* x, const HaloOffset& o, int d) {
  double t[3] = {0.0, 0.0, 0.0};
  // unrolled over the 3 axes (a runtime bound put t[] in local memory: a
  // 48-B stack frame per thread in the halo selection kernels)
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a >= d) break;
    const double p = __dadd_rn(x[a], o.shift[a]);
    const double below = fmax(__dsub_rn(o.lo[a], p), 0.0);
    const double above = fmax(__dsub_rn(p, o.hi[a]), 0.0);
    const double s = __dadd_rn(below, above);
    t[a] = __dmul_rn(s, s);
  }
  if (d == 3) return __dadd_rn(__dadd_rn(t[0], t[2]), t[1]);
  if (d == 2) return __dadd_rn(t[0], t[1]);
  return t[0];
}

// Per particle: best image per destination (strict <, first offset in
// product order wins ties), export iff best d2 < w^2.  Writes flags[slot][i]
// (0/1 int32) and the winning offset per slot.
__global__ void halo_plan_kernel(const double* __restrict__ x, int64_t n, HaloTable t,
                                 int* __restrict__ flags, int8_t* __restrict__ best_off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xi[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < t.d; ++a) xi[a] = x[i * t.d + a];
  double best[kMaxSlots];
  int bo[kMaxSlots];
  for (int s = 0; s < t.n_slots; ++s) { best[s] = INFINITY; bo[s] = -1; }
  for (int k = 0; k < t.n_off; ++k) {
    const int s = t.off[k].slot;
    const double d2 = dist2_box(xi, t.off[k], t.d);
    if (bo[s] < 0 || d2 < best[s]) { best[s] = d2; bo[s] = k; }
  }
  for (int s = 0; s < t.n_slots; ++s) {
    flags[(int64_t)s * n + i] = best[s] < t.w2 ? 1 : 0;
    best_off[(int64_t)s * n + i] = (int8_t)bo[s];
  }
}

// ---- fused halo selection (decomposed MD engine) ----------------------------
// The export set of build_halo (ref decomp.py:143-228: best image per
// destination slot, export iff its d^2 < w^2, entries ordered by (slot,
// particle index)) in two passes over the particles, without the per-slot
// flag matrix: (1) per 1024-particle chunk and slot, the number of exported
// particles; (2) after a scan of those counts (slot-major, chunk-minor: the
// (slot, index) order), each particle writes its index and its ghost row
// (x, y, z, global-id bits, shift of the winning image) at its place.
constexpr int kSelChunk = 1024;

// winning image of slot q (strict <, first offset in product order wins)
__device__ __forceinline__ int halo_best_offset(const double* xi, const HaloTable& t, int q,
                                                double& best) {
  best = INFINITY;
  int bo = -1;
  for (int k = 0; k < t.n_off; ++k) {
    if (t.off[k].slot != q) continue;
    const double d2 = dist2_box(xi, t.off[k], t.d);
    if (bo < 0 || d2 < best) { best = d2; bo = k; }
  }
  return bo;
}

// export mask over slots; `ident`: slots 1:1 with offsets (one slot per image,
// the decomposed engine's layout) -- no per-slot minimum, no local arrays
__device__ __forceinline__ unsigned halo_select_mask(const double* xi, const HaloTable& t,
                                                     bool ident) {
  unsigned m = 0u;
  if (t.has_in && xi[0] > t.in_lo[0] && xi[0] < t.in_hi[0] && xi[1] > t.in_lo[1] &&
      xi[1] < t.in_hi[1] && xi[2] > t.in_lo[2] && xi[2] < t.in_hi[2])
    return 0u;                     // deep inside the own block (most particles)
  if (ident) {
    for (int k = 0; k < t.n_off; ++k)
      if (dist2_box(xi, t.off[k], t.d) < t.w2) m |= 1u << k;
  } else {
    for (int q = 0; q < t.n_slots; ++q) {
      double best;
      halo_best_offset(xi, t, q, best);
      if (best < t.w2) m |= 1u << q;
    }
  }
  return m;
}

__device__ __forceinline__ bool halo_ident(const HaloTable& t) {
  bool id = t.n_slots == t.n_off;
  for (int k = 0; k < t.n_off; ++k) id &= t.off[k].slot == k;
  return id;
}

__global__ void __launch_bounds__(kSelChunk)
halo_select_count_kernel(const double* __restrict__ pos4, int64_t n, HaloTable t, int nchunks,
                         int* __restrict__ hist) {
  __shared__ int h[kMaxSlots];
  if (threadIdx.x < kMaxSlots) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kSelChunk + threadIdx.x;
  unsigned m = 0u;
  if (i < n) {
    const double xi[3] = {pos4[i * 4], pos4[i * 4 + 1], pos4[i * 4 + 2]};
    m = halo_select_mask(xi, t, halo_ident(t));
  }
  const int lane = threadIdx.x & 31;
  const unsigned any = __reduce_or_sync(0xffffffffu, m);
  for (int q = 0; q < t.n_slots; ++q) {
    if (!((any >> q) & 1u)) continue;               // warp-uniform
    const unsigned b = __ballot_sync(0xffffffffu, (m >> q) & 1u);
    if (lane == 0) atomicAdd(&h[q], __popc(b));
  }
  __syncthreads();
  if (threadIdx.x < t.n_slots) hist[(int64_t)threadIdx.x * nchunks + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSelChunk)
halo_select_place_kernel(const double* __restrict__ pos4, int64_t n, HaloTable t, int nchunks,
                         const int* __restrict__ off, int* __restrict__ out_idx,
                         double* __restrict__ out_rows) {
  __shared__ int wc[kSelChunk / 32][kMaxSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kSelChunk + threadIdx.x;
  const bool ident = halo_ident(t);
  double xi[3] = {0.0, 0.0, 0.0};
  unsigned m = 0u;
  if (i < n) {
    xi[0] = pos4[i * 4];
    xi[1] = pos4[i * 4 + 1];
    xi[2] = pos4[i * 4 + 2];
    m = halo_select_mask(xi, t, ident);
  }
  const unsigned any = __reduce_or_sync(0xffffffffu, m);
  for (int q = lane; q < t.n_slots; q += 32) wc[warp][q] = 0;
  __syncwarp();
  for (int q = 0; q < t.n_slots; ++q) {
    if (!((any >> q) & 1u)) continue;
    const unsigned b = __ballot_sync(0xffffffffu, (m >> q) & 1u);
    if (lane == 0) wc[warp][q] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x < t.n_slots) {              // exclusive prefix over the warps, per slot
    int run = 0;
    for (int w = 0; w < kSelChunk / 32; ++w) {
      const int v = wc[w][threadIdx.x];
      wc[w][threadIdx.x] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int q = 0; q < t.n_slots; ++q) {
    if (!((any >> q) & 1u)) continue;
    const unsigned b = __ballot_sync(0xffffffffu, (m >> q) & 1u);
    if (!((m >> q) & 1u)) continue;
    const int64_t at = off[(int64_t)q * nchunks + blockIdx.x] + wc[warp][q] +
                       __popc(b & ((1u << lane) - 1u));
    double best;
    const int k = ident ? q : halo_best_offset(xi, t, q, best);
    out_idx[at] = (int)i;
    const HaloOffset& o = t.off[k];
    double* r = out_rows + at * 7;
    r[0] = xi[0];
    r[1] = xi[1];
    r[2] = xi[2];
    r[3] = pos4[i * 4 + 3];
    r[4] = o.shift[0];
    r[5] = o.shift[1];
    r[6] = o.shift[2];
  }
}

// ---- reverse halo of the half-list (Newton-3) MD engine --------------------
// ref decomp.py:263-300 (halo_scatter): ghost rows' accumulated forces go
// back to their owners.  Pack: buf[k] = f[:, rows[k]] (planar force, stride
// fs) and the ghost row's force is cleared (so the kick leaves ghost
// velocities at zero); add: f[:, rows[k]] += buf[k] with FP64 atomics (a
// particle exported as several images appears several times in `rows`).
__global__ void halo_force_pack_kernel(double* __restrict__ f, int64_t fs,
                                       const int* __restrict__ rows, int64_t m,
                                       double* __restrict__ buf) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t r = rows[k];
  for (int a = 0; a < 3; ++a) {
    buf[k * 3 + a] = f[a * fs + r];
    f[a * fs + r] = 0.0;
  }
}

__global__ void halo_force_add_kernel(double* __restrict__ f, int64_t fs,
                                      const int* __restrict__ rows, int64_t m,
                                      const double* __restrict__ buf) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t r = rows[k];
  for (int a = 0; a < 3; ++a) atomicAdd(f + a * fs + r, buf[k * 3 + a]);
}

// Stable compaction of one slot: idx[pos[i]] = i where flag[i].
__global__ void compact_kernel(const int* __restrict__ flag, const int* __restrict__ pos,
                               int64_t n, int* __restrict__ out_idx,
                               const int8_t* __restrict__ best_off, int8_t* __restrict__ out_off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  out_idx[pos[i]] = (int)i;
  out_off[pos[i]] = best_off[i];
}

// dst[k] = src[idx[k]] (+ shift[k] for the position field): (m, w) doubles.
__global__ void gather_shift_kernel(const double* __restrict__ src, const int* __restrict__ idx,
                                    int64_t m, int w, const double* __restrict__ shift,
                                    double* __restrict__ dst) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t k = t / w;
  int c = (int)(t - k * w);
  if (k >= m) return;
  double v = src[(int64_t)idx[k] * w + c];
  if (shift) v = __dadd_rn(v, shift[k * w + c]);
  dst[t] = v;
}

// dst[idx[k]] += src[k] over (m, w) doubles; idx distinct within one call.
__global__ void scatter_add_kernel(double* __restrict__ dst, const int* __restrict__ idx,
                                   int64_t m, int w, const double* __restrict__ src) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t k = t / w;
  int c = (int)(t - k * w);
  if (k >= m) return;
  double* p = dst + (int64_t)idx[k] * w + c;
  *p = __dadd_rn(*p, src[t]);
}

// Per-step halo refresh (ref md.py:192-200 / decomp.py:231-260 with the
// plan cached): pack the raw x, y, z of exported rows into a contiguous send
// buffer; unpack a received buffer into the ghost rows (+ planar copy).
__global__ void halo_pack_kernel(const double* __restrict__ pos, const int* __restrict__ rows,
                                 int64_t m, double* __restrict__ buf) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const double4 p = ld_pos4(pos + 4 * (int64_t)rows[k]);
  buf[3 * k] = p.x;
  buf[3 * k + 1] = p.y;
  buf[3 * k + 2] = p.z;
}

__global__ void halo_pack_planar_kernel(const double* __restrict__ pl, int64_t ps,
                                        const int* __restrict__ rows, int64_t m,
                                        double* __restrict__ buf) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int r = rows[k];
  buf[3 * k] = pl[r];
  buf[3 * k + 1] = pl[ps + r];
  buf[3 * k + 2] = pl[2 * ps + r];
}

__global__ void halo_unpack_kernel(const double* __restrict__ buf, const int* __restrict__ rows,
                                   int64_t m, double* __restrict__ pos,
                                   double* __restrict__ planar, int64_t ps) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int r = rows[k];
  const double x = buf[3 * k], y = buf[3 * k + 1], z = buf[3 * k + 2];
  if (pos) {
    pos[4 * (int64_t)r] = x;
    pos[4 * (int64_t)r + 1] = y;
    pos[4 * (int64_t)r + 2] = z;
  }
  if (planar) {
    planar[r] = x;
    planar[ps + r] = y;
    planar[2 * ps + r] = z;
  }
}

}  // namespace pc

using namespace pc;

extern "C" {

int pc_owner_of(const double* d_x, int64_t n, int32_t d, const pc_grid* fabric,
                int32_t* d_owner, int32_t* d_flag, void* stream) {
  return pc_owner_of_domain(d_x, n, d, fabric, nullptr, 0, d_owner, d_flag, stream);
}

int pc_owner_of_domain(const double* d_x, int64_t n, int32_t d, const pc_grid* fabric,
                       const int32_t* d_skip, int32_t skip_owner, int32_t* d_owner,
                       int32_t* d_flag, void* stream) {
  if (n <= 0) return PC_OK;
  owner_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_x, n, d, *fabric, d_owner, d_flag, d_skip, skip_owner);
  return check_launch("pc_owner_of");
}

int pc_check_nonperiodic(const double* d_x, int64_t n, int32_t d, const pc_box* box,
                         int32_t* d_flag, void* stream) {
  if (n <= 0) return PC_OK;
  nonperiodic_check_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_x, n, d, *box, d_flag);
  return check_launch("pc_check_nonperiodic");
}

static int make_halo_table(const char* who, int32_t d, int32_t n_off, const int32_t* h_slot,
                           const double* h_shift, const double* h_lo, const double* h_hi,
                           int32_t n_slots, double w2, HaloTable& t,
                           const double* h_in_lo = nullptr, const double* h_in_hi = nullptr) {
  if (n_off > kMaxSlots || n_slots > kMaxSlots || d < 1 || d > 3) {
    set_error("%s: too many offsets or bad dimension", who);
    return PC_ERR_VALUE;
  }
  t.n_off = n_off;
  t.n_slots = n_slots;
  t.d = d;
  t.w2 = w2;
  t.has_in = h_in_lo && h_in_hi && d == 3;
  for (int a = 0; a < 3; ++a) {
    t.in_lo[a] = t.has_in ? h_in_lo[a] : 0.0;
    t.in_hi[a] = t.has_in ? h_in_hi[a] : 0.0;
  }
  for (int k = 0; k < n_off; ++k) {
    t.off[k].slot = h_slot[k];
    for (int a = 0; a < 3; ++a) {
      t.off[k].shift[a] = a < d ? h_shift[k * d + a] : 0.0;
      t.off[k].lo[a] = a < d ? h_lo[k * d + a] : 0.0;
      t.off[k].hi[a] = a < d ? h_hi[k * d + a] : 0.0;
    }
  }
  return PC_OK;
}

int64_t pc_halo_select_chunks(int64_t n) { return (n + kSelChunk - 1) / kSelChunk; }

int pc_halo_select_count(const double* d_pos4, int64_t n, int32_t d, int32_t n_off,
                         const int32_t* h_slot, const double* h_shift, const double* h_lo,
                         const double* h_hi, int32_t n_slots, double w2, int32_t* d_hist,
                         void* stream, const double* h_in_lo, const double* h_in_hi) {
  if (n <= 0) return PC_OK;
  HaloTable t;
  const int rc = make_halo_table("pc_halo_select_count", d, n_off, h_slot, h_shift, h_lo, h_hi,
                                 n_slots, w2, t, h_in_lo, h_in_hi);
  if (rc != PC_OK) return rc;
  const int64_t nch = pc_halo_select_chunks(n);
  halo_select_count_kernel<<<(unsigned)nch, kSelChunk, 0, as_stream(stream)>>>(d_pos4, n, t,
                                                                              (int)nch, d_hist);
  return check_launch("pc_halo_select_count");
}

int pc_halo_select_place(const double* d_pos4, int64_t n, int32_t d, int32_t n_off,
                         const int32_t* h_slot, const double* h_shift, const double* h_lo,
                         const double* h_hi, int32_t n_slots, double w2, const int32_t* d_off,
                         int32_t* d_out_idx, double* d_out_rows, void* stream,
                         const double* h_in_lo, const double* h_in_hi) {
  if (n <= 0) return PC_OK;
  HaloTable t;
  const int rc = make_halo_table("pc_halo_select_place", d, n_off, h_slot, h_shift, h_lo, h_hi,
                                 n_slots, w2, t, h_in_lo, h_in_hi);
  if (rc != PC_OK) return rc;
  const int64_t nch = pc_halo_select_chunks(n);
  halo_select_place_kernel<<<(unsigned)nch, kSelChunk, 0, as_stream(stream)>>>(
      d_pos4, n, t, (int)nch, d_off, d_out_idx, d_out_rows);
  return check_launch("pc_halo_select_place");
}

int pc_halo_plan(const double* d_x, int64_t n, int32_t d, int32_t n_off, const int32_t* h_slot,
                 const double* h_shift, const double* h_lo, const double* h_hi, int32_t n_slots,
                 double w2, int32_t* d_flags, int8_t* d_best_off, void* stream) {
  if (n <= 0) return PC_OK;
  if (n_off > kMaxSlots || n_slots > kMaxSlots || d < 1 || d > 3) {
    set_error("pc_halo_plan: too many offsets or bad dimension");
    return PC_ERR_VALUE;
  }
  HaloTable t;
  t.n_off = n_off;
  t.n_slots = n_slots;
  t.d = d;
  t.w2 = w2;
  for (int k = 0; k < n_off; ++k) {
    t.off[k].slot = h_slot[k];
    for (int a = 0; a < 3; ++a) {
      t.off[k].shift[a] = a < d ? h_shift[k * d + a] : 0.0;
      t.off[k].lo[a] = a < d ? h_lo[k * d + a] : 0.0;
      t.off[k].hi[a] = a < d ? h_hi[k * d + a] : 0.0;
    }
  }
  halo_plan_kernel<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(d_x, n, t, d_flags,
                                                                               d_best_off);
  return check_launch("pc_halo_plan");
}

int pc_halo_force_pack(double* d_f3, int64_t f_stride, const int32_t* d_rows, int64_t m,
                       double* d_buf, void* stream) {
  if (m <= 0) return PC_OK;
  halo_force_pack_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_f3, f_stride, d_rows, m, d_buf);
  return check_launch("pc_halo_force_pack");
}

int pc_halo_force_add(double* d_f3, int64_t f_stride, const int32_t* d_rows, int64_t m,
                      const double* d_buf, void* stream) {
  if (m <= 0) return PC_OK;
  halo_force_add_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_f3, f_stride, d_rows, m, d_buf);
  return check_launch("pc_halo_force_add");
}

int pc_compact(const int32_t* d_flag, const int32_t* d_pos, int64_t n, int32_t* d_out_idx,
               const int8_t* d_best_off, int8_t* d_out_off, void* stream) {
  if (n <= 0) return PC_OK;
  compact_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_flag, d_pos, n, d_out_idx, d_best_off, d_out_off);
  return check_launch("pc_compact");
}

int pc_gather_shift(const double* d_src, const int32_t* d_idx, int64_t m, int32_t w,
                    const double* d_shift, double* d_dst, void* stream) {
  int64_t t = m * w;
  if (t <= 0) return PC_OK;
  gather_shift_kernel<<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_src, d_idx, m, w, d_shift, d_dst);
  return check_launch("pc_gather_shift");
}

int pc_halo_pack(const double* d_pos, const int32_t* d_rows, int64_t m, double* d_buf,
                 void* stream) {
  if (m <= 0) return PC_OK;
  halo_pack_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(d_pos, d_rows, m,
                                                                               d_buf);
  return check_launch("pc_halo_pack");
}

int pc_halo_pack_planar(const double* d_planar, int64_t planar_stride, const int32_t* d_rows,
                        int64_t m, double* d_buf, void* stream) {
  if (m <= 0) return PC_OK;
  halo_pack_planar_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_planar, planar_stride, d_rows, m, d_buf);
  return check_launch("pc_halo_pack_planar");
}

int pc_halo_unpack(const double* d_buf, const int32_t* d_rows, int64_t m, double* d_pos,
                   double* d_planar, int64_t planar_stride, void* stream) {
  if (m <= 0) return PC_OK;
  halo_unpack_kernel<<<(unsigned)((m + 255) / 256), 256, 0, as_stream(stream)>>>(
      d_buf, d_rows, m, d_pos, d_planar, planar_stride);
  return check_launch("pc_halo_unpack");
}

int pc_scatter_add(double* d_dst, const int32_t* d_idx, int64_t m, int32_t w,
                   const double* d_src, void* stream) {
  int64_t t = m * w;
  if (t <= 0) return PC_OK;
  scatter_add_kernel<<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(d_dst, d_idx,
                                                                                 m, w, d_src);
  return check_launch("pc_scatter_add");
}

}  // extern "C"
