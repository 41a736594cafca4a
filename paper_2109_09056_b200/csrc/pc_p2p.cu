// Peer-memory halo exchange (NVLink P2P stores between processes, CUDA IPC).
//
// The per-step ghost refresh of a decomposed domain (ref md.py:192-200,
// decomp.py:231-260) moves each exported particle's x, y, z to the ranks
// that hold it as a ghost.  Over NCCL that is an all_to_all_single: SM
// kernels plus protocol overhead on every step.  Here every rank owns a
// receive window in device memory, exported with cudaIpcGetMemHandle and
// mapped by its peers: the sender's put kernel stores the packed rows
// straight into each destination's window over NVLink, then raises the
// destination's arrival flag; the receiver waits for its sources' flags on
// the device (no host round trip), unpacks, and acknowledges.
//
// Window layout (one per rank and channel):
//   [2 parities x cap rows x w doubles][arrive: world int64][ack: world int64]
// Step k of a channel uses parity k & 1.  arrive[s] = k: source s has stored
// its step-k rows here; ack[d] = k: destination d has unpacked this rank's
// step-k rows (so parity k & 1 of d's window may be written again at k + 2).
// Ordering: the put kernel's threads fence (system scope) after their stores;
// the signal kernel, launched after it on the same stream, fences and writes
// the flags with volatile stores; waits spin on volatile loads and fence.
#include <string.h>

#include "pc_common.cuh"

namespace pc {

struct P2PDest {          // one destination of a put
  double* window;         // destination window base (IPC-mapped, or own)
  int64_t src0;           // first row in the send buffer
  int64_t count;          // rows
  int64_t dst0;           // first row in the destination's window parity block
};

__global__ void p2p_wait_kernel(const volatile long long* __restrict__ flags,
                                const int* __restrict__ ranks, int n, long long target,
                                int* __restrict__ err, long long spin_limit) {
  // one thread per awaited flag
  const int t = threadIdx.x;
  if (t < n) {
    const volatile long long* f = flags + ranks[t];
    long long spins = 0;
    while (*f < target) {
      __nanosleep(200);
      if (++spins > spin_limit) {
        atomicOr(err, 1);
        break;
      }
    }
  }
  __threadfence_system();
}

__global__ void p2p_put_kernel(const double* __restrict__ send, const P2PDest* __restrict__ dst,
                               int w, int64_t cap, int parity) {
  const P2PDest D = dst[blockIdx.y];
  double* out = D.window + ((int64_t)parity * cap + D.dst0) * w;
  const double* in = send + D.src0 * w;
  const int64_t n = D.count * w;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[k];
  __threadfence_system();
}

// K11: the refresh's pack fused into the put -- exported row k of
// destination D is gathered from the planar positions and stored straight
// into D's window (no send buffer)
__global__ void p2p_pack_put_kernel(const double* __restrict__ pl, int64_t ps,
                                    const int* __restrict__ rows,
                                    const P2PDest* __restrict__ dst, int64_t cap, int parity) {
  const P2PDest D = dst[blockIdx.y];
  double* out = D.window + ((int64_t)parity * cap + D.dst0) * 3;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < D.count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = rows[D.src0 + k];
    out[3 * k] = pl[r];
    out[3 * k + 1] = pl[ps + r];
    out[3 * k + 2] = pl[2 * ps + r];
  }
  __threadfence_system();
}

// flag[me] = value in each window of the table (arrive or ack region)
__global__ void p2p_signal_kernel(const P2PDest* __restrict__ dst, int n, int64_t flag_off,
                                  int me, long long value) {
  __threadfence_system();
  const int t = threadIdx.x;
  if (t < n) {
    volatile long long* f =
        reinterpret_cast<volatile long long*>(dst[t].window + flag_off) + me;
    *f = value;
  }
  __threadfence_system();
}

}  // namespace pc

using namespace pc;

extern "C" {

int pc_p2p_window_bytes(int64_t cap_rows, int32_t width, int32_t world, int64_t* bytes) {
  if (cap_rows < 0 || width <= 0 || world <= 0) {
    set_error("pc_p2p_window_bytes: bad capacity / width / world");
    return PC_ERR_VALUE;
  }
  *bytes = (2 * cap_rows * width + 2 * (int64_t)world) * (int64_t)sizeof(double);
  return PC_OK;
}

int pc_p2p_window_alloc(int64_t cap_rows, int32_t width, int32_t world, void** d_window,
                        void* h_handle) {
  int64_t bytes = 0;
  int rc = pc_p2p_window_bytes(cap_rows, width, world, &bytes);
  if (rc != PC_OK) return rc;
  void* p = nullptr;
  if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) {
    cudaGetLastError();
    set_error("pc_p2p_window_alloc: cudaMalloc of %lld B failed", (long long)bytes);
    return PC_ERR_CAPACITY;
  }
  cudaMemset(p, 0, (size_t)bytes);
  if (h_handle) {
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(p);
      set_error("pc_p2p_window_alloc: cudaIpcGetMemHandle failed");
      return PC_ERR_CUDA;
    }
    memcpy(h_handle, &h, sizeof(h));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error("pc_p2p_window_alloc: %s", cudaGetErrorString(cudaGetLastError()));
    return PC_ERR_CUDA;
  }
  *d_window = p;
  return PC_OK;
}

int pc_p2p_window_free(void* d_window) {
  if (d_window && cudaFree(d_window) != cudaSuccess) {
    set_error("pc_p2p_window_free: %s", cudaGetErrorString(cudaGetLastError()));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

int32_t pc_p2p_handle_bytes(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

int pc_p2p_open(const void* h_handle, void** d_peer) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  if (cudaIpcOpenMemHandle(d_peer, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    set_error("pc_p2p_open: cudaIpcOpenMemHandle: %s", cudaGetErrorString(cudaGetLastError()));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

int pc_p2p_close(void* d_peer) {
  if (d_peer && cudaIpcCloseMemHandle(d_peer) != cudaSuccess) {
    set_error("pc_p2p_close: %s", cudaGetErrorString(cudaGetLastError()));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

// Wait (on the stream) until flags[ranks[t]] >= target for every t < n: the
// arrive region of this rank's own window (sources) or its ack region
// (destinations).  A wait that exceeds ~spin_limit x 200 ns sets *d_err.
int pc_p2p_wait(const void* d_window, int64_t flag_off, const int32_t* d_ranks, int32_t n,
                int64_t target, int32_t* d_err, int64_t spin_limit, void* stream) {
  if (n <= 0) return PC_OK;
  if (n > 1024) {
    set_error("pc_p2p_wait: at most 1024 peers");
    return PC_ERR_VALUE;
  }
  const volatile long long* f = reinterpret_cast<const volatile long long*>(
      static_cast<const double*>(d_window) + flag_off);
  p2p_wait_kernel<<<1, ((n + 31) / 32) * 32, 0, as_stream(stream)>>>(f, d_ranks, n, target,
                                                                       d_err, spin_limit);
  return check_launch("pc_p2p_wait");
}

// Store the rows of each destination of the table (n_dst entries, device
// memory) into its window's parity block.
int pc_p2p_put(const double* d_send, const void* d_dests, int32_t n_dst, int64_t max_rows,
               int32_t width, int64_t cap_rows, int32_t parity, void* stream) {
  if (n_dst <= 0 || max_rows <= 0) return PC_OK;
  const int64_t tot = max_rows * width;
  unsigned bx = (unsigned)((tot + 255) / 256);
  if (bx > 1184) bx = 1184;
  p2p_put_kernel<<<dim3(bx, (unsigned)n_dst), 256, 0, as_stream(stream)>>>(
      d_send, static_cast<const P2PDest*>(d_dests), width, cap_rows, parity & 1);
  return check_launch("pc_p2p_put");
}

// Fused pack + put of the ghost refresh: rows[src0 + k] of the planar x|y|z
// positions to each destination window's parity block (width 3).
int pc_p2p_pack_put(const double* d_planar, int64_t planar_stride, const int32_t* d_rows,
                    const void* d_dests, int32_t n_dst, int64_t max_rows, int64_t cap_rows,
                    int32_t parity, void* stream) {
  if (n_dst <= 0 || max_rows <= 0) return PC_OK;
  unsigned bx = (unsigned)((max_rows + 255) / 256);
  if (bx > 1184) bx = 1184;
  p2p_pack_put_kernel<<<dim3(bx, (unsigned)n_dst), 256, 0, as_stream(stream)>>>(
      d_planar, planar_stride, d_rows, static_cast<const P2PDest*>(d_dests), cap_rows,
      parity & 1);
  return check_launch("pc_p2p_pack_put");
}

// flags[me] = value in every window of the table (flag_off: the arrive or
// the ack region, in doubles from the window base).
int pc_p2p_signal(const void* d_dests, int32_t n_dst, int64_t flag_off, int32_t me,
                  int64_t value, void* stream) {
  if (n_dst <= 0) return PC_OK;
  p2p_signal_kernel<<<1, ((n_dst + 31) / 32) * 32, 0, as_stream(stream)>>>(
      static_cast<const P2PDest*>(d_dests), n_dst, flag_off, me, (long long)value);
  return check_launch("pc_p2p_signal");
}

int32_t pc_p2p_dest_bytes(void) { return (int32_t)sizeof(P2PDest); }

}  // extern "C"
