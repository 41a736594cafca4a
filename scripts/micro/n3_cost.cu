// Cost of the j-side force accumulation a Newton-3 (half-list) tile force
// pass would add: per pair evaluated once, three
// atomic adds to the neighbour's accumulator --
//   (a) FP32 atomicAdd in shared memory (the staged neighbourhood's slots;
//       sm_100a has no native shared FP32 add: ATOMS.CAST.SPIN CAS loop),
//   (b) FP64 red.global.add at scattered addresses (a neighbour's global
//       force row), (c) the same, lane-coalesced (a per-tile flush of staged
//       slots), against (d) the plain LDS + FADD + STS of one warp (no race),
// all at full occupancy, 3 ops per "pair" as the x, y, z components.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o n3_cost n3_cost.cu
#include <cstdio>
#include <cstdint>

constexpr int kSlots = 2304;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// (a) shared FP32 atomics, random slots (distinct per lane with high probability)
__global__ void smem_atomic(float* out, int iters) {
  __shared__ float acc[3 * kSlots];
  for (int i = threadIdx.x; i < 3 * kSlots; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  uint32_t h = hash(blockIdx.x * blockDim.x + threadIdx.x);
  const float f = 1e-3f * (threadIdx.x & 7);
  for (int it = 0; it < iters; ++it) {
    h = hash(h);
    const int s = h % kSlots;
    atomicAdd(&acc[s], f);
    atomicAdd(&acc[kSlots + s], f);
    atomicAdd(&acc[2 * kSlots + s], f);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[threadIdx.x % (3 * kSlots)];
}

// (d) plain read-modify-write (each warp its own region: no race)
__global__ void smem_plain(float* out, int iters) {
  __shared__ float acc[32][3 * 64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 3 * 64; i += 32) acc[w][i] = 0.f;
  __syncwarp();
  uint32_t h = hash(blockIdx.x * blockDim.x + threadIdx.x);
  const float f = 1e-3f * (threadIdx.x & 7);
  for (int it = 0; it < iters; ++it) {
    h = hash(h);
    const int s = (lane + (h & 1) * 32) & 63;       // distinct per lane
    acc[w][s] += f;
    acc[w][64 + s] += f;
    acc[w][128 + s] += f;
  }
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[w][lane];
}

// (b) / (c) FP64 reductions into a global array of n rows (planar x|y|z)
template <bool COALESCED>
__global__ void global_red(double* f, int64_t n, int iters) {
  uint32_t h = hash(blockIdx.x * blockDim.x + threadIdx.x);
  const double v = 1e-3 * (threadIdx.x & 7);
  const int64_t base = (int64_t)(blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    h = hash(h);
    int64_t j;
    if (COALESCED) j = (base + (int64_t)it * gridDim.x * blockDim.x) % n;
    else j = (int64_t)(h % (uint32_t)n);
    atomicAdd(&f[j], v);                 // no return value used: RED.E.ADD.F64
    atomicAdd(&f[n + j], v);
    atomicAdd(&f[2 * n + j], v);
  }
}

template <typename K>
float timed(K kernel) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kernel();                              // warm-up
  cudaEventRecord(a);
  kernel();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 1024, iters = 4000;
  float* outf;
  cudaMalloc(&outf, (size_t)sms * threads * 4);
  const int64_t n = 8388608;
  double* f;
  cudaMalloc(&f, 3 * n * 8);
  cudaMemset(f, 0, 3 * n * 8);
  const double warp_ops = (double)sms * (threads / 32) * iters * 3;   // warp-level ops
  const double lane_ops = warp_ops * 32;
  const double clk = 1.965e9;
  float ms = timed([&] { smem_atomic<<<sms, threads>>>(outf, iters); });
  printf("(a) shared FP32 atomicAdd (CAS loop), random slots: %.3f ms  %.2f SM-cycles per warp op  %.1f G lane-ops/s\n",
         ms, ms * 1e-3 * clk / (warp_ops / sms), lane_ops / (ms * 1e-3) / 1e9);
  ms = timed([&] { smem_plain<<<sms, threads>>>(outf, iters); });
  printf("(d) shared FP32 LDS+FADD+STS, no race:              %.3f ms  %.2f SM-cycles per warp op  %.1f G lane-ops/s\n",
         ms, ms * 1e-3 * clk / (warp_ops / sms), lane_ops / (ms * 1e-3) / 1e9);
  const int gblocks = sms * 4, gthreads = 256, giters = 200;
  const double g_ops = (double)gblocks * gthreads * giters * 3;
  ms = timed([&] { global_red<false><<<gblocks, gthreads>>>(f, n, giters); });
  printf("(b) global FP64 red.add, scattered rows (8.4M):     %.3f ms  %.1f G lane-ops/s\n", ms,
         g_ops / (ms * 1e-3) / 1e9);
  ms = timed([&] { global_red<true><<<gblocks, gthreads>>>(f, n, giters); });
  printf("(c) global FP64 red.add, lane-coalesced rows:        %.3f ms  %.1f G lane-ops/s\n", ms,
         g_ops / (ms * 1e-3) / 1e9);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
