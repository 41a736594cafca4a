// LDS.64 wavefront model: does a warp need max-distinct-addresses-per-bank-pair over the
// whole warp (warp model) or per fixed half-warp (half model)?
#include <cstdio>
__device__ int pat(int P, int lane) {
  switch (P) {
    case 0: return lane;                                        // distinct residues per half
    case 1: return (lane & 7) + ((lane >> 3) & 1) * 16 + (lane >> 4) * 8;  // half: 2/res, warp: 2/res
    case 2: return lane < 16 ? (lane & 7) + ((lane >> 3) & 1) * 16 : 40 + lane;  // half0: 2/res; half1 distinct
    case 3: return lane * 16;                                   // all residue 0: 32 distinct
    case 4: return (lane & 15) + (lane >> 4) * 16;              // each residue: 2 slots (one per half)
    case 5: return (lane & 15) + (lane & 16 ? 32 : 0) + ((lane & 1) ? 64 : 0); // 3-4 per residue? (mixed)
  }
  return 0;
}
template <int P>
__global__ void k(double* out, int iters) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int off = pat(P, lane);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += s[(off + u * 128 + (it & 7) * 512) & 4095];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int P> void run(const char* name) {
  double* out; cudaMalloc(&out, 148 * 1024 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 2000;
  k<P><<<148, 1024>>>(out, 10);
  cudaEventRecord(a); k<P><<<148, 1024>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double lds = 148.0 * 32 * iters * 16;   // warp-level LDS per SM summed
  double cyc = ms * 1e-3 * 1.965e9;
  printf("%-44s %.3f ms  %.2f SM-cycles per warp LDS.64\n", name, ms, cyc / (lds / 148));
  cudaFree(out);
}
int main() {
  run<0>("P0 distinct residues per half");
  run<1>("P1 half: 2/res ; warp: 2/res (split)");
  run<2>("P2 half0 2/res, half1 distinct");
  run<3>("P3 all residue 0 (32 distinct)");
  run<4>("P4 each residue 2 slots, one per half");
  return 0;
}
