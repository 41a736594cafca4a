// Does __reduce_max_sync work with per-lane group masks (disjoint groups in one instruction)?
#include <cstdio>
__global__ void k(int* out) {
  const int lane = threadIdx.x & 31;
  const unsigned key = (lane * 7) % 5;                       // 5 groups
  const unsigned m = __match_any_sync(0xffffffffu, key);
  const int v = (lane * 13) % 17;
  out[lane] = __reduce_max_sync(m, v);
  // reference
  int best = -1;
  for (int l = 0; l < 32; ++l) if ((m >> l) & 1) { int vv = (l * 13) % 17; best = vv > best ? vv : best; }
  out[32 + lane] = best;
}
int main() {
  int* d; cudaMalloc(&d, 64 * 4); k<<<1, 32>>>(d); int h[64]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 32; ++i) bad += h[i] != h[32 + i];
  printf("redux with group masks: %s\n", bad ? "MISMATCH" : "ok"); for (int i = 0; i < 32; ++i) printf("%d/%d ", h[i], h[32+i]); printf("\n");
  return 0;
}
