// Microbenchmark: per-SM throughput of DFMA, F2F (f64<->f32), MUFU.RCP64H, FFMA on B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-3 + a, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float f0 = x0, f1 = x1, f2 = x2, f3 = x3, f4 = x4, f5 = x5, f6 = x6, f7 = x7;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) { x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
                   x4 = fma(x4, a, 1e-9); x5 = fma(x5, a, 1e-9); x6 = fma(x6, a, 1e-9); x7 = fma(x7, a, 1e-9); }
    if (OP == 1) { f0 = (float)x0; f1 = (float)x1; f2 = (float)x2; f3 = (float)x3; f4 = (float)x4; f5 = (float)x5; f6=(float)x6; f7=(float)x7;
                   x0 = (double)f1 + 1e-30; x1 = (double)f2; x2 = (double)f3; x3 = (double)f4; x4=(double)f5; x5=(double)f6; x6=(double)f7; x7=(double)f0; }
    if (OP == 2) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x0)); x0 = r + 1.0;
                   asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x1)); x1 = r + 1.0;
                   asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x2)); x2 = r + 1.0;
                   asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x3)); x3 = r + 1.0; }
    if (OP == 3) { f0 = fmaf(f0, 0.999f, 1e-3f); f1 = fmaf(f1, 0.999f, 1e-3f); f2 = fmaf(f2, 0.999f, 1e-3f); f3 = fmaf(f3, 0.999f, 1e-3f);
                   f4 = fmaf(f4, 0.999f, 1e-3f); f5 = fmaf(f5, 0.999f, 1e-3f); f6 = fmaf(f6, 0.999f, 1e-3f); f7 = fmaf(f7, 0.999f, 1e-3f); }
    if (OP == 4) { x0 = x0 * a; x1 = x1 * a; x2 = x2*a; x3 = x3*a; x4 = x4*a; x5=x5*a; x6=x6*a; x7=x7*a; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7;
}
template <int OP> void run(const char* name, int ops_per_iter) {
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<OP><<<148 * 8, 1024>>>(out, 16, 0.9999);
  cudaEventRecord(a); k<OP><<<148 * 8, 1024>>>(out, iters, 0.9999); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = 148.0 * 8 * 1024 * iters * ops_per_iter;
  printf("%-22s %8.3f ms  %8.2f Gop/s  %7.1f lane-ops/clk/SM @1.965GHz\n", name, ms, ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
}
int main() { run<0>("DFMA", 8); run<4>("DMUL", 8); run<1>("F2F f64->f32->f64", 16); run<2>("MUFU.RCP64H(+DADD)", 4); run<3>("FFMA", 8); return 0; }
