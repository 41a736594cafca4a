// Microbenchmark: per-SM lane-op throughput of the ops the force kernel mixes.
#include <cstdio>
#include <cuda_runtime.h>
#define R8(S) S(0) S(1) S(2) S(3) S(4) S(5) S(6) S(7)
template <int OP>
__global__ void k(float* out, int iters, double a, float af, int ai) {
  double d[8]; float f[8]; int q[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) { d[t] = threadIdx.x * 1e-3 + t; f[t] = (float)d[t]; q[t] = threadIdx.x + t; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (OP == 0) d[t] = fma(d[t], a, 1e-9);                 // DFMA
      if (OP == 1) d[t] = d[t] + a;                           // DADD
      if (OP == 2) f[t] = __double2float_rn(d[t] + (double)f[t]); // DADD + F2F.F32.F64
      if (OP == 3) { d[t] = d[t] + (double)f[t]; f[t] = f[t] * af; }  // F2F.F64.F32 + DADD + FMUL
      if (OP == 4) f[t] = fmaf(f[t], af, 1e-3f);              // FFMA
      if (OP == 5) { q[t] += ai; f[t] += (float)q[t]; }        // IADD + I2F + FADD
      if (OP == 6) f[t] = __frcp_rn(f[t]) + af;               // MUFU.RCP (+fixup) 
      if (OP == 7) { float r; asm volatile("rcp.approx.ftz.f32 %0,%1;" : "=f"(r) : "f"(f[t])); f[t] = r + af; }
      if (OP == 8) q[t] = (q[t] ^ ai) + (q[t] >> 3);          // ALU
      if (OP == 9) d[t] = (d[t] < a) ? d[t] + 1.0 : d[t];     // DSETP + DADD + sel
      if (OP == 10) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d[t])); d[t] = r + a; }
      if (OP == 11) d[t] = (double)f[t] * a + d[t], f[t] = f[t] + af; // F2F.F64.F32 + DFMA + FADD
      if (OP == 12) {                                           // FFMA2 (two FP32 lanes per op)
        unsigned long long x, y = ((unsigned long long)__float_as_uint(af) << 32) | __float_as_uint(af);
        asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(f[t]), "f"(f[(t + 1) & 7]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x) : "l"(y));
        float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x)); f[t] = lo + hi * 0.f;
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += (float)d[t] + f[t] + (float)q[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP> void run(const char* name, double ops_per_iter) {
  float* out; cudaMalloc(&out, 148 * 8 * 512 * 4);
  int iters = 2048;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<OP><<<148 * 8, 512>>>(out, 16, 0.9999, 0.999f, 3);
  cudaEventRecord(a); k<OP><<<148 * 8, 512>>>(out, iters, 0.9999, 0.999f, 3); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = 148.0 * 8 * 512 * iters * ops_per_iter;
  printf("%-28s %8.3f ms  %7.1f lane-ops/clk/SM @1.965GHz\n", name, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
}
int main() {
  run<0>("DFMA", 8); run<1>("DADD", 8); run<2>("DADD+F2F.F32.F64 (pairs)", 8);
  run<3>("F2F.F64.F32+DMUL (pairs)", 8); run<4>("FFMA", 8); run<5>("IADD+I2F (pairs)", 8);
  run<6>("__frcp_rn (+FADD)", 8); run<7>("rcp.approx.f32 (+FADD)", 8); run<8>("LOP/SHF/IADD (x3)", 8);
  run<9>("DSETP+DADD+FSEL", 8); run<10>("MUFU.RCP64H(+DADD)", 8);
  run<11>("F2F.F64.F32+DFMA+FADD (trip)", 8); run<12>("FFMA2 (+pack)", 8);
  return 0;
}
