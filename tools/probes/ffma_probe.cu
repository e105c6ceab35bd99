// Why does the same FFMA chain pattern issue at rt 1 in one probe and rt 2 in another?
#include <cstdint>
#include <cstdio>
#include "warm.cuh"
__global__ void k1(float* out, int iters, float s) {   // alu_rates style: 8 chains, 1 FFMA each
  float a[8];
  for (int q = 0; q < 8; ++q) a[q] = (float)(threadIdx.x + q) * 1e-9f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(s), "f"(s));
  float t = 0;
  for (int q = 0; q < 8; ++q) t += a[q];
  if (t == 12345.f) out[0] = t;
}
__global__ void __launch_bounds__(256) k2(float* out, int iters, float s) {   // imad_mix mode-6 style
  float f[8];
  for (int q = 0; q < 8; ++q) f[q] = threadIdx.x * 1e-9f + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[2 * q]) : "f"(s), "f"(s));
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[2 * q + 1]) : "f"(s), "f"(s));
    }
  float g = 0;
  for (int q = 0; q < 8; ++q) g += f[q];
  if (g == 1.2345f) out[0] = g;
}
__global__ void k3(float* out, int iters, float s) {   // k1 with values that grow large (like k2's init)
  float a[8];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-9f + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(s), "f"(s));
  float t = 0;
  for (int q = 0; q < 8; ++q) t += a[q];
  if (t == 12345.f) out[0] = t;
}
__global__ void k4(float* out, int iters, float s) {   // k1 with s = 0.5 (exact values)
  float a[8];
  for (int q = 0; q < 8; ++q) a[q] = (float)(threadIdx.x + q) * 1e-9f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(s), "f"(s));
  float t = 0;
  for (int q = 0; q < 8; ++q) t += a[q];
  if (t == 12345.f) out[0] = t;
}
int main() {
  const double clk = warm_and_clock_mhz();
  float* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = 148 * 8, iters = 4096;
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 5; ++m) {
      cudaEventRecord(e0);
      if (m == 0) k1<<<blocks, threads>>>(d, iters, 0.999f);
      if (m == 1) k2<<<blocks, threads>>>(d, iters, 0.999f);
      if (m == 2) k3<<<blocks, threads>>>(d, iters, 0.999f);
      if (m == 3) k4<<<blocks, threads>>>(d, iters, 0.5f);
      if (m == 4) k2<<<blocks, threads>>>(d, iters, 0.5f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double wi = 8.0 * iters * blocks * (threads / 32);
      if (rep) printf("k%d s=%s %7.3f ms  %.3f FFMA warp-instr per SMSP per clock\n", m < 4 ? m + 1 : 2,
                      m >= 3 ? "0.5" : "0.999", ms, wi / (ms * 1e-3 * clk * 1e6 * 148 * 4));
    }
  return 0;
}
