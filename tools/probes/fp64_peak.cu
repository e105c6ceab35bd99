// FP64 peak probe on B200: DFMA (CUDA cores) vs DMMA.8x8x4 (tensor cores), plus
// FFMA and IMAD.WIDE issue probes for the k_pmc roofline (run under gpurun).
#include <cstdio>
#include <cstdint>
__global__ void dfma_loop(double* out, int iters, double s) {
  double a[8];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-9 + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = fma(a[q], s, 1e-12);
  double t = 0; for (int q = 0; q < 8; ++q) t += a[q];
  if (t == 12345.0) out[0] = t;
}
__global__ void dmma_loop(double* out, int iters, double s) {
  double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double a = threadIdx.x * 1e-9 + s, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[2 * q]), "+d"(c[2 * q + 1]) : "d"(a), "d"(b));
  }
  double t = 0; for (int q = 0; q < 8; ++q) t += c[q];
  if (t == 12345.0) out[0] = t;
}
__global__ void ffma_loop(float* out, int iters, float s) {
  float a[8];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-9f + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = fmaf(a[q], s, 1e-12f);
  float t = 0; for (int q = 0; q < 8; ++q) t += a[q];
  if (t == 12345.0f) out[0] = t;
}
__global__ void imadwide_loop(uint32_t* out, int iters, uint32_t s) {
  uint32_t a[8];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint64_t p = (uint64_t)0xD2511F53u * a[q];
      a[q] = (uint32_t)(p >> 32) ^ (uint32_t)p ^ s;
    }
  uint32_t t = 0; for (int q = 0; q < 8; ++q) t ^= a[q];
  if (t == 12345u) out[0] = t;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8, threads = 256, iters = 20000;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(d, iters, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    if (rep) printf("DFMA  : %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(d, iters / 4, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 4 * (iters / 4) * (double)blocks * (threads / 32);
    if (rep) printf("DMMA  : %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); ffma_loop<<<blocks, threads>>>((float*)d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * iters * (double)blocks * threads;
    if (rep) printf("FFMA  : %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); imadwide_loop<<<blocks, threads>>>((uint32_t*)d, iters, 7u); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 8.0 * iters * (double)blocks * threads;
    if (rep) printf("IMAD.WIDE+LOP3 pairs: %.3f T/s (%.3f ms)\n", fl / ms / 1e12, ms);
  }
  return 0;
}
