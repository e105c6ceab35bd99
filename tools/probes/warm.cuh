// Shared by the probes: spin the GPU up to its boost clock, then report the SM clock
// measured as clock64() cycles per event-timed microsecond.
#pragma once
#include <cstdio>
__global__ void k_spin(long long cycles, int* sink) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 9999) sink[0] = 1;
}
inline double warm_and_clock_mhz() {
  int* d;
  cudaMalloc(&d, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 20; ++i) k_spin<<<148 * 4, 128>>>(200000000LL / 2, d);   // ~1 s at 2 GHz
  cudaDeviceSynchronize();
  const long long cyc = 400000000LL;
  cudaEventRecord(e0);
  k_spin<<<148 * 4, 128>>>(cyc, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double mhz = cyc / (ms * 1e3);
  printf("measured SM clock after warm-up: %.0f MHz\n", mhz);
  cudaFree(d);
  return mhz;
}
