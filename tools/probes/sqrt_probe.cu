// sqrt_probe.cu -- accuracy of the brick's FP64 sqrt from the MUFU.RSQ64H seed with one or two
// Newton steps on 1/sqrt plus the final sqrt correction, against the correctly rounded sqrt.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 sqrt_probe.cu -o sqrt_probe && ./sqrt_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NEWTON>
__device__ __forceinline__ double sqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < NEWTON; ++i) y = y * fma(-0.5 * x, y * y, 1.5);
  const double r = x * y;
  return fma(0.5 * y, fma(-r, r, x), r);
}

__global__ void probe(int64_t n, unsigned long long* maxulp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // log-uniform x over [1e-12, 1e12] plus tiny values
  const double u = (double)(i * 2654435761ull % 1000003ull) / 1000003.0;
  const double x = exp((u * 2.0 - 1.0) * 27.63) * (1.0 + 1e-7 * (double)(i % 977));
  const double ref = __dsqrt_rn(x);
  const double a1 = sqrt_seed<1>(x), a2 = sqrt_seed<2>(x), a0 = sqrt_seed<0>(x);
  const long long r = __double_as_longlong(ref);
  atomicMax(maxulp + 0, (unsigned long long)llabs(__double_as_longlong(a0) - r));
  atomicMax(maxulp + 1, (unsigned long long)llabs(__double_as_longlong(a1) - r));
  atomicMax(maxulp + 2, (unsigned long long)llabs(__double_as_longlong(a2) - r));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  const int64_t n = 1 << 26;
  probe<<<(unsigned)((n + 255) / 256), 256>>>(n, d);
  unsigned long long h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("max ulp vs correctly rounded sqrt over %lld values: 0 Newton steps %llu, 1 step %llu, 2 steps %llu\n",
         (long long)n, h[0], h[1], h[2]);
  return 0;
}
