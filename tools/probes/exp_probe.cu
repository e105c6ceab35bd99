// Accuracy of the brick kernel's exp_neg_fast (brick.cu) against libm exp(-x).
#include <cstdio>
#include <cmath>
__constant__ double c_exp_taylor[13] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29};
__constant__ double c_exp_consts[4] = {1.4426950408889634074, 6755399441055744.0, 0x1.62e42fefa39efp-1,
                                       0x1.abc9e3b39803fp-56};
__device__ __forceinline__ double exp_neg_fast(double x) {
  const double t = fma(-x, c_exp_consts[0], c_exp_consts[1]);
  const double n = t - c_exp_consts[1];
  double f = fma(n, -c_exp_consts[2], -x);
  f = fma(n, -c_exp_consts[3], f);
  double p = c_exp_taylor[12];
#pragma unroll
  for (int i = 11; i >= 0; --i) p = fma(p, f, c_exp_taylor[i]);
  const int ni = __double2loint(t);
  const double scale = __hiloint2double((ni + 1023) << 20, 0);
  return ni < -1022 ? 0.0 : p * scale;
}
__device__ __forceinline__ double sqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  double r = x * y;
  r = fma(0.5 * y, fma(-r, r, x), r);
  return x > 0.0 ? r : 0.0;
}
__global__ void ks(double* err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = i == 0 ? 0.0 : exp2(-60.0 + 120.0 * ((double)i / n));
  double a = sqrt_fast(x), b = sqrt(x);
  err[i] = b > 0 ? fabs(a - b) / b : fabs(a - b);
}
__global__ void k(double* err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = 745.0 * ((double)i / n);          // covers the whole range
  double a = exp_neg_fast(x), b = exp(-x);
  double e = b > 1e-300 ? fabs(a - b) / b : fabs(a - b);
  err[i] = e;
}
int main() {
  int n = 1 << 24;
  double* d;
  cudaMalloc(&d, sizeof(double) * n);
  k<<<(n + 255) / 256, 256>>>(d, n);
  double* h = new double[n];
  cudaMemcpy(h, d, sizeof(double) * n, cudaMemcpyDeviceToHost);
  double mx = 0, mx40 = 0;
  for (int i = 0; i < n; ++i) {
    double x = 745.0 * ((double)i / n);
    if (h[i] > mx) mx = h[i];
    if (x < 40 && h[i] > mx40) mx40 = h[i];
  }
  printf("exp_neg_fast max rel err: %.3e overall (x in [0,745)), %.3e for x < 40 (ulp = 1.1e-16)\n", mx, mx40);
  ks<<<(n + 255) / 256, 256>>>(d, n);
  cudaMemcpy(h, d, sizeof(double) * n, cudaMemcpyDeviceToHost);
  mx = 0;
  for (int i = 0; i < n; ++i) if (h[i] > mx) mx = h[i];
  printf("sqrt_fast max rel err: %.3e (x in {0} U [2^-60, 2^60])\n", mx);
  return 0;
}
