// Accuracy of the brick kernels' exp_neg_tab / exp_neg_fast / sqrt_fast (csrc/expfast.cuh)
// against libm on the device.  nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2512_12442_b200/csrc
#include <cstdio>
#include <cmath>
#include "expfast.cuh"
using namespace lcp;

__global__ void k(double* e_tab, double* e_fast, int n) {
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = c_exp2_64[threadIdx.x];
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = 745.0 * ((double)i / n);
  double b = exp(-x);
  double a = exp_neg_tab(x, tab), f = exp_neg_fast(x);
  e_tab[i] = b > 1e-300 ? fabs(a - b) / b : fabs(a - b);
  e_fast[i] = b > 1e-300 ? fabs(f - b) / b : fabs(f - b);
}
int main() {
  int n = 1 << 24;
  double *d1, *d2;
  cudaMalloc(&d1, sizeof(double) * n);
  cudaMalloc(&d2, sizeof(double) * n);
  k<<<(n + 255) / 256, 256>>>(d1, d2, n);
  double* h1 = new double[n];
  double* h2 = new double[n];
  cudaMemcpy(h1, d1, sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, d2, sizeof(double) * n, cudaMemcpyDeviceToHost);
  double m1 = 0, m2 = 0, m140 = 0, m240 = 0;
  for (int i = 0; i < n; ++i) {
    double x = 745.0 * ((double)i / n);
    m1 = fmax(m1, h1[i]); m2 = fmax(m2, h2[i]);
    if (x < 40) { m140 = fmax(m140, h1[i]); m240 = fmax(m240, h2[i]); }
  }
  printf("exp_neg_tab  max rel err %.3e (x < 745), %.3e (x < 40); ulp = 1.1e-16\n", m1, m140);
  printf("exp_neg_fast max rel err %.3e (x < 745), %.3e (x < 40)\n", m2, m240);
  return 0;
}
