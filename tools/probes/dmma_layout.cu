// Probe of the mma.sync m8n8k4 f64 fragment layout on sm_100a (run under gpurun).
#include <cstdio>
__device__ void mma(double a, double b, double& d0, double& d1) {
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__global__ void k(double* out) {
  int l = threadIdx.x;
  double d0, d1;
  mma((double)l, 1.0, d0, d1);   // D[r][c] = sum_k A[r][k]
  out[4 * l + 0] = d0; out[4 * l + 1] = d1;
  mma(1.0, (double)l, d0, d1);   // D[r][c] = sum_k B[k][c]
  out[4 * l + 2] = d0; out[4 * l + 3] = d1;
}
int main() {
  double* d; cudaMalloc(&d, 32 * 4 * sizeof(double));
  k<<<1, 32>>>(d);
  double h[128]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int ok = 1;
  for (int l = 0; l < 32; ++l) {
    double ea = 16 * (l >> 2) + 6;                      // A row r = lane >> 2 holds lanes 4r..4r+3
    double eb0 = 16 * (2 * (l % 4)) + 6, eb1 = 16 * (2 * (l % 4) + 1) + 6;   // B col c = lane >> 2
    printf("lane %2d: rowsumA %.0f %.0f  colsumB %.0f %.0f  expect %.0f | %.0f %.0f\n", l, h[4*l], h[4*l+1], h[4*l+2], h[4*l+3], ea, eb0, eb1);
    ok &= h[4*l] == ea && h[4*l+1] == ea && h[4*l+2] == eb0 && h[4*l+3] == eb1;
  }
  printf("layout %s\n", ok ? "CONFIRMED" : "DIFFERENT");
  return 0;
}
