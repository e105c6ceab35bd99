// Decomposition probe for k_pmc phase 1 on B200 (run under gpurun): samples/s of
//   A  Philox4x32-10 only (one block per sample)
//   B  A + two Box-Muller pairs
//   C  B + the 26 FFMA of the partial L z and the bound/decision logic (no queue)
//   D  C with 2 samples per lane per iteration (ILP 2)
// Each warp runs N samples of one synthetic cell, lane per sample, like k_pmc.
#include <cstdint>
#include <cstdio>
#include "warm.cuh"

struct Keys { uint32_t k[20]; };

__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const Keys& K,
                                       uint32_t* r) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k[2 * i];
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k[2 * i + 1];
    c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
  }
  r[0] = c0; r[1] = c1; r[2] = c2; r[3] = c3;
}
__device__ __forceinline__ float u23(uint32_t r) {
  return __uint_as_float(0x3f800000u | (r & 0x7fffffu)) - (1.0f - 0x1p-24f);
}
__device__ __forceinline__ void bm(uint32_t ra, uint32_t rb, float& z0, float& z1) {
  float ua = u23(ra);
  float fb = __uint_as_float(0x3f800000u | (rb & 0x7fffffu));
  float lg, R;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(ua));
  float r2 = fmaxf(-1.3862943611198906f * lg, 0.0f);
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(R) : "f"(r2));
  float s, co;
  __sincosf(fmaf(6.283185307179586f, fb, -9.424777586727f), &s, &co);
  z0 = -R * co;
  z1 = -R * s;
}

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(n) : "memory"); }

// H: warp-specialised -- warps 0-3 draw Philox blocks into a double-buffered
// shared ring, warps 4-7 finish (Box-Muller, L z, decision) the samples of the
// same cell.  Named barriers 4p + {0,1} (full) and 4p + {2,3} (empty) per pair p.
template <int PAIRS_ILP>
__global__ void __launch_bounds__(256, 2) k_ws(const float* __restrict__ Lg, uint32_t N, Keys K,
                                               uint32_t* __restrict__ out) {
  __shared__ uint4 ring[4][2][PAIRS_ILP * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, p = w & 3;
  const bool producer = w < 4;
  const uint32_t cell = blockIdx.x * 4 + p;
  const uint32_t nb = N / (32 * PAIRS_ILP);
  if (producer) {
    for (uint32_t b = 0; b < nb; ++b) {
      const int k = b & 1;
      if (b >= 2) bar_sync(4 * p + 2 + k, 64);
#pragma unroll
      for (int i = 0; i < PAIRS_ILP; ++i) {
        uint32_t r[4];
        philox(2u * (b * 32 * PAIRS_ILP + i * 32 + lane), cell, 0u, 0u, K, r);
        ring[p][k][i * 32 + lane] = make_uint4(r[0], r[1], r[2], r[3]);
      }
      bar_arrive(4 * p + k, 64);
    }
    return;
  }
  float L[36], m[8], B[4];
#pragma unroll
  for (int q = 0; q < 36; ++q) L[q] = Lg[q];
#pragma unroll
  for (int c = 0; c < 8; ++c) m[c] = Lg[36 + c];
#pragma unroll
  for (int c = 0; c < 4; ++c) B[c] = Lg[44 + c];
  uint32_t acc = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    const int k = b & 1;
    bar_sync(4 * p + k, 64);
    uint4 rr[PAIRS_ILP];
#pragma unroll
    for (int i = 0; i < PAIRS_ILP; ++i) rr[i] = ring[p][k][i * 32 + lane];
    if (b + 2 < nb) bar_arrive(4 * p + 2 + k, 64);
#pragma unroll
    for (int i = 0; i < PAIRS_ILP; ++i) {
      float z[4];
      bm(rr[i].x, rr[i].y, z[0], z[1]);
      bm(rr[i].z, rr[i].w, z[2], z[3]);
      float yp[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float y = m[c];
#pragma unroll
        for (int d = 0; d < 4 && d <= c; ++d) y = fmaf(L[c * (c + 1) / 2 + d], z[d], y);
        yp[c] = y;
      }
      const float mx03 = fmaxf(fmaxf(yp[0], yp[1]), fmaxf(yp[2], yp[3]));
      const float mn03 = fminf(fminf(yp[0], yp[1]), fminf(yp[2], yp[3]));
      float hi_max = mx03, lo_min = mn03, lo_max = mx03, hi_min = mn03;
#pragma unroll
      for (int c = 4; c < 8; ++c) {
        const float lo = yp[c] - B[c - 4], hi = yp[c] + B[c - 4];
        hi_max = fmaxf(hi_max, hi); lo_min = fminf(lo_min, lo);
        lo_max = fmaxf(lo_max, lo); hi_min = fminf(hi_min, hi);
      }
      const bool cross = lo_max >= 0.0f && hi_min <= 0.0f;
      const bool decided = hi_max < 0.0f || lo_min > 0.0f || cross;
      acc += cross ? 1u : 0u;
      acc += decided ? 0u : 65536u;
    }
  }
  if (acc == 0x12345) out[0] = acc;
  if (lane == 0) out[1 + cell % 1024] = acc;
}

// I: one warp per CTA, so the cell index (blockIdx.x) and its L, m, B are
// warp-uniform: the compiler may keep them in uniform registers (UR operands of
// FFMA / FFMA2), freeing vector-register bandwidth and capacity.
__global__ void __launch_bounds__(32) k_uniform(const float* __restrict__ Lcells, uint32_t N, Keys K,
                                                uint32_t* __restrict__ out) {
  const int lane = threadIdx.x;
  const uint32_t cell = blockIdx.x;
  const float* Lg = Lcells + 48 * (cell & 1023);
  float L[36], m[8], B[4];
#pragma unroll
  for (int q = 0; q < 36; ++q) L[q] = Lg[q];
#pragma unroll
  for (int c = 0; c < 8; ++c) m[c] = Lg[36 + c];
#pragma unroll
  for (int c = 0; c < 4; ++c) B[c] = Lg[44 + c];
  uint32_t acc = 0;
  auto one = [&](uint32_t s) {
    uint32_t r[4];
    philox(2u * s, cell, 0u, 0u, K, r);
    float z[4];
    bm(r[0], r[1], z[0], z[1]);
    bm(r[2], r[3], z[2], z[3]);
    float yp[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float y = m[c];
#pragma unroll
      for (int d = 0; d < 4 && d <= c; ++d) y = fmaf(L[c * (c + 1) / 2 + d], z[d], y);
      yp[c] = y;
    }
    const float mx03 = fmaxf(fmaxf(yp[0], yp[1]), fmaxf(yp[2], yp[3]));
    const float mn03 = fminf(fminf(yp[0], yp[1]), fminf(yp[2], yp[3]));
    float hi_max = mx03, lo_min = mn03, lo_max = mx03, hi_min = mn03;
#pragma unroll
    for (int c = 4; c < 8; ++c) {
      const float lo = yp[c] - B[c - 4], hi = yp[c] + B[c - 4];
      hi_max = fmaxf(hi_max, hi); lo_min = fminf(lo_min, lo);
      lo_max = fmaxf(lo_max, lo); hi_min = fminf(hi_min, hi);
    }
    const bool cross = lo_max >= 0.0f && hi_min <= 0.0f;
    const bool decided = hi_max < 0.0f || lo_min > 0.0f || cross;
    acc += cross ? 1u : 0u;
    acc += decided ? 0u : 65536u;
  };
  for (uint32_t b = 0; b < N; b += 64) { one(b + lane); one(b + 32 + lane); }
  if (acc == 0x12345) out[0] = acc;
  if (lane == 0) out[1 + cell % 1024] = acc;
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_part(const float* __restrict__ Lg, uint32_t N, Keys K,
                                                 uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint32_t cell = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float L[36], m[8], B[4];
#pragma unroll
  for (int p = 0; p < 36; ++p) L[p] = Lg[p];
#pragma unroll
  for (int c = 0; c < 8; ++c) m[c] = Lg[36 + c];
#pragma unroll
  for (int c = 0; c < 4; ++c) B[c] = Lg[44 + c];
  uint32_t acc = 0;
  float facc = 0.f;
  auto draw = [&](uint32_t s, uint32_t (&r)[4]) {
    if (MODE == 4) {   // cheap hash instead of Philox (isolates the rest)
      uint32_t h = s * 0x9E3779B9u + cell;
      r[0] = h; r[1] = h ^ 0x5bd1e995u; r[2] = h * 3u; r[3] = h ^ 0x1b873593u;
    } else {
      philox(2u * s, cell, 0u, 0u, K, r);
    }
  };
  auto finish = [&](const uint32_t (&r)[4]) {
    if (MODE == 0) { acc ^= r[0] ^ r[1] ^ r[2] ^ r[3]; return; }
    float z[4];
    if (MODE == 5) {   // no Box-Muller: uniforms as stand-in normals
#pragma unroll
      for (int i = 0; i < 4; ++i) z[i] = __uint_as_float(0x3f800000u | (r[i] >> 9)) - 1.5f;
    } else {
      bm(r[0], r[1], z[0], z[1]);
      bm(r[2], r[3], z[2], z[3]);
    }
    if (MODE == 1) { facc += z[0] + z[1] + z[2] + z[3]; return; }
    float yp[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float y = m[c];
#pragma unroll
      for (int d = 0; d < 4 && d <= c; ++d) y = fmaf(L[c * (c + 1) / 2 + d], z[d], y);
      yp[c] = y;
    }
    const float mx03 = fmaxf(fmaxf(yp[0], yp[1]), fmaxf(yp[2], yp[3]));
    const float mn03 = fminf(fminf(yp[0], yp[1]), fminf(yp[2], yp[3]));
    float hi_max = mx03, lo_min = mn03, lo_max = mx03, hi_min = mn03;
#pragma unroll
    for (int c = 4; c < 8; ++c) {
      const float lo = yp[c] - B[c - 4], hi = yp[c] + B[c - 4];
      hi_max = fmaxf(hi_max, hi); lo_min = fminf(lo_min, lo);
      lo_max = fmaxf(lo_max, lo); hi_min = fminf(hi_min, hi);
    }
    const bool cross = lo_max >= 0.0f && hi_min <= 0.0f;
    const bool decided = hi_max < 0.0f || lo_min > 0.0f || cross;
    acc += cross ? 1u : 0u;
    acc += decided ? 0u : 65536u;
  };
  auto one = [&](uint32_t s) {
    uint32_t r[4];
    draw(s, r);
    finish(r);
  };
  if (MODE == 3 || MODE == 4 || MODE == 5) {
    for (uint32_t b = 0; b < N; b += 64) { one(b + lane); one(b + 32 + lane); }
  } else if (MODE == 6) {   // software-pipelined D
    uint32_t ra[4], rb[4];
    draw(lane, ra);
    draw(32 + lane, rb);
    for (uint32_t b = 0; b < N; b += 64) {
      uint32_t na[4], nb[4];
      draw(b + 64 + lane, na);
      draw(b + 96 + lane, nb);
      finish(ra);
      finish(rb);
#pragma unroll
      for (int i = 0; i < 4; ++i) { ra[i] = na[i]; rb[i] = nb[i]; }
    }
  } else {
    for (uint32_t b = 0; b < N; b += 32) one(b + lane);
  }
  if (acc == 0x12345 || facc == 1.2345f) out[0] = acc;
  if (lane == 0) out[1 + cell % 1024] = acc;
}

int main() {
  const double clk_mhz = warm_and_clock_mhz();
  float hL[48];
  for (int p = 0; p < 36; ++p) hL[p] = 0.05f + 0.01f * (p % 7);
  for (int c = 0; c < 8; ++c) hL[36 + c] = 0.1f * (c - 4);
  for (int c = 0; c < 4; ++c) hL[44 + c] = 0.2f;
  float* dL; uint32_t* dout;
  cudaMalloc(&dL, sizeof hL); cudaMalloc(&dout, 4 * 2048);
  cudaMemcpy(dL, hL, sizeof hL, cudaMemcpyHostToDevice);
  Keys K;
  for (int r = 0; r < 10; ++r) { K.k[2 * r] = 7u + r * 0x9E3779B9u; K.k[2 * r + 1] = 9u + r * 0xBB67AE85u; }
  const uint32_t N = 4096;
  const int cells = 148 * 16 * 64, threads = 256, blocks = cells * 32 / threads;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[7] = {"A philox", "B +box-muller", "C +Lz+decision", "D C with ILP2",
                          "E D, hash not philox", "F D, no box-muller", "G D software-pipelined"};
  {
    float* dLc;
    cudaMalloc(&dLc, sizeof(float) * 48 * 1024);
    float hc[48 * 1024];
    for (int c = 0; c < 1024; ++c) for (int q = 0; q < 48; ++q) hc[48 * c + q] = hL[q] * (1.0f + 1e-3f * (c % 7));
    cudaMemcpy(dLc, hc, sizeof hc, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_uniform<<<cells, 32>>>(dLc, N, K, dout);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double sps = (double)cells * N / (ms * 1e-3);
      if (rep) printf("I warp-per-CTA uniform L %8.3f ms  %.3e samples/s  %.1f SMSP-cycles per warp-step\n", ms, sps,
                      148.0 * 4 * (clk_mhz * 1e6) / (sps / 32));
    }
  }
  for (int rep = 0; rep < 2; ++rep)
    for (int ilp = 1; ilp <= 2; ++ilp) {
      // warp-specialised: 4 cells per block of 8 warps -> half the blocks' cells per launch
      const int wblocks = cells / 4;
      cudaEventRecord(e0);
      if (ilp == 1) k_ws<1><<<wblocks, threads>>>(dL, N, K, dout);
      else k_ws<2><<<wblocks, threads>>>(dL, N, K, dout);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double sps = (double)cells * N / (ms * 1e-3);
      if (rep) printf("H warp-specialised ilp%d %8.3f ms  %.3e samples/s  %.1f SMSP-cycles per 32 samples\n", ilp, ms,
                      sps, 148.0 * 4 * (clk_mhz * 1e6) / (sps / 32));
    }
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 7; ++mode) {
      cudaEventRecord(e0);
      if (mode == 0) k_part<0><<<blocks, threads>>>(dL, N, K, dout);
      if (mode == 1) k_part<1><<<blocks, threads>>>(dL, N, K, dout);
      if (mode == 2) k_part<2><<<blocks, threads>>>(dL, N, K, dout);
      if (mode == 3) k_part<3><<<blocks, threads>>>(dL, N, K, dout);
      if (mode == 4) k_part<4><<<blocks, threads>>>(dL, N, K, dout);
      if (mode == 5) k_part<5><<<blocks, threads>>>(dL, N, K, dout);
      if (mode == 6) k_part<6><<<blocks, threads>>>(dL, N, K, dout);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double sps = (double)cells * N / (ms * 1e-3);
      if (rep) printf("%-16s %8.3f ms  %.3e samples/s  %.1f SMSP-cycles per warp-step\n", names[mode], ms, sps,
                      148.0 * 4 * (clk_mhz * 1e6) / (sps / 32));
    }
  return 0;
}
