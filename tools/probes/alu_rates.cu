// Issue-rate probe for the k_pmc instruction mix on B200 (run under gpurun).
// Each kernel runs 8 independent chains of one instruction class per thread over
// a full-occupancy grid; the printed number is warp-instructions per SM per clock
// at the measured time (4.0 = one per SMSP per clock = full issue).
#include <cstdint>
#include <cstdio>
#include "warm.cuh"

#define CHAINS 8
#define DEFK(name, T, init, ...)                                          \
  __global__ void name(T* out, int iters, T s) {                          \
    T a[CHAINS];                                                          \
    for (int q = 0; q < CHAINS; ++q) a[q] = (T)(threadIdx.x + q) * init;  \
    for (int it = 0; it < iters; ++it) {                                  \
      _Pragma("unroll") for (int q = 0; q < CHAINS; ++q) { __VA_ARGS__; }      \
    }                                                                     \
    T t = 0;                                                              \
    for (int q = 0; q < CHAINS; ++q) t += a[q];                           \
    if (t == (T)12345) out[0] = t;                                        \
  }

// one IMAD.WIDE.U32 per chain step (hi and lo folded by a 3-input LOP3 every 2nd step)
DEFK(k_imadwide, uint32_t, 1u, {
  uint32_t lo, hi;
  asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(*(uint64_t*)&lo) : "r"(a[q]), "r"(0xD2511F53u));
  (void)hi;
  a[q] = lo;
})
DEFK(k_lop3, uint32_t, 1u, { asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[q]) : "r"(s), "r"(q * 77u)); })
DEFK(k_ffma3, float, 1e-9f, { asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(s), "f"(s)); })
DEFK(k_fmul, float, 1e-9f, { asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(s)); })
DEFK(k_fadd, float, 1e-9f, { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(s)); })
DEFK(k_fmnmx, float, 1e-9f, { asm volatile("max.f32 %0, %0, %1;" : "+f"(a[q]) : "f"(s)); })
DEFK(k_lg2, float, 1e-3f, { asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(a[q])); })
DEFK(k_sin, float, 1e-3f, { asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(a[q])); })
DEFK(k_sqrt, float, 1e-3f, { asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(a[q])); })
// Philox round shape: IMAD.WIDE + LOP3 pairs
DEFK(k_philox_pair, uint32_t, 1u, {
  uint64_t p;
  asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[q]), "r"(0xD2511F53u));
  uint32_t h = (uint32_t)(p >> 32), l = (uint32_t)p;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(a[q]) : "r"(h), "r"(l), "r"(s));
})
// FFMA 3-reg + LOP3 alternating (fma pipe + alu pipe)
DEFK(k_ffma_lop3, float, 1e-9f, {
  asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[q]) : "f"(s), "f"(s));
  uint32_t u = __float_as_uint(a[q]);
  asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u) : "r"(7u), "r"(q * 77u));
  a[q] = __uint_as_float(u);
})

typedef void (*kfn_u)(uint32_t*, int, uint32_t);
typedef void (*kfn_f)(float*, int, float);

int main() {
  const double clk_mhz = warm_and_clock_mhz();
  void* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  auto report = [&](const char* name, float ms, double instr_per_step) {
    double warp_instr = instr_per_step * CHAINS * (double)iters * blocks * (threads / 32);
    double per_sm_clk = warp_instr / (ms * 1e-3) / sms / (clk_mhz * 1e6);
    printf("%-14s %7.3f ms  %.3f warp-instr/SM/clk (at 1.965 GHz)\n", name, ms, per_sm_clk);
  };
  struct U { const char* n; kfn_u f; double ipc; } us[] = {
      {"IMAD.WIDE", k_imadwide, 1}, {"LOP3", k_lop3, 1}, {"IMADW+LOP3", k_philox_pair, 2}};
  struct F { const char* n; kfn_f f; double ipc; } fs[] = {
      {"FFMA(3reg)", k_ffma3, 1}, {"FMUL", k_fmul, 1}, {"FADD", k_fadd, 1}, {"FMNMX", k_fmnmx, 1},
      {"MUFU.LG2", k_lg2, 1},    {"MUFU.SIN", k_sin, 1}, {"MUFU.SQRT", k_sqrt, 1}, {"FFMA+LOP3", k_ffma_lop3, 2}};
  printf("sms=%d clock attr=%d kHz\n", sms, clk_khz);
  for (int rep = 0; rep < 2; ++rep) {
    for (auto& u : us) {
      float ms;
      cudaEventRecord(e0);
      u.f<<<blocks, threads>>>((uint32_t*)d, iters, 3u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) report(u.n, ms, u.ipc);
    }
    for (auto& f : fs) {
      float ms;
      cudaEventRecord(e0);
      f.f<<<blocks, threads>>>((float*)d, iters, 0.999f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) report(f.n, ms, f.ipc);
    }
  }
  return 0;
}
