// Instruction-throughput microbenchmarks on B200 (sm_100a): lane-ops/clk/SM
// of the instruction classes the decode kernel uses, 8 independent chains
// per thread, 64 warps/SM, and the same at 12 warps/SM (the decode's
// occupancy). Build+run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ub ubench.cu && ./ub
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t h2u(half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ half2 u2h(uint32_t u) { return *reinterpret_cast<half2*>(&u); }

template <int OP>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  const uint32_t c = seed ^ 0x3C003C00u, d = seed ^ 0x57F057F0u;
  __shared__ uint16_t sm[8192];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t x = a[i];
      if (OP == 0) x = h2u(__hmin2(u2h(x), __habs2(u2h(d))));                       // HMNMX2
      if (OP == 1) x = h2u(__hfma2(u2h(x), u2h(c), u2h(d)));                         // HFMA2
      if (OP == 2) x = h2u(__hadd2(u2h(x), u2h(d)));                                 // HADD2
      if (OP == 3) asm volatile("prmt.b32 %0, %0, %1, 0x4140;" : "+r"(x) : "r"(d));  // PRMT
      if (OP == 4) x = (x & 0x80008000u) | c;                                        // LOP3
      if (OP == 5) { uint32_t y = x + c; x = min(y, y - d); }                         // VIADD+VIADDMNMX
      if (OP == 6) x = h2u(__hmin2(__hmin2(u2h(x), u2h(c)), u2h(d)));                 // VHMNMX
      if (OP == 7) x = h2u(__hsub2_sat(__habs2(u2h(x)), u2h(d)));                     // HADD2.SAT
      if (OP == 10) x = __float_as_uint(fmaf(__uint_as_float(x), __uint_as_float(c), __uint_as_float(d)));  // FFMA
      if (OP == 11) x = __float_as_uint(__uint_as_float(x) + __uint_as_float(d));     // FADD
      if (OP == 12) x = __float_as_uint(fminf(__uint_as_float(x), fabsf(__uint_as_float(d))));  // FMNMX
      if (OP == 13) x = x * c + d;                                                    // IMAD
      if (OP == 14) x = x + c + d;                                                    // IADD3
      if (OP == 15) x = __vadd2(x, d);                                                // VIADD.16x2
      if (OP == 16) x = __vmins2(x, d);                                               // VIMNMX.S16x2
      if (OP == 17) x = __viaddmax_s16x2(x, c, d);                                    // VIADDMNMX.S16x2
      if (OP == 18) x = __vimin3_s16x2(x, c, d);                                      // VIMNMX3.S16x2
      if (OP == 19) x = __funnelshift_l(x, d, 7);                                     // SHF
      if (OP == 20) x = __heq2_mask(u2h(x), u2h(d)) ^ x;                              // HSET2 + LOP
      if (OP == 21) x = h2u(__hmax2(u2h(x), u2h(d)));                                 // HMNMX2 max no abs
      if (OP == 22) x = __float_as_uint(fminf(fmaxf(__uint_as_float(x), __uint_as_float(c)), __uint_as_float(d)));
      a[i] = x;
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  if (r == 0x12345678u) out[0] = r;
}

template <int OP>
void run(const char* name, int blocks_per_sm, int threads) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* d;
  cudaMalloc(&d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<OP><<<sms * blocks_per_sm, threads>>>(d, iters, 0x1234 + rep);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = ms < best ? ms : best;
  }
  const double ops = 8.0 * iters * (double)threads * blocks_per_sm * sms;
  const double per_clk_sm = ops / (best * 1e-3) / (clk * 1e3) / sms;
  printf("%-18s warps/SM=%2d  %7.1f lane-ops/clk/SM  (%.3f warp-inst/clk/SMSP)\n", name,
         blocks_per_sm * threads / 32, per_clk_sm, per_clk_sm / 32 / 4);
}

int main() {
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int bps = cfg ? 1 : 4, thr = cfg ? 384 : 512;
    run<0>("HMNMX2|abs", bps, thr);
    run<1>("HFMA2", bps, thr);
    run<2>("HADD2", bps, thr);
    run<3>("PRMT", bps, thr);
    run<4>("LOP3", bps, thr);
    run<5>("VIADD+VIADDMNMX/2", bps, thr);
    run<6>("VHMNMX(3in)", bps, thr);
    run<7>("HADD2.SAT|abs", bps, thr);
    run<10>("FFMA", bps, thr);
    run<11>("FADD", bps, thr);
    run<12>("FMNMX|abs", bps, thr);
    run<13>("IMAD", bps, thr);
    run<14>("IADD3", bps, thr);
    run<15>("VIADD.16x2", bps, thr);
    run<16>("VIMNMX.S16x2", bps, thr);
    run<17>("VIADDMNMX.S16x2", bps, thr);
    run<18>("VIMNMX3.S16x2", bps, thr);
    run<19>("SHF", bps, thr);
    run<20>("HSET2+LOP3/2", bps, thr);
    run<21>("HMNMX2 max", bps, thr);
    run<22>("FMNMX x2/2", bps, thr);
  }
  return 0;
}
