// TMEM as per-thread scratch: alloc 512 columns in a 384-thread CTA, then
// tcgen05.st / tcgen05.ld (32x32b, x1/x2/x4) at unaligned column offsets,
// each warp in its lane quarter (warp % 4) and column slot (warp / 4).
// Checks the round trip and prints PASS/FAIL.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void st1(uint32_t a, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void st2(uint32_t a, uint32_t v0, uint32_t v1) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(v0), "r"(v1));
}
__device__ __forceinline__ void st4(uint32_t a, uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v0), "r"(v1),
               "r"(v2), "r"(v3));
}
__device__ __forceinline__ void ld4(uint32_t a, uint32_t& v0, uint32_t& v1, uint32_t& v2, uint32_t& v3) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
}
__device__ __forceinline__ void ld1(uint32_t a, uint32_t& v0) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v0) : "r"(a));
}

__global__ void __launch_bounds__(384, 1) k(uint32_t* out, int* err) {
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t taddr;
  const int w = threadIdx.x / 32;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr + ((uint32_t)(32 * (w % 4)) << 16) + (uint32_t)(w / 4) * 170u;
  const uint32_t t = threadIdx.x;
  // write 170 columns: x4 at col 0, x1 at 4, x2 at 5, x4 at 7, x1 ... then x1 fill
  st4(base + 0, t * 1000 + 0, t * 1000 + 1, t * 1000 + 2, t * 1000 + 3);
  st1(base + 4, t * 1000 + 4);
  st2(base + 5, t * 1000 + 5, t * 1000 + 6);
  st4(base + 7, t * 1000 + 7, t * 1000 + 8, t * 1000 + 9, t * 1000 + 10);
  for (int c = 11; c < 170; ++c) st1(base + c, t * 1000 + c);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  int bad = 0;
  for (int c = 0; c + 4 <= 170; c += 3) {  // unaligned x4 loads
    uint32_t v0, v1, v2, v3;
    ld4(base + c, v0, v1, v2, v3);
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v0), "+r"(v1), "+r"(v2), "+r"(v3));
    bad += (v0 != t * 1000 + c) + (v1 != t * 1000 + c + 1) + (v2 != t * 1000 + c + 2) + (v3 != t * 1000 + c + 3);
  }
  // overwrite then read back immediately (st -> ld ordering with wait::st)
  st1(base + 50, 7);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t v;
  ld1(base + 50, v);
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v));
  bad += v != 7;
  // and without wait::st
  st1(base + 51, 9);
  ld1(base + 51, v);
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v));
  const int nowait_ok = v == 9;
  if (bad) atomicAdd(err, bad);
  if (!nowait_ok) atomicAdd(err + 1, 1);
  sm[t] = v;
  out[blockIdx.x * 384 + t] = sm[t];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}

int main() {
  uint32_t* out;
  int* err;
  cudaMalloc(&out, 148 * 4 * 384 * 4);
  cudaMalloc(&err, 8);
  cudaMemset(err, 0, 8);
  const int smem = 210 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148 * 4, 384, smem>>>(out, err);
  cudaError_t e = cudaDeviceSynchronize();
  int h[2];
  cudaMemcpy(h, err, 8, cudaMemcpyDeviceToHost);
  printf("%s: cuda=%s mismatches=%d st->ld-without-wait failures=%d\n", (e == cudaSuccess && !h[0]) ? "PASS" : "FAIL",
         cudaGetErrorString(e), h[0], h[1]);
  return 0;
}
