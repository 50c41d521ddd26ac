// Device-side building blocks shared by the nrldpc kernels (sm_100a).
//
// Exact int8 layered min-sum in packed half2 arithmetic
// -----------------------------------------------------
// The reference's int8 engine (/root/reference/pkg/src/ldpclab/decoder.py:
// 295-320) widens int8 posteriors L and messages M to int32 and computes
//     t   = clamp127(L - M)          (decoder.py:300)
//     m1, m2, S over |t|, sign(t)    (decoder.py:305, kernels.py:246-257)
//     b   = floor(beta * m)          (decoder.py:208-212)
//     out = (S ^ sign t) ? -b : b    (decoder.py:315-316)
//     L'  = clamp127(t + out)        (decoder.py:318)
// Every intermediate is an integer with |x| <= 254, so IEEE half represents
// it exactly and HADD2/HFMA2/HMNMX2 reproduce the integer results bit for
// bit. Two codewords ride in the two half lanes of one 32-bit register
// (LANES=2), so one SASS instruction does the work of two codeword-edges;
// |x| comes for free as an HMNMX2 operand modifier.
//
// Storage is one biased byte per value and codeword: u = v + 128 (the int8
// bit pattern with the top bit flipped). One PRMT with the byte 0x64 turns a
// pair of stored bytes into the half2 {1024+u_a, 1024+u_b} = {1152+v_a,
// 1152+v_b}; subtracting two such values yields the exact unbiased t, and
// HFMA2(y, +-1, 1152) maps a result back into the same biased form, whose
// low byte is again u. The bias also makes a -0.0 result impossible to store.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#define NR_MAX_ROWS 46
#define NR_MAX_EDGES 316
#define NR_MAX_BLOCKS 68
#define NR_MAX_TAB 456

namespace nr {

struct alignas(16) KParams {
  int z;
  int k_b;
  int rows;          // rows_used
  int n_blocks;      // k_b + rows_used
  int n_edges;       // sum of w_r over the used rows
  int groups;        // codeword groups per CTA (a group = Z threads)
  int max_iter;
  int early_stop;    // NRLDPC_STOP_*
  int crc_len;
  uint32_t crc_poly;
  int trace;         // nonzero: record per-iteration trace, never exit early
  int vec_load;      // rows are 16-byte aligned: vectorized prologue
  int words;         // ceil(K/32)
  long long batch;
  uint32_t l_bytes;  // per group: n_blocks*z*LANES rounded up to 16
  uint32_t m_bytes;  // per group: z * m_stride rounded up to 16
  uint32_t m_stride; // bytes between consecutive z message rows (odd # words)
  int e_reg;         // edges whose messages live in registers (rows < nreg)
  uint32_t magic;    // 0x64646464: PRMT filler byte (half exponent of 1024)
  uint32_t one;      // 0x3C003C00: half2 {1.0, 1.0}
  uint32_t abs_base; // nonzero: cb holds shared-window addresses, L starts here
  uint32_t tm_cols;  // TM layout: tensor-memory message columns per thread
  uint32_t tm_slot;  // TM layout: columns per thread slot (512 / warps per lane quarter, rounded down)
  uint32_t tm_r45[2];  // TM layout, register-row shapes: TMEM columns of rows 4 and 5
  uint16_t row_start[NR_MAX_ROWS + 1];  // first edge of each row (message offsets)
  uint16_t tab_start[NR_MAX_ROWS + 1];  // row's first slot in sh/cb (multiple of 4)
  uint8_t bar_after[NR_MAX_ROWS];       // 0: next row is column-disjoint from this layer
  // layer units of the BG1/BG2 kernels after the register rows (one row or
  // two fused column-disjoint rows): a = {code wa | wb << 8, barrier after,
  // table slot / 4 of row a, message byte offset of row a}, b = {table slot
  // / 4 of row b, message byte offset of row b, odd-edge slot offsets of rows
  // a and b (paired message layout)}. One spare entry for the prefetch.
  int n_units;
  alignas(16) uint4 unit_a[NR_MAX_ROWS + 1];
  alignas(16) uint4 unit_b[NR_MAX_ROWS + 1];
  // per-edge graph tables, each row padded to a multiple of 4 slots so a row
  // loads them with 128-bit uniform constant loads
  alignas(16) uint32_t sh[NR_MAX_TAB];  // shift * LANES (bytes)
  alignas(16) uint32_t cb[NR_MAX_TAB];  // col * z * LANES (bytes) [+ abs_base]
  const uint32_t* crc_tab;          // crc mode: rem(x^(K-1-i+L), g), device memory
  uint32_t beta_f;                  // float engines: dtype(beta) (f32 bits or half2)
  int beta_mode;                    // 1: half-arithmetic beta (beta_h, ndelta_h, c_h)
  uint32_t beta_h, ndelta_h, c_h;   // half2 constants of the arithmetic beta rule
  uint16_t lut[128];                // floor(beta*m) as half bits, m = 0..127
};

struct KOut {
  uint32_t* bits;
  int32_t* iters;
  int32_t* synd;
  uint8_t* success;
  uint8_t* crc_ok;
  int32_t* trace_w;
  float* trace_m;
  int32_t* status;
  int32_t* work;  // lane-refill kernel: next-codeword counter (zeroed per launch)
};

// Several shapes in one decode launch (k_decode_i8_multi): the parameter
// block holds each shape's KParams (5.8 KB each; kernel parameters are
// limited to 32 KB), its input and outputs, and its last CTA + 1.
constexpr int kMultiShapes = 5;
struct alignas(16) KMulti {
  KParams s[kMultiShapes];
  const int8_t* llr[kMultiShapes];
  KOut o[kMultiShapes];
  int cta_end[kMultiShapes];
  int n;
};
static_assert(sizeof(KMulti) <= 32764, "kernel parameter block limit");

__device__ __forceinline__ uint32_t h2u(half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ half2 u2h(uint32_t u) { return *reinterpret_cast<half2*>(&u); }

// biased byte(s) -> half2 {1152+v_a, 1152+v_b}
// `magic` must hold 0x64646464 in a register (kept opaque so ptxas puts the
// selector, not the constant, in PRMT's immediate slot).
template <int LANES>
__device__ __forceinline__ half2 unpack_elem(uint32_t raw, uint32_t magic) {
  uint32_t d;
  if (LANES == 2)
    asm("prmt.b32 %0, %1, %2, 0x4140;" : "=r"(d) : "r"(raw), "r"(magic));
  else
    asm("prmt.b32 %0, %1, %2, 0x4040;" : "=r"(d) : "r"(raw), "r"(magic));
  return u2h(d);
}

// biased half2 -> stored byte(s) (low byte of each lane)
template <int LANES>
__device__ __forceinline__ uint32_t pack_elem(half2 h) {
  return LANES == 2 ? __byte_perm(h2u(h), 0, 0x0020) : h2u(h);
}

// ---- checked build (NRLDPC_CHECKED, libnrldpc_checked.so) ------------------
// compute-sanitizer is not available on the GPU pool, so the checked build
// carries its own device-side checks: every shared-memory access through the
// helpers below must fall inside the CTA's dynamic shared memory and be
// naturally aligned; every tensor-memory access must stay in the executing
// warp's lane quarter and below column 512; result writes must index a
// codeword of the batch (NR_CHECK at the call sites). A violation traps.
#ifdef NRLDPC_CHECKED
extern __shared__ __align__(16) uint8_t nr_chk_dyn_smem[];
__device__ __forceinline__ void chk_smem(uint32_t a, uint32_t n) {
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(nr_chk_dyn_smem);
  if (a < base || a + n > base + dyn || (a & (n - 1)) != 0) __trap();
}
__device__ __forceinline__ void chk_tmem(uint32_t a, uint32_t n) {
  if ((a >> 16) != 32u * ((threadIdx.x >> 5) & 3u) || (a & 0xFFFFu) + n > 512u) __trap();
}
#define NR_CHECK(c)       \
  do {                    \
    if (!(c)) __trap();   \
  } while (0)
#else
__device__ __forceinline__ void chk_smem(uint32_t, uint32_t) {}
__device__ __forceinline__ void chk_tmem(uint32_t, uint32_t) {}
#define NR_CHECK(c) \
  do {              \
  } while (0)
#endif

template <int LANES>
__device__ __forceinline__ uint32_t ld_elem(const uint8_t* p) {
  chk_smem((uint32_t)__cvta_generic_to_shared(p), LANES);
  if (LANES == 2) return *reinterpret_cast<const uint16_t*>(p);
  return *p;
}

template <int LANES>
__device__ __forceinline__ void st_elem(uint8_t* p, uint32_t v) {
  chk_smem((uint32_t)__cvta_generic_to_shared(p), LANES);
  if (LANES == 2) *reinterpret_cast<uint16_t*>(p) = (uint16_t)v;
  else *p = (uint8_t)v;
}

// Predicated shared store (no branch): padding threads compute but never
// store. All loads of a row precede its stores through register
// dependences (every stored value depends on m1/m2/S of the whole row),
// and rows are separated by __syncthreads, so no memory clobber is needed.
template <int LANES>
__device__ __forceinline__ void st_elem_if(uint8_t* p, uint32_t v, bool ok) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  chk_smem(a, LANES);
  if (LANES == 2)
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u16 [%0], %1; }" ::"r"(a), "h"((uint16_t)v),
                 "r"((uint32_t)ok));
  else
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u8 [%0], %1; }" ::"r"(a), "h"((uint16_t)v),
                 "r"((uint32_t)ok));
}

// The same accesses on absolute shared-window addresses. With the graph
// table already holding (column base + window base), ptxas folds the add into
// the load/store as [R + UR] and the per-edge address costs two instructions.
// volatile keeps NVVM from moving the loads across barriers.
template <int LANES>
__device__ __forceinline__ uint32_t lds_elem(uint32_t a) {
  chk_smem(a, LANES);
  uint16_t v;
  if (LANES == 2)
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  else
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

template <int LANES>
__device__ __forceinline__ void sts_elem_if(uint32_t a, uint32_t v, bool ok) {
  chk_smem(a, LANES);
  if (LANES == 2)
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u16 [%0], %1; }" ::"r"(a), "h"((uint16_t)v),
                 "r"((uint32_t)ok));
  else
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u8 [%0], %1; }" ::"r"(a), "h"((uint16_t)v),
                 "r"((uint32_t)ok));
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  chk_smem(a, 4);
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void sts_u32_if(uint32_t a, uint32_t v, bool ok) {
  chk_smem(a, 4);
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u32 [%0], %1; }" ::"r"(a), "r"(v),
               "r"((uint32_t)ok));
}

__device__ __forceinline__ void lds_v2(uint32_t a, uint32_t& x, uint32_t& y) {
  chk_smem(a, 8);
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
}

__device__ __forceinline__ void sts_v2(uint32_t a, uint32_t x, uint32_t y) {
  chk_smem(a, 8);
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}

__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  chk_smem(a, 4);
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}

// Tensor memory as per-thread message storage (TM layout, see k_decode_i8).
// tcgen05.ld / tcgen05.st with the 32x32b shape move N consecutive 32-bit
// columns of the executing thread's own TMEM lane; the address is warp-uniform
// (lane quarter in bits 31:16, column in bits 15:0) and the instructions are
// warp-collective. A row of W messages is one x4 plus an x2 / x1 remainder.
__device__ __forceinline__ void tm_ld1(uint32_t a, uint32_t& r0) {
  chk_tmem(a, 1);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(a));
}
__device__ __forceinline__ void tm_ld2(uint32_t a, uint32_t& r0, uint32_t& r1) {
  chk_tmem(a, 2);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(a));
}
__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  chk_tmem(a, 4);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void tm_st1(uint32_t a, uint32_t r0) {
  chk_tmem(a, 1);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "r"(r0));
}
__device__ __forceinline__ void tm_st2(uint32_t a, uint32_t r0, uint32_t r1) {
  chk_tmem(a, 2);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(r0), "r"(r1));
}
__device__ __forceinline__ void tm_st4(uint32_t a, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  chk_tmem(a, 4);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3));
}

template <int W>
__device__ __forceinline__ void tm_ld_row(uint32_t a, uint32_t (&r)[W]) {
#pragma unroll
  for (int k = 0; k + 4 <= W; k += 4) tm_ld4(a + k, r[k], r[k + 1], r[k + 2], r[k + 3]);
  constexpr int k2 = W / 4 * 4;
  if constexpr ((W & 2) != 0) tm_ld2(a + k2, r[k2], r[k2 + 1]);
  if constexpr ((W & 1) != 0) tm_ld1(a + W - 1, r[W - 1]);
}

template <int W>
__device__ __forceinline__ void tm_st_row(uint32_t a, const uint32_t (&r)[W]) {
#pragma unroll
  for (int k = 0; k + 4 <= W; k += 4) tm_st4(a + k, r[k], r[k + 1], r[k + 2], r[k + 3]);
  constexpr int k2 = W / 4 * 4;
  if constexpr ((W & 2) != 0) tm_st2(a + k2, r[k2], r[k2 + 1]);
  if constexpr ((W & 1) != 0) tm_st1(a + W - 1, r[W - 1]);
}

// Waits for this thread's outstanding tcgen05.ld; the empty "+r" statements
// after it make every later use of r depend on the wait.
template <int W>
__device__ __forceinline__ void tm_wait_ld(uint32_t (&r)[W]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int j = 0; j < W; ++j) asm volatile("" : "+r"(r[j]));
}

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }

// beta LUT on a half2 of integer magnitudes 0..127
__device__ __forceinline__ half2 beta_lut2(const uint16_t* lut, half2 m) {
  const uint32_t x = h2u(__hadd2(m, u2h(0x64006400u)));  // lanes 0x6400|m
  const uint32_t lo = lut[x & 0x7Fu];
  const uint32_t hi = lut[(x >> 16) & 0x7Fu];
  return u2h(lo | (hi << 16));
}

}  // namespace nr
