// nrldpc: B200-native layered min-sum LDPC decoder (sm_100a) + C ABI.
//
// Hot path replaced: ldpclab.decoder.decode / _run_schedule / layered_iteration
// / _scalar_layer (/root/reference/pkg/src/ldpclab/decoder.py:295-320,
// 459-469, 486-566) and ldpclab.channel.quantize (channel.py:64-83).
// See DESIGN.md for the layout and roofline; nrldpc_kernels.cuh for the exact
// half2 arithmetic argument.

#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <bitset>
#include <vector>

#include "nrldpc_kernels.cuh"
#include "../../include/nrldpc.h"

using namespace nr;

namespace {

thread_local std::string g_last_error;
thread_local int g_launches = 0;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return NRLDPC_ECUDA;
}

#define NR_CUDA(call)                                    \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------
// Device code

namespace nr {

struct GroupState {
  int synd[2];
  int minabs[2];
  int done[2];
  int accept[2];
};

struct CtaState {
  int n_done;
  int n_valid;
  uint32_t kc[6];  // Consts, staged so every thread loads them once
};

constexpr int kLutBytes = 256;
constexpr int kCtaBytes = 32;
static_assert(sizeof(CtaState) == kCtaBytes, "CtaState layout");

// k_decode_i8's shared layout: LUT, CTA state, group states, then per group
// L and messages from this 16-aligned offset
__host__ __device__ constexpr uint32_t data_offset(int groups) {
  return (kLutBytes + kCtaBytes + (uint32_t)sizeof(GroupState) * groups + 15u) & ~15u;
}

// (z + s) mod Z for one edge, as a byte offset into the group's L array.
// codeword-load steps whose global loads are issued together
constexpr int kLoadBatch = 4;

__device__ __forceinline__ uint32_t edge_offset(uint32_t shift, uint32_t colbase, uint32_t zl, uint32_t ZL) {
  uint32_t a = zl + shift;
  a = min(a, a - ZL);  // unsigned: picks a-ZL only when a >= ZL  (one VIADDMNMX)
  return a + colbase;
}

// A row's shift/column tables (tq = its first slot / 4; rows are padded to
// 4 slots): 128-bit uniform loads.
template <int MAXW>
__device__ __forceinline__ void load_row_tables(const KParams& p, uint32_t tq, int w, uint32_t (&sh)[MAXW],
                                                uint32_t (&cb)[MAXW]) {
  const uint4* S = reinterpret_cast<const uint4*>(p.sh) + tq;
  const uint4* C = reinterpret_cast<const uint4*>(p.cb) + tq;
#pragma unroll
  for (int k = 0; k < (MAXW + 3) / 4; ++k) {
    if (4 * k < w) {
      const uint4 a = S[k], b = C[k];
      const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (4 * k + i < MAXW) {
          sh[4 * k + i] = av[i];
          cb[4 * k + i] = bv[i];
        }
      }
    }
  }
}

// Message access for one edge. Shared memory: thread-major rows (Mrow =
// this thread's messages of the current base row, edge j at Mrow + j*LANES).
// Registers (REGMSG, LANES=2): two 16-bit message pairs per 32-bit register,
// edge e in half (e & 1) of mreg[e >> 1]; e is a compile-time constant after
// the schedule is unrolled, so mreg stays in registers.
template <int LANES, bool REGMSG, bool ABS = false>
__device__ __forceinline__ half2 msg_load(const uint8_t* Mrow, uint32_t Ms, const uint32_t* mreg, int j, int e,
                                          uint32_t magic) {
  if constexpr (REGMSG) {
    uint32_t d;
    if (e & 1) asm("prmt.b32 %0, %1, %2, 0x4342;" : "=r"(d) : "r"(mreg[e >> 1]), "r"(magic));
    else asm("prmt.b32 %0, %1, %2, 0x4140;" : "=r"(d) : "r"(mreg[e >> 1]), "r"(magic));
    return u2h(d);
  } else {
    const uint32_t raw = ABS ? lds_elem<LANES>(Ms + j * LANES) : ld_elem<LANES>(Mrow + j * LANES);
    return unpack_elem<LANES>(raw, magic);
  }
}

template <int LANES, bool REGMSG, bool ABS = false>
__device__ __forceinline__ void msg_store(uint8_t* Mrow, uint32_t Ms, uint32_t* mreg, int j, int e, half2 biased,
                                          bool st_ok) {
  if constexpr (REGMSG) {
    mreg[e >> 1] = __byte_perm(h2u(biased), mreg[e >> 1], (e & 1) ? 0x2054 : 0x7620);
  } else {
    if constexpr (ABS) sts_elem_if<LANES>(Ms + j * LANES, pack_elem<LANES>(biased), st_ok);
    else st_elem_if<LANES>(Mrow + j * LANES, pack_elem<LANES>(biased), st_ok);
  }
}

// Two smallest of |t_0..t_{W-1}| capped at the fold identity 127
// (kernels.py:246-257 folded from m1 = m2 = 127), as a pairwise tree: the
// same min/max work as the sequential fold but ~log2(W) deep instead of ~2W,
// so the scheduler can overlap it. Pairs give (lo, hi); two pairs merge as
// lo = min(lo_a, lo_b), hi = min(max(lo_a, lo_b), hi_a, hi_b).
template <int N>
__device__ __forceinline__ void mm_merge_level(half2 (&lo)[N], half2 (&hi)[N]) {
  if constexpr (N > 1) {
    constexpr int M = (N + 1) / 2;
    half2 nlo[M], nhi[M];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      nlo[i] = __hmin2(lo[2 * i], lo[2 * i + 1]);
      nhi[i] = __hmin2(__hmin2(__hmax2(lo[2 * i], lo[2 * i + 1]), hi[2 * i]), hi[2 * i + 1]);
    }
    if constexpr (N & 1) {
      nlo[M - 1] = lo[N - 1];
      nhi[M - 1] = hi[N - 1];
    }
    mm_merge_level<M>(nlo, nhi);
    lo[0] = nlo[0];
    hi[0] = nhi[0];
  }
}

template <int W>
__device__ __forceinline__ void two_smallest(const half2 (&t)[W], half2& m1, half2& m2) {
  const half2 H127 = u2h(0x57F057F0u);
  constexpr int P = (W + 1) / 2;
  half2 lo[P], hi[P];
#pragma unroll
  for (int i = 0; i < W / 2; ++i) {
    lo[i] = __hmin2(__habs2(t[2 * i]), __habs2(t[2 * i + 1]));
    hi[i] = __hmax2(__habs2(t[2 * i]), __habs2(t[2 * i + 1]));
  }
  if constexpr (W & 1) {
    lo[P - 1] = __habs2(t[W - 1]);
    hi[P - 1] = H127;
  }
  mm_merge_level<P>(lo, hi);
  m1 = __hmin2(lo[0], H127);
  m2 = __hmin2(hi[0], H127);
}

// One layer (base row r) for thread (group, z): gather, min-sum check-node
// update, scatter. decoder.py:295-320. t0 is the row's slot in the graph
// tables; me0 is the row's first edge in this thread's shared-memory message
// row. Split in two phases so that column-disjoint rows can be interleaved
// in one basic block (process_rows2).
// Per-kernel constants kept in registers for the whole decode. They are
// staged through shared memory and loaded once, so ptxas keeps them live
// instead of re-reading the constant bank in every layer unit.
struct Consts {
  uint32_t magic;       // 0x64646464: PRMT filler byte
  uint32_t one;         // half2 {1.0, 1.0}
  uint32_t bh, nd, cc;  // arithmetic beta rule (beta_h, -delta, C)
};

__device__ __forceinline__ uint32_t lds_u32(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(a)));
  return v;
}

// ABS: the graph table's column bases are absolute shared-window addresses
// (single-group CTAs); otherwise byte offsets from the group's L array.
template <int MAXW, int LANES, bool REGMSG, bool ABS = false>
struct RowWork {
  // ABS pair shapes store a row's messages two edges per 32-bit word (one
  // LDS.32 / STS.32 per two edges); an odd row's last edge sits in a
  // half-word slot shared with another odd row (Mh). Host: msg_layout().
  static constexpr bool PAIRED = ABS && LANES == 2 && !REGMSG;
  uint32_t off[MAXW];
  half2 t[MAXW];
  half2 m1, m2;
  uint32_t S;
  uint8_t* Mrow;
  uint32_t Ms;  // ABS: shared-window address of Mrow
  uint32_t Mh;  // PAIRED: shared-window address of the odd edge's slot
  int w;

  // phase 1: gather L and the old messages, t = L - M, fold (m1, m2, S).
  // Split in two: gather_pro touches only this thread's own state (graph
  // tables, edge addresses, its messages), so it may run before the layer
  // barrier that orders the previous layer's posterior stores; gather_main
  // reads the posteriors.
  // tb: the row's table slot / 4; mb: byte offset of its first
  // message in this thread's shared-memory message row
  uint32_t mw[(MAXW + 1) / 2];
  __device__ __forceinline__ void gather_pro(const KParams& p, const uint32_t tb, const uint32_t mb, const int w_,
                                             uint32_t zl, uint32_t ZL, uint8_t* __restrict__ Mz, uint32_t Mzs,
                                             uint32_t mh_off) {
    w = w_;
    Mrow = Mz + mb;
    Ms = Mzs + mb;
    Mh = Mzs + mh_off;
    uint32_t tsh[MAXW], tcb[MAXW];
    load_row_tables<MAXW>(p, tb, w, tsh, tcb);
    if constexpr (PAIRED) {
#pragma unroll
      for (int i = 0; i < MAXW / 2; ++i)
        if (2 * i + 1 < w) mw[i] = lds_u32(Ms + 4 * i);
      // (paired rows always run with w == MAXW: compile-time row bodies)
      if (MAXW & 1) mw[MAXW / 2] = lds_elem<2>(Mh);
    }
#pragma unroll
    for (int j = 0; j < MAXW; ++j)
      if (j < w) off[j] = edge_offset(tsh[j], tcb[j], zl, ZL);
  }
  __device__ __forceinline__ void gather_main(const uint8_t* __restrict__ Lg, const uint32_t* mreg,
                                              uint32_t magic) {
    const half2 H127 = u2h(0x57F057F0u);
    m1 = H127;
    m2 = H127;
    S = 0;
#pragma unroll
    for (int j = 0; j < MAXW; ++j) {
      if (j < w) {
        const uint32_t raw = ABS ? lds_elem<LANES>(off[j]) : ld_elem<LANES>(Lg + off[j]);
        const half2 lh = unpack_elem<LANES>(raw, magic);
        half2 mh;
        if constexpr (PAIRED) {
          uint32_t d;
          if (j & 1) asm("prmt.b32 %0, %1, %2, 0x4342;" : "=r"(d) : "r"(mw[j >> 1]), "r"(magic));
          else asm("prmt.b32 %0, %1, %2, 0x4140;" : "=r"(d) : "r"(mw[j >> 1]), "r"(magic));
          mh = u2h(d);
        } else {
          mh = msg_load<LANES, REGMSG, ABS>(Mrow, Ms, mreg, j, j, magic);
        }
        const half2 tj = __hsub2(lh, mh);           // exact: L - M
        S ^= h2u(tj);                               // sign product (bits 15/31)
        t[j] = tj;
      }
    }
    if (w == MAXW) {
      two_smallest<MAXW>(t, m1, m2);                // kernels.py:247-250, as a tree
    } else {
#pragma unroll
      for (int j = 0; j < MAXW; ++j) {
        if (j < w) {
          const half2 aj = __habs2(t[j]);
          m2 = __hmin2(m2, __hmax2(m1, aj));        // kernels.py:247-250
          m1 = __hmin2(m1, aj);
        }
      }
    }
  }
  __device__ __forceinline__ void gather(const KParams& p, const uint32_t tb, const uint32_t mb, const int w_,
                                         uint32_t zl, uint32_t ZL, const uint8_t* __restrict__ Lg,
                                         uint8_t* __restrict__ Mz, uint32_t Mzs, const uint32_t* mreg,
                                         uint32_t magic, uint32_t mh_off = 0, bool bar = false) {
    gather_pro(p, tb, mb, w_, zl, ZL, Mz, Mzs, mh_off);
    if (bar) __syncthreads();
    gather_main(Lg, mreg, magic);
  }

  // beta-scaled magnitudes with the row sign folded in: b' = (-1)^S * b.
  // Split from the scatter so that fused rows share one branch on beta_mode
  // and their scatters stay in one basic block.
  half2 dd, b2s;  // (b1 - b2)' and b2'
  __device__ __forceinline__ void beta_arith(const Consts& k) {
    // floor(beta*m) == RN(beta_h*(m - delta) + C) - C for every m in [0,127]
    // (verified exhaustively on the host); all FMA-pipe, no table lookups
    const half2 sig = u2h((S & 0x80008000u) | k.one);
    const half2 bh = u2h(k.bh), nd = u2h(k.nd), cc = u2h(k.cc);
    const half2 B1 = __hfma2(__hadd2(m1, nd), bh, cc);
    const half2 B2 = __hfma2(__hadd2(m2, nd), bh, cc);
    dd = __hmul2(__hsub2(B1, B2), sig);
    b2s = __hmul2(__hsub2(B2, cc), sig);
  }
  __device__ __forceinline__ void beta_lut(const uint16_t* __restrict__ lut, uint32_t one) {
    const half2 sig = u2h((S & 0x80008000u) | one);
    const half2 b1 = beta_lut2(lut, m1);
    const half2 b2 = beta_lut2(lut, m2);
    dd = __hmul2(__hsub2(b1, b2), sig);
    b2s = __hmul2(b2, sig);
  }

  // phase 2: new messages and posteriors, scatter
  __device__ __forceinline__ void scatter(uint8_t* __restrict__ Lg, uint32_t* mreg, uint32_t one,
                                          bool st_ok) {
    const half2 H127 = u2h(0x57F057F0u);   // 127.0
    const half2 H1152 = u2h(0x64806480u);  // 1152.0
#pragma unroll
    for (int j = 0; j < MAXW; ++j) {
      if (j < w) {
        // x = 0 for the edge holding the minimum (it gets m2; a tie implies
        // m1 == m2), else 1: |t| - m1 is a non-negative integer, saturated.
        const half2 x = __hsub2_sat(__habs2(t[j]), m1);
        const half2 mag = __hfma2(x, dd, b2s);       // +-b1 or +-b2
        // L' = clamp127(clamp127(t) + out) with clamp127(t) = sign(t)*a,
        // a = min(|t|,127), out = sign(t)*mag':  L' = sign(t)*min(a + mag', 127)
        // (a + mag' >= -127, so the lower clamp never binds). The two mins are
        // full-rate ALU ops; the FP16 pipe is the busier one in this phase.
        const half2 a = __hmin2(__habs2(t[j]), H127);
        const half2 y = __hmin2(__hadd2(a, mag), H127);
        const half2 sg = u2h((h2u(t[j]) & 0x80008000u) | one);
        const uint32_t lnew = pack_elem<LANES>(__hfma2(y, sg, H1152));
        if constexpr (ABS) sts_elem_if<LANES>(off[j], lnew, st_ok);
        else st_elem_if<LANES>(Lg + off[j], lnew, st_ok);
        const half2 mb = __hfma2(mag, sg, H1152);
        if constexpr (PAIRED) {
          // two edges' biased messages -> one word: low bytes of each half
          if (j & 1) sts_u32_if(Ms + 4 * (j >> 1), __byte_perm(h2u(mprev), h2u(mb), 0x6420), st_ok);
          else if (j == w - 1) sts_elem_if<2>(Mh, pack_elem<2>(mb), st_ok);
          mprev = mb;
        } else {
          msg_store<LANES, REGMSG, ABS>(Mrow, Ms, mreg, j, j, mb, st_ok);
        }
      }
    }
  }
  half2 mprev;
};

// LUT: the beta rule may be the table (generic schedule); the compile-time
// BG1/BG2 schedules are only used with the arithmetic rule (smaller bodies).
template <int MAXW, int LANES, bool REGMSG, bool ABS = false, bool LUT = true>
__device__ __forceinline__ void process_row(const KParams& p, const uint32_t tb, const uint32_t mb, const int w,
                                            uint32_t zl, uint32_t ZL, uint8_t* __restrict__ Lg,
                                            uint8_t* __restrict__ Mz, uint32_t Mzs, uint32_t* mreg,
                                            const uint16_t* __restrict__ lut, const Consts& k, bool st_ok,
                                            uint32_t mh = 0, bool bar = false) {
  RowWork<MAXW, LANES, REGMSG, ABS> r;
  r.gather(p, tb, mb, w, zl, ZL, Lg, Mz, Mzs, mreg, k.magic, mh, bar);
  if (!LUT || p.beta_mode) r.beta_arith(k);
  else r.beta_lut(lut, k.one);
  r.scatter(Lg, mreg, k.one, st_ok);
}

// Two consecutive column-disjoint rows as one basic block: no barrier between
// them is needed and the scheduler interleaves their independent chains.
template <int WA, int WB, int LANES, bool ABS = false, bool LUT = true>
__device__ __forceinline__ void process_rows2(const KParams& p, uint32_t tba, uint32_t mba, uint32_t tbb,
                                              uint32_t mbb,
                                              uint32_t zl, uint32_t ZL, uint8_t* __restrict__ Lg,
                                              uint8_t* __restrict__ Mz, uint32_t Mzs, uint32_t* mreg,
                                              const uint16_t* __restrict__ lut, const Consts& k, bool st_ok,
                                              uint32_t mha = 0, uint32_t mhb = 0, bool bar = false) {
  RowWork<WA, LANES, false, ABS> a;
  RowWork<WB, LANES, false, ABS> b;
  a.gather_pro(p, tba, mba, WA, zl, ZL, Mz, Mzs, mha);
  b.gather_pro(p, tbb, mbb, WB, zl, ZL, Mz, Mzs, mhb);
  if (bar) __syncthreads();
  a.gather_main(Lg, mreg, k.magic);
  b.gather_main(Lg, mreg, k.magic);
  if (!LUT || p.beta_mode) {
    a.beta_arith(k);
    b.beta_arith(k);
  } else {
    a.beta_lut(lut, k.one);
    b.beta_lut(lut, k.one);
  }
  a.scatter(Lg, mreg, k.one, st_ok);
  b.scatter(Lg, mreg, k.one, st_ok);
}

// ---- TM layout (single-group pair shapes that hold an SM alone) -----------
// L holds the biased half2 itself, 4 bytes per position ({1152+v_a,
// 1152+v_b}; the low byte of each half is the biased byte u = v + 128), so
// the gather needs no unpack and the scatter no pack. That doubles L
// (104 KB at BG1 Z=384), so the messages leave shared memory: rows with
// w >= SMW keep one biased half2 per edge in shared memory (thread-major, odd
// word stride), the other rows in tensor memory (tcgen05.ld/st, 32x32b: the
// thread's own TMEM lane; the warps sharing a lane quarter each own a slot
// of p.tm_slot columns). BG1 register-row shapes keep rows 0..5 in byte-pair
// registers. The message kind follows from the compile-time row weight
// (host: tm_shape); SMW per schedule: tm_smw.
template <int BG, int NREG>
__host__ __device__ constexpr int tm_smw() {
  return BG == 2 ? 8 : NREG == 6 ? 7 : 11;
}

// Rows whose last edge is their degree-1 extension column, with shift 0 in
// every lifting (TS 38.212 base graphs: BG1 rows >= 4, BG2 rows >= 4; the
// host checks the tables, tm_shape). Told apart by weight: the core rows are
// the only ones of weight 19 (BG1) or 8 and 10 (BG2). Thread z's position in
// that column is z itself, so its address needs no modular arithmetic.
template <int BG>
__host__ __device__ constexpr bool tm_diag(int w) {
  return BG == 1 ? w != 19 : w <= 6;
}

template <int MAXW, bool REGMSG, int SMW = 7, bool DIAG = false>
struct RowWorkTM {
  static constexpr bool TMEM = !REGMSG && MAXW < SMW;
  // shared kind, BG1 register-row shapes (SMW 7): 8-byte aligned rows padded
  // to an even word count (host: tm_shape), two messages per LDS.64/STS.64
  // (measured +0.7% there, -0.7% for BG2, so only there)
  static constexpr bool V2 = !REGMSG && !TMEM && SMW == 7;
  uint32_t off[MAXW];
  half2 t[MAXW];
  uint32_t mw[MAXW];  // the row's messages (shared / tensor memory kinds)
  half2 m1, m2;
  uint32_t S;
  uint32_t Ma;  // shared address (w >= SMW) or tensor-memory address (w < SMW) of the row's messages

  // thread-private part (tables, addresses, own messages): may run before the
  // barrier that closes the previous layer
  __device__ __forceinline__ void gather_pro(const KParams& p, uint32_t tb, uint32_t mb, uint32_t zl, uint32_t ZL,
                                             uint32_t Mzs, uint32_t tbase) {
    uint32_t tsh[MAXW], tcb[MAXW];
    load_row_tables<MAXW>(p, tb, MAXW, tsh, tcb);
    if constexpr (TMEM) {
      Ma = tbase + mb;
      tm_ld_row<MAXW>(Ma, mw);
    } else if constexpr (!REGMSG) {
      Ma = Mzs + mb;
      if constexpr (V2) {
#pragma unroll
        for (int j = 0; j + 1 < MAXW; j += 2) lds_v2(Ma + 4 * j, mw[j], mw[j + 1]);
        if constexpr ((MAXW & 1) != 0) mw[MAXW - 1] = lds_u32(Ma + 4 * (MAXW - 1));
      } else {
#pragma unroll
        for (int j = 0; j < MAXW; ++j) mw[j] = lds_u32(Ma + 4 * j);
      }
    }
#pragma unroll
    for (int j = 0; j < MAXW; ++j)
      off[j] = DIAG && j == MAXW - 1 ? zl + tcb[j] : edge_offset(tsh[j], tcb[j], zl, ZL);
  }
  __device__ __forceinline__ void gather_main(const uint32_t* mreg, uint32_t magic) {
    if constexpr (TMEM) tm_wait_ld<MAXW>(mw);
    S = 0;
#pragma unroll
    for (int j = 0; j < MAXW; ++j) {
      const half2 lh = u2h(lds_u32(off[j]));
      const half2 mh = REGMSG ? msg_load<2, true>(nullptr, 0, mreg, j, j, magic) : u2h(mw[j]);
      const half2 tj = __hsub2(lh, mh);  // exact: L - M
      S ^= h2u(tj);
      t[j] = tj;
    }
    two_smallest<MAXW>(t, m1, m2);  // kernels.py:247-250
  }
  half2 dd, b2s;
  __device__ __forceinline__ void beta_arith(const Consts& k) {
    const half2 sig = u2h((S & 0x80008000u) | k.one);
    const half2 bh = u2h(k.bh), nd = u2h(k.nd), cc = u2h(k.cc);
    const half2 B1 = __hfma2(__hadd2(m1, nd), bh, cc);
    const half2 B2 = __hfma2(__hadd2(m2, nd), bh, cc);
    dd = __hmul2(__hsub2(B1, B2), sig);
    b2s = __hmul2(__hsub2(B2, cc), sig);
  }
  __device__ __forceinline__ void scatter(uint32_t* mreg, uint32_t one) {
    const half2 H127 = u2h(0x57F057F0u);   // 127.0
    const half2 H1152 = u2h(0x64806480u);  // 1152.0
#pragma unroll
    for (int j = 0; j < MAXW; ++j) {
      const half2 x = __hsub2_sat(__habs2(t[j]), m1);
      const half2 mag = __hfma2(x, dd, b2s);
      const half2 a = __hmin2(__habs2(t[j]), H127);
      const half2 y = __hmin2(__hadd2(a, mag), H127);
      const half2 sg = u2h((h2u(t[j]) & 0x80008000u) | one);
      sts_u32(off[j], h2u(__hfma2(y, sg, H1152)));
      const half2 mb = __hfma2(mag, sg, H1152);
      if constexpr (REGMSG) msg_store<2, true>(nullptr, 0, mreg, j, j, mb, true);
      else if constexpr (TMEM || V2) mw[j] = h2u(mb);
      else sts_u32(Ma + 4 * j, h2u(mb));
    }
    if constexpr (TMEM) {
      tm_st_row<MAXW>(Ma, mw);
    } else if constexpr (V2) {
#pragma unroll
      for (int j = 0; j + 1 < MAXW; j += 2) sts_v2(Ma + 4 * j, mw[j], mw[j + 1]);
      if constexpr ((MAXW & 1) != 0) sts_u32(Ma + 4 * (MAXW - 1), mw[MAXW - 1]);
    }
  }
};

struct TmCtx {
  uint32_t zl, ZL;
  uint32_t Ms;     // shared-window address of this thread's message row
  uint32_t tbase;  // tensor-memory address of this thread's column slot
  Consts k;
};

template <int W, bool REGMSG, int SMW, bool DIAG>
__device__ __forceinline__ void process_row_tm(const KParams& p, uint32_t tb, uint32_t mb, const TmCtx& c,
                                               uint32_t* mreg, bool bar) {
  RowWorkTM<W, REGMSG, SMW, DIAG> r;
  r.gather_pro(p, tb, mb, c.zl, c.ZL, c.Ms, c.tbase);
  if (bar) __syncthreads();
  r.gather_main(mreg, c.k.magic);
  r.beta_arith(c.k);
  r.scatter(mreg, c.k.one);
}

template <int WA, int WB, int SMW, bool DIAG>
__device__ __forceinline__ void process_rows2_tm(const KParams& p, uint32_t tba, uint32_t mba, uint32_t tbb,
                                                 uint32_t mbb, const TmCtx& c, bool bar) {
  RowWorkTM<WA, false, SMW, DIAG> a;
  RowWorkTM<WB, false, SMW, DIAG> b;
  a.gather_pro(p, tba, mba, c.zl, c.ZL, c.Ms, c.tbase);
  b.gather_pro(p, tbb, mbb, c.zl, c.ZL, c.Ms, c.tbase);
  if (bar) __syncthreads();
  a.gather_main(nullptr, c.k.magic);
  b.gather_main(nullptr, c.k.magic);
  a.beta_arith(c.k);
  b.beta_arith(c.k);
  a.scatter(nullptr, c.k.one);
  b.scatter(nullptr, c.k.one);
}

template <int MAXW, bool DIAG>
__device__ __forceinline__ void row_parity_tm(const KParams& p, const uint32_t tb, uint32_t zl, uint32_t ZL,
                                              int& wa, int& wb) {
  uint32_t tsh[MAXW], tcb[MAXW];
  load_row_tables<MAXW>(p, tb, MAXW, tsh, tcb);
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < MAXW; ++j)
    x ^= lds_u32(DIAG && j == MAXW - 1 ? zl + tcb[j] : edge_offset(tsh[j], tcb[j], zl, ZL));
  // bit 7 of each half's low byte is 1 for a non-negative value
  if (MAXW & 1) x ^= 0x00800080u;
  wa += (x >> 7) & 1u;
  wb += (x >> 23) & 1u;
}

// Syndrome weight (decoder.py:323-329) and min|L| (decoder.py:480-483) over
// the thread's check rows / columns.
template <int MAXW, int LANES, bool ABS = false>
__device__ __forceinline__ void row_parity(const KParams& p, const uint32_t tb, const int w, uint32_t zl,
                                           uint32_t ZL, const uint8_t* __restrict__ Lg, int& wa,
                                           int& wb) {
  uint32_t tsh[MAXW], tcb[MAXW];
  load_row_tables<MAXW>(p, tb, w, tsh, tcb);
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < MAXW; ++j) {
    if (j < w) {
      const uint32_t a = edge_offset(tsh[j], tcb[j], zl, ZL);
      x ^= ABS ? lds_elem<LANES>(a) : ld_elem<LANES>(Lg + a);
    }
  }
  // bit 7 of a stored byte is 1 for a non-negative value
  if (w & 1) x ^= 0x8080u;
  wa += (x >> 7) & 1u;
  wb += (x >> 15) & 1u;
}

// Layer schedules. Generic: row tables read at run time. BG1/BG2: the row
// weights are compile-time (they are fixed by the base graph), so every
// edge's shift/column becomes a constant-bank operand and the 46 (42)
// layers are straight-line code with one uniform early-out on rows_used.
template <int BG>
struct RowW;
template <>
struct RowW<1> {
  static constexpr int n = 46;
  static constexpr int w[46] = {19, 19, 19, 19, 3, 8, 9, 7, 10, 9, 7, 8, 7, 6, 7, 7, 6, 6, 6, 6, 6, 6, 5,
                                5,  6,  5,  5,  4, 5, 5, 5, 5,  5, 5, 5, 5, 5, 4, 5, 5, 4, 5, 4, 5, 5, 4};
  static constexpr int e0[47] = {0, 19, 38, 57, 76, 79, 87, 96, 103, 113, 122, 129, 137, 144, 150, 157, 164, 170, 176, 182, 188, 194, 200, 205, 210, 216, 221, 226, 230, 235, 240, 245, 250, 255, 260, 265, 270, 275, 279, 284, 289, 293, 298, 302, 307, 312, 316};
};
template <>
struct RowW<2> {
  static constexpr int n = 42;
  static constexpr int w[42] = {8, 10, 8, 10, 4, 6, 6, 6, 4, 5, 5, 5, 4, 5, 5, 4, 5, 5, 4, 4, 4,
                                4, 3,  4, 4,  3, 5, 3, 4, 3, 5, 3, 4, 4, 4, 4, 4, 3, 4, 4, 4, 4};
  static constexpr int e0[43] = {0, 8, 18, 26, 36, 40, 46, 52, 58, 62, 67, 72, 77, 81, 86, 91, 95, 100, 105, 109, 113, 117, 121, 124, 128, 132, 135, 140, 143, 147, 150, 155, 158, 162, 166, 170, 174, 178, 181, 185, 189, 193, 197};
};

struct RowCtx {
  uint32_t zl, ZL;
  uint8_t* Lg;
  uint8_t* Mz;
  uint32_t Ms;  // shared-window address of Mz
  const uint16_t* lut;
  Consts k;
  bool st_ok;
};

template <int N>
struct IC {
  static constexpr int value = N;
};

// Calls f(IC<W>{}) for the row weights that occur in the base graph, so each
// layer body is compiled once per weight (not once per row): the whole
// iteration stays within the instruction cache.
// w == k through inline PTX, so LLVM cannot fold the chain below back into a
// switch (jump table)
__device__ __forceinline__ bool weq(int w, int k) {
  int r;
  asm("{ .reg .pred q; setp.eq.s32 q, %1, %2; selp.s32 %0, 1, 0, q; }" : "=r"(r) : "r"(w), "r"(k));
  return r != 0;
}

template <int BG, typename F>
__device__ __forceinline__ void dispatch_w(int w, F&& f) {
  // an if-chain on a uniform value compiles to uniform branches (BRA.U);
  // a switch becomes BRX on a vector register, which makes ptxas demote the
  // row index and every graph-table load to per-thread registers
  if constexpr (BG == 1) {
    if (weq(w, 5)) f(IC<5>{});
    else if (weq(w, 6)) f(IC<6>{});
    else if (weq(w, 4)) f(IC<4>{});
    else if (weq(w, 7)) f(IC<7>{});
    else if (weq(w, 19)) f(IC<19>{});
    else if (weq(w, 9)) f(IC<9>{});
    else if (weq(w, 8)) f(IC<8>{});
    else if (weq(w, 10)) f(IC<10>{});
    else if (weq(w, 3)) f(IC<3>{});
  } else {
    if (weq(w, 4)) f(IC<4>{});
    else if (weq(w, 5)) f(IC<5>{});
    else if (weq(w, 3)) f(IC<3>{});
    else if (weq(w, 6)) f(IC<6>{});
    else if (weq(w, 8)) f(IC<8>{});
    else if (weq(w, 10)) f(IC<10>{});
  }
}

// Layer units of the compile-time schedules: code = wa | wb << 8 (wb = 0: a
// single row). Fused pairs are the column-disjoint consecutive rows that
// occur in the base graphs (BG1 rows 16..45, BG2 rows 11..41); the host
// (build_units) fuses exactly these. The chain is ordered by how often each
// unit occurs per iteration of the full graph.
// NREG: rows 0..NREG-1 run from registers, so their weights (19 for the four
// core rows, 3 for row 4) never reach the unit loop and get no body.
__device__ __forceinline__ bool wge(int w, int k) {
  int r;
  asm("{ .reg .pred q; setp.ge.s32 q, %1, %2; selp.s32 %0, 1, 0, q; }" : "=r"(r) : "r"(w), "r"(k));
  return r != 0;
}

template <int BG, int NREG, typename F>
__device__ __forceinline__ void dispatch_unit(uint32_t code, F&& f) {
  const int c = (int)code;
  // pairs (code >= 256) and single rows get separate chains
#define NR_U(a, b) else if (weq(c, (a) | ((b) << 8))) f(IC<a>{}, IC<b>{})
  if constexpr (BG == 1) {
    if (wge(c, 256)) {
      if (false) {}
      NR_U(5, 5); NR_U(5, 4); NR_U(6, 6); NR_U(6, 5);
    } else {
      if (false) {}
      NR_U(7, 0); NR_U(6, 0); NR_U(9, 0); NR_U(10, 0); NR_U(8, 0); NR_U(5, 0); NR_U(4, 0);
      else if constexpr (NREG < 6) {
        if (weq(c, 3)) f(IC<3>{}, IC<0>{});
        else if constexpr (NREG < 4) {
          if (weq(c, 19)) f(IC<19>{}, IC<0>{});
        }
      }
    }
  } else {
    if (wge(c, 256)) {
      if (false) {}
      NR_U(4, 4); NR_U(4, 3); NR_U(5, 4); NR_U(5, 3);
    } else {
      if (false) {}
      NR_U(4, 0); NR_U(5, 0); NR_U(6, 0); NR_U(8, 0); NR_U(10, 0); NR_U(3, 0);
    }
  }
#undef NR_U
}

// Register-resident messages (BG1 pairs at the largest Z, see choose_shape):
// the four 19-edge core rows keep their messages in a rotating queue of
// 4 x 10 registers (the head is always the row being processed, so one loop
// body serves all four rows); rows 4 and 5 (weights 3 and 8) use their own
// registers when NREG == 6.
template <int NREG>
struct RegMsg {
  static constexpr int nq = NREG >= 4 ? 4 : NREG;
  uint32_t q[nq > 0 ? nq : 1][10];
  uint32_t r4[2];
  uint32_t r5[4];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int k = 0; k < (nq > 0 ? nq : 1); ++k)
#pragma unroll
      for (int i = 0; i < 10; ++i) q[k][i] = 0x80808080u;  // zero messages (biased)
#pragma unroll
    for (int i = 0; i < 2; ++i) r4[i] = 0x80808080u;
#pragma unroll
    for (int i = 0; i < 4; ++i) r5[i] = 0x80808080u;
  }
  // zero (biased 0x80) one lane's bytes of every register message
  __device__ __forceinline__ void reset_lane(uint32_t keep) {
    const uint32_t z = 0x80808080u & ~keep;
#pragma unroll
    for (int k = 0; k < (nq > 0 ? nq : 1); ++k)
#pragma unroll
      for (int i = 0; i < 10; ++i) q[k][i] = (q[k][i] & keep) | z;
#pragma unroll
    for (int i = 0; i < 2; ++i) r4[i] = (r4[i] & keep) | z;
#pragma unroll
    for (int i = 0; i < 4; ++i) r5[i] = (r5[i] & keep) | z;
  }
  // rows come in twos: after rows (2k, 2k+1) swap the head pair with the
  // tail pair (nq == 4); nq == 2 needs no movement at all
  __device__ __forceinline__ void rotate2() {
    if constexpr (nq == 4) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < 10; ++i) {
          const uint32_t h = q[k][i];
          q[k][i] = q[k + 2][i];
          q[k + 2][i] = h;
        }
    }
  }
};

template <int BG, int MAXW, int LANES, int NREG, bool ABS>
__device__ __forceinline__ void one_iteration(const KParams& p, const RowCtx& c, RegMsg<NREG>& rm) {
  if constexpr (BG == 0) {
    for (int r = 0; r < p.rows; ++r) {
      const int e0 = p.row_start[r];
      process_row<MAXW, LANES, false>(p, p.tab_start[r] / 4u, (uint32_t)e0 * LANES, p.row_start[r + 1] - e0, c.zl, c.ZL, c.Lg, c.Mz, c.Ms,
                                      rm.r4, c.lut, c.k, c.st_ok);
      if (p.bar_after[r]) __syncthreads();
    }
  } else {
    bool bar_prev = false;  // a layer barrier is owed before the next posterior load
    if constexpr (NREG > 0) {
      // each row runs its table/address prologue before the barrier that
      // closes the previous row (the iteration starts after a barrier)
#pragma unroll 1
      for (int r = 0; r < RegMsg<NREG>::nq; r += 2) {
        process_row<19, LANES, true, ABS, false>(p, 5u * r, 0, 19, c.zl, c.ZL, c.Lg, c.Mz, c.Ms, rm.q[0], c.lut, c.k,
                                                 c.st_ok, 0, r != 0);
        process_row<19, LANES, true, ABS, false>(p, 5u * r + 5u, 0, 19, c.zl, c.ZL, c.Lg, c.Mz, c.Ms, rm.q[1], c.lut,
                                                 c.k, c.st_ok, 0, true);
        rm.rotate2();
      }
      if constexpr (NREG == 6) {
        process_row<3, LANES, true, ABS, false>(p, 20u, 0, 3, c.zl, c.ZL, c.Lg, c.Mz, c.Ms, rm.r4, c.lut, c.k,
                                                c.st_ok, 0, true);
        process_row<8, LANES, true, ABS, false>(p, 21u, 0, 8, c.zl, c.ZL, c.Lg, c.Mz, c.Ms, rm.r5, c.lut, c.k,
                                                c.st_ok, 0, true);
      }
      bar_prev = true;
    }
    // The remaining rows run as host-built units (a single row, or two
    // consecutive column-disjoint rows fused into one basic block) with
    // precomputed offsets; each unit's dispatch code is loaded one unit
    // ahead so the dispatch does not wait on the constant cache.
    uint32_t ncode = p.unit_a[0].x;
    // The barrier that closes a layer runs inside the next unit, after its
    // thread-private prologue (tables, addresses, own messages) and before
    // its first posterior load, so warps arriving early do useful work.
#pragma unroll 1
    for (int u = 0; u < p.n_units; ++u) {
      // only the dispatch code is prefetched (one loop-carried copy); the
      // offsets are needed inside the body, where their load overlaps the
      // dispatch
      const uint32_t code = ncode;
      const uint4 A = p.unit_a[u];
      const uint4 B = p.unit_b[u];
      ncode = p.unit_a[u + 1].x;
      dispatch_unit<BG, NREG>(code, [&](auto WA, auto WB) {
        constexpr int wa = decltype(WA)::value, wb = decltype(WB)::value;
        if constexpr (wb == 0)
          process_row<wa, LANES, false, ABS, false>(p, A.z, A.w, wa, c.zl, c.ZL, c.Lg, c.Mz, c.Ms, rm.r4, c.lut, c.k,
                                                    c.st_ok, B.z, bar_prev);
        else
          process_rows2<wa, wb, LANES, ABS, false>(p, A.z, A.w, B.x, B.y, c.zl, c.ZL, c.Lg, c.Mz, c.Ms, rm.r4, c.lut,
                                                   c.k, c.st_ok, B.z, B.w, bar_prev);
      });
      // consecutive column-disjoint rows form one layer: the next unit reads
      // no column this one wrote, so warps may run ahead into it
      bar_prev = A.y != 0;
    }
    if (bar_prev) __syncthreads();
  }
}

// one_iteration for the TM layout: same schedule, units and barrier placement
template <int BG, int NREG>
__device__ __forceinline__ void one_iteration_tm(const KParams& p, const TmCtx& c, RegMsg<NREG>& rm) {
  constexpr int SMW = tm_smw<BG, NREG>();
  bool bar_prev = false;
  if constexpr (NREG == 6) {
#pragma unroll 1
    for (int r = 0; r < 4; r += 2) {
      process_row_tm<19, true, SMW, false>(p, 5u * r, 0, c, rm.q[0], r != 0);
      process_row_tm<19, true, SMW, false>(p, 5u * r + 5u, 0, c, rm.q[1], true);
      rm.rotate2();
    }
    // rows 4 and 5 keep their messages in tensor memory (SMW 9: both weights
    // below it), so their byte-pair registers and PRMTs go away
    process_row_tm<3, false, 9, tm_diag<BG>(3)>(p, 20u, p.tm_r45[0], c, nullptr, true);
    process_row_tm<8, false, 9, tm_diag<BG>(8)>(p, 21u, p.tm_r45[1], c, nullptr, true);
    bar_prev = true;
  }
  uint32_t ncode = p.unit_a[0].x;
#pragma unroll 1
  for (int u = 0; u < p.n_units; ++u) {
    const uint32_t code = ncode;
    const uint4 A = p.unit_a[u];
    const uint4 B = p.unit_b[u];
    ncode = p.unit_a[u + 1].x;
    dispatch_unit<BG, NREG>(code, [&](auto WA, auto WB) {
      constexpr int wa = decltype(WA)::value, wb = decltype(WB)::value;
      if constexpr (wb == 0) process_row_tm<wa, false, SMW, tm_diag<BG>(wa)>(p, A.z, A.w, c, nullptr, bar_prev);
      else process_rows2_tm<wa, wb, SMW, tm_diag<BG>(wa) && tm_diag<BG>(wb)>(p, A.z, A.w, B.x, B.y, c, bar_prev);
    });
    bar_prev = A.y != 0;
  }
  if (bar_prev) __syncthreads();
  // the next iteration reads these messages back
  tm_wait_st();
}

// min |L| over this thread's positions of both lanes (decoder.py:480-483)
// (four independent min chains, so the loads overlap; the posteriors are
// the biased half2 {1152+v_a, 1152+v_b}, so |v| is one HADD2 plus the |.|
// operand of HMNMX2 for both lanes)
__device__ __forceinline__ void margin_tm(const KParams& p, uint32_t zl, uint32_t ZL, uint32_t Ls, int* mabs) {
  const half2 H255 = u2h(0x5BF85BF8u), H1152 = u2h(0x64806480u);
  half2 acc[4] = {H255, H255, H255, H255};
  int c = 0;
  for (; c + 4 <= p.n_blocks; c += 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      acc[i] = __hmin2(acc[i], __habs2(__hsub2(u2h(lds_u32(Ls + (uint32_t)(c + i) * ZL + zl)), H1152)));
  }
  for (; c < p.n_blocks; ++c)
    acc[0] = __hmin2(acc[0], __habs2(__hsub2(u2h(lds_u32(Ls + (uint32_t)c * ZL + zl)), H1152)));
  const half2 m = __hmin2(__hmin2(acc[0], acc[1]), __hmin2(acc[2], acc[3]));
  mabs[0] = (int)__low2float(m);   // exact small integers
  mabs[1] = (int)__high2float(m);
}

// Table slot quad of row R in the compile-time schedules (rows padded to 4
// slots; host: nrldpc_plan_create's table builder).
template <int BG, int R>
__host__ __device__ constexpr uint32_t row_tq() {
  uint32_t t = 0;
  for (int r = 0; r < R; ++r) t += (uint32_t)(RowW<BG>::w[r] + 3) / 4u;
  return t;
}

// Full syndrome of a full compile-time graph (rows R..E-1) as one
// straight-line block (no per-row dispatch), so the loads of many rows are in
// flight together.
template <int BG, int R = 0, int E = RowW<BG>::n>
__device__ __forceinline__ void parity_rows_tm(const KParams& p, uint32_t zl, uint32_t ZL, int& wa, int& wb) {
  if constexpr (R < E) {
    constexpr int w = RowW<BG>::w[R];
    row_parity_tm<w, tm_diag<BG>(w)>(p, row_tq<BG, R>(), zl, ZL, wa, wb);
    parity_rows_tm<BG, R + 1, E>(p, zl, ZL, wa, wb);
  }
}

// The same for a partial graph (rows < p.rows): straight-line rows with a
// uniform bound test before each.
template <int BG, int R = 0>
__device__ __forceinline__ void parity_rows_part_tm(const KParams& p, uint32_t zl, uint32_t ZL, int& wa, int& wb) {
  if constexpr (R < RowW<BG>::n) {
    if (R >= p.rows) return;
    constexpr int w = RowW<BG>::w[R];
    row_parity_tm<w, tm_diag<BG>(w)>(p, row_tq<BG, R>(), zl, ZL, wa, wb);
    parity_rows_part_tm<BG, R + 1>(p, zl, ZL, wa, wb);
  }
}

// Early-mode scan of a full compile-time graph (see local_check_tm): blocks
// of STEP straight-line rows, then publish this warp's failures and stop
// once every live lane has one. Returns when done or stopped.
template <int BG, int R, int STEP>
__device__ __forceinline__ void parity_rows_early_tm(const KParams& p, uint32_t zl, uint32_t ZL, int& wa, int& wb,
                                                     bool need_a, bool need_b, bool& pub_a, bool& pub_b,
                                                     int* synd) {
  if constexpr (R < RowW<BG>::n) {
    constexpr int E = R + STEP < RowW<BG>::n ? R + STEP : RowW<BG>::n;
    parity_rows_tm<BG, R, E>(p, zl, ZL, wa, wb);
    const bool leader = (threadIdx.x & 31) == 0;
    if (!pub_a && __any_sync(0xFFFFFFFFu, wa != 0)) {
      if (leader) atomicAdd(&synd[0], 1);
      pub_a = true;
    }
    if (!pub_b && __any_sync(0xFFFFFFFFu, wb != 0)) {
      if (leader) atomicAdd(&synd[1], 1);
      pub_b = true;
    }
    const volatile int* vs = synd;
    if ((!need_a || vs[0] != 0) && (!need_b || vs[1] != 0)) return;
    parity_rows_early_tm<BG, E, STEP>(p, zl, ZL, wa, wb, need_a, need_b, pub_a, pub_b, synd);
  }
}

// local_check for the TM layout (Z % 32 == 0, one group). Early mode (an
// early-stop iteration that is neither traced nor final) needs only "does
// any check fail" per lane, so the warps cooperate: a warp that holds a
// failing check of a live lane publishes it at once in the group's syndrome
// counter (synd), and every warp stops scanning rows as soon as the counters
// show a failure for every live lane. wcnt then returns 0 (already counted),
// and the margin (min |L|) is left out (mabs = 255): it only matters for a
// lane whose syndrome is zero, and the caller computes it in a second pass
// only then.
template <int BG>
__device__ __forceinline__ void local_check_tm(const KParams& p, uint32_t zl, uint32_t ZL, uint32_t Ls, int* wcnt,
                                               int* mabs, bool early, bool need_a, bool need_b, int* synd) {
  int wa = 0, wb = 0;
  bool pub_a = !need_a, pub_b = !need_b;  // nothing to publish for a lane not being decoded
  const bool leader = (threadIdx.x & 31) == 0;
  if (p.rows == RowW<BG>::n) {
    mabs[0] = mabs[1] = 255;
    if (early) {
      parity_rows_early_tm<BG, 0, 4>(p, zl, ZL, wa, wb, need_a, need_b, pub_a, pub_b, synd);
      wcnt[0] = wcnt[1] = 0;
    } else {
      parity_rows_tm<BG>(p, zl, ZL, wa, wb);
      margin_tm(p, zl, ZL, Ls, mabs);
      wcnt[0] = wa;
      wcnt[1] = wb;
    }
    return;
  }
  if (!early) {
    parity_rows_part_tm<BG>(p, zl, ZL, wa, wb);
    margin_tm(p, zl, ZL, Ls, mabs);
    wcnt[0] = wa;
    wcnt[1] = wb;
    return;
  }
  // early mode, partial graph: row loop with the cooperative exit test
#pragma unroll 1
  for (int r = 0; r < p.rows; ++r) {
    const int e0 = p.row_start[r];
    const int t0 = p.tab_start[r];
    const int w = p.row_start[r + 1] - e0;
    dispatch_w<BG>(w, [&](auto W) {
      constexpr int wv = decltype(W)::value;
      row_parity_tm<wv, tm_diag<BG>(wv)>(p, t0 / 4u, zl, ZL, wa, wb);
    });
    if (!pub_a && __any_sync(0xFFFFFFFFu, wa != 0)) {
      if (leader) atomicAdd(&synd[0], 1);
      pub_a = true;
    }
    if (!pub_b && __any_sync(0xFFFFFFFFu, wb != 0)) {
      if (leader) atomicAdd(&synd[1], 1);
      pub_b = true;
    }
    const volatile int* vs = synd;
    if ((!need_a || vs[0] != 0) && (!need_b || vs[1] != 0)) break;
  }
  mabs[0] = mabs[1] = 255;
  wcnt[0] = wcnt[1] = 0;
}

// The byte-pair layout's full-graph syndrome as straight-line code (see
// parity_rows_tm).
template <int BG, int LANES, bool ABS, int R = 0, int E = RowW<BG>::n>
__device__ __forceinline__ void parity_rows(const KParams& p, uint32_t zl, uint32_t ZL,
                                            const uint8_t* __restrict__ Lg, int& wa, int& wb) {
  if constexpr (R < E) {
    constexpr int w = RowW<BG>::w[R];
    row_parity<w, LANES, ABS>(p, row_tq<BG, R>(), w, zl, ZL, Lg, wa, wb);
    parity_rows<BG, LANES, ABS, R + 1, E>(p, zl, ZL, Lg, wa, wb);
  }
}

// Early-mode scan of a full graph in the byte-pair layout: straight-line
// blocks of STEP rows, then publish this warp's failures in the group's
// counters and stop once every live lane has one (see local_check_tm).
template <int BG, int LANES, bool ABS, int R, int STEP>
__device__ __forceinline__ void parity_rows_early(const KParams& p, uint32_t zl, uint32_t ZL,
                                                  const uint8_t* __restrict__ Lg, int& wa, int& wb, bool need_a,
                                                  bool need_b, bool& pub_a, bool& pub_b, int* synd) {
  if constexpr (R < RowW<BG>::n) {
    constexpr int E = R + STEP < RowW<BG>::n ? R + STEP : RowW<BG>::n;
    parity_rows<BG, LANES, ABS, R, E>(p, zl, ZL, Lg, wa, wb);
    const bool leader = (threadIdx.x & 31) == 0;
    if (!pub_a && __any_sync(0xFFFFFFFFu, wa != 0)) {
      if (leader) atomicAdd(&synd[0], 1);
      pub_a = true;
    }
    if (!pub_b && __any_sync(0xFFFFFFFFu, wb != 0)) {
      if (leader) atomicAdd(&synd[1], 1);
      pub_b = true;
    }
    const volatile int* vs = synd;
    if ((!need_a || vs[0] != 0) && (!need_b || vs[1] != 0)) return;
    parity_rows_early<BG, LANES, ABS, E, STEP>(p, zl, ZL, Lg, wa, wb, need_a, need_b, pub_a, pub_b, synd);
  }
}

// early: only "any unsatisfied check" matters (an early-stop iteration that
// is neither traced nor the last). A warp then stops scanning rows once it
// holds a failing check of every lane still being decoded (need_a/need_b):
// one failure anywhere in the group already rules the codeword out. Only
// when warps never straddle groups (Z % 32 == 0). wcnt is then a lower
// bound of the weight (>0 iff some check fails), and mabs is left at 255 for
// lanes known to fail.
template <int BG, int MAXW, int LANES, bool ABS>
__device__ __forceinline__ void local_check(const KParams& p, uint32_t zl, uint32_t ZL,
                                            const uint8_t* __restrict__ Lg, int* wcnt, int* mabs,
                                            bool early = false, bool need_a = true, bool need_b = true,
                                            int* synd = nullptr) {
  int wa = 0, wb = 0;
  bool stopped = false;
  if constexpr (BG != 0) {
    // full graph, early mode, group counters given: cooperative straight-line scan
    if (early && synd && p.rows == RowW<BG>::n) {
      const bool nb = LANES == 2 && need_b;
      bool pub_a = !need_a, pub_b = !nb;
      parity_rows_early<BG, LANES, ABS, 0, 4>(p, zl, ZL, Lg, wa, wb, need_a, nb, pub_a, pub_b, synd);
      wcnt[0] = wcnt[1] = 0;  // already counted in synd
      mabs[0] = mabs[1] = 255;  // only failing lanes stop early; the margin pass below is skipped
      const volatile int* vs = synd;
      if ((need_a && vs[0] == 0) || (nb && vs[1] == 0)) {
        // a live lane may have a zero syndrome: its margin is needed
        int ma[2] = {255, 255}, mb[2] = {255, 255};
        for (int c = 0; c < p.n_blocks; ++c) {
          const uint32_t u = ld_elem<LANES>(Lg + (uint32_t)c * ZL + zl);
          ma[c & 1] = min(ma[c & 1], abs((int)(u & 0xFFu) - 128));
          mb[c & 1] = min(mb[c & 1], abs((int)((u >> 8) & 0xFFu) - 128));
        }
        mabs[0] = min(ma[0], ma[1]);
        mabs[1] = min(mb[0], mb[1]);
      }
      return;
    }
  }
  if constexpr (BG == 0) {
    for (int r = 0; r < p.rows; ++r) {
      const int e0 = p.row_start[r];
      row_parity<MAXW, LANES>(p, p.tab_start[r] / 4u, p.row_start[r + 1] - e0, zl, ZL, Lg, wa, wb);
    }
  } else if (!early && p.rows == RowW<BG>::n) {
    parity_rows<BG, LANES, ABS>(p, zl, ZL, Lg, wa, wb);  // full graph: straight-line
  } else {
#pragma unroll 1
    for (int r = 0; r < p.rows; ++r) {
      const int e0 = p.row_start[r];
      const int t0 = p.tab_start[r];
      dispatch_w<BG>(p.row_start[r + 1] - e0, [&](auto W) {
        row_parity<decltype(W)::value, LANES, ABS>(p, t0 / 4u, decltype(W)::value, zl, ZL, Lg, wa, wb);
      });
      if (early) {
        const bool fa = !need_a || __any_sync(0xFFFFFFFFu, wa != 0);
        const bool fb = LANES == 1 || !need_b || __any_sync(0xFFFFFFFFu, wb != 0);
        if (fa && fb) {
          stopped = true;
          break;
        }
      }
    }
  }
  int ma[2] = {255, 255}, mb[2] = {255, 255};  // two chains, so the loads overlap
  if (!stopped) {
    int c = 0;
    for (; c + 2 <= p.n_blocks; c += 2) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t u = ld_elem<LANES>(Lg + (uint32_t)(c + i) * ZL + zl);
        ma[i] = min(ma[i], abs((int)(u & 0xFFu) - 128));
        mb[i] = min(mb[i], abs((int)((u >> 8) & 0xFFu) - 128));
      }
    }
    if (c < p.n_blocks) {
      const uint32_t u = ld_elem<LANES>(Lg + (uint32_t)c * ZL + zl);
      ma[0] = min(ma[0], abs((int)(u & 0xFFu) - 128));
      mb[0] = min(mb[0], abs((int)((u >> 8) & 0xFFu) - 128));
    }
  }
  wcnt[0] = wa;
  wcnt[1] = wb;
  mabs[0] = min(ma[0], ma[1]);
  mabs[1] = min(mb[0], mb[1]);
}

// Hard decisions of the first K positions, bit-packed LSB-first
// (decoder.py:332-334).
template <int LANES>
__device__ __forceinline__ void write_bits(const KParams& p, const uint8_t* __restrict__ Lg, int z,
                                           int lane, long long cw, uint32_t* __restrict__ bits) {
  const int K = p.k_b * p.z;
  for (int wi = z; wi < p.words; wi += p.z) {
    const int base = wi * 32;
    const int nb = min(32, K - base);
    uint32_t word = 0;
    for (int i = 0; i < nb; ++i) {
      const uint32_t u = Lg[(base + i) * LANES + lane];
      word |= (u < 128u ? 1u : 0u) << i;
    }
    bits[cw * p.words + wi] = word;
  }
}

// The same with whole warps when Z % 32 == 0 (warps never straddle groups):
// lane t of a warp reads position 32*w + t of both codewords with one
// coalesced load and two ballots build the two packed words.
template <int LANES, uint32_t ES = LANES>
__device__ __forceinline__ void write_bits_warp(const KParams& p, const uint8_t* __restrict__ Lg, int z,
                                                const int (&need)[2], long long cw0,
                                                uint32_t* __restrict__ bits, long long cw1 = -1) {
  if (cw1 < 0) cw1 = cw0 + 1;
  const int K = p.k_b * p.z;
  const int lid = z & 31;
  for (int wi = z >> 5; wi < p.words; wi += p.z >> 5) {
    const int pos = wi * 32 + lid;
    // lane b's byte: byte 1 (byte pairs) or byte 2 (TM half2)
    constexpr int sb = ES == 4 ? 16 : 8;
    const uint32_t u = pos < K ? (ES == 4 ? *reinterpret_cast<const uint32_t*>(Lg + pos * 4) : ld_elem<LANES>(Lg + pos * LANES))
                               : (0x80u | (0x80u << sb));
    const uint32_t wa = __ballot_sync(0xFFFFFFFFu, (u & 0xFFu) < 128u);
    const uint32_t wb = __ballot_sync(0xFFFFFFFFu, ((u >> sb) & 0xFFu) < 128u);
    if (lid == 0) {
      if (need[0]) bits[cw0 * p.words + wi] = wa;
      if (LANES == 2 && need[1]) bits[cw1 * p.words + wi] = wb;
    }
  }
}

// CRC over the K hard bits (codec.py:183-213) computed by the whole group.
// The bit-serial register is linear over GF(2): after all K bits it equals
// XOR over set bits i of rem(x^(K-1-i+L), g), tabulated on the host
// (crc_tab[i]). Each thread folds positions i = z, z+Z, ... and XORs its
// partial into the group's accumulator; the check passes when the XOR is 0.
template <int LANES, uint32_t ES = LANES>
__device__ __forceinline__ uint32_t crc_partial(const KParams& p, const uint8_t* __restrict__ Lg, int z,
                                                int lane) {
  const int K = p.k_b * p.z;
  uint32_t acc = 0;
  for (int i = z; i < K; i += p.z) {
    const uint32_t neg = Lg[i * ES + (ES == 4 ? 2 : 1) * lane] < 128u ? 0xFFFFFFFFu : 0u;
    acc ^= __ldg(p.crc_tab + i) & neg;
  }
  return acc;
}

// Layered decode of G groups x LANES codewords per CTA, everything resident
// in shared memory for the whole decode (decoder.py:486-540).
// Threads beyond G*Z (warp padding) shadow the last group's z = tid - (G-1)*Z
// clamp but never store, so the layer loop runs warp-uniform and the graph
// tables stay in uniform registers.
template <int BG, int MAXW, int LANES, int NREG, bool ABS, bool TM = false>
__global__ void __launch_bounds__(NREG ? 384 : 512, 1) k_decode_i8(const __grid_constant__ KParams p,
                                                                   const int8_t* __restrict__ llr, KOut o) {
  static_assert(NREG == 0 || (BG == 1 && LANES == 2), "register messages: BG1 pairs only");
  static_assert(!ABS || BG != 0, "absolute addressing: compile-time schedules only");
  static_assert(!TM || (BG != 0 && LANES == 2 && (NREG == 6 || NREG == 0) && ABS), "TM layout: pair shapes");
  constexpr uint32_t ES = TM ? 4 : LANES;  // bytes per position of L
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* lut = reinterpret_cast<uint16_t*>(smem);
  CtaState* cta = reinterpret_cast<CtaState*>(smem + kLutBytes);
  GroupState* gstate = reinterpret_cast<GroupState*>(smem + kLutBytes + kCtaBytes);
  const uint32_t data_off = data_offset(p.groups);

  const int tid = threadIdx.x;
  // not a padding thread; register-row shapes have one group of Z threads
  // with Z in {288, 320, 352, 384}, a whole number of warps (host-checked)
  const bool st_ok = NREG > 0 || tid < p.groups * p.z;
  const int g = st_ok ? tid / p.z : p.groups - 1;
  const int z = st_ok ? tid - g * p.z : (tid - g * p.z) % p.z;
  const long long cw0 = ((long long)blockIdx.x * p.groups + g) * LANES;
  const bool active = st_ok && cw0 < p.batch;        // owns real codewords
  const uint32_t ZL = (uint32_t)p.z * ES;
  const uint32_t zl = (uint32_t)z * ES;
  const long long n_c = (long long)p.n_blocks * p.z;
  uint8_t* Lg = smem + data_off + (uint32_t)g * (p.l_bytes + p.m_bytes);
  uint8_t* Mz = Lg + p.l_bytes + (uint32_t)z * p.m_stride;
  GroupState& gs = gstate[g];
  if constexpr (ABS) {
    // the host folded the L array's shared-window address into the graph
    // table (one group per CTA); a different window layout is a hard error
    if ((uint32_t)__cvta_generic_to_shared(Lg) != p.abs_base) __trap();
  }

  for (int i = tid; i < 128; i += blockDim.x) lut[i] = p.lut[i];
  if (tid == 0) {
    const long long first = (long long)blockIdx.x * p.groups * LANES;
    const long long rem = p.batch - first;
    cta->n_done = 0;
    cta->n_valid = (int)min(rem, (long long)p.groups * LANES);
    cta->kc[0] = p.magic;
    cta->kc[1] = p.one;
    cta->kc[2] = p.beta_h;
    cta->kc[3] = p.ndelta_h;
    cta->kc[4] = p.c_h;
  }
  if (st_ok && z == 0) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      gs.synd[l] = 0;
      gs.minabs[l] = 255;
      gs.done[l] = 0;
      gs.accept[l] = 0;
    }
  }

  uint32_t tbase = 0;  // TM: this thread's tensor-memory column slot
  if constexpr (TM) {
    if (tid < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&cta->kc[5])));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int warp = tid >> 5;
    // the warps of a lane quarter own consecutive slots (host: tm_shape)
    tbase = lds_u32(&cta->kc[5]) + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * p.tm_slot;
  }

  bool lane_valid[2];
  lane_valid[0] = active;
  lane_valid[1] = active && LANES == 2 && cw0 + 1 < p.batch;

  // load: int8 -> biased byte (x ^ 0x80), lanes interleaved; messages = 0.
  // The group's Z threads cooperate; with 16-byte aligned rows each thread
  // moves 16 positions per step (LDG.128 per codeword, PRMT interleave,
  // STS.128), otherwise one position per thread per step.
  if (st_ok) {
    uint32_t bad = 0;
    const uint4 zero4 = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    if (p.vec_load) {
      const int chunks = (int)(n_c >> 4);
      const uint4* rowA = reinterpret_cast<const uint4*>(llr + cw0 * n_c);
      const uint4* rowB = reinterpret_cast<const uint4*>(llr + (cw0 + 1) * n_c);
      // kLoadBatch steps' loads are issued before any is consumed: one HBM
      // round trip per batch instead of one per step
      for (int k0 = z; k0 < chunks; k0 += kLoadBatch * p.z) {
        uint4 ra[kLoadBatch], rb[kLoadBatch];
#pragma unroll
        for (int u = 0; u < kLoadBatch; ++u) {
          const int k = k0 + u * p.z;
          ra[u] = lane_valid[0] && k < chunks ? rowA[k] : make_uint4(0, 0, 0, 0);
          rb[u] = LANES == 2 && lane_valid[1] && k < chunks ? rowB[k] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kLoadBatch; ++u) {
        const int k = k0 + u * p.z;
        if (k >= chunks) break;
        uint4 a = ra[u];
        a.x ^= 0x80808080u; a.y ^= 0x80808080u; a.z ^= 0x80808080u; a.w ^= 0x80808080u;
        bad |= (a.x - 0x01010101u) & ~a.x; bad |= (a.y - 0x01010101u) & ~a.y;
        bad |= (a.z - 0x01010101u) & ~a.z; bad |= (a.w - 0x01010101u) & ~a.w;
        if (LANES == 2) {
          uint4 b = rb[u];
          b.x ^= 0x80808080u; b.y ^= 0x80808080u; b.z ^= 0x80808080u; b.w ^= 0x80808080u;
          if (lane_valid[1]) {
            bad |= (b.x - 0x01010101u) & ~b.x; bad |= (b.y - 0x01010101u) & ~b.y;
            bad |= (b.z - 0x01010101u) & ~b.z; bad |= (b.w - 0x01010101u) & ~b.w;
          }
          if constexpr (TM) {
            // position i of the chunk -> {0x64, u_b, 0x64, u_a} (biased half2)
            uint4* dst = reinterpret_cast<uint4*>(Lg) + 4 * k;
            const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t w4[4];
#pragma unroll
              for (int i = 0; i < 4; ++i)
                w4[i] = (__byte_perm(av[q], bv[q], 0x0400u + 0x0101u * i) & 0x00FF00FFu) | 0x64006400u;
              dst[q] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
          } else {
          uint4* dst = reinterpret_cast<uint4*>(Lg) + 2 * k;
          dst[0] = make_uint4(__byte_perm(a.x, b.x, 0x5140), __byte_perm(a.x, b.x, 0x7362),
                              __byte_perm(a.y, b.y, 0x5140), __byte_perm(a.y, b.y, 0x7362));
          dst[1] = make_uint4(__byte_perm(a.z, b.z, 0x5140), __byte_perm(a.z, b.z, 0x7362),
                              __byte_perm(a.w, b.w, 0x5140), __byte_perm(a.w, b.w, 0x7362));
          }
        } else {
          reinterpret_cast<uint4*>(Lg)[k] = a;
        }
        }
      }
      bad &= 0x80808080u;
    } else {
      for (int c = 0; c < p.n_blocks; ++c) {
        const long long n = (long long)c * p.z + z;
        uint32_t v = 0;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          uint32_t u = 0x80u;
          if (lane_valid[l]) {
            const int8_t x = llr[(cw0 + l) * n_c + n];
            bad |= (x == -128);
            u = (uint32_t)(uint8_t)x ^ 0x80u;
          }
          v |= u << (8 * l);
        }
        if constexpr (TM)
          *reinterpret_cast<uint32_t*>(Lg + (uint32_t)n * 4) = (v & 0xFFu) | ((v & 0xFF00u) << 8) | 0x64006400u;
        else
          st_elem<LANES>(Lg + (uint32_t)n * LANES, v);
      }
    }
    // messages: the group's whole message area is contiguous (m_bytes % 16 == 0)
    uint4* m4 = reinterpret_cast<uint4*>(Lg + p.l_bytes);
    if constexpr (TM) {
      // biased zero half2 (1152.0) in shared and tensor memory
      const uint4 hz = make_uint4(0x64806480u, 0x64806480u, 0x64806480u, 0x64806480u);
      for (uint32_t k = z; k < (p.m_bytes >> 4); k += p.z) m4[k] = hz;
      const uint32_t h = 0x64806480u;
      uint32_t c = 0;
      for (; c + 4 <= p.tm_cols; c += 4) tm_st4(tbase + c, h, h, h, h);
      for (; c < p.tm_cols; ++c) tm_st1(tbase + c, h);
      tm_wait_st();
    } else {
    for (uint32_t k = z; k < (p.m_bytes >> 4); k += p.z) m4[k] = zero4;
    }
    if (bad && o.status) atomicOr(o.status, 1);
  }
  __syncthreads();

  const Consts kc{lds_u32(&cta->kc[0]), lds_u32(&cta->kc[1]), lds_u32(&cta->kc[2]), lds_u32(&cta->kc[3]),
                  lds_u32(&cta->kc[4])};
  const RowCtx rc{zl, ZL, Lg, Mz, (uint32_t)__cvta_generic_to_shared(Mz), lut, kc, st_ok};
  const TmCtx tc{zl, ZL, (uint32_t)__cvta_generic_to_shared(Mz), tbase, kc};
  RegMsg<NREG> rm;
  rm.init();
  for (int it = 1; it <= p.max_iter; ++it) {
    if constexpr (TM) one_iteration_tm<BG, NREG>(p, tc, rm);
    else one_iteration<BG, MAXW, LANES, NREG, ABS>(p, rc, rm);
    const bool last = it == p.max_iter;
    if (!(p.early_stop != NRLDPC_STOP_NONE || p.trace || last)) continue;

    // ---- end-of-iteration check (decoder.py:497-536) ----
    // weights are only needed in full when traced or final
    const bool early = BG != 0 && !p.trace && !last && p.z % 32 == 0;
    {
      int wc[2], ma[2];
      if constexpr (TM)
        local_check_tm<BG>(p, zl, ZL, p.abs_base, wc, ma, early, lane_valid[0] && !gs.done[0],
                           lane_valid[1] && !gs.done[1], gs.synd);
      else
        local_check<BG, MAXW, LANES, ABS>(p, zl, ZL, Lg, wc, ma, early, lane_valid[0] && !gs.done[0],
                                          lane_valid[1] && !gs.done[1], gs.synd);
      if (active) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (wc[l]) atomicAdd(&gs.synd[l], wc[l]);
          atomicMin(&gs.minabs[l], ma[l]);
        }
      }
    }
    __syncthreads();
    if constexpr (TM) {
      // second pass: the margin, only when a live lane's syndrome is zero
      // (block-uniform: shared state read after the barrier)
      if (early && ((lane_valid[0] && !gs.done[0] && gs.synd[0] == 0) ||
                    (lane_valid[1] && !gs.done[1] && gs.synd[1] == 0))) {
        int ma[2];
        margin_tm(p, zl, ZL, p.abs_base, ma);
        atomicMin(&gs.minabs[0], ma[0]);
        atomicMin(&gs.minabs[1], ma[1]);
        __syncthreads();
      }
    }
    int cand[2] = {0, 0};
    if (active && p.early_stop != NRLDPC_STOP_NONE) {
#pragma unroll
      for (int l = 0; l < LANES; ++l)
        cand[l] = lane_valid[l] && !gs.done[l] && gs.synd[l] == 0 && gs.minabs[l] > 0;
    }
    if (p.early_stop == NRLDPC_STOP_CRC) {
      if (active) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (cand[l]) {
            const uint32_t part = p.crc_tab ? crc_partial<LANES, ES>(p, Lg, z, l) : 1u;
            if (part) atomicXor(reinterpret_cast<unsigned int*>(&gs.accept[l]), part);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int l = 0; l < LANES; ++l) cand[l] = cand[l] && p.crc_tab != nullptr && gs.accept[l] == 0;
    }
    int fin[2] = {0, 0};  // not frozen at the last iteration: final values
    if (active && last) {
#pragma unroll
      for (int l = 0; l < LANES; ++l) fin[l] = lane_valid[l] && !gs.done[l] && !cand[l];
    }
    if (active) {
      const int need[2] = {cand[0] || fin[0], LANES == 2 && (cand[1] || fin[1])};
      if (p.z % 32 == 0) {
        // group-uniform condition, whole warps per group: ballots are safe
        if (need[0] || need[1]) write_bits_warp<LANES, ES>(p, Lg, z, need, cw0, o.bits);
      } else {
#pragma unroll
        for (int l = 0; l < LANES; ++l)
          if (need[l]) write_bits<LANES>(p, Lg, z, l, cw0 + l, o.bits);
      }
      if (z == 0) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (!lane_valid[l]) continue;
          const long long cw = cw0 + l;
          const int wgt = gs.synd[l];
          const int mar = gs.minabs[l];
          if (p.trace) {
            o.trace_w[cw * p.max_iter + (it - 1)] = wgt;
            o.trace_m[cw * p.max_iter + (it - 1)] = (float)mar;
          }
          if (cand[l]) {
            o.iters[cw] = it;
            o.synd[cw] = 0;
            o.success[cw] = 1;
            if (o.crc_ok) o.crc_ok[cw] = 1;
          } else if (fin[l]) {
            o.iters[cw] = p.max_iter;
            o.synd[cw] = wgt;
            o.success[cw] = (p.early_stop == NRLDPC_STOP_NONE && wgt == 0 && mar > 0) ? 1 : 0;
            if (o.crc_ok) o.crc_ok[cw] = 0;
          }
        }
      }
    }
    __syncthreads();
    if (active && z == 0) {
      int newly = 0;
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if (cand[l]) {
          gs.done[l] = 1;
          ++newly;
        }
        gs.synd[l] = 0;
        gs.minabs[l] = 255;
        gs.accept[l] = 0;
      }
      if (newly) atomicAdd(&cta->n_done, newly);
    }
    __syncthreads();
    // block-wide vote: provably uniform, so the layer loop stays on the
    // uniform datapath (graph tables in uniform registers)
    if (__syncthreads_and(!p.trace && cta->n_done >= cta->n_valid)) break;
  }
  if constexpr (TM) {
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(lds_u32(&cta->kc[5])));
  }
}

// ---- lane-refill decode (early-stop modes) --------------------------------
// The pair kernel above runs a CTA until both of its codewords stop, so in
// syndrome/CRC modes a lane idles once its codeword converges. This
// persistent variant refills a lane as soon as its codeword stops: the CTA
// writes that codeword's results, takes the next codeword index from a
// global counter, loads it into the lane's bytes of L and zeroes the lane's
// messages, while the other lane keeps iterating. Each lane counts its own
// iterations; every codeword runs exactly the reference's schedule
// (decoder.py:486-540), so results are unchanged. One group of Z threads per
// CTA (Z % 32 == 0), two lanes, absolute addressing; not for traced runs.
struct LaneState {
  long long cw[2];  // codeword in each lane (-1: idle)
  int it[2];        // iterations run on it
  int pad[2];
};

template <int BG, int MAXW, int NREG, bool TM = false>
__global__ void __launch_bounds__(NREG ? 384 : 512, 1) k_decode_i8_refill(const __grid_constant__ KParams p,
                                                                          const int8_t* __restrict__ llr, KOut o) {
  constexpr int LANES = 2;
  constexpr bool ABS = true;
  static_assert(!TM || NREG == 6 || NREG == 0, "TM layout: pair shapes");
  constexpr uint32_t ES = TM ? 4 : LANES;  // bytes per position of L
  extern __shared__ __align__(16) uint8_t smem[];
  LaneState* ls = reinterpret_cast<LaneState*>(smem);  // the (unused) beta-table area
  CtaState* cta = reinterpret_cast<CtaState*>(smem + kLutBytes);
  GroupState& gs = *reinterpret_cast<GroupState*>(smem + kLutBytes + kCtaBytes);
  const uint32_t data_off = data_offset(1);
  const int tid = threadIdx.x;
  const int z = tid;
  const bool st_ok = true;
  const uint32_t ZL = (uint32_t)p.z * ES;
  const uint32_t zl = (uint32_t)z * ES;
  const long long n_c = (long long)p.n_blocks * p.z;
  uint8_t* Lg = smem + data_off;
  uint8_t* Mz = Lg + p.l_bytes + (uint32_t)z * p.m_stride;
  if ((uint32_t)__cvta_generic_to_shared(Lg) != p.abs_base) __trap();

  if (tid == 0) {
    cta->kc[0] = p.magic;
    cta->kc[1] = p.one;
    cta->kc[2] = p.beta_h;
    cta->kc[3] = p.ndelta_h;
    cta->kc[4] = p.c_h;
    for (int l = 0; l < 2; ++l) {
      const long long c = 2LL * blockIdx.x + l;
      ls->cw[l] = c < p.batch ? c : -1;
      ls->it[l] = 0;
      gs.synd[l] = 0;
      gs.minabs[l] = 255;
      gs.done[l] = 0;
      gs.accept[l] = 0;
    }
  }
  uint32_t tbase = 0;  // TM: this thread's tensor-memory column slot (see k_decode_i8)
  if constexpr (TM) {
    if (tid < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&cta->kc[5])));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int warp = tid >> 5;
    tbase = lds_u32(&cta->kc[5]) + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * p.tm_slot;
  }
  // messages: all zero (biased)
  {
    uint4* m4 = reinterpret_cast<uint4*>(Lg + p.l_bytes);
    const uint32_t zw = TM ? 0x64806480u : 0x80808080u;
    const uint4 zero4 = make_uint4(zw, zw, zw, zw);
    for (uint32_t k = z; k < (p.m_bytes >> 4); k += p.z) m4[k] = zero4;
    if constexpr (TM) {
      uint32_t c = 0;
      for (; c + 4 <= p.tm_cols; c += 4) tm_st4(tbase + c, zw, zw, zw, zw);
      for (; c < p.tm_cols; ++c) tm_st1(tbase + c, zw);
      tm_wait_st();
    }
  }
  __syncthreads();

  // load one lane's codeword (int8 -> biased byte) into its bytes of L:
  // 16 positions per thread and step when the row is 16-byte aligned (one
  // LDG.128, byte-interleaved into the other lane's bytes with PRMT)
  auto load_lane = [&](int l, long long cw) {
    uint32_t bad = 0;
    const int8_t* src = llr + cw * n_c;
    if (p.vec_load) {
      const uint4* row = reinterpret_cast<const uint4*>(src);
      uint4* dst = reinterpret_cast<uint4*>(Lg);
      const uint32_t keep = l ? 0x00FF00FFu : 0xFF00FF00u;
      const int chunks = (int)(n_c >> 4);
      for (int k0 = z; k0 < chunks; k0 += kLoadBatch * p.z) {
        uint4 ra[kLoadBatch];
#pragma unroll
        for (int u = 0; u < kLoadBatch; ++u) {
          const int k = k0 + u * p.z;
          ra[u] = k < chunks ? row[k] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kLoadBatch; ++u) {
        const int k = k0 + u * p.z;
        if (k >= chunks) break;
        uint4 a = ra[u];
        a.x ^= 0x80808080u; a.y ^= 0x80808080u; a.z ^= 0x80808080u; a.w ^= 0x80808080u;
        bad |= (a.x - 0x01010101u) & ~a.x; bad |= (a.y - 0x01010101u) & ~a.y;
        bad |= (a.z - 0x01010101u) & ~a.z; bad |= (a.w - 0x01010101u) & ~a.w;
        // spread 4 bytes to the lane's byte of 4 positions: 0x5140 -> lane 0,
        // then shift up by 8 for lane 1
        const uint32_t in4[4] = {a.x, a.y, a.z, a.w};
        if constexpr (TM) {
          // position -> the lane's half of its half2 word: {0x64, u}
          uint4* dh = reinterpret_cast<uint4*>(Lg) + 4 * k;
          const uint32_t keep_h = l ? 0x0000FFFFu : 0xFFFF0000u;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 d = dh[q];
            const uint32_t v0 = __byte_perm(in4[q], 0x64646464u, 0x4040u), v1 = __byte_perm(in4[q], 0x64646464u, 0x4141u);
            const uint32_t v2 = __byte_perm(in4[q], 0x64646464u, 0x4242u), v3 = __byte_perm(in4[q], 0x64646464u, 0x4343u);
            d.x = (d.x & keep_h) | (v0 & ~keep_h);
            d.y = (d.y & keep_h) | (v1 & ~keep_h);
            d.z = (d.z & keep_h) | (v2 & ~keep_h);
            d.w = (d.w & keep_h) | (v3 & ~keep_h);
            dh[q] = d;
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint4 d = dst[2 * k + h];
            const uint32_t u0 = __byte_perm(in4[2 * h], 0, 0x4140), u1 = __byte_perm(in4[2 * h], 0, 0x4342);
            const uint32_t u2 = __byte_perm(in4[2 * h + 1], 0, 0x4140), u3 = __byte_perm(in4[2 * h + 1], 0, 0x4342);
            const int sh = 8 * l;
            d.x = (d.x & keep) | ((u0 << sh) & ~keep);
            d.y = (d.y & keep) | ((u1 << sh) & ~keep);
            d.z = (d.z & keep) | ((u2 << sh) & ~keep);
            d.w = (d.w & keep) | ((u3 << sh) & ~keep);
            dst[2 * k + h] = d;
          }
        }
        }
      }
      bad &= 0x80808080u;
    } else {
      for (long long n = z; n < n_c; n += p.z) {
        const int8_t x = src[n];
        bad |= (x == -128);
        if constexpr (TM) reinterpret_cast<uint16_t*>(Lg)[n * 2 + l] = (uint16_t)(0x6400u | ((uint8_t)x ^ 0x80u));
        else Lg[n * 2 + l] = (uint8_t)x ^ 0x80u;
      }
    }
    if (bad && o.status) atomicOr(o.status, 1);
  };
  long long cw[2] = {ls->cw[0], ls->cw[1]};
  for (int l = 0; l < 2; ++l) {
    if (cw[l] >= 0) load_lane(l, cw[l]);
    else if constexpr (TM) for (long long n = z; n < n_c; n += p.z) reinterpret_cast<uint16_t*>(Lg)[n * 2 + l] = 0x6480u;
    else for (long long n = z; n < n_c; n += p.z) Lg[n * 2 + l] = 0x80u;
  }
  __syncthreads();

  const Consts kc{lds_u32(&cta->kc[0]), lds_u32(&cta->kc[1]), lds_u32(&cta->kc[2]), lds_u32(&cta->kc[3]),
                  lds_u32(&cta->kc[4])};
  const RowCtx rc{zl, ZL, Lg, Mz, (uint32_t)__cvta_generic_to_shared(Mz), nullptr, kc, st_ok};
  const TmCtx tc{zl, ZL, (uint32_t)__cvta_generic_to_shared(Mz), tbase, kc};
  RegMsg<NREG> rm;
  rm.init();
  int it[2] = {0, 0};
  while (cw[0] >= 0 || cw[1] >= 0) {
    if constexpr (TM) one_iteration_tm<BG, NREG>(p, tc, rm);
    else one_iteration<BG, MAXW, LANES, NREG, ABS>(p, rc, rm);
    bool act[2], last[2];
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      act[l] = cw[l] >= 0;
      it[l] += act[l] ? 1 : 0;
      last[l] = act[l] && it[l] == p.max_iter;
    }
    {
      int wc[2], ma[2];
      if constexpr (TM) local_check_tm<BG>(p, zl, ZL, p.abs_base, wc, ma, !last[0] && !last[1], act[0], act[1], gs.synd);
      else local_check<BG, MAXW, LANES, ABS>(p, zl, ZL, Lg, wc, ma, !last[0] && !last[1], act[0], act[1], gs.synd);
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        if (wc[l]) atomicAdd(&gs.synd[l], wc[l]);
        atomicMin(&gs.minabs[l], ma[l]);
      }
    }
    __syncthreads();
    if constexpr (TM) {
      // second pass: the margin, only when a live lane's syndrome is zero
      if (!last[0] && !last[1] && ((act[0] && gs.synd[0] == 0) || (act[1] && gs.synd[1] == 0))) {
        int ma[2];
        margin_tm(p, zl, ZL, p.abs_base, ma);
        atomicMin(&gs.minabs[0], ma[0]);
        atomicMin(&gs.minabs[1], ma[1]);
        __syncthreads();
      }
    }
    int cand[2], fin[2];
#pragma unroll
    for (int l = 0; l < 2; ++l) cand[l] = act[l] && gs.synd[l] == 0 && gs.minabs[l] > 0;
    if (p.early_stop == NRLDPC_STOP_CRC) {
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        if (cand[l]) {
          const uint32_t part = p.crc_tab ? crc_partial<LANES, ES>(p, Lg, z, l) : 1u;
          if (part) atomicXor(reinterpret_cast<unsigned int*>(&gs.accept[l]), part);
        }
      }
      __syncthreads();
#pragma unroll
      for (int l = 0; l < 2; ++l) cand[l] = cand[l] && p.crc_tab != nullptr && gs.accept[l] == 0;
    }
#pragma unroll
    for (int l = 0; l < 2; ++l) fin[l] = last[l] && !cand[l];
    const int need[2] = {cand[0] || fin[0], cand[1] || fin[1]};
    if (need[0] || need[1]) {
      write_bits_warp<LANES, ES>(p, Lg, z, need, cw[0], o.bits, cw[1]);
      if (z == 0) {
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          if (!need[l]) continue;
          const long long c = cw[l];
          o.iters[c] = cand[l] ? it[l] : p.max_iter;
          o.synd[c] = cand[l] ? 0 : gs.synd[l];
          o.success[c] = cand[l] ? 1 : 0;
          if (o.crc_ok) o.crc_ok[c] = cand[l] ? 1 : 0;
          // the next codeword for this lane
          const long long nxt = 2LL * gridDim.x + atomicAdd(o.work, 1);
          ls->cw[l] = nxt < p.batch ? nxt : -1;
        }
      }
    }
    __syncthreads();
    if (z == 0) {
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        gs.synd[l] = 0;
        gs.minabs[l] = 255;
        gs.accept[l] = 0;
      }
    }
    if (need[0] || need[1]) {
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        if (!need[l]) continue;
        cw[l] = ls->cw[l];
        it[l] = 0;
        if (cw[l] >= 0) {
          load_lane(l, cw[l]);
          // this lane's messages back to zero (bytes l of every 16-bit pair)
          const uint32_t keep = l ? 0x00FF00FFu : 0xFF00FF00u;  // register byte pairs
          const uint32_t keep_m = TM ? (l ? 0x0000FFFFu : 0xFFFF0000u) : keep;
          const uint32_t zb = (TM ? 0x64806480u : 0x80808080u) & ~keep_m;
          if constexpr (TM) {
            uint32_t c = 0;
            for (; c + 4 <= p.tm_cols; c += 4) {
              uint32_t r[4];
              tm_ld4(tbase + c, r[0], r[1], r[2], r[3]);
              tm_wait_ld<4>(r);
              tm_st4(tbase + c, (r[0] & keep_m) | zb, (r[1] & keep_m) | zb, (r[2] & keep_m) | zb,
                     (r[3] & keep_m) | zb);
            }
            for (; c < p.tm_cols; ++c) {
              uint32_t r[1];
              tm_ld1(tbase + c, r[0]);
              tm_wait_ld<1>(r);
              tm_st1(tbase + c, (r[0] & keep_m) | zb);
            }
            tm_wait_st();
          }
          uint4* m4 = reinterpret_cast<uint4*>(Lg + p.l_bytes);
          for (uint32_t k = z; k < (p.m_bytes >> 4); k += p.z) {
            uint4 v = m4[k];
            v.x = (v.x & keep_m) | zb;
            v.y = (v.y & keep_m) | zb;
            v.z = (v.z & keep_m) | zb;
            v.w = (v.w & keep_m) | zb;
            m4[k] = v;
          }
          rm.reset_lane(keep);
        }
      }
    }
    __syncthreads();
  }
  if constexpr (TM) {
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(lds_u32(&cta->kc[5])));
  }
}

// ---- quantize: depuncture + channel-domain -> decoder-domain LLRs ---------
// channel.py:64-83; arithmetic in float64 like the reference.
// With DEMAP the input is received BPSK symbols y and the LLR is formed first
// exactly as channel.demap_llr does it: (2.0 * y) / (sigma * sigma), float64
// (channel.py:57-61), with sigma2 = sigma*sigma computed on the host.
template <typename Tin, int MODE, bool DEMAP>
__device__ __forceinline__ void quant_one(double v, bool pad, double scale, double clip, double sigma2,
                                          void* __restrict__ out, long long i) {
  if (pad) v = 0.0;
  else if (DEMAP) v = __ddiv_rn(__dmul_rn(2.0, v), sigma2);
  if (MODE == NRLDPC_INT8) {
    double q = rint(v * scale);
    q = fmin(fmax(q, -127.0), 127.0);
    reinterpret_cast<int8_t*>(out)[i] = (int8_t)q;
  } else if (MODE == NRLDPC_F16) {
    double c = fmin(fmax(v, -clip), clip);
    c = fmin(fmax(c, -65504.0), 65504.0);
    reinterpret_cast<__half*>(out)[i] = __double2half(c);
  } else {
    const double c = fmin(fmax(v, -clip), clip);
    reinterpret_cast<float*>(out)[i] = __double2float_rn(c);
  }
}

// One thread per 8 consecutive output positions of one codeword row (grid:
// x over the row, y over codewords). Rows whose input is 16-byte aligned take
// two-to-four 128-bit loads per thread and one packed store; the 2Z punctured
// head and unaligned shapes (odd Z) use the per-element path. HBM-bound:
// 8 B (f64) or 4 B (f32) in per position, 1/2/4 B out.
template <typename Tin, int MODE, bool DEMAP = false>
__global__ void __launch_bounds__(256) k_quantize(const Tin* __restrict__ in, long long batch, int n_tx,
                                                  int n_c, int two_z, double scale, double clip,
                                                  void* __restrict__ out, double sigma2, int vec) {
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (j0 >= n_c) return;
  for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
    const Tin* row = in + b * n_tx;
    const long long o0 = b * n_c + j0;
    if (vec && j0 >= two_z && j0 + 8 <= n_c) {
      double v[8];
      if (sizeof(Tin) == 8) {
        const double2* q = reinterpret_cast<const double2*>(row + (j0 - two_z));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 d = __ldcs(q + k);
          v[2 * k] = d.x;
          v[2 * k + 1] = d.y;
        }
      } else {
        const float4* q = reinterpret_cast<const float4*>(row + (j0 - two_z));
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float4 f = __ldcs(q + k);
          v[4 * k] = f.x;
          v[4 * k + 1] = f.y;
          v[4 * k + 2] = f.z;
          v[4 * k + 3] = f.w;
        }
      }
      if (MODE == NRLDPC_INT8) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double x = DEMAP ? __ddiv_rn(__dmul_rn(2.0, v[k]), sigma2) : v[k];
          double q = rint(x * scale);
          q = fmin(fmax(q, -127.0), 127.0);
          const uint32_t byte = (uint32_t)(uint8_t)(int8_t)q;
          if (k < 4) lo |= byte << (8 * k);
          else hi |= byte << (8 * (k - 4));
        }
        if (vec == 2) {
          *reinterpret_cast<uint2*>(reinterpret_cast<int8_t*>(out) + o0) = make_uint2(lo, hi);
        } else {
          uint32_t* o = reinterpret_cast<uint32_t*>(reinterpret_cast<int8_t*>(out) + o0);
          o[0] = lo;
          o[1] = hi;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) quant_one<Tin, MODE, DEMAP>(v[k], false, scale, clip, sigma2, out, o0 + k);
      }
    } else {
      for (int k = 0; k < 8 && j0 + k < n_c; ++k) {
        const int j = j0 + k;
        const bool pad = j < two_z;
        quant_one<Tin, MODE, DEMAP>(pad ? 0.0 : (double)row[j - two_z], pad, scale, clip, sigma2, out, o0 + k);
      }
    }
  }
}

// ---- ALU roofline microbenchmark -----------------------------------------
// Eight independent half2 chains per thread; MIXED interleaves HMNMX2 (ALU
// pipe) with HFMA2 (FMA pipe) 1:1 to find the dual-issue ceiling, otherwise
// HMNMX2 only (ALU-pipe ceiling). Same instruction classes as the decode.
template <bool MIXED>
__global__ void __launch_bounds__(512) k_alu_peak(uint32_t* out, int iters, uint32_t seed) {
  half2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = u2h(seed + threadIdx.x * 7919u + i * 104729u);
  const half2 c = u2h(seed ^ 0x3C003C00u);
  const half2 d = u2h(seed ^ 0x57F057F0u);
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __hmin2(a[i], __habs2(d));
      if (MIXED) a[i] = __hfma2(a[i], c, d);
      else a[i] = __hmax2(a[i], c);
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= h2u(a[i]);
  if (x == 0x12345678u) out[0] = x;  // keep the chains alive
}

}  // namespace nr

#include "nrldpc_float.cuh"
#include "nrldpc_codec.cuh"
#include "nrldpc_flood.cuh"

// ---------------------------------------------------------------------------
// Host side

// Stream-ordered scratch (lane-refill work counters, float-engine message
// workspaces) comes from a library-private pool per device. Reuse of a freed
// block is limited to orderings the caller's own streams/events establish:
// with the default pool's internal-dependency reuse, a launch on stream B
// could be made to wait for an earlier launch on stream A whose block it
// recycles, which serialises independent batches on separate streams. The
// release threshold keeps freed blocks cached across synchronisations.
cudaError_t scratch_alloc(void** ptr, size_t bytes, int device, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    cudaMemPool_t& slot = pools[device & 63];
    if (!slot) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      cudaError_t e = cudaMemPoolCreate(&slot, &props);
      int off = 0;
      uint64_t keep = ~0ull;
      if (e == cudaSuccess) e = cudaMemPoolSetAttribute(slot, cudaMemPoolReuseAllowOpportunistic, &off);
      if (e == cudaSuccess) e = cudaMemPoolSetAttribute(slot, cudaMemPoolReuseAllowInternalDependencies, &off);
      if (e == cudaSuccess) e = cudaMemPoolSetAttribute(slot, cudaMemPoolAttrReleaseThreshold, &keep);
      if (e != cudaSuccess) {
        if (slot) cudaMemPoolDestroy(slot);
        slot = nullptr;
        return e;
      }
    }
    pool = slot;
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pool, st);
}

// One launch configuration of the decode kernel.
struct Shape {
  int lanes = 1;    // codewords per half2 lane pair
  int nreg = 0;     // leading rows whose messages live in registers (BG1 pairs)
  int groups = 1;   // codeword groups (of Z threads) per CTA
  int threads = 0;  // 0: no feasible shape
  size_t smem = 0;
  int occ = 0;      // resident CTAs per SM (0: not queried yet)
  int refill_occ = 0;  // the same for this shape's lane-refill kernel
  bool abs = false; // kp.cb holds absolute shared-window addresses
  bool tm = false;  // TM layout (half2 L, shared/tensor-memory messages)
  KParams kp{};
};

struct nrldpc_plan {
  int device = 0;
  bool coscheduled = false;  // launches share SMs with other plans' launches
  int precision = NRLDPC_INT8;
  int early_stop = NRLDPC_STOP_SYNDROME;
  int crc_kind = NRLDPC_CRC24B;
  uint32_t* d_crc_tab = nullptr;  // device: rem(x^(K-1-i+L), g) for i < K (crc mode)
  EncSched enc{};                 // systematic-encoder schedule (enc_ok)
  FloodTables flood{};            // column-major edge lists (flooding schedule)
  bool enc_ok = false;
  double beta = 0.75;
  int max_iter = 20;
  int k_b = 0, z = 0, rows = 0, n_blocks = 0, n_edges = 0, maxw = 0;
  int schedule = 0;  // 0 generic, 1/2: compile-time BG1/BG2 row schedule
  KParams base{};    // graph tables + config, before the shape-dependent scaling
  Shape main;        // the launch shape
  // host-path staging (nrldpc_decode_host[_async])
  std::mutex host_mu;
  // host pipeline: streams[0] copies inputs in (in chunk order), streams[1]
  // copies results out, the rest decode chunks as their input lands (one
  // event per chunk). Two slots of device buffers let one call's copies and
  // decode overlap the next call's (nrldpc_decode_host_async).
  static constexpr int kHostStreams = 18;
  static constexpr int kSlots = 2;
  cudaStream_t streams[kHostStreams] = {};
  std::vector<cudaEvent_t> chunk_ev;
  struct Slot {
    void* d_buf = nullptr;
    size_t d_cap = 0;
    int32_t* h_status = nullptr;  // pinned: the slot's status word lands here
    cudaEvent_t done = nullptr;   // recorded after the slot's result copies
    int64_t ticket = -1;          // call in flight in this slot (-1: none)
    // pageable callers: inputs are staged through h_in (parallel host copy
    // into pinned memory, chunk by chunk, overlapped with the chunks' DMA);
    // results land in h_out and are copied to the caller's buffers when the
    // call retires
    uint8_t* h_in = nullptr;
    size_t h_in_cap = 0;
    uint8_t* h_out = nullptr;
    size_t h_out_cap = 0;
    struct Dst {
      void* p;
      size_t off, n;
    } dst[5] = {};
    int n_dst = 0;
  } slot[kSlots];
  int64_t next_ticket = 0;
  // Calls retired on behalf of a later call (slot reuse, or a synchronous
  // call draining the pipeline) whose input was rejected: their status is
  // kept here until their own nrldpc_host_wait, so an error is reported
  // against the call that caused it and never fails the call reusing the
  // slot. Bounded: the oldest entries go first.
  std::vector<int64_t> failed;
  static constexpr size_t kMaxFailed = 4096;
};

namespace {

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Per-thread message rows are padded so the row stride is an odd number of
// 32-bit words: 32 consecutive z then hit 32 distinct banks.
size_t padded_edges(int n_edges, int lanes) {
  const size_t unit = lanes == 2 ? 2 : 4;  // stride bytes = e_pad*lanes = 4*(odd)
  size_t e = (size_t)n_edges;
  while (((e * lanes) % 4) != 0 || (((e * lanes) / 4) % 2) == 0) ++e;
  (void)unit;
  return e;
}

// dynamic shared memory's offset in the CTA's shared window (sm_90+ reserve
// 1 KB per CTA; no static __shared__ in k_decode_i8, no clusters)
constexpr uint32_t kSmemWindowBase = 0x400;

size_t smem_for(int groups, size_t l_bytes, size_t m_bytes) {
  return kLutBytes + kCtaBytes + sizeof(GroupState) * groups + 16 + groups * (l_bytes + m_bytes);
}

// Launch (or, with llr == nullptr, only prepare: set the smem attribute and
// query occupancy) one decode kernel instance for `sh`.
template <int BG, int MAXW, int LANES, int NREG = 0, bool ABS = false, bool TM = false>
cudaError_t launch_i8(Shape& sh, int device, const int8_t* llr, long long batch, const KOut& o,
                      cudaStream_t st) {
  static bool attr_done[64] = {};
  auto kern = k_decode_i8<BG, MAXW, LANES, NREG, ABS, TM>;
  if (!attr_done[device & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    attr_done[device & 63] = true;
  }
  if (!sh.occ) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sh.threads, sh.smem);
    if (e != cudaSuccess) return e;
    sh.occ = occ > 0 ? occ : 1;
  }
  if (!llr) return cudaSuccess;
  KParams kp = sh.kp;
  kp.batch = batch;
  kp.trace = o.trace_w != nullptr;
  kp.vec_load = ((long long)kp.n_blocks * kp.z) % 16 == 0 && ((uintptr_t)llr & 15) == 0;
  const long long per_cta = (long long)sh.groups * LANES;
  const long long grid = (batch + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid, sh.threads, sh.smem, st>>>(kp, llr, o);
  ++g_launches;
  return cudaGetLastError();
}

int crc_params(int kind, int* len, uint32_t* poly) {
  switch (kind) {
    case NRLDPC_CRC24A: *len = 24; *poly = 0x864CFB; return 0;
    case NRLDPC_CRC24B: *len = 24; *poly = 0x800063; return 0;
    case NRLDPC_CRC16: *len = 16; *poly = 0x1021; return 0;
    default: return -1;
  }
}

uint16_t float_to_half_bits(float f) {
  __half h = __float2half_rn(f);
  uint16_t b;
  std::memcpy(&b, &h, 2);
  return b;
}

// Half-precision arithmetic form of the int8 beta rule, if one exists:
// floor(beta*m) == RN_half(bh*(m - delta) + C) - C for all m in [0,127], with
// bh, delta, C halves and the FMA rounded once (HFMA2). Checked exhaustively
// here, so the device never depends on an unverified identity; otherwise the
// kernel falls back to the 128-entry LUT.
double half_round(double x) {  // x in [1024, 2048): half ulp is 1
  return std::nearbyint(x);
}

void find_beta_arith(double beta, KParams* kp) {
  kp->beta_mode = 0;
  const float bf = (float)beta;
  const __half bh0 = __float2half_rn(bf);
  uint16_t b0;
  std::memcpy(&b0, &bh0, 2);
  for (int db = 0; db <= 64; ++db) {
    for (int sgn = 0; sgn < 2; ++sgn) {
      const int bits = sgn ? (int)b0 - db : (int)b0 + db;
      if (bits <= 0 || bits >= 0x3C01) continue;  // (0, 1]
      __half hb;
      const uint16_t ub = (uint16_t)bits;
      std::memcpy(&hb, &ub, 2);
      const double bh = (double)__half2float(hb);
      for (int d16 = 0; d16 <= 16; ++d16) {
        const double delta = d16 / 16.0;
        for (int c = 1025; c <= 1040; ++c) {
          bool ok = true;
          for (int m = 0; m < 128 && ok; ++m) {
            const double x = bh * ((double)m - delta) + (double)c;  // exact in double
            if (x < 1024.0 || x >= 2048.0) { ok = false; break; }
            ok = half_round(x) - c == std::floor(beta * (double)m);
          }
          if (ok) {
            kp->beta_mode = 1;
            kp->beta_h = (uint32_t)ub * 0x10001u;
            kp->ndelta_h = (uint32_t)float_to_half_bits((float)-delta) * 0x10001u;
            kp->c_h = (uint32_t)float_to_half_bits((float)c) * 0x10001u;
            return;
          }
        }
      }
      if (db == 0) break;
    }
  }
}

// Pick lanes (codewords per half2), register-resident message rows and
// groups per CTA. Two codewords per lane (half2) whenever the pair's state
// fits on chip; for BG1 at the largest Z the first rows' messages move from
// shared memory into registers to make room. Smaller CTAs keep the per-layer
// barrier cheap; more codewords per SM come from more CTAs.
// Float engines: 4 bytes per position per group (one f32 codeword, or a
// half2 pair of f16 codewords); messages go to a global workspace.
Shape choose_shape_float(const nrldpc_plan* p) {
  const size_t smem_max = 232448;
  const size_t lb = align16((size_t)p->n_blocks * p->z * 4);
  auto smem_f = [&](int g) { return (size_t)kCtaBytes + 16 + sizeof(FltState) * g + g * lb; };
  int best_g = 1;
  double best_waste = 1e9;
  for (int g = 1; g * p->z <= 512; ++g) {
    if (smem_f(g) > smem_max) break;
    const int thr = g * p->z, thr32 = (thr + 31) / 32 * 32;
    const double waste = double(thr32 - thr) / thr32;
    if (thr32 < 64 && (g + 1) * p->z <= 512 && smem_f(g + 1) <= smem_max) continue;
    if (waste < best_waste - 1e-9) {
      best_waste = waste;
      best_g = g;
    }
    if (waste <= 1.0 / 16) break;
  }
  Shape sh;
  sh.lanes = p->precision == NRLDPC_F16 ? 2 : 1;
  sh.groups = best_g;
  sh.threads = (best_g * p->z + 31) / 32 * 32;
  sh.smem = smem_f(best_g);
  sh.kp = p->base;
  sh.kp.groups = best_g;
  sh.kp.l_bytes = (uint32_t)lb;
  for (int t = 0; t < NR_MAX_TAB; ++t) {
    sh.kp.sh[t] = p->base.sh[t] * 4u;
    sh.kp.cb[t] = p->base.cb[t] * (uint32_t)p->z * 4u;
  }
  return sh;
}

// Host side of dispatch_unit: which consecutive column-disjoint row pairs
// have a fused body.
bool fused_pair(int schedule, int wa, int wb) {
  static const int bg1[][2] = {{5, 5}, {5, 4}, {6, 6}, {4, 5}, {6, 5}};
  static const int bg2[][2] = {{4, 4}, {4, 3}, {5, 4}, {5, 3}, {3, 4}};
  const auto& t = schedule == 1 ? bg1 : bg2;
  for (const auto& q : t)
    if (q[0] == wa && q[1] == wb) return true;
  return false;
}

// Layer units for rows nreg.. of a BG1/BG2 kernel (see KParams::unit_a).
// Per-thread shared-memory message slots of rows nreg.. (byte offsets).
// Edge-ordered: row r's edges at (row_start[r] - e_reg) * lanes. Paired (ABS
// pair shapes): each row's first 2*floor(w/2) edges as whole 32-bit words;
// the last edge of an odd row takes half of a word whose other half holds
// another odd row's last edge. Returns the slot count in edges.
struct MsgLayout {
  uint32_t mb[NR_MAX_ROWS];  // first (paired) slot
  uint32_t mh[NR_MAX_ROWS];  // odd edge's half-word slot (paired only)
  int slots = 0;
};

MsgLayout msg_layout(const nrldpc_plan* p, int nreg, int e_reg, int lanes, bool paired) {
  const KParams& b = p->base;
  MsgLayout m{};
  if (!paired) {
    for (int r = nreg; r < p->rows; ++r) m.mb[r] = (uint32_t)(b.row_start[r] - e_reg) * lanes;
    m.slots = b.row_start[p->rows] - e_reg;
    return m;
  }
  int cur = 0, free_half = -1;  // in edge slots (2 bytes each)
  for (int r = nreg; r < p->rows; ++r) {
    const int w = b.row_start[r + 1] - b.row_start[r];
    m.mb[r] = (uint32_t)cur * 2u;
    cur += 2 * (w / 2);
    if (w & 1) {
      if (free_half >= 0) {
        m.mh[r] = (uint32_t)free_half * 2u;
        free_half = -1;
      } else {
        m.mh[r] = (uint32_t)cur * 2u;
        free_half = cur + 1;
        cur += 2;
      }
    }
  }
  m.slots = cur;
  return m;
}

// On-chip message variant of a float shape (k_decode_flt FTM): single-group
// BG1/BG2 shapes (Z % 32 == 0, Z <= 384). Rows by ftm_kind: global rows keep
// workspace slots (they must be the leading rows: e_reg edges), shared rows
// one word per edge in a thread-major row (odd word stride), tensor rows one
// TMEM column per edge. Expects build_units to run with the returned layout;
// returns false (shape unchanged) when the layout does not fit.
// NRLDPC_NO_TM=1 disables it.
bool ftm_layout(const nrldpc_plan* p, Shape& sh, MsgLayout& ml) {
  if (p->schedule == 0 || sh.groups != 1 || p->z % 32 != 0 || p->z > 384 || getenv("NRLDPC_NO_TM")) return false;
  const size_t smem_max = 232448, one_per_sm = smem_max / 2 + 1024;
  const KParams& b = p->base;
  const int warps = p->z / 32;
  const uint32_t slot = 512u / (uint32_t)((warps + 3) / 4);
  uint32_t sm_slots = 0, tm_cols = 0;
  int e_glob = 0;
  bool leading = true;
  for (int r = 0; r < p->rows; ++r) {
    const int w = b.row_start[r + 1] - b.row_start[r];
    const int kind = p->schedule == 1 ? ftm_kind<1>(w) : ftm_kind<2>(w);
    if (kind == 0) {
      if (!leading) return false;
      ml.mb[r] = (uint32_t)b.row_start[r];
      e_glob = b.row_start[r + 1];
    } else {
      leading = false;
      if (kind == 1) {
        ml.mb[r] = sm_slots * 4u;
        sm_slots += (uint32_t)w;
      } else {
        ml.mb[r] = tm_cols;
        tm_cols += (uint32_t)w;
      }
    }
  }
  if (tm_cols > slot) return false;
  const uint32_t e = sm_slots | 1u;
  const size_t mb = align16((size_t)p->z * e * 4);
  const size_t need = sh.smem + mb;  // header + L (one group) + shared message rows
  if (need > smem_max) return false;
  sh.tm = true;
  sh.smem = std::max(need, one_per_sm);
  sh.kp.m_bytes = (uint32_t)mb;
  sh.kp.m_stride = e * 4u;
  sh.kp.e_reg = e_glob;
  sh.kp.tm_cols = tm_cols;
  sh.kp.tm_slot = slot;
  return true;
}

void build_units(const nrldpc_plan* p, int nreg, const MsgLayout& ml, KParams& kp) {
  const KParams& b = p->base;
  int n = 0;
  for (int r = nreg; r < p->rows;) {
    const int wa = b.row_start[r + 1] - b.row_start[r];
    const uint32_t ta = b.tab_start[r] / 4u;
    if (p->schedule != 0 && !b.bar_after[r] && r + 1 < p->rows) {
      const int wb = b.row_start[r + 2] - b.row_start[r + 1];
      if (fused_pair(p->schedule, wa, wb)) {
        // the two rows share no column, so their order inside the fused body
        // is free: the heavier row goes first and (4,5) runs on the (5,4)
        // body, (3,4) on (4,3) (fewer bodies in the hot loop)
        const int f = wa < wb ? 1 : 0;  // row r + f becomes row a
        const int ra = r + f, rb = r + 1 - f;
        kp.unit_a[n] = make_uint4((uint32_t)(std::max(wa, wb) | std::min(wa, wb) << 8), b.bar_after[r + 1],
                                  b.tab_start[ra] / 4u, ml.mb[ra]);
        kp.unit_b[n] = make_uint4(b.tab_start[rb] / 4u, ml.mb[rb], ml.mh[ra], ml.mh[rb]);
        ++n;
        r += 2;
        continue;
      }
    }
    kp.unit_a[n] = make_uint4((uint32_t)wa, b.bar_after[r], ta, ml.mb[r]);
    kp.unit_b[n] = make_uint4(0, 0, ml.mh[r], 0);
    ++n;
    r += 1;
  }
  kp.n_units = n;
  kp.unit_a[n] = make_uint4(0, 0, 0, 0);
  kp.unit_b[n] = make_uint4(0, 0, 0, 0);
}

Shape choose_shape(const nrldpc_plan* p, int max_lanes) {
  const size_t smem_max = 232448;
  const size_t n_pos = (size_t)p->n_blocks * p->z;
  auto msg_bytes = [&](int lanes, int e_reg) {
    return align16((size_t)p->z * padded_edges(p->n_edges - e_reg, lanes) * lanes);
  };
  int lanes = 1, nreg = 0;
  if (max_lanes >= 2) {
    const bool fits = smem_for(1, align16(n_pos * 2), msg_bytes(2, 0)) <= smem_max;
    // BG1 pairs with Z > 256 run one group per CTA; they keep the messages
    // of rows 0..5 in registers whenever those rows exist (fewer shared
    // accesses, and one kernel for all large Z, which matters when many Z
    // decode concurrently). Rows 0..1 / 0..3 when rows_used < 6.
    const bool big = p->schedule == 1 && p->z > 256 && p->z <= 384 && p->z % 32 == 0;
    if (fits && !big) {
      lanes = 2;
    } else if (p->schedule == 1 && p->z <= 384 && p->z % 32 == 0) {
      for (int nr : {6, 4, 2}) {
        if (nr > p->rows) continue;
        if (smem_for(1, align16(n_pos * 2), msg_bytes(2, RowW<1>::e0[nr])) <= smem_max) {
          lanes = 2;
          nreg = nr;
          break;
        }
      }
      if (!nreg && fits) lanes = 2;
    }
  }
  const int e_reg = nreg ? RowW<1>::e0[nreg] : 0;
  const size_t lb = align16(n_pos * lanes);
  size_t e_pad = padded_edges(p->n_edges - e_reg, lanes);
  size_t mb = msg_bytes(lanes, e_reg);
  int best_g = 1;
  double best_waste = 1e9;
  const int max_thr = nreg ? 384 : 512;
  for (int g = 1; g * p->z <= max_thr; ++g) {
    if (smem_for(g, lb, mb) > smem_max) break;
    const int thr = g * p->z;
    const int thr32 = (thr + 31) / 32 * 32;
    const double waste = double(thr32 - thr) / thr32;
    if (thr32 < 64 && (g + 1) * p->z <= max_thr && smem_for(g + 1, lb, mb) <= smem_max) continue;
    if (waste < best_waste - 1e-9) {
      best_waste = waste;
      best_g = g;
    }
    if (waste <= 1.0 / 16) break;
  }
  // single-group pair shapes of the BG1/BG2 schedules address L absolutely:
  // the table holds column base + the L array's shared-window address (the
  // dynamic window starts after the 1 KB system reservation; the kernel
  // verifies), and their messages use the paired word layout.
  // Absolute L addressing is ~5% faster for one decode alone, but measured
  // ~12% slower when many plans' kernels share the SMs (mixed-shape batches,
  // nrldpc_plan_set_coscheduled); register-row shapes always use it.
  bool abs = best_g == 1 && lanes == 2 && p->schedule != 0 && (nreg > 0 || !p->coscheduled);
  MsgLayout ml = msg_layout(p, nreg, e_reg, lanes, abs);
  if (abs) {
    const size_t e_pad_p = padded_edges(ml.slots, lanes);
    const size_t mb_p = align16((size_t)p->z * e_pad_p * lanes);
    if (smem_for(1, lb, mb_p) <= smem_max) {
      e_pad = e_pad_p;
      mb = mb_p;
    } else if (nreg == 0) {
      abs = false;
      ml = msg_layout(p, nreg, e_reg, lanes, false);
    } else {
      return Shape{};  // no feasible layout (threads == 0: plan creation fails)
    }
  }
  Shape sh;
  sh.lanes = lanes;
  sh.nreg = nreg;
  sh.groups = best_g;
  sh.threads = (best_g * p->z + 31) / 32 * 32;
  sh.smem = smem_for(best_g, lb, mb);
  sh.kp = p->base;
  sh.kp.groups = best_g;
  sh.kp.l_bytes = (uint32_t)lb;
  sh.kp.m_bytes = (uint32_t)mb;
  sh.kp.m_stride = (uint32_t)(e_pad * lanes);
  sh.kp.e_reg = e_reg;
  build_units(p, nreg, ml, sh.kp);
  sh.kp.magic = 0x64646464u;
  sh.kp.one = 0x3C003C00u;
  sh.kp.abs_base = abs ? kSmemWindowBase + data_offset(1) : 0u;
  sh.abs = sh.kp.abs_base != 0;
  for (int t = 0; t < NR_MAX_TAB; ++t) {
    sh.kp.sh[t] = p->base.sh[t] * lanes;
    sh.kp.cb[t] = p->base.cb[t] * (uint32_t)p->z * lanes + sh.kp.abs_base;
  }
  return sh;
}

// TM layout (k_decode_i8 TM) of a single-group pair shape that holds an SM
// alone: L as biased half2, messages of rows >= nreg with w >= SMW in
// shared memory (one half2 per edge, odd word stride) and the others in
// tensor memory (one column per edge). The CTA allocates all 512 TMEM
// columns, so the shape keeps one CTA per SM (shared memory is padded to
// force it). Returns the byte-pair shape unchanged when the layout does not
// apply or fit; NRLDPC_NO_TM=1 disables it.
Shape tm_shape(const nrldpc_plan* p, const Shape& leg) {
  const size_t smem_max = 232448, one_per_sm = smem_max / 2 + 1024;
  if (!leg.abs || leg.groups != 1 || leg.lanes != 2 || p->z % 32 != 0 || p->z > 384 || getenv("NRLDPC_NO_TM"))
    return leg;
  int smw = 0;
  if (p->schedule == 1 && leg.nreg == 6) smw = tm_smw<1, 6>();
  else if (p->schedule == 1 && leg.nreg == 0) smw = tm_smw<1, 0>();
  else if (p->schedule == 2 && leg.nreg == 0) smw = tm_smw<2, 0>();
  // byte-pair shapes with several CTAs per SM keep them (register-row shapes
  // hold an SM alone through their register count)
  if (!smw || (leg.nreg == 0 && leg.smem < one_per_sm)) return leg;
  const int warps = p->z / 32;
  const uint32_t slot = 512u / (uint32_t)((warps + 3) / 4);
  const KParams& b = p->base;
  // the row bodies take the last edge of every non-core row as the degree-1
  // extension column at shift 0 (tm_diag)
  for (int r = 0; r < p->rows; ++r) {
    const int w = b.row_start[r + 1] - b.row_start[r];
    const bool diag = p->schedule == 1 ? tm_diag<1>(w) : tm_diag<2>(w);
    if (diag && b.sh[b.tab_start[r] + w - 1] != 0) return leg;
  }
  MsgLayout ml{};
  uint32_t sm_slots = 0, tm_cols = 0;
  uint32_t r45[2] = {0, 0};
  if (leg.nreg == 6) {  // rows 4 and 5: tensor memory (one_iteration_tm)
    r45[0] = 0;
    r45[1] = (uint32_t)(b.row_start[5] - b.row_start[4]);
    tm_cols = (uint32_t)(b.row_start[6] - b.row_start[4]);
  }
  for (int r = leg.nreg; r < p->rows; ++r) {
    const int w = b.row_start[r + 1] - b.row_start[r];
    if (w >= smw) {
      ml.mb[r] = sm_slots * 4u;
      sm_slots += (uint32_t)(leg.nreg == 6 ? w + (w & 1) : w);  // RowWorkTM::V2: 8-byte aligned rows
    } else {
      ml.mb[r] = tm_cols;
      tm_cols += (uint32_t)w;
    }
  }
  if (tm_cols > slot) return leg;
  // word stride: odd (32-bit accesses), or 2 x odd for the LDS.64 rows, so
  // the accesses of consecutive z hit distinct banks
  uint32_t e = sm_slots | 1u;
  if (leg.nreg == 6) {
    e = std::max<uint32_t>(sm_slots, 2u);
    if ((e / 2) % 2 == 0) e += 2;
  }
  const size_t lb = align16((size_t)p->n_blocks * p->z * 4);
  const size_t mb = align16((size_t)p->z * e * 4);
  if (smem_for(1, lb, mb) > smem_max) return leg;
  Shape sh = leg;
  sh.tm = true;
  sh.occ = 0;
  sh.refill_occ = 0;
  sh.smem = std::max(smem_for(1, lb, mb), one_per_sm);
  sh.kp.l_bytes = (uint32_t)lb;
  sh.kp.m_bytes = (uint32_t)mb;
  sh.kp.m_stride = e * 4u;
  sh.kp.tm_cols = tm_cols;
  sh.kp.tm_slot = slot;
  sh.kp.tm_r45[0] = r45[0];
  sh.kp.tm_r45[1] = r45[1];
  build_units(p, leg.nreg, ml, sh.kp);
  for (int t = 0; t < NR_MAX_TAB; ++t) {
    sh.kp.sh[t] = b.sh[t] * 4u;
    sh.kp.cb[t] = b.cb[t] * (uint32_t)p->z * 4u + sh.kp.abs_base;
  }
  return sh;
}

}  // namespace

// Persistent lane-refill launch (early-stop modes, single-group pair shapes):
// one CTA per resident slot, each refilling its lanes from a per-launch
// codeword counter.
template <int BG, int MAXW, int NREG, bool TM = false>
static cudaError_t launch_refill(Shape& sh, int device, const int8_t* llr, long long batch, const KOut& o,
                                 cudaStream_t st) {
  static bool attr_done[64] = {};
  static int sms[64] = {};
  auto kern = k_decode_i8_refill<BG, MAXW, NREG, TM>;
  const int d = device & 63;
  if (!attr_done[d]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    attr_done[d] = true;
  }
  // occupancy depends on this shape's threads and shared memory (one
  // instantiation serves several Z / rows_used): cached in the Shape, set at
  // plan creation (the llr == nullptr call)
  if (!sh.refill_occ) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sh.threads, sh.smem);
    if (e != cudaSuccess) return e;
    sh.refill_occ = occ > 0 ? occ : 1;
  }
  if (!llr) return cudaSuccess;
  KParams kp = sh.kp;
  kp.batch = batch;
  kp.trace = 0;
  kp.vec_load = ((long long)kp.n_blocks * kp.z) % 16 == 0 && ((uintptr_t)llr & 15) == 0;
  const long long pairs = (batch + 1) / 2;
  const long long grid = std::min<long long>(pairs, (long long)sh.refill_occ * sms[d]);
  int32_t* work = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&work), sizeof(int32_t), device, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e == cudaSuccess) {
    KOut oo = o;
    oo.work = work;
    kern<<<(unsigned)grid, sh.threads, sh.smem, st>>>(kp, llr, oo);
    ++g_launches;
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(work, st);
  return e != cudaSuccess ? e : f;
}

static cudaError_t launch_shape(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch,
                                const KOut& o, cudaStream_t st) {
  if (sh.threads == 0) return cudaErrorInvalidConfiguration;  // no feasible shape
  const bool two = sh.lanes == 2;
  const int dev = plan->device;
  // early-stop modes without a trace: refill lanes as codewords stop
  const bool refill = plan->early_stop != NRLDPC_STOP_NONE && o.trace_w == nullptr && sh.abs && two &&
                      sh.groups == 1 && plan->z % 32 == 0 && !getenv("NRLDPC_NO_REFILL");
  if (refill && (in == nullptr || batch > 2)) {
    cudaError_t e = cudaSuccess;
    if (sh.tm && sh.nreg == 6) e = launch_refill<1, 19, 6, true>(sh, dev, in, batch, o, st);
    else if (sh.tm && plan->schedule == 1) e = launch_refill<1, 19, 0, true>(sh, dev, in, batch, o, st);
    else if (sh.tm) e = launch_refill<2, 10, 0, true>(sh, dev, in, batch, o, st);
    else if (plan->schedule == 1 && sh.nreg == 6) e = launch_refill<1, 19, 6>(sh, dev, in, batch, o, st);
    else if (plan->schedule == 1 && sh.nreg == 0) e = launch_refill<1, 19, 0>(sh, dev, in, batch, o, st);
    else if (plan->schedule == 2 && sh.nreg == 0) e = launch_refill<2, 10, 0>(sh, dev, in, batch, o, st);
    else goto plain;
    if (in != nullptr || e != cudaSuccess) return e;
  }
plain:
  if (sh.tm) {
    if (sh.nreg == 6) return launch_i8<1, 19, 2, 6, true, true>(sh, dev, in, batch, o, st);
    if (plan->schedule == 1) return launch_i8<1, 19, 2, 0, true, true>(sh, dev, in, batch, o, st);
    return launch_i8<2, 10, 2, 0, true, true>(sh, dev, in, batch, o, st);
  }
  switch (plan->schedule) {
    case 1:
      if (!two) return launch_i8<1, 19, 1>(sh, dev, in, batch, o, st);
      if (sh.nreg == 0)
        return sh.abs ? launch_i8<1, 19, 2, 0, true>(sh, dev, in, batch, o, st)
                      : launch_i8<1, 19, 2>(sh, dev, in, batch, o, st);
      if (!sh.abs) return cudaErrorInvalidConfiguration;
      if (sh.nreg == 2) return launch_i8<1, 19, 2, 2, true>(sh, dev, in, batch, o, st);
      if (sh.nreg == 4) return launch_i8<1, 19, 2, 4, true>(sh, dev, in, batch, o, st);
      return launch_i8<1, 19, 2, 6, true>(sh, dev, in, batch, o, st);
    case 2:
      if (!two) return launch_i8<2, 10, 1>(sh, dev, in, batch, o, st);
      return sh.abs ? launch_i8<2, 10, 2, 0, true>(sh, dev, in, batch, o, st)
                    : launch_i8<2, 10, 2>(sh, dev, in, batch, o, st);
    default:
      if (plan->maxw > 10)
        return two ? launch_i8<0, 19, 2>(sh, dev, in, batch, o, st) : launch_i8<0, 19, 1>(sh, dev, in, batch, o, st);
      return two ? launch_i8<0, 10, 2>(sh, dev, in, batch, o, st) : launch_i8<0, 10, 1>(sh, dev, in, batch, o, st);
  }
}

template <int PREC, int BG, bool FTM = false>
static cudaError_t launch_float_bg(Shape& sh, int device, const void* llr, long long batch, const KOut& o,
                                cudaStream_t st) {
  static bool attr_done[64] = {};
  auto kern = k_decode_flt<PREC, BG, FTM>;
  if (!attr_done[device & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    attr_done[device & 63] = true;
  }
  if (!sh.occ) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sh.threads, sh.smem);
    if (e != cudaSuccess) return e;
    sh.occ = occ > 0 ? occ : 1;
  }
  if (!llr) return cudaSuccess;
  KParams kp = sh.kp;
  kp.batch = batch;
  kp.trace = o.trace_w != nullptr;
  const long long per_cta = (long long)sh.groups * sh.lanes;
  const long long grid = (batch + per_cta - 1) / per_cta;
  // messages: stream-ordered workspace, [group][edge][z] x 4 bytes (FTM:
  // only the rows kept in global memory)
  uint32_t* ws = nullptr;
  const size_t ws_bytes = std::max<size_t>(16, (size_t)grid * sh.groups * (FTM ? kp.e_reg : kp.n_edges) * kp.z * 4);
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&ws), ws_bytes, device, st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, sh.threads, sh.smem, st>>>(kp, llr, ws, o);
  ++g_launches;
  e = cudaGetLastError();
  const cudaError_t f = cudaFreeAsync(ws, st);
  return e != cudaSuccess ? e : f;
}

// compile-time row bodies for the BG1/BG2 schedules, generic loop otherwise
template <int PREC>
static cudaError_t launch_float(int schedule, Shape& sh, int device, const void* llr, long long batch,
                                const KOut& o, cudaStream_t st) {
  if (schedule == 1) return sh.tm ? launch_float_bg<PREC, 1, true>(sh, device, llr, batch, o, st)
                                  : launch_float_bg<PREC, 1>(sh, device, llr, batch, o, st);
  if (schedule == 2) return sh.tm ? launch_float_bg<PREC, 2, true>(sh, device, llr, batch, o, st)
                                  : launch_float_bg<PREC, 2>(sh, device, llr, batch, o, st);
  return launch_float_bg<PREC, 0>(sh, device, llr, batch, o, st);
}

// ---- host worker pool -------------------------------------------------------
// A few persistent threads for the host side of the end-to-end path: copying
// a pageable caller's input into pinned staging memory, and unpacking packed
// hard decisions into the reference's (B, K) byte layout. One copy thread
// moves ~10 GB/s; the pool splits each chunk so the host copy keeps ahead
// of the PCIe DMA it feeds. NRLDPC_HOST_THREADS overrides the size.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return (int)workers_.size() + 1; }
  // f(i) for i in [0, n): the caller runs tasks too; returns when all done
  void run(int n, const std::function<void(int)>& f) {
    if (n <= 0) return;
    if (n == 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      n_ = n;
      next_.store(0);
      left_.store(n);
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return left_.load() == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = std::getenv("NRLDPC_HOST_THREADS")) n = std::atoi(e);
    n = std::max(1, std::min(n, 8));
    for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) return;
      (*job_)(i);
      if (left_.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (!job_) continue;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0}, left_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

static void host_copy(void* dst, const void* src, size_t n) {
  constexpr size_t kPiece = 1u << 20;
  HostPool& pool = HostPool::get();
  const int parts = (int)std::min<size_t>((size_t)pool.size(), (n + kPiece - 1) / kPiece);
  if (parts <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t per = ((n + parts - 1) / parts + 4095) & ~size_t(4095);
  pool.run(parts, [&](int i) {
    const size_t o = (size_t)i * per;
    if (o < n) std::memcpy(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o, std::min(per, n - o));
  });
}

static bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

static cudaError_t grow_pinned(uint8_t*& buf, size_t& cap, size_t need) {
  if (need <= cap) return cudaSuccess;
  if (buf) cudaFreeHost(buf);
  buf = nullptr;
  cap = 0;
  const cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&buf), need);
  if (e == cudaSuccess) cap = need;
  return e;
}

extern "C" {

const char* nrldpc_last_error(void) { return g_last_error.c_str(); }

int nrldpc_beta_rule(double beta, int* mode, float* beta_h, float* delta, float* c) {
  KParams kp{};
  find_beta_arith(beta, &kp);
  if (mode) *mode = kp.beta_mode;
  if (kp.beta_mode) {
    __half h;
    uint16_t u = (uint16_t)(kp.beta_h & 0xFFFF);
    std::memcpy(&h, &u, 2);
    if (beta_h) *beta_h = __half2float(h);
    u = (uint16_t)(kp.ndelta_h & 0xFFFF);
    std::memcpy(&h, &u, 2);
    if (delta) *delta = -__half2float(h);
    u = (uint16_t)(kp.c_h & 0xFFFF);
    std::memcpy(&h, &u, 2);
    if (c) *c = __half2float(h);
  }
  return NRLDPC_OK;
}

int nrldpc_decode_flooding(nrldpc_plan* plan, const void* llr, int64_t batch, uint32_t* bits,
                           int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok,
                           int32_t* trace_w, float* trace_m, int32_t* status, void* stream) {
  g_launches = 0;
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (batch < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
  if (batch == 0) return NRLDPC_OK;
  if (!llr || !bits || !iters || !synd || !success) return fail(NRLDPC_EINVAL, "NULL buffer");
  if ((trace_w == nullptr) != (trace_m == nullptr))
    return fail(NRLDPC_EINVAL, "trace_w and trace_m must both be set or both NULL");
  if (plan->early_stop == NRLDPC_STOP_CRC && !crc_ok)
    return fail(NRLDPC_EINVAL, "crc mode needs a crc_ok buffer");
  NR_CUDA(cudaSetDevice(plan->device));
  cudaStream_t st = (cudaStream_t)stream;
  KParams kp = plan->base;
  kp.batch = batch;
  kp.trace = trace_w != nullptr;
  if (plan->precision == NRLDPC_F32) {
    const float bf = (float)plan->beta;
    std::memcpy(&kp.beta_f, &bf, 4);
  } else if (plan->precision == NRLDPC_F16) {
    const __half bh = __double2half(plan->beta);
    uint16_t u;
    std::memcpy(&u, &bh, 2);
    kp.beta_f = (uint32_t)u * 0x10001u;
  }
  const size_t n_c = (size_t)plan->n_blocks * plan->z;
  const size_t smem = 2 * n_c * 4;
  const int threads = (plan->z + 31) / 32 * 32;
  void* ws = nullptr;
  NR_CUDA(scratch_alloc(&ws, (size_t)batch * plan->n_edges * plan->z * 4, plan->device, st));
  KOut o{bits, iters, synd, success, crc_ok, trace_w, trace_m, status};
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)batch, threads, smem, st>>>(kp, plan->flood, llr, ws, o);
    return cudaGetLastError();
  };
  cudaError_t e = plan->precision == NRLDPC_INT8  ? go(k_decode_flood<NRLDPC_INT8>)
                  : plan->precision == NRLDPC_F32 ? go(k_decode_flood<NRLDPC_F32>)
                                                  : go(k_decode_flood<NRLDPC_F16>);
  ++g_launches;
  const cudaError_t f = cudaFreeAsync(ws, st);
  if (e != cudaSuccess) return cuda_fail(e, "flooding decode launch");
  if (f != cudaSuccess) return cuda_fail(f, "workspace free");
  return NRLDPC_OK;
}

int nrldpc_encode(const nrldpc_plan* plan, const uint8_t* msgs, int64_t batch, uint8_t* out,
                  void* stream) {
  g_launches = 0;
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (!plan->enc_ok) return fail(NRLDPC_EINVAL, "graph does not have the systematic-encoder structure");
  if (batch < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
  if (batch == 0) return NRLDPC_OK;
  if (!msgs || !out) return fail(NRLDPC_EINVAL, "NULL buffer");
  NR_CUDA(cudaSetDevice(plan->device));
  const int threads = (plan->z + 31) / 32 * 32;
  const size_t smem = (size_t)(plan->n_blocks + 4) * plan->z;
  k_encode<<<(unsigned)batch, threads, smem, (cudaStream_t)stream>>>(plan->base, plan->enc, msgs, batch, out);
  ++g_launches;
  NR_CUDA(cudaGetLastError());
  return NRLDPC_OK;
}

int nrldpc_channel_awgn(const nrldpc_plan* plan, const uint8_t* bits, int64_t batch, double sigma,
                        double scale, uint64_t seed, int8_t* out, void* stream) {
  g_launches = 0;
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (!(sigma > 0.0)) return fail(NRLDPC_EINVAL, "sigma must be positive");
  if (!(scale > 0.0)) return fail(NRLDPC_EINVAL, "scale must be positive");
  if (batch < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
  if (batch == 0) return NRLDPC_OK;
  if (!bits || !out) return fail(NRLDPC_EINVAL, "NULL buffer");
  NR_CUDA(cudaSetDevice(plan->device));
  const int n_c = plan->n_blocks * plan->z;
  const long long total = batch * (long long)n_c;
  const int grid = (int)std::min<long long>((total + 1023) / 1024, 148LL * 16);
  k_channel_awgn<<<grid, 256, 0, (cudaStream_t)stream>>>(bits, batch, n_c, 2 * plan->z, sigma, scale,
                                                         (unsigned long long)seed, out);
  ++g_launches;
  NR_CUDA(cudaGetLastError());
  return NRLDPC_OK;
}

int nrldpc_alu_peak(int device, double* alu_lane_ops_per_s, double* mixed_lane_ops_per_s) {
  NR_CUDA(cudaSetDevice(device));
  int sms = 0;
  NR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  uint32_t* d_out = nullptr;
  NR_CUDA(cudaMalloc(&d_out, 16));
  cudaEvent_t e0, e1;
  NR_CUDA(cudaEventCreate(&e0));
  NR_CUDA(cudaEventCreate(&e1));
  const int threads = 512, blocks = sms * 4, iters = 4096;
  double res[2] = {0, 0};
  for (int mixed = 0; mixed < 2; ++mixed) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      NR_CUDA(cudaEventRecord(e0));
      if (mixed) k_alu_peak<true><<<blocks, threads>>>(d_out, iters, 0x1234u + rep);
      else k_alu_peak<false><<<blocks, threads>>>(d_out, iters, 0x1234u + rep);
      NR_CUDA(cudaEventRecord(e1));
      NR_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      NR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0) best = std::min(best, ms);
    }
    // two half2 instructions per chain step, 8 chains, iters steps, per thread
    const double lane_ops = 2.0 * 8.0 * iters * (double)threads * blocks;
    res[mixed] = lane_ops / (best * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_out);
  if (alu_lane_ops_per_s) *alu_lane_ops_per_s = res[0];
  if (mixed_lane_ops_per_s) *mixed_lane_ops_per_s = res[1];
  return NRLDPC_OK;
}

int nrldpc_launch_count(void) { return g_launches; }

int nrldpc_unpack_bits(const uint32_t* words, int64_t batch, int64_t words_per_cw, int64_t k, uint8_t* out) {
  if (batch < 0 || k < 0 || words_per_cw * 32 < k) return fail(NRLDPC_EINVAL, "bad unpack shape");
  if (batch == 0 || k == 0) return NRLDPC_OK;
  if (!words || !out) return fail(NRLDPC_EINVAL, "NULL buffer");
  // byte b of a packed word -> 8 output bytes 0/1, LSB first
  static const auto lut = [] {
    std::vector<uint64_t> t(256);
    for (int b = 0; b < 256; ++b) {
      uint64_t v = 0;
      for (int i = 0; i < 8; ++i) v |= (uint64_t)((b >> i) & 1) << (8 * i);
      t[b] = v;
    }
    return t;
  }();
  HostPool& pool = HostPool::get();
  const int64_t per = std::max<int64_t>(1, (batch + 4 * pool.size() - 1) / (4 * pool.size()));
  const int parts = (int)((batch + per - 1) / per);
  pool.run(parts, [&](int part) {
    const int64_t c0 = part * per, c1 = std::min(batch, c0 + per);
    for (int64_t c = c0; c < c1; ++c) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(words + c * words_per_cw);
      uint8_t* dst = out + c * k;
      const int64_t full = k / 8;
      for (int64_t i = 0; i < full; ++i) std::memcpy(dst + 8 * i, &lut[src[i]], 8);
      for (int64_t i = full * 8; i < k; ++i) dst[i] = (src[i >> 3] >> (i & 7)) & 1u;
    }
  });
  return NRLDPC_OK;
}

int nrldpc_plan_create(int device, int k_b, int z, int rows_used, const int32_t* row_start,
                       const int16_t* cols, const int16_t* shifts, int precision, double beta,
                       int max_iter, int early_stop, int crc_kind, nrldpc_plan** out) {
  if (!out) return fail(NRLDPC_EINVAL, "out is NULL");
  *out = nullptr;
  if (!row_start || !cols || !shifts) return fail(NRLDPC_EINVAL, "graph tables are NULL");
  if (z < 2 || z > 384) return fail(NRLDPC_EINVAL, "Z must be in [2, 384]");
  if (k_b != 22 && k_b != 10) return fail(NRLDPC_EINVAL, "k_b must be 22 (BG1) or 10 (BG2)");
  if (rows_used < 4 || rows_used > NR_MAX_ROWS)
    return fail(NRLDPC_EINVAL, "rows_used must be in [4, 46]");
  if (!(beta > 0.0 && beta <= 1.0)) return fail(NRLDPC_EINVAL, "beta must be in (0, 1]");
  if (max_iter < 1) return fail(NRLDPC_EINVAL, "max_iter must be at least 1");
  if (precision != NRLDPC_INT8 && precision != NRLDPC_F16 && precision != NRLDPC_F32)
    return fail(NRLDPC_EINVAL, "unknown precision");
  if (early_stop < NRLDPC_STOP_SYNDROME || early_stop > NRLDPC_STOP_NONE)
    return fail(NRLDPC_EINVAL, "unknown early_stop mode");
  int crc_len = 0;
  uint32_t crc_poly = 0;
  if (crc_params(crc_kind, &crc_len, &crc_poly) != 0) return fail(NRLDPC_EINVAL, "unknown crc kind");
  const int n_edges = row_start[rows_used];
  if (row_start[0] != 0 || n_edges <= 0 || n_edges > NR_MAX_EDGES)
    return fail(NRLDPC_EINVAL, "bad row_start table");
  const int n_blocks = k_b + rows_used;
  int maxw = 0;
  for (int r = 0; r < rows_used; ++r) {
    const int w = row_start[r + 1] - row_start[r];
    if (w < 2 || w > 19) return fail(NRLDPC_EINVAL, "row weight must be in [2, 19]");
    maxw = std::max(maxw, w);
  }
  for (int e = 0; e < n_edges; ++e) {
    if (cols[e] < 0 || cols[e] >= n_blocks) return fail(NRLDPC_EINVAL, "edge column out of range");
    if (shifts[e] < 0 || shifts[e] >= z) return fail(NRLDPC_EINVAL, "edge shift must be in [0, Z)");
  }
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(NRLDPC_EINVAL, "device index out of range");

  nrldpc_plan* p = new (std::nothrow) nrldpc_plan();
  if (!p) return fail(NRLDPC_ENOMEM, "plan allocation failed");
  p->device = device;
  p->precision = precision;
  p->early_stop = early_stop;
  p->crc_kind = crc_kind;
  p->beta = beta;
  p->max_iter = max_iter;
  p->k_b = k_b;
  p->z = z;
  p->rows = rows_used;
  p->n_blocks = n_blocks;
  p->n_edges = n_edges;
  p->maxw = maxw;
  KParams& kp = p->base;
  std::memset(&kp, 0, sizeof(kp));
  kp.z = z;
  kp.k_b = k_b;
  kp.rows = rows_used;
  kp.n_blocks = n_blocks;
  kp.n_edges = n_edges;
  kp.max_iter = max_iter;
  kp.early_stop = early_stop;
  kp.crc_len = crc_len;
  kp.crc_poly = crc_poly;
  kp.words = (k_b * z + 31) / 32;
  for (int r = 0; r <= rows_used; ++r) kp.row_start[r] = (uint16_t)row_start[r];
  {
    int t = 0;
    for (int r = 0; r < rows_used; ++r) {
      kp.tab_start[r] = (uint16_t)t;
      for (int e = row_start[r]; e < row_start[r + 1]; ++e, ++t) {
        kp.sh[t] = (uint32_t)shifts[e];
        kp.cb[t] = (uint32_t)cols[e];
      }
      t = (t + 3) & ~3;
    }
    kp.tab_start[rows_used] = (uint16_t)t;
  }
  // layers: a barrier after row r unless row r+1 shares no column with any
  // row since the last barrier (then r+1 can run concurrently with them).
  // Rows 0..5 keep their barriers (register-message rows are straight-line).
  {
    std::bitset<NR_MAX_BLOCKS> layer_cols;
    for (int r = 0; r < rows_used; ++r) {
      for (int e = row_start[r]; e < row_start[r + 1]; ++e) layer_cols.set(cols[e]);
      std::bitset<NR_MAX_BLOCKS> next;
      if (r + 1 < rows_used)
        for (int e = row_start[r + 1]; e < row_start[r + 2]; ++e) next.set(cols[e]);
      const bool disjoint = r + 1 < rows_used && r >= 6 && (next & layer_cols).none();
      kp.bar_after[r] = disjoint ? 0 : 1;
      if (!disjoint) layer_cols.reset();
    }
  }
  // int8 beta rule: floor(beta * m) computed in float64 (decoder.py:208-212)
  for (int m = 0; m < 128; ++m) kp.lut[m] = float_to_half_bits((float)std::floor(beta * (double)m));
  find_beta_arith(beta, &kp);
  p->schedule = 0;
  for (int bg = 1; bg <= 2; ++bg) {
    const int kb_bg = bg == 1 ? 22 : 10;
    const int nrows = bg == 1 ? RowW<1>::n : RowW<2>::n;
    if (k_b != kb_bg || rows_used > nrows) continue;
    bool same = true;
    for (int r = 0; r <= rows_used && same; ++r)
      same = row_start[r] == (bg == 1 ? RowW<1>::e0[r] : RowW<2>::e0[r]);
    // the compile-time schedules carry only the arithmetic beta rule; a
    // table-only beta decodes on the generic schedule
    if (same && kp.beta_mode) p->schedule = bg;
  }
  // flooding: per column, its edges in row order (decoder.py:362-364)
  {
    int k = 0;
    for (int c = 0; c < n_blocks; ++c) {
      p->flood.col_start[c] = (uint16_t)k;
      for (int e = 0; e < n_edges; ++e)
        if (cols[e] == c) {
          p->flood.col_edge[k] = (uint16_t)e;
          p->flood.col_shift[k] = (uint16_t)shifts[e];
          ++k;
        }
    }
    p->flood.col_start[n_blocks] = (uint16_t)k;
  }
  // systematic-encoder schedule (basegraph.py:175-207, codec.py:85-125)
  {
    const int p0 = k_b;
    std::vector<int> core[4];
    bool ok = true;
    for (int r = 0; r < 4 && ok; ++r)
      for (int e = row_start[r]; e < row_start[r + 1]; ++e)
        if (cols[e] >= p0 && cols[e] < p0 + 4) core[cols[e] - p0].push_back(shifts[e]);
        else if (cols[e] >= p0 + 4) ok = false;
    for (int c = 1; c < 4 && ok; ++c) {
      if (core[c].size() % 2) ok = false;
      for (int v : core[c]) ok = ok && v == core[c][0];
    }
    // the shift value occurring an odd number of times at p0 (exactly one)
    int odd = -1, n_odd = 0;
    for (size_t i = 0; i < core[0].size(); ++i) {
      bool first = true;
      for (size_t k = 0; k < i; ++k) first = first && core[0][k] != core[0][i];
      if (!first) continue;
      int cnt = 0;
      for (int u : core[0]) cnt += (u == core[0][i]);
      if (cnt % 2) {
        odd = core[0][i];
        ++n_odd;
      }
    }
    ok = ok && n_odd == 1;
    EncSched es{};
    es.css = odd;
    bool known[4] = {true, false, false, false};
    std::vector<int> pending = {0, 1, 2, 3};
    while (ok && !pending.empty()) {
      bool progressed = false;
      for (size_t i = 0; i < pending.size(); ++i) {
        const int r = pending[i];
        int n_unknown = 0, uc = -1, us = 0;
        for (int e = row_start[r]; e < row_start[r + 1]; ++e)
          if (cols[e] >= p0 && !known[cols[e] - p0]) ++n_unknown, uc = cols[e], us = shifts[e];
        if (n_unknown > 1) continue;
        if (n_unknown == 1) {
          es.row[es.nsteps] = r;
          es.col[es.nsteps] = uc;
          es.shift[es.nsteps] = us;
          ++es.nsteps;
          known[uc - p0] = true;
        }
        pending.erase(pending.begin() + i);
        progressed = true;
        break;
      }
      if (!progressed) ok = false;
    }
    for (int r = 4; r < rows_used && ok; ++r) {
      int own = 0;
      for (int e = row_start[r]; e < row_start[r + 1]; ++e)
        if (cols[e] == p0 + r) own += shifts[e] == 0 ? 1 : 100;
        else if (cols[e] >= p0 + 4) own += 100;
      ok = own == 1;
    }
    p->enc = es;
    p->enc_ok = ok;
  }
  if (early_stop == NRLDPC_STOP_CRC && k_b * z >= crc_len) {
    // rem(x^(K-1-i+L), g) for i = K-1 down to 0: start at x^L mod g = poly
    const int K = k_b * z;
    std::vector<uint32_t> tab(K);
    const uint32_t mask = (crc_len == 32) ? 0xFFFFFFFFu : ((1u << crc_len) - 1u);
    uint32_t r = crc_poly & mask;
    for (int i = K - 1; i >= 0; --i) {
      tab[i] = r;
      const bool top = (r >> (crc_len - 1)) & 1u;
      r = ((r << 1) & mask) ^ (top ? crc_poly : 0u);
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    ce = cudaMalloc(&p->d_crc_tab, sizeof(uint32_t) * K);
    if (ce == cudaSuccess)
      ce = cudaMemcpy(p->d_crc_tab, tab.data(), sizeof(uint32_t) * K, cudaMemcpyHostToDevice);
    cudaSetDevice(prev);
    if (ce != cudaSuccess) {
      if (p->d_crc_tab) cudaFree(p->d_crc_tab);
      delete p;
      return cuda_fail(ce, "crc table");
    }
    p->base.crc_tab = p->d_crc_tab;
  }
  const char* force = std::getenv("NRLDPC_FORCE_LANES");
  if (precision == NRLDPC_INT8) {
    p->main = choose_shape(p, force && force[0] == '1' ? 1 : 2);
    p->main = tm_shape(p, p->main);
  } else {
    p->main = choose_shape_float(p);
    if (p->schedule != 0) {
      // layer units with messages addressed by edge index ([edge][z]
      // workspace), or by their on-chip slots
      MsgLayout ml{};
      if (!ftm_layout(p, p->main, ml))
        for (int r = 0; r < p->rows; ++r) ml.mb[r] = (uint32_t)p->base.row_start[r];
      build_units(p, 0, ml, p->main.kp);
    }
    if (precision == NRLDPC_F32) {
      const float bf = (float)beta;  // np.float32(beta)
      std::memcpy(&p->main.kp.beta_f, &bf, 4);
    } else {
      const __half bh = __double2half(beta);  // np.float16(beta): one RNE rounding
      uint16_t u;
      std::memcpy(&u, &bh, 2);
      p->main.kp.beta_f = (uint32_t)u * 0x10001u;
    }
  }
  // set kernel attributes and cache occupancy now, so decode never mutates
  // the plan (concurrent decodes on one plan are then race-free)
  {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    KOut none{};
    const cudaError_t e1 =
        precision == NRLDPC_INT8 ? launch_shape(p, p->main, nullptr, 0, none, nullptr)
        : precision == NRLDPC_F32 ? launch_float<NRLDPC_F32>(p->schedule, p->main, device, nullptr, 0, none, nullptr)
                                  : launch_float<NRLDPC_F16>(p->schedule, p->main, device, nullptr, 0, none, nullptr);
    cudaSetDevice(prev);
    if (e1 != cudaSuccess) {
      delete p;
      return cuda_fail(e1, "kernel setup");
    }
  }
  *out = p;
  return NRLDPC_OK;
}

int nrldpc_plan_set_coscheduled(nrldpc_plan* plan, int on) {
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (plan->precision != NRLDPC_INT8 || plan->coscheduled == (on != 0)) return NRLDPC_OK;
  plan->coscheduled = on != 0;
  const char* force = std::getenv("NRLDPC_FORCE_LANES");
  Shape sh = tm_shape(plan, choose_shape(plan, force && force[0] == '1' ? 1 : 2));
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  KOut none{};
  const cudaError_t e = launch_shape(plan, sh, nullptr, 0, none, nullptr);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, "kernel setup");
  plan->main = sh;
  return NRLDPC_OK;
}

int nrldpc_plan_destroy(nrldpc_plan* plan) {
  if (!plan) return NRLDPC_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  for (auto& s : plan->streams)
    if (s) cudaStreamDestroy(s);
  for (auto& e : plan->chunk_ev) cudaEventDestroy(e);
  for (auto& sl : plan->slot) {
    if (sl.done) cudaEventSynchronize(sl.done), cudaEventDestroy(sl.done);
    if (sl.d_buf) cudaFree(sl.d_buf);
    if (sl.h_status) cudaFreeHost(sl.h_status);
    if (sl.h_in) cudaFreeHost(sl.h_in);
    if (sl.h_out) cudaFreeHost(sl.h_out);
  }
  if (plan->d_crc_tab) cudaFree(plan->d_crc_tab);
  cudaSetDevice(prev);
  delete plan;
  return NRLDPC_OK;
}

int nrldpc_plan_info(const nrldpc_plan* plan, int64_t* k, int64_t* n_c, int64_t* n_tx,
                     int64_t* words_per_cw, int* lanes, int* groups_per_cta, int* threads_per_cta,
                     int64_t* smem_bytes) {
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (k) *k = (int64_t)plan->k_b * plan->z;
  if (n_c) *n_c = (int64_t)plan->n_blocks * plan->z;
  if (n_tx) *n_tx = (int64_t)(plan->n_blocks - 2) * plan->z;
  if (words_per_cw) *words_per_cw = plan->base.words;
  if (lanes) *lanes = plan->main.lanes;
  if (groups_per_cta) *groups_per_cta = plan->main.groups;
  if (threads_per_cta) *threads_per_cta = plan->main.threads;
  if (smem_bytes) *smem_bytes = (int64_t)plan->main.smem;
  return NRLDPC_OK;
}

static int quantize_impl(const nrldpc_plan* plan, const void* llr_in, int in_dtype, int64_t batch,
                         double scale, double clip, void* out, int out_mode, void* stream, bool demap,
                         double sigma) {
  g_launches = 0;
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (batch < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
  if (!(scale > 0.0)) return fail(NRLDPC_EINVAL, "scale must be positive");
  if (demap && !(sigma > 0.0)) return fail(NRLDPC_EINVAL, "sigma must be positive");
  if (batch == 0) return NRLDPC_OK;
  if (!llr_in || !out) return fail(NRLDPC_EINVAL, "NULL buffer");
  const int n_c = plan->n_blocks * plan->z;
  const int n_tx = n_c - 2 * plan->z;
  cudaStream_t st = (cudaStream_t)stream;
  NR_CUDA(cudaSetDevice(plan->device));
  const double sigma2 = sigma * sigma;
  // row-vector path: 16-byte aligned input rows (and int8 output rows of at
  // least 4-byte alignment: vec 1 = two 32-bit stores, 2 = one 64-bit store)
  const size_t in_bytes = in_dtype == NRLDPC_IN_F64 ? 8 : 4;
  const bool in_ok = ((size_t)n_tx * in_bytes) % 16 == 0 && ((size_t)2 * plan->z * in_bytes) % 16 == 0 &&
                     ((uintptr_t)llr_in & 15) == 0;
  int vec = 0;
  if (in_ok) {
    if (out_mode != NRLDPC_INT8) vec = 1;
    else if (n_c % 8 == 0 && ((uintptr_t)out & 7) == 0) vec = 2;
    else if (n_c % 4 == 0 && ((uintptr_t)out & 3) == 0) vec = 1;
  }
  const dim3 grid((unsigned)((n_c + 8 * 256 - 1) / (8 * 256)), (unsigned)std::min<int64_t>(batch, 65535));
  auto go = [&](auto k_plain, auto k_demap, auto* typed_in) {
    if (demap)
      k_demap<<<grid, 256, 0, st>>>(typed_in, (long long)batch, n_tx, n_c, 2 * plan->z, scale, clip, out, sigma2, vec);
    else
      k_plain<<<grid, 256, 0, st>>>(typed_in, (long long)batch, n_tx, n_c, 2 * plan->z, scale, clip, out, 1.0, vec);
  };
  if (in_dtype == NRLDPC_IN_F64) {
    const double* in = static_cast<const double*>(llr_in);
    if (out_mode == NRLDPC_INT8) go(k_quantize<double, NRLDPC_INT8, false>, k_quantize<double, NRLDPC_INT8, true>, in);
    else if (out_mode == NRLDPC_F16) go(k_quantize<double, NRLDPC_F16, false>, k_quantize<double, NRLDPC_F16, true>, in);
    else if (out_mode == NRLDPC_F32) go(k_quantize<double, NRLDPC_F32, false>, k_quantize<double, NRLDPC_F32, true>, in);
    else return fail(NRLDPC_EINVAL, "unknown quantize out_mode");
  } else if (in_dtype == NRLDPC_IN_F32) {
    const float* in = static_cast<const float*>(llr_in);
    if (out_mode == NRLDPC_INT8) go(k_quantize<float, NRLDPC_INT8, false>, k_quantize<float, NRLDPC_INT8, true>, in);
    else if (out_mode == NRLDPC_F16) go(k_quantize<float, NRLDPC_F16, false>, k_quantize<float, NRLDPC_F16, true>, in);
    else if (out_mode == NRLDPC_F32) go(k_quantize<float, NRLDPC_F32, false>, k_quantize<float, NRLDPC_F32, true>, in);
    else return fail(NRLDPC_EINVAL, "unknown quantize out_mode");
  } else {
    return fail(NRLDPC_EINVAL, "unknown quantize input dtype");
  }
  ++g_launches;
  NR_CUDA(cudaGetLastError());
  return NRLDPC_OK;
}

int nrldpc_quantize(const nrldpc_plan* plan, const void* llr_in, int in_dtype, int64_t batch,
                    double scale, double clip, void* out, int out_mode, void* stream) {
  return quantize_impl(plan, llr_in, in_dtype, batch, scale, clip, out, out_mode, stream, false, 1.0);
}

int nrldpc_demap_quantize(const nrldpc_plan* plan, const void* symbols, int in_dtype, int64_t batch,
                          double sigma, double scale, double clip, void* out, int out_mode,
                          void* stream) {
  return quantize_impl(plan, symbols, in_dtype, batch, scale, clip, out, out_mode, stream, true, sigma);
}

static int decode_impl(nrldpc_plan* plan, const void* llr, int64_t batch, const KOut& o,
                       cudaStream_t st) {
  if (plan->precision != NRLDPC_INT8) {
    const cudaError_t e = plan->precision == NRLDPC_F32
                              ? launch_float<NRLDPC_F32>(plan->schedule, plan->main, plan->device, llr, batch, o, st)
                              : launch_float<NRLDPC_F16>(plan->schedule, plan->main, plan->device, llr, batch, o, st);
    if (e != cudaSuccess) return cuda_fail(e, "decode launch");
    return NRLDPC_OK;
  }
  const cudaError_t e = launch_shape(plan, plan->main, static_cast<const int8_t*>(llr), batch, o, st);
  if (e != cudaSuccess) return cuda_fail(e, "decode launch");
  return NRLDPC_OK;
}

int nrldpc_decode(nrldpc_plan* plan, const void* llr, int64_t batch, uint32_t* bits,
                  int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok, int32_t* trace_w,
                  float* trace_m, int32_t* status, void* stream) {
  g_launches = 0;
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (batch < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
  if (batch == 0) return NRLDPC_OK;
  if (!llr || !bits || !iters || !synd || !success) return fail(NRLDPC_EINVAL, "NULL buffer");
  if ((trace_w == nullptr) != (trace_m == nullptr))
    return fail(NRLDPC_EINVAL, "trace_w and trace_m must both be set or both NULL");
  if (plan->early_stop == NRLDPC_STOP_CRC && !crc_ok)
    return fail(NRLDPC_EINVAL, "crc mode needs a crc_ok buffer");
  NR_CUDA(cudaSetDevice(plan->device));
  KOut o{bits, iters, synd, success, crc_ok, trace_w, trace_m, status};
  return decode_impl(plan, llr, batch, o, (cudaStream_t)stream);
}

// Enqueue one host-buffer decode into slot `si` (caller holds host_mu and has
// retired the slot's previous call). Returns the number of decode launches
// through *launches.
static int host_enqueue(nrldpc_plan* plan, int si, const void* llr_host, int64_t batch, uint32_t* bits,
                        int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok, int chunks,
                        int* launches_out) {
  auto& sl = plan->slot[si];
  const size_t esz = plan->precision == NRLDPC_INT8 ? 1 : (plan->precision == NRLDPC_F16 ? 2 : 4);
  const size_t n_c = (size_t)plan->n_blocks * plan->z;
  const size_t words = plan->base.words;
  const size_t per_cw_in = n_c * esz;
  const size_t need = align16(batch * per_cw_in) + align16(batch * words * 4) + align16(batch * 4) * 2 +
                      align16(batch) * 2 + 16;
  if (need > sl.d_cap) {
    if (sl.d_buf) cudaFree(sl.d_buf);
    sl.d_buf = nullptr;
    sl.d_cap = 0;
    NR_CUDA(cudaMalloc(&sl.d_buf, need));
    sl.d_cap = need;
  }
  if (!sl.h_status) NR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&sl.h_status), sizeof(int32_t)));
  if (!sl.done) NR_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
  for (auto& s : plan->streams)
    if (!s) NR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint8_t* base = static_cast<uint8_t*>(sl.d_buf);
  uint8_t* d_llr = base;
  uint32_t* d_bits = reinterpret_cast<uint32_t*>(base + align16(batch * per_cw_in));
  int32_t* d_iters = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(d_bits) + align16(batch * words * 4));
  int32_t* d_synd = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(d_iters) + align16(batch * 4));
  uint8_t* d_succ = reinterpret_cast<uint8_t*>(d_synd) + align16(batch * 4);
  uint8_t* d_crc = d_succ + align16(batch);
  int32_t* d_status = reinterpret_cast<int32_t*>(d_crc + align16(batch));
  // Pipeline: the copy-in stream moves the chunks in order at full link
  // rate, each chunk's decode waits only for its own input, and many chunk
  // kernels are in flight at once so their partial waves pack the SMs.
  // Results come back in one pass on the copy-out stream (they are ~4% of
  // the input bytes), so the next call's inputs never queue behind them.
  cudaStream_t cin = plan->streams[0], cout = plan->streams[1];
  constexpr int n_comp = nrldpc_plan::kHostStreams - 2;
  NR_CUDA(cudaMemsetAsync(d_status, 0, 4, cin));
  if (chunks < 1) chunks = 1;
  const int64_t per_lane_cta = (int64_t)plan->main.groups * plan->main.lanes;
  int64_t chunk = (batch + chunks - 1) / chunks;
  chunk = (chunk + per_lane_cta - 1) / per_lane_cta * per_lane_cta;
  const int n_chunks = (int)((batch + chunk - 1) / chunk);
  while ((int)plan->chunk_ev.size() < n_chunks + n_comp) {
    cudaEvent_t e;
    NR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    plan->chunk_ev.push_back(e);
  }
  int launches = 0;
  // a pageable input is staged through pinned memory chunk by chunk: the
  // host copy of chunk i+1 overlaps the DMA of chunk i (a pageable source
  // would make every cudaMemcpyAsync a synchronous, driver-staged copy)
  const bool stage_in = is_pageable(llr_host);
  if (stage_in) NR_CUDA(grow_pinned(sl.h_in, sl.h_in_cap, batch * per_cw_in));
  for (int idx = 0; idx < n_chunks; ++idx) {
    const int64_t b0 = idx * chunk;
    const int64_t nb = std::min<int64_t>(chunk, batch - b0);
    const uint8_t* src = static_cast<const uint8_t*>(llr_host) + b0 * per_cw_in;
    if (stage_in) {
      host_copy(sl.h_in + b0 * per_cw_in, src, nb * per_cw_in);
      src = sl.h_in + b0 * per_cw_in;
    }
    NR_CUDA(cudaMemcpyAsync(d_llr + b0 * per_cw_in, src, nb * per_cw_in, cudaMemcpyHostToDevice, cin));
    NR_CUDA(cudaEventRecord(plan->chunk_ev[idx], cin));
    cudaStream_t st = plan->streams[2 + idx % n_comp];
    NR_CUDA(cudaStreamWaitEvent(st, plan->chunk_ev[idx], 0));
    KOut o{d_bits + b0 * words, d_iters + b0, d_synd + b0, d_succ + b0,
           crc_ok ? d_crc + b0 : nullptr, nullptr, nullptr, d_status};
    g_launches = 0;
    const int rc = decode_impl(plan, d_llr + b0 * per_cw_in, nb, o, st);
    if (rc != NRLDPC_OK) return rc;
    launches += g_launches;
  }
  for (int c = 0; c < n_comp; ++c) {
    NR_CUDA(cudaEventRecord(plan->chunk_ev[n_chunks + c], plan->streams[2 + c]));
    NR_CUDA(cudaStreamWaitEvent(cout, plan->chunk_ev[n_chunks + c], 0));
  }
  // results: straight into pinned caller buffers; pageable ones get the
  // slot's pinned staging area and a host copy when the call retires (a D2H
  // copy into pageable memory would block this enqueue until it completes)
  struct Out {
    void* host;
    const void* dev;
    size_t n;
  } outs[5] = {{bits, d_bits, (size_t)batch * words * 4}, {iters, d_iters, (size_t)batch * 4},
               {synd, d_synd, (size_t)batch * 4}, {success, d_succ, (size_t)batch},
               {crc_ok, d_crc, crc_ok ? (size_t)batch : 0}};
  sl.n_dst = 0;
  size_t stage_bytes = 0;
  bool staged[5] = {};
  for (int i = 0; i < 5; ++i) {
    if (outs[i].n && is_pageable(outs[i].host)) {
      staged[i] = true;
      stage_bytes += align16(outs[i].n);
    }
  }
  if (stage_bytes) NR_CUDA(grow_pinned(sl.h_out, sl.h_out_cap, stage_bytes));
  size_t so = 0;
  for (int i = 0; i < 5; ++i) {
    if (!outs[i].n) continue;
    void* dst = outs[i].host;
    if (staged[i]) {
      sl.dst[sl.n_dst++] = {outs[i].host, so, outs[i].n};
      dst = sl.h_out + so;
      so += align16(outs[i].n);
    }
    NR_CUDA(cudaMemcpyAsync(dst, outs[i].dev, outs[i].n, cudaMemcpyDeviceToHost, cout));
  }
  NR_CUDA(cudaMemcpyAsync(sl.h_status, d_status, 4, cudaMemcpyDeviceToHost, cout));
  NR_CUDA(cudaEventRecord(sl.done, cout));
  *launches_out = launches;
  return NRLDPC_OK;
}

// Retire the call in slot `si`: wait for its results and report its status.
// own == false: the retire happens on behalf of another call (the slot is
// being reused, or a synchronous call drains the pipeline); a rejected input
// is then recorded against the retired call's ticket for its own wait
// instead of failing the caller.
static int host_retire(nrldpc_plan* plan, int si, bool own) {
  auto& sl = plan->slot[si];
  if (sl.ticket < 0) return NRLDPC_OK;
  const int64_t t = sl.ticket;
  sl.ticket = -1;
  NR_CUDA(cudaEventSynchronize(sl.done));
  for (int i = 0; i < sl.n_dst; ++i) host_copy(sl.dst[i].p, sl.h_out + sl.dst[i].off, sl.dst[i].n);
  sl.n_dst = 0;
  if (!*sl.h_status) return NRLDPC_OK;
  if (own) return fail(NRLDPC_EINVAL, "int8 LLR magnitudes must be at most 127");
  if (plan->failed.size() >= nrldpc_plan::kMaxFailed) plan->failed.erase(plan->failed.begin());
  plan->failed.push_back(t);
  return NRLDPC_OK;
}

static int host_check_args(const nrldpc_plan* plan, int64_t batch, const void* llr_host, const void* bits,
                           const void* iters, const void* synd, const void* success, const void* crc_ok) {
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (batch < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
  if (batch == 0) return NRLDPC_OK;
  if (!llr_host || !bits || !iters || !synd || !success) return fail(NRLDPC_EINVAL, "NULL buffer");
  if (plan->early_stop == NRLDPC_STOP_CRC && !crc_ok)
    return fail(NRLDPC_EINVAL, "crc mode needs a crc_ok buffer");
  return NRLDPC_OK;
}

int nrldpc_decode_host(nrldpc_plan* plan, const void* llr_host, int64_t batch, uint32_t* bits,
                       int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok, int chunks) {
  g_launches = 0;
  int rc = host_check_args(plan, batch, llr_host, bits, iters, synd, success, crc_ok);
  if (rc != NRLDPC_OK || batch == 0) return rc;
  std::lock_guard<std::mutex> lock(plan->host_mu);
  NR_CUDA(cudaSetDevice(plan->device));
  // a synchronous call retires whatever is still in flight first
  for (int i = 0; i < nrldpc_plan::kSlots; ++i) {
    rc = host_retire(plan, i, false);
    if (rc != NRLDPC_OK) return rc;
  }
  static const bool dbg = getenv("NRLDPC_HOST_TIMING") != nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (dbg) {
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, plan->streams[0] ? plan->streams[0] : nullptr);
  }
  int launches = 0;
  rc = host_enqueue(plan, 0, llr_host, batch, bits, iters, synd, success, crc_ok, chunks, &launches);
  if (rc != NRLDPC_OK) return rc;
  plan->slot[0].ticket = plan->next_ticket++;
  if (dbg) cudaEventRecord(t1, plan->streams[1]);
  rc = host_retire(plan, 0, true);
  if (dbg) {
    float ms = 0;
    cudaEventSynchronize(t1);
    cudaEventElapsedTime(&ms, t0, t1);
    fprintf(stderr, "decode_host gpu span %.3f ms\n", ms);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  g_launches = launches;
  return rc;
}

int nrldpc_decode_host_async(nrldpc_plan* plan, const void* llr_host, int64_t batch, uint32_t* bits,
                             int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok, int chunks,
                             int64_t* ticket) {
  g_launches = 0;
  if (!ticket) return fail(NRLDPC_EINVAL, "NULL ticket");
  *ticket = -1;
  int rc = host_check_args(plan, batch, llr_host, bits, iters, synd, success, crc_ok);
  if (rc != NRLDPC_OK) return rc;
  std::lock_guard<std::mutex> lock(plan->host_mu);
  NR_CUDA(cudaSetDevice(plan->device));
  const int64_t t = plan->next_ticket++;
  if (batch == 0) {
    *ticket = t;
    return NRLDPC_OK;
  }
  const int si = (int)(t % nrldpc_plan::kSlots);
  // the slot's previous call; its status stays with its own ticket
  rc = host_retire(plan, si, false);
  if (rc != NRLDPC_OK) return rc;
  int launches = 0;
  rc = host_enqueue(plan, si, llr_host, batch, bits, iters, synd, success, crc_ok, chunks, &launches);
  if (rc != NRLDPC_OK) return rc;
  plan->slot[si].ticket = t;
  *ticket = t;
  g_launches = launches;
  return NRLDPC_OK;
}

int nrldpc_host_wait(nrldpc_plan* plan, int64_t ticket) {
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  std::lock_guard<std::mutex> lock(plan->host_mu);
  NR_CUDA(cudaSetDevice(plan->device));
  for (int i = 0; i < nrldpc_plan::kSlots; ++i)
    if (plan->slot[i].ticket == ticket) return host_retire(plan, i, true);
  // already retired on behalf of a later call: report its own status
  for (auto it = plan->failed.begin(); it != plan->failed.end(); ++it) {
    if (*it == ticket) {
      plan->failed.erase(it);
      return fail(NRLDPC_EINVAL, "int8 LLR magnitudes must be at most 127");
    }
  }
  return NRLDPC_OK;  // retired ok (or an empty batch)
}

}  // extern "C"
