// nrldpc device code shared by the translation units: the int8 layered
// decode kernels (k_decode_i8, lane refill), the quantize and ALU-peak
// kernels, and (included at the end) the float / codec / flooding kernels.
// Kernels are templates, instantiated only by the TU that launches them.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "nrldpc_kernels.cuh"
#include "../../include/nrldpc.h"

// ---------------------------------------------------------------------------
// Device code

namespace nr {

struct GroupState {
  int synd[2];
  int minabs[2];
  int done[2];
  int accept[2];
};

// Add a thread's unsatisfied-check count and min |L| into its group's
// counters. When warps never straddle groups (Z % 32 == 0) the warp reduces
// first (REDUX) and one lane issues the shared-memory atomic: 32x fewer
// atomics on the same two addresses, which otherwise serialise (up to 768
// per check at 384 threads). on: this thread contributes (padding threads
// and idle lanes pass false). Every thread of the warp must call it.
__device__ __forceinline__ void group_accumulate(int* synd, int* minabs, int wc, int ma, bool on, bool whole_warps) {
  if (whole_warps) {
    const int s = __reduce_add_sync(0xFFFFFFFFu, on ? wc : 0);
    const int m = __reduce_min_sync(0xFFFFFFFFu, on ? ma : 255);
    if ((threadIdx.x & 31) == 0) {
      if (s) atomicAdd(synd, s);
      if (m < 255) atomicMin(minabs, m);
    }
  } else if (on) {
    if (wc) atomicAdd(synd, wc);
    atomicMin(minabs, ma);
  }
}

// Phase stamps (NRLDPC_PHASES builds only, tools/phase_probe.py): per CTA,
// globaltimer at kernel entry, after the prologue, before the final check,
// after the results, at exit.
#ifdef NRLDPC_PHASES
__device__ unsigned long long nr_phase_stamps[4096 * 16];
__device__ __forceinline__ void phase_stamp(long long cta, int k) {
  if (threadIdx.x == 0 && cta < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    nr_phase_stamps[cta * 16 + k] = t;
  }
}
#else
__device__ __forceinline__ void phase_stamp(long long, int) {}
#endif

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
  chk_smem((uint32_t)__cvta_generic_to_shared(a), 4);
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
#ifdef NRLDPC_CHECKED
    // every gathered position lies in this group's L array; the row's
    // messages lie in this thread's message row
    for (int j = 0; j < w; ++j)
      NR_CHECK(ABS ? off[j] >= p.abs_base && off[j] + LANES <= p.abs_base + p.l_bytes : off[j] + LANES <= p.l_bytes);
    if (!REGMSG) NR_CHECK(mb + (uint32_t)w * LANES <= p.m_stride || PAIRED);
#endif
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
    // (verified exhaustively on the host); no table lookups
    const half2 bh = u2h(k.bh), nd = u2h(k.nd), cc = u2h(k.cc);
    const half2 B1 = __hfma2(__hadd2(m1, nd), bh, cc);
    const half2 B2 = __hfma2(__hadd2(m2, nd), bh, cc);
    // times (-1)^S as a sign-bit flip: one LOP3 each instead of forming
    // +-1.0 and two HMUL2 (exact, including the sign of a zero)
    const uint32_t sflip = S & 0x80008000u;
    dd = u2h(h2u(__hsub2(B1, B2)) ^ sflip);
    b2s = u2h(h2u(__hsub2(B2, cc)) ^ sflip);
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
#ifdef NRLDPC_CHECKED
    for (int j = 0; j < MAXW; ++j) NR_CHECK(off[j] >= p.abs_base && off[j] + 4 <= p.abs_base + p.l_bytes);
    if constexpr (TMEM) NR_CHECK(mb + MAXW <= p.tm_cols && p.tm_cols <= p.tm_slot);
    else if constexpr (!REGMSG) NR_CHECK(mb + 4 * MAXW <= p.m_stride);
#endif
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
    const half2 bh = u2h(k.bh), nd = u2h(k.nd), cc = u2h(k.cc);
    const half2 B1 = __hfma2(__hadd2(m1, nd), bh, cc);
    const half2 B2 = __hfma2(__hadd2(m2, nd), bh, cc);
    // times (-1)^S as a sign-bit flip: one LOP3 each instead of forming
    // +-1.0 and two HMUL2 (exact, including the sign of a zero)
    const uint32_t sflip = S & 0x80008000u;
    dd = u2h(h2u(__hsub2(B1, B2)) ^ sflip);
    b2s = u2h(h2u(__hsub2(B2, cc)) ^ sflip);
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

// Bit-sliced final check of the TM layout (Z % 32 == 0, one group per CTA).
// The hard decisions (decoder.py:323-334: L < 0) of every position are
// packed once into words, one coalesced LDS and two ballots per 32
// positions, with the margin min |L| (decoder.py:480-483) folded into the
// same pass. Check (r, z) is the XOR over the row's edges of the hard bit at
// ((z + s) mod Z) of the edge's column, so the parities of 32 consecutive
// checks z = 32i..32i+31 are the XOR of one funnel-shifted word pair per
// edge: about 1/16 of the instructions of the per-check scan
// (row_parity_tm). W holds {lane a, lane b} per word, word k covering
// positions 32k..32k+31 (bit t = position 32k + t); it lives in the message
// area, dead after the last iteration.
__device__ __forceinline__ void pack_hard_tm(const KParams& p, uint32_t Ls, uint2* W, int* mabs) {
  constexpr int PB = 8;  // words per warp per batch: their loads are all in flight together
  const half2 H255 = u2h(0x5BF85BF8u), H1152 = u2h(0x64806480u);
  const int lid = threadIdx.x & 31, nwarp = p.z >> 5;
  const int warp = (int)__reduce_max_sync(0xFFFFFFFFu, threadIdx.x >> 5);  // REDUX: a warp-uniform value for ptxas
  const int total = p.n_blocks * nwarp;  // words per lane (positions / 32)
  NR_CHECK((uint32_t)total * 8u <= p.m_bytes);
  half2 acc = H255;
  for (int k0 = warp; k0 < total; k0 += PB * nwarp) {
    uint32_t u[PB];
#pragma unroll
    for (int i = 0; i < PB; ++i) {
      const int k = k0 + i * nwarp;
      // past the end: a biased +127, which moves neither the margin (the
      // true minimum is <= 127) nor a stored word
      u[i] = k < total ? lds_u32(Ls + (uint32_t)(k * 32 + lid) * 4u) : 0x64FF64FFu;
    }
    uint32_t va = 0, vb = 0;
#pragma unroll
    for (int i = 0; i < PB; ++i) {
      acc = __hmin2(acc, __habs2(__hsub2(u2h(u[i]), H1152)));
      // the biased half2's low byte has bit 7 clear exactly for v < 0
      // (lane a: bit 7, lane b: bit 23)
      const uint32_t a = __ballot_sync(0xFFFFFFFFu, !(u[i] & 0x80u));
      const uint32_t b = __ballot_sync(0xFFFFFFFFu, !(u[i] & 0x800000u));
      if (lid == i) {
        va = a;
        vb = b;
      }
    }
    const int k = k0 + lid * nwarp;  // lane i stores the batch's word i
    if (lid < PB && k < total) W[k] = make_uint2(va, vb);
  }
  mabs[0] = (int)__low2float(acc);  // exact small integers
  mabs[1] = (int)__high2float(acc);
}

// Parities of checks 32i..32i+31 (lane i < Z/32) of one row of compile-time
// weight W from the packed hard decisions: the row's table loads (uniform,
// 128-bit) and all its word loads are in flight together.
template <int MAXW>
__device__ __forceinline__ void packed_row_parity(const KParams& p, uint32_t tq, const uint2* W, uint32_t lid,
                                                  uint32_t nw, int& wa, int& wb) {
  uint32_t tsh[MAXW], tcb[MAXW];
  load_row_tables<MAXW>(p, tq, MAXW, tsh, tcb);
  uint32_t xa = 0, xb = 0;
#pragma unroll
  for (int j = 0; j < MAXW; ++j) {
    const uint32_t s = tsh[j] >> 2;                  // TM tables: shift * 4
    const uint32_t cw = (tcb[j] - p.abs_base) >> 7;  // column * Z * 4 + base -> column * Z / 32
    uint32_t q = 32u * (lid < nw ? lid : 0u) + s;
    if (q >= (uint32_t)p.z) q -= (uint32_t)p.z;
    const uint32_t k = q >> 5, o = q & 31u;
    const uint32_t k1 = k + 1 == nw ? 0u : k + 1;
    NR_CHECK((cw + nw) * 8u <= p.m_bytes);
    const uint2 lo = W[cw + k], hi = W[cw + k1];
    xa ^= __funnelshift_r(lo.x, hi.x, o);
    xb ^= __funnelshift_r(lo.y, hi.y, o);
  }
  if (lid < nw) {  // the other lanes ran on a copy of lane 0's checks
    wa += __popc(xa);
    wb += __popc(xb);
  }
}

// Syndrome weights from the packed hard decisions: warp w takes the rows
// r with r % (Z/32) == w, lane i the checks 32i..32i+31 (lanes >= Z/32 run
// a copy of lane 0's checks and do not count them). The phase is latency-
// bound (dependent table and word loads per row); a per-thread row loop and
// tables staged in shared memory measured no faster
// (profiles/r02_cta_phases.txt).
template <int BG>
__device__ __forceinline__ void packed_parity_tm(const KParams& p, const uint2* W, int& wa, int& wb) {
  const uint32_t lid = threadIdx.x & 31, nw = (uint32_t)p.z >> 5;
  const int warp = (int)__reduce_max_sync(0xFFFFFFFFu, threadIdx.x >> 5);  // REDUX: warp-uniform
  wa = wb = 0;
  int owner = 0;  // r % (Z/32)
  for (int r = 0; r < p.rows; ++r) {
    if (owner == warp) {  // warp-uniform: the whole warp runs the row
      const uint32_t tq = (uint32_t)p.tab_start[r] / 4u;
      dispatch_w<BG>(p.row_start[r + 1] - p.row_start[r],
                     [&](auto WW) { packed_row_parity<decltype(WW)::value>(p, tq, W, lid, nw, wa, wb); });
    }
    owner = owner + 1 == (int)nw ? 0 : owner + 1;
  }
}

// The hard-decision words of the first K positions straight from the packed
// words (K = k_b * Z, a whole number of words): coalesced stores.
__device__ __forceinline__ void write_bits_packed(const KParams& p, const uint2* W, int z, const int (&need)[2],
                                                  long long cw0, uint32_t* __restrict__ bits) {
  for (int k = z; k < p.words; k += p.z) {
    const uint2 v = W[k];
    NR_CHECK(!need[0] || cw0 < p.batch);
    NR_CHECK(!need[1] || cw0 + 1 < p.batch);
    if (need[0]) bits[cw0 * p.words + k] = v.x;
    if (need[1]) bits[(cw0 + 1) * p.words + k] = v.y;
  }
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
// once every live lane has one. Returns when done or stopped. The first
// block is one row: a codeword still far from convergence fails there
// already (config 3: +2.5% against a first block of four rows), and the
// later blocks are eight rows.
#ifndef NRLDPC_EARLY_FIRST
#define NRLDPC_EARLY_FIRST 1
#endif
#ifndef NRLDPC_EARLY_NEXT
#define NRLDPC_EARLY_NEXT 8
#endif
template <int BG, int R, int STEP, int NEXT = STEP>
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
    parity_rows_early_tm<BG, E, NEXT, NEXT>(p, zl, ZL, wa, wb, need_a, need_b, pub_a, pub_b, synd);
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
      parity_rows_early_tm<BG, 0, NRLDPC_EARLY_FIRST, NRLDPC_EARLY_NEXT>(p, zl, ZL, wa, wb, need_a, need_b, pub_a, pub_b, synd);
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
template <int BG, int LANES, bool ABS, int R, int STEP, int NEXT = STEP>
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
    parity_rows_early<BG, LANES, ABS, E, NEXT, NEXT>(p, zl, ZL, Lg, wa, wb, need_a, need_b, pub_a, pub_b, synd);
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
      parity_rows_early<BG, LANES, ABS, 0, NRLDPC_EARLY_FIRST, NRLDPC_EARLY_NEXT>(p, zl, ZL, Lg, wa, wb, need_a, nb,
                                                                              pub_a, pub_b, synd);
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
    NR_CHECK(cw < p.batch && wi < p.words);
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
      NR_CHECK(!need[0] || cw0 < p.batch);
      NR_CHECK(LANES != 2 || !need[1] || cw1 < p.batch);
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
__device__ __forceinline__ void decode_i8_cta(const KParams& p, const int8_t* __restrict__ llr, const KOut o,
                                              const long long cta_idx) {
  static_assert(NREG == 0 || (BG == 1 && LANES == 2), "register messages: BG1 pairs only");
  static_assert(!ABS || BG != 0, "absolute addressing: compile-time schedules only");
  static_assert(!TM || (BG != 0 && LANES == 2 && (NREG == 6 || NREG == 0) && ABS), "TM layout: pair shapes");
  constexpr uint32_t ES = TM ? 4 : LANES;  // bytes per position of L
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* lut = reinterpret_cast<uint16_t*>(smem);
  CtaState* cta = reinterpret_cast<CtaState*>(smem + kLutBytes);
  GroupState* gstate = reinterpret_cast<GroupState*>(smem + kLutBytes + kCtaBytes);
  const uint32_t data_off = data_offset(p.groups);

  phase_stamp(cta_idx, 0);
  const int tid = threadIdx.x;
  // not a padding thread; register-row shapes have one group of Z threads
  // with Z in {288, 320, 352, 384}, a whole number of warps (host-checked)
  const bool st_ok = NREG > 0 || tid < p.groups * p.z;
  const int g = st_ok ? tid / p.z : p.groups - 1;
  const int z = st_ok ? tid - g * p.z : (tid - g * p.z) % p.z;
  const long long cw0 = (cta_idx * p.groups + g) * LANES;
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
    const long long first = cta_idx * p.groups * LANES;
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
  phase_stamp(cta_idx, 1);

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
    if (last) phase_stamp(cta_idx, 2);

    // ---- end-of-iteration check (decoder.py:497-536) ----
    // weights are only needed in full when traced or final
    const bool early = BG != 0 && !p.trace && !last && p.z % 32 == 0;
    // TM, final and untraced: the bit-sliced check (pack_hard_tm), whose
    // words also give the result bits; the message area is dead by now
    const bool packed = TM && last && !p.trace;
    uint2* W = reinterpret_cast<uint2*>(Lg + p.l_bytes);
    {
      int wc[2], ma[2];
      if constexpr (TM) {
        if (packed) {
          __syncthreads();  // every message store of the last layer has landed before W reuses the area
          phase_stamp(cta_idx, 8);
          pack_hard_tm(p, p.abs_base, W, ma);
          phase_stamp(cta_idx, 9);
          __syncthreads();
          phase_stamp(cta_idx, 10);
          packed_parity_tm<BG>(p, W, wc[0], wc[1]);
        } else {
          local_check_tm<BG>(p, zl, ZL, p.abs_base, wc, ma, early, lane_valid[0] && !gs.done[0],
                             lane_valid[1] && !gs.done[1], gs.synd);
        }
      } else
        local_check<BG, MAXW, LANES, ABS>(p, zl, ZL, Lg, wc, ma, early, lane_valid[0] && !gs.done[0],
                                          lane_valid[1] && !gs.done[1], gs.synd);
      if (last) phase_stamp(cta_idx, 5);
      // minabs starts at 255 and |L| <= 127, so 255 never needs storing
#pragma unroll
      for (int l = 0; l < LANES; ++l)
        group_accumulate(&gs.synd[l], &gs.minabs[l], wc[l], ma[l], active, p.z % 32 == 0);
    }
    __syncthreads();
    if (last) phase_stamp(cta_idx, 6);
    if constexpr (TM) {
      // second pass: the margin, only when a live lane's syndrome is zero
      // (block-uniform: shared state read after the barrier)
      if (early && ((lane_valid[0] && !gs.done[0] && gs.synd[0] == 0) ||
                    (lane_valid[1] && !gs.done[1] && gs.synd[1] == 0))) {
        int ma[2];
        margin_tm(p, zl, ZL, p.abs_base, ma);
        group_accumulate(&gs.synd[0], &gs.minabs[0], 0, ma[0], true, true);
        group_accumulate(&gs.synd[1], &gs.minabs[1], 0, ma[1], true, true);
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
        if (need[0] || need[1]) {
          if (packed) write_bits_packed(p, W, z, need, cw0, o.bits);
          else write_bits_warp<LANES, ES>(p, Lg, z, need, cw0, o.bits);
        }
        if (last) phase_stamp(cta_idx, 7);
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
          NR_CHECK(cw < p.batch);
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
  phase_stamp(cta_idx, 3);
  if constexpr (TM) {
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(lds_u32(&cta->kc[5])));
  }
  phase_stamp(cta_idx, 4);
}

// One launch, one shape: CTA blockIdx.x decodes codewords
// [blockIdx.x * groups * LANES, ...).
template <int BG, int MAXW, int LANES, int NREG, bool ABS, bool TM = false>
__global__ void __launch_bounds__(NREG ? 384 : 512, 1) k_decode_i8(const __grid_constant__ KParams p,
                                                                   const int8_t* __restrict__ llr, KOut o) {
  decode_i8_cta<BG, MAXW, LANES, NREG, ABS, TM>(p, llr, o, (long long)blockIdx.x);
}

// One launch, up to kMultiShapes shapes of the same kernel variant and CTA
// size (mixed-size batches, BASELINE config 4): shape s owns CTAs
// [cta_end[s-1], cta_end[s]). Each shape's full KParams sits in the
// parameter block, so its graph tables are read from the constant bank with
// a uniform shape offset, exactly as in the one-shape launch. This replaces
// per-shape launches whose number, not their work, limited a mixed batch:
// a CUDA-graph replay runs about 32 kernels concurrently (tools/cfg4_probe.py).
template <int BG, int MAXW, int LANES, int NREG, bool ABS, bool TM = false>
__global__ void __launch_bounds__(NREG ? 384 : 512, 1) k_decode_i8_multi(const __grid_constant__ KMulti P) {
  int s = 0;  // block-uniform
#pragma unroll
  for (int i = 0; i + 1 < kMultiShapes; ++i) s += (i + 1 < P.n && (int)blockIdx.x >= P.cta_end[i]) ? 1 : 0;
  const int begin = s ? P.cta_end[s - 1] : 0;
  decode_i8_cta<BG, MAXW, LANES, NREG, ABS, TM>(P.s[s], P.llr[s], P.o[s], (long long)blockIdx.x - begin);
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
      for (int l = 0; l < 2; ++l) group_accumulate(&gs.synd[l], &gs.minabs[l], wc[l], ma[l], true, true);
    }
    __syncthreads();
    if constexpr (TM) {
      // second pass: the margin, only when a live lane's syndrome is zero
      if (!last[0] && !last[1] && ((act[0] && gs.synd[0] == 0) || (act[1] && gs.synd[1] == 0))) {
        int ma[2];
        margin_tm(p, zl, ZL, p.abs_base, ma);
        group_accumulate(&gs.synd[0], &gs.minabs[0], 0, ma[0], true, true);
        group_accumulate(&gs.synd[1], &gs.minabs[1], 0, ma[1], true, true);
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
          NR_CHECK(c >= 0 && c < p.batch);
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
            // 16 columns per round trip: four loads in flight, one wait
            for (; c + 16 <= p.tm_cols; c += 16) {
              uint32_t r[16];
#pragma unroll
              for (int q = 0; q < 16; q += 4) tm_ld4(tbase + c + q, r[q], r[q + 1], r[q + 2], r[q + 3]);
              tm_wait_ld<16>(r);
#pragma unroll
              for (int q = 0; q < 16; q += 4)
                tm_st4(tbase + c + q, (r[q] & keep_m) | zb, (r[q + 1] & keep_m) | zb, (r[q + 2] & keep_m) | zb,
                       (r[q + 3] & keep_m) | zb);
            }
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
