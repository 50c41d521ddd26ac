// Floating-point layered min-sum engines (Precision.F32 / Precision.F16),
// bit-exact restatements of the reference's float paths:
//   f32: lvc = lv - msg, b = float32(beta) * m, new = lvc + out, no clamp
//   f16: every op rounded to half (numpy float16 ufuncs are correctly
//        rounded), lvc and new clamped to +-65504 (decoder.py:227-240)
// (/root/reference/pkg/src/ldpclab/decoder.py:295-320). f16 carries two
// codewords per half2 lane; f32 one codeword per thread. Posteriors live in
// shared memory (4 bytes per position per group); messages (4 bytes per edge
// and z per group) live in a stream-ordered global workspace, coalesced as
// [group][edge][z]. On-chip variant (FTM, single-group BG1/BG2 shapes that
// hold an SM alone): the messages of most rows move on chip, into shared
// memory (thread-major, odd word stride) or tensor memory (tcgen05.ld/st,
// the thread's own lane, as in k_decode_i8's TM layout); the kind follows
// from the row weight (ftm_kind). Included by nrldpc.cu.
#pragma once

namespace nr {

// Per-lane arithmetic on a 32-bit element (one float, or a half2 pair).
template <int PREC>
struct FOps;

template <>
struct FOps<NRLDPC_F32> {
  static constexpr int lanes = 1;
  static constexpr uint32_t sign = 0x80000000u;
  __device__ static uint32_t sat() { return 0x7F800000u; }  // +inf: the f32 fold identity
  __device__ static uint32_t sub_clamp(uint32_t a, uint32_t b) {
    return __float_as_uint(__fsub_rn(__uint_as_float(a), __uint_as_float(b)));
  }
  __device__ static uint32_t add_clamp(uint32_t a, uint32_t b) {
    return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(b)));
  }
  __device__ static uint32_t absv(uint32_t a) { return a & 0x7FFFFFFFu; }
  __device__ static uint32_t minv(uint32_t a, uint32_t b) {
    return __float_as_uint(fminf(__uint_as_float(a), __uint_as_float(b)));
  }
  __device__ static uint32_t maxv(uint32_t a, uint32_t b) {
    return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b)));
  }
  __device__ static uint32_t mul(uint32_t a, uint32_t b) {
    return __float_as_uint(__fmul_rn(__uint_as_float(a), __uint_as_float(b)));
  }
  __device__ static uint32_t neg_mask(uint32_t a) { return __uint_as_float(a) < 0.0f ? 0xFFFFFFFFu : 0u; }
  __device__ static uint32_t eq_mask(uint32_t a, uint32_t b) {
    return __uint_as_float(a) == __uint_as_float(b) ? 0xFFFFFFFFu : 0u;
  }
  __device__ static float lane_abs(uint32_t a, int) { return fabsf(__uint_as_float(a)); }
  __device__ static bool lane_neg(uint32_t a, int) { return __uint_as_float(a) < 0.0f; }
};

template <>
struct FOps<NRLDPC_F16> {
  static constexpr int lanes = 2;
  static constexpr uint32_t sign = 0x80008000u;
  __device__ static uint32_t sat() { return 0x7BFF7BFFu; }  // 65504 (F16_SAT)
  __device__ static half2 clamp(half2 x) {
    return __hmin2(__hmax2(x, u2h(0xFBFFFBFFu)), u2h(0x7BFF7BFFu));  // np.clip(+-65504)
  }
  __device__ static uint32_t sub_clamp(uint32_t a, uint32_t b) { return h2u(clamp(__hsub2(u2h(a), u2h(b)))); }
  __device__ static uint32_t add_clamp(uint32_t a, uint32_t b) { return h2u(clamp(__hadd2(u2h(a), u2h(b)))); }
  __device__ static uint32_t absv(uint32_t a) { return a & 0x7FFF7FFFu; }
  __device__ static uint32_t minv(uint32_t a, uint32_t b) { return h2u(__hmin2(u2h(a), u2h(b))); }
  __device__ static uint32_t maxv(uint32_t a, uint32_t b) { return h2u(__hmax2(u2h(a), u2h(b))); }
  __device__ static uint32_t mul(uint32_t a, uint32_t b) { return h2u(__hmul2(u2h(a), u2h(b))); }
  // a < 0 per lane (-0 is not negative) in the lane's sign bit only, which is
  // all the callers read (sign products, parity bits 15/31): sign bit AND a
  // nonzero magnitude. |a| + 0x7FFF sets bit 15 exactly when |a| != 0 and
  // cannot carry into the other lane (|a| <= 0x7C00). Integer ops instead of
  // HSET2, which issues at a quarter of the full rate on sm_100.
  __device__ static uint32_t neg_mask(uint32_t a) { return a & ((a & 0x7FFF7FFFu) + 0x7FFF7FFFu) & sign; }
  // a == b per lane as a full-lane mask, for non-negative a and b (|t| and
  // m1): equal halves have equal bits, so a ^ b is zero exactly there; the
  // same carry-free test marks nonzero lanes in bit 15, and PRMT replicates
  // that bit over the lane (0xbb99: the sign bits of bytes 1 and 3)
  __device__ static uint32_t eq_mask(uint32_t a, uint32_t b) {
    uint32_t ne;
    asm("prmt.b32 %0, %1, 0, 0xbb99;" : "=r"(ne) : "r"((a ^ b) + 0x7FFF7FFFu));
    return ~ne;
  }
  __device__ static float lane_abs(uint32_t a, int l) {
    return fabsf(__half2float(l ? __high2half(u2h(a)) : __low2half(u2h(a))));
  }
  __device__ static bool lane_neg(uint32_t a, int l) {
    return __half2float(l ? __high2half(u2h(a)) : __low2half(u2h(a))) < 0.0f;
  }
};

// Message store of a row in the on-chip variant: 0 global workspace, 1 shared
// memory, 2 tensor memory. BG1: the four 19-edge core rows (76 edges) stay
// global, rows with w >= 7 go to shared memory, the rest to tensor memory;
// BG2: w >= 8 shared, the rest tensor memory (host: ftm_shape).
template <int BG>
__host__ __device__ constexpr int ftm_kind(int w) {
  return BG == 1 ? (w == 19 ? 0 : w >= 7 ? 1 : 2) : (w >= 8 ? 1 : 2);
}

// Two smallest of a[0..W-1] (non-negative, NaN-free) from the fold identity
// F::sat(), as a pairwise tree (see two_smallest in nrldpc_device.cuh).
template <typename F, int N>
__device__ __forceinline__ void flt_merge(uint32_t (&lo)[N], uint32_t (&hi)[N]) {
  if constexpr (N > 1) {
    constexpr int M = (N + 1) / 2;
    uint32_t nlo[M], nhi[M];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      nlo[i] = F::minv(lo[2 * i], lo[2 * i + 1]);
      nhi[i] = F::minv(F::minv(F::maxv(lo[2 * i], lo[2 * i + 1]), hi[2 * i]), hi[2 * i + 1]);
    }
    if constexpr ((N & 1) != 0) {
      nlo[M - 1] = lo[N - 1];
      nhi[M - 1] = hi[N - 1];
    }
    flt_merge<F, M>(nlo, nhi);
    lo[0] = nlo[0];
    hi[0] = nhi[0];
  }
}

template <typename F, int W>
__device__ __forceinline__ void flt_two_smallest(const uint32_t (&a)[W], uint32_t& m1, uint32_t& m2) {
  constexpr int P = (W + 1) / 2;
  uint32_t lo[P], hi[P];
#pragma unroll
  for (int i = 0; i < W / 2; ++i) {
    lo[i] = F::minv(a[2 * i], a[2 * i + 1]);
    hi[i] = F::maxv(a[2 * i], a[2 * i + 1]);
  }
  if constexpr ((W & 1) != 0) {
    lo[P - 1] = a[W - 1];
    hi[P - 1] = F::sat();
  }
  flt_merge<F, P>(lo, hi);
  if constexpr (F::lanes == 2) {
    // f16: every |t| is already clipped to 65504 = sat (FRow::main), so the
    // cap at the fold identity is a no-op
    m1 = lo[0];
    m2 = hi[0];
  } else {
    m1 = F::minv(lo[0], F::sat());
    m2 = F::minv(hi[0], F::sat());
  }
}

// Posterior access: relative to the group's L array, or (ABSL, the on-chip
// single-group shapes) at an absolute shared-window address already folded
// into the graph table's column base, so a gather is LDS [R + UR] with no
// per-edge address add (as in k_decode_i8's ABS shapes).
template <bool ABSL>
__device__ __forceinline__ uint32_t ld_L(const uint8_t* Lg, uint32_t off) {
  if constexpr (ABSL) return lds_u32(off);
  else return *reinterpret_cast<const uint32_t*>(Lg + off);
}
template <bool ABSL>
__device__ __forceinline__ void st_L(uint8_t* Lg, uint32_t off, uint32_t v) {
  if constexpr (ABSL) sts_u32(off, v);
  else *reinterpret_cast<uint32_t*>(Lg + off) = v;
}

// One row of a compile-time (BG1/BG2) layer unit in the float engines,
// split like the int8 RowWork: pro() touches only this thread's own state
// (graph tables, edge addresses, its messages from the global workspace), so
// it runs before the barrier that closes the previous layer; main() reads
// the posteriors.
template <int PREC, int W, int KIND = 0, bool ABSL = false>
struct FRow {
  using F = FOps<PREC>;
  uint32_t off[W], t[W], neg[W], msg[W], a[W];
  uint32_t m1, m2, S, beta;
  uint4* Me;     // global kind: this row's first quad, edges 4q..4q+3 at Me[q * Z]
  uint32_t Ma;   // shared kind: shared address of the row's first message; tensor kind: TMEM address
  // e0: the row's first edge (global kind), byte offset in this thread's
  // shared message row (shared kind) or column in its TMEM slot (tensor kind)
  static constexpr int NQ = (W + 3) / 4;
  __device__ __forceinline__ void pro(const KParams& p, uint32_t tq, uint32_t e0, uint32_t zl, uint32_t ZL,
                                      uint4* Mg, bool active, uint32_t Ms = 0, uint32_t tbase = 0) {
    uint32_t tsh[W], tcb[W];
    load_row_tables<W>(p, tq, W, tsh, tcb);
    if constexpr (KIND == 0) {
      // quad-interleaved workspace: one coalesced 16-byte load per four
      // edges (e0: the row's first slot, a multiple of 4)
      Me = Mg + (long long)(e0 >> 2) * p.z;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const uint4 v = active ? Me[(long long)q * p.z] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * q + k < W) msg[4 * q + k] = vv[k];
      }
    } else if constexpr (KIND == 1) {
      Ma = Ms + e0;
    } else {
      Ma = tbase + e0;
      tm_ld_row<W>(Ma, msg);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
      off[j] = edge_offset(tsh[j], tcb[j], zl, ZL);
      if constexpr (KIND == 1) msg[j] = lds_u32(Ma + 4u * j);
    }
  }
  __device__ __forceinline__ void main(const uint8_t* Lg, uint32_t beta_) {
    if constexpr (KIND == 2) tm_wait_ld<W>(msg);
    S = 0;
    beta = beta_;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const uint32_t lv = ld_L<ABSL>(Lg, off[j]);
      if constexpr (PREC == NRLDPC_F16) {
        // lvc = clip(lv - msg, +-65504) (decoder.py:300, 231): the clipped
        // magnitude is min(|d|, 65504) (one HMNMX2 with the |.| modifier;
        // the clip only maps +-inf), the sign is d's. No posterior is -0
        // (the prologue loads -0 as +0), so d is never -0 and lvc < 0 is
        // its sign bit.
        const uint32_t d = h2u(__hsub2(u2h(lv), u2h(msg[j])));
        a[j] = h2u(__hmin2(__habs2(u2h(d)), u2h(F::sat())));
        t[j] = (d & F::sign) | a[j];
        neg[j] = t[j];  // sign bits only are read
      } else {
        // f32 has no clip (decoder.py:300); with no -0 posterior (the
        // prologue loads -0 as +0) lvc < 0 is again the sign bit of t for
        // finite posteriors
        t[j] = F::sub_clamp(lv, msg[j]);
        a[j] = F::absv(t[j]);
        neg[j] = t[j];  // sign bits only are read
      }
      S ^= neg[j];
    }
    // the two smallest |t| (kernels.py:247-250 fold from the saturation
    // identity) as a pairwise tree: the same values as the sequential fold
    // (ties give m1 == m2 either way), ~log2(W) deep instead of ~2W
    flt_two_smallest<F, W>(a, m1, m2);
  }
  __device__ __forceinline__ void scatter(uint8_t* Lg, const KParams& p, bool active) {
    const uint32_t x12 = m1 ^ m2;
    // the row sign S folded into beta, so dtype(beta) * other carries
    // it and the edge's own sign is one XOR; a zero magnitude keeps the
    // sign the reference gives -0 (np.where(sign, -b, b))
    const uint32_t beta_s = beta ^ (S & F::sign);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      // the reference's magnitude b = dtype(beta) * (j == argmin ? m2 : m1)
      // (decoder.py:306-316). Every edge but the argmin has |t| >= m2, the
      // argmin has |t| = m1 <= m2, so min(|t|, m2) is m1 there and m2
      // elsewhere, and (m1 ^ m2) ^ min(|t|, m2) selects the other one
      // bitwise (non-negative values; a tie has m1 == m2 either way). The
      // multiply runs per edge on the otherwise idle FMA pipe instead of a
      // compare + select on the busy ALU pipe.
      const uint32_t other = x12 ^ F::minv(a[j], m2);
      const uint32_t out = F::mul(beta_s, other) ^ (neg[j] & F::sign);  // -mag flips the sign bit
      if constexpr (KIND == 2 || KIND == 0) msg[j] = out;
      if (active) {
        if constexpr (KIND == 1) sts_u32(Ma + 4u * j, out);
        st_L<ABSL>(Lg, off[j], F::add_clamp(t[j], out));  // decoder.py:318
      }
    }
    if constexpr (KIND == 2) tm_st_row<W>(Ma, msg);  // warp-collective: every thread of an FTM CTA is active
    if constexpr (KIND == 0) {
      if (active) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          Me[(long long)q * p.z] = make_uint4(msg[4 * q], 4 * q + 1 < W ? msg[4 * q + 1] : 0u,
                                              4 * q + 2 < W ? msg[4 * q + 2] : 0u,
                                              4 * q + 3 < W ? msg[4 * q + 3] : 0u);
      }
    }
  }
};

// One row's parity of hard decisions (lvc < 0) for the
// end-of-iteration check, with the row weight known at compile time.
template <int PREC, int W, bool ABSL = false>
__device__ __forceinline__ void flt_row_parity(const KParams& p, uint32_t tq, const uint8_t* Lg, uint32_t zl,
                                               uint32_t ZL, int (&wc)[2]) {
  using F = FOps<PREC>;
  uint32_t tsh[W], tcb[W];
  load_row_tables<W>(p, tq, W, tsh, tcb);
  uint32_t par = 0;
#pragma unroll
  // no posterior is -0 (the prologue loads -0 as +0), so lvc < 0 is the
  // sign bit and the row parity is the XOR of the raw words' sign bits
  for (int j = 0; j < W; ++j) par ^= ld_L<ABSL>(Lg, edge_offset(tsh[j], tcb[j], zl, ZL));
  if (F::lanes == 1) {
    wc[0] += par >> 31;
  } else {  // half2 masks: lane 0 in bits 0-15, lane 1 in bits 16-31
    wc[0] += (par >> 15) & 1u;
    wc[1] += par >> 31;
  }
}

// The full syndrome of a full compile-time graph (rows R..E-1) as
// straight-line code.
template <int PREC, int BG, bool ABSL, int R = 0, int E = RowW<BG>::n>
__device__ __forceinline__ void flt_parity_rows(const KParams& p, const uint8_t* Lg, uint32_t zl, uint32_t ZL,
                                                int (&wc)[2]) {
  if constexpr (R < E) {
    flt_row_parity<PREC, RowW<BG>::w[R], ABSL>(p, row_tq<BG, R>(), Lg, zl, ZL, wc);
    flt_parity_rows<PREC, BG, ABSL, R + 1, E>(p, Lg, zl, ZL, wc);
  }
}

// Early-stop iterations (see local_check_tm): blocks of STEP straight-line
// rows; a warp publishes a failing check of a live lane in the group's
// counters at once, and all warps stop when every live lane has one.
template <int PREC, int BG, bool ABSL, int R, int STEP, int NEXT = STEP>
__device__ __forceinline__ void flt_parity_rows_early(const KParams& p, const uint8_t* Lg, uint32_t zl, uint32_t ZL,
                                                      int (&wc)[2], bool need_a, bool need_b, bool& pub_a,
                                                      bool& pub_b, int* synd) {
  if constexpr (R < RowW<BG>::n) {
    constexpr int E = R + STEP < RowW<BG>::n ? R + STEP : RowW<BG>::n;
    flt_parity_rows<PREC, BG, ABSL, R, E>(p, Lg, zl, ZL, wc);
    const bool leader = (threadIdx.x & 31) == 0;
    if (!pub_a && __any_sync(0xFFFFFFFFu, wc[0] != 0)) {
      if (leader) atomicAdd(&synd[0], 1);
      pub_a = true;
    }
    if (!pub_b && __any_sync(0xFFFFFFFFu, wc[1] != 0)) {
      if (leader) atomicAdd(&synd[1], 1);
      pub_b = true;
    }
    const volatile int* vs = synd;
    if ((!need_a || vs[0] != 0) && (!need_b || vs[1] != 0)) return;
    flt_parity_rows_early<PREC, BG, ABSL, E, NEXT, NEXT>(p, Lg, zl, ZL, wc, need_a, need_b, pub_a, pub_b, synd);
  }
}

struct FltState {
  int synd[2];
  float minabs[2];
  int done[2];
  uint32_t accept[2];
};

template <int PREC, int BG = 0, bool FTM = false>
__global__ void __launch_bounds__(512) k_decode_flt(const __grid_constant__ KParams p,
                                                    const void* __restrict__ llr,
                                                    uint32_t* __restrict__ ws, KOut o) {
  static_assert(!FTM || BG != 0, "on-chip messages: compile-time schedules only");
  using F = FOps<PREC>;
  constexpr int LANES = F::lanes;
  extern __shared__ __align__(16) uint8_t smem[];
  CtaState* cta = reinterpret_cast<CtaState*>(smem);
  FltState* gstate = reinterpret_cast<FltState*>(smem + kCtaBytes);
  const uint32_t data_off = ((uint32_t)kCtaBytes + (uint32_t)sizeof(FltState) * p.groups + 15u) & ~15u;

  const int tid = threadIdx.x;
  const bool st_ok = tid < p.groups * p.z;
  const int g = st_ok ? tid / p.z : p.groups - 1;
  const int z = st_ok ? tid - g * p.z : (tid - g * p.z) % p.z;
  const long long gg = (long long)blockIdx.x * p.groups + g;  // global group index
  const long long cw0 = gg * LANES;
  const bool active = st_ok && cw0 < p.batch;
  // ZL through an opaque move: otherwise the compiler rewrites edge_offset's
  // (zl + s) - ZL as (z - Z) * 4 + s, one more instruction per edge than the
  // fused add-min (VIADDMNMX) it emits for the int8 kernels
  uint32_t ZL;
  asm("mov.b32 %0, %1;" : "=r"(ZL) : "r"((uint32_t)p.z * 4u));
  const uint32_t zl = (uint32_t)z * 4u;
  const long long n_c = (long long)p.n_blocks * p.z;
  uint8_t* Lg = smem + data_off + (uint32_t)g * p.l_bytes;
  // generic schedule: edge e at Mg[e * Z]. Compile-time schedules: e_reg
  // padded slots per group as [quad][z][4] (FTM: only the global rows)
  uint32_t* Mg = ws + gg * (long long)p.n_edges * p.z + z;
  uint4* Mg4 = reinterpret_cast<uint4*>(ws) + gg * (long long)(p.e_reg >> 2) * p.z + z;
  FltState& gs = gstate[g];
  // FTM: shared message rows after L (one group), tensor-memory slot
  const uint32_t Ms = (uint32_t)__cvta_generic_to_shared(Lg + p.l_bytes) + (uint32_t)z * p.m_stride;
  // FTM: the host folded L's shared-window address into the column bases
  if (FTM && (uint32_t)__cvta_generic_to_shared(Lg) != p.abs_base) __trap();
  uint32_t tbase = 0;
  if constexpr (FTM) {
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

  if (tid == 0) {
    const long long first = (long long)blockIdx.x * p.groups * LANES;
    cta->n_done = 0;
    cta->n_valid = (int)min(p.batch - first, (long long)p.groups * LANES);
  }
  if (st_ok && z == 0) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      gs.synd[l] = 0;
      gs.minabs[l] = __int_as_float(0x7F800000);
      gs.done[l] = 0;
      gs.accept[l] = 0;
    }
  }
  bool lane_valid[2];
  lane_valid[0] = active;
  lane_valid[1] = active && LANES == 2 && cw0 + 1 < p.batch;

  // load posteriors (decoder.py:286: astype to the engine dtype, done by the
  // caller) and zero the messages of this group
  if (st_ok) {
    for (int c = 0; c < p.n_blocks; ++c) {
      const long long n = (long long)c * p.z + z;
      uint32_t v = 0;
      if (PREC == NRLDPC_F32) {
        if (lane_valid[0]) v = reinterpret_cast<const uint32_t*>(llr)[cw0 * n_c + n];
        if (v == 0x80000000u) v = 0u;  // -0 loads as +0, as for f16 below
      } else {
        const uint16_t* h = reinterpret_cast<const uint16_t*>(llr);
        uint32_t lo = lane_valid[0] ? h[cw0 * n_c + n] : 0u;
        uint32_t hi = lane_valid[1] ? h[(cw0 + 1) * n_c + n] : 0u;
        // -0 inputs load as +0. The decode never creates a -0 posterior
        // itself (x - y and x + y are -0 only for a -0 operand, and messages
        // are subtracted/added to posteriors), so afterwards "lvc < 0" is the
        // sign bit alone. Every output is unchanged: -0 and +0 compare and
        // order the same, and only lvc < 0 / |L| reach the results
        // (decoder.py:300-334).
        if (lo == 0x8000u) lo = 0u;
        if (hi == 0x8000u) hi = 0u;
        v = lo | (hi << 16);
      }
      *reinterpret_cast<uint32_t*>(Lg + (uint32_t)n * 4u) = v;
    }
    if constexpr (BG != 0) {
      if (active)
        for (int q = 0; q < (p.e_reg >> 2); ++q) Mg4[(long long)q * p.z] = make_uint4(0u, 0u, 0u, 0u);
    }
    if constexpr (FTM) {
      uint4* m4 = reinterpret_cast<uint4*>(Lg + p.l_bytes);
      for (uint32_t k = z; k < (p.m_bytes >> 4); k += p.z) m4[k] = make_uint4(0u, 0u, 0u, 0u);
      uint32_t c = 0;
      for (; c + 4 <= p.tm_cols; c += 4) tm_st4(tbase + c, 0u, 0u, 0u, 0u);
      for (; c < p.tm_cols; ++c) tm_st1(tbase + c, 0u);
      tm_wait_st();
    } else if (BG == 0 && active) {
      for (int e = 0; e < p.n_edges; ++e) Mg[(long long)e * p.z] = 0u;
    }
  }
  __syncthreads();

  const uint32_t beta = p.beta_f;
  for (int it = 1; it <= p.max_iter; ++it) {
   if constexpr (BG != 0) {
    // host-built layer units (KParams::unit_a/b, edge indices for messages)
    bool bar_prev = false;
    // an on-chip (FTM) CTA is one group of exactly blockDim threads and the
    // grid never holds a CTA without a codeword, so every thread is active:
    // known at compile time, the message loads and stores need no branch
    const bool act = FTM ? true : active;
    // the dispatch code is loaded one unit ahead (as in one_iteration), so
    // the dispatch branch does not wait on the constant load
    uint32_t ncode = p.unit_a[0].x;
#pragma unroll 1
    for (int u = 0; u < p.n_units; ++u) {
      const uint32_t code = ncode;
      const uint4 A = p.unit_a[u];
      const uint4 B = p.unit_b[u];
      ncode = p.unit_a[u + 1].x;
      dispatch_unit<BG, 0>(code, [&](auto WA, auto WB) {
        constexpr int wa = decltype(WA)::value, wb = decltype(WB)::value;
        FRow<PREC, wa, FTM ? ftm_kind<BG>(wa) : 0, FTM> ra;
        ra.pro(p, A.z, A.w, zl, ZL, Mg4, act, Ms, tbase);
        if constexpr (wb == 0) {
          if (bar_prev) __syncthreads();
          ra.main(Lg, beta);
          ra.scatter(Lg, p, act);
        } else {
          FRow<PREC, wb, FTM ? ftm_kind<BG>(wb) : 0, FTM> rb;
          rb.pro(p, B.x, B.y, zl, ZL, Mg4, act, Ms, tbase);
          if (bar_prev) __syncthreads();
          ra.main(Lg, beta);
          rb.main(Lg, beta);
          ra.scatter(Lg, p, act);
          rb.scatter(Lg, p, act);
        }
      });
      bar_prev = A.y != 0;
    }
    if (bar_prev) __syncthreads();
    if constexpr (FTM) tm_wait_st();  // the next iteration reads these messages back
   } else {
    for (int r = 0; r < p.rows; ++r) {
      const int e0 = p.row_start[r];
      const int w = p.row_start[r + 1] - e0;
      uint32_t tsh[19], tcb[19];
      load_row_tables<19>(p, p.tab_start[r] / 4u, w, tsh, tcb);
      uint32_t off[19], t[19], neg[19];
      uint32_t m1 = F::sat(), m2 = F::sat(), S = 0;
#pragma unroll
      for (int j = 0; j < 19; ++j) {
        if (j < w) {
          off[j] = edge_offset(tsh[j], tcb[j], zl, ZL);
          const uint32_t lv = *reinterpret_cast<const uint32_t*>(Lg + off[j]);
          const uint32_t mv = Mg[(long long)(e0 + j) * p.z];
          t[j] = F::sub_clamp(lv, mv);                 // decoder.py:300
          const uint32_t a = F::absv(t[j]);
          neg[j] = F::neg_mask(t[j]);                  // lvc < 0 (-0 is not negative)
          m2 = F::minv(m2, F::maxv(m1, a));            // kernels.py:247-250
          m1 = F::minv(m1, a);
          S ^= neg[j];
        }
      }
      const uint32_t b1 = F::mul(beta, m1), b2 = F::mul(beta, m2);  // dtype(beta) * m
#pragma unroll
      for (int j = 0; j < 19; ++j) {
        if (j < w) {
          const uint32_t eq = F::eq_mask(F::absv(t[j]), m1);        // the argmin edge (ties: m1 == m2)
          const uint32_t mag = (eq & b2) | (~eq & b1);
          const uint32_t out = mag ^ ((S ^ neg[j]) & F::sign);       // -mag flips the sign bit
          if (active) {
            Mg[(long long)(e0 + j) * p.z] = out;
            *reinterpret_cast<uint32_t*>(Lg + off[j]) = F::add_clamp(t[j], out);  // decoder.py:318
          }
        }
      }
      __syncthreads();
    }
   }
    const bool last = it == p.max_iter;
    if (!(p.early_stop != NRLDPC_STOP_NONE || p.trace || last)) continue;

    // end-of-iteration check (decoder.py:497-536); early-stop iterations of
    // full graphs cooperate (whole warps per group when Z % 32 == 0)
    const bool early = BG != 0 && !p.trace && !last && p.z % 32 == 0 && p.early_stop != NRLDPC_STOP_NONE;
    if (active) {
      int wc[2] = {0, 0};
      bool straight = false, coop = false;
      const bool need_a = lane_valid[0] && !gs.done[0];
      const bool need_b = LANES == 2 && lane_valid[1] && !gs.done[1];
      if constexpr (BG != 0) {
        if (p.rows == RowW<BG>::n) {
          if (early) {
            bool pub_a = !need_a, pub_b = !need_b;
            // first block one row, then eight (as the int8 kernels, parity_rows_early_tm)
            flt_parity_rows_early<PREC, BG, FTM, 0, 1, 8>(p, Lg, zl, ZL, wc, need_a, need_b, pub_a, pub_b, gs.synd);
            wc[0] = wc[1] = 0;  // already counted in gs.synd
            coop = true;
          } else {
            flt_parity_rows<PREC, BG, FTM>(p, Lg, zl, ZL, wc);
          }
          straight = true;
        }
      }
      for (int r = 0; r < p.rows && !straight; ++r) {
        const int w = p.row_start[r + 1] - p.row_start[r];
        uint32_t tsh[19], tcb[19];
        load_row_tables<19>(p, p.tab_start[r] / 4u, w, tsh, tcb);
        uint32_t par = 0;
#pragma unroll
        for (int j = 0; j < 19; ++j)
          if (j < w) par ^= F::neg_mask(ld_L<FTM>(Lg, edge_offset(tsh[j], tcb[j], zl, ZL)));
        if (LANES == 1) {
          wc[0] += par >> 31;
        } else {  // half2 masks: lane 0 in bits 0-15, lane 1 in bits 16-31
          wc[0] += (par >> 15) & 1u;
          wc[1] += par >> 31;
        }
      }
      float ma[2] = {__int_as_float(0x7F800000), __int_as_float(0x7F800000)};
      // the margin matters only for a lane whose syndrome is zero
      const volatile int* vs = gs.synd;
      const bool margin = !coop || (need_a && vs[0] == 0) || (need_b && vs[1] == 0);
      for (int c = 0; c < p.n_blocks && margin; ++c) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(Lg + (uint32_t)c * ZL + zl);
#pragma unroll
        for (int l = 0; l < LANES; ++l) ma[l] = fminf(ma[l], F::lane_abs(v, l));
      }
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        // non-negative floats order as their bit patterns; with whole warps
        // per group (Z % 32 == 0, group-uniform `active`) the warp reduces
        // first and one lane issues the atomics (see group_accumulate)
        if (p.z % 32 == 0) {
          const int s = __reduce_add_sync(0xFFFFFFFFu, wc[l]);
          const int m = __reduce_min_sync(0xFFFFFFFFu, __float_as_int(ma[l]));
          if ((threadIdx.x & 31) == 0) {
            if (s) atomicAdd(&gs.synd[l], s);
            atomicMin(reinterpret_cast<int*>(&gs.minabs[l]), m);
          }
        } else {
          if (wc[l]) atomicAdd(&gs.synd[l], wc[l]);
          atomicMin(reinterpret_cast<int*>(&gs.minabs[l]), __float_as_int(ma[l]));
        }
      }
    }
    __syncthreads();
    int cand[2] = {0, 0};
    if (active && p.early_stop != NRLDPC_STOP_NONE) {
#pragma unroll
      for (int l = 0; l < LANES; ++l)
        cand[l] = lane_valid[l] && !gs.done[l] && gs.synd[l] == 0 && gs.minabs[l] > 0.0f;
    }
    if (p.early_stop == NRLDPC_STOP_CRC) {
      if (active) {
        const int K = p.k_b * p.z;
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (!cand[l]) continue;
          uint32_t acc = p.crc_tab ? 0u : 1u;
          if (p.crc_tab)
            for (int i = z; i < K; i += p.z) {
              const uint32_t v = *reinterpret_cast<const uint32_t*>(Lg + (uint32_t)i * 4u);
              if (F::lane_neg(v, l)) acc ^= __ldg(p.crc_tab + i);
            }
          if (acc) atomicXor(&gs.accept[l], acc);
        }
      }
      __syncthreads();
#pragma unroll
      for (int l = 0; l < LANES; ++l) cand[l] = cand[l] && p.crc_tab != nullptr && gs.accept[l] == 0;
    }
    int fin[2] = {0, 0};
    if (active && last) {
#pragma unroll
      for (int l = 0; l < LANES; ++l) fin[l] = lane_valid[l] && !gs.done[l] && !cand[l];
    }
    if (active) {
      const int K = p.k_b * p.z;
#pragma unroll
      for (int l = 0; l < LANES; ++l) {
        if (!(cand[l] || fin[l])) continue;
        for (int wi = z; wi < p.words; wi += p.z) {
          const int base = wi * 32;
          const int nb = min(32, K - base);
          uint32_t word = 0;
          for (int i = 0; i < nb; ++i)
            word |= (F::lane_neg(*reinterpret_cast<const uint32_t*>(Lg + (uint32_t)(base + i) * 4u), l) ? 1u : 0u) << i;
          o.bits[(cw0 + l) * p.words + wi] = word;
        }
      }
      if (z == 0) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) {
          if (!lane_valid[l]) continue;
          const long long cw = cw0 + l;
          const int wgt = gs.synd[l];
          const float mar = gs.minabs[l];
          if (p.trace) {
            o.trace_w[cw * p.max_iter + (it - 1)] = wgt;
            o.trace_m[cw * p.max_iter + (it - 1)] = mar;
          }
          if (cand[l]) {
            o.iters[cw] = it;
            o.synd[cw] = 0;
            o.success[cw] = 1;
            if (o.crc_ok) o.crc_ok[cw] = 1;
          } else if (fin[l]) {
            o.iters[cw] = p.max_iter;
            o.synd[cw] = wgt;
            o.success[cw] = (p.early_stop == NRLDPC_STOP_NONE && wgt == 0 && mar > 0.0f) ? 1 : 0;
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
        gs.minabs[l] = __int_as_float(0x7F800000);
        gs.accept[l] = 0;
      }
      if (newly) atomicAdd(&cta->n_done, newly);
    }
    __syncthreads();
    if (__syncthreads_and(!p.trace && cta->n_done >= cta->n_valid)) break;
  }
  if constexpr (FTM) {
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(lds_u32(&cta->kc[5])));
  }
}

}  // namespace nr
