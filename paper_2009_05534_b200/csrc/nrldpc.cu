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
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <bitset>
#include <vector>

#define NRLDPC_AUX_KERNELS  // k_encode / k_channel_awgn live in this TU
#include "nrldpc_host.h"

namespace nrh {

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

}  // namespace nrh

using nrh::cuda_fail;
using nrh::fail;
using nrh::g_last_error;

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
      // workspace rows: slots padded to whole uint4 quads ([quad][z][4])
      if (!leading) return false;
      ml.mb[r] = (uint32_t)e_glob;
      e_glob += (w + 3) & ~3;
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
  // absolute L addressing (one group per CTA): L starts after the CTA state
  // and one FltState, in the dynamic window after the 1 KB system area
  // (k_decode_flt checks the address)
  sh.kp.abs_base = 0x400u + (((uint32_t)kCtaBytes + (uint32_t)sizeof(FltState) + 15u) & ~15u);
  for (int t = 0; t < NR_MAX_TAB; ++t) sh.kp.cb[t] += sh.kp.abs_base;
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

static cudaError_t launch_shape(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch,
                                const KOut& o, cudaStream_t st) {
  if (sh.threads == 0) return cudaErrorInvalidConfiguration;  // no feasible shape
  // early-stop modes without a trace: refill lanes as codewords stop
  const bool refill = plan->early_stop != NRLDPC_STOP_NONE && o.trace_w == nullptr && sh.abs && sh.lanes == 2 &&
                      sh.groups == 1 && plan->z % 32 == 0 && !getenv("NRLDPC_NO_REFILL");
  if (sh.tm) return launch_int8_tm(plan, sh, in, batch, o, st, refill);
  if (plan->schedule == 1) return launch_int8_bg1(plan, sh, in, batch, o, st, refill);
  return launch_int8_bg2(plan, sh, in, batch, o, st, refill);
}

// The int8 kernel instantiation launch_shape would use for `sh` (plain pair
// kernel, no refill): the grouping key of multi-shape launches. 0: none.
static int kernel_variant(const nrldpc_plan* plan, const Shape& sh) {
  if (plan->precision != NRLDPC_INT8 || sh.threads == 0) return 0;
  const bool two = sh.lanes == 2;
  if (sh.tm) return sh.nreg == 6 ? 1 : plan->schedule == 1 ? 2 : 3;
  if (plan->schedule == 1) {
    if (!two) return 10;
    if (sh.nreg == 0) return sh.abs ? 11 : 12;
    if (!sh.abs) return 0;
    return sh.nreg == 2 ? 13 : sh.nreg == 4 ? 14 : 15;
  }
  if (plan->schedule == 2) return !two ? 20 : sh.abs ? 21 : 22;
  if (plan->maxw > 10) return two ? 30 : 31;
  return two ? 32 : 33;
}

// ---- host worker pool -------------------------------------------------------
// A few persistent threads for the host side of the end-to-end path: copying
// a pageable caller's input into pinned staging memory, and unpacking packed
// hard decisions into the reference's (B, K) byte layout. One copy thread
// moves ~10 GB/s; the pool splits each chunk so the host copy keeps ahead
// of the PCIe DMA it feeds. NRLDPC_HOST_THREADS overrides the size.
class HostPool {
 public:
  // One parallel job: f(i) for i in [0, n), tasks handed out in index order.
  struct Job {
    std::function<void(int)> f;
    int n = 0;
    std::atomic<int> next{0}, left{0};
  };
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int workers() const { return (int)workers_.size(); }
  // Start a job on the worker threads and return at once; the caller may do
  // other work (e.g. issue DMAs as pieces complete) before wait(). One job
  // at a time: submit holds the pool until the matching wait.
  std::shared_ptr<Job> submit(int n, std::function<void(int)> f) {
    auto job = std::make_shared<Job>();
    job->f = std::move(f);
    job->n = n;
    job->left.store(n);
    call_mu_.lock();
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = job;
      ++gen_;
    }
    cv_.notify_all();
    return job;
  }
  // The caller helps with the remaining tasks, then waits for the job.
  void wait(const std::shared_ptr<Job>& job) {
    work(*job);
    {
      std::unique_lock<std::mutex> lk(mu_);
      done_cv_.wait(lk, [&] { return job->left.load() == 0; });
      job_.reset();
    }
    call_mu_.unlock();
  }
  void run(int n, std::function<void(int)> f) {
    if (n <= 0) return;
    if (n == 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    wait(submit(n, std::move(f)));
  }

 private:
  HostPool() {
    int n = std::min((int)std::thread::hardware_concurrency(), 8);
    if (const char* e = std::getenv("NRLDPC_HOST_THREADS")) n = std::min(std::atoi(e), 64);
    n = std::max(1, n);
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
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
  void work(Job& job) {
    for (;;) {
      const int i = job.next.fetch_add(1);
      if (i >= job.n) return;
      job.f(i);
      if (job.left.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      if (job) work(*job);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Copy into pinned staging memory that only the DMA engine reads next:
// streaming (non-temporal) stores skip the read-for-ownership of the
// destination, so the copy moves 2 instead of 3 bytes of host memory traffic
// per byte, the resource it shares with the DMA (NRLDPC_NO_NT=1: memcpy).
#if defined(__x86_64__) && !defined(__CUDA_ARCH__)
__attribute__((target("avx2"))) static void stream_copy_avx2(uint8_t* d, const uint8_t* s, size_t n) {
  size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
  }
  std::memcpy(d + i, s + i, n - i);
  _mm_sfence();  // the streaming stores are visible before the task reports completion
}
#endif

static void staging_copy(uint8_t* d, const uint8_t* s, size_t n) {
#if defined(__x86_64__) && !defined(__CUDA_ARCH__)
  static const bool nt = __builtin_cpu_supports("avx2") && !std::getenv("NRLDPC_NO_NT");
  if (nt) {
    stream_copy_avx2(d, s, n);
    return;
  }
#endif
  std::memcpy(d, s, n);
}

static void host_copy(void* dst, const void* src, size_t n, bool streaming = false) {
  constexpr size_t kPiece = 256u << 10;
  HostPool& pool = HostPool::get();
  const int parts = (int)std::min<size_t>((size_t)pool.workers() + 1, (n + kPiece - 1) / kPiece);
  auto copy = [streaming](uint8_t* d, const uint8_t* s, size_t len) {
    if (streaming) staging_copy(d, s, len);
    else std::memcpy(d, s, len);
  };
  if (parts <= 1) {
    copy(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), n);
    return;
  }
  const size_t per = ((n + parts - 1) / parts + 4095) & ~size_t(4095);
  pool.run(parts, [=](int i) {
    const size_t o = (size_t)i * per;
    if (o < n) copy(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o, std::min(per, n - o));
  });
}

// Packed hard-decision words -> the reference's (B, K) bytes 0/1, LSB first
// (decoder.py:332-334), rows split over the host pool.
static void unpack_rows_parallel(const uint32_t* words, int64_t batch, int64_t words_per_cw, int64_t k,
                                 uint8_t* out) {
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
  const int nt = pool.workers() + 1;
  const int64_t per = std::max<int64_t>(1, (batch + 4 * nt - 1) / (4 * nt));
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
  unpack_rows_parallel(words, batch, words_per_cw, k, out);
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
      if (!ftm_layout(p, p->main, ml)) {
        // every row in the workspace, [quad][z][4] with rows padded to
        // whole quads (FRow kind 0); e_reg = padded slots per group
        int slots = 0;
        for (int r = 0; r < p->rows; ++r) {
          ml.mb[r] = (uint32_t)slots;
          slots += (p->base.row_start[r + 1] - p->base.row_start[r] + 3) & ~3;
        }
        p->main.kp.e_reg = slots;
      }
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
                                  : launch_float_any(precision, p->schedule, p->main, device, nullptr, 0, none, nullptr);
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
  for (auto& e : plan->word_ev) cudaEventDestroy(e);
  if (plan->h_words) cudaFreeHost(plan->h_words);
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

int nrldpc_plan_kernel(const nrldpc_plan* plan, int* kernel, int* threads, int64_t* smem_bytes) {
  if (!plan) return fail(NRLDPC_EINVAL, "plan is NULL");
  if (kernel) *kernel = kernel_variant(plan, plan->main);
  if (threads) *threads = plan->main.threads;
  if (smem_bytes) *smem_bytes = (int64_t)plan->main.smem;
  return NRLDPC_OK;
}

int nrldpc_decode_multi(nrldpc_plan* const* plans, int n, const void* const* llr, const int64_t* batch,
                        uint32_t* const* bits, int32_t* const* iters, int32_t* const* synd,
                        uint8_t* const* success, uint8_t* const* crc_ok, int32_t* status, void* stream) {
  g_launches = 0;
  if (!plans || !llr || !batch || !bits || !iters || !synd || !success)
    return fail(NRLDPC_EINVAL, "NULL array");
  if (n < 1 || n > NRLDPC_MULTI_MAX) return fail(NRLDPC_EINVAL, "n must be in [1, NRLDPC_MULTI_MAX]");
  const nrldpc_plan* p0 = plans[0];
  if (!p0) return fail(NRLDPC_EINVAL, "plan is NULL");
  const int kern = kernel_variant(p0, p0->main);
  if (kern == 0) return fail(NRLDPC_EINVAL, "multi-shape launches need int8 plans");
  Shape* sh[kMultiShapes];
  const int8_t* in[kMultiShapes];
  long long nb[kMultiShapes];
  KOut o[kMultiShapes];
  for (int i = 0; i < n; ++i) {
    nrldpc_plan* p = plans[i];
    if (!p) return fail(NRLDPC_EINVAL, "plan is NULL");
    if (p->device != p0->device) return fail(NRLDPC_EINVAL, "plans of one multi-shape launch share a device");
    if (kernel_variant(p, p->main) != kern || p->main.threads != p0->main.threads)
      return fail(NRLDPC_EINVAL, "plans of one multi-shape launch need the same kernel variant and CTA size");
    if (batch[i] < 0) return fail(NRLDPC_EINVAL, "batch must be non-negative");
    if (batch[i] > 0 && (!llr[i] || !bits[i] || !iters[i] || !synd[i] || !success[i]))
      return fail(NRLDPC_EINVAL, "NULL buffer");
    if (p->early_stop == NRLDPC_STOP_CRC && batch[i] > 0 && (!crc_ok || !crc_ok[i]))
      return fail(NRLDPC_EINVAL, "crc mode needs a crc_ok buffer");
    sh[i] = &p->main;
    in[i] = static_cast<const int8_t*>(llr[i]);
    nb[i] = batch[i];
    o[i] = KOut{bits[i], iters[i], synd[i], success[i], crc_ok ? crc_ok[i] : nullptr, nullptr, nullptr, status,
                nullptr};
  }
  NR_CUDA(cudaSetDevice(p0->device));
  cudaStream_t st = (cudaStream_t)stream;
  const cudaError_t e = kern <= 3    ? launch_int8_multi_tm(kern, sh, n, in, nb, o, p0->device, st)
                        : kern < 20  ? launch_int8_multi_bg1(kern, sh, n, in, nb, o, p0->device, st)
                                     : launch_int8_multi_bg2(kern, sh, n, in, nb, o, p0->device, st);
  if (e != cudaSuccess) return cuda_fail(e, "multi-shape decode launch");
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
    const cudaError_t e = launch_float_any(plan->precision, plan->schedule, plan->main, plan->device, llr, batch, o, st);
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
// chunk_words (nrldpc_decode_host_bytes): each chunk's packed words come back
// on its own decode stream right after its kernel, into plan->h_words, with
// plan->word_ev[chunk] recorded; `bits` is then unused and the chunk
// geometry is returned in *n_chunks_out / *chunk_out.
static int host_enqueue(nrldpc_plan* plan, int si, const void* llr_host, int64_t batch, uint32_t* bits,
                        int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok, int chunks,
                        int* launches_out, bool chunk_words = false, int* n_chunks_out = nullptr,
                        int64_t* chunk_out = nullptr) {
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
  if (chunk_words) {
    while ((int)plan->word_ev.size() < n_chunks) {
      cudaEvent_t e;
      NR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      plan->word_ev.push_back(e);
    }
    if (batch * words * 4 > plan->h_words_cap) {
      uint8_t* hw = reinterpret_cast<uint8_t*>(plan->h_words);
      NR_CUDA(grow_pinned(hw, plan->h_words_cap, batch * words * 4));
      plan->h_words = reinterpret_cast<uint32_t*>(hw);
    }
    *n_chunks_out = n_chunks;
    *chunk_out = chunk;
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
      // host copy of this chunk on the pool (the DMA of the previous chunk
      // runs meanwhile). Measured on the GPU box: the staging is bound by
      // host memory bandwidth (copy read + write + the DMA's read); letting
      // the copy run ahead of the DMA on all workers was slower (2.0 vs
      // 1.3 ms per 26.7 MB batch, tools/api_phase_probe.py)
      host_copy(sl.h_in + b0 * per_cw_in, src, nb * per_cw_in, true);
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
    if (chunk_words) {
      NR_CUDA(cudaMemcpyAsync(plan->h_words + b0 * words, d_bits + b0 * words, nb * words * 4,
                              cudaMemcpyDeviceToHost, st));
      NR_CUDA(cudaEventRecord(plan->word_ev[idx], st));
    }
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
  } outs[5] = {{bits, d_bits, chunk_words ? 0 : (size_t)batch * words * 4}, {iters, d_iters, (size_t)batch * 4},
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

int nrldpc_decode_host_bytes(nrldpc_plan* plan, const void* llr_host, int64_t batch, uint8_t* bits,
                             int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok, int chunks) {
  g_launches = 0;
  int rc = host_check_args(plan, batch, llr_host, bits, iters, synd, success, crc_ok);
  if (rc != NRLDPC_OK || batch == 0) return rc;
  std::lock_guard<std::mutex> lock(plan->host_mu);
  NR_CUDA(cudaSetDevice(plan->device));
  for (int i = 0; i < nrldpc_plan::kSlots; ++i) {
    rc = host_retire(plan, i, false);
    if (rc != NRLDPC_OK) return rc;
  }
  int launches = 0, n_chunks = 0;
  int64_t chunk = 0;
  rc = host_enqueue(plan, 0, llr_host, batch, nullptr, iters, synd, success, crc_ok, chunks, &launches, true,
                    &n_chunks, &chunk);
  if (rc != NRLDPC_OK) return rc;
  plan->slot[0].ticket = plan->next_ticket++;
  // unpack each chunk's words as soon as they land, while later chunks
  // still decode: only the last chunk's unpack is exposed
  const int64_t words = plan->base.words, k = (int64_t)plan->k_b * plan->z;
  for (int idx = 0; idx < n_chunks; ++idx) {
    const int64_t b0 = idx * chunk, nb = std::min<int64_t>(chunk, batch - b0);
    NR_CUDA(cudaEventSynchronize(plan->word_ev[idx]));
    unpack_rows_parallel(plan->h_words + b0 * words, nb, words, k, bits + b0 * k);
  }
  rc = host_retire(plan, 0, true);
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

