// Flooding-schedule min-sum (decoder.py:337-365 _scalar_flood, 569-581
// decode_flooding). Every row reads the previous iteration's posteriors; then
// each posterior is rebuilt as L_b + sum of its incoming messages, widened
// (int64 / float64 in the reference) and saturated once per iteration.
// One codeword per CTA, thread per check row z; posteriors L and channel
// values L_b in shared memory as 4-byte values (int32, or float holding the
// f32/f16 value); messages in a global workspace [cw][edge][z].
// Float sums run in double in the reference's order (rows ascending, then
// edges), so the final rounding to float/half matches numpy bit for bit.
// Included by nrldpc.cu.
#pragma once

namespace nr {

// column-major edge lists in the reference's accumulation order
struct FloodTables {
  uint16_t col_start[NR_MAX_BLOCKS + 1];
  uint16_t col_edge[NR_MAX_EDGES];
  uint16_t col_shift[NR_MAX_EDGES];
};

template <int PREC>
struct FloodOps;

template <>
struct FloodOps<NRLDPC_INT8> {
  using V = int;
  using Acc = int;
  __device__ static V from_in(const void* in, long long i) { return ((const int8_t*)in)[i]; }
  __device__ static V sat() { return 127; }
  __device__ static V sub_clamp(V a, V b) { return min(max(a - b, -127), 127); }
  __device__ static V absv(V a) { return abs(a); }
  __device__ static bool neg(V a) { return a < 0; }
  __device__ static V beta_mul(const KParams& p, V m) { return (int)__half2float(__ushort_as_half(p.lut[m])); }
  __device__ static V negate(V a) { return -a; }
  __device__ static Acc acc0(V a) { return a; }
  __device__ static Acc add(Acc a, V b) { return a + b; }
  __device__ static V finish(Acc a) { return min(max(a, -127), 127); }
  __device__ static float mag_f(V a) { return (float)abs(a); }
};

template <>
struct FloodOps<NRLDPC_F32> {
  using V = float;
  using Acc = double;
  __device__ static V from_in(const void* in, long long i) { return ((const float*)in)[i]; }
  __device__ static V sat() { return __int_as_float(0x7F800000); }
  __device__ static V sub_clamp(V a, V b) { return __fsub_rn(a, b); }
  __device__ static V absv(V a) { return fabsf(a); }
  __device__ static bool neg(V a) { return a < 0.0f; }
  __device__ static V beta_mul(const KParams& p, V m) { return __fmul_rn(__uint_as_float(p.beta_f), m); }
  __device__ static V negate(V a) { return -a; }
  __device__ static Acc acc0(V a) { return (double)a; }
  __device__ static Acc add(Acc a, V b) { return __dadd_rn(a, (double)b); }
  __device__ static V finish(Acc a) { return __double2float_rn(a); }
  __device__ static float mag_f(V a) { return fabsf(a); }
};

template <>
struct FloodOps<NRLDPC_F16> {
  using V = float;  // always an exactly representable half value
  using Acc = double;
  __device__ static float h(float x) { return __half2float(__float2half_rn(x)); }
  __device__ static V from_in(const void* in, long long i) { return __half2float(((const __half*)in)[i]); }
  __device__ static V sat() { return 65504.0f; }
  __device__ static V sub_clamp(V a, V b) {
    // half subtraction (one rounding), overflow to inf, then np.clip(+-65504)
    const float d = __half2float(__hsub(__float2half_rn(a), __float2half_rn(b)));
    return fminf(fmaxf(d, -65504.0f), 65504.0f);
  }
  __device__ static V absv(V a) { return fabsf(a); }
  __device__ static bool neg(V a) { return a < 0.0f; }
  __device__ static V beta_mul(const KParams& p, V m) {
    return __half2float(__hmul(__low2half(u2h(p.beta_f)), __float2half_rn(m)));
  }
  __device__ static V negate(V a) { return -a; }
  __device__ static Acc acc0(V a) { return (double)a; }
  __device__ static Acc add(Acc a, V b) { return __dadd_rn(a, (double)b); }
  __device__ static V finish(Acc a) {
    const double c = fmin(fmax(a, -65504.0), 65504.0);
    return __half2float(__double2half(c));
  }
  __device__ static float mag_f(V a) { return fabsf(a); }
};

template <int PREC>
__global__ void __launch_bounds__(384) k_decode_flood(const __grid_constant__ KParams p,
                                                      const __grid_constant__ FloodTables ft,
                                                      const void* __restrict__ llr, void* __restrict__ ws,
                                                      KOut o) {
  using F = FloodOps<PREC>;
  using V = typename F::V;
  extern __shared__ __align__(16) uint8_t smem[];
  const int Z = p.z;
  const long long n_c = (long long)p.n_blocks * Z;
  V* L = reinterpret_cast<V*>(smem);
  V* Lb = L + n_c;
  __shared__ int s_synd, s_done, s_accept;
  __shared__ float s_min;
  const long long cw = blockIdx.x;
  const int z = threadIdx.x;
  const bool on = z < Z;
  V* M = reinterpret_cast<V*>(ws) + cw * (long long)p.n_edges * Z;  // [edge][z]

  bool bad = false;
  for (long long n = z; n < n_c; n += blockDim.x) {
    const V v = F::from_in(llr, cw * n_c + n);
    // int8 inputs must satisfy |x| <= 127 (decoder.py:287-288): -128 is the
    // only int8 value outside, and the host raises the reference's ValueError
    if (PREC == NRLDPC_INT8) bad |= ((const int8_t*)llr)[cw * n_c + n] == -128;
    L[n] = v;
    Lb[n] = v;
  }
  if (bad && o.status) atomicOr(o.status, 1);
  for (long long i = z; i < (long long)p.n_edges * Z; i += blockDim.x) M[i] = V(0);
  if (z == 0) {
    s_synd = 0;
    s_done = 0;
    s_accept = 0;
    s_min = __int_as_float(0x7F800000);
  }
  __syncthreads();

  for (int it = 1; it <= p.max_iter; ++it) {
    // check-node update of every row from the previous posteriors
    if (on) {
      for (int r = 0; r < p.rows; ++r) {
        const int e0 = p.row_start[r], w = p.row_start[r + 1] - e0, t0 = p.tab_start[r];
        V t[19];
        V m1 = F::sat(), m2 = F::sat();
        int tag = -1;
        bool S = false;
        for (int j = 0; j < w; ++j) {
          const int c = (int)p.cb[t0 + j], s = (int)p.sh[t0 + j];
          t[j] = F::sub_clamp(L[c * Z + (z + s) % Z], M[(long long)(e0 + j) * Z + z]);
          const V a = F::absv(t[j]);
          const bool y_wins = a < m1;                       // kernels.py:247-250
          const V loser = y_wins ? m1 : a;
          m1 = y_wins ? a : m1;
          m2 = loser < m2 ? loser : m2;
          tag = y_wins ? j : tag;
          S ^= F::neg(t[j]);
        }
        const V b1 = F::beta_mul(p, m1), b2 = F::beta_mul(p, m2);
        for (int j = 0; j < w; ++j) {
          const V mag = (tag == j) ? b2 : b1;
          M[(long long)(e0 + j) * Z + z] = (S ^ F::neg(t[j])) ? F::negate(mag) : mag;
        }
      }
    }
    __syncthreads();
    // variable-node update: L = sat(L_b + sum of rolled messages), per column
    if (on) {
      for (int c = 0; c < p.n_blocks; ++c) {
        typename F::Acc acc = F::acc0(Lb[c * Z + z]);
        for (int k = ft.col_start[c]; k < ft.col_start[c + 1]; ++k) {
          const int e = ft.col_edge[k], s = ft.col_shift[k];
          acc = F::add(acc, M[(long long)e * Z + (z - s + Z) % Z]);   // np.roll(msg, s)
        }
        L[c * Z + z] = F::finish(acc);
      }
    }
    __syncthreads();

    const bool last = it == p.max_iter;
    if (!(p.early_stop != NRLDPC_STOP_NONE || p.trace || last)) continue;
    if (on) {
      int wc = 0;
      for (int r = 0; r < p.rows; ++r) {
        const int w = p.row_start[r + 1] - p.row_start[r], t0 = p.tab_start[r];
        bool par = false;
        for (int j = 0; j < w; ++j) par ^= F::neg(L[(int)p.cb[t0 + j] * Z + (z + (int)p.sh[t0 + j]) % Z]);
        wc += par;
      }
      float mn = __int_as_float(0x7F800000);
      for (int c = 0; c < p.n_blocks; ++c) mn = fminf(mn, F::mag_f(L[c * Z + z]));
      if (wc) atomicAdd(&s_synd, wc);
      atomicMin(reinterpret_cast<int*>(&s_min), __float_as_int(mn));
    }
    __syncthreads();
    const int wgt = s_synd;
    const float mar = s_min;
    bool cand = p.early_stop != NRLDPC_STOP_NONE && !s_done && wgt == 0 && mar > 0.0f;
    const int K = p.k_b * Z;
    if (p.early_stop == NRLDPC_STOP_CRC) {
      if (cand && on && p.crc_tab) {
        uint32_t acc = 0;
        for (int i = z; i < K; i += Z)
          if (F::neg(L[i])) acc ^= __ldg(p.crc_tab + i);
        if (acc) atomicXor(reinterpret_cast<unsigned int*>(&s_accept), acc);
      }
      __syncthreads();
      cand = cand && p.crc_tab != nullptr && s_accept == 0;
    }
    const bool fin = last && !s_done && !cand;
    if ((cand || fin) && on) {
      for (int wi = z; wi < p.words; wi += Z) {
        const int base = wi * 32, nb = min(32, K - base);
        uint32_t word = 0;
        for (int i = 0; i < nb; ++i) word |= (F::neg(L[base + i]) ? 1u : 0u) << i;
        o.bits[cw * p.words + wi] = word;
      }
    }
    if (z == 0) {
      if (p.trace) {
        o.trace_w[cw * p.max_iter + (it - 1)] = wgt;
        o.trace_m[cw * p.max_iter + (it - 1)] = mar;
      }
      if (cand) {
        o.iters[cw] = it;
        o.synd[cw] = 0;
        o.success[cw] = 1;
        if (o.crc_ok) o.crc_ok[cw] = 1;
      } else if (fin) {
        o.iters[cw] = p.max_iter;
        o.synd[cw] = wgt;
        o.success[cw] = (p.early_stop == NRLDPC_STOP_NONE && wgt == 0 && mar > 0.0f) ? 1 : 0;
        if (o.crc_ok) o.crc_ok[cw] = 0;
      }
    }
    __syncthreads();
    if (z == 0) {
      if (cand) s_done = 1;
      s_synd = 0;
      s_accept = 0;
      s_min = __int_as_float(0x7F800000);
    }
    __syncthreads();
    if (__syncthreads_and(!p.trace && s_done)) break;
  }
}

}  // namespace nr
