// GPU synthetic-traffic kernels: systematic encoder and a
// fused BPSK + AWGN + demapper + quantizer, so BLER sweeps and slot-scale
// batches are generated at GPU speed. Included by nrldpc.cu.
//
// Encoder: the reference's algorithm (codec.py:66-139). Core rows' info part
// t_r, first parity column p0 = roll(t0^t1^t2^t3, core_sum_shift), the three
// other core columns by back-substitution in the reference's order, then
// every extension row through its identity column. Bit-exact.
//
// Channel: y = (1 - 2b) + sigma*n, L = (2y)/(sigma*sigma), q = clip(rint(L*scale))
// (channel.py:47-83). The reference draws n from numpy's PCG64; here n comes
// from a counter-based Philox4x32-10 + Box-Muller, so traffic is statistically
// equivalent (N(0, sigma^2)), not draw-for-draw identical.
#pragma once

namespace nr {

struct EncSched {
  int css;            // core_sum_shift
  int nsteps;         // back-substitution steps (3 for the 5G-NR-style core)
  int row[4], col[4], shift[4];
};

// Non-template kernels: compiled only in the TU that launches them.
#ifdef NRLDPC_AUX_KERNELS
// One codeword per CTA, Z threads; x holds one byte per codeword bit.
__global__ void __launch_bounds__(512) k_encode(const __grid_constant__ KParams p, EncSched es,
                                                const uint8_t* __restrict__ msgs, long long batch,
                                                uint8_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int Z = p.z;
  const int p0 = p.k_b;
  uint8_t* x = smem;                             // (k_b + rows) * Z
  uint8_t* t = smem + p.n_blocks * Z;            // 4 * Z
  const long long cw = blockIdx.x;
  const int z = threadIdx.x;
  const bool on = z < Z;
  const int K = p.k_b * Z;
  const long long n_c = (long long)p.n_blocks * Z;
  auto edge_col = [&](int r, int j) { return (int)p.cb[p.tab_start[r] + j]; };
  auto edge_shift = [&](int r, int j) { return (int)p.sh[p.tab_start[r] + j]; };
  auto rw = [&](int r) { return (int)(p.row_start[r + 1] - p.row_start[r]); };

  for (int i = z; i < K; i += blockDim.x) x[i] = msgs[cw * K + i];
  __syncthreads();
  if (on) {
    for (int r = 0; r < 4; ++r) {                // info part of each core row
      uint32_t acc = 0;
      for (int j = 0; j < rw(r); ++j) {
        const int c = edge_col(r, j);
        if (c < p0) acc ^= x[c * Z + (z + edge_shift(r, j)) % Z];
      }
      t[r * Z + z] = (uint8_t)acc;
    }
  }
  __syncthreads();
  if (on) {                                      // p0 = roll(t0^t1^t2^t3, css)
    const int q = (z - es.css % Z + Z) % Z;
    x[p0 * Z + z] = t[q] ^ t[Z + q] ^ t[2 * Z + q] ^ t[3 * Z + q];
  }
  __syncthreads();
  for (int k = 0; k < es.nsteps; ++k) {          // back-substitution, reference order
    const int r = es.row[k], cu = es.col[k], su = es.shift[k];
    if (on) {
      const int q = (z - su % Z + Z) % Z;        // x[cu] = roll(u, su)
      uint32_t u = t[r * Z + q];
      for (int j = 0; j < rw(r); ++j) {
        const int c = edge_col(r, j);
        if (c >= p0 && c != cu) u ^= x[c * Z + (q + edge_shift(r, j)) % Z];
      }
      x[cu * Z + z] = (uint8_t)u;
    }
    __syncthreads();
  }
  if (on) {                                      // extension rows: independent of each other
    for (int r = 4; r < p.rows; ++r) {
      uint32_t acc = 0;
      for (int j = 0; j < rw(r); ++j) {
        const int c = edge_col(r, j);
        if (c != p0 + r) acc ^= x[c * Z + (z + edge_shift(r, j)) % Z];
      }
      x[(p0 + r) * Z + z] = (uint8_t)acc;
    }
  }
  __syncthreads();
  for (long long i = z; i < n_c; i += blockDim.x) out[cw * n_c + i] = x[i];
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// bits (batch, n_c) 0/1 -> int8 decoder-domain LLR blocks (batch, n_c), the
// first 2Z positions punctured (zero). Four positions per thread per step.
__global__ void __launch_bounds__(256) k_channel_awgn(const uint8_t* __restrict__ bits, long long batch,
                                                      int n_c, int two_z, double sigma, double scale,
                                                      unsigned long long seed, int8_t* __restrict__ out) {
  const long long total = batch * (long long)n_c;
  const double inv_s2 = 1.0 / (sigma * sigma);
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i0 < total;
       i0 += (long long)gridDim.x * blockDim.x * 4) {
    const uint4 r = philox4x32_10(make_uint4((uint32_t)i0, (uint32_t)(i0 >> 32), 0x4C445043u, 0u), key);
    const uint32_t rv[4] = {r.x, r.y, r.z, r.w};
    double n[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {               // Box-Muller on two uniform pairs
      const double u1 = ((double)rv[2 * h] + 1.0) * (1.0 / 4294967296.0);   // (0, 1]
      const double u2 = (double)rv[2 * h + 1] * (1.0 / 4294967296.0);
      const double rad = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      n[2 * h] = rad * cs;
      n[2 * h + 1] = rad * sn;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long i = i0 + k;
      if (i >= total) break;
      const int j = (int)(i % n_c);
      if (j < two_z) {
        out[i] = 0;
        continue;
      }
      const double y = (bits[i] ? -1.0 : 1.0) + sigma * n[k];
      double q = rint((2.0 * y) * inv_s2 * scale);
      q = fmin(fmax(q, -127.0), 127.0);
      out[i] = (int8_t)q;
    }
  }
}

#endif  // NRLDPC_AUX_KERNELS

}  // namespace nr
