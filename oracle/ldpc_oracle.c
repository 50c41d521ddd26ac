/*
 * ldpc_oracle.c — CPU restatement of the reference's layered min-sum decoder.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker (tests/,
 * __graft_entry__.smoke) and the CPU baseline (bench.py --impl reference and
 * the cpu_baseline leg). The product path (paper_2009_05534_b200) never links
 * or calls it.
 *
 * It restates, per codeword, /root/reference/pkg/src/ldpclab/decoder.py:
 *   init_workspace        :256-292  (rows_used from n_c, zero messages)
 *   _scalar_layer         :295-320  (gather, clamp, fold, beta, scatter)
 *   ValueAccumulator.merge kernels.py:246-257 (strict '<' keeps the first tag)
 *   _beta_mag             :208-212  (int: floor(beta*m) in double; float:
 *                                    dtype(beta)*m in the engine dtype)
 *   _clamp / _sat_value   :227-240
 *   _scalar_syndrome      :323-329, _min_abs_lv :480-483, hard bits :332-334
 *   _run_schedule         :486-540  (freeze at first w==0 && margin>0, CRC)
 *   codec._crc_remainder  codec.py:201-213
 * Codewords are independent, so the batch is split over threads (OpenMP).
 * For trace parity every codeword runs max_iter iterations when a trace
 * buffer is given; the caller truncates like the reference's batch loop.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/*.npz, tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PREC_INT8 0
#define PREC_F16 1
#define PREC_F32 2
#define STOP_SYNDROME 0
#define STOP_CRC 1
#define STOP_NONE 2

typedef struct {
  int k_b, z, rows, n_blocks, n_edges;
  const int32_t* row_start;
  const int16_t* cols;
  const int16_t* shifts;
  double beta;
  int max_iter, early_stop, crc_len;
  uint32_t crc_poly;
} graph_t;

static int crc_pass(const uint8_t* bits, int k, int len, uint32_t poly) {
  /* codec.py:183-191, 201-213 */
  if (k < len) return 0;
  const uint32_t top = 1u << (len - 1);
  const uint32_t mask = (len == 32) ? 0xFFFFFFFFu : ((1u << len) - 1u);
  uint32_t reg = 0;
  for (int i = 0; i < k; ++i) {
    const uint32_t fb = ((reg & top) ? 1u : 0u) ^ (uint32_t)bits[i];
    reg = ((reg << 1) & mask) ^ (fb ? poly : 0u);
  }
  return reg == 0;
}

/* ---------------- int8 engine (widened to int32) ---------------- */

static inline int32_t clamp127(int32_t x) { return x < -127 ? -127 : (x > 127 ? 127 : x); }

static void layer_i8(const graph_t* g, int32_t* L, int32_t* M, const int32_t* lut, int r) {
  const int Z = g->z;
  const int e0 = g->row_start[r], w = g->row_start[r + 1] - e0;
  int32_t t[32];
  int idx[32];
  for (int z = 0; z < Z; ++z) {
    int32_t m1 = 127, m2 = 127, tag = -1, s = 0;
    for (int j = 0; j < w; ++j) {
      const int e = e0 + j;
      idx[j] = g->cols[e] * Z + (z + g->shifts[e]) % Z;
      t[j] = clamp127(L[idx[j]] - M[e * Z + z]);
      const int32_t mag = t[j] < 0 ? -t[j] : t[j];
      /* merge(acc, edge{m1=mag, m2=sat, tag=j}) */
      const int y_wins = mag < m1;
      const int32_t loser = y_wins ? m1 : mag;
      m1 = y_wins ? mag : m1;
      m2 = loser < m2 ? loser : m2;
      tag = y_wins ? j : tag;
      s ^= (t[j] < 0);
    }
    const int32_t b1 = lut[m1], b2 = lut[m2];
    for (int j = 0; j < w; ++j) {
      const int32_t mag = (tag == j) ? b2 : b1;
      const int32_t out = (s ^ (t[j] < 0)) ? -mag : mag;
      M[(e0 + j) * Z + z] = out;
      L[idx[j]] = clamp127(t[j] + out);
    }
  }
}

/* ---------------- float engines ---------------- */

static void layer_f32(const graph_t* g, float* L, float* M, float beta32, int r) {
  const int Z = g->z;
  const int e0 = g->row_start[r], w = g->row_start[r + 1] - e0;
  float t[32];
  int idx[32];
  for (int z = 0; z < Z; ++z) {
    float m1 = INFINITY, m2 = INFINITY;
    int tag = -1, s = 0;
    for (int j = 0; j < w; ++j) {
      const int e = e0 + j;
      idx[j] = g->cols[e] * Z + (z + g->shifts[e]) % Z;
      t[j] = L[idx[j]] - M[e * Z + z];
      const float mag = fabsf(t[j]);
      const int y_wins = mag < m1;
      const float loser = y_wins ? m1 : mag;
      m1 = y_wins ? mag : m1;
      m2 = loser < m2 ? loser : m2;
      tag = y_wins ? j : tag;
      s ^= (t[j] < 0.0f);
    }
    const float b1 = beta32 * m1, b2 = beta32 * m2;
    for (int j = 0; j < w; ++j) {
      const float mag = (tag == j) ? b2 : b1;
      const float out = (s ^ (t[j] < 0.0f)) ? -mag : mag;
      M[(e0 + j) * Z + z] = out;
      L[idx[j]] = t[j] + out;
    }
  }
}

typedef _Float16 h16;
static inline h16 clamp_h(h16 x) {
  const h16 hi = (h16)65504.0f, lo = (h16)-65504.0f;
  return x < lo ? lo : (x > hi ? hi : x);
}

static void layer_f16(const graph_t* g, h16* L, h16* M, h16 beta16, int r) {
  const int Z = g->z;
  const int e0 = g->row_start[r], w = g->row_start[r + 1] - e0;
  h16 t[32];
  int idx[32];
  const h16 sat = (h16)65504.0f;
  for (int z = 0; z < Z; ++z) {
    h16 m1 = sat, m2 = sat;
    int tag = -1, s = 0;
    for (int j = 0; j < w; ++j) {
      const int e = e0 + j;
      idx[j] = g->cols[e] * Z + (z + g->shifts[e]) % Z;
      h16 d = (h16)(L[idx[j]] - M[e * Z + z]); /* one float16 rounding */
      t[j] = clamp_h(d);
      const h16 mag = t[j] < (h16)0.0f ? (h16)(-t[j]) : t[j];
      const int y_wins = mag < m1;
      const h16 loser = y_wins ? m1 : mag;
      m1 = y_wins ? mag : m1;
      m2 = loser < m2 ? loser : m2;
      tag = y_wins ? j : tag;
      s ^= (t[j] < (h16)0.0f);
    }
    const h16 b1 = (h16)(beta16 * m1), b2 = (h16)(beta16 * m2);
    for (int j = 0; j < w; ++j) {
      const h16 mag = (tag == j) ? b2 : b1;
      const h16 out = (s ^ (t[j] < (h16)0.0f)) ? (h16)(-mag) : mag;
      M[(e0 + j) * Z + z] = out;
      L[idx[j]] = clamp_h((h16)(t[j] + out));
    }
  }
}

/* ---------------- flooding schedule (decoder.py:337-365) ----------------
 * Check-node update of every row from the previous posteriors (messages are
 * per row, updated in place after the row's gather), then
 * L = sat(L_b + sum over the column's edges of roll(msg_e, s_e)), summed in
 * int64 (int8) or float64 (floats) in row order, saturated once. */
static void flood_i8(const graph_t* g, int32_t* L, const int32_t* Lb, int32_t* M, const int32_t* lut) {
  const int Z = g->z;
  for (int r = 0; r < g->rows; ++r) {
    const int e0 = g->row_start[r], w = g->row_start[r + 1] - e0;
    for (int z = 0; z < Z; ++z) {
      int32_t t[32];
      int32_t m1 = 127, m2 = 127, tag = -1, s = 0;
      for (int j = 0; j < w; ++j) {
        const int e = e0 + j;
        t[j] = clamp127(L[g->cols[e] * Z + (z + g->shifts[e]) % Z] - M[e * Z + z]);
        const int32_t mag = t[j] < 0 ? -t[j] : t[j];
        const int y_wins = mag < m1;
        const int32_t loser = y_wins ? m1 : mag;
        m1 = y_wins ? mag : m1;
        m2 = loser < m2 ? loser : m2;
        tag = y_wins ? j : tag;
        s ^= (t[j] < 0);
      }
      for (int j = 0; j < w; ++j) {
        const int32_t mag = lut[(tag == j) ? m2 : m1];
        M[(e0 + j) * Z + z] = (s ^ (t[j] < 0)) ? -mag : mag;
      }
    }
  }
  for (int c = 0; c < g->n_blocks; ++c)
    for (int i = 0; i < Z; ++i) {
      int64_t acc = Lb[c * Z + i];
      for (int e = 0; e < g->n_edges; ++e)
        if (g->cols[e] == c) acc += M[e * Z + ((i - g->shifts[e]) % Z + Z) % Z];
      L[c * Z + i] = (int32_t)(acc < -127 ? -127 : (acc > 127 ? 127 : acc));
    }
}

static void flood_f32(const graph_t* g, float* L, const float* Lb, float* M, float beta32) {
  const int Z = g->z;
  for (int r = 0; r < g->rows; ++r) {
    const int e0 = g->row_start[r], w = g->row_start[r + 1] - e0;
    for (int z = 0; z < Z; ++z) {
      float t[32];
      float m1 = INFINITY, m2 = INFINITY;
      int tag = -1, s = 0;
      for (int j = 0; j < w; ++j) {
        const int e = e0 + j;
        t[j] = L[g->cols[e] * Z + (z + g->shifts[e]) % Z] - M[e * Z + z];
        const float mag = fabsf(t[j]);
        const int y_wins = mag < m1;
        const float loser = y_wins ? m1 : mag;
        m1 = y_wins ? mag : m1;
        m2 = loser < m2 ? loser : m2;
        tag = y_wins ? j : tag;
        s ^= (t[j] < 0.0f);
      }
      const float b1 = beta32 * m1, b2 = beta32 * m2;
      for (int j = 0; j < w; ++j) {
        const float mag = (tag == j) ? b2 : b1;
        M[(e0 + j) * Z + z] = (s ^ (t[j] < 0.0f)) ? -mag : mag;
      }
    }
  }
  for (int c = 0; c < g->n_blocks; ++c)
    for (int i = 0; i < Z; ++i) {
      double acc = (double)Lb[c * Z + i];
      for (int e = 0; e < g->n_edges; ++e)
        if (g->cols[e] == c) acc += (double)M[e * Z + ((i - g->shifts[e]) % Z + Z) % Z];
      L[c * Z + i] = (float)acc;
    }
}

static void flood_f16(const graph_t* g, h16* L, const h16* Lb, h16* M, h16 beta16) {
  const int Z = g->z;
  const h16 sat = (h16)65504.0f;
  for (int r = 0; r < g->rows; ++r) {
    const int e0 = g->row_start[r], w = g->row_start[r + 1] - e0;
    for (int z = 0; z < Z; ++z) {
      h16 t[32];
      h16 m1 = sat, m2 = sat;
      int tag = -1, s = 0;
      for (int j = 0; j < w; ++j) {
        const int e = e0 + j;
        h16 d = (h16)(L[g->cols[e] * Z + (z + g->shifts[e]) % Z] - M[e * Z + z]);
        t[j] = clamp_h(d);
        const h16 mag = t[j] < (h16)0.0f ? (h16)(-t[j]) : t[j];
        const int y_wins = mag < m1;
        const h16 loser = y_wins ? m1 : mag;
        m1 = y_wins ? mag : m1;
        m2 = loser < m2 ? loser : m2;
        tag = y_wins ? j : tag;
        s ^= (t[j] < (h16)0.0f);
      }
      const h16 b1 = (h16)(beta16 * m1), b2 = (h16)(beta16 * m2);
      for (int j = 0; j < w; ++j) {
        const h16 mag = (tag == j) ? b2 : b1;
        M[(e0 + j) * Z + z] = (s ^ (t[j] < (h16)0.0f)) ? (h16)(-mag) : mag;
      }
    }
  }
  for (int c = 0; c < g->n_blocks; ++c)
    for (int i = 0; i < Z; ++i) {
      double acc = (double)Lb[c * Z + i];
      for (int e = 0; e < g->n_edges; ++e)
        if (g->cols[e] == c) acc += (double)M[e * Z + ((i - g->shifts[e]) % Z + Z) % Z];
      if (acc < -65504.0) acc = -65504.0;
      if (acc > 65504.0) acc = 65504.0;
      L[c * Z + i] = (h16)acc; /* double -> half, one RNE rounding (astype) */
    }
}

/* syndrome weight and min|L| of the current posteriors; sign test is v < 0 */
#define DEF_CHECK(NAME, T, NEG, ABS)                                                \
  static void NAME(const graph_t* g, const T* L, int64_t* wgt, double* margin) {   \
    const int Z = g->z;                                                             \
    int64_t w = 0;                                                                  \
    for (int r = 0; r < g->rows; ++r) {                                             \
      const int e0 = g->row_start[r], n = g->row_start[r + 1] - e0;                 \
      for (int z = 0; z < Z; ++z) {                                                 \
        int p = 0;                                                                  \
        for (int j = 0; j < n; ++j) {                                               \
          const int e = e0 + j;                                                     \
          p ^= NEG(L[g->cols[e] * Z + (z + g->shifts[e]) % Z]);                     \
        }                                                                           \
        w += p;                                                                     \
      }                                                                             \
    }                                                                               \
    double m = INFINITY;                                                            \
    for (int i = 0; i < g->n_blocks * Z; ++i) {                                     \
      const double a = ABS(L[i]);                                                   \
      if (a < m) m = a;                                                             \
    }                                                                               \
    *wgt = w;                                                                       \
    *margin = m;                                                                    \
  }
#define NEG_I(x) ((x) < 0)
#define ABS_I(x) ((double)((x) < 0 ? -(x) : (x)))
#define NEG_F(x) ((x) < 0.0f)
#define ABS_F(x) ((double)fabsf(x))
#define NEG_H(x) ((x) < (h16)0.0f)
#define ABS_H(x) ((double)fabsf((float)(x)))
DEF_CHECK(check_i8, int32_t, NEG_I, ABS_I)
DEF_CHECK(check_f32, float, NEG_F, ABS_F)
DEF_CHECK(check_f16, h16, NEG_H, ABS_H)

typedef struct {
  uint8_t* bits;
  int64_t* iters;
  int64_t* synd;
  uint8_t* success;
  uint8_t* crc_ok;
  int32_t* trace_w;
  double* trace_m;
} outs_t;

static void decode_one(const graph_t* g, int prec, const void* llr_cw, int64_t b, const outs_t* o,
                       void* Lbuf, void* Mbuf, uint8_t* hard, void* LBbuf, int flooding) {
  const int Z = g->z, K = g->k_b * Z, NC = g->n_blocks * Z, E = g->n_edges;
  int32_t lut[128];
  for (int m = 0; m < 128; ++m) lut[m] = (int32_t)floor(g->beta * (double)m);
  const float beta32 = (float)g->beta;
  const h16 beta16 = (h16)g->beta; /* np.float16(beta): double -> half, RNE */
  if (prec == PREC_INT8) {
    int32_t* L = (int32_t*)Lbuf;
    const int8_t* in = (const int8_t*)llr_cw;
    for (int i = 0; i < NC; ++i) L[i] = in[i];
    memset(Mbuf, 0, sizeof(int32_t) * (size_t)E * Z);
  } else if (prec == PREC_F32) {
    memcpy(Lbuf, llr_cw, sizeof(float) * NC);
    memset(Mbuf, 0, sizeof(float) * (size_t)E * Z);
  } else {
    memcpy(Lbuf, llr_cw, sizeof(h16) * NC);
    memset(Mbuf, 0, sizeof(h16) * (size_t)E * Z);
  }
  if (flooding) {
    const size_t esz = prec == PREC_F16 ? 2 : 4;
    memcpy(LBbuf, Lbuf, esz * (size_t)NC);
  }
  const int tracing = o->trace_w != NULL;
  int done = 0;
  int64_t wgt = 0;
  double margin = 0.0;
  int it;
  for (it = 1; it <= g->max_iter; ++it) {
    if (flooding) {
      if (prec == PREC_INT8) flood_i8(g, (int32_t*)Lbuf, (const int32_t*)LBbuf, (int32_t*)Mbuf, lut);
      else if (prec == PREC_F32) flood_f32(g, (float*)Lbuf, (const float*)LBbuf, (float*)Mbuf, beta32);
      else flood_f16(g, (h16*)Lbuf, (const h16*)LBbuf, (h16*)Mbuf, beta16);
    } else {
      for (int r = 0; r < g->rows; ++r) {
        if (prec == PREC_INT8) layer_i8(g, (int32_t*)Lbuf, (int32_t*)Mbuf, lut, r);
        else if (prec == PREC_F32) layer_f32(g, (float*)Lbuf, (float*)Mbuf, beta32, r);
        else layer_f16(g, (h16*)Lbuf, (h16*)Mbuf, beta16, r);
      }
    }
    if (prec == PREC_INT8) check_i8(g, (const int32_t*)Lbuf, &wgt, &margin);
    else if (prec == PREC_F32) check_f32(g, (const float*)Lbuf, &wgt, &margin);
    else check_f16(g, (const h16*)Lbuf, &wgt, &margin);
    if (tracing) {
      o->trace_w[b * g->max_iter + (it - 1)] = (int32_t)wgt;
      o->trace_m[b * g->max_iter + (it - 1)] = margin;
    }
    if (g->early_stop == STOP_NONE || done) {
      if (done && !tracing) break;
      continue;
    }
    if (wgt == 0 && margin > 0.0) {
      for (int i = 0; i < K; ++i) {
        if (prec == PREC_INT8) hard[i] = ((int32_t*)Lbuf)[i] < 0;
        else if (prec == PREC_F32) hard[i] = ((float*)Lbuf)[i] < 0.0f;
        else hard[i] = ((h16*)Lbuf)[i] < (h16)0.0f;
      }
      int accept = 1;
      if (g->early_stop == STOP_CRC) {
        accept = crc_pass(hard, K, g->crc_len, g->crc_poly);
        o->crc_ok[b] = (uint8_t)accept;
      }
      if (accept) {
        memcpy(o->bits + b * K, hard, K);
        o->iters[b] = it;
        o->synd[b] = 0;
        o->success[b] = 1;
        done = 1;
        if (!tracing) break;
      }
    }
  }
  if (!done) {
    for (int i = 0; i < K; ++i) {
      if (prec == PREC_INT8) hard[i] = ((int32_t*)Lbuf)[i] < 0;
      else if (prec == PREC_F32) hard[i] = ((float*)Lbuf)[i] < 0.0f;
      else hard[i] = ((h16*)Lbuf)[i] < (h16)0.0f;
    }
    memcpy(o->bits + b * K, hard, K);
    o->iters[b] = g->max_iter;
    o->synd[b] = wgt;
    o->success[b] = (wgt == 0 && margin > 0.0);
    if (g->early_stop == STOP_CRC) {
      if (o->success[b]) {
        o->crc_ok[b] = (uint8_t)crc_pass(hard, K, g->crc_len, g->crc_poly);
        o->success[b] = o->crc_ok[b];
      } else {
        o->crc_ok[b] = 0;
      }
    }
  }
}

int oracle_decode(int precision, const void* llr, int64_t batch, int k_b, int z, int rows_used,
                  const int32_t* row_start, const int16_t* cols, const int16_t* shifts, double beta,
                  int max_iter, int early_stop, int crc_len, uint32_t crc_poly, uint8_t* bits,
                  int64_t* iters, int64_t* synd, uint8_t* success, uint8_t* crc_ok,
                  int32_t* trace_w, double* trace_m, int n_threads, int flooding) {
  graph_t g = {k_b, z, rows_used, k_b + rows_used, row_start[rows_used], row_start, cols, shifts,
               beta, max_iter, early_stop, crc_len, crc_poly};
  outs_t o = {bits, iters, synd, success, crc_ok, trace_w, trace_m};
  const size_t esz = precision == PREC_INT8 ? 4 : (precision == PREC_F32 ? 4 : 2);
  const size_t in_sz = precision == PREC_INT8 ? 1 : esz;
  const int64_t NC = (int64_t)g.n_blocks * z;
  int rc = 0;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel
#endif
  {
    void* Lbuf = malloc(esz * (size_t)NC);
    void* Mbuf = malloc(esz * (size_t)g.n_edges * z);
    void* LBbuf = malloc(esz * (size_t)NC);
    uint8_t* hard = (uint8_t*)malloc((size_t)k_b * z);
    if (!Lbuf || !Mbuf || !hard || !LBbuf) {
      rc = -3;
    } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
      for (int64_t b = 0; b < batch; ++b)
        decode_one(&g, precision, (const uint8_t*)llr + (size_t)b * NC * in_sz, b, &o, Lbuf, Mbuf, hard,
                   LBbuf, flooding);
    }
    free(LBbuf);
    free(Lbuf);
    free(Mbuf);
    free(hard);
  }
  return rc;
}

/* depuncture + quantize (channel.py:64-83), float64 in; int8 mode only */
void oracle_quantize_i8(const double* in, int64_t batch, int n_tx, int two_z, double scale,
                        int8_t* out) {
  const int n_c = n_tx + two_z;
  for (int64_t b = 0; b < batch; ++b) {
    for (int j = 0; j < n_c; ++j) {
      const double v = j < two_z ? 0.0 : in[b * n_tx + (j - two_z)];
      double s = nearbyint(v * scale); /* default rounding mode: half-to-even */
      if (s < -127.0) s = -127.0;
      if (s > 127.0) s = 127.0;
      out[b * n_c + j] = (int8_t)s;
    }
  }
}
