/*
 * moe_oracle.c — CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the MoE-layer data path that MoEless balances, used
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER.  Nothing in the product (paper_2603_06350_b200/) links, loads or
 * calls this file.
 *
 * Provenance of each piece (reference = /root/reference, arXiv 2603.06350):
 *   - keyed RNG streams ............ proj/include/moeless/rng.hpp:12-32
 *   - popularity permutation ....... proj/src/workload.cpp:30-88
 *   - route_tokens id replay ....... proj/src/workload.cpp:188-230 (same stream,
 *                                    same arithmetic, but also emits the ids)
 *   - even replica split ........... proj/src/cost_model.cpp:98-106 made integer
 *                                    (SURVEY.md §8a "integer dispatch rule")
 *   - gate / FFN / combine ......... no reference code exists (SURVEY §8a row
 *                                    a14); Mixtral conventions stated in
 *                                    softmax over E then top-k
 *                                    (== softmax over the k selected logits),
 *                                    lowest expert index wins ties, no bias, no
 *                                    token dropping, y = sum_j w_j FFN_e(x),
 *                                    FFN = (silu(x W1^T) * (x W3^T)) W2^T.
 * Parity of the route replay is PINNED against the compiled reference
 * (oracle/_ref).  Parity of gate/FFN/combine numerics is UNPINNED by the
 * reference (it has none); those are pinned by the committed golden fixtures.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG */
/* rng.hpp:12-17 */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 restated (the reference builds its streams on it). */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;

static void mt_seed(orc_mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt_next(orc_mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* rng.hpp:21-25 */
static void keyed_engine(orc_mt64* g, uint64_t seed, uint64_t a, uint64_t b, uint64_t tag) {
  mt_seed(g, orc_mix64(seed ^ orc_mix64(a ^ orc_mix64(b ^ orc_mix64(tag)))));
}

/* rng.hpp:30-32 */
static double uniform01(orc_mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

/* first n raw draws of a keyed stream — lets tests pin the MT restatement */
void orc_keyed_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag, int n, uint64_t* out) {
  orc_mt64 g;
  keyed_engine(&g, seed, a, b, tag);
  for (int i = 0; i < n; ++i) out[i] = mt_next(&g);
}

/* --------------------------------------------------------- popularity */
#define ROUTE_TAG 0x726f757465ULL /* workload.cpp:19 */
#define DRIFT_TAG 0x7065726dULL   /* workload.cpp:20 */

/* workload.cpp:30-75: base Fisher-Yates permutation per layer, re-permuted per
 * drift epoch. */
void orc_popularity_perm(int experts, uint64_t seed, int layer, long iteration, int drift_period,
                         int* perm) {
  orc_mt64 g;
  for (int i = 0; i < experts; ++i) perm[i] = i;
  keyed_engine(&g, seed, (uint64_t)layer, 0, DRIFT_TAG);
  for (int i = experts - 1; i > 0; --i) {
    int j = (int)(mt_next(&g) % (uint64_t)(i + 1));
    int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  if (drift_period > 0 && iteration / drift_period > 0) {
    long epoch = iteration / drift_period;
    keyed_engine(&g, seed, (uint64_t)epoch, (uint64_t)layer, DRIFT_TAG + 1);
    for (int i = experts - 1; i > 0; --i) {
      int j = (int)(mt_next(&g) % (uint64_t)(i + 1));
      int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
  }
}

/* workload.cpp:77-88 */
void orc_popularity_weights(int experts, double s, const int* perm, double* w) {
  double norm = 0.0;
  for (int r = 0; r < experts; ++r) norm += 1.0 / pow((double)(r + 1), s);
  for (int r = 0; r < experts; ++r) w[perm[r]] = (1.0 / pow((double)(r + 1), s)) / norm;
}

/* workload.cpp:188-230 replayed: same keyed stream, same inverse-CDF draw and
 * duplicate rejection, but the chosen expert ids are emitted per token (in
 * draw order), so their histogram equals route_tokens().loads exactly. */
int orc_route_tokens_ids(int64_t tokens, int layer, long iteration, int experts, double s,
                         uint64_t seed, int top_k, int drift_period, int32_t* ids,
                         int64_t* loads) {
  if (top_k < 1 || top_k > experts || tokens < 0) return 1;
  int* perm = (int*)malloc(sizeof(int) * experts);
  double* cum = (double*)malloc(sizeof(double) * experts);
  orc_popularity_perm(experts, seed, layer, iteration, drift_period, perm);
  double norm = 0.0;
  for (int r = 0; r < experts; ++r) {
    norm += 1.0 / pow((double)(r + 1), s);
    cum[r] = norm;
  }
  if (loads) memset(loads, 0, sizeof(int64_t) * experts);
  orc_mt64 g;
  keyed_engine(&g, seed, (uint64_t)iteration, (uint64_t)layer, ROUTE_TAG);
  for (int64_t t = 0; t < tokens; ++t) {
    int chosen = 0;
    int32_t* picked = ids + t * top_k;
    while (chosen < top_k) {
      double u = uniform01(&g) * norm;
      int lo = 0, hi = experts; /* lower_bound */
      while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (cum[mid] < u) lo = mid + 1; else hi = mid;
      }
      int e = perm[lo < experts - 1 ? lo : experts - 1];
      int dup = 0;
      for (int c = 0; c < chosen; ++c) if (picked[c] == e) dup = 1;
      if (dup) continue;
      picked[chosen++] = e;
      if (loads) ++loads[e];
    }
  }
  free(perm);
  free(cum);
  return 0;
}

/* ------------------------------------------------------------- bf16 */
static inline float bf2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f2bf(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
uint16_t orc_f2bf(float f) { return f2bf(f); }

/* ------------------------------------------------ synthetic layer inputs */
/* Counter-based streams (DESIGN.md §"Synthetic inputs"): value i of stream
 * `key` is r = mix64(key ^ (i * K)).  Restated independently of the product
 * so that the product's generator is itself checked. */
#define SYN_K 0xD1B54A32D192ED03ULL
static inline uint64_t syn(uint64_t key, uint64_t i) { return orc_mix64(key ^ (i * SYN_K)); }

uint64_t orc_stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag) {
  return orc_mix64(seed ^ orc_mix64(a ^ orc_mix64(b ^ orc_mix64(tag))));
}

static int gumbel_q16(uint64_t r) {
  double u = ((double)(r >> 11) + 0.5) * 0x1.0p-53;
  double g = -log(-log(u));
  long q = lrint(g * 16.0);
  if (q > 255) q = 255;
  if (q < -255) q = -255;
  return (int)q;
}

/* Token activations x[T, d] (bf16): column 0 is the constant-1 bias feature,
 * columns 1..E carry Gumbel noise on the 1/16 grid, the rest are q/16 with
 * |q| <= 16.  Every value is exact in bf16. */
void orc_synth_tokens(uint64_t key, int64_t t0, int64_t tokens, int d, int experts, uint16_t* x) {
  for (int64_t t = 0; t < tokens; ++t) {
    uint16_t* row = x + t * d;
    int64_t gt = t0 + t;
    for (int c = 0; c < d; ++c) {
      uint64_t r = syn(key, (uint64_t)(gt * d + c));
      float v;
      if (c == 0) v = 1.0f;
      else if (c <= experts) v = (float)gumbel_q16(r) / 16.0f;
      else v = (float)((int)(r % 33) - 16) / 16.0f;
      row[c] = f2bf(v);
    }
  }
}

/* Gate weights Wg[E, d] (bf16, nn.Linear layout): column 0 carries the Zipf
 * log-popularity rounded to 1/16, column 1+noise_perm[e] is 1 (so logit_e
 * gets its own iid Gumbel feature), bulk columns are q/4096, |q| <= 16.
 * Gumbel-top-k of log w + G samples k experts without replacement with
 * probabilities proportional to w — the distribution route_tokens draws. */
void orc_synth_gate(uint64_t key, int d, int experts, const double* pop_w, const int* noise_perm,
                    uint16_t* wg) {
  for (int e = 0; e < experts; ++e) {
    uint16_t* row = wg + (int64_t)e * d;
    for (int c = 0; c < d; ++c) {
      float v;
      if (c == 0) {
        long q = lrint(log(pop_w[e]) * 16.0);
        if (q < -255) q = -255;
        v = (float)q / 16.0f;
      } else if (c <= experts) {
        v = (c - 1 == noise_perm[e]) ? 1.0f : 0.0f;
      } else {
        uint64_t r = syn(key, (uint64_t)((int64_t)e * d + c));
        v = (float)((int)(r % 33) - 16) / 4096.0f;
      }
      row[c] = f2bf(v);
    }
  }
}

/* Expert weights, nn.Linear layout: W1,W3 [ff, d], W2 [d, ff]; entries are
 * bf16(q/64 * scale) with q uniform in [-64, 64] and scale 1/sqrt(fan_in). */
void orc_synth_expert(uint64_t key, int d, int ff, uint16_t* w1, uint16_t* w3, uint16_t* w2) {
  const float s1 = 1.0f / sqrtf((float)d), s2 = 1.0f / sqrtf((float)ff);
  const int64_t n = (int64_t)d * ff;
  for (int64_t i = 0; i < n; ++i) {
    w1[i] = f2bf((float)((int)(syn(key, (uint64_t)i) % 129) - 64) / 64.0f * s1);
    w3[i] = f2bf((float)((int)(syn(key, (uint64_t)(n + i)) % 129) - 64) / 64.0f * s1);
    w2[i] = f2bf((float)((int)(syn(key, (uint64_t)(2 * n + i)) % 129) - 64) / 64.0f * s2);
  }
}

/* ----------------------------------------------------------- gate (K1) */
/* logits = x Wg^T in fp32 (exact for the synthetic grid); top-k by repeated
 * argmax with strict '>' so the lowest expert index wins ties; weights =
 * softmax over the k selected logits (== softmax over E, top-k, renormalise);
 * counts = per-expert histogram. */
void orc_gate(const uint16_t* x, int64_t tokens, int d, const uint16_t* wg, int experts, int top_k,
              int32_t* ids, float* w, int32_t* counts, float* logits_out) {
  float* logit = (float*)malloc(sizeof(float) * experts);
  int* used = (int*)malloc(sizeof(int) * experts);
  memset(counts, 0, sizeof(int32_t) * experts);
  for (int64_t t = 0; t < tokens; ++t) {
    const uint16_t* xr = x + t * d;
    for (int e = 0; e < experts; ++e) {
      const uint16_t* wr = wg + (int64_t)e * d;
      float acc = 0.0f;
      for (int c = 0; c < d; ++c) acc += bf2f(xr[c]) * bf2f(wr[c]);
      logit[e] = acc;
      used[e] = 0;
      if (logits_out) logits_out[t * experts + e] = acc;
    }
    float sel[64];
    for (int j = 0; j < top_k; ++j) {
      int best = -1;
      for (int e = 0; e < experts; ++e)
        if (!used[e] && (best < 0 || logit[e] > logit[best])) best = e;
      used[best] = 1;
      ids[t * top_k + j] = best;
      sel[j] = logit[best];
      counts[best]++;
    }
    float m = sel[0], z = 0.0f;
    for (int j = 0; j < top_k; ++j) { sel[j] = expf(sel[j] - m); z += sel[j]; }
    for (int j = 0; j < top_k; ++j) w[t * top_k + j] = sel[j] / z;
  }
  free(logit);
  free(used);
}

/* The batched predictor MLP (moe_set_predictor_mlp; the learned stand-in
 * for LayerAwarePredictor::predict's scoring, predictor.cpp:38-62):
 * hidden_j = relu(x . W1_j) (E units, fp32 dot products as in orc_gate),
 * out_e = fmaf chain over j ascending of W2[e][j] * hidden_j from 0, then
 * top-k of out with the same lowest-index tie rule; counts = histogram. */
void orc_predict_mlp(const uint16_t* x, int64_t tokens, int d, const uint16_t* w1, int experts,
                     const float* w2, int top_k, int32_t* counts) {
  float* h = (float*)malloc(sizeof(float) * experts);
  float* out = (float*)malloc(sizeof(float) * experts);
  int* used = (int*)malloc(sizeof(int) * experts);
  memset(counts, 0, sizeof(int32_t) * experts);
  for (int64_t t = 0; t < tokens; ++t) {
    const uint16_t* xr = x + t * d;
    for (int j = 0; j < experts; ++j) {
      const uint16_t* wr = w1 + (int64_t)j * d;
      float acc = 0.0f;
      for (int c = 0; c < d; ++c) acc += bf2f(xr[c]) * bf2f(wr[c]);
      h[j] = acc > 0.0f ? acc : 0.0f;
    }
    for (int e = 0; e < experts; ++e) {
      float acc = 0.0f;
      for (int j = 0; j < experts; ++j) acc = fmaf(w2[(int64_t)e * experts + j], h[j], acc);
      out[e] = acc;
      used[e] = 0;
    }
    for (int j = 0; j < top_k; ++j) {
      int best = -1;
      for (int e = 0; e < experts; ++e)
        if (!used[e] && (best < 0 || out[e] > out[best])) best = e;
      used[best] = 1;
      counts[best]++;
    }
  }
  free(h);
  free(out);
  free(used);
}

/* ----------------------------------------------------- dispatch (K3/K6) */
/* Integer replica split (cost_model.cpp:98-106 made integer):
 * expert e's n_e assignments, ordered by (source rank, token index), are cut
 * into R_e contiguous ranges; replica r takes floor(n/R) + [r < n mod R].
 * Every rank lays out its received rows as segments ordered by (expert,
 * ordinal) over the replicas placed on it; inside a segment rows keep the
 * global order.
 *
 * Inputs: ids of every source rank (ids_all[src] -> [T_src, k]), tokens[src],
 * replica_counts[E], replica_gpu[sum R] (flattened (e, r)).
 * Outputs for every (src, t, j): dest_gpu and dest_row (row in dest's receive
 * layout); per gpu: seg_start/seg_rows indexed by flat replica id (or -1 /0 if
 * not on that gpu) and rows_on_gpu[G]. */
int orc_dispatch(int ranks, const int32_t* const* ids_all, const int64_t* tokens, int top_k,
                 int experts, const int32_t* replica_counts, const int32_t* replica_gpu,
                 int32_t* const* dest_gpu, int64_t* const* dest_row, int64_t* seg_start,
                 int64_t* seg_rows, int64_t* rows_on_gpu) {
  int64_t* n_src = (int64_t*)calloc((size_t)ranks * experts, sizeof(int64_t));
  int64_t* n_tot = (int64_t*)calloc((size_t)experts, sizeof(int64_t));
  int* rep_base = (int*)malloc(sizeof(int) * (experts + 1));
  rep_base[0] = 0;
  for (int e = 0; e < experts; ++e) rep_base[e + 1] = rep_base[e] + replica_counts[e];
  const int total_rep = rep_base[experts];
  for (int s = 0; s < ranks; ++s)
    for (int64_t i = 0; i < tokens[s] * top_k; ++i) {
      int e = ids_all[s][i];
      if (e < 0 || e >= experts) { free(n_src); free(n_tot); free(rep_base); return 1; }
      n_src[(size_t)s * experts + e]++;
      n_tot[e]++;
    }
  /* segment layout per gpu: (expert, ordinal) order */
  int64_t* fill = (int64_t*)calloc((size_t)ranks, sizeof(int64_t));
  for (int e = 0; e < experts; ++e) {
    int64_t n = n_tot[e], R = replica_counts[e], q = n / R, rem = n % R;
    for (int r = 0; r < R; ++r) {
      int f = rep_base[e] + r;
      int g = replica_gpu[f];
      seg_rows[f] = q + (r < rem ? 1 : 0);
      seg_start[f] = fill[g];
      fill[g] += seg_rows[f];
    }
  }
  for (int g = 0; g < ranks; ++g) rows_on_gpu[g] = fill[g];
  /* per-assignment destination */
  int64_t* run = (int64_t*)calloc((size_t)experts, sizeof(int64_t));
  for (int s = 0; s < ranks; ++s) {
    for (int e = 0; e < experts; ++e) {
      int64_t off = 0;
      for (int p = 0; p < s; ++p) off += n_src[(size_t)p * experts + e];
      run[e] = off;
    }
    for (int64_t i = 0; i < tokens[s] * top_k; ++i) {
      int e = ids_all[s][i];
      int64_t gr = run[e]++;
      int64_t n = n_tot[e], R = replica_counts[e], q = n / R, rem = n % R;
      int64_t r, start;
      if (gr < rem * (q + 1)) { r = gr / (q + 1); start = r * (q + 1); }
      else { r = rem + (gr - rem * (q + 1)) / q; start = rem * (q + 1) + (r - rem) * q; }
      int f = rep_base[e] + (int)r;
      dest_gpu[s][i] = replica_gpu[f];
      dest_row[s][i] = seg_start[f] + (gr - start);
    }
  }
  (void)total_rep;
  free(run); free(fill); free(n_src); free(n_tot); free(rep_base);
  return 0;
}

/* ------------------------------------------------------- expert FFN (K4) */
/* Y[r] = W2 (silu(W1 x_r) * (W3 x_r)) for rows [0, rows) of one segment, fp32
 * accumulate.  round_h mirrors the device's bf16 intermediate; round_y rounds
 * the output to bf16 values (kept in float). */
void orc_expert_ffn(const uint16_t* x, int64_t rows, int d, int ff, const uint16_t* w1,
                    const uint16_t* w3, const uint16_t* w2, int round_h, int round_y, float* y) {
  float* h = (float*)malloc(sizeof(float) * (size_t)rows * ff);
#pragma omp parallel for schedule(static)
  for (int f = 0; f < ff; ++f) {
    const uint16_t* a = w1 + (int64_t)f * d;
    const uint16_t* b = w3 + (int64_t)f * d;
    for (int64_t r = 0; r < rows; ++r) {
      const uint16_t* xr = x + r * d;
      float g = 0.0f, u = 0.0f;
#pragma omp simd reduction(+ : g, u)
      for (int c = 0; c < d; ++c) {
        float xv = bf2f(xr[c]);
        g += xv * bf2f(a[c]);
        u += xv * bf2f(b[c]);
      }
      float hv = g / (1.0f + expf(-g)) * u;
      h[r * ff + f] = round_h ? bf2f(f2bf(hv)) : hv;
    }
  }
#pragma omp parallel for schedule(static)
  for (int n = 0; n < d; ++n) {
    const uint16_t* wr = w2 + (int64_t)n * ff;
    for (int64_t r = 0; r < rows; ++r) {
      const float* hr = h + r * ff;
      float acc = 0.0f;
#pragma omp simd reduction(+ : acc)
      for (int f = 0; f < ff; ++f) acc += hr[f] * bf2f(wr[f]);
      y[r * d + n] = round_y ? bf2f(f2bf(acc)) : acc;
    }
  }
  free(h);
}

/* ----------------------------------------------------------- combine (K5) */
/* y_t = sum_j w[t,j] * Y[row(t,j)], fp32 in slot order j = 0..k-1. */
void orc_combine(const float* Y, int d, const int64_t* rows, const float* w, int64_t tokens,
                 int top_k, float* y) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < tokens; ++t) {
    float* out = y + t * d;
    for (int c = 0; c < d; ++c) out[c] = 0.0f;
    for (int j = 0; j < top_k; ++j) {
      const float* src = Y + rows[t * top_k + j] * d;
      float wj = w[t * top_k + j];
      for (int c = 0; c < d; ++c) out[c] += wj * src[c];
    }
  }
}

/* ----------------------------------------------- whole layer, one rank */
/* gate -> dispatch (G = 1) -> FFN per segment -> combine.  weights are given
 * per expert (replicas on one GPU share their expert's weights).  Used for the
 * bench's cpu_baseline ("port") and for the end-to-end parity test. */
int orc_layer_forward(const uint16_t* x, int64_t tokens, int d, int ff, int experts, int top_k,
                      const uint16_t* wg, const uint16_t* const* w1, const uint16_t* const* w3,
                      const uint16_t* const* w2, const int32_t* replica_counts, int round_h,
                      float* y, int32_t* ids_out, float* w_out, int32_t* counts_out) {
  int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * tokens * top_k);
  float* w = (float*)malloc(sizeof(float) * tokens * top_k);
  int32_t* counts = (int32_t*)malloc(sizeof(int32_t) * experts);
  orc_gate(x, tokens, d, wg, experts, top_k, ids, w, counts, NULL);
  int total_rep = 0;
  for (int e = 0; e < experts; ++e) total_rep += replica_counts[e];
  int32_t* rgpu = (int32_t*)calloc((size_t)total_rep, sizeof(int32_t));
  int32_t* dgpu = (int32_t*)malloc(sizeof(int32_t) * tokens * top_k);
  int64_t* drow = (int64_t*)malloc(sizeof(int64_t) * tokens * top_k);
  int64_t* sstart = (int64_t*)malloc(sizeof(int64_t) * total_rep);
  int64_t* srows = (int64_t*)malloc(sizeof(int64_t) * total_rep);
  int64_t rows_total = 0;
  const int32_t* ids_c = ids;
  int rc = orc_dispatch(1, &ids_c, &tokens, top_k, experts, replica_counts, rgpu, &dgpu, &drow,
                        sstart, srows, &rows_total);
  if (rc) return rc;
  uint16_t* xp = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)rows_total * d);
  for (int64_t i = 0; i < tokens * top_k; ++i)
    memcpy(xp + drow[i] * d, x + (i / top_k) * d, sizeof(uint16_t) * d);
  float* Y = (float*)malloc(sizeof(float) * (size_t)rows_total * d);
  int f = 0;
  for (int e = 0; e < experts; ++e)
    for (int r = 0; r < replica_counts[e]; ++r, ++f)
      if (srows[f] > 0)
        orc_expert_ffn(xp + sstart[f] * d, srows[f], d, ff, w1[e], w3[e], w2[e], round_h, round_h,
                       Y + sstart[f] * d);
  orc_combine(Y, d, drow, w, tokens, top_k, y);
  if (ids_out) memcpy(ids_out, ids, sizeof(int32_t) * tokens * top_k);
  if (w_out) memcpy(w_out, w, sizeof(float) * tokens * top_k);
  if (counts_out) memcpy(counts_out, counts, sizeof(int32_t) * experts);
  free(ids); free(w); free(counts); free(rgpu); free(dgpu); free(drow); free(sstart);
  free(srows); free(xp); free(Y);
  return 0;
}
