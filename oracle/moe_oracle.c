/*
 * moe_oracle.c -- plain-C restatement of the reference CPU layer.
 * TEST INFRASTRUCTURE ONLY (see moe_oracle.h).  Parity: PINNED (golden vector,
 * reference hand cases, and bit-for-bit against oracle/_ref).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared moe_oracle.c -lm
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#include "moe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */

/* include/sparsekit/rng.hpp:20-25 -- state += golden gamma, then the
 * three-step xor-shift/multiply avalanche. */
uint64_t ork_splitmix_next(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

/* rng.hpp:31-34 (next_symmetric) applied over a buffer, model.cpp:20-24.
 * draw_offset skips that many draws: the state is linear in the draw index,
 * so a matrix deep inside the stream can be produced without the prefix. */
void ork_fill_symmetric(float *dst, uint64_t count, uint64_t seed, uint64_t draw_offset,
                        float scale) {
  uint64_t st = seed + draw_offset * 0x9E3779B97F4A7C15ull;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t r = ork_splitmix_next(&st);
    const float u = (float)(r >> 40) * 0x1.0p-24f;
    dst[i] = (2.0f * u - 1.0f) * scale;
  }
}

/* rng.hpp:28 (next_unit), :42-55 (next_gaussian), model.cpp:168-178. */
void ork_fill_gaussian(float *dst, uint64_t count, uint64_t seed) {
  uint64_t st = seed;
  int have_spare = 0;
  double spare = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    double g;
    if (have_spare) {
      have_spare = 0;
      g = spare;
    } else {
      double u1 = (double)(ork_splitmix_next(&st) >> 11) * 0x1.0p-53;
      const double u2 = (double)(ork_splitmix_next(&st) >> 11) * 0x1.0p-53;
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      const double radius = sqrt(-2.0 * log(u1));
      const double angle = 2.0 * 3.14159265358979323846 * u2;
      spare = radius * sin(angle);
      have_spare = 1;
      g = radius * cos(angle);
    }
    dst[i] = (float)g;
  }
}

/* model.cpp:129-166 fill order: router, then per expert gate/up/down_t, then
 * shared gate/up/down_t; one draw per element. */
uint64_t ork_synth_offset_router(const ork_config *c) {
  (void)c;
  return 0;
}
uint64_t ork_synth_offset_expert(const ork_config *c, int e, int which) {
  const uint64_t nd = (uint64_t)c->d_ffn * (uint64_t)c->d_model;
  return (uint64_t)c->n_experts * (uint64_t)c->d_model + ((uint64_t)e * 3u + (uint64_t)which) * nd;
}
uint64_t ork_synth_offset_shared(const ork_config *c, int which) {
  const uint64_t sd = (uint64_t)c->d_shared * (uint64_t)c->d_model;
  return ork_synth_offset_expert(c, c->n_experts, 0) + (uint64_t)which * sd;
}

void ork_round_bf16(float *v, uint64_t count) {
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t bits;
    memcpy(&bits, &v[i], 4);
    if ((bits & 0x7f800000u) != 0x7f800000u) {
      bits += 0x7fffu + ((bits >> 16) & 1u);
    }
    bits &= 0xffff0000u;
    memcpy(&v[i], &bits, 4);
  }
}

/* model.cpp:113-127 */
int ork_config_validate(const ork_config *c) {
  if (c->n_experts < 1) return ORK_ECONFIG;
  if (c->top_k < 1 || c->top_k > c->n_experts) return ORK_ECONFIG;
  if (c->d_model < 1 || c->d_ffn < 1 || c->d_shared < 0) return ORK_ECONFIG;
  if ((c->has_shared != 0) != (c->d_shared > 0)) return ORK_ECONFIG;
  if (c->align_block < 1) return ORK_ECONFIG;
  return ORK_OK;
}

/* --------------------------------------------------------------- linalg */

/* linalg.cpp:10-20 */
float ork_dot(const float *a, const float *b, int n) {
  float acc = 0.0f;
  for (int i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

/* linalg.cpp:22-40 */
void ork_matvec(const float *w, int rows, int cols, const float *x, float *y) {
  for (int r = 0; r < rows; ++r) y[r] = ork_dot(w + (size_t)r * cols, x, cols);
}

/* linalg.cpp:56-81: y[d] += w_t[idx[k]][d] * h[k], k outer & ascending. */
int ork_gathered_matvec_t(const float *w_t, int rows, int cols, const int32_t *idx, const float *h,
                          int m, float *y) {
  for (int d = 0; d < cols; ++d) y[d] = 0.0f;
  for (int k = 0; k < m; ++k) {
    const int32_t r = idx[k];
    if (r < 0 || r >= rows) return ORK_EINDEX;
    const float *row = w_t + (size_t)r * cols;
    const float hk = h[k];
    for (int d = 0; d < cols; ++d) y[d] += row[d] * hk;
  }
  return ORK_OK;
}

/* --------------------------------------------------------------- router */

/* router.cpp:13-68.  Softmax with max subtraction, ascending-sum denominator,
 * then the K best by (probability descending, id ascending). */
int ork_route(const float *logits, int batch, int n_experts, int top_k, int renorm, int32_t *ids,
              float *weights) {
  if (batch < 1) return ORK_ESHAPE;
  if (top_k < 1 || top_k > n_experts) return ORK_ECONFIG;
  float *p = (float *)malloc(sizeof(float) * (size_t)n_experts);
  uint8_t *taken = (uint8_t *)malloc((size_t)n_experts);
  for (int t = 0; t < batch; ++t) {
    const float *row = logits + (size_t)t * n_experts;
    float mx = row[0];
    for (int e = 1; e < n_experts; ++e) mx = row[e] > mx ? row[e] : mx;
    float denom = 0.0f;
    for (int e = 0; e < n_experts; ++e) {
      p[e] = expf(row[e] - mx);
      denom += p[e];
    }
    for (int e = 0; e < n_experts; ++e) p[e] /= denom;

    memset(taken, 0, (size_t)n_experts);
    float picked_sum = 0.0f;
    for (int s = 0; s < top_k; ++s) {
      int best = -1;
      for (int e = 0; e < n_experts; ++e) {
        if (taken[e]) continue;
        if (best < 0 || p[e] > p[best]) best = e; /* strict > keeps the lower id on ties */
      }
      taken[best] = 1;
      ids[(size_t)t * top_k + s] = best;
      picked_sum += p[best];
    }
    for (int s = 0; s < top_k; ++s) {
      const float pe = p[ids[(size_t)t * top_k + s]];
      weights[(size_t)t * top_k + s] = renorm ? pe / picked_sum : pe;
    }
  }
  free(p);
  free(taken);
  return ORK_OK;
}

/* router.cpp:70-107.  Flat slots i = t*K+s bucketed by expert in ascending i,
 * experts ascending, each bucket padded with -1 to a multiple of `block`. */
int ork_align_dispatch(const int32_t *ids, int batch, int top_k, int n_experts, int block,
                       int32_t *sorted_out, int32_t *expert_of_block, int32_t *n_padded,
                       int32_t *n_blocks) {
  if (block < 1) return ORK_ECONFIG;
  const int flat = batch * top_k;
  int32_t *count = (int32_t *)calloc((size_t)n_experts, sizeof(int32_t));
  for (int i = 0; i < flat; ++i) {
    if (ids[i] < 0 || ids[i] >= n_experts) {
      free(count);
      return ORK_EINDEX;
    }
    count[ids[i]]++;
  }
  int32_t *start = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_experts);
  int32_t pos = 0, blocks = 0;
  for (int e = 0; e < n_experts; ++e) {
    start[e] = pos;
    if (count[e] == 0) continue;
    const int32_t padded = (count[e] + block - 1) / block * block;
    for (int32_t j = count[e]; j < padded; ++j) sorted_out[pos + j] = ORK_PAD_INDEX;
    for (int32_t b = 0; b < padded / block; ++b) expert_of_block[blocks++] = e;
    pos += padded;
  }
  for (int i = 0; i < flat; ++i) sorted_out[start[ids[i]]++] = i;
  *n_padded = pos;
  *n_blocks = blocks;
  free(count);
  free(start);
  return ORK_OK;
}

/* router.cpp:109-132 */
void ork_combine(const float *slot_outputs, const float *weights, int batch, int top_k, int d_model,
                 float *y) {
  for (int t = 0; t < batch; ++t) {
    float *dst = y + (size_t)t * d_model;
    for (int d = 0; d < d_model; ++d) dst[d] = 0.0f;
    for (int s = 0; s < top_k; ++s) {
      const float wt = weights[(size_t)t * top_k + s];
      const float *src = slot_outputs + ((size_t)t * top_k + s) * d_model;
      for (int d = 0; d < d_model; ++d) dst[d] += wt * src[d];
    }
  }
}

/* ----------------------------------------------------------- activation */

/* activation.cpp:15 */
float ork_silu(float x) { return x / (1.0f + expf(-x)); }

/* activation.cpp:17-29 */
void ork_swiglu_rows(const float *gate_out, const float *up_out, int n, float *h) {
  for (int i = 0; i < n; ++i) h[i] = ork_silu(gate_out[i]) * up_out[i];
}

/* activation.cpp:57-58: round-half-up of s*n in double, clamped to [0,n]. */
int ork_n_off(double s, int n) {
  long raw = (long)floor(s * (double)n + 0.5);
  if (raw < 0) raw = 0;
  if (raw > n) raw = n;
  return (int)raw;
}

typedef struct {
  float mag;
  int32_t idx;
} ork_mag_idx;

static int ork_cmp_mag_idx(const void *pa, const void *pb) {
  const ork_mag_idx *a = (const ork_mag_idx *)pa, *b = (const ork_mag_idx *)pb;
  if (a->mag < b->mag) return -1;
  if (b->mag < a->mag) return 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}

/* activation.cpp:31-52.  A stable sort on |h| over the identity permutation is
 * the lexicographic order (|h|, index); the first `count` entries are cleared. */
void ork_mask_smallest(const float *h, int n, int count, uint8_t *mask) {
  if (count <= 0) {
    memset(mask, 1, (size_t)n);
    return;
  }
  if (count >= n) {
    memset(mask, 0, (size_t)n);
    return;
  }
  ork_mag_idx *order = (ork_mag_idx *)malloc(sizeof(ork_mag_idx) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    order[i].mag = fabsf(h[i]);
    order[i].idx = i;
  }
  qsort(order, (size_t)n, sizeof(ork_mag_idx), ork_cmp_mag_idx);
  memset(mask, 1, (size_t)n);
  for (int k = 0; k < count; ++k) mask[order[k].idx] = 0;
  free(order);
}

/* activation.cpp:54-60 (+ SparsityLevel range check, activation.hpp:18-22) */
int ork_topk_mask(const float *h, int n, double s, uint8_t *mask) {
  if (!(s >= 0.0 && s <= 1.0)) return ORK_ECONFIG;
  ork_mask_smallest(h, n, ork_n_off(s, n), mask);
  return ORK_OK;
}

/* activation.cpp:62-72 */
int ork_threshold_mask(const float *gate_out, int n, float threshold, uint8_t *mask) {
  if (!(threshold >= 0.0f)) return ORK_ECONFIG;
  for (int i = 0; i < n; ++i) mask[i] = fabsf(ork_silu(gate_out[i])) >= threshold ? 1 : 0;
  return ORK_OK;
}

/* activation.cpp:74-77 */
int ork_default_capacity(int top_k, int d_ffn) { return (top_k * d_ffn + 31) / 32 * 32; }

/* activation.cpp:79-114 */
int ork_compact_active(const uint8_t *masks, const int32_t *topk_ids, int n_slots, int d_ffn,
                       int capacity, int32_t *flat, int32_t *active_per_slot,
                       int32_t *total_active) {
  if (capacity < 0) return ORK_ECONFIG;
  for (int i = 0; i < capacity; ++i) flat[i] = ORK_PAD_INDEX;
  int32_t write_base = 0;
  for (int s = 0; s < n_slots; ++s) {
    const uint8_t *m = masks + (size_t)s * d_ffn;
    int32_t seen = 0;
    for (int i = 0; i < d_ffn; ++i) {
      if (!m[i]) continue;
      if (write_base + seen < capacity) flat[write_base + seen] = topk_ids[s] * d_ffn + i;
      ++seen;
    }
    const int32_t room = capacity - write_base;
    const int32_t kept = seen < room ? seen : room;
    active_per_slot[s] = kept;
    write_base += kept;
  }
  *total_active = write_base;
  return ORK_OK;
}

/* ---------------------------------------------------------------- layer */

static void ork_router_logits(const ork_weights *w, const float *x, int batch, float *logits) {
  /* engine.cpp:43-53 */
  for (int t = 0; t < batch; ++t)
    ork_matvec(w->router, w->cfg.n_experts, w->cfg.d_model, x + (size_t)t * w->cfg.d_model,
               logits + (size_t)t * w->cfg.n_experts);
}

/* profiler.cpp:101-150 */
int ork_build_topk_masks(const ork_weights *w, const float *x, int batch, double s, int mode,
                         uint8_t *routed_masks, uint8_t *shared_masks) {
  const ork_config *c = &w->cfg;
  if (!(s >= 0.0 && s <= 1.0)) return ORK_ECONFIG;
  const int E = c->n_experts, K = c->top_k, D = c->d_model, N = c->d_ffn, S = c->d_shared;
  float *logits = (float *)malloc(sizeof(float) * (size_t)batch * E);
  int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)batch * K);
  float *wts = (float *)malloc(sizeof(float) * (size_t)batch * K);
  ork_router_logits(w, x, batch, logits);
  int rc = ork_route(logits, batch, E, K, c->renormalize, ids, wts);
  const int widest = N > S ? N : S;
  float *g = (float *)malloc(sizeof(float) * (size_t)widest * 3);
  float *u = g + widest, *h = u + widest;
  for (int t = 0; rc == ORK_OK && t < batch; ++t) {
    const float *xt = x + (size_t)t * D;
    for (int slot = 0; slot < K; ++slot) {
      const size_t e = (size_t)ids[(size_t)t * K + slot];
      ork_matvec(w->gate + e * N * D, N, D, xt, g);
      ork_matvec(w->up + e * N * D, N, D, xt, u);
      ork_swiglu_rows(g, u, N, h);
      ork_topk_mask(h, N, s, routed_masks + ((size_t)t * K + slot) * N);
    }
    if (mode == 1 && c->has_shared && shared_masks) {
      ork_matvec(w->shared_gate, S, D, xt, g);
      ork_matvec(w->shared_up, S, D, xt, u);
      ork_swiglu_rows(g, u, S, h);
      ork_topk_mask(h, S, s, shared_masks + (size_t)t * S);
    }
  }
  free(g);
  free(wts);
  free(ids);
  free(logits);
  return rc;
}

/* engine.cpp:55-84 */
static void ork_add_shared(const ork_weights *w, const float *x, int batch,
                           const uint8_t *shared_masks, float *y, float *h_shared_out,
                           uint64_t *other_macs) {
  const ork_config *c = &w->cfg;
  if (!c->has_shared) return;
  const int D = c->d_model, S = c->d_shared;
  float *g = (float *)malloc(sizeof(float) * ((size_t)S * 3 + D));
  float *u = g + S, *h = u + S, *contrib = h + S;
  int32_t *all = (int32_t *)malloc(sizeof(int32_t) * (size_t)S);
  for (int i = 0; i < S; ++i) all[i] = i;
  for (int t = 0; t < batch; ++t) {
    const float *xt = x + (size_t)t * D;
    ork_matvec(w->shared_gate, S, D, xt, g);
    ork_matvec(w->shared_up, S, D, xt, u);
    ork_swiglu_rows(g, u, S, h);
    if (h_shared_out) memcpy(h_shared_out + (size_t)t * S, h, sizeof(float) * (size_t)S);
    if (shared_masks)
      for (int i = 0; i < S; ++i)
        if (!shared_masks[(size_t)t * S + i]) h[i] = 0.0f;
    ork_gathered_matvec_t(w->shared_down_t, S, D, all, h, S, contrib);
    for (int d = 0; d < D; ++d) y[(size_t)t * D + d] += contrib[d];
    *other_macs += 3ull * (uint64_t)S * (uint64_t)D;
  }
  free(all);
  free(g);
}

/* engine.cpp:94-191 (forward_dense_impl).  Per-slot results do not depend on
 * the dispatch-plan visiting order, so slots are visited directly. */
int ork_forward_masked(const ork_weights *w, const float *x, int batch, const uint8_t *routed_masks,
                       const uint8_t *shared_masks, float *y, ork_report *rep, int32_t *ids_out,
                       float *weights_out, float *h_routed_out, float *h_shared_out) {
  const ork_config *c = &w->cfg;
  int rc = ork_config_validate(c);
  if (rc != ORK_OK) return rc;
  const int E = c->n_experts, K = c->top_k, D = c->d_model, N = c->d_ffn;
  float *logits = (float *)malloc(sizeof(float) * (size_t)batch * E);
  int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)batch * K);
  float *wts = (float *)malloc(sizeof(float) * (size_t)batch * K);
  ork_router_logits(w, x, batch, logits);
  rc = ork_route(logits, batch, E, K, c->renormalize, ids, wts);
  if (rc != ORK_OK) {
    free(logits);
    free(ids);
    free(wts);
    return rc;
  }
  float *slot_out = (float *)malloc(sizeof(float) * (size_t)batch * K * D);
  float *g = (float *)malloc(sizeof(float) * (size_t)N * 3);
  float *u = g + N, *h = u + N;
  int32_t *all = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  for (int i = 0; i < N; ++i) all[i] = i;

  uint64_t active = 0;
  for (int t = 0; t < batch; ++t) {
    const float *xt = x + (size_t)t * D;
    for (int s = 0; s < K; ++s) {
      const size_t slot = (size_t)t * K + s;
      const size_t e = (size_t)ids[slot];
      ork_matvec(w->gate + e * N * D, N, D, xt, g);
      ork_matvec(w->up + e * N * D, N, D, xt, u);
      ork_swiglu_rows(g, u, N, h);
      if (h_routed_out) memcpy(h_routed_out + slot * N, h, sizeof(float) * (size_t)N);
      if (routed_masks) {
        const uint8_t *m = routed_masks + slot * N;
        for (int n = 0; n < N; ++n) {
          if (!m[n]) h[n] = 0.0f;
          else ++active;
        }
      }
      ork_gathered_matvec_t(w->down_t + e * N * D, N, D, all, h, N, slot_out + slot * D);
    }
  }
  ork_combine(slot_out, wts, batch, K, D, y);

  uint64_t other = (uint64_t)batch * (uint64_t)E * (uint64_t)D;
  ork_add_shared(w, x, batch, shared_masks, y, h_shared_out, &other);

  if (rep) {
    const uint64_t routed = (uint64_t)batch * K * (uint64_t)N;
    memset(rep, 0, sizeof(*rep));
    rep->gate_macs = rep->up_macs = rep->down_macs = routed * (uint64_t)D;
    rep->other_macs = other;
    rep->active_neurons_total = routed_masks ? active : routed;
    rep->achieved_routed_sparsity = 1.0 - (double)rep->active_neurons_total / (double)routed;
    rep->path_used = 0;
  }
  if (ids_out) memcpy(ids_out, ids, sizeof(int32_t) * (size_t)batch * K);
  if (weights_out) memcpy(weights_out, wts, sizeof(float) * (size_t)batch * K);
  free(all);
  free(g);
  free(slot_out);
  free(wts);
  free(ids);
  free(logits);
  return ORK_OK;
}

/* engine.cpp:229-369 (forward_sparse): dense gate, threshold mask on
 * |silu(gate)|, compaction, then 64-neuron tiles of gathered up+down. */
int ork_forward_sparse(const ork_weights *w, const float *x, int batch, float threshold, float *y,
                       ork_report *rep) {
  const ork_config *c = &w->cfg;
  int rc = ork_config_validate(c);
  if (rc != ORK_OK) return rc;
  if (!(threshold >= 0.0f)) return ORK_ECONFIG;
  const int E = c->n_experts, K = c->top_k, D = c->d_model, N = c->d_ffn;
  const int capacity = ork_default_capacity(K, N);
  const uint64_t token_tiles = ((uint64_t)capacity + ORK_TILE - 1) / ORK_TILE;

  float *logits = (float *)malloc(sizeof(float) * (size_t)batch * E);
  int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)batch * K);
  float *wts = (float *)malloc(sizeof(float) * (size_t)batch * K);
  ork_router_logits(w, x, batch, logits);
  rc = ork_route(logits, batch, E, K, c->renormalize, ids, wts);
  if (rc != ORK_OK) {
    free(logits);
    free(ids);
    free(wts);
    return rc;
  }
  float *gate_raw = (float *)malloc(sizeof(float) * (size_t)K * N);
  uint8_t *masks = (uint8_t *)malloc((size_t)K * N);
  int32_t *flat = (int32_t *)malloc(sizeof(int32_t) * (size_t)capacity);
  int32_t *per_slot = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
  float *partial = (float *)malloc(sizeof(float) * (size_t)D);

  uint64_t active_sum = 0, skipped = 0, padded_sum = 0;
  for (int t = 0; t < batch; ++t) {
    const float *xt = x + (size_t)t * D;
    const int32_t *tid = ids + (size_t)t * K;
    for (int s = 0; s < K; ++s) {
      ork_matvec(w->gate + (size_t)tid[s] * N * D, N, D, xt, gate_raw + (size_t)s * N);
      ork_threshold_mask(gate_raw + (size_t)s * N, N, threshold, masks + (size_t)s * N);
    }
    int32_t total = 0;
    ork_compact_active(masks, tid, K, N, capacity, flat, per_slot, &total);

    float *yt = y + (size_t)t * D;
    for (int d = 0; d < D; ++d) yt[d] = 0.0f;
    for (uint64_t tile = 0; tile < token_tiles; ++tile) {
      const int32_t lo = (int32_t)tile * ORK_TILE;
      if (lo >= total) continue;
      int32_t hi = lo + ORK_TILE;
      if (hi > capacity) hi = capacity;
      if (hi > total) hi = total;
      for (int d = 0; d < D; ++d) partial[d] = 0.0f;
      for (int32_t k = lo; k < hi; ++k) {
        const int e = flat[k] / N, n = flat[k] % N;
        int s = 0;
        while (s < K && tid[s] != e) ++s;
        const float h_up = ork_dot(w->up + ((size_t)e * N + n) * D, xt, D);
        const float hval = wts[(size_t)t * K + s] * ork_silu(gate_raw[(size_t)s * N + n]) * h_up;
        const float *drow = w->down_t + ((size_t)e * N + n) * D;
        for (int d = 0; d < D; ++d) partial[d] += drow[d] * hval;
      }
      for (int d = 0; d < D; ++d) yt[d] += partial[d];
    }
    const uint64_t exec_tiles = ((uint64_t)total + ORK_TILE - 1) / ORK_TILE;
    padded_sum += exec_tiles * ORK_TILE;
    active_sum += (uint64_t)total;
    skipped += token_tiles - exec_tiles;
  }
  uint64_t other = (uint64_t)batch * (uint64_t)E * (uint64_t)D;
  ork_add_shared(w, x, batch, NULL, y, NULL, &other);
  if (rep) {
    const uint64_t routed = (uint64_t)batch * K * (uint64_t)N;
    memset(rep, 0, sizeof(*rep));
    rep->gate_macs = routed * (uint64_t)D;
    rep->up_macs = rep->down_macs = padded_sum * (uint64_t)D;
    rep->other_macs = other;
    rep->active_neurons_total = active_sum;
    rep->achieved_routed_sparsity = 1.0 - (double)active_sum / (double)routed;
    rep->tiles_total = (uint64_t)batch * token_tiles;
    rep->tiles_skipped = skipped;
    rep->path_used = 1;
  }
  free(partial);
  free(per_slot);
  free(flat);
  free(masks);
  free(gate_raw);
  free(wts);
  free(ids);
  free(logits);
  return ORK_OK;
}

/* tests/support.hpp:55-152.  Router in float (so expert choice agrees), the
 * rest in double with plain loops. */
int ork_scalar_forward(const ork_weights *w, const float *x, int batch, const uint8_t *routed_masks,
                       const uint8_t *shared_masks, float *y) {
  const ork_config *c = &w->cfg;
  const int E = c->n_experts, K = c->top_k, D = c->d_model, N = c->d_ffn, S = c->d_shared;
  float *logits = (float *)malloc(sizeof(float) * (size_t)E);
  int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
  float *pw = (float *)malloc(sizeof(float) * (size_t)K);
  double *acc = (double *)malloc(sizeof(double) * (size_t)D);
  for (int t = 0; t < batch; ++t) {
    const float *xt = x + (size_t)t * D;
    ork_matvec(w->router, E, D, xt, logits);
    ork_route(logits, 1, E, K, 0, ids, pw); /* raw probabilities, float */
    double wsum = 0.0;
    for (int s = 0; s < K; ++s) wsum += (double)pw[s];
    for (int d = 0; d < D; ++d) acc[d] = 0.0;
    for (int s = 0; s < K; ++s) {
      const size_t e = (size_t)ids[s];
      const double wt = c->renormalize ? (double)pw[s] / wsum : (double)pw[s];
      for (int n = 0; n < N; ++n) {
        const float *gr = w->gate + (e * N + n) * D, *ur = w->up + (e * N + n) * D;
        double g = 0.0, u = 0.0;
        for (int d = 0; d < D; ++d) {
          g += (double)gr[d] * xt[d];
          u += (double)ur[d] * xt[d];
        }
        double h = g / (1.0 + exp(-g)) * u;
        if (routed_masks && !routed_masks[((size_t)t * K + s) * N + n]) h = 0.0;
        const double wh = wt * h;
        const float *dr = w->down_t + (e * N + n) * D;
        for (int d = 0; d < D; ++d) acc[d] += wh * (double)dr[d];
      }
    }
    if (c->has_shared) {
      for (int n = 0; n < S; ++n) {
        const float *gr = w->shared_gate + (size_t)n * D, *ur = w->shared_up + (size_t)n * D;
        double g = 0.0, u = 0.0;
        for (int d = 0; d < D; ++d) {
          g += (double)gr[d] * xt[d];
          u += (double)ur[d] * xt[d];
        }
        double h = g / (1.0 + exp(-g)) * u;
        if (shared_masks && !shared_masks[(size_t)t * S + n]) h = 0.0;
        const float *dr = w->shared_down_t + (size_t)n * D;
        for (int d = 0; d < D; ++d) acc[d] += h * (double)dr[d];
      }
    }
    for (int d = 0; d < D; ++d) y[(size_t)t * D + d] = (float)acc[d];
  }
  free(acc);
  free(pw);
  free(ids);
  free(logits);
  return ORK_OK;
}

/* tests/support.hpp:32-42 */
double ork_max_rel_diff(const float *a, const float *b, uint64_t count) {
  double worst = 0.0, ref = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    const double d = fabs((double)a[i] - (double)b[i]);
    if (d > worst) worst = d;
    const double r = fabs((double)b[i]);
    if (r > ref) ref = r;
  }
  return worst / (ref > 1.0 ? ref : 1.0);
}
