/*
 * samo_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference algorithm on the SAMO per-step path
 * (/root/reference/proj/include/samo/*.hpp).  It is the checker the parity
 * tests compare the CUDA path against, and the "port" CPU baseline of
 * bench.py.  Nothing in the product path (paper_2302_05045_b200/) may link,
 * load or call it.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * reference's own known-answer tests (half_test.cpp, store_test.cpp,
 * prune_test.cpp, train_test.cpp) and against golden vectors produced by the
 * unmodified reference headers compiled into oracle/_ref/libsamo_ref.so
 * (tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no -march, so no FMA
 * contraction — the reference's Adam is FMA-free on x86-64).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------------- */
/* binary16 (half.hpp:13-71)                                               */

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* float_to_half_bits, half.hpp:13-49: RNE in integer arithmetic. */
EXPORT uint16_t or_float_to_half(float value) {
  const uint32_t w = f2u(value);
  const uint16_t sign = (uint16_t)((w >> 16) & 0x8000u);
  const uint32_t mag = w & 0x7FFFFFFFu;
  if (mag > 0x7F800000u) /* NaN: quiet bit forced, top payload bits kept (18-24) */
    return (uint16_t)(sign | 0x7E00u | ((mag >> 13) & 0x03FFu));
  if (mag == 0x7F800000u || mag >= 0x47800000u) /* inf, or >= 2^16 (25-27) */
    return (uint16_t)(sign | 0x7C00u);
  if (mag < 0x33000000u) /* below 2^-25 -> signed zero (37-39) */
    return sign;
  int32_t e = (int32_t)(mag >> 23) - 127;      /* unbiased exponent */
  uint32_t sig = (mag & 0x7FFFFFu) | 0x800000u; /* 24-bit significand */
  uint32_t drop;                                /* bits dropped from sig */
  uint32_t base;                                /* encoding before rounding */
  if (e >= -14) { /* normal half (28-36) */
    drop = 13;
    base = ((uint32_t)(e + 15) << 10) | ((sig >> 13) & 0x3FFu);
  } else {        /* subnormal half (40-48): value = q * 2^-24 */
    drop = (uint32_t)(-1 - e); /* 14..24 for e in [-25, -15] */
    base = sig >> drop;
  }
  const uint32_t rem = sig & ((1u << drop) - 1u);
  const uint32_t half = 1u << (drop - 1u);
  if (rem > half || (rem == half && (base & 1u))) base += 1u; /* carry may reach inf / normal */
  return (uint16_t)(sign | base);
}

/* half_bits_to_float, half.hpp:52-71: exact. */
EXPORT float or_half_to_float(uint16_t h) {
  const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu;
  uint32_t m = h & 0x3FFu;
  if (e == 0x1Fu) return u2f(sign | 0x7F800000u | (m << 13));
  if (e == 0) {
    if (m == 0) return u2f(sign);
    int32_t ex = -14; /* normalise the subnormal */
    while (!(m & 0x400u)) { m <<= 1; --ex; }
    return u2f(sign | ((uint32_t)(ex + 127) << 23) | ((m & 0x3FFu) << 13));
  }
  return u2f(sign | ((e + 112u) << 23) | (m << 13));
}

EXPORT void or_f2h(const float* in, uint16_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = or_float_to_half(in[i]);
}
EXPORT void or_h2f(const uint16_t* in, float* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = or_half_to_float(in[i]);
}

/* ---------------------------------------------------------------------- */
/* compress / expand (store.hpp:58-87).  Return 1 on DimensionError.      */

EXPORT int or_compress_u16(const uint16_t* dense, uint64_t dense_len, const uint32_t* idx,
                           uint64_t n, uint64_t ind_dense_len, uint16_t* out) {
  if (dense_len != ind_dense_len) return 1; /* store.hpp:60-62 */
  for (uint64_t k = 0; k < n; ++k) out[k] = dense[idx[k]];
  return 0;
}
EXPORT int or_compress_u32(const uint32_t* dense, uint64_t dense_len, const uint32_t* idx,
                           uint64_t n, uint64_t ind_dense_len, uint32_t* out) {
  if (dense_len != ind_dense_len) return 1;
  for (uint64_t k = 0; k < n; ++k) out[k] = dense[idx[k]];
  return 0;
}
EXPORT int or_expand_u16(const uint16_t* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                         uint64_t ind_dense_len, uint64_t shape_numel, uint16_t* dense) {
  if (n_values != n || shape_numel != ind_dense_len) return 1; /* store.hpp:75-80 */
  memset(dense, 0, shape_numel * 2);
  for (uint64_t k = 0; k < n; ++k) dense[idx[k]] = values[k];
  return 0;
}
EXPORT int or_expand_u32(const uint32_t* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                         uint64_t ind_dense_len, uint64_t shape_numel, uint32_t* dense) {
  if (n_values != n || shape_numel != ind_dense_len) return 1;
  memset(dense, 0, shape_numel * 4);
  for (uint64_t k = 0; k < n; ++k) dense[idx[k]] = values[k];
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Adam (train.hpp:320-347).                                               */

typedef struct {
  float lr, beta1, beta2, eps, loss_scale, wd;
} or_cfg;

EXPORT void or_adam_update(float* theta, float* m, float* v, const float* g, uint64_t n,
                           const or_cfg* c, float bias1, float bias2) {
  const float omb1 = 1.0f - c->beta1; /* train.hpp:335-336 */
  const float omb2 = 1.0f - c->beta2;
  for (uint64_t i = 0; i < n; ++i) { /* train.hpp:337-346, one rounding per op */
    const float gi = g[i];
    const float mi = c->beta1 * m[i] + omb1 * gi;
    const float vi = c->beta2 * v[i] + omb2 * (gi * gi);
    const float mh = mi / bias1;
    const float vh = vi / bias2;
    float t = theta[i] - c->lr * (mh / (sqrtf(vh) + c->eps));
    if (c->wd != 0.0f) t = t - (c->lr * c->wd) * t;
    m[i] = mi;
    v[i] = vi;
    theta[i] = t;
  }
}

/* ---------------------------------------------------------------------- */
/* One optimizer step over a flat arena (SamoTrainer::optimizer_step,      */
/* train.hpp:617-656), with the backward-sink gather (train.hpp:598-611)   */
/* folded in: grad16[k] = dense_grad_l[idx[k]].                            */
/*                                                                          */
/* Layers are given as arrays; compressed arenas are layer-concatenated.   */
/* state: [0]=t, [1]=skipped (as uint64), beta pows in bp[2].              */

typedef struct {
  uint64_t t;
  uint64_t skipped;
  float beta1_pow;
  float beta2_pow;
  float grad_norm;
  uint32_t last_skipped;
} or_step_state;

/* bfloat16 -> binary32 (the north_star's other 16-bit gradient type; no
 * reference code — an extension paralleling half_bits_to_float,
 * half.hpp:52-71): bfloat16 is the top half of a binary32, so the widening is
 * exact for every input, NaN payloads included. */
EXPORT float or_bf16_to_float(uint16_t h) {
  const uint32_t w = (uint32_t)h << 16;
  float f;
  memcpy(&f, &w, 4);
  return f;
}

EXPORT void or_bf16_to_float_n(const uint16_t* in, float* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = or_bf16_to_float(in[i]);
}

/* grad_bf16 = 0: binary16 dense gradients (the reference); 1: bfloat16. */
EXPORT int or_optimizer_step_ex(int nlayers, const uint64_t* dense_len, const uint64_t* nnz,
                                const uint32_t* idx, const uint16_t* const* dense_grads,
                                float* theta, float* m, float* v, float* g32,
                                uint16_t* const* theta16, const or_cfg* c, or_step_state* st,
                                int grad_bf16) {
  const float inv_scale = 1.0f / c->loss_scale; /* train.hpp:619 */
  int finite = 1;
  float norm_acc = 0.0f;
  uint64_t k0 = 0;
  for (int l = 0; l < nlayers; ++l) { /* train.hpp:622-629, serial over layers then k */
    for (uint64_t k = 0; k < nnz[l]; ++k) {
      const uint16_t h = dense_grads[l][idx[k0 + k]];
      const float gv = (grad_bf16 ? or_bf16_to_float(h) : or_half_to_float(h)) * inv_scale;
      g32[k0 + k] = gv;
      finite = finite && isfinite(gv);
      norm_acc += gv * gv;
    }
    k0 += nnz[l];
  }
  st->grad_norm = sqrtf(norm_acc);
  if (!finite) { /* train.hpp:632-639 */
    st->skipped += 1;
    st->last_skipped = 1;
    memset(g32, 0, k0 * 4);
    return 0;
  }
  st->t += 1; /* AdamScalars::advance, train.hpp:325-329 */
  st->beta1_pow *= c->beta1;
  st->beta2_pow *= c->beta2;
  st->last_skipped = 0;
  const float bias1 = 1.0f - st->beta1_pow, bias2 = 1.0f - st->beta2_pow;
  k0 = 0;
  for (int l = 0; l < nlayers; ++l) { /* train.hpp:643-654 */
    or_adam_update(theta + k0, m + k0, v + k0, g32 + k0, nnz[l], c, bias1, bias2);
    memset(theta16[l], 0, dense_len[l] * 2);
    for (uint64_t k = 0; k < nnz[l]; ++k) theta16[l][idx[k0 + k]] = or_float_to_half(theta[k0 + k]);
    memset(g32 + k0, 0, nnz[l] * 4);
    k0 += nnz[l];
  }
  return 1;
}

EXPORT int or_optimizer_step(int nlayers, const uint64_t* dense_len, const uint64_t* nnz,
                             const uint32_t* idx, const uint16_t* const* dense_grads,
                             float* theta, float* m, float* v, float* g32,
                             uint16_t* const* theta16, const or_cfg* c, or_step_state* st) {
  return or_optimizer_step_ex(nlayers, dense_len, nnz, idx, dense_grads, theta, m, v, g32, theta16, c, st, 0);
}

/* ---------------------------------------------------------------------- */
/* Index construction (prune.hpp:61-170).                                  */

/* detail::unpruned_count, prune.hpp:76-79 (double arithmetic). */
EXPORT uint64_t or_unpruned_count(double p, uint64_t n) {
  const double exact = (1.0 - p) * (double)n;
  return (uint64_t)floor(exact + 0.5 + 1e-9);
}

/* Key of a parameter under the ranking |v| (as float) — the bit pattern of
 * fabsf(v) is monotone in |v| for non-NaN floats. */
static uint32_t mag_key(float v) { return f2u(v) & 0x7FFFFFFFu; }

/* Threshold of a problem (a list of (values, len) segments): the keep-th
 * largest key T and how many key==T elements are kept.  Two 16-bit counting
 * passes instead of the reference's partial_sort; same selected set. */
static void select_threshold(const float* const* vals, const uint64_t* lens, const int* segs,
                             int nsegs, uint64_t keep, uint32_t* T_out, uint64_t* need_eq) {
  if (keep == 0) { *T_out = 0xFFFFFFFFu; *need_eq = 0; return; }
  uint64_t* hist = (uint64_t*)calloc(65536, sizeof(uint64_t));
  for (int s = 0; s < nsegs; ++s)
    for (uint64_t i = 0; i < lens[segs[s]]; ++i) hist[mag_key(vals[segs[s]][i]) >> 16]++;
  uint64_t r = keep, above = 0;
  int hi = 65535;
  for (; hi >= 0; --hi) {
    if (above + hist[hi] >= r) break;
    above += hist[hi];
  }
  r -= above;
  memset(hist, 0, 65536 * sizeof(uint64_t));
  for (int s = 0; s < nsegs; ++s)
    for (uint64_t i = 0; i < lens[segs[s]]; ++i) {
      const uint32_t key = mag_key(vals[segs[s]][i]);
      if ((int)(key >> 16) == hi) hist[key & 0xFFFFu]++;
    }
  above = 0;
  int lo = 65535;
  for (; lo >= 0; --lo) {
    if (above + hist[lo] >= r) break;
    above += hist[lo];
  }
  free(hist);
  *T_out = ((uint32_t)hi << 16) | (uint32_t)lo;
  *need_eq = r - above;
}

/* magnitude_prune (prune.hpp:99-170).  scope 0 = per_layer, 1 = global.
 * idx_out[l] has room for lens[l]; counts_out[l] receives the kept count.
 * Returns 0, or 2 (ParameterError) for p outside [0,1) or a layer >= 2^32. */
EXPORT int or_magnitude_prune(const float* const* vals, const uint64_t* lens,
                              const uint8_t* prunable, int nlayers, double p, int scope,
                              uint32_t* const* idx_out, uint64_t* counts_out) {
  if (!(p >= 0.0 && p < 1.0)) return 2;
  for (int l = 0; l < nlayers; ++l)
    if (lens[l] >= (1ull << 32)) return 2;
  int* segs = (int*)malloc(sizeof(int) * (nlayers > 0 ? nlayers : 1));
  uint32_t T_glob = 0;
  uint64_t need_glob = 0;
  if (scope == 1) {
    int ns = 0;
    uint64_t total = 0;
    for (int l = 0; l < nlayers; ++l)
      if (prunable[l]) { segs[ns++] = l; total += lens[l]; }
    select_threshold(vals, lens, segs, ns, or_unpruned_count(p, total), &T_glob, &need_glob);
  }
  uint64_t eq_seen_glob = 0; /* global tie-break: layer asc, then index asc */
  for (int l = 0; l < nlayers; ++l) {
    uint64_t cnt = 0;
    if (!prunable[l]) { /* iota, prune.hpp:117-120 */
      for (uint64_t i = 0; i < lens[l]; ++i) idx_out[l][i] = (uint32_t)i;
      counts_out[l] = lens[l];
      continue;
    }
    uint32_t T;
    uint64_t need;
    uint64_t eq_seen = 0;
    uint64_t* eq_ctr = &eq_seen;
    if (scope == 1) {
      T = T_glob; need = need_glob; eq_ctr = &eq_seen_glob;
    } else {
      segs[0] = l;
      select_threshold(vals, lens, segs, 1, or_unpruned_count(p, lens[l]), &T, &need);
    }
    for (uint64_t i = 0; i < lens[l]; ++i) {
      const uint32_t key = mag_key(vals[l][i]);
      int keep = 0;
      if (T != 0xFFFFFFFFu && key > T) keep = 1;
      else if (key == T) { keep = (*eq_ctr < need); (*eq_ctr)++; }
      if (keep) idx_out[l][cnt++] = (uint32_t)i;
    }
    counts_out[l] = cnt;
  }
  free(segs);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Synthetic data — mirror of the product's counter-based generator        */
/* (paper_2302_05045_b200/csrc/common.cuh synth_mix64) so tests can        */
/* regenerate any element of a GPT-scale input on the host.                */

static uint64_t mix64(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t x = i + stream * 0xD1B54A32D192ED03ull + seed * 0x9E3779B97F4A7C15ull;
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

static float synth_value(uint64_t seed, uint64_t sid, uint64_t i, float bound) {
  const float c = (float)(mix64(seed, sid, i) >> 40) * 0x1.0p-24f; /* train.hpp:93-96 */
  return (2.0f * c - 1.0f) * bound;                                 /* train.hpp:98-100 */
}

EXPORT void or_synth_f32(float* out, uint64_t first, uint64_t n, uint64_t seed, uint64_t sid,
                         float bound) {
  for (uint64_t i = 0; i < n; ++i) out[i] = synth_value(seed, sid, first + i, bound);
}
EXPORT void or_synth_f16(uint16_t* out, uint64_t first, uint64_t n, uint64_t seed, uint64_t sid,
                         float bound, float scale) {
  for (uint64_t i = 0; i < n; ++i) out[i] = or_float_to_half(synth_value(seed, sid, first + i, bound) * scale);
}

/* mt19937_64 (the engine the reference seeds, train.hpp:90-100) so tests can
 * reproduce init_params / uniform_symmetric streams without the reference. */
typedef struct { uint64_t mt[312]; int mti; } or_mt64;

EXPORT void or_mt64_seed(or_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

EXPORT uint64_t or_mt64_next(or_mt64* s) {
  static const uint64_t MAG[2] = {0ull, 0xB5026F5AA96619E9ull};
  if (s->mti >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      s->mt[i] = s->mt[(i + 156) % 312] ^ (x >> 1) ^ MAG[x & 1ull];
    }
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* n draws of uniform_symmetric(eng, bound) (train.hpp:98-100). */
EXPORT void or_mt64_uniform(or_mt64* s, float* out, uint64_t n, float bound) {
  for (uint64_t i = 0; i < n; ++i) {
    const float c = (float)(or_mt64_next(s) >> 40) * 0x1.0p-24f;
    out[i] = (2.0f * c - 1.0f) * bound;
  }
}

/* ---------------------------------------------------------------------- */
/* Data-parallel exchange oracle (no reference code exists; the reference  */
/* only models it, sim.hpp:110-117).  Rank-ascending fp32 sum, plus the    */
/* fp64 sum of |g_r| for the error bound.                                  */
EXPORT void or_dp_sum(const float* const* bufs, int G, uint64_t n, float* out, double* abs_sum) {
  for (uint64_t i = 0; i < n; ++i) {
    float s = 0.0f;
    double a = 0.0;
    for (int r = 0; r < G; ++r) { s += bufs[r][i]; a += fabs((double)bufs[r][i]); }
    out[i] = s;
    if (abs_sum) abs_sum[i] = a;
  }
}

/* dW = matmul(transpose(x), dy) (train.hpp:304, tensor.hpp:88-105): exact
 * half x half products, serial fp32 adds in ascending batch order, one
 * rounding to binary16.  x [batch x in], dy [batch x out], dw [in x out]. */
EXPORT void or_dw_matmul(const uint16_t* x, const uint16_t* dy, uint64_t batch, uint64_t in,
                         uint64_t out, uint16_t* dw) {
  for (uint64_t i = 0; i < in; ++i) {
    for (uint64_t j = 0; j < out; ++j) {
      float acc = 0.0f;
      for (uint64_t b = 0; b < batch; ++b)
        acc += or_half_to_float(x[b * in + i]) * or_half_to_float(dy[b * out + j]);
      dw[i * out + j] = or_float_to_half(acc);
    }
  }
}
