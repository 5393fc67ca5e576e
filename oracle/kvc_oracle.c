/* kvc_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker; see kvc_oracle.h).
 *
 * Plain-C restatement of the reference arithmetic on the hot path. Every function cites
 * the reference file:line it follows (paths relative to /root/reference/proj/core).
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, matching the reference's
 * -ffp-contract=off at /root/reference/proj/CMakeLists.txt:11-13).
 */
#include "kvc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ rng
 * std::mt19937_64 as specified by [rand.eng.mers] (rng.hpp:41 uses the standard engine),
 * the 53-bit uniform (rng.hpp:19), modulo index (rng.hpp:21) and Box-Muller with a cached
 * spare (rng.hpp:26-38). */
#define MT_N 312
#define MT_M 156

void kvo_rng_init(kvo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

static void mt_twist(kvo_rng* r) {
  const uint64_t hi = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & hi) | (r->mt[(i + 1) % MT_N] & lo);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t kvo_rng_u64(kvo_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

double kvo_rng_uniform(kvo_rng* r) { return (double)(kvo_rng_u64(r) >> 11) * 0x1.0p-53; }

uint64_t kvo_rng_index(kvo_rng* r, uint64_t n) { return kvo_rng_u64(r) % n; }

double kvo_rng_gaussian(kvo_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = kvo_rng_uniform(r);
  double u2 = kvo_rng_uniform(r);
  double rad = sqrt(-2.0 * log1p(-u1));
  double th = 2.0 * M_PI * u2;
  r->spare = rad * sin(th);
  r->has_spare = 1;
  return rad * cos(th);
}

/* rng.hpp:47-52 (splitmix64 finalizer) */
uint64_t kvo_mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* ------------------------------------------------------------------ vecmath
 * vecmath.hpp:27-61: fp64 sequential accumulation of fp32->fp64 products, no FMA. */
double kvo_dot_fd(const float* a, const double* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += (double)a[i] * b[i];
  return s;
}
double kvo_dot_ff(const float* a, const float* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += (double)a[i] * (double)b[i];
  return s;
}
static double dot_dd(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += a[i] * b[i];
  return s;
}
double kvo_norm_f(const float* a, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += (double)a[i] * (double)a[i];
  return sqrt(s);
}
double kvo_norm_d(const double* a, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += a[i] * a[i];
  return sqrt(s);
}
static double clamp1(double x) { return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x); }

/* vecmath.hpp:54-61; kDegenerateNorm = 1e-12 (vecmath.hpp:19) */
double kvo_cosine_fd(const float* a, const double* b, int d, int* err) {
  double na = kvo_norm_f(a, d), nb = kvo_norm_d(b, d);
  if (na < 1e-12 || nb < 1e-12) {
    if (err) *err = -2;
    return 0.0;
  }
  if (err) *err = 0;
  return clamp1(kvo_dot_fd(a, b, d) / (na * nb));
}
double kvo_cosine_dd(const double* a, const double* b, int d, int* err) {
  double na = kvo_norm_d(a, d), nb = kvo_norm_d(b, d);
  if (na < 1e-12 || nb < 1e-12) {
    if (err) *err = -2;
    return 0.0;
  }
  if (err) *err = 0;
  return clamp1(dot_dd(a, b, d) / (na * nb));
}

/* vecmath.hpp:71-77 */
static int dnormalize(double* v, int d) {
  double n = kvo_norm_d(v, d);
  if (n < 1e-12) return -2;
  for (int i = 0; i < d; ++i) v[i] = v[i] / n;
  return 0;
}

/* ------------------------------------------------------------------ maintainer
 * maintainer.cpp:11-14 */
double kvo_tau(int64_t n, double tau_min, double tau_max, double n0) {
  return tau_min + (tau_max - tau_min) * exp(-(double)n / n0);
}

/* maintainer.cpp:16-25 -- r' = (n r + k)/(n+1); var' = (n var + |k - r'|^2)/(n+1) */
void kvo_updated_stats(const double* rep, double var, int64_t n, const float* key, int d,
                       double* rep_out, double* var_out) {
  double dn = (double)n;
  for (int i = 0; i < d; ++i) rep_out[i] = (dn * rep[i] + (double)key[i]) / (dn + 1.0);
  double sq = 0.0; /* sq_dist(key, rep') : vecmath.hpp:42-51 */
  for (int i = 0; i < d; ++i) {
    double diff = (double)key[i] - rep_out[i];
    sq += diff * diff;
  }
  *var_out = (dn * var + sq) / (dn + 1.0);
}

/* ------------------------------------------------------------------ gen_stream
 * workload.cpp:30-54 helpers, 56-187 generator. */
static void gauss_vec(kvo_rng* r, double* v, int d) {
  for (int i = 0; i < d; ++i) v[i] = kvo_rng_gaussian(r);
}
static int unit_vec(kvo_rng* r, double* v, int d) {
  gauss_vec(r, v, d);
  return dnormalize(v, d);
}
static int perturb(kvo_rng* r, const double* base, double scale, double* out, int d) {
  if (out != base) memcpy(out, base, sizeof(double) * (size_t)d);
  for (int i = 0; i < d; ++i) out[i] += scale * kvo_rng_gaussian(r);
  return dnormalize(out, d);
}

typedef struct {
  double sim;
  int64_t id;
} simid;
static int cmp_simid(const void* a, const void* b) {
  const simid* x = (const simid*)a;
  const simid* y = (const simid*)b;
  if (x->sim != y->sim) return x->sim > y->sim ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}
static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int kvo_gen_stream(const kvo_stream_cfg* c, int32_t* kinds, float* visual, float* keys,
                   float* values, float* qout, int64_t* gt, int32_t* n_gt) {
  const int d = c->d, L = c->L, T = c->tokens_per_frame, S = c->n_scenes, F = c->frames_per_scene;
  if (S < 1 || F < 1 || T < 1 || d < 1 || L < 1 || c->n_queries < 0 || c->gt_top_m < 1)
    return -10;
  kvo_rng rng;
  kvo_rng_init(&rng, c->seed);
  int n_base = c->scene_cycle > 0 ? (c->scene_cycle < S ? c->scene_cycle : S) : S;

  double* vc = (double*)calloc((size_t)n_base * d, sizeof(double));
  double* tmp = (double*)calloc((size_t)d, sizeof(double));
  int have = 0, retries = 0;
  while (have < n_base) { /* workload.cpp:67-82: rejection sampling, cos < 0.5 */
    unit_vec(&rng, tmp, d);
    int ok = 1;
    for (int j = 0; j < have; ++j) {
      int e = 0;
      if (kvo_cosine_dd(tmp, vc + (size_t)j * d, d, &e) >= 0.5) {
        ok = 0;
        break;
      }
    }
    if (ok) {
      memcpy(vc + (size_t)have * d, tmp, sizeof(double) * (size_t)d);
      ++have;
    } else if (++retries > 20000) {
      free(vc);
      free(tmp);
      return -10;
    }
  }
  /* workload.cpp:86-97: semantic base = normalize(mix * visual + (1-mix) * dir) */
  double* sb = (double*)calloc((size_t)n_base * L * d, sizeof(double));
  for (int s = 0; s < n_base; ++s)
    for (int l = 0; l < L; ++l) {
      unit_vec(&rng, tmp, d);
      double* m = sb + ((size_t)s * L + l) * d;
      for (int i = 0; i < d; ++i)
        m[i] = c->cross_modal_mix * vc[(size_t)s * d + i] + (1.0 - c->cross_modal_mix) * tmp[i];
      dnormalize(m, d);
    }

  int per_scene = c->n_queries / S, extra = c->n_queries % S;
  double* final_c = (double*)calloc((size_t)S * L * d, sizeof(double));
  double* means = (double*)calloc((size_t)S * F * d, sizeof(double));
  double* centers = (double*)calloc((size_t)L * d, sizeof(double));
  double* key = (double*)calloc((size_t)d, sizeof(double));
  double* qd = (double*)calloc((size_t)d, sizeof(double));
  float* qf = (float*)calloc((size_t)d, sizeof(float));
  simid* scored = (simid*)calloc((size_t)F, sizeof(simid));
  int n_events = 0, n_queries = 0;
  int held_first = -1;
  int32_t* held = (int32_t*)calloc((size_t)(c->n_queries + 1), sizeof(int32_t));
  int n_held = 0;
  int64_t frame_id = 0;
  (void)held_first;

  for (int s = 0; s < S; ++s) {
    int base = c->scene_cycle > 0 ? s % n_base : s;
    const double* vcen = vc + (size_t)base * d;
    memcpy(centers, sb + (size_t)base * L * d, sizeof(double) * (size_t)L * d);
    for (int f = 0; f < F; ++f) {
      size_t fi = (size_t)frame_id;
      perturb(&rng, vcen, c->visual_noise, tmp, d);
      for (int i = 0; i < d; ++i) visual[fi * d + i] = (float)tmp[i];
      if (f > 0)
        for (int l = 0; l < L; ++l) perturb(&rng, centers + (size_t)l * d, c->drift_rate, centers + (size_t)l * d, d);
      double* ks = means + ((size_t)s * F + f) * d;
      for (int i = 0; i < d; ++i) ks[i] = 0.0;
      for (int l = 0; l < L; ++l)
        for (int t = 0; t < T; ++t) {
          size_t off = ((fi * L + l) * T + t) * (size_t)d;
          perturb(&rng, centers + (size_t)l * d, c->semantic_noise, key, d);
          for (int i = 0; i < d; ++i) keys[off + i] = (float)key[i];
          gauss_vec(&rng, tmp, d);
          for (int i = 0; i < d; ++i) values[off + i] = (float)tmp[i];
          if (l == 0)
            for (int i = 0; i < d; ++i) ks[i] += key[i];
        }
      for (int i = 0; i < d; ++i) ks[i] /= (double)T;
      kinds[n_events++] = 0;
      frame_id += 1;
    }
    memcpy(final_c + (size_t)s * L * d, centers, sizeof(double) * (size_t)L * d);

    int allotted = per_scene + (s < extra ? 1 : 0);
    for (int qi = 0; qi < allotted; ++qi) {
      int target = (int)kvo_rng_index(&rng, (uint64_t)(s + 1));
      size_t qo = (size_t)n_queries * L * d;
      memcpy(qd, final_c + (size_t)target * L * d, sizeof(double) * (size_t)d);
      for (int i = 0; i < d; ++i) qout[qo + i] = (float)qd[i];
      for (int l = 1; l < L; ++l) {
        perturb(&rng, qd, c->cross_layer_eps, qd, d);
        for (int i = 0; i < d; ++i) qout[qo + (size_t)l * d + i] = (float)qd[i];
      }
      /* ground truth: workload.cpp:158-168, cosine of the float layer-0 query to frame means */
      for (int f = 0; f < F; ++f) {
        int e = 0;
        scored[f].sim = kvo_cosine_fd(qout + qo, means + ((size_t)target * F + f) * d, d, &e);
        scored[f].id = (int64_t)target * F + f; /* frame ids of scene `target` */
      }
      /* frame ids are contiguous per scene: scene t's frames are t*F .. t*F+F-1 */
      qsort(scored, (size_t)F, sizeof(simid), cmp_simid);
      int m = F < c->gt_top_m ? F : c->gt_top_m;
      int64_t* g = gt + (size_t)n_queries * c->gt_top_m;
      for (int i = 0; i < m; ++i) g[i] = scored[i].id;
      qsort(g, (size_t)m, sizeof(int64_t), cmp_i64);
      n_gt[n_queries] = m;
      if (c->queries_at_end)
        held[n_held++] = n_queries;
      else
        kinds[n_events++] = 1;
      n_queries += 1;
    }
  }
  for (int i = 0; i < n_held; ++i) kinds[n_events++] = 1;
  (void)qf;
  free(vc);
  free(tmp);
  free(sb);
  free(final_c);
  free(means);
  free(centers);
  free(key);
  free(qd);
  free(qf);
  free(scored);
  free(held);
  return 0;
}

/* ------------------------------------------------------------------ ranking */
typedef struct {
  double sim;
  int64_t key;
  int32_t pos;
} rk;
static int cmp_rk(const void* a, const void* b) {
  const rk* x = (const rk*)a;
  const rk* y = (const rk*)b;
  if (x->sim != y->sim) return x->sim > y->sim ? -1 : 1;
  return x->key < y->key ? -1 : (x->key > y->key ? 1 : 0);
}

int kvo_rank(const double* sims, const int64_t* keys, int n, int k, int32_t* order) {
  rk* v = (rk*)malloc(sizeof(rk) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) {
    v[i].sim = sims[i];
    v[i].key = keys[i];
    v[i].pos = i;
  }
  qsort(v, (size_t)n, sizeof(rk), cmp_rk);
  int take = n < k ? n : k;
  for (int i = 0; i < take; ++i) order[i] = v[i].pos;
  free(v);
  return take;
}

/* ------------------------------------------------------------------ attention (fp64) */
void kvo_attend_f32(const float* q, const float* K, const float* V, int n, int d, double scale,
                    double* out) {
  for (int c = 0; c < d; ++c) out[c] = 0.0;
  if (n <= 0) return;
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  double mx = -INFINITY;
  for (int t = 0; t < n; ++t) {
    s[t] = kvo_dot_ff(q, K + (size_t)t * d, d) * scale;
    if (s[t] > mx) mx = s[t];
  }
  double den = 0.0;
  for (int t = 0; t < n; ++t) {
    double w = exp(s[t] - mx);
    den += w;
    for (int c = 0; c < d; ++c) out[c] += w * (double)V[(size_t)t * d + c];
  }
  for (int c = 0; c < d; ++c) out[c] /= den;
  free(s);
}

/* ------------------------------------------------------------------ token baseline */
typedef struct {
  double sim;
  int64_t frame;
  int32_t token;
  int32_t pos;
} tk;
static int cmp_tk(const void* a, const void* b) {
  const tk* x = (const tk*)a;
  const tk* y = (const tk*)b;
  if (x->sim != y->sim) return x->sim > y->sim ? -1 : 1;
  if (x->frame != y->frame) return x->frame < y->frame ? -1 : 1;
  return x->token < y->token ? -1 : (x->token > y->token ? 1 : 0);
}

int kvo_token_rank(const float* q, const float* keys, const int64_t* frames,
                   const int32_t* tokens, int n, int d, int k, int32_t* order) {
  tk* v = (tk*)malloc(sizeof(tk) * (size_t)(n > 0 ? n : 1));
  double nq = kvo_norm_f(q, d);
  for (int i = 0; i < n; ++i) {
    const float* kk = keys + (size_t)i * d;
    double nk = kvo_norm_f(kk, d);
    double c = kvo_dot_ff(q, kk, d) / (nq * nk);
    v[i].sim = clamp1(c);
    v[i].frame = frames[i];
    v[i].token = tokens[i];
    v[i].pos = i;
  }
  qsort(v, (size_t)n, sizeof(tk), cmp_tk);
  int take = n < k ? n : k;
  for (int i = 0; i < take; ++i) order[i] = v[i].pos;
  free(v);
  return take;
}
