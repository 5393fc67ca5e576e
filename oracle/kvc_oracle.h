/* kvc_oracle.h -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference's
 * hot-path arithmetic (kvclust, /root/reference/proj/core). Used as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg; never by the product.
 *
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   - bit-for-bit against the compiled reference (oracle/_ref/libkvclust_ref.so) on random
 *     inputs, when that library is present;
 *   - against the reference tests' known answers (tests/golden/kats.json).
 * The attention restatement has no reference counterpart (attention is a
 * non-goal of the reference) -- "parity unpinned" for attention values; see DESIGN.md.
 */
#ifndef KVC_ORACLE_H
#define KVC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:14-52 ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
  int has_spare;
  double spare;
} kvo_rng;
void kvo_rng_init(kvo_rng* r, uint64_t seed);
uint64_t kvo_rng_u64(kvo_rng* r);
double kvo_rng_uniform(kvo_rng* r);
uint64_t kvo_rng_index(kvo_rng* r, uint64_t n);
double kvo_rng_gaussian(kvo_rng* r);
uint64_t kvo_mix_seed(uint64_t a, uint64_t b);

/* ---- vecmath.hpp:27-77 (fp64 sequential sums) ---- */
double kvo_dot_fd(const float* a, const double* b, int d);
double kvo_dot_ff(const float* a, const float* b, int d);
double kvo_norm_f(const float* a, int d);
double kvo_norm_d(const double* a, int d);
/* returns the clamped cosine; *err = -2 (DegenerateVector) if a norm < 1e-12 */
double kvo_cosine_fd(const float* a, const double* b, int d, int* err);
double kvo_cosine_dd(const double* a, const double* b, int d, int* err);

/* ---- maintainer.cpp:11-25 ---- */
double kvo_tau(int64_t n, double tau_min, double tau_max, double n0);
void kvo_updated_stats(const double* rep, double var, int64_t n, const float* key, int d,
                       double* rep_out, double* var_out);

/* ---- workload.cpp:56-187 (gen_stream) ---- */
typedef struct {
  int n_scenes, frames_per_scene, tokens_per_frame, d, L;
  double visual_noise, semantic_noise, drift_rate, cross_layer_eps;
  int n_queries;
  double cross_modal_mix;
  int gt_top_m, scene_cycle, queries_at_end;
  uint64_t seed;
} kvo_stream_cfg;
/* Output buffers (caller-allocated):
 *   kinds[n_frames + n_queries]        0 frame / 1 query, in event order
 *   visual[n_frames][d], keys/values[n_frames][L][T][d]
 *   q[n_queries][L][d], gt[n_queries][gt_top_m], n_gt[n_queries]
 * Frames and queries are numbered in event order (frame_id = frame index, query_id =
 * query index). Returns 0, or -10 (ConfigError/ConfigInfeasible). */
int kvo_gen_stream(const kvo_stream_cfg* cfg, int32_t* kinds, float* visual, float* keys,
                   float* values, float* q, int64_t* gt, int32_t* n_gt);

/* ---- ranking: index.cpp:192-240, retrieval.cpp:145-164 ----
 * Sorts n candidates by (sim desc, key asc) and writes the first k positions into order[].
 * key = 2*cluster_id + is_buffer reproduces CandidateRef's (cluster_id, is_buffer) order
 * (index.hpp:62-68). Returns min(n, k). */
int kvo_rank(const double* sims, const int64_t* keys, int n, int k, int32_t* order);

/* ---- attention restatement (no reference counterpart) ----
 * out[d] = sum_t softmax(q.k_t * scale) v_t over n tokens, fp64. K,V row-major [n][d]. */
void kvo_attend_f32(const float* q, const float* K, const float* V, int n, int d, double scale,
                    double* out);

/* ---- token baseline ranking: retrieval.cpp:185-204 ----
 * cosine of q to every key, order by (sim desc, frame asc, token asc); first k indices. */
int kvo_token_rank(const float* q, const float* keys, const int64_t* frames,
                   const int32_t* tokens, int n, int d, int k, int32_t* order);

#ifdef __cplusplus
}
#endif
#endif
