// token.hpp -- token-level top-k retrieval baseline (retrieval.cpp:166-254): device arguments and
// the host context that drives it (token_context.cpp). Selected by kvc_cfg.token_mode, like the
// reference's RetrievalMode::TokenBaseline (engine.cpp:153-158, 179-203).
#pragma once

#include <cstdint>
#include <deque>
#include <vector>

#include "../../include/kvc.h"
#include "kvc_core.hpp"

namespace kvc {

struct TokArgs {
  int32_t L, d, es;
  int64_t cap;                // pool rows per domain
  int64_t wcap;               // 32-row words per domain
  uint8_t* pk;                // [L][cap][d] keys (kv dtype)
  uint8_t* pv;                // [L][cap][d] values
  double* kn64;               // [L][cap] exact key norms (vecmath.hpp:35-40)
  float* kn32;                // [L][cap] fp32 key norms (approximate scan)
  float* approx;              // [L][cap] approximate cosines of the current query
  uint32_t* pick;             // [L][wcap] picked rows (top token_budget)
  uint32_t* attw;             // [L][wcap] attended rows (picked | window)
  int32_t* att_idx;           // [L][max_att] attended rows in order
  int32_t* bidx;              // [L][cap] boundary rows (scratch)
  double* bsim;               // [L][cap] their exact cosines (scratch)
  long long* btie;            // [L][cap] their (frame id << 24 | token) tie-break keys (scratch)
  int32_t max_att, pages_per_dom;
  const int32_t* fidx;        // [cap] frame ordinal of each pool row (same for every domain)
  const int64_t* fid;         // [frames] frame id of each ordinal
  const int64_t* fstart;      // [frames] first pool row of each ordinal
  uint8_t* frame_hit;         // [frames] frame has an attended row in some domain
  int32_t* stats;             // [L][4] attended rows, host-side runs, host-side rows, boundary size
  const float* q;             // [L][d] current query
  int32_t* work_ctr;          // K6 work counter (reset by the select kernel)
  long long* prof;            // [L][8] clock64 cycles per select phase (instrumentation)
  int32_t* err;               // error bits (1: degenerate vector)
};

int launch_tok_append(const TokArgs& a, const void* fk, const void* fv, int T, int tmax, int64_t n0, cudaStream_t st);
// approx scan + select + gather + K6 (attention over the attended rows). Returns launches.
int launch_tok_decode(const TokArgs& a, const DevTables& stage, const DecodeArgs& da, int64_t n, int budget,
                      int64_t win_lo, cudaStream_t st);

class TokenContext {
 public:
  TokenContext(const kvc_cfg& cfg, int d, int L);
  ~TokenContext();
  void ingest_frame(std::int64_t frame_id, const void* keys, const void* values, int T, int mem);
  void decode_step(std::int64_t qid, const float* q, int q_mem, float* out, int out_mem, const std::int64_t* gt,
                   int n_gt);
  // views of the last query (RetrievalResult, retrieval.hpp:49-71)
  int attended(int layer, std::int64_t* frames, std::int32_t* tokens, int cap) const;
  void layer_meta(int layer, double* lat, std::int64_t* ints) const;
  double ttft() const { return ttft_; }
  double recall() const { return recall_; }
  std::uint64_t digest() const { return digest_; }
  std::int64_t ledger(std::int64_t* ops, std::int64_t* bytes, double* cost) const;
  cudaStream_t stream() const { return st_; }
  int L() const { return L_; }
  std::int64_t launches() const { return launches_; }
  void set_timing(bool on) { timing_ = on; }
  void set_head_dim(int d_logical);
  const double* step_timing() const { return step_t_; }
  void profile(double* out);  // mean select-phase cycles over domains (out[8])
  // the baseline's window_frames argument (retrieval.cpp:166-254) empty: nothing attended without
  // a fetch (the component-level retrieve_token_baseline call)
  void reset_window() { window_.clear(); }
  // RetrievalResult fetched_frames / context_frames of the last query (parity mode)
  const std::vector<std::int64_t>& last_frames(int which) const { return which == 0 ? fetched_ : context_; }

 private:
  kvc_cfg cfg_;
  int d_, L_, es_;
  int dl_ = 0;  // the caller's head width (kvc_set_head_dim)
  cudaStream_t st_ = nullptr;
  std::vector<void*> dev_, host_;
  void* dalloc(std::size_t bytes);
  TokArgs ta_{};
  DevTables stage_{};
  DecodeArgs da_{};
  void* d_fk_ = nullptr;
  void* d_fv_ = nullptr;
  float* d_q_ = nullptr;
  float* d_out_ = nullptr;
  std::int32_t* d_fidx_ = nullptr;
  std::int64_t* d_fid_ = nullptr;
  std::int64_t* d_fstart_ = nullptr;
  std::int32_t* h_stats_ = nullptr;
  std::uint8_t* h_hit_ = nullptr;
  std::int32_t* h_err_ = nullptr;
  std::int64_t max_frames_ = 0, tmax_ = 0;
  // host view of the pool: frames in ingest order
  std::vector<std::int64_t> fid_, fstart_;
  std::vector<int> ft_;
  std::int64_t n_ = 0;
  std::deque<std::int64_t> window_;  // ordinals of the last W frames
  // last query
  std::vector<std::vector<std::pair<std::int64_t, std::int32_t>>> att_;
  std::vector<double> lat_;  // [L][5]
  std::vector<std::int64_t> attc_, bnd_;
  double ttft_ = 0.0, recall_ = -1.0;
  std::uint64_t digest_ = 0;
  std::vector<std::int64_t> fetched_, context_;
  // baseline ledger totals (cause Retrieval, retrieval.cpp:224-229)
  std::int64_t led_ops_ = 0, led_bytes_ = 0;
  double led_cost_ = 0.0;
  std::int64_t launches_ = 0;
  bool timing_ = false;
  double step_t_[10] = {0};
  cudaEvent_t ev_[4];
};

}  // namespace kvc
