// token_context.cpp -- host side of the token-level baseline (engine.cpp:153-158 ingest into the
// per-layer pools, engine.cpp:179-203 + retrieval.cpp:166-254 per query). The pools, the scan,
// the selection and the attention run on the GPU (token.cu); the host keeps the frame table, the
// window, the latency model and the ledger totals, from per-domain counts the kernels produce.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "token.hpp"

namespace kvc {

namespace {

std::uint64_t fnv1a(std::uint64_t h, std::uint64_t x) {  // engine.cpp:18-24
  for (int i = 0; i < 8; ++i) {
    h ^= (x >> (8 * i)) & 0xffu;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace

void* TokenContext::dalloc(std::size_t bytes) {
  void* p = nullptr;
  KVC_CUDA(cudaMalloc(&p, std::max<std::size_t>(bytes, 16)));
  KVC_CUDA(cudaMemsetAsync(p, 0, std::max<std::size_t>(bytes, 16), st_));
  dev_.push_back(p);
  return p;
}

TokenContext::TokenContext(const kvc_cfg& cfg, int d, int L) : cfg_(cfg), d_(d), L_(L) {
  if (cfg_.k_v <= 0 || cfg_.k_s <= 0 || cfg_.window_frames <= 0 || cfg_.prefetch_k <= 0)
    fail(-10, "retrieval budgets must be positive");  // RetrievalConfig::validate (retrieval.cpp:10-16)
  if (cfg_.token_budget < 1) fail(-10, "token budget must be at least 1");
  if (cfg_.lookup_cost_per_candidate_us < 0.0 || cfg_.compute_cost_per_token_us < 0.0)
    fail(-10, "cost constants must be non-negative");
  if (cfg_.kv_dtype != KVC_DTYPE_F32 && cfg_.kv_dtype != KVC_DTYPE_BF16) fail(-10, "kv_dtype");
  if (d < 1 || L < 1 || d % 8 != 0 || d > 256) fail(-10, "the device path supports d % 8 == 0 and d <= 256");
  if (cfg_.page_tokens != 0 && (cfg_.page_tokens < 8 || cfg_.page_tokens > 64 || cfg_.page_tokens % 8))
    fail(-10, "page_tokens must be 0 (auto) or 8..64, a multiple of 8");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(-22, "no CUDA device: the B200 path has no CPU fallback");
  es_ = cfg_.kv_dtype == KVC_DTYPE_BF16 ? 2 : 4;
  if (cfg_.page_tokens == 0) cfg_.page_tokens = auto_page_tokens(d, cfg_.kv_dtype == KVC_DTYPE_BF16);
  if (d * es_ > 512) fail(-10, "token baseline rows are at most 512 bytes (fp32 d <= 128, bf16 d <= 256)");
  KVC_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  for (auto& e : ev_) KVC_CUDA(cudaEventCreate(&e));
  const std::int64_t rb = static_cast<std::int64_t>(d) * es_;
  tmax_ = cfg_.max_tokens;
  // pool rows per domain: pool_bytes holds the K/V of every domain
  const std::int64_t cap = std::max<std::int64_t>(64, cfg_.pool_bytes / (2 * rb * L));
  max_frames_ = cap + 1;  // at least one row per frame
  ta_.L = L;
  ta_.d = d;
  ta_.es = es_;
  ta_.cap = cap;
  ta_.wcap = (cap + 31) / 32;
  ta_.pk = static_cast<std::uint8_t*>(dalloc(static_cast<std::size_t>(L) * cap * rb));
  ta_.pv = static_cast<std::uint8_t*>(dalloc(static_cast<std::size_t>(L) * cap * rb));
  ta_.kn64 = static_cast<double*>(dalloc(static_cast<std::size_t>(L) * cap * 8));
  ta_.kn32 = static_cast<float*>(dalloc(static_cast<std::size_t>(L) * cap * 4));
  ta_.approx = static_cast<float*>(dalloc(static_cast<std::size_t>(L) * cap * 4));
  ta_.pick = static_cast<std::uint32_t*>(dalloc(static_cast<std::size_t>(L) * ta_.wcap * 4));
  ta_.attw = static_cast<std::uint32_t*>(dalloc(static_cast<std::size_t>(L) * ta_.wcap * 4));
  const std::int64_t max_att = std::min<std::int64_t>(cap, cfg_.token_budget + static_cast<std::int64_t>(cfg_.window_frames) * tmax_);
  ta_.max_att = static_cast<std::int32_t>(max_att);
  ta_.att_idx = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(L) * max_att * 4));
  ta_.bidx = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(L) * cap * 4));
  ta_.bsim = static_cast<double*>(dalloc(static_cast<std::size_t>(L) * cap * 8));
  ta_.btie = static_cast<long long*>(dalloc(static_cast<std::size_t>(L) * cap * 8));
  d_fidx_ = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(cap) * 4));
  d_fid_ = static_cast<std::int64_t*>(dalloc(static_cast<std::size_t>(max_frames_) * 8));
  d_fstart_ = static_cast<std::int64_t*>(dalloc(static_cast<std::size_t>(max_frames_) * 8));
  ta_.fidx = d_fidx_;
  ta_.fid = d_fid_;
  ta_.fstart = d_fstart_;
  ta_.frame_hit = static_cast<std::uint8_t*>(dalloc(static_cast<std::size_t>(max_frames_)));
  ta_.stats = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(L) * 16));
  ta_.err = static_cast<std::int32_t*>(dalloc(16));
  ta_.prof = static_cast<long long*>(dalloc(static_cast<std::size_t>(L) * 8 * 8));
  ta_.work_ctr = static_cast<std::int32_t*>(dalloc(64));
  d_q_ = static_cast<float*>(dalloc(static_cast<std::size_t>(L) * d * 4));
  d_out_ = static_cast<float*>(dalloc(static_cast<std::size_t>(L) * d * 4));
  d_fk_ = dalloc(static_cast<std::size_t>(L) * tmax_ * rb);
  d_fv_ = dalloc(static_cast<std::size_t>(L) * tmax_ * rb);
  // staging pages (the gathered attended rows) and K6's work list
  const int P = cfg_.page_tokens;
  ta_.pages_per_dom = static_cast<std::int32_t>((max_att + P - 1) / P);
  stage_.d = d;
  stage_.L = L;
  stage_.P = P;
  stage_.es = es_;
  stage_.kv_bf16 = es_ == 2;
  stage_.max_pages = static_cast<std::int64_t>(L) * ta_.pages_per_dom;
  stage_.page_bytes = 2LL * P * rb;
  stage_.pool = static_cast<std::uint8_t*>(dalloc(static_cast<std::size_t>(stage_.max_pages) * stage_.page_bytes));
  stage_.err = ta_.err;
  da_.chunk_pages = 8;
  da_.max_desc = ta_.pages_per_dom;
  da_.max_items = (da_.max_desc + da_.chunk_pages - 1) / da_.chunk_pages;
  da_.desc = static_cast<int4*>(dalloc(static_cast<std::size_t>(L) * da_.max_desc * sizeof(int4)));
  da_.n_desc = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(L) * 4));
  da_.n_items = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(L) * 4));
  da_.part_ml = static_cast<float*>(dalloc(static_cast<std::size_t>(L) * da_.max_items * 2 * 4));
  da_.part_o = static_cast<float*>(dalloc(static_cast<std::size_t>(L) * da_.max_items * d * 4));
  da_.dom_done = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(L) * 4));
  da_.work_ctr = ta_.work_ctr;
  da_.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d)));
  {
    const char* pf = std::getenv("KVC_ATT_PF");  // K6: L2 prefetch distance in pages (0: off)
    da_.att_pf = pf ? std::atoi(pf) : 0;
  }
  da_.q = d_q_;
  ta_.q = d_q_;
  void* hs = nullptr;
  KVC_CUDA(cudaMallocHost(&hs, static_cast<std::size_t>(L) * 16 + 64));
  host_.push_back(hs);
  h_stats_ = static_cast<std::int32_t*>(hs);
  h_err_ = h_stats_ + L * 4;
  void* hh = nullptr;
  KVC_CUDA(cudaMallocHost(&hh, static_cast<std::size_t>(max_frames_)));
  host_.push_back(hh);
  h_hit_ = static_cast<std::uint8_t*>(hh);
  att_.resize(static_cast<std::size_t>(L));
  lat_.assign(static_cast<std::size_t>(L) * 5, 0.0);
  attc_.assign(static_cast<std::size_t>(L), 0);
  bnd_.assign(static_cast<std::size_t>(L), 0);
  KVC_CUDA(cudaStreamSynchronize(st_));
}

TokenContext::~TokenContext() {
  if (st_) cudaStreamSynchronize(st_);
  for (void* p : dev_) cudaFree(p);
  for (void* p : host_) cudaFreeHost(p);
  for (auto& e : ev_) cudaEventDestroy(e);
  if (st_) cudaStreamDestroy(st_);
}

// engine.cpp:153-158: every entry joins its layer's pool; the frame joins the window.
void TokenContext::ingest_frame(std::int64_t frame_id, const void* keys, const void* values, int T, int mem) {
  if (T < 1 || T > tmax_) fail(-10, "tokens per frame outside [1, max_tokens]");
  if (!keys || !values) fail(-10, "null frame buffer");
  if (frame_id < 0 || frame_id >= (1LL << 39)) fail(-10, "token baseline frame ids must be in [0, 2^39)");
  if (n_ + T > ta_.cap) fail(-21, "token pool full (raise kvc_cfg.pool_bytes)");
  const std::size_t row = static_cast<std::size_t>(T) * d_ * es_;
  const std::size_t pitch = static_cast<std::size_t>(tmax_) * d_ * es_;
  const cudaMemcpyKind kind = mem == KVC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  KVC_CUDA(cudaMemcpy2DAsync(d_fk_, pitch, keys, row, row, L_, kind, st_));
  KVC_CUDA(cudaMemcpy2DAsync(d_fv_, pitch, values, row, row, L_, kind, st_));
  launches_ += launch_tok_append(ta_, d_fk_, d_fv_, T, static_cast<int>(tmax_), n_, st_);
  const std::int64_t ord = static_cast<std::int64_t>(fid_.size());
  fid_.push_back(frame_id);
  fstart_.push_back(n_);
  ft_.push_back(T);
  std::vector<std::int32_t> fx(static_cast<std::size_t>(T), static_cast<std::int32_t>(ord));
  KVC_CUDA(cudaMemcpyAsync(d_fidx_ + n_, fx.data(), fx.size() * 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_fid_ + ord, &fid_.back(), 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_fstart_ + ord, &fstart_.back(), 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));  // pageable sources above
  KVC_CUDA(cudaGetLastError());
  n_ += T;
  window_.push_back(ord);  // engine.cpp:54-57
  while (static_cast<int>(window_.size()) > cfg_.window_frames) window_.pop_front();
}

void TokenContext::decode_step(std::int64_t qid, const float* q, int q_mem, float* out, int out_mem,
                               const std::int64_t* gt, int n_gt) {
  (void)qid;
  if (!q) fail(-10, "null query");
  const float* dq = q;
  if (q_mem != KVC_MEM_DEVICE) {
    KVC_CUDA(cudaMemcpyAsync(d_q_, q, static_cast<std::size_t>(L_) * d_ * 4, cudaMemcpyHostToDevice, st_));
  } else {
    KVC_CUDA(cudaMemcpyAsync(d_q_, dq, static_cast<std::size_t>(L_) * d_ * 4, cudaMemcpyDeviceToDevice, st_));
  }
  da_.out = (out && out_mem == KVC_MEM_DEVICE) ? out : d_out_;
  const std::int64_t win_lo = window_.empty() ? n_ : fstart_[static_cast<std::size_t>(window_.front())];
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[0], st_));
  if (n_ > 0) {
    KVC_CUDA(cudaMemsetAsync(ta_.frame_hit, 0, static_cast<std::size_t>(fid_.size()), st_));
    launches_ += launch_tok_decode(ta_, stage_, da_, n_, static_cast<int>(std::min<std::int64_t>(cfg_.token_budget, 1 << 30)),
                                   win_lo, st_);
    KVC_CUDA(cudaGetLastError());
  } else if (out) {
    KVC_CUDA(cudaMemsetAsync(da_.out, 0, static_cast<std::size_t>(L_) * d_ * 4, st_));
  }
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[1], st_));
  if (out && out_mem != KVC_MEM_DEVICE)
    KVC_CUDA(cudaMemcpyAsync(out, d_out_, static_cast<std::size_t>(L_) * d_ * 4, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(h_stats_, ta_.stats, static_cast<std::size_t>(L_) * 16, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(h_err_, ta_.err, 4, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(h_hit_, ta_.frame_hit, fid_.size(), cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));
  if (timing_) {
    float ms = 0.f;
    KVC_CUDA(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
    step_t_[1] = ms * 1e3;
  }
  if (*h_err_) {
    const int e = *h_err_;
    KVC_CUDA(cudaMemsetAsync(ta_.err, 0, 4, st_));
    KVC_CUDA(cudaStreamSynchronize(st_));
    if (e & 1) fail(-2, "cosine of zero vector");
    if (e & 64) fail(-21, "more than 1024 rows share the exact boundary value");
    fail(-1, "device error");
  }
  // latency model and ledger (retrieval.cpp:185-242): one op per run of adjacent host-side tokens
  const std::int64_t eb = cfg_.bytes_per_entry > 0 ? cfg_.bytes_per_entry : static_cast<std::int64_t>(dl_ ? dl_ : d_) * 2 * 4;
  ttft_ = 0.0;
  std::int64_t tok_total = 0;
  for (int l = 0; l < L_; ++l) {
    double* lt = &lat_[static_cast<std::size_t>(l) * 5];
    for (int i = 0; i < 5; ++i) lt[i] = 0.0;
    attc_[static_cast<std::size_t>(l)] = 0;
    if (n_ == 0) continue;  // empty pool
    const std::int64_t ops = h_stats_[l * 4 + 1], htok = h_stats_[l * 4 + 2];
    lt[0] = cfg_.lookup_cost_per_candidate_us * static_cast<double>(n_);
    lt[1] = static_cast<double>(ops) * cfg_.alpha_us + static_cast<double>(htok * eb) * cfg_.beta_us_per_byte;
    lt[4] = cfg_.compute_cost_per_token_us * static_cast<double>(h_stats_[l * 4 + 0]);
    attc_[static_cast<std::size_t>(l)] = h_stats_[l * 4 + 0];
    bnd_[static_cast<std::size_t>(l)] = h_stats_[l * 4 + 3];
    led_ops_ += ops;
    led_bytes_ += htok * eb;
    led_cost_ += lt[1];
    tok_total += h_stats_[l * 4 + 0];
    ttft_ += lt[0] + lt[1] + lt[2] + lt[3] + lt[4];
  }
  step_t_[4] = static_cast<double>(tok_total) * 2.0 * d_ * es_;
  recall_ = -1.0;
  if (gt && n_gt > 0) {
    std::vector<std::int64_t> ctx;
    for (std::size_t o = 0; o < fid_.size(); ++o)
      if (h_hit_[o]) ctx.push_back(fid_[o]);
    std::sort(ctx.begin(), ctx.end());
    std::int64_t hit = 0;
    for (int i = 0; i < n_gt; ++i)
      if (std::binary_search(ctx.begin(), ctx.end(), gt[i])) hit += 1;
    recall_ = static_cast<double>(hit) / static_cast<double>(n_gt);
  }
  fetched_.clear();
  context_.clear();
  if (cfg_.parity_mode) {  // attended (frame, token) lists and the digest
    std::vector<std::uint32_t> w(static_cast<std::size_t>(L_) * ta_.wcap), pk(static_cast<std::size_t>(L_) * ta_.wcap);
    KVC_CUDA(cudaMemcpyAsync(w.data(), ta_.attw, w.size() * 4, cudaMemcpyDeviceToHost, st_));
    KVC_CUDA(cudaMemcpyAsync(pk.data(), ta_.pick, pk.size() * 4, cudaMemcpyDeviceToHost, st_));
    KVC_CUDA(cudaStreamSynchronize(st_));
    // fetched_frames: frames of the picked tokens (retrieval.cpp:210-213); context_frames: frames
    // with attended entries
    for (std::size_t o = 0; o < fid_.size(); ++o) {
      if (h_hit_[o]) context_.push_back(fid_[o]);
      bool picked = false;
      for (int l = 0; l < L_ && !picked; ++l)
        for (std::int64_t i = fstart_[o]; i < fstart_[o] + ft_[o] && !picked; ++i)
          picked = (pk[static_cast<std::size_t>(l) * ta_.wcap + i / 32] >> (i % 32)) & 1u;
      if (picked) fetched_.push_back(fid_[o]);
    }
    std::sort(context_.begin(), context_.end());
    std::sort(fetched_.begin(), fetched_.end());
    std::uint64_t h = 1469598103934665603ull;
    for (int l = 0; l < L_; ++l) {
      auto& a = att_[static_cast<std::size_t>(l)];
      a.clear();
      std::size_t o = 0;
      for (std::int64_t i = 0; i < n_; ++i) {
        if (!((w[static_cast<std::size_t>(l) * ta_.wcap + i / 32] >> (i % 32)) & 1u)) continue;
        while (o + 1 < fstart_.size() && fstart_[o + 1] <= i) ++o;
        a.push_back({fid_[o], static_cast<std::int32_t>(i - fstart_[o])});
      }
      std::sort(a.begin(), a.end());
      for (const auto& x : a) {
        h = fnv1a(h, static_cast<std::uint64_t>(l));
        h = fnv1a(h, static_cast<std::uint64_t>(x.first));
        h = fnv1a(h, static_cast<std::uint64_t>(x.second));
      }
    }
    digest_ = h;
  }
}

int TokenContext::attended(int layer, std::int64_t* frames, std::int32_t* tokens, int cap) const {
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range");
  const auto& a = att_[static_cast<std::size_t>(layer)];
  const int n = static_cast<int>(a.size());
  for (int i = 0; i < n && i < cap; ++i) {
    frames[i] = a[static_cast<std::size_t>(i)].first;
    tokens[i] = a[static_cast<std::size_t>(i)].second;
  }
  return n;
}

void TokenContext::layer_meta(int layer, double* lat, std::int64_t* ints) const {
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range");
  for (int i = 0; i < 5; ++i) lat[i] = lat_[static_cast<std::size_t>(layer) * 5 + i];
  ints[0] = ints[1] = ints[2] = 0;
  ints[3] = bnd_[static_cast<std::size_t>(layer)];  // (token mode) rows re-scored exactly at the boundary
  ints[4] = attc_[static_cast<std::size_t>(layer)];
}

std::int64_t TokenContext::ledger(std::int64_t* ops, std::int64_t* bytes, double* cost) const {
  for (int i = 0; i < 5; ++i) {
    ops[i] = 0;
    bytes[i] = 0;
    cost[i] = 0.0;
  }
  ops[0] = led_ops_;  // TransferCause::Retrieval
  bytes[0] = led_bytes_;
  cost[0] = led_cost_;
  return 0;
}

void TokenContext::profile(double* out) {
  std::vector<long long> p(static_cast<std::size_t>(L_) * 8);
  KVC_CUDA(cudaMemcpyAsync(p.data(), ta_.prof, p.size() * 8, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));
  for (int k = 0; k < 8; ++k) {
    double s = 0.0;
    for (int l = 0; l < L_; ++l) s += static_cast<double>(p[static_cast<std::size_t>(l) * 8 + k]);
    out[k] = s / L_;
  }
}

void TokenContext::set_head_dim(int d_logical) {
  if (d_logical < 1 || d_logical > d_) fail(-10, "head width must be in [1, d]");
  dl_ = d_logical;
  da_.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d_logical)));
}

}  // namespace kvc
