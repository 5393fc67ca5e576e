// context.cpp -- host control plane of one stream (see context.hpp).
//
// Reference semantics followed (paths under /root/reference/proj/core):
//   engine.cpp:54-174     window / repin / build / cadence / ingest order
//   engine.cpp:176-237    query path
//   maintainer.cpp:37-242 placement, insert branches (decided on the GPU, replayed here),
//                         split_members / materialize (host slow path)
//   store.cpp:67-189      residency state machine and ledger arithmetic
//   retrieval.cpp:45-143  per-layer bookkeeping around the GPU rankings
//   index.cpp:97-190      cluster registration, frame -> cluster map, buffers
#include "context.hpp"

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include "kmeans.hpp"

namespace kvc {

namespace {

inline double tau_of(std::int64_t n, const kvc_cfg& c) {  // maintainer.cpp:11-14
  return c.tau_min + (c.tau_max - c.tau_min) * std::exp(-static_cast<double>(n) / c.n0);
}

inline float bf16_to_f32(std::uint16_t h) {
  std::uint32_t u = static_cast<std::uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

void rows_to_f32(const void* src, int bf16, std::size_t n, float* dst) {
  if (!bf16) {
    std::memcpy(dst, src, n * sizeof(float));
    return;
  }
  const auto* h = static_cast<const std::uint16_t*>(src);
  for (std::size_t i = 0; i < n; ++i) dst[i] = bf16_to_f32(h[i]);
}

}  // namespace

// ============================================================================ lifetime

Context::Context(const kvc_cfg& cfg, int d, int L) : cfg_(cfg), d_(d), L_(L), dl_(d) {
  // EngineConfig::validate (engine.cpp:9-14), RetrievalConfig::validate (retrieval.cpp:10-16)
  if (cfg_.k_v <= 0 || cfg_.k_s <= 0 || cfg_.window_frames <= 0 || cfg_.prefetch_k <= 0)
    fail(-10, "retrieval budgets must be positive");
  if (cfg_.token_budget < 1) fail(-10, "token budget must be at least 1");
  if (cfg_.lookup_cost_per_candidate_us < 0.0 || cfg_.compute_cost_per_token_us < 0.0)
    fail(-10, "cost constants must be non-negative");
  if (cfg_.build_batch_frames < 1) fail(-10, "build batch must be at least 1 frame");
  if (cfg_.ingest_overhead_us < 0.0) fail(-10, "ingestion overhead must be non-negative");
  if (cfg_.offload_horizon_frames < 1) fail(-10, "offload horizon must be at least 1 frame");
  if (d < 1 || L < 1) fail(-10, "stream dimensions must be positive");
  // TieredStore / Maintainer constructor checks (store.cpp:67-74, maintainer.cpp:27-35)
  if (cfg_.alpha_us < 0.0 || cfg_.beta_us_per_byte < 0.0) fail(-10, "transfer costs must be non-negative");
  if (cfg_.device_capacity_entries <= 0) fail(-10, "device capacity must be positive");
  if (cfg_.tau_min < 0.0 || cfg_.tau_max < cfg_.tau_min)
    fail(-10, "variance thresholds must satisfy 0 <= tau_min <= tau_max");
  if (cfg_.n0 <= 0.0) fail(-10, "threshold horizon must be positive");
  if (cfg_.max_split_depth < 1) fail(-10, "split depth must be at least 1");
  if (cfg_.visual_floor < -1.0 || cfg_.visual_floor > 1.0) fail(-10, "visual floor must be a cosine value");
  if (cfg_.token_mode) fail(-10, "token-baseline mode is served by TokenContext (kvc_create dispatches on cfg.token_mode)");
  if (cfg_.kv_dtype != KVC_DTYPE_F32 && cfg_.kv_dtype != KVC_DTYPE_BF16) fail(-10, "kv_dtype");
  // (<= 64: a window page's dedup mask is one 64-bit word of its attention descriptor)
  if (cfg_.page_tokens != 0 && (cfg_.page_tokens < 8 || cfg_.page_tokens > 64 || cfg_.page_tokens % 8))
    fail(-10, "page_tokens must be 0 (auto) or 8..64, a multiple of 8");
  if (cfg_.max_candidates < 1 || cfg_.max_candidates > 6144)
    fail(-10, "max_candidates must be 1..6144 (the ingest top-M keeps 8 candidate rows in shared memory)");
  if (d % 8 != 0 || d > 256) fail(-10, "the device path supports d % 8 == 0 and d <= 256");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(-22, "no CUDA device: the B200 path has no CPU fallback");
  es_ = cfg_.kv_dtype == KVC_DTYPE_BF16 ? 2 : 4;
  if (cfg_.page_tokens == 0) cfg_.page_tokens = auto_page_tokens(d, cfg_.kv_dtype == KVC_DTYPE_BF16);
  if (d == 32 || d == 64 || d == 128 || d == 256) {
    // K6 stages whole pages (K + V) in shared memory: e.g. fp32, d = 256, 64-token pages needs
    // 2 x 128 KB, more than a CTA can have -- reject here instead of failing every decode step
    const std::size_t att = attend_smem_bytes(d, cfg_.page_tokens, cfg_.kv_dtype == KVC_DTYPE_BF16);
    if (att > static_cast<std::size_t>(device_smem_optin()))
      fail(-10, "page_tokens * d * sizeof(kv) too large for the attention kernel's shared-memory ring (" +
                    std::to_string(att) + " B > " + std::to_string(device_smem_optin()) +
                    " B per CTA): use a smaller page_tokens");
  }
  try {
    KVC_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    for (auto& e : ev_) KVC_CUDA(cudaEventCreate(&e));
    alloc_device();
    upload_tau();
  } catch (...) {  // a failed construction (e.g. the pool does not fit) releases what it took
    release();
    throw;
  }
  mstats_[0] = 0;
  last_.resize(static_cast<std::size_t>(L_));
}

Context::~Context() { release(); }

void Context::release() {
  if (st_) cudaStreamSynchronize(st_);
  waves_free();
  if (spec_st_) {
    cudaStreamSynchronize(spec_st_);
    cudaStreamDestroy(spec_st_);
  }
  if (spec_.ev) cudaEventDestroy(spec_.ev);
  if (xs_) {
    cudaStreamSynchronize(xs_);
    cudaStreamDestroy(xs_);
  }
  for (const TierBatch& b : tier_fl_)
    if (b.ev) cudaEventDestroy(b.ev);
  for (cudaEvent_t e : tier_ev_free_) cudaEventDestroy(e);
  for (void* p : dev_allocs_) cudaFree(p);
  for (void* p : host_allocs_) cudaFreeHost(p);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_step_)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_k4_)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_out_)
    if (e) cudaEventDestroy(e);
  if (cs_) cudaStreamDestroy(cs_);
  if (in_st_) {
    cudaStreamSynchronize(in_st_);
    cudaStreamDestroy(in_st_);
  }
  if (ev_init_) cudaEventDestroy(ev_init_);
  for (cudaEvent_t e : ev_act_)
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t e : {ev_ing_[b], ev_in_[b], ev_buf_[b]})
      if (e) cudaEventDestroy(e);
  for (auto& row : evb_)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  if (st_) cudaStreamDestroy(st_);
  cudaGetLastError();  // nothing of a released context may surface in a later launch check
}

void* Context::dalloc(std::size_t bytes) {
  void* p = nullptr;
  KVC_CUDA(cudaMalloc(&p, std::max<std::size_t>(bytes, 16)));
  KVC_CUDA(cudaMemsetAsync(p, 0, std::max<std::size_t>(bytes, 16), st_));
  dev_allocs_.push_back(p);
  return p;
}

void* Context::dalloc_scratch(std::size_t bytes) {
  if (bytes > scratch_cap_) {
    scratch_cap_ = std::max(bytes, scratch_cap_ * 2);
    scratch_ = dalloc(scratch_cap_);
  }
  return scratch_;
}

void* Context::halloc(std::size_t bytes) {
  void* p = nullptr;
  KVC_CUDA(cudaMallocHost(&p, std::max<std::size_t>(bytes, 16)));
  std::memset(p, 0, std::max<std::size_t>(bytes, 16));
  host_allocs_.push_back(p);
  return p;
}

void Context::alloc_device() {
  const std::int64_t S = cfg_.max_slots, d = d_, L = L_;
  t_.d = d_;
  t_.L = L_;
  t_.P = cfg_.page_tokens;
  t_.es = es_;
  t_.kv_bf16 = cfg_.kv_dtype == KVC_DTYPE_BF16;
  t_.max_slots = cfg_.max_slots;
  t_.maxp = cfg_.max_cluster_pages;
  t_.maxbp = cfg_.max_buffer_pages;
  t_.max_parts = cfg_.max_partitions;
  t_.cmax = cfg_.max_candidates;
  t_.tmax = cfg_.max_tokens;
  t_.W = cfg_.window_frames;
  t_.page_bytes = 2LL * t_.P * d * es_;
  t_.rpp = (t_.tmax + t_.P - 1) / t_.P;
  const std::int64_t ring_pages = L * t_.W * t_.rpp;
  t_.max_pages = cfg_.max_pages > 0 ? cfg_.max_pages : cfg_.pool_bytes / t_.page_bytes;
  if (t_.max_pages <= ring_pages + 16) fail(-21, "page pool too small for the window ring");
  t_.max_hpages = cfg_.host_pool_bytes > 0 ? cfg_.host_pool_bytes / t_.page_bytes : 0;
  if (t_.max_pages + t_.max_hpages >= (1LL << 31)) fail(-10, "page pool + host tier exceed 2^31 pages");

  t_.rep64 = static_cast<double*>(dalloc(S * d * 8));
  t_.rep32 = static_cast<float*>(dalloc(S * d * 4));
  t_.rnorm = static_cast<double*>(dalloc(S * 8));
  t_.brep64 = static_cast<double*>(dalloc(S * d * 8));
  t_.brep32 = static_cast<float*>(dalloc(S * d * 4));
  t_.bnorm = static_cast<double*>(dalloc(S * 8));
  t_.var = static_cast<double*>(dalloc(S * 8));
  t_.stat = static_cast<std::int64_t*>(dalloc(S * 8));
  t_.nmem = static_cast<std::int64_t*>(dalloc(S * 8));
  t_.nbuf = static_cast<std::int32_t*>(dalloc(S * 4));
  t_.lazy = static_cast<std::uint8_t*>(dalloc(S));
  t_.resid = static_cast<std::uint8_t*>(dalloc(S));
  t_.cid = static_cast<std::int64_t*>(dalloc(S * 8));
  t_.npages = static_cast<std::int32_t*>(dalloc(S * 4));
  t_.pages = static_cast<std::int32_t*>(dalloc(S * t_.maxp * 4));
  t_.nbpages = static_cast<std::int32_t*>(dalloc(S * 4));
  t_.bpages = static_cast<std::int32_t*>(dalloc(S * t_.maxbp * 4));
  t_.pg_fill = static_cast<std::int32_t*>(dalloc((t_.max_pages + t_.max_hpages) * 4));
  t_.free_stack = static_cast<std::int32_t*>(dalloc(t_.max_pages * 4));
  t_.free_top = static_cast<std::int32_t*>(dalloc(16));
  t_.pool = static_cast<std::uint8_t*>(dalloc(static_cast<std::size_t>(t_.max_pages) * t_.page_bytes));
  t_.ring_pages = static_cast<std::int32_t*>(dalloc(ring_pages * 4));
  t_.ring_owner = static_cast<std::int32_t*>(dalloc(L * t_.W * t_.tmax * 4));
  t_.ring_count = static_cast<std::int32_t*>(dalloc(t_.W * 4));
  t_.vrep = static_cast<double*>(dalloc(static_cast<std::int64_t>(t_.max_parts) * d * 8));
  t_.vnorm = static_cast<double*>(dalloc(static_cast<std::int64_t>(t_.max_parts) * 8));
  t_.n_parts = static_cast<std::int32_t*>(dalloc(16));
  t_.pl_off = static_cast<std::int32_t*>(dalloc(static_cast<std::int64_t>(t_.max_parts) * L * 4));
  t_.pl_cnt = static_cast<std::int32_t*>(dalloc(static_cast<std::int64_t>(t_.max_parts) * L * 4));
  t_.pl_pool_cap = S * 4 + 1024;
  t_.pl_pool = static_cast<std::int32_t*>(dalloc(t_.pl_pool_cap * 4));
  h_err_ = static_cast<std::int32_t*>(halloc(16));
  tier_alloc();

  // page stack: ring pages are [0, ring_pages); the stack holds the rest
  {
    std::vector<std::int32_t> stack(static_cast<std::size_t>(t_.max_pages - ring_pages));
    for (std::size_t i = 0; i < stack.size(); ++i)
      stack[i] = static_cast<std::int32_t>(t_.max_pages - 1 - static_cast<std::int64_t>(i));
    KVC_CUDA(cudaMemcpyAsync(t_.free_stack, stack.data(), stack.size() * 4, cudaMemcpyHostToDevice, st_));
    std::int32_t top = static_cast<std::int32_t>(stack.size());
    KVC_CUDA(cudaMemcpyAsync(t_.free_top, &top, 4, cudaMemcpyHostToDevice, st_));
    std::vector<std::int32_t> rp(static_cast<std::size_t>(ring_pages));
    std::iota(rp.begin(), rp.end(), 0);
    KVC_CUDA(cudaMemcpyAsync(t_.ring_pages, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice, st_));
    ring_owner_h_.assign(static_cast<std::size_t>(L * t_.W * t_.tmax), -1);
    ring_frame_.assign(static_cast<std::size_t>(t_.W), RingFrame{});
    KVC_CUDA(cudaMemcpyAsync(t_.ring_owner, ring_owner_h_.data(), ring_owner_h_.size() * 4, cudaMemcpyHostToDevice, st_));
    // dalloc zero-fills on st_ (a non-blocking stream): every initial upload goes on st_ too and
    // completes before the pageable sources die
    KVC_CUDA(cudaStreamSynchronize(st_));
  }
  slot_id_.assign(static_cast<std::size_t>(S), -1);
  free_slots_.resize(static_cast<std::size_t>(S));
  for (std::int64_t i = 0; i < S; ++i) free_slots_[static_cast<std::size_t>(i)] = static_cast<std::int32_t>(S - 1 - i);
  resid_h_.assign(static_cast<std::size_t>(S), 0);
  layer_live_count_.assign(static_cast<std::size_t>(L), 0);

  // frame input (kv dtype, [L][tmax][d])
  const std::size_t frame_bytes = static_cast<std::size_t>(L) * t_.tmax * d * es_;
  for (int b = 0; b < 2; ++b) {  // double-buffered frame input (pipelined ingest)
    fkbuf_[b] = dalloc(frame_bytes);
    fvbuf_[b] = dalloc(frame_bytes);
  }
  d_fk_ = fkbuf_[0];
  d_fv_ = fvbuf_[0];
  ensure_stage(static_cast<std::int64_t>(t_.maxp + t_.maxbp) * t_.P + 1);
  ensure_idx(1 << 16, 1 << 12);

  // ingest arrays
  ia_.cand_n = static_cast<std::int32_t*>(dalloc(L * 4));
  ia_.cand_slot = static_cast<std::int32_t*>(dalloc(L * t_.cmax * 4));
  ia_.cand_buf = static_cast<std::uint8_t*>(dalloc(L * t_.cmax));
  ia_.approx = static_cast<float*>(dalloc(L * t_.tmax * t_.cmax * 4));
  // outcome words in one block (ev_kind | ev_slot | stop_t | stop_kind | stop_slot): one D2H per launch
  // ... | error word | tie flags [L] (k_resolve)
  ia_.ev_kind = static_cast<std::int32_t*>(dalloc(L * t_.tmax * 4 * 2 + L * 4 * 4 + 16));
  ia_.ev_slot = ia_.ev_kind + L * t_.tmax;
  ia_.stop_t = ia_.ev_slot + L * t_.tmax;
  ia_.stop_kind = ia_.stop_t + L;
  ia_.stop_slot = ia_.stop_t + 2 * L;
  ia_.n_exact = static_cast<std::int32_t*>(dalloc(L * 4));
  ia_.topm_idx = static_cast<std::int16_t*>(dalloc(L * t_.tmax * TOPM * 2));
  ia_.topm_val = static_cast<float*>(dalloc(L * t_.tmax * TOPM * 4));
  ia_.topm_next = static_cast<float*>(dalloc(L * t_.tmax * 4));
  ia_.topm_exact = static_cast<double*>(dalloc(L * t_.tmax * TOPM * 8));
  ia_.ev_page = static_cast<std::int32_t*>(dalloc(L * t_.tmax * 4));
  ia_.ev_row = static_cast<std::int32_t*>(dalloc(L * t_.tmax * 4));
  ia_.dom_pool = static_cast<std::int32_t*>(dalloc(L * POOL * 4));
  ia_.prof = static_cast<long long*>(dalloc(L * 16 * 8));
  ia_.dom_pool_n = static_cast<std::int32_t*>(dalloc(L * 4));
  ia_.rsnap = static_cast<double*>(dalloc(static_cast<std::int64_t>(L) * d * t_.tmax * 8));
  ia_.bsnap = static_cast<double*>(dalloc(static_cast<std::int64_t>(L) * d * t_.tmax * 8));
  {
    const char* e = std::getenv("KVC_RESOLVE");  // "seq": the sequential resolve kernel
    resolve_seq_ = e && std::string(e) == "seq";
    const char* rl = std::getenv("KVC_RELAUNCH");  // "seq": the sequential kernel for relaunches
    relaunch_seq_ = rl && std::string(rl) == "seq";
    const char* wv = std::getenv("KVC_WAVES");  // 0: settle host events one domain at a time
    waves_ = !(wv && std::string(wv) == "0");
    const char* wp = std::getenv("KVC_WAVES_PERTURB");
    waves_perturb_ = wp && std::string(wp) == "1";
    const char* wl = std::getenv("KVC_WAVES_LOG");
    waves_log_ = wl && std::string(wl) == "1";
    const char* we = std::getenv("KVC_WAVES_EAGER");
    waves_eager_ = we && std::string(we) == "1";
    const char* ss = std::getenv("KVC_SPEC_SPLIT");  // 0: no speculative split k-means
    spec_split_ = !(ss && std::string(ss) == "0");
    const char* g = std::getenv("KVC_ASSIGN");  // "simt": the fp32 CUDA-core tile
    assign_tc_ = !(g && std::string(g) == "simt") && assign_tc_supported(t_) &&
                 make_key_tensor_map(key_maps_[0], fkbuf_[0], d, t_.tmax, L) &&
                 make_key_tensor_map(key_maps_[1], fkbuf_[1], d, t_.tmax, L);
    std::memcpy(key_map_, key_maps_[0], sizeof(key_map_));
    const char* sp = std::getenv("KVC_INGEST_SPEC");  // 0: no speculative next-frame round
    spec_ingest_ = !(sp && std::string(sp) == "0");
    const char* sm = std::getenv("KVC_SPLIT_DEV_MIN");  // smallest group split on the GPU (0: never)
    if (sm) split_dev_min_ = std::atoi(sm);
  }
  d_active_ = static_cast<std::int32_t*>(dalloc(L * 4 * 2));
  d_cursor_ = d_active_ + L;
  h_active_ = static_cast<std::int32_t*>(halloc(L * 4 * 2 * kActSlots));  // kActSlots staging slots
  h_cursor_ = h_active_ + L;
  d_evflags_ = static_cast<std::int32_t*>(dalloc(16));  // per frame buffer: first round stopped
  for (int b = 0; b < 2; ++b) {
    h_out_[b] = static_cast<std::int32_t*>(halloc(L * t_.tmax * 4 * 2 + L * 4 * 4 + 16));
    h_errb_[b] = static_cast<std::int32_t*>(halloc(16));
    KVC_CUDA(cudaEventCreateWithFlags(&ev_ing_[b], cudaEventDisableTiming));
    if (b == 0) KVC_CUDA(cudaEventCreateWithFlags(&ev_init_, cudaEventDisableTiming));
    KVC_CUDA(cudaEventCreateWithFlags(&ev_in_[b], cudaEventDisableTiming));
    KVC_CUDA(cudaEventCreateWithFlags(&ev_buf_[b], cudaEventDisableTiming));
    KVC_CUDA(cudaEventRecord(ev_buf_[b], st_));
  }
  h_evk_ = h_out_[0];
  h_evs_ = h_evk_ + L * t_.tmax;
  h_stop_ = h_evs_ + L * t_.tmax;
  ia_.active = d_active_;
  ia_.cursor = d_cursor_;
  ia_.err_copy = ia_.ev_kind + 2 * static_cast<std::int64_t>(L) * t_.tmax + 3 * L;
  ia_.tie = ia_.err_copy + 1;
  // every domain from token 0 (a frame's first round): constant device arrays, no staging copy
  d_all_active_ = static_cast<std::int32_t*>(dalloc(L * 4 * 2));
  {
    std::vector<std::int32_t> h(static_cast<std::size_t>(2 * L), 0);
    for (int l = 0; l < L; ++l) h[static_cast<std::size_t>(l)] = l;
    KVC_CUDA(cudaMemcpyAsync(d_all_active_, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st_));
    KVC_CUDA(cudaStreamSynchronize(st_));
  }
  ia_.fk = d_fk_;
  ia_.fv = d_fv_;
  ia_.defer = cfg_.defer_host_splits;

  // decode result block
  // ranked lists never exceed the candidate count (take = min(k, candidates)), so the result
  // blocks are sized by the clamped budgets (k_s = 10^6 "exhaustive" budgets stay small)
  const std::int32_t kv = std::min(cfg_.k_v, t_.max_parts), ks = std::min(cfg_.k_s, t_.cmax),
                     kp = std::min(cfg_.prefetch_k, t_.cmax);
  da_.chunk_pages = 8;
  da_.max_desc = 4096;
  da_.max_items = da_.max_desc / da_.chunk_pages;
  t_.err = static_cast<std::int32_t*>(dalloc(16));
  KVC_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
  KVC_CUDA(cudaStreamCreateWithFlags(&in_st_, cudaStreamNonBlocking));
  alloc_result_blocks(kv, ks, kp);
  for (int b = 0; b < 2; ++b) {
    KVC_CUDA(cudaEventCreateWithFlags(&ev_k4_[b], cudaEventDisableTiming));
    KVC_CUDA(cudaEventCreateWithFlags(&ev_out_[b], cudaEventDisableTiming));
    KVC_CUDA(cudaEventCreateWithFlags(&ev_step_[b], cudaEventDisableTiming));
    for (auto& e : evb_[b]) KVC_CUDA(cudaEventCreate(&e));
  }
  set_result_block(0);
  da_.desc = static_cast<int4*>(dalloc(L * da_.max_desc * sizeof(int4)));
  da_.n_desc = static_cast<std::int32_t*>(dalloc(L * 4));
  da_.n_items = static_cast<std::int32_t*>(dalloc(L * 4));
  da_.part_ml = static_cast<float*>(dalloc(L * da_.max_items * 2 * 4));
  da_.part_o = static_cast<float*>(dalloc(L * da_.max_items * d * 4));
  da_.dom_done = static_cast<std::int32_t*>(dalloc(L * 4));
  da_.k4prof = static_cast<long long*>(dalloc(L * 16 * 8));
  da_.work_ctr = static_cast<std::int32_t*>(dalloc(64));
  da_.k_v = kv;
  da_.k_s = ks;
  da_.prefetch_k = kp;
  da_.prefetch = cfg_.prefetch_enabled;
  da_.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d)));
  {
    const char* e = std::getenv("KVC_ATT_DEBUG");  // bit 0: attention consumers skip the math
    da_.debug_flags = e ? std::atoi(e) : 0;
    const char* pf = std::getenv("KVC_ATT_PF");  // K6: L2 prefetch distance in pages (0: off)
    da_.att_pf = pf ? std::atoi(pf) : 0;
  }
  d_q_ = static_cast<float*>(dalloc(L * d * 4));
  d_out_ = static_cast<float*>(dalloc(L * d * 4));
  if (t_.max_hpages > 0) {  // fetch-on-read (DecodeArgs::fr_*): copy lists, one per domain
    const char* e = std::getenv("KVC_FETCH_ON_READ");
    fr_enabled_ = !(e && e[0] == '0');
    da_.fr_jobs = static_cast<int4*>(dalloc(L * da_.max_desc * sizeof(int4)));
    da_.fr_nj = static_cast<std::int32_t*>(dalloc(L * 4));
    da_.fr_reserve = static_cast<std::int32_t>(std::min<std::int64_t>(t_.max_pages / 16 + 2LL * t_.maxp, t_.max_pages));
  } else {
    fr_enabled_ = false;
  }
  KVC_CUDA(cudaStreamSynchronize(st_));
}

void Context::upload_tau() {
  const std::int64_t len = static_cast<std::int64_t>(t_.maxp) * t_.P + 2;
  tau_host_.resize(static_cast<std::size_t>(len));
  for (std::int64_t n = 0; n < len; ++n) tau_host_[static_cast<std::size_t>(n)] = tau_of(n, cfg_);
  t_.tau_tab = static_cast<double*>(dalloc(len * 8));
  t_.tau_len = static_cast<std::int32_t>(len);
  KVC_CUDA(cudaMemcpyAsync(t_.tau_tab, tau_host_.data(), len * 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));
}

void Context::ensure_stage(std::int64_t rows) {
  if (rows <= stage_rows_) return;
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  stage_rows_ = std::max<std::int64_t>(rows, stage_rows_ * 2);
  // old buffers stay allocated until destruction (rare growth)
  d_stage_k_ = dalloc(stage_rows_ * rb);
  d_stage_v_ = dalloc(stage_rows_ * rb);
  d_stage_f32_ = static_cast<float*>(dalloc(stage_rows_ * d_ * 4));
  h_stage_f32_ = static_cast<float*>(halloc(stage_rows_ * d_ * 4));
}

void Context::ensure_idx(std::int64_t n, std::int64_t runs) {
  if (n > idx_cap_) {
    idx_cap_ = std::max(n, idx_cap_ * 2);
    d_idx_ = static_cast<std::int32_t*>(dalloc(idx_cap_ * 4));
    h_idx_ = static_cast<std::int32_t*>(halloc(idx_cap_ * 4));
  }
  if (runs > runs_cap_) {
    runs_cap_ = std::max(runs, runs_cap_ * 2);
    d_runs_ = static_cast<AppendRun*>(dalloc(runs_cap_ * sizeof(AppendRun)));
    h_runs_ = static_cast<AppendRun*>(halloc(runs_cap_ * sizeof(AppendRun)));
  }
}

void Context::debug_assign_check(const void* keys, int T, std::int64_t pid, int mem, double* out) {
  if (T < 1 || T > t_.tmax) fail(-10, "tokens per frame outside [1, max_tokens]");
  tier_kick();
  if (pid < 0 || pid >= static_cast<std::int64_t>(parts_.size())) fail(-3, "unknown partition");
  flush_pending();
  const std::size_t row = static_cast<std::size_t>(T) * d_ * es_;
  const std::size_t pitch = static_cast<std::size_t>(t_.tmax) * d_ * es_;
  const cudaMemcpyKind kind = mem == KVC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  KVC_CUDA(cudaMemcpy2DAsync(d_fk_, pitch, keys, row, row, L_, kind, st_));
  flush_resid();
  ia_.T = T;
  ia_.pid = static_cast<std::int32_t>(pid);
  ia_.n_active = L_;
  ia_.active = d_active_;
  ia_.cursor = d_cursor_;
  ia_.my_events = nullptr;
  for (int l = 0; l < L_; ++l) {
    h_active_[l] = l;
    h_cursor_[l] = 0;
  }
  KVC_CUDA(cudaMemcpyAsync(d_active_, h_active_, L_ * 8, cudaMemcpyHostToDevice, st_));
  launches_ += launch_build_cands(t_, ia_, st_);
  if (assign_tc_) {
    ia_.margin = kTcMargin;
    launches_ += launch_assign_tc(t_, ia_, key_map_, st_);
  } else {
    ia_.margin = kSimtMargin;
    launches_ += launch_approx(t_, ia_, st_);
    launches_ += launch_topm(t_, ia_, st_);
  }
  if (!d_check_) d_check_ = dalloc(64);
  unsigned long long* dres = static_cast<unsigned long long*>(d_check_);
  KVC_CUDA(cudaMemsetAsync(dres, 0, 24, st_));
  launches_ += launch_assign_err(t_, ia_, dres, st_);
  unsigned long long h[3];
  KVC_CUDA(cudaMemcpyAsync(h, dres, 24, cudaMemcpyDeviceToHost, st_));
  sync();
  check_dev_err();
  double e;
  std::memcpy(&e, &h[0], 8);
  out[0] = e;
  out[1] = static_cast<double>(h[1]);
  out[2] = static_cast<double>(h[2]);
  out[3] = ia_.margin;
}

// Points the decode arguments' result fields at device result block b (two blocks: the kernels
// of step i+1 write one while step i's block is copied to the host and replayed).
// Decode result blocks (device + pinned host, double-buffered): the step's ranked / prefetch /
// verified lists and counters, carved for budgets kv / ks / kp per domain.
void Context::alloc_result_blocks(std::int32_t kv, std::int32_t ks, std::int32_t kp) {
  const std::size_t L = static_cast<std::size_t>(L_);
  std::size_t off = 0;
  auto carve = [&](std::size_t bytes) {
    std::size_t o = off;
    off += (bytes + 15) & ~std::size_t(15);
    return o;
  };
  const std::size_t o_parts = carve(L * kv * 4), o_nps = carve(L * 4), o_rs = carve(L * ks * 4),
                    o_rb = carve(L * ks), o_nr = carve(L * 4), o_ps = carve(L * kp * 4),
                    o_pb = carve(L * kp), o_np = carve(L * 4), o_vs = carve(L * ks * 4),
                    o_nv = carve(L * 4), o_att = carve(L * 8), o_nc = carve(L * 4), o_fl = carve(L * 4), o_ew = carve(L * 4),
                    o_frn = carve(L * 4);
  dec_lean_bytes_ = off;  // the fetch-on-read records go last: copied only by steps that use them
  const std::size_t o_frr = carve(L * std::min<std::int32_t>(std::max<std::int32_t>(ks, 1), 64) * 16);
  dec_bytes_ = off;
  res_off_ = {o_parts, o_nps, o_rs, o_rb, o_nr, o_ps, o_pb, o_np, o_vs, o_nv, o_att, o_nc, o_fl, o_ew, o_frn, o_frr};
  for (int b = 0; b < 2; ++b) {
    d_blk_[b] = dalloc(dec_bytes_);
    h_blk_[b] = halloc(dec_bytes_);
  }
  kv_cap_ = kv;
  ks_cap_ = ks;
  kp_cap_ = kp;
  set_result_block(cur_);
}

void Context::set_result_block(int b) {
  auto* base = static_cast<std::uint8_t*>(d_blk_[b]);
  const ResultOffsets& o = res_off_;
  da_.parts = reinterpret_cast<std::int32_t*>(base + o.parts);
  da_.n_parts_sel = reinterpret_cast<std::int32_t*>(base + o.nps);
  da_.ranked_slot = reinterpret_cast<std::int32_t*>(base + o.rs);
  da_.ranked_buf = base + o.rb;
  da_.n_ranked = reinterpret_cast<std::int32_t*>(base + o.nr);
  da_.pf_slot = reinterpret_cast<std::int32_t*>(base + o.ps);
  da_.pf_buf = base + o.pb;
  da_.n_pf = reinterpret_cast<std::int32_t*>(base + o.np);
  da_.ver_slot = reinterpret_cast<std::int32_t*>(base + o.vs);
  da_.n_ver = reinterpret_cast<std::int32_t*>(base + o.nv);
  da_.attended = reinterpret_cast<std::int64_t*>(base + o.att);
  da_.n_cand = reinterpret_cast<std::int32_t*>(base + o.nc);
  da_.flags = reinterpret_cast<std::int32_t*>(base + o.fl);
  da_.errw = reinterpret_cast<std::int32_t*>(base + o.ew);
  da_.fr_n = reinterpret_cast<std::int32_t*>(base + o.frn);
  da_.fr_rec = reinterpret_cast<int4*>(base + o.frr);
  da_.fr_max = std::min<std::int32_t>(std::max<std::int32_t>(ks_cap_, 1), 64);
  d_dec_ = d_blk_[b];
}

void Context::resolve_profile(double* out) {
  const bool dec = out[0] < 0;
  const int W = 16;  // K4 and resolve: [L][16]
  std::vector<long long> p(static_cast<std::size_t>(L_) * W);
  KVC_CUDA(cudaMemcpyAsync(p.data(), dec ? da_.k4prof : ia_.prof, p.size() * 8, cudaMemcpyDeviceToHost, st_));
  sync();
  for (int k = 0; k < 16; ++k) {
    double s = 0.0;
    if (k < W)
      for (int l = 0; l < L_; ++l) s += static_cast<double>(p[static_cast<std::size_t>(l) * W + k]);
    out[k] = s / L_;
  }
  if (dec) {  // K4 v3 global-timer stamps: block-start skew, span, mean block duration (ns)
    long long s0 = LLONG_MAX, s1 = LLONG_MIN, e1 = LLONG_MIN;
    double dur = 0.0;
    for (int l = 0; l < L_; ++l) {
      const long long a0 = p[static_cast<std::size_t>(l) * W + 13], a1 = p[static_cast<std::size_t>(l) * W + 14];
      s0 = std::min(s0, a0);
      s1 = std::max(s1, a0);
      e1 = std::max(e1, a1);
      dur += static_cast<double>(a1 - a0);
    }
    out[13] = static_cast<double>(s1 - s0);
    out[14] = static_cast<double>(e1 - s0);
    out[15] = dur / L_;
  }
}

void Context::sync() { KVC_CUDA(cudaStreamSynchronize(st_)); }

void Context::set_head_dim(int d_logical) {
  if (d_logical < 1 || d_logical > d_) fail(-10, "head width must be in [1, d]");
  flush_pending();
  da_.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d_logical)));
  dl_ = d_logical;  // CostModel::entry_bytes counts the caller's width (store.hpp:27-30)
}

void Context::check_dev_err() {
  std::int32_t e = 0;
  KVC_CUDA(cudaMemcpyAsync(&e, t_.err, 4, cudaMemcpyDeviceToHost, st_));  // (st_ is non-blocking:
  sync();                                                                 //  not the legacy stream)
  check_err_word(e);
}

void Context::check_err_word(std::int32_t e) {
  if (!e) return;
  KVC_CUDA(cudaMemsetAsync(t_.err, 0, 4, st_));
  sync();
  if (e & DERR_DEGENERATE) fail(-2, "cosine of zero vector");
  if (e & DERR_PAGES) fail(-21, "page pool exhausted (raise kvc_cfg.pool_bytes)");
  if (e & DERR_CLUSTER_PAGES) fail(-21, "cluster exceeds max_cluster_pages / max_buffer_pages");
  if (e & DERR_CANDIDATES) fail(-21, "more candidates than max_candidates");
  if (e & DERR_ITEMS) fail(-21, "attention work list overflow");
  if (e & DERR_TIER) fail(-11, "host-tier page outside its cluster's extent");
  if (e & DERR_TAKE)
    fail(-21, "more than 64 ranked clusters per domain (min(k_s, candidates) and min(prefetch_k, candidates) must be <= 64)");
  fail(-1, "device error");
}

// ============================================================================ index (host)

Cluster& Context::C(std::int64_t id) {
  if (id < 0 || id >= static_cast<std::int64_t>(clusters_.size()) || !clusters_[static_cast<std::size_t>(id)])
    fail(-8, "unknown cluster id: " + std::to_string(id));
  return *clusters_[static_cast<std::size_t>(id)];
}

const Cluster* Context::cluster(std::int64_t id) const {
  if (id < 0 || id >= static_cast<std::int64_t>(clusters_.size())) return nullptr;
  return clusters_[static_cast<std::size_t>(id)].get();
}

std::vector<std::int64_t> Context::cluster_ids() const {
  std::vector<std::int64_t> out;
  out.reserve(static_cast<std::size_t>(n_live_));
  for (std::size_t i = 0; i < clusters_.size(); ++i)
    if (clusters_[i]) out.push_back(static_cast<std::int64_t>(i));
  return out;
}

std::int32_t Context::take_slot() {
  if (free_slots_.empty()) fail(-21, "cluster table full (raise kvc_cfg.max_slots)");
  std::int32_t s = free_slots_.back();
  free_slots_.pop_back();
  return s;
}

void Context::frame_add(std::int64_t frame, std::int64_t cid) {
  auto& v = frame_clusters_[frame];
  auto it = std::lower_bound(v.begin(), v.end(), cid);
  if (it == v.end() || *it != cid) v.insert(it, cid);
}

// The replay's frame -> cluster entries of one frame, merged in one sorted pass.
void Context::frame_add_flush(std::int64_t frame) {
  if (fc_pending_.empty()) return;
  std::sort(fc_pending_.begin(), fc_pending_.end());
  fc_pending_.erase(std::unique(fc_pending_.begin(), fc_pending_.end()), fc_pending_.end());
  auto& v = frame_clusters_[frame];
  if (v.empty()) {
    v.swap(fc_pending_);
  } else {
    std::vector<std::int64_t> m;
    m.reserve(v.size() + fc_pending_.size());
    std::set_union(v.begin(), v.end(), fc_pending_.begin(), fc_pending_.end(), std::back_inserter(m));
    v.swap(m);
  }
  fc_pending_.clear();
}

void Context::frame_del(std::int64_t frame, std::int64_t cid) {
  auto f = frame_clusters_.find(frame);
  if (f == frame_clusters_.end()) return;
  auto it = std::lower_bound(f->second.begin(), f->second.end(), cid);
  if (it != f->second.end() && *it == cid) f->second.erase(it);
  if (f->second.empty()) frame_clusters_.erase(f);
}

// HierIndex::add_cluster (index.cpp:97-120) for a cluster whose statistics the caller
// installs on the device. Returns the id; assigns a device slot.
std::int64_t Context::new_cluster(std::int32_t layer, std::int64_t parent,
                                  std::vector<Member>&& members, bool host) {
  if (members.empty()) fail(-5, "cluster with no members");
  return new_cluster_at(take_slot(), layer, parent, std::move(members), host);
}

std::int64_t Context::new_cluster_at(std::int32_t slot, std::int32_t layer, std::int64_t parent,
                                     std::vector<Member>&& members, bool host) {
  if (members.empty()) fail(-5, "cluster with no members");
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range: " + std::to_string(layer));
  auto c = std::make_unique<Cluster>();
  c->id = static_cast<std::int64_t>(clusters_.size());
  c->layer = layer;
  c->parent = parent;
  c->members = MemberList(members);
  c->stat_count = static_cast<std::int64_t>(c->members.size());
  c->first_frame = c->members.front().frame;
  c->last_touch = c->members.front().frame;
  for (const MemberList::Run& r : c->members.runs()) {
    c->first_frame = std::min(c->first_frame, r.frame);
    c->last_touch = std::max(c->last_touch, r.frame);
    frame_add(r.frame, c->id);
  }
  cflags_.push_back(host ? CF_HOST : 0);
  last_use_.push_back(0);
  if (!host) min_lt_ = std::min(min_lt_, c->last_touch);
  c->slot = slot;
  slot_id_[static_cast<std::size_t>(c->slot)] = c->id;
  resid_h_[static_cast<std::size_t>(c->slot)] = host ? 1 : 0;
  parts_[static_cast<std::size_t>(parent)].per_layer[static_cast<std::size_t>(layer)].push_back(c->id);
  layer_live_count_[static_cast<std::size_t>(layer)] += 1;
  n_live_ += 1;
  std::int64_t id = c->id;
  clusters_.push_back(std::move(c));
  return id;
}

// HierIndex::remove_cluster (index.cpp:122-145); device pages are released by the caller.
void Context::drop_cluster(std::int64_t id) {
  const std::int32_t s = C(id).slot;
  launches_ += launch_free_slot_pages(t_, s, st_);  // HBM pages only
  drop_cluster_host(id);
  free_slots_.push_back(s);
}

void Context::drop_cluster_host(std::int64_t id) {
  Cluster& c = C(id);
  auto& sib = parts_[static_cast<std::size_t>(c.parent)].per_layer[static_cast<std::size_t>(c.layer)];
  sib.erase(std::remove(sib.begin(), sib.end(), id), sib.end());
  for (const MemberList::Run& r : c.members.runs()) frame_del(r.frame, id);
  for (const MemberList::Run& r : c.buffer.runs()) frame_del(r.frame, id);
  layer_live_count_[static_cast<std::size_t>(c.layer)] -= 1;
  n_live_ -= 1;
  const std::int32_t s = c.slot;
  tier_forget(id);  // the host-tier extent
  slot_id_[static_cast<std::size_t>(s)] = -1;
  clusters_[static_cast<std::size_t>(id)].reset();
}

// Device copy of per_layer_clusters[layer] of a partition, as slots.
void Context::pl_upload(std::int64_t pid, int layer) {
  Partition& p = parts_[static_cast<std::size_t>(pid)];
  const auto& ids = p.per_layer[static_cast<std::size_t>(layer)];
  const std::int32_t n = static_cast<std::int32_t>(ids.size());
  pl_reserve(pid, layer, n);
  const std::int32_t off = p.dev_off[static_cast<std::size_t>(layer)];
  std::vector<std::int32_t> tmp(static_cast<std::size_t>(n));
  for (std::int32_t i = 0; i < n; ++i) tmp[static_cast<std::size_t>(i)] = C(ids[static_cast<std::size_t>(i)]).slot;
  // the stream is synchronised below, so pageable sources may be locals
  if (n > 0) KVC_CUDA(cudaMemcpyAsync(t_.pl_pool + off, tmp.data(), n * 4, cudaMemcpyHostToDevice, st_));
  const std::int64_t k = pid * L_ + layer;
  KVC_CUDA(cudaMemcpyAsync(t_.pl_off + k, &off, 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(t_.pl_cnt + k, &n, 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));
}

void Context::pl_reserve(std::int64_t pid, int layer, std::int32_t n) {
  Partition& p = parts_[static_cast<std::size_t>(pid)];
  std::int32_t& off = p.dev_off[static_cast<std::size_t>(layer)];
  std::int32_t& cap = p.dev_cap[static_cast<std::size_t>(layer)];
  if (n > cap) {
    std::int32_t ncap = std::max<std::int32_t>(16, std::max(n, cap * 2));
    if (pl_bump_ + ncap > t_.pl_pool_cap) {
      // compact: re-lay every list contiguously
      pl_bump_ = 0;
      for (std::size_t q = 0; q < parts_.size(); ++q)
        for (int l = 0; l < L_; ++l) {
          parts_[q].dev_cap[static_cast<std::size_t>(l)] = 0;
        }
      for (std::size_t q = 0; q < parts_.size(); ++q)
        for (int l = 0; l < L_; ++l) {
          const std::int32_t m = static_cast<std::int32_t>(parts_[q].per_layer[static_cast<std::size_t>(l)].size());
          std::int32_t c2 = (static_cast<std::int64_t>(q) == pid && l == layer) ? ncap : m;
          const std::size_t fk = q * static_cast<std::size_t>(L_) + static_cast<std::size_t>(l);
          if (fk < pl_floor_.size()) c2 = std::max(c2, pl_floor_[fk]);  // lists the wave engine holds
          if (pl_bump_ + c2 > t_.pl_pool_cap) fail(-21, "partition-list pool full");
          parts_[q].dev_off[static_cast<std::size_t>(l)] = static_cast<std::int32_t>(pl_bump_);
          parts_[q].dev_cap[static_cast<std::size_t>(l)] = c2;
          pl_bump_ += c2;
          if (!(static_cast<std::int64_t>(q) == pid && l == layer) && m > 0) pl_upload(static_cast<std::int64_t>(q), l);
        }
    } else {
      off = static_cast<std::int32_t>(pl_bump_);
      cap = ncap;
      pl_bump_ += ncap;
    }
  }
}

// Partition representative -> device without a host sync: the values go through a pinned ring
// (the stream is synchronised at least once per ingested frame, long before a slot is reused).
void Context::upload_partition(std::int64_t pid) {
  const Partition& p = parts_[static_cast<std::size_t>(pid)];
  constexpr int kRing = 64;
  if (!h_part_ring_) h_part_ring_ = static_cast<double*>(halloc(static_cast<std::size_t>(kRing) * (d_ + 2) * 8));
  double* slot = h_part_ring_ + static_cast<std::size_t>(part_ring_pos_++ % kRing) * (d_ + 2);
  std::memcpy(slot, p.vrep.data(), d_ * 8);
  slot[d_] = norm_d(p.vrep.data(), d_);
  std::int32_t np = static_cast<std::int32_t>(parts_.size());
  std::memcpy(&slot[d_ + 1], &np, 4);
  KVC_CUDA(cudaMemcpyAsync(t_.vrep + pid * d_, slot, d_ * 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(t_.vnorm + pid, &slot[d_], 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(t_.n_parts, &slot[d_ + 1], 4, cudaMemcpyHostToDevice, st_));
}

void Context::flush_resid() {
  if (!resid_dirty_) return;
  KVC_CUDA(cudaMemcpyAsync(t_.resid, resid_h_.data(), resid_h_.size(), cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));
  resid_dirty_ = false;
}

// ============================================================================ store (host)

std::int64_t Context::entry_bytes() const {  // CostModel::entry_bytes (store.hpp:27-30)
  return cfg_.bytes_per_entry > 0 ? cfg_.bytes_per_entry
                                  : static_cast<std::int64_t>(dl_) * 2 * static_cast<std::int64_t>(sizeof(float));
}

std::int64_t Context::side_entries(const Cluster& c) const {  // store.cpp:76-80
  const std::int64_t buffered = static_cast<std::int64_t>(c.buffer.size());
  if (!is_host(c.id)) return static_cast<std::int64_t>(c.members.size()) + buffered;
  return c.device_tail + buffered;
}

void Context::adopt(std::int64_t id) {  // store.cpp:82-86
  Cluster& c = C(id);
  device_entries_ += side_entries(c);
  std::int64_t tk = tick_++;
  if (!flag(id, CF_TRACKED)) {
    set_flag(id, CF_TRACKED, true);
    last_use_[static_cast<std::size_t>(id)] = tk;
  }
}

void Context::forget(std::int64_t id) {  // store.cpp:88-93
  Cluster& c = C(id);
  device_entries_ -= side_entries(c);
  set_flag(id, CF_TRACKED, false);
  if (flag(id, CF_PINNED)) {
    set_flag(id, CF_PINNED, false);
    pinned_ids_.erase(std::remove(pinned_ids_.begin(), pinned_ids_.end(), id), pinned_ids_.end());
  }
}

void Context::touch(std::int64_t id) {  // store.cpp:139-141
  set_flag(id, CF_TRACKED, true);
  last_use_[static_cast<std::size_t>(id)] = tick_++;
}

void Context::record(int cause, bool to_dev, std::int64_t id, std::int64_t bytes) {
  LedgerOp op{cause, to_dev, id, 1, bytes,
              1.0 * cfg_.alpha_us + static_cast<double>(bytes) * cfg_.beta_us_per_byte};
  ledger_.push_back(op);
}

double Context::fetch(std::int64_t id, int cause) {  // store.cpp:95-113
  if (id < 0 || id >= static_cast<std::int64_t>(clusters_.size()) || !clusters_[static_cast<std::size_t>(id)])
    fail(-8, "unknown cluster id: " + std::to_string(id));
  touch(id);
  if (!is_host(id)) return 0.0;  // resident: only the LRU tick moves (no object access)
  Cluster& c = C(id);
  const std::int64_t moved = static_cast<std::int64_t>(c.members.size()) - c.device_tail;
  if (moved < 0) fail(-11, "device tail exceeds member count");
  double paid = 0.0;
  if (moved > 0) {
    const std::int64_t bytes = moved * entry_bytes();
    record(cause, true, id, bytes);
    paid = ledger_.back().cost_us;
    device_entries_ += moved;
  }
  set_flag(id, CF_HOST, false);
  tier_note(id, false);  // physical: the host extent comes back to HBM (context_tiers.cpp)
  c.device_tail = 0;
  min_lt_ = std::min(min_lt_, c.last_touch);
  resid_h_[static_cast<std::size_t>(c.slot)] = 0;
  resid_dirty_ = true;
  paid += enforce_capacity();
  return paid;
}

double Context::offload(std::int64_t id) {  // store.cpp:115-130
  Cluster& c = C(id);
  const std::int64_t moved = !is_host(id) ? static_cast<std::int64_t>(c.members.size()) : c.device_tail;
  double paid = 0.0;
  if (moved > 0) {
    const std::int64_t bytes = moved * entry_bytes();
    record(KVC_CAUSE_OFFLOAD, false, id, bytes);
    paid = ledger_.back().cost_us;
    device_entries_ -= moved;
  }
  set_flag(id, CF_HOST, true);
  tier_note(id, true);  // physical: member pages move to the host tier (context_tiers.cpp)
  c.device_tail = 0;
  resid_h_[static_cast<std::size_t>(c.slot)] = 1;
  resid_dirty_ = true;
  return paid;
}

double Context::enforce_capacity() {  // store.cpp:156-164
  double paid = 0.0;
  while (device_entries_ > cfg_.device_capacity_entries) {
    const double cost = evict_one();
    if (cost < 0.0) break;
    paid += cost;
  }
  return paid;
}

double Context::evict_one() {  // store.cpp:166-181
  std::int64_t victim = -1, vt = 0;
  for (const auto& up : clusters_) {
    if (!up) continue;
    const std::uint8_t f = cflags_[static_cast<std::size_t>(up->id)];
    if (!(f & CF_TRACKED) || (f & CF_PINNED)) continue;
    if (side_entries(*up) == 0) continue;
    if (!up->buffer.empty()) continue;
    const std::int64_t lu = last_use_[static_cast<std::size_t>(up->id)];
    if (victim < 0 || lu < vt) {
      victim = up->id;
      vt = lu;
    }
  }
  if (victim < 0) return -1.0;
  return offload(victim);
}

// ============================================================================ engine (host)

void Context::push_window(std::int64_t frame_id, int T, int slot) {  // engine.cpp:54-57
  window_.push_back({frame_id, slot, T});
  while (static_cast<int>(window_.size()) > t_.W) window_.pop_front();
}

std::vector<std::int64_t> Context::window_owner_ids() const {
  std::vector<std::int64_t> out;
  for (const WinFrame& w : window_) {
    auto it = frame_clusters_.find(w.frame_id);
    if (it != frame_clusters_.end()) out.insert(out.end(), it->second.begin(), it->second.end());
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

void Context::repin() {  // engine.cpp:67-75 + TieredStore::pin (store.cpp:143-145)
  for (std::int64_t id : pinned_ids_)
    if (clusters_[static_cast<std::size_t>(id)]) set_flag(id, CF_PINNED, false);
  pinned_ids_ = window_owner_ids();
  for (std::int64_t id : pinned_ids_) set_flag(id, CF_PINNED, true);
}

void Context::apply_cadence(std::int64_t frame_id, std::int64_t pid) {  // engine.cpp:95-132
  if (last_partition_ >= 0 && pid >= 0 && pid != last_partition_) {
    const Partition& closed = parts_[static_cast<std::size_t>(last_partition_)];
    std::vector<std::int64_t> ids;
    for (const auto& list : closed.per_layer) ids.insert(ids.end(), list.begin(), list.end());
    for (std::int64_t cid : ids) {
      const Cluster& c = C(cid);
      if (!is_host(cid) && !is_lazy(cid)) {
        const auto owners = window_owner_ids();
        if (!std::binary_search(owners.begin(), owners.end(), cid)) offload(cid);
      }
    }
  }
  if (pid >= 0) last_partition_ = pid;
  // no Device, non-lazy cluster can be stale while the lower bound on their last_touch is recent
  if (min_lt_ == INT64_MAX || min_lt_ + cfg_.offload_horizon_frames >= frame_id) {
    enforce_capacity();
    return;
  }
  std::vector<std::int64_t> stale;
  std::int64_t lo = INT64_MAX;
  for (const auto& up : clusters_)
    if (up && !(cflags_[static_cast<std::size_t>(up->id)] & (CF_HOST | CF_LAZY))) lo = std::min(lo, up->last_touch);
  min_lt_ = lo;
  for (const auto& up : clusters_)
    if (up && !(cflags_[static_cast<std::size_t>(up->id)] & (CF_HOST | CF_LAZY)) &&
        up->last_touch + cfg_.offload_horizon_frames < frame_id)
      stale.push_back(up->id);
  if (!stale.empty()) {
    const auto owners = window_owner_ids();
    for (std::int64_t cid : stale)
      if (!std::binary_search(owners.begin(), owners.end(), cid)) offload(cid);
  }
  enforce_capacity();
}

std::int64_t Context::place_frame(std::int64_t frame_id, const float* visual) {
  // maintainer.cpp:37-53
  std::int64_t best = -1;
  double best_sim = -2.0;
  for (std::size_t p = 0; p < parts_.size(); ++p) {
    const double sim = cosine_fd(visual, parts_[p].vrep.data(), d_);
    if (sim > best_sim) {
      best_sim = sim;
      best = static_cast<std::int64_t>(p);
    }
  }
  if (best >= 0 && best_sim >= cfg_.visual_floor) {  // HierIndex::append_frame (index.cpp:71-79)
    Partition& p = parts_[static_cast<std::size_t>(best)];
    p.frames.push_back(frame_id);
    const double n = static_cast<double>(p.stat);
    for (int i = 0; i < d_; ++i) p.vrep[static_cast<std::size_t>(i)] = (n * p.vrep[static_cast<std::size_t>(i)] + visual[i]) / (n + 1.0);
    p.stat += 1;
    upload_partition(best);
    return best;
  }
  mstats_[8] += 1;  // partitions_opened
  if (static_cast<std::int32_t>(parts_.size()) >= t_.max_parts) fail(-21, "too many partitions (raise max_partitions)");
  Partition p;  // HierIndex::add_partition (index.cpp:59-69)
  p.frames.push_back(frame_id);
  p.vrep.assign(visual, visual + d_);
  p.stat = 1;
  p.per_layer.resize(static_cast<std::size_t>(L_));
  p.dev_off.assign(static_cast<std::size_t>(L_), 0);
  p.dev_cap.assign(static_cast<std::size_t>(L_), 0);
  parts_.push_back(std::move(p));
  const std::int64_t pid = static_cast<std::int64_t>(parts_.size()) - 1;
  upload_partition(pid);
  // empty device lists
  std::vector<std::int32_t> z(static_cast<std::size_t>(L_), 0);
  KVC_CUDA(cudaMemcpyAsync(t_.pl_cnt + pid * L_, z.data(), L_ * 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaStreamSynchronize(st_));
  return pid;
}

void Context::select_frame_buffer(int b) {
  d_fk_ = fkbuf_[b];
  d_fv_ = fvbuf_[b];
  ia_.fk = d_fk_;
  ia_.fv = d_fv_;
  std::memcpy(key_map_, key_maps_[b], sizeof(key_map_));
  h_evk_ = h_out_[b];
  h_evs_ = h_evk_ + static_cast<std::size_t>(L_) * t_.tmax;
  h_stop_ = h_evs_ + static_cast<std::size_t>(L_) * t_.tmax;
  h_err_ = h_out_[b] + 2 * static_cast<std::size_t>(L_) * t_.tmax + 3 * static_cast<std::size_t>(L_);
}

// Replay (+ host events) of the pending frame, then window / repin / cadence (engine.cpp:168-173).
void Context::finish_frame(std::int64_t* assigned) {
  PendingIngest p = ping_;
  ping_.active = false;
  ping_wait_ = p.ev;
  select_frame_buffer(p.buf);
  ia_.T = p.T;
  ia_.pid = static_cast<std::int32_t>(p.pid);
  ia_.ring_slot = p.ring_slot;
  ia_.my_events = d_evflags_ + p.buf;
  ia_.prev_events = nullptr;
  const std::int64_t l0 = launches_;
  run_inserts(p.frame_id, p.pid, p.T, assigned, true);
  // re-launches (host events) read the frame buffer again; they happen before any later frame is
  // launched, so the buffer's release event can be moved after them
  if (launches_ != l0) KVC_CUDA(cudaEventRecord(ev_buf_[p.buf], st_));
  push_window(p.frame_id, p.T, p.ring_slot);
  repin();
  apply_cadence(p.frame_id, p.pid);
  tier_kick();
}

// Replays the frame held in pong_ (its kernels are complete and it had no host events).
void Context::finish_pong() {
  if (!pong_.active) return;
  const PendingIngest keep = ping_;
  ping_ = pong_;
  pong_.active = false;
  finish_frame(nullptr);
  ping_ = keep;
}

void Context::flush_ingest() {
  finish_pong();
  if (!ping_.active) return;
  KVC_CUDA(cudaEventSynchronize(ping_.ev));
  finish_frame(nullptr);
}

void Context::ingest_frame(std::int64_t frame_id, const float* visual, const void* keys,
                           const void* values, int T, int mem, std::int64_t* assigned,
                           std::int64_t* partition) {
  if (T < 1 || T > t_.tmax) fail(-10, "tokens per frame outside [1, max_tokens]");
  tier_kick();
  if (!visual || !keys || !values) fail(-10, "null frame buffer");
  if (assigned) std::fill(assigned, assigned + static_cast<std::int64_t>(L_) * T, -1);
  if (partition) *partition = -1;
  // Pipelined ingest (no per-entry outputs requested): this frame is launched before the previous
  // frame's host replay, which then overlaps this frame's kernels. A previous frame that needs
  // host events (seeds / splits change the device index) is completed first.
  static const bool force_sync = std::getenv("KVC_INGEST_SYNC") != nullptr;
  const bool async_ok = !assigned && !cfg_.parity_mode && !cfg_.check_invariants && built_ && cfg_.defer_host_splits &&
                        !timing_ && !force_sync;
  const int b = ping_.active ? (ping_.buf ^ 1) : (ibuf_ ^ 1);
  ibuf_ = b;
  // The payload crosses on the input stream first, overlapping the pending frame's kernels
  // (buffer b's last reader, two frames back, is complete: ordered by ev_buf_[b]).
  {
    const std::size_t row = static_cast<std::size_t>(T) * d_ * es_;
    const std::size_t pitch = static_cast<std::size_t>(t_.tmax) * d_ * es_;
    const cudaMemcpyKind kind = mem == KVC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    KVC_CUDA(cudaStreamWaitEvent(in_st_, ev_buf_[b], 0));
    if (pitch == row) {  // frames of max_tokens tokens: one linear copy each
      KVC_CUDA(cudaMemcpyAsync(fkbuf_[b], keys, row * L_, kind, in_st_));
      KVC_CUDA(cudaMemcpyAsync(fvbuf_[b], values, row * L_, kind, in_st_));
    } else {
      KVC_CUDA(cudaMemcpy2DAsync(fkbuf_[b], pitch, keys, row, row, L_, kind, in_st_));
      KVC_CUDA(cudaMemcpy2DAsync(fvbuf_[b], pitch, values, row, row, L_, kind, in_st_));
    }
    KVC_CUDA(cudaEventRecord(ev_in_[b], in_st_));
  }
  // the frame before the previous one is replayed now, after this frame's payload copy was queued
  // (so the copies run back to back while the host replays)
  finish_pong();
  // Speculation: this frame's first round is queued behind the pending frame's before that
  // frame's outcome is known (no device idle while the host waits and launches). It commits
  // nothing if the pending frame stopped for host events; this frame is then launched again.
  const bool spec = ping_.active && async_ok && spec_ingest_;
  if (ping_.active && !spec) {
    KVC_CUDA(cudaEventSynchronize(ping_.ev));
    bool events = false;
    const std::int32_t* stp = h_out_[ping_.buf] + 2 * static_cast<std::size_t>(L_) * t_.tmax;
    for (int l = 0; l < L_ && !events; ++l) events = stp[l] < ping_.T;
    if (!async_ok || events || stp[3 * L_]) finish_frame(nullptr);
  }
  select_frame_buffer(b);
  KVC_CUDA(cudaStreamWaitEvent(st_, ev_in_[b], 0));
  const int ring_slot = static_cast<int>(frames_seen_ % t_.W);
  launches_ += launch_ring_write(t_, d_fk_, d_fv_, T, ring_slot, st_);
  for (int l = 0; l < L_; ++l)
    std::fill_n(&ring_owner_h_[(static_cast<std::size_t>(l) * t_.W + ring_slot) * t_.tmax], t_.tmax, -1);
  ring_frame_[static_cast<std::size_t>(ring_slot)] = RingFrame{frame_id, T};

  if (!built_) {  // engine.cpp:161-166
    launches_ += launch_ring_rows(t_, d_fk_, d_fv_, T, ring_slot, st_);
    PendingFrame pf;
    pf.frame_id = frame_id;
    pf.visual.assign(visual, visual + d_);
    pf.T = T;
    const std::size_t n = static_cast<std::size_t>(L_) * T * d_;
    pf.keys_raw.resize(n * es_);
    pf.vals_raw.resize(n * es_);
    if (mem == KVC_MEM_DEVICE) {
      KVC_CUDA(cudaMemcpyAsync(pf.keys_raw.data(), keys, n * es_, cudaMemcpyDeviceToHost, st_));
      KVC_CUDA(cudaMemcpyAsync(pf.vals_raw.data(), values, n * es_, cudaMemcpyDeviceToHost, st_));
      sync();
    } else {
      std::memcpy(pf.keys_raw.data(), keys, n * es_);
      std::memcpy(pf.vals_raw.data(), values, n * es_);
    }
    pf.keys_f32.resize(n);
    rows_to_f32(pf.keys_raw.data(), es_ == 2, n, pf.keys_f32.data());
    pending_.push_back(std::move(pf));
    KVC_CUDA(cudaEventRecord(ev_buf_[b], st_));
    push_window(frame_id, T, ring_slot);
    frames_seen_ += 1;
    if (static_cast<int>(pending_.size()) >= cfg_.build_batch_frames) build_now();
    return;
  }

  const std::int64_t pid = place_frame(frame_id, visual);
  if (partition) *partition = pid;
  frames_seen_ += 1;
  if (!async_ok) {
    ia_.T = T;
    ia_.pid = static_cast<std::int32_t>(pid);
    ia_.ring_slot = ring_slot;
    run_inserts(frame_id, pid, T, assigned, false);
    KVC_CUDA(cudaEventRecord(ev_buf_[b], st_));
    push_window(frame_id, T, ring_slot);
    repin();
    apply_cadence(frame_id, pid);
    tier_kick();
    return;
  }
  // launch this frame (all domains from token 0), its outcome block copied back on the stream
  ia_.T = T;
  ia_.pid = static_cast<std::int32_t>(pid);
  ia_.ring_slot = ring_slot;
  std::vector<int> all_doms(static_cast<std::size_t>(L_)), zero_cursor(static_cast<std::size_t>(L_), 0);
  std::iota(all_doms.begin(), all_doms.end(), 0);
  ia_.my_events = d_evflags_ + b;
  ia_.prev_events = spec ? d_evflags_ + ping_.buf : nullptr;
  launch_round(all_doms, zero_cursor);
  ia_.prev_events = nullptr;
  KVC_CUDA(cudaEventRecord(ev_buf_[b], st_));  // the frame buffer's readers are all launched
  PendingIngest next;
  next.active = true;
  next.frame_id = frame_id;
  next.pid = pid;
  next.T = T;
  next.ring_slot = ring_slot;
  next.buf = b;
  next.ev = ev_ing_[b];
  KVC_CUDA(cudaEventRecord(next.ev, st_));
  if (spec) {  // now the pending frame's outcome
    KVC_CUDA(cudaEventSynchronize(ping_.ev));
    bool events = false;
    const std::int32_t* stp = h_out_[ping_.buf] + 2 * static_cast<std::size_t>(L_) * t_.tmax;
    for (int l = 0; l < L_ && !events; ++l) events = stp[l] < ping_.T;
    if (events || stp[3 * L_]) {
      // host events: settle the pending frame (its relaunches queue behind the skipped round),
      // then launch this frame again on the settled index
      finish_frame(nullptr);
      select_frame_buffer(b);
      ia_.T = T;
      ia_.pid = static_cast<std::int32_t>(pid);
      ia_.ring_slot = ring_slot;
      ia_.my_events = d_evflags_ + b;
      launch_round(all_doms, zero_cursor);
      KVC_CUDA(cudaEventRecord(ev_buf_[b], st_));
      KVC_CUDA(cudaEventRecord(next.ev, st_));
      ping_ = next;
      return;
    }
  }
  // the previous frame (no host events, kernels complete) is replayed at the start of the next
  // call (or by any reader of host state: flush_ingest), overlapping this frame's kernels
  if (ping_.active) pong_ = ping_;
  ping_ = next;
}

// Runs on_insert for every (layer, token) of the frame in layer-major order
// (engine.cpp:169-170). The GPU resolves every domain in parallel until a host event; the
// host replays the outcomes in reference order and settles host events domain by domain so
// ids, split seeds and LRU ticks are assigned exactly as the sequential reference does.
// One resolve round for `active` domains from their cursors: candidates, distance tile, resolve,
// row store, and the outcome block / error word copied back (not waited for).
void Context::launch_round(const std::vector<int>& active, const std::vector<int>& cursor) {
  flush_resid();
  ia_.n_active = static_cast<std::int32_t>(active.size());
  bool first = static_cast<int>(active.size()) == L_;
  for (int l = 0; l < L_ && first; ++l) first = active[static_cast<std::size_t>(l)] == l && cursor[static_cast<std::size_t>(l)] == 0;
  if (first) {  // a frame's first round: the constant arrays
    ia_.active = d_all_active_;
    ia_.cursor = d_all_active_ + L_;
  } else {
    ia_.active = d_active_;
    ia_.cursor = d_cursor_;
  }
  // rotating pinned staging: a round may be queued behind another whose copy has not run yet
  // (speculative next frame), so consecutive rounds never share a staging slot
  const int slot = act_next_;
  act_next_ = (act_next_ + 1) % kActSlots;
  if (ev_act_[slot]) KVC_CUDA(cudaEventSynchronize(ev_act_[slot]));
  std::int32_t* ha = h_active_ + static_cast<std::size_t>(slot) * 2 * L_;
  for (std::size_t i = 0; i < active.size(); ++i) ha[i] = active[i];
  for (int l = 0; l < L_; ++l) ha[L_ + l] = cursor[static_cast<std::size_t>(l)];
  if (!first) {
    KVC_CUDA(cudaMemcpyAsync(d_active_, ha, L_ * 8, cudaMemcpyHostToDevice, st_));
    if (!ev_act_[slot]) KVC_CUDA(cudaEventCreateWithFlags(&ev_act_[slot], cudaEventDisableTiming));
    KVC_CUDA(cudaEventRecord(ev_act_[slot], st_));
  }
  round_timed_ = timing_;
  static const bool exact_all_env = [] {  // KVC_EXACT_ALL=1: every round as a relaunch round (profiling)
    const char* e = std::getenv("KVC_EXACT_ALL");
    return e && e[0] == '1';
  }();
  ia_.exact_all = round_after_event_ || exact_all_env ? 1 : 0;
  static const bool resolve_prof = [] {  // KVC_RESOLVE_PROF=1: the sequential resolve's phase clocks
    const char* e = std::getenv("KVC_RESOLVE_PROF");
    return e && e[0] == '1';
  }();
  ia_.prof_on = resolve_prof ? 1 : 0;
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[0], st_));
  launches_ += launch_build_cands(t_, ia_, st_);
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[1], st_));
  if (assign_tc_) {
    ia_.margin = kTcMargin;
    launches_ += launch_assign_tc(t_, ia_, key_map_, st_);
    if (timing_) KVC_CUDA(cudaEventRecord(ev_[2], st_));
  } else {
    ia_.margin = kSimtMargin;
    launches_ += launch_approx(t_, ia_, st_);
    if (timing_) KVC_CUDA(cudaEventRecord(ev_[2], st_));
    launches_ += launch_topm(t_, ia_, st_);
  }
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[3], st_));
  {
    const bool seq = resolve_seq_ || (round_after_event_ && relaunch_seq_);
    const int n = seq ? 0 : launch_resolve_spec(t_, ia_, st_);
    launches_ += n ? n : launch_resolve(t_, ia_, st_);
  }
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[4], st_));
  launches_ += launch_store_rows(t_, ia_, st_);
  KVC_CUDA(cudaGetLastError());
  if (timing_) KVC_CUDA(cudaEventRecord(ev_[5], st_));
  // outcome block + the error word K3 copied after it, in one copy
  KVC_CUDA(cudaMemcpyAsync(h_evk_, ia_.ev_kind, (static_cast<std::size_t>(L_) * t_.tmax * 2 + static_cast<std::size_t>(L_) * 4 + 1) * 4,
                           cudaMemcpyDeviceToHost, st_));
}

// launched: the first round (all domains from token 0) is already in flight with its outcome
// block in h_evk_ (pipelined ingest); otherwise it is launched here.
namespace {
// First index in [u, stop) whose (slot, kind) differs from the run's: blocks of 8 compared without
// branches (vectorised), then the differing block scanned.
inline int run_end(const std::int32_t* evs, const std::int32_t* evk, int u, int stop, std::int32_t slot,
                   std::int32_t kind) {
  while (u + 8 <= stop) {
    int diff = 0;
    for (int j = 0; j < 8; ++j) diff |= (evs[u + j] != slot) | (evk[u + j] != kind);
    if (diff) break;
    u += 8;
  }
  while (u < stop && evs[u] == slot && evk[u] == kind) ++u;
  return u;
}
}  // namespace

void Context::run_inserts(std::int64_t frame_id, std::int64_t pid, int T, std::int64_t* assigned, bool launched,
                          int l_lo, int l_hi, int tok0) {
  const int ring_slot = ia_.ring_slot;
  const bool eager = !cfg_.defer_host_splits;
  if (l_hi < 0) l_hi = L_;
  if (waves_ && !eager && l_lo == 0 && l_hi == L_ && tok0 == 0) {
    run_inserts_waves(frame_id, pid, T, assigned, launched);
    return;
  }
  if (spec_.active) {  // a speculation of an earlier frame is never consumed
    KVC_CUDA(cudaEventSynchronize(spec_.ev));
    spec_.active = false;
  }
  std::vector<int> cursor(static_cast<std::size_t>(L_), 0), replayed(static_cast<std::size_t>(L_), 0);
  for (int l = l_lo; l < l_hi; ++l) cursor[static_cast<std::size_t>(l)] = replayed[static_cast<std::size_t>(l)] = tok0;
  std::vector<int> active;
  if (eager)
    active.push_back(l_lo);
  else
    for (int l = l_lo; l < l_hi; ++l) active.push_back(l);
  int frontier = l_lo;
  bool launch = true;
  bool relaunch_after_event = false;
  ia_.T = T;
  ia_.pid = static_cast<std::int32_t>(pid);
  ia_.ring_slot = ring_slot;
  double t_wait = 0.0, t_replay = 0.0, t_launch = 0.0;
  for (double& x : ingest_t_) x = 0.0;
  const auto r0 = std::chrono::steady_clock::now();
  while (frontier < l_hi) {
    if (launch) {
      const auto lc0 = std::chrono::steady_clock::now();
      cudaEvent_t done = nullptr;
      if (launched) {
        launched = false;  // the first round was launched by ingest_frame: wait for its outcome
        done = ping_wait_;  // block only (the next frame's kernels may already be queued behind it)
      } else {
        round_after_event_ = relaunch_after_event;
        launch_round(active, cursor);
        round_after_event_ = false;
      }
      const auto w0 = std::chrono::steady_clock::now();
      t_launch += std::chrono::duration<double, std::micro>(w0 - lc0).count();
      if (done)
        KVC_CUDA(cudaEventSynchronize(done));
      else
        sync();
      t_wait += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w0).count();
      if (relaunch_after_event) evt_t_[5] += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - lc0).count();
      relaunch_after_event = false;
      check_err_word(*h_err_);
      if (round_timed_) {  // (the round may have been launched before timing was switched on)
        float ms = 0.f;
        for (int i = 0; i < 5; ++i) {
          KVC_CUDA(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]));
          ingest_t_[i] += ms * 1e3;
        }
      }
      launch = false;
      // the replay below is bound by cache misses on scattered per-cluster state: touch every
      // pending domain's first cluster now, with the loads independent of each other
      for (int pass = 0; pass < 2; ++pass)
        for (int l = frontier; l < l_hi; ++l) {
          const int t0 = replayed[static_cast<std::size_t>(l)];
          if (t0 >= h_stop_[l]) continue;
          const std::int32_t sl = h_evs_[static_cast<std::size_t>(l) * t_.tmax + t0];
          if (sl < 0 || static_cast<std::size_t>(sl) >= slot_id_.size()) continue;
          const std::int64_t cid = slot_id_[static_cast<std::size_t>(sl)];
          if (cid < 0 || static_cast<std::size_t>(cid) >= clusters_.size() || !clusters_[static_cast<std::size_t>(cid)]) continue;
          const Cluster* cp = clusters_[static_cast<std::size_t>(cid)].get();
          if (pass == 0) {
            __builtin_prefetch(cp);
            __builtin_prefetch(&last_use_[static_cast<std::size_t>(cid)], 1);
            __builtin_prefetch(&cflags_[static_cast<std::size_t>(cid)], 1);
          } else if (!cp->members.runs().empty()) {
            __builtin_prefetch(&cp->members.runs().back(), 1);
          }
        }
    }
    const int l = frontier;
    const int stop = h_stop_[l];
    const std::int32_t* evk = h_evk_ + static_cast<std::size_t>(l) * t_.tmax;
    const std::int32_t* evs = h_evs_ + static_cast<std::size_t>(l) * t_.tmax;
    std::int32_t* owner = ring_slot >= 0 ? &ring_owner_h_[(static_cast<std::size_t>(l) * t_.W + ring_slot) * t_.tmax] : nullptr;
    std::int64_t last_cid = -1;
    const auto rp0 = std::chrono::steady_clock::now();
    // replay in runs of equal (cluster, outcome): ticks are consecutive within a run, so the run
    // moves the LRU tick once (store.cpp:139-141) and appends its members in one go
    for (int t = replayed[static_cast<std::size_t>(l)]; t < stop;) {
      const std::int32_t slot = evs[t];
      const std::int32_t kind = evk[t];
      int u = t + 1;
      if (kind != EV_DEFER) u = run_end(evs, evk, u, stop, slot, kind);
      const int n = u - t;
      const std::int64_t cid = slot_id_[static_cast<std::size_t>(slot)];
      Cluster& c = *clusters_[static_cast<std::size_t>(cid)];
      mstats_[0] += n;  // inserts
      c.stat_count += n;
      c.last_touch = std::max(c.last_touch, frame_id);
      if (cid != last_cid) {
        fc_pending_.push_back(cid);  // frame -> cluster map entries, merged once (frame_add_flush)
        last_cid = cid;
      }
      if (owner) std::fill(owner + t, owner + u, slot);
      (kind == EV_ABSORB ? c.members : c.buffer).push_run(frame_id, t, n);
      device_entries_ += n;
      set_flag(cid, CF_TRACKED, true);
      tick_ += n;
      last_use_[static_cast<std::size_t>(cid)] = tick_ - 1;
      switch (kind) {
        case EV_ABSORB:  // add_member + note_device_append (index.cpp:170-175, store.cpp:132-137)
          if (is_host(cid)) c.device_tail += n;
          mstats_[1] += n;
          break;
        case EV_BUFJOIN:  // add_to_buffer + note_device_buffer_append
          mstats_[3] += n;
          break;
        case EV_DEFER:  // lazy mark + buffer + register (maintainer.cpp:170-175)
          mstats_[6] += n;
          set_flag(cid, CF_LAZY, true);
          mstats_[3] += n;
          break;
        default:
          fail(-11, "unexpected device event kind");
      }
      if (assigned) std::fill(assigned + static_cast<std::size_t>(l) * T + t, assigned + static_cast<std::size_t>(l) * T + u, cid);
      t = u;
    }
    t_replay += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - rp0).count();
    replayed[static_cast<std::size_t>(l)] = stop;
    if (stop >= T) {
      frontier += 1;
      if (eager && frontier < l_hi) {
        active.assign(1, frontier);
        launch = true;
      }
      continue;
    }
    frame_add_flush(frame_id);  // host events add / remove map entries themselves
    if (h_stop_[L_ + l] == EV_SPLIT && is_host(slot_id_[static_cast<std::size_t>(h_stop_[2 * L_ + l])])) {
      // Pipelined ingest launched this frame before the previous frame's cadence offloaded the
      // cluster (residence only turns Device -> Host between frames): the device decided with the
      // old residence. Nothing of this token was committed; resolve the domain again from it.
      cursor[static_cast<std::size_t>(l)] = stop;
      active.assign(1, l);
      launch = true;
      continue;
    }
    const std::int64_t id = handle_host_event(frame_id, pid, l, stop, h_stop_[L_ + l], h_stop_[2 * L_ + l]);
    ingest_t_[9] += 1.0;  // host events this frame
    // the next domain's pending split, 2-means'd on the side while this domain is relaunched
    if (spec_split_ && l + 1 < l_hi && split_dev_min_ > 0) spec_split_launch(l + 1, T);
    if (assigned) assigned[static_cast<std::size_t>(l) * T + stop] = id;
    cursor[static_cast<std::size_t>(l)] = stop + 1;
    replayed[static_cast<std::size_t>(l)] = stop + 1;
    if (stop + 1 < T) {
      active.assign(1, l);
      launch = true;
      relaunch_after_event = true;
    } else {
      frontier += 1;
      if (eager && frontier < l_hi) {
        active.assign(1, frontier);
        launch = true;
      }
    }
  }
  frame_add_flush(frame_id);
  ingest_t_[5] = t_wait;
  ingest_t_[6] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - r0).count() - t_wait;
  ingest_t_[7] = t_replay;  // (part of [6]) the outcome replay loop
  ingest_t_[8] = t_launch;  // (part of [6]) relaunch issue
}

// ============================================================================ slow path

std::int64_t Context::stage_cluster(std::int32_t slot, bool with_buffer) {
  const Cluster& c = C(slot_id_[static_cast<std::size_t>(slot)]);
  const std::int64_t rows = static_cast<std::int64_t>(c.members.size()) + (with_buffer ? static_cast<std::int64_t>(c.buffer.size()) : 0);
  ensure_stage(rows + 1);
  launches_ += launch_gather_cluster(t_, slot, with_buffer ? 1 : 0, d_stage_k_, d_stage_v_, 0, st_);
  return rows;
}

void Context::stage_download(std::int64_t rows) {
  launches_ += launch_to_f32(t_, d_stage_k_, d_stage_f32_, rows * d_, st_);
  KVC_CUDA(cudaMemcpyAsync(h_stage_f32_, d_stage_f32_, static_cast<std::size_t>(rows) * d_ * 4, cudaMemcpyDeviceToHost, st_));
  sync();
}

void Context::init_slots(const std::vector<std::int32_t>& slots,
                         const std::vector<std::vector<double>>& reps,
                         const std::vector<double>& vars, const std::vector<std::int64_t>& stats,
                         const std::vector<std::int64_t>& nmem, const std::vector<std::int64_t>& cids,
                         const std::vector<std::uint8_t>& resid, const std::vector<std::int32_t>* nbuf,
                         const std::vector<std::vector<double>>* breps) {
  // Host-computed exact statistics -> device tables: one packed record per slot in pinned
  // staging, one copy, one scatter kernel; then the fp32 mirrors are refreshed on device.
  const std::size_t n = slots.size();
  if (n == 0) return;
  const std::size_t rb = slot_init_bytes(d_), bytes = n * rb + n * 4;  // records | slot list
  if (static_cast<std::int64_t>(bytes) > init_cap_) {
    if (h_init_) KVC_CUDA(cudaStreamSynchronize(st_));
    init_cap_ = static_cast<std::int64_t>(std::max(bytes, static_cast<std::size_t>(init_cap_) * 2));
    h_init_ = halloc(static_cast<std::size_t>(init_cap_));
    d_init_ = dalloc(static_cast<std::size_t>(init_cap_));
  } else {
    KVC_CUDA(cudaEventSynchronize(ev_init_));  // the previous batch's copy has left the staging
  }
  auto* h = static_cast<std::uint8_t*>(h_init_);
  for (std::size_t i = 0; i < n; ++i) {
    auto* r = h + i * rb;
    SlotInit x{};
    x.slot = slots[i];
    x.nb = nbuf ? (*nbuf)[i] : 0;
    x.stat = stats[i];
    x.nmem = nmem[i];
    x.cid = cids[i];
    x.resid = resid[i];
    x.lazy = x.nb > 0 ? 1 : 0;
    x.has_brep = (breps && x.nb > 0) ? 1 : 0;
    x.rnorm = norm_d(reps[i].data(), d_);
    x.var = vars[i];
    x.bnorm = x.has_brep ? norm_d((*breps)[i].data(), d_) : 0.0;
    std::memcpy(r, &x, sizeof(x));
    std::memcpy(r + sizeof(SlotInit), reps[i].data(), static_cast<std::size_t>(d_) * 8);
    if (x.has_brep) std::memcpy(r + sizeof(SlotInit) + static_cast<std::size_t>(d_) * 8, (*breps)[i].data(), static_cast<std::size_t>(d_) * 8);
  }
  std::memcpy(h + n * rb, slots.data(), n * 4);
  KVC_CUDA(cudaMemcpyAsync(d_init_, h_init_, bytes, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaEventRecord(ev_init_, st_));
  launches_ += launch_init_slots(t_, d_init_, static_cast<std::int32_t>(n), st_);
  launches_ += launch_refresh_mirror(
      t_, reinterpret_cast<const std::int32_t*>(static_cast<std::uint8_t*>(d_init_) + n * rb), static_cast<std::int32_t>(n), st_);
}

void Context::append_runs_idx(const std::vector<AppendRun>& runs, const std::vector<std::int32_t>& idx,
                              const void* src_k, const void* src_v) {
  if (runs.empty()) return;
  ensure_idx(static_cast<std::int64_t>(idx.size()), static_cast<std::int64_t>(runs.size()));
  std::memcpy(h_idx_, idx.data(), idx.size() * 4);
  std::memcpy(h_runs_, runs.data(), runs.size() * sizeof(AppendRun));
  KVC_CUDA(cudaMemcpyAsync(d_idx_, h_idx_, idx.size() * 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_runs_, h_runs_, runs.size() * sizeof(AppendRun), cudaMemcpyHostToDevice, st_));
  launches_ += launch_append_runs(t_, d_runs_, static_cast<std::int32_t>(runs.size()), d_idx_,
                                  src_k ? src_k : d_stage_k_, src_v ? src_v : d_stage_v_, st_);
  sync();
}

// Points the ring entries of the given tokens at `slot`. The ring holds the frames of the
// device view (including a frame being ingested, whose slot already replaced the oldest window
// frame), so lookups go through ring_frame_, not the reference-order window_.
void Context::ring_owner_patch(int layer, const std::vector<Member>& ids, std::int32_t slot) {
  // only members of the few window frames matter: one range test rejects the others
  std::int64_t lo = INT64_MAX, hi = INT64_MIN;
  for (int rs = 0; rs < t_.W; ++rs) {
    const RingFrame& rf = ring_frame_[static_cast<std::size_t>(rs)];
    if (rf.T <= 0) continue;
    lo = std::min(lo, rf.frame_id);
    hi = std::max(hi, rf.frame_id);
  }
  if (lo > hi) return;
  for (const Member& m : ids) {
    if (m.frame < lo || m.frame > hi) continue;
    for (int rs = 0; rs < t_.W; ++rs) {
      const RingFrame& rf = ring_frame_[static_cast<std::size_t>(rs)];
      if (rf.frame_id == m.frame && m.token < rf.T)
        ring_owner_h_[(static_cast<std::size_t>(layer) * t_.W + rs) * t_.tmax + m.token] = slot;
    }
  }
}

void Context::ring_owner_upload(int layer) {
  const std::size_t off = static_cast<std::size_t>(layer) * t_.W * t_.tmax;
  KVC_CUDA(cudaMemcpyAsync(t_.ring_owner + off, &ring_owner_h_[off], static_cast<std::size_t>(t_.W) * t_.tmax * 4,
                           cudaMemcpyHostToDevice, st_));
  sync();
}

// Maintainer::split_members (maintainer.cpp:195-242) over the staged pool rows
// [0, ids.size()). Emits children in reference order; installs their exact statistics and
// repacks their payload rows into fresh pages. Returns the new ids.
std::vector<std::int64_t> Context::split_pool(std::int64_t pid, int layer, bool host,
                                              std::vector<Member>&& ids, std::int64_t rows, int) {
  if (static_cast<std::int64_t>(ids.size()) != rows) fail(-11, "pool size mismatch");
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count();
  };
  const auto sd0 = now();
  stage_download(rows);
  evt_t_[1] += us(sd0, now());
  const float* keys = h_stage_f32_;
  std::vector<std::int64_t> out;
  std::vector<std::int32_t> slots;
  std::vector<std::vector<double>> reps;
  std::vector<double> vars;
  std::vector<std::int64_t> stats, nmem, cids;
  std::vector<std::uint8_t> res;
  std::vector<AppendRun> runs;
  std::vector<std::int32_t> idx;

  auto emit = [&](const std::vector<int>& g, std::vector<double>&& rep, double var) {
    std::vector<Member> m;
    m.reserve(g.size());
    for (int r : g) m.push_back(ids[static_cast<std::size_t>(r)]);
    const std::int64_t id = new_cluster(layer, pid, std::move(m), host);
    Cluster& c = C(id);
    adopt(id);
    out.push_back(id);
    slots.push_back(c.slot);
    reps.push_back(std::move(rep));
    vars.push_back(var);
    stats.push_back(static_cast<std::int64_t>(g.size()));
    nmem.push_back(static_cast<std::int64_t>(g.size()));
    cids.push_back(id);
    res.push_back(host ? 1 : 0);
    runs.push_back({c.slot, static_cast<std::int32_t>(idx.size()), static_cast<std::int32_t>(g.size()), 0});
    idx.insert(idx.end(), g.begin(), g.end());
  };

  auto rec = [&](auto&& self, std::vector<int> grp, int depth) -> void {
    if (grp.size() < 2) {
      std::vector<double> rep(static_cast<std::size_t>(d_));
      representative(keys, grp.data(), static_cast<int>(grp.size()), d_, rep.data());
      const double var = variance(keys, grp.data(), static_cast<int>(grp.size()), d_, rep.data());
      emit(grp, std::move(rep), var);
      return;
    }
    const auto k0 = now();
    KMeansOut halves;
    const std::uint64_t ctr = static_cast<std::uint64_t>(split_counter_++);
    if (!(depth == 0 && static_cast<std::int64_t>(grp.size()) == rows && spec_split_take(spec_slot_hint_, static_cast<int>(grp.size()), ctr, halves)))
      halves = split_two_staged(grp, mix_seed(maint_seed_, ctr));
    evt_t_[2] += us(k0, now());
    evt_t_[7] += 1.0;
    mstats_[5] += 1;  // split_ops_total
    std::vector<int> g2[2];
    for (std::size_t i = 0; i < grp.size(); ++i) g2[halves.assign[i]].push_back(grp[i]);
    for (auto& g : g2) {
      if (g.empty()) continue;
      std::vector<double> rep(static_cast<std::size_t>(d_));
      const auto h0 = now();
      representative(keys, g.data(), static_cast<int>(g.size()), d_, rep.data());
      const double var = variance(keys, g.data(), static_cast<int>(g.size()), d_, rep.data());
      evt_t_[3] += us(h0, now());
      if (depth + 1 < cfg_.max_split_depth && g.size() >= 2 &&
          var > tau_of(static_cast<std::int64_t>(g.size()), cfg_)) {
        self(self, std::move(g), depth + 1);
      } else {
        emit(g, std::move(rep), var);
      }
    }
  };
  std::vector<int> all(static_cast<std::size_t>(rows));
  std::iota(all.begin(), all.end(), 0);
  rec(rec, std::move(all), 0);

  const auto u0 = now();
  init_slots(slots, reps, vars, stats, nmem, cids, res, nullptr, nullptr);
  append_runs_idx(runs, idx);
  pl_upload(pid, layer);
  for (std::size_t i = 0; i < out.size(); ++i) ring_owner_patch(layer, C(out[i]).members, slots[i]);
  ring_owner_upload(layer);
  evt_t_[4] += us(u0, now());
  return out;
}

// split_two (kmeans.cpp, clustering.cpp:180-208) of the staged rows grp[]: on the GPU (split.cu)
// for groups of at least split_dev_min_ rows, else on the host. Both are bit-identical; the host
// owns the generator, so the device gets the seeding's two draws (first index, uniform) in the
// order plus_plus makes them.
KMeansOut Context::split_two_staged(const std::vector<int>& grp, std::uint64_t seed) {
  const int n = static_cast<int>(grp.size());
  if (split_dev_min_ <= 0 || n < std::max(2, split_dev_min_) || d_ > 256) {
    std::vector<float> sub(static_cast<std::size_t>(n) * d_);
    for (int i = 0; i < n; ++i)
      std::memcpy(&sub[static_cast<std::size_t>(i) * d_], h_stage_f32_ + static_cast<std::size_t>(grp[i]) * d_,
                  static_cast<std::size_t>(d_) * 4);
    return split_two(sub.data(), n, d_, seed);
  }
  Rng64 rng(seed);
  const int first = static_cast<int>(rng.index(static_cast<std::size_t>(n)));
  const double uni = rng.uniform();
  const std::size_t dbl = (static_cast<std::size_t>(n) * (2 * d_ + 3) + 1) * 8;
  const std::size_t ints = (2 * static_cast<std::size_t>(n) + 4) * 4;
  auto* base = static_cast<std::uint8_t*>(dalloc_scratch(dbl + ints));
  auto* u = reinterpret_cast<double*>(base);
  double* d_obj = u + static_cast<std::size_t>(n) * (2 * d_ + 3);
  auto* d_i = reinterpret_cast<std::int32_t*>(base + dbl);  // idx[n] | assign[n] | meta[4]
  const std::size_t hobj = (ints + 7) & ~std::size_t{7};
  if (static_cast<std::int64_t>(hobj + 8) > split_cap_) {
    split_cap_ = static_cast<std::int64_t>(hobj + 8) * 2;
    h_split_ = halloc(static_cast<std::size_t>(split_cap_));
  }
  auto* h_i = static_cast<std::int32_t*>(h_split_);
  auto* h_obj = reinterpret_cast<double*>(static_cast<std::uint8_t*>(h_split_) + hobj);
  std::memcpy(h_i, grp.data(), static_cast<std::size_t>(n) * 4);
  KVC_CUDA(cudaMemcpyAsync(d_i, h_i, static_cast<std::size_t>(n) * 4, cudaMemcpyHostToDevice, st_));
  launches_ += launch_split_two(d_stage_f32_, d_i, n, d_, first, uni, u, d_i + n, d_i + 2 * n, d_obj, st_);
  KVC_CUDA(cudaMemcpyAsync(h_i + n, d_i + n, static_cast<std::size_t>(n + 4) * 4, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(h_obj, d_obj, 8, cudaMemcpyDeviceToHost, st_));
  sync();
  const std::int32_t* meta = h_i + 2 * n;
  if (meta[3] != 0) fail(-2, "normalize of zero vector");
  KMeansOut o;
  o.assign.assign(h_i + n, h_i + 2 * n);
  o.k_live = meta[0];
  o.iterations = meta[1];
  o.degenerate = meta[2] != 0;
  o.objective = *h_obj;
  return o;
}

// Stage + 2-means of the first pending split of domains [from_layer, L) on the side stream, with
// the seed of the current split counter (see SpecSplit in context.hpp).
void Context::spec_split_launch(int from_layer, int T) {
  int l = -1;
  for (int x = from_layer; x < L_; ++x)
    if (h_stop_[x] < T) {
      l = x;
      break;
    }
  if (l < 0) return;
  const int kind = h_stop_[L_ + l];
  if (kind != EV_SPLIT && kind != EV_EAGER) return;  // seeds need no k-means
  const std::int32_t slot = h_stop_[2 * L_ + l];
  const int tok = h_stop_[l];
  if (slot < 0 || static_cast<std::size_t>(slot) >= slot_id_.size() || slot_id_[static_cast<std::size_t>(slot)] < 0) return;
  const std::int64_t cid = slot_id_[static_cast<std::size_t>(slot)];
  if (is_host(cid)) return;  // the settle re-resolves such a token (residence changed between frames)
  const Cluster& c = C(cid);
  // rows at the event = the cluster's rows before this frame + this domain's tokens routed to it
  // before the stop (committed on the device by the first round, replayed on the host later)
  std::int64_t n = static_cast<std::int64_t>(c.members.size() + c.buffer.size()) + 1;
  const std::int32_t* evs = h_evs_ + static_cast<std::size_t>(l) * t_.tmax;
  for (int t = 0; t < tok; ++t) n += evs[t] == slot ? 1 : 0;
  if (n < std::max(2, split_dev_min_) || d_ > 256) return;
  if (!spec_st_) {
    KVC_CUDA(cudaStreamCreateWithFlags(&spec_st_, cudaStreamNonBlocking));
    KVC_CUDA(cudaEventCreateWithFlags(&spec_.ev, cudaEventDisableTiming));
  }
  if (spec_.active) KVC_CUDA(cudaEventSynchronize(spec_.ev));  // its buffers are about to be reused
  if (n + 1 > spec_.cap) {
    spec_.cap = std::max<std::int64_t>(n + 1, spec_.cap * 2);
    const std::size_t rb = static_cast<std::size_t>(d_) * es_;
    spec_.dk = dalloc(static_cast<std::size_t>(spec_.cap) * rb);
    spec_.dv = dalloc(static_cast<std::size_t>(spec_.cap) * rb);
    spec_.df32 = static_cast<float*>(dalloc(static_cast<std::size_t>(spec_.cap) * d_ * 4));
    spec_.scratch = static_cast<double*>(dalloc((static_cast<std::size_t>(spec_.cap) * (2 * d_ + 3) + 1) * 8));
    spec_.d_i = static_cast<std::int32_t*>(dalloc((2 * static_cast<std::size_t>(spec_.cap) + 4) * 4));
    spec_.d_obj = static_cast<double*>(dalloc(8));
    spec_.h_i = static_cast<std::int32_t*>(halloc((2 * static_cast<std::size_t>(spec_.cap) + 4) * 4));
    spec_.h_obj = static_cast<double*>(halloc(8));
  }
  const std::uint64_t counter = static_cast<std::uint64_t>(split_counter_);
  Rng64 rng(mix_seed(maint_seed_, counter));
  const int first = static_cast<int>(rng.index(static_cast<std::size_t>(n)));
  const double uni = rng.uniform();
  // the side stream starts after everything queued so far (the first round's commits)
  KVC_CUDA(cudaEventRecord(spec_.ev, st_));
  KVC_CUDA(cudaStreamWaitEvent(spec_st_, spec_.ev, 0));
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  launches_ += launch_gather_cluster(t_, slot, 1, spec_.dk, spec_.dv, 0, spec_st_);
  const std::size_t frow = static_cast<std::size_t>(l) * t_.tmax + tok;
  KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(spec_.dk) + static_cast<std::size_t>(n - 1) * rb,
                           static_cast<std::uint8_t*>(d_fk_) + frow * rb, rb, cudaMemcpyDeviceToDevice, spec_st_));
  launches_ += launch_to_f32(t_, spec_.dk, spec_.df32, n * d_, spec_st_);
  for (std::int64_t i = 0; i < n; ++i) spec_.h_i[i] = static_cast<std::int32_t>(i);
  KVC_CUDA(cudaMemcpyAsync(spec_.d_i, spec_.h_i, static_cast<std::size_t>(n) * 4, cudaMemcpyHostToDevice, spec_st_));
  launches_ += launch_split_two(spec_.df32, spec_.d_i, static_cast<int>(n), d_, first, uni, spec_.scratch, spec_.d_i + n,
                                spec_.d_i + 2 * n, spec_.d_obj, spec_st_);
  KVC_CUDA(cudaMemcpyAsync(spec_.h_i + n, spec_.d_i + n, static_cast<std::size_t>(n + 4) * 4, cudaMemcpyDeviceToHost, spec_st_));
  KVC_CUDA(cudaMemcpyAsync(spec_.h_obj, spec_.d_obj, 8, cudaMemcpyDeviceToHost, spec_st_));
  KVC_CUDA(cudaEventRecord(spec_.ev, spec_st_));
  spec_.active = true;
  spec_.layer = l;
  spec_.tok = tok;
  spec_.slot = slot;
  spec_.rows = n;
  spec_.counter = counter;
  spec_tries_ += 1;
}

bool Context::spec_split_take(std::int32_t slot, int n, std::uint64_t counter, KMeansOut& out) {
  if (!spec_.active || slot < 0) return false;
  const bool hit = spec_.slot == slot && spec_.rows == n && spec_.counter == counter;
  if (!hit) return false;
  KVC_CUDA(cudaEventSynchronize(spec_.ev));
  spec_.active = false;
  const std::int32_t* meta = spec_.h_i + 2 * static_cast<std::size_t>(n);
  if (meta[3] != 0) return false;  // a degenerate row: the normal path raises it
  out.assign.assign(spec_.h_i + n, spec_.h_i + 2 * static_cast<std::size_t>(n));
  out.k_live = meta[0];
  out.iterations = meta[1];
  out.degenerate = meta[2] != 0;
  out.objective = *spec_.h_obj;
  spec_hits_ += 1;
  return true;
}

KMeansOut Context::debug_split_two_dev(const float* pts, int n, std::uint64_t seed) {
  if (n < 2) fail(-6, "split_two: need at least 2 points");
  ensure_stage(n + 1);
  KVC_CUDA(cudaMemcpyAsync(d_stage_f32_, pts, static_cast<std::size_t>(n) * d_ * 4, cudaMemcpyHostToDevice, st_));
  std::vector<int> grp(static_cast<std::size_t>(n));
  std::iota(grp.begin(), grp.end(), 0);
  const int keep = split_dev_min_;
  split_dev_min_ = 2;
  KMeansOut o;
  try {
    o = split_two_staged(grp, seed);
  } catch (...) {
    split_dev_min_ = keep;
    throw;
  }
  split_dev_min_ = keep;
  return o;
}

std::int64_t Context::handle_host_event(std::int64_t frame_id, std::int64_t pid, int layer, int tok,
                                        int kind, std::int32_t slot) {
  struct Tm {
    double* acc;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~Tm() { *acc += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(); }
  } tm{&evt_t_[0]};
  evt_t_[6] += 1.0;
  mstats_[0] += 1;  // inserts (maintainer.cpp:89)
  const std::size_t frow = static_cast<std::size_t>(layer) * t_.tmax + tok;
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  if (kind == EV_SEED) {  // seed_cluster (maintainer.cpp:74-86)
    ensure_stage(2);
    KVC_CUDA(cudaMemcpyAsync(d_stage_k_, static_cast<std::uint8_t*>(d_fk_) + frow * rb, rb, cudaMemcpyDeviceToDevice, st_));
    KVC_CUDA(cudaMemcpyAsync(d_stage_v_, static_cast<std::uint8_t*>(d_fv_) + frow * rb, rb, cudaMemcpyDeviceToDevice, st_));
    stage_download(1);
    std::vector<Member> m{{frame_id, tok}};
    const std::int64_t id = new_cluster(layer, pid, std::move(m), false);
    Cluster& c = C(id);
    std::vector<double> rep(h_stage_f32_, h_stage_f32_ + d_);
    init_slots({c.slot}, {rep}, {0.0}, {1}, {1}, {id}, {0}, nullptr, nullptr);
    append_runs_idx({{c.slot, 0, 1, 0}}, {0});
    adopt(id);
    pl_upload(pid, layer);
    ring_owner_patch(layer, c.members, c.slot);
    ring_owner_upload(layer);
    return id;
  }
  const std::int64_t cid = slot_id_[static_cast<std::size_t>(slot)];
  Cluster& c = C(cid);
  if (kind == EV_EAGER) {  // maintainer.cpp:151-158
    mstats_[6] += 1;
    fetch(cid, KVC_CAUSE_MAINTENANCE);
    mstats_[7] += 1;
  } else if (kind != EV_SPLIT) {
    fail(-11, "unknown host event");
  }
  mstats_[2] += 1;  // immediate_splits
  const auto ts0 = std::chrono::steady_clock::now();
  const std::int64_t rows = stage_cluster(c.slot, true);
  KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(d_stage_k_) + rows * rb,
                           static_cast<std::uint8_t*>(d_fk_) + frow * rb, rb, cudaMemcpyDeviceToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(d_stage_v_) + rows * rb,
                           static_cast<std::uint8_t*>(d_fv_) + frow * rb, rb, cudaMemcpyDeviceToDevice, st_));
  std::vector<Member> ids = c.members;
  for (const Member& m : c.buffer) ids.push_back(m);
  ids.push_back({frame_id, tok});
  forget(cid);
  drop_cluster(cid);
  spec_slot_hint_ = slot;
  const std::vector<std::int64_t> kids = split_pool(pid, layer, false, std::move(ids), rows + 1, 0);
  spec_slot_hint_ = -1;
  for (std::int64_t k : kids)  // home_of (maintainer.cpp:62-70)
    for (const Member& m : C(k).members)
      if (m.frame == frame_id && m.token == tok) return k;
  return kids.front();
}

std::vector<std::int64_t> Context::materialize(std::int64_t id) {  // maintainer.cpp:178-193
  Cluster& c = C(id);
  if (!is_lazy(id)) return {id};
  if (is_host(id)) fail(-11, "pending split settled without fetching the payload first");
  mstats_[4] += 1;  // settled_splits
  const std::int64_t rows = stage_cluster(c.slot, true);
  std::vector<Member> ids = c.members;
  for (const Member& m : c.buffer) ids.push_back(m);
  const std::int64_t pid = c.parent;
  const int layer = c.layer;
  const bool host = is_host(id);
  forget(id);
  drop_cluster(id);
  return split_pool(pid, layer, host, std::move(ids), rows, 0);
}

// ============================================================================ build

// Batch spherical k-means of host point sets on the GPU (the index build's per-(partition, layer)
// pools, index.cpp:405-425): one CTA per set, all sets of a chunk in one launch.
std::vector<KMeansOut> Context::kmeans_pools(const std::vector<const float*>& pts, const std::vector<int>& n,
                                             const std::vector<int>& k_req, const std::vector<std::uint64_t>& seeds,
                                             int max_iters, double tol, bool stats) {
  const std::size_t np = pts.size();
  std::vector<KMeansOut> out(np);
  const bool host_only = std::getenv("KVC_BUILD_HOST") != nullptr;  // ablation: host k-means
  std::vector<std::size_t> dev;
  for (std::size_t i = 0; i < np; ++i) {
    const int k = std::max(1, std::min(k_req[i], n[i]));
    if (!host_only && n[i] >= 1 && kmeans_smem_bytes(k, d_) <= 227 * 1024)
      dev.push_back(i);
    else
      out[i] = spherical_kmeans(pts[i], n[i], d_, k_req[i], max_iters, tol, seeds[i]);
  }
  const std::size_t budget = std::size_t{3} << 30;  // scratch bytes per launch
  for (std::size_t b = 0; b < dev.size();) {
    std::size_t e = b, rows = 0, scr = 0, unis = 0;
    int kmax = 1;
    while (e < dev.size()) {
      const std::size_t i = dev[e];
      const std::size_t s = kmeans_scratch_doubles(n[i], d_) * 8;
      if (e > b && scr + s > budget) break;
      const int k = std::max(1, std::min(k_req[i], n[i]));
      rows += static_cast<std::size_t>(n[i]);
      scr += s;
      unis += static_cast<std::size_t>(k);
      kmax = std::max(kmax, k);
      ++e;
    }
    const std::size_t nj = e - b;
    // device: rows f32 | uniforms | jobs | assign (padded) | meta[4] | objective | reps | vars | scratch
    std::size_t kd = 0, ksum = 0;
    for (std::size_t q = 0; q < nj; ++q) {
      const std::size_t i = dev[b + q];
      const std::size_t k = static_cast<std::size_t>(std::max(1, std::min(k_req[i], n[i])));
      ksum += k;
      kd += k * d_;
    }
    const std::size_t rows_pad = (rows + 1) & ~std::size_t{1};
    const std::size_t rows_b = rows * d_ * 4, uni_b = unis * 8, job_b = nj * sizeof(KmJob);
    const std::size_t out_b = rows_pad * 4 + nj * 16 + nj * 8 + (stats ? (kd + ksum) * 8 : 0);
    const std::size_t in_b = rows_b + uni_b + job_b;
    void* dp = nullptr;
    struct Free {
      void*& d;
      ~Free() {
        if (d) cudaFree(d);
      }
    } guard{dp};
    KVC_CUDA(cudaMalloc(&dp, in_b + out_b + scr));
    auto* d8 = static_cast<std::uint8_t*>(dp);
    std::vector<double> huni(unis);
    std::vector<KmJob> hjob(nj);
    std::size_t r0 = 0, s0 = 0, u0 = 0, k0 = 0;
    for (std::size_t q = 0; q < nj; ++q) {
      const std::size_t i = dev[b + q];
      const int k = std::max(1, std::min(k_req[i], n[i]));
      KVC_CUDA(cudaMemcpyAsync(d8 + r0 * d_ * 4, pts[i], static_cast<std::size_t>(n[i]) * d_ * 4,
                               cudaMemcpyHostToDevice, st_));
      Rng64 rng(seeds[i]);  // plus_plus's draws in order: the first index, then one uniform per pick
      KmJob j{};
      j.row0 = static_cast<std::int64_t>(r0);
      j.scratch0 = static_cast<std::int64_t>(s0);
      j.rep0 = stats ? static_cast<std::int64_t>(k0 * d_) : -1;
      j.var0 = static_cast<std::int32_t>(k0);
      j.n = n[i];
      j.k = k;
      j.first = static_cast<std::int32_t>(rng.index(static_cast<std::size_t>(n[i])));
      j.out0 = static_cast<std::int32_t>(r0);
      j.uni0 = static_cast<std::int32_t>(u0);
      for (int t = 0; t + 1 < k; ++t) huni[u0 + t] = rng.uniform();
      hjob[q] = j;
      r0 += static_cast<std::size_t>(n[i]);
      s0 += kmeans_scratch_doubles(n[i], d_);
      u0 += static_cast<std::size_t>(k);
      k0 += static_cast<std::size_t>(k);
    }
    KVC_CUDA(cudaMemcpyAsync(d8 + rows_b, huni.data(), uni_b, cudaMemcpyHostToDevice, st_));
    KVC_CUDA(cudaMemcpyAsync(d8 + rows_b + uni_b, hjob.data(), job_b, cudaMemcpyHostToDevice, st_));
    auto* d_assign = reinterpret_cast<std::int32_t*>(d8 + in_b);
    auto* d_meta = d_assign + rows_pad;
    auto* d_obj = reinterpret_cast<double*>(d_meta + nj * 4);
    auto* d_reps = d_obj + nj;
    auto* d_vars = d_reps + kd;
    auto* d_scr = reinterpret_cast<double*>(d8 + in_b + out_b);
    KVC_CUDA(cudaMemsetAsync(d_meta, 0, nj * 16, st_));
    launches_ += launch_kmeans(reinterpret_cast<const float*>(d8), reinterpret_cast<const KmJob*>(d8 + rows_b + uni_b),
                               static_cast<int>(nj), reinterpret_cast<const double*>(d8 + rows_b), d_scr, d_assign,
                               d_meta, d_obj, d_reps, d_vars, d_, kmax, max_iters, tol, st_);
    KVC_CUDA(cudaGetLastError());
    std::vector<std::uint8_t> hout(out_b);
    KVC_CUDA(cudaMemcpyAsync(hout.data(), d_assign, out_b, cudaMemcpyDeviceToHost, st_));
    sync();
    const auto* ha = reinterpret_cast<const std::int32_t*>(hout.data());
    const auto* hm = ha + rows_pad;
    const auto* ho = reinterpret_cast<const double*>(hm + nj * 4);
    const double* hr = ho + nj;
    const double* hv = hr + kd;
    for (std::size_t q = 0; q < nj; ++q) {
      const std::size_t i = dev[b + q];
      if (hm[q * 4 + 3] != 0) fail(-2, "normalize of zero vector");
      KMeansOut& o = out[i];
      const KmJob& j = hjob[q];
      o.assign.assign(ha + j.out0, ha + j.out0 + n[i]);
      o.k_live = hm[q * 4 + 0];
      o.iterations = hm[q * 4 + 1];
      o.objective = ho[q];
      if (stats) {
        o.reps.assign(hr + j.rep0, hr + j.rep0 + static_cast<std::size_t>(o.k_live) * d_);
        o.vars.assign(hv + j.var0, hv + j.var0 + o.k_live);
      }
    }
    b = e;
  }
  return out;
}

void Context::build_now() {  // engine.cpp:77-93 + build_index (index.cpp:364-450)
  if (built_) return;
  if (pending_.empty()) fail(-9, "no frames available to build from");
  // engine.cpp:79: BuildConfig::seed = mix_seed(engine seed, 1); a direct build_index call passes
  // its BuildConfig's seed verbatim (kvc_reconfigure bit 8)
  const std::uint64_t bseed = build_seed_set_ ? build_seed_ : mix_seed(cfg_.seed, 1);
  maint_seed_ = mix_seed(cfg_.seed, 2);
  const int n = static_cast<int>(pending_.size());
  std::vector<float> vis(static_cast<std::size_t>(n) * d_);
  for (int i = 0; i < n; ++i) std::memcpy(&vis[static_cast<std::size_t>(i) * d_], pending_[static_cast<std::size_t>(i)].visual.data(), d_ * 4);
  const int kv = (n + cfg_.target_visual_cluster_size - 1) / cfg_.target_visual_cluster_size;
  const KMeansOut vk = spherical_kmeans(vis.data(), n, d_, kv, cfg_.kmeans_max_iters, cfg_.kmeans_tol, bseed);
  std::vector<std::vector<int>> pf(static_cast<std::size_t>(vk.k_live));
  for (int i = 0; i < n; ++i) pf[static_cast<std::size_t>(vk.assign[static_cast<std::size_t>(i)])].push_back(i);
  for (std::size_t p = 0; p < pf.size(); ++p) {
    Partition part;
    std::vector<double> acc(static_cast<std::size_t>(d_), 0.0);  // dmean (vecmath.hpp:80-92)
    for (int fi : pf[p]) {
      part.frames.push_back(pending_[static_cast<std::size_t>(fi)].frame_id);
      for (int c = 0; c < d_; ++c) acc[static_cast<std::size_t>(c)] += static_cast<double>(pending_[static_cast<std::size_t>(fi)].visual[static_cast<std::size_t>(c)]);
    }
    const double inv = 1.0 / static_cast<double>(pf[p].size());
    for (double& x : acc) x *= inv;
    part.vrep = std::move(acc);
    part.stat = static_cast<std::int64_t>(pf[p].size());
    part.per_layer.resize(static_cast<std::size_t>(L_));
    part.dev_off.assign(static_cast<std::size_t>(L_), 0);
    part.dev_cap.assign(static_cast<std::size_t>(L_), 0);
    if (static_cast<std::int32_t>(parts_.size()) >= t_.max_parts) fail(-21, "too many partitions");
    parts_.push_back(std::move(part));
    upload_partition(static_cast<std::int64_t>(parts_.size()) - 1);
  }
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  // every (partition, layer) pool's semantic k-means at once on the GPU (index.cpp:405-425)
  std::vector<std::vector<float>> pool_keys;
  std::vector<const float*> pool_ptr;
  std::vector<int> pool_n, pool_k;
  std::vector<std::uint64_t> pool_seed;
  for (std::size_t p = 0; p < pf.size(); ++p)
    for (int layer = 0; layer < L_; ++layer) {
      std::int64_t rows = 0;
      for (int fi : pf[p]) rows += pending_[static_cast<std::size_t>(fi)].T;
      std::vector<float> keys(static_cast<std::size_t>(rows) * d_);
      std::int64_t r = 0;
      for (int fi : pf[p]) {
        const PendingFrame& f = pending_[static_cast<std::size_t>(fi)];
        const std::size_t base = static_cast<std::size_t>(layer) * f.T;
        std::memcpy(&keys[static_cast<std::size_t>(r) * d_], &f.keys_f32[base * d_], static_cast<std::size_t>(f.T) * d_ * 4);
        r += f.T;
      }
      pool_n.push_back(static_cast<int>(rows));
      pool_k.push_back(static_cast<int>((rows + cfg_.target_semantic_cluster_size - 1) / cfg_.target_semantic_cluster_size));
      pool_seed.push_back(mix_seed(bseed, (static_cast<std::uint64_t>(p) << 8) | static_cast<std::uint64_t>(layer) | 0x100u));
      pool_keys.push_back(std::move(keys));
      pool_ptr.push_back(pool_keys.back().data());
    }
  const auto bt0 = std::chrono::steady_clock::now();
  std::vector<KMeansOut> pool_km;
  {
    std::vector<const float*> ptr;
    std::vector<int> nn, kk;
    std::vector<std::uint64_t> ss;
    std::vector<std::size_t> which;
    for (std::size_t i = 0; i < pool_n.size(); ++i)
      if (pool_n[i] > 0) {
        ptr.push_back(pool_keys[i].data());
        nn.push_back(pool_n[i]);
        kk.push_back(pool_k[i]);
        ss.push_back(pool_seed[i]);
        which.push_back(i);
      }
    std::vector<KMeansOut> r = kmeans_pools(ptr, nn, kk, ss, cfg_.kmeans_max_iters, cfg_.kmeans_tol, true);
    pool_km.resize(pool_n.size());
    for (std::size_t q = 0; q < which.size(); ++q) pool_km[which[q]] = std::move(r[q]);
  }
  const auto bt1 = std::chrono::steady_clock::now();
  double t_repvar = 0.0, t_dev = 0.0;
  for (std::size_t p = 0; p < pf.size(); ++p) {
    for (int layer = 0; layer < L_; ++layer) {
      // pool = frames of the partition in order, tokens in order (index.cpp:405-409)
      const std::size_t pool = p * static_cast<std::size_t>(L_) + static_cast<std::size_t>(layer);
      std::vector<Member> ids;
      const std::int64_t rows = pool_n[pool];
      if (rows == 0) continue;
      ensure_stage(rows + 1);
      const std::vector<float>& keys = pool_keys[pool];
      std::vector<std::uint8_t> kraw(static_cast<std::size_t>(rows) * rb), vraw(static_cast<std::size_t>(rows) * rb);
      std::int64_t r = 0;
      for (int fi : pf[p]) {
        const PendingFrame& f = pending_[static_cast<std::size_t>(fi)];
        const std::size_t base = static_cast<std::size_t>(layer) * f.T;
        std::memcpy(&kraw[static_cast<std::size_t>(r) * rb], &f.keys_raw[base * rb], static_cast<std::size_t>(f.T) * rb);
        std::memcpy(&vraw[static_cast<std::size_t>(r) * rb], &f.vals_raw[base * rb], static_cast<std::size_t>(f.T) * rb);
        for (int t = 0; t < f.T; ++t) ids.push_back({f.frame_id, t});
        r += f.T;
      }
      KVC_CUDA(cudaMemcpyAsync(d_stage_k_, kraw.data(), kraw.size(), cudaMemcpyHostToDevice, st_));
      KVC_CUDA(cudaMemcpyAsync(d_stage_v_, vraw.data(), vraw.size(), cudaMemcpyHostToDevice, st_));
      const KMeansOut& sk = pool_km[pool];
      std::vector<std::vector<int>> groups(static_cast<std::size_t>(sk.k_live));
      for (std::int64_t i = 0; i < rows; ++i) groups[static_cast<std::size_t>(sk.assign[static_cast<std::size_t>(i)])].push_back(static_cast<int>(i));
      std::vector<std::int32_t> slots;
      std::vector<std::vector<double>> reps;
      std::vector<double> vars;
      std::vector<std::int64_t> stats, nmem, cids;
      std::vector<std::uint8_t> res;
      std::vector<AppendRun> runs;
      std::vector<std::int32_t> idx;
      for (auto& g : groups) {
        const auto rv0 = std::chrono::steady_clock::now();
        const std::size_t gi = static_cast<std::size_t>(&g - groups.data());
        std::vector<double> rep(static_cast<std::size_t>(d_));
        double var;
        if (!sk.vars.empty()) {  // computed by the device build with the k-means
          std::copy_n(&sk.reps[gi * d_], d_, rep.begin());
          var = sk.vars[gi];
        } else {
          representative(keys.data(), g.data(), static_cast<int>(g.size()), d_, rep.data());
          var = variance(keys.data(), g.data(), static_cast<int>(g.size()), d_, rep.data());
        }
        t_repvar += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - rv0).count();
        std::vector<Member> m;
        for (int i : g) m.push_back(ids[static_cast<std::size_t>(i)]);
        const std::int64_t id = new_cluster(layer, static_cast<std::int64_t>(p), std::move(m), false);
        const Cluster& c = C(id);
        slots.push_back(c.slot);
        reps.push_back(std::move(rep));
        vars.push_back(var);
        stats.push_back(static_cast<std::int64_t>(g.size()));
        nmem.push_back(static_cast<std::int64_t>(g.size()));
        cids.push_back(id);
        res.push_back(0);
        runs.push_back({c.slot, static_cast<std::int32_t>(idx.size()), static_cast<std::int32_t>(g.size()), 0});
        idx.insert(idx.end(), g.begin(), g.end());
      }
      const auto dv0 = std::chrono::steady_clock::now();
      init_slots(slots, reps, vars, stats, nmem, cids, res, nullptr, nullptr);
      append_runs_idx(runs, idx);
      pl_upload(static_cast<std::int64_t>(p), layer);
      t_dev += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - dv0).count();
    }
  }
  const auto bt2 = std::chrono::steady_clock::now();
  if (std::getenv("KVC_BUILD_TIMING"))
    std::fprintf(stderr, "build: kmeans %.1f ms, pools %.1f ms (rep/var %.1f, device %.1f)\n",
                 std::chrono::duration<double, std::milli>(bt1 - bt0).count(),
                 std::chrono::duration<double, std::milli>(bt2 - bt1).count(), t_repvar, t_dev);
  // TieredStore(index, cost) adopts every cluster in id order (store.cpp:67-74)
  for (std::int64_t id : cluster_ids()) adopt(id);
  built_ = true;
  const auto bt3 = std::chrono::steady_clock::now();
  const std::int64_t last = pending_.back().frame_id;
  pending_.clear();
  // ring owners of the window frames
  for (int layer = 0; layer < L_; ++layer) {
    for (const auto& up : clusters_)
      if (up && up->layer == layer) ring_owner_patch(layer, up->members, up->slot);
    ring_owner_upload(layer);
  }
  repin();
  apply_cadence(last, -1);
  tier_kick();
  if (std::getenv("KVC_BUILD_TIMING"))
    std::fprintf(stderr, "build: adopt %.1f ms, ring/repin/cadence %.1f ms\n",
                 std::chrono::duration<double, std::milli>(bt3 - bt2).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - bt3).count());
  if (cfg_.check_invariants) check();
}

}  // namespace kvc
