// context_api.cpp -- component-level operations of the reference's C++ API on the device engine
// (HierIndex / TieredStore / Maintainer / retrieve as separate calls), used by the
// C++ drop-in (include/kvclust_b200.hpp) through the C-ABI. The engine-level path
// (StreamEngine: kvc_ingest_frame / kvc_decode_step) does not go through here.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "context.hpp"

namespace kvc {

// HierIndex::add_partition (index.cpp:59-69): a partition with one frame, not counted as opened
// by the maintainer.
std::int64_t Context::api_add_partition(std::int64_t first_frame, const float* visual) {
  flush_pending();
  if (static_cast<std::int32_t>(parts_.size()) >= t_.max_parts) fail(-21, "too many partitions (raise max_partitions)");
  if (!built_) {
    built_ = true;  // an index assembled by hand is "built" (no batch build pending)
    maint_seed_ = mix_seed(cfg_.seed, 2);
  }
  Partition p;
  p.frames.push_back(first_frame);
  p.vrep.assign(visual, visual + d_);
  p.stat = 1;
  p.per_layer.resize(static_cast<std::size_t>(L_));
  p.dev_off.assign(static_cast<std::size_t>(L_), 0);
  p.dev_cap.assign(static_cast<std::size_t>(L_), 0);
  parts_.push_back(std::move(p));
  const std::int64_t pid = static_cast<std::int64_t>(parts_.size()) - 1;
  upload_partition(pid);
  std::vector<std::int32_t> z(static_cast<std::size_t>(L_), 0);
  KVC_CUDA(cudaMemcpyAsync(t_.pl_cnt + pid * L_, z.data(), L_ * 4, cudaMemcpyHostToDevice, st_));
  sync();
  return pid;
}

// HierIndex::append_frame (index.cpp:71-79)
void Context::api_append_frame(std::int64_t pid, std::int64_t frame, const float* visual) {
  flush_pending();
  if (pid < 0 || pid >= static_cast<std::int64_t>(parts_.size())) fail(-8, "unknown partition id");
  Partition& p = parts_[static_cast<std::size_t>(pid)];
  p.frames.push_back(frame);
  const double n = static_cast<double>(p.stat);
  for (int i = 0; i < d_; ++i) p.vrep[static_cast<std::size_t>(i)] = (n * p.vrep[static_cast<std::size_t>(i)] + visual[i]) / (n + 1.0);
  p.stat += 1;
  upload_partition(pid);
  sync();
}

// HierIndex::add_cluster (index.cpp:97-120) of one cluster with members keys/values [n][d] f32
// (host), exact Eq. 1/2 statistics computed on the device, plus TieredStore::adopt when `adopt`.
std::int64_t Context::api_add_cluster(int layer, std::int64_t parent, int n, const float* keys, const float* values,
                                      const std::int64_t* frames, const std::int32_t* tokens, bool host, bool adopt_it) {
  flush_pending();
  if (n < 1) fail(-5, "cluster with no members");
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range: " + std::to_string(layer));
  if (parent < 0 || parent >= static_cast<std::int64_t>(parts_.size())) fail(-8, "unknown partition id");
  if (cfg_.kv_dtype != KVC_DTYPE_F32) fail(-10, "add_cluster takes f32 payloads (kv_dtype f32 contexts)");
  std::vector<Member> m(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) m[static_cast<std::size_t>(i)] = {frames[i], tokens[i]};
  const std::int64_t id = new_cluster(layer, parent, std::move(m), host);
  const Cluster& cl = C(id);
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  ensure_stage(n + 1);
  KVC_CUDA(cudaMemcpyAsync(d_stage_k_, keys, static_cast<std::size_t>(n) * rb, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_stage_v_, values, static_cast<std::size_t>(n) * rb, cudaMemcpyHostToDevice, st_));
  {
    SlotHeader hd{cl.slot, 0, id, static_cast<std::int64_t>(n)};
    auto* dh = static_cast<SlotHeader*>(dalloc_scratch(sizeof(SlotHeader)));
    KVC_CUDA(cudaMemcpyAsync(dh, &hd, sizeof(SlotHeader), cudaMemcpyHostToDevice, st_));
    launches_ += launch_slot_headers(t_, dh, 1, st_);
    sync();
  }
  std::vector<std::int32_t> idx(static_cast<std::size_t>(n));
  std::iota(idx.begin(), idx.end(), 0);
  ensure_idx(n, 1);
  std::memcpy(h_idx_, idx.data(), idx.size() * 4);
  AppendRun run{cl.slot, 0, n, 0};
  std::memcpy(h_runs_, &run, sizeof(AppendRun));
  KVC_CUDA(cudaMemcpyAsync(d_idx_, h_idx_, idx.size() * 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_runs_, h_runs_, sizeof(AppendRun), cudaMemcpyHostToDevice, st_));
  launches_ += launch_exact_stats(t_, d_runs_, 1, d_idx_, d_stage_k_, st_);
  launches_ += launch_append_runs(t_, d_runs_, 1, d_idx_, d_stage_k_, d_stage_v_, st_);
  sync();
  check_dev_err();
  resid_h_[static_cast<std::size_t>(cl.slot)] = host ? 1 : 0;
  resid_dirty_ = true;
  flush_resid();
  pl_upload(parent, layer);
  if (adopt_it) adopt(id);
  return id;
}

// A VisualPartition installed verbatim (frames, fp64 visual_rep, visual_stat_count): a parsed
// index (HierIndex::from_json_string) or a host-assembled one whose frames were appended.
std::int64_t Context::api_add_partition_ex(const std::int64_t* frames, int n_frames, const double* visual_rep,
                                           std::int64_t stat) {
  flush_pending();
  if (n_frames < 1) fail(-10, "a partition needs at least one frame");
  const std::int64_t pid = api_add_partition(frames[0], std::vector<float>(static_cast<std::size_t>(d_), 0.f).data());
  Partition& p = parts_[static_cast<std::size_t>(pid)];
  p.frames.assign(frames, frames + n_frames);
  p.vrep.assign(visual_rep, visual_rep + d_);
  p.stat = stat;
  upload_partition(pid);
  sync();
  return pid;
}

// A ClusterRecord installed verbatim (index.hpp:29-50): members and pending-split buffer entries
// (f32 payloads), rep / variance / stat_count / buffer_rep as given (the caller's statistics,
// not recomputed), lazy flag (= registered buffer), residence, device tail. want_id >= the next
// id keeps the caller's id (ids are never reused: index.cpp:105).
std::int64_t Context::api_add_cluster_ex(int layer, std::int64_t parent, int n_mem, const float* mk, const float* mv,
                                         const std::int64_t* mf, const std::int32_t* mt, int n_buf, const float* bk,
                                         const float* bv, const std::int64_t* bf, const std::int32_t* bt, const double* rep,
                                         double var, std::int64_t stat, const double* brep, bool lazy, bool host,
                                         std::int64_t device_tail, bool adopt_it, std::int64_t want_id) {
  flush_pending();
  if (n_mem < 1) fail(-5, "cluster with no members");
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range: " + std::to_string(layer));
  if (parent < 0 || parent >= static_cast<std::int64_t>(parts_.size())) fail(-8, "unknown partition id");
  if (cfg_.kv_dtype != KVC_DTYPE_F32) fail(-10, "add_cluster takes f32 payloads (kv_dtype f32 contexts)");
  if (want_id >= 0) {
    if (want_id < static_cast<std::int64_t>(clusters_.size())) fail(-10, "cluster ids are never reused");
    while (static_cast<std::int64_t>(clusters_.size()) < want_id) {  // skipped ids stay dead
      clusters_.push_back(nullptr);
      cflags_.push_back(0);
      last_use_.push_back(0);
    }
  }
  std::vector<Member> m(static_cast<std::size_t>(n_mem));
  for (int i = 0; i < n_mem; ++i) m[static_cast<std::size_t>(i)] = {mf[i], mt[i]};
  const std::int64_t id = new_cluster(layer, parent, std::move(m), host);
  Cluster& c = C(id);
  if (n_buf > 0) {
    std::vector<Member> b(static_cast<std::size_t>(n_buf));
    for (int i = 0; i < n_buf; ++i) b[static_cast<std::size_t>(i)] = {bf[i], bt[i]};
    c.buffer = MemberList(b);
    for (const MemberList::Run& r : c.buffer.runs()) frame_add(r.frame, id);
  }
  c.stat_count = stat;
  c.device_tail = device_tail;
  if (lazy) set_flag(id, CF_LAZY, true);
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  ensure_stage(n_mem + n_buf + 1);
  KVC_CUDA(cudaMemcpyAsync(d_stage_k_, mk, static_cast<std::size_t>(n_mem) * rb, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_stage_v_, mv, static_cast<std::size_t>(n_mem) * rb, cudaMemcpyHostToDevice, st_));
  if (n_buf > 0) {
    KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(d_stage_k_) + static_cast<std::size_t>(n_mem) * rb, bk,
                             static_cast<std::size_t>(n_buf) * rb, cudaMemcpyHostToDevice, st_));
    KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(d_stage_v_) + static_cast<std::size_t>(n_mem) * rb, bv,
                             static_cast<std::size_t>(n_buf) * rb, cudaMemcpyHostToDevice, st_));
  }
  std::vector<double> r(rep, rep + d_), b(static_cast<std::size_t>(d_), 0.0);
  if (brep) b.assign(brep, brep + d_);
  const std::vector<std::int32_t> nb{n_buf};
  const std::vector<std::vector<double>> breps{b};
  init_slots({c.slot}, {r}, {var}, {stat}, {static_cast<std::int64_t>(n_mem)}, {id}, {static_cast<std::uint8_t>(host ? 1 : 0)},
             &nb, &breps);
  std::vector<AppendRun> runs{{c.slot, 0, n_mem, 0}};
  if (n_buf > 0) runs.push_back({c.slot, n_mem, n_buf, 1});
  std::vector<std::int32_t> idx(static_cast<std::size_t>(n_mem + n_buf));
  std::iota(idx.begin(), idx.end(), 0);
  append_runs_idx(runs, idx);
  check_dev_err();
  resid_h_[static_cast<std::size_t>(c.slot)] = host ? 1 : 0;
  resid_dirty_ = true;
  flush_resid();
  pl_upload(parent, layer);
  if (adopt_it) adopt(id);
  return id;
}

void Context::api_adopt(std::int64_t id) {
  flush_pending();
  C(id);
  adopt(id);
}

// retrieve()'s explicit window argument (retrieval.cpp:99-110) empty: no window tokens attended.
void Context::api_reset_window() {
  flush_pending();
  window_.clear();
  for (auto& rf : ring_frame_) rf = RingFrame{};
  std::fill(ring_owner_h_.begin(), ring_owner_h_.end(), -1);
  KVC_CUDA(cudaMemcpyAsync(t_.ring_owner, ring_owner_h_.data(), ring_owner_h_.size() * 4, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemsetAsync(t_.ring_count, 0, static_cast<std::size_t>(t_.W) * 4, st_));
  sync();
  repin();
}

// Per-call RetrievalConfig (retrieval.hpp:20-32): budgets and simulated-cost constants.
void Context::api_set_retrieval(const kvc_cfg& c) {
  flush_pending();
  if (c.k_v <= 0 || c.k_s <= 0 || c.prefetch_k <= 0) fail(-10, "retrieval budgets must be positive");
  if (c.lookup_cost_per_candidate_us < 0.0 || c.compute_cost_per_token_us < 0.0)
    fail(-10, "cost constants must be non-negative");
  const std::int32_t kv = std::min(c.k_v, t_.max_parts), ks = std::min(c.k_s, t_.cmax),
                     kp = std::min(c.prefetch_k, t_.cmax);
  if (kv > kv_cap_ || ks > ks_cap_ || kp > kp_cap_) alloc_result_blocks(kv, ks, kp);
  cfg_.k_v = c.k_v;
  cfg_.k_s = c.k_s;
  cfg_.prefetch_k = c.prefetch_k;
  cfg_.prefetch_enabled = c.prefetch_enabled;
  cfg_.lookup_cost_per_candidate_us = c.lookup_cost_per_candidate_us;
  cfg_.compute_cost_per_token_us = c.compute_cost_per_token_us;
  da_.k_v = kv;
  da_.k_s = ks;
  da_.prefetch_k = kp;
  da_.prefetch = cfg_.prefetch_enabled;
}

// TieredStore's CostModel (store.hpp:17-31) / Maintainer's config (maintainer.hpp:28-34) of a
// component-level caller; the maintainer's split seeds come from cfg.seed directly
// (MaintainerConfig::seed, maintainer.cpp:222), not from an engine seed.
void Context::api_reconfigure(const kvc_cfg& c, int what) {
  flush_pending();
  if (what & 1) api_set_retrieval(c);
  if (what & 2) {
    if (c.alpha_us < 0.0 || c.beta_us_per_byte < 0.0) fail(-10, "transfer costs must be non-negative");
    if (c.device_capacity_entries <= 0) fail(-10, "device capacity must be positive");
    cfg_.alpha_us = c.alpha_us;
    cfg_.beta_us_per_byte = c.beta_us_per_byte;
    cfg_.bytes_per_entry = c.bytes_per_entry;
    cfg_.device_capacity_entries = c.device_capacity_entries;
  }
  if (what & 8) {  // BuildConfig of a direct build_index call (index.hpp:76-82), seed verbatim
    if (c.target_visual_cluster_size < 1 || c.target_semantic_cluster_size < 1)
      fail(-10, "target cluster sizes must be positive");
    cfg_.target_visual_cluster_size = c.target_visual_cluster_size;
    cfg_.target_semantic_cluster_size = c.target_semantic_cluster_size;
    cfg_.kmeans_max_iters = c.kmeans_max_iters;
    cfg_.kmeans_tol = c.kmeans_tol;
    build_seed_set_ = true;
    build_seed_ = c.seed;
  }
  if (what & 4) {
    if (c.tau_min < 0.0 || c.tau_max < c.tau_min) fail(-10, "variance thresholds must satisfy 0 <= tau_min <= tau_max");
    if (c.n0 <= 0.0) fail(-10, "threshold horizon must be positive");
    if (c.max_split_depth < 1) fail(-10, "split depth must be at least 1");
    if (c.visual_floor < -1.0 || c.visual_floor > 1.0) fail(-10, "visual floor must be a cosine value");
    cfg_.tau_min = c.tau_min;
    cfg_.tau_max = c.tau_max;
    cfg_.n0 = c.n0;
    cfg_.defer_host_splits = c.defer_host_splits;
    cfg_.max_split_depth = c.max_split_depth;
    cfg_.visual_floor = c.visual_floor;
    ia_.defer = cfg_.defer_host_splits;
    maint_seed_ = c.seed;
    upload_tau();
  }
}

// A Maintainer may start on an empty HierIndex (maintainer.cpp:37-53 opens the first partition):
// the component API owns the index from then on (no engine batch build pending).
void Context::component_index() {
  if (built_) return;
  if (!pending_.empty()) fail(-9, "the engine is still collecting its build batch (ingest_frame before build)");
  built_ = true;
}

std::int64_t Context::api_place_frame(std::int64_t frame, const float* visual) {  // maintainer.cpp:37-53
  flush_pending();
  component_index();
  return place_frame(frame, visual);
}

// Maintainer::on_insert (maintainer.cpp:88-176) of one entry: the device resolve (candidate scan,
// exact Eq. 3/4, Eq. 5 decision) of a single token of one domain, with host events (seed / split)
// settled exactly as in a frame; no window ring row (ia_.ring_slot = -1). Returns the routed id.
std::int64_t Context::api_insert(std::int64_t pid, int layer, int token, std::int64_t frame, const float* key,
                                 const float* value) {
  flush_pending();
  component_index();
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range: " + std::to_string(layer));
  if (pid < 0 || pid >= static_cast<std::int64_t>(parts_.size())) fail(-8, "unknown partition id");
  if (token < 0 || token >= t_.tmax) fail(-10, "token id outside [0, max_tokens)");
  if (cfg_.kv_dtype != KVC_DTYPE_F32) fail(-10, "on_insert takes f32 payloads (kv_dtype f32 contexts)");
  select_frame_buffer(0);
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  const std::size_t row = static_cast<std::size_t>(layer) * t_.tmax + token;
  KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(d_fk_) + row * rb, key, rb, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(static_cast<std::uint8_t*>(d_fv_) + row * rb, value, rb, cudaMemcpyHostToDevice, st_));
  ia_.T = token + 1;
  ia_.pid = static_cast<std::int32_t>(pid);
  ia_.ring_slot = -1;
  ia_.my_events = nullptr;
  ia_.prev_events = nullptr;
  std::vector<std::int64_t> assigned(static_cast<std::size_t>(L_) * (token + 1), -1);
  run_inserts(frame, pid, token + 1, assigned.data(), false, layer, layer + 1, token);
  KVC_CUDA(cudaEventRecord(ev_buf_[0], st_));
  sync();
  return assigned[static_cast<std::size_t>(layer) * (token + 1) + token];
}

std::vector<std::int64_t> Context::api_materialize(std::int64_t id) {  // maintainer.cpp:178-193
  flush_pending();
  C(id);
  return materialize(id);
}

void Context::api_touch(std::int64_t id) {  // store.cpp:139-141
  flush_pending();
  C(id);
  touch(id);
}

// TieredStore::pin (store.cpp:143-145): the pinned set is replaced
void Context::api_pin(const std::vector<std::int64_t>& ids) {
  flush_pending();
  for (std::int64_t id : pinned_ids_)
    if (clusters_[static_cast<std::size_t>(id)]) set_flag(id, CF_PINNED, false);
  pinned_ids_.clear();
  for (std::int64_t id : ids) {
    if (id < 0 || id >= static_cast<std::int64_t>(clusters_.size()) || !clusters_[static_cast<std::size_t>(id)]) continue;
    set_flag(id, CF_PINNED, true);
    pinned_ids_.push_back(id);
  }
  std::sort(pinned_ids_.begin(), pinned_ids_.end());
}

double Context::api_enforce_capacity() {
  flush_pending();
  return enforce_capacity();
}

// visual_topk (index.cpp:192-208) / semantic_topk (index.cpp:210-240) on the device: exact fp64
// cosines and the reference's tie-breaks through the flat top-k kernel over an explicit list.
std::vector<std::int64_t> Context::api_visual_topk(const float* q, int k) {
  flush_pending();
  if (k <= 0) fail(-10, "visual top-k must be positive");
  if (parts_.empty()) fail(-9, "visual_topk on an empty index");
  const int n = static_cast<int>(parts_.size());
  ensure_idx(static_cast<std::int64_t>(n) + d_, 1);
  KVC_CUDA(cudaMemcpyAsync(d_q_, q, d_ * 4, cudaMemcpyHostToDevice, st_));
  auto* gs = static_cast<std::uint8_t*>(dalloc_scratch(static_cast<std::size_t>(n) * 17 + 16));
  const int nl = launch_flat_topk(t_, d_q_, nullptr, nullptr, n, k, d_idx_, gs, st_);
  if (nl == 0) fail(-20, "visual top-k kernel could not be launched");
  launches_ += nl;
  KVC_CUDA(cudaGetLastError());
  const int take = std::min(n, k);
  std::vector<std::int32_t> order(static_cast<std::size_t>(take));
  KVC_CUDA(cudaMemcpyAsync(order.data(), d_idx_, take * 4, cudaMemcpyDeviceToHost, st_));
  sync();
  check_dev_err();
  return std::vector<std::int64_t>(order.begin(), order.end());
}

std::vector<std::pair<std::int64_t, int>> Context::api_semantic_topk(const float* q, int layer,
                                                                     const std::vector<std::int64_t>& part_ids, int k) {
  flush_pending();
  if (k <= 0) fail(-10, "semantic top-k must be positive");
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range: " + std::to_string(layer));
  // candidates: the partitions' clusters at this layer + their registered buffers (index.cpp:216-229)
  std::vector<std::int32_t> slots;
  std::vector<std::uint8_t> bufs;
  for (std::int64_t p : part_ids) {
    if (p < 0 || p >= static_cast<std::int64_t>(parts_.size())) fail(-8, "unknown partition id");
    for (std::int64_t id : parts_[static_cast<std::size_t>(p)].per_layer[static_cast<std::size_t>(layer)]) {
      slots.push_back(C(id).slot);
      bufs.push_back(0);
      if (is_lazy(id)) {
        slots.push_back(C(id).slot);
        bufs.push_back(1);
      }
    }
  }
  const int n = static_cast<int>(slots.size());
  std::vector<std::pair<std::int64_t, int>> out;
  if (n == 0) return out;
  ensure_idx(static_cast<std::int64_t>(n) * 2 + k + d_, 1);
  std::memcpy(h_idx_, slots.data(), n * 4);
  std::memcpy(reinterpret_cast<std::uint8_t*>(h_idx_ + n), bufs.data(), n);
  KVC_CUDA(cudaMemcpyAsync(d_idx_, h_idx_, static_cast<std::size_t>(n) * 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_q_, q, d_ * 4, cudaMemcpyHostToDevice, st_));
  std::int32_t* d_out = d_idx_ + 2 * n;
  auto* gs = static_cast<std::uint8_t*>(dalloc_scratch(static_cast<std::size_t>(n) * 17 + 16));
  const int nl = launch_flat_topk(t_, d_q_, d_idx_, reinterpret_cast<std::uint8_t*>(d_idx_ + n), n, k, d_out, gs, st_);
  if (nl == 0) fail(-20, "semantic top-k kernel could not be launched");
  launches_ += nl;
  KVC_CUDA(cudaGetLastError());
  const int take = std::min(n, k);
  std::vector<std::int32_t> order(static_cast<std::size_t>(take));
  KVC_CUDA(cudaMemcpyAsync(order.data(), d_out, take * 4, cudaMemcpyDeviceToHost, st_));
  sync();
  check_dev_err();
  for (int i = 0; i < take; ++i) {
    const int j = order[static_cast<std::size_t>(i)];
    out.push_back({slot_id_[static_cast<std::size_t>(slots[static_cast<std::size_t>(j)])], bufs[static_cast<std::size_t>(j)]});
  }
  return out;
}

}  // namespace kvc
