// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// A C-ABI driver over the *unmodified* reference library (kvclust, compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/libkvclust_ref.so).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it.
//
// What it exposes:
//   * ref_stream_*   : gen_stream() (workload.cpp:56-187) output as flat float arrays.
//   * ref_drv_*      : a driver that follows StreamEngine's control flow
//                      (engine.cpp:67-174 ingest/build/cadence/repin, engine.cpp:176-237 query)
//                      through the public component API (HierIndex / TieredStore / Maintainer /
//                      retrieve), so the per-insert routed cluster id (maintainer.cpp:88-176) and
//                      the full RetrievalResult (retrieval.hpp:49-71) are observable. Its fidelity
//                      to StreamEngine is itself checked by comparing attended digests with
//                      ref_eng_* (the real StreamEngine) in tests/test_oracle.py.
//   * ref_eng_*      : the real StreamEngine / run_stream (engine.cpp:266-271).
//   * ref_prim_*     : reference primitives (vecmath.hpp, maintainer.cpp:11-25, rng.hpp:47-52,
//                      clustering.cpp:180-208) used to pin the C restatement (kvc_oracle.c).
//   * ref_time_*     : CPU-baseline timers.
//
// Errors: every entry point catches kvclust::Error and returns a negative code
// (see kvc.h's KVC_E_* values, which mirror error.hpp:9-82).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "kvclust/clustering.hpp"
#include "kvclust/engine.hpp"
#include "kvclust/error.hpp"
#include "kvclust/index.hpp"
#include "kvclust/maintainer.hpp"
#include "kvclust/retrieval.hpp"
#include "kvclust/rng.hpp"
#include "kvclust/store.hpp"
#include "kvclust/vecmath.hpp"
#include "kvclust/workload.hpp"

using namespace kvclust;

namespace {

thread_local std::string g_err;

// Same numbering as include/kvc.h (KVC_E_*).
int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const DegenerateVector*>(&e)) return -2;
  if (dynamic_cast<const DimMismatch*>(&e)) return -3;
  if (dynamic_cast<const EmptyInput*>(&e)) return -4;
  if (dynamic_cast<const EmptyCluster*>(&e)) return -5;
  if (dynamic_cast<const TooFewPoints*>(&e)) return -6;
  if (dynamic_cast<const BadLayer*>(&e)) return -7;
  if (dynamic_cast<const UnknownCluster*>(&e)) return -8;
  if (dynamic_cast<const EmptyIndex*>(&e)) return -9;
  if (dynamic_cast<const ConfigError*>(&e)) return -10;
  if (dynamic_cast<const InvariantViolation*>(&e)) return -11;
  return -1;
}

#define GUARD_BEGIN try {
#define GUARD_END                         \
  }                                       \
  catch (const std::exception& e) {       \
    return code_of(e);                    \
  }                                       \
  return 0;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- streams

struct ref_stream_cfg {
  int n_scenes, frames_per_scene, tokens_per_frame, d, L;
  double visual_noise, semantic_noise, drift_rate, cross_layer_eps;
  int n_queries;
  double cross_modal_mix;
  int gt_top_m, scene_cycle, queries_at_end;
  std::uint64_t seed;
};

void ref_stream_cfg_default(ref_stream_cfg* c) {
  StreamConfig s;
  c->n_scenes = s.n_scenes;
  c->frames_per_scene = s.frames_per_scene;
  c->tokens_per_frame = s.tokens_per_frame;
  c->d = s.d;
  c->L = s.L;
  c->visual_noise = s.visual_noise;
  c->semantic_noise = s.semantic_noise;
  c->drift_rate = s.drift_rate;
  c->cross_layer_eps = s.cross_layer_eps;
  c->n_queries = s.n_queries;
  c->cross_modal_mix = s.cross_modal_mix;
  c->gt_top_m = s.gt_top_m;
  c->scene_cycle = s.scene_cycle;
  c->queries_at_end = s.queries_at_end ? 1 : 0;
  c->seed = s.seed;
}

static StreamConfig to_stream_cfg(const ref_stream_cfg* c) {
  StreamConfig s;
  s.n_scenes = c->n_scenes;
  s.frames_per_scene = c->frames_per_scene;
  s.tokens_per_frame = c->tokens_per_frame;
  s.d = c->d;
  s.L = c->L;
  s.visual_noise = c->visual_noise;
  s.semantic_noise = c->semantic_noise;
  s.drift_rate = c->drift_rate;
  s.cross_layer_eps = c->cross_layer_eps;
  s.n_queries = c->n_queries;
  s.cross_modal_mix = c->cross_modal_mix;
  s.gt_top_m = c->gt_top_m;
  s.scene_cycle = c->scene_cycle;
  s.queries_at_end = c->queries_at_end != 0;
  s.seed = c->seed;
  return s;
}

struct RefStream {
  StreamConfig cfg;
  std::vector<StreamEvent> events;
};

int ref_stream_gen(const ref_stream_cfg* c, void** out) {
  GUARD_BEGIN
  auto* s = new RefStream;
  s->cfg = to_stream_cfg(c);
  s->events = gen_stream(s->cfg);
  *out = s;
  GUARD_END
}

void ref_stream_free(void* h) { delete static_cast<RefStream*>(h); }

int ref_stream_n_events(void* h) { return static_cast<int>(static_cast<RefStream*>(h)->events.size()); }

// kind: 0 frame, 1 query
int ref_stream_kind(void* h, int i) {
  return static_cast<RefStream*>(h)->events[static_cast<std::size_t>(i)].kind ==
                 StreamEvent::Kind::Frame
             ? 0
             : 1;
}

// visual[d]; keys/values[L][T][d]
int ref_stream_frame(void* h, int i, std::int64_t* frame_id, float* visual, float* keys,
                     float* values) {
  const auto& ev = static_cast<RefStream*>(h)->events[static_cast<std::size_t>(i)];
  if (ev.kind != StreamEvent::Kind::Frame) return -10;
  *frame_id = ev.frame.frame_id;
  std::memcpy(visual, ev.frame.visual.data(), ev.frame.visual.size() * sizeof(float));
  std::size_t off = 0;
  for (const auto& layer : ev.frame.layers)
    for (const KVEntry& e : layer) {
      std::memcpy(keys + off, e.key.data(), e.key.size() * sizeof(float));
      std::memcpy(values + off, e.value.data(), e.value.size() * sizeof(float));
      off += e.key.size();
    }
  return 0;
}

// q[L][d]; gt up to gt_cap entries; returns n_gt
int ref_stream_query(void* h, int i, std::int64_t* query_id, float* q, std::int64_t* gt,
                     int gt_cap) {
  const auto& ev = static_cast<RefStream*>(h)->events[static_cast<std::size_t>(i)];
  if (ev.kind != StreamEvent::Kind::Query) return -10;
  *query_id = ev.query.query_id;
  std::size_t off = 0;
  for (const Embedding& v : ev.query.q) {
    std::memcpy(q + off, v.data(), v.size() * sizeof(float));
    off += v.size();
  }
  int n = 0;
  for (std::int64_t f : ev.query.ground_truth_frames)
    if (n < gt_cap) gt[n++] = f;
  return static_cast<int>(ev.query.ground_truth_frames.size());
}

// ---------------------------------------------------------------- engine config

struct ref_engine_cfg {
  // RetrievalConfig (retrieval.hpp:20-32)
  int k_v, k_s, window_frames, prefetch_k, prefetch_enabled, token_mode;
  std::int64_t token_budget;
  double lookup_cost_per_candidate_us, compute_cost_per_token_us;
  // MaintainerConfig (maintainer.hpp:18-34)
  double tau_min, tau_max, n0;
  int defer_host_splits, max_split_depth;
  double visual_floor;
  // BuildConfig (index.hpp:76-82)
  int target_visual_cluster_size, target_semantic_cluster_size, kmeans_max_iters;
  double kmeans_tol;
  // CostModel (store.hpp:17-31)
  double alpha_us, beta_us_per_byte;
  std::int64_t bytes_per_entry, device_capacity_entries;
  // EngineConfig (engine.hpp:21-33)
  int build_batch_frames, batched_ingest;
  double ingest_overhead_us;
  int offload_horizon_frames;
  std::uint64_t seed;
};

void ref_engine_cfg_default(ref_engine_cfg* c) {
  EngineConfig e;
  c->k_v = e.retrieval.k_v;
  c->k_s = e.retrieval.k_s;
  c->window_frames = e.retrieval.window_frames;
  c->prefetch_k = e.retrieval.prefetch_k;
  c->prefetch_enabled = e.retrieval.prefetch_enabled ? 1 : 0;
  c->token_mode = e.retrieval.mode == RetrievalMode::TokenBaseline ? 1 : 0;
  c->token_budget = e.retrieval.token_budget;
  c->lookup_cost_per_candidate_us = e.retrieval.lookup_cost_per_candidate_us;
  c->compute_cost_per_token_us = e.retrieval.compute_cost_per_token_us;
  c->tau_min = e.maintainer.threshold.tau_min;
  c->tau_max = e.maintainer.threshold.tau_max;
  c->n0 = e.maintainer.threshold.n0;
  c->defer_host_splits = e.maintainer.defer_host_splits ? 1 : 0;
  c->max_split_depth = e.maintainer.max_split_depth;
  c->visual_floor = e.maintainer.visual_floor;
  c->target_visual_cluster_size = e.build.target_visual_cluster_size;
  c->target_semantic_cluster_size = e.build.target_semantic_cluster_size;
  c->kmeans_max_iters = e.build.kmeans_max_iters;
  c->kmeans_tol = e.build.kmeans_tol;
  c->alpha_us = e.cost.alpha_us;
  c->beta_us_per_byte = e.cost.beta_us_per_byte;
  c->bytes_per_entry = e.cost.bytes_per_entry;
  c->device_capacity_entries = e.cost.device_capacity_entries;
  c->build_batch_frames = e.build_batch_frames;
  c->batched_ingest = e.batched_ingest ? 1 : 0;
  c->ingest_overhead_us = e.ingest_overhead_us;
  c->offload_horizon_frames = e.offload_horizon_frames;
  c->seed = e.seed;
}

static EngineConfig to_engine_cfg(const ref_engine_cfg* c) {
  EngineConfig e;
  e.retrieval.k_v = c->k_v;
  e.retrieval.k_s = c->k_s;
  e.retrieval.window_frames = c->window_frames;
  e.retrieval.prefetch_k = c->prefetch_k;
  e.retrieval.prefetch_enabled = c->prefetch_enabled != 0;
  e.retrieval.mode = c->token_mode ? RetrievalMode::TokenBaseline : RetrievalMode::Cluster;
  e.retrieval.token_budget = c->token_budget;
  e.retrieval.lookup_cost_per_candidate_us = c->lookup_cost_per_candidate_us;
  e.retrieval.compute_cost_per_token_us = c->compute_cost_per_token_us;
  e.maintainer.threshold.tau_min = c->tau_min;
  e.maintainer.threshold.tau_max = c->tau_max;
  e.maintainer.threshold.n0 = c->n0;
  e.maintainer.defer_host_splits = c->defer_host_splits != 0;
  e.maintainer.max_split_depth = c->max_split_depth;
  e.maintainer.visual_floor = c->visual_floor;
  e.build.target_visual_cluster_size = c->target_visual_cluster_size;
  e.build.target_semantic_cluster_size = c->target_semantic_cluster_size;
  e.build.kmeans_max_iters = c->kmeans_max_iters;
  e.build.kmeans_tol = c->kmeans_tol;
  e.cost.alpha_us = c->alpha_us;
  e.cost.beta_us_per_byte = c->beta_us_per_byte;
  e.cost.bytes_per_entry = c->bytes_per_entry;
  e.cost.device_capacity_entries = c->device_capacity_entries;
  e.build_batch_frames = c->build_batch_frames;
  e.batched_ingest = c->batched_ingest != 0;
  e.ingest_overhead_us = c->ingest_overhead_us;
  e.offload_horizon_frames = c->offload_horizon_frames;
  e.seed = c->seed;
  return e;
}

static FrameInput make_frame(int d, int L, int T, std::int64_t frame_id, const float* visual,
                             const float* keys, const float* values) {
  FrameInput f;
  f.frame_id = frame_id;
  f.visual.assign(visual, visual + d);
  f.layers.resize(static_cast<std::size_t>(L));
  for (int l = 0; l < L; ++l)
    for (int t = 0; t < T; ++t) {
      KVEntry e;
      std::size_t off = (static_cast<std::size_t>(l) * T + t) * static_cast<std::size_t>(d);
      e.key.assign(keys + off, keys + off + d);
      e.value.assign(values + off, values + off + d);
      e.frame_id = frame_id;
      e.layer_id = l;
      e.token_id = t;
      f.layers[static_cast<std::size_t>(l)].push_back(std::move(e));
    }
  return f;
}

static QueryBundle make_query(int d, int L, std::int64_t qid, const float* q, const std::int64_t* gt,
                              int n_gt) {
  QueryBundle b;
  b.query_id = qid;
  for (int l = 0; l < L; ++l) b.q.emplace_back(q + static_cast<std::size_t>(l) * d, q + static_cast<std::size_t>(l + 1) * d);
  for (int i = 0; i < n_gt; ++i) b.ground_truth_frames.push_back(gt[i]);
  return b;
}

// ---------------------------------------------------------------- driver

// Follows StreamEngine (engine.cpp) step for step in cluster mode, but keeps the
// per-insert routing result and the last RetrievalResult observable.
struct Driver {
  EngineConfig cfg;
  int d, L;
  bool built = false;
  std::vector<FrameInput> pending;
  std::optional<HierIndex> index;
  std::optional<TieredStore> store;
  std::optional<Maintainer> maint;
  std::deque<FrameInput> window;
  std::int64_t last_partition = -1;
  bool check = true;  // run check_invariants / audit like engine.cpp:91-92,234-236

  // token-baseline mode (engine.cpp:153-158, 179-203)
  std::vector<std::vector<KVEntry>> pools;
  TransferLedger baseline_ledger;

  std::vector<std::int64_t> last_assign;  // [L*T] routed cluster ids of the last frame
  std::int64_t last_pid = -1;
  RetrievalResult last_rr;

  void repin() {  // engine.cpp:67-75
    if (!store) return;
    std::set<std::int64_t> pins;
    for (const FrameInput& f : window) {
      auto o = index->clusters_of_frame(f.frame_id);
      pins.insert(o.begin(), o.end());
    }
    store->pin(pins);
  }

  void push_window(const FrameInput& f) {  // engine.cpp:54-57
    window.push_back(f);
    while (static_cast<int>(window.size()) > cfg.retrieval.window_frames) window.pop_front();
  }

  std::vector<KVEntry> window_entries() const {  // engine.cpp:59-65
    std::vector<KVEntry> out;
    for (const FrameInput& f : window)
      for (const auto& layer : f.layers)
        for (const KVEntry& e : layer) out.push_back(e);
    return out;
  }

  std::set<std::int64_t> window_owners() const {
    std::set<std::int64_t> owners;
    for (const FrameInput& f : window) {
      auto o = index->clusters_of_frame(f.frame_id);
      owners.insert(o.begin(), o.end());
    }
    return owners;
  }

  void apply_cadence(std::int64_t frame_id, std::int64_t pid) {  // engine.cpp:95-132
    if (last_partition >= 0 && pid >= 0 && pid != last_partition) {
      const VisualPartition& closed = index->partition(last_partition);
      std::vector<std::int64_t> ids;
      for (const auto& [layer, list] : closed.per_layer_clusters) ids.insert(ids.end(), list.begin(), list.end());
      for (std::int64_t cid : ids) {
        const ClusterRecord& rec = index->cluster(cid);
        if (rec.residence == Residence::Device && !rec.lazy_split) {
          auto owners = window_owners();
          if (!owners.count(cid)) store->offload(cid);
        }
      }
    }
    if (pid >= 0) last_partition = pid;
    std::vector<std::int64_t> stale;
    for (const auto& [cid, rec] : index->clusters())
      if (rec.residence == Residence::Device && !rec.lazy_split &&
          rec.last_touch_frame + cfg.offload_horizon_frames < frame_id)
        stale.push_back(cid);
    if (!stale.empty()) {
      auto owners = window_owners();
      for (std::int64_t cid : stale)
        if (!owners.count(cid)) store->offload(cid);
    }
    store->enforce_capacity();
  }

  void build_now() {  // engine.cpp:77-93
    if (pending.empty()) throw EmptyIndex("no frames available to build from");
    BuildConfig b = cfg.build;
    b.seed = mix_seed(cfg.seed, 1);
    index.emplace(build_index(pending, b));
    store.emplace(*index, cfg.cost);
    MaintainerConfig m = cfg.maintainer;
    m.seed = mix_seed(cfg.seed, 2);
    maint.emplace(*index, *store, m);
    built = true;
    std::int64_t last = pending.back().frame_id;
    pending.clear();
    repin();
    apply_cadence(last, -1);
    if (check) {
      index->check_invariants();
      store->audit();
    }
  }

  void frame(FrameInput&& f) {  // engine.cpp:134-174 (cluster mode)
    last_assign.assign(static_cast<std::size_t>(L) * f.layers[0].size(), -1);
    last_pid = -1;
    if (cfg.retrieval.mode == RetrievalMode::TokenBaseline) {  // engine.cpp:153-158
      pools.resize(static_cast<std::size_t>(L));
      for (std::size_t l = 0; l < f.layers.size(); ++l)
        for (const KVEntry& e : f.layers[l]) pools[l].push_back(e);
      push_window(f);
      return;
    }
    if (!built) {
      pending.push_back(f);
      push_window(f);
      if (static_cast<int>(pending.size()) >= cfg.build_batch_frames) build_now();
      return;
    }
    std::int64_t pid = maint->place_frame(f.frame_id, f.visual);
    last_pid = pid;
    std::size_t i = 0;
    for (const auto& layer : f.layers)
      for (const KVEntry& e : layer) last_assign[i++] = maint->on_insert(pid, e);
    std::int64_t fid = f.frame_id;
    push_window(f);
    repin();
    apply_cadence(fid, pid);
  }

  void query(const QueryBundle& b) {  // engine.cpp:176-237 (cluster mode)
    if (cfg.retrieval.mode == RetrievalMode::TokenBaseline) {  // engine.cpp:179-203
      std::set<std::int64_t> window_frames;
      for (const FrameInput& f : window) window_frames.insert(f.frame_id);
      pools.resize(static_cast<std::size_t>(L));
      last_rr = retrieve_token_baseline(b, cfg.retrieval, pools, window_frames, cfg.cost, baseline_ledger);
      return;
    }
    if (!built) build_now();
    last_rr = retrieve(b, cfg.retrieval, *index, *store, *maint, window_entries());
    repin();
    if (check) {
      index->check_invariants();
      store->audit();
    }
  }
};

int ref_drv_create(const ref_engine_cfg* c, int d, int L, void** out) {
  GUARD_BEGIN
  auto* drv = new Driver;
  drv->cfg = to_engine_cfg(c);
  drv->cfg.validate();
  drv->d = d;
  drv->L = L;
  *out = drv;
  GUARD_END
}

void ref_drv_free(void* h) { delete static_cast<Driver*>(h); }

void ref_drv_set_checks(void* h, int on) { static_cast<Driver*>(h)->check = on != 0; }

// assigned[L*T] <- routed cluster id per (layer, token); -1 while frames are pending the build.
int ref_drv_frame(void* h, std::int64_t frame_id, const float* visual, const float* keys,
                  const float* values, int T, std::int64_t* assigned, std::int64_t* pid) {
  GUARD_BEGIN
  auto* drv = static_cast<Driver*>(h);
  drv->frame(make_frame(drv->d, drv->L, T, frame_id, visual, keys, values));
  if (assigned)
    std::memcpy(assigned, drv->last_assign.data(), drv->last_assign.size() * sizeof(std::int64_t));
  if (pid) *pid = drv->last_pid;
  GUARD_END
}

int ref_drv_build_now(void* h) {
  GUARD_BEGIN
  auto* drv = static_cast<Driver*>(h);
  if (!drv->built) drv->build_now();
  GUARD_END
}

int ref_drv_query(void* h, std::int64_t qid, const float* q, const std::int64_t* gt, int n_gt) {
  GUARD_BEGIN
  auto* drv = static_cast<Driver*>(h);
  drv->query(make_query(drv->d, drv->L, qid, q, gt, n_gt));
  GUARD_END
}

// Per-layer views of the last RetrievalResult. Each returns the element count and copies
// at most cap elements.
int ref_drv_q_ranked(void* h, int l, std::int64_t* ids, std::int32_t* is_buffer, int cap) {
  const auto& lr = static_cast<Driver*>(h)->last_rr.layers[static_cast<std::size_t>(l)];
  int n = 0;
  for (const CandidateRef& r : lr.ranked) {
    if (n < cap) {
      ids[n] = r.cluster_id;
      is_buffer[n] = r.is_buffer ? 1 : 0;
    }
    ++n;
  }
  return n;
}

int ref_drv_q_selected(void* h, int l, std::int64_t* ids, int cap) {
  const auto& lr = static_cast<Driver*>(h)->last_rr.layers[static_cast<std::size_t>(l)];
  int n = 0;
  for (std::int64_t id : lr.selected) {
    if (n < cap) ids[n] = id;
    ++n;
  }
  return n;
}

int ref_drv_q_attended(void* h, int l, std::int64_t* frames, std::int32_t* tokens, int cap) {
  const auto& lr = static_cast<Driver*>(h)->last_rr.layers[static_cast<std::size_t>(l)];
  int n = 0;
  for (const auto& [f, t] : lr.attended_tokens) {
    if (n < cap) {
      frames[n] = f;
      tokens[n] = t;
    }
    ++n;
  }
  return n;
}

// lat[5] = lookup, transfer, stall, completion, compute (retrieval.hpp:39-47);
// ints[4] = verified_clusters, prefetch_hits, rep_count, n_predicted
void ref_drv_q_layer_meta(void* h, int l, double* lat, std::int64_t* ints) {
  const auto& lr = static_cast<Driver*>(h)->last_rr.layers[static_cast<std::size_t>(l)];
  lat[0] = lr.latency.lookup_us;
  lat[1] = lr.latency.transfer_us;
  lat[2] = lr.latency.stall_us;
  lat[3] = lr.latency.completion_us;
  lat[4] = lr.latency.compute_us;
  ints[0] = lr.verified_clusters;
  ints[1] = lr.prefetch_hits;
  ints[2] = lr.rep_count;
  ints[3] = static_cast<std::int64_t>(lr.predicted.size());
}

// d[2] = ttft_us, recall
void ref_drv_q_meta(void* h, double* dd) {
  const auto& rr = static_cast<Driver*>(h)->last_rr;
  dd[0] = rr.ttft_us;
  dd[1] = rr.recall;
}

// FNV-1a attended digest of the last query (engine.cpp:18-35)
std::uint64_t ref_drv_q_digest(void* h) {
  const auto& r = static_cast<Driver*>(h)->last_rr;
  auto fnv = [](std::uint64_t hh, std::uint64_t x) {
    for (int i = 0; i < 8; ++i) {
      hh ^= (x >> (8 * i)) & 0xffu;
      hh *= 1099511628211ull;
    }
    return hh;
  };
  std::uint64_t hh = 1469598103934665603ull;
  for (std::size_t l = 0; l < r.layers.size(); ++l)
    for (const auto& [frame, token] : r.layers[l].attended_tokens) {
      hh = fnv(hh, l);
      hh = fnv(hh, static_cast<std::uint64_t>(frame));
      hh = fnv(hh, static_cast<std::uint64_t>(token));
    }
  return hh;
}

// MaintainerStats (maintainer.hpp:36-46) -> out[9]
void ref_drv_maint_stats(void* h, std::int64_t* o) {
  auto* drv = static_cast<Driver*>(h);
  MaintainerStats s = drv->maint ? drv->maint->stats() : MaintainerStats{};
  o[0] = s.inserts;
  o[1] = s.absorbed;
  o[2] = s.immediate_splits;
  o[3] = s.deferred_marks;
  o[4] = s.settled_splits;
  o[5] = s.split_ops_total;
  o[6] = s.host_over_threshold;
  o[7] = s.maintenance_fetches;
  o[8] = s.partitions_opened;
}

// Ledger totals per cause (retrieval, maintenance, prefetch, completion, offload):
// ops[5], bytes[5], cost[5]; returns device_entries
std::int64_t ref_drv_ledger(void* h, std::int64_t* ops, std::int64_t* bytes, double* cost) {
  auto* drv = static_cast<Driver*>(h);
  const bool tok = drv->cfg.retrieval.mode == RetrievalMode::TokenBaseline;
  if (!drv->store && !tok) return 0;
  const TransferLedger& lg = tok ? drv->baseline_ledger : drv->store->ledger();
  const TransferCause causes[5] = {TransferCause::Retrieval, TransferCause::Maintenance,
                                   TransferCause::Prefetch, TransferCause::Completion,
                                   TransferCause::Offload};
  for (int i = 0; i < 5; ++i) {
    CauseTotals t = lg.cause(causes[i]);
    ops[i] = t.n_ops;
    bytes[i] = t.bytes;
    cost[i] = t.cost_us;
  }
  return tok ? 0 : drv->store->device_entries();
}

int ref_drv_ledger_log_size(void* h) {
  auto* drv = static_cast<Driver*>(h);
  return drv->store ? static_cast<int>(drv->store->ledger().log().size()) : 0;
}

// op i: ints[4] = cause, to_device, cluster_id, bytes
void ref_drv_ledger_op(void* h, int i, std::int64_t* ints) {
  const TransferOp& op = static_cast<Driver*>(h)->store->ledger().log()[static_cast<std::size_t>(i)];
  ints[0] = static_cast<std::int64_t>(op.cause);
  ints[1] = op.to_device ? 1 : 0;
  ints[2] = op.cluster_id;
  ints[3] = op.bytes;
}

int ref_drv_n_partitions(void* h) {
  auto* drv = static_cast<Driver*>(h);
  return drv->index ? static_cast<int>(drv->index->partitions().size()) : 0;
}

// visual_rep[d], frames up to cap; returns frame count
int ref_drv_partition(void* h, int p, double* visual_rep, std::int64_t* frames, int cap) {
  const VisualPartition& vp = static_cast<Driver*>(h)->index->partition(p);
  std::memcpy(visual_rep, vp.visual_rep.data(), vp.visual_rep.size() * sizeof(double));
  int n = 0;
  for (std::int64_t f : vp.frame_ids) {
    if (n < cap) frames[n] = f;
    ++n;
  }
  return n;
}

int ref_drv_n_clusters(void* h) {
  auto* drv = static_cast<Driver*>(h);
  return drv->index ? static_cast<int>(drv->index->clusters().size()) : 0;
}

int ref_drv_cluster_ids(void* h, std::int64_t* ids, int cap) {
  int n = 0;
  for (const auto& [id, rec] : static_cast<Driver*>(h)->index->clusters()) {
    if (n < cap) ids[n] = id;
    ++n;
  }
  return n;
}

// info[10] = layer, parent, n_members, n_buffer, stat_count, lazy, residence(0 dev,1 host),
//            device_tail, first_frame, last_touch ; dd[1] = variance; rep[d]; buffer_rep[d]
int ref_drv_cluster(void* h, std::int64_t id, std::int64_t* info, double* var, double* rep,
                    double* buffer_rep) {
  GUARD_BEGIN
  const ClusterRecord& r = static_cast<Driver*>(h)->index->cluster(id);
  info[0] = r.layer_id;
  info[1] = r.visual_parent;
  info[2] = r.n();
  info[3] = static_cast<std::int64_t>(r.buffer.size());
  info[4] = r.stat_count;
  info[5] = r.lazy_split ? 1 : 0;
  info[6] = r.residence == Residence::Device ? 0 : 1;
  info[7] = r.device_tail;
  info[8] = r.first_frame_id;
  info[9] = r.last_touch_frame;
  *var = r.variance;
  if (rep) std::memcpy(rep, r.rep.data(), r.rep.size() * sizeof(double));
  if (buffer_rep && !r.buffer_rep.empty())
    std::memcpy(buffer_rep, r.buffer_rep.data(), r.buffer_rep.size() * sizeof(double));
  GUARD_END
}

// members (which=0) or buffer (which=1) as (frame, token) in stored order; returns count
int ref_drv_cluster_entries(void* h, std::int64_t id, int which, std::int64_t* frames,
                            std::int32_t* tokens, int cap) {
  const ClusterRecord& r = static_cast<Driver*>(h)->index->cluster(id);
  const auto& v = which == 0 ? r.members : r.buffer;
  int n = 0;
  for (const KVEntry& e : v) {
    if (n < cap) {
      frames[n] = e.frame_id;
      tokens[n] = e.token_id;
    }
    ++n;
  }
  return n;
}

// per_layer_clusters[layer] of partition p, in stored order; returns count
int ref_drv_partition_layer(void* h, int p, int layer, std::int64_t* ids, int cap) {
  const VisualPartition& vp = static_cast<Driver*>(h)->index->partition(p);
  auto it = vp.per_layer_clusters.find(layer);
  if (it == vp.per_layer_clusters.end()) return 0;
  int n = 0;
  for (std::int64_t id : it->second) {
    if (n < cap) ids[n] = id;
    ++n;
  }
  return n;
}

// oracle_flat_topk (retrieval.cpp:145-164) against the driver's current index.
int ref_drv_flat_topk(void* h, const float* q, int layer, int k, std::int64_t* ids,
                      std::int32_t* is_buffer) {
  auto* drv = static_cast<Driver*>(h);
  try {
    Embedding qq(q, q + drv->d);
    auto refs = oracle_flat_topk(*drv->index, qq, layer, k);
    for (std::size_t i = 0; i < refs.size(); ++i) {
      ids[i] = refs[i].cluster_id;
      is_buffer[i] = refs[i].is_buffer ? 1 : 0;
    }
    return static_cast<int>(refs.size());
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// ---------------------------------------------------------------- real StreamEngine

struct Eng {
  std::unique_ptr<StreamEngine> eng;
  int d, L;
  RunOutput out;
};

int ref_eng_create(const ref_engine_cfg* c, int d, int L, void** o) {
  GUARD_BEGIN
  auto* e = new Eng;
  e->eng = std::make_unique<StreamEngine>(to_engine_cfg(c), d, L);
  e->d = d;
  e->L = L;
  *o = e;
  GUARD_END
}

void ref_eng_free(void* h) { delete static_cast<Eng*>(h); }

int ref_eng_frame(void* h, std::int64_t frame_id, const float* visual, const float* keys,
                  const float* values, int T) {
  GUARD_BEGIN
  auto* e = static_cast<Eng*>(h);
  StreamEvent ev;
  ev.kind = StreamEvent::Kind::Frame;
  ev.frame = make_frame(e->d, e->L, T, frame_id, visual, keys, values);
  e->eng->process(ev);
  GUARD_END
}

int ref_eng_query(void* h, std::int64_t qid, const float* q, const std::int64_t* gt, int n_gt) {
  GUARD_BEGIN
  auto* e = static_cast<Eng*>(h);
  StreamEvent ev;
  ev.kind = StreamEvent::Kind::Query;
  ev.query = make_query(e->d, e->L, qid, q, gt, n_gt);
  e->eng->process(ev);
  GUARD_END
}

int ref_eng_finish(void* h) {
  GUARD_BEGIN
  auto* e = static_cast<Eng*>(h);
  e->out = e->eng->finish();
  GUARD_END
}

int ref_eng_n_rows(void* h) { return static_cast<int>(static_cast<Eng*>(h)->out.rows.size()); }

// row i: digest, ops, bytes, realized_frames, context_frames ; dd[2] = ttft_us, recall
std::uint64_t ref_eng_row(void* h, int i, std::int64_t* ints, double* dd) {
  const QueryRow& r = static_cast<Eng*>(h)->out.rows[static_cast<std::size_t>(i)];
  ints[0] = r.ops;
  ints[1] = r.bytes;
  ints[2] = r.realized_frames;
  ints[3] = r.context_frames;
  dd[0] = r.ttft_us;
  dd[1] = r.recall;
  return r.attended_digest;
}

void ref_eng_maint_stats(void* h, std::int64_t* o) {
  const MaintainerStats& s = static_cast<Eng*>(h)->out.maintainer;
  o[0] = s.inserts;
  o[1] = s.absorbed;
  o[2] = s.immediate_splits;
  o[3] = s.deferred_marks;
  o[4] = s.settled_splits;
  o[5] = s.split_ops_total;
  o[6] = s.host_over_threshold;
  o[7] = s.maintenance_fetches;
  o[8] = s.partitions_opened;
}

// ---------------------------------------------------------------- primitives

double ref_prim_cosine_fd(const float* a, const double* b, int d) {
  Embedding x(a, a + d);
  DVec y(b, b + d);
  try {
    return cosine_sim(x, y);
  } catch (const std::exception& e) {
    return static_cast<double>(code_of(e)) * 10.0;  // <= -20: an error marker, never a cosine
  }
}

double ref_prim_cosine_ff(const float* a, const float* b, int d) {
  Embedding x(a, a + d), y(b, b + d);
  try {
    return cosine_sim(x, y);
  } catch (const std::exception& e) {
    return static_cast<double>(code_of(e)) * 10.0;
  }
}

double ref_prim_dot_fd(const float* a, const double* b, int d) {
  Embedding x(a, a + d);
  DVec y(b, b + d);
  return dot(x, y);
}

double ref_prim_norm_d(const double* a, int d) { return norm(DVec(a, a + d)); }

double ref_prim_tau(std::int64_t n, double tau_min, double tau_max, double n0) {
  return tau(n, ThresholdConfig{tau_min, tau_max, n0});
}

void ref_prim_updated_stats(const double* rep, double var, std::int64_t n, const float* key, int d,
                            double* rep_out, double* var_out) {
  StatUpdate up = updated_stats(DVec(rep, rep + d), var, n, Embedding(key, key + d));
  std::memcpy(rep_out, up.rep.data(), static_cast<std::size_t>(d) * sizeof(double));
  *var_out = up.variance;
}

std::uint64_t ref_prim_mix_seed(std::uint64_t a, std::uint64_t b) { return mix_seed(a, b); }

// first n outputs of Rng(seed): u64[n], uniform[n], gaussian[n] (separate generators)
void ref_prim_rng(std::uint64_t seed, int n, std::uint64_t* u64, double* uni, double* gau) {
  Rng a(seed), b(seed), c(seed);
  for (int i = 0; i < n; ++i) {
    u64[i] = a.u64();
    uni[i] = b.uniform();
    gau[i] = c.gaussian();
  }
}

// split_two (clustering.cpp:180-208): points[n][d]; assignments[n]; returns degenerate flag
int ref_prim_split_two(const float* pts, int n, int d, std::uint64_t seed, std::int32_t* assign) {
  std::vector<Embedding> p;
  for (int i = 0; i < n; ++i) p.emplace_back(pts + static_cast<std::size_t>(i) * d, pts + static_cast<std::size_t>(i + 1) * d);
  try {
    KMeansResult r = split_two(p, seed);
    for (int i = 0; i < n; ++i) assign[i] = r.assignments[static_cast<std::size_t>(i)];
    return r.degenerate ? 1 : 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// spherical_kmeans (clustering.cpp:80-178); returns k_live; objective out
int ref_prim_kmeans(const float* pts, int n, int d, int k, int max_iters, double tol,
                    std::uint64_t seed, std::int32_t* assign, double* objective, int* iters) {
  std::vector<Embedding> p;
  for (int i = 0; i < n; ++i) p.emplace_back(pts + static_cast<std::size_t>(i) * d, pts + static_cast<std::size_t>(i + 1) * d);
  try {
    KMeansConfig cfg;
    cfg.k = k;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.seed = seed;
    KMeansResult r = spherical_kmeans(p, cfg);
    for (int i = 0; i < n; ++i) assign[i] = r.assignments[static_cast<std::size_t>(i)];
    *objective = r.objective;
    *iters = r.iterations_run;
    return static_cast<int>(r.centroids.size());
  } catch (const std::exception& e) {
    return code_of(e);
  }
}


// Installs one partition's pre-clustered state through the public HierIndex API, the way
// kvc_bulk_load documents it (include/kvc.h): add_partition (index.cpp:59-69) for the
// visual, the partition's frame list set to the members' distinct frames (the product records
// every loaded frame with visual_stat_count = #frames), then per layer, per cluster index
// ascending, add_cluster (index.cpp:97-120) with the exact Eq. 1/2 statistics
// (compute_representative / compute_variance, index.cpp:345-362). Members keep row order.
// keys/values [L][N][d]; assign [L][N]; frame_ids / token_ids [N] (NULL: i / 196, i % 196).
static std::int64_t install_clusters(HierIndex& index, int d, int L, int N, int C, const float* keys,
                                     const float* values, const std::int32_t* assign, const float* visual,
                                     const std::int64_t* frame_ids, const std::int32_t* token_ids,
                                     bool full_partition) {
  Embedding vis(static_cast<std::size_t>(d), 0.0f);
  if (visual) vis.assign(visual, visual + d); else vis[0] = 1.0f;
  auto fid = [&](int i) -> std::int64_t { return frame_ids ? frame_ids[i] : i / 196; };
  auto tid = [&](int i) -> std::int32_t { return token_ids ? token_ids[i] : i % 196; };
  std::vector<std::int64_t> fr;
  for (int i = 0; i < N; ++i) fr.push_back(fid(i));
  std::sort(fr.begin(), fr.end());
  fr.erase(std::unique(fr.begin(), fr.end()), fr.end());
  const std::int64_t pid = index.add_partition(fr.empty() ? 0 : fr.front(), vis);
  if (full_partition) {
    VisualPartition& p = index.partition(pid);
    p.frame_ids = fr;
    p.visual_stat_count = static_cast<std::int64_t>(fr.size());
  }
  for (int l = 0; l < L; ++l) {
    std::vector<std::vector<KVEntry>> groups(static_cast<std::size_t>(C));
    for (int i = 0; i < N; ++i) {
      KVEntry e;
      std::size_t off = (static_cast<std::size_t>(l) * N + i) * d;
      e.key.assign(keys + off, keys + off + d);
      e.value.assign(values + off, values + off + d);
      e.frame_id = fid(i);
      e.layer_id = l;
      e.token_id = tid(i);
      const std::int32_t a = assign[static_cast<std::size_t>(l) * N + i];
      if (a < 0 || a >= C) throw ConfigError("cluster index out of range");
      groups[static_cast<std::size_t>(a)].push_back(std::move(e));
    }
    for (auto& g : groups) {
      if (g.empty()) continue;
      ClusterRecord rec;
      rec.layer_id = l;
      rec.visual_parent = pid;
      rec.rep = compute_representative(g);
      rec.variance = compute_variance(g, rec.rep);
      rec.stat_count = static_cast<std::int64_t>(g.size());
      rec.members = std::move(g);
      index.add_cluster(std::move(rec));
    }
  }
  return pid;
}

// Bulk construction on the driver (the checker side of kvc_bulk_load): the index is built by
// install_clusters, then the store adopts every cluster in id order (store.cpp:67-74) and the
// maintainer is created with the engine's seed (engine.cpp:84), as after StreamEngine's build.
int ref_drv_bulk_load(void* h, const float* visual, const float* keys, const float* values, int N, int C,
                      const std::int32_t* assign, const std::int64_t* frame_ids, const std::int32_t* token_ids,
                      std::int64_t* partition) {
  GUARD_BEGIN
  auto* drv = static_cast<Driver*>(h);
  if (drv->built || !drv->pending.empty()) throw ConfigError("bulk load needs a fresh driver");
  drv->index.emplace(drv->d, drv->L);
  *partition = install_clusters(*drv->index, drv->d, drv->L, N, C, keys, values, assign, visual, frame_ids,
                                token_ids, true);
  drv->store.emplace(*drv->index, drv->cfg.cost);
  MaintainerConfig m = drv->cfg.maintainer;
  m.seed = mix_seed(drv->cfg.seed, 2);
  drv->maint.emplace(*drv->index, *drv->store, m);
  drv->built = true;
  GUARD_END
}

// ---------------------------------------------------------------- CPU baseline timers

// Builds a reference HierIndex directly from a synthetic clustered state (one partition,
// L layers, C clusters/layer, members given as keys/values [L][N][d] with assignment
// [L][N]); then times `steps` retrieve() calls (retrieval.cpp:45-143) plus the fp64
// attention restatement over each layer's attended set. Returns microseconds per step
// for retrieve (t[0]) and attention (t[1]).
int ref_time_decode(int d, int L, int N, int C, const float* keys, const float* values,
                    const std::int32_t* assign, const float* queries /*[steps][L][d]*/,
                    int steps, int k_s, int window_tokens, double* t) {
  GUARD_BEGIN
  HierIndex index(d, L);
  install_clusters(index, d, L, N, C, keys, values, assign, nullptr, nullptr, nullptr, false);
  const int T = 196;
  CostModel cost;
  cost.device_capacity_entries = static_cast<std::int64_t>(L) * N + 1;
  TieredStore store(index, cost);
  MaintainerConfig mc;
  Maintainer maint(index, store, mc);
  RetrievalConfig rc;
  rc.k_v = 1;
  rc.k_s = k_s;
  // window: the last window_tokens tokens of every layer
  std::vector<KVEntry> window;
  for (int l = 0; l < L; ++l)
    for (int i = N - window_tokens; i < N; ++i) {
      KVEntry e;
      std::size_t off = (static_cast<std::size_t>(l) * N + i) * d;
      e.key.assign(keys + off, keys + off + d);
      e.value.assign(values + off, values + off + d);
      e.frame_id = i / T;
      e.layer_id = l;
      e.token_id = i % T;
      window.push_back(std::move(e));
    }
  double t_ret = 0.0, t_att = 0.0;
  double sink = 0.0;
  for (int s = 0; s < steps; ++s) {
    QueryBundle b;
    for (int l = 0; l < L; ++l) {
      const float* q = queries + (static_cast<std::size_t>(s) * L + l) * d;
      b.q.emplace_back(q, q + d);
    }
    auto t0 = std::chrono::steady_clock::now();
    RetrievalResult r = retrieve(b, rc, index, store, maint, window);
    auto t1 = std::chrono::steady_clock::now();
    // fp64 attention restatement over the attended set
    for (int l = 0; l < L; ++l) {
      const auto& att = r.layers[static_cast<std::size_t>(l)].attended_tokens;
      const float* q = queries + (static_cast<std::size_t>(s) * L + l) * d;
      std::vector<double> sc(att.size());
      double mx = -1e300;
      const double scale = 1.0 / std::sqrt(static_cast<double>(d));
      for (std::size_t j = 0; j < att.size(); ++j) {
        std::size_t i = static_cast<std::size_t>(att[j].first) * T + static_cast<std::size_t>(att[j].second);
        const float* k = keys + (static_cast<std::size_t>(l) * N + i) * d;
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += static_cast<double>(q[c]) * k[c];
        sc[j] = acc * scale;
        mx = std::max(mx, sc[j]);
      }
      std::vector<double> o(static_cast<std::size_t>(d), 0.0);
      double den = 0.0;
      for (std::size_t j = 0; j < att.size(); ++j) {
        std::size_t i = static_cast<std::size_t>(att[j].first) * T + static_cast<std::size_t>(att[j].second);
        const float* v = values + (static_cast<std::size_t>(l) * N + i) * d;
        double w = std::exp(sc[j] - mx);
        den += w;
        for (int c = 0; c < d; ++c) o[static_cast<std::size_t>(c)] += w * v[c];
      }
      sink += o[0] / den;
    }
    auto t2 = std::chrono::steady_clock::now();
    t_ret += std::chrono::duration<double, std::micro>(t1 - t0).count();
    t_att += std::chrono::duration<double, std::micro>(t2 - t1).count();
  }
  t[0] = t_ret / steps;
  t[1] = t_att / steps;
  t[2] = sink;
  GUARD_END
}

// Multi-threaded CPU baseline: `threads` independent reference instances,
// each over the same `L`-domain sample (state built with add_cluster as in ref_time_decode),
// run concurrently. mode 0: `steps` retrieve() + fp64 attention per instance (queries
// [steps][L][d]); mode 1: place_frame + on_insert for `steps` frames per instance (frames:
// visual [steps][d], keys/values [steps][L][T][d]). out[0] = wall microseconds per step
// (max over threads), out[1] = mean per-thread microseconds per step.
int ref_time_mt(int mode, int threads, int d, int L, int N, int C, const float* keys,
                const float* values, const std::int32_t* assign, const float* queries, int warmup,
                int steps, int k_s, int window_tokens, const float* fvis, const float* fkeys,
                const float* fvals, int T, double* out) {
  GUARD_BEGIN
  std::vector<double> per(static_cast<std::size_t>(threads), 0.0);
  std::vector<std::string> errs(static_cast<std::size_t>(threads));
  auto worker = [&](int ti) {
    try {
      HierIndex index(d, L);
      install_clusters(index, d, L, N, C, keys, values, assign, fvis, nullptr, nullptr, false);
      const int TT = 196;
      CostModel cost;
      cost.device_capacity_entries = static_cast<std::int64_t>(L) * (N + (warmup + steps) * T + 1) + 1;
      TieredStore store(index, cost);
      MaintainerConfig mc;
      Maintainer maint(index, store, mc);
      RetrievalConfig rc;
      rc.k_v = 1;
      rc.k_s = k_s;
      std::vector<KVEntry> window;
      for (int l = 0; l < L; ++l)
        for (int i = N - window_tokens; i < N; ++i) {
          KVEntry e;
          std::size_t off = (static_cast<std::size_t>(l) * N + i) * d;
          e.key.assign(keys + off, keys + off + d);
          e.value.assign(values + off, values + off + d);
          e.frame_id = i / TT;
          e.layer_id = l;
          e.token_id = i % TT;
          window.push_back(std::move(e));
        }
      double sink = 0.0;
      auto t0 = std::chrono::steady_clock::now();
      for (int s = 0; s < warmup + steps; ++s) {
        if (s == warmup) t0 = std::chrono::steady_clock::now();
        if (mode == 0) {
          QueryBundle b;
          for (int l = 0; l < L; ++l) {
            const float* q = queries + (static_cast<std::size_t>(s) * L + l) * d;
            b.q.emplace_back(q, q + d);
          }
          RetrievalResult r = retrieve(b, rc, index, store, maint, window);
          for (int l = 0; l < L; ++l) {  // fp64 attention restatement over the attended set
            const auto& att = r.layers[static_cast<std::size_t>(l)].attended_tokens;
            const float* q = queries + (static_cast<std::size_t>(s) * L + l) * d;
            const double scale = 1.0 / std::sqrt(static_cast<double>(d));
            std::vector<double> sc(att.size());
            double mx = -1e300;
            for (std::size_t j = 0; j < att.size(); ++j) {
              std::size_t i = static_cast<std::size_t>(att[j].first) * TT + static_cast<std::size_t>(att[j].second);
              const float* k = keys + (static_cast<std::size_t>(l) * N + i) * d;
              double acc = 0.0;
              for (int c = 0; c < d; ++c) acc += static_cast<double>(q[c]) * k[c];
              sc[j] = acc * scale;
              mx = std::max(mx, sc[j]);
            }
            std::vector<double> o(static_cast<std::size_t>(d), 0.0);
            double den = 0.0;
            for (std::size_t j = 0; j < att.size(); ++j) {
              std::size_t i = static_cast<std::size_t>(att[j].first) * TT + static_cast<std::size_t>(att[j].second);
              const float* v = values + (static_cast<std::size_t>(l) * N + i) * d;
              double w = std::exp(sc[j] - mx);
              den += w;
              for (int c = 0; c < d; ++c) o[static_cast<std::size_t>(c)] += w * v[c];
            }
            sink += o[0] / den;
          }
        } else {
          const std::int64_t fid = 1000000 + s;
          Embedding fv(fvis + static_cast<std::size_t>(s) * d, fvis + static_cast<std::size_t>(s + 1) * d);
          std::int64_t p = maint.place_frame(fid, fv);
          for (int l = 0; l < L; ++l)
            for (int t = 0; t < T; ++t) {
              KVEntry e;
              std::size_t off = ((static_cast<std::size_t>(s) * L + l) * T + t) * d;
              e.key.assign(fkeys + off, fkeys + off + d);
              e.value.assign(fvals + off, fvals + off + d);
              e.frame_id = fid;
              e.layer_id = l;
              e.token_id = t;
              maint.on_insert(p, e);
            }
        }
      }
      auto t1 = std::chrono::steady_clock::now();
      per[static_cast<std::size_t>(ti)] = std::chrono::duration<double, std::micro>(t1 - t0).count() / steps;
      if (sink == 12345.678) per[static_cast<std::size_t>(ti)] += 0.0;
    } catch (const std::exception& e) {
      errs[static_cast<std::size_t>(ti)] = e.what();
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < threads; ++i) pool.emplace_back(worker, i);
  for (auto& th : pool) th.join();
  for (const auto& e : errs)
    if (!e.empty()) throw Error(e);
  double mx = 0.0, mean = 0.0;
  for (double v : per) {
    mx = std::max(mx, v);
    mean += v / threads;
  }
  out[0] = mx;
  out[1] = mean;
  GUARD_END
}

}  // extern "C"
