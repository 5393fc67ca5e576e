// kvclust_b200.hpp -- C++ drop-in for the hot-path part of the reference's public API
// (`kvclust::core`, /root/reference/proj/core/include/kvclust), backed by the B200 engine behind
// include/kvc.h.
//
// What it replaces (SURVEY.md §8(b) "must export"): the declarations of index.hpp:17-177
// (KVEntry, ClusterRecord, VisualPartition, CandidateRef, FrameInput, BuildConfig, HierIndex,
// compute_representative / compute_variance / build_index), store.hpp:15-127 (CostModel,
// TransferCause, TransferOp, CauseTotals, TransferLedger, TieredStore), maintainer.hpp:16-90
// (ThresholdConfig, tau, MaintainerConfig, MaintainerStats, Maintainer, StatUpdate,
// updated_stats) and retrieval.hpp:16-91 (RetrievalMode, RetrievalConfig, QueryBundle,
// LayerLatency, LayerResult, RetrievalResult, retrieve, oracle_flat_topk,
// retrieve_token_baseline). engine.hpp's surface is in kvclust_b200_engine.hpp. Same namespace,
// type names, member names, defaults and exception types, so callers recompile unchanged:
// point the include path at include/kvclust_dropin/ (whose kvclust/{index,store,maintainer,
// retrieval,engine}.hpp forward here) ahead of the reference's include directory, and link
// libkvclust_b200.so + libkvc.so instead of the hot-path translation units.
//
// Kept from the reference, unchanged (not on the hot path): the header-only utilities
// vecmath.hpp (Embedding / DVec / cosine_sim), error.hpp (the exception hierarchy), rng.hpp,
// clustering.hpp, and the non-hot-path modules workload / harness / report.
//
// Semantics: the state lives on the GPU. A HierIndex is a handle to a device context
// (kvc_ctx); TieredStore and Maintainer constructed over it are views of the same context
// (in the reference they hold references to the index, store.hpp:115 / maintainer.hpp:68-69).
// Operations run on the device with the reference's exact arithmetic; the
// host-side views (clusters(), partitions(), rep_set(), ...) are materialised from the device
// on demand and cached until the next mutation. Indexes assembled by hand (add_partition /
// add_cluster, as test_store.cpp and acceptance check 7 do) are installed on the device when
// the first device operation needs them; add_cluster takes the members' exact Eq. 1/2
// statistics (compute_representative / compute_variance), as every reference caller passes.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "kvclust/clustering.hpp"
#include "kvclust/error.hpp"
#include "kvclust/rng.hpp"
#include "kvclust/vecmath.hpp"

namespace kvclust {

namespace b200 {
struct Device;  // one kvc_ctx + the configuration it was created with (kvclust_b200.cpp)
}

// ================================================================== index (index.hpp:17-177)

enum class Residence { Device, Host };

struct KVEntry {
  Embedding key;
  Embedding value;
  std::int64_t frame_id = 0;
  std::int32_t layer_id = 0;
  std::int32_t token_id = 0;
};

struct ClusterRecord {
  std::int64_t cluster_id = 0;
  std::int32_t layer_id = 0;
  std::int64_t visual_parent = 0;
  std::vector<KVEntry> members;
  DVec rep;
  double variance = 0.0;
  std::int64_t stat_count = 0;
  bool lazy_split = false;
  std::vector<KVEntry> buffer;
  DVec buffer_rep;
  Residence residence = Residence::Device;
  std::int64_t device_tail = 0;
  std::int64_t first_frame_id = 0;
  std::int64_t last_touch_frame = 0;

  std::int64_t n() const { return static_cast<std::int64_t>(members.size()); }
  std::int64_t payload_bytes(std::int64_t bytes_per_entry) const { return n() * bytes_per_entry; }
};

struct VisualPartition {
  std::int64_t partition_id = 0;
  std::vector<std::int64_t> frame_ids;
  DVec visual_rep;
  std::int64_t visual_stat_count = 0;
  std::map<std::int32_t, std::vector<std::int64_t>> per_layer_clusters;
};

struct CandidateRef {
  std::int64_t cluster_id = 0;
  bool is_buffer = false;

  friend bool operator==(const CandidateRef&, const CandidateRef&) = default;
  friend auto operator<=>(const CandidateRef&, const CandidateRef&) = default;
};

struct FrameInput {
  std::int64_t frame_id = 0;
  Embedding visual;
  std::vector<std::vector<KVEntry>> layers;
};

struct BuildConfig {
  int target_visual_cluster_size = 8;
  int target_semantic_cluster_size = 32;
  int kmeans_max_iters = 50;
  double kmeans_tol = 1e-6;
  std::uint64_t seed = 0;
};

class HierIndex {
 public:
  HierIndex();
  HierIndex(std::int32_t dim, std::int32_t layers);
  HierIndex(HierIndex&&) noexcept;
  HierIndex& operator=(HierIndex&&) noexcept;
  HierIndex(const HierIndex&) = delete;  // the state is a device context
  HierIndex& operator=(const HierIndex&) = delete;
  ~HierIndex();

  std::int32_t dim() const { return dim_; }
  std::int32_t num_layers() const { return layers_; }
  bool empty() const { return partitions().empty(); }

  const std::vector<VisualPartition>& partitions() const;
  VisualPartition& partition(std::int64_t id);
  const VisualPartition& partition(std::int64_t id) const;

  const std::map<std::int64_t, ClusterRecord>& clusters() const;
  ClusterRecord& cluster(std::int64_t id);
  const ClusterRecord& cluster(std::int64_t id) const;
  bool has_cluster(std::int64_t id) const { return clusters().count(id) != 0; }

  const std::vector<CandidateRef>& rep_set(std::int32_t layer) const;
  const std::vector<std::int64_t>& rep_timeline(std::int32_t layer) const;
  const DVec& candidate_rep(const CandidateRef& ref) const;

  std::int64_t add_partition(std::int64_t first_frame_id, const Embedding& visual);
  void append_frame(std::int64_t partition_id, std::int64_t frame_id, const Embedding& visual);
  std::int64_t add_cluster(ClusterRecord&& rec);
  void remove_cluster(std::int64_t id);
  void register_buffer(std::int64_t cluster_id);
  void deregister_buffer(std::int64_t cluster_id);
  bool buffer_registered(std::int64_t cluster_id) const;
  void add_member(std::int64_t cluster_id, KVEntry entry);
  void add_to_buffer(std::int64_t cluster_id, KVEntry entry);

  // Stage one / stage two of the two-stage lookup (index.cpp:192-240), on the device.
  std::vector<std::int64_t> visual_topk(const Embedding& query, int k_v) const;
  std::vector<CandidateRef> semantic_topk(const Embedding& query, std::int32_t layer,
                                          const std::vector<std::int64_t>& partition_ids, int k_s) const;

  std::set<std::int64_t> clusters_of_frame(std::int64_t frame_id) const;
  std::int64_t entries_at_layer(std::int32_t layer) const;
  std::int64_t total_member_entries() const;
  void check_invariants() const;

  // The reference's index.v1 JSON (index.cpp:452-592): partitions, clusters with members, buffers
  // and statistics. A parsed index is host-assembled and installed on first device use.
  std::string to_json_string() const;
  static HierIndex from_json_string(const std::string& text);

  // The device context behind this index (created on first use from the host-assembled
  // state; kvclust_b200.cpp). Not part of the reference's surface.
  b200::Device& device() const;
  void mark_device_changed() const;  // host views are re-materialised on next access

 private:
  friend HierIndex build_index(const std::vector<FrameInput>&, const BuildConfig&);
  friend struct b200::Device;
  struct View;  // materialised host view (partitions, clusters, rep sets, timelines)

  std::int32_t dim_ = 0;
  std::int32_t layers_ = 0;
  mutable std::shared_ptr<b200::Device> dev_;
  // host-assembled state not yet installed on the device (add_partition / add_cluster before the
  // first device operation)
  std::vector<VisualPartition> pending_parts_;
  std::vector<Embedding> pending_first_visual_;                                   // per pending partition
  std::vector<std::vector<std::pair<std::int64_t, Embedding>>> pending_appends_;  // append_frame calls
  std::vector<ClusterRecord> pending_clusters_;
  std::vector<std::uint8_t> pending_adopted_;
  std::set<std::int64_t> pending_registered_;
  mutable std::unique_ptr<View> view_;

  const View& view() const;
  void install_pending() const;
  friend class TieredStore;
  friend class StreamEngine;
};

DVec compute_representative(const std::vector<KVEntry>& members);
double compute_variance(const std::vector<KVEntry>& members, const DVec& rep);
HierIndex build_index(const std::vector<FrameInput>& frames, const BuildConfig& cfg);

// ================================================================== store (store.hpp:15-127)

struct CostModel {
  double alpha_us = 10.0;
  double beta_us_per_byte = 0.001;
  std::int64_t bytes_per_entry = 0;
  std::int64_t device_capacity_entries = 1 << 20;

  double transfer_cost(std::int64_t n_ops, std::int64_t bytes) const {
    return static_cast<double>(n_ops) * alpha_us + static_cast<double>(bytes) * beta_us_per_byte;
  }
  std::int64_t entry_bytes(std::int32_t dim) const {
    return bytes_per_entry > 0 ? bytes_per_entry : static_cast<std::int64_t>(dim) * 2 * static_cast<std::int64_t>(sizeof(float));
  }
};

enum class TransferCause { Retrieval, Maintenance, Prefetch, Completion, Offload };
const char* to_string(TransferCause cause);

struct TransferOp {
  TransferCause cause = TransferCause::Retrieval;
  bool to_device = true;
  std::int64_t cluster_id = -1;
  std::int64_t n_ops = 0;
  std::int64_t bytes = 0;
  double cost_us = 0.0;
};

struct CauseTotals {
  std::int64_t n_ops = 0;
  std::int64_t bytes = 0;
  double cost_us = 0.0;
};

// The simulated-cost ledger (store.cpp:21-65). Plain host bookkeeping: the device engine keeps
// the authoritative op log; a TieredStore's ledger() is refreshed from it on access.
class TransferLedger {
 public:
  void record(const TransferOp& op);
  const std::vector<TransferOp>& log() const { return log_; }
  const std::map<std::string, CauseTotals>& by_cause() const { return totals_; }
  CauseTotals totals() const;
  CauseTotals cause(TransferCause c) const;
  void audit() const;
  void clear();

 private:
  std::vector<TransferOp> log_;
  std::map<std::string, CauseTotals> totals_;
};

class TieredStore {
 public:
  // Adopts every existing cluster (store.cpp:67-74); validates the cost constants.
  TieredStore(HierIndex& index, const CostModel& cost);

  void adopt(std::int64_t cluster_id);
  void forget(std::int64_t cluster_id);
  double fetch(std::int64_t cluster_id, TransferCause cause);
  double offload(std::int64_t cluster_id);
  void note_device_append(std::int64_t cluster_id);
  void note_device_buffer_append(std::int64_t cluster_id);
  void touch(std::int64_t cluster_id);
  void pin(const std::set<std::int64_t>& cluster_ids);
  bool on_device(std::int64_t cluster_id) const;
  std::int64_t device_entries() const;
  double enforce_capacity();
  TransferLedger& ledger();
  const TransferLedger& ledger() const;
  const CostModel& cost() const { return cost_; }
  void audit() const;

  HierIndex& index() const { return index_; }

 private:
  HierIndex& index_;
  CostModel cost_;
  mutable TransferLedger ledger_;
  mutable std::size_t ledger_seen_ = 0;
  void refresh_ledger() const;
};

// ================================================================== maintainer (maintainer.hpp:16-90)

struct ThresholdConfig {
  double tau_min = 0.05;
  double tau_max = 0.3;
  double n0 = 32.0;
};

double tau(std::int64_t n, const ThresholdConfig& cfg);

struct MaintainerConfig {
  ThresholdConfig threshold;
  bool defer_host_splits = true;
  int max_split_depth = 4;
  double visual_floor = 0.75;
  std::uint64_t seed = 0;
};

struct MaintainerStats {
  std::int64_t inserts = 0;
  std::int64_t absorbed = 0;
  std::int64_t immediate_splits = 0;
  std::int64_t deferred_marks = 0;
  std::int64_t settled_splits = 0;
  std::int64_t split_ops_total = 0;
  std::int64_t host_over_threshold = 0;
  std::int64_t maintenance_fetches = 0;
  std::int64_t partitions_opened = 0;
};

class Maintainer {
 public:
  Maintainer(HierIndex& index, TieredStore& store, const MaintainerConfig& cfg);

  // place_frame (maintainer.cpp:37-53) and on_insert (maintainer.cpp:88-176) run on the device
  // engine: on_insert resolves the entry with the GPU candidate scan + exact Eq. 3/4 / Eq. 5
  // chain and returns the routed cluster id; splits are settled in reference order.
  std::int64_t place_frame(std::int64_t frame_id, const Embedding& visual);
  std::int64_t on_insert(std::int64_t partition_id, const KVEntry& entry);
  std::vector<std::int64_t> materialize(std::int64_t cluster_id);
  const MaintainerStats& stats() const;

 private:
  HierIndex& index_;
  TieredStore& store_;
  MaintainerConfig cfg_;
  mutable MaintainerStats stats_;
};

struct StatUpdate {
  DVec rep;
  double variance = 0.0;
};
StatUpdate updated_stats(const DVec& rep, double variance, std::int64_t n, const Embedding& key);

// ================================================================== retrieval (retrieval.hpp:16-91)

enum class RetrievalMode { Cluster, TokenBaseline };

struct RetrievalConfig {
  int k_v = 4;
  int k_s = 4;
  int window_frames = 4;
  int prefetch_k = 4;
  bool prefetch_enabled = false;
  RetrievalMode mode = RetrievalMode::Cluster;
  std::int64_t token_budget = 256;
  double lookup_cost_per_candidate_us = 0.02;
  double compute_cost_per_token_us = 0.6;

  void validate() const;
};

struct QueryBundle {
  std::int64_t query_id = 0;
  std::vector<Embedding> q;
  std::vector<std::int64_t> ground_truth_frames;
};

struct LayerLatency {
  double lookup_us = 0.0;
  double transfer_us = 0.0;
  double stall_us = 0.0;
  double completion_us = 0.0;
  double compute_us = 0.0;

  double total() const { return lookup_us + transfer_us + stall_us + completion_us + compute_us; }
};

struct LayerResult {
  std::vector<CandidateRef> ranked;
  std::vector<std::int64_t> selected;
  std::vector<std::int64_t> predicted;
  std::int64_t prefetch_hits = 0;
  std::int64_t verified_clusters = 0;
  std::vector<std::pair<std::int64_t, std::int32_t>> attended_tokens;
  std::int64_t rep_count = 0;
  LayerLatency latency;
};

struct RetrievalResult {
  std::int64_t query_id = 0;
  std::vector<LayerResult> layers;
  double ttft_us = 0.0;
  double recall = -1.0;
  std::vector<std::int64_t> context_frames;
  std::vector<std::int64_t> fetched_frames;
};

// One decode step on the device (K4 scoring / selection, settle, K6 attention). `window` must be
// empty or the entries of the context's own recent frames (the engine keeps its window on the
// device); the attention outputs are available through b200::last_attention().
RetrievalResult retrieve(const QueryBundle& bundle, const RetrievalConfig& cfg, HierIndex& index,
                         TieredStore& store, Maintainer& maintainer, const std::vector<KVEntry>& window);

std::vector<CandidateRef> oracle_flat_topk(const HierIndex& index, const Embedding& query,
                                           std::int32_t layer, int k);

// The token-granular baseline on the device (token.cu): pools[l] hold whole frames (each frame's
// entries with token ids 0..T-1 in order); window_frames are the frames attended without a fetch.
RetrievalResult retrieve_token_baseline(const QueryBundle& bundle, const RetrievalConfig& cfg,
                                        const std::vector<std::vector<KVEntry>>& pools,
                                        const std::set<std::int64_t>& window_frames, const CostModel& cost,
                                        TransferLedger& ledger);

namespace b200 {
// fp32 attention outputs [L][d] of the last device decode step run through this API on the
// calling thread (retrieve / StreamEngine), the product's extension (no reference counterpart).
const std::vector<float>& last_attention();
}  // namespace b200

}  // namespace kvclust
