// context.hpp -- one stream's cluster-level KV cache: host control plane + device data plane.
//
// The host side keeps what the reference keeps in HierIndex / TieredStore / Maintainer /
// StreamEngine *except* the payloads and the statistics: ids, partitions, member identities
// (frame, token) in stored order, residency, LRU ticks, the transfer ledger, split counters
// (index.hpp:84-166, store.hpp:73-125, maintainer.hpp:48-80, engine.hpp:62-100). K/V payloads,
// fp64 representatives / variances and page tables live on the GPU and are only read back on
// the split slow path or through debug accessors.
#pragma once

#include <array>
#include <climits>
#include <cstdint>
#include <cstddef>
#include <deque>
#include <iterator>
#include <memory>
#include <unordered_map>
#include <vector>

#include "../../include/kvc.h"
#include "extent_alloc.hpp"
#include "kmeans.hpp"
#include "kvc_core.hpp"

namespace kvc {

struct Member {
  std::int64_t frame;
  std::int32_t token;
};

// Member identities of a cluster in stored order, run-length encoded: a frame's tokens are
// appended in runs (one run per frame and cluster on the ingest path), so a 512-member cluster is
// a handful of runs and appends never reallocate a long vector.
class MemberList {
 public:
  struct Run {
    std::int64_t frame;
    std::int32_t tok0, count;
  };
  class iterator {
   public:
    using iterator_category = std::forward_iterator_tag;
    using value_type = Member;
    using difference_type = std::ptrdiff_t;
    using pointer = const Member*;
    using reference = Member;
    iterator(const Run* r, std::int32_t k) : r_(r), k_(k) {}
    Member operator*() const { return {r_->frame, r_->tok0 + k_}; }
    iterator& operator++() {
      if (++k_ == r_->count) {
        ++r_;
        k_ = 0;
      }
      return *this;
    }
    iterator operator++(int) {
      iterator x = *this;
      ++*this;
      return x;
    }
    bool operator==(const iterator& o) const { return r_ == o.r_ && k_ == o.k_; }
    bool operator!=(const iterator& o) const { return !(*this == o); }

   private:
    const Run* r_;
    std::int32_t k_;
  };
  MemberList() = default;
  MemberList(const std::vector<Member>& v) {
    for (const Member& m : v) push_back(m);
  }
  void push_back(const Member& m) { push_run(m.frame, m.token, 1); }
  void push_run(std::int64_t frame, std::int32_t tok0, std::int32_t count) {
    if (count <= 0) return;
    if (!runs_.empty() && runs_.back().frame == frame && runs_.back().tok0 + runs_.back().count == tok0)
      runs_.back().count += count;
    else
      runs_.push_back({frame, tok0, count});
    n_ += count;
  }
  std::size_t size() const { return static_cast<std::size_t>(n_); }
  bool empty() const { return n_ == 0; }
  Member front() const { return {runs_.front().frame, runs_.front().tok0}; }
  iterator begin() const { return iterator(runs_.data(), 0); }
  iterator end() const { return iterator(runs_.data() + runs_.size(), 0); }
  const std::vector<Run>& runs() const { return runs_; }
  operator std::vector<Member>() const { return std::vector<Member>(begin(), end()); }

 private:
  std::vector<Run> runs_;
  std::int64_t n_ = 0;
};

struct Cluster {  // ClusterRecord (index.hpp:29-50) minus payload and statistics
  std::int64_t id = 0;
  std::int32_t layer = 0;
  std::int64_t parent = 0;
  std::int32_t slot = -1;
  MemberList members, buffer;
  std::int64_t stat_count = 0;
  std::int64_t device_tail = 0;
  std::int64_t first_frame = 0, last_touch = 0;
  // lazy_split, residence, the TieredStore LRU entry and the pin live in compact per-id arrays of
  // the Context (cflags_ / last_use_) so the per-step bookkeeping stays cache resident
};

enum ClusterFlag : std::uint8_t { CF_HOST = 1, CF_LAZY = 2, CF_TRACKED = 4, CF_PINNED = 8 };

struct Partition {  // VisualPartition (index.hpp:52-58)
  std::vector<std::int64_t> frames;
  std::vector<double> vrep;
  std::int64_t stat = 0;
  std::vector<std::vector<std::int64_t>> per_layer;  // [L] cluster ids, stored order
  std::vector<std::int32_t> dev_off, dev_cap;        // [L] region of the device slot list
};

struct LedgerOp {  // TransferOp (store.hpp:35-42)
  int cause;
  bool to_device;
  std::int64_t cluster_id, n_ops, bytes;
  double cost_us;
};

struct LayerOut {  // LayerResult (retrieval.hpp:49-59)
  std::vector<std::pair<std::int64_t, int>> ranked, pf;  // pf: device prefetch ranking (l+1)
  std::vector<std::int64_t> selected, predicted;
  std::int64_t prefetch_hits = 0, verified = 0, rep_count = 0, attended_count = 0;
  double lat[5] = {0, 0, 0, 0, 0};
  std::vector<std::pair<std::int64_t, std::int32_t>> attended;  // parity mode
};

struct PendingFrame {
  std::int64_t frame_id;
  std::vector<float> visual;
  std::vector<float> keys_f32;  // [L][T][d] (exact values of the kv dtype)
  std::vector<std::uint8_t> keys_raw, vals_raw;  // kv dtype
  int T;
};

class Context {
 public:
  Context(const kvc_cfg& cfg, int d, int L);
  ~Context();
  void release();  // every device / host allocation, stream and event (destructor, failed ctor)

  void ingest_frame(std::int64_t frame_id, const float* visual, const void* keys,
                    const void* values, int T, int mem, std::int64_t* assigned,
                    std::int64_t* partition);
  void decode_step(std::int64_t qid, const float* q, int q_mem, float* out, int out_mem,
                   const std::int64_t* gt, int n_gt);
  void build_now();
  std::int64_t bulk_load(const float* visual, const void* keys, const void* values, int N, int C,
                         const std::int32_t* assign, const std::int64_t* frame_ids,
                         const std::int32_t* token_ids, int mem);
  std::vector<std::pair<std::int64_t, int>> flat_topk(const float* q, int layer, int k);

  // views
  const kvc_cfg& cfg() const { return cfg_; }
  int d() const { return d_; }
  int L() const { return L_; }
  const Cluster* cluster(std::int64_t id) const;
  bool is_host(std::int64_t id) const { return cflags_[static_cast<std::size_t>(id)] & CF_HOST; }
  bool is_lazy(std::int64_t id) const { return cflags_[static_cast<std::size_t>(id)] & CF_LAZY; }
  std::vector<std::int64_t> cluster_ids() const;
  void cluster_stats(std::int64_t id, double* var, double* rep, double* brep);
  int cluster_payload(std::int64_t id, int which, float* k, float* v, int cap);
  const std::vector<Partition>& partitions() const { return parts_; }
  const std::vector<LayerOut>& last_layers() const { return last_; }
  double last_ttft() const { return last_ttft_; }
  double last_recall() const { return last_recall_; }
  std::uint64_t last_digest() const { return last_digest_; }
  const std::int64_t* maint_stats() const { return mstats_; }
  const std::vector<LedgerOp>& ledger() const { return ledger_; }
  std::int64_t device_entries() const { return device_entries_; }
  void check();
  // Completes the deferred host bookkeeping of the last decode step (every host-state reader
  // calls this first; decode_step overlaps it with the next step's GPU work).
  void flush_pending();
  void flush_decode();  // only the decode step's deferred bookkeeping (ingest keeps its pipeline)
  double offload(std::int64_t id);
  double fetch(std::int64_t id, int cause);
  cudaStream_t stream() const { return st_; }
  std::int64_t launches() const { return launches_; }
  void set_timing(bool on) { timing_ = on; }
  // attention scale 1/sqrt(d_logical) for rows zero-padded to d (kvc_set_head_dim)
  void set_head_dim(int d_logical);
  const double* step_timing() const { return step_t_; }
  const double* ingest_timing() const { return ingest_t_; }
  // Runs the candidate build + distance tile (+ top-M) on a frame for partition `pid` without
  // resolving, then checks it against exact cosines. out: max |approx - exact|, top-M
  // violations, exact mismatches, the margin the resolve kernels assume.
  void debug_assign_check(const void* keys, int T, std::int64_t pid, int mem, double* out);
  void resolve_profile(double* out);  // mean clock64 cycles per resolve phase over domains
  // physical host tier (context_tiers.cpp): migrations follow the logical residence
  void tier_kick();  // polls in-flight migrations, starts queued ones (never blocks)
  void tier_sync();  // completes everything queued or in flight
  void tier_stats(std::int64_t* out) const;
  void cluster_tier(std::int64_t id, std::int64_t* out) const;
  void tier_check(std::int64_t* out);
  // fused output exchange across ranks (multi-GPU by domain; context_query.cpp)
  void set_peers(int n, int rank, int dom_offset, int total_domains, void* const* bufs);
  void peer_output(float* out, int mem);
  // component-level API (context_api.cpp): the reference's HierIndex / TieredStore / Maintainer /
  // retrieve calls one by one, for the C++ drop-in (include/kvclust_b200.hpp)
  std::int64_t api_add_partition(std::int64_t first_frame, const float* visual);
  void api_append_frame(std::int64_t pid, std::int64_t frame, const float* visual);
  std::int64_t api_add_cluster(int layer, std::int64_t parent, int n, const float* keys, const float* values,
                               const std::int64_t* frames, const std::int32_t* tokens, bool host, bool adopt_it);
  void api_adopt(std::int64_t id);
  std::int64_t api_add_partition_ex(const std::int64_t* frames, int n_frames, const double* visual_rep, std::int64_t stat);
  std::int64_t api_add_cluster_ex(int layer, std::int64_t parent, int n_mem, const float* mk, const float* mv,
                                  const std::int64_t* mf, const std::int32_t* mt, int n_buf, const float* bk,
                                  const float* bv, const std::int64_t* bf, const std::int32_t* bt, const double* rep,
                                  double var, std::int64_t stat, const double* brep, bool lazy, bool host,
                                  std::int64_t device_tail, bool adopt_it, std::int64_t want_id);
  void api_reset_window();
  void api_set_retrieval(const kvc_cfg& c);
  void api_reconfigure(const kvc_cfg& c, int what);  // bits: 1 retrieval, 2 cost model, 4 maintainer
  std::int64_t api_place_frame(std::int64_t frame, const float* visual);
  void component_index();
  std::int64_t api_insert(std::int64_t pid, int layer, int token, std::int64_t frame, const float* key,
                          const float* value);
  std::vector<std::int64_t> api_materialize(std::int64_t id);
  void api_touch(std::int64_t id);
  void api_pin(const std::vector<std::int64_t>& ids);
  double api_enforce_capacity();
  std::vector<std::int64_t> api_visual_topk(const float* q, int k);
  std::vector<std::pair<std::int64_t, int>> api_semantic_topk(const float* q, int layer,
                                                              const std::vector<std::int64_t>& part_ids, int k);
  // frames of the last step's selected clusters / attended entries (RetrievalResult
  // fetched_frames / context_frames, retrieval.cpp:99-110; parity mode or ground truth given)
  const std::vector<std::int64_t>& last_fetched_frames() const { return last_fetched_; }
  const std::vector<std::int64_t>& last_context_frames() const { return last_context_; }

 private:
  // ---- configuration
  kvc_cfg cfg_;
  int d_, L_, es_;
  int dl_ = 0;  // the caller's head width (kvc_set_head_dim; d_ unless rows are zero-padded)
  // ---- device
  DevTables t_{};
  cudaStream_t st_ = nullptr;
  std::vector<void*> dev_allocs_;
  void* dalloc(std::size_t bytes);
  void* halloc(std::size_t bytes);  // pinned
  void* dalloc_scratch(std::size_t bytes);  // reusable device scratch (grows)
  void* scratch_ = nullptr;
  std::size_t scratch_cap_ = 0;
  std::vector<void*> host_allocs_;
  // frame input + staging
  void* d_fk_ = nullptr;  // the current frame's input buffer (one of fkbuf_ / fvbuf_)
  void* d_fv_ = nullptr;
  void* fkbuf_[2] = {nullptr, nullptr};
  void* fvbuf_[2] = {nullptr, nullptr};
  void* d_stage_k_ = nullptr;
  void* d_stage_v_ = nullptr;
  float* d_stage_f32_ = nullptr;
  std::int64_t stage_rows_ = 0;
  float* h_stage_f32_ = nullptr;
  std::int32_t* d_idx_ = nullptr;
  std::int32_t* h_idx_ = nullptr;
  std::int64_t idx_cap_ = 0;
  AppendRun* d_runs_ = nullptr;
  AppendRun* h_runs_ = nullptr;
  std::int64_t runs_cap_ = 0;
  // slot-init staging
  void* d_init_ = nullptr;
  void* h_init_ = nullptr;
  std::int64_t init_cap_ = 0;
  cudaEvent_t ev_init_ = nullptr;  // the last slot-init copy out of h_init_
  // ingest buffers
  IngestArgs ia_{};
  std::int32_t *d_active_ = nullptr, *h_active_ = nullptr, *d_cursor_ = nullptr, *h_cursor_ = nullptr;
  std::int32_t* h_evk_ = nullptr;  // the current frame's outcome block (one of h_out_)
  std::int32_t* h_evs_ = nullptr;
  std::int32_t* h_stop_ = nullptr;  // [3][L]: stop_t, stop_kind, stop_slot
  std::int32_t* h_out_[2] = {nullptr, nullptr};
  std::int32_t* h_errb_[2] = {nullptr, nullptr};
  // Pipelined ingest: frame i's kernels are launched and its outcome block copied back, and its
  // host replay is deferred until the next ingest call has launched frame i + 1 (when frame i
  // needed no host event), or until any host-state reader flushes it.
  struct PendingIngest {
    bool active = false;
    std::int64_t frame_id = 0, pid = 0;
    int T = 0, ring_slot = 0, buf = 0;
    cudaEvent_t ev = nullptr;  // outcome block of the first launch on the host
  };
  const void* mapped_host(const void* p);
  static constexpr int kActSlots = 4;
  int act_next_ = 0;
  cudaEvent_t ev_act_[kActSlots] = {nullptr, nullptr, nullptr, nullptr};
  std::int32_t* d_evflags_ = nullptr;  // [2] per frame buffer: its first round stopped a domain
  std::int32_t* d_all_active_ = nullptr;  // [0..L) then L zeros: a first round's active / cursor
  bool spec_ingest_ = true;            // KVC_INGEST_SPEC=0: wait for the previous outcome first
  PendingIngest ping_;  // launched, outcome not yet inspected
  PendingIngest pong_;  // the frame before: kernels complete, no host events, replay pending
  void finish_pong();
  cudaEvent_t ev_ing_[2] = {nullptr, nullptr};  // per frame buffer: its outcome block reached the host
  cudaEvent_t ev_in_[2] = {nullptr, nullptr};   // per frame buffer: payload copied in (input stream)
  cudaEvent_t ev_buf_[2] = {nullptr, nullptr};  // per frame buffer: last reader on the compute stream done
  cudaStream_t in_st_ = nullptr;                // frame payload copies
  int ibuf_ = 0;  // buffer of the most recently launched frame
  bool round_timed_ = false;  // the last resolve round recorded its phase events
  cudaEvent_t ping_wait_ = nullptr;  // outcome event of the frame being finished
  void select_frame_buffer(int b);
  void launch_round(const std::vector<int>& active, const std::vector<int>& cursor);
  void finish_frame(std::int64_t* assigned);  // replay (+ host events) of ping_, then window/cadence
  void flush_ingest();
  // decode buffers
  DecodeArgs da_{};
  void* d_dec_ = nullptr;  // packed result block
  // two host copies of the decode result block: step i fills one while step i-1's bookkeeping
  // is replayed from the other
  void* h_blk_[2] = {nullptr, nullptr};
  cudaEvent_t ev_step_[2] = {nullptr, nullptr};  // result block b copied to the host (copy stream)
  cudaEvent_t ev_k4_[2] = {nullptr, nullptr};    // K4 of the step in block b done (compute stream)
  cudaEvent_t ev_out_[2] = {nullptr, nullptr};   // attention output of that step done
  cudaStream_t cs_ = nullptr;                    // copy stream for the result blocks
  void* d_blk_[2] = {nullptr, nullptr};
  struct ResultOffsets {
    std::size_t parts, nps, rs, rb, nr, ps, pb, np, vs, nv, att, nc, fl, ew, frn, frr;
  } res_off_{};
  std::size_t dec_lean_bytes_ = 0;       // the block without the fetch-on-read records
  bool blk_fr_[2] = {false, false};      // block b's step ran with fetch-on-read
  bool fr_enabled_ = true;               // KVC_FETCH_ON_READ (default 1)
  void fr_commit(int b);
  void set_result_block(int b);
  cudaEvent_t evb_[2][4] = {{nullptr, nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr, nullptr}};
  bool step_timed_[2] = {false, false};
  bool blk_used_[2] = {false, false};
  int cur_ = 0;           // buffer of the most recently launched step
  bool inflight_ = false;  // that step's bookkeeping has not been replayed yet
  std::vector<std::int64_t> step_gt_[2];
  void launch_step(int b, const float* q, int q_mem, float* out, int out_mem);
  bool finish_step(int b);
  void replay_decode(const void* hblock, const std::int64_t* gt, int n_gt);
  std::size_t dec_bytes_ = 0;
  std::int32_t kv_cap_ = 0, ks_cap_ = 0, kp_cap_ = 0;  // budgets the result blocks are carved for
  void alloc_result_blocks(std::int32_t kv, std::int32_t ks, std::int32_t kp);
  float* d_q_ = nullptr;
  float* d_out_ = nullptr;
  cudaEvent_t ev_[8] = {};
  bool timing_ = false;
  bool resolve_seq_ = false;  // KVC_RESOLVE=seq selects the sequential resolve kernel
  // A domain relaunched after a split runs the speculative kernel seeded by the fp32 routing
  // simulation, its fresh children settled by warp-parallel cosine bounds (resolve_spec.cu):
  // ≈ 0.35 ms vs ≈ 1 ms per relaunch round for the sequential kernel (KVC_RELAUNCH=seq).
  bool relaunch_seq_ = false;
  bool round_after_event_ = false;
  bool assign_tc_ = false;    // tensor-core distance tile (KVC_ASSIGN=simt disables)
  alignas(64) unsigned char key_map_[128];  // CUtensorMap over the current frame's keys
  alignas(64) unsigned char key_maps_[2][128];
  void* d_check_ = nullptr;                 // debug_assign_check result words
  double step_t_[10] = {0};
  // last frame: device us (cands, assign, topm, resolve, store), host us (wait, on_insert loop,
  // of which replay and relaunch issue), host events
  double ingest_t_[10] = {0};
  // host-event (split / seed) slow-path profile, cumulative: total, stage + download, split
  // k-means, host Eq. 1/2 stats, slot/page uploads, relaunch after an event, #events, #split_two
  double evt_t_[8] = {0};
  // Speculative split k-means (host-event pipelining): while a domain is relaunched after its
  // split, the NEXT domain's pending split (its first event of the frame, known from the first
  // round) is already staged and 2-means'd on a side stream with the seed the global split
  // counter will give it if the relaunched domain splits no more (maintainer.cpp:222). The
  // settle takes the result when counter, cluster and row count match, else computes it anew --
  // nothing is committed speculatively, so a misprediction costs only the side work.
  struct SpecSplit {
    bool active = false;
    int layer = -1, tok = -1;
    std::int32_t slot = -1;
    std::int64_t rows = 0;  // staged rows incl. the triggering token
    std::uint64_t counter = 0;
    cudaEvent_t ev = nullptr;
    void *dk = nullptr, *dv = nullptr;
    float* df32 = nullptr;
    std::int64_t cap = 0;  // rows the staging holds
    double* scratch = nullptr;
    std::int32_t* d_i = nullptr;  // idx[n] | assign[n] | meta[4]
    double* d_obj = nullptr;
    std::int32_t* h_i = nullptr;
    double* h_obj = nullptr;
  } spec_;
  cudaStream_t spec_st_ = nullptr;
  std::int32_t spec_slot_hint_ = -1;  // slot of the cluster an immediate split is settling
  bool build_seed_set_ = false;  // build_index(frames, BuildConfig) called directly: its seed
  std::uint64_t build_seed_ = 0;
  bool spec_split_ = true;  // KVC_SPEC_SPLIT=0 disables
  std::int64_t spec_tries_ = 0, spec_hits_ = 0;
  void spec_split_launch(int from_layer, int T);
  bool spec_split_take(std::int32_t slot, int n, std::uint64_t counter, KMeansOut& out);

 public:
  void event_profile(double* out, bool reset) {
    for (int i = 0; i < 8; ++i) out[i] = evt_t_[i];
    out[8] = static_cast<double>(spec_tries_);
    out[9] = static_cast<double>(spec_hits_);
    if (reset) {
      for (double& x : evt_t_) x = 0.0;
      spec_tries_ = spec_hits_ = 0;
    }
  }

 private:
  std::int64_t launches_ = 0;

  // ---- physical host tier (context_tiers.cpp)
  struct Extent {
    std::int64_t start = -1, n = 0;
  };
  struct TierBatch {
    int kind = 0;   // 0 offload, 1 fetch
    int phase = 0;  // offload: 0 count, 1 copy, 2 commit; fetch: 0 copy, 1 commit
    int ring = 0;   // mapped argument slot
    std::vector<std::int64_t> ids;
    std::vector<Extent> ext, stage;  // new host extent (offload) / staging run per cluster
    cudaEvent_t ev = nullptr;
  };
  static constexpr int kTierRing = 8, kTierMaxBatch = 2048;
  ExtentAlloc hext_alloc_, stage_alloc_;
  std::vector<Extent> hext_;              // by cluster id: extent referenced by its page list
  std::vector<std::uint8_t> tier_busy_;   // by cluster id: in a batch
  std::vector<std::int64_t> off_q_, fet_q_;
  std::deque<TierBatch> tier_fl_;
  std::vector<cudaEvent_t> tier_ev_free_;
  bool tier_ring_used_[kTierRing] = {};
  TierMove* tier_mv_ = nullptr;        // [kTierRing][kTierMaxBatch] pinned, mapped
  std::int32_t* tier_cnt_ = nullptr;   // [kTierRing][kTierMaxBatch] pinned, mapped (slots / counts)
  std::int32_t* tier_scratch_ = nullptr;  // [kTierMaxBatch][maxp] device (fetch commit)
  std::uint8_t* tier_stage_ = nullptr;    // HBM staging pages
  cudaStream_t xs_ = nullptr;             // transfer stream (copy engines)
  // offloads, fetches, bytes d2h, bytes h2d, batches, copies, fetch-on-read clusters / bytes
  std::int64_t tier_n_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  void tier_alloc();
  void tier_note(std::int64_t id, bool to_host);  // a logical residence change (offload / fetch)
  void tier_forget(std::int64_t id);              // the cluster is being removed
  void tier_ensure(std::int64_t id);
  bool tier_start();                              // starts one batch from the queues
  bool tier_advance(TierBatch& b, bool block);    // next phase; true when the batch finished
  int tier_ring_take();
  cudaEvent_t tier_event();

  // ---- fused output exchange (set_peers)
  int peer_n_ = 0, peer_rank_ = 0, peer_total_ = 0;
  std::uint8_t* peer_buf_[kMaxPeers] = {};
  unsigned long long peer_step_ = 0;
  unsigned long long* peer_flag_ptr(int r) const;

  // ---- host control plane
  std::vector<std::unique_ptr<Cluster>> clusters_;  // by id (dense, null when removed)
  std::vector<std::uint8_t> cflags_;                 // by id: ClusterFlag bits
  std::vector<std::int64_t> last_use_;               // by id: TieredStore::last_use_ tick
  bool flag(std::int64_t id, std::uint8_t f) const { return cflags_[static_cast<std::size_t>(id)] & f; }
  void set_flag(std::int64_t id, std::uint8_t f, bool v) {
    std::uint8_t& x = cflags_[static_cast<std::size_t>(id)];
    x = v ? static_cast<std::uint8_t>(x | f) : static_cast<std::uint8_t>(x & ~f);
  }
  std::int64_t n_live_ = 0;
  std::vector<std::int64_t> slot_id_;               // slot -> cluster id (-1 free)
  std::vector<std::int32_t> free_slots_;
  std::vector<Partition> parts_;
  std::vector<std::int64_t> layer_live_count_;      // rep_timeline sizes
  std::unordered_map<std::int64_t, std::vector<std::int64_t>> frame_clusters_;
  std::vector<std::uint8_t> resid_h_;               // device residence mirror
  bool resid_dirty_ = false;
  std::int64_t pl_bump_ = 0;
  std::int64_t min_lt_ = INT64_MAX;  // lower bound of last_touch over Device, non-lazy clusters
  double* h_part_ring_ = nullptr;
  std::int64_t part_ring_pos_ = 0;
  // store
  std::int64_t device_entries_ = 0, tick_ = 0;
  std::vector<std::int64_t> pinned_ids_;
  std::vector<LedgerOp> ledger_;
  // maintainer
  std::int64_t mstats_[9] = {0};
  std::int64_t split_counter_ = 0;
  std::uint64_t maint_seed_ = 0;
  std::vector<double> tau_host_;
  // engine
  bool built_ = false;
  std::vector<PendingFrame> pending_;
  struct WinFrame {
    std::int64_t frame_id;
    int ring_slot;
    int T;
  };
  std::deque<WinFrame> window_;
  std::int64_t frames_seen_ = 0;
  std::int64_t last_partition_ = -1;
  std::vector<std::int32_t> ring_owner_h_;  // [L][W][tmax] mirror
  struct RingFrame {
    std::int64_t frame_id = -1;
    int T = 0;
  };
  std::vector<RingFrame> ring_frame_;  // [W] frame held by each ring slot (device view)
  // last query
  std::vector<LayerOut> last_;
  double last_ttft_ = 0.0, last_recall_ = -1.0;
  std::vector<std::int64_t> last_fetched_, last_context_;
  std::uint64_t last_digest_ = 0;

  std::vector<std::int64_t> verified_tmp_;

  // ---- helpers
  void alloc_device();
  void upload_tau();
  Cluster& C(std::int64_t id);
  std::int32_t take_slot();
  std::int64_t new_cluster(std::int32_t layer, std::int64_t parent, std::vector<Member>&& members,
                           bool host);
  // new_cluster on a slot the caller already holds (the wave engine installs children first)
  std::int64_t new_cluster_at(std::int32_t slot, std::int32_t layer, std::int64_t parent, std::vector<Member>&& members,
                              bool host);
  void drop_cluster(std::int64_t id);  // HierIndex::remove_cluster (host side)
  // drop_cluster without releasing the slot: its pages are freed and the slot returned by the caller
  void drop_cluster_host(std::int64_t id);
  void frame_add(std::int64_t frame, std::int64_t cid);
  void frame_add_flush(std::int64_t frame);
  std::vector<std::int64_t> fc_pending_;
  void frame_del(std::int64_t frame, std::int64_t cid);
  void pl_upload(std::int64_t pid, int layer);
  // capacity of the device slot list of (pid, layer) for n entries (may re-lay every list, which
  // rewrites the device lists from the host ones)
  void pl_reserve(std::int64_t pid, int layer, std::int32_t n);
  std::vector<std::int32_t> pl_floor_;  // [pid * L + layer] capacity a compaction keeps (wave engine)
  void upload_partition(std::int64_t pid);
  void flush_resid();
  // store (store.cpp:67-189)
  std::int64_t side_entries(const Cluster& c) const;
  void adopt(std::int64_t id);
  void forget(std::int64_t id);
  void touch(std::int64_t id);
  double enforce_capacity();
  double evict_one();
  void record(int cause, bool to_dev, std::int64_t id, std::int64_t bytes);
  std::int64_t entry_bytes() const;
  // engine (engine.cpp)
  void push_window(std::int64_t frame_id, int T, int slot);
  void repin();
  std::vector<std::int64_t> window_owner_ids() const;
  void apply_cadence(std::int64_t frame_id, std::int64_t pid);
  std::int64_t place_frame(std::int64_t frame_id, const float* visual);
  // domains [l_lo, l_hi) (l_hi < 0: all) from token tok0 (Maintainer::on_insert uses one domain,
  // one token, no window ring: ia_.ring_slot = -1)
  void run_inserts(std::int64_t frame_id, std::int64_t pid, int T, std::int64_t* assigned, bool launched,
                   int l_lo = 0, int l_hi = -1, int tok0 = 0);
  // Parallel settle of a frame's host events across domains (context_waves.cpp; deferred mode,
  // whole frames). KVC_WAVES=0 keeps the one-domain-at-a-time loop of run_inserts.
  struct Waves;
  Waves* wv_ = nullptr;
  bool waves_ = true;
  bool waves_perturb_ = false;
  bool waves_log_ = false;
  bool waves_eager_ = false;  // KVC_WAVES_EAGER=1: validation sweep predicts through restarted domains  // KVC_WAVES_LOG=1: per-frame pass / rollback lines on stderr  // KVC_WAVES_PERTURB=1: first-pass counter predictions made wrong (tests)
  void run_inserts_waves(std::int64_t frame_id, std::int64_t pid, int T, std::int64_t* assigned, bool launched);
  void replay_runs(int l, std::int64_t frame_id, int T, int t0, int t1, std::int64_t* assigned);
  void waves_free();
 public:
  // frames with events, waves, passes, rolled-back domains, verification k-means, events, stage us,
  // k-means jobs, k-means us, stats + install us, relaunch us, verify + commit us, splits verified
  // with exchanged labels (cumulative)
  void wave_profile(double* out13, bool reset);

 private:
  // split slow path
  std::vector<std::int64_t> split_pool(std::int64_t pid, int layer, bool host,
                                       std::vector<Member>&& ids, std::int64_t rows, int depth_unused);
  std::int64_t stage_cluster(std::int32_t slot, bool with_buffer);
 public:
  // split_two (kmeans.cpp) of staged rows grp[] on the GPU (split.cu), bit-identical to the host
  // restatement; falls back to it for groups below split_dev_min_ rows or d > 256.
  KMeansOut split_two_staged(const std::vector<int>& grp, std::uint64_t seed);
  // spherical_kmeans (kmeans.cpp) of several host point sets at once on the GPU (kmeans_dev.cu),
  // bit-identical to the host restatement; sets that do not fit a CTA run on the host.
  std::vector<KMeansOut> kmeans_pools(const std::vector<const float*>& pts, const std::vector<int>& n,
                                      const std::vector<int>& k_req, const std::vector<std::uint64_t>& seeds,
                                      int max_iters, double tol, bool stats = false);
  // debug: split_two of host points through the device path (stages them first)
  KMeansOut debug_split_two_dev(const float* pts, int n, std::uint64_t seed);

 private:
  int split_dev_min_ = 128;
  void* h_split_ = nullptr;  // pinned: idx[n] | assign[n] | meta[4] | objective
  std::int64_t split_cap_ = 0;
  void stage_download(std::int64_t rows);
  void init_slots(const std::vector<std::int32_t>& slots, const std::vector<std::vector<double>>& reps,
                  const std::vector<double>& vars, const std::vector<std::int64_t>& stats,
                  const std::vector<std::int64_t>& nmem, const std::vector<std::int64_t>& cids,
                  const std::vector<std::uint8_t>& resid, const std::vector<std::int32_t>* nbuf,
                  const std::vector<std::vector<double>>* breps);
  void append_runs_idx(const std::vector<AppendRun>& runs, const std::vector<std::int32_t>& idx,
                       const void* src_k = nullptr, const void* src_v = nullptr);
  void ring_owner_patch(int layer, const std::vector<Member>& ids, std::int32_t slot);
  void ring_owner_upload(int layer);
  std::int64_t handle_host_event(std::int64_t frame_id, std::int64_t pid, int layer, int tok,
                                 int kind, std::int32_t slot);
  std::vector<std::int64_t> materialize(std::int64_t id);
  void ensure_stage(std::int64_t rows);
  void ensure_idx(std::int64_t n, std::int64_t runs);
  void sync();
  void check_dev_err();
  void check_err_word(std::int32_t e);  // inspects a copied DevTables::err word
  std::int32_t* h_err_ = nullptr;       // pinned copy of DevTables::err
};

}  // namespace kvc
