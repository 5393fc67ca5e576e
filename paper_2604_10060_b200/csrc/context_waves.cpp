// context_waves.cpp -- parallel settle of a frame's host events (seeds / immediate splits) in
// deferred mode, bit-identical to the reference's sequential order.
//
// The reference inserts a frame layer by layer, token by token (engine.cpp:169-170 ->
// Maintainer::on_insert, maintainer.cpp:88-176). An immediate split (maintainer.cpp:139-149)
// draws its k-means seed from ONE global counter, mix_seed(seed, split_counter_++)
// (maintainer.cpp:222), and its children take the next global cluster ids (index.cpp:105); both
// are numbered in that layer-major order. Everything else a split touches belongs to its own
// domain: the parent, its siblings of the same (partition, layer) list, the tokens after it.
// Residence does not change inside a frame in deferred mode (fetch / enforce_capacity run only on
// the eager path), so domains are independent apart from the two counters.
//
// The engine therefore settles the pending events of ALL domains at once, in waves:
//   wave: stage every pending event's pool (parent members, buffer, token) in one launch ->
//         split_two of every pool in one launch (counter PREDICTED from the other domains' event
//         counts) -> exact children statistics in one launch -> recursion (Eq. 5 on a child,
//         maintainer.cpp:232-236) as further sub-waves -> children installed (provisional ids
//         above every existing id, in creation order: the same order relations as the final ids)
//         -> one relaunch round of every such domain from its next token.
//   verify: when no domain has events left, the exact counter of every split_two follows from
//         the final event counts; a split whose predicted counter differs is recomputed with the
//         exact seed (one launch) and compared. If any assignment differs, that domain is rolled
//         back to the snapshot taken at its first event (device statistics, page counts and tail
//         fills of its (partition, layer) clusters; its speculative children freed) and settled
//         again with the corrected counts. The lowest failing domain is always exact on its next
//         pass, so the loop terminates.
//   commit: the host replays every domain in reference order -- outcome runs, events, final ids,
//         counters, LRU ticks (store.cpp:82-86, 139-141) -- exactly as the sequential path does,
//         then uploads the final cluster ids, partition lists and window-ring owners.
// The host state (Cluster objects, ticks, counters) is only touched at commit, so a rollback is a
// device-side restore plus a reset of the domain's wave record.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <numeric>

#include "context.hpp"
#include "kmeans.hpp"

namespace kvc {

namespace {

inline double tau_at(std::int64_t n, const kvc_cfg& c) {  // maintainer.cpp:11-14 (as context.cpp tau_of)
  return c.tau_min + (c.tau_max - c.tau_min) * std::exp(-static_cast<double>(n) / c.n0);
}

struct DBuf {  // growable device buffer
  void* p = nullptr;
  std::size_t cap = 0;
  // keep: the first `keep` bytes survive a growth (copied on the stream, which is synchronised)
  void ensure(std::size_t bytes, cudaStream_t st, std::size_t keep = 0) {
    if (bytes <= cap) return;
    static const bool log = [] {
      const char* e = std::getenv("KVC_WAVES_LOG");
      return e && e[0] == '1';
    }();
    if (log) std::fprintf(stderr, "[waves] device buffer growth %zu -> %zu bytes\n", cap, bytes);
    // 2x headroom: a growth (allocation + synchronisation) stays a rare event across frames
    std::size_t n = std::max<std::size_t>(bytes * 2, cap * 2);
    n = std::max<std::size_t>(n, 1 << 16);
    void* q = nullptr;
    KVC_CUDA(cudaMalloc(&q, n));
    if (p) {
      if (keep) KVC_CUDA(cudaMemcpyAsync(q, p, std::min(keep, cap), cudaMemcpyDeviceToDevice, st));
      KVC_CUDA(cudaStreamSynchronize(st));
      KVC_CUDA(cudaFree(p));
    }
    p = q;
    cap = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as(std::size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<std::uint8_t*>(p) + byte_off);
  }
};

struct HBuf {  // growable pinned host buffer (contents not kept)
  void* p = nullptr;
  std::size_t cap = 0;
  void ensure(std::size_t bytes, cudaStream_t st) {
    if (bytes <= cap) return;
    const std::size_t n = std::max<std::size_t>({bytes * 2, cap * 2, std::size_t{1} << 16});
    static const bool log = [] {
      const char* e = std::getenv("KVC_WAVES_LOG");
      return e && e[0] == '1';
    }();
    if (log) std::fprintf(stderr, "[waves] pinned buffer growth %zu -> %zu bytes\n", cap, bytes);
    if (p) {
      KVC_CUDA(cudaStreamSynchronize(st));
      KVC_CUDA(cudaFreeHost(p));
    }
    KVC_CUDA(cudaHostAlloc(&p, n, cudaHostAllocDefault));
    cap = n;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as(std::size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<std::uint8_t*>(p) + byte_off);
  }
};

// Packs several arrays into one pinned buffer and moves them in one H2D copy.
struct Upload {
  HBuf h;
  DBuf d;
  std::size_t used = 0;
  std::vector<std::pair<const void*, std::size_t>> parts;
  void reset() {
    used = 0;
    parts.clear();
  }
  std::size_t add(const void* src, std::size_t bytes) {
    const std::size_t off = (used + 15) & ~std::size_t{15};
    parts.emplace_back(src, bytes);
    used = off + bytes;
    return off;
  }
  cudaEvent_t copied = nullptr;  // the last H2D out of the pinned buffer
  // copies the parts (in add order) into the pinned buffer and sends them; returns device base.
  // The device copy is only read by kernels queued before the next send (stream order); the
  // pinned side must wait until the previous copy has left it.
  std::uint8_t* send(cudaStream_t st) {
    if (copied) KVC_CUDA(cudaEventSynchronize(copied));
    h.ensure(used, st);
    d.ensure(used, st);
    std::size_t off = 0;
    for (auto& pr : parts) {
      off = (off + 15) & ~std::size_t{15};
      if (pr.second) std::memcpy(h.as<std::uint8_t>(off), pr.first, pr.second);
      off += pr.second;
    }
    if (used) KVC_CUDA(cudaMemcpyAsync(d.p, h.p, used, cudaMemcpyHostToDevice, st));
    if (!copied) KVC_CUDA(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    KVC_CUDA(cudaEventRecord(copied, st));
    return static_cast<std::uint8_t*>(d.p);
  }
};

constexpr int kNoKid = -1;
inline int leaf_code(int i) { return -2 - i; }
inline bool is_leaf_code(int k) { return k <= -2; }
inline int leaf_of(int k) { return -2 - k; }

}  // namespace

struct Context::Waves {
  struct Op {  // one split_two call
    int ev = -1, depth = 0;
    std::vector<int> rows;  // pool rows (relative to the event's staged pool)
    std::uint64_t ctr = 0;  // the counter its k-means used
    std::int64_t ok_ctr = -1;  // a counter its result was verified for
    bool ok_swap = false;      // ... as the same partition with the two labels exchanged
    std::vector<std::int32_t> assign;
    int kids[2] = {kNoKid, kNoKid};  // op index, leaf_code(leaf), or kNoKid (empty group)
  };
  struct Leaf {
    std::vector<int> rows;
    std::int32_t slot = -1;
  };
  struct Event {
    int layer = 0, tok = 0, kind = 0;
    std::int32_t parent_slot = -1;
    std::int64_t row0 = 0;  // staged pool rows [row0, row0 + n)
    int n = 0;
    int root = -1;              // root op (splits) or leaf (seeds: leaf_code)
    std::vector<int> ops;       // DFS preorder = counter order
    std::vector<int> stack;     // ops still to run (top = next in preorder)
    std::vector<int> emitted;   // leaves in emission order (filled at the end of the event)
    std::uint64_t ctr0 = 0;     // predicted counter of the first op
  };
  struct Dom {
    bool active = false;  // has events this frame (snapshot taken)
    bool done = true;
    int cur = 0;          // next token to resolve
    int pend_tok = -1, pend_kind = 0;
    std::int32_t pend_slot = -1;
    bool pend_valid = false;  // a pending event not yet turned into an Event
    bool retry = false;   // relaunch from pend_tok without an event (stale residence)
    bool first_retry = false;
    int cur_ev = -1;      // the event being settled (its ops still to run count in predictions)
    int first_tok = -1, first_kind = 0;
    std::int32_t first_slot = -1;
    int snap0 = 0, snap_n = 0;
    std::vector<int> events;
    std::vector<std::int32_t> pl;     // speculative (partition, layer) slot list
    std::vector<std::int32_t> taken;  // leaf slots created by this pass
    int ops = 0, prev_ops = -1;
    std::uint64_t epoch = 0;
    bool tie = false;  // a relaunch decision of this pass was an exact tie broken by the id key
    bool restarted = false;  // rolled back and not finished since (its event count is uncertain)
  };
  std::vector<Op> ops;
  std::vector<Leaf> leaves;
  std::vector<Event> evs;
  std::vector<Dom> dom;
  // per-slot pool sizes during speculation (valid when stamp == the owning domain's epoch)
  std::vector<std::int64_t> sz;
  std::vector<std::uint64_t> sz_stamp;
  std::uint64_t epoch_next = 1;
  // device
  DBuf stage_k, stage_v, stage_f32;  // staged pools (kv dtype, f32), append-only within a frame
  std::int64_t rows_used = 0;
  DBuf snap;                          // slot snapshots
  std::int64_t snap_used = 0;
  DBuf km_scratch, km_out;            // k-means scratch / assign | meta | counts
  HBuf h_out;
  Upload up;
  std::int64_t prov_next = 0;
  // stats (cumulative; kvc_debug_wave_profile)
  double st[16] = {0};
};

void Context::waves_free() {
  if (!wv_) return;
  wv_->stage_k.release();
  wv_->stage_v.release();
  wv_->stage_f32.release();
  wv_->snap.release();
  wv_->km_scratch.release();
  wv_->km_out.release();
  wv_->h_out.release();
  wv_->up.h.release();
  wv_->up.d.release();
  if (wv_->up.copied) cudaEventDestroy(wv_->up.copied);
  delete wv_;
  wv_ = nullptr;
}

void Context::wave_profile(double* out, bool reset) {
  for (int i = 0; i < 13; ++i) out[i] = wv_ ? wv_->st[i] : 0.0;
  if (reset && wv_)
    for (double& x : wv_->st) x = 0.0;
}

// Replays device outcomes of domain l, tokens [t0, t1) (the outcome runs of run_inserts).
void Context::replay_runs(int l, std::int64_t frame_id, int T, int t0, int t1, std::int64_t* assigned) {
  const int ring_slot = ia_.ring_slot;
  const std::int32_t* evk = h_evk_ + static_cast<std::size_t>(l) * t_.tmax;
  const std::int32_t* evs = h_evs_ + static_cast<std::size_t>(l) * t_.tmax;
  std::int32_t* owner = ring_slot >= 0 ? &ring_owner_h_[(static_cast<std::size_t>(l) * t_.W + ring_slot) * t_.tmax] : nullptr;
  std::int64_t last_cid = -1;
  for (int t = t0; t < t1;) {
    const std::int32_t slot = evs[t];
    const std::int32_t kind = evk[t];
    int u = t + 1;
    if (kind != EV_DEFER)
      while (u < t1 && evs[u] == slot && evk[u] == kind) ++u;
    const int n = u - t;
    if (slot < 0 || static_cast<std::size_t>(slot) >= slot_id_.size() || slot_id_[static_cast<std::size_t>(slot)] < 0) {
      std::string m = "wave replay: outcome names an unknown slot: domain " + std::to_string(l) + " token " +
                      std::to_string(t) + " of [" + std::to_string(t0) + "," + std::to_string(t1) + ") slot " +
                      std::to_string(slot) + " kind " + std::to_string(kind);
      if (wv_ && static_cast<std::size_t>(l) < wv_->dom.size()) {
        const Waves::Dom& D = wv_->dom[static_cast<std::size_t>(l)];
        m += "; first event " + std::to_string(D.first_tok) + " kind " + std::to_string(D.first_kind) + " events:";
        for (int ei : D.events) {
          const Waves::Event& e = wv_->evs[static_cast<std::size_t>(ei)];
          m += " (tok " + std::to_string(e.tok) + " kind " + std::to_string(e.kind) + " parent " + std::to_string(e.parent_slot) + " leaves";
          for (int li : e.emitted) m += " " + std::to_string(wv_->leaves[static_cast<std::size_t>(li)].slot);
          m += ")";
        }
        m += " pl:";
        for (std::int32_t x : D.pl) m += " " + std::to_string(x);
      }
      fail(-11, m);
    }
    const std::int64_t cid = slot_id_[static_cast<std::size_t>(slot)];
    Cluster& c = *clusters_[static_cast<std::size_t>(cid)];
    mstats_[0] += n;
    c.stat_count += n;
    c.last_touch = std::max(c.last_touch, frame_id);
    if (cid != last_cid) {
      fc_pending_.push_back(cid);
      last_cid = cid;
    }
    if (owner) std::fill(owner + t, owner + u, slot);
    (kind == EV_ABSORB ? c.members : c.buffer).push_run(frame_id, t, n);
    device_entries_ += n;
    set_flag(cid, CF_TRACKED, true);
    tick_ += n;
    last_use_[static_cast<std::size_t>(cid)] = tick_ - 1;
    switch (kind) {
      case EV_ABSORB:
        if (is_host(cid)) c.device_tail += n;
        mstats_[1] += n;
        break;
      case EV_BUFJOIN:
        mstats_[3] += n;
        break;
      case EV_DEFER:
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
}

void Context::run_inserts_waves(std::int64_t frame_id, std::int64_t pid, int T, std::int64_t* assigned, bool launched) {
  using clk = std::chrono::steady_clock;
  auto us = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  const auto t_start = clk::now();
  if (!wv_) {
    wv_ = new Waves();
    // staging for a typical frame's pools up front (about one 1,000-member pool per domain)
    const std::size_t rows0 = static_cast<std::size_t>(L_) * 3072;
    const std::size_t rb0 = static_cast<std::size_t>(d_) * es_;
    wv_->stage_k.ensure(rows0 * rb0 / 2, st_);  // (ensure doubles: rows0 rows)
    wv_->stage_v.ensure(rows0 * rb0 / 2, st_);
    wv_->stage_f32.ensure(rows0 * d_ * 2, st_);
    wv_->km_scratch.ensure(rows0 * (2 * d_ + 3) * 4, st_);
    // snapshots of every domain's (partition, layer) clusters, the packed uploads and results
    wv_->snap.ensure(static_cast<std::size_t>(L_) * 192 * slot_snap_bytes(d_), st_);
    wv_->up.h.ensure(std::size_t{2} << 20, st_);
    wv_->up.d.ensure(std::size_t{2} << 20, st_);
    wv_->km_out.ensure(std::size_t{2} << 20, st_);
    wv_->h_out.ensure(std::size_t{2} << 20, st_);
  }
  Waves& W = *wv_;
  if (spec_.active) {
    KVC_CUDA(cudaEventSynchronize(spec_.ev));
    spec_.active = false;
  }
  ia_.T = T;
  ia_.pid = static_cast<std::int32_t>(pid);
  const int ring_slot = ia_.ring_slot;
  for (double& x : ingest_t_) x = 0.0;
  double t_wait = 0.0;

  // ---- the first round (all domains from token 0)
  if (launched) {
    KVC_CUDA(cudaEventSynchronize(ping_wait_));
  } else {
    std::vector<int> all(static_cast<std::size_t>(L_)), zero(static_cast<std::size_t>(L_), 0);
    std::iota(all.begin(), all.end(), 0);
    launch_round(all, zero);
    const auto w0 = clk::now();
    sync();
    t_wait += us(w0, clk::now());
  }
  check_err_word(*h_err_);
  if (round_timed_) {
    float ms = 0.f;
    for (int i = 0; i < 5; ++i) {
      KVC_CUDA(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]));
      ingest_t_[i] += ms * 1e3;
    }
  }

  W.ops.clear();
  W.leaves.clear();
  W.evs.clear();
  W.dom.assign(static_cast<std::size_t>(L_), Waves::Dom{});
  W.rows_used = 0;
  W.snap_used = 0;
  if (W.sz.size() < slot_id_.size()) {
    W.sz.resize(slot_id_.size(), 0);
    W.sz_stamp.resize(slot_id_.size(), 0);
  }
  const std::uint64_t ctr_base = static_cast<std::uint64_t>(split_counter_);
  W.prov_next = std::int64_t{1} << 40;

  auto size_of = [&](std::int32_t slot, Waves::Dom& D) -> std::int64_t& {
    const std::size_t s = static_cast<std::size_t>(slot);
    if (W.sz_stamp[s] != D.epoch) {
      W.sz_stamp[s] = D.epoch;
      const std::int64_t cid = slot_id_[s];
      W.sz[s] = cid >= 0 && clusters_[static_cast<std::size_t>(cid)]
                    ? static_cast<std::int64_t>(clusters_[static_cast<std::size_t>(cid)]->members.size() +
                                                clusters_[static_cast<std::size_t>(cid)]->buffer.size())
                    : 0;
    }
    return W.sz[s];
  };
  // counts the outcome of tokens [a, b) of domain l into the pool sizes
  auto count_outcome = [&](int l, int a, int b) {
    Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
    const std::int32_t* evs = h_evs_ + static_cast<std::size_t>(l) * t_.tmax;
    for (int t = a; t < b; ++t) size_of(evs[t], D) += 1;
  };
  auto host_slots = [&](int l) {
    std::vector<std::int32_t> v;
    const auto& ids = parts_[static_cast<std::size_t>(pid)].per_layer[static_cast<std::size_t>(l)];
    v.reserve(ids.size());
    for (std::int64_t id : ids) v.push_back(C(id).slot);
    return v;
  };
  // a stop reported by a round for domain l
  auto take_stop = [&](int l) {
    Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
    const int stop = h_stop_[l];
    count_outcome(l, D.cur, std::min(stop, T));
    if (stop >= T) {
      D.done = true;
      D.restarted = false;
      D.cur = T;
      return;
    }
    D.done = false;
    D.cur = stop;
    D.pend_tok = stop;
    D.pend_kind = h_stop_[L_ + l];
    D.pend_slot = h_stop_[2 * L_ + l];
    D.retry = false;
    D.pend_valid = true;
    if (D.pend_kind == EV_EAGER) fail(-11, "wave engine: eager event in deferred mode");
    if (D.pend_kind == EV_SPLIT && is_host(slot_id_[static_cast<std::size_t>(D.pend_slot)])) {
      // the pipelined launch decided with the residence before the previous frame's cadence
      // offloaded the cluster (residence only turns Device -> Host between frames): nothing of
      // this token was committed; resolve the domain again from it
      D.retry = true;
      D.pend_valid = false;
    }
    if (D.pend_kind != EV_SEED && D.pend_kind != EV_SPLIT) fail(-11, "wave engine: unexpected host event");
  };

  // ---- domains with events after the first round: snapshot their (partition, layer) clusters
  std::vector<std::int32_t> snap_slots;
  bool any_events = false;
  for (int l = 0; l < L_; ++l) {
    Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
    D.epoch = W.epoch_next++;
    D.cur = 0;
    take_stop(l);
    if (D.done) continue;
    D.active = true;
    any_events = true;
    D.first_tok = D.pend_tok;
    D.first_kind = D.pend_kind;
    D.first_slot = D.pend_slot;
    D.first_retry = D.retry;
    D.pl = host_slots(l);
    D.snap0 = static_cast<int>(snap_slots.size());
    D.snap_n = static_cast<int>(D.pl.size());
    snap_slots.insert(snap_slots.end(), D.pl.begin(), D.pl.end());
  }
  if (!any_events) {  // no host events: plain replay
    for (int l = 0; l < L_; ++l) replay_runs(l, frame_id, T, 0, T, assigned);
    frame_add_flush(frame_id);
    ingest_t_[5] = t_wait;
    ingest_t_[6] = us(t_start, clk::now()) - t_wait;
    return;
  }
  const std::size_t snap_rb = slot_snap_bytes(d_);
  W.snap.ensure(snap_slots.size() * snap_rb, st_);
  if (!snap_slots.empty()) {
    W.up.reset();
    const std::size_t o = W.up.add(snap_slots.data(), snap_slots.size() * 4);
    std::uint8_t* db = W.up.send(st_);
    launches_ += launch_snap_slots(t_, reinterpret_cast<const std::int32_t*>(db + o), static_cast<std::int32_t>(snap_slots.size()),
                                   W.snap.p, st_);
  }
  W.st[0] += 1;  // frames with events

  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  const std::int64_t frame_rows = static_cast<std::int64_t>(L_) * t_.tmax;
  double t_stage = 0, t_km = 0, t_stats = 0, t_inst = 0, t_relaunch = 0, t_verify = 0;

  int passes = 1;  // 1 + waves whose validation rolled domains back
  // predicted counter of the next op of domain l
  auto predict = [&](int l) -> std::uint64_t {
    std::uint64_t c = ctr_base;
    for (int k = 0; k < l; ++k) {
      const Waves::Dom& E = W.dom[static_cast<std::size_t>(k)];
      if (!E.active) continue;
      std::int64_t est = E.ops;
      if (!E.done) {
        std::int64_t left = E.pend_valid && E.pend_kind == EV_SPLIT ? 1 : 0;
        if (E.cur_ev >= 0) left += static_cast<std::int64_t>(W.evs[static_cast<std::size_t>(E.cur_ev)].stack.size());
        est = std::max<std::int64_t>(E.ops + left, E.prev_ops);
      }
      c += static_cast<std::uint64_t>(est);
    }
    // test hook (KVC_WAVES_PERTURB=1): every first-pass prediction is wrong, so every split is
    // re-verified and (almost) every domain with events is rolled back and settled again
    if (waves_perturb_ && W.dom[static_cast<std::size_t>(l)].prev_ops < 0) c += 7;
    return c + static_cast<std::uint64_t>(W.dom[static_cast<std::size_t>(l)].ops);
  };

  // One launch of split jobs (k_split_two_batch): k-means of an op's pool rows with the seed of
  // `ctr` (or the labels `given`), and, for jobs with slots, its two groups' Eq. 1/2 statistics
  // installed into those slots with their variances returned.
  struct Job {
    int op = -1;                       // op whose rows are used (or -1: a seed's single row)
    int ev = -1;                       // event (row base) when op < 0
    std::uint64_t ctr = 0;
    std::int32_t slot[2] = {-1, -1};
    bool want_var = false;
    const std::vector<std::int32_t>* given = nullptr;
    // results
    std::vector<std::int32_t> assign;
    double var[2] = {0.0, 0.0};
  };
  const std::vector<int> one_row = {0};
  const std::vector<std::int32_t> label0 = {0};
  auto run_jobs = [&](std::vector<Job>& jobs) {
    const auto k0 = clk::now();
    const std::size_t nj = jobs.size();
    if (nj == 0) return 0.0;
    std::vector<std::int32_t> idx, given;
    std::vector<std::size_t> idx_off(nj), scr_off(nj), out_off(nj), giv_off(nj, 0);
    std::size_t scr = 0, outw = 0;
    for (std::size_t j = 0; j < nj; ++j) {
      const Job& J = jobs[j];
      const std::vector<int>& rows = J.op >= 0 ? W.ops[static_cast<std::size_t>(J.op)].rows : one_row;
      const Waves::Event& e = W.evs[static_cast<std::size_t>(J.op >= 0 ? W.ops[static_cast<std::size_t>(J.op)].ev : J.ev)];
      idx_off[j] = idx.size();
      for (int r : rows) idx.push_back(static_cast<std::int32_t>(e.row0 + r));
      scr_off[j] = scr;
      scr += ((rows.size() * (2 * static_cast<std::size_t>(d_) + 3) + 2) * 8 + 15) & ~std::size_t{15};  // 16-byte rows
      out_off[j] = outw;
      outw += rows.size() + 4;
      if (J.given) {
        giv_off[j] = given.size();
        given.insert(given.end(), J.given->begin(), J.given->end());
      }
    }
    W.km_scratch.ensure(scr, st_);
    const std::size_t var_off = (outw * 4 + 7) & ~std::size_t{7};
    const std::size_t obj_off = var_off + nj * 16;
    W.km_out.ensure(obj_off + nj * 8 + 64, st_);
    std::vector<SplitJob> sj(nj);
    std::int32_t* dout = W.km_out.as<std::int32_t>();
    W.up.reset();
    const std::size_t o_idx = W.up.add(idx.data(), idx.size() * 4);
    const std::size_t o_giv = W.up.add(given.data(), given.size() * 4);
    const std::size_t o_jobs = W.up.add(sj.data(), nj * sizeof(SplitJob));  // filled below
    // the jobs point into the uploaded arrays: size the device side first, then fill them
    W.up.h.ensure(W.up.used, st_);
    W.up.d.ensure(W.up.used, st_);
    std::uint8_t* dbase = static_cast<std::uint8_t*>(W.up.d.p);
    for (std::size_t j = 0; j < nj; ++j) {
      const Job& J = jobs[j];
      const int n = static_cast<int>(J.op >= 0 ? W.ops[static_cast<std::size_t>(J.op)].rows.size() : 1);
      SplitJob& X = sj[j];
      X.rows = W.stage_f32.as<float>();
      X.idx = reinterpret_cast<const std::int32_t*>(dbase + o_idx) + idx_off[j];
      X.scratch = W.km_scratch.as<double>(scr_off[j]);
      X.assign = dout + out_off[j];
      X.meta = dout + out_off[j] + n;
      X.objective = W.km_out.as<double>(obj_off) + j;
      X.n = n;
      X.slot[0] = J.slot[0];
      X.slot[1] = J.slot[1];
      X.var_out = (J.want_var || J.slot[0] >= 0 || J.slot[1] >= 0) ? W.km_out.as<double>(var_off) + 2 * j : nullptr;
      X.assign_in = J.given ? reinterpret_cast<const std::int32_t*>(dbase + o_giv) + giv_off[j] : nullptr;
      if (!J.given) {  // Rng64::index then Rng64::uniform (rng.hpp:14-44) from the first two draws
        std::uint64_t r2[2];
        mt64_first2(mix_seed(maint_seed_, J.ctr), r2);
        X.first = static_cast<std::int32_t>(r2[0] % static_cast<std::uint64_t>(n));
        X.uni = static_cast<double>(r2[1] >> 11) * 0x1.0p-53;
      } else {
        X.first = 0;
        X.uni = 0.0;
      }
    }
    std::uint8_t* db = W.up.send(st_);
    static long long* sprof = [] {  // KVC_SPLIT_PROF=1: per-job phase clocks (development)
      const char* e = std::getenv("KVC_SPLIT_PROF");
      long long* p = nullptr;
      if (e && e[0] == '1') {
        KVC_CUDA(cudaMalloc(&p, 8192 * 16 * 8));
        split_prof_set(p);
      }
      return p;
    }();
    launches_ += launch_split_two_batch(t_, reinterpret_cast<const SplitJob*>(db + o_jobs), static_cast<int>(nj), d_, st_);
    W.h_out.ensure(obj_off, st_);
    KVC_CUDA(cudaMemcpyAsync(W.h_out.p, dout, obj_off, cudaMemcpyDeviceToHost, st_));
    sync();
    if (sprof && nj <= 8192) {
      std::vector<long long> pr(nj * 16);
      KVC_CUDA(cudaMemcpy(pr.data(), sprof, pr.size() * 8, cudaMemcpyDeviceToHost));
      std::size_t jm = 0;
      for (std::size_t j = 0; j < nj; ++j)
        if (!jobs[j].given && (jobs[jm].given || pr[j * 16 + 11] > pr[jm * 16 + 11])) jm = j;
      if (!jobs[jm].given) {
        std::string m = "[split-prof] jobs " + std::to_string(nj) + " max-n job:";
        for (int k = 0; k < 12; ++k) m += " " + std::to_string(pr[jm * 16 + k]);
        std::fprintf(stderr, "%s\n", m.c_str());
      }
    }
    if (waves_log_) {
      std::size_t nmax = 0, nsum = 0;
      int itmax = 0;
      for (std::size_t j = 0; j < nj; ++j) {
        const std::size_t n = jobs[j].op >= 0 ? W.ops[static_cast<std::size_t>(jobs[j].op)].rows.size() : 1;
        nmax = std::max(nmax, n);
        nsum += n;
        itmax = std::max(itmax, W.h_out.as<std::int32_t>()[out_off[j] + n + 1]);
      }
      std::fprintf(stderr, "[waves] jobs %zu rows max %zu mean %.0f iters max %d: %.0f us\n", nj, nmax,
                   static_cast<double>(nsum) / static_cast<double>(nj), itmax, us(k0, clk::now()));
    }
    for (std::size_t j = 0; j < nj; ++j) {
      Job& J = jobs[j];
      const std::size_t n = J.op >= 0 ? W.ops[static_cast<std::size_t>(J.op)].rows.size() : 1;
      const std::int32_t* a = W.h_out.as<std::int32_t>() + out_off[j];
      if (a[n + 3] != 0) fail(-2, "normalize of zero vector");
      J.assign.assign(a, a + n);
      J.var[0] = W.h_out.as<double>(var_off)[2 * j];
      J.var[1] = W.h_out.as<double>(var_off)[2 * j + 1];
      if (!J.given) W.st[7] += 1;  // k-means jobs
    }
    return us(k0, clk::now());
  };

  // ---------------------------------------------------------------- the wave loop
  // Each iteration: (1) a validation sweep over the prefix of finished domains, where the split
  // counters are exact: every split whose k-means ran with another counter is recomputed with the
  // exact one (in the same launch as this wave's new splits); a domain whose result changes is
  // rolled back to its first event and restarted in this same wave, its first split taking the
  // exact result just computed. (2) The pending events of all unfinished domains are settled
  // (staging, k-means, children statistics, recursion as sub-waves, install) and (3) their domains
  // relaunched from the next token in one round.
  std::vector<std::uint64_t> first_ctr(static_cast<std::size_t>(L_), 0);
  // restart of a rolled-back domain: its first event again, with the staged pool of the previous
  // attempt (the snapshot restores exactly the state it was staged from) and, for a split, the
  // k-means result for the exact counter
  struct Prefab {
    bool on = false;
    std::int64_t row0 = 0;
    int n = 0;
    std::uint64_t ctr = 0;
    std::vector<std::int32_t> assign;
  };
  std::vector<Prefab> prefab(static_cast<std::size_t>(L_));
  auto new_event = [&](int l) -> int {
    Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
    Waves::Event e;
    e.layer = l;
    e.tok = D.pend_tok;
    e.kind = D.pend_kind;
    e.parent_slot = D.pend_kind == EV_SPLIT ? D.pend_slot : -1;
    e.n = e.kind == EV_SPLIT ? static_cast<int>(size_of(e.parent_slot, D)) + 1 : 1;
    e.row0 = -1;
    const int ei = static_cast<int>(W.evs.size());
    D.cur_ev = ei;
    D.pend_valid = false;
    D.events.push_back(ei);
    W.evs.push_back(std::move(e));
    return ei;
  };
  auto root_op = [&](int ei) {
    Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
    if (e.kind == EV_SEED) {
      Waves::Leaf lf;
      lf.rows = {0};
      W.leaves.push_back(std::move(lf));
      e.root = leaf_code(static_cast<int>(W.leaves.size()) - 1);
      return;
    }
    Waves::Op o;
    o.ev = ei;
    o.depth = 0;
    o.rows.resize(static_cast<std::size_t>(e.n));
    std::iota(o.rows.begin(), o.rows.end(), 0);
    W.ops.push_back(std::move(o));
    e.root = static_cast<int>(W.ops.size()) - 1;
    e.stack.push_back(e.root);
  };
  auto rollback = [&](const std::vector<int>& doms) {
    std::vector<std::int32_t> ridx, fslots;
    for (int l : doms) {
      Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
      for (int i = 0; i < D.snap_n; ++i) ridx.push_back(D.snap0 + i);
      fslots.insert(fslots.end(), D.taken.begin(), D.taken.end());
    }
    W.up.reset();
    const std::size_t o_f = W.up.add(fslots.data(), fslots.size() * 4);
    const std::size_t o_x = W.up.add(ridx.data(), ridx.size() * 4);
    std::uint8_t* db = W.up.send(st_);
    launches_ += launch_free_slots(t_, reinterpret_cast<const std::int32_t*>(db + o_f), static_cast<std::int32_t>(fslots.size()), st_);
    launches_ += launch_restore_slots(t_, reinterpret_cast<const std::int32_t*>(db + o_x), static_cast<std::int32_t>(ridx.size()),
                                      W.snap.p, st_);
    for (std::int32_t sl : fslots) free_slots_.push_back(sl);
    for (int l : doms) {
      Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
      D.prev_ops = D.ops;
      D.ops = 0;
      D.events.clear();
      D.taken.clear();
      D.tie = false;
      D.restarted = true;
      D.pl = host_slots(l);
      D.epoch = W.epoch_next++;
      D.cur = D.first_tok;
      D.done = false;
      D.pend_tok = D.first_tok;
      D.pend_kind = D.first_kind;
      D.pend_slot = D.first_slot;
      D.retry = D.first_retry;
      D.pend_valid = !D.retry;
      D.cur_ev = -1;
      count_outcome(l, 0, D.first_tok);
    }
  };

  for (;;) {
    // ---- (1) validation sweep
    const auto v0 = clk::now();
    std::vector<int> chk;
    std::vector<std::uint64_t> chk_ctr;
    bool any_undone = false;
    {
      // exact over the prefix of finished domains; past the first unfinished one the counters are
      // the current best prediction (an unfinished domain counts as predict() counts it), so a
      // finished domain whose split ran with a counter that is now predicted wrong is corrected
      // (recomputed and, if its result changes, restarted) without waiting for the domains before
      // it to finish; the final sweep, with every domain finished, is exact
      std::uint64_t c = ctr_base;
      bool uncertain = false;
      for (int l = 0; l < L_; ++l) {
        const Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
        if (!D.active) continue;
        if (!D.done) {
          any_undone = true;
          // past a restarted domain the counters move with its new event count: wait for it
          // (KVC_WAVES_EAGER=1 predicts through it as through any unfinished domain)
          if (D.restarted && !waves_eager_) uncertain = true;
          std::int64_t left = D.pend_valid && D.pend_kind == EV_SPLIT ? 1 : 0;
          if (D.cur_ev >= 0) left += static_cast<std::int64_t>(W.evs[static_cast<std::size_t>(D.cur_ev)].stack.size());
          c += static_cast<std::uint64_t>(std::max<std::int64_t>(D.ops + left, D.prev_ops));
          continue;
        }
        if (uncertain) continue;
        first_ctr[static_cast<std::size_t>(l)] = c;
        for (int ei : D.events)
          for (int oi : W.evs[static_cast<std::size_t>(ei)].ops) {
            const Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
            if (o.ctr != c && o.ok_ctr != static_cast<std::int64_t>(c)) {
              chk.push_back(oi);
              chk_ctr.push_back(c);
            }
            ++c;
          }
      }
    }
    t_verify += us(v0, clk::now());
    if (!any_undone && chk.empty()) break;
    // ---- (2) this wave's events
    std::vector<int> relaunch, rcur, new_evs;
    for (int l = 0; l < L_; ++l) {
      Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
      if (!D.active || D.done) continue;
      if (D.retry) {
        relaunch.push_back(l);
        rcur.push_back(D.pend_tok);
        D.cur = D.pend_tok;
        D.retry = false;
        continue;
      }
      if (D.pend_valid) new_evs.push_back(new_event(l));
    }
    W.st[1] += 1;  // waves
    const auto s0 = clk::now();
    // stage the new pools
    auto stage = [&](const std::vector<int>& evl) {
      std::vector<GatherJob> gj;
      std::vector<int> staged;
      std::int64_t rows_need = W.rows_used;
      for (int ei : evl) {
        Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
        if (e.row0 >= 0) continue;  // reused
        e.row0 = rows_need;
        rows_need += e.n;
        staged.push_back(ei);
      }
      if (staged.empty()) return;
      const std::int64_t keep_rows = W.rows_used;
      W.stage_k.ensure(static_cast<std::size_t>(rows_need) * rb, st_, static_cast<std::size_t>(keep_rows) * rb);
      W.stage_v.ensure(static_cast<std::size_t>(rows_need) * rb, st_, static_cast<std::size_t>(keep_rows) * rb);
      W.stage_f32.ensure(static_cast<std::size_t>(rows_need) * d_ * 4, st_, static_cast<std::size_t>(keep_rows) * d_ * 4);
      W.rows_used = rows_need;
      W.km_out.ensure(staged.size() * 4 + 64, st_);
      for (std::size_t i = 0; i < staged.size(); ++i) {
        const Waves::Event& e = W.evs[static_cast<std::size_t>(staged[i])];
        GatherJob g{};
        g.slot = e.parent_slot;
        g.with_buf = 1;
        g.row0 = e.row0;
        g.frame_row = static_cast<std::int64_t>(e.layer) * t_.tmax + e.tok;
        g.count_out = W.km_out.as<std::int32_t>() + i;
        gj.push_back(g);
      }
      W.up.reset();
      const std::size_t o = W.up.add(gj.data(), gj.size() * sizeof(GatherJob));
      std::uint8_t* db = W.up.send(st_);
      launches_ += launch_gather_batch(t_, reinterpret_cast<const GatherJob*>(db + o), static_cast<std::int32_t>(gj.size()),
                                       d_fk_, d_fv_, W.stage_k.p, W.stage_v.p, st_);
      launches_ += launch_to_f32(t_, W.stage_k.as<std::uint8_t>(static_cast<std::size_t>(keep_rows) * rb),
                                 W.stage_f32.as<float>(static_cast<std::size_t>(keep_rows) * d_ * 4),
                                 (rows_need - keep_rows) * d_, st_);
      W.h_out.ensure(gj.size() * 4, st_);
      KVC_CUDA(cudaMemcpyAsync(W.h_out.p, W.km_out.p, gj.size() * 4, cudaMemcpyDeviceToHost, st_));
      sync();
      for (std::size_t i = 0; i < staged.size(); ++i)
        if (W.h_out.as<std::int32_t>()[i] != W.evs[static_cast<std::size_t>(staged[i])].n)
          fail(-11, "wave engine: staged pool size differs from the host's count");
    };
    stage(new_evs);
    t_stage += us(s0, clk::now());
    for (int ei : new_evs) root_op(ei);
    // ---- sub-waves: one op per event at a time, in DFS preorder (its counter order); the first
    // also carries the validation sweep's recomputations and the seeds' statistics
    std::vector<int> seed_evs;  // events whose root is a seed leaf
    for (int ei : new_evs)
      if (is_leaf_code(W.evs[static_cast<std::size_t>(ei)].root)) seed_evs.push_back(ei);
    bool first_sub = true;
    for (;;) {
      std::vector<Job> jobs;
      std::vector<int> settled;  // ops whose groups are decided this sub-wave (jobs[0 .. n_settle))
      for (int ei : new_evs) {
        Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
        if (e.stack.empty()) continue;
        const int oi = e.stack.back();
        e.stack.pop_back();
        Waves::Dom& D = W.dom[static_cast<std::size_t>(e.layer)];
        Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
        o.ctr = predict(e.layer);
        D.ops += 1;
        e.ops.push_back(oi);
        settled.push_back(oi);
        Job J;
        J.op = oi;
        J.ctr = o.ctr;
        J.slot[0] = take_slot();
        J.slot[1] = take_slot();
        jobs.push_back(std::move(J));
      }
      const std::size_t n_settle = jobs.size();
      auto add_seed_jobs = [&](const std::vector<int>& evl) {
        for (int ei : evl) {
          const Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
          Waves::Leaf& lf = W.leaves[static_cast<std::size_t>(leaf_of(e.root))];
          lf.slot = take_slot();
          W.dom[static_cast<std::size_t>(e.layer)].taken.push_back(lf.slot);
          Job J;
          J.ev = ei;
          J.slot[0] = lf.slot;
          J.given = &label0;
          jobs.push_back(std::move(J));
        }
      };
      if (first_sub) {
        add_seed_jobs(seed_evs);
        for (std::size_t j = 0; j < chk.size(); ++j) {
          Job J;
          J.op = chk[j];
          J.ctr = chk_ctr[j];
          jobs.push_back(std::move(J));
        }
      }
      if (jobs.empty()) break;
      t_km += run_jobs(jobs);
      const std::size_t chk0 = jobs.size() - (first_sub ? chk.size() : 0);
      for (std::size_t j = 0; j < n_settle; ++j) W.ops[static_cast<std::size_t>(settled[j])].assign = jobs[j].assign;
      std::vector<Job> done_jobs(jobs.begin(), jobs.begin() + static_cast<std::ptrdiff_t>(n_settle));
      if (first_sub && !chk.empty()) {
        // ---- validation results: failing domains are rolled back and restarted in this wave
        const auto c0 = clk::now();
        W.st[4] += static_cast<double>(chk.size());
        std::vector<int> bad_dom;
        std::vector<std::vector<std::int32_t>> exact_first(static_cast<std::size_t>(L_));
        for (std::size_t j = 0; j < chk.size(); ++j) {
          std::vector<std::int32_t>& r = jobs[chk0 + j].assign;
          Waves::Op& o = W.ops[static_cast<std::size_t>(chk[j])];
          const int l = W.evs[static_cast<std::size_t>(o.ev)].layer;
          const Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
          const bool is_first = !D.events.empty() && W.evs[static_cast<std::size_t>(D.events.front())].root == chk[j];
          // the same two groups with the labels exchanged: only the children's emission order (and
          // so their ids) changes. Valid when neither group was split further (the sub-splits'
          // counters would follow the other order) and no relaunch decision of the domain was a
          // tie broken by the provisional ids (every other decision is order-independent).
          bool swapped = !D.tie && is_leaf_code(o.kids[0]) && is_leaf_code(o.kids[1]) && r.size() == o.assign.size();
          for (std::size_t i = 0; swapped && i < r.size(); ++i) swapped = r[i] == 1 - o.assign[i];
          if (r == o.assign || swapped) {
            o.ok_ctr = static_cast<std::int64_t>(chk_ctr[j]);
            o.ok_swap = swapped;
            W.st[12] += swapped ? 1 : 0;
          } else if (bad_dom.empty() || bad_dom.back() != l) {
            bad_dom.push_back(l);
          }
          if (is_first) exact_first[static_cast<std::size_t>(l)] = std::move(r);
        }
        if (!bad_dom.empty()) {
          passes += 1;
          W.st[3] += static_cast<double>(bad_dom.size());
          if (waves_log_) {
            std::string m = "[waves] frame " + std::to_string(frame_id) + " wave " + std::to_string(W.st[1]) + " checked " +
                            std::to_string(chk.size()) + " failed domains " + std::to_string(bad_dom.size()) + ":";
            for (int l : bad_dom) {
              const Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
              m += " " + std::to_string(l) + "(ops " + std::to_string(D.ops) + " prev " + std::to_string(D.prev_ops) + ")";
            }
            std::fprintf(stderr, "%s\n", m.c_str());
          }
          // the exact result of each failing domain's first split (for its restart)
          for (int l : bad_dom) {
            Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
            Prefab& pf = prefab[static_cast<std::size_t>(l)];
            pf = Prefab{};
            const Waves::Event& e1 = W.evs[static_cast<std::size_t>(D.events.front())];
            pf.row0 = e1.row0;
            pf.n = e1.n;
            if (e1.kind != EV_SPLIT) continue;
            const Waves::Op& o1 = W.ops[static_cast<std::size_t>(e1.root)];
            const std::uint64_t c1 = first_ctr[static_cast<std::size_t>(l)];
            pf.on = true;
            pf.ctr = c1;
            if (!exact_first[static_cast<std::size_t>(l)].empty()) {
              pf.assign = exact_first[static_cast<std::size_t>(l)];
            } else {
              pf.assign = o1.assign;
              if (o1.ctr != c1 && o1.ok_swap)
                for (std::int32_t& a : pf.assign) a = 1 - a;
            }
          }
          rollback(bad_dom);
          // restart: first event again (pool reused), its root split from the exact result; the
          // restarted splits' (and seeds') statistics in one more launch
          std::vector<Job> rj;
          std::vector<int> restart_seeds;
          for (int l : bad_dom) {
            Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
            if (D.retry) {  // the first stop was a stale-residence retry: relaunch it
              relaunch.push_back(l);
              rcur.push_back(D.pend_tok);
              D.cur = D.pend_tok;
              D.retry = false;
              continue;
            }
            const Prefab& pf = prefab[static_cast<std::size_t>(l)];
            const int ei = new_event(l);
            Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
            if (e.n != pf.n) fail(-11, "wave engine: restarted pool size differs");
            e.row0 = pf.row0;
            root_op(ei);
            new_evs.push_back(ei);
            if (is_leaf_code(e.root)) {
              restart_seeds.push_back(ei);
              continue;
            }
            Waves::Op& o = W.ops[static_cast<std::size_t>(e.root)];
            e.stack.pop_back();
            o.ctr = pf.ctr;
            o.assign = pf.assign;
            D.ops += 1;
            e.ops.push_back(e.root);
            settled.push_back(e.root);
            Job J;
            J.op = e.root;
            J.given = &prefab[static_cast<std::size_t>(l)].assign;
            J.slot[0] = take_slot();
            J.slot[1] = take_slot();
            rj.push_back(std::move(J));
          }
          const std::size_t n_rs = rj.size();
          std::swap(jobs, rj);
          add_seed_jobs(restart_seeds);
          if (!jobs.empty()) t_km += run_jobs(jobs);
          for (std::size_t j = 0; j < n_rs; ++j) done_jobs.push_back(std::move(jobs[j]));
        }
        t_verify += us(c0, clk::now());
      }
      first_sub = false;
      const auto st0 = clk::now();
      // groups (their statistics are installed in the jobs' slots) and the recursion decisions
      // (maintainer.cpp:228-238)
      for (std::size_t j = 0; j < settled.size(); ++j) {
        const int oi = settled[j];
        const Job& J = done_jobs[j];
        const int o_ev = W.ops[static_cast<std::size_t>(oi)].ev, o_depth = W.ops[static_cast<std::size_t>(oi)].depth;
        const int layer = W.evs[static_cast<std::size_t>(o_ev)].layer;
        std::vector<int> g2[2];
        {
          const Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
          for (std::size_t i = 0; i < o.rows.size(); ++i) g2[o.assign[i]].push_back(o.rows[i]);
        }
        for (int g = 0; g < 2; ++g) {
          if (g2[g].empty()) {
            free_slots_.push_back(J.slot[g]);
            continue;
          }
          const std::int64_t sz = static_cast<std::int64_t>(g2[g].size());
          if (o_depth + 1 < cfg_.max_split_depth && sz >= 2 && J.var[g] > tau_at(sz, cfg_)) {
            free_slots_.push_back(J.slot[g]);  // no pages were attached
            Waves::Op c;
            c.ev = o_ev;
            c.depth = o_depth + 1;
            c.rows = std::move(g2[g]);
            W.ops.push_back(std::move(c));
            W.ops[static_cast<std::size_t>(oi)].kids[g] = static_cast<int>(W.ops.size()) - 1;
          } else {
            Waves::Leaf lf;
            lf.rows = std::move(g2[g]);
            lf.slot = J.slot[g];
            W.leaves.push_back(std::move(lf));
            W.ops[static_cast<std::size_t>(oi)].kids[g] = leaf_code(static_cast<int>(W.leaves.size()) - 1);
            W.dom[static_cast<std::size_t>(layer)].taken.push_back(J.slot[g]);
          }
        }
      }
      // children to run: push kid 1 first so kid 0 (its subtree) runs first (preorder)
      for (int oi : settled) {
        const Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
        Waves::Event& e = W.evs[static_cast<std::size_t>(o.ev)];
        for (int g = 1; g >= 0; --g)
          if (o.kids[g] >= 0) e.stack.push_back(o.kids[g]);
      }
      t_stats += us(st0, clk::now());
    }
    // ---- install children: headers, pages, partition lists; relaunch the domains
    const auto i0 = clk::now();
    std::vector<SlotHeader> hd;
    std::vector<AppendRun> runs;
    std::vector<std::int32_t> idx;
    for (int ei : new_evs) {
      Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
      Waves::Dom& D = W.dom[static_cast<std::size_t>(e.layer)];
      if (D.events.empty() || std::find(D.events.begin(), D.events.end(), ei) == D.events.end())
        continue;  // an event of an attempt rolled back in this wave
      // emission order: in-order over the split tree (maintainer.cpp:224-238)
      if (is_leaf_code(e.root)) {
        e.emitted.push_back(leaf_of(e.root));
      } else {
        auto walk = [&](auto&& self, int oi) -> void {
          const Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
          for (int g = 0; g < 2; ++g) {
            if (o.kids[g] == kNoKid) continue;
            if (is_leaf_code(o.kids[g]))
              e.emitted.push_back(leaf_of(o.kids[g]));
            else
              self(self, o.kids[g]);
          }
        };
        walk(walk, e.root);
      }
      if (e.kind == EV_SPLIT) D.pl.erase(std::remove(D.pl.begin(), D.pl.end(), e.parent_slot), D.pl.end());
      for (int li : e.emitted) {
        const Waves::Leaf& lf = W.leaves[static_cast<std::size_t>(li)];
        const std::int64_t n = static_cast<std::int64_t>(lf.rows.size());
        hd.push_back({lf.slot, 0, W.prov_next++, n});
        runs.push_back({lf.slot, static_cast<std::int32_t>(idx.size()), static_cast<std::int32_t>(n), 0});
        for (int r : lf.rows) idx.push_back(static_cast<std::int32_t>(e.row0 + r));
        D.pl.push_back(lf.slot);
        W.sz_stamp[static_cast<std::size_t>(lf.slot)] = D.epoch;
        W.sz[static_cast<std::size_t>(lf.slot)] = n;
      }
      D.cur = e.tok + 1;
      D.cur_ev = -1;
      if (D.cur >= T) {
        D.done = true;
        D.restarted = false;
      } else {
        relaunch.push_back(e.layer);
        rcur.push_back(D.cur);
      }
    }
    // partition lists of every domain in speculation (capacity first: a compaction rewrites
    // the device lists from the host ones)
    std::vector<std::int32_t> plrec, ploff;
    pl_floor_.assign(parts_.size() * static_cast<std::size_t>(L_), 0);
    for (int l = 0; l < L_; ++l)
      if (W.dom[static_cast<std::size_t>(l)].active)
        pl_floor_[static_cast<std::size_t>(pid) * L_ + l] = static_cast<std::int32_t>(W.dom[static_cast<std::size_t>(l)].pl.size());
    for (int l = 0; l < L_; ++l)
      if (W.dom[static_cast<std::size_t>(l)].active)
        pl_reserve(pid, l, static_cast<std::int32_t>(W.dom[static_cast<std::size_t>(l)].pl.size()));
    pl_floor_.clear();
    for (int l = 0; l < L_; ++l) {
      const Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
      if (!D.active) continue;
      ploff.push_back(static_cast<std::int32_t>(plrec.size()));
      plrec.push_back(static_cast<std::int32_t>(pid * L_ + l));
      plrec.push_back(parts_[static_cast<std::size_t>(pid)].dev_off[static_cast<std::size_t>(l)]);
      plrec.push_back(static_cast<std::int32_t>(D.pl.size()));
      plrec.insert(plrec.end(), D.pl.begin(), D.pl.end());
    }
    W.up.reset();
    const std::size_t o_h = W.up.add(hd.data(), hd.size() * sizeof(SlotHeader));
    const std::size_t o_r = W.up.add(runs.data(), runs.size() * sizeof(AppendRun));
    const std::size_t o_i = W.up.add(idx.data(), idx.size() * 4);
    const std::size_t o_p = W.up.add(plrec.data(), plrec.size() * 4);
    const std::size_t o_q = W.up.add(ploff.data(), ploff.size() * 4);
    std::uint8_t* db = W.up.send(st_);
    launches_ += launch_slot_headers(t_, reinterpret_cast<const SlotHeader*>(db + o_h), static_cast<std::int32_t>(hd.size()), st_);
    launches_ += launch_append_runs(t_, reinterpret_cast<const AppendRun*>(db + o_r), static_cast<std::int32_t>(runs.size()),
                                    reinterpret_cast<const std::int32_t*>(db + o_i), W.stage_k.p, W.stage_v.p, st_);
    launches_ += launch_pl_scatter(t_, reinterpret_cast<const std::int32_t*>(db + o_p), reinterpret_cast<const std::int32_t*>(db + o_q),
                                   static_cast<std::int32_t>(ploff.size()), st_);
    t_inst += us(i0, clk::now());
    // ---- relaunch
    if (!relaunch.empty()) {
      const auto r0 = clk::now();
      std::vector<int> cursor(static_cast<std::size_t>(L_), 0);
      for (std::size_t i = 0; i < relaunch.size(); ++i) cursor[static_cast<std::size_t>(relaunch[i])] = rcur[i];
      round_after_event_ = true;
      launch_round(relaunch, cursor);
      round_after_event_ = false;
      sync();
      check_err_word(*h_err_);
      for (int l : relaunch) {  // (both resolve kernels report key-decided exact ties)
        W.dom[static_cast<std::size_t>(l)].tie |= h_err_[1 + l] != 0;
        take_stop(l);
      }
      if (waves_log_) {
        int cmin = T;
        for (int c : rcur) cmin = std::min(cmin, c);
        std::string kt;
        if (round_timed_) {  // (timing mode) the round's kernels: cands, tile, top-M, resolve, store
          for (int i = 0; i < 5; ++i) {
            float ms = 0.f;
            KVC_CUDA(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]));
            kt += " " + std::to_string(static_cast<int>(ms * 1e3));
          }
          kt = "; kernels us" + kt;
        }
        if (!relaunch_seq_) {  // the speculative kernel's rounds (prof[10]) over the relaunched domains
          std::vector<long long> pr(static_cast<std::size_t>(L_) * 16);
          KVC_CUDA(cudaMemcpy(pr.data(), ia_.prof, pr.size() * 8, cudaMemcpyDeviceToHost));
          long long mx = 0, sm = 0;
          for (int l : relaunch) {
            mx = std::max(mx, pr[static_cast<std::size_t>(l) * 16 + 10]);
            sm += pr[static_cast<std::size_t>(l) * 16 + 10];
          }
          kt += "; spec rounds max " + std::to_string(mx) + " mean " + std::to_string(sm / std::max<long long>(1, static_cast<long long>(relaunch.size())));
          long long best = -1;
          int bl = relaunch[0];
          for (int l : relaunch) {
            long long tot = 0;
            for (int k = 0; k < 10; ++k) tot += pr[static_cast<std::size_t>(l) * 16 + k];
            if (tot > best) {
              best = tot;
              bl = l;
            }
          }
          kt += "; slowest domain phases";
          for (int k = 0; k < 10; ++k) kt += " " + std::to_string(pr[static_cast<std::size_t>(bl) * 16 + k]);
        }
        std::fprintf(stderr, "[waves] relaunch %zu domains (first token %d, seq %d): %.0f us incl. install (install %.0f)%s\n",
                     relaunch.size(), cmin, relaunch_seq_ ? 1 : 0, us(i0, clk::now()), us(i0, r0), kt.c_str());
      }
      t_relaunch += us(r0, clk::now());
    } else {
      sync();
    }
  }
  W.st[2] += passes;
  if (waves_log_) {
    int act = 0, ops = 0, multi = 0;
    for (const Waves::Dom& D : W.dom) {
      act += D.active ? 1 : 0;
      ops += D.ops;
      multi += D.ops > 1 ? 1 : 0;
    }
    std::fprintf(stderr, "[waves] frame %lld done: passes %d, domains with events %d, ops %d, domains with >1 op %d\n",
                 static_cast<long long>(frame_id), passes, act, ops, multi);
  }

  // ---------------------------------------------------------------- commit in reference order
  const auto c0 = clk::now();
  std::vector<SlotCid> cids;
  std::vector<std::int32_t> parents;
  for (int l = 0; l < L_; ++l) {
    Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
    int t = 0;
    for (int ei : D.events) {
      const Waves::Event& e = W.evs[static_cast<std::size_t>(ei)];
      replay_runs(l, frame_id, T, t, e.tok, assigned);
      frame_add_flush(frame_id);  // host events add / remove map entries themselves
      mstats_[0] += 1;            // inserts (maintainer.cpp:89)
      evt_t_[6] += 1.0;
      W.st[5] += 1;
      std::vector<Member> ids;
      if (e.kind == EV_SPLIT) {
        const std::int64_t cid = slot_id_[static_cast<std::size_t>(e.parent_slot)];
        Cluster& c = C(cid);
        mstats_[2] += 1;  // immediate_splits
        ids.reserve(static_cast<std::size_t>(e.n));
        for (const Member& m : c.members) ids.push_back(m);
        for (const Member& m : c.buffer) ids.push_back(m);
        ids.push_back({frame_id, e.tok});
        if (static_cast<int>(ids.size()) != e.n) fail(-11, "wave commit: pool size mismatch");
        forget(cid);
        drop_cluster_host(cid);
        parents.push_back(e.parent_slot);
        for (int oi : e.ops) {
          Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
          const std::uint64_t ctr = static_cast<std::uint64_t>(split_counter_++);
          if (o.ctr == ctr) o.ok_swap = false;
          else if (o.ok_ctr != static_cast<std::int64_t>(ctr)) fail(-11, "wave commit: unverified split counter");
          mstats_[5] += 1;  // split_ops_total
          evt_t_[7] += 1.0;
        }
      } else {
        ids.push_back({frame_id, e.tok});
      }
      std::vector<int> emitted;  // the reference's emission order (labels as the exact seed gives them)
      if (is_leaf_code(e.root)) {
        emitted.push_back(leaf_of(e.root));
      } else {
        auto walk = [&](auto&& self, int oi) -> void {
          const Waves::Op& o = W.ops[static_cast<std::size_t>(oi)];
          for (int k = 0; k < 2; ++k) {
            const int g = o.ok_swap ? 1 - k : k;
            if (o.kids[g] == kNoKid) continue;
            if (is_leaf_code(o.kids[g]))
              emitted.push_back(leaf_of(o.kids[g]));
            else
              self(self, o.kids[g]);
          }
        };
        walk(walk, e.root);
      }
      std::int64_t home = -1;
      for (int li : emitted) {
        const Waves::Leaf& lf = W.leaves[static_cast<std::size_t>(li)];
        std::vector<Member> m;
        m.reserve(lf.rows.size());
        bool has_tok = false;
        for (int r : lf.rows) {
          m.push_back(ids[static_cast<std::size_t>(r)]);
          has_tok |= r == e.n - 1;
        }
        const std::int64_t id = new_cluster_at(lf.slot, l, pid, std::move(m), false);
        adopt(id);
        ring_owner_patch(l, C(id).members, lf.slot);
        cids.push_back({id, lf.slot, 0});
        if (has_tok && home < 0) home = id;  // home_of (maintainer.cpp:62-70)
      }
      if (home < 0) home = slot_id_[static_cast<std::size_t>(W.leaves[static_cast<std::size_t>(emitted.front())].slot)];
      if (assigned) assigned[static_cast<std::size_t>(l) * T + e.tok] = home;
      t = e.tok + 1;
    }
    replay_runs(l, frame_id, T, t, T, assigned);
  }
  frame_add_flush(frame_id);
  const auto c1 = clk::now();
  // device: final ids, released parents, final partition lists, window-ring owners
  std::vector<std::int32_t> plrec, ploff;
  for (int l = 0; l < L_; ++l) {
    const Waves::Dom& D = W.dom[static_cast<std::size_t>(l)];
    if (!D.active) continue;
    const auto& ids = parts_[static_cast<std::size_t>(pid)].per_layer[static_cast<std::size_t>(l)];
    pl_reserve(pid, l, static_cast<std::int32_t>(ids.size()));
    ploff.push_back(static_cast<std::int32_t>(plrec.size()));
    plrec.push_back(static_cast<std::int32_t>(pid * L_ + l));
    plrec.push_back(parts_[static_cast<std::size_t>(pid)].dev_off[static_cast<std::size_t>(l)]);
    plrec.push_back(static_cast<std::int32_t>(ids.size()));
    for (std::int64_t id : ids) plrec.push_back(C(id).slot);
  }
  const auto c2 = clk::now();
  W.up.reset();
  const std::size_t o_c = W.up.add(cids.data(), cids.size() * sizeof(SlotCid));
  const std::size_t o_f = W.up.add(parents.data(), parents.size() * 4);
  const std::size_t o_p = W.up.add(plrec.data(), plrec.size() * 4);
  const std::size_t o_q = W.up.add(ploff.data(), ploff.size() * 4);
  const std::size_t o_o = W.up.add(ring_owner_h_.data(), ring_owner_h_.size() * 4);
  std::uint8_t* db = W.up.send(st_);
  launches_ += launch_set_cids(t_, reinterpret_cast<const SlotCid*>(db + o_c), static_cast<std::int32_t>(cids.size()), st_);
  launches_ += launch_free_slots(t_, reinterpret_cast<const std::int32_t*>(db + o_f), static_cast<std::int32_t>(parents.size()), st_);
  launches_ += launch_pl_scatter(t_, reinterpret_cast<const std::int32_t*>(db + o_p), reinterpret_cast<const std::int32_t*>(db + o_q),
                                 static_cast<std::int32_t>(ploff.size()), st_);
  KVC_CUDA(cudaMemcpyAsync(t_.ring_owner, db + o_o, ring_owner_h_.size() * 4, cudaMemcpyDeviceToDevice, st_));
  for (std::int32_t s : parents) free_slots_.push_back(s);
  const auto c3 = clk::now();
  sync();  // the upload staging is reused by the next frame
  (void)ring_slot;
  const double t_commit = us(c0, clk::now());
  if (waves_log_)
    std::fprintf(stderr, "[waves] commit us: replay %.0f lists %.0f upload %.0f sync %.0f\n", us(c0, c1), us(c1, c2), us(c2, c3),
                 us(c3, clk::now()));
  if (waves_log_)
    std::fprintf(stderr, "[waves] frame %lld times us: stage %.0f kmeans %.0f stats %.0f install %.0f relaunch %.0f verify %.0f commit %.0f total %.0f\n",
                 static_cast<long long>(frame_id), t_stage, t_km, t_stats, t_inst, t_relaunch, t_verify, t_commit,
                 us(t_start, clk::now()));
  W.st[6] += t_stage;
  W.st[8] += t_km;
  W.st[9] += t_stats + t_inst;
  W.st[10] += t_relaunch;
  W.st[11] += t_verify + t_commit;
  evt_t_[0] += us(t_start, clk::now());
  evt_t_[1] += t_stage;
  evt_t_[2] += t_km;
  evt_t_[3] += t_stats;
  evt_t_[4] += t_inst + t_commit;
  evt_t_[5] += t_relaunch;
  ingest_t_[5] = t_wait;
  ingest_t_[6] = us(t_start, clk::now()) - t_wait;
  ingest_t_[9] = W.st[5];
}

}  // namespace kvc
