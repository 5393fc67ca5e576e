// context_query.cpp -- decode step (retrieve + attend), bulk load, views and self-checks.
//
// Reference semantics (paths under /root/reference/proj/core):
//   retrieval.cpp:45-143  retrieve(): per-layer rankings (computed on the GPU for all layers at
//                         once -- rankings depend only on representatives, which nothing in the
//                         per-layer loop changes for a later layer), then fetch / materialize /
//                         touch / latency bookkeeping replayed here in layer order.
//   retrieval.cpp:145-164 oracle_flat_topk
//   engine.cpp:176-237    answer_query: repin + checks after the query
//   index.cpp:263-343     check_invariants;  store.cpp:183-189 audit
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include "context.hpp"
#include "kmeans.hpp"

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

// Asynchronous step pipeline. decode_step(i) enqueues the scoring/selection and attention
// kernels of step i and the device->host copy of its result block, THEN replays the host
// bookkeeping of step i-1 (fetch / touch / materialize / latency model, retrieval.cpp:58-128)
// while the GPU runs step i, and returns without waiting for step i (outputs in device memory
// follow stream order on kvc_stream()). Step i's kernels read only the device index, which the
// bookkeeping of step i-1 changes only when it settles a pending split (the K4 flag): then step i
// is relaunched after the settle. Host outputs, parity / check / recall modes and per-step timing
// complete the step before returning.
// Device address of pinned (page-locked, mapped) host memory, or nullptr for pageable memory.
// Asked every step (a buffer may be freed and its address reused by pageable memory).
const void* Context::mapped_host(const void* p) {
  if (!p) return nullptr;
  static const bool off = std::getenv("KVC_NO_ZERO_COPY") != nullptr;
  if (off) return nullptr;
  cudaPointerAttributes at{};
  const void* dp = nullptr;
  const cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
    dp = at.devicePointer;
  else if (e != cudaSuccess)
    cudaGetLastError();  // clear only this query's own error (an unknown pointer is pageable memory)
  return dp;
}

void Context::launch_step(int b, const float* q, int q_mem, float* out, int out_mem) {
  if (blk_used_[b]) KVC_CUDA(cudaStreamWaitEvent(st_, ev_step_[b], 0));  // block b's last copy done
  blk_used_[b] = true;
  set_result_block(b);
  // Host query / output in pinned memory are used in place (zero-copy): K4 reads the query over
  // the link and leaves the device copy for K6, K6's combine writes the rows to the host; no
  // separate copies (and their launch latencies) on the critical path of an end-to-end step.
  const float* dq = q;
  da_.q_src = nullptr;
  const float* q_map = q_mem != KVC_MEM_DEVICE ? static_cast<const float*>(mapped_host(q)) : nullptr;
  float* out_map = (out && out_mem != KVC_MEM_DEVICE) ? static_cast<float*>(const_cast<void*>(mapped_host(out))) : nullptr;
  if (q_map) {
    da_.q_src = q_map;
    dq = d_q_;
  } else if (q_mem != KVC_MEM_DEVICE) {
    KVC_CUDA(cudaMemcpyAsync(d_q_, q, static_cast<std::size_t>(L_) * d_ * 4, cudaMemcpyHostToDevice, st_));
    dq = d_q_;
  }
  da_.q = dq;
  da_.out = (out && out_mem == KVC_MEM_DEVICE) ? out : (out_map ? out_map : d_out_);
  da_.n_parts_host = static_cast<std::int32_t>(parts_.size());
  da_.fr_on = fr_enabled_ && hext_alloc_.used() > 0 ? 1 : 0;  // some cluster has host pages
  blk_fr_[b] = da_.fr_on != 0;
  const int nl = launch_decode(t_, da_, st_, timing_ ? evb_[b] : nullptr, ev_k4_[b]);
  if (nl < 2)
    fail(-20, "decode kernels could not be launched for d = " + std::to_string(d_) +
                  " (attention is instantiated for d in {32, 64, 128, 256}; or a shared-memory opt-in was refused)");
  launches_ += nl;
  KVC_CUDA(cudaGetLastError());  // launch-configuration failures surface here, not as empty results
  // the result block goes to the host on the copy stream as soon as K4 is done (overlaps K6)
  KVC_CUDA(cudaStreamWaitEvent(cs_, ev_k4_[b], 0));
  KVC_CUDA(cudaMemcpyAsync(h_blk_[b], d_blk_[b], da_.fr_on ? dec_bytes_ : dec_lean_bytes_, cudaMemcpyDeviceToHost, cs_));
  KVC_CUDA(cudaEventRecord(ev_step_[b], cs_));
  if (out && out_mem != KVC_MEM_DEVICE && !out_map)
    KVC_CUDA(cudaMemcpyAsync(out, d_out_, static_cast<std::size_t>(L_) * d_ * 4, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaEventRecord(ev_out_[b], st_));
  step_timed_[b] = timing_;
}

// Waits for step buffer b's result block and replays its bookkeeping. Returns the settle flag.
bool Context::finish_step(int b) {
  const auto w0 = std::chrono::steady_clock::now();
  KVC_CUDA(cudaEventSynchronize(ev_step_[b]));
  const auto w1 = std::chrono::steady_clock::now();
  auto hoff = [&](const void* dptr) {
    return static_cast<const std::uint8_t*>(h_blk_[b]) +
           (static_cast<const std::uint8_t*>(dptr) - static_cast<const std::uint8_t*>(d_dec_));
  };
  std::int32_t err = 0;
  bool settle = false;
  {
    const auto* hew = reinterpret_cast<const std::int32_t*>(hoff(da_.errw));
    const auto* hfl = reinterpret_cast<const std::int32_t*>(hoff(da_.flags));
    for (int l = 0; l < L_; ++l) {
      err |= hew[l];
      settle |= hfl[l] != 0;
    }
  }
  check_err_word(err);
  if (step_timed_[b]) {  // per-kernel events of this step (recorded when it was launched)
    KVC_CUDA(cudaEventSynchronize(evb_[b][3]));
    float ms = 0.f;
    for (int i = 0; i < 3; ++i) {
      KVC_CUDA(cudaEventElapsedTime(&ms, evb_[b][i], evb_[b][i + 1]));
      step_t_[i] = ms * 1e3;
    }
    KVC_CUDA(cudaEventElapsedTime(&ms, evb_[b][0], evb_[b][3]));
    step_t_[3] = ms * 1e3;
  }
  fr_commit(b);
  std::vector<std::int64_t> gt;
  gt.swap(step_gt_[b]);
  const auto w2 = std::chrono::steady_clock::now();  // (after the instrumentation's event wait)
  replay_decode(h_blk_[b], gt.empty() ? nullptr : gt.data(), static_cast<int>(gt.size()));
  step_t_[5] = std::chrono::duration<double, std::micro>(w1 - w0).count();
  step_t_[6] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w2).count();
  return settle;
}

// Fetch-on-read bookkeeping of step buffer b (select.cu / tiers.cu k_fetch_read): each listed
// cluster's host pages now have HBM copies the page table names, so its extent is released here
// -- the physical side of the fetch the replay records for it (store.cpp:95-116). A record whose
// extent is no longer the cluster's current one (re-offloaded meanwhile, or the cluster gone) is
// skipped: the migration that replaced it already released the old extent.
void Context::fr_commit(int b) {
  if (!blk_fr_[b]) return;
  blk_fr_[b] = false;
  const auto* base = static_cast<const std::uint8_t*>(h_blk_[b]);
  const auto* n = reinterpret_cast<const std::int32_t*>(base + res_off_.frn);
  const auto* rec = reinterpret_cast<const std::int32_t*>(base + res_off_.frr);
  for (int l = 0; l < L_; ++l)
    for (int j = 0; j < n[l]; ++j) {
      const std::int32_t* r = rec + (static_cast<std::int64_t>(l) * da_.fr_max + j) * 4;
      const std::int64_t id = static_cast<std::int64_t>(static_cast<std::uint32_t>(r[0])) |
                              (static_cast<std::int64_t>(r[1]) << 32);
      if (id < 0 || id >= static_cast<std::int64_t>(clusters_.size()) || !clusters_[static_cast<std::size_t>(id)] ||
          static_cast<std::size_t>(id) >= hext_.size())
        continue;
      const Extent e = hext_[static_cast<std::size_t>(id)];
      if (e.n != r[3] || e.start != r[2]) continue;
      tier_forget(id);
      tier_n_[1] += 1;
      tier_n_[3] += e.n * t_.page_bytes;
      tier_n_[6] += 1;
      tier_n_[7] += e.n * t_.page_bytes;
    }
}

// Exchange buffer of rank r: [2 step parities][total domains][d] f32, then n u64 arrival flags.
unsigned long long* Context::peer_flag_ptr(int r) const {
  return reinterpret_cast<unsigned long long*>(peer_buf_[r] + 2LL * peer_total_ * d_ * 4);
}

void Context::set_peers(int n, int rank, int dom_offset, int total_domains, void* const* bufs) {
  flush_pending();
  if (n < 0 || n > kMaxPeers) fail(-10, "at most 8 ranks in the fused output exchange");
  if (n > 0 && (rank < 0 || rank >= n || dom_offset < 0 || dom_offset + L_ > total_domains || !bufs))
    fail(-10, "bad peer configuration");
  peer_n_ = n;
  peer_rank_ = rank;
  peer_total_ = total_domains;
  peer_step_ = 0;
  for (int r = 0; r < kMaxPeers; ++r) peer_buf_[r] = r < n ? static_cast<std::uint8_t*>(bufs[r]) : nullptr;
  da_.peer.n = 0;
  da_.peer.dom_offset = dom_offset;
}

void Context::peer_output(float* out, int mem) {
  if (peer_n_ == 0) fail(-10, "no fused output exchange configured");
  if (peer_step_ == 0) fail(-10, "no decode step yet");
  const std::uint8_t* src = peer_buf_[peer_rank_] + static_cast<std::int64_t>(peer_step_ % 2) * peer_total_ * d_ * 4;
  KVC_CUDA(cudaMemcpyAsync(out, src, static_cast<std::size_t>(peer_total_) * d_ * 4,
                           mem == KVC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st_));
  if (mem != KVC_MEM_DEVICE) sync();
}

void Context::decode_step(std::int64_t qid, const float* q, int q_mem, float* out, int out_mem,
                          const std::int64_t* gt, int n_gt) {
  (void)qid;
  flush_ingest();  // a frame whose replay is still deferred (pipelined ingest)
  if (!built_) {
    flush_pending();
    build_now();  // engine.cpp:202
  }
  if (parts_.empty()) fail(-9, "retrieve before any index was built");
  if (!q) fail(-10, "null query");
  const bool overlap = inflight_;
  const int pb = cur_;
  if (overlap) cur_ ^= 1;
  if (peer_n_ > 0) {  // this step's rows go to buffer parity (step % 2) of every rank
    peer_step_ += 1;
    da_.peer.n = peer_n_;
    for (int r = 0; r < peer_n_; ++r)
      da_.peer.out[r] = reinterpret_cast<float*>(peer_buf_[r] + static_cast<std::int64_t>(peer_step_ % 2) * peer_total_ * d_ * 4);
  }
  launch_step(cur_, q, q_mem, out, out_mem);
  step_gt_[cur_].assign(gt ? gt : nullptr, gt ? gt + (n_gt > 0 ? n_gt : 0) : nullptr);
  inflight_ = true;
  if (overlap) {
    // the previous step's bookkeeping runs on the host while this step runs on the GPU
    if (finish_step(pb)) {  // it settled a split: this step saw the pre-settle index
      KVC_CUDA(cudaStreamSynchronize(st_));
      KVC_CUDA(cudaEventSynchronize(ev_step_[cur_]));
      fr_commit(cur_);  // the discarded launch's fetch-on-read copies did happen
      launch_step(cur_, q, q_mem, out, out_mem);
    }
  }
  if (peer_n_ > 0) {
    // the step's launch is final: publish it to every rank, then wait until every rank has
    // published it (their rows are in this rank's buffer); the next step's writes into parity
    // (step + 1) % 2 are ordered after this wait in every rank's stream
    unsigned long long* flags[kMaxPeers];
    for (int r = 0; r < peer_n_; ++r) flags[r] = peer_flag_ptr(r);
    launches_ += launch_peer_signal(flags, peer_n_, peer_rank_, peer_step_, st_);
    launches_ += launch_peer_wait(peer_flag_ptr(peer_rank_), peer_n_, peer_step_, st_);
  }
  // parity / recall / self-check callers need the bookkeeping now; a host output only needs the
  // step's data (its bookkeeping still overlaps the next step)
  if (cfg_.parity_mode || cfg_.check_invariants || (gt && n_gt > 0))
    flush_pending();
  else if (out && out_mem != KVC_MEM_DEVICE)
    KVC_CUDA(cudaEventSynchronize(ev_out_[cur_]));
}

void Context::flush_pending() {
  flush_ingest();
  flush_decode();
}

void Context::flush_decode() {
  if (!inflight_) return;
  inflight_ = false;
  if (finish_step(cur_)) {
    // nothing launched after it: the settle is already reflected in the device index
  }
}

void Context::replay_decode(const void* hblock, const std::int64_t* gt, int n_gt) {
  {  // algorithmic bytes of the attention launch: attended tokens x (K + V)
    const auto* ha = reinterpret_cast<const std::int64_t*>(
        static_cast<const std::uint8_t*>(hblock) +
        (reinterpret_cast<const std::uint8_t*>(da_.attended) - static_cast<const std::uint8_t*>(d_dec_)));
    std::int64_t tok = 0;
    for (int l = 0; l < L_; ++l) tok += ha[l];
    step_t_[4] = static_cast<double>(tok) * 2.0 * d_ * es_;
    // L2 prefetch budget for the next steps: the first domains K6 will stream (KVC_L2PF_MB, default 0 = off: measured no net gain, the per-SM prefetch issue delays K4 as much as it saves in K6)
    static const double budget = [] {
      const char* e = std::getenv("KVC_L2PF_MB");
      return (e ? std::atof(e) : 0.0) * 1048576.0;
    }();
    da_.l2pf_pages = static_cast<std::int32_t>(budget / (static_cast<double>(std::max(1, L_)) * t_.page_bytes));
  }
  // host copies of the device rankings (same carve offsets as alloc_device)
  auto hp = [&](const void* dptr) {
    return static_cast<const std::uint8_t*>(hblock) +
           (static_cast<const std::uint8_t*>(dptr) - static_cast<const std::uint8_t*>(d_dec_));
  };
  const auto* h_parts = reinterpret_cast<const std::int32_t*>(hp(da_.parts));
  const auto* h_nps = reinterpret_cast<const std::int32_t*>(hp(da_.n_parts_sel));
  const auto* h_rs = reinterpret_cast<const std::int32_t*>(hp(da_.ranked_slot));
  const auto* h_rb = hp(da_.ranked_buf);
  const auto* h_nr = reinterpret_cast<const std::int32_t*>(hp(da_.n_ranked));
  const auto* h_ps = reinterpret_cast<const std::int32_t*>(hp(da_.pf_slot));
  const auto* h_pb = hp(da_.pf_buf);
  const auto* h_np = reinterpret_cast<const std::int32_t*>(hp(da_.n_pf));
  const auto* h_att = reinterpret_cast<const std::int64_t*>(hp(da_.attended));
  const auto* h_nc = reinterpret_cast<const std::int32_t*>(hp(da_.n_cand));
  (void)h_parts;
  (void)h_nps;

  // Translate every layer's slots to ids before any settle frees / reuses a slot.
  for (int l = 0; l < L_; ++l) {
    LayerOut& lo = last_[static_cast<std::size_t>(l)];
    lo.ranked.clear();
    lo.pf.clear();
    for (int i = 0; i < h_nr[l]; ++i)
      lo.ranked.push_back({slot_id_[static_cast<std::size_t>(h_rs[l * da_.k_s + i])], h_rb[l * da_.k_s + i]});
    for (int i = 0; i < h_np[l]; ++i)
      lo.pf.push_back({slot_id_[static_cast<std::size_t>(h_ps[l * da_.prefetch_k + i])], h_pb[l * da_.prefetch_k + i]});
  }

  const auto tl0 = std::chrono::steady_clock::now();
  // retrieval.cpp:58-128, layer by layer
  const bool parity = cfg_.parity_mode != 0 || (gt && n_gt > 0);
  std::vector<std::int64_t> predicted_next;
  double stall_next = 0.0;
  std::vector<std::int64_t> context_frames, fetched_frames;
  last_ttft_ = 0.0;
  for (int l = 0; l < L_; ++l) {
    LayerOut& lo = last_[static_cast<std::size_t>(l)];
    lo.selected.clear();
    lo.predicted.clear();
    lo.attended.clear();
    lo.prefetch_hits = lo.verified = lo.rep_count = lo.attended_count = 0;
    for (double& x : lo.lat) x = 0.0;
    const std::int64_t compared = static_cast<std::int64_t>(parts_.size()) + h_nc[l];
    lo.lat[0] = cfg_.lookup_cost_per_candidate_us * static_cast<double>(compared);
    std::vector<std::int64_t>& verified = verified_tmp_;
    verified.clear();
    for (const auto& r : lo.ranked)
      if (std::find(verified.begin(), verified.end(), r.first) == verified.end()) verified.push_back(r.first);
    lo.verified = static_cast<std::int64_t>(verified.size());
    if (cfg_.prefetch_enabled && l > 0) {
      lo.predicted = predicted_next;
      lo.lat[2] = stall_next;
      for (std::int64_t cid : verified) {
        if (std::find(lo.predicted.begin(), lo.predicted.end(), cid) != lo.predicted.end()) lo.prefetch_hits += 1;
        lo.lat[3] += fetch(cid, KVC_CAUSE_COMPLETION);
      }
    } else {
      for (std::int64_t cid : verified) lo.lat[1] += fetch(cid, KVC_CAUSE_RETRIEVAL);
    }
    predicted_next.clear();
    stall_next = 0.0;
    for (std::int64_t cid : verified) {
      if (!is_lazy(cid)) {  // materialize() is the identity for clusters without a pending split
        lo.selected.push_back(cid);
        continue;
      }
      std::vector<std::int64_t> s = materialize(cid);
      lo.selected.insert(lo.selected.end(), s.begin(), s.end());
    }
    std::sort(lo.selected.begin(), lo.selected.end());
    for (std::int64_t cid : lo.selected) touch(cid);
    lo.attended_count = h_att[l];
    if (parity) {
      auto& att = lo.attended;
      for (std::int64_t cid : lo.selected)
        for (const Member& m : C(cid).members) {
          att.push_back({m.frame, m.token});
          fetched_frames.push_back(m.frame);  // retrieval.cpp:101-105
        }
      for (const WinFrame& w : window_)
        for (int t = 0; t < w.T; ++t) att.push_back({w.frame_id, t});
      std::sort(att.begin(), att.end());
      att.erase(std::unique(att.begin(), att.end()), att.end());
      if (static_cast<std::int64_t>(att.size()) != lo.attended_count) {
        std::int64_t members = 0;
        for (std::int64_t cid : lo.selected) members += static_cast<std::int64_t>(C(cid).members.size());
        fail(-11, "device attended count disagrees with the attended set: layer " + std::to_string(l) +
                      " device " + std::to_string(lo.attended_count) + " host " + std::to_string(att.size()) +
                      " selected members " + std::to_string(members) + " window frames " +
                      std::to_string(window_.size()));
      }
      for (const auto& a : att) context_frames.push_back(a.first);
    }
    lo.rep_count = layer_live_count_[static_cast<std::size_t>(l)];
    lo.lat[4] = cfg_.compute_cost_per_token_us * static_cast<double>(lo.attended_count + lo.rep_count);
    if (cfg_.prefetch_enabled && l + 1 < L_) {
      for (const auto& r : lo.pf)
        if (std::find(predicted_next.begin(), predicted_next.end(), r.first) == predicted_next.end())
          predicted_next.push_back(r.first);
      double pf_cost = 0.0;
      for (std::int64_t cid : predicted_next) pf_cost += fetch(cid, KVC_CAUSE_PREFETCH);
      stall_next = std::max(0.0, pf_cost - lo.lat[4]);
    }
  }
  step_t_[8] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tl0).count();
  for (const LayerOut& lo : last_) last_ttft_ += lo.lat[0] + lo.lat[1] + lo.lat[2] + lo.lat[3] + lo.lat[4];
  last_recall_ = -1.0;
  last_fetched_.clear();
  last_context_.clear();
  if (parity) {
    std::sort(context_frames.begin(), context_frames.end());
    context_frames.erase(std::unique(context_frames.begin(), context_frames.end()), context_frames.end());
    std::sort(fetched_frames.begin(), fetched_frames.end());
    fetched_frames.erase(std::unique(fetched_frames.begin(), fetched_frames.end()), fetched_frames.end());
    last_context_ = context_frames;
    last_fetched_ = fetched_frames;
    if (gt && n_gt > 0) {
      std::int64_t hit = 0;
      for (int i = 0; i < n_gt; ++i)
        if (std::binary_search(context_frames.begin(), context_frames.end(), gt[i])) hit += 1;
      last_recall_ = static_cast<double>(hit) / static_cast<double>(n_gt);
    }
    std::uint64_t h = 1469598103934665603ull;
    for (int l = 0; l < L_; ++l)
      for (const auto& a : last_[static_cast<std::size_t>(l)].attended) {
        h = fnv1a(h, static_cast<std::uint64_t>(l));
        h = fnv1a(h, static_cast<std::uint64_t>(a.first));
        h = fnv1a(h, static_cast<std::uint64_t>(a.second));
      }
    last_digest_ = h;
  }
  const auto th2 = std::chrono::steady_clock::now();
  repin();  // engine.cpp:234
  tier_kick();  // migrations for this step's fetches / evictions (asynchronous)
  if (cfg_.check_invariants) check();
  step_t_[7] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th2).count();
}

// ---------------------------------------------------------------------------- bulk load

std::int64_t Context::bulk_load(const float* visual, const void* keys, const void* values, int N,
                                int C_, const std::int32_t* assign, const std::int64_t* frame_ids,
                                const std::int32_t* token_ids, int mem) {
  if (!pending_.empty()) fail(-10, "bulk load after frames are pending the batch build");
  if (N < 1 || C_ < 1) fail(-4, "bulk load needs members and clusters");
  if (!built_) {
    built_ = true;
    maint_seed_ = mix_seed(cfg_.seed, 2);
  }
  if (static_cast<std::int32_t>(parts_.size()) >= t_.max_parts) fail(-21, "too many partitions");
  Partition p;
  std::vector<std::int64_t> fr(frame_ids, frame_ids + N);
  std::sort(fr.begin(), fr.end());
  fr.erase(std::unique(fr.begin(), fr.end()), fr.end());
  p.frames = fr;
  p.vrep.assign(visual, visual + d_);
  p.stat = static_cast<std::int64_t>(fr.size());
  p.per_layer.resize(static_cast<std::size_t>(L_));
  p.dev_off.assign(static_cast<std::size_t>(L_), 0);
  p.dev_cap.assign(static_cast<std::size_t>(L_), 0);
  parts_.push_back(std::move(p));
  const std::int64_t pid = static_cast<std::int64_t>(parts_.size()) - 1;
  upload_partition(pid);
  std::vector<std::int32_t> z(static_cast<std::size_t>(L_), 0);
  KVC_CUDA(cudaMemcpyAsync(t_.pl_cnt + pid * L_, z.data(), L_ * 4, cudaMemcpyHostToDevice, st_));
  sync();

  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  ensure_stage(N + 1);
  std::vector<std::int64_t> new_ids;
  for (int l = 0; l < L_; ++l) {
    const auto* kb = static_cast<const std::uint8_t*>(keys) + static_cast<std::size_t>(l) * N * rb;
    const auto* vb = static_cast<const std::uint8_t*>(values) + static_cast<std::size_t>(l) * N * rb;
    const cudaMemcpyKind kind = mem == KVC_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    KVC_CUDA(cudaMemcpyAsync(d_stage_k_, kb, static_cast<std::size_t>(N) * rb, kind, st_));
    KVC_CUDA(cudaMemcpyAsync(d_stage_v_, vb, static_cast<std::size_t>(N) * rb, kind, st_));
    // stable grouping by cluster index (members keep row order)
    const std::int32_t* a = assign + static_cast<std::size_t>(l) * N;
    std::vector<std::int32_t> cnt(static_cast<std::size_t>(C_) + 1, 0);
    for (int i = 0; i < N; ++i) {
      if (a[i] < 0 || a[i] >= C_) fail(-10, "cluster index out of range");
      cnt[static_cast<std::size_t>(a[i]) + 1] += 1;
    }
    for (int c = 0; c < C_; ++c) cnt[static_cast<std::size_t>(c) + 1] += cnt[static_cast<std::size_t>(c)];
    std::vector<std::int32_t> idx(static_cast<std::size_t>(N));
    {
      std::vector<std::int32_t> pos(cnt.begin(), cnt.end() - 1);
      for (int i = 0; i < N; ++i) idx[static_cast<std::size_t>(pos[static_cast<std::size_t>(a[i])]++)] = i;
    }
    std::vector<AppendRun> runs;
    std::vector<std::int32_t> slots;
    std::vector<std::int64_t> cids;
    for (int c = 0; c < C_; ++c) {
      const std::int32_t b = cnt[static_cast<std::size_t>(c)], e = cnt[static_cast<std::size_t>(c) + 1];
      if (b == e) continue;
      std::vector<Member> m;
      m.reserve(static_cast<std::size_t>(e - b));
      for (std::int32_t j = b; j < e; ++j) {
        const std::int32_t i = idx[static_cast<std::size_t>(j)];
        m.push_back({frame_ids[i], token_ids[i]});
      }
      const std::int64_t id = new_cluster(l, pid, std::move(m), false);
      const Cluster& cl = C(id);
      runs.push_back({cl.slot, b, e - b, 0});
      slots.push_back(cl.slot);
      cids.push_back(id);
      new_ids.push_back(id);
    }
    // headers (counts / ids / residence) in one batch; statistics are computed exactly on the
    // device from the staged rows
    {
      std::vector<SlotHeader> hd(slots.size());
      for (std::size_t i = 0; i < slots.size(); ++i)
        hd[i] = SlotHeader{slots[i], 0, cids[i], static_cast<std::int64_t>(C(cids[i]).members.size())};
      auto* dh = static_cast<SlotHeader*>(dalloc_scratch(hd.size() * sizeof(SlotHeader)));
      KVC_CUDA(cudaMemcpyAsync(dh, hd.data(), hd.size() * sizeof(SlotHeader), cudaMemcpyHostToDevice, st_));
      launches_ += launch_slot_headers(t_, dh, static_cast<std::int32_t>(hd.size()), st_);
      sync();
    }
    ensure_idx(N, static_cast<std::int64_t>(runs.size()));
    std::memcpy(h_idx_, idx.data(), idx.size() * 4);
    std::memcpy(h_runs_, runs.data(), runs.size() * sizeof(AppendRun));
    KVC_CUDA(cudaMemcpyAsync(d_idx_, h_idx_, idx.size() * 4, cudaMemcpyHostToDevice, st_));
    KVC_CUDA(cudaMemcpyAsync(d_runs_, h_runs_, runs.size() * sizeof(AppendRun), cudaMemcpyHostToDevice, st_));
    launches_ += launch_exact_stats(t_, d_runs_, static_cast<std::int32_t>(runs.size()), d_idx_, d_stage_k_, st_);
    launches_ += launch_append_runs(t_, d_runs_, static_cast<std::int32_t>(runs.size()), d_idx_, d_stage_k_, d_stage_v_, st_);
    sync();
    check_dev_err();
    pl_upload(pid, l);
  }
  for (std::int64_t id : new_ids) adopt(id);
  return pid;
}

// ---------------------------------------------------------------------------- flat top-k

std::vector<std::pair<std::int64_t, int>> Context::flat_topk(const float* q, int layer, int k) {
  if (k <= 0) fail(-10, "oracle top-k must be positive");
  if (layer < 0 || layer >= L_) fail(-7, "layer out of range: " + std::to_string(layer));
  std::vector<std::int32_t> slots;
  std::vector<std::uint8_t> bufs;
  for (const auto& up : clusters_) {
    if (!up || up->layer != layer) continue;
    slots.push_back(up->slot);
    bufs.push_back(0);
    if (is_lazy(up->id)) {
      slots.push_back(up->slot);
      bufs.push_back(1);
    }
  }
  const int n = static_cast<int>(slots.size());
  std::vector<std::pair<std::int64_t, int>> out;
  if (n == 0) return out;
  ensure_idx(static_cast<std::int64_t>(n) * 2 + k + d_, 1);
  std::memcpy(h_idx_, slots.data(), n * 4);
  auto* hb = reinterpret_cast<std::uint8_t*>(h_idx_ + n);
  std::memcpy(hb, bufs.data(), n);
  KVC_CUDA(cudaMemcpyAsync(d_idx_, h_idx_, static_cast<std::size_t>(n) * 8, cudaMemcpyHostToDevice, st_));
  KVC_CUDA(cudaMemcpyAsync(d_q_, q, d_ * 4, cudaMemcpyHostToDevice, st_));
  std::int32_t* d_out = d_idx_ + 2 * n;
  auto* gs = static_cast<std::uint8_t*>(dalloc_scratch(static_cast<std::size_t>(n) * 17 + 16));
  const int nl = launch_flat_topk(t_, d_q_, d_idx_, reinterpret_cast<std::uint8_t*>(d_idx_ + n), n, k, d_out, gs, st_);
  if (nl == 0) fail(-20, "flat top-k kernel could not be launched");
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

// ---------------------------------------------------------------------------- views

void Context::cluster_stats(std::int64_t id, double* var, double* rep, double* brep) {
  const Cluster& c = C(id);
  const std::int64_t s = c.slot;
  KVC_CUDA(cudaMemcpyAsync(var, t_.var + s, 8, cudaMemcpyDeviceToHost, st_));
  if (rep) KVC_CUDA(cudaMemcpyAsync(rep, t_.rep64 + s * d_, d_ * 8, cudaMemcpyDeviceToHost, st_));
  if (brep && !c.buffer.empty())
    KVC_CUDA(cudaMemcpyAsync(brep, t_.brep64 + s * d_, d_ * 8, cudaMemcpyDeviceToHost, st_));
  sync();
}

int Context::cluster_payload(std::int64_t id, int which, float* k, float* v, int cap) {
  const Cluster& c = C(id);
  const std::int64_t nm = static_cast<std::int64_t>(c.members.size());
  const std::int64_t nb = static_cast<std::int64_t>(c.buffer.size());
  const std::int64_t rows = stage_cluster(c.slot, true);
  const std::int64_t first = which == 0 ? 0 : nm;
  const std::int64_t n = which == 0 ? nm : nb;
  (void)rows;
  const std::size_t rb = static_cast<std::size_t>(d_) * es_;
  const int take = static_cast<int>(std::min<std::int64_t>(n, cap));
  if (take > 0) {
    launches_ += launch_to_f32(t_, static_cast<std::uint8_t*>(d_stage_k_) + first * rb, d_stage_f32_, static_cast<std::int64_t>(take) * d_, st_);
    KVC_CUDA(cudaMemcpyAsync(k, d_stage_f32_, static_cast<std::size_t>(take) * d_ * 4, cudaMemcpyDeviceToHost, st_));
    sync();
    launches_ += launch_to_f32(t_, static_cast<std::uint8_t*>(d_stage_v_) + first * rb, d_stage_f32_, static_cast<std::int64_t>(take) * d_, st_);
    KVC_CUDA(cudaMemcpyAsync(v, d_stage_f32_, static_cast<std::size_t>(take) * d_ * 4, cudaMemcpyDeviceToHost, st_));
    sync();
  }
  return static_cast<int>(n);
}

// ---------------------------------------------------------------------------- self-check

void Context::check() {
  auto bad = [](const std::string& w) { fail(-11, w); };
  // index.cpp:266-282: partitions
  for (std::size_t p = 0; p < parts_.size(); ++p) {
    const Partition& part = parts_[p];
    if (!std::is_sorted(part.frames.begin(), part.frames.end())) bad("partition frame list not in temporal order");
    for (int l = 0; l < L_; ++l)
      for (std::int64_t cid : part.per_layer[static_cast<std::size_t>(l)]) {
        const Cluster* c = cluster(cid);
        if (!c) bad("partition lists a cluster that does not exist");
        if (c->parent != static_cast<std::int64_t>(p)) bad("cluster parent does not match the partition listing it");
        if (c->layer != l) bad("cluster filed under the wrong layer");
      }
  }
  // index.cpp:284-307 + device agreement
  std::vector<std::int64_t> live(static_cast<std::size_t>(L_), 0);
  std::unordered_map<std::int64_t, std::vector<std::int64_t>> frames;
  std::vector<std::int64_t> dstat(static_cast<std::size_t>(t_.max_slots)), dnmem(static_cast<std::size_t>(t_.max_slots));
  std::vector<std::int32_t> dnbuf(static_cast<std::size_t>(t_.max_slots));
  std::vector<std::uint8_t> dlazy(static_cast<std::size_t>(t_.max_slots));
  KVC_CUDA(cudaMemcpyAsync(dstat.data(), t_.stat, dstat.size() * 8, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(dnmem.data(), t_.nmem, dnmem.size() * 8, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(dnbuf.data(), t_.nbuf, dnbuf.size() * 4, cudaMemcpyDeviceToHost, st_));
  KVC_CUDA(cudaMemcpyAsync(dlazy.data(), t_.lazy, dlazy.size(), cudaMemcpyDeviceToHost, st_));
  sync();
  std::int64_t recount = 0;
  for (const auto& up : clusters_) {
    if (!up) continue;
    const Cluster& c = *up;
    const std::size_t s = static_cast<std::size_t>(c.slot);
    if (slot_id_[s] != c.id) bad("slot map out of step");
    if (c.members.empty()) bad("cluster with no members");
    if (c.stat_count != static_cast<std::int64_t>(c.members.size() + c.buffer.size()))
      bad("statistics count out of step with held entries");
    if (is_lazy(c.id) != !c.buffer.empty()) bad("deferred-split flag out of step with buffer");
    if (!is_host(c.id) && c.device_tail != 0) bad("device-resident cluster with a device tail");
    if (c.device_tail < 0 || c.device_tail > static_cast<std::int64_t>(c.members.size()))
      bad("device tail outside the member count");
    if (dstat[s] != c.stat_count || dnmem[s] != static_cast<std::int64_t>(c.members.size()) ||
        dnbuf[s] != static_cast<std::int32_t>(c.buffer.size()) || (dlazy[s] != 0) != is_lazy(c.id))
      bad("device cluster table out of step with the host control plane");
    std::int64_t first = c.members.front().frame;
    for (const Member& m : c.members) {
      first = std::min(first, m.frame);
      frames[m.frame].push_back(c.id);
    }
    for (const Member& m : c.buffer) frames[m.frame].push_back(c.id);
    if (first != c.first_frame) bad("first-frame marker out of step with members");
    live[static_cast<std::size_t>(c.layer)] += 1;
    recount += side_entries(c);
  }
  for (auto& kv : frames) {
    std::sort(kv.second.begin(), kv.second.end());
    kv.second.erase(std::unique(kv.second.begin(), kv.second.end()), kv.second.end());
    auto it = frame_clusters_.find(kv.first);
    if (it == frame_clusters_.end() || it->second != kv.second) bad("frame lookup map out of step with cluster contents");
  }
  if (frames.size() != frame_clusters_.size()) bad("frame lookup map out of step with cluster contents");
  for (int l = 0; l < L_; ++l)
    if (live[static_cast<std::size_t>(l)] != layer_live_count_[static_cast<std::size_t>(l)])
      bad("timeline length out of step with live clusters");
  // store.cpp:183-189 + ledger replay (store.cpp:44-60 is trivially consistent here: totals are
  // always derived from the op log)
  if (recount != device_entries_) bad("device occupancy out of step with residency");
}

}  // namespace kvc
