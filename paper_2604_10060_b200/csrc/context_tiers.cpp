// context_tiers.cpp -- physical host tier: migrations that make the page placement follow the
// TieredStore residence (store.cpp:95-130) kept by the host control plane.
//
// Logical residence changes (offload / fetch, store.cpp:95-130, decided exactly as the reference
// decides them) queue the cluster; migrations run asynchronously in batches, one cudaMemcpyAsync
// per cluster on the transfer stream xs_ (copy engines) between the cluster's contiguous pinned
// host extent and a contiguous HBM staging run:
//   offload: count pages (K) -> gather pages to staging + seal them (K) -> D2H per cluster (xs_)
//            -> commit: page ids become host ids, HBM pages return to the free stack (K)
//   fetch:   H2D per cluster (xs_) -> commit: fresh HBM pages filled from staging, ids rewritten (K)
//   fetch-on-read: a decode step's selected Host clusters are copied by the step itself (K4 takes
//            the pages, k_fetch_read copies, tiers.cu); Context::fr_commit then drops the extent,
//            so the queued fetch finds nothing left to move
// Phases advance when their event has completed (tier_kick polls; nothing blocks the decode
// pipeline). Until a migration commits, every kernel keeps addressing the pages where they are
// (page_k/page_v resolve host ids through the mapping), so results never depend on migration
// progress -- only where the bytes come from does.
//
// Ordering argument (why no extra synchronisation is needed):
//  * an offload's snapshot stays valid until its commit: the gather seals the copied pages
//    (appends start a new page, kernels.cu warp_append / resolve_spec.cu), splits only drop
//    clusters (the commit then skips them), and decode kernels only read pages;
//  * host extents are written only by D2H copies on xs_ that wait on a compute-stream event recorded
//    after the extent was allocated; every read of a freed extent was enqueued (on the compute
//    stream or on xs_) before that event, so an extent can return to the allocator immediately;
//  * HBM pages are popped / pushed only by compute-stream kernels (stream order).
#include <algorithm>
#include <cstring>

#include "context.hpp"

namespace kvc {

namespace {

// One copy per cluster, merged with its predecessor when both its staging run and its host extent
// continue the previous cluster's (first-fit over a quiet allocator hands out consecutive runs), so
// a batch usually crosses the host link in a few large DMA transfers.
struct CopyRun {
  std::int64_t dev, host, n;
};

void add_run(std::vector<CopyRun>& runs, std::int64_t dev, std::int64_t host, std::int64_t n) {
  if (!runs.empty() && runs.back().dev + runs.back().n == dev && runs.back().host + runs.back().n == host)
    runs.back().n += n;
  else
    runs.push_back({dev, host, n});
}

// Submits the runs as one cudaMemcpyAsync each on the transfer stream (runs are already merged, so
// a batch usually crosses the host link in a few large transfers).
void submit_runs(const std::vector<CopyRun>& runs, std::uint8_t* dev_base, std::uint8_t* host_base,
                 std::int64_t page_bytes, bool to_host, cudaStream_t st) {
  for (const CopyRun& r : runs) {
    std::uint8_t* d = dev_base + r.dev * page_bytes;
    std::uint8_t* h = host_base + r.host * page_bytes;
    KVC_CUDA(cudaMemcpyAsync(to_host ? static_cast<void*>(h) : static_cast<void*>(d),
                             to_host ? static_cast<const void*>(d) : static_cast<const void*>(h),
                             static_cast<std::size_t>(r.n * page_bytes),
                             to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st));
  }
}

}  // namespace

void Context::tier_alloc() {
  KVC_CUDA(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
  t_.seal = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(cfg_.max_slots) * 4));
  if (t_.max_hpages > 0) {
    void* p = nullptr;
    KVC_CUDA(cudaHostAlloc(&p, static_cast<std::size_t>(t_.max_hpages) * t_.page_bytes,
                           cudaHostAllocMapped | cudaHostAllocPortable));
    host_allocs_.push_back(p);
    void* dp = nullptr;
    KVC_CUDA(cudaHostGetDevicePointer(&dp, p, 0));
    t_.hpool = static_cast<std::uint8_t*>(dp);
    hext_alloc_.reset(t_.max_hpages);
    const std::int64_t sp = std::max<std::int64_t>(cfg_.tier_stage_pages, t_.maxp);
    tier_stage_ = static_cast<std::uint8_t*>(dalloc(static_cast<std::size_t>(sp) * t_.page_bytes));
    stage_alloc_.reset(sp);
    void* mv = nullptr;
    KVC_CUDA(cudaHostAlloc(&mv, sizeof(TierMove) * kTierRing * kTierMaxBatch, cudaHostAllocMapped));
    host_allocs_.push_back(mv);
    tier_mv_ = static_cast<TierMove*>(mv);
    void* cn = nullptr;
    KVC_CUDA(cudaHostAlloc(&cn, sizeof(std::int32_t) * kTierRing * kTierMaxBatch, cudaHostAllocMapped));
    host_allocs_.push_back(cn);
    tier_cnt_ = static_cast<std::int32_t*>(cn);
    tier_scratch_ = static_cast<std::int32_t*>(dalloc(static_cast<std::size_t>(kTierMaxBatch) * t_.maxp * 4));
  }
}

void Context::tier_ensure(std::int64_t id) {
  if (static_cast<std::size_t>(id) >= hext_.size()) {
    const std::size_t n = std::max<std::size_t>(static_cast<std::size_t>(id) + 1, hext_.size() * 2);
    hext_.resize(n);
    tier_busy_.resize(n, 0);
  }
}

void Context::tier_note(std::int64_t id, bool to_host) {
  if (t_.max_hpages <= 0) return;  // no host tier configured: residence stays logical
  tier_ensure(id);
  // bit 2/4: already queued for offload / fetch
  std::uint8_t& b = tier_busy_[static_cast<std::size_t>(id)];
  const std::uint8_t q = to_host ? 2 : 4;
  if (b & q) return;
  b |= q;
  (to_host ? off_q_ : fet_q_).push_back(id);
}

void Context::tier_forget(std::int64_t id) {
  if (static_cast<std::size_t>(id) >= hext_.size()) return;
  Extent& e = hext_[static_cast<std::size_t>(id)];
  if (e.n > 0) hext_alloc_.release(e.start, e.n);
  e = Extent{};
}

int Context::tier_ring_take() {
  for (int i = 0; i < kTierRing; ++i)
    if (!tier_ring_used_[i]) {
      tier_ring_used_[i] = true;
      return i;
    }
  return -1;
}

cudaEvent_t Context::tier_event() {
  if (!tier_ev_free_.empty()) {
    cudaEvent_t e = tier_ev_free_.back();
    tier_ev_free_.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  KVC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

// Starts one batch (offloads first: they free HBM). Returns false when nothing could start.
bool Context::tier_start() {
  const auto alive = [&](std::int64_t id) {
    return id >= 0 && id < static_cast<std::int64_t>(clusters_.size()) && clusters_[static_cast<std::size_t>(id)];
  };
  for (int kind = 0; kind < 2; ++kind) {
    std::vector<std::int64_t>& q = kind == 0 ? off_q_ : fet_q_;
    if (q.empty()) continue;
    const int ring = tier_ring_take();
    if (ring < 0) return false;
    TierBatch b;
    b.kind = kind;
    b.ring = ring;
    std::vector<std::int64_t> keep;
    const std::uint8_t qbit = kind == 0 ? 2 : 4;
    if (kind == 1)  // in host-address order: neighbouring extents merge into one DMA transfer
      std::sort(q.begin(), q.end(), [&](std::int64_t x, std::int64_t y) {
        return hext_[static_cast<std::size_t>(x)].start < hext_[static_cast<std::size_t>(y)].start;
      });
    for (std::int64_t id : q) {
      if (!alive(id)) continue;  // removed: its extent was released with it
      std::uint8_t& bz = tier_busy_[static_cast<std::size_t>(id)];
      const bool want = kind == 0 ? is_host(id) : !is_host(id) && hext_[static_cast<std::size_t>(id)].n > 0;
      if (!want) {
        bz &= static_cast<std::uint8_t>(~qbit);
        continue;
      }
      if ((bz & 1) || static_cast<int>(b.ids.size()) >= kTierMaxBatch) {
        keep.push_back(id);  // in another batch / batch full: later
        continue;
      }
      if (kind == 1) {  // fetch: staging for the whole extent now
        const Extent& e = hext_[static_cast<std::size_t>(id)];
        const std::int64_t s0 = stage_alloc_.alloc(e.n);
        if (s0 < 0) {
          keep.push_back(id);
          continue;
        }
        b.stage.push_back({s0, e.n});
        b.ext.push_back(e);
      }
      bz = static_cast<std::uint8_t>((bz & ~qbit) | 1);
      b.ids.push_back(id);
    }
    q.swap(keep);
    if (b.ids.empty()) {
      tier_ring_used_[ring] = false;
      continue;
    }
    const std::int32_t n = static_cast<std::int32_t>(b.ids.size());
    std::int32_t* cnt = tier_cnt_ + static_cast<std::size_t>(ring) * kTierMaxBatch;
    TierMove* mv = tier_mv_ + static_cast<std::size_t>(ring) * kTierMaxBatch;
    b.ev = tier_event();
    if (kind == 0) {
      for (std::int32_t i = 0; i < n; ++i) cnt[i] = C(b.ids[static_cast<std::size_t>(i)]).slot;
      launches_ += launch_tier_count(t_, cnt, n, cnt, st_);
      KVC_CUDA(cudaEventRecord(b.ev, st_));
    } else {
      std::vector<CopyRun> runs;
      for (std::int32_t i = 0; i < n; ++i) {
        const Extent& e = b.ext[static_cast<std::size_t>(i)];
        const Extent& s = b.stage[static_cast<std::size_t>(i)];
        mv[i] = TierMove{C(b.ids[static_cast<std::size_t>(i)]).slot, static_cast<std::int32_t>(e.n), s.start, e.start};
        add_run(runs, s.start, e.start, e.n);
      }
      submit_runs(runs, tier_stage_, t_.hpool, t_.page_bytes, false, xs_);
      tier_n_[5] += static_cast<std::int64_t>(runs.size());
      KVC_CUDA(cudaEventRecord(b.ev, xs_));
    }
    tier_n_[4] += 1;
    tier_fl_.push_back(std::move(b));
    return true;
  }
  return false;
}

bool Context::tier_advance(TierBatch& b, bool block) {
  if (block) {
    KVC_CUDA(cudaEventSynchronize(b.ev));
  } else {
    const cudaError_t e = cudaEventQuery(b.ev);
    if (e == cudaErrorNotReady) return false;
    if (e != cudaSuccess) KVC_CUDA(e);
  }
  const auto alive = [&](std::int64_t id) {
    return id >= 0 && id < static_cast<std::int64_t>(clusters_.size()) && clusters_[static_cast<std::size_t>(id)];
  };
  const std::int32_t n = static_cast<std::int32_t>(b.ids.size());
  std::int32_t* cnt = tier_cnt_ + static_cast<std::size_t>(b.ring) * kTierMaxBatch;
  TierMove* mv = tier_mv_ + static_cast<std::size_t>(b.ring) * kTierMaxBatch;
  const std::int64_t pb = t_.page_bytes;
  auto finish = [&]() {
    for (std::int64_t id : b.ids)
      if (static_cast<std::size_t>(id) < tier_busy_.size()) tier_busy_[static_cast<std::size_t>(id)] &= static_cast<std::uint8_t>(~1);
    tier_ring_used_[b.ring] = false;
    tier_ev_free_.push_back(b.ev);
    return true;
  };
  if (b.kind == 0 && b.phase == 0) {  // counts known: allocate extents, gather, copy out
    b.ext.assign(static_cast<std::size_t>(n), Extent{});
    b.stage.assign(static_cast<std::size_t>(n), Extent{});
    int moves = 0, failed = 0;
    std::int32_t maxnp = 1;
    // the batch's extents and staging runs are carved from one run each when the allocators have
    // room, so the whole batch crosses the link as one DMA transfer
    std::int64_t total = 0;
    for (std::int32_t i = 0; i < n; ++i) {
      const std::int64_t id = b.ids[static_cast<std::size_t>(i)];
      if (alive(id) && is_host(id) && cnt[i] > 0) total += cnt[i];
    }
    std::int64_t hbig = total > 0 ? hext_alloc_.alloc(total) : -1;
    std::int64_t sbig = hbig >= 0 ? stage_alloc_.alloc(total) : -1;
    if (sbig < 0 && hbig >= 0) {
      hext_alloc_.release(hbig, total);
      hbig = -1;
    }
    for (std::int32_t i = 0; i < n; ++i) {
      const std::int64_t id = b.ids[static_cast<std::size_t>(i)];
      const std::int32_t np = cnt[i];
      mv[i] = TierMove{-1, 0, 0, 0};
      if (!alive(id) || !is_host(id) || np <= 0) continue;  // np == 0: every page already in the host tier
      std::int64_t h0, s0;
      if (hbig >= 0) {
        h0 = hbig;
        s0 = sbig;
        hbig += np;
        sbig += np;
      } else {
        h0 = hext_alloc_.alloc(np);
        s0 = h0 >= 0 ? stage_alloc_.alloc(np) : -1;
      }
      if (s0 < 0) {  // tier or staging full: retry after in-flight batches release space
        if (h0 >= 0) hext_alloc_.release(h0, np);
        tier_note(id, true);
        failed += 1;
        continue;
      }
      b.ext[static_cast<std::size_t>(i)] = {h0, np};
      b.stage[static_cast<std::size_t>(i)] = {s0, np};
      mv[i] = TierMove{C(id).slot, np, s0, h0};
      maxnp = std::max(maxnp, np);
      moves += 1;
    }
    if (failed > 0 && moves == 0 && tier_fl_.size() <= 1)  // nothing in flight can release space
      fail(-21, "host tier full: raise kvc_cfg.host_pool_bytes / tier_stage_pages");
    if (moves == 0) return finish();
    launches_ += launch_tier_gather(t_, mv, n, maxnp, tier_stage_, st_);
    KVC_CUDA(cudaEventRecord(b.ev, st_));
    KVC_CUDA(cudaStreamWaitEvent(xs_, b.ev, 0));
    std::vector<CopyRun> runs;
    for (std::int32_t i = 0; i < n; ++i) {
      if (mv[i].slot < 0) continue;
      add_run(runs, b.stage[static_cast<std::size_t>(i)].start, b.ext[static_cast<std::size_t>(i)].start,
              b.ext[static_cast<std::size_t>(i)].n);
    }
    submit_runs(runs, tier_stage_, t_.hpool, pb, true, xs_);
    tier_n_[5] += static_cast<std::int64_t>(runs.size());
    KVC_CUDA(cudaEventRecord(b.ev, xs_));
    b.phase = 1;
    return false;
  }
  if (b.kind == 0 && b.phase == 1) {  // copies done: commit the surviving moves
    for (std::int32_t i = 0; i < n; ++i) {
      if (mv[i].slot < 0) continue;
      const std::int64_t id = b.ids[static_cast<std::size_t>(i)];
      const Extent e = b.ext[static_cast<std::size_t>(i)];
      stage_alloc_.release(b.stage[static_cast<std::size_t>(i)].start, b.stage[static_cast<std::size_t>(i)].n);
      if (!alive(id) || !is_host(id)) {  // removed or fetched again meanwhile: keep the old placement
        hext_alloc_.release(e.start, e.n);
        mv[i].slot = -1;
        continue;
      }
      tier_forget(id);  // a previous extent (re-offload of a device tail) is superseded
      hext_[static_cast<std::size_t>(id)] = e;
      tier_n_[0] += 1;
      tier_n_[2] += e.n * pb;
    }
    launches_ += launch_tier_commit_offload(t_, mv, n, st_);
    KVC_CUDA(cudaEventRecord(b.ev, st_));
    b.phase = 2;
    return false;
  }
  if (b.kind == 0) return finish();  // phase 2: commit done, argument slot reusable
  if (b.phase == 0) {  // fetch: extents are in staging
    std::int32_t maxnp = 1;
    for (std::int32_t i = 0; i < n; ++i) {
      const std::int64_t id = b.ids[static_cast<std::size_t>(i)];
      const Extent e = b.ext[static_cast<std::size_t>(i)];
      if (!alive(id) || is_host(id) || hext_[static_cast<std::size_t>(id)].start != e.start) {
        mv[i].slot = -1;  // removed / offloaded again: the extent stays (or went with the cluster)
        continue;
      }
      maxnp = std::max<std::int32_t>(maxnp, static_cast<std::int32_t>(e.n));
      tier_forget(id);
      tier_n_[1] += 1;
      tier_n_[3] += e.n * pb;
    }
    launches_ += launch_tier_commit_fetch(t_, mv, n, std::max<std::int32_t>(maxnp, t_.maxp), tier_stage_,
                                          tier_scratch_, st_);
    KVC_CUDA(cudaEventRecord(b.ev, st_));
    b.phase = 1;
    return false;
  }
  for (const Extent& s : b.stage) stage_alloc_.release(s.start, s.n);
  return finish();
}

void Context::tier_kick() {
  if (t_.max_hpages <= 0) return;
  for (auto it = tier_fl_.begin(); it != tier_fl_.end();) {
    bool done = false;
    // a batch may move through several phases at once when its events already completed
    while (!done) {
      const int ph = it->phase;
      done = tier_advance(*it, false);
      if (!done && it->phase == ph) break;
    }
    it = done ? tier_fl_.erase(it) : std::next(it);
  }
  while ((!off_q_.empty() || !fet_q_.empty()) && tier_start()) {
  }
}

void Context::tier_sync() {
  flush_pending();
  if (t_.max_hpages <= 0) return;
  for (int guard = 0;; ++guard) {
    tier_kick();
    if (tier_fl_.empty()) {
      if (off_q_.empty() && fet_q_.empty()) break;
      if (!tier_start()) fail(-21, "host tier full: raise kvc_cfg.host_pool_bytes / tier_stage_pages");
      continue;
    }
    TierBatch& b = tier_fl_.front();
    if (tier_advance(b, true)) tier_fl_.pop_front();
    if (guard > 1000000) fail(-11, "host-tier migrations do not converge");
  }
  sync();
  check_dev_err();
}

void Context::tier_stats(std::int64_t* out) const {
  std::int64_t hc = 0;
  for (std::size_t i = 0; i < hext_.size(); ++i)
    if (hext_[i].n > 0) hc += 1;
  out[0] = hext_alloc_.used();
  out[1] = t_.max_hpages;
  out[2] = hc;
  out[3] = tier_n_[0];
  out[4] = tier_n_[1];
  out[5] = tier_n_[2];
  out[6] = tier_n_[3];
  out[7] = static_cast<std::int64_t>(off_q_.size() + fet_q_.size());
  out[8] = static_cast<std::int64_t>(tier_fl_.size());
  out[9] = stage_alloc_.used();
  out[10] = tier_n_[4];
  out[11] = tier_n_[5];
  out[12] = tier_n_[6];
  out[13] = tier_n_[7];
}

void Context::cluster_tier(std::int64_t id, std::int64_t* out) const {
  if (id < 0 || id >= static_cast<std::int64_t>(clusters_.size()) || !clusters_[static_cast<std::size_t>(id)])
    fail(-8, "unknown cluster id: " + std::to_string(id));
  out[0] = -1;
  out[1] = 0;
  out[2] = 0;
  if (static_cast<std::size_t>(id) < hext_.size()) {
    out[0] = hext_[static_cast<std::size_t>(id)].start;
    out[1] = hext_[static_cast<std::size_t>(id)].n;
    out[2] = tier_busy_[static_cast<std::size_t>(id)] & 1;
  }
}

// Debug: page tables vs the host's view of the tiers (small contexts; reads each live slot's list).
// out[4]: host page ids outside the cluster's extent, Device clusters holding host pages, Host
// clusters whose member pages are all still in HBM, clusters whose page fills disagree with the
// member count (or whose HBM tail exceeds the logical device tail).
void Context::tier_check(std::int64_t* out) {
  flush_pending();
  sync();
  for (int i = 0; i < 4; ++i) out[i] = 0;
  std::vector<std::int32_t> fill(static_cast<std::size_t>(t_.max_pages + t_.max_hpages));
  KVC_CUDA(cudaMemcpyAsync(fill.data(), t_.pg_fill, fill.size() * 4, cudaMemcpyDeviceToHost, st_));
  sync();
  std::vector<std::int32_t> list(static_cast<std::size_t>(t_.maxp));
  for (const auto& up : clusters_) {
    if (!up) continue;
    const Cluster& c = *up;
    std::int32_t np = 0;
    KVC_CUDA(cudaMemcpyAsync(&np, t_.npages + c.slot, 4, cudaMemcpyDeviceToHost, st_));
    sync();
    if (np > 0) {
      KVC_CUDA(cudaMemcpyAsync(list.data(), t_.pages + static_cast<std::int64_t>(c.slot) * t_.maxp, np * 4,
                               cudaMemcpyDeviceToHost, st_));
      sync();
    }
    const Extent e = static_cast<std::size_t>(c.id) < hext_.size() ? hext_[static_cast<std::size_t>(c.id)] : Extent{};
    std::int64_t rows = 0, tail_rows = 0, nhost = 0;
    for (std::int32_t p = 0; p < np; ++p) {
      const std::int32_t pg = list[static_cast<std::size_t>(p)];
      rows += fill[static_cast<std::size_t>(pg)];
      if (pg >= t_.max_pages) {
        nhost += 1;
        if (p >= e.n || pg != t_.max_pages + e.start + p) out[0] += 1;
      } else if (p >= e.n) {
        tail_rows += fill[static_cast<std::size_t>(pg)];
      }
    }
    if (!is_host(c.id) && nhost > 0) out[1] += 1;
    if (is_host(c.id) && nhost == 0 && np > 0) out[2] += 1;
    if (rows != static_cast<std::int64_t>(c.members.size()) || (is_host(c.id) && tail_rows > c.device_tail)) out[3] += 1;
  }
}

}  // namespace kvc
