// abi.cpp -- the extern "C" boundary (include/kvc.h). Every entry point catches kvc::Error and
// returns its code; no exception crosses the ABI (SURVEY.md §8(b) "Errors").
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/kvc.h"
#include "context.hpp"
#include "kmeans.hpp"
#include "token.hpp"

using kvc::Context;
using kvc::TokenContext;

// One of the two is set: the cluster path (Context) or the token-level baseline
// (TokenContext, cfg.token_mode -- RetrievalMode::TokenBaseline, engine.cpp:153-158,179-203).
struct kvc_ctx {
  std::unique_ptr<Context> impl;
  std::unique_ptr<TokenContext> tok;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return KVC_OK;
  } catch (const kvc::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return KVC_E_GENERIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KVC_E_GENERIC;
  }
}

// Host-state readers first complete the deferred bookkeeping of the last decode step. Only call
// inside guard(): it throws (a failed replay must surface as the reader's status, never leave
// stale views behind a success count) and a token-baseline context has no cluster index.
Context& F(kvc_ctx* c) {
  if (!c->impl) kvc::fail(KVC_E_CONFIG, "not available in token-baseline mode (cfg.token_mode)");
  c->impl->flush_pending();
  return *c->impl;
}

// Entry points that return a count (not wrapped in guard): the cluster path only.
#define KVC_CLUSTER_ONLY(ctx)                                                   \
  do {                                                                          \
    if (!(ctx)->impl) {                                                         \
      g_err = "not available in token-baseline mode (cfg.token_mode)";          \
      return KVC_E_CONFIG;                                                      \
    }                                                                           \
  } while (0)

// Readers that return a count (not wrapped in guard): the cluster path, with the deferred
// decode bookkeeping completed first; a replay failure is returned as the reader's status.
#define KVC_READER(ctx)                                                         \
  do {                                                                          \
    KVC_CLUSTER_ONLY(ctx);                                                      \
    const int rc_ = guard([&] { (ctx)->impl->flush_pending(); });               \
    if (rc_ != KVC_OK) return rc_;                                              \
  } while (0)

// After KVC_READER: the flushed context.
inline Context& R(kvc_ctx* c) { return *c->impl; }

template <class T>
int copy_out(const std::vector<T>& v, T* dst, int cap) {
  const int n = static_cast<int>(v.size());
  if (dst)
    for (int i = 0; i < n && i < cap; ++i) dst[i] = v[static_cast<std::size_t>(i)];
  return n;
}

}  // namespace

extern "C" {

void kvc_cfg_default(kvc_cfg* c) {
  std::memset(c, 0, sizeof(*c));
  // EngineConfig defaults (engine.hpp:21-33 and the nested structs)
  c->k_v = 4;
  c->k_s = 4;
  c->window_frames = 4;
  c->prefetch_k = 4;
  c->prefetch_enabled = 0;
  c->token_mode = 0;
  c->token_budget = 256;
  c->lookup_cost_per_candidate_us = 0.02;
  c->compute_cost_per_token_us = 0.6;
  c->tau_min = 0.05;
  c->tau_max = 0.3;
  c->n0 = 32.0;
  c->defer_host_splits = 1;
  c->max_split_depth = 4;
  c->visual_floor = 0.75;
  c->target_visual_cluster_size = 8;
  c->target_semantic_cluster_size = 32;
  c->kmeans_max_iters = 50;
  c->kmeans_tol = 1e-6;
  c->alpha_us = 10.0;
  c->beta_us_per_byte = 0.001;
  c->bytes_per_entry = 0;
  c->device_capacity_entries = 1 << 20;
  c->build_batch_frames = 32;
  c->batched_ingest = 0;
  c->ingest_overhead_us = 10.0;
  c->offload_horizon_frames = 16;
  c->seed = 0;
  // device data plane
  c->kv_dtype = KVC_DTYPE_F32;
  c->page_tokens = 0;  // auto: 64, halved while the attention kernel's page ring does not fit
  c->max_pages = 0;
  c->pool_bytes = 1LL << 30;
  c->max_slots = 65536;
  c->max_cluster_pages = 256;
  c->max_buffer_pages = 64;
  c->max_partitions = 4096;
  c->max_candidates = 1024;
  c->max_tokens = 256;
  c->parity_mode = 0;
  c->check_invariants = 0;
  c->tier_stage_pages = 2048;
  c->host_pool_bytes = 256LL << 20;
}

const char* kvc_last_error(void) { return g_err.c_str(); }

int kvc_create(const kvc_cfg* cfg, int32_t d, int32_t L, kvc_ctx** out) {
  return guard([&] {
    if (!cfg || !out) kvc::fail(KVC_E_CONFIG, "null argument");
    auto* h = new kvc_ctx;
    try {
      if (cfg->token_mode)
        h->tok = std::make_unique<TokenContext>(*cfg, d, L);
      else
        h->impl = std::make_unique<Context>(*cfg, d, L);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void kvc_destroy(kvc_ctx* ctx) { delete ctx; }

void* kvc_stream(kvc_ctx* ctx) {
  if (!ctx) return nullptr;
  return ctx->tok ? static_cast<void*>(ctx->tok->stream()) : static_cast<void*>(ctx->impl->stream());
}

int kvc_ingest_frame(kvc_ctx* ctx, int64_t frame_id, const float* visual, const void* keys,
                     const void* values, int32_t T, int32_t mem, int64_t* assigned,
                     int64_t* partition) {
  return guard([&] {
    if (ctx->tok) {  // engine.cpp:153-158: the entries join the pools
      if (assigned) std::fill(assigned, assigned + static_cast<int64_t>(ctx->tok->L()) * (T > 0 ? T : 0), -1);
      if (partition) *partition = -1;
      ctx->tok->ingest_frame(frame_id, keys, values, T, mem);
      return;
    }
    if (!ctx->impl) kvc::fail(KVC_E_CONFIG, "no context");
    ctx->impl->flush_decode();  // (not F: the previous frame's deferred replay overlaps this frame)
    ctx->impl->ingest_frame(frame_id, visual, keys, values, T, mem, assigned, partition);
  });
}

int kvc_decode_step(kvc_ctx* ctx, int64_t query_id, const float* q, int32_t q_mem, float* out,
                    int32_t out_mem, const int64_t* gt, int32_t n_gt) {
  return guard([&] {
    if (ctx->tok)
      ctx->tok->decode_step(query_id, q, q_mem, out, out_mem, gt, n_gt);
    else
      ctx->impl->decode_step(query_id, q, q_mem, out, out_mem, gt, n_gt);
  });
}

int kvc_last_ranked(kvc_ctx* ctx, int32_t layer, int64_t* ids, int32_t* is_buffer, int32_t cap) {
  if (ctx->tok) return 0;  // no cluster ranking in the token baseline
  KVC_READER(ctx);
  const auto& ls = R(ctx).last_layers();
  if (layer < 0 || layer >= static_cast<int>(ls.size())) return KVC_E_BAD_LAYER;
  const auto& r = ls[static_cast<std::size_t>(layer)].ranked;
  for (int i = 0; i < static_cast<int>(r.size()) && i < cap; ++i) {
    ids[i] = r[static_cast<std::size_t>(i)].first;
    is_buffer[i] = r[static_cast<std::size_t>(i)].second;
  }
  return static_cast<int>(r.size());
}

int kvc_last_selected(kvc_ctx* ctx, int32_t layer, int64_t* ids, int32_t cap) {
  if (ctx->tok) return 0;
  KVC_READER(ctx);
  const auto& ls = R(ctx).last_layers();
  if (layer < 0 || layer >= static_cast<int>(ls.size())) return KVC_E_BAD_LAYER;
  return copy_out(ls[static_cast<std::size_t>(layer)].selected, ids, cap);
}

int kvc_last_attended(kvc_ctx* ctx, int32_t layer, int64_t* frames, int32_t* tokens, int32_t cap) {
  if (ctx->tok) {
    int n = 0;
    const int rc = guard([&] { n = ctx->tok->attended(layer, frames, tokens, cap); });
    return rc != KVC_OK ? rc : n;
  }
  KVC_READER(ctx);
  const auto& ls = R(ctx).last_layers();
  if (layer < 0 || layer >= static_cast<int>(ls.size())) return KVC_E_BAD_LAYER;
  const auto& a = ls[static_cast<std::size_t>(layer)].attended;
  for (int i = 0; i < static_cast<int>(a.size()) && i < cap; ++i) {
    frames[i] = a[static_cast<std::size_t>(i)].first;
    tokens[i] = a[static_cast<std::size_t>(i)].second;
  }
  return static_cast<int>(a.size());
}

int kvc_last_layer_meta(kvc_ctx* ctx, int32_t layer, double* lat, int64_t* ints) {
  if (ctx->tok) return guard([&] { ctx->tok->layer_meta(layer, lat, ints); });
  KVC_READER(ctx);
  const auto& ls = R(ctx).last_layers();
  if (layer < 0 || layer >= static_cast<int>(ls.size())) return KVC_E_BAD_LAYER;
  const auto& lo = ls[static_cast<std::size_t>(layer)];
  for (int i = 0; i < 5; ++i) lat[i] = lo.lat[i];
  ints[0] = lo.verified;
  ints[1] = lo.prefetch_hits;
  ints[2] = lo.rep_count;
  ints[3] = static_cast<int64_t>(lo.predicted.size());
  ints[4] = lo.attended_count;
  return KVC_OK;
}

int kvc_last_query_meta(kvc_ctx* ctx, double* dd) {
  if (ctx->tok) {
    dd[0] = ctx->tok->ttft();
    dd[1] = ctx->tok->recall();
    return KVC_OK;
  }
  KVC_READER(ctx);
  dd[0] = R(ctx).last_ttft();
  dd[1] = R(ctx).last_recall();
  return KVC_OK;
}

// 0 (with kvc_last_error set) when the deferred bookkeeping of the step failed
uint64_t kvc_last_digest(kvc_ctx* ctx) {
  if (ctx->tok) return ctx->tok->digest();
  uint64_t h = 0;
  const int rc = guard([&] { h = F(ctx).last_digest(); });
  return rc == KVC_OK ? h : 0;
}

int kvc_flat_topk(kvc_ctx* ctx, const float* q, int32_t layer, int32_t k, int64_t* ids,
                  int32_t* is_buffer) {
  int n = 0;
  const int rc = guard([&] {
    auto r = F(ctx).flat_topk(q, layer, k);
    n = static_cast<int>(r.size());
    for (int i = 0; i < n; ++i) {
      ids[i] = r[static_cast<std::size_t>(i)].first;
      is_buffer[i] = r[static_cast<std::size_t>(i)].second;
    }
  });
  return rc != KVC_OK ? rc : n;
}

int kvc_build_now(kvc_ctx* ctx) {
  return guard([&] { F(ctx).build_now(); });
}

int kvc_bulk_load(kvc_ctx* ctx, const float* visual, const void* keys, const void* values,
                  int32_t N, int32_t C, const int32_t* assign, const int64_t* frame_ids,
                  const int32_t* token_ids, int32_t mem, int64_t* partition) {
  return guard([&] {
    const int64_t p = F(ctx).bulk_load(visual, keys, values, N, C, assign, frame_ids, token_ids, mem);
    if (partition) *partition = p;
  });
}

int kvc_n_clusters(kvc_ctx* ctx) {
  if (ctx->tok) return 0;
  KVC_READER(ctx);
  return static_cast<int>(R(ctx).cluster_ids().size());
}

int kvc_cluster_ids(kvc_ctx* ctx, int64_t* ids, int32_t cap) {
  if (ctx->tok) return 0;
  KVC_READER(ctx);
  return copy_out(R(ctx).cluster_ids(), ids, cap);
}

int kvc_cluster(kvc_ctx* ctx, int64_t id, int64_t* info, double* var, double* rep,
                double* buffer_rep) {
  return guard([&] {
    const kvc::Cluster* c = F(ctx).cluster(id);
    if (!c) kvc::fail(KVC_E_UNKNOWN_CLUSTER, "unknown cluster id: " + std::to_string(id));
    info[0] = c->layer;
    info[1] = c->parent;
    info[2] = static_cast<int64_t>(c->members.size());
    info[3] = static_cast<int64_t>(c->buffer.size());
    info[4] = c->stat_count;
    info[5] = F(ctx).is_lazy(id) ? 1 : 0;
    info[6] = F(ctx).is_host(id) ? 1 : 0;
    info[7] = c->device_tail;
    info[8] = c->first_frame;
    info[9] = c->last_touch;
    double v = 0.0;
    F(ctx).cluster_stats(id, &v, rep, buffer_rep);
    if (var) *var = v;
  });
}

int kvc_cluster_entries(kvc_ctx* ctx, int64_t id, int32_t which, int64_t* frames, int32_t* tokens,
                        int32_t cap) {
  KVC_READER(ctx);
  const kvc::Cluster* c = R(ctx).cluster(id);
  if (!c) return KVC_E_UNKNOWN_CLUSTER;
  const auto& v = which == 0 ? c->members : c->buffer;
  int i = 0;
  for (const kvc::Member& m : v) {
    if (i >= cap) break;
    frames[i] = m.frame;
    tokens[i] = m.token;
    ++i;
  }
  return static_cast<int>(v.size());
}

int kvc_cluster_payload(kvc_ctx* ctx, int64_t id, int32_t which, float* keys, float* values,
                        int32_t cap) {
  int n = 0;
  const int rc = guard([&] { n = F(ctx).cluster_payload(id, which, keys, values, cap); });
  return rc != KVC_OK ? rc : n;
}

int kvc_n_partitions(kvc_ctx* ctx) {
  if (ctx->tok) return 0;
  KVC_READER(ctx);
  return static_cast<int>(R(ctx).partitions().size());
}

int kvc_partition(kvc_ctx* ctx, int32_t p, double* visual_rep, int64_t* frames, int32_t cap) {
  KVC_READER(ctx);
  const auto& ps = R(ctx).partitions();
  if (p < 0 || p >= static_cast<int>(ps.size())) return KVC_E_UNKNOWN_CLUSTER;
  const auto& part = ps[static_cast<std::size_t>(p)];
  if (visual_rep) std::memcpy(visual_rep, part.vrep.data(), part.vrep.size() * sizeof(double));
  return copy_out(part.frames, frames, cap);
}

int kvc_partition_layer(kvc_ctx* ctx, int32_t p, int32_t layer, int64_t* ids, int32_t cap) {
  KVC_READER(ctx);
  const auto& ps = R(ctx).partitions();
  if (p < 0 || p >= static_cast<int>(ps.size())) return KVC_E_UNKNOWN_CLUSTER;
  if (layer < 0 || layer >= R(ctx).L()) return KVC_E_BAD_LAYER;
  return copy_out(ps[static_cast<std::size_t>(p)].per_layer[static_cast<std::size_t>(layer)], ids, cap);
}

int kvc_maint_stats(kvc_ctx* ctx, int64_t* out) {
  if (ctx->tok) {  // the baseline never runs the maintainer
    std::memset(out, 0, 9 * sizeof(int64_t));
    return KVC_OK;
  }
  KVC_READER(ctx);
  std::memcpy(out, R(ctx).maint_stats(), 9 * sizeof(int64_t));
  return KVC_OK;
}

int64_t kvc_ledger(kvc_ctx* ctx, int64_t* ops, int64_t* bytes, double* cost_us) {
  if (ctx->tok) return ctx->tok->ledger(ops, bytes, cost_us);  // the baseline ledger (engine.cpp:184)
  KVC_READER(ctx);
  for (int i = 0; i < 5; ++i) {
    ops[i] = 0;
    bytes[i] = 0;
    cost_us[i] = 0.0;
  }
  for (const auto& op : R(ctx).ledger()) {  // TransferLedger::record (store.cpp:21-27)
    ops[op.cause] += op.n_ops;
    bytes[op.cause] += op.bytes;
    cost_us[op.cause] += op.cost_us;
  }
  return R(ctx).device_entries();
}

// (token baseline: totals only -- one op per coalesced run would be thousands per query)
int kvc_ledger_log_size(kvc_ctx* ctx) {
  if (ctx->tok) return 0;
  KVC_READER(ctx);
  return static_cast<int>(R(ctx).ledger().size());
}

int kvc_ledger_op(kvc_ctx* ctx, int32_t i, int64_t* ints) {
  KVC_READER(ctx);
  const auto& lg = R(ctx).ledger();
  if (i < 0 || i >= static_cast<int>(lg.size())) return KVC_E_CONFIG;
  const auto& op = lg[static_cast<std::size_t>(i)];
  ints[0] = op.cause;
  ints[1] = op.to_device ? 1 : 0;
  ints[2] = op.cluster_id;
  ints[3] = op.bytes;
  return KVC_OK;
}

int kvc_check(kvc_ctx* ctx) {
  return guard([&] { F(ctx).check(); });
}

int kvc_offload(kvc_ctx* ctx, int64_t id, double* cost_us) {
  return guard([&] {
    const double c = F(ctx).offload(id);
    F(ctx).tier_kick();
    if (cost_us) *cost_us = c;
  });
}

int kvc_fetch(kvc_ctx* ctx, int64_t id, int32_t cause, double* cost_us) {
  return guard([&] {
    if (cause < 0 || cause > 4) kvc::fail(KVC_E_CONFIG, "unknown transfer cause");
    const double c = F(ctx).fetch(id, cause);
    F(ctx).tier_kick();
    if (cost_us) *cost_us = c;
  });
}

int kvc_tier_sync(kvc_ctx* ctx) {
  return guard([&] { F(ctx).tier_sync(); });
}

int kvc_tier_stats(kvc_ctx* ctx, int64_t* out) {
  return guard([&] { F(ctx).tier_stats(out); });
}

size_t kvc_exchange_bytes(int32_t n_ranks, int32_t total_domains, int32_t d) {
  return 2ull * static_cast<size_t>(total_domains) * static_cast<size_t>(d) * 4 + static_cast<size_t>(n_ranks) * 8;
}

int kvc_ipc_alloc(size_t bytes, void** dptr, uint8_t* handle64) {
  return guard([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) kvc::fail(KVC_E_NO_DEVICE, "no CUDA device");
    KVC_CUDA(cudaMalloc(dptr, bytes));
    KVC_CUDA(cudaMemset(*dptr, 0, bytes));
    cudaIpcMemHandle_t h;
    KVC_CUDA(cudaIpcGetMemHandle(&h, *dptr));
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int kvc_ipc_open(const uint8_t* handle64, void** dptr) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    KVC_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int kvc_ipc_close(void* dptr) {
  return guard([&] { KVC_CUDA(cudaIpcCloseMemHandle(dptr)); });
}

int kvc_ipc_free(void* dptr) {
  return guard([&] { KVC_CUDA(cudaFree(dptr)); });
}

int kvc_set_peers(kvc_ctx* ctx, int32_t n_ranks, int32_t rank, int32_t dom_offset, int32_t total_domains,
                  void* const* bufs) {
  return guard([&] { F(ctx).set_peers(n_ranks, rank, dom_offset, total_domains, bufs); });
}

int kvc_peer_output(kvc_ctx* ctx, float* out, int32_t mem) {
  return guard([&] { F(ctx).peer_output(out, mem); });
}

int kvc_debug_tier_check(kvc_ctx* ctx, int64_t* out) {
  return guard([&] { F(ctx).tier_check(out); });
}

int kvc_debug_split_two(kvc_ctx* ctx, const float* pts, int32_t n, uint64_t seed, int32_t* assign, int32_t* meta3,
                        double* objective) {
  int live = 0;
  const int rc = guard([&] {
    const kvc::KMeansOut o = F(ctx).debug_split_two_dev(pts, n, seed);
    for (int i = 0; i < n; ++i) assign[i] = o.assign[static_cast<std::size_t>(i)];
    if (meta3) {
      meta3[0] = o.k_live;
      meta3[1] = o.iterations;
      meta3[2] = o.degenerate ? 1 : 0;
    }
    if (objective) *objective = o.objective;
    live = o.k_live;
  });
  return rc != KVC_OK ? rc : live;
}

int kvc_debug_kmeans(kvc_ctx* ctx, const float* pts, int32_t n_sets, const int32_t* n, const int32_t* k,
                     int32_t max_iters, double tol, const uint64_t* seeds, int32_t* assign, int32_t* meta2,
                     double* objective) {
  int rc = guard([&] {
    std::vector<const float*> ptr;
    std::vector<int> nn, kk;
    std::vector<std::uint64_t> ss;
    std::size_t off = 0;
    const int d = F(ctx).d();
    for (int i = 0; i < n_sets; ++i) {
      ptr.push_back(pts + off * d);
      nn.push_back(n[i]);
      kk.push_back(k[i]);
      ss.push_back(seeds[i]);
      off += static_cast<std::size_t>(n[i]);
    }
    const std::vector<kvc::KMeansOut> o = F(ctx).kmeans_pools(ptr, nn, kk, ss, max_iters, tol);
    off = 0;
    for (int i = 0; i < n_sets; ++i) {
      for (int t = 0; t < n[i]; ++t) assign[off + t] = o[static_cast<std::size_t>(i)].assign[static_cast<std::size_t>(t)];
      off += static_cast<std::size_t>(n[i]);
      meta2[2 * i] = o[static_cast<std::size_t>(i)].k_live;
      meta2[2 * i + 1] = o[static_cast<std::size_t>(i)].iterations;
      objective[i] = o[static_cast<std::size_t>(i)].objective;
    }
  });
  return rc;
}

int kvc_cluster_tier(kvc_ctx* ctx, int64_t id, int64_t* out) {
  return guard([&] { F(ctx).cluster_tier(id, out); });
}

int64_t kvc_launch_count(kvc_ctx* ctx) { return ctx->tok ? ctx->tok->launches() : ctx->impl->launches(); }

int kvc_last_step_timing(kvc_ctx* ctx, double* t) {
  const double* s = ctx->tok ? ctx->tok->step_timing() : ctx->impl->step_timing();
  for (int i = 0; i < 10; ++i) t[i] = s[i];
  return KVC_OK;
}

int kvc_set_head_dim(kvc_ctx* ctx, int32_t d_logical) {
  return guard([&] {
    if (ctx->tok)
      ctx->tok->set_head_dim(d_logical);
    else
      ctx->impl->set_head_dim(d_logical);
  });
}

void kvc_set_timing(kvc_ctx* ctx, int32_t on) {
  if (ctx->tok)
    ctx->tok->set_timing(on != 0);
  else
    ctx->impl->set_timing(on != 0);
}

int kvc_debug_assign_check(kvc_ctx* ctx, const void* keys, int32_t T, int64_t partition, int32_t mem,
                           double* out4) {
  return guard([&] { F(ctx).debug_assign_check(keys, T, partition, mem, out4); });
}

int kvc_debug_div_check(uint64_t n, uint64_t seed, int32_t max_den, uint64_t* mismatches) {
  int dev = 0;
  if (cudaGetDeviceCount(&dev) != cudaSuccess || dev == 0) return KVC_E_NO_DEVICE;
  *mismatches = kvc::debug_div_check(n, seed, max_den);
  return *mismatches == ~0ull ? KVC_E_CUDA : KVC_OK;
}

// ------------------------------------------------------------------ component-level API
int kvc_add_partition(kvc_ctx* ctx, int64_t first_frame, const float* visual, int64_t* partition) {
  return guard([&] {
    const int64_t p = F(ctx).api_add_partition(first_frame, visual);
    if (partition) *partition = p;
  });
}

int kvc_append_frame(kvc_ctx* ctx, int64_t partition, int64_t frame_id, const float* visual) {
  return guard([&] { F(ctx).api_append_frame(partition, frame_id, visual); });
}

int kvc_add_cluster(kvc_ctx* ctx, int32_t layer, int64_t partition, int32_t n, const float* keys,
                    const float* values, const int64_t* frames, const int32_t* tokens, int32_t residence,
                    int32_t adopt, int64_t* id) {
  return guard([&] {
    const int64_t c = F(ctx).api_add_cluster(layer, partition, n, keys, values, frames, tokens, residence != 0, adopt != 0);
    if (id) *id = c;
  });
}

int kvc_add_partition_ex(kvc_ctx* ctx, const int64_t* frames, int32_t n_frames, const double* visual_rep,
                         int64_t visual_stat_count, int64_t* partition) {
  return guard([&] {
    const int64_t p = F(ctx).api_add_partition_ex(frames, n_frames, visual_rep, visual_stat_count);
    if (partition) *partition = p;
  });
}

int kvc_add_cluster_ex(kvc_ctx* ctx, const kvc_cluster_record* r, int64_t* id) {
  return guard([&] {
    if (!r) kvc::fail(KVC_E_CONFIG, "null record");
    const int64_t c = F(ctx).api_add_cluster_ex(
        r->layer, r->partition, r->n_members, r->member_keys, r->member_values, r->member_frames, r->member_tokens,
        r->n_buffer, r->buffer_keys, r->buffer_values, r->buffer_frames, r->buffer_tokens, r->rep, r->variance,
        r->stat_count, r->buffer_rep, r->lazy_split != 0, r->residence != 0, r->device_tail, r->adopt != 0, r->want_id);
    if (id) *id = c;
  });
}

int kvc_adopt(kvc_ctx* ctx, int64_t id) {
  return guard([&] { F(ctx).api_adopt(id); });
}

int kvc_reset_window(kvc_ctx* ctx) {
  return guard([&] {
    if (ctx->tok)
      ctx->tok->reset_window();
    else
      F(ctx).api_reset_window();
  });
}

int kvc_set_retrieval(kvc_ctx* ctx, const kvc_cfg* cfg) {
  return guard([&] {
    if (!cfg) kvc::fail(KVC_E_CONFIG, "null config");
    if (ctx->tok) kvc::fail(KVC_E_CONFIG, "token-baseline contexts take their budget at creation");
    F(ctx).api_set_retrieval(*cfg);
  });
}

int kvc_reconfigure(kvc_ctx* ctx, const kvc_cfg* cfg, int32_t what) {
  return guard([&] {
    if (!cfg) kvc::fail(KVC_E_CONFIG, "null config");
    F(ctx).api_reconfigure(*cfg, what);
  });
}

int kvc_place_frame(kvc_ctx* ctx, int64_t frame_id, const float* visual, int64_t* partition) {
  return guard([&] {
    const int64_t p = F(ctx).api_place_frame(frame_id, visual);
    if (partition) *partition = p;
  });
}

int kvc_insert(kvc_ctx* ctx, int64_t partition, int32_t layer, int32_t token, int64_t frame_id, const float* key,
               const float* value, int64_t* cluster) {
  return guard([&] {
    const int64_t c = F(ctx).api_insert(partition, layer, token, frame_id, key, value);
    if (cluster) *cluster = c;
  });
}

int kvc_materialize(kvc_ctx* ctx, int64_t id, int64_t* ids, int32_t cap) {
  std::vector<int64_t> r;
  const int rc = guard([&] { r = F(ctx).api_materialize(id); });
  return rc != KVC_OK ? rc : copy_out(r, ids, cap);
}

int kvc_touch(kvc_ctx* ctx, int64_t id) {
  return guard([&] { F(ctx).api_touch(id); });
}

int kvc_pin(kvc_ctx* ctx, const int64_t* ids, int32_t n) {
  return guard([&] { F(ctx).api_pin(std::vector<int64_t>(ids, ids + (n > 0 ? n : 0))); });
}

int kvc_enforce_capacity(kvc_ctx* ctx, double* cost_us) {
  return guard([&] {
    const double c = F(ctx).api_enforce_capacity();
    if (cost_us) *cost_us = c;
  });
}

int kvc_visual_topk(kvc_ctx* ctx, const float* q, int32_t k, int64_t* ids) {
  std::vector<int64_t> r;
  const int rc = guard([&] { r = F(ctx).api_visual_topk(q, k); });
  return rc != KVC_OK ? rc : copy_out(r, ids, k);
}

int kvc_semantic_topk(kvc_ctx* ctx, const float* q, int32_t layer, const int64_t* partitions, int32_t n_parts,
                      int32_t k, int64_t* ids, int32_t* is_buffer) {
  int n = 0;
  const int rc = guard([&] {
    auto r = F(ctx).api_semantic_topk(q, layer, std::vector<int64_t>(partitions, partitions + (n_parts > 0 ? n_parts : 0)), k);
    n = static_cast<int>(r.size());
    for (int i = 0; i < n; ++i) {
      ids[i] = r[static_cast<std::size_t>(i)].first;
      is_buffer[i] = r[static_cast<std::size_t>(i)].second;
    }
  });
  return rc != KVC_OK ? rc : n;
}

int kvc_last_frames(kvc_ctx* ctx, int32_t which, int64_t* frames, int32_t cap) {
  if (which != 0 && which != 1) return KVC_E_CONFIG;
  if (ctx->tok) return copy_out(ctx->tok->last_frames(which), frames, cap);
  KVC_READER(ctx);
  return copy_out(which == 0 ? R(ctx).last_fetched_frames() : R(ctx).last_context_frames(), frames, cap);
}

int kvc_last_predicted(kvc_ctx* ctx, int32_t layer, int64_t* ids, int32_t cap) {
  if (ctx->tok) return 0;
  KVC_READER(ctx);
  const auto& ls = R(ctx).last_layers();
  if (layer < 0 || layer >= static_cast<int>(ls.size())) return KVC_E_BAD_LAYER;
  return copy_out(ls[static_cast<std::size_t>(layer)].predicted, ids, cap);
}

int kvc_debug_event_profile(kvc_ctx* ctx, double* out10, int32_t reset) {
  return guard([&] { F(ctx).event_profile(out10, reset != 0); });
}

int kvc_debug_wave_profile(kvc_ctx* ctx, double* out13, int32_t reset) {
  KVC_CLUSTER_ONLY(ctx);
  return guard([&] { ctx->impl->wave_profile(out13, reset != 0); });
}

int kvc_debug_resolve_profile(kvc_ctx* ctx, double* out) {
  if (ctx->tok) return guard([&] { ctx->tok->profile(out); });  // token-baseline select phases
  ctx->impl->resolve_profile(out);
  return KVC_OK;
}

int kvc_last_ingest_timing(kvc_ctx* ctx, double* t) {
  KVC_CLUSTER_ONLY(ctx);
  const double* s = ctx->impl->ingest_timing();
  for (int i = 0; i < 10; ++i) t[i] = s[i];
  return KVC_OK;
}

int kvc_host_split_two(const float* pts, int32_t n, int32_t d, uint64_t seed, int32_t* assign,
                       int32_t* degenerate) {
  int live = 0;
  const int rc = guard([&] {
    const kvc::KMeansOut o = kvc::split_two(pts, n, d, seed);
    for (int i = 0; i < n; ++i) assign[i] = o.assign[static_cast<std::size_t>(i)];
    if (degenerate) *degenerate = o.degenerate ? 1 : 0;
    live = o.k_live;
  });
  return rc != KVC_OK ? rc : live;
}

int kvc_host_kmeans(const float* pts, int32_t n, int32_t d, int32_t k, int32_t max_iters, double tol,
                    uint64_t seed, int32_t* assign, double* objective, int32_t* iterations) {
  int live = 0;
  const int rc = guard([&] {
    const kvc::KMeansOut o = kvc::spherical_kmeans(pts, n, d, k, max_iters, tol, seed);
    for (int i = 0; i < n; ++i) assign[i] = o.assign[static_cast<std::size_t>(i)];
    if (objective) *objective = o.objective;
    if (iterations) *iterations = o.iterations;
    live = o.k_live;
  });
  return rc != KVC_OK ? rc : live;
}

double kvc_host_tau(int64_t n, double tau_min, double tau_max, double n0) {
  return tau_min + (tau_max - tau_min) * std::exp(-static_cast<double>(n) / n0);  // maintainer.cpp:11-14
}

uint64_t kvc_host_mix_seed(uint64_t a, uint64_t b) { return kvc::mix_seed(a, b); }

void kvc_host_rng_first2(uint64_t seed, uint64_t* fast2, uint64_t* std2) {
  kvc::mt64_first2(seed, fast2);
  kvc::Rng64 r(seed);
  std2[0] = r.u64();
  std2[1] = r.u64();
}

}  // extern "C"
