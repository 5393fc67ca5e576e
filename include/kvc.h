/* kvc.h -- C-ABI of the B200-native cluster-level KV-cache hot path (Mosaic, arXiv 2604.10060).
 *
 * Drop-in boundary for the reference's `kvclust::core` hot path. The
 * reference has no FFI; its boundary is the C++ API of HierIndex / TieredStore / Maintainer /
 * retrieve driven by StreamEngine. Each entry point below names the reference interface it
 * replaces (paths relative to /root/reference/proj/core). Conventions:
 *   - plain pointers and sizes only; no C++ or torch types cross this ABI;
 *   - every call returns an int status (KVC_OK or a negative KVC_E_* code); C++ exceptions of
 *     the reference's kvclust::Error hierarchy (include/kvclust/error.hpp:9-82) map one-to-one
 *     onto the codes, and kvc_last_error() returns the message;
 *   - `mem` arguments say where a buffer lives: KVC_MEM_HOST (pageable or pinned host memory;
 *     the call copies it in/out on the context's stream) or KVC_MEM_DEVICE (device pointer on
 *     the context's GPU, consumed/produced in stream order);
 *   - a context is single-threaded like the reference: one writer.
 */
#ifndef KVC_H
#define KVC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status codes */
#define KVC_OK 0
#define KVC_E_GENERIC -1
#define KVC_E_DEGENERATE -2      /* DegenerateVector   error.hpp:15 */
#define KVC_E_DIM -3             /* DimMismatch        error.hpp:20 */
#define KVC_E_EMPTY_INPUT -4     /* EmptyInput         error.hpp:26 */
#define KVC_E_EMPTY_CLUSTER -5   /* EmptyCluster       error.hpp:31 */
#define KVC_E_TOO_FEW -6         /* TooFewPoints       error.hpp:36 */
#define KVC_E_BAD_LAYER -7       /* BadLayer           error.hpp:41 */
#define KVC_E_UNKNOWN_CLUSTER -8 /* UnknownCluster     error.hpp:46 */
#define KVC_E_EMPTY_INDEX -9     /* EmptyIndex         error.hpp:51 */
#define KVC_E_CONFIG -10         /* ConfigError        error.hpp:57 */
#define KVC_E_INVARIANT -11      /* InvariantViolation error.hpp:69 */
#define KVC_E_CUDA -20           /* CUDA runtime failure (no reference counterpart) */
#define KVC_E_CAPACITY -21       /* a device table/page pool is full (raise the kvc_cfg limit) */
#define KVC_E_NO_DEVICE -22      /* no CUDA device: the product has no CPU fallback */

#define KVC_MEM_HOST 0
#define KVC_MEM_DEVICE 1

#define KVC_DTYPE_F32 0
#define KVC_DTYPE_BF16 1

/* TransferCause (store.hpp:33) */
#define KVC_CAUSE_RETRIEVAL 0
#define KVC_CAUSE_MAINTENANCE 1
#define KVC_CAUSE_PREFETCH 2
#define KVC_CAUSE_COMPLETION 3
#define KVC_CAUSE_OFFLOAD 4

#if defined(__GNUC__)
#define KVC_API __attribute__((visibility("default")))
#else
#define KVC_API
#endif

typedef struct kvc_ctx kvc_ctx;

/* ------------------------------------------------------------------ configuration
 * The first block is EngineConfig flattened (engine.hpp:21-33 with RetrievalConfig
 * retrieval.hpp:20-32, MaintainerConfig maintainer.hpp:18-34, BuildConfig index.hpp:76-82,
 * CostModel store.hpp:17-31), field-for-field, same defaults (kvc_cfg_default). The second
 * block sizes the device data plane (no reference counterpart). */
typedef struct {
  int32_t k_v, k_s, window_frames, prefetch_k, prefetch_enabled, token_mode;
  int64_t token_budget;
  double lookup_cost_per_candidate_us, compute_cost_per_token_us;
  double tau_min, tau_max, n0;
  int32_t defer_host_splits, max_split_depth;
  double visual_floor;
  int32_t target_visual_cluster_size, target_semantic_cluster_size, kmeans_max_iters;
  double kmeans_tol;
  double alpha_us, beta_us_per_byte;
  int64_t bytes_per_entry, device_capacity_entries;
  int32_t build_batch_frames, batched_ingest;
  double ingest_overhead_us;
  int32_t offload_horizon_frames;
  uint64_t seed;
  /* ---- device data plane ---- */
  int32_t kv_dtype;            /* KVC_DTYPE_F32 (bit-exact fp32 keys) or KVC_DTYPE_BF16 */
  int32_t page_tokens;         /* tokens per K/V page (cluster-contiguous store); 0 (default) = auto:
                                  64, halved while the attention kernel's page ring does not fit */
  int64_t max_pages;           /* page-pool size (0 = derive from pool_bytes) */
  int64_t pool_bytes;          /* page-pool bytes when max_pages == 0, default 1 GiB */
  int32_t max_slots;           /* live-cluster table capacity, default 65536 */
  int32_t max_cluster_pages;   /* member pages per cluster, default 256 */
  int32_t max_buffer_pages;    /* pending-split buffer pages per cluster, default 64 */
  int32_t max_partitions;      /* visual partitions, default 4096 */
  int32_t max_candidates;      /* clusters (+ buffers) scored per domain per call, default 1024 */
  int32_t max_tokens;          /* tokens per frame, default 256 */
  int32_t parity_mode;         /* materialise attended (frame, token) sets on the host */
  int32_t check_invariants;    /* run the structural self-check after build/query (engine.cpp:91,235) */
  int32_t tier_stage_pages;    /* HBM staging pages for in-flight host-tier migrations, default 2048 */
  int64_t host_pool_bytes;     /* pinned host tier for Host-resident clusters, default 256 MiB */
} kvc_cfg;

KVC_API void kvc_cfg_default(kvc_cfg* cfg);

/* ------------------------------------------------------------------ lifetime
 * StreamEngine(const EngineConfig&, int d, int L)  (engine.hpp:64, engine.cpp:37-44).
 * L is the number of clustering domains (the reference's layer_id space; on a GQA model one
 * domain per (layer, KV head)). Binds the calling thread's current CUDA device. */
KVC_API int kvc_create(const kvc_cfg* cfg, int32_t d, int32_t L, kvc_ctx** out);
KVC_API void kvc_destroy(kvc_ctx* ctx);
KVC_API const char* kvc_last_error(void);
/* The context's compute stream (cudaStream_t as void*), for event timing / interop. */
KVC_API void* kvc_stream(kvc_ctx* ctx);

/* ------------------------------------------------------------------ hot path
 * Frame ingest: StreamEngine::process(Frame) (engine.cpp:134-174) = build buffering
 * (engine.cpp:161-166 -> build_index index.cpp:364-450), Maintainer::place_frame
 * (maintainer.cpp:37-53), Maintainer::on_insert for every (layer, token) in layer-major order
 * (maintainer.cpp:88-176), push_window / repin / apply_cadence (engine.cpp:54-132).
 * visual: [d] f32 host. keys/values: [L][T][d] in cfg.kv_dtype, host or device (`mem`).
 * assigned (optional, host [L*T]): routed cluster id per entry, the return value of
 * on_insert (-1 while the frame waits for the batch build). partition (optional): placed id. */
KVC_API int kvc_ingest_frame(kvc_ctx* ctx, int64_t frame_id, const float* visual, const void* keys,
                     const void* values, int32_t T, int32_t mem, int64_t* assigned,
                     int64_t* partition);

/* Decode step: StreamEngine::process(Query) (engine.cpp:176-237) -> retrieve()
 * (retrieval.cpp:45-143), then attention over each domain's attended set (members of the
 * selected clusters U the local window; no reference counterpart):
 * out[l] = sum_t softmax(q_l . k_t / sqrt(d)) v_t, fp32.
 * q: [L][d] f32 (`q_mem`); out: [L][d] f32 (`out_mem`), may be NULL. gt: ground-truth frames
 * for recall (host, may be NULL).
 * Asynchronous with device buffers: the call returns once the step is enqueued on kvc_stream();
 * a device `out` is valid in that stream's order and a device `q` must stay valid until then.
 * Host `out` is complete on return. The step's bookkeeping (the views below, ledger, stats) is
 * replayed while the next step runs, or on first read. */
KVC_API int kvc_decode_step(kvc_ctx* ctx, int64_t query_id, const float* q, int32_t q_mem, float* out,
                    int32_t out_mem, const int64_t* gt, int32_t n_gt);

/* Views of the last decode step's RetrievalResult (retrieval.hpp:49-71). Each returns the
 * element count and copies at most `cap` elements. */
KVC_API int kvc_last_ranked(kvc_ctx* ctx, int32_t layer, int64_t* ids, int32_t* is_buffer, int32_t cap);
KVC_API int kvc_last_selected(kvc_ctx* ctx, int32_t layer, int64_t* ids, int32_t cap);
/* attended (frame, token), sorted; needs cfg.parity_mode */
KVC_API int kvc_last_attended(kvc_ctx* ctx, int32_t layer, int64_t* frames, int32_t* tokens, int32_t cap);
/* lat[5] = lookup, transfer, stall, completion, compute (retrieval.hpp:39-47);
 * ints[5] = verified_clusters, prefetch_hits, rep_count, n_predicted, attended_count */
KVC_API int kvc_last_layer_meta(kvc_ctx* ctx, int32_t layer, double* lat, int64_t* ints);
/* dd[2] = ttft_us, recall */
KVC_API int kvc_last_query_meta(kvc_ctx* ctx, double* dd);
/* FNV-1a attended digest (engine.cpp:18-35); needs cfg.parity_mode */
KVC_API uint64_t kvc_last_digest(kvc_ctx* ctx);

/* oracle_flat_topk (retrieval.cpp:145-164) computed on the device: k best candidates of
 * rep_set(layer) for q ([d] f32 host). Returns the count. */
KVC_API int kvc_flat_topk(kvc_ctx* ctx, const float* q, int32_t layer, int32_t k, int64_t* ids,
                  int32_t* is_buffer);

/* Forces the batch build of buffered frames (engine.cpp:202 "a query cannot wait"). */
KVC_API int kvc_build_now(kvc_ctx* ctx);

/* Bulk construction: HierIndex::add_partition (index.cpp:59-69) + add_cluster
 * (index.cpp:97-120) for every cluster of one partition + TieredStore::adopt (store.cpp:82-86).
 * Installs, for each domain l, n_clusters[l] clusters whose members are the rows of
 * keys/values [L][N][d] (kv dtype, `mem`) with cluster index assign[l*N + i] in [0,C);
 * member (frame, token) = (frame_ids[i], token_ids[i]). Representatives / variances are the
 * exact Eq. 1/2 statistics (compute_representative / compute_variance, index.cpp:345-362).
 * Clusters are created layer by layer, cluster index ascending. Returns the partition id. */
KVC_API int kvc_bulk_load(kvc_ctx* ctx, const float* visual, const void* keys, const void* values,
                  int32_t N, int32_t C, const int32_t* assign, const int64_t* frame_ids,
                  const int32_t* token_ids, int32_t mem, int64_t* partition);

/* ------------------------------------------------------------------ index / store views */
KVC_API int kvc_n_clusters(kvc_ctx* ctx);
KVC_API int kvc_cluster_ids(kvc_ctx* ctx, int64_t* ids, int32_t cap);
/* info[10] = layer, parent, n_members, n_buffer, stat_count, lazy, residence (0 device,
 * 1 host), device_tail, first_frame, last_touch; var; rep[d]; buffer_rep[d] (fp64, read
 * back from the device masters). Mirrors ClusterRecord (index.hpp:29-50). */
KVC_API int kvc_cluster(kvc_ctx* ctx, int64_t id, int64_t* info, double* var, double* rep,
                double* buffer_rep);
/* members (which=0) or buffer (which=1) as (frame, token) in stored order */
KVC_API int kvc_cluster_entries(kvc_ctx* ctx, int64_t id, int32_t which, int64_t* frames,
                        int32_t* tokens, int32_t cap);
/* member / buffer payload rows read back from the device store: keys/values [n][d] f32 */
KVC_API int kvc_cluster_payload(kvc_ctx* ctx, int64_t id, int32_t which, float* keys, float* values,
                        int32_t cap);
KVC_API int kvc_n_partitions(kvc_ctx* ctx);
KVC_API int kvc_partition(kvc_ctx* ctx, int32_t p, double* visual_rep, int64_t* frames, int32_t cap);
KVC_API int kvc_partition_layer(kvc_ctx* ctx, int32_t p, int32_t layer, int64_t* ids, int32_t cap);
/* MaintainerStats (maintainer.hpp:36-46) -> out[9] */
KVC_API int kvc_maint_stats(kvc_ctx* ctx, int64_t* out);
/* TransferLedger totals per cause (store.cpp:21-65): ops[5], bytes[5], cost_us[5];
 * returns TieredStore::device_entries (store.hpp:97) */
KVC_API int64_t kvc_ledger(kvc_ctx* ctx, int64_t* ops, int64_t* bytes, double* cost_us);
KVC_API int kvc_ledger_log_size(kvc_ctx* ctx);
/* op i: ints[4] = cause, to_device, cluster_id, bytes */
KVC_API int kvc_ledger_op(kvc_ctx* ctx, int32_t i, int64_t* ints);
/* HierIndex::check_invariants (index.cpp:263-343) + TieredStore::audit (store.cpp:183-189),
 * including device-vs-host agreement of counts and page tables. */
KVC_API int kvc_check(kvc_ctx* ctx);

/* TieredStore::offload / fetch (store.cpp:95-130) for one cluster. Returns the simulated cost
 * in *cost_us (the reference's ledger arithmetic). */
KVC_API int kvc_offload(kvc_ctx* ctx, int64_t id, double* cost_us);
KVC_API int kvc_fetch(kvc_ctx* ctx, int64_t id, int32_t cause, double* cost_us);

/* ------------------------------------------------------------------ physical host tier
 * TieredStore's Host residence is physical: a Host cluster's member pages live in one contiguous
 * extent of pinned host memory and every residence change is migrated by one cudaMemcpyAsync
 * per cluster on a transfer stream (K5), asynchronously. Kernels address pages wherever they
 * physically are, so results never depend on migration progress.
 * kvc_tier_sync completes every queued / in-flight migration (physical == logical residence).
 * A decode step copies the host pages of the clusters it selected into HBM itself, between
 * selection and attention (fetch-on-read: one crossing of the host link; KVC_FETCH_ON_READ=0
 * leaves them to the queued fetch migrations while attention reads them in place).
 * kvc_tier_stats out[14]: host pages in use, host-tier capacity (pages), clusters with host pages,
 * offloads committed, fetches committed, bytes device->host, bytes host->device, migrations
 * queued, batches in flight, HBM staging pages in use, batches started, DMA copies issued
 * (per-cluster copies merged when both sides are contiguous), fetches done by fetch-on-read and
 * their bytes (included in the fetch / host->device totals). */
KVC_API int kvc_tier_sync(kvc_ctx* ctx);
KVC_API int kvc_tier_stats(kvc_ctx* ctx, int64_t* out);
/* out[3]: first host page of the cluster's extent (-1 none), its length in pages, migration busy */
KVC_API int kvc_cluster_tier(kvc_ctx* ctx, int64_t id, int64_t* out);
/* Debug: every live page table against the host's view of the tiers (reads each list; small
 * contexts). out[4]: host page ids outside their cluster's extent, Device clusters holding host
 * pages, Host clusters with all member pages in HBM, clusters whose page fills disagree with the
 * member count / logical device tail. All zero after kvc_tier_sync. */
KVC_API int kvc_debug_tier_check(kvc_ctx* ctx, int64_t* out4);
/* split_two (clustering.cpp:180-208) of n host points (the context's d) through the device split
 * kernel the maintenance slow path uses (split.cu); meta3 = {k_live, iterations, degenerate}.
 * Bit-identical to kvc_host_split_two / kvc_host_kmeans(k=2, 50, 1e-9). Returns k_live or < 0. */
/* spherical_kmeans (clustering.cpp:80-178) of n_sets host point sets (rows concatenated, the
 * context's d) through the batch-build device kernel (kmeans_dev.cu), as the index build runs it;
 * meta2[2i] = k_live, meta2[2i+1] = iterations. Bit-identical to kvc_host_kmeans. */
KVC_API int kvc_debug_kmeans(kvc_ctx* ctx, const float* pts, int32_t n_sets, const int32_t* n, const int32_t* k,
                             int32_t max_iters, double tol, const uint64_t* seeds, int32_t* assign, int32_t* meta2,
                             double* objective);
KVC_API int kvc_debug_split_two(kvc_ctx* ctx, const float* pts, int32_t n, uint64_t seed, int32_t* assign,
                                int32_t* meta3, double* objective);

/* ------------------------------------------------------------------ multi-GPU: fused output exchange
 * Domains are sharded over ranks (one process per GPU). Instead of an all-gather pass after each
 * decode step, the attention kernel's split-KV combine stores every finished output row directly
 * into every rank's exchange buffer over peer memory (NVLink; CUDA IPC mappings), and a per-step
 * signal/wait pair orders the ranks. Exchange buffer of a rank (kvc_ipc_alloc,
 * kvc_exchange_bytes): [2 step parities][total_domains][d] f32 followed by n_ranks u64 flags,
 * zero-initialised. Each rank passes the mapped buffers of all ranks (its own included), in rank
 * order, to kvc_set_peers; every rank must then run the same number of decode steps.
 * kvc_peer_output copies the last step's gathered [total_domains][d] outputs (stream order). */
KVC_API size_t kvc_exchange_bytes(int32_t n_ranks, int32_t total_domains, int32_t d);
KVC_API int kvc_ipc_alloc(size_t bytes, void** dptr, uint8_t* handle64);
KVC_API int kvc_ipc_open(const uint8_t* handle64, void** dptr);
KVC_API int kvc_ipc_close(void* dptr);
KVC_API int kvc_ipc_free(void* dptr);
KVC_API int kvc_set_peers(kvc_ctx* ctx, int32_t n_ranks, int32_t rank, int32_t dom_offset, int32_t total_domains,
                          void* const* bufs);
KVC_API int kvc_peer_output(kvc_ctx* ctx, float* out, int32_t mem);

/* ------------------------------------------------------------------ component-level API
 * The reference's HierIndex / TieredStore / Maintainer / retrieve calls one at a time (the C++
 * drop-in include/kvclust_b200.hpp is built on these; engine-level callers use the hot path
 * above). Payloads are f32 (kv_dtype f32 contexts). */
/* HierIndex::add_partition (index.cpp:59-69) / append_frame (index.cpp:71-79) */
KVC_API int kvc_add_partition(kvc_ctx* ctx, int64_t first_frame, const float* visual, int64_t* partition);
KVC_API int kvc_append_frame(kvc_ctx* ctx, int64_t partition, int64_t frame_id, const float* visual);
/* HierIndex::add_cluster (index.cpp:97-120) + TieredStore::adopt (store.cpp:82-86) when `adopt`:
 * n members keys/values [n][d] f32 host with their (frame, token) ids; representative and variance
 * are the exact Eq. 1/2 statistics (compute_representative / compute_variance), computed on the
 * device; residence 0 Device / 1 Host. *id receives the new cluster id. */
KVC_API int kvc_add_cluster(kvc_ctx* ctx, int32_t layer, int64_t partition, int32_t n, const float* keys,
                            const float* values, const int64_t* frames, const int32_t* tokens, int32_t residence,
                            int32_t adopt, int64_t* id);
KVC_API int kvc_adopt(kvc_ctx* ctx, int64_t id);
/* Verbatim installs (a parsed or host-assembled index, index.hpp:29-58): a VisualPartition with its
 * frame list, fp64 visual_rep and visual_stat_count; a ClusterRecord with members AND pending-split
 * buffer entries and the caller's rep / variance / stat_count / buffer_rep / lazy flag / residence /
 * device tail (not recomputed). want_id >= the next id keeps the record's id (ids are never reused,
 * index.cpp:105); -1 assigns the next one. */
typedef struct {
  int32_t layer;
  int64_t partition;
  int32_t n_members;
  const float *member_keys, *member_values; /* [n_members][d] f32 */
  const int64_t* member_frames;
  const int32_t* member_tokens;
  int32_t n_buffer;
  const float *buffer_keys, *buffer_values; /* [n_buffer][d] f32 */
  const int64_t* buffer_frames;
  const int32_t* buffer_tokens;
  const double* rep;        /* [d] */
  double variance;
  int64_t stat_count;
  const double* buffer_rep; /* [d] or NULL */
  int32_t lazy_split, residence, adopt;
  int64_t device_tail, want_id;
} kvc_cluster_record;
KVC_API int kvc_add_partition_ex(kvc_ctx* ctx, const int64_t* frames, int32_t n_frames, const double* visual_rep,
                                 int64_t visual_stat_count, int64_t* partition);
KVC_API int kvc_add_cluster_ex(kvc_ctx* ctx, const kvc_cluster_record* record, int64_t* id);
/* retrieve()'s explicit local window (retrieval.hpp:73-75) empty: no window entries attended */
KVC_API int kvc_reset_window(kvc_ctx* ctx);
/* Per-call RetrievalConfig (retrieval.hpp:20-32): k_v, k_s, prefetch_k, prefetch_enabled and the
 * lookup / compute cost constants are taken from cfg (other fields ignored). */
KVC_API int kvc_set_retrieval(kvc_ctx* ctx, const kvc_cfg* cfg);
/* Re-configures a live context from cfg, `what` bits: 1 the RetrievalConfig fields (as
 * kvc_set_retrieval), 2 the CostModel (TieredStore(index, cost), store.hpp:17-31: alpha_us,
 * beta_us_per_byte, bytes_per_entry, device_capacity_entries), 4 the MaintainerConfig
 * (Maintainer(index, store, cfg), maintainer.hpp:28-34: tau_min / tau_max / n0, defer_host_splits,
 * max_split_depth, visual_floor; cfg.seed is taken as MaintainerConfig::seed itself), 8 the
 * BuildConfig of a direct build_index call (index.hpp:76-82: target sizes, k-means iterations /
 * tolerance; cfg.seed is taken as BuildConfig::seed itself). */
KVC_API int kvc_reconfigure(kvc_ctx* ctx, const kvc_cfg* cfg, int32_t what);
/* Maintainer::place_frame (maintainer.cpp:37-53) / on_insert (maintainer.cpp:88-176): one entry of
 * one domain resolved on the device (no window row); *cluster receives the routed id. */
KVC_API int kvc_place_frame(kvc_ctx* ctx, int64_t frame_id, const float* visual, int64_t* partition);
KVC_API int kvc_insert(kvc_ctx* ctx, int64_t partition, int32_t layer, int32_t token, int64_t frame_id,
                       const float* key, const float* value, int64_t* cluster);
/* Maintainer::materialize (maintainer.cpp:178-193): returns the count of replacement ids */
KVC_API int kvc_materialize(kvc_ctx* ctx, int64_t id, int64_t* ids, int32_t cap);
/* TieredStore::touch / pin (replaces the pinned set) / enforce_capacity (store.cpp:139-164) */
KVC_API int kvc_touch(kvc_ctx* ctx, int64_t id);
KVC_API int kvc_pin(kvc_ctx* ctx, const int64_t* ids, int32_t n);
KVC_API int kvc_enforce_capacity(kvc_ctx* ctx, double* cost_us);
/* visual_topk (index.cpp:192-208) / semantic_topk (index.cpp:210-240) on the device; return counts */
KVC_API int kvc_visual_topk(kvc_ctx* ctx, const float* q, int32_t k, int64_t* ids);
KVC_API int kvc_semantic_topk(kvc_ctx* ctx, const float* q, int32_t layer, const int64_t* partitions, int32_t n_parts,
                              int32_t k, int64_t* ids, int32_t* is_buffer);
/* RetrievalResult fetched_frames (which = 0) / context_frames (which = 1) of the last decode step
 * (retrieval.cpp:99-110; needs cfg.parity_mode or ground truth). Returns the count. */
KVC_API int kvc_last_frames(kvc_ctx* ctx, int32_t which, int64_t* frames, int32_t cap);
/* LayerResult::predicted of the last decode step (clusters prefetched for this layer) */
KVC_API int kvc_last_predicted(kvc_ctx* ctx, int32_t layer, int64_t* ids, int32_t cap);

/* ------------------------------------------------------------------ instrumentation */
/* Kernel launches issued by this context since creation (for bench gpu_launches). */
KVC_API int64_t kvc_launch_count(kvc_ctx* ctx);
/* Timing of the last decode step (needs kvc_set_timing(1)), t[8]: device phases in
 * microseconds from CUDA events -- t[0] score/select, t[1] attention (+ fused combine), t[2]
 * unused, t[3] launch-to-end on the device; t[4] algorithmic bytes of the attention launch;
 * host phases in microseconds -- t[5] wait for the device, t[6] retrieve bookkeeping replay,
 * t[7] repin + checks; t[8], t[9] unused. t has 10 entries. */
KVC_API int kvc_last_step_timing(kvc_ctx* ctx, double* t);
/* Timing of the last ingested frame (needs kvc_set_timing(1)), t[8]: device microseconds of
 * the candidate lists, approximate tile, top-M + exact pre-scores, sequential resolve and row
 * store kernels (t[0..4], summed over launches); host microseconds waiting for the device (t[5])
 * and of everything else in the on_insert loop incl. replay and host events (t[6]), of which the
 * outcome replay loop (t[7]) and relaunch issue (t[8]); t[9] the number of host events (seeds /
 * splits) the frame needed. t must hold 10 doubles. */
KVC_API int kvc_last_ingest_timing(kvc_ctx* ctx, double* t);
/* Host slow-path primitives (no GPU needed), exported so the split / batch-build arithmetic can
 * be checked bit-for-bit against the reference on CPU:
 * split_two (clustering.cpp:180-208) and spherical_kmeans (clustering.cpp:80-178) over
 * pts[n][d] f32; assign[n] receives the dense cluster index. Return the live cluster count
 * (split_two: 2; *degenerate set for the (n-1, 1) rule) or a negative KVC_E_* code. tau
 * (maintainer.cpp:11-14) and mix_seed (rng.hpp:47-52) as used by the device threshold table and
 * the split seed sequence. */
KVC_API int kvc_host_split_two(const float* pts, int32_t n, int32_t d, uint64_t seed, int32_t* assign,
                               int32_t* degenerate);
KVC_API int kvc_host_kmeans(const float* pts, int32_t n, int32_t d, int32_t k, int32_t max_iters, double tol,
                            uint64_t seed, int32_t* assign, double* objective, int32_t* iterations);
KVC_API double kvc_host_tau(int64_t n, double tau_min, double tau_max, double n0);
KVC_API uint64_t kvc_host_mix_seed(uint64_t a, uint64_t b);
/* Test hook: the first two outputs of mt19937_64(seed) from the wave engine's shortcut (fast2)
 * and from std::mt19937_64 (std2). */
KVC_API void kvc_host_rng_first2(uint64_t seed, uint64_t* fast2, uint64_t* std2);
/* Instrumentation: mean clock64 cycles per phase of the last resolve launch (out[16]; with
 * out[0] < 0 on entry: of the last decode's score/select kernel, first 8 entries). */
/* Device self-check of the reciprocal-based correctly rounded division used on the resolve
 * chains against __ddiv_rn: n random (a, b) pairs, integer b in [1, max_den]; *mismatches
 * receives the count of differing results. */
/* Device self-check of the frame-ingest distance tile: runs the candidate build and the distance
 * tile (tensor-core or SIMT, whichever the context uses) + top-M for a frame keys[L][T][d] (kv
 * dtype, host or device) against `partition` without inserting anything, then compares every
 * (token, candidate) approximate cosine with the exact fp64 cosine. out4: max |approx - exact|,
 * candidates outside a top-M list scoring above its (M+1)-th value, top-M exact values that differ
 * from a fresh exact cosine, and the margin the resolve kernels certify with. */
KVC_API int kvc_debug_assign_check(kvc_ctx* ctx, const void* keys, int32_t T, int64_t partition, int32_t mem,
                                   double* out4);
/* Debug: the kernels' reciprocal division (one RN(1/b) + two FMA corrections) against __ddiv_rn on
 * n random operands: integer divisors in [1, max_den], or (max_den <= 0) real divisors in
 * [2^-8, 2^8) with float numerators (the unit rows of the split k-means). */
KVC_API int kvc_debug_div_check(uint64_t n, uint64_t seed, int32_t max_den, uint64_t* mismatches);
/* Debug: per-domain averages of the last resolve round's phase clocks, out16 (the speculative
 * kernel always records them; the sequential kernel only with KVC_RESOLVE_PROF=1); out[0] < 0 on
 * entry selects the decode step's K4 clocks instead. */
KVC_API int kvc_debug_resolve_profile(kvc_ctx* ctx, double* out);
/* Host-event slow path profile (cumulative since creation / the last reset), out10: microseconds in
 * host events (split / seed) total, of which staging + download of the cluster rows, split k-means
 * (split_two calls), host Eq. 1/2 statistics of the children, slot / page / list uploads; then the
 * relaunch-and-wait of a domain after an event; the number of host events and of split_two calls;
 * speculative split k-means launched / consumed (the next domain's split 2-means'd on a side
 * stream during a relaunch). */
KVC_API int kvc_debug_event_profile(kvc_ctx* ctx, double* out10, int32_t reset);
/* Wave engine profile (parallel settle of a frame's host events across domains; cumulative), out13:
 * frames with events, waves, verification passes, rolled-back domains, verification k-means jobs,
 * host events, then microseconds in pool staging, k-means jobs (count), k-means, children
 * statistics + install, relaunch rounds, verification + commit; splits verified as the same
 * partition with exchanged labels. */
KVC_API int kvc_debug_wave_profile(kvc_ctx* ctx, double* out13, int32_t reset);
/* Enables per-phase CUDA-event timing (off by default: it adds event records). */
KVC_API void kvc_set_timing(kvc_ctx* ctx, int32_t on);
/* Rows zero-padded to the context's width d (a caller with a narrower head width, e.g. the C++
 * drop-in for d % 8 != 0): attention keeps the softmax scale 1/sqrt(d_logical). Everything else
 * of the path is a sequential sum over the elements, unchanged by trailing zeros. */
KVC_API int kvc_set_head_dim(kvc_ctx* ctx, int32_t d_logical);

#ifdef __cplusplus
}
#endif
#endif /* KVC_H */
