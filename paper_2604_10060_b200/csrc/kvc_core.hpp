// kvc_core.hpp -- declarations shared by the host control plane (context.cpp) and the
// sm_100a kernels (kernels.cu). Plain structs of device pointers; no torch.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

namespace kvc {

// ----------------------------------------------------------------------------- errors
// One exception type carrying a KVC_E_* code; the C-ABI turns it into the return value.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define KVC_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      ::kvc::fail(-20, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #expr); \
  } while (0)

// ----------------------------------------------------------------------------- events
// Per-(domain, token) outcome of the device resolve kernel (maintainer.cpp:88-176 branches).
enum EventKind : int32_t {
  EV_NONE = 0,
  EV_ABSORB = 1,   // add_member + note_device_append          (maintainer.cpp:132-137)
  EV_BUFJOIN = 2,  // buffer candidate won: add_to_buffer        (maintainer.cpp:112-123)
  EV_DEFER = 3,    // over threshold on a Host cluster: lazy mark (maintainer.cpp:170-175)
  EV_SEED = 4,     // host: empty candidate set -> seed_cluster   (maintainer.cpp:93-94)
  EV_SPLIT = 5,    // host: over threshold on a Device cluster    (maintainer.cpp:139-149)
  EV_EAGER = 6,    // host: eager policy fetch + split            (maintainer.cpp:153-166)
};

// Device error flags (bit set in DevTables::err).
enum DevErr : int32_t {
  DERR_DEGENERATE = 1,  // a norm below 1e-12 met a cosine (vecmath.hpp:59)
  DERR_PAGES = 2,       // page pool exhausted
  DERR_CLUSTER_PAGES = 4,
  DERR_CANDIDATES = 8,  // more candidates than max_candidates
  DERR_ITEMS = 16,      // attention work list overflow
  DERR_TIER = 32,       // a host-tier page outside its cluster's extent
  DERR_TAKE = 64,       // more than 64 ranked candidates per domain (k_s / prefetch_k x candidates)
};

// ----------------------------------------------------------------------------- device state
// Cluster tables are SoA indexed by a device *slot*; the host maps slots <-> cluster ids.
// K/V live in a page pool: page p = [K: page_tokens x d][V: page_tokens x d] in kv dtype,
// cluster-contiguous (a cluster's members are its pages in order; buffered entries of a
// pending split use a second page list).
struct DevTables {
  int32_t d, L, P, es;  // dim, domains, page tokens, element size (4 f32 / 2 bf16)
  int32_t kv_bf16;
  int32_t max_slots, maxp, maxbp, max_parts, cmax, tmax, W;
  int64_t max_pages, page_bytes;

  double* rep64;   // [S][d] running centroid (Eq. 3), fp64 master
  float* rep32;    // [S][d] fp32 mirror for the approximate tile
  double* rnorm;   // [S]    norm(rep) (vecmath.hpp:35-40), cached bit-exactly
  double* brep64;  // [S][d] pending-buffer running mean (index.cpp:177-190)
  float* brep32;
  double* bnorm;
  double* var;     // [S]    running variance (Eq. 4)
  int64_t* stat;   // [S]    stat_count
  int64_t* nmem;   // [S]    members
  int32_t* nbuf;   // [S]    buffered entries
  uint8_t* lazy;   // [S]    lazy_split (== buffer registered)
  uint8_t* resid;  // [S]    0 Device, 1 Host
  int64_t* cid;    // [S]    cluster id (tie-break key)
  int32_t* npages; // [S]
  int32_t* pages;  // [S][maxp]
  int32_t* nbpages;
  int32_t* bpages; // [S][maxbp]
  int32_t* pg_fill;     // [max_pages + max_hpages] rows used in each page (HBM, then host tier)
  int32_t* free_stack;  // [max_pages]
  int32_t* free_top;    // [1]
  uint8_t* pool;        // page pool (HBM)
  // host tier (TieredStore Host residence, store.cpp:95-130): pinned, mapped host pages in the
  // same page format. Page ids >= max_pages name host page (id - max_pages); every kernel reaches
  // them through page_k/page_v, so attention over a not-yet-fetched cluster reads host memory.
  uint8_t* hpool;
  int64_t max_hpages;
  // [S] leading member pages that are sealed (moved to / copied for the host tier): appends
  // never write into them, so an offload's snapshot stays valid while its copy is in flight
  int32_t* seal;
  // window ring (engine.cpp:54-65): W frame slots per domain, each ceil(tmax/P) pages
  int32_t* ring_pages;  // [L][W][rpp]
  int32_t* ring_owner;  // [L][W][tmax] owning slot of each window token (-1 none)
  int32_t* ring_count;  // [W] tokens in the frame held by each ring slot (0 empty)
  int32_t rpp;          // ring pages per frame slot
  // visual partitions (index.hpp:52-58)
  double* vrep;   // [max_parts][d]
  double* vnorm;  // [max_parts]
  int32_t* n_parts;  // [1]
  // per (partition, domain) live-cluster slot lists (per_layer_clusters order)
  int32_t* pl_off;   // [max_parts * L]
  int32_t* pl_cnt;   // [max_parts * L]
  int32_t* pl_pool;
  int64_t pl_pool_cap;
  // Eq. 5 threshold table tau[n] computed on the host with libm exp (maintainer.cpp:11-14)
  double* tau_tab;
  int32_t tau_len;
  int32_t* err;  // [1] DevErr bits
};

inline __host__ __device__ bool is_host_page(const DevTables& t, int32_t page) {
  return page >= t.max_pages;
}
inline __host__ __device__ uint8_t* page_k(const DevTables& t, int32_t page) {
  return page < t.max_pages ? t.pool + static_cast<int64_t>(page) * t.page_bytes
                            : t.hpool + (static_cast<int64_t>(page) - t.max_pages) * t.page_bytes;
}
inline __host__ __device__ uint8_t* page_v(const DevTables& t, int32_t page) {
  return page_k(t, page) + static_cast<int64_t>(t.P) * t.d * t.es;
}

// ----------------------------------------------------------------------------- ingest
struct IngestArgs {
  int32_t T, pid, ring_slot, n_active;
  const int32_t* active;   // [n_active] domains to run (device)
  const int32_t* cursor;   // [L] first token to process per domain (device)
  const void* fk;          // [L][tmax][d] frame keys (kv dtype)
  const void* fv;
  // candidate lists (built per launch)
  int32_t* cand_n;         // [L]
  int32_t* cand_slot;      // [L][cmax]
  uint8_t* cand_buf;       // [L][cmax]
  float* approx;           // [L][tmax][cmax] approximate cosines (K1)
  float margin;            // certified bound on |approx - exact| (cosine units)
  int32_t defer;           // MaintainerConfig::defer_host_splits
  // the tile's epilogue computes the exact cosine of every top-M candidate, not only those within
  // 2 margins of the best (a relaunch after a split: the new children take the best tokens, so
  // the resolve would otherwise re-score the runner-up candidates from global memory per token)
  int32_t exact_all;
  // outputs
  int32_t* ev_kind;        // [L][tmax]
  int32_t* ev_slot;        // [L][tmax]
  int32_t* stop_t;         // [L] token index of the host event (T when done)
  int32_t* stop_kind;      // [L]
  int32_t* stop_slot;      // [L]
  int32_t* n_exact;        // [L] exact re-scores performed (instrumentation)
  int32_t* tie;            // [L] (k_resolve) 1: a decision of the launch was an exact cosine tie
                           // broken by the cluster-id key (in the outcome block, after the error word)
  // per-token approximate top-M (K1b): candidate index, value, and the (M+1)-th value
  int16_t* topm_idx;       // [L][tmax][TOPM]
  float* topm_val;         // [L][tmax][TOPM]
  float* topm_next;        // [L][tmax]
  double* topm_exact;      // [L][tmax][TOPM] exact cosine vs the launch-time representative (K1c)
  // destination of each committed row (page, row) for the parallel store pass (K3)
  int32_t* ev_page;        // [L][tmax]
  int32_t* ev_row;         // [L][tmax]
  // per-domain reserve of free pages carried between resolve launches (no pushes to the
  // shared free stack while pops may run concurrently)
  long long* prof;         // [L][16] clock64 cycles per resolve phase (instrumentation)
  int32_t prof_on;         // the sequential resolve records its per-token phase clocks (timing mode)
  int32_t* dom_pool;       // [L][POOL]
  int32_t* dom_pool_n;     // [L]
  // speculative resolve (resolve_spec.cu): per-token state snapshots, column-major so that
  // one thread per token reads them coalesced
  // speculative next frame: a round launched behind the previous frame's first round before
  // its outcome is known; it commits nothing if that round stopped any domain (*prev_events)
  int32_t* err_copy;            // the error word, copied by K3 into the outcome block (one D2H)
  const int32_t* prev_events;  // null: not speculative
  int32_t* my_events;          // this frame's first-round flag: some domain stopped early
  double* rsnap;           // [L][d][tmax] representative after each token's insert
  double* bsnap;           // [L][d][tmax] buffer mean after each buffer-moving insert
};
constexpr int TOPM = 8;
constexpr int POOL = 16;

// ----------------------------------------------------------------------------- decode
// Fused output exchange across ranks (multi-GPU by domain): K6's combine (and K4's path for a
// domain with nothing attended) stores each finished output row straight into every rank's full
// output buffer over peer memory (NVLink P2P stores; CUDA IPC mappings), instead of a separate
// all-gather pass; a per-step signal/wait pair of tiny kernels orders the ranks.
constexpr int kMaxPeers = 8;
struct PeerOut {
  int32_t n;           // ranks (0: no fused exchange)
  int32_t dom_offset;  // this rank's first global domain
  float* out[kMaxPeers];  // rank p's full output buffer [total domains][d] (mapped)
};

struct DecodeArgs {
  const float* q;          // [L][d] (device)
  const float* q_src;      // non-null: the query lives in pinned host memory; K4 reads it from
                           // there (zero-copy) and writes the device copy q for K6
  int32_t k_v, k_s, prefetch_k, prefetch;
  int32_t n_parts_host;    // partitions known to the host (== device count)
  // outputs (device)
  int32_t* parts;          // [L][k_v]    visual_topk partition ids
  int32_t* n_parts_sel;    // [L]
  int32_t* ranked_slot;    // [L][k_s]
  uint8_t* ranked_buf;     // [L][k_s]
  int32_t* n_ranked;       // [L]
  int32_t* pf_slot;        // [L][prefetch_k] ranking of layer l+1 candidates with q_l
  uint8_t* pf_buf;
  int32_t* n_pf;           // [L]
  int32_t* ver_slot;       // [L][k_s]    verified (dedup, rank order)
  int32_t* n_ver;          // [L]
  int64_t* attended;       // [L]        attended-set size (members+buffers of verified U window)
  int32_t* n_cand;         // [L]        candidates compared (count_candidates)
  int32_t* flags;          // [L] 1: a verified cluster of the domain has a pending split (host settle)
  int32_t* errw;           // [L] the device error word as seen by the domain's K4 block at its end
  // attention work list: page descriptors per domain (x page, y fill, z kind | ring_slot << 8,
  // w first token of the page within its frame); an item = chunk_pages consecutive descriptors
  int4* desc;              // [L][max_desc]
  int32_t* n_desc;         // [L]
  int32_t* n_items;        // [L] = ceil(n_desc / chunk_pages)
  int32_t max_desc, max_items, chunk_pages;
  // attention partials / output
  float* part_ml;          // [L][max_items][2]
  float* part_o;           // [L][max_items][d]
  int32_t* dom_done;       // [L] completion counters (reset by the combine)
  float* out;              // [L][d]
  float scale_log2;        // log2(e) / sqrt(d)
  long long* k4prof;       // [L][8] clock64 phase cycles (instrumentation; may be null)
  int32_t* work_ctr;       // attention work-claim counter (per context: contexts may run concurrently)
  int32_t debug_flags;     // instrumentation experiments only (KVC_ATT_DEBUG); 0 in production
  int32_t l2pf_pages;      // pages per domain K4 prefetches into L2 while it is latency bound
  int32_t att_pf;          // K6 producer: the item's page this many pages ahead prefetched into L2 (0: off)
  PeerOut peer;            // fused output exchange (multi-GPU); peer.n == 0 when unused
  // fetch-on-read (select.cu R6 + tiers.cu k_fetch_read): a verified cluster whose member pages
  // are in the host tier gets fresh HBM pages in K4 (all of its host pages or none, never below
  // fr_reserve free pages); K4 points the work list at them and lists the copies, which
  // k_fetch_read performs between K4 and K6 (one crossing of the host link instead of K6 reading
  // in place and the fetch migration reading again). The host drops the cluster's extent from
  // fr_rec when it replays the step (the reference's fetch of that cluster, store.cpp:95-116).
  int32_t fr_on;           // 0: off (no host pages, K4 v1/v2, KVC_FETCH_ON_READ=0)
  int32_t fr_reserve;      // free HBM pages K4 leaves untouched
  int32_t fr_max;          // records per domain in fr_rec (>= k_s)
  int4* fr_jobs;           // [L][max_desc] {host page, HBM page, slot, page index}
  int32_t* fr_nj;          // [L] copies listed by K4
  int32_t* fr_n;           // [L] migrated clusters (result block; written by K4 in every mode)
  int4* fr_rec;            // [L][fr_max] {cluster id lo, hi, extent's first host page, pages}
};

// ----------------------------------------------------------------------------- launchers
// Implemented in kernels.cu. All launch on `st`; each returns the number of kernel launches.
int launch_build_cands(const DevTables& t, const IngestArgs& a, cudaStream_t st);
int launch_approx(const DevTables& t, const IngestArgs& a, cudaStream_t st);
int launch_resolve(const DevTables& t, const IngestArgs& a, cudaStream_t st);
// Speculate-and-verify resolve (resolve_spec.cu). Returns 0 (nothing launched) when the
// shape does not fit its shared-memory plan; the caller then uses launch_resolve.
int launch_resolve_spec(const DevTables& t, const IngestArgs& a, cudaStream_t st);
// Tensor-core distance tile + top-M (assign_tc.cu) for bf16 frames with d in {64, 128}: replaces
// launch_approx + launch_topm. key_map: a CUtensorMap over the frame keys [L][tmax][d] made by
// make_key_tensor_map (128-byte swizzle, 64 x 128 boxes).
bool assign_tc_supported(const DevTables& t);
bool make_key_tensor_map(void* map, const void* keys, int d, int tmax, int L);
int launch_assign_tc(const DevTables& t, const IngestArgs& a, const void* key_map, cudaStream_t st);
int launch_assign_err(const DevTables& t, const IngestArgs& a, unsigned long long* out, cudaStream_t st);
constexpr float kSimtMargin = 1e-4f;  // |approx - exact| bound of the fp32 SIMT tile
constexpr float kTcMargin = 2e-4f;    // ... of the bf16 hi/lo tensor-core tile
// Counts div_rcp != __ddiv_rn over n random operands on the device (~0 on CUDA failure).
uint64_t debug_div_check(uint64_t n, uint64_t seed, int max_den);
int launch_topm(const DevTables& t, const IngestArgs& a, cudaStream_t st);
// The launch's frame rows [cursor, T) of every active domain -> window ring; committed ones also
// -> the (page, row) the resolve kernel reserved.
int launch_store_rows(const DevTables& t, const IngestArgs& a, cudaStream_t st);
// Frame start: the ring slot's owner entries / page fills / token count. Its rows are written by
// launch_store_rows (routed frames) or launch_ring_rows (frames pending the batch build).
int launch_ring_rows(const DevTables& t, const void* fk, const void* fv, int32_t T, int32_t rs, cudaStream_t st);
int launch_ring_write(const DevTables& t, const void* fk, const void* fv, int32_t T,
                      int32_t ring_slot, cudaStream_t st);
// K6 alone over a prepared work list (desc / n_desc / n_items / partials / out of `a`; the work
// counter a.work_ctr must be zero). Used by the token-level baseline.
int launch_attend(const DevTables& t, const DecodeArgs& a, cudaStream_t st);

// Fused exchange signalling: rank `rank` publishes `step` into slot `rank` of every rank's flag
// array (after a system-scope fence, so its output stores are visible first); the wait kernel
// blocks the stream until every slot of this rank's flag array has reached `step`.
int launch_peer_signal(unsigned long long* const* flags, int n, int rank, unsigned long long step, cudaStream_t st);
int launch_peer_wait(const unsigned long long* my_flags, int n, unsigned long long step, cudaStream_t st);

// K4 v3 (select.cu); false when the shape does not fit it.
bool launch_select3(const DevTables& t, const DecodeArgs& a, cudaStream_t st);
// k4_done (may be null) is recorded between the score/select and attention kernels.
int launch_decode(const DevTables& t, const DecodeArgs& a, cudaStream_t st, cudaEvent_t* ev,
                  cudaEvent_t k4_done = nullptr);

// Slot initialisation from host-computed exact statistics: rep64 rows (rep, norm, var,
// counts) uploaded by the host; this kernel fills the fp32 mirrors.
int launch_refresh_mirror(const DevTables& t, const int32_t* slots, int32_t n, cudaStream_t st);

// Appends staged rows (kv dtype, [rows][d] K and V) to slots: run r appends rows
// idx[first .. first + n_rows) in order to the member (or buffer) pages of run.slot.
// One warp per run (runs must name distinct slots).
struct AppendRun {
  int32_t slot, first_row, n_rows, to_buffer;
};
int launch_append_runs(const DevTables& t, const AppendRun* runs, int32_t n_runs,
                       const int32_t* idx, const void* stage_k, const void* stage_v,
                       cudaStream_t st);

// ---- host tier migrations (tiers.cu). One entry per cluster of a batch.
struct TierMove {
  int32_t slot, n_pages;  // pages [0, n_pages) of the member list move
  int64_t stage0;         // first staging page of the cluster's contiguous copy
  int64_t host0;          // first host page of the cluster's extent
};
// Offload, step 1: npages of each slot -> out[i] (for extent sizing).
int launch_tier_count(const DevTables& t, const int32_t* slots, int32_t n, int32_t* out, cudaStream_t st);
// fetch-on-read copies listed by K4 (DecodeArgs::fr_jobs), launched between K4 and K6 as a
// programmatic dependent of K4 (K6 then depends on it); pdl as for K6.
int launch_fetch_read(const DevTables& t, const DecodeArgs& a, cudaStream_t st, bool pdl);
// Offload, step 2: pages [0, n_pages) of each slot (HBM or host) -> staging, seals them.
int launch_tier_gather(const DevTables& t, const TierMove* mv, int32_t n, int32_t max_pages_per_cluster,
                       uint8_t* stage, cudaStream_t st);
// Offload, step 3 (after the staging -> host copies completed): member pages [0, n_pages) become
// host pages host0 + i; their HBM pages return to the free stack.
int launch_tier_commit_offload(const DevTables& t, const TierMove* mv, int32_t n, cudaStream_t st);
// Fetch (after the host extent -> staging copies completed): every host page of the slot's member
// list gets a fresh HBM page filled from staging page stage0 + (id - max_pages - host0).
// scratch: [n][maxp] int32 (new page ids between the copy and the table pass).
int launch_tier_commit_fetch(const DevTables& t, const TierMove* mv, int32_t n, int32_t max_pages_per_cluster,
                             const uint8_t* stage, int32_t* scratch, cudaStream_t st);

// Gathers a cluster's members (then its buffer) into staging rows [n][d] K and V.
int launch_gather_cluster(const DevTables& t, int32_t slot, int32_t include_buffer,
                          void* stage_k, void* stage_v, int64_t row0, cudaStream_t st);
// Returns a slot's member and buffer pages to the free stack and clears its page lists.
int launch_free_slot_pages(const DevTables& t, int32_t slot, cudaStream_t st);

// Exact compute_representative / compute_variance (index.cpp:345-362) over staged rows
// idx[first .. first+n) for each run; writes rep64/rep32/rnorm/var of run.slot.
int launch_exact_stats(const DevTables& t, const AppendRun* runs, int32_t n_runs,
                       const int32_t* idx, const void* stage_k, cudaStream_t st);

// Flat top-k (oracle_flat_topk) of one query over an explicit candidate list.
// gscratch: n * 17 + 16 bytes of global scratch, used when the arrays exceed shared memory;
// slots == nullptr ranks the visual partitions 0..n-1 instead (visual_topk)
int launch_flat_topk(const DevTables& t, const float* q, const int32_t* slots,
                     const uint8_t* bufs, int32_t n, int32_t k, int32_t* out_idx,
                     uint8_t* gscratch, cudaStream_t st);

// Fresh-slot headers for a batch of clusters: counts, ids, Device residence, no buffer.
struct SlotHeader {
  int32_t slot, pad;
  int64_t cid, n;
};
int launch_slot_headers(const DevTables& t, const SlotHeader* h, int32_t n, cudaStream_t st);
// Exact statistics of host-built slots (split children, seeds, batch build): one packed record
// per slot, SlotInit followed by rep[d] and brep[d] doubles (slot_init_bytes(d) apart).
struct SlotInit {
  int32_t slot, nb;
  int64_t stat, nmem, cid;
  uint8_t resid, lazy, has_brep, pad[5];
  double rnorm, var, bnorm;
};
inline __host__ __device__ size_t slot_init_bytes(int d) { return sizeof(SlotInit) + 2 * static_cast<size_t>(d) * 8; }
int launch_init_slots(const DevTables& t, const void* recs, int32_t n, cudaStream_t st);
// kmeans_dev.cu: batch spherical k-means, one CTA per pool (rows [row0, row0 + n) of `rows`,
// final k = max(1, min(k_req, n)), the host's draws: first index + k - 1 uniforms at uni0).
struct KmJob {
  int64_t row0, scratch0, rep0;  // rep0: k x d doubles of Eq. 1 representatives (-1: not wanted)
  int32_t n, k, first, out0, uni0, var0;  // var0: k doubles of Eq. 2 variances
};
size_t kmeans_smem_bytes(int k, int d);
size_t kmeans_scratch_doubles(int n, int d);
int launch_kmeans(const float* rows, const KmJob* jobs, int n_jobs, const double* uniforms, double* scratch,
                  int32_t* assign, int32_t* meta, double* objective, double* reps, double* vars, int d, int k_max,
                  int max_iters, double tol, cudaStream_t st);

// Converts staged kv-dtype rows to fp32 (for host read-back).
// split.cu: split_two of rows[idx[i]] (i < n), one CTA; scratch n * (2d + 3) doubles; returns 0
// (nothing launched) for n < 2 or d > 256.
int launch_split_two(const float* rows, const int32_t* idx, int n, int d, int first, double uni, double* scratch,
                     int32_t* assign, int32_t* meta, double* objective, cudaStream_t st);
int launch_to_f32(const DevTables& t, const void* src, float* dst, int64_t n_elems,
                  cudaStream_t st);
// split_two for many independent point sets in one launch (one CTA per job).
struct SplitJob {
  const float* rows;
  const int32_t* idx;
  double* scratch;  // n * (2d + 3) doubles
  int32_t* assign;  // [n]
  int32_t* meta;    // [4]
  double* objective;
  double uni;
  int32_t n, first;
  // wave engine: group g's Eq. 1/2 statistics installed into slot[g] (>= 0) and its variance
  // written to var_out[g]; assign_in (non-null): no k-means, these labels
  int32_t slot[2];
  double* var_out;
  const int32_t* assign_in;
};
int launch_split_two_batch(const DevTables& t, const SplitJob* jobs, int n_jobs, int d, cudaStream_t st);
void split_prof_set(long long* p);  // KVC_SPLIT_PROF: per-job phase clocks [job][16] (nullptr: off)

// ---- ingest wave engine (waves.cu, context_waves.cpp)
// Staging of a slot's members (then its buffer when with_buf) and/or one frame row at row0.
struct GatherJob {
  int32_t slot, with_buf;  // slot -1: no cluster rows
  int64_t row0;
  int64_t frame_row;  // row of the frame buffer [L][tmax] appended after the cluster's rows (-1 none)
  int32_t* count_out;  // rows staged (checked by the host against its own count; may be null)
};
int launch_gather_batch(const DevTables& t, const GatherJob* jobs, int32_t n, const void* fk, const void* fv,
                        void* sk, void* sv, cudaStream_t st);
int launch_free_slots(const DevTables& t, const int32_t* slots, int32_t n, cudaStream_t st);
// Snapshot of a slot's ingest-mutable state: header, then rep64[d], brep64[d], rep32[d], brep32[d].
struct SlotSnap {
  int32_t slot, npages, nbpages, nbuf;
  int64_t stat, nmem, cid;
  int32_t fill_m, fill_b;
  uint8_t lazy, resid, pad[6];
  double var, rnorm, bnorm;
};
inline __host__ __device__ size_t slot_snap_bytes(int d) { return sizeof(SlotSnap) + static_cast<size_t>(d) * 24; }
int launch_snap_slots(const DevTables& t, const int32_t* slots, int32_t n, void* arena, cudaStream_t st);
int launch_restore_slots(const DevTables& t, const int32_t* idx, int32_t n, const void* arena, cudaStream_t st);
// Partition lists from packed records {pid * L + layer, pool offset, n, slots[n]} at rec_off[i].
int launch_pl_scatter(const DevTables& t, const int32_t* recs, const int32_t* rec_off, int32_t n, cudaStream_t st);
struct SlotCid {
  int64_t cid;
  int32_t slot, pad;
};
int launch_set_cids(const DevTables& t, const SlotCid* x, int32_t n, cudaStream_t st);
int launch_read_vars(const DevTables& t, const int32_t* slots, int32_t n, double* out, cudaStream_t st);

// launch_util.cu: per-device launch state. smem_optin raises a kernel's dynamic shared-memory
// attribute on the current device when `bytes` exceeds what was set there (false: the device's
// opt-in limit is smaller); occupancy is cached per (kernel, device, block, smem).
int current_device();
int device_sms();
int device_smem_optin();
bool smem_optin(const void* fn, size_t bytes);
int occupancy(const void* fn, int threads, size_t smem);
// K6 dynamic shared memory for a context's shape (kernels.cu); kvc::Context rejects shapes whose
// K6 ring does not fit the device.
size_t attend_smem_bytes(int d, int page_tokens, bool bf16);
// kvc_cfg.page_tokens == 0: 64 tokens per page, halved (down to 8) while K6's ring does not fit
int auto_page_tokens(int d, bool bf16);

#ifdef __CUDACC__
// Launch as a programmatic dependent of the previous kernel on the stream (its launch and block
// scheduling overlap the predecessor's tail; the kernel must execute griddepcontrol.wait before
// touching global memory). KVC_INGEST_PDL=0 launches normally.
inline bool ingest_pdl_enabled() {
  static const int on = [] {
    const char* e = std::getenv("KVC_INGEST_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return on != 0;
}
template <class K, class... A>
inline void launch_pdl(K kernel, dim3 g, dim3 b, size_t smem, cudaStream_t st, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ingest_pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}
#endif

}  // namespace kvc
