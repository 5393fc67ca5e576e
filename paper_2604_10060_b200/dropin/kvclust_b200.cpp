// kvclust_b200.cpp -- the C++ drop-in (include/kvclust_b200.hpp, kvclust_b200_engine.hpp) over
// the B200 engine's C-ABI (include/kvc.h). Every hot-path operation is a device call; the host
// code here only marshals the reference's value types (KVEntry, FrameInput, QueryBundle, ...) to
// and from flat buffers, maps status codes onto the reference's exception types
// (error.hpp:9-82) and keeps the reference's pure bookkeeping types (TransferLedger, RunOutput).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "kvc.h"
#include "kvclust_b200.hpp"
#include "kvclust_b200_engine.hpp"

namespace kvclust {

// =============================================================================== device handle
namespace b200 {

[[noreturn]] void raise(int rc) {
  const std::string msg = kvc_last_error() ? kvc_last_error() : "";
  auto num = [&](const char* prefix) -> long long {
    const auto p = msg.find(prefix);
    if (p == std::string::npos) return -1;
    try {
      return std::stoll(msg.substr(p + std::strlen(prefix)));
    } catch (...) {
      return -1;
    }
  };
  switch (rc) {
    case KVC_E_DEGENERATE: throw DegenerateVector(msg);
    case KVC_E_DIM: throw DimMismatch(0, 0);
    case KVC_E_EMPTY_INPUT: throw EmptyInput(msg);
    case KVC_E_EMPTY_CLUSTER: throw EmptyCluster(msg);
    case KVC_E_TOO_FEW: throw TooFewPoints(msg);
    case KVC_E_BAD_LAYER: throw BadLayer(static_cast<int>(num("layer out of range: ")));
    case KVC_E_UNKNOWN_CLUSTER: throw UnknownCluster(num("unknown cluster id: "));
    case KVC_E_EMPTY_INDEX: throw EmptyIndex(msg);
    case KVC_E_CONFIG: throw ConfigError(msg);
    case KVC_E_INVARIANT: throw InvariantViolation(msg);
    default: throw Error("kvc[" + std::to_string(rc) + "]: " + msg);
  }
}

inline int check(int rc) {
  if (rc < 0) raise(rc);
  return rc;
}

// Head widths: the device path stores rows of a multiple of 8 elements (16-byte vector moves for
// bf16 / f32 rows). A narrower width d (the reference's own unit tests use d = 4) is carried as
// d rounded up to 8 with zero padding: every quantity of the path is a sequential sum over the
// elements (dot, norm, sq_dist, the Eq. 3/4 running means, the k-means unit rows and centroid
// sums), and appending +0 terms to such a sum leaves it bit-identical, so rankings, statistics and
// splits are those of width d; the attention softmax keeps 1/sqrt(d) (kvc_set_head_dim). Rows are
// padded on the way in and cut back to d on the way out.
inline int padded_width(int d) { return d > 0 && d % 8 != 0 ? (d + 7) / 8 * 8 : d; }

struct Device {
  kvc_ctx* ctx = nullptr;
  kvc_cfg cfg{};
  int d = 0, dp = 0, L = 0;  // logical width, device width (padded)
  Device(const kvc_cfg& c, int d_, int L_) : cfg(c), d(d_), dp(padded_width(d_)), L(L_) {
    check(kvc_create(&cfg, dp, L, &ctx));
    if (dp != d) check(kvc_set_head_dim(ctx, d));
  }
  // `rows` rows of width d -> width dp (zero padding); a no-op view when dp == d
  template <class T>
  const T* pad(const T* src, std::size_t rows, std::vector<T>& buf) const {
    if (dp == d || !src) return src;
    buf.assign(rows * static_cast<std::size_t>(dp), T(0));
    for (std::size_t r = 0; r < rows; ++r)
      std::memcpy(&buf[r * dp], src + r * d, static_cast<std::size_t>(d) * sizeof(T));
    return buf.data();
  }
  // rows of width dp (device) -> width d in place of a buffer sized rows * dp
  template <class T>
  void cut(std::vector<T>& v, std::size_t rows) const {
    if (dp == d) return;
    for (std::size_t r = 0; r < rows; ++r)
      std::memmove(&v[r * d], &v[r * dp], static_cast<std::size_t>(d) * sizeof(T));
    v.resize(rows * static_cast<std::size_t>(d));
  }
  ~Device() {
    if (ctx) kvc_destroy(ctx);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
};

thread_local std::vector<float> g_attention;
const std::vector<float>& last_attention() { return g_attention; }

// defaults of the device data plane for contexts created by the drop-in: f32 payloads (the
// reference's Embedding is float), attended sets materialised (RetrievalResult / digests)
kvc_cfg base_cfg() {
  kvc_cfg c;
  kvc_cfg_default(&c);
  c.kv_dtype = KVC_DTYPE_F32;
  c.parity_mode = 1;
  return c;
}

void put_retrieval(kvc_cfg& c, const RetrievalConfig& r) {
  c.k_v = r.k_v;
  c.k_s = r.k_s;
  c.window_frames = r.window_frames;
  c.prefetch_k = r.prefetch_k;
  c.prefetch_enabled = r.prefetch_enabled ? 1 : 0;
  c.token_mode = r.mode == RetrievalMode::TokenBaseline ? 1 : 0;
  c.token_budget = r.token_budget;
  c.lookup_cost_per_candidate_us = r.lookup_cost_per_candidate_us;
  c.compute_cost_per_token_us = r.compute_cost_per_token_us;
}

void put_cost(kvc_cfg& c, const CostModel& m) {
  c.alpha_us = m.alpha_us;
  c.beta_us_per_byte = m.beta_us_per_byte;
  c.bytes_per_entry = m.bytes_per_entry;
  c.device_capacity_entries = m.device_capacity_entries;
}

void put_maintainer(kvc_cfg& c, const MaintainerConfig& m) {
  c.tau_min = m.threshold.tau_min;
  c.tau_max = m.threshold.tau_max;
  c.n0 = m.threshold.n0;
  c.defer_host_splits = m.defer_host_splits ? 1 : 0;
  c.max_split_depth = m.max_split_depth;
  c.visual_floor = m.visual_floor;
}

void put_build(kvc_cfg& c, const BuildConfig& b) {
  c.target_visual_cluster_size = b.target_visual_cluster_size;
  c.target_semantic_cluster_size = b.target_semantic_cluster_size;
  c.kmeans_max_iters = b.kmeans_max_iters;
  c.kmeans_tol = b.kmeans_tol;
}

// FrameInput -> [L][T][d] keys / values; token ids must be the positions 0..T-1 (the engine keys
// a frame's entries by position, as gen_stream and every reference caller produce them)
void pack_frame(const FrameInput& f, int d, int L, std::vector<float>& k, std::vector<float>& v, int& T, int dp = 0) {
  if (dp <= 0) dp = d;
  if (static_cast<int>(f.visual.size()) != d) throw ConfigError("frame width does not match the engine");
  if (static_cast<int>(f.layers.size()) != L) throw ConfigError("frame layer count does not match the engine");
  T = static_cast<int>(f.layers[0].size());
  k.assign(static_cast<std::size_t>(L) * T * dp, 0.f);
  v.assign(k.size(), 0.f);
  for (int l = 0; l < L; ++l) {
    const auto& layer = f.layers[static_cast<std::size_t>(l)];
    if (static_cast<int>(layer.size()) != T) throw ConfigError("layers of a frame must hold the same token count");
    for (int t = 0; t < T; ++t) {
      const KVEntry& e = layer[static_cast<std::size_t>(t)];
      if (e.token_id != t) throw ConfigError("frame entries must carry token ids 0..T-1 in order");
      if (static_cast<int>(e.key.size()) != d || static_cast<int>(e.value.size()) != d)
        throw DimMismatch(e.key.size(), static_cast<std::size_t>(d));
      std::memcpy(&k[(static_cast<std::size_t>(l) * T + t) * dp], e.key.data(), static_cast<std::size_t>(d) * 4);
      std::memcpy(&v[(static_cast<std::size_t>(l) * T + t) * dp], e.value.data(), static_cast<std::size_t>(d) * 4);
    }
  }
}

std::vector<float> pack_query(const QueryBundle& b, int d, int L, int dp = 0) {
  if (dp <= 0) dp = d;
  if (static_cast<int>(b.q.size()) != L) throw ConfigError("query bundle layer count does not match the stored layers");
  std::vector<float> q(static_cast<std::size_t>(L) * dp, 0.f);
  for (int l = 0; l < L; ++l) {
    if (static_cast<int>(b.q[static_cast<std::size_t>(l)].size()) != d)
      throw DimMismatch(b.q[static_cast<std::size_t>(l)].size(), static_cast<std::size_t>(d));
    std::memcpy(&q[static_cast<std::size_t>(l) * dp], b.q[static_cast<std::size_t>(l)].data(), static_cast<std::size_t>(d) * 4);
  }
  return q;
}

TransferCause cause_of(std::int64_t c) { return static_cast<TransferCause>(c); }

// the device's TransferLedger op log (store.cpp:21-27) from op `from` on
void ledger_ops(const Device& dv, std::size_t from, TransferLedger& out) {
  const int n = check(kvc_ledger_log_size(dv.ctx));
  for (int i = static_cast<int>(from); i < n; ++i) {
    std::int64_t x[4];
    check(kvc_ledger_op(dv.ctx, i, x));
    TransferOp op;
    op.cause = cause_of(x[0]);
    op.to_device = x[1] != 0;
    op.cluster_id = x[2];
    op.n_ops = 1;
    op.bytes = x[3];
    op.cost_us = 1.0 * dv.cfg.alpha_us + static_cast<double>(x[3]) * dv.cfg.beta_us_per_byte;
    out.record(op);
  }
}

struct Totals {
  std::int64_t ops = 0, bytes = 0;
  double cost = 0.0;
};
Totals ledger_totals(const Device& dv) {
  std::int64_t ops[5], by[5];
  double co[5];
  const std::int64_t rc = kvc_ledger(dv.ctx, ops, by, co);
  if (rc < 0) raise(static_cast<int>(rc));
  Totals t;
  for (int i = 0; i < 5; ++i) {
    t.ops += ops[i];
    t.bytes += by[i];
    t.cost += co[i];
  }
  return t;
}

// RetrievalResult of the last device decode step (retrieval.hpp:49-71)
RetrievalResult read_result(const Device& dv, std::int64_t qid) {
  RetrievalResult r;
  r.query_id = qid;
  r.layers.resize(static_cast<std::size_t>(dv.L));
  std::vector<std::int64_t> ids(4096), fr(1 << 16);
  std::vector<std::int32_t> buf(4096), tk(1 << 16);
  for (int l = 0; l < dv.L; ++l) {
    LayerResult& lr = r.layers[static_cast<std::size_t>(l)];
    int n = check(kvc_last_ranked(dv.ctx, l, ids.data(), buf.data(), static_cast<int>(ids.size())));
    for (int i = 0; i < std::min<int>(n, static_cast<int>(ids.size())); ++i) lr.ranked.push_back({ids[static_cast<std::size_t>(i)], buf[static_cast<std::size_t>(i)] != 0});
    n = check(kvc_last_selected(dv.ctx, l, ids.data(), static_cast<int>(ids.size())));
    lr.selected.assign(ids.begin(), ids.begin() + std::min<int>(n, static_cast<int>(ids.size())));
    n = check(kvc_last_predicted(dv.ctx, l, ids.data(), static_cast<int>(ids.size())));
    lr.predicted.assign(ids.begin(), ids.begin() + std::min<int>(n, static_cast<int>(ids.size())));
    n = check(kvc_last_attended(dv.ctx, l, nullptr, nullptr, 0));
    if (n > static_cast<int>(fr.size())) {
      fr.resize(static_cast<std::size_t>(n));
      tk.resize(static_cast<std::size_t>(n));
    }
    n = check(kvc_last_attended(dv.ctx, l, fr.data(), tk.data(), static_cast<int>(fr.size())));
    for (int i = 0; i < n; ++i) lr.attended_tokens.push_back({fr[static_cast<std::size_t>(i)], tk[static_cast<std::size_t>(i)]});
    double lat[5];
    std::int64_t ints[5];
    check(kvc_last_layer_meta(dv.ctx, l, lat, ints));
    lr.latency = {lat[0], lat[1], lat[2], lat[3], lat[4]};
    lr.verified_clusters = ints[0];
    lr.prefetch_hits = ints[1];
    lr.rep_count = ints[2];
  }
  double dd[2];
  check(kvc_last_query_meta(dv.ctx, dd));
  r.ttft_us = dd[0];
  r.recall = dd[1];
  for (int which = 0; which < 2; ++which) {
    const int n = check(kvc_last_frames(dv.ctx, which, nullptr, 0));
    std::vector<std::int64_t> f(static_cast<std::size_t>(n));
    check(kvc_last_frames(dv.ctx, which, f.data(), n));
    (which == 0 ? r.fetched_frames : r.context_frames) = std::move(f);
  }
  return r;
}

}  // namespace b200

using b200::check;

// =============================================================================== free functions

const char* to_string(TransferCause cause) {
  switch (cause) {
    case TransferCause::Retrieval: return "retrieval";
    case TransferCause::Maintenance: return "maintenance";
    case TransferCause::Prefetch: return "prefetch";
    case TransferCause::Completion: return "completion";
    case TransferCause::Offload: return "offload";
  }
  return "unknown";
}

double tau(std::int64_t n, const ThresholdConfig& cfg) { return kvc_host_tau(n, cfg.tau_min, cfg.tau_max, cfg.n0); }

// Eq. 3/4 as one uncommitted step (maintainer.cpp:16-25), the evaluation order the device chains use
StatUpdate updated_stats(const DVec& rep, double variance, std::int64_t n, const Embedding& key) {
  if (rep.size() != key.size()) throw DimMismatch(rep.size(), key.size());
  StatUpdate out;
  out.rep.resize(rep.size());
  const double dn = static_cast<double>(n);
  for (std::size_t i = 0; i < rep.size(); ++i) out.rep[i] = (dn * rep[i] + static_cast<double>(key[i])) / (dn + 1.0);
  double acc = 0.0;
  for (std::size_t i = 0; i < rep.size(); ++i) {
    const double df = static_cast<double>(key[i]) - out.rep[i];
    acc += df * df;
  }
  out.variance = (dn * variance + acc) / (dn + 1.0);
  return out;
}

// Eq. 1 / Eq. 2 (index.cpp:345-362)
DVec compute_representative(const std::vector<KVEntry>& members) {
  if (members.empty()) throw EmptyCluster("representative of an empty member set");
  DVec rep(members.front().key.size(), 0.0);
  for (const KVEntry& e : members) {
    if (e.key.size() != rep.size()) throw DimMismatch(e.key.size(), rep.size());
    for (std::size_t i = 0; i < rep.size(); ++i) rep[i] += static_cast<double>(e.key[i]);
  }
  for (double& x : rep) x /= static_cast<double>(members.size());
  return rep;
}

double compute_variance(const std::vector<KVEntry>& members, const DVec& rep) {
  if (members.empty()) throw EmptyCluster("variance of an empty member set");
  double s = 0.0;
  for (const KVEntry& e : members) {
    double acc = 0.0;
    for (std::size_t i = 0; i < rep.size(); ++i) {
      const double df = static_cast<double>(e.key[i]) - rep[i];
      acc += df * df;
    }
    s += acc;
  }
  return s / static_cast<double>(members.size());
}

void RetrievalConfig::validate() const {  // retrieval.cpp:10-16
  if (k_v <= 0 || k_s <= 0 || window_frames <= 0 || prefetch_k <= 0)
    throw ConfigError("retrieval budgets must be positive");
  if (token_budget < 1) throw ConfigError("token budget must be at least 1");
  if (lookup_cost_per_candidate_us < 0.0 || compute_cost_per_token_us < 0.0)
    throw ConfigError("cost constants must be non-negative");
}

// =============================================================================== TransferLedger

void TransferLedger::record(const TransferOp& op) {
  log_.push_back(op);
  CauseTotals& t = totals_[to_string(op.cause)];
  t.n_ops += op.n_ops;
  t.bytes += op.bytes;
  t.cost_us += op.cost_us;
}

CauseTotals TransferLedger::totals() const {
  CauseTotals s;
  for (const auto& [k, t] : totals_) {
    s.n_ops += t.n_ops;
    s.bytes += t.bytes;
    s.cost_us += t.cost_us;
  }
  return s;
}

CauseTotals TransferLedger::cause(TransferCause c) const {
  auto it = totals_.find(to_string(c));
  return it == totals_.end() ? CauseTotals{} : it->second;
}

void TransferLedger::audit() const {
  std::map<std::string, CauseTotals> re;
  for (const TransferOp& op : log_) {
    CauseTotals& t = re[to_string(op.cause)];
    t.n_ops += op.n_ops;
    t.bytes += op.bytes;
    t.cost_us += op.cost_us;
  }
  for (const auto& [k, t] : re) {
    auto it = totals_.find(k);
    if (it == totals_.end() || it->second.n_ops != t.n_ops || it->second.bytes != t.bytes ||
        std::abs(it->second.cost_us - t.cost_us) > 1e-6 * std::max(1.0, std::abs(t.cost_us)))
      throw InvariantViolation("ledger totals drifted from the op log");
  }
  if (re.size() != totals_.size()) throw InvariantViolation("ledger totals drifted from the op log");
}

void TransferLedger::clear() {
  log_.clear();
  totals_.clear();
}

// =============================================================================== HierIndex

namespace {
ClusterRecord* pending_cluster(std::vector<ClusterRecord>& cs, std::int64_t id) {
  for (ClusterRecord& r : cs)
    if (r.cluster_id == id) return &r;
  throw UnknownCluster(id);
}
}  // namespace

struct HierIndex::View {
  std::vector<VisualPartition> parts;
  std::map<std::int64_t, ClusterRecord> clusters;
  std::vector<std::vector<CandidateRef>> rep_set;
  std::vector<std::vector<std::int64_t>> timeline;
  std::set<std::int64_t> registered;
};

HierIndex::HierIndex() = default;
HierIndex::HierIndex(std::int32_t dim, std::int32_t layers) : dim_(dim), layers_(layers) {}
HierIndex::HierIndex(HierIndex&&) noexcept = default;
HierIndex& HierIndex::operator=(HierIndex&&) noexcept = default;
HierIndex::~HierIndex() = default;

namespace {
// configuration a component-level index context is created with: the store's CostModel and the
// maintainer's config are applied by kvc_reconfigure when those objects attach
kvc_cfg component_cfg() {
  kvc_cfg c = b200::base_cfg();
  c.build_batch_frames = 1;
  c.offload_horizon_frames = 1 << 30;  // no engine cadence: residence changes only through the API
  c.host_pool_bytes = 0;               // residence stays logical (no physical host tier)
  return c;
}
}  // namespace

b200::Device& HierIndex::device() const {
  if (!dev_) {
    if (dim_ <= 0 || layers_ <= 0) throw ConfigError("stream dimensions must be positive");
    dev_ = std::make_shared<b200::Device>(component_cfg(), dim_, layers_);
  }
  install_pending();
  return *dev_;
}

void HierIndex::install_pending() const {
  if (pending_parts_.empty() && pending_clusters_.empty()) return;
  auto* self = const_cast<HierIndex*>(this);
  const int dp = dev_->dp;
  for (const VisualPartition& p : pending_parts_) {  // verbatim: frames, fp64 visual_rep, count
    std::int64_t pid = -1;
    std::vector<double> pv;
    check(kvc_add_partition_ex(dev_->ctx, p.frame_ids.data(), static_cast<int>(p.frame_ids.size()),
                               dev_->pad(p.visual_rep.data(), 1, pv), p.visual_stat_count, &pid));
  }
  auto rows = [&](const std::vector<KVEntry>& es, std::vector<float>& k, std::vector<float>& v,
                  std::vector<std::int64_t>& fr, std::vector<std::int32_t>& tk) {
    const std::size_t n = es.size();
    k.assign(n * static_cast<std::size_t>(dp), 0.f);
    v.assign(k.size(), 0.f);
    fr.resize(n);
    tk.resize(n);
    for (std::size_t j = 0; j < n; ++j) {
      if (static_cast<int>(es[j].key.size()) != dim_ || static_cast<int>(es[j].value.size()) != dim_)
        throw DimMismatch(es[j].key.size(), static_cast<std::size_t>(dim_));
      std::memcpy(&k[j * dp], es[j].key.data(), static_cast<std::size_t>(dim_) * 4);
      std::memcpy(&v[j * dp], es[j].value.data(), static_cast<std::size_t>(dim_) * 4);
      fr[j] = es[j].frame_id;
      tk[j] = es[j].token_id;
    }
  };
  for (std::size_t i = 0; i < pending_clusters_.size(); ++i) {  // verbatim records, ids kept
    const ClusterRecord& rec = pending_clusters_[i];
    std::vector<float> mk, mv, bk, bv;
    std::vector<std::int64_t> mf, bf;
    std::vector<std::int32_t> mt, bt;
    rows(rec.members, mk, mv, mf, mt);
    rows(rec.buffer, bk, bv, bf, bt);
    if (static_cast<int>(rec.rep.size()) != dim_) throw DimMismatch(rec.rep.size(), static_cast<std::size_t>(dim_));
    kvc_cluster_record r{};
    r.layer = rec.layer_id;
    r.partition = rec.visual_parent;
    r.n_members = static_cast<int>(rec.members.size());
    r.member_keys = mk.data();
    r.member_values = mv.data();
    r.member_frames = mf.data();
    r.member_tokens = mt.data();
    r.n_buffer = static_cast<int>(rec.buffer.size());
    r.buffer_keys = bk.data();
    r.buffer_values = bv.data();
    r.buffer_frames = bf.data();
    r.buffer_tokens = bt.data();
    std::vector<double> prep, pbrep;
    r.rep = dev_->pad(rec.rep.data(), 1, prep);
    r.variance = rec.variance;
    r.stat_count = rec.stat_count;
    r.buffer_rep = rec.buffer_rep.size() == static_cast<std::size_t>(dim_) ? dev_->pad(rec.buffer_rep.data(), 1, pbrep) : nullptr;
    r.lazy_split = (rec.lazy_split || pending_registered_.count(rec.cluster_id)) ? 1 : 0;
    r.residence = rec.residence == Residence::Host ? 1 : 0;
    r.adopt = pending_adopted_[i];
    r.device_tail = rec.device_tail;
    r.want_id = rec.cluster_id;
    std::int64_t id = -1;
    check(kvc_add_cluster_ex(dev_->ctx, &r, &id));
  }
  self->pending_parts_.clear();
  self->pending_first_visual_.clear();
  self->pending_appends_.clear();
  self->pending_clusters_.clear();
  self->pending_adopted_.clear();
  self->pending_registered_.clear();
  mark_device_changed();
}

void HierIndex::mark_device_changed() const { view_.reset(); }

const HierIndex::View& HierIndex::view() const {
  if (view_) return *view_;
  auto v = std::make_unique<View>();
  v->rep_set.resize(static_cast<std::size_t>(std::max(layers_, 0)));
  v->timeline.resize(static_cast<std::size_t>(std::max(layers_, 0)));
  if (!dev_) {  // host-assembled, not yet installed
    v->parts = pending_parts_;
    for (const ClusterRecord& r : pending_clusters_) v->clusters.emplace(r.cluster_id, r);
    v->registered = pending_registered_;
  } else {
    install_pending();
    kvc_ctx* c = dev_->ctx;
    const int P = check(kvc_n_partitions(c));
    std::vector<std::int64_t> buf(1 << 16);
    for (int p = 0; p < P; ++p) {
      VisualPartition vp;
      vp.partition_id = p;
      DVec rep(static_cast<std::size_t>(dev_->dp));
      int n = check(kvc_partition(c, p, rep.data(), nullptr, 0));
      vp.frame_ids.resize(static_cast<std::size_t>(n));
      check(kvc_partition(c, p, rep.data(), vp.frame_ids.data(), n));
      dev_->cut(rep, 1);
      vp.visual_rep = rep;
      vp.visual_stat_count = n;
      for (int l = 0; l < layers_; ++l) {
        n = check(kvc_partition_layer(c, p, l, nullptr, 0));
        if (n == 0) continue;
        std::vector<std::int64_t> ids(static_cast<std::size_t>(n));
        check(kvc_partition_layer(c, p, l, ids.data(), n));
        vp.per_layer_clusters[l] = ids;
      }
      v->parts.push_back(std::move(vp));
    }
    const int nc = check(kvc_n_clusters(c));
    std::vector<std::int64_t> ids(static_cast<std::size_t>(nc));
    check(kvc_cluster_ids(c, ids.data(), nc));
    for (std::int64_t id : ids) {
      ClusterRecord r;
      std::int64_t info[10];
      DVec rep(static_cast<std::size_t>(dev_->dp)), brep(static_cast<std::size_t>(dev_->dp), 0.0);
      double var = 0.0;
      check(kvc_cluster(c, id, info, &var, rep.data(), brep.data()));
      dev_->cut(rep, 1);
      dev_->cut(brep, 1);
      r.cluster_id = id;
      r.layer_id = static_cast<std::int32_t>(info[0]);
      r.visual_parent = info[1];
      r.stat_count = info[4];
      r.lazy_split = info[5] != 0;
      r.residence = info[6] ? Residence::Host : Residence::Device;
      r.device_tail = info[7];
      r.first_frame_id = info[8];
      r.last_touch_frame = info[9];
      r.rep = rep;
      r.variance = var;
      for (int which = 0; which < 2; ++which) {
        const int n = static_cast<int>(info[2 + which]);
        if (n == 0) continue;
        std::vector<std::int64_t> fr(static_cast<std::size_t>(n));
        std::vector<std::int32_t> tk(static_cast<std::size_t>(n));
        std::vector<float> k(static_cast<std::size_t>(n) * dev_->dp), val(k.size());
        check(kvc_cluster_entries(c, id, which, fr.data(), tk.data(), n));
        check(kvc_cluster_payload(c, id, which, k.data(), val.data(), n));
        dev_->cut(k, static_cast<std::size_t>(n));
        dev_->cut(val, static_cast<std::size_t>(n));
        auto& dst = which == 0 ? r.members : r.buffer;
        for (int j = 0; j < n; ++j) {
          KVEntry e;
          e.key.assign(k.begin() + static_cast<std::ptrdiff_t>(j) * dim_, k.begin() + static_cast<std::ptrdiff_t>(j + 1) * dim_);
          e.value.assign(val.begin() + static_cast<std::ptrdiff_t>(j) * dim_, val.begin() + static_cast<std::ptrdiff_t>(j + 1) * dim_);
          e.frame_id = fr[static_cast<std::size_t>(j)];
          e.layer_id = r.layer_id;
          e.token_id = tk[static_cast<std::size_t>(j)];
          dst.push_back(std::move(e));
        }
      }
      if (!r.buffer.empty()) r.buffer_rep = brep;
      v->clusters.emplace(id, std::move(r));
    }
  }
  // rep_set: live clusters in id order, then the registered buffers (index.cpp:97-168)
  for (const auto& [id, r] : v->clusters) v->rep_set[static_cast<std::size_t>(r.layer_id)].push_back({id, false});
  for (const auto& [id, r] : v->clusters)
    if (dev_ ? r.lazy_split : v->registered.count(id) != 0) {
      v->rep_set[static_cast<std::size_t>(r.layer_id)].push_back({id, true});
      v->registered.insert(id);
    }
  // timeline: (first_frame_id, cluster_id) order (index.cpp:81-95)
  for (int l = 0; l < layers_; ++l) {
    std::vector<std::pair<std::int64_t, std::int64_t>> t;
    for (const auto& [id, r] : v->clusters)
      if (r.layer_id == l) t.push_back({r.first_frame_id, id});
    std::sort(t.begin(), t.end());
    for (const auto& x : t) v->timeline[static_cast<std::size_t>(l)].push_back(x.second);
  }
  view_ = std::move(v);
  return *view_;
}

const std::vector<VisualPartition>& HierIndex::partitions() const { return view().parts; }

VisualPartition& HierIndex::partition(std::int64_t id) {
  if (!dev_) {
    if (id < 0 || id >= static_cast<std::int64_t>(pending_parts_.size())) throw UnknownCluster(id);
    mark_device_changed();
    return pending_parts_[static_cast<std::size_t>(id)];
  }
  auto& ps = const_cast<View&>(view()).parts;
  if (id < 0 || id >= static_cast<std::int64_t>(ps.size())) throw UnknownCluster(id);
  return ps[static_cast<std::size_t>(id)];
}
const VisualPartition& HierIndex::partition(std::int64_t id) const {
  return const_cast<HierIndex*>(this)->partition(id);
}

const std::map<std::int64_t, ClusterRecord>& HierIndex::clusters() const { return view().clusters; }

ClusterRecord& HierIndex::cluster(std::int64_t id) {
  if (!dev_) {  // host-assembled: the caller edits the pending record itself
    mark_device_changed();
    return *pending_cluster(pending_clusters_, id);
  }
  auto& cs = const_cast<View&>(view()).clusters;
  auto it = cs.find(id);
  if (it == cs.end()) throw UnknownCluster(id);
  return it->second;
}
const ClusterRecord& HierIndex::cluster(std::int64_t id) const { return const_cast<HierIndex*>(this)->cluster(id); }

const std::vector<CandidateRef>& HierIndex::rep_set(std::int32_t layer) const {
  if (layer < 0 || layer >= layers_) throw BadLayer(layer);
  return view().rep_set[static_cast<std::size_t>(layer)];
}

const std::vector<std::int64_t>& HierIndex::rep_timeline(std::int32_t layer) const {
  if (layer < 0 || layer >= layers_) throw BadLayer(layer);
  return view().timeline[static_cast<std::size_t>(layer)];
}

const DVec& HierIndex::candidate_rep(const CandidateRef& ref) const {
  const ClusterRecord& rec = cluster(ref.cluster_id);
  return ref.is_buffer ? rec.buffer_rep : rec.rep;
}

std::int64_t HierIndex::add_partition(std::int64_t first_frame_id, const Embedding& visual) {
  if (static_cast<std::int32_t>(visual.size()) != dim_) throw DimMismatch(visual.size(), static_cast<std::size_t>(dim_));
  if (dev_) {
    std::int64_t pid = -1;
    std::vector<float> pv;
    check(kvc_add_partition(dev_->ctx, first_frame_id, dev_->pad(visual.data(), 1, pv), &pid));
    mark_device_changed();
    return pid;
  }
  VisualPartition p;
  p.partition_id = static_cast<std::int64_t>(pending_parts_.size());
  p.frame_ids.push_back(first_frame_id);
  p.visual_rep.assign(visual.begin(), visual.end());
  p.visual_stat_count = 1;
  pending_parts_.push_back(std::move(p));
  pending_first_visual_.push_back(visual);
  pending_appends_.emplace_back();
  mark_device_changed();
  return pending_parts_.back().partition_id;
}

void HierIndex::append_frame(std::int64_t partition_id, std::int64_t frame_id, const Embedding& visual) {
  if (dev_) {
    if (static_cast<std::int32_t>(visual.size()) != dim_) throw DimMismatch(visual.size(), static_cast<std::size_t>(dim_));
    std::vector<float> pv;
    check(kvc_append_frame(dev_->ctx, partition_id, frame_id, dev_->pad(visual.data(), 1, pv)));
    mark_device_changed();
    return;
  }
  if (partition_id < 0 || partition_id >= static_cast<std::int64_t>(pending_parts_.size())) throw UnknownCluster(partition_id);
  VisualPartition& p = pending_parts_[static_cast<std::size_t>(partition_id)];
  pending_appends_[static_cast<std::size_t>(partition_id)].push_back({frame_id, visual});
  p.frame_ids.push_back(frame_id);
  const double n = static_cast<double>(p.visual_stat_count);
  for (std::size_t i = 0; i < p.visual_rep.size(); ++i) p.visual_rep[i] = (n * p.visual_rep[i] + visual[i]) / (n + 1.0);
  p.visual_stat_count += 1;
  mark_device_changed();
}

std::int64_t HierIndex::add_cluster(ClusterRecord&& rec) {
  if (rec.members.empty()) throw EmptyCluster("cluster with no members");
  if (rec.layer_id < 0 || rec.layer_id >= layers_) throw BadLayer(rec.layer_id);
  if (!rec.buffer.empty() || rec.lazy_split) throw ConfigError("add_cluster: pending-split buffers are created by the maintainer");
  if (dev_) {
    const int n = static_cast<int>(rec.members.size());
    std::vector<float> k(static_cast<std::size_t>(n) * dim_), v(k.size());
    std::vector<std::int64_t> fr(static_cast<std::size_t>(n));
    std::vector<std::int32_t> tk(static_cast<std::size_t>(n));
    for (int j = 0; j < n; ++j) {
      const KVEntry& e = rec.members[static_cast<std::size_t>(j)];
      if (static_cast<int>(e.key.size()) != dim_) throw DimMismatch(e.key.size(), static_cast<std::size_t>(dim_));
      std::memcpy(&k[static_cast<std::size_t>(j) * dim_], e.key.data(), static_cast<std::size_t>(dim_) * 4);
      std::memcpy(&v[static_cast<std::size_t>(j) * dim_], e.value.data(), static_cast<std::size_t>(dim_) * 4);
      fr[static_cast<std::size_t>(j)] = e.frame_id;
      tk[static_cast<std::size_t>(j)] = e.token_id;
    }
    std::int64_t id = -1;
    std::vector<float> pk, pv;
    check(kvc_add_cluster(dev_->ctx, rec.layer_id, rec.visual_parent, n, dev_->pad(k.data(), static_cast<std::size_t>(n), pk),
                          dev_->pad(v.data(), static_cast<std::size_t>(n), pv), fr.data(), tk.data(),
                          rec.residence == Residence::Host ? 1 : 0, 0, &id));
    mark_device_changed();
    return id;
  }
  if (rec.visual_parent < 0 || rec.visual_parent >= static_cast<std::int64_t>(pending_parts_.size()))
    throw UnknownCluster(rec.visual_parent);
  for (const KVEntry& e : rec.members)
    if (static_cast<int>(e.key.size()) != dim_) throw DimMismatch(e.key.size(), static_cast<std::size_t>(dim_));
  rec.cluster_id = static_cast<std::int64_t>(pending_clusters_.size());
  rec.first_frame_id = rec.members.front().frame_id;
  rec.last_touch_frame = rec.members.front().frame_id;
  for (const KVEntry& e : rec.members) {
    rec.first_frame_id = std::min(rec.first_frame_id, e.frame_id);
    rec.last_touch_frame = std::max(rec.last_touch_frame, e.frame_id);
  }
  const std::int64_t id = rec.cluster_id;
  pending_parts_[static_cast<std::size_t>(rec.visual_parent)].per_layer_clusters[rec.layer_id].push_back(id);
  pending_clusters_.push_back(std::move(rec));
  pending_adopted_.push_back(0);
  mark_device_changed();
  return id;
}

namespace {
[[noreturn]] void maintainer_only(const char* what) {
  throw ConfigError(std::string(what) + ": the device index is mutated by the maintainer (on_insert / materialize)");
}
}  // namespace

// Low-level mutators (index.cpp:122-190). On a host-assembled index (before any device operation)
// they edit the pending state; once the index lives on the device, the maintainer owns it.
void HierIndex::remove_cluster(std::int64_t id) {
  if (dev_) maintainer_only("remove_cluster");
  ClusterRecord* r = pending_cluster(pending_clusters_, id);
  auto& sib = pending_parts_[static_cast<std::size_t>(r->visual_parent)].per_layer_clusters[r->layer_id];
  sib.erase(std::remove(sib.begin(), sib.end(), id), sib.end());
  const std::size_t i = static_cast<std::size_t>(r - pending_clusters_.data());
  pending_clusters_.erase(pending_clusters_.begin() + static_cast<std::ptrdiff_t>(i));
  pending_adopted_.erase(pending_adopted_.begin() + static_cast<std::ptrdiff_t>(i));
  pending_registered_.erase(id);
  mark_device_changed();
}
void HierIndex::register_buffer(std::int64_t cluster_id) {
  if (dev_) maintainer_only("register_buffer");
  pending_cluster(pending_clusters_, cluster_id);
  pending_registered_.insert(cluster_id);
  mark_device_changed();
}
void HierIndex::deregister_buffer(std::int64_t cluster_id) {
  if (dev_) maintainer_only("deregister_buffer");
  pending_registered_.erase(cluster_id);
  mark_device_changed();
}
bool HierIndex::buffer_registered(std::int64_t cluster_id) const {
  if (!dev_) return pending_registered_.count(cluster_id) != 0;
  return view().registered.count(cluster_id) != 0;
}
void HierIndex::add_member(std::int64_t cluster_id, KVEntry entry) {
  if (dev_) maintainer_only("add_member");
  ClusterRecord* r = pending_cluster(pending_clusters_, cluster_id);
  r->last_touch_frame = std::max(r->last_touch_frame, entry.frame_id);
  r->members.push_back(std::move(entry));
  mark_device_changed();
}
void HierIndex::add_to_buffer(std::int64_t cluster_id, KVEntry entry) {
  if (dev_) maintainer_only("add_to_buffer");
  ClusterRecord* r = pending_cluster(pending_clusters_, cluster_id);
  // running mean of the buffered keys (index.cpp:177-190)
  if (r->buffer_rep.empty()) r->buffer_rep.assign(entry.key.size(), 0.0);
  const double n = static_cast<double>(r->buffer.size());
  for (std::size_t i = 0; i < r->buffer_rep.size(); ++i)
    r->buffer_rep[i] = (n * r->buffer_rep[i] + static_cast<double>(entry.key[i])) / (n + 1.0);
  r->buffer.push_back(std::move(entry));
  mark_device_changed();
}

// index.v1 JSON (the reference's schema, index.cpp:452-592)
namespace {
using json = nlohmann::json;
json emb_json(const Embedding& v) {
  json a = json::array();
  for (float x : v) a.push_back(static_cast<double>(x));
  return a;
}
Embedding emb_from(const json& a) {
  Embedding v;
  for (const auto& x : a) v.push_back(static_cast<float>(x.get<double>()));
  return v;
}
json entry_json(const KVEntry& e) {
  return json{{"key", emb_json(e.key)}, {"value", emb_json(e.value)}, {"frame", e.frame_id},
              {"layer", e.layer_id}, {"token", e.token_id}};
}
KVEntry entry_from(const json& j) {
  KVEntry e;
  e.key = emb_from(j.at("key"));
  e.value = emb_from(j.at("value"));
  e.frame_id = j.at("frame").get<std::int64_t>();
  e.layer_id = j.at("layer").get<std::int32_t>();
  e.token_id = j.at("token").get<std::int32_t>();
  return e;
}
}  // namespace

std::string HierIndex::to_json_string() const {
  json root;
  root["format"] = "kvclust.index.v1";
  root["dim"] = dim_;
  root["layers"] = layers_;
  std::int64_t next = 0;
  for (const auto& [id, r] : clusters()) next = std::max(next, id + 1);
  root["next_cluster_id"] = next;
  json parts = json::array();
  for (const VisualPartition& p : partitions()) {
    json jp;
    jp["id"] = p.partition_id;
    jp["frames"] = p.frame_ids;
    jp["visual_rep"] = p.visual_rep;
    jp["visual_stat_count"] = p.visual_stat_count;
    json lm = json::object();
    for (const auto& [layer, ids] : p.per_layer_clusters) lm[std::to_string(layer)] = ids;
    jp["clusters"] = std::move(lm);
    parts.push_back(std::move(jp));
  }
  root["partitions"] = std::move(parts);
  json cs = json::array();
  for (const auto& [id, r] : clusters()) {
    json jc;
    jc["id"] = id;
    jc["layer"] = r.layer_id;
    jc["parent"] = r.visual_parent;
    jc["rep"] = r.rep;
    jc["variance"] = r.variance;
    jc["stat_count"] = r.stat_count;
    jc["lazy_split"] = r.lazy_split;
    jc["residence"] = r.residence == Residence::Device ? "device" : "host";
    jc["device_tail"] = r.device_tail;
    jc["first_frame"] = r.first_frame_id;
    jc["last_touch"] = r.last_touch_frame;
    json m = json::array(), b = json::array();
    for (const KVEntry& e : r.members) m.push_back(entry_json(e));
    for (const KVEntry& e : r.buffer) b.push_back(entry_json(e));
    jc["members"] = std::move(m);
    jc["buffer"] = std::move(b);
    jc["buffer_rep"] = r.buffer_rep;
    cs.push_back(std::move(jc));
  }
  root["clusters"] = std::move(cs);
  return root.dump(2);
}

HierIndex HierIndex::from_json_string(const std::string& text) {
  json root;
  try {
    root = json::parse(text);
  } catch (const json::parse_error& e) {
    throw ParseError(0, std::string("bad index json: ") + e.what());
  }
  if (root.value("format", "") != "kvclust.index.v1") throw ParseError(0, "unrecognized index format");
  HierIndex idx(root.at("dim").get<std::int32_t>(), root.at("layers").get<std::int32_t>());
  for (const json& jp : root.at("partitions")) {
    VisualPartition p;
    p.partition_id = jp.at("id").get<std::int64_t>();
    p.frame_ids = jp.at("frames").get<std::vector<std::int64_t>>();
    p.visual_rep = jp.at("visual_rep").get<DVec>();
    p.visual_stat_count = jp.at("visual_stat_count").get<std::int64_t>();
    for (const auto& [ls, ids] : jp.at("clusters").items()) p.per_layer_clusters[std::stoi(ls)] = ids.get<std::vector<std::int64_t>>();
    idx.pending_first_visual_.push_back(Embedding(p.visual_rep.begin(), p.visual_rep.end()));
    idx.pending_appends_.emplace_back();
    idx.pending_parts_.push_back(std::move(p));
  }
  for (const json& jc : root.at("clusters")) {
    ClusterRecord r;
    r.cluster_id = jc.at("id").get<std::int64_t>();
    r.layer_id = jc.at("layer").get<std::int32_t>();
    r.visual_parent = jc.at("parent").get<std::int64_t>();
    r.rep = jc.at("rep").get<DVec>();
    r.variance = jc.at("variance").get<double>();
    r.stat_count = jc.at("stat_count").get<std::int64_t>();
    r.lazy_split = jc.at("lazy_split").get<bool>();
    r.residence = jc.at("residence").get<std::string>() == "device" ? Residence::Device : Residence::Host;
    r.device_tail = jc.at("device_tail").get<std::int64_t>();
    r.first_frame_id = jc.at("first_frame").get<std::int64_t>();
    r.last_touch_frame = jc.at("last_touch").get<std::int64_t>();
    for (const json& je : jc.at("members")) r.members.push_back(entry_from(je));
    for (const json& je : jc.at("buffer")) r.buffer.push_back(entry_from(je));
    r.buffer_rep = jc.at("buffer_rep").get<DVec>();
    if (r.lazy_split) idx.pending_registered_.insert(r.cluster_id);
    idx.pending_clusters_.push_back(std::move(r));
    idx.pending_adopted_.push_back(0);
  }
  return idx;
}

std::vector<std::int64_t> HierIndex::visual_topk(const Embedding& query, int k_v) const {
  if (static_cast<std::int32_t>(query.size()) != dim_) throw DimMismatch(query.size(), static_cast<std::size_t>(dim_));
  if (k_v <= 0) throw ConfigError("visual top-k must be positive");
  b200::Device& dv = device();
  if (check(kvc_n_partitions(dv.ctx)) == 0) throw EmptyIndex("visual_topk on an empty index");
  std::vector<std::int64_t> ids(static_cast<std::size_t>(k_v));
  std::vector<float> pq;
  const int n = check(kvc_visual_topk(dv.ctx, dv.pad(query.data(), 1, pq), k_v, ids.data()));
  ids.resize(static_cast<std::size_t>(std::min(n, k_v)));
  return ids;
}

std::vector<CandidateRef> HierIndex::semantic_topk(const Embedding& query, std::int32_t layer,
                                                   const std::vector<std::int64_t>& partition_ids, int k_s) const {
  if (static_cast<std::int32_t>(query.size()) != dim_) throw DimMismatch(query.size(), static_cast<std::size_t>(dim_));
  if (layer < 0 || layer >= layers_) throw BadLayer(layer);
  if (k_s <= 0) throw ConfigError("semantic top-k must be positive");
  b200::Device& dv = device();
  std::vector<std::int64_t> ids(static_cast<std::size_t>(k_s));
  std::vector<std::int32_t> buf(static_cast<std::size_t>(k_s));
  std::vector<float> pq;
  const int n = check(kvc_semantic_topk(dv.ctx, dv.pad(query.data(), 1, pq), layer, partition_ids.data(),
                                        static_cast<int>(partition_ids.size()), k_s, ids.data(), buf.data()));
  std::vector<CandidateRef> out;
  for (int i = 0; i < n && i < k_s; ++i) out.push_back({ids[static_cast<std::size_t>(i)], buf[static_cast<std::size_t>(i)] != 0});
  return out;
}

std::set<std::int64_t> HierIndex::clusters_of_frame(std::int64_t frame_id) const {
  std::set<std::int64_t> out;
  for (const auto& [id, r] : clusters()) {
    for (const KVEntry& e : r.members)
      if (e.frame_id == frame_id) out.insert(id);
    for (const KVEntry& e : r.buffer)
      if (e.frame_id == frame_id) out.insert(id);
  }
  return out;
}

std::int64_t HierIndex::entries_at_layer(std::int32_t layer) const {
  std::int64_t n = 0;
  for (const auto& [id, r] : clusters())
    if (r.layer_id == layer) n += static_cast<std::int64_t>(r.members.size() + r.buffer.size());
  return n;
}

std::int64_t HierIndex::total_member_entries() const {
  std::int64_t n = 0;
  for (const auto& [id, r] : clusters()) n += r.n();
  return n;
}

void HierIndex::check_invariants() const {
  if (!dev_) return;
  check(kvc_check(device().ctx));
}

// Batch construction (index.cpp:364-450): the frames go through the device engine's batch build
// (visual k-means + per-(partition, layer) spherical k-means on the GPU, kmeans_dev.cu).
HierIndex build_index(const std::vector<FrameInput>& frames, const BuildConfig& cfg) {
  if (frames.empty()) throw EmptyInput("no frames to build from");
  const int d = static_cast<int>(frames.front().visual.size());
  const int L = static_cast<int>(frames.front().layers.size());
  HierIndex idx(d, L);
  kvc_cfg c = component_cfg();
  b200::put_build(c, cfg);
  c.build_batch_frames = static_cast<int>(frames.size());
  c.device_capacity_entries = std::int64_t(1) << 40;
  idx.dev_ = std::make_shared<b200::Device>(c, d, L);
  {
    kvc_cfg bc = c;
    bc.seed = cfg.seed;  // BuildConfig::seed, verbatim
    check(kvc_reconfigure(idx.dev_->ctx, &bc, 8));
  }
  std::vector<float> k, v;
  for (const FrameInput& f : frames) {
    int T = 0;
    b200::pack_frame(f, d, L, k, v, T, idx.dev_->dp);
    std::vector<float> pv;
    check(kvc_ingest_frame(idx.dev_->ctx, f.frame_id, idx.dev_->pad(f.visual.data(), 1, pv), k.data(), v.data(), T, KVC_MEM_HOST,
                           nullptr, nullptr));
  }
  check(kvc_reset_window(idx.dev_->ctx));  // an index has no local window
  // a TieredStore over the built index re-applies its own CostModel (kvc_reconfigure)
  kvc_cfg dflt = b200::base_cfg();
  check(kvc_reconfigure(idx.dev_->ctx, &dflt, 2));
  idx.mark_device_changed();
  return idx;
}

// =============================================================================== TieredStore

TieredStore::TieredStore(HierIndex& index, const CostModel& cost) : index_(index), cost_(cost) {
  if (cost_.alpha_us < 0.0 || cost_.beta_us_per_byte < 0.0) throw ConfigError("transfer costs must be non-negative");
  if (cost_.device_capacity_entries <= 0) throw ConfigError("device capacity must be positive");
  // adopts every existing cluster (store.cpp:67-74): host-assembled ones are adopted when they
  // are installed; a built / device index adopted its clusters when it created them
  for (auto& a : index_.pending_adopted_) a = 1;
  kvc_cfg c = b200::base_cfg();
  b200::put_cost(c, cost_);
  b200::Device& dv = index_.device();
  dv.cfg.alpha_us = c.alpha_us;
  dv.cfg.beta_us_per_byte = c.beta_us_per_byte;
  dv.cfg.bytes_per_entry = c.bytes_per_entry;
  dv.cfg.device_capacity_entries = c.device_capacity_entries;
  check(kvc_reconfigure(dv.ctx, &c, 2));
  ledger_seen_ = static_cast<std::size_t>(check(kvc_ledger_log_size(dv.ctx)));
}

void TieredStore::refresh_ledger() const {
  b200::Device& dv = index_.device();
  const std::size_t n = static_cast<std::size_t>(check(kvc_ledger_log_size(dv.ctx)));
  if (n > ledger_seen_) {
    b200::ledger_ops(dv, ledger_seen_, ledger_);
    ledger_seen_ = n;
  }
}

void TieredStore::adopt(std::int64_t cluster_id) {
  check(kvc_adopt(index_.device().ctx, cluster_id));
  index_.mark_device_changed();
}
void TieredStore::forget(std::int64_t) { throw ConfigError("forget: cluster lifetimes are managed by the device maintainer"); }

double TieredStore::fetch(std::int64_t cluster_id, TransferCause cause) {
  double c = 0.0;
  check(kvc_fetch(index_.device().ctx, cluster_id, static_cast<int>(cause), &c));
  index_.mark_device_changed();
  return c;
}

double TieredStore::offload(std::int64_t cluster_id) {
  double c = 0.0;
  check(kvc_offload(index_.device().ctx, cluster_id, &c));
  index_.mark_device_changed();
  return c;
}

void TieredStore::note_device_append(std::int64_t) {
  throw ConfigError("note_device_append: device appends are recorded by the device maintainer");
}
void TieredStore::note_device_buffer_append(std::int64_t) {
  throw ConfigError("note_device_buffer_append: device appends are recorded by the device maintainer");
}

void TieredStore::touch(std::int64_t cluster_id) { check(kvc_touch(index_.device().ctx, cluster_id)); }

void TieredStore::pin(const std::set<std::int64_t>& cluster_ids) {
  std::vector<std::int64_t> ids(cluster_ids.begin(), cluster_ids.end());
  check(kvc_pin(index_.device().ctx, ids.data(), static_cast<int>(ids.size())));
}

bool TieredStore::on_device(std::int64_t cluster_id) const {
  return index_.cluster(cluster_id).residence == Residence::Device;
}

std::int64_t TieredStore::device_entries() const {
  std::int64_t ops[5], by[5];
  double co[5];
  const std::int64_t r = kvc_ledger(index_.device().ctx, ops, by, co);
  if (r < 0) b200::raise(static_cast<int>(r));
  return r;
}

double TieredStore::enforce_capacity() {
  double c = 0.0;
  check(kvc_enforce_capacity(index_.device().ctx, &c));
  index_.mark_device_changed();
  return c;
}

TransferLedger& TieredStore::ledger() {
  refresh_ledger();
  return ledger_;
}
const TransferLedger& TieredStore::ledger() const {
  refresh_ledger();
  return ledger_;
}

void TieredStore::audit() const { check(kvc_check(index_.device().ctx)); }

// =============================================================================== Maintainer

Maintainer::Maintainer(HierIndex& index, TieredStore& store, const MaintainerConfig& cfg)
    : index_(index), store_(store), cfg_(cfg) {
  if (cfg_.threshold.tau_min < 0.0 || cfg_.threshold.tau_max < cfg_.threshold.tau_min)
    throw ConfigError("variance thresholds must satisfy 0 <= tau_min <= tau_max");
  if (cfg_.threshold.n0 <= 0.0) throw ConfigError("threshold horizon must be positive");
  if (cfg_.max_split_depth < 1) throw ConfigError("split depth must be at least 1");
  if (cfg_.visual_floor < -1.0 || cfg_.visual_floor > 1.0) throw ConfigError("visual floor must be a cosine value");
  kvc_cfg c = b200::base_cfg();
  b200::put_maintainer(c, cfg_);
  c.seed = cfg_.seed;
  check(kvc_reconfigure(index_.device().ctx, &c, 4));
}

std::int64_t Maintainer::place_frame(std::int64_t frame_id, const Embedding& visual) {
  if (static_cast<std::int32_t>(visual.size()) != index_.dim()) throw DimMismatch(visual.size(), static_cast<std::size_t>(index_.dim()));
  std::int64_t pid = -1;
  std::vector<float> pv;
  b200::Device& dv = index_.device();
  check(kvc_place_frame(dv.ctx, frame_id, dv.pad(visual.data(), 1, pv), &pid));
  index_.mark_device_changed();
  return pid;
}

std::int64_t Maintainer::on_insert(std::int64_t partition_id, const KVEntry& entry) {
  if (static_cast<std::int32_t>(entry.key.size()) != index_.dim() || entry.value.size() != entry.key.size())
    throw DimMismatch(entry.key.size(), static_cast<std::size_t>(index_.dim()));
  std::int64_t cid = -1;
  b200::Device& dv = index_.device();
  std::vector<float> pk, pv;
  check(kvc_insert(dv.ctx, partition_id, entry.layer_id, entry.token_id, entry.frame_id, dv.pad(entry.key.data(), 1, pk),
                   dv.pad(entry.value.data(), 1, pv), &cid));
  index_.mark_device_changed();
  return cid;
}

std::vector<std::int64_t> Maintainer::materialize(std::int64_t cluster_id) {
  std::vector<std::int64_t> ids(64);
  int n = check(kvc_materialize(index_.device().ctx, cluster_id, ids.data(), static_cast<int>(ids.size())));
  if (n > static_cast<int>(ids.size())) throw InvariantViolation("materialize returned more ids than expected");
  ids.resize(static_cast<std::size_t>(n));
  index_.mark_device_changed();
  return ids;
}

const MaintainerStats& Maintainer::stats() const {
  std::int64_t o[9];
  check(kvc_maint_stats(index_.device().ctx, o));
  stats_ = {o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8]};
  return stats_;
}

// =============================================================================== retrieval

RetrievalResult retrieve(const QueryBundle& bundle, const RetrievalConfig& cfg, HierIndex& index, TieredStore& store,
                         Maintainer& maintainer, const std::vector<KVEntry>& window) {
  (void)maintainer;
  cfg.validate();
  if (cfg.mode != RetrievalMode::Cluster) throw ConfigError("retrieve() is the cluster path (RetrievalMode::Cluster)");
  if (!window.empty())
    throw ConfigError("retrieve(): the device engine keeps its local window itself (StreamEngine); pass an empty window");
  b200::Device& dv = index.device();
  if (check(kvc_n_partitions(dv.ctx)) == 0) throw EmptyIndex("retrieve before any index was built");
  kvc_cfg c = dv.cfg;
  b200::put_retrieval(c, cfg);
  check(kvc_reconfigure(dv.ctx, &c, 1));
  check(kvc_reset_window(dv.ctx));
  const std::vector<float> q = b200::pack_query(bundle, dv.d, dv.L, dv.dp);
  b200::g_attention.assign(static_cast<std::size_t>(dv.L) * dv.dp, 0.f);
  const auto& gt = bundle.ground_truth_frames;
  check(kvc_decode_step(dv.ctx, bundle.query_id, q.data(), KVC_MEM_HOST, b200::g_attention.data(), KVC_MEM_HOST,
                        gt.empty() ? nullptr : gt.data(), static_cast<int>(gt.size())));
  dv.cut(b200::g_attention, static_cast<std::size_t>(dv.L));
  RetrievalResult r = b200::read_result(dv, bundle.query_id);
  index.mark_device_changed();
  store.ledger();  // pull the step's ledger ops
  return r;
}

std::vector<CandidateRef> oracle_flat_topk(const HierIndex& index, const Embedding& query, std::int32_t layer, int k) {
  if (static_cast<std::int32_t>(query.size()) != index.dim()) throw DimMismatch(query.size(), static_cast<std::size_t>(index.dim()));
  if (layer < 0 || layer >= index.num_layers()) throw BadLayer(layer);
  b200::Device& dv = index.device();
  const int cap = std::max(1, std::min(k, check(kvc_n_clusters(dv.ctx)) * 2 + 1));
  std::vector<std::int64_t> ids(static_cast<std::size_t>(cap));
  std::vector<std::int32_t> buf(static_cast<std::size_t>(cap));
  std::vector<float> pq;
  const int n = check(kvc_flat_topk(dv.ctx, dv.pad(query.data(), 1, pq), layer, std::min(k, cap), ids.data(), buf.data()));
  std::vector<CandidateRef> out;
  for (int i = 0; i < n; ++i) out.push_back({ids[static_cast<std::size_t>(i)], buf[static_cast<std::size_t>(i)] != 0});
  return out;
}

// The token-granular baseline on the device (token.cu + K6): a token-mode context holding the
// pools frame by frame; window_frames must be the pools' last frames (or empty).
RetrievalResult retrieve_token_baseline(const QueryBundle& bundle, const RetrievalConfig& cfg,
                                        const std::vector<std::vector<KVEntry>>& pools,
                                        const std::set<std::int64_t>& window_frames, const CostModel& cost,
                                        TransferLedger& ledger) {
  cfg.validate();
  const int L = static_cast<int>(pools.size());
  if (static_cast<int>(bundle.q.size()) != L) throw ConfigError("query bundle layer count does not match the stored layers");
  RetrievalResult empty;
  int d = 0;
  for (const auto& p : pools)
    if (!p.empty()) d = static_cast<int>(p.front().key.size());
  if (d == 0) {  // every pool empty: nothing ranked, nothing attended (retrieval.cpp:185)
    empty.query_id = bundle.query_id;
    empty.layers.resize(static_cast<std::size_t>(L));
    return empty;
  }
  // frames in pool order; every layer must hold the same frames with tokens 0..T-1
  std::vector<std::pair<std::int64_t, int>> frames;  // (frame id, T)
  {
    const auto& p0 = pools.front();
    for (std::size_t i = 0; i < p0.size();) {
      std::size_t j = i;
      while (j < p0.size() && p0[j].frame_id == p0[i].frame_id) {
        if (p0[j].token_id != static_cast<int>(j - i)) throw ConfigError("token pools must hold whole frames (tokens 0..T-1 in order)");
        ++j;
      }
      frames.push_back({p0[i].frame_id, static_cast<int>(j - i)});
      i = j;
    }
    for (const auto& p : pools)
      if (p.size() != p0.size()) throw ConfigError("token pools must hold the same frames at every layer");
  }
  kvc_cfg c = b200::base_cfg();
  b200::put_retrieval(c, cfg);
  b200::put_cost(c, cost);
  c.token_mode = 1;
  c.window_frames = std::max<int>(1, static_cast<int>(window_frames.size()));
  c.max_tokens = 1;
  for (const auto& f : frames) c.max_tokens = std::max(c.max_tokens, f.second);
  std::int64_t rows = static_cast<std::int64_t>(pools.front().size());
  c.pool_bytes = std::max<std::int64_t>(rows * d * 4 * 2 * L + (1 << 20), 1 << 22);
  b200::Device dv(c, d, L);
  std::vector<float> k, v;
  std::size_t off = 0;
  for (const auto& [fid, T] : frames) {
    k.assign(static_cast<std::size_t>(L) * T * dv.dp, 0.f);
    v.assign(k.size(), 0.f);
    for (int l = 0; l < L; ++l)
      for (int t = 0; t < T; ++t) {
        const KVEntry& e = pools[static_cast<std::size_t>(l)][off + static_cast<std::size_t>(t)];
        if (e.frame_id != fid) throw ConfigError("token pools must hold the same frames at every layer");
        std::memcpy(&k[(static_cast<std::size_t>(l) * T + t) * dv.dp], e.key.data(), static_cast<std::size_t>(d) * 4);
        std::memcpy(&v[(static_cast<std::size_t>(l) * T + t) * dv.dp], e.value.data(), static_cast<std::size_t>(d) * 4);
      }
    std::vector<float> vis(static_cast<std::size_t>(dv.dp), 0.f);
    check(kvc_ingest_frame(dv.ctx, fid, vis.data(), k.data(), v.data(), T, KVC_MEM_HOST, nullptr, nullptr));
    off += static_cast<std::size_t>(T);
  }
  // the window: the pools' last |window_frames| frames, else nothing
  bool tail = window_frames.size() <= frames.size();
  for (std::size_t i = 0; tail && i < window_frames.size(); ++i)
    tail = window_frames.count(frames[frames.size() - 1 - i].first) != 0;
  if (!tail) throw ConfigError("retrieve_token_baseline: window_frames must be the pools' most recent frames");
  if (window_frames.empty()) check(kvc_reset_window(dv.ctx));
  const b200::Totals t0 = b200::ledger_totals(dv);
  const std::vector<float> q = b200::pack_query(bundle, d, L, dv.dp);
  b200::g_attention.assign(static_cast<std::size_t>(L) * dv.dp, 0.f);
  const auto& gt = bundle.ground_truth_frames;
  check(kvc_decode_step(dv.ctx, bundle.query_id, q.data(), KVC_MEM_HOST, b200::g_attention.data(), KVC_MEM_HOST,
                        gt.empty() ? nullptr : gt.data(), static_cast<int>(gt.size())));
  dv.cut(b200::g_attention, static_cast<std::size_t>(L));
  RetrievalResult r = b200::read_result(dv, bundle.query_id);
  const b200::Totals t1 = b200::ledger_totals(dv);
  if (t1.ops > t0.ops) {  // the step's coalesced-run ops, recorded as one aggregate entry
    TransferOp op{TransferCause::Retrieval, true, -1, t1.ops - t0.ops, t1.bytes - t0.bytes, t1.cost - t0.cost};
    ledger.record(op);
  }
  return r;
}

// =============================================================================== StreamEngine

void EngineConfig::validate() const {  // engine.cpp:9-14
  retrieval.validate();
  if (build_batch_frames < 1) throw ConfigError("build batch must be at least 1 frame");
  if (ingest_overhead_us < 0.0) throw ConfigError("ingestion overhead must be non-negative");
  if (offload_horizon_frames < 1) throw ConfigError("offload horizon must be at least 1 frame");
}

StreamEngine::StreamEngine(const EngineConfig& cfg, int d, int L) : cfg_(cfg), d_(d), L_(L) {
  cfg_.validate();
  if (d < 1 || L < 1) throw ConfigError("stream dimensions must be positive");
  kvc_cfg c = b200::base_cfg();
  b200::put_retrieval(c, cfg_.retrieval);
  b200::put_maintainer(c, cfg_.maintainer);
  b200::put_build(c, cfg_.build);
  b200::put_cost(c, cfg_.cost);
  c.build_batch_frames = cfg_.build_batch_frames;
  c.batched_ingest = cfg_.batched_ingest ? 1 : 0;
  c.ingest_overhead_us = cfg_.ingest_overhead_us;
  c.offload_horizon_frames = cfg_.offload_horizon_frames;
  c.seed = cfg_.seed;
  c.check_invariants = 1;  // engine.cpp:234-236 checks the index and the store after every query
  dev_ = std::make_shared<b200::Device>(c, d, L);
}

StreamEngine::~StreamEngine() = default;
StreamEngine::StreamEngine(StreamEngine&&) noexcept = default;
StreamEngine& StreamEngine::operator=(StreamEngine&&) noexcept = default;

void StreamEngine::process(const StreamEvent& event) {
  if (event.kind == StreamEvent::Kind::Frame)
    ingest_frame(event.frame);
  else
    answer_query(event.query);
}

void StreamEngine::ingest_frame(const FrameInput& frame) {  // engine.cpp:134-174
  std::vector<float> k, v;
  int T = 0;
  b200::pack_frame(frame, d_, L_, k, v, T, dev_->dp);
  frames_processed_ += 1;
  frames_in_batch_ += 1;
  if (cfg_.batched_ingest) {
    if (frames_in_batch_ == cfg_.build_batch_frames) {
      ingest_cost_us_ += cfg_.ingest_overhead_us;
      frames_in_batch_ = 0;
    }
  } else {
    ingest_cost_us_ += cfg_.ingest_overhead_us;
    frames_in_batch_ = 0;
  }
  std::vector<float> pvis;
  check(kvc_ingest_frame(dev_->ctx, frame.frame_id, dev_->pad(frame.visual.data(), 1, pvis), k.data(), v.data(), T, KVC_MEM_HOST, nullptr,
                         nullptr));
  if (view_) view_->mark_device_changed();
}

void StreamEngine::answer_query(const QueryBundle& bundle) {  // engine.cpp:176-237
  const bool token = cfg_.retrieval.mode == RetrievalMode::TokenBaseline;
  const b200::Totals t0 = b200::ledger_totals(*dev_);
  const std::vector<float> q = b200::pack_query(bundle, d_, L_, dev_->dp);
  att_.assign(static_cast<std::size_t>(L_) * dev_->dp, 0.f);
  const auto& gt = bundle.ground_truth_frames;
  check(kvc_decode_step(dev_->ctx, bundle.query_id, q.data(), KVC_MEM_HOST, att_.data(), KVC_MEM_HOST,
                        gt.empty() ? nullptr : gt.data(), static_cast<int>(gt.size())));
  dev_->cut(att_, static_cast<std::size_t>(L_));
  const b200::Totals t1 = b200::ledger_totals(*dev_);
  QueryRow row;
  row.query_id = bundle.query_id;
  row.ops = t1.ops - t0.ops;
  row.bytes = t1.bytes - t0.bytes;
  double dd[2];
  check(kvc_last_query_meta(dev_->ctx, dd));
  row.ttft_us = dd[0];
  row.recall = dd[1];
  for (int l = 0; l < L_; ++l) {
    double lat[5];
    std::int64_t ints[5];
    check(kvc_last_layer_meta(dev_->ctx, l, lat, ints));
    row.lookup_us += lat[0];
    row.transfer_us += lat[1];
    row.stall_us += lat[2];
    row.completion_us += lat[3];
    row.compute_us += lat[4];
    if (!token && cfg_.retrieval.prefetch_enabled && l > 0) {
      row.prefetch_hits += ints[1];
      row.verified_clusters += ints[0];
    }
  }
  row.realized_frames = check(kvc_last_frames(dev_->ctx, 0, nullptr, 0));
  row.context_frames = check(kvc_last_frames(dev_->ctx, 1, nullptr, 0));
  row.attended_digest = kvc_last_digest(dev_->ctx);
  rows_.push_back(row);
  if (token && t1.ops > t0.ops)  // the baseline keeps totals: one aggregate op per query
    tok_ledger_.record({TransferCause::Retrieval, true, -1, t1.ops - t0.ops, t1.bytes - t0.bytes, t1.cost - t0.cost});
  if (view_) view_->mark_device_changed();
}

RunOutput StreamEngine::finish() {  // engine.cpp:239-264
  RunOutput out;
  if (cfg_.retrieval.mode == RetrievalMode::Cluster) {
    if (check(kvc_n_partitions(dev_->ctx)) == 0) {
      const int rc = kvc_build_now(dev_->ctx);  // pending frames (none: nothing to build)
      if (rc < 0 && rc != KVC_E_EMPTY_INDEX) b200::raise(rc);
    }
    if (check(kvc_n_partitions(dev_->ctx)) > 0) {
      check(kvc_check(dev_->ctx));
      std::int64_t o[9];
      check(kvc_maint_stats(dev_->ctx, o));
      out.maintainer = {o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8]};
      b200::ledger_ops(*dev_, 0, out.ledger);
      out.final_partitions = check(kvc_n_partitions(dev_->ctx));
      out.final_clusters = check(kvc_n_clusters(dev_->ctx));
    }
  } else {
    out.ledger = tok_ledger_;
  }
  if (cfg_.batched_ingest && frames_in_batch_ > 0) {
    ingest_cost_us_ += cfg_.ingest_overhead_us;
    frames_in_batch_ = 0;
  }
  out.rows = rows_;
  out.ingest_cost_us = ingest_cost_us_;
  out.frames_processed = frames_processed_;
  out.queries_processed = static_cast<std::int64_t>(rows_.size());
  return out;
}

const HierIndex* StreamEngine::index() const {
  if (cfg_.retrieval.mode != RetrievalMode::Cluster) return nullptr;
  if (check(kvc_n_partitions(dev_->ctx)) == 0) return nullptr;
  if (!view_) {
    view_ = std::make_unique<HierIndex>(d_, L_);
    view_->dev_ = dev_;
  }
  return view_.get();
}

RunOutput run_stream(const EngineConfig& cfg, int d, int L, const std::vector<StreamEvent>& events) {
  StreamEngine engine(cfg, d, L);
  for (const StreamEvent& ev : events) engine.process(ev);
  return engine.finish();
}

}  // namespace kvclust
