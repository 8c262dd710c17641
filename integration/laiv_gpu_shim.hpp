// laiv_gpu_shim.hpp — the C++ shim a laiv maintainer adds to run the
// reference's hot path (proj/core, namespace laiv) on a B200 through the C ABI
// of liblaivg.so (include/laivg.h).
//
// Every function below has the reference's signature, in namespace laiv::gpu,
// with one type swapped: laiv::gpu::TieredStore is a TieredStore whose fast
// tier is a GPU's HBM cluster cache (same member functions as
// laiv::TieredStore, tiered.hpp:22-56; constructed with the index it caches).
// Re-pointing the reference's caller (pipeline.cpp serve_microbatch /
// run_batch) is a namespace change plus that constructor:
//
//   laiv::gpu::TieredStore store(capacity, ix, db, /*device=*/w);
//   auto plan = laiv::gpu::plan_prefetch(ix, q_in, budget, store);
//   laiv::gpu::execute_prefetch(store, plan, chan, window, ix, db);
//   auto [res, t] = laiv::gpu::hybrid_search(ix, db, store, q_out, L, k, cost);
//
// A channel of mode laiv::gpu::kDevice (the ChannelMode::Device extension of
// tiered.hpp:65) streams the lists host->HBM on a copy stream while a timed
// generation-window kernel occupies the GPU; SimulatedClock and Measured keep
// the reference's meaning.
//
// Binding: the first TieredStore (or DeviceIndex) of an (IvfIndex,
// EmbeddingMatrix) pair gathers the rows ONCE, list by list (the LAIX order
// load_index produces, ivf.cpp:437-455), straight into pinned host memory the
// library borrows (laivg_host_alloc + LAIVG_INDEX_BORROW): one host copy of
// the datastore, which every GPU's cache copies from. Functions without a
// store argument (ivf_search, rank_clusters, ...) run on the most recent
// TieredStore of their index.
//
// Header-only; needs the reference headers (laiv/*.hpp) and include/laivg.h.
// Errors come back as the reference's exception classes.
#pragma once

#include <laiv/budget.hpp>
#include <laiv/cache.hpp>
#include <laiv/ivf.hpp>
#include <laiv/sched.hpp>
#include <laiv/tiered.hpp>
#include <laiv/vectorstore.hpp>

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "laivg.h"

namespace laiv::gpu {

[[noreturn]] inline void raise(int rc) {
  const std::string m = laivg_last_error();
  switch (rc) {
    case LAIVG_EINVAL: throw std::invalid_argument(m);
    case LAIVG_ELOGIC: throw std::logic_error(m);
    default: throw std::runtime_error(m); // ERUNTIME, ECUDA
  }
}
inline void ck(int rc) {
  if (rc != LAIVG_OK) raise(rc);
}

/// tiered.hpp:65 extension: ChannelMode::Device.
inline constexpr ChannelMode kDevice = static_cast<ChannelMode>(2);

inline int channel_mode(ChannelMode m) {
  switch (m) {
    case ChannelMode::SimulatedClock: return LAIVG_CHAN_SIMULATED;
    case ChannelMode::Measured: return LAIVG_CHAN_MEASURED;
    default: return LAIVG_CHAN_DEVICE;
  }
}

class TieredStore;

/// An index + datastore bound into the library's list-major pinned store.
class DeviceIndex {
 public:
  DeviceIndex(const IvfIndex& ix, const EmbeddingMatrix& db) : ix_ref_(&ix), db_ref_(&db) {
    const uint32_t d = ix.dim(), nc = ix.num_clusters();
    if (db.dim() != d && db.count()) throw std::invalid_argument("index/datastore dim mismatch");
    std::vector<uint64_t> off(nc + 1, 0);
    for (uint32_t c = 0; c < nc; ++c) off[c + 1] = off[c] + ix.list(c).size();
    const uint64_t n = off[nc];
    const uint64_t vb = n * d * sizeof(float), ib = n * sizeof(uint64_t);
    ck(laivg_host_alloc(vb + ib + 16, &block_));
    float* vecs = static_cast<float*>(block_);
    uint64_t* ids = reinterpret_cast<uint64_t*>(static_cast<char*>(block_) + ((vb + 15) & ~15ull));
    for (uint32_t c = 0; c < nc; ++c) {
      const auto& lst = ix.list(c);
      for (size_t i = 0; i < lst.size(); ++i) {
        const auto r = db.row_of(lst[i]);
        if (!r) {
          laivg_host_free(block_);
          throw std::runtime_error("index references id " + std::to_string(lst[i]) +
                                   " missing from the datastore");
        }
        const auto row = db.row(*r);
        std::copy(row.begin(), row.end(), vecs + (off[c] + i) * d);
        ids[off[c] + i] = lst[i];
      }
    }
    // rows were validated by EmbeddingMatrix::append (vectorstore.cpp:66-85)
    const int rc = laivg_index_create(ix.centroids().data().data(), nc, d, int(ix.metric()), vecs,
                                      ids, off.data(), LAIVG_INDEX_BORROW | LAIVG_INDEX_TRUST, &h_);
    if (rc != LAIVG_OK) {
      laivg_host_free(block_);
      raise(rc);
    }
  }
  /// Straight from a LAIX file (what load_index reads, ivf.hpp:98): the
  /// library reads the lists into its pinned store in parallel.
  explicit DeviceIndex(const std::string& laix_path, uint32_t threads = 0) {
    ck(laivg_index_load(laix_path.c_str(), threads, &h_));
  }
  ~DeviceIndex() {
    laivg_index_destroy(h_);
    if (block_) laivg_host_free(block_);
  }
  DeviceIndex(const DeviceIndex&) = delete;
  DeviceIndex& operator=(const DeviceIndex&) = delete;

  laivg_index* handle() const { return h_; }
  uint32_t dim() const { return laivg_index_dim(h_); }
  uint32_t num_clusters() const { return laivg_index_num_clusters(h_); }
  Metric metric() const { return static_cast<Metric>(laivg_index_metric(h_)); }
  uint64_t cluster_bytes(uint32_t c) const { return laivg_index_cluster_bytes(h_, c); }
  uint64_t list_len(uint32_t c) const { return laivg_index_list_len(h_, c); }
  // save_index (ivf.hpp:96) of the bound store
  void save(const std::string& path, uint32_t threads = 0) const {
    ck(laivg_index_save(h_, path.c_str(), threads));
  }

 private:
  friend class TieredStore;
  const IvfIndex* ix_ref_ = nullptr;
  const EmbeddingMatrix* db_ref_ = nullptr;
  laivg_index* h_ = nullptr;
  void* block_ = nullptr;
};

namespace detail {
// bound indexes by (IvfIndex, EmbeddingMatrix) address; the stores of each
struct Registry {
  std::mutex mu;
  std::map<std::pair<const void*, const void*>, std::weak_ptr<DeviceIndex>> bound;
  std::map<const void*, TieredStore*> last_store;  // by IvfIndex or EmbeddingMatrix
  std::vector<TieredStore*> all;
};
inline Registry& reg() {
  static Registry r;
  return r;
}
} // namespace detail

/// The GPU fast tier: laiv::TieredStore's interface (tiered.hpp:22-56) over
/// one device context (its HBM cluster cache, streams, host miss pool).
class TieredStore {
 public:
  TieredStore(uint64_t capacity_bytes, const IvfIndex& ix, const EmbeddingMatrix& db,
              int device = 0, const laivg_opts* opts = nullptr) {
    auto& r = detail::reg();
    {
      std::lock_guard<std::mutex> g(r.mu);
      auto& w = r.bound[{&ix, &db}];
      index_ = w.lock();
      if (!index_) {
        index_ = std::make_shared<DeviceIndex>(ix, db);
        w = index_;
      }
    }
    open(capacity_bytes, device, opts);
    keys_ = {&ix, &db};
    register_self();
  }
  TieredStore(uint64_t capacity_bytes, std::shared_ptr<DeviceIndex> index, int device = 0,
              const laivg_opts* opts = nullptr)
      : index_(std::move(index)) {
    open(capacity_bytes, device, opts);
    register_self();
  }
  ~TieredStore() {
    auto& r = detail::reg();
    {
      std::lock_guard<std::mutex> g(r.mu);
      for (auto it = r.last_store.begin(); it != r.last_store.end();) {
        it = it->second == this ? r.last_store.erase(it) : std::next(it);
      }
      r.all.erase(std::remove(r.all.begin(), r.all.end(), this), r.all.end());
    }
    laivg_ctx_destroy(ctx_);
  }
  TieredStore(const TieredStore&) = delete;
  TieredStore& operator=(const TieredStore&) = delete;

  // ---- tiered.hpp:26-51 ----
  uint64_t capacity_bytes() const { return laivg_store_capacity_bytes(ctx_); }
  uint64_t used_bytes() const { return laivg_store_used_bytes(ctx_); }
  uint64_t free_bytes() const { return laivg_store_free_bytes(ctx_); }
  bool contains(uint32_t cluster) const { return laivg_store_contains(ctx_, cluster) != 0; }
  size_t resident_count() const { return laivg_store_resident_count(ctx_); }
  std::map<uint32_t, std::pair<Residency, uint64_t>> resident() const {
    const uint32_t n = laivg_store_resident_count(ctx_);
    std::vector<uint32_t> cl(n ? n : 1);
    std::vector<uint8_t> tg(n ? n : 1);
    std::vector<uint64_t> by(n ? n : 1);
    uint32_t got = 0;
    ck(laivg_store_resident(ctx_, cl.data(), tg.data(), by.data(), &got));
    std::map<uint32_t, std::pair<Residency, uint64_t>> m;
    for (uint32_t i = 0; i < got; ++i) m[cl[i]] = {static_cast<Residency>(tg[i]), by[i]};
    return m;
  }
  /// Makes the cluster resident with its payload copied into HBM. `bytes`
  /// is the reference's accounting (IvfIndex::cluster_bytes).
  void insert(uint32_t cluster, uint64_t bytes, Residency tag) {
    if (cluster < index_->num_clusters() && bytes != index_->cluster_bytes(cluster)) {
      throw std::invalid_argument("insert: bytes must be cluster_bytes(" +
                                  std::to_string(cluster) + ")");
    }
    ck(laivg_store_insert(ctx_, cluster, int(tag)));
  }
  uint64_t evict(uint32_t cluster) {
    uint64_t b = 0;
    ck(laivg_store_evict(ctx_, cluster, &b));
    return b;
  }
  void retag_all(Residency tag) { ck(laivg_store_retag_all(ctx_, int(tag))); }
  void clear() { ck(laivg_store_clear(ctx_)); }
  uint64_t bytes_with_tag(Residency tag) const { return laivg_store_bytes_with_tag(ctx_, int(tag)); }
  uint64_t recompute_used_bytes() const { return laivg_store_recompute_used_bytes(ctx_); }

  // ---- device-side extras ----
  laivg_ctx* ctx() const { return ctx_; }
  const DeviceIndex& index() const { return *index_; }
  /// Slab compaction (paper: consolidate GPU memory after a batch).
  void compact() { ck(laivg_store_compact(ctx_)); }

 private:
  void open(uint64_t capacity_bytes, int device, const laivg_opts* opts) {
    laivg_opts o;
    if (opts) o = *opts;
    else laivg_opts_default(&o);
    o.device = device;
    o.capacity_bytes = capacity_bytes;
    ck(laivg_ctx_create(index_->handle(), &o, &ctx_));
  }
  void register_self() {
    auto& r = detail::reg();
    std::lock_guard<std::mutex> g(r.mu);
    if (keys_.first) r.last_store[keys_.first] = this;
    if (keys_.second) r.last_store[keys_.second] = this;
    r.all.push_back(this);
  }
  std::shared_ptr<DeviceIndex> index_;
  laivg_ctx* ctx_ = nullptr;
  std::pair<const void*, const void*> keys_{nullptr, nullptr};
};

namespace detail {
inline TieredStore& store_for(const void* key, const char* what) {
  auto& r = reg();
  std::lock_guard<std::mutex> g(r.mu);
  auto it = r.last_store.find(key);
  if (it == r.last_store.end()) {
    throw std::logic_error(std::string(what) +
                           ": no laiv::gpu::TieredStore is bound to this index/datastore");
  }
  return *it->second;
}
inline TieredStore& any_store(const char* what) {
  auto& r = reg();
  std::lock_guard<std::mutex> g(r.mu);
  if (r.all.empty()) throw std::logic_error(std::string(what) + ": no GPU context is open");
  return *r.all.back();
}
inline TopK to_topk(int k, const uint64_t* ids, const float* sc, uint32_t n) {
  TopK t{k, {}};
  t.entries.reserve(n);
  for (uint32_t i = 0; i < n; ++i) t.entries.push_back({ids[i], sc[i]});
  return t;
}
inline void check_dim(const TieredStore& s, std::span<const float> q) {
  if (q.size() != s.index().dim()) throw std::invalid_argument("query dim mismatch");
}
} // namespace detail

// ---- ivf.hpp ----------------------------------------------------------------
/// ivf.hpp:68-69
inline std::vector<uint32_t> rank_clusters(const IvfIndex& ix, std::span<const float> q) {
  auto& s = detail::store_for(&ix, "rank_clusters");
  detail::check_dim(s, q);
  std::vector<uint32_t> out(s.index().num_clusters());
  ck(laivg_rank_clusters(s.ctx(), q.data(), 1, out.data(), nullptr));
  return out;
}

/// ivf.hpp:72-73
inline std::vector<uint32_t> coarse_probe(const IvfIndex& ix, std::span<const float> q, int L) {
  auto& s = detail::store_for(&ix, "coarse_probe");
  detail::check_dim(s, q);
  std::vector<uint32_t> out(std::max<uint32_t>(1, s.index().num_clusters()));
  uint32_t lp = 0;
  ck(laivg_coarse_probe(s.ctx(), q.data(), 1, L, out.data(), &lp));
  out.resize(lp);
  return out;
}

/// ivf.hpp:75-81
inline std::vector<ScoredId> score_clusters(const IvfIndex& ix, const EmbeddingMatrix& db,
                                            std::span<const float> q,
                                            std::span<const uint32_t> clusters) {
  (void)db;
  auto& s = detail::store_for(&ix, "score_clusters");
  detail::check_dim(s, q);
  uint64_t n = 0;
  for (uint32_t c : clusters) {
    if (c >= s.index().num_clusters()) {
      throw std::invalid_argument("unknown cluster id " + std::to_string(c));
    }
    n += s.index().list_len(c);
  }
  std::vector<uint64_t> ids(n ? n : 1);
  std::vector<float> sc(n ? n : 1);
  uint64_t got = 0;
  ck(laivg_score_clusters(s.ctx(), q.data(), clusters.data(), uint32_t(clusters.size()), n,
                          ids.data(), sc.data(), &got));
  std::vector<ScoredId> out(got);
  for (uint64_t i = 0; i < got; ++i) out[i] = {ids[i], sc[i]};
  return out;
}

/// ivf.hpp:85-87
inline TopK search_clusters(const IvfIndex& ix, const EmbeddingMatrix& db,
                            std::span<const float> q, std::span<const uint32_t> clusters,
                            int k) {
  (void)db;
  auto& s = detail::store_for(&ix, "search_clusters");
  detail::check_dim(s, q);
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  std::vector<uint64_t> ids(k);
  std::vector<float> sc(k);
  uint32_t n = 0;
  ck(laivg_search_clusters(s.ctx(), q.data(), clusters.data(), uint32_t(clusters.size()), k,
                           ids.data(), sc.data(), &n));
  return detail::to_topk(k, ids.data(), sc.data(), n);
}

/// ivf.hpp:90-91
inline TopK ivf_search(const IvfIndex& ix, const EmbeddingMatrix& db, std::span<const float> q,
                       int L, int k) {
  (void)db;
  auto& s = detail::store_for(&ix, "ivf_search");
  detail::check_dim(s, q);
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  std::vector<uint64_t> ids(k);
  std::vector<float> sc(k);
  uint32_t n = 0;
  ck(laivg_ivf_search(s.ctx(), q.data(), 1, L, k, ids.data(), sc.data(), &n));
  return detail::to_topk(k, ids.data(), sc.data(), n);
}

/// ivf_search over a batch (extension point (2): one device pass per
/// max_batch queries; the reference loops ivf_search).
inline std::vector<TopK> ivf_search_batch(const IvfIndex& ix, const EmbeddingMatrix& db,
                                          const EmbeddingMatrix& queries, int L, int k) {
  (void)db;
  auto& s = detail::store_for(&ix, "ivf_search_batch");
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  const uint32_t nq = uint32_t(queries.count());
  std::vector<uint64_t> ids(size_t(nq) * k + 1);
  std::vector<float> sc(size_t(nq) * k + 1);
  std::vector<uint32_t> cnt(nq + 1);
  if (nq) {
    ck(laivg_ivf_search(s.ctx(), queries.data().data(), nq, L, k, ids.data(), sc.data(),
                        cnt.data()));
  }
  std::vector<TopK> out;
  for (uint32_t q = 0; q < nq; ++q) {
    out.push_back(detail::to_topk(k, ids.data() + size_t(q) * k, sc.data() + size_t(q) * k, cnt[q]));
  }
  return out;
}

// ---- vectorstore.hpp --------------------------------------------------------
/// vectorstore.hpp:94-98: over the bound datastore `db` (the union of the
/// index's lists).
inline TopK exact_search(const EmbeddingMatrix& db, std::span<const float> q, int k, Metric m) {
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  auto& s = detail::store_for(&db, "exact_search");
  if (db.count() && q.size() != db.dim()) {
    throw std::invalid_argument("query dim " + std::to_string(q.size()) +
                                " does not match db dim " + std::to_string(db.dim()));
  }
  if (m != s.index().metric()) {
    throw std::invalid_argument("exact_search: metric differs from the bound index's");
  }
  std::vector<uint64_t> ids(k);
  std::vector<float> sc(k);
  uint32_t n = 0;
  ck(laivg_exact_search(s.ctx(), q.data(), 1, k, ids.data(), sc.data(), &n));
  return detail::to_topk(k, ids.data(), sc.data(), n);
}

/// vectorstore.hpp:100-102 (on the GPU of any open store)
inline std::vector<float> pairwise_l2(const EmbeddingMatrix& a, const EmbeddingMatrix& b) {
  if (a.dim() != b.dim()) throw std::invalid_argument("pairwise_l2: dim mismatch");
  std::vector<float> out(a.count() * b.count());
  if (out.empty()) return out;
  auto& s = detail::any_store("pairwise_l2");
  ck(laivg_pairwise_l2(s.ctx(), a.data().data(), a.count(), b.data().data(), b.count(), a.dim(),
                       out.data()));
  return out;
}

// ---- tiered.hpp -------------------------------------------------------------
/// tiered.hpp:97-98 (against the GPU cache's residency)
inline PrefetchPlan plan_prefetch(const IvfIndex& ix, std::span<const float> q_in,
                                  uint64_t budget_bytes, const TieredStore& resident) {
  (void)ix;
  detail::check_dim(resident, q_in);
  const uint32_t nc = resident.index().num_clusters();
  std::vector<uint32_t> plan(nc + 1), skipped(nc + 1);
  uint32_t np = 0, ns = 0;
  uint64_t pb = 0;
  ck(laivg_plan_prefetch(resident.ctx(), q_in.data(), budget_bytes, plan.data(), &np, &pb,
                         skipped.data(), &ns));
  plan.resize(np);
  skipped.resize(ns);
  return PrefetchPlan{std::move(plan), pb, std::move(skipped)};
}

namespace detail {
inline TransferReport to_report(const laivg_transfer_report& rep, std::vector<uint32_t> moved) {
  moved.resize(rep.n_transferred);
  return TransferReport{rep.t_p, std::move(moved), rep.bytes, rep.overshoot_s};
}
} // namespace detail

/// tiered.hpp:104-107. kDevice: the copies run on a copy stream while a
/// generation-window kernel of overlap_window_s occupies the GPU.
inline TransferReport execute_prefetch(TieredStore& store, const PrefetchPlan& plan,
                                       const TransferChannel& chan, double overlap_window_s,
                                       const IvfIndex& ix, const EmbeddingMatrix& db) {
  (void)ix;
  (void)db;
  std::vector<uint32_t> moved(plan.clusters.size() + 1);
  const laivg_channel ch{chan.bandwidth_bytes_per_s, channel_mode(chan.mode)};
  laivg_transfer_report rep{};
  ck(laivg_execute_prefetch(store.ctx(), plan.clusters.data(), uint32_t(plan.clusters.size()),
                            &ch, overlap_window_s, moved.data(), &rep));
  return detail::to_report(rep, std::move(moved));
}

/// tiered.hpp:111-116
inline TransferReport incremental_prefetch(TieredStore& store, const IvfIndex& ix,
                                           std::span<const float> q_round, uint64_t budget_bytes,
                                           const TransferChannel& chan, const EmbeddingMatrix& db,
                                           double overlap_window_s = 0.0) {
  (void)ix;
  (void)db;
  detail::check_dim(store, q_round);
  std::vector<uint32_t> moved(store.index().num_clusters() + 1);
  const laivg_channel ch{chan.bandwidth_bytes_per_s, channel_mode(chan.mode)};
  laivg_transfer_report rep{};
  ck(laivg_incremental_prefetch(store.ctx(), q_round.data(), budget_bytes, &ch, overlap_window_s,
                                moved.data(), &rep));
  return detail::to_report(rep, std::move(moved));
}

/// The prefetch loop of serve_microbatch (pipeline.cpp:357-371) as one call:
/// one coarse pass over the batch's predictor embeddings, query i planned
/// against the store holding plans 0..i-1 with min(budgets[i], free), ONE
/// generation window for all copies (kDevice only). nplan (optional) gets
/// each query's planned count.
inline TransferReport prefetch_batch(TieredStore& store, const EmbeddingMatrix& q_in,
                                     const std::vector<uint64_t>& budgets,
                                     const TransferChannel& chan, double overlap_window_s,
                                     std::vector<uint32_t>* nplan = nullptr) {
  const uint32_t nq = uint32_t(q_in.count());
  if (budgets.size() != nq) throw std::invalid_argument("one budget per query");
  std::vector<uint32_t> moved(store.index().num_clusters() + 1), np(nq + 1);
  const laivg_channel ch{chan.bandwidth_bytes_per_s, LAIVG_CHAN_DEVICE};
  laivg_transfer_report rep{};
  ck(laivg_prefetch_batch(store.ctx(), q_in.data().data(), nq, budgets.data(), &ch,
                          overlap_window_s, moved.data(), np.data(), &rep));
  if (nplan) nplan->assign(np.begin(), np.begin() + nq);
  return detail::to_report(rep, std::move(moved));
}

namespace detail {
inline HybridTiming timing(const laivg_hybrid_timing& t, const CostModel& cost) {
  (void)cost;
  return HybridTiming{t.t_g, t.t_c, t.t_2};
}
} // namespace detail

/// tiered.hpp:121-124; HybridTiming carries measured times (GPU events /
/// host wall clock).
inline std::pair<HybridResult, HybridTiming> hybrid_search(const IvfIndex& ix,
                                                           const EmbeddingMatrix& db,
                                                           const TieredStore& store,
                                                           std::span<const float> q_out, int L,
                                                           int k, const CostModel& cost) {
  (void)ix;
  (void)db;
  detail::check_dim(store, q_out);
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  cost.validate();
  const uint32_t nc = store.index().num_clusters();
  std::vector<uint64_t> ids(k);
  std::vector<float> sc(k);
  std::vector<uint32_t> fast(nc + 1), slow(nc + 1);
  uint32_t n = 0, nf = 0, ns = 0;
  double hit = 0;
  laivg_hybrid_timing t{};
  const laivg_cost_model cm{cost.bandwidth_bytes_per_s, cost.t_cc, cost.t_gc,
                            cost.parallel_slots};
  ck(laivg_hybrid_search(store.ctx(), q_out.data(), L, k, &cm, ids.data(), sc.data(), &n,
                         fast.data(), &nf, slow.data(), &ns, &hit, &t));
  HybridResult r;
  r.topk = detail::to_topk(k, ids.data(), sc.data(), n);
  r.fast_clusters.assign(fast.begin(), fast.begin() + nf);
  r.slow_clusters.assign(slow.begin(), slow.begin() + ns);
  r.hit_rate = hit;
  return {std::move(r), detail::timing(t, cost)};
}

/// The retrieval loop of serve_microbatch (pipeline.cpp:391-428) as one
/// device pass per max_batch queries; per query equal to hybrid_search.
inline std::vector<TopK> hybrid_search_batch(const IvfIndex& ix, const EmbeddingMatrix& db,
                                             const TieredStore& store,
                                             const EmbeddingMatrix& queries, int L, int k,
                                             const CostModel& cost, HybridTiming* timing = nullptr) {
  (void)ix;
  (void)db;
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  const uint32_t nq = uint32_t(queries.count());
  std::vector<uint64_t> ids(size_t(nq) * k + 1);
  std::vector<float> sc(size_t(nq) * k + 1);
  std::vector<uint32_t> cnt(nq + 1);
  const laivg_cost_model cm{cost.bandwidth_bytes_per_s, cost.t_cc, cost.t_gc,
                            cost.parallel_slots};
  laivg_hybrid_timing t{};
  if (nq) {
    ck(laivg_hybrid_search_batch(store.ctx(), queries.data().data(), nq, L, k, &cm, ids.data(),
                                 sc.data(), cnt.data(), nullptr, &t));
  }
  if (timing) *timing = detail::timing(t, cost);
  std::vector<TopK> out;
  for (uint32_t q = 0; q < nq; ++q) {
    out.push_back(detail::to_topk(k, ids.data() + size_t(q) * k, sc.data() + size_t(q) * k, cnt[q]));
  }
  return out;
}

/// tiered.hpp:129-130
inline double coverage(const IvfIndex& ix, std::span<const float> q_in,
                       std::span<const float> q_out, int L) {
  auto& s = detail::store_for(&ix, "coverage");
  detail::check_dim(s, q_in);
  detail::check_dim(s, q_out);
  double out = 0;
  ck(laivg_coverage(s.ctx(), q_in.data(), q_out.data(), L, &out));
  return out;
}

// ---- sched.hpp --------------------------------------------------------------
namespace detail {
inline std::vector<MicroBatch> from_csr(const std::vector<uint64_t>& order,
                                        const std::vector<uint64_t>& off, uint32_t nb) {
  std::vector<MicroBatch> out(nb);
  for (uint32_t b = 0; b < nb; ++b) {
    out[b].queries.assign(order.begin() + off[b], order.begin() + off[b + 1]);
  }
  return out;
}
inline void to_csr(const std::vector<MicroBatch>& batches, std::vector<uint64_t>& off,
                   std::vector<uint64_t>& mem) {
  off.assign(1, 0);
  mem.clear();
  for (const auto& b : batches) {
    for (size_t q : b.queries) mem.push_back(q);
    off.push_back(mem.size());
  }
  if (mem.empty()) mem.push_back(0);
}
inline std::vector<uint8_t> resident_matrix(const std::vector<WorkerState>& workers, uint32_t nc) {
  std::vector<uint8_t> r(size_t(workers.size()) * nc + 1, 0);
  for (size_t w = 0; w < workers.size(); ++w) {
    for (uint32_t c : workers[w].resident_clusters) {
      if (c < nc) r[w * nc + c] = 1;
    }
  }
  return r;
}
} // namespace detail

/// sched.hpp:31-32 (the library's threaded host scheduler; the GPU one is
/// laivg_group_microbatches_gpu)
inline std::vector<MicroBatch> group_microbatches(const EmbeddingMatrix& queries, size_t m) {
  const uint64_t n = queries.count();
  std::vector<uint64_t> order(n + 1), off(n + 2);
  uint32_t nb = 0;
  ck(laivg_group_microbatches(queries.data().data(), n, queries.dim(), m, order.data(),
                              off.data(), &nb));
  return detail::from_csr(order, off, nb);
}

/// sched.hpp:36
inline std::vector<MicroBatch> chunk_microbatches(size_t n, size_t m) {
  std::vector<uint64_t> order(n + 1), off(n + 2);
  uint32_t nb = 0;
  ck(laivg_chunk_microbatches(n, m, order.data(), off.data(), &nb));
  return detail::from_csr(order, off, nb);
}

/// sched.hpp:42-45: probe unions from the GPU coarse quantizer of the
/// index's store.
inline std::vector<uint32_t> assign_cache_aware(const std::vector<MicroBatch>& batches,
                                                const std::vector<WorkerState>& workers,
                                                const IvfIndex& ix,
                                                const EmbeddingMatrix& queries, int L) {
  auto& s = detail::store_for(&ix, "assign_cache_aware");
  std::vector<uint64_t> off, mem;
  detail::to_csr(batches, off, mem);
  const auto res = detail::resident_matrix(workers, s.index().num_clusters());
  std::vector<uint32_t> out(batches.size() + 1);
  ck(laivg_assign_cache_aware(s.ctx(), off.data(), mem.data(), uint32_t(batches.size()),
                              res.data(), uint32_t(workers.size()), queries.data().data(),
                              queries.count(), L, out.data()));
  out.resize(batches.size());
  return out;
}

/// sched.hpp:48
inline std::vector<uint32_t> assign_round_robin(size_t n_batches, size_t n_workers) {
  std::vector<uint32_t> out(n_batches + 1);
  ck(laivg_assign_round_robin(n_batches, n_workers, out.data()));
  out.resize(n_batches);
  return out;
}

/// sched.hpp:51-55
inline uint64_t assignment_overlap(const std::vector<MicroBatch>& batches,
                                   const std::vector<WorkerState>& workers,
                                   const std::vector<uint32_t>& assignment, const IvfIndex& ix,
                                   const EmbeddingMatrix& queries, int L) {
  auto& s = detail::store_for(&ix, "assignment_overlap");
  std::vector<uint64_t> off, mem;
  detail::to_csr(batches, off, mem);
  const auto res = detail::resident_matrix(workers, s.index().num_clusters());
  uint64_t out = 0;
  ck(laivg_assignment_overlap(s.ctx(), off.data(), mem.data(), uint32_t(batches.size()),
                              res.data(), uint32_t(workers.size()), assignment.data(),
                              queries.data().data(), queries.count(), L, &out));
  return out;
}

/// sched.hpp:59-60
inline std::vector<uint64_t> split_budget(uint64_t total_budget_bytes, const MicroBatch& batch) {
  std::vector<uint64_t> b(batch.queries.begin(), batch.queries.end()), out(b.size() + 1);
  ck(laivg_split_budget(total_budget_bytes, b.data(), b.size(), out.data()));
  out.resize(b.size());
  return out;
}

// ---- cache.hpp --------------------------------------------------------------
/// cache.hpp:28-56 over the GPU store.
class HotnessTable {
 public:
  explicit HotnessTable(CacheParams params = {}) : params_(params) {
    params_.validate();
    ck(laivg_hotness_create(params_.h_init, params_.h_inc, params_.decay, params_.cache_fraction,
                            &h_));
  }
  ~HotnessTable() { laivg_hotness_destroy(h_); }
  HotnessTable(const HotnessTable&) = delete;
  HotnessTable& operator=(const HotnessTable&) = delete;

  const CacheParams& params() const { return params_; }
  void on_fetch(uint32_t cluster) { ck(laivg_hotness_on_fetch(h_, cluster)); }
  void end_of_round(const std::unordered_set<uint32_t>& used) {
    std::vector<uint32_t> u(used.begin(), used.end());
    ck(laivg_hotness_end_of_round(h_, u.data(), uint32_t(u.size())));
  }
  std::vector<uint32_t> evict_to_fraction(TieredStore& store) {
    std::vector<uint32_t> ev(store.resident_count() + 1);
    uint32_t n = 0;
    ck(laivg_hotness_evict_to_fraction(h_, store.ctx(), ev.data(), &n));
    ev.resize(n);
    return ev;
  }
  void forget(uint32_t cluster) { ck(laivg_hotness_forget(h_, cluster)); }
  void clear() { ck(laivg_hotness_clear(h_)); }
  bool tracked(uint32_t cluster) const { return laivg_hotness_get(h_, cluster) >= 0.0f; }
  float hotness(uint32_t cluster) const {
    const float h = laivg_hotness_get(h_, cluster);
    if (h < 0.0f) throw std::out_of_range("cluster not tracked");
    return h;
  }

 private:
  CacheParams params_;
  laivg_hotness* h_ = nullptr;
};

} // namespace laiv::gpu
