// laiv_gpu_shim.hpp — the C++ shim a laiv maintainer adds to run the
// reference's hot path (proj/core, namespace laiv) on a B200 through the C ABI
// of liblaivg.so (include/laivg.h). The laiv:: signatures stay; the index and
// datastore are bound once, each GPU with its cluster cache once.
//
// Header-only; needs the reference headers (laiv/*.hpp) and include/laivg.h.
// Errors come back as the reference's exception classes.
#pragma once

#include <laiv/budget.hpp>
#include <laiv/ivf.hpp>
#include <laiv/tiered.hpp>
#include <laiv/vectorstore.hpp>

#include <span>
#include <stdexcept>
#include <string>
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

// One-time binding of the reference's IvfIndex + EmbeddingMatrix: rows are
// gathered in list order (what load_index produces, ivf.cpp:437-455) into the
// library's pinned list-major store; `device` + `capacity_bytes` make the
// cluster cache (TieredStore) of one GPU.
class Bound {
 public:
  Bound(const IvfIndex& ix, const EmbeddingMatrix& db, uint64_t capacity_bytes, int device = 0,
        uint32_t max_batch = 0) {
    const uint32_t d = ix.dim(), nc = ix.num_clusters();
    std::vector<uint64_t> off(nc + 1, 0), ids;
    for (uint32_t c = 0; c < nc; ++c) off[c + 1] = off[c] + ix.list(c).size();
    std::vector<float> vecs(off[nc] * d);
    ids.reserve(off[nc]);
    for (uint32_t c = 0; c < nc; ++c) {
      for (size_t i = 0; i < ix.list(c).size(); ++i) {
        const uint64_t id = ix.list(c)[i];
        const auto r = db.row_of(id);
        if (!r) throw std::runtime_error("id " + std::to_string(id) + " missing from datastore");
        const auto row = db.row(*r);
        std::copy(row.begin(), row.end(), vecs.begin() + (off[c] + i) * d);
        ids.push_back(id);
      }
    }
    ck(laivg_index_create(ix.centroids().data().data(), nc, d, int(ix.metric()), vecs.data(),
                          ids.data(), off.data(), 0, &ix_));
    open_ctx(capacity_bytes, device, max_batch);
  }
  // Straight from a LAIX file (what load_index reads, ivf.hpp:98), without
  // materialising the reference's EmbeddingMatrix: the library reads the
  // lists into its pinned store in parallel (laivg_index_load).
  Bound(const std::string& laix_path, uint64_t capacity_bytes, int device = 0,
        uint32_t max_batch = 0, uint32_t threads = 0) {
    ck(laivg_index_load(laix_path.c_str(), threads, &ix_));
    open_ctx(capacity_bytes, device, max_batch);
  }
  ~Bound() {
    laivg_ctx_destroy(ctx_);
    laivg_index_destroy(ix_);
  }
  Bound(const Bound&) = delete;
  Bound& operator=(const Bound&) = delete;

  // save_index (ivf.hpp:96) of the bound store
  void save(const std::string& path, uint32_t threads = 0) const {
    ck(laivg_index_save(ix_, path.c_str(), threads));
  }

  laivg_ctx* ctx() const { return ctx_; }
  uint32_t dim() const { return d_; }
  uint32_t num_clusters() const { return nc_; }

  // TieredStore view of the GPU cache (tiered.hpp:22-56)
  void insert(uint32_t c, Residency tag = Residency::Prefetched) {
    ck(laivg_store_insert(ctx_, c, int(tag)));
  }
  uint64_t evict(uint32_t c) {
    uint64_t b = 0;
    ck(laivg_store_evict(ctx_, c, &b));
    return b;
  }
  void clear() { ck(laivg_store_clear(ctx_)); }
  uint64_t free_bytes() const { return laivg_store_free_bytes(ctx_); }

 private:
  void open_ctx(uint64_t capacity_bytes, int device, uint32_t max_batch) {
    laivg_opts o;
    laivg_opts_default(&o);
    o.device = device;
    o.capacity_bytes = capacity_bytes;
    o.max_batch = max_batch;
    const int rc = laivg_ctx_create(ix_, &o, &ctx_);
    if (rc != LAIVG_OK) {
      laivg_index_destroy(ix_);
      raise(rc);
    }
    d_ = laivg_index_dim(ix_);
    nc_ = laivg_index_num_clusters(ix_);
  }

  laivg_index* ix_ = nullptr;
  laivg_ctx* ctx_ = nullptr;
  uint32_t d_ = 0, nc_ = 0;
};

inline TopK to_topk(int k, const uint64_t* ids, const float* sc, uint32_t n) {
  TopK t{k, {}};
  for (uint32_t i = 0; i < n; ++i) t.entries.push_back({ids[i], sc[i]});
  return t;
}

// ivf.hpp:72-73
inline std::vector<uint32_t> coarse_probe(Bound& b, std::span<const float> q, int L) {
  std::vector<uint32_t> out(b.num_clusters());
  uint32_t lp = 0;
  ck(laivg_coarse_probe(b.ctx(), q.data(), 1, L, out.data(), &lp));
  out.resize(lp);
  return out;
}

// ivf.hpp:90-91
inline TopK ivf_search(Bound& b, std::span<const float> q, int L, int k) {
  std::vector<uint64_t> ids(k > 0 ? k : 1);
  std::vector<float> sc(k > 0 ? k : 1);
  uint32_t n = 0;
  ck(laivg_ivf_search(b.ctx(), q.data(), 1, L, k, ids.data(), sc.data(), &n));
  return to_topk(k, ids.data(), sc.data(), n);
}

// ivf_search over a batch (one device pass per max_batch queries)
inline std::vector<TopK> ivf_search_batch(Bound& b, const EmbeddingMatrix& queries, int L,
                                          int k) {
  const uint32_t nq = uint32_t(queries.count());
  std::vector<uint64_t> ids(size_t(nq) * k);
  std::vector<float> sc(size_t(nq) * k);
  std::vector<uint32_t> cnt(nq);
  ck(laivg_ivf_search(b.ctx(), queries.data().data(), nq, L, k, ids.data(), sc.data(),
                      cnt.data()));
  std::vector<TopK> out;
  for (uint32_t q = 0; q < nq; ++q) {
    out.push_back(to_topk(k, ids.data() + size_t(q) * k, sc.data() + size_t(q) * k, cnt[q]));
  }
  return out;
}

// tiered.hpp:100-101 (against the GPU cache's residency)
inline PrefetchPlan plan_prefetch(Bound& b, std::span<const float> q_in, uint64_t budget) {
  std::vector<uint32_t> plan(b.num_clusters()), skipped(b.num_clusters());
  uint32_t np = 0, ns = 0;
  uint64_t pb = 0;
  ck(laivg_plan_prefetch(b.ctx(), q_in.data(), budget, plan.data(), &np, &pb, skipped.data(),
                         &ns));
  plan.resize(np);
  skipped.resize(ns);
  return PrefetchPlan{std::move(plan), pb, std::move(skipped)};
}

// tiered.hpp:107-110; the device channel streams the lists on a copy stream
// while a generation-window kernel of window_s runs
inline TransferReport execute_prefetch(Bound& b, const PrefetchPlan& plan,
                                       const TransferChannel& chan, double window_s) {
  std::vector<uint32_t> moved(plan.clusters.size() + 1);
  const laivg_channel ch{chan.bandwidth_bytes_per_s, LAIVG_CHAN_DEVICE};
  laivg_transfer_report rep{};
  ck(laivg_execute_prefetch(b.ctx(), plan.clusters.data(), uint32_t(plan.clusters.size()), &ch,
                            window_s, moved.data(), &rep));
  moved.resize(rep.n_transferred);
  return TransferReport{rep.t_p, std::move(moved), rep.bytes, rep.overshoot_s};
}

// tiered.hpp:125-128; HybridTiming carries measured times
inline std::pair<HybridResult, HybridTiming> hybrid_search(Bound& b, std::span<const float> q_out,
                                                           int L, int k, const CostModel& cost) {
  const uint32_t nc = b.num_clusters();
  std::vector<uint64_t> ids(k > 0 ? k : 1);
  std::vector<float> sc(k > 0 ? k : 1);
  std::vector<uint32_t> fast(nc), slow(nc);
  uint32_t n = 0, nf = 0, ns = 0;
  double hit = 0;
  laivg_hybrid_timing t{};
  const laivg_cost_model cm{cost.bandwidth_bytes_per_s, cost.t_cc, cost.t_gc,
                            cost.parallel_slots};
  ck(laivg_hybrid_search(b.ctx(), q_out.data(), L, k, &cm, ids.data(), sc.data(), &n,
                         fast.data(), &nf, slow.data(), &ns, &hit, &t));
  HybridResult r;
  r.topk = to_topk(k, ids.data(), sc.data(), n);
  r.fast_clusters.assign(fast.begin(), fast.begin() + nf);
  r.slow_clusters.assign(slow.begin(), slow.begin() + ns);
  r.hit_rate = hit;
  return {std::move(r), HybridTiming{t.t_g, t.t_c, t.t_2}};
}

} // namespace laiv::gpu
