// ref_shim.cpp — extern "C" wrapper around the UNMODIFIED reference `laiv`
// core, compiled from /root/reference/proj/core/src/*.cpp by oracle/Makefile
// into oracle/_ref/libref.so (git-ignored; travels to the GPU box prebuilt).
//
// TEST INFRASTRUCTURE ONLY: used to make golden fixtures (tests/golden/), to
// cross-check the C restatement (oracle.c), and as the CPU baseline arm of
// bench.py (`--impl reference`). Never linked into the product.
//
// Every entry point returns >= 0 on success, -1 on a reference exception
// (message via ref_last_error()).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <set>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "laiv/cache.hpp"
#include "laiv/ivf.hpp"
#include "laiv/rng.hpp"
#include "laiv/sched.hpp"
#include "laiv/tiered.hpp"
#include "laiv/vectorstore.hpp"

namespace {
thread_local std::string g_err;

struct RefIndex {
  laiv::IvfIndex ix;
  laiv::EmbeddingMatrix db;
};

struct RefCache {
  laiv::TieredStore store;
  laiv::HotnessTable hot;
  RefCache(uint64_t cap, laiv::CacheParams p) : store(cap), hot(p) {}
};

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

laiv::TieredStore make_store(const RefIndex* h, const uint8_t* resident) {
  laiv::TieredStore store(1ull << 62);
  if (resident) {
    for (uint32_t c = 0; c < h->ix.num_clusters(); ++c) {
      if (resident[c]) {
        store.insert(c, h->ix.cluster_bytes(c), laiv::Residency::Prefetched);
      }
    }
  }
  return store;
}

int write_topk(const laiv::TopK& t, uint64_t* ids, float* scores) {
  for (size_t i = 0; i < t.entries.size(); ++i) {
    ids[i] = t.entries[i].id;
    scores[i] = t.entries[i].score;
  }
  return static_cast<int>(t.entries.size());
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Rng stream check (rng.hpp): n gaussians from Rng(seed).
void ref_rng_gaussians(uint64_t seed, uint64_t n, double* out) {
  laiv::Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.gaussian();
}
uint64_t ref_derive_seed(uint64_t seed, const char* label) {
  return laiv::derive_seed(seed, label);
}

// Builds IvfIndex + EmbeddingMatrix from a list-major store, appending rows
// in list order exactly as load_index does (ivf.cpp:437-455).
void* ref_index_create(const float* centroids, uint32_t nc, uint32_t d,
                       int metric, const float* vecs, const uint64_t* ids,
                       const uint64_t* list_off) {
  try {
    laiv::EmbeddingMatrix cen(d);
    cen.reserve(nc);
    for (uint32_t c = 0; c < nc; ++c) {
      cen.append(c, std::span<const float>(centroids + uint64_t(c) * d, d));
    }
    laiv::EmbeddingMatrix db(d);
    db.reserve(list_off[nc]);
    std::vector<std::vector<uint64_t>> lists(nc);
    for (uint32_t c = 0; c < nc; ++c) {
      for (uint64_t r = list_off[c]; r < list_off[c + 1]; ++r) {
        lists[c].push_back(ids[r]);
        db.append(ids[r], std::span<const float>(vecs + r * d, d));
      }
    }
    auto* h = new RefIndex{
        laiv::IvfIndex(std::move(cen), std::move(lists),
                       static_cast<laiv::Metric>(metric)),
        std::move(db)};
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_index_destroy(void* h) { delete static_cast<RefIndex*>(h); }

uint64_t ref_cluster_bytes(void* hv, uint32_t c) {
  return static_cast<RefIndex*>(hv)->ix.cluster_bytes(c);
}

int ref_rank_clusters(void* hv, const float* q, uint32_t* order) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    auto o = laiv::rank_clusters(h->ix, {q, h->ix.dim()});
    std::memcpy(order, o.data(), o.size() * sizeof(uint32_t));
    return static_cast<int>(o.size());
  });
}

int ref_coarse_probe(void* hv, const float* q, int L, uint32_t* out) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    auto o = laiv::coarse_probe(h->ix, {q, h->ix.dim()}, L);
    std::memcpy(out, o.data(), o.size() * sizeof(uint32_t));
    return static_cast<int>(o.size());
  });
}

int ref_search_clusters(void* hv, const float* q, const uint32_t* clusters,
                        uint32_t n, int k, uint64_t* ids, float* scores) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    auto t = laiv::search_clusters(h->ix, h->db, {q, h->ix.dim()},
                                   {clusters, n}, k);
    return write_topk(t, ids, scores);
  });
}

int ref_ivf_search(void* hv, const float* q, int L, int k, uint64_t* ids,
                   float* scores) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    return write_topk(laiv::ivf_search(h->ix, h->db, {q, h->ix.dim()}, L, k),
                      ids, scores);
  });
}

int ref_exact_search(void* hv, const float* q, int k, uint64_t* ids,
                     float* scores) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    return write_topk(
        laiv::exact_search(h->db, {q, h->ix.dim()}, k, h->ix.metric()), ids,
        scores);
  });
}

// score_clusters: the raw candidate list (returns its length; -1 on a throw).
int64_t ref_score_clusters(void* hv, const float* q, const uint32_t* clusters, uint32_t n,
                           uint64_t cap, uint64_t* ids, float* scores) {
  auto* h = static_cast<RefIndex*>(hv);
  try {
    auto v = laiv::score_clusters(h->ix, h->db, {q, h->ix.dim()}, {clusters, n});
    if (v.size() > cap) {
      g_err = "capacity";
      return -1;
    }
    for (size_t i = 0; i < v.size(); ++i) {
      ids[i] = v[i].id;
      scores[i] = v[i].score;
    }
    return static_cast<int64_t>(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// pairwise_l2 over two row-major matrices (ids 0..n-1).
int ref_pairwise_l2(const float* a, uint64_t na, const float* b, uint64_t nb, uint32_t d,
                    float* out) {
  return guard([&] {
    laiv::EmbeddingMatrix A(d), B(d);
    for (uint64_t i = 0; i < na; ++i) A.append(i, {a + i * d, d});
    for (uint64_t i = 0; i < nb; ++i) B.append(i, {b + i * d, d});
    auto v = laiv::pairwise_l2(A, B);
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return 0;
  });
}

// hybrid_search with a store holding exactly the clusters marked resident.
int ref_hybrid_search(void* hv, const uint8_t* resident, const float* q, int L,
                      int k, uint64_t* ids, float* scores, uint32_t* fast,
                      uint32_t* nfast, uint32_t* slow, uint32_t* nslow,
                      double* hit_rate) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    const auto store = make_store(h, resident);
    auto [res, timing] = laiv::hybrid_search(h->ix, h->db, store,
                                             {q, h->ix.dim()}, L, k, {});
    (void)timing;
    std::memcpy(fast, res.fast_clusters.data(),
                res.fast_clusters.size() * sizeof(uint32_t));
    std::memcpy(slow, res.slow_clusters.data(),
                res.slow_clusters.size() * sizeof(uint32_t));
    *nfast = static_cast<uint32_t>(res.fast_clusters.size());
    *nslow = static_cast<uint32_t>(res.slow_clusters.size());
    *hit_rate = res.hit_rate;
    return write_topk(res.topk, ids, scores);
  });
}

int ref_plan_prefetch(void* hv, const float* q, uint64_t budget,
                      const uint8_t* resident, uint32_t* plan, uint32_t* nplan,
                      uint64_t* planned_bytes, uint32_t* skipped,
                      uint32_t* nskipped) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    const auto store = make_store(h, resident);
    auto p = laiv::plan_prefetch(h->ix, {q, h->ix.dim()}, budget, store);
    std::memcpy(plan, p.clusters.data(), p.clusters.size() * sizeof(uint32_t));
    std::memcpy(skipped, p.skipped.data(), p.skipped.size() * sizeof(uint32_t));
    *nplan = static_cast<uint32_t>(p.clusters.size());
    *nskipped = static_cast<uint32_t>(p.skipped.size());
    *planned_bytes = p.planned_bytes;
    return 0;
  });
}

double ref_coverage(void* hv, const float* q_in, const float* q_out, int L) {
  auto* h = static_cast<RefIndex*>(hv);
  return laiv::coverage(h->ix, {q_in, h->ix.dim()}, {q_out, h->ix.dim()}, L);
}

// build_index (k-means++ / Lloyd) on a row-major db with ids 0..n-1. Writes
// centroids[nc*d], list_off[nc+1] and members[n] (ids in member order).
int ref_build_index(const float* db, uint64_t n, uint32_t d, uint32_t nc,
                    uint64_t seed, int max_iters, int spherical, int metric,
                    float* centroids, uint64_t* list_off, uint64_t* members) {
  return guard([&] {
    laiv::EmbeddingMatrix m(d);
    m.reserve(n);
    for (uint64_t i = 0; i < n; ++i) m.append(i, {db + i * d, d});
    laiv::IvfBuildOptions o;
    o.seed = seed;
    o.max_iters = max_iters;
    o.spherical = spherical != 0;
    auto ix = laiv::build_index(m, nc, o, static_cast<laiv::Metric>(metric));
    uint64_t w = 0;
    for (uint32_t c = 0; c < nc; ++c) {
      auto row = ix.centroids().row(c);
      std::memcpy(centroids + uint64_t(c) * d, row.data(), d * sizeof(float));
      list_off[c] = w;
      for (uint64_t id : ix.list(c)) members[w++] = id;
    }
    list_off[nc] = w;
    return 0;
  });
}

int ref_group_microbatches(const float* q, uint64_t n, uint32_t d, uint64_t m,
                           uint64_t* order, uint64_t* batch_off) {
  return guard([&] {
    laiv::EmbeddingMatrix qs(d);
    for (uint64_t i = 0; i < n; ++i) qs.append(i, {q + i * d, d});
    auto b = laiv::group_microbatches(qs, m);
    uint64_t w = 0;
    batch_off[0] = 0;
    for (size_t i = 0; i < b.size(); ++i) {
      for (size_t x : b[i].queries) order[w++] = x;
      batch_off[i + 1] = w;
    }
    return static_cast<int>(b.size());
  });
}

namespace {
std::vector<laiv::MicroBatch> csr_batches(const uint64_t* off,
                                          const uint64_t* mem, uint32_t nb) {
  std::vector<laiv::MicroBatch> b(nb);
  for (uint32_t i = 0; i < nb; ++i) {
    for (uint64_t j = off[i]; j < off[i + 1]; ++j) b[i].queries.push_back(mem[j]);
  }
  return b;
}
std::vector<laiv::WorkerState> workers_of(const uint8_t* res, uint32_t nw,
                                          uint32_t nc) {
  std::vector<laiv::WorkerState> w(nw);
  for (uint32_t i = 0; i < nw; ++i) {
    w[i].worker_id = i;
    for (uint32_t c = 0; c < nc; ++c) {
      if (res[uint64_t(i) * nc + c]) w[i].resident_clusters.insert(c);
    }
  }
  return w;
}
laiv::EmbeddingMatrix query_matrix(const float* q, uint64_t n, uint32_t d) {
  laiv::EmbeddingMatrix qs(d);
  for (uint64_t i = 0; i < n; ++i) qs.append(i, {q + i * d, d});
  return qs;
}
} // namespace

int ref_assign_cache_aware(void* hv, const uint64_t* off, const uint64_t* mem,
                           uint32_t nb, const uint8_t* resident, uint32_t nw,
                           const float* queries, uint64_t nq, int L,
                           uint32_t* assignment) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    auto a = laiv::assign_cache_aware(csr_batches(off, mem, nb),
                                      workers_of(resident, nw,
                                                 h->ix.num_clusters()),
                                      h->ix, query_matrix(queries, nq, h->ix.dim()),
                                      L);
    std::memcpy(assignment, a.data(), a.size() * sizeof(uint32_t));
    return 0;
  });
}

int64_t ref_assignment_overlap(void* hv, const uint64_t* off,
                               const uint64_t* mem, uint32_t nb,
                               const uint8_t* resident, uint32_t nw,
                               const uint32_t* assignment,
                               const float* queries, uint64_t nq, int L) {
  auto* h = static_cast<RefIndex*>(hv);
  try {
    std::vector<uint32_t> a(assignment, assignment + nb);
    return static_cast<int64_t>(laiv::assignment_overlap(
        csr_batches(off, mem, nb), workers_of(resident, nw, h->ix.num_clusters()),
        a, h->ix, query_matrix(queries, nq, h->ix.dim()), L));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_split_budget(uint64_t total, const uint64_t* batch, uint64_t n,
                     uint64_t* out) {
  return guard([&] {
    laiv::MicroBatch b;
    b.queries.assign(batch, batch + n);
    auto s = laiv::split_budget(total, b);
    std::memcpy(out, s.data(), s.size() * sizeof(uint64_t));
    return 0;
  });
}

// --- TieredStore + HotnessTable scripting (cache.cpp / tiered.cpp) ---------
void* ref_cache_create(uint64_t capacity, float h_init, float h_inc,
                       float decay, double fraction) {
  try {
    return new RefCache(capacity, laiv::CacheParams{h_init, h_inc, decay, fraction});
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_cache_destroy(void* c) { delete static_cast<RefCache*>(c); }
int ref_cache_insert(void* cv, uint32_t c, uint64_t bytes, int tag) {
  auto* x = static_cast<RefCache*>(cv);
  return guard([&] {
    x->store.insert(c, bytes, static_cast<laiv::Residency>(tag));
    return 0;
  });
}
void ref_cache_on_fetch(void* cv, uint32_t c) {
  static_cast<RefCache*>(cv)->hot.on_fetch(c);
}
void ref_cache_end_of_round(void* cv, const uint32_t* used, uint32_t n) {
  std::unordered_set<uint32_t> u(used, used + n);
  static_cast<RefCache*>(cv)->hot.end_of_round(u);
}
int ref_cache_evict_to_fraction(void* cv, uint32_t* evicted) {
  auto* x = static_cast<RefCache*>(cv);
  auto e = x->hot.evict_to_fraction(x->store);
  std::memcpy(evicted, e.data(), e.size() * sizeof(uint32_t));
  return static_cast<int>(e.size());
}
float ref_cache_hotness(void* cv, uint32_t c) {
  auto* x = static_cast<RefCache*>(cv);
  return x->hot.tracked(c) ? x->hot.hotness(c) : -1.0f;
}
uint64_t ref_cache_used(void* cv) { return static_cast<RefCache*>(cv)->store.used_bytes(); }
int ref_cache_contains(void* cv, uint32_t c) {
  return static_cast<RefCache*>(cv)->store.contains(c) ? 1 : 0;
}

// --- CPU baseline runner: the reference search, one query per thread -------
// mode 0 = ivf_search (ivf.cpp:345), 1 = hybrid_search with an empty store
// (tiered.cpp:148). Queries are claimed from a shared counter by `threads`
// host threads (ivf.hpp:25: concurrent searches are safe).
int ref_search_many(void* hv, int mode, const float* Q, uint64_t nq, int L,
                    int k, int threads, uint64_t* ids, float* scores,
                    double* latency_s) {
  auto* h = static_cast<RefIndex*>(hv);
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  const laiv::TieredStore empty(1ull << 62);
  auto work = [&] {
    for (;;) {
      const uint64_t i = next.fetch_add(1);
      if (i >= nq) return;
      try {
        const auto t0 = std::chrono::steady_clock::now();
        laiv::TopK t;
        const std::span<const float> q(Q + i * h->ix.dim(), h->ix.dim());
        if (mode == 0) {
          t = laiv::ivf_search(h->ix, h->db, q, L, k);
        } else {
          t = laiv::hybrid_search(h->ix, h->db, empty, q, L, k, {}).first.topk;
        }
        for (size_t j = 0; j < t.entries.size(); ++j) {
          ids[i * k + j] = t.entries[j].id;
          scores[i * k + j] = t.entries[j].score;
        }
        if (latency_s) {
          latency_s[i] = std::chrono::duration<double>(
                             std::chrono::steady_clock::now() - t0).count();
        }
      } catch (const std::exception& e) {
        failed = 1;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return failed ? -1 : 0;
}

// save_index (ivf.cpp:351-392) of an index built by ref_index_create.
int ref_save_index(void* hv, const char* path) {
  return guard([&] {
    const auto* h = static_cast<RefIndex*>(hv);
    laiv::save_index(path, h->ix, h->db);
    return 0;
  });
}

// load_index (ivf.cpp:394-458): 0 and a new handle in *out, or the class of
// the exception (1 runtime_error, 2 invalid_argument, 3 logic_error, 4 other)
// with its message in ref_last_error().
int ref_load_index(const char* path, void** out) {
  *out = nullptr;
  try {
    auto [ix, db] = laiv::load_index(path);
    *out = new RefIndex{std::move(ix), std::move(db)};
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// The list-major store of a loaded index: list_off[nc+1], ids[N], vecs[N*d]
// (any pointer may be NULL to skip it).
void ref_index_lists(void* hv, uint64_t* list_off, uint64_t* ids, float* vecs) {
  const auto* h = static_cast<RefIndex*>(hv);
  const uint32_t d = h->ix.dim();
  uint64_t r = 0;
  if (list_off) list_off[0] = 0;
  for (uint32_t c = 0; c < h->ix.num_clusters(); ++c) {
    for (uint64_t id : h->ix.list(c)) {
      if (ids) ids[r] = id;
      if (vecs) {
        const auto row = h->db.row(*h->db.row_of(id));
        std::memcpy(vecs + r * d, row.data(), d * sizeof(float));
      }
      ++r;
    }
    if (list_off) list_off[c + 1] = r;
  }
}

} // extern "C"
