// host.cpp — CPU side of the retrieval path (see host.hpp).
// Built with -ffp-contract=off: every fp64 add/mul rounds separately, as the
// reference's scalar loops do (vectorstore.cpp:93-108).
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include <immintrin.h>

namespace laivg {

// ==========================================================================
// ThreadPool
// ==========================================================================
ThreadPool::ThreadPool(unsigned n) {
  for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::loop(unsigned wid) {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(size_t, unsigned)>* job;
    size_t n;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      job = job_;
      n = n_;
      if (job == nullptr) continue; // woke after that job already finished
      ++active_;
    }
    for (size_t i; (i = next_.fetch_add(1)) < n;) (*job)(i, wid);
    {
      std::lock_guard<std::mutex> g(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
}

void ThreadPool::parallel_for(size_t n,
                              const std::function<void(size_t, unsigned)>& fn) {
  if (n == 0) return;
  if (workers_.empty() || n == 1) {
    for (size_t i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  {
    std::lock_guard<std::mutex> g(mu_);
    job_ = &fn;
    n_ = n;
    next_ = 0;
    ++gen_;
  }
  cv_.notify_all();
  for (size_t i; (i = next_.fetch_add(1)) < n;) fn(i, 0);
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return active_ == 0 && next_ >= n; });
  job_ = nullptr;
}

// ==========================================================================
// miss scan
// ==========================================================================
namespace {

// fp64 dot / squared L2 over fp32 inputs, 16 partial sums (vectorised).
__attribute__((target_clones("arch=sapphirerapids", "default")))
double dot_f64(const float* a, const float* b, uint32_t d) {
  double acc[16] = {0};
  uint32_t j = 0;
  for (; j + 16 <= d; j += 16) {
    for (int t = 0; t < 16; ++t) {
      acc[t] += static_cast<double>(a[j + t]) * static_cast<double>(b[j + t]);
    }
  }
  for (int t = 0; t < 8; ++t) acc[t] += acc[t + 8];
  for (int t = 0; t < 4; ++t) acc[t] += acc[t + 4];
  double s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  for (; j < d; ++j) s += static_cast<double>(a[j]) * static_cast<double>(b[j]);
  return s;
}

__attribute__((target_clones("arch=sapphirerapids", "default")))
double l2sq_f64(const float* a, const float* b, uint32_t d) {
  double acc[16] = {0};
  uint32_t j = 0;
  for (; j + 16 <= d; j += 16) {
    for (int t = 0; t < 16; ++t) {
      const double x = static_cast<double>(a[j + t]) - static_cast<double>(b[j + t]);
      acc[t] += x * x;
    }
  }
  for (int t = 0; t < 8; ++t) acc[t] += acc[t + 8];
  for (int t = 0; t < 4; ++t) acc[t] += acc[t + 4];
  double s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  for (; j < d; ++j) {
    const double x = static_cast<double>(a[j]) - static_cast<double>(b[j]);
    s += x * x;
  }
  return s;
}

// Sorted best-first list of at most k entries.
struct TopList {
  int metric;
  int k;
  std::vector<Scored> e;
  void push(const Scored& c) {
    if (static_cast<int>(e.size()) == k && !ranks_before(metric, c, e.back())) return;
    auto it = std::upper_bound(e.begin(), e.end(), c, [this](const Scored& a, const Scored& b) {
      return ranks_before(metric, a, b);
    });
    e.insert(it, c);
    if (static_cast<int>(e.size()) > k) e.pop_back();
  }
};


// Register-blocked host scoring of one fp32 row against G queries held in
// fp64 (converted once per batch): the row is read from memory once and
// every term is the reference's (vectorstore.cpp:93-108). IP uses FMA, which
// is exact here: the product of two fp32 values is exact in fp64, so
// fma(q, x, acc) == acc + q * x. L2 keeps the separately rounded sub/mul/add.
// Partial sums run over 4 lanes x 2 chains, reduced at the end (any order is
// within the parity rule; see the GPU scan).
template <int G, bool kIP>
__attribute__((target("avx2,fma"))) void score_rows_avx2(const float* x, const double* const* q,
                                                         uint32_t d, double* out) {
  __m256d a0[G], a1[G];
  for (int g = 0; g < G; ++g) {
    a0[g] = _mm256_setzero_pd();
    a1[g] = _mm256_setzero_pd();
  }
  uint32_t j = 0;
  for (; j + 8 <= d; j += 8) {
    const __m256d x0 = _mm256_cvtps_pd(_mm_loadu_ps(x + j));
    const __m256d x1 = _mm256_cvtps_pd(_mm_loadu_ps(x + j + 4));
    for (int g = 0; g < G; ++g) {
      const __m256d q0 = _mm256_loadu_pd(q[g] + j), q1 = _mm256_loadu_pd(q[g] + j + 4);
      if constexpr (kIP) {
        a0[g] = _mm256_fmadd_pd(q0, x0, a0[g]);
        a1[g] = _mm256_fmadd_pd(q1, x1, a1[g]);
      } else {
        const __m256d t0 = _mm256_sub_pd(q0, x0), t1 = _mm256_sub_pd(q1, x1);
        a0[g] = _mm256_add_pd(a0[g], _mm256_mul_pd(t0, t0));
        a1[g] = _mm256_add_pd(a1[g], _mm256_mul_pd(t1, t1));
      }
    }
  }
  for (int g = 0; g < G; ++g) {
    alignas(32) double l[4];
    _mm256_store_pd(l, _mm256_add_pd(a0[g], a1[g]));
    double sacc = (l[0] + l[1]) + (l[2] + l[3]);
    for (uint32_t t = j; t < d; ++t) {
      const double xv = static_cast<double>(x[t]);
      if constexpr (kIP) {
        sacc += q[g][t] * xv;
      } else {
        const double u = q[g][t] - xv;
        sacc += u * u;
      }
    }
    out[g] = sacc;
  }
}

template <int G, bool kIP>
__attribute__((target("avx512f"))) void score_rows_avx512(const float* x, const double* const* q,
                                                         uint32_t d, double* out) {
  __m512d a0[G], a1[G];
  for (int g = 0; g < G; ++g) {
    a0[g] = _mm512_setzero_pd();
    a1[g] = _mm512_setzero_pd();
  }
  uint32_t j = 0;
  for (; j + 16 <= d; j += 16) {
    const __m512d x0 = _mm512_cvtps_pd(_mm256_loadu_ps(x + j));
    const __m512d x1 = _mm512_cvtps_pd(_mm256_loadu_ps(x + j + 8));
    for (int g = 0; g < G; ++g) {
      const __m512d q0 = _mm512_loadu_pd(q[g] + j), q1 = _mm512_loadu_pd(q[g] + j + 8);
      if constexpr (kIP) {
        a0[g] = _mm512_fmadd_pd(q0, x0, a0[g]);
        a1[g] = _mm512_fmadd_pd(q1, x1, a1[g]);
      } else {
        const __m512d t0 = _mm512_sub_pd(q0, x0), t1 = _mm512_sub_pd(q1, x1);
        a0[g] = _mm512_add_pd(a0[g], _mm512_mul_pd(t0, t0));
        a1[g] = _mm512_add_pd(a1[g], _mm512_mul_pd(t1, t1));
      }
    }
  }
  for (int g = 0; g < G; ++g) {
    alignas(64) double l[8];
    _mm512_store_pd(l, _mm512_add_pd(a0[g], a1[g]));
    double sacc = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
    for (uint32_t t = j; t < d; ++t) {
      const double xv = static_cast<double>(x[t]);
      if constexpr (kIP) {
        sacc += q[g][t] * xv;
      } else {
        const double u = q[g][t] - xv;
        sacc += u * u;
      }
    }
    out[g] = sacc;
  }
}

bool host_has_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f");
  return ok;
}

bool host_has_avx2() {
  static const bool ok = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
  return ok;
}

template <bool kIP>
void score_row_blocked(const float* x, const double* const* q, uint32_t n, uint32_t d,
                       double* out) {
  uint32_t g = 0;
  if (host_has_avx512()) {
    for (; g + 4 <= n; g += 4) score_rows_avx512<4, kIP>(x, q + g, d, out + g);
    switch (n - g) {
      case 3: score_rows_avx512<3, kIP>(x, q + g, d, out + g); break;
      case 2: score_rows_avx512<2, kIP>(x, q + g, d, out + g); break;
      case 1: score_rows_avx512<1, kIP>(x, q + g, d, out + g); break;
      default: break;
    }
    return;
  }
  for (; g + 4 <= n; g += 4) score_rows_avx2<4, kIP>(x, q + g, d, out + g);
  switch (n - g) {
    case 3: score_rows_avx2<3, kIP>(x, q + g, d, out + g); break;
    case 2: score_rows_avx2<2, kIP>(x, q + g, d, out + g); break;
    case 1: score_rows_avx2<1, kIP>(x, q + g, d, out + g); break;
    default: break;
  }
}

} // namespace

std::vector<Scored> miss_scan(const Index& ix, const float* q,
                              const std::vector<uint32_t>& lists, int k,
                              ThreadPool& pool) {
  struct Task {
    uint64_t r0, r1;
  };
  std::vector<Task> tasks;
  for (uint32_t c : lists) {
    for (uint64_t r = ix.list_off[c]; r < ix.list_off[c + 1]; r += kMissChunkSingle) {
      tasks.push_back({r, std::min(r + kMissChunkSingle, ix.list_off[c + 1])});
    }
  }
  std::vector<TopList> per(pool.size(), TopList{ix.metric, k, {}});
  const uint32_t d = ix.d;
  const bool fast = host_has_avx2();
  std::vector<double> qd(fast ? d : 0);
  for (uint32_t j = 0; fast && j < d; ++j) qd[j] = q[j];
  const double* qp = qd.data();
  pool.parallel_for(tasks.size(), [&](size_t t, unsigned wid) {
    TopList& tl = per[wid];
    for (uint64_t r = tasks[t].r0; r < tasks[t].r1; ++r) {
      const float* x = ix.vecs + r * d;
      float s;
      if (fast) { // same per-query arithmetic as the batched miss scan
        double v;
        if (ix.metric == kMetricIP) {
          score_row_blocked<true>(x, &qp, 1, d, &v);
          s = static_cast<float>(v);
        } else {
          score_row_blocked<false>(x, &qp, 1, d, &v);
          s = static_cast<float>(std::sqrt(v));
        }
        tl.push({s, ix.ids[r]});
        continue;
      }
      if (ix.metric == kMetricIP) {
        s = static_cast<float>(dot_f64(q, x, d));
      } else {
        s = static_cast<float>(std::sqrt(l2sq_f64(q, x, d)));
      }
      tl.push({s, ix.ids[r]});
    }
  });
  TopList all{ix.metric, k, {}};
  for (auto& tl : per) {
    for (const auto& e : tl.e) all.push(e);
  }
  return std::move(all.e);
}

void score_lists(const Index& ix, const float* q,
                 const std::vector<std::pair<uint32_t, uint64_t>>& items, float* s_out,
                 uint64_t* id_out, ThreadPool& pool) {
  struct Task {
    uint64_t r0, r1, out;
  };
  std::vector<Task> tasks;
  for (const auto& [c, o] : items) {
    const uint64_t b = ix.list_off[c], e = ix.list_off[c + 1];
    for (uint64_t r = b; r < e; r += kMissChunk) {
      tasks.push_back({r, std::min(r + kMissChunk, e), o + (r - b)});
    }
  }
  const uint32_t d = ix.d;
  const bool fast = host_has_avx2();
  std::vector<double> qd(fast ? d : 0);
  for (uint32_t j = 0; fast && j < d; ++j) qd[j] = q[j];
  const double* qp = qd.data();
  pool.parallel_for(tasks.size(), [&](size_t t, unsigned) {
    uint64_t o = tasks[t].out;
    for (uint64_t r = tasks[t].r0; r < tasks[t].r1; ++r, ++o) {
      const float* x = ix.vecs + r * d;
      float sc;
      if (fast) { // the miss scan's arithmetic
        double v;
        if (ix.metric == kMetricIP) {
          score_row_blocked<true>(x, &qp, 1, d, &v);
          sc = static_cast<float>(v);
        } else {
          score_row_blocked<false>(x, &qp, 1, d, &v);
          sc = static_cast<float>(std::sqrt(v));
        }
      } else {
        sc = ix.metric == kMetricIP ? static_cast<float>(dot_f64(q, x, d))
                                    : static_cast<float>(std::sqrt(l2sq_f64(q, x, d)));
      }
      s_out[o] = sc;
      id_out[o] = ix.ids[r];
    }
  });
}

std::vector<std::vector<Scored>> miss_scan_batch(const Index& ix, const float* Q, uint32_t nq,
                                                 const std::vector<std::vector<uint32_t>>& slow,
                                                 int k, ThreadPool& pool) {
  // list-major: every missed list is streamed once per chunk and scored
  // against all queries that miss it
  std::map<uint32_t, std::vector<uint32_t>> by_list;
  for (uint32_t q = 0; q < nq; ++q) {
    for (uint32_t c : slow[q]) by_list[c].push_back(q);
  }
  struct Task {
    uint64_t r0, r1;
    const std::vector<uint32_t>* qs;
  };
  std::vector<Task> tasks;
  for (auto& [c, qs] : by_list) {
    for (uint64_t r = ix.list_off[c]; r < ix.list_off[c + 1]; r += kMissChunk) {
      tasks.push_back({r, std::min(r + kMissChunk, ix.list_off[c + 1]), &qs});
    }
  }
  const unsigned nw = pool.size();
  std::vector<TopList> per(size_t(nw) * nq, TopList{ix.metric, k, {}});
  const uint32_t d = ix.d;
  const bool fast = host_has_avx2();
  // queries in fp64 once per batch (only those with misses)
  std::vector<double> Qd;
  std::vector<int64_t> qslot(nq, -1);
  if (fast) {
    size_t n = 0;
    for (uint32_t q = 0; q < nq; ++q) {
      if (!slow[q].empty()) qslot[q] = int64_t(n++);
    }
    Qd.resize(n * d);
    for (uint32_t q = 0; q < nq; ++q) {
      if (qslot[q] < 0) continue;
      for (uint32_t j = 0; j < d; ++j) Qd[size_t(qslot[q]) * d + j] = Q[size_t(q) * d + j];
    }
  }
  pool.parallel_for(tasks.size(), [&](size_t t, unsigned wid) {
    const Task& tk = tasks[t];
    if (fast) {
      const std::vector<uint32_t>& qs = *tk.qs;
      std::vector<const double*> qp(qs.size());
      for (size_t i = 0; i < qs.size(); ++i) qp[i] = Qd.data() + size_t(qslot[qs[i]]) * d;
      std::vector<double> sc(qs.size());
      for (uint64_t r = tk.r0; r < tk.r1; ++r) {
        const float* x = ix.vecs + r * d;
        if (ix.metric == kMetricIP) {
          score_row_blocked<true>(x, qp.data(), uint32_t(qs.size()), d, sc.data());
        } else {
          score_row_blocked<false>(x, qp.data(), uint32_t(qs.size()), d, sc.data());
        }
        for (size_t i = 0; i < qs.size(); ++i) {
          const float s = ix.metric == kMetricIP ? static_cast<float>(sc[i])
                                                 : static_cast<float>(std::sqrt(sc[i]));
          per[size_t(wid) * nq + qs[i]].push({s, ix.ids[r]});
        }
      }
      return;
    }
    for (uint64_t r = tk.r0; r < tk.r1; ++r) {
      const float* x = ix.vecs + r * d;
      for (uint32_t q : *tk.qs) {
        const float* qv = Q + size_t(q) * d;
        const float s = ix.metric == kMetricIP
                            ? static_cast<float>(dot_f64(qv, x, d))
                            : static_cast<float>(std::sqrt(l2sq_f64(qv, x, d)));
        per[size_t(wid) * nq + q].push({s, ix.ids[r]});
      }
    }
  });
  std::vector<std::vector<Scored>> out(nq);
  for (uint32_t q = 0; q < nq; ++q) {
    TopList all{ix.metric, k, {}};
    for (unsigned w = 0; w < nw; ++w) {
      for (const auto& e : per[size_t(w) * nq + q].e) all.push(e);
    }
    out[q] = std::move(all.e);
  }
  return out;
}

std::vector<Scored> merge_topk(int metric, const std::vector<Scored>& a,
                               const std::vector<Scored>& b, int k) {
  std::vector<Scored> out;
  out.reserve(std::min<size_t>(a.size() + b.size(), static_cast<size_t>(k)));
  size_t i = 0, j = 0;
  while (static_cast<int>(out.size()) < k && (i < a.size() || j < b.size())) {
    if (j >= b.size() || (i < a.size() && ranks_before(metric, a[i], b[j]))) {
      out.push_back(a[i++]);
    } else {
      out.push_back(b[j++]);
    }
  }
  return out;
}

// ==========================================================================
// planner (tiered.cpp:67-84)
// ==========================================================================
void plan_walk(const Index& ix, const uint32_t* order,
               const std::function<bool(uint32_t)>& resident, uint64_t budget,
               std::vector<uint32_t>& plan, uint64_t& planned,
               std::vector<uint32_t>& skipped) {
  plan.clear();
  skipped.clear();
  planned = 0;
  uint64_t remaining = budget;
  for (uint32_t i = 0; i < ix.nc; ++i) {
    const uint32_t c = order[i];
    if (resident(c)) continue;
    const uint64_t b = ix.cluster_bytes(c);
    if (b <= remaining) {
      plan.push_back(c);
      planned += b;
      remaining -= b;
    } else {
      skipped.push_back(c);
    }
  }
}

// ==========================================================================
// schedulers (sched.cpp)
// ==========================================================================
namespace {
double l2sq_serial(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double t = static_cast<double>(a[j]) - static_cast<double>(b[j]);
    acc += t * t;
  }
  return acc;
}
} // namespace

void group_microbatches(const float* q, uint64_t n, uint32_t d, uint64_t m,
                        std::vector<uint64_t>& order,
                        std::vector<uint64_t>& off, ThreadPool* pool) {
  if (m < 1) throw std::invalid_argument("micro-batch size must be >= 1");
  // fp64 L2^2 with the reference's serial accumulation (symmetric bit for
  // bit: (a-b)^2 == (b-a)^2). Small n: the whole upper triangle at once, rows
  // in parallel. Larger n: each seed's row over its unassigned later queries
  // only (what sched.cpp:52-56 computes), so memory stays O(n).
  constexpr uint64_t kMatrixMax = 2048; // 32 MB of pair distances
  const bool matrix = n <= kMatrixMax;
  std::vector<double> dist(matrix ? n * n : n, 0.0);
  if (matrix) {
    auto row = [&](size_t i, unsigned) {
      for (uint64_t j = i + 1; j < n; ++j) dist[i * n + j] = l2sq_serial(q + i * d, q + j * d, d);
    };
    if (pool) pool->parallel_for(n, row);
    else for (size_t i = 0; i < n; ++i) row(i, 0);
  }
  order.clear();
  off.assign(1, 0);
  std::vector<char> assigned(n, 0);
  std::vector<std::pair<double, uint64_t>> cand;
  std::vector<uint64_t> open;
  for (uint64_t seed = 0; seed < n; ++seed) {
    if (assigned[seed]) continue;
    order.push_back(seed);
    assigned[seed] = 1;
    cand.clear();
    if (m > 1) {
      if (matrix) {
        for (uint64_t j = seed + 1; j < n; ++j) {
          if (!assigned[j]) cand.emplace_back(dist[seed * n + j], j);
        }
      } else {
        open.clear();
        for (uint64_t j = seed + 1; j < n; ++j) {
          if (!assigned[j]) open.push_back(j);
        }
        constexpr size_t kChunk = 256;
        auto part = [&](size_t c, unsigned) {
          const size_t e = std::min(open.size(), (c + 1) * kChunk);
          for (size_t x = c * kChunk; x < e; ++x) {
            dist[open[x]] = l2sq_serial(q + seed * d, q + open[x] * d, d);
          }
        };
        const size_t nch = (open.size() + kChunk - 1) / kChunk;
        if (pool && nch > 1) pool->parallel_for(nch, part);
        else for (size_t c = 0; c < nch; ++c) part(c, 0);
        for (uint64_t j : open) cand.emplace_back(dist[j], j);
      }
    }
    const size_t take = std::min<size_t>(m - 1, cand.size());
    std::partial_sort(cand.begin(), cand.begin() + take, cand.end());
    for (size_t t = 0; t < take; ++t) {
      order.push_back(cand[t].second);
      assigned[cand[t].second] = 1;
    }
    off.push_back(order.size());
  }
}

std::vector<uint32_t> greedy_assign(const std::vector<uint64_t>& overlap,
                                    uint32_t nb, uint32_t nw) {
  if (nw == 0) throw std::invalid_argument("need at least one worker");
  const uint64_t cap = (uint64_t(nb) + nw - 1) / nw;
  std::vector<uint32_t> a(nb, 0);
  std::vector<char> placed(nb, 0);
  std::vector<uint64_t> load(nw, 0);
  for (uint32_t step = 0; step < nb; ++step) {
    uint32_t bb = nb, bw = nw;
    uint64_t best = 0;
    bool found = false;
    for (uint32_t b = 0; b < nb; ++b) {
      if (placed[b]) continue;
      for (uint32_t w = 0; w < nw; ++w) {
        if (load[w] >= cap) continue;
        const uint64_t o = overlap[uint64_t(b) * nw + w];
        const bool better =
            !found || o > best ||
            (o == best && (b < bb || (b == bb && (load[w] < load[bw] ||
                                                  (load[w] == load[bw] && w < bw)))));
        if (better) {
          found = true;
          bb = b;
          bw = w;
          best = o;
        }
      }
    }
    a[bb] = bw;
    placed[bb] = 1;
    ++load[bw];
  }
  return a;
}

std::vector<uint64_t> split_budget(uint64_t total, const uint64_t* batch,
                                   uint64_t n) {
  if (n == 0) throw std::invalid_argument("cannot split a budget over an empty batch");
  const uint64_t base = total / n, rem = total % n;
  std::vector<size_t> by_id(n);
  std::iota(by_id.begin(), by_id.end(), size_t{0});
  std::stable_sort(by_id.begin(), by_id.end(),
                   [&](size_t a, size_t b) { return batch[a] < batch[b]; });
  std::vector<uint64_t> out(n, base);
  for (uint64_t r = 0; r < rem; ++r) out[by_id[r]] += 1;
  return out;
}

// ==========================================================================
// hotness (cache.cpp)
// ==========================================================================
Hotness::Hotness(float h_init, float h_inc, float decay, double fraction)
    : h_init_(h_init), h_inc_(h_inc), decay_(decay), fraction_(fraction) {
  if (h_init <= 0.0f || h_inc <= 0.0f) {
    throw std::invalid_argument("h_init and h_inc must be positive");
  }
  if (decay <= 1.0f) throw std::invalid_argument("decay factor must exceed 1");
  if (fraction <= 0.0 || fraction > 1.0) {
    throw std::invalid_argument("cache_fraction must be in (0, 1]");
  }
}

void Hotness::end_of_round(const std::unordered_set<uint32_t>& used) {
  for (auto& [c, h] : h_) {
    float v = h / decay_;
    if (used.count(c)) v = v + h_inc_;
    h = v;
  }
}

std::vector<uint32_t> Hotness::eviction_order(const std::vector<uint32_t>& resident) const {
  std::vector<uint32_t> o(resident);
  std::sort(o.begin(), o.end(), [this](uint32_t a, uint32_t b) {
    const auto ia = h_.find(a), ib = h_.find(b);
    const float ha = ia == h_.end() ? 0.0f : ia->second;
    const float hb = ib == h_.end() ? 0.0f : ib->second;
    if (ha != hb) return ha < hb;
    return a < b;
  });
  return o;
}

} // namespace laivg
