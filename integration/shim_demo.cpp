// shim_demo.cpp — drop-in check of laiv_gpu_shim.hpp against the UNMODIFIED
// reference (proj/core sources compiled in place by integration/Makefile).
//
// One caller (caller_body.inc: grouping, cache-aware routing, lookahead
// plan + transfer, hybrid retrieval, hotness eviction, incremental prefetch,
// rank / probe / score / search_clusters / ivf / exact / pairwise / coverage)
// is compiled twice from the same source: against namespace laiv (the
// reference) and against laiv::gpu (the B200 path). The two runs start from
// the same index (the reference's own build_index) and must make the same
// decisions and return the same results (ids exact, scores within 1e-5
// relative: SURVEY §8c). Also: the batched entry points, and a LAIX file
// written by the reference's save_index, loaded by the library and written
// back byte for byte. Prints one JSON line; exit code 0 = everything agrees.
// Test infrastructure: the reference here is the checker.
#include <laiv/cache.hpp>
#include <laiv/ivf.hpp>
#include <laiv/sched.hpp>
#include <laiv/tiered.hpp>
#include <laiv/vectorstore.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <unordered_set>

#include "laiv_gpu_shim.hpp"

namespace ref_run {
namespace impl = ::laiv;
using Store = ::laiv::TieredStore;
#include "caller_body.inc"
} // namespace ref_run

namespace gpu_run {
namespace impl = ::laiv::gpu;
using Store = ::laiv::gpu::TieredStore;
#include "caller_body.inc"
} // namespace gpu_run

namespace {

bool agree(const laiv::TopK& a, const laiv::TopK& b, int& exact) {
  if (a.entries.size() != b.entries.size()) return false;
  bool same = true;
  for (size_t i = 0; i < a.entries.size(); ++i) {
    const float x = a.entries[i].score, y = b.entries[i].score;
    if (a.entries[i].id != b.entries[i].id) {
      if (std::fabs(x - y) > 1e-5f * std::fabs(y)) return false; // swap only across a near-tie
      same = false;
    } else if (std::fabs(x - y) > 1e-5f * std::fabs(y)) {
      return false;
    } else if (x != y) {
      same = false;
    }
  }
  exact += same;
  return true;
}

int agree_all(const std::vector<laiv::TopK>& a, const std::vector<laiv::TopK>& b, int& exact,
              int& total) {
  int ok = 0;
  for (size_t i = 0; i < std::min(a.size(), b.size()); ++i) ok += agree(a[i], b[i], exact);
  total += int(b.size());
  return a.size() == b.size() ? ok : -1;
}

std::string slurp(const std::string& p) {
  std::FILE* f = std::fopen(p.c_str(), "rb");
  std::string s;
  if (!f) return s;
  char buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, n);
  std::fclose(f);
  return s;
}

} // namespace

int main(int argc, char** argv) {
  const uint32_t n = 20000, d = 64, nc = 64;
  const int L = 8, k = 10, nq = 64;
  const laiv::Metric metric = argc > 1 && std::string(argv[1]) == "l2" ? laiv::Metric::L2
                                                                        : laiv::Metric::InnerProduct;
  std::mt19937_64 rng(7);
  std::normal_distribution<float> g(0.f, 1.f);
  laiv::EmbeddingMatrix db(d);
  db.reserve(n);
  std::vector<float> row(d), row2(d);
  for (uint32_t i = 0; i < n; ++i) {
    for (auto& x : row) x = g(rng);
    db.append(1000 + uint64_t(i) * 3, row); // non-contiguous ids
  }
  const laiv::IvfIndex ix = laiv::build_index(db, nc, laiv::IvfBuildOptions{1, 8, false}, metric);
  laiv::EmbeddingMatrix q_in(d), q_out(d);
  for (int t = 0; t < nq; ++t) {
    for (size_t j = 0; j < d; ++j) {
      row[j] = g(rng);
      row2[j] = row[j] + 0.3f * g(rng);
    }
    q_in.append(uint64_t(t), row);
    q_out.append(uint64_t(t), row2);
  }
  const uint64_t cap = uint64_t(12) << 20; // ~1/3 of the lists
  laiv::TransferChannel ref_chan;          // SimulatedClock
  laiv::TransferChannel gpu_chan{50e9, laiv::gpu::kDevice};

  laiv::TieredStore ref_store(cap);
  const auto want = ref_run::run(ix, db, q_in, q_out, ref_store, ref_chan, L, k);
  laiv::gpu::TieredStore gpu_store(cap, ix, db, /*device=*/0);
  const auto got = gpu_run::run(ix, db, q_in, q_out, gpu_store, gpu_chan, L, k);

  int exact = 0, total = 0;
  const int hybrid_ok = agree_all(got.hybrid, want.hybrid, exact, total);
  const int ivf_ok = agree_all(got.ivf, want.ivf, exact, total);
  const int clusters_ok = agree_all(got.clusters, want.clusters, exact, total);
  const int exact_ok = agree_all(got.exact, want.exact, exact, total);
  bool scored_ok = got.scored.size() == want.scored.size();
  for (size_t i = 0; scored_ok && i < want.scored.size(); ++i) {
    scored_ok = got.scored[i].size() == want.scored[i].size();
    for (size_t j = 0; scored_ok && j < want.scored[i].size(); ++j) {
      const float x = got.scored[i][j].score, y = want.scored[i][j].score;
      scored_ok = got.scored[i][j].id == want.scored[i][j].id &&
                  std::fabs(x - y) <= 1e-5f * std::fabs(y);
    }
  }
  const bool decisions = got.groups == want.groups && got.assignment == want.assignment &&
                         got.overlap == want.overlap && got.split == want.split &&
                         got.plans == want.plans && got.transferred == want.transferred &&
                         got.fast == want.fast && got.slow == want.slow &&
                         got.evicted == want.evicted && got.used_after == want.used_after;
  const bool ranks = got.ranks == want.ranks && got.probes == want.probes &&
                     got.coverage == want.coverage;
  const bool pairwise = got.pairwise == want.pairwise; // bit-identical

  // store accounting through the TieredStore interface
  const bool store_ok = gpu_store.recompute_used_bytes() == gpu_store.used_bytes() &&
                        ref_store.resident_count() == gpu_store.resident_count() &&
                        ref_store.bytes_with_tag(laiv::Residency::Cached) ==
                            gpu_store.bytes_with_tag(laiv::Residency::Cached);

  // batched entry points (one device pass per max_batch queries)
  int batch_ok = 0, e = 0;
  const auto batch = laiv::gpu::ivf_search_batch(ix, db, q_out, L, k);
  const auto hbatch = laiv::gpu::hybrid_search_batch(ix, db, gpu_store, q_out, L, k, laiv::CostModel{});
  for (int t = 0; t < nq; ++t) {
    const auto w = laiv::ivf_search(ix, db, q_out.row(t), L, k);
    batch_ok += agree(batch[size_t(t)], w, e) && agree(hbatch[size_t(t)], w, e);
  }

  // LAIX: the reference's save_index, loaded by the library, written back
  const std::string dir = argc > 2 ? argv[2] : "/tmp";
  const std::string f1 = dir + "/shim_demo_ref.laix", f2 = dir + "/shim_demo_gpu.laix";
  laiv::save_index(f1, ix, db);
  int file_ok = 0;
  {
    auto di = std::make_shared<laiv::gpu::DeviceIndex>(f1);
    di->save(f2);
    laiv::gpu::TieredStore fs(uint64_t(1) << 30, di, /*device=*/0);
    for (int t = 0; t < nq; ++t) {
      std::vector<uint64_t> ids(k);
      std::vector<float> sc(k);
      uint32_t cnt = 0;
      laiv::gpu::ck(laivg_ivf_search(fs.ctx(), q_out.row(t).data(), 1, L, k, ids.data(), sc.data(),
                                     &cnt));
      int e2 = 0;
      file_ok += agree(laiv::gpu::detail::to_topk(k, ids.data(), sc.data(), cnt),
                       laiv::ivf_search(ix, db, q_out.row(t), L, k), e2);
    }
  }
  const bool same_bytes = slurp(f1) == slurp(f2) && !slurp(f1).empty();
  std::remove(f1.c_str());
  std::remove(f2.c_str());

  const bool all = hybrid_ok == int(want.hybrid.size()) && ivf_ok == int(want.ivf.size()) &&
                   clusters_ok == int(want.clusters.size()) &&
                   exact_ok == int(want.exact.size()) && scored_ok && decisions && ranks &&
                   pairwise && store_ok && batch_ok == nq && file_ok == nq && same_bytes;
  std::printf("{\"metric\": \"%s\", \"queries\": %d, \"hybrid_agree\": %d, \"ivf_agree\": %d, "
              "\"search_clusters_k300_agree\": %d, \"exact_agree\": %d, \"topk_lists\": %d, "
              "\"bit_identical_lists\": %d, \"score_clusters_agree\": %s, "
              "\"decisions_identical\": %s, \"rank_probe_coverage_identical\": %s, "
              "\"pairwise_bit_identical\": %s, \"store_accounting\": %s, \"batch_agree\": %d, "
              "\"laix_agree\": %d, \"laix_same_bytes\": %s, \"plans\": %zu, \"evictions\": %zu, "
              "\"all\": %s}\n",
              metric == laiv::Metric::L2 ? "l2" : "ip", nq, hybrid_ok, ivf_ok, clusters_ok,
              exact_ok, total, exact, scored_ok ? "true" : "false", decisions ? "true" : "false",
              ranks ? "true" : "false", pairwise ? "true" : "false", store_ok ? "true" : "false",
              batch_ok, file_ok, same_bytes ? "true" : "false", want.plans.size(),
              want.evicted.size(), all ? "true" : "false");
  return all ? 0 : 1;
}
