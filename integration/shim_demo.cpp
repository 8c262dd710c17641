// shim_demo.cpp — drop-in check of laiv_gpu_shim.hpp against the UNMODIFIED
// reference (proj/core sources compiled in place by integration/Makefile).
//
// Builds a random datastore and an IvfIndex with the reference's own
// build_index, then runs the reference's laiv::ivf_search / hybrid_search
// and the shim's laiv::gpu:: versions on the same inputs and compares them
// (ids exact, scores within 1e-5 relative: SURVEY §8c). Prints one JSON line;
// exit code 0 = all queries agree. Test infrastructure: the reference here
// is the checker, the GPU path the thing checked.
#include <laiv/ivf.hpp>
#include <laiv/rng.hpp>
#include <laiv/tiered.hpp>
#include <laiv/vectorstore.hpp>

#include <cmath>
#include <cstdio>
#include <string>
#include <random>

#include "laiv_gpu_shim.hpp"

namespace {

bool agree(const laiv::TopK& a, const laiv::TopK& b, int& exact) {
  if (a.entries.size() != b.entries.size()) return false;
  bool same = true;
  for (size_t i = 0; i < a.entries.size(); ++i) {
    const float x = a.entries[i].score, y = b.entries[i].score;
    if (a.entries[i].id != b.entries[i].id) {
      // a swap is allowed only across a near-tie
      if (std::fabs(x - y) > 1e-5f * std::fabs(y)) return false;
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
  std::vector<float> row(d);
  for (uint32_t i = 0; i < n; ++i) {
    for (auto& x : row) x = g(rng);
    db.append(1000 + uint64_t(i) * 3, row); // non-contiguous ids
  }
  const laiv::IvfIndex ix = laiv::build_index(db, nc, laiv::IvfBuildOptions{1, 8, false}, metric);
  laiv::EmbeddingMatrix queries(d);
  for (int t = 0; t < nq; ++t) {
    for (auto& x : row) x = g(rng);
    queries.append(uint64_t(t), row);
  }

  laiv::gpu::Bound gpu(ix, db, uint64_t(1) << 30, /*device=*/0);
  // half of the lists cached on the GPU: hybrid splits hits and misses
  for (uint32_t c = 0; c < nc; c += 2) gpu.insert(c);
  laiv::TieredStore store(uint64_t(1) << 30);
  for (uint32_t c = 0; c < nc; c += 2) store.insert(c, ix.cluster_bytes(c), laiv::Residency::Prefetched);

  int ok = 0, exact = 0, probe_eq = 0;
  const laiv::CostModel cost;
  for (int t = 0; t < nq; ++t) {
    const auto q = queries.row(t);
    const laiv::TopK want = laiv::ivf_search(ix, db, q, L, k);
    const laiv::TopK got = laiv::gpu::ivf_search(gpu, q, L, k);
    auto [hr_ref, tm_ref] = laiv::hybrid_search(ix, db, store, q, L, k, cost);
    auto [hr_gpu, tm_gpu] = laiv::gpu::hybrid_search(gpu, q, L, k, cost);
    probe_eq += laiv::coarse_probe(ix, q, L) == laiv::gpu::coarse_probe(gpu, q, L);
    const bool a = agree(got, want, exact);
    const bool b = agree(hr_gpu.topk, hr_ref.topk, exact) &&
                   hr_gpu.fast_clusters == hr_ref.fast_clusters &&
                   hr_gpu.slow_clusters == hr_ref.slow_clusters &&
                   hr_gpu.hit_rate == hr_ref.hit_rate;
    ok += a && b;
  }
  // the batch entry point
  const auto batch = laiv::gpu::ivf_search_batch(gpu, queries, L, k);
  int batch_ok = 0;
  for (int t = 0; t < nq; ++t) {
    int e = 0;
    batch_ok += agree(batch[size_t(t)], laiv::ivf_search(ix, db, queries.row(t), L, k), e);
  }
  // LAIX: the reference's save_index, bound straight from the file; the
  // library's save writes the same bytes back
  const std::string dir = argc > 2 ? argv[2] : "/tmp";
  const std::string f1 = dir + "/shim_demo_ref.laix", f2 = dir + "/shim_demo_gpu.laix";
  laiv::save_index(f1, ix, db);
  int file_ok = 0;
  {
    laiv::gpu::Bound fromfile(f1, uint64_t(1) << 30, /*device=*/0);
    fromfile.save(f2);
    for (int t = 0; t < nq; ++t) {
      int e = 0;
      file_ok += agree(laiv::gpu::ivf_search(fromfile, queries.row(t), L, k),
                       laiv::ivf_search(ix, db, queries.row(t), L, k), e);
    }
  }
  auto slurp = [](const std::string& p) {
    std::FILE* f = std::fopen(p.c_str(), "rb");
    std::string s;
    if (!f) return s;
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, n);
    std::fclose(f);
    return s;
  };
  const bool same_bytes = slurp(f1) == slurp(f2) && !slurp(f1).empty();
  std::remove(f1.c_str());
  std::remove(f2.c_str());
  std::printf("{\"metric\": \"%s\", \"queries\": %d, \"agree\": %d, \"bit_identical_pairs\": %d, "
              "\"probe_identical\": %d, \"batch_agree\": %d, \"laix_agree\": %d, "
              "\"laix_same_bytes\": %s}\n",
              metric == laiv::Metric::L2 ? "l2" : "ip", nq, ok, exact, probe_eq, batch_ok, file_ok,
              same_bytes ? "true" : "false");
  return (ok == nq && batch_ok == nq && probe_eq == nq && file_ok == nq && same_bytes) ? 0 : 1;
}
