// synth_capi.cpp — C entry points of oracle/libsynth.so: the synthetic
// workload generator (paper_2502_20969_b200/csrc/synth.cpp, the SAME source
// and flags liblaivg.so compiles) on its own, so bench.py's reference arm and
// the checkers draw the bench datastore without loading the product library.
// Workload generation only: no search code lives here.
#include <algorithm>
#include <stdexcept>
#include <thread>
#include <string>

#include "synth.hpp"

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
} // namespace

extern "C" {
const char* lsynth_last_error(void) { return g_err.c_str(); }

int lsynth_centroids(uint64_t seed, uint32_t nc, uint32_t d, float* out) {
  return guard([&] { laivg::synth_centroids(seed, nc, d, out); });
}

int lsynth_lists(uint64_t seed, const float* centroids, uint32_t nc, uint32_t d,
                 uint64_t per_list, float spread, uint32_t c_begin, uint32_t c_end, float* vecs,
                 uint64_t* ids, int threads) {
  return guard([&] {
    if (c_end > nc || c_begin > c_end) throw std::invalid_argument("bad cluster range");
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    laivg::synth_lists(seed, centroids, d, per_list, spread, c_begin, c_end, vecs, ids,
                       threads);
  });
}

int lsynth_queries(uint64_t seed, const float* vecs, uint64_t n_rows, uint32_t d, uint32_t nq,
                   float sigma, float* q_in, float* q_out, uint64_t* rows) {
  return guard([&] { laivg::synth_queries(seed, vecs, n_rows, d, nq, sigma, q_in, q_out, rows); });
}

int lsynth_queries_topical(uint64_t seed, const float* centroids, uint32_t nc, const float* vecs,
                           const uint64_t* list_off, uint32_t d, uint32_t n_topics, double zipf_s,
                           uint32_t neigh, uint32_t nq, float sigma, float* q_in, float* q_out,
                           uint64_t* rows, uint32_t* topic) {
  return guard([&] {
    laivg::synth_queries_topical(seed, centroids, nc, vecs, list_off, d, n_topics, zipf_s, neigh,
                                 nq, sigma, q_in, q_out, rows, topic);
  });
}
}
