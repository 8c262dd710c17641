// synth.cpp — the synthetic workload generator of SURVEY §8d (planted
// clusters, queries, topical queries). Not on the retrieval path: it makes the
// bench / test datastores. Compiled into liblaivg.so (laivg_synth_*) and, from
// this same file with the same flags, into oracle/libsynth.so so the
// reference arm of bench.py draws identical data without loading the product.
#include "synth.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <thread>
#include <vector>

namespace laivg {

// ==========================================================================
// synthetic workload
// ==========================================================================
namespace {
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// Approximately standard normal: Irwin-Hall sum of four 16-bit uniforms,
// scaled to unit variance. Exact integer + IEEE arithmetic only, so the
// stream is identical on every platform.
inline double gauss(uint64_t key) {
  const uint64_t h = mix64(key);
  const double s = double(h & 0xffff) + double((h >> 16) & 0xffff) +
                   double((h >> 32) & 0xffff) + double(h >> 48);
  // each term uniform on {0..65535}: mean 32767.5, var (65536^2-1)/12
  return (s - 4.0 * 32767.5) * (1.7320508075688772 / 65536.0);
}
inline uint64_t stream(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(mix64(seed ^ 0x6c61697667ull) + a * 0x100000001b3ull + b);
}
void normalize_into(const double* v, uint32_t d, float* out) {
  double ss = 0.0;
  for (uint32_t t = 0; t < d; ++t) ss += v[t] * v[t];
  const double n = std::sqrt(ss);
  for (uint32_t t = 0; t < d; ++t) out[t] = static_cast<float>(n > 0.0 ? v[t] / n : v[t]);
}
} // namespace

void synth_centroids(uint64_t seed, uint32_t nc, uint32_t d, float* out) {
  std::vector<double> v(d);
  for (uint32_t j = 0; j < nc; ++j) {
    const uint64_t s = stream(seed, 1, j);
    for (uint32_t t = 0; t < d; ++t) v[t] = gauss(s * 0x9e3779b97f4a7c15ull + t);
    normalize_into(v.data(), d, out + uint64_t(j) * d);
  }
}

void synth_lists(uint64_t seed, const float* centroids, uint32_t d,
                 uint64_t per_list, float spread, uint32_t c_begin,
                 uint32_t c_end, float* vecs, uint64_t* ids, int threads) {
  const uint32_t n = c_end - c_begin;
  auto work = [&](uint32_t lo, uint32_t hi) {
    std::vector<double> v(d);
    for (uint32_t j = lo; j < hi; ++j) {
      const float* mu = centroids + uint64_t(j) * d;
      for (uint64_t i = 0; i < per_list; ++i) {
        const uint64_t row = uint64_t(j - c_begin) * per_list + i;
        const uint64_t s = stream(seed, 2 + (uint64_t(j) << 32), i);
        for (uint32_t t = 0; t < d; ++t) {
          v[t] = static_cast<double>(mu[t]) +
                 static_cast<double>(spread) * gauss(s * 0x9e3779b97f4a7c15ull + t);
        }
        normalize_into(v.data(), d, vecs + row * d);
        ids[row] = uint64_t(j) * per_list + i;
      }
    }
  };
  const int nt = std::max(1, threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) {
    const uint32_t lo = c_begin + uint32_t(uint64_t(n) * t / nt);
    const uint32_t hi = c_begin + uint32_t(uint64_t(n) * (t + 1) / nt);
    pool.emplace_back(work, lo, hi);
  }
  for (auto& t : pool) t.join();
}

namespace {
// q_in = normalize(x_r + 0.01 g), q_out = normalize(q_in + sigma g) for query i
void query_pair(uint64_t seed, uint32_t i, const float* x, uint32_t d, float sigma, float* q_in,
                float* q_out, std::vector<double>& v) {
  const uint64_t s1 = stream(seed, 4, i), s2 = stream(seed, 5, i);
  for (uint32_t t = 0; t < d; ++t) {
    v[t] = static_cast<double>(x[t]) + 0.01 * gauss(s1 * 0x9e3779b97f4a7c15ull + t);
  }
  normalize_into(v.data(), d, q_in);
  for (uint32_t t = 0; t < d; ++t) {
    v[t] = static_cast<double>(q_in[t]) +
           static_cast<double>(sigma) * gauss(s2 * 0x9e3779b97f4a7c15ull + t);
  }
  normalize_into(v.data(), d, q_out);
}
} // namespace

void synth_queries(uint64_t seed, const float* vecs, uint64_t n_rows,
                   uint32_t d, uint32_t nq, float sigma, float* q_in,
                   float* q_out, uint64_t* rows) {
  std::vector<double> v(d);
  for (uint32_t i = 0; i < nq; ++i) {
    const uint64_t r = mix64(stream(seed, 3, i)) % n_rows;
    rows[i] = r;
    query_pair(seed, i, vecs + r * d, d, sigma, q_in + uint64_t(i) * d, q_out + uint64_t(i) * d,
               v);
  }
}

void synth_queries_topical(uint64_t seed, const float* centroids, uint32_t nc,
                           const float* vecs, const uint64_t* list_off, uint32_t d,
                           uint32_t n_topics, double zipf_s, uint32_t neigh, uint32_t nq,
                           float sigma, float* q_in, float* q_out, uint64_t* rows,
                           uint32_t* topic) {
  if (n_topics == 0 || n_topics > nc) throw std::invalid_argument("bad topic count");
  neigh = std::max(1u, std::min(neigh, nc));
  // topic centres: distinct random lists
  std::vector<uint32_t> centre;
  std::vector<uint8_t> used(nc, 0);
  for (uint64_t t = 0; centre.size() < n_topics; ++t) {
    const uint32_t c = uint32_t(mix64(stream(seed, 7, t)) % nc);
    if (!used[c]) {
      used[c] = 1;
      centre.push_back(c);
    }
  }
  // neighbourhood of each topic: the `neigh` nearest centroids (fp64 L2,
  // ties by id)
  std::vector<uint32_t> hood(size_t(n_topics) * neigh);
  std::vector<std::pair<double, uint32_t>> dist(nc);
  for (uint32_t t = 0; t < n_topics; ++t) {
    const float* a = centroids + uint64_t(centre[t]) * d;
    for (uint32_t c = 0; c < nc; ++c) {
      const float* b = centroids + uint64_t(c) * d;
      double s2 = 0;
      for (uint32_t j = 0; j < d; ++j) {
        const double x = double(a[j]) - double(b[j]);
        s2 += x * x;
      }
      dist[c] = {s2, c};
    }
    std::partial_sort(dist.begin(), dist.begin() + neigh, dist.end());
    for (uint32_t j = 0; j < neigh; ++j) hood[size_t(t) * neigh + j] = dist[j].second;
  }
  // Zipf popularity over topics
  std::vector<double> cdf(n_topics);
  double acc = 0;
  for (uint32_t t = 0; t < n_topics; ++t) {
    acc += 1.0 / std::pow(double(t + 1), zipf_s);
    cdf[t] = acc;
  }
  std::vector<double> v(d);
  for (uint32_t i = 0; i < nq; ++i) {
    const double u = double(mix64(stream(seed, 6, i)) >> 11) * 0x1.0p-53 * acc;
    const uint32_t t = uint32_t(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    const uint32_t tt = std::min(t, n_topics - 1);
    const uint32_t c = hood[size_t(tt) * neigh + mix64(stream(seed, 8, i)) % neigh];
    const uint64_t len = list_off[c + 1] - list_off[c];
    if (len == 0) throw std::invalid_argument("topic neighbourhood holds an empty list");
    const uint64_t r = list_off[c] + mix64(stream(seed, 3, i)) % len;
    rows[i] = r;
    if (topic) topic[i] = tt;
    query_pair(seed, i, vecs + r * d, d, sigma, q_in + uint64_t(i) * d, q_out + uint64_t(i) * d,
               v);
  }
}

} // namespace laivg
