// host.hpp — host-side (CPU) parts of the retrieval path: the index model,
// the cache-miss scanner and its thread pool, the prefetch planner, the
// schedulers, the hotness policy and the synthetic workload generator.
// Pure C++; ctx.cu couples these to the device.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "synth.hpp"

namespace laivg {

constexpr int kMetricIP = 0;
constexpr int kMetricL2 = 1;
constexpr uint64_t kMissChunk = 512; // vectors per host miss-scan task (batched scan)
// single query: a missed list is usually the only host work and must finish
// inside the GPU's hit scan, so it is cut finer to occupy every host thread
constexpr uint64_t kMissChunkSingle = 128;

// CUDA failures map to LAIVG_ECUDA at the ABI.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Scored {
  float s;
  uint64_t id;
};

// vectorstore.hpp:34-39
inline bool ranks_before(int metric, const Scored& a, const Scored& b) {
  if (a.s != b.s) return metric == kMetricIP ? a.s > b.s : a.s < b.s;
  return a.id < b.id;
}

// IvfIndex + EmbeddingMatrix over a list-major host store (ivf.hpp:26-50).
struct Index {
  uint32_t nc = 0, d = 0;
  int metric = kMetricL2;
  std::vector<float> centroids;     // nc * d
  std::vector<uint64_t> list_off;   // nc + 1
  const float* vecs = nullptr;      // list_off[nc] * d (pinned when owned)
  const uint64_t* ids = nullptr;    // list_off[nc]
  void* owned_block = nullptr;      // pinned allocation when copied
  bool owned_pageable = false;      // owned_block came from aligned_alloc
  bool owned_registered = false;    // ... and is pinned in place (cudaHostRegister)
  uint64_t member_bytes() const { return 4ull * d + 8ull; } // ivf.cpp:23
  uint64_t list_len(uint32_t c) const { return list_off[c + 1] - list_off[c]; }
  uint64_t cluster_bytes(uint32_t c) const { return list_len(c) * member_bytes(); }
  uint64_t total() const { return list_off[nc]; }
};

// Fixed pool; parallel_for blocks until every task ran. The calling thread
// participates, so a pool of n threads uses n + 1 cores.
class ThreadPool {
 public:
  explicit ThreadPool(unsigned n);
  ~ThreadPool();
  unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }
  void parallel_for(size_t n, const std::function<void(size_t, unsigned)>& fn);

 private:
  void loop(unsigned wid);
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t, unsigned)>* job_ = nullptr;
  size_t n_ = 0;
  std::atomic<size_t> next_{0};
  unsigned active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// LAIX files (laix.cpp). first_invalid_row: the first row of a list-major
// store that EmbeddingMatrix::append would reject (vectorstore.cpp:66-85),
// n when none; validate_store throws the reference's invalid_argument for it.
uint64_t first_invalid_row(const float* vecs, const uint64_t* ids, uint64_t n, uint32_t d,
                           unsigned threads, bool* dup);
void validate_store(const Index& ix, unsigned threads);
// load_index (ivf.cpp:394-458) / save_index (ivf.cpp:351-392) against the
// list-major store; alloc(bytes, user) provides the block for rows + ids.
void laix_load(const std::string& path, unsigned threads, Index& ix,
               void* (*alloc)(uint64_t bytes, void* user), void* user);
void laix_save(const std::string& path, const Index& ix, unsigned threads);

// Cache-miss path (the slow tier of hybrid_search, tiered.cpp:169): scores
// every member of `lists` with fp64 accumulation rounded to fp32
// (vectorstore.cpp:93-115) and returns the best-k, best-first.
std::vector<Scored> miss_scan(const Index& ix, const float* q,
                              const std::vector<uint32_t>& lists, int k,
                              ThreadPool& pool);

// score_clusters' host half (ivf.cpp:301-324): every row of list c scored
// (the miss scan's arithmetic) into s_out / id_out starting at offset o, for
// each (c, o) of items.
void score_lists(const Index& ix, const float* q,
                 const std::vector<std::pair<uint32_t, uint64_t>>& items, float* s_out,
                 uint64_t* id_out, ThreadPool& pool);

// Batched miss path: slow[q] are the missed lists of query q (rows of Q).
// List-major: each missed list is read once and scored for every query that
// misses it. Returns each query's best-k, best-first.
std::vector<std::vector<Scored>> miss_scan_batch(const Index& ix, const float* Q, uint32_t nq,
                                                 const std::vector<std::vector<uint32_t>>& slow,
                                                 int k, ThreadPool& pool);

// Best-k merge of two best-first lists (the hybrid merge, tiered.cpp:172-185:
// a global sort of the concatenation truncated to k equals this merge).
std::vector<Scored> merge_topk(int metric, const std::vector<Scored>& a,
                               const std::vector<Scored>& b, int k);

// plan_prefetch walk (tiered.cpp:67-84) over a full ranking.
void plan_walk(const Index& ix, const uint32_t* order,
               const std::function<bool(uint32_t)>& resident, uint64_t budget,
               std::vector<uint32_t>& plan, uint64_t& planned,
               std::vector<uint32_t>& skipped);

// sched.cpp:39-70 / 72-85 / 146-155 / 170-192
void group_microbatches(const float* q, uint64_t n, uint32_t d, uint64_t m,
                        std::vector<uint64_t>& order,
                        std::vector<uint64_t>& off, ThreadPool* pool);
// sched.cpp:114-142: greedy over an nb x nw overlap matrix.
std::vector<uint32_t> greedy_assign(const std::vector<uint64_t>& overlap,
                                    uint32_t nb, uint32_t nw);
std::vector<uint64_t> split_budget(uint64_t total, const uint64_t* batch,
                                   uint64_t n);

// cache.hpp:28-56
class Hotness {
 public:
  Hotness(float h_init, float h_inc, float decay, double fraction);
  void on_fetch(uint32_t c) { h_[c] = h_init_; }
  void end_of_round(const std::unordered_set<uint32_t>& used);
  // Order in which evict_to_fraction removes clusters: ascending
  // (hotness, id) over the given resident ids (cache.cpp:48-56).
  std::vector<uint32_t> eviction_order(const std::vector<uint32_t>& resident) const;
  void forget(uint32_t c) { h_.erase(c); }
  void clear() { h_.clear(); }
  bool tracked(uint32_t c) const { return h_.count(c) != 0; }
  float get(uint32_t c) const { return h_.at(c); }
  double fraction() const { return fraction_; }

 private:
  float h_init_, h_inc_, decay_;
  double fraction_;
  std::map<uint32_t, float> h_;
};

} // namespace laivg
