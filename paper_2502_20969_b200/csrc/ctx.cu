// ctx.cu — device context (one GPU + its cluster cache) and the C ABI of
// include/laivg.h. Host orchestration only; kernels live in kernels.cu and the
// CPU side (miss scan, planner, schedulers, hotness, synth) in host.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <unordered_set>
#include <sys/mman.h>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/laivg.h"
#include "host.hpp"
#include "kernels.cuh"

namespace laivg {
namespace {

thread_local std::string g_err;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      throw ::laivg::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    }                                                                           \
  } while (0)

using Clock = std::chrono::steady_clock;

// LAIVG_TRACE=1: per-call host phase timestamps of the single-query search,
// printed to stderr (diagnostics for the latency budget; off by default).
struct PhaseTrace {
  bool on = std::getenv("LAIVG_TRACE") != nullptr;
  Clock::time_point t[16];
  const char* name[16];
  int n = 0;
  void mark(const char* nm) {
    if (!on || n >= 16) return;
    t[n] = Clock::now();
    name[n++] = nm;
  }
  void dump() {
    if (!on || n < 2) return;
    std::string s = "[laivg trace]";
    for (int i = 1; i < n; ++i) {
      s += std::string(" ") + name[i] + "=" +
           std::to_string(std::chrono::duration<double, std::micro>(t[i] - t[i - 1]).count());
    }
    std::fprintf(stderr, "%s\n", s.c_str());
  }
};
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

template <class T>
T* dev_alloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}
template <class T>
T* pin_alloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable));
  return static_cast<T*>(p);
}

// Pinned host memory the device also addresses (kernels write results
// straight into it: no copy nodes on the latency path).
template <class T>
T* pin_alloc_mapped(size_t n, T** dev) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable | cudaHostAllocMapped));
  void* d = nullptr;
  CK(cudaHostGetDevicePointer(&d, p, 0));
  *dev = static_cast<T*>(d);
  return static_cast<T*>(p);
}

// First-fit allocator over the device slab, in vectors.
class SlabAlloc {
 public:
  void reset(uint64_t total) {
    total_ = total;
    free_.clear();
    if (total) free_[0] = total;
  }
  bool alloc(uint64_t n, uint64_t& off) {
    if (n == 0) {
      off = 0;
      return true;
    }
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second >= n) {
        off = it->first;
        const uint64_t rest = it->second - n;
        free_.erase(it);
        if (rest) free_[off + n] = rest;
        return true;
      }
    }
    return false;
  }
  void release(uint64_t off, uint64_t n) {
    if (n == 0) return;
    auto it = free_.emplace(off, n).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
      }
    }
  }

 private:
  uint64_t total_ = 0;
  std::map<uint64_t, uint64_t> free_;
};

constexpr uint32_t kMaxFetchChunks = 128;

// Enqueues host->device copies, one cudaMemcpyAsync per (already coalesced)
// run of adjacent lists.
void h2d_batch(std::vector<void*>& dst, std::vector<void*>& src, std::vector<size_t>& size,
               cudaStream_t st) {
  for (size_t i = 0; i < dst.size(); ++i) {
    CK(cudaMemcpyAsync(dst[i], src[i], size[i], cudaMemcpyHostToDevice, st));
  }
}

struct Resident {
  int tag;
  uint64_t bytes;
};

} // namespace

// ============================================================================
// context
// ============================================================================
struct Ctx {
  const Index* ix = nullptr;
  int dev = 0;
  int sms = 148;
  bool acc_fp64 = true;
  ScanImpl scan_impl = ScanImpl::kTma;
  ScanTune tune{};
  cudaStream_t comp = nullptr, copy = nullptr, aux = nullptr;

  // static device data
  float* d_cen = nullptr;
  uint64_t* d_list_off = nullptr;
  uint64_t* d_ids = nullptr;

  // cluster cache (TieredStore, tiered.hpp:22-56)
  uint64_t capacity = 0, used = 0;
  std::map<uint32_t, Resident> resident;
  std::vector<int64_t> h_res;  // slab vector offset per cluster, -1 if absent
  int64_t* d_res = nullptr;
  bool res_dirty = true;
  int64_t* res_stage[2] = {nullptr, nullptr};
  cudaEvent_t res_ev[2] = {nullptr, nullptr};
  int res_slot = 0;
  float* d_slab = nullptr;
  uint64_t slab_vecs = 0;
  SlabAlloc alloc;
  float* d_tmp = nullptr;       // one-list bounce buffer for compaction
  uint64_t tmp_vecs = 0;

  // scratch
  uint32_t max_batch = 256, max_probe = 0;
  // batched coarse quantizer on tensor cores (coarse_tc.cu)
  uint32_t coarse_impl = 0; // 0 auto, 1 fp64 SIMT, 2 tensor cores
  bool tc_ok = false;
  float* d_approx = nullptr; // [max_batch][nc] tf32 scores
  float* d_cnorm = nullptr;  // [nc] ||c|| rounded up
  TcSelectScratch tcs{};     // three-kernel exact selection scratch
  // list-major tensor-core batched scan (listscan.cu), allocated on first use
  ListScanScratch lss{};
  unsigned* h_ls_flag = nullptr;
  unsigned* dm_ls_flag = nullptr;
  bool ls_result = false;    // the last batch's scan results came from the list scan
  double ls_qpl = 0;         // EMA of queries per resident probed list (batches)
  uint64_t ls_runs = 0, ls_fallbacks = 0;
  bool want_list_scan(uint32_t nq, uint32_t lp, int k) const;
  double list_scan_sharing(uint32_t nq, uint32_t lp) const {
    return ls_qpl > 0 ? ls_qpl : double(nq) * lp / std::max(1u, ix->nc);
  }
  void ensure_list_scan();
  void run_list_scan(const float* dQ, uint32_t nq, uint32_t lp, int k, cudaStream_t st);
  float* d_Q = nullptr;
  double* d_scores = nullptr;
  uint32_t* d_order = nullptr;
  uint64_t* d_run_k = nullptr;  // selection scratch (sorted runs)
  uint32_t* d_run_v = nullptr;
  FastTable ft{};
  ScanOut so{};
  // runtime-fetch miss path (batched search): missed lists stream host->HBM
  // through a 2-slot ring and are scanned there, in parallel with the host
  // scan of the remaining misses
  uint32_t miss_fetch = 1;       // 0 off, 1 adaptive split, 2 every fetchable miss
  uint64_t ring_vecs = 0;        // vectors per ring slot
  float* d_ring = nullptr;       // [2][ring_vecs][d]
  int64_t* d_res_ring[2] = {nullptr, nullptr};
  int64_t* h_res_ring = nullptr; // pinned [kMaxFetchChunks][nc] staging
  FastTable fft{};
  ScanOut fso{};
  float* h_fetch_s = nullptr;    // pinned [chunk][fetch_nq][k] chunk results
  uint64_t* h_fetch_id = nullptr;
  uint32_t* h_fetch_cnt = nullptr; // [chunk][max_batch]
  size_t fetch_cap = 0;          // entries h_fetch_s / h_fetch_id hold
  uint32_t fetch_nq = 0;         // queries of the call the chunk results belong to
  void fetch_results_for(size_t entries) {
    if (entries <= fetch_cap) return;
    if (h_fetch_s) cudaFreeHost(h_fetch_s);
    if (h_fetch_id) cudaFreeHost(h_fetch_id);
    h_fetch_s = nullptr;
    h_fetch_id = nullptr;
    fetch_cap = std::max(entries, fetch_cap + fetch_cap / 2);
    h_fetch_s = pin_alloc<float>(fetch_cap);
    h_fetch_id = pin_alloc<uint64_t>(fetch_cap);
  }
  cudaEvent_t ev_landed[2] = {nullptr, nullptr}, ev_freed[2] = {nullptr, nullptr};
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr, ev_fdone = nullptr;
  double link_rate = 50e9;       // EMA of fetch H2D bytes/s
  double scan_rate = 6e12;       // EMA of the GPU scan's vector bytes/s
  bool want_timing = true;       // the current call reports device timings
  uint64_t link_h2d_total = 0, link_d2h_total = 0; // host-link bytes of all searches
  uint64_t fast_vecs(const std::vector<uint32_t>& fast) const {
    uint64_t v = 0;
    for (uint32_t c : fast) v += ix->list_len(c);
    return v;
  }
  // Modeled seconds the batched / single hit scan of these vectors takes.
  double busy_of(const std::vector<uint64_t>& v) const {
    uint64_t t = 0;
    for (uint64_t x : v) t += x;
    return double(t) * ix->d * 4 / scan_rate;
  }
  void note_scan(uint64_t vecs, double t_scan) {
    if (vecs > 0 && t_scan > 0) {
      scan_rate = 0.8 * scan_rate + 0.2 * (double(vecs) * ix->d * 4 / t_scan);
    }
  }
  double cpu_rate = 0;           // EMA of the host miss scan rate on distinct list bytes
  void alloc_scan_set(FastTable& f, ScanOut& o, bool device_outputs = true);
  // The scan's result for query q: the device-merged top-k, or (host-final
  // mode) the k-way merge of the G CTA lists with ids looked up here.
  std::vector<Scored> scan_result(uint32_t q, uint32_t G, int k, uint64_t V) const;
  // Host-link bytes of the scan results of nq queries (G CTAs each): the
  // per-CTA lists (host-final mode) or the device-merged top-k, read from
  // mapped host memory; and of the fetch chunks' result lists.
  uint64_t result_bytes(uint32_t nq, uint32_t G, int k) const {
    const uint64_t e = sizeof(float) + sizeof(uint64_t);
    if (k > kMaxK) return uint64_t(nq) * (k * e + sizeof(uint32_t));
    return host_final ? uint64_t(nq) * G * scan_kk(k, acc_fp64) * e
                      : uint64_t(nq) * (k * e + sizeof(uint32_t));
  }
  uint64_t fetch_result_bytes(size_t nchunks, uint32_t nq, int k) const {
    return uint64_t(nchunks) * nq * (k * (sizeof(float) + sizeof(uint64_t)) + sizeof(uint32_t));
  }

  // GPU schedulers (sched.cu): grown on demand, freed with the context
  struct SchedBufs {
    float* q = nullptr;
    double* dist = nullptr;
    uint64_t* order = nullptr;
    uint64_t* off = nullptr;
    uint32_t* nb = nullptr;
    uint32_t* probes = nullptr;
    unsigned long long* resident = nullptr;
    unsigned long long* overlap = nullptr;
    uint64_t n = 0, L = 0, nw = 0;
  } sb;
  GroupScratch gs{};
  uint64_t dist_n = 0;
  void sched_reserve(uint64_t n, uint64_t L, uint64_t nw) {
    const uint32_t words = (ix->nc + 63) / 64;
    if (n > sb.n) {
      for (void* p : {(void*)sb.q, (void*)sb.order, (void*)sb.off, (void*)sb.nb}) {
        if (p) cudaFree(p);
      }
      sb.q = dev_alloc<float>(n * ix->d);
      sb.order = dev_alloc<uint64_t>(n);
      sb.off = dev_alloc<uint64_t>(n + 1);
      sb.nb = dev_alloc<uint32_t>(1);
    }
    // grouping scratch: the n x n pair matrix up to group_max_queries(), the
    // streaming kernel's O(n) state above
    if (n <= group_max_queries()) {
      if (n > dist_n) {
        if (sb.dist) cudaFree(sb.dist);
        sb.dist = dev_alloc<double>(n * n);
        dist_n = n;
      }
    } else if (n > gs.n) {
      for (void* p : {(void*)gs.taken, (void*)gs.dist_row}) {
        if (p) cudaFree(p);
      }
      gs.taken = dev_alloc<unsigned char>(n);
      gs.dist_row = dev_alloc<double>(n);
      if (!gs.slot_d) {
        gs.slot_d = dev_alloc<double>(2 * kGroupLargeMaxGrid);
        gs.slot_i = dev_alloc<uint32_t>(2 * kGroupLargeMaxGrid);
        gs.bar = dev_alloc<uint64_t>(1);
      }
      gs.n = n;
    }
    if (n * L > sb.n * sb.L || sb.probes == nullptr) {
      if (sb.probes) cudaFree(sb.probes);
      sb.probes = dev_alloc<uint32_t>(std::max<uint64_t>(1, n * L));
    }
    if (n > sb.n || nw > sb.nw) {
      if (sb.resident) cudaFree(sb.resident);
      if (sb.overlap) cudaFree(sb.overlap);
      sb.resident = dev_alloc<unsigned long long>(std::max<uint64_t>(1, nw) * words);
      sb.overlap = dev_alloc<unsigned long long>(std::max<uint64_t>(1, n * nw));
    }
    sb.n = std::max(sb.n, n);
    sb.L = std::max(sb.L, L);
    sb.nw = std::max(sb.nw, nw);
  }
  // ---- size-unbounded paths (wide.cu) ----
  // k > kMaxK: every fast-list member of a query becomes one 64-bit key
  // (score key, datastore-id rank); a radix sort orders them exactly as the
  // reference's partial_sort (ivf.cpp:336-341). Also score_clusters' raw list.
  uint32_t* d_rank_of_row = nullptr; // built on first use
  uint32_t* d_row_of_rank = nullptr;
  uint64_t* d_wkeys = nullptr;
  uint64_t* d_wkeys_alt = nullptr;
  uint64_t wcap = 0;
  void* d_wtmp = nullptr;
  size_t wtmp_bytes = 0;
  float* d_wout_s = nullptr; // [max_batch][wk] device top-k of the wide scan
  uint64_t* d_wout_id = nullptr;
  uint32_t* d_wout_cnt = nullptr;
  float* h_wout_s = nullptr; // pinned copies the host merges from
  uint64_t* h_wout_id = nullptr;
  uint32_t* h_wout_cnt = nullptr;
  int wk = 0;
  float* d_wraw_s = nullptr; // score_clusters raw candidates
  uint64_t* d_wraw_id = nullptr;
  float* h_wraw_s = nullptr;
  uint64_t* h_wraw_id = nullptr;
  uint64_t wraw_cap = 0;
  // nc > kMaxSortNc: ranking by a multi-CTA radix sort per query
  RankScratch rs{};
  bool large_nc() const { return ix->nc > kMaxSortNc; }
  void wide_reserve(uint64_t V, int k);
  void wide_raw_reserve(uint64_t V);
  // Top-k of nq queries over their fast lists (table f over `slab`, V[q]
  // members each) for any k: results to d_wout_* [q * k], fcount_out[q]
  // (nullable) gets the partition's fast-list count.
  void scan_wide(const float* dQ, uint32_t nq, const FastTable& f, const float* slab,
                 const std::vector<uint64_t>& V, int k, uint32_t* fcount_out, cudaStream_t st);
  // score_clusters (ivf.cpp:301-324): the raw candidate list of one query
  // over `cl` in order; resident lists scored on the GPU, the rest by the
  // host at the same time. Returns the candidate count.
  uint64_t score_clusters(const float* hq, const uint32_t* cl, uint32_t n, uint64_t cap,
                          float* s_out, uint64_t* id_out);
  // d_wout_* of nq queries -> the pinned h_wout_* scan_result reads.
  void wide_results(uint32_t nq, int k, cudaStream_t st);
  // First n_out entries of each query's coarse ranking into `order` (device),
  // with the residency split into ft when `part`.
  void select_order(const double* scores, uint32_t nq, uint32_t n_out, uint32_t* order, bool part,
                    cudaStream_t st, bool scan_sorted) {
    if (!large_nc()) {
      launch_select(scores, nq, ix->nc, ix->metric, n_out, order, d_run_k, d_run_v,
                    part ? d_res : nullptr, part ? d_list_off : nullptr, part ? &ft : nullptr, st,
                    scan_sorted);
      return;
    }
    launch_rank_large(scores, nq, ix->nc, ix->metric, n_out, order, rs, st);
    if (part) launch_partition(order, nq, n_out, d_res, d_list_off, ft, st);
  }
  int part_cap = 0; // partial top-k rows available (CTAs x queries)
  float* h_Q = nullptr;
  const float* volatile* h_qslot = nullptr; // staged-query source of the captured chain (mapped)
  const float* const* dm_qslot = nullptr;
  uint32_t* h_order = nullptr;
  float* h_out_s = nullptr;
  uint64_t* h_out_id = nullptr;
  uint32_t* h_out_cnt = nullptr;
  uint32_t* h_fcount = nullptr;
  float* h_cta_s = nullptr;      // host-final grid merge input [part_cap][kMaxK]
  unsigned long long* h_probe = nullptr; // LAIVG_SCAN_PROBE stamps [part_cap][4]
  void print_probe(uint32_t nq, uint32_t G) const {
    for (uint32_t q = 0; q < nq; ++q) {
      const unsigned long long* p = h_probe + size_t(q) * G * 4;
      unsigned long long t0 = ~0ull, e_max = 0, f_min = ~0ull, f_max = 0, l_min = ~0ull, l_max = 0,
                         x_max = 0;
      for (uint32_t b = 0; b < G; ++b) t0 = std::min(t0, p[b * 4]);
      for (uint32_t b = 0; b < G; ++b) {
        e_max = std::max(e_max, p[b * 4] - t0);
        f_min = std::min(f_min, p[b * 4 + 1] - t0);
        f_max = std::max(f_max, p[b * 4 + 1] - t0);
        l_min = std::min(l_min, p[b * 4 + 2] - t0);
        l_max = std::max(l_max, p[b * 4 + 2] - t0);
        x_max = std::max(x_max, p[b * 4 + 3] - t0);
      }
      std::vector<unsigned long long> epi(G);
      for (uint32_t b = 0; b < G; ++b) epi[b] = p[b * 4 + 3] - p[b * 4 + 2];
      std::sort(epi.begin(), epi.end());
      std::fprintf(stderr,
                   "[laivg] scan probe q%u G=%u (us from first CTA entry): entry<=%.2f "
                   "first tile %.2f..%.2f loop end %.2f..%.2f done %.2f epilogue p50 %.2f max "
                   "%.2f\n",
                   q, G, e_max / 1e3, f_min / 1e3, f_max / 1e3, l_min / 1e3, l_max / 1e3,
                   x_max / 1e3, epi[G / 2] / 1e3, epi[G - 1] / 1e3);
    }
  }
  uint64_t* h_cta_r = nullptr;
  bool host_final = false;
  uint32_t* dm_order = nullptr; // device aliases of the mapped buffers above
  float* dm_out_s = nullptr;
  uint64_t* dm_out_id = nullptr;
  uint32_t* dm_out_cnt = nullptr;
  uint32_t* dm_fcount = nullptr;
  float* d_staged = nullptr;
  uint32_t n_staged = 0;
  std::vector<float> staged_host;

  // events
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_p = nullptr, ev_s = nullptr, ev_c = nullptr,
              ev_probe = nullptr, ev_base = nullptr, ev_win = nullptr, ev_cp0 = nullptr,
              ev_cp1 = nullptr, ev_copy_tail = nullptr, ev_comp_tail = nullptr;

  std::unique_ptr<ThreadPool> pool;

  ~Ctx();
  void init(const Index* index, const laivg_opts& o);

  // ---- residency -----------------------------------------------------------
  // Uploads the residency table if it changed; returns the bytes copied.
  uint64_t commit_res(cudaStream_t st) {
    if (!res_dirty) return 0;
    const int s = res_slot;
    res_slot ^= 1;
    CK(cudaEventSynchronize(res_ev[s]));
    std::memcpy(res_stage[s], h_res.data(), h_res.size() * sizeof(int64_t));
    CK(cudaMemcpyAsync(d_res, res_stage[s], h_res.size() * sizeof(int64_t),
                       cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(res_ev[s], st));
    res_dirty = false;
    return h_res.size() * sizeof(int64_t);
  }
  // Copy-stream work issued after this point is ordered after all compute
  // work issued so far (scans may still read slab regions being reused).
  void copy_after_comp() {
    CK(cudaEventRecord(ev_comp_tail, comp));
    CK(cudaStreamWaitEvent(copy, ev_comp_tail, 0));
  }
  void compact();
  // TieredStore::insert + payload upload on the copy stream (no sync).
  void insert_async(uint32_t c, int tag);
  // insert_async that, inside a peer epoch, returns false instead of
  // compacting when the slab is too fragmented for the list
  bool try_insert_async(uint32_t c, int tag);
  uint64_t evict(uint32_t c);
  void clear_store();

  // ---- peer caches ------------------------------------
  // During an epoch this context's resident lists are published to peers,
  // which may copy them out of the slab: evicted ranges are quarantined (not
  // reused) and the slab is not compacted until the epoch closes.
  bool epoch = false;
  std::vector<uint8_t> pinned; // the lists published at epoch open
  std::vector<std::pair<uint64_t, uint64_t>> quarantine; // (vector offset, count)
  uint64_t quarantined = 0;                              // reference bytes held back
  struct Peer {
    const float* slab = nullptr; // the peer's slab (same process or CUDA IPC)
    int dev = -1;                // CUDA ordinal the slab lives on
    void* ipc = nullptr;         // cudaIpcOpenMemHandle mapping to close
    std::vector<int64_t> off;    // the peer's published offsets (-1 absent)
  };
  std::vector<Peer> peers;
  // Publishes (pins) every list resident now: until the epoch closes a
  // pinned list keeps its slab range (an eviction quarantines it, the hotness
  // policy passes over it) and the slab is not compacted. Lists inserted
  // during the epoch are not published and churn as usual.
  void epoch_open() {
    pinned.assign(ix->nc, 0);
    for (auto& [c, r] : resident) pinned[c] = 1;
    epoch = true;
  }
  void epoch_close() {
    for (auto& [o, n] : quarantine) alloc.release(o, n);
    quarantine.clear();
    quarantined = 0;
    for (auto& p : peers) p.off.clear();
    pinned.clear();
    epoch = false;
  }
  bool is_pinned(uint32_t c) const { return epoch && !pinned.empty() && pinned[c]; }
  uint64_t free_bytes() const { return capacity - used - quarantined; }

  // ---- search --------------------------------------------------------------
  bool use_tc(uint32_t nq, uint32_t n_out) const {
    if (coarse_impl == 1 || !tc_ok || n_out == 0) return false;
    if (coarse_impl == 2) return true;
    return nq >= kTcMinBatch && n_out < ix->nc;
  }
  // Coarse ranking prefix of nq queries into d_order[q * n_out + i]; with
  // `part`, also the residency split into ft (ft.grid scan CTAs per query).
  void coarse(const float* dQ, uint32_t nq, uint32_t n_out, cudaStream_t st, bool part = false,
              bool need_scores = false);
  struct Result {
    std::vector<Scored> top;
    std::vector<uint32_t> fast, slow;
    double t_g = 0, t_c = 0, t_2 = 0, t_coarse = 0, t_scan = 0;
    double t_kernel = 0; // fused single-query kernel (events), 0 for the chain
    uint64_t vecs_gpu = 0, bytes_gpu = 0;
    uint32_t fetch_lists = 0, peer_lists = 0;
    uint64_t fetch_bytes = 0, peer_bytes = 0;
    double t_fetch = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0; // host-link bytes of this call
  };
  // One query: dq on device, hq on host (miss path). With `explicit_probe`
  // the probe is those clusters (search_clusters), otherwise the coarse
  // quantizer picks min(L, nc) of them (hybrid/ivf search).
  Result search(const float* dq, const float* hq, int L, int k,
                const std::vector<uint32_t>* explicit_probe);
  // Batched hybrid search of nq <= max_batch queries (dQ on device, hQ on
  // host): one coarse + partition launch and one scan launch for the batch,
  // the misses scanned list-major on the host while the GPU scans the hits.
  struct BatchResult {
    std::vector<std::vector<Scored>> top;
    std::vector<uint32_t> nfast, nslow;
    double t_g = 0, t_c = 0, t_2 = 0, t_coarse = 0, t_scan = 0;
    uint64_t vecs_gpu = 0, bytes_gpu = 0;
    // runtime fetch: misses scanned on the GPU after an on-demand H2D
    uint32_t fetch_lists = 0, cpu_lists = 0, peer_lists = 0;
    uint64_t fetch_bytes = 0, cpu_query_bytes = 0, peer_bytes = 0;
    double t_fetch = 0; // copy-stream time of the fetch copies
    uint64_t h2d_bytes = 0, d2h_bytes = 0; // host-link bytes of this call
    uint32_t list_scan = 0;                // hits ran on the list-major scan
    uint64_t distinct_bytes = 0;           // 4·d·n over distinct resident probed lists
  };
  BatchResult search_batch(const float* dQ, const float* hQ, uint32_t nq, int L, int k);
  // The GPU side of the miss path, shared by both searches: peer-resident
  // misses, then runtime fetch of host lists (rate model), copied through
  // the ring and scanned there; slow[q] loses what goes to the GPU. Returns
  // the chunks issued (results in h_fetch_*, ev_fdone after the last scan).
  struct FetchStats {
    uint32_t fetch_lists = 0, peer_lists = 0;
    uint64_t fetch_bytes = 0, peer_bytes = 0;
    double t_fetch = 0;
  };
  // gpu_busy: modeled seconds the GPU still spends scanning the hits once the
  // probe is known (the host scans misses for free during that time)
  size_t issue_fetch(std::vector<std::vector<uint32_t>>& slow, bool& any_slow, double gpu_busy,
                     const float* dQ,
                     uint32_t nq, uint32_t lp, const uint32_t* probe_dev, int k, int G,
                     FetchStats& st);
  void merge_fetch(uint32_t q, size_t nchunks, int k, std::vector<Scored>& gpu) const;
  void finish_fetch(size_t nchunks, FetchStats& st);

  // ---- generation window (execute_prefetch / prefetch_batch / window) ----
  // With a load buffer set (laivg_window_load), the window streams it like a
  // memory-bound decode (one full read per token period) instead of idling.
  float* d_wbuf = nullptr;
  uint64_t wbuf_bytes = 0;
  double w_rate = 0;                       // target read rate, bytes/s
  float* d_wsink = nullptr;
  unsigned long long* d_wread = nullptr;   // bytes the last window read
  void launch_window_any(double seconds) {
    if (!(seconds > 0)) return;
    if (d_wbuf && w_rate > 0) {
      CK(cudaMemsetAsync(d_wread, 0, sizeof(unsigned long long), comp));
      const uint64_t period = uint64_t(double(wbuf_bytes) / w_rate * 1e9);
      launch_window_stream(d_wbuf, wbuf_bytes, uint64_t(seconds * 1e9), std::max<uint64_t>(1, period),
                           sms, d_wsink, d_wread, comp);
    } else {
      launch_window(uint64_t(seconds * 1e9), sms, comp);
    }
  }
  // Read rate of the last window (after it completed), GB/s.
  double window_read_gbps(double window_s) {
    if (!d_wbuf || !(w_rate > 0) || !(window_s > 0)) return 0.0;
    unsigned long long b = 0;
    CK(cudaMemcpy(&b, d_wread, sizeof(b), cudaMemcpyDeviceToHost));
    return double(b) / window_s / 1e9;
  }

  // ---- fused single-query kernel (one cooperative launch per query) ----
  bool fused_on = true;               // opts.single_chain == 0
  uint64_t* d_keys = nullptr;         // [nc] order keys of the coarse scores
  unsigned* d_ctl = nullptr;          // [2] grid barrier word, call sequence
  unsigned* h_flag = nullptr;         // mapped: sequence number once the probe is out
  unsigned* dm_flag = nullptr;
  unsigned long long* h_stamps = nullptr; // mapped [6] phase stamps of CTA 0
  unsigned long long* dm_stamps = nullptr;
  unsigned long long* h_cta_stamps = nullptr; // LAIVG_SCAN_PROBE: [sms][3]
  unsigned long long* dm_cta_stamps = nullptr;
  unsigned fused_seq = 0;             // launches of the fused kernel executed
  bool last_fused = false;            // the last single-query chain was fused
  std::map<uint64_t, size_t> fused_fit; // (L, k) -> smem (0: does not fit)
  bool use_fused(uint32_t lp, int k, int G) {
    if (!fused_on || large_nc() || scan_impl != ScanImpl::kTma || G > sms || k > kMaxK) {
      return false;
    }
    const uint64_t key = (uint64_t(lp) << 32) | uint32_t(k);
    auto it = fused_fit.find(key);
    if (it == fused_fit.end()) {
      it = fused_fit.emplace(key, fused_query_smem(ix->nc, ix->d, lp, k, acc_fp64, uint32_t(G),
                                                   tune)).first;
    }
    return it->second != 0;
  }
  // Waits until the fused kernel of call `seq` has published its probe
  // (word 0) or all of its results (word 1).
  void wait_probe_flag(unsigned seq, int word = 0) {
    const volatile unsigned* f = h_flag + word;
    uint32_t spins = 0;
    while (*f != seq) {
      if ((++spins & 0x3fffu) == 0) {
        const cudaError_t e = cudaStreamQuery(comp);
        if (e == cudaSuccess) {
          if (*f == seq) break;
          throw std::runtime_error("fused query kernel finished without publishing its probe");
        }
        if (e != cudaErrorNotReady) throw CudaError(cudaGetErrorString(e));
      }
    }
  }

  // ---- the coarse -> select -> scan chain as one CUDA graph per (L, k) ----
  bool use_graphs = std::getenv("LAIVG_GRAPHS") ? std::atoi(std::getenv("LAIVG_GRAPHS")) != 0 : true;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr; // capture-internal fork/join
  bool capturing = false;
  // Timing events stay host-visible inside a captured graph (external record
  // nodes); the external flag is only legal while capturing.
  void rec(cudaEvent_t e, cudaStream_t st) {
    if (capturing) CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CK(cudaEventRecord(e, st));
  }
  // The scan's final CTA wrote the results (and the fast-list count) into
  // mapped host memory; completion (event synchronize) orders those writes
  // before the host reads them.
  void enqueue_results(int) { rec(ev_c, comp); }
  // The chain's first node, a one-CTA kernel, copies the query into d_Q:
  // from the pinned staging row h_Q (a fixed argument), or from whatever a
  // mapped pointer slot holds (staged HBM rows, which change per call). Both
  // graphs keep fixed parameters: a memcpy node costs 2-4 us more launch and
  // re-pointing a node per call ~4 us plus a slower launch. Then coarse
  // scores, ranking + residency split, scan, results; the probe lands in
  // mapped host memory as soon as it exists.
  void enqueue_coarse_path(uint32_t lp, int k, int G, const float* src,
                           PhaseTrace* tr = nullptr) {
    if (use_fused(lp, k, G)) {
      // launched directly (not captured): the query row is a kernel
      // argument. A staged row (HBM) is read by every CTA; the pinned host
      // row once by CTA 0 (a read of mapped host memory costs microseconds).
      FusedQuery fq;
      fq.src = src;
      fq.qdirect = src != h_Q || std::getenv("LAIVG_FUSED_QDIRECT") ? 1 : 0;
      fq.dQ = d_Q;
      fq.cen = d_cen;
      fq.nc = ix->nc;
      fq.d = ix->d;
      fq.L = lp;
      fq.metric = ix->metric;
      fq.k = k;
      fq.keys = d_keys;
      fq.res_off = d_res;
      fq.list_off = d_list_off;
      fq.order_out = dm_order;
      fq.fcount_out = dm_fcount;
      fq.flag_out = dm_flag;
      fq.done_out = dm_flag + 1;
      fq.ctl = d_ctl;
      fq.stamps = dm_stamps;
      fq.cta_stamps = dm_cta_stamps;
      fq.slab = d_slab;
      fq.ids = d_ids;
      fq.grid = uint32_t(G);
      if (tr) tr->mark("prep");
      rec(ev_a, comp);
      if (tr) tr->mark("ev_a");
      launch_fused_query(fq, so, acc_fp64, tune, comp);
      if (tr) tr->mark("kernel");
      rec(ev_s, comp); // also marks the results in mapped host memory complete
      return;
    }
    if (src == h_Q) {
      launch_fetch_query(h_Q, nullptr, d_Q, ix->d, comp);
    } else {
      *h_qslot = src;
      launch_fetch_query(nullptr, dm_qslot, d_Q, ix->d, comp);
    }
    rec(ev_a, comp);
    launch_coarse_scores(d_Q, 1, d_cen, ix->nc, ix->d, ix->metric, d_scores, comp);
    if (large_nc()) {
      select_order(d_scores, 1, lp, d_order, /*part=*/true, comp, false);
      CK(cudaMemcpyAsync(h_order, d_order, size_t(lp) * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                         comp));
    } else {
      launch_select(d_scores, 1, ix->nc, ix->metric, lp, dm_order, d_run_k, d_run_v, d_res,
                    d_list_off, &ft, comp);
    }
    rec(ev_b, comp);
    launch_scan(d_Q, 1, ix->d, ix->metric, k, ft, d_slab, d_ids, so, G, acc_fp64, scan_impl,
                tune, comp);
    rec(ev_s, comp); // also marks the results in mapped host memory complete
  }
  struct GraphEntry {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    uint64_t kernels = 0; // kernel nodes (launch accounting)
  };
  std::map<uint64_t, GraphEntry> graph_tab;
  void run_coarse_path(uint32_t lp, int k, int G, const float* src, PhaseTrace* tr = nullptr) {
    const bool staged = src != h_Q;
    last_fused = use_fused(lp, k, G);
    if (last_fused) {
      ++fused_seq; // this call executes one fused launch
      // host row (fixed arguments): a captured graph of event + kernel +
      // event; a staged row is a per-call argument: direct launch
      static const bool fgraph =
          std::getenv("LAIVG_FUSED_GRAPH") ? std::atoi(std::getenv("LAIVG_FUSED_GRAPH")) != 0 : true;
      if (!fgraph || staged || !use_graphs) {
        enqueue_coarse_path(lp, k, G, src, tr);
        return;
      }
      const uint64_t key = (1ull << 63) | (uint64_t(lp) << 33) | (uint64_t(uint32_t(k)) << 1);
      auto it = graph_tab.find(key);
      if (it != graph_tab.end()) {
        CK(cudaGraphLaunch(it->second.ge, comp));
        launch_counter() += it->second.kernels;
        if (tr) tr->mark("kernel");
        return;
      }
      enqueue_coarse_path(lp, k, G, src, tr); // runs this call, sets attributes
      GraphEntry e;
      const uint64_t launched = launch_counter().load();
      bool ok = cudaStreamBeginCapture(comp, cudaStreamCaptureModeRelaxed) == cudaSuccess;
      if (ok) {
        capturing = true;
        try {
          enqueue_coarse_path(lp, k, G, src);
        } catch (...) {
          ok = false;
        }
        capturing = false;
        ok = (cudaStreamEndCapture(comp, &e.g) == cudaSuccess) && ok && e.g != nullptr;
      }
      e.kernels = launch_counter().load() - launched;
      launch_counter() = launched; // captured launches did not run
      ok = ok && cudaGraphInstantiate(&e.ge, e.g, 0) == cudaSuccess;
      ok = ok && cudaGraphUpload(e.ge, comp) == cudaSuccess;
      cudaGetLastError();
      if (ok) {
        graph_tab[key] = e;
      } else {
        if (e.g) cudaGraphDestroy(e.g);
        use_graphs = false; // capture unsupported here: stay eager
      }
      return;
    }
    if (staged) *h_qslot = src; // read by the chain's first kernel
    const uint64_t key = (uint64_t(lp) << 33) | (uint64_t(uint32_t(k)) << 1) | (staged ? 1 : 0);
    auto it = graph_tab.find(key);
    if (it == graph_tab.end() && use_graphs) {
      // first call for this shape runs eagerly (sets kernel attributes), then
      // the chain is captured for the following calls
      enqueue_coarse_path(lp, k, G, src);
      GraphEntry e;
      const uint64_t launched = launch_counter().load();
      bool ok = cudaStreamBeginCapture(comp, cudaStreamCaptureModeRelaxed) == cudaSuccess;
      if (ok) {
        capturing = true;
        try {
          enqueue_coarse_path(lp, k, G, src);
        } catch (...) {
          ok = false;
        }
        capturing = false;
        ok = (cudaStreamEndCapture(comp, &e.g) == cudaSuccess) && ok && e.g != nullptr;
      }
      e.kernels = launch_counter().load() - launched;
      launch_counter() = launched; // captured launches did not run
      ok = ok && cudaGraphInstantiate(&e.ge, e.g, 0) == cudaSuccess;
      ok = ok && cudaGraphUpload(e.ge, comp) == cudaSuccess;
      cudaGetLastError();
      if (ok) {
        graph_tab[key] = e;
      } else {
        if (e.g) cudaGraphDestroy(e.g);
        use_graphs = false; // capture unsupported here: stay eager
      }
      return;
    }
    if (it != graph_tab.end()) {
      if (tr) tr->mark("glookup");
      CK(cudaGraphLaunch(it->second.ge, comp));
      launch_counter() += it->second.kernels;
      return;
    }
    enqueue_coarse_path(lp, k, G, src);
  }
};


Ctx::~Ctx() {
  if (comp) cudaStreamSynchronize(comp);
  if (copy) cudaStreamSynchronize(copy);
  if (aux) cudaStreamSynchronize(aux);
  for (void* p : {(void*)d_cen, (void*)d_list_off, (void*)d_ids, (void*)d_res,
                  (void*)d_slab, (void*)d_tmp, (void*)d_Q, (void*)d_scores,
                  (void*)d_order, (void*)d_run_k, (void*)d_run_v, (void*)ft.slab, (void*)ft.row, (void*)ft.len,
                  (void*)ft.cluster, (void*)ft.pre, (void*)ft.count, (void*)ft.cta,
                  (void*)so.part_s, (void*)so.part_id, (void*)so.part_vi, (void*)so.ticket,
                  (void*)so.gpart_s, (void*)so.gpart_id, (void*)so.gpart_vi,
                  (void*)d_staged, (void*)d_approx, (void*)d_cnorm, (void*)d_keys,
                  (void*)tcs.cand, (void*)tcs.key, (void*)tcs.ncand, (void*)tcs.qmask,
                  (void*)lss.qcount, (void*)lss.lists, (void*)lss.lq_off, (void*)lss.item_off,
                  (void*)lss.qidx, (void*)lss.meta, (void*)lss.gtau, (void*)lss.gcnt, lss.cand,
                  (void*)d_ctl, (void*)d_wbuf, (void*)d_wsink, (void*)d_wread}) {
    if (p) cudaFree(p);
  }
  for (void* p : {(void*)res_stage[0], (void*)res_stage[1], (void*)h_Q, (void*)h_qslot,
                  (void*)h_order, (void*)h_out_s, (void*)h_out_id,
                  (void*)h_out_cnt, (void*)h_fcount, (void*)h_flag, (void*)h_stamps,
                  (void*)h_cta_stamps, (void*)h_ls_flag}) {
    if (p) cudaFreeHost(p);
  }
  for (void* p : {(void*)fft.slab, (void*)fft.row, (void*)fft.len, (void*)fft.cluster,
                  (void*)fft.pre, (void*)fft.count, (void*)fft.cta, (void*)fso.part_s,
                  (void*)fso.part_id, (void*)fso.part_vi, (void*)fso.ticket, (void*)fso.gpart_s,
                  (void*)fso.gpart_id, (void*)fso.gpart_vi, (void*)fso.out_s,
                  (void*)fso.out_id, (void*)fso.out_count, (void*)d_ring,
                  (void*)d_res_ring[0], (void*)d_res_ring[1]}) {
    if (p) cudaFree(p);
  }
  for (void* p : {(void*)h_res_ring, (void*)h_fetch_s, (void*)h_fetch_id, (void*)h_fetch_cnt,
                  (void*)h_cta_s, (void*)h_cta_r, (void*)h_probe}) {
    if (p) cudaFreeHost(p);
  }
  for (cudaEvent_t e : {ev_landed[0], ev_landed[1], ev_freed[0], ev_freed[1], ev_f0, ev_f1,
                        ev_fdone}) {
    if (e) cudaEventDestroy(e);
  }
  for (void* p : {(void*)sb.q, (void*)sb.dist, (void*)sb.order, (void*)sb.off, (void*)sb.nb,
                  (void*)sb.probes, (void*)sb.resident, (void*)sb.overlap, (void*)gs.taken,
                  (void*)gs.dist_row, (void*)gs.slot_d, (void*)gs.slot_i, gs.bar}) {
    if (p) cudaFree(p);
  }
  for (void* p : {(void*)d_rank_of_row, (void*)d_row_of_rank, (void*)d_wkeys, (void*)d_wkeys_alt,
                  (void*)d_wtmp, (void*)d_wout_s, (void*)d_wout_id, (void*)d_wout_cnt,
                  (void*)d_wraw_s, (void*)d_wraw_id, (void*)rs.keys, (void*)rs.keys_alt,
                  (void*)rs.vals, (void*)rs.vals_alt, rs.tmp}) {
    if (p) cudaFree(p);
  }
  for (void* p : {(void*)h_wout_s, (void*)h_wout_id, (void*)h_wout_cnt, (void*)h_wraw_s,
                  (void*)h_wraw_id}) {
    if (p) cudaFreeHost(p);
  }
  for (auto& p : peers) {
    if (p.ipc) cudaIpcCloseMemHandle(p.ipc);
  }
  for (auto& [key, e] : graph_tab) {
    if (e.ge) cudaGraphExecDestroy(e.ge);
    if (e.g) cudaGraphDestroy(e.g);
  }
  for (cudaEvent_t e : {ev_a, ev_b, ev_p, ev_s, ev_c, ev_probe, ev_base, ev_win,
                        ev_cp0, ev_cp1, ev_copy_tail, ev_comp_tail, res_ev[0],
                        res_ev[1], ev_fork, ev_join}) {
    if (e) cudaEventDestroy(e);
  }
  if (comp) cudaStreamDestroy(comp);
  if (copy) cudaStreamDestroy(copy);
  if (aux) cudaStreamDestroy(aux);
}

void Ctx::init(const Index* index, const laivg_opts& o) {
  ix = index;
  dev = o.device;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (dev < 0 || dev >= ndev) {
    throw CudaError("device ordinal " + std::to_string(dev) + " not present (" +
                    std::to_string(ndev) + " devices)");
  }
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) {
    throw CudaError(std::string("device is ") + prop.name +
                    " (sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                    "); this build targets sm_100a");
  }
  sms = prop.multiProcessorCount;
  acc_fp64 = o.acc_fp64 != 0;
  if (o.scan_impl > 1) throw std::invalid_argument("scan_impl must be 0 (TMA) or 1 (LDG)");
  scan_impl = static_cast<ScanImpl>(o.scan_impl);
  tune.tile = o.tma_tile;
  tune.stages = o.tma_stages;
  tune.ctas_per_sm = o.ctas_per_sm;
  if (o.ctas_per_sm > 6) throw std::invalid_argument("ctas_per_sm must be <= 6");
  CK(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&ev_a, &ev_b, &ev_p, &ev_s, &ev_c, &ev_probe, &ev_base,
                         &ev_win, &ev_cp0, &ev_cp1, &ev_copy_tail, &ev_comp_tail,
                         &res_ev[0], &res_ev[1], &ev_fork, &ev_join}) {
    CK(cudaEventCreate(e));
  }
  CK(cudaEventRecord(ev_copy_tail, copy));
  CK(cudaEventRecord(res_ev[0], copy));
  CK(cudaEventRecord(res_ev[1], copy));

  const uint32_t nc = ix->nc, d = ix->d;
  d_cen = dev_alloc<float>(size_t(nc) * d);
  CK(cudaMemcpy(d_cen, ix->centroids.data(), size_t(nc) * d * sizeof(float),
                cudaMemcpyHostToDevice));
  d_list_off = dev_alloc<uint64_t>(nc + 3); // padded: the fused kernel bulk-copies 16 B multiples
  CK(cudaMemcpy(d_list_off, ix->list_off.data(), (nc + 1) * sizeof(uint64_t),
                cudaMemcpyHostToDevice));
  d_ids = dev_alloc<uint64_t>(ix->total());
  if (ix->total()) {
    CK(cudaMemcpy(d_ids, ix->ids, ix->total() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  }

  capacity = o.capacity_bytes;
  h_res.assign(nc, -1);
  d_res = dev_alloc<int64_t>(nc + 2); // padded (see d_list_off)
  res_stage[0] = pin_alloc<int64_t>(nc);
  res_stage[1] = pin_alloc<int64_t>(nc);
  slab_vecs = capacity / ix->member_bytes();
  d_slab = dev_alloc<float>(slab_vecs * d);
  alloc.reset(slab_vecs);
  uint64_t maxlen = 1;
  for (uint32_t c = 0; c < nc; ++c) maxlen = std::max(maxlen, ix->list_len(c));
  tmp_vecs = maxlen;

  coarse_impl = o.coarse_impl;
  if (coarse_impl > 2) throw std::invalid_argument("coarse_impl must be 0 (auto), 1 or 2");
  tc_ok = coarse_tc_supported(nc, d);
  if (coarse_impl == 2 && !tc_ok) {
    throw std::invalid_argument("tensor-core coarse quantizer needs d % 4 == 0 and nc <= " +
                                std::to_string(kTcMaxNc));
  }
  max_batch = o.max_batch ? o.max_batch : 256;
  max_probe = o.max_probe ? std::min(o.max_probe, nc) : nc;
  if (max_probe == 0) max_probe = 1;
  d_Q = dev_alloc<float>(size_t(max_batch) * d);
  if (tc_ok) {
    d_approx = dev_alloc<float>(size_t(kTcMaxSplit) * max_batch * nc);
    std::vector<float> cn(nc);
    for (uint32_t c = 0; c < nc; ++c) {
      double s2 = 0.0;
      for (uint32_t j = 0; j < d; ++j) {
        const double x = ix->centroids[size_t(c) * d + j];
        s2 += x * x;
      }
      cn[c] = std::nextafter(static_cast<float>(std::sqrt(s2) * (1.0 + 1e-9)), INFINITY);
    }
    d_cnorm = dev_alloc<float>(nc);
    CK(cudaMemcpy(d_cnorm, cn.data(), nc * sizeof(float), cudaMemcpyHostToDevice));
    if (!std::getenv("LAIVG_TC_SELECT1")) { // (A/B: the single-kernel selection)
      uint32_t cap = 2;
      while (cap < nc) cap <<= 1;
      tcs.cand = dev_alloc<uint32_t>(size_t(max_batch) * cap);
      tcs.key = dev_alloc<uint64_t>(size_t(max_batch) * cap);
      tcs.ncand = dev_alloc<uint32_t>(max_batch);
      tcs.qmask = dev_alloc<uint32_t>(size_t((max_batch + 31) / 32) * nc);
    }
  }
  d_scores = dev_alloc<double>(size_t(max_batch) * nc);
  d_order = dev_alloc<uint32_t>(size_t(max_batch) * std::max(nc, 1u));
  if (!large_nc()) {
    d_run_k = dev_alloc<uint64_t>(select_scratch_entries(max_batch, nc));
    d_run_v = dev_alloc<uint32_t>(select_scratch_entries(max_batch, nc));
  } else {
    const size_t n = size_t(max_batch) * nc;
    rs.keys = dev_alloc<uint64_t>(n);
    rs.keys_alt = dev_alloc<uint64_t>(n);
    rs.vals = dev_alloc<uint32_t>(n);
    rs.vals_alt = dev_alloc<uint32_t>(n);
    rs.tmp_bytes = rank_large_temp_bytes(nc);
    rs.tmp = dev_alloc<unsigned char>(rs.tmp_bytes);
  }
  const int per_sm = std::max<int>(2, int(tune.ctas_per_sm));
  part_cap = std::max<int>(per_sm * sms, int(max_batch)) + per_sm * sms;
  alloc_scan_set(ft, so, /*device_outputs=*/false);
  miss_fetch = o.miss_fetch;
  if (miss_fetch > 2) throw std::invalid_argument("miss_fetch must be 0, 1 or 2");
  if (miss_fetch) {
    const uint64_t chunk_mb = o.fetch_chunk_mb ? o.fetch_chunk_mb : 512;
    ring_vecs = std::max<uint64_t>(maxlen, (chunk_mb << 20) / (uint64_t(d) * 4));
    d_ring = dev_alloc<float>(2 * ring_vecs * d);
    for (int i = 0; i < 2; ++i) {
      d_res_ring[i] = dev_alloc<int64_t>(nc);
      CK(cudaEventCreate(&ev_landed[i]));
      CK(cudaEventCreate(&ev_freed[i]));
      CK(cudaEventRecord(ev_freed[i], comp));
    }
    CK(cudaEventCreate(&ev_f0));
    CK(cudaEventCreate(&ev_f1));
    CK(cudaEventCreate(&ev_fdone));
    h_res_ring = pin_alloc<int64_t>(size_t(kMaxFetchChunks) * nc);
    alloc_scan_set(fft, fso);
    h_fetch_cnt = pin_alloc<uint32_t>(size_t(kMaxFetchChunks) * max_batch);
  }
  {
    // the query staging rows: written by the host, read only by the GPU (a
    // kernel or a copy), so write-combined (PCIe reads need no CPU snoop)
    void* p = nullptr;
    const unsigned fl = std::getenv("LAIVG_HQ_NOWC") ? cudaHostAllocPortable
                                                    : (cudaHostAllocPortable | cudaHostAllocWriteCombined);
    CK(cudaHostAlloc(&p, std::max<size_t>(1, size_t(max_batch) * d) * sizeof(float), fl));
    h_Q = static_cast<float*>(p);
  }
  h_order = pin_alloc_mapped<uint32_t>(size_t(max_batch) * std::max(nc, 1u), &dm_order);
  {
    const float** dslot = nullptr;
    h_qslot = pin_alloc_mapped<const float*>(1, &dslot);
    dm_qslot = dslot;
  }
  h_out_s = pin_alloc_mapped<float>(size_t(max_batch) * kMaxK, &dm_out_s);
  h_out_id = pin_alloc_mapped<uint64_t>(size_t(max_batch) * kMaxK, &dm_out_id);
  h_out_cnt = pin_alloc_mapped<uint32_t>(max_batch, &dm_out_cnt);
  h_fcount = pin_alloc_mapped<uint32_t>(max_batch, &dm_fcount);
  fused_on = o.single_chain == 0 && !std::getenv("LAIVG_CHAIN");
  d_keys = dev_alloc<uint64_t>(std::max(nc, 1u));
  d_ctl = dev_alloc<unsigned>(3);
  CK(cudaMemset(d_ctl, 0, 3 * sizeof(unsigned)));
  h_flag = pin_alloc_mapped<unsigned>(2, &dm_flag); // [0] probe out, [1] results out
  h_flag[0] = h_flag[1] = 0;
  h_stamps = pin_alloc_mapped<unsigned long long>(32, &dm_stamps);
  if (std::getenv("LAIVG_SCAN_PROBE")) {
    h_cta_stamps = pin_alloc_mapped<unsigned long long>(size_t(sms) * 4, &dm_cta_stamps);
  }
  // the main scan writes its results straight into host memory
  so.out_s = dm_out_s;
  so.out_id = dm_out_id;
  so.out_count = dm_out_cnt;
  so.fcount_in = ft.count;
  so.fcount_out = dm_fcount;
  // fp64 accumulation needs no device re-score: the host merges the scan
  // CTAs' lists (saves the device grid merge chain)
  host_final = acc_fp64 && !(std::getenv("LAIVG_DEVICE_MERGE"));
  if (host_final) {
    float* ds = nullptr;
    uint64_t* dr = nullptr;
    h_cta_s = pin_alloc_mapped<float>(size_t(part_cap) * kMaxK, &ds);
    h_cta_r = pin_alloc_mapped<uint64_t>(size_t(part_cap) * kMaxK, &dr);
    so.cta_s = ds;
    so.cta_r = dr;
  }
  if (std::getenv("LAIVG_SCAN_PROBE")) {
    unsigned long long* dp = nullptr;
    h_probe = pin_alloc_mapped<unsigned long long>(size_t(part_cap) * 4, &dp);
    so.probe = dp;
  }

  unsigned threads = o.miss_threads;
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  pool = std::make_unique<ThreadPool>(threads - 1);
  CK(cudaDeviceSynchronize());
}

void Ctx::alloc_scan_set(FastTable& f, ScanOut& o, bool device_outputs) {
  f.stride = max_probe;
  f.slab = dev_alloc<int64_t>(size_t(max_batch) * max_probe);
  f.row = dev_alloc<uint64_t>(size_t(max_batch) * max_probe);
  f.len = dev_alloc<uint32_t>(size_t(max_batch) * max_probe);
  f.cluster = dev_alloc<uint32_t>(size_t(max_batch) * max_probe);
  f.pre = dev_alloc<uint64_t>(size_t(max_batch) * (max_probe + 1));
  f.count = dev_alloc<uint32_t>(max_batch);
  f.cta = dev_alloc<CtaStart>(size_t(part_cap));
  o.part_s = dev_alloc<float>(size_t(part_cap) * kMaxK);
  o.part_id = dev_alloc<uint64_t>(size_t(part_cap) * kMaxK);
  o.part_vi = dev_alloc<uint32_t>(size_t(part_cap) * kMaxK);
  o.gpart_s = dev_alloc<float>(size_t(max_batch) * kMaxGroups * kMaxK);
  o.gpart_id = dev_alloc<uint64_t>(size_t(max_batch) * kMaxGroups * kMaxK);
  o.gpart_vi = dev_alloc<uint32_t>(size_t(max_batch) * kMaxGroups * kMaxK);
  o.ticket = dev_alloc<unsigned>(size_t(max_batch) * (kMaxGroups + 1));
  CK(cudaMemset(o.ticket, 0, size_t(max_batch) * (kMaxGroups + 1) * sizeof(unsigned)));
  if (device_outputs) {
    o.out_s = dev_alloc<float>(size_t(max_batch) * kMaxK);
    o.out_id = dev_alloc<uint64_t>(size_t(max_batch) * kMaxK);
    o.out_count = dev_alloc<uint32_t>(max_batch);
  }
}

void Ctx::wide_results(uint32_t nq, int k, cudaStream_t st) {
  CK(cudaMemcpyAsync(h_wout_s, d_wout_s, size_t(nq) * k * sizeof(float), cudaMemcpyDeviceToHost,
                     st));
  CK(cudaMemcpyAsync(h_wout_id, d_wout_id, size_t(nq) * k * sizeof(uint64_t),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_wout_cnt, d_wout_cnt, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
}

std::vector<Scored> Ctx::scan_result(uint32_t q, uint32_t G, int k, uint64_t V) const {
  if (k > kMaxK) { // wide path (wide_results copied them)
    std::vector<Scored> g(h_wout_cnt[q]);
    for (uint32_t i = 0; i < h_wout_cnt[q]; ++i) {
      g[i] = {h_wout_s[size_t(q) * k + i], h_wout_id[size_t(q) * k + i]};
    }
    return g;
  }
  const int kk = scan_kk(k, acc_fp64);
  if (!host_final || ls_result) {
    std::vector<Scored> g(h_out_cnt[q]);
    for (uint32_t i = 0; i < h_out_cnt[q]; ++i) {
      g[i] = {h_out_s[size_t(q) * k + i], h_out_id[size_t(q) * k + i]};
    }
    return g;
  }
  // Best `want` of G sorted lists (score, then id: vectorstore.hpp:34-39):
  // one pass over the lists with a sorted buffer; a list is left at its
  // first entry that does not beat the buffer's last (the lists are sorted),
  // so most lists cost one read. Ids are looked up only to break an exact
  // score tie and for the output.
  const size_t base = size_t(q) * G * kk;
  const int metric = ix->metric;
  const uint64_t* idt = ix->ids;
  struct E {
    float s;
    uint64_t row;
  };
  auto before = [&](const E& a, const E& b) { // a ranks before b
    if (a.s != b.s) return metric == kMetricIP ? a.s > b.s : a.s < b.s;
    return idt[a.row] < idt[b.row];
  };
  const size_t want = size_t(std::min<uint64_t>(V, uint64_t(k)));
  E best[kMaxK + 1];
  size_t n = 0;
  for (uint32_t l = 0; l < G && want; ++l) {
    const float* ls = h_cta_s + base + size_t(l) * kk;
    const uint64_t* lr = h_cta_r + base + size_t(l) * kk;
    for (int p = 0; p < kk; ++p) {
      const E e{ls[p], lr[p]};
      if (e.row == ~0ull) break;
      if (n == want && !before(e, best[n - 1])) break;
      size_t i = n < want ? n++ : n - 1; // drop the last when full
      while (i > 0 && before(e, best[i - 1])) {
        best[i] = best[i - 1];
        --i;
      }
      best[i] = e;
    }
  }
  std::vector<Scored> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = {best[i].s, idt[best[i].row]};
  return out;
}

void Ctx::wide_reserve(uint64_t V, int k) {
  if (!d_rank_of_row) {
    const uint64_t n = ix->total();
    d_rank_of_row = dev_alloc<uint32_t>(n);
    d_row_of_rank = dev_alloc<uint32_t>(n);
    build_id_rank(d_ids, n, d_rank_of_row, d_row_of_rank, comp);
  }
  if (V > wcap) {
    for (void* p : {(void*)d_wkeys, (void*)d_wkeys_alt, d_wtmp}) {
      if (p) cudaFree(p);
    }
    // one allocation serves later calls: grow by 1.5x
    wcap = std::max<uint64_t>(V, wcap + wcap / 2);
    d_wkeys = dev_alloc<uint64_t>(wcap);
    d_wkeys_alt = dev_alloc<uint64_t>(wcap);
    wtmp_bytes = wide_sort_temp_bytes(wcap);
    d_wtmp = dev_alloc<unsigned char>(wtmp_bytes);
  }
  if (k > wk) {
    for (void* p : {(void*)d_wout_s, (void*)d_wout_id, (void*)d_wout_cnt}) {
      if (p) cudaFree(p);
    }
    for (void* p : {(void*)h_wout_s, (void*)h_wout_id, (void*)h_wout_cnt}) {
      if (p) cudaFreeHost(p);
    }
    wk = k;
    d_wout_s = dev_alloc<float>(size_t(max_batch) * wk);
    d_wout_id = dev_alloc<uint64_t>(size_t(max_batch) * wk);
    d_wout_cnt = dev_alloc<uint32_t>(max_batch);
    h_wout_s = pin_alloc<float>(size_t(max_batch) * wk);
    h_wout_id = pin_alloc<uint64_t>(size_t(max_batch) * wk);
    h_wout_cnt = pin_alloc<uint32_t>(max_batch);
  }
}

void Ctx::wide_raw_reserve(uint64_t V) {
  if (V <= wraw_cap) return;
  for (void* p : {(void*)d_wraw_s, (void*)d_wraw_id}) {
    if (p) cudaFree(p);
  }
  for (void* p : {(void*)h_wraw_s, (void*)h_wraw_id}) {
    if (p) cudaFreeHost(p);
  }
  wraw_cap = std::max<uint64_t>(V, wraw_cap + wraw_cap / 2);
  d_wraw_s = dev_alloc<float>(wraw_cap);
  d_wraw_id = dev_alloc<uint64_t>(wraw_cap);
  h_wraw_s = pin_alloc<float>(wraw_cap);
  h_wraw_id = pin_alloc<uint64_t>(wraw_cap);
}

void Ctx::scan_wide(const float* dQ, uint32_t nq, const FastTable& f, const float* slab,
                    const std::vector<uint64_t>& V, int k, uint32_t* fcount_out, cudaStream_t st) {
  uint64_t vmax = 0;
  for (uint32_t q = 0; q < nq; ++q) vmax = std::max(vmax, V[q]);
  wide_reserve(vmax, k);
  for (uint32_t q = 0; q < nq; ++q) {
    launch_score_all(dQ + size_t(q) * ix->d, q, ix->d, ix->metric, f, slab, d_rank_of_row, d_ids,
                     V[q], d_wkeys, nullptr, nullptr, sms, st);
    launch_wide_topk(d_wkeys, d_wkeys_alt, V[q], k, ix->metric, d_wtmp, wtmp_bytes,
                     d_row_of_rank, d_ids, d_wout_s + size_t(q) * k, d_wout_id + size_t(q) * k,
                     d_wout_cnt + q, f.count, fcount_out ? fcount_out + q : nullptr, q, st);
  }
}

uint64_t Ctx::score_clusters(const float* hq, const uint32_t* cl, uint32_t n, uint64_t cap,
                             float* s_out, uint64_t* id_out) {
  std::vector<uint64_t> base(size_t(n) + 1, 0);
  for (uint32_t i = 0; i < n; ++i) {
    if (cl[i] >= ix->nc) throw std::invalid_argument("unknown cluster id " + std::to_string(cl[i]));
    base[i + 1] = base[i] + ix->list_len(cl[i]);
  }
  const uint64_t total = base[n];
  if (total > cap) {
    throw std::invalid_argument("score_clusters: " + std::to_string(total) +
                                " candidates exceed the output capacity " + std::to_string(cap));
  }
  if (n == 0 || total == 0) return total;
  if (n > max_probe) {
    throw std::invalid_argument("score_clusters over " + std::to_string(n) +
                                " clusters exceeds the context's max_probe " +
                                std::to_string(max_probe));
  }
  CK(cudaStreamWaitEvent(comp, ev_copy_tail, 0));
  commit_res(comp);
  std::memcpy(h_Q, hq, ix->d * sizeof(float));
  CK(cudaMemcpyAsync(d_Q, h_Q, ix->d * sizeof(float), cudaMemcpyHostToDevice, comp));
  std::memcpy(h_order, cl, n * sizeof(uint32_t));
  CK(cudaMemcpyAsync(d_order, h_order, n * sizeof(uint32_t), cudaMemcpyHostToDevice, comp));
  ft.grid = 1;
  launch_partition(d_order, 1, n, d_res, d_list_off, ft, comp);
  uint64_t vf = 0;
  std::vector<std::pair<uint32_t, uint64_t>> host_items;
  for (uint32_t i = 0; i < n; ++i) {
    if (h_res[cl[i]] >= 0) vf += ix->list_len(cl[i]);
    else host_items.emplace_back(cl[i], base[i]);
  }
  if (vf) {
    wide_raw_reserve(vf);
    launch_score_all(d_Q, 0, ix->d, ix->metric, ft, d_slab, nullptr, d_ids, vf, nullptr, d_wraw_s,
                     d_wraw_id, sms, comp);
    CK(cudaMemcpyAsync(h_wraw_s, d_wraw_s, vf * sizeof(float), cudaMemcpyDeviceToHost, comp));
    CK(cudaMemcpyAsync(h_wraw_id, d_wraw_id, vf * sizeof(uint64_t), cudaMemcpyDeviceToHost, comp));
  }
  CK(cudaEventRecord(ev_c, comp));
  if (!host_items.empty()) score_lists(*ix, hq, host_items, s_out, id_out, *pool);
  CK(cudaEventSynchronize(ev_c));
  // the GPU's list is the resident entries in probe order: place each at
  // its position in the full candidate list
  uint64_t g = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (h_res[cl[i]] < 0) continue;
    const uint64_t len = ix->list_len(cl[i]);
    std::memcpy(s_out + base[i], h_wraw_s + g, len * sizeof(float));
    std::memcpy(id_out + base[i], h_wraw_id + g, len * sizeof(uint64_t));
    g += len;
  }
  return total;
}

void Ctx::compact() {
  if (epoch) throw std::logic_error("the device slab cannot be compacted during a peer epoch");
  // Slide every resident list down to the lowest free offset (slab order),
  // through a bounce buffer so source and destination never overlap.
  copy_after_comp();
  std::vector<std::pair<int64_t, uint32_t>> by_off;
  for (auto& [c, r] : resident) by_off.emplace_back(h_res[c], c);
  std::sort(by_off.begin(), by_off.end());
  const uint32_t d = ix->d;
  if (!d_tmp) d_tmp = dev_alloc<float>(tmp_vecs * d);
  uint64_t cursor = 0;
  for (auto& [off, c] : by_off) {
    const uint64_t n = ix->list_len(c);
    if (uint64_t(off) != cursor && n) {
      CK(cudaMemcpyAsync(d_tmp, d_slab + uint64_t(off) * d, n * d * sizeof(float),
                         cudaMemcpyDeviceToDevice, copy));
      CK(cudaMemcpyAsync(d_slab + cursor * d, d_tmp, n * d * sizeof(float),
                         cudaMemcpyDeviceToDevice, copy));
    }
    h_res[c] = int64_t(cursor);
    cursor += n;
  }
  alloc.reset(slab_vecs);
  uint64_t dummy;
  if (cursor) alloc.alloc(cursor, dummy);
  res_dirty = true;
}

void Ctx::insert_async(uint32_t c, int tag) {
  if (!try_insert_async(c, tag)) {
    throw std::runtime_error("device cache slab too fragmented inserting cluster " +
                             std::to_string(c) + " during a peer epoch");
  }
}

bool Ctx::try_insert_async(uint32_t c, int tag) {
  if (c >= ix->nc) throw std::invalid_argument("unknown cluster id " + std::to_string(c));
  if (resident.count(c)) {
    throw std::logic_error("cluster " + std::to_string(c) + " is already resident");
  }
  const uint64_t bytes = ix->cluster_bytes(c);
  if (used + quarantined + bytes > capacity) {
    throw std::runtime_error("fast tier capacity exceeded inserting cluster " +
                             std::to_string(c));
  }
  const uint64_t n = ix->list_len(c);
  uint64_t off = 0;
  if (!alloc.alloc(n, off)) {
    if (epoch) return false; // peers may be reading: no compaction now
    compact();
    if (!alloc.alloc(n, off)) {
      throw std::runtime_error("device cache slab exhausted inserting cluster " +
                               std::to_string(c));
    }
  }
  if (n) {
    const uint32_t d = ix->d;
    CK(cudaMemcpyAsync(d_slab + off * d, ix->vecs + ix->list_off[c] * d,
                       n * d * sizeof(float), cudaMemcpyHostToDevice, copy));
  }
  resident[c] = {tag, bytes};
  used += bytes;
  h_res[c] = int64_t(off);
  res_dirty = true;
  return true;
}

uint64_t Ctx::evict(uint32_t c) {
  auto it = resident.find(c);
  if (it == resident.end()) {
    throw std::logic_error("evicting non-resident cluster " + std::to_string(c));
  }
  const uint64_t bytes = it->second.bytes;
  used -= bytes;
  if (is_pinned(c)) { // a peer may still copy it out of the slab this epoch
    quarantine.emplace_back(uint64_t(h_res[c]), ix->list_len(c));
    quarantined += bytes;
    pinned[c] = 0;
  } else {
    alloc.release(uint64_t(h_res[c]), ix->list_len(c));
  }
  h_res[c] = -1;
  res_dirty = true;
  resident.erase(it);
  return bytes;
}

void Ctx::clear_store() {
  if (epoch) {
    std::vector<uint32_t> all;
    for (auto& [c, r] : resident) all.push_back(c);
    for (uint32_t c : all) evict(c);
    return;
  }
  resident.clear();
  used = 0;
  std::fill(h_res.begin(), h_res.end(), -1);
  alloc.reset(slab_vecs);
  res_dirty = true;
}

void Ctx::coarse(const float* dQ, uint32_t nq, uint32_t n_out, cudaStream_t st, bool part,
                 bool need_scores) {
  const FastTable* f = part ? &ft : nullptr;
  if (!need_scores && use_tc(nq, n_out)) {
    const uint32_t S = launch_coarse_tc(dQ, nq, d_cen, ix->nc, ix->d, d_approx, sms, st);
    launch_tc_select(d_approx, S, dQ, nq, ix->d, d_cen, d_cnorm, ix->nc, ix->metric, n_out,
                     d_order, part ? d_res : nullptr, part ? d_list_off : nullptr, f, st,
                     /*scan_sorted=*/part && nq > 1, &tcs);
    return;
  }
  launch_coarse_scores(dQ, nq, d_cen, ix->nc, ix->d, ix->metric, d_scores, st);
  (void)f;
  select_order(d_scores, nq, n_out, d_order, part, st, /*scan_sorted=*/part && nq > 1);
}

size_t Ctx::issue_fetch(std::vector<std::vector<uint32_t>>& slow, bool& any_slow,
                        double gpu_busy, const float* dQ, uint32_t nq, uint32_t lp, const uint32_t* probe_dev,
                        int k, int G, FetchStats& st) {
  // Misses scanned on the GPU from the 2-slot ring: first every missed list
  // a peer GPU holds (copied over NVLink from the peer's slab, published for
  // this epoch), then — runtime fetch — the most-shared remaining misses
  // copied from host memory until the modeled GPU time meets the host's.
  const uint32_t d = ix->d;
  struct FetchItem {
    uint32_t c;
    const float* src;
    bool host;
    int dev = -1; // device of a peer slab
  };
  std::vector<std::vector<FetchItem>> chunks;
  uint64_t fill = 0;
  auto add_item = [&](const FetchItem& it) {
    const uint64_t len = ix->list_len(it.c);
    if (chunks.empty() || fill + len > ring_vecs) {
      if (chunks.size() == kMaxFetchChunks) return false;
      chunks.emplace_back();
      fill = 0;
    }
    chunks.back().push_back(it);
    fill += len;
    return true;
  };
  if (miss_fetch && any_slow) {
    std::map<uint32_t, uint32_t> share;
    for (uint32_t q = 0; q < nq; ++q) {
      for (uint32_t c : slow[q]) ++share[c];
    }
    std::vector<std::pair<uint32_t, uint32_t>> cand; // (share, list)
    for (auto& [c, n] : share) cand.emplace_back(n, c);
    std::sort(cand.begin(), cand.end(), [](auto& a, auto& b) {
      return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    std::vector<uint8_t> on_gpu(ix->nc, 0);
    // 1. peer-resident misses (peer copies outrun both the host link and the
    //    host scan)
    if (!peers.empty()) {
      std::vector<std::pair<uint32_t, uint32_t>> rest;
      for (auto& [n, c] : cand) {
        const float* src = nullptr;
        int sdev = -1;
        for (auto& pr : peers) {
          if (pr.slab && !pr.off.empty() && pr.off[c] >= 0) {
            src = pr.slab + uint64_t(pr.off[c]) * d;
            sdev = pr.dev;
            break;
          }
        }
        if (src && ix->list_len(c) && add_item({c, src, false, sdev})) {
          on_gpu[c] = 1;
          ++st.peer_lists;
          st.peer_bytes += ix->list_len(c) * d * 4;
        } else {
          rest.emplace_back(n, c);
        }
      }
      cand.swap(rest);
    }
    // 2. runtime fetch from host memory. Host model: memory-bound on the
    //    distinct missed bytes (each row is read once for all queries sharing
    //    its list) at the measured rate, scaled by the parallelism the tasks
    //    allow; GPU model: fetched bytes over the measured link rate plus a
    //    per-chunk launch cost.
    const double threads = double(pool->size());
    const double cr = cpu_rate > 0 ? cpu_rate : 6e9 * threads;
    auto tasks_of = [&](uint32_t c) {
      const uint64_t ch = nq == 1 ? kMissChunkSingle : kMissChunk; // miss_scan / _batch
      return double((ix->list_len(c) + ch - 1) / ch);
    };
    double host_bytes = 0, host_tasks = 0;
    for (auto& [n, c] : cand) {
      host_bytes += double(ix->list_len(c)) * d * 4;
      host_tasks += tasks_of(c);
    }
    auto host_time = [&](double bytes, double tasks) {
      return tasks <= 0 ? 0.0 : bytes / (cr * std::min(1.0, tasks / threads));
    };
    // GPU side: the hit scan keeps the GPU busy for gpu_busy; fetched lists
    // are copied meanwhile and their chunks scanned after it (a launch of
    // partition + scan per chunk). Host side: the host scan, which runs
    // during the hit scan. A list moves to the GPU only if that lowers the
    // later of the two finishes.
    double copy_t = 0, over_t = double(chunks.size()) * 50e-6;
    bool gpu_any = !chunks.empty();
    auto gpu_end = [&](double cp, double ov, bool any) {
      return any ? std::max(gpu_busy, cp) + ov : gpu_busy;
    };
    for (auto& [n, c] : cand) {
      const uint64_t len = ix->list_len(c);
      if (len == 0) continue;
      const double b = double(len) * d * 4;
      const bool new_chunk = chunks.empty() || fill + len > ring_vecs;
      const double ncp = copy_t + b / link_rate;
      const double nov = over_t + (new_chunk ? 50e-6 : 0.0) + b / scan_rate;
      const double nct = host_time(host_bytes - b, host_tasks - tasks_of(c));
      if (miss_fetch == 1 &&
          std::max(gpu_end(ncp, nov, true), nct) >=
              std::max(gpu_end(copy_t, over_t, gpu_any), host_time(host_bytes, host_tasks))) {
        break;
      }
      if (!add_item({c, ix->vecs + ix->list_off[c] * d, true})) break;
      on_gpu[c] = 1;
      ++st.fetch_lists;
      copy_t = ncp;
      over_t = nov;
      gpu_any = true;
      host_bytes -= b;
      host_tasks -= tasks_of(c);
    }
    if (st.fetch_lists || st.peer_lists) {
      any_slow = false;
      for (uint32_t q = 0; q < nq; ++q) {
        auto& v = slow[q];
        v.erase(std::remove_if(v.begin(), v.end(), [&](uint32_t c) { return on_gpu[c] != 0; }),
                v.end());
        any_slow = any_slow || !v.empty();
      }
    }
  }
  if (!chunks.empty()) {
    fetch_results_for(chunks.size() * nq * size_t(k));
    fetch_nq = nq;
    const bool wide = k > kMaxK;
    CK(cudaEventRecord(ev_f0, copy));
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    for (size_t j = 0; j < chunks.size(); ++j) {
      const int slot = int(j & 1);
      float* ring = d_ring + size_t(slot) * ring_vecs * d;
      int64_t* hres = h_res_ring + j * ix->nc;
      std::fill(hres, hres + ix->nc, int64_t(-1));
      // ring order = cluster order, so lists adjacent in the list-major host
      // store become one copy
      std::sort(chunks[j].begin(), chunks[j].end(),
                [](const FetchItem& a, const FetchItem& b) { return a.c < b.c; });
      dsts.clear();
      srcs.clear();
      sizes.clear();
      CK(cudaStreamWaitEvent(copy, ev_freed[slot], 0));
      uint64_t off = 0;
      for (const FetchItem& it : chunks[j]) {
        const uint64_t len = ix->list_len(it.c);
        hres[it.c] = int64_t(off);
        float* dst = ring + off * d;
        const size_t bytes = len * d * sizeof(float);
        if (!it.host) { // peer slab (same process or CUDA IPC): over NVLink when the
                        // peer is another device (peer access enabled at attach)
          CK(cudaMemcpyPeerAsync(dst, dev, it.src, it.dev >= 0 ? it.dev : dev, bytes, copy));
        } else if (!srcs.empty() && static_cast<float*>(srcs.back()) +
                                            sizes.back() / sizeof(float) == it.src) {
          sizes.back() += bytes;
          st.fetch_bytes += bytes;
        } else {
          dsts.push_back(dst);
          srcs.push_back(const_cast<float*>(it.src));
          sizes.push_back(bytes);
          st.fetch_bytes += bytes;
        }
        off += len;
      }
      CK(cudaMemcpyAsync(d_res_ring[slot], hres, ix->nc * sizeof(int64_t),
                         cudaMemcpyHostToDevice, copy));
      h2d_batch(dsts, srcs, sizes, copy);
      CK(cudaEventRecord(ev_landed[slot], copy));
      if (j + 1 == chunks.size()) CK(cudaEventRecord(ev_f1, copy));
      CK(cudaStreamWaitEvent(comp, ev_landed[slot], 0));
      fft.grid = static_cast<uint32_t>(G);
      launch_partition(probe_dev, nq, lp, d_res_ring[slot], d_list_off, fft, comp);
      const float* rs_s = fso.out_s;
      const uint64_t* rs_id = fso.out_id;
      const uint32_t* rs_cnt = fso.out_count;
      if (wide) { // members per query in this chunk, from the host copy of the probe
        std::vector<uint64_t> V(nq, 0);
        for (uint32_t q = 0; q < nq; ++q) {
          for (uint32_t i = 0; i < lp; ++i) {
            const uint32_t c = h_order[size_t(q) * lp + i];
            if (hres[c] >= 0) V[q] += ix->list_len(c);
          }
        }
        scan_wide(dQ, nq, fft, ring, V, k, nullptr, comp);
        rs_s = d_wout_s;
        rs_id = d_wout_id;
        rs_cnt = d_wout_cnt;
      } else {
        launch_scan(dQ, nq, d, ix->metric, k, fft, ring, d_ids, fso, G, acc_fp64, scan_impl, tune,
                    comp);
      }
      CK(cudaEventRecord(ev_freed[slot], comp));
      const size_t o = j * nq;
      CK(cudaMemcpyAsync(h_fetch_s + o * k, rs_s, size_t(nq) * k * sizeof(float),
                         cudaMemcpyDeviceToHost, comp));
      CK(cudaMemcpyAsync(h_fetch_id + o * k, rs_id, size_t(nq) * k * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost, comp));
      CK(cudaMemcpyAsync(h_fetch_cnt + j * max_batch, rs_cnt, nq * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost, comp));
    }
    rec(ev_fdone, comp);
  }
  return chunks.size();
}

void Ctx::merge_fetch(uint32_t q, size_t nchunks, int k, std::vector<Scored>& gpu) const {
  for (size_t j = 0; j < nchunks; ++j) {
    const uint32_t n = h_fetch_cnt[j * max_batch + q];
    const size_t o = j * fetch_nq + q;
    std::vector<Scored> f(n);
    for (uint32_t i = 0; i < n; ++i) {
      f[i] = {h_fetch_s[o * k + i], h_fetch_id[o * k + i]};
    }
    gpu = merge_topk(ix->metric, gpu, f, k);
  }
}

void Ctx::finish_fetch(size_t nchunks, FetchStats& st) {
  if (nchunks == 0) return;
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, ev_f0, ev_f1));
  st.t_fetch = ms * 1e-3;
  if (ms > 0 && st.fetch_bytes > (64ull << 20) && st.peer_lists == 0) {
    link_rate = 0.5 * link_rate + 0.5 * double(st.fetch_bytes) / (ms * 1e-3);
  }
}

// List-major scan policy (LAIVG_LIST_SCAN): "0" off, "1" whenever the shape
// allows, default auto: when the previous batches' queries per resident
// probed list (EMA) reach LAIVG_LIST_SCAN_QPL (default 1.5; measured
// crossover ~1.3, profiles/r02/list_scan_sharing.jsonl). Before any batch
// the estimate is the uniform-probe prior nq * L / nc (topical batches share
// more than that).
bool Ctx::want_list_scan(uint32_t nq, uint32_t lp, int k) const {
  const char* em = std::getenv("LAIVG_LIST_SCAN"); // read per call (tests switch it)
  const int mode = em ? std::atoi(em) : 2;
  const char* eq = std::getenv("LAIVG_LIST_SCAN_QPL");
  const double qpl_min = eq ? std::atof(eq) : 1.5;
  if (mode == 0 || nq < 2 || !list_scan_supported(ix->d, k) || slab_vecs == 0) return false;
  return mode == 1 || list_scan_sharing(nq, lp) >= qpl_min;
}

void Ctx::ensure_list_scan() {
  if (lss.cand) return;
  const uint32_t nc = ix->nc;
  lss.gcap = 16384;
  lss.qcount = dev_alloc<uint32_t>(std::max(nc, 1u));
  lss.lists = dev_alloc<uint32_t>(std::max(nc, 1u));
  lss.lq_off = dev_alloc<uint32_t>(nc + 1);
  lss.item_off = dev_alloc<uint32_t>(nc + 1);
  lss.qidx = dev_alloc<uint32_t>(std::max<size_t>(1, size_t(max_batch) * max_probe));
  lss.meta = dev_alloc<uint32_t>(4);
  lss.gtau = dev_alloc<uint32_t>(max_batch);
  lss.gcnt = dev_alloc<uint32_t>(max_batch);
  lss.cand = dev_alloc<uint4>(size_t(max_batch) * lss.gcap);
  h_ls_flag = pin_alloc_mapped<unsigned>(1, &dm_ls_flag);
}

void Ctx::run_list_scan(const float* dQ, uint32_t nq, uint32_t lp, int k, cudaStream_t st) {
  ensure_list_scan();
  *reinterpret_cast<volatile unsigned*>(h_ls_flag) = 0u;
  ListScan p;
  p.Q = dQ;
  p.nq = nq;
  p.d = ix->d;
  p.nc = ix->nc;
  p.lp = lp;
  p.metric = ix->metric;
  p.k = k;
  p.order = d_order;
  p.res = d_res;
  p.list_off = d_list_off;
  p.slab = d_slab;
  p.slab_rows = slab_vecs;
  p.ids = d_ids;
  p.out_s = dm_out_s;
  p.out_id = dm_out_id;
  p.out_count = dm_out_cnt;
  p.fcount_in = ft.count;
  p.fcount_out = dm_fcount;
  p.flag_host = dm_ls_flag;
  p.grid = sms;
  p.scratch = lss;
  // 32-query items once lists are shared by >= 12 queries (each 16-query
  // group streams its chunk again); LAIVG_LIST_SCAN_N forces 16 / 32
  const char* en = std::getenv("LAIVG_LIST_SCAN_N");
  const uint32_t forced = en ? uint32_t(std::atoi(en)) : 0u;
  p.group = forced == 16 || forced == 32 ? forced
            : (list_scan_sharing(nq, lp) >= 12.0 ? 32u : 16u);
  if (!list_scan_supported(ix->d, k, p.group)) p.group = 16;
  // whole lists per item (4096-row chunks: fewer item boundaries, c2b 48.4 ->
  // 51.0 K q/s) once the batch touches >= 8 lists per SM; 1024-row chunks
  // keep the tail balanced for smaller batches. LAIVG_LIST_SCAN_CHUNK forces.
  const double lists_est =
      double(nq) * lp / std::max(1.0, list_scan_sharing(nq, lp));
  p.chunk = lists_est >= 8.0 * sms ? 4096u : 1024u;
  if (const char* ec = std::getenv("LAIVG_LIST_SCAN_CHUNK")) p.chunk = uint32_t(std::atol(ec));
  launch_list_scan(p, st);
  ++ls_runs;
}

Ctx::BatchResult Ctx::search_batch(const float* dQ, const float* hQ, uint32_t nq, int L,
                                   int k) {
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  const bool wide = k > kMaxK; // top-k by radix sort of every candidate (wide.cu)
  if (nq > max_batch) throw std::invalid_argument("batch exceeds the context's max_batch");
  const auto t0 = Clock::now();
  BatchResult r;
  r.top.resize(nq);
  r.nfast.assign(nq, 0);
  r.nslow.assign(nq, 0);
  const uint32_t lp = uint32_t(std::min<int64_t>(std::max(L, 0), ix->nc));
  if (lp > max_probe) {
    throw std::invalid_argument("probe of " + std::to_string(lp) +
                                " clusters exceeds the context's max_probe " +
                                std::to_string(max_probe));
  }
  if (nq == 0) return r;
  if (lp == 0) {
    r.t_2 = secs(t0, Clock::now());
    return r;
  }
  CK(cudaStreamWaitEvent(comp, ev_copy_tail, 0));
  r.h2d_bytes += commit_res(comp);
  const int G = std::max(1, std::min(scan_grid_x(nq, sms, scan_impl, tune), part_cap / int(nq)));
  ft.grid = static_cast<uint32_t>(G);
  rec(ev_a, comp);
  coarse(dQ, nq, lp, comp, /*part=*/true);
  rec(ev_b, comp);
  CK(cudaEventRecord(ev_fork, comp));
  CK(cudaStreamWaitEvent(aux, ev_fork, 0));
  CK(cudaMemcpyAsync(h_order, d_order, size_t(nq) * lp * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost, aux));
  rec(ev_probe, aux);
  rec(ev_p, comp);
  bool use_ls = !wide && want_list_scan(nq, lp, k);
  if (!wide) {
    if (use_ls) {
      run_list_scan(dQ, nq, lp, k, comp);
    } else {
      launch_scan(dQ, nq, ix->d, ix->metric, k, ft, d_slab, d_ids, so, G, acc_fp64, scan_impl,
                  tune, comp);
    }
    rec(ev_s, comp);
    rec(ev_c, comp); // results are in mapped host memory
  }

  // host: split every probe by residency and scan the misses list-major
  CK(cudaEventSynchronize(ev_probe));
  std::vector<std::vector<uint32_t>> slow(nq);
  std::vector<uint64_t> vfast(nq, 0);
  bool any_slow = false;
  for (uint32_t q = 0; q < nq; ++q) {
    for (uint32_t i = 0; i < lp; ++i) {
      const uint32_t c = h_order[size_t(q) * lp + i];
      if (h_res[c] >= 0) {
        ++r.nfast[q];
        vfast[q] += ix->list_len(c);
        r.vecs_gpu += ix->list_len(c);
        r.bytes_gpu += ix->cluster_bytes(c);
      } else {
        slow[q].push_back(c);
        any_slow = true;
      }
    }
    r.nslow[q] = uint32_t(slow[q].size());
  }
  {
    // sharing of the resident lists across the batch (list-scan policy)
    std::vector<unsigned char> seen(ix->nc, 0);
    uint64_t pairs = 0, lists = 0;
    for (uint32_t q = 0; q < nq; ++q) {
      for (uint32_t i = 0; i < lp; ++i) {
        const uint32_t c = h_order[size_t(q) * lp + i];
        if (h_res[c] < 0) continue;
        ++pairs;
        if (!seen[c]) {
          seen[c] = 1;
          ++lists;
          r.distinct_bytes += ix->list_len(c) * uint64_t(ix->d) * 4;
        }
      }
    }
    if (lists) {
      const double qpl = double(pairs) / double(lists);
      ls_qpl = ls_qpl > 0 ? 0.5 * ls_qpl + 0.5 * qpl : qpl;
    }
  }
  if (wide) { // the candidate sort is sized by the probe split
    scan_wide(dQ, nq, ft, d_slab, vfast, k, dm_fcount, comp);
    wide_results(nq, k, comp);
    rec(ev_s, comp);
    rec(ev_c, comp);
  }
  const uint32_t d = ix->d;
  FetchStats fst;
  const size_t nchunks = (miss_fetch && any_slow)
                             ? issue_fetch(slow, any_slow, busy_of(vfast), dQ, nq, lp, d_order, k,
                                           G, fst)
                             : 0;
  std::vector<std::vector<Scored>> miss(nq);
  if (any_slow) {
    std::map<uint32_t, uint32_t> cl;
    for (uint32_t q = 0; q < nq; ++q) {
      for (uint32_t c : slow[q]) {
        ++cl[c];
        r.cpu_query_bytes += ix->list_len(c) * d * 4;
      }
    }
    r.cpu_lists = uint32_t(cl.size());
    const auto tc = Clock::now();
    miss = miss_scan_batch(*ix, hQ, nq, slow, k, *pool);
    r.t_c = secs(tc, Clock::now());
    // measured host rate on distinct bytes, parallelism-corrected
    double dbytes = 0, dtasks = 0;
    for (auto& [c, n] : cl) {
      dbytes += double(ix->list_len(c)) * d * 4;
      dtasks += double((ix->list_len(c) + kMissChunk - 1) / kMissChunk);
    }
    if (r.t_c > 0 && dbytes > double(16ull << 20)) {
      const double eff = std::min(1.0, dtasks / double(pool->size()));
      const double rate = dbytes / (r.t_c * eff);
      cpu_rate = cpu_rate > 0 ? 0.5 * cpu_rate + 0.5 * rate : rate;
    }
  }
  CK(cudaEventSynchronize(ev_c));
  if (use_ls && *reinterpret_cast<volatile unsigned*>(h_ls_flag)) {
    // a candidate buffer overflowed (e.g. many equal scores): per-query scan
    ++ls_fallbacks;
    use_ls = false;
    launch_scan(dQ, nq, ix->d, ix->metric, k, ft, d_slab, d_ids, so, G, acc_fp64, scan_impl, tune,
                comp);
    rec(ev_s, comp);
    rec(ev_c, comp);
    CK(cudaEventSynchronize(ev_c));
  }
  ls_result = use_ls;
  r.list_scan = use_ls ? 1u : 0u;
  if (nchunks) CK(cudaEventSynchronize(ev_fdone));
  for (uint32_t q = 0; q < nq; ++q) {
    if (h_fcount[q] != r.nfast[q]) {
      throw std::runtime_error("device residency table disagrees with the store");
    }
    std::vector<Scored> gpu = scan_result(q, uint32_t(G), k, vfast[q]);
    merge_fetch(q, nchunks, k, gpu);
    r.top[q] = merge_topk(ix->metric, gpu, miss[q], k);
  }
  r.t_2 = secs(t0, Clock::now()); // merged results exist: timing bookkeeping follows
  finish_fetch(nchunks, fst);
  r.fetch_lists = fst.fetch_lists;
  r.peer_lists = fst.peer_lists;
  r.fetch_bytes = fst.fetch_bytes;
  r.peer_bytes = fst.peer_bytes;
  r.t_fetch = fst.t_fetch;
  r.h2d_bytes += fst.fetch_bytes;
  r.d2h_bytes += uint64_t(nq) * lp * sizeof(uint32_t) + uint64_t(nq) * sizeof(uint32_t) +
                 (use_ls ? uint64_t(nq) * (k * (sizeof(float) + sizeof(uint64_t)) + 4)
                         : result_bytes(nq, uint32_t(G), k)) +
                 fetch_result_bytes(nchunks, nq, k);
  ls_result = false;
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, ev_a, nchunks ? ev_fdone : ev_s));
  r.t_g = ms * 1e-3;
  CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
  r.t_coarse = ms * 1e-3;
  CK(cudaEventElapsedTime(&ms, ev_p, ev_s));
  r.t_scan = ms * 1e-3;
  {
    uint64_t v = 0;
    for (uint64_t x : vfast) v += x;
    note_scan(v, r.t_scan);
  }
  return r;
}

Ctx::Result Ctx::search(const float* dq, const float* hq, int L, int k,
                        const std::vector<uint32_t>* explicit_probe) {
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  const bool wide = k > kMaxK; // top-k by radix sort of every candidate (wide.cu)
  const auto t0 = Clock::now();
  PhaseTrace tr;
  tr.mark("start");
  Result r;
  uint32_t lp;
  if (explicit_probe) {
    for (uint32_t c : *explicit_probe) {
      if (c >= ix->nc) throw std::invalid_argument("unknown cluster id " + std::to_string(c));
    }
    lp = uint32_t(explicit_probe->size());
  } else {
    lp = uint32_t(std::min<int64_t>(std::max(L, 0), ix->nc));
  }
  if (lp > max_probe) {
    throw std::invalid_argument("probe of " + std::to_string(lp) +
                                " clusters exceeds the context's max_probe " +
                                std::to_string(max_probe));
  }
  // Retrieval is ordered after every prefetch copy issued so far, then sees
  // the residency table of the host store state.
  CK(cudaStreamWaitEvent(comp, ev_copy_tail, 0));
  r.h2d_bytes += commit_res(comp);
  tr.mark("commit");
  const int G = std::min(scan_grid_x(1, sms, scan_impl, tune), part_cap);
  ft.grid = static_cast<uint32_t>(G); // the partition step lays out G scan CTAs
  if (explicit_probe) {
    CK(cudaMemcpyAsync(d_Q, dq, ix->d * sizeof(float), cudaMemcpyDefault, comp));
    CK(cudaEventRecord(ev_a, comp));
    if (lp) {
      std::memcpy(h_order, explicit_probe->data(), lp * sizeof(uint32_t));
      CK(cudaMemcpyAsync(d_order, h_order, lp * sizeof(uint32_t), cudaMemcpyHostToDevice, comp));
    }
    CK(cudaEventRecord(ev_b, comp));
    launch_partition(d_order, 1, lp, d_res, d_list_off, ft, comp);
    CK(cudaEventRecord(ev_p, comp));
    if (wide) {
      std::vector<uint64_t> V(1, 0);
      for (uint32_t c : *explicit_probe) {
        if (h_res[c] >= 0) V[0] += ix->list_len(c);
      }
      scan_wide(d_Q, 1, ft, d_slab, V, k, dm_fcount, comp);
      wide_results(1, k, comp);
    } else {
      launch_scan(d_Q, 1, ix->d, ix->metric, k, ft, d_slab, d_ids, so, G, acc_fp64, scan_impl,
                  tune, comp);
    }
    CK(cudaEventRecord(ev_s, comp));
    enqueue_results(k);
  } else if (wide) {
    // eager chain: query -> coarse -> ranking + residency split; the host
    // needs the probe to size the candidate sort
    CK(cudaMemcpyAsync(d_Q, dq, ix->d * sizeof(float), cudaMemcpyDefault, comp));
    CK(cudaEventRecord(ev_a, comp));
    coarse(d_Q, 1, lp, comp, /*part=*/true);
    if (lp) {
      CK(cudaMemcpyAsync(h_order, d_order, lp * sizeof(uint32_t), cudaMemcpyDeviceToHost, comp));
    }
    CK(cudaEventRecord(ev_b, comp));
    CK(cudaEventSynchronize(ev_b));
    std::vector<uint64_t> V(1, 0);
    for (uint32_t i = 0; i < lp; ++i) {
      if (h_res[h_order[i]] >= 0) V[0] += ix->list_len(h_order[i]);
    }
    scan_wide(d_Q, 1, ft, d_slab, V, k, dm_fcount, comp);
    wide_results(1, k, comp);
    CK(cudaEventRecord(ev_s, comp));
    enqueue_results(k);
  } else {
    // the query always runs from d_Q so one captured graph serves every call
    run_coarse_path(lp, k, G, dq, &tr);
  }
  tr.mark("launch");

  // Host: split the probe by residency (tiered.cpp:155-161) and scan the
  // misses while the GPU scans the hits.
  const bool fused = !explicit_probe && !wide && last_fused;
  if (fused && lp) wait_probe_flag(fused_seq);
  else if (!explicit_probe && lp) CK(cudaEventSynchronize(ev_b));
  tr.mark("probe_wait");
  for (uint32_t i = 0; i < lp; ++i) {
    const uint32_t c = h_order[i];
    (h_res[c] >= 0 ? r.fast : r.slow).push_back(c);
  }
  // The misses (r.slow keeps the reference's meaning: not cached here) go
  // to the GPU (peer copies, runtime fetch) and/or the host scan.
  std::vector<std::vector<uint32_t>> host(1, r.slow);
  bool any_host = !r.slow.empty();
  FetchStats fst;
  const size_t nchunks =
      (miss_fetch && any_host)
          ? issue_fetch(host, any_host, busy_of(std::vector<uint64_t>(1, fast_vecs(r.fast))), d_Q,
                        1, lp, (explicit_probe || wide) ? d_order : dm_order, k, G, fst)
          : 0;
  std::vector<Scored> miss;
  if (any_host) {
    const auto tc = Clock::now();
    miss = miss_scan(*ix, hq, host[0], k, *pool);
    r.t_c = secs(tc, Clock::now());
  }
  tr.mark("split_miss");
  if (fused) wait_probe_flag(fused_seq, 1); // results out (before the kernel's teardown)
  else CK(cudaEventSynchronize((explicit_probe || wide) ? ev_c : ev_s));
  if (nchunks) CK(cudaEventSynchronize(ev_fdone));
  tr.mark("scan_wait");
  if (*h_fcount != r.fast.size()) {
    throw std::runtime_error("device residency table disagrees with the store");
  }
  uint64_t vfast = 0;
  for (uint32_t c : r.fast) vfast += ix->list_len(c);
  std::vector<Scored> gpu = scan_result(0, uint32_t(G), k, vfast);
  tr.mark("scanres");
  if (h_probe) print_probe(1, uint32_t(G));
  merge_fetch(0, nchunks, k, gpu);
  r.top = merge_topk(ix->metric, gpu, miss, k);
  r.t_2 = secs(t0, Clock::now()); // the merged result exists: timing bookkeeping follows
  tr.mark("mtopk");
  finish_fetch(nchunks, fst);
  tr.mark("fetchfin");
  r.fetch_lists = fst.fetch_lists;
  r.peer_lists = fst.peer_lists;
  r.fetch_bytes = fst.fetch_bytes;
  r.peer_bytes = fst.peer_bytes;
  r.t_fetch = fst.t_fetch;
  r.h2d_bytes += fst.fetch_bytes + (explicit_probe ? uint64_t(lp) * sizeof(uint32_t) : 0);
  r.d2h_bytes += uint64_t(lp) * sizeof(uint32_t) + sizeof(uint32_t) +
                 result_bytes(1, uint32_t(G), k) + fetch_result_bytes(nchunks, 1, k);
  float ms = 0;
  link_h2d_total += r.h2d_bytes;
  link_d2h_total += r.d2h_bytes;
  if (!want_timing) {
    // the caller asked for no timing: skip the event queries (they cost
    // microseconds of the call); the scan-rate model still learns from the
    // fused kernel's own stamps
    if (fused && h_stamps[7] > h_stamps[5]) {
      uint64_t v = 0;
      for (uint32_t c : r.fast) v += ix->list_len(c);
      note_scan(v, double(h_stamps[7] - h_stamps[5]) * 1e-9);
    }
    return r;
  }
  if (fused) {
    // one kernel: its event time; the coarse + selection phase from CTA 0's
    // globaltimer stamps (entry -> scan ranges ready)
    CK(cudaEventSynchronize(ev_s)); // the host only waited for the results flag
    CK(cudaEventElapsedTime(&ms, ev_a, ev_s));
    r.t_kernel = ms * 1e-3;
    r.t_coarse = std::min(r.t_kernel, double(h_stamps[5] - h_stamps[0]) * 1e-9);
    r.t_scan = r.t_kernel - r.t_coarse;
    if (tr.on) {
      std::fprintf(stderr,
                   "[laivg fused] us from CTA 0 entry: query %.2f keys %.2f loaded %.2f "
                   "selected %.2f ranges %.2f loop end %.2f done %.2f | kernel (events) %.2f\n",
                   (h_stamps[1] - h_stamps[0]) * 1e-3, (h_stamps[2] - h_stamps[0]) * 1e-3,
                   (h_stamps[3] - h_stamps[0]) * 1e-3, (h_stamps[4] - h_stamps[0]) * 1e-3,
                   (h_stamps[5] - h_stamps[0]) * 1e-3, (h_stamps[6] - h_stamps[0]) * 1e-3,
                   (h_stamps[7] - h_stamps[0]) * 1e-3, r.t_kernel * 1e6);
      std::string sel = "[laivg fused] select us from keys loaded:";
      for (int i = 8; i < 19; ++i) {
        if (h_stamps[i] >= h_stamps[3]) {
          sel += " " + std::to_string(i - 8) + ":" + std::to_string((h_stamps[i] - h_stamps[3]) * 1e-3);
        }
      }
      sel += " passes " + std::to_string(h_stamps[19]);
      std::fprintf(stderr, "%s\n", sel.c_str());
      std::fprintf(stderr, "[laivg fused] CTA 0 epilogue: lists stored %.2f, CTA merge done %.2f\n",
                   (h_stamps[21] - h_stamps[0]) * 1e-3, (h_stamps[22] - h_stamps[0]) * 1e-3);
      if (h_cta_stamps) {
        unsigned long long e0 = ~0ull, e1 = 0, b1a = ~0ull, b1b = 0, b2a = ~0ull, b2b = 0,
                           da = ~0ull, db = 0;
        for (int b = 0; b < sms; ++b) {
          const unsigned long long* p = h_cta_stamps + 4 * b;
          e0 = std::min(e0, p[0]);
          e1 = std::max(e1, p[0]);
          b1a = std::min(b1a, p[1]);
          b1b = std::max(b1b, p[1]);
          b2a = std::min(b2a, p[2]);
          b2b = std::max(b2b, p[2]);
          da = std::min(da, p[3]);
          db = std::max(db, p[3]);
        }
        std::fprintf(stderr,
                     "[laivg fused] CTAs (us from first entry): entry <= %.2f, barrier 1 exit "
                     "%.2f..%.2f, barrier 2 exit %.2f..%.2f, done %.2f..%.2f (CTA 0 %.2f)\n",
                     (e1 - e0) * 1e-3, (b1a - e0) * 1e-3, (b1b - e0) * 1e-3, (b2a - e0) * 1e-3,
                     (b2b - e0) * 1e-3, (da - e0) * 1e-3, (db - e0) * 1e-3,
                     (h_cta_stamps[3] - e0) * 1e-3);
      }
    }
  } else {
    CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
    r.t_coarse = ms * 1e-3;
    tr.mark("ev1");
    CK(cudaEventElapsedTime(&ms, explicit_probe ? ev_p : ev_b, ev_s));
    r.t_scan = ms * 1e-3;
  }
  tr.mark("ev2");
  if (nchunks || explicit_probe || wide) {
    CK(cudaEventElapsedTime(&ms, ev_a, nchunks ? ev_fdone : ev_s));
    r.t_g = ms * 1e-3;
  } else {
    r.t_g = r.t_coarse + r.t_scan; // one query: a -> b -> s back to back
  }
  for (uint32_t c : r.fast) {
    r.vecs_gpu += ix->list_len(c);
    r.bytes_gpu += ix->cluster_bytes(c);
  }
  note_scan(r.vecs_gpu, r.t_scan);
  tr.mark("merge");
  tr.dump();
  return r;
}

} // namespace laivg

// ============================================================================
// C ABI
// ============================================================================
using laivg::Ctx;
using laivg::Index;
using laivg::Clock;

struct laivg_index {
  Index ix;
};
struct laivg_ctx {
  Ctx c;
};
struct laivg_hotness {
  laivg::Hotness h;
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return LAIVG_OK;
  } catch (const laivg::CudaError& e) {
    laivg::g_err = e.what();
    return LAIVG_ECUDA;
  } catch (const std::invalid_argument& e) {
    laivg::g_err = e.what();
    return LAIVG_EINVAL;
  } catch (const std::logic_error& e) {
    laivg::g_err = e.what();
    return LAIVG_ELOGIC;
  } catch (const std::runtime_error& e) {
    laivg::g_err = e.what();
    return LAIVG_ERUNTIME;
  } catch (const std::exception& e) {
    laivg::g_err = e.what();
    return LAIVG_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + " is null");
}

void set_ctx_device(const laivg_ctx* ctx) {
  need(ctx, "ctx");
  CK(cudaSetDevice(ctx->c.dev));
}

void fill_timing(laivg_hybrid_timing* t, const Ctx::Result& r,
                 const laivg_cost_model* cost) {
  if (!t) return;
  t->t_g = r.t_g;
  t->t_c = r.t_c;
  t->t_2 = r.t_2;
  t->t_coarse = r.t_coarse;
  t->t_scan = r.t_scan;
  t->t_kernel = r.t_kernel;
  t->scanned_vectors = r.vecs_gpu;
  t->scanned_bytes = r.bytes_gpu;
  t->fetched_lists = r.fetch_lists;
  t->cpu_lists = uint32_t(r.slow.size()) - r.fetch_lists - r.peer_lists;
  t->fetched_bytes = r.fetch_bytes;
  t->t_fetch = r.t_fetch;
  t->peer_lists = r.peer_lists;
  t->peer_bytes = r.peer_bytes;
  t->list_scan = 0;
  t->distinct_bytes = 0;
  t->h2d_bytes = r.h2d_bytes;
  t->d2h_bytes = r.d2h_bytes;
  if (cost) { // tiered.cpp:190-196
    const double miss = double(r.slow.size());
    t->model_t_c = std::ceil(miss / cost->parallel_slots) * cost->t_cc;
    t->model_t_g = double(r.fast.size()) * cost->t_gc;
    t->model_t_2 = std::max(t->model_t_c, t->model_t_g);
  } else {
    t->model_t_c = t->model_t_g = t->model_t_2 = 0.0;
  }
}

void write_top(const std::vector<laivg::Scored>& top, int k, uint64_t* ids,
               float* scores, uint32_t* count) {
  for (size_t i = 0; i < top.size(); ++i) {
    ids[i] = top[i].id;
    scores[i] = top[i].s;
  }
  for (size_t i = top.size(); i < size_t(k); ++i) {
    ids[i] = ~0ull;
    scores[i] = std::nanf("");
  }
  if (count) *count = uint32_t(top.size());
}

void stage_batch(Ctx& c, const float* Q, uint32_t nq) {
  const size_t n = size_t(nq) * c.ix->d;
  std::memcpy(c.h_Q, Q, n * sizeof(float));
  CK(cudaMemcpyAsync(c.d_Q, c.h_Q, n * sizeof(float), cudaMemcpyHostToDevice, c.comp));
}

void fill_batch_timing(laivg_hybrid_timing* t, const Ctx::BatchResult& r,
                       const laivg_cost_model* cost) {
  if (!t) return;
  t->t_g = r.t_g;
  t->t_c = r.t_c;
  t->t_2 = r.t_2;
  t->t_coarse = r.t_coarse;
  t->t_scan = r.t_scan;
  t->t_kernel = 0.0;
  t->scanned_vectors = r.vecs_gpu;
  t->scanned_bytes = r.bytes_gpu;
  t->fetched_lists = r.fetch_lists;
  t->cpu_lists = r.cpu_lists;
  t->fetched_bytes = r.fetch_bytes;
  t->t_fetch = r.t_fetch;
  t->peer_lists = r.peer_lists;
  t->peer_bytes = r.peer_bytes;
  t->h2d_bytes = r.h2d_bytes;
  t->d2h_bytes = r.d2h_bytes;
  t->list_scan = r.list_scan;
  t->distinct_bytes = r.distinct_bytes;
  if (cost) { // tiered.cpp:190-196 summed over the batch
    double miss = 0, hit = 0;
    for (size_t q = 0; q < r.nfast.size(); ++q) {
      miss += r.nslow[q];
      hit += r.nfast[q];
    }
    t->model_t_c = std::ceil(miss / cost->parallel_slots) * cost->t_cc;
    t->model_t_g = hit * cost->t_gc;
    t->model_t_2 = std::max(t->model_t_c, t->model_t_g);
  } else {
    t->model_t_c = t->model_t_g = t->model_t_2 = 0.0;
  }
}

// The query goes to the pinned staging row; the search's first node copies
// it to the device.
void stage_query(Ctx& c, const float* q) {
  need(q, "query");
  std::memcpy(c.h_Q, q, c.ix->d * sizeof(float));
}

} // namespace

extern "C" {

const char* laivg_last_error(void) { return laivg::g_err.c_str(); }
uint32_t laivg_version(void) { return (1u << 16) | 0u; }

int laivg_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    need(out, "out");
    CK(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}
int laivg_host_free(void* p) {
  return guard([&] {
    if (p) CK(cudaFreeHost(p));
  });
}
int laivg_host_register(void* p, uint64_t bytes) {
  return guard([&] {
    need(p, "pointer");
    CK(cudaHostRegister(p, bytes, cudaHostRegisterPortable));
  });
}
int laivg_host_unregister(void* p) {
  return guard([&] {
    need(p, "pointer");
    CK(cudaHostUnregister(p));
  });
}
uint64_t laivg_kernel_launches(void) { return laivg::launch_counter().load(); }

// ---- index -----------------------------------------------------------------
int laivg_index_create(const float* centroids, uint32_t nc, uint32_t d, int metric,
                       const float* vecs, const uint64_t* ids, const uint64_t* list_off,
                       uint32_t flags, laivg_index** out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (d == 0) throw std::invalid_argument("matrix has no dimension set");
    if (metric != LAIVG_METRIC_IP && metric != LAIVG_METRIC_L2) {
      throw std::invalid_argument("bad metric");
    }
    need(list_off, "list_off");
    if (nc) need(centroids, "centroids");
    auto h = std::make_unique<laivg_index>();
    Index& ix = h->ix;
    ix.nc = nc;
    ix.d = d;
    ix.metric = metric;
    ix.centroids.assign(centroids, centroids + size_t(nc) * d);
    ix.list_off.assign(list_off, list_off + nc + 1);
    if (ix.list_off[0] != 0) throw std::invalid_argument("list_off[0] must be 0");
    for (uint32_t c = 0; c < nc; ++c) {
      if (ix.list_off[c + 1] < ix.list_off[c]) {
        throw std::invalid_argument("list_off must be non-decreasing");
      }
    }
    const uint64_t n = ix.list_off[nc];
    if (n) {
      need(vecs, "vecs");
      need(ids, "ids");
    }
    if (!(flags & LAIVG_INDEX_TRUST)) { // vectorstore.cpp:66-85, first bad row in append order
      ix.vecs = vecs;
      ix.ids = ids;
      laivg::validate_store(ix, 0);
    }
    if (flags & LAIVG_INDEX_BORROW) {
      ix.vecs = vecs;
      ix.ids = ids;
    } else {
      const size_t vb = size_t(n) * d * sizeof(float), ib = size_t(n) * sizeof(uint64_t);
      // Pinned when a driver is present; pageable host memory otherwise (the
      // index itself is host data -- only the device context needs a GPU).
      void* blk = nullptr;
      if (cudaHostAlloc(&blk, vb + ib + 16, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        blk = std::aligned_alloc(64, ((vb + ib + 16) + 63) & ~size_t(63));
        if (!blk) throw std::runtime_error("host allocation failed");
        ix.owned_pageable = true;
      }
      ix.owned_block = blk;
      float* v = static_cast<float*>(blk);
      uint64_t* id = reinterpret_cast<uint64_t*>(static_cast<char*>(blk) + ((vb + 15) & ~size_t(15)));
      if (n) {
        std::memcpy(v, vecs, vb);
        std::memcpy(id, ids, ib);
      }
      ix.vecs = v;
      ix.ids = id;
    }
    *out = h.release();
  });
}

namespace {
void* laix_alloc(uint64_t bytes, void* user) {
  // 2 MB aligned and backed by huge pages where the kernel allows: the
  // readers fault the block in 512x fewer times
  const size_t b = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  void* p = std::aligned_alloc(size_t(2) << 20, b);
  if (!p) throw std::runtime_error("host allocation failed");
  madvise(p, b, MADV_HUGEPAGE);
  *static_cast<size_t*>(user) = b;
  return p;
}
} // namespace

int laivg_index_load(const char* path, uint32_t threads, laivg_index** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = nullptr;
    auto h = std::make_unique<laivg_index>();
    size_t bytes = 0;
    const auto t0 = Clock::now();
    try {
      laivg::laix_load(path, threads, h->ix, laix_alloc, &bytes);
    } catch (...) {
      std::free(h->ix.owned_block);
      throw;
    }
    h->ix.owned_pageable = true;
    const auto t1 = Clock::now();
    // pin the store in place (the rows are already resident): every device
    // copies lists from it; without a driver it stays pageable
    if (bytes && cudaHostRegister(h->ix.owned_block, bytes, cudaHostRegisterPortable) ==
                     cudaSuccess) {
      h->ix.owned_registered = true;
    } else {
      cudaGetLastError();
    }
    if (std::getenv("LAIVG_TRACE")) {
      std::fprintf(stderr, "[laivg] index_load %s: read+validate %.3f s, pin %.3f s (%.2f GB)\n",
                   path, std::chrono::duration<double>(t1 - t0).count(),
                   std::chrono::duration<double>(Clock::now() - t1).count(), bytes / 1e9);
    }
    *out = h.release();
  });
}

int laivg_index_save(const laivg_index* ix, const char* path, uint32_t threads) {
  return guard([&] {
    need(ix, "index");
    need(path, "path");
    laivg::laix_save(path, ix->ix, threads);
  });
}

int laivg_index_store(const laivg_index* ix, const float** vecs, const uint64_t** ids,
                      const uint64_t** list_off, const float** centroids) {
  return guard([&] {
    need(ix, "index");
    if (vecs) *vecs = ix->ix.vecs;
    if (ids) *ids = ix->ix.ids;
    if (list_off) *list_off = ix->ix.list_off.data();
    if (centroids) *centroids = ix->ix.centroids.data();
  });
}

void laivg_index_destroy(laivg_index* ix) {
  if (!ix) return;
  if (ix->ix.owned_block) {
    if (ix->ix.owned_registered) cudaHostUnregister(ix->ix.owned_block);
    if (ix->ix.owned_pageable) std::free(ix->ix.owned_block);
    else cudaFreeHost(ix->ix.owned_block);
  }
  delete ix;
}
uint32_t laivg_index_num_clusters(const laivg_index* ix) { return ix ? ix->ix.nc : 0; }
uint32_t laivg_index_dim(const laivg_index* ix) { return ix ? ix->ix.d : 0; }
int laivg_index_metric(const laivg_index* ix) { return ix ? ix->ix.metric : -1; }
uint64_t laivg_index_total_vectors(const laivg_index* ix) { return ix ? ix->ix.total() : 0; }
uint64_t laivg_index_cluster_bytes(const laivg_index* ix, uint32_t c) {
  return (ix && c < ix->ix.nc) ? ix->ix.cluster_bytes(c) : 0;
}
uint64_t laivg_index_list_len(const laivg_index* ix, uint32_t c) {
  return (ix && c < ix->ix.nc) ? ix->ix.list_len(c) : 0;
}
uint64_t laivg_index_total_payload_bytes(const laivg_index* ix) {
  return ix ? ix->ix.total() * ix->ix.member_bytes() : 0;
}

// ---- context ---------------------------------------------------------------
void laivg_opts_default(laivg_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->acc_fp64 = 1;
  o->scan_impl = 0;
  o->miss_fetch = 1;
}

int laivg_ctx_create(const laivg_index* ix, const laivg_opts* opts, laivg_ctx** out) {
  return guard([&] {
    need(ix, "index");
    need(out, "out");
    *out = nullptr;
    laivg_opts o;
    if (opts) o = *opts;
    else laivg_opts_default(&o);
    auto h = std::make_unique<laivg_ctx>();
    h->c.init(&ix->ix, o);
    *out = h.release();
  });
}

void laivg_ctx_destroy(laivg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.dev);
  delete ctx;
}

int laivg_ctx_sync(laivg_ctx* ctx) {
  return guard([&] {
    set_ctx_device(ctx);
    CK(cudaStreamSynchronize(ctx->c.copy));
    CK(cudaStreamSynchronize(ctx->c.aux));
    CK(cudaStreamSynchronize(ctx->c.comp));
  });
}

// ---- coarse ----------------------------------------------------------------
namespace {
void coarse_batch(Ctx& c, const float* Q, uint32_t nq, uint32_t n_out,
                  uint32_t* order_out, double* scores_out) {
  need(Q, "queries");
  const uint32_t d = c.ix->d, nc = c.ix->nc;
  for (uint32_t q0 = 0; q0 < nq; q0 += c.max_batch) {
    const uint32_t b = std::min(c.max_batch, nq - q0);
    std::memcpy(c.h_Q, Q + size_t(q0) * d, size_t(b) * d * sizeof(float));
    CK(cudaMemcpyAsync(c.d_Q, c.h_Q, size_t(b) * d * sizeof(float), cudaMemcpyHostToDevice, c.comp));
    c.coarse(c.d_Q, b, n_out, c.comp, false, scores_out != nullptr);
    if (n_out) {
      CK(cudaMemcpyAsync(c.h_order, c.d_order, size_t(b) * n_out * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost, c.comp));
    }
    if (scores_out) {
      CK(cudaMemcpyAsync(scores_out + size_t(q0) * nc, c.d_scores, size_t(b) * nc * sizeof(double),
                         cudaMemcpyDeviceToHost, c.comp));
    }
    CK(cudaStreamSynchronize(c.comp));
    if (n_out) std::memcpy(order_out + size_t(q0) * n_out, c.h_order, size_t(b) * n_out * sizeof(uint32_t));
  }
}
} // namespace

int laivg_rank_clusters(laivg_ctx* ctx, const float* Q, uint32_t nq, uint32_t* order_out,
                        double* scores_out) {
  return guard([&] {
    set_ctx_device(ctx);
    need(order_out, "order_out");
    coarse_batch(ctx->c, Q, nq, ctx->c.ix->nc, order_out, scores_out);
  });
}

int laivg_coarse_probe(laivg_ctx* ctx, const float* Q, uint32_t nq, int L, uint32_t* probe_out,
                       uint32_t* lp_out) {
  return guard([&] {
    set_ctx_device(ctx);
    const uint32_t lp = uint32_t(std::min<int64_t>(std::max(L, 0), ctx->c.ix->nc));
    if (lp_out) *lp_out = lp;
    if (lp) need(probe_out, "probe_out");
    coarse_batch(ctx->c, Q, nq, lp, probe_out, nullptr);
  });
}

// ---- fine search -------------------------------------------------------------
int laivg_search_clusters(laivg_ctx* ctx, const float* q, const uint32_t* clusters, uint32_t n,
                          int k, uint64_t* ids_out, float* scores_out, uint32_t* count_out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    need(ids_out, "ids_out");
    need(scores_out, "scores_out");
    if (n) need(clusters, "clusters");
    Ctx& c = ctx->c;
    stage_query(c, q);
    std::vector<uint32_t> probe(clusters, clusters + n);
    auto r = c.search(c.h_Q, q, 0, k, &probe);
    write_top(r.top, k, ids_out, scores_out, count_out);
  });
}

int laivg_ivf_search(laivg_ctx* ctx, const float* Q, uint32_t nq, int L, int k, uint64_t* ids_out,
                     float* scores_out, uint32_t* count_out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    need(ids_out, "ids_out");
    need(scores_out, "scores_out");
    Ctx& c = ctx->c;
    if (nq) need(Q, "queries");
    if (nq == 1) {
      stage_query(c, Q);
      auto r = c.search(c.h_Q, Q, L, k, nullptr);
      write_top(r.top, k, ids_out, scores_out, count_out);
      return;
    }
    for (uint32_t q0 = 0; q0 < nq; q0 += c.max_batch) {
      const uint32_t b = std::min(c.max_batch, nq - q0);
      const float* Qb = Q + size_t(q0) * c.ix->d;
      stage_batch(c, Qb, b);
      auto r = c.search_batch(c.d_Q, Qb, b, L, k);
      for (uint32_t i = 0; i < b; ++i) {
        write_top(r.top[i], k, ids_out + size_t(q0 + i) * k, scores_out + size_t(q0 + i) * k,
                  count_out ? count_out + q0 + i : nullptr);
      }
    }
  });
}

int laivg_score_clusters(laivg_ctx* ctx, const float* q, const uint32_t* clusters, uint32_t n,
                         uint64_t cap, uint64_t* ids_out, float* scores_out, uint64_t* count_out) {
  return guard([&] {
    set_ctx_device(ctx);
    need(q, "query");
    if (n) need(clusters, "clusters");
    if (cap) {
      need(ids_out, "ids_out");
      need(scores_out, "scores_out");
    }
    const uint64_t m = ctx->c.score_clusters(q, clusters, n, cap, scores_out, ids_out);
    if (count_out) *count_out = m;
  });
}

int laivg_exact_search(laivg_ctx* ctx, const float* Q, uint32_t nq, int k, uint64_t* ids_out,
                       float* scores_out, uint32_t* count_out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    if (nq) {
      need(Q, "queries");
      need(ids_out, "ids_out");
      need(scores_out, "scores_out");
    }
    Ctx& c = ctx->c;
    // every row of the datastore is a member of exactly one list: the union
    // of all lists is the datastore (test_ivf.cpp:213-222)
    std::vector<uint32_t> all(c.ix->nc);
    for (uint32_t i = 0; i < c.ix->nc; ++i) all[i] = i;
    for (uint32_t i = 0; i < nq; ++i) {
      const float* q = Q + size_t(i) * c.ix->d;
      stage_query(c, q);
      auto r = c.search(c.h_Q, q, 0, k, &all);
      write_top(r.top, k, ids_out + size_t(i) * k, scores_out + size_t(i) * k,
                count_out ? count_out + i : nullptr);
    }
  });
}

int laivg_pairwise_l2(laivg_ctx* ctx, const float* a, uint64_t na, const float* b, uint64_t nb,
                      uint32_t d, float* out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (na == 0 || nb == 0) return;
    need(a, "a");
    need(b, "b");
    need(out, "out");
    if (d == 0) throw std::invalid_argument("pairwise_l2: dimension must be > 0");
    Ctx& c = ctx->c;
    // rows of a in chunks so one chunk's output stays <= 256 MB of HBM
    const uint64_t rows = std::max<uint64_t>(1, std::min<uint64_t>(na, (64ull << 20) / nb));
    float* dA = laivg::dev_alloc<float>(rows * d);
    float* dB = laivg::dev_alloc<float>(nb * d);
    float* dO = laivg::dev_alloc<float>(rows * nb);
    try {
      CK(cudaMemcpyAsync(dB, b, nb * d * sizeof(float), cudaMemcpyDefault, c.comp));
      for (uint64_t r0 = 0; r0 < na; r0 += rows) {
        const uint64_t m = std::min(rows, na - r0);
        CK(cudaMemcpyAsync(dA, a + r0 * d, m * d * sizeof(float), cudaMemcpyDefault, c.comp));
        laivg::launch_pairwise_l2(dA, m, dB, nb, d, dO, nullptr, c.comp);
        CK(cudaMemcpyAsync(out + r0 * nb, dO, m * nb * sizeof(float), cudaMemcpyDefault, c.comp));
      }
      CK(cudaStreamSynchronize(c.comp));
    } catch (...) {
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dO);
      throw;
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
  });
}

// ---- store -------------------------------------------------------------------
uint64_t laivg_store_capacity_bytes(const laivg_ctx* ctx) { return ctx ? ctx->c.capacity : 0; }
uint64_t laivg_store_used_bytes(const laivg_ctx* ctx) { return ctx ? ctx->c.used : 0; }
uint64_t laivg_store_free_bytes(const laivg_ctx* ctx) {
  return ctx ? ctx->c.free_bytes() : 0;
}
int laivg_store_contains(const laivg_ctx* ctx, uint32_t c) {
  return ctx && ctx->c.resident.count(c) ? 1 : 0;
}
uint32_t laivg_store_resident_count(const laivg_ctx* ctx) {
  return ctx ? uint32_t(ctx->c.resident.size()) : 0;
}
int laivg_store_resident(const laivg_ctx* ctx, uint32_t* clusters_out, uint8_t* tags_out,
                         uint64_t* bytes_out, uint32_t* n_out) {
  return guard([&] {
    need(ctx, "ctx");
    uint32_t i = 0;
    for (auto& [c, r] : ctx->c.resident) {
      if (clusters_out) clusters_out[i] = c;
      if (tags_out) tags_out[i] = uint8_t(r.tag);
      if (bytes_out) bytes_out[i] = r.bytes;
      ++i;
    }
    if (n_out) *n_out = i;
  });
}
int laivg_store_insert(laivg_ctx* ctx, uint32_t c, int tag) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    x.copy_after_comp();
    x.insert_async(c, tag);
    x.commit_res(x.copy);
    CK(cudaEventRecord(x.ev_copy_tail, x.copy));
    CK(cudaStreamSynchronize(x.copy));
  });
}
int laivg_store_evict(laivg_ctx* ctx, uint32_t c, uint64_t* bytes_out) {
  return guard([&] {
    set_ctx_device(ctx);
    const uint64_t b = ctx->c.evict(c);
    if (bytes_out) *bytes_out = b;
  });
}
int laivg_store_retag_all(laivg_ctx* ctx, int tag) {
  return guard([&] {
    need(ctx, "ctx");
    for (auto& [c, r] : ctx->c.resident) r.tag = tag;
  });
}
int laivg_store_clear(laivg_ctx* ctx) {
  return guard([&] {
    set_ctx_device(ctx);
    ctx->c.clear_store();
  });
}
uint64_t laivg_store_bytes_with_tag(const laivg_ctx* ctx, int tag) {
  uint64_t s = 0;
  if (ctx) {
    for (auto& [c, r] : ctx->c.resident) {
      if (r.tag == tag) s += r.bytes;
    }
  }
  return s;
}
uint64_t laivg_store_recompute_used_bytes(const laivg_ctx* ctx) {
  uint64_t s = 0;
  if (ctx) {
    for (auto& [c, r] : ctx->c.resident) s += r.bytes;
  }
  return s;
}
int laivg_store_compact(laivg_ctx* ctx) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    x.compact();
    x.commit_res(x.copy);
    CK(cudaEventRecord(x.ev_copy_tail, x.copy));
    CK(cudaStreamSynchronize(x.copy));
  });
}

// ---- prefetch ------------------------------------------------------------------
int laivg_plan_prefetch(laivg_ctx* ctx, const float* q_in, uint64_t budget_bytes,
                        uint32_t* plan_out, uint32_t* nplan_out, uint64_t* planned_bytes_out,
                        uint32_t* skipped_out, uint32_t* nskipped_out) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    std::vector<uint32_t> order(x.ix->nc);
    coarse_batch(x, q_in, 1, x.ix->nc, order.data(), nullptr);
    std::vector<uint32_t> plan, skipped;
    uint64_t planned = 0;
    laivg::plan_walk(*x.ix, order.data(), [&](uint32_t c) { return x.h_res[c] >= 0; },
                     budget_bytes, plan, planned, skipped);
    if (plan_out) std::copy(plan.begin(), plan.end(), plan_out);
    if (skipped_out) std::copy(skipped.begin(), skipped.end(), skipped_out);
    if (nplan_out) *nplan_out = uint32_t(plan.size());
    if (nskipped_out) *nskipped_out = uint32_t(skipped.size());
    if (planned_bytes_out) *planned_bytes_out = planned;
  });
}

int laivg_execute_prefetch(laivg_ctx* ctx, const uint32_t* plan, uint32_t n,
                           const laivg_channel* chan, double overlap_window_s,
                           uint32_t* transferred_out, laivg_transfer_report* rep) {
  return guard([&] {
    set_ctx_device(ctx);
    need(chan, "chan");
    if (n) need(plan, "plan");
    Ctx& x = ctx->c;
    laivg_transfer_report r{};
    const int mode = chan->mode;
    if (mode != LAIVG_CHAN_SIMULATED && mode != LAIVG_CHAN_MEASURED && mode != LAIVG_CHAN_DEVICE) {
      throw std::invalid_argument("bad channel mode");
    }
    if (mode == LAIVG_CHAN_SIMULATED && !(chan->bandwidth_bytes_per_s > 0)) {
      throw std::invalid_argument("bandwidth must be positive");
    }
    uint64_t bytes = 0;
    const auto w0 = Clock::now();
    CK(cudaEventRecord(x.ev_base, x.comp));
    CK(cudaStreamWaitEvent(x.copy, x.ev_base, 0));
    const bool win = mode == LAIVG_CHAN_DEVICE && overlap_window_s > 0;
    if (win) x.launch_window_any(overlap_window_s);
    CK(cudaEventRecord(x.ev_win, x.comp));
    CK(cudaEventRecord(x.ev_cp0, x.copy));
    uint32_t done = 0;
    try {
      for (uint32_t i = 0; i < n; ++i) {
        if (!x.try_insert_async(plan[i], LAIVG_TAG_PREFETCHED)) continue; // fragmented epoch
        bytes += x.ix->cluster_bytes(plan[i]);
        if (transferred_out) transferred_out[done] = plan[i];
        ++done;
      }
    } catch (...) {
      // Reference semantics: clusters inserted before the failure stay.
      x.commit_res(x.copy);
      CK(cudaEventRecord(x.ev_copy_tail, x.copy));
      CK(cudaStreamSynchronize(x.copy));
      CK(cudaStreamSynchronize(x.comp));
      throw;
    }
    x.commit_res(x.copy);
    CK(cudaEventRecord(x.ev_cp1, x.copy));
    CK(cudaEventRecord(x.ev_copy_tail, x.copy));
    CK(cudaEventSynchronize(x.ev_cp1));
    CK(cudaEventSynchronize(x.ev_win));
    const double wall = std::chrono::duration<double>(Clock::now() - w0).count();
    float ms_cp = 0, ms_win = 0, ms_end = 0;
    CK(cudaEventElapsedTime(&ms_cp, x.ev_cp0, x.ev_cp1));
    CK(cudaEventElapsedTime(&ms_win, x.ev_base, x.ev_win));
    CK(cudaEventElapsedTime(&ms_end, x.ev_base, x.ev_cp1));
    r.bytes = bytes;
    r.n_transferred = done;
    r.window_s = win ? ms_win * 1e-3 : 0.0;
    r.h2d_gbps = ms_cp > 0 ? double(bytes) / (ms_cp * 1e-3) / 1e9 : 0.0;
    r.window_read_gbps = win ? x.window_read_gbps(r.window_s) : 0.0;
    if (mode == LAIVG_CHAN_SIMULATED) {
      r.t_p = double(bytes) / chan->bandwidth_bytes_per_s; // tiered.cpp:131
      r.overshoot_s = std::max(0.0, r.t_p - overlap_window_s);
    } else if (mode == LAIVG_CHAN_MEASURED) {
      r.t_p = wall;
      r.overshoot_s = std::max(0.0, r.t_p - overlap_window_s);
    } else {
      r.t_p = ms_cp * 1e-3;
      // exposed transfer: copy end past window end (both from ev_base)
      r.overshoot_s = std::max(0.0, double(ms_end - (win ? ms_win : 0.0f)) * 1e-3);
    }
    if (rep) *rep = r;
  });
}

int laivg_prefetch_batch(laivg_ctx* ctx, const float* Q_in, uint32_t nq,
                         const uint64_t* budgets, const laivg_channel* chan,
                         double overlap_window_s, uint32_t* transferred_out,
                         uint32_t* nplan_out, laivg_transfer_report* rep) {
  return guard([&] {
    set_ctx_device(ctx);
    need(chan, "chan");
    if (chan->mode != LAIVG_CHAN_DEVICE) {
      throw std::invalid_argument("prefetch_batch runs on the device channel");
    }
    Ctx& x = ctx->c;
    const uint32_t nc = x.ix->nc;
    if (nq) {
      need(Q_in, "queries");
      need(budgets, "budgets");
    }
    // one coarse pass ranks every predictor embedding of the micro-batch
    std::vector<uint32_t> order(size_t(nq) * nc);
    if (nq) coarse_batch(x, Q_in, nq, nc, order.data(), nullptr);
    laivg_transfer_report r{};
    const auto w0 = Clock::now();
    (void)w0;
    CK(cudaEventRecord(x.ev_base, x.comp));
    CK(cudaStreamWaitEvent(x.copy, x.ev_base, 0));
    const bool win = overlap_window_s > 0;
    if (win) x.launch_window_any(overlap_window_s);
    CK(cudaEventRecord(x.ev_win, x.comp));
    CK(cudaEventRecord(x.ev_cp0, x.copy));
    uint64_t bytes = 0;
    uint32_t done = 0;
    try {
      // pipeline.cpp:357-371: each query plans against the store already
      // holding the earlier plans (shared clusters travel once), with budget
      // min(budget_i, free bytes); the transfers share the copy stream
      for (uint32_t q = 0; q < nq; ++q) {
        std::vector<uint32_t> plan, skipped;
        uint64_t planned = 0;
        const uint64_t budget = std::min<uint64_t>(budgets[q], x.free_bytes());
        laivg::plan_walk(*x.ix, order.data() + size_t(q) * nc,
                         [&](uint32_t c) { return x.h_res[c] >= 0; }, budget, plan, planned,
                         skipped);
        for (uint32_t c : plan) {
          if (!x.try_insert_async(c, LAIVG_TAG_PREFETCHED)) continue; // fragmented epoch
          bytes += x.ix->cluster_bytes(c);
          if (transferred_out) transferred_out[done] = c;
          ++done;
        }
        if (nplan_out) nplan_out[q] = uint32_t(plan.size());
      }
    } catch (...) {
      x.commit_res(x.copy);
      CK(cudaEventRecord(x.ev_copy_tail, x.copy));
      CK(cudaStreamSynchronize(x.copy));
      CK(cudaStreamSynchronize(x.comp));
      throw;
    }
    x.commit_res(x.copy);
    CK(cudaEventRecord(x.ev_cp1, x.copy));
    CK(cudaEventRecord(x.ev_copy_tail, x.copy));
    CK(cudaEventSynchronize(x.ev_cp1));
    CK(cudaEventSynchronize(x.ev_win));
    float ms_cp = 0, ms_win = 0, ms_end = 0;
    CK(cudaEventElapsedTime(&ms_cp, x.ev_cp0, x.ev_cp1));
    CK(cudaEventElapsedTime(&ms_win, x.ev_base, x.ev_win));
    CK(cudaEventElapsedTime(&ms_end, x.ev_base, x.ev_cp1));
    r.bytes = bytes;
    r.n_transferred = done;
    r.window_s = win ? ms_win * 1e-3 : 0.0;
    r.h2d_gbps = ms_cp > 0 ? double(bytes) / (ms_cp * 1e-3) / 1e9 : 0.0;
    r.window_read_gbps = win ? x.window_read_gbps(r.window_s) : 0.0;
    r.t_p = ms_cp * 1e-3;
    r.overshoot_s = std::max(0.0, double(ms_end - (win ? ms_win : 0.0f)) * 1e-3);
    if (rep) *rep = r;
  });
}

int laivg_incremental_prefetch(laivg_ctx* ctx, const float* q_round, uint64_t budget_bytes,
                               const laivg_channel* chan, double overlap_window_s,
                               uint32_t* transferred_out, laivg_transfer_report* rep) {
  return guard([&] {
    need(ctx, "ctx");
    std::vector<uint32_t> plan(ctx->c.ix->nc), skipped(ctx->c.ix->nc);
    uint32_t np = 0, ns = 0;
    uint64_t pb = 0;
    int rc = laivg_plan_prefetch(ctx, q_round, budget_bytes, plan.data(), &np, &pb,
                                 skipped.data(), &ns);
    if (rc) throw std::runtime_error(laivg::g_err);
    rc = laivg_execute_prefetch(ctx, plan.data(), np, chan, overlap_window_s, transferred_out, rep);
    if (rc == LAIVG_ELOGIC) throw std::logic_error(laivg::g_err);
    if (rc == LAIVG_ECUDA) throw laivg::CudaError(laivg::g_err);
    if (rc == LAIVG_EINVAL) throw std::invalid_argument(laivg::g_err);
    if (rc) throw std::runtime_error(laivg::g_err);
  });
}

int laivg_window(laivg_ctx* ctx, double seconds, double* measured_s) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    CK(cudaEventRecord(x.ev_base, x.comp));
    x.launch_window_any(seconds);
    CK(cudaEventRecord(x.ev_win, x.comp));
    CK(cudaEventSynchronize(x.ev_win));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, x.ev_base, x.ev_win));
    if (measured_s) *measured_s = ms * 1e-3;
  });
}

int laivg_window_load(laivg_ctx* ctx, uint64_t buffer_bytes, double read_gbps) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    if (read_gbps < 0) throw std::invalid_argument("read_gbps must be >= 0");
    CK(cudaStreamSynchronize(x.comp));
    if (x.d_wbuf && (buffer_bytes == 0 || buffer_bytes != x.wbuf_bytes)) {
      CK(cudaFree(x.d_wbuf));
      x.d_wbuf = nullptr;
      x.wbuf_bytes = 0;
    }
    buffer_bytes &= ~uint64_t(63);
    if (buffer_bytes && !x.d_wbuf) {
      x.d_wbuf = laivg::dev_alloc<float>(buffer_bytes / sizeof(float));
      CK(cudaMemset(x.d_wbuf, 0, buffer_bytes));
      x.wbuf_bytes = buffer_bytes;
      if (!x.d_wsink) x.d_wsink = laivg::dev_alloc<float>(1);
      if (!x.d_wread) x.d_wread = laivg::dev_alloc<unsigned long long>(1);
    }
    x.w_rate = read_gbps * 1e9;
  });
}

int laivg_link_bytes(const laivg_ctx* ctx, uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  return guard([&] {
    need(ctx, "ctx");
    if (h2d_bytes) *h2d_bytes = ctx->c.link_h2d_total;
    if (d2h_bytes) *d2h_bytes = ctx->c.link_d2h_total;
  });
}

int laivg_list_scan_stats(const laivg_ctx* ctx, uint64_t* runs, uint64_t* fallbacks,
                          double* queries_per_list) {
  return guard([&] {
    need(ctx, "ctx");
    if (runs) *runs = ctx->c.ls_runs;
    if (fallbacks) *fallbacks = ctx->c.ls_fallbacks;
    if (queries_per_list) *queries_per_list = ctx->c.ls_qpl;
  });
}

int laivg_link_peak(laivg_ctx* ctx, uint64_t bytes, double* h2d_gbps, double* d2h_gbps) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    if (bytes == 0) throw std::invalid_argument("bytes must be > 0");
    void* h = nullptr;
    void* d = nullptr;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocPortable));
    try {
      std::memset(h, 1, bytes);
      d = laivg::dev_alloc<unsigned char>(bytes);
      cudaStream_t st = x.aux;
      auto timed = [&](cudaMemcpyKind kind) {
        void* dst = kind == cudaMemcpyHostToDevice ? d : h;
        const void* src = kind == cudaMemcpyHostToDevice ? h : d;
        CK(cudaMemcpyAsync(dst, src, bytes, kind, st)); // warm the path
        CK(cudaEventRecord(x.ev_cp0, st));
        for (int i = 0; i < 3; ++i) CK(cudaMemcpyAsync(dst, src, bytes, kind, st));
        CK(cudaEventRecord(x.ev_cp1, st));
        CK(cudaEventSynchronize(x.ev_cp1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, x.ev_cp0, x.ev_cp1));
        return 3.0 * double(bytes) / (ms * 1e-3) / 1e9;
      };
      const double a = timed(cudaMemcpyHostToDevice);
      const double b = timed(cudaMemcpyDeviceToHost);
      if (h2d_gbps) *h2d_gbps = a;
      if (d2h_gbps) *d2h_gbps = b;
    } catch (...) {
      if (d) cudaFree(d);
      cudaFreeHost(h);
      throw;
    }
    CK(cudaFree(d));
    CK(cudaFreeHost(h));
  });
}

// ---- hybrid ----------------------------------------------------------------------
int laivg_hybrid_search(laivg_ctx* ctx, const float* q_out, int L, int k,
                        const laivg_cost_model* cost, uint64_t* ids_out, float* scores_out,
                        uint32_t* count_out, uint32_t* fast_out, uint32_t* nfast_out,
                        uint32_t* slow_out, uint32_t* nslow_out, double* hit_rate_out,
                        laivg_hybrid_timing* timing) {
  return guard([&] {
    set_ctx_device(ctx);
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    need(ids_out, "ids_out");
    need(scores_out, "scores_out");
    Ctx& c = ctx->c;
    stage_query(c, q_out);
    c.want_timing = timing != nullptr;
    auto r = [&] {
      try {
        return c.search(c.h_Q, q_out, L, k, nullptr);
      } catch (...) {
        c.want_timing = true;
        throw;
      }
    }();
    c.want_timing = true;
    r.h2d_bytes += uint64_t(c.ix->d) * sizeof(float); // the query row
    c.link_h2d_total += uint64_t(c.ix->d) * sizeof(float);
    write_top(r.top, k, ids_out, scores_out, count_out);
    if (fast_out) std::copy(r.fast.begin(), r.fast.end(), fast_out);
    if (slow_out) std::copy(r.slow.begin(), r.slow.end(), slow_out);
    if (nfast_out) *nfast_out = uint32_t(r.fast.size());
    if (nslow_out) *nslow_out = uint32_t(r.slow.size());
    const size_t probed = r.fast.size() + r.slow.size();
    if (hit_rate_out) *hit_rate_out = probed ? double(r.fast.size()) / double(probed) : 0.0;
    fill_timing(timing, r, cost);
  });
}

int laivg_coverage(laivg_ctx* ctx, const float* q_in, const float* q_out, int L, double* out) {
  return guard([&] {
    set_ctx_device(ctx);
    need(q_in, "q_in");
    need(q_out, "q_out");
    need(out, "out");
    Ctx& c = ctx->c;
    const uint32_t d = c.ix->d;
    const uint32_t lp = uint32_t(std::min<int64_t>(std::max(L, 0), c.ix->nc));
    if (lp == 0) {
      *out = 0.0;
      return;
    }
    std::vector<float> Q(size_t(2) * d);
    std::memcpy(Q.data(), q_in, d * sizeof(float));
    std::memcpy(Q.data() + d, q_out, d * sizeof(float));
    std::vector<uint32_t> probe(size_t(2) * lp);
    coarse_batch(c, Q.data(), 2, lp, probe.data(), nullptr);
    std::unordered_set<uint32_t> in(probe.begin(), probe.begin() + lp);
    size_t overlap = 0;
    for (uint32_t i = 0; i < lp; ++i) overlap += in.count(probe[lp + i]);
    *out = double(overlap) / double(lp);
  });
}

int laivg_stage_queries(laivg_ctx* ctx, const float* Q, uint32_t nq) {
  return guard([&] {
    set_ctx_device(ctx);
    need(Q, "queries");
    Ctx& c = ctx->c;
    if (c.d_staged) {
      CK(cudaFree(c.d_staged));
      c.d_staged = nullptr;
    }
    const size_t n = size_t(nq) * c.ix->d;
    c.d_staged = laivg::dev_alloc<float>(n);
    CK(cudaMemcpy(c.d_staged, Q, n * sizeof(float), cudaMemcpyHostToDevice));
    c.staged_host.assign(Q, Q + n);
    c.n_staged = nq;
  });
}

int laivg_hybrid_search_staged(laivg_ctx* ctx, uint32_t qi, int L, int k, uint64_t* ids_out,
                               float* scores_out, uint32_t* count_out, uint32_t* nfast_out,
                               laivg_hybrid_timing* timing) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& c = ctx->c;
    if (qi >= c.n_staged) throw std::invalid_argument("staged query index out of range");
    const size_t off = size_t(qi) * c.ix->d;
    auto r = c.search(c.d_staged + off, c.staged_host.data() + off, L, k, nullptr);
    if (ids_out && scores_out) write_top(r.top, k, ids_out, scores_out, count_out);
    if (nfast_out) *nfast_out = uint32_t(r.fast.size());
    fill_timing(timing, r, nullptr);
  });
}

int laivg_hybrid_search_batch(laivg_ctx* ctx, const float* Q, uint32_t nq, int L, int k,
                              const laivg_cost_model* cost, uint64_t* ids_out,
                              float* scores_out, uint32_t* count_out, uint32_t* nfast_out,
                              laivg_hybrid_timing* timing) {
  return guard([&] {
    set_ctx_device(ctx);
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    need(ids_out, "ids_out");
    need(scores_out, "scores_out");
    if (nq) need(Q, "queries");
    Ctx& c = ctx->c;
    if (nq > c.max_batch) throw std::invalid_argument("batch exceeds the context's max_batch");
    stage_batch(c, Q, nq);
    auto r = c.search_batch(c.d_Q, Q, nq, L, k);
    r.h2d_bytes += uint64_t(nq) * c.ix->d * sizeof(float); // the query rows
    for (uint32_t i = 0; i < nq; ++i) {
      write_top(r.top[i], k, ids_out + size_t(i) * k, scores_out + size_t(i) * k,
                count_out ? count_out + i : nullptr);
      if (nfast_out) nfast_out[i] = r.nfast[i];
    }
    fill_batch_timing(timing, r, cost);
  });
}

int laivg_hybrid_search_batch_staged(laivg_ctx* ctx, uint32_t q0, uint32_t nq, int L, int k,
                                     uint64_t* ids_out, float* scores_out, uint32_t* count_out,
                                     uint32_t* nfast_out, laivg_hybrid_timing* timing) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& c = ctx->c;
    if (uint64_t(q0) + nq > c.n_staged) throw std::invalid_argument("staged range out of range");
    if (nq > c.max_batch) throw std::invalid_argument("batch exceeds the context's max_batch");
    const size_t off = size_t(q0) * c.ix->d;
    auto r = c.search_batch(c.d_staged + off, c.staged_host.data() + off, nq, L, k);
    for (uint32_t i = 0; i < nq; ++i) {
      if (ids_out && scores_out) {
        write_top(r.top[i], k, ids_out + size_t(i) * k, scores_out + size_t(i) * k,
                  count_out ? count_out + i : nullptr);
      }
      if (nfast_out) nfast_out[i] = r.nfast[i];
    }
    fill_batch_timing(timing, r, nullptr);
  });
}

int laivg_debug_coarse_approx(laivg_ctx* ctx, const float* Q, uint32_t nq, float* approx_out) {
  return guard([&] {
    set_ctx_device(ctx);
    need(Q, "queries");
    need(approx_out, "approx_out");
    Ctx& c = ctx->c;
    if (!c.tc_ok) throw std::invalid_argument("tensor-core coarse quantizer unsupported here");
    const uint32_t nc = c.ix->nc;
    for (uint32_t q0 = 0; q0 < nq; q0 += c.max_batch) {
      const uint32_t b = std::min(c.max_batch, nq - q0);
      stage_batch(c, Q + size_t(q0) * c.ix->d, b);
      const uint32_t S =
          laivg::launch_coarse_tc(c.d_Q, b, c.d_cen, nc, c.ix->d, c.d_approx, c.sms, c.comp);
      std::vector<float> planes(size_t(S) * b * nc);
      CK(cudaMemcpyAsync(planes.data(), c.d_approx, planes.size() * sizeof(float),
                         cudaMemcpyDeviceToHost, c.comp));
      CK(cudaStreamSynchronize(c.comp));
      for (size_t i = 0; i < size_t(b) * nc; ++i) { // plane sum, as tc_select forms it
        double a = planes[i];
        for (uint32_t z = 1; z < S; ++z) a += planes[size_t(z) * b * nc + i];
        approx_out[size_t(q0) * nc + i] = static_cast<float>(a);
      }
      CK(cudaStreamSynchronize(c.comp));
    }
  });
}

// ---- the slow tier on its own ---------------------------------------------------
int laivg_slow_tier_scan(const laivg_index* ix, const float* Q, uint32_t nq,
                         const uint32_t* lists, const uint32_t* lists_off, int k,
                         uint32_t threads, uint64_t* ids_out, float* scores_out,
                         uint32_t* count_out) {
  return guard([&] {
    need(ix, "index");
    if (k < 1) throw std::invalid_argument("k must be >= 1");
    if (nq) {
      need(Q, "queries");
      need(lists_off, "lists_off");
      need(ids_out, "ids_out");
      need(scores_out, "scores_out");
    }
    const laivg::Index& x = ix->ix;
    std::vector<std::vector<uint32_t>> slow(nq);
    for (uint32_t q = 0; q < nq; ++q) {
      for (uint32_t i = lists_off[q]; i < lists_off[q + 1]; ++i) {
        if (lists[i] >= x.nc) {
          throw std::invalid_argument("unknown cluster id " + std::to_string(lists[i]));
        }
        slow[q].push_back(lists[i]);
      }
    }
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    laivg::ThreadPool pool(threads - 1);
    const auto top = laivg::miss_scan_batch(x, Q, nq, slow, k, pool);
    for (uint32_t q = 0; q < nq; ++q) {
      write_top(top[q], k, ids_out + size_t(q) * k, scores_out + size_t(q) * k,
                count_out ? count_out + q : nullptr);
    }
  });
}

// ---- peer caches ---------------------------------------------------------------
int laivg_epoch_open(laivg_ctx* ctx) {
  return guard([&] {
    set_ctx_device(ctx);
    if (ctx->c.epoch) throw std::logic_error("a peer epoch is already open");
    ctx->c.epoch_open();
  });
}
int laivg_epoch_close(laivg_ctx* ctx) {
  return guard([&] {
    set_ctx_device(ctx);
    Ctx& c = ctx->c;
    // peer copies issued by this context must be done before its own
    // view of the peers is dropped; its quarantine returns to the allocator
    CK(cudaStreamSynchronize(c.copy));
    c.epoch_close();
  });
}
int laivg_store_offsets(const laivg_ctx* ctx, int64_t* off_out) {
  return guard([&] {
    need(ctx, "ctx");
    need(off_out, "off_out");
    const Ctx& c = ctx->c;
    for (uint32_t i = 0; i < c.ix->nc; ++i) { // inside an epoch: the published lists
      off_out[i] = (!c.epoch || c.is_pinned(i)) ? c.h_res[i] : -1;
    }
  });
}
int laivg_slab_ipc_handle(laivg_ctx* ctx, void* handle_out) {
  return guard([&] {
    set_ctx_device(ctx);
    need(handle_out, "handle_out");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ctx->c.d_slab));
    std::memcpy(handle_out, &h, sizeof(h));
  });
}
namespace {
laivg::Ctx::Peer& peer_slot(Ctx& c, uint32_t peer) {
  if (peer > 1024) throw std::invalid_argument("peer index out of range");
  if (c.peers.size() <= peer) c.peers.resize(peer + 1);
  return c.peers[peer];
}
} // namespace
int laivg_peer_attach_ipc(laivg_ctx* ctx, uint32_t peer, const void* handle) {
  return guard([&] {
    set_ctx_device(ctx);
    need(handle, "handle");
    auto& p = peer_slot(ctx->c, peer);
    if (p.ipc) throw std::logic_error("peer already attached");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p.ipc = ptr;
    p.slab = static_cast<const float*>(ptr);
    cudaPointerAttributes at{};
    CK(cudaPointerGetAttributes(&at, ptr));
    p.dev = at.device;
  });
}
int laivg_peer_attach_local(laivg_ctx* ctx, uint32_t peer, const laivg_ctx* other) {
  return guard([&] {
    set_ctx_device(ctx);
    need(other, "other");
    if (other->c.ix->nc != ctx->c.ix->nc || other->c.ix->d != ctx->c.ix->d) {
      throw std::invalid_argument("peer serves a different index");
    }
    if (other->c.dev != ctx->c.dev) {
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, ctx->c.dev, other->c.dev));
      if (!ok) throw laivg::CudaError("no peer access between the two devices");
      const cudaError_t e = cudaDeviceEnablePeerAccess(other->c.dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
    peer_slot(ctx->c, peer).slab = other->c.d_slab;
    peer_slot(ctx->c, peer).dev = other->c.dev;
  });
}
int laivg_peer_publish(laivg_ctx* ctx, uint32_t peer, const int64_t* offsets) {
  return guard([&] {
    need(ctx, "ctx");
    if (!ctx->c.epoch) {
      throw std::logic_error("peer offsets are only valid inside an open epoch");
    }
    auto& p = peer_slot(ctx->c, peer);
    if (!p.slab) throw std::logic_error("peer not attached");
    if (offsets) p.off.assign(offsets, offsets + ctx->c.ix->nc);
    else p.off.clear();
  });
}

// ---- schedulers ----------------------------------------------------------------
int laivg_group_microbatches(const float* queries, uint64_t n, uint32_t d, uint64_t m,
                             uint64_t* order_out, uint64_t* batch_off_out, uint32_t* nb_out) {
  return guard([&] {
    if (n) need(queries, "queries");
    std::vector<uint64_t> order, off;
    static laivg::ThreadPool pool(std::max(1u, std::thread::hardware_concurrency()) - 1);
    laivg::group_microbatches(queries, n, d, m, order, off, &pool);
    std::copy(order.begin(), order.end(), order_out);
    std::copy(off.begin(), off.end(), batch_off_out);
    if (nb_out) *nb_out = uint32_t(off.size() - 1);
  });
}

int laivg_chunk_microbatches(uint64_t n, uint64_t m, uint64_t* order_out, uint64_t* batch_off_out,
                             uint32_t* nb_out) {
  return guard([&] {
    if (m < 1) throw std::invalid_argument("micro-batch size must be >= 1");
    uint32_t nb = 0;
    batch_off_out[0] = 0;
    for (uint64_t i = 0; i < n; i += m) {
      for (uint64_t j = i; j < std::min(i + m, n); ++j) order_out[j] = j;
      batch_off_out[++nb] = std::min(i + m, n);
    }
    if (nb_out) *nb_out = nb;
  });
}

namespace {
// overlap[b][w] = |probe union of batch b  ∩  resident set of worker w|
// (sched.cpp:15-35, 99-108); probes from the GPU coarse quantizer.
std::vector<uint64_t> overlap_matrix(Ctx& c, const uint64_t* off, const uint64_t* mem,
                                     uint32_t nb, const uint8_t* resident, uint32_t nw,
                                     const float* queries, uint64_t nq, int L) {
  const uint32_t nc = c.ix->nc;
  const uint32_t lp = uint32_t(std::min<int64_t>(std::max(L, 0), nc));
  std::vector<uint32_t> probe(size_t(nq) * lp);
  if (lp && nq) coarse_batch(c, queries, uint32_t(nq), lp, probe.data(), nullptr);
  std::vector<uint64_t> ov(size_t(nb) * nw, 0);
  std::vector<uint8_t> mark(nc);
  for (uint32_t b = 0; b < nb; ++b) {
    std::fill(mark.begin(), mark.end(), 0);
    for (uint64_t i = off[b]; i < off[b + 1]; ++i) {
      if (mem[i] >= nq) throw std::out_of_range("query index out of range");
      for (uint32_t j = 0; j < lp; ++j) mark[probe[size_t(mem[i]) * lp + j]] = 1;
    }
    for (uint32_t w = 0; w < nw; ++w) {
      uint64_t s = 0;
      const uint8_t* r = resident + size_t(w) * nc;
      for (uint32_t x = 0; x < nc; ++x) s += mark[x] & (r[x] != 0);
      ov[size_t(b) * nw + w] = s;
    }
  }
  return ov;
}
} // namespace

int laivg_assign_cache_aware(laivg_ctx* ctx, const uint64_t* batch_off, const uint64_t* members,
                             uint32_t nb, const uint8_t* resident, uint32_t nw,
                             const float* queries, uint64_t nq, int L, uint32_t* assignment_out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (nw == 0) throw std::invalid_argument("need at least one worker");
    auto ov = overlap_matrix(ctx->c, batch_off, members, nb, resident, nw, queries, nq, L);
    auto a = laivg::greedy_assign(ov, nb, nw);
    std::copy(a.begin(), a.end(), assignment_out);
  });
}

namespace {
// group_microbatches on the device: queries already in c.sb.q; fills order /
// off on the host.
uint32_t group_on_device(Ctx& c, uint64_t n, uint64_t m, std::vector<uint64_t>& order,
                         std::vector<uint64_t>& off) {
  if (n >= (1ull << 32) || m >= (1ull << 32)) throw std::invalid_argument("too many queries");
  if (n <= laivg::group_max_queries()) {
    laivg::launch_pair_dist(c.sb.q, uint32_t(n), c.ix->d, c.sb.dist, c.comp);
    laivg::launch_group(c.sb.dist, uint32_t(n), uint32_t(m), c.sb.order, c.sb.off, c.sb.nb,
                        c.comp);
  } else {
    laivg::launch_group_large(c.sb.q, uint32_t(n), c.ix->d, uint32_t(m), c.gs, c.sb.order,
                              c.sb.off, c.sb.nb, c.sms, c.comp);
  }
  uint32_t nb = 0;
  CK(cudaMemcpyAsync(&nb, c.sb.nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, c.comp));
  CK(cudaStreamSynchronize(c.comp));
  order.resize(n);
  off.resize(size_t(nb) + 1);
  CK(cudaMemcpyAsync(order.data(), c.sb.order, n * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                     c.comp));
  CK(cudaMemcpyAsync(off.data(), c.sb.off, (size_t(nb) + 1) * sizeof(uint64_t),
                     cudaMemcpyDeviceToHost, c.comp));
  CK(cudaStreamSynchronize(c.comp));
  return nb;
}

void upload_queries(Ctx& c, const float* Q, uint64_t n) {
  CK(cudaMemcpyAsync(c.sb.q, Q, n * c.ix->d * sizeof(float), cudaMemcpyHostToDevice, c.comp));
}
} // namespace

int laivg_group_microbatches_gpu(laivg_ctx* ctx, const float* queries, uint64_t n, uint64_t m,
                                 uint64_t* order_out, uint64_t* batch_off_out, uint32_t* nb_out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (m < 1) throw std::invalid_argument("micro-batch size must be >= 1");
    Ctx& c = ctx->c;
    if (n == 0) {
      if (batch_off_out) batch_off_out[0] = 0;
      if (nb_out) *nb_out = 0;
      return;
    }
    need(queries, "queries");
    c.sched_reserve(n, 0, 0);
    upload_queries(c, queries, n);
    std::vector<uint64_t> order, off;
    const uint32_t nb = group_on_device(c, n, m, order, off);
    std::copy(order.begin(), order.end(), order_out);
    std::copy(off.begin(), off.end(), batch_off_out);
    if (nb_out) *nb_out = nb;
  });
}

int laivg_schedule(laivg_ctx* ctx, const float* queries, uint64_t n, uint64_t m, int L,
                   const uint8_t* resident, uint32_t nw, uint64_t* order_out,
                   uint64_t* batch_off_out, uint32_t* nb_out, uint32_t* assignment_out,
                   uint64_t* overlap_out) {
  return guard([&] {
    set_ctx_device(ctx);
    if (m < 1) throw std::invalid_argument("micro-batch size must be >= 1");
    if (nw == 0) throw std::invalid_argument("need at least one worker");
    Ctx& c = ctx->c;
    if (n == 0) {
      if (batch_off_out) batch_off_out[0] = 0;
      if (nb_out) *nb_out = 0;
      return;
    }
    need(queries, "queries");
    need(resident, "resident");
    const uint32_t nc = c.ix->nc, d = c.ix->d;
    const uint32_t lp = uint32_t(std::min<int64_t>(std::max(L, 0), nc));
    c.sched_reserve(n, lp, nw);
    upload_queries(c, queries, n);
    // 1. group_microbatches (sched.cpp:39-70) on the device
    std::vector<uint64_t> order, off;
    const uint32_t nb = group_on_device(c, n, m, order, off);
    // 2. every query's probe (coarse_probe, batched: tensor cores for >= 16)
    for (uint64_t q0 = 0; q0 < n && lp; q0 += c.max_batch) {
      const uint32_t b = uint32_t(std::min<uint64_t>(c.max_batch, n - q0));
      c.coarse(c.sb.q + q0 * d, b, lp, c.comp);
      CK(cudaMemcpyAsync(c.sb.probes + q0 * lp, c.d_order, size_t(b) * lp * sizeof(uint32_t),
                         cudaMemcpyDeviceToDevice, c.comp));
    }
    // 3. overlap[b][w] = |probe union of b  ∩  resident_w| as bitset popcounts
    const uint32_t words = (nc + 63) / 64;
    std::vector<unsigned long long> bits(size_t(nw) * words, 0ull);
    for (uint32_t w = 0; w < nw; ++w) {
      for (uint32_t cl = 0; cl < nc; ++cl) {
        if (resident[size_t(w) * nc + cl]) bits[size_t(w) * words + cl / 64] |= 1ull << (cl % 64);
      }
    }
    CK(cudaMemcpyAsync(c.sb.resident, bits.data(), bits.size() * sizeof(unsigned long long),
                       cudaMemcpyHostToDevice, c.comp));
    std::vector<uint64_t> ov(size_t(nb) * nw, 0);
    if (lp) {
      laivg::launch_overlap(c.sb.probes, lp, c.sb.order, c.sb.off, nb, c.sb.resident, nw, words,
                            c.sb.overlap, c.comp);
      CK(cudaMemcpyAsync(ov.data(), c.sb.overlap, ov.size() * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost, c.comp));
    }
    CK(cudaStreamSynchronize(c.comp));
    // 4. the greedy (sched.cpp:114-142) on the host
    const auto a = laivg::greedy_assign(ov, nb, nw);
    std::copy(order.begin(), order.end(), order_out);
    std::copy(off.begin(), off.end(), batch_off_out);
    if (nb_out) *nb_out = nb;
    if (assignment_out) std::copy(a.begin(), a.end(), assignment_out);
    if (overlap_out) std::copy(ov.begin(), ov.end(), overlap_out);
  });
}

int laivg_greedy_assign(const uint64_t* overlap, uint32_t nb, uint32_t nw,
                        uint32_t* assignment_out) {
  return guard([&] {
    if (nw == 0) throw std::invalid_argument("need at least one worker");
    if (nb) {
      need(overlap, "overlap");
      need(assignment_out, "assignment_out");
    }
    std::vector<uint64_t> ov(overlap, overlap + size_t(nb) * nw);
    auto a = laivg::greedy_assign(ov, nb, nw);
    std::copy(a.begin(), a.end(), assignment_out);
  });
}

int laivg_assign_round_robin(uint64_t nb, uint64_t nw, uint32_t* out) {
  return guard([&] {
    if (nw == 0) throw std::invalid_argument("need at least one worker");
    for (uint64_t b = 0; b < nb; ++b) out[b] = uint32_t(b % nw);
  });
}

int laivg_assignment_overlap(laivg_ctx* ctx, const uint64_t* batch_off, const uint64_t* members,
                             uint32_t nb, const uint8_t* resident, uint32_t nw,
                             const uint32_t* assignment, const float* queries, uint64_t nq, int L,
                             uint64_t* out) {
  return guard([&] {
    set_ctx_device(ctx);
    auto ov = overlap_matrix(ctx->c, batch_off, members, nb, resident, nw, queries, nq, L);
    uint64_t s = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      if (assignment[b] >= nw) throw std::out_of_range("assignment out of range");
      s += ov[size_t(b) * nw + assignment[b]];
    }
    *out = s;
  });
}

int laivg_split_budget(uint64_t total, const uint64_t* batch, uint64_t n, uint64_t* out) {
  return guard([&] {
    auto s = laivg::split_budget(total, batch, n);
    std::copy(s.begin(), s.end(), out);
  });
}

// ---- hotness ---------------------------------------------------------------------
int laivg_hotness_create(float h_init, float h_inc, float decay, double cache_fraction,
                         laivg_hotness** out) {
  return guard([&] {
    need(out, "out");
    *out = new laivg_hotness{laivg::Hotness(h_init, h_inc, decay, cache_fraction)};
  });
}
void laivg_hotness_destroy(laivg_hotness* h) { delete h; }
int laivg_hotness_on_fetch(laivg_hotness* h, uint32_t c) {
  return guard([&] {
    need(h, "hotness");
    h->h.on_fetch(c);
  });
}
int laivg_hotness_end_of_round(laivg_hotness* h, const uint32_t* used, uint32_t n) {
  return guard([&] {
    need(h, "hotness");
    std::unordered_set<uint32_t> u;
    if (n) u.insert(used, used + n);
    h->h.end_of_round(u);
  });
}
int laivg_hotness_evict_to_fraction(laivg_hotness* h, laivg_ctx* ctx, uint32_t* evicted_out,
                                    uint32_t* n_out) {
  return guard([&] {
    need(h, "hotness");
    set_ctx_device(ctx);
    Ctx& x = ctx->c;
    for (auto& [c, r] : x.resident) r.tag = LAIVG_TAG_CACHED; // cache.cpp:41
    const auto budget = uint64_t(h->h.fraction() * double(x.capacity));
    std::vector<uint32_t> ids;
    for (auto& [c, r] : x.resident) ids.push_back(c);
    uint32_t n = 0;
    for (uint32_t c : h->h.eviction_order(ids)) {
      if (x.used <= budget) break;
      if (x.is_pinned(c)) continue; // published to peers for this epoch
      x.evict(c);
      h->h.forget(c);
      if (evicted_out) evicted_out[n] = c;
      ++n;
    }
    if (n_out) *n_out = n;
  });
}
float laivg_hotness_get(const laivg_hotness* h, uint32_t c) {
  return h && h->h.tracked(c) ? h->h.get(c) : -1.0f;
}
int laivg_hotness_forget(laivg_hotness* h, uint32_t c) {
  return guard([&] {
    need(h, "hotness");
    h->h.forget(c);
  });
}
int laivg_hotness_clear(laivg_hotness* h) {
  return guard([&] {
    need(h, "hotness");
    h->h.clear();
  });
}

// ---- synthetic workload -------------------------------------------------------------
int laivg_synth_centroids(uint64_t seed, uint32_t nc, uint32_t d, float* centroids_out) {
  return guard([&] {
    need(centroids_out, "centroids_out");
    laivg::synth_centroids(seed, nc, d, centroids_out);
  });
}
int laivg_synth_lists(uint64_t seed, const float* centroids, uint32_t nc, uint32_t d,
                      uint64_t per_list, float spread, uint32_t c_begin, uint32_t c_end,
                      float* vecs_out, uint64_t* ids_out, int threads) {
  return guard([&] {
    need(centroids, "centroids");
    if (c_end > nc || c_begin > c_end) throw std::invalid_argument("bad cluster range");
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    laivg::synth_lists(seed, centroids, d, per_list, spread, c_begin, c_end, vecs_out,
                       ids_out, threads);
  });
}
int laivg_synth_queries(uint64_t seed, const float* vecs, uint64_t n_rows, uint32_t d, uint32_t nq,
                        float sigma, float* q_in_out, float* q_out_out, uint64_t* rows_out) {
  return guard([&] {
    need(vecs, "vecs");
    if (n_rows == 0) throw std::invalid_argument("no rows");
    laivg::synth_queries(seed, vecs, n_rows, d, nq, sigma, q_in_out, q_out_out, rows_out);
  });
}

int laivg_synth_queries_topical(uint64_t seed, const float* centroids, uint32_t nc,
                                const float* vecs, const uint64_t* list_off, uint32_t d,
                                uint32_t n_topics, double zipf_s, uint32_t neigh, uint32_t nq,
                                float sigma, float* q_in_out, float* q_out_out,
                                uint64_t* rows_out, uint32_t* topic_out) {
  return guard([&] {
    need(centroids, "centroids");
    need(vecs, "vecs");
    need(list_off, "list_off");
    laivg::synth_queries_topical(seed, centroids, nc, vecs, list_off, d, n_topics, zipf_s, neigh,
                                 nq, sigma, q_in_out, q_out_out, rows_out, topic_out);
  });
}

} // extern "C"
