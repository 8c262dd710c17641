// kernels.cu — sm_100a kernels of the lookahead IVF retrieval path.
//
//   coarse_scores_kernel : query x centroid scores in fp64 (ivf.cpp:269-281)
//   select_kernel        : full on-chip ranking (register/shuffle/smem bitonic
//                          sort), ascending cluster id on ties
//                          (ivf.cpp:282-299), fused split of the probe by
//                          device-cache residency (tiered.cpp:155-161)
//   partition_kernel     : the same split for an explicit cluster list
//                          (search_clusters, ivf.cpp:301-323)
//   scan_tma_kernel      : IVF-Flat list scan. One producer warp streams
//                          list tiles HBM -> shared memory with cp.async.bulk
//                          (TMA) into an mbarrier ring; eight consumer warps
//                          score vectors from shared memory, keep a register
//                          top-k, merge per CTA, and the last CTA merges the
//                          grid and re-scores the survivors exactly
//                          (ivf.cpp:301-343, tiered.cpp:172-185)
//   scan_ldg_kernel      : the same scan with direct 128-bit register loads
//                          (rows that are not 16-byte aligned; A/B baseline)
//   window_kernel        : %globaltimer spin standing in for LLM generation
//
// Reference semantics kept on device: per-term arithmetic of dot_d / l2_sq_d
// (vectorstore.cpp:93-108; products are exact in fp64, so DFMA == mul+add for
// IP; L2 uses separately rounded sub/mul/add), fp32 rounding of the final
// score, sqrt for L2, and the (score, ascending id) total order with
// -0.0 == +0.0 (vectorstore.hpp:34-39). Only the summation order differs
// (parallel tree instead of a serial chain).
//
// Accumulation: the scan accumulates in fp32 (FMA) to stay HBM-bound and keeps
// k + kRerankMargin survivors; the last CTA recomputes their scores with the
// fp64 arithmetic above and re-ranks, so reported scores and the boundary
// order are the reference's. acc_fp64 instead accumulates every candidate in
// fp64 (no re-score needed).
#include <algorithm>
#include <mutex>
#include <map>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "host.hpp"
#include "kernels.cuh"
#include "dev_common.cuh"

namespace laivg {
using namespace dev;

// Raises a kernel's dynamic shared-memory limit once per (kernel, device):
// function attributes are per device, so one process driving several GPUs
// must set them on each.
void ensure_dyn_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = done[{fn, dev}];
  if (bytes > cur) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    cur = bytes;
  }
}

// Counts the launch and surfaces launch-configuration errors immediately.
void after_launch() {
  launch_counter()++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    throw CudaError(std::string("kernel launch failed: ") + cudaGetErrorString(e));
  }
}

namespace {

// --------------------------------------------------------------------------
// total order (vectorstore.hpp:34-39)
// --------------------------------------------------------------------------
__device__ __forceinline__ float sentinel_score(int metric) {
  return metric == kIP ? -INFINITY : INFINITY;
}

// Warp-resident sorted top-k with a payload (slab vector index, for the exact
// re-score): entry j = i * 32 + lane lives in slot i of that lane. Entries
// j >= k are scratch.
//
// `id` holds the candidate's host-store ROW when `ids` is set: the datastore
// id is only looked up (ids[row]) to break an exact score tie, and once at
// output. A scan therefore never waits on an id load to admit a candidate.
template <int KPL>
struct WarpTopK {
  float s[KPL];
  uint64_t id[KPL];
  uint32_t vi[KPL];
  float worst_s;
  uint64_t worst_id;
  const uint64_t* ids = nullptr; // row -> id table (nullptr: keys are ids)

  // (score, id) total order on keys (vectorstore.hpp:34-39)
  __device__ __forceinline__ bool ranks_before(int metric, float sa, uint64_t ka, float sb,
                                               uint64_t kb) const {
    if (sa != sb) return metric == kIP ? sa > sb : sa < sb;
    if (ids == nullptr || ka == ~0ull || kb == ~0ull) return ka < kb;
    return __ldg(reinterpret_cast<const unsigned long long*>(ids) + ka) <
           __ldg(reinterpret_cast<const unsigned long long*>(ids) + kb);
  }

  __device__ void init(int metric) {
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      s[i] = sentinel_score(metric);
      id[i] = ~0ull;
      vi[i] = ~0u;
    }
    worst_s = sentinel_score(metric);
    worst_id = ~0ull;
  }

  __device__ void refresh_worst(int k) {
    const int wi = (k - 1) >> 5, wl = (k - 1) & 31;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      if (i == wi) {
        worst_s = __shfl_sync(kFull, s[i], wl);
        worst_id = __shfl_sync(kFull, id[i], wl);
      }
    }
  }

  // Score-only pre-check: could (cs, any id) enter?
  __device__ __forceinline__ bool may_enter(int metric, float cs) const {
    return metric == kIP ? cs >= worst_s : cs <= worst_s;
  }
  __device__ __forceinline__ bool enters(int metric, float cs, uint64_t cid) const {
    return ranks_before(metric, cs, cid, worst_s, worst_id);
  }

  // Warp-uniform insertion of a candidate known to enter.
  __device__ void insert(int metric, int k, float cs, uint64_t cid, uint32_t cvi) {
    const int lane = threadIdx.x & 31;
    int pos = 0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      const bool b = j < k && ranks_before(metric, s[i], id[i], cs, cid);
      pos += __popc(__ballot_sync(kFull, b));
    }
    float ps[KPL];
    uint64_t pid[KPL];
    uint32_t pvi[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      float us = __shfl_up_sync(kFull, s[i], 1);
      uint64_t uid = __shfl_up_sync(kFull, id[i], 1);
      uint32_t uvi = __shfl_up_sync(kFull, vi[i], 1);
      if (i > 0) {
        const float ts = __shfl_sync(kFull, s[i - 1], 31);
        const uint64_t tid = __shfl_sync(kFull, id[i - 1], 31);
        const uint32_t tvi = __shfl_sync(kFull, vi[i - 1], 31);
        if (lane == 0) {
          us = ts;
          uid = tid;
          uvi = tvi;
        }
      }
      ps[i] = us;
      pid[i] = uid;
      pvi[i] = uvi;
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      if (j > pos) {
        s[i] = ps[i];
        id[i] = pid[i];
        vi[i] = pvi[i];
      } else if (j == pos) {
        s[i] = cs;
        id[i] = cid;
        vi[i] = cvi;
      }
    }
    refresh_worst(k);
  }

  __device__ __forceinline__ void offer(int metric, int k, float cs, uint64_t cid,
                                        uint32_t cvi) {
    if (may_enter(metric, cs) && enters(metric, cs, cid)) insert(metric, k, cs, cid, cvi);
  }

  // Merge a best-first list of n entries (sentinels allowed) from memory.
  // Stops at the first entry that cannot enter (the list is sorted).
  template <bool kCG>
  __device__ void merge_list(int metric, int k, const float* ls, const uint64_t* lid,
                             const uint32_t* lvi, int n) {
    for (int e = 0; e < n; ++e) {
      const float cs = kCG ? __ldcg(ls + e) : ls[e];
      if (!may_enter(metric, cs)) break;
      const uint64_t cid =
          kCG ? __ldcg(reinterpret_cast<const unsigned long long*>(lid) + e) : lid[e];
      if (!enters(metric, cs, cid)) break;
      insert(metric, k, cs, cid, kCG ? __ldcg(lvi + e) : lvi[e]);
    }
  }

  __device__ void store(int k, float* ls, uint64_t* lid, uint32_t* lvi) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      if (j < k) {
        ls[j] = s[i];
        lid[j] = id[i];
        lvi[j] = vi[i];
      }
    }
  }
};

// --------------------------------------------------------------------------
// coarse scores
// --------------------------------------------------------------------------
template <int QT>
__global__ void __launch_bounds__(256)
    coarse_scores_kernel(const float* __restrict__ Q, uint32_t nq,
                         const float* __restrict__ cen, uint32_t nc, uint32_t d,
                         int metric, double* __restrict__ scores) {
  extern __shared__ float sq[];
  const uint32_t q0 = blockIdx.y * QT;
  const int nqt = min(QT, static_cast<int>(nq - q0));
  for (uint32_t i = threadIdx.x; i < nqt * d; i += blockDim.x) {
    sq[i] = Q[static_cast<uint64_t>(q0) * d + i];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= nc) return;
  const float* row = cen + static_cast<uint64_t>(c) * d;
  double acc[QT];
#pragma unroll
  for (int t = 0; t < QT; ++t) acc[t] = 0.0;
  if ((d & 3u) == 0 && d <= 1024) {
    // all of the row's loads in flight before any math (d <= 1024: <= 8 per lane)
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const uint32_t d4 = d >> 2;
    float4 xs[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t j = lane + 32u * c;
      xs[c] = j < d4 ? __ldg(r4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t j = lane + 32u * c;
      if (j < d4) {
#pragma unroll
        for (int t = 0; t < QT; ++t) {
          if (t < nqt) {
            const float4 qq = reinterpret_cast<const float4*>(sq + t * d)[j];
            const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
            Acc4<true>::run(metric, qd, xs[c], acc[t]);
          }
        }
      }
    }
  } else if ((d & 3u) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (uint32_t j = lane; j < d / 4; j += 32) {
      const float4 x = __ldg(r4 + j);
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        if (t < nqt) {
          const float4 qq = reinterpret_cast<const float4*>(sq + t * d)[j];
          const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
          Acc4<true>::run(metric, qd, x, acc[t]);
        }
      }
    }
  } else {
    for (uint32_t j = lane; j < d; j += 32) {
      const float x = __ldg(row + j);
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        if (t < nqt) {
          acc[t] = metric == kIP ? term_ip_d(sq[t * d + j], x, acc[t])
                                 : term_l2_d(sq[t * d + j], x, acc[t]);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < QT; ++t) {
    const double v = warp_sum(acc[t]);
    if (lane == 0 && t < nqt) {
      scores[static_cast<uint64_t>(q0 + t) * nc + c] = v;
    }
  }
}

// Single query, d % 4 == 0, d <= 1024: each warp scores kCPW centroids with
// all of their row loads in flight (about one wave for nc = 4096). Per
// centroid the arithmetic is exactly warp_coarse_score's, so scores are
// bit-identical to every other coarse path.
constexpr int kCPW = 2;
template <int NCH> // float4 chunks per lane: d <= 128 * NCH
__global__ void __launch_bounds__(256, 2)
    coarse_scores_q1_kernel(const float* __restrict__ Q, const float* __restrict__ cen,
                            uint32_t nc, uint32_t d, int metric, double* __restrict__ scores) {
  __shared__ __align__(16) float sq[128 * NCH];
  const uint32_t q = blockIdx.y;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) sq[i] = Q[static_cast<uint64_t>(q) * d + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c0 = (blockIdx.x * (blockDim.x >> 5) + warp) * kCPW;
  if (c0 >= nc) return;
  const uint32_t d4 = d >> 2;
  float4 xs[kCPW][NCH];
#pragma unroll
  for (int u = 0; u < kCPW; ++u) {
    const uint32_t c = c0 + u < nc ? c0 + u : c0;
    const float4* r4 = reinterpret_cast<const float4*>(cen + static_cast<uint64_t>(c) * d);
#pragma unroll
    for (int t = 0; t < NCH; ++t) {
      const uint32_t j = lane + 32u * t;
      xs[u][t] = j < d4 ? __ldg(r4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  double acc[kCPW];
#pragma unroll
  for (int u = 0; u < kCPW; ++u) acc[u] = 0.0;
#pragma unroll
  for (int t = 0; t < NCH; ++t) {
    const uint32_t j = lane + 32u * t;
    if (j < d4) {
      const float4 qq = reinterpret_cast<const float4*>(sq)[j];
      const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
      for (int u = 0; u < kCPW; ++u) Acc4<true>::run(metric, qd, xs[u][t], acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < kCPW; ++u) {
    const double v = warp_sum(acc[u]);
    if (lane == 0 && c0 + u < nc) scores[static_cast<uint64_t>(q) * nc + c0 + u] = v;
  }
}

// --------------------------------------------------------------------------
// residency split of a probe held in memory (block-wide, any blockDim <= 1024)
// --------------------------------------------------------------------------
__device__ void partition_block(const uint32_t* probe, uint32_t lp, const int64_t* res_off,
                                const uint64_t* list_off, const FastTable& ft, uint32_t q) {
  __shared__ uint32_t w_cnt[32];
  __shared__ uint64_t w_len[32];
  __shared__ uint32_t base_cnt;
  __shared__ uint64_t base_len;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = (blockDim.x + 31) >> 5;
  const uint64_t tb = static_cast<uint64_t>(q) * ft.stride;
  uint64_t* pre = ft.pre + static_cast<uint64_t>(q) * (ft.stride + 1);
  if (threadIdx.x == 0) {
    base_cnt = 0;
    base_len = 0;
  }
  __syncthreads();
  for (uint32_t t0 = 0; t0 < lp; t0 += blockDim.x) {
    const uint32_t i = t0 + threadIdx.x;
    uint32_t c = 0;
    int64_t so = -1;
    uint64_t lo0 = 0, lo1 = 0;
    if (i < lp) { // all three loads in flight together
      c = probe[i];
      so = res_off[c];
      lo0 = list_off[c];
      lo1 = list_off[c + 1];
    }
    const bool fast = so >= 0;
    const uint64_t len = fast ? lo1 - lo0 : 0;
    uint32_t ic = fast ? 1u : 0u;
    uint64_t il = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t nc_ = __shfl_up_sync(kFull, ic, o);
      const uint64_t nl = __shfl_up_sync(kFull, il, o);
      if (lane >= o) {
        ic += nc_;
        il += nl;
      }
    }
    if (lane == 31) {
      w_cnt[warp] = ic;
      w_len[warp] = il;
    }
    __syncthreads();
    uint32_t pc = base_cnt;
    uint64_t pl = base_len;
    for (int w = 0; w < warp; ++w) {
      pc += w_cnt[w];
      pl += w_len[w];
    }
    if (fast) {
      const uint32_t ex_c = pc + ic - 1u;
      ft.slab[tb + ex_c] = so;
      ft.row[tb + ex_c] = lo0;
      ft.len[tb + ex_c] = static_cast<uint32_t>(len);
      ft.cluster[tb + ex_c] = c;
      pre[ex_c] = pl + il - len;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tc = base_cnt;
      uint64_t tl = base_len;
      for (int w = 0; w < nwarps; ++w) {
        tc += w_cnt[w];
        tl += w_len[w];
      }
      base_cnt = tc;
      base_len = tl;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ft.count[q] = base_cnt;
    pre[base_cnt] = base_len;
  }
  if (ft.cta == nullptr) return;
  // Scan CTA b covers [V*b/G, V*(b+1)/G): record the list and offset it
  // starts at, so the scan's producer needs no search. CTA b starts inside
  // list i iff b in [ceil(p*G/V), ceil((p+len)*G/V)), p = pre[i].
  __syncthreads();
  const uint32_t G = ft.grid, nf = base_cnt;
  const uint64_t V = base_len;
  CtaStart* cs = ft.cta + static_cast<uint64_t>(q) * G;
  for (uint32_t b = threadIdx.x; b < G; b += blockDim.x) {
    if (V == 0 || V * b / G >= V) cs[b] = CtaStart{0u, 0u, 0u, 0u};
  }
  if (V == 0) return;
  for (uint32_t i = threadIdx.x; i < nf; i += blockDim.x) {
    const uint64_t p = pre[i];
    const uint64_t len = ft.len[tb + i];
    if (len == 0) continue;
    const uint64_t b0 = (p * G + V - 1) / V, b1 = ((p + len) * G + V - 1) / V;
    for (uint64_t b = b0; b < b1 && b < G; ++b) {
      const uint64_t v0 = V * b / G, v1 = V * (b + 1) / G;
      cs[b] = CtaStart{i, static_cast<uint32_t>(v0 - p), static_cast<uint32_t>(v1 - v0), 0u};
    }
  }
}

__global__ void __launch_bounds__(256)
    partition_kernel(const uint32_t* __restrict__ probe, uint32_t lp,
                     const int64_t* __restrict__ res_off,
                     const uint64_t* __restrict__ list_off, FastTable ft) {
  partition_block(probe + static_cast<uint64_t>(blockIdx.x) * lp, lp, res_off, list_off, ft,
                  blockIdx.x);
}

// --------------------------------------------------------------------------
// selection: block bitonic sort of (orderable key, cluster id); strides below
// E stay in registers, below 32E use warp shuffles, the rest shared memory
// --------------------------------------------------------------------------
__device__ __forceinline__ bool kv_gt(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
  return ka > kb || (ka == kb && va > vb);
}

// Compare-exchange stage with stride J < E inside one thread's registers.
template <int E, int J>
__device__ __forceinline__ void inthread_stage(uint64_t (&k)[E], uint32_t (&v)[E], uint32_t kk) {
  if constexpr (J < E) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = e ^ J;
      if (p > e) {
        const uint32_t i = threadIdx.x * E + e;
        const bool up = (i & kk) == 0;
        if (kv_gt(k[e], v[e], k[p], v[p]) == up) {
          const uint64_t tk = k[e];
          k[e] = k[p];
          k[p] = tk;
          const uint32_t tv = v[e];
          v[e] = v[p];
          v[p] = tv;
        }
      }
    }
  }
}

template <int E>
__device__ void block_bitonic_sort(uint64_t (&k)[E], uint32_t (&v)[E], uint64_t* sk,
                                   uint32_t* sv, uint32_t n) {
  const uint32_t t = threadIdx.x;
  for (uint32_t kk = 2; kk <= n; kk <<= 1) {
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      if (j < static_cast<uint32_t>(E)) {
        if (j == 1) inthread_stage<E, 1>(k, v, kk);
        else if (j == 2) inthread_stage<E, 2>(k, v, kk);
        else if (j == 4) inthread_stage<E, 4>(k, v, kk);
        else if (j == 8) inthread_stage<E, 8>(k, v, kk);
        else inthread_stage<E, 16>(k, v, kk);
      } else if (j < 32u * E) {
        const int lm = static_cast<int>(j / E);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t ok = __shfl_xor_sync(kFull, k[e], lm);
          const uint32_t ov = __shfl_xor_sync(kFull, v[e], lm);
          const uint32_t i = t * E + e;
          const bool up = (i & kk) == 0, lower = (i & j) == 0;
          const bool gt = kv_gt(k[e], v[e], ok, ov);
          if (lower == up ? gt : !gt) {
            k[e] = ok;
            v[e] = ov;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          sk[t * E + e] = k[e];
          sv[t * E + e] = v[e];
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t i = t * E + e, p = i ^ j;
          const uint64_t ok = sk[p];
          const uint32_t ov = sv[p];
          const bool up = (i & kk) == 0, lower = (i & j) == 0;
          const bool gt = kv_gt(k[e], v[e], ok, ov);
          if (lower == up ? gt : !gt) {
            k[e] = ok;
            v[e] = ov;
          }
        }
        __syncthreads();
      }
    }
  }
}

// Selection runs in two kernels so that no single SM sorts the whole ranking:
//   seg_sort_kernel   — CTA (s, q) sorts the 256 scores of segment s of query
//                       q (register/shuffle/smem bitonic) into a sorted run;
//   merge_runs_kernel — one CTA per query merges the runs pairwise with the
//                       bitonic min/max construction (C = min(A_i, B_{m-1-i})
//                       holds the m smallest of A u B as a bitonic sequence),
//                       keeping only the best P >= n_out per run when the
//                       caller needs a prefix (coarse_probe) and every entry
//                       when it needs the full ranking (rank_clusters).
constexpr uint32_t kSeg = 256;

// Ascending in-place bitonic sort of a[0, n) in shared memory (the buffer
// holds at least pow2(n) entries; the tail is overwritten with sentinels).
// Used to hand the scan each query's lists in cluster order: queries of a
// batch that share lists then stream them at about the same time, so the
// second and later reads of a list are L2 hits.
__device__ void sort_ids_block(uint32_t* a, uint32_t n) {
  uint32_t m = 1;
  while (m < n) m <<= 1;
  for (uint32_t i = n + threadIdx.x; i < m; i += blockDim.x) a[i] = 0xffffffffu;
  __syncthreads();
  for (uint32_t kk = 2; kk <= m; kk <<= 1) {
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t p = i ^ j;
        if (p > i && ((a[i] > a[p]) == ((i & kk) == 0))) {
          const uint32_t t = a[i];
          a[i] = a[p];
          a[p] = t;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSeg)
    seg_sort_kernel(const double* __restrict__ scores, uint32_t nc, int metric,
                    uint64_t* __restrict__ run_k, uint32_t* __restrict__ run_v,
                    uint32_t nseg_pad) {
  __shared__ uint64_t sk[kSeg];
  __shared__ uint32_t sv[kSeg];
  const uint32_t q = blockIdx.y, s = blockIdx.x;
  const uint32_t i = s * kSeg + threadIdx.x;
  uint64_t k[1];
  uint32_t v[1];
  if (i < nc) {
    k[0] = order_key(scores[static_cast<uint64_t>(q) * nc + i], metric);
    v[0] = i;
  } else {
    k[0] = ~0ull;
    v[0] = ~0u;
  }
  block_bitonic_sort<1>(k, v, sk, sv, kSeg);
  const uint64_t o = (static_cast<uint64_t>(q) * nseg_pad + s) * kSeg + threadIdx.x;
  run_k[o] = k[0];
  run_v[o] = v[0];
}

__device__ __forceinline__ void cswap_up(uint64_t* k, uint32_t* v, uint32_t a, uint32_t b) {
  // ascending compare-exchange of positions a < b
  if (kv_gt(k[a], v[a], k[b], v[b])) {
    const uint64_t tk = k[a];
    k[a] = k[b];
    k[b] = tk;
    const uint32_t tv = v[a];
    v[a] = v[b];
    v[b] = tv;
  }
}

// One merge step of the prefix tree, by one warp: runs A and B (ascending by
// (key, cluster), P = 32 * E entries each) -> the best P of A u B, ascending,
// at `o`. C_i = min(A_i, B_{P-1-i}) holds exactly those P as a bitonic
// sequence; a bitonic clean (strides >= E across lanes by shuffle, < E in
// registers) sorts it. No block barrier inside.
template <int E>
__device__ __forceinline__ void warp_merge_best(const uint64_t* ak, const uint32_t* av,
                                                const uint64_t* bk, const uint32_t* bv,
                                                uint64_t* ok, uint32_t* ov) {
  constexpr uint32_t P = 32u * E;
  const uint32_t lane = threadIdx.x & 31u;
  uint64_t k[E];
  uint32_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = lane * E + e;
    const uint64_t ka = ak[i], kb = bk[P - 1 - i];
    const uint32_t va = av[i], vb = bv[P - 1 - i];
    const bool take_b = kv_gt(ka, va, kb, vb);
    k[e] = take_b ? kb : ka;
    v[e] = take_b ? vb : va;
  }
#pragma unroll
  for (uint32_t st = P / 2; st > 0; st >>= 1) {
    if (st >= static_cast<uint32_t>(E)) {
      const int lm = static_cast<int>(st / E);
      const bool lower = (lane & static_cast<uint32_t>(lm)) == 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint64_t pk = __shfl_xor_sync(kFull, k[e], lm);
        const uint32_t pv = __shfl_xor_sync(kFull, v[e], lm);
        // the lower index keeps the smaller of the pair
        const bool gt = kv_gt(k[e], v[e], pk, pv);
        if (lower == gt) {
          k[e] = pk;
          v[e] = pv;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int pe = e ^ static_cast<int>(st);
        if (pe > e && kv_gt(k[e], v[e], k[pe], v[pe])) {
          const uint64_t tk = k[e];
          k[e] = k[pe];
          k[pe] = tk;
          const uint32_t tv = v[e];
          v[e] = v[pe];
          v[pe] = tv;
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    ok[lane * E + e] = k[e];
    ov[lane * E + e] = v[e];
  }
}

template <int E>
__device__ void warp_merge_tree(uint64_t*& ak, uint32_t*& av, uint64_t*& bk, uint32_t*& bv,
                                uint32_t nruns) {
  constexpr uint32_t P = 32u * E;
  const uint32_t warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t lists = nruns; lists > 1; lists >>= 1) {
    for (uint32_t pr = warp; pr < lists / 2; pr += nw) {
      warp_merge_best<E>(ak + 2 * pr * P, av + 2 * pr * P, ak + (2 * pr + 1) * P,
                         av + (2 * pr + 1) * P, bk + pr * P, bv + pr * P);
    }
    __syncthreads();
    uint64_t* tk = ak;
    ak = bk;
    bk = tk;
    uint32_t* tv = av;
    av = bv;
    bv = tv;
  }
}

// nseg_pad runs of kSeg sorted entries per query (power of two, sentinel
// padded); P = run length kept per level (power of two, <= kSeg) or kSeg with
// `full` to keep everything.
__global__ void __launch_bounds__(1024)
    merge_runs_kernel(const uint64_t* __restrict__ run_k, const uint32_t* __restrict__ run_v,
                      uint32_t nseg_pad, uint32_t P, bool full, uint32_t n_out,
                      uint32_t* __restrict__ order, const int64_t* res_off,
                      const uint64_t* list_off, FastTable ft, bool do_partition,
                      bool scan_sorted) {
  extern __shared__ uint64_t mk[];
  const uint32_t total = nseg_pad * P;
  uint32_t* mv = reinterpret_cast<uint32_t*>(mk + total);
  const uint32_t q = blockIdx.x;
  const uint64_t base = static_cast<uint64_t>(q) * nseg_pad * kSeg;
  // every size here is a power of two: index with shifts and masks
  const uint32_t lP = __ffs(P) - 1;
  for (uint32_t x = threadIdx.x; x < total; x += blockDim.x) {
    const uint32_t r = x >> lP, i = x & (P - 1);
    mk[x] = run_k[base + static_cast<uint64_t>(r) * kSeg + i];
    mv[x] = run_v[base + static_cast<uint64_t>(r) * kSeg + i];
  }
  __syncthreads();
  if (!full) {
    // prefix mode: merge-path tree, the best P of each pair per level (one
    // co-rank binary search per output, one barrier per level)
    uint64_t* ak = mk;
    uint32_t* av = mv;
    uint64_t* bk = reinterpret_cast<uint64_t*>(mv + total);
    bk = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bk) + 7) & ~uintptr_t(7));
    uint32_t* bv = reinterpret_cast<uint32_t*>(bk + total);
    if (P >= 32 && P <= 256) {
      // one warp per pair: min-trick + in-warp bitonic clean, one barrier
      // per level (the merge-path search below costs ~4x more)
      if (P == 32) warp_merge_tree<1>(ak, av, bk, bv, nseg_pad);
      else if (P == 64) warp_merge_tree<2>(ak, av, bk, bv, nseg_pad);
      else if (P == 128) warp_merge_tree<4>(ak, av, bk, bv, nseg_pad);
      else warp_merge_tree<8>(ak, av, bk, bv, nseg_pad);
    }
    for (uint32_t lists = (P >= 32 && P <= 256) ? 1 : nseg_pad; lists > 1; lists >>= 1) {
      for (uint32_t x = threadIdx.x; x < (lists / 2) << lP; x += blockDim.x) {
        const uint32_t pr = x >> lP, p = x & (P - 1);
        const uint32_t A = 2 * pr * P, B = A + P;
        uint32_t lo = 0, hi = p;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (!kv_gt(ak[A + mid], av[A + mid], ak[B + p - mid - 1], av[B + p - mid - 1])) {
            lo = mid + 1;
          } else {
            hi = mid;
          }
        }
        const uint32_t i = lo, j = p - i;
        const bool from_a = j >= P || (i < P && !kv_gt(ak[A + i], av[A + i], ak[B + j], av[B + j]));
        bk[pr * P + p] = from_a ? ak[A + i] : ak[B + j];
        bv[pr * P + p] = from_a ? av[A + i] : av[B + j];
      }
      __syncthreads();
      uint64_t* tk = ak;
      ak = bk;
      bk = tk;
      uint32_t* tv = av;
      av = bv;
      bv = tv;
    }
    uint32_t* out = order + static_cast<uint64_t>(q) * n_out;
    for (uint32_t i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = av[i];
    if (do_partition) {
      __syncthreads();
      if (scan_sorted) sort_ids_block(av, n_out);
      partition_block(av, n_out, res_off, list_off, ft, q);
    }
    return;
  }
  uint32_t nruns = nseg_pad, ls = lP, lm = lP;
  while (nruns > 1) {
    const uint32_t pairs = nruns >> 1, m = 1u << lm, stride = 1u << ls;
    // min/max pass: A[i] <-> B[m-1-i]
    for (uint32_t x = threadIdx.x; x < (pairs << lm); x += blockDim.x) {
      const uint32_t p = x >> lm, i = x & (m - 1);
      const uint32_t a = (p << (ls + 1)) + i, b = (p << (ls + 1)) + stride + (m - 1 - i);
      cswap_up(mk, mv, a, b);
    }
    __syncthreads();
    // bitonic clean of the low half (and of the high half in full mode)
    const uint32_t lh = full ? 1 : 0, lper = lm - 1;
    for (uint32_t lj = lm; lj-- > 0;) {
      const uint32_t j = 1u << lj;
      for (uint32_t x = threadIdx.x; x < (pairs << (lh + lper)); x += blockDim.x) {
        const uint32_t hp = x >> lper, t = x & ((1u << lper) - 1);
        const uint32_t p = hp >> lh, h = hp & lh;
        const uint32_t lo = ((t >> lj) << (lj + 1)) + (t & (j - 1));
        const uint32_t o = (p << (ls + 1)) + (h << ls);
        cswap_up(mk, mv, o + lo, o + lo + j);
      }
      __syncthreads();
    }
    nruns = pairs;
    ++ls;
    if (full) ++lm;
  }
  uint32_t* out = order + static_cast<uint64_t>(q) * n_out;
  for (uint32_t i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = mv[i];
  if (do_partition) {
    __syncthreads();
    if (scan_sorted) sort_ids_block(mv, n_out);
    partition_block(mv, n_out, res_off, list_off, ft, q);
  }
}


// --------------------------------------------------------------------------
// exact selection from tensor-core scores (batched coarse_probe)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t float_order(float f) { // ascending with f
  const uint32_t b = __float_as_uint(f + 0.0f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float order_float(uint32_t u) {
  return __uint_as_float((u >> 31) ? (u & 0x7fffffffu) : ~u);
}

// Bounds on the exact "goodness" g (IP: score, L2: -squared distance) of
// centroid c from its tensor-core score a: g in [lo, hi].
__device__ __forceinline__ void tc_bounds(int metric, double a, double qn, double qn2, float cn,
                                          float& lo, float& hi) {
  const double cnd = cn;
  double g, e;
  if (metric == kIP) {
    g = a;
    e = kTcErr * qn * cnd;
  } else {
    const double cn2 = cnd * cnd;
    g = -(qn2 + cn2 - 2.0 * a);
    e = 2.0 * kTcErr * qn * cnd + 1e-6 * (qn2 + cn2);
  }
  lo = __double2float_rd(g - e);
  hi = __double2float_ru(g + e);
}

// One CTA (1024 threads) per query. smem: q[d], 32-bit keys of the lower
// bounds[nc], upper bounds[nc], candidate keys/ids[cap] (cap = pow2 >= nc,
// so every centroid fits).
// Threads per query CTA: 1024 for small batches; 512 (two CTAs per SM) once
// the batch exceeds the SM count, so a 256-query batch runs in one wave
// (1024-thread CTAs are held to one per SM by the register file)
constexpr int kSelThreads = 1024;
// LAIVG_TC_PROBE diagnostics: query 0's CTA stamps its phases here
__device__ unsigned long long g_tc_dbg[8];
template <int NT>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1)
    tc_select_kernel(const float* __restrict__ approx, uint32_t splits,
                     const float* __restrict__ Q, uint32_t d,
                     const float* __restrict__ cen, const float* __restrict__ cnorm,
                     uint32_t nc, int metric, uint32_t n_out, uint32_t cap,
                     uint32_t* __restrict__ order, const int64_t* res_off,
                     const uint64_t* list_off, FastTable ft, bool do_partition,
                     bool scan_sorted, bool probe_on) {
  extern __shared__ __align__(16) unsigned char sm[];
  float* sq = reinterpret_cast<float*>(sm);
  uint32_t* lok = reinterpret_cast<uint32_t*>(sm + ((static_cast<size_t>(d) * 4 + 15) & ~size_t(15)));
  float* hik = reinterpret_cast<float*>(
      reinterpret_cast<unsigned char*>(lok) + ((static_cast<size_t>(nc) * 4 + 15) & ~size_t(15)));
  uint64_t* ck = reinterpret_cast<uint64_t*>(
      reinterpret_cast<unsigned char*>(hik) + ((static_cast<size_t>(nc) * 4 + 15) & ~size_t(15)));
  uint32_t* cv = reinterpret_cast<uint32_t*>(ck + cap);
  __shared__ uint32_t hist[256];
  __shared__ double red[32];
  __shared__ uint32_t s_prefix, s_rank, s_count;
  const uint32_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* qv = Q + static_cast<uint64_t>(q) * d;
  const float* aq = approx + static_cast<uint64_t>(q) * nc;
  const uint64_t plane = static_cast<uint64_t>(gridDim.x) * nc; // split-K partial planes
  const bool dbg = probe_on && q == 0 && threadIdx.x == 0;
  if (dbg) g_tc_dbg[0] = globaltimer();

  // ||q||^2 in fp64
  double part = 0.0;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
    const float x = qv[i];
    sq[i] = x;
    part += static_cast<double>(x) * x;
  }
  part = warp_sum(part);
  if (lane == 0) red[warp] = part;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_rank = n_out - 1;
    s_count = 0;
  }
  __syncthreads();
  double qn2 = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) qn2 += red[w];
  const double qn = sqrt(qn2) * (1.0 + 1e-12);

  // bounds of every cluster, once: lower-bound keys (inverted so that
  // ascending key = best first) and upper bounds; 4 clusters per thread with
  // all their loads in flight
  for (uint32_t c0 = threadIdx.x; c0 < nc; c0 += 4 * blockDim.x) {
    double a[4];
    float cn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t c = c0 + u * blockDim.x;
      a[u] = 0.0;
      cn[u] = 0.0f;
      if (c < nc) {
        cn[u] = cnorm[c];
        for (uint32_t z = 0; z < splits; ++z) a[u] += aq[z * plane + c];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t c = c0 + u * blockDim.x;
      if (c < nc) {
        float lo, hi;
        tc_bounds(metric, a[u], qn, qn2, cn[u], lo, hi);
        lok[c] = ~float_order(lo);
        hik[c] = hi;
      }
    }
  }
  __syncthreads();
  if (dbg) g_tc_dbg[1] = globaltimer();
  // radix select: the (n_out-1)-th smallest key, 8 bits at a time
  uint32_t mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (uint32_t c0 = 0; c0 < nc; c0 += blockDim.x) { // warp-uniform trip count
      const uint32_t c = c0 + threadIdx.x;
      const bool in = c < nc && (lok[c] & mask) == prefix;
      const uint32_t bin = in ? (lok[c] >> shift) & 255u : 256u;
      // one atomic per distinct bin per warp (the top digits are shared by
      // almost every key)
      const unsigned peers = __match_any_sync(kFull, bin);
      if (in && (__ffs(peers) - 1) == lane) atomicAdd(&hist[bin], __popc(peers));
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t h[8], tot = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        h[i] = hist[lane * 8 + i];
        tot += h[i];
      }
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += t;
      }
      const uint32_t rank = s_rank, excl = inc - tot;
      if (rank >= excl && rank < inc) { // exactly one lane
        uint32_t r = rank - excl, b = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (r >= h[i] && b == static_cast<uint32_t>(i)) {
            r -= h[i];
            ++b;
          }
        }
        s_rank = r;
        s_prefix = prefix | ((lane * 8u + b) << shift);
      }
    }
    mask |= 255u << shift;
    __syncthreads();
  }
  const float T = order_float(~s_prefix); // the n_out-th best lower bound
  if (dbg) g_tc_dbg[2] = globaltimer();

  // candidates: upper bound reaches T (includes every exact top-n_out member)
  for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
    if (hik[c] >= T) cv[atomicAdd(&s_count, 1u)] = c;
  }
  __syncthreads();
  if (dbg) g_tc_dbg[3] = globaltimer();
  const uint32_t n = s_count;
  uint32_t m = 2;
  while (m < n) m <<= 1;
  // exact fp64 re-score (same arithmetic as coarse_scores_kernel)
  const uint32_t nwarps = blockDim.x >> 5;
  for (uint32_t i = warp; i < n; i += nwarps) {
    double sc[1];
    warp_coarse_score_n<1>(sq, cen, cv + i, 1, d, metric, lane, sc);
    if (lane == 0) ck[i] = order_key(sc[0], metric);
  }
  for (uint32_t i = n + threadIdx.x; i < m; i += blockDim.x) {
    ck[i] = ~0ull;
    cv[i] = ~0u;
  }
  __syncthreads();
  if (dbg) {
    g_tc_dbg[4] = globaltimer();
    g_tc_dbg[7] = n;
  }
  // bitonic sort on (key, cluster id)
  for (uint32_t kk = 2; kk <= m; kk <<= 1) {
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t p = i ^ j;
        if (p > i) {
          const bool up = (i & kk) == 0;
          if (kv_gt(ck[i], cv[i], ck[p], cv[p]) == up) {
            const uint64_t tk = ck[i];
            ck[i] = ck[p];
            ck[p] = tk;
            const uint32_t tv = cv[i];
            cv[i] = cv[p];
            cv[p] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
  if (dbg) g_tc_dbg[5] = globaltimer();
  uint32_t* out = order + static_cast<uint64_t>(q) * n_out;
  for (uint32_t i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = cv[i];
  if (do_partition) {
    __syncthreads();
    if (scan_sorted) sort_ids_block(cv, n_out);
    partition_block(cv, n_out, res_off, list_off, ft, q);
  }
  if (dbg) g_tc_dbg[6] = globaltimer();
}

// ---- batched exact selection, three kernels ------------------------------
// tc_filter_kernel   per query: the bounds pass, radix select and candidate
//                    collection of tc_select_kernel; candidates to global
// tc_rescore_stream  one CTA per SM over the flattened (query, candidate)
//                    pairs: a producer warp gathers candidate centroid rows
//                    with bulk copies into a two-stage ring (the scan's
//                    design), eight consumer warps score them with
//                    warp_coarse_score's arithmetic (same lane-strided fp64
//                    terms, same butterfly) -> exact order keys
// tc_sort_kernel     per query: register/shuffle bitonic sort on (key, id),
//                    first n_out, fused residency split
template <int NT>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1)
    tc_filter_kernel(const float* __restrict__ approx, uint32_t splits,
                     const float* __restrict__ Q, uint32_t d, const float* __restrict__ cnorm,
                     uint32_t nc, int metric, uint32_t n_out, uint32_t cap,
                     uint32_t* __restrict__ cand, uint32_t* __restrict__ ncand,
                     uint32_t* __restrict__ qmask) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint32_t* lok = reinterpret_cast<uint32_t*>(sm);
  float* hik = reinterpret_cast<float*>(sm + ((static_cast<size_t>(nc) * 4 + 15) & ~size_t(15)));
  __shared__ uint32_t hist[256];
  __shared__ double red[32];
  __shared__ uint32_t s_prefix, s_rank, s_count;
  const uint32_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* qv = Q + static_cast<uint64_t>(q) * d;
  const float* aq = approx + static_cast<uint64_t>(q) * nc;
  const uint64_t plane = static_cast<uint64_t>(gridDim.x) * nc;
  double part = 0.0;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
    const float x = qv[i];
    part += static_cast<double>(x) * x;
  }
  part = warp_sum(part);
  if (lane == 0) red[warp] = part;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_rank = n_out - 1;
    s_count = 0;
  }
  __syncthreads();
  double qn2 = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) qn2 += red[w];
  const double qn = sqrt(qn2) * (1.0 + 1e-12);
  for (uint32_t c0 = threadIdx.x; c0 < nc; c0 += 4 * blockDim.x) {
    double a[4];
    float cn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t c = c0 + u * blockDim.x;
      a[u] = 0.0;
      cn[u] = 0.0f;
      if (c < nc) {
        cn[u] = cnorm[c];
        for (uint32_t z = 0; z < splits; ++z) a[u] += aq[z * plane + c];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t c = c0 + u * blockDim.x;
      if (c < nc) {
        float lo, hi;
        tc_bounds(metric, a[u], qn, qn2, cn[u], lo, hi);
        lok[c] = ~float_order(lo);
        hik[c] = hi;
      }
    }
  }
  uint32_t mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (uint32_t c0 = 0; c0 < nc; c0 += blockDim.x) {
      const uint32_t c = c0 + threadIdx.x;
      const bool in = c < nc && (lok[c] & mask) == prefix;
      const uint32_t bin = in ? (lok[c] >> shift) & 255u : 256u;
      const unsigned peers = __match_any_sync(kFull, bin);
      if (in && (__ffs(peers) - 1) == lane) atomicAdd(&hist[bin], __popc(peers));
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t h[8], tot = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        h[i] = hist[lane * 8 + i];
        tot += h[i];
      }
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += t;
      }
      const uint32_t rank = s_rank, excl = inc - tot;
      if (rank >= excl && rank < inc) {
        uint32_t r = rank - excl, b = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (r >= h[i] && b == static_cast<uint32_t>(i)) {
            r -= h[i];
            ++b;
          }
        }
        s_rank = r;
        s_prefix = prefix | ((lane * 8u + b) << shift);
      }
    }
    mask |= 255u << shift;
    __syncthreads();
  }
  const float T = order_float(~s_prefix);
  uint32_t* out = cand + static_cast<uint64_t>(q) * cap;
  for (uint32_t c0 = 0; c0 < nc; c0 += blockDim.x) {
    const uint32_t c = c0 + threadIdx.x;
    const bool take = c < nc && hik[c] >= T;
    const unsigned m = __ballot_sync(kFull, take);
    uint32_t base = 0;
    if (lane == 0 && m) base = atomicAdd(&s_count, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(kFull, base, 0);
    if (take) {
      out[base + __popc(m & ((1u << lane) - 1u))] = c;
      if (qmask) atomicOr(qmask + static_cast<uint64_t>(q >> 5) * nc + c, 1u << (q & 31));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ncand[q] = s_count;
}

// List-major exact re-score: CTA (x, y) holds the 32 queries of block y in
// shared memory and walks centroids [x * chunk, (x + 1) * chunk); each warp
// loads a centroid row once into registers (the next one in flight) and
// scores it for every block query that kept it as a candidate (qmask), two
// queries at a time, with warp_coarse_score's exact sequence (lane-strided
// float4 terms, Acc4, butterfly), so the keys are the ones the per-pair
// re-score computes. Centroid rows leave L2 once per 32-query block instead
// of once per (query, candidate) pair.
template <int NCH>
__global__ void __launch_bounds__(256, 2)
    tc_rescore_lm_kernel(const float* __restrict__ Q, uint32_t d, const float* __restrict__ cen,
                         int metric, uint32_t nq, uint32_t nc, uint32_t cap, uint32_t chunk,
                         const uint32_t* __restrict__ qmask, uint64_t* __restrict__ key) {
  extern __shared__ __align__(16) unsigned char smq[];
  float4* sq4 = reinterpret_cast<float4*>(smq);
  const uint32_t qb = blockIdx.y, q0 = qb * 32, nb = min(32u, nq - q0);
  const uint32_t d4 = d >> 2;
  const uint32_t c0 = blockIdx.x * chunk, c1 = min(nc, c0 + chunk);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smq + static_cast<size_t>(32) * d * 4);
  __shared__ __align__(8) uint64_t qbar;
  // the block's query rows are contiguous: one bulk copy
  const uint32_t qbytes = nb * d * 4;
  if (threadIdx.x == 0) {
    mbar_init(&qbar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&qbar, qbytes);
    bulk_g2s(sq4, Q + static_cast<uint64_t>(q0) * d, qbytes, &qbar);
  }
  for (uint32_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    smask[c - c0] = qmask[static_cast<uint64_t>(qb) * nc + c];
  }
  __syncthreads();
  mbar_wait(&qbar, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t W = 8; // warps per CTA
  const float4* cen4 = reinterpret_cast<const float4*>(cen);
  auto next = [&](uint32_t c) { // next centroid of this warp with a candidate query
    while (c < c1 && smask[c - c0] == 0) c += W;
    return c;
  };
  auto load_row = [&](uint32_t c, float4 (&r)[NCH]) {
#pragma unroll
    for (int t = 0; t < NCH; ++t) {
      const uint32_t jj = lane + 32u * t;
      r[t] = jj < d4 ? __ldg(cen4 + static_cast<uint64_t>(c) * d4 + jj)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 r[NCH], rn[NCH];
  uint32_t c = next(c0 + warp);
  if (c < c1) load_row(c, r);
  while (c < c1) {
    const uint32_t cn = next(c + W);
    if (cn < c1) load_row(cn, rn); // in flight while this row is scored
    uint32_t m = smask[c - c0];
    while (m) {
      // two block queries at a time (independent accumulation chains)
      const uint32_t b0 = __ffs(m) - 1;
      m &= m - 1;
      const bool two = m != 0;
      const uint32_t b1 = two ? __ffs(m) - 1 : b0;
      if (two) m &= m - 1;
      const float4* qv0 = sq4 + static_cast<size_t>(b0) * d4;
      const float4* qv1 = sq4 + static_cast<size_t>(b1) * d4;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int t = 0; t < NCH; ++t) {
        const uint32_t jj = lane + 32u * t;
        if (jj < d4) {
          const float4 x0 = qv0[jj], x1 = qv1[jj];
          const double qd0[4] = {x0.x, x0.y, x0.z, x0.w};
          const double qd1[4] = {x1.x, x1.y, x1.z, x1.w};
          Acc4<true>::run(metric, qd0, r[t], a0);
          Acc4<true>::run(metric, qd1, r[t], a1);
        }
      }
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      if (lane == 0) {
        key[static_cast<uint64_t>(q0 + b0) * cap + c] = order_key(a0, metric);
        if (two) key[static_cast<uint64_t>(q0 + b1) * cap + c] = order_key(a1, metric);
      }
    }
    c = cn;
#pragma unroll
    for (int t = 0; t < NCH; ++t) r[t] = rn[t];
  }
}

constexpr int kRsConsumers = 8;
constexpr int kRsThreads = 32 * (kRsConsumers + 1);
constexpr uint32_t kRsTile = 32; // rows per ring stage
constexpr uint32_t kRsMaxPairs = 2048; // pairs one CTA resolves up front (grid sized to fit)
template <int NCH>
__global__ void __launch_bounds__(kRsThreads, 1)
    tc_rescore_stream_kernel(const float* __restrict__ Q, uint32_t d,
                             const float* __restrict__ cen, int metric, uint32_t nq, uint32_t cap,
                             const uint32_t* __restrict__ cand, const uint32_t* __restrict__ ncand,
                             uint64_t* __restrict__ ckey) {
  extern __shared__ __align__(128) unsigned char smr[];
  constexpr uint32_t S = 2;
  const size_t row_f = d;
  float* ring = reinterpret_cast<float*>(smr);
  uint64_t* full = reinterpret_cast<uint64_t*>(smr + S * kRsTile * row_f * 4);
  uint64_t* empty = full + S;
  uint32_t* mq = reinterpret_cast<uint32_t*>(empty + S);  // [S][T] query of the row
  uint32_t* mi = mq + S * kRsTile;                         // [S][T] candidate index
  uint32_t* mn = mi + S * kRsTile;                         // [S] rows in the stage
  uint32_t* pref = mn + S;                                 // [nq + 1]
  uint32_t* rq = pref + nq + 1;                            // this CTA's pairs: query,
  uint32_t* ri = rq + kRsMaxPairs;                         //   candidate index,
  uint32_t* rc = ri + kRsMaxPairs;                         //   centroid
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // exclusive prefix of the candidate counts (every CTA, in shared memory)
  if (warp == 0) {
    uint32_t run = 0;
    for (uint32_t b = 0; b < nq; b += 32) {
      const uint32_t q = b + lane;
      const uint32_t v = q < nq ? ncand[q] : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += t;
      }
      if (q < nq) pref[q] = run + inc - v;
      run += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) pref[nq] = run;
  }
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kRsConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t P = pref[nq];
  const uint64_t p0 = P * blockIdx.x / gridDim.x, p1 = P * (blockIdx.x + 1) / gridDim.x;
  uint32_t tg = 0; // ring tiles issued / consumed so far (stage parity)
  uint32_t cur_q = 0xffffffffu;
  double qd[NCH * 4];
  for (uint64_t c0 = p0; c0 < p1; c0 += kRsMaxPairs) {
    const uint32_t np = static_cast<uint32_t>(min(static_cast<uint64_t>(kRsMaxPairs), p1 - c0));
    // resolve this chunk's pairs once, every thread, all candidate loads in flight
    for (uint32_t x = threadIdx.x; x < np; x += blockDim.x) {
      const uint64_t p = c0 + x;
      uint32_t lo = 0, hi = nq - 1; // last q with pref[q] <= p
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (pref[mid] <= p) lo = mid;
        else hi = mid - 1;
      }
      const uint32_t i = static_cast<uint32_t>(p - pref[lo]);
      rq[x] = lo;
      ri[x] = i;
      rc[x] = cand[static_cast<uint64_t>(lo) * cap + i];
    }
    __syncthreads();
    const uint32_t ntiles = (np + kRsTile - 1) / kRsTile;
    if (warp == 0) {
      // producer: one lane issues the row copies, the others publish metadata
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t tt = tg + t, s = tt % S;
        mbar_wait(empty + s, ((tt / S) & 1u) ^ 1u);
        const uint32_t x0 = t * kRsTile;
        const uint32_t n = min(kRsTile, np - x0);
        if (static_cast<uint32_t>(lane) < n) {
          mq[s * kRsTile + lane] = rq[x0 + lane];
          mi[s * kRsTile + lane] = ri[x0 + lane];
        }
        if (lane == 0) mn[s] = n;
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_expect_tx(full + s, n * d * 4u);
          for (uint32_t j = 0; j < n; ++j) {
            bulk_g2s(ring + (static_cast<size_t>(s) * kRsTile + j) * row_f,
                     cen + static_cast<uint64_t>(rc[x0 + j]) * d, d * 4u, full + s);
          }
        }
        __syncwarp();
      }
    } else {
      const int cw = warp - 1;
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t tt = tg + t, s = tt % S;
        mbar_wait(full + s, (tt / S) & 1u);
        const uint32_t n = mn[s];
        auto stage_query = [&](uint32_t q) { // this query's terms in registers (fp64)
          const float4* q4 = reinterpret_cast<const float4*>(Q + static_cast<uint64_t>(q) * d);
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const uint32_t jj = lane + 32u * c;
            const float4 v = jj < d / 4 ? __ldg(q4 + jj) : make_float4(0.f, 0.f, 0.f, 0.f);
            qd[4 * c + 0] = v.x;
            qd[4 * c + 1] = v.y;
            qd[4 * c + 2] = v.z;
            qd[4 * c + 3] = v.w;
          }
          cur_q = q;
        };
        // rows cw, cw + 8, cw + 16, cw + 24 of the stage: four independent
        // accumulator chains when they share a query (the usual case)
        constexpr int kR = static_cast<int>(kRsTile) / kRsConsumers;
        const uint32_t j0 = cw;
        bool same = j0 + (kR - 1) * kRsConsumers < n;
        const uint32_t q0 = j0 < n ? mq[s * kRsTile + j0] : 0u;
#pragma unroll
        for (int u = 1; u < kR; ++u) {
          same = same && mq[s * kRsTile + j0 + u * kRsConsumers] == q0;
        }
        if (same) {
          if (q0 != cur_q) stage_query(q0);
          double acc[kR];
          const float4* r4[kR];
#pragma unroll
          for (int u = 0; u < kR; ++u) {
            acc[u] = 0.0;
            r4[u] = reinterpret_cast<const float4*>(
                ring + (static_cast<size_t>(s) * kRsTile + j0 + u * kRsConsumers) * row_f);
          }
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const uint32_t jj = lane + 32u * c;
            if (jj < d / 4) {
#pragma unroll
              for (int u = 0; u < kR; ++u) Acc4<true>::run(metric, qd + 4 * c, r4[u][jj], acc[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < kR; ++u) acc[u] = warp_sum(acc[u]);
          if (lane == 0) {
#pragma unroll
            for (int u = 0; u < kR; ++u) {
              ckey[static_cast<uint64_t>(q0) * cap + mi[s * kRsTile + j0 + u * kRsConsumers]] =
                  order_key(acc[u], metric);
            }
          }
        } else {
          for (uint32_t j = j0; j < n; j += kRsConsumers) {
            const uint32_t q = mq[s * kRsTile + j];
            if (q != cur_q) stage_query(q);
            const float4* r4 = reinterpret_cast<const float4*>(
                ring + (static_cast<size_t>(s) * kRsTile + j) * row_f);
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              const uint32_t jj = lane + 32u * c;
              if (jj < d / 4) Acc4<true>::run(metric, qd + 4 * c, r4[jj], acc);
            }
            acc = warp_sum(acc);
            if (lane == 0) {
              ckey[static_cast<uint64_t>(q) * cap + mi[s * kRsTile + j]] = order_key(acc, metric);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
      }
    }
    tg += ntiles;
    __syncthreads(); // the chunk's metadata arrays are rewritten next
  }
}

constexpr int kSortThreads = 256;
template <int E>
__device__ void tc_sort_run(const uint64_t* kq, const uint32_t* cq, uint32_t n, uint64_t* sk,
                            uint32_t* sv, bool dense) {
  uint64_t k[E];
  uint32_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = threadIdx.x * E + e;
    v[e] = i < n ? cq[i] : ~0u;
    k[e] = i < n ? kq[dense ? v[e] : i] : ~0ull; // dense: keys indexed by centroid id
  }
  block_bitonic_sort<E>(k, v, sk, sv, static_cast<uint32_t>(kSortThreads) * E);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    sk[threadIdx.x * E + e] = k[e];
    sv[threadIdx.x * E + e] = v[e];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSortThreads)
    tc_sort_kernel(uint32_t cap, const uint32_t* __restrict__ cand,
                   const uint32_t* __restrict__ ncand, const uint64_t* __restrict__ ckey,
                   uint32_t n_out, uint32_t* __restrict__ order, const int64_t* res_off,
                   const uint64_t* list_off, FastTable ft, bool do_partition, bool scan_sorted,
                   bool dense) {
  extern __shared__ __align__(16) unsigned char smx[];
  const uint32_t q = blockIdx.x, n = ncand[q];
  uint32_t m = kSortThreads;
  while (m < n) m <<= 1;
  uint64_t* sk = reinterpret_cast<uint64_t*>(smx);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + m);
  const uint64_t* kq = ckey + static_cast<uint64_t>(q) * cap;
  const uint32_t* cq = cand + static_cast<uint64_t>(q) * cap;
  switch (m / kSortThreads) {
    case 1: tc_sort_run<1>(kq, cq, n, sk, sv, dense); break;
    case 2: tc_sort_run<2>(kq, cq, n, sk, sv, dense); break;
    case 4: tc_sort_run<4>(kq, cq, n, sk, sv, dense); break;
    case 8: tc_sort_run<8>(kq, cq, n, sk, sv, dense); break;
    case 16: tc_sort_run<16>(kq, cq, n, sk, sv, dense); break;
    default: tc_sort_run<32>(kq, cq, n, sk, sv, dense); break;
  }
  uint32_t* out = order + static_cast<uint64_t>(q) * n_out;
  for (uint32_t i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = sv[i];
  if (do_partition) {
    __syncthreads();
    if (scan_sorted) sort_ids_block(sv, n_out);
    partition_block(sv, n_out, res_off, list_off, ft, q);
  }
}


// --------------------------------------------------------------------------
// shared scan epilogue: CTA merge, grid merge, exact re-score of survivors
// --------------------------------------------------------------------------
// Epilogue candidates: (score, host-store row, slab vector index) in three
// shared-memory arrays. Rows stand in for datastore ids until the output; an
// exact score tie is broken by looking both ids up (vectorstore.hpp:34-39).
struct Cands {
  float* s;
  uint64_t* r;
  uint32_t* vi;
};

__host__ __device__ inline uint32_t pow2_ceil(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Entries of one ping-pong buffer: the largest level, power-of-two lists of
// power-of-two length.
__host__ __device__ inline uint32_t epilogue_entries(int nw, int kk, uint32_t grid) {
  const uint32_t m = pow2_ceil(static_cast<uint32_t>(kk));
  const uint32_t groups = (grid + kGroup - 1) / kGroup;
  uint32_t lists = pow2_ceil(static_cast<uint32_t>(nw));
  lists = lists > kGroup ? lists : kGroup;
  lists = lists > pow2_ceil(groups) ? lists : pow2_ceil(groups);
  return lists * m;
}
// Scratch bytes the epilogue needs (two ping-pong buffers).
__host__ __device__ inline size_t epilogue_scratch(int nw, int kk, uint32_t grid) {
  return 2 * (static_cast<size_t>(epilogue_entries(nw, kk, grid)) * 16 + 16);
}

__device__ inline Cands cands_at(unsigned char* base, uint32_t cap) {
  Cands c;
  c.s = reinterpret_cast<float*>(base);
  c.r = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(c.s + cap) + 7) & ~uintptr_t(7));
  c.vi = reinterpret_cast<uint32_t*>(c.r + cap);
  return c;
}

__device__ __forceinline__ bool cand_before(int metric, const uint64_t* ids, float sa,
                                            uint64_t ra, float sb, uint64_t rb) {
  if (sa != sb) return metric == kIP ? sa > sb : sa < sb;
  if (ra == rb || ra == ~0ull) return false;
  if (rb == ~0ull) return true;
  return __ldg(reinterpret_cast<const unsigned long long*>(ids) + ra) <
         __ldg(reinterpret_cast<const unsigned long long*>(ids) + rb);
}

__device__ __forceinline__ void cand_copy(Cands d, uint32_t i, Cands s, uint32_t j) {
  d.s[i] = s.s[j];
  d.r[i] = s.r[j];
  d.vi[i] = s.vi[j];
}

// One merge-path level: `lists` sorted lists of length m in `a` (list l at
// l * m) merge pairwise into lists / 2 lists of the best m in `b`. Every
// output is one co-rank binary search, so a level costs log2(m) steps.
__device__ void merge_level(int metric, const uint64_t* ids, Cands a, Cands b, uint32_t lists,
                            uint32_t m) {
  const uint32_t lm = __ffs(m) - 1;
  for (uint32_t x = threadIdx.x; x < (lists / 2) << lm; x += blockDim.x) {
    const uint32_t pr = x >> lm, p = x & (m - 1);
    const uint32_t A = 2 * pr * m, B = A + m;
    uint32_t lo = p > m ? p - m : 0, hi = p < m ? p : m;
    while (lo < hi) { // i = how many of the first p outputs come from A
      const uint32_t mid = (lo + hi) >> 1;
      if (cand_before(metric, ids, a.s[A + mid], a.r[A + mid], a.s[B + p - mid - 1],
                      a.r[B + p - mid - 1])) {
        lo = mid + 1;
      } else {
        hi = mid;
      }
    }
    const uint32_t i = lo, j = p - i;
    const bool from_a =
        j >= m || (i < m && cand_before(metric, ids, a.s[A + i], a.r[A + i], a.s[B + j], a.r[B + j]));
    cand_copy(b, pr * m + p, a, from_a ? A + i : B + j);
  }
}

// Reduces `lists` (power of two) sorted lists of length m held in *cur down
// to one (the best m) at (*cur)[0, m), ping-ponging with *alt.
__device__ void merge_tree(int metric, const uint64_t* ids, Cands* cur, Cands* alt,
                           uint32_t lists, uint32_t m) {
  while (lists > 1) {
    merge_level(metric, ids, *cur, *alt, lists, m);
    __syncthreads();
    const Cands t = *cur;
    *cur = *alt;
    *alt = t;
    lists >>= 1;
  }
}

// Block bitonic sort of n (power of two) candidates, best first.
__device__ void cands_sort(int metric, const uint64_t* ids, Cands c, uint32_t n) {
  for (uint32_t kk = 2; kk <= n; kk <<= 1) {
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t x = threadIdx.x; x < n / 2; x += blockDim.x) {
        const uint32_t lo = 2 * x - (x & (j - 1)), hi = lo + j;
        const bool up = (lo & kk) == 0;
        if (up == cand_before(metric, ids, c.s[hi], c.r[hi], c.s[lo], c.r[lo])) {
          const float ts = c.s[lo];
          c.s[lo] = c.s[hi];
          c.s[hi] = ts;
          const uint64_t tr = c.r[lo];
          c.r[lo] = c.r[hi];
          c.r[hi] = tr;
          const uint32_t tv = c.vi[lo];
          c.vi[lo] = c.vi[hi];
          c.vi[hi] = tv;
        }
      }
      __syncthreads();
    }
  }
}

__device__ void cands_fill(int metric, Cands c, uint32_t from, uint32_t to) {
  for (uint32_t x = from + threadIdx.x; x < to; x += blockDim.x) {
    c.s[x] = sentinel_score(metric);
    c.r[x] = ~0ull;
    c.vi[x] = ~0u;
  }
}

// Loads `lists` global lists of kk entries (written by other CTAs: L2, not
// L1) into lists of length m (padded with sentinels), then pads the list
// count to `lists2`; all loads in flight together.
__device__ void cands_load(int metric, Cands c, const float* ps, const uint64_t* pr,
                           const uint32_t* pvi, uint32_t lists, uint32_t kk, uint32_t m,
                           uint32_t lists2) {
  const uint32_t lm = __ffs(m) - 1;
  for (uint32_t x = threadIdx.x; x < lists2 << lm; x += blockDim.x) {
    const uint32_t l = x >> lm, e = x & (m - 1);
    if (l < lists && e < kk) {
      const uint64_t g = static_cast<uint64_t>(l) * kk + e;
      c.s[x] = __ldcg(ps + g);
      c.r[x] = __ldcg(reinterpret_cast<const unsigned long long*>(pr) + g);
      c.vi[x] = __ldcg(pvi + g);
    } else {
      c.s[x] = sentinel_score(metric);
      c.r[x] = ~0ull;
      c.vi[x] = ~0u;
    }
  }
}

// Exact fp64 re-score (vectorstore.cpp:93-115 arithmetic) of c[0, n) by the
// warps [first, first + nw), four candidates per warp in flight together.
__device__ void cands_rescore(int metric, Cands c, uint32_t n, const float* __restrict__ slab,
                              const float* sq, uint32_t d, int first, int nw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < first || warp >= first + nw) return;
  const int w = warp - first;
  for (uint32_t c0 = w; c0 < n; c0 += 4 * nw) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const float* rows[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t ci = c0 + u * nw;
      rows[u] = slab + static_cast<uint64_t>(ci < n ? c.vi[ci] : c.vi[c0]) * d;
    }
    if ((d & 3u) == 0) {
      const uint32_t d4 = d >> 2;
#pragma unroll 2
      for (uint32_t j4 = lane; j4 < d4; j4 += 32) {
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(rows[u]) + j4);
        const float4 qq = reinterpret_cast<const float4*>(sq)[j4];
        const double q4[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) Acc4<true>::run(metric, q4, x[u], acc[u]);
      }
    } else {
      for (uint32_t j = lane; j < d; j += 32) {
        const double qj = sq[j];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[u] = metric == kIP ? term_ip_d(qj, __ldg(rows[u] + j), acc[u])
                                 : term_l2_d(qj, __ldg(rows[u] + j), acc[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = warp_sum(acc[u]);
      const uint32_t ci = c0 + u * nw;
      if (lane == 0 && ci < n) c.s[ci] = finish_score<double>(metric, t);
    }
  }
}

// Scan epilogue, called by every thread once the warps [first, first + nw)
// hold their top-kk (keys = host-store rows) in registers and `scratch`
// (>= epilogue_scratch bytes) is free. Merges are merge-path trees over
// sorted lists:
//   1. CTA:   the nw warp lists -> the CTA's top-kk partial
//   2. group: the last of each kGroup CTAs merges the group's partials
//   3. final: the last group merges the group results, re-scores the
//             survivors exactly (fp32 accumulation), resolves rows to ids and
//             writes the top-k.
// Tickets self-reset, so the same buffers serve the next launch.
template <int KPL>
__device__ void scan_epilogue(WarpTopK<KPL>& top, int metric, int k, int kk, bool rerank,
                              unsigned char* scratch, const ScanOut& out, const float* sq,
                              const float* __restrict__ slab, const uint64_t* __restrict__ ids,
                              uint32_t d, uint64_t V, int first, int nw,
                              unsigned long long* t_merged = nullptr) {
  __shared__ bool last;
  const int warp = threadIdx.x >> 5;
  const uint32_t q = blockIdx.y, G = gridDim.x;
  const uint32_t ngroups = (G + kGroup - 1) / kGroup, g = blockIdx.x / kGroup;
  const uint32_t gsize = min(kGroup, G - g * kGroup);
  const uint32_t m = pow2_ceil(static_cast<uint32_t>(kk));
  const uint32_t cap = epilogue_entries(nw, kk, G);
  Cands cur = cands_at(scratch, cap);
  Cands alt = cands_at(scratch + cap * 16 + 16, cap);
  unsigned* tickets = out.ticket + static_cast<uint64_t>(q) * (kMaxGroups + 1);

  // ---- 1. CTA level ----
  const uint32_t wl = pow2_ceil(static_cast<uint32_t>(nw));
  if (warp >= first && warp < first + nw) {
    const uint32_t o = (warp - first) * m;
    top.store(kk, cur.s + o, cur.r + o, cur.vi + o);
  }
  for (uint32_t x = threadIdx.x; x < wl * m; x += blockDim.x) {
    if ((x & (m - 1)) >= static_cast<uint32_t>(kk) || (x >> (__ffs(m) - 1)) >= static_cast<uint32_t>(nw)) {
      cur.s[x] = sentinel_score(metric);
      cur.r[x] = ~0ull;
      cur.vi[x] = ~0u;
    }
  }
  __syncthreads();
  if (t_merged && threadIdx.x == 0) t_merged[0] = globaltimer();
  merge_tree(metric, ids, &cur, &alt, wl, m);
  if (t_merged && threadIdx.x == 0) t_merged[1] = globaltimer();
  const uint64_t pbase = static_cast<uint64_t>(q) * G * kk;
  if (out.cta_s != nullptr && !rerank) {
    // host-final mode: the host merges the grid's sorted lists
    for (uint32_t x = threadIdx.x; x < static_cast<uint32_t>(kk); x += blockDim.x) {
      const uint64_t o = pbase + static_cast<uint64_t>(blockIdx.x) * kk + x;
      out.cta_s[o] = cur.s[x];
      out.cta_r[o] = cur.r[x];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && out.fcount_out) {
      out.fcount_out[q] = out.fcount_in[q];
    }
    return;
  }
  for (uint32_t x = threadIdx.x; x < static_cast<uint32_t>(kk); x += blockDim.x) {
    const uint64_t o = pbase + static_cast<uint64_t>(blockIdx.x) * kk + x;
    out.part_s[o] = cur.s[x];
    out.part_id[o] = cur.r[x];
    out.part_vi[o] = cur.vi[x];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(tickets + g, 1u) == gsize - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();

  // ---- 2. group level ----
  const uint64_t gofs = pbase + static_cast<uint64_t>(g) * kGroup * kk;
  const uint32_t gl = pow2_ceil(gsize);
  cands_load(metric, cur, out.part_s + gofs, out.part_id + gofs, out.part_vi + gofs, gsize, kk,
             m, gl);
  __syncthreads();
  merge_tree(metric, ids, &cur, &alt, gl, m);
  const uint64_t gbase = static_cast<uint64_t>(q) * kMaxGroups * kk;
  for (uint32_t x = threadIdx.x; x < static_cast<uint32_t>(kk); x += blockDim.x) {
    const uint64_t o = gbase + static_cast<uint64_t>(g) * kk + x;
    out.gpart_s[o] = cur.s[x];
    out.gpart_id[o] = cur.r[x];
    out.gpart_vi[o] = cur.vi[x];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(tickets + kMaxGroups, 1u) == ngroups - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();

  // ---- 3. final ----
  const uint32_t fl = pow2_ceil(ngroups);
  cands_load(metric, cur, out.gpart_s + gbase, out.gpart_id + gbase, out.gpart_vi + gbase,
             ngroups, kk, m, fl);
  __syncthreads();
  merge_tree(metric, ids, &cur, &alt, fl, m);
  const uint32_t navail = static_cast<uint32_t>(V < static_cast<uint64_t>(kk) ? V : kk);
  if (rerank && navail > 0) {
    cands_fill(metric, cur, navail, m);
    cands_rescore(metric, cur, navail, slab, sq, d, first, nw);
    __syncthreads();
    cands_sort(metric, ids, cur, m);
  }
  for (uint32_t x = threadIdx.x; x < static_cast<uint32_t>(k); x += blockDim.x) {
    const uint64_t r = cur.r[x];
    out.out_s[static_cast<uint64_t>(q) * k + x] = cur.s[x];
    out.out_id[static_cast<uint64_t>(q) * k + x] = r == ~0ull ? ~0ull : ids[r]; // row -> id
  }
  for (uint32_t x = threadIdx.x; x <= ngroups; x += blockDim.x) {
    tickets[x == ngroups ? kMaxGroups : x] = 0;
  }
  if (threadIdx.x == 0) {
    out.out_count[q] = static_cast<uint32_t>(V < static_cast<uint64_t>(k) ? V : k);
    if (out.fcount_out) out.fcount_out[q] = out.fcount_in[q];
  }
}

// Cursor over a query's flattened fast-list vector space.
struct Cursor {
  uint32_t li;
  uint32_t len;
  uint64_t o;
  int64_t slab;
  uint64_t row;
  __device__ void load(const FastTable& ft, uint64_t tb) {
    len = ft.len[tb + li];
    slab = ft.slab[tb + li];
    row = ft.row[tb + li];
  }
  // position at flattened index v (pre: exclusive prefix over nf lists)
  __device__ void seek(const FastTable& ft, uint64_t tb, const uint64_t* pre, uint32_t nf,
                       uint64_t v) {
    uint32_t lo = 0, hi = nf - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= v) lo = mid;
      else hi = mid - 1;
    }
    li = lo;
    load(ft, tb);
    o = v - pre[lo];
    while (o >= len) { // skip empty lists
      ++li;
      load(ft, tb);
      o = 0;
    }
  }
  // Move forward n vectors; only called when the target position exists.
  __device__ void advance(const FastTable& ft, uint64_t tb, uint64_t n) {
    o += n;
    while (o >= len) {
      o -= len;
      ++li;
      load(ft, tb);
    }
  }
};

// --------------------------------------------------------------------------
// TMA-staged scan
// --------------------------------------------------------------------------
constexpr int kConsumers = 8;
constexpr int kTmaThreads = 32 * (kConsumers + 1);

// One CTA's share of a query's TMA scan: the range `cs` of the query's
// flattened fast-list vector space (V vectors in all), tiles streamed through
// the ring at `stage` (S stages of T rows), then the CTA merge and the
// epilogue. sq: the query in shared memory. Shared by scan_tma_kernel and
// fused_query_kernel. Returns the time the last tile was consumed when
// `probe` stamps are on.
template <bool kFp64, int KPL, int NCH>
__device__ __forceinline__ unsigned long long scan_tma_cta(
    const float* sq, uint32_t d, int metric, int k, int kk, const FastTable& ft, uint64_t tb,
    CtaStart cs, uint64_t V, const float* __restrict__ slab, const uint64_t* __restrict__ ids_all,
    const ScanOut& out, uint32_t T, uint32_t S, unsigned char* smem, uint64_t* full,
    uint64_t* empty, uint64_t* mrow, uint32_t* mvi, uint32_t* mn, bool probe,
    unsigned long long* s_first_tile, unsigned long long* t_merged = nullptr) {
  using ACC = typename std::conditional<kFp64, double, float>::type;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t stage_floats = static_cast<size_t>(T) * d;
  float* stage = reinterpret_cast<float*>(smem);
  const uint32_t nvec = cs.n;
  const uint32_t ntiles = (nvec + T - 1) / T;

  WarpTopK<KPL> top;
  top.ids = ids_all; // keys are host-store rows
  top.init(metric);

  if (warp == 0) {
    // ---------------- producer: one lane drives the bulk copies ----------
    if (lane == 0 && ntiles) {
      const uint64_t pol = l2_evict_first_policy();
      Cursor cur;
      cur.li = cs.li;
      cur.load(ft, tb);
      cur.o = cs.o;
      for (uint32_t i = 0; i < ntiles; ++i) {
        const uint32_t s = i % S;
        mbar_wait(empty + s, ((i / S) & 1u) ^ 1u);
        const uint32_t tile0 = i * T;
        const uint32_t n = min(T, nvec - tile0);
        // tile metadata first (published by the arrive), then the copies
        uint32_t j = 0;
        Cursor c2 = cur;
        while (true) {
          const uint32_t take = static_cast<uint32_t>(umin64(n - j, c2.len - c2.o));
          for (uint32_t t = 0; t < take; ++t) {
            mrow[s * T + j + t] = c2.row + c2.o + t;
            mvi[s * T + j + t] = static_cast<uint32_t>(c2.slab + c2.o + t);
          }
          j += take;
          if (j >= n) break;
          c2.advance(ft, tb, take);
        }
        mn[s] = n;
        mbar_arrive_expect_tx(full + s, n * d * 4u);
        j = 0;
        while (true) {
          const uint32_t take = static_cast<uint32_t>(umin64(n - j, cur.len - cur.o));
          bulk_g2s_hint(stage + s * stage_floats + static_cast<size_t>(j) * d,
                        slab + static_cast<uint64_t>(cur.slab + static_cast<int64_t>(cur.o)) * d,
                        take * d * 4u, full + s, pol);
          j += take;
          if (tile0 + j >= nvec) break;
          cur.advance(ft, tb, take);
          if (j >= n) break;
        }
      }
    }
  } else if (warp <= kConsumers) { // (the fused kernel's host I/O warp idles)
    // ---------------- consumers ----------------
    const int cw = warp - 1;
    float qf[NCH > 0 ? NCH * 4 : 1];
    double qd[(NCH > 0 && kFp64) ? NCH * 4 : 1];
    if constexpr (NCH > 0) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const float4 t = reinterpret_cast<const float4*>(sq)[c * 32 + lane];
        qf[4 * c + 0] = t.x;
        qf[4 * c + 1] = t.y;
        qf[4 * c + 2] = t.z;
        qf[4 * c + 3] = t.w;
        if constexpr (kFp64) {
          qd[4 * c + 0] = t.x;
          qd[4 * c + 1] = t.y;
          qd[4 * c + 2] = t.z;
          qd[4 * c + 3] = t.w;
        }
      }
    }
    for (uint32_t i = 0; i < ntiles; ++i) {
      const uint32_t s = i % S;
      mbar_wait(full + s, (i / S) & 1u);
      if (probe && i == 0 && cw == 0 && lane == 0) *s_first_tile = globaltimer();
      const uint32_t n = mn[s];
      const float* base = stage + s * stage_floats;
      for (uint32_t j = cw; j < n; j += 2 * kConsumers) {
        const uint32_t j2 = j + kConsumers;
        const bool two = j2 < n;
        const float4* r0 = reinterpret_cast<const float4*>(base + static_cast<size_t>(j) * d);
        const float4* r1 =
            reinterpret_cast<const float4*>(base + static_cast<size_t>(two ? j2 : j) * d);
        ACC a0 = ACC(0), a1 = ACC(0);
        if constexpr (NCH > 0) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const float4 x0 = r0[c * 32 + lane];
            const float4 x1 = r1[c * 32 + lane];
            if constexpr (kFp64) {
              Acc4<true>::run(metric, qd + 4 * c, x0, a0);
              Acc4<true>::run(metric, qd + 4 * c, x1, a1);
            } else {
              Acc4<false>::run(metric, qf + 4 * c, x0, a0);
              Acc4<false>::run(metric, qf + 4 * c, x1, a1);
            }
          }
        } else {
          const uint32_t d4 = d >> 2;
          for (uint32_t j4 = lane; j4 < d4; j4 += 32) {
            const float4 qq = reinterpret_cast<const float4*>(sq)[j4];
            if constexpr (kFp64) {
              const double q4[4] = {qq.x, qq.y, qq.z, qq.w};
              Acc4<true>::run(metric, q4, r0[j4], a0);
              Acc4<true>::run(metric, q4, r1[j4], a1);
            } else {
              const float q4[4] = {qq.x, qq.y, qq.z, qq.w};
              Acc4<false>::run(metric, q4, r0[j4], a0);
              Acc4<false>::run(metric, q4, r1[j4], a1);
            }
          }
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        const float s0 = finish_score<ACC>(metric, a0);
        top.offer(metric, kk, s0, mrow[s * T + j], mvi[s * T + j]);
        if (two) {
          const float s1 = finish_score<ACC>(metric, a1);
          top.offer(metric, kk, s1, mrow[s * T + j2], mvi[s * T + j2]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
  }
  __syncthreads(); // every tile consumed: the stage ring is free for merging
  const unsigned long long t_loop = probe ? globaltimer() : 0ull;
  scan_epilogue<KPL>(top, metric, k, kk, !kFp64, smem, out, sq, slab, ids_all, d, V, 1,
                     kConsumers, t_merged);
  return t_loop;
}

// Shared-memory layout of the TMA ring (scan_tma_kernel, fused_query_kernel):
// [S stages of T rows | >= the epilogue's merge scratch] [full[S] empty[S]]
// [mrow[S][T]] [mvi[S][T]] [mn[S]] [sq[d]] — then the fused kernel's tables.
struct RingSmem {
  uint64_t* full;
  uint64_t* empty;
  uint64_t* mrow;
  uint32_t* mvi;
  uint32_t* mn;
  float* sq;
  unsigned char* end; // first byte after sq[d]
};
__device__ __forceinline__ RingSmem ring_smem(unsigned char* smem, uint32_t T, uint32_t S,
                                              uint32_t d, int kk) {
  RingSmem r;
  const size_t stage_floats = static_cast<size_t>(T) * d;
  size_t off = (static_cast<size_t>(S) * stage_floats * 4 + 127) & ~size_t(127);
  const size_t merge_bytes = epilogue_scratch(kConsumers, kk, gridDim.x);
  if (off < merge_bytes) off = (merge_bytes + 127) & ~size_t(127);
  r.full = reinterpret_cast<uint64_t*>(smem + off);
  r.empty = r.full + S;
  r.mrow = r.empty + S;                                  // [S][T]
  r.mvi = reinterpret_cast<uint32_t*>(r.mrow + S * T);   // [S][T]
  r.mn = r.mvi + S * T;                                  // [S]
  r.sq = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(r.mn + S) + 15) & ~uintptr_t(15));
  r.end = reinterpret_cast<unsigned char*>(r.sq + d);
  return r;
}

__device__ __forceinline__ void ring_init(const RingSmem& r, uint32_t S) {
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(r.full + s, 1);
      mbar_init(r.empty + s, kConsumers);
    }
    fence_mbar_init();
  }
}

template <bool kFp64, int KPL, int NCH>
__global__ void __launch_bounds__(kTmaThreads, 1)
    scan_tma_kernel(const float* __restrict__ Q, uint32_t d, int metric, int k, int kk,
                    FastTable ft, const float* __restrict__ slab,
                    const uint64_t* __restrict__ ids_all, ScanOut out, uint32_t T, uint32_t S) {
  extern __shared__ __align__(128) unsigned char smem[];
  const RingSmem rs = ring_smem(smem, T, S, d, kk);
  const uint32_t q = blockIdx.y;
  // probe stamps stay on chip until the end: a store to mapped host memory
  // stalls the issuing warp for microseconds
  unsigned long long* probe =
      out.probe ? out.probe + (static_cast<uint64_t>(q) * gridDim.x + blockIdx.x) * 4 : nullptr;
  __shared__ unsigned long long s_first_tile;
  const unsigned long long t_entry = probe ? globaltimer() : 0ull;
  const float* qv = Q + static_cast<uint64_t>(q) * d;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) rs.sq[i] = qv[i];
  ring_init(rs, S);
  __syncthreads();

  const uint64_t tb = static_cast<uint64_t>(q) * ft.stride;
  const uint64_t* pre = ft.pre + static_cast<uint64_t>(q) * (ft.stride + 1);
  // this CTA's range, precomputed by the partition step (no search here)
  const CtaStart cs = ft.cta[static_cast<uint64_t>(q) * gridDim.x + blockIdx.x];
  const uint64_t V = pre[ft.count[q]];
  const unsigned long long t_loop = scan_tma_cta<kFp64, KPL, NCH>(
      rs.sq, d, metric, k, kk, ft, tb, cs, V, slab, ids_all, out, T, S, smem, rs.full, rs.empty,
      rs.mrow, rs.mvi, rs.mn, probe != nullptr, &s_first_tile);
  if (probe && threadIdx.x == 0) {
    const unsigned long long t_done = globaltimer();
    probe[0] = t_entry;
    probe[1] = s_first_tile;
    probe[2] = t_loop;
    probe[3] = t_done;
  }
}

// --------------------------------------------------------------------------
// fused single-query kernel: query fetch -> coarse scores -> top-L selection
// -> residency split -> TMA scan, one cooperative launch (ivf.cpp:269-343,
// tiered.cpp:148-185). The multi-kernel chain pays a launch gap per kernel and
// ranks on one SM; here every CTA scores a slice of the centroids, two grid
// barriers publish the query and the scores, and every CTA then ranks all nc
// keys itself (radix select in shared memory), splits the probe by residency
// and derives its own scan range, so the scan starts with no further barrier.
// --------------------------------------------------------------------------
constexpr int kFusedWarps = kConsumers + 2; // producer, 8 consumers, host I/O
constexpr int kFusedThreads = 32 * kFusedWarps;

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier of a cooperative launch (every CTA co-resident). The
// word's top bit flips once all gridDim.x CTAs have arrived (CTA 0 adds
// 2^31 - (G - 1), the others 1), so it needs no reset between barriers or
// launches. A watchdog turns a broken barrier into a launch error instead
// of a hung device.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned add = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
    __threadfence();
    const unsigned old = atomicAdd(bar, add);
    const uint64_t t0 = globaltimer();
    while (((old ^ ld_acquire_gpu(bar)) & 0x80000000u) == 0u) {
      if (globaltimer() - t0 > 20000000000ull) __trap(); // 20 s: far beyond any time slice
    }
    __threadfence();
  }
  __syncthreads();
}

struct FusedArgs {
  const float* src;             // query row (pinned host or HBM), unless
  const float* const* slot;     // set: mapped word holding the row pointer
  float* dQ;                    // HBM copy of the query, read by every CTA
  const float* cen;
  uint32_t nc, d, L;
  int metric;
  uint64_t* keys;               // [nc] order keys of the coarse scores
  const int64_t* res_off;
  const uint64_t* list_off;
  uint32_t* order_out;          // [L] the probe (mapped host memory)
  uint32_t* fcount_out;         // fast-list count (mapped)
  unsigned* flag_out;           // mapped: call sequence number, probe is out
  unsigned* done_out;           // mapped: call sequence number, results are out
  unsigned* ctl;                // [0] grid barrier word, [1] call sequence, [2] done ticket
  unsigned long long* stamps;   // [32] phase stamps of CTA 0 (mapped), nullable
  unsigned long long* cta_stamps; // [G][4] entry, query ready, keys ready, done; nullable
  int tables;                   // residency + list offsets bulk-copied into shared memory
  int qdirect;                  // every CTA reads a host row itself (diagnostics)
  const float* slab;
  const uint64_t* ids;
  ScanOut out;
  uint32_t T, S;
  int k, kk;
};

// Shared memory of the fused kernel beyond the ring (host and device agree):
// fast table (slab, row, pre, len, cluster) for L lists + G scan starts.
__host__ __device__ inline size_t fused_tables_bytes(uint32_t L, uint32_t G) {
  return 16 + static_cast<size_t>(L) * (8 + 8 + 4 + 4) + (static_cast<size_t>(L) + 1) * 8 +
         static_cast<size_t>(G) * sizeof(CtaStart) + 16;
}
// Selection scratch, aliased onto the ring before the scan starts.
__host__ __device__ inline size_t fused_select_bytes(uint32_t nc, uint32_t L) {
  return 2 * (static_cast<size_t>(nc) * 12 + 16) + static_cast<size_t>(L) * (8 + 4 + 4) + 64;
}
// Bytes of the residency table and list offsets as bulk-copied (16-byte
// multiples; the device arrays are padded for it).
__host__ __device__ inline size_t fused_res_bytes(uint32_t nc) {
  return (static_cast<size_t>(nc) * 8 + 15) & ~size_t(15);
}
__host__ __device__ inline size_t fused_off_bytes(uint32_t nc) {
  return (static_cast<size_t>(nc + 1) * 8 + 15) & ~size_t(15);
}
__host__ __device__ inline size_t fused_tables_at(uint32_t nc, uint32_t L) {
  return (fused_select_bytes(nc, L) + 127) & ~size_t(127);
}

template <int R, int NCHC>
__device__ __forceinline__ void fused_load_rows(const float* __restrict__ cen, uint32_t nc,
                                                uint32_t d4, uint32_t c0, int lane,
                                                float4 (&xs)[R][NCHC]) {
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const uint32_t c = c0 + u < nc ? c0 + u : 0u;
    const float4* r4 = reinterpret_cast<const float4*>(cen + static_cast<uint64_t>(c) * d4 * 4);
#pragma unroll
    for (int t = 0; t < NCHC; ++t) {
      const uint32_t j = lane + 32u * t;
      xs[u][t] = (c0 + u < nc && j < d4) ? __ldg(r4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// Scores of rows c0..c0+R-1 with exactly warp_coarse_score's sequence
// (lane-strided fp64 terms, then the butterfly), stored as order keys.
template <int R, int NCHC>
__device__ __forceinline__ void fused_score_rows(const float* sq, uint32_t nc, uint32_t d4,
                                                 uint32_t c0, int lane, int metric,
                                                 const float4 (&xs)[R][NCHC], uint64_t* keys) {
  double acc[R];
#pragma unroll
  for (int u = 0; u < R; ++u) acc[u] = 0.0;
#pragma unroll
  for (int t = 0; t < NCHC; ++t) {
    const uint32_t j = lane + 32u * t;
    if (j < d4) {
      const float4 qq = reinterpret_cast<const float4*>(sq)[j];
      const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
      for (int u = 0; u < R; ++u) Acc4<true>::run(metric, qd, xs[u][t], acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const double v = warp_sum(acc[u]);
    if (lane == 0 && c0 + u < nc) __stcg(reinterpret_cast<unsigned long long*>(keys) + c0 + u,
                                         static_cast<unsigned long long>(order_key(v, metric)));
  }
}

// ---- top-L selection inside one CTA -------------------------------------
// The ranking order is (key, cluster id) ascending (ivf.cpp:282-289), i.e.
// the unique 96-bit composite key:id. A radix select walks its digits from
// the highest bit where the keys differ; each pass histograms the current
// group (the entries sharing the resolved prefix), moves the entries of lower
// bins to the selection and keeps the boundary bin as the next, much smaller
// group. It stops when the boundary bin is taken whole or the group is small
// enough to rank directly. The selected L entries are then ordered by rank
// counting.
constexpr uint32_t kRankCap = 64;

__device__ __forceinline__ bool comp_less(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
  return ka < kb || (ka == kb && va < vb);
}
// Bits [shift, shift + w) of the composite (key << 32 | id), w <= 8.
__device__ __forceinline__ uint32_t comp_digit(uint64_t key, uint32_t id, int shift, uint32_t mask) {
  const uint64_t v = shift >= 32 ? (key >> (shift - 32))
                                 : ((key << (32 - shift)) | (static_cast<uint64_t>(id) >> shift));
  return static_cast<uint32_t>(v) & mask;
}

struct SelectScratch {
  uint64_t* gk[2]; // group keys, ping-pong (nc entries each)
  uint32_t* gv[2]; // group ids
  uint64_t* sel_k; // the L selected
  uint32_t* sel_v;
};

// The first L (L <= nc) of the ranking of sk[0, nc) into probe[0, L). va /
// vo / kmin: the AND, OR and minimum of all keys (computed while loading
// them). sk may be overwritten (its space backs group buffer 1).
//
// Fast path: warp 0 ranks 64 evenly spaced keys; the one of rank ~3L*64/nc
// is a threshold with about 3L keys below it. One pass histograms only the
// keys at or below it (few, so the shared-memory atomics hardly collide) into
// 256 bins relative to kmin; the lower bins go to the selection and the
// boundary bin becomes the group. If fewer than L keys fall below the
// threshold (an unlucky sample) the selection restarts on the general path:
// radix passes over the composite bits from the highest differing one.
__device__ void block_select_topL(const uint64_t* sk, uint32_t nc, uint32_t L,
                                  unsigned long long va, unsigned long long vo,
                                  unsigned long long kmin, const SelectScratch& sc,
                                  uint32_t* probe, unsigned long long* dbg = nullptr) {
  // dbg (thread 0, diagnostics): [0] start, [1..8] after each pass,
  // [9] selected, [10] ranked, [11] passes run
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_nsel, s_ng, s_need, s_m, s_dsel, s_before, s_flag;
  __shared__ unsigned long long s_test, s_and, s_or, w_ka[32], w_ko[32], w_ia[32], w_io[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  if (L == 0) return;
  if (dbg && threadIdx.x == 0) dbg[0] = globaltimer();
  uint64_t* gk[2] = {sc.gk[0], sc.gk[1]};
  uint32_t* gv[2] = {sc.gv[0], sc.gv[1]};
  uint64_t* selk = sc.sel_k;
  uint32_t* selv = sc.sel_v;
  int npass = 0;

  // the boundary bin of a histogram (warp 0): s_dsel, s_before (entries in
  // lower bins), s_m (boundary bin size), s_flag = 1 if it is taken whole,
  // 2 if the histogram holds fewer than `need` entries
  auto find_boundary = [&](uint32_t need) {
    uint32_t h[8], sum = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      h[e] = hist[lane * 8 + e];
      sum += h[e];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    uint32_t before = incl - sum;
    if (before < need && need <= incl) {
      int e = 0;
      while (before + h[e] < need) before += h[e++];
      s_dsel = static_cast<uint32_t>(lane * 8 + e);
      s_before = before;
      s_flag = h[e] == need - before ? 1u : 0u;
      s_m = h[e];
    }
    if (lane == 31 && incl < need) s_flag = 2u;
    if (lane == 0) s_ng = 0;
  };

  if (L >= nc) {
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
      selk[i] = sk[i];
      selv[i] = i;
    }
  } else {
    if (threadIdx.x == 0) {
      s_nsel = 0;
      s_need = L;
      s_test = ~0ull;
    }
    // ---- threshold from a 64-key sample -------------------------------
    const uint32_t rs = static_cast<uint32_t>((3ull * L * 64 + nc - 1) / nc);
    const bool sampled = rs < 48 && nc >= 512;
    if (sampled) {
      // rank of each sample among the 64 (ties by sample index): every
      // thread compares one sample with a slice of the others
      __shared__ uint32_t srank[64];
      __shared__ unsigned long long sval[64];
      if (threadIdx.x < 64) {
        srank[threadIdx.x] = 0;
        sval[threadIdx.x] = sk[static_cast<uint64_t>(threadIdx.x) * nc / 64];
      }
      __syncthreads();
      const uint32_t parts = max(1u, blockDim.x / 64u);
      if (threadIdx.x < parts * 64u) {
        const uint32_t si = threadIdx.x & 63u, part = threadIdx.x >> 6;
        const unsigned long long v = sval[si];
        uint32_t r = 0;
        for (uint32_t j = part * 64u / parts; j < (part + 1) * 64u / parts; ++j) {
          const unsigned long long b = sval[j];
          r += (b < v || (b == v && j < si)) ? 1u : 0u;
        }
        atomicAdd(&srank[si], r);
      }
      __syncthreads();
      if (threadIdx.x < 64 && srank[threadIdx.x] == rs) s_test = sval[threadIdx.x];
    }
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned long long T = s_test;
    int cur = -1; // -1: the group is sk with ids 0..nc-1
    bool done = false, general = T == ~0ull;
    if (!general) {
      const unsigned long long span = T - kmin;
      const int sh = span ? max(0, 64 - __clzll(static_cast<long long>(span)) - 8) : 0;
      for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
        const unsigned long long k = sk[i];
        if (k <= T) atomicAdd(&hist[static_cast<uint32_t>((k - kmin) >> sh)], 1u);
      }
      __syncthreads();
      if (warp == 0) find_boundary(L);
      __syncthreads();
      if (s_flag == 2u) {
        general = true; // fewer than L keys at or below the sample threshold
      } else {
        const uint32_t dsel = s_dsel, whole = s_flag;
        for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
          const unsigned long long k = sk[i];
          if (k > T) continue;
          const uint32_t bn = static_cast<uint32_t>((k - kmin) >> sh);
          if (bn < dsel || (bn == dsel && whole)) {
            const uint32_t p = atomicAdd(&s_nsel, 1u);
            selk[p] = k;
            selv[p] = i;
          } else if (bn == dsel) {
            const uint32_t p = atomicAdd(&s_ng, 1u);
            gk[0][p] = k;
            gv[0][p] = i;
          }
        }
        ++npass;
        __syncthreads();
        if (dbg && threadIdx.x == 0) dbg[npass] = globaltimer();
        if (whole) {
          done = true;
        } else {
          if (threadIdx.x == 0) s_need = L - s_before;
          cur = 0;
        }
      }
    }
    int top = 0;
    if (!done) {
      if (general) {
        const unsigned long long diff = va ^ vo;
        top = diff ? 32 + (63 - __clzll(static_cast<long long>(diff)))
                   : (nc > 1 ? 31 - __clz(static_cast<int>(nc - 1)) : 0);
        if (threadIdx.x == 0) {
          s_nsel = 0;
          s_need = L;
          s_m = nc;
        }
        __syncthreads();
      } else if (s_m > kRankCap) {
        // the group shares the bits above the highest one its composites
        // differ in
        unsigned long long ka = ~0ull, ko = 0ull, ia = ~0ull, io = 0ull;
        for (uint32_t i = threadIdx.x; i < s_m; i += blockDim.x) {
          ka &= gk[0][i];
          ko |= gk[0][i];
          ia &= gv[0][i];
          io |= gv[0][i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ka &= __shfl_xor_sync(kFull, ka, o);
          ko |= __shfl_xor_sync(kFull, ko, o);
          ia &= __shfl_xor_sync(kFull, ia, o);
          io |= __shfl_xor_sync(kFull, io, o);
        }
        if (lane == 0) {
          w_ka[warp] = ka;
          w_ko[warp] = ko;
          w_ia[warp] = ia;
          w_io[warp] = io;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long a1 = ~0ull, o1 = 0ull, a2 = ~0ull, o2 = 0ull;
          for (int w = 0; w < nwarps; ++w) {
            a1 &= w_ka[w];
            o1 |= w_ko[w];
            a2 &= w_ia[w];
            o2 |= w_io[w];
          }
          s_and = a1 ^ o1; // bits the group's keys differ in
          s_or = a2 ^ o2;  // ... and its ids
        }
        __syncthreads();
        const unsigned long long dk = s_and, di = s_or;
        top = dk ? 32 + (63 - __clzll(static_cast<long long>(dk)))
                 : (di ? 63 - __clzll(static_cast<long long>(di)) : 0);
      }
    }
    while (!done) {
      if (cur >= 0 && s_m <= kRankCap) {
        // rank the small group directly; composites are unique
        const uint32_t gm = s_m, need = s_need;
        for (uint32_t e = threadIdx.x; e < gm; e += blockDim.x) {
          const uint64_t ke = gk[cur][e];
          const uint32_t ve = gv[cur][e];
          uint32_t r = 0;
          for (uint32_t j = 0; j < gm; ++j) r += comp_less(gk[cur][j], gv[cur][j], ke, ve);
          if (r < need) {
            const uint32_t p = atomicAdd(&s_nsel, 1u);
            selk[p] = ke;
            selv[p] = ve;
          }
        }
        break;
      }
      const int w = top >= 7 ? 8 : top + 1;
      const int shift = top + 1 - w;
      const uint32_t dmask = (1u << w) - 1u;
      const uint32_t m = s_m;
      const uint64_t* ck = cur < 0 ? sk : gk[cur];
      const uint32_t* cv = cur < 0 ? nullptr : gv[cur];
      for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        atomicAdd(&hist[comp_digit(ck[i], cv ? cv[i] : i, shift, dmask)], 1u);
      }
      __syncthreads();
      if (warp == 0) find_boundary(s_need);
      __syncthreads();
      const uint32_t dsel = s_dsel, whole = s_flag == 1u;
      const int nxt = cur < 0 ? 0 : cur ^ 1;
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint64_t key = ck[i];
        const uint32_t id = cv ? cv[i] : i;
        const uint32_t dg = comp_digit(key, id, shift, dmask);
        if (dg < dsel || (dg == dsel && whole)) {
          const uint32_t p = atomicAdd(&s_nsel, 1u);
          selk[p] = key;
          selv[p] = id;
        } else if (dg == dsel) {
          const uint32_t p = atomicAdd(&s_ng, 1u);
          gk[nxt][p] = key;
          gv[nxt][p] = id;
        }
      }
      __syncthreads();
      ++npass;
      if (dbg && threadIdx.x == 0 && npass <= 8) dbg[npass] = globaltimer();
      if (whole) break;
      if (threadIdx.x == 0) s_need = s_need - s_before;
      cur = nxt;
      top = shift - 1;
      __syncthreads();
    }
  }
  __syncthreads();
  if (dbg && threadIdx.x == 0) dbg[9] = globaltimer();
  // order the L selected by rank counting, every thread one (entry, slice
  // of the others) pair; the counters reuse group buffer 0
  {
    uint32_t* rank = gv[0];
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) rank[i] = 0;
    __syncthreads();
    const uint32_t parts = max(1u, blockDim.x / L);
    for (uint32_t t = threadIdx.x; t < parts * L; t += blockDim.x) {
      const uint32_t e = t % L, part = t / L;
      const uint64_t ke = selk[e];
      const uint32_t ve = selv[e];
      uint32_t r = 0;
      const uint32_t j1 = (part + 1) * L / parts;
#pragma unroll 4
      for (uint32_t j = part * L / parts; j < j1; ++j) r += comp_less(selk[j], selv[j], ke, ve);
      atomicAdd(&rank[e], r);
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < L; e += blockDim.x) probe[rank[e]] = selv[e];
  }
  __syncthreads();
  if (dbg && threadIdx.x == 0) {
    dbg[10] = globaltimer();
    dbg[11] = static_cast<unsigned long long>(npass);
  }
}

template <bool kFp64, int KPL, int NCH>
__global__ void __launch_bounds__(kFusedThreads, 1) fused_query_kernel(FusedArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const RingSmem rs = ring_smem(smem, a.T, a.S, a.d, a.kk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t d4 = a.d >> 2, L = a.L, G = gridDim.x;
  const bool stamp = a.stamps != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __shared__ unsigned long long s_dbg[12];
  const unsigned long long t_in = a.cta_stamps ? globaltimer() : 0ull;
  if (stamp) st[0] = globaltimer();

  // fast table of this query (shared memory after the ring's sq)
  unsigned char* tp = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(rs.end) + 15) & ~uintptr_t(15));
  int64_t* f_slab = reinterpret_cast<int64_t*>(tp);
  uint64_t* f_row = reinterpret_cast<uint64_t*>(f_slab + L);
  uint64_t* f_pre = f_row + L;
  CtaStart* f_cta = reinterpret_cast<CtaStart*>(f_pre + L + 1);
  uint32_t* f_len = reinterpret_cast<uint32_t*>(f_cta + G);
  uint32_t* f_clu = f_len + L;
  __shared__ uint32_t f_count;
  FastTable ft;
  ft.slab = f_slab;
  ft.row = f_row;
  ft.len = f_len;
  ft.cluster = f_clu;
  ft.pre = f_pre;
  ft.count = &f_count;
  ft.cta = f_cta;
  ft.stride = L;
  ft.grid = G;

  // ---- 0. the query -> HBM; meanwhile the first centroid rows load --------
  constexpr int NCHC = NCH > 0 ? NCH : 8; // float4 chunks per lane (d <= 1024)
  constexpr int R = NCH > 0 ? 4 : 2;      // centroid rows per warp per round
  const uint32_t gw = blockIdx.x * kFusedWarps + warp, GW = G * kFusedWarps;
  // A staged query (HBM row named by the mapped slot) is read by every CTA
  // straight into shared memory; a host row (pinned, PCIe) is copied to HBM
  // once by CTA 0 behind a grid barrier.
  unsigned long long q_st[3] = {0, 0, 0};
  const bool direct = a.slot != nullptr || a.qdirect;
  const float* src = nullptr;
  if (direct || blockIdx.x == 0) {
    src = a.slot ? *reinterpret_cast<const float* const volatile*>(a.slot) : a.src;
  }
  float4 xs[R][NCHC];
  fused_load_rows<R, NCHC>(a.cen, a.nc, d4, gw * R, lane, xs);
  if (direct) {
    if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
      for (uint32_t i = threadIdx.x; i < d4; i += blockDim.x) {
        reinterpret_cast<float4*>(rs.sq)[i] = reinterpret_cast<const float4*>(src)[i];
      }
    } else {
      for (uint32_t i = threadIdx.x; i < a.d; i += blockDim.x) rs.sq[i] = src[i];
    }
    if (stamp) q_st[1] = globaltimer();
    ring_init(rs, a.S);
    __syncthreads();
    // the row also lands in dQ: the miss path's chunk scans that follow this
    // kernel on the stream (runtime fetch, peer copies) read the query there
    if (blockIdx.x == 0) {
      for (uint32_t i = threadIdx.x; i < a.d; i += blockDim.x) a.dQ[i] = rs.sq[i];
    }
  } else {
    if (blockIdx.x == 0) {
      if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
        for (uint32_t i = threadIdx.x; i < d4; i += blockDim.x) {
          reinterpret_cast<float4*>(a.dQ)[i] = reinterpret_cast<const float4*>(src)[i];
        }
      } else {
        for (uint32_t i = threadIdx.x; i < a.d; i += blockDim.x) a.dQ[i] = src[i];
      }
      if (stamp) q_st[1] = globaltimer();
    }
    ring_init(rs, a.S);
    if (stamp) q_st[2] = globaltimer();
    grid_sync(a.ctl);
    for (uint32_t i = threadIdx.x; i < d4; i += blockDim.x) {
      reinterpret_cast<float4*>(rs.sq)[i] = __ldcg(reinterpret_cast<const float4*>(a.dQ) + i);
    }
    __syncthreads();
  }
  // the residency table and list offsets stream into shared memory while the
  // coarse phase and the selection run (the split needs them after)
  __shared__ __align__(8) uint64_t tbar;
  const int64_t* res_tab = a.res_off;
  const uint64_t* off_tab = a.list_off;
  if (a.tables) {
    unsigned char* tb0 = smem + fused_tables_at(a.nc, L);
    if (threadIdx.x == 0) {
      mbar_init(&tbar, 1);
      fence_mbar_init();
      const uint32_t rb = static_cast<uint32_t>(fused_res_bytes(a.nc));
      const uint32_t ob = static_cast<uint32_t>(fused_off_bytes(a.nc));
      mbar_arrive_expect_tx(&tbar, rb + ob);
      bulk_g2s(tb0, a.res_off, rb, &tbar);
      bulk_g2s(tb0 + rb, a.list_off, ob, &tbar);
    }
    res_tab = reinterpret_cast<const int64_t*>(tb0);
    off_tab = reinterpret_cast<const uint64_t*>(tb0 + fused_res_bytes(a.nc));
  }
  if (stamp) st[1] = globaltimer();
  const unsigned long long t_b1 = a.cta_stamps ? globaltimer() : 0ull;

  // ---- 1. coarse scores of this CTA's centroid rows -> order keys ---------
  for (uint32_t c0 = gw * R; c0 < a.nc; c0 += GW * R) {
    if (c0 != gw * R) fused_load_rows<R, NCHC>(a.cen, a.nc, d4, c0, lane, xs);
    fused_score_rows<R, NCHC>(rs.sq, a.nc, d4, c0, lane, a.metric, xs, a.keys);
  }
  grid_sync(a.ctl);
  if (stamp) st[2] = globaltimer();
  if (a.cta_stamps && threadIdx.x == 0) {
    unsigned long long* cs3 = a.cta_stamps + 4ull * blockIdx.x;
    cs3[0] = t_in;
    cs3[1] = t_b1;
    cs3[2] = globaltimer();
  }

  // ---- 2. every CTA ranks all nc keys (scratch aliased on the ring) -------
  // [keys / group 1: nc x 12 B][group 0: nc x 12 B][selection: L x 12 B][probe]
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem);
  SelectScratch sc;
  sc.gk[1] = sk;
  sc.gv[1] = reinterpret_cast<uint32_t*>(sk + a.nc);
  sc.gk[0] = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(sc.gv[1] + a.nc) + 15) & ~uintptr_t(15));
  sc.gv[0] = reinterpret_cast<uint32_t*>(sc.gk[0] + a.nc);
  sc.sel_k = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(sc.gv[0] + a.nc) + 15) & ~uintptr_t(15));
  sc.sel_v = reinterpret_cast<uint32_t*>(sc.sel_k + L);
  uint32_t* probe = sc.sel_v + L;
  unsigned long long va = ~0ull, vo = 0ull, vmin = ~0ull;
  {
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(a.keys);
    // eight 16-byte loads per thread in flight per round (the stores to
    // shared memory would otherwise serialise them behind each other)
    constexpr int kB = 8;
    const uint32_t n2 = a.nc / 2;
    for (uint32_t base = 0; base < n2; base += kB * blockDim.x) {
      ulonglong2 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        v[u] = i < n2 ? __ldcg(k2 + i) : make_ulonglong2(~0ull, ~0ull);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        if (i < n2) {
          sk[2 * i] = v[u].x;
          sk[2 * i + 1] = v[u].y;
          va &= v[u].x & v[u].y;
          vo |= v[u].x | v[u].y;
          vmin = min(vmin, min(v[u].x, v[u].y));
        }
      }
    }
    if ((a.nc & 1u) && threadIdx.x == 0) {
      const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(a.keys) + a.nc - 1);
      sk[a.nc - 1] = v;
      va &= v;
      vo |= v;
      vmin = min(vmin, v);
    }
  }
  {
    __shared__ unsigned long long w_and[32], w_or[32], w_min[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      va &= __shfl_xor_sync(kFull, va, o);
      vo |= __shfl_xor_sync(kFull, vo, o);
      vmin = min(vmin, __shfl_xor_sync(kFull, vmin, o));
    }
    if (lane == 0) {
      w_and[warp] = va;
      w_or[warp] = vo;
      w_min[warp] = vmin;
    }
    __syncthreads();
    va = ~0ull;
    vo = 0ull;
    vmin = ~0ull;
    for (int w = 0; w < kFusedWarps; ++w) {
      va &= w_and[w];
      vo |= w_or[w];
      vmin = min(vmin, w_min[w]);
    }
  }
  if (stamp) st[3] = globaltimer();
  block_select_topL(sk, a.nc, L, va, vo, vmin, sc, probe,
                    a.stamps && blockIdx.x == 0 ? s_dbg : nullptr);
  if (stamp) st[4] = globaltimer();
  // residency split + this query's scan-CTA start table (partition step)
  if (a.tables) mbar_wait(&tbar, 0);
  partition_block(probe, L, res_tab, off_tab, ft, 0);
  __syncthreads();
  if (blockIdx.x == 0 && warp == kFusedWarps - 1) {
    // host I/O warp: the probe and the fast count go out, then the flag
    for (uint32_t i = lane; i < L; i += 32) a.order_out[i] = probe[i];
    if (lane == 0) {
      *a.fcount_out = f_count;
      const unsigned s = a.ctl[1] + 1u;
      a.ctl[1] = s;
      __threadfence_system();
      *reinterpret_cast<volatile unsigned*>(a.flag_out) = s;
    }
  }
  if (stamp) st[5] = globaltimer();
  // the scratch was written through the generic proxy; the ring's bulk
  // copies write the same bytes through the async proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  // ---- 3. scan of this CTA's range of the fast lists ----------------------
  const uint64_t V = f_pre[f_count];
  const CtaStart cs = (L > 0 && f_count > 0) ? f_cta[blockIdx.x] : CtaStart{0u, 0u, 0u, 0u};
  __shared__ unsigned long long s_first_tile;
  const unsigned long long t_loop = scan_tma_cta<kFp64, KPL, NCH>(
      rs.sq, a.d, a.metric, a.k, a.kk, ft, 0, cs, V, a.slab, a.ids, a.out, a.T, a.S, smem, rs.full,
      rs.empty, rs.mrow, rs.mvi, rs.mn, stamp, &s_first_tile, stamp ? &q_st[1] : nullptr);
  if (a.cta_stamps && threadIdx.x == 0) a.cta_stamps[4ull * blockIdx.x + 3] = globaltimer();
  if (stamp) {
    st[6] = t_loop;
    st[7] = globaltimer();
    for (int i = 0; i < 8; ++i) a.stamps[i] = st[i];
    for (int i = 0; i < 12; ++i) a.stamps[8 + i] = s_dbg[i];
    for (int i = 0; i < 3; ++i) a.stamps[20 + i] = q_st[i];
  }
  // completion: the last CTA to finish publishes the call's sequence number
  // after every CTA's results (mapped host memory) are visible, so the host
  // need not wait for the kernel's teardown and its event
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(a.ctl + 2, 1u) == gridDim.x - 1) {
      a.ctl[2] = 0u;
      const unsigned s = *reinterpret_cast<volatile unsigned*>(a.ctl + 1);
      __threadfence_system();
      *reinterpret_cast<volatile unsigned*>(a.done_out) = s;
    }
  }
}

// --------------------------------------------------------------------------
// LDG scan (direct 128-bit loads into registers)
// --------------------------------------------------------------------------
constexpr int kScanWarps = 8;
constexpr int kScanThreads = kScanWarps * 32;
constexpr int kU = 2; // vectors in flight per warp iteration

template <bool kFp64, int KPL, int NCH>
__global__ void __launch_bounds__(kScanThreads, 2)
    scan_ldg_kernel(const float* __restrict__ Q, uint32_t d, int metric, int k, int kk,
                    FastTable ft, const float* __restrict__ slab_vecs,
                    const uint64_t* __restrict__ ids_all, ScanOut out) {
  using ACC = typename std::conditional<kFp64, double, float>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sq = reinterpret_cast<float*>(smem_raw);
  unsigned char* scratch = smem_raw + ((static_cast<size_t>(d) * 4 + 15) & ~size_t(15));

  const uint32_t q = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* qv = Q + static_cast<uint64_t>(q) * d;
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) sq[i] = qv[i];
  __syncthreads();

  const uint64_t tb = static_cast<uint64_t>(q) * ft.stride;
  const uint64_t* pre = ft.pre + static_cast<uint64_t>(q) * (ft.stride + 1);
  const uint32_t nf = ft.count[q];
  const uint64_t V = pre[nf];

  WarpTopK<KPL> top;
  top.ids = ids_all; // keys are host-store rows
  top.init(metric);

  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kScanWarps;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kScanWarps + warp;
  const uint64_t v0 = V * gw / tw, v1 = V * (gw + 1) / tw;

  float qf[NCH > 0 ? NCH * 4 : 1];
  if constexpr (NCH > 0) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const float4 t = reinterpret_cast<const float4*>(sq)[c * 32 + lane];
      qf[4 * c + 0] = t.x;
      qf[4 * c + 1] = t.y;
      qf[4 * c + 2] = t.z;
      qf[4 * c + 3] = t.w;
    }
  }

  if (v0 < v1) {
    Cursor cur;
    cur.seek(ft, tb, pre, nf, v0);
    for (uint64_t v = v0; v < v1; v += kU) {
      int64_t vec[kU];
      uint64_t rowi[kU];
      bool valid[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        valid[u] = v + u < v1;
        vec[u] = cur.slab + static_cast<int64_t>(cur.o);
        rowi[u] = cur.row + cur.o;
        if (valid[u] && v + u + 1 < v1) cur.advance(ft, tb, 1);
      }
      ACC acc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) acc[u] = ACC(0);
      if constexpr (NCH > 0) {
        float4 x[kU][NCH];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const float4* p =
              reinterpret_cast<const float4*>(slab_vecs + static_cast<uint64_t>(vec[u]) * (NCH * 128)) +
              lane;
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            x[u][c] = valid[u] ? ldg_stream(p + c * 32) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if constexpr (kFp64) {
              const double q4[4] = {qf[4 * c], qf[4 * c + 1], qf[4 * c + 2], qf[4 * c + 3]};
              Acc4<true>::run(metric, q4, x[u][c], acc[u]);
            } else {
              Acc4<false>::run(metric, qf + 4 * c, x[u][c], acc[u]);
            }
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (!valid[u]) continue;
          const float* p = slab_vecs + static_cast<uint64_t>(vec[u]) * d;
          for (uint32_t j = lane; j < d; j += 32) {
            const float xv = __ldg(p + j);
            if constexpr (kFp64) {
              acc[u] = metric == kIP ? term_ip_d(sq[j], xv, acc[u]) : term_l2_d(sq[j], xv, acc[u]);
            } else {
              acc[u] = metric == kIP ? term_ip_f(sq[j], xv, acc[u]) : term_l2_f(sq[j], xv, acc[u]);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const ACC tot = warp_sum(acc[u]);
        if (!valid[u]) continue;
        const float cs = finish_score<ACC>(metric, tot);
        top.offer(metric, kk, cs, rowi[u], static_cast<uint32_t>(vec[u]));
      }
    }
  }
  __syncthreads();
  scan_epilogue<KPL>(top, metric, k, kk, !kFp64, scratch, out, sq, slab_vecs, ids_all, d, V, 0,
                     kScanWarps);
}

// --------------------------------------------------------------------------
// generation window
// --------------------------------------------------------------------------
// First node of the captured single-query chain: copies the query into d_Q
// from `src` (the pinned staging row: a fixed argument) or, when `slot` is
// set, from the pointer the host left in that mapped word (a staged HBM row
// that changes per call). Both are device-addressable under UVA; neither
// needs the graph node re-pointed (that costs ~4 us + a slower launch).
__global__ void __launch_bounds__(256) fetch_query_kernel(const float* src,
                                                          const float* const* slot, float* dQ,
                                                          uint32_t d) {
  if (slot != nullptr) src = *reinterpret_cast<const float* const volatile*>(slot);
  if ((d & 3u) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    for (uint32_t i = threadIdx.x; i < d / 4; i += blockDim.x) {
      reinterpret_cast<float4*>(dQ)[i] = reinterpret_cast<const float4*>(src)[i];
    }
  } else {
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) dQ[i] = src[i];
  }
}

__global__ void window_kernel(uint64_t ns) {
  const uint64_t t0 = globaltimer();
  while (globaltimer() - t0 < ns) {
    __nanosleep(2000);
  }
}

// Decode-like generation window: for `ns` nanoseconds, one "token" every
// period_ns streams the whole buffer (an LLM decode step reads every weight
// once) at full speed, then idles until the next token is due. The HBM,
// L2 and SM load of a memory-bound decode thus share the device with the
// lookahead copies. Bytes read are counted into *bytes_read.
__global__ void __launch_bounds__(512) window_stream_kernel(const float4* __restrict__ buf,
                                                            uint64_t n16, uint64_t ns,
                                                            uint64_t period_ns, float* sink,
                                                            unsigned long long* bytes_read) {
  const uint64_t t0 = globaltimer();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  float acc = 0.f;
  uint64_t mine = 0;
  for (uint64_t tok = 0;; ++tok) {
    const uint64_t due = tok * period_ns;
    uint64_t now = globaltimer() - t0;
    if (now >= ns) break;
    while (now < due) {
      __nanosleep(1000);
      now = globaltimer() - t0;
      if (now >= ns) break;
    }
    if (now >= ns) break;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n16;
         i += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t j = i + u * stride;
        v[u] = j < n16 ? ldg_stream(buf + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
      mine += 4;
    }
  }
  if (acc == 1234.5f) *sink = acc; // keeps the loads; never true for the zeroed buffer
  const uint64_t tot = __reduce_add_sync(kFull, static_cast<unsigned>(mine));
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(bytes_read, static_cast<unsigned long long>(tot) * 16ull);
}

// --------------------------------------------------------------------------
// launch plumbing
// --------------------------------------------------------------------------
struct TmaGeom {
  uint32_t T, S;
  size_t smem;
};

TmaGeom tma_geom(uint32_t d, int kk, uint32_t grid, const ScanTune& tune) {
  const size_t row = size_t(d) * 4;
  TmaGeom g;
  // ~96 KB stages in a ~192 KB ring: measured best at d = 768 (32 rows x 2
  // stages: 7.0 TB/s marginal vs 6.6 for 16 x 4; tiles that are not a
  // multiple of the 16 rows a consumer pass covers idle warps)
  g.T = tune.tile ? tune.tile
                  : static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(32, 98304 / row)));
  const size_t stage = g.T * row;
  g.S = tune.stages
            ? tune.stages
            : static_cast<uint32_t>(std::max<size_t>(2, std::min<size_t>(8, 196608 / stage)));
  size_t off = (g.S * stage + 127) & ~size_t(127);
  const size_t merge = epilogue_scratch(kConsumers, kk, grid);
  if (off < merge) off = (merge + 127) & ~size_t(127);
  off += g.S * 16 + g.S * g.T * 12 + g.S * 4 + 16;
  off += row + 16;
  g.smem = off;
  return g;
}

template <bool kFp64, int KPL, int NCH>
void launch_tma_t(const float* Q, uint32_t nq, uint32_t d, int metric, int k, int kk,
                  const FastTable& ft, const float* slab, const uint64_t* ids,
                  const ScanOut& out, int gx, const ScanTune& tune, cudaStream_t st) {
  const TmaGeom g = tma_geom(d, kk, static_cast<uint32_t>(gx), tune);
  if (g.smem > 227 * 1024) throw CudaError("TMA ring does not fit shared memory");
  auto fn = scan_tma_kernel<kFp64, KPL, NCH>;
  ensure_dyn_smem(reinterpret_cast<const void*>(fn), g.smem);
  fn<<<dim3(gx, nq), kTmaThreads, g.smem, st>>>(Q, d, metric, k, kk, ft, slab, ids, out, g.T, g.S);
  after_launch();
}

template <bool kFp64, int KPL, int NCH>
void launch_ldg_t(const float* Q, uint32_t nq, uint32_t d, int metric, int k, int kk,
                  const FastTable& ft, const float* slab, const uint64_t* ids,
                  const ScanOut& out, int gx, cudaStream_t st) {
  const size_t smem = ((size_t(d) * 4 + 15) & ~size_t(15)) +
                      epilogue_scratch(kScanWarps, kk, static_cast<uint32_t>(gx));
  if (smem > 227 * 1024) throw CudaError("LDG scan epilogue does not fit shared memory");
  auto fn = scan_ldg_kernel<kFp64, KPL, NCH>;
  ensure_dyn_smem(reinterpret_cast<const void*>(fn), smem);
  fn<<<dim3(gx, nq), kScanThreads, smem, st>>>(Q, d, metric, k, kk, ft, slab, ids, out);
  after_launch();
}

template <bool kFp64, int NCH>
void dispatch_k(bool tma, const float* Q, uint32_t nq, uint32_t d, int metric, int k, int kk,
                const FastTable& ft, const float* slab, const uint64_t* ids,
                const ScanOut& out, int gx, const ScanTune& tune, cudaStream_t st) {
#define LAIVG_SCAN(KPL)                                                                    \
  do {                                                                                     \
    if (tma) launch_tma_t<kFp64, KPL, NCH>(Q, nq, d, metric, k, kk, ft, slab, ids, out, gx, tune, st); \
    else launch_ldg_t<kFp64, KPL, NCH>(Q, nq, d, metric, k, kk, ft, slab, ids, out, gx, st);     \
  } while (0)
  if (kk <= 32) LAIVG_SCAN(1);
  else if (kk <= 64) LAIVG_SCAN(2);
  else if (kk <= 128) LAIVG_SCAN(4);
  else LAIVG_SCAN(8);
#undef LAIVG_SCAN
}

} // namespace

// ==========================================================================
// launchers
// ==========================================================================
std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> n{0};
  return n;
}

void launch_coarse_scores(const float* Q, uint32_t nq, const float* centroids,
                          uint32_t nc, uint32_t d, int metric, double* scores,
                          cudaStream_t st) {
  const int warps = 8;
  const dim3 block(warps * 32);
  if (nq >= 8) {
    const size_t smem = size_t(8) * d * sizeof(float);
    if (smem > 48 * 1024) {
      ensure_dyn_smem(reinterpret_cast<const void*>(coarse_scores_kernel<8>), smem);
    }
    coarse_scores_kernel<8><<<dim3((nc + warps - 1) / warps, (nq + 7) / 8), block, smem, st>>>(
        Q, nq, centroids, nc, d, metric, scores);
  } else if ((d & 3u) == 0 && d <= 1024) {
    const uint32_t per_cta = warps * kCPW;
    const dim3 grid((nc + per_cta - 1) / per_cta, nq);
    if (d <= 768) coarse_scores_q1_kernel<6><<<grid, block, 0, st>>>(Q, centroids, nc, d, metric, scores);
    else coarse_scores_q1_kernel<8><<<grid, block, 0, st>>>(Q, centroids, nc, d, metric, scores);
  } else {
    const size_t smem = size_t(d) * sizeof(float);
    if (smem > 48 * 1024) {
      ensure_dyn_smem(reinterpret_cast<const void*>(coarse_scores_kernel<1>), smem);
    }
    coarse_scores_kernel<1><<<dim3((nc + warps - 1) / warps, nq), block, smem, st>>>(
        Q, nq, centroids, nc, d, metric, scores);
  }
  after_launch();
}

uint32_t select_runs(uint32_t nc) {
  uint32_t nseg = (nc + kSeg - 1) / kSeg, pad = 1;
  while (pad < nseg) pad <<= 1;
  return pad;
}

size_t select_scratch_entries(uint32_t nq, uint32_t nc) {
  return size_t(nq) * select_runs(nc) * kSeg;
}

void launch_select(const double* scores, uint32_t nq, uint32_t nc, int metric,
                   uint32_t n_out, uint32_t* order, uint64_t* run_k, uint32_t* run_v,
                   const int64_t* res_off, const uint64_t* list_off, const FastTable* ft,
                   cudaStream_t st, bool scan_sorted) {
  const uint32_t nseg_pad = select_runs(nc);
  seg_sort_kernel<<<dim3(nseg_pad, nq), kSeg, 0, st>>>(scores, nc, metric, run_k, run_v,
                                                       nseg_pad);
  after_launch();
  // keep the best P per run when only a prefix is needed
  const bool full = n_out > kSeg;
  uint32_t P = kSeg;
  if (!full) {
    P = 32; // warp-merge granularity; runs hold kSeg >= 32 entries
    while (P < n_out) P <<= 1;
  }
  // prefix mode ping-pongs between two buffers
  const size_t smem = size_t(nseg_pad) * P * (sizeof(uint64_t) + sizeof(uint32_t)) *
                          (full ? 1 : 2) + 16;
  // dynamic + the partition statics may pass 48 KB
  ensure_dyn_smem(reinterpret_cast<const void*>(merge_runs_kernel), smem);
  const FastTable f = ft ? *ft : FastTable{};
  const uint32_t total = nseg_pad * P;
  const uint32_t threads = std::min<uint32_t>(1024, std::max<uint32_t>(256, (total / 2 + 31) & ~31u));
  merge_runs_kernel<<<nq, threads, smem, st>>>(run_k, run_v, nseg_pad, P, full, n_out, order,
                                            res_off, list_off, f, ft != nullptr, scan_sorted);
  after_launch();
}


size_t tc_select_smem(uint32_t nc, uint32_t d) {
  uint32_t cap = 2;
  while (cap < nc) cap <<= 1;
  return ((size_t(d) * 4 + 15) & ~size_t(15)) + 2 * ((size_t(nc) * 4 + 15) & ~size_t(15)) +
         size_t(cap) * 12;
}

void launch_tc_select(const float* approx, uint32_t splits, const float* Q, uint32_t nq,
                      uint32_t d, const float* centroids, const float* cnorm, uint32_t nc, int metric,
                      uint32_t n_out, uint32_t* order, const int64_t* res_off,
                      const uint64_t* list_off, const FastTable* ft, cudaStream_t st,
                      bool scan_sorted, const TcSelectScratch* sc) {
  if (nq == 0 || n_out == 0) return;
  uint32_t cap = 2;
  while (cap < nc) cap <<= 1;
  const FastTable f = ft ? *ft : FastTable{};
  int nsm = 148;
  {
    int dv = 0;
    cudaGetDevice(&dv);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dv);
  }
  const bool half = nq > uint32_t(nsm);
  if (sc != nullptr && sc->cand != nullptr && cap <= 8192 && (d % 4) == 0 && d <= 1024) {
    // filter (per query) -> streamed exact re-score (one CTA per SM) -> sort
    const size_t fs = 2 * ((size_t(nc) * 4 + 15) & ~size_t(15));
    auto ffn = half ? tc_filter_kernel<512> : tc_filter_kernel<kSelThreads>;
    ensure_dyn_smem(reinterpret_cast<const void*>(ffn), fs);
    // per-pair streamed re-score by default; LAIVG_TC_RESCORE=lm selects the
    // list-major re-score (measured: 13.4 vs ~11-23 us at nq 32, 46.8 vs ~54
    // us at nq 256, whole call no faster: profiles/r02/tc_rescore_lm.jsonl)
    const char* lm_env = std::getenv("LAIVG_TC_RESCORE"); // read per call (tests switch it)
    const bool lm_on = lm_env && std::string(lm_env) == "lm";
    const bool lm = lm_on && sc->qmask != nullptr;
    if (lm) {
      if (cudaMemsetAsync(sc->qmask, 0, size_t((nq + 31) / 32) * nc * sizeof(uint32_t), st) !=
          cudaSuccess) {
        throw CudaError("tc_select: qmask reset failed");
      }
    }
    ffn<<<nq, half ? 512 : kSelThreads, fs, st>>>(approx, splits, Q, d, cnorm, nc, metric, n_out,
                                                 cap, sc->cand, sc->ncand,
                                                 lm ? sc->qmask : nullptr);
    after_launch();
    if (lm) {
      const uint32_t nqb = (nq + 31) / 32;
      const uint32_t chunks = std::max<uint32_t>(1, (2u * uint32_t(nsm) + nqb - 1) / nqb);
      const uint32_t chunk = (nc + chunks - 1) / chunks;
      const size_t qs = size_t(32) * d * 4 + size_t(chunk) * 4;
      auto lfn = d <= 768 ? tc_rescore_lm_kernel<6> : tc_rescore_lm_kernel<8>;
      ensure_dyn_smem(reinterpret_cast<const void*>(lfn), qs);
      lfn<<<dim3((nc + chunk - 1) / chunk, nqb), 256, qs, st>>>(Q, d, centroids, metric, nq, nc,
                                                                cap, chunk, sc->qmask, sc->key);
      after_launch();
    } else {
      const size_t rs = 2 * size_t(kRsTile) * d * 4 + 2 * 16 + 2 * kRsTile * 8 + 16 +
                        (size_t(nq) + 1) * 4 + size_t(kRsMaxPairs) * 12 + 64;
      auto rfn = d <= 768 ? tc_rescore_stream_kernel<6> : tc_rescore_stream_kernel<8>;
      ensure_dyn_smem(reinterpret_cast<const void*>(rfn), rs);
      rfn<<<nsm, kRsThreads, rs, st>>>(Q, d, centroids, metric, nq, cap, sc->cand, sc->ncand,
                                        sc->key);
      after_launch();
    }
    const size_t ss = size_t(std::max<uint32_t>(cap, kSortThreads)) * 12 + 16;
    ensure_dyn_smem(reinterpret_cast<const void*>(tc_sort_kernel), ss);
    tc_sort_kernel<<<nq, kSortThreads, ss, st>>>(cap, sc->cand, sc->ncand, sc->key, n_out, order,
                                                 res_off, list_off, f, ft != nullptr, scan_sorted,
                                                 lm);
    after_launch();
    return;
  }
  const size_t smem = tc_select_smem(nc, d);
  if (smem > 227 * 1024) throw CudaError("tc_select: shared memory exceeds 227 KB");
  auto kfn = half ? tc_select_kernel<512> : tc_select_kernel<kSelThreads>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kfn), smem);
  static const bool probe = std::getenv("LAIVG_TC_PROBE") != nullptr;
  kfn<<<nq, half ? 512 : kSelThreads, smem, st>>>(approx, splits, Q, d, centroids, cnorm, nc, metric,
                                           n_out,
                                           cap, order, res_off, list_off, f, ft != nullptr,
                                           scan_sorted, probe);
  after_launch();
  if (probe) {
    unsigned long long t[8];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(t, g_tc_dbg, sizeof(t));
    std::fprintf(stderr,
                 "[laivg tc_select] q0 us: bounds %.2f radix %.2f collect %.2f rescore %.2f "
                 "sort %.2f out+partition %.2f (candidates %llu, nq %u, L %u)\n",
                 (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3,
                 (t[4] - t[3]) * 1e-3, (t[5] - t[4]) * 1e-3, (t[6] - t[5]) * 1e-3, t[7], nq, n_out);
  }
}

void launch_partition(const uint32_t* probe, uint32_t nq, uint32_t lp,
                      const int64_t* res_off, const uint64_t* list_off,
                      FastTable ft, cudaStream_t st) {
  partition_kernel<<<nq, 256, 0, st>>>(probe, lp, res_off, list_off, ft);
  after_launch();
}

int scan_grid_x(uint32_t nq, int num_sms, ScanImpl impl, const ScanTune& tune) {
  const int per_sm = tune.ctas_per_sm ? static_cast<int>(tune.ctas_per_sm)
                                      : (impl == ScanImpl::kTma ? 1 : 2);
  int gx = per_sm * num_sms / static_cast<int>(nq ? nq : 1);
  return gx < 1 ? 1 : gx;
}

int scan_kk(int k, bool acc_fp64) {
  if (acc_fp64) return k;
  return k + kRerankMargin < kMaxK ? k + kRerankMargin : kMaxK;
}

void launch_scan(const float* Q, uint32_t nq, uint32_t d, int metric, int k,
                 const FastTable& ft, const float* slab_vecs,
                 const uint64_t* ids_all, const ScanOut& out, int grid_x,
                 bool acc_fp64, ScanImpl impl, const ScanTune& tune, cudaStream_t st) {
  // fp32 accumulation keeps k + kRerankMargin survivors for the exact
  // re-score; where that margin no longer fits the register top-k, every
  // candidate is accumulated in fp64 instead (no survivor cut to get wrong)
  if (!acc_fp64 && k + kRerankMargin > kMaxK) acc_fp64 = true;
  const int kk = scan_kk(k, acc_fp64);
  const bool tma = impl == ScanImpl::kTma && (d % 4) == 0;
  const bool d768 = d == 768;
#define LAIVG_D(F64, NCH) \
  dispatch_k<F64, NCH>(tma, Q, nq, d, metric, k, kk, ft, slab_vecs, ids_all, out, grid_x, tune, st)
  if (acc_fp64) {
    if (d768) LAIVG_D(true, 6);
    else LAIVG_D(true, 0);
  } else {
    if (d768) LAIVG_D(false, 6);
    else LAIVG_D(false, 0);
  }
#undef LAIVG_D
}

// The two tables fit in the ring region next to the selection scratch.
bool fused_tables_fit(uint32_t nc, uint32_t d, uint32_t L, int kk, uint32_t G,
                      const ScanTune& tune) {
  const TmaGeom g = tma_geom(d, kk, G, tune);
  size_t region = (size_t(g.S) * g.T * d * 4 + 127) & ~size_t(127);
  const size_t merge = epilogue_scratch(kConsumers, kk, G);
  if (region < merge) region = (merge + 127) & ~size_t(127);
  return fused_tables_at(nc, L) + fused_res_bytes(nc) + fused_off_bytes(nc) <= region &&
         !std::getenv("LAIVG_NO_TABLES");
}

size_t fused_query_smem(uint32_t nc, uint32_t d, uint32_t L, int k, bool acc_fp64, uint32_t G,
                        const ScanTune& tune) {
  if (!acc_fp64 && k + kRerankMargin > kMaxK) acc_fp64 = true;
  const int kk = scan_kk(k, acc_fp64);
  if (k > kMaxK || (d % 4) != 0 || d > 1024 || nc == 0) return 0;
  const TmaGeom g = tma_geom(d, kk, G, tune);
  // the selection scratch lives in the ring region (ring or merge scratch)
  size_t region = (size_t(g.S) * g.T * d * 4 + 127) & ~size_t(127);
  const size_t merge = epilogue_scratch(kConsumers, kk, G);
  if (region < merge) region = (merge + 127) & ~size_t(127);
  if (fused_select_bytes(nc, L) > region) return 0;
  const size_t smem = g.smem + fused_tables_bytes(L, G);
  return smem > 227 * 1024 ? 0 : smem;
}

template <bool kFp64, int KPL, int NCH>
void launch_fused_t(const FusedArgs& a, uint32_t G, size_t smem, cudaStream_t st) {
  auto fn = fused_query_kernel<kFp64, KPL, NCH>;
  ensure_dyn_smem(reinterpret_cast<const void*>(fn), smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1; // (measured: no launch-latency cost over a plain launch)
  const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
  if (e != cudaSuccess) {
    throw CudaError(std::string("fused query launch failed: ") + cudaGetErrorString(e));
  }
  after_launch();
}

void launch_fused_query(const FusedQuery& q, const ScanOut& out, bool acc_fp64,
                        const ScanTune& tune, cudaStream_t st) {
  if (!acc_fp64 && q.k + kRerankMargin > kMaxK) acc_fp64 = true;
  const int kk = scan_kk(q.k, acc_fp64);
  const size_t smem = fused_query_smem(q.nc, q.d, q.L, q.k, acc_fp64, q.grid, tune);
  if (smem == 0) throw CudaError("fused query kernel: shape does not fit shared memory");
  const TmaGeom g = tma_geom(q.d, kk, q.grid, tune);
  FusedArgs a;
  a.src = q.src;
  a.slot = q.slot;
  a.dQ = q.dQ;
  a.cen = q.cen;
  a.nc = q.nc;
  a.d = q.d;
  a.L = q.L;
  a.metric = q.metric;
  a.keys = q.keys;
  a.res_off = q.res_off;
  a.list_off = q.list_off;
  a.order_out = q.order_out;
  a.fcount_out = q.fcount_out;
  a.flag_out = q.flag_out;
  a.done_out = q.done_out;
  a.ctl = q.ctl;
  a.stamps = q.stamps;
  a.cta_stamps = q.cta_stamps;
  a.tables = fused_tables_fit(q.nc, q.d, q.L, kk, q.grid, tune) ? 1 : 0;
  a.qdirect = q.qdirect;
  a.slab = q.slab;
  a.ids = q.ids;
  a.out = out;
  a.out.fcount_out = nullptr; // the I/O warp publishes the fast count
  a.out.fcount_in = nullptr;
  a.out.probe = nullptr;
  a.T = g.T;
  a.S = g.S;
  a.k = q.k;
  a.kk = kk;
#define LAIVG_FUSED(F64, NCH)                                   \
  do {                                                          \
    if (kk <= 32) launch_fused_t<F64, 1, NCH>(a, q.grid, smem, st);  \
    else if (kk <= 64) launch_fused_t<F64, 2, NCH>(a, q.grid, smem, st); \
    else if (kk <= 128) launch_fused_t<F64, 4, NCH>(a, q.grid, smem, st); \
    else launch_fused_t<F64, 8, NCH>(a, q.grid, smem, st);       \
  } while (0)
  if (acc_fp64) {
    if (q.d == 768) LAIVG_FUSED(true, 6);
    else LAIVG_FUSED(true, 0);
  } else {
    if (q.d == 768) LAIVG_FUSED(false, 6);
    else LAIVG_FUSED(false, 0);
  }
#undef LAIVG_FUSED
}

void launch_fetch_query(const float* src, const float* const* slot, float* dQ, uint32_t d,
                        cudaStream_t st) {
  fetch_query_kernel<<<1, 256, 0, st>>>(src, slot, dQ, d);
  after_launch();
}

void launch_window(uint64_t ns, int num_sms, cudaStream_t st) {
  window_kernel<<<num_sms, 32, 0, st>>>(ns);
  after_launch();
}

void launch_window_stream(const float* buf, uint64_t bytes, uint64_t ns, uint64_t period_ns,
                          int num_sms, float* sink, unsigned long long* bytes_read,
                          cudaStream_t st) {
  window_stream_kernel<<<num_sms * 2, 512, 0, st>>>(reinterpret_cast<const float4*>(buf),
                                                    bytes / 16, ns, period_ns, sink, bytes_read);
  after_launch();
}

} // namespace laivg
