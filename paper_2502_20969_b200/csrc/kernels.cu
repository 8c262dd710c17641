// kernels.cu — sm_100a kernels of the lookahead IVF retrieval path.
//
//   coarse_scores_kernel : query x centroid scores in fp64 (ivf.cpp:269-281)
//   select_kernel        : full on-chip ranking, ascending cluster id on ties
//                          (ivf.cpp:282-299)
//   partition_kernel     : probe split by device-cache residency
//                          (tiered.cpp:155-161), exclusive prefix of lengths
//   scan_kernel          : IVF-Flat list scan over the resident probed lists,
//                          per-warp register top-k, CTA merge, last-CTA grid
//                          merge (ivf.cpp:301-343, tiered.cpp:172-185)
//   window_kernel        : %globaltimer spin standing in for LLM generation
//
// Reference semantics kept on device: per-term arithmetic of dot_d / l2_sq_d
// (vectorstore.cpp:93-108; products are exact in fp64, so DFMA == mul+add for
// IP; L2 uses separately rounded sub/mul/add), fp32 rounding of the final
// score, sqrt for L2, and the (score, ascending id) total order with
// -0.0 == +0.0 (vectorstore.hpp:34-39). Only the summation order differs
// (parallel tree instead of a serial chain).
#include <cfloat>
#include <cstdint>
#include <cstdio>

#include "kernels.cuh"

namespace laivg {
namespace {

constexpr int kIP = 0;
constexpr unsigned kFull = 0xffffffffu;

// --------------------------------------------------------------------------
// scoring terms
// --------------------------------------------------------------------------
template <typename ACC>
__device__ __forceinline__ ACC term_ip(float q, float x, ACC acc);
template <>
__device__ __forceinline__ double term_ip<double>(float q, float x, double acc) {
  return __fma_rn(static_cast<double>(q), static_cast<double>(x), acc);
}
template <>
__device__ __forceinline__ float term_ip<float>(float q, float x, float acc) {
  return __fmaf_rn(q, x, acc);
}
template <typename ACC>
__device__ __forceinline__ ACC term_l2(float q, float x, ACC acc);
template <>
__device__ __forceinline__ double term_l2<double>(float q, float x, double acc) {
  const double t = __dsub_rn(static_cast<double>(q), static_cast<double>(x));
  return __dadd_rn(acc, __dmul_rn(t, t));
}
template <>
__device__ __forceinline__ float term_l2<float>(float q, float x, float acc) {
  const float t = q - x;
  return __fmaf_rn(t, t, acc);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <typename ACC>
__device__ __forceinline__ float finish_score(int metric, ACC acc) {
  if (metric == kIP) return static_cast<float>(acc);
  return static_cast<float>(sqrt(static_cast<double>(acc)));
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// --------------------------------------------------------------------------
// total order (vectorstore.hpp:34-39)
// --------------------------------------------------------------------------
__device__ __forceinline__ bool ranks_before(int metric, float sa, uint64_t ia,
                                             float sb, uint64_t ib) {
  if (sa != sb) return metric == kIP ? sa > sb : sa < sb;
  return ia < ib;
}
__device__ __forceinline__ float sentinel_score(int metric) {
  return metric == kIP ? -INFINITY : INFINITY;
}

// Warp-resident sorted top-k: entry j = i * 32 + lane lives in slot i of that
// lane. Entries j >= k are scratch.
template <int KPL>
struct WarpTopK {
  float s[KPL];
  uint64_t id[KPL];
  float worst_s;
  uint64_t worst_id;

  __device__ void init(int metric) {
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      s[i] = sentinel_score(metric);
      id[i] = ~0ull;
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
  __device__ __forceinline__ bool enters(int metric, float cs,
                                         uint64_t cid) const {
    return ranks_before(metric, cs, cid, worst_s, worst_id);
  }

  // Warp-uniform insertion of a candidate known to enter.
  __device__ void insert(int metric, int k, float cs, uint64_t cid) {
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
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      float us = __shfl_up_sync(kFull, s[i], 1);
      uint64_t uid = __shfl_up_sync(kFull, id[i], 1);
      if (i > 0) {
        const float ts = __shfl_sync(kFull, s[i - 1], 31);
        const uint64_t tid = __shfl_sync(kFull, id[i - 1], 31);
        if (lane == 0) {
          us = ts;
          uid = tid;
        }
      }
      ps[i] = us;
      pid[i] = uid;
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      if (j > pos) {
        s[i] = ps[i];
        id[i] = pid[i];
      } else if (j == pos) {
        s[i] = cs;
        id[i] = cid;
      }
    }
    refresh_worst(k);
  }

  // Merge a best-first list of n entries (sentinels allowed) from memory.
  // Stops at the first entry that cannot enter (the list is sorted).
  template <bool kCG>
  __device__ void merge_list(int metric, int k, const float* ls,
                             const uint64_t* lid, int n) {
    for (int e = 0; e < n; ++e) {
      const float cs = kCG ? __ldcg(ls + e) : ls[e];
      if (!may_enter(metric, cs)) break;
      const uint64_t cid = kCG ? __ldcg(reinterpret_cast<const unsigned long long*>(lid) + e)
                               : lid[e];
      if (!enters(metric, cs, cid)) break;
      insert(metric, k, cs, cid);
    }
  }

  __device__ void store(int k, float* ls, uint64_t* lid) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      if (j < k) {
        ls[j] = s[i];
        lid[j] = id[i];
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
  if ((d & 3u) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (uint32_t j = lane; j < d / 4; j += 32) {
      const float4 x = __ldg(r4 + j);
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        if (t < nqt) {
          const float4 qq = reinterpret_cast<const float4*>(sq + t * d)[j];
          if (metric == kIP) {
            acc[t] = term_ip<double>(qq.x, x.x, acc[t]);
            acc[t] = term_ip<double>(qq.y, x.y, acc[t]);
            acc[t] = term_ip<double>(qq.z, x.z, acc[t]);
            acc[t] = term_ip<double>(qq.w, x.w, acc[t]);
          } else {
            acc[t] = term_l2<double>(qq.x, x.x, acc[t]);
            acc[t] = term_l2<double>(qq.y, x.y, acc[t]);
            acc[t] = term_l2<double>(qq.z, x.z, acc[t]);
            acc[t] = term_l2<double>(qq.w, x.w, acc[t]);
          }
        }
      }
    }
  } else {
    for (uint32_t j = lane; j < d; j += 32) {
      const float x = __ldg(row + j);
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        if (t < nqt) {
          acc[t] = metric == kIP ? term_ip<double>(sq[t * d + j], x, acc[t])
                                 : term_l2<double>(sq[t * d + j], x, acc[t]);
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

// --------------------------------------------------------------------------
// selection: bitonic sort of (orderable key, cluster id) in shared memory
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t order_key(double s, int metric) {
  s = s + 0.0;                      // -0.0 -> +0.0: equal scores tie on id
  if (metric == kIP) s = -s;        // descending -> ascending
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

__global__ void __launch_bounds__(1024)
    select_kernel(const double* __restrict__ scores, uint32_t nc, int metric,
                  uint32_t p2, uint32_t n_out, uint32_t* __restrict__ order) {
  extern __shared__ uint64_t skey[];
  uint32_t* sid = reinterpret_cast<uint32_t*>(skey + p2);
  const uint32_t q = blockIdx.x;
  const double* sc = scores + static_cast<uint64_t>(q) * nc;
  for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
    if (i < nc) {
      skey[i] = order_key(sc[i], metric);
      sid[i] = i;
    } else {
      skey[i] = ~0ull;
      sid[i] = ~0u;
    }
  }
  __syncthreads();
  for (uint32_t kk = 2; kk <= p2; kk <<= 1) {
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint64_t ka = skey[i], kb = skey[l];
          const uint32_t ia = sid[i], ib = sid[l];
          const bool a_gt_b = ka > kb || (ka == kb && ia > ib);
          const bool up = (i & kk) == 0;
          if (up == a_gt_b) {
            skey[i] = kb;
            skey[l] = ka;
            sid[i] = ib;
            sid[l] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  uint32_t* out = order + static_cast<uint64_t>(q) * n_out;
  for (uint32_t i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = sid[i];
}

// --------------------------------------------------------------------------
// partition by residency (tiered.cpp:155-161) + exclusive prefix of lengths
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    partition_kernel(const uint32_t* __restrict__ probe, uint32_t lp,
                     const int64_t* __restrict__ res_off,
                     const uint64_t* __restrict__ list_off, FastTable ft) {
  __shared__ uint32_t w_cnt[8];
  __shared__ uint64_t w_len[8];
  __shared__ uint32_t base_cnt;
  __shared__ uint64_t base_len;
  const uint32_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tb = static_cast<uint64_t>(q) * ft.stride;
  if (threadIdx.x == 0) {
    base_cnt = 0;
    base_len = 0;
  }
  __syncthreads();
  for (uint32_t t0 = 0; t0 < lp; t0 += 256) {
    const uint32_t i = t0 + threadIdx.x;
    uint32_t c = 0;
    int64_t so = -1;
    if (i < lp) {
      c = probe[static_cast<uint64_t>(q) * lp + i];
      so = res_off[c];
    }
    const bool fast = so >= 0;
    const uint64_t len = fast ? list_off[c + 1] - list_off[c] : 0;
    // warp inclusive scans
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
    const uint32_t ex_c = pc + ic - (fast ? 1u : 0u);
    const uint64_t ex_l = pl + il - len;
    if (fast) {
      ft.slab[tb + ex_c] = so;
      ft.row[tb + ex_c] = list_off[c];
      ft.len[tb + ex_c] = static_cast<uint32_t>(len);
      ft.cluster[tb + ex_c] = c;
      ft.pre[static_cast<uint64_t>(q) * (ft.stride + 1) + ex_c] = ex_l;
    }
    __syncthreads();
    if (threadIdx.x == 255) {
      base_cnt = pc + ic;
      base_len = pl + il;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ft.count[q] = base_cnt;
    ft.pre[static_cast<uint64_t>(q) * (ft.stride + 1) + base_cnt] = base_len;
  }
}

// --------------------------------------------------------------------------
// list scan
// --------------------------------------------------------------------------
constexpr int kScanWarps = 8;
constexpr int kScanThreads = kScanWarps * 32;
constexpr int kU = 2; // vectors in flight per warp iteration

// Cursor over a query's flattened fast-list vector space.
struct Cursor {
  uint32_t li;
  uint32_t len;
  uint64_t o;
  int64_t slab;
  uint64_t row;
};

template <typename ACC, int KPL, int NCH>
__global__ void __launch_bounds__(kScanThreads, 2)
    scan_kernel(const float* __restrict__ Q, uint32_t d, int metric, int k,
                FastTable ft, const float* __restrict__ slab_vecs,
                const uint64_t* __restrict__ ids_all, ScanOut out) {
  extern __shared__ unsigned char smem_raw[];
  float* sq = reinterpret_cast<float*>(smem_raw);                  // d floats
  float* ms = sq + ((d + 3) & ~3u);                                // [W][k]
  uint64_t* mid = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(ms + kScanWarps * k) + 7) & ~uintptr_t(7)); // [W][k]
  __shared__ bool am_last;

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
  top.init(metric);

  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * kScanWarps;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kScanWarps + warp;
  const uint64_t v0 = V * gw / tw, v1 = V * (gw + 1) / tw;

  // q slice in registers for the fixed-D fast path
  float4 qr[NCH > 0 ? NCH : 1];
  if constexpr (NCH > 0) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      qr[c] = reinterpret_cast<const float4*>(sq)[c * 32 + lane];
    }
  }

  if (v0 < v1) {
    // locate the list holding v0: last li with pre[li] <= v0
    uint32_t lo = 0, hi = nf - 1;
    while (lo < hi) {
      const uint32_t mid_ = (lo + hi + 1) >> 1;
      if (pre[mid_] <= v0) lo = mid_;
      else hi = mid_ - 1;
    }
    Cursor cur;
    cur.li = lo;
    cur.len = ft.len[tb + lo];
    cur.o = v0 - pre[lo];
    cur.slab = ft.slab[tb + lo];
    cur.row = ft.row[tb + lo];
    while (cur.o >= cur.len) { // skip empty lists
      ++cur.li;
      cur.len = ft.len[tb + cur.li];
      cur.o = 0;
      cur.slab = ft.slab[tb + cur.li];
      cur.row = ft.row[tb + cur.li];
    }

    for (uint64_t v = v0; v < v1; v += kU) {
      int64_t vec[kU];
      uint64_t rowi[kU];
      bool valid[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        valid[u] = v + u < v1;
        vec[u] = cur.slab + static_cast<int64_t>(cur.o);
        rowi[u] = cur.row + cur.o;
        if (valid[u] && v + u + 1 < v1) {
          ++cur.o;
          while (cur.o >= cur.len) {
            ++cur.li;
            cur.len = ft.len[tb + cur.li];
            cur.o = 0;
            cur.slab = ft.slab[tb + cur.li];
            cur.row = ft.row[tb + cur.li];
          }
        }
      }
      ACC acc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) acc[u] = ACC(0);
      if constexpr (NCH > 0) {
        float4 x[kU][NCH];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const float4* p = reinterpret_cast<const float4*>(
                                slab_vecs + static_cast<uint64_t>(vec[u]) * (NCH * 128)) +
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
            if (metric == kIP) {
              acc[u] = term_ip<ACC>(qr[c].x, x[u][c].x, acc[u]);
              acc[u] = term_ip<ACC>(qr[c].y, x[u][c].y, acc[u]);
              acc[u] = term_ip<ACC>(qr[c].z, x[u][c].z, acc[u]);
              acc[u] = term_ip<ACC>(qr[c].w, x[u][c].w, acc[u]);
            } else {
              acc[u] = term_l2<ACC>(qr[c].x, x[u][c].x, acc[u]);
              acc[u] = term_l2<ACC>(qr[c].y, x[u][c].y, acc[u]);
              acc[u] = term_l2<ACC>(qr[c].z, x[u][c].z, acc[u]);
              acc[u] = term_l2<ACC>(qr[c].w, x[u][c].w, acc[u]);
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
            acc[u] = metric == kIP ? term_ip<ACC>(sq[j], xv, acc[u])
                                   : term_l2<ACC>(sq[j], xv, acc[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const ACC tot = warp_sum(acc[u]);
        if (!valid[u]) continue;
        const float cs = finish_score<ACC>(metric, tot);
        if (top.may_enter(metric, cs)) {
          const uint64_t cid = ids_all[rowi[u]];
          if (top.enters(metric, cs, cid)) top.insert(metric, k, cs, cid);
        }
      }
    }
  }

  // ---- CTA merge: warps -> smem -> warp 0 ----
  top.store(k, ms + warp * k, mid + warp * k);
  __syncthreads();
  const uint64_t part = (static_cast<uint64_t>(q) * gridDim.x + blockIdx.x) * k;
  if (warp == 0) {
    for (int w = 1; w < kScanWarps; ++w) {
      top.template merge_list<false>(metric, k, ms + w * k, mid + w * k, k);
    }
    top.store(k, out.part_s + part, out.part_id + part);
    __threadfence();
    if (lane == 0) {
      const unsigned t = atomicAdd(out.ticket + q, 1u);
      am_last = (t == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!am_last) return;

  // ---- grid merge in the last CTA ----
  __threadfence();
  top.init(metric);
  const uint64_t pbase = static_cast<uint64_t>(q) * gridDim.x * k;
  for (uint32_t g = warp; g < gridDim.x; g += kScanWarps) {
    top.template merge_list<true>(metric, k, out.part_s + pbase + g * k,
                                  out.part_id + pbase + g * k, k);
  }
  top.store(k, ms + warp * k, mid + warp * k);
  __syncthreads();
  if (warp == 0) {
    for (int w = 1; w < kScanWarps; ++w) {
      top.template merge_list<false>(metric, k, ms + w * k, mid + w * k, k);
    }
    top.store(k, out.out_s + static_cast<uint64_t>(q) * k,
              out.out_id + static_cast<uint64_t>(q) * k);
    if (lane == 0) {
      out.out_count[q] = static_cast<uint32_t>(V < static_cast<uint64_t>(k) ? V : k);
      out.ticket[q] = 0; // self-reset for the next launch / graph replay
    }
  }
}

// --------------------------------------------------------------------------
// generation window
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void window_kernel(uint64_t ns) {
  const uint64_t t0 = globaltimer();
  while (globaltimer() - t0 < ns) {
    __nanosleep(2000);
  }
}

template <typename ACC, int KPL, int NCH>
void launch_scan_t(const float* Q, uint32_t nq, uint32_t d, int metric, int k,
                   const FastTable& ft, const float* slab, const uint64_t* ids,
                   const ScanOut& out, int gx, cudaStream_t st) {
  const size_t smem = ((d + 3) & ~3u) * sizeof(float) +
                      kScanWarps * k * (sizeof(float) + sizeof(uint64_t)) + 16;
  auto fn = scan_kernel<ACC, KPL, NCH>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr_set = true;
  }
  fn<<<dim3(gx, nq), kScanThreads, smem, st>>>(Q, d, metric, k, ft, slab, ids, out);
  launch_counter()++;
}

template <typename ACC, int NCH>
void launch_scan_k(const float* Q, uint32_t nq, uint32_t d, int metric, int k,
                   const FastTable& ft, const float* slab, const uint64_t* ids,
                   const ScanOut& out, int gx, cudaStream_t st) {
  if (k <= 32) launch_scan_t<ACC, 1, NCH>(Q, nq, d, metric, k, ft, slab, ids, out, gx, st);
  else if (k <= 64) launch_scan_t<ACC, 2, NCH>(Q, nq, d, metric, k, ft, slab, ids, out, gx, st);
  else if (k <= 128) launch_scan_t<ACC, 4, NCH>(Q, nq, d, metric, k, ft, slab, ids, out, gx, st);
  else launch_scan_t<ACC, 8, NCH>(Q, nq, d, metric, k, ft, slab, ids, out, gx, st);
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
      cudaFuncSetAttribute(coarse_scores_kernel<8>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
    coarse_scores_kernel<8><<<dim3((nc + warps - 1) / warps, (nq + 7) / 8), block, smem, st>>>(
        Q, nq, centroids, nc, d, metric, scores);
    launch_counter()++;
  } else {
    const size_t smem = size_t(d) * sizeof(float);
    if (smem > 48 * 1024) {
      cudaFuncSetAttribute(coarse_scores_kernel<1>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
    coarse_scores_kernel<1><<<dim3((nc + warps - 1) / warps, nq), block, smem, st>>>(
        Q, nq, centroids, nc, d, metric, scores);
    launch_counter()++;
  }
}

void launch_select(const double* scores, uint32_t nq, uint32_t nc, int metric,
                   uint32_t n_out, uint32_t* order, cudaStream_t st) {
  uint32_t p2 = 1;
  while (p2 < nc) p2 <<= 1;
  const size_t smem = size_t(p2) * (sizeof(uint64_t) + sizeof(uint32_t));
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    attr = smem;
  }
  const int threads = p2 >= 2048 ? 1024 : (p2 >= 64 ? int(p2 / 2) : 32);
  select_kernel<<<nq, threads, smem, st>>>(scores, nc, metric, p2, n_out, order);
  launch_counter()++;
}

void launch_partition(const uint32_t* probe, uint32_t nq, uint32_t lp,
                      const int64_t* res_off, const uint64_t* list_off,
                      FastTable ft, cudaStream_t st) {
  partition_kernel<<<nq, 256, 0, st>>>(probe, lp, res_off, list_off, ft);
  launch_counter()++;
}

int scan_grid_x(uint32_t nq, int num_sms) {
  const int ctas = 2 * num_sms; // 2 CTAs of 8 warps per SM
  int gx = ctas / static_cast<int>(nq ? nq : 1);
  return gx < 1 ? 1 : gx;
}

void launch_scan(const float* Q, uint32_t nq, uint32_t d, int metric, int k,
                 const FastTable& ft, const float* slab_vecs,
                 const uint64_t* ids_all, const ScanOut& out, int grid_x,
                 bool acc_fp64, cudaStream_t st) {
  const bool d768 = d == 768;
  if (acc_fp64) {
    if (d768) launch_scan_k<double, 6>(Q, nq, d, metric, k, ft, slab_vecs, ids_all, out, grid_x, st);
    else launch_scan_k<double, 0>(Q, nq, d, metric, k, ft, slab_vecs, ids_all, out, grid_x, st);
  } else {
    if (d768) launch_scan_k<float, 6>(Q, nq, d, metric, k, ft, slab_vecs, ids_all, out, grid_x, st);
    else launch_scan_k<float, 0>(Q, nq, d, metric, k, ft, slab_vecs, ids_all, out, grid_x, st);
  }
}

void launch_window(uint64_t ns, int num_sms, cudaStream_t st) {
  window_kernel<<<num_sms, 32, 0, st>>>(ns);
  launch_counter()++;
}

} // namespace laivg
