// dev_common.cuh — device primitives shared by the sm_100a kernels: the
// reference's per-term scoring arithmetic (vectorstore.cpp:93-115), warp
// reductions, streaming loads, and the mbarrier / bulk-copy (TMA) helpers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace laivg {
namespace dev {

constexpr int kIP = 0;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : : "memory");
  return t;
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// --------------------------------------------------------------------------
// scoring terms
// --------------------------------------------------------------------------
__device__ __forceinline__ double term_ip_d(double q, float x, double acc) {
  return __fma_rn(q, static_cast<double>(x), acc); // exact product: == mul+add
}
__device__ __forceinline__ double term_l2_d(double q, float x, double acc) {
  const double t = __dsub_rn(q, static_cast<double>(x));
  return __dadd_rn(acc, __dmul_rn(t, t));
}
__device__ __forceinline__ float term_ip_f(float q, float x, float acc) {
  return __fmaf_rn(q, x, acc);
}
__device__ __forceinline__ float term_l2_f(float q, float x, float acc) {
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

// Accumulates one float4 of a row into acc with the metric's term.
template <bool kFp64>
struct Acc4;
template <>
struct Acc4<true> {
  __device__ __forceinline__ static void run(int metric, const double* q, float4 x,
                                             double& a) {
    if (metric == kIP) {
      a = term_ip_d(q[0], x.x, a);
      a = term_ip_d(q[1], x.y, a);
      a = term_ip_d(q[2], x.z, a);
      a = term_ip_d(q[3], x.w, a);
    } else {
      a = term_l2_d(q[0], x.x, a);
      a = term_l2_d(q[1], x.y, a);
      a = term_l2_d(q[2], x.z, a);
      a = term_l2_d(q[3], x.w, a);
    }
  }
};
template <>
struct Acc4<false> {
  __device__ __forceinline__ static void run(int metric, const float* q, float4 x, float& a) {
    if (metric == kIP) {
      a = term_ip_f(q[0], x.x, a);
      a = term_ip_f(q[1], x.y, a);
      a = term_ip_f(q[2], x.z, a);
      a = term_ip_f(q[3], x.w, a);
    } else {
      a = term_l2_f(q[0], x.x, a);
      a = term_l2_f(q[1], x.y, a);
      a = term_l2_f(q[2], x.z, a);
      a = term_l2_f(q[3], x.w, a);
    }
  }
};

// --------------------------------------------------------------------------
// mbarrier + bulk copy (TMA) primitives
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 policy for data read once (the scanned lists): evict first, so a
// ~1 GB scan does not flush what the next query needs from L2 (centroids,
// tables).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Orderable 64-bit key of an fp64 score: ascending key == best first
// (IP descending, L2 ascending); -0.0 == +0.0 so equal scores tie on id.
__device__ __forceinline__ uint64_t order_key(double s, int metric) {
  s = s + 0.0;
  if (metric == kIP) s = -s;
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

// Exact coarse score of one centroid row for one query (ivf.cpp:276-280), by
// one warp: lane-strided per-term fp64 accumulation then a butterfly sum.
// Every kernel that needs a coarse score uses this sequence, so scores (and
// therefore rankings) agree bit for bit across code paths.
__device__ __forceinline__ double warp_coarse_score(const float* sq, const float* row,
                                                    uint32_t d, int metric, int lane) {
  double acc = 0.0;
  if ((d & 3u) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const float4* q4 = reinterpret_cast<const float4*>(sq);
    for (uint32_t j = lane; j < (d >> 2); j += 32) {
      const float4 qq = q4[j];
      const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
      Acc4<true>::run(metric, qd, __ldg(r4 + j), acc);
    }
  } else {
    for (uint32_t j = lane; j < d; j += 32) {
      const float x = __ldg(row + j);
      acc = metric == kIP ? term_ip_d(sq[j], x, acc) : term_l2_d(sq[j], x, acc);
    }
  }
  return warp_sum(acc);
}

// warp_coarse_score for up to R centroid rows at once (rows cen + c[u] * d):
// every row follows exactly warp_coarse_score's sequence of operations, the
// rows only share the warp's load latency.
template <int R>
__device__ __forceinline__ void warp_coarse_score_n(const float* sq, const float* cen,
                                                    const uint32_t* c, uint32_t nr, uint32_t d,
                                                    int metric, int lane, double (&out)[R]) {
  if ((d & 3u) != 0 || d > 1024) {
    for (uint32_t u = 0; u < R; ++u) {
      out[u] = u < nr ? warp_coarse_score(sq, cen + static_cast<uint64_t>(c[u]) * d, d, metric,
                                          lane)
                      : 0.0;
    }
    return;
  }
  const uint32_t d4 = d >> 2;
  const float4* q4 = reinterpret_cast<const float4*>(sq);
  float4 x[R][8];
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const float4* r4 = reinterpret_cast<const float4*>(cen + static_cast<uint64_t>(
                                                                 c[u < static_cast<int>(nr) ? u : 0]) * d);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t j = lane + 32u * t;
      x[u][t] = (u < static_cast<int>(nr) && j < d4) ? __ldg(r4 + j)
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  double acc[R];
#pragma unroll
  for (int u = 0; u < R; ++u) acc[u] = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const uint32_t j = lane + 32u * t;
    if (j < d4) {
      const float4 qq = q4[j];
      const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
      for (int u = 0; u < R; ++u) Acc4<true>::run(metric, qd, x[u][t], acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < R; ++u) out[u] = warp_sum(acc[u]);
}

} // namespace dev
} // namespace laivg
