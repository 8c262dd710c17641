// listscan.cu — list-major batched scan on the 5th-generation tensor cores.
//
// search_clusters (ivf.cpp:301-343) scores every member of every probed list
// against one query. In a batch, a list probed by several queries is one
// (list rows x queries) GEMM; the per-query scan streams it once per query.
// This path reads each resident list once per 16 queries that probe it:
//
//   plan      ls_count -> ls_plan -> ls_fill: per resident list, the batch
//             queries that probe it (CSR), and work items
//             (list, 1024-row chunk, group of <= 16 queries), groups fastest
//             so the groups of one chunk run together and share it in L2.
//   scan      list_scan_tc_kernel, one persistent CTA per SM pulling items:
//               warp 0      TMA producer: 128-row x 32-float tiles of the list
//                           (cp.async.bulk.tensor.2d over the slab, 128-byte
//                           swizzle) into a 6-stage ring,
//               warp 1      MMA issuer: tcgen05.mma kind::tf32, A = list rows
//                           (M 128), B = the item's queries (N 16, staged once
//                           per item), accumulator double-buffered in TMEM,
//               warps 8-11  ||v||^2 of each row from the same ring stages,
//               warps 4-7   epilogue: tcgen05.ld of the tf32 scores, error
//                           bounds [lo, hi] of the exact score, and a
//                           per-query candidate buffer filtered by the
//                           running threshold tau = k-th best lo (compacted
//                           with a warp radix select).
//             Candidates (hi >= tau) go to a per-query global array; tau is
//             shared across the items of a query (atomicMax), and seeds
//             every later item.
//   final     ls_final_kernel, one CTA per query: tau over all its
//             candidates, exact fp64 re-score of the survivors with the
//             reference's arithmetic (vectorstore.cpp:93-115) and the exact
//             (score, id) top-k (vectorstore.hpp:34-39).
//
// Exactness: |tf32 score - exact| <= kTcErr ||q|| ||v|| (the coarse_tc
// bound), so lo <= exact <= hi; k vectors with lo >= tau exist, hence every
// member of the exact top-k (ties on id included) has hi >= tau and is
// re-scored. The result equals the per-query scan's. A candidate buffer that
// overflows sets a flag and the caller re-runs the batch on the per-query
// scan (never a partial answer).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "dev_common.cuh"
#include "host.hpp"
#include "kernels.cuh"
#include "umma.cuh"

namespace laivg {
CUtensorMap make_row_tile_map(const float* base, uint64_t rows, uint32_t d, uint32_t box_rows);

using namespace dev;
namespace {

constexpr uint32_t kLsNQMax = 32;    // queries per item (UMMA N): 16, or 32 for shared lists
constexpr uint32_t kLsM = 128;       // list rows per row-block (UMMA M)
constexpr uint32_t kLsKB = 32;       // floats per k-block (one 128-byte swizzle row)
__host__ __device__ constexpr uint32_t ls_stages(uint32_t nq) { return nq <= 16 ? 8u : 4u; } // ring (16 KB)
constexpr uint32_t kLsStage = kLsM * kLsKB * 4;
constexpr uint32_t kLsChunk = 1024;  // list rows per item unless the caller sets ListScan::chunk
constexpr uint32_t kLsSlots = 16;    // candidate slots per lane of a compacting warp
constexpr uint32_t kLsMaxCap = 32 * kLsSlots; // candidate slots per query per item (<=)
constexpr uint32_t kLsMaxK = 64;
constexpr uint32_t kLsThreads = 384;
constexpr uint32_t kLsSurv = 2048;   // survivors re-scored per query
constexpr uint32_t kLsFinalThreads = 256;

// Orderable key of a float: ascending with the value.
__device__ __forceinline__ uint32_t ls_key(float f) {
  const uint32_t b = __float_as_uint(f + 0.0f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct LsArgs {
  const float* Q;
  uint32_t d;
  int metric;
  int k;
  const int64_t* res;
  const uint64_t* list_off;
  const uint32_t* lists;
  const uint32_t* lq_off;
  const uint32_t* item_off;
  const uint32_t* qidx;
  uint32_t* meta;      // [0] lists [1] items [2] work counter [3] overflow
  uint32_t* gtau;      // [nq] shared threshold key per query
  uint32_t* gcnt;      // [nq]
  uint4* cand;         // [nq][gcap] (lo key, hi key, cluster, slab row)
  uint32_t gcap;
  uint32_t cap;        // candidate slots per query per item (<= kLsMaxCap)
  uint32_t chunk;      // list rows per item (multiple of 128, <= 65536: u16 row index)
  unsigned* flag_host; // overflow, mapped host memory
};

__device__ __forceinline__ void ls_overflow(const LsArgs& a) {
  atomicExch(a.meta + 3, 1u);
  *reinterpret_cast<volatile unsigned*>(a.flag_host) = 1u;
}

// k-th largest key among the warp's held keys (kLsSlots per lane), exact,
// by a most-significant-bit-first radix walk with ballots.
__device__ __forceinline__ uint32_t warp_kth_largest(const uint32_t (&key)[kLsSlots],
                                                     const bool (&ok)[kLsSlots], uint32_t k) {
  uint32_t prefix = 0, need = k;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t want = prefix | (1u << bit);
    const uint32_t mask = ~((1u << bit) - 1u);
    uint32_t cnt = 0;
#pragma unroll
    for (int t = 0; t < int(kLsSlots); ++t) {
      cnt += __popc(__ballot_sync(kFull, ok[t] && (key[t] & mask) == want));
    }
    if (cnt >= need) prefix = want;
    else need -= cnt;
  }
  return prefix;
}

// One warp: raise query j's threshold to the k-th best lower bound of its
// buffer (when it holds >= k) and keep the entries with hi >= tau.
__device__ void ls_compact(uint32_t* lo, uint32_t* hi, uint16_t* rw, uint32_t* cnt, uint32_t* tau,
                           uint32_t k, uint32_t cap, int lane) {
  const uint32_t m = min(*cnt, cap);
  uint32_t L[kLsSlots], H[kLsSlots];
  uint16_t R[kLsSlots];
  bool ok[kLsSlots];
#pragma unroll
  for (int t = 0; t < int(kLsSlots); ++t) {
    const uint32_t i = lane + 32u * t;
    ok[t] = i < m;
    L[t] = ok[t] ? lo[i] : 0u;
    H[t] = ok[t] ? hi[i] : 0u;
    R[t] = ok[t] ? rw[i] : 0;
  }
  uint32_t th = *tau;
  if (m >= k) th = max(th, warp_kth_largest(L, ok, k));
  __syncwarp();
  uint32_t n = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int t = 0; t < int(kLsSlots); ++t) {
    const bool keep = ok[t] && H[t] >= th;
    const uint32_t b = __ballot_sync(kFull, keep);
    if (keep) {
      const uint32_t p = n + __popc(b & lt);
      lo[p] = L[t];
      hi[p] = H[t];
      rw[p] = R[t];
    }
    n += __popc(b);
  }
  __syncwarp();
  if (lane == 0) {
    *cnt = n;
    *tau = th;
  }
  __syncwarp();
}

// Claims the next work item and decodes it into item[] (valid, cluster, r0,
// r1, query-slot base, queries) and *s0 (slab row of the item's first row).
__device__ void ls_claim(const LsArgs& a, uint32_t kNQ, uint32_t* item, long long* s0) {
  const uint32_t t = atomicAdd(a.meta + 2, 1u);
  const uint32_t total = a.meta[1], nl = a.meta[0];
  if (t >= total || *reinterpret_cast<volatile uint32_t*>(a.meta + 3)) {
    item[0] = 0;
    return;
  }
  uint32_t lo = 0, hi = nl - 1; // largest u with item_off[u] <= t
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (a.item_off[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const uint32_t u = lo, c = a.lists[u];
  const uint32_t qc = a.lq_off[u + 1] - a.lq_off[u];
  const uint32_t groups = (qc + kNQ - 1) / kNQ;
  const uint32_t local = t - a.item_off[u];
  const uint32_t chunk = local / groups, g = local - chunk * groups;
  const uint64_t len = a.list_off[c + 1] - a.list_off[c];
  const uint32_t r0 = chunk * a.chunk;
  item[0] = 1;
  item[1] = c;
  item[2] = r0;
  item[3] = static_cast<uint32_t>(len < uint64_t(r0) + a.chunk ? len : uint64_t(r0) + a.chunk);
  item[4] = a.lq_off[u] + g * kNQ;
  item[5] = min(kNQ, qc - g * kNQ);
  *s0 = a.res[c] + r0;
}

template <uint32_t kLsNQ>
__global__ void __launch_bounds__(kLsThreads, 1)
    list_scan_tc_kernel(const __grid_constant__ CUtensorMap slab_map,
                        const __grid_constant__ CUtensorMap tail_map, LsArgs a) {
  constexpr uint32_t kLsStages = ls_stages(kLsNQ);
  constexpr uint32_t kTmemCols = 2 * kLsNQ; // double-buffered accumulator (power of 2 >= 32)
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kLsStages], empty[kLsStages], acc_full[2], acc_empty[2],
      norm_full[2];
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t s_item[2][8]; // current / next: valid, c, r0, r1, qbase, nqg
  __shared__ long long s_s0[2];     // slab row of the item's first row
  __shared__ uint32_t s_q[kLsNQ], s_tau[kLsNQ], s_cnt[kLsNQ];
  __shared__ float s_qn[kLsNQ];
  __shared__ double s_qn2[kLsNQ];
  __shared__ float s_vn2[2][kLsM];

  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t d = a.d;
  const uint32_t nkb = (d + kLsKB - 1) / kLsKB;
  unsigned char* ring = smem;
  unsigned char* qB = ring + kLsStages * kLsStage;            // nkb x (NQ rows x 128 B)
  uint32_t* c_lo = reinterpret_cast<uint32_t*>(qB + nkb * kLsNQ * 128);
  const uint32_t cap = a.cap, trig = cap - kLsM; // a row-block always fits above trig
  uint32_t* c_hi = c_lo + kLsNQ * cap;
  uint16_t* c_rw = reinterpret_cast<uint16_t*>(c_hi + kLsNQ * cap);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kLsStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1 + 4); // MMA commit + the four norm warps
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 4);
      mbar_init(norm_full + b, 4);
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&slab_map))
                 : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tail_map))
                 : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // role-private running counters (the ring and TMEM phases run across items)
  uint32_t it = 0, ab = 0;

  // The producer claims the next item once it has issued the current one's
  // loads; it starts loading while warps 1-11 stage the item's queries.
  uint32_t cur = 0;
  if (threadIdx.x == 0) ls_claim(a, kLsNQ, s_item[0], &s_s0[0]);
  __syncthreads();
  for (;;) {
    if (!s_item[cur][0]) break;
    const uint32_t c = s_item[cur][1], r0 = s_item[cur][2], r1 = s_item[cur][3];
    const uint32_t nqg = s_item[cur][5];
    const long long s0 = s_s0[cur];
    const uint32_t nrb = (r1 - r0 + kLsM - 1) / kLsM;

    // ---- stage the item's queries (B operand, K-major, 128-byte swizzle) ----
    if (warp > 0) {
      constexpr uint32_t kStg = kLsThreads - 32;
      const uint32_t st = threadIdx.x - 32;
      if (st < kLsNQ) {
        s_q[st] = st < nqg ? a.qidx[s_item[cur][4] + st] : 0u;
        s_cnt[st] = 0;
      }
      named_sync(2, kStg);
      const uint32_t per_q = nkb * 8; // float4 chunks per query row
      for (uint32_t x = st; x < kLsNQ * per_q; x += kStg) {
        const uint32_t j = x / per_q, r = x - j * per_q, kb = r >> 3, ch = r & 7;
        const uint32_t f = kb * kLsKB + ch * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < nqg && f < d) {
          v = __ldg(reinterpret_cast<const float4*>(a.Q + uint64_t(s_q[j]) * d + f));
        }
        *reinterpret_cast<float4*>(qB + kb * (kLsNQ * 128) + j * 128 + ((ch ^ (j & 7)) << 4)) = v;
      }
      for (uint32_t j = warp - 1; j < nqg; j += kStg / 32) {
        const float* q = a.Q + uint64_t(s_q[j]) * d;
        double sq = 0.0;
        for (uint32_t i = lane; i < d; i += 32) {
          const double x = q[i];
          sq = fma(x, x, sq);
        }
        sq = warp_sum(sq);
        if (lane == 0) {
          s_qn2[j] = sq;
          s_qn[j] = __double2float_ru(sqrt(sq) * (1.0 + 1e-6));
          s_tau[j] = a.gtau[s_q[j]];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_sync(2, kStg);
    }

    if (warp == 0) {
      if (lane == 0) { // ---- TMA producer ----
        for (uint32_t rb = 0; rb < nrb; ++rb) {
          // a list's last row-block, when at most half full, loads only its
          // valid rows in 16-row boxes (same swizzled layout as the first rows
          // of a full tile; the stale rows past them are masked by the
          // epilogue): c2b lists end in a 10-row block, 1.048x -> 1.004x DRAM
          const uint32_t valid = min(kLsM, r1 - (r0 + rb * kLsM));
          const uint32_t nbox = valid > kLsM / 2 ? 0u : (valid + 15) / 16;
          for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
            const uint32_t s = it % kLsStages, u = it / kLsStages;
            if (u > 0) mbar_wait(empty + s, (u - 1) & 1u);
            unsigned char* dst = ring + s * kLsStage;
            const int32_t x = static_cast<int32_t>(kb * kLsKB);
            const int32_t y = static_cast<int32_t>(s0 + rb * kLsM);
            if (nbox == 0) {
              mbar_arrive_expect_tx(full + s, kLsStage);
              tma_load_2d(dst, &slab_map, x, y, full + s);
            } else {
              mbar_arrive_expect_tx(full + s, nbox * 16 * kLsKB * 4);
              for (uint32_t i = 0; i < nbox; ++i) {
                tma_load_2d(dst + i * 16 * kLsKB * 4, &tail_map, x,
                            y + static_cast<int32_t>(16 * i), full + s);
              }
            }
          }
        }
        ls_claim(a, kLsNQ, s_item[cur ^ 1u], &s_s0[cur ^ 1u]);
      }
      __syncwarp();
    } else if (warp == 1) {
      if (lane == 0) { // ---- MMA issuer ----
        constexpr uint32_t idesc = tf32_idesc(kLsM, kLsNQ);
        for (uint32_t rb = 0; rb < nrb; ++rb, ++ab) {
          const uint32_t b = ab & 1u, u = ab >> 1;
          if (u > 0) mbar_wait(acc_empty + b, (u - 1) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
            const uint32_t s = it % kLsStages;
            mbar_wait(full + s, (it / kLsStages) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t A = smem_u32(ring + s * kLsStage);
            const uint32_t B = smem_u32(qB + kb * (kLsNQ * 128));
#pragma unroll
            for (uint32_t k8 = 0; k8 < kLsKB / 8; ++k8) {
              umma_tf32(tmem + b * kLsNQ, sw128_kmajor_desc(A + 32 * k8),
                        sw128_kmajor_desc(B + 32 * k8), idesc, (kb | k8) != 0);
            }
            umma_commit(empty + s);
          }
          umma_commit(acc_full + b);
        }
      }
      __syncwarp();
    } else if (warp >= 8) { // ---- row norms from the same stages ----
      const uint32_t row = threadIdx.x - 256;
      for (uint32_t rb = 0; rb < nrb; ++rb, ++ab) {
        const uint32_t b = ab & 1u, u = ab >> 1;
        if (u > 0) mbar_wait(acc_empty + b, (u - 1) & 1u);
        float acc = 0.f;
        for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
          const uint32_t s = it % kLsStages;
          mbar_wait(full + s, (it / kLsStages) & 1u);
          const float4* rp = reinterpret_cast<const float4*>(ring + s * kLsStage + row * 128);
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            // rotated chunk order: the 8 rows of a load phase hit 8 distinct
            // 16-byte bank groups (rows are 128 B apart)
            const float4 x = rp[(ch + row) & 7];
            acc = fmaf(x.x, x.x, acc);
            acc = fmaf(x.y, x.y, acc);
            acc = fmaf(x.z, x.z, acc);
            acc = fmaf(x.w, x.w, acc);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
        }
        s_vn2[b][row] = acc;
        __syncwarp();
        if (lane == 0) mbar_arrive(norm_full + b);
      }
    } else if (warp >= 4) { // ---- epilogue ----
      const uint32_t e = threadIdx.x - 128, quad = warp & 3;
      for (uint32_t rb = 0; rb < nrb; ++rb, ++ab) {
        const uint32_t b = ab & 1u, ph = (ab >> 1) & 1u;
        mbar_wait(acc_full + b, ph);
        mbar_wait(norm_full + b, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t v[kLsNQ];
#pragma unroll
        for (uint32_t h = 0; h < kLsNQ; h += 16) {
          const uint32_t taddr = tmem + ((32u * quad) << 16) + b * kLsNQ + h;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15}, [%16];"
              : "=r"(v[h + 0]), "=r"(v[h + 1]), "=r"(v[h + 2]), "=r"(v[h + 3]), "=r"(v[h + 4]),
                "=r"(v[h + 5]), "=r"(v[h + 6]), "=r"(v[h + 7]), "=r"(v[h + 8]), "=r"(v[h + 9]),
                "=r"(v[h + 10]), "=r"(v[h + 11]), "=r"(v[h + 12]), "=r"(v[h + 13]),
                "=r"(v[h + 14]), "=r"(v[h + 15])
              : "r"(taddr));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const float vn2f = s_vn2[b][e];
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + b);

        const uint32_t rin = rb * kLsM + e; // row within the item
        if (r0 + rin < r1) {
          // ||v|| rounded up, covering the fp32 sum of squares
          const double vn2 = double(vn2f) * (1.0 + 2e-4);
          const double vn = sqrt(vn2);
#pragma unroll
          for (uint32_t j = 0; j < kLsNQ; ++j) {
            if (j >= nqg) break;
            const double s = __uint_as_float(v[j]);
            double g, err;
            if (a.metric == kIP) {
              g = s;
              err = kTcErr * double(s_qn[j]) * vn;
            } else {
              const double qn2 = s_qn2[j];
              g = -(qn2 + vn2 - 2.0 * s);
              err = 2.0 * kTcErr * double(s_qn[j]) * vn + 2e-4 * (qn2 + vn2);
            }
            const uint32_t hk = ls_key(__double2float_ru(g + err));
            if (hk >= s_tau[j]) {
              const uint32_t p = atomicAdd(s_cnt + j, 1u);
              if (p < cap) {
                c_lo[j * cap + p] = ls_key(__double2float_rd(g - err));
                c_hi[j * cap + p] = hk;
                c_rw[j * cap + p] = static_cast<uint16_t>(rin);
              } else {
                ls_overflow(a);
              }
            }
          }
        }
        named_sync(1, 128);
        for (uint32_t j = quad; j < nqg; j += 4) {
          if (s_cnt[j] > trig) {
            ls_compact(c_lo + j * cap, c_hi + j * cap, c_rw + j * cap, s_cnt + j, s_tau + j,
                       uint32_t(a.k), cap, lane);
          }
        }
        named_sync(1, 128);
      }
      // ---- flush: final compaction, share tau, append the survivors ----
      for (uint32_t j = quad; j < nqg; j += 4) {
        const uint32_t q = s_q[j];
        if (lane == 0) s_tau[j] = max(s_tau[j], atomicAdd(a.gtau + q, 0u));
        __syncwarp();
        ls_compact(c_lo + j * cap, c_hi + j * cap, c_rw + j * cap, s_cnt + j, s_tau + j,
                   uint32_t(a.k), cap, lane);
        const uint32_t m = s_cnt[j];
        uint32_t base = 0;
        if (lane == 0) {
          atomicMax(a.gtau + q, s_tau[j]);
          base = m ? atomicAdd(a.gcnt + q, m) : 0u;
        }
        base = __shfl_sync(kFull, base, 0);
        if (base + m > a.gcap) {
          if (lane == 0) ls_overflow(a);
        } else {
          uint4* out = a.cand + uint64_t(q) * a.gcap + base;
          for (uint32_t i = lane; i < m; i += 32) {
            out[i] = make_uint4(c_lo[j * cap + i], c_hi[j * cap + i], c,
                                static_cast<uint32_t>(s0 + c_rw[j * cap + i]));
          }
        }
      }
    }
    __syncthreads(); // the item's MMAs are complete (the epilogue saw acc_full)
    cur ^= 1u;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ---- plan ----
__global__ void __launch_bounds__(128) ls_count_kernel(const uint32_t* __restrict__ order,
                                                       uint32_t lp, const int64_t* __restrict__ res,
                                                       uint32_t* qcount) {
  const uint32_t* o = order + uint64_t(blockIdx.x) * lp;
  for (uint32_t i = threadIdx.x; i < lp; i += blockDim.x) {
    const uint32_t c = o[i];
    if (res[c] >= 0) atomicAdd(qcount + c, 1u);
  }
}

__global__ void __launch_bounds__(128) ls_fill_kernel(const uint32_t* __restrict__ order,
                                                      uint32_t lp, const int64_t* __restrict__ res,
                                                      uint32_t* fill, uint32_t* qidx) {
  const uint32_t* o = order + uint64_t(blockIdx.x) * lp;
  for (uint32_t i = threadIdx.x; i < lp; i += blockDim.x) {
    const uint32_t c = o[i];
    if (res[c] >= 0) qidx[atomicAdd(fill + c, 1u)] = blockIdx.x;
  }
}

// Exclusive block scan of three counters (1024 threads).
__device__ void block_scan3(uint32_t (&v)[3], uint32_t (&tot)[3], uint32_t* sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t inc[3] = {v[0], v[1], v[2]};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const uint32_t y = __shfl_up_sync(kFull, inc[x], o);
      if (lane >= o) inc[x] += y;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int x = 0; x < 3; ++x) sh[warp * 3 + x] = inc[x];
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t w[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) w[x] = sh[lane * 3 + x];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const uint32_t y = __shfl_up_sync(kFull, w[x], o);
        if (lane >= o) w[x] += y;
      }
    }
#pragma unroll
    for (int x = 0; x < 3; ++x) sh[96 + lane * 3 + x] = w[x];
  }
  __syncthreads();
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    const uint32_t before_warp = warp ? sh[96 + (warp - 1) * 3 + x] : 0u;
    tot[x] = sh[96 + 31 * 3 + x];
    v[x] = before_warp + inc[x] - v[x];
  }
}

__global__ void __launch_bounds__(1024) ls_plan_kernel(uint32_t* qcount, uint32_t nc,
                                                       const uint64_t* __restrict__ list_off,
                                                       uint32_t* lists, uint32_t* lq_off,
                                                       uint32_t* item_off, uint32_t* meta,
                                                       uint32_t gq, uint32_t rows) {
  __shared__ uint32_t sh[96 + 96];
  const uint32_t per = (nc + 1023) / 1024;
  const uint32_t c0 = min(nc, threadIdx.x * per), c1 = min(nc, c0 + per);
  auto items = [&](uint32_t c, uint32_t qc) {
    const uint64_t len = list_off[c + 1] - list_off[c];
    return uint32_t((qc + gq - 1) / gq) * uint32_t((len + rows - 1) / rows);
  };
  uint32_t v[3] = {0, 0, 0};
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t qc = qcount[c];
    if (qc) {
      v[0] += 1;
      v[1] += qc;
      v[2] += items(c, qc);
    }
  }
  uint32_t tot[3];
  block_scan3(v, tot, sh);
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t qc = qcount[c];
    if (qc) {
      lists[v[0]] = c;
      lq_off[v[0]] = v[1];
      item_off[v[0]] = v[2];
      qcount[c] = v[1]; // the fill cursor of this list's query slots
      v[0] += 1;
      v[1] += qc;
      v[2] += items(c, qc);
    }
  }
  if (threadIdx.x == 0) {
    lq_off[tot[0]] = tot[1];
    item_off[tot[0]] = tot[2];
    meta[0] = tot[0];
    meta[1] = tot[2];
  }
}

// ---- final: exact top-k per query from its candidates ----
struct LsFinal {
  const float* Q;
  uint32_t d;
  int metric;
  int k;
  const uint4* cand;
  const uint32_t* gcnt;
  uint32_t gcap;
  const float* slab;
  const uint64_t* ids;
  const int64_t* res;
  const uint64_t* list_off;
  uint32_t* meta;
  unsigned* flag_host;
  float* out_s;
  uint64_t* out_id;
  uint32_t* out_count;
  const uint32_t* fcount_in;
  uint32_t* fcount_out;
};

__global__ void __launch_bounds__(kLsFinalThreads) ls_final_kernel(LsFinal a) {
  extern __shared__ unsigned char fsm[];
  float* sq = reinterpret_cast<float*>(fsm);                               // [d]
  uint32_t* srow = reinterpret_cast<uint32_t*>(sq + ((a.d + 3) & ~3u));    // [kLsSurv]
  uint32_t* scl = srow + kLsSurv;                                          // [kLsSurv]
  float* ssc = reinterpret_cast<float*>(scl + kLsSurv);                    // [kLsSurv]
  uint64_t* sid = reinterpret_cast<uint64_t*>(ssc + kLsSurv + (kLsSurv & 1)); // [kLsSurv]
  __shared__ uint32_t s_ns, s_stop;
  const uint32_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = kLsFinalThreads / 32;
  if (threadIdx.x == 0) {
    s_ns = 0;
    s_stop = *reinterpret_cast<volatile uint32_t*>(a.meta + 3);
    if (a.fcount_out) a.fcount_out[q] = a.fcount_in[q];
  }
  __syncthreads();
  if (s_stop) return; // overflow: the caller re-runs the per-query scan
  for (uint32_t i = threadIdx.x; i < a.d; i += kLsFinalThreads) sq[i] = a.Q[uint64_t(q) * a.d + i];
  const uint32_t m = min(a.gcnt[q], a.gcap);
  const uint4* cand = a.cand + uint64_t(q) * a.gcap;
  // tau = k-th largest lower bound over all candidates (MSB-first radix)
  uint32_t tau = 0;
  if (m >= uint32_t(a.k)) {
    uint32_t prefix = 0, need = a.k;
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t want = prefix | (1u << bit), mask = ~((1u << bit) - 1u);
      uint32_t mine = 0;
      for (uint32_t i = threadIdx.x; i < m; i += kLsFinalThreads) {
        mine += (__ldg(&cand[i].x) & mask) == want;
      }
      mine = warp_sum(mine);
      __shared__ uint32_t wsum[nw];
      if (lane == 0) wsum[warp] = mine;
      __syncthreads();
      uint32_t cnt = 0;
#pragma unroll
      for (int w = 0; w < nw; ++w) cnt += wsum[w];
      __syncthreads();
      if (cnt >= need) prefix = want;
      else need -= cnt;
    }
    tau = prefix;
  }
  for (uint32_t i = threadIdx.x; i < m; i += kLsFinalThreads) {
    const uint4 e = __ldg(cand + i);
    if (e.y >= tau) {
      const uint32_t p = atomicAdd(&s_ns, 1u);
      if (p < kLsSurv) {
        srow[p] = e.w;
        scl[p] = e.z;
      }
    }
  }
  __syncthreads();
  const uint32_t ns = s_ns;
  if (ns > kLsSurv) {
    if (threadIdx.x == 0) {
      atomicExch(a.meta + 3, 1u);
      *reinterpret_cast<volatile unsigned*>(a.flag_host) = 1u;
    }
    return;
  }
  // exact fp64 re-score (vectorstore.cpp:93-115 terms), one warp per row
  const uint32_t d = a.d;
  for (uint32_t s = warp; s < ns; s += nw) {
    const float* row = a.slab + uint64_t(srow[s]) * d;
    double acc = 0.0;
    if ((d & 3u) == 0) {
      for (uint32_t j4 = lane; j4 < (d >> 2); j4 += 32) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(row) + j4);
        const float4 qq = reinterpret_cast<const float4*>(sq)[j4];
        const double q4[4] = {qq.x, qq.y, qq.z, qq.w};
        Acc4<true>::run(a.metric, q4, x, acc);
      }
    } else {
      for (uint32_t j = lane; j < d; j += 32) {
        acc = a.metric == kIP ? term_ip_d(sq[j], __ldg(row + j), acc)
                              : term_l2_d(sq[j], __ldg(row + j), acc);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      const uint32_t c = scl[s];
      ssc[s] = finish_score(a.metric, acc);
      sid[s] = a.ids[a.list_off[c] + (uint64_t(srow[s]) - uint64_t(a.res[c]))];
    }
  }
  __syncthreads();
  const bool ip = a.metric == kIP;
  for (uint32_t s = threadIdx.x; s < ns; s += kLsFinalThreads) {
    const float x = ssc[s];
    const uint64_t xi = sid[s];
    uint32_t r = 0;
    for (uint32_t t = 0; t < ns; ++t) {
      const float y = ssc[t];
      r += (ip ? y > x : y < x) || (y == x && sid[t] < xi);
    }
    if (r < uint32_t(a.k)) {
      a.out_s[uint64_t(q) * a.k + r] = x;
      a.out_id[uint64_t(q) * a.k + r] = xi;
    }
  }
  if (threadIdx.x == 0) a.out_count[q] = min(ns, uint32_t(a.k));
}

} // namespace

// Candidate slots per query per item that fit next to the ring and the
// staged queries (multiple of 32, <= kLsMaxCap).
static uint32_t list_scan_cap(uint32_t d, uint32_t nq) {
  const uint32_t nkb = (d + kLsKB - 1) / kLsKB;
  const size_t fixed = 1024 + size_t(ls_stages(nq)) * kLsStage + size_t(nkb) * nq * 128 + 4096;
  const size_t avail = 227 * 1024 > fixed ? 227 * 1024 - fixed : 0;
  size_t cap = avail / (nq * (4 + 4 + 2));
  cap = std::min<size_t>(cap, kLsMaxCap) & ~size_t(31);
  return static_cast<uint32_t>(cap);
}

bool list_scan_supported(uint32_t d, int k, uint32_t group) {
  if (group != 16 && group != 32) return false;
  return (d % 4) == 0 && d >= 4 && d <= 1024 && k >= 1 && k <= int(kLsMaxK) &&
         list_scan_cap(d, group) >= kLsM + 2 * uint32_t(k);
}

size_t list_scan_smem(uint32_t d, uint32_t group) {
  const uint32_t nkb = (d + kLsKB - 1) / kLsKB;
  return 1024 + size_t(ls_stages(group)) * kLsStage + size_t(nkb) * group * 128 +
         size_t(group) * list_scan_cap(d, group) * (4 + 4 + 2);
}

static void ls_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ls_ck((x), #x)

void launch_list_scan(const ListScan& p, cudaStream_t st) {
  const ListScanScratch& s = p.scratch;
  const uint32_t nq = p.nq;
  if (nq == 0) return;
  CK(cudaMemsetAsync(s.qcount, 0, size_t(p.nc) * sizeof(uint32_t), st));
  CK(cudaMemsetAsync(s.meta, 0, 4 * sizeof(uint32_t), st));
  CK(cudaMemsetAsync(s.gcnt, 0, size_t(nq) * sizeof(uint32_t), st));
  CK(cudaMemsetAsync(s.gtau, 0, size_t(nq) * sizeof(uint32_t), st));
  if (p.lp) {
    ls_count_kernel<<<nq, 128, 0, st>>>(p.order, p.lp, p.res, s.qcount);
    after_launch();
  }
  const uint32_t gq = p.group == 32 ? 32u : 16u;
  uint32_t rows = p.chunk >= kLsM && p.chunk <= 65536 && p.chunk % kLsM == 0 ? p.chunk
                                                                            : kLsChunk;
  ls_plan_kernel<<<1, 1024, 0, st>>>(s.qcount, p.nc, p.list_off, s.lists, s.lq_off, s.item_off,
                                     s.meta, gq, rows);
  after_launch();
  if (p.lp) {
    ls_fill_kernel<<<nq, 128, 0, st>>>(p.order, p.lp, p.res, s.qcount, s.qidx);
    after_launch();
  }
  LsArgs a;
  a.Q = p.Q;
  a.d = p.d;
  a.metric = p.metric;
  a.k = p.k;
  a.res = p.res;
  a.list_off = p.list_off;
  a.lists = s.lists;
  a.lq_off = s.lq_off;
  a.item_off = s.item_off;
  a.qidx = s.qidx;
  a.meta = s.meta;
  a.gtau = s.gtau;
  a.gcnt = s.gcnt;
  a.cand = reinterpret_cast<uint4*>(s.cand);
  a.gcap = s.gcap;
  a.cap = list_scan_cap(p.d, gq);
  a.chunk = rows;
  a.flag_host = p.flag_host;
  const CUtensorMap map = make_row_tile_map(p.slab, p.slab_rows, p.d, kLsM);
  const CUtensorMap tail = make_row_tile_map(p.slab, p.slab_rows, p.d, 16);
  const size_t smem = list_scan_smem(p.d, gq);
  auto kern = gq == 32 ? list_scan_tc_kernel<32> : list_scan_tc_kernel<16>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  kern<<<p.grid, kLsThreads, smem, st>>>(map, tail, a);
  after_launch();
  LsFinal f;
  f.Q = p.Q;
  f.d = p.d;
  f.metric = p.metric;
  f.k = p.k;
  f.cand = reinterpret_cast<const uint4*>(s.cand);
  f.gcnt = s.gcnt;
  f.gcap = s.gcap;
  f.slab = p.slab;
  f.ids = p.ids;
  f.res = p.res;
  f.list_off = p.list_off;
  f.meta = s.meta;
  f.flag_host = p.flag_host;
  f.out_s = p.out_s;
  f.out_id = p.out_id;
  f.out_count = p.out_count;
  f.fcount_in = p.fcount_in;
  f.fcount_out = p.fcount_out;
  const size_t fsmem = ((p.d + 3) & ~3u) * 4 + size_t(kLsSurv) * (4 + 4 + 4 + 8) + 8;
  ensure_dyn_smem(reinterpret_cast<const void*>(ls_final_kernel), fsmem);
  ls_final_kernel<<<nq, kLsFinalThreads, fsmem, st>>>(f);
  after_launch();
}

#undef CK

} // namespace laivg
