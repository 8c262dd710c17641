// wide.cu — the size-unbounded device paths of the drop-in (VERDICT r01
// Missing #1/#2): what the reference accepts for any size and the on-chip
// kernels of kernels.cu cap.
//
//   score_all_kernel    every member of the fast lists of one query, scored
//                       with the scan's arithmetic (fp64 per term, lane-strided
//                       float4 order + butterfly, rounded to f32), written as
//                       one orderable 64-bit key per candidate:
//                         (score key << 32) | rank of the datastore id
//                       so that ascending keys are exactly the reference's
//                       total order (score by metric, then ascending id;
//                       vectorstore.hpp:34-39) with no ties left to break.
//                       Raw mode writes (score, id) in candidate order instead:
//                       score_clusters (ivf.cpp:301-324).
//   (radix sort)        the keys of one query (CUB's multi-CTA onesweep radix
//                       sort), then the first k are the top-k: search_clusters
//                       for any k (ivf.cpp:326-343: partial_sort).
//   wide_emit_kernel    key -> (score, id) for the first min(k, V).
//   rank_keys_kernel    coarse ranking for any number of clusters: fp64 score
//                       -> orderable key, cluster id as the value; a stable
//                       radix sort leaves equal scores in ascending cluster
//                       order (rank_clusters, ivf.cpp:269-291).
//   pairwise_l2_kernel  pairwise_l2 (vectorstore.cpp:141-153): serial fp64
//                       l2_sq_d per pair, separately rounded like the
//                       reference, sqrt, f32 — bit-identical; 32x32 pair tiles
//                       staged through shared memory, four independent chains
//                       per thread.
//
// Everything here is opt-in by size: k <= kMaxK and nc <= kMaxSortNc stay on
// the register/shared-memory kernels.
#include <cub/device/device_radix_sort.cuh>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "dev_common.cuh"
#include "host.hpp"
#include "kernels.cuh"

namespace laivg {
using namespace dev;
namespace {

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      throw ::laivg::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t float_order_w(float f) { // ascending with f
  const uint32_t b = __float_as_uint(f + 0.0f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float order_float_w(uint32_t u) {
  return __uint_as_float((u >> 31) ? (u & 0x7fffffffu) : ~u);
}
// ascending == best first
__device__ __forceinline__ uint32_t score_key(int metric, float s) {
  const uint32_t o = float_order_w(s);
  return metric == kIP ? ~o : o;
}
__device__ __forceinline__ float key_score(int metric, uint32_t k) {
  return order_float_w(metric == kIP ? ~k : k);
}

// One query; warp w of the grid scores the flattened fast-list range
// [V*w/W, V*(w+1)/W) two rows at a time. The per-row arithmetic is the
// scan's (kernels.cu scan_tma_kernel / scan_ldg_kernel, fp64 mode): lane l
// accumulates float4 chunks l, l+32, ... with Acc4<true>, then warp_sum; for
// d % 4 != 0 scalar terms j = l, l+32, ...
__global__ void __launch_bounds__(256)
    score_all_kernel(const float* __restrict__ q, uint32_t qi, uint32_t d, int metric,
                     FastTable ft, const float* __restrict__ slab,
                     const uint32_t* __restrict__ rank_of_row, const uint64_t* __restrict__ ids,
                     uint64_t V, uint64_t* __restrict__ keys, float* __restrict__ raw_s,
                     uint64_t* __restrict__ raw_id) {
  extern __shared__ __align__(16) float sq[];
  for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) sq[i] = q[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tb = static_cast<uint64_t>(qi) * ft.stride;
  const uint64_t* pre = ft.pre + static_cast<uint64_t>(qi) * (ft.stride + 1);
  const uint32_t nf = ft.count[qi];
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
  const uint64_t v0 = V * gw / tw, v1 = V * (gw + 1) / tw;
  if (v0 >= v1 || nf == 0) return;
  // cursor over the fast lists (same walk as the scans)
  uint32_t li;
  {
    uint32_t lo = 0, hi = nf - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= v0) lo = mid;
      else hi = mid - 1;
    }
    li = lo;
  }
  uint64_t o = v0 - pre[li];
  uint64_t len = ft.len[tb + li];
  while (o >= len) {
    o -= len;
    ++li;
    len = ft.len[tb + li];
  }
  int64_t slab0 = ft.slab[tb + li];
  uint64_t row0 = ft.row[tb + li];
  const bool vec4 = (d & 3u) == 0;
  for (uint64_t v = v0; v < v1; v += 2) {
    int64_t sv[2];
    uint64_t rw[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      ok[u] = v + u < v1;
      sv[u] = slab0 + static_cast<int64_t>(o);
      rw[u] = row0 + o;
      if (ok[u] && v + u + 1 < v1) {
        ++o;
        while (o >= len) {
          o -= len;
          ++li;
          len = ft.len[tb + li];
          slab0 = ft.slab[tb + li];
          row0 = ft.row[tb + li];
        }
      }
    }
    double a[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      const float* x = slab + static_cast<uint64_t>(sv[u]) * d;
      if (vec4) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* q4 = reinterpret_cast<const float4*>(sq);
        for (uint32_t j4 = lane; j4 < (d >> 2); j4 += 32) {
          const float4 qq = q4[j4];
          const double qd[4] = {qq.x, qq.y, qq.z, qq.w};
          Acc4<true>::run(metric, qd, ldg_stream(x4 + j4), a[u]);
        }
      } else {
        for (uint32_t j = lane; j < d; j += 32) {
          const float xv = __ldg(x + j);
          a[u] = metric == kIP ? term_ip_d(sq[j], xv, a[u]) : term_l2_d(sq[j], xv, a[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double t = warp_sum(a[u]);
      if (!ok[u] || lane != 0) continue;
      const float s = finish_score<double>(metric, t);
      if (keys) {
        keys[v + u] = (static_cast<uint64_t>(score_key(metric, s)) << 32) | rank_of_row[rw[u]];
      } else {
        raw_s[v + u] = s;
        raw_id[v + u] = ids[rw[u]];
      }
    }
  }
}

__global__ void __launch_bounds__(256)
    wide_emit_kernel(const uint64_t* __restrict__ sorted, uint64_t V, int k, int metric,
                     const uint32_t* __restrict__ row_of_rank, const uint64_t* __restrict__ ids,
                     float* out_s, uint64_t* out_id, uint32_t* out_count,
                     const uint32_t* fcount_in, uint32_t* fcount_out, uint32_t qi) {
  const uint64_t n = V < static_cast<uint64_t>(k) ? V : static_cast<uint64_t>(k);
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = sorted[i];
    out_s[i] = key_score(metric, static_cast<uint32_t>(key >> 32));
    out_id[i] = ids[row_of_rank[static_cast<uint32_t>(key)]];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out_count[0] = static_cast<uint32_t>(n);
    if (fcount_out) fcount_out[0] = fcount_in[qi];
  }
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    v[i] = static_cast<uint32_t>(i);
  }
}

__global__ void invert_kernel(const uint32_t* __restrict__ row_of_rank, uint64_t n,
                              uint32_t* __restrict__ rank_of_row) {
  for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    rank_of_row[row_of_rank[r]] = static_cast<uint32_t>(r);
  }
}

// keys[q][c] = order_key(score) (ascending = best first), vals = c
__global__ void __launch_bounds__(256)
    rank_keys_kernel(const double* __restrict__ scores, uint64_t n, uint32_t nc, int metric,
                     uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    keys[i] = order_key(scores[i], metric);
    vals[i] = static_cast<uint32_t>(i % nc);
  }
}

__global__ void take_prefix_kernel(const uint32_t* __restrict__ sorted_v, uint32_t nc,
                                   uint32_t n_out, uint32_t* __restrict__ order) {
  const uint32_t q = blockIdx.y;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += gridDim.x * blockDim.x) {
    order[static_cast<uint64_t>(q) * n_out + i] = sorted_v[static_cast<uint64_t>(q) * nc + i];
  }
}

// 32 x 32 output tile per CTA (16 x 16 threads, 2 x 2 pairs each: four
// independent serial chains); A and B tiles staged 32 components at a time.
constexpr int kPT = 32;
__global__ void __launch_bounds__(256)
    pairwise_l2_kernel(const float* __restrict__ A, uint64_t na, const float* __restrict__ B,
                       uint64_t nb, uint32_t d, float* __restrict__ out, bool squared_f64,
                       double* __restrict__ out_sq) {
  __shared__ float sa[kPT][kPT + 1];
  __shared__ float sb[kPT][kPT + 1];
  const uint32_t tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const uint64_t i0 = static_cast<uint64_t>(blockIdx.y) * kPT, j0 = static_cast<uint64_t>(blockIdx.x) * kPT;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (uint32_t t0 = 0; t0 < d; t0 += kPT) {
    for (uint32_t e = threadIdx.x; e < kPT * kPT; e += blockDim.x) {
      const uint32_t r = e / kPT, c = e % kPT;
      const uint64_t ia = i0 + r, jb = j0 + r;
      sa[r][c] = (ia < na && t0 + c < d) ? A[ia * d + t0 + c] : 0.f;
      sb[r][c] = (jb < nb && t0 + c < d) ? B[jb * d + t0 + c] : 0.f;
    }
    __syncthreads();
    const uint32_t tn = min(static_cast<uint32_t>(kPT), d - t0);
    for (uint32_t t = 0; t < tn; ++t) { // serial in t: the reference's order
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const double x = __dsub_rn(static_cast<double>(sa[ty + 16 * u][t]),
                                     static_cast<double>(sb[tx + 16 * w][t]));
          acc[u][w] = __dadd_rn(acc[u][w], __dmul_rn(x, x));
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const uint64_t i = i0 + ty + 16 * u, j = j0 + tx + 16 * w;
      if (i < na && j < nb) {
        if (squared_f64) out_sq[i * nb + j] = acc[u][w];
        else out[i * nb + j] = static_cast<float>(sqrt(acc[u][w]));
      }
    }
  }
}

int grid_for(uint64_t n, int threads = 256) {
  const uint64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 4096 ? (b ? b : 1) : 4096);
}

} // namespace

// ---- id ranks -------------------------------------------------------------
void build_id_rank(const uint64_t* ids, uint64_t n, uint32_t* rank_of_row, uint32_t* row_of_rank,
                   cudaStream_t st) {
  if (n == 0) return;
  if (n >= (1ull << 32)) throw std::invalid_argument("wide path supports < 2^32 rows");
  uint64_t* ids_sorted = nullptr;
  uint32_t* rows = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  CK(cudaMalloc(&ids_sorted, n * sizeof(uint64_t)));
  CK(cudaMalloc(&rows, n * sizeof(uint32_t)));
  iota_kernel<<<grid_for(n), 256, 0, st>>>(rows, n);
  after_launch();
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ids, ids_sorted, rows, row_of_rank,
                                     static_cast<int64_t>(n), 0, 64, st));
  CK(cudaMalloc(&tmp, tmp_bytes));
  CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ids, ids_sorted, rows, row_of_rank,
                                     static_cast<int64_t>(n), 0, 64, st));
  invert_kernel<<<grid_for(n), 256, 0, st>>>(row_of_rank, n, rank_of_row);
  after_launch();
  CK(cudaStreamSynchronize(st));
  cudaFree(ids_sorted);
  cudaFree(rows);
  cudaFree(tmp);
}

// ---- wide scan --------------------------------------------------------------
size_t wide_sort_temp_bytes(uint64_t n) {
  size_t b = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, b, static_cast<const uint64_t*>(nullptr),
                                    static_cast<uint64_t*>(nullptr), static_cast<int64_t>(n), 0,
                                    64, nullptr));
  return b;
}

void launch_score_all(const float* q, uint32_t qi, uint32_t d, int metric, const FastTable& ft,
                      const float* slab, const uint32_t* rank_of_row, const uint64_t* ids,
                      uint64_t V, uint64_t* keys, float* raw_s, uint64_t* raw_id, int num_sms,
                      cudaStream_t st) {
  if (V == 0) return;
  const uint64_t warps = (V + 15) / 16; // >= 16 rows per warp
  uint64_t ctas = (warps + 7) / 8;
  const uint64_t cap = uint64_t(num_sms) * 8;
  if (ctas > cap) ctas = cap;
  const size_t smem = ((size_t(d) * 4 + 15) & ~size_t(15));
  if (smem > 48 * 1024) ensure_dyn_smem(reinterpret_cast<const void*>(score_all_kernel), smem);
  score_all_kernel<<<static_cast<unsigned>(ctas), 256, smem, st>>>(
      q, qi, d, metric, ft, slab, rank_of_row, ids, V, keys, raw_s, raw_id);
  after_launch();
}

void launch_wide_topk(uint64_t* keys, uint64_t* keys_alt, uint64_t V, int k, int metric,
                      void* tmp, size_t tmp_bytes, const uint32_t* row_of_rank,
                      const uint64_t* ids, float* out_s, uint64_t* out_id, uint32_t* out_count,
                      const uint32_t* fcount_in, uint32_t* fcount_out, uint32_t qi,
                      cudaStream_t st) {
  if (V) {
    size_t b = tmp_bytes;
    CK(cub::DeviceRadixSort::SortKeys(tmp, b, keys, keys_alt, static_cast<int64_t>(V), 0, 64, st));
  }
  const uint64_t n = V < uint64_t(k) ? V : uint64_t(k);
  wide_emit_kernel<<<grid_for(n ? n : 1), 256, 0, st>>>(keys_alt, V, k, metric, row_of_rank, ids,
                                                        out_s, out_id, out_count, fcount_in,
                                                        fcount_out, qi);
  after_launch();
}

// ---- ranking for any nc -----------------------------------------------------
size_t rank_large_temp_bytes(uint32_t nc) {
  size_t b = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const uint64_t*>(nullptr),
                                     static_cast<uint64_t*>(nullptr),
                                     static_cast<const uint32_t*>(nullptr),
                                     static_cast<uint32_t*>(nullptr), static_cast<int64_t>(nc), 0,
                                     64, nullptr));
  return b;
}

void launch_rank_large(const double* scores, uint32_t nq, uint32_t nc, int metric, uint32_t n_out,
                       uint32_t* order, RankScratch& rs, cudaStream_t st) {
  if (nq == 0 || nc == 0 || n_out == 0) return;
  const uint64_t n = uint64_t(nq) * nc;
  rank_keys_kernel<<<grid_for(n), 256, 0, st>>>(scores, n, nc, metric, rs.keys, rs.vals);
  after_launch();
  for (uint32_t q = 0; q < nq; ++q) {
    size_t b = rs.tmp_bytes;
    const uint64_t o = uint64_t(q) * nc;
    // stable: equal keys keep ascending cluster order (ivf.cpp:282-289)
    CK(cub::DeviceRadixSort::SortPairs(rs.tmp, b, rs.keys + o, rs.keys_alt + o, rs.vals + o,
                                       rs.vals_alt + o, static_cast<int64_t>(nc), 0, 64, st));
  }
  take_prefix_kernel<<<dim3((n_out + 255) / 256, nq), 256, 0, st>>>(rs.vals_alt, nc, n_out, order);
  after_launch();
}

// ---- pairwise_l2 ------------------------------------------------------------
void launch_pairwise_l2(const float* A, uint64_t na, const float* B, uint64_t nb, uint32_t d,
                        float* out, double* out_sq, cudaStream_t st) {
  if (na == 0 || nb == 0) return;
  if ((nb + kPT - 1) / kPT > 0x7fffffffull || (na + kPT - 1) / kPT > 65535ull) {
    throw std::invalid_argument("pairwise_l2: matrix too large for one launch");
  }
  const dim3 grid(static_cast<unsigned>((nb + kPT - 1) / kPT), static_cast<unsigned>((na + kPT - 1) / kPT));
  pairwise_l2_kernel<<<grid, 256, 0, st>>>(A, na, B, nb, d, out, out_sq != nullptr, out_sq);
  after_launch();
}

} // namespace laivg
