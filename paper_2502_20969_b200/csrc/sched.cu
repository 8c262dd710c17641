// sched.cu — the micro-batch schedulers on the GPU.
//
//   pair_dist_kernel   : fp64 L2^2 of every query pair (i < j) with the
//                        reference's serial per-term arithmetic
//                        (l2_sq_d, vectorstore.cpp:101-108), one pair per
//                        thread, so distances are bit-identical to the CPU
//   group_kernel       : the greedy of group_microbatches (sched.cpp:39-70)
//                        in one CTA: lowest unassigned seed, then its m-1
//                        nearest unassigned later queries by (distance,
//                        index), as partial_sort on pairs orders them
//   overlap_kernel     : assign_cache_aware's overlap matrix
//                        (sched.cpp:99-108): per micro-batch, the union of
//                        its queries' probes as a bitset in shared memory,
//                        then popcount(union & resident_w) for every worker
//
// The greedy assignment over the nb x nw overlap matrix stays on the host
// (greedy_assign, host.cpp): it is O(nb^2 nw) on a few hundred entries.
#include <cstdint>
#include <stdexcept>

#include "dev_common.cuh"
#include "host.hpp"
#include "kernels.cuh"

namespace laivg {
using namespace dev;
namespace {

__global__ void __launch_bounds__(256)
    pair_dist_kernel(const float* __restrict__ Q, uint32_t n, uint32_t d,
                     double* __restrict__ dist) {
  const uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t np = static_cast<uint64_t>(n) * n;
  if (p >= np) return;
  const uint32_t i = static_cast<uint32_t>(p / n), j = static_cast<uint32_t>(p % n);
  if (j <= i) return;
  const float* a = Q + static_cast<uint64_t>(i) * d;
  const float* b = Q + static_cast<uint64_t>(j) * d;
  double acc = 0.0;
  for (uint32_t t = 0; t < d; ++t) { // serial, separately rounded: the reference order
    const double u = __dsub_rn(static_cast<double>(__ldg(a + t)), static_cast<double>(__ldg(b + t)));
    acc = __dadd_rn(acc, __dmul_rn(u, u));
  }
  dist[p] = acc;
}

__device__ __forceinline__ bool pair_less(double da, uint32_t ia, double db, uint32_t ib) {
  return da < db || (da == db && ia < ib);
}

// One CTA of kGroupThreads threads; n <= kGroupThreads * kGroupPer.
// order_out[n] = the queries batch by batch, off_out[nb + 1] CSR offsets,
// *nb_out = number of batches. The seed's distance row is read once into
// registers; the assigned flags live in shared memory.
constexpr int kGroupThreads = 1024;
constexpr int kGroupPer = 8;
__global__ void __launch_bounds__(kGroupThreads)
    group_kernel(const double* __restrict__ dist, uint32_t n, uint32_t m,
                 uint64_t* __restrict__ order_out, uint64_t* __restrict__ off_out,
                 uint32_t* __restrict__ nb_out) {
  extern __shared__ unsigned char taken[];
  __shared__ double wd[32];
  __shared__ uint32_t wi[32];
  __shared__ uint32_t s_pick;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) taken[j] = 0;
  __syncthreads();
  uint32_t pos = 0, nb = 0;
  if (threadIdx.x == 0) off_out[0] = 0;
  for (uint32_t seed = 0; seed < n; ++seed) {
    if (taken[seed]) continue; // uniform: every thread reads the same byte
    __syncthreads();
    if (threadIdx.x == 0) {
      taken[seed] = 1;
      order_out[pos] = seed;
    }
    ++pos;
    const double* row = dist + static_cast<uint64_t>(seed) * n;
    double rd[kGroupPer];
#pragma unroll
    for (int u = 0; u < kGroupPer; ++u) {
      const uint32_t j = threadIdx.x + u * blockDim.x;
      rd[u] = (j > seed && j < n) ? row[j] : INFINITY;
    }
    for (uint32_t t = 1; t < m; ++t) {
      __syncthreads();
      // (distance, index)-smallest unassigned j > seed
      double bd = INFINITY;
      uint32_t bi = 0xffffffffu;
#pragma unroll
      for (int u = 0; u < kGroupPer; ++u) {
        const uint32_t j = threadIdx.x + u * blockDim.x;
        if (j > seed && j < n && !taken[j] && pair_less(rd[u], j, bd, bi)) {
          bd = rd[u];
          bi = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, bd, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (pair_less(od, oi, bd, bi)) {
          bd = od;
          bi = oi;
        }
      }
      if (lane == 0) {
        wd[warp] = bd;
        wi[warp] = bi;
      }
      __syncthreads();
      if (warp == 0) {
        bd = lane < nwarps ? wd[lane] : INFINITY;
        bi = lane < nwarps ? wi[lane] : 0xffffffffu;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (pair_less(od, oi, bd, bi)) {
            bd = od;
            bi = oi;
          }
        }
        if (lane == 0) {
          s_pick = bi;
          if (bi != 0xffffffffu) {
            taken[bi] = 1;
            order_out[pos] = bi;
          }
        }
      }
      __syncthreads();
      if (s_pick == 0xffffffffu) break; // fewer than m-1 unassigned remain
      ++pos;
    }
    ++nb;
    if (threadIdx.x == 0) off_out[nb] = pos;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nb_out = nb;
}

// One CTA per micro-batch. probes[q * L + i]; members of batch b are
// order[off[b] .. off[b + 1]); resident bitsets [nw][words].
__global__ void __launch_bounds__(256)
    overlap_kernel(const uint32_t* __restrict__ probes, uint32_t L,
                   const uint64_t* __restrict__ order, const uint64_t* __restrict__ off,
                   const unsigned long long* __restrict__ resident, uint32_t nw, uint32_t words,
                   unsigned long long* __restrict__ overlap) {
  extern __shared__ unsigned long long uni[];
  const uint32_t b = blockIdx.x;
  for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) uni[w] = 0ull;
  __syncthreads();
  const uint64_t m0 = off[b], m1 = off[b + 1];
  for (uint64_t x = threadIdx.x; x < (m1 - m0) * L; x += blockDim.x) {
    const uint64_t q = order[m0 + x / L];
    const uint32_t c = probes[q * L + x % L];
    atomicOr(&uni[c >> 6], 1ull << (c & 63));
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t wk = warp; wk < nw; wk += blockDim.x >> 5) {
    unsigned long long cnt = 0;
    const unsigned long long* r = resident + static_cast<uint64_t>(wk) * words;
    for (uint32_t w = lane; w < words; w += 32) cnt += __popcll(uni[w] & r[w]);
    cnt = warp_sum(cnt);
    if (lane == 0) overlap[static_cast<uint64_t>(b) * nw + wk] = cnt;
  }
}

} // namespace

void launch_pair_dist(const float* Q, uint32_t n, uint32_t d, double* dist, cudaStream_t st) {
  const uint64_t np = static_cast<uint64_t>(n) * n;
  if (np == 0) return;
  pair_dist_kernel<<<static_cast<unsigned>((np + 255) / 256), 256, 0, st>>>(Q, n, d, dist);
  after_launch();
}

uint32_t group_max_queries() { return kGroupThreads * kGroupPer; }

void launch_group(const double* dist, uint32_t n, uint32_t m, uint64_t* order, uint64_t* off,
                  uint32_t* nb, cudaStream_t st) {
  if (n > group_max_queries()) throw std::invalid_argument("too many queries for GPU grouping");
  group_kernel<<<1, kGroupThreads, n, st>>>(dist, n, m, order, off, nb);
  after_launch();
}

void launch_overlap(const uint32_t* probes, uint32_t L, const uint64_t* order,
                    const uint64_t* off, uint32_t nb, const unsigned long long* resident,
                    uint32_t nw, uint32_t words, unsigned long long* overlap, cudaStream_t st) {
  if (nb == 0 || nw == 0) return;
  overlap_kernel<<<nb, 256, words * sizeof(unsigned long long), st>>>(probes, L, order, off,
                                                                      resident, nw, words,
                                                                      overlap);
  after_launch();
}

} // namespace laivg
