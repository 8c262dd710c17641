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
#include <algorithm>
#include <stdexcept>
#include <string>

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

// ---------------------------------------------------------------------------
// group_microbatches for any n (no n x n matrix): one persistent grid, every
// CTA co-resident (cooperative launch), walking the seeds in order. Thread t
// owns queries j = t, t + T, ... (T = grid threads). Per seed s: each owner
// computes l2_sq_d(q_s, q_j) for its unassigned j > s (serial, the
// reference's order), then m-1 rounds pick the (distance, index)-smallest
// unassigned j: thread -> warp -> CTA minimum into a per-CTA slot, one grid
// barrier, then every CTA reduces the slots itself (no second barrier); the
// owner of the pick marks it taken. A barrier ends each seed so every CTA
// sees the same taken flags.
// ---------------------------------------------------------------------------
struct GridBar {
  unsigned count;
  unsigned gen;
};

__device__ __forceinline__ void grid_barrier(GridBar* b, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &b->gen;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(&b->count, 1u) == nblocks - 1) {
      b->count = 0;
      __threadfence();
      atomicAdd(&b->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kGLThreads = 256;
__global__ void __launch_bounds__(kGLThreads)
    group_large_kernel(const float* __restrict__ Q, uint32_t n, uint32_t d, uint32_t m,
                       unsigned char* taken, double* dist_row, double* slot_d, uint32_t* slot_i,
                       GridBar* bar, uint64_t* __restrict__ order_out,
                       uint64_t* __restrict__ off_out, uint32_t* __restrict__ nb_out) {
  extern __shared__ float sseed[];
  __shared__ double wd[kGLThreads / 32];
  __shared__ uint32_t wi[kGLThreads / 32];
  const unsigned G = gridDim.x;
  const uint32_t T = G * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  volatile unsigned char* vt = taken;
  uint64_t pos = 0;
  uint32_t nb = 0, round = 0;
  if (t == 0) off_out[0] = 0;
  for (uint32_t s = 0; s < n; ++s) {
    if (vt[s]) continue; // uniform: read after the last barrier
    if (t == 0) order_out[pos] = s;
    ++pos;
    if (m > 1 && s + 1 < n) {
      for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) sseed[i] = Q[static_cast<uint64_t>(s) * d + i];
      __syncthreads();
      for (uint32_t j = t; j < n; j += T) {
        if (j <= s || vt[j]) continue;
        const float* b = Q + static_cast<uint64_t>(j) * d;
        double acc = 0.0;
        for (uint32_t e = 0; e < d; ++e) { // serial, separately rounded (l2_sq_d)
          const double u = __dsub_rn(static_cast<double>(sseed[e]), static_cast<double>(__ldg(b + e)));
          acc = __dadd_rn(acc, __dmul_rn(u, u));
        }
        dist_row[j] = acc;
      }
      for (uint32_t r = 1; r < m; ++r, ++round) {
        double bd = INFINITY;
        uint32_t bi = 0xffffffffu;
        for (uint32_t j = t; j < n; j += T) {
          if (j <= s || vt[j]) continue;
          const double dj = dist_row[j];
          if (pair_less(dj, j, bd, bi)) {
            bd = dj;
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
        const uint32_t par = (round & 1u) * G;
        if (threadIdx.x == 0) {
          double cd = wd[0];
          uint32_t ci = wi[0];
          for (int w = 1; w < kGLThreads / 32; ++w) {
            if (pair_less(wd[w], wi[w], cd, ci)) {
              cd = wd[w];
              ci = wi[w];
            }
          }
          slot_d[par + blockIdx.x] = cd;
          slot_i[par + blockIdx.x] = ci;
        }
        grid_barrier(bar, G);
        // every CTA reduces the slots: same answer everywhere
        bd = INFINITY;
        bi = 0xffffffffu;
        for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) {
          const double od = __ldcg(slot_d + par + g);
          const uint32_t oi = __ldcg(slot_i + par + g);
          if (pair_less(od, oi, bd, bi)) {
            bd = od;
            bi = oi;
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
        __syncthreads();
        if (lane == 0) {
          wd[warp] = bd;
          wi[warp] = bi;
        }
        __syncthreads();
        bd = wd[0];
        bi = wi[0];
        for (int w = 1; w < kGLThreads / 32; ++w) {
          if (pair_less(wd[w], wi[w], bd, bi)) {
            bd = wd[w];
            bi = wi[w];
          }
        }
        __syncthreads();
        if (bi == 0xffffffffu) break; // fewer than m-1 unassigned remain
        if (bi % T == t) taken[bi] = 1; // the owner: only it reads taken[bi] this seed
        if (t == 0) order_out[pos] = bi;
        ++pos;
      }
    }
    ++nb;
    if (t == 0) off_out[nb] = pos;
    grid_barrier(bar, G); // every owner's taken flags visible before the next seed
  }
  if (t == 0) *nb_out = nb;
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

void launch_group_large(const float* Q, uint32_t n, uint32_t d, uint32_t m, GroupScratch& gs,
                        uint64_t* order, uint64_t* off, uint32_t* nb, int num_sms,
                        cudaStream_t st) {
  if (n == 0) return;
  const size_t smem = size_t(d) * sizeof(float);
  auto fn = group_large_kernel;
  if (smem > 48 * 1024) ensure_dyn_smem(reinterpret_cast<const void*>(fn), smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGLThreads, smem);
  if (per_sm < 1) throw std::runtime_error("group_large_kernel does not fit an SM");
  unsigned G = static_cast<unsigned>(std::min(per_sm, 2) * num_sms);
  // at least ~16 queries per thread before adding CTAs
  const unsigned want = static_cast<unsigned>((uint64_t(n) + 16 * kGLThreads - 1) / (16 * kGLThreads));
  if (want < G) G = want < 1 ? 1 : want;
  cudaMemsetAsync(gs.taken, 0, n, st);
  cudaMemsetAsync(gs.bar, 0, sizeof(GridBar), st);
  const float* q = Q;
  unsigned char* tk = gs.taken;
  double* dr = gs.dist_row;
  double* sd = gs.slot_d;
  uint32_t* si = gs.slot_i;
  GridBar* b = reinterpret_cast<GridBar*>(gs.bar);
  void* args[] = {(void*)&q, (void*)&n, (void*)&d, (void*)&m, (void*)&tk, (void*)&dr, (void*)&sd,
                  (void*)&si, (void*)&b, (void*)&order, (void*)&off, (void*)&nb};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(G),
                                                    dim3(kGLThreads), args, smem, st);
  if (e != cudaSuccess) {
    throw CudaError(std::string("group_large_kernel launch: ") + cudaGetErrorString(e));
  }
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
