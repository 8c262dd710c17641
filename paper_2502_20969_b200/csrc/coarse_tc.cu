// coarse_tc.cu — batched coarse quantizer on the 5th-generation tensor cores.
//
// For a batch of queries the query x centroid scores (rank_clusters'
// `dot`, ivf.cpp:276-280) form a dense GEMM: S[nq][nc] = Q[nq][d] . C[nc][d]^T.
// This kernel computes it with tcgen05.mma kind::tf32:
//
//   * CTA (m, n) owns 128 centroids (UMMA M) x N queries (UMMA N <= 256),
//   * warp 0 / lane 0 streams 32-float k-blocks of both operands into a
//     4-stage shared-memory ring with TMA tensor copies
//     (cp.async.bulk.tensor.2d, 128-byte swizzle, K-major: the natural
//     row-major layout of centroids and queries),
//   * warp 1 / lane 0 issues 4 MMAs (K = 8) per k-block into a TMEM
//     accumulator (128 lanes x N fp32 columns) and frees each stage with
//     tcgen05.commit on its mbarrier,
//   * all 4 warps drain TMEM with tcgen05.ld (warp w owns lanes 32w..32w+31 =
//     its 32 centroids) and store the approximate scores, coalesced along
//     the centroid axis.
//
// TF32 keeps 10 mantissa bits, so these scores are APPROXIMATE: |s~ - s| <=
// kTcErr * ||q|| * ||c||. They are never reported. The selection kernel
// (tc_select_kernel, kernels.cu) turns them into the exact ranking: it keeps
// every centroid whose upper bound reaches the L-th best lower bound,
// re-scores those candidates with the reference's fp64 arithmetic and sorts
// them exactly. The probe is therefore bit-identical to the fp64 path.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dev_common.cuh"
#include "host.hpp"
#include "kernels.cuh"
#include "umma.cuh"

namespace laivg {
using namespace dev;
namespace {

constexpr uint32_t kTcM = 128;     // centroids per CTA (UMMA M)
constexpr uint32_t kTcKB = 32;     // fp32 elements per k-block = one 128-byte swizzle row
constexpr uint32_t kTcStages = 4;  // TMA ring depth
constexpr uint32_t kTcThreads = 128;

template <uint32_t N>
__global__ void __launch_bounds__(kTcThreads, 1)
    coarse_tc_kernel(const __grid_constant__ CUtensorMap cen_map,
                     const __grid_constant__ CUtensorMap q_map, uint32_t nc, uint32_t nq,
                     uint32_t d, float* __restrict__ approx) {
  constexpr uint32_t kABytes = kTcM * kTcKB * 4;   // 16 KB
  constexpr uint32_t kBBytes = N * kTcKB * 4;      // N * 128 B
  constexpr uint32_t kStage = kABytes + kBBytes;
  constexpr uint32_t kCols = N < 32 ? 32 : N;      // TMEM columns (power of two)
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kTcStages], empty[kTcStages], done;
  __shared__ uint32_t tmem_slot;

  // 1024-byte alignment for the swizzle atoms
  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t m0 = blockIdx.x * kTcM, q0 = blockIdx.y * N;
  // split-K: CTA z accumulates k-blocks [kb0, kb1) into partial plane z
  const uint32_t nkb_all = (d + kTcKB - 1) / kTcKB;
  const uint32_t kb0 = nkb_all * blockIdx.z / gridDim.z;
  const uint32_t kb1 = nkb_all * (blockIdx.z + 1) / gridDim.z;
  const uint32_t nkb = kb1 - kb0;
  approx += static_cast<uint64_t>(blockIdx.z) * nq * nc;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kTcStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&cen_map)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&q_map)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (uint32_t kb = 0; kb < nkb; ++kb) {
      const uint32_t s = kb % kTcStages;
      if (kb >= kTcStages) mbar_wait(empty + s, ((kb / kTcStages) - 1) & 1u);
      unsigned char* a = smem + s * kStage;
      mbar_arrive_expect_tx(full + s, kStage);
      tma_load_2d(a, &cen_map, static_cast<int32_t>((kb0 + kb) * kTcKB),
                  static_cast<int32_t>(m0), full + s);
      tma_load_2d(a + kABytes, &q_map, static_cast<int32_t>((kb0 + kb) * kTcKB),
                  static_cast<int32_t>(q0), full + s);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (one thread for the whole CTA) ----
    constexpr uint32_t idesc = tf32_idesc(kTcM, N);
    for (uint32_t kb = 0; kb < nkb; ++kb) {
      const uint32_t s = kb % kTcStages;
      mbar_wait(full + s, (kb / kTcStages) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = smem_u32(smem + s * kStage), b = a + kABytes;
#pragma unroll
      for (uint32_t k = 0; k < kTcKB / 8; ++k) { // K = 8 tf32 = 32 bytes per MMA
        umma_tf32(tmem, sw128_kmajor_desc(a + 32 * k), sw128_kmajor_desc(b + 32 * k), idesc,
                  (kb | k) != 0);
      }
      umma_commit(empty + s); // frees the stage once these MMAs have read it
    }
    umma_commit(&done);
  }
  __syncwarp();

  // ---- epilogue: TMEM -> registers -> global (all 4 warps) ----
  mbar_wait(&done, 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t row = m0 + 32u * warp + lane; // centroid of this thread's TMEM lane
#pragma unroll 1
  for (uint32_t c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((32u * warp) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < nc) {
#pragma unroll
      for (uint32_t j = 0; j < 32; ++j) {
        const uint32_t q = q0 + c0 + j;
        if (q < nq) approx[static_cast<uint64_t>(q) * nc + row] = __uint_as_float(v[j]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kCols)
                 : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr) {
      cudaGetLastError();
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Row-major fp32 matrix [rows][d] as a 2D tensor map with a (32 x box_rows)
// box and 128-byte swizzle; out-of-range rows/columns read as zero.
CUtensorMap make_map(const float* base, uint64_t rows, uint32_t d, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable from the driver");
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {d, rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 4};
  const cuuint32_t box[2] = {kTcKB, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  }
  return m;
}

template <uint32_t N>
void launch_tc_n(const float* Q, uint32_t nq, const float* cen, uint32_t nc, uint32_t d,
                 float* approx, uint32_t splits, cudaStream_t st) {
  const CUtensorMap cm = make_map(cen, nc, d, kTcM);
  const CUtensorMap qm = make_map(Q, nq, d, N);
  const size_t smem = size_t(kTcStages) * (kTcM + N) * kTcKB * 4 + 1024;
  auto fn = coarse_tc_kernel<N>;
  ensure_dyn_smem(reinterpret_cast<const void*>(fn), smem);
  fn<<<dim3((nc + kTcM - 1) / kTcM, (nq + N - 1) / N, splits), kTcThreads, smem, st>>>(
      cm, qm, nc, nq, d, approx);
  after_launch();
}

} // namespace

CUtensorMap make_row_tile_map(const float* base, uint64_t rows, uint32_t d, uint32_t box_rows) {
  return make_map(base, rows, d, box_rows);
}

bool coarse_tc_supported(uint32_t nc, uint32_t d) {
  return (d % 4) == 0 && d >= 4 && nc <= kTcMaxNc && encode_fn() != nullptr;
}

// Query tile (UMMA N): LAIVG_TC_N overrides (diagnostics / tuning).
uint32_t tc_tile_n(uint32_t nq) {
  static const uint32_t forced = [] {
    const char* e = std::getenv("LAIVG_TC_N");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
  }();
  if (forced == 32 || forced == 64 || forced == 128 || forced == 256) return forced;
  return nq <= 32 ? 32 : nq <= 64 ? 64 : nq <= 128 ? 128 : 256;
}

uint32_t coarse_tc_splits(uint32_t nq, uint32_t nc, uint32_t d, int num_sms) {
  const uint32_t N = tc_tile_n(nq);
  const uint32_t tiles = ((nc + kTcM - 1) / kTcM) * ((nq + N - 1) / N);
  const uint32_t nkb = (d + kTcKB - 1) / kTcKB;
  uint32_t s = tiles >= uint32_t(num_sms) ? 1u : uint32_t(num_sms) / tiles;
  s = std::min<uint32_t>(std::min<uint32_t>(s, kTcMaxSplit), nkb);
  return std::max(1u, s);
}

uint32_t launch_coarse_tc(const float* Q, uint32_t nq, const float* centroids, uint32_t nc,
                          uint32_t d, float* approx, int num_sms, cudaStream_t st) {
  if (nq == 0 || nc == 0) return 1;
  const uint32_t S = coarse_tc_splits(nq, nc, d, num_sms);
  switch (tc_tile_n(nq)) {
    case 32: launch_tc_n<32>(Q, nq, centroids, nc, d, approx, S, st); break;
    case 64: launch_tc_n<64>(Q, nq, centroids, nc, d, approx, S, st); break;
    case 128: launch_tc_n<128>(Q, nq, centroids, nc, d, approx, S, st); break;
    default: launch_tc_n<256>(Q, nq, centroids, nc, d, approx, S, st); break;
  }
  return S;
}

} // namespace laivg
