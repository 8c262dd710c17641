// stream_probe.cu — bandwidth ceilings of the two scan feeding strategies on
// this B200 (developer tool): a cp.async.bulk (TMA) ring with empty consumers
// and a plain 128-bit LDG stream, over a 1 GB buffer (> L2), timed with CUDA
// events. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu
//   /tmp/stream_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// producer warp 0 lane 0; `cons` consumer warps touch one word per stage
__global__ void tma_ring(const char* src, size_t bytes_per_cta, uint32_t stage_bytes,
                         uint32_t S, uint32_t chunks, int cons, float* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * stage_bytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, cons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const char* base = src + blockIdx.x * bytes_per_cta;
  const uint32_t ntiles = static_cast<uint32_t>(bytes_per_cta / stage_bytes);
  float acc = 0.f;
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t i = 0; i < ntiles; ++i) {
        const uint32_t s = i % S;
        mbar_wait(empty + s, ((i / S) & 1u) ^ 1u);
        mbar_expect(full + s, stage_bytes);
        const uint32_t cb = stage_bytes / chunks;
        for (uint32_t c = 0; c < chunks; ++c) {
          bulk(smem + size_t(s) * stage_bytes + c * cb, base + size_t(i) * stage_bytes + c * cb,
               cb, full + s);
        }
      }
    }
  } else {
    for (uint32_t i = 0; i < ntiles; ++i) {
      const uint32_t s = i % S;
      mbar_wait(full + s, (i / S) & 1u);
      acc += reinterpret_cast<const float*>(smem + size_t(s) * stage_bytes)[threadIdx.x];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

// The scan's shape: 768-float rows, T rows per stage, consumers score two
// rows per pass from shared memory (fp32 FMA + warp tree reduction);
// `meta` adds the producer's per-row metadata stores.
__global__ void tma_scan_shape(const char* src, size_t bytes_per_cta, uint32_t T, uint32_t S,
                               int meta, float* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t stage_bytes = T * 3072;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* mrow = empty + S;
  const int cons = 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, cons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const char* base = src + blockIdx.x * bytes_per_cta;
  const uint32_t ntiles = static_cast<uint32_t>(bytes_per_cta / stage_bytes);
  float best = -1e30f;
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t i = 0; i < ntiles; ++i) {
        const uint32_t s = i % S;
        mbar_wait(empty + s, ((i / S) & 1u) ^ 1u);
        if (meta) {
          for (uint32_t t = 0; t < T; ++t) mrow[s * T + t] = uint64_t(i) * T + t;
        }
        mbar_expect(full + s, stage_bytes);
        bulk(smem + size_t(s) * stage_bytes, base + size_t(i) * stage_bytes, stage_bytes, full + s);
      }
    }
  } else {
    float q[24];
    for (int c = 0; c < 24; ++c) q[c] = 0.001f * (lane + c);
    const int cw = warp - 1;
    for (uint32_t i = 0; i < ntiles; ++i) {
      const uint32_t s = i % S;
      mbar_wait(full + s, (i / S) & 1u);
      const float* st = reinterpret_cast<const float*>(smem + size_t(s) * stage_bytes);
      for (uint32_t j = cw; j < T; j += 2 * cons) {
        const float4* r0 = reinterpret_cast<const float4*>(st + j * 768);
        const float4* r1 = reinterpret_cast<const float4*>(st + (j + cons < T ? j + cons : j) * 768);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const float4 x0 = r0[c * 32 + lane], x1 = r1[c * 32 + lane];
          a0 = fmaf(q[4 * c], x0.x, a0); a0 = fmaf(q[4 * c + 1], x0.y, a0);
          a0 = fmaf(q[4 * c + 2], x0.z, a0); a0 = fmaf(q[4 * c + 3], x0.w, a0);
          a1 = fmaf(q[4 * c], x1.x, a1); a1 = fmaf(q[4 * c + 1], x1.y, a1);
          a1 = fmaf(q[4 * c + 2], x1.z, a1); a1 = fmaf(q[4 * c + 3], x1.w, a1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a0 += __shfl_xor_sync(0xffffffffu, a0, o);
          a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        best = fmaxf(best, fmaxf(a0, a1));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
  }
  if (best == 12345.f) sink[0] = best;
}

__global__ void ldg_stream(const float4* src, size_t n4, float* sink) {
  float acc = 0.f;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    acc += a.x + b.y + c.z + d.w;
  }
  for (; i < n4; i += stride) acc += src[i].x;
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const size_t bytes = size_t(1) << 30;
  char* buf;
  float* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { uint32_t stage, S, chunks; int cons, ctas_per_sm; };
  Cfg cfgs[] = {{49152, 4, 1, 8, 1}, {49152, 4, 4, 8, 1}, {49152, 4, 12, 8, 1},
                {24576, 8, 1, 8, 1}, {16384, 12, 1, 8, 1}, {98304, 2, 1, 8, 1},
                {24576, 4, 1, 8, 2}, {16384, 6, 1, 4, 2}, {12288, 4, 1, 4, 4},
                {49152, 4, 1, 1, 1}, {4096, 48, 1, 8, 1}};
  for (const Cfg& c : cfgs) {
    const int grid = sms * c.ctas_per_sm;
    const size_t per = (bytes / grid) / c.stage * c.stage;
    const size_t smem = size_t(c.S) * c.stage + 16 * c.S;
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      tma_ring<<<grid, 32 * (c.cons + 1), smem>>>(buf, per, c.stage, c.S, c.chunks, c.cons, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const cudaError_t e = cudaGetLastError();
    printf("tma stage=%6u S=%2u chunks=%2u cons=%d ctas/sm=%d : %7.1f GB/s %s\n", c.stage, c.S,
           c.chunks, c.cons, c.ctas_per_sm, per * grid / (best * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(tma_scan_shape, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Shape { uint32_t T, S; int meta; };
  for (const Shape& c : {Shape{16, 4, 0}, Shape{16, 4, 1}, Shape{8, 8, 0}, Shape{32, 2, 0},
                         Shape{16, 4, 1}}) {
    const int grid = sms;
    const size_t stage = size_t(c.T) * 3072;
    const size_t per = (bytes / grid) / stage * stage;
    const size_t smem = c.S * stage + 16 * c.S + 8 * c.S * c.T + 16;
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      tma_scan_shape<<<grid, 32 * 9, smem>>>(buf, per, c.T, c.S, c.meta, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const cudaError_t e = cudaGetLastError();
    printf("scan-shape T=%2u S=%u meta=%d : %7.1f GB/s %s\n", c.T, c.S, c.meta,
           per * grid / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {256, 512, 1024}) {
      float best = 1e9f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        ldg_stream<<<sms * bpsm, threads>>>(reinterpret_cast<const float4*>(buf), bytes / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("ldg blocks/sm=%d threads=%4d : %7.1f GB/s\n", bpsm, threads, bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
