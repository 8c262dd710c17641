// CPU cost of cudaGraphLaunch for graph shapes like the single-query chain:
// which node kinds make the launch expensive. nvcc -O2 -arch=sm_100a -o /tmp/glp tools/graph_launch_probe.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__global__ void k_small(float* p) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1.f; }
__global__ void k_big(float* p) {
  extern __shared__ float sm[];
  if (threadIdx.x == 0) sm[0] = p[0];
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) p[1] = sm[0];
}

double launch_us(cudaGraphExec_t ge, cudaStream_t st) {
  std::vector<double> v;
  for (int i = 0; i < 200; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    cudaGraphLaunch(ge, st);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    v.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  float *d, *h;
  cudaMalloc(&d, 1 << 20);
  cudaHostAlloc(&h, 1 << 20, cudaHostAllocMapped);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  auto capture = [&](int variant) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    if (variant & 1) cudaMemcpyAsync(d, h, 3072, cudaMemcpyHostToDevice, st);
    if (variant & 4) cudaEventRecordWithFlags(ev[0], st, cudaEventRecordExternal);
    k_small<<<512, 256, 0, st>>>(d);
    k_small<<<16, 256, 0, st>>>(d);
    k_small<<<1, 1024, 0, st>>>(d);
    if (variant & 4) cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal);
    if (variant & 2) k_big<<<148, 288, 200 * 1024, st>>>(d);
    else k_small<<<148, 288, 0, st>>>(d);
    if (variant & 4) cudaEventRecordWithFlags(ev[2], st, cudaEventRecordExternal);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphUpload(ge, st);
    cudaStreamSynchronize(st);
    return ge;
  };
  const char* names[] = {"4 kernels", "memcpy + 4 kernels", "4 kernels (one 200KB smem)",
                         "memcpy + 4 kernels (200KB)", "4 kernels + 3 events",
                         "memcpy + 4k + 3 ev", "4k(200KB) + 3 ev", "memcpy + 4k(200KB) + 3 ev"};
  for (int v = 0; v < 8; ++v) {
    auto ge = capture(v);
    std::printf("{\"graph\": \"%s\", \"launch_us_p50\": %.2f}\n", names[v], launch_us(ge, st));
  }
  // eager equivalents
  std::vector<double> e;
  for (int i = 0; i < 200; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    cudaMemcpyAsync(d, h, 3072, cudaMemcpyHostToDevice, st);
    k_small<<<512, 256, 0, st>>>(d);
    k_small<<<16, 256, 0, st>>>(d);
    k_small<<<1, 1024, 0, st>>>(d);
    k_big<<<148, 288, 200 * 1024, st>>>(d);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    e.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(e.begin(), e.end());
  std::printf("{\"eager\": \"memcpy + 4 kernels (200KB)\", \"submit_us_p50\": %.2f}\n", e[100]);
  return 0;
}
