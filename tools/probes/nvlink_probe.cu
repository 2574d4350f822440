// NVLink SM-copy probe: remote load / remote store / local bandwidth from a
// kernel on GPU 0 against GPU 1 memory (peer access), various unrolls.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void rd(const double2* __restrict__ src, double2* __restrict__ dst, long long n) {
  long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
}

int main() {
  int n_dev = 0;
  CK(cudaGetDeviceCount(&n_dev));
  if (n_dev < 2) { printf("need 2 GPUs\n"); return 1; }
  const long long bytes = 256ll << 20, n = bytes / 16;
  double2 *a0, *b0, *a1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMemset(a1, 0, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 0, bytes));
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, const double2* s, double2* d, int blocks) {
    kern<<<blocks, 256>>>(s, d, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<blocks, 256>>>(s, d, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s blocks %5d: %7.1f GB/s\n", name, blocks, bytes * 5 / (ms * 1e-3) / 1e9);
  };
  for (int bpsm : {1, 2, 4, 8}) {
    const int blocks = nsm * bpsm;
    run("remote load  U=1", rd<1>, a1, b0, blocks);
    run("remote load  U=4", rd<4>, a1, b0, blocks);
    run("remote store U=1", rd<1>, a0, a1, blocks);
    run("remote store U=4", rd<4>, a0, a1, blocks);
    run("local copy   U=4", rd<4>, a0, b0, blocks);
  }
  // copy engine
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cudaMemcpyPeer 0->1: %.1f GB/s\n", bytes * 5 / (ms * 1e-3) / 1e9);
  return 0;
}
