// Green-context probe: can runtime <<<>>> launches go to streams of SM
// partitions (cuGreenCtxStreamCreate), and do they stay on their SMs?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* m; cuGetErrorString(r_, &m); printf("%s -> %s\n", #x, m); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

int main(int argc, char** argv) {
  const unsigned su = argc > 1 ? atoi(argv[1]) : 32;
  RK(cudaSetDevice(0));
  RK(cudaFree(nullptr));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all, part, rest;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned n = 1;
  CK(cuDevSmResourceSplitByCount(&part, &n, &all, &rest, 0, su));
  printf("total SMs %u, part %u, rest %u\n", all.sm.smCount, part.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d1, d2;
  CK(cuDevResourceGenerateDesc(&d1, &part, 1));
  CK(cuDevResourceGenerateDesc(&d2, &rest, 1));
  CUgreenCtx g1, g2;
  CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2;
  CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
  int *o1, *o2;
  RK(cudaMalloc(&o1, 4096 * 4));
  RK(cudaMalloc(&o2, 4096 * 4));
  const int nb = 1000;
  smid_kernel<<<nb, 64, 0, (cudaStream_t)s1>>>(o1);
  RK(cudaGetLastError());
  smid_kernel<<<nb, 64, 0, (cudaStream_t)s2>>>(o2);
  RK(cudaGetLastError());
  // cross-stream event from the primary context
  cudaEvent_t ev;
  RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  RK(cudaEventRecord(ev, (cudaStream_t)s1));
  cudaStream_t ps;
  RK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
  RK(cudaStreamWaitEvent(ps, ev, 0));
  RK(cudaDeviceSynchronize());
  std::vector<int> h1(nb), h2(nb);
  RK(cudaMemcpy(h1.data(), o1, nb * 4, cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(h2.data(), o2, nb * 4, cudaMemcpyDeviceToHost));
  std::set<int> a(h1.begin(), h1.end()), b(h2.begin(), h2.end());
  int overlap = 0;
  for (int x : a) overlap += b.count(x);
  printf("stream1 used %zu SMs, stream2 used %zu SMs, shared %d\n", a.size(), b.size(), overlap);
  // attribute: the kernel's smem opt-in from the primary context applies?
  printf("ok\n");
  return 0;
}
