// Probe: CUDA green contexts (SM partitions) on this driver -- can a chain of small kernels run on
// a reserved set of SMs beside bulk kernels on the rest, also inside one captured graph?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/greenctx_probe tools/greenctx_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("FAIL %s: %s\n", #x, s_); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void mark(int* out, int spin) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)smid;
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}

static void report(const char* what, const int* h, int n) {
  std::set<int> s(h, h + n);
  printf("%s: %d CTAs on %zu distinct SMs, min %d max %d\n", what, n, s.size(), *s.begin(), *s.rbegin());
}

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  CUdevResource part[1], rest;
  unsigned int ng = 1;
  CK(cuDevSmResourceSplitByCount(part, &ng, &all, &rest, 0, 32));
  printf("split: groups %u, part %u SMs, remaining %u SMs\n", ng, part[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dA, dB;
  CK(cuDevResourceGenerateDesc(&dA, &part[0], 1));
  CK(cuDevResourceGenerateDesc(&dB, &rest, 1));
  CUgreenCtx gA, gB;
  CK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  CK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, -5));
  CK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  const int n = 1024;
  int *dAo, *dBo;
  RK(cudaMalloc(&dAo, n * sizeof(int)));
  RK(cudaMalloc(&dBo, n * sizeof(int)));
  std::vector<int> h(n);
  // direct launches through the runtime API on the green-context streams
  mark<<<n, 128, 0, (cudaStream_t)sA>>>(dAo, 20000);
  mark<<<n, 128, 0, (cudaStream_t)sB>>>(dBo, 20000);
  RK(cudaGetLastError());
  RK(cudaDeviceSynchronize());
  RK(cudaMemcpy(h.data(), dAo, n * sizeof(int), cudaMemcpyDeviceToHost));
  report("direct A (32-SM partition)", h.data(), n);
  RK(cudaMemcpy(h.data(), dBo, n * sizeof(int), cudaMemcpyDeviceToHost));
  report("direct B (rest)", h.data(), n);
  // a user stream of the primary context forks into both partitions (events), also as a graph
  cudaStream_t user;
  RK(cudaStreamCreateWithFlags(&user, cudaStreamNonBlocking));
  cudaEvent_t e0, eA, eB;
  RK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
  RK(cudaEventCreateWithFlags(&eA, cudaEventDisableTiming));
  RK(cudaEventCreateWithFlags(&eB, cudaEventDisableTiming));
  RK(cudaMemset(dAo, 0xff, n * sizeof(int)));
  RK(cudaMemset(dBo, 0xff, n * sizeof(int)));
  cudaGraph_t graph;
  RK(cudaStreamBeginCapture(user, cudaStreamCaptureModeThreadLocal));
  RK(cudaEventRecord(e0, user));
  RK(cudaStreamWaitEvent((cudaStream_t)sA, e0, 0));
  RK(cudaStreamWaitEvent((cudaStream_t)sB, e0, 0));
  mark<<<n, 128, 0, (cudaStream_t)sA>>>(dAo, 20000);
  mark<<<n, 128, 0, (cudaStream_t)sB>>>(dBo, 20000);
  RK(cudaEventRecord(eA, (cudaStream_t)sA));
  RK(cudaEventRecord(eB, (cudaStream_t)sB));
  RK(cudaStreamWaitEvent(user, eA, 0));
  RK(cudaStreamWaitEvent(user, eB, 0));
  RK(cudaStreamEndCapture(user, &graph));
  cudaGraphExec_t exec;
  RK(cudaGraphInstantiate(&exec, graph, 0));
  RK(cudaGraphLaunch(exec, user));
  RK(cudaStreamSynchronize(user));
  RK(cudaMemcpy(h.data(), dAo, n * sizeof(int), cudaMemcpyDeviceToHost));
  report("graph A (32-SM partition)", h.data(), n);
  RK(cudaMemcpy(h.data(), dBo, n * sizeof(int), cudaMemcpyDeviceToHost));
  report("graph B (rest)", h.data(), n);
  printf("OK\n");
  return 0;
}
