// green_probe.cu — can runtime-API kernels / graphs run on streams of a green context (SM partition)?
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/gp green_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#define CKD(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
#define CKR(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void k_smid(unsigned* out, int iters) {
  unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64(); while (clock64() - t0 < iters) {}
  if (threadIdx.x == 0) atomicMax(out, s), atomicAdd(out + 1, 1u);
  __shared__ unsigned seen; if (threadIdx.x == 0) { seen = s; out[2 + s] = 1; }
}

int main() {
  CKR(cudaSetDevice(0));
  CKR(cudaFree(0));   // primary context
  CUdevice dev; CKD(cuDeviceGet(&dev, 0));
  CUdevResource all; CKD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("SMs in device resource: %u\n", all.sm.smCount);
  CUdevResource parts[2], rest; unsigned n = 1;
  CKD(cuDevSmResourceSplitByCount(parts, &n, &all, &rest, 0, 40));
  printf("split: %u group(s) of %u SMs, remaining %u SMs\n", n, parts[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d0, d1; CKD(cuDevResourceGenerateDesc(&d0, &parts[0], 1)); CKD(cuDevResourceGenerateDesc(&d1, &rest, 1));
  CUgreenCtx g0, g1; CKD(cuGreenCtxCreate(&g0, d0, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CKD(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s0, s1; CKD(cuGreenCtxStreamCreate(&s0, g0, CU_STREAM_NON_BLOCKING, 0)); CKD(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
  unsigned* buf; CKR(cudaMalloc(&buf, 4096));   // primary-context allocation
  for (int which = 0; which < 2; ++which) {
    CKR(cudaMemsetAsync(buf, 0, 4096, (cudaStream_t)(which ? s1 : s0)));
    k_smid<<<296, 128, 0, (cudaStream_t)(which ? s1 : s0)>>>(buf, 200000);
    CKR(cudaGetLastError());
    CKR(cudaStreamSynchronize((cudaStream_t)(which ? s1 : s0)));
    unsigned h[2 + 256]; CKR(cudaMemcpy(h, buf, sizeof h, cudaMemcpyDeviceToHost));
    int used = 0; for (int i = 0; i < 256; ++i) used += h[2 + i] ? 1 : 0;
    printf("stream of green ctx %d: CTAs %u, distinct SMs used %d\n", which, h[1], used);
  }
  // graph capture on a green-context stream
  cudaGraph_t g; cudaGraphExec_t ge;
  CKR(cudaStreamBeginCapture((cudaStream_t)s0, cudaStreamCaptureModeThreadLocal));
  k_smid<<<296, 128, 0, (cudaStream_t)s0>>>(buf, 1000);
  CKR(cudaStreamEndCapture((cudaStream_t)s0, &g));
  CKR(cudaGraphInstantiate(&ge, g, 0));
  CKR(cudaMemset(buf, 0, 4096));
  CKR(cudaGraphLaunch(ge, (cudaStream_t)s0)); CKR(cudaStreamSynchronize((cudaStream_t)s0));
  unsigned h[2 + 256]; CKR(cudaMemcpy(h, buf, sizeof h, cudaMemcpyDeviceToHost));
  int used = 0; for (int i = 0; i < 256; ++i) used += h[2 + i] ? 1 : 0;
  printf("graph on green stream 0: CTAs %u, distinct SMs %d\n", h[1], used);
  // events across contexts
  cudaEvent_t ev; CKR(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CKR(cudaEventRecord(ev, (cudaStream_t)s0)); CKR(cudaStreamWaitEvent((cudaStream_t)s1, ev, 0));
  CKR(cudaStreamSynchronize((cudaStream_t)s1));
  printf("cross-context event wait OK\n");
  return 0;
}
