// pdl_floor.cu — cost of one dependent kernel in a CUDA graph with programmatic dependent launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pf pdl_floor.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_empty(int* p, int mode) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (mode == 1 && threadIdx.x == 0) { int v = *(volatile int*)p; if (v == 12345) p[1] = v; }      // one dependent L2 read
  if (mode == 2 && threadIdx.x == 0) { int v = *(volatile int*)p; p[blockIdx.x + 2] = v + 1; }     // read + write
}

int main() {
  int* p; CK(cudaMalloc(&p, 1 << 20)); CK(cudaMemset(p, 0, 1 << 20));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int mode = 0; mode < 3; ++mode)
      for (int blocks : {1, 4, 148}) {
        const int N = 200;
        cudaGraph_t g; cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < N; ++i) {
          cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(128); cfg.stream = st;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = pdl; cfg.attrs = at; cfg.numAttrs = 1;
          CK(cudaLaunchKernelEx(&cfg, k_empty, p, mode));
        }
        CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, st); CK(cudaGraphLaunch(ge, st)); cudaEventRecord(b, st); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("pdl %d mode %d (%s) blocks %3d: %.2f us per kernel\n", pdl, mode,
               mode == 0 ? "empty" : mode == 1 ? "1 dependent read" : "read+write", blocks, 1000 * ms / N);
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
      }
  return 0;
}
