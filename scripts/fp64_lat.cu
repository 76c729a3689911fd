// Dependent-chain latency of fp64 / fp32 FMA and fp64 exp on this GPU (one warp, clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat scripts/fp64_lat.cu && ./fp64_lat
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* outf, long long* cyc, double x0, float y0, int n) {
  double a = x0, b = 1.0000001;
  float fa = y0, fb = 1.0000001f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __fma_rn(a, b, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) fa = __fmaf_rn(fa, fb, 1e-9f);
  long long t2 = clock64();
  double e = x0;
  for (int i = 0; i < n / 16; ++i) e = exp(-e * 1e-3);
  long long t3 = clock64();
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, (double)fa * i);
  long long t4 = clock64();
  out[threadIdx.x] = a + e + s;
  outf[threadIdx.x] = fa;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&of, 1024 * 4); cudaMalloc(&c, 64);
  const int n = 4096;
  for (int warps : {1, 4, 16, 32}) {
    k<<<1, 32 * warps>>>(o, of, c, 1.0, 1.0f, n);
    long long h[4];
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d: fp64 FMA chain %.1f cyc/op, fp32 FMA %.1f, fp64 exp %.1f cyc, fp64 add(+cvt,mul) %.1f\n", warps,
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / (n / 16), (double)h[3] / n);
  }
  return 0;
}
