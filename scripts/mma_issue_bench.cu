// Microbenchmark: cost of a chain of tcgen05.mma.kind::i8 (M = 128, K = 32 per instruction) issued
// by one thread from operands already resident in shared memory, by N and by the per-K-block
// bookkeeping of k_gemm_i8's MMA loop (mbarrier wait + tcgen05.fence::after_thread_sync every 4
// MMAs, a commit per K block).  One CTA, %clock64 around the issue loop and the final commit wait.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1805_12096_b200/csrc \
//        scripts/mma_issue_bench.cu -o scripts/mma_issue_bench -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "ptx.cuh"

using namespace mnmt;

template <int N>
__global__ void k_bench(int kblocks, int mode, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar_full, bar_done, bar_kb;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // operands: A 128 x 128 B, B N x 128 B (contents irrelevant; zero-filled)
  for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_done, 1);
    mbar_init(&bar_kb, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<N < 32 ? 32 : N>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar_full, 0);   // completes phase 0 at once
  __syncthreads();
  if (mode >= 3) {
    // the whole warp runs the loop (warp-uniform: descriptors and the TMEM address stay in
    // uniform registers); one elected lane issues each MMA
    if (warp == 1) {
      constexpr uint32_t idesc = idesc_i8<128, N>();
      const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
      const uint64_t adesc = umma_desc_sw128(sa), bdesc = umma_desc_sw128(sb);
      const uint32_t tm = slot;
      const unsigned long long t0 = clock64();
      for (int kb = 0; kb < kblocks; ++kb) {
        if (mode >= 4) {
          mbar_wait(&bar_full, 0);
          tc_fence_after();
        }
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_i8(tm, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
          if (mode >= 4) mma_commit(&bar_kb);
        }
        __syncwarp();
      }
      const unsigned long long t1 = clock64();
      if (elect_one()) mma_commit(&bar_done);
      __syncwarp();
      mbar_wait(&bar_done, 0);
      const unsigned long long t2 = clock64();
      if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_i8<128, N>();
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    const uint64_t adesc = umma_desc_sw128(sa), bdesc = umma_desc_sw128(sb);
    const unsigned long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      if (mode >= 1) {   // the MMA loop's per-K-block wait (already complete) + fence
        mbar_wait(&bar_full, 0);
        tc_fence_after();
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_i8(slot, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
      if (mode >= 2) mma_commit(&bar_kb);   // per-K-block commit (frees a stage in k_gemm_i8)
    }
    const unsigned long long t1 = clock64();
    mma_commit(&bar_done);
    mbar_wait(&bar_done, 0);
    const unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<N < 32 ? 32 : N>(slot);
}

template <int N>
static void run(int kblocks, int mode, unsigned long long* d) {
  const int smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(k_bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long h[2] = {0, 0};
  for (int rep = 0; rep < 3; ++rep) {
    k_bench<N><<<1, 128, smem>>>(kblocks, mode, d);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const int n = 4 * kblocks;
  static const char* names[] = {"MMAs only", "+ wait/fence per K block", "+ commit per K block",
                                "warp-uniform + elect", "warp-uniform + elect + wait/fence/commit"};
  printf("N %3d  K blocks %2d  mode %d (%s): issue %6llu cyc, complete %6llu cyc = %6.1f cyc per MMA (%.2f us at 1.965 GHz)\n",
         N, kblocks, mode, names[mode],
         h[0], h[1], (double)h[1] / n, h[1] / 1965.0);
  (void)names;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  for (int mode = 0; mode < 5; ++mode)
    for (int kb : {1, 8, 32}) {
      run<16>(kb, mode, d);
      run<64>(kb, mode, d);
      run<256>(kb, mode, d);
    }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
