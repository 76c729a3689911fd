// cluster_microbench.cu — measurements that decide the cluster decoder's exchange design.
// Standalone (not part of libmnmt):  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cmb
//   1. max active clusters of size 8 / 16 at ~200 KB smem
//   2. DSMEM all-gather: each CTA pushes a 4 KB slice (16-byte st.shared::cluster) to all 8
//      CTAs of its cluster, then one remote mbarrier arrive per destination; wait for 8 arrivals
//   3. the same all-gather through L2: st.global of the slice, release/acquire flag, then every
//      CTA reads the cluster's 32 KB
//   4. remote mbarrier ping-pong latency between two CTAs of a cluster
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t a, uint4 v) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void wait_parity_cluster(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
               :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int CS = 8;
constexpr int SLICE = 4096;        // bytes per CTA per all-gather (128 rows x 32 codes)
constexpr int THREADS = 256;

// 2. DSMEM all-gather, `iters` times (two buffers alternate).
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(THREADS, 1)
k_dsmem_ag(int iters, unsigned long long* cycles, int sink_only) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t me = cl.block_rank();
  if (threadIdx.x == 0) { mbar_init(&bar[0], CS); mbar_init(&bar[1], CS); asm volatile("fence.mbarrier_init.release.cluster;"); }
  cl.sync();
  const uint32_t base = smem_u32(sm);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    const uint32_t buf = base + b * (CS * SLICE);
    // this thread's 16 bytes of the slice -> every CTA, at offset me * SLICE + tid * 16
    uint4 v = make_uint4(it, me, threadIdx.x, 0);
    for (int d = 0; d < CS; ++d) st_cluster_v4(mapa(buf + me * SLICE + threadIdx.x * 16, d), v);
    asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
    asm volatile("bar.sync 1, %0;" :: "r"(THREADS));
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      for (int d = 0; d < CS; ++d) arrive_remote(mapa(smem_u32(&bar[b]), d));
    }
    wait_parity_cluster(&bar[b], (it >> 1) & 1);
    if (!sink_only) {
      // read one value from each slice (checks arrival)
      const uint4* p = reinterpret_cast<const uint4*>(sm + b * (CS * SLICE) + (threadIdx.x % CS) * SLICE);
      if (p->x != (uint32_t)it) { printf("bad %d\n", it); asm volatile("trap;"); }
    }
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// 2b. variants. mode: 0 stores+cluster.sync (bandwidth), 1 sync only (arrive/wait, no data),
// 2 st.async with mbarrier complete_tx, 3 one thread bulk-copies the 4 KB slice to 8 CTAs.
__device__ __forceinline__ void st_async_v4(uint32_t a, uint4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];"
               :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar) : "memory");
}
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(THREADS, 1)
k_ag_var(int iters, int mode, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t me = cl.block_rank();
  if (threadIdx.x == 0) { mbar_init(&bar[0], mode >= 2 ? 1 : CS); mbar_init(&bar[1], mode >= 2 ? 1 : CS); asm volatile("fence.mbarrier_init.release.cluster;"); }
  cl.sync();
  const uint32_t base = smem_u32(sm);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    const uint32_t buf = base + b * (CS * SLICE);
    uint4 v = make_uint4(it, me, threadIdx.x, 0);
    if (mode == 0) {
      for (int d = 0; d < CS; ++d) st_cluster_v4(mapa(buf + me * SLICE + threadIdx.x * 16, d), v);
      cluster_sync_all();
    } else if (mode == 1) {
      asm volatile("bar.sync 1, %0;" :: "r"(THREADS));
      if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        for (int d = 0; d < CS; ++d) arrive_remote(mapa(smem_u32(&bar[b]), d));
      }
      wait_parity_cluster(&bar[b], (it >> 1) & 1);
    } else if (mode == 2) {
      // consumer arms its own barrier for 8 x 4 KB; producers st.async into it
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[b])), "r"(CS * SLICE) : "memory");
      for (int d = 0; d < CS; ++d)
        st_async_v4(mapa(buf + me * SLICE + threadIdx.x * 16, d), v, mapa(smem_u32(&bar[b]), d));
      wait_parity_cluster(&bar[b], (it >> 1) & 1);
      // (reuse of buffer b two iterations later is safe: every peer has waited on this phase)
      cluster_sync_all();
    } else {
      // stage locally, one thread bulk-copies to the 8 CTAs
      reinterpret_cast<uint4*>(sm + 2 * CS * SLICE)[threadIdx.x] = v;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" :: "r"(THREADS));
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[b])), "r"(CS * SLICE) : "memory");
        for (int d = 0; d < CS; ++d)
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(mapa(buf + me * SLICE, d)), "r"(base + 2 * CS * SLICE), "r"(SLICE), "r"(mapa(smem_u32(&bar[b]), d)) : "memory");
      }
      wait_parity_cluster(&bar[b], (it >> 1) & 1);
      cluster_sync_all();
    }
    const uint4* p = reinterpret_cast<const uint4*>(sm + b * (CS * SLICE) + (threadIdx.x % CS) * SLICE);
    if (mode != 1 && p->x != (uint32_t)it) { printf("bad mode %d it %d\n", mode, it); asm volatile("trap;"); }
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// 3. L2 all-gather: slice -> global, flag (release), wait flags of the cluster (acquire), read 32 KB.
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(THREADS, 1)
k_l2_ag(int iters, uint8_t* gbuf, unsigned int* flags, unsigned long long* cycles) {
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t me = cl.block_rank();
  const int cid = blockIdx.x / CS;
  uint8_t* cb = gbuf + (size_t)cid * 2 * CS * SLICE;
  unsigned int* cf = flags + cid * CS * 32;
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    uint4 v = make_uint4(it, me, threadIdx.x, 0);
    reinterpret_cast<uint4*>(cb + b * CS * SLICE + me * SLICE)[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("st.release.gpu.u32 [%0], %1;" :: "l"(cf + me * 32), "r"(it + 1) : "memory");
    }
    if (threadIdx.x < CS) {
      unsigned int f;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(f) : "l"(cf + threadIdx.x * 32) : "memory"); } while (f < (unsigned)(it + 1));
    }
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(cb + b * CS * SLICE);
    for (int i = threadIdx.x; i < CS * SLICE / 16; i += THREADS) {
      uint4 x;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(src + i));
      acc += x.x;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (acc == 0xdeadbeef) cycles[0] = 0;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// 4. ping-pong between CTA 0 and CTA 1 of each cluster via remote mbarrier arrivals.
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(THREADS, 1)
k_pingpong(int iters, unsigned long long* cycles) {
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t me = cl.block_rank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  cl.sync();
  long long t0 = clock64();
  if (threadIdx.x == 0 && me < 2) {
    const uint32_t peer = mapa(smem_u32(&bar), me ^ 1);
    for (int it = 0; it < iters; ++it) {
      if (me == 0) { arrive_remote(peer); wait_parity_cluster(&bar, it & 1); }
      else { wait_parity_cluster(&bar, it & 1); arrive_remote(peer); }
    }
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// 5. cluster.sync cost
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(THREADS, 1)
k_csync(int iters, unsigned long long* cycles) {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) cluster_sync_all();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

static double avg(unsigned long long* h, int n) { double s = 0; for (int i = 0; i < n; ++i) s += h[i]; return s / n; }

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("SMs %d clock %d kHz\n", pr.multiProcessorCount, pr.clockRate);
  const int smem = 200 * 1024;
  CK(cudaFuncSetAttribute(k_dsmem_ag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 32); cfg.blockDim = dim3(THREADS); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim = {(unsigned)cs, 1, 1};
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = -1;
    if (cs == 16) cudaFuncSetAttribute(k_csync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k_dsmem_ag, &cfg);
    printf("cluster %2d: max active clusters %d (%s) -> %d SMs\n", cs, ncl, cudaGetErrorString(e), ncl * cs);
    cudaGetLastError();
  }
  const int NCL = 16, nblk = NCL * CS, iters = 2000;
  unsigned long long *d_cyc, h[1024];
  CK(cudaMalloc(&d_cyc, 1024 * 8));
  const double ghz = pr.clockRate * 1e-6;
  for (int sink = 0; sink < 2; ++sink) {
    k_dsmem_ag<<<nblk, THREADS, smem>>>(iters, d_cyc, sink); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d_cyc, nblk * 8, cudaMemcpyDeviceToHost));
    double c = avg(h, nblk) / iters;
    printf("DSMEM all-gather (%d clusters, 8 x 4 KB pushed per CTA): %.0f cyc/iter = %.2f us, %.1f B/cyc/SM out\n", NCL, c, c / ghz / 1e3, 8.0 * SLICE / c);
  }
  for (int ncl : {1, 16}) {
    k_dsmem_ag<<<ncl * CS, THREADS, smem>>>(iters, d_cyc, 1); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d_cyc, ncl * CS * 8, cudaMemcpyDeviceToHost));
    double c = avg(h, ncl * CS) / iters;
    printf("DSMEM all-gather %2d cluster(s): %.0f cyc/iter = %.2f us\n", ncl, c, c / ghz / 1e3);
  }
  CK(cudaFuncSetAttribute(k_ag_var, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[] = {"stores + cluster.sync", "sync only (fence + 8 remote arrives)", "st.async complete_tx (+cluster.sync)", "bulk copy 8 x 4 KB (+cluster.sync)"};
  for (int mode = 0; mode < 4; ++mode) for (int ncl : {1, 15}) {
    k_ag_var<<<ncl * CS, THREADS, smem>>>(iters, mode, d_cyc); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d_cyc, ncl * CS * 8, cudaMemcpyDeviceToHost));
    double c = avg(h, ncl * CS) / iters;
    printf("variant %-40s %2d cl: %.0f cyc/iter = %.2f us\n", names[mode], ncl, c, c / ghz / 1e3);
  }
  uint8_t* g; unsigned int* fl;
  CK(cudaMalloc(&g, NCL * 2 * CS * SLICE)); CK(cudaMalloc(&fl, NCL * CS * 32 * 4));
  for (int ncl : {1, 16}) {
    CK(cudaMemset(fl, 0, NCL * CS * 32 * 4));
    k_l2_ag<<<ncl * CS, THREADS>>>(iters, g, fl, d_cyc); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d_cyc, ncl * CS * 8, cudaMemcpyDeviceToHost));
    double c = avg(h, ncl * CS) / iters;
    printf("L2 all-gather %2d cluster(s) (4 KB write + 32 KB read per CTA): %.0f cyc/iter = %.2f us\n", ncl, c, c / ghz / 1e3);
  }
  k_pingpong<<<CS, THREADS>>>(iters, d_cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d_cyc, CS * 8, cudaMemcpyDeviceToHost));
  printf("remote mbarrier ping-pong round trip: %.0f cyc\n", (double)h[0] / iters);
  k_csync<<<NCL * CS, THREADS>>>(iters, d_cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d_cyc, NCL * CS * 8, cudaMemcpyDeviceToHost));
  printf("cluster.sync: %.0f cyc\n", avg(h, NCL * CS) / iters);
  return 0;
}
