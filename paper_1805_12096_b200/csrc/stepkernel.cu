// stepkernel.cu — persistent decode-step kernel for sm_100a.
//
// Why: a decoder step is a chain of ~75 dependent operations (SURVEY 8(a) A5-A10 x 6
// layers).  As separate kernels each link costs ~2.5-4 us of launch/drain latency even with
// PDL (measured), which bounds a step at ~390 us whatever the batch size.  Here the whole
// chain runs inside one cooperative launch: phases are separated by a grid barrier
// (atomic counter + generation flag), and the GEMM machinery is persistent:
//   warp 0     TMA producer over a 3-stage smem ring (pipeline counters persist across
//              phases and steps);
//   warp 1     TMEM allocation (512 columns = two 128x256 s32 accumulators) and the single
//              MMA-issuing thread (tcgen05.mma .kind::i8, M=128, N=bn, K=32);
//   warps 4-11 epilogue: two warps per TMEM lane quarter, one column half each; the
//              accumulator buffer is released (mbarrier) as soon as it has been read, so
//              the next tile's MMAs overlap this tile's epilogue;
//   all 12 warps run the row phases (embedding, LayerNorm, attention) with the same
//   device functions as the standalone kernels (rowdev.cuh); CTA 0 runs the finish /
//   compaction.
// Numerics are those of the standalone kernels (numerics.cuh): bit-identical results.
#include <cstdio>

#include "numerics.cuh"
#include "ptx.cuh"
#include "rowdev.cuh"
#include "stepkernel.h"

namespace mnmt {

namespace {

constexpr int SK_THREADS = 384;               // 12 warps
constexpr int SK_WARPS = SK_THREADS / 32;
constexpr int SK_BM = 128;
constexpr int SK_BK = 128;
constexpr int SK_A_BYTES = SK_BM * SK_BK;     // 16 KB
constexpr int SK_B_MAX = 256 * SK_BK;         // 32 KB (bn <= 256)
constexpr int SK_STAGE = SK_A_BYTES + SK_B_MAX;
constexpr int SK_STAGES = 3;
constexpr int SK_RING = SK_STAGES * SK_STAGE;                       // 144 KB
constexpr int SK_SCRATCH = SK_WARPS * (MNMT_MAX_KV + 64) * 8;       // 54 KB attention scratch
constexpr int SK_SMEM = SK_RING + SK_SCRATCH + 1024;
constexpr int SK_TMEM_COLS = 512;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier for a co-resident (cooperative) grid.  bar[0] = arrivals,
// bar[32] = generation (separate 128-byte lines).
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen;
    __threadfence();
    const unsigned prev = atomicAdd(bar, 1u);
    if (prev == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicExch(bar + 32, g + 1);
    } else {
      // watchdog: a barrier that never completes traps (kernel error) instead of hanging
      long long spins = 0;
      while (ld_acquire_gpu(bar + 32) == g) {
        __nanosleep(20);
        if (++spins > (1ll << 25)) __trap();
      }
    }
    gen = g + 1;
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t idesc_rt(int bn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) | ((128u >> 4) << 24);
}

struct Pipe {
  uint32_t ps = 0, pph = 0;   // producer ring position / phase
  uint32_t cs = 0, cph = 0;   // MMA ring position / phase
  uint32_t ab = 0, aph = 0;   // accumulator buffer / phase (MMA and epilogue keep own copies)
};

// The k-th tile of this CTA in the phase -> (problem, m0, n0); false when exhausted.
//   grid-wide: tiles i = blockIdx.x + k * gridDim.x of all live tiles (problem 0 first);
//   row-local: the CTA owns 128-row tiles mt = blockIdx.x + j * gridDim.x and runs every
//              column tile of every problem of those rows.
__device__ __forceinline__ bool tile_k(const Phase& P, const int* mt_live, int k, int& p, int& m0,
                                       int& n0) {
  if (P.rowlocal) {
    const int tpm = P.g[0].n_tiles + (P.nprob > 1 ? P.g[1].n_tiles : 0);
    const int j = k / tpm;
    int r = k - j * tpm;
    const int mt = blockIdx.x + j * gridDim.x;
    if (mt >= mt_live[0]) return false;
    p = 0;
    if (r >= P.g[0].n_tiles) { p = 1; r -= P.g[0].n_tiles; }
    m0 = mt * SK_BM;
    n0 = r * P.g[p].bn;
    return true;
  }
  int i = blockIdx.x + k * gridDim.x;
  const int T = mt_live[0] * P.g[0].n_tiles + (P.nprob > 1 ? mt_live[1] * P.g[1].n_tiles : 0);
  if (i >= T) return false;
  p = 0;
  const int t0 = mt_live[0] * P.g[0].n_tiles;
  if (i >= t0) { p = 1; i -= t0; }
  const int nt = P.g[p].n_tiles;
  m0 = (i / nt) * SK_BM;
  n0 = (i % nt) * P.g[p].bn;
  return true;
}

// Epilogue of one 32-column chunk of one row (same arithmetic as k_gemm_i8).
__device__ __forceinline__ void epi_chunk(int epi, const GemmArgs a, int row, bool row_ok, int n,
                                          const int32_t* acc, float& best_v, int& best_j) {
  if (n >= a.N) return;
  if (epi == EPI_ARGMAX) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (n + j < a.N) {
        const float b = a.bias ? __ldg(a.bias + n + j) : 0.0f;
        const float v = dequant(acc[j], a.scale, b);
        if (v > best_v) { best_v = v; best_j = n + j; }
      }
    }
    return;
  }
  if (!row_ok) return;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float b = (a.bias && n + j < a.N) ? __ldg(a.bias + n + j) : 0.0f;
    v[j] = dequant(acc[j], a.scale, b);
    if (epi == EPI_RELU_Q || epi == EPI_RELU_F32_Q) v[j] = relu(v[j]);
  }
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int ng = n + 16 * g;
    if (ng >= a.N) break;
    const float* vg = v + 16 * g;
    if (epi == EPI_F32 || epi == EPI_F32_Q || epi == EPI_RELU_F32_Q) {
      const int blk = ng / a.col_block;
      float* dst = a.out_f + (int64_t)blk * a.block_stride + (int64_t)row * a.ldo + (ng - blk * a.col_block);
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int j = 0; j < 4; ++j) d4[j] = make_float4(vg[4 * j], vg[4 * j + 1], vg[4 * j + 2], vg[4 * j + 3]);
    }
    if (epi == EPI_F32_Q || epi == EPI_RELU_Q || epi == EPI_RELU_F32_Q) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t b0 = (uint32_t)(q8(vg[4 * j + 0], a.clip, a.sigma) & 0xff);
        uint32_t b1 = (uint32_t)(q8(vg[4 * j + 1], a.clip, a.sigma) & 0xff);
        uint32_t b2 = (uint32_t)(q8(vg[4 * j + 2], a.clip, a.sigma) & 0xff);
        uint32_t b3 = (uint32_t)(q8(vg[4 * j + 3], a.clip, a.sigma) & 0xff);
        w[j] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
      }
      *reinterpret_cast<uint4*>(a.out_q + (int64_t)row * a.ldo + ng) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

}  // namespace

template <int NV>
__global__ void __launch_bounds__(SK_THREADS, 1) k_step(const StepArgs s) {
  extern __shared__ uint8_t sk_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[SK_STAGES];
  __shared__ __align__(8) uint64_t empty_bar[SK_STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int32_t fin_warp_cnt[32];
  __shared__ int32_t fin_base;
  __shared__ int mt_live_s[2];
  __shared__ __align__(16) Phase sP;   // current phase descriptor (copied from global once)

  const uint32_t warp = warp_id(), lane = lane_id();
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sk_smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  double* scratch = reinterpret_cast<double*>(ring + SK_RING);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < SK_STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 8);   // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<SK_TMEM_COLS>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  unsigned gen = 0;
  if (s.cluster) {
    cluster_sync();
  } else {
    gen = ld_acquire_gpu(s.bar + 32);
    grid_sync(s.bar, gen);   // everybody has read the generation before anyone moves on
  }

  Pipe pp;   // each role only touches its own fields
  const int gwarp = blockIdx.x * SK_WARPS + warp;
  const int nwarps_all = gridDim.x * SK_WARPS;

  for (int step = 0; step < s.max_steps; ++step) {
    if (*reinterpret_cast<const volatile int32_t*>(s.ctrl) <= 0) break;   // uniform
    if (s.timing && blockIdx.x == 0 && threadIdx.x == 0)
      s.timing[(size_t)step * (s.n_phases + 1)] = globaltimer_ns();
    for (int ph = 0; ph < s.n_phases; ++ph) {
      {
        const int4* src = reinterpret_cast<const int4*>(s.phases + ph);
        int4* dst = reinterpret_cast<int4*>(&sP);
        for (int i = threadIdx.x; i < (int)(sizeof(Phase) / 16); i += blockDim.x) dst[i] = src[i];
      }
      __syncthreads();
      const Phase& P = sP;
      switch (P.type) {
        case PH_GEMM: {
          if (threadIdx.x == 0) {
            for (int p = 0; p < 2; ++p) {
              int mt = 0;
              if (p < P.nprob) {
                const GemmArgs& a = P.g[p].a;
                const int ml = a.M_dyn ? min(a.M, *a.M_dyn) : a.M;
                mt = (ml + SK_BM - 1) / SK_BM;
              }
              mt_live_s[p] = mt;
            }
          }
          __syncthreads();
          int p, m0, n0;
          if (warp == 0) {
            if (lane == 0) {
              fence_proxy_async();   // activations written by the previous phase -> TMA reads
              for (int k = 0; tile_k(P, mt_live_s, k, p, m0, n0); ++k) {
                const CUtensorMap* tmA = P.g[p].tmA;
                const CUtensorMap* tmB = P.g[p].tmB;
                const int bn = P.g[p].bn;
                const int nkb = (P.g[p].a.K + SK_BK - 1) / SK_BK;
                const uint32_t bytes = SK_A_BYTES + bn * SK_BK;
                for (int kb = 0; kb < nkb; ++kb) {
                  mbar_wait(&empty_bar[pp.ps], pp.pph ^ 1);
                  uint8_t* sa = ring + pp.ps * SK_STAGE;
                  uint8_t* sb = sa + SK_A_BYTES;
                  mbar_arrive_expect_tx(&full_bar[pp.ps], bytes);
                  tma_load_2d(sa, tmA, &full_bar[pp.ps], kb * SK_BK, m0);
                  tma_load_2d(sa + 64 * SK_BK, tmA, &full_bar[pp.ps], kb * SK_BK, m0 + 64);
                  for (int j = 0; j < bn / 64; ++j)
                    tma_load_2d(sb + j * 64 * SK_BK, tmB, &full_bar[pp.ps], kb * SK_BK, n0 + j * 64);
                  if (++pp.ps == SK_STAGES) { pp.ps = 0; pp.pph ^= 1; }
                }
              }
            }
          } else if (warp == 1) {
            if (lane == 0) {
              for (int k = 0; tile_k(P, mt_live_s, k, p, m0, n0); ++k) {
                const int nkb = (P.g[p].a.K + SK_BK - 1) / SK_BK;
                const uint32_t idesc = idesc_rt(P.g[p].bn);
                mbar_wait(&tempty_bar[pp.ab], pp.aph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + pp.ab * 256;
                for (int kb = 0; kb < nkb; ++kb) {
                  mbar_wait(&full_bar[pp.cs], pp.cph);
                  tc_fence_after();
                  const uint32_t sa = smem_u32(ring + pp.cs * SK_STAGE);
                  const uint64_t adesc = umma_desc_sw128(sa);
                  const uint64_t bdesc = umma_desc_sw128(sa + SK_A_BYTES);
#pragma unroll
                  for (int k = 0; k < SK_BK / 32; ++k)
                    mma_i8(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc,
                           (kb | k) != 0);
                  mma_commit(&empty_bar[pp.cs]);
                  if (++pp.cs == SK_STAGES) { pp.cs = 0; pp.cph ^= 1; }
                }
                mma_commit(&tfull_bar[pp.ab]);
                pp.ab ^= 1;
                if (pp.ab == 0) pp.aph ^= 1;
              }
            }
          } else if (warp >= 4) {
            const int q = warp & 3, half = (warp - 4) >> 2;
            bool wrote = false;
            for (int k = 0; tile_k(P, mt_live_s, k, p, m0, n0); ++k) {
              const GemmArgs a = P.g[p].a;     // registers: no reloads around global stores
              const int epi = P.g[p].epi;
              const int bn = P.g[p].bn;
              const int ml = a.M_dyn ? min(a.M, *a.M_dyn) : a.M;
              const int row = m0 + q * 32 + (int)lane;
              const bool row_ok = row < ml;
              mbar_wait(&tfull_bar[pp.ab], pp.aph);
              tc_fence_after();
              const int HALF = bn >> 1;
              const uint32_t t_row = tmem_base + pp.ab * 256 + ((uint32_t)(q * 32) << 16) + half * HALF;
              float best_v = -INFINITY;
              int best_j = -1;
              for (int c = 0; c < HALF; c += 32) {
                int32_t acc[32];
                tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
                tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
                tmem_ld_wait();
                epi_chunk(epi, a, row, row_ok, n0 + half * HALF + c, acc, best_v, best_j);
              }
              if (epi == EPI_ARGMAX && row_ok && best_j >= 0)
                atomicMax(a.keys + row, argmax_key(best_v, (uint32_t)best_j));
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty_bar[pp.ab]);
              pp.ab ^= 1;
              if (pp.ab == 0) pp.aph ^= 1;
              wrote = true;
            }
            if (wrote) fence_proxy_async();   // our global writes -> next phase's TMA reads
          }
          break;
        }
        case PH_EMBED: {
          const EmbedTgtArgs a = P.em;
          const int n_live = a.ctrl[0];
          if (P.rowlocal) {
            for (int t0 = blockIdx.x * SK_BM; t0 < n_live; t0 += gridDim.x * SK_BM)
              for (int r = t0 + (int)warp; r < min(n_live, t0 + SK_BM); r += SK_WARPS) embed_tgt_row<NV>(a, r);
          } else {
            for (int r = gwarp; r < n_live; r += nwarps_all) embed_tgt_row<NV>(a, r);
          }
          fence_proxy_async();
          break;
        }
        case PH_LN: {
          const LnArgs a = P.ln;
          const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
          if (P.rowlocal) {
            for (int t0 = blockIdx.x * SK_BM; t0 < n_live; t0 += gridDim.x * SK_BM)
              for (int r = t0 + (int)warp; r < min(n_live, t0 + SK_BM); r += SK_WARPS) ln_row<NV>(a, r);
          } else {
            for (int r = gwarp; r < n_live; r += nwarps_all) ln_row<NV>(a, r);
          }
          fence_proxy_async();
          break;
        }
        case PH_ATTN: {
          const AttnArgs a = P.at;
          const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
          const int total = n_live * a.H;
          for (int i = gwarp; i < total; i += nwarps_all) {
            const int r = i / a.H, h = i - r * a.H;
            attn_row_head(a, r, h, scratch + (size_t)warp * (MNMT_MAX_KV + 64), MNMT_MAX_KV);
          }
          fence_proxy_async();
          break;
        }
        case PH_FINISH: {
          if (blockIdx.x == 0) finish_block(P.fi, fin_warp_cnt, fin_base);
          __syncthreads();
          break;
        }
      }
      if (P.sync_grid) {
        if (s.cluster) {
          __syncwarp();
          cluster_sync();   // release/acquire at cluster scope orders the global writes too
        } else {
          grid_sync(s.bar, gen);
        }
      } else {
        fence_proxy_async();   // this CTA's global writes -> its own TMA reads in the next phase
        __syncthreads();
      }
      if (s.timing && blockIdx.x == 0 && threadIdx.x == 0)
        s.timing[(size_t)step * (s.n_phases + 1) + ph + 1] = globaltimer_ns();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<SK_TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ barrier microbenchmark
// mode 0: atomic counter + generation (as used);  mode 1: same without nanosleep;
// mode 2: per-CTA arrival flags (no contended atomic) gathered by CTA 0, generation release.
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_sync_flags(unsigned* flags, unsigned* genp, unsigned& gen) {
  __syncthreads();
  const unsigned g = gen + 1;
  if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * 32, g);   // one line per CTA
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    for (unsigned i = threadIdx.x; i < gridDim.x; i += 32)
      while (ld_acquire_gpu(flags + i * 32) < g) __nanosleep(0);
    __syncwarp();
    if (threadIdx.x == 0) st_release_gpu(genp, g);
  }
  if (threadIdx.x == 0)
    while (ld_acquire_gpu(genp) < g) {}
  gen = g;
  __syncthreads();
}

__global__ void k_barrier_bench(unsigned* bar, int mode, int iters, unsigned long long* out) {
  unsigned gen = ld_acquire_gpu(mode == 2 ? bar + 16384 : bar + 32);
  __syncthreads();
  grid_sync(bar, gen);
  if (mode == 2) gen = ld_acquire_gpu(bar + 16384);
  unsigned long long t0 = globaltimer_ns();
  for (int i = 0; i < iters; ++i) {
    if (mode == 2) {
      grid_sync_flags(bar + 4096, bar + 16384, gen);
    } else if (mode == 1) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned g = gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
          atomicExch(bar, 0u);
          __threadfence();
          atomicExch(bar + 32, g + 1);
        } else {
          while (ld_acquire_gpu(bar + 32) == g) {}
        }
        gen = g + 1;
      }
      __syncthreads();
    } else {
      grid_sync(bar, gen);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = (globaltimer_ns() - t0) / iters;
}

// ------------------------------------------------------------------ host side
int step_kernel_grid() {
  static int grid[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
  if (grid[dev]) return grid[dev];
  const void* fns[4] = {(const void*)k_step<1>, (const void*)k_step<2>, (const void*)k_step<4>,
                        (const void*)k_step<8>};
  for (const void* f : fns) {
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SK_SMEM) != cudaSuccess)
      return -1;
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaGetLastError();
  }
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step<2>, SK_THREADS, SK_SMEM) !=
          cudaSuccess ||
      per_sm < 1)
    return -1;
  grid[dev] = sms;   // one CTA per SM (smem use admits exactly one)
  return grid[dev];
}

cudaError_t launch_step_kernel(const StepArgs& a, int d, cudaStream_t st, int grid_cap) {
  int grid = step_kernel_grid();
  if (grid <= 0) return cudaErrorInvalidConfiguration;
  if (grid_cap > 0 && grid_cap < grid) grid = grid_cap;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SK_THREADS);
  cfg.dynamicSmemBytes = SK_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (a.cluster) {
    if (grid > 16) return cudaErrorInvalidConfiguration;
    attr[0].id = cudaLaunchAttributeClusterDimension;   // one cluster: co-scheduled by construction
    attr[0].val.clusterDim.x = grid;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int nv = (d / 4 + 31) / 32;
  switch (nv) {
    case 1: return cudaLaunchKernelEx(&cfg, k_step<1>, a);
    case 2: return cudaLaunchKernelEx(&cfg, k_step<2>, a);
    case 4: return cudaLaunchKernelEx(&cfg, k_step<4>, a);
    case 8: return cudaLaunchKernelEx(&cfg, k_step<8>, a);
  }
  return cudaErrorInvalidValue;
}


extern "C" long long mnmt_debug_barrier_ns(int mode, int iters) {
  unsigned* bar = nullptr;
  unsigned long long* out = nullptr;
  if (cudaMalloc(&bar, 65536 * 4) != cudaSuccess) return -1;
  cudaMemset(bar, 0, 65536 * 4);
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(SK_THREADS);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_barrier_bench, bar, mode, iters, out);
  unsigned long long ns = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
  cudaFree(bar);
  cudaFree(out);
  return e == cudaSuccess ? (long long)ns : -1;
}

}  // namespace mnmt
