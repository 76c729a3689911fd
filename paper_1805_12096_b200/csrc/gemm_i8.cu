// gemm_i8.cu — int8 x int8 -> s32 tensor-core GEMM for sm_100a (tcgen05.mma .kind::i8).
//
// Computes, for every product with a parameter, dotint(quant(A), quant(B^T)) = A . B^T
// with exact s32 accumulation (R3) and a fused epilogue
// fmaf((float)acc, s, b) (R5) followed by ReLU / quantization / sigmoid / argmax.
//
// Structure (one CTA per 128 x BN output tile, 10 warps):
//   warp 0      TMA producer: A tile [128 x 128B] + B tile [BN x 128B] per K-block into a
//               ring of min(K-blocks, STAGES) stages (128-byte swizzle), completion on
//               mbarriers.  The weight (B) tiles of the first stages are requested BEFORE
//               griddepcontrol.wait, overlapping the previous kernel (weights are constant);
//   warp 1      allocates BN TMEM columns, one lane issues 4 x tcgen05.mma
//               (M=128, N=BN, K=32) per K-block, tcgen05.commit frees the smem stage;
//   warps 2..9  epilogue: two warps per TMEM lane quarter (each half of the columns):
//               tcgen05.ld 32 lanes x 32 columns -> registers -> fused op -> HBM.
// Rows beyond the live-row count (M_dyn, read on device) are computed but never stored,
// and whole M-tiles beyond it exit before allocating TMEM.
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace mnmt {

constexpr int BM = 128;           // MMA M (rows of A per tile)
constexpr int BK = 128;           // K bytes per stage = one 128B swizzle atom row
constexpr int EPI_WARPS = 8;      // two warps per TMEM lane quarter, splitting the columns
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK;
  static constexpr int B_BYTES = BN * BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196 * 1024 / STAGE_BYTES) > 8 ? 8 : (196 * 1024 / STAGE_BYTES);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int smem_for(int stages) { return stages * STAGE_BYTES + 1024; }
};

template <int BN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[Cfg::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[Cfg::STAGES];
  __shared__ __align__(8) uint64_t tmem_full_bar;
  __shared__ uint32_t tmem_slot;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int n_tile = blockIdx.x, m_tile = blockIdx.y;
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  const int num_kb = (args.K + BK - 1) / BK;
  // ring depth chosen at launch (dynamic smem); at most Cfg::STAGES
  const int stages = min(Cfg::STAGES, num_kb);

  // 1024-byte aligned stage ring (required by the 128B swizzle atom).
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tmem_full_bar, 1);
    fence_barrier_init();
    // Weights are constant for the life of the model: fetch the first stages' B tiles
    // before waiting on the previous kernel (programmatic dependent launch).
    for (int s = 0; s < stages; ++s) {
      mbar_arrive_expect_tx(&full_bar[s], Cfg::STAGE_BYTES);
      uint8_t* sb = smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES;
#pragma unroll
      for (int j = 0; j < BN / 64; ++j)
        tma_load_2d(sb + j * 64 * BK, &tmB, &full_bar[s], s * BK, n0 + j * 64);
    }
  }
  pdl_wait();   // everything below may read the previous kernel's outputs
  const int M_live = args.M_dyn ? min(args.M, *args.M_dyn) : args.M;
  if (m0 >= M_live) {
    // Tile has no live rows.  Complete the in-flight weight copies before leaving.
    if (warp == 0 && lane == 0) {
      for (int s = 0; s < stages; ++s) {
        uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
        tma_load_2d(sa, &tmA, &full_bar[s], s * BK, m0);
        tma_load_2d(sa + 64 * BK, &tmA, &full_bar[s], s * BK, m0 + 64);
      }
      for (int s = 0; s < stages; ++s) mbar_wait(&full_bar[s], 0);
    }
    return;
  }

  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % stages;
        uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        if (kb >= stages) {
          mbar_wait(&empty_bar[s], ((kb / stages) - 1) & 1);
          mbar_arrive_expect_tx(&full_bar[s], Cfg::STAGE_BYTES);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(sb + j * 64 * BK, &tmB, &full_bar[s], kb * BK, n0 + j * 64);
        }
        tma_load_2d(sa, &tmA, &full_bar[s], kb * BK, m0);
        tma_load_2d(sa + 64 * BK, &tmA, &full_bar[s], kb * BK, m0 + 64);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      constexpr uint32_t idesc = idesc_i8<BM, BN>();
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % stages;
        mbar_wait(&full_bar[s], (kb / stages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t sb = sa + Cfg::A_BYTES;
        const uint64_t adesc = umma_desc_sw128(sa);
        const uint64_t bdesc = umma_desc_sw128(sb);
#pragma unroll
        for (int k = 0; k < BK / 32; ++k) {
          // advance the start address by k * 32 bytes (encoded >> 4) inside the swizzle atom
          mma_i8(tmem_base, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc,
                 (kb | k) != 0);
        }
        mma_commit(&empty_bar[s]);  // smem stage free once these MMAs have read it
      }
      mma_commit(&tmem_full_bar);   // accumulator complete
    }
  } else {
    // ---------------- epilogue: warps 2..9; TMEM lane quarter = warp % 4 (hardware rule),
    // column half = (warp - 2) / 4.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < M_live;
    constexpr int HALF = BN / 2;
    mbar_wait(&tmem_full_bar, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) pdl_launch_dependents();
    const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + half * HALF;
    float best_v = -INFINITY;
    int best_j = -1;
#pragma unroll 1
    for (int c = 0; c < HALF; c += 32) {
      int32_t acc[32];
      tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
      tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
      tmem_ld_wait();
      const int n = n0 + half * HALF + c;
      if (n >= args.N) break;  // warp-uniform
      if constexpr (EPI == EPI_ARGMAX) {
        // strict '>' over increasing columns keeps the lowest column among equal logits (R15)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (n + j < args.N) {
            const float b = args.bias ? __ldg(args.bias + n + j) : 0.0f;
            const float v = dequant(acc[j], args.scale, b);
            if (v > best_v) { best_v = v; best_j = n + j; }
          }
        }
      } else if constexpr (EPI == EPI_ACC) {
        if (row_ok) {
          int4* dst = reinterpret_cast<int4*>(args.out_i + (int64_t)row * args.ldo + n);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (n + 4 * j < args.N)
              dst[j] = make_int4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
        }
      } else {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float b = (args.bias && n + j < args.N) ? __ldg(args.bias + n + j) : 0.0f;
          v[j] = dequant(acc[j], args.scale, b);
          if constexpr (EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) v[j] = relu(v[j]);
          if constexpr (EPI == EPI_SIGMOID) v[j] = sigmoid_f64(v[j]);
        }
        if (row_ok) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {          // two 16-column groups (N % 16 == 0)
            const int ng = n + 16 * g;
            if (ng >= args.N) break;
            const float* vg = v + 16 * g;
            if constexpr (EPI == EPI_F32 || EPI == EPI_F32_Q || EPI == EPI_RELU_F32_Q ||
                          EPI == EPI_SIGMOID) {
              const int blk = ng / args.col_block;
              float* dst = args.out_f + (int64_t)blk * args.block_stride +
                           (int64_t)row * args.ldo + (ng - blk * args.col_block);
              float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                d4[j] = make_float4(vg[4 * j], vg[4 * j + 1], vg[4 * j + 2], vg[4 * j + 3]);
            }
            if constexpr (EPI == EPI_F32_Q || EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) {
              uint32_t w[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint32_t b0 = (uint32_t)(q8(vg[4 * j + 0], args.clip, args.sigma) & 0xff);
                uint32_t b1 = (uint32_t)(q8(vg[4 * j + 1], args.clip, args.sigma) & 0xff);
                uint32_t b2 = (uint32_t)(q8(vg[4 * j + 2], args.clip, args.sigma) & 0xff);
                uint32_t b3 = (uint32_t)(q8(vg[4 * j + 3], args.clip, args.sigma) & 0xff);
                w[j] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
              }
              *reinterpret_cast<uint4*>(args.out_q + (int64_t)row * args.ldo + ng) =
                  make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      }
    }
    if constexpr (EPI == EPI_ARGMAX) {
      if (row_ok && best_j >= 0) atomicMax(args.keys + row, argmax_key(best_v, (uint32_t)best_j));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_tmap_i8(CUtensorMap* map, const void* base, int64_t rows, int64_t K) {
  auto enc = get_encode();
  if (!enc || K % 16 != 0 || rows < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {(cuuint32_t)BK, 64u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MNMT_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

int gemm_pick_bn(int M, int N) {
  const int mt = (M + BM - 1) / BM;
  if (((N + 255) / 256) * mt >= 148) return 256;
  if (((N + 127) / 128) * mt >= 74) return 128;
  return 64;
}

template <int BN, int EPI>
static cudaError_t launch_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                            cudaStream_t st) {
  using Cfg = GemmCfg<BN>;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  const int num_kb = (a.K + BK - 1) / BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg::smem_for(num_kb < Cfg::STAGES ? num_kb : Cfg::STAGES);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_i8<BN, EPI>, tmA, tmB, a);
}

template <int BN, int EPI>
static cudaError_t set_attr() {
  return cudaFuncSetAttribute(k_gemm_i8<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GemmCfg<BN>::smem_for(GemmCfg<BN>::STAGES));
}
template <int BN>
static cudaError_t set_attr_bn() {
  cudaError_t e;
  if ((e = set_attr<BN, EPI_F32>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, EPI_F32_Q>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, EPI_RELU_Q>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, EPI_RELU_F32_Q>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, EPI_SIGMOID>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, EPI_ARGMAX>()) != cudaSuccess) return e;
  return set_attr<BN, EPI_ACC>();
}

static cudaError_t gemm_init_all();

// Opt every GEMM instantiation into its dynamic shared memory size on the current
// device (once per device).  Must run before any launch (never inside a stream capture).
cudaError_t gemm_init() {
  static bool done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  e = gemm_init_all();
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

static cudaError_t gemm_init_all() {
  cudaError_t e;
  if ((e = set_attr_bn<64>()) != cudaSuccess) return e;
  if ((e = set_attr_bn<128>()) != cudaSuccess) return e;
  return set_attr_bn<256>();
}

template <int BN>
static cudaError_t launch_bn(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                             int epi, cudaStream_t st) {
  switch (epi) {
    case EPI_F32: return launch_t<BN, EPI_F32>(tmA, tmB, a, st);
    case EPI_F32_Q: return launch_t<BN, EPI_F32_Q>(tmA, tmB, a, st);
    case EPI_RELU_Q: return launch_t<BN, EPI_RELU_Q>(tmA, tmB, a, st);
    case EPI_RELU_F32_Q: return launch_t<BN, EPI_RELU_F32_Q>(tmA, tmB, a, st);
    case EPI_SIGMOID: return launch_t<BN, EPI_SIGMOID>(tmA, tmB, a, st);
    case EPI_ARGMAX: return launch_t<BN, EPI_ARGMAX>(tmA, tmB, a, st);
    case EPI_ACC: return launch_t<BN, EPI_ACC>(tmA, tmB, a, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemm_i8(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                           int epi, int bn, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return cudaSuccess;
  if (bn == 0) bn = gemm_pick_bn(a.M, a.N);
  switch (bn) {
    case 64: return launch_bn<64>(tmA, tmB, a, epi, st);
    case 128: return launch_bn<128>(tmA, tmB, a, epi, st);
    case 256: return launch_bn<256>(tmA, tmB, a, epi, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mnmt
