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
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"
#include "rowdev.cuh"

namespace mnmt {

static int num_sms();
bool gemm_persistent(int M, int N, int bn, int sms = 0);

constexpr int BM = 128;           // MMA M (rows of A per tile)
constexpr int BK = 128;           // K bytes per stage = one 128B swizzle atom row
constexpr int EPI_WARPS = 8;      // two warps per TMEM lane quarter, splitting the columns
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_STAGE_LD = 36;                       // row stride (floats): 16-byte rows, and
                                                       // conflict-free STS.128 / LDS.128
constexpr int EPI_STAGE_FLOATS = 32 * EPI_STAGE_LD;    // per epilogue warp
constexpr int EPI_STAGE_BYTES = EPI_WARPS * EPI_STAGE_FLOATS * 4;
constexpr int GEMM_SMEM_MAX = 220 * 1024;                // dynamic smem cap of a split-K launch

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK;
  static constexpr int B_ROWS = BN < 64 ? 64 : BN;   // TMA box is 64 rows: BN = 32 loads 64
  static constexpr int B_BYTES = B_ROWS * BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (190 * 1024 / STAGE_BYTES) > 8 ? 8 : (190 * 1024 / STAGE_BYTES);
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int smem_for(int stages) { return stages * STAGE_BYTES + 1024 + EPI_STAGE_BYTES; }
  // split-K (gridDim.z > 1, one cluster along z): CTA z > 0 stores its s32 partial tile into
  // slot z - 1 of CTA 0's buffer [ks - 1][128][BN + 4]; CTA 0 adds the slots (exact integers)
  static constexpr int RED_LD = BN + 4;
  static constexpr int RED_SLOT_BYTES = BM * RED_LD * 4;
};

// 16-byte store into another CTA's shared memory (distributed shared memory).
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, int32_t a, int32_t b, int32_t c, int32_t d) {
  asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d) : "memory");
}

// Exact (float)acc for |acc| < 2^22 without the quarter-rate I2F: place acc in the
// mantissa of 1.5 * 2^23 and subtract.  Used when K <= 256 (|acc| <= 127^2 * 256 < 2^22).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// debug trace (GemmArgs::trace): CTA (0,0) records entry, after the PDL wait, operands landed,
// accumulator complete, epilogue done
#define GEMM_TRACE(i)                                                              \
  do {                                                                             \
    if (args.trace && blockIdx.x == 0 && blockIdx.y == 0) args.trace[i] = gtimer(); \
  } while (0)

__device__ __forceinline__ float acc_to_float(int32_t acc, bool small) {
  return small ? __fsub_rn(__int_as_float(0x4B400000 + acc), 12582912.0f) : __int2float_rn(acc);
}


// Packed fp32 pairs (sm_100a FFMA2 / FADD2): each half is one IEEE round-to-nearest op.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}

// v[j] = fmaf((float)acc[j], s, bias[j]) for one 32-column chunk.
// Fast path (K <= 256, whole chunk in range): exact magic-number conversion + packed ops.
// bsrc: the bias indexed by global column (args.bias, or the CTA's shared-memory copy shifted by
// its first column) or null.
template <int CW = 32>
__device__ __forceinline__ void dequant32(const GemmArgs& args, const float* bsrc, int n, bool fast,
                                          const int32_t (&acc)[32], float (&v)[32]) {
  if (fast) {
    float bias[32];
    if (bsrc) {
#pragma unroll
      for (int j = 0; j < CW; j += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(bsrc + n + j);
        bias[j] = b4.x; bias[j + 1] = b4.y; bias[j + 2] = b4.z; bias[j + 3] = b4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < CW; ++j) bias[j] = 0.0f;
    }
    const unsigned long long negc = pk2(-12582912.0f, -12582912.0f);
    const unsigned long long s2 = pk2(args.scale, args.scale);
#pragma unroll
    for (int j = 0; j < CW; j += 2) {
      unsigned long long t = pk2(__int_as_float(0x4B400000 + acc[j]), __int_as_float(0x4B400000 + acc[j + 1]));
      asm("add.rn.f32x2 %0, %0, %1;" : "+l"(t) : "l"(negc));
      unsigned long long r;
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(t), "l"(s2), "l"(pk2(bias[j], bias[j + 1])));
      upk2(r, v[j], v[j + 1]);
    }
  } else {
    const bool small = args.K <= 256;
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const float b = (bsrc && n + j < args.N) ? bsrc[n + j] : 0.0f;
      v[j] = __fmaf_rn(acc_to_float(acc[j], small), args.scale, b);
    }
  }
}

// Shortlist (F2): the row's group words for the HALF columns from nb (one 32-bit word per
// 32-column chunk, zero past N), so the epilogue masks with no further loads.
template <int HALF>
__device__ __forceinline__ void sl_words(const GemmArgs& args, int row, bool row_ok, int nb,
                                         uint32_t (&w)[HALF / 32]) {
  if (!args.colbits) {
#pragma unroll
    for (int c = 0; c < HALF / 32; ++c) w[c] = 0xffffffffu;
    return;
  }
  const int g = row_ok ? args.row_grp[args.row_live ? args.row_live[row] : row] : 0;
  const uint32_t* gb = args.colbits + (int64_t)g * args.colbits_ld;
#pragma unroll
  for (int c = 0; c < HALF / 32; ++c) {
    const int n = nb + c * 32;
    w[c] = n < args.N ? gb[n >> 5] : 0u;
  }
}

// One 32-column chunk of the 32 rows of this warp (lane = row): dequant + fused op +
// store, or running argmax.  fp32 outputs go through a padded per-warp smem tile so each
// store instruction writes four full 128-byte lines.
template <int EPI, int CW = 32>
__device__ __forceinline__ void epi_store_chunk(const GemmArgs& args, const float* bsrc, int row,
                                                bool row_ok, int n, const int32_t (&acc)[32],
                                                float& best_v, int& best_j, float* stage,
                                                uint32_t slw = 0xffffffffu) {
  static_assert(CW == 32 || (CW == 16 && EPI != EPI_ARGMAX && EPI != EPI_ACC),
                "16-column chunks: the fp32 / code epilogues only");
  const bool full = n + CW <= args.N;
  const bool fast = full && args.K <= 256;
  if constexpr (EPI == EPI_ARGMAX) {
    // Branch-free chunk maximum; the lowest column holding it is searched only when the
    // chunk beats the running best, and a strictly greater value is required, so among
    // equal logits the lowest column wins (R15).
    float v[32];
    dequant32(args, bsrc, n, fast, acc, v);
    if (args.colbits) {   // shortlist union: only the columns of the row's own batch (F2);
      // slw = the row's group word of this chunk (zero past N), loaded before the MMA wait
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (!((slw >> j) & 1u)) v[j] = -INFINITY;
    } else if (!full) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n + j >= args.N) v[j] = -INFINITY;
    }
    float m[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) m[j] = fmaxf(v[j], v[j + 16]);
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
      for (int j = 0; j < w; ++j) m[j] = fmaxf(m[j], m[j + w]);
    if (m[0] > best_v) {
      int jj = 31;
#pragma unroll
      for (int j = 31; j >= 0; --j) jj = (v[j] == m[0]) ? j : jj;
      best_v = m[0];
      best_j = n + jj;
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
    dequant32<CW>(args, bsrc, n, fast, acc, v);
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      if constexpr (EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) v[j] = relu(v[j]);
      if constexpr (EPI == EPI_SIGMOID) v[j] = sigmoid_f64(v[j]);
    }
    if constexpr (EPI == EPI_F32 || EPI == EPI_F32_Q || EPI == EPI_RELU_F32_Q || EPI == EPI_SIGMOID) {
      // stage [32 rows][CW cols] then write rows cooperatively (CW / 4 lanes x float4 per row)
      const int lane = threadIdx.x & 31;
      if (threadIdx.x == 64) GEMM_TRACE(7);   // warp 2 lane 0: dequant done
      const unsigned okm = __ballot_sync(0xffffffffu, row_ok);   // live rows of this warp
#pragma unroll
      for (int j = 0; j < CW; j += 4)
        *reinterpret_cast<float4*>(stage + lane * EPI_STAGE_LD + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      __syncwarp();
      if (threadIdx.x == 64) GEMM_TRACE(8);   // staged
      const int row0 = row - lane;
      const int blk = n / args.col_block;   // chunks never straddle a block (16 | col_block)
      float* base = args.out_f + (int64_t)blk * args.block_stride + (n - blk * args.col_block);
      constexpr int LPR = CW / 4, RPI = 32 / LPR;   // lanes per row, rows per store instruction
      constexpr unsigned GM = (1u << RPI) - 1u;
      const int sub = lane / LPR, c4 = (lane % LPR) * 4;
#pragma unroll
      for (int it = 0; it < 32 / RPI; ++it) {
        if (((okm >> (RPI * it)) & GM) == 0) continue;   // warp-uniform: no live row in the group
        const int r = it * RPI + sub;
        if (((okm >> r) & 1u) && n + c4 < args.N)
          *reinterpret_cast<float4*>(base + (int64_t)(row0 + r) * args.ldo + c4) =
              *reinterpret_cast<const float4*>(stage + r * EPI_STAGE_LD + c4);
      }
      __syncwarp();
    }
    if constexpr (EPI == EPI_F32_Q || EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) {
      if (row_ok) {
#pragma unroll
        for (int g = 0; g < CW / 16; ++g) {    // 16-column groups (N % 16 == 0)
          const int ng = n + 16 * g;
          if (ng >= args.N) break;
          const float* vg = v + 16 * g;
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


// EPI_TOPK* (beam search, F1): one 32-column chunk at a time, the row's running maximum m,
// the fp64 sum z = sum exp(v - m) (rescaled by exp(m_old - m_new) when a chunk raises m) and
// the TK largest (v, column) in descending v, ascending column on ties (columns arrive in
// ascending order and only a strictly larger value displaces an entry).
__host__ __device__ constexpr bool is_topk(int epi) {
  return epi == EPI_TOPK || epi == EPI_TOPK2 || epi == EPI_TOPK4;
}
__host__ __device__ constexpr int topk_k(int epi) {
  return epi == EPI_TOPK2 ? 2 : epi == EPI_TOPK4 ? 4 : TOPK_MAX;
}

// 2^(i/64), i = 0..63, correctly rounded (staged in shared memory by the TOPK epilogue)
__device__ const double c_exp2_64[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284, 1.0442737824274138,
    1.0556451783605572, 1.0671404006768237, 1.0787607977571199, 1.0905077326652577,
    1.102382583307841, 1.1143867425958924, 1.1265216186082418, 1.1387886347566916,
    1.1511892299529827, 1.1637248587775775, 1.1763969916502812, 1.189207115002721,
    1.202156731452703, 1.215247359980469, 1.22848053610687, 1.241857812073484,
    1.255380757024691, 1.2690509571917332, 1.2828700160787783, 1.2968395546510096,
    1.3109612115247644, 1.3252366431597413, 1.339667524053303, 1.3542555469368927,
    1.3690024229745905, 1.383909881963832, 1.3989796725383112, 1.4142135623730951,
    1.42961333839197, 1.4451808069770467, 1.460917794180647, 1.4768261459394993,
    1.4929077282912648, 1.5091644275934228, 1.5255981507445384, 1.5422108254079407,
    1.559004400237837, 1.5759808451078865, 1.593142151342267, 1.6104903319492543,
    1.6280274218573478, 1.645755478153965, 1.6636765803267364, 1.681792830507429,
    1.7001063537185235, 1.718619298122478, 1.7373338352737062, 1.7562521603732995,
    1.7753764925265212, 1.7947090750031072, 1.8142521755003989, 1.8340080864093424,
    1.8539791250833855, 1.8741676341103, 1.8945759815869656, 1.9152065613971474,
    1.9360617934922943, 1.9571441241754002, 1.978456026387951};

// exp(x) for x <= 0 in fp64 (relative error ~2 ulp; R26): x = k ln2/64 + r with |r| <= ln2/128,
// exp(x) = 2^floor(k/64) * 2^((k mod 64)/64) * e^r, e^r by its degree-5 Taylor polynomial
// (truncation < 4e-17).  k ln2/64 is split hi (32 significant bits, so k*hi is exact) + lo.
// x < -707: 0 (the sums it feeds are >= 1, so such terms are far below their last bit).
__device__ __forceinline__ double exp_neg(double x, const double* tab) {
  if (x < -707.0) return 0.0;
  const double kd = rint(x * 92.33248261689366);          // 64 / ln2
  double r = fma(kd, -0.01083042469326756, x);             // ln2/64, high 32 bits
  r = fma(kd, -2.9815858269852933e-12, r);                 // ln2/64, low part
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = (int)kd;
  const double v = p * tab[k & 63];
  // multiply by 2^(k >> 6) through the exponent field (v in [0.99, 2), result normal)
  return __hiloint2double(__double2hiint(v) + ((k >> 6) << 20), __double2loint(v));
}

template <int BN, int TK>
__device__ __forceinline__ void topk_epilogue(const GemmArgs& args, const float* bsrc, uint32_t t_row,
                                              int row, bool row_ok, int half, int n0,
                                              const double* tab) {
  constexpr int HALF = BN / 2;
  float tv[TK];
  int tj[TK];
#pragma unroll
  for (int i = 0; i < TK; ++i) { tv[i] = -INFINITY; tj[i] = -1; }
  float run_m = -INFINITY;
  double z = 0.0;
#pragma unroll 1
  for (int c = 0; c < HALF; c += 32) {
    int32_t acc[32];
    tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
    tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
    tmem_ld_wait();
    const int n = n0 + half * HALF + c;
    if (n >= args.N) break;   // warp-uniform
    const bool full = n + 32 <= args.N;
    float v[32];
    dequant32(args, bsrc, n, full && args.K <= 256, acc, v);
    if (!full) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n + j >= args.N) v[j] = -INFINITY;
    }
    float cm = v[0];
#pragma unroll
    for (int j = 1; j < 32; ++j) cm = fmaxf(cm, v[j]);
    if (cm > run_m) {
      if (run_m != -INFINITY) z = __dmul_rn(z, exp_neg(__dsub_rn((double)run_m, (double)cm), tab));
      run_m = cm;
    }
    // four independent partial sums (columns j mod 4), combined in a fixed order
    const double md = (double)run_m;
    double zp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (v[j] != -INFINITY) zp[j & 3] = __dadd_rn(zp[j & 3], exp_neg(__dsub_rn((double)v[j], md), tab));
    z = __dadd_rn(z, __dadd_rn(__dadd_rn(zp[0], zp[1]), __dadd_rn(zp[2], zp[3])));
    if (cm > tv[TK - 1]) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (v[j] > tv[TK - 1]) {
          float cv = v[j];
          int cj = n + j;
          bool sh = false;
#pragma unroll
          for (int i = 0; i < TK; ++i) {
            const bool take = sh || cv > tv[i];
            const float ov = tv[i];
            const int oj = tj[i];
            tv[i] = take ? cv : ov;
            tj[i] = take ? cj : oj;
            cv = take ? ov : cv;
            cj = take ? oj : cj;
            sh = take;
          }
        }
      }
    }
  }
  if (row_ok) {
    TopkPart* p = args.part + (int64_t)row * args.part_ld + blockIdx.x * 2 + half;
    p->m = run_m;
    p->pad = 0;
    p->z = z;
#pragma unroll
    for (int i = 0; i < TOPK_MAX; ++i) {
      p->v[i] = i < TK ? tv[i < TK ? i : 0] : -INFINITY;
      p->j[i] = i < TK ? tj[i < TK ? i : 0] : -1;
    }
  }
}

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
  __shared__ double exp_tab[is_topk(EPI) ? 64 : 1];   // 2^(i/64) for exp_neg (EPI_TOPK*)
  __shared__ __align__(16) float bias_s[BN];   // the tile's bias, staged before the PDL wait

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int n_tile = blockIdx.x, m_tile = blockIdx.y;
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  // split-K: the ks CTAs of a cluster (along z) take consecutive K-block ranges; CTA z = 0
  // reduces (launch_t guarantees every range is non-empty)
  const int ks = gridDim.z, kz = blockIdx.z;
  const int kb_all = (args.K + BK - 1) / BK, kb_per = (kb_all + ks - 1) / ks;
  const int kb0 = kz * kb_per;
  const int num_kb = min(kb_all, kb0 + kb_per) - kb0;
  // ring depth chosen at launch (dynamic smem; the same layout in every CTA of a cluster)
  const int ring = min(min(Cfg::STAGES, kb_per), args.ring_cap > 0 ? args.ring_cap : Cfg::STAGES);
  const int stages = min(ring, num_kb);
  if (threadIdx.x == 0) GEMM_TRACE(0);

  // 1024-byte aligned stage ring (required by the 128B swizzle atom).
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  int32_t* red = reinterpret_cast<int32_t*>(smem + ring * Cfg::STAGE_BYTES + EPI_STAGE_BYTES);
  if (ks > 1) cluster_arrive_relaxed();   // phase 1: this CTA is running (DSMEM valid)

  // a_box > 0: tmA holds one a_box-row box per K block (a_box < 128: the launch's a.M <= 64 rows;
  // the rest of the A tile stays stale, those accumulator rows are never stored); b_box > 0: tmB
  // holds one b_box-row box (BN = 32: 32 rows; else the whole B tile).  Otherwise 64-row boxes.
  // boxes (BN = 32 loads only its own weight rows)
  const int a_bytes = args.a_box > 0 ? args.a_box * BK : Cfg::A_BYTES;
  const int b_bytes = args.b_box > 0 ? args.b_box * BK : Cfg::B_BYTES;
  const int tx_bytes = a_bytes + b_bytes;
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
      mbar_arrive_expect_tx(&full_bar[s], tx_bytes);
      uint8_t* sb = smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES;
      if (args.b_box > 0) {
        tma_load_2d(sb, &tmB, &full_bar[s], (kb0 + s) * BK, n0);
      } else {
#pragma unroll
        for (int j = 0; j < Cfg::B_ROWS / 64; ++j)
          tma_load_2d(sb + j * 64 * BK, &tmB, &full_bar[s], (kb0 + s) * BK, n0 + j * 64);
      }
    }
  }
  // TMEM and the bias do not depend on the previous kernel either: both before the wait
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(&tmem_slot);
  if constexpr (is_topk(EPI)) {
    if (warp >= 2 && threadIdx.x - 64 < 64) exp_tab[threadIdx.x - 64] = c_exp2_64[threadIdx.x - 64];
  }
  if (args.bias && warp >= 2)
    for (int i = (int)threadIdx.x - 64; i < BN; i += 32 * EPI_WARPS)
      bias_s[i] = n0 + i < args.N ? __ldg(args.bias + n0 + i) : 0.0f;
  if (args.npsync) {   // the CTA barrier before the PDL wait (as the persistent kernel; A/B)
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  pdl_wait();   // everything below may read the previous kernel's outputs
  if (threadIdx.x == 0) GEMM_TRACE(1);
  // The A tiles of the first ring stages are requested right away, in parallel with the
  // live-row read (rows beyond it are loaded but never stored; an idle tile drains them).
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
      tma_load_2d(sa, &tmA, &full_bar[s], (kb0 + s) * BK, m0);
      if (args.a_box == 0) tma_load_2d(sa + 64 * BK, &tmA, &full_bar[s], (kb0 + s) * BK, m0 + 64);
    }
  }
  const int M_live = args.M_dyn ? min(args.M, *args.M_dyn) : args.M;
  if (m0 >= M_live) {   // (uniform over a split-K cluster: one M tile)
    // Tile has no live rows.  Complete the in-flight copies before leaving.
    if (warp == 0 && lane == 0)
      for (int s = 0; s < stages; ++s) mbar_wait(&full_bar[s], 0);
    __syncwarp();   // bar.sync is .aligned: reconverge warp 0 after its single-lane work
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_slot);
    return;
  }

  if (!args.npsync) {
    __syncwarp();   // (compute-sanitizer synccheck: divergent warp 0 at the barrier otherwise)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t tmem_base = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (stages 0..stages-1 were issued above)
      for (int kb = stages; kb < num_kb; ++kb) {
        const int s = kb % stages;
        uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        mbar_wait(&empty_bar[s], ((kb / stages) - 1) & 1);
        mbar_arrive_expect_tx(&full_bar[s], tx_bytes);
        if (args.b_box > 0) {
          tma_load_2d(sb, &tmB, &full_bar[s], (kb0 + kb) * BK, n0);
        } else {
#pragma unroll
          for (int j = 0; j < Cfg::B_ROWS / 64; ++j)
            tma_load_2d(sb + j * 64 * BK, &tmB, &full_bar[s], (kb0 + kb) * BK, n0 + j * 64);
        }
        tma_load_2d(sa, &tmA, &full_bar[s], (kb0 + kb) * BK, m0);
        if (args.a_box == 0) tma_load_2d(sa + 64 * BK, &tmA, &full_bar[s], (kb0 + kb) * BK, m0 + 64);
      }
    }
    __syncwarp();
    if (ks > 1) {   // phase 1 wait + phase 2 (partials added) of the split-K exchange
      cluster_wait();
      cluster_arrive();
      cluster_wait();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp walks the K blocks (warp-uniform, so the
    // descriptors live in uniform registers), one elected lane issues the MMAs and their commits
    // (measured: 100-107 -> 72-82 cycles per tcgen05.mma with the per-K-block bookkeeping,
    // profiles/r2_mma_issue_bench.txt; small-N MMAs are issue-bound)
    constexpr uint32_t idesc = idesc_i8<BM, BN>();
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % stages;
      mbar_wait(&full_bar[s], (kb / stages) & 1);
      if (kb == 0 && lane == 0) GEMM_TRACE(2);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
      const uint32_t sb = sa + Cfg::A_BYTES;
      const uint64_t adesc = umma_desc_sw128(sa);
      const uint64_t bdesc = umma_desc_sw128(sb);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BK / 32; ++k) {
          // advance the start address by k * 32 bytes (encoded >> 4) inside the swizzle atom
          mma_i8(tmem_base, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc,
                 (kb | k) != 0);
        }
        mma_commit(&empty_bar[s]);  // smem stage free once these MMAs have read it
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&tmem_full_bar);   // accumulator complete
    __syncwarp();
    if (ks > 1) {
      cluster_wait();
      cluster_arrive();
      cluster_wait();
    }
  } else {
    // ---------------- epilogue: warps 2..9; TMEM lane quarter = warp % 4 (hardware rule),
    // column half = (warp - 2) / 4.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < M_live;
    constexpr int HALF = BN / 2;
    constexpr int CW = HALF < 32 ? 16 : 32;   // chunk width (BN = 32: 16 columns per warp)
    uint32_t slw[HALF >= 32 ? HALF / 32 : 1];
    if constexpr (EPI == EPI_ARGMAX) sl_words<HALF>(args, row, row_ok, n0 + half * HALF, slw);
    mbar_wait(&tmem_full_bar, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) GEMM_TRACE(3);
    // dependents launch once the accumulator is complete (measured: at entry is slower, and
    // from the MMA warp after its last commit no different)
    if (warp == 2 && lane == 0) pdl_launch_dependents();
    const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + half * HALF;
    float* stage = reinterpret_cast<float*>(smem + ring * Cfg::STAGE_BYTES) +
                   (warp - 2) * EPI_STAGE_FLOATS;
    float best_v = -INFINITY;
    int best_j = -1;
    const int rl = q * 32 + lane;   // row within the tile (TMEM lane)
    if (ks > 1) {
      // split-K exchange: CTAs z > 0 add the live lane quarters of their partial accumulators
      // into the leader's buffer; the leader adds the buffer to its own before the epilogue
      __syncwarp();
      cluster_wait();   // phase 1: every CTA of the cluster is running
      if (kz > 0 && m0 + q * 32 < M_live) {
        constexpr int CWX = HALF < 32 ? 16 : 32;
        const uint32_t base = mapa_shared(
            smem_u32(red + (kz - 1) * (Cfg::RED_SLOT_BYTES / 4) + rl * Cfg::RED_LD + half * HALF), 0);
#pragma unroll 1
        for (int c = 0; c < HALF; c += CWX) {
          int32_t acc[32];
          tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
          if constexpr (CWX == 32) tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CWX; j += 4)
            st_cluster_v4(base + 4 * (c + j), acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        }
      }
      __syncwarp();
      cluster_arrive();   // phase 2 (release): partials added
      cluster_wait();
    }
    if (ks > 1 && kz > 0) {
      // partials delivered; nothing to store
    } else if constexpr (is_topk(EPI)) {
      topk_epilogue<BN, topk_k(EPI)>(args, args.bias ? bias_s - n0 : nullptr, t_row, row, row_ok,
                                     half, n0, exp_tab);
    } else
#pragma unroll 1
    for (int c = 0; c < HALF; c += CW) {
      int32_t acc[32];
      tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
      if constexpr (CW == 32) tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
      tmem_ld_wait();
      if (ks > 1) {   // + the other K ranges' partials (exact s32)
        for (int z = 1; z < ks; ++z) {
          const int4* rp = reinterpret_cast<const int4*>(red + (z - 1) * (Cfg::RED_SLOT_BYTES / 4) +
                                                         rl * Cfg::RED_LD + half * HALF + c);
#pragma unroll
          for (int j = 0; j < CW / 4; ++j) {
            const int4 p = rp[j];
            acc[4 * j] += p.x; acc[4 * j + 1] += p.y; acc[4 * j + 2] += p.z; acc[4 * j + 3] += p.w;
          }
        }
      }
      if (c == 0 && warp == 2 && lane == 0) GEMM_TRACE(6);
      const int n = n0 + half * HALF + c;
      if (n >= args.N) break;  // warp-uniform
      if constexpr (CW == 32)
        epi_store_chunk<EPI>(args, args.bias ? bias_s - n0 : nullptr, row, row_ok, n, acc, best_v,
                             best_j, stage, EPI == EPI_ARGMAX ? slw[c / 32] : 0u);
      else
        epi_store_chunk<EPI, 16>(args, args.bias ? bias_s - n0 : nullptr, row, row_ok, n, acc,
                                 best_v, best_j, stage);
    }
    if constexpr (EPI == EPI_ARGMAX) {
      if (row_ok && best_j >= 0) atomicMax(args.keys + row, argmax_key(best_v, (uint32_t)best_j));
    }
    (void)rl;
    if (warp == 2 && lane == 0) GEMM_TRACE(4);   // this warp's stores issued
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  if (warp == 1 && lane == 0) GEMM_TRACE(5);     // after the barrier and the dealloc
}

// ------------------------------------------------------------------ persistent variant
// For large problems (encoder GEMMs at tens of thousands of rows, the output layer at
// thousands of rows): one CTA per SM loops over 128 x BN tiles (n fastest, so consecutive
// tiles share the A tile in L2).  Two TMEM accumulators (2 x BN columns) let the
// epilogue of tile i overlap the MMAs of tile i+1; the TMA ring keeps streaming across
// tile boundaries.  Same numerics and epilogues as k_gemm_i8.
template <int BN>
struct PersCfg {
  static constexpr int A_BYTES = BM * BK;
  static constexpr int STAGE_BYTES = A_BYTES + BN * BK;
  static constexpr int STAGES = (190 * 1024 / STAGE_BYTES) > 8 ? 8 : (190 * 1024 / STAGE_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + EPI_STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN;
};

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int BN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_pers(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const GemmArgs args) {
  using Cfg = PersCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_slot;
  const uint32_t warp = warp_id(), lane = lane_id();
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(&tmem_slot);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  pdl_wait();
  const int M_live = args.M_dyn ? min(args.M, *args.M_dyn) : args.M;
  const int m_tiles = (M_live + BM - 1) / BM;
  const int n_tiles = (args.N + BN - 1) / BN;
  const int T = m_tiles * n_tiles;
  const int num_kb = (args.K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t ps = 0, pph = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int m0 = (t / n_tiles) * BM, n0 = (t % n_tiles) * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[ps], pph ^ 1);
          uint8_t* sa = smem + ps * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[ps], Cfg::STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full_bar[ps], kb * BK, m0);
          tma_load_2d(sa + 64 * BK, &tmA, &full_bar[ps], kb * BK, m0 + 64);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(sb + j * 64 * BK, &tmB, &full_bar[ps], kb * BK, n0 + j * 64);
          if (++ps == STAGES) { ps = 0; pph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: warp-uniform loop, one elected lane issues (as in k_gemm_i8)
    constexpr uint32_t idesc = idesc_i8<BM, BN>();
    uint32_t cs = 0, cph = 0, ab = 0, aph = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      mbar_wait(&tempty_bar[ab], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + ab * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[cs], cph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + cs * Cfg::STAGE_BYTES);
        const uint64_t adesc = umma_desc_sw128(sa);
        const uint64_t bdesc = umma_desc_sw128(sa + Cfg::A_BYTES);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 32; ++k)
            mma_i8(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
          mma_commit(&empty_bar[cs]);
        }
        __syncwarp();
        if (++cs == STAGES) { cs = 0; cph ^= 1; }
      }
      if (elect_one()) mma_commit(&tfull_bar[ab]);
      __syncwarp();
      ab ^= 1;
      if (ab == 0) aph ^= 1;
    }
  } else {
    const int q = warp & 3, half = (warp - 2) >> 2;
    constexpr int HALF = BN / 2;
    uint32_t ab = 0, aph = 0;
    bool first = true;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const int m0 = (t / n_tiles) * BM, n0 = (t % n_tiles) * BN;
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < M_live;
      uint32_t slw[HALF / 32];
      if constexpr (EPI == EPI_ARGMAX) sl_words<HALF>(args, row, row_ok, n0 + half * HALF, slw);
      mbar_wait(&tfull_bar[ab], aph);
      tc_fence_after();
      if (first && warp == 2 && lane == 0) pdl_launch_dependents();
      first = false;
      const uint32_t t_row = tmem_base + ab * BN + ((uint32_t)(q * 32) << 16) + half * HALF;
      float* stage = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES) +
                     (warp - 2) * EPI_STAGE_FLOATS;
      float best_v = -INFINITY;
      int best_j = -1;
#pragma unroll 1
      for (int c = 0; c < HALF; c += 32) {
        int32_t acc[32];
        tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
        tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
        tmem_ld_wait();
        const int n = n0 + half * HALF + c;
        if (n >= args.N) break;
        epi_store_chunk<EPI>(args, args.bias, row, row_ok, n, acc, best_v, best_j, stage,
                             EPI == EPI_ARGMAX ? slw[c / 32] : 0u);
      }
      if constexpr (EPI == EPI_ARGMAX) {
        if (row_ok && best_j >= 0) atomicMax(args.keys + row, argmax_key(best_v, (uint32_t)best_j));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&tempty_bar[ab]);
      ab ^= 1;
      if (ab == 0) aph ^= 1;
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ CTA-pair persistent variant
// For the many-row GEMMs (encoder, K|V, the output layer at hundreds of rows) the one-CTA
// persistent kernel is bound by L2 -> SM traffic: a 128 x 256 tile streams 48 KB per K block for
// 4.2 M MACs (ncu: ~50 % of the int8 pipe).  k_gemm_pers2 runs a 256 x 256 tile on a CTA pair
// (thread-block cluster of 2, tcgen05 cta_group::2): each CTA loads its 128 rows of A and its
// 128 rows of B (32 KB per K block, both completing on the leader's barrier), the leader issues
// M = 256 MMAs that read both CTAs' shared memory, and each CTA's TMEM receives its 128 rows of
// the accumulator (two 256-column buffers).  Commits are multicast to both CTAs; each CTA's
// epilogue warps release an accumulator buffer on the leader's barrier.  Numerics and epilogues
// are k_gemm_pers's (exact s32 sums; outputs identical).
constexpr int P2_BN = 256;
struct Pers2Cfg {
  static constexpr int A_BYTES = BM * BK;              // this CTA's 128 rows of A
  static constexpr int B_BYTES = (P2_BN / 2) * BK;     // this CTA's 128 rows of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = 5;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + EPI_STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * P2_BN;          // two accumulator buffers
};

template <int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_pers2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const GemmArgs args) {
  using Cfg = Pers2Cfg;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];    // leader: both CTAs' bytes
  __shared__ __align__(8) uint64_t empty_bar[STAGES];   // both: the leader's commit (multicast)
  __shared__ __align__(8) uint64_t tfull_bar[2];        // both: accumulator buffer complete
  __shared__ __align__(8) uint64_t tempty_bar[2];       // leader: both CTAs' epilogue warps
  __shared__ uint32_t tmem_slot;
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<Cfg::TMEM_COLS>(&tmem_slot);
  __syncwarp();
  tc_fence_before();
  cluster_sync();   // both CTAs' barriers initialised and TMEM allocated before any remote use
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  pdl_wait();
  const int M_live = args.M_dyn ? min(args.M, *args.M_dyn) : args.M;
  const int m_tiles = (M_live + 2 * BM - 1) / (2 * BM);
  const int n_tiles = (args.N + P2_BN - 1) / P2_BN;
  const int T = m_tiles * n_tiles;
  const int num_kb = (args.K + BK - 1) / BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs): this CTA's A and B halves, counted on the
      // leader's full barrier
      uint32_t ps = 0, pph = 0;
      for (int t = pair; t < T; t += npairs) {
        const int m0 = (t / n_tiles) * 2 * BM + (int)rank * BM, n0 = (t % n_tiles) * P2_BN + (int)rank * (P2_BN / 2);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[ps], pph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[ps], 2 * Cfg::STAGE_BYTES);
          const uint32_t fb = mapa_shared(smem_u32(&full_bar[ps]), 0);
          uint8_t* sa = smem + ps * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          tma_load_2d_pair(sa, &tmA, fb, kb * BK, m0);
          tma_load_2d_pair(sa + 64 * BK, &tmA, fb, kb * BK, m0 + 64);
          tma_load_2d_pair(sb, &tmB, fb, kb * BK, n0);
          tma_load_2d_pair(sb + 64 * BK, &tmB, fb, kb * BK, n0 + 64);
          if (++ps == STAGES) { ps = 0; pph ^= 1; }
        }
      }
      // drain: every stage's last use released (the commits that arrive here have landed)
      for (int i = 0; i < STAGES; ++i) {
        mbar_wait(&empty_bar[ps], pph ^ 1);
        if (++ps == STAGES) { ps = 0; pph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader's warp 1, warp-uniform; one elected lane issues):
      // 256 x 256 x 32 per instruction for the pair
      constexpr uint32_t idesc = idesc_i8<2 * BM, P2_BN>();
      uint32_t cs = 0, cph = 0, ab = 0, aph = 0;
      for (int t = pair; t < T; t += npairs) {
        mbar_wait_cluster(&tempty_bar[ab], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + ab * P2_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait_cluster(&full_bar[cs], cph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + cs * Cfg::STAGE_BYTES);
          const uint64_t adesc = umma_desc_sw128(sa);
          const uint64_t bdesc = umma_desc_sw128(sa + Cfg::A_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 32; ++k)
              mma_i8_pair(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
            mma_commit_pair(&empty_bar[cs], 0x3);
          }
          __syncwarp();
          if (++cs == STAGES) { cs = 0; cph ^= 1; }
        }
        if (elect_one()) mma_commit_pair(&tfull_bar[ab], 0x3);
        __syncwarp();
        ab ^= 1;
        if (ab == 0) aph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): this CTA's 128 rows x 256 columns
    const int q = warp & 3, half = (warp - 2) >> 2;
    constexpr int HALF = P2_BN / 2;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    uint32_t ab = 0, aph = 0;
    bool first = true;
    for (int t = pair; t < T; t += npairs) {
      const int m0 = (t / n_tiles) * 2 * BM + (int)rank * BM, n0 = (t % n_tiles) * P2_BN;
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < M_live;
      uint32_t slw[HALF / 32];
      if constexpr (EPI == EPI_ARGMAX) sl_words<HALF>(args, row, row_ok, n0 + half * HALF, slw);
      mbar_wait_cluster(&tfull_bar[ab], aph);
      tc_fence_after();
      if (first && warp == 2 && lane == 0) pdl_launch_dependents();
      first = false;
      const uint32_t t_row = tmem_base + ab * P2_BN + ((uint32_t)(q * 32) << 16) + half * HALF;
      float* stage = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES) + (warp - 2) * EPI_STAGE_FLOATS;
      float best_v = -INFINITY;
      int best_j = -1;
#pragma unroll 1
      for (int c = 0; c < HALF; c += 32) {
        int32_t acc[32];
        tmem_ld16(t_row + c, *reinterpret_cast<int32_t(*)[16]>(acc));
        tmem_ld16(t_row + c + 16, *reinterpret_cast<int32_t(*)[16]>(acc + 16));
        tmem_ld_wait();
        const int n = n0 + half * HALF + c;
        if (n >= args.N) break;
        epi_store_chunk<EPI>(args, args.bias, row, row_ok, n, acc, best_v, best_j, stage,
                             EPI == EPI_ARGMAX ? slw[c / 32] : 0u);
      }
      if constexpr (EPI == EPI_ARGMAX) {
        if (row_ok && best_j >= 0) atomicMax(args.keys + row, argmax_key(best_v, (uint32_t)best_j));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + ab * 8);
      ab ^= 1;
      if (ab == 0) aph ^= 1;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();   // both CTAs done: every MMA has completed and been read
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ swap-AB variant
// For a handful of live rows (a decoder step of the critical lane, <= 64 rows) the 128-row A
// tile of k_gemm_i8 is mostly padding, yet every CTA streams it from L2 after the PDL wait (the
// per-launch critical path at deep K: 8 x 16 KB per CTA at K = 1024, DESIGN 12.3).  k_gemm_sab
// computes the transposed product D^T = W . A^T on the same tensor cores: the 128 weight rows
// of an N tile are the MMA's M = 128 operand (constant, all of a CTA's K blocks requested
// before griddepcontrol.wait), the live rows are its N = MP operand (MP = 16 / 32 / 64 / 128,
// MP x 128 bytes per K block after the wait), and the s32 accumulator D^T[n][m] lives in MP
// TMEM columns.  Deep K is split over a cluster along z exactly as in k_gemm_i8 (partials into
// the leader's slots, exact integer adds).  Epilogue: TMEM lane = output column n, column =
// row m, so each epilogue warp holds 32 consecutive columns of a row and its fp32 stores are
// full 128-byte lines without staging.  The arithmetic per element is k_gemm_i8's
// (v = fmaf((float)acc, s, b[n]), then ReLU / sigmoid / Q / argmax key), so outputs are
// bit-identical to the other paths.
constexpr int SAB_STAGES = 8;   // K blocks per CTA kept in flight (the launch splits K to fit)
constexpr int SAB_STAGE_LD = 36;   // epilogue staging row stride (floats): 32 columns + pad
template <int MP>
struct SabCfg {
  static constexpr int W_BYTES = BM * BK;   // 128 weight rows x 128 K bytes
  static constexpr int A_BYTES = MP * BK;   // MP activation rows x 128 K bytes
  static constexpr int STAGE_BYTES = W_BYTES + A_BYTES;
  static constexpr int TMEM_COLS = MP < 32 ? 32 : MP;
  static constexpr int RED_LD = MP + 4;     // split-K slot row stride (s32): 16-byte rows
  static constexpr int RED_SLOT_BYTES = BM * RED_LD * 4;
};

// acc[0..CH) = the accumulator's columns at taddr
template <int CH>
__device__ __forceinline__ void sab_ld_acc(uint32_t taddr, int32_t (&acc)[16]) {
  if constexpr (CH == 16) tmem_ld16(taddr, acc);
  else tmem_ld8(taddr, *reinterpret_cast<int32_t(*)[8]>(acc));
  tmem_ld_wait();
}

template <int MP, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_sab(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const GemmArgs args) {
  using Cfg = SabCfg<MP>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[SAB_STAGES];
  __shared__ __align__(8) uint64_t empty_bar[SAB_STAGES];
  __shared__ __align__(8) uint64_t tmem_full_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ float bias_s[BM];
  __shared__ unsigned long long amax_s[EPI == EPI_ARGMAX ? MP : 1];   // the CTA's row maxima

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int n0 = blockIdx.x * BM;
  const int ks = gridDim.z, kz = blockIdx.z;
  const int kb_all = (args.K + BK - 1) / BK, kb_per = (kb_all + ks - 1) / ks;
  const int kb0 = kz * kb_per;
  const int num_kb = min(kb_all, kb0 + kb_per) - kb0;
  const int stages = min(args.ring_cap, num_kb);   // ring depth chosen at launch
  if (threadIdx.x == 0) GEMM_TRACE(0);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  int32_t* red = reinterpret_cast<int32_t*>(smem + args.ring_cap * Cfg::STAGE_BYTES);
  if (ks > 1) cluster_arrive_relaxed();   // phase 1: this CTA is running (DSMEM valid)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tmem_full_bar, 1);
    fence_barrier_init();
    // the constant weight rows of the first stages before the PDL wait
    for (int s = 0; s < stages; ++s) {
      mbar_arrive_expect_tx(&full_bar[s], Cfg::STAGE_BYTES);
      uint8_t* sw = smem + s * Cfg::STAGE_BYTES;
      tma_load_2d(sw, &tmB, &full_bar[s], (kb0 + s) * BK, n0);
      tma_load_2d(sw + 64 * BK, &tmB, &full_bar[s], (kb0 + s) * BK, n0 + 64);
    }
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(&tmem_slot);
  if (args.bias && warp >= 2)
    for (int i = (int)threadIdx.x - 64; i < BM; i += 32 * EPI_WARPS)
      bias_s[i] = n0 + i < args.N ? __ldg(args.bias + n0 + i) : 0.0f;
  if constexpr (EPI == EPI_ARGMAX)
    if (warp >= 2 && (int)threadIdx.x - 64 < MP) amax_s[threadIdx.x - 64] = 0ull;
  // the CTA barrier before the PDL wait (measured faster than after it, as in k_gemm_i8)
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) GEMM_TRACE(1);
  if (warp == 0 && lane == 0)
    for (int s = 0; s < stages; ++s)
      tma_load_2d(smem + s * Cfg::STAGE_BYTES + Cfg::W_BYTES, &tmA, &full_bar[s], (kb0 + s) * BK, 0);
  const int M_live = args.M_dyn ? min(args.M, *args.M_dyn) : args.M;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (stages 0..stages-1 were issued above)
      for (int kb = stages; kb < num_kb; ++kb) {
        const int s = kb % stages;
        uint8_t* sw = smem + s * Cfg::STAGE_BYTES;
        mbar_wait(&empty_bar[s], ((kb / stages) - 1) & 1);
        mbar_arrive_expect_tx(&full_bar[s], Cfg::STAGE_BYTES);
        tma_load_2d(sw, &tmB, &full_bar[s], (kb0 + kb) * BK, n0);
        tma_load_2d(sw + 64 * BK, &tmB, &full_bar[s], (kb0 + kb) * BK, n0 + 64);
        tma_load_2d(sw + Cfg::W_BYTES, &tmA, &full_bar[s], (kb0 + kb) * BK, 0);
      }
    }
    __syncwarp();
    if (ks > 1) {
      cluster_wait();
      cluster_arrive();
      cluster_wait();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform, one elected lane issues):
    // D^T[128 x MP] (+)= W[128 x 32] . A[MP x 32]^T per step
    constexpr uint32_t idesc = idesc_i8<BM, MP>();
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % stages;
      mbar_wait(&full_bar[s], (kb / stages) & 1);
      if (kb == 0 && lane == 0) GEMM_TRACE(2);
      tc_fence_after();
      const uint32_t sw = smem_u32(smem + s * Cfg::STAGE_BYTES);
      const uint64_t wdesc = umma_desc_sw128(sw);
      const uint64_t adesc = umma_desc_sw128(sw + Cfg::W_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BK / 32; ++k)
          mma_i8(tmem_base, wdesc + (uint64_t)(2 * k), adesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
        mma_commit(&empty_bar[s]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&tmem_full_bar);
    __syncwarp();
    if (ks > 1) {
      cluster_wait();
      cluster_arrive();
      cluster_wait();
    }
  } else {
    // ---------------- epilogue: warps 2..9; TMEM lane quarter q = warp % 4 holds output columns
    // n0 + 32 q .. + 31 (lane = column); half = (warp - 2) / 4 takes rows [half MP/2, +MP/2)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HR = MP / 2;              // rows per warp
    constexpr int CH = HR < 16 ? 8 : 16;    // rows per tcgen05.ld
    const int cl = q * 32 + (int)lane;      // column within the tile (TMEM lane)
    const int n = n0 + cl;
    const bool col_ok = n < args.N;
    const float b = args.bias ? bias_s[cl] : 0.0f;
    const uint32_t t_lane = tmem_base + ((uint32_t)(q * 32) << 16);
    const int r_beg = half * HR;
    mbar_wait(&tmem_full_bar, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) GEMM_TRACE(3);
    if (warp == 2 && lane == 0) pdl_launch_dependents();
    if (ks > 1) {
      // split-K exchange: CTAs z > 0 store the live rows of their partial accumulators into
      // the leader's slot z - 1; the leader adds the slots to its own before the epilogue
      __syncwarp();
      cluster_wait();   // phase 1: every CTA of the cluster is running
      if (kz > 0) {
        const uint32_t base = mapa_shared(
            smem_u32(red + (kz - 1) * (Cfg::RED_SLOT_BYTES / 4) + cl * Cfg::RED_LD), 0);
#pragma unroll 1
        for (int r0 = r_beg; r0 < r_beg + HR && r0 < M_live; r0 += CH) {
          int32_t acc[16];
          sab_ld_acc<CH>(t_lane + r0, acc);
#pragma unroll
          for (int j = 0; j < CH; j += 4)
            st_cluster_v4(base + 4 * (r0 + j), acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        }
      }
      __syncwarp();
      cluster_arrive();   // phase 2 (release): partials stored
      cluster_wait();
    }
    if (!(ks > 1 && kz > 0)) {
      const bool small = args.K <= 256;
      // per-warp staging tile [CH rows][32 columns] in the ring (free: every MMA has completed)
      float* stage = reinterpret_cast<float*>(smem) + (warp - 2) * (16 * SAB_STAGE_LD);
      const int nw = n0 + q * 32;                 // the warp's first column
      const int sub = (int)lane >> 3, c4 = ((int)lane & 7) * 4;   // store phase: 4 rows x 8 lanes
#pragma unroll 1
      for (int r0 = r_beg; r0 < r_beg + HR && r0 < M_live; r0 += CH) {   // warp-uniform
        int32_t acc[16];
        sab_ld_acc<CH>(t_lane + r0, acc);
        if (ks > 1) {   // + the other K ranges' partials (exact s32)
          for (int z = 1; z < ks; ++z) {
            const int4* rp = reinterpret_cast<const int4*>(red + (z - 1) * (Cfg::RED_SLOT_BYTES / 4) +
                                                           cl * Cfg::RED_LD + r0);
#pragma unroll
            for (int j = 0; j < CH / 4; ++j) {
              const int4 p = rp[j];
              acc[4 * j] += p.x; acc[4 * j + 1] += p.y; acc[4 * j + 2] += p.z; acc[4 * j + 3] += p.w;
            }
          }
        }
        if (r0 == r_beg && warp == 2 && lane == 0) GEMM_TRACE(6);
        const int nr = min(CH, M_live - r0);   // live rows of this chunk
        if constexpr (EPI == EPI_ACC) {
#pragma unroll
          for (int j = 0; j < CH; ++j)
            if (j < nr && col_ok) args.out_i[(int64_t)(r0 + j) * args.ldo + n] = acc[j];
        } else if constexpr (EPI == EPI_ARGMAX) {
          // the row's maximum over this warp's 32 columns, lowest column on ties (R15): the
          // order key's warp maximum (redux), then the lowest lane holding it (columns ascend
          // with the lane) -- the packed key of k_gemm_i8 maximised over the same columns
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            if (j < nr) {
              const float v = __fmaf_rn(acc_to_float(acc[j], small), args.scale, b);
              const uint32_t k32 = col_ok ? float_order_key(v) : 0u;
              const uint32_t mk = __reduce_max_sync(0xffffffffu, k32);
              const uint32_t hit = __ballot_sync(0xffffffffu, col_ok && k32 == mk);
              if (lane == 0 && hit) {   // the CTA's maximum first (one global atomic per row)
                const uint32_t jcol = (uint32_t)(nw + __ffs(hit) - 1);
                atomicMax(amax_s + r0 + j,
                          ((unsigned long long)mk << 32) | (unsigned long long)(0xFFFFFFFFu - jcol));
              }
            }
          }
        } else {
          // dequant + fused op per element, staged [row][column] so each store instruction
          // writes whole 128-byte row segments (fp32) / 32-byte code segments
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            float v = __fmaf_rn(acc_to_float(acc[j], small), args.scale, b);
            if constexpr (EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) v = relu(v);
            if constexpr (EPI == EPI_SIGMOID) v = sigmoid_f64(v);
            stage[j * SAB_STAGE_LD + lane] = v;
          }
          __syncwarp();
          const int nc = nw + c4;
          const bool c_ok = nc < args.N;   // N % 16 == 0: whole 4-column groups
#pragma unroll
          for (int it = 0; it < CH / 4; ++it) {
            const int j = it * 4 + sub;
            if (j < nr && c_ok) {
              const float4 v4 = *reinterpret_cast<const float4*>(stage + j * SAB_STAGE_LD + c4);
              const int r = r0 + j;
              if constexpr (EPI == EPI_F32 || EPI == EPI_F32_Q || EPI == EPI_RELU_F32_Q || EPI == EPI_SIGMOID) {
                const int blk = nc / args.col_block;   // 4-column groups never straddle a block
                *reinterpret_cast<float4*>(args.out_f + (int64_t)blk * args.block_stride +
                                           (int64_t)r * args.ldo + (nc - blk * args.col_block)) = v4;
              }
              if constexpr (EPI == EPI_F32_Q || EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) {
                const uint32_t w = (uint32_t)(q8(v4.x, args.clip, args.sigma) & 0xff) |
                                   ((uint32_t)(q8(v4.y, args.clip, args.sigma) & 0xff) << 8) |
                                   ((uint32_t)(q8(v4.z, args.clip, args.sigma) & 0xff) << 16) |
                                   ((uint32_t)(q8(v4.w, args.clip, args.sigma) & 0xff) << 24);
                *reinterpret_cast<uint32_t*>(args.out_q + (int64_t)r * args.ldo + nc) = w;
              }
            }
          }
          __syncwarp();
        }
      }
      if constexpr (EPI == EPI_ARGMAX) {   // the 8 epilogue warps' row maxima -> global keys
        named_bar_sync(1, 32 * EPI_WARPS);
        const int i = (int)threadIdx.x - 64;
        if (i < M_live && i < MP && amax_s[i]) atomicMax(args.keys + i, amax_s[i]);
      }
    }
    if (warp == 2 && lane == 0) GEMM_TRACE(4);
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  if (warp == 1 && lane == 0) GEMM_TRACE(5);
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

bool make_tmap_kv(CUtensorMap* map, const void* base, int64_t rows, int64_t cols) {
  auto enc = get_encode();
  if (!enc || rows < 1 || cols % 4 != 0 || ((uintptr_t)base & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32u, 8u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
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

// Persistent tile loop once the grid would exceed two waves of one CTA per SM
// (env MNMT_GEMM_PERSISTENT=0/1 forces it off/on for A/B tests).
// sms: the SMs the launch may use (a lane's partition / pers_grid cap); 0 = the device's.
bool gemm_persistent(int M, int N, int bn, int sms) {
  static const int force = [] {
    const char* e = getenv("MNMT_GEMM_PERSISTENT");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  if (force >= 0) return force == 1;
  const long tiles = (long)((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  // also every launch with more than 64 rows: the persistent kernel is 0.3-4 us faster per launch
  // at 128-630 rows even with one tile per CTA (d x d 4.84 -> 4.03 us at 128 rows, FFN1 11.2 ->
  // 7.1 at 630, FFN2 9.8 -> 7.4 at 128; big job 83.4 -> 81.3 ms, profiles/r2_gemm_persistent_ab.txt)
  return tiles > 2L * (sms > 0 ? sms : num_sms()) || M > 64;
}

int gemm_pick_bn(int M, int N, int sms) {
  const int S = sms > 0 ? sms : num_sms();
  const int mt = (M + BM - 1) / BM;
  if ((long)mt * ((N + 255) / 256) > 2L * S) return 256;   // persistent, widest tile
  if (((N + 255) / 256) * mt >= S) return 256;
  // few rows, very wide N (the output layer at <= 128 rows): 128-wide tiles would need two waves,
  // 256-wide ones fit one (output GEMM + argmax at 1-64 rows, d 1024: 11.1 -> 8.2 us; d 256:
  // 7.2 -> 5.3 us; profiles/r2_out_gemm_tiles.txt)
  if (M <= 128 && (long)((N + 127) / 128) * mt > S) return 256;
  if (((N + 127) / 128) * mt >= S / 2) return 128;
  return 64;
}

static int num_sms() {
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
  return n[dev] > 0 ? n[dev] : 148;
}

// Persistent launch: grid = min(tiles, SMs), one CTA per SM.
template <int BN, int EPI>
static cudaError_t launch_pers_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                                 cudaStream_t st) {
  const int tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  int cap = num_sms();
  if (a.pers_grid > 0 && a.pers_grid < cap) cap = a.pers_grid;
  cfg.gridDim = dim3(tiles < cap ? tiles : cap);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = PersCfg<BN>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_pers<BN, EPI>, tmA, tmB, a);
}

// CTA-pair persistent launch: one cluster of 2 per pair of SMs, 256 x 256 tiles.  Taken for the
// BN = 256 persistent launches with deep K (>= 2048: the operand stream, not the epilogue's
// stores, bounds the tile; measured encoder FFN2 of the big student, 33k rows, K 4096: 70.6 ->
// 81.8 % of the int8 peak, while the K = 1024 GEMMs with fp32 outputs lose 3-10 %,
// profiles/r2_pair_micro.txt).  env MNMT_PERS2 = 0 / 1 forces it off / on (A/B).
static int pers2_mode() {
  static const int v = [] {
    const char* e = getenv("MNMT_PERS2");
    return e ? atoi(e) : -1;
  }();
  return v;
}
static bool pers2_take(const GemmArgs& a) {
  if (a.pers2 != 0) return a.pers2 > 0;
  const int mode = pers2_mode();
  return mode >= 0 ? mode == 1 : a.K >= 2048;
}

template <int EPI>
static cudaError_t launch_pers2_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                                  cudaStream_t st) {
  const int tiles = ((a.M + 2 * BM - 1) / (2 * BM)) * ((a.N + P2_BN - 1) / P2_BN);
  int cap = num_sms();
  if (a.pers_grid > 0 && a.pers_grid < cap) cap = a.pers_grid;
  const int pairs = std::max(1, std::min(tiles, cap / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Pers2Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_pers2<EPI>, tmA, tmB, a);
}

static cudaError_t launch_pers2(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, int epi,
                                cudaStream_t st) {
  switch (epi) {
    case EPI_F32: return launch_pers2_t<EPI_F32>(tmA, tmB, a, st);
    case EPI_F32_Q: return launch_pers2_t<EPI_F32_Q>(tmA, tmB, a, st);
    case EPI_RELU_Q: return launch_pers2_t<EPI_RELU_Q>(tmA, tmB, a, st);
    case EPI_RELU_F32_Q: return launch_pers2_t<EPI_RELU_F32_Q>(tmA, tmB, a, st);
    case EPI_SIGMOID: return launch_pers2_t<EPI_SIGMOID>(tmA, tmB, a, st);
    case EPI_ARGMAX: return launch_pers2_t<EPI_ARGMAX>(tmA, tmB, a, st);
    case EPI_ACC: return launch_pers2_t<EPI_ACC>(tmA, tmB, a, st);
  }
  return cudaErrorNotSupported;
}

// Split-K factor of a non-persistent launch (GemmArgs::split_k: 0 none, > 1 forced, -1 the rule
// below): deep K and a grid that leaves most SMs idle (FFN2 of the base / big students at small
// row counts, where each CTA would stream its whole K = F range alone).  Powers of two while the split grid fits the launch's SM budget, every
// CTA keeps >= 1 K block and the leader's partial slots fit its shared memory (<= 4 for
// BN = 64).  Measured (profiles/r2_gemm_splitk.txt, warm PDL chain): big FFN2 (K = 4096)
// 10.5 -> 6.0 us at <= 32 rows, 10.7 -> 8.7 at 128; base FFN2 (K = 2048) 6.5 -> 5.0 at <= 32
// rows but 6.7 -> 7.6 at 128; K = 1024 neutral at <= 32 rows and slower at 128-256 (the
// partial tiles cross distributed shared memory).  Hence the rule: K >= 4096, or K >= 2048 with
// a <= 32-row bound.  In the whole big-student job it still loses (3 lanes: 118.4-119.2 ms per
// job without, 122.0-122.6 with; profiles/r2_gemm_splitk.txt), so the model path leaves it off
// unless the model option "split_k" = 1 asks for the rule.
static int gemm_split_k(const GemmArgs& a, int bn, int epi) {
  if (a.split_k == 0 || a.split_k == 1 || bn > 128) return 1;
  if (a.split_k < 0 && !(a.K >= 4096 || (a.K >= 2048 && a.M <= 32))) return 1;
  if (!(epi == EPI_F32 || epi == EPI_F32_Q || epi == EPI_RELU_Q || epi == EPI_RELU_F32_Q ||
        epi == EPI_SIGMOID || epi == EPI_ACC))
    return 1;
  const int sms = a.pers_grid > 0 ? a.pers_grid : num_sms();
  const long tiles = (long)((a.N + bn - 1) / bn) * ((a.M + BM - 1) / BM);
  const int kb_all = (a.K + BK - 1) / BK;
  int ks = 1;
  // the leader holds ks - 1 partial slots next to its ring and epilogue staging
  const int slot = BM * (bn + 4) * 4;
  const int want = a.split_k > 1 ? a.split_k : 8;
  while (ks < want && (a.split_k > 1 || tiles * ks * 2 <= sms) && kb_all >= ks * 2 &&
         (long)(2 * ks - 1) * slot + 1024 + EPI_STAGE_BYTES + 2 * (BM + 64) * BK <= GEMM_SMEM_MAX)
    ks *= 2;
  while (ks > 1 && kb_all - (ks - 1) * ((kb_all + ks - 1) / ks) < 1) ks /= 2;   // no empty range
  return ks;
}

static bool make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld,
                           int box_rows);

// Live-row A boxes (env MNMT_ABOX=0 disables; A/B): a launch whose row bound a.M is <= 64 and
// whose raw A pointer is known loads only ceil16(a.M) rows of A per K block instead of 128.
static bool abox_on() {
  static const bool on = [] {
    const char* e = getenv("MNMT_ABOX");
    return !(e && e[0] == '0');
  }();
  return on;
}

// The one-shot kernel's CTA barrier before the PDL wait instead of after it (the persistent
// kernel's order): d x d 4.21 -> 3.90 us at 8 rows, 4.84 -> 4.37 at 128, FFN2 (K 4096) 9.0 -> 8.8
// (profiles/r2_gemm_npsync_ab.txt).  env MNMT_NPSYNC = 0 restores the old order (A/B).
static int gemm_npsync() {
  static const int v = [] {
    const char* e = getenv("MNMT_NPSYNC");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int BN, int EPI>
static cudaError_t launch_t(const CUtensorMap& tmA_in, const CUtensorMap& tmB_in, const GemmArgs& a,
                            cudaStream_t st) {
  if constexpr (BN >= 64)   // BN = 32 (16-column epilogue chunks) is never persistent
    if (gemm_persistent(a.M, a.N, BN, a.pers_grid) && gemm_split_k(a, BN, EPI) == 1) {
      if (BN == 256 && pers2_take(a))
        return launch_pers2_t<EPI>(tmA_in, tmB_in, a, st);
      return launch_pers_t<BN, EPI>(tmA_in, tmB_in, a, st);
    }
  using Cfg = GemmCfg<BN>;
  const int ks = gemm_split_k(a, BN, EPI);
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, ks);
  const int num_kb = (a.K + BK - 1) / BK, kb_per = (num_kb + ks - 1) / ks;
  GemmArgs b = a;
  b.npsync = gemm_npsync();
  CUtensorMap tmA = tmA_in, tmB = tmB_in;
  b.a_box = 0;
  b.b_box = 0;
  if (abox_on() && a.a_ptr && a.M <= 64 && a.K % 16 == 0 && a.lda % 16 == 0) {
    const int box = a.M <= 16 ? 16 : a.M <= 32 ? 32 : 64;
    if (make_tmap_rows(&tmA, a.a_ptr, a.M, a.K, a.lda, box)) b.a_box = box;
    else tmA = tmA_in;
  }
  if (abox_on() && a.b_ptr && BN == 32) {
    if (make_tmap_rows(&tmB, a.b_ptr, a.N, a.K, a.K, 32)) b.b_box = 32;
    else tmB = tmB_in;
  }
  int ring = kb_per < Cfg::STAGES ? kb_per : Cfg::STAGES;
  size_t smem = Cfg::smem_for(ring);
  if (ks > 1) {   // + the leader's partial buffer; the ring shrinks to fit
    const int red_bytes = (ks - 1) * Cfg::RED_SLOT_BYTES;
    const int cap = (int)((GEMM_SMEM_MAX - 1024 - EPI_STAGE_BYTES - red_bytes) / Cfg::STAGE_BYTES);
    if (ring > cap) ring = cap;
    b.ring_cap = ring;
    smem = Cfg::smem_for(ring) + red_bytes;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = ks;
  cfg.attrs = attr;
  cfg.numAttrs = ks > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_i8<BN, EPI>, tmA, tmB, b);
}

template <int BN, int EPI>
static cudaError_t set_attr() {
  cudaError_t e = cudaFuncSetAttribute(k_gemm_i8<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       std::max<int>(GemmCfg<BN>::smem_for(GemmCfg<BN>::STAGES), GEMM_SMEM_MAX));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_gemm_pers<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              PersCfg<BN>::SMEM);
}
// BN = 32 (non-persistent, fp32 / code epilogues only): 16 columns per epilogue warp
static cudaError_t set_attr_bn32() {
  for (const void* f : {(const void*)k_gemm_i8<32, EPI_F32>, (const void*)k_gemm_i8<32, EPI_F32_Q>,
                        (const void*)k_gemm_i8<32, EPI_RELU_Q>, (const void*)k_gemm_i8<32, EPI_RELU_F32_Q>,
                        (const void*)k_gemm_i8<32, EPI_SIGMOID>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         std::max<int>(GemmCfg<32>::smem_for(GemmCfg<32>::STAGES), GEMM_SMEM_MAX));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
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
template <int MP>
static cudaError_t set_attr_sab();

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
  if ((e = set_attr_bn32()) != cudaSuccess) return e;
  if ((e = set_attr_bn<64>()) != cudaSuccess) return e;
  if ((e = set_attr_bn<128>()) != cudaSuccess) return e;
  for (const void* f : {(const void*)k_gemm_pers2<EPI_F32>, (const void*)k_gemm_pers2<EPI_F32_Q>,
                        (const void*)k_gemm_pers2<EPI_RELU_Q>, (const void*)k_gemm_pers2<EPI_RELU_F32_Q>,
                        (const void*)k_gemm_pers2<EPI_SIGMOID>, (const void*)k_gemm_pers2<EPI_ARGMAX>,
                        (const void*)k_gemm_pers2<EPI_ACC>})
    if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, Pers2Cfg::SMEM)) != cudaSuccess)
      return e;
  if ((e = set_attr_sab<16>()) != cudaSuccess) return e;
  if ((e = set_attr_sab<32>()) != cudaSuccess) return e;
  if ((e = set_attr_sab<64>()) != cudaSuccess) return e;
  if ((e = set_attr_sab<128>()) != cudaSuccess) return e;
  for (const void* f : {(const void*)k_gemm_i8<TOPK_BN, EPI_TOPK>, (const void*)k_gemm_i8<TOPK_BN, EPI_TOPK2>,
                        (const void*)k_gemm_i8<TOPK_BN, EPI_TOPK4>})
    if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  GemmCfg<TOPK_BN>::smem_for(GemmCfg<TOPK_BN>::STAGES))) != cudaSuccess)
      return e;
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

// non-persistent launch of one instantiation
template <int BN, int EPI>
static cudaError_t launch_np(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                             cudaStream_t st) {
  using Cfg = GemmCfg<BN>;
  const int num_kb = (a.K + BK - 1) / BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg::smem_for(num_kb < Cfg::STAGES ? num_kb : Cfg::STAGES);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GemmArgs b = a;
  b.npsync = gemm_npsync();
  return cudaLaunchKernelEx(&cfg, k_gemm_i8<BN, EPI>, tmA, tmB, b);
}


// ------------------------------------------------------------------ small-M path
// At <= 32 live rows a decoder GEMM is latency-bound: the tcgen05 kernel's A-tile TMA round
// trip, MMA commit and TMEM load sit on the critical path of every launch (DESIGN 12.3).
// k_gemm_smallm computes the same s32 accumulators with IDP4A on CUDA cores: lane = row,
// warp = (column, K segment), CN = 8 / S columns per CTA, S K segments per column combined
// in shared memory.  Integer sums are exact in any order, and the epilogue is the tcgen05
// kernel's arithmetic element by element (v = fmaf(float(acc), s, b), then ReLU / sigmoid /
// Q), so outputs are bit-identical.  The weight row segment (constant) is loaded before the
// PDL wait; A rows are read straight from L2 after it.
template <int EPI, int S, int CPW>
__global__ void __launch_bounds__(256) k_gemm_smallm(const GemmArgs args) {
  constexpr int CN = 8 / S, CT = CN * CPW;   // column groups / columns per CTA
  extern __shared__ __align__(16) int8_t wsm[];   // [CT][K] the CTA's weight rows
  __shared__ int32_t red[8][CPW][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cw = warp % CN, seg = warp / CN;
  const int nbase = blockIdx.x * CT;
  const int K = args.K, KS = K / S, k0 = seg * KS, k16 = K >> 4;
  // constant operands before the PDL wait: weight rows staged in shared memory, bias
  const int ncols = min(CT, args.N - nbase);
  for (int i = threadIdx.x; i < ncols * k16; i += 256) {
    const int c = i / k16, kk = i - c * k16;
    *reinterpret_cast<uint4*>(wsm + c * K + 16 * kk) =
        __ldg(reinterpret_cast<const uint4*>(args.b_ptr + (int64_t)(nbase + c) * K + 16 * kk));
  }
  float b[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int n = nbase + cw * CPW + c;
    b[c] = (args.bias && seg == 0 && n < args.N) ? __ldg(args.bias + n) : 0.0f;
  }
  __syncthreads();   // weights staged (the barrier before the PDL wait, as in k_gemm_i8)
  pdl_wait();
  const int n_live = args.M_dyn ? min(args.M, *args.M_dyn) : args.M;
  const bool row_ok = lane < n_live;
  int32_t acc[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) acc[c] = 0;
  if (row_ok) {
    const int8_t* arow = args.a_ptr + (int64_t)lane * args.lda + k0;
    const int8_t* wb = wsm + (cw * CPW) * K + k0;
    for (int k = 0; k < KS; k += 64) {
      uint4 av[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + 16 * u < KS) av[u] = *reinterpret_cast<const uint4*>(arow + k + 16 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k + 16 * u < KS) {
#pragma unroll
          for (int c = 0; c < CPW; ++c) {   // broadcast reads: every lane the same address
            const uint4 wv = *reinterpret_cast<const uint4*>(wb + c * K + k + 16 * u);
            acc[c] = __dp4a((int)av[u].x, (int)wv.x, acc[c]);
            acc[c] = __dp4a((int)av[u].y, (int)wv.y, acc[c]);
            acc[c] = __dp4a((int)av[u].z, (int)wv.z, acc[c]);
            acc[c] = __dp4a((int)av[u].w, (int)wv.w, acc[c]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPW; ++c) red[warp][c][lane] = acc[c];
  __syncthreads();
  if (threadIdx.x == 0) pdl_launch_dependents();
  if (seg != 0 || !row_ok) return;   // no block-wide barrier below
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int n = nbase + cw * CPW + c;
    if (n >= args.N) break;
    int32_t a = 0;
#pragma unroll
    for (int g = 0; g < S; ++g) a += red[g * CN + cw][c][lane];
    float v = __fmaf_rn(acc_to_float(a, K <= 256), args.scale, b[c]);
    if constexpr (EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q) v = relu(v);
    if constexpr (EPI == EPI_SIGMOID) v = sigmoid_f64(v);
    if constexpr (EPI == EPI_F32 || EPI == EPI_F32_Q || EPI == EPI_RELU_F32_Q || EPI == EPI_SIGMOID) {
      const int blk = n / args.col_block;
      args.out_f[(int64_t)blk * args.block_stride + (int64_t)lane * args.ldo + (n - blk * args.col_block)] = v;
    }
    if constexpr (EPI == EPI_F32_Q || EPI == EPI_RELU_Q || EPI == EPI_RELU_F32_Q)
      args.out_q[(int64_t)lane * args.ldo + n] = (int8_t)q8(v, args.clip, args.sigma);
  }
}


template <int EPI, int CPW>
static cudaError_t launch_smallm_c(const GemmArgs& a, int S, cudaStream_t st) {
  const int CT = (8 / S) * CPW;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.N + CT - 1) / CT);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = (size_t)CT * a.K;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (S) {
    case 1: return cudaLaunchKernelEx(&cfg, k_gemm_smallm<EPI, 1, CPW>, a);
    case 2: return cudaLaunchKernelEx(&cfg, k_gemm_smallm<EPI, 2, CPW>, a);
    case 4: return cudaLaunchKernelEx(&cfg, k_gemm_smallm<EPI, 4, CPW>, a);
    case 8: return cudaLaunchKernelEx(&cfg, k_gemm_smallm<EPI, 8, CPW>, a);
  }
  return cudaErrorInvalidValue;
}

// CPW columns per warp: 4, or 8 where the 4-column grid would exceed 64 CTAs (wide N) or K is
// deep (every CTA reads all live rows of A, so fewer, wider CTAs cut the redundant A traffic)
// The grid must fit the launch's SM budget in one wave (3 resident CTAs per SM): in a small
// SM partition a multi-wave small-M grid is slower than the tcgen05 kernel (measured: base
// self-attention student, 24-SM critical lane, 66.4 -> 71.5 ms per job without this bound).
template <int EPI>
static cudaError_t launch_smallm_e(const GemmArgs& a, int S, cudaStream_t st) {
  const int cn = 8 / S;
  const int ctas4 = (a.N + cn * 4 - 1) / (cn * 4), ctas8 = (a.N + cn * 8 - 1) / (cn * 8);
  const int cap = a.smallm_force ? (1 << 30) : 3 * (a.pers_grid > 0 ? a.pers_grid : num_sms());
  // dynamic weight staging + the static reduction array red[8][CPW][32] within the 48 KB a
  // launch gets without an opt-in
  const bool fit8 = (size_t)cn * 8 * a.K + 8 * 8 * 32 * 4 <= 48 * 1024;
  const bool fit4 = (size_t)cn * 4 * a.K + 8 * 4 * 32 * 4 <= 48 * 1024;
  if (fit8 && (ctas4 > 64 || a.K >= 1024 || (ctas4 > cap && ctas8 <= cap)))
    return ctas8 <= cap ? launch_smallm_c<EPI, 8>(a, S, st) : cudaErrorNotSupported;
  if (!fit4 || ctas4 > cap) return cudaErrorNotSupported;
  return launch_smallm_c<EPI, 4>(a, S, st);
}

// Returns cudaErrorNotSupported when the launch does not qualify (the caller takes the
// tcgen05 path).
static cudaError_t launch_smallm(const GemmArgs& a, int epi, cudaStream_t st) {
  if (!a.a_ptr || !a.b_ptr || a.M > SMALLM_MAX) return cudaErrorNotSupported;
  if (!a.smallm_force && (a.smallm_rows <= 0 || a.M > a.smallm_rows || a.K > a.smallm_kmax ||
                          (int64_t)a.N * a.K > a.smallm_wmax))
    return cudaErrorNotSupported;
  if (a.K % 16 || a.lda % 16 || ((uintptr_t)a.a_ptr & 15) || ((uintptr_t)a.b_ptr & 15))
    return cudaErrorNotSupported;
  int S = 8;   // K segments per column: the largest power of two <= 8 leaving >= 64 bytes
  while (S > 1 && ((a.K % S) || (a.K / S) % 16 || a.K / S < 64)) S >>= 1;
  switch (epi) {
    case EPI_F32: return launch_smallm_e<EPI_F32>(a, S, st);
    case EPI_F32_Q: return launch_smallm_e<EPI_F32_Q>(a, S, st);
    case EPI_RELU_Q: return launch_smallm_e<EPI_RELU_Q>(a, S, st);
    case EPI_RELU_F32_Q: return launch_smallm_e<EPI_RELU_F32_Q>(a, S, st);
    case EPI_SIGMOID: return launch_smallm_e<EPI_SIGMOID>(a, S, st);
  }
  return cudaErrorNotSupported;
}

// ------------------------------------------------------------------ swap-AB launch
// Tensor map over the live rows of A with an MP-row box: rows beyond the launch's row bound
// a.M are outside the map (zero-filled by the TMA, never read from memory).  Encoded on the
// host at launch (graph capture) time; the kernel receives it by value.
static bool make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld,
                           int box_rows) {
  auto enc = get_encode();
  if (!enc || K % 16 != 0 || ld % 16 != 0 || rows < 1 || ((uintptr_t)base & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// K blocks per CTA of the swap-AB launch before K is split over a cluster (env MNMT_SAB_KB, A/B)
static int sab_kb_max() {
  static const int v = [] {
    const char* e = getenv("MNMT_SAB_KB");
    const int x = e ? atoi(e) : SAB_STAGES;
    return x < 1 ? 1 : x > SAB_STAGES ? SAB_STAGES : x;
  }();
  return v;
}

template <int MP, int EPI>
static cudaError_t launch_sab_t(const CUtensorMap& tmB, const GemmArgs& a, cudaStream_t st) {
  using Cfg = SabCfg<MP>;
  CUtensorMap tmA;
  if (!make_tmap_rows(&tmA, a.a_ptr, a.M, a.K, a.lda, MP)) return cudaErrorInvalidValue;
  const int kb_all = (a.K + BK - 1) / BK;
  const int kbm = a.sab_kb > 0 ? std::min(a.sab_kb, SAB_STAGES) : sab_kb_max();
  int ks = 1;
  while (ks < 8 && (kb_all + ks - 1) / ks > kbm && kb_all >= 2 * ks) ks *= 2;
  // the leader's partial slots plus at least two ring stages must fit its shared memory
  while (ks > 1 && (ks - 1) * Cfg::RED_SLOT_BYTES + 2 * Cfg::STAGE_BYTES + 1024 > GEMM_SMEM_MAX) ks /= 2;
  while (ks > 1 && kb_all - (ks - 1) * ((kb_all + ks - 1) / ks) < 1) ks /= 2;   // no empty range
  const int kb_per = (kb_all + ks - 1) / ks;
  const int red_bytes = ks > 1 ? (ks - 1) * Cfg::RED_SLOT_BYTES : 0;
  int ring = std::min(kb_per, SAB_STAGES);
  const int cap = (GEMM_SMEM_MAX - 1024 - red_bytes) / Cfg::STAGE_BYTES;
  if (cap < 1) return cudaErrorNotSupported;
  if (ring > cap) ring = cap;
  GemmArgs b = a;
  b.ring_cap = ring;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.N + BM - 1) / BM, 1, ks);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = 1024 + (size_t)ring * Cfg::STAGE_BYTES + red_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = ks;
  cfg.attrs = attr;
  cfg.numAttrs = ks > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_sab<MP, EPI>, tmA, tmB, b);
}

template <int MP>
static cudaError_t launch_sab_mp(const CUtensorMap& tmB, const GemmArgs& a, int epi, cudaStream_t st) {
  switch (epi) {
    case EPI_F32: return launch_sab_t<MP, EPI_F32>(tmB, a, st);
    case EPI_F32_Q: return launch_sab_t<MP, EPI_F32_Q>(tmB, a, st);
    case EPI_RELU_Q: return launch_sab_t<MP, EPI_RELU_Q>(tmB, a, st);
    case EPI_RELU_F32_Q: return launch_sab_t<MP, EPI_RELU_F32_Q>(tmB, a, st);
    case EPI_SIGMOID: return launch_sab_t<MP, EPI_SIGMOID>(tmB, a, st);
    case EPI_ARGMAX: return launch_sab_t<MP, EPI_ARGMAX>(tmB, a, st);
    case EPI_ACC: return launch_sab_t<MP, EPI_ACC>(tmB, a, st);
  }
  return cudaErrorNotSupported;
}

template <int MP>
static cudaError_t set_attr_sab() {
  for (const void* f : {(const void*)k_gemm_sab<MP, EPI_F32>, (const void*)k_gemm_sab<MP, EPI_F32_Q>,
                        (const void*)k_gemm_sab<MP, EPI_RELU_Q>, (const void*)k_gemm_sab<MP, EPI_RELU_F32_Q>,
                        (const void*)k_gemm_sab<MP, EPI_SIGMOID>, (const void*)k_gemm_sab<MP, EPI_ARGMAX>,
                        (const void*)k_gemm_sab<MP, EPI_ACC>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM_MAX);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Returns cudaErrorNotSupported when the launch does not qualify (the caller takes the
// 128-row tcgen05 path): needs the raw A pointer, a row bound <= the swap-AB bound
// (sab_rows, or any M <= 128 under sab_force), no shortlist / beam epilogue.
static cudaError_t launch_sab(const CUtensorMap& tmB, const GemmArgs& a, int epi, cudaStream_t st) {
  const int bound = a.sab_force ? 128 : a.sab_rows;
  if (!a.a_ptr || bound <= 0 || a.M > bound || a.M > 128 || a.colbits || is_topk(epi))
    return cudaErrorNotSupported;
  if (!a.sab_force && a.K < a.sab_kmin) return cudaErrorNotSupported;
  if (a.K % 16 || a.lda % 16 || ((uintptr_t)a.a_ptr & 15)) return cudaErrorNotSupported;
  if (a.M <= 16) return launch_sab_mp<16>(tmB, a, epi, st);
  if (a.M <= 32) return launch_sab_mp<32>(tmB, a, epi, st);
  if (a.M <= 64) return launch_sab_mp<64>(tmB, a, epi, st);
  return launch_sab_mp<128>(tmB, a, epi, st);
}

cudaError_t launch_gemm_i8(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                           int epi, int bn, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return cudaSuccess;
  if (!a.sab_force) {
    const cudaError_t e = launch_smallm(a, epi, st);
    // op level (smallm_force): a launch the small-M kernel cannot take is an error, never a
    // silent tcgen05 run
    if (e != cudaErrorNotSupported || a.smallm_force) return e;
  }
  {
    const cudaError_t e = launch_sab(tmB, a, epi, st);
    if (e != cudaErrorNotSupported || a.sab_force) return e;   // op level: never a silent fallback
  }
  if (is_topk(epi)) {   // fixed tile (the partial layout depends on it), never persistent
    if (a.part_ld < 2 * ((a.N + TOPK_BN - 1) / TOPK_BN)) return cudaErrorInvalidValue;
    if (epi == EPI_TOPK2) return launch_np<TOPK_BN, EPI_TOPK2>(tmA, tmB, a, st);
    if (epi == EPI_TOPK4) return launch_np<TOPK_BN, EPI_TOPK4>(tmA, tmB, a, st);
    return launch_np<TOPK_BN, EPI_TOPK>(tmA, tmB, a, st);
  }
  if (bn == -3) return launch_pers2(tmA, tmB, a, epi, st);   // op level: the CTA-pair kernel
  if (bn == 0) bn = gemm_pick_bn(a.M, a.N, a.pers_grid);
  // 32-wide tiles halve each epilogue warp's columns where the 64-wide grid is small
  // (env MNMT_BN32=0 disables; A/B)
  static const bool bn32 = [] {
    const char* e = getenv("MNMT_BN32");
    return !(e && e[0] == '0');
  }();
  if (bn32 && bn == 64 && (epi == EPI_F32 || epi == EPI_F32_Q || epi == EPI_RELU_Q ||
                           epi == EPI_RELU_F32_Q || epi == EPI_SIGMOID)) {
    const int tiles64 = ((a.N + 63) / 64) * ((a.M + BM - 1) / BM);
    const int sms = a.pers_grid > 0 ? a.pers_grid : num_sms();   // the launch's SM budget
    // K <= 512 only: the 32-wide tile still receives a 64-row B box, which costs more than
    // it saves for deep K (measured: big student 126 -> 131 ms per job without this bound)
    static const int bn32_kmax = [] {   // env MNMT_BN32_KMAX: deepest K of the 32-wide tiles (A/B)
      const char* e = getenv("MNMT_BN32_KMAX");
      return e ? atoi(e) : 512;
    }();
    if (tiles64 * 2 <= sms && a.N % 32 == 0 && (a.K <= bn32_kmax || (a.b_ptr && a.M <= 64 && abox_on())))
      bn = 32;
  }
  switch (bn) {
    case 32:
      switch (epi) {
        case EPI_F32: return launch_t<32, EPI_F32>(tmA, tmB, a, st);
        case EPI_F32_Q: return launch_t<32, EPI_F32_Q>(tmA, tmB, a, st);
        case EPI_RELU_Q: return launch_t<32, EPI_RELU_Q>(tmA, tmB, a, st);
        case EPI_RELU_F32_Q: return launch_t<32, EPI_RELU_F32_Q>(tmA, tmB, a, st);
        case EPI_SIGMOID: return launch_t<32, EPI_SIGMOID>(tmA, tmB, a, st);
      }
      return cudaErrorInvalidValue;
    case 64: return launch_bn<64>(tmA, tmB, a, epi, st);
    case 128: return launch_bn<128>(tmA, tmB, a, epi, st);
    case 256: return launch_bn<256>(tmA, tmB, a, epi, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mnmt
