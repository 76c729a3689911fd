// kernels.h — host-side launch interface of the sm_100a kernels (internal to libmnmt).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "rowops.h"

namespace mnmt {

// Epilogues of the int8 GEMM (acc = exact s32; v = fmaf((float)acc, s, bias)).
enum Epi : int {
  EPI_F32 = 0,        // out_f = v                       (projections, residual deltas)
  EPI_F32_Q = 1,      // out_f = v, out_q = Q(v)         (AAN FFN output a, needed as both)
  EPI_RELU_Q = 2,     // out_q = Q(ReLU(v))              (FFN1: ReLU straight to codes)
  EPI_RELU_F32_Q = 3, // out_f = ReLU(v), out_q = Q(.)   (AAN FFN depth 1)
  EPI_SIGMOID = 4,    // out_f = sigmoid(v)              (AAN gates)
  EPI_ARGMAX = 5,     // keys[row] = max packed(v, col)  (output layer, A9)
  EPI_ACC = 6,        // out_i = acc                     (test hook: raw accumulators)
  EPI_TOPK = 9,       // beam search (F1): per (row, N-tile half) the running max m, the fp64
                      // sum z = sum exp(v - m) and the TOPK_MAX largest (v, col) -> part[]
  EPI_TOPK2 = 10,     // as EPI_TOPK with the 2 / 4 largest (beam <= 2 / <= 4; the other
  EPI_TOPK4 = 11,     // record entries are empty)
};

// Beam-search partial of one row over one half of one N tile (EPI_TOPK).  v sorted by
// descending value, ties by ascending column; unused entries v = -inf, j = -1.
constexpr int TOPK_MAX = 8;
constexpr int TOPK_BN = 256;   // N tile of the EPI_TOPK launch: 2 partials per tile
struct __align__(16) TopkPart {
  float m;          // max v of the range (-inf: empty)
  int32_t pad;
  double z;         // sum over the range of exp((double)v - m)
  float v[TOPK_MAX];
  int32_t j[TOPK_MAX];
};

struct GemmArgs {
  int M;                       // rows covered by the grid (static upper bound)
  const int32_t* M_dyn;        // optional device row count (live rows), <= M
  int N, K;
  float scale;                 // s = fl32(c^2 / 127^2)
  const float* bias;           // [N] or nullptr
  float clip, sigma;
  float* out_f;
  int8_t* out_q;
  int32_t* out_i;
  int64_t ldo;                 // output row stride (elements)
  int col_block;               // scatter: out + (n / col_block) * block_stride + m * ldo + n % col_block
  int64_t block_stride;
  unsigned long long* keys;    // [rows] for EPI_ARGMAX
  // EPI_ARGMAX over a shortlist union (F2): column n is a candidate for row r only if bit n % 32
  // of colbits[g * colbits_ld + n / 32] is set, g = row_grp[row_live[r]] (colbits null: every
  // column)
  const uint32_t* colbits;
  int colbits_ld;
  const int32_t* row_grp;
  const int32_t* row_live;
  int pers_grid;               // persistent variant: CTA cap (0 = one per SM)
  unsigned long long* trace;   // debug: CTA (0,0) %globaltimer stamps [9] (null = off)
  TopkPart* part;              // EPI_TOPK: [rows][part_ld] partials (part_ld >= 2 * N tiles)
  int part_ld;
  // optional raw operands (row-major codes, K contiguous) for the small-M path: with
  // M <= the small-M row bound (<= SMALLM_MAX), a_ptr and b_ptr set, the fp32 / code epilogues
  // run as a CUDA-core IDP4A kernel (k_gemm_smallm) instead of the tcgen05 one
  const int8_t* a_ptr;
  int64_t lda;
  const int8_t* b_ptr;         // [N x K]
  int smallm_force;            // op level: take the small-M path whenever it can run (M <= 32)
  int smallm_rows;             // small-M path row bound of the launch (0 = off, <= SMALLM_MAX)
  int smallm_kmax;             // deepest K the small-M path takes
  int64_t smallm_wmax;         // largest weight matrix (N x K bytes) the small-M path takes
  // swap-AB tcgen05 path (k_gemm_sab): with a_ptr set and M <= sab_rows, the weights are the
  // MMA's 128-row operand and the M live rows its N = 16 / 32 / 64 / 128 operand
  int sab_rows;                // row bound of the swap-AB path (0 = off, <= 128)
  int sab_kmin;                // shallowest K the swap-AB path takes (model path; 0 = any)
  int sab_force;               // op level: take the swap-AB path for any M <= 128 (error otherwise)
  int sab_kb;                  // K blocks per CTA before K is split over a cluster (0 = default 8)
  int pers2;                   // BN = 256 persistent launches on CTA pairs (k_gemm_pers2): 1 on,
                               // -1 off, 0 the library default (env MNMT_PERS2)
  int a_box;                   // (launch-internal) k_gemm_i8: A loaded as one a_box-row box (0: 2 x 64)
  int b_box;                   // (launch-internal) k_gemm_i8: B loaded as one b_box-row box (0: 64-row boxes)
  int npsync;                  // (launch-internal) k_gemm_i8: CTA barrier before the PDL wait
  int ring_cap;                // (launch-internal) TMA ring depth cap of a split-K launch
  int split_k;                 // 0 / 1: no split-K; -1: the K / row-bound rule; 2, 4, 8: forced
                               // (capped by the leader's shared memory and the K blocks)
};

constexpr int SMALLM_MAX = 32;

// Tensor map over a row-major int8 matrix [rows x K] (K contiguous, K % 16 == 0):
// box {128 bytes, 64 rows}, 128-byte swizzle (the UMMA K-major SW128 atom).
bool make_tmap_i8(CUtensorMap* map, const void* base, int64_t rows, int64_t K);
// Tensor map over fp32 key/value rows [rows x cols] (cols contiguous, row stride = cols): box
// {32 floats, 8 rows} (one 128-byte swizzle atom), 128-byte swizzle (the attention K / V tiles).
bool make_tmap_kv(CUtensorMap* map, const void* base, int64_t rows, int64_t cols);

// A is [>= M x K] activation codes, B is [N x K] weight codes (both via make_tmap_i8).
// bn = 0 picks the N tile; -3 forces the CTA-pair persistent kernel (256 x 256 tiles).
cudaError_t launch_gemm_i8(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                           int epi, int bn, cudaStream_t st);

int gemm_pick_bn(int M, int N, int sms = 0);   // 64, 128 or 256 (sms: SM budget, 0 = device)

// Programmatic dependent launch on every kernel (env MNMT_NO_PDL=1 disables; A/B testing).
bool pdl_enabled();

// Sets the dynamic-smem attribute of every GEMM instantiation on the current device.
cudaError_t gemm_init();

}  // namespace mnmt
