// rowfused.h — fused per-row decoder blocks for small live-row counts (internal to libmnmt).
//
// At a few dozen live rows every decoder GEMM is one 128-row tile whose cost is latency (an
// operand round trip, the MMA, the epilogue, the release of the next kernel: ~3 us each, 42 of
// them on a step's critical path).  For such steps the d x d projections of a block run inside
// one kernel per block, one CTA per row, as exact int8 dot products (IDP4A, s32) against a
// k4-major copy of the weight codes: the s32 sums, the fmaf dequantization, the sigmoid, the
// residuals and the LayerNorm are the same arithmetic as the GEMM + row-kernel path (R3, R5, R8,
// R20), so the ids are identical; only the fp64 LayerNorm sums are ordered differently.
//   k_aan_block  a1 -> ReLU -> a2, i/f gates, gate combine, LN1      (A6)
//   k_src_block  q projection, source attention, o projection, LN2   (A7)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rowops.h"

namespace mnmt {

// One int8 linear map on the row path: out[c] = fmaf((float)(codes . W[c]), s, b[c]).
struct RowLin {
  const int32_t* W4;   // [d_in / 4][d_out]: W4[k4 * d_out + c] packs W[c][4 k4 .. 4 k4 + 3]
  const float* b;      // [d_out] or null
};

struct AanBlockArgs {
  int n;                     // static row bound (grid)
  const int32_t* n_dyn;      // live rows
  int d, depth, gate;        // AAN FFN depth 0/1/2, gated
  float scale, clip, sigma, eps;
  const float* y;            // [n x d] layer input
  const int8_t* yq;          // Q(y)
  const float* g_f;          // depth 0: g (a = g)
  const int8_t* g_q;         // Q(g)
  RowLin a1, a2, gi, gf;
  const float* gamma;        // LN1
  const float* beta;
  float* x1;                 // outputs
  int8_t* x1q;
};

struct SrcBlockArgs {
  int n;
  const int32_t* n_dyn;
  int d, H, span;            // span: longest source (sizes the score scratch)
  float scale, clip, sigma, eps;
  const float* x1;
  const int8_t* x1q;
  RowLin sq, so;
  const float* kv;           // source K|V of the layer, rows of ldkv floats
  int64_t ldkv;
  int k_off, v_off;
  const int32_t* live_start; // compact-order source spans
  const int32_t* live_len;
  const float* gamma;        // LN2
  const float* beta;
  float* x2;
  int8_t* x2q;
};

// W4 from row-major codes W [N x K] (K % 4 == 0).
cudaError_t launch_repack_k4(const int8_t* W, int N, int K, int32_t* W4, cudaStream_t st);
// d % 32 == 0, d <= 1024, d / H <= 64.
cudaError_t launch_aan_block(const AanBlockArgs& a, cudaStream_t st);
cudaError_t launch_src_block(const SrcBlockArgs& a, cudaStream_t st);
cudaError_t rowfused_init();   // dynamic-smem attributes (once per device, outside capture)

}  // namespace mnmt
