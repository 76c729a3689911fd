// beam.h — beam-search step kernels (internal to libmnmt).
//
// Beam search of the b = 2 / 4 systems of Table 3, readings R26-R29
// (DESIGN.md).  A hypothesis is a decoder row; its SLOT is sentence * beam + k, so the
// per-row state the step kernels keep by slot (AAN running sums, self-attention cache) is the
// hypothesis' own.  Per step, after the EPI_TOPK output GEMM:
//   k_beam_rows     one warp per live row: log-sum-exp and the row's top-beam (logit, id)
//                   from the GEMM's per-tile partials;
//   k_beam_select   one CTA: per sentence, the best beam - finished candidates (R28),
//                   finished hypotheses written out, children stably compacted into slots;
//   k_beam_reorder  one CTA per sentence with children: state of parent -> child slot.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace mnmt {

struct BeamArgs {
  int beam;                  // b, 1..TOPK_MAX
  int n;                     // static row bound of the step (grids)
  int32_t* ctrl;             // [0] live rows, [1] t, [2] sentences of the batch, [3] sentences with children
  int32_t* live;             // compact row -> slot
  int32_t* prev_live;        // compact row -> input id of the next step
  int32_t* live_start;       // compact row -> source span
  int32_t* live_len;
  const int32_t* row_start;  // [sentence] source span (batch row order)
  const int32_t* row_len;
  const int32_t* max_len;    // [sentence]
  const int64_t* out_off;    // [sentence] prefix sum of max_len in the job
  const int32_t* len_idx;    // [sentence] -> job sentence index
  int eos;
  const TopkPart* part;      // [rows][part_ld] (EPI_TOPK)
  int part_ld, n_part;
  float* row_lse;            // [rows]
  float* row_v;              // [rows][TOPK_MAX]
  int32_t* row_j;
  int32_t* sent_row0;        // [sentence] first compact row this step
  int32_t* sent_nlive;       // [sentence] live hypotheses
  int32_t* sent_nfin;        // [sentence] finished hypotheses
  int32_t* sent_list;        // sentences with children, in order (k_beam_reorder grid)
  float* hscore;             // [slot] cumulative score of the live hypothesis
  int32_t* child_par;        // [slot] (sentence * beam + c): parent slot of child c
  int32_t* child_tok;
  float* child_score;
  int32_t* hist;             // [slot][t_cap] emitted ids
  int32_t* anc;              // [slot][t_cap] self-attention cache rows, or null (AAN)
  int t_cap;
  float* C;                  // AAN running sums [L][c_stride] (slot rows of d), or null
  int64_t c_stride;
  int L, d;
  const float* logits;       // beam_fused = 0: fp32 logits [rows][V] of the step (EPI_F32 GEMM)
  int V;
  int64_t ld_logits;         // row stride of logits (V rounded up to 16: aligned float4 rows)
  int32_t* out_ids;          // job outputs (see mnmt_beam_translate)
  int32_t* out_len;
  float* out_score;
  int32_t* n_hyp;
};

cudaError_t launch_beam_init(const BeamArgs& a, int n_sent, cudaStream_t st);
cudaError_t launch_beam_rows(const BeamArgs& a, cudaStream_t st);
// Same outputs as k_beam_rows, from materialised fp32 logits: one CTA per live row.
cudaError_t launch_beam_logits(const BeamArgs& a, cudaStream_t st);
cudaError_t launch_beam_select(const BeamArgs& a, cudaStream_t st);
cudaError_t launch_beam_reorder(const BeamArgs& a, cudaStream_t st);
cudaError_t launch_beam_final(const BeamArgs& a, int n_sent, cudaStream_t st);

}  // namespace mnmt
