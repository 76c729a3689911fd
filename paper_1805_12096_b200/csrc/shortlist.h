// shortlist.h — batch vocabulary shortlist kernels (internal to libmnmt).
//
// "the union of the 100 most frequent target words and the 100 most probable
// translations for every source word in a batch" (readings R32-R34 in DESIGN.md).
// Per word-budget batch b (the paper's batch):
//   k_sl_mark     bitmap[b] |= freq ∪ {lex[s][k] : s a source id of b} ∪ {EOS, UNK}
//                 (ids outside [0, V) ignored), one CTA group per batch, atomicOr into V/32 words;
//   k_sl_compact  one CTA per batch: ids of the set bits in ascending order (block prefix scan
//                 of the word popcounts) -> sl_ids[b][0..n_b), n_b -> sl_n[b];
//   k_sl_gather   per decode unit: the n_b rows of the memoized int8 E (and of the output bias)
//                 copied into the lane's contiguous [n_b x d] operand, plus the id map, so the
//                 output GEMM + argmax runs over n_b columns and k_finish maps column -> id.
// Integer work only: bit-exact by construction.  The shortlist is ascending, so the lowest
// column on an argmax tie is the lowest id (R15).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mnmt {

struct SlMarkArgs {
  int V, W;                  // vocabulary, bitmap words per batch (ceil(V / 32))
  const int32_t* src_ids;    // [tokens] job source ids
  const int32_t* sent_start; // [sentences of all batches, batch-major] first token in src_ids
  const int32_t* sent_len;
  const int32_t* bb_off;     // [n_bb + 1] sentence offsets of each word-budget batch
  const int32_t* freq;       // [n_freq]
  int n_freq;
  const int32_t* lex;        // [V][k_lex]
  int k_lex;
  int eos, unk;
  uint32_t* bits;            // [n_bb][W], zeroed by the caller
};

cudaError_t launch_sl_build(const SlMarkArgs& a, int n_bb, int32_t* sl_ids /*[n_bb][V]*/,
                            int32_t* sl_n /*[n_bb]*/, cudaStream_t st);

// dst_q[r] = qE[ids[r]] (d int8), dst_b[r] = bias[ids[r]] (bias may be null), dst_map[r] = ids[r],
// r < n; d % 16 == 0.
cudaError_t launch_sl_gather(const int32_t* ids, int n, const int8_t* qE, const float* bias, int d,
                             int8_t* dst_q, float* dst_b, int32_t* dst_map, cudaStream_t st);

}  // namespace mnmt
