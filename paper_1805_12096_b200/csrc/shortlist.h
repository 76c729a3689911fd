// shortlist.h — batch vocabulary shortlist kernels (internal to libmnmt).
//
// "the union of the 100 most frequent target words and the 100 most probable
// translations for every source word in a batch" (readings R32-R34 in DESIGN.md).
// Per word-budget batch b (the paper's batch):
//   k_sl_mark     bitmap[b] |= freq ∪ {lex[s][k] : s a source id of b} ∪ {EOS, UNK}
//                 (ids outside [0, V) ignored), one CTA group per batch, atomicOr into V/32 words;
// Per decode wave w (up to SL_MAX_GROUPS consecutive batches decoded together):
//   k_sl_wave     one CTA per wave: U_w = the union of its batches' bitmaps, in ascending id
//                 order (block prefix scan of the word popcounts) -> ids[w][0..n_w), and per
//                 column u the group mask  mask[w][u] bit g = (U_w[u] is in batch b0 + g's list);
//   k_sl_gather   per decode unit: the n_w rows of the memoized int8 E (and of the output bias)
//                 copied into the lane's contiguous [n_w x d] operand with the id map, and the
//                 masks transposed into one column bitmap per group (a warp ballot per 32
//                 columns), so the output GEMM + argmax runs over n_w columns, each row only
//                 over the columns of its own batch's shortlist (one 32-bit word per 32-column
//                 chunk), and k_finish maps column -> id.
// Integer work only: bit-exact by construction.  The union is ascending and a row's allowed
// columns are exactly its batch's shortlist, so the lowest id still wins ties (R15).
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

constexpr int SL_MAX_GROUPS = 64;   // batches per decode wave (bits of a column mask)

// Marks every batch's bitmap, then builds every wave's union, ids and masks.
// wave_off: [n_waves + 1] first batch of each wave.
cudaError_t launch_sl_build(const SlMarkArgs& a, int n_bb, const int32_t* wave_off, int n_waves,
                            int32_t* wave_ids /*[n_waves][V]*/,
                            unsigned long long* wave_mask /*[n_waves][V]*/,
                            int32_t* wave_n /*[n_waves]*/, cudaStream_t st);

// r < n: dst_q[r] = qE[ids[r]] (d int8), dst_b[r] = bias[ids[r]] (dst_b null: skipped),
// dst_map[r] = ids[r]; for g < n_groups, bit r % 32 of dst_bits[g * ld + r / 32] = bit g of
// mask[r] (ld >= ceil(n / 32)); d % 16 == 0.
cudaError_t launch_sl_gather(const int32_t* ids, const unsigned long long* mask, int n,
                             int n_groups, const int8_t* qE, const float* bias, int d,
                             int8_t* dst_q, float* dst_b, int32_t* dst_map, uint32_t* dst_bits,
                             int ld, cudaStream_t st);

}  // namespace mnmt
