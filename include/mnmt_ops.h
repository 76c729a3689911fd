/*
 * mnmt_ops.h — op-level C ABI of libmnmt: each step of the decode path
 * as one call on caller-owned DEVICE memory.
 * Used by the kernel-level parity tests (P-1 of the parity protocol: inject the
 * oracle's exact operands) and by the benchmark's per-kernel timing.  The
 * model-level path (mnmt.h) runs the very same kernels.
 *
 * Conventions: every *_dev pointer is device memory on the current CUDA device,
 * row-major, 16-byte aligned; work is enqueued on `stream` and NOT synchronized.
 * Errors: MNMT_ERR_ARG for bad sizes/NULL pointers, MNMT_ERR_CUDA for launch
 * failures (no handle is involved, so nothing becomes fail-stop).
 * Quantization everywhere: Q(x) = RNE(clip(x, +-c) * 127/c) (R1, R2);
 * dequantization: fmaf((float)acc, s, b), s = fl32(c^2/127^2) (R5).
 */
#ifndef MNMT_OPS_H_
#define MNMT_OPS_H_

#include <stdint.h>

#include "mnmt.h"

#ifdef __cplusplus
extern "C" {
#endif

/* A1 / activation quantization: out[i] = Q(x[i]), n elements. */
mnmt_status mnmt_op_quantize(const float* x_dev, int64_t n, float clip, int8_t* out_dev,
                             void* stream);

/* Epilogues of mnmt_op_gemm_i8 (v = fmaf((float)acc, s, bias)). */
#define MNMT_EPI_F32 0        /* out fp32 [M x N] = v                              */
#define MNMT_EPI_F32_Q 1      /* out fp32 = v and out2 int8 = Q(v)                 */
#define MNMT_EPI_RELU_Q 2     /* out int8 = Q(ReLU(v))                             */
#define MNMT_EPI_RELU_F32_Q 3 /* out fp32 = ReLU(v), out2 int8 = Q(ReLU(v))        */
#define MNMT_EPI_SIGMOID 4    /* out fp32 = sigmoid(v) (fp64 exp, R20)             */
#define MNMT_EPI_ARGMAX 5     /* out u64 [M] = max over columns of packed (v, col); caller zeroes it */
#define MNMT_EPI_ACC 6        /* out int32 [M x N] = exact s32 accumulator         */
#define MNMT_EPI_TOPK 9       /* beam search (F1): out = [M][2 * ceil(N / 256)] records of 80 bytes,
                               * one per (row, 128-column half tile): {float m; int32 pad; double z;
                               * float v[8]; int32 j[8]} = max v, sum exp(v - m) in fp64, the 8
                               * largest (v, column) by (v desc, column asc); n_tile = 2 / 4 keeps
                               * only the 2 / 4 largest (the rest empty: v = -inf, column = -1) */

/* dotint(quant(A), quant(B^T)) = A . W^T on the int8 tensor cores (R3):
 * A [M x K] codes, W [N x K] codes (K % 16 == 0), bias [N] fp32 or NULL.
 * For EPI_F32* / SIGMOID / ACC, N % 16 == 0; out row stride = N.
 * n_tile = 0 (auto), 64, 128 or 256; -1 = the small-M CUDA-core kernel (IDP4A, same s32 sums and
 * epilogue arithmetic; M <= 32, EPI_F32 .. EPI_SIGMOID, A and W 16-byte aligned);
 * -2 = the swap-AB tcgen05 kernel (D^T = W . A^T: W's 128-row tiles as the MMA's M operand, the
 * M <= 128 rows of A as its N = 16 / 32 / 64 / 128 operand; same s32 sums and epilogue
 * arithmetic; every epilogue but EPI_TOPK; A 16-byte aligned); -3 = the CTA-pair persistent
 * kernel (256 x 256 tiles on a 2-CTA cluster, tcgen05 cta_group::2; any M; every epilogue but
 * EPI_TOPK).  Argument errors (not a silent fallback) when the chosen kernel cannot take the call. */
mnmt_status mnmt_op_gemm_i8(const int8_t* A_dev, const int8_t* W_dev, int32_t M, int32_t N,
                            int32_t K, const float* bias_dev, float clip, int32_t epilogue,
                            void* out_dev, void* out2_dev, int32_t n_tile, void* stream);

/* Argmax key -> id (the packed key of MNMT_EPI_ARGMAX; lowest id wins ties, R15). */
/* As mnmt_op_gemm_i8 with split-K: split_k = 2, 4, 8 spreads the K blocks of every output tile
 * over a thread-block cluster of that many CTAs (fewer when K has fewer 128-byte blocks or the
 * leader's shared memory cannot hold the partial slots; BN <= 128), whose exact s32 partials are
 * added in the leader before the epilogue; -1 = the library's rule (K >= 4096, or K >= 2048 at
 * <= 32 rows); 1 = none.  With n_tile = -2 (swap-AB) split_k = 1, 2, 4, 8 caps each CTA at
 * ceil(K blocks / split_k) K blocks (the kernel picks the power-of-two cluster that fits).
 * Outputs identical to mnmt_op_gemm_i8 (integer sums). */
mnmt_status mnmt_op_gemm_i8_split(const int8_t* A_dev, const int8_t* W_dev, int32_t M, int32_t N,
                                  int32_t K, const float* bias_dev, float clip, int32_t epi,
                                  void* out_dev, void* out2_dev, int32_t n_tile, int32_t split_k,
                                  void* stream);

mnmt_status mnmt_op_argmax_ids(const uint64_t* keys_dev, int32_t n, int32_t* ids_dev,
                               void* stream);

/* A3/A6-A8: out = LN(fl(x + delta)) (post-norm, fp64 statistics; R10, R20) and
 * out_q = Q(out).  Gate form (gi_dev != NULL, R8): gi/gf are the gate LOGITS of the two gate
 * products; out = LN(fl(x + fl(fl(s(gi)*x) + fl(s(gf)*delta)))), s = fp64 sigmoid (R20). */
mnmt_status mnmt_op_layernorm(const float* x_dev, const float* delta_dev, const float* gi_dev,
                              const float* gf_dev, const float* gamma_dev, const float* beta_dev,
                              int32_t n, int32_t d, float eps, float clip, float* out_dev,
                              int8_t* out_q_dev, void* stream);

/* A6 (AAN): one step t of the running sum for n rows: C <- fl(C + y),
 * g = fl(C / t); writes g (fp32, may be NULL) and Q(g) (may be NULL). */
mnmt_status mnmt_op_aan_step(float* C_dev, const float* y_dev, int32_t n, int32_t d, int32_t t,
                             float clip, float* g_dev, int8_t* g_q_dev, void* stream);

/* A2/A5: x = fl(fl(E[id] * fl32(sqrt d)) + PE[pos]) (id < 0: zero vector, R13) and Q(x). */
mnmt_status mnmt_op_embed(const float* E_dev, int32_t d, const int32_t* ids_dev,
                          const int32_t* pos_dev, int32_t n, float clip, float* x_dev,
                          int8_t* x_q_dev, void* stream);

/* A3/A7: attention of n query rows over per-row key/value spans (fp64, R20):
 * row r attends over kv rows kv_start[r] .. kv_start[r] + kv_len[r] - 1;
 * query at q + r*ldq, key j at kv + j*ldkv + k_off, value at kv + j*ldkv + v_off.
 * Head h uses columns [h*d/H, (h+1)*d/H) (R11).  out_q = Q(ctx) [n x d];
 * out_f (may be NULL) = ctx fp32.  kv_len[r] <= MNMT_MAX_SPAN. */
mnmt_status mnmt_op_attention(const float* q_dev, int64_t ldq, const float* kv_dev, int64_t ldkv,
                              int32_t k_off, int32_t v_off, const int32_t* kv_start_dev,
                              const int32_t* kv_len_dev, int32_t n, int32_t d, int32_t H,
                              float clip, int8_t* out_q_dev, float* out_f_dev, void* stream);

/* A3: encoder self-attention of n_sent sentences with the encoder's kernels (R20, R24):
 * qkv_dev [rows x 3d] holds each token's query | key | value (the fused QKV GEMM's output);
 * sentence s is rows sent_start[s] .. sent_start[s] + sent_len[s] - 1 and attends over itself;
 * s_max >= every sent_len (<= MNMT_MAX_KV; sizes shared memory).  out_q [rows x d] = Q(ctx).
 * variant 0 = the library's choice, 1 = the generic warp-per-query kernel, 2 / 3 = the d/H = 64
 * multi-query kernel with 4 / 8 queries per warp pass (s_max <= 100; argument error otherwise).
 * Every variant computes the same values in the same order (identical codes). */
mnmt_status mnmt_op_attention_enc(const float* qkv_dev, const int32_t* sent_start_dev,
                                  const int32_t* sent_len_dev, int32_t n_sent, int32_t d, int32_t H,
                                  int32_t s_max, float clip, int8_t* out_q_dev, int32_t variant,
                                  void* stream);

/* A7 with the decode path's kernel choice (the TMA-tiled source-attention kernel for fp32 K/V
 * and d/H = 32 or 64, else as mnmt_op_attention): row r attends kv rows
 * [kv_start[r], kv_start[r] + kv_len[r]) of the kv_rows-row buffer kv_dev (ldkv floats per row,
 * 16-byte aligned; the TMA tensor map is bounded by kv_rows); max_span >= every kv_len[r]
 * (<= MNMT_MAX_KV; sizes shared memory).  Same outputs as mnmt_op_attention. */
mnmt_status mnmt_op_src_attention(const float* q_dev, int64_t ldq, const float* kv_dev,
                                  int64_t kv_rows, int64_t ldkv, int32_t k_off, int32_t v_off,
                                  const int32_t* kv_start_dev, const int32_t* kv_len_dev,
                                  int32_t max_span, int32_t n, int32_t d, int32_t H, float clip,
                                  int8_t* out_q_dev, float* out_f_dev, void* stream);

/* As mnmt_op_src_attention with the one-warp TMA kernel in fp32 arithmetic (the model option
 * "attn_f32"): fp32 dot products in order, expf, fp32 normaliser and context sums.  It departs
 * from R20 (fp64 sums): ctx agrees with the oracle to ~1e-6 relative and codes differ only at
 * rounding boundaries; long spans at <= 128 rows still take the fp64 split kernel.  d / H = 32
 * or 64 (argument error otherwise). */
mnmt_status mnmt_op_src_attention_f32(const float* q_dev, int64_t ldq, const float* kv_dev,
                                      int64_t kv_rows, int64_t ldkv, int32_t k_off, int32_t v_off,
                                      const int32_t* kv_start_dev, const int32_t* kv_len_dev,
                                      int32_t max_span, int32_t n, int32_t d, int32_t H, float clip,
                                      int8_t* out_q_dev, float* out_f_dev, void* stream);

/* As mnmt_op_attention with bf16 keys / values: kv16 holds bfloat16 bit
 * patterns (uint16) in the same layout (strides and offsets in elements, multiples of 4). */
mnmt_status mnmt_op_attention_bf16(const float* q_dev, int64_t ldq, const uint16_t* kv16_dev,
                                   int64_t ldkv, int32_t k_off, int32_t v_off,
                                   const int32_t* kv_start_dev, const int32_t* kv_len_dev,
                                   int32_t n, int32_t d, int32_t H, float clip, int8_t* out_q_dev,
                                   float* out_f_dev, void* stream);


/* A11 on several GPUs: ids back in input order after the id gather of a
 * strong-scaling run.  Source row i (ids src_dev[src_off[i] .. + src_len[i]), src_len[i] >= 0)
 * is copied to dst_dev[dst_off[dst_row[i]] ..] and dst_len[dst_row[i]] = src_len[i].
 * src_off_dev, dst_off_dev: int64 [n] / [max dst_row + 1]; dst_row_dev: int32 [n], distinct.
 * Rows may not overlap in dst.  One warp per row. */
mnmt_status mnmt_op_gather_rows(const int32_t* src_dev, const int64_t* src_off_dev,
                                const int32_t* src_len_dev, const int32_t* dst_row_dev,
                                const int64_t* dst_off_dev, int32_t n, int32_t* dst_dev,
                                int32_t* dst_len_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MNMT_OPS_H_ */
