/*
 * mnmt.h — C ABI of libmnmt: batched greedy (beam-1) decoding of a distilled
 * Transformer / AAN student with int8 matrix products on one B200 (sm_100a).
 *
 * The calls follow the paper's statement of the problem (arXiv 1805.12096,
 * /root/reference/PAPER.md, cited P:L<n>): load a student of Table 1's
 * dimensions with tied source/target/output embeddings over a
 * 36,000-entry joint vocabulary; quantize every parameter matrix once
 * (memoization of quant(B^T); int8 clip [-2,2] -> [-127,127],
 * P:L94); sort sentences by source length and cut word-budget batches
 * (P:L42); decode with beam 1, softmax skipped, "select the output word with
 * highest activation".  Readings of points the paper leaves open are
 * numbered R<k> in DESIGN.md.
 *
 * Conventions shared by every call:
 *   - Every call returns an mnmt_status; nothing throws or aborts across the ABI.
 *     mnmt_last_error() describes the last failure of the calling thread.
 *   - Pointers named *_host are host memory owned by the caller, read or written
 *     only during the call.  Pointers named *_dev are device memory on the
 *     model's GPU, owned by the caller.
 *   - One host thread per model handle at a time; handles are independent.
 *   - A CUDA failure returns MNMT_ERR_CUDA once and makes the handle fail-stop:
 *     every later call on it returns MNMT_ERR_STATE.
 */
#ifndef MNMT_H_
#define MNMT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MNMT_ABI_VERSION 2

typedef enum {
  MNMT_OK = 0,
  MNMT_ERR_ARG = 1,       /* bad argument: budget < 1, n < 0, bad config field, NULL pointer */
  MNMT_ERR_DIM = 2,       /* unknown parameter name or wrong element count */
  MNMT_ERR_VOCAB = 3,     /* token id < 0 or >= vocab */
  MNMT_ERR_STATE = 4,     /* call-order violation, missing parameters, or fail-stopped handle */
  MNMT_ERR_CAPACITY = 5,  /* output capacity too small, or a span > MNMT_MAX_SPAN */
  MNMT_ERR_CUDA = 6,      /* CUDA runtime/driver failure (handle becomes fail-stop) */
  MNMT_ERR_OOM = 7        /* device allocation failed */
} mnmt_status;

/* Longest source sentence / number of decoder steps per sentence. */
#define MNMT_MAX_SPAN 512

/* Student configuration (Table 1; AAN block P:L70-72). */
typedef struct {
  int32_t abi_version;    /* = MNMT_ABI_VERSION */
  int32_t d_model;        /* embedding / model width d; d % 16 == 0, d % n_heads == 0, d <= 1024 */
  int32_t d_ffn;          /* FFN width F; F % 16 == 0 */
  int32_t n_heads;        /* H; d / H <= 64 and (d / H) % 4 == 0 (R11) */
  int32_t enc_layers;     /* 6 in the paper */
  int32_t dec_layers;     /* 6 in the paper */
  int32_t vocab;          /* V = 36000 */
  int32_t decoder;        /* 1 = AAN; 0 = self-attention with a KV cache */
  int32_t aan_ffn_depth;  /* AAN FFN, hidden width = d (R9): 0 = "-ffn", 1, 2 (default) */
  int32_t aan_gate;       /* 1 = gated AAN (default; R8), 0 = "-gate" */
  int32_t out_bias;       /* 1 = output bias present (default; R14) */
  int32_t eos_id;         /* end-of-sentence id, default 0 (R16) */
  float clip;             /* quantization clip c = 2.0 */
  float ln_eps;           /* LayerNorm epsilon, default 1e-6 (R10) */
  int32_t src_kv_bf16;    /* 0 (default): the source keys / values K_l, V_l are fp32 (R4);
                           * 1: they are rounded (RNE) to bf16 once per batch and source
                           * attention reads them at half the bytes */
} mnmt_config;

typedef struct mnmt_model mnmt_model;   /* opaque; owns all of its device memory */

/* Fills *cfg with the defaults above and the given Table-1 widths. */
void mnmt_config_default(mnmt_config* cfg, int32_t d_model, int32_t d_ffn, int32_t n_heads);

/* Creates a model on CUDA device `cuda_device` (the caller's current device is
 * restored).  Errors: MNMT_ERR_ARG (bad config), MNMT_ERR_CUDA, MNMT_ERR_OOM. */
mnmt_status mnmt_model_create(const mnmt_config* cfg, int32_t cuda_device, mnmt_model** out);

/* Copies one fp32 parameter.  `name` is a manifest name (DESIGN.md "Parameter
 * manifest"), e.g. "emb.E" [V x d], "dec.3.src.q.W" [d x d]; every W is row-major
 * [out x in], i.e. already the B^T operand of dotint(A, B).
 * Errors: MNMT_ERR_DIM (unknown name / wrong numel), MNMT_ERR_STATE (after quantize). */
mnmt_status mnmt_model_set_param(mnmt_model* m, const char* name, const float* host,
                                 int64_t numel);

/* One-time weight preparation: quantizes every parameter matrix to int8 codes on
 * the device and builds its TMA descriptors — the memoized quant(B^T) of
 * P:L100-105.  Errors: MNMT_ERR_STATE (missing parameters; names listed in
 * mnmt_last_error()), MNMT_ERR_CUDA, MNMT_ERR_OOM. */
mnmt_status mnmt_model_quantize(mnmt_model* m);

/* Length-sorted word-budget batching (R17).  Stable sort of sentence
 * indices by (src_len, index); a batch closes as soon as it holds >= budget
 * words; the last batch may be short.  order[n], batch_off[n+1] (only the first
 * *n_batches + 1 entries are written).  Host-only.  Errors: MNMT_ERR_ARG. */
mnmt_status mnmt_batch_by_words(const int32_t* src_len_host, int32_t n, int32_t word_budget,
                                int32_t* order_host, int32_t* batch_off_host,
                                int32_t* n_batches);

/* Greedy decode of n sentences as ONE batch (rows are independent: static
 * scales).  Source sentence i is src_ids[src_off[i] .. src_off[i+1]);
 * it decodes at most max_len[i] steps, stopping at EOS (not emitted) (R16).
 * Its ids are written to out_ids[O_i ...] with O_i = sum_{k<i} max_len[k];
 * out_len[i] = number written.  Work is enqueued on `cuda_stream` (NULL =
 * legacy default stream) and the stream is synchronized before returning.
 * Errors: MNMT_ERR_ARG, MNMT_ERR_VOCAB, MNMT_ERR_CAPACITY (out_cap < sum max_len,
 * or a span > MNMT_MAX_SPAN), MNMT_ERR_STATE (before quantize), MNMT_ERR_CUDA. */
mnmt_status mnmt_decode(mnmt_model* m, const int32_t* src_ids_host, const int64_t* src_off_host,
                        int32_t n, const int32_t* max_len_host, int32_t* out_ids_host,
                        int64_t out_cap, int32_t* out_len_host, void* cuda_stream);

/* The whole translation job: batch_by_words(word_budget), then every batch is
 * decoded back to back on one stream (one synchronization at the end); outputs
 * are in INPUT order with the layout of mnmt_decode.
 * flags & MNMT_DEVICE_IO: src_ids and out_ids/out_len are device pointers (the
 * ids are already resident in HBM; offsets and max_len stay host arrays).
 * Errors as mnmt_decode. */
#define MNMT_DEVICE_IO 1u
/* flags & MNMT_SHORTLIST: vocabulary shortlist ("the union of the 100
 * most frequent target words and the 100 most probable translations for every source word in a
 * batch").  Every word-budget batch decodes with the argmax restricted to its
 * shortlist = freq ∪ {lex[s][k] : s a source id of the batch} ∪ {eos_id, MNMT_UNK_ID} (the
 * tables of mnmt_model_set_shortlist; ids outside [0, vocab) ignored), ascending, so the lowest
 * id still wins ties (R15, R32-R34).  Batches co-scheduled in one decode wave (at most 64
 * with a shortlist) share one output GEMM over the union of their shortlists, each row masked
 * to its own batch's columns, so ids do not depend on the scheduling.  Greedy only.
 * Errors: MNMT_ERR_STATE without tables, MNMT_ERR_ARG with beam search. */
#define MNMT_SHORTLIST 2u
#define MNMT_UNK_ID 1   /* reserved ids EOS/UNK/PAD = 0/1/2 */
mnmt_status mnmt_translate(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off_host,
                           int32_t n, const int32_t* max_len_host, int32_t word_budget,
                           int32_t* out_ids, int64_t out_cap, int32_t* out_len, uint32_t flags,
                           void* cuda_stream);

/* Shortlist tables (S:L435-443, S:L497 format), copied to the device:
 *   freq[0..n_freq)          the most frequent target ids (host int32; any order)
 *   lex[s * k_lex + k]       the k_lex most probable translations of source id s, s < vocab
 *                            (host int32 [vocab x k_lex]; entries outside [0, vocab), e.g. -1
 *                            as padding, are ignored)
 * Replaces earlier tables.  Errors: MNMT_ERR_ARG (negative sizes, NULL non-empty table),
 * MNMT_ERR_CUDA. */
mnmt_status mnmt_model_set_shortlist(mnmt_model* m, const int32_t* freq, int32_t n_freq,
                                     const int32_t* lex, int32_t k_lex);

/* Beam search over the same word-budget batches as mnmt_translate: the
 * b = 2 / 4 systems of Table 3 (rows 5, 6, 8, 9, 11, 12).  Per step,
 * every live hypothesis is expanded over log-softmax(logits) (lse = fl32(M + log sum exp(l - M)),
 * fp64 sum, R26); a candidate scores fl32(score + fl32(l_j - lse)) (R27); per sentence the best
 * beam - (finished so far) candidates are kept in the order (score desc, logit desc, hypothesis
 * rank asc, id asc) (R28); a kept EOS candidate is finished (EOS not emitted), and at step
 * max_len[i] every kept candidate is; the search of a sentence ends when it has beam finished
 * hypotheses.  No length normalisation.  Decoder state (AAN running sums, self-attention cache
 * through per-position ancestor rows, R29) follows each hypothesis.
 * beam: 1..8 (1 = greedy decoding through the log-softmax path; ids equal mnmt_translate's).
 * Outputs, sentence i in INPUT order, O_i = sum_{k<i} max_len[k]:
 *   hypothesis r (r < n_hyp[i], by descending score) at out_ids[beam * O_i + r * max_len[i] ...],
 *   length out_len[i * beam + r], score out_score[i * beam + r] (fp32 sum of log-probabilities).
 * n_hyp[i] = beam when max_len[i] >= 1, else 0.  out_cap >= beam * sum(max_len).
 * flags & MNMT_DEVICE_IO: src_ids and every output are device pointers.
 * Errors as mnmt_translate; MNMT_ERR_ARG for beam outside 1..8 or beam > vocab. */
mnmt_status mnmt_beam_translate(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off_host,
                                int32_t n, const int32_t* max_len_host, int32_t word_budget,
                                int32_t beam, int32_t* out_ids, int64_t out_cap, int32_t* out_len,
                                float* out_score, int32_t* n_hyp, uint32_t flags,
                                void* cuda_stream);

/* Teacher-forced decode (test hook for the parity protocol):
 * sentence i runs T_i = forced_off[i+1] - forced_off[i] steps; the input at step
 * t >= 2 is forced_ids[forced_off[i] + t - 2]; argmax_ids[forced_off[i] + t - 1]
 * receives the model's argmax at step t.  No EOS stop.
 * dump_mask selects intermediates copied to dump_host (sections in bit order):
 *   MNMT_DUMP_ENC_OUT   fp32 [sum S_i][d]         encoder output
 *   MNMT_DUMP_SRC_KV    fp32 [L][sum S_i][2][d]   source keys | values per layer
 *   MNMT_DUMP_DEC_OUT   fp32 [sum T_i][d]         last decoder layer output per step
 *   MNMT_DUMP_OUT_CODES int8 [sum T_i][d]         Q(dec_out): the output-layer operand
 *   MNMT_DUMP_LAYERS    fp32 [sum T_i][L][3][d]   x1, x2, x3 of every decoder layer
 *   MNMT_DUMP_MARGIN    fp32 [sum T_i]            top2_margin: largest minus second largest
 *                                                 output logit of the step (near-tie flag of
 *                                                 the parity protocol), (float)((double)v1 - v2)
 * Errors as mnmt_decode; MNMT_ERR_CAPACITY if dump_cap is too small. */
#define MNMT_DUMP_ENC_OUT 1u
#define MNMT_DUMP_SRC_KV 2u
#define MNMT_DUMP_DEC_OUT 4u
#define MNMT_DUMP_OUT_CODES 8u
#define MNMT_DUMP_LAYERS 16u
#define MNMT_DUMP_MARGIN 32u
mnmt_status mnmt_decode_forced(mnmt_model* m, const int32_t* src_ids_host,
                               const int64_t* src_off_host, int32_t n,
                               const int32_t* forced_ids_host, const int64_t* forced_off_host,
                               int32_t* argmax_ids_host, uint32_t dump_mask, void* dump_host,
                               int64_t dump_cap, void* cuda_stream);

/* Teacher-forced decode through the whole mnmt_translate schedule (test hook, P-2 at the
 * launch configuration the benchmark times): word-budget batches, co-scheduled waves,
 * decoder lanes / length tiers / SM partitions and small-M GEMMs as set by the options, every
 * step replayed from its captured CUDA graph.  Inputs, outputs and the DEC_OUT / OUT_CODES /
 * LAYERS dump sections as mnmt_decode_forced (rows in forced_off order); the dumps are written
 * by a copy kernel captured in the step graphs, so the kernels under test run unchanged.
 * Errors as mnmt_decode_forced; MNMT_ERR_ARG for word_budget < 1 or the encoder dump bits
 * (ENC_OUT, SRC_KV: one-batch calls only). */
mnmt_status mnmt_translate_forced(mnmt_model* m, const int32_t* src_ids_host,
                                  const int64_t* src_off_host, int32_t n,
                                  const int32_t* forced_ids_host, const int64_t* forced_off_host,
                                  int32_t word_budget, int32_t* argmax_ids_host,
                                  uint32_t dump_mask, void* dump_host, int64_t dump_cap,
                                  void* cuda_stream);

/* Runtime options (not part of the method; they change scheduling only, never results —
 * rows are independent, so ids are identical for every setting):
 *   "max_concurrent_rows"  mnmt_translate co-schedules consecutive word-budget batches in
 *                          one decode wave while the wave holds at most this many sentences
 *                          (0 = default = one batch at a time).  A single >=8192-word batch
 *                          (~375 sentences) cannot fill 148 SMs.
 *   "lanes"                1..16 independent decoders (workspace + stream + step graph);
 *                          each wave's sentences are dealt round-robin to the lanes in
 *                          length order and the lanes' kernel chains overlap (default 1).
 *   "steps_per_graph"      1..63 consecutive decoder steps captured in one CUDA graph (default 1).
 *   "smallm"               0..32 row bound (default 32): greedy decoder steps with at most this many
 *                          live rows run their fp32 / code-output GEMMs with K <= "smallm_kmax" as
 *                          IDP4A CUDA-core kernels (same s32 accumulators, same epilogue arithmetic,
 *                          bit-identical outputs); 0: tcgen05 always.  Per model.
 *   "smallm_kmax"          deepest K the small-M path takes (default 512, per model).
 *   "smallm_wmax"          largest weight matrix N x K (bytes) the small-M path takes (default
 *                          2^20: the d x d maps of the big student, not its FFN / Q|K|V maps).
 *   "attn_tma_self"        self-attention decoder: 1 = long decodes at <= 128 rows attend through
 *                          the TMA-tiled split kernel, 2 (default) = every step through TMA tiles,
 *                          0 = the generic kernels (identical results up to fp64 summation order,
 *                          R25; measured: 2 fastest on base and big).
 *   "split_k"              1: decoder GEMMs with K >= 4096 (or >= 2048 at <= 32 rows) spread their
 *                          K blocks over a 2-4 CTA cluster (exact s32 partials added in the
 *                          leader); 0 (default; measured slower in the 3-lane job).
 *   "lane_tiers"           0 (default): a wave's sentences are dealt round-robin to the lanes;
 *                          10*p: contiguous length tiers of equal sum S_i^p, the last lane (the
 *                          longest sentences, the job's critical path) on the highest-priority stream.
 *   "pers_reserve"         SMs the persistent GEMMs of the other lanes leave free (default 0).
 *   "green_sms"            0 (default) or a multiple of 8: with tiered lanes, the critical lane's
 *                          streams live in a green context (SM partition) of this many SMs and the
 *                          other lanes' in one holding the rest.
 *   "beam_fused"           beam search: 1 = log-sum-exp partials and top-k fused into the output
 *                          GEMM epilogue (EPI_TOPK*, logits never reach HBM); 0 (default, measured
 *                          faster) = fp32 logits written by the GEMM, reduced by one CTA per row.
 * Errors: MNMT_ERR_ARG (unknown name or negative value). */
mnmt_status mnmt_model_set_option(mnmt_model* m, const char* name, int64_t value);

/* Statistics of the last mnmt_translate / mnmt_decode call. */
typedef struct {
  int64_t gpu_launches;     /* kernels launched (graph nodes counted per replay) */
  int64_t decode_steps;     /* decoder steps summed over batches */
  int64_t batches;
  int64_t target_words;     /* ids emitted (EOS excluded) */
  int64_t h2d_bytes, d2h_bytes;
} mnmt_stats;
mnmt_status mnmt_get_stats(const mnmt_model* m, mnmt_stats* out);

/* Thread-local description of the last failure; valid until the next call. */
const char* mnmt_last_error(void);

/* Frees every device allocation of the handle.  NULL is a no-op. */
void mnmt_model_destroy(mnmt_model* m);

#ifdef __cplusplus
}
#endif
#endif /* MNMT_H_ */
