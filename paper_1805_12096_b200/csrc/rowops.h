// rowops.h — launch interface of the HBM-bound kernels (internal to libmnmt).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#define MNMT_MAX_KV 512   // longest attended span (source length or decoder steps)

namespace mnmt {

// Optional "next layer AAN step" fused into a row kernel (R6/R7):
// C[orig] <- fl(C + y); g = fl(C / t); writes g (fp32, for -ffn) and/or Q(g).
struct AanOut {
  float* C;          // [rows_cap x d] state of the layer being entered, indexed by orig row; null = off
  float* g_f;        // compact [n x d] or null
  int8_t* g_q;       // compact [n x d] or null
  float clip, sigma;
};

struct EmbedTgtArgs {
  int n;                    // static row bound (grid)
  const int32_t* ctrl;      // [0] = live rows, [1] = t
  const int32_t* live;      // compact -> original row
  const int32_t* prev_id;   // [orig] previous output id
  const int32_t* prev_live; // optional: [compact] previous output id (written by k_finish)
  const float* E;
  const float* PE;
  int d;
  float rsd;                // fl32(sqrt d)
  float* y;                 // compact [n x d]
  int8_t* yq;
  AanOut aan;
};

struct LnArgs {
  int n;                    // static row bound
  const int32_t* n_dyn;     // live rows (device) or null
  const int32_t* ctrl;      // for t when aan.C is set
  const int32_t* live;      // for orig when aan.C is set
  int d;
  float eps;
  const float* x;           // residual input (for the gate form: y)
  const float* delta;       // added to x (for the gate form: a)
  const float* gi;          // gate form when non-null: gate LOGITS; r = x + (s(gi)*x + s(gf)*delta)
  const float* gf;
  const float* gamma;
  const float* beta;
  float* out;               // fp32 output or null
  int8_t* out_q;            // Q(out) or null
  float clip, sigma;
  AanOut aan;
};

enum AttnMode : int { ATTN_ENC = 0, ATTN_SRC = 1, ATTN_SELF = 2 };

struct bf16s { uint16_t u; };   // bf16 bits (source K/V storage, F3)

struct AttnArgs {
  int mode;
  int span;                 // longest attended span of the launch (<= MNMT_MAX_KV; sizes smem)
  int n;                    // static row bound
  const int32_t* n_dyn;
  const int32_t* ctrl;      // t (self mode)
  const int32_t* live;      // compact -> orig (src / self)
  int H, dh, d;
  const float* q;           // query rows, row stride ldq (self mode: the qkv rows)
  int64_t ldq;
  const float* kv;          // key/value rows, row stride ldkv; K at +k_off, V at +v_off
  float* kv_w;              // self mode: writable cache (same as kv)
  const bf16s* kv16;        // src mode, optional: bf16 copy of kv (same layout), read instead (F3)
  int64_t ldkv;
  int k_off, v_off;
  const int32_t* kv_start;  // enc: [row]; src: [orig]
  const int32_t* kv_len;
  const int32_t* live_start;   // optional (src): kv_start / kv_len in compact row order
  const int32_t* live_len;
  int t_cap;                // self mode: cache rows per sentence
  int32_t* anc;             // self mode, beam search: [slot][t_cap] cache row of each position (R29)
  float clip, sigma;
  int8_t* out_q;            // Q(ctx) [n x d]
  float* out_f;             // optional fp32 ctx (tests)
  // optional TMA path (SRC / op-level ENC, fp32 K/V, d_h = 32 / 64): a make_tmap_kv map over
  // the K/V rows; this launch's kv == the map's base + kv_row0 rows
  const CUtensorMap* tmap;
  int64_t kv_row0;
  int tma_self;             // self mode: 0 generic kernels, 1 TMA split kernel for long decodes at
                            // <= 128 rows, 2 also the one-warp TMA kernel (measured per workload)
  int f32;                  // one-warp TMA kernel in fp32 arithmetic (model option attn_f32; departs
                            // from R20: ids exact or near-tie-explained, intermediates not within 1e-4)
};

// Encoder self-attention over Q|K|V rows [M x 3d] (A3), one CTA per (sentence, head).
struct EncAttnArgs {
  const float* qkv;
  const int32_t* sent_start;   // [n_sent] first token row of each sentence
  const int32_t* sent_len;     // [n_sent]
  const int32_t* sent_order;   // optional: CTA x -> sentence sent_order[x] (a length bucket)
  int n_sent, H, dh, d;        // n_sent: CTAs in x (sentences of this launch)
  int s_max;                   // longest sentence of the launch (sizes shared memory)
  float clip, sigma;
  int8_t* out_q;               // Q(ctx) [M x d]
};

struct FinishArgs {
  int32_t* ctrl;
  int32_t* live;
  unsigned long long* keys;
  int32_t* prev_id;
  const int32_t* max_len;   // [orig]
  const int64_t* out_off;   // [orig]
  int32_t* out_ids;
  int32_t* out_len;         // [len_idx[orig]] (len_idx null: [orig])
  const int32_t* len_idx;   // batch row -> sentence index in the job
  int eos;
  const int32_t* forced;    // teacher forcing ids (flat) or null
  const int64_t* forced_off;
  // optional compact-order copies for the next step (written at each kept row's new index)
  int32_t* prev_live;       // next input id
  const int32_t* row_start; // [orig] source span
  const int32_t* row_len;
  int32_t* live_start;
  int32_t* live_len;
  const int32_t* id_map;    // shortlist (F2): GEMM column -> vocabulary id, or null
};

// Teacher-forced dumps (test hook): live row r of src [n x d] (elem bytes per element) is
// copied to dst + ((foff[live[r]] + t - 1) * slots + slot) * d * elem.
struct DumpArgs {
  int n;                    // static row bound
  const int32_t* ctrl;      // [0] live rows, [1] t
  const int32_t* live;      // compact -> batch row
  const int64_t* foff;      // [batch row] forced offset
  int d, elem;
  const void* src;
  void* dst;
  int64_t slot, slots;
};

cudaError_t launch_quantize(const float* x, int64_t n, float clip, int8_t* out, cudaStream_t st);
cudaError_t launch_pe_table(float* pe, int max_pos, int d, cudaStream_t st);
// x[i] = emb(ids[idx[i]], pos[i]) (idx may be null; id < 0 = zero vector) and Q(x).
cudaError_t launch_embed_src(const int32_t* ids, const int32_t* idx, const int32_t* pos, int M,
                             const float* E, const float* PE, int d, float clip, float* x,
                             int8_t* xq, cudaStream_t st);
cudaError_t launch_embed_tgt(const EmbedTgtArgs& a, int rows, cudaStream_t st);
cudaError_t launch_ln(const LnArgs& a, cudaStream_t st);
cudaError_t launch_attn(const AttnArgs& a, cudaStream_t st);
cudaError_t launch_kv_bf16(float* kv, bf16s* kv16, int L, int64_t n, int64_t stride, cudaStream_t st);
cudaError_t launch_attn_enc(const EncAttnArgs& a, cudaStream_t st);
// variant 0: the library's choice; 1: the generic warp-per-query kernel; 2 / 3: the d_h = 64
// multi-query kernel with 4 / 8 queries per warp pass (cudaErrorNotSupported otherwise)
cudaError_t launch_attn_enc_v(const EncAttnArgs& a, int variant, cudaStream_t st);
cudaError_t attn_init();   // dynamic-smem attribute (call once per device, outside capture)
cudaError_t launch_finish(const FinishArgs& a, cudaStream_t st);
cudaError_t launch_dump_rows(const DumpArgs& a, cudaStream_t st);
// Teacher-forced top-2 margin dump (test hook): live row r's output
// logits' largest minus second largest value, (float)((double)v1 - (double)v2), from the
// per-tile top-2 partials of an EPI_TOPK2 output GEMM ([rows][part_ld], n_part used), written
// to dst[foff[live[r]] + t - 1].
struct TopkPart;
cudaError_t launch_top2_margin(const TopkPart* part, int part_ld, int n_part, int n,
                               const int32_t* ctrl, const int32_t* live, const int64_t* foff,
                               float* dst, cudaStream_t st);
// live[r] = r, keys = 0, ctrl = {B, 1}; live_start/live_len (optional) = row_start/row_len.
cudaError_t launch_decode_init(int32_t* ctrl, int32_t* live, int B, unsigned long long* keys,
                               const int32_t* row_start, const int32_t* row_len,
                               int32_t* live_start, int32_t* live_len, cudaStream_t st);
cudaError_t launch_aan_step_rows(float* C, const float* y, int n, int d, int t, const AanOut& o,
                                 cudaStream_t st);
cudaError_t launch_argmax_ids(const unsigned long long* keys, int n, int32_t* ids, cudaStream_t st);

}  // namespace mnmt
