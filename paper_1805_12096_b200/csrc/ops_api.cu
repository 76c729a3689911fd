// ops_api.cu — op-level C ABI (include/mnmt_ops.h): each decode-path kernel on caller memory.
#include <cstdio>
#include <string>
#include <cstdlib>
#include <vector>

#include "../../include/mnmt_ops.h"
#include "kernels.h"
#include "rowops.h"

using namespace mnmt;

// defined in mnmt.cu
extern "C" const char* mnmt_last_error(void);
void mnmt_set_error_str(const char* s);

namespace {
mnmt_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MNMT_OK;
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  mnmt_set_error_str(buf);
  return MNMT_ERR_CUDA;
}
mnmt_status arg_error(const char* what) {
  mnmt_set_error_str(what);
  return MNMT_ERR_ARG;
}
float sigma_of(float clip) { return 127.0f / clip; }
}  // namespace

extern "C" {

mnmt_status mnmt_op_quantize(const float* x, int64_t n, float clip, int8_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!x || !out)) || !(clip > 0.0f)) return arg_error("mnmt_op_quantize: bad arguments");
  return cuda_status(launch_quantize(x, n, clip, out, (cudaStream_t)stream), "quantize");
}

static mnmt_status gemm_op(const int8_t* A, const int8_t* W, int32_t M, int32_t N, int32_t K,
                           const float* bias, float clip, int32_t epi, void* out, void* out2,
                           int32_t n_tile, int32_t split_k, void* stream);

mnmt_status mnmt_op_gemm_i8(const int8_t* A, const int8_t* W, int32_t M, int32_t N, int32_t K,
                            const float* bias, float clip, int32_t epi, void* out, void* out2,
                            int32_t n_tile, void* stream) {
  return gemm_op(A, W, M, N, K, bias, clip, epi, out, out2, n_tile, 0, stream);
}

mnmt_status mnmt_op_gemm_i8_split(const int8_t* A, const int8_t* W, int32_t M, int32_t N, int32_t K,
                                  const float* bias, float clip, int32_t epi, void* out, void* out2,
                                  int32_t n_tile, int32_t split_k, void* stream) {
  if (split_k != -1 && split_k != 1 && split_k != 2 && split_k != 4 && split_k != 8)
    return arg_error("mnmt_op_gemm_i8_split: split_k must be -1, 1, 2, 4 or 8");
  if (n_tile == -1) return arg_error("mnmt_op_gemm_i8_split: no split-K for the small-M kernel");
  if (n_tile == -2 && split_k < 1) return arg_error("mnmt_op_gemm_i8_split: swap-AB takes split_k 1, 2, 4 or 8");
  return gemm_op(A, W, M, N, K, bias, clip, epi, out, out2, n_tile, split_k, stream);
}

}  // extern "C"

static mnmt_status gemm_op(const int8_t* A, const int8_t* W, int32_t M, int32_t N, int32_t K,
                           const float* bias, float clip, int32_t epi, void* out, void* out2,
                           int32_t n_tile, int32_t split_k, void* stream) {
  if (!A || !W || !out || M < 1 || N < 1 || K < 16 || K % 16 || !(clip > 0.0f))
    return arg_error("mnmt_op_gemm_i8: bad arguments (K must be a positive multiple of 16)");
  if ((epi < MNMT_EPI_F32 || epi > MNMT_EPI_ACC) && epi != MNMT_EPI_TOPK)
    return arg_error("mnmt_op_gemm_i8: bad epilogue");
  if (epi != MNMT_EPI_ARGMAX && epi != MNMT_EPI_TOPK && N % 16) return arg_error("mnmt_op_gemm_i8: N % 16 != 0");
  if ((epi == MNMT_EPI_F32_Q || epi == MNMT_EPI_RELU_F32_Q) && !out2)
    return arg_error("mnmt_op_gemm_i8: epilogue needs out2");
  const bool small = n_tile == -1;   // the small-M CUDA-core kernel (k_gemm_smallm)
  if (small && (M > 32 || epi > MNMT_EPI_SIGMOID || (uintptr_t)A % 16 || (uintptr_t)W % 16))
    return arg_error("mnmt_op_gemm_i8: n_tile -1 needs M <= 32, an fp32 / code epilogue and 16-byte aligned A, W");
  const bool sab = n_tile == -2;     // the swap-AB tcgen05 kernel (k_gemm_sab)
  const bool pair = n_tile == -3;    // the CTA-pair persistent kernel (k_gemm_pers2)
  if (pair && (epi == MNMT_EPI_TOPK || split_k > 1))
    return arg_error("mnmt_op_gemm_i8: n_tile -3 takes no TOPK epilogue and no split-K");
  if (sab && (M > 128 || epi == MNMT_EPI_TOPK || (uintptr_t)A % 16))
    return arg_error("mnmt_op_gemm_i8: n_tile -2 needs M <= 128, a non-TOPK epilogue and 16-byte aligned A");
  if (epi != MNMT_EPI_TOPK && n_tile != 0 && n_tile != 64 && n_tile != 128 && n_tile != 256 && !small && !sab &&
      !pair)
    return arg_error("mnmt_op_gemm_i8: n_tile must be -3, -2, -1, 0, 64, 128 or 256");
  int n_tile_topk = 0;
  if (cudaError_t e = gemm_init(); e != cudaSuccess) return cuda_status(e, "gemm init");
  CUtensorMap ta, tb;
  if (!make_tmap_i8(&ta, A, M, K) || !make_tmap_i8(&tb, W, N, K))
    return cuda_status(cudaErrorInvalidValue, "tensor map encode");
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.scale = (float)(((double)clip * (double)clip) / (127.0 * 127.0));
  a.bias = bias;
  a.clip = clip;
  a.sigma = sigma_of(clip);
  a.ldo = N;
  a.col_block = N;
  a.block_stride = 0;
  a.split_k = split_k;
  // raw operands: the launch may load only the live rows of A (a.M <= 64) and 32-row weight boxes
  a.a_ptr = A;
  a.lda = K;
  a.b_ptr = W;
  if (small) {
    a.a_ptr = A;
    a.lda = K;
    a.b_ptr = W;
    a.smallm_force = 1;
    n_tile = 0;
  }
  if (sab) {
    a.a_ptr = A;
    a.lda = K;
    a.b_ptr = W;
    a.sab_force = 1;
    // split_k > 1: at most ceil(K blocks / split_k) K blocks per CTA (the cluster splits K)
    a.sab_kb = split_k > 1 ? ((K + 127) / 128 + split_k - 1) / split_k : 0;
    a.split_k = 0;
    n_tile = 0;
  }
  switch (epi) {
    case MNMT_EPI_F32:
    case MNMT_EPI_SIGMOID: a.out_f = (float*)out; break;
    case MNMT_EPI_F32_Q:
    case MNMT_EPI_RELU_F32_Q: a.out_f = (float*)out; a.out_q = (int8_t*)out2; break;
    case MNMT_EPI_RELU_Q: a.out_q = (int8_t*)out; break;
    case MNMT_EPI_ARGMAX: a.keys = (unsigned long long*)out; break;
    case MNMT_EPI_ACC: a.out_i = (int32_t*)out; break;
    case MNMT_EPI_TOPK:
      a.part = (TopkPart*)out;
      a.part_ld = 2 * ((N + TOPK_BN - 1) / TOPK_BN);
      n_tile_topk = n_tile;
      n_tile = 0;
      break;
  }
  // MNMT_EPI_TOPK keeps the 8 largest per record; n_tile 2 / 4 selects the top-2 / top-4 variant
  if (epi == MNMT_EPI_TOPK && n_tile_topk == 2) epi = EPI_TOPK2;
  if (epi == MNMT_EPI_TOPK && n_tile_topk == 4) epi = EPI_TOPK4;
  return cuda_status(launch_gemm_i8(ta, tb, a, epi, n_tile, (cudaStream_t)stream), "gemm_i8");
}

extern "C" {

mnmt_status mnmt_op_argmax_ids(const uint64_t* keys, int32_t n, int32_t* ids, void* stream) {
  if (n < 0 || (n > 0 && (!keys || !ids))) return arg_error("mnmt_op_argmax_ids: bad arguments");
  return cuda_status(launch_argmax_ids((const unsigned long long*)keys, n, ids, (cudaStream_t)stream),
                     "argmax_ids");
}

mnmt_status mnmt_op_layernorm(const float* x, const float* delta, const float* gi, const float* gf,
                              const float* gamma, const float* beta, int32_t n, int32_t d,
                              float eps, float clip, float* out, int8_t* out_q, void* stream) {
  if (n < 0 || d < 4 || d % 4 || d > 1024 || !x || !delta || !gamma || !beta || (!out && !out_q) ||
      ((gi == nullptr) != (gf == nullptr)) || !(clip > 0.0f))
    return arg_error("mnmt_op_layernorm: bad arguments");
  LnArgs a{};
  a.n = n;
  a.d = d;
  a.eps = eps;
  a.x = x;
  a.delta = delta;
  a.gi = gi;
  a.gf = gf;
  a.gamma = gamma;
  a.beta = beta;
  a.out = out;
  a.out_q = out_q;
  a.clip = clip;
  a.sigma = sigma_of(clip);
  return cuda_status(launch_ln(a, (cudaStream_t)stream), "layernorm");
}

mnmt_status mnmt_op_aan_step(float* C, const float* y, int32_t n, int32_t d, int32_t t, float clip,
                             float* g, int8_t* g_q, void* stream) {
  if (n < 0 || d < 4 || d % 4 || t < 1 || !C || !y || !(clip > 0.0f))
    return arg_error("mnmt_op_aan_step: bad arguments");
  AanOut o{};
  o.C = C;
  o.g_f = g;
  o.g_q = g_q;
  o.clip = clip;
  o.sigma = sigma_of(clip);
  return cuda_status(launch_aan_step_rows(C, y, n, d, t, o, (cudaStream_t)stream), "aan_step");
}

mnmt_status mnmt_op_embed(const float* E, int32_t d, const int32_t* ids, const int32_t* pos,
                          int32_t n, float clip, float* x, int8_t* x_q, void* stream) {
  if (n < 0 || d < 4 || d % 4 || d > 1024 || !E || !ids || !pos || !x || !x_q || !(clip > 0.0f))
    return arg_error("mnmt_op_embed: bad arguments");
  // positions come from a table of MNMT_MAX_SPAN + 1 rows built on the device
  static thread_local float* pe = nullptr;
  static thread_local int pe_d = 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (pe_d != d) {
    if (pe) cudaFree(pe);
    pe = nullptr;
    if (cudaMalloc(&pe, sizeof(float) * (size_t)(MNMT_MAX_SPAN + 1) * d) != cudaSuccess)
      return cuda_status(cudaGetLastError(), "embed: PE table");
    pe_d = d;
    cudaError_t e = launch_pe_table(pe, MNMT_MAX_SPAN + 1, d, st);
    if (e != cudaSuccess) return cuda_status(e, "embed: PE table");
  }
  return cuda_status(launch_embed_src(ids, nullptr, pos, n, E, pe, d, clip, x, x_q, st), "embed");
}

mnmt_status mnmt_op_attention(const float* q, int64_t ldq, const float* kv, int64_t ldkv,
                              int32_t k_off, int32_t v_off, const int32_t* kv_start,
                              const int32_t* kv_len, int32_t n, int32_t d, int32_t H, float clip,
                              int8_t* out_q, float* out_f, void* stream) {
  if (n < 0 || H < 1 || d % H || (d / H) % 4 || d / H > 64 || !q || !kv || !kv_start || !kv_len ||
      !out_q || ldq % 4 || ldkv % 4 || k_off % 4 || v_off % 4 || !(clip > 0.0f))
    return arg_error("mnmt_op_attention: bad arguments");
  if (cudaError_t e = attn_init(); e != cudaSuccess) return cuda_status(e, "attention init");
  AttnArgs a{};
  a.mode = ATTN_ENC;
  a.n = n;
  a.H = H;
  a.dh = d / H;
  a.d = d;
  a.q = q;
  a.ldq = ldq;
  a.kv = kv;
  a.ldkv = ldkv;
  a.k_off = k_off;
  a.v_off = v_off;
  a.kv_start = kv_start;
  a.kv_len = kv_len;
  a.clip = clip;
  a.sigma = sigma_of(clip);
  a.out_q = out_q;
  a.out_f = out_f;
  return cuda_status(launch_attn(a, (cudaStream_t)stream), "attention");
}

mnmt_status mnmt_op_attention_enc(const float* qkv, const int32_t* sent_start, const int32_t* sent_len,
                                  int32_t n_sent, int32_t d, int32_t H, int32_t s_max, float clip,
                                  int8_t* out_q, int32_t variant, void* stream) {
  if (n_sent < 0 || H < 1 || d % H || (d / H) % 4 || d / H > 64 || !qkv || !sent_start || !sent_len ||
      !out_q || s_max < 1 || s_max > MNMT_MAX_KV || variant < 0 || variant > 3 || !(clip > 0.0f))
    return arg_error("mnmt_op_attention_enc: bad arguments");
  if (cudaError_t e = attn_init(); e != cudaSuccess) return cuda_status(e, "attention init");
  EncAttnArgs a{};
  a.qkv = qkv;
  a.sent_start = sent_start;
  a.sent_len = sent_len;
  a.n_sent = n_sent;
  a.H = H;
  a.dh = d / H;
  a.d = d;
  a.s_max = s_max;
  a.clip = clip;
  a.sigma = sigma_of(clip);
  a.out_q = out_q;
  const cudaError_t e = launch_attn_enc_v(a, variant, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) return arg_error("mnmt_op_attention_enc: variant needs d / H = 64, s_max <= 100");
  return cuda_status(e, "encoder attention");
}

static mnmt_status src_attention_op(const float* q, int64_t ldq, const float* kv, int64_t kv_rows,
                                    int64_t ldkv, int32_t k_off, int32_t v_off,
                                    const int32_t* kv_start, const int32_t* kv_len, int32_t max_span,
                                    int32_t n, int32_t d, int32_t H, float clip, int8_t* out_q,
                                    float* out_f, int f32, void* stream);

mnmt_status mnmt_op_src_attention(const float* q, int64_t ldq, const float* kv, int64_t kv_rows,
                                  int64_t ldkv, int32_t k_off, int32_t v_off,
                                  const int32_t* kv_start, const int32_t* kv_len, int32_t max_span,
                                  int32_t n, int32_t d, int32_t H, float clip, int8_t* out_q,
                                  float* out_f, void* stream) {
  return src_attention_op(q, ldq, kv, kv_rows, ldkv, k_off, v_off, kv_start, kv_len, max_span, n, d,
                          H, clip, out_q, out_f, 0, stream);
}

mnmt_status mnmt_op_src_attention_f32(const float* q, int64_t ldq, const float* kv, int64_t kv_rows,
                                      int64_t ldkv, int32_t k_off, int32_t v_off,
                                      const int32_t* kv_start, const int32_t* kv_len, int32_t max_span,
                                      int32_t n, int32_t d, int32_t H, float clip, int8_t* out_q,
                                      float* out_f, void* stream) {
  if (d % H || (d / H != 32 && d / H != 64))
    return arg_error("mnmt_op_src_attention_f32: d / H must be 32 or 64 (the TMA kernel)");
  return src_attention_op(q, ldq, kv, kv_rows, ldkv, k_off, v_off, kv_start, kv_len, max_span, n, d,
                          H, clip, out_q, out_f, 1, stream);
}

static mnmt_status src_attention_op(const float* q, int64_t ldq, const float* kv, int64_t kv_rows,
                                    int64_t ldkv, int32_t k_off, int32_t v_off,
                                    const int32_t* kv_start, const int32_t* kv_len, int32_t max_span,
                                    int32_t n, int32_t d, int32_t H, float clip, int8_t* out_q,
                                    float* out_f, int f32, void* stream) {
  if (n < 0 || H < 1 || d % H || (d / H) % 4 || d / H > 64 || !q || !kv || kv_rows < 1 ||
      max_span < 0 || max_span > MNMT_MAX_KV ||
      !kv_start || !kv_len || !out_q || ldq % 4 || ldkv % 4 || k_off % 4 || v_off % 4 ||
      !(clip > 0.0f))
    return arg_error("mnmt_op_src_attention: bad arguments");
  if (cudaError_t e = attn_init(); e != cudaSuccess) return cuda_status(e, "attention init");
  CUtensorMap tm;
  if (!make_tmap_kv(&tm, kv, kv_rows, ldkv)) return cuda_status(cudaErrorInvalidValue, "tensor map encode");
  AttnArgs a{};
  a.mode = ATTN_ENC;   // row r attends kv rows [kv_start[r], + kv_len[r])
  a.span = (max_span + 31) / 32 * 32;
  a.n = n;
  a.H = H;
  a.dh = d / H;
  a.d = d;
  a.q = q;
  a.ldq = ldq;
  a.kv = kv;
  a.ldkv = ldkv;
  a.k_off = k_off;
  a.v_off = v_off;
  a.kv_start = kv_start;
  a.kv_len = kv_len;
  a.clip = clip;
  a.sigma = sigma_of(clip);
  a.out_q = out_q;
  a.out_f = out_f;
  a.tmap = &tm;
  a.kv_row0 = 0;
  a.f32 = f32;
  return cuda_status(launch_attn(a, (cudaStream_t)stream), "source attention");
}

mnmt_status mnmt_op_attention_bf16(const float* q, int64_t ldq, const uint16_t* kv16, int64_t ldkv,
                                   int32_t k_off, int32_t v_off, const int32_t* kv_start,
                                   const int32_t* kv_len, int32_t n, int32_t d, int32_t H,
                                   float clip, int8_t* out_q, float* out_f, void* stream) {
  if (n < 0 || H < 1 || d % H || (d / H) % 4 || d / H > 64 || !q || !kv16 || !kv_start ||
      !kv_len || !out_q || ldq % 4 || ldkv % 4 || k_off % 4 || v_off % 4 || !(clip > 0.0f))
    return arg_error("mnmt_op_attention_bf16: bad arguments");
  if (cudaError_t e = attn_init(); e != cudaSuccess) return cuda_status(e, "attention init");
  AttnArgs a{};
  a.mode = ATTN_ENC;
  a.n = n;
  a.H = H;
  a.dh = d / H;
  a.d = d;
  a.q = q;
  a.ldq = ldq;
  a.kv16 = reinterpret_cast<const bf16s*>(kv16);
  a.ldkv = ldkv;
  a.k_off = k_off;
  a.v_off = v_off;
  a.kv_start = kv_start;
  a.kv_len = kv_len;
  a.clip = clip;
  a.sigma = sigma_of(clip);
  a.out_q = out_q;
  a.out_f = out_f;
  return cuda_status(launch_attn(a, (cudaStream_t)stream), "attention (bf16 K/V)");
}

}  // extern "C"

// Debug: a chain of `n` identical int8 GEMMs (M x N x K, EPI_F32, A -> out, PDL, captured in a CUDA
// graph) replayed once; res[0] = mean per-launch time (us); res[1..5] = CTA (0,0)'s stamps relative
// to its entry: after the PDL wait, operands landed, accumulator complete, warp 2's stores issued,
// after the final barrier + TMEM dealloc; res[6] = entry-to-entry; res[7] = next kernel's wait
// release minus our end.  Not part of the documented ABI.
extern "C" mnmt_status mnmt_debug_gemm_chain(const int8_t* A, const int8_t* W, int32_t M, int32_t N,
                                            int32_t K, float* out, int32_t n, double* res6) {
  if (!A || !W || !out || n < 2 || !res6) return arg_error("mnmt_debug_gemm_chain: bad arguments");
  cudaError_t e = gemm_init();
  if (e != cudaSuccess) return cuda_status(e, "gemm_init");
  CUtensorMap ta, tb;
  if (!make_tmap_i8(&ta, A, M, K) || !make_tmap_i8(&tb, W, N, K)) return arg_error("tensor map");
  unsigned long long* tr = nullptr;
  if ((e = cudaMalloc(&tr, (size_t)n * 9 * 8)) != cudaSuccess) return cuda_status(e, "malloc");
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const char* ebn = getenv("MNMT_CHAIN_BN");   // N tile override (64 / 128 / 256), A/B only
  const int bn = ebn ? atoi(ebn) : 0;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n; ++i) {
    GemmArgs a{};
    a.M = M; a.N = N; a.K = K; a.scale = 1.0f / 4032.25f; a.clip = 2.0f; a.sigma = 63.5f;
    a.out_f = out; a.ldo = N; a.col_block = N; a.trace = tr + (size_t)i * 9;
    launch_gemm_i8(ta, tb, a, EPI_F32, bn, st);
  }
  e = cudaStreamEndCapture(st, &g);
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
  if (e == cudaSuccess) e = cudaGraphLaunch(ge, st);   // warm
  cudaEvent_t a0, a1;
  cudaEventCreate(&a0);
  cudaEventCreate(&a1);
  if (e == cudaSuccess) e = cudaEventRecord(a0, st);
  if (e == cudaSuccess) e = cudaGraphLaunch(ge, st);
  if (e == cudaSuccess) e = cudaEventRecord(a1, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  std::vector<unsigned long long> h((size_t)n * 9);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
  float ms = 0;
  cudaEventElapsedTime(&ms, a0, a1);
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 1; i + 1 < n; ++i) {
    const unsigned long long* t = h.data() + (size_t)i * 9;
    for (int k = 0; k < 5; ++k) acc[k] += (double)(t[k + 1] - t[0]);
    acc[5] += (double)(t[0] - h[(size_t)(i - 1) * 9]);
    acc[6] += (double)(h[(size_t)(i + 1) * 9 + 1]) - (double)t[5];   // next kernel's wait release - our end
    for (int k = 0; k < 3; ++k) acc[7 + k] += (double)(t[6 + k] - t[0]);
  }
  res6[0] = 1000.0 * ms / n;
  for (int k = 0; k < 10; ++k) res6[k + 1] = acc[k] / (n - 2) / 1000.0;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaEventDestroy(a0);
  cudaEventDestroy(a1);
  cudaStreamDestroy(st);
  cudaFree(tr);
  return cuda_status(e, "gemm chain");
}


// ------------------------------------------------------------------ A11: multi-GPU id unshard
namespace {
__global__ void k_gather_rows(const int32_t* __restrict__ src, const int64_t* __restrict__ src_off,
                              const int32_t* __restrict__ src_len, const int32_t* __restrict__ dst_row,
                              const int64_t* __restrict__ dst_off, int n, int32_t* __restrict__ dst,
                              int32_t* __restrict__ dst_len) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  const int len = src_len[i], r = dst_row[i];
  const int32_t* s = src + src_off[i];
  int32_t* o = dst + dst_off[r];
  for (int j = lane; j < len; j += 32) o[j] = s[j];
  if (lane == 0) dst_len[r] = len;
}
}  // namespace

extern "C" mnmt_status mnmt_op_gather_rows(const int32_t* src, const int64_t* src_off,
                                           const int32_t* src_len, const int32_t* dst_row,
                                           const int64_t* dst_off, int32_t n, int32_t* dst,
                                           int32_t* dst_len, void* stream) {
  if (n < 0 || (n > 0 && (!src || !src_off || !src_len || !dst_row || !dst_off || !dst || !dst_len)))
    return arg_error("mnmt_op_gather_rows: bad arguments");
  if (n == 0) return MNMT_OK;
  k_gather_rows<<<(n + 7) / 8, 256, 0, (cudaStream_t)stream>>>(src, src_off, src_len, dst_row, dst_off,
                                                                n, dst, dst_len);
  return cuda_status(cudaGetLastError(), "gather_rows");
}
