// mnmt.cu — libmnmt runtime: the C ABI of include/mnmt.h on top of the sm_100a kernels.
//
// Host side only schedules; every step of the decode path runs in kernels
// (gemm_i8.cu, rowops.cu).  Per batch (PAPER.md:L42 length-sorted word batches):
//   encoder: embed -> L x [QKV GEMM -> attn -> O GEMM -> LN -> FFN1(ReLU->codes) -> FFN2 -> LN]
//            -> one GEMM for every decoder layer's source K|V (N = 2 d L), scattered per layer;
//   decoder step (one CUDA graph, replayed max_len times; live-row count and t live on device):
//            embed(+AAN step of layer 0) -> L x [AAN FFN / gates | self-attn] -> LN1
//            -> src-q GEMM -> src attention -> src-o GEMM -> LN2 -> FFN1 -> FFN2
//            -> LN3 (+AAN step of the next layer) -> output GEMM fused with argmax -> finish.
#include <algorithm>
#include <cuda.h>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/mnmt.h"
#include "../../include/mnmt_ops.h"
#include "beam.h"
#include "kernels.h"
#include "rowops.h"
#include "shortlist.h"

using namespace mnmt;

static thread_local std::string g_err;

static void set_err(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

extern "C" const char* mnmt_last_error(void) { return g_err.c_str(); }
void mnmt_set_error_str(const char* s) { g_err = s; }

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct Lin {
  int8_t* q = nullptr;
  float* b = nullptr;
  int out = 0, in = 0;
  CUtensorMap tm;
};

struct EncLayer {
  Lin qkv, o, f1, f2;
  float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
};
struct DecLayer {
  Lin a1, a2, gi, gf, qkv, o, sq, so, f1, f2;
  float* ln[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
};

struct Workspace {
  int64_t M_cap = 0, B_cap = 0, T_cap = 0, O_cap = 0;
  std::vector<void*> allocs;
  // encoder (token rows)
  float *x = nullptr, *qkv = nullptr, *o = nullptr, *kv = nullptr;
  bf16s* kv16 = nullptr;   // src_kv_bf16 (F3): bf16 copy of kv read by source attention
  int8_t *cx = nullptr, *cctx = nullptr, *ch = nullptr;
  CUtensorMap tm_cx, tm_cctx, tm_ch;
  // decoder (compact live rows)
  int32_t *ctrl = nullptr, *live = nullptr, *prev_id = nullptr;
  int32_t *prev_live = nullptr, *live_start = nullptr, *live_len = nullptr;   // compact order
  int32_t *row_start = nullptr, *row_len = nullptr, *max_len = nullptr, *len_idx = nullptr;
  int64_t *out_off = nullptr, *forced_off = nullptr;
  unsigned long long* keys = nullptr;
  float *C = nullptr, *y = nullptr, *g = nullptr, *a = nullptr, *gi = nullptr, *gf = nullptr;
  float *x1 = nullptr, *qs = nullptr, *od = nullptr, *x2 = nullptr, *f = nullptr, *qkvd = nullptr;
  float* selfkv = nullptr;
  int8_t *cy = nullptr, *cg = nullptr, *ch1 = nullptr, *ca = nullptr, *cx1 = nullptr;
  int8_t *cctxd = nullptr, *cx2 = nullptr, *chd = nullptr;
  CUtensorMap tm_cy, tm_cg, tm_ch1, tm_ca, tm_cx1, tm_cctxd, tm_cx2, tm_chd;
  CUtensorMap tm_kv;   // fp32 source K|V rows of every layer [L * M_cap][2d] (TMA attention)
  CUtensorMap tm_self; // self-attention cache rows [L * B_cap * T_cap][2d] (decoder 0)
  // beam search (F1; allocated on first use by beam_ensure, sized B_cap x T_cap)
  std::vector<void*> beam_allocs;
  int64_t beam_rows = 0, beam_T = 0;
  TopkPart* part = nullptr;
  int part_ld = 0;
  float *row_lse = nullptr, *row_v = nullptr, *hscore = nullptr, *child_score = nullptr;
  int32_t *row_j = nullptr, *sent_row0 = nullptr, *sent_nlive = nullptr, *sent_nfin = nullptr;
  int32_t *sent_list = nullptr, *child_par = nullptr, *child_tok = nullptr, *hist = nullptr;
  int32_t* anc = nullptr;
  float* logits = nullptr;   // [B_cap][V] (beam_fused = 0)
  // vocabulary shortlist (F2; allocated on first use by sl_lane_ensure): the decode unit's
  // shortlist rows of the int8 E and of the output bias, and column -> id
  std::vector<void*> sl_allocs;
  int8_t* sl_q = nullptr;
  float* sl_b = nullptr;
  int32_t* sl_map = nullptr;
  uint32_t* sl_bits = nullptr;             // [SL_MAX_GROUPS][ceil(V/32)] per-group column bitmaps
  int32_t* sl_rgrp = nullptr;              // [B_cap] batch row -> group in the wave
  CUtensorMap tm_sl;
};

// Job-level device buffers shared by all lanes.
struct JobBuf {
  int64_t O_cap = 0, N_cap = 0, tok_cap = 0, meta_cap = 0, rows_cap = 0;
  std::vector<void*> allocs;
  int32_t* out_ids = nullptr;   // [sum max_len] output ids, input-order layout
  int32_t* out_len = nullptr;   // [n]
  int32_t* src_ids = nullptr;   // [sum S_i]
  int32_t* meta = nullptr;      // token metadata of all batches: idx|pos|start|len per batch
  int32_t* rmeta32 = nullptr;   // row metadata of all batches: [start|len|max_len|len_idx|order] x B_b
  int64_t* rmeta64 = nullptr;   // [out_off|forced_off] x B_b
  int32_t* forced = nullptr;    // teacher forcing: [sum T_i] input ids (forced_off layout)
  float* out_score = nullptr;   // beam search: [n x beam] hypothesis scores
  int32_t* n_hyp = nullptr;     // beam search: [n] hypotheses per sentence
  // vocabulary shortlist (F2): per word-budget batch bitmap, ascending ids and count, and the
  // batch-major sentence spans the bitmap kernel walks
  std::vector<void*> sl_allocs;
  int64_t sl_bb_cap = 0, sl_sent_cap = 0, sl_wave_cap = 0, sl_rows_cap = 0;
  uint32_t* sl_bits = nullptr;  // [bb][ceil(V/32)]
  int32_t* sl_ids = nullptr;    // [wave][V] union of the wave's shortlists, ascending
  unsigned long long* sl_mask = nullptr;   // [wave][V] per column: bit g = in group g's list
  int32_t* sl_n = nullptr;      // [wave]
  int32_t* sl_span = nullptr;   // [start | len] x sentences (batch-major), bb_off, wave_off
  int32_t* sl_rgrp = nullptr;   // [job rows] group (batch within its wave) of every row
};

// A lane = one independent decoder (workspace + stream + step graphs).  Rows are
// independent, so lanes run concurrently and their kernel chains overlap on the GPU.
struct Lane {
  Workspace ws;
  cudaStream_t st = nullptr;
  cudaEvent_t ev = nullptr;
  cudaStream_t side = nullptr;                 // fork stream for independent GEMMs (graph branch)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::map<int64_t, cudaGraphExec_t> graphs;   // key: padded live-row bound
  std::map<int64_t, int64_t> graph_launches;   // kernels per launch of graphs[key]
  int span_cap = 0;                            // attention span the step kernels are sized for
  int kind = -1;                               // streams from: 0 runtime, 1 critical / 2 bulk green context
  int sl_n = 0;                             // columns of the shortlisted output GEMM (0 = full V)
};

// Device-side dumps of a teacher-forced run (call state, MNMT_DUMP_*): k_dump_rows copies the
// live rows of a step's activations to row foff[orig] + t - 1 of these buffers.  Launched
// inside the step graphs, so dumps cover the same scheduling (lanes, tiers, SM partitions,
// small-M GEMMs) as an untouched run.
struct DevDump {
  float* layers = nullptr;      // [O][L][3][d]: x1, x2, x3 of every decoder layer
  float* dec_out = nullptr;     // [O][d]
  int8_t* out_codes = nullptr;  // [O][d]
  float* margin = nullptr;      // [O]: top-1 minus top-2 logit of each step
  bool any() const { return layers || dec_out || out_codes || margin; }
};

}  // namespace

struct mnmt_model {
  mnmt_config c;
  int dev = 0;
  bool quantized = false, failed = false;
  std::map<std::string, int64_t> manifest;               // name -> numel
  std::map<std::string, std::vector<float>> host;        // set parameters (until quantize)
  std::vector<void*> allocs;
  float *E = nullptr, *out_b = nullptr, *PE = nullptr;
  int8_t* qE = nullptr;
  CUtensorMap tmE;
  std::vector<EncLayer> enc;
  std::vector<DecLayer> dec;
  Lin kv_all;
  std::vector<Lane> lanes;      // lanes[0] always exists after create
  int n_lanes = 1;               // option "lanes"
  JobBuf jb;
  cudaStream_t st = nullptr;     // main stream: uploads, joins, output copies
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_job = nullptr;
  mnmt_stats stats{};
  int max_pos = MNMT_MAX_SPAN + 1;
  int64_t max_concurrent_rows = 0;   // option: co-schedule batches in waves of <= this many rows
  int steps_per_graph = 1;             // option: decoder steps captured per CUDA graph
  int smallm = 32;                     // option: row bound of the small-M GEMM path (0 = off)
  int sab_kmin = 0;                    // option: shallowest K of the swap-AB path
  int sab_out = 0;                     // option: row bound of the swap-AB output GEMM + argmax (A9)
  int sab_kb = 0;                      // option: K blocks per swap-AB CTA before K is split (0 = 8)
  int sab = 0;                         // option: row bound of the swap-AB tcgen05 GEMM path (0 = off,
                                       // <= 128); steps at <= sab rows run in 16 / 32 / 64 / 128-row graphs
  int smallm_kmax = 512;               // option: deepest K the small-M path takes
  int64_t smallm_wmax = 1 << 20;       // option: largest weight matrix (N x K bytes) of the small-M path
  int attn_tma_self = 2;               // option: self-attention through TMA tiles (0 / 1 / 2)
  int attn_f32 = 0;                    // option: decoder attention in fp32 (departs from R20; off)
  int split_k = 0;                     // option: 1 = split-K clusters by the measured rule (off: slower in the job)
  DevDump dump;                        // (call state) device dumps of a teacher-forced run
  int green_sms = 0;                   // option: SMs of the critical lane's green context (0 = off)
  CUgreenCtx green[2] = {nullptr, nullptr};   // [0] critical lane, [1] the other lanes
  int green_count[2] = {0, 0};                // SMs of each partition
  int pers_reserve = 0;                // option: SMs the persistent GEMMs of non-critical lanes leave free
  int cur_pers_grid = 0;               // (launch state) persistent-GEMM CTA cap of the lane being issued
  int lane_tiers = 0;                  // option: 0 = deal sentences round-robin to lanes;
                                       // p*10 = contiguous length tiers of equal sum S^p
  int beam = 0;                        // (call state) beam size of the running call; 0 = greedy
  int beam_fused = 0;                  // option: 1 = log-sum-exp / top-k in the output GEMM epilogue
                                       // (EPI_TOPK*), 0 = fp32 logits + k_beam_logits (faster)
  // vocabulary shortlist tables (F2, mnmt_model_set_shortlist)
  int32_t *sl_freq = nullptr, *sl_lex = nullptr;
  int sl_nfreq = 0, sl_k = 0;
  bool sl_tables = false;
  bool sl_active = false;              // (call state) MNMT_SHORTLIST
  std::vector<int32_t> sl_count;       // (call state) union size of each decode wave
  std::vector<int32_t> sl_groups;      // (call state) word-budget batches of each decode wave
};

namespace {

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_err("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, __LINE__, \
              cudaGetErrorString(e_));                                              \
      return MNMT_ERR_CUDA;                                                         \
    }                                                                               \
  } while (0)

#define CKS(call)                    \
  do {                               \
    mnmt_status s_ = (call);         \
    if (s_ != MNMT_OK) return s_;    \
  } while (0)

// CUDA failure -> fail-stop handle.
static mnmt_status fail(mnmt_model* m, mnmt_status s) {
  if (s == MNMT_ERR_CUDA) m->failed = true;
  return s;
}

static float sigma_of(const mnmt_model* m) { return 127.0f / m->c.clip; }
static float scale_of(const mnmt_model* m) {
  return (float)(((double)m->c.clip * (double)m->c.clip) / (127.0 * 127.0));
}

static mnmt_status dmalloc(std::vector<void*>& list, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_err("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    return MNMT_ERR_OOM;
  }
  list.push_back(*p);
  return MNMT_OK;
}
template <typename T>
static mnmt_status dalloc(std::vector<void*>& list, T** p, int64_t n) {
  return dmalloc(list, reinterpret_cast<void**>(p), (size_t)std::max<int64_t>(n, 1) * sizeof(T));
}

static void build_manifest(mnmt_model* m) {
  const auto& c = m->c;
  const int64_t d = c.d_model, F = c.d_ffn, V = c.vocab;
  auto& mf = m->manifest;
  mf["emb.E"] = V * d;
  if (c.out_bias) mf["out.b"] = V;
  auto lin = [&](const std::string& p, int64_t out, int64_t in) {
    mf[p + ".W"] = out * in;
    mf[p + ".b"] = out;
  };
  auto ln = [&](const std::string& p) {
    mf[p + ".g"] = d;
    mf[p + ".b"] = d;
  };
  for (int l = 0; l < c.enc_layers; ++l) {
    const std::string p = "enc." + std::to_string(l) + ".";
    for (const char* s : {"q", "k", "v", "o"}) lin(p + "self." + s, d, d);
    lin(p + "ffn.1", F, d);
    lin(p + "ffn.2", d, F);
    ln(p + "ln1");
    ln(p + "ln2");
  }
  for (int l = 0; l < c.dec_layers; ++l) {
    const std::string p = "dec." + std::to_string(l) + ".";
    if (c.decoder == 1) {
      if (c.aan_ffn_depth >= 1) lin(p + "aan.ffn.1", d, d);
      if (c.aan_ffn_depth >= 2) lin(p + "aan.ffn.2", d, d);
      if (c.aan_gate) {
        lin(p + "aan.gate.i", d, d);
        lin(p + "aan.gate.f", d, d);
      }
    } else {
      for (const char* s : {"q", "k", "v", "o"}) lin(p + "self." + s, d, d);
    }
    for (const char* s : {"q", "k", "v", "o"}) lin(p + "src." + s, d, d);
    lin(p + "ffn.1", F, d);
    lin(p + "ffn.2", d, F);
    ln(p + "ln1");
    ln(p + "ln2");
    ln(p + "ln3");
  }
}

static const char* cfg_problem(const mnmt_config* c) {
  if (!c) return "config is NULL";
  if (c->abi_version != MNMT_ABI_VERSION) return "abi_version mismatch";
  if (c->d_model < 16 || c->d_model > 1024 || c->d_model % 16) return "d_model must be 16..1024, multiple of 16";
  if (c->d_ffn < 16 || c->d_ffn % 16) return "d_ffn must be a positive multiple of 16";
  if (c->n_heads < 1 || c->d_model % c->n_heads) return "d_model must be divisible by n_heads";
  const int dh = c->d_model / c->n_heads;
  if (dh % 4 || dh > 64) return "head width d/H must be a multiple of 4 and <= 64";
  if (c->enc_layers < 0 || c->enc_layers > 64 || c->dec_layers < 1 || c->dec_layers > 64) return "layer count out of range";
  if (c->vocab < 1) return "vocab must be >= 1";
  if (c->decoder != 0 && c->decoder != 1) return "decoder must be 0 or 1";
  if (c->aan_ffn_depth < 0 || c->aan_ffn_depth > 2) return "aan_ffn_depth must be 0, 1 or 2";
  if (c->aan_gate != 0 && c->aan_gate != 1) return "aan_gate must be 0 or 1";
  if (c->out_bias != 0 && c->out_bias != 1) return "out_bias must be 0 or 1";
  if (c->eos_id < 0 || c->eos_id >= c->vocab) return "eos_id out of range";
  if (!(c->clip > 0.0f) || !std::isfinite(c->clip)) return "clip must be > 0";
  if (!(c->ln_eps >= 0.0f)) return "ln_eps must be >= 0";
  if (c->src_kv_bf16 != 0 && c->src_kv_bf16 != 1) return "src_kv_bf16 must be 0 or 1";
  return nullptr;
}

// Upload and quantize a (possibly concatenated) weight: rows from `names` stacked in order.
static mnmt_status prep_lin(mnmt_model* m, Lin& L, const std::vector<std::string>& names,
                            int rows_each, int in, float* tmp) {
  const int out = rows_each * (int)names.size();
  L.out = out;
  L.in = in;
  CKS(dalloc(m->allocs, &L.q, (int64_t)out * in));
  CKS(dalloc(m->allocs, &L.b, out));
  for (size_t i = 0; i < names.size(); ++i) {
    const auto& W = m->host[names[i] + ".W"];
    const auto& b = m->host[names[i] + ".b"];
    CK(cudaMemcpyAsync(tmp, W.data(), W.size() * sizeof(float), cudaMemcpyHostToDevice, m->st));
    CK(launch_quantize(tmp, (int64_t)W.size(), m->c.clip, L.q + (int64_t)i * rows_each * in, m->st));
    CK(cudaMemcpyAsync(L.b + (int64_t)i * rows_each, b.data(), b.size() * sizeof(float),
                       cudaMemcpyHostToDevice, m->st));
    CK(cudaStreamSynchronize(m->st));  // tmp is reused
  }
  if (!make_tmap_i8(&L.tm, L.q, out, in)) {
    set_err("cuTensorMapEncodeTiled failed for %s", names[0].c_str());
    return MNMT_ERR_CUDA;
  }
  return MNMT_OK;
}

static mnmt_status upload_vec(mnmt_model* m, float** dst, const std::string& name) {
  const auto& v = m->host[name];
  CKS(dalloc(m->allocs, dst, (int64_t)v.size()));
  CK(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice, m->st));
  return MNMT_OK;
}

// ------------------------------------------------------------------ workspace
static void lane_free(Lane& L) {
  for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
  L.graphs.clear();
  for (void* p : L.ws.allocs) cudaFree(p);
  for (void* p : L.ws.beam_allocs) cudaFree(p);
  for (void* p : L.ws.sl_allocs) cudaFree(p);
  L.sl_n = 0;
  L.ws = Workspace();
}

static void jb_free(mnmt_model* m) {
  for (void* p : m->jb.allocs) cudaFree(p);
  for (void* p : m->jb.sl_allocs) cudaFree(p);
  m->jb = JobBuf();
}

// ------------------------------------------------------------------ green contexts
// SM partitions (driver API, resolved through cudaGetDriverEntryPoint like the tensor-map
// encoder, so the library needs no -lcuda): with tiered lanes and option green_sms = N, the
// critical lane's streams live in a green context of N SMs and the other lanes' in one holding
// the rest, so the bulk can never occupy the SMs the critical path waits for.
struct GreenApi {
  CUresult (*dev_get)(CUdevice*, int) = nullptr;
  CUresult (*get_res)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                    unsigned) = nullptr;
  CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*destroy)(CUgreenCtx) = nullptr;
  CUresult (*stream_create)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  bool ok = false;
};
static const GreenApi& green_api() {
  static GreenApi g;
  static bool tried = false;
  if (tried) return g;
  tried = true;
  auto get = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess;
  };
  g.ok = get("cuDeviceGet", (void**)&g.dev_get) && get("cuDeviceGetDevResource", (void**)&g.get_res) &&
         get("cuDevSmResourceSplitByCount", (void**)&g.split) &&
         get("cuDevResourceGenerateDesc", (void**)&g.gen_desc) &&
         get("cuGreenCtxCreate", (void**)&g.create) && get("cuGreenCtxDestroy", (void**)&g.destroy) &&
         get("cuGreenCtxStreamCreate", (void**)&g.stream_create);
  return g;
}

static mnmt_status green_ensure(mnmt_model* m) {
  if (m->green[0] || m->green_sms <= 0) return MNMT_OK;
  const GreenApi& g = green_api();
  if (!g.ok) { set_err("green contexts unavailable in this driver"); return MNMT_ERR_CUDA; }
  CUdevice dev;
  CUdevResource all, part[1], rest;
  CUdevResourceDesc d0, d1;
  unsigned n = 1;
  if (g.dev_get(&dev, m->dev) != CUDA_SUCCESS || g.get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      g.split(part, &n, &all, &rest, 0, (unsigned)m->green_sms) != CUDA_SUCCESS || n != 1 ||
      g.gen_desc(&d0, part, 1) != CUDA_SUCCESS || g.gen_desc(&d1, &rest, 1) != CUDA_SUCCESS ||
      g.create(&m->green[0], d0, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      g.create(&m->green[1], d1, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    set_err("green context creation failed (green_sms %d)", m->green_sms);
    return MNMT_ERR_CUDA;
  }
  m->green_count[0] = (int)part[0].sm.smCount;
  m->green_count[1] = (int)rest.sm.smCount;
  return MNMT_OK;
}

static void lane_streams_free(Lane& L) {
  for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
  L.graphs.clear();
  if (L.st) cudaStreamDestroy(L.st);
  if (L.side) cudaStreamDestroy(L.side);
  if (L.ev) cudaEventDestroy(L.ev);
  if (L.ev_fork) cudaEventDestroy(L.ev_fork);
  if (L.ev_join) cudaEventDestroy(L.ev_join);
  L.st = L.side = nullptr;
  L.ev = L.ev_fork = L.ev_join = nullptr;
  L.kind = -1;
}

// Lane li's streams get priority li steps above the lowest (clamped): with length tiers the
// last lane holds the longest sentences, i.e. the job's critical path.  With green_sms the
// streams come from the lane's SM partition.
static mnmt_status lane_init(mnmt_model* m, Lane& L, int li) {
  const bool tiered = m->n_lanes > 1 && m->lane_tiers > 0;
  const int kind = (m->green_sms > 0 && tiered) ? (li == m->n_lanes - 1 ? 1 : 2) : 0;
  if (L.st && L.kind == kind) return MNMT_OK;
  if (L.st) {
    cudaDeviceSynchronize();
    lane_streams_free(L);
  }
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  const int prio = std::max(greatest, least - li);
  bool ok;
  if (kind) {
    mnmt_status gs = green_ensure(m);
    if (gs != MNMT_OK) return gs;
    const GreenApi& g = green_api();
    CUstream a = nullptr, b = nullptr;
    ok = g.stream_create(&a, m->green[kind - 1], CU_STREAM_NON_BLOCKING, prio) == CUDA_SUCCESS &&
         g.stream_create(&b, m->green[kind - 1], CU_STREAM_NON_BLOCKING, prio) == CUDA_SUCCESS;
    L.st = (cudaStream_t)a;
    L.side = (cudaStream_t)b;
  } else {
    ok = cudaStreamCreateWithPriority(&L.st, cudaStreamNonBlocking, prio) == cudaSuccess &&
         cudaStreamCreateWithPriority(&L.side, cudaStreamNonBlocking, prio) == cudaSuccess;
  }
  if (!ok || cudaEventCreateWithFlags(&L.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L.ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L.ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    set_err("lane stream/event creation failed");
    return MNMT_ERR_CUDA;
  }
  L.kind = kind;
  return MNMT_OK;
}

static mnmt_status ws_tmap(CUtensorMap* tm, const void* p, int64_t rows, int64_t K) {
  if (!make_tmap_i8(tm, p, rows, K)) {
    set_err("cuTensorMapEncodeTiled failed (workspace)");
    return MNMT_ERR_CUDA;
  }
  return MNMT_OK;
}

// Job buffers for O output ids, N sentences, tok source tokens, token/row metadata.
static mnmt_status jb_ensure(mnmt_model* m, int64_t O, int64_t N, int64_t tok, int64_t meta,
                             int64_t rows) {
  JobBuf& j = m->jb;
  if (O <= j.O_cap && N <= j.N_cap && tok <= j.tok_cap && meta <= j.meta_cap && rows <= j.rows_cap)
    return MNMT_OK;
  CK(cudaDeviceSynchronize());
  const int64_t Oc = std::max(O, j.O_cap), Nc = std::max(N, j.N_cap), tc = std::max(tok, j.tok_cap);
  const int64_t mc = std::max(meta, j.meta_cap), rc = std::max(rows, j.rows_cap);
  jb_free(m);
  for (Lane& L : m->lanes) {   // captured graphs / step programs point at the job buffers
    for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
    L.graphs.clear();
  }
  JobBuf& z = m->jb;
  z.O_cap = Oc; z.N_cap = Nc; z.tok_cap = tc; z.meta_cap = mc; z.rows_cap = rc;
  CKS(dalloc(z.allocs, &z.out_ids, Oc));
  CKS(dalloc(z.allocs, &z.forced, Oc));
  CKS(dalloc(z.allocs, &z.out_len, Nc));
  CKS(dalloc(z.allocs, &z.src_ids, tc));
  CKS(dalloc(z.allocs, &z.meta, mc));
  CKS(dalloc(z.allocs, &z.rmeta32, 5 * rc));
  CKS(dalloc(z.allocs, &z.rmeta64, 2 * rc));
  CKS(dalloc(z.allocs, &z.out_score, Nc));
  CKS(dalloc(z.allocs, &z.n_hyp, Nc));
  return MNMT_OK;
}

// Beam-search buffers of a lane (F1): TOPK partials and per-row / per-slot / per-sentence
// state for the lane's B_cap rows and T_cap steps.
static mnmt_status beam_ensure(mnmt_model* m, Lane& Ln) {
  Workspace& w = Ln.ws;
  if (w.beam_rows >= w.B_cap && w.beam_T >= w.T_cap) return MNMT_OK;
  CK(cudaDeviceSynchronize());
  for (void* p : w.beam_allocs) cudaFree(p);
  w.beam_allocs.clear();
  for (auto& kv : Ln.graphs) cudaGraphExecDestroy(kv.second);
  Ln.graphs.clear();
  const int64_t R = w.B_cap, T = w.T_cap;
  auto& A = w.beam_allocs;
  w.part_ld = 2 * ((m->c.vocab + TOPK_BN - 1) / TOPK_BN);
  CKS(dalloc(A, &w.part, R * w.part_ld));
  CKS(dalloc(A, &w.row_lse, R));
  CKS(dalloc(A, &w.row_v, R * TOPK_MAX));
  CKS(dalloc(A, &w.row_j, R * TOPK_MAX));
  for (int32_t** p : {&w.sent_row0, &w.sent_nlive, &w.sent_nfin, &w.sent_list, &w.child_par,
                      &w.child_tok})
    CKS(dalloc(A, p, R));
  CKS(dalloc(A, &w.hscore, R));
  CKS(dalloc(A, &w.child_score, R));
  CKS(dalloc(A, &w.hist, R * T));
  if (m->c.decoder == 0) CKS(dalloc(A, &w.anc, R * T));
  CKS(dalloc(A, &w.logits, R * (((int64_t)m->c.vocab + 15) / 16 * 16)));
  w.beam_rows = R;
  w.beam_T = T;
  return MNMT_OK;
}

// Shortlist operand of a lane (F2): [V x d] int8 rows + bias + id map, allocated once.
static mnmt_status sl_lane_ensure(mnmt_model* m, Lane& Ln) {
  Workspace& w = Ln.ws;
  if (w.sl_q) return MNMT_OK;
  const int64_t V = m->c.vocab, d = m->c.d_model;
  CKS(dalloc(w.sl_allocs, &w.sl_q, V * d));
  CKS(dalloc(w.sl_allocs, &w.sl_b, V));
  CKS(dalloc(w.sl_allocs, &w.sl_map, V));
  CKS(dalloc(w.sl_allocs, &w.sl_bits, (int64_t)SL_MAX_GROUPS * ((V + 31) / 32)));
  CKS(dalloc(w.sl_allocs, &w.sl_rgrp, w.B_cap));
  if (!make_tmap_i8(&w.tm_sl, w.sl_q, V, d)) { set_err("tensor map (shortlist) failed"); return MNMT_ERR_CUDA; }
  return MNMT_OK;
}

// Job-level shortlist buffers.
static mnmt_status sl_job_ensure(mnmt_model* m, int64_t n_bb, int64_t n, int64_t n_waves,
                                 int64_t rows) {
  JobBuf& j = m->jb;
  if (n_bb <= j.sl_bb_cap && n <= j.sl_sent_cap && n_waves <= j.sl_wave_cap && rows <= j.sl_rows_cap)
    return MNMT_OK;
  CK(cudaDeviceSynchronize());
  for (void* p : j.sl_allocs) cudaFree(p);
  j.sl_allocs.clear();
  const int64_t V = m->c.vocab, W = (V + 31) / 32;
  j.sl_bb_cap = std::max(n_bb, j.sl_bb_cap);
  j.sl_sent_cap = std::max(n, j.sl_sent_cap);
  j.sl_wave_cap = std::max(n_waves, j.sl_wave_cap);
  j.sl_rows_cap = std::max(rows, j.sl_rows_cap);
  CKS(dalloc(j.sl_allocs, &j.sl_bits, j.sl_bb_cap * W));
  CKS(dalloc(j.sl_allocs, &j.sl_ids, j.sl_wave_cap * V));
  CKS(dalloc(j.sl_allocs, &j.sl_mask, j.sl_wave_cap * V));
  CKS(dalloc(j.sl_allocs, &j.sl_n, j.sl_wave_cap));
  CKS(dalloc(j.sl_allocs, &j.sl_span, 2 * j.sl_sent_cap + j.sl_bb_cap + j.sl_wave_cap + 2));
  CKS(dalloc(j.sl_allocs, &j.sl_rgrp, std::max<int64_t>(j.sl_rows_cap, 1)));
  return MNMT_OK;
}

// Builds every word-budget batch's shortlist and every decode wave's union (with per-column
// group masks) on the device, and reads the union sizes back (one synchronisation per job,
// before decoding: the output GEMM's N is a launch parameter of the step graphs).
// bb_sents: batch-major sentence indices; bb_off: [n_bb + 1]; wave_off: [n_waves + 1] first
// batch of each wave; rgrp: group of every job row (rmeta row order).
static mnmt_status sl_build_job(mnmt_model* m, const int64_t* src_off,
                                const std::vector<int32_t>& bb_sents,
                                const std::vector<int32_t>& bb_off,
                                const std::vector<int32_t>& wave_off,
                                const std::vector<int32_t>& rgrp) {
  const int n_bb = (int)bb_off.size() - 1, n_waves = (int)wave_off.size() - 1;
  const int64_t ns = (int64_t)bb_sents.size();
  CKS(sl_job_ensure(m, n_bb, ns, n_waves, (int64_t)rgrp.size()));
  JobBuf& j = m->jb;
  std::vector<int32_t> span(2 * ns + n_bb + 1 + n_waves + 1);
  for (int64_t i = 0; i < ns; ++i) {
    const int s = bb_sents[i];
    span[i] = (int32_t)src_off[s];
    span[ns + i] = (int32_t)(src_off[s + 1] - src_off[s]);
  }
  std::copy(bb_off.begin(), bb_off.end(), span.begin() + 2 * ns);
  std::copy(wave_off.begin(), wave_off.end(), span.begin() + 2 * ns + n_bb + 1);
  CK(cudaMemcpyAsync(j.sl_span, span.data(), span.size() * 4, cudaMemcpyHostToDevice, m->st));
  if (!rgrp.empty())
    CK(cudaMemcpyAsync(j.sl_rgrp, rgrp.data(), rgrp.size() * 4, cudaMemcpyHostToDevice, m->st));
  m->stats.h2d_bytes += (int64_t)(span.size() + rgrp.size()) * 4;
  SlMarkArgs a{};
  a.V = m->c.vocab;
  a.W = (m->c.vocab + 31) / 32;
  a.src_ids = j.src_ids;
  a.sent_start = j.sl_span;
  a.sent_len = j.sl_span + ns;
  a.bb_off = j.sl_span + 2 * ns;
  a.freq = m->sl_freq;
  a.n_freq = m->sl_nfreq;
  a.lex = m->sl_lex;
  a.k_lex = m->sl_k;
  a.eos = m->c.eos_id;
  a.unk = MNMT_UNK_ID;
  a.bits = j.sl_bits;
  CK(launch_sl_build(a, n_bb, j.sl_span + 2 * ns + n_bb + 1, n_waves, j.sl_ids, j.sl_mask,
                     j.sl_n, m->st));
  m->stats.gpu_launches += 2;
  m->sl_count.assign(n_waves, 0);
  m->sl_groups.resize(n_waves);
  for (int i = 0; i < n_waves; ++i) m->sl_groups[i] = wave_off[i + 1] - wave_off[i];
  if (n_waves > 0) {
    CK(cudaMemcpyAsync(m->sl_count.data(), j.sl_n, n_waves * 4, cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
  }
  return MNMT_OK;
}

static BeamArgs beam_args(mnmt_model* m, Lane& Ln, int n) {
  auto& w = Ln.ws;
  BeamArgs b{};
  b.beam = m->beam;
  b.n = n;
  b.ctrl = w.ctrl;
  b.live = w.live;
  b.prev_live = w.prev_live;
  b.live_start = w.live_start;
  b.live_len = w.live_len;
  b.row_start = w.row_start;
  b.row_len = w.row_len;
  b.max_len = w.max_len;
  b.out_off = w.out_off;
  b.len_idx = w.len_idx;
  b.eos = m->c.eos_id;
  b.part = w.part;
  b.part_ld = w.part_ld;
  b.n_part = 2 * ((m->c.vocab + TOPK_BN - 1) / TOPK_BN);
  b.row_lse = w.row_lse;
  b.row_v = w.row_v;
  b.row_j = w.row_j;
  b.sent_row0 = w.sent_row0;
  b.sent_nlive = w.sent_nlive;
  b.sent_nfin = w.sent_nfin;
  b.sent_list = w.sent_list;
  b.hscore = w.hscore;
  b.child_par = w.child_par;
  b.child_tok = w.child_tok;
  b.child_score = w.child_score;
  b.hist = w.hist;
  b.anc = w.anc;
  b.t_cap = (int)w.T_cap;
  b.C = m->c.decoder == 1 ? w.C : nullptr;
  b.c_stride = w.B_cap * m->c.d_model;
  b.L = m->c.dec_layers;
  b.d = m->c.d_model;
  b.logits = w.logits;
  b.V = m->c.vocab;
  b.ld_logits = ((int64_t)m->c.vocab + 15) / 16 * 16;
  b.out_ids = m->jb.out_ids;
  b.out_len = m->jb.out_len;
  b.out_score = m->jb.out_score;
  b.n_hyp = m->jb.n_hyp;
  return b;
}

// Grows a lane's workspace to hold M tokens, B rows, T steps, O forced ids.
static mnmt_status lane_ensure(mnmt_model* m, Lane& Ln, int64_t M, int64_t B, int64_t T, int64_t O) {
  Workspace& w = Ln.ws;
  if (M <= w.M_cap && B <= w.B_cap && T <= w.T_cap && O <= w.O_cap) return MNMT_OK;
  CK(cudaDeviceSynchronize());
  auto rnd = [](int64_t v, int64_t a) { return (std::max<int64_t>(v, 1) + a - 1) / a * a; };
  const int64_t Mc = rnd(std::max(M, w.M_cap), 128), Bc = rnd(std::max(B, w.B_cap), 128);
  const int64_t Tc = std::max(T, w.T_cap), Oc = std::max<int64_t>(std::max(O, w.O_cap), 1);
  lane_free(Ln);
  Workspace& z = Ln.ws;
  z.M_cap = Mc; z.B_cap = Bc; z.T_cap = Tc; z.O_cap = Oc;
  const auto& c = m->c;
  const int64_t d = c.d_model, F = c.d_ffn, L = c.dec_layers;
  auto& A = z.allocs;
  CKS(dalloc(A, &z.x, Mc * d));
  CKS(dalloc(A, &z.qkv, Mc * 3 * d));
  CKS(dalloc(A, &z.o, Mc * d));
  CKS(dalloc(A, &z.kv, L * Mc * 2 * d));
  if (c.src_kv_bf16) CKS(dalloc(A, &z.kv16, L * Mc * 2 * d));
  CKS(dalloc(A, &z.cx, Mc * d));
  CKS(dalloc(A, &z.cctx, Mc * d));
  CKS(dalloc(A, &z.ch, Mc * F));
  CKS(dalloc(A, &z.ctrl, 64));
  CKS(dalloc(A, &z.live, Bc));
  CKS(dalloc(A, &z.prev_id, Bc));
  CKS(dalloc(A, &z.prev_live, Bc));
  CKS(dalloc(A, &z.live_start, Bc));
  CKS(dalloc(A, &z.live_len, Bc));
  CKS(dalloc(A, &z.row_start, Bc));
  CKS(dalloc(A, &z.row_len, Bc));
  CKS(dalloc(A, &z.max_len, Bc));
  CKS(dalloc(A, &z.len_idx, Bc));
  CKS(dalloc(A, &z.out_off, Bc));
  CKS(dalloc(A, &z.forced_off, Bc));
  CKS(dalloc(A, &z.keys, Bc));
  CKS(dalloc(A, &z.C, L * Bc * d));
  for (float** p : {&z.y, &z.g, &z.a, &z.gi, &z.gf, &z.x1, &z.qs, &z.od, &z.x2, &z.f})
    CKS(dalloc(A, p, Bc * d));
  CKS(dalloc(A, &z.qkvd, Bc * 3 * d));
  if (c.decoder == 0) CKS(dalloc(A, &z.selfkv, L * Bc * Tc * 2 * d));
  for (int8_t** p : {&z.cy, &z.cg, &z.ch1, &z.ca, &z.cx1, &z.cctxd, &z.cx2})
    CKS(dalloc(A, p, Bc * d));
  CKS(dalloc(A, &z.chd, Bc * F));
  CKS(ws_tmap(&z.tm_cx, z.cx, Mc, d));
  CKS(ws_tmap(&z.tm_cctx, z.cctx, Mc, d));
  CKS(ws_tmap(&z.tm_ch, z.ch, Mc, F));
  CKS(ws_tmap(&z.tm_cy, z.cy, Bc, d));
  CKS(ws_tmap(&z.tm_cg, z.cg, Bc, d));
  CKS(ws_tmap(&z.tm_ch1, z.ch1, Bc, d));
  CKS(ws_tmap(&z.tm_ca, z.ca, Bc, d));
  CKS(ws_tmap(&z.tm_cx1, z.cx1, Bc, d));
  CKS(ws_tmap(&z.tm_cctxd, z.cctxd, Bc, d));
  CKS(ws_tmap(&z.tm_cx2, z.cx2, Bc, d));
  CKS(ws_tmap(&z.tm_chd, z.chd, Bc, F));
  if (!make_tmap_kv(&z.tm_kv, z.kv, L * Mc, 2 * d) ||
      (c.decoder == 0 && !make_tmap_kv(&z.tm_self, z.selfkv, L * Bc * Tc, 2 * d))) {
    set_err("cuTensorMapEncodeTiled failed (attention K/V)");
    return MNMT_ERR_CUDA;
  }
  return MNMT_OK;
}

// ------------------------------------------------------------------ launch helpers
static cudaError_t gemm(mnmt_model* m, cudaStream_t st, const CUtensorMap& tmA, const Lin& W, int M,
                        const int32_t* M_dyn, int epi, float* out_f, int8_t* out_q, int64_t ldo,
                        unsigned long long* keys = nullptr, int col_block = 0,
                        int64_t block_stride = 0, const int8_t* A = nullptr) {
  GemmArgs a{};
  a.a_ptr = A;   // raw A codes [M x W.in] (small-M path), or null
  a.lda = W.in;
  a.b_ptr = W.q;
  a.M = M;
  a.M_dyn = M_dyn;
  a.N = W.out;
  a.K = W.in;
  a.scale = scale_of(m);
  a.bias = W.b;
  a.clip = m->c.clip;
  a.sigma = sigma_of(m);
  a.out_f = out_f;
  a.out_q = out_q;
  a.ldo = ldo;
  a.col_block = col_block > 0 ? col_block : W.out;
  a.block_stride = block_stride;
  a.keys = keys;
  a.pers_grid = m->cur_pers_grid;
  a.smallm_rows = m->smallm;
  a.smallm_kmax = m->smallm_kmax;
  a.smallm_wmax = m->smallm_wmax;
  a.sab_rows = m->sab;
  a.sab_kmin = m->sab_kmin;
  a.sab_kb = m->sab_kb;
  a.split_k = m->split_k ? -1 : 0;
  return launch_gemm_i8(tmA, W.tm, a, epi, 0, st);
}

// Decoder GEMM that may take the small-M path (A also passed as a raw pointer).
static cudaError_t gemm_r(mnmt_model* m, cudaStream_t st, const CUtensorMap& tmA, const int8_t* A,
                          const Lin& W, int M, const int32_t* M_dyn, int epi, float* out_f,
                          int8_t* out_q, int64_t ldo) {
  return gemm(m, st, tmA, W, M, M_dyn, epi, out_f, out_q, ldo, nullptr, 0, 0, A);
}

static LnArgs ln_args(mnmt_model* m, const Workspace& w, int n, const int32_t* n_dyn, const float* x,
                      const float* delta, const float* gamma, const float* beta, float* out,
                      int8_t* out_q) {
  LnArgs a{};
  a.n = n;
  a.n_dyn = n_dyn;
  a.ctrl = w.ctrl;
  a.live = w.live;
  a.d = m->c.d_model;
  a.eps = m->c.ln_eps;
  a.x = x;
  a.delta = delta;
  a.gamma = gamma;
  a.beta = beta;
  a.out = out;
  a.out_q = out_q;
  a.clip = m->c.clip;
  a.sigma = sigma_of(m);
  a.aan.clip = m->c.clip;
  a.aan.sigma = sigma_of(m);
  return a;
}

// AAN step of decoder layer l fused into the producer of that layer's input.
static AanOut aan_for_layer(mnmt_model* m, const Workspace& w, int l) {
  AanOut o{};
  o.clip = m->c.clip;
  o.sigma = sigma_of(m);
  if (m->c.decoder != 1 || l >= m->c.dec_layers) return o;
  const int64_t d = m->c.d_model;
  o.C = w.C + (int64_t)l * w.B_cap * d;
  if (m->c.aan_ffn_depth == 0) {
    o.g_f = w.g;                       // a = g (fp32) for the residual / gate
    if (m->c.aan_gate) o.g_q = w.cg;   // Q(a) = Q(g) feeds the f-gate
  } else {
    o.g_q = w.cg;                      // Q(g) feeds the AAN FFN
  }
  return o;
}

// Encoder over M tokens (A2-A4).  meta: [idx M][pos M][start M][len M].
// order: the batch's rows in (length, row) order (device); buckets: {first, count, longest} ranges
// of it, one encoder-attention launch each.
static cudaError_t launch_encoder(mnmt_model* m, Lane& Ln, int M, const int32_t* order,
                                  const std::vector<std::array<int, 3>>& buckets,
                                  const int32_t* tok_idx, const int32_t* tok_pos,
                                  const int32_t* tok_start, const int32_t* tok_len, int64_t* nlaunch) {
  (void)tok_start;
  (void)tok_len;   // sentence spans come from the row metadata (row_start / row_len)
  auto& w = Ln.ws;
  cudaStream_t st = Ln.st;
  const auto& c = m->c;
  const int d = c.d_model;
  cudaError_t e;
  if ((e = launch_embed_src(m->jb.src_ids, tok_idx, tok_pos, M, m->E, m->PE, d, c.clip, w.x, w.cx,
                            st)) != cudaSuccess)
    return e;
  ++*nlaunch;
  for (int l = 0; l < c.enc_layers; ++l) {
    const EncLayer& E = m->enc[l];
    if ((e = gemm(m, st, w.tm_cx, E.qkv, M, nullptr, EPI_F32, w.qkv, nullptr, 3 * d)) != cudaSuccess) return e;
    EncAttnArgs at{};
    at.qkv = w.qkv;
    at.sent_start = w.row_start;
    at.sent_len = w.row_len;
    at.H = c.n_heads;
    at.dh = d / c.n_heads;
    at.d = d;
    at.clip = c.clip;
    at.sigma = sigma_of(m);
    at.out_q = w.cctx;
    for (const auto& bk : buckets) {
      at.sent_order = order + bk[0];
      at.n_sent = bk[1];
      at.s_max = bk[2];
      if ((e = launch_attn_enc(at, st)) != cudaSuccess) return e;
      ++*nlaunch;
    }
    --*nlaunch;   // counted below with the layer's other kernels
    LnArgs la = ln_args(m, w, M, nullptr, w.x, w.o, E.ln1g, E.ln1b, w.x, w.cx);
    LnArgs lb = ln_args(m, w, M, nullptr, w.x, w.o, E.ln2g, E.ln2b, w.x, w.cx);
    if ((e = gemm(m, st, w.tm_cctx, E.o, M, nullptr, EPI_F32, w.o, nullptr, d)) != cudaSuccess) return e;
    if ((e = launch_ln(la, st)) != cudaSuccess) return e;
    if ((e = gemm(m, st, w.tm_cx, E.f1, M, nullptr, EPI_RELU_Q, nullptr, w.ch, c.d_ffn)) != cudaSuccess) return e;
    if ((e = gemm(m, st, w.tm_ch, E.f2, M, nullptr, EPI_F32, w.o, nullptr, d)) != cudaSuccess) return e;
    if ((e = launch_ln(lb, st)) != cudaSuccess) return e;
    *nlaunch += 7;
  }
  // Source keys/values of all decoder layers in one GEMM, scattered to [L][M_cap][2d].
  if ((e = gemm(m, st, w.tm_cx, m->kv_all, M, nullptr, EPI_F32, w.kv, nullptr, 2 * d, nullptr, 2 * d,
                w.M_cap * 2 * d)) != cudaSuccess)
    return e;
  ++*nlaunch;
  if (c.src_kv_bf16) {   // F3 (R35): K/V rounded to bf16 once per batch; attention reads kv16
    if ((e = launch_kv_bf16(w.kv, w.kv16, c.dec_layers, (int64_t)M * 2 * d, w.M_cap * 2 * d, st)) !=
        cudaSuccess)
      return e;
    ++*nlaunch;
  }
  return cudaSuccess;
}


static cudaError_t dump_rows(mnmt_model* m, Lane& Ln, int n, const void* src, bool codes,
                             void* dst, int64_t slot, int64_t slots, int64_t* k) {
  auto& w = Ln.ws;
  DumpArgs a{};
  a.n = n;
  a.ctrl = w.ctrl;
  a.live = w.live;
  a.foff = w.forced_off;
  a.d = m->c.d_model;
  a.src = src;
  a.elem = codes ? 1 : 4;
  a.dst = dst;
  a.slot = slot;
  a.slots = slots;
  ++*k;
  return launch_dump_rows(a, Ln.st);
}

// One decoder step for up to `n` live rows (A5-A10).  Returns kernels launched via *nlaunch.
static cudaError_t launch_step(mnmt_model* m, Lane& Ln, int n, bool forced, int64_t* nlaunch) {
  auto& w = Ln.ws;
  cudaStream_t st = Ln.st;
  const auto& c = m->c;
  const int d = c.d_model, L = c.dec_layers, H = c.n_heads;
  const int32_t* nd = w.ctrl;  // ctrl[0] = live rows
  const DevDump& dd = m->dump;
  cudaError_t e;
  int64_t k = 0;
  EmbedTgtArgs ea{};
  ea.ctrl = w.ctrl;
  ea.live = w.live;
  ea.prev_id = w.prev_id;
  ea.prev_live = w.prev_live;
  ea.E = m->E;
  ea.PE = m->PE;
  ea.d = d;
  ea.rsd = (float)std::sqrt((double)d);
  ea.y = w.y;
  ea.yq = w.cy;
  ea.aan = aan_for_layer(m, w, 0);
  if ((e = launch_embed_tgt(ea, n, st)) != cudaSuccess) return e;
  ++k;
  for (int l = 0; l < L; ++l) {
    const DecLayer& D = m->dec[l];
    LnArgs l1;
    if (c.decoder == 1) {
      // A6: AAN block. g (or its codes) was produced with this layer's input.
      const float* a_f = w.g;
      // The i-gate GEMM needs only Q(y): it runs on a forked branch beside the AAN FFN.
      // (measured: in-line is slower; the branch runs beside the AAN FFN)
      const bool fork = c.aan_gate && c.aan_ffn_depth > 0;
      if (fork) {
        if ((e = cudaEventRecord(Ln.ev_fork, st)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(Ln.side, Ln.ev_fork, 0)) != cudaSuccess) return e;
        if ((e = gemm(m, Ln.side, w.tm_cy, D.gi, n, nd, EPI_F32, w.gi, nullptr, d)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(Ln.ev_join, Ln.side)) != cudaSuccess) return e;
      }
      if (c.aan_ffn_depth == 2) {
        if ((e = gemm_r(m, st, w.tm_cg, w.cg, D.a1, n, nd, EPI_RELU_Q, nullptr, w.ch1, d)) != cudaSuccess) return e;
        if ((e = gemm_r(m, st, w.tm_ch1, w.ch1, D.a2, n, nd, EPI_F32_Q, w.a, w.ca, d)) != cudaSuccess) return e;
        a_f = w.a;
        k += 2;
      } else if (c.aan_ffn_depth == 1) {
        if ((e = gemm_r(m, st, w.tm_cg, w.cg, D.a1, n, nd, EPI_RELU_F32_Q, w.a, w.ca, d)) != cudaSuccess) return e;
        a_f = w.a;
        k += 1;
      }
      l1 = ln_args(m, w, n, nd, w.y, a_f, D.ln[0][0], D.ln[0][1], w.x1, w.cx1);
      if (c.aan_gate) {
        // gate (R8): logits W_i Q(y) + b_i and W_f Q(a) + b_f (for -ffn, Q(a) = Q(g));
        // the sigmoids are applied in the gate-LayerNorm kernel
        const CUtensorMap& tm_a = c.aan_ffn_depth == 0 ? w.tm_cg : w.tm_ca;
        const int8_t* a_ptr = c.aan_ffn_depth == 0 ? w.cg : w.ca;
        if (!fork) {
          if ((e = gemm_r(m, st, w.tm_cy, w.cy, D.gi, n, nd, EPI_F32, w.gi, nullptr, d)) != cudaSuccess) return e;
        }
        if ((e = gemm_r(m, st, tm_a, a_ptr, D.gf, n, nd, EPI_F32, w.gf, nullptr, d)) != cudaSuccess) return e;
        if (fork && (e = cudaStreamWaitEvent(st, Ln.ev_join, 0)) != cudaSuccess)
          return e;   // join before the gate LayerNorm reads gi
        l1.gi = w.gi;
        l1.gf = w.gf;
        k += 2;
      }
    } else {
      // A6': self-attention with a KV cache
      if ((e = gemm_r(m, st, w.tm_cy, w.cy, D.qkv, n, nd, EPI_F32, w.qkvd, nullptr, 3 * d)) != cudaSuccess) return e;
      AttnArgs at{};
      at.mode = ATTN_SELF;
      at.span = Ln.span_cap;
      at.n = n;
      at.n_dyn = nd;
      at.ctrl = w.ctrl;
      at.live = w.live;
      at.H = H;
      at.dh = d / H;
      at.d = d;
      at.q = w.qkvd;
      at.ldq = 3 * d;
      at.kv = w.selfkv + (int64_t)l * w.B_cap * w.T_cap * 2 * d;
      at.kv_w = const_cast<float*>(at.kv);
      at.ldkv = 2 * d;
      at.k_off = 0;
      at.v_off = d;
      at.t_cap = (int)w.T_cap;
      at.anc = m->beam > 0 ? w.anc : nullptr;
      at.tmap = &w.tm_self;             // TMA tiles (greedy; beam search reads through anc)
      at.tma_self = m->attn_tma_self;
      at.f32 = m->attn_f32;
      at.kv_row0 = (int64_t)l * w.B_cap * w.T_cap;
      at.clip = c.clip;
      at.sigma = sigma_of(m);
      at.out_q = w.cctxd;
      if ((e = launch_attn(at, st)) != cudaSuccess) return e;
      if ((e = gemm_r(m, st, w.tm_cctxd, w.cctxd, D.o, n, nd, EPI_F32, w.od, nullptr, d)) != cudaSuccess) return e;
      k += 3;
      l1 = ln_args(m, w, n, nd, w.y, w.od, D.ln[0][0], D.ln[0][1], w.x1, w.cx1);
    }
    if ((e = launch_ln(l1, st)) != cudaSuccess) return e;
    ++k;
    if (dd.layers && (e = dump_rows(m, Ln, n, w.x1, false, dd.layers, 3 * l + 0, 3 * L, &k)) != cudaSuccess)
      return e;
    // A7: source attention
    if ((e = gemm_r(m, st, w.tm_cx1, w.cx1, D.sq, n, nd, EPI_F32, w.qs, nullptr, d)) != cudaSuccess) return e;
    AttnArgs as{};
    as.mode = ATTN_SRC;
    as.span = Ln.span_cap;
    as.n = n;
    as.n_dyn = nd;
    as.ctrl = w.ctrl;
    as.live = w.live;
    as.H = H;
    as.dh = d / H;
    as.d = d;
    as.q = w.qs;
    as.ldq = d;
    as.kv = w.kv + (int64_t)l * w.M_cap * 2 * d;
    as.kv16 = c.src_kv_bf16 ? w.kv16 + (int64_t)l * w.M_cap * 2 * d : nullptr;
    as.tmap = &w.tm_kv;                // TMA tiles (fp32 K/V)
    as.f32 = m->attn_f32;
    as.kv_row0 = (int64_t)l * w.M_cap;
    as.ldkv = 2 * d;
    as.k_off = 0;
    as.v_off = d;
    as.kv_start = w.row_start;
    as.kv_len = w.row_len;
    as.live_start = w.live_start;
    as.live_len = w.live_len;
    as.clip = c.clip;
    as.sigma = sigma_of(m);
    as.out_q = w.cctxd;
    if ((e = launch_attn(as, st)) != cudaSuccess) return e;
    LnArgs l2 = ln_args(m, w, n, nd, w.x1, w.od, D.ln[1][0], D.ln[1][1], w.x2, w.cx2);
    if ((e = gemm_r(m, st, w.tm_cctxd, w.cctxd, D.so, n, nd, EPI_F32, w.od, nullptr, d)) != cudaSuccess) return e;
    if ((e = launch_ln(l2, st)) != cudaSuccess) return e;
    k += 4;
    if (dd.layers && (e = dump_rows(m, Ln, n, w.x2, false, dd.layers, 3 * l + 1, 3 * L, &k)) != cudaSuccess)
      return e;
    // A8: FFN
    if ((e = gemm_r(m, st, w.tm_cx2, w.cx2, D.f1, n, nd, EPI_RELU_Q, nullptr, w.chd, c.d_ffn)) != cudaSuccess) return e;
    LnArgs l3 = ln_args(m, w, n, nd, w.x2, w.f, D.ln[2][0], D.ln[2][1], w.y, w.cy);
    l3.aan = aan_for_layer(m, w, l + 1);
    if ((e = gemm_r(m, st, w.tm_chd, w.chd, D.f2, n, nd, EPI_F32, w.f, nullptr, d)) != cudaSuccess) return e;
    if ((e = launch_ln(l3, st)) != cudaSuccess) return e;
    k += 3;
    if (dd.layers && (e = dump_rows(m, Ln, n, w.y, false, dd.layers, 3 * l + 2, 3 * L, &k)) != cudaSuccess)
      return e;
  }
  if (dd.dec_out && (e = dump_rows(m, Ln, n, w.y, false, dd.dec_out, 0, 1, &k)) != cudaSuccess) return e;
  if (dd.out_codes && (e = dump_rows(m, Ln, n, w.cy, true, dd.out_codes, 0, 1, &k)) != cudaSuccess) return e;
  if (m->beam > 0) {
    // beam search (F1): output GEMM with per-tile log-sum-exp partials and top-k (EPI_TOPK),
    // then row merge, per-sentence selection + compaction, state reorder (beam.h)
    GemmArgs a{};
    a.M = n;
    a.M_dyn = nd;
    a.N = c.vocab;
    a.K = d;
    a.scale = scale_of(m);
    a.bias = c.out_bias ? m->out_b : nullptr;
    a.clip = c.clip;
    a.sigma = sigma_of(m);
    a.col_block = c.vocab;
    const BeamArgs ba = beam_args(m, Ln, n);
    if (m->beam_fused) {
      a.part = w.part;
      a.part_ld = w.part_ld;
      const int epi = m->beam <= 2 ? EPI_TOPK2 : m->beam <= 4 ? EPI_TOPK4 : EPI_TOPK;
      if ((e = launch_gemm_i8(w.tm_cy, m->tmE, a, epi, 0, st)) != cudaSuccess) return e;
      if ((e = launch_beam_rows(ba, st)) != cudaSuccess) return e;
    } else {
      a.out_f = w.logits;
      a.ldo = ba.ld_logits;
      a.pers_grid = m->cur_pers_grid;
      if ((e = launch_gemm_i8(w.tm_cy, m->tmE, a, EPI_F32, 0, st)) != cudaSuccess) return e;
      if ((e = launch_beam_logits(ba, st)) != cudaSuccess) return e;
    }
    if ((e = launch_beam_select(ba, st)) != cudaSuccess) return e;
    if ((e = launch_beam_reorder(ba, st)) != cudaSuccess) return e;
    k += 4;
    *nlaunch += k;
    return cudaSuccess;
  }
  if (dd.margin) {
    // test hook: the step's top-2 logit margin from an EPI_TOPK2 pass over the same operands
    GemmArgs a{};
    a.M = n;
    a.M_dyn = nd;
    a.N = c.vocab;
    a.K = d;
    a.scale = scale_of(m);
    a.bias = c.out_bias ? m->out_b : nullptr;
    a.clip = c.clip;
    a.sigma = sigma_of(m);
    a.col_block = c.vocab;
    a.part = w.part;
    a.part_ld = w.part_ld;
    if ((e = launch_gemm_i8(w.tm_cy, m->tmE, a, EPI_TOPK2, 0, st)) != cudaSuccess) return e;
    if ((e = launch_top2_margin(w.part, w.part_ld, 2 * ((c.vocab + TOPK_BN - 1) / TOPK_BN), n, w.ctrl,
                                w.live, w.forced_off, dd.margin, st)) != cudaSuccess)
      return e;
    k += 2;
  }
  // A9: tied output projection fused with the argmax (softmax skipped)
  {
    GemmArgs a{};
    // shortlist (F2): the GEMM runs over the decode unit's Ln.sl_n gathered rows of qE
    const bool sl = Ln.sl_n > 0;
    a.M = n;
    a.M_dyn = nd;
    a.N = sl ? Ln.sl_n : c.vocab;
    a.K = d;
    a.scale = scale_of(m);
    a.bias = c.out_bias ? (sl ? w.sl_b : m->out_b) : nullptr;
    a.clip = c.clip;
    a.sigma = sigma_of(m);
    a.col_block = a.N;
    a.keys = w.keys;
    a.a_ptr = w.cy;   // swap-AB path at <= sab_out rows
    a.lda = d;
    a.sab_rows = m->sab_out;
    a.sab_kb = m->sab_kb;
    if (sl) {
      a.colbits = w.sl_bits;
      a.colbits_ld = (c.vocab + 31) / 32;
      a.row_grp = w.sl_rgrp;
      a.row_live = w.live;
    }
    a.pers_grid = m->cur_pers_grid;
    if ((e = launch_gemm_i8(w.tm_cy, sl ? w.tm_sl : m->tmE, a, EPI_ARGMAX, 0, st)) != cudaSuccess)
      return e;
  }
  // A10: finish + compaction
  FinishArgs fa{};
  fa.ctrl = w.ctrl;
  fa.live = w.live;
  fa.keys = w.keys;
  fa.prev_id = w.prev_id;
  fa.max_len = w.max_len;
  fa.out_off = w.out_off;
  fa.out_ids = m->jb.out_ids;
  fa.out_len = m->jb.out_len;
  fa.len_idx = w.len_idx;
  fa.eos = c.eos_id;
  fa.forced = forced ? m->jb.forced : nullptr;
  fa.forced_off = forced ? w.forced_off : nullptr;
  fa.prev_live = w.prev_live;
  fa.row_start = w.row_start;
  fa.row_len = w.row_len;
  fa.live_start = w.live_start;
  fa.live_len = w.live_len;
  fa.id_map = Ln.sl_n > 0 ? w.sl_map : nullptr;
  if ((e = launch_finish(fa, st)) != cudaSuccess) return e;
  k += 2;
  *nlaunch += k;
  return cudaSuccess;
}

// ------------------------------------------------------------------ job planning
struct Batch {
  std::vector<int32_t> rows;  // sentence indices in row order
  int64_t tok0 = 0;           // first token of this batch in the job's token metadata
  int64_t M = 0;
  int T = 0;                  // max steps
  int lane = 0;               // decoder lane (stream) that runs this batch
  int S_max = 1;              // longest source sentence
  int bb = -1;                // shortlist (F2): decode wave whose union this unit uses, -1 = none
  std::vector<int32_t> alive; // alive[t-1] = rows with max_len >= t (upper bound of live rows)
  // encoder attention launches: {first index into the length-sorted row order, rows, longest}
  std::vector<std::array<int, 3>> enc_buckets;
};

struct Job {
  std::vector<Batch> batches;
  std::vector<int32_t> meta;  // per batch: tok_idx, tok_pos, tok_start, tok_len (4 x M)
  std::vector<int64_t> out_off;  // per sentence: output offset (prefix sum of max_len)
  std::vector<int32_t> rmeta32;  // per batch: [row_start|row_len|max_len|len_idx|len_order] x B
  std::vector<int64_t> rmeta64;  // per batch: [out_off|forced_off] x B
  std::vector<int64_t> r0;       // per batch: first row in rmeta
  int64_t out_total = 0, tok_total = 0, rows_total = 0;
  int64_t maxM = 0, maxB = 0;
  int maxT = 0;
  std::vector<int64_t> lane_M, lane_B, lane_T;   // per-lane maxima (workspace sizing)
};

static mnmt_status check_inputs(mnmt_model* m, const int64_t* src_off, int32_t n,
                                const int32_t* max_len) {
  if (n < 0) { set_err("n < 0"); return MNMT_ERR_ARG; }
  if (n > 0 && (!src_off || !max_len)) { set_err("NULL src_off / max_len"); return MNMT_ERR_ARG; }
  if (n > 0 && src_off[0] != 0) { set_err("src_off[0] must be 0"); return MNMT_ERR_ARG; }
  for (int i = 0; i < n; ++i) {
    const int64_t S = src_off[i + 1] - src_off[i];
    if (S < 0) { set_err("src_off not monotone at %d", i); return MNMT_ERR_ARG; }
    if (S > MNMT_MAX_SPAN) { set_err("sentence %d longer than MNMT_MAX_SPAN", i); return MNMT_ERR_CAPACITY; }
    if (max_len[i] < 0) { set_err("max_len[%d] < 0", i); return MNMT_ERR_ARG; }
    if (max_len[i] > MNMT_MAX_SPAN) { set_err("max_len[%d] > MNMT_MAX_SPAN", i); return MNMT_ERR_CAPACITY; }
  }
  return MNMT_OK;
}

static void plan_job(const int64_t* src_off, int32_t n, const int32_t* max_len,
                     const std::vector<std::vector<int32_t>>& batch_rows,
                     const std::vector<int>& batch_lane, int n_lanes, Job& job,
                     const std::vector<int>* batch_bb = nullptr) {
  job.lane_M.assign(n_lanes, 0);
  job.lane_B.assign(n_lanes, 0);
  job.lane_T.assign(n_lanes, 0);
  size_t bi_in = 0;
  job.out_off.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) job.out_off[i + 1] = job.out_off[i] + max_len[i];
  job.out_total = job.out_off[n];
  job.tok_total = n > 0 ? src_off[n] : 0;
  for (const auto& rows_all : batch_rows) {
    Batch b;
    b.lane = batch_lane.empty() ? 0 : batch_lane[bi_in];
    b.bb = batch_bb ? (*batch_bb)[bi_in] : -1;
    ++bi_in;
    for (int32_t s : rows_all)
      if (max_len[s] > 0) b.rows.push_back(s);   // max_len 0: nothing to decode
    if (b.rows.empty()) continue;
    b.tok0 = (int64_t)job.meta.size();
    int64_t M = 0;
    for (int32_t s : b.rows) {
      M += src_off[s + 1] - src_off[s];
      b.T = std::max(b.T, max_len[s]);
      b.S_max = std::max<int>(b.S_max, (int)(src_off[s + 1] - src_off[s]));
    }
    b.M = M;
    b.alive.assign(b.T, 0);
    for (int32_t s : b.rows)
      for (int t = 0; t < max_len[s]; ++t) ++b.alive[t];
    job.meta.resize(job.meta.size() + 4 * M);
    int32_t* idx = job.meta.data() + b.tok0;
    int32_t *pos = idx + M, *st = idx + 2 * M, *ln = idx + 3 * M;
    int64_t t = 0;
    for (int32_t s : b.rows) {
      const int64_t S = src_off[s + 1] - src_off[s];
      for (int64_t j = 0; j < S; ++j) {
        idx[t + j] = (int32_t)(src_off[s] + j);
        pos[t + j] = (int32_t)j;
        st[t + j] = (int32_t)t;
        ln[t + j] = (int32_t)S;
      }
      t += S;
    }
    job.maxM = std::max(job.maxM, M);
    job.maxB = std::max<int64_t>(job.maxB, (int64_t)b.rows.size());
    job.maxT = std::max(job.maxT, b.T);
    job.lane_M[b.lane] = std::max(job.lane_M[b.lane], M);
    job.lane_B[b.lane] = std::max<int64_t>(job.lane_B[b.lane], (int64_t)b.rows.size());
    job.lane_T[b.lane] = std::max<int64_t>(job.lane_T[b.lane], b.T);
    job.batches.push_back(std::move(b));
  }
}

// Row metadata of every batch, staged host-side once per job (uploaded in one copy).
static void plan_rows(Job& job, const int64_t* src_off, const int32_t* max_len, bool forced,
                      const int64_t* forced_off, int d_model) {
  job.rmeta32.clear();
  job.rmeta64.clear();
  job.r0.clear();
  int64_t r0 = 0;
  for (Batch& b : job.batches) {
    const int B = (int)b.rows.size();
    job.r0.push_back(r0);
    job.rmeta32.resize((size_t)5 * (r0 + B));
    int32_t* rs = job.rmeta32.data() + 5 * r0;
    int32_t *rl = rs + B, *ml = rs + 2 * B, *li = rs + 3 * B, *ord = rs + 4 * B;
    job.rmeta64.resize((size_t)2 * (r0 + B));
    int64_t* oo = job.rmeta64.data() + 2 * r0;
    int64_t* fo = oo + B;
    int64_t t = 0;
    for (int r = 0; r < B; ++r) {
      const int s = b.rows[r];
      const int64_t S = src_off[s + 1] - src_off[s];
      rs[r] = (int32_t)t;
      rl[r] = (int32_t)S;
      ml[r] = max_len[s];
      li[r] = s;
      oo[r] = job.out_off[s];
      fo[r] = forced ? forced_off[s] : 0;
      t += S;
    }
    // rows in (length, row) order, cut into length buckets for the encoder attention
    for (int r = 0; r < B; ++r) ord[r] = r;
    std::stable_sort(ord, ord + B, [&](int32_t x, int32_t y) { return rl[x] < rl[y]; });
    // (one launch per bucket: shared memory and warps per CTA follow the bucket's longest).  The
    // fine edges keep the multi-query kernel's warps busy where the encoder attention is heavy
    // (d >= 512; measured: big 86.5 -> 84.8 ms per job, base-AAN 50.9 -> 50.5, small-AAN 37.4 ->
    // 38.3 from the extra launches, profiles/r2_sab_enc_ab.txt); env MNMT_ENC_FINE = 0 / 1 forces
    static const int kCoarse[] = {32, 64, 128, MNMT_MAX_SPAN};
    static const int kFine[] = {8, 12, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 100, 128, MNMT_MAX_SPAN};
    static const int fine_env = [] {
      const char* e = getenv("MNMT_ENC_FINE");
      return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const bool fine = fine_env >= 0 ? fine_env == 1 : d_model >= 512;
    const int* kEdges = fine ? kFine : kCoarse;
    b.enc_buckets.clear();
    for (int i = 0, e = 0; i < B;) {
      while (rl[ord[i]] > kEdges[e]) ++e;
      int j = i;
      while (j < B && rl[ord[j]] <= kEdges[e]) ++j;
      b.enc_buckets.push_back({i, j - i, rl[ord[j - 1]]});
      i = j;
    }
    r0 += B;
  }
  job.rows_total = r0;
}

// Runs every batch of a job on m->st.  Source ids must already be in ws.src_ids and
// the metadata in ws.meta / ws.rmeta* (upload_job).
static mnmt_status upload_job(mnmt_model* m, const Job& job) {
  auto& w = m->jb;
  if (!job.meta.empty())
    CK(cudaMemcpyAsync(w.meta, job.meta.data(), job.meta.size() * 4, cudaMemcpyHostToDevice, m->st));
  if (!job.rmeta32.empty()) {
    CK(cudaMemcpyAsync(w.rmeta32, job.rmeta32.data(), job.rmeta32.size() * 4, cudaMemcpyHostToDevice, m->st));
    CK(cudaMemcpyAsync(w.rmeta64, job.rmeta64.data(), job.rmeta64.size() * 8, cudaMemcpyHostToDevice, m->st));
  }
  m->stats.h2d_bytes += (int64_t)job.meta.size() * 4 + (int64_t)job.rmeta32.size() * 4 +
                        (int64_t)job.rmeta64.size() * 8;
  // pageable host memory: the copies above are staged before cudaMemcpyAsync returns
  return MNMT_OK;
}

static mnmt_status run_job(mnmt_model* m, const Job& job, bool forced) {
  const auto& c = m->c;
  const int64_t d = c.d_model;
  int64_t launches = 0, steps = 0;
  // fan out: every lane waits for the uploads on the main stream
  CK(cudaEventRecord(m->ev_job, m->st));
  std::vector<char> used(m->lanes.size(), 0);
  for (const Batch& b : job.batches) used[b.lane] = 1;
  for (size_t li = 0; li < m->lanes.size(); ++li)
    if (used[li]) CK(cudaStreamWaitEvent(m->lanes[li].st, m->ev_job, 0));
  for (size_t bi = 0; bi < job.batches.size(); ++bi) {
    const Batch& b = job.batches[bi];
    Lane& Ln = m->lanes[b.lane];
    auto& w = Ln.ws;
    cudaStream_t st = Ln.st;
    const int B = (int)b.rows.size();
    const int32_t* r32 = m->jb.rmeta32 + 5 * job.r0[bi];
    const int64_t* r64 = m->jb.rmeta64 + 2 * job.r0[bi];
    CK(cudaMemcpyAsync(w.row_start, r32, B * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(w.row_len, r32 + B, B * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(w.max_len, r32 + 2 * B, B * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(w.len_idx, r32 + 3 * B, B * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(w.out_off, r64, B * 8, cudaMemcpyDeviceToDevice, st));
    if (forced) CK(cudaMemcpyAsync(w.forced_off, r64 + B, B * 8, cudaMemcpyDeviceToDevice, st));
    // tiered lanes: the last lane (longest sentences) is the critical path; the persistent
    // GEMMs of the other lanes leave pers_reserve SMs free for it
    {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->dev);
      const bool critical = b.lane == m->n_lanes - 1 || m->n_lanes <= 1 || m->lane_tiers == 0;
      m->cur_pers_grid = (!critical && m->pers_reserve > 0) ? std::max(1, sms - m->pers_reserve) : 0;
      if (Ln.kind > 0) m->cur_pers_grid = m->green_count[Ln.kind - 1];   // the lane's SM partition
    }
    const int32_t* base = m->jb.meta + b.tok0;
    const int M = (int)b.M;
    CK(launch_encoder(m, Ln, M, r32 + 4 * B, b.enc_buckets, base, base + M, base + 2 * M, base + 3 * M,
                      &launches));
    if (c.decoder == 1)
      CK(cudaMemsetAsync(w.C, 0, (size_t)c.dec_layers * w.B_cap * d * sizeof(float), st));
    if (m->beam > 0) {
      CK(launch_beam_init(beam_args(m, Ln, B), B, st));
    } else {
      CK(launch_decode_init(w.ctrl, w.live, B, w.keys, w.row_start, w.row_len, w.live_start,
                            w.live_len, st));
    }
    launches += 1;
    if (m->sl_active && b.bb >= 0) {
      const int nsl = m->sl_count[b.bb];
      CK(launch_sl_gather(m->jb.sl_ids + (int64_t)b.bb * c.vocab,
                          m->jb.sl_mask + (int64_t)b.bb * c.vocab, nsl, m->sl_groups[b.bb], m->qE,
                          c.out_bias ? m->out_b : nullptr, (int)d, w.sl_q,
                          c.out_bias ? w.sl_b : nullptr, w.sl_map, w.sl_bits,
                          (c.vocab + 31) / 32, st));
      CK(cudaMemcpyAsync(w.sl_rgrp, m->jb.sl_rgrp + job.r0[bi], B * 4, cudaMemcpyDeviceToDevice, st));
      launches += 1;
      Ln.sl_n = nsl;
    } else {
      Ln.sl_n = 0;
    }
    const int npad = (B + 127) / 128 * 128;
    // attention scratch is sized by the longest span a step can attend (source length, or the
    // step count for the self-attention decoder); it only grows, and captured graphs are
    // rebuilt when it does
    {
      const int need = std::max(b.S_max, c.decoder == 0 ? b.T : 0);
      if (need > Ln.span_cap) {
        for (auto& kv : Ln.graphs) cudaGraphExecDestroy(kv.second);
        Ln.graphs.clear();
        Ln.span_cap = std::min(MNMT_MAX_KV, (need + 31) / 32 * 32);
      }
    }
    // per-step row bound: rows are compacted to the front and a row never outlives its
    // max_len, so step t needs at most alive[t-1] rows -> the smallest cached graph that fits
    // (128-row multiples; the small-M GEMM bound below that)
    const int rows_per = std::max(1, m->beam);   // beam search: up to beam rows per sentence
    auto pad_at = [&](int t) {
      const int a = b.alive[t] * rows_per;
      if (a <= std::max(m->sab, m->sab_out) && m->beam == 0)   // swap-AB row tiers
        return a <= 16 ? 16 : a <= 32 ? 32 : a <= 64 ? 64 : 128;
      if (a <= m->smallm && m->beam == 0) return m->smallm;   // small-M GEMMs
      return (a + 127) / 128 * 128;
    };
    // k consecutive steps per graph (PDL chains the kernels inside a graph, not across graph
    // launches), sized for the first step's row bound (rows only decrease)
    const int K = std::max(1, m->steps_per_graph);
    for (int t = 0; t < b.T;) {
      const int np = pad_at(t), k = std::min(K, b.T - t);
      const int64_t key = ((((int64_t)np * 64 + k) * 16 + m->beam) * ((int64_t)c.vocab + 1) + Ln.sl_n) * 2 +
                          (m->dump.any() ? 1 : 0);
      auto it = Ln.graphs.find(key);
      if (it == Ln.graphs.end()) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int64_t per_step = 0;
        cudaError_t e = cudaSuccess;
        for (int u = 0; u < k && e == cudaSuccess; ++u) e = launch_step(m, Ln, np, forced, &per_step);
        cudaError_t e2 = cudaStreamEndCapture(st, &g);
        CK(e);
        CK(e2);
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        if (Ln.graphs.size() >= 2048) {   // bound the cache (shortlist sizes vary per batch)
          CK(cudaStreamSynchronize(st));
          for (auto& kv : Ln.graphs) cudaGraphExecDestroy(kv.second);
          Ln.graphs.clear();
        }
        it = Ln.graphs.emplace(key, ge).first;
        Ln.graph_launches[key] = per_step;
      }
      CK(cudaGraphLaunch(it->second, st));
      launches += Ln.graph_launches[key];
      t += k;
    }
    if (m->beam > 0) {
      CK(launch_beam_final(beam_args(m, Ln, B), B, st));
      launches += 1;
    }
    steps += b.T;
  }
  // join: the main stream waits for every lane
  for (size_t li = 0; li < m->lanes.size(); ++li)
    if (used[li]) {
      CK(cudaEventRecord(m->lanes[li].ev, m->lanes[li].st));
      CK(cudaStreamWaitEvent(m->st, m->lanes[li].ev, 0));
    }
  m->stats.gpu_launches += launches;
  m->stats.decode_steps += steps;
  m->stats.batches += (int64_t)job.batches.size();
  return MNMT_OK;
}

// Sizes every lane a job uses.
static mnmt_status ensure_lanes(mnmt_model* m, const Job& job, int64_t forced_O) {
  for (size_t li = 0; li < job.lane_M.size(); ++li) {
    if (job.lane_B[li] == 0) continue;
    CKS(lane_init(m, m->lanes[li], (int)li));
    CKS(lane_ensure(m, m->lanes[li], job.lane_M[li], job.lane_B[li] * std::max(1, m->beam),
                    job.lane_T[li], forced_O));
    if (m->beam > 0) CKS(beam_ensure(m, m->lanes[li]));
    if (m->sl_active) CKS(sl_lane_ensure(m, m->lanes[li]));
  }
  return MNMT_OK;
}

static mnmt_status begin_call(mnmt_model* m, void* cuda_stream) {
  if (m->failed) { set_err("handle is fail-stopped after an earlier CUDA error"); return MNMT_ERR_STATE; }
  if (!m->quantized) { set_err("decode before mnmt_model_quantize"); return MNMT_ERR_STATE; }
  m->stats = mnmt_stats{};
  CK(cudaEventRecord(m->ev_in, (cudaStream_t)cuda_stream));
  CK(cudaStreamWaitEvent(m->st, m->ev_in, 0));
  return MNMT_OK;
}

static mnmt_status end_call(mnmt_model* m, void* cuda_stream) {
  CK(cudaEventRecord(m->ev_out, m->st));
  CK(cudaStreamWaitEvent((cudaStream_t)cuda_stream, m->ev_out, 0));
  CK(cudaStreamSynchronize(m->st));
  return MNMT_OK;
}

static mnmt_status check_ids_host(const mnmt_model* m, const int32_t* ids, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= m->c.vocab) {
      set_err("token id %d at %lld out of range [0, %d)", ids[i], (long long)i, m->c.vocab);
      return MNMT_ERR_VOCAB;
    }
  return MNMT_OK;
}

// Device-side id validation (DEVICE_IO mode): counts out-of-range ids.
__global__ void k_count_bad_ids(const int32_t* ids, int64_t n, int V, int32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (ids[i] < 0 || ids[i] >= V) atomicAdd(bad, 1);
}

}  // namespace

// ======================================================================== C ABI
extern "C" {

void mnmt_config_default(mnmt_config* c, int32_t d_model, int32_t d_ffn, int32_t n_heads) {
  if (!c) return;
  c->abi_version = MNMT_ABI_VERSION;
  c->d_model = d_model;
  c->d_ffn = d_ffn;
  c->n_heads = n_heads;
  c->enc_layers = 6;
  c->dec_layers = 6;
  c->vocab = 36000;
  c->decoder = 1;
  c->aan_ffn_depth = 2;
  c->aan_gate = 1;
  c->out_bias = 1;
  c->eos_id = 0;
  c->clip = 2.0f;
  c->ln_eps = 1e-6f;
  c->src_kv_bf16 = 0;
}

mnmt_status mnmt_model_create(const mnmt_config* cfg, int32_t cuda_device, mnmt_model** out) {
  if (!out) { set_err("out is NULL"); return MNMT_ERR_ARG; }
  *out = nullptr;
  if (const char* p = cfg_problem(cfg)) { set_err("bad config: %s", p); return MNMT_ERR_ARG; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) {
    cudaGetLastError();
    set_err("CUDA device %d not available", cuda_device);
    return MNMT_ERR_CUDA;
  }
  DeviceGuard g(cuda_device);
  {
    DeviceGuard g0(cuda_device);
    cudaError_t e = gemm_init();
    if (e == cudaSuccess) e = attn_init();
    if (e != cudaSuccess) {
      set_err("kernel init failed: %s", cudaGetErrorString(e));
      return MNMT_ERR_CUDA;
    }
  }
  mnmt_model* m = new mnmt_model();
  m->c = *cfg;
  m->dev = cuda_device;
  build_manifest(m);
  m->lanes.resize(1);
  if (cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&m->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&m->ev_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&m->ev_job, cudaEventDisableTiming) != cudaSuccess ||
      lane_init(m, m->lanes[0], 0) != MNMT_OK) {
    set_err("stream/event creation failed");
    delete m;
    return MNMT_ERR_CUDA;
  }
  *out = m;
  return MNMT_OK;
}

mnmt_status mnmt_model_set_param(mnmt_model* m, const char* name, const float* host,
                                 int64_t numel) {
  if (!m || !name || (!host && numel > 0)) { set_err("NULL argument"); return MNMT_ERR_ARG; }
  if (m->failed) { set_err("handle is fail-stopped"); return MNMT_ERR_STATE; }
  if (m->quantized) { set_err("set_param after quantize (weights are immutable)"); return MNMT_ERR_STATE; }
  auto it = m->manifest.find(name);
  if (it == m->manifest.end()) { set_err("unknown parameter '%s' for this config", name); return MNMT_ERR_DIM; }
  if (it->second != numel) {
    set_err("parameter '%s': numel %lld, expected %lld", name, (long long)numel, (long long)it->second);
    return MNMT_ERR_DIM;
  }
  m->host[name].assign(host, host + numel);
  return MNMT_OK;
}

mnmt_status mnmt_model_quantize(mnmt_model* m) {
  if (!m) { set_err("NULL model"); return MNMT_ERR_ARG; }
  if (m->failed) { set_err("handle is fail-stopped"); return MNMT_ERR_STATE; }
  if (m->quantized) { set_err("already quantized"); return MNMT_ERR_STATE; }
  std::string missing;
  for (const auto& kv : m->manifest)
    if (!m->host.count(kv.first)) missing += (missing.empty() ? "" : ", ") + kv.first;
  if (!missing.empty()) {
    if (missing.size() > 900) missing = missing.substr(0, 900) + "...";
    set_err("missing parameters: %s", missing.c_str());
    return MNMT_ERR_STATE;
  }
  DeviceGuard g(m->dev);
  const auto& c = m->c;
  const int d = c.d_model, F = c.d_ffn, L = c.dec_layers;
  mnmt_status s;
  float* tmp = nullptr;
  int64_t tmp_n = std::max<int64_t>((int64_t)c.vocab * d, (int64_t)F * d);
  if ((s = dmalloc(m->allocs, reinterpret_cast<void**>(&tmp), tmp_n * 4)) != MNMT_OK) return s;
  auto done = [&](mnmt_status st) { return fail(m, st); };
  // tied embedding: fp32 for gathers (A2/A5), int8 codes for the output layer (A9)
  if ((s = upload_vec(m, &m->E, "emb.E")) != MNMT_OK) return done(s);
  if ((s = dalloc(m->allocs, &m->qE, (int64_t)c.vocab * d)) != MNMT_OK) return done(s);
  if (launch_quantize(m->E, (int64_t)c.vocab * d, c.clip, m->qE, m->st) != cudaSuccess) {
    set_err("quantize launch failed");
    return done(MNMT_ERR_CUDA);
  }
  if (!make_tmap_i8(&m->tmE, m->qE, c.vocab, d)) { set_err("tensor map (E) failed"); return done(MNMT_ERR_CUDA); }
  if (c.out_bias && (s = upload_vec(m, &m->out_b, "out.b")) != MNMT_OK) return done(s);
  if ((s = dalloc(m->allocs, &m->PE, (int64_t)m->max_pos * d)) != MNMT_OK) return done(s);
  if (launch_pe_table(m->PE, m->max_pos, d, m->st) != cudaSuccess) { set_err("PE launch failed"); return done(MNMT_ERR_CUDA); }
  m->enc.resize(c.enc_layers);
  m->dec.resize(L);
  for (int l = 0; l < c.enc_layers; ++l) {
    const std::string p = "enc." + std::to_string(l) + ".";
    EncLayer& E = m->enc[l];
    if ((s = prep_lin(m, E.qkv, {p + "self.q", p + "self.k", p + "self.v"}, d, d, tmp)) != MNMT_OK) return done(s);
    if ((s = prep_lin(m, E.o, {p + "self.o"}, d, d, tmp)) != MNMT_OK) return done(s);
    if ((s = prep_lin(m, E.f1, {p + "ffn.1"}, F, d, tmp)) != MNMT_OK) return done(s);
    if ((s = prep_lin(m, E.f2, {p + "ffn.2"}, d, F, tmp)) != MNMT_OK) return done(s);
    if ((s = upload_vec(m, &E.ln1g, p + "ln1.g")) != MNMT_OK) return done(s);
    if ((s = upload_vec(m, &E.ln1b, p + "ln1.b")) != MNMT_OK) return done(s);
    if ((s = upload_vec(m, &E.ln2g, p + "ln2.g")) != MNMT_OK) return done(s);
    if ((s = upload_vec(m, &E.ln2b, p + "ln2.b")) != MNMT_OK) return done(s);
  }
  std::vector<std::string> kv_names;
  for (int l = 0; l < L; ++l) {
    const std::string p = "dec." + std::to_string(l) + ".";
    DecLayer& D = m->dec[l];
    if (c.decoder == 1) {
      if (c.aan_ffn_depth >= 1 && (s = prep_lin(m, D.a1, {p + "aan.ffn.1"}, d, d, tmp)) != MNMT_OK) return done(s);
      if (c.aan_ffn_depth >= 2 && (s = prep_lin(m, D.a2, {p + "aan.ffn.2"}, d, d, tmp)) != MNMT_OK) return done(s);
      if (c.aan_gate) {
        if ((s = prep_lin(m, D.gi, {p + "aan.gate.i"}, d, d, tmp)) != MNMT_OK) return done(s);
        if ((s = prep_lin(m, D.gf, {p + "aan.gate.f"}, d, d, tmp)) != MNMT_OK) return done(s);
      }
    } else {
      if ((s = prep_lin(m, D.qkv, {p + "self.q", p + "self.k", p + "self.v"}, d, d, tmp)) != MNMT_OK) return done(s);
      if ((s = prep_lin(m, D.o, {p + "self.o"}, d, d, tmp)) != MNMT_OK) return done(s);
    }
    if ((s = prep_lin(m, D.sq, {p + "src.q"}, d, d, tmp)) != MNMT_OK) return done(s);
    if ((s = prep_lin(m, D.so, {p + "src.o"}, d, d, tmp)) != MNMT_OK) return done(s);
    if ((s = prep_lin(m, D.f1, {p + "ffn.1"}, F, d, tmp)) != MNMT_OK) return done(s);
    if ((s = prep_lin(m, D.f2, {p + "ffn.2"}, d, F, tmp)) != MNMT_OK) return done(s);
    for (int i = 0; i < 3; ++i) {
      const std::string ln = p + "ln" + std::to_string(i + 1);
      if ((s = upload_vec(m, &D.ln[i][0], ln + ".g")) != MNMT_OK) return done(s);
      if ((s = upload_vec(m, &D.ln[i][1], ln + ".b")) != MNMT_OK) return done(s);
    }
    kv_names.push_back(p + "src.k");
    kv_names.push_back(p + "src.v");
  }
  if ((s = prep_lin(m, m->kv_all, kv_names, d, d, tmp)) != MNMT_OK) return done(s);
  if (cudaStreamSynchronize(m->st) != cudaSuccess) {
    set_err("weight preparation failed: %s", cudaGetErrorString(cudaGetLastError()));
    return done(MNMT_ERR_CUDA);
  }
  cudaFree(tmp);
  m->allocs.erase(std::remove(m->allocs.begin(), m->allocs.end(), (void*)tmp), m->allocs.end());
  m->host.clear();
  m->quantized = true;
  return MNMT_OK;
}

mnmt_status mnmt_batch_by_words(const int32_t* len, int32_t n, int32_t budget, int32_t* order,
                                int32_t* off, int32_t* n_batches) {
  if (budget < 1) { set_err("word_budget < 1"); return MNMT_ERR_ARG; }
  if (n < 0) { set_err("n < 0"); return MNMT_ERR_ARG; }
  if (!off || !n_batches || (n > 0 && (!len || !order))) { set_err("NULL argument"); return MNMT_ERR_ARG; }
  std::vector<int32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return len[a] < len[b]; });
  int nb = 0;
  int64_t words = 0;
  off[0] = 0;
  for (int i = 0; i < n; ++i) {
    order[i] = idx[i];
    words += len[idx[i]];
    if (words >= budget) {
      off[++nb] = i + 1;
      words = 0;
    }
  }
  if (n > 0 && off[nb] != n) off[++nb] = n;
  *n_batches = nb;
  return MNMT_OK;
}

// Teacher forcing (test hook of the parity protocol): sentence i runs T_i steps with the
// given input ids; dumps as in mnmt.h.
struct Forced {
  const int32_t* ids;
  const int64_t* off;
  uint32_t dump_mask;
  void* dump_host;
};

static mnmt_status translate_impl(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off,
                                  int32_t n, const int32_t* max_len, int32_t budget,
                                  bool sorted_batches, int32_t* out_ids, int64_t out_cap,
                                  int32_t* out_len, uint32_t flags, void* cuda_stream,
                                  int32_t beam = 0, float* out_score = nullptr,
                                  int32_t* n_hyp = nullptr, const Forced* fz = nullptr) {
  if (!m) { set_err("NULL model"); return MNMT_ERR_ARG; }
  const bool forced = fz != nullptr;   // teacher forcing: max_len[i] = T_i, no EOS stop
  mnmt_status s;
  if ((s = check_inputs(m, src_off, n, max_len)) != MNMT_OK) return s;
  if (beam < 0 || beam > TOPK_MAX || beam > m->c.vocab) {
    set_err("beam must be in 1..%d (and <= vocab)", TOPK_MAX);
    return MNMT_ERR_ARG;
  }
  if (beam > 0 && n > 0 && (!out_score || !n_hyp)) { set_err("NULL beam outputs"); return MNMT_ERR_ARG; }
  const bool dev_io = (flags & MNMT_DEVICE_IO) != 0;
  const bool use_sl = (flags & MNMT_SHORTLIST) != 0;
  if (use_sl && (beam > 0 || !sorted_batches)) {
    set_err("MNMT_SHORTLIST: greedy mnmt_translate only");
    return MNMT_ERR_ARG;
  }
  if (use_sl && !m->sl_tables) { set_err("MNMT_SHORTLIST before mnmt_model_set_shortlist"); return MNMT_ERR_STATE; }
  const int64_t bm = std::max(1, beam);   // output slots per sentence
  int64_t O = 0, ntok = n > 0 ? src_off[n] : 0;
  for (int i = 0; i < n; ++i) O += max_len[i] * bm;
  if (out_cap < O) { set_err("out_cap %lld < sum(max_len) %lld", (long long)out_cap, (long long)O); return MNMT_ERR_CAPACITY; }
  if (n > 0 && (!src_ids && ntok > 0)) { set_err("NULL src_ids"); return MNMT_ERR_ARG; }
  if (n > 0 && (!out_len || (!out_ids && O > 0))) { set_err("NULL outputs"); return MNMT_ERR_ARG; }
  if (!dev_io && (s = check_ids_host(m, src_ids, ntok)) != MNMT_OK) return s;
  DeviceGuard g(m->dev);
  if ((s = begin_call(m, cuda_stream)) != MNMT_OK) return fail(m, s);
  std::vector<std::vector<int32_t>> rows;
  std::vector<int> lanes_of, wave_of;
  // shortlist scopes (F2): word-budget batches (sentences batch-major), waves of batches, and
  // every sentence's group (batch index within its wave)
  std::vector<int32_t> bb_sents, bb_off(1, 0), wave_off(1, 0), grp_of(std::max(n, 1), 0);
  if (sorted_batches) {
    if (budget < 1) { set_err("word_budget < 1"); return MNMT_ERR_ARG; }
    std::vector<int32_t> L(n), order(std::max(n, 1)), off(n + 2);
    for (int i = 0; i < n; ++i) L[i] = (int32_t)(src_off[i + 1] - src_off[i]);
    int32_t nb = 0;
    mnmt_batch_by_words(L.data(), n, budget, order.data(), off.data(), &nb);
    // Waves: consecutive batches decoded together while the wave holds at most
    // max_concurrent_rows sentences; each wave's sentences are dealt round-robin (in
    // length order) to the decoder lanes, which run concurrently.  Scheduling only:
    // rows are independent, so the ids do not depend on it.
    const int P = std::max(1, m->n_lanes);
    for (int b = 0; b < nb;) {
      int e = b + 1;
      // with a shortlist a wave holds at most SL_MAX_GROUPS batches (bits of a column mask)
      if (m->max_concurrent_rows > 0)
        while (e < nb && off[e + 1] - off[b] <= m->max_concurrent_rows &&
               (!use_sl || e - b < SL_MAX_GROUPS))
          ++e;
      for (int bb = b; bb < e; ++bb) {
        for (int i = off[bb]; i < off[bb + 1]; ++i) {
          bb_sents.push_back(order[i]);
          grp_of[order[i]] = bb - b;
        }
        bb_off.push_back((int32_t)bb_sents.size());
      }
      wave_off.push_back(e);
      if (m->lane_tiers > 0 && P > 1) {
        // contiguous length tiers: lane li takes the li-th of P equal shares of
        // sum_i S_i^p (p = lane_tiers / 10) in length order, so the long-sentence tail runs on
        // its own lane beside the bulk instead of stretching every lane's step count
        const double pw = m->lane_tiers / 10.0;
        double tot = 0.0;
        for (int i = off[b]; i < off[e]; ++i) tot += std::pow((double)L[order[i]], pw);
        double acc = 0.0;
        int li = 0;
        std::vector<int32_t> part;
        for (int i = off[b]; i < off[e]; ++i) {
          part.push_back(order[i]);
          acc += std::pow((double)L[order[i]], pw);
          if (li < P - 1 && acc >= tot * (li + 1) / P) {
            rows.push_back(std::move(part));
            lanes_of.push_back(li++);
            part.clear();
          }
        }
        if (!part.empty()) {
          rows.push_back(std::move(part));
          lanes_of.push_back(li);
        }
      } else {
        for (int li = 0; li < P; ++li) {
          std::vector<int32_t> part;
          for (int i = off[b] + li; i < off[e]; i += P) part.push_back(order[i]);
          if (!part.empty()) {
            rows.push_back(std::move(part));
            lanes_of.push_back(li);
          }
        }
      }
      wave_of.resize(rows.size(), (int)wave_off.size() - 2);
      b = e;
    }
  } else {
    rows.emplace_back(n);
    std::iota(rows[0].begin(), rows[0].end(), 0);
    lanes_of.push_back(0);
  }
  Job job;
  plan_job(src_off, n, max_len, rows, lanes_of, (int)m->lanes.size(), job, use_sl ? &wave_of : nullptr);
  plan_rows(job, src_off, max_len, forced, forced ? fz->off : nullptr, m->c.d_model);
  std::vector<int32_t> rgrp;
  if (use_sl) {
    rgrp.assign(job.rows_total, 0);
    for (size_t bi = 0; bi < job.batches.size(); ++bi)
      for (size_t i = 0; i < job.batches[bi].rows.size(); ++i)
        rgrp[job.r0[bi] + i] = grp_of[job.batches[bi].rows[i]];
  }
  if ((s = jb_ensure(m, std::max<int64_t>(O, 1), std::max<int64_t>((int64_t)n * bm, 1),
                     std::max<int64_t>(ntok, 1), (int64_t)job.meta.size(), job.rows_total)) != MNMT_OK)
    return fail(m, s);
  m->beam = beam;
  m->sl_active = use_sl;
  struct BeamReset {
    mnmt_model* m;
    ~BeamReset() { m->beam = 0; m->sl_active = false; }
  } beam_reset{m};
  if ((s = ensure_lanes(m, job, 1)) != MNMT_OK) return fail(m, s);
  auto& w = m->jb;
  if ((s = upload_job(m, job)) != MNMT_OK) return fail(m, s);
  if (ntok > 0) {
    CK(cudaMemcpyAsync(w.src_ids, src_ids, ntok * 4,
                       dev_io ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, m->st));
    if (!dev_io) m->stats.h2d_bytes += ntok * 4;
  }
  if (dev_io && ntok > 0) {
    int32_t* bad = m->lanes[0].ws.ctrl + 32;
    CK(cudaMemsetAsync(bad, 0, 4, m->st));
    k_count_bad_ids<<<148, 256, 0, m->st>>>(w.src_ids, ntok, m->c.vocab, bad);
    int32_t hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
    if (hbad) { set_err("%d source ids out of range", hbad); return MNMT_ERR_VOCAB; }
  }
  if (use_sl && (s = sl_build_job(m, src_off, bb_sents, bb_off, wave_off, rgrp)) != MNMT_OK)
    return fail(m, s);
  CK(cudaMemsetAsync(w.out_len, 0, (size_t)n * bm * 4, m->st));
  if (beam > 0) {
    CK(cudaMemsetAsync(w.n_hyp, 0, (size_t)n * 4, m->st));
    CK(cudaMemsetAsync(w.out_score, 0, (size_t)n * bm * 4, m->st));
  }
  if (forced && O > 0) {
    CK(cudaMemcpyAsync(w.forced, fz->ids, O * 4, cudaMemcpyHostToDevice, m->st));
    m->stats.h2d_bytes += O * 4;
  }
  // device dumps of a teacher-forced run: written inside the step graphs, copied out below
  struct DumpReset {
    mnmt_model* m;
    std::vector<void*> bufs;
    ~DumpReset() {
      if (bufs.empty()) return;
      cudaStreamSynchronize(m->st);
      for (void* p : bufs) cudaFree(p);
      m->dump = DevDump();
      for (Lane& L : m->lanes) {   // graphs captured with dump kernels point at freed buffers
        for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
        L.graphs.clear();
      }
    }
  } dump_reset{m, {}};
  const int64_t dL = m->c.dec_layers, dd = m->c.d_model;
  const uint32_t dmask = forced ? fz->dump_mask : 0u;
  if (dmask & (MNMT_DUMP_LAYERS | MNMT_DUMP_DEC_OUT | MNMT_DUMP_OUT_CODES | MNMT_DUMP_MARGIN)) {
    auto dev = [&](void** p, int64_t bytes) -> mnmt_status {
      CK(cudaMalloc(p, std::max<int64_t>(bytes, 1)));
      dump_reset.bufs.push_back(*p);
      return MNMT_OK;
    };
    if (dmask & MNMT_DUMP_LAYERS) CKS(dev((void**)&m->dump.layers, O * dL * 3 * dd * 4));
    if (dmask & MNMT_DUMP_DEC_OUT) CKS(dev((void**)&m->dump.dec_out, O * dd * 4));
    if (dmask & MNMT_DUMP_OUT_CODES) CKS(dev((void**)&m->dump.out_codes, O * dd));
    if (dmask & MNMT_DUMP_MARGIN) {
      CKS(dev((void**)&m->dump.margin, O * 4));
      for (size_t li = 0; li < m->lanes.size(); ++li)   // the EPI_TOPK2 partials
        if (li < job.lane_B.size() && job.lane_B[li] > 0) CKS(beam_ensure(m, m->lanes[li]));
    }
    for (Lane& L : m->lanes) {   // capture fresh graphs with the dump kernels
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
  }
  if ((s = run_job(m, job, forced)) != MNMT_OK) return fail(m, s);
  if (forced && fz->dump_host) {
    // sections in bit order (mnmt.h); the encoder sections exist only for one-batch calls
    char* p = static_cast<char*>(fz->dump_host);
    const Workspace& w0 = m->lanes[0].ws;
    if (dmask & (MNMT_DUMP_ENC_OUT | MNMT_DUMP_SRC_KV)) {
      char* enc_out = nullptr;
      char* src_kv = nullptr;
      if (dmask & MNMT_DUMP_ENC_OUT) { enc_out = p; p += ntok * dd * 4; }
      if (dmask & MNMT_DUMP_SRC_KV) { src_kv = p; p += dL * ntok * 2 * dd * 4; }
      // the encoder buffers still hold the (single) batch: sentences in input order, those
      // with T_i = 0 or S_i = 0 skipped
      int64_t t = 0;
      for (int i = 0; i < n; ++i) {
        const int64_t S = src_off[i + 1] - src_off[i];
        if (max_len[i] == 0 || S == 0) continue;
        if (enc_out) CK(cudaMemcpyAsync(enc_out + src_off[i] * dd * 4, w0.x + t * dd, S * dd * 4, cudaMemcpyDeviceToHost, m->st));
        if (src_kv)
          for (int64_t l = 0; l < dL; ++l)
            CK(cudaMemcpyAsync(src_kv + ((l * ntok + src_off[i]) * 2 * dd) * 4,
                               w0.kv + (l * w0.M_cap + t) * 2 * dd, S * 2 * dd * 4, cudaMemcpyDeviceToHost, m->st));
        t += S;
      }
    }
    if (m->dump.dec_out) { CK(cudaMemcpyAsync(p, m->dump.dec_out, O * dd * 4, cudaMemcpyDeviceToHost, m->st)); p += O * dd * 4; }
    if (m->dump.out_codes) { CK(cudaMemcpyAsync(p, m->dump.out_codes, O * dd, cudaMemcpyDeviceToHost, m->st)); p += O * dd; }
    if (m->dump.layers) { CK(cudaMemcpyAsync(p, m->dump.layers, O * dL * 3 * dd * 4, cudaMemcpyDeviceToHost, m->st)); p += O * dL * 3 * dd * 4; }
    if (m->dump.margin) { CK(cudaMemcpyAsync(p, m->dump.margin, O * 4, cudaMemcpyDeviceToHost, m->st)); p += O * 4; }
  }
  const cudaMemcpyKind dk = dev_io ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (O > 0) CK(cudaMemcpyAsync(out_ids, w.out_ids, O * 4, dk, m->st));
  if (n > 0) CK(cudaMemcpyAsync(out_len, w.out_len, (size_t)n * bm * 4, dk, m->st));
  if (beam > 0 && n > 0) {
    CK(cudaMemcpyAsync(out_score, w.out_score, (size_t)n * bm * 4, dk, m->st));
    CK(cudaMemcpyAsync(n_hyp, w.n_hyp, (size_t)n * 4, dk, m->st));
  }
  if (!dev_io) m->stats.d2h_bytes += O * 4 + (int64_t)n * bm * 4 + (beam > 0 ? (int64_t)n * (bm + 1) * 4 : 0);
  if ((s = end_call(m, cuda_stream)) != MNMT_OK) return fail(m, s);
  if (!dev_io) {
    int64_t words = 0;
    if (beam > 0) {
      for (int i = 0; i < n; ++i) words += n_hyp[i] > 0 ? out_len[(int64_t)i * bm] : 0;   // best hypothesis
    } else {
      for (int i = 0; i < n; ++i) words += out_len[i];
    }
    m->stats.target_words = words;
  }
  return MNMT_OK;
}

mnmt_status mnmt_decode(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off, int32_t n,
                        const int32_t* max_len, int32_t* out_ids, int64_t out_cap,
                        int32_t* out_len, void* cuda_stream) {
  return translate_impl(m, src_ids, src_off, n, max_len, 1, false, out_ids, out_cap, out_len, 0,
                        cuda_stream);
}

mnmt_status mnmt_translate(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off, int32_t n,
                           const int32_t* max_len, int32_t budget, int32_t* out_ids,
                           int64_t out_cap, int32_t* out_len, uint32_t flags, void* cuda_stream) {
  if (budget < 1) { set_err("word_budget < 1"); return MNMT_ERR_ARG; }
  return translate_impl(m, src_ids, src_off, n, max_len, budget, true, out_ids, out_cap, out_len,
                        flags, cuda_stream);
}

mnmt_status mnmt_model_set_shortlist(mnmt_model* m, const int32_t* freq, int32_t n_freq,
                                     const int32_t* lex, int32_t k_lex) {
  if (!m) { set_err("NULL model"); return MNMT_ERR_ARG; }
  if (m->failed) { set_err("handle failed earlier (fail-stop)"); return MNMT_ERR_STATE; }
  if (n_freq < 0 || k_lex < 0 || (n_freq > 0 && !freq) || (k_lex > 0 && !lex)) {
    set_err("bad shortlist tables (n_freq, k_lex >= 0; non-NULL when non-empty)");
    return MNMT_ERR_ARG;
  }
  DeviceGuard g(m->dev);
  CK(cudaDeviceSynchronize());
  if (m->sl_freq) cudaFree(m->sl_freq);
  if (m->sl_lex) cudaFree(m->sl_lex);
  m->sl_freq = m->sl_lex = nullptr;
  m->sl_tables = false;
  const int64_t nl = (int64_t)m->c.vocab * k_lex;
  CK(cudaMalloc(&m->sl_freq, std::max<int64_t>(n_freq, 1) * 4));
  CK(cudaMalloc(&m->sl_lex, std::max<int64_t>(nl, 1) * 4));
  if (n_freq > 0) CK(cudaMemcpy(m->sl_freq, freq, (size_t)n_freq * 4, cudaMemcpyHostToDevice));
  if (nl > 0) CK(cudaMemcpy(m->sl_lex, lex, (size_t)nl * 4, cudaMemcpyHostToDevice));
  m->sl_nfreq = n_freq;
  m->sl_k = k_lex;
  m->sl_tables = true;
  return MNMT_OK;
}

mnmt_status mnmt_beam_translate(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off,
                                int32_t n, const int32_t* max_len, int32_t word_budget,
                                int32_t beam, int32_t* out_ids, int64_t out_cap, int32_t* out_len,
                                float* out_score, int32_t* n_hyp, uint32_t flags,
                                void* cuda_stream) {
  if (word_budget < 1) { set_err("word_budget < 1"); return MNMT_ERR_ARG; }
  if (beam < 1) { set_err("beam < 1"); return MNMT_ERR_ARG; }
  return translate_impl(m, src_ids, src_off, n, max_len, word_budget, true, out_ids, out_cap,
                        out_len, flags, cuda_stream, beam, out_score, n_hyp);
}

}  // extern "C"

// ------------------------------------------------------------------ teacher forcing
static mnmt_status forced_impl(mnmt_model* m, const int32_t* src_ids, const int64_t* src_off,
                               int32_t n, const int32_t* forced_ids, const int64_t* forced_off,
                               int32_t word_budget, bool sorted_batches, int32_t* argmax_ids,
                               uint32_t dump_mask, void* dump_host, int64_t dump_cap,
                               void* cuda_stream) {
  if (!m) { set_err("NULL model"); return MNMT_ERR_ARG; }
  if (n < 0 || (n > 0 && (!src_off || !forced_off))) { set_err("bad arguments"); return MNMT_ERR_ARG; }
  if (n > 0 && forced_off[0] != 0) { set_err("forced_off[0] must be 0"); return MNMT_ERR_ARG; }
  std::vector<int32_t> ml(std::max(n, 1));
  for (int i = 0; i < n; ++i) {
    const int64_t T = forced_off[i + 1] - forced_off[i];
    if (T < 0) { set_err("forced_off not monotone"); return MNMT_ERR_ARG; }
    ml[i] = (int32_t)std::min<int64_t>(T, MNMT_MAX_SPAN + 1);   // > MAX_SPAN: rejected below
  }
  mnmt_status s;
  if ((s = check_inputs(m, src_off, n, ml.data())) != MNMT_OK) return s;
  const int64_t ntok = n > 0 ? src_off[n] : 0, O = n > 0 ? forced_off[n] : 0;
  if ((ntok > 0 && !src_ids) || (O > 0 && (!forced_ids || !argmax_ids))) { set_err("NULL arrays"); return MNMT_ERR_ARG; }
  if ((s = check_ids_host(m, forced_ids, O)) != MNMT_OK) return s;
  if (sorted_batches && (dump_mask & (MNMT_DUMP_ENC_OUT | MNMT_DUMP_SRC_KV))) {
    set_err("encoder dumps need one batch (mnmt_decode_forced)");
    return MNMT_ERR_ARG;
  }
  const int64_t d = m->c.d_model, L = m->c.dec_layers;
  int64_t need = 0;
  if (dump_mask & MNMT_DUMP_ENC_OUT) need += ntok * d * 4;
  if (dump_mask & MNMT_DUMP_SRC_KV) need += L * ntok * 2 * d * 4;
  if (dump_mask & MNMT_DUMP_DEC_OUT) need += O * d * 4;
  if (dump_mask & MNMT_DUMP_OUT_CODES) need += O * d;
  if (dump_mask & MNMT_DUMP_LAYERS) need += O * L * 3 * d * 4;
  if (dump_mask & MNMT_DUMP_MARGIN) need += O * 4;
  if (need > 0 && (!dump_host || dump_cap < need)) { set_err("dump_cap %lld < %lld", (long long)dump_cap, (long long)need); return MNMT_ERR_CAPACITY; }
  std::vector<int32_t> lens(std::max(n, 1));
  const Forced fz{forced_ids, forced_off, dump_mask, need > 0 ? dump_host : nullptr};
  return translate_impl(m, src_ids, src_off, n, ml.data(), sorted_batches ? word_budget : 1,
                        sorted_batches, argmax_ids, O, lens.data(), 0, cuda_stream, 0, nullptr,
                        nullptr, &fz);
}

extern "C" mnmt_status mnmt_decode_forced(mnmt_model* m, const int32_t* src_ids,
                                          const int64_t* src_off, int32_t n,
                                          const int32_t* forced_ids, const int64_t* forced_off,
                                          int32_t* argmax_ids, uint32_t dump_mask,
                                          void* dump_host, int64_t dump_cap, void* cuda_stream) {
  return forced_impl(m, src_ids, src_off, n, forced_ids, forced_off, 1, false, argmax_ids,
                     dump_mask, dump_host, dump_cap, cuda_stream);
}

extern "C" mnmt_status mnmt_translate_forced(mnmt_model* m, const int32_t* src_ids,
                                             const int64_t* src_off, int32_t n,
                                             const int32_t* forced_ids, const int64_t* forced_off,
                                             int32_t word_budget, int32_t* argmax_ids,
                                             uint32_t dump_mask, void* dump_host,
                                             int64_t dump_cap, void* cuda_stream) {
  if (word_budget < 1) { set_err("word_budget < 1"); return MNMT_ERR_ARG; }
  return forced_impl(m, src_ids, src_off, n, forced_ids, forced_off, word_budget, true,
                     argmax_ids, dump_mask, dump_host, dump_cap, cuda_stream);
}

extern "C" mnmt_status mnmt_model_set_option(mnmt_model* m, const char* name, int64_t value) {
  if (!m || !name) { set_err("NULL argument"); return MNMT_ERR_ARG; }
  if (std::string(name) == "max_concurrent_rows") {
    if (value < 0) { set_err("max_concurrent_rows < 0"); return MNMT_ERR_ARG; }
    m->max_concurrent_rows = value;
    return MNMT_OK;
  }
  if (std::string(name) == "pers_reserve") {
    if (value < 0 || value > 128) { set_err("pers_reserve must be in [0, 128]"); return MNMT_ERR_ARG; }
    m->pers_reserve = (int)value;
    for (Lane& L : m->lanes) {   // captured graphs encode the old grid sizes
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "beam_fused") {
    if (value < 0 || value > 1) { set_err("beam_fused must be 0 or 1"); return MNMT_ERR_ARG; }
    m->beam_fused = (int)value;
    for (Lane& L : m->lanes) {   // captured graphs encode the old kernel sequence
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "green_sms") {
    if (value < 0 || value > 136 || value % 8) { set_err("green_sms must be 0 or a multiple of 8 up to 136"); return MNMT_ERR_ARG; }
    if (value != m->green_sms) {
      DeviceGuard g(m->dev);
      cudaDeviceSynchronize();
      for (Lane& L : m->lanes) lane_streams_free(L);   // recreated (in the new partitions) on use
      const GreenApi& ga = green_api();
      for (auto& gc : m->green)
        if (gc) { ga.destroy(gc); gc = nullptr; }
      m->green_sms = (int)value;
    }
    return MNMT_OK;
  }
  if (std::string(name) == "lane_tiers") {
    if (value < 0 || value > 100) { set_err("lane_tiers must be in [0, 100]"); return MNMT_ERR_ARG; }
    m->lane_tiers = (int)value;
    return MNMT_OK;
  }
  if (std::string(name) == "smallm") {
    if (value < 0 || value > SMALLM_MAX) { set_err("smallm must be in [0, 32]"); return MNMT_ERR_ARG; }
    m->smallm = (int)value;
    for (Lane& L : m->lanes) {     // captured graphs encode the old kernel sequence
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "sab") {
    if (value < 0 || value > 128) { set_err("sab must be in [0, 128]"); return MNMT_ERR_ARG; }
    m->sab = (int)value;
    for (Lane& L : m->lanes) {     // captured graphs encode the old kernel sequence and row tiers
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "sab_out" || std::string(name) == "sab_kb") {
    if (value < 0 || value > 128) { set_err("%s must be in [0, 128]", name); return MNMT_ERR_ARG; }
    (std::string(name) == "sab_out" ? m->sab_out : m->sab_kb) = (int)value;
    for (Lane& L : m->lanes) {
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "sab_kmin") {
    if (value < 0 || value > (1 << 16)) { set_err("sab_kmin must be in [0, 65536]"); return MNMT_ERR_ARG; }
    m->sab_kmin = (int)value;
    for (Lane& L : m->lanes) {
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "smallm_kmax") {
    if (value < 0 || value > (1 << 16)) { set_err("smallm_kmax must be in [0, 65536]"); return MNMT_ERR_ARG; }
    m->smallm_kmax = (int)value;
    for (Lane& L : m->lanes) {
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "smallm_wmax") {
    if (value < 0) { set_err("smallm_wmax < 0"); return MNMT_ERR_ARG; }
    m->smallm_wmax = value;
    for (Lane& L : m->lanes) {
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "attn_f32") {
    if (value != 0 && value != 1) { set_err("attn_f32 must be 0 or 1"); return MNMT_ERR_ARG; }
    m->attn_f32 = (int)value;
    for (Lane& L : m->lanes) {
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "attn_tma_self") {
    if (value < 0 || value > 2) { set_err("attn_tma_self must be 0, 1 or 2"); return MNMT_ERR_ARG; }
    m->attn_tma_self = (int)value;
    for (Lane& L : m->lanes) {
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "split_k") {
    if (value != 0 && value != 1) { set_err("split_k must be 0 or 1"); return MNMT_ERR_ARG; }
    m->split_k = (int)value;
    for (Lane& L : m->lanes) {   // captured graphs encode the old grids
      for (auto& kv : L.graphs) cudaGraphExecDestroy(kv.second);
      L.graphs.clear();
    }
    return MNMT_OK;
  }
  if (std::string(name) == "steps_per_graph") {
    if (value < 1 || value > 63) { set_err("steps_per_graph must be in [1, 63]"); return MNMT_ERR_ARG; }
    m->steps_per_graph = (int)value;
    return MNMT_OK;
  }
  if (std::string(name) == "lanes") {
    if (value < 1 || value > 16) { set_err("lanes must be 1..16"); return MNMT_ERR_ARG; }
    DeviceGuard g(m->dev);
    cudaDeviceSynchronize();
    if ((int64_t)m->lanes.size() < value) m->lanes.resize(value);
    m->n_lanes = (int)value;
    return MNMT_OK;
  }
  set_err("unknown option '%s'", name);
  return MNMT_ERR_ARG;
}

extern "C" mnmt_status mnmt_get_stats(const mnmt_model* m, mnmt_stats* out) {
  if (!m || !out) { set_err("NULL argument"); return MNMT_ERR_ARG; }
  *out = m->stats;
  return MNMT_OK;
}

extern "C" void mnmt_model_destroy(mnmt_model* m) {
  if (!m) return;
  {
    DeviceGuard g(m->dev);
    cudaDeviceSynchronize();
    for (Lane& L : m->lanes) {
      lane_free(L);
      lane_streams_free(L);
    }
    jb_free(m);
    if (m->sl_freq) cudaFree(m->sl_freq);
    if (m->sl_lex) cudaFree(m->sl_lex);
    for (void* p : m->allocs) cudaFree(p);
    for (auto& gc : m->green)
      if (gc) green_api().destroy(gc);
    if (m->st) cudaStreamDestroy(m->st);
    if (m->ev_in) cudaEventDestroy(m->ev_in);
    if (m->ev_out) cudaEventDestroy(m->ev_out);
    if (m->ev_job) cudaEventDestroy(m->ev_job);
    cudaGetLastError();
  }
  delete m;
}
