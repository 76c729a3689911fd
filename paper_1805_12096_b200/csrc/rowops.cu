// rowops.cu — the HBM-bound kernels of the decode path (sm_100a).
//
// One warp per row (d <= 1024 held in registers as float4), fp64 reductions
// (R20), explicit single-rounding fp32 elementwise ops.
//   k_quantize     weight/activation quantization Q(x)            (A1)
//   k_pe_table     sinusoidal positions                           (R12)
//   k_embed_src    x = E[id]*sqrt(d) + PE[pos], Q(x)              (A2)
//   k_embed_tgt    decoder input + first AAN step                 (A5, A6)
//   k_ln           residual/gate combine + LayerNorm + Q + next-layer AAN step (A6-A8)
//   k_attn         attention, one warp per (row, head), fp64      (A3, A6', A7)
//   k_finish       argmax decode + EOS/max_len + stable live-row compaction (A9, A10)
#include <cstdio>
#include <utility>

#include "numerics.cuh"
#include "ptx.cuh"
#include "rowops.h"

namespace mnmt {

// ------------------------------------------------------------------ quantize
__global__ void k_quantize(const float* __restrict__ x, int64_t n, float clip, float sigma,
                           int8_t* __restrict__ out) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (int8_t)q8(x[i], clip, sigma);
}

cudaError_t launch_quantize(const float* x, int64_t n, float clip, int8_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_quantize<<<(int)blocks, 256, 0, st>>>(x, n, clip, 127.0f / clip, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ positions
__global__ void k_pe_table(float* pe, int max_pos, int d) {
  const int pos = blockIdx.x;
  for (int i = threadIdx.x; 2 * i < d; i += blockDim.x) {
    const double ang = (double)pos / pow(10000.0, (double)(2 * i) / (double)d);
    pe[(int64_t)pos * d + 2 * i] = (float)sin(ang);
    if (2 * i + 1 < d) pe[(int64_t)pos * d + 2 * i + 1] = (float)cos(ang);
  }
}

cudaError_t launch_pe_table(float* pe, int max_pos, int d, cudaStream_t st) {
  k_pe_table<<<max_pos, 128, 0, st>>>(pe, max_pos, d);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ helpers
template <int NV>
struct RowVec {
  float4 v[NV];
};

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ uint32_t q8x4(float4 v, float clip, float sigma) {
  return (uint32_t)(q8(v.x, clip, sigma) & 0xff) | ((uint32_t)(q8(v.y, clip, sigma) & 0xff) << 8) |
         ((uint32_t)(q8(v.z, clip, sigma) & 0xff) << 16) |
         ((uint32_t)(q8(v.w, clip, sigma) & 0xff) << 24);
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 mul4(float4 a, float4 b) {
  return make_float4(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y), __fmul_rn(a.z, b.z),
                     __fmul_rn(a.w, b.w));
}
__device__ __forceinline__ float4 muls4(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}
__device__ __forceinline__ float4 divs4(float4 a, float s) {
  return make_float4(__fdiv_rn(a.x, s), __fdiv_rn(a.y, s), __fdiv_rn(a.z, s), __fdiv_rn(a.w, s));
}

// AAN step on one float4 of a row: C <- fl(C + y); g = fl(C / t)  (R6, R7).
__device__ __forceinline__ void aan4(float* C, float4 y, float tf, const AanOut& o, int64_t off_row,
                                     int col) {
  float4 c = add4(ld4(C + col), y);
  st4(C + col, c);
  float4 g = divs4(c, tf);
  if (o.g_f) st4(o.g_f + off_row + col, g);
  if (o.g_q) *reinterpret_cast<uint32_t*>(o.g_q + off_row + col) = q8x4(g, o.clip, o.sigma);
}

// ------------------------------------------------------------------ source embedding (A2)
template <int NV>
__global__ void k_embed_src(const int32_t* __restrict__ ids, const int32_t* __restrict__ idx,
                            const int32_t* __restrict__ pos, int M, const float* __restrict__ E,
                            const float* __restrict__ PE, int d, float rsd, float clip,
                            float sigma, float* __restrict__ x, int8_t* __restrict__ xq) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  if (row >= M) return;
  const int lane = threadIdx.x & 31, d4 = d >> 2;
  const int id = ids[idx ? idx[row] : row], p = pos[row];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    if (c4 < d4) {
      float4 e = id >= 0 ? muls4(ld4(E + (int64_t)id * d + 4 * c4), rsd)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 v = add4(e, ld4(PE + (int64_t)p * d + 4 * c4));
      st4(x + (int64_t)row * d + 4 * c4, v);
      *reinterpret_cast<uint32_t*>(xq + (int64_t)row * d + 4 * c4) = q8x4(v, clip, sigma);
    }
  }
}

// ------------------------------------------------------------------ target embedding (A5)
template <int NV>
__global__ void k_embed_tgt(EmbedTgtArgs a) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  const int n_live = a.ctrl[0];
  if (r >= n_live) return;
  const int lane = threadIdx.x & 31, d = a.d, d4 = d >> 2;
  const int t = a.ctrl[1];
  const int orig = a.live[r];
  const int id = t == 1 ? -1 : a.prev_id[orig];   // zero embedding at t = 1 (R13)
  const float tf = (float)t;
  const int64_t off = (int64_t)r * d;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    if (c4 < d4) {
      float4 e = id >= 0 ? muls4(ld4(a.E + (int64_t)id * d + 4 * c4), a.rsd)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 v = add4(e, ld4(a.PE + (int64_t)(t - 1) * d + 4 * c4));
      st4(a.y + off + 4 * c4, v);
      *reinterpret_cast<uint32_t*>(a.yq + off + 4 * c4) = q8x4(v, a.aan.clip, a.aan.sigma);
      if (a.aan.C) aan4(a.aan.C + (int64_t)orig * d, v, tf, a.aan, off, 4 * c4);
    }
  }
}

// ------------------------------------------------------------------ residual + LayerNorm (+AAN)
template <int NV>
__global__ void k_ln(LnArgs a) {
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  if (r >= n_live) return;
  const int lane = threadIdx.x & 31, d = a.d, d4 = d >> 2;
  const int64_t off = (int64_t)r * d;
  float4 v[NV];
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    if (c4 < d4) {
      float4 x = ld4(a.x + off + 4 * c4);
      float4 z;
      if (a.gi) {
        // AAN gate (R8): i = sigmoid(gi), f = sigmoid(gf) from the gate GEMMs' logits;
        // z = fl(fl(i*y) + fl(f*a)), residual r = fl(y + z)
        float4 li = ld4(a.gi + off + 4 * c4), lf = ld4(a.gf + off + 4 * c4);
        float4 si = make_float4(sigmoid_f64(li.x), sigmoid_f64(li.y), sigmoid_f64(li.z), sigmoid_f64(li.w));
        float4 sf = make_float4(sigmoid_f64(lf.x), sigmoid_f64(lf.y), sigmoid_f64(lf.z), sigmoid_f64(lf.w));
        float4 iy = mul4(si, x);
        float4 fa = mul4(sf, ld4(a.delta + off + 4 * c4));
        z = add4(iy, fa);
      } else {
        z = ld4(a.delta + off + 4 * c4);
      }
      v[i] = add4(x, z);
      s = __dadd_rn(s, (double)v[i].x);
      s = __dadd_rn(s, (double)v[i].y);
      s = __dadd_rn(s, (double)v[i].z);
      s = __dadd_rn(s, (double)v[i].w);
    }
  }
  const double mu = __ddiv_rn(warp_sum_f64(s), (double)d);
  double q = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    if (c4 < d4) {
      double t0 = __dsub_rn((double)v[i].x, mu), t1 = __dsub_rn((double)v[i].y, mu);
      double t2 = __dsub_rn((double)v[i].z, mu), t3 = __dsub_rn((double)v[i].w, mu);
      q = __dadd_rn(q, __dmul_rn(t0, t0));
      q = __dadd_rn(q, __dmul_rn(t1, t1));
      q = __dadd_rn(q, __dmul_rn(t2, t2));
      q = __dadd_rn(q, __dmul_rn(t3, t3));
    }
  }
  const double var = __ddiv_rn(warp_sum_f64(q), (double)d);
  const double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, (double)a.eps)));
  const int orig = a.aan.C ? a.live[r] : 0;
  const float tf = a.aan.C ? (float)a.ctrl[1] : 1.0f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    if (c4 < d4) {
      const float4 g = ld4(a.gamma + 4 * c4), b = ld4(a.beta + 4 * c4);
      float4 o;
      o.x = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].x, mu), inv), (double)g.x), (double)b.x);
      o.y = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].y, mu), inv), (double)g.y), (double)b.y);
      o.z = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].z, mu), inv), (double)g.z), (double)b.z);
      o.w = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].w, mu), inv), (double)g.w), (double)b.w);
      if (a.out) st4(a.out + off + 4 * c4, o);
      if (a.out_q) *reinterpret_cast<uint32_t*>(a.out_q + off + 4 * c4) = q8x4(o, a.clip, a.sigma);
      if (a.aan.C) aan4(a.aan.C + (int64_t)orig * d, o, tf, a.aan, off, 4 * c4);
    }
  }
}

// ------------------------------------------------------------------ attention
// fp64 scores / softmax / context (R20).  Dot products run over the head dimension in
// order and context sums over positions in order (the plain definition); the max and the
// normaliser Z use warp tree reductions.
//
// warp_attend: one warp computes one (query row, head): lane j scores positions j, j+32,
// ...; probabilities go to a per-warp scratch in shared memory; lane c then sums column c
// over the positions in order (V loads issued 4 ahead).
__device__ __forceinline__ void warp_attend(const float* __restrict__ q, const float* k,
                                            const float* v, int64_t ld, int len, int dh,
                                            double* sc, float clip, float sigma,
                                            int8_t* out_q, float* out_f) {
  const int lane = threadIdx.x & 31;
  const double inv_sqrt = 1.0 / sqrt((double)dh);
  double mx = -INFINITY;
  for (int j = lane; j < len; j += 32) {
    const float* kr = k + (int64_t)j * ld;
    double dot = 0.0;
    for (int c = 0; c < dh; c += 4) {
      const float4 k4 = *reinterpret_cast<const float4*>(kr + c);
      const float4 q4 = *reinterpret_cast<const float4*>(q + c);
      dot = __dadd_rn(dot, __dmul_rn((double)q4.x, (double)k4.x));
      dot = __dadd_rn(dot, __dmul_rn((double)q4.y, (double)k4.y));
      dot = __dadd_rn(dot, __dmul_rn((double)q4.z, (double)k4.z));
      dot = __dadd_rn(dot, __dmul_rn((double)q4.w, (double)k4.w));
    }
    const double s = __dmul_rn(dot, inv_sqrt);
    sc[j] = s;
    mx = fmax(mx, s);
  }
  mx = warp_max_f64(mx);
  double z = 0.0;
  for (int j = lane; j < len; j += 32) {
    const double p = exp(__dsub_rn(sc[j], mx));
    sc[j] = p;
    z = __dadd_rn(z, p);
  }
  z = warp_sum_f64(z);
  __syncwarp();
  for (int c = lane; c < dh; c += 32) {
    double acc = 0.0;
    int j = 0;
    for (; j + 4 <= len; j += 4) {
      const float v0 = v[(int64_t)(j + 0) * ld + c], v1 = v[(int64_t)(j + 1) * ld + c];
      const float v2 = v[(int64_t)(j + 2) * ld + c], v3 = v[(int64_t)(j + 3) * ld + c];
      acc = __dadd_rn(acc, __dmul_rn(sc[j + 0], (double)v0));
      acc = __dadd_rn(acc, __dmul_rn(sc[j + 1], (double)v1));
      acc = __dadd_rn(acc, __dmul_rn(sc[j + 2], (double)v2));
      acc = __dadd_rn(acc, __dmul_rn(sc[j + 3], (double)v3));
    }
    for (; j < len; ++j) acc = __dadd_rn(acc, __dmul_rn(sc[j], (double)v[(int64_t)j * ld + c]));
    const float ctx = len > 0 ? (float)__ddiv_rn(acc, z) : 0.0f;
    out_q[c] = (int8_t)q8(ctx, clip, sigma);
    if (out_f) out_f[c] = ctx;
  }
  __syncwarp();
}

constexpr int ATTN_WARPS = 8;

// Decoder (SRC, SELF) and op-level (ENC) attention: one warp per (row, head).
__global__ void __launch_bounds__(ATTN_WARPS * 32) k_attn(AttnArgs a) {
  __shared__ double sc_all[ATTN_WARPS][MNMT_MAX_KV];
  pdl_wait();
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * ATTN_WARPS + wi;
  const int H = a.H, dh = a.dh;
  const int r = (int)(gw / H), h = (int)(gw - (int64_t)r * H);
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  if (r >= n_live) return;
  int start, len;
  const float* q = a.q + (int64_t)r * a.ldq + h * dh;
  if (a.mode == ATTN_ENC) {
    start = a.kv_start[r];
    len = a.kv_len[r];
  } else if (a.mode == ATTN_SRC) {
    const int orig = a.live[r];
    start = a.kv_start[orig];
    len = a.kv_len[orig];
  } else {  // ATTN_SELF: append this step's k, v (head slice), attend over positions 1..t
    const int orig = a.live[r];
    const int t = a.ctrl[1];
    start = orig * a.t_cap;
    len = t;
    float* dst = a.kv_w + (int64_t)(start + t - 1) * a.ldkv + h * dh;
    for (int c = lane; c < dh; c += 32) {
      dst[a.k_off + c] = q[a.d + c];        // k at qkv columns [d, 2d)
      dst[a.v_off + c] = q[2 * a.d + c];    // v at qkv columns [2d, 3d)
    }
    __syncwarp();
  }
  const float* K = a.kv + (int64_t)start * a.ldkv + a.k_off + h * dh;
  const float* V = a.kv + (int64_t)start * a.ldkv + a.v_off + h * dh;
  warp_attend(q, K, V, a.ldkv, len, dh, sc_all[wi], a.clip, a.sigma,
              a.out_q + (int64_t)r * a.d + h * dh, a.out_f ? a.out_f + (int64_t)r * a.d + h * dh : nullptr);
}

// Encoder self-attention: one CTA per (sentence, head).  The sentence's K and V head
// slices are staged in shared memory once (rows padded by 4 floats) and reused by all of
// its query rows (warp per query).  Sentences longer than ENC_STAGE_MAX read from L2/HBM.
constexpr int ENC_STAGE_MAX = 160;

__host__ __device__ inline size_t enc_attn_smem(int dh) {
  return (size_t)ATTN_WARPS * MNMT_MAX_KV * sizeof(double) +
         2 * (size_t)ENC_STAGE_MAX * (dh + 4) * sizeof(float);
}

__global__ void __launch_bounds__(ATTN_WARPS * 32) k_attn_enc(EncAttnArgs a) {
  extern __shared__ __align__(16) uint8_t enc_smem[];
  double* sc = reinterpret_cast<double*>(enc_smem);                       // [warps][MAX_KV]
  float* ks = reinterpret_cast<float*>(sc + (size_t)ATTN_WARPS * MNMT_MAX_KV);
  pdl_wait();
  const int s = blockIdx.x, h = blockIdx.y;
  const int dh = a.dh, d = a.d, ld3 = 3 * d, lds = dh + 4;
  const int start = a.sent_start[s], len = a.sent_len[s];
  const float* base = a.qkv + (int64_t)start * ld3 + h * dh;
  const float *K, *V;
  int64_t ldk;
  if (len <= ENC_STAGE_MAX) {
    float* vs = ks + (size_t)ENC_STAGE_MAX * lds;
    const int d4 = dh >> 2;
    for (int i = threadIdx.x; i < len * d4; i += blockDim.x) {
      const int j = i / d4, c4 = i - j * d4;
      *reinterpret_cast<float4*>(ks + j * lds + 4 * c4) =
          *reinterpret_cast<const float4*>(base + (int64_t)j * ld3 + d + 4 * c4);
      *reinterpret_cast<float4*>(vs + j * lds + 4 * c4) =
          *reinterpret_cast<const float4*>(base + (int64_t)j * ld3 + 2 * d + 4 * c4);
    }
    __syncthreads();
    K = ks;
    V = vs;
    ldk = lds;
  } else {
    K = base + d;
    V = base + 2 * d;
    ldk = ld3;
  }
  const int wi = threadIdx.x >> 5;
  for (int i = wi; i < len; i += ATTN_WARPS) {
    warp_attend(base + (int64_t)i * ld3, K, V, ldk, len, dh, sc + (size_t)wi * MNMT_MAX_KV,
                a.clip, a.sigma, a.out_q + (int64_t)(start + i) * d + h * dh, nullptr);
  }
}

// ------------------------------------------------------------------ finish + compaction
// Single CTA.  For each live row: id = argmax (lowest column on ties); write it
// unless it is EOS; row is done at EOS or t == max_len (R16).  Then the live
// list is compacted stably in place (new index <= old index, chunk by chunk).
constexpr int FIN_THREADS = 1024;

__global__ void __launch_bounds__(FIN_THREADS) k_finish(FinishArgs a) {
  __shared__ int32_t warp_cnt[FIN_THREADS / 32];
  __shared__ int32_t base_s;
  pdl_wait();
  const int n_live = a.ctrl[0];
  const int t = a.ctrl[1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n_live; c0 += FIN_THREADS) {
    const int r = c0 + tid;
    int keep = 0, orig = 0;
    if (r < n_live) {
      orig = a.live[r];
      const unsigned long long key = a.keys[r];
      a.keys[r] = 0ull;
      const int id = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
      const int ml = a.max_len[orig];
      int32_t* out = a.out_ids + a.out_off[orig];
      if (a.forced) {
        out[t - 1] = id;
        a.out_len[a.len_idx ? a.len_idx[orig] : orig] = t;
        if (t < ml) a.prev_id[orig] = a.forced[a.forced_off[orig] + t - 1];
        keep = t < ml;
      } else if (id == a.eos) {
        keep = 0;
      } else {
        out[t - 1] = id;
        a.out_len[a.len_idx ? a.len_idx[orig] : orig] = t;
        a.prev_id[orig] = id;
        keep = t < ml;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_cnt[w] = __popc(bal);
    __syncthreads();
    if (w == 0) {
      int v = warp_cnt[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      warp_cnt[lane] = v;  // inclusive prefix over warps
    }
    __syncthreads();
    const int before = (w ? warp_cnt[w - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
    const int base = base_s;
    if (keep) a.live[base + before] = orig;
    __syncthreads();
    if (tid == 0) base_s = base + warp_cnt[31];
    __syncthreads();
  }
  if (tid == 0) {
    a.ctrl[0] = base_s;
    a.ctrl[1] = t + 1;
  }
}

// ------------------------------------------------------------------ decode init
__global__ void k_decode_init(int32_t* ctrl, int32_t* live, int B, unsigned long long* keys) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    live[i] = i;
    keys[i] = 0ull;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctrl[0] = B;
    ctrl[1] = 1;
  }
}

// ------------------------------------------------------------------ launchers
static inline int nv_for(int d) { return (d / 4 + 31) / 32; }

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int ROW_WARPS = 4;

cudaError_t launch_embed_src(const int32_t* ids, const int32_t* idx, const int32_t* pos, int M,
                             const float* E, const float* PE, int d, float clip, float* x,
                             int8_t* xq, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  const float rsd = (float)sqrt((double)d);
  dim3 grid((M + ROW_WARPS - 1) / ROW_WARPS), block(32 * ROW_WARPS);
  switch (nv_for(d)) {
    case 1: return launch_pdl(k_embed_src<1>, grid, block, 0, st, ids, idx, pos, M, E, PE, d, rsd, clip, 127.0f / clip, x, xq);
    case 2: return launch_pdl(k_embed_src<2>, grid, block, 0, st, ids, idx, pos, M, E, PE, d, rsd, clip, 127.0f / clip, x, xq);
    case 4: return launch_pdl(k_embed_src<4>, grid, block, 0, st, ids, idx, pos, M, E, PE, d, rsd, clip, 127.0f / clip, x, xq);
    case 8: return launch_pdl(k_embed_src<8>, grid, block, 0, st, ids, idx, pos, M, E, PE, d, rsd, clip, 127.0f / clip, x, xq);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_embed_tgt(const EmbedTgtArgs& a, int rows, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  dim3 grid((rows + ROW_WARPS - 1) / ROW_WARPS), block(32 * ROW_WARPS);
  switch (nv_for(a.d)) {
    case 1: return launch_pdl(k_embed_tgt<1>, grid, block, 0, st, a);
    case 2: return launch_pdl(k_embed_tgt<2>, grid, block, 0, st, a);
    case 4: return launch_pdl(k_embed_tgt<4>, grid, block, 0, st, a);
    case 8: return launch_pdl(k_embed_tgt<8>, grid, block, 0, st, a);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_ln(const LnArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  dim3 grid((a.n + ROW_WARPS - 1) / ROW_WARPS), block(32 * ROW_WARPS);
  switch (nv_for(a.d)) {
    case 1: return launch_pdl(k_ln<1>, grid, block, 0, st, a);
    case 2: return launch_pdl(k_ln<2>, grid, block, 0, st, a);
    case 4: return launch_pdl(k_ln<4>, grid, block, 0, st, a);
    case 8: return launch_pdl(k_ln<8>, grid, block, 0, st, a);
  }
  return cudaErrorInvalidValue;
}

cudaError_t attn_init() {   // once per device
  static bool done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(k_attn_enc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)enc_attn_smem(64));
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

cudaError_t launch_attn(const AttnArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int64_t warps = (int64_t)a.n * a.H;
  return launch_pdl(k_attn, dim3((unsigned)((warps + ATTN_WARPS - 1) / ATTN_WARPS)),
                    dim3(ATTN_WARPS * 32), 0, st, a);
}

cudaError_t launch_attn_enc(const EncAttnArgs& a, cudaStream_t st) {
  if (a.n_sent <= 0) return cudaSuccess;
  return launch_pdl(k_attn_enc, dim3(a.n_sent, a.H), dim3(ATTN_WARPS * 32), enc_attn_smem(a.dh),
                    st, a);
}

cudaError_t launch_finish(const FinishArgs& a, cudaStream_t st) {
  return launch_pdl(k_finish, dim3(1), dim3(FIN_THREADS), 0, st, a);
}

cudaError_t launch_decode_init(int32_t* ctrl, int32_t* live, int B, unsigned long long* keys,
                               cudaStream_t st) {
  int blocks = (B + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148) blocks = 148;
  return launch_pdl(k_decode_init, dim3(blocks), dim3(256), 0, st, ctrl, live, B, keys);
}

// ------------------------------------------------------------------ op-level helpers (tests)
__global__ void k_aan_step_rows(float* C, const float* y, int n, int d, int t, AanOut o) {
  pdl_wait();
  const int64_t total = (int64_t)n * (d / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (d / 4);
    const int col = (int)(i - r * (d / 4)) * 4;
    aan4(C + r * d, ld4(y + r * d + col), (float)t, o, r * d, col);
  }
}

cudaError_t launch_aan_step_rows(float* C, const float* y, int n, int d, int t, const AanOut& o,
                                 cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_aan_step_rows<<<148, 256, 0, st>>>(C, y, n, d, t, o);
  return cudaGetLastError();
}

__global__ void k_argmax_ids(const unsigned long long* keys, int n, int32_t* ids) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    ids[i] = (int32_t)(0xFFFFFFFFu - (uint32_t)(keys[i] & 0xFFFFFFFFull));
}

cudaError_t launch_argmax_ids(const unsigned long long* keys, int n, int32_t* ids, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_argmax_ids<<<(n + 255) / 256, 256, 0, st>>>(keys, n, ids);
  return cudaGetLastError();
}

}  // namespace mnmt
