// rowdev.cuh — device bodies of the HBM-bound row operations, shared by the standalone
// kernels (rowops.cu) and the fused GEMM epilogues.
#pragma once
#include <cstdint>

#include "numerics.cuh"
#include "ptx.cuh"
#include "rowops.h"

namespace mnmt {

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

// ------------------------------------------------------------------ target embedding (A5)
// r < a.n; the live-count check is taken together with the first loads (ctrl, live,
// prev_live are independent), so the row costs two dependent memory round trips.
template <int NV>
__device__ __forceinline__ void embed_tgt_row(const EmbedTgtArgs a, int r) {
  const int lane = threadIdx.x & 31, d = a.d, d4 = d >> 2;
  const int n_live = a.ctrl[0];
  const int t = a.ctrl[1];
  const int orig = a.live[r];
  const int pl = a.prev_live ? a.prev_live[r] : 0;
  if (r >= n_live) return;
  const int id = t == 1 ? -1 : (a.prev_live ? pl : a.prev_id[orig]);   // zero embedding at t = 1 (R13)
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
// r < a.n (static bound); rows at or beyond the live count are computed but not stored, so
// every load of the row is issued without waiting for the live-count read.
// vsm (optional, fused GEMM epilogue): the producing GEMM's output row staged in shared memory,
// read in place of delta (or of the f-gate logits gf in the gate form).
template <int NV>
__device__ __forceinline__ void ln_row(const LnArgs a, int r, const float* vsm = nullptr) {
  const int lane = threadIdx.x & 31, d = a.d, d4 = d >> 2;
  const int64_t off = (int64_t)r * d;
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  const int orig = a.aan.C ? a.live[r] : 0;
  const float tf = a.aan.C ? (float)a.ctrl[1] : 1.0f;
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
        float4 li = ld4(a.gi + off + 4 * c4), lf = vsm ? ld4(vsm + 4 * c4) : ld4(a.gf + off + 4 * c4);
        float4 si = make_float4(sigmoid_f64(li.x), sigmoid_f64(li.y), sigmoid_f64(li.z), sigmoid_f64(li.w));
        float4 sf = make_float4(sigmoid_f64(lf.x), sigmoid_f64(lf.y), sigmoid_f64(lf.z), sigmoid_f64(lf.w));
        float4 iy = mul4(si, x);
        float4 fa = mul4(sf, ld4(a.delta + off + 4 * c4));
        z = add4(iy, fa);
      } else {
        z = vsm ? ld4(vsm + 4 * c4) : ld4(a.delta + off + 4 * c4);
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
  if (r >= n_live) return;   // warp-uniform
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

// ------------------------------------------------------------------ residual + LayerNorm, W warps per row
// For wide rows (d = 256 W: 8 elements per thread, float4 columns lane + 32 w and that + d/8)
// the row is split over W warps so the fp64 sums run as short per-thread chains: per-thread
// partial sums (its elements in order), warp tree, then the W warp partials combined in warp
// order through shared memory (red: [rows per block][W] doubles).  Same arithmetic as ln_row
// (R20: fp64 sums in another order, one rounding to fp32).
// gamma / beta of the thread's NV float4 columns, loaded by the caller before the PDL wait
// (model constants), or null (loaded at the output stage)
template <int W, int NV = 2>
__device__ __forceinline__ void ln_row_split(const LnArgs a, int r, double* red, bool store,
                                             const float4* gpre = nullptr, const float4* bpre = nullptr) {
  // NV float4 columns per thread: d = 128 W NV (NV = 2: 8 elements per thread; NV = 1: 4)
  const int tid = threadIdx.x % (32 * W), wr = tid >> 5, lane = threadIdx.x & 31;
  const int d = a.d;
  const int64_t off = (int64_t)r * d;
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  const int orig = a.aan.C ? a.live[r] : 0;
  const float tf = a.aan.C ? (float)a.ctrl[1] : 1.0f;
  // the division by d is exact as a multiplication when d is a power of two
  const bool pow2 = (d & (d - 1)) == 0;
  const double rd = 1.0 / (double)d;
  float4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 4 * (tid + 32 * W * i);
    const float4 x = ld4(a.x + off + c);
    float4 z;
    if (a.gi) {
      // AAN gate (R8): r = fl(y + fl(fl(s(gi) * y) + fl(s(gf) * a)))
      const float4 li = ld4(a.gi + off + c), lf = ld4(a.gf + off + c);
      const float4 si = make_float4(sigmoid_f64(li.x), sigmoid_f64(li.y), sigmoid_f64(li.z), sigmoid_f64(li.w));
      const float4 sf = make_float4(sigmoid_f64(lf.x), sigmoid_f64(lf.y), sigmoid_f64(lf.z), sigmoid_f64(lf.w));
      z = add4(mul4(si, x), mul4(sf, ld4(a.delta + off + c)));
    } else {
      z = ld4(a.delta + off + c);
    }
    v[i] = add4(x, z);
  }
  double s = __dadd_rn(__dadd_rn(__dadd_rn((double)v[0].x, (double)v[0].y), (double)v[0].z), (double)v[0].w);
#pragma unroll
  for (int i = 1; i < NV; ++i)
    s = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s, (double)v[i].x), (double)v[i].y), (double)v[i].z), (double)v[i].w);
  s = warp_sum_f64(s);
  if (lane == 0) red[wr] = s;
  __syncthreads();
  double tot = red[0];
#pragma unroll
  for (int k = 1; k < W; ++k) tot = __dadd_rn(tot, red[k]);
  const double mu = pow2 ? __dmul_rn(tot, rd) : __ddiv_rn(tot, (double)d);
  double q = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double t0 = __dsub_rn((double)v[i].x, mu), t1 = __dsub_rn((double)v[i].y, mu);
    const double t2 = __dsub_rn((double)v[i].z, mu), t3 = __dsub_rn((double)v[i].w, mu);
    q = __dadd_rn(q, __dmul_rn(t0, t0));
    q = __dadd_rn(q, __dmul_rn(t1, t1));
    q = __dadd_rn(q, __dmul_rn(t2, t2));
    q = __dadd_rn(q, __dmul_rn(t3, t3));
  }
  q = warp_sum_f64(q);
  __syncthreads();   // every thread has read red[] (mean) before it is reused
  if (lane == 0) red[wr] = q;
  __syncthreads();
  double qt = red[0];
#pragma unroll
  for (int k = 1; k < W; ++k) qt = __dadd_rn(qt, red[k]);
  const double var = pow2 ? __dmul_rn(qt, rd) : __ddiv_rn(qt, (double)d);
  const double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, (double)a.eps)));
  if (!store || r >= n_live) return;   // after the last barrier
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 4 * (tid + 32 * W * i);
    const float4 g = gpre ? gpre[i] : ld4(a.gamma + c), b = bpre ? bpre[i] : ld4(a.beta + c);
    float4 o;
    o.x = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].x, mu), inv), (double)g.x), (double)b.x);
    o.y = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].y, mu), inv), (double)g.y), (double)b.y);
    o.z = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].z, mu), inv), (double)g.z), (double)b.z);
    o.w = (float)__dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn((double)v[i].w, mu), inv), (double)g.w), (double)b.w);
    if (a.out) st4(a.out + off + c, o);
    if (a.out_q) *reinterpret_cast<uint32_t*>(a.out_q + off + c) = q8x4(o, a.clip, a.sigma);
    if (a.aan.C) aan4(a.aan.C + (int64_t)orig * d, o, tf, a.aan, off, c);
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
__device__ __forceinline__ double to_f64(float x) { return (double)x; }
__device__ __forceinline__ double to_f64(double x) { return x; }
// bf16 storage of the source keys / values: the upper half of an fp32
__device__ __forceinline__ double to_f64(bf16s x) { return (double)__uint_as_float((uint32_t)x.u << 16); }
// four consecutive K elements (16-byte fp32 or 8-byte bf16 load), widened exactly to fp64
__device__ __forceinline__ void ld4_f64(const float* p, double (&o)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void ld4_f64(const bf16s* p, double (&o)[4]) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  o[0] = (double)__uint_as_float(v.x << 16);
  o[1] = (double)__uint_as_float(v.x & 0xffff0000u);
  o[2] = (double)__uint_as_float(v.y << 16);
  o[3] = (double)__uint_as_float(v.y & 0xffff0000u);
}

// KT = float / bf16s: K/V rows in global memory (each element converted once, when used);
// KT = double: K/V already converted (staged in shared memory by the caller).
// qd: per-warp scratch of dh doubles (the query converted once).
// IND: rows[j] is the row of position j (beam search: the self-attention cache rows of a
// hypothesis' ancestors, R29); otherwise position j is row j.
template <typename KT, bool IND = false>
__device__ __forceinline__ void warp_attend(const float* __restrict__ q, const KT* k, const KT* v,
                                            int64_t ld, int len, int dh, double* sc, double* qd,
                                            float clip, float sigma, int8_t* out_q, float* out_f,
                                            const int32_t* rows = nullptr) {
  const int lane = threadIdx.x & 31;
  // the query converted once into the warp's scratch: the dot loop then reads shared memory
  // (broadcasts) instead of global memory inside its fp64 chain
  for (int c = lane; c < dh; c += 32) qd[c] = (double)q[c];
  __syncwarp();
  const double inv_sqrt = 1.0 / sqrt((double)dh);
  double mx = -INFINITY;
  for (int j = lane; j < len; j += 32) {
    const KT* kr = k + (int64_t)(IND ? rows[j] : j) * ld;
    double dot = 0.0;
    for (int c = 0; c < dh; c += 4) {
      double kk[4], qq[4];
      if constexpr (sizeof(KT) <= 4) {
        ld4_f64(kr + c, kk);
        qq[0] = qd[c]; qq[1] = qd[c + 1]; qq[2] = qd[c + 2]; qq[3] = qd[c + 3];
      } else {
        const double2 a = *reinterpret_cast<const double2*>(kr + c);
        const double2 b = *reinterpret_cast<const double2*>(kr + c + 2);
        kk[0] = a.x; kk[1] = a.y; kk[2] = b.x; kk[3] = b.y;
        qq[0] = qd[c]; qq[1] = qd[c + 1]; qq[2] = qd[c + 2]; qq[3] = qd[c + 3];
      }
      dot = __fma_rn(qq[0], kk[0], dot);   // fused product-accumulate (R24)
      dot = __fma_rn(qq[1], kk[1], dot);
      dot = __fma_rn(qq[2], kk[2], dot);
      dot = __fma_rn(qq[3], kk[3], dot);
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
  if constexpr (IND) {
    for (int c = lane; c < dh; c += 32) {
      double acc = 0.0;
      for (int j = 0; j < len; ++j) acc = __fma_rn(sc[j], to_f64(v[(int64_t)rows[j] * ld + c]), acc);
      const float ctx = len > 0 ? (float)__ddiv_rn(acc, z) : 0.0f;
      out_q[c] = (int8_t)q8(ctx, clip, sigma);
      if (out_f) out_f[c] = ctx;
    }
    __syncwarp();
    return;
  }
  for (int c = lane; c < dh; c += 32) {
    double acc = 0.0;
    int j = 0;
    for (; j + 4 <= len; j += 4) {
      const double v0 = to_f64(v[(int64_t)(j + 0) * ld + c]), v1 = to_f64(v[(int64_t)(j + 1) * ld + c]);
      const double v2 = to_f64(v[(int64_t)(j + 2) * ld + c]), v3 = to_f64(v[(int64_t)(j + 3) * ld + c]);
      acc = __fma_rn(sc[j + 0], v0, acc);
      acc = __fma_rn(sc[j + 1], v1, acc);
      acc = __fma_rn(sc[j + 2], v2, acc);
      acc = __fma_rn(sc[j + 3], v3, acc);
    }
    for (; j < len; ++j) acc = __fma_rn(sc[j], to_f64(v[(int64_t)j * ld + c]), acc);
    const float ctx = len > 0 ? (float)__ddiv_rn(acc, z) : 0.0f;
    out_q[c] = (int8_t)q8(ctx, clip, sigma);
    if (out_f) out_f[c] = ctx;
  }
  __syncwarp();
}

// Attention of one (row, head) by one warp (SRC, SELF and ENC modes); sc = per-warp scratch
// of span + 64 doubles (scores, then the converted query).
// pre_start / pre_len: the row's source span when a.live_start is set (src mode; loaded by the
// caller together with the live-row count).
__device__ __forceinline__ void attn_row_head(const AttnArgs a, int r, int h, double* sc, int span,
                                              int pre_start = 0, int pre_len = 0) {
  const int lane = threadIdx.x & 31;
  const int dh = a.dh;
  int start, len;
  const float* q = a.q + (int64_t)r * a.ldq + h * dh;
  if (a.mode == ATTN_ENC) {
    start = a.kv_start[r];
    len = a.kv_len[r];
  } else if (a.mode == ATTN_SRC) {
    if (a.live_start) {
      start = pre_start;
      len = pre_len;
    } else {
      const int orig = a.live[r];
      start = a.kv_start[orig];
      len = a.kv_len[orig];
    }
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
    if (a.anc) {
      // beam search (R29): positions 0..t-2 live in the rows of the hypothesis' ancestors,
      // position t-1 in its own slot's row (written above)
      int32_t* rows = a.anc + (int64_t)orig * a.t_cap;
      if (lane == 0) rows[t - 1] = start + t - 1;
      __syncwarp();
      warp_attend<float, true>(q, a.kv + a.k_off + h * dh, a.kv + a.v_off + h * dh, a.ldkv, len, dh,
                               sc, sc + span, a.clip, a.sigma, a.out_q + (int64_t)r * a.d + h * dh,
                               a.out_f ? a.out_f + (int64_t)r * a.d + h * dh : nullptr, rows);
      return;
    }
    __syncwarp();
  }
  if (a.kv16) {   // bf16 source K/V (F3): same layout, half the bytes
    const bf16s* K16 = a.kv16 + (int64_t)start * a.ldkv + a.k_off + h * dh;
    const bf16s* V16 = a.kv16 + (int64_t)start * a.ldkv + a.v_off + h * dh;
    warp_attend<bf16s>(q, K16, V16, a.ldkv, len, dh, sc, sc + span, a.clip, a.sigma,
                       a.out_q + (int64_t)r * a.d + h * dh,
                       a.out_f ? a.out_f + (int64_t)r * a.d + h * dh : nullptr);
    return;
  }
  const float* K = a.kv + (int64_t)start * a.ldkv + a.k_off + h * dh;
  const float* V = a.kv + (int64_t)start * a.ldkv + a.v_off + h * dh;
  warp_attend<float>(q, K, V, a.ldkv, len, dh, sc, sc + span, a.clip, a.sigma,
              a.out_q + (int64_t)r * a.d + h * dh, a.out_f ? a.out_f + (int64_t)r * a.d + h * dh : nullptr);
}

// ------------------------------------------------------------------ finish + compaction
// Single CTA.  For each live row: id = argmax (lowest column on ties); write it
// unless it is EOS; row is done at EOS or t == max_len (R16).  Then the live
// list is compacted stably in place (new index <= old index, chunk by chunk).
// Block-wide (any blockDim multiple of 32, <= 1024).  warp_cnt: smem [32], base_s: smem.
__device__ __forceinline__ void finish_block(const FinishArgs a, int32_t* warp_cnt,
                                             int32_t& base_s) {
  const int n_live = a.ctrl[0];
  const int t = a.ctrl[1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nthreads = blockDim.x, nw = nthreads >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n_live; c0 += nthreads) {
    const int r = c0 + tid;
    int keep = 0, orig = 0, next_id = 0;
    if (r < n_live) {
      orig = a.live[r];
      const unsigned long long key = a.keys[r];
      a.keys[r] = 0ull;
      int id = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
      if (a.id_map) id = a.id_map[id];
      const int ml = a.max_len[orig];
      int32_t* out = a.out_ids + a.out_off[orig];
      if (a.forced) {
        out[t - 1] = id;
        a.out_len[a.len_idx ? a.len_idx[orig] : orig] = t;
        if (t < ml) next_id = a.prev_id[orig] = a.forced[a.forced_off[orig] + t - 1];
        keep = t < ml;
      } else if (id == a.eos) {
        keep = 0;
      } else {
        out[t - 1] = id;
        a.out_len[a.len_idx ? a.len_idx[orig] : orig] = t;
        a.prev_id[orig] = next_id = id;
        keep = t < ml;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_cnt[w] = __popc(bal);
    __syncthreads();
    if (w == 0) {
      int v = lane < nw ? warp_cnt[lane] : 0;
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
    if (keep) {
      const int nr = base + before;
      a.live[nr] = orig;
      if (a.prev_live) a.prev_live[nr] = next_id;
      if (a.live_start) {
        a.live_start[nr] = a.row_start[orig];
        a.live_len[nr] = a.row_len[orig];
      }
    }
    __syncthreads();
    if (tid == 0) base_s = base + warp_cnt[nw - 1];
    __syncthreads();
  }
  if (tid == 0) {
    a.ctrl[0] = base_s;
    a.ctrl[1] = t + 1;
  }
  __syncthreads();
}

}  // namespace mnmt
