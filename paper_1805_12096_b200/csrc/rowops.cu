// rowops.cu — the HBM-bound kernels of the decode path (sm_100a).
//
// One warp per row (d <= 1024 held in registers as float4), fp64 reductions
// (R20), explicit single-rounding fp32 elementwise ops.
//   k_quantize     weight/activation quantization Q(x)            (A1)
//   k_pe_table     sinusoidal positions                           (R12)
//   k_embed_src    x = E[id]*sqrt(d) + PE[pos], Q(x)              (A2)
//   k_embed_tgt    decoder input + first AAN step                 (A5, A6)
//   k_ln           residual/gate combine + LayerNorm + Q + next-layer AAN step (A6-A8)
//   k_attn         decoder attention, one warp per (row, head), fp64 (A6', A7; op-level A3)
//   k_attn_enc_r   encoder self-attention, lane per query row, dh <= 32, <= 128 positions (A3)
//   k_attn_enc     encoder self-attention, warp per query row (other shapes)          (A3)
//   k_finish       argmax decode + EOS/max_len + stable live-row compaction (A9, A10)
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "numerics.cuh"
#include "ptx.cuh"
#include "rowops.h"
#include "rowdev.cuh"
#include "kernels.h"

namespace mnmt {
__constant__ int c_pdl_early = 1;
// Let the next kernel of the chain launch (and run its prologue) right away; its
// griddepcontrol.wait still waits for this grid to complete (env MNMT_PDL_EARLY=0 disables).
__device__ __forceinline__ void pdl_trigger_early() {
  if (c_pdl_early) pdl_launch_dependents();
}
}  // namespace mnmt

namespace mnmt {

// ------------------------------------------------------------------ quantize
__global__ void k_quantize(const float* __restrict__ x, int64_t n, float clip, float sigma,
                           int8_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger_early();
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

// ------------------------------------------------------------------ source embedding (A2)
template <int NV>
__global__ void k_embed_src(const int32_t* __restrict__ ids, const int32_t* __restrict__ idx,
                            const int32_t* __restrict__ pos, int M, const float* __restrict__ E,
                            const float* __restrict__ PE, int d, float rsd, float clip,
                            float sigma, float* __restrict__ x, int8_t* __restrict__ xq) {
  pdl_wait();
  pdl_trigger_early();
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

// ------------------------------------------------------------------ standalone row kernels
template <int NV>
__global__ void k_embed_tgt(EmbedTgtArgs a) {
  pdl_wait();
  pdl_trigger_early();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= a.n) return;
  embed_tgt_row<NV>(a, r);   // checks the live-row count itself
}

template <int NV>
__global__ void k_ln(LnArgs a) {
  pdl_wait();
  pdl_trigger_early();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= a.n) return;
  ln_row<NV>(a, r);   // checks the live-row count itself, after issuing its loads
}

// Wide rows (d = 256 W, W >= 2): W warps per row, 256-thread blocks (256 / (32 W) rows each).
template <int W, int NV = 2>
__global__ void __launch_bounds__(256) k_ln_split(LnArgs a) {
  __shared__ double red[256 / 32];
  // gamma / beta are model constants: loaded before the PDL wait (off the dependent chain)
  const int tid = threadIdx.x % (32 * W);
  float4 g[NV], b[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 4 * (tid + 32 * W * i);
    g[i] = ld4(a.gamma + c);
    b[i] = ld4(a.beta + c);
  }
  pdl_wait();
  pdl_trigger_early();
  constexpr int RPB = 256 / (32 * W);
  const int rb = threadIdx.x / (32 * W);
  const int r = blockIdx.x * RPB + rb;
  // rows past the static bound compute a clamped row (every thread reaches every barrier)
  // and store nothing
  ln_row_split<W, NV>(a, min(r, a.n - 1), red + rb * W, r < a.n, g, b);
}

constexpr int ATTN_WARPS = 8;

// Decoder (SRC, SELF) and op-level (ENC) attention: one warp per (row, head) (warp_attend).
// Dynamic smem: ATTN_WARPS x (span + 64) doubles.  (A variant that staged 32-position V tiles
// with cp.async measured no faster in the decode: its V tile halved the resident CTAs.)
__global__ void __launch_bounds__(ATTN_WARPS * 32) k_attn(AttnArgs a) {
  extern __shared__ double sc_dyn[];
  pdl_wait();
  pdl_trigger_early();
  const int wi = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * ATTN_WARPS + wi;
  const int r = (int)(gw / a.H), h = (int)(gw - (int64_t)r * a.H);
  if (r >= a.n) return;
  // independent loads first: live-row count and (src mode) the row's span in compact order
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  const int pst = a.live_start ? a.live_start[r] : 0, pln = a.live_start ? a.live_len[r] : 0;
  if (r >= n_live) return;
  attn_row_head(a, r, h, sc_dyn + (size_t)wi * (a.span + 64), a.span, pst, pln);
}

// Source attention with the head's K / V tiles moved by TMA (A7; fp32 K/V, d_h = 32 / 64).
// One warp per (row, head), AT_WARPS warps per CTA.  Lane 0 of a warp issues, before any
// arithmetic, the bulk tensor copies of the first 32 positions' K tile and V tile (d_h / 32
// boxes of 32 rows x 128 B each, 128-byte swizzle) into the warp's shared memory, completing
// on two mbarriers; later 32-position chunks are requested as soon as the previous chunk of the
// same buffer has been consumed.  No register holds a load in flight, so every warp keeps its
// whole tile in flight (the generic kernel's lanes wait on one K row / four V rows at a time:
// ncu, long-scoreboard stalls at 45 % occupancy).  The swizzle makes both access patterns
// conflict-free: lane = position reading 16-byte column groups of its row (scores), lane =
// column reading one row (context).  Arithmetic and order are warp_attend's (identical outputs).
constexpr int AT_WARPS = 4;       // warps per CTA of the one-warp TMA kernels (default)
constexpr int AT_WARPS_MAX = 8;
constexpr int AT_TILE = 32 * 128;   // one 32-position chunk of 32 floats (four 8-row boxes)
constexpr int AT_BOX = 8 * 128;     // one TMA box: 8 rows x 32 floats = one 128B-swizzle atom

__device__ __forceinline__ int at_swz(int j, int cc) {   // byte offset of (row j, float cc) in a box
  return j * 128 + ((((cc >> 2) ^ (j & 7)) << 4) | ((cc & 3) << 2));
}

// SHARE (default): the V chunks reuse the K buffer (the first requested as soon as the last K
// chunk's scores are formed, overlapping the normaliser): half the shared memory per warp, twice
// the resident warps (six CTAs of 4 warps per SM instead of three), one more round trip per warp.
// Measured: 630 rows d = 1024 33.8 -> 23.9 us (warm), big job 106.9 -> 102.0 ms.
// F32 (model option attn_f32, off by default -- it departs from R20's fp64 sums): the same kernel
// with fp32 dot products (FMA chains in order), expf, normaliser and context sums; measured 7-18 %
// faster per launch and 5.6 % on the big job (profiles/r2_attn_f32_measure.txt).
__device__ __forceinline__ float at_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double at_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float at_exp(float x) { return expf(x); }
__device__ __forceinline__ double at_exp(double x) { return exp(x); }
__device__ __forceinline__ float at_wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double at_wmax(double v) { return warp_max_f64(v); }
__device__ __forceinline__ float at_wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double at_wsum(double v) { return warp_sum_f64(v); }

template <int DH, bool SHARE, bool F32 = false>
__global__ void __launch_bounds__(AT_WARPS_MAX * 32) k_attn_tma(const __grid_constant__ CUtensorMap tm,
                                                            AttnArgs a) {
  constexpr int HB = DH / 32;                 // 32-column boxes per head slice
  constexpr int WB = (SHARE ? 1 : 2) * HB * AT_TILE;   // this warp's K (and V) tiles
  extern __shared__ uint8_t at_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(at_raw) + 1023) & ~uintptr_t(1023));
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* kt = base + wi * WB;
  uint8_t* vt = SHARE ? kt : kt + HB * AT_TILE;
  const int nw = blockDim.x >> 5;   // warps per CTA (AT_WARPS, or the launch's choice)
  double* sc = reinterpret_cast<double*>(base + nw * WB) + (size_t)wi * a.span;
  // per warp: two mbarriers, then its query (DH floats)
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + nw * WB + (size_t)nw * a.span * 8) +
                  (2 + DH / 2) * wi;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm);
  }
  __syncwarp();
  // Source attention (and the op-level ENC mode) reads only data written before the previous
  // kernel started: the source K / V cache (encoder), the live-row metadata and count (k_finish of
  // the previous step).  Its metadata loads and the first K tile's copy are issued BEFORE the PDL
  // wait, overlapping the previous kernel (the query projection); only the query needs the wait.
  // Self-attention appends this step's k, v (from the previous kernel) first, so it waits.
  const bool pre = a.mode != ATTN_SELF;
  const int64_t gw = (int64_t)blockIdx.x * nw + wi;
  const int r = (int)(gw / a.H), h = (int)(gw - (int64_t)r * a.H);
  int n_live = 0, start = 0, len = 0;
  auto meta = [&]() {
    n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
    if (a.mode == ATTN_ENC) {   // op level: row r's own span
      start = a.kv_start[r];
      len = a.kv_len[r];
    } else if (a.mode == ATTN_SELF) {   // cache rows of positions 1..t of this row's slot
      start = a.live[r] * a.t_cap;
      len = a.ctrl[1];
    } else if (a.live_start) {
      start = a.live_start[r];
      len = a.live_len[r];
    } else {
      const int orig = a.live[r];
      start = a.kv_start[orig];
      len = a.kv_len[orig];
    }
  };
  const int kc = a.k_off + h * DH, vc = a.v_off + h * DH;
  // chunk c0 (positions c0 .. c0 + 31 of the span): only the 8-row boxes holding positions < len
  auto load = [&](uint64_t* b, uint8_t* dst, int col, int c0) {
    const int row0 = (int)(a.kv_row0 + start);
    const int nb = min(4, (len - c0 + 7) >> 3);
    mbar_arrive_expect_tx(b, HB * nb * AT_BOX);
    for (int hb = 0; hb < HB; ++hb)
      for (int x = 0; x < nb; ++x)
        tma_load_2d(dst + hb * AT_TILE + x * AT_BOX, &tm, b, col + 32 * hb, row0 + c0 + 8 * x);
  };
  if (pre && r < a.n) {
    meta();
    if (lane == 0 && r < n_live && len > 0) {
      load(&bar[0], kt, kc, 0);
      if constexpr (!SHARE) load(&bar[1], vt, vc, 0);
    }
  }
  pdl_wait();
  pdl_trigger_early();
  if (r >= a.n) return;
  if (!pre) meta();
  if (r >= n_live) return;
  if (!pre) {
    // append this step's k, v (head slice, qkv columns [d, 2d) / [2d, 3d)) at position t, then
    // order the generic-proxy stores before the tensor copies that read them
    const float* qk = a.q + (int64_t)r * a.ldq + h * DH;
    float* dst = a.kv_w + (int64_t)(start + len - 1) * a.ldkv + h * DH;
    for (int c = lane; c < DH; c += 32) {
      dst[a.k_off + c] = qk[a.d + c];
      dst[a.v_off + c] = qk[2 * a.d + c];
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    if (lane == 0 && len > 0) {
      load(&bar[0], kt, kc, 0);
      if constexpr (!SHARE) load(&bar[1], vt, vc, 0);
    }
  }
  const float* q = a.q + (int64_t)r * a.ldq + h * DH;
  // the query staged in shared memory while the tiles are in flight (the dot loop then reads
  // only shared memory: one broadcast per float4)
  float4* qv = reinterpret_cast<float4*>(bar + 2);
  if (lane < DH / 4) qv[lane] = *reinterpret_cast<const float4*>(q + 4 * lane);
  __syncwarp();
  using T = typename std::conditional<F32, float, double>::type;
  const T inv_sqrt = (T)(1.0 / sqrt((double)DH));
  T mx = -INFINITY;
  uint32_t kph = 0, vph = 0;
  for (int c0 = 0; c0 < len; c0 += 32) {
    mbar_wait(&bar[0], kph);
    kph ^= 1;
    const int j = c0 + lane;
    if (j < len) {
      T dot = 0;
#pragma unroll
      for (int c = 0; c < DH; c += 4) {
        const float4 k4 = *reinterpret_cast<const float4*>(kt + (c >> 5) * AT_TILE + at_swz(lane, c & 31));
        const float4 q4 = qv[c >> 2];
        dot = at_fma((T)q4.x, (T)k4.x, dot);
        dot = at_fma((T)q4.y, (T)k4.y, dot);
        dot = at_fma((T)q4.z, (T)k4.z, dot);
        dot = at_fma((T)q4.w, (T)k4.w, dot);
      }
      const T s = dot * inv_sqrt;
      sc[j] = s;
      mx = mx > s ? mx : s;
    }
    __syncwarp();
    if (lane == 0 && c0 + 32 < len) load(&bar[0], kt, kc, c0 + 32);
  }
  // SHARE: every lane has read the K buffer (the __syncwarp above); the first V chunk goes into
  // it while the normaliser is formed
  if constexpr (SHARE)
    if (lane == 0 && len > 0) load(&bar[1], vt, vc, 0);
  mx = at_wmax(mx);
  T z = 0;
  for (int j = lane; j < len; j += 32) {
    const T p = at_exp((T)sc[j] - mx);
    sc[j] = p;
    z = z + p;
  }
  z = at_wsum(z);
  __syncwarp();
  T acc[HB];
#pragma unroll
  for (int i = 0; i < HB; ++i) acc[i] = 0;
  for (int c0 = 0; c0 < len; c0 += 32) {
    mbar_wait(&bar[1], vph);
    vph ^= 1;
    const int je = min(32, len - c0);
    for (int jj = 0; jj < je; ++jj) {
      const T p = (T)sc[c0 + jj];
#pragma unroll
      for (int i = 0; i < HB; ++i)
        acc[i] = at_fma(p, (T)*reinterpret_cast<const float*>(vt + i * AT_TILE + at_swz(jj, lane)), acc[i]);
    }
    __syncwarp();
    if (lane == 0 && c0 + 32 < len) load(&bar[1], vt, vc, c0 + 32);
  }
  int8_t* out = a.out_q + (int64_t)r * a.d + h * DH;
#pragma unroll
  for (int i = 0; i < HB; ++i) {
    const int c = lane + 32 * i;
    const float ctx = len > 0 ? (float)(acc[i] / z) : 0.0f;
    out[c] = (int8_t)q8(ctx, a.clip, a.sigma);
    if (a.out_f) a.out_f[(int64_t)r * a.d + h * DH + c] = ctx;
  }
}

inline size_t attn_tma_smem(int dh, int span, bool share, int nw = AT_WARPS) {
  return 1024 + (size_t)nw * ((share ? 1 : 2) * (dh / 32) * AT_TILE + (size_t)span * 8 + 16 +
                              (size_t)dh * 4);
}

// Long spans at small row counts, split over NS warps per (row, head) with TMA tiles (A7 and the
// greedy A6' self-attention; fp32 K/V, d_h = 32 / 64): one (row, head) per CTA of NS warps; warp
// w takes the 32-position chunks w, w + NS, ... and requests each chunk's K tile by bulk tensor
// copy (the first before any arithmetic), then its V tiles into the same buffer (the first while
// the row max is exchanged).  The row max is exchanged first; Z and
// the context are per-warp partial sums over the warp's positions in order, combined in warp
// order (R25) -- k_attn_split's arithmetic and order, so outputs are identical to it.  In self
// mode warp 0 appends this step's k, v before the copies are issued.
template <int NS, int DH>
__global__ void __launch_bounds__(NS * 32) k_attn_split_tma(const __grid_constant__ CUtensorMap tm,
                                                            AttnArgs a) {
  constexpr int HB = DH / 32, WB = HB * AT_TILE;   // one buffer: V chunks reuse the K buffer
  extern __shared__ uint8_t ast_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ast_raw) + 1023) & ~uintptr_t(1023));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* kt = base + w * WB;
  uint8_t* vt = kt;
  double* sc = reinterpret_cast<double*>(base + NS * WB);   // [span]
  double* pm = sc + a.span;                                 // [NS]
  double* pacc = pm + NS;                                   // [NS][DH]
  uint64_t* bar = reinterpret_cast<uint64_t*>(pacc + NS * DH) + (2 + DH / 2) * w;   // + query
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm);
  }
  __syncwarp();
  // source mode: metadata and the warp's first K tile before the PDL wait (written before the
  // previous kernel started, as in k_attn_tma); self mode appends k, v after the wait first
  const bool pre = a.mode != ATTN_SELF;
  const int r = (int)(blockIdx.x / a.H), h = (int)(blockIdx.x - (int64_t)r * a.H);
  int n_live = 0, start = 0, len = 0;
  auto meta = [&]() {
    n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
    if (a.mode == ATTN_SELF) {
      start = a.live[r] * a.t_cap;
      len = a.ctrl[1];
    } else if (a.live_start) {
      start = a.live_start[r];
      len = a.live_len[r];
    } else {
      const int orig = a.live[r];
      start = a.kv_start[orig];
      len = a.kv_len[orig];
    }
  };
  const int kc = a.k_off + h * DH, vc = a.v_off + h * DH;
  // chunk c0 (positions c0 .. c0 + 31 of the span): only the 8-row boxes holding positions < len
  auto load = [&](uint64_t* b, uint8_t* dst, int col, int c0) {
    const int row0 = (int)(a.kv_row0 + start);
    const int nb = min(4, (len - c0 + 7) >> 3);
    mbar_arrive_expect_tx(b, HB * nb * AT_BOX);
    for (int hb = 0; hb < HB; ++hb)
      for (int x = 0; x < nb; ++x)
        tma_load_2d(dst + hb * AT_TILE + x * AT_BOX, &tm, b, col + 32 * hb, row0 + c0 + 8 * x);
  };
  if (pre) {
    meta();
    if (lane == 0 && r < n_live && w * 32 < len) load(&bar[0], kt, kc, w * 32);
  }
  pdl_wait();
  pdl_trigger_early();
  if (!pre) meta();
  if (r >= n_live) return;   // uniform over the CTA
  const float* q = a.q + (int64_t)r * a.ldq + h * DH;
  if (!pre) {
    if (w == 0) {
      float* dst = a.kv_w + (int64_t)(start + len - 1) * a.ldkv + h * DH;
      for (int c = lane; c < DH; c += 32) {
        dst[a.k_off + c] = q[a.d + c];
        dst[a.v_off + c] = q[2 * a.d + c];
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
    if (lane == 0 && w * 32 < len) load(&bar[0], kt, kc, w * 32);
  }
  // the query staged in shared memory while the tiles are in flight (broadcast reads)
  float4* qv = reinterpret_cast<float4*>(bar + 2);
  if (lane < DH / 4) qv[lane] = *reinterpret_cast<const float4*>(q + 4 * lane);
  __syncwarp();
  const double inv_sqrt = 1.0 / sqrt((double)DH);
  // ---- scores of this warp's chunks, local max
  double mx = -INFINITY;
  uint32_t kph = 0, vph = 0;
  for (int j0 = w * 32; j0 < len; j0 += NS * 32) {
    mbar_wait(&bar[0], kph);
    kph ^= 1;
    const int j = j0 + lane;
    if (j < len) {
      double dot = 0.0;
#pragma unroll
      for (int c = 0; c < DH; c += 4) {
        const float4 k4 = *reinterpret_cast<const float4*>(kt + (c >> 5) * AT_TILE + at_swz(lane, c & 31));
        const float4 q4 = qv[c >> 2];
        dot = __fma_rn((double)q4.x, (double)k4.x, dot);
        dot = __fma_rn((double)q4.y, (double)k4.y, dot);
        dot = __fma_rn((double)q4.z, (double)k4.z, dot);
        dot = __fma_rn((double)q4.w, (double)k4.w, dot);
      }
      const double sj = __dmul_rn(dot, inv_sqrt);
      sc[j] = sj;
      mx = fmax(mx, sj);
    }
    __syncwarp();
    if (lane == 0 && j0 + NS * 32 < len) load(&bar[0], kt, kc, j0 + NS * 32);
  }
  // every lane has read the buffer: the warp's first V chunk goes into it during the exchange
  if (lane == 0 && w * 32 < len) load(&bar[1], vt, vc, w * 32);
  mx = warp_max_f64(mx);
  if (lane == 0) pm[w] = mx;
  __syncthreads();
  double m = -INFINITY;
  for (int k = 0; k < NS; ++k) m = fmax(m, pm[k]);
  __syncthreads();   // pm is reused for the partial Z below
  // ---- p_j and the partial normaliser
  double z = 0.0;
  for (int j0 = w * 32; j0 < len; j0 += NS * 32) {
    const int j = j0 + lane;
    if (j < len) {
      const double p = exp(__dsub_rn(sc[j], m));
      sc[j] = p;
      z = __dadd_rn(z, p);
    }
  }
  z = warp_sum_f64(z);
  if (lane == 0) pm[w] = z;
  __syncwarp();
  // ---- partial context over this warp's positions, in order
  double acc[HB];
#pragma unroll
  for (int i = 0; i < HB; ++i) acc[i] = 0.0;
  for (int j0 = w * 32; j0 < len; j0 += NS * 32) {
    mbar_wait(&bar[1], vph);
    vph ^= 1;
    const int je = min(32, len - j0);
    for (int jj = 0; jj < je; ++jj) {
      const double p = sc[j0 + jj];
#pragma unroll
      for (int i = 0; i < HB; ++i)
        acc[i] = __fma_rn(p, (double)*reinterpret_cast<const float*>(vt + i * AT_TILE + at_swz(jj, lane)), acc[i]);
    }
    __syncwarp();
    if (lane == 0 && j0 + NS * 32 < len) load(&bar[1], vt, vc, j0 + NS * 32);
  }
#pragma unroll
  for (int i = 0; i < HB; ++i) pacc[w * DH + lane + 32 * i] = acc[i];
  __syncthreads();
  if (w != 0) return;
  double zt = 0.0;
  for (int k = 0; k < NS; ++k) zt = __dadd_rn(zt, pm[k]);
  int8_t* out = a.out_q + (int64_t)r * a.d + h * DH;
#pragma unroll
  for (int i = 0; i < HB; ++i) {
    const int c = lane + 32 * i;
    double s = 0.0;
    for (int k = 0; k < NS; ++k) s = __dadd_rn(s, pacc[k * DH + c]);
    const float ctx = len > 0 ? (float)__ddiv_rn(s, zt) : 0.0f;
    out[c] = (int8_t)q8(ctx, a.clip, a.sigma);
    if (a.out_f) a.out_f[(int64_t)r * a.d + h * DH + c] = ctx;
  }
}

inline size_t attn_split_tma_smem(int ns, int dh, int span) {
  return 1024 + (size_t)ns * (dh / 32) * AT_TILE + ((size_t)span + ns + (size_t)ns * dh) * 8 +
         (16 + (size_t)dh * 4) * ns;
}

// Source attention split over NS warps per (row, head) for long spans (A7): warp w of a group
// scores the 32-position chunks w, w + NS, ...; the row max is exchanged first, so every
// p_j = exp(s_j - max) is the value of the one-warp kernel; Z and the context are per-warp
// partial sums (positions in order inside a warp) combined in warp order (R25).
template <int NS, typename KT>
__global__ void __launch_bounds__(ATTN_WARPS * 32) k_attn_split(AttnArgs a) {
  constexpr int G = ATTN_WARPS / NS;                      // (row, head) groups per CTA
  extern __shared__ __align__(16) double as_smem[];
  const int span = a.span;
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = wi / NS, w = wi % NS;
  double* sc = as_smem + (size_t)g * span;                // [G][span] scores, then p
  double* pm = as_smem + (size_t)G * span;                // [G][NS] partial max, then partial Z
  double* pacc = pm + G * NS;                             // [G][NS][64] partial contexts
  double* qs = pacc + G * NS * 64;                        // [G][64] the group's query
  pdl_wait();
  pdl_trigger_early();
  const int64_t gw = (int64_t)blockIdx.x * G + g;
  const int r = (int)(gw / a.H), h = (int)(gw - (int64_t)r * a.H);
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  if ((int64_t)blockIdx.x * G / a.H >= n_live) return;    // uniform: no live row in this CTA
  const bool live = r < n_live;
  const int dh = a.dh;
  int start = 0, len = 0;
  if (live) {
    start = a.live_start ? a.live_start[r] : a.kv_start[a.live[r]];
    len = a.live_start ? a.live_len[r] : a.kv_len[a.live[r]];
  }
  const float* q = a.q + (int64_t)(live ? r : 0) * a.ldq + h * dh;
  const KT* kvb;
  if constexpr (sizeof(KT) == 2) kvb = a.kv16; else kvb = a.kv;   // bf16 source K/V (F3)
  const KT* K = kvb + (int64_t)start * a.ldkv + a.k_off + h * dh;
  const KT* V = kvb + (int64_t)start * a.ldkv + a.v_off + h * dh;
  double* qg = qs + g * 64;   // the query, converted once by warp 0 of the group
  if (w == 0)
    for (int c = lane; c < dh; c += 32) qg[c] = (double)q[c];
  __syncthreads();
  const double inv_sqrt = 1.0 / sqrt((double)dh);
  // ---- scores of this warp's chunks, local max
  double mx = -INFINITY;
  for (int j0 = w * 32; j0 < len; j0 += NS * 32) {
    const int j = j0 + lane;
    if (j < len) {
      const KT* kr = K + (int64_t)j * a.ldkv;
      double dot = 0.0;
      for (int c = 0; c < dh; c += 4) {
        double kk[4];
        ld4_f64(kr + c, kk);
        dot = __fma_rn(qg[c], kk[0], dot);
        dot = __fma_rn(qg[c + 1], kk[1], dot);
        dot = __fma_rn(qg[c + 2], kk[2], dot);
        dot = __fma_rn(qg[c + 3], kk[3], dot);
      }
      const double sj = __dmul_rn(dot, inv_sqrt);
      sc[j] = sj;
      mx = fmax(mx, sj);
    }
  }
  mx = warp_max_f64(mx);
  if (lane == 0) pm[g * NS + w] = mx;
  __syncthreads();
  double m = -INFINITY;
  for (int k = 0; k < NS; ++k) m = fmax(m, pm[g * NS + k]);
  __syncthreads();   // pm is reused for the partial Z below
  // ---- p_j and the partial normaliser
  double z = 0.0;
  for (int j0 = w * 32; j0 < len; j0 += NS * 32) {
    const int j = j0 + lane;
    if (j < len) {
      const double p = exp(__dsub_rn(sc[j], m));
      sc[j] = p;
      z = __dadd_rn(z, p);
    }
  }
  z = warp_sum_f64(z);
  if (lane == 0) pm[g * NS + w] = z;
  __syncwarp();
  // ---- partial context over this warp's positions, in order
  for (int c = lane; c < dh; c += 32) {
    double acc = 0.0;
    for (int j0 = w * 32; j0 < len; j0 += NS * 32) {
      const int je = min(j0 + 32, len);
      int j = j0;
      for (; j + 4 <= je; j += 4) {
        const double v0 = to_f64(V[(int64_t)(j + 0) * a.ldkv + c]);
        const double v1 = to_f64(V[(int64_t)(j + 1) * a.ldkv + c]);
        const double v2 = to_f64(V[(int64_t)(j + 2) * a.ldkv + c]);
        const double v3 = to_f64(V[(int64_t)(j + 3) * a.ldkv + c]);
        acc = __fma_rn(sc[j + 0], v0, acc);
        acc = __fma_rn(sc[j + 1], v1, acc);
        acc = __fma_rn(sc[j + 2], v2, acc);
        acc = __fma_rn(sc[j + 3], v3, acc);
      }
      for (; j < je; ++j) acc = __fma_rn(sc[j], to_f64(V[(int64_t)j * a.ldkv + c]), acc);
    }
    pacc[(g * NS + w) * 64 + c] = acc;
  }
  __syncthreads();
  if (w != 0 || !live) return;
  double zt = 0.0;
  for (int k = 0; k < NS; ++k) zt = __dadd_rn(zt, pm[g * NS + k]);
  int8_t* out = a.out_q + (int64_t)r * a.d + h * dh;
  for (int c = lane; c < dh; c += 32) {
    double acc = 0.0;
    for (int k = 0; k < NS; ++k) acc = __dadd_rn(acc, pacc[(g * NS + k) * 64 + c]);
    const float ctx = len > 0 ? (float)__ddiv_rn(acc, zt) : 0.0f;
    out[c] = (int8_t)q8(ctx, a.clip, a.sigma);
    if (a.out_f) a.out_f[(int64_t)r * a.d + h * dh + c] = ctx;
  }
}

inline size_t attn_split_smem(int ns, int span) {
  const int G = ATTN_WARPS / ns;
  return ((size_t)G * span + (size_t)G * ns + (size_t)G * ns * 64 + (size_t)G * 64) * sizeof(double);
}

constexpr int FIN_THREADS = 1024;

__global__ void __launch_bounds__(FIN_THREADS) k_finish(FinishArgs a) {
  __shared__ int32_t warp_cnt[32];
  __shared__ int32_t base_s;
  pdl_wait();
  pdl_trigger_early();
  finish_block(a, warp_cnt, base_s);
}

// Teacher-forced dumps (test hook): live row r of a step's activations -> row
// foff[live[r]] + t - 1, slot `slot` of `slots`.  One warp per row, 16-byte copies.
__global__ void k_dump_rows(DumpArgs a) {
  pdl_wait();
  pdl_trigger_early();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= a.n || r >= a.ctrl[0]) return;
  const int64_t row = a.foff[a.live[r]] + a.ctrl[1] - 1;
  const int64_t bytes = (int64_t)a.d * a.elem;
  const uint4* src = reinterpret_cast<const uint4*>(static_cast<const char*>(a.src) + r * bytes);
  uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(a.dst) + (row * a.slots + a.slot) * bytes);
  for (int64_t i = lane; i < bytes / 16; i += 32) dst[i] = src[i];
}

// Encoder self-attention: one CTA per (sentence, head).  The sentence's K and V head
// slices are staged in shared memory once (rows padded by 4 floats) and reused by all of
// its query rows (warp per query).  Sentences longer than ENC_STAGE_MAX read from L2/HBM.
constexpr int ENC_STAGE_MAX = 160;

// Launches are bucketed by sentence length (sent_order + s_max per bucket) so that shared
// memory, and with it the number of resident CTAs, follows the bucket's longest sentence.
__host__ __device__ inline size_t enc_attn_smem(int dh, int s_max, int warps) {
  const int staged = s_max < ENC_STAGE_MAX ? s_max : ENC_STAGE_MAX;
  return (size_t)warps * (s_max + 64) * sizeof(double) +
         2 * (size_t)staged * (dh + 2) * sizeof(double);
}
inline int enc_attn_warps(int s_max) { return s_max <= 8 ? 4 : ATTN_WARPS; }

__global__ void __launch_bounds__(ATTN_WARPS * 32) k_attn_enc(EncAttnArgs a) {
  extern __shared__ __align__(16) uint8_t enc_smem[];
  const int nw = blockDim.x >> 5;
  double* sc = reinterpret_cast<double*>(enc_smem);                       // [warps][s_max + 64]
  double* ks = sc + (size_t)nw * (a.s_max + 64);
  pdl_wait();
  pdl_trigger_early();
  const int s = a.sent_order ? a.sent_order[blockIdx.x] : (int)blockIdx.x, h = blockIdx.y;
  const int dh = a.dh, d = a.d, ld3 = 3 * d, lds = dh + 2;
  const int start = a.sent_start[s], len = a.sent_len[s];
  const int staged = a.s_max < ENC_STAGE_MAX ? a.s_max : ENC_STAGE_MAX;
  const float* base = a.qkv + (int64_t)start * ld3 + h * dh;
  const int wi = threadIdx.x >> 5;
  double* scw = sc + (size_t)wi * (a.s_max + 64);
  if (len <= staged) {
    // K and V head slices converted to fp64 once, reused by all of the sentence's queries
    double* vs = ks + (size_t)staged * lds;
    const int d4 = dh >> 2;
    for (int i = threadIdx.x; i < len * d4; i += blockDim.x) {
      const int j = i / d4, c4 = i - j * d4;
      const float4 k4 = *reinterpret_cast<const float4*>(base + (int64_t)j * ld3 + d + 4 * c4);
      const float4 v4 = *reinterpret_cast<const float4*>(base + (int64_t)j * ld3 + 2 * d + 4 * c4);
      double* kd = ks + j * lds + 4 * c4;
      double* vd = vs + j * lds + 4 * c4;
      kd[0] = k4.x; kd[1] = k4.y; kd[2] = k4.z; kd[3] = k4.w;
      vd[0] = v4.x; vd[1] = v4.y; vd[2] = v4.z; vd[3] = v4.w;
    }
    __syncthreads();
    for (int i = wi; i < len; i += nw)
      warp_attend<double>(base + (int64_t)i * ld3, ks, vs, lds, len, dh, scw, scw + a.s_max, a.clip,
                          a.sigma, a.out_q + (int64_t)(start + i) * d + h * dh, nullptr);
  } else {
    for (int i = wi; i < len; i += nw)
      warp_attend<float>(base + (int64_t)i * ld3, base + d, base + 2 * d, ld3, len, dh, scw,
                         scw + a.s_max, a.clip, a.sigma, a.out_q + (int64_t)(start + i) * d + h * dh,
                         nullptr);
  }
}

// Encoder self-attention, lane = query row (A3), dh <= 32: one CTA per (sentence, head) with
// ceil(len / 32) warps.  K and V head slices are staged once as fp64 in shared memory and read as
// warp-wide broadcasts (one wavefront feeds 32 lanes x 2 FMAs); each lane keeps its query in
// registers.  No score matrix is stored: pass A forms each row's max, pass B recomputes every
// dot (same order, same value) and accumulates p, Z and the context in one sweep.  The
// arithmetic and its order are the plain definition (R20): dot over c in order, scale, max,
// p_j = exp(s_j - max), Z = sum_j p_j in order, ctx_c = (sum_j p_j v_jc in order) / Z, with
// the product-accumulate steps fused (fp64 FMA, R24).
constexpr int ENC_R_MAX = 128;   // longest sentence this kernel stages (4 warps)
__host__ __device__ inline size_t enc_r_smem(int s_max) { return (size_t)2 * 32 * s_max * sizeof(double); }

__device__ __forceinline__ double dot32(const double (&q)[32], const double* kr, int dh) {
  double dot = 0.0;
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    if (c < dh) {
      const double2 k2 = *reinterpret_cast<const double2*>(kr + c);   // broadcast
      dot = __fma_rn(q[c], k2.x, dot);
      dot = __fma_rn(q[c + 1], k2.y, dot);
    }
  }
  return dot;
}

__global__ void __launch_bounds__(ENC_R_MAX) k_attn_enc_r(EncAttnArgs a) {
  extern __shared__ __align__(16) double es[];
  const int S = a.s_max, dh = a.dh, d = a.d, ld3 = 3 * d;
  double* Ks = es;                 // [S][32]
  double* Vs = Ks + S * 32;        // [S][32]
  pdl_wait();
  pdl_trigger_early();
  const int s = a.sent_order ? a.sent_order[blockIdx.x] : (int)blockIdx.x, h = blockIdx.y;
  const int start = a.sent_start[s], len = a.sent_len[s];
  const float* base = a.qkv + (int64_t)start * ld3 + h * dh;
  const int d4 = dh >> 2;
  for (int idx = threadIdx.x; idx < len * d4; idx += blockDim.x) {
    const int j = idx / d4, c4 = idx - j * d4;
    const float4 k4 = *reinterpret_cast<const float4*>(base + (int64_t)j * ld3 + d + 4 * c4);
    const float4 v4 = *reinterpret_cast<const float4*>(base + (int64_t)j * ld3 + 2 * d + 4 * c4);
    double* kd = Ks + j * 32 + 4 * c4;
    double* vd = Vs + j * 32 + 4 * c4;
    kd[0] = k4.x; kd[1] = k4.y; kd[2] = k4.z; kd[3] = k4.w;
    vd[0] = v4.x; vd[1] = v4.y; vd[2] = v4.z; vd[3] = v4.w;
  }
  __syncthreads();
  const int i = threadIdx.x;
  if (i >= len) return;            // no further block-wide barriers
  const float* qrow = base + (int64_t)i * ld3;
  double q[32];
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < dh) q4 = *reinterpret_cast<const float4*>(qrow + c);
    q[c] = q4.x; q[c + 1] = q4.y; q[c + 2] = q4.z; q[c + 3] = q4.w;
  }
  const double inv_sqrt = 1.0 / sqrt((double)dh);
  // ---- pass A: row max of the scaled scores
  double mx = -INFINITY;
#pragma unroll 4
  for (int j = 0; j < len; ++j) mx = fmax(mx, __dmul_rn(dot32(q, Ks + j * 32, dh), inv_sqrt));
  // ---- pass B: p_j, Z and the context, in order of j
  double z = 0.0, acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.0;
#pragma unroll 2
  for (int j = 0; j < len; ++j) {
    const double p = exp(__dsub_rn(__dmul_rn(dot32(q, Ks + j * 32, dh), inv_sqrt), mx));
    z = __dadd_rn(z, p);
    const double* vr = Vs + j * 32;
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      if (c < dh) {
        const double2 v2 = *reinterpret_cast<const double2*>(vr + c);   // broadcast
        acc[c] = __fma_rn(p, v2.x, acc[c]);
        acc[c + 1] = __fma_rn(p, v2.y, acc[c + 1]);
      }
    }
  }
  int8_t* orow = a.out_q + (int64_t)(start + i) * d + h * dh;
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    if (c < dh) {
      uint32_t w = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        w |= (uint32_t)(q8((float)__ddiv_rn(acc[c + u], z), a.clip, a.sigma) & 0xff) << (8 * u);
      *reinterpret_cast<uint32_t*>(orow + c) = w;
    }
  }
}

// Encoder self-attention for d_h = 64 (A3; small / base / big students), QW query rows per warp
// pass: one CTA per (sentence, head) stages the head's queries (transposed), keys and values once
// as fp64 in shared memory; a warp takes QW queries at a time, so every K / V element read from
// shared memory feeds QW FMAs (the one-query warp_attend is bound by shared-memory wavefronts:
// one K load per FMA).
//   pass 1  lane = position j (slots of 32): K row j's 64 elements in registers, 16 at a time,
//           QW dot chains over c in order (fused, R24), the QW queries' element c read as
//           broadcasts from QT[c][i0 .. i0 + QW);
//   pass 2  max (warp tree), p = exp(s - max), z per lane over its positions then the warp tree;
//   pass 3  lane = columns c, c + 32: context sums over positions in order, p read as
//           broadcasts from P[QW][SP].
// Every step and its order is warp_attend's (the generic encoder kernel), so outputs are
// bit-identical to it; the arithmetic is the plain definition of R20 / R24.
constexpr int ENC_MQ_DH = 64;
constexpr int ENC_MQ_SMAX = 100;   // longest sentence of a launch this kernel takes (smem)
__host__ __device__ inline int enc_mq_sp(int s_max) { return (s_max + 7) & ~7; }   // QT row length
// shared memory (doubles): K [S][65] (rounded to even), V [S][66], QT [64][SP], P per warp [QW][SP]
// (row paddings: the staging stores of consecutive positions j and the lane-j K reads hit
// distinct banks)
constexpr int ENC_MQ_LDV = ENC_MQ_DH + 2;
__host__ __device__ inline int enc_mq_kd(int s_max) { return (s_max * (ENC_MQ_DH + 1) + 1) & ~1; }
__host__ __device__ inline size_t enc_mq_smem(int s_max, int warps, int qw) {
  return ((size_t)enc_mq_kd(s_max) + (size_t)s_max * ENC_MQ_LDV + (size_t)ENC_MQ_DH * enc_mq_sp(s_max) +
          (size_t)warps * qw * enc_mq_sp(s_max)) * sizeof(double);
}

template <int QW>
__global__ void __launch_bounds__(ATTN_WARPS * 32) k_attn_enc_mq(EncAttnArgs a) {
  constexpr int DH = ENC_MQ_DH, LDK = DH + 1;   // K rows padded: lanes j hit distinct banks
  extern __shared__ __align__(16) double ems[];
  const int nw = blockDim.x >> 5, S = a.s_max, SP = enc_mq_sp(S);
  double* Ks = ems;                                 // [S][65]
  double* Vs = Ks + enc_mq_kd(S);                   // [S][66]
  double* QT = Vs + (size_t)S * ENC_MQ_LDV;         // [64][SP]
  pdl_wait();
  pdl_trigger_early();
  const int s = a.sent_order ? a.sent_order[blockIdx.x] : (int)blockIdx.x, h = blockIdx.y;
  const int d = a.d, ld3 = 3 * d;
  const int start = a.sent_start[s], len = a.sent_len[s];
  const float* base = a.qkv + (int64_t)start * ld3 + h * DH;
  for (int i = threadIdx.x; i < len * (DH / 4); i += blockDim.x) {
    const int j = i % len, c4 = (i / len) * 4;   // consecutive threads: consecutive positions
    const float* rj = base + (int64_t)j * ld3 + c4;
    const float4 q4 = *reinterpret_cast<const float4*>(rj);
    const float4 k4 = *reinterpret_cast<const float4*>(rj + d);
    const float4 v4 = *reinterpret_cast<const float4*>(rj + 2 * d);
    double* kd = Ks + j * LDK + c4;
    kd[0] = k4.x; kd[1] = k4.y; kd[2] = k4.z; kd[3] = k4.w;
    *reinterpret_cast<double2*>(Vs + j * ENC_MQ_LDV + c4) = make_double2(v4.x, v4.y);
    *reinterpret_cast<double2*>(Vs + j * ENC_MQ_LDV + c4 + 2) = make_double2(v4.z, v4.w);
    QT[(c4 + 0) * SP + j] = q4.x; QT[(c4 + 1) * SP + j] = q4.y;
    QT[(c4 + 2) * SP + j] = q4.z; QT[(c4 + 3) * SP + j] = q4.w;
  }
  for (int i = threadIdx.x; i < DH * (SP - len); i += blockDim.x)   // padding queries: zeros
    QT[(i / (SP - len)) * SP + len + i % (SP - len)] = 0.0;
  __syncthreads();
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* P = QT + (size_t)DH * SP + (size_t)wi * QW * SP;   // [QW][SP]
  const double inv_sqrt = 1.0 / sqrt((double)DH);
  for (int i0 = wi * QW; i0 < len; i0 += nw * QW) {
    const int nq = min(QW, len - i0);
    // ---- pass 1: scaled scores
    double mx[QW];
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) mx[qq] = -INFINITY;
    for (int j = lane; j < len; j += 32) {
      const double* kr = Ks + j * LDK;
      double dot[QW];
#pragma unroll
      for (int qq = 0; qq < QW; ++qq) dot[qq] = 0.0;
#pragma unroll 1
      for (int c0 = 0; c0 < DH; c0 += 16) {
        double kk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) kk[u] = kr[c0 + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double2* qp = reinterpret_cast<const double2*>(QT + (c0 + u) * SP + i0);
#pragma unroll
          for (int q2 = 0; q2 < QW / 2; ++q2) {
            const double2 qv = qp[q2];   // broadcast
            dot[2 * q2] = __fma_rn(qv.x, kk[u], dot[2 * q2]);
            dot[2 * q2 + 1] = __fma_rn(qv.y, kk[u], dot[2 * q2 + 1]);
          }
        }
      }
#pragma unroll
      for (int qq = 0; qq < QW; ++qq) {
        const double sv = __dmul_rn(dot[qq], inv_sqrt);
        P[qq * SP + j] = sv;
        mx[qq] = fmax(mx[qq], sv);
      }
    }
    // ---- pass 2: p = exp(s - max), z
    double z[QW];
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) {
      mx[qq] = warp_max_f64(mx[qq]);
      z[qq] = 0.0;
    }
    for (int j = lane; j < len; j += 32) {
#pragma unroll
      for (int qq = 0; qq < QW; ++qq) {
        const double p = exp(__dsub_rn(P[qq * SP + j], mx[qq]));
        P[qq * SP + j] = p;
        z[qq] = __dadd_rn(z[qq], p);
      }
    }
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) z[qq] = warp_sum_f64(z[qq]);
    __syncwarp();
    // ---- pass 3: context, positions in order
    double acc[QW][2];
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) acc[qq][0] = acc[qq][1] = 0.0;
#pragma unroll 2
    for (int j = 0; j < len; ++j) {
      const double v0 = Vs[j * ENC_MQ_LDV + lane], v1 = Vs[j * ENC_MQ_LDV + lane + 32];
#pragma unroll
      for (int qq = 0; qq < QW; ++qq) {
        const double p = P[qq * SP + j];   // broadcast
        acc[qq][0] = __fma_rn(p, v0, acc[qq][0]);
        acc[qq][1] = __fma_rn(p, v1, acc[qq][1]);
      }
    }
#pragma unroll
    for (int qq = 0; qq < QW; ++qq) {
      if (qq < nq) {
        int8_t* orow = a.out_q + (int64_t)(start + i0 + qq) * d + h * DH;
        orow[lane] = (int8_t)q8((float)__ddiv_rn(acc[qq][0], z[qq]), a.clip, a.sigma);
        orow[lane + 32] = (int8_t)q8((float)__ddiv_rn(acc[qq][1], z[qq]), a.clip, a.sigma);
      }
    }
    __syncwarp();   // P reused by the next pass
  }
}

// ------------------------------------------------------------------ decode init
__global__ void k_decode_init(int32_t* ctrl, int32_t* live, int B, unsigned long long* keys,
                              const int32_t* row_start, const int32_t* row_len,
                              int32_t* live_start, int32_t* live_len) {
  pdl_wait();
  pdl_trigger_early();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B; i += gridDim.x * blockDim.x) {
    live[i] = i;
    keys[i] = 0ull;
    if (live_start) {
      live_start[i] = row_start[i];
      live_len[i] = row_len[i];
    }
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
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
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

cudaError_t launch_embed_tgt(const EmbedTgtArgs& a_in, int rows, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  EmbedTgtArgs a = a_in;
  a.n = rows;
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
  // wide rows: W = d / 256 warps per row (env MNMT_LN_SPLIT=0: warp per row, A/B)
  static const bool split = [] {
    const char* e = getenv("MNMT_LN_SPLIT");
    return !(e && e[0] == '0');
  }();
  // one float4 per thread (W = d / 128 warps per row): measured 300.7 -> 283.3 us per big decoder
  // step at 1 row, 413 -> 391 at 64 rows, base-AAN job 50.0 -> 48.7 ms (profiles/r2_ln_nv1.txt);
  // env MNMT_LN_NV1=0: two float4 per thread (W = d / 256; A/B)
  static const bool nv1 = [] {
    const char* e = getenv("MNMT_LN_NV1");
    return !(e && e[0] == '0');
  }();
  // d = 256 (small students) over 2 warps per row: small-AAN decoder step 205 -> 180 us at 1 row,
  // job 37.3-37.6 -> 36.4 ms (profiles/r2_ln_split256.txt); env MNMT_LN_SPLIT256=0 disables (A/B)
  static const bool s256 = [] {
    const char* e = getenv("MNMT_LN_SPLIT256");
    return !(e && e[0] == '0');
  }();
  if (split && nv1 && (a.d == 512 || a.d == 1024 || (a.d == 256 && s256))) {
    const int W = a.d / 128, rpb = 256 / (32 * W);
    dim3 grid((a.n + rpb - 1) / rpb), block(256);
    return W == 2 ? launch_pdl(k_ln_split<2, 1>, grid, block, 0, st, a)
         : W == 4 ? launch_pdl(k_ln_split<4, 1>, grid, block, 0, st, a)
                  : launch_pdl(k_ln_split<8, 1>, grid, block, 0, st, a);
  }
  if (split && (a.d == 512 || a.d == 1024)) {
    const int W = a.d / 256, rpb = 256 / (32 * W);
    dim3 grid((a.n + rpb - 1) / rpb), block(256);
    return W == 2 ? launch_pdl(k_ln_split<2>, grid, block, 0, st, a)
                  : launch_pdl(k_ln_split<4>, grid, block, 0, st, a);
  }
  dim3 grid((a.n + ROW_WARPS - 1) / ROW_WARPS), block(32 * ROW_WARPS);
  switch (nv_for(a.d)) {
    case 1: return launch_pdl(k_ln<1>, grid, block, 0, st, a);
    case 2: return launch_pdl(k_ln<2>, grid, block, 0, st, a);
    case 4: return launch_pdl(k_ln<4>, grid, block, 0, st, a);
    case 8: return launch_pdl(k_ln<8>, grid, block, 0, st, a);
  }
  return cudaErrorInvalidValue;
}

// Optional (env MNMT_CARVEOUT=1): every row kernel prefers the maximum shared-memory
// carveout, the same L1/shared split as the GEMM kernels, so consecutive kernels of a
// decoder step never need an SM reconfiguration.
static cudaError_t set_carveouts() {
  const char* e = getenv("MNMT_CARVEOUT");
  if (!(e && e[0] == '1')) return cudaSuccess;
  const void* fns[] = {(const void*)k_quantize, (const void*)k_embed_src<1>, (const void*)k_embed_src<2>,
                       (const void*)k_embed_src<4>, (const void*)k_embed_src<8>,
                       (const void*)k_embed_tgt<1>, (const void*)k_embed_tgt<2>,
                       (const void*)k_embed_tgt<4>, (const void*)k_embed_tgt<8>,
                       (const void*)k_ln<1>, (const void*)k_ln<2>, (const void*)k_ln<4>, (const void*)k_ln<8>,
                       (const void*)k_attn, (const void*)k_attn_enc, (const void*)k_finish,
                       (const void*)k_decode_init};
  for (const void* f : fns) {
    cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (r != cudaSuccess) return r;
  }
  return cudaSuccess;
}

cudaError_t attn_init() {   // once per device
  static bool done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(k_attn_enc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)enc_attn_smem(64, MNMT_MAX_KV, ATTN_WARPS));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_enc_r, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)enc_r_smem(ENC_R_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_enc_mq<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)enc_mq_smem(ENC_MQ_SMAX, ATTN_WARPS, 4));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_enc_mq<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)enc_mq_smem(ENC_MQ_SMAX, ATTN_WARPS, 8));

  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ATTN_WARPS * (MNMT_MAX_KV + 64) * (int)sizeof(double));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_tma<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_tma_smem(64, MNMT_MAX_KV, false, AT_WARPS_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_tma<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_tma_smem(32, MNMT_MAX_KV, false, AT_WARPS_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_tma<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_tma_smem(64, MNMT_MAX_KV, true, AT_WARPS_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_tma<64, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_tma_smem(64, MNMT_MAX_KV, true, AT_WARPS_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_tma<32, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_tma_smem(32, MNMT_MAX_KV, true, AT_WARPS_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_tma<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_tma_smem(32, MNMT_MAX_KV, true, AT_WARPS_MAX));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split_tma<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_tma_smem(4, 64, MNMT_MAX_KV));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split_tma<2, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_tma_smem(2, 64, MNMT_MAX_KV));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split_tma<4, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_tma_smem(4, 32, MNMT_MAX_KV));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split_tma<2, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_tma_smem(2, 32, MNMT_MAX_KV));

  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split<2, bf16s>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_smem(2, MNMT_MAX_KV));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split<4, bf16s>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_smem(4, MNMT_MAX_KV));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split<2, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_smem(2, MNMT_MAX_KV));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_attn_split<4, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)attn_split_smem(4, MNMT_MAX_KV));
  if (e == cudaSuccess) e = set_carveouts();
  if (e == cudaSuccess) {
    const char* pe = getenv("MNMT_PDL_EARLY");
    const int v = (pe && pe[0] == '0') ? 0 : 1;
    e = cudaMemcpyToSymbol(c_pdl_early, &v, sizeof v);
  }
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

// Source K/V to bf16 (F3, R35): kv16 = RNE bf16 of kv, and kv itself rounded to the same value
// (so every reader of the fp32 copy sees the rounded keys / values).  L slices of n elements
// at stride `stride`.
__global__ void k_kv_bf16(float* __restrict__ kv, bf16s* __restrict__ kv16, int64_t n,
                          int64_t stride) {
  pdl_wait();
  pdl_trigger_early();
  const int64_t off = (int64_t)blockIdx.y * stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = __float_as_uint(kv[off + i]);
    const uint32_t r = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;   // RNE (finite inputs)
    kv16[off + i].u = (uint16_t)(r >> 16);
    kv[off + i] = __uint_as_float(r);
  }
}

cudaError_t launch_kv_bf16(float* kv, bf16s* kv16, int L, int64_t n, int64_t stride,
                           cudaStream_t st) {
  if (n <= 0 || L <= 0) return cudaSuccess;
  int64_t bx = (n + 255) / 256;
  if (bx > 148 * 4) bx = 148 * 4;
  return launch_pdl(k_kv_bf16, dim3((unsigned)bx, L), dim3(256), 0, st, kv, kv16, n, stride);
}

cudaError_t launch_attn(const AttnArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int64_t warps = (int64_t)a.n * a.H;
  AttnArgs b = a;
  if (b.span <= 0 || b.span > MNMT_MAX_KV) b.span = MNMT_MAX_KV;

  if (b.dh > 64 || (b.dh & 3)) return cudaErrorInvalidValue;
  // long source spans at small row counts: several warps per (row, head) (measured: -6 % per
  // step at 64 rows with 100-word sources; at 206 rows the extra warps cost more than they save)
  static const bool tma = [] {   // env MNMT_ATTN_TMA=0: the generic kernels (A/B)
    const char* e = getenv("MNMT_ATTN_TMA");
    return !(e && e[0] == '0');
  }();
  // self-attention through TMA tiles: AttnArgs::tma_self (model option "attn_tma_self": 0 off,
  // 1 the split kernel for long decodes at <= 128 rows, 2 also the one-warp kernel); A/B switch
  // MNMT_ATTN_TMA_SPLIT=0: long spans at <= 128 rows through the generic split kernel
  const int tma_self = b.tma_self;
  static const int tma_split = [] {
    const char* e = getenv("MNMT_ATTN_TMA_SPLIT");
    return e ? atoi(e) : 1;
  }();
  const bool use_tma = tma && b.tmap && !b.kv16 && !b.anc && (b.dh == 64 || b.dh == 32) &&
                       (b.mode != ATTN_SELF || tma_self > 0);
  const int ns = (b.mode == ATTN_SRC && b.n <= 128) ? (b.span >= 128 ? 4 : b.span >= 64 ? 2 : 1) : 1;
  // with TMA tiles the self-attention of long decodes splits the same way (R25)
  const int ns_t = !tma_split ? 1 : ((b.mode == ATTN_SRC || b.mode == ATTN_SELF) && b.n <= 128)
                       ? (b.span >= 128 ? 4 : b.span >= 64 ? 2 : 1) : 1;
  if (use_tma && (ns_t == 2 || ns_t == 4)) {
    const dim3 grid((unsigned)warps), block(ns_t * 32);
    const size_t smem = attn_split_tma_smem(ns_t, b.dh, b.span);
    if (ns_t == 4)
      return b.dh == 64 ? launch_pdl(k_attn_split_tma<4, 64>, grid, block, smem, st, *b.tmap, b)
                        : launch_pdl(k_attn_split_tma<4, 32>, grid, block, smem, st, *b.tmap, b);
    return b.dh == 64 ? launch_pdl(k_attn_split_tma<2, 64>, grid, block, smem, st, *b.tmap, b)
                      : launch_pdl(k_attn_split_tma<2, 32>, grid, block, smem, st, *b.tmap, b);
  }
  if (ns == 2 || ns == 4) {
    const int G = ATTN_WARPS / ns;
    const dim3 grid((unsigned)((warps + G - 1) / G)), block(ATTN_WARPS * 32);
    if (b.kv16)
      return ns == 2 ? launch_pdl(k_attn_split<2, bf16s>, grid, block, attn_split_smem(2, b.span), st, b)
                     : launch_pdl(k_attn_split<4, bf16s>, grid, block, attn_split_smem(4, b.span), st, b);
    return ns == 2 ? launch_pdl(k_attn_split<2, float>, grid, block, attn_split_smem(2, b.span), st, b)
                   : launch_pdl(k_attn_split<4, float>, grid, block, attn_split_smem(4, b.span), st, b);
  }
  if (use_tma && (b.mode != ATTN_SELF || tma_self == 2)) {
    static const bool share = [] {   // V reuses the K buffer (env MNMT_ATTN_SHARE=0: separate, A/B)
      const char* e = getenv("MNMT_ATTN_SHARE");
      return !(e && e[0] == '0');
    }();
    static const int atw = [] {   // warps per CTA (env MNMT_AT_WARPS = 2 / 4 / 8; A/B)
      const char* e = getenv("MNMT_AT_WARPS");
      const int v = e ? atoi(e) : AT_WARPS;
      return (v == 2 || v == 8) ? v : AT_WARPS;
    }();
    const dim3 grid((unsigned)((warps + atw - 1) / atw)), block(atw * 32);
    const size_t smem = attn_tma_smem(b.dh, b.span, share, atw);
    static const bool f32 = [] {   // env MNMT_ATTN_F32=1: the fp32 variant everywhere (A/B)
      const char* e = getenv("MNMT_ATTN_F32");
      return e && e[0] == '1';
    }();
    if (share && (f32 || b.f32))
      return b.dh == 64 ? launch_pdl(k_attn_tma<64, true, true>, grid, block, smem, st, *b.tmap, b)
                        : launch_pdl(k_attn_tma<32, true, true>, grid, block, smem, st, *b.tmap, b);
    if (share)
      return b.dh == 64 ? launch_pdl(k_attn_tma<64, true>, grid, block, smem, st, *b.tmap, b)
                        : launch_pdl(k_attn_tma<32, true>, grid, block, smem, st, *b.tmap, b);
    return b.dh == 64 ? launch_pdl(k_attn_tma<64, false>, grid, block, smem, st, *b.tmap, b)
                      : launch_pdl(k_attn_tma<32, false>, grid, block, smem, st, *b.tmap, b);
  }
  const dim3 grid((unsigned)((warps + ATTN_WARPS - 1) / ATTN_WARPS)), block(ATTN_WARPS * 32);
  const size_t smem = (size_t)ATTN_WARPS * (b.span + 64) * 8;
  return launch_pdl(k_attn, grid, block, smem, st, b);
}

cudaError_t launch_attn_enc(const EncAttnArgs& a, cudaStream_t st) { return launch_attn_enc_v(a, 0, st); }

cudaError_t launch_attn_enc_v(const EncAttnArgs& a, int variant, cudaStream_t st) {
  if (a.n_sent <= 0) return cudaSuccess;
  if (a.s_max < 1 || a.s_max > MNMT_MAX_KV) return cudaErrorInvalidValue;
  if (variant == 1) {   // forced: the generic warp-per-query kernel
    const int nw = enc_attn_warps(a.s_max);
    return launch_pdl(k_attn_enc, dim3(a.n_sent, a.H), dim3(nw * 32), enc_attn_smem(a.dh, a.s_max, nw),
                      st, a);
  }
  if (variant == 2 || variant == 3) {   // forced: the d_h = 64 multi-query kernel, QW = 4 / 8
    if (a.dh != ENC_MQ_DH || a.s_max > ENC_MQ_SMAX) return cudaErrorNotSupported;
    const int qw = variant == 2 ? 4 : 8;
    const int nw = std::min(ATTN_WARPS, (a.s_max + qw - 1) / qw);
    const size_t smem = enc_mq_smem(a.s_max, nw, qw);
    return qw == 4 ? launch_pdl(k_attn_enc_mq<4>, dim3(a.n_sent, a.H), dim3(nw * 32), smem, st, a)
                   : launch_pdl(k_attn_enc_mq<8>, dim3(a.n_sent, a.H), dim3(nw * 32), smem, st, a);
  }
  if (a.dh <= 32 && (a.dh & 3) == 0 && a.s_max <= ENC_R_MAX) {
    const dim3 grid(a.n_sent, a.H), block((a.s_max + 31) / 32 * 32);
    return launch_pdl(k_attn_enc_r, grid, block, enc_r_smem(a.s_max), st, a);
  }
  // d_h = 64: QW queries per warp pass (env MNMT_ENC_MQ = 0 / 4 / 8 selects; default 4), as many
  // warps as the bucket's longest sentence fills
  static const int mq = [] {
    const char* e = getenv("MNMT_ENC_MQ");
    return e ? atoi(e) : 4;
  }();
  if (a.dh == ENC_MQ_DH && a.s_max <= ENC_MQ_SMAX && (mq == 4 || mq == 8)) {
    const int nw = std::min(ATTN_WARPS, (a.s_max + mq - 1) / mq);
    const size_t smem = enc_mq_smem(a.s_max, nw, mq);
    return mq == 4 ? launch_pdl(k_attn_enc_mq<4>, dim3(a.n_sent, a.H), dim3(nw * 32), smem, st, a)
                   : launch_pdl(k_attn_enc_mq<8>, dim3(a.n_sent, a.H), dim3(nw * 32), smem, st, a);
  }
  const int nw = enc_attn_warps(a.s_max);
  return launch_pdl(k_attn_enc, dim3(a.n_sent, a.H), dim3(nw * 32), enc_attn_smem(a.dh, a.s_max, nw),
                    st, a);
}

cudaError_t launch_finish(const FinishArgs& a, cudaStream_t st) {
  return launch_pdl(k_finish, dim3(1), dim3(FIN_THREADS), 0, st, a);
}

// One warp per live row: each lane keeps the two largest values of its partials (a multiset:
// equal values both count), then a warp merge.
__global__ void k_top2_margin(const TopkPart* __restrict__ part, int part_ld, int n_part, int n,
                              const int32_t* ctrl, const int32_t* live, const int64_t* foff,
                              float* dst) {
  pdl_wait();
  pdl_trigger_early();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= n || r >= ctrl[0]) return;
  float a = -INFINITY, b = -INFINITY;   // a >= b
  for (int p = lane; p < n_part; p += 32) {
    const TopkPart& P = part[(int64_t)r * part_ld + p];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float v = P.v[i];
      if (v > a) { b = a; a = v; } else if (v > b) { b = v; }
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float oa = __shfl_xor_sync(0xffffffffu, a, o), ob = __shfl_xor_sync(0xffffffffu, b, o);
    const float hi = fmaxf(a, oa), lo = fminf(a, oa);
    b = fmaxf(lo, fmaxf(b, ob));
    a = hi;
  }
  if (lane == 0)
    dst[foff[live[r]] + ctrl[1] - 1] = b == -INFINITY ? INFINITY : (float)__dsub_rn((double)a, (double)b);
}

cudaError_t launch_top2_margin(const TopkPart* part, int part_ld, int n_part, int n,
                               const int32_t* ctrl, const int32_t* live, const int64_t* foff,
                               float* dst, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(k_top2_margin, dim3((n + ROW_WARPS - 1) / ROW_WARPS), dim3(32 * ROW_WARPS), 0, st,
                    part, part_ld, n_part, n, ctrl, live, foff, dst);
}

cudaError_t launch_dump_rows(const DumpArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  return launch_pdl(k_dump_rows, dim3((a.n + ROW_WARPS - 1) / ROW_WARPS), dim3(32 * ROW_WARPS), 0,
                    st, a);
}

cudaError_t launch_decode_init(int32_t* ctrl, int32_t* live, int B, unsigned long long* keys,
                               const int32_t* row_start, const int32_t* row_len,
                               int32_t* live_start, int32_t* live_len, cudaStream_t st) {
  int blocks = (B + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148) blocks = 148;
  return launch_pdl(k_decode_init, dim3(blocks), dim3(256), 0, st, ctrl, live, B, keys, row_start,
                    row_len, live_start, live_len);
}

// ------------------------------------------------------------------ op-level helpers (tests)
__global__ void k_aan_step_rows(float* C, const float* y, int n, int d, int t, AanOut o) {
  pdl_wait();
  pdl_trigger_early();
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
