// rowfused.cu — fused per-row decoder blocks for small live-row counts (see rowfused.h).
//
// One CTA per live row, one output column per thread (blockDim = max(d, 32 H) rounded to a
// warp).  A d x d projection is an exact s32 dot product per column: the row's activation codes
// sit in shared memory as packed int32 (read as warp-wide broadcasts) and each thread streams
// its column of the k4-major weight copy (coalesced across the warp) through IDP4A.  The
// dequantization, ReLU, quantizer, sigmoid, gate combine and residual are the same single-
// rounding operations as the GEMM epilogues and ln_row; the LayerNorm statistics are fp64 block
// sums (R20).
#include <cstdio>
#include <utility>

#include "kernels.h"
#include "numerics.cuh"
#include "ptx.cuh"
#include "rowdev.cuh"
#include "rowfused.h"

namespace mnmt {

namespace {

// exact s32 dot of the packed row codes (shared memory) with output column c of W4
__device__ __forceinline__ int32_t dot_k4(const int32_t* __restrict__ act4,
                                          const int32_t* __restrict__ W4, int d_in, int d_out,
                                          int c) {
  int32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  const int K4 = d_in >> 2;
  int k = 0;
  for (; k + 4 <= K4; k += 4) {
    const int32_t w0 = __ldg(W4 + (size_t)(k + 0) * d_out + c);
    const int32_t w1 = __ldg(W4 + (size_t)(k + 1) * d_out + c);
    const int32_t w2 = __ldg(W4 + (size_t)(k + 2) * d_out + c);
    const int32_t w3 = __ldg(W4 + (size_t)(k + 3) * d_out + c);
    a0 = __dp4a(act4[k + 0], w0, a0);
    a1 = __dp4a(act4[k + 1], w1, a1);
    a2 = __dp4a(act4[k + 2], w2, a2);
    a3 = __dp4a(act4[k + 3], w3, a3);
  }
  for (; k < K4; ++k) a0 = __dp4a(act4[k], __ldg(W4 + (size_t)k * d_out + c), a0);
  return (a0 + a1) + (a2 + a3);   // exact: |sum| <= 127^2 * 1024 < 2^31
}

__device__ __forceinline__ float lin_col(const RowLin& L, const int32_t* act4, int d, int c,
                                         float s) {
  return dequant(dot_k4(act4, L.W4, d, d, c), s, L.b ? __ldg(L.b + c) : 0.0f);
}

// fp64 sum over the block, the same value in every thread (warp trees, then warps in order)
__device__ __forceinline__ double block_sum_f64(double v, double* red) {
  v = warp_sum_f64(v);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();   // red may still be read by the previous call
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t = __dadd_rn(t, red[i]);
  return t;
}

// LayerNorm of the row (one column per thread, `on` = column exists): ln_row's arithmetic
__device__ __forceinline__ void row_ln(float v, bool on, int d, float eps, const float* gamma,
                                       const float* beta, int c, double* red, float* out,
                                       int8_t* out_q, float clip, float sigma) {
  const double mu = __ddiv_rn(block_sum_f64(on ? (double)v : 0.0, red), (double)d);
  const double t = on ? __dsub_rn((double)v, mu) : 0.0;
  const double var = __ddiv_rn(block_sum_f64(__dmul_rn(t, t), red), (double)d);
  const double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, (double)eps)));
  if (!on) return;
  const float o = (float)__dadd_rn(__dmul_rn(__dmul_rn(t, inv), (double)gamma[c]), (double)beta[c]);
  out[c] = o;
  out_q[c] = (int8_t)q8(o, clip, sigma);
}

}  // namespace

__global__ void k_repack_k4(const int8_t* __restrict__ W, int N, int K, int32_t* __restrict__ W4) {
  const int64_t total = (int64_t)N * (K / 4);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k4 = (int)(i / N), c = (int)(i - (int64_t)k4 * N);
    W4[i] = *reinterpret_cast<const int32_t*>(W + (int64_t)c * K + 4 * k4);
  }
}

// ---------------------------------------------------------------- AAN block (A6)
__global__ void __launch_bounds__(1024) k_aan_block(AanBlockArgs a) {
  extern __shared__ __align__(16) uint8_t rf_smem[];
  const int d = a.d, d4 = d >> 2;
  int32_t* act = reinterpret_cast<int32_t*>(rf_smem);   // [d/4] Q(g), then Q(h1), then Q(a)
  int32_t* yq4 = act + d4;                                // [d/4] Q(y)
  double* red = reinterpret_cast<double*>(yq4 + d4);      // [32]
  pdl_wait();
  pdl_launch_dependents();   // as the row kernels: let the next kernel launch now
  const int r = blockIdx.x;
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  if (r >= n_live) return;   // uniform over the CTA
  const int c = threadIdx.x;
  const bool on = c < d;
  const int64_t off = (int64_t)r * d;
  for (int i = threadIdx.x; i < d4; i += blockDim.x) {
    act[i] = reinterpret_cast<const int32_t*>(a.g_q + off)[i];
    yq4[i] = reinterpret_cast<const int32_t*>(a.yq + off)[i];
  }
  const float y = on ? a.y[off + c] : 0.0f;
  const float gf0 = (on && a.depth == 0) ? a.g_f[off + c] : 0.0f;
  __syncthreads();
  const float s = a.scale;
  float gi_logit = 0.0f;
  if (a.gate && on) gi_logit = lin_col(a.gi, yq4, d, c, s);        // W_i Q(y) + b_i
  float af;                                                          // AAN output a
  if (a.depth == 2) {
    const float h = on ? relu(lin_col(a.a1, act, d, c, s)) : 0.0f;  // RELU_Q: codes only
    const int8_t hq = (int8_t)q8(h, a.clip, a.sigma);
    __syncthreads();
    if (on) reinterpret_cast<int8_t*>(act)[c] = hq;
    __syncthreads();
    af = on ? lin_col(a.a2, act, d, c, s) : 0.0f;                   // F32_Q
  } else if (a.depth == 1) {
    af = on ? relu(lin_col(a.a1, act, d, c, s)) : 0.0f;             // RELU_F32_Q
  } else {
    af = gf0;                                                        // a = g
  }
  float v;
  if (a.gate) {
    if (a.depth > 0) {   // Q(a) feeds the f gate (for depth 0, Q(a) = Q(g) is already in act)
      const int8_t aq = (int8_t)q8(af, a.clip, a.sigma);
      __syncthreads();
      if (on) reinterpret_cast<int8_t*>(act)[c] = aq;
      __syncthreads();
    }
    const float gf_logit = on ? lin_col(a.gf, act, d, c, s) : 0.0f;
    // R8: z = fl(fl(i*y) + fl(f*a)), residual fl(y + z)
    const float iy = __fmul_rn(sigmoid_f64(gi_logit), y);
    const float fa = __fmul_rn(sigmoid_f64(gf_logit), af);
    v = __fadd_rn(y, __fadd_rn(iy, fa));
  } else {
    v = __fadd_rn(y, af);
  }
  row_ln(v, on, d, a.eps, a.gamma, a.beta, c, red, a.x1 + off, a.x1q + off, a.clip, a.sigma);
}

// ---------------------------------------------------------------- source-attention block (A7)
__global__ void __launch_bounds__(1024) k_src_block(SrcBlockArgs a) {
  extern __shared__ __align__(16) uint8_t rf_smem[];
  const int d = a.d, d4 = d >> 2, dh = d / a.H;
  float* qf = reinterpret_cast<float*>(rf_smem);           // [d] projected query
  int32_t* act = reinterpret_cast<int32_t*>(qf + d);       // [d/4] Q(x1), then Q(ctx)
  double* red = reinterpret_cast<double*>(act + d4 + (d4 & 1));   // [32]
  double* scr = red + 32;                                   // [H][span + 64]
  pdl_wait();
  pdl_launch_dependents();   // as the row kernels: let the next kernel launch now
  const int r = blockIdx.x;
  const int n_live = a.n_dyn ? min(a.n, *a.n_dyn) : a.n;
  if (r >= n_live) return;
  const int c = threadIdx.x, warp = threadIdx.x >> 5;
  const bool on = c < d;
  const int64_t off = (int64_t)r * d;
  const int start = a.live_start[r], len = a.live_len[r];
  for (int i = threadIdx.x; i < d4; i += blockDim.x) act[i] = reinterpret_cast<const int32_t*>(a.x1q + off)[i];
  const float x1 = on ? a.x1[off + c] : 0.0f;
  __syncthreads();
  if (on) qf[c] = lin_col(a.sq, act, d, c, a.scale);          // q = W_q Q(x1) + b_q
  __syncthreads();                                            // q complete, Q(x1) no longer read
  if (warp < a.H) {
    const int h = warp;
    const float* K = a.kv + (int64_t)start * a.ldkv + a.k_off + h * dh;
    const float* V = a.kv + (int64_t)start * a.ldkv + a.v_off + h * dh;
    double* sc = scr + (size_t)h * (a.span + 64);
    warp_attend<float>(qf + h * dh, K, V, a.ldkv, len, dh, sc, sc + a.span, a.clip, a.sigma,
                       reinterpret_cast<int8_t*>(act) + h * dh, nullptr);   // Q(ctx) of head h
  }
  __syncthreads();
  const float o = on ? lin_col(a.so, act, d, c, a.scale) : 0.0f;   // W_o Q(ctx) + b_o
  row_ln(on ? __fadd_rn(x1, o) : 0.0f, on, d, a.eps, a.gamma, a.beta, c, red, a.x2 + off,
         a.x2q + off, a.clip, a.sigma);
}

// ---------------------------------------------------------------- host side
namespace {
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_rf(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
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
int block_threads(int d, int H) {
  int t = d > 32 * H ? d : 32 * H;
  return (t + 31) / 32 * 32;
}
size_t src_smem(int d, int H, int span) {
  const int d4 = d / 4;
  return (size_t)d * 4 + (size_t)(d4 + (d4 & 1)) * 4 + 32 * 8 + (size_t)H * (span + 64) * 8;
}
}  // namespace

cudaError_t launch_repack_k4(const int8_t* W, int N, int K, int32_t* W4, cudaStream_t st) {
  if (N <= 0 || K <= 0 || K % 4) return cudaErrorInvalidValue;
  k_repack_k4<<<256, 256, 0, st>>>(W, N, K, W4);
  return cudaGetLastError();
}

cudaError_t launch_aan_block(const AanBlockArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (a.d % 32 || a.d > 1024) return cudaErrorInvalidValue;
  const size_t smem = (size_t)2 * a.d + 32 * 8;
  return launch_pdl_rf(k_aan_block, dim3(a.n), dim3(block_threads(a.d, 1)), smem, st, a);
}

cudaError_t launch_src_block(const SrcBlockArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int nt = block_threads(a.d, a.H);
  if (a.d % 32 || nt > 1024 || a.d / a.H > 64 || (a.d / a.H) % 4 || a.span < 1 || a.span > MNMT_MAX_KV)
    return cudaErrorInvalidValue;
  return launch_pdl_rf(k_src_block, dim3(a.n), dim3(nt), src_smem(a.d, a.H, a.span), st, a);
}

cudaError_t rowfused_init() {
  static bool done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(k_src_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)src_smem(1024, 32, MNMT_MAX_KV));
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

}  // namespace mnmt
