// shortlist.cu — batch vocabulary shortlist.  See shortlist.h.
#include "shortlist.h"

namespace mnmt {

constexpr int SL_THREADS = 1024;

__device__ __forceinline__ void sl_set(uint32_t* bits, int j, int V) {
  if (j >= 0 && j < V) atomicOr(bits + (j >> 5), 1u << (j & 31));
}

// grid (n_bb, G): CTA (b, g) marks the lex rows of every G-th token of batch b; (b, 0) also
// marks freq, EOS and UNK.  A warp walks one token's k_lex translations (coalesced row read).
__global__ void __launch_bounds__(256) k_sl_mark(SlMarkArgs a) {
  const int b = blockIdx.x;
  uint32_t* bits = a.bits + (int64_t)b * a.W;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (blockIdx.y == 0) {
    for (int i = threadIdx.x; i < a.n_freq; i += blockDim.x) sl_set(bits, a.freq[i], a.V);
    if (threadIdx.x == 0) {
      sl_set(bits, a.eos, a.V);
      sl_set(bits, a.unk, a.V);
    }
  }
  const int s0 = a.bb_off[b], s1 = a.bb_off[b + 1];
  // tokens of the batch, enumerated sentence by sentence; warp-strided over (sentence, token)
  int64_t gw = (int64_t)blockIdx.y * nw + warp;
  const int64_t stride = (int64_t)gridDim.y * nw;
  int64_t base = 0;   // tokens of the sentences before s
  for (int s = s0; s < s1; ++s) {
    const int len = a.sent_len[s], st = a.sent_start[s];
    for (; gw < base + len; gw += stride) {
      const int sid = a.src_ids[st + (gw - base)];
      if (sid < 0 || sid >= a.V) continue;
      const int32_t* row = a.lex + (int64_t)sid * a.k_lex;
      for (int k = lane; k < a.k_lex; k += 32) sl_set(bits, row[k], a.V);
    }
    base += len;
  }
}

// One CTA per wave: union of the wave's batch bitmaps, exclusive prefix of the word popcounts,
// then each thread emits its words' set bits in ascending order with their group masks.
__global__ void __launch_bounds__(SL_THREADS) k_sl_wave(const uint32_t* __restrict__ bits_all,
                                                        int W, int V,
                                                        const int32_t* __restrict__ wave_off,
                                                        int32_t* wave_ids,
                                                        unsigned long long* wave_mask,
                                                        int32_t* wave_n) {
  __shared__ int warp_sum[SL_THREADS / 32];
  const int wv = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b0 = wave_off[wv], ng = wave_off[wv + 1] - b0;
  const uint32_t* bits = bits_all + (int64_t)b0 * W;
  int32_t* out = wave_ids + (int64_t)wv * V;
  unsigned long long* omask = wave_mask + (int64_t)wv * V;
  const int per = (W + SL_THREADS - 1) / SL_THREADS;   // consecutive words per thread
  const int w0 = tid * per, w1 = min(W, w0 + per);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) {
    uint32_t u = 0;
    for (int g = 0; g < ng; ++g) u |= bits[(int64_t)g * W + w];
    cnt += __popc(u);
  }
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) warp_sum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int x = warp_sum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += u;
    }
    warp_sum[lane] = x;   // inclusive over warps
  }
  __syncthreads();
  int pos = (warp ? warp_sum[warp - 1] : 0) + v - cnt;
  for (int w = w0; w < w1; ++w) {
    uint32_t gw[SL_MAX_GROUPS];
    uint32_t u = 0;
    for (int g = 0; g < ng; ++g) u |= (gw[g] = bits[(int64_t)g * W + w]);
    while (u) {
      const int bit = __ffs(u) - 1;
      unsigned long long mk = 0ull;
      for (int g = 0; g < ng; ++g) mk |= (unsigned long long)((gw[g] >> bit) & 1u) << g;
      out[pos] = w * 32 + bit;
      omask[pos] = mk;
      ++pos;
      u &= u - 1;
    }
  }
  if (tid == SL_THREADS - 1) wave_n[wv] = pos;
}

cudaError_t launch_sl_build(const SlMarkArgs& a, int n_bb, const int32_t* wave_off, int n_waves,
                            int32_t* wave_ids, unsigned long long* wave_mask, int32_t* wave_n,
                            cudaStream_t st) {
  if (n_bb <= 0 || n_waves <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(a.bits, 0, (size_t)n_bb * a.W * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  const int G = n_bb >= 148 ? 1 : (148 * 4 + n_bb - 1) / n_bb;
  k_sl_mark<<<dim3(n_bb, G), 256, 0, st>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_sl_wave<<<n_waves, SL_THREADS, 0, st>>>(a.bits, a.W, a.V, wave_off, wave_ids, wave_mask,
                                            wave_n);
  return cudaGetLastError();
}

// A warp per shortlist row: d / 16 lanes copy 16-byte chunks of the E code row; then a warp per
// 32 columns: lane = column, one ballot per group gives that group's bitmap word.
__global__ void __launch_bounds__(256) k_sl_gather(const int32_t* __restrict__ ids,
                                                   const unsigned long long* __restrict__ mask,
                                                   int n, int n_groups,
                                                   const int8_t* __restrict__ qE,
                                                   const float* __restrict__ bias, int d,
                                                   int8_t* __restrict__ dst_q,
                                                   float* __restrict__ dst_b,
                                                   int32_t* __restrict__ dst_map,
                                                   uint32_t* __restrict__ dst_bits, int ld) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5, chunks = d >> 4;
  for (int r = warp; r < n; r += nwarps) {
    const int id = ids[r];
    const int4* src = reinterpret_cast<const int4*>(qE + (int64_t)id * d);
    int4* dst = reinterpret_cast<int4*>(dst_q + (int64_t)r * d);
    for (int c = lane; c < chunks; c += 32) dst[c] = src[c];
    if (lane == 0) {
      dst_map[r] = id;
      if (dst_b) dst_b[r] = bias ? bias[id] : 0.0f;
    }
  }
  for (int wd = warp; wd < (n + 31) / 32; wd += nwarps) {
    const int r = wd * 32 + lane;
    const unsigned long long mk = r < n ? mask[r] : 0ull;
    for (int g = 0; g < n_groups; ++g) {
      const uint32_t b = __ballot_sync(0xffffffffu, (mk >> g) & 1ull);
      if (lane == 0) dst_bits[(int64_t)g * ld + wd] = b;
    }
  }
}

cudaError_t launch_sl_gather(const int32_t* ids, const unsigned long long* mask, int n,
                             int n_groups, const int8_t* qE, const float* bias, int d,
                             int8_t* dst_q, float* dst_b, int32_t* dst_map, uint32_t* dst_bits,
                             int ld, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_sl_gather<<<blocks, 256, 0, st>>>(ids, mask, n, n_groups, qE, bias, d, dst_q, dst_b, dst_map,
                                      dst_bits, ld);
  return cudaGetLastError();
}

}  // namespace mnmt
