// beam.cu — beam-search step kernels (see beam.h).
//
// Numerics (R26-R28): a row's log-sum-exp is lse = fl32(M + log Z) with
// Z = sum_j exp((double)l_j - M) accumulated in fp64 (per 32-column chunk in the GEMM
// epilogue, then across tiles here: a reordering of the same fp64 sum, R20); the candidate
// score is fl32(score + fl32(l_j - lse)); candidates rank by (score desc, logit desc,
// hypothesis rank asc, id asc).  Every selection is taken on those fp32 values.
#include <cstdint>
#include <utility>

#include "beam.h"
#include "numerics.cuh"
#include "ptx.cuh"

namespace mnmt {

constexpr int BEAM_SELECT_THREADS = 1024;
constexpr int BEAM_ROWS_WARPS = 4;
constexpr int BEAM_REORDER_THREADS = 256;

// ------------------------------------------------------------------ init
__global__ void k_beam_init(BeamArgs a, int n_sent) {
  pdl_wait();
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_sent; s += gridDim.x * blockDim.x) {
    a.live[s] = s * a.beam;
    a.prev_live[s] = 0;
    a.live_start[s] = a.row_start[s];
    a.live_len[s] = a.row_len[s];
    a.sent_row0[s] = s;
    a.sent_nlive[s] = 1;
    a.sent_nfin[s] = 0;
    a.hscore[s * a.beam] = 0.0f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctrl[0] = n_sent;
    a.ctrl[1] = 1;
    a.ctrl[2] = n_sent;
    a.ctrl[3] = 0;
  }
}

// ------------------------------------------------------------------ per-row merge
// (v, j) ranks before (w, k): larger value, then lower id.
__device__ __forceinline__ bool vj_before(float v, int j, float w, int k) {
  return v > w || (v == w && (unsigned)j < (unsigned)k);   // j = -1 (empty) ranks last
}

__global__ void __launch_bounds__(BEAM_ROWS_WARPS * 32) k_beam_rows(BeamArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * BEAM_ROWS_WARPS + (threadIdx.x >> 5);
  if (r >= a.n || r >= a.ctrl[0]) return;
  const TopkPart* P = a.part + (int64_t)r * a.part_ld;
  float M = -INFINITY;
  for (int p = lane; p < a.n_part; p += 32) M = fmaxf(M, P[p].m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  double Z = 0.0;
  float lv[TOPK_MAX];
  int lj[TOPK_MAX];
#pragma unroll
  for (int i = 0; i < TOPK_MAX; ++i) { lv[i] = -INFINITY; lj[i] = -1; }
  for (int p = lane; p < a.n_part; p += 32) {
    const float pm = P[p].m;
    if (pm == -INFINITY) continue;
    Z = __dadd_rn(Z, __dmul_rn(P[p].z, exp(__dsub_rn((double)pm, (double)M))));
    for (int i = 0; i < TOPK_MAX; ++i) {
      float cv = P[p].v[i];
      int cj = P[p].j[i];
      if (cj < 0 || !vj_before(cv, cj, lv[TOPK_MAX - 1], lj[TOPK_MAX - 1])) break;   // sorted
      bool sh = false;
#pragma unroll
      for (int u = 0; u < TOPK_MAX; ++u) {
        const bool take = sh || vj_before(cv, cj, lv[u], lj[u]);
        const float ov = lv[u];
        const int oj = lj[u];
        lv[u] = take ? cv : ov;
        lj[u] = take ? cj : oj;
        cv = take ? ov : cv;
        cj = take ? oj : cj;
        sh = take;
      }
    }
  }
  Z = warp_sum_f64(Z);
  const float lse = (float)__dadd_rn((double)M, log(Z));
  // warp merge of the per-lane lists: beam rounds of a packed (value, lowest id) maximum
  int head = 0;
  for (int i = 0; i < a.beam; ++i) {
    float hv = -INFINITY;
    int hj = -1;
#pragma unroll
    for (int u = 0; u < TOPK_MAX; ++u)
      if (u == head) { hv = lv[u]; hj = lj[u]; }
    const unsigned long long key = hj >= 0 ? argmax_key(hv, (uint32_t)hj) : 0ull;
    unsigned long long mk = key;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, mk, o);
      mk = other > mk ? other : mk;
    }
    const unsigned win = __ballot_sync(0xffffffffu, key == mk && mk != 0ull);
    const int wl = win ? __ffs(win) - 1 : 0;
    const float wv = __shfl_sync(0xffffffffu, hv, wl);
    const int wj = __shfl_sync(0xffffffffu, hj, wl);
    if (lane == wl && win) ++head;
    if (lane == 0) {
      a.row_v[(int64_t)r * TOPK_MAX + i] = win ? wv : -INFINITY;
      a.row_j[(int64_t)r * TOPK_MAX + i] = win ? wj : -1;
    }
  }
  if (lane == 0) a.row_lse[r] = lse;
}

// ------------------------------------------------------------------ selection + compaction
// Block-wide exclusive scan of one int per thread (blockDim multiple of 32, <= 1024).
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += u;
    }
    wsum[lane] = x;   // inclusive over warps
  }
  __syncthreads();
  total = wsum[nw - 1];
  const int excl = (w ? wsum[w - 1] : 0) + incl - v;
  __syncthreads();
  return excl;
}

// candidate a ranks before candidate b (R28)
__device__ __forceinline__ bool cand_before(float sa, float la, int ka, int ja, float sb, float lb,
                                            int kb, int jb) {
  if (sa != sb) return sa > sb;
  if (la != lb) return la > lb;
  if (ka != kb) return ka < kb;
  return ja < jb;
}

__global__ void __launch_bounds__(BEAM_SELECT_THREADS) k_beam_select(BeamArgs a) {
  __shared__ int wsum[32];
  __shared__ int base_rows_s, base_sents_s;
  pdl_wait();
  pdl_launch_dependents();
  const int t = a.ctrl[1], n_sent = a.ctrl[2], B = a.beam;
  // phase 1: every sentence's selection (reads the compact rows of this step)
  for (int s = threadIdx.x; s < n_sent; s += blockDim.x) {
    const int nl = a.sent_nlive[s];
    if (nl == 0) continue;
    const int r0 = a.sent_row0[s], ml = a.max_len[s];
    int nfin = a.sent_nfin[s];
    const int nkeep = B - nfin;
    const int li = a.len_idx ? a.len_idx[s] : s;
    int32_t* out_base = a.out_ids + (int64_t)B * a.out_off[s];
    uint64_t taken = 0;
    int n_next = 0;
    for (int rank = 0; rank < nkeep; ++rank) {
      int bk = -1, bi = -1, bj = -1;
      float bs = 0.0f, bv = 0.0f;
      for (int k = 0; k < nl; ++k) {
        const int r = r0 + k;
        const float sc = a.hscore[a.live[r]], lse = a.row_lse[r];
        for (int i = 0; i < B; ++i) {
          if ((taken >> (k * TOPK_MAX + i)) & 1ull) continue;
          const int j = a.row_j[(int64_t)r * TOPK_MAX + i];
          if (j < 0) continue;
          const float v = a.row_v[(int64_t)r * TOPK_MAX + i];
          const float cs = __fadd_rn(sc, __fsub_rn(v, lse));
          if (bk < 0 || cand_before(cs, v, k, j, bs, bv, bk, bj)) {
            bk = k; bi = i; bj = j; bs = cs; bv = v;
          }
        }
      }
      if (bk < 0) break;
      taken |= 1ull << (bk * TOPK_MAX + bi);
      const int ps = a.live[r0 + bk];
      if (bj == a.eos || t == ml) {
        // finished: the parent's ids (steps 1..t-1) plus this id unless it is EOS (R16)
        int32_t* dst = out_base + (int64_t)nfin * ml;
        const int32_t* h = a.hist + (int64_t)ps * a.t_cap;
        for (int u = 0; u < t - 1; ++u) dst[u] = h[u];
        int len = t - 1;
        if (bj != a.eos) dst[len++] = bj;
        a.out_len[(int64_t)li * B + nfin] = len;
        a.out_score[(int64_t)li * B + nfin] = bs;
        ++nfin;
      } else {
        const int c = s * B + n_next++;
        a.child_par[c] = ps;
        a.child_tok[c] = bj;
        a.child_score[c] = bs;
      }
    }
    a.sent_nfin[s] = nfin;
    a.sent_nlive[s] = n_next;
  }
  __syncthreads();
  // phase 2: stable compaction of the children into the next step's compact rows
  if (threadIdx.x == 0) { base_rows_s = 0; base_sents_s = 0; }
  __syncthreads();
  for (int c0 = 0; c0 < n_sent; c0 += blockDim.x) {
    const int s = c0 + threadIdx.x;
    const int cnt = s < n_sent ? a.sent_nlive[s] : 0;
    int tot_rows = 0, tot_sents = 0;
    const int er = block_excl_scan(cnt, wsum, tot_rows);
    const int es = block_excl_scan(cnt > 0 ? 1 : 0, wsum, tot_sents);
    const int br = base_rows_s, bs = base_sents_s;
    if (cnt > 0) {
      const int row0 = br + er;
      a.sent_row0[s] = row0;
      a.sent_list[bs + es] = s;
      for (int c = 0; c < cnt; ++c) {
        a.live[row0 + c] = s * B + c;
        a.prev_live[row0 + c] = a.child_tok[s * B + c];
        a.live_start[row0 + c] = a.row_start[s];
        a.live_len[row0 + c] = a.row_len[s];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) { base_rows_s = br + tot_rows; base_sents_s = bs + tot_sents; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.ctrl[0] = base_rows_s;
    a.ctrl[1] = t + 1;
    a.ctrl[3] = base_sents_s;
  }
}

// ------------------------------------------------------------------ state reorder
// One CTA per sentence with children: child c (slot s * beam + c) takes its parent's AAN
// running sums, emitted ids and (self-attention) ancestor rows, staged through shared
// memory because parents and children share the sentence's slots.
__global__ void __launch_bounds__(BEAM_REORDER_THREADS) k_beam_reorder(BeamArgs a) {
  extern __shared__ __align__(16) float rb[];
  __shared__ int par[TOPK_MAX];
  __shared__ int ident;
  pdl_wait();
  pdl_launch_dependents();
  if ((int)blockIdx.x >= a.ctrl[3]) return;
  const int s = a.sent_list[blockIdx.x];
  const int nn = a.sent_nlive[s], B = a.beam, t = a.ctrl[1] - 1, tid = threadIdx.x;
  if (tid == 0) ident = 1;
  __syncthreads();
  if (tid < nn) {
    par[tid] = a.child_par[s * B + tid];
    if (par[tid] != s * B + tid) ident = 0;
  }
  __syncthreads();
  if (!ident) {
    const int d = a.d;
    if (a.C) {
      for (int l = 0; l < a.L; ++l) {
        float* Cl = a.C + (int64_t)l * a.c_stride;
        for (int i = tid; i < nn * d; i += blockDim.x) {
          const int c = i / d;
          rb[i] = Cl[(int64_t)par[c] * d + (i - c * d)];
        }
        __syncthreads();
        for (int i = tid; i < nn * d; i += blockDim.x) {
          const int c = i / d;
          Cl[(int64_t)(s * B + c) * d + (i - c * d)] = rb[i];
        }
        __syncthreads();
      }
    }
    int32_t* ib = reinterpret_cast<int32_t*>(rb);
    const int w_h = t - 1;   // ids of steps 1..t-1
    for (int i = tid; i < nn * w_h; i += blockDim.x) {
      const int c = i / w_h;
      ib[i] = a.hist[(int64_t)par[c] * a.t_cap + (i - c * w_h)];
    }
    __syncthreads();
    for (int i = tid; i < nn * w_h; i += blockDim.x) {
      const int c = i / w_h;
      a.hist[(int64_t)(s * B + c) * a.t_cap + (i - c * w_h)] = ib[i];
    }
    __syncthreads();
    if (a.anc) {
      for (int i = tid; i < nn * t; i += blockDim.x) {
        const int c = i / t;
        ib[i] = a.anc[(int64_t)par[c] * a.t_cap + (i - c * t)];
      }
      __syncthreads();
      for (int i = tid; i < nn * t; i += blockDim.x) {
        const int c = i / t;
        a.anc[(int64_t)(s * B + c) * a.t_cap + (i - c * t)] = ib[i];
      }
      __syncthreads();
    }
  }
  if (tid < nn) {
    a.hist[(int64_t)(s * B + tid) * a.t_cap + t - 1] = a.child_tok[s * B + tid];
    a.hscore[s * B + tid] = a.child_score[s * B + tid];
  }
}

// ------------------------------------------------------------------ n-best order
// Thread per sentence: finished hypotheses stably sorted by descending score (the hist rows
// of the sentence's slots are free after the last step and serve as scratch).
__global__ void k_beam_final(BeamArgs a, int n_sent) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sent) return;
  const int B = a.beam, nf = a.sent_nfin[s], ml = a.max_len[s];
  const int li = a.len_idx ? a.len_idx[s] : s;
  int ord[TOPK_MAX];
  for (int f = 0; f < nf; ++f) {
    const float sc = a.out_score[(int64_t)li * B + f];
    int j = f - 1;
    while (j >= 0 && a.out_score[(int64_t)li * B + ord[j]] < sc) { ord[j + 1] = ord[j]; --j; }
    ord[j + 1] = f;
  }
  int32_t* ids = a.out_ids + (int64_t)B * a.out_off[s];
  float sc[TOPK_MAX];
  int ln[TOPK_MAX];
  for (int f = 0; f < nf; ++f) {
    int32_t* tmp = a.hist + (int64_t)(s * B + f) * a.t_cap;
    for (int u = 0; u < ml; ++u) tmp[u] = ids[(int64_t)f * ml + u];
    sc[f] = a.out_score[(int64_t)li * B + f];
    ln[f] = a.out_len[(int64_t)li * B + f];
  }
  for (int f = 0; f < nf; ++f) {
    const int o = ord[f];
    const int32_t* tmp = a.hist + (int64_t)(s * B + o) * a.t_cap;
    for (int u = 0; u < ml; ++u) ids[(int64_t)f * ml + u] = tmp[u];
    a.out_score[(int64_t)li * B + f] = sc[o];
    a.out_len[(int64_t)li * B + f] = ln[o];
  }
  a.n_hyp[li] = nf;
}

// ------------------------------------------------------------------ launchers
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

cudaError_t launch_beam_init(const BeamArgs& a, int n_sent, cudaStream_t st) {
  if (n_sent <= 0) return cudaSuccess;
  return launch_pdl(k_beam_init, dim3((n_sent + 255) / 256), dim3(256), 0, st, a, n_sent);
}
cudaError_t launch_beam_rows(const BeamArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  return launch_pdl(k_beam_rows, dim3((a.n + BEAM_ROWS_WARPS - 1) / BEAM_ROWS_WARPS),
                    dim3(32 * BEAM_ROWS_WARPS), 0, st, a);
}
cudaError_t launch_beam_select(const BeamArgs& a, cudaStream_t st) {
  return launch_pdl(k_beam_select, dim3(1), dim3(BEAM_SELECT_THREADS), 0, st, a);
}
cudaError_t launch_beam_reorder(const BeamArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const size_t smem = (size_t)a.beam * (size_t)(a.d > a.t_cap ? a.d : a.t_cap) * 4;
  return launch_pdl(k_beam_reorder, dim3(a.n), dim3(BEAM_REORDER_THREADS), smem, st, a);
}
cudaError_t launch_beam_final(const BeamArgs& a, int n_sent, cudaStream_t st) {
  if (n_sent <= 0) return cudaSuccess;
  return launch_pdl(k_beam_final, dim3((n_sent + 127) / 128), dim3(128), 0, st, a, n_sent);
}

}  // namespace mnmt
