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

// exp(x) for x <= 0 in fp64 (same construction as the GEMM epilogue's exp_neg; R26).
__device__ const double c_beam_exp2_64[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284, 1.0442737824274138,
    1.0556451783605572, 1.0671404006768237, 1.0787607977571199, 1.0905077326652577,
    1.102382583307841, 1.1143867425958924, 1.1265216186082418, 1.1387886347566916,
    1.1511892299529827, 1.1637248587775775, 1.1763969916502812, 1.189207115002721,
    1.202156731452703, 1.215247359980469, 1.22848053610687, 1.241857812073484,
    1.255380757024691, 1.2690509571917332, 1.2828700160787783, 1.2968395546510096,
    1.3109612115247644, 1.3252366431597413, 1.339667524053303, 1.3542555469368927,
    1.3690024229745905, 1.383909881963832, 1.3989796725383112, 1.4142135623730951,
    1.42961333839197, 1.4451808069770467, 1.460917794180647, 1.4768261459394993,
    1.4929077282912648, 1.5091644275934228, 1.5255981507445384, 1.5422108254079407,
    1.559004400237837, 1.5759808451078865, 1.593142151342267, 1.6104903319492543,
    1.6280274218573478, 1.645755478153965, 1.6636765803267364, 1.681792830507429,
    1.7001063537185235, 1.718619298122478, 1.7373338352737062, 1.7562521603732995,
    1.7753764925265212, 1.7947090750031072, 1.8142521755003989, 1.8340080864093424,
    1.8539791250833855, 1.8741676341103, 1.8945759815869656, 1.9152065613971474,
    1.9360617934922943, 1.9571441241754002, 1.978456026387951};

__device__ __forceinline__ double beam_exp_neg(double x, const double* tab) {
  if (x < -707.0) return 0.0;
  const double kd = rint(x * 92.33248261689366);
  double r = fma(kd, -0.01083042469326756, x);
  r = fma(kd, -2.9815858269852933e-12, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = (int)kd;
  const double v = p * tab[k & 63];
  return __hiloint2double(__double2hiint(v) + ((k >> 6) << 20), __double2loint(v));
}

constexpr int BEAM_LOGITS_THREADS = 512;

// One CTA per live row of materialised logits: the row maximum M (pass 1), then
// Z = sum exp((double)l - M) in fp64 per thread (4 partial sums) + block tree, and the row's
// top-beam (value desc, id asc) from per-thread sorted lists merged in beam block rounds.
template <int TK>
__global__ void __launch_bounds__(BEAM_LOGITS_THREADS) k_beam_logits(BeamArgs a) {
  __shared__ double tab[64];
  __shared__ double zs[BEAM_LOGITS_THREADS / 32];
  __shared__ float ms[BEAM_LOGITS_THREADS / 32];
  __shared__ unsigned long long ks[BEAM_LOGITS_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = BEAM_LOGITS_THREADS / 32;
  if (tid < 64) tab[tid] = c_beam_exp2_64[tid];
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x;
  if (r >= a.ctrl[0]) return;   // block-uniform
  const float* L = a.logits + (int64_t)r * a.ld_logits;
  const int V = a.V, V4 = V >> 2;
  const float4* L4 = reinterpret_cast<const float4*>(L);
  // pass 1: maximum and per-thread top-TK
  float mx = -INFINITY;
  float tv[TK];
  int tj[TK];
#pragma unroll
  for (int i = 0; i < TK; ++i) { tv[i] = -INFINITY; tj[i] = -1; }
  auto ins = [&](float cv, int cj) {
    bool sh = false;
#pragma unroll
    for (int i = 0; i < TK; ++i) {
      const bool take = sh || cv > tv[i];
      const float ov = tv[i];
      const int oj = tj[i];
      tv[i] = take ? cv : ov;
      tj[i] = take ? cj : oj;
      cv = take ? ov : cv;
      cj = take ? oj : cj;
      sh = take;
    }
  };
  for (int q = tid; q < V4; q += BEAM_LOGITS_THREADS) {   // columns ascending per thread
    const float4 x = L4[q];
    mx = fmaxf(mx, fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
    if (x.x > tv[TK - 1]) ins(x.x, 4 * q);
    if (x.y > tv[TK - 1]) ins(x.y, 4 * q + 1);
    if (x.z > tv[TK - 1]) ins(x.z, 4 * q + 2);
    if (x.w > tv[TK - 1]) ins(x.w, 4 * q + 3);
  }
  for (int j = 4 * V4 + tid; j < V; j += BEAM_LOGITS_THREADS) {
    const float x = L[j];
    mx = fmaxf(mx, x);
    if (x > tv[TK - 1]) ins(x, j);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) ms[w] = mx;
  __syncthreads();
  mx = ms[0];
  for (int i = 1; i < nw; ++i) mx = fmaxf(mx, ms[i]);
  // pass 2: Z (the row is re-read from L2)
  const double md = (double)mx;
  double zp[4] = {0.0, 0.0, 0.0, 0.0};
  for (int q = tid; q < V4; q += BEAM_LOGITS_THREADS) {
    const float4 x = L4[q];
    zp[0] = __dadd_rn(zp[0], beam_exp_neg(__dsub_rn((double)x.x, md), tab));
    zp[1] = __dadd_rn(zp[1], beam_exp_neg(__dsub_rn((double)x.y, md), tab));
    zp[2] = __dadd_rn(zp[2], beam_exp_neg(__dsub_rn((double)x.z, md), tab));
    zp[3] = __dadd_rn(zp[3], beam_exp_neg(__dsub_rn((double)x.w, md), tab));
  }
  for (int j = 4 * V4 + tid; j < V; j += BEAM_LOGITS_THREADS)
    zp[0] = __dadd_rn(zp[0], beam_exp_neg(__dsub_rn((double)L[j], md), tab));
  double z = __dadd_rn(__dadd_rn(zp[0], zp[1]), __dadd_rn(zp[2], zp[3]));
  z = warp_sum_f64(z);
  if (lane == 0) zs[w] = z;
  __syncthreads();
  if (tid == 0) {
    double Z = 0.0;
    for (int i = 0; i < nw; ++i) Z = __dadd_rn(Z, zs[i]);
    a.row_lse[r] = (float)__dadd_rn(md, log(Z));
  }
  // top-beam: beam rounds of a block-wide packed (value, lowest id) maximum over list heads
  int head = 0;
  for (int i = 0; i < a.beam; ++i) {
    float hv = -INFINITY;
    int hj = -1;
#pragma unroll
    for (int u = 0; u < TK; ++u)
      if (u == head) { hv = tv[u]; hj = tj[u]; }
    const unsigned long long key = hj >= 0 ? argmax_key(hv, (uint32_t)hj) : 0ull;
    unsigned long long mk = key;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, mk, o);
      mk = other > mk ? other : mk;
    }
    __syncthreads();
    if (lane == 0) ks[w] = mk;
    __syncthreads();
    mk = ks[0];
    for (int u = 1; u < nw; ++u) mk = ks[u] > mk ? ks[u] : mk;
    if (key == mk && mk != 0ull) {   // exactly one thread holds the winning (value, id)
      ++head;
      a.row_v[(int64_t)r * TOPK_MAX + i] = hv;
      a.row_j[(int64_t)r * TOPK_MAX + i] = hj;
    }
  }
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
cudaError_t launch_beam_logits(const BeamArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (a.beam <= 2)
    return launch_pdl(k_beam_logits<2>, dim3(a.n), dim3(BEAM_LOGITS_THREADS), 0, st, a);
  if (a.beam <= 4)
    return launch_pdl(k_beam_logits<4>, dim3(a.n), dim3(BEAM_LOGITS_THREADS), 0, st, a);
  return launch_pdl(k_beam_logits<8>, dim3(a.n), dim3(BEAM_LOGITS_THREADS), 0, st, a);
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
