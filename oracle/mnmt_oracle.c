/*
 * mnmt_oracle.c — plain, slow, obviously-correct CPU oracle for batched greedy
 * decoding of a distilled Transformer / AAN student with int8 products
 * (arXiv 1805.12096, "Marian: Cost-effective High-Quality Neural Machine
 * Translation in C++", WNMT 2018).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1805_12096_b200/, libmnmt) never links, imports or calls
 * it, and it shares no code, header, table or constant generator with it.
 *
 * Citations: P:L<n> = /root/reference/PAPER.md line n; "R<k>" = the reading
 * numbered k in DESIGN.md section "Readings of the paper".
 *
 * Numeric contract (R1-R6, R20):
 *   - activations are stored in fp32 (Marian tensors);
 *   - every product with a parameter is int8 x int8 -> exact int32 (P:L94,
 *     P:L100; R3), dequantized as fmaf((float)acc, s, b) (R5);
 *   - LayerNorm / attention / softmax / sigmoid accumulate in fp64 and round
 *     once to fp32 (R20);
 *   - elementwise adds/multiplies/divides are single fp32 operations
 *     (compile with -ffp-contract=off so nothing is fused).
 *
 * Parity pins: tests/test_oracle_pins.py.  Functions with no independent pin
 * would be marked "parity unpinned" here; see the per-function notes.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_LAYERS 16

/* ---------------------------------------------------------------- config */
typedef struct {
    int32_t d_model, d_ffn, n_heads, enc_layers, dec_layers, vocab;
    int32_t decoder;        /* 0 = self-attention + KV cache, 1 = AAN */
    int32_t aan_ffn_depth;  /* 0 (= "-ffn"), 1, 2 (R9) */
    int32_t aan_gate;       /* 1 or 0 (= "-gate") */
    int32_t out_bias;       /* 1 or 0 (R14) */
    int32_t eos_id;         /* R16 */
    float clip;             /* c = 2 */
    float ln_eps;           /* R10 */
    int32_t arith;          /* integer products (oracle only):
                             * 0 = int8 codes, exact int32 accumulation (R3; the GPU path);
                             * 1 = int8 codes, saturating int16 accumulation of adjacent pairs
                             *     ("accumulated in 16-bit integers with saturation");
                             * 2 = int16 codes RNE(x * 2^10), wrapping int32 accumulation */
    int32_t src_kv_bf16;    /* 1 = each source key / value element is
                             * rounded to the nearest bfloat16 (ties to even) after its
                             * projection; attention then uses the rounded values */
} orc_cfg;

typedef struct { float *W, *b; int16_t *qW; int out, in; } orc_lin;   /* codes of arith (int8 range for 0/1) */
typedef struct { float *g, *b; } orc_ln;
typedef struct { orc_lin q, k, v, o, f1, f2; orc_ln ln1, ln2; } orc_enc_layer;
typedef struct {
    orc_lin a1, a2, gi, gf;          /* AAN FFN and gates (R8, R9) */
    orc_lin q, k, v, o;              /* decoder self-attention */
    orc_lin sq, sk, sv, so;          /* source attention */
    orc_lin f1, f2;                  /* FFN */
    orc_ln ln1, ln2, ln3;
} orc_dec_layer;

typedef struct {
    orc_cfg c;
    float *E, *out_b;                /* tied embedding [V x d] */
    int16_t *qE;
    orc_enc_layer enc[ORC_MAX_LAYERS];
    orc_dec_layer dec[ORC_MAX_LAYERS];
    int quantized;
} orc_model;

/* ------------------------------------------------------------- scalars */
/* sigma = 127/c, s = c^2/127^2 ("scaled linearly to [-127,127]"; R2). */
float orc_sigma(float clip) { return 127.0f / clip; }

/* Nearest bfloat16 of a finite fp32 x, ties to even (R35): bfloat16 keeps the
 * sign, the 8 exponent bits and the top 7 mantissa bits of the fp32 encoding, so x is rounded
 * to a multiple of 2^16 in its bit pattern; the returned float is that bfloat16 value. */
float orc_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    uint32_t low = u & 0xFFFFu, keep = u & 0xFFFF0000u;
    if (low > 0x8000u || (low == 0x8000u && (keep & 0x10000u))) keep += 0x10000u;   /* round up */
    float r;
    memcpy(&r, &keep, 4);
    return r;
}
float orc_dequant_scale(float clip) {
    return (float)(((double)clip * (double)clip) / (127.0 * 127.0));
}

/* Q(x) = RNE(clip(x, +-c) * sigma) ("clipped to a range ... scaled
 * linearly to [-127,127] and rounded to integers"; rounding mode R1). */
int8_t orc_q(float x, float clip) {
    float v = x;
    if (v > clip) v = clip;
    if (v < -clip) v = -clip;
    float y = v * orc_sigma(clip);
    return (int8_t)nearbyintf(y);   /* FE_TONEAREST: ties to even */
}

void orc_quantize(const float *x, int64_t n, float clip, int8_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_q(x[i], clip);
}

/* dotint(quant(A), quant(B^T)) = A . B^T with int32 accumulation (
 * exact s32 accumulation R3).  acc[i][j] = sum_k a[i][k] * w[j][k]. */
void orc_gemm_acc(const int8_t *a, const int8_t *w, int M, int N, int K, int32_t *acc) {
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            int32_t s = 0;
            const int8_t *ar = a + (int64_t)i * K, *wr = w + (int64_t)j * K;
            for (int k = 0; k < K; ++k) s += (int32_t)ar[k] * (int32_t)wr[k];
            acc[(int64_t)i * N + j] = s;
        }
}

/* lin over M rows: out[i][j] = fmaf((float)sum_k qa[i][k] qw[j][k], s, b[j]) (R5). */
void orc_linear(const int8_t *qa, const int8_t *qw, int M, int N, int K, const float *b,
                float clip, float *out) {
    float s = orc_dequant_scale(clip);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            int32_t acc = 0;
            for (int k = 0; k < K; ++k)
                acc += (int32_t)qa[(int64_t)i * K + k] * (int32_t)qw[(int64_t)j * K + k];
            out[(int64_t)i * N + j] = fmaf((float)acc, s, b ? b[j] : 0.0f);
        }
}

/* ------------------------------------------------ F4: integer arithmetic variants */
/* int16 quantization of P:L92 ("multiplying parameters and inputs by 2^10 before rounding
 * to signed integers"): RNE(x * 1024) (R1's rounding), saturated to +-32767. */
int16_t orc_q16(float x) {
    float y = nearbyintf(x * 1024.0f);   /* x * 2^10 is exact */
    if (y > 32767.0f) y = 32767.0f;
    if (y < -32767.0f) y = -32767.0f;
    return (int16_t)y;
}

static int16_t code1(const orc_cfg *c, float x) {
    return c->arith == 2 ? orc_q16(x) : (int16_t)orc_q(x, c->clip);
}
static void qcodes(const orc_cfg *c, const float *x, int64_t n, int16_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = code1(c, x[i]);
}
/* dequantization scale of a product: s = c^2/127^2 (int8, R2) or 2^-20 (int16). */
static float code_scale(const orc_cfg *c) {
    return c->arith == 2 ? (float)(1.0 / 1048576.0) : orc_dequant_scale(c->clip);
}

static int16_t sat16(int32_t v) { return (int16_t)(v > 32767 ? 32767 : v < -32768 ? -32768 : v); }

/* One dot product of codes under arithmetic `arith`:
 *   0: exact int32 sum;
 *   1: k in adjacent pairs, p = sat16(a0*b0 + a1*b1), acc = sat16(acc + p), ascending pairs
 *      (the pair-then-accumulate order of vpmaddubsw + vpaddsw; odd K padded with a zero);
 *   2: products in int32, sum wrapping modulo 2^32 (no 32-bit saturating add in AVX512F,
 *      P:L92), ascending k. */
int32_t orc_dot_codes(int arith, const int16_t *a, const int16_t *w, int K) {
    if (arith == 1) {
        int16_t acc = 0;
        for (int k = 0; k < K; k += 2) {
            int32_t p = (int32_t)a[k] * w[k];
            if (k + 1 < K) p += (int32_t)a[k + 1] * w[k + 1];
            acc = sat16((int32_t)acc + (int32_t)sat16(p));
        }
        return acc;
    }
    if (arith == 2) {
        uint32_t acc = 0;
        for (int k = 0; k < K; ++k) acc += (uint32_t)((int32_t)a[k] * (int32_t)w[k]);
        return (int32_t)acc;
    }
    int32_t acc = 0;
    for (int k = 0; k < K; ++k) acc += (int32_t)a[k] * (int32_t)w[k];
    return acc;
}

/* lin(qa; W, b)[j] = fmaf((float)acc_j, s, b_j)  (R5). b may be NULL (= 0). */
static void lin1(const orc_cfg *c, const orc_lin *L, const int16_t *qa, float *out) {
    float s = code_scale(c);
    for (int j = 0; j < L->out; ++j) {
        int32_t acc = orc_dot_codes(c->arith, qa, L->qW + (int64_t)j * L->in, L->in);
        out[j] = fmaf((float)acc, s, L->b ? L->b[j] : 0.0f);
    }
}

void orc_sigmoid_array(const float *x, int64_t n, float *out);

/* LayerNorm, post-norm (P:L65 Vaswani recipe; R10), fp64 accumulation (R20):
 * mu = sum r / d; var = sum (r-mu)^2 / d; out = (r-mu)/sqrt(var+eps)*g + b. */
void orc_layernorm(const float *r, int d, const float *g, const float *b, float eps, float *out) {
    double mu = 0.0, var = 0.0;
    for (int k = 0; k < d; ++k) mu += (double)r[k];
    mu /= (double)d;
    for (int k = 0; k < d; ++k) { double t = (double)r[k] - mu; var += t * t; }
    var /= (double)d;
    double inv = 1.0 / sqrt(var + (double)eps);
    for (int k = 0; k < d; ++k)
        out[k] = (float)((((double)r[k] - mu) * inv) * (double)g[k] + (double)b[k]);
}

/* Scaled dot-product attention of one query row over n key/value rows
 * (Vaswani et al.).  Head h uses columns [h*dh, (h+1)*dh) (R11).
 * fp64 accumulation, one rounding to fp32 per context element (R20).
 * k, v: row j at k + j*ld. */
void orc_attention(const float *q, const float *k, const float *v, int64_t ld, int n,
                   int d, int H, float *ctx) {
    int dh = d / H;
    double inv_sqrt = 1.0 / sqrt((double)dh);
    double *sc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int h = 0; h < H; ++h) {
        double mx = -INFINITY;
        for (int j = 0; j < n; ++j) {
            double dot = 0.0;
            for (int c = 0; c < dh; ++c)
                dot += (double)q[h * dh + c] * (double)k[(int64_t)j * ld + h * dh + c];
            sc[j] = dot * inv_sqrt;
            if (sc[j] > mx) mx = sc[j];
        }
        double Z = 0.0;
        for (int j = 0; j < n; ++j) { sc[j] = exp(sc[j] - mx); Z += sc[j]; }
        for (int c = 0; c < dh; ++c) {
            double acc = 0.0;
            for (int j = 0; j < n; ++j) acc += sc[j] * (double)v[(int64_t)j * ld + h * dh + c];
            ctx[h * dh + c] = (float)(acc / Z);
        }
    }
    free(sc);
}

/* AAN cumulative average, incremental form ("cumulative uniform
 * averaging ... computed based on the single last step"): the state is the
 * running sum C (R6); C <- fl(C + y); g = fl(C / t), t = 1, 2, ... (R7). */
void orc_aan_step(float *C, const float *y, int t, int d, float *g) {
    for (int k = 0; k < d; ++k) {
        C[k] = C[k] + y[k];
        g[k] = C[k] / (float)t;
    }
}

/* sigma(x) = 1/(1+exp(-x)), fp64 then rounded (R20). */
float orc_sigmoid(float x) { return (float)(1.0 / (1.0 + exp(-(double)x))); }
void orc_sigmoid_array(const float *x, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_sigmoid(x[i]);
}

/* Residual + LayerNorm of one row: out = LN(fl(x + z)) with z = delta, or, in the gate
 * form (gi != NULL; R8), z = fl(fl(sig_i * x) + fl(sig_f * delta)) where gi/gf are the
 * gate activations after the sigmoid. */
void orc_residual_ln(const float *x, const float *delta, const float *gi, const float *gf, int d,
                     const float *g, const float *b, float eps, float *out) {
    float *r = (float *)malloc(sizeof(float) * (size_t)d);
    for (int k = 0; k < d; ++k) {
        float z = delta[k];
        if (gi) {
            float iy = gi[k] * x[k];
            float fa = gf[k] * delta[k];
            z = iy + fa;
        }
        r[k] = x[k] + z;
    }
    orc_layernorm(r, d, g, b, eps, out);
    free(r);
}

/* Sinusoidal position encoding (P:L65 Vaswani recipe; R12):
 * PE[pos][2i] = sin(pos / 10000^(2i/d)), PE[pos][2i+1] = cos(same). */
void orc_pe(int pos, int d, float *out) {
    for (int i = 0; 2 * i < d; ++i) {
        double ang = (double)pos / pow(10000.0, (double)(2 * i) / (double)d);
        out[2 * i] = (float)sin(ang);
        if (2 * i + 1 < d) out[2 * i + 1] = (float)cos(ang);
    }
}

/* emb(id, pos) = fl(fl(E[id] * fl32(sqrt d)) + PE[pos]); id < 0 = zero vector
 * (the start symbol, R13).  Tied embedding E. */
void orc_embed_row(const float *E, int d, int id, int pos, float *out) {
    float r = (float)sqrt((double)d);
    float *pe = (float *)malloc(sizeof(float) * (size_t)d);
    orc_pe(pos, d, pe);
    for (int k = 0; k < d; ++k) {
        float e = id >= 0 ? E[(int64_t)id * d + k] * r : 0.0f;
        out[k] = e + pe[k];
    }
    free(pe);
}

static void embed(const orc_model *m, int id, int pos, float *out, float *pe_tmp) {
    (void)pe_tmp;
    orc_embed_row(m->E, m->c.d_model, id, pos, out);
}

/* ----------------------------------------------------- model assembly */
static int cfg_ok(const orc_cfg *c) {
    if (c->d_model <= 0 || c->d_ffn <= 0 || c->n_heads <= 0 || c->vocab <= 0) return 0;
    if (c->d_model % c->n_heads) return 0;
    if (c->enc_layers < 0 || c->dec_layers < 1) return 0;
    if (c->enc_layers > ORC_MAX_LAYERS || c->dec_layers > ORC_MAX_LAYERS) return 0;
    if (c->decoder != 0 && c->decoder != 1) return 0;
    if (c->aan_ffn_depth < 0 || c->aan_ffn_depth > 2) return 0;
    if (!(c->clip > 0.0f)) return 0;
    if (c->eos_id < 0 || c->eos_id >= c->vocab) return 0;
    return 1;
}

orc_model *orc_model_new(const orc_cfg *c) {
    if (!cfg_ok(c)) return NULL;
    orc_model *m = (orc_model *)calloc(1, sizeof(orc_model));
    m->c = *c;
    return m;
}

static void free_lin(orc_lin *l) { free(l->W); free(l->b); free(l->qW); }
static void free_ln(orc_ln *l) { free(l->g); free(l->b); }

void orc_model_free(orc_model *m) {
    if (!m) return;
    free(m->E); free(m->out_b); free(m->qE);
    for (int l = 0; l < ORC_MAX_LAYERS; ++l) {
        orc_enc_layer *e = &m->enc[l];
        free_lin(&e->q); free_lin(&e->k); free_lin(&e->v); free_lin(&e->o);
        free_lin(&e->f1); free_lin(&e->f2); free_ln(&e->ln1); free_ln(&e->ln2);
        orc_dec_layer *D = &m->dec[l];
        free_lin(&D->a1); free_lin(&D->a2); free_lin(&D->gi); free_lin(&D->gf);
        free_lin(&D->q); free_lin(&D->k); free_lin(&D->v); free_lin(&D->o);
        free_lin(&D->sq); free_lin(&D->sk); free_lin(&D->sv); free_lin(&D->so);
        free_lin(&D->f1); free_lin(&D->f2);
        free_ln(&D->ln1); free_ln(&D->ln2); free_ln(&D->ln3);
    }
    free(m);
}

static float *dup(const float *p, int64_t n) {
    float *q = (float *)malloc(sizeof(float) * (size_t)n);
    memcpy(q, p, sizeof(float) * (size_t)n);
    return q;
}

/* Resolve a manifest name to its slot.  Returns element count expected, or -1. */
static int64_t slot(orc_model *m, const char *name, float ***dst, orc_lin **lin_out) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, F = c->d_ffn;
    *lin_out = NULL;
    if (!strcmp(name, "emb.E")) { *dst = &m->E; return (int64_t)c->vocab * d; }
    if (!strcmp(name, "out.b")) { if (!c->out_bias) return -1; *dst = &m->out_b; return c->vocab; }
    int l = -1, n = 0;
    char rest[64];
    if (sscanf(name, "enc.%d.%63s%n", &l, rest, &n) == 2 && l >= 0 && l < c->enc_layers) {
        orc_enc_layer *e = &m->enc[l];
        struct { const char *nm; orc_lin *L; int out, in; } lt[] = {
            {"self.q", &e->q, d, d}, {"self.k", &e->k, d, d}, {"self.v", &e->v, d, d},
            {"self.o", &e->o, d, d}, {"ffn.1", &e->f1, F, d}, {"ffn.2", &e->f2, d, F}};
        for (size_t i = 0; i < sizeof(lt) / sizeof(lt[0]); ++i) {
            size_t ln = strlen(lt[i].nm);
            if (!strncmp(rest, lt[i].nm, ln) && rest[ln] == '.') {
                lt[i].L->out = lt[i].out; lt[i].L->in = lt[i].in; *lin_out = lt[i].L;
                if (!strcmp(rest + ln, ".W")) { *dst = &lt[i].L->W; return (int64_t)lt[i].out * lt[i].in; }
                if (!strcmp(rest + ln, ".b")) { *dst = &lt[i].L->b; return lt[i].out; }
                return -1;
            }
        }
        if (!strcmp(rest, "ln1.g")) { *dst = &e->ln1.g; return d; }
        if (!strcmp(rest, "ln1.b")) { *dst = &e->ln1.b; return d; }
        if (!strcmp(rest, "ln2.g")) { *dst = &e->ln2.g; return d; }
        if (!strcmp(rest, "ln2.b")) { *dst = &e->ln2.b; return d; }
        return -1;
    }
    if (sscanf(name, "dec.%d.%63s%n", &l, rest, &n) == 2 && l >= 0 && l < c->dec_layers) {
        orc_dec_layer *D = &m->dec[l];
        int aan = c->decoder == 1;
        struct { const char *nm; orc_lin *L; int out, in; int present; } lt[] = {
            {"aan.ffn.1", &D->a1, d, d, aan && c->aan_ffn_depth >= 1},
            {"aan.ffn.2", &D->a2, d, d, aan && c->aan_ffn_depth >= 2},
            {"aan.gate.i", &D->gi, d, d, aan && c->aan_gate},
            {"aan.gate.f", &D->gf, d, d, aan && c->aan_gate},
            {"self.q", &D->q, d, d, !aan}, {"self.k", &D->k, d, d, !aan},
            {"self.v", &D->v, d, d, !aan}, {"self.o", &D->o, d, d, !aan},
            {"src.q", &D->sq, d, d, 1}, {"src.k", &D->sk, d, d, 1},
            {"src.v", &D->sv, d, d, 1}, {"src.o", &D->so, d, d, 1},
            {"ffn.1", &D->f1, F, d, 1}, {"ffn.2", &D->f2, d, F, 1}};
        for (size_t i = 0; i < sizeof(lt) / sizeof(lt[0]); ++i) {
            size_t ln = strlen(lt[i].nm);
            if (!strncmp(rest, lt[i].nm, ln) && rest[ln] == '.' &&
                (!strcmp(rest + ln, ".W") || !strcmp(rest + ln, ".b"))) {
                if (!lt[i].present) return -1;
                lt[i].L->out = lt[i].out; lt[i].L->in = lt[i].in; *lin_out = lt[i].L;
                if (rest[ln + 1] == 'W') { *dst = &lt[i].L->W; return (int64_t)lt[i].out * lt[i].in; }
                *dst = &lt[i].L->b; return lt[i].out;
            }
        }
        orc_ln *lns[3] = {&D->ln1, &D->ln2, &D->ln3};
        for (int i = 0; i < 3; ++i) {
            char nm[16];
            snprintf(nm, sizeof nm, "ln%d.g", i + 1);
            if (!strcmp(rest, nm)) { *dst = &lns[i]->g; return d; }
            snprintf(nm, sizeof nm, "ln%d.b", i + 1);
            if (!strcmp(rest, nm)) { *dst = &lns[i]->b; return d; }
        }
    }
    return -1;
}

/* 0 ok, 2 = unknown name or wrong numel, 4 = after quantize. */
int orc_model_set(orc_model *m, const char *name, const float *data, int64_t numel) {
    if (m->quantized) return 4;
    float **dst = NULL; orc_lin *L = NULL;
    int64_t want = slot(m, name, &dst, &L);
    if (want < 0 || want != numel) return 2;
    free(*dst);
    *dst = dup(data, numel);
    return 0;
}

static int lin_ready(const orc_lin *l) { return l->W && l->b; }

/* One-time quantization of every parameter matrix: the memoized
 * quant(B^T) of P:L100-105.  Returns 0, or 4 if any parameter is missing. */
int orc_model_quantize(orc_model *m) {
    const orc_cfg *c = &m->c;
    float clip = c->clip;
    if (!m->E || (c->out_bias && !m->out_b)) return 4;
    for (int l = 0; l < c->enc_layers; ++l) {
        orc_enc_layer *e = &m->enc[l];
        orc_lin *ls[6] = {&e->q, &e->k, &e->v, &e->o, &e->f1, &e->f2};
        for (int i = 0; i < 6; ++i) if (!lin_ready(ls[i])) return 4;
        if (!e->ln1.g || !e->ln1.b || !e->ln2.g || !e->ln2.b) return 4;
    }
    for (int l = 0; l < c->dec_layers; ++l) {
        orc_dec_layer *D = &m->dec[l];
        if (c->decoder == 1) {
            if (c->aan_ffn_depth >= 1 && !lin_ready(&D->a1)) return 4;
            if (c->aan_ffn_depth >= 2 && !lin_ready(&D->a2)) return 4;
            if (c->aan_gate && (!lin_ready(&D->gi) || !lin_ready(&D->gf))) return 4;
        } else {
            if (!lin_ready(&D->q) || !lin_ready(&D->k) || !lin_ready(&D->v) || !lin_ready(&D->o)) return 4;
        }
        orc_lin *ls[6] = {&D->sq, &D->sk, &D->sv, &D->so, &D->f1, &D->f2};
        for (int i = 0; i < 6; ++i) if (!lin_ready(ls[i])) return 4;
        if (!D->ln1.g || !D->ln1.b || !D->ln2.g || !D->ln2.b || !D->ln3.g || !D->ln3.b) return 4;
    }
    int64_t nE = (int64_t)c->vocab * c->d_model;
    (void)clip;
    m->qE = (int16_t *)malloc(sizeof(int16_t) * (size_t)nE);
    qcodes(c, m->E, nE, m->qE);
#define QL(L) do { if ((L).W) { int64_t n_ = (int64_t)(L).out * (L).in; \
        (L).qW = (int16_t *)malloc(sizeof(int16_t) * (size_t)n_); qcodes(c, (L).W, n_, (L).qW); } } while (0)
    for (int l = 0; l < c->enc_layers; ++l) {
        orc_enc_layer *e = &m->enc[l];
        QL(e->q); QL(e->k); QL(e->v); QL(e->o); QL(e->f1); QL(e->f2);
    }
    for (int l = 0; l < c->dec_layers; ++l) {
        orc_dec_layer *D = &m->dec[l];
        QL(D->a1); QL(D->a2); QL(D->gi); QL(D->gf);
        QL(D->q); QL(D->k); QL(D->v); QL(D->o);
        QL(D->sq); QL(D->sk); QL(D->sv); QL(D->so); QL(D->f1); QL(D->f2);
    }
#undef QL
    m->quantized = 1;
    return 0;
}

/* ------------------------------------------------------------ encoder */
/* Encoder: x = emb(src, 0..S-1); per layer
 *   qkv = lin(Q(x)); ctx = attn; x = LN1(fl(x + lin(Q(ctx))));
 *   h = Q(ReLU(lin(Q(x)))); x = LN2(fl(x + lin(h))).
 * Then the source keys/values of every decoder layer: K_l = lin(Q(x); Wk_l),
 * V_l = lin(Q(x); Wv_l).  enc_out [S x d] and kv [L][2][S][d] may be NULL. */
int orc_encode(const orc_model *m, const int32_t *src, int S, float *enc_out, float *kv) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, F = c->d_ffn, H = c->n_heads;
    if (!m->quantized) return 4;
    for (int i = 0; i < S; ++i) if (src[i] < 0 || src[i] >= c->vocab) return 3;
    float *x = (float *)malloc(sizeof(float) * (size_t)S * d);
    float *Q = (float *)malloc(sizeof(float) * (size_t)S * d);
    float *Kt = (float *)malloc(sizeof(float) * (size_t)S * d);
    float *Vt = (float *)malloc(sizeof(float) * (size_t)S * d);
    float *ctx = (float *)malloc(sizeof(float) * d);
    float *o = (float *)malloc(sizeof(float) * d);
    float *r = (float *)malloc(sizeof(float) * d);
    float *h = (float *)malloc(sizeof(float) * F);
    int16_t *qa = (int16_t *)malloc(sizeof(int16_t) * (size_t)(F > d ? F : d));
    float *pe = (float *)malloc(sizeof(float) * d);
    for (int i = 0; i < S; ++i) embed(m, src[i], i, x + (int64_t)i * d, pe);
    for (int l = 0; l < c->enc_layers; ++l) {
        const orc_enc_layer *e = &m->enc[l];
        for (int i = 0; i < S; ++i) {
            qcodes(c, x + (int64_t)i * d, d, qa);
            lin1(c, &e->q, qa, Q + (int64_t)i * d);
            lin1(c, &e->k, qa, Kt + (int64_t)i * d);
            lin1(c, &e->v, qa, Vt + (int64_t)i * d);
        }
        for (int i = 0; i < S; ++i) {
            float *xi = x + (int64_t)i * d;
            orc_attention(Q + (int64_t)i * d, Kt, Vt, d, S, d, H, ctx);
            qcodes(c, ctx, d, qa);
            lin1(c, &e->o, qa, o);
            orc_residual_ln(xi, o, NULL, NULL, d, e->ln1.g, e->ln1.b, c->ln_eps, r);
            memcpy(xi, r, sizeof(float) * d);
            qcodes(c, xi, d, qa);
            lin1(c, &e->f1, qa, h);
            for (int k = 0; k < F; ++k) qa[k] = code1(c, h[k] > 0.0f ? h[k] : 0.0f);
            lin1(c, &e->f2, qa, o);
            orc_residual_ln(xi, o, NULL, NULL, d, e->ln2.g, e->ln2.b, c->ln_eps, r);
            memcpy(xi, r, sizeof(float) * d);
        }
    }
    if (enc_out) memcpy(enc_out, x, sizeof(float) * (size_t)S * d);
    if (kv) {
        for (int l = 0; l < c->dec_layers; ++l) {
            const orc_dec_layer *D = &m->dec[l];
            for (int i = 0; i < S; ++i) {
                qcodes(c, x + (int64_t)i * d, d, qa);
                lin1(c, &D->sk, qa, kv + (((int64_t)l * 2 + 0) * S + i) * d);
                lin1(c, &D->sv, qa, kv + (((int64_t)l * 2 + 1) * S + i) * d);
            }
            if (c->src_kv_bf16)
                for (int64_t k = 0; k < 2 * (int64_t)S * d; ++k)
                    kv[(int64_t)l * 2 * S * d + k] = orc_bf16(kv[(int64_t)l * 2 * S * d + k]);
        }
    }
    free(x); free(Q); free(Kt); free(Vt); free(ctx); free(o); free(r); free(h); free(qa); free(pe);
    return 0;
}

/* ------------------------------------------------------------ decoder */
typedef struct {
    int32_t *ids;        /* [T] model argmax at each step */
    int32_t *second;     /* [T] runner-up id */
    float *margin;       /* [T] top-1 minus top-2 logit (fp32 difference in double) */
    float *dec_out;      /* [T][d] decoder output of the last layer */
    float *layer_out;    /* [T][L][3][d] x1, x2, x3 of every layer */
    int8_t *out_codes;   /* [T][d] Q(dec_out): the output-layer A operand */
} orc_trace;

/* The decoder state of ONE hypothesis (one sentence for greedy decoding):
 * the AAN running sums C_l (R6; C_l = 0 before t = 1) or the self-attention
 * cache of positions 1..t. */
typedef struct {
    float *C;            /* [L][d] */
    float *Ks, *Vs;      /* [L][Tcap][d] (decoder == 0) */
    int Tcap;
} orc_dstate;

static void dstate_init(const orc_model *m, orc_dstate *s, int Tcap) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, L = c->dec_layers;
    s->Tcap = Tcap > 0 ? Tcap : 1;
    s->C = (float *)calloc((size_t)L * d, sizeof(float));
    s->Ks = s->Vs = NULL;
    if (c->decoder == 0) {
        s->Ks = (float *)calloc((size_t)L * s->Tcap * d, sizeof(float));
        s->Vs = (float *)calloc((size_t)L * s->Tcap * d, sizeof(float));
    }
}
static void dstate_copy(const orc_model *m, orc_dstate *dst, const orc_dstate *src) {
    const orc_cfg *c = &m->c;
    size_t n = (size_t)c->dec_layers * c->d_model;
    memcpy(dst->C, src->C, sizeof(float) * n);
    if (c->decoder == 0) {
        memcpy(dst->Ks, src->Ks, sizeof(float) * n * src->Tcap);
        memcpy(dst->Vs, src->Vs, sizeof(float) * n * src->Tcap);
    }
}
static void dstate_free(orc_dstate *s) { free(s->C); free(s->Ks); free(s->Vs); }

/* Scratch rows of one decoder step. */
typedef struct {
    float *y, *g, *a, *t1, *gi, *gf, *r, *x1, *x2, *ctx, *h, *pe, *qs;
    int16_t *qa, *qy;
} orc_scratch;

static void scratch_init(const orc_model *m, orc_scratch *w) {
    int d = m->c.d_model, F = m->c.d_ffn;
    float **f[] = {&w->y, &w->g, &w->a, &w->t1, &w->gi, &w->gf, &w->r, &w->x1, &w->x2,
                   &w->ctx, &w->pe, &w->qs};
    for (size_t i = 0; i < sizeof(f) / sizeof(f[0]); ++i) *f[i] = (float *)malloc(sizeof(float) * d);
    w->h = (float *)malloc(sizeof(float) * F);
    w->qa = (int16_t *)malloc(sizeof(int16_t) * (size_t)(F > d ? F : d));
    w->qy = (int16_t *)malloc(sizeof(int16_t) * (size_t)d);
}
static void scratch_free(orc_scratch *w) {
    free(w->y); free(w->g); free(w->a); free(w->t1); free(w->gi); free(w->gf); free(w->r);
    free(w->x1); free(w->x2); free(w->ctx); free(w->pe); free(w->qs); free(w->h); free(w->qa);
    free(w->qy);
}

/* One decoder step t of one hypothesis (A5-A8): input in_id (< 0: the start
 * symbol, R13) at position t-1; updates the state; the last layer's output is
 * left in w->y.  kv: the source keys/values [L][2][S][d] (orc_encode).
 * layer_out: optional [L][3][d] x1, x2, x3 of every layer. */
static void dec_step(const orc_model *m, const float *kv, int S, orc_dstate *st, int in_id,
                     int t, orc_scratch *w, float *layer_out) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, F = c->d_ffn, H = c->n_heads, L = c->dec_layers;
    float *y = w->y, *g = w->g, *a = w->a, *t1 = w->t1, *gi = w->gi, *gf = w->gf;
    float *x1 = w->x1, *x2 = w->x2, *ctx = w->ctx, *h = w->h, *qs = w->qs;
    int16_t *qa = w->qa, *qy = w->qy;
    /* A5: decoder input y = emb(id_{t-1}, t-1); zero embedding at t=1 (R13). */
    embed(m, in_id, t - 1, y, w->pe);
    for (int l = 0; l < L; ++l) {
        const orc_dec_layer *D = &m->dec[l];
        if (c->decoder == 1) {
            /* A6: AAN.  C <- fl(C + y); g = fl(C / t) (R6, R7). */
            orc_aan_step(st->C + (int64_t)l * d, y, t, d, g);
            if (c->aan_ffn_depth == 0) {
                memcpy(a, g, sizeof(float) * d);
            } else {
                qcodes(c, g, d, qa);
                lin1(c, &D->a1, qa, t1);
                if (c->aan_ffn_depth == 1) {
                    for (int k = 0; k < d; ++k) a[k] = t1[k] > 0.0f ? t1[k] : 0.0f;
                } else {
                    for (int k = 0; k < d; ++k) qa[k] = code1(c, t1[k] > 0.0f ? t1[k] : 0.0f);
                    lin1(c, &D->a2, qa, a);
                }
            }
            if (c->aan_gate) {
                /* Gate (R8): i = sig(W_i y + b_i), f = sig(W_f a + b_f), z = i*y + f*a. */
                qcodes(c, y, d, qy);
                lin1(c, &D->gi, qy, gi);
                qcodes(c, a, d, qa);
                lin1(c, &D->gf, qa, gf);
                orc_sigmoid_array(gi, d, gi);
                orc_sigmoid_array(gf, d, gf);
                orc_residual_ln(y, a, gi, gf, d, D->ln1.g, D->ln1.b, c->ln_eps, x1);
            } else {
                orc_residual_ln(y, a, NULL, NULL, d, D->ln1.g, D->ln1.b, c->ln_eps, x1);
            }
        } else {
            /* A6': self-attention over positions 1..t with a KV cache. */
            float *Kl = st->Ks + (int64_t)l * st->Tcap * d, *Vl = st->Vs + (int64_t)l * st->Tcap * d;
            qcodes(c, y, d, qy);
            lin1(c, &D->q, qy, qs);
            lin1(c, &D->k, qy, Kl + (int64_t)(t - 1) * d);
            lin1(c, &D->v, qy, Vl + (int64_t)(t - 1) * d);
            orc_attention(qs, Kl, Vl, d, t, d, H, ctx);
            qcodes(c, ctx, d, qa);
            lin1(c, &D->o, qa, a);
            orc_residual_ln(y, a, NULL, NULL, d, D->ln1.g, D->ln1.b, c->ln_eps, x1);
        }
        /* A7: source attention. */
        qcodes(c, x1, d, qa);
        lin1(c, &D->sq, qa, qs);
        if (S > 0) {
            orc_attention(qs, kv + ((int64_t)l * 2 + 0) * S * d, kv + ((int64_t)l * 2 + 1) * S * d,
                          d, S, d, H, ctx);
        } else {
            memset(ctx, 0, sizeof(float) * d);
        }
        qcodes(c, ctx, d, qa);
        lin1(c, &D->so, qa, a);
        orc_residual_ln(x1, a, NULL, NULL, d, D->ln2.g, D->ln2.b, c->ln_eps, x2);
        /* A8: FFN; ReLU output goes straight to int8 codes. */
        qcodes(c, x2, d, qa);
        lin1(c, &D->f1, qa, h);
        for (int k = 0; k < F; ++k) qa[k] = code1(c, h[k] > 0.0f ? h[k] : 0.0f);
        lin1(c, &D->f2, qa, a);
        orc_residual_ln(x2, a, NULL, NULL, d, D->ln3.g, D->ln3.b, c->ln_eps, y);
        if (layer_out) {
            float *dst = layer_out + (int64_t)l * 3 * d;
            memcpy(dst, x1, sizeof(float) * d);
            memcpy(dst + d, x2, sizeof(float) * d);
            memcpy(dst + 2 * d, y, sizeof(float) * d);
        }
    }
}

/* A9: tied output projection: logit_j = fmaf((float)acc_j, s, b_j)
 * with acc_j = sum_k Q(y)_k * Q(E)[j,k]; out_bias = 0: b_j = 0 (R14).
 * qy receives Q(y). */
static void out_logits(const orc_model *m, const float *y, int16_t *qy, float *logits) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, V = c->vocab;
    float s = code_scale(c);
    qcodes(c, y, d, qy);
    for (int j = 0; j < V; ++j) {
        int32_t acc = orc_dot_codes(c->arith, qy, m->qE + (int64_t)j * d, d);
        logits[j] = fmaf((float)acc, s, c->out_bias ? m->out_b[j] : 0.0f);
    }
}

/* Greedy decode of ONE sentence (beam 1, softmax skipped, "select the
 * output word with highest activation").
 * forced == NULL: free-running; stop at EOS (not emitted) or t == max_len (R16).
 * forced != NULL: teacher forcing for max_len steps; the input at step t >= 2
 * is forced[t-2]; every step's argmax is recorded in trace/out_ids.
 * Returns the number of ids written to out_ids, or <0 on error. */
static int decode_impl(const orc_model *m, const int32_t *src, int S, int max_len,
                       const int32_t *forced, const int32_t *sl, int n_sl, int32_t *out_ids,
                       orc_trace *tr);

int orc_decode_one(const orc_model *m, const int32_t *src, int S, int max_len,
                   const int32_t *forced, int32_t *out_ids, orc_trace *tr) {
    return decode_impl(m, src, S, max_len, forced, NULL, 0, out_ids, tr);
}

/* Greedy decode restricted to a vocabulary shortlist: the argmax runs
 * over the ids sl[0..n_sl) only (ascending, so the lowest id still wins ties, R15). */
int orc_decode_one_sl(const orc_model *m, const int32_t *src, int S, int max_len,
                      const int32_t *sl, int n_sl, int32_t *out_ids) {
    return decode_impl(m, src, S, max_len, NULL, sl, n_sl, out_ids, NULL);
}

static int decode_impl(const orc_model *m, const int32_t *src, int S, int max_len,
                       const int32_t *forced, const int32_t *sl, int n_sl, int32_t *out_ids,
                       orc_trace *tr) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, L = c->dec_layers, V = c->vocab;
    if (!m->quantized) return -4;
    if (max_len < 0) return -1;
    for (int i = 0; i < S; ++i) if (src[i] < 0 || src[i] >= V) return -3;
    if (forced) for (int i = 0; i + 1 < max_len; ++i) if (forced[i] < 0 || forced[i] >= V) return -3;
    float *kv = (float *)malloc(sizeof(float) * (size_t)L * 2 * (S > 0 ? S : 1) * d);
    if (S > 0) orc_encode(m, src, S, NULL, kv);
    orc_dstate st;
    dstate_init(m, &st, max_len);
    orc_scratch w;
    scratch_init(m, &w);
    float *logits = (float *)malloc(sizeof(float) * (size_t)V);
    int n_out = 0, prev = -1;
    for (int t = 1; t <= max_len; ++t) {
        int in_id = t == 1 ? -1 : (forced ? forced[t - 2] : prev);
        dec_step(m, kv, S, &st, in_id, t, &w,
                 tr && tr->layer_out ? tr->layer_out + (int64_t)(t - 1) * L * 3 * d : NULL);
        /* A9: argmax of the logits, softmax skipped; lowest j wins ties (R15). */
        out_logits(m, w.y, w.qy, logits);
        int best = -1, second = -1;
        float bv = 0.0f, sv = 0.0f;
        for (int u = 0; u < (sl ? n_sl : V); ++u) {
            int j = sl ? sl[u] : u;
            float lg = logits[j];
            if (best < 0 || lg > bv) { second = best; sv = bv; best = j; bv = lg; }
            else if (second < 0 || lg > sv) { second = j; sv = lg; }
        }
        if (tr) {
            int i = t - 1;
            if (tr->ids) tr->ids[i] = best;
            if (tr->second) tr->second[i] = second;
            if (tr->margin) tr->margin[i] = second >= 0 ? (float)((double)bv - (double)sv) : INFINITY;
            if (tr->dec_out) memcpy(tr->dec_out + (int64_t)i * d, w.y, sizeof(float) * d);
            if (tr->out_codes)
                for (int k = 0; k < d; ++k) tr->out_codes[(int64_t)i * d + k] = (int8_t)w.qy[k];
        }
        if (forced) {
            out_ids[n_out++] = best;
        } else {
            /* A10: EOS is not emitted and ends the sentence (R16). */
            if (best == c->eos_id) break;
            out_ids[n_out++] = best;
            prev = best;
        }
    }
    free(kv); free(logits);
    dstate_free(&st);
    scratch_free(&w);
    return n_out;
}

/* ------------------------------------------------------------ beam search */
/* log-softmax of one row of logits (readings R26-R27):
 * M = max_j l_j; Z = sum_j exp((double)l_j - M) in ascending j, fp64;
 * lse = fl32(M + log Z); log p_j = fl32(l_j - lse). */
float orc_logsumexp(const float *l, int n) {
    float M = l[0];
    for (int j = 1; j < n; ++j) if (l[j] > M) M = l[j];
    double Z = 0.0;
    for (int j = 0; j < n; ++j) Z += exp((double)l[j] - (double)M);
    return (float)((double)M + log(Z));
}

typedef struct {
    orc_dstate st;
    int32_t *toks;     /* [max_len] emitted ids */
    int len;
    float score;       /* sum of fp32 log-probabilities (R27) */
} orc_hyp;

/* Candidate order (R28): score desc, then logit desc, then hypothesis rank asc,
 * then id asc.  Returns 1 if candidate a ranks before b. */
static int cand_before(float sa, float la, int ka, int ja, float sb, float lb, int kb, int jb) {
    if (sa != sb) return sa > sb;
    if (la != lb) return la > lb;
    if (ka != kb) return ka < kb;
    return ja < jb;
}

/* Beam search of ONE sentence with beam size b (the b=2 systems of
 * Table 3 rows 6 and 12), in the plain textbook form:
 *   - step 1 expands the start hypothesis; every later step expands each live
 *     hypothesis k over log-softmax(logits) (R26);
 *   - a candidate (k, j) scores fl32(score_k + log p_j) (R27); the top
 *     b - (finished so far) candidates in the order of R28 are kept;
 *   - a kept candidate with j = EOS is set aside as finished (EOS not emitted);
 *     at t = max_len every kept candidate is finished;
 *   - the search ends when no live hypothesis remains;
 *   - the finished list is stably sorted by descending score (no length
 *     normalization).
 * Outputs up to b hypotheses: ids of hypothesis r at hyp_ids[r * max_len ...],
 * hyp_len[r], hyp_score[r].  Returns their number (0 when max_len == 0) or <0. */
int orc_beam_one(const orc_model *m, const int32_t *src, int S, int max_len, int b,
                 int32_t *hyp_ids, int32_t *hyp_len, float *hyp_score) {
    const orc_cfg *c = &m->c;
    int d = c->d_model, L = c->dec_layers, V = c->vocab;
    if (!m->quantized) return -4;
    if (max_len < 0 || b < 1 || b > V) return -1;
    for (int i = 0; i < S; ++i) if (src[i] < 0 || src[i] >= V) return -3;
    if (max_len == 0) return 0;
    float *kv = (float *)malloc(sizeof(float) * (size_t)L * 2 * (S > 0 ? S : 1) * d);
    if (S > 0) orc_encode(m, src, S, NULL, kv);
    orc_scratch w;
    scratch_init(m, &w);
    orc_hyp *live = (orc_hyp *)calloc((size_t)b, sizeof(orc_hyp));
    orc_hyp *next = (orc_hyp *)calloc((size_t)b, sizeof(orc_hyp));
    for (int k = 0; k < b; ++k) {
        dstate_init(m, &live[k].st, max_len);
        dstate_init(m, &next[k].st, max_len);
        live[k].toks = (int32_t *)calloc((size_t)max_len, sizeof(int32_t));
        next[k].toks = (int32_t *)calloc((size_t)max_len, sizeof(int32_t));
    }
    float *logits = (float *)malloc(sizeof(float) * (size_t)b * V);
    float *cand = (float *)malloc(sizeof(float) * (size_t)b * V);
    char *taken = (char *)malloc((size_t)b * V);
    int n_live = 1, n_fin = 0;
    live[0].len = 0;
    live[0].score = 0.0f;
    for (int t = 1; t <= max_len && n_live > 0; ++t) {
        /* expand every live hypothesis: logits, log-softmax, candidate scores */
        for (int k = 0; k < n_live; ++k) {
            int in_id = t == 1 ? -1 : live[k].toks[live[k].len - 1];
            dec_step(m, kv, S, &live[k].st, in_id, t, &w, NULL);
            float *lk = logits + (int64_t)k * V;
            out_logits(m, w.y, w.qy, lk);
            float lse = orc_logsumexp(lk, V);
            for (int j = 0; j < V; ++j) {
                float lp = lk[j] - lse;
                cand[(int64_t)k * V + j] = live[k].score + lp;
            }
        }
        /* keep the best b - n_fin candidates, in rank order (repeated scans) */
        int n_keep = b - n_fin, n_next = 0;
        memset(taken, 0, (size_t)n_live * V);
        for (int r = 0; r < n_keep; ++r) {
            int bk = -1, bj = -1;
            for (int k = 0; k < n_live; ++k)
                for (int j = 0; j < V; ++j) {
                    int64_t i = (int64_t)k * V + j;
                    if (taken[i]) continue;
                    if (bk < 0 || cand_before(cand[i], logits[i], k, j,
                                              cand[(int64_t)bk * V + bj], logits[(int64_t)bk * V + bj], bk, bj)) {
                        bk = k; bj = j;
                    }
                }
            taken[(int64_t)bk * V + bj] = 1;
            float sc = cand[(int64_t)bk * V + bj];
            const orc_hyp *p = &live[bk];
            if (bj == c->eos_id || t == max_len) {
                int32_t *dst = hyp_ids + (int64_t)n_fin * max_len;
                memcpy(dst, p->toks, sizeof(int32_t) * (size_t)p->len);
                int len = p->len;
                if (bj != c->eos_id) dst[len++] = bj;   /* EOS is not emitted (R16) */
                hyp_len[n_fin] = len;
                hyp_score[n_fin] = sc;
                ++n_fin;
            } else {
                orc_hyp *q = &next[n_next++];
                dstate_copy(m, &q->st, &p->st);
                memcpy(q->toks, p->toks, sizeof(int32_t) * (size_t)p->len);
                q->toks[p->len] = bj;
                q->len = p->len + 1;
                q->score = sc;
            }
        }
        orc_hyp *tmp = live; live = next; next = tmp;
        n_live = n_next;
    }
    /* stable insertion sort of the finished list by descending score */
    for (int i = 1; i < n_fin; ++i) {
        float sc = hyp_score[i];
        int len = hyp_len[i];
        int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)max_len);
        memcpy(row, hyp_ids + (int64_t)i * max_len, sizeof(int32_t) * (size_t)max_len);
        int j = i - 1;
        while (j >= 0 && hyp_score[j] < sc) {
            hyp_score[j + 1] = hyp_score[j];
            hyp_len[j + 1] = hyp_len[j];
            memcpy(hyp_ids + (int64_t)(j + 1) * max_len, hyp_ids + (int64_t)j * max_len,
                   sizeof(int32_t) * (size_t)max_len);
            --j;
        }
        hyp_score[j + 1] = sc;
        hyp_len[j + 1] = len;
        memcpy(hyp_ids + (int64_t)(j + 1) * max_len, row, sizeof(int32_t) * (size_t)max_len);
        free(row);
    }
    for (int k = 0; k < b; ++k) {
        dstate_free(&live[k].st); dstate_free(&next[k].st);
        free(live[k].toks); free(next[k].toks);
    }
    free(live); free(next); free(logits); free(cand); free(taken); free(kv);
    scratch_free(&w);
    return n_fin;
}

/* Beam search of n independent sentences (OpenMP over sentences, timing only).
 * Sentence i's hypotheses occupy hyp_ids[b * out_off[i] + r * max_len[i] ...],
 * hyp_len / hyp_score [i * b + r], n_hyp[i]; out_off = prefix sum of max_len. */
int orc_beam_many(const orc_model *m, const int32_t *src_ids, const int64_t *src_off, int n,
                  const int32_t *max_len, int b, int32_t *hyp_ids, int32_t *hyp_len,
                  float *hyp_score, int32_t *n_hyp, int nthreads) {
    int64_t *oo = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    oo[0] = 0;
    for (int i = 0; i < n; ++i) oo[i + 1] = oo[i] + max_len[i];
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int i = 0; i < n; ++i) {
        int r = orc_beam_one(m, src_ids + src_off[i], (int)(src_off[i + 1] - src_off[i]), max_len[i],
                             b, hyp_ids + (int64_t)b * oo[i], hyp_len + (int64_t)i * b,
                             hyp_score + (int64_t)i * b);
        if (r < 0) err = -r; else n_hyp[i] = r;
    }
    free(oo);
    return err;
}

/* Decode n independent sentences (rows are independent: static scales,
 * P:L94), parallel over sentences with OpenMP for timing only.  Sentence i's
 * ids go to out_ids[out_off[i] ...], out_off = exclusive prefix sum of max_len.
 * nthreads <= 0: library default.  Returns 0 or a status code. */
int orc_decode_many(const orc_model *m, const int32_t *src_ids, const int64_t *src_off, int n,
                    const int32_t *max_len, int32_t *out_ids, int32_t *out_len, int nthreads) {
    int64_t *oo = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    oo[0] = 0;
    for (int i = 0; i < n; ++i) oo[i + 1] = oo[i] + max_len[i];
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int i = 0; i < n; ++i) {
        int r = orc_decode_one(m, src_ids + src_off[i], (int)(src_off[i + 1] - src_off[i]),
                               max_len[i], NULL, out_ids + oo[i], NULL);
        if (r < 0) err = -r; else out_len[i] = r;
    }
    free(oo);
    return err;
}

/* ------------------------------------------------------------ shortlist (F2) */
/* Vocabulary shortlist of one batch ("the union of the 100 most frequent target words and
 * the 100 most probable translations for every source word in a batch"):
 *   freq[0..n_freq)                      the most frequent target ids (in frequency order)
 *   lex[s * k_lex + 0..k_lex)            the most probable translations of source id s
 * shortlist = freq ∪ {lex[s][k] : s a source id of the batch} ∪ {EOS, UNK}, deduplicated,
 * ascending.  Ids outside [0, V) are ignored.  Writes out[0..count) (capacity V), returns count. */
int orc_build_shortlist(int V, const int32_t *freq, int n_freq, const int32_t *lex, int k_lex,
                        const int32_t *src_ids, int64_t n_src, int eos, int unk, int32_t *out) {
    char *in = (char *)calloc((size_t)V, 1);
    for (int i = 0; i < n_freq; ++i) if (freq[i] >= 0 && freq[i] < V) in[freq[i]] = 1;
    for (int64_t t = 0; t < n_src; ++t) {
        int s = src_ids[t];
        if (s < 0 || s >= V) continue;
        for (int k = 0; k < k_lex; ++k) {
            int j = lex[(int64_t)s * k_lex + k];
            if (j >= 0 && j < V) in[j] = 1;
        }
    }
    if (eos >= 0 && eos < V) in[eos] = 1;
    if (unk >= 0 && unk < V) in[unk] = 1;
    int n = 0;
    for (int j = 0; j < V; ++j) if (in[j]) out[n++] = j;
    free(in);
    return n;
}

/* orc_decode_many with every sentence restricted to the same shortlist (one batch). */
int orc_decode_many_sl(const orc_model *m, const int32_t *src_ids, const int64_t *src_off, int n,
                       const int32_t *max_len, const int32_t *sl, int n_sl, int32_t *out_ids,
                       int32_t *out_len, int nthreads) {
    int64_t *oo = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    oo[0] = 0;
    for (int i = 0; i < n; ++i) oo[i + 1] = oo[i] + max_len[i];
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int i = 0; i < n; ++i) {
        int r = orc_decode_one_sl(m, src_ids + src_off[i], (int)(src_off[i + 1] - src_off[i]),
                                  max_len[i], sl, n_sl, out_ids + oo[i]);
        if (r < 0) err = -r; else out_len[i] = r;
    }
    free(oo);
    return err;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------ batcher */
/* Length-sorted word-budget batching ("sorted by source length ...
 * batch based on number of words ... at least 384 words"; R17).
 * Stable sort ascending by (S_i, i); append sentences while the batch holds
 * fewer than `budget` words; close it once it holds >= budget words.
 * Returns 0, or 1 for budget < 1 / n < 0. */
int orc_batch_by_words(const int32_t *len, int n, int budget, int32_t *order, int32_t *off,
                       int32_t *n_batches) {
    if (budget < 1 || n < 0) return 1;
    for (int i = 0; i < n; ++i) order[i] = i;
    /* insertion sort: obviously stable */
    for (int i = 1; i < n; ++i) {
        int32_t v = order[i];
        int j = i - 1;
        while (j >= 0 && len[order[j]] > len[v]) { order[j + 1] = order[j]; --j; }
        order[j + 1] = v;
    }
    int nb = 0;
    int64_t words = 0;
    off[0] = 0;
    for (int i = 0; i < n; ++i) {
        words += len[order[i]];
        if (words >= budget) { off[++nb] = i + 1; words = 0; }
    }
    if (n > 0 && off[nb] != n) off[++nb] = n;
    *n_batches = nb;
    return 0;
}

/* ---------------------------------------------------- size arithmetic */
/* Parameter count of a Table-1 student: tied embedding V*d
 * (P:L31), 6+6 layers, biases, LayerNorm gain/bias, output bias. */
int64_t orc_param_count(const orc_cfg *c) {
    int64_t d = c->d_model, F = c->d_ffn, V = c->vocab;
    int64_t lin_dd = d * d + d;
    int64_t ffn = (F * d + F) + (d * F + d);
    int64_t enc = 4 * lin_dd + ffn + 2 * 2 * d;
    int64_t self_blk;
    if (c->decoder == 1)
        self_blk = (c->aan_ffn_depth >= 1 ? lin_dd : 0) + (c->aan_ffn_depth >= 2 ? lin_dd : 0) +
                   (c->aan_gate ? 2 * lin_dd : 0);
    else
        self_blk = 4 * lin_dd;
    int64_t dec = self_blk + 4 * lin_dd + ffn + 3 * 2 * d;
    return V * d + c->enc_layers * enc + c->dec_layers * dec + (c->out_bias ? V : 0);
}
