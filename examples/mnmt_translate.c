/* mnmt_translate.c — a plain C client of the libmnmt ABI (include/mnmt.h), no Python involved.
 *
 * usage: mnmt_translate <weights.bin> <sentences.bin> d_model d_ffn n_heads layers vocab
 *                       decoder aan_ffn_depth aan_gate word_budget [shortlist.bin]
 *
 *   weights.bin    records {int32 name_len, name bytes, int64 numel, float32[numel]} — every
 *                  parameter of the manifest (DESIGN.md §1 / SURVEY §8(b)), W row-major [out][in]
 *   sentences.bin  {int32 n, int64 offsets[n+1], int32 ids[offsets[n]], int32 max_len[n]}
 *   shortlist.bin  optional {int32 n_freq, int32 freq[n_freq], int32 k_lex, int32 lex[vocab*k_lex]}
 *
 * Prints one line per sentence (input order): the decoded target ids.  Exit status: 0 on
 * success, otherwise the mnmt_status of the failing call with mnmt_last_error() on stderr
 * (nonzero exit with a one-line diagnostic). */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mnmt.h"

static int die(mnmt_status s, const char* what) {
  fprintf(stderr, "mnmt_translate: %s failed (status %d): %s\n", what, (int)s, mnmt_last_error());
  return s ? (int)s : 1;
}

static void* read_all(const char* path, long* size) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *size = ftell(f);
  fseek(f, 0, SEEK_SET);
  void* buf = malloc(*size > 0 ? (size_t)*size : 1);
  if (buf && fread(buf, 1, (size_t)*size, f) != (size_t)*size) { free(buf); buf = NULL; }
  fclose(f);
  return buf;
}

int main(int argc, char** argv) {
  if (argc < 12) {
    fprintf(stderr, "usage: %s weights.bin sentences.bin d F H L V decoder depth gate budget [shortlist.bin]\n", argv[0]);
    return 1;
  }
  mnmt_config cfg;
  mnmt_config_default(&cfg, atoi(argv[3]), atoi(argv[4]), atoi(argv[5]));
  cfg.enc_layers = cfg.dec_layers = atoi(argv[6]);
  cfg.vocab = atoi(argv[7]);
  cfg.decoder = atoi(argv[8]);
  cfg.aan_ffn_depth = atoi(argv[9]);
  cfg.aan_gate = atoi(argv[10]);
  const int budget = atoi(argv[11]);
  mnmt_model* m = NULL;
  mnmt_status s;
  if ((s = mnmt_model_create(&cfg, 0, &m)) != MNMT_OK) return die(s, "mnmt_model_create");

  long wsize = 0;
  char* w = (char*)read_all(argv[1], &wsize);
  if (!w) { fprintf(stderr, "mnmt_translate: cannot read %s\n", argv[1]); return 1; }
  for (long p = 0; p < wsize;) {
    int32_t len;
    int64_t numel;
    char name[256];
    memcpy(&len, w + p, 4);
    p += 4;
    if (len <= 0 || len >= (int32_t)sizeof name) { fprintf(stderr, "bad record\n"); return 1; }
    memcpy(name, w + p, (size_t)len);
    name[len] = 0;
    p += len;
    memcpy(&numel, w + p, 8);
    p += 8;
    if ((s = mnmt_model_set_param(m, name, (const float*)(w + p), numel)) != MNMT_OK)
      return die(s, name);
    p += numel * 4;
  }
  free(w);
  if ((s = mnmt_model_quantize(m)) != MNMT_OK) return die(s, "mnmt_model_quantize");

  long ssize = 0;
  char* sb = (char*)read_all(argv[2], &ssize);
  if (!sb) { fprintf(stderr, "mnmt_translate: cannot read %s\n", argv[2]); return 1; }
  int32_t n;
  memcpy(&n, sb, 4);
  const int64_t* off = (const int64_t*)(sb + 4);
  const int32_t* ids = (const int32_t*)(sb + 4 + 8 * (size_t)(n + 1));
  const int32_t* max_len = ids + off[n];
  int64_t cap = 0;
  for (int i = 0; i < n; ++i) cap += max_len[i];
  int32_t* out = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  int32_t* out_len = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));

  uint32_t flags = 0;
  if (argc > 12) {   /* batch vocabulary shortlist */
    long lsize = 0;
    char* lb = (char*)read_all(argv[12], &lsize);
    if (!lb) { fprintf(stderr, "mnmt_translate: cannot read %s\n", argv[12]); return 1; }
    int32_t n_freq, k_lex;
    memcpy(&n_freq, lb, 4);
    const int32_t* freq = (const int32_t*)(lb + 4);
    memcpy(&k_lex, lb + 4 + 4 * (size_t)n_freq, 4);
    const int32_t* lex = (const int32_t*)(lb + 8 + 4 * (size_t)n_freq);
    if ((s = mnmt_model_set_shortlist(m, freq, n_freq, lex, k_lex)) != MNMT_OK)
      return die(s, "mnmt_model_set_shortlist");
    free(lb);
    flags |= MNMT_SHORTLIST;
  }
  if ((s = mnmt_translate(m, ids, off, n, max_len, budget, out, cap, out_len, flags, NULL)) != MNMT_OK)
    return die(s, "mnmt_translate");
  int64_t o = 0;
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < out_len[i]; ++k) printf(k ? " %d" : "%d", out[o + k]);
    printf("\n");
    o += max_len[i];
  }
  mnmt_stats st;
  if (mnmt_get_stats(m, &st) == MNMT_OK)
    fprintf(stderr, "mnmt_translate: %lld target words, %lld decoder steps, %lld kernel launches\n",
            (long long)st.target_words, (long long)st.decode_steps, (long long)st.gpu_launches);
  free(out);
  free(out_len);
  free(sb);
  mnmt_model_destroy(m);
  return 0;
}
