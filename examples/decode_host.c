/* decode_host.c -- a plain C client of libfwbf_b200.so (no CUDA, no Python):
 * the binding a maintainer of a compiled caller would write.
 *
 *   decode_host OFFSETS_FILE Y_FILE N B P ALPHA KMAX > results
 *
 * OFFSETS_FILE: the circulant first row (int32, ascending); Y_FILE: B*N float32
 * channel values.  Prints one line per frame: iterations flags z-words(hex).
 * Build: gcc -O2 -I include examples/decode_host.c -L paper_1206_3362_b200
 *        -lfwbf_b200 -Wl,-rpath,$PWD/paper_1206_3362_b200 -o decode_host        */
#include <stdio.h>
#include <stdlib.h>

#include "fwbf_b200.h"

static void *slurp(const char *path, size_t *len) {
  FILE *f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *len = (size_t)ftell(f);
  fseek(f, 0, SEEK_SET);
  void *buf = malloc(*len ? *len : 1);
  if (fread(buf, 1, *len, f) != *len) { free(buf); buf = NULL; }
  fclose(f);
  return buf;
}

int main(int argc, char **argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: %s OFFSETS Y N B P ALPHA KMAX\n", argv[0]);
    return 2;
  }
  size_t olen = 0, ylen = 0;
  int32_t *offs = (int32_t *)slurp(argv[1], &olen);
  float *y = (float *)slurp(argv[2], &ylen);
  const int n = atoi(argv[3]), B = atoi(argv[4]);
  if (!offs || !y || ylen != (size_t)n * B * sizeof(float)) {
    fprintf(stderr, "bad inputs\n");
    return 2;
  }
  fwbf_code_desc d = {0};
  d.n_cols = n;
  d.n_rows = n;
  d.circulant = 1;
  d.n_offsets = (int32_t)(olen / sizeof(int32_t));
  d.offsets = offs;
  fwbf_code *code = NULL;
  if (fwbf_code_create(&d, 0, &code) != FWBF_OK) {
    fprintf(stderr, "code_create: %s\n", fwbf_last_error());
    return 1;
  }
  fwbf_params p = {0};
  p.algorithm = FWBF_ALG_FWBF;
  p.weight_mode = FWBF_WEIGHTS_IMWBF;
  p.alpha = atof(argv[6]);
  p.k_max = atoi(argv[7]);
  p.lam = 1;
  p.block_len_p = atoi(argv[5]);
  p.stall = FWBF_STALL_FLIP_GLOBAL_MAX;
  p.mlp_threshold = 1;
  const int zw = (n + 31) / 32;
  uint32_t *z = (uint32_t *)calloc((size_t)B * zw, 4);
  int32_t *it = (int32_t *)calloc((size_t)B, 4);
  uint8_t *fl = (uint8_t *)calloc((size_t)B, 1);
  int64_t cnt[FWBF_NCOUNTERS] = {0};
  if (fwbf_decode_host_f32(code, &p, y, B, n, z, zw, it, fl, cnt, 0) != FWBF_OK) {
    fprintf(stderr, "decode: %s\n", fwbf_last_error());
    return 1;
  }
  for (int f = 0; f < B; ++f) {
    printf("%d %d", it[f], fl[f]);
    for (int w = 0; w < zw; ++w) printf(" %08x", z[(size_t)f * zw + w]);
    printf("\n");
  }
  fprintf(stderr, "frames %lld word errors %lld\n", (long long)cnt[FWBF_CNT_FRAMES],
          (long long)cnt[FWBF_CNT_WORD_ERRORS]);
  fwbf_code_destroy(code);
  return 0;
}
