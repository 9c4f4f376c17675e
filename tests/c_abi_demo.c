/* A reference-style C caller of libcve_b200.so: the same calls a program
 * linked against the reference's libcve.so makes (cve.h), compiled as C99
 * against include/cve_b200.h.  Used by tests/test_capi_host.py (CPU: header
 * and link check, no-GPU failure mode) and tests/test_gpu_parity.py (GPU:
 * round trip and ciphertext digest).
 *
 *   argv[1]: key hex (PLCM or LASM);  prints "ok <xor of all ciphertext bytes>" on success,
 *   "nogpu <status>" when the cipher cannot be created. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cve_b200.h"

int main(int argc, char** argv) {
  const char* key = argc > 1 ? argv[1]
                             : "005f633937dd9abf3f93ba8c762f1bd43fb8560e3cdd9aef3f7c74d008a265d13f";
  cve_map_kind kind;
  if (cve_key_validate(key, &kind) != CVE_OK || (kind != CVE_MAP_PLCM && kind != CVE_MAP_LASM)) {
    printf("badkey %s\n", cve_last_error());
    return 2;
  }
  char fresh[80];
  if (cve_key_generate(CVE_MAP_PLCM, fresh, sizeof fresh) != CVE_OK || strlen(fresh) != 66) {
    printf("keygen failed\n");
    return 2;
  }
  if (strcmp(cve_status_message(CVE_ERROR_MISMATCH), "") == 0) return 2;

  cve_cipher* c = NULL;
  cve_status st = cve_cipher_create(key, 8, 5, 1, &c);
  if (st != CVE_OK) {
    printf("nogpu %d\n", (int)st);
    return 0;
  }
  const uint32_t side = 96;
  const size_t n = (size_t)side * side * 3;
  uint8_t* px = (uint8_t*)malloc(n);
  uint8_t* orig = (uint8_t*)malloc(n);
  for (size_t i = 0; i < n; ++i) orig[i] = px[i] = (uint8_t)(i * 2654435761u >> 24);
  if (cve_cipher_encrypt_frame(c, px, side) != CVE_OK) return 3;
  unsigned x = 0;
  for (size_t i = 0; i < n; ++i) x ^= (unsigned)px[i] << (8 * (i & 3));
  uint64_t seeds = 0;
  cve_cipher_seeds_drawn(c, &seeds);
  /* side % workers != 0: MISMATCH after the seed draw (reference order) */
  if (cve_cipher_encrypt_frame(c, px, 97) != CVE_ERROR_MISMATCH) return 4;
  cve_cipher_destroy(c);

  cve_cipher* d = NULL;
  if (cve_cipher_create(key, 8, 5, 0, &d) != CVE_OK) return 5;
  /* decrypt the ciphertext with a fresh handle: frame 0 again */
  uint8_t* ct = (uint8_t*)malloc(n);
  memcpy(ct, px, n);
  if (cve_cipher_decrypt_frame(d, ct, side) != CVE_OK) return 6;
  if (memcmp(ct, orig, n) != 0) {
    printf("roundtrip mismatch\n");
    return 7;
  }
  cve_cipher_destroy(d);

  /* the reference's sweep and bench entry points through its option structs */
  cve_sweep_options sw;
  memset(&sw, 0, sizeof sw);
  sw.key_hex = key;
  sw.synth_side = 32;
  sw.workers = 2;
  sw.max_rounds = 2;
  sw.seed = 5;
  char* csv = NULL;
  if (cve_sweep_rounds(&sw, &csv) != CVE_OK || csv == NULL) return 8;
  if (strncmp(csv, "round,npcr_r,", 13) != 0) return 9;
  unsigned lines = 0;
  for (const char* q = csv; *q; ++q) lines += *q == '\n';
  cve_string_free(csv);
  if (lines != 4) return 10; /* header + rounds 0..2 */
  const uint32_t sides[1] = {32};
  cve_bench_video_options bv;
  memset(&bv, 0, sizeof bv);
  bv.key_hex = key;
  bv.sides = sides;
  bv.side_len = 1;
  bv.workers = 2;
  bv.frames = 3;
  csv = NULL;
  if (cve_bench_video(&bv, &csv) != CVE_OK || csv == NULL) return 11;
  if (strncmp(csv, "map,side,workers,rounds,frames,fps,", 35) != 0) return 12;
  cve_string_free(csv);
  sw.synth_side = 33; /* not divisible by 2 workers */
  if (cve_sweep_rounds(&sw, &csv) != CVE_ERROR_MISMATCH) return 13;
  printf("ok %08x seeds=%llu\n", x, (unsigned long long)seeds);
  free(px);
  free(orig);
  free(ct);
  return 0;
}
