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
  printf("ok %08x seeds=%llu\n", x, (unsigned long long)seeds);
  free(px);
  free(orig);
  free(ct);
  return 0;
}
