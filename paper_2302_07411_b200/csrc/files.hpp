// File pipelines (P6 / directory / raw <-> CVE1) on the GPU engine.
#pragma once

#include <cstdint>

namespace cveb {

// Resolved cve_io_options (defaults applied: workers 8, rounds 5, fps 20).
struct FileOptions {
  uint32_t workers = 8;
  uint32_t rounds = 5;
  uint16_t fps = 20;
  uint32_t raw_width = 0, raw_height = 0;
};

void encrypt_file(const char* key_hex, const FileOptions& opt, const char* in_path,
                  const char* out_path, int device);
// format: 0 auto (P6 / directory of P6), 1 P6, 2 raw RGB24.  opt may be null
// (follow the container header).
void decrypt_file(const char* key_hex, const FileOptions* opt, int format,
                  const char* in_path, const char* out_path, int device);

// Reference cve_nist_export: byte_count generator bytes split over the
// workers derived from the key, written worker after worker.
void keystream_export(const char* key_hex, uint32_t workers, uint64_t byte_count,
                      const char* out_path, int device);

}  // namespace cveb
