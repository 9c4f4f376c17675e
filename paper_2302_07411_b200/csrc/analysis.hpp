// Row f4: the reference's statistical analysis and its two
// image tools (analysis.cpp:51-361, capi.cpp:109-141, 335-383).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace cveb {

// One square frame loaded from a P6 image or a CVE1 container (load_frame_any,
// capi.cpp:109-121).
struct HostFrame {
  uint32_t side = 0, orig_width = 0, orig_height = 0;
  std::vector<uint8_t> px;
};
HostFrame load_frame_any(const char* path, uint32_t frame_index);

// GPU reductions (stats.cu) over nbytes of interleaved RGB24: d_hist[c*256+v]
// (768 counters, zeroed here) and, with d_b, d_diff = {differing positions
// per channel, sum |a-b| per channel}.  Ordered on stream s.
void launch_frame_stats(const uint8_t* d_a, const uint8_t* d_b, uint64_t nbytes,
                        unsigned long long* d_hist, unsigned long long* d_diff,
                        cudaStream_t s);

// cve_analyze: the key=value report (csv == false) or the CSV table, with
// the histograms and NPCR/UACI counts taken on `device`.
std::string analyze(const HostFrame& frame, const HostFrame* second, uint32_t samples,
                    uint64_t seed, bool csv, int device);

struct CropBlock {
  uint32_t x = 0, y = 0, side = 0;
  uint8_t fill = 0;
};
// cve_add_noise_file / cve_crop_file: every frame of a CVE1 container, or the
// single square P6 image, rewritten.
void add_noise_file(const char* in_path, const char* out_path, double rate, uint64_t seed);
void crop_file(const char* in_path, const char* out_path, const std::vector<CropBlock>& blocks);

}  // namespace cveb
