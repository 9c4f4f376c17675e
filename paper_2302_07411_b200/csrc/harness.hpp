// The reference library's timing and sweep entry points (cve.h:153-206,
// capi.cpp:417-505, bench.cpp:60-315) over THIS engine: the same options,
// defaults, CSV schemas and error behaviour, with the B200 generator and
// rounds doing the work that is timed.  cve_sweep_rounds is deterministic and
// byte-identical to the reference's; the three bench tables hold this
// engine's own timings in the reference's columns.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "analysis.hpp"
#include "keying.hpp"

namespace cveb {

// Synthetic inputs of the reference's harness (synth.cpp:12-100): uniform
// noise from mt19937_64 bytes, and the smooth "natural" test image.
HostFrame noise_frame(uint32_t side, uint64_t seed);
HostFrame natural_frame(uint32_t side, uint64_t seed);

// bench.cpp:60-123.  One row per worker count: `iterations` map iterations in
// total, split across the workers' generators, which advance together on the
// GPU (derivation and warm-up outside the timed window, no copy to the host).
std::string bytegen_table(const Key& key, const std::vector<uint32_t>& counts,
                          uint64_t iterations, int device);
// bench.cpp:125-184: confusion-only and diffusion-only transforms of noise
// images, timed on the host clock (the diffusion column includes generation).
std::string phases_table(const Key& key, uint32_t side, uint32_t workers, uint32_t rounds,
                         uint32_t images, int device);
// bench.cpp:186-257: per-frame cve_cipher_encrypt_frame-equivalent calls on
// noise frames.  bytegen_mean_ms = generator kernels' device time per frame;
// confuse_mean_ms = the fused confusion+diffusion round kernels' device time;
// diffuse_mean_ms = 0 (there is no separate diffusion pass to time).
std::string video_table(const Key& key, const std::vector<uint32_t>& sides, uint32_t workers,
                        uint32_t rounds, uint32_t frames, uint16_t fps, int device);
// bench.cpp:259-315.
std::string sweep_table(const Key& key, const HostFrame& plain, uint32_t workers,
                        uint32_t max_rounds, uint64_t seed, int device);

}  // namespace cveb
