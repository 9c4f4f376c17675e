#include "harness.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <optional>
#include <random>

#include "engine.hpp"

namespace cveb {
namespace {

using Clock = std::chrono::steady_clock;

double elapsed_ms(Clock::time_point from) {
  return std::chrono::duration<double, std::milli>(Clock::now() - from).count();
}

const char* map_label(MapKind k) { return k == MapKind::Plcm ? "plcm" : "lasm"; }

// "%.3f" / "%.6f" fields, as the reference prints them (bench.cpp:29-39)
void put_fixed(std::string& out, double v, int digits) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.*f", digits, v);
  out += ',';
  out += buf;
}

void put_uint(std::string& out, uint64_t v, bool comma = true) {
  if (comma) out += ',';
  out += std::to_string(v);
}

struct Spread {
  double total = 0, lo = std::numeric_limits<double>::infinity(),
         hi = -std::numeric_limits<double>::infinity();
  uint64_t count = 0;
  void take(double v) {
    total += v;
    lo = std::min(lo, v);
    hi = std::max(hi, v);
    ++count;
  }
  double mean() const { return count ? total / double(count) : 0.0; }
};

constexpr double kMiB = 1024.0 * 1024.0;

std::vector<HostFrame> noise_pool(uint32_t side, uint32_t count, uint64_t seed0) {
  std::vector<HostFrame> pool;
  pool.reserve(count);
  for (uint32_t i = 0; i < count; ++i) pool.push_back(noise_frame(side, seed0 + i));
  return pool;
}

// Pearson correlation of channel `ch` between two frames at the same
// positions, with the reference's two passes and summation order
// (analysis.cpp:124-165), so the printed digits agree.
std::optional<double> channel_correlation(const uint8_t* a, const uint8_t* b, size_t pixels,
                                          int ch) {
  const double n = double(pixels);
  double ma = 0, mb = 0;
  for (size_t i = 0; i < pixels; ++i) {
    ma += a[3 * i + ch];
    mb += b[3 * i + ch];
  }
  ma /= n;
  mb /= n;
  double cov = 0, va = 0, vb = 0;
  for (size_t i = 0; i < pixels; ++i) {
    const double da = double(a[3 * i + ch]) - ma;
    const double db = double(b[3 * i + ch]) - mb;
    cov += da * db;
    va += da * da;
    vb += db * db;
  }
  if (va == 0.0 || vb == 0.0) return std::nullopt;
  return (cov / n) / (std::sqrt(va / n) * std::sqrt(vb / n));
}

// NPCR / UACI of one channel in percent (analysis.cpp:203-220).
void channel_diff(const uint8_t* a, const uint8_t* b, size_t pixels, int ch, double& npcr,
                  double& uaci) {
  uint64_t changed = 0, magnitude = 0;
  for (size_t i = 0; i < pixels; ++i) {
    const int d = int(a[3 * i + ch]) - int(b[3 * i + ch]);
    changed += d != 0;
    magnitude += uint64_t(d < 0 ? -d : d);
  }
  npcr = 100.0 * double(changed) / double(pixels);
  uaci = 100.0 * double(magnitude) / (255.0 * double(pixels));
}

}  // namespace

HostFrame noise_frame(uint32_t side, uint64_t seed) {
  if (side == 0) raise(Errc::invalid_argument, "frame side must be >= 1");
  HostFrame f;
  f.side = f.orig_width = f.orig_height = side;
  f.px.resize(size_t(side) * side * 3);
  std::mt19937_64 rng(seed);
  // eight bytes per draw, least significant first; the last draw is partial
  for (size_t at = 0; at < f.px.size(); at += 8) {
    const uint64_t v = rng();
    const size_t take = std::min<size_t>(8, f.px.size() - at);
    for (size_t k = 0; k < take; ++k) f.px[at + k] = uint8_t(v >> (8 * k));
  }
  return f;
}

HostFrame natural_frame(uint32_t side, uint64_t seed) {
  if (side == 0) raise(Errc::invalid_argument, "frame side must be >= 1");
  HostFrame f;
  f.side = f.orig_width = f.orig_height = side;
  f.px.resize(size_t(side) * side * 3);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
  // per channel: two sinusoid products, drawn in this order (synth.cpp:36-46)
  struct Wave {
    double f_row, f_col, f_diag, ph_row, ph_col, ph_diag, amp_rc, amp_diag;
  } wave[3];
  for (Wave& w : wave) {
    w.f_row = 1.0 + 3.0 * u01(rng);
    w.f_col = 1.0 + 3.0 * u01(rng);
    w.f_diag = 0.5 + 2.0 * u01(rng);
    w.ph_row = two_pi * u01(rng);
    w.ph_col = two_pi * u01(rng);
    w.ph_diag = two_pi * u01(rng);
    w.amp_rc = 50.0 + 25.0 * u01(rng);
    w.amp_diag = 30.0 + 20.0 * u01(rng);
  }
  uint8_t* px = f.px.data();
  for (uint32_t r = 0; r < side; ++r) {
    const double u = double(r) / double(side);
    for (uint32_t c = 0; c < side; ++c, px += 3) {
      const double v = double(c) / double(side);
      for (int ch = 0; ch < 3; ++ch) {
        const Wave& w = wave[ch];
        double level = 118.0 +
                       w.amp_rc * std::sin(two_pi * w.f_row * u + w.ph_row) *
                           std::cos(two_pi * w.f_col * v + w.ph_col) +
                       w.amp_diag * std::sin(two_pi * w.f_diag * (u + v) + w.ph_diag);
        level = std::min(255.0, std::max(0.0, level));
        px[ch] = uint8_t(std::lround(level));
      }
    }
  }
  // four flat ellipses (synth.cpp:66-96)
  for (int e = 0; e < 4; ++e) {
    const double cx = double(side) * u01(rng);
    const double cy = double(side) * u01(rng);
    const double rx = double(side) * (0.05 + 0.10 * u01(rng));
    const double ry = double(side) * (0.05 + 0.10 * u01(rng));
    uint8_t rgb[3];
    for (uint8_t& v : rgb) v = uint8_t(40 + 180 * u01(rng));
    const uint32_t top = uint32_t(std::max(0.0, cy - ry));
    const uint32_t bottom = uint32_t(std::min(double(side) - 1, cy + ry));
    for (uint32_t r = top; r <= bottom; ++r) {
      for (uint32_t c = 0; c < side; ++c) {
        const double dx = (double(c) - cx) / rx;
        const double dy = (double(r) - cy) / ry;
        if (dx * dx + dy * dy <= 1.0)
          std::memcpy(f.px.data() + (size_t(r) * side + c) * 3, rgb, 3);
      }
    }
  }
  return f;
}

std::string bytegen_table(const Key& key, const std::vector<uint32_t>& counts,
                          uint64_t iterations, int device) {
  if (iterations == 0) raise(Errc::invalid_argument, "need iterations >= 1");
  const uint64_t bpi = key.kind == MapKind::Plcm ? 6 : 12;
  std::string out = "map,workers,iterations,bytes,elapsed_ms,throughput_mbps\n";
  for (const uint32_t n : counts) {
    if (n == 0) raise(Errc::invalid_argument, "worker count must be >= 1");
    Coordinator coord(key);
    const std::vector<WorkerLanes> lanes = coord.derive_workers(n);
    // the workers' generators advance in lockstep: every worker runs the
    // largest share, ceil(iterations / n) (the reference gives the remainder
    // to worker 0 alone)
    const uint64_t share = (iterations + n - 1) / n;
    KeystreamSource src(lanes, key.kind, device, share * bpi);
    const auto t0 = Clock::now();
    src.burn(share);
    const double ms = elapsed_ms(t0);
    const uint64_t bytes = iterations * bpi;
    out += map_label(key.kind);
    put_uint(out, n);
    put_uint(out, iterations);
    put_uint(out, bytes);
    put_fixed(out, ms, 3);
    put_fixed(out, double(bytes) / kMiB / (ms / 1000.0), 3);
    out += '\n';
  }
  return out;
}

std::string phases_table(const Key& key, uint32_t side, uint32_t workers, uint32_t rounds,
                         uint32_t images, int device) {
  if (images == 0) raise(Errc::invalid_argument, "need images >= 1");
  Engine engine(key, workers, rounds, device);
  const std::vector<HostFrame> pool = noise_pool(side, std::min(images, 16u), 0xB0);
  Spread confuse, diffuse;
  std::vector<uint8_t> work;
  for (uint32_t i = 0; i < images; ++i) {
    const HostFrame& img = pool[i % pool.size()];
    Engine::PhaseMs t{};
    work = img.px;
    engine.transform_host(work.data(), side, rounds, true, false, nullptr, &t);
    confuse.take(t.confuse_ms);
    t = Engine::PhaseMs{};
    work = img.px;
    engine.transform_host(work.data(), side, rounds, false, true, nullptr, &t);
    diffuse.take(t.bytegen_ms + t.diffuse_ms);
  }
  std::string out =
      "map,side,workers,rounds,images,confuse_mean_ms,confuse_min_ms,"
      "confuse_max_ms,diffuse_mean_ms,diffuse_min_ms,diffuse_max_ms\n";
  out += map_label(key.kind);
  put_uint(out, side);
  put_uint(out, workers);
  put_uint(out, rounds);
  put_uint(out, images);
  for (const Spread* s : {&confuse, &diffuse}) {
    put_fixed(out, s->mean(), 3);
    put_fixed(out, s->lo, 3);
    put_fixed(out, s->hi, 3);
  }
  out += '\n';
  return out;
}

std::string video_table(const Key& key, const std::vector<uint32_t>& sides, uint32_t workers,
                        uint32_t rounds, uint32_t frames, uint16_t fps, int device) {
  std::string out =
      "map,side,workers,rounds,frames,fps,bytegen_mean_ms,confuse_mean_ms,"
      "diffuse_mean_ms,total_mean_ms,total_min_ms,total_max_ms,"
      "throughput_mbps,realtime_ok\n";
  for (const uint32_t side : sides) {
    if (frames == 0) raise(Errc::invalid_argument, "need frames >= 1");
    if (fps == 0) raise(Errc::invalid_argument, "need fps >= 1");
    Engine engine(key, workers, rounds, device);
    const std::vector<HostFrame> pool = noise_pool(side, std::min(frames, 32u), 0xF0);
    Spread total;
    std::vector<uint8_t> work;
    const EngineStats before = engine.stats();
    for (uint32_t i = 0; i < frames; ++i) {
      // The call is in place, so each frame needs a fresh plaintext: that
      // copy is inside the window, like the reference's copy-in
      // (engine.cpp:219).  Outside it, the generator's run-ahead would work
      // during the copy and the mean would undercut the frame period.
      const auto t0 = Clock::now();
      work = pool[i % pool.size()].px;
      engine.run_host(work.data(), side, 1, false);
      total.take(elapsed_ms(t0));
    }
    const EngineStats after = engine.stats();
    const double mean = total.mean();
    out += map_label(key.kind);
    put_uint(out, side);
    put_uint(out, workers);
    put_uint(out, rounds);
    put_uint(out, frames);
    put_uint(out, fps);
    put_fixed(out, (after.prbg_ms - before.prbg_ms) / double(frames), 3);
    put_fixed(out, (after.cipher_ms - before.cipher_ms) / double(frames), 3);
    put_fixed(out, 0.0, 3);
    put_fixed(out, mean, 3);
    put_fixed(out, total.lo, 3);
    put_fixed(out, total.hi, 3);
    put_fixed(out, double(side) * side * 3 / kMiB / (mean / 1000.0), 3);
    out += mean <= 1000.0 / double(fps) ? ",1\n" : ",0\n";
  }
  return out;
}

std::string sweep_table(const Key& key, const HostFrame& plain, uint32_t workers,
                        uint32_t max_rounds, uint64_t seed, int device) {
  if (max_rounds == 0) raise(Errc::invalid_argument, "need max_rounds >= 1");
  const uint32_t side = plain.side;
  const size_t pixels = size_t(side) * side;
  // one byte of one pixel raised by one (bench.cpp:264-268)
  std::mt19937_64 rng(seed);
  HostFrame changed = plain;
  const uint32_t row = uint32_t(rng() % side);
  const uint32_t col = uint32_t(rng() % side);
  const int ch0 = int(rng() % 3);
  uint8_t& target = changed.px[(size_t(row) * side + col) * 3 + ch0];
  target = uint8_t(target + 1);

  // every run on a fresh engine, so each sees the same stream bytes
  const auto states_of = [&](const HostFrame& in, bool confusion, bool diffusion) {
    Engine engine(key, workers, max_rounds, device);
    std::vector<std::vector<uint8_t>> states;
    states.reserve(max_rounds);
    std::vector<uint8_t> work = in.px;
    engine.transform_host(work.data(), side, max_rounds, confusion, diffusion,
                          [&](uint32_t, const uint8_t* s) { states.emplace_back(s, s + work.size()); },
                          nullptr);
    return states;
  };
  const auto base = states_of(plain, false, true);
  const auto other = states_of(changed, false, true);
  const auto scrambled = states_of(plain, true, false);

  std::string out =
      "round,npcr_r,npcr_g,npcr_b,uaci_r,uaci_g,uaci_b,conf_corr_r,"
      "conf_corr_g,conf_corr_b\n";
  for (uint32_t k = 0; k <= max_rounds; ++k) {
    const uint8_t* a = k ? base[k - 1].data() : plain.px.data();
    const uint8_t* b = k ? other[k - 1].data() : changed.px.data();
    const uint8_t* s = k ? scrambled[k - 1].data() : plain.px.data();
    double npcr[3], uaci[3], corr[3];
    for (int ch = 0; ch < 3; ++ch) {
      channel_diff(a, b, pixels, ch, npcr[ch], uaci[ch]);
      corr[ch] = channel_correlation(plain.px.data(), s, pixels, ch).value_or(0.0);
    }
    put_uint(out, k, false);
    for (double v : npcr) put_fixed(out, v, 6);
    for (double v : uaci) put_fixed(out, v, 6);
    for (double v : corr) put_fixed(out, v, 6);
    out += '\n';
  }
  return out;
}

}  // namespace cveb
