// Row f4: the reference's statistical analysis report and its
// salt-and-pepper / crop tools, on this engine.
//
// Split: the O(side^2) integer reductions -- per-channel histograms and the
// NPCR/UACI counts -- run on the GPU (stats.cu).  The rest is O(samples) or
// O(blocks) and depends on the reference's exact sequential arithmetic and
// random draws, so it runs on the host in the reference's order:
//   histogram_variance / chi_square / entropy   analysis.cpp:62-95
//   sample_adjacent_pairs (mt19937_64 + uniform_int_distribution, dedup by
//     index, pairs in draw order)                analysis.cpp:97-122
//   correlation (two-pass, sequential sums)      analysis.cpp:124-146
//   local_entropy (30 disjoint 44x44 blocks)     analysis.cpp:163-198
//   channel_stats / report / CSV                 analysis.cpp:259-359
// With the same libstdc++ the draws are identical, and with the same
// libm and -ffp-contract=off every printed value is identical.
#include "analysis.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <optional>
#include <random>
#include <unordered_set>

#include "engine.hpp"
#include "fileio.hpp"
#include "keying.hpp"

namespace cveb {
namespace {

constexpr double kChiSquare05Df255 = 293.25;  // analysis.hpp:28
constexpr uint32_t kLocalEntropyBlocks = 30;    // analysis.hpp:54
constexpr uint32_t kLocalEntropyBlockSide = 44; // analysis.hpp:55

using Hist = std::array<uint64_t, 256>;

double hist_variance(const Hist& h) {
  double acc = 0;
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 256; ++j) {
      const double d = double(h[size_t(i)]) - double(h[size_t(j)]);
      acc += 0.5 * d * d;
    }
  return acc / (256.0 * 256.0);
}

double chi_square(const Hist& h, uint64_t total) {
  if (total == 0) raise(Errc::invalid_argument, "empty histogram");
  const double expected = double(total) / 256.0;
  double acc = 0;
  for (const uint64_t c : h) {
    const double d = double(c) - expected;
    acc += d * d / expected;
  }
  return acc;
}

double entropy(const Hist& h, uint64_t total) {
  if (total == 0) raise(Errc::invalid_argument, "empty histogram");
  double acc = 0;
  for (const uint64_t c : h) {
    if (c == 0) continue;
    const double p = double(c) / double(total);
    acc -= p * std::log2(p);
  }
  return acc;
}

std::optional<double> correlation(const std::vector<uint8_t>& x, const std::vector<uint8_t>& y) {
  const double n = double(x.size());
  double ex = 0, ey = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    ex += x[i];
    ey += y[i];
  }
  ex /= n;
  ey /= n;
  double cov = 0, dx = 0, dy = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    const double a = double(x[i]) - ex;
    const double b = double(y[i]) - ey;
    cov += a * b;
    dx += a * a;
    dy += b * b;
  }
  if (dx == 0.0 || dy == 0.0) return std::nullopt;
  return (cov / n) / (std::sqrt(dx / n) * std::sqrt(dy / n));
}

enum class Dir { H, V, D };

// Adjacent-pair correlation of one channel over `count` distinct random
// positions (draws that repeat a position are skipped).
std::optional<double> pair_correlation(const HostFrame& f, int ch, Dir d, uint32_t samples,
                                       uint64_t seed) {
  const uint32_t w = f.side;
  if (w < 2) return std::nullopt;
  const uint32_t rows = d == Dir::H ? w : w - 1, cols = d == Dir::V ? w : w - 1;
  const uint64_t available = uint64_t(rows) * cols;
  const uint32_t count = uint32_t(std::min<uint64_t>(samples, available));
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<uint64_t> dist(0, available - 1);
  std::unordered_set<uint64_t> chosen;
  chosen.reserve(size_t(count) * 2);
  std::vector<uint8_t> x, y;
  x.reserve(count);
  y.reserve(count);
  const uint32_t dr = d == Dir::H ? 0 : 1, dc = d == Dir::V ? 0 : 1;
  while (x.size() < count) {
    const uint64_t idx = dist(rng);
    if (!chosen.insert(idx).second) continue;
    const uint32_t r = uint32_t(idx / cols), c = uint32_t(idx % cols);
    x.push_back(f.px[(size_t(r) * w + c) * 3 + ch]);
    y.push_back(f.px[(size_t(r + dr) * w + c + dc) * 3 + ch]);
  }
  return correlation(x, y);
}

struct Rect {
  uint32_t x, y;
};

// The disjoint block set of local_entropy, or nothing when the frame cannot
// hold it within the attempt cap.  It depends only on the seed and the side,
// so it is drawn once and shared by the three channels.
std::optional<std::vector<Rect>> entropy_blocks(uint32_t side, uint64_t seed) {
  const uint32_t blocks = kLocalEntropyBlocks, bs = kLocalEntropyBlockSide;
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<uint32_t> dist(0, side - bs);
  std::vector<Rect> accepted;
  accepted.reserve(blocks);
  uint64_t attempts = 0;
  const uint64_t cap = uint64_t(blocks) * 100000;
  while (accepted.size() < blocks) {
    if (++attempts > cap) return std::nullopt;
    const uint32_t cx = dist(rng);
    const uint32_t cy = dist(rng);
    bool overlaps = false;
    for (const Rect& r : accepted)
      if (cx < r.x + bs && r.x < cx + bs && cy < r.y + bs && r.y < cy + bs) {
        overlaps = true;
        break;
      }
    if (!overlaps) accepted.push_back(Rect{cx, cy});
  }
  return accepted;
}

double local_entropy(const HostFrame& f, int ch, const std::vector<Rect>& blocks) {
  const uint32_t bs = kLocalEntropyBlockSide;
  double acc = 0;
  for (const Rect& b : blocks) {
    Hist h{};
    for (uint32_t r = 0; r < bs; ++r)
      for (uint32_t c = 0; c < bs; ++c) ++h[f.px[(size_t(b.y + r) * f.side + b.x + c) * 3 + ch]];
    acc += entropy(h, uint64_t(bs) * bs);
  }
  return acc / double(blocks.size());
}

std::string fmt(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.6f", v);
  return buf;
}
std::string fmt(const std::optional<double>& v) { return v ? fmt(*v) : "undefined"; }

struct ChannelStats {
  double variance = 0, chi2 = 0, ent = 0;
  std::optional<double> local_ent, corr_h, corr_v, corr_d;
  bool has_diff = false;
  double npcr = 0, uaci = 0;
};

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::internal, std::string(what) + ": " + cudaGetErrorString(e));
}

// Histograms (768) and NPCR/UACI counts (6) of the frames on the GPU.
void gpu_counts(const HostFrame& a, const HostFrame* b, int device, uint64_t hist[768],
                uint64_t diff[6]) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    raise(Errc::internal, "no CUDA device: the analysis reductions run on the GPU");
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  const uint64_t nbytes = a.px.size();
  cudaStream_t s = nullptr;
  uint8_t *da = nullptr, *db = nullptr;
  unsigned long long* dout = nullptr;
  // stream-ordered allocations: cudaFree would synchronise the whole device
  // (and wait for any other handle's work); cudaFreeAsync does not
  auto cleanup = [&] {
    if (s) {
      if (da) cudaFreeAsync(da, s);
      if (db) cudaFreeAsync(db, s);
      if (dout) cudaFreeAsync(dout, s);
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  };
  try {
    check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&da), std::max<uint64_t>(nbytes, 16), s),
               "cudaMallocAsync");
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&dout), 774 * sizeof(unsigned long long), s),
               "cudaMallocAsync");
    check_cuda(cudaMemcpyAsync(da, a.px.data(), nbytes, cudaMemcpyHostToDevice, s), "H2D");
    if (b) {
      check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&db), std::max<uint64_t>(nbytes, 16), s),
                 "cudaMallocAsync");
      check_cuda(cudaMemcpyAsync(db, b->px.data(), nbytes, cudaMemcpyHostToDevice, s), "H2D");
    }
    launch_frame_stats(da, db, nbytes, dout, b ? dout + 768 : nullptr, s);
    unsigned long long host[774] = {};
    check_cuda(cudaMemcpyAsync(host, dout, sizeof host, cudaMemcpyDeviceToHost, s), "D2H");
    check_cuda(cudaStreamSynchronize(s), "frame statistics");
    for (int i = 0; i < 768; ++i) hist[i] = host[i];
    for (int i = 0; i < 6; ++i) diff[i] = host[768 + i];
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

std::vector<ChannelStats> all_stats(const HostFrame& f, const HostFrame* second, uint32_t samples,
                                    uint64_t seed, int device) {
  uint64_t hist[768], diff[6] = {};
  gpu_counts(f, second, device, hist, diff);
  const uint64_t total = uint64_t(f.side) * f.side;
  std::optional<std::vector<Rect>> blocks;
  if (f.side >= kLocalEntropyBlockSide) blocks = entropy_blocks(f.side, seed);
  std::vector<ChannelStats> out(3);
  for (int ch = 0; ch < 3; ++ch) {
    ChannelStats& s = out[size_t(ch)];
    Hist h;
    std::copy(hist + 256 * ch, hist + 256 * (ch + 1), h.begin());
    s.variance = hist_variance(h);
    s.chi2 = chi_square(h, total);
    s.ent = entropy(h, total);
    if (blocks) s.local_ent = local_entropy(f, ch, *blocks);
    s.corr_h = pair_correlation(f, ch, Dir::H, samples, seed + 0x68);
    s.corr_v = pair_correlation(f, ch, Dir::V, samples, seed + 0x76);
    s.corr_d = pair_correlation(f, ch, Dir::D, samples, seed + 0x64);
    if (second) {
      s.has_diff = true;
      s.npcr = 100.0 * double(diff[ch]) / double(total);
      s.uaci = 100.0 * double(diff[3 + ch]) / (255.0 * double(total));
    }
  }
  return out;
}

void square_p6_check(const P6Image& img) {
  if (img.width != img.height)
    raise(Errc::invalid_argument, "this operation needs a square image");
}

bool is_container(const std::vector<uint8_t>& d) {
  return d.size() >= 4 && std::memcmp(d.data(), "CVE1", 4) == 0;
}

// Applies fn to every frame of a container (header copied), or to the single
// square P6 image (capi.cpp:123-141).
template <typename Fn>
void rewrite_frames(const char* in_path, const char* out_path, Fn&& fn) {
  const std::vector<uint8_t> data = read_whole_file(in_path);
  if (is_container(data)) {
    ContainerIn in(in_path);
    ContainerOut out(out_path, in.header());
    const CveHeader& h = in.header();
    HostFrame f;
    f.side = h.side;
    f.orig_width = h.orig_width;
    f.orig_height = h.orig_height;
    f.px.resize(size_t(h.side) * h.side * 3);
    for (uint32_t i = 0; i < h.frame_count; ++i) {
      in.next(f.px.data(), 1);
      fn(f, i);
      out.put(f.px.data(), 1);
    }
    out.finish();
    return;
  }
  P6Image img = p6_parse(data.data(), data.size());
  square_p6_check(img);
  HostFrame f;
  f.side = f.orig_width = img.width;
  f.orig_height = img.height;
  f.px = std::move(img.rgb);
  fn(f, 0);
  const std::string hdr = p6_header(f.side, f.side);
  std::vector<uint8_t> bytes(hdr.begin(), hdr.end());
  bytes.insert(bytes.end(), f.px.begin(), f.px.end());
  write_whole_file(out_path, bytes.data(), bytes.size());
}

}  // namespace

HostFrame load_frame_any(const char* path, uint32_t frame_index) {
  const std::vector<uint8_t> data = read_whole_file(path);
  HostFrame f;
  if (is_container(data)) {
    ContainerIn in(path);
    const CveHeader& h = in.header();
    if (frame_index >= h.frame_count) raise(Errc::invalid_argument, "frame index out of range");
    f.side = h.side;
    f.orig_width = h.orig_width;
    f.orig_height = h.orig_height;
    f.px.resize(size_t(h.side) * h.side * 3);
    for (uint32_t i = 0; i <= frame_index; ++i) in.next(f.px.data(), 1);
    return f;
  }
  P6Image img = p6_parse(data.data(), data.size());
  square_p6_check(img);
  f.side = f.orig_width = img.width;
  f.orig_height = img.height;
  f.px = std::move(img.rgb);
  return f;
}

std::string analyze(const HostFrame& frame, const HostFrame* second, uint32_t samples,
                    uint64_t seed, bool csv, int device) {
  NvtxRange nvtx("cve: analyze");
  static const char* names[3] = {"R", "G", "B"};
  const std::vector<ChannelStats> st = all_stats(frame, second, samples, seed, device);
  std::string out;
  if (csv) {
    out = "channel,variance,chi_square,entropy,local_entropy,corr_horizontal,corr_vertical,"
          "corr_diagonal";
    if (second) out += ",npcr,uaci";
    out += "\n";
    for (int ch = 0; ch < 3; ++ch) {
      const ChannelStats& s = st[size_t(ch)];
      out += names[ch];
      for (const std::string& v : {fmt(s.variance), fmt(s.chi2), fmt(s.ent), fmt(s.local_ent),
                                   fmt(s.corr_h), fmt(s.corr_v), fmt(s.corr_d)})
        out += "," + v;
      if (s.has_diff) out += "," + fmt(s.npcr) + "," + fmt(s.uaci);
      out += "\n";
    }
    return out;
  }
  out += "side=" + std::to_string(frame.side) + "\n";
  out += "orig_width=" + std::to_string(frame.orig_width) + "\n";
  out += "orig_height=" + std::to_string(frame.orig_height) + "\n";
  out += "samples=" + std::to_string(samples) + "\n";
  out += "seed=" + std::to_string(seed) + "\n";
  for (int ch = 0; ch < 3; ++ch) {
    const ChannelStats& s = st[size_t(ch)];
    const std::string p = std::string("channel.") + names[ch] + ".";
    out += p + "variance=" + fmt(s.variance) + "\n";
    out += p + "chi_square=" + fmt(s.chi2) + "\n";
    out += p + "chi_square_uniform=" + (s.chi2 < kChiSquare05Df255 ? "yes" : "no") + "\n";
    out += p + "entropy=" + fmt(s.ent) + "\n";
    out += p + "local_entropy=" + fmt(s.local_ent) + "\n";
    out += p + "corr_horizontal=" + fmt(s.corr_h) + "\n";
    out += p + "corr_vertical=" + fmt(s.corr_v) + "\n";
    out += p + "corr_diagonal=" + fmt(s.corr_d) + "\n";
    if (s.has_diff) {
      out += p + "npcr=" + fmt(s.npcr) + "\n";
      out += p + "uaci=" + fmt(s.uaci) + "\n";
    }
  }
  return out;
}

// add_salt_pepper (analysis.cpp:220-241) per frame, seed + frame index.
void add_noise_file(const char* in_path, const char* out_path, double rate, uint64_t seed) {
  rewrite_frames(in_path, out_path, [&](HostFrame& f, uint32_t index) {
    if (!(rate >= 0.0 && rate <= 1.0)) raise(Errc::invalid_argument, "noise rate must be in [0,1]");
    if (f.side == 0) raise(Errc::invalid_argument, "empty frame");
    const uint64_t positions = uint64_t(f.side) * f.side;
    const uint64_t hits = uint64_t(std::llround(rate * double(positions)));
    std::mt19937_64 rng(seed + index);
    std::uniform_int_distribution<uint64_t> dist(0, positions - 1);
    std::unordered_set<uint64_t> chosen;
    chosen.reserve(size_t(hits) * 2);
    while (chosen.size() < hits) {
      const uint64_t idx = dist(rng);
      if (!chosen.insert(idx).second) continue;
      const uint8_t v = (rng() & 1) ? 0xFF : 0x00;
      std::memset(f.px.data() + idx * 3, v, 3);
    }
  });
}

// crop_fill (analysis.cpp:243-257): blocks checked and filled in order.
void crop_file(const char* in_path, const char* out_path, const std::vector<CropBlock>& blocks) {
  rewrite_frames(in_path, out_path, [&](HostFrame& f, uint32_t) {
    for (const CropBlock& b : blocks) {
      if (b.side == 0 || b.x + b.side > f.side || b.y + b.side > f.side)
        raise(Errc::invalid_argument, "crop block outside the frame");
      if (b.fill != 0x00 && b.fill != 0xFF)
        raise(Errc::invalid_argument, "crop fill must be 0x00 or 0xFF");
      for (uint32_t r = 0; r < b.side; ++r)
        std::memset(f.px.data() + (size_t(b.y + r) * f.side + b.x) * 3, b.fill, size_t(b.side) * 3);
    }
  });
}

}  // namespace cveb
