#include "fileio.hpp"

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <filesystem>

namespace fs = std::filesystem;

namespace cveb {
namespace {

bool ws(uint8_t c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; }

uint32_t le32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 |
         uint32_t(p[3]) << 24;
}
uint16_t le16(const uint8_t* p) { return uint16_t(p[0] | (p[1] << 8)); }
void put32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = uint8_t(v >> (8 * i));
}
void put16(uint8_t* p, uint16_t v) {
  p[0] = uint8_t(v);
  p[1] = uint8_t(v >> 8);
}

// container.cpp:31-50
void check_header(const CveHeader& h) {
  if (h.version != 1) raise(Errc::bad_format, "container: unsupported version");
  if (h.map_kind > 1) raise(Errc::bad_format, "container: unknown map kind");
  if (h.side == 0) raise(Errc::bad_format, "container: zero frame side");
  if (h.workers == 0) raise(Errc::bad_format, "container: zero worker count");
  if (h.side % h.workers)
    raise(Errc::bad_format, "container: side not divisible by worker count");
  if (h.rounds == 0) raise(Errc::bad_format, "container: zero rounds");
  if (h.orig_width == 0 || h.orig_width > h.side || h.orig_height == 0 ||
      h.orig_height > h.side)
    raise(Errc::bad_format, "container: original dimensions outside the frame");
  if (h.fps == 0) raise(Errc::bad_format, "container: zero fps");
}

std::FILE* open_or_raise(const std::string& path, const char* mode, bool writing) {
  std::FILE* f = std::fopen(path.c_str(), mode);
  if (!f)
    raise(Errc::io, std::string(writing ? "cannot open for writing: "
                                        : "cannot open for reading: ") + path);
  return f;
}

}  // namespace

std::vector<uint8_t> read_whole_file(const std::string& path) {
  std::FILE* f = open_or_raise(path, "rb", false);
  std::vector<uint8_t> out;
  uint8_t buf[1 << 16];
  size_t k;
  while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) out.insert(out.end(), buf, buf + k);
  const bool bad = std::ferror(f);
  std::fclose(f);
  if (bad) raise(Errc::io, "read failed: " + path);
  return out;
}

void write_whole_file(const std::string& path, const uint8_t* data, size_t n) {
  std::FILE* f = open_or_raise(path, "wb", true);
  const bool ok = std::fwrite(data, 1, n, f) == n;
  const bool closed = std::fclose(f) == 0;
  if (!ok || !closed) raise(Errc::io, "write failed: " + path);
}

// image_io.cpp:34-93
P6Image p6_parse(const uint8_t* d, size_t n) {
  if (n < 2 || d[0] != 'P' || d[1] != '6') raise(Errc::bad_format, "ppm: not a P6 file");
  size_t pos = 2;
  auto field = [&]() -> uint32_t {
    while (pos < n) {
      if (d[pos] == '#') {
        while (pos < n && d[pos] != '\n') ++pos;
      } else if (ws(d[pos])) {
        ++pos;
      } else {
        break;
      }
    }
    if (pos >= n || d[pos] < '0' || d[pos] > '9')
      raise(Errc::bad_format, "ppm: expected a decimal header field");
    uint64_t v = 0;
    while (pos < n && d[pos] >= '0' && d[pos] <= '9') {
      v = v * 10 + uint64_t(d[pos] - '0');
      if (v > 0xFFFFFFFFull) raise(Errc::bad_format, "ppm: header field overflow");
      ++pos;
    }
    return uint32_t(v);
  };
  P6Image img;
  img.width = field();
  img.height = field();
  const uint32_t maxval = field();
  if (img.width == 0 || img.height == 0) raise(Errc::bad_format, "ppm: zero dimension");
  if (maxval != 255) raise(Errc::bad_format, "ppm: only maxval 255 is supported");
  if (pos >= n) raise(Errc::bad_format, "ppm: truncated header");
  if (!ws(d[pos])) raise(Errc::bad_format, "ppm: missing separator after maxval");
  ++pos;
  const size_t need = size_t(img.width) * img.height * 3;
  if (n - pos < need) raise(Errc::bad_format, "ppm: truncated pixels");
  img.rgb.assign(d + pos, d + pos + need);
  return img;
}

std::string p6_header(uint32_t width, uint32_t height) {
  char b[64];
  std::snprintf(b, sizeof b, "P6\n%u %u\n255\n", width, height);
  return b;
}

uint32_t padded_side_of(uint32_t width, uint32_t height, uint32_t workers) {
  if (width == 0 || height == 0) raise(Errc::invalid_argument, "frame dimensions must be >= 1");
  if (workers == 0) raise(Errc::invalid_argument, "worker count must be >= 1");
  const uint64_t m = std::max(width, height);
  const uint64_t s = (m + workers - 1) / workers * workers;
  if (s > 0xFFFFFFFFull) raise(Errc::invalid_argument, "padded side overflows");
  return uint32_t(s);
}

// image_io.cpp:138-212
PlainSource::PlainSource(const std::string& path, uint32_t raw_w, uint32_t raw_h) {
  if (raw_w || raw_h) {
    if (!raw_w || !raw_h) raise(Errc::invalid_argument, "raw input needs explicit dimensions");
    kind_ = Kind::Raw;
    w_ = raw_w;
    h_ = raw_h;
    std::error_code ec;
    const uint64_t bytes = fs::exists(path, ec) ? fs::file_size(path, ec) : 0;
    const uint64_t fb = uint64_t(w_) * h_ * 3;
    if (bytes == 0 || bytes % fb) raise(Errc::bad_format, "raw input is not a whole number of frames");
    count_ = uint32_t(bytes / fb);
    raw_ = open_or_raise(path, "rb", false);
    return;
  }
  std::error_code ec;
  if (fs::is_directory(path, ec)) {
    kind_ = Kind::Dir;
    for (const auto& e : fs::directory_iterator(path))
      if (e.is_regular_file() && e.path().extension() == ".ppm") paths_.push_back(e.path().string());
    if (paths_.empty()) raise(Errc::io, "no .ppm frames in: " + path);
    std::sort(paths_.begin(), paths_.end());
    const auto first = read_whole_file(paths_[0]);
    const P6Image img = p6_parse(first.data(), first.size());
    w_ = img.width;
    h_ = img.height;
    count_ = uint32_t(paths_.size());
    return;
  }
  kind_ = Kind::File;
  const auto data = read_whole_file(path);
  const P6Image img = p6_parse(data.data(), data.size());
  w_ = img.width;
  h_ = img.height;
  count_ = 1;
  paths_.push_back(path);
}

PlainSource::~PlainSource() {
  if (raw_) std::fclose(raw_);
}

void PlainSource::next(uint8_t* dst) {
  if (cursor_ >= count_) raise(Errc::invalid_argument, "frame source drained");
  const size_t fb = size_t(w_) * h_ * 3;
  if (kind_ == Kind::Raw) {
    if (std::fread(dst, 1, fb, raw_) != fb) raise(Errc::io, "raw input truncated");
  } else {
    const auto data = read_whole_file(paths_[cursor_]);
    const P6Image img = p6_parse(data.data(), data.size());
    if (img.width != w_ || img.height != h_)
      raise(Errc::bad_format, "frame dimensions differ across the sequence: " + paths_[cursor_]);
    std::memcpy(dst, img.rgb.data(), fb);
  }
  ++cursor_;
}

// image_io.cpp:230-277
PlainSink::PlainSink(const std::string& path, bool raw, uint32_t count)
    : path_(path), raw_mode_(raw), expected_(count) {
  if (raw) {
    raw_ = open_or_raise(path, "wb", true);
  } else if (count > 1) {
    std::error_code ec;
    fs::create_directories(path, ec);
    if (!fs::is_directory(path, ec)) raise(Errc::io, "cannot create frame directory: " + path);
  }
}

PlainSink::~PlainSink() {
  if (raw_) std::fclose(raw_);
}

void PlainSink::put(const uint8_t* rgb, uint32_t width, uint32_t height) {
  if (written_ >= expected_) raise(Errc::invalid_argument, "frame sink received too many frames");
  const size_t fb = size_t(width) * height * 3;
  if (raw_mode_) {
    if (std::fwrite(rgb, 1, fb, raw_) != fb) raise(Errc::io, "write failed: " + path_);
  } else {
    std::string target = path_;
    if (expected_ > 1) {
      char name[32];
      std::snprintf(name, sizeof name, "frame_%06u.ppm", written_);
      target = (fs::path(path_) / name).string();
    }
    const std::string hdr = p6_header(width, height);
    std::vector<uint8_t> out(hdr.begin(), hdr.end());
    out.insert(out.end(), rgb, rgb + fb);
    write_whole_file(target, out.data(), out.size());
  }
  ++written_;
}

void PlainSink::finish() {
  if (written_ != expected_) raise(Errc::io, "frame sink closed before all frames were written");
  if (raw_) {
    const bool ok = std::fclose(raw_) == 0;
    raw_ = nullptr;
    if (!ok) raise(Errc::io, "write failed: " + path_);
  }
}

// container.cpp:53-90
void cve_header_encode(const CveHeader& h, uint8_t out[kCveHeaderBytes]) {
  check_header(h);
  std::memcpy(out, "CVE1", 4);
  out[4] = h.version;
  out[5] = h.map_kind;
  put32(out + 6, h.side);
  put32(out + 10, h.orig_width);
  put32(out + 14, h.orig_height);
  put16(out + 18, h.workers);
  out[20] = h.rounds;
  put16(out + 21, h.fps);
  put32(out + 23, h.frame_count);
}

CveHeader cve_header_decode(const uint8_t* d, size_t n) {
  if (n < kCveHeaderBytes) raise(Errc::bad_format, "container: truncated header");
  if (std::memcmp(d, "CVE1", 4) != 0) raise(Errc::bad_format, "container: bad magic");
  CveHeader h;
  h.version = d[4];
  if (d[5] > 1) raise(Errc::bad_format, "container: unknown map kind");
  h.map_kind = d[5];
  h.side = le32(d + 6);
  h.orig_width = le32(d + 10);
  h.orig_height = le32(d + 14);
  h.workers = le16(d + 18);
  h.rounds = d[20];
  h.fps = le16(d + 21);
  h.frame_count = le32(d + 23);
  check_header(h);
  return h;
}

ContainerOut::ContainerOut(const std::string& path, const CveHeader& h) : path_(path), h_(h) {
  f_ = open_or_raise(path, "wb", true);  // opened first, like the reference
  uint8_t hdr[kCveHeaderBytes];
  cve_header_encode(h_, hdr);
  if (std::fwrite(hdr, 1, sizeof hdr, f_) != sizeof hdr) raise(Errc::io, "write failed: " + path_);
}

ContainerOut::~ContainerOut() {
  if (f_) std::fclose(f_);
}

void ContainerOut::put(const uint8_t* frames, uint32_t count) {
  if (uint64_t(written_) + count > h_.frame_count)
    raise(Errc::invalid_argument, "container: too many frames");
  const size_t bytes = size_t(count) * h_.side * h_.side * 3;
  if (std::fwrite(frames, 1, bytes, f_) != bytes) raise(Errc::io, "write failed: " + path_);
  written_ += count;
}

void ContainerOut::finish() {
  if (written_ != h_.frame_count) raise(Errc::io, "container: fewer frames written than declared");
  const bool ok = std::fclose(f_) == 0;
  f_ = nullptr;
  if (!ok) raise(Errc::io, "close failed: " + path_);
}

// container.cpp:125-158
ContainerIn::ContainerIn(const std::string& path) : path_(path) {
  f_ = open_or_raise(path, "rb", false);
  uint8_t hdr[kCveHeaderBytes];
  if (std::fread(hdr, 1, sizeof hdr, f_) != sizeof hdr)
    raise(Errc::bad_format, "container: truncated header");
  h_ = cve_header_decode(hdr, sizeof hdr);
  std::error_code ec;
  const uint64_t total = fs::file_size(path, ec);
  const uint64_t want =
      kCveHeaderBytes + uint64_t(h_.frame_count) * h_.side * h_.side * 3;
  if (ec || total != want) raise(Errc::bad_format, "container: payload size does not match header");
}

ContainerIn::~ContainerIn() {
  if (f_) std::fclose(f_);
}

void ContainerIn::next(uint8_t* frames, uint32_t count) {
  if (count > remaining()) raise(Errc::invalid_argument, "container: no frames left");
  const size_t bytes = size_t(count) * h_.side * h_.side * 3;
  if (std::fread(frames, 1, bytes, f_) != bytes)
    raise(Errc::bad_format, "container: truncated frame payload");
  cursor_ += count;
}

}  // namespace cveb
