// Host-side file formats around the cipher path:
// binary P6 images, frame sequences (one P6, a directory of P6 files, raw
// RGB24), and the CVE1 container.  Semantics and error codes follow the
// reference (image_io.cpp:15-279, container.cpp:31-158, README.md:69-89);
// the implementation is this engine's own.
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "keying.hpp"

namespace cveb {

std::vector<uint8_t> read_whole_file(const std::string& path);
void write_whole_file(const std::string& path, const uint8_t* data, size_t n);

struct P6Image {
  uint32_t width = 0, height = 0;
  std::vector<uint8_t> rgb;
};
// Binary P6, maxval 255; '#' comments and any whitespace in the header.
P6Image p6_parse(const uint8_t* data, size_t n);
std::string p6_header(uint32_t width, uint32_t height);

// smallest multiple of n covering max(w, h) (frame.cpp:19-26)
uint32_t padded_side_of(uint32_t width, uint32_t height, uint32_t workers);

// Unpadded plaintext frames from a P6 file, a directory of *.ppm (sorted by
// name, equal dimensions) or raw RGB24 of declared dimensions.
class PlainSource {
 public:
  PlainSource(const std::string& path, uint32_t raw_w, uint32_t raw_h);
  ~PlainSource();
  uint32_t width() const { return w_; }
  uint32_t height() const { return h_; }
  uint32_t count() const { return count_; }
  // next frame's w*h*3 bytes into dst
  void next(uint8_t* dst);

 private:
  enum class Kind { File, Dir, Raw } kind_ = Kind::File;
  uint32_t w_ = 0, h_ = 0, count_ = 0, cursor_ = 0;
  std::vector<std::string> paths_;
  std::FILE* raw_ = nullptr;
};

// Cropped plaintext frames to one P6 (single frame), a directory of
// frame_NNNNNN.ppm, or a raw RGB24 stream.
class PlainSink {
 public:
  PlainSink(const std::string& path, bool raw, uint32_t count);
  ~PlainSink();
  void put(const uint8_t* rgb, uint32_t width, uint32_t height);
  void finish();

 private:
  std::string path_;
  bool raw_mode_;
  uint32_t expected_, written_ = 0;
  std::FILE* raw_ = nullptr;
};

// CVE1: 27-byte little-endian header, then frame_count * side*side*3 bytes.
struct CveHeader {
  uint8_t version = 1;
  uint8_t map_kind = 0;
  uint32_t side = 0, orig_width = 0, orig_height = 0;
  uint16_t workers = 0;
  uint8_t rounds = 0;
  uint16_t fps = 0;
  uint32_t frame_count = 0;
};
constexpr size_t kCveHeaderBytes = 27;
void cve_header_encode(const CveHeader& h, uint8_t out[kCveHeaderBytes]);
CveHeader cve_header_decode(const uint8_t* data, size_t n);  // bad_format

class ContainerOut {
 public:
  ContainerOut(const std::string& path, const CveHeader& h);
  ~ContainerOut();
  void put(const uint8_t* square_frames, uint32_t count);
  void finish();

 private:
  std::string path_;
  CveHeader h_;
  uint32_t written_ = 0;
  std::FILE* f_ = nullptr;
};

class ContainerIn {
 public:
  explicit ContainerIn(const std::string& path);
  ~ContainerIn();
  const CveHeader& header() const { return h_; }
  uint32_t remaining() const { return h_.frame_count - cursor_; }
  void next(uint8_t* square_frames, uint32_t count);

 private:
  std::string path_;
  CveHeader h_;
  uint32_t cursor_ = 0;
  std::FILE* f_ = nullptr;
};

}  // namespace cveb
