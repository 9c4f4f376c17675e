// Host-side keying for the B200 engine: hex keys, the coordinator generator,
// per-subframe lane parameters and per-frame confusion seeds.
//
// This is O(n) work per clip plus 4 bytes per frame, so it stays on the host
// (SURVEY.md §8(a) rows A1-A4).  The per-subframe keystream generators -- the
// hot loop -- run on the GPU (prbg.cu).  All arithmetic is IEEE binary64 with
// contraction disabled (-ffp-contract=off), matching the reference's x86-64
// Release build bit for bit.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace cveb {

// Error taxonomy of the reference (errors.hpp:8-28); values equal cve_status.
enum class Errc : int {
  invalid_argument = 1,
  bad_key = 2,
  io = 3,
  bad_format = 4,
  mismatch = 5,
  internal = 6,
};

struct Error : std::runtime_error {
  Errc code;
  Error(Errc c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void raise(Errc c, const std::string& what) {
  throw Error(c, what);
}

enum class MapKind : uint8_t { Plcm = 0, Lasm = 1 };

struct Lane {  // one PLCM orbit: start point and control parameter
  double x0 = 0;
  double p = 0;
};

struct LasmLane {  // one LASM orbit (chaos.hpp LasmParams): start point, mu
  double x0 = 0;
  double y0 = 0;
  double mu = 0;
};

struct Key {
  MapKind kind = MapKind::Plcm;
  Lane a, b;                          // PLCM
  double lx0 = 0, ly0 = 0, lmu = 0;   // LASM
};

// Reference parse_key_hex (keying.cpp:77-107): trailing whitespace trimmed,
// 66 (PLCM) or 50 (LASM) hex digits, tag byte, little-endian binary64s,
// domain checks (chaos.cpp:58-76).  Throws Error{bad_key}.
Key parse_key(const char* hex);
std::string key_hex(const Key& k);
Key fresh_key(MapKind kind);  // OS entropy, like generate_key (keying.cpp:131-143)

// PLCM map, one guarded iteration (chaos.cpp:18-32, 109-117).  Host copy used
// by the coordinator only.
double plcm_iterate(double x, double p);
double plcm_guard(double x, double p);

// LASM map, one iteration (chaos.cpp:34-38) with the host's libm sin -- the
// coordinator's copy; the subframe generators run on the GPU (lasm.cu).
void lasm_iterate(double& x, double& y, double mu);
void check_lasm_lane(const LasmLane& l);  // chaos.cpp:67-77, throws bad_key

// Two-lane byte generator with a chunk-invariant byte cursor: 6 bytes per
// PLCM iteration, 12 per LASM iteration (x bytes, then y bytes)
// (chaos.cpp:79-107, 119-153).
class HostPrbg {
 public:
  HostPrbg() = default;
  HostPrbg(Lane a, Lane b);
  HostPrbg(LasmLane a, LasmLane b);
  void fill(uint8_t* out, size_t n);

 private:
  void step();
  bool lasm_ = false;
  double xa_ = 0, pa_ = 0, xb_ = 0, pb_ = 0;  // LASM: pa_/pb_ hold mu
  double ya_ = 0, yb_ = 0;
  uint8_t buf_[12] = {};
  int pos_ = 0, len_ = 0;  // pos_ == len_: empty
};

// Lane pair of subframe generator i, in reference derivation order; the
// PLCM pair (a, b) or the LASM pair (la, lb), by the key's map.
struct WorkerLanes {
  Lane a, b;
  LasmLane la, lb;
};

// Coordinator (keying.cpp:164-218): seeded from the key lanes, derives the
// subframe lanes (6-byte unit draws, clamped one ulp inside), then yields one
// 32-bit confusion seed per frame.
class Coordinator {
 public:
  explicit Coordinator(const Key& key);
  MapKind kind() const { return kind_; }
  std::vector<WorkerLanes> derive_workers(uint32_t n);
  uint32_t next_seed();
  uint64_t seeds_drawn() const { return seeds_; }

 private:
  double next_unit();
  MapKind kind_ = MapKind::Plcm;
  HostPrbg prbg_;
  uint64_t seeds_ = 0;
};

// S[alpha] = sin(((2*pi)*alpha)/side), the seed-independent half of the
// confusion shift (engine.cpp:19-22).  glibc sin, evaluated once per side.
std::vector<double> sine_table(uint32_t side);

}  // namespace cveb
