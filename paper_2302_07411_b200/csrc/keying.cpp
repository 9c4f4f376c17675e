#include "keying.hpp"

#include <cmath>
#include <cstring>
#include <fstream>
#include <random>

namespace cveb {
namespace {

int nibble(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return 10 + (c - 'a');
  if (c >= 'A' && c <= 'F') return 10 + (c - 'A');
  return -1;
}

double f64_le(const uint8_t* p) {
  uint64_t bits = 0;
  for (int i = 7; i >= 0; --i) bits = (bits << 8) | p[i];
  double v;
  std::memcpy(&v, &bits, 8);
  return v;
}

void put_f64_le(std::string& s, double v) {
  static const char* digits = "0123456789abcdef";
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  for (int i = 0; i < 8; ++i) {
    const unsigned byte = unsigned(bits >> (8 * i)) & 0xFFu;
    s += digits[byte >> 4];
    s += digits[byte & 15];
  }
}

void check_plcm(const Lane& l) {
  if (!(std::isfinite(l.x0) && l.x0 >= 0.0 && l.x0 <= 1.0))
    raise(Errc::bad_key, "plcm x0 outside [0,1]");
  if (!(std::isfinite(l.p) && l.p > 0.0 && l.p < 0.5))
    raise(Errc::bad_key, "plcm p outside (0,0.5)");
}

bool lasm_mu_ok(double mu) {  // chaos.cpp:41-44
  return (mu >= 0.37 && mu <= 0.38) || (mu >= 0.40 && mu <= 0.42) ||
         (mu >= 0.44 && mu <= 0.93) || mu == 1.0;
}

void check_lasm(const Key& k) { check_lasm_lane(LasmLane{k.lx0, k.ly0, k.lmu}); }

double rotate_half(double v) {  // keying.cpp:67-73
  v += 0.5;
  if (v >= 1.0) v -= 1.0;
  return v;
}

double inside(double v, double lo, double hi) {  // keying.cpp:61-65
  if (v <= lo) return std::nextafter(lo, hi);
  if (v >= hi) return std::nextafter(hi, lo);
  return v;
}

double entropy_unit(std::random_device& rd) {  // keying.cpp:52-59
  for (;;) {
    const uint64_t v = (uint64_t(rd()) << 32) | rd();
    const double u = double(v >> 11) * 0x1p-53;
    if (u > 0.0 && u < 1.0) return u;
  }
}

}  // namespace

void check_lasm_lane(const LasmLane& l) {  // chaos.cpp:67-77
  auto unit = [](double v) { return std::isfinite(v) && v >= 0.0 && v <= 1.0; };
  if (!unit(l.x0)) raise(Errc::bad_key, "lasm x0 outside [0,1]");
  if (!unit(l.y0)) raise(Errc::bad_key, "lasm y0 outside [0,1]");
  if (!(std::isfinite(l.mu) && lasm_mu_ok(l.mu)))
    raise(Errc::bad_key, "lasm mu outside the chaotic bands");
}

Key parse_key(const char* hex) {
  size_t len = std::strlen(hex);
  while (len > 0 && (hex[len - 1] == '\n' || hex[len - 1] == '\r' ||
                     hex[len - 1] == ' ' || hex[len - 1] == '\t'))
    --len;
  if (len != 66 && len != 50) raise(Errc::bad_key, "key hex has wrong length");
  std::vector<uint8_t> raw(len / 2);
  for (size_t i = 0; i < raw.size(); ++i) {
    const int hi = nibble(hex[2 * i]), lo = nibble(hex[2 * i + 1]);
    if (hi < 0 || lo < 0) raise(Errc::bad_key, "key hex has a non-hex digit");
    raw[i] = uint8_t(hi << 4 | lo);
  }
  Key k;
  if (raw[0] == 0x00) {
    if (raw.size() != 33) raise(Errc::bad_key, "plcm key truncated");
    k.kind = MapKind::Plcm;
    k.a = {f64_le(&raw[1]), f64_le(&raw[9])};
    k.b = {f64_le(&raw[17]), f64_le(&raw[25])};
    check_plcm(k.a);
    check_plcm(k.b);
  } else if (raw[0] == 0x01) {
    if (raw.size() != 25) raise(Errc::bad_key, "lasm key truncated");
    k.kind = MapKind::Lasm;
    k.lx0 = f64_le(&raw[1]);
    k.ly0 = f64_le(&raw[9]);
    k.lmu = f64_le(&raw[17]);
    check_lasm(k);
  } else {
    raise(Errc::bad_key, "unknown key map tag");
  }
  return k;
}

std::string key_hex(const Key& k) {
  std::string s;
  if (k.kind == MapKind::Plcm) {
    check_plcm(k.a);
    check_plcm(k.b);
    s = "00";
    put_f64_le(s, k.a.x0);
    put_f64_le(s, k.a.p);
    put_f64_le(s, k.b.x0);
    put_f64_le(s, k.b.p);
  } else {
    check_lasm(k);
    s = "01";
    put_f64_le(s, k.lx0);
    put_f64_le(s, k.ly0);
    put_f64_le(s, k.lmu);
  }
  return s;
}

Key fresh_key(MapKind kind) {
  std::random_device rd;
  Key k;
  k.kind = kind;
  if (kind == MapKind::Plcm) {
    k.a.x0 = entropy_unit(rd);
    k.a.p = 0.5 * entropy_unit(rd);
    k.b.x0 = entropy_unit(rd);
    k.b.p = 0.5 * entropy_unit(rd);
  } else {
    k.lx0 = entropy_unit(rd);
    k.ly0 = entropy_unit(rd);
    k.lmu = 0.44 + entropy_unit(rd) * (0.93 - 0.44);
  }
  return k;
}

double plcm_guard(double x, double p) {
  if (x == 0.0 || x == p || x == 0.5 || x == 1.0) {
    x += 0x1p-52;
    if (x > 1.0) x -= 1.0;
  }
  return x;
}

double plcm_iterate(double x, double p) {
  const double f = x > 0.5 ? 1.0 - x : x;
  const double y = f < p ? f / p : (f - p) / (0.5 - p);
  return plcm_guard(y, p);
}

void lasm_iterate(double& x, double& y, double mu) {
  const double pi = 3.14159265358979323846;  // std::numbers::pi
  const double xn = std::sin(pi * mu * (y + 3.0) * x * (1.0 - x));
  const double yn = std::sin(pi * mu * (xn + 3.0) * y * (1.0 - y));
  x = xn;
  y = yn;
}

HostPrbg::HostPrbg(Lane a, Lane b) : pa_(a.p), pb_(b.p) {
  check_plcm(a);
  check_plcm(b);
  xa_ = plcm_guard(a.x0, pa_);
  xb_ = plcm_guard(b.x0, pb_);
  for (int i = 0; i < 256; ++i) step();  // kWarmupSteps (chaos.hpp:14)
}

HostPrbg::HostPrbg(LasmLane a, LasmLane b)
    : lasm_(true), xa_(a.x0), pa_(a.mu), xb_(b.x0), pb_(b.mu), ya_(a.y0), yb_(b.y0) {
  check_lasm_lane(a);  // chaos.cpp:93-107: no guard for LASM
  check_lasm_lane(b);
  for (int i = 0; i < 256; ++i) step();
}

void HostPrbg::step() {
  if (lasm_) {
    lasm_iterate(xa_, ya_, pa_);
    lasm_iterate(xb_, yb_, pb_);
  } else {
    xa_ = plcm_iterate(xa_, pa_);
    xb_ = plcm_iterate(xb_, pb_);
  }
}

void HostPrbg::fill(uint8_t* out, size_t n) {
  auto put48 = [](uint8_t* dst, double a, double b) {
    uint64_t ba, bb;
    std::memcpy(&ba, &a, 8);
    std::memcpy(&bb, &b, 8);
    for (int k = 0; k < 6; ++k) dst[k] = uint8_t((ba ^ bb) >> (8 * k));
  };
  for (size_t i = 0; i < n; ++i) {
    if (pos_ == len_) {
      step();
      put48(buf_, xa_, xb_);
      if (lasm_) put48(buf_ + 6, ya_, yb_);
      len_ = lasm_ ? 12 : 6;
      pos_ = 0;
    }
    out[i] = buf_[pos_++];
  }
}

Coordinator::Coordinator(const Key& key) : kind_(key.kind) {
  if (key.kind == MapKind::Plcm) {
    prbg_ = HostPrbg(key.a, key.b);
  } else {  // keying.cpp:164-170: lane b is the key rotated by one half
    prbg_ = HostPrbg(LasmLane{key.lx0, key.ly0, key.lmu},
                     LasmLane{rotate_half(key.lx0), rotate_half(key.ly0), key.lmu});
  }
}

double Coordinator::next_unit() {
  uint8_t b[6];
  prbg_.fill(b, 6);
  uint64_t v = 0;
  for (int i = 5; i >= 0; --i) v = (v << 8) | b[i];
  return double(v) / double((uint64_t(1) << 48) - 1);
}

std::vector<WorkerLanes> Coordinator::derive_workers(uint32_t n) {  // keying.cpp:180-207
  std::vector<WorkerLanes> out(n);
  for (auto& w : out) {
    if (kind_ == MapKind::Plcm) {
      for (Lane* l : {&w.a, &w.b}) {
        l->x0 = inside(next_unit(), 0.0, 1.0);
        l->p = inside(next_unit() * 0.5, 0.0, 0.5);
      }
    } else {
      for (LasmLane* l : {&w.la, &w.lb}) {
        l->x0 = inside(next_unit(), 0.0, 1.0);
        l->y0 = inside(next_unit(), 0.0, 1.0);
        l->mu = inside(0.44 + next_unit() * (0.93 - 0.44), 0.44, 0.93);
      }
    }
  }
  return out;
}

uint32_t Coordinator::next_seed() {
  uint8_t b[4];
  prbg_.fill(b, 4);
  const uint64_t u = uint64_t(b[0]) | uint64_t(b[1]) << 8 |
                     uint64_t(b[2]) << 16 | uint64_t(b[3]) << 24;
  ++seeds_;
  return uint32_t(u % 0xFFFFFFFFull) + 1;
}

std::vector<double> sine_table(uint32_t side) {
  const double two_pi = 2.0 * 3.14159265358979323846;
  std::vector<double> s(side);
  for (uint32_t a = 0; a < side; ++a)
    s[a] = std::sin(two_pi * double(a) / double(side));
  return s;
}

}  // namespace cveb
