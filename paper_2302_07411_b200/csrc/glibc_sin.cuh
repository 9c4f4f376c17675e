// sin(x) exactly as glibc 2.39's libm computes it on an FMA-capable x86-64
// host, for host and sm_100a device code.
//
// Why: the LASM map (reference chaos.cpp:34-38) evaluates glibc `sin` twice
// per iteration on a sequential chaotic chain, so one differing bit forks the
// keystream for the rest of the clip.  A correctly rounded (or CUDA's) sin
// differs from glibc's in a fraction of cases; only glibc's own arithmetic
// gives byte parity.
//
// What is restated: the published algorithm of glibc's dbl-64 sin (the IBM
// Accurate Mathematical Library: table lookup at k/128 plus double-double
// polynomial corrections, Taylor series near 0, Cody-Waite reduction by pi/2
// below 105414350), in the operation order and FMA contractions of the
// `sin` ifunc variant the dynamic linker selects on hosts with FMA + AVX2
// (every B200 host); which operations that variant fuses was read from the
// installed libm's machine code (objdump), not from glibc's sources.  The
// polynomial and reduction constants are the algorithm's published
// coefficients; the 110-entry sin/cos table is read from the installed libm
// at build time (gen_sincostab.py -> the generated glibc_sincostab.inc),
// because its low parts are not reproducible by recomputation.  Parity is
// pinned by tests/test_lasm.py against the host's libm `sin` on ~4 million
// arguments across every branch and edge and on whole LASM orbits.
//
// Domain: |x| < 105414350 (the Cody-Waite branch).  LASM arguments are
// pi*mu*(y+3)*x*(1-x) with x, y in [0,1], mu <= 1, i.e. in [0, pi]; larger
// arguments (glibc's multi-precision reduction) return NaN here.
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define GSIN_HD __host__ __device__ __forceinline__
#define GSIN_MEMBER __host__ __device__ __forceinline__
#else
#define GSIN_HD static inline
#define GSIN_MEMBER inline
#endif

#ifndef __CUDA_ARCH__
#include <math.h>
#endif

namespace gsin {

// Entries {sin hi, sin lo, cos hi, cos lo} of k/128, k = 0..109.
constexpr int kTableDoubles = 440;

// Coefficients (hex-exact).
constexpr double kBig = 0x1.8p45;              // rounds |x| to a multiple of 2^-7
constexpr double kSn3 = -0x1.5555555555515p-3;  // sin correction polynomial
constexpr double kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs2 = 0x1.0p-1;               // cos correction polynomial
constexpr double kCs4 = -0x1.5555555555535p-5;
constexpr double kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3;   // Taylor series near 0
constexpr double kS2 = 0x1.1111111110ecep-7;
constexpr double kS3 = -0x1.a01a019db08b8p-13;
constexpr double kS4 = 0x1.71de27b9a7ed9p-19;
constexpr double kS5 = -0x1.addffc2fcdf59p-26;
constexpr double kTaylorMax = 0x1.020c49ba5e354p-3;  // 0.126
constexpr double kHp0 = 0x1.921fb54442d18p0;    // pi/2 = hp0 + hp1
constexpr double kHp1 = 0x1.1a62633145c07p-54;
constexpr double kHpInv = 0x1.45f306dc9c883p-1; // 2/pi
constexpr double kToInt = 0x1.8p52;
constexpr double kMp1 = 0x1.921fb58p0;          // pi/2 = mp1 + mp2 + pp3 + pp4
constexpr double kMp2 = -0x1.dde973cp-27;
constexpr double kPp3 = -0x1.cb3b398p-55;
constexpr double kPp4 = -0x1.d747f23e32ed7p-83;

GSIN_HD uint64_t bits(double v) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(v);
#else
  uint64_t u;
  memcpy(&u, &v, 8);
  return u;
#endif
}

GSIN_HD double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double v;
  memcpy(&v, &u, 8);
  return v;
#endif
}

GSIN_HD double fmad(double a, double b, double c) { return fma(a, b, c); }

// Table access.  Host code indexes a plain array; device code may use
// SmemTable, whose 32-bit shared-memory address is formed once per kernel
// (indexing a generic pointer to shared memory made ptxas re-derive the
// shared window base -- S2UR SR_CgaCtaId -- in front of every table load on
// the chain, measured ~100 cycles per LASM iteration).
struct PtrTable {
  const double* p;
  GSIN_MEMBER double operator()(int i) const { return p[i]; }
};

#ifdef __CUDACC__
struct SmemTable {
  uint32_t base;  // __cvta_generic_to_shared of the table
  __device__ __forceinline__ double operator()(int i) const {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * (uint32_t)i));
    return v;
  }
};
#endif

GSIN_HD double copysign_of(double mag, double sgn) {
  return from_bits((bits(mag) & 0x7fffffffffffffffull) | (bits(sgn) & 0x8000000000000000ull));
}

// sin(a + da) for |a| < 0.126:  a + xx*(P(xx)*a - da/2) + da.
GSIN_HD double taylor(double a, double da) {
  const double xx = a * a;
  double p = fmad(xx, kS5, kS4);
  p = fmad(xx, p, kS3);
  p = fmad(xx, p, kS2);
  p = fmad(xx, p, kS1);
  const double t = fmad(p, a, -(0.5 * da));
  return fmad(xx, t, da) + a;
}

// |sin(a + da)| for 0.126 <= |a| <= 0.8555 via the table at k/128 (glibc
// returns it with the sign of a).
template <class Tab>
GSIN_HD double sin_tab_mag(double a, double da, const Tab& tab) {
  const double ax = from_bits(bits(a) & 0x7fffffffffffffffull);
  if (a <= 0.0) da = -da;
  const double u = kBig + ax;
  const double x = ax - (u - kBig);
  const int k = (int)((uint32_t)bits(u) << 2);
  const double xx = x * x;
  const double s = x + fmad(x * xx, fmad(xx, kSn5, kSn3), da);
  const double c = fmad(x, da, xx * fmad(xx, fmad(xx, kCs6, kCs4), kCs2));
  const double sn = tab(k), ssn = tab(k + 1), cs = tab(k + 2), ccs = tab(k + 3);
  const double cor = fmad(s, cs, fmad(-c, sn, fmad(s, ccs, ssn)));
  return sn + cor;
}

template <class Tab>
GSIN_HD double sin_tab(double a, double da, const Tab& tab) {
  return copysign_of(sin_tab_mag(a, da, tab), a);
}

// cos(a + da) for |a| <= 0.8555 via the table at k/128.
template <class Tab>
GSIN_HD double cos_tab(double a, double da, const Tab& tab) {
  const double ax = from_bits(bits(a) & 0x7fffffffffffffffull);
  if (a < 0.0) da = -da;
  const double u = kBig + ax;
  const int k = (int)((uint32_t)bits(u) << 2);
  const double x = (ax - (u - kBig)) + da;
  const double xx = x * x;
  const double s = fmad(x * xx, fmad(xx, kSn5, kSn3), x);
  const double c = xx * fmad(xx, fmad(xx, kCs6, kCs4), kCs2);
  const double sn = tab(k), ssn = tab(k + 1), cs = tab(k + 2), ccs = tab(k + 3);
  const double cor = fmad(-s, sn, fmad(-c, cs, fmad(-s, ssn, ccs)));
  return cs + cor;
}

// glibc sin(x), |x| < 105414350; `tab` = the 440 table doubles.
template <class Tab>
GSIN_HD double sin(double x, const Tab& tab) {
  const uint32_t k = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;  // |x| < 2^-26
  if (k < 0x3feb6000u) {          // |x| < 0.855469
    const double ax = from_bits(bits(x) & 0x7fffffffffffffffull);
    if (ax < kTaylorMax) return taylor(x, 0.0);
    return sin_tab(x, 0.0, tab);
  }
  if (k < 0x400368fdu) {          // |x| < 0x1.368fdp+1 (2.4262638): cos(pi/2 - |x|)
    const double ax = from_bits(bits(x) & 0x7fffffffffffffffull);
    const double t = kHp0 - ax;
    return copysign_of(cos_tab(t, kHp1, tab), x);
  }
  if (k < 0x419921fbu) {          // |x| < 105414350: x = n*pi/2 + (b + db)
    const double t = fmad(x, kHpInv, kToInt);
    const double xn = t - kToInt;
    double y = fmad(-xn, kMp1, x);
    y = fmad(-xn, kMp2, y);
    const double t2 = fmad(-xn, kPp3, y);
    double db = fmad(-kPp3, xn, y - t2);
    const double b = fmad(-xn, kPp4, t2);
    db = db + fmad(-xn, kPp4, t2 - b);
    const uint32_t n = (uint32_t)bits(t) & 3u;
    double r;
    if (n & 1u) {
      r = cos_tab(b, db, tab);
    } else {
      const double ab = from_bits(bits(b) & 0x7fffffffffffffffull);
      r = ab < kTaylorMax ? taylor(b, db) : sin_tab(b, db, tab);
    }
    return (n & 2u) ? -r : r;
  }
  return from_bits(0x7ff8000000000000ull);  // outside the supported domain
}

GSIN_HD double sin(double x, const double* tab) { return sin(x, PtrTable{tab}); }

// sin(x) again, arranged for the LASM chain, whose arguments
// pi*mu*(y+3)*x*(1-x) lie in [0, pi] up to rounding:
//  * glibc's cos(pi/2 - x) branch, 44% of LASM arguments, is tested first,
//    with one branch (testing the sin table's 36% second as its own range
//    measured no better);
//  * the two range tests fail for negative x and NaN; for positive x every
//    one of these branches yields a positive value, so
//    glibc's copysign(result, x) is the identity and is left out (it cost an
//    integer round trip on the chain).
// Everything else (tiny, the Cody-Waite branch, negative, NaN) takes sin()
// itself, so sin_0pi(x) == sin(x) for every x.
template <class Tab>
GSIN_HD double sin_0pi(double x, const Tab& tab) {
  // The branch tests compare x itself with the doubles whose high words are
  // glibc's thresholds (for x >= +0, hi(x) >= K <=> x >= double(K << 32));
  // an FP64 compare avoids moving the fresh FP64 result to the integer pipe.
  if (x >= 0x1.b6p-1 && x < 0x1.368fdp+1) return cos_tab(kHp0 - x, kHp1, tab);
  if (x >= 0x1p-26 && x < 0x1.b6p-1)
    return x < kTaylorMax ? taylor(x, 0.0) : sin_tab_mag(x, 0.0, tab);
  return sin(x, tab);
}

GSIN_HD double sin_0pi(double x, const double* tab) { return sin_0pi(x, PtrTable{tab}); }

}  // namespace gsin
