// Test helper (tests/test_lasm.py): compares the product's host/device
// restatement of glibc sin (paper_2302_07411_b200/csrc/glibc_sin.cuh, host
// build: gsin::sin and the chain's arrangement gsin::sin_0pi) with this
// host's libm sin() bit for bit, over seeded random
// arguments in every branch of the algorithm, every double around the
// branch edges, and whole LASM orbits (chaos.cpp:34-38).
// Prints "<cases> <mismatches>" and the first mismatches.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "glibc_sin.cuh"

static const double kTab[gsin::kTableDoubles] = {
#include "glibc_sincostab.inc"
};

static long cases = 0, bad = 0;

// sin_0pi: the LASM chain's arrangement of the same function
static void check_0pi(double x) {
  const double a = gsin::sin_0pi(x, kTab), w = std::sin(x);
  if (std::memcmp(&a, &w, 8) != 0) {
    if (bad < 5) std::printf("sin_0pi x=%a ours=%a libm=%a\n", x, a, w);
    ++bad;
  }
}

static void check(double x) {
  const double a = gsin::sin(x, kTab), w = std::sin(x);
  ++cases;
  check_0pi(x);
  if (std::memcmp(&a, &w, 8) != 0) {
    if (bad < 5) std::printf("x=%a ours=%a libm=%a\n", x, a, w);
    ++bad;
  }
}

int main(int argc, char** argv) {
  const long per = argc > 1 ? std::atol(argv[1]) : 200000;
  std::mt19937_64 rng(20230214);
  const double ranges[][2] = {
      {0.0, 0x1p-26},        {0x1p-26, 0.126},      {0.126, 0.85546875},
      {0.85546875, 2.4262639}, {2.4262600, 2.4262700}, {2.4262638, 3.1415927},
      {3.1415927, 26.0},     {26.0, 1.0e6},         {-26.0, 0.0},
      {0.1259, 0.1261},      {0.8554, 0.8556},      {2.356, 2.357}};
  for (const auto& r : ranges) {
    std::uniform_real_distribution<double> u(r[0], r[1]);
    for (long i = 0; i < per; ++i) check(u(rng));
  }
  // every double around the branch thresholds
  const double edges[] = {0x1p-26, 0.126, 0.85546875, 0x1.368fdp+1, 2.42626953125,
                          3.14159265358979, 105414350.0 * 0.999999};
  for (double e : edges) {
    double v = e;
    for (int k = 0; k < 2000; ++k) v = std::nextafter(v, 0.0);
    for (int k = 0; k < 4000; ++k, v = std::nextafter(v, 1e300)) check(v);
  }
  // LASM orbits, as the reference iterates them
  std::uniform_real_distribution<double> u01(0.0, 1.0), umu(0.44, 0.93);
  const double pi = 3.14159265358979323846;
  for (int lane = 0; lane < 16; ++lane) {
    double x = u01(rng), y = u01(rng);
    const double mu = lane == 0 ? 1.0 : umu(rng);
    for (long i = 0; i < per / 2; ++i) {
      const double ax = pi * mu * (y + 3.0) * x * (1.0 - x);
      check(ax);
      x = std::sin(ax);
      const double ay = pi * mu * (x + 3.0) * y * (1.0 - y);
      check(ay);
      y = std::sin(ay);
    }
  }
  std::printf("%ld %ld\n", cases, bad);
  return 0;
}
