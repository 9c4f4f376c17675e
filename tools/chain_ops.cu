// FP64 issue pressure in the chain step.  Tool, not product.
// The product step (A) issues 14 FP64 instructions per iteration (3 DSETP,
// 3 DADD, 1 DMUL, 7 DFMA) at one per 2 cycles per SM sub-partition, next to
// a ~40-cycle dependent path.  The variants compute bit-identical orbits with
// fewer FP64 instructions:
//   B  fold predicate from the high word (ISETP; exact for every x != 0.5,
//      and x == 0.5 is a guard value the verifier re-decides anyway)
//   C  B + x<p and x>cthr as 64-bit integer compares of the bit patterns
//   D  one correction FMA per divisor, constants selected by fold
//      (cases A/C share corr_p, B/D share corr_q): 11 FP64 instead of 14
//   E  C + D (9 FP64)
//   F  C, case D selected last: other = cc ? yc : (a ? ya : yb) (cc implies
//      fold, a implies !fold), x' = (fold & !cc) ? yd : other
//   G  F with the last select as a LOP3 bit-select per 32-bit half (mask from
//      the predicates), which ptxas cannot re-canonicalise into FSEL levels
//   H  C with cc ? yc : (fold ? yd : (a ? ya : yb))
//   J  C as predicated assignments: y = yb; if (a) y = ya; if (fold) y = yd;
//      if (cc) y = yc
//   N  C unrolled by 16
//   K  C with each orbit store as `asm volatile` st.global.f64 (not sunk)
//   L  C with __stcg stores
//   U4, U2  C unrolled by 4 / 2
// Prints ns/iteration and checks every variant's orbit against A's.
// Measured (B200, 1965 MHz, 128 lanes x 2^18 iterations), ns/iteration:
//   A 26.18  B 25.61  C 25.36  D 31.85  E 31.91  F 28.79  G 28.67  H 28.72
//   J 28.67  N 25.29  K 25.36  L 25.35  U4 28.02  U2 25.67
// C is the product step since r01h (N's gain reverses inside the product).
// Selecting case D last (F, G) or sharing corrections (D, E) lengthens the
// path the hardware actually sees; the store form (K, L) does not matter;
// the 2 IMAD.MOV per 8 steps come from the halves of a predicated select
// landing in unpaired registers and survive every unroll factor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/chain_ops.cu -o tools/chain_ops
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

struct LaneConst {
  double p, q, yh_p, yl_p, yh_q, yl_q, cthr, a_b, a_d;
};

__device__ __forceinline__ bool gt_bits(double x, double y) {  // x, y >= 0
  return __double_as_longlong(x) > __double_as_longlong(y);
}

template <int V>
__device__ __forceinline__ double step(double x, const LaneConst& c) {
  const bool fold = (V == 0) ? x > 0.5 : __double2hiint(x) >= 0x3FE00000;
  const bool int_cmp = V == 2 || V >= 4;
  const bool a = int_cmp ? gt_bits(c.p, x) : x < c.p;
  const bool cc = int_cmp ? gt_bits(x, c.cthr) : x > c.cthr;
  const double t1 = __dsub_rn(1.0, x);
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  if (V >= 5) {
    const double ya = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
    const double yb = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
    const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
    const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
    const double other = cc ? yc : (a ? ya : yb);
    const bool isd = fold & !cc;
    if (V == 5) return isd ? yd : other;
    const unsigned m = isd ? 0xFFFFFFFFu : 0u;
    unsigned lo, hi;
    // (yd & m) | (other & ~m): LUT 0xCA over (m, yd, other) = (a & b) | (~a & c)
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(lo) : "r"(m), "r"(unsigned(__double2loint(yd))),
        "r"(unsigned(__double2loint(other))));
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(hi) : "r"(m), "r"(unsigned(__double2hiint(yd))),
        "r"(unsigned(__double2hiint(other))));
    return __hiloint2double(int(hi), int(lo));
  }
  if (V == 7 || V == 8) {
    const double ya = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
    const double yb = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
    const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
    const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
    if (V == 7) return cc ? yc : (fold ? yd : (a ? ya : yb));
    double y = yb;
    if (a) y = ya;
    if (fold) y = yd;
    if (cc) y = yc;
    return y;
  }
  if (V == 3 || V == 4) {
    const double gp = fold ? -c.yl_p : c.yl_p, ap = fold ? c.yl_p : 0.0;
    const double gq = fold ? -c.yl_q : c.yl_q, aq = fold ? c.a_d : c.a_b;
    const double cp = __fma_rn(x, gp, ap), cq = __fma_rn(x, gq, aq);
    const double ya = __fma_rn(x, c.yh_p, cp), yc = __fma_rn(t1, c.yh_p, cp);
    const double yb = __fma_rn(nb, c.yh_q, cq), yd = __fma_rn(nd, c.yh_q, cq);
    return fold ? (cc ? yc : yd) : (a ? ya : yb);
  }
  const double ya = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
  const double yb = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
  const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
  const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
  return fold ? (cc ? yc : yd) : (a ? ya : yb);
}

template <int V>
__global__ void __launch_bounds__(128, 1)
    k(double* state, const LaneConst* lcs, double* orbit, uint32_t iters, uint32_t nl) {
  constexpr int S = V >= 9 ? 2 : V;  // N, K, L: the C step
  constexpr int U = V == 9 ? 16 : V == 12 ? 4 : V == 13 ? 2 : 8;
  const uint32_t l = threadIdx.x;
  const LaneConst c = lcs[l];
  double x = state[l];
  double* o = orbit + l;
  for (uint32_t i = 0; i < iters; i += U) {
#pragma unroll
    for (int t = 0; t < U; ++t) {
      x = step<S>(x, c);
      if (V == 10)
        asm volatile("st.global.f64 [%0], %1;" ::"l"(o + size_t(t) * nl), "d"(x) : "memory");
      else if (V == 11)
        __stcg(o + size_t(t) * nl, x);
      else
        o[size_t(t) * nl] = x;
    }
    o += size_t(U) * nl;
  }
  state[l] = x;
}

static LaneConst make(double p) {
  LaneConst c{};
  volatile double half = 0.5, one = 1.0;
  c.p = p;
  c.q = half - p;
  c.yh_p = one / c.p;
  c.yl_p = std::fma(-c.p, c.yh_p, 1.0) / c.p;
  c.yh_q = one / c.q;
  c.yl_q = std::fma(-c.q, c.yh_q, 1.0) / c.q;
  double t = one - c.p;
  volatile double d = t - one;
  if (d + c.p < 0.0) t = std::nextafter(t, 0.0);
  c.cthr = t;
  c.a_b = -c.p * c.yl_q;
  c.a_d = (one - c.p) * c.yl_q;
  return c;
}

int main() {
  const int T = 128;
  const uint32_t iters = 1u << 18;
  std::vector<LaneConst> h(T);
  std::vector<double> x0(T);
  for (int i = 0; i < T; ++i) {
    h[i] = make(0.01 + 0.48 * ((i * 37 % 101) / 101.0));
    x0[i] = (i * 53 % 97) / 97.0 + 0.001;
  }
  LaneConst* dl;
  double *dx, *dorb;
  cudaMalloc(&dl, T * sizeof(LaneConst));
  cudaMalloc(&dx, T * 8);
  cudaMalloc(&dorb, size_t(iters) * T * 8);
  cudaMemcpy(dl, h.data(), T * sizeof(LaneConst), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  void (*ks[])(double*, const LaneConst*, double*, uint32_t, uint32_t) = {k<0>, k<1>, k<2>,
                                                                         k<3>, k<4>, k<5>, k<6>,
                                                                         k<7>, k<8>, k<9>, k<10>, k<11>, k<12>, k<13>};
  const char* names[] = {"A product (14 FP64)", "B fold from hi word", "C integer predicates",
                         "D shared corrections", "E C + D",
                         "F C, case D selected last", "G F with LOP3 bit-select",
                         "H C, cc-first select", "J C, predicated assigns", "N C, unroll 16",
                         "K C, asm volatile stores", "L C, __stcg stores",
                         "U4 C, unroll 4", "U2 C, unroll 2"};
  std::vector<double> ref(size_t(iters) * T), got(size_t(iters) * T);
  for (int m = 0; m < 14; ++m) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(dx, x0.data(), T * 8, cudaMemcpyHostToDevice);
      cudaEventRecord(a);
      ks[m]<<<1, T>>>(dx, dl, dorb, iters, T);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::fmin(best, ms);
    }
    cudaMemcpy(m ? got.data() : ref.data(), dorb, ref.size() * 8, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    if (m)
      for (size_t i = 0; i < ref.size(); ++i) bad += std::memcmp(&ref[i], &got[i], 8) != 0;
    printf("%-26s %.2f ns/iter  orbit mismatches vs A: %zu\n", names[m], best * 1e6 / iters,
           bad);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
