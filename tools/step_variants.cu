// Time per dependent PLCM iteration for alternative step formulations.
// Tool, not product.  Each variant: 128 threads (4 warps, one per SMSP),
// one chain per thread, N iterations; reports ns/iteration and checks the
// orbit against the IEEE-division reference step (mismatch count).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/step_variants.cu -o tools/step_variants
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>

struct LC {
  double p, q, rp, rq, hp, hq;  // Markstein constants
  double yhp, ylp, yhq, ylq;    // 1/p, 1/q as double-double
  double cthr;                  // largest double <= 1 - p  (x > cthr <=> 1-x < p)
  double aB, aD;                // alpha of the correction term, cases B and D
  unsigned plo;
};

__device__ __forceinline__ double ref_step(double x, double p, double q) {
  const double f = x > 0.5 ? __dsub_rn(1.0, x) : x;
  double y = f < p ? __ddiv_rn(f, p) : __ddiv_rn(__dsub_rn(f, p), q);
  if (y == 0.0 || y == p || y == 0.5 || y == 1.0) {
    y = __dadd_rn(y, 0x1p-52);
    if (y > 1.0) y = __dsub_rn(y, 1.0);
  }
  return y;
}

// V0: current product step (fold select, Markstein 3-op, verify)
__device__ __forceinline__ double v0(double x, const LC& c, bool& flag) {
  const double folded = __dsub_rn(1.0, x);
  const double f = x > 0.5 ? folded : x;
  const bool low = f < c.p;
  const double shifted = __dsub_rn(f, c.p);
  const double num = low ? f : shifted;
  const double rcp = low ? c.rp : c.rq;
  const double den = low ? c.p : c.q;
  const double q0 = __dmul_rn(num, rcp);
  const double r0 = __fma_rn(-q0, den, num);
  const double y = __fma_rn(r0, rcp, q0);
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y)), lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

// V1: V0 without verification (chain floor of the current formulation)
__device__ __forceinline__ double v1(double x, const LC& c, bool& flag) {
  const double folded = __dsub_rn(1.0, x);
  const double f = x > 0.5 ? folded : x;
  const bool low = f < c.p;
  const double shifted = __dsub_rn(f, c.p);
  const double num = low ? f : shifted;
  const double rcp = low ? c.rp : c.rq;
  const double den = low ? c.p : c.q;
  const double q0 = __dmul_rn(num, rcp);
  const double r0 = __fma_rn(-q0, den, num);
  return __fma_rn(r0, rcp, q0);
}

// V2: compares straight from x, numerator = base - sub (one DADD after the
// fold select), 2-op double-double division, verify.
__device__ __forceinline__ double v2(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool low = c1 ? (x > c.cthr) : (x < c.p);
  const double t1 = __dsub_rn(1.0, x);
  const double base = c1 ? t1 : x;
  const double sub = low ? 0.0 : c.p;
  const double num = __dsub_rn(base, sub);
  const double yh = low ? c.yhp : c.yhq;
  const double yl = low ? c.ylp : c.ylq;
  const double den = low ? c.p : c.q;
  const double e = __dmul_rn(num, yl);
  const double y = __fma_rn(num, yh, e);
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y)), lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

// V3: V2 without verification
__device__ __forceinline__ double v3(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool low = c1 ? (x > c.cthr) : (x < c.p);
  const double t1 = __dsub_rn(1.0, x);
  const double base = c1 ? t1 : x;
  const double sub = low ? 0.0 : c.p;
  const double num = __dsub_rn(base, sub);
  const double yh = low ? c.yhp : c.yhq;
  const double yl = low ? c.ylp : c.ylq;
  const double e = __dmul_rn(num, yl);
  return __fma_rn(num, yh, e);
}

// V4: numerator via two predicated subtractions (no fold select):
// num = c1 ? (t1 - sub) : (x - sub) computed as both then select.
__device__ __forceinline__ double v4(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool low = c1 ? (x > c.cthr) : (x < c.p);
  const double t1 = __dsub_rn(1.0, x);
  const double sub = low ? 0.0 : c.p;
  const double n1 = __dsub_rn(t1, sub);
  const double n0 = __dsub_rn(x, sub);
  const double num = c1 ? n1 : n0;
  const double yh = low ? c.yhp : c.yhq;
  const double yl = low ? c.ylp : c.ylq;
  const double den = low ? c.p : c.q;
  const double e = __dmul_rn(num, yl);
  const double y = __fma_rn(num, yh, e);
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y)), lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

// V5: PTX with predicated writes of the numerator (cases are disjoint).
__device__ __forceinline__ double v5(double x, const LC& c, bool& flag) {
  double num, yh, yl, den, dh;
  asm volatile(
      "{\n\t.reg .pred c1, pl, pA, pB, pC, pD;\n\t"
      ".reg .f64 t1;\n\t"
      "setp.gt.f64 c1, %5, 0d3FE0000000000000;\n\t"
      "sub.rn.f64 t1, 0d3FF0000000000000, %5;\n\t"
      "setp.gt.f64 pC, %5, %7;\n\t"       // x > cthr  (case C, implies c1)
      "setp.lt.f64 pA, %5, %6;\n\t"       // x < p     (case A, implies !c1)
      "or.pred pl, pA, pC;\n\t"           // low
      "not.pred pB, c1;\n\t"
      "and.pred pB, pB, !pA;\n\t"         // B: !c1 & !A
      "and.pred pD, c1, !pC;\n\t"         // D: c1 & !C
      "@pA mov.f64 %0, %5;\n\t"
      "@pB sub.rn.f64 %0, %5, %6;\n\t"
      "@pC mov.f64 %0, t1;\n\t"
      "@pD sub.rn.f64 %0, t1, %6;\n\t"
      "selp.f64 %1, %8, %10, pl;\n\t"
      "selp.f64 %2, %9, %11, pl;\n\t"
      "selp.f64 %3, %6, %12, pl;\n\t"
      "selp.f64 %4, %13, %14, pl;\n\t"
      "}"
      : "=d"(num), "=d"(yh), "=d"(yl), "=d"(den), "=d"(dh)
      : "d"(x), "d"(c.p), "d"(c.cthr), "d"(c.yhp), "d"(c.ylp), "d"(c.yhq), "d"(c.ylq),
        "d"(c.q), "d"(c.hp), "d"(c.hq));
  const double e = __dmul_rn(num, yl);
  const double y = __fma_rn(num, yh, e);
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y)), lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(dh, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

// V6: all four quotients speculated from x, final 4-way select.
__device__ __forceinline__ double v6(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool lowA = x < c.p, lowC = x > c.cthr;
  const double t1 = __dsub_rn(1.0, x);
  const double n0 = __dsub_rn(x, c.p);
  const double n1 = __dsub_rn(t1, c.p);
  const double yA = __fma_rn(x, c.yhp, __dmul_rn(x, c.ylp));
  const double yB = __fma_rn(n0, c.yhq, __dmul_rn(n0, c.ylq));
  const double yC = __fma_rn(t1, c.yhp, __dmul_rn(t1, c.ylp));
  const double yD = __fma_rn(n1, c.yhq, __dmul_rn(n1, c.ylq));
  const double y = c1 ? (lowC ? yC : yD) : (lowA ? yA : yB);
  const bool low = c1 ? lowC : lowA;
  const double num = c1 ? (lowC ? t1 : n1) : (lowA ? x : n0);
  const double den = low ? c.p : c.q;
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y)), lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

// V7: correction term from x (4 FMAs, selected), num via base-sub, 1 DFMA on
// the chain after num.  No verification.
__device__ __forceinline__ double v7(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool low = (x < c.p) | (x > c.cthr);
  const double t1 = __dsub_rn(1.0, x);
  const double base = c1 ? t1 : x;
  const double sub = low ? 0.0 : c.p;
  const double num = __dsub_rn(base, sub);
  const double yh = low ? c.yhp : c.yhq;
  const double cA = __dmul_rn(x, c.ylp);
  const double cB = __fma_rn(x, c.ylq, c.aB);
  const double cC = __fma_rn(-x, c.ylp, c.ylp);
  const double cD = __fma_rn(-x, c.ylq, c.aD);
  const double cl = c1 ? cC : cA;
  const double ch = c1 ? cD : cB;
  const double corr = low ? cl : ch;
  return __fma_rn(num, yh, corr);
}

// V8: V7 + producer-side cost of handing y to a verifier warp (STS per step)
template <int K>
__device__ __forceinline__ double v8(double x, const LC& c, bool& flag, double* ring, int t) {
  const double y = v7(x, c, flag);
  ring[(t & 15) * 128 + threadIdx.x] = y;
  return y;
}

// V9: V7 but numerator via predicated subtraction (asm), correction as V7
__device__ __forceinline__ double v9(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const double cA = __dmul_rn(x, c.ylp);
  const double cB = __fma_rn(x, c.ylq, c.aB);
  const double cC = __fma_rn(-x, c.ylp, c.ylp);
  const double cD = __fma_rn(-x, c.ylq, c.aD);
  double num, yh, corr;
  asm volatile(
      "{\n\t.reg .pred c1, pl, pA, pC;\n\t.reg .f64 t1, b, cl, ch;\n\t"
      "setp.gt.f64 c1, %3, 0d3FE0000000000000;\n\t"
      "setp.lt.f64 pA, %3, %4;\n\t"
      "setp.gt.f64 pC, %3, %5;\n\t"
      "or.pred pl, pA, pC;\n\t"
      "sub.rn.f64 t1, 0d3FF0000000000000, %3;\n\t"
      "selp.f64 b, t1, %3, c1;\n\t"
      "mov.f64 %0, b;\n\t"
      "@!pl sub.rn.f64 %0, b, %4;\n\t"
      "selp.f64 %1, %6, %7, pl;\n\t"
      "selp.f64 cl, %10, %8, c1;\n\t"
      "selp.f64 ch, %11, %9, c1;\n\t"
      "selp.f64 %2, cl, ch, pl;\n\t"
      "}"
      : "=d"(num), "=d"(yh), "=d"(corr)
      : "d"(x), "d"(c.p), "d"(c.cthr), "d"(c.yhp), "d"(c.yhq), "d"(cA), "d"(cB), "d"(cC),
        "d"(cD));
  return __fma_rn(num, yh, corr);
}

// V10: V7 with the verification inline (for comparison with V2)
__device__ __forceinline__ double v10(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool low = (x < c.p) | (x > c.cthr);
  const double t1 = __dsub_rn(1.0, x);
  const double base = c1 ? t1 : x;
  const double sub = low ? 0.0 : c.p;
  const double num = __dsub_rn(base, sub);
  const double yh = low ? c.yhp : c.yhq;
  const double cA = __dmul_rn(x, c.ylp);
  const double cB = __fma_rn(x, c.ylq, c.aB);
  const double cC = __fma_rn(-x, c.ylp, c.ylp);
  const double cD = __fma_rn(-x, c.ylq, c.aD);
  const double cl = c1 ? cC : cA;
  const double ch = c1 ? cD : cB;
  const double corr = low ? cl : ch;
  const double y = __fma_rn(num, yh, corr);
  const double den = low ? c.p : c.q;
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y)), lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

// V11: product formulation (4 numerators, single 4-way select)
__device__ __forceinline__ double v11(double x, const LC& c, bool& flag) {
  const bool c1 = x > 0.5;
  const bool low = (x < c.p) | (x > c.cthr);
  const double t1 = __dsub_rn(1.0, x);
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  const double num = low ? (c1 ? t1 : x) : (c1 ? nd : nb);
  const double yh = low ? c.yhp : c.yhq;
  const double ca = __dmul_rn(x, c.ylp);
  const double cb = __fma_rn(x, c.ylq, c.aB);
  const double cc = __fma_rn(-x, c.ylp, c.ylp);
  const double cd = __fma_rn(-x, c.ylq, c.aD);
  const double corr = low ? (c1 ? cc : ca) : (c1 ? cd : cb);
  return __fma_rn(num, yh, corr);
}

template <int V>
__device__ __forceinline__ double stepv(double x, const LC& c, bool& f) {
  if (V == 0) return v0(x, c, f);
  if (V == 1) return v1(x, c, f);
  if (V == 2) return v2(x, c, f);
  if (V == 3) return v3(x, c, f);
  if (V == 4) return v4(x, c, f);
  if (V == 5) return v5(x, c, f);
  if (V == 6) return v6(x, c, f);
  if (V == 7) return v7(x, c, f);
  if (V == 9) return v9(x, c, f);
  if (V == 11) return v11(x, c, f);
  return v10(x, c, f);
}

template <int V>
__global__ void k_run(const LC* lcs, double* xs, int iters, int* flags) {
  __shared__ double ring[16 * 128];
  const LC c = lcs[threadIdx.x];
  double x = xs[threadIdx.x];
  bool flag = false;
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (V == 8) x = v8<0>(x, c, flag, ring, i + t);
      else x = stepv<V>(x, c, flag);
    }
  }
  if (V == 8) x += ring[threadIdx.x] * 0.0;
  xs[threadIdx.x] = x;
  flags[threadIdx.x] = flag;
}

template <int V>
__global__ void k_sparse(const LC* lcs, double* xs, int iters, int* flags, int per_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane >= per_warp) return;
  const int l = warp * per_warp + lane;
  const LC c = lcs[l];
  double x = xs[l];
  bool flag = false;
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) x = stepv<V>(x, c, flag);
  }
  xs[l] = x;
  flags[l] = flag;
}

__global__ void k_ref(const LC* lcs, double* xs, int iters) {
  const LC c = lcs[threadIdx.x];
  double x = xs[threadIdx.x];
  for (int i = 0; i < iters; ++i) x = ref_step(x, c.p, c.q);
  xs[threadIdx.x] = x;
}

static LC make(double p) {
  LC c{};
  volatile double half = 0.5, one = 1.0;
  c.p = p;
  c.q = half - p;
  c.rp = one / c.p;
  c.rq = one / c.q;
  c.hp = 0.5 * c.p;
  c.hq = 0.5 * c.q;
  // 1/d = yh + yl to ~2^-106: the residual 1 - d*yh is exact under FMA
  c.yhp = one / c.p;
  c.ylp = std::fma(-c.p, c.yhp, 1.0) / c.p;
  c.yhq = one / c.q;
  c.ylq = std::fma(-c.q, c.yhq, 1.0) / c.q;
  // cthr = largest double <= 1 - p; t - 1 is exact and sign(RN(d + p)) is exact
  double t = one - c.p;
  volatile double d = t - one;
  if (d + c.p < 0.0) t = nextafter(t, 0.0);
  c.cthr = t;
  c.aB = -c.p * c.ylq;
  c.aD = (1.0 - c.p) * c.ylq;
  uint64_t b;
  memcpy(&b, &c.p, 8);
  c.plo = unsigned(b);
  return c;
}

int main() {
  const int T = 128, iters = 1 << 20;
  std::vector<LC> h(T);
  std::vector<double> x0(T);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&] { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return double(s >> 11) * 0x1p-53; };
  for (int i = 0; i < T; ++i) {
    h[i] = make(0.01 + 0.48 * rnd());
    x0[i] = rnd();
  }
  LC* d_lc;
  double *d_x, *d_ref;
  int* d_f;
  cudaMalloc(&d_lc, T * sizeof(LC));
  cudaMalloc(&d_x, T * 8);
  cudaMalloc(&d_ref, T * 8);
  cudaMalloc(&d_f, T * 4);
  cudaMemcpy(d_lc, h.data(), T * sizeof(LC), cudaMemcpyHostToDevice);
  cudaMemcpy(d_ref, x0.data(), T * 8, cudaMemcpyHostToDevice);
  k_ref<<<1, T>>>(d_lc, d_ref, iters);
  std::vector<double> ref(T);
  cudaMemcpy(ref.data(), d_ref, T * 8, cudaMemcpyDeviceToHost);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, void (*k)(const LC*, double*, int, int*)) {
    cudaMemcpy(d_x, x0.data(), T * 8, cudaMemcpyHostToDevice);
    k<<<1, T>>>(d_lc, d_x, 1024, d_f);  // warm
    cudaMemcpy(d_x, x0.data(), T * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    k<<<1, T>>>(d_lc, d_x, iters, d_f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<double> got(T);
    std::vector<int> fl(T);
    cudaMemcpy(got.data(), d_x, T * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(fl.data(), d_f, T * 4, cudaMemcpyDeviceToHost);
    int mism = 0, flags = 0;
    for (int i = 0; i < T; ++i) {
      mism += got[i] != ref[i];
      flags += fl[i];
    }
    printf("%-34s %7.2f ns/iter  (%6.1f cyc@1965)  orbit mismatches %d/%d  flagged lanes %d\n",
           name, ms * 1e6 / iters, ms * 1e6 / iters * 1.965, mism, T, flags);
  };
  run("V0 current (Markstein+verify)", k_run<0>);
  run("V1 current, no verify", k_run<1>);
  run("V2 direct cmp, base-sub, DD div, verify", k_run<2>);
  run("V3 V2 no verify", k_run<3>);
  run("V4 two subs + select, verify", k_run<4>);
  run("V5 PTX predicated num, verify", k_run<5>);
  run("V6 4 quotients + select, verify", k_run<6>);
  run("V7 corr-from-x, no verify", k_run<7>);
  run("V8 V7 + STS y (verifier hand-off)", k_run<8>);
  run("V9 V7 w/ predicated sub (asm)", k_run<9>);
  run("V10 V7 + inline verify", k_run<10>);
  run("V11 product (4 nums, 1 select)", k_run<11>);
  for (int pw : {32, 16, 8, 4, 2}) {
    cudaMemcpy(d_x, x0.data(), T * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    k_sparse<11><<<1, 128>>>(d_lc, d_x, iters, d_f, pw);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(d_x, x0.data(), T * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    k_sparse<9><<<1, 128>>>(d_lc, d_x, iters, d_f, pw);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms9;
    cudaEventElapsedTime(&ms9, a, b);
    printf("lanes/warp %2d: V11 %6.2f ns/iter   V9 %6.2f ns/iter\n", pw, ms * 1e6 / iters,
           ms9 * 1e6 / iters);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
