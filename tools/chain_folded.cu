// Folded-state chain step (experiment; tool, not product).  The product step
// carries x and computes four quotient candidates (11 FP64 instructions).
// Here the loop carries u = min(x, 1 - x) (the map is symmetric: F(x) =
// F(1 - x)), so only the two unfolded candidates are needed, plus their
// complements for the next fold: 7 FP64 instructions
//   nb = u - p; cA = u*yl_p; cB = fma(u, yl_q, a_b);
//   ya = fma(u, yh_p, cA); yb = fma(nb, yh_q, cB); ta = 1 - ya; tb = 1 - yb
//   u' = a ? (ya >= 0.5 ? ta : ya) : (yb >= 0.5 ? tb : yb)
// Checkpoint form (one store per 8 steps); the check folds the product
// step's orbit and compares.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/chain_folded.cu -o tools/chain_folded
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

struct LaneConst {
  double p, q, yh_p, yl_p, yh_q, yl_q, cthr, a_b, a_d;
};

__device__ __forceinline__ bool gt_bits(double x, double y) {
  return __double_as_longlong(x) > __double_as_longlong(y);
}

__device__ __forceinline__ double step_product(double x, const LaneConst& c) {
  const bool a = gt_bits(c.p, x), cc = gt_bits(x, c.cthr);
  const bool fold = __double2hiint(x) >= 0x3FE00000;
  const double t1 = __dsub_rn(1.0, x);
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  const double ya = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
  const double yb = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
  const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
  const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
  return fold ? (cc ? yc : yd) : (a ? ya : yb);
}

template <int V>
__device__ __forceinline__ double step_folded(double u, const LaneConst& c) {
  const bool a = gt_bits(c.p, u);
  const double nb = __dsub_rn(u, c.p);
  const double ya = __fma_rn(u, c.yh_p, __dmul_rn(u, c.yl_p));
  const double yb = __fma_rn(nb, c.yh_q, __fma_rn(u, c.yl_q, c.a_b));
  const double ta = __dsub_rn(1.0, ya);
  const double tb = __dsub_rn(1.0, yb);
  const bool fa = __double2hiint(ya) >= 0x3FE00000, fb = __double2hiint(yb) >= 0x3FE00000;
  if (V == 0) return a ? (fa ? ta : ya) : (fb ? tb : yb);
  if (V == 1) {  // tb last
    const double wa = fa ? ta : ya;
    const double other = a ? wa : yb;
    return (!a && fb) ? tb : other;
  }
  if (V == 2) {  // select y first, then complement of the selected
    const double y = a ? ya : yb;
    const double t = a ? ta : tb;
    return __double2hiint(y) >= 0x3FE00000 ? t : y;
  }
  if (V == 3) {  // four predicated assignments
    const bool pa1 = a & fa, pa0 = a & !fa, pb1 = (!a) & fb;
    double r = yb;
    if (pb1) r = tb;
    if (pa0) r = ya;
    if (pa1) r = ta;
    return r;
  }
  if (V == 4) {  // 64-bit integer selects
    const long long ia = fa ? __double_as_longlong(ta) : __double_as_longlong(ya);
    const long long ib = fb ? __double_as_longlong(tb) : __double_as_longlong(yb);
    return __longlong_as_double(a ? ia : ib);
  }
  // V == 5: halves selected separately and re-paired
  const int lo = a ? (fa ? __double2loint(ta) : __double2loint(ya))
                   : (fb ? __double2loint(tb) : __double2loint(yb));
  const int hi = a ? (fa ? __double2hiint(ta) : __double2hiint(ya))
                   : (fb ? __double2hiint(tb) : __double2hiint(yb));
  return __hiloint2double(hi, lo);
}

template <int V>
__global__ void __launch_bounds__(128, 1)
    k(double* state, const LaneConst* lcs, double* ck, uint32_t iters, uint32_t nl) {
  const uint32_t l = threadIdx.x;
  const LaneConst c = lcs[l];
  double x = state[l];
  if (V > 0 && x >= 0.5) x = 1.0 - x;
  double* o = ck + l;
  for (uint32_t i = 0; i < iters; i += 32) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
#pragma unroll
      for (int t = 0; t < 8; ++t) x = V == 0 ? step_product(x, c) : step_folded<V - 1>(x, c);
      o[size_t(g) * nl] = x;
    }
    o += size_t(4) * nl;
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
  const uint32_t iters = 1u << 20;
  std::vector<LaneConst> h(T);
  std::vector<double> x0(T);
  for (int i = 0; i < T; ++i) {
    h[i] = make(0.01 + 0.48 * ((i * 37 % 101) / 101.0));
    x0[i] = (i * 53 % 97) / 97.0 + 0.001;
  }
  LaneConst* dl;
  double *dx, *dck;
  const size_t nck = size_t(iters / 8) * T;
  cudaMalloc(&dl, T * sizeof(LaneConst));
  cudaMalloc(&dx, T * 8);
  cudaMalloc(&dck, nck * 8);
  cudaMemcpy(dl, h.data(), T * sizeof(LaneConst), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  void (*ks[])(double*, const LaneConst*, double*, uint32_t, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  const char* names[] = {"product step (11 FP64)", "folded, nested selects (7 FP64)",
                         "folded, tb selected last", "folded, select then fold",
                         "folded, predicated assigns", "folded, 64-bit int selects",
                         "folded, halves re-paired"};
  std::vector<double> ref(nck), got(nck);
  for (int m = 0; m < 7; ++m) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(dx, x0.data(), T * 8, cudaMemcpyHostToDevice);
      cudaEventRecord(a);
      ks[m]<<<1, T>>>(dx, dl, dck, iters, T);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::fmin(best, ms);
    }
    cudaMemcpy(m ? got.data() : ref.data(), dck, nck * 8, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    if (m)
      for (size_t i = 0; i < nck; ++i) {
        const double f = ref[i] >= 0.5 ? 1.0 - ref[i] : ref[i];
        bad += std::memcmp(&f, &got[i], 8) != 0;
      }
    printf("%-34s %.2f ns/iter (%.1f cycles at 1965 MHz)  mismatches vs folded product orbit: %zu\n",
           names[m], best * 1e6 / iters, best * 1e6 / iters * 1.965, bad);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
