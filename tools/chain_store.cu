// Dynamic cost of the orbit stores in the chain kernel.  Tool, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/chain_store.cu -o tools/chain_store
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
struct LaneConst { double p, q, yh_p, yl_p, yh_q, yl_q, cthr, a_b, a_d, hp, hq; uint32_t plo, pad; };
__device__ __forceinline__ double step(double x, const LaneConst& c) {
  const bool c1 = x > 0.5;
  const bool low = (x < c.p) | (x > c.cthr);
  const double t1 = __dsub_rn(1.0, x);
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  const double f = c1 ? t1 : x;
  const double g = low ? c.yl_p : c.yl_q;
  const double a = low ? 0.0 : c.a_b;
  const double corr = __fma_rn(f, g, a);
  const double num = low ? f : (c1 ? nd : nb);
  const double yh = low ? c.yh_p : c.yh_q;
  return __fma_rn(num, yh, corr);
}
__device__ __forceinline__ double step4(double x, const LaneConst& c) {
  const bool pA = x < c.p, pC = x > c.cthr, c1 = x > 0.5;
  const double t1 = __dsub_rn(1.0, x);
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  const double yA = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
  const double yB = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
  const double yC = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
  const double yD = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
  return c1 ? (pC ? yC : yD) : (pA ? yA : yB);
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(double* state, const LaneConst* lcs, double* orbit, uint32_t iters, uint32_t nl) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  const LaneConst c = lcs[l];
  double x = state[l];
  double acc = 0;
  if (MODE == 0) {  // no stores
    for (uint32_t i = 0; i < iters; i += 8) {
#pragma unroll
      for (int t = 0; t < 8; ++t) { x = step(x, c); acc += 0.0 * x; }
    }
  } else if (MODE == 1) {  // STG.64 per step, iteration-major
    double* o = orbit + l;
    for (uint32_t i = 0; i < iters; i += 8) {
#pragma unroll
      for (int t = 0; t < 8; ++t) { x = step(x, c); o[size_t(t) * nl] = x; }
      o += size_t(8) * nl;
    }
  } else if (MODE == 2) {  // 8 steps then 4 x STG.128 (lane-major chunks)
    double* o = orbit + size_t(l) * 8;
    for (uint32_t i = 0; i < iters; i += 8) {
      double v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) { x = step(x, c); v[t] = x; }
#pragma unroll
      for (int t = 0; t < 8; t += 2) *reinterpret_cast<double2*>(o + t) = make_double2(v[t], v[t + 1]);
      o += size_t(8) * nl;
    }
  } else if (MODE == 4) {  // 4-quotient formulation, STG.64 per step
    double* o = orbit + l;
    for (uint32_t i = 0; i < iters; i += 8) {
#pragma unroll
      for (int t = 0; t < 8; ++t) { x = step4(x, c); o[size_t(t) * nl] = x; }
      o += size_t(8) * nl;
    }
  } else {  // 8 steps buffered then 8 STG.64 (iteration-major)
    double* o = orbit + l;
    for (uint32_t i = 0; i < iters; i += 8) {
      double v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) { x = step(x, c); v[t] = x; }
#pragma unroll
      for (int t = 0; t < 8; ++t) o[size_t(t) * nl] = v[t];
      o += size_t(8) * nl;
    }
  }
  state[l] = x + acc;
}
static LaneConst make(double p) {
  LaneConst c{};
  volatile double half = 0.5, one = 1.0;
  c.p = p; c.q = half - p;
  c.yh_p = one / c.p; c.yl_p = std::fma(-c.p, c.yh_p, 1.0) / c.p;
  c.yh_q = one / c.q; c.yl_q = std::fma(-c.q, c.yh_q, 1.0) / c.q;
  double t = one - c.p; volatile double d = t - one;
  if (d + c.p < 0.0) t = std::nextafter(t, 0.0);
  c.cthr = t; c.a_b = -c.p * c.yl_q; c.a_d = (one - c.p) * c.yl_q;
  return c;
}
int main() {
  const int T = 128, iters = 1 << 19;
  std::vector<LaneConst> h(T); std::vector<double> x0(T);
  for (int i = 0; i < T; ++i) { h[i] = make(0.01 + 0.48 * ((i * 37 % 101) / 101.0)); x0[i] = (i * 53 % 97) / 97.0 + 0.001; }
  LaneConst* dl; double *dx, *dorb;
  cudaMalloc(&dl, T * sizeof(LaneConst)); cudaMalloc(&dx, T * 8); cudaMalloc(&dorb, size_t(iters) * T * 8);
  cudaMemcpy(dl, h.data(), T * sizeof(LaneConst), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  void (*ks[])(double*, const LaneConst*, double*, uint32_t, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>};
  const char* names[] = {"no stores", "STG.64 per step", "4x STG.128 per 8 (lane-major)", "8x STG.64 per 8 buffered", "4-quotient step, STG.64"};
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(dx, x0.data(), T * 8, cudaMemcpyHostToDevice);
      cudaEventRecord(a);
      ks[m]<<<1, T>>>(dx, dl, dorb, iters, T);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%-34s %.2f ns/iter\n", names[m], ms * 1e6 / iters);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
