// Chain with inline verification + keystream emission vs the product chain
// (speculative step + orbit store, verified by a separate kernel).  Tool,
// not product: measures ns/iteration of the chain loop in both forms.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/chain_inline.cu -o tools/chain_inline
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

struct LaneConst {
  double p, q, yh_p, yl_p, yh_q, yl_q, cthr, a_b, a_d, hp, hq;
  uint32_t plo, pad;
};

__device__ __noinline__ double plcm_exact(double x, double p, double q) {
  if (x > 0.5) x = __dsub_rn(1.0, x);
  double y = x < p ? __ddiv_rn(x, p) : __ddiv_rn(__dsub_rn(x, p), q);
  if (y == 0.0 || y == p || y == 0.5 || y == 1.0) {
    y = __dadd_rn(y, 0x1p-52);
    if (y > 1.0) y = __dsub_rn(y, 1.0);
  }
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(128, 1)
    k(double* state, const LaneConst* lcs, double* orbit, uint8_t* ring, uint32_t iters,
      uint32_t nl, unsigned* redo) {
  const uint32_t l = threadIdx.x;
  const LaneConst c = lcs[l];
  double x = state[l];
  if (MODE == 0) {  // product: speculative step, orbit store per step
    double* o = orbit + l;
    for (uint32_t i = 0; i < iters; i += 8) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const bool a = x < c.p, cc = x > c.cthr, fold = x > 0.5;
        const double t1 = __dsub_rn(1.0, x), nb = __dsub_rn(x, c.p), nd = __dsub_rn(t1, c.p);
        const double ya = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
        const double yb = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
        const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
        const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
        x = fold ? (cc ? yc : yd) : (a ? ya : yb);
        o[size_t(t) * nl] = x;
      }
      o += size_t(8) * nl;
    }
  } else {  // inline verification of each step, block redo, direct emission
    const uint32_t odd = l & 1u;
    uint8_t* rb = ring + size_t(l >> 1) * size_t(iters) * 6 + (odd ? 24 : 0);
    unsigned nredo = 0;
    for (uint32_t i = 0; i < iters; i += 8) {
      const double xs = x;
      double y[8];
      bool bad = false;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double xi = x;
        const bool a = xi < c.p, cc = xi > c.cthr, fold = xi > 0.5;
        const double t1 = __dsub_rn(1.0, xi), nb = __dsub_rn(xi, c.p), nd = __dsub_rn(t1, c.p);
        const double ya = __fma_rn(xi, c.yh_p, __dmul_rn(xi, c.yl_p));
        const double yb = __fma_rn(nb, c.yh_q, __fma_rn(xi, c.yl_q, c.a_b));
        const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-xi, c.yl_p, c.yl_p));
        const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-xi, c.yl_q, c.a_d));
        x = fold ? (cc ? yc : yd) : (a ? ya : yb);
        y[t] = x;
        // verify x == RN(num / den) off the critical path
        const bool low = fold ? cc : a;
        const double num = fold ? (cc ? t1 : nd) : (a ? xi : nb);
        const double den = low ? c.p : c.q;
        const unsigned hi = unsigned(__double2hiint(x)), lo = unsigned(__double2loint(x));
        const unsigned ex = hi & 0x7FF00000u;
        const double r = __fma_rn(-x, den, num);
        const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
        const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
        bad |= !(fabs(r) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
      }
      if (bad) {  // rare: the block exactly
        ++nredo;
        x = xs;
        for (int t = 0; t < 8; ++t) {
          x = plcm_exact(x, c.p, c.q);
          y[t] = x;
        }
      }
      uint32_t mlo[4], mhi[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double sv = odd ? y[t] : y[t + 4];
        const double kv = odd ? y[t + 4] : y[t];
        const uint32_t rlo = __shfl_xor_sync(0xFFFFFFFFu, unsigned(__double2loint(sv)), 1);
        const uint32_t rhi = __shfl_xor_sync(0xFFFFFFFFu, unsigned(__double2hiint(sv)), 1);
        mlo[t] = unsigned(__double2loint(kv)) ^ rlo;
        mhi[t] = (unsigned(__double2hiint(kv)) ^ rhi) & 0xFFFFu;
      }
      const uint32_t w0 = mlo[0], w1 = mhi[0] | (mlo[1] << 16), w2 = (mlo[1] >> 16) | (mhi[1] << 16),
                     w3 = mlo[2], w4 = mhi[2] | (mlo[3] << 16), w5 = (mlo[3] >> 16) | (mhi[3] << 16);
      uint8_t* dst = rb + size_t(i) * 6;
      if (!odd) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(w0, w1, w2, w3);
        *reinterpret_cast<uint2*>(dst + 16) = make_uint2(w4, w5);
      } else {
        *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
        *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w2, w3, w4, w5);
      }
    }
    if (nredo) atomicAdd(redo, nredo);
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
  c.hp = 0.5 * c.p;
  c.hq = 0.5 * c.q;
  uint64_t bits;
  std::memcpy(&bits, &c.p, 8);
  c.plo = uint32_t(bits);
  return c;
}

int main() {
  const int T = 128;
  const uint32_t iters = 1u << 19;
  std::vector<LaneConst> h(T);
  std::vector<double> x0(T);
  for (int i = 0; i < T; ++i) {
    h[i] = make(0.01 + 0.48 * ((i * 37 % 101) / 101.0));
    x0[i] = (i * 53 % 97) / 97.0 + 0.001;
  }
  LaneConst* dl;
  double *dx, *dorb;
  uint8_t* dring;
  unsigned* dredo;
  cudaMalloc(&dl, T * sizeof(LaneConst));
  cudaMalloc(&dx, T * 8);
  cudaMalloc(&dorb, size_t(iters) * T * 8);
  cudaMalloc(&dring, size_t(iters) * 6 * (T / 2));
  cudaMalloc(&dredo, 4);
  cudaMemcpy(dl, h.data(), T * sizeof(LaneConst), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<double> end[2];
  const char* names[] = {"product: step + orbit STG", "inline verify + emit"};
  for (int m = 0; m < 2; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(dx, x0.data(), T * 8, cudaMemcpyHostToDevice);
      cudaMemset(dredo, 0, 4);
      cudaEventRecord(a);
      if (m == 0)
        k<0><<<1, T>>>(dx, dl, dorb, dring, iters, T, dredo);
      else
        k<1><<<1, T>>>(dx, dl, dorb, dring, iters, T, dredo);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned redo = 0;
      cudaMemcpy(&redo, dredo, 4, cudaMemcpyDeviceToHost);
      if (rep)
        printf("%-28s %.2f ns/iter  (redo blocks %u of %u)\n", names[m], ms * 1e6 / iters, redo,
               iters / 8 * T);
    }
    end[m].resize(T);
    cudaMemcpy(end[m].data(), dx, T * 8, cudaMemcpyDeviceToHost);
  }
  printf("final states identical: %s\n", end[0] == end[1] ? "yes" : "NO");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
