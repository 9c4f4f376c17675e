// Latency probe for the LASM chain (not product code): cycles per dependent
// iteration of several variants, one thread, clock64 around the loop.
// Measured on B200 (r01): arg only 67, LASM step 504, 16 x DFMA 140,
// 16 x DADD 133, 2 x Taylor 150, 2 x sin_tab 260 cycles per iteration.  A
// branch-free arrangement of the Taylor/sin-table/cos-table branches
// (selects instead of branches) also measured 504: the step is bound by its
// ~25 dependent FP64 operations per half step, not by branching.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
//        -I paper_2302_07411_b200/csrc -I build/csrc tools/lasm_latency.cu -o tools/lasm_latency
#include <cstdio>
#include <cuda_runtime.h>
#include "glibc_sin.cuh"

__device__ const double g_tab[gsin::kTableDoubles] = {
#include "glibc_sincostab.inc"
};

template <int V>
__global__ void k(double* out, long long* cyc, int iters, double x0, double y0, double mu) {
  __shared__ double smem[gsin::kTableDoubles];
  for (int i = threadIdx.x; i < gsin::kTableDoubles; i += blockDim.x) smem[i] = g_tab[i];
  __syncthreads();
  const gsin::SmemTable tab{uint32_t(__cvta_generic_to_shared(smem))};
  if (threadIdx.x) return;
  double x = x0, y = y0;
  const double pm = 0x1.921fb54442d18p1 * mu;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    if (V == 0) {         // arg only (4 dependent ops per half)
      x = pm * (y + 3.0) * x * (1.0 - x);
      y = pm * (x + 3.0) * y * (1.0 - y);
    } else if (V == 1) {  // general glibc sin
      x = gsin::sin(pm * (y + 3.0) * x * (1.0 - x), tab);
      y = gsin::sin(pm * (x + 3.0) * y * (1.0 - y), tab);
    } else if (V == 2) {  // the chain's arrangement
      x = gsin::sin_0pi(pm * (y + 3.0) * x * (1.0 - x), tab);
      y = gsin::sin_0pi(pm * (x + 3.0) * y * (1.0 - y), tab);
    } else if (V == 3) {  // 16 dependent DFMA
#pragma unroll
      for (int j = 0; j < 16; ++j) x = fma(x, y, 1e-3);
    } else if (V == 4) {  // 16 dependent DADD
#pragma unroll
      for (int j = 0; j < 16; ++j) x = x + y;
    } else if (V == 5) {  // taylor only
      x = gsin::taylor(x * 1e-3, 0.0);
      y = gsin::taylor(y * 1e-3 + x, 0.0);
    } else if (V == 7) {  // arg + glibc's cos(pi/2 - x) branch body, forced (no range tests)
      // keeps the argument in the C range: pm' = 1.3/0.25 scale keeps a in ~[0.9, 1.6]
      x = gsin::cos_tab(gsin::kHp0 - (0.9 + pm * (y + 3.0) * x * (1.0 - x)), gsin::kHp1, tab);
      y = gsin::cos_tab(gsin::kHp0 - (0.9 + pm * (x + 3.0) * y * (1.0 - y)), gsin::kHp1, tab);
    } else if (V == 8) {  // the same through sin_0pi (range tests + branch)
      x = gsin::sin_0pi(0.9 + pm * (y + 3.0) * x * (1.0 - x), tab);
      y = gsin::sin_0pi(0.9 + pm * (x + 3.0) * y * (1.0 - y), tab);
    } else if (V == 9) {  // 17 dependent FP64 ops per half: the C path's op count
#pragma unroll
      for (int j = 0; j < 17; ++j) x = fma(x, 0.999, y * 0.0);
#pragma unroll
      for (int j = 0; j < 17; ++j) y = fma(y, 0.999, x * 0.0);
    } else if (V == 6) {  // sin_tab only
      x = gsin::sin_tab(0.2 + x * 1e-3, 0.0, tab);
      y = gsin::sin_tab(0.2 + y * 1e-3 + x * 1e-3, 0.0, tab);
    }
  }
  long long t1 = clock64();
  out[0] = x + y;
  cyc[0] = t1 - t0;
}

template <int V>
void run(const char* name, double x0, double y0, double mu) {
  double* d; long long* c;
  cudaMalloc(&d, 8); cudaMalloc(&c, 8);
  const int iters = 20000;
  k<V><<<1, 128>>>(d, c, 100, x0, y0, mu);
  k<V><<<1, 128>>>(d, c, iters, x0, y0, mu);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %8.1f cycles/iter\n", name, double(h) / iters);
  cudaFree(d); cudaFree(c);
}

// The product's configuration: one active lane per warp, `warps` warps per
// CTA, optionally storing each (x, y) like k_lasm_chain.
__global__ void k_multi(double2* orbit, long long* cyc, int iters, int warps, int store) {
  __shared__ double smem[gsin::kTableDoubles];
  for (int i = threadIdx.x; i < gsin::kTableDoubles; i += blockDim.x) smem[i] = g_tab[i];
  __syncthreads();
  const gsin::SmemTable tab{uint32_t(__cvta_generic_to_shared(smem))};
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) || w >= warps) return;
  double x = 0.3 + 0.01 * w, y = 0.7, pm = 0x1.921fb54442d18p1 * 0.9;
  double2* out = orbit + (size_t)w * iters;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    x = gsin::sin(pm * (y + 3.0) * x * (1.0 - x), tab);
    y = gsin::sin(pm * (x + 3.0) * y * (1.0 - y), tab);
    if (store) out[i] = make_double2(x, y);
  }
  long long t1 = clock64();
  if (w == 0) cyc[0] = t1 - t0;
}

void run_multi(int warps, int store) {
  double2* o; long long* c;
  const int iters = 20000;
  cudaMalloc(&o, sizeof(double2) * iters * 8); cudaMalloc(&c, 8);
  k_multi<<<1, 256>>>(o, c, 100, warps, store);
  k_multi<<<1, 256>>>(o, c, iters, warps, store);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("lasm step, %d warps/CTA, store %d %8.1f cycles/iter\n", warps, store, double(h) / iters);
  cudaFree(o); cudaFree(c);
}

int main() {
  for (int w : {1, 2, 4, 8})
    for (int st : {0, 1}) run_multi(w, st);
  run<0>("arg only (2 halves)", 0.3, 0.7, 0.9);
  run<1>("lasm step, gsin::sin", 0.3, 0.7, 0.9);
  run<2>("lasm step, sin_0pi", 0.3, 0.7, 0.9);
  run<3>("16 x DFMA", 0.3, 0.999, 0.9);
  run<4>("16 x DADD", 0.3, 1e-9, 0.9);
  run<5>("2 x taylor", 0.3, 0.7, 0.9);
  run<7>("2 x (arg + cos branch body)", 0.3, 0.7, 0.05);
  run<8>("2 x (arg + sin_0pi, C path)", 0.3, 0.7, 0.05);
  run<9>("2 x 17 dependent DFMA", 0.3, 0.7, 0.9);
  run<6>("2 x sin_tab", 0.3, 0.7, 0.9);
  return 0;
}
