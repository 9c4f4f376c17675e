// FP64 issue rate of one warp (not product code): cycles per DFMA when a
// warp has 1, 2, 4, 8 independent dependency chains, with 1 or 32 active
// lanes.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
//   tools/fp64_issue_probe.cu -o tools/fp64_issue_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(double* out, long long* cyc, int iters, int lanes) {
  if (threadIdx.x >= lanes) return;
  double v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) v[c] = 0.1 * (c + 1) + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int c = 0; c < C; ++c) v[c] = fma(v[c], 0.999, 1e-3);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += v[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
void run(int lanes) {
  double* o; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
  const int iters = 4000;
  k<C><<<1, 32>>>(o, c, 100, lanes);
  k<C><<<1, 32>>>(o, c, iters, lanes);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%d chains, %2d lanes: %.2f cycles per DFMA\n", C, lanes, double(h) / (iters * 8.0 * C));
  cudaFree(o); cudaFree(c);
}

int main() {
  for (int lanes : {1, 32}) { run<1>(lanes); run<2>(lanes); run<4>(lanes); run<8>(lanes); }
  return 0;
}
