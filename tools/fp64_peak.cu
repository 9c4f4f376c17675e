// Dense FP64 FMA throughput of this B200 (the FP64 side of the
// BASELINE roofline must be measured).  Tool, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/fp64_peak
#include <cstdio>

constexpr int kChains = 16;  // independent FMA chains per thread (hide latency)

__global__ void __launch_bounds__(256) k(double* out, int iters, double a, double b) {
  double v[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) v[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) v[i] = __fma_rn(v[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += v[i];
  if (s == 42.0) out[threadIdx.x] = s;  // keep the work alive
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks_per_sm : {2, 4, 8}) {
    const int grid = sms * blocks_per_sm;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double flops = 2.0 * kChains * iters * double(grid) * 256;
      if (rep) printf("%d blocks/SM: %.2f TFLOP/s FP64 (FMA = 2 flops)\n", blocks_per_sm,
                      flops / (ms * 1e-3) / 1e12);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
