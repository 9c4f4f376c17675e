// Dependent-latency microbenchmark for the instructions on the PLCM chain
// (one warp, clock64 around a 1024-long dependency chain).  Tool, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/latency_probe.cu -o latency_probe
#include <cstdio>
#include <cstdint>

#define CHAIN 1024

__global__ void k_dadd(double* out, long long* cyc, double a) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dmul(double* out, long long* cyc, double a) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = __dmul_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(double* out, long long* cyc, double a) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = __fma_rn(x, a, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// DSETP -> FSEL pair: x = (x > a) ? x*?:... keep it a select chain
__global__ void k_dsetp_sel(double* out, long long* cyc, double a) {
  double x = out[threadIdx.x];
  const double b = a * 0.5;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = (x > a) ? b : x + 0.0 * i;  // compiler: DSETP+FSEL
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// DADD feeding DADD through a select on an independent predicate
__global__ void k_fsel(double* out, long long* cyc, double a) {
  double x = out[threadIdx.x];
  const bool p = threadIdx.x & 1;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) {
    double y = __dadd_rn(x, a);
    x = p ? y : x;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dmnmx(double* out, long long* cyc, double a) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = fmin(__dadd_rn(x, a), x);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_iadd(double* out, long long* cyc, double a) {
  unsigned x = __double2loint(out[threadIdx.x]);
  const unsigned b = __double2hiint(a);
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = (x ^ b) + 0x9E3779B9u;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_fadd(double* out, long long* cyc, double a) {
  float x = out[threadIdx.x];
  const float b = a;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < CHAIN; ++i) x = __fadd_rn(x, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

typedef void (*K)(double*, long long*, double);

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 32 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  cudaMemset(d, 0, 32 * sizeof(double));
  struct { const char* name; K k; int ops; } ks[] = {
      {"DADD", k_dadd, 1}, {"DMUL", k_dmul, 1}, {"DFMA", k_dfma, 1},
      {"DSETP+FSEL(+DADD)", k_dsetp_sel, 1}, {"DADD+FSEL", k_fsel, 1},
      {"DADD+DMNMX", k_dmnmx, 1}, {"LOP3+IADD", k_iadd, 1}, {"FADD", k_fadd, 1}};
  for (auto& e : ks) {
    long long best = 1LL << 60;
    for (int r = 0; r < 5; ++r) {
      e.k<<<1, 32>>>(d, c, 0.25);
      long long h;
      cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
      if (h < best) best = h;
    }
    printf("%-22s %.2f cycles per dependent step\n", e.name, double(best) / CHAIN);
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz, err %s\n", clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
