// Dependency-pair latencies on the PLCM chain (one warp, clock64).  Tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/latency_probe2.cu -o tools/latency_probe2
#include <cstdio>

#define N 1024
#define BODY_BEGIN                                  \
  double x = out[threadIdx.x];                      \
  long long t0 = clock64();                         \
  _Pragma("unroll 32") for (int i = 0; i < N; ++i) {
#define BODY_END                                    \
  }                                                 \
  long long t1 = clock64();                         \
  out[threadIdx.x] = x;                             \
  if (threadIdx.x == 0) cyc[0] = t1 - t0;

// DSETP -> FSEL (predicate operand on the chain)
__global__ void k_pred_sel(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("{.reg .pred p; setp.gt.f64 p, %0, %1; selp.f64 %0, %2, %1, p;}"
               : "+d"(x) : "d"(a), "d"(b));
  BODY_END
}
// DSETP -> DSETP.OR -> FSEL
__global__ void k_pred2_sel(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("{.reg .pred p, q; setp.gt.f64 p, %0, %1; setp.lt.or.f64 q, %0, %2, p;"
               " selp.f64 %0, %2, %1, q;}"
               : "+d"(x) : "d"(a), "d"(b));
  BODY_END
}
// DSETP, DSETP -> or.pred -> FSEL
__global__ void k_pred_or_sel(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("{.reg .pred p, q, r; setp.gt.f64 p, %0, %1; setp.lt.f64 q, %0, %2;"
               " or.pred r, p, q; selp.f64 %0, %2, %1, r;}"
               : "+d"(x) : "d"(a), "d"(b));
  BODY_END
}
// DADD -> FSEL (data operand), predicate loop-invariant
__global__ void k_add_sel(double* out, long long* cyc, double a, double b) {
  const bool pr = threadIdx.x & 1;
  BODY_BEGIN
  asm volatile("{.reg .pred p; .reg .f64 t; setp.ne.b32 p, %3, 0; add.rn.f64 t, %0, %1;"
               " selp.f64 %0, t, %2, p;}"
               : "+d"(x) : "d"(a), "d"(b), "r"(int(pr)));
  BODY_END
}
// DADD -> DADD
__global__ void k_add_add(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(a));
  BODY_END
}
// DSETP -> predicated FP64 add (keeps value otherwise)
__global__ void k_pred_padd(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("{.reg .pred p; setp.gt.f64 p, %0, %1; @p add.rn.f64 %0, %0, %2;}"
               : "+d"(x) : "d"(a), "d"(b));
  BODY_END
}
// DFMA -> DFMA
__global__ void k_fma(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(a), "d"(b));
  BODY_END
}
// integer compare on the hi word -> FSEL
__global__ void k_isetp_sel(double* out, long long* cyc, double a, double b) {
  BODY_BEGIN
  asm volatile("{.reg .pred p; .reg .b32 lo, hi; mov.b64 {lo, hi}, %0;"
               " setp.gt.s32 p, hi, 1071644672; selp.f64 %0, %2, %1, p;}"
               : "+d"(x) : "d"(a), "d"(b));
  BODY_END
}
// DADD -> FSEL -> FSEL (two selects in series, data path)
__global__ void k_add_sel_sel(double* out, long long* cyc, double a, double b) {
  const bool pr = threadIdx.x & 1, pr2 = threadIdx.x & 2;
  BODY_BEGIN
  asm volatile("{.reg .pred p, q; .reg .f64 t, u; setp.ne.b32 p, %3, 0; setp.ne.b32 q, %4, 0;"
               " add.rn.f64 t, %0, %1; selp.f64 u, t, %2, p; selp.f64 %0, u, %1, q;}"
               : "+d"(x) : "d"(a), "d"(b), "r"(int(pr)), "r"(int(pr2)));
  BODY_END
}

typedef void (*K)(double*, long long*, double, double);

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 32 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  cudaMemset(d, 0, 32 * sizeof(double));
  struct { const char* name; K k; } ks[] = {
      {"DADD->DADD", k_add_add},           {"DFMA->DFMA", k_fma},
      {"DSETP->FSEL", k_pred_sel},         {"DSETP->DSETP.OR->FSEL", k_pred2_sel},
      {"DSETPx2->PLOP->FSEL", k_pred_or_sel}, {"DADD->FSEL", k_add_sel},
      {"DADD->FSEL->FSEL", k_add_sel_sel}, {"DSETP->@P DADD", k_pred_padd},
      {"ISETP(hi)->FSEL", k_isetp_sel}};
  for (auto& e : ks) {
    long long best = 1LL << 60;
    for (int r = 0; r < 5; ++r) {
      e.k<<<1, 32>>>(d, c, 0.25, 0.75);
      long long h;
      cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
      if (h < best) best = h;
    }
    printf("%-26s %6.2f cycles per step\n", e.name, double(best) / N);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
