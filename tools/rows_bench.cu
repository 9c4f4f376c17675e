// One cipher round, kernels alone: K2r/K3r (rows.cu) against K2s/K3t
// (cipher.cu) and a CPU restatement of the reference round
// (engine.cpp:32-83, 207-284).  Random frame, keystream ring, shift table.
// Tool (not the product):
//   make -C paper_2302_07411_b200/csrc && nvcc ... tools/rows_bench.cu build/csrc/{cipher,rows,keying}.o
//   tools/rows_bench SIDE N [REPS]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "kernels.hpp"

using namespace cveb;
#ifdef ROWS_PROF
namespace cveb {
void rows_prof_read(unsigned long long* host, size_t n);
}
#endif

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(2);                                                                \
    }                                                                              \
  } while (0)

static uint32_t euclid(int64_t v, uint32_t m) {
  int64_t r = v % int64_t(m);
  return uint32_t(r < 0 ? r + m : r);
}

__global__ void k_empty(int x) {
  extern __shared__ uint8_t sm[];
  if (x == 12345) sm[threadIdx.x] = 1;
}

static void empty_launch(dim3 grid, uint32_t threads, size_t smem, uint32_t cl, bool pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (cl > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cl;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k_empty, 0);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const uint32_t side = argc > 1 ? atoi(argv[1]) : 1920;
  const uint32_t n = argc > 2 ? atoi(argv[2]) : 64;
  const int reps = argc > 3 ? atoi(argv[3]) : 50;
  const uint32_t rows = side / n;
  const uint64_t region = uint64_t(rows) * side * 3, F = uint64_t(side) * side * 3;
  const uint64_t ring_bytes = ((4 * 5 * region + 47) / 48) * 48 + 48 * 7;
  std::mt19937_64 rng(12345 + side);
  std::vector<uint8_t> X(F), ring(n * ring_bytes);
  for (auto& v : X) v = uint8_t(rng());
  for (auto& v : ring) v = uint8_t(rng());
  const uint32_t seed = uint32_t(rng());
  std::vector<double> sine(side);
  for (uint32_t a = 0; a < side; ++a) sine[a] = std::sin(2.0 * M_PI * double(a) / double(side));
  std::vector<int32_t> shift(side);
  for (uint32_t a = 0; a < side; ++a) {
    volatile double v = double(seed) * sine[a];
    shift[a] = int32_t(euclid(int64_t(std::floor(v)), side));
  }
  // a window that wraps the ring inside the frame
  const uint64_t pos = ((ring_bytes - region / 2) / 48) * 48;
  auto ks = [&](uint32_t band, uint64_t j) { return ring[band * ring_bytes + (pos + j) % ring_bytes]; };

  // CPU forward round: confuse_rows + diffuse_region (s_d of the next band)
  std::vector<uint8_t> Y(F), C(F), P(F), D(F);
  for (uint32_t a = 0; a < side; ++a)
    for (uint32_t o = 0; o < side; ++o) {
      const uint32_t al = (a + o) % side, be = euclid(int64_t(o) + shift[al], side);
      std::memcpy(&Y[(uint64_t(al) * side + be) * 3], &X[(uint64_t(a) * side + o) * 3], 3);
    }
  for (uint32_t i = 0; i < n; ++i) {
    uint8_t prev = Y[((i + 1) % n + 1) * region - 1];
    for (uint64_t j = 0; j < region; ++j) {
      const uint8_t b = ks(i, j);
      prev = uint8_t(b ^ ((Y[i * region + j] + b) & 0xFF) ^ prev);
      C[i * region + j] = prev;
    }
  }
  // CPU inverse round of X (as a cipher frame): inverse diffusion + heads,
  // then inverse confusion
  std::vector<uint8_t> T(F);
  for (uint32_t i = 0; i < n; ++i)
    for (uint64_t j = 1; j < region; ++j) {
      const uint8_t b = ks(i, j);
      T[i * region + j] = uint8_t(((b ^ X[i * region + j] ^ X[i * region + j - 1]) - b) & 0xFF);
    }
  for (uint32_t i = 0; i < n; ++i) {
    const uint8_t sd = T[((i + 1) % n + 1) * region - 1];
    const uint8_t b = ks(i, 0);
    T[i * region] = uint8_t(((b ^ X[i * region] ^ sd) - b) & 0xFF);
  }
  for (uint32_t al = 0; al < side; ++al)
    for (uint32_t be = 0; be < side; ++be) {
      const uint32_t o = euclid(int64_t(be) - shift[al], side);
      const uint32_t a = euclid(int64_t(al) - int64_t(o), side);
      std::memcpy(&P[(uint64_t(a) * side + o) * 3], &T[(uint64_t(al) * side + be) * 3], 3);
    }

  uint8_t *dX, *dO, *dR, *dS;
  double* dSine;
  int32_t* dShift;
  CK(cudaMalloc(&dX, F));
  CK(cudaMalloc(&dO, F));
  CK(cudaMalloc(&dS, 2 * F + 4096));
  CK(cudaMalloc(&dR, n * ring_bytes));
  CK(cudaMalloc(&dSine, side * 8));
  CK(cudaMalloc(&dShift, side * 4));
  CK(cudaMemcpy(dX, X.data(), F, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dR, ring.data(), n * ring_bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dSine, sine.data(), side * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dShift, shift.data(), side * 4, cudaMemcpyHostToDevice));
  configure_cipher_kernels();
  configure_rows_kernels();
  Geom g{side, n, rows, region, F};
  KsWindow w{dR, ring_bytes, pos};
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  uint64_t launches = 0;
  std::vector<uint8_t> out(F);
  auto check = [&](const char* what, const std::vector<uint8_t>& want) {
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(out.data(), dO, F, cudaMemcpyDeviceToHost));
    uint64_t bad = 0, first = ~0ull;
    for (uint64_t i = 0; i < F; ++i)
      if (out[i] != want[i]) {
        if (!bad) first = i;
        ++bad;
      }
    std::printf("%-22s %s", what, bad ? "MISMATCH" : "ok");
    if (bad) std::printf(" (%llu bytes, first at %llu: row %llu col %llu ch %llu)", (unsigned long long)bad,
                         (unsigned long long)first, (unsigned long long)(first / (3ull * side)),
                         (unsigned long long)(first % (3ull * side) / 3), (unsigned long long)(first % 3));
    return bad == 0;
  };
  auto timeit = [&](const char* what, auto&& fn) {
    for (int i = 0; i < 3; ++i) fn();
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) fn();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / reps;
    std::printf("   %7.2f us/round  %6.0f GB/s (3F)\n", us, 3.0 * F / us / 1e3);
    (void)what;
  };
  std::printf("side %u n %u rows %u region %llu\n", side, n, rows, (unsigned long long)region);
  if (getenv("EMPTY_PROBE")) {
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (uint32_t cl : {1u, 2u}) for (size_t sm : {size_t(0), size_t(90000)}) for (int pdl = 0; pdl < 2; ++pdl) {
      std::printf("empty grid 128 x 512 thr, cluster %u smem %zu pdl %d:", cl, sm, pdl);
      timeit("empty", [&] { empty_launch(dim3(128), 512, sm, cl, pdl, s); });
    }
  }

  RowPlan rp;
  if (plan_rows_encrypt(g, rp)) {
    std::printf("K2r plan: cr %u h %u bpw %u nb %u L %u smem %zu\n", rp.cr, rp.h, rp.bpw, rp.nb,
                rp.L, rp.smem);
    CK(cudaMemset(dO, 0, F));
    launch_encrypt_round_rows(rp, g, dX, dO, w, dSine, seed, s);
    CK(cudaGetLastError());
    check("K2r encrypt", C);
    timeit("K2r", [&] { launch_encrypt_round_rows(rp, g, dX, dO, w, dSine, seed, s); });
#ifdef ROWS_PROF
    {
      CK(cudaDeviceSynchronize());
      launch_encrypt_round_rows(rp, g, dX, dO, w, dSine, seed, s);
      CK(cudaDeviceSynchronize());
      const size_t nc = g.n * rp.h;
      std::vector<unsigned long long> pr(nc * 8);
      rows_prof_read(pr.data(), nc);
      unsigned long long t0 = ~0ull, tend = 0;
      double avg[8] = {0};
      for (size_t c = 0; c < nc; ++c) {
        t0 = std::min(t0, pr[c * 8]);
        tend = std::max(tend, pr[c * 8 + 6]);
        for (int i = 1; i < 7; ++i) avg[i] += double(pr[c * 8 + i] - pr[c * 8 + i - 1]) / nc;
      }
      unsigned long long lastStart = 0;
      for (size_t c = 0; c < nc; ++c) lastStart = std::max(lastStart, pr[c * 8]);
      std::printf("   phases (us, mean over CTAs): prologue %.2f  lanes %.2f  bar %.2f  rowscan %.2f  cluster %.2f  copyout %.2f | first start->last end %.2f, last start %.2f\n",
                  avg[1] / 1e3, avg[2] / 1e3, avg[3] / 1e3, avg[4] / 1e3, avg[5] / 1e3, avg[6] / 1e3,
                  (tend - t0) / 1e3, (lastStart - t0) / 1e3);
    }
#endif
  } else {
    std::printf("K2r: no plan\n");
  }
  {
    const EncPlan ep = plan_encrypt(g);
    CK(cudaMemset(dO, 0, F));
    launch_encrypt_round(ep, g, dX, dO, w, dShift, dS, s, &launches);
    check("K2s encrypt (r02)", C);
    timeit("K2s", [&] { launch_encrypt_round(ep, g, dX, dO, w, dShift, dS, s, &launches); });
  }
  if (plan_rows_decrypt(g, rp)) {
    std::printf("K3r plan: cr %u bpw %u nb %u L %u smem %zu\n", rp.cr, rp.bpw, rp.nb, rp.L, rp.smem);
    CK(cudaMemset(dO, 0, F));
    launch_decrypt_round_rows(rp, g, dX, dO, w, dShift, s);
    CK(cudaGetLastError());
    check("K3r decrypt", P);
    timeit("K3r", [&] { launch_decrypt_round_rows(rp, g, dX, dO, w, dShift, s); });
  }
  {
    CK(cudaMemset(dO, 0, F));
    launch_decrypt_round(g, dX, dO, w, dShift, s, &launches);
    check("K3t decrypt (r02)", P);
    timeit("K3t", [&] { launch_decrypt_round(g, dX, dO, w, dShift, s, &launches); });
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
