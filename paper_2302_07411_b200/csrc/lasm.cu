// LASM keystream generator for sm_100a.
//
// The reference's LASM lane (chaos.cpp:34-38, 93-107, 119-141) iterates
//   x' = sin(pi*mu*(y+3)*x*(1-x)),  y' = sin(pi*mu*(x'+3)*y*(1-y))
// with glibc's libm sin, and emits 12 bytes per iteration: lo48(x_a ^ x_b)
// then lo48(y_a ^ y_b), least significant byte first.  Each lane is a
// sequential chain with no jump-ahead, so -- as for PLCM -- the bound is the
// dependent latency of one iteration: two glibc sin evaluations in series.
//
// Unlike the PLCM chain there is no speculation and no verifier: gsin::sin
// (glibc_sin.cuh) performs glibc's own operation sequence, so every value is
// the reference's by construction (pinned by tests/test_lasm.py).  sin's
// branches depend on the argument, so lanes in one warp would diverge and
// serialise their paths; each lane therefore runs alone in its own CTA, as
// thread 0 (`if (threadIdx.x) return`): the compiler then knows the thread
// is alone in its warp and emits the branches without reconvergence
// barriers (BSSY/BSYNC), 600 -> 504 cycles per iteration on B200
// (tools/lasm_latency.cu).  The orbit values go to a lane-major buffer, and a
// second, fully parallel kernel XORs the two lanes of each worker into the
// keystream ring.
//
// Compiled with -fmad=false: every fused multiply-add is an explicit fma()
// mirroring glibc's, nothing else is contracted.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "glibc_sin.cuh"
#include "kernels.hpp"

namespace cveb {
namespace {

__device__ const double g_sintab[gsin::kTableDoubles] = {
#include "glibc_sincostab.inc"
};

constexpr double kPi = 0x1.921fb54442d18p1;  // std::numbers::pi
constexpr int kCtaThreads = 32;  // thread 0 runs the lane; the warp loads the table

// Copies the table into shared memory; returns its shared-window address.
__device__ __forceinline__ gsin::SmemTable load_table(double* tab) {
  for (int i = threadIdx.x; i < gsin::kTableDoubles; i += blockDim.x) tab[i] = g_sintab[i];
  __syncthreads();
  return gsin::SmemTable{uint32_t(__cvta_generic_to_shared(tab))};
}

// `iters` LASM iterations of one lane from (x, y); orbit values to out[i]
// when kStore.  chaos.cpp:34-38, evaluated left to right:
// ((((pi*mu)*(y+3))*x)*(1-x)).  sin_0pi is sin() with the branches LASM
// arguments take ordered for the chain.
template <bool kStore>
__device__ __forceinline__ void lasm_walk(double& x, double& y, double pm,
                                          const gsin::SmemTable& tab, uint32_t iters,
                                          double2* out) {
#pragma unroll 1
  for (uint32_t i = 0; i < iters; ++i) {
    x = gsin::sin_0pi(pm * (y + 3.0) * x * (1.0 - x), tab);
    y = gsin::sin_0pi(pm * (x + 3.0) * y * (1.0 - y), tab);
    if (kStore) out[i] = make_double2(x, y);
  }
}

// 256 warm-up iterations from the derived start points (chaos.cpp:93-107).
__global__ void __launch_bounds__(kCtaThreads)
    k_lasm_init(double2* state, const double* mu, const double2* xy0, uint32_t nlanes) {
  __shared__ double smem[gsin::kTableDoubles];
  const gsin::SmemTable tab = load_table(smem);
  const uint32_t lane = blockIdx.x;
  if (threadIdx.x || lane >= nlanes) return;
  double x = xy0[lane].x, y = xy0[lane].y;
  lasm_walk<false>(x, y, kPi * mu[lane], tab, 256, nullptr);
  state[lane] = make_double2(x, y);
}

// Chain: every lane advances `iters` iterations; orbit[lane*max_iters + i].
__global__ void __launch_bounds__(kCtaThreads)
    k_lasm_chain(double2* state, const double* mu, double2* orbit, uint32_t max_iters,
                 uint32_t iters, uint32_t nlanes) {
  __shared__ double smem[gsin::kTableDoubles];
  const gsin::SmemTable tab = load_table(smem);
  const uint32_t lane = blockIdx.x;
  if (threadIdx.x || lane >= nlanes) return;
  double x = state[lane].x, y = state[lane].y;
  lasm_walk<true>(x, y, kPi * mu[lane], tab, iters, orbit + uint64_t(lane) * max_iters);
  state[lane] = make_double2(x, y);
}

// Emission: thread = (worker, 4 iterations) -> 48 keystream bytes at stream
// byte 12*(it0 + 4g) of the worker's ring (48-aligned: it0 % 8 == 0 and
// ring_bytes % 48 == 0, so a group never wraps).
__global__ void k_lasm_emit(const double2* __restrict__ orbit, uint32_t max_iters,
                            uint8_t* __restrict__ ring, uint64_t ring_bytes, uint64_t it0,
                            uint32_t iters, uint32_t nworkers) {
  const uint32_t groups = iters / 4;
  const uint64_t total = uint64_t(groups) * nworkers;
  for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t w = uint32_t(idx / groups), g = uint32_t(idx % groups);
    const double2* A = orbit + uint64_t(2 * w) * max_iters + 4ull * g;
    const double2* B = orbit + uint64_t(2 * w + 1) * max_iters + 4ull * g;
    uint64_t word[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // piece j: bits [48j, 48j+48)
      const double2 a = A[j / 2], b = B[j / 2];
      const uint64_t v =
          (j & 1) ? (uint64_t(__double_as_longlong(a.y)) ^ uint64_t(__double_as_longlong(b.y)))
                  : (uint64_t(__double_as_longlong(a.x)) ^ uint64_t(__double_as_longlong(b.x)));
      const uint64_t p = v & 0xFFFFFFFFFFFFull;
      const int bit = 48 * j, wi = bit / 64, sh = bit % 64;
      word[wi] |= p << sh;
      if (sh > 16) word[wi + 1] |= p >> (64 - sh);
    }
    uint8_t* dst = ring + uint64_t(w) * ring_bytes + (12 * (it0 + 4ull * g)) % ring_bytes;
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 3; ++q)
      d[q] = make_uint4(uint32_t(word[2 * q]), uint32_t(word[2 * q] >> 32),
                        uint32_t(word[2 * q + 1]), uint32_t(word[2 * q + 1] >> 32));
  }
}

__global__ void k_glibc_sin(const double* __restrict__ x, double* __restrict__ y, size_t n) {
  __shared__ double smem[gsin::kTableDoubles];
  const gsin::SmemTable tab = load_table(smem);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    y[i] = gsin::sin(x[i], tab);
}


}  // namespace

void launch_lasm_init(double2* state, const double* mu, const double2* xy0, uint32_t nlanes,
                      cudaStream_t s) {
  k_lasm_init<<<nlanes, kCtaThreads, 0, s>>>(state, mu, xy0, nlanes);
}

void launch_lasm_chain(const LasmBuffers& b, int slot, uint32_t iters, uint32_t nlanes,
                       cudaStream_t s) {
  k_lasm_chain<<<nlanes, kCtaThreads, 0, s>>>(
      b.state, b.mu, b.orbit[slot], b.max_iters, iters, nlanes);
}

void launch_lasm_emit(const LasmBuffers& b, int slot, uint8_t* ring, uint64_t ring_bytes,
                      uint64_t it0, uint32_t iters, uint32_t nlanes, cudaStream_t s) {
  const uint64_t total = uint64_t(iters / 4) * (nlanes / 2);
  const uint32_t blocks = uint32_t(std::min<uint64_t>((total + 255) / 256, 148 * 8));
  k_lasm_emit<<<blocks ? blocks : 1, 256, 0, s>>>(b.orbit[slot], b.max_iters, ring, ring_bytes,
                                                  it0, iters, nlanes / 2);
}

void launch_glibc_sin(const double* x, double* y, size_t n, cudaStream_t s) {
  const uint32_t blocks = uint32_t(std::min<size_t>((n + 255) / 256, 148 * 8));
  k_glibc_sin<<<blocks ? blocks : 1, 256, 0, s>>>(x, y, n);
}

}  // namespace cveb
