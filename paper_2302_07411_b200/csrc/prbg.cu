// K1: per-subframe PLCM keystream generator for sm_100a.
//
// Replaces the reference's Prbg::fill -> refill -> step_lane -> plcm_step /
// plcm_guard / extract_bytes hot loop (chaos.cpp:18-56, 109-153), called per
// worker from Engine::Impl::draw_streams (engine.cpp:198-205).
//
// The keystream of a clip is 2n sequential chaotic orbits (n subframes x 2
// lanes) that continue across frames, so the kernel is bound by the latency
// of ONE dependent PLCM iteration, not by bandwidth or FP64 throughput.
// Everything here serves that chain:
//   * one orbit per thread; the two lanes of a worker sit in adjacent
//     threads and meet through one shuffle per iteration (keeps a warp's
//     issue demand below the chain latency);
//   * branch-free iteration (selects), division by the loop-invariant
//     divisor done as RN(1/d) multiply + two FMA corrections (Markstein);
//   * the exactness of that quotient and the reference's endpoint guard are
//     both verified OFF the dependency chain: a cheap pre-filter flags any
//     iteration whose result might be wrong or might hit the guard set
//     {0, p, 0.5, 1}; a flagged 8-iteration block is replayed with IEEE
//     __ddiv_rn and the exact guard.  Output is therefore bit-identical to
//     the reference's IEEE binary64 loop by construction, not by statistics.
//
// Compiled with -fmad=false; every FP64 operation below is an explicit _rn
// intrinsic anyway, so no contraction can change a result.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "kernels.hpp"

namespace cveb {

LaneConst make_lane_const(double p) {
  LaneConst c{};
  volatile double half = 0.5, one = 1.0;  // keep host evaluation IEEE
  c.p = p;
  c.q = half - p;
  c.rp = one / c.p;
  c.rq = one / c.q;
  c.hp = 0.5 * c.p;
  c.hq = 0.5 * c.q;
  uint64_t bits;
  std::memcpy(&bits, &c.p, 8);
  c.plo = uint32_t(bits);
  return c;
}

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Reference step + guard in plain IEEE arithmetic (chaos.cpp:18-32).
__device__ __forceinline__ double plcm_exact(double x, double p, double q) {
  const double f = x > 0.5 ? __dsub_rn(1.0, x) : x;
  double y = f < p ? __ddiv_rn(f, p) : __ddiv_rn(__dsub_rn(f, p), q);
  if (y == 0.0 || y == p || y == 0.5 || y == 1.0) {
    y = __dadd_rn(y, 0x1p-52);
    if (y > 1.0) y = __dsub_rn(y, 1.0);
  }
  return y;
}

// Speculative step: branch-free, division via reciprocal + FMA correction.
// `flag` accumulates "this result may differ from plcm_exact".
__device__ __forceinline__ double plcm_fast(double x, const LaneConst& c,
                                            bool& flag) {
  const double folded = __dsub_rn(1.0, x);
  const double f = x > 0.5 ? folded : x;
  const bool low = f < c.p;
  const double shifted = __dsub_rn(f, c.p);
  const double num = low ? f : shifted;
  const double rcp = low ? c.rp : c.rq;
  const double den = low ? c.p : c.q;
  const double q0 = __dmul_rn(num, rcp);
  const double r0 = __fma_rn(-q0, den, num);
  const double y = __fma_rn(r0, rcp, q0);

  // --- off the chain: is y == RN(num/den), and is y outside the guard set?
  // y = RN(num/den)  <=>  |num - den*y| < den*ulp(y)/2  when y is not a power
  // of two (no quotient is a midpoint).  Powers of two, 0, 0.5, 1 and p all
  // have low word 0 or equal to p's low word, so the pre-filter sends them
  // to the exact replay.
  const double r1 = __fma_rn(-y, den, num);
  const unsigned hi = unsigned(__double2hiint(y));
  const unsigned lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  flag |= !(fabs(r1) < thr) | (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return y;
}

__global__ void __launch_bounds__(128)
    k_prbg_init(double* __restrict__ state, const LaneConst* __restrict__ lc,
                const double* __restrict__ x0, uint32_t nlanes) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlanes) return;
  const double p = lc[l].p, q = lc[l].q;
  double x = x0[l];
  if (x == 0.0 || x == p || x == 0.5 || x == 1.0) {  // plcm_guard on the seed
    x = __dadd_rn(x, 0x1p-52);
    if (x > 1.0) x = __dsub_rn(x, 1.0);
  }
  for (int i = 0; i < 256; ++i) x = plcm_exact(x, p, q);
  state[l] = x;
}

// One thread per lane; lanes 2w and 2w+1 (worker w's lanes a and b) are
// shuffle partners.  Per 8-iteration block the pair emits 48 keystream bytes:
// the even thread stores bytes 0..23 (iterations 0-3), the odd one 24..47.
__global__ void __launch_bounds__(128)
    k_prbg_generate(double* __restrict__ state,
                    const LaneConst* __restrict__ lc, uint8_t* __restrict__ ring,
                    uint64_t ring_bytes, uint64_t it0, uint32_t nblk,
                    uint32_t nlanes, unsigned long long* __restrict__ replays) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = l < nlanes;
  const uint32_t me = live ? l : (l & 1u);  // idle threads shadow lane 0/1
  const LaneConst c = lc[me];
  const uint32_t odd = me & 1u;
  uint8_t* const base = ring + uint64_t(me >> 1) * ring_bytes + (odd ? 24 : 0);
  uint64_t off = (it0 * 6u) % ring_bytes;
  double x = state[me];
  uint32_t nreplay = 0;

  for (uint32_t b = 0; b < nblk; ++b) {
    uint32_t lo[8], hi[8];
    const double x_start = x;
    bool flag = false;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      x = plcm_fast(x, c, flag);
      lo[t] = unsigned(__double2loint(x));
      hi[t] = unsigned(__double2hiint(x));
    }
    if (flag) {  // rare: replay the block with IEEE division + exact guard
      ++nreplay;
      x = x_start;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        x = plcm_exact(x, c.p, c.q);
        lo[t] = unsigned(__double2loint(x));
        hi[t] = unsigned(__double2hiint(x));
      }
    }
    // Even thread needs the partner's iterations 0-3, odd one 4-7.
    uint32_t w[6];
    uint32_t mlo[4], mhi[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t slo = odd ? lo[t] : lo[t + 4];
      const uint32_t shi = odd ? hi[t] : hi[t + 4];
      const uint32_t rlo = __shfl_xor_sync(kFull, slo, 1);
      const uint32_t rhi = __shfl_xor_sync(kFull, shi, 1);
      mlo[t] = (odd ? lo[t + 4] : lo[t]) ^ rlo;
      mhi[t] = ((odd ? hi[t + 4] : hi[t]) ^ rhi) & 0xFFFFu;
    }
    // 4 iterations x 6 bytes, little-endian mantissa bytes (extract_bytes).
    w[0] = mlo[0];
    w[1] = mhi[0] | (mlo[1] << 16);
    w[2] = (mlo[1] >> 16) | (mhi[1] << 16);
    w[3] = mlo[2];
    w[4] = mhi[2] | (mlo[3] << 16);
    w[5] = (mlo[3] >> 16) | (mhi[3] << 16);
    if (live) {
      uint8_t* dst = base + off;
      if (!odd) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint2*>(dst + 16) = make_uint2(w[4], w[5]);
      } else {
        *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
        *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w[2], w[3], w[4], w[5]);
      }
    }
    off += 48;
    if (off == ring_bytes) off = 0;
  }
  if (live) {
    state[l] = x;
    if (nreplay) atomicAdd(replays, (unsigned long long)nreplay);
  }
}

}  // namespace

void launch_prbg_init(double* state, const LaneConst* lc, const double* x0,
                      uint32_t nlanes, cudaStream_t s) {
  const uint32_t threads = 128;
  k_prbg_init<<<(nlanes + threads - 1) / threads, threads, 0, s>>>(state, lc,
                                                                    x0, nlanes);
}

void launch_prbg_generate(double* state, const LaneConst* lc, uint8_t* ring,
                          uint64_t ring_bytes, uint64_t it0, uint32_t nblk,
                          uint32_t nlanes, unsigned long long* replays,
                          uint32_t reserve_smem, cudaStream_t s) {
  // At most 4 warps per CTA: one warp per SM sub-partition, so each warp
  // owns its scheduler.  `reserve_smem` (optional) keeps smem-hungry cipher
  // CTAs off the generator's SMs.
  const uint32_t warps = (nlanes + 31) / 32;
  const uint32_t per_cta = warps < 4 ? warps : 4;
  const uint32_t ctas = (warps + per_cta - 1) / per_cta;
  static bool attr_done = false;
  if (reserve_smem && !attr_done) {
    cudaFuncSetAttribute(k_prbg_generate,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_done = true;
  }
  k_prbg_generate<<<ctas, per_cta * 32, reserve_smem, s>>>(
      state, lc, ring, ring_bytes, it0, nblk, nlanes, replays);
}

}  // namespace cveb
