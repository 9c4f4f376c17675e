// Row f4: the O(side^2) reductions of the reference's
// statistical analysis on sm_100a -- per-channel byte histograms
// (analysis.cpp:51-60 channel_histogram) and NPCR/UACI counts
// (analysis.cpp:200-218 npcr_uaci).  Everything downstream of these integer
// counts (variance, chi^2, entropy, the percentages) is evaluated on the
// host in the reference's order, so the printed statistics are identical.
//
// One kernel walks the frame(s) in 48-byte granules (16 pixels): the channel
// of byte j of a granule is j mod 3, a compile-time constant per register
// byte.  Counts are exact integers, so the reduction order is free.
#include <cuda_runtime.h>

#include <cstdint>

#include "analysis.hpp"
#include "keying.hpp"

namespace cveb {
namespace {

constexpr int kStatThreads = 512;
constexpr int kSubHists = 8;  // shared-memory copies (2 warps each): less contention

__device__ __forceinline__ void hist_word(uint32_t* h, uint32_t w, int byte0) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int ch = (byte0 + j) % 3;
    atomicAdd(h + ch * 256 + ((w >> (8 * j)) & 0xFFu), 1u);
  }
}

// One pass over frame a (and b when diff != nullptr): hist[c*256 + v] of a;
// diff[c] = positions where channel c differs, diff[3 + c] = sum |a - b|.
__global__ void __launch_bounds__(kStatThreads)
    k_frame_stats(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, uint64_t nbytes,
                  bool vec, unsigned long long* __restrict__ hist,
                  unsigned long long* __restrict__ diff) {
  __shared__ uint32_t h[kSubHists][768];
  if (hist) {
    for (int i = threadIdx.x; i < kSubHists * 768; i += kStatThreads) (&h[0][0])[i] = 0;
    __syncthreads();
  }
  uint32_t* mine = h[(threadIdx.x >> 6) % kSubHists];
  // scalar accumulators (a dynamically indexed array would live in local memory)
  unsigned long long c0 = 0, c1 = 0, c2 = 0, s0 = 0, s1 = 0, s2 = 0;
  const uint64_t stride = uint64_t(gridDim.x) * kStatThreads;
  const uint64_t t0 = uint64_t(blockIdx.x) * kStatThreads + threadIdx.x;
  uint64_t done = 0;
  if (vec) {
    const uint64_t G = nbytes / 48;
    const uint4* pa = reinterpret_cast<const uint4*>(a);
    const uint4* pb = reinterpret_cast<const uint4*>(b);
#pragma unroll 2
    for (uint64_t g = t0; g < G; g += stride) {
      uint32_t wa[12], wb[12];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const uint4 x = __ldg(pa + 3 * g + i);
        wa[4 * i] = x.x; wa[4 * i + 1] = x.y; wa[4 * i + 2] = x.z; wa[4 * i + 3] = x.w;
        if (diff) {
          const uint4 y = __ldg(pb + 3 * g + i);
          wb[4 * i] = y.x; wb[4 * i + 1] = y.y; wb[4 * i + 2] = y.z; wb[4 * i + 3] = y.w;
        }
      }
      if (hist) {
#pragma unroll
        for (int k = 0; k < 12; ++k) hist_word(mine, wa[k], 4 * k);
      }
      if (diff) {
        uint32_t c32[3] = {0, 0, 0}, s32[3] = {0, 0, 0};
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          const uint32_t d = __vabsdiffu4(wa[k], wb[k]);  // native VABSDIFF4
          const uint32_t x = wa[k] ^ wb[k];                // 0x01 per nonzero byte of x
          const uint32_t ne = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) >> 7 & 0x01010101u;
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            uint32_t m = 0;  // bytes of word k in channel ch
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if ((4 * k + j) % 3 == ch) m |= 0xFFu << (8 * j);
            s32[ch] = __dp4a(d & m, 0x01010101u, s32[ch]);
            c32[ch] = __dp4a(ne & m, 0x01010101u, c32[ch]);
          }
        }
        c0 += c32[0];
        c1 += c32[1];
        c2 += c32[2];
        s0 += s32[0];
        s1 += s32[1];
        s2 += s32[2];
      }
    }
    done = G * 48;
  }
  for (uint64_t i = done + t0; i < nbytes; i += stride) {  // tail / unaligned frames
    if (hist) atomicAdd(mine + (i % 3) * 256 + a[i], 1u);
    if (diff) {
      const int d = int(a[i]) - int(b[i]);
      const uint32_t ch = uint32_t(i % 3), ad = uint32_t(d < 0 ? -d : d);
      c0 += ch == 0 && d; c1 += ch == 1 && d; c2 += ch == 2 && d;
      s0 += ch == 0 ? ad : 0u; s1 += ch == 1 ? ad : 0u; s2 += ch == 2 ? ad : 0u;
    }
  }
  if (diff) {  // warp shuffles, then the CTA's warps through shared memory:
               // 6 global atomics per CTA (same-address atomics serialise in L2)
    __shared__ unsigned long long part[kStatThreads / 32][6];
    unsigned long long v[6] = {c0, c1, c2, s0, s1, s2};
#pragma unroll
    for (int k = 0; k < 6; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xFFFFFFFFu, v[k], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) part[threadIdx.x >> 5][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 6) {
      unsigned long long t = 0;
      for (int w = 0; w < kStatThreads / 32; ++w) t += part[w][threadIdx.x];
      if (t) atomicAdd(diff + threadIdx.x, t);
    }
  }
  if (hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < 768; i += kStatThreads) {
      uint32_t sum = 0;
#pragma unroll
      for (int k = 0; k < kSubHists; ++k) sum += h[k][i];
      if (sum) atomicAdd(hist + i, (unsigned long long)sum);
    }
  }
}

uint32_t stat_grid(uint64_t nbytes) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // <= 2 CTAs per SM (measured best for histogram + NPCR/UACI); each
  // CTA issues 768 + 6 global atomics
  const uint64_t want = (nbytes / 48 + kStatThreads - 1) / kStatThreads;
  return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sms) * 2)));
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::internal, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void launch_frame_stats(const uint8_t* d_a, const uint8_t* d_b, uint64_t nbytes,
                        unsigned long long* d_hist, unsigned long long* d_diff,
                        cudaStream_t s) {
  if (!d_b) d_diff = nullptr;
  if (!d_hist && !d_diff) return;
  if (d_hist) check(cudaMemsetAsync(d_hist, 0, 768 * sizeof(unsigned long long), s), "memset");
  if (d_diff) check(cudaMemsetAsync(d_diff, 0, 6 * sizeof(unsigned long long), s), "memset");
  const bool vec =
      ((reinterpret_cast<uintptr_t>(d_a) | (d_diff ? reinterpret_cast<uintptr_t>(d_b) : 0)) & 15) == 0;
  k_frame_stats<<<stat_grid(nbytes), kStatThreads, 0, s>>>(d_a, d_b, nbytes, vec, d_hist, d_diff);
  check(cudaGetLastError(), "frame_stats launch");
}

}  // namespace cveb
