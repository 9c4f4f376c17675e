// Row f4: the O(side^2) reductions of the reference's
// statistical analysis on sm_100a -- per-channel byte histograms
// (analysis.cpp:51-60 channel_histogram) and NPCR/UACI counts
// (analysis.cpp:200-218 npcr_uaci).  Everything downstream of these integer
// counts (variance, chi^2, entropy, the percentages) is evaluated on the
// host in the reference's order, so the printed statistics are identical.
//
// Both kernels walk the frame in 48-byte granules (16 pixels): the channel
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

__global__ void __launch_bounds__(kStatThreads)
    k_channel_hist(const uint8_t* __restrict__ px, uint64_t nbytes, bool vec,
                   unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[kSubHists][768];
  for (int i = threadIdx.x; i < kSubHists * 768; i += kStatThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  uint32_t* mine = h[(threadIdx.x >> 6) % kSubHists];
  const uint64_t stride = uint64_t(gridDim.x) * kStatThreads;
  const uint64_t t0 = uint64_t(blockIdx.x) * kStatThreads + threadIdx.x;
  uint64_t done = 0;
  if (vec) {
    const uint64_t G = nbytes / 48;
    const uint4* p = reinterpret_cast<const uint4*>(px);
    for (uint64_t g = t0; g < G; g += stride) {
      const uint4 a = __ldg(p + 3 * g), b = __ldg(p + 3 * g + 1), c = __ldg(p + 3 * g + 2);
      const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 12; ++k) hist_word(mine, w[k], 4 * k);
    }
    done = G * 48;
  }
  for (uint64_t i = done + t0; i < nbytes; i += stride)  // tail / unaligned frames
    atomicAdd(mine + (i % 3) * 256 + px[i], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 768; i += kStatThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kSubHists; ++k) s += h[k][i];
    if (s) atomicAdd(hist + i, (unsigned long long)s);
  }
}

// out[c] = positions where channel c differs, out[3 + c] = sum |a - b|.
__global__ void __launch_bounds__(kStatThreads)
    k_diff_stats(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                 uint64_t nbytes, bool vec, unsigned long long* __restrict__ out) {
  unsigned long long cnt[3] = {0, 0, 0}, abs_sum[3] = {0, 0, 0};
  const uint64_t stride = uint64_t(gridDim.x) * kStatThreads;
  const uint64_t t0 = uint64_t(blockIdx.x) * kStatThreads + threadIdx.x;
  uint64_t done = 0;
  if (vec) {
    const uint64_t G = nbytes / 48;
    const uint4* pa = reinterpret_cast<const uint4*>(a);
    const uint4* pb = reinterpret_cast<const uint4*>(b);
    for (uint64_t g = t0; g < G; g += stride) {
      uint32_t wa[12], wb[12];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const uint4 x = __ldg(pa + 3 * g + i), y = __ldg(pb + 3 * g + i);
        wa[4 * i] = x.x; wa[4 * i + 1] = x.y; wa[4 * i + 2] = x.z; wa[4 * i + 3] = x.w;
        wb[4 * i] = y.x; wb[4 * i + 1] = y.y; wb[4 * i + 2] = y.z; wb[4 * i + 3] = y.w;
      }
      uint32_t c32[3] = {0, 0, 0}, s32[3] = {0, 0, 0};
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const uint32_t d = __vabsdiffu4(wa[k], wb[k]);
        const uint32_t ne = __vcmpne4(wa[k], wb[k]) & 0x01010101u;
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
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        cnt[ch] += c32[ch];
        abs_sum[ch] += s32[ch];
      }
    }
    done = G * 48;
  }
  for (uint64_t i = done + t0; i < nbytes; i += stride) {
    const int d = int(a[i]) - int(b[i]);
    cnt[i % 3] += d != 0;
    abs_sum[i % 3] += uint64_t(d < 0 ? -d : d);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cnt[k] += __shfl_down_sync(0xFFFFFFFFu, cnt[k], o);
      abs_sum[k] += __shfl_down_sync(0xFFFFFFFFu, abs_sum[k], o);
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (cnt[k]) atomicAdd(out + k, cnt[k]);
      if (abs_sum[k]) atomicAdd(out + 3 + k, abs_sum[k]);
    }
  }
}

uint32_t stat_grid(uint64_t nbytes) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (nbytes / 48 + kStatThreads - 1) / kStatThreads;
  return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sms) * 4)));
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::internal, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void launch_frame_stats(const uint8_t* d_a, const uint8_t* d_b, uint64_t nbytes,
                        unsigned long long* d_hist, unsigned long long* d_diff,
                        cudaStream_t s) {
  if (d_hist) {
    check(cudaMemsetAsync(d_hist, 0, 768 * sizeof(unsigned long long), s), "memset");
    const bool vec = (reinterpret_cast<uintptr_t>(d_a) & 15) == 0;
    k_channel_hist<<<stat_grid(nbytes), kStatThreads, 0, s>>>(d_a, nbytes, vec, d_hist);
    check(cudaGetLastError(), "channel_hist launch");
  }
  if (d_b && d_diff) {
    check(cudaMemsetAsync(d_diff, 0, 6 * sizeof(unsigned long long), s), "memset");
    const bool vec = ((reinterpret_cast<uintptr_t>(d_a) | reinterpret_cast<uintptr_t>(d_b)) & 15) == 0;
    k_diff_stats<<<stat_grid(nbytes), kStatThreads, 0, s>>>(d_a, d_b, nbytes, vec, d_diff);
    check(cudaGetLastError(), "diff_stats launch");
  }
}

}  // namespace cveb
