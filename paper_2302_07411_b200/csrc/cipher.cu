// K2/K3/K4: confusion + diffusion round kernels for sm_100a.
//
//   K2s k_encrypt_round_slots / K3s k_decrypt_round_slots: the production
//       rounds (side % 16 == 0, 16-byte aligned frames and keystream):
//       cp.async-staged source runs, 32-bit pixel slots in shared memory,
//       cluster DSMEM band prefix (K2s).  Every benchmark config takes these.
//   K2 k_encrypt_round / K3 k_decrypt_round: byte-staged rounds for any side.
//   k_gather + k_gen_*: generic multi-kernel forward round for bands no
//       cluster can hold.
//   K4 k_shift: the per-frame shift table.
//
// Reference semantics (paths relative to /root/reference/proj):
//   confusion   confuse_rows            src/engine.cpp:32-47   (scatter form)
//               inverse_confuse_rows    src/engine.cpp:49-64
//   diffusion   diffuse_region          src/engine.cpp:66-73, engine.hpp:32-34
//               seed byte s_d           src/engine.cpp:237
//   inverse     inverse_diffuse_region  src/engine.cpp:75-83, engine.hpp:36-38
//               head fix-up             src/engine.cpp:271-276
//   shift table build_shift_table       src/engine.cpp:14-30
//
// Restated for the GPU (probe P1):
//   confusion as a GATHER: y[al][be] = x[(al-o) mod w][o], o = (be-shift[al]) mod w.
//     Destination rows [al0, al0+R) read, from EVERY source row a, the
//     contiguous run o in [al0-a, al0-a+R) -- a diagonal stripe.
//   diffusion as an XOR PREFIX SCAN: with t_j = b_j ^ ((y_j + b_j) mod 256),
//     c_j = s_d ^ t_0 ^ ... ^ t_j   over the bytes of one row band.
//   inverse diffusion is elementwise: d_j = ((b_j ^ c_j ^ c_{j-1}) - b_j),
//     the band head using the next band's recovered last byte.
//
// Data layout in HBM: frames are the reference's square row-major
// interleaved RGB24 buffers; band i = bytes [i*region, (i+1)*region).
// Keystream: one ring per worker, stream byte s at ring[i*R + s % R]; the
// bytes of round k of a frame start at the frame's stream position + k*region
// (engine.cpp:198-205, 227-230).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.hpp"
#include "keying.hpp"

namespace cg = cooperative_groups;

namespace cveb {
namespace {

// Device-side bounds checks (make BOUNDS=1): every global address the round
// kernels form is checked against its buffer before use; a failure prints
// and traps.  Compiled out otherwise.
#ifdef CVE_B200_BOUNDS
#define CVE_CHECK(cond)                                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("cve bounds check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define CVE_CHECK(cond) ((void)0)
#endif
__device__ __forceinline__ bool within(const void* p, uint64_t n, const void* base,
                                       uint64_t bytes) {
  const uint8_t* q = static_cast<const uint8_t*>(p);
  const uint8_t* b = static_cast<const uint8_t*>(base);
  return q >= b && q + n <= b + bytes;
}

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kEncThreads = 512;
constexpr int kSeg = 4;  // granules per thread per super-tile
constexpr uint32_t kDecThreads = 512;
constexpr size_t kSmemBudget = 200 * 1024;
constexpr int kStageBatch = 8;  // pixels in flight per thread while staging

// floor(n / d) for 32-bit n, d via one 64x64 high multiply.
struct FastDiv {
  uint32_t d;
  uint64_t m;  // floor((2^64-1)/d) + 1, or 0 when d == 1
};

FastDiv make_div(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.m = d == 1 ? 0 : (~uint64_t(0)) / d + 1;
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.d == 1 ? n : uint32_t(__umul64hi(uint64_t(n), f.m));
}

// Keystream bytes are read exactly once per frame: they are loaded with an
// L2 evict-first policy (KS_HINT, default on), so the stream of keystream
// does not push the round's frame buffers (re-read by the next round) out
// of L2.
#ifndef KS_HINT
#define KS_HINT 1
#endif
__device__ __forceinline__ uint64_t ks_policy() {
  uint64_t pol = 0;
#if KS_HINT
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}

__device__ __forceinline__ uint4 ld_stream(const uint8_t* p, uint64_t pol = ks_policy()) {
  uint4 v;
#if KS_HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
#else
  (void)pol;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
#endif
  return v;
}

// Byte lanes of a word: (y + b) mod 256 without cross-byte carries.
__device__ __forceinline__ uint32_t add_bytes(uint32_t y, uint32_t b) {
  return ((y & 0x7F7F7F7Fu) + (b & 0x7F7F7F7Fu)) ^ ((y ^ b) & 0x80808080u);
}

// t = b ^ (y + b) on 8 bytes, then inclusive XOR prefix across the bytes
// (byte k of the result = t_0 ^ ... ^ t_k, little-endian byte order).
__device__ __forceinline__ uint64_t t_prefix8(uint32_t y0, uint32_t y1,
                                              uint32_t b0, uint32_t b1) {
  const uint64_t t = uint64_t(b0 ^ add_bytes(y0, b0)) |
                     (uint64_t(b1 ^ add_bytes(y1, b1)) << 32);
  uint64_t s = t ^ (t << 8);
  s ^= s << 16;
  s ^= s << 32;
  return s;
}

constexpr uint64_t kBcast = 0x0101010101010101ull;

// Exclusive XOR scan of one byte per thread across the CTA.  `wsum` holds
// 2 x 32 words (double-buffered by `phase` so one barrier per call suffices).
__device__ __forceinline__ uint32_t block_xor_scan(uint32_t v, uint32_t* wsum,
                                                   uint32_t phase,
                                                   uint32_t& total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nwarps = blockDim.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(kFull, inc, d);
    if (lane >= uint32_t(d)) inc ^= u;
  }
  uint32_t* ws = wsum + 32 * (phase & 1);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint32_t wprefix = 0, tot = 0;
  // every warp scans the (<=32) warp totals redundantly: no second barrier
  const uint32_t w = lane < nwarps ? ws[lane] : 0u;
  uint32_t winc = w;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(kFull, winc, d);
    if (lane >= uint32_t(d)) winc ^= u;
  }
  wprefix = __shfl_sync(kFull, winc ^ w, warp);  // exclusive for this warp
  tot = __shfl_sync(kFull, winc, 31);
  total = tot;
  return wprefix ^ inc ^ v;
}

// ---------------------------------------------------------------------------
// K4: per-frame shift table.
__global__ void k_shift(const double* __restrict__ sine, uint32_t seed,
                        int32_t* __restrict__ shift, uint32_t side) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= side) return;
  const double v = __dmul_rn(double(seed), sine[a]);
  const long long s = (long long)floor(v);
  long long r = s % (long long)side;
  if (r < 0) r += side;
  shift[a] = int32_t(r);
}

// ---------------------------------------------------------------------------
// K2: fused forward round.  One CTA per (band, chunk of chunk_rows rows);
// the h chunks of a band form one thread-block cluster and exchange their
// XOR aggregates through distributed shared memory.
struct EncArgs {
  const uint8_t* src;
  uint8_t* dst;
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;
  const int32_t* shift;
  uint32_t side, n, rows, chunk_rows, h;
  uint64_t region;
  FastDiv div_cr;
  uint64_t frame_bytes;  // bounds checks only
};

__device__ __forceinline__ uint8_t seed_byte(const EncArgs& a, uint32_t band) {
  // s_d = post-confusion byte ((band+1) mod n + 1)*region - 1: pixel
  // (last row of the next band, column side-1), channel 2.
  const uint32_t nb = band + 1 == a.n ? 0 : band + 1;
  const uint32_t al = nb * a.rows + a.rows - 1;
  int o = int(a.side - 1) - a.shift[al];
  if (o < 0) o += a.side;
  int sr = int(al) - o;
  if (sr < 0) sr += a.side;
  return a.src[(uint64_t(sr) * a.side + uint32_t(o)) * 3 + 2];
}

// Layout of one CTA's work: the chunk's G 16-byte granules (destination
// order) are split into super-tiles of blockDim*kSeg granules; thread t owns
// the contiguous granules [t*kSeg, (t+1)*kSeg) of each super-tile, keeps
// their keystream and results in registers, and the CTA needs one barrier
// per super-tile for the XOR scan.
template <bool VEC>
__device__ __forceinline__ uint4 load_ks16(const uint8_t* ks, uint64_t ring_bytes,
                                           uint64_t kp, uint32_t valid) {
  if (VEC) return ld_stream(ks + kp);
  uint32_t w[4] = {0, 0, 0, 0};
  for (uint32_t i = 0; i < valid; ++i) {
    uint64_t q = kp + i;
    if (q >= ring_bytes) q -= ring_bytes;
    w[i >> 2] |= uint32_t(__ldg(ks + q)) << (8 * (i & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <bool VEC>
__global__ void __launch_bounds__(kEncThreads)
    k_encrypt_round(const EncArgs a) {
  extern __shared__ uint4 smem[];
  __shared__ uint32_t wsum[64];
  __shared__ uint32_t agg_share;
  __shared__ uint32_t prefix_share;

  uint8_t* ys = reinterpret_cast<uint8_t*>(smem);
  const uint32_t tid = threadIdx.x;
  const uint32_t band = blockIdx.x / a.h;
  const uint32_t chunk = blockIdx.x - band * a.h;
  const uint32_t cr = a.chunk_rows, side = a.side;
  const uint32_t al0 = band * a.rows + chunk * cr;
  const uint32_t cb = cr * side * 3;  // chunk bytes
  const uint32_t cb16 = (cb + 15) & ~15u;
  const uint32_t G = cb16 / 16;
  const uint32_t tile = blockDim.x * kSeg;  // granules per super-tile
  int32_t* shs = reinterpret_cast<int32_t*>(ys + cb16);
  const uint8_t* ks = a.ring + uint64_t(band) * a.ring_bytes;
  uint64_t kbase = a.pos + uint64_t(chunk) * cb;  // < 2R
  if (kbase >= a.ring_bytes) kbase -= a.ring_bytes;
  auto ks_at = [&](uint32_t g) {
    uint64_t kp = kbase + 16ull * g;
    if (kp >= a.ring_bytes) kp -= a.ring_bytes;
    return kp;
  };

  // 1. keystream of this thread's first super-tile segment: in flight while
  //    the frame is staged.
  uint4 kv[kSeg];
#pragma unroll
  for (int k = 0; k < kSeg; ++k) {
    const uint32_t g = tid * kSeg + k;
    kv[k] = make_uint4(0, 0, 0, 0);
    if (g < G) kv[k] = load_ks16<VEC>(ks, a.ring_bytes, ks_at(g), min(16u, cb - 16 * g));
  }

  for (uint32_t t = tid; t < cr; t += blockDim.x) shs[t] = a.shift[al0 + t];
  if (!VEC)
    for (uint32_t i = cb + tid; i < cb16; i += blockDim.x) ys[i] = 0;
  if (tid == 0) prefix_share = seed_byte(a, band);
  __syncthreads();

  // 2. Stage + permute: source pixel (sr, o) with sr + o == al (mod side)
  //    lands at chunk row al - al0, column (o + shift[al]) mod side.
  //    kStageBatch pixels per thread per pass, all loads before any store.
  const uint32_t items = side * cr;
  for (uint32_t base = tid; base < items; base += kStageBatch * blockDim.x) {
    uint8_t v[kStageBatch][3];
    uint32_t dofs[kStageBatch];
#pragma unroll
    for (int k = 0; k < kStageBatch; ++k) {
      const uint32_t idx = base + k * blockDim.x;
      dofs[k] = ~0u;
      if (idx < items) {
        const uint32_t sr = fdiv(idx, a.div_cr);
        const uint32_t t = idx - sr * cr;
        int o = int(al0 + t) - int(sr);
        if (o < 0) o += side;
        uint32_t be = uint32_t(o) + uint32_t(shs[t]);
        if (be >= side) be -= side;
        const uint8_t* sp = a.src + (uint64_t(sr) * side + uint32_t(o)) * 3;
        v[k][0] = __ldg(sp);
        v[k][1] = __ldg(sp + 1);
        v[k][2] = __ldg(sp + 2);
        dofs[k] = (t * side + be) * 3;
      }
    }
#pragma unroll
    for (int k = 0; k < kStageBatch; ++k) {
      if (dofs[k] != ~0u) {
        ys[dofs[k]] = v[k][0];
        ys[dofs[k] + 1] = v[k][1];
        ys[dofs[k] + 2] = v[k][2];
      }
    }
  }
  __syncthreads();

  // 3. Chunk XOR scan of t = b ^ (y + b), super-tile by super-tile.  The
  //    chunk prefix (s_d ^ earlier chunks of the band) is applied at the end,
  //    so the results stay in registers (single super-tile) or in smem.
  uint32_t carry = 0;  // XOR of every t in earlier super-tiles
  uint4 res[kSeg];
  uint32_t excl_last = 0;
  const uint32_t ntiles = (G + tile - 1) / tile;
  for (uint32_t st = 0; st < ntiles; ++st) {
    const uint32_t gs = st * tile + tid * kSeg;
    if (st > 0) {
#pragma unroll
      for (int k = 0; k < kSeg; ++k) {
        const uint32_t g = gs + k;
        kv[k] = make_uint4(0, 0, 0, 0);
        if (g < G) kv[k] = load_ks16<VEC>(ks, a.ring_bytes, ks_at(g), min(16u, cb - 16 * g));
      }
    }
    uint32_t run = 0;  // running XOR within the thread's segment
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
      const uint32_t g = gs + k;
      const uint4 y = g < G ? smem[g] : make_uint4(0, 0, 0, 0);
      uint64_t lo = t_prefix8(y.x, y.y, kv[k].x, kv[k].y);
      uint64_t hi = t_prefix8(y.z, y.w, kv[k].z, kv[k].w);
      hi ^= (lo >> 56) * kBcast;
      const uint64_t m = uint64_t(run) * kBcast;
      lo ^= m;
      hi ^= m;
      run = uint32_t(hi >> 56);
      res[k] = make_uint4(uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi), uint32_t(hi >> 32));
    }
    uint32_t total;
    const uint32_t excl = block_xor_scan(run, wsum, st, total) ^ carry;
    if (ntiles > 1) {  // park this super-tile's results (prefix not known yet)
      const uint32_t m = excl * 0x01010101u;
#pragma unroll
      for (int k = 0; k < kSeg; ++k) {
        const uint32_t g = gs + k;
        if (g < G) smem[g] = make_uint4(res[k].x ^ m, res[k].y ^ m, res[k].z ^ m, res[k].w ^ m);
      }
    } else {
      excl_last = excl;
    }
    carry ^= total;
  }

  // 4. Band prefix: s_d ^ aggregates of the chunks before this one.
  if (a.h > 1) {
    cg::cluster_group cluster = cg::this_cluster();
    if (tid == 0) agg_share = carry;
    cluster.sync();
    if (tid == 0) {
      uint32_t p = prefix_share;
      const uint32_t me = cluster.block_rank();
      for (uint32_t j = 0; j < me; ++j) p ^= *cluster.map_shared_rank(&agg_share, j);
      prefix_share = p;
    }
    cluster.sync();
  } else {
    __syncthreads();
  }

  // 5. Output.
  uint8_t* out = a.dst + uint64_t(band) * a.region + uint64_t(chunk) * cb;
  if (ntiles == 1) {
    const uint32_t m = (prefix_share ^ excl_last) * 0x01010101u;
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
      const uint32_t g = tid * kSeg + k;
      if (g >= G) continue;
      const uint4 v = make_uint4(res[k].x ^ m, res[k].y ^ m, res[k].z ^ m, res[k].w ^ m);
      if (VEC) {
        reinterpret_cast<uint4*>(out)[g] = v;
      } else {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        for (uint32_t i = 0; i < 16 && 16 * g + i < cb; ++i)
          out[16 * g + i] = uint8_t(w[i >> 2] >> (8 * (i & 3)));
      }
    }
  } else {
    const uint32_t m = prefix_share * 0x01010101u;
    if (VEC) {
      uint4* out4 = reinterpret_cast<uint4*>(out);
      for (uint32_t g = tid; g < G; g += blockDim.x) {
        const uint4 v = smem[g];
        out4[g] = make_uint4(v.x ^ m, v.y ^ m, v.z ^ m, v.w ^ m);
      }
    } else {
      for (uint32_t j = tid; j < cb; j += blockDim.x) out[j] = ys[j] ^ uint8_t(m);
    }
  }
}

// ---------------------------------------------------------------------------
// K2s: the forward round for side % 16 == 0 with 16-byte aligned frames and
// keystream.  Same work split as K2 (one CTA per chunk of cr <= 16
// destination rows al0 .. al0+cr-1, the h chunks of a band in one cluster):
//
//  1. Staging.  Source row sr holds the chunk's pixels at columns
//     o0 .. o0+cr-1, o0 = (al0 - sr) mod side -- one contiguous run of 3*cr
//     bytes (pixel k belongs to destination row al0 + k).  The runs' aligned
//     64-byte windows are copied global -> shared with cp.async (four threads
//     per row, so a warp covers 8 rows per instruction), 512 rows per stage,
//     double-buffered.  Each stage is then repacked by thread = row: the
//     window is realigned in registers and pixel k is stored as one 32-bit
//     slot at k*side + (o0 + c_k) mod side, c_k = (k + shift[al0+k]) mod side
//     (consecutive rows -> consecutive columns: no bank conflicts).  Runs
//     that wrap past the row end (cr - 1 rows per chunk) are read pixel by
//     pixel from global.
//  2. Scan.  One 48-byte granule (16 slots -> 12 packed words) per thread per
//     super-tile, 32-bit SWAR diffusion, the next super-tile's keystream in
//     flight during the current one; one CTA-wide XOR scan per super-tile.
//  3. Band prefix across the cluster (DSMEM), 4. 16-byte stores.
//
// Slot layout: granule u = slots [16u, 16u+16); its 4-slot quarter c lives
// at quarter c ^ ((u >> 1) & 3), so the 8 granules a quarter-warp reads with
// one LDS.128 cover all 32 banks.  Window layout: row r's 16-byte chunk c at
// chunk c ^ ((r >> 1) & 3) of its 64-byte slot, same reason.
constexpr uint32_t kSlotThreads = 512;
constexpr uint32_t kMaxChunkRows = 16;
constexpr uint32_t kStageRows = kSlotThreads;  // rows per staging stage
constexpr uint32_t kWinBytes = 64;
constexpr uint32_t kStageBytes = kStageRows * kWinBytes;
constexpr size_t kSlotSmemMax = 224 * 1024;

__device__ __forceinline__ uint32_t slot_word(uint32_t s) {
  return s ^ ((s >> 3) & 12u);  // quarter bits (2,3) ^= granule bits (5,6)
}

// t = b ^ ((y + b) mod 256) per byte, then the inclusive XOR prefix across the
// word's bytes (little-endian order).
__device__ __forceinline__ uint32_t t_prefix4(uint32_t y, uint32_t b) {
  uint32_t t = b ^ add_bytes(y, b);
  t ^= t << 8;
  t ^= t << 16;
  return t;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(pred ? 16 : 0)
               : "memory");
}
// keystream windows: with the evict-first L2 policy (see ld_stream)
__device__ __forceinline__ void cp_async16_ks(uint32_t dst, const void* src, bool pred,
                                              uint64_t pol) {
#if KS_HINT
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst),
               "l"(src), "r"(pred ? 16 : 0), "l"(pol)
               : "memory");
#else
  (void)pol;
  cp_async16(dst, src, pred);
#endif
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kSlotThreads, 1)
    k_encrypt_round_slots(const EncArgs a) {
  extern __shared__ uint4 smem[];
  __shared__ uint32_t cks[kMaxChunkRows];
  __shared__ uint32_t wsum[64];
  __shared__ uint32_t agg_in[16];  // aggregates of earlier chunks (cluster rank j)
  __shared__ uint32_t agg_share;
  __shared__ uint32_t prefix_share;

  const uint32_t tid = threadIdx.x;
  const uint32_t band = blockIdx.x / a.h;
  const uint32_t chunk = blockIdx.x - band * a.h;
  const uint32_t cr = a.chunk_rows, side = a.side;
  const uint32_t al0 = band * a.rows + chunk * cr;
  const uint32_t G = (cr * side) >> 4;  // 48-byte granules in the chunk
  const uint32_t cb = cr * side * 3;
  const uint32_t slots_base = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t win_base = slots_base + cr * side * 4u;  // 2 stages of windows
  const uint8_t* ks = a.ring + uint64_t(band) * a.ring_bytes;
  uint64_t kbase = a.pos + uint64_t(chunk) * cb;
  if (kbase >= a.ring_bytes) kbase -= a.ring_bytes;
  // kbase and ring_bytes are multiples of 48 (launch condition): a granule
  // never straddles the ring end
  auto load_ks = [&](uint32_t g, uint4 (&kv)[3]) {
    uint64_t kp = kbase + 48ull * g;
    if (kp >= a.ring_bytes) kp -= a.ring_bytes;
    const uint8_t* p = ks + kp;
    if (g < G) CVE_CHECK(within(p, 48, ks, a.ring_bytes));
#pragma unroll
    for (int i = 0; i < 3; ++i) kv[i] = g < G ? ld_stream(p + 16 * i) : make_uint4(0, 0, 0, 0);
  };
  // source run of row sr: first column and byte offset
  auto run_of = [&](uint32_t sr, uint32_t& o0, uint32_t& b0) {
    int o = int(al0) - int(sr);
    o += o < 0 ? int(side) : 0;
    o0 = uint32_t(o);
    b0 = (sr * side + o0) * 3u;
  };
  const uint32_t nstages = (side + kStageRows - 1) / kStageRows;
  // Thread tid owns source row st * kStageRows + tid of stage st: it copies
  // the row's aligned 64-byte window (the chunks its run touches) into its
  // own window slot of buffer st & 1, and repacks it once its copies land --
  // no CTA barrier between stages.  Stage st + 1 is in flight during st.
  auto issue_row = [&](uint32_t st) {
    const uint32_t sr = st * kStageRows + tid;
    const uint32_t w = win_base + (st & 1u) * kStageBytes + tid * kWinBytes;
    const uint32_t sw = (tid >> 1) & 3u;
    uint32_t o0 = 0, b0 = 0;
    if (sr < side) run_of(sr, o0, b0);
    // runs that wrap past the row end are read by the deferred pass (their
    // window could run past the end of the frame: last chunk, row side-1)
    const bool live = sr < side && o0 + cr <= side;
    const uint8_t* src = a.src + (b0 & ~15u);
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
      const bool need = live && 16u * c < (b0 & 15u) + 3u * cr;
      if (need) CVE_CHECK(within(src + 16u * c, 16, a.src, a.frame_bytes));
      cp_async16(w + 16u * (c ^ sw), src + 16u * c, need);
    }
    cp_async_commit();
  };

  // Programmatic dependent launch: the next round may be scheduled as soon
  // as SMs free up; it runs its independent prologue (first keystream tile,
  // cluster arrive) and waits for this grid before touching the frame.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // cluster phase 1 (arrive now, wait before the DSMEM stores): every CTA of
  // the cluster has started before any remote store lands in it
  if (a.h > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  uint4 kv[3];
  load_ks(tid, kv);  // first super-tile's keystream (independent of the frame)
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous round / shift table done
  issue_row(0);
  for (uint32_t t = tid; t < cr; t += kSlotThreads) {
    uint32_t c = t + uint32_t(a.shift[al0 + t]);
    cks[t] = c >= side ? c - side : c;
  }
  if (tid == 0) prefix_share = seed_byte(a, band);
  __syncthreads();

  // 1. Staging.
  {
    uint32_t dk[kMaxChunkRows], ek[kMaxChunkRows];
#pragma unroll
    for (int k = 0; k < int(kMaxChunkRows); ++k) {
      const uint32_t c = uint32_t(k) < cr ? cks[k] : 0u;
      dk[k] = uint32_t(k) * side + c;
      ek[k] = side - c;  // o0 >= ek  <=>  o0 + c_k >= side
    }
    auto put = [&](int k, uint32_t o0, uint32_t pix) {
      const uint32_t sl = dk[k] + o0 - (o0 >= ek[k] ? side : 0u);
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots_base + 4u * slot_word(sl)), "r"(pix));
    };
    for (uint32_t st = 0; st < nstages; ++st) {
      if (st + 1 < nstages) {
        issue_row(st + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      const uint32_t sr = st * kStageRows + tid;
      if (sr < side) {
        uint32_t o0, b0;
        run_of(sr, o0, b0);
        if (o0 + cr <= side) {
          const uint32_t w = win_base + (st & 1u) * kStageBytes + tid * kWinBytes;
          const uint32_t sw = (tid >> 1) & 3u;
          uint32_t V[16];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(V[4 * c]), "=r"(V[4 * c + 1]), "=r"(V[4 * c + 2]), "=r"(V[4 * c + 3])
                         : "r"(w + 16u * (uint32_t(c) ^ sw)));
          const uint32_t ws = (b0 >> 2) & 3u, bs = (b0 & 3u) * 8u;
          uint32_t X[14], U[13], A[12];
#pragma unroll
          for (int i = 0; i < 14; ++i) X[i] = (ws & 2u) ? V[i + 2] : V[i];
#pragma unroll
          for (int i = 0; i < 13; ++i) U[i] = (ws & 1u) ? X[i + 1] : X[i];
#pragma unroll
          for (int i = 0; i < 12; ++i) A[i] = __funnelshift_r(U[i], U[i + 1], bs);
#pragma unroll
          for (int k = 0; k < int(kMaxChunkRows); ++k) {
            if (uint32_t(k) >= cr) break;
            const int j = (3 * k) >> 2, sh = ((3 * k) & 3) * 8;
            put(k, o0, sh <= 8 ? (A[j] >> sh) : __funnelshift_r(A[j], A[j + 1], sh));
          }
        }  // runs that wrap past the row end: deferred, below
      }
    }
    // The cr - 1 source rows whose run wraps past the row end are rows
    // al0 + i (i = 1 .. cr-1, o0 = side - i): one thread per pixel, every
    // load in flight at once.
    const uint32_t nwrap = min(cr, side) - 1;
    for (uint32_t it = tid; it < nwrap * cr; it += kSlotThreads) {
      const uint32_t i = it / cr + 1, k = it - (i - 1) * cr;
      uint32_t sr = al0 + i;
      sr -= sr >= side ? side : 0u;
      const uint32_t o0 = side - i;
      uint32_t o = o0 + k;
      o -= o >= side ? side : 0u;
      const uint8_t* sp = a.src + (uint64_t(sr) * side + o) * 3;
      CVE_CHECK(within(sp, 3, a.src, a.frame_bytes));
      const uint32_t pix = uint32_t(__ldg(sp)) | (uint32_t(__ldg(sp + 1)) << 8) |
                           (uint32_t(__ldg(sp + 2)) << 16);
      uint32_t be = o0 + cks[k];
      be -= be >= side ? side : 0u;
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots_base + 4u * slot_word(k * side + be)),
                   "r"(pix));
    }
  }
  __syncthreads();

  // 2. Chunk XOR scan, one granule per thread per super-tile.
  uint32_t carry = 0, excl_last = 0;
  uint32_t res[12];
  const uint32_t ntiles = (G + kSlotThreads - 1) / kSlotThreads;
  for (uint32_t st = 0; st < ntiles; ++st) {
    const uint32_t g = st * kSlotThreads + tid;
    uint4 kn[3];
    if (st + 1 < ntiles) load_ks(g + kSlotThreads, kn);
    uint32_t y[12];
    const uint32_t sw = (g >> 1) & 3u;
    if (g < G) {
      const uint4* q = smem + 4 * g;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 s = q[c ^ sw];  // 4 slots (3 bytes each) -> 3 packed words
        y[3 * c] = __byte_perm(s.x, s.y, 0x4210);
        y[3 * c + 1] = __byte_perm(s.y, s.z, 0x5421);
        y[3 * c + 2] = __byte_perm(s.z, s.w, 0x6542);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 12; ++i) y[i] = 0;
    }
    const uint32_t kw[12] = {kv[0].x, kv[0].y, kv[0].z, kv[0].w, kv[1].x, kv[1].y,
                             kv[1].z, kv[1].w, kv[2].x, kv[2].y, kv[2].z, kv[2].w};
    uint32_t E = 0;  // XOR of every earlier t byte, broadcast to 4 bytes
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const uint32_t t = t_prefix4(y[i], kw[i]);
      res[i] = t ^ E;
      E ^= __byte_perm(t, 0, 0x3333);
    }
    uint32_t total;
    const uint32_t excl = block_xor_scan(E & 0xFFu, wsum, st, total) ^ carry;
    if (ntiles > 1) {  // park the results in the granule's own slots
      if (g < G) {
        const uint32_t m = excl * 0x01010101u;
        uint4* q = smem + 4 * g;
        q[0 ^ sw] = make_uint4(res[0] ^ m, res[1] ^ m, res[2] ^ m, res[3] ^ m);
        q[1 ^ sw] = make_uint4(res[4] ^ m, res[5] ^ m, res[6] ^ m, res[7] ^ m);
        q[2 ^ sw] = make_uint4(res[8] ^ m, res[9] ^ m, res[10] ^ m, res[11] ^ m);
      }
    } else {
      excl_last = excl;
    }
    carry ^= total;
    if (st + 1 < ntiles) {
#pragma unroll
      for (int i = 0; i < 3; ++i) kv[i] = kn[i];
    }
  }

  // 3. Band prefix: s_d ^ aggregates of the chunks before this one.  Each
  //    CTA pushes its aggregate into the later CTAs' agg_in[] (DSMEM stores),
  //    then one release/acquire cluster barrier.
  if (a.h > 1) {
    const uint32_t me = blockIdx.x - band * a.h;  // == cluster rank
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (tid > me && tid < a.h) {
      const uint32_t local = uint32_t(__cvta_generic_to_shared(&agg_in[me]));
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(tid));
      asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(carry) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (tid == 0) {
      uint32_t p = prefix_share;
      for (uint32_t j = 0; j < me; ++j) p ^= agg_in[j];
      prefix_share = p;
    }
  }
  __syncthreads();

  // 4. Output (16-byte stores, consecutive threads on consecutive pieces).
  uint4* out4 = reinterpret_cast<uint4*>(a.dst + uint64_t(band) * a.region +
                                         uint64_t(chunk) * cb);
  if (ntiles == 1) {
    if (tid < G) {
      CVE_CHECK(within(out4 + 3 * tid, 48, a.dst, a.frame_bytes));
      const uint32_t m = (prefix_share ^ excl_last) * 0x01010101u;
      out4[3 * tid] = make_uint4(res[0] ^ m, res[1] ^ m, res[2] ^ m, res[3] ^ m);
      out4[3 * tid + 1] = make_uint4(res[4] ^ m, res[5] ^ m, res[6] ^ m, res[7] ^ m);
      out4[3 * tid + 2] = make_uint4(res[8] ^ m, res[9] ^ m, res[10] ^ m, res[11] ^ m);
    }
  } else {
    const uint32_t m = prefix_share * 0x01010101u;
    for (uint32_t q = tid; q < 3 * G; q += kSlotThreads) {
      const uint32_t g = q / 3, c = q - 3 * g;
      const uint4 v = smem[4 * g + (c ^ ((g >> 1) & 3u))];
      CVE_CHECK(within(out4 + q, 16, a.dst, a.frame_bytes));
      out4[q] = make_uint4(v.x ^ m, v.y ^ m, v.z ^ m, v.w ^ m);
    }
  }
}

// ---------------------------------------------------------------------------
// K3: fused inverse round.  One CTA per tile of T output rows; for every
// cipher row al it gathers the contiguous run of T pixels that lands in the
// tile, inverse-diffuses them elementwise, and writes the tile back with
// coalesced stores.
struct DecArgs {
  const uint8_t* src;
  uint8_t* dst;
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;
  const int32_t* shift;
  uint32_t side, n, rows, T;
  uint64_t region;
  FastDiv div_T, div_rows;
  uint64_t frame_bytes;  // bounds checks only
};

__device__ __forceinline__ uint8_t ks_byte(const DecArgs& a, uint32_t band,
                                           uint64_t j) {
  uint64_t kp = a.pos + j;
  if (kp >= a.ring_bytes) kp -= a.ring_bytes;
  return __ldg(a.ring + uint64_t(band) * a.ring_bytes + kp);
}

template <bool VEC>
__global__ void __launch_bounds__(kDecThreads)
    k_decrypt_round(const DecArgs a) {
  extern __shared__ uint4 smem[];
  uint8_t* tile = reinterpret_cast<uint8_t*>(smem);
  const uint32_t side = a.side, T = a.T;
  const uint32_t a0 = blockIdx.x * T;
  const uint32_t tv = min(T, side - a0);
  const uint32_t items = side * T;
  for (uint32_t base = threadIdx.x; base < items; base += kStageBatch * blockDim.x) {
    uint8_t c[kStageBatch][4], k3[kStageBatch][3];
    uint32_t dofs[kStageBatch];
#pragma unroll
    for (int k = 0; k < kStageBatch; ++k) {
      const uint32_t idx = base + k * blockDim.x;
      dofs[k] = ~0u;
      if (idx >= items) continue;
      const uint32_t al = fdiv(idx, a.div_T);
      const uint32_t t = idx - al * T;
      if (t >= tv) continue;
      int o = int(al) - int(a0 + t);
      if (o < 0) o += side;
      uint32_t be = uint32_t(o) + uint32_t(__ldg(a.shift + al));
      if (be >= side) be -= side;
      const uint64_t P = (uint64_t(al) * side + be) * 3;
      const uint32_t band = fdiv(al, a.div_rows);
      const uint64_t j0 = P - uint64_t(band) * a.region;
      c[k][1] = __ldg(a.src + P);
      c[k][2] = __ldg(a.src + P + 1);
      c[k][3] = __ldg(a.src + P + 2);
      if (j0 == 0) {  // band head: next band's recovered last byte
        const uint32_t nb = band + 1 == a.n ? 0 : band + 1;
        const uint64_t L = (uint64_t(nb) + 1) * a.region - 1;
        const uint8_t kl = ks_byte(a, nb, a.region - 1);
        c[k][0] = uint8_t((kl ^ a.src[L] ^ a.src[L - 1]) - kl);
      } else {
        c[k][0] = __ldg(a.src + P - 1);
      }
      k3[k][0] = ks_byte(a, band, j0);
      k3[k][1] = ks_byte(a, band, j0 + 1);
      k3[k][2] = ks_byte(a, band, j0 + 2);
      dofs[k] = (t * side + uint32_t(o)) * 3;
    }
#pragma unroll
    for (int k = 0; k < kStageBatch; ++k) {
      if (dofs[k] == ~0u) continue;
      uint8_t* d = tile + dofs[k];
      d[0] = uint8_t((k3[k][0] ^ c[k][1] ^ c[k][0]) - k3[k][0]);
      d[1] = uint8_t((k3[k][1] ^ c[k][2] ^ c[k][1]) - k3[k][1]);
      d[2] = uint8_t((k3[k][2] ^ c[k][3] ^ c[k][2]) - k3[k][2]);
    }
  }
  __syncthreads();
  const uint32_t bytes = tv * side * 3;
  uint8_t* out = a.dst + uint64_t(a0) * side * 3;
  if (VEC) {
    uint4* out4 = reinterpret_cast<uint4*>(out);
    for (uint32_t g = threadIdx.x; g < bytes / 16; g += blockDim.x) out4[g] = smem[g];
  } else {
    for (uint32_t j = threadIdx.x; j < bytes; j += blockDim.x) out[j] = tile[j];
  }
}

// ---------------------------------------------------------------------------
// K3s: the inverse round for side % 16 == 0 (16-byte aligned frames and
// keystream).  One CTA per tile of T destination rows a0 .. a0+tv-1 (no
// cluster: the inverse diffusion is elementwise).  Source (cipher) row al
// holds the tile's pixels at columns be_lo .. be_lo+tv-1,
// be_lo = (al - a0 - tv + 1 + shift[al]) mod side -- one contiguous run; its
// keystream bytes are one contiguous run of the band's stream too.  Per
// stage of 256 source rows both 64-byte windows are copied with cp.async
// (8 threads per row), then thread = row realigns them, inverse-diffuses
// d = ((b ^ c ^ c_prev) - b) four bytes at a time and stores pixel m as a
// slot of destination row a0 + tv-1-m, column (al - a0 - tv+1 + m) mod side.
// Band heads (which need the next band's recovered last byte) and runs that
// wrap past the row end go byte by byte.  The tile's rows are contiguous in
// the frame: output is packed 48-byte granules.
constexpr uint32_t kDecStageRows = 256;
constexpr uint32_t kDecWin = 128;  // 64 B cipher window + 64 B keystream window
constexpr uint32_t kDecStageBytes = kDecStageRows * kDecWin;
constexpr uint32_t kDecDefer = 256;

// bytewise (x - y) mod 256
__device__ __forceinline__ uint32_t sub_bytes(uint32_t x, uint32_t y) {
  return ((x | 0x80808080u) - (y & 0x7F7F7F7Fu)) ^ ((x ^ ~y) & 0x80808080u);
}

// 12 words starting `off` (0..15) bytes into a 16-word window
__device__ __forceinline__ void realign12(const uint32_t (&V)[16], uint32_t off,
                                          uint32_t (&A)[12]) {
  const uint32_t ws = off >> 2, bs = (off & 3u) * 8u;
  uint32_t X[14], U[13];
#pragma unroll
  for (int i = 0; i < 14; ++i) X[i] = (ws & 2u) ? V[i + 2] : V[i];
#pragma unroll
  for (int i = 0; i < 13; ++i) U[i] = (ws & 1u) ? X[i + 1] : X[i];
#pragma unroll
  for (int i = 0; i < 12; ++i) A[i] = __funnelshift_r(U[i], U[i + 1], bs);
}

__global__ void __launch_bounds__(kSlotThreads, 1)
    k_decrypt_round_slots(const DecArgs a) {
  extern __shared__ uint4 smem[];
  const uint32_t tid = threadIdx.x, side = a.side, T = a.T;
  const uint32_t a0 = blockIdx.x * T;
  const uint32_t tv = min(T, side - a0);
  const uint32_t slots_base = uint32_t(__cvta_generic_to_shared(smem));
  int32_t* sht = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(smem) + T * side * 4u);
  // per-row run info of 3 stages (P0, keystream position, band | fast<<31)
  uint4* rinfo = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(smem) + T * side * 4u +
                                          side * 4u);
  const uint32_t win_base = slots_base + T * side * 4u + side * 4u + 3u * kDecStageRows * 16u;
  const uint32_t region = uint32_t(a.region);

  __shared__ uint32_t dlist[kDecDefer];  // rows deferred to the per-pixel pass
  __shared__ uint32_t dcount;
  // programmatic dependent launch: hides the launch gap between rounds; the
  // shift table and the frame are read only after the previous grid is done
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (uint32_t i = tid; i < side; i += kSlotThreads) sht[i] = a.shift[i];
  if (tid == 0) dcount = 0;
  __syncthreads();

  struct Run {
    uint32_t band, be_lo, P0;
    uint64_t kp0;
    bool fast;
  };
  auto run_of = [&](uint32_t al) {
    Run r;
    r.band = fdiv(al, a.div_rows);
    int b = int(al) - int(a0) - int(tv) + 1 + sht[al];  // in (-side, 2 side)
    b += b < 0 ? int(side) : 0;
    b -= b >= int(side) ? int(side) : 0;
    r.be_lo = uint32_t(b);
    r.P0 = (al * side + r.be_lo) * 3u;
    uint64_t kp = a.pos + (r.P0 - r.band * region);
    if (kp >= a.ring_bytes) kp -= a.ring_bytes;
    r.kp0 = kp;
    const bool head = (al - r.band * a.rows) == 0 && r.be_lo == 0;
    r.fast = r.be_lo + tv <= side && !head;
    return r;
  };
  const uint32_t nstages = (side + kDecStageRows - 1) / kDecStageRows;
  auto fill_info = [&](uint32_t st, uint32_t r) {  // r < kDecStageRows
    const uint32_t al = st * kDecStageRows + r;
    uint4 e = make_uint4(0, 0, 0, 0);
    if (al < side) {
      const Run q = run_of(al);
      e = make_uint4(q.P0, uint32_t(q.kp0), uint32_t(q.kp0 >> 32),
                     q.band | (q.fast ? 0x80000000u : 0u));
    }
    rinfo[(st % 3u) * kDecStageRows + r] = e;
  };
  const uint32_t cps = tid & 7u, cpr = tid >> 3;  // chunk, row (+64 i) of a stage
  auto issue_stage = [&](uint32_t st) {
    const uint32_t dst0 = win_base + (st & 1u) * kDecStageBytes;
    const uint4* info = rinfo + (st % 3u) * kDecStageRows;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t r = cpr + 64u * i;
      const uint4 e = info[r];
      const uint32_t dst = dst0 + r * kDecWin + 16u * (cps ^ (r & 7u));
      bool need = false;
      const uint8_t* src = a.src;
      if (e.w >> 31) {  // fast run (implies a row inside the frame)
        if (cps < 4) {
          const uint32_t base = (e.x - 1) & ~15u;  // fast runs have P0 >= 1
          need = base + 16u * cps < e.x + 3u * tv;
          if (need) src = a.src + base + 16u * cps;
        } else {
          const uint32_t c = cps - 4;
          const uint64_t kp0 = (uint64_t(e.z) << 32) | e.y;
          uint64_t kp = (kp0 & ~uint64_t(15)) + 16u * c;
          if (kp >= a.ring_bytes) kp -= a.ring_bytes;
          need = 16u * c < (e.y & 15u) + 3u * tv;
          if (need) src = a.ring + uint64_t(e.w & 0x7FFFFFFFu) * a.ring_bytes + kp;
        }
      }
      if (need && cps < 4) CVE_CHECK(within(src, 16, a.src, a.frame_bytes));
      if (need && cps >= 4)
        CVE_CHECK(within(src, 16, a.ring + uint64_t(e.w & 0x7FFFFFFFu) * a.ring_bytes,
                         a.ring_bytes));
      if (cps >= 4)
        cp_async16_ks(dst, src, need, ks_policy());
      else
        cp_async16(dst, src, need);
    }
    cp_async_commit();
  };
  if (tid < kDecStageRows)
    fill_info(0, tid);
  else if (nstages > 1)
    fill_info(1, tid - kDecStageRows);
  __syncthreads();
  issue_stage(0);
  if (nstages > 1) issue_stage(1);

  auto put = [&](uint32_t m, uint32_t q0, uint32_t pix) {
    uint32_t o = q0 + m;
    o -= o >= side ? side : 0u;
    const uint32_t sl = (tv - 1u - m) * side + o;
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots_base + 4u * slot_word(sl)), "r"(pix));
  };
  auto ks_at = [&](uint32_t band, uint32_t j) {  // keystream byte j of the round
    uint64_t kp = a.pos + j;
    if (kp >= a.ring_bytes) kp -= a.ring_bytes;
    CVE_CHECK(band < a.n && kp < a.ring_bytes);
    return uint32_t(__ldg(a.ring + uint64_t(band) * a.ring_bytes + kp));
  };
  // pixel m of source row al's run, byte by byte from global
  auto slow_pixel = [&](uint32_t al, const Run& q, uint32_t m) {
    const uint32_t nb = q.band + 1 == a.n ? 0 : q.band + 1;
    uint32_t be = q.be_lo + m;
    be -= be >= side ? side : 0u;
    const uint32_t P = (al * side + be) * 3u;
    uint32_t pix = 0;
#pragma unroll
    for (uint32_t ch = 0; ch < 3; ++ch) {
      const uint32_t j = P + ch - q.band * region;
      const uint32_t b = ks_at(q.band, j);
      uint32_t prev;
      if (j == 0) {  // band head: the next band's recovered last byte
        const uint32_t L = (nb + 1) * region - 1;
        const uint32_t bl = ks_at(nb, region - 1);
        prev = (bl ^ __ldg(a.src + L) ^ __ldg(a.src + L - 1)) - bl;
      } else {
        prev = __ldg(a.src + P + ch - 1);
      }
      CVE_CHECK(P + ch < a.frame_bytes && (j == 0 || P + ch >= 1));
      pix |= (((b ^ __ldg(a.src + P + ch) ^ prev) - b) & 0xFFu) << (8 * ch);
    }
    return pix;
  };

  for (uint32_t st = 0; st < nstages; ++st) {
    if (st + 1 < nstages)
      cp_async_wait<1>();
    else
      cp_async_wait<0>();
    __syncthreads();
    const uint32_t al = st * kDecStageRows + tid;
    if (tid >= kDecStageRows) {  // idle during the repack: run info two stages ahead
      if (st + 2 < nstages) fill_info(st + 2, tid - kDecStageRows);
    } else if (al < side) {
      const uint4 e = rinfo[(st % 3u) * kDecStageRows + tid];
      int q0i = int(al) - int(a0) - int(tv) + 1;  // in (-side, side)
      q0i += q0i < 0 ? int(side) : 0;
      const uint32_t q0 = uint32_t(q0i);
      if (e.w >> 31) {
        struct {
          uint32_t P0;
          uint64_t kp0;
        } q{e.x, (uint64_t(e.z) << 32) | e.y};
        const uint32_t w = win_base + (st & 1u) * kDecStageBytes + tid * kDecWin;
        uint32_t V[16], R[12], K[12];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(V[4 * c]), "=r"(V[4 * c + 1]), "=r"(V[4 * c + 2]), "=r"(V[4 * c + 3])
                       : "r"(w + 16u * (uint32_t(c) ^ (tid & 7u))));
        realign12(V, (q.P0 - 1) & 15u, R);  // R byte 0 = c[P0-1], then c[P0..]
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(V[4 * c]), "=r"(V[4 * c + 1]), "=r"(V[4 * c + 2]), "=r"(V[4 * c + 3])
                       : "r"(w + 16u * (uint32_t(c + 4) ^ (tid & 7u))));
        realign12(V, uint32_t(q.kp0 & 15u), K);
        uint32_t D[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          const uint32_t cur = i < 11 ? __funnelshift_r(R[i], R[i + 1], 8) : (R[11] >> 8);
          D[i] = sub_bytes(K[i] ^ cur ^ R[i], K[i]);
        }
#pragma unroll
        for (int m = 0; m < int(kMaxChunkRows); ++m) {
          if (uint32_t(m) >= tv) break;
          const int j = (3 * m) >> 2, sh = ((3 * m) & 3) * 8;
          put(m, q0, sh <= 8 ? (D[j] >> sh) : __funnelshift_r(D[j], D[j + 1], sh));
        }
      } else {  // band head or wrapping run: deferred (inline if the list is full)
        const uint32_t i = atomicAdd(&dcount, 1u);
        if (i < kDecDefer) {
          dlist[i] = al;
        } else {
          const Run q = run_of(al);
          for (uint32_t m = 0; m < tv; ++m) put(m, q0, slow_pixel(al, q, m));
        }
      }
    }
    if (st + 2 < nstages) {
      __syncthreads();
      issue_stage(st + 2);
    }
  }
  __syncthreads();
  {  // deferred rows: one thread per pixel
    const uint32_t nd = min(dcount, kDecDefer);
    for (uint32_t it = tid; it < nd * tv; it += kSlotThreads) {
      const uint32_t al = dlist[it / tv], m = it % tv;
      const Run q = run_of(al);
      int q0i = int(al) - int(a0) - int(tv) + 1;
      q0i += q0i < 0 ? int(side) : 0;
      put(m, uint32_t(q0i), slow_pixel(al, q, m));
    }
  }
  __syncthreads();

  // Output: the tile = rows a0 .. a0+tv-1, contiguous in the frame.
  const uint32_t G = (tv * side) >> 4;
  uint4* out4 = reinterpret_cast<uint4*>(a.dst + uint64_t(a0) * side * 3);
  for (uint32_t g = tid; g < G; g += kSlotThreads) {
    const uint4* q = smem + 4 * g;
    const uint32_t sw = (g >> 1) & 3u;
    uint32_t y[12];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = q[c ^ sw];
      y[3 * c] = __byte_perm(v.x, v.y, 0x4210);
      y[3 * c + 1] = __byte_perm(v.y, v.z, 0x5421);
      y[3 * c + 2] = __byte_perm(v.z, v.w, 0x6542);
    }
    CVE_CHECK(within(out4 + 3 * g, 48, a.dst, a.frame_bytes));
    out4[3 * g] = make_uint4(y[0], y[1], y[2], y[3]);
    out4[3 * g + 1] = make_uint4(y[4], y[5], y[6], y[7]);
    out4[3 * g + 2] = make_uint4(y[8], y[9], y[10], y[11]);
  }
}

// ---------------------------------------------------------------------------
// K3t: the inverse round on 2-D output tiles (side % 16 == 0, 16-byte
// aligned frames and keystream) -- the production decrypt round.
//
// Output tile = rows a0 .. a0+tv-1 x columns o0 .. o0+wv-1 (tv <= 15,
// wv <= W, W % 16 == 0).  Output pixel (a0+i, o0+j) is cipher pixel
// (al, be) with al = (a0 + o0 + i + j) mod side, be = (o0 + j + shift[al])
// mod side (inverse_confuse_rows, engine.cpp:49-64), inverse-diffused
// elementwise from the cipher byte, the byte before it and the keystream
// byte (engine.hpp:36-38).  The pixels with i + j = s all come from cipher
// row al_s = (a0 + o0 + s) mod side, at the consecutive columns of
// j in [max(0, s-tv+1), min(wv-1, s)]: the tile reads tv + wv - 1 runs of
// <= tv pixels.  One staging phase: 64-byte cipher and keystream windows of
// every run by cp.async, thread = run realigns, inverse-diffuses four bytes
// at a time and stores its pixels as 32-bit slots of the tile; runs through
// a band head (which needs the next band's recovered last byte, engine.cpp:
// 271-276) or wrapping past the row end go pixel by pixel.  Then the tile's
// tv row segments of 3 wv bytes are written with 16-byte stores.
//
// Unlike K3s (full-width tiles, 184-215 KB of shared memory, one CTA per
// SM), a tile needs ~25 KB, so ~8 CTAs share an SM and hide each other's
// staging latency.
#ifndef TILE_THREADS
#define TILE_THREADS 160
#endif
#ifndef TILE_TMA
#define TILE_TMA 0  // experiment: 1-D TMA bulk copies for K3t's windows
#endif
constexpr uint32_t kTileThreads = TILE_THREADS;  // >= the runs of the largest tile
constexpr uint32_t kTileMaxT = 15;
constexpr uint32_t kTileMaxW = 128;
constexpr uint32_t kTileMaxRuns = kTileMaxT + kTileMaxW - 1;
static_assert(kTileMaxRuns <= kTileThreads, "thread = run");
constexpr uint32_t kTileDefer = 64;

struct TileArgs {
  const uint8_t* src;
  uint8_t* dst;
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;
  const int32_t* shift;
  uint32_t side, n, rows, T, W;
  uint32_t region;
  FastDiv div_rows;
  uint64_t frame_bytes;  // bounds checks only
};

__global__ void __launch_bounds__(kTileThreads)
    k_decrypt_round_tiles(const TileArgs a) {
  extern __shared__ uint4 smem[];
  __shared__ uint32_t dlist[kTileDefer];
  __shared__ uint32_t dcount;
  const uint32_t tid = threadIdx.x, side = a.side, W = a.W;
  const uint32_t a0 = blockIdx.y * a.T, o0 = blockIdx.x * W;
  const uint32_t tv = min(a.T, side - a0), wv = min(W, side - o0);
  const uint32_t nruns = tv + wv - 1;
  const uint32_t slots_base = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t win_base = slots_base + a.T * W * 4u;
  const uint32_t region = a.region;
  uint32_t diag = a0 + o0;  // al of run 0
  diag -= diag >= side ? side : 0u;

  // geometry of run s: cipher row al, first j, length, first column
  struct Run {
    uint32_t al, jlo, len, be_lo, band;
  };
  auto run_of = [&](uint32_t s) {
    Run r;
    r.al = diag + s;
    r.al -= r.al >= side ? side : 0u;
    r.jlo = s + 1 > tv ? s + 1 - tv : 0u;
    r.len = min(wv - 1, s) - r.jlo + 1;
    uint32_t b = o0 + r.jlo + uint32_t(a.shift[r.al]);  // < 3 side
    b -= b >= side ? side : 0u;
    b -= b >= side ? side : 0u;
    r.be_lo = b;
    r.band = fdiv(r.al, a.div_rows);
    return r;
  };
  // slot of tile pixel (i, j); granules of 16 slots swizzled as in K2s/K3s
  auto put = [&](uint32_t i, uint32_t j, uint32_t pix) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(slots_base + 4u * slot_word(i * W + j)),
                 "r"(pix));
  };
  auto ks_at = [&](uint32_t band, uint32_t j) {  // keystream byte j of this round
    uint64_t kp = a.pos + j;
    if (kp >= a.ring_bytes) kp -= a.ring_bytes;
    CVE_CHECK(band < a.n && kp < a.ring_bytes);
    return uint32_t(__ldg(a.ring + uint64_t(band) * a.ring_bytes + kp));
  };
  // pixel m of run r, byte by byte from global
  auto slow_pixel = [&](const Run& r, uint32_t m) {
    const uint32_t nb = r.band + 1 == a.n ? 0 : r.band + 1;
    uint32_t be = r.be_lo + m;
    be -= be >= side ? side : 0u;
    const uint32_t P = (r.al * side + be) * 3u;
    uint32_t pix = 0;
#pragma unroll
    for (uint32_t ch = 0; ch < 3; ++ch) {
      const uint32_t j = P + ch - r.band * region;
      const uint32_t b = ks_at(r.band, j);
      uint32_t prev;
      if (j == 0) {  // band head: the next band's recovered last byte
        const uint32_t L = (nb + 1) * region - 1;
        const uint32_t bl = ks_at(nb, region - 1);
        prev = (bl ^ __ldg(a.src + L) ^ __ldg(a.src + L - 1)) - bl;
      } else {
        prev = __ldg(a.src + P + ch - 1);
      }
      CVE_CHECK(P + ch < a.frame_bytes && (j == 0 || P + ch >= 1));
      pix |= (((b ^ __ldg(a.src + P + ch) ^ prev) - b) & 0xFFu) << (8 * ch);
    }
    return pix;
  };

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if TILE_TMA
  __shared__ uint64_t tbar;
  const uint32_t mbar = uint32_t(__cvta_generic_to_shared(&tbar));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(kTileThreads));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
#endif
  if (tid == 0) dcount = 0;
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // previous round / shift table done
#if TILE_TMA
  bool arrived = false;
#endif
  if (tid < nruns) {
    // thread = run: its own windows (cp.async), realigned once they land
    const Run r = run_of(tid);
    const uint32_t P0 = (r.al * side + r.be_lo) * 3u;
    uint64_t kp = a.pos + (P0 - r.band * region);
    if (kp >= a.ring_bytes) kp -= a.ring_bytes;
    const bool head = r.al == r.band * a.rows && r.be_lo == 0;
    const bool fast = r.be_lo + r.len <= side && !head;
    const uint32_t w = win_base + tid * (TILE_TMA ? 144u : 128u);
    if (fast) {
      const uint32_t cb = (P0 - 1) & ~15u;  // fast runs have P0 >= 1
      const uint32_t nc = (P0 + 3u * r.len - cb + 15u) >> 4;  // bytes P0-1 .. P0+3len-1
      const uint8_t* ks = a.ring + uint64_t(r.band) * a.ring_bytes;
      const uint64_t kb = kp & ~uint64_t(15);
      const uint32_t nk = (uint32_t(kp & 15u) + 3u * r.len + 15u) >> 4;
      const uint64_t kpol = ks_policy();
#if TILE_TMA
      // experiment: 1-D TMA bulk copies of the needed chunks (windows
      // unswizzled, 144-byte stride), completion on the CTA's mbarrier
      {
        const uint64_t kroom = a.ring_bytes - kb;
        const uint32_t kfirst = kroom < 16u * nk ? uint32_t(kroom) : 16u * nk;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                     "r"(16u * nc + 16u * nk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(w), "l"(a.src + cb), "r"(16u * nc), "r"(mbar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(w + 64u), "l"(ks + kb), "r"(kfirst), "r"(mbar) : "memory");
        if (kfirst < 16u * nk)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(w + 64u + kfirst), "l"(ks), "r"(16u * nk - kfirst), "r"(mbar) : "memory");
        arrived = true;
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
              : "=r"(done) : "r"(mbar) : "memory");
      }
#else
#pragma unroll
      for (uint32_t c = 0; c < 4; ++c) {
        if (c < nc) CVE_CHECK(within(a.src + cb + 16u * c, 16, a.src, a.frame_bytes));
        cp_async16(w + 16u * (c ^ (tid & 7u)), a.src + cb + 16u * c, c < nc);
      }
#pragma unroll
      for (uint32_t c = 0; c < 4; ++c) {
        uint64_t q = kb + 16u * c;
        q -= q >= a.ring_bytes ? a.ring_bytes : 0;
        if (c < nk) CVE_CHECK(within(ks + q, 16, ks, a.ring_bytes));
        cp_async16_ks(w + 16u * ((c + 4) ^ (tid & 7u)), ks + q, c < nk, kpol);
      }
      cp_async_commit();
      cp_async_wait<0>();  // this thread's own copies: no CTA barrier needed
#endif
      uint32_t V[16], R[12], K[12];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(V[4 * c]), "=r"(V[4 * c + 1]), "=r"(V[4 * c + 2]), "=r"(V[4 * c + 3])
                     : "r"(w + 16u * (uint32_t(c) ^ (TILE_TMA ? 0u : tid & 7u))));
      realign12(V, (P0 - 1) & 15u, R);  // R byte 0 = c[P0-1], then c[P0..]
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(V[4 * c]), "=r"(V[4 * c + 1]), "=r"(V[4 * c + 2]), "=r"(V[4 * c + 3])
                     : "r"(w + 16u * (uint32_t(c + 4) ^ (TILE_TMA ? 0u : tid & 7u))));
      realign12(V, uint32_t(kp & 15u), K);
      uint32_t D[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const uint32_t cur = i < 11 ? __funnelshift_r(R[i], R[i + 1], 8) : (R[11] >> 8);
        D[i] = sub_bytes(K[i] ^ cur ^ R[i], K[i]);
      }
#pragma unroll
      for (int m = 0; m < int(kTileMaxT); ++m) {
        if (uint32_t(m) >= r.len) break;
        const int j = (3 * m) >> 2, sh = ((3 * m) & 3) * 8;
        put(tid - r.jlo - uint32_t(m), r.jlo + uint32_t(m),
            sh <= 8 ? (D[j] >> sh) : __funnelshift_r(D[j], D[j + 1], sh));
      }
    } else {  // band head or wrapping run: deferred (inline if the list is full)
      const uint32_t i = atomicAdd(&dcount, 1u);
      if (i < kTileDefer) {
        dlist[i] = tid;
      } else {
        for (uint32_t m = 0; m < r.len; ++m) put(tid - r.jlo - m, r.jlo + m, slow_pixel(r, m));
      }
    }
  }
#if TILE_TMA
  if (!arrived) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
#endif
  __syncthreads();
  {  // deferred runs: one thread per pixel
    const uint32_t nd = min(dcount, kTileDefer);
    for (uint32_t it = tid; it < nd * kTileMaxT; it += kTileThreads) {
      const uint32_t s = dlist[it / kTileMaxT], m = it % kTileMaxT;
      const Run r = run_of(s);
      if (m < r.len) put(s - r.jlo - m, r.jlo + m, slow_pixel(r, m));
    }
  }
  __syncthreads();
  // Output: row a0+i, columns o0 .. o0+wv-1 = 3 wv contiguous bytes, 16-byte
  // aligned (o0, wv multiples of 16): 48-byte granules of 16 slots.
  const uint32_t gpr = wv >> 4;  // granules per row
  for (uint32_t q = tid; q < tv * gpr; q += kTileThreads) {
    const uint32_t i = q / gpr, g = q - i * gpr;
    const uint32_t u = (i * W >> 4) + g;  // granule index in the slot array
    const uint4* sl = smem + 4 * u;
    const uint32_t sw = (u >> 1) & 3u;
    uint32_t y[12];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 v = sl[c ^ sw];
      y[3 * c] = __byte_perm(v.x, v.y, 0x4210);
      y[3 * c + 1] = __byte_perm(v.y, v.z, 0x5421);
      y[3 * c + 2] = __byte_perm(v.z, v.w, 0x6542);
    }
    uint4* out4 = reinterpret_cast<uint4*>(a.dst + (uint64_t(a0 + i) * side + o0 + 16u * g) * 3u);
    CVE_CHECK(within(out4, 48, a.dst, a.frame_bytes));
    out4[0] = make_uint4(y[0], y[1], y[2], y[3]);
    out4[1] = make_uint4(y[4], y[5], y[6], y[7]);
    out4[2] = make_uint4(y[8], y[9], y[10], y[11]);
  }
}

// ---------------------------------------------------------------------------
// K6: ALL rounds of one frame in one thread-block cluster (frames up to
// ~768^2).  CTA q of the CL-CTA cluster owns the R = side/CL
// destination rows al0 = qR .. qR+R-1 -- whole bands (R % rows == 0), so the
// diffusion scan never crosses a CTA -- as a packed slab of R*side*3 bytes
// in each of two shared-memory buffers.
//   load:  one TMA bulk copy (cp.async.bulk, mbarrier completion) of the
//          CTA's slab of the plaintext into buffer 0;
//   round: gather y = confuse(x) from the cluster's source buffers through
//          distributed shared memory (every source row sr holds the CTA's
//          run of R pixels at columns (al0 - sr) mod side ...: 16-pixel
//          pieces, a 64-byte window each) into the local other buffer; then
//          the XOR-prefix diffusion of each local band in place, with the
//          keystream of round k from the ring and s_d gathered from the
//          round's source buffers (engine.cpp:237); one cluster barrier;
//   store: one TMA bulk copy of the final slab to the frame.
// The frame is read from and written to HBM once, with no kernel boundary
// between rounds (reference: the r-round loop of engine.cpp:207-250).
#ifndef CL_THREADS
#define CL_THREADS 512
#endif
constexpr uint32_t kClThreads = CL_THREADS;
constexpr int kClBatch = 4;  // gather pieces per thread with loads in flight together
constexpr uint32_t kClMax = 16;  // CTAs per cluster (non-portable above 8)
constexpr size_t kClSmemMax = 227 * 1024;

struct ClusterArgs {
  const uint8_t* src;  // plaintext (global)
  uint8_t* dst;        // ciphertext (global; may alias src)
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;  // stream position of round 0 (round k: pos + k * region)
  const int32_t* shift;
  uint32_t side, n, rows, R, rounds;
  uint32_t region, slab;  // slab = R * side * 3
  uint32_t cks_off;       // shared-memory offset of the c_k table (after 2 slabs)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(kClThreads, 1)
    k_encrypt_frame_cluster(const ClusterArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t q = cluster.block_rank();
  const uint32_t tid = threadIdx.x, side = a.side, R = a.R;
  const uint32_t al0 = q * R;
  uint8_t* const buf0 = sm;
  uint32_t* const cks = reinterpret_cast<uint32_t*>(sm + a.cks_off);  // R entries
  uint32_t* const wsum = cks + ((R + 3u) & ~3u);                       // 64 words
  uint32_t* const bseed = wsum + 64;                                   // 8 words
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(bseed + 8);

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // shift table and frame ready
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
                 "r"(a.slab)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(buf0)),
        "l"(a.src + uint64_t(q) * a.slab), "r"(a.slab), "r"(smem_u32(mbar))
        : "memory");
  }
  for (uint32_t k = tid; k < R; k += kClThreads) {
    uint32_t c = k + uint32_t(a.shift[al0 + k]);
    cks[k] = c >= side ? c - side : c;
  }
  {  // wait for the slab (phase 0)
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(mbar))
          : "memory");
  }
  cluster.sync();  // every slab is loaded before any CTA gathers from it

  const uint32_t np = (R + 15u) >> 4;  // 16-pixel pieces of a run
  const uint32_t nbl = R / a.rows;     // local bands
  const uint32_t ngr = a.region / 48u; // 48-byte granules per band
  uint32_t phase = 0;                  // block_xor_scan calls (alternating workspace)
  for (uint32_t rk = 0; rk < a.rounds; ++rk) {
    const uint8_t* S = sm + (rk & 1u) * a.slab;  // this round's source (every CTA)
    uint8_t* Y = sm + ((rk & 1u) ^ 1u) * a.slab;  // local destination
    // 1. Gather: piece (sr, p) = pixels k in [16p, 16p+16) of source row sr's
    //    run, source columns o0 + k, o0 = (al0 - sr) mod side; pixel k goes to
    //    local row k, column (o0 + c_k) mod side.
    // The windows of up to kClBatch pieces of the thread are loaded (remote
    // DSMEM, long latency) before any is used, then realigned and stored.
    struct Piece {
      uint32_t o0, k0, len, b0;
      bool fast, live;
      const uint8_t* rs;
      uint32_t rowb;
    };
    auto piece_of = [&](uint32_t w) {
      Piece pc;
      pc.live = w < side * np;
      const uint32_t sr = pc.live ? w / np : 0u, p = pc.live ? w - sr * np : 0u;
      int oi = int(al0) - int(sr);
      oi += oi < 0 ? int(side) : 0;
      pc.o0 = uint32_t(oi);
      pc.k0 = 16u * p;
      pc.len = min(16u, R - pc.k0);
      const uint32_t qs = sr / R;  // owner of source row sr
      pc.rs = cluster.map_shared_rank(S, qs);
      pc.rowb = (sr - qs * R) * side * 3u;
      pc.fast = pc.live && pc.o0 + pc.k0 + pc.len <= side;
      pc.b0 = pc.rowb + (pc.o0 + pc.k0) * 3u;
      return pc;
    };
    const uint32_t npieces = side * np;
    for (uint32_t w0 = 0; w0 < npieces; w0 += kClBatch * kClThreads) {
      Piece pc[kClBatch];
      uint4 V4[kClBatch][4];
#pragma unroll
      for (int b = 0; b < kClBatch; ++b) {
        pc[b] = piece_of(w0 + uint32_t(b) * kClThreads + tid);
        const uint4* win = reinterpret_cast<const uint4*>(pc[b].rs + (pc[b].b0 & ~15u));
        CVE_CHECK(!pc[b].fast ||
                  (pc[b].b0 & ~15u) + 16u * (((pc[b].b0 & 15u) + 3u * pc[b].len + 15u) / 16u) <= a.slab);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          V4[b][c] = (pc[b].fast && 16u * c < (pc[b].b0 & 15u) + 3u * pc[b].len)
                         ? win[c] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int b = 0; b < kClBatch; ++b) {
        const Piece& q = pc[b];
        if (q.fast) {
          uint32_t V[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            V[4 * c] = V4[b][c].x;
            V[4 * c + 1] = V4[b][c].y;
            V[4 * c + 2] = V4[b][c].z;
            V[4 * c + 3] = V4[b][c].w;
          }
          uint32_t A[12];
          realign12(V, q.b0 & 15u, A);
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            if (uint32_t(m) >= q.len) break;
            const int j = (3 * m) >> 2, sh = ((3 * m) & 3) * 8;
            const uint32_t pix = sh <= 8 ? (A[j] >> sh) : __funnelshift_r(A[j], A[j + 1], sh);
            const uint32_t k = q.k0 + uint32_t(m);
            uint32_t col = q.o0 + cks[k];
            col -= col >= side ? side : 0u;
            uint8_t* d = Y + (k * side + col) * 3u;
            CVE_CHECK(k < R && col < side);
            d[0] = uint8_t(pix);
            d[1] = uint8_t(pix >> 8);
            d[2] = uint8_t(pix >> 16);
          }
        } else if (q.live) {  // the run wraps past the row end: pixel by pixel
          for (uint32_t m = 0; m < q.len; ++m) {
            const uint32_t k = q.k0 + m;
            uint32_t o = q.o0 + k;
            o -= o >= side ? side : 0u;
            const uint8_t* sp = q.rs + q.rowb + o * 3u;
            CVE_CHECK(k < R && q.rowb + o * 3u + 3u <= a.slab);
            uint32_t col = q.o0 + cks[k];
            col -= col >= side ? side : 0u;
            uint8_t* d = Y + (k * side + col) * 3u;
            d[0] = sp[0];
            d[1] = sp[1];
            d[2] = sp[2];
          }
        }
      }
    }
    // s_d of each local band: the post-confusion byte ((band+1) mod n + 1) *
    // region - 1 = pixel (last row of the next band, column side-1), channel
    // 2, gathered straight from this round's source buffers.
    if (tid < nbl) {
      const uint32_t band = al0 / a.rows + tid;
      const uint32_t nb = band + 1 == a.n ? 0 : band + 1;
      const uint32_t al = nb * a.rows + a.rows - 1;
      int o = int(side - 1) - a.shift[al];
      o += o < 0 ? int(side) : 0;
      int sr = int(al) - o;
      sr += sr < 0 ? int(side) : 0;
      const uint32_t qs = uint32_t(sr) / R;
      const uint8_t* rs = cluster.map_shared_rank(S, qs);
      bseed[tid] = rs[((uint32_t(sr) - qs * R) * side + uint32_t(o)) * 3u + 2u];
    }
    __syncthreads();  // Y complete, seeds set
    // 2. Diffusion of each local band, in place on Y (one granule of 48 bytes
    //    per thread per super-tile, one CTA-wide XOR scan per super-tile).
    uint64_t kbase = a.pos + uint64_t(rk) * a.region;
    kbase %= a.ring_bytes;
    // keystream granule g of local band lb (48-byte granules never straddle
    // the ring end: positions and ring size are multiples of 48)
    auto load_kw = [&](uint32_t lb, uint32_t g, uint4 (&kv)[3]) {
      const uint8_t* ks = a.ring + uint64_t(al0 / a.rows + lb) * a.ring_bytes;
      uint64_t kp = kbase + 48ull * g;
      kp -= kp >= a.ring_bytes ? a.ring_bytes : 0;
      if (g < ngr) CVE_CHECK(within(ks + kp, 48, ks, a.ring_bytes));
#pragma unroll
      for (int i = 0; i < 3; ++i)
        kv[i] = g < ngr ? ld_stream(ks + kp + 16 * i) : make_uint4(0, 0, 0, 0);
    };
    uint4 kv[3];
    load_kw(0, tid, kv);
    for (uint32_t lb = 0; lb < nbl; ++lb) {
      uint32_t carry = bseed[lb];
      uint8_t* yb = Y + lb * a.region;
      for (uint32_t st = 0; st * kClThreads < ngr; ++st) {
        const uint32_t g = st * kClThreads + tid;
        // next super-tile's keystream (or the next band's first) in flight
        uint4 kn[3];
        const bool last = (st + 1) * kClThreads >= ngr;
        if (!last)
          load_kw(lb, g + kClThreads, kn);
        else if (lb + 1 < nbl)
          load_kw(lb + 1, tid, kn);
        uint32_t yv[12];
        const uint32_t kw[12] = {kv[0].x, kv[0].y, kv[0].z, kv[0].w, kv[1].x, kv[1].y,
                                 kv[1].z, kv[1].w, kv[2].x, kv[2].y, kv[2].z, kv[2].w};
        if (g < ngr) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const uint4 v = reinterpret_cast<const uint4*>(yb + 48u * g)[i];
            yv[4 * i] = v.x;
            yv[4 * i + 1] = v.y;
            yv[4 * i + 2] = v.z;
            yv[4 * i + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 12; ++i) yv[i] = 0;
        }
        uint32_t res[12], E = 0;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          const uint32_t t = t_prefix4(yv[i], kw[i]);
          res[i] = t ^ E;
          E ^= __byte_perm(t, 0, 0x3333);
        }
        uint32_t total;
        const uint32_t excl = block_xor_scan(E & 0xFFu, wsum, phase++, total) ^ carry;
        if (g < ngr) {
          const uint32_t m = excl * 0x01010101u;
          uint4* o4 = reinterpret_cast<uint4*>(yb + 48u * g);
          o4[0] = make_uint4(res[0] ^ m, res[1] ^ m, res[2] ^ m, res[3] ^ m);
          o4[1] = make_uint4(res[4] ^ m, res[5] ^ m, res[6] ^ m, res[7] ^ m);
          o4[2] = make_uint4(res[8] ^ m, res[9] ^ m, res[10] ^ m, res[11] ^ m);
        }
        carry ^= total;
#pragma unroll
        for (int i = 0; i < 3; ++i) kv[i] = kn[i];
      }
    }
    cluster.sync();  // Y complete everywhere; every read of this round's S done
  }
  // 3. Store the final slab with one TMA bulk copy.
  const uint8_t* fin = sm + (a.rounds & 1u) * a.slab;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     a.dst + uint64_t(q) * a.slab),
                 "r"(smem_u32(fin)), "r"(a.slab)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---------------------------------------------------------------------------
// Generic forward round for geometries whose band chunks do not fit one
// cluster's shared memory: gather -> chunk aggregates -> band prefixes ->
// chunk scans, through global scratch.
constexpr uint32_t kGenChunk = 4096;  // bytes per chunk (256 threads x 16 B)

__global__ void k_gather(const uint8_t* __restrict__ src, uint8_t* __restrict__ y,
                         const int32_t* __restrict__ shift, uint32_t side) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= uint64_t(side) * side) return;
  const uint32_t al = uint32_t(q / side), be = uint32_t(q - uint64_t(al) * side);
  int o = int(be) - shift[al];
  if (o < 0) o += side;
  int sr = int(al) - o;
  if (sr < 0) sr += side;
  const uint8_t* sp = src + (uint64_t(sr) * side + uint32_t(o)) * 3;
  y[q * 3] = sp[0];
  y[q * 3 + 1] = sp[1];
  y[q * 3 + 2] = sp[2];
}

struct GenArgs {
  const uint8_t* y;
  uint8_t* dst;
  const uint8_t* ring;
  uint64_t ring_bytes, pos, region;
  uint32_t n, nch;
  uint32_t* agg;  // n * nch
};

__device__ __forceinline__ void gen_chunk_values(const GenArgs& a, uint32_t band,
                                                 uint32_t ch, uint64_t& lo,
                                                 uint64_t& hi, uint32_t& agg) {
  uint32_t yw[4] = {0, 0, 0, 0}, kw[4] = {0, 0, 0, 0};
  const uint64_t j = uint64_t(ch) * kGenChunk + 16ull * threadIdx.x;
  for (uint32_t i = 0; i < 16; ++i) {
    if (j + i < a.region) {
      yw[i >> 2] |= uint32_t(a.y[uint64_t(band) * a.region + j + i]) << (8 * (i & 3));
      uint64_t kp = (a.pos + j + i) % a.ring_bytes;
      kw[i >> 2] |= uint32_t(a.ring[uint64_t(band) * a.ring_bytes + kp]) << (8 * (i & 3));
    }
  }
  lo = t_prefix8(yw[0], yw[1], kw[0], kw[1]);
  hi = t_prefix8(yw[2], yw[3], kw[2], kw[3]);
  hi ^= (lo >> 56) * kBcast;
  agg = uint32_t(hi >> 56);
}

__global__ void __launch_bounds__(256) k_gen_aggregate(const GenArgs a) {
  __shared__ uint32_t wsum[64];
  const uint32_t band = blockIdx.y, ch = blockIdx.x;
  uint64_t lo, hi;
  uint32_t agg, total;
  gen_chunk_values(a, band, ch, lo, hi, agg);
  block_xor_scan(agg, wsum, 0, total);
  if (threadIdx.x == 0) a.agg[band * a.nch + ch] = total;
}

__global__ void k_gen_prefix(const GenArgs a) {
  const uint32_t band = blockIdx.x * blockDim.x + threadIdx.x;
  if (band >= a.n) return;
  const uint32_t nb = band + 1 == a.n ? 0 : band + 1;
  uint32_t p = a.y[(uint64_t(nb) + 1) * a.region - 1];
  for (uint32_t c = 0; c < a.nch; ++c) {
    const uint32_t v = a.agg[band * a.nch + c];
    a.agg[band * a.nch + c] = p;  // exclusive prefix incl. s_d
    p ^= v;
  }
}

__global__ void __launch_bounds__(256) k_gen_scan(const GenArgs a) {
  __shared__ uint32_t wsum[64];
  const uint32_t band = blockIdx.y, ch = blockIdx.x;
  uint64_t lo, hi;
  uint32_t agg, total;
  gen_chunk_values(a, band, ch, lo, hi, agg);
  const uint32_t excl = block_xor_scan(agg, wsum, 0, total) ^ a.agg[band * a.nch + ch];
  const uint64_t m = uint64_t(excl) * kBcast;
  lo ^= m;
  hi ^= m;
  const uint64_t j = uint64_t(ch) * kGenChunk + 16ull * threadIdx.x;
  uint8_t* out = a.dst + uint64_t(band) * a.region;
  for (uint32_t i = 0; i < 16; ++i)
    if (j + i < a.region) out[j + i] = uint8_t((i < 8 ? lo >> (8 * i) : hi >> (8 * (i - 8))));
}

__global__ void k_ring_move(const uint8_t* __restrict__ src, uint64_t sb,
                            uint8_t* __restrict__ dst, uint64_t db, uint64_t lo,
                            uint64_t hi, uint32_t workers) {
  const uint64_t span = hi - lo;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       i < span * workers; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t w = i / span, s = lo + (i - w * span);
    dst[w * db + s % db] = src[w * sb + s % sb];
  }
}

inline void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char msg[256];
    std::snprintf(msg, sizeof msg, "%s launch failed: %s", what,
                  cudaGetErrorString(e));
    throw Error(Errc::internal, msg);
  }
}

}  // namespace

void configure_cipher_kernels() {
  // once per device (Engine ctor): large dynamic smem and 16-CTA clusters
  for (auto k : {k_encrypt_round<true>, k_encrypt_round<false>}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBudget));
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaFuncSetAttribute(k_encrypt_round_slots, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(kSlotSmemMax));
  cudaFuncSetAttribute(k_encrypt_round_slots, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_decrypt_round_slots, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(kSlotSmemMax));
  cudaFuncSetAttribute(k_encrypt_frame_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(kClSmemMax));
  cudaFuncSetAttribute(k_encrypt_frame_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // K3t: ~26 KB tiles, 8 per SM need the whole carveout as shared memory
  cudaFuncSetAttribute(k_decrypt_round_tiles, cudaFuncAttributePreferredSharedMemoryCarveout,
                       int(cudaSharedmemCarveoutMaxShared));
  for (auto k : {k_decrypt_round<true>, k_decrypt_round<false>})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBudget));
}

void launch_shift_table(const double* sine, uint32_t seed, int32_t* shift,
                        uint32_t side, cudaStream_t s) {
  k_shift<<<(side + 255) / 256, 256, 0, s>>>(sine, seed, shift, side);
  check_launch("shift_table");
}

// Slot-staged plan: chunk rows cr | rows, cr <= 16, h = rows / cr <= 16 (one
// cluster); shared memory = 4 B of slots per chunk pixel + 2 stages of source
// windows.  Longer chunks mean longer contiguous source runs; take the
// largest cr with >= 64 CTAs per frame.
void plan_slots(const Geom& g, EncPlan& p) {
  p.slots = false;
  if (g.side % 16 || g.frame_bytes >= (uint64_t(1) << 32)) return;
  uint32_t forced = 0;
  if (const char* e = std::getenv("CVE_B200_ENC_CR")) forced = uint32_t(std::atoi(e));  // experiments only
  bool enough = false;
  for (uint32_t cr = 1; cr <= std::min(g.rows, kMaxChunkRows); ++cr) {
    if (g.rows % cr || g.rows / cr > 16) continue;
    const size_t smem = size_t(cr) * g.side * 4 + 2 * kStageBytes;
    if (smem > kSlotSmemMax) continue;
    if (forced && cr != forced) continue;
    const bool ok = uint64_t(g.n) * (g.rows / cr) >= 64;
    if (!ok && enough) continue;
    enough = enough || ok;
    p.slots = true;
    p.s_rows = cr;
    p.s_h = g.rows / cr;
    p.s_smem = smem;
  }
}

EncPlan plan_encrypt(const Geom& g) {
  // Chunks of a band: h | rows, h <= 16 (one cluster; > 8 is non-portable).
  // The staging loads runs of rows/h pixels from every source row, so long
  // runs (small h) cost fewer L1 wavefronts per byte: measured on B200 at
  // 1920^2 / n=64, h = 2/3/5/6 -> 27.0/31.1/34.5/35.3 us per round.  Take
  // the smallest h with <= 120 KB of shared memory and >= 64 CTAs per frame.
  const uint64_t row_bytes = uint64_t(g.side) * 3;
  auto make = [&](uint32_t h) {
    const uint64_t cb = uint64_t(g.rows / h) * row_bytes;
    const size_t smem = size_t(((cb + 15) & ~uint64_t(15)) + 4 * (g.rows / h));
    return EncPlan{smem <= kSmemBudget, g.rows / h, h, smem, false, 0, 0, 0};
  };
  EncPlan out{false, 0, 0, 0, false, 0, 0, 0};
  bool done = false;
  if (const char* e = std::getenv("CVE_B200_ENC_H")) {  // experiments only
    const uint32_t h = uint32_t(std::atoi(e));
    if (h >= 1 && h <= 16 && g.rows % h == 0 && make(h).fused) {
      out = make(h);
      done = true;
    }
  }
  for (uint32_t h = 1; h <= 16 && !done; ++h) {
    if (g.rows % h) continue;
    const EncPlan p = make(h);
    if (!p.fused) continue;
    out = p;  // largest feasible h so far
    if (p.smem <= 120 * 1024 && uint64_t(g.n) * h >= 64) done = true;
  }
  if (!std::getenv("CVE_B200_NO_SLOTS")) plan_slots(g, out);  // experiments only
  return out;
}

// K6 plan: the largest cluster (<= 16 CTAs) whose CTAs own whole bands
// (R = side / CL rows, R % rows == 0) and fit two packed slabs of R rows plus
// the c_k table in shared memory.  0: the frame does not fit one cluster.
uint32_t plan_cluster(const Geom& g, size_t& smem) {
  if (g.side % 16 || std::getenv("CVE_B200_NO_CLUSTER")) return 0;  // experiments only
  for (uint32_t cl = kClMax; cl >= 1; --cl) {
    if (g.side % cl) continue;
    const uint32_t R = g.side / cl;
    if (R % g.rows) continue;
    const size_t slab = size_t(R) * g.side * 3;
    const size_t need = 2 * slab + 4 * ((R + 3) & ~3u) + 4 * 64 + 4 * 8 + 16;
    if (need > kClSmemMax || R / g.rows > 8) continue;
    smem = need;
    return cl;
  }
  return 0;
}

bool launch_encrypt_frame(const Geom& g, uint8_t* buf, KsWindow ks, const int32_t* shift,
                          uint32_t rounds, cudaStream_t s, uint64_t* launches) {
  size_t smem = 0;
  const uint32_t cl = plan_cluster(g, smem);
  const bool aligned = ks.pos % 48 == 0 && ks.ring_bytes % 48 == 0 && g.region % 48 == 0 &&
                       ((reinterpret_cast<uintptr_t>(buf) | reinterpret_cast<uintptr_t>(ks.ring)) % 16 == 0);
  if (!cl || !aligned) return false;
  const uint32_t R = g.side / cl;
  ClusterArgs a{buf, buf, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n, g.rows, R,
                rounds, uint32_t(g.region), R * g.side * 3, 2 * R * g.side * 3};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = std::getenv("CVE_B200_NO_PDL") ? 1 : 2;  // experiments only
  cudaLaunchKernelEx(&cfg, k_encrypt_frame_cluster, a);
  check_launch("encrypt_frame_cluster");
  ++*launches;
  return true;
}

void launch_encrypt_round(const EncPlan& plan, const Geom& g,
                          const uint8_t* src, uint8_t* dst, KsWindow ks,
                          const int32_t* shift, uint8_t* scratch,
                          cudaStream_t s, uint64_t* launches) {
  const bool aligned = (g.side % 16 == 0) && (ks.pos % 16 == 0) &&
                       (ks.ring_bytes % 16 == 0) &&
                       ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                         reinterpret_cast<uintptr_t>(ks.ring)) % 16 == 0);
  if (plan.slots && aligned && ks.pos % 48 == 0 && ks.ring_bytes % 48 == 0) {
    EncArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n,
              g.rows, plan.s_rows, plan.s_h, g.region, make_div(plan.s_rows), g.frame_bytes};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.n * plan.s_h);
    cfg.blockDim = dim3(kSlotThreads);
    cfg.dynamicSmemBytes = plan.s_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = plan.s_h;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchAttribute attr2[2] = {attr[0], {}};
    if (!std::getenv("CVE_B200_NO_PDL")) {  // experiments only
      attr2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr2[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr2;
      cfg.numAttrs = 2;
    }
    cudaLaunchKernelEx(&cfg, k_encrypt_round_slots, a);
    check_launch("encrypt_round_slots");
    ++*launches;
    return;
  }
  if (plan.fused) {
    EncArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n,
              g.rows, plan.chunk_rows, plan.h, g.region, make_div(plan.chunk_rows),
              g.frame_bytes};
    const bool vec = aligned;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.n * plan.h);
    cfg.blockDim = dim3(kEncThreads);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = plan.h;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto kern = vec ? k_encrypt_round<true> : k_encrypt_round<false>;
    cudaLaunchKernelEx(&cfg, kern, a);
    check_launch("encrypt_round");
    ++*launches;
    return;
  }
  // generic path: scratch holds y (frame_bytes) followed by chunk aggregates
  launch_confuse_only(g, src, scratch, shift, s, launches);
  uint32_t* agg = reinterpret_cast<uint32_t*>(scratch + ((g.frame_bytes + 255) & ~uint64_t(255)));
  launch_diffuse_only(g, scratch, dst, ks, agg, s, launches);
}

// Confusion alone (confuse_rows, engine.cpp:32-47): dst = the permuted src.
void launch_confuse_only(const Geom& g, const uint8_t* src, uint8_t* dst, const int32_t* shift,
                         cudaStream_t s, uint64_t* launches) {
  const uint64_t pix = uint64_t(g.side) * g.side;
  k_gather<<<uint32_t((pix + 255) / 256), 256, 0, s>>>(src, dst, shift, g.side);
  check_launch("gather");
  ++*launches;
}

// Diffusion alone (diffuse_region per band, engine.cpp:232-244): dst = the
// band-wise chained rewrite of y with the round's keystream window; agg holds
// n * ceil(region / 4096) chunk aggregates.
void launch_diffuse_only(const Geom& g, const uint8_t* y, uint8_t* dst, KsWindow ks,
                         uint32_t* agg, cudaStream_t s, uint64_t* launches) {
  const uint32_t nch = uint32_t((g.region + kGenChunk - 1) / kGenChunk);
  GenArgs a{y, dst, ks.ring, ks.ring_bytes, ks.pos, g.region, g.n, nch, agg};
  k_gen_aggregate<<<dim3(nch, g.n), 256, 0, s>>>(a);
  check_launch("gen_aggregate");
  k_gen_prefix<<<(g.n + 127) / 128, 128, 0, s>>>(a);
  check_launch("gen_prefix");
  k_gen_scan<<<dim3(nch, g.n), 256, 0, s>>>(a);
  check_launch("gen_scan");
  *launches += 3;
}

// Slot-staged inverse round: tile rows T in [6, 15] (<= side) minimising the
// destination rows per SM, ceil(ceil(side / T) / SMs') * T (ties: larger T),
// with T*side*4 (slots) + side*4 (shift table) + 2 window stages of shared
// memory.  SMs' = SMs - 8: while its clip runs, each generator chain holds
// one SM (K1 reserves it), and a CTA count equal to the SM count would then
// need a second wave (measured at 1920^2: T = 13 -> 148 CTAs ran at 2x the
// single-wave time next to a chain).
uint32_t plan_decrypt_slots(const Geom& g, size_t& smem) {
  if (g.side % 16 || g.frame_bytes >= (uint64_t(1) << 32) || std::getenv("CVE_B200_NO_SLOTS"))
    return 0;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t best = 0;
  uint64_t best_load = ~uint64_t(0);
  for (uint32_t T = std::min<uint32_t>(6, g.side); T <= std::min<uint32_t>(kMaxChunkRows - 1, g.side); ++T) {
    const size_t need = size_t(T) * g.side * 4 + size_t(g.side) * 4 +
                        3 * kDecStageRows * 16 + 2 * kDecStageBytes;
    if (need > kSlotSmemMax) continue;
    const uint64_t ctas = (g.side + T - 1) / T;
    const uint64_t free_sms = uint64_t(std::max(1, sms - 8));
    const uint64_t load = (ctas + free_sms - 1) / free_sms * T;
    if (load <= best_load) {
      best_load = load;
      best = T;
      smem = need;
    }
  }
  return best;
}

// K3t tile: T = 15 rows (fewer if the side is smaller), W = the largest
// multiple of 16 dividing the side, <= 128 (the runs tv + wv - 1 <= 142 fit
// one CTA); shared memory = T*W slots + 128 B of windows per run.
bool plan_decrypt_tiles(const Geom& g, uint32_t& T, uint32_t& W, size_t& smem) {
  if (g.side % 16 || g.frame_bytes >= (uint64_t(1) << 32) || std::getenv("CVE_B200_NO_TILES"))
    return false;  // experiments only: CVE_B200_NO_TILES selects K3s
  T = std::min<uint32_t>(kTileMaxT, g.side);
  if (const char* e = std::getenv("CVE_B200_TILE_T")) T = std::max(1, std::min(atoi(e), int(T)));
  W = 16;
  for (uint32_t w = kTileMaxW; w >= 16; w -= 16)
    if (g.side % w == 0) {
      W = w;
      break;
    }
  if (const char* e = std::getenv("CVE_B200_TILE_W")) {
    const uint32_t w = uint32_t(atoi(e));
    if (w >= 16 && w <= kTileMaxW && w % 16 == 0) W = w;
  }
  smem = size_t(T) * W * 4 + size_t(T + W - 1) * (TILE_TMA ? 144 : 128);
  return true;
}

void launch_decrypt_round(const Geom& g, const uint8_t* src, uint8_t* dst,
                          KsWindow ks, const int32_t* shift, cudaStream_t s,
                          uint64_t* launches) {
  const bool aligned = (g.side % 16 == 0) && (ks.pos % 16 == 0) && (ks.ring_bytes % 16 == 0) &&
                       ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                         reinterpret_cast<uintptr_t>(ks.ring)) % 16 == 0);
  size_t smem = 0;
  uint32_t tT = 0, tW = 0;
  if (aligned && plan_decrypt_tiles(g, tT, tW, smem)) {
    TileArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n, g.rows,
               tT, tW, uint32_t(g.region), make_div(g.rows), g.frame_bytes};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((g.side + tW - 1) / tW, (g.side + tT - 1) / tT);
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = std::getenv("CVE_B200_NO_PDL") ? 0 : 1;  // experiments only
    cudaLaunchKernelEx(&cfg, k_decrypt_round_tiles, a);
    check_launch("decrypt_round_tiles");
    ++*launches;
    return;
  }
  const uint32_t Ts = aligned ? plan_decrypt_slots(g, smem) : 0;
  if (Ts) {
    DecArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n, g.rows,
              Ts, g.region, make_div(Ts), make_div(g.rows), g.frame_bytes};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((g.side + Ts - 1) / Ts);
    cfg.blockDim = dim3(kSlotThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = std::getenv("CVE_B200_NO_PDL") ? 0 : 1;  // experiments only
    cudaLaunchKernelEx(&cfg, k_decrypt_round_slots, a);
    check_launch("decrypt_round_slots");
    ++*launches;
    return;
  }
  const uint64_t row_bytes = uint64_t(g.side) * 3;
  uint32_t T = uint32_t(std::max<uint64_t>(1, (96 * 1024) / row_bytes));
  const uint32_t want = std::max<uint32_t>(8, (g.side + 147) / 148);
  T = std::min(T, want);
  T = std::min(T, g.side);
  smem = ((uint64_t(T) * row_bytes + 15) & ~uint64_t(15));
  if (smem > kSmemBudget) throw Error(Errc::invalid_argument, "frame side too large");
  DecArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n, g.rows,
            T, g.region, make_div(T), make_div(g.rows), g.frame_bytes};
  const uint32_t grid = (g.side + T - 1) / T;
  if (aligned)
    k_decrypt_round<true><<<grid, kDecThreads, smem, s>>>(a);
  else
    k_decrypt_round<false><<<grid, kDecThreads, smem, s>>>(a);
  check_launch("decrypt_round");
  ++*launches;
}

void launch_ring_move(const uint8_t* src, uint64_t src_bytes, uint8_t* dst,
                      uint64_t dst_bytes, uint64_t lo, uint64_t hi,
                      uint32_t workers, cudaStream_t s) {
  if (hi <= lo) return;
  k_ring_move<<<1024, 256, 0, s>>>(src, src_bytes, dst, dst_bytes, lo, hi, workers);
  check_launch("ring_move");
}

}  // namespace cveb
