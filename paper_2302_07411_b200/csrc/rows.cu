// K2r / K3r: the cipher rounds with one lane per destination row (r02).
//
// Forward round (K2r, k_encrypt_round_rows).  Reference: confuse_rows
// (src/engine.cpp:32-47), diffuse_region (engine.cpp:66-73, engine.hpp:32-34)
// with the neighbour seed byte s_d (engine.cpp:237).  One CTA per chunk of cr
// destination rows al0 .. al0+cr-1 of a band; the h = rows/cr chunks of a
// band form one thread-block cluster (band prefix through DSMEM).
//
//   Destination row al0+k is the source anti-diagonal {(sr, (al0+k-sr) mod
//   side)} rotated by c_k = (k + shift[al0+k]) mod side: source row sr puts
//   its pixel o = (al0 - sr + k) mod side at destination column
//   (al0 - sr + c_k) mod side.  So lane k walks the source rows DOWNWARD and
//   produces destination row k left to right, one pixel per source row; the
//   cr lanes of a block read the same source row at consecutive columns (one
//   coalesced 3*cr-byte run per warp instruction and block).  A warp holds
//   32/cr blocks; block j owns source rows [j*L, (j+1)*L).
//
//   Keystream: each destination row's 3*side stream bytes are copied into
//   shared memory by TMA bulk copies (cp.async.bulk + mbarrier), ROTATED so
//   the row's pixel order as the lanes produce it -- position i <-> column
//   (rho_k + i) mod side, rho_k = (al0 + 1 + c_k) mod side, i = side-1-sr --
//   is linear: every lane's segment is one contiguous, unwrapped smem range.
//   The diffusion output overwrites the keystream in place.
//
//   Diffusion: t = b ^ ((y + b) mod 256), c_j = s_d ^ t_0 ^ .. ^ t_j is an
//   XOR prefix scan.  Each lane scans its own segment
//   (relative to the segment start), the per-row order of the segments gives
//   each segment's offset, the rows of the chunk and the chunks of the band
//   (cluster) give the row's; the copy-out to global XORs the constant of the
//   segment each 16-byte unit lies in.
//
//   k_encrypt_round_rows<true> runs every round of a frame in one
//   cooperative launch (grid barrier between rounds, the next round's
//   keystream rows prefetched into a second row buffer).  It is opt-in: it
//   measured slower than per-round launches chained by programmatic
//   dependent launch.
//
// Inverse round (K3r, k_decrypt_round_rows): inverse_diffuse_region
// (engine.cpp:75-83, engine.hpp:36-38), head fix-up (engine.cpp:271-276),
// inverse_confuse_rows (engine.cpp:49-64).  Output row a0+k, column o comes
// from cipher row al = (a0 + k + o) mod side, column (o + shift[al]) mod
// side; lane k walks the cipher rows upward (o ascending), the lanes of a
// block read one run of consecutive cipher columns (and their keystream
// bytes).  Inverse diffusion is elementwise (d = ((b ^ c ^ c_prev) - b)
// bytewise), so there is no scan and no cluster.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.hpp"
#include "keying.hpp"

namespace cveb {
namespace {

#ifdef ROWS_PROF
// phase timestamps of each CTA's thread 0 (tools/rows_bench.cu): %globaltimer
__device__ unsigned long long g_rows_prof[8192][8];
#define ROWS_STAMP(i)                                                         \
  do {                                                                        \
    if (threadIdx.x == 0 && blockIdx.x < 8192) {                              \
      unsigned long long t_;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_rows_prof[blockIdx.x][i] = t_;                                        \
    }                                                                         \
  } while (0)
#else
#define ROWS_STAMP(i) ((void)0)
#endif
// Device-side bounds checks (make BOUNDS=1): global frame / ring addresses
// and shared-memory row-slot addresses the row kernels form are checked
// against their buffers; a failure prints and traps.  Compiled out otherwise.
#ifdef CVE_B200_BOUNDS
#define RCHECK(cond)                                                                  \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      printf("cve rows bounds check failed: %s (%s:%d) block %d thread %d\n", #cond,  \
             __FILE__, __LINE__, blockIdx.x, threadIdx.x);                            \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define RCHECK(cond) ((void)0)
#endif
constexpr uint32_t kRowThreads = 1024;  // K2r maximum (the plan picks the count)
constexpr uint32_t kDecRowThreads = 512;  // K3r maximum
constexpr uint32_t kRowMaxCr = 16;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

// t = b ^ ((y + b) mod 256) per byte, then the inclusive XOR prefix across
// the word's bytes (little-endian order).
__device__ __forceinline__ uint32_t tprefix(uint32_t y, uint32_t b) {
  uint32_t t = b ^ (((y & 0x7F7F7F7Fu) + (b & 0x7F7F7F7Fu)) ^ ((y ^ b) & 0x80808080u));
  t ^= t << 8;
  t ^= t << 16;
  return t;
}

// The three bytes at frame byte offset a (any alignment) in the low bytes.
__device__ __forceinline__ uint32_t ld_pixel(const uint8_t* __restrict__ f, uint32_t a) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(f + (a & ~3u));
  return __funnelshift_r(__ldg(w), __ldg(w + 1), a << 3);
}
// Same, never touching the word after the pixel's last byte (the frame's
// final pixel: its second word would lie past the end of the buffer).
__device__ __forceinline__ uint32_t ld_pixel_safe(const uint8_t* __restrict__ f, uint32_t a) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(f + (a & ~3u));
  const uint32_t v1 = (a & 3u) >= 2u ? __ldg(w + 1) : 0u;
  return __funnelshift_r(__ldg(w), v1, a << 3);
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Stream bytes [off, off + len) of one worker's ring (off < ring_bytes, the
// range may wrap once) -> shared memory at dst, completing on mbar.  All of
// dst, the ring positions and len are multiples of 16.
__device__ __forceinline__ void bulk_stream(uint32_t dst, const uint8_t* ring,
                                            uint64_t ring_bytes, uint64_t off, uint32_t len,
                                            uint32_t mbar, uint64_t pol) {
  while (len) {
    const uint64_t room = ring_bytes - off;
    const uint32_t n = room < len ? uint32_t(room) : len;
    RCHECK(off < ring_bytes && off + n <= ring_bytes && (off & 15) == 0 && (n & 15) == 0 &&
           (dst & 15) == 0);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(ring + off), "r"(n), "r"(mbar), "l"(pol)
        : "memory");
    dst += n;
    len -= n;
    off += n;
    if (off >= ring_bytes) off -= ring_bytes;
  }
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000; selp.u32 %0, "
        "1, 0, p; }"
        : "=r"(done)
        : "r"(mbar), "r"(parity)
        : "memory");
}

// shift[a] exactly as k_shift computes it (engine.cpp:14-30).
__device__ __forceinline__ uint32_t shift_of(const double* sine, uint32_t seed, uint32_t a,
                                             uint32_t side) {
  const double v = __dmul_rn(double(seed), sine[a]);
  const long long s = (long long)floor(v);
  long long r = s % (long long)side;
  if (r < 0) r += side;
  return uint32_t(r);
}

// ---------------------------------------------------------------------------
// K2r
struct RowEncArgs {
  const uint8_t* src;
  uint8_t* dst;
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;
  const double* sine;  // sin(2 pi a / side) (K4's table input): shifts from it and the seed
  uint32_t seed;
  uint32_t side, n, rows, cr, h;
  uint32_t bpw;     // blocks (of cr lanes) per warp = 32 / cr
  uint32_t nb;      // blocks = segments per destination row
  uint32_t L;       // source rows per block, multiple of 4
  uint32_t rs;      // shared-memory row stride, multiple of 16
  uint32_t magic_L; // ceil(2^32 / L): floor(x / L) = umulhi(x, magic_L) for x < side
  uint64_t region;
  uint32_t pdl_early;  // trigger the next round at entry (else after the band prefix)
  uint32_t magic_3L;   // ceil(2^32 / 3L)
  // all rounds in one launch (k_encrypt_round_rows<true>): round k reads
  // k == 0 ? src : sc[(k-1) & 1] and writes k == rounds-1 ? dst : sc[k & 1];
  // gbar counts CTAs through the grid barrier between rounds (zeroed per launch)
  uint32_t rounds;
  uint8_t* sc[2];
  unsigned* gbar;
};

// PERSIST: every round of the frame in one cooperative launch (co-resident
// grid, a grid barrier after each round's copy-out); the next round's
// keystream rows land in the other of two shared-memory row buffers while
// this round runs.  Otherwise one round per launch.
template <bool PERSIST>
__global__ void __launch_bounds__(kRowThreads) k_encrypt_round_rows(const RowEncArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t s_rho[kRowMaxCr], s_d[kRowMaxCr], s_iz[kRowMaxCr], s_jz[kRowMaxCr];
  __shared__ uint32_t s_a1[kRowMaxCr], s_x1[kRowMaxCr], s_tot[kRowMaxCr];
  __shared__ __align__(8) uint64_t pmbar;  // chunk prefixes from the earlier chunks
  __shared__ uint32_t agg_in[16];
  __shared__ uint32_t s_prefix, s_chunk;

  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t band = blockIdx.x / a.h, chunk = blockIdx.x - band * a.h;
  const uint32_t side = a.side, cr = a.cr, nb = a.nb;
  const uint32_t RB = 3u * side;
  const uint32_t al0 = band * a.rows + chunk * cr;
  const uint32_t bufb = cr * a.rs;  // bytes of one row buffer
  uint8_t* aggb = sm + (PERSIST ? 2u : 1u) * bufb;  // cr * nb bytes: segment aggregates
  // cr * (nb + 2) words: per row, the segments' constants in row order
  uint32_t* rowc_all = reinterpret_cast<uint32_t*>(aggb + ((cr * nb + 15u) & ~15u));
  const uint32_t pmb = su32(&pmbar);
  ROWS_STAMP(0);

  // 0. Rotation of each destination row (from the sine table and the seed,
  //    so it does not wait for the shift-table kernel), smem placement.
  if (tid < cr) {
    uint32_t c = tid + shift_of(a.sine, a.seed, al0 + tid, side);
    c -= c >= side ? side : 0u;
    uint32_t rho = al0 + 1u + c;
    rho -= rho >= side ? side : 0u;
    rho -= rho >= side ? side : 0u;
    s_rho[tid] = rho;
    s_iz[tid] = rho == 0 ? 0u : side - rho;  // pixel index of column 0
    s_jz[tid] = ~0u;
    s_a1[tid] = 0;
    // row k's data starts at D_k = k*rs + 16 + (3 rho_k mod 16): the TMA
    // copies keep the stream's alignment mod 16
    s_d[tid] = tid * a.rs + 16u + ((3u * rho) & 15u);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar[0])), "r"(cr));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar[1])), "r"(cr));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pmb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the earlier chunks' totals: 4 bytes each
    if (chunk)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pmb), "r"(4u * chunk)
                   : "memory");
  }
  __syncthreads();
  // 1. Keystream of every destination row into shared memory, rotated:
  //    round kk's rows into row buffer bi (its mbarrier mbar[bi]).
  auto issue_keystream = [&](uint32_t kk, uint32_t bi) {
    if (tid < cr) {
      const uint32_t k = tid, rho = s_rho[k];
      uint64_t r0 = (a.pos + uint64_t(kk) * a.region) % a.ring_bytes + uint64_t(chunk) * cr * RB +
                    uint64_t(k) * RB;
      r0 %= a.ring_bytes;
      const uint8_t* ring = a.ring + uint64_t(band) * a.ring_bytes;
      const uint32_t cut = (3u * rho) & ~15u;  // part 1: [cut, RB) of the row
      const uint32_t len1 = RB - cut, len2 = (3u * rho + 15u) & ~15u;
      const uint32_t base = su32(sm) + bi * bufb + s_d[k] - ((3u * rho) & 15u);
      const uint32_t mb = su32(&mbar[bi]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                   "r"(len1 + len2)
                   : "memory");
      const uint64_t pol = evict_first_policy();
      uint64_t o1 = r0 + cut;
      o1 -= o1 >= a.ring_bytes ? a.ring_bytes : 0;
      bulk_stream(base, ring, a.ring_bytes, o1, len1, mb, pol);
      if (len2) bulk_stream(base + len1, ring, a.ring_bytes, r0, len2, mb, pol);
    }
  };
  issue_keystream(0, 0);
  if (!PERSIST && a.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.h > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (!PERSIST) asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous round wrote src

  const uint32_t nrounds = PERSIST ? a.rounds : 1u;
  for (uint32_t kr = 0; kr < nrounds; ++kr) {
  const uint32_t bi = PERSIST ? (kr & 1u) : 0u;  // this round's row buffer
  const uint8_t* __restrict__ src = !PERSIST || kr == 0 ? a.src : a.sc[(kr - 1u) & 1u];
  uint8_t* __restrict__ dst = !PERSIST || kr + 1u == nrounds ? a.dst : a.sc[kr & 1u];
  // frames written by this launch (rounds >= 1 of PERSIST) are read through
  // L2 only: L1 lines cached in an earlier round would be stale
  const bool coherent = PERSIST && kr > 0;
  auto ldf = [&](const uint32_t* p) { return coherent ? __ldcg(p) : __ldg(p); };
  if (PERSIST && kr + 1u < nrounds) {
    // the next round's rows into the other buffer (its last reader, the
    // copy-out of round kr-1, finished before the grid barrier)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue_keystream(kr + 1u, bi ^ 1u);
  }

  ROWS_STAMP(1);
  // s_d (engine.cpp:237): the post-confusion byte ((band+1) mod n + 1)*region
  // - 1 = pixel (last row of the next band, column side-1), channel 2.  The
  // load is issued now and consumed after the lane loop.
  uint32_t sd_val = 0;
  if (tid == 0) {
    const uint32_t nbd = band + 1 == a.n ? 0 : band + 1;
    const uint32_t al = nbd * a.rows + a.rows - 1;
    int o = int(side - 1) - int(shift_of(a.sine, a.seed, al, side));
    if (o < 0) o += side;
    int sr = int(al) - o;
    if (sr < 0) sr += side;
    const uint64_t ba = (uint64_t(sr) * side + uint32_t(o)) * 3 + 2;
    sd_val = coherent ? __ldcg(src + ba) : src[ba];
  }
  // 2. Lanes.  Block j = warp * bpw + lane / cr, lane row k = lane % cr.
  const uint32_t bw = lane / cr, k = lane - bw * cr;
  const uint32_t j = warp * a.bpw + bw;
  const bool active = bw < a.bpw && j < nb;
  const unsigned amask = __ballot_sync(0xFFFFFFFFu, active);
  uint32_t R = 0;   // running XOR byte, broadcast to the 4 bytes of a word
  if (active) {
    const uint32_t L = a.L, hi = (j + 1u) * L;
    const uint32_t D = bi * bufb + s_d[k], iz = s_iz[k];
    const uint32_t i0 = side - hi;  // first pixel index of the segment
    // frame offset of source row sr's pixel for this lane
    auto addr_of = [&](uint32_t sr) {
      uint32_t col = al0 + k + side - sr;
      col -= col >= side ? side : 0u;
      return sr * RB + 3u * col;
    };
    // Group g = source rows sr_g .. sr_g-3, sr_g = hi-1-4g.  Its pixel loads
    // are issued two groups ahead.  A lane's column wraps between rows
    // al0+k+1 and al0+k: groups that have (or follow) such a step take exact
    // per-pixel addresses, and never read the word after a pixel that ends
    // on a word boundary (the frame's last pixel, row side-1 / column side-1,
    // is read by lane side-2-al0 of the last chunk, whose wrap zone it is in).
    struct Grp {
      uint32_t w0[4], w1[4], sh[4];
    };
    const uint32_t ngroups = L >> 2;
    uint32_t fa = addr_of(hi - 1u);  // address of the next group to load (fast path)
    auto load = [&](Grp& G, uint32_t g) {
      const uint32_t sr = hi - 1u - 4u * g;
      const bool slow = __any_sync(amask, sr >= al0 && sr - 3u <= al0 + cr);
      if (!slow) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t at = fa - uint32_t(t) * (RB - 3u);
          const uint32_t* w = reinterpret_cast<const uint32_t*>(src + (at & ~3u));
          RCHECK(at == addr_of(sr - uint32_t(t)) && uint64_t(at & ~3u) + 8 <= uint64_t(side) * RB);
          G.w0[t] = ldf(w);
          G.w1[t] = ldf(w + 1);
          G.sh[t] = at << 3;
        }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t at = addr_of(sr - uint32_t(t));
          const uint32_t* w = reinterpret_cast<const uint32_t*>(src + (at & ~3u));
          RCHECK(uint64_t(at & ~3u) + ((at & 3u) >= 2u ? 8 : 4) <= uint64_t(side) * RB);
          G.w0[t] = ldf(w);
          G.w1[t] = ldf(w + ((at & 3u) >= 2u ? 1 : 0));
          G.sh[t] = at << 3;
        }
        fa = addr_of(sr - 3u);
      }
      fa -= 4u * (RB - 3u) - (slow ? 3u * (RB - 3u) : 0u);
    };
    Grp GA, GB;
    load(GA, 0);
    if (ngroups > 1) load(GB, 1);
    // smem byte of the segment's first pixel; alignment m is the same for
    // every 4-pixel group (12 bytes)
    // (shared-memory byte offsets; plain C++ accesses, so the compiler may
    // overlap one group's keystream loads with the previous group's stores:
    // they never touch the same word)
    const uint32_t q0 = D + 3u * i0;
    const uint32_t m8 = (q0 & 3u) * 8u;
    uint32_t qw = q0 & ~3u;  // aligned word of the current group's first byte
    mbar_wait(su32(&mbar[bi]), PERSIST ? (kr >> 1) & 1u : 0u);  // keystream in shared memory
    auto smw = [&](uint32_t off) -> uint32_t& { return *reinterpret_cast<uint32_t*>(sm + off); };
    uint32_t W0 = smw(qw);
    uint32_t prev = 0;  // previous group's out2 (its top bytes precede this group)
    auto step = [&](Grp& G, uint32_t g) {
      uint32_t p[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) p[t] = __funnelshift_r(G.w0[t], G.w1[t], G.sh[t]);
      if (g + 2u < ngroups) load(G, g + 2u);
      // keystream words of the group (12 bytes at q0 + 12 g)
      uint32_t W1, W2, W3;
      RCHECK(qw >= bi * bufb + k * a.rs && qw + 16u <= bi * bufb + (k + 1u) * a.rs);
      W1 = smw(qw + 4u);
      W2 = smw(qw + 8u);
      W3 = smw(qw + 12u);
      const uint32_t b0 = __funnelshift_r(W0, W1, m8), b1 = __funnelshift_r(W1, W2, m8),
                     b2 = __funnelshift_r(W2, W3, m8);
      const uint32_t y0 = __byte_perm(p[0], p[1], 0x4210), y1 = __byte_perm(p[1], p[2], 0x5421),
                     y2 = __byte_perm(p[2], p[3], 0x6542);
      const uint32_t t0 = tprefix(y0, b0), t1 = tprefix(y1, b1), t2 = tprefix(y2, b2);
      const uint32_t B0 = __byte_perm(t0, 0, 0x3333), B1 = __byte_perm(t1, 0, 0x3333),
                     B2 = __byte_perm(t2, 0, 0x3333);
      const uint32_t o0 = t0 ^ R, o1 = t1 ^ R ^ B0, o2 = t2 ^ R ^ B0 ^ B1;
      // exclusive running value at column 0 of the row (pixel index iz)
      const uint32_t ig = i0 + 4u * g;
      if (iz - ig < 4u) {
        const uint32_t pp = iz - ig;
        const uint32_t e = pp == 0 ? R : pp == 1 ? __byte_perm(o0, 0, 0x2222)
                                     : pp == 2 ? __byte_perm(o1, 0, 0x1111)
                                               : __byte_perm(o2, 0, 0x0000);
        s_a1[k] = e & 0xFFu;
        s_jz[k] = j;
      }
      R ^= B0 ^ B1 ^ B2;
      // store the group's 12 bytes in place (aligned words; the first word of
      // the segment is shared with the neighbouring segment: bytes only)
      const uint32_t A0 = m8 ? __funnelshift_l(prev, o0, m8) : o0;
      const uint32_t A1 = m8 ? __funnelshift_l(o0, o1, m8) : o1;
      const uint32_t A2 = m8 ? __funnelshift_l(o1, o2, m8) : o2;
      if (g == 0 && m8) {
        for (uint32_t bb = m8 >> 3; bb < 4u; ++bb) sm[qw + bb] = uint8_t(A0 >> (8u * bb));
      } else {
        smw(qw) = A0;
      }
      smw(qw + 4u) = A1;
      smw(qw + 8u) = A2;
      prev = o2;
      W0 = W3;
      qw += 12u;
    };
    for (uint32_t g = 0; g < ngroups; g += 2) {
      step(GA, g);
      if (g + 1u < ngroups) step(GB, g + 1u);
    }
    // tail: the top m bytes of the last group go into the low bytes of the
    // next word (shared with the next segment: bytes only)
    for (uint32_t bb = 0; bb < (m8 >> 3); ++bb)
      sm[qw + bb] = uint8_t(prev >> (8u * (4u - (m8 >> 3) + bb)));
    aggb[k * nb + j] = uint8_t(R);
  }
  ROWS_STAMP(2);
  __syncthreads();
  ROWS_STAMP(3);

  // 3. Per row (one warp per row): segment offsets in ROW ORDER.  The row
  //    starts at column 0 = pixel index iz, inside segment jz, and runs to
  //    higher pixel indices = lower j, cyclically: s_0 = jz from column 0 on,
  //    s_t = segment (jz - t) mod nb (t = 1 .. nb-1), s_nb = jz before column
  //    0.  rowc[t] = the XOR to apply to s_t's stored bytes (relative to the
  //    row start; broadcast), s_x1 = byte offset of s_1 in the row.
  for (uint32_t kk = warp; kk < cr; kk += blockDim.x >> 5) {
    const uint32_t jz = s_jz[kk], a1 = s_a1[kk];
    const uint8_t* ag = aggb + kk * nb;
    uint32_t* rowc = rowc_all + kk * (nb + 2);
    uint32_t carry = 0;
    for (uint32_t t0 = 0; t0 < nb; t0 += 32) {
      const uint32_t t = t0 + lane;
      const uint32_t jj = jz >= t ? jz - t : jz + nb - t;
      const uint32_t v = t < nb ? (t == 0 ? ag[jz] ^ a1 : ag[jj]) : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= uint32_t(d)) inc ^= u;
      }
      const uint32_t ex = (inc ^ v ^ carry) & 0xFFu;
      if (t < nb && t > 0) rowc[t] = ex * 0x01010101u;
      carry ^= __shfl_sync(0xFFFFFFFFu, inc, 31);
    }
    if (lane == 0) {
      rowc[0] = (a1 & 0xFFu) * 0x01010101u;  // stored bytes of s_0 include a1
      rowc[nb] = (carry & 0xFFu) * 0x01010101u;
      s_tot[kk] = (carry ^ a1) & 0xFFu;
      s_x1[kk] = 3u * (side - jz * a.L - s_iz[kk]);
    }
  }
  __syncthreads();
  ROWS_STAMP(4);
  // 4. Chunk prefix within the band: each chunk sends its total to the later
  //    chunks of the cluster (st.async into their agg_in, completing on
  //    their mbarrier); a chunk waits only for the earlier ones.
  if (tid == 0) {
    uint32_t tot = 0;
    for (uint32_t kk = 0; kk < cr; ++kk) tot ^= s_tot[kk];
    s_chunk = tot;
  }
  if (a.h > 1) {
    // every CTA of the cluster has started (phase 0: the arrive at entry)
    if (kr == 0) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (tid > chunk && tid < a.h) {
      uint32_t ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(&agg_in[chunk])), "r"(tid));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(pmb), "r"(tid));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(ra),
                   "r"(s_chunk), "r"(rb)
                   : "memory");
    }
    if (tid == 0) {
      uint32_t p = sd_val;
      if (chunk) {
        mbar_wait(pmb, kr & 1u);
        for (uint32_t jj = 0; jj < chunk; ++jj) p ^= agg_in[jj];
        // re-armed for the next round before the grid barrier, so no earlier
        // chunk's next total can arrive before its expectation
        if (PERSIST && kr + 1u < nrounds)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pmb),
                       "r"(4u * chunk)
                       : "memory");
      }
      s_prefix = p;
    }
  } else if (tid == 0) {
    s_prefix = sd_val;
  }
  __syncthreads();
  ROWS_STAMP(5);
  if (!PERSIST && !a.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // 5. Copy-out, one warp per row: unit x = 16u of row k lives at smem
  //    D_k + ((x - 3 rho_k) mod 3 side) (16-byte aligned) and belongs to
  //    s_t, t = x < x1 ? 0 : 1 + (x - x1) / 3L; at most one segment boundary
  //    per unit (segments are >= 8 pixels); the constant is E_k ^ rowc[t],
  //    E_k = s_d ^ chunk prefix ^ rows before k (engine.cpp:237, 66-73).
  const uint32_t U = RB >> 4;
  const uint32_t L3 = 3u * a.L;
  for (uint32_t kk = warp; kk < cr; kk += blockDim.x >> 5) {
    const uint32_t D = bi * bufb + s_d[kk], rho3 = 3u * s_rho[kk], x1 = s_x1[kk];
    const uint32_t* rowc = rowc_all + kk * (nb + 2);
    uint32_t e = s_prefix;
    for (uint32_t r = 0; r < kk; ++r) e ^= s_tot[r];
    e = (e & 0xFFu) * 0x01010101u;
    uint4* out = reinterpret_cast<uint4*>(dst + uint64_t(al0 + kk) * RB);
    for (uint32_t u = lane; u < U; u += 32) {
      const uint32_t x = 16u * u;
      int sgn = int(x) - int(rho3);
      sgn += sgn < 0 ? int(RB) : 0;
      const uint32_t su = uint32_t(sgn);
      RCHECK(D + su >= bi * bufb + kk * a.rs && D + su + 16u <= bi * bufb + (kk + 1u) * a.rs);
      uint4 v = *reinterpret_cast<const uint4*>(sm + D + su);
      uint32_t t = x < x1 ? 0u : 1u + __umulhi(x - x1, a.magic_3L);
      t = t > nb ? nb : t;
      const uint32_t xb = t == 0 ? x1 : (t == nb ? RB : x1 + L3 * t);  // next boundary
      const uint32_t bo = xb - x;
      const uint32_t c0 = rowc[t] ^ e, c1 = rowc[t + 1] ^ e;
      // branch-free: word w keeps c0 on its bytes before the boundary
      // (funnel shift with clamp: 0 -> no byte, >= 32 -> all four)
      const int sb = int(min(bo, 16u) * 8u);
      uint32_t cw[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t keep = __funnelshift_lc(~0u, 0u, uint32_t(max(sb - 32 * w, 0)));
        cw[w] = (c0 & keep) | (c1 & ~keep);
      }
      if (su + 16u > RB) {  // the rotation seam: bytes past the row wrap to D
        uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int bb = 0; bb < 16; ++bb) {
          if (uint32_t(bb) >= RB - su) {
            const uint32_t byte = sm[D + su + bb - RB];
            vw[bb >> 2] = (vw[bb >> 2] & ~(0xFFu << (8 * (bb & 3)))) | (byte << (8 * (bb & 3)));
          }
        }
        v = make_uint4(vw[0], vw[1], vw[2], vw[3]);
      }
      v.x ^= cw[0];
      v.y ^= cw[1];
      v.z ^= cw[2];
      v.w ^= cw[3];
      out[u] = v;
    }
  }
  ROWS_STAMP(6);
  if (PERSIST && kr + 1u < nrounds) {
    // grid barrier: every CTA's copy-out of this round is visible before any
    // CTA's next round reads it (release before the arrival, acquire after)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(a.gbar, 1u);
      const unsigned want = (kr + 1u) * gridDim.x;
      unsigned seen;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(a.gbar) : "memory");
      } while (seen < want);
      __threadfence();
    }
    __syncthreads();
  }
  }  // rounds
}

// ---------------------------------------------------------------------------
// K3r
struct RowDecArgs {
  const uint8_t* src;   // cipher frame of this round
  uint8_t* dst;
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;
  const int32_t* shift;
  uint32_t side, n, rows, cr;
  uint32_t bpw, nb, L, rs;
  uint64_t region;
  uint32_t magic_rows;    // ceil(2^32 / rows) (unused when rows == 1)
  uint32_t pos32, ring32; // pos, ring_bytes (< 2^32: checked by the plan)
};

// Row k of the CTA out by TMA bulk stores: global byte x of the row is at
// smem D + ((x - rho3) mod RB) (D == rho3 mod 16).  The parts before and
// after the rotation seam are 16-byte aligned on both sides; the 16-byte
// unit across the seam goes by hand.
__device__ __forceinline__ void row_store_tma(uint8_t* grow, uint32_t D, uint32_t rho3,
                                              uint32_t RB) {
  const uint32_t f = rho3 & ~15u, c = (rho3 + 15u) & ~15u;
  if (f)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(grow),
                 "r"(D + RB - rho3), "r"(f)
                 : "memory");
  if (c < RB)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(grow + c),
                 "r"(D + c - rho3), "r"(RB - c)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  if (c != f) {
    uint32_t vw[4] = {0, 0, 0, 0};
#pragma unroll
    for (int bb = 0; bb < 16; ++bb) {
      const uint32_t x = f + uint32_t(bb);
      const uint32_t sa = x < rho3 ? D + RB - rho3 + x : D + x - rho3;
      uint32_t byte;
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(byte) : "r"(sa));
      vw[bb >> 2] |= byte << (8 * (bb & 3));
    }
    *reinterpret_cast<uint4*>(grow + f) = make_uint4(vw[0], vw[1], vw[2], vw[3]);
  }
  // the shared memory must stay until the stores have read it; the writes
  // complete with the grid
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Inverse diffusion of one pixel (engine.hpp:36-38): cv = cipher bytes
// [ca-1, ca+3) (the byte before the pixel, then the pixel), kv = its
// keystream bytes; d = ((b ^ c ^ c_prev) - b) bytewise.
__device__ __forceinline__ uint32_t inv_pixel(uint32_t cv, uint32_t kv) {
  const uint32_t x = kv ^ (cv >> 8) ^ (cv & 0xFFFFFFu);
  return ((x | 0x80808080u) - (kv & 0x7F7F7F7Fu)) ^ ((x ^ ~kv) & 0x80808080u);
}

__global__ void __launch_bounds__(kDecRowThreads) k_decrypt_round_rows(const RowDecArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t s_d[kRowMaxCr], s_rho[kRowMaxCr];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t side = a.side, cr = a.cr, RB = 3u * side;
  const uint32_t a0 = blockIdx.x * cr;
  // band of cipher row c: c / rows (magic_rows = ceil(2^32 / rows) is 0 for
  // rows == 1, which does not fit 32 bits)
  auto band_of = [&](uint32_t c) { return a.rows == 1 ? c : __umulhi(c, a.magic_rows); };
  // per cipher row c: be0[c] = column of output row a0's pixel in row c,
  // ko[c] = stream offset (mod ring) of row c's first byte in its worker's
  // round window
  uint32_t* t_be0 = reinterpret_cast<uint32_t*>(sm + cr * a.rs);
  uint32_t* t_ko = t_be0 + side;
  if (tid < cr) {
    // output row a0+k, column o <- cipher row al = (a0 + k + o) mod side:
    // smem position i = al  <->  o = (rho_k + i) mod side, rho_k = (-a0-k) mod side
    uint32_t rho = 2u * side - a0 - tid;
    rho -= rho >= side ? side : 0u;
    rho -= rho >= side ? side : 0u;
    s_rho[tid] = rho;
    s_d[tid] = tid * a.rs + 16u + ((3u * rho) & 15u);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (uint32_t c = tid; c < side; c += blockDim.x) {
    uint32_t be = c + side - a0 + uint32_t(a.shift[c]);
    be -= be >= side ? side : 0u;
    be -= be >= side ? side : 0u;
    const uint32_t bandc = band_of(c);
    uint32_t ko = a.pos32 + (c - bandc * a.rows) * RB;
    ko -= ko >= a.ring32 ? a.ring32 : 0u;
    t_be0[c] = be;
    t_ko[c] = ko;
  }
  __syncthreads();

  const uint32_t bw = lane / cr, k = lane - bw * cr;
  const uint32_t j = warp * a.bpw + bw;
  const bool active = bw < a.bpw && j < a.nb && a0 + k < side;
  if (active) {
    const uint32_t L = a.L, lo = j * L;
    const uint32_t D = s_d[k];
    uint32_t qw = su32(sm) + D + 3u * lo;
    const uint32_t m8 = (qw & 3u) * 8u;
    qw &= ~3u;
    uint32_t prev = 0;
    // group g = cipher rows lo+4g .. lo+4g+3; loads issued two groups ahead
    struct Grp {
      uint32_t c0[4], c1[4], csh[4], k0[4], k1[4], ksh[4];
      uint32_t head;  // bit t: pixel t is a band head (or the frame's first pixel)
    };
    auto load = [&](Grp& G, uint32_t g) {
      G.head = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t c = lo + 4u * g + uint32_t(t);
        const uint32_t be0 = t_be0[c], ko = t_ko[c];
        uint32_t be = be0 - k;
        be += be0 < k ? side : 0u;
        const uint32_t ca = c * RB + 3u * be;  // the pixel's cipher byte offset
        const uint32_t cm = ca ? ca - 1u : 0u;
        const uint8_t* cw = a.src + (cm & ~3u);
        RCHECK(uint64_t(cm & ~3u) + ((cm & 3u) ? 8 : 4) <= uint64_t(side) * RB);
        G.c0[t] = __ldg(reinterpret_cast<const uint32_t*>(cw));
        G.c1[t] = __ldg(reinterpret_cast<const uint32_t*>(cw + ((cm & 3u) ? 4 : 0)));
        G.csh[t] = cm << 3;
        uint32_t kp = ko + 3u * be;
        kp -= kp >= a.ring32 ? a.ring32 : 0u;
        const uint8_t* kw = a.ring + uint64_t(band_of(c)) * a.ring_bytes + (kp & ~3u);
        RCHECK(kp + 3u <= a.ring32 && uint64_t(kp & ~3u) + ((kp & 3u) >= 2u ? 8 : 4) <= a.ring_bytes &&
               band_of(c) < a.n);
        G.k0[t] = __ldg(reinterpret_cast<const uint32_t*>(kw));
        G.k1[t] = __ldg(reinterpret_cast<const uint32_t*>(kw + ((kp & 3u) >= 2u ? 4 : 0)));
        G.ksh[t] = kp << 3;
        if (be == 0 && ko == a.pos32) G.head |= 1u << t;
      }
    };
    const uint32_t ngroups = L >> 2;
    Grp GA, GB;
    load(GA, 0);
    if (ngroups > 1) load(GB, 1);
    auto step = [&](Grp& G, uint32_t g) {
      uint32_t d[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t cv = __funnelshift_r(G.c0[t], G.c1[t], G.csh[t]);
        const uint32_t kv = __funnelshift_r(G.k0[t], G.k1[t], G.ksh[t]);
        d[t] = inv_pixel(cv, kv);
      }
      if (G.head) {
        // band head (engine.cpp:271-276): its first byte uses the next band's
        // recovered last byte, inverse-diffused here from the cipher
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (!((G.head >> t) & 1u)) continue;
          const uint32_t c = lo + 4u * g + uint32_t(t);
          const uint32_t bandc = band_of(c);
          const uint32_t nbd = bandc + 1 == a.n ? 0 : bandc + 1;
          const uint64_t last = (uint64_t(nbd) + 1) * a.region - 1;
          uint64_t kq = a.pos + a.region - 1;
          kq -= kq >= a.ring_bytes ? a.ring_bytes : 0;
          const uint32_t bl = a.ring[uint64_t(nbd) * a.ring_bytes + kq];
          const uint32_t sd = ((bl ^ a.src[last] ^ a.src[last - 1]) - bl) & 0xFFu;
          uint32_t cv = __funnelshift_r(G.c0[t], G.c1[t], G.csh[t]);
          if (c == 0) cv <<= 8;  // the frame's first pixel: bytes [0, 3)
          cv = (cv & ~0xFFu) | sd;
          d[t] = inv_pixel(cv, __funnelshift_r(G.k0[t], G.k1[t], G.ksh[t]));
        }
      }
      if (g + 2u < ngroups) load(G, g + 2u);
      const uint32_t o0 = __byte_perm(d[0], d[1], 0x4210), o1 = __byte_perm(d[1], d[2], 0x5421),
                     o2 = __byte_perm(d[2], d[3], 0x6542);
      const uint32_t A0 = m8 ? __funnelshift_l(prev, o0, m8) : o0;
      const uint32_t A1 = m8 ? __funnelshift_l(o0, o1, m8) : o1;
      const uint32_t A2 = m8 ? __funnelshift_l(o1, o2, m8) : o2;
      if (g == 0 && m8) {
        for (uint32_t bb = m8 >> 3; bb < 4u; ++bb)
          asm volatile("st.shared.u8 [%0], %1;" ::"r"(qw + bb), "r"(A0 >> (8u * bb)));
      } else {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(qw), "r"(A0));
      }
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(qw + 4u), "r"(A1));
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(qw + 8u), "r"(A2));
      prev = o2;
      qw += 12u;
    };
    for (uint32_t g = 0; g < ngroups; g += 2) {
      step(GA, g);
      if (g + 1u < ngroups) step(GB, g + 1u);
    }
    for (uint32_t bb = 0; bb < (m8 >> 3); ++bb)
      asm volatile("st.shared.u8 [%0], %1;" ::"r"(qw + bb), "r"(prev >> (8u * (4u - (m8 >> 3) + bb))));
  }
  // the next round is released only now: triggered at entry, its CTAs were
  // co-scheduled two per SM with this round's
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid < cr && a0 + tid < side)
    row_store_tma(a.dst + uint64_t(a0 + tid) * RB, su32(sm) + s_d[tid], 3u * s_rho[tid], RB);
}

}  // namespace

// ---------------------------------------------------------------------------
// Plans.  Lanes: a warp holds 32/cr blocks of cr lanes; nb = blocks per CTA
// must divide side/4 (4-pixel groups).  Shared memory: cr rows of 3*side + 64
// bytes (+ the segment tables).
// Row slot: 16 bytes before the row, up to 15 of alignment, 3*side bytes,
// up to 15 bytes of the rotated copy's overshoot; the stride is == 16 mod
// 128 bytes, so the lanes' rows start 4 banks apart.
static uint32_t row_stride(uint32_t side) {
  return ((3 * side + 48 - 16 + 127) / 128) * 128 + 16;
}

bool plan_rows_encrypt(const Geom& g, RowPlan& p) {
  if (g.side % 16 || g.frame_bytes >= (uint64_t(1) << 32) || std::getenv("CVE_B200_NO_ROWS"))
    return false;
  uint32_t forced = 0;
  if (const char* e = std::getenv("CVE_B200_ROWS_CR")) forced = uint32_t(std::atoi(e));
  // 1024 threads for 3840^2 (41 vs 48 us per round), 512 below (C4: 11.4 vs 12.1)
  uint32_t threads = g.side >= 3072 ? 1024 : 512;
  if (const char* e = std::getenv("CVE_B200_ROWS_THREADS")) threads = uint32_t(std::atoi(e));
  threads = std::min(threads, kRowThreads);
  const uint32_t nw = threads / 32;
  bool found = false;
  for (uint32_t cr = std::min(g.rows, kRowMaxCr - 1); cr >= 1; --cr) {
    if (g.rows % cr || g.rows / cr > 16) continue;
    if (forced && cr != forced) continue;
    const uint32_t bpw = 32 / cr;
    uint32_t nb = nw * bpw;
    // segments of L = side/nb pixels, L % 4 == 0 (4-pixel groups) and L >= 8
    // (a 16-byte unit of the copy-out meets at most one segment boundary)
    while (nb > 1 && ((g.side / 4) % nb || g.side / nb < 8)) --nb;
    if ((g.side / 4) % nb || g.side / nb < 8) continue;
    const uint32_t rs = row_stride(g.side);
    const size_t smem = size_t(cr) * rs + ((cr * nb + 15) & ~15u) + 4 * cr * (nb + 2);
    if (smem > 200 * 1024) continue;
    p = RowPlan{cr, g.rows / cr, bpw, nb, g.side / nb, rs, smem, threads};
    found = true;
    // prefer >= 128 CTAs per frame (the GPU has 148 SMs)
    if (uint64_t(g.n) * (g.rows / cr) >= 128 || forced) break;
  }
  return found;
}

bool plan_rows_decrypt(const Geom& g, RowPlan& p) {
  if (g.side % 16 || g.frame_bytes >= (uint64_t(1) << 32) || std::getenv("CVE_B200_NO_ROWS"))
    return false;
  uint32_t cr = 15;
  if (const char* e = std::getenv("CVE_B200_ROWS_DCR")) cr = uint32_t(std::atoi(e));
  cr = std::max(1u, std::min(cr, std::min(g.side, kRowMaxCr)));
  uint32_t threads = 512;
  if (const char* e = std::getenv("CVE_B200_ROWS_THREADS")) threads = uint32_t(std::atoi(e));
  threads = std::min(threads, kDecRowThreads);
  const uint32_t bpw = 32 / cr, nw = threads / 32;
  uint32_t nb = nw * bpw;
  while (nb > 1 && (g.side / 4) % nb) --nb;
  if ((g.side / 4) % nb || g.rows == 0) return false;
  const uint32_t rs = row_stride(g.side);
  const size_t smem = size_t(cr) * rs + 8 * size_t(g.side);
  if (smem > 200 * 1024) return false;
  p = RowPlan{cr, 1, bpw, nb, g.side / nb, rs, smem, threads};
  return true;
}

void configure_rows_kernels() {
  cudaFuncSetAttribute(k_encrypt_round_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 * 1024);
  cudaFuncSetAttribute(k_encrypt_round_rows<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_encrypt_round_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       227 * 1024);
  cudaFuncSetAttribute(k_encrypt_round_rows<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_decrypt_round_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 * 1024);
}

static void rows_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char msg[256];
    std::snprintf(msg, sizeof msg, "%s launch failed: %s", what, cudaGetErrorString(e));
    throw Error(Errc::internal, msg);
  }
}

void launch_encrypt_round_rows(const RowPlan& p, const Geom& g, const uint8_t* src,
                               uint8_t* dst, KsWindow ks, const double* sine, uint32_t seed,
                               cudaStream_t s, bool pdl) {
  RowEncArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, sine, seed, g.side, g.n,
               g.rows, p.cr, p.h, p.bpw, p.nb, p.L, p.rs,
               uint32_t((uint64_t(1) << 32) / p.L + ((uint64_t(1) << 32) % p.L ? 1 : 0)),
               g.region, 0,
               uint32_t((uint64_t(1) << 32) / (3 * p.L) + ((uint64_t(1) << 32) % (3 * p.L) ? 1 : 0)),
               1u, {nullptr, nullptr}, nullptr};
  if (const char* e = std::getenv("CVE_B200_ROWS_PDL_EARLY")) a.pdl_early = uint32_t(std::atoi(e));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.n * p.h);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.h;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && !std::getenv("CVE_B200_NO_PDL")) ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k_encrypt_round_rows<false>, a);
  rows_check("encrypt_round_rows");
}

bool launch_encrypt_frame_rows(const RowPlan& p, const Geom& g, uint8_t* buf, uint8_t* sc0,
                               uint8_t* sc1, KsWindow ks, const double* sine, uint32_t seed,
                               uint32_t rounds, unsigned* gbar, cudaStream_t s) {
  const size_t smem = p.smem + size_t(p.cr) * p.rs;  // a second row buffer
  if (rounds < 2 || smem > 227 * 1024) return false;
  RowEncArgs a{buf, buf, ks.ring, ks.ring_bytes, ks.pos, sine, seed, g.side, g.n,
               g.rows, p.cr, p.h, p.bpw, p.nb, p.L, p.rs,
               uint32_t((uint64_t(1) << 32) / p.L + ((uint64_t(1) << 32) % p.L ? 1 : 0)),
               g.region, 0,
               uint32_t((uint64_t(1) << 32) / (3 * p.L) + ((uint64_t(1) << 32) % (3 * p.L) ? 1 : 0)),
               rounds, {sc0, sc1}, gbar};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.n * p.h);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.h;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // the grid barrier needs a co-resident grid
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (cudaMemsetAsync(gbar, 0, sizeof(unsigned), s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (cudaLaunchKernelEx(&cfg, k_encrypt_round_rows<true>, a) != cudaSuccess) {
    cudaGetLastError();  // e.g. the grid cannot be co-resident: per-round launches
    return false;
  }
  return true;
}

void launch_decrypt_round_rows(const RowPlan& p, const Geom& g, const uint8_t* src,
                               uint8_t* dst, KsWindow ks, const int32_t* shift, cudaStream_t s) {
  RowDecArgs a{src, dst, ks.ring, ks.ring_bytes, ks.pos, shift, g.side, g.n, g.rows,
               p.cr, p.bpw, p.nb, p.L, p.rs, g.region,
               uint32_t((uint64_t(1) << 32) / g.rows + ((uint64_t(1) << 32) % g.rows ? 1 : 0)),
               uint32_t(ks.pos), uint32_t(ks.ring_bytes)};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((g.side + p.cr - 1) / p.cr);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = std::getenv("CVE_B200_NO_PDL") ? 0 : 1;
  cudaLaunchKernelEx(&cfg, k_decrypt_round_rows, a);
  rows_check("decrypt_round_rows");
}

}  // namespace cveb

#ifdef ROWS_PROF
namespace cveb {
void rows_prof_read(unsigned long long* host, size_t n) {
  cudaMemcpyFromSymbol(host, g_rows_prof, n * 8 * sizeof(unsigned long long));
}
}  // namespace cveb
#endif
