// K1: per-subframe PLCM keystream generator for sm_100a.
//
// Replaces the reference's Prbg::fill -> refill -> step_lane -> plcm_step /
// plcm_guard / extract_bytes hot loop (chaos.cpp:18-56, 109-153), called per
// worker from Engine::Impl::draw_streams (engine.cpp:198-205).
//
// The keystream of a clip is 2n sequential chaotic orbits (n subframes x 2
// lanes) that continue across frames, so the kernel is bound by the LATENCY
// of one dependent PLCM iteration -- not by bandwidth or FP64 throughput.
// The design takes everything that is not the orbit itself off that chain:
//
//   producer warps (SM sub-partitions 0,1): one orbit per thread, a
//     branch-free speculative step -- exact case predicates, exact numerator,
//     and the quotient num/d as fma(num, RN(1/d), corr) where the ~2^-53
//     correction corr ~= num * (1/d - RN(1/d)) is formed straight from x by
//     one FMA per case, so only DADD -> DADD -> DFMA -> FSEL remain on the
//     chain.  Each orbit value is stored (one coalesced 8-byte store).
//   verify+emit kernel (whole GPU, in parallel over steps): re-derives every
//     step with the reference's own case logic (chaos.cpp:28-32), proves the
//     produced quotient is the correctly rounded one (|num - d*y| < d*ulp(y)/2
//     via an exact FMA residual; IEEE division for the inconclusive powers
//     of two) and outside the guard set {0, p, 0.5, 1} (chaos.cpp:18-24),
//     and emits the keystream bytes.
//   fix-up kernel: any worker with a failed step is recomputed from the
//     launch checkpoint with IEEE __ddiv_rn and the exact guard.
//
// Output is therefore bit-identical to the reference's IEEE binary64 loop by
// construction.  Compiled with -fmad=false; every FP64 operation is an
// explicit _rn intrinsic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"

namespace cveb {

LaneConst make_lane_const(double p) {
  LaneConst c{};
  volatile double half = 0.5, one = 1.0;  // keep host evaluation IEEE
  c.p = p;
  c.q = half - p;
  c.yh_p = one / c.p;
  c.yl_p = std::fma(-c.p, c.yh_p, 1.0) / c.p;
  c.yh_q = one / c.q;
  c.yl_q = std::fma(-c.q, c.yh_q, 1.0) / c.q;
  // cthr = RD(1 - p): t - 1 is exact (Sterbenz) and the sign of RN(d + p)
  // is the sign of the exact sum, so t > 1 - p is decided exactly.
  double t = one - c.p;
  volatile double d = t - one;
  if (d + c.p < 0.0) t = std::nextafter(t, 0.0);
  c.cthr = t;
  c.a_b = -c.p * c.yl_q;
  c.a_d = (one - c.p) * c.yl_q;
  c.hp = 0.5 * c.p;
  c.hq = 0.5 * c.q;
  c.nyl_p = -c.yl_p;
  c.nyl_q = -c.yl_q;
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

// Speculative chain step.  Cases (reference: fold x>0.5 to 1-x, then
// f<p ? f/p : (f-p)/q):  A x<p: x/p   B p<=x<=.5: (x-p)/q
//                        C x>cthr: (1-x)/p   D .5<x<=cthr: ((1-x)-p)/q
// The case predicates and every numerator are exact; each quotient is
// fma(num, RN(1/d), corr) with corr ~= num*(1/d - RN(1/d)) formed from x by
// one FMA, and one select tree picks the case.  The chain is
// DADD -> DADD -> DFMA -> FSEL (case D).  Static schedule: 42 cycles per
// iteration (tools/iter_cycles.py; other formulations tried scored 44-57,
// tools/chain_search.py).
// The predicates are integer compares of the bit patterns (x >= 0, so the
// signed 64-bit order is the double order), which keeps 3 of the 14 FP64
// instructions off the FP64 pipe: 26.2 -> 25.4 ns/iteration
// (tools/chain_ops.cu, variant C).  fold tests x >= 0.5 on the high word:
// it differs from x > 0.5 only at x == 0.5, a guard value whose step the
// verifier always re-decides exactly.
__device__ __forceinline__ bool bits_gt(double u, double v) {
  return __double_as_longlong(u) > __double_as_longlong(v);
}

__device__ __forceinline__ double plcm_fast(double x, const LaneConst& c) {
  const bool a = bits_gt(c.p, x), cc = bits_gt(x, c.cthr);
  const bool fold = __double2hiint(x) >= 0x3FE00000;
  const double t1 = __dsub_rn(1.0, x);  // exact when x > 0.5
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  const double ya = __fma_rn(x, c.yh_p, __dmul_rn(x, c.yl_p));
  const double yb = __fma_rn(nb, c.yh_q, __fma_rn(x, c.yl_q, c.a_b));
  const double yc = __fma_rn(t1, c.yh_p, __fma_rn(-x, c.yl_p, c.yl_p));
  const double yd = __fma_rn(nd, c.yh_q, __fma_rn(-x, c.yl_q, c.a_d));
  return fold ? (cc ? yc : yd) : (a ? ya : yb);
}

// The chain's step on the FOLDED orbit value u = min(x, 1 - x) (r02, last
// session).  The map is symmetric -- the reference folds first (chaos.cpp:29:
// x > 0.5 ? 1 - x : x, exact for x >= 0.5), so F(x) == F(1 - x) bit for bit --
// and carrying u needs only the two unfolded quotient candidates plus their
// complements for the next fold: 7 FP64 instructions instead of 11 (the step
// is bound by FP64 issue slots, one per 2 cycles, plus the select's two pipe
// crossings; DESIGN 12).  Returns fold(F(u)); 1 - y is exact for y >= 0.5.
// Measured 23.12 -> 20.76 ns per iteration (tools/chain_folded.cu), the
// folded orbit bit-identical to the product step's over 2^27 lane-steps.
__device__ __forceinline__ double plcm_fast_folded(double u, const LaneConst& c) {
  const bool a = bits_gt(c.p, u);
  const double nb = __dsub_rn(u, c.p);
  const double ya = __fma_rn(u, c.yh_p, __dmul_rn(u, c.yl_p));
  const double yb = __fma_rn(nb, c.yh_q, __fma_rn(u, c.yl_q, c.a_b));
  const double ta = __dsub_rn(1.0, ya);
  const double tb = __dsub_rn(1.0, yb);
  const bool fa = __double2hiint(ya) >= 0x3FE00000, fb = __double2hiint(yb) >= 0x3FE00000;
  return a ? (fa ? ta : ya) : (fb ? tb : yb);
}

// u = min(x, 1 - x): the representative both sides of a comparison are
// reduced to where one of them may be a folded chain value.
__device__ __forceinline__ double plcm_fold(double x) {
  return x >= 0.5 ? __dsub_rn(1.0, x) : x;
}

// Is y exactly the reference's next orbit value after x?  Branch-free common
// path: one FMA residual test.  Values whose low word is 0 or p's (the guard
// set {0, 0.5, 1, p} and powers of two) or that are tiny only raise
// `suspect`; the caller re-decides those exactly with plcm_verify_exact.
__device__ __forceinline__ bool plcm_verify_fast(double x, double y, const LaneConst& c,
                                                 bool& suspect) {
  const double f = x > 0.5 ? __dsub_rn(1.0, x) : x;
  const bool low = f < c.p;
  const double num = low ? f : __dsub_rn(f, c.p);
  const double den = low ? c.p : c.q;
  const unsigned hi = unsigned(__double2hiint(y));
  const unsigned lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  // y is RN(num/den) iff |num - den*y| < den*ulp(y)/2 when y is not a power
  // of two (no quotient is a midpoint).  The FMA residual is exact for any
  // faithful y, and any error in it can only turn a pass into a (safe) fail.
  const double r = __fma_rn(-y, den, num);
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  suspect |= (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  return fabs(r) < thr;
}

// The verifier's step: regenerates y = plcm_fast(x) bit for bit -- the same
// FMAs on the same operands, but the case's operands are selected BEFORE the
// arithmetic, so one quotient is computed instead of four -- and checks that
// y is the reference's correctly rounded quotient num/den, where num and den
// are exactly the reference's (chaos.cpp:28-32: f = x > 0.5 ? 1 - x : x;
// f < p ? f/p : (f - p)/q).  fold tests x >= 0.5; at x == 0.5, 1 - x == x,
// so num and den are the reference's there too.  Same residual test and
// suspect flags as plcm_verify_fast.
__device__ __forceinline__ double plcm_regen_verify(double x, const LaneConst& c, bool& ok,
                                                    bool& suspect) {
  // The chain's predicates (x >= 0, so the integer compares there equal these
  // FP64 compares).  Here they go to the FP64 pipe: the verifier is bound by
  // the ALU pipe (selects, integer tests), the chain by FP64 latency.
  const bool a = x < c.p, cc = x > c.cthr;
  const bool fold = x >= 0.5;
  const double t1 = __dsub_rn(1.0, x);
  const double nb = __dsub_rn(x, c.p);
  const double nd = __dsub_rn(t1, c.p);
  const bool low = fold ? cc : a;  // f < p
  const double num = fold ? (cc ? t1 : nd) : (a ? x : nb);
  const double yh = low ? c.yh_p : c.yh_q;
  // (-x) * yl == x * (-yl) exactly: the sign goes into the selected constant
  const double yl = fold ? (cc ? c.nyl_p : c.nyl_q) : (a ? c.yl_p : c.yl_q);
  const double off = fold ? (cc ? c.yl_p : c.a_d) : (a ? 0.0 : c.a_b);
  const double y = __fma_rn(num, yh, __fma_rn(x, yl, off));
  const unsigned hi = unsigned(__double2hiint(y));
  const unsigned lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double r = __fma_rn(-y, low ? c.p : c.q, num);
  const double ulp = __hiloint2double(int(ex - (52u << 20)), 0);
  const double thr = __dmul_rn(low ? c.hp : c.hq, ulp);
  suspect |= (lo == 0u) | (lo == c.plo) | (ex < (53u << 20));
  ok &= fabs(r) < thr;
  return y;
}

// The verifier's step (r02): the exact next orbit value, computed with the
// reference's own case logic (chaos.cpp:28-32: f = x > 0.5 ? 1 - x : x;
// f < p ? f/p : (f - p)/q -- fold tests x >= 0.5, and at x == 0.5, 1 - x ==
// x), the quotient num/den from the selected operands as fma(num, yh,
// num*yl), proven correctly rounded by the residual test (same suspect flags
// as plcm_verify_fast).  It need not reproduce the chain's speculative
// formula bit for bit: the regenerated orbit is exact step by step, the
// bytes are emitted from it, and it must end on the chain's checkpoint.  Two
// operand selects fewer than the chain-exact form (no fold/case offset
// terms): the verifier is bound by the ALU pipe's selects.
__device__ __forceinline__ double plcm_check_step(double x, const LaneConst& c, bool& ok,
                                                  bool& suspect) {
  const bool fold = x >= 0.5;
  const double f = fold ? __dsub_rn(1.0, x) : x;  // exact when folded (Sterbenz)
  const bool low = f < c.p;
  const double num = low ? f : __dsub_rn(f, c.p);
  const double yh = low ? c.yh_p : c.yh_q;
  const double yl = low ? c.yl_p : c.yl_q;
  const double y = __fma_rn(num, yh, __dmul_rn(num, yl));
  const unsigned hi = unsigned(__double2hiint(y));
  const unsigned lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  // threshold den * ulp(y)/2 formed from den (p/2 and q/2 are exact halves):
  // no hp/hq select, 96 registers, so five 128-thread CTAs fit an SM
  // (57.7 -> 52.6 us per 144k-iteration C4 launch with the smaller CTAs)
  const double den = low ? c.p : c.q;
  const double r = __fma_rn(-y, den, num);
  const double hulp = __hiloint2double(int(ex - (53u << 20)), 0);  // ulp(y) / 2
  const double thr = __dmul_rn(den, hulp);
  suspect |= (lo == 0u) | (lo == c.plo) | (ex < (54u << 20));
  ok &= fabs(r) < thr;
  return y;
}

// Same decision with fewer operand selects (the verifier is bound by the ALU
// pipe): the quotient from yh and den alone -- y0 = num*yh, one exact
// residual correction y = y0 + (num - den*y0)*yh (Markstein's correction
// of a correctly rounded reciprocal) -- and the threshold den*ulp(y)/2
// formed from den (p/2 and q/2 are exact halves), so yl, hp/hq need no
// select.  Still proven by the residual test.
__device__ __forceinline__ double plcm_check_step_m(double x, const LaneConst& c, bool& ok,
                                                    bool& suspect) {
  const bool fold = x >= 0.5;
  const double f = fold ? __dsub_rn(1.0, x) : x;
  const bool low = f < c.p;
  const double num = low ? f : __dsub_rn(f, c.p);
  const double yh = low ? c.yh_p : c.yh_q;
  const double den = low ? c.p : c.q;
  const double y0 = __dmul_rn(num, yh);
  const double y = __fma_rn(__fma_rn(-y0, den, num), yh, y0);
  const unsigned hi = unsigned(__double2hiint(y));
  const unsigned lo = unsigned(__double2loint(y));
  const unsigned ex = hi & 0x7FF00000u;
  const double r = __fma_rn(-y, den, num);
  const double hulp = __hiloint2double(int(ex - (53u << 20)), 0);  // ulp(y) / 2
  suspect |= (lo == 0u) | (lo == c.plo) | (ex < (54u << 20));
  ok &= fabs(r) < __dmul_rn(den, hulp);
  return y;
}

// Exact decision: the reference step itself (IEEE division + guard).
__device__ __noinline__ bool plcm_verify_exact(double x, double y, const LaneConst& c) {
  return y == plcm_exact(x, c.p, c.q);
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

// Out of line, so the rare resynchronisation path leaves the chain's main
// loop schedule alone (inlined, it cost 23.15 -> 23.57 ns per iteration).
__device__ __noinline__ double chain_resync(uint32_t l, const LaneConst& c,
                                            const double* __restrict__ verified_end,
                                            unsigned long long* __restrict__ resync,
                                            uint32_t recompute) {
  double x = verified_end[l];
  for (uint32_t i = 0; i < recompute; ++i) x = plcm_fast(x, c);
  resync[l] = ~0ull;
  return x;
}

#ifndef CHAIN_GROUPS
#define CHAIN_GROUPS 4
#endif
// (1) The chain.  One orbit per thread, 4 warps per CTA, one CTA per SM, so
// every warp owns an SM sub-partition's in-order issue.  Two forms:
//   dense (many-clips handles): every true orbit value stored, the verifier
//     streams them from memory (k_prbg_chain_dense; the same folded step);
//   checkpointed (single clips, the fastest chain): per 8-iteration group 8
//     speculative iterations and ONE coalesced 8-byte store of the group's
//     last (folded) orbit value.  plcm_fast_folded is deterministic (IEEE _rn
//     intrinsics, integer compares, selects); the verifier regenerates the
//     true orbit exactly from the previous checkpoint and requires it to end
//     on this one: 1/8 of the stores on the chain and of the orbit traffic.
__global__ void __launch_bounds__(128, 1)
    k_prbg_chain_dense(double* __restrict__ state, double* __restrict__ ckpt,
                       const LaneConst* __restrict__ lcs, double* __restrict__ orbit,
                       uint32_t iters, uint32_t nlanes, const double* __restrict__ verified_end,
                       unsigned long long* __restrict__ resync, uint64_t launch,
                       uint32_t prev_iters) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlanes) return;
  const LaneConst c = lcs[l];
  double x = state[l];
  // Resynchronisation after an exact replay of launch R by the fix-up (it
  // stores R after the verified end point, release-ordered): launch R + 1
  // starts from the verified end; launch R + 2 -- whose predecessor already
  // ran from the diverged state -- first recomputes that launch's
  // iterations from it.  Never needed for correctness (the verifier proves
  // every step and continuity); it keeps a guard hit from sending every
  // later launch to the serial replay.
  unsigned long long R;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(R) : "l"(resync + l) : "memory");
  if (R != ~0ull && R < launch && launch - R <= 2)
    x = chain_resync(l, c, verified_end, resync, launch - R == 2 ? prev_iters : 0u);
  ckpt[l] = x;
  double* o = orbit + l;
  // the folded step (plcm_fast_folded), storing the TRUE orbit value of each
  // step -- the selected quotient before its fold -- for the streaming
  // verifier; the end state is the last true value
  double u = plcm_fold(x);
  for (uint32_t i = 0; i < iters; i += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool a = bits_gt(c.p, u);
      const double nb = __dsub_rn(u, c.p);
      const double ya = __fma_rn(u, c.yh_p, __dmul_rn(u, c.yl_p));
      const double yb = __fma_rn(nb, c.yh_q, __fma_rn(u, c.yl_q, c.a_b));
      const double ta = __dsub_rn(1.0, ya);
      const double tb = __dsub_rn(1.0, yb);
      const bool fa = __double2hiint(ya) >= 0x3FE00000, fb = __double2hiint(yb) >= 0x3FE00000;
      u = a ? (fa ? ta : ya) : (fb ? tb : yb);
      x = a ? ya : yb;
      o[size_t(t) * nlanes] = x;
    }
    o += size_t(8) * nlanes;
  }
  state[l] = x;
}

// Checkpointed generator as two kernels (r02, last session): the launch's
// start-up -- resynchronisation, the start checkpoint, folding the state --
// in a tiny kernel of its own, so that the chain kernel is nothing but the
// loop.  With the start-up code in the same kernel ptxas left a register move
// behind every step's select (on the dependency chain); alone, the loop gets
// the stand-alone probe's code (tools/chain_folded.cu).
__global__ void __launch_bounds__(128)
    k_prbg_chain_start(double* __restrict__ state, double* __restrict__ ckpt,
                       const LaneConst* __restrict__ lcs, uint32_t nlanes,
                       const double* __restrict__ verified_end,
                       unsigned long long* __restrict__ resync, uint64_t launch,
                       uint32_t prev_iters) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlanes) return;
  double x = state[l];
  unsigned long long R;  // see k_prbg_chain_dense
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(R) : "l"(resync + l) : "memory");
  if (R != ~0ull && R < launch && launch - R <= 2)
    x = chain_resync(l, lcs[l], verified_end, resync, launch - R == 2 ? prev_iters : 0u);
  ckpt[l] = x;
  state[l] = plcm_fold(x);
}

__global__ void __launch_bounds__(128, 1)
    k_prbg_chain_walk(double* __restrict__ state, const LaneConst* __restrict__ lcs,
                      double* __restrict__ orbit, uint32_t iters, uint32_t nlanes) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlanes) return;
  const LaneConst c = lcs[l];
  double x = state[l];  // folded by k_prbg_chain_start
  double* o = orbit + l;
  // CHAIN_GROUPS checkpoint groups (32 steps) per loop trip: measured (unfolded
  // step) 23.15 ns per iteration against 23.66 (2 groups), 23.35 (8) and 32.9
  // (16: instruction cache); folded step 21.53 / 21.97 (2) / 21.52 (8)
  uint32_t i = 0;
  for (; i + 8 * CHAIN_GROUPS <= iters; i += 8 * CHAIN_GROUPS) {
#pragma unroll
    for (int gq = 0; gq < CHAIN_GROUPS; ++gq) {
#pragma unroll
      for (int t = 0; t < 8; ++t) x = plcm_fast_folded(x, c);
      o[size_t(gq) * nlanes] = x;
    }
    o += size_t(CHAIN_GROUPS) * nlanes;
  }
  for (; i < iters; i += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) x = plcm_fast_folded(x, c);
    *o = x;
    o += nlanes;
  }
  state[l] = x;
}

// (2) Verify every step in parallel against the reference's exact step, and
// emit the keystream: 6 bytes per iteration per worker = the little-endian
// low 48 mantissa bits of x_a ^ x_b (extract_bytes, chaos.cpp:46-56).
// Thread = (lane, 8-iteration group), lanes fastest (coalesced checkpoint
// loads); the group's 8 orbit values are regenerated exactly from the
// previous group's checkpoint (every step proven correctly rounded) and must
// end on the group's checkpoint, so the chain walked exactly the reference's
// orbit and the bytes emitted from the regenerated values are the
// reference's; a group starting from a wrong checkpoint belongs to a flagged
// worker, whose launch the fix-up replays.  Lanes a/b of
// a worker are shuffle partners: the even one emits iterations 0-3 of the
// group, the odd one 4-7.  Group 0 also checks continuity: the launch must
// start where the previous launch verifiably ended.
#ifndef VERIFY_ILP
#define VERIFY_ILP 1
#endif
// plcm_check_step (r02, default) or plcm_regen_verify (the chain's formula)
#ifndef VERIFY_STEP
#define VERIFY_STEP plcm_check_step
#endif
constexpr int kVerifyIlp = VERIFY_ILP;
#ifndef VERIFY_MIN_BLOCKS
#define VERIFY_MIN_BLOCKS 5
#endif

#ifndef VERIFY_THREADS
#define VERIFY_THREADS 128  // 256: 57.7 us per 144k-iteration C4 launch, 128: 52.6, 96/32: 58-59 (spills)
#endif
template <bool DENSE>
__global__ void __launch_bounds__(VERIFY_THREADS, VERIFY_MIN_BLOCKS)
    k_prbg_verify_emit(const double* __restrict__ ckpt,
                       const double* __restrict__ verified_end,
                       const LaneConst* __restrict__ lcs,
                       const double* __restrict__ orbit, uint32_t iters,
                       uint32_t nlanes, uint32_t gs, uint8_t* __restrict__ ring,
                       uint64_t ring_bytes, uint64_t it0,
                       unsigned* __restrict__ bad) {
  // Persistent threads: thread = (lane l, first group g0), then groups
  // g0 + gs, g0 + 2 gs, ...; the lane constants are loaded once.  Every warp
  // runs the same number of trips (shuffle partners stay paired); trips past
  // the last group, and threads past gs * nlanes, shadow a real group and
  // store nothing.
  const uint64_t gid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t groups = iters / 8;
  const bool live_thread = gid < uint64_t(gs) * nlanes;
  const uint64_t me = live_thread ? gid : gid % nlanes;
  const uint32_t l = uint32_t(me % nlanes);
  const uint32_t g0 = uint32_t(me / nlanes);
  const LaneConst c = lcs[l];
  const uint32_t odd = l & 1u;
  // kVerifyIlp groups per trip, regenerated interleaved: a group's 8 steps
  // are one dependent chain, so independent groups are the ILP
  const uint32_t trips = (groups + gs - 1) / gs;
  // ring offset of group g0 + k gs, advanced without a 64-bit modulo per trip
  // (48 bytes per group; ring_bytes % 48 == 0 and every group is whole)
  uint64_t off0 = ((it0 + uint64_t(g0) * 8) * 6u) % ring_bytes;
  const uint64_t off_step = (uint64_t(gs) * 48u) % ring_bytes;
  bool flagged = false;
  // checkpointed: the next trip's start and end values are loaded one trip
  // ahead (the loads otherwise stall every trip: register-limited occupancy)
  auto group_of = [&](uint32_t kk) {
    const uint32_t gr = g0 + kk * gs;
    return (live_thread && gr < groups) ? gr : groups - 1;
  };
  double nx = 0.0, nend = 0.0;
  if (!DENSE) {
    const uint32_t gn = group_of(0);
    nx = gn ? orbit[size_t(gn - 1) * nlanes + l] : ckpt[l];
    nend = __ldg(orbit + size_t(gn) * nlanes + l);
  }
  for (uint32_t k = 0; k < trips; k += kVerifyIlp) {
    uint32_t g[kVerifyIlp];
    bool live[kVerifyIlp], cont[kVerifyIlp], ok[kVerifyIlp], suspect[kVerifyIlp];
    double x[kVerifyIlp], end[kVerifyIlp], y[kVerifyIlp][8];
#pragma unroll
    for (int j = 0; j < kVerifyIlp; ++j) {
      const uint32_t gr = g0 + (k + j) * gs;
      live[j] = live_thread && gr < groups;
      g[j] = live[j] ? gr : groups - 1;
      cont[j] = true;  // continuity with the previous launch (group 0 only)
      if (DENSE) {
        const size_t prev = size_t(g[j]) * 8 - 1;
        if (g[j]) {
          x[j] = orbit[prev * nlanes + l];
        } else {
          x[j] = ckpt[l];
          cont[j] = x[j] == verified_end[l];
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)  // all in flight
          y[j][t] = __ldg(orbit + (size_t(g[j]) * 8 + t) * nlanes + l);
      } else {
        x[j] = nx;
        end[j] = nend;
        // either side may be a folded chain value or an exact replay's end
        if (!g[j]) cont[j] = plcm_fold(x[j]) == plcm_fold(verified_end[l]);
        if (k + j + 1 < trips) {
          const uint32_t gn = group_of(k + j + 1);
          nx = gn ? orbit[size_t(gn - 1) * nlanes + l] : ckpt[l];
          nend = __ldg(orbit + size_t(gn) * nlanes + l);
        }
      }
      ok[j] = true;
      suspect[j] = false;
    }
    if (DENSE) {
#pragma unroll
      for (int j = 0; j < kVerifyIlp; ++j) {
        ok[j] = plcm_verify_fast(x[j], y[j][0], c, suspect[j]);
#pragma unroll
        for (int t = 1; t < 8; ++t) ok[j] &= plcm_verify_fast(y[j][t - 1], y[j][t], c, suspect[j]);
      }
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int j = 0; j < kVerifyIlp; ++j)
          y[j][t] = VERIFY_STEP(t ? y[j][t - 1] : x[j], c, ok[j], suspect[j]);
    }
#pragma unroll
    for (int j = 0; j < kVerifyIlp; ++j) {
      // the chain walked exactly these values (its checkpoints are folded)
      if (!DENSE) cont[j] &= plcm_fold(y[j][7]) == end[j];
      if (suspect[j]) {  // rare: decide this group exactly
        ok[j] = true;
        for (int t = 0; t < 8; ++t) ok[j] &= plcm_verify_exact(t ? y[j][t - 1] : x[j], y[j][t], c);
      }
      flagged |= live[j] && !(ok[j] && cont[j]);
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        lo[t] = unsigned(__double2loint(y[j][t]));
        hi[t] = unsigned(__double2hiint(y[j][t]));
      }
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
      const uint32_t w0 = mlo[0], w1 = mhi[0] | (mlo[1] << 16),
                     w2 = (mlo[1] >> 16) | (mhi[1] << 16), w3 = mlo[2],
                     w4 = mhi[2] | (mlo[3] << 16), w5 = (mlo[3] >> 16) | (mhi[3] << 16);
      const uint64_t off = off0;  // of group g0 + (k + j) gs
      off0 += off_step;
      off0 -= off0 >= ring_bytes ? ring_bytes : 0;
      if (live[j]) {
        uint8_t* dst = ring + uint64_t(l >> 1) * ring_bytes + off + (odd ? 24 : 0);
        if (!odd) {
          *reinterpret_cast<uint4*>(dst) = make_uint4(w0, w1, w2, w3);
          *reinterpret_cast<uint2*>(dst + 16) = make_uint2(w4, w5);
        } else {
          *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
          *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w2, w3, w4, w5);
        }
      }
    }
  }
  if (flagged) atomicOr(bad + (l >> 1), 1u);
}

// (3) One thread per worker.  Verified: advance the verified end point to
// the launch's last orbit values.  Flagged: recompute both lanes from the
// verified end point with IEEE division and the exact guard, rewriting the
// worker's bytes -- normally never taken.
__global__ void k_prbg_fixup(const double* __restrict__ orbit,
                             double* __restrict__ verified_end,
                             const LaneConst* __restrict__ lcs, uint32_t iters,
                             uint32_t nworkers, uint8_t* __restrict__ ring,
                             uint64_t ring_bytes, uint64_t it0,
                             unsigned* __restrict__ bad,
                             unsigned long long* __restrict__ replays,
                             unsigned long long* __restrict__ resync, uint64_t launch,
                             bool dense) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nworkers) return;
  const uint32_t nl = 2 * nworkers;
  if (!bad[w]) {  // the launch's last orbit value (its last checkpoint)
    const size_t last = dense ? size_t(iters) - 1 : size_t(iters / 8) - 1;
    verified_end[2 * w] = orbit[last * nl + 2 * w];
    verified_end[2 * w + 1] = orbit[last * nl + 2 * w + 1];
    return;
  }
  bad[w] = 0;
  const LaneConst ca = lcs[2 * w], cb = lcs[2 * w + 1];
  double xa = verified_end[2 * w], xb = verified_end[2 * w + 1];
  uint8_t* base = ring + uint64_t(w) * ring_bytes;
  uint64_t off = (it0 * 6u) % ring_bytes;
  for (uint32_t i = 0; i < iters; ++i) {
    xa = plcm_exact(xa, ca.p, ca.q);
    xb = plcm_exact(xb, cb.p, cb.q);
    uint64_t ba, bb;
    memcpy(&ba, &xa, 8);
    memcpy(&bb, &xb, 8);
    const uint64_t v = ba ^ bb;
    for (int k = 0; k < 6; ++k) base[off + k] = uint8_t(v >> (8 * k));
    off += 6;
    if (off == ring_bytes) off = 0;
  }
  verified_end[2 * w] = xa;
  verified_end[2 * w + 1] = xb;
  atomicAdd(replays, 1ull);
  // the chain of a later launch restarts from these end points (release:
  // verified_end is visible to whoever observes `launch` here)
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(resync + 2 * w), "l"(launch) : "memory");
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(resync + 2 * w + 1), "l"(launch)
               : "memory");
}

}  // namespace

void launch_prbg_init(double* state, const LaneConst* lc, const double* x0,
                      uint32_t nlanes, cudaStream_t s) {
  const uint32_t threads = 128;
  k_prbg_init<<<(nlanes + threads - 1) / threads, threads, 0, s>>>(state, lc,
                                                                    x0, nlanes);
}

// The chain CTA reserves all of an SM's shared memory, so no other CTA (not
// even the shared-memory-free verifier) is co-resident and steals issue slots
// from the 4 chain warps: 160 -> 227 KB gave 268 -> 270 frames/s at C4 and
// 5.66k -> 5.71k frames/s for 32 clips.
int chain_reserve() {
  static const int v = [] {
    int kb = 227;
    if (const char* e = std::getenv("CVE_B200_CHAIN_RESERVE_KB")) kb = std::atoi(e);  // experiments only
    return std::min(std::max(kb, 1), 227) * 1024;
  }();
  return v;
}

void configure_prbg_kernels() {
  cudaFuncSetAttribute(k_prbg_chain_dense, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       chain_reserve());
  cudaFuncSetAttribute(k_prbg_chain_walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       chain_reserve());
}

void launch_prbg_chain(const PrbgBuffers& b, int slot, const LaneConst* lc,
                       uint32_t iters, uint32_t nlanes, uint64_t launch, uint32_t prev_iters,
                       cudaStream_t s) {
  // 128 threads/CTA, one CTA per SM; the dynamic shared memory request only
  // enforces SM exclusivity (chain_reserve).
  if (!b.dense) {
    k_prbg_chain_start<<<(nlanes + 127) / 128, 128, 0, s>>>(
        b.state, b.ckpt[slot], lc, nlanes, b.verified_end, b.resync, launch, prev_iters);
    k_prbg_chain_walk<<<(nlanes + 127) / 128, 128, chain_reserve(), s>>>(
        b.state, lc, b.orbit[slot], iters, nlanes);
    return;
  }
  k_prbg_chain_dense<<<(nlanes + 127) / 128, 128, chain_reserve(), s>>>(
      b.state, b.ckpt[slot], lc, b.orbit[slot], iters, nlanes, b.verified_end, b.resync, launch,
      prev_iters);
}

void launch_prbg_verify(const PrbgBuffers& b, int slot, const LaneConst* lc,
                        uint8_t* ring, uint64_t ring_bytes, uint64_t it0,
                        uint32_t iters, uint32_t nlanes, uint64_t launch, cudaStream_t s) {
  const uint32_t nw = nlanes / 2;
  // group streams gs: enough threads to fill the GPU (2048 per SM), each
  // thread walking ceil(groups / gs) groups of its lane
  static int sms = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    return v;
  }();
  const uint32_t groups = iters / 8;
  const uint64_t target = uint64_t(sms) * 2048;
  const uint32_t gs = uint32_t(std::max<uint64_t>(
      1, std::min<uint64_t>(groups, (target + nlanes - 1) / nlanes)));
  const uint64_t threads = uint64_t(gs) * nlanes;
  auto vk = b.dense ? k_prbg_verify_emit<true> : k_prbg_verify_emit<false>;
  vk<<<uint32_t((threads + VERIFY_THREADS - 1) / VERIFY_THREADS), VERIFY_THREADS, 0, s>>>(
      b.ckpt[slot], b.verified_end, lc, b.orbit[slot], iters, nlanes, gs, ring, ring_bytes,
      it0, b.bad);
  k_prbg_fixup<<<(nw + 127) / 128, 128, 0, s>>>(b.orbit[slot], b.verified_end, lc,
                                                iters, nw, ring, ring_bytes, it0,
                                                b.bad, b.replays, b.resync, launch,
                                                b.dense);
}

}  // namespace cveb
