// Host-callable launchers of the sm_100a kernels (prbg.cu, cipher.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace cveb {

// Per-lane constants of one PLCM orbit, precomputed on the host so the
// device loop has no division and no loop-invariant reciprocal to hoist.
//   q        = RN(0.5 - p)           the reference's (0.5 - p), chaos.cpp:31
//   yh_*+yl_* = 1/p, 1/q to ~2^-106   (yh = RN(1/d), yl = RN((1 - d*yh)/d))
//   cthr     = largest double <= 1-p  (x > cthr  <=>  1 - x < p, exactly)
//   a_b, a_d = offsets of the quotient correction term for cases B and D
//   hp, hq   = p/2, q/2               (rounding-verification thresholds)
//   nyl_*    = -yl_p, -yl_q           (the verifier's operand-selected step)
//   plo      = low 32 bits of p
struct LaneConst {
  double p, q;
  double yh_p, yl_p, yh_q, yl_q;
  double cthr, a_b, a_d;
  double hp, hq;
  double nyl_p, nyl_q;
  uint32_t plo, pad;
};

LaneConst make_lane_const(double p);

// Kernel attributes (dynamic smem limits, cluster sizes); once per device.
void configure_prbg_kernels();
void configure_cipher_kernels();
void configure_kernels_once(int device);

// Lane layout: lane l = 2*worker + (0 for the reference's lane a, 1 for b).

// x <- guard(x0); 256 exact warm-up iterations (chaos.cpp:79-91).
void launch_prbg_init(double* state, const LaneConst* lc, const double* x0,
                      uint32_t nlanes, cudaStream_t s);

// Device state of the generator.  Chain launches run back to back on one
// stream; verification/emission of launch L runs on another stream while
// the chain computes L+1, so every per-launch buffer is double-buffered.
struct PrbgBuffers {
  double* state;          // nlanes: chain position (written by the chain)
  double* ckpt[2];        // nlanes: start point of launch L (slot L&1)
  double* orbit[2];       // launch L's orbit: the value ending each 8-iteration group
                          // ((max_iters / 8) * nlanes), or every value if dense
  double* verified_end;   // nlanes: verified end point of the last launch
  unsigned* bad;          // nworkers: verification failure flags
  unsigned long long* replays;  // workers recomputed exactly (cumulative)
  unsigned long long* resync;   // nlanes: index of the launch last replayed (~0: none)
  uint32_t max_iters;           // per launch, multiple of 8
  // Dense orbit: the chain stores every value and the verifier streams them
  // (DRAM-bound, leaves SM issue slots to other clips' kernels: the
  // many-clips configuration); otherwise one checkpoint per 8 iterations and
  // the verifier regenerates the rest (the fastest chain: one clip).
  bool dense;
};

// (1) Chain: advances every lane by `iters` (multiple of 8, <= max_iters)
// iterations, group checkpoints into orbit[slot], start point into ckpt[slot].
// `launch` counts the generator's chain launches (0, 1, ...); `prev_iters`
// is the previous launch's iteration count.  A lane whose launch R was
// replayed exactly by the fix-up restarts from the verified end point in
// launch R + 1 (same-stream pipelines) or R + 2 (the chain of R + 1 already
// ran: its iterations are recomputed first), instead of continuing from its
// diverged speculative state forever.
void launch_prbg_chain(const PrbgBuffers& b, int slot, const LaneConst* lc,
                       uint32_t iters, uint32_t nlanes, uint64_t launch, uint32_t prev_iters,
                       cudaStream_t s);
// (2) Verify every step of launch `slot` against the reference's exact step
// (and that it starts where the previous launch verifiably ended), emit the
// keystream bytes of iterations [it0, it0+iters) into the ring at stream
// byte 6*it (mod ring_bytes, ring_bytes % 48 == 0), and (3) recompute any
// failed worker exactly from the verified end point.
void launch_prbg_verify(const PrbgBuffers& b, int slot, const LaneConst* lc,
                        uint8_t* ring, uint64_t ring_bytes, uint64_t it0,
                        uint32_t iters, uint32_t nlanes, uint64_t launch, cudaStream_t s);

// LASM generator (lasm.cu, row f2).  Lane layout as above; per lane the
// chain position (x, y) and mu.  Orbit values are lane-major:
// orbit[slot][lane * max_iters + i] = (x, y) after iteration i of the launch.
struct LasmBuffers {
  double2* state;
  double* mu;
  double2* orbit[2];
  uint32_t max_iters;  // per launch, multiple of 8
};
// 256 warm-up iterations from the start points xy0 (chaos.cpp:93-107).
void launch_lasm_init(double2* state, const double* mu, const double2* xy0, uint32_t nlanes,
                      cudaStream_t s);
// Advances every lane by `iters` (multiple of 8) iterations into orbit[slot].
void launch_lasm_chain(const LasmBuffers& b, int slot, uint32_t iters, uint32_t nlanes,
                       cudaStream_t s);
// Emits the 12 bytes per iteration of launch `slot` (iterations
// [it0, it0+iters), it0 % 8 == 0) into the ring at stream byte 12*it
// (mod ring_bytes, ring_bytes % 48 == 0).
void launch_lasm_emit(const LasmBuffers& b, int slot, uint8_t* ring, uint64_t ring_bytes,
                      uint64_t it0, uint32_t iters, uint32_t nlanes, cudaStream_t s);
// y[i] = glibc sin(x[i]) (glibc_sin.cuh), for parity tests.
void launch_glibc_sin(const double* x, double* y, size_t n, cudaStream_t s);

// Geometry of one square frame split into n row bands.
struct Geom {
  uint32_t side, n, rows;  // rows = side / n
  uint64_t region;         // rows * side * 3
  uint64_t frame_bytes;    // side * side * 3
};

// Keystream window of one round of one frame: worker i's byte j of this round
// is ring[i*ring_bytes + (pos + j) % ring_bytes].
struct KsWindow {
  const uint8_t* ring;
  uint64_t ring_bytes;
  uint64_t pos;
};

// shift[a] = euclid(floor(double(seed) * sine[a]), side)  (engine.cpp:14-30)
void launch_shift_table(const double* sine, uint32_t seed, int32_t* shift,
                        uint32_t side, cudaStream_t s);

// One forward round (confusion gather fused with the band XOR-scan
// diffusion).  plan_encrypt picks the slot-staged kernel when the geometry
// allows it (side % 16 == 0, <= 16 rows per chunk), else the byte-staged
// fused kernel, else (fused == false) the generic multi-kernel path.
struct EncPlan {
  bool fused;
  uint32_t chunk_rows, h;  // h chunks (one cluster) per band
  size_t smem;
  // slot-staged variant (side % 16 == 0); used when the launch's frames and
  // keystream window are 16-byte aligned, else the byte-staged one above
  bool slots;
  uint32_t s_rows, s_h;
  size_t s_smem;
};
EncPlan plan_encrypt(const Geom& g);
void launch_encrypt_round(const EncPlan& plan, const Geom& g,
                          const uint8_t* src, uint8_t* dst, KsWindow ks,
                          const int32_t* shift, uint8_t* scratch,
                          cudaStream_t s, uint64_t* launches);

// The two halves of the generic forward round on their own (the reference's
// Engine::transform with confusion or diffusion switched off,
// engine.cpp:207-250): the permutation src -> dst, and the band-wise chained
// rewrite y -> dst with one round's keystream window (agg: n * ceil(region /
// 4096) words of scratch).
void launch_confuse_only(const Geom& g, const uint8_t* src, uint8_t* dst, const int32_t* shift,
                         cudaStream_t s, uint64_t* launches);
void launch_diffuse_only(const Geom& g, const uint8_t* y, uint8_t* dst, KsWindow ks,
                         uint32_t* agg, cudaStream_t s, uint64_t* launches);

// K6: all `rounds` forward rounds of one frame (in place in `buf`) in one
// thread-block cluster, when the frame fits one (side % 16 == 0, up to
// ~768^2); false: not applicable, nothing launched.
bool launch_encrypt_frame(const Geom& g, uint8_t* buf, KsWindow ks, const int32_t* shift,
                          uint32_t rounds, cudaStream_t s, uint64_t* launches);

// One inverse round (elementwise inverse diffusion fused with the inverse
// confusion gather).
void launch_decrypt_round(const Geom& g, const uint8_t* src, uint8_t* dst,
                          KsWindow ks, const int32_t* shift, cudaStream_t s,
                          uint64_t* launches);

// K2r / K3r (rows.cu): rounds with one lane per destination row; a warp holds
// bpw = 32/cr blocks of cr lanes, block j of the nb blocks walks L = side/nb
// source rows.  plan_rows_* returns false when the geometry does not allow
// them (side % 16, 4-pixel groups, shared memory).
struct RowPlan {
  uint32_t cr, h;     // destination rows per CTA; CTAs (one cluster) per band
  uint32_t bpw, nb, L;
  uint32_t rs;        // shared-memory row stride
  size_t smem;
  uint32_t threads;   // per CTA
};
bool plan_rows_encrypt(const Geom& g, RowPlan& p);
bool plan_rows_decrypt(const Geom& g, RowPlan& p);
void configure_rows_kernels();
// K4 is folded in (the row rotations and s_d's row shift from the sine table
// and the seed), so no shift-table kernel precedes the first round.  pdl:
// launched as a programmatic dependent of the previous kernel in the stream
// (rounds 2..r: its keystream copies start before that round ends); the
// first round of a frame is launched plainly, behind every earlier stream
// operation (the waits for its keystream and input).
void launch_encrypt_round_rows(const RowPlan& p, const Geom& g, const uint8_t* src,
                               uint8_t* dst, KsWindow ks, const double* sine, uint32_t seed,
                               cudaStream_t s, bool pdl = true);
// Every round of one frame in one cooperative launch (K2r with a grid
// barrier between rounds; the next round's keystream rows load during the
// current one): buf -> sc0 -> sc1 -> ... -> buf.  gbar: one device counter.
// false: not applicable or not launchable (e.g. the grid cannot be
// co-resident); nothing was launched and the caller runs the rounds one by one.
bool launch_encrypt_frame_rows(const RowPlan& p, const Geom& g, uint8_t* buf, uint8_t* sc0,
                               uint8_t* sc1, KsWindow ks, const double* sine, uint32_t seed,
                               uint32_t rounds, unsigned* gbar, cudaStream_t s);
void launch_decrypt_round_rows(const RowPlan& p, const Geom& g, const uint8_t* src,
                               uint8_t* dst, KsWindow ks, const int32_t* shift, cudaStream_t s);

// Copies stream bytes [lo, hi) of every worker from one ring to another
// (ring growth).
void launch_ring_move(const uint8_t* src, uint64_t src_bytes, uint8_t* dst,
                      uint64_t dst_bytes, uint64_t lo, uint64_t hi,
                      uint32_t workers, cudaStream_t s);

}  // namespace cveb
