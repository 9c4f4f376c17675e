// Host-callable launchers of the sm_100a kernels (prbg.cu, cipher.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace cveb {

// Per-lane constants of one PLCM orbit, precomputed on the host so the
// device loop has no division and no loop-invariant reciprocal to hoist:
//   q  = RN(0.5 - p)         (the reference's (0.5 - p), chaos.cpp:31)
//   rp = RN(1/p), rq = RN(1/q)
//   hp = p/2, hq = q/2       (exact; rounding-verification thresholds)
//   plo = low 32 bits of p   (guard pre-filter)
struct LaneConst {
  double p, q, rp, rq, hp, hq;
  uint32_t plo, pad;
};

LaneConst make_lane_const(double p);

// Lane layout: lane l = 2*worker + (0 for the reference's lane a, 1 for b).

// x <- guard(x0); 256 exact warm-up iterations (chaos.cpp:79-91).
void launch_prbg_init(double* state, const LaneConst* lc, const double* x0,
                      uint32_t nlanes, cudaStream_t s);

// Advances every lane by 8*nblk iterations starting at iteration `it0`
// (multiple of 8) and writes each worker's 6 bytes/iteration at stream byte
// 6*it (mod ring_bytes) of that worker's ring.  ring_bytes % 48 == 0.
void launch_prbg_generate(double* state, const LaneConst* lc, uint8_t* ring,
                          uint64_t ring_bytes, uint64_t it0, uint32_t nblk,
                          uint32_t nlanes, unsigned long long* replays,
                          uint32_t reserve_smem, cudaStream_t s);

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
// diffusion).  Returns false if this geometry needs the generic path.
struct EncPlan {
  bool fused;
  uint32_t chunk_rows, h;  // h chunks (one cluster) per band
  size_t smem;
};
EncPlan plan_encrypt(const Geom& g);
void launch_encrypt_round(const EncPlan& plan, const Geom& g,
                          const uint8_t* src, uint8_t* dst, KsWindow ks,
                          const int32_t* shift, uint8_t* scratch,
                          cudaStream_t s, uint64_t* launches);

// One inverse round (elementwise inverse diffusion fused with the inverse
// confusion gather).
void launch_decrypt_round(const Geom& g, const uint8_t* src, uint8_t* dst,
                          KsWindow ks, const int32_t* shift, cudaStream_t s,
                          uint64_t* launches);

// Copies stream bytes [lo, hi) of every worker from one ring to another
// (ring growth).
void launch_ring_move(const uint8_t* src, uint64_t src_bytes, uint8_t* dst,
                      uint64_t dst_bytes, uint64_t lo, uint64_t hi,
                      uint32_t workers, cudaStream_t s);

}  // namespace cveb
