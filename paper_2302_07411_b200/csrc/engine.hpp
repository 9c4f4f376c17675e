// Host engine behind one cve_cipher handle: keying on the host, keystream
// ring + cipher rounds on the GPU, copies and kernels overlapped on streams.
//
// Mirrors the reference Engine (engine.hpp:66-95, engine.cpp:156-301):
// same constructor checks, same seed-before-validation order, same stream
// accounting (r * side^2 * 3 keystream bytes per frame), but the n worker
// threads + barrier pool become one sm_100a kernel per phase, and the
// synchronous frame loop becomes a pipeline:
//
//   s_gen : K1 chain kernels, back to back, ahead of the frames that need them
//           (the same stream as s_work with cve_set_streams_per_handle(1))
//   s_work: K1 verification + keystream emission (+ exact fix-up) of each
//           chain launch, then K4 shift table and K2/K3 rounds of the frames
//           whose keystream it verified (waits on s_gen and s_h2d events)
//   s_h2d : host->device frame copies  } CipherCtx streams, created on the
//   s_d2h : device->host copies        } first host-API call (wait on s_work)
//
// The keystream lives in one ring per worker (ring_bytes each).  Stream byte
// s of worker i sits at ring[i*ring_bytes + s % ring_bytes]; the generator
// never overwrites bytes a frame still has to read (event gating).
//
// A handle may also shard ONE clip across several devices (north star:
// "independent frames of a clip are partitioned across the B200s"): the
// generator (chain, verify, ring) stays on devices[0]; frame k is ciphered on
// shard k mod G, which first pulls that frame's keystream window (r * region
// bytes per worker, engine.cpp:198-205) from the ring with one peer copy per
// contiguous piece, then runs the shift table and the rounds on its own
// device and streams.  Frames stay independent given (seed, window), so no
// collective is needed; only the copy crosses NVLink.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "kernels.hpp"
#include "keying.hpp"

namespace cveb {

// NVTX range for the host-side phases (enqueue of frames, generator
// launches, ring growth, file pipelines).  NVTX v3 is header-only and a
// no-op unless a profiler (Nsight Systems) injects itself.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct EngineStats {
  uint64_t frames = 0;
  uint64_t keystream_iters = 0;
  uint64_t kernel_launches = 0;
  uint64_t prbg_launches = 0;
  uint64_t guard_replays = 0;
  double prbg_ms = 0;    // all generator kernels
  double chain_ms = 0;   // of which the sequential chain kernel
  double cipher_ms = 0;
};

// Streams per handle created from now on (process-wide): 2 (default) puts the
// generator chain on its own stream, so a single clip never waits for its
// cipher rounds; 1 keeps every handle on one hardware queue, so up to
// CUDA_DEVICE_MAX_CONNECTIONS (32) concurrent handles never share a queue
// (measured: 16 clips 3.5k frames/s with 2, 32 clips 5.4k frames/s with 1;
// a lone clip 261 vs 251 frames/s).  Initial value: CVE_B200_STREAMS_PER_HANDLE.
void set_streams_per_handle(int n);
int streams_per_handle();

// Round fusion (process-wide, read when a handle is created): whether the
// forward rounds of frames that fit one thread-block cluster (<= ~768^2) run
// as ONE cluster kernel (K6: the frame is read and written once, every round
// on-chip in distributed shared memory, 8-16 SMs per frame) or as one
// grid-wide kernel per round (K2s, all SMs).  0 (default) = one kernel per
// round: measured faster per frame (C1 37 vs 112-120 us) and in aggregate for
// 16-32 concurrent clips (C1 4.4k vs 4.2k, C3 6.5k vs 5.8k frames/s);
// 1 = K6 wherever the frame fits.  Initial value: $CVE_B200_ROUND_FUSION.
void set_round_fusion(int mode);
int round_fusion();

// Runs on `dev` until the scope ends, then restores the caller's device.  If
// no device can be queried (no driver), does nothing and lets the first CUDA
// call report INTERNAL, after the host-side checks ran (reference order).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev);
  ~DeviceScope();
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

// Pool of CUDA events created on one device (events can only be recorded
// on streams of their own device).
class EventPool {
 public:
  explicit EventPool(int dev = 0) : dev_(dev) {}
  ~EventPool() { release(); }
  EventPool(const EventPool&) = delete;
  EventPool& operator=(const EventPool&) = delete;
  int device() const { return dev_; }
  cudaEvent_t get(bool timing = false);
  void put(cudaEvent_t e, bool timing = false) { (timing ? timed_ : plain_).push_back(e); }
  void release() noexcept;

 private:
  int dev_;
  std::vector<cudaEvent_t> plain_, timed_;
};

// Per-device resources of the cipher rounds of one handle: the handle's own
// device, or one shard of a clip sharded across devices.
struct CipherCtx {
  static constexpr uint32_t kWindows = 2;  // keystream windows in flight (shards)
  explicit CipherCtx(int device) : dev(device), events(device) {}
  ~CipherCtx() { release(); }
  CipherCtx(const CipherCtx&) = delete;
  CipherCtx& operator=(const CipherCtx&) = delete;

  int dev;
  cudaStream_t s_work = nullptr;  // rounds (for the handle's own device: shared with verify)
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // created on first host-API use
  bool owns_work = false;
  uint8_t* scratch[3] = {nullptr, nullptr, nullptr};
  uint64_t scratch_bytes = 0;
  int32_t* d_shift = nullptr;
  unsigned* d_gbar = nullptr;  // grid-barrier counter of the all-rounds K2r launch
  uint32_t shift_cap = 0;
  std::map<uint32_t, double*> sines;
  std::vector<uint8_t*> slots;  // host-API frame slots
  uint64_t slot_bytes = 0;
  std::vector<cudaEvent_t> slot_free;
  uint32_t slot_next = 0;
  // sharded handles: keystream windows pulled from the generator's ring
  uint8_t* win[kWindows] = {nullptr, nullptr};
  uint64_t win_bytes = 0;
  cudaEvent_t win_free[kWindows] = {nullptr, nullptr};
  uint32_t win_next = 0;
  EventPool events;

  void ensure_copy_streams();
  void ensure_buffers(const Geom& g, uint32_t nslots);
  void ensure_windows(uint64_t bytes_per_worker, uint32_t workers);
  void set_l2_window();
  const double* sine_for(uint32_t side);
  void sync();
  // Frees everything in the stream order of s_work (after all queued work).
  void release() noexcept;
};

// Keystream generator of 2n lanes of either map on one device: the PLCM
// kernels (prbg.cu: speculative chain, verify/emit, fix-up) or the LASM
// kernels (lasm.cu: chain, emit).  chain(slot) advances every lane and writes
// orbit buffer `slot`; emit(slot) turns that orbit into keystream bytes.  The
// two orbit buffers let emission of launch L overlap the chain of launch L+1.
class Generator {
 public:
  Generator() = default;
  ~Generator() { release(); }
  Generator(const Generator&) = delete;
  Generator& operator=(const Generator&) = delete;

  // Uploads the lanes and runs the warm-up on `s` (synchronously).
  // orbit_iters = 0: no orbit buffers yet (see resize).
  // dense: PLCM chain stores every orbit value (see PrbgBuffers::dense).
  void init(const std::vector<WorkerLanes>& lanes, MapKind kind, cudaStream_t s,
            uint32_t orbit_iters, bool dense = false);
  // after == nullptr: nothing may still use the buffers; otherwise they are
  // released in the stream order of `after`, behind every user of them.
  void release(cudaStream_t after = nullptr) noexcept;
  MapKind kind() const { return kind_; }
  uint32_t bytes_per_iter() const { return kind_ == MapKind::Lasm ? 12 : 6; }
  // kernels one chain() + emit() pair launches: PLCM chain (start + walk when
  // checkpointed, one kernel when dense), verify/emit, fix-up; LASM chain, emit
  uint32_t kernels_per_launch() const {
    return kind_ == MapKind::Lasm ? 2u : (pb_.dense ? 3u : 4u);
  }
  uint32_t max_iters() const { return kind_ == MapKind::Lasm ? lb_.max_iters : pb_.max_iters; }
  // Largest launch (iterations, multiple of 8) the orbit memory budget allows.
  uint32_t orbit_cap_iters() const;
  // Regrows both orbit buffers to `iters` per launch (caller synchronised).
  void resize(uint32_t iters);
  void chain(int slot, uint32_t iters, cudaStream_t s);
  // Iterations [it0, it0+iters) of launch `slot` into the ring at stream byte
  // bytes_per_iter()*it (mod ring_bytes).
  void emit(int slot, uint8_t* ring, uint64_t ring_bytes, uint64_t it0, uint32_t iters,
            cudaStream_t s);
  uint64_t replays();  // PLCM workers recomputed exactly (always 0 for LASM)

 private:
  MapKind kind_ = MapKind::Plcm;
  uint32_t nl_ = 0;
  uint64_t chains_ = 0;          // chain launches so far (resync bookkeeping)
  uint32_t last_iters_ = 0;      // iterations of the latest chain launch
  uint64_t launch_of_[2] = {0, 0};  // launch index that wrote orbit slot k
  PrbgBuffers pb_{};
  LaneConst* d_lc_ = nullptr;
  LasmBuffers lb_{};
};

class Engine {
 public:
  Engine(const Key& key, uint32_t workers, uint32_t rounds, int device);
  // One clip sharded over `devices` (size >= 1, entries may repeat): the
  // generator runs on devices[0], frame k of the clip on devices[k mod G].
  Engine(const Key& key, uint32_t workers, uint32_t rounds, const std::vector<int>& devices);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  uint32_t workers() const { return n_; }
  uint32_t rounds() const { return r_; }
  uint64_t seeds_drawn() const { return coord_.seeds_drawn(); }
  int device() const { return dev_; }
  // Cipher shards: 1 for a single-device handle.
  uint32_t shard_count() const { return shards_.empty() ? 1u : uint32_t(shards_.size()); }
  int shard_device(uint32_t i) const { return shards_.empty() ? dev_ : shards_[i]->dev; }

  // `count` frames in host memory, in place.
  void run_host(uint8_t* px, uint32_t side, uint32_t count, bool decrypt);
  // Host frames whose input/output may be smaller than the side x side
  // working square: input w*h regions are padded on the device (zero rows
  // bottom, zero columns right, frame.cpp:28-39); output regions are the
  // top-left w*h crop (frame.cpp:41-51).  Frames are packed densely.
  struct HostIo {
    const uint8_t* in;
    uint32_t in_w, in_h;
    uint8_t* out;
    uint32_t out_w, out_h;
  };
  void run_host_io(const HostIo& io, uint32_t side, uint32_t count, bool decrypt);
  // `count` frames in device memory, in place, ordered on `user` stream.
  void run_device(uint8_t* d_px, uint32_t side, uint32_t count, bool decrypt,
                  cudaStream_t user);
  // Sharded handles: batch frame f lives on shard f % G at
  // shard_px[f % G] + (f / G) * frame_bytes, ordered on users[f % G]
  // (entries may be null: the legacy default stream of that device).
  void run_device_sharded(uint8_t* const* shard_px, uint32_t side, uint32_t count, bool decrypt,
                          const cudaStream_t* users);
  // The reference's Engine::transform (engine.cpp:302-307, forward 207-250):
  // one frame in host memory, in place, through `rounds` rounds with
  // confusion and/or diffusion switched off -- the two halves of the generic
  // round as separate kernels, not the fused production rounds.  Draws one
  // confusion seed (and, with diffusion, rounds * region stream bytes per
  // worker) like a frame call.  per_round(k, state) sees the frame after
  // round k = 1..rounds.  `t` (optional) receives host-clock phase times.
  struct PhaseMs {
    double bytegen_ms = 0, confuse_ms = 0, diffuse_ms = 0;
  };
  void transform_host(uint8_t* px, uint32_t side, uint32_t rounds, bool confusion,
                      bool diffusion,
                      const std::function<void(uint32_t, const uint8_t*)>& per_round,
                      PhaseMs* t);
  void synchronize();
  void peek(uint32_t worker, uint8_t* out, size_t len);
  void prefetch(uint64_t bytes);
  EngineStats stats();
  // Per-launch device times (ms) of the chain kernel since the last call,
  // for the bench's live roofline numbers.
  std::vector<float> take_prbg_times();

 private:
  struct Consumer {
    uint64_t lo, hi;
    cudaEvent_t done;
    EventPool* pool;  // the device the event belongs to
  };
  struct GenMark {
    uint64_t end_byte;
    cudaEvent_t ev;
  };
  struct Timed {
    cudaEvent_t a, b;
    EventPool* pool;
    bool chain, verify;  // neither: cipher rounds
  };

  void init(const std::vector<int>& devices);
  Geom geometry(uint32_t side) const;
  uint32_t draw_and_check(uint32_t side, uint32_t count);
  void ensure_ring(uint64_t need);
  void gen_until(uint64_t end_byte);
  cudaEvent_t gen_event_covering(uint64_t end_byte);
  // Rounds of one frame on ctx (the keystream is read from `ks`); returns
  // the event recorded on ctx.s_work behind them.
  cudaEvent_t enqueue_rounds(CipherCtx& c, uint8_t* buf, const Geom& g, uint32_t seed,
                             bool decrypt, KsWindow ks);
  // Single-device handle: rounds read the ring directly.
  cudaEvent_t enqueue_frame(uint8_t* buf, const Geom& g, uint32_t seed, bool decrypt);
  // Sharded handle: pull the window into the shard, then the rounds there.
  cudaEvent_t enqueue_shard_frame(CipherCtx& c, uint8_t* buf, const Geom& g, uint32_t seed,
                                  bool decrypt);
  void after_frame(uint64_t need);
  void timed_begin(EventPool& pool, cudaStream_t s, bool chain, bool verify = false);
  void timed_end(cudaStream_t s);
  void fold_timings(bool wait);
  void acquire(const std::vector<WorkerLanes>& lanes);  // constructor's CUDA resources
  void release() noexcept;

  Key key_;
  uint32_t n_, r_;
  int dev_;
  Coordinator coord_;

  cudaStream_t s_gen_ = nullptr, s_work_ = nullptr;
  cudaEvent_t chain_done_[2] = {nullptr, nullptr};
  cudaEvent_t ver_done_[2] = {nullptr, nullptr};
  uint64_t launches_ = 0;  // generator launches (slot = launches_ & 1)
  uint64_t gen_chunk_cap_ = 0;  // optional cap on iterations per generator launch
  bool one_stream_ = false;     // generator shares the rounds stream
  bool fuse_rounds_ = false;    // K6 cluster kernel for frames that fit
  Generator gen_;
  uint32_t bpi_ = 6;  // keystream bytes per generator iteration (6 PLCM, 12 LASM)

  uint8_t* ring_ = nullptr;
  uint64_t ring_bytes_ = 0;
  uint64_t cons_ = 0;       // stream bytes assigned to submitted frames
  uint64_t gen_iters_ = 0;  // iterations enqueued on s_gen
  std::deque<Consumer> consumers_;
  std::deque<GenMark> gens_;

  std::unique_ptr<CipherCtx> local_;                // rounds on dev_ (single-device handles)
  std::vector<std::unique_ptr<CipherCtx>> shards_;  // sharded handles
  uint64_t shard_rr_ = 0;                           // host-API frames dealt so far

  std::unique_ptr<EventPool> gen_events_;  // events of dev_
  std::vector<Timed> timed_;
  Timed open_{};
  std::vector<float> prbg_times_;
  EngineStats st_;
};

// Reference Prbg with explicit lanes, generated on the current device.
// launch_iters: cap on iterations per generator launch (0: none); replays
// (may be null): workers the fix-up recomputed exactly.
void standalone_stream(const Lane& a, const Lane& b, uint8_t* out, size_t len,
                       uint32_t launch_iters = 0, uint64_t* replays = nullptr,
                       bool dense = false);
void standalone_stream(const LasmLane& a, const LasmLane& b, uint8_t* out, size_t len);

// Fresh generators for a set of workers (reference WorkerParams::make_prbg,
// keying.cpp:154-162), advanced together on the GPU; next() copies the next
// `bytes` (<= chunk_bytes()) of every worker to host memory, worker-major
// with a stride of chunk_bytes().
class KeystreamSource {
 public:
  // max_bytes: the most any worker will be asked for (sizes the chunks)
  KeystreamSource(const std::vector<WorkerLanes>& lanes, MapKind kind, int device,
                  uint64_t max_bytes = ~uint64_t(0));
  ~KeystreamSource();
  KeystreamSource(const KeystreamSource&) = delete;
  KeystreamSource& operator=(const KeystreamSource&) = delete;
  uint64_t chunk_bytes() const { return uint64_t(gen_.max_iters()) * gen_.bytes_per_iter(); }
  void next(uint8_t* host, uint64_t bytes);
  // Advances every worker by `iters` iterations (rounded up to a multiple of
  // 8) and drops the bytes on the device: generation alone, for timing.
  // Not to be mixed with next() on one source.
  void burn(uint64_t iters);

 private:
  void release() noexcept;
  uint32_t n_;
  int dev_;
  Generator gen_;
  uint8_t* d_buf_ = nullptr;
  cudaStream_t s_ = nullptr;
  int slot_ = 0;
  uint64_t carry_ = 0;   // bytes of the current chunk already handed out
  uint64_t have_ = 0;    // bytes generated in the current chunk
};

}  // namespace cveb
