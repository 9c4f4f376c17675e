#include "engine.hpp"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

namespace cveb {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
    throw Error(Errc::internal, msg);
  }
}

uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

// ---- process-wide device resources -----------------------------------------
// Handles are cheap to create and destroy (a one-frame clip is a real use,
// BASELINE config C1): device buffers come from the device's stream-ordered
// memory pool, which keeps freed memory for the next handle, and streams
// from a free list.  Measured before: cudaMalloc/cudaFree and stream
// create/destroy made a C1 handle's create + first frame + destroy cost
// ~9 ms, as much as the reference's whole CPU frame.
constexpr uint64_t kPoolRetainBytes = 4ull << 30;  // kept by the pool when freed

struct DevPool {
  std::mutex mu;
  std::map<int, std::vector<cudaStream_t>> idle;  // idle non-blocking streams
  std::map<int, cudaStream_t> alloc;              // allocation stream per device
  std::map<int, cudaMemPool_t> pools;             // the library's private memory pools
  std::set<std::pair<int, int>> access;           // (pool device, peer) granted
};

DevPool& devpool() {
  static DevPool* p = new DevPool;  // process lifetime (no teardown-order issues at exit)
  return *p;
}

int current_dev() {
  int d = 0;
  ck(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}

cudaStream_t alloc_stream(int dev) {
  DevPool& P = devpool();
  std::lock_guard<std::mutex> lock(P.mu);
  cudaStream_t& s = P.alloc[dev];
  if (!s) ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  return s;
}

// The library's own stream-ordered memory pool of `dev` (not the device's
// default pool, which the host application -- e.g. PyTorch's cudaMallocAsync
// backend -- owns and tunes): it keeps up to kPoolRetainBytes of freed
// handle buffers for the next handle.
cudaMemPool_t mem_pool(int dev) {
  DevPool& P = devpool();
  std::lock_guard<std::mutex> lock(P.mu);
  cudaMemPool_t& pool = P.pools[dev];
  if (!pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t fresh = nullptr;
    ck(cudaMemPoolCreate(&fresh, &props), "cudaMemPoolCreate");
    uint64_t retain = kPoolRetainBytes;
    ck(cudaMemPoolSetAttribute(fresh, cudaMemPoolAttrReleaseThreshold, &retain), "mempool");
    pool = fresh;
  }
  return pool;
}

// Lets `peer` read and write allocations of `dev`'s pool (a sharded handle's
// shards pull keystream windows out of the generator device's ring).  A
// no-op without peer capability: the copies are then staged by the driver.
void grant_peer_access(int dev, int peer) {
  if (dev == peer) return;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, peer, dev) != cudaSuccess || !can) {
    cudaGetLastError();
    return;
  }
  const cudaMemPool_t pool = mem_pool(dev);
  DevPool& P = devpool();
  std::lock_guard<std::mutex> lock(P.mu);
  if (P.access.count({dev, peer})) return;
  cudaMemAccessDesc d{};
  d.location.type = cudaMemLocationTypeDevice;
  d.location.id = peer;
  d.flags = cudaMemAccessFlagsProtReadWrite;
  ck(cudaMemPoolSetAccess(pool, &d, 1), "cudaMemPoolSetAccess");
  P.access.insert({dev, peer});
}

// Device memory of the current device, usable from any stream on return.
template <class T>
void dmalloc(T** p, uint64_t bytes, const char* what) {
  *p = nullptr;
  if (!bytes) return;
  const int dev = current_dev();
  const cudaStream_t s = alloc_stream(dev);
  void* v = nullptr;
  ck(cudaMallocFromPoolAsync(&v, bytes, mem_pool(dev), s), what);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFreeAsync(v, s);
    ck(e, what);
  }
  *p = static_cast<T*>(v);
}

// Returns memory to the pool.  s == nullptr: no stream may still use it
// (callers synchronise first); otherwise the memory is released when `s`
// reaches this point, and every user of it must be ordered before.
void dfree(void* p, cudaStream_t s = nullptr) noexcept {
  if (!p) return;
  if (!s) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return;
    try {
      s = alloc_stream(d);
    } catch (...) {
      return;
    }
  }
  cudaFreeAsync(p, s);
}

// An idle pooled stream (streams of destroyed handles may still be
// finishing their last work: those are skipped), else a new one.
cudaStream_t stream_get() {
  const int dev = current_dev();
  DevPool& P = devpool();
  {
    std::lock_guard<std::mutex> lock(P.mu);
    auto& v = P.idle[dev];
    for (size_t i = v.size(); i-- > 0;) {
      if (cudaStreamQuery(v[i]) == cudaSuccess) {
        cudaStream_t s = v[i];
        v.erase(v.begin() + long(i));
        return s;
      }
    }
    cudaGetLastError();  // cudaErrorNotReady from the queries is not an error
  }
  cudaStream_t s = nullptr;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  return s;
}

// Back to the pool (it may still be finishing queued work).
void stream_put(cudaStream_t s) noexcept {
  if (!s) return;
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) return;
  DevPool& P = devpool();
  std::lock_guard<std::mutex> lock(P.mu);
  try {
    P.idle[d].push_back(s);
  } catch (...) {
    cudaStreamDestroy(s);
  }
}

constexpr uint32_t kSlots = 3;  // host frames in flight (H2D / work / D2H)
constexpr uint64_t kOrbitBytes = 128ull << 20;  // per generator launch

void free_prbg(PrbgBuffers& b, cudaStream_t s = nullptr) {
  dfree(b.state, s);
  dfree(b.verified_end, s);
  for (int k = 0; k < 2; ++k) {
    dfree(b.ckpt[k], s);
    dfree(b.orbit[k], s);
  }
  dfree(b.bad, s);
  dfree(b.replays, s);
  dfree(b.resync, s);
  b = PrbgBuffers{};
}

// Every upload / memset below is ordered on the stream that consumes it: the
// synchronous cudaMemcpy / cudaMemset run on the legacy default stream, which
// does not order against our non-blocking streams (a pageable H2D cudaMemcpy
// may even return before its DMA lands).
// orbit_iters = 0: no orbit buffers yet (an Engine sizes them from its ring,
// resize_orbit); otherwise capacity for launches of orbit_iters iterations.
PrbgBuffers alloc_prbg(uint32_t nlanes, cudaStream_t s, uint32_t orbit_iters, bool dense) {
  PrbgBuffers b{};
  b.dense = dense;
  try {
    const size_t lanes_bytes = nlanes * sizeof(double);
    dmalloc(&b.state, lanes_bytes, "cudaMalloc state");
    dmalloc(&b.verified_end, lanes_bytes, "cudaMalloc state");
    for (int k = 0; k < 2; ++k) {
      dmalloc(&b.ckpt[k], lanes_bytes, "cudaMalloc ckpt");
      if (orbit_iters)  // one checkpoint per 8 iterations, or every value
        dmalloc(&b.orbit[k], uint64_t(dense ? orbit_iters : orbit_iters / 8) * lanes_bytes,
                "cudaMalloc orbit");
    }
    b.max_iters = orbit_iters;
    dmalloc(&b.bad, (nlanes / 2) * sizeof(unsigned), "cudaMalloc flags");
    dmalloc(&b.replays, sizeof(unsigned long long), "cudaMalloc");
    dmalloc(&b.resync, nlanes * sizeof(unsigned long long), "cudaMalloc");
    ck(cudaMemsetAsync(b.bad, 0, (nlanes / 2) * sizeof(unsigned), s), "memset");
    ck(cudaMemsetAsync(b.replays, 0, sizeof(unsigned long long), s), "memset");
    ck(cudaMemsetAsync(b.resync, 0xFF, nlanes * sizeof(unsigned long long), s), "memset");
  } catch (...) {
    free_prbg(b);
    throw;
  }
  return b;
}

// Grows both orbit buffers to launches of `iters` iterations (caller has
// synchronised: no kernel may be using them).
void resize_orbit(PrbgBuffers& b, uint32_t nlanes, uint32_t iters) {
  for (int k = 0; k < 2; ++k) {
    dfree(b.orbit[k]);
    b.orbit[k] = nullptr;
  }
  b.max_iters = 0;
  for (int k = 0; k < 2; ++k)  // one checkpoint per 8 iterations, or every value
    dmalloc(&b.orbit[k], uint64_t(b.dense ? iters : iters / 8) * nlanes * sizeof(double),
            "cudaMalloc orbit");
  b.max_iters = iters;
}

// x <- guard(x0) + 256 warm-up steps; the warm state is the first verified
// end point.
void init_prbg(const PrbgBuffers& b, const LaneConst* d_lc, const double* x0,
               uint32_t nlanes, cudaStream_t s) {
  struct Staging {  // freed on every path, once the stream is done with it
    double* p = nullptr;
    cudaStream_t s;
    ~Staging() {
      if (p) cudaStreamSynchronize(s);
      dfree(p);
    }
  } x0d{nullptr, s};
  dmalloc(&x0d.p, nlanes * sizeof(double), "cudaMalloc x0");
  ck(cudaMemcpyAsync(x0d.p, x0, nlanes * sizeof(double), cudaMemcpyHostToDevice, s),
     "upload x0");
  launch_prbg_init(b.state, d_lc, x0d.p, nlanes, s);
  ck(cudaGetLastError(), "prbg_init launch");
  ck(cudaMemcpyAsync(b.verified_end, b.state, nlanes * sizeof(double),
                     cudaMemcpyDeviceToDevice, s), "copy state");
  ck(cudaStreamSynchronize(s), "prbg_init");
}

void free_lasm(LasmBuffers& b, cudaStream_t s = nullptr) {
  dfree(b.state, s);
  dfree(b.mu, s);
  for (auto& o : b.orbit) dfree(o, s);
  b = LasmBuffers{};
}
}  // namespace

void Generator::init(const std::vector<WorkerLanes>& lanes, MapKind kind, cudaStream_t s,
                     uint32_t orbit_iters, bool dense) {
  release();
  kind_ = kind;
  chains_ = 0;
  last_iters_ = 0;
  nl_ = uint32_t(2 * lanes.size());
  if (kind_ == MapKind::Plcm) {
    std::vector<LaneConst> lc(nl_);
    std::vector<double> x0(nl_);
    for (size_t i = 0; i < lanes.size(); ++i) {
      lc[2 * i] = make_lane_const(lanes[i].a.p);
      lc[2 * i + 1] = make_lane_const(lanes[i].b.p);
      x0[2 * i] = lanes[i].a.x0;
      x0[2 * i + 1] = lanes[i].b.x0;
    }
    pb_ = alloc_prbg(nl_, s, orbit_iters, dense);
    dmalloc(&d_lc_, nl_ * sizeof(LaneConst), "cudaMalloc lanes");
    ck(cudaMemcpyAsync(d_lc_, lc.data(), nl_ * sizeof(LaneConst), cudaMemcpyHostToDevice, s),
       "upload lanes");
    init_prbg(pb_, d_lc_, x0.data(), nl_, s);
    return;
  }
  std::vector<double> mu(nl_);
  std::vector<double2> xy0(nl_);
  for (size_t i = 0; i < lanes.size(); ++i) {
    mu[2 * i] = lanes[i].la.mu;
    mu[2 * i + 1] = lanes[i].lb.mu;
    xy0[2 * i] = make_double2(lanes[i].la.x0, lanes[i].la.y0);
    xy0[2 * i + 1] = make_double2(lanes[i].lb.x0, lanes[i].lb.y0);
  }
  struct Staging {  // freed on every path, once the stream is done with it
    double2* p = nullptr;
    cudaStream_t s;
    ~Staging() {
      if (p) cudaStreamSynchronize(s);
      dfree(p);
    }
  } d_xy0{nullptr, s};
  dmalloc(&lb_.state, nl_ * sizeof(double2), "cudaMalloc lasm state");
  dmalloc(&lb_.mu, nl_ * sizeof(double), "cudaMalloc lasm mu");
  dmalloc(&d_xy0.p, nl_ * sizeof(double2), "cudaMalloc lasm x0");
  ck(cudaMemcpyAsync(lb_.mu, mu.data(), nl_ * sizeof(double), cudaMemcpyHostToDevice, s),
     "upload mu");
  ck(cudaMemcpyAsync(d_xy0.p, xy0.data(), nl_ * sizeof(double2), cudaMemcpyHostToDevice, s),
     "upload x0");
  launch_lasm_init(lb_.state, lb_.mu, d_xy0.p, nl_, s);
  ck(cudaGetLastError(), "lasm_init launch");
  if (orbit_iters) resize(orbit_iters);
  ck(cudaStreamSynchronize(s), "lasm_init");
}

void Generator::release(cudaStream_t after) noexcept {
  free_prbg(pb_, after);
  dfree(d_lc_, after);
  d_lc_ = nullptr;
  free_lasm(lb_, after);
}

uint32_t Generator::orbit_cap_iters() const {
  // orbit bytes per iteration: LASM keeps every (x, y); PLCM one 8-byte
  // checkpoint per 8 iterations (or every value, dense)
  const uint64_t per = (kind_ == MapKind::Lasm ? 16ull : pb_.dense ? 8ull : 1ull) * nl_;
  const uint64_t iters = std::min<uint64_t>(kOrbitBytes / per, 1u << 20) / 8 * 8;
  return uint32_t(std::max<uint64_t>(iters, 8));
}

void Generator::resize(uint32_t iters) {
  if (kind_ == MapKind::Plcm) {
    resize_orbit(pb_, nl_, iters);
    return;
  }
  for (auto& o : lb_.orbit) {
    dfree(o);
    o = nullptr;
  }
  lb_.max_iters = 0;
  for (auto& o : lb_.orbit)
    dmalloc(&o, uint64_t(iters) * nl_ * sizeof(double2), "cudaMalloc lasm orbit");
  lb_.max_iters = iters;
}

void Generator::chain(int slot, uint32_t iters, cudaStream_t s) {
  if (kind_ == MapKind::Plcm)
    launch_prbg_chain(pb_, slot, d_lc_, iters, nl_, chains_, last_iters_, s);
  else
    launch_lasm_chain(lb_, slot, iters, nl_, s);
  ck(cudaGetLastError(), "generator chain launch");
  launch_of_[slot & 1] = chains_;
  ++chains_;
  last_iters_ = iters;
}

void Generator::emit(int slot, uint8_t* ring, uint64_t ring_bytes, uint64_t it0,
                     uint32_t iters, cudaStream_t s) {
  if (kind_ == MapKind::Plcm)
    launch_prbg_verify(pb_, slot, d_lc_, ring, ring_bytes, it0, iters, nl_, launch_of_[slot & 1],
                       s);
  else
    launch_lasm_emit(lb_, slot, ring, ring_bytes, it0, iters, nl_, s);
  ck(cudaGetLastError(), "generator emit launch");
}

uint64_t Generator::replays() {
  if (kind_ != MapKind::Plcm || !pb_.replays) return 0;
  unsigned long long rep = 0;
  ck(cudaMemcpy(&rep, pb_.replays, sizeof rep, cudaMemcpyDeviceToHost), "stats");
  return rep;
}

namespace {
std::atomic<int> g_streams{0};  // 0: not yet read from the environment
std::atomic<int> g_fusion{-1};  // -1: not yet read from the environment
}

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

void set_streams_per_handle(int n) {
  if (n != 1 && n != 2) raise(Errc::invalid_argument, "streams per handle must be 1 or 2");
  g_streams.store(n);
}

int streams_per_handle() {
  int v = g_streams.load();
  if (v == 0) {
    const char* e = std::getenv("CVE_B200_STREAMS_PER_HANDLE");
    v = (e && std::atoi(e) == 1) ? 1 : 2;
    int expected = 0;
    if (!g_streams.compare_exchange_strong(expected, v)) v = expected;
  }
  return v;
}

void set_round_fusion(int mode) {
  if (mode < 0 || mode > 1) raise(Errc::invalid_argument, "round fusion mode must be 0 or 1");
  g_fusion.store(mode);
}

int round_fusion() {
  int v = g_fusion.load();
  if (v < 0) {
    const char* e = std::getenv("CVE_B200_ROUND_FUSION");
    v = e ? std::atoi(e) : 0;
    if (v < 0 || v > 1) v = 0;
    int expected = -1;
    if (!g_fusion.compare_exchange_strong(expected, v)) v = expected;
  }
  return v;
}

void configure_kernels_once(int device) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(device)) return;
  DeviceScope scope(device);
  configure_prbg_kernels();
  configure_cipher_kernels();
  configure_rows_kernels();
  ck(cudaGetLastError(), "kernel attributes");
  done.insert(device);
}

DeviceScope::DeviceScope(int dev) {
  if (cudaGetDevice(&prev) != cudaSuccess) {
    cudaGetLastError();
    prev = -1;
    return;
  }
  if (prev != dev && cudaSetDevice(dev) != cudaSuccess)
    raise(Errc::internal, "cannot select the handle's CUDA device");
}

DeviceScope::~DeviceScope() {
  if (prev >= 0) cudaSetDevice(prev);
}

cudaEvent_t EventPool::get(bool timing) {
  auto& v = timing ? timed_ : plain_;
  if (!v.empty()) {
    cudaEvent_t e = v.back();
    v.pop_back();
    return e;
  }
  DeviceScope scope(dev_);
  cudaEvent_t e;
  ck(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming),
     "cudaEventCreate");
  return e;
}

void EventPool::release() noexcept {
  for (cudaEvent_t e : plain_) cudaEventDestroy(e);
  for (cudaEvent_t e : timed_) cudaEventDestroy(e);
  plain_.clear();
  timed_.clear();
}

void CipherCtx::ensure_copy_streams() {
  if (s_h2d) return;
  s_h2d = stream_get();
  s_d2h = stream_get();
}

void CipherCtx::sync() {
  for (cudaStream_t s : {s_h2d, s_work, s_d2h})
    if (s) ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

void CipherCtx::ensure_buffers(const Geom& g, uint32_t nslots) {
  const uint64_t fb = g.frame_bytes;
  const uint64_t scratch_need =
      round_up(fb, 256) + 4 * uint64_t(g.n) * ((g.region + 4095) / 4096) + 256;
  const bool generic = !plan_encrypt(g).fused;
  if (scratch_bytes < scratch_need || (generic && !scratch[2])) {
    sync();
    dfree(scratch[0]);  // scratch[1] lives in the same allocation
    dfree(scratch[2]);
    for (auto& p : scratch) p = nullptr;
    scratch_bytes = 0;
    // the two ping-pong frames of the middle rounds in one allocation, so one
    // L2 access-policy window can cover both
    dmalloc(&scratch[0], 2 * scratch_need, "cudaMalloc scratch");
    scratch[1] = scratch[0] + scratch_need;
    if (generic) dmalloc(&scratch[2], scratch_need, "cudaMalloc scratch");
    scratch_bytes = scratch_need;
    set_l2_window();
  }
  if (shift_cap < g.side) {
    sync();
    dfree(d_shift);
    d_shift = nullptr;
    shift_cap = 0;
    dmalloc(&d_shift, sizeof(int32_t) * g.side, "cudaMalloc shift");
    shift_cap = g.side;
  }
  if (!d_gbar) dmalloc(&d_gbar, 256, "cudaMalloc grid barrier");
  if (nslots && (slots.size() < nslots || slot_bytes < fb)) {
    sync();
    for (uint8_t* p : slots) dfree(p);
    slots.assign(nslots, nullptr);
    slot_bytes = 0;
    for (auto& p : slots) dmalloc(&p, fb, "cudaMalloc frame slot");
    slot_bytes = fb;
    while (slot_free.size() < nslots) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventRecord(e, s_d2h), "cudaEventRecord");
      slot_free.push_back(e);
    }
  }
}

// Experiment ($CVE_B200_L2_WINDOW=1): an L2 access-policy window marking the
// two scratch frames persisting on the rounds stream (the middle rounds
// read and write them; the keystream streams through evict-first).
void CipherCtx::set_l2_window() {
  static const bool on = [] {
    const char* e = std::getenv("CVE_B200_L2_WINDOW");
    return e && std::atoi(e) == 1;
  }();
  if (!on || !s_work || !scratch[0]) return;
  int max_win = 0, max_persist = 0;
  if (cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
      max_win <= 0 || max_persist <= 0) {
    cudaGetLastError();
    return;
  }
  const uint64_t bytes = std::min<uint64_t>(2 * scratch_bytes, uint64_t(max_win));
  const uint64_t persist = std::min<uint64_t>(bytes, uint64_t(max_persist));
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = scratch[0];
  v.accessPolicyWindow.num_bytes = bytes;
  v.accessPolicyWindow.hitRatio = float(double(persist) / double(bytes));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(s_work, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

void CipherCtx::ensure_windows(uint64_t bytes_per_worker, uint32_t workers) {
  const uint64_t need = bytes_per_worker * workers;
  if (win_bytes >= need) return;
  sync();
  for (auto& w : win) {
    dfree(w);
    w = nullptr;
  }
  win_bytes = 0;
  for (auto& w : win) dmalloc(&w, need, "cudaMalloc keystream window");
  win_bytes = need;
  for (auto& e : win_free) {
    if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(e, s_work), "cudaEventRecord");
  }
}

const double* CipherCtx::sine_for(uint32_t side) {
  auto it = sines.find(side);
  if (it != sines.end()) return it->second;
  const std::vector<double> sv = sine_table(side);
  double* d = nullptr;
  dmalloc(&d, sizeof(double) * side, "cudaMalloc sine");
  sines[side] = d;
  // ordered before k_shift, which runs on s_work
  // (pageable source: the call returns once the bytes are staged)
  ck(cudaMemcpyAsync(d, sv.data(), sizeof(double) * side, cudaMemcpyHostToDevice, s_work),
     "upload sine");
  return d;
}

void CipherCtx::release() noexcept {
  int prev = -1;  // everything below belongs to `dev` (stream pools are per device)
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != dev) cudaSetDevice(dev);
  cudaStream_t fin = s_work;
  for (cudaStream_t s : {s_h2d, s_d2h}) {
    if (!s) continue;
    cudaEvent_t e = nullptr;
    if (fin && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventRecord(e, s) == cudaSuccess && cudaStreamWaitEvent(fin, e, 0) == cudaSuccess) {
      cudaEventDestroy(e);
    } else {
      if (e) cudaEventDestroy(e);
      cudaStreamSynchronize(s);
    }
  }
  for (cudaEvent_t e : slot_free) cudaEventDestroy(e);
  slot_free.clear();
  for (auto& e : win_free) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  for (uint8_t* p : slots) dfree(p, fin);
  slots.clear();
  for (auto& w : win) {
    dfree(w, fin);
    w = nullptr;
  }
  for (auto& kv : sines) dfree(kv.second, fin);
  sines.clear();
  dfree(scratch[0], fin);  // scratch[1] lives in the same allocation
  dfree(scratch[2], fin);
  for (uint8_t*& p : scratch) p = nullptr;
  dfree(d_shift, fin);
  d_shift = nullptr;
  dfree(d_gbar, fin);
  d_gbar = nullptr;
  events.release();
  for (cudaStream_t s : {owns_work ? s_work : nullptr, s_h2d, s_d2h}) stream_put(s);
  s_work = s_h2d = s_d2h = nullptr;
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
}

Engine::Engine(const Key& key, uint32_t workers, uint32_t rounds, int device)
    : Engine(key, workers, rounds, std::vector<int>{device}) {}

Engine::Engine(const Key& key, uint32_t workers, uint32_t rounds,
               const std::vector<int>& devices)
    : key_(key), n_(workers), r_(rounds), dev_(devices.empty() ? 0 : devices[0]), coord_(key) {
  // engine.cpp:168-179: coordinator first, then workers/rounds checks.
  if (workers == 0) raise(Errc::invalid_argument, "workers must be >= 1");
  if (rounds == 0 || rounds > 255)
    raise(Errc::invalid_argument, "rounds must be in 1..255");
  if (devices.empty()) raise(Errc::invalid_argument, "no device given");
  const std::vector<WorkerLanes> lanes = coord_.derive_workers(n_);

  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    raise(Errc::internal, "no CUDA device: the B200 engine has no CPU path");
  for (int d : devices) {
    if (d < 0 || d >= count) raise(Errc::invalid_argument, "device index out of range");
    int major = 0;
    ck(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d), "device query");
    if (major != 10) {
      cudaDeviceProp prop{};
      cudaGetDeviceProperties(&prop, d);
      raise(Errc::internal, std::string("engine is built for sm_100a; device is ") + prop.name);
    }
  }
  if (const char* e = std::getenv("CVE_B200_GEN_CHUNK")) {  // experiments only; 0 = unset
    const uint64_t v = std::strtoull(e, nullptr, 10) / 8 * 8;
    if (v) gen_chunk_cap_ = v;
  }
  one_stream_ = streams_per_handle() == 1;
  fuse_rounds_ = round_fusion() == 1;
  try {
    for (int d : devices) configure_kernels_once(d);
    DeviceScope scope(dev_);  // the caller's device is restored on return
    acquire(lanes);
    init(devices);
  } catch (...) {
    release();  // the destructor does not run for a throwing constructor
    throw;
  }
}

void Engine::acquire(const std::vector<WorkerLanes>& lanes) {
  gen_events_ = std::make_unique<EventPool>(dev_);
  s_gen_ = stream_get();
  for (auto& e : ver_done_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (auto& e : chain_done_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  s_work_ = stream_get();
  // Verification runs on s_work: every frame's rounds wait for their
  // keystream's verify anyway, and a device-API handle then occupies two
  // hardware queues, so 16 concurrent handles fit CUDA_DEVICE_MAX_CONNECTIONS
  // = 32 without sharing a queue with another handle's long chain launches.
  if (one_stream_) {  // generator on the rounds stream too: one hardware queue per handle
    stream_put(s_gen_);
    s_gen_ = s_work_;
  }

  // dense orbit in the many-clips configuration (one stream per handle):
  // the verifier then streams the orbit instead of regenerating it, which
  // leaves SM issue slots to the other clips' kernels
  bool dense = one_stream_;
  if (const char* e = std::getenv("CVE_B200_DENSE")) dense = std::atoi(e) != 0;  // experiments only
  gen_.init(lanes, key_.kind, s_gen_, 0, dense);  // orbit buffers sized by ensure_ring
  bpi_ = gen_.bytes_per_iter();
  ++st_.kernel_launches;
}

// Cipher contexts: the handle's own device (rounds share s_work with the
// verifier), or one shard per entry of `devices` with its own streams.
void Engine::init(const std::vector<int>& devices) {
  if (devices.size() == 1) {
    local_ = std::make_unique<CipherCtx>(dev_);
    local_->s_work = s_work_;
    return;
  }
  for (int d : devices) {
    grant_peer_access(dev_, d);  // the shard reads the generator's ring
    if (d != dev_) {
      DeviceScope scope(d);
      const cudaError_t e = cudaDeviceEnablePeerAccess(dev_, 0);
      if (e != cudaSuccess) cudaGetLastError();  // already enabled / not capable: copies still work
    }
    DeviceScope scope(d);
    auto c = std::make_unique<CipherCtx>(d);
    c->s_work = stream_get();
    c->owns_work = true;
    shards_.push_back(std::move(c));
  }
}

Engine::~Engine() { release(); }

// Frees everything the engine holds; safe on a partially constructed engine
// and idempotent.  Restores the caller's device.
void Engine::release() noexcept {
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  cudaSetDevice(dev_);
  // Asynchronous teardown: work still queued -- typically the generator's
  // run-ahead for a next frame that will never come -- finishes on the
  // device, and every buffer goes back to the pool in stream order after it,
  // so destroying a handle does not wait for it.  `fin` joins every stream.
  cudaStream_t fin = s_work_;
  std::vector<cudaStream_t> others = {s_gen_};
  if (local_) others.insert(others.end(), {local_->s_h2d, local_->s_d2h});
  for (cudaStream_t s : others) {
    if (!s || s == fin) continue;
    cudaEvent_t e = nullptr;
    if (fin && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventRecord(e, s) == cudaSuccess && cudaStreamWaitEvent(fin, e, 0) == cudaSuccess) {
      cudaEventDestroy(e);
    } else {
      if (e) cudaEventDestroy(e);
      cudaStreamSynchronize(s);
    }
  }
  for (auto& c : consumers_) {
    // a shard's last window copy out of the ring must finish before the
    // ring is freed behind `fin`
    if (fin && c.pool->device() != dev_ && cudaStreamWaitEvent(fin, c.done, 0) != cudaSuccess)
      cudaDeviceSynchronize();
    c.pool->put(c.done);
  }
  consumers_.clear();
  for (auto& c : shards_) c->release();  // each in its own stream order
  cudaSetDevice(dev_);
  for (auto& e : ver_done_) {
    if (e) cudaEventDestroy(e);  // pending events are released once complete
    e = nullptr;
  }
  for (auto& e : chain_done_) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  for (auto& g : gens_) gen_events_->put(g.ev);
  gens_.clear();
  for (auto& t : timed_) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  timed_.clear();
  if (local_) {
    local_->s_work = s_work_;  // freed below, in the order of s_work_
    local_->release();
    local_.reset();
  }
  shards_.clear();
  if (gen_events_) gen_events_->release();
  dfree(ring_, fin);
  ring_ = nullptr;
  gen_.release(fin);
  for (cudaStream_t s : {s_gen_ == s_work_ ? nullptr : s_gen_, s_work_}) stream_put(s);
  s_gen_ = s_work_ = nullptr;
  if (prev >= 0) cudaSetDevice(prev);
}

Geom Engine::geometry(uint32_t side) const {
  Geom g;
  g.side = side;
  g.n = n_;
  g.rows = side / n_;
  g.region = uint64_t(g.rows) * side * 3;
  g.frame_bytes = uint64_t(side) * side * 3;
  return g;
}

// Seed drawn before the side check, like Engine::encrypt (engine.cpp:293-296)
// followed by check_frame (engine.cpp:189-196).  Returns nothing useful; the
// seeds are drawn again per frame by the caller after this check passes.
uint32_t Engine::draw_and_check(uint32_t side, uint32_t count) {
  (void)count;
  if (side % n_ != 0) {
    coord_.next_seed();
    raise(Errc::mismatch, "frame side is not divisible by the worker count");
  }
  if (side > 65536) {
    coord_.next_seed();
    raise(Errc::invalid_argument, "frame side above 65536 is not supported");
  }
  return 0;
}

void Engine::timed_begin(EventPool& pool, cudaStream_t s, bool chain, bool verify) {
  Timed t{};
  t.a = pool.get(true);
  t.b = pool.get(true);
  t.pool = &pool;
  t.chain = chain;
  t.verify = verify;
  ck(cudaEventRecord(t.a, s), "cudaEventRecord");
  open_ = t;
}

void Engine::timed_end(cudaStream_t s) {
  ck(cudaEventRecord(open_.b, s), "cudaEventRecord");
  timed_.push_back(open_);
  open_ = Timed{};
  if (timed_.size() > 256) fold_timings(false);
}

void Engine::fold_timings(bool wait) {
  std::vector<Timed> keep;
  for (auto& t : timed_) {
    if (!wait && cudaEventQuery(t.b) != cudaSuccess) {
      keep.push_back(t);
      continue;
    }
    float ms = 0;
    ck(cudaEventSynchronize(t.b), "timing event");
    ck(cudaEventElapsedTime(&ms, t.a, t.b), "cudaEventElapsedTime");
    if (t.chain) {
      st_.prbg_ms += ms;
      st_.chain_ms += ms;
      if (prbg_times_.size() < (1u << 20)) prbg_times_.push_back(ms);
    } else if (t.verify) {
      st_.prbg_ms += ms;
    } else {
      st_.cipher_ms += ms;
    }
    t.pool->put(t.a, true);
    t.pool->put(t.b, true);
  }
  cudaGetLastError();  // cudaErrorNotReady from the queries is not an error
  timed_.swap(keep);
}

// Ring of >= 4 frames of keystream per worker, so the generator can run one
// frame ahead while up to two frames are still being ciphered.
void Engine::ensure_ring(uint64_t need) {
  NvtxRange nvtx("cve: keystream ring grow");
  if (ring_bytes_ >= 4 * need) return;
  const uint64_t want = round_up(4 * need + 48 * 1024, 48 * 1024);
  synchronize();
  uint8_t* fresh = nullptr;
  dmalloc(&fresh, want * n_, "cudaMalloc keystream ring");
  const uint64_t gen_bytes = gen_iters_ * bpi_;
  if (ring_ && gen_bytes > cons_) {
    launch_ring_move(ring_, ring_bytes_, fresh, want, cons_, gen_bytes, n_, s_gen_);
    ++st_.kernel_launches;
    ck(cudaStreamSynchronize(s_gen_), "ring move");
  }
  dfree(ring_);
  ring_ = fresh;
  ring_bytes_ = want;
  // orbit buffers for the longest launch gen_until will issue (a quarter of
  // the ring), within the orbit budget: a small clip holds MBs, not 256 MB
  const uint32_t cap = gen_.orbit_cap_iters();
  const uint64_t launch = std::max<uint64_t>(8, ring_bytes_ / 4 / bpi_ / 8 * 8);
  const uint32_t iters = uint32_t(std::min<uint64_t>(launch, cap));
  if (iters > gen_.max_iters()) gen_.resize(iters);
  for (auto& c : consumers_) c.pool->put(c.done);
  consumers_.clear();
  for (auto& g : gens_) gen_events_->put(g.ev);
  gens_.clear();
}

// Enqueue generator launches on s_gen until stream byte `end_byte` (per
// worker) is produced.  Launches cover whole 8-iteration (48-byte) blocks.
// Runs on dev_ (the caller's scope).
void Engine::gen_until(uint64_t end_byte) {
  NvtxRange nvtx("cve: generator launches");
  uint64_t target = round_up((end_byte + bpi_ - 1) / bpi_, 8);
  // never produce beyond what the ring can hold ahead of unassigned bytes
  const uint64_t cap = (cons_ + ring_bytes_) / bpi_ / 8 * 8;
  target = std::min(target, cap);
  while (gen_iters_ < target) {
    uint64_t chunk = target - gen_iters_;
    uint64_t max_chunk = std::max<uint64_t>(8, ring_bytes_ / 4 / bpi_ / 8 * 8);
    if (gen_chunk_cap_) max_chunk = std::min(max_chunk, gen_chunk_cap_);
    chunk = std::min<uint64_t>({chunk, max_chunk, uint64_t(gen_.max_iters())});
    if (chunk == 0) raise(Errc::internal, "generator launch without orbit buffers");
    const int slot = int(launches_ & 1);
    // (1) chain on s_gen, once the verifier is done with this slot's buffers
    if (launches_ >= 2) ck(cudaStreamWaitEvent(s_gen_, ver_done_[slot], 0), "wait slot");
    timed_begin(*gen_events_, s_gen_, true);
    gen_.chain(slot, uint32_t(chunk), s_gen_);
    timed_end(s_gen_);
    ck(cudaEventRecord(chain_done_[slot], s_gen_), "cudaEventRecord");
    // (2)+(3) verify, emit, fix up on s_work while the next chain runs.
    // Ring bytes below write_end - R get overwritten: their readers must be
    // done (the rounds of a single-device handle, the window copies of a
    // sharded one).
    ck(cudaStreamWaitEvent(s_work_, chain_done_[slot], 0), "wait chain");
    const uint64_t write_end = (gen_iters_ + chunk) * bpi_;
    if (write_end > ring_bytes_) {
      const uint64_t dead = write_end - ring_bytes_;
      while (!consumers_.empty() && consumers_.front().lo < dead) {
        ck(cudaStreamWaitEvent(s_work_, consumers_.front().done, 0), "wait");
        if (consumers_.front().hi <= dead) {
          consumers_.front().pool->put(consumers_.front().done);
          consumers_.pop_front();
        } else {
          break;
        }
      }
    }
    timed_begin(*gen_events_, s_work_, false, true);
    gen_.emit(slot, ring_, ring_bytes_, gen_iters_, uint32_t(chunk), s_work_);
    timed_end(s_work_);
    ck(cudaEventRecord(ver_done_[slot], s_work_), "cudaEventRecord");
    st_.kernel_launches += gen_.kernels_per_launch();
    ++st_.prbg_launches;
    ++launches_;
    gen_iters_ += chunk;
    st_.keystream_iters += chunk;
    GenMark m{gen_iters_ * bpi_, gen_events_->get()};
    ck(cudaEventRecord(m.ev, s_work_), "cudaEventRecord");
    gens_.push_back(m);
  }
}

cudaEvent_t Engine::gen_event_covering(uint64_t end_byte) {
  while (!gens_.empty() && gens_.front().end_byte < end_byte) {
    gen_events_->put(gens_.front().ev);
    gens_.pop_front();
  }
  return gens_.empty() ? nullptr : gens_.front().ev;  // null: already synced
}

// K4 + r rounds of one frame on c.s_work, which already waits for the
// frame's input and keystream.  Round 0 reads buf; middle rounds ping-pong
// the two scratch frames; the last round writes buf (r == 1 goes through
// scratch and a copy).  The generic encrypt path stages y in a third
// scratch frame.
cudaEvent_t Engine::enqueue_rounds(CipherCtx& c, uint8_t* buf, const Geom& g, uint32_t seed,
                                   bool decrypt, KsWindow ks) {
  timed_begin(c.events, c.s_work, false, false);
  // K2r (rows.cu) for the forward rounds where it applies: 16-byte aligned
  // frames and keystream, side % 16 == 0 (every benchmark config).  It forms
  // the frame's shifts itself (sine table and seed), so K4 runs only for the
  // other round kernels.
  RowPlan rplan{};
  const bool rows = !decrypt && !fuse_rounds_ && plan_rows_encrypt(g, rplan) &&
                    ks.pos % 16 == 0 && ks.ring_bytes % 16 == 0 &&
                    ((reinterpret_cast<uintptr_t>(buf) | reinterpret_cast<uintptr_t>(ks.ring) |
                      reinterpret_cast<uintptr_t>(c.scratch[0]) |
                      reinterpret_cast<uintptr_t>(c.scratch[1])) % 16 == 0);
  if (!rows) {
    launch_shift_table(c.sine_for(g.side), seed, c.d_shift, g.side, c.s_work);
    ++st_.kernel_launches;
  }
  const uint64_t base = ks.pos;
  // K2r with every round in one cooperative launch, opt-in
  // (CVE_B200_ROWS_PERSIST=1): a grid barrier per round costs more than the
  // programmatic-dependent launches it replaces (C1 34 -> 40, C4 72 -> 74 us
  // per frame; DESIGN 6a)
  if (rows && c.d_gbar && std::getenv("CVE_B200_ROWS_PERSIST") &&
      launch_encrypt_frame_rows(rplan, g, buf, c.scratch[0], c.scratch[1], ks, c.sine_for(g.side),
                                seed, r_, c.d_gbar, c.s_work)) {
    ++st_.kernel_launches;
    timed_end(c.s_work);
    cudaEvent_t done = c.events.get();
    ck(cudaEventRecord(done, c.s_work), "cudaEventRecord");
    ++st_.frames;
    return done;
  }
  if (!decrypt && fuse_rounds_ &&
      launch_encrypt_frame(g, buf, ks, c.d_shift, r_, c.s_work, &st_.kernel_launches)) {
    timed_end(c.s_work);  // K6: every round in one cluster kernel
    cudaEvent_t done = c.events.get();
    ck(cudaEventRecord(done, c.s_work), "cudaEventRecord");
    ++st_.frames;
    return done;
  }
  const EncPlan plan = decrypt ? EncPlan{} : plan_encrypt(g);
  // K3r (rows.cu) for the inverse rounds: opt-in (CVE_B200_ROWS_DECRYPT=1).
  // Alone it matches K3t (1920^2: 14.8 vs 14.1 us per round, 768^2: 7.4 vs
  // 8.5), chained in a frame it is slower (768^2: 46 vs 36 us per frame).
  RowPlan dplan{};
  const bool drows = decrypt && std::getenv("CVE_B200_ROWS_DECRYPT") && plan_rows_decrypt(g, dplan) &&
                     ks.pos % 16 == 0 && ks.ring_bytes % 48 == 0 &&
                     ks.ring_bytes < (uint64_t(1) << 31) &&
                     ((reinterpret_cast<uintptr_t>(buf) | reinterpret_cast<uintptr_t>(ks.ring) |
                       reinterpret_cast<uintptr_t>(c.scratch[0]) |
                       reinterpret_cast<uintptr_t>(c.scratch[1])) % 16 == 0);
  const double* sine = c.sine_for(g.side);
  const uint8_t* src = buf;
  for (uint32_t step = 0; step < r_; ++step) {
    const uint32_t k = decrypt ? r_ - 1 - step : step;
    uint8_t* dst = (step + 1 == r_ && r_ > 1)
                       ? buf
                       : (src == c.scratch[0] ? c.scratch[1] : c.scratch[0]);
    ks.pos = (base + uint64_t(k) * g.region) % ks.ring_bytes;
    if (drows) {
      launch_decrypt_round_rows(dplan, g, src, dst, ks, c.d_shift, c.s_work);
      ++st_.kernel_launches;
    } else if (decrypt) {
      launch_decrypt_round(g, src, dst, ks, c.d_shift, c.s_work, &st_.kernel_launches);
    } else if (rows) {
      launch_encrypt_round_rows(rplan, g, src, dst, ks, sine, seed, c.s_work, step > 0);
      ++st_.kernel_launches;
    } else {
      launch_encrypt_round(plan, g, src, dst, ks, c.d_shift, c.scratch[2], c.s_work,
                           &st_.kernel_launches);
    }
    src = dst;
  }
  if (r_ == 1)
    ck(cudaMemcpyAsync(buf, src, g.frame_bytes, cudaMemcpyDeviceToDevice, c.s_work), "d2d");
  timed_end(c.s_work);
  cudaEvent_t done = c.events.get();
  ck(cudaEventRecord(done, c.s_work), "cudaEventRecord");
  ++st_.frames;
  return done;
}

// Run-ahead: start the next frame's keystream behind this one's, so a
// caller's next call finds it (partly) generated.  Not after a handle's
// first frame: a one-frame clip (BASELINE config C1) would leave a whole
// frame of chain + verify work running after it is destroyed, where the
// next clip's work collides with it.  From the second frame on the clip is
// a stream of frames and the run-ahead pays.
void Engine::after_frame(uint64_t need) {
  if (st_.frames >= 2) gen_until(cons_ + need);
}

cudaEvent_t Engine::enqueue_frame(uint8_t* buf, const Geom& g, uint32_t seed, bool decrypt) {
  NvtxRange nvtx("cve: frame");
  const uint64_t need = uint64_t(r_) * g.region;
  const uint64_t lo = cons_;
  cons_ += need;
  gen_until(lo + need);
  if (cudaEvent_t ge = gen_event_covering(lo + need))
    ck(cudaStreamWaitEvent(s_work_, ge, 0), "wait keystream");
  cudaEvent_t done =
      enqueue_rounds(*local_, buf, g, seed, decrypt, KsWindow{ring_, ring_bytes_, lo % ring_bytes_});
  // the rounds read the ring: they are its consumer
  consumers_.push_back(Consumer{lo, lo + need, done, &local_->events});
  after_frame(need);
  return done;
}

// Copies `rows` rows of `width` bytes between (possibly different) devices.
static void copy_rows(uint8_t* dst, uint64_t dpitch, int ddev, const uint8_t* src, uint64_t spitch,
               int sdev, uint64_t width, uint32_t rows, cudaStream_t s) {
  if (ddev == sdev) {
    ck(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToDevice, s),
       "keystream window copy");
    return;
  }
  cudaMemcpy3DPeerParms p{};
  p.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(src), spitch, width, rows);
  p.srcDevice = sdev;
  p.dstPtr = make_cudaPitchedPtr(dst, dpitch, width, rows);
  p.dstDevice = ddev;
  p.extent = make_cudaExtent(width, rows, 1);
  ck(cudaMemcpy3DPeerAsync(&p, s), "keystream window peer copy");
}

cudaEvent_t Engine::enqueue_shard_frame(CipherCtx& c, uint8_t* buf, const Geom& g,
                                        uint32_t seed, bool decrypt) {
  NvtxRange nvtx("cve: frame (shard)");
  const uint64_t need = uint64_t(r_) * g.region;
  const uint64_t lo = cons_;
  cons_ += need;
  gen_until(lo + need);
  cudaEvent_t ge = gen_event_covering(lo + need);
  DeviceScope scope(c.dev);
  c.ensure_windows(need, n_);
  const uint32_t w = c.win_next;
  c.win_next = (c.win_next + 1) % CipherCtx::kWindows;
  ck(cudaStreamWaitEvent(c.s_work, c.win_free[w], 0), "wait window");
  if (ge) ck(cudaStreamWaitEvent(c.s_work, ge, 0), "wait keystream");
  // worker i's window = ring stream bytes [lo, lo + need), wrapping at most once
  const uint64_t pos = lo % ring_bytes_;
  const uint64_t first = std::min(need, ring_bytes_ - pos);
  copy_rows(c.win[w], need, c.dev, ring_ + pos, ring_bytes_, dev_, first, n_, c.s_work);
  if (first < need)
    copy_rows(c.win[w] + first, need, c.dev, ring_, ring_bytes_, dev_, need - first, n_,
              c.s_work);
  cudaEvent_t copied = c.events.get();
  ck(cudaEventRecord(copied, c.s_work), "cudaEventRecord");
  consumers_.push_back(Consumer{lo, lo + need, copied, &c.events});
  cudaEvent_t done = enqueue_rounds(c, buf, g, seed, decrypt, KsWindow{c.win[w], need, 0});
  ck(cudaEventRecord(c.win_free[w], c.s_work), "cudaEventRecord");
  return done;
}

void Engine::run_host(uint8_t* px, uint32_t side, uint32_t count, bool decrypt) {
  run_host_io(HostIo{px, side, side, px, side, side}, side, count, decrypt);
}

void Engine::run_host_io(const HostIo& io, uint32_t side, uint32_t count, bool decrypt) {
  NvtxRange nvtx("cve: frames (host buffers)");
  draw_and_check(side, count);
  if (io.in_w > side || io.in_h > side || io.out_w > side || io.out_h > side ||
      !io.in_w || !io.in_h || !io.out_w || !io.out_h)
    raise(Errc::invalid_argument, "frame region exceeds the padded side");
  const Geom g = geometry(side);
  ensure_ring(uint64_t(r_) * g.region);
  std::vector<CipherCtx*> ctxs;
  if (shards_.empty()) {
    ctxs.push_back(local_.get());
  } else {
    for (auto& c : shards_) ctxs.push_back(c.get());
  }
  for (CipherCtx* c : ctxs) {
    DeviceScope scope(c->dev);
    c->ensure_copy_streams();  // copy streams only for handles that use the host API
    c->ensure_buffers(g, kSlots);
  }
  const uint64_t row = uint64_t(side) * 3;
  const uint64_t in_fb = uint64_t(io.in_w) * io.in_h * 3;
  const uint64_t out_fb = uint64_t(io.out_w) * io.out_h * 3;

  for (uint32_t f = 0; f < count; ++f) {
    const uint32_t seed = coord_.next_seed();
    CipherCtx& c = shards_.empty() ? *local_ : *shards_[shard_rr_++ % shards_.size()];
    const uint32_t slot = c.slot_next;
    c.slot_next = (c.slot_next + 1) % kSlots;
    const uint8_t* hin = io.in + uint64_t(f) * in_fb;
    uint8_t* hout = io.out + uint64_t(f) * out_fb;
    uint8_t* dbuf = c.slots[slot];
    cudaEvent_t done;
    {
      DeviceScope scope(c.dev);
      ck(cudaStreamWaitEvent(c.s_h2d, c.slot_free[slot], 0), "wait slot");
      if (io.in_w == side && io.in_h == side) {
        ck(cudaMemcpyAsync(dbuf, hin, g.frame_bytes, cudaMemcpyHostToDevice, c.s_h2d), "H2D");
      } else {  // pad on the device: only the w*h payload crosses PCIe
        ck(cudaMemcpy2DAsync(dbuf, row, hin, uint64_t(io.in_w) * 3, uint64_t(io.in_w) * 3,
                             io.in_h, cudaMemcpyHostToDevice, c.s_h2d), "H2D 2D");
        if (io.in_w < side)
          ck(cudaMemset2DAsync(dbuf + uint64_t(io.in_w) * 3, row, 0,
                               uint64_t(side - io.in_w) * 3, io.in_h, c.s_h2d), "pad right");
        if (io.in_h < side)
          ck(cudaMemsetAsync(dbuf + uint64_t(io.in_h) * row, 0,
                             uint64_t(side - io.in_h) * row, c.s_h2d), "pad bottom");
      }
      cudaEvent_t in = c.events.get();
      ck(cudaEventRecord(in, c.s_h2d), "record");
      ck(cudaStreamWaitEvent(c.s_work, in, 0), "wait H2D");
      c.events.put(in);
    }
    if (shards_.empty()) {
      done = enqueue_frame(dbuf, g, seed, decrypt);  // the consumer list owns `done`
    } else {
      done = enqueue_shard_frame(c, dbuf, g, seed, decrypt);
      after_frame(uint64_t(r_) * g.region);
    }
    DeviceScope scope(c.dev);
    ck(cudaStreamWaitEvent(c.s_d2h, done, 0), "wait work");
    if (!shards_.empty()) c.events.put(done);
    if (io.out_w == side && io.out_h == side) {
      ck(cudaMemcpyAsync(hout, dbuf, g.frame_bytes, cudaMemcpyDeviceToHost, c.s_d2h), "D2H");
    } else {  // crop on the way out
      ck(cudaMemcpy2DAsync(hout, uint64_t(io.out_w) * 3, dbuf, row, uint64_t(io.out_w) * 3,
                           io.out_h, cudaMemcpyDeviceToHost, c.s_d2h), "D2H 2D");
    }
    ck(cudaEventRecord(c.slot_free[slot], c.s_d2h), "record");
  }
  for (CipherCtx* c : ctxs) ck(cudaStreamSynchronize(c->s_d2h), "frame pipeline");
}

void Engine::run_device(uint8_t* d_px, uint32_t side, uint32_t count,
                        bool decrypt, cudaStream_t user) {
  NvtxRange nvtx("cve: frames (device-resident)");
  if (!shards_.empty()) {
    // a sharded handle's frames live on all its devices: run_device_sharded
    raise(Errc::invalid_argument, "sharded handle: use the per-shard device API");
  }
  draw_and_check(side, count);
  const Geom g = geometry(side);
  ensure_ring(uint64_t(r_) * g.region);
  local_->ensure_buffers(g, 0);
  cudaEvent_t in = gen_events_->get();
  ck(cudaEventRecord(in, user), "record user stream");
  ck(cudaStreamWaitEvent(s_work_, in, 0), "wait user stream");
  gen_events_->put(in);
  cudaEvent_t done = nullptr;
  for (uint32_t f = 0; f < count; ++f) {
    const uint32_t seed = coord_.next_seed();
    done = enqueue_frame(d_px + uint64_t(f) * g.frame_bytes, g, seed, decrypt);
  }
  ck(cudaStreamWaitEvent(user, done, 0), "join user stream");
}

// Reference Engine::transform (engine.cpp:302-307 -> forward, 207-250): seed
// first, then the geometry check, the streams only when diffusion is on, and
// per round the confusion half (a -> b, swap), the diffusion half (a -> b,
// swap; s_d from the pre-diffusion snapshot a), then the callback.
void Engine::transform_host(uint8_t* px, uint32_t side, uint32_t rounds, bool confusion,
                            bool diffusion,
                            const std::function<void(uint32_t, const uint8_t*)>& per_round,
                            PhaseMs* t) {
  NvtxRange nvtx("cve: transform");
  if (!shards_.empty())
    raise(Errc::invalid_argument, "sharded handle: transform runs on single-device handles");
  draw_and_check(side, 1);
  const uint32_t seed = coord_.next_seed();
  const Geom g = geometry(side);
  CipherCtx& c = *local_;
  c.ensure_buffers(g, 0);
  using Clock = std::chrono::steady_clock;
  const auto since = [](Clock::time_point a) {
    return std::chrono::duration<double, std::milli>(Clock::now() - a).count();
  };
  const uint64_t need = diffusion ? uint64_t(rounds) * g.region : 0;
  uint64_t lo = 0;
  if (need) {
    const auto t0 = Clock::now();
    ensure_ring(need);
    lo = cons_;
    cons_ += need;
    gen_until(lo + need);
    if (cudaEvent_t ge = gen_event_covering(lo + need))
      ck(cudaStreamWaitEvent(c.s_work, ge, 0), "wait keystream");
    if (t) {
      ck(cudaStreamSynchronize(c.s_work), "keystream");
      t->bytegen_ms += since(t0);
    }
  }
  uint8_t* a = c.scratch[0];
  uint8_t* b = c.scratch[1];
  const uint64_t agg_off = round_up(g.frame_bytes, 256);
  ck(cudaMemcpyAsync(a, px, g.frame_bytes, cudaMemcpyHostToDevice, c.s_work), "H2D");
  if (confusion) {
    launch_shift_table(c.sine_for(side), seed, c.d_shift, side, c.s_work);
    ++st_.kernel_launches;
  }
  if (t) ck(cudaStreamSynchronize(c.s_work), "transform input");
  std::vector<uint8_t> state(per_round ? g.frame_bytes : 0);
  for (uint32_t k = 0; k < rounds; ++k) {
    if (confusion) {
      const auto t0 = Clock::now();
      launch_confuse_only(g, a, b, c.d_shift, c.s_work, &st_.kernel_launches);
      std::swap(a, b);
      if (t) {
        ck(cudaStreamSynchronize(c.s_work), "confusion");
        t->confuse_ms += since(t0);
      }
    }
    if (diffusion) {
      const auto t0 = Clock::now();
      const KsWindow ks{ring_, ring_bytes_, (lo + uint64_t(k) * g.region) % ring_bytes_};
      launch_diffuse_only(g, a, b, ks, reinterpret_cast<uint32_t*>(b + agg_off), c.s_work,
                          &st_.kernel_launches);
      std::swap(a, b);
      if (t) {
        ck(cudaStreamSynchronize(c.s_work), "diffusion");
        t->diffuse_ms += since(t0);
      }
    }
    if (per_round) {
      ck(cudaMemcpyAsync(state.data(), a, g.frame_bytes, cudaMemcpyDeviceToHost, c.s_work),
         "D2H");
      ck(cudaStreamSynchronize(c.s_work), "transform round");
      per_round(k + 1, state.data());
    }
  }
  ck(cudaMemcpyAsync(px, a, g.frame_bytes, cudaMemcpyDeviceToHost, c.s_work), "D2H");
  cudaEvent_t done = c.events.get();
  ck(cudaEventRecord(done, c.s_work), "cudaEventRecord");
  if (need) {
    consumers_.push_back(Consumer{lo, lo + need, done, &c.events});  // read the ring
  } else {
    c.events.put(done);
  }
  ck(cudaStreamSynchronize(c.s_work), "transform");
}

void Engine::run_device_sharded(uint8_t* const* shard_px, uint32_t side, uint32_t count,
                                bool decrypt, const cudaStream_t* users) {
  NvtxRange nvtx("cve: frames (device-resident, sharded)");
  if (shards_.empty()) {
    run_device(shard_px[0], side, count, decrypt, users ? users[0] : nullptr);
    return;
  }
  draw_and_check(side, count);
  const Geom g = geometry(side);
  ensure_ring(uint64_t(r_) * g.region);
  const uint32_t G = uint32_t(shards_.size());
  for (uint32_t i = 0; i < G && i < count; ++i) {
    CipherCtx& c = *shards_[i];
    DeviceScope scope(c.dev);
    c.ensure_buffers(g, 0);
    cudaEvent_t in = c.events.get();
    ck(cudaEventRecord(in, users ? users[i] : nullptr), "record user stream");
    ck(cudaStreamWaitEvent(c.s_work, in, 0), "wait user stream");
    c.events.put(in);
  }
  std::vector<cudaEvent_t> last(G, nullptr);
  for (uint32_t f = 0; f < count; ++f) {
    const uint32_t seed = coord_.next_seed();
    const uint32_t i = f % G;
    CipherCtx& c = *shards_[i];
    if (last[i]) c.events.put(last[i]);
    last[i] = enqueue_shard_frame(c, shard_px[i] + uint64_t(f / G) * g.frame_bytes, g, seed,
                                  decrypt);
    after_frame(uint64_t(r_) * g.region);
  }
  for (uint32_t i = 0; i < G; ++i) {
    if (!last[i]) continue;
    DeviceScope scope(shards_[i]->dev);
    ck(cudaStreamWaitEvent(users ? users[i] : nullptr, last[i], 0), "join user stream");
    shards_[i]->events.put(last[i]);
  }
}

void Engine::synchronize() {
  for (cudaStream_t s : {s_gen_, s_work_})
    if (s) ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  if (local_) local_->sync();
  for (auto& c : shards_) c->sync();
}

void Engine::peek(uint32_t worker, uint8_t* out, size_t len) {
  if (worker >= n_) raise(Errc::invalid_argument, "worker index out of range");
  if (len == 0) return;
  ensure_ring(std::max<uint64_t>(len, 48));
  if (len > ring_bytes_ / 2) raise(Errc::invalid_argument, "peek too long");
  gen_until(cons_ + len);
  synchronize();
  const uint64_t start = cons_ % ring_bytes_;
  const uint8_t* base = ring_ + uint64_t(worker) * ring_bytes_;
  const uint64_t first = std::min<uint64_t>(len, ring_bytes_ - start);
  ck(cudaMemcpy(out, base + start, first, cudaMemcpyDeviceToHost), "peek");
  if (first < len)
    ck(cudaMemcpy(out + first, base, len - first, cudaMemcpyDeviceToHost), "peek");
}

void Engine::prefetch(uint64_t bytes) {
  ensure_ring(std::max<uint64_t>(bytes, 48));
  gen_until(cons_ + bytes);
}

EngineStats Engine::stats() {
  synchronize();
  fold_timings(true);
  st_.guard_replays = gen_.replays();
  return st_;
}

std::vector<float> Engine::take_prbg_times() {
  synchronize();
  fold_timings(true);
  std::vector<float> out;
  out.swap(prbg_times_);
  return out;
}

namespace {
// The reference's Prbg{lane_a, lane_b}.take(len) (chaos.cpp:79-107, 143-153)
// on the GPU: explicit lanes, one worker.  The generator is pipelined like an
// Engine's: chain L+1 runs on one stream while launch L is verified and
// emitted on another.  launch_iters (0: as large as the orbit budget allows)
// caps the iterations per generator launch.
void standalone(const WorkerLanes& w, MapKind kind, uint8_t* out, size_t len,
                uint32_t launch_iters, uint64_t* replays, bool dense) {
  cudaStream_t sg = nullptr, sw = nullptr;
  cudaEvent_t chain_done[2] = {nullptr, nullptr}, ver_done[2] = {nullptr, nullptr};
  uint8_t* d_out = nullptr;
  Generator gen;
  auto cleanup = [&] {
    for (cudaStream_t s : {sg, sw})
      if (s) cudaStreamSynchronize(s);
    gen.release();
    dfree(d_out);
    for (auto* evs : {chain_done, ver_done})
      for (int k = 0; k < 2; ++k)
        if (evs[k]) cudaEventDestroy(evs[k]);
    stream_put(sg);
    stream_put(sw);
  };
  try {
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    configure_kernels_once(dev);
    sg = stream_get();
    sw = stream_get();
    for (auto* evs : {chain_done, ver_done})
      for (int k = 0; k < 2; ++k)
        ck(cudaEventCreateWithFlags(&evs[k], cudaEventDisableTiming), "cudaEventCreate");
    gen.init({w}, kind, sg, 0, dense);
    const uint32_t bpi = gen.bytes_per_iter();
    const uint64_t iters = round_up((len + bpi - 1) / bpi, 8);
    uint64_t chunk = std::min<uint64_t>(gen.orbit_cap_iters(), iters);
    if (launch_iters) chunk = std::min<uint64_t>(chunk, std::max<uint32_t>(8, launch_iters / 8 * 8));
    gen.resize(uint32_t(chunk));
    const uint64_t ring = iters * bpi;  // multiple of 48
    dmalloc(&d_out, ring, "cudaMalloc");
    uint64_t L = 0;
    for (uint64_t it = 0; it < iters; it += chunk, ++L) {
      const int slot = int(L & 1);
      const uint32_t n = uint32_t(std::min<uint64_t>(chunk, iters - it));
      if (L >= 2) ck(cudaStreamWaitEvent(sg, ver_done[slot], 0), "wait slot");
      gen.chain(slot, n, sg);
      ck(cudaEventRecord(chain_done[slot], sg), "record");
      ck(cudaStreamWaitEvent(sw, chain_done[slot], 0), "wait chain");
      gen.emit(slot, d_out, ring, it, n, sw);
      ck(cudaEventRecord(ver_done[slot], sw), "record");
    }
    ck(cudaStreamSynchronize(sw), "keystream");
    ck(cudaMemcpy(out, d_out, len, cudaMemcpyDeviceToHost), "download");
    if (replays) *replays = gen.replays();
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}
}  // namespace

void standalone_stream(const Lane& a, const Lane& b, uint8_t* out, size_t len,
                       uint32_t launch_iters, uint64_t* replays, bool dense) {
  if (replays) *replays = 0;
  if (len == 0) return;
  HostPrbg validate(a, b);  // domain checks (bad_key), cheap
  (void)validate;
  WorkerLanes w;
  w.a = a;
  w.b = b;
  standalone(w, MapKind::Plcm, out, len, launch_iters, replays, dense);
}

void standalone_stream(const LasmLane& a, const LasmLane& b, uint8_t* out, size_t len) {
  if (len == 0) return;
  check_lasm_lane(a);
  check_lasm_lane(b);
  WorkerLanes w;
  w.la = a;
  w.lb = b;
  standalone(w, MapKind::Lasm, out, len, 0, nullptr, false);
}

KeystreamSource::KeystreamSource(const std::vector<WorkerLanes>& lanes, MapKind kind,
                                 int device, uint64_t max_bytes)
    : n_(uint32_t(lanes.size())), dev_(device) {
  configure_kernels_once(device);
  DeviceScope scope(device);  // the caller's device is restored on return
  try {
    s_ = stream_get();
    gen_.init(lanes, kind, s_, 0);
    // chunks no longer than the whole request: a short export generates
    // (and allocates for) only what it returns
    const uint64_t bpi = gen_.bytes_per_iter();
    const uint64_t need = round_up((std::max<uint64_t>(max_bytes, 1) + bpi - 1) / bpi, 8);
    gen_.resize(uint32_t(std::min<uint64_t>(gen_.orbit_cap_iters(), need)));
    dmalloc(&d_buf_, chunk_bytes() * n_, "cudaMalloc keystream");
  } catch (...) {
    release();
    throw;
  }
}

KeystreamSource::~KeystreamSource() { release(); }

void KeystreamSource::release() noexcept {
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != dev_) cudaSetDevice(dev_);
  if (s_) cudaStreamSynchronize(s_);
  gen_.release();
  dfree(d_buf_);
  d_buf_ = nullptr;
  stream_put(s_);
  s_ = nullptr;
  if (prev >= 0 && prev != dev_) cudaSetDevice(prev);
}

// Generates whole chunks of max_iters iterations; a request that does not
// end on a chunk boundary leaves the rest of the chunk for the next call.
void KeystreamSource::next(uint8_t* host, uint64_t bytes) {
  DeviceScope scope(dev_);
  const uint64_t cb = chunk_bytes();
  if (bytes > cb) raise(Errc::invalid_argument, "request larger than a chunk");
  uint64_t got = 0;
  while (got < bytes) {
    if (carry_ == have_) {
      gen_.chain(slot_, gen_.max_iters(), s_);
      gen_.emit(slot_, d_buf_, cb, 0, gen_.max_iters(), s_);
      slot_ ^= 1;
      carry_ = 0;
      have_ = cb;
    }
    const uint64_t take = std::min(bytes - got, have_ - carry_);
    ck(cudaMemcpy2DAsync(host + got, cb, d_buf_ + carry_, cb, take, n_,
                         cudaMemcpyDeviceToHost, s_), "D2H keystream");
    ck(cudaStreamSynchronize(s_), "keystream");
    carry_ += take;
    got += take;
  }
}

void KeystreamSource::burn(uint64_t iters) {
  DeviceScope scope(dev_);
  const uint64_t cb = chunk_bytes();
  while (iters > 0) {
    const uint32_t now = uint32_t(std::min<uint64_t>(round_up(iters, 8), gen_.max_iters()));
    gen_.chain(slot_, now, s_);
    gen_.emit(slot_, d_buf_, cb, 0, now, s_);
    slot_ ^= 1;
    iters -= std::min<uint64_t>(iters, now);
  }
  carry_ = have_ = 0;
  ck(cudaStreamSynchronize(s_), "keystream");
}

}  // namespace cveb
