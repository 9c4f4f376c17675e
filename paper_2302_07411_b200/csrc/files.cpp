// File pipelines on the GPU engine: plaintext frames
// (P6 / directory / raw) -> CVE1 container and back, through the same Engine
// as the per-frame ABI.  Order of checks and error codes follow the
// reference's cve_encrypt_file / cve_decrypt_file (capi.cpp:143-164,
// 262-333).  Differences: frames travel to the GPU unpadded and are padded
// (and, on decrypt, cropped) on the device; the next batch is read from disk
// and the previous one written while the GPU works on the current one.
#include "files.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <future>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "engine.hpp"
#include "fileio.hpp"

namespace cveb {
namespace {

constexpr uint64_t kBatchBytes = 64ull << 20;  // host staging per batch

// Pinned staging buffers are cached process-wide: pinning ~100 MB per call
// costs 0.1-1 s and varies, more than the GPU work of a short clip.
class PinnedCache {
 public:
  static PinnedCache& get() {
    static PinnedCache* c = new PinnedCache();  // never destroyed: the CUDA
    return *c;                                  // runtime may be gone at exit
  }
  uint8_t* take(size_t n) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      size_t best = free_.size();
      for (size_t i = 0; i < free_.size(); ++i)
        if (free_[i].second >= n && (best == free_.size() || free_[i].second < free_[best].second))
          best = i;
      if (best != free_.size()) {
        uint8_t* p = free_[best].first;
        cached_ -= free_[best].second;
        sizes_[p] = free_[best].second;
        free_.erase(free_.begin() + long(best));
        return p;
      }
    }
    uint8_t* p = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&p), n, cudaHostAllocDefault) != cudaSuccess)
      raise(Errc::internal, "cudaHostAlloc failed");
    std::lock_guard<std::mutex> lock(mu_);
    sizes_[p] = n;
    return p;
  }
  void give(uint8_t* p) {
    std::lock_guard<std::mutex> lock(mu_);
    const size_t n = sizes_[p];
    sizes_.erase(p);
    if (cached_ + n > kCacheCap) {
      cudaFreeHost(p);
      return;
    }
    free_.emplace_back(p, n);
    cached_ += n;
  }

 private:
  static constexpr size_t kCacheCap = size_t(512) << 20;
  std::mutex mu_;
  std::vector<std::pair<uint8_t*, size_t>> free_;
  std::map<uint8_t*, size_t> sizes_;
  size_t cached_ = 0;
};

struct Pinned {
  uint8_t* p = nullptr;
  explicit Pinned(size_t n) : p(PinnedCache::get().take(std::max<size_t>(n, 1))) {}
  ~Pinned() { PinnedCache::get().give(p); }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
};

uint32_t batch_frames(uint64_t frame_bytes, uint32_t total) {
  const uint64_t b = std::max<uint64_t>(1, kBatchBytes / std::max<uint64_t>(frame_bytes, 1));
  return uint32_t(std::min<uint64_t>(b, std::max<uint32_t>(total, 1)));
}

}  // namespace

void encrypt_file(const char* key_hex, const FileOptions& opt, const char* in_path,
                  const char* out_path, int device) {
  NvtxRange nvtx("cve: encrypt_file");
  if (!key_hex) raise(Errc::invalid_argument, "key_hex is null");
  if (!in_path || !out_path) raise(Errc::invalid_argument, "path is null");
  if (opt.raw_width || opt.raw_height) {
    if (!opt.raw_width || !opt.raw_height)
      raise(Errc::invalid_argument, "raw input needs both dimensions");
  }
  if (opt.workers > 0xFFFF) raise(Errc::invalid_argument, "workers must fit the container header");
  if (opt.rounds < 1 || opt.rounds > 255) raise(Errc::invalid_argument, "rounds must be in 1..255");
  const Key key = parse_key(key_hex);

  PlainSource src(in_path, opt.raw_width, opt.raw_height);
  CveHeader h;
  h.map_kind = uint8_t(key.kind);
  h.side = padded_side_of(src.width(), src.height(), opt.workers);
  h.orig_width = src.width();
  h.orig_height = src.height();
  h.workers = uint16_t(opt.workers);
  h.rounds = uint8_t(opt.rounds);
  h.fps = opt.fps;
  h.frame_count = src.count();

  Engine engine(key, opt.workers, opt.rounds, device);
  ContainerOut out(out_path, h);
  const uint64_t in_fb = uint64_t(h.orig_width) * h.orig_height * 3;
  const uint64_t sq_fb = uint64_t(h.side) * h.side * 3;
  const uint32_t B = batch_frames(sq_fb, h.frame_count);
  Pinned in_buf[2] = {Pinned(B * in_fb), Pinned(B * in_fb)};
  Pinned out_buf[2] = {Pinned(B * sq_fb), Pinned(B * sq_fb)};

  auto read_batch = [&](uint8_t* dst, uint32_t nb) {
    for (uint32_t i = 0; i < nb; ++i) src.next(dst + i * in_fb);
  };
  // batch k: read ahead (k+1) and write behind (k-1) overlap the GPU work
  uint32_t done = 0, cur = 0;
  uint32_t nb = std::min(B, h.frame_count);
  read_batch(in_buf[0].p, nb);
  std::future<void> writing;
  while (done < h.frame_count) {
    const uint32_t next_nb = std::min(B, h.frame_count - done - nb);
    std::future<void> prefetch;
    if (next_nb)
      prefetch = std::async(std::launch::async, read_batch, in_buf[cur ^ 1].p, next_nb);
    engine.run_host_io(Engine::HostIo{in_buf[cur].p, h.orig_width, h.orig_height,
                                      out_buf[cur].p, h.side, h.side},
                       h.side, nb, /*decrypt=*/false);
    if (writing.valid()) writing.get();  // batch k-1 written: its buffer is free
    writing = std::async(std::launch::async, [&out, p = out_buf[cur].p, nb] { out.put(p, nb); });
    if (prefetch.valid()) prefetch.get();
    done += nb;
    nb = next_nb;
    cur ^= 1;
  }
  if (writing.valid()) writing.get();
  out.finish();
}

void decrypt_file(const char* key_hex, const FileOptions* opt, int format,
                  const char* in_path, const char* out_path, int device) {
  NvtxRange nvtx("cve: decrypt_file");
  if (!key_hex) raise(Errc::invalid_argument, "key_hex is null");
  if (!in_path || !out_path) raise(Errc::invalid_argument, "path is null");
  if (format < 0 || format > 2) raise(Errc::invalid_argument, "unknown output format");
  const Key key = parse_key(key_hex);

  ContainerIn in(in_path);
  const CveHeader h = in.header();
  if (uint8_t(key.kind) != h.map_kind)
    raise(Errc::mismatch, "key map kind does not match the container");
  if (opt) {
    if (opt->workers && opt->workers != h.workers)
      raise(Errc::mismatch, "workers does not match the container");
    if (opt->rounds && opt->rounds != h.rounds)
      raise(Errc::mismatch, "rounds does not match the container");
  }
  Engine engine(key, h.workers, h.rounds, device);
  PlainSink sink(out_path, /*raw=*/format == 2, h.frame_count);
  const uint64_t out_fb = uint64_t(h.orig_width) * h.orig_height * 3;
  const uint64_t sq_fb = uint64_t(h.side) * h.side * 3;
  const uint32_t B = batch_frames(sq_fb, h.frame_count);
  Pinned in_buf[2] = {Pinned(B * sq_fb), Pinned(B * sq_fb)};
  Pinned out_buf[2] = {Pinned(B * out_fb), Pinned(B * out_fb)};

  uint32_t done = 0, cur = 0;
  uint32_t nb = std::min(B, h.frame_count);
  in.next(in_buf[0].p, nb);
  std::future<void> writing;
  while (done < h.frame_count) {
    const uint32_t next_nb = std::min(B, h.frame_count - done - nb);
    std::future<void> prefetch;
    if (next_nb)
      prefetch = std::async(std::launch::async,
                            [&, dst = in_buf[cur ^ 1].p, k = next_nb] { in.next(dst, k); });
    engine.run_host_io(Engine::HostIo{in_buf[cur].p, h.side, h.side, out_buf[cur].p,
                                      h.orig_width, h.orig_height},
                       h.side, nb, /*decrypt=*/true);
    if (writing.valid()) writing.get();
    writing = std::async(std::launch::async, [&sink, &h, out_fb, p = out_buf[cur].p, nb] {
      for (uint32_t i = 0; i < nb; ++i) sink.put(p + i * out_fb, h.orig_width, h.orig_height);
    });
    if (prefetch.valid()) prefetch.get();
    done += nb;
    nb = next_nb;
    cur ^= 1;
  }
  if (writing.valid()) writing.get();
  sink.finish();
}

// Reference cve_nist_export (capi.cpp:385-415): the byte budget split over
// the n workers derived from the key (the first byte_count % n workers get
// one extra byte); each worker's fresh generator stream is written in
// worker order.  All n generators run at once on the GPU (K1); chunks are
// copied back and written at each worker's file offset.
void keystream_export(const char* key_hex, uint32_t workers, uint64_t byte_count,
                      const char* out_path, int device) {
  NvtxRange nvtx("cve: nist_export");
  if (!key_hex) raise(Errc::invalid_argument, "key_hex is null");
  if (!out_path) raise(Errc::invalid_argument, "path is null");
  if (byte_count == 0) raise(Errc::invalid_argument, "byte_count must be >= 1");
  const uint32_t n = workers ? workers : 8;
  const Key key = parse_key(key_hex);
  Coordinator coord(key);
  const std::vector<WorkerLanes> lanes = coord.derive_workers(n);

  std::FILE* out = std::fopen(out_path, "wb");
  if (!out) raise(Errc::io, "cannot open output file");
  struct Closer {
    std::FILE* f;
    ~Closer() {
      if (f) std::fclose(f);
    }
  } closer{out};

  const uint64_t base = byte_count / n, extra = byte_count % n;
  const uint64_t longest = base + (extra ? 1 : 0);
  std::vector<uint64_t> start(n), len(n);
  for (uint32_t i = 0; i < n; ++i) {
    len[i] = base + (i < extra ? 1 : 0);
    start[i] = i ? start[i - 1] + len[i - 1] : 0;
  }
  KeystreamSource src(lanes, key.kind, device, longest);
  const uint64_t chunk = src.chunk_bytes();
  Pinned host(size_t(chunk) * n);
  for (uint64_t done = 0; done < longest; done += chunk) {
    const uint64_t now = std::min(chunk, longest - done);
    src.next(host.p, now);  // now bytes per worker, worker-major
    for (uint32_t i = 0; i < n; ++i) {
      if (done >= len[i]) continue;
      const uint64_t take = std::min(now, len[i] - done);
      if (std::fseek(out, long(start[i] + done), SEEK_SET) != 0 ||
          std::fwrite(host.p + uint64_t(i) * chunk, 1, take, out) != take)
        raise(Errc::io, "short write");
    }
  }
  if (std::fflush(out) != 0) raise(Errc::io, "short write");
}

}  // namespace cveb
