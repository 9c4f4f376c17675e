// C ABI of libcve_b200.so (include/cve_b200.h).
//
// Status mapping and argument-check order follow the reference C ABI
// (capi.cpp:36-67 `guarded`, 166-181 `run_frame`, 187-260 exports): argument
// errors are reported before any seed is drawn; exceptions map to
// cve_status; the detail string is thread-local and only set on failure.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/cve_b200.h"
#include "analysis.hpp"
#include "engine.hpp"
#include "fileio.hpp"
#include "files.hpp"
#include "harness.hpp"
#include "keying.hpp"

struct cve_cipher {
  std::unique_ptr<cveb::Engine> engine;
};

namespace {

thread_local std::string g_last_error;
thread_local int g_device = -1;

template <typename Fn>
cve_status guarded(Fn&& fn) {
  try {
    fn();
    return CVE_OK;
  } catch (const cveb::Error& e) {
    g_last_error = e.what();
    return static_cast<cve_status>(e.code);
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return CVE_ERROR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CVE_ERROR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown failure";
    return CVE_ERROR_INTERNAL;
  }
}

void require(bool ok, const char* what) {
  if (!ok) cveb::raise(cveb::Errc::invalid_argument, what);
}

using cveb::DeviceScope;  // runs the handle's work on its device, restoring the caller's

cve_status run_frames(cve_cipher* c, uint8_t* px, uint32_t side,
                      uint32_t count, bool decrypt) {
  return guarded([&] {
    require(c != nullptr, "cipher is null");
    require(px != nullptr, "pixels is null");
    require(side != 0, "side must be >= 1");
    require(count != 0, "count must be >= 1");
    DeviceScope scope(c->engine->device());
    c->engine->run_host(px, side, count, decrypt);
  });
}

cve_status run_frames_async(cve_cipher* c, uint8_t* d_px, uint32_t side,
                            uint32_t count, void* stream, bool decrypt) {
  return guarded([&] {
    require(c != nullptr, "cipher is null");
    require(d_px != nullptr, "pixels is null");
    require(side != 0, "side must be >= 1");
    require(count != 0, "count must be >= 1");
    DeviceScope scope(c->engine->device());
    c->engine->run_device(d_px, side, count, decrypt,
                          static_cast<cudaStream_t>(stream));
  });
}

int current_device() {
  int dev = g_device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev;
}

}  // namespace

extern "C" {

const char* cve_version(void) { return "1.0.0-b200"; }

const char* cve_status_message(cve_status status) {
  switch (status) {
    case CVE_OK:
      return "ok";
    case CVE_ERROR_INVALID_ARGUMENT:
      return "invalid argument";
    case CVE_ERROR_BAD_KEY:
      return "malformed or out-of-domain key";
    case CVE_ERROR_IO:
      return "file i/o failure";
    case CVE_ERROR_BAD_FORMAT:
      return "unrecognized or corrupt input format";
    case CVE_ERROR_MISMATCH:
      return "parameters do not match the input";
    case CVE_ERROR_INTERNAL:
      return "internal failure";
  }
  return "unknown status";
}

const char* cve_last_error(void) { return g_last_error.c_str(); }

void cve_string_free(char* s) { std::free(s); }

cve_status cve_key_generate(cve_map_kind kind, char* hex_out, size_t hex_cap) {
  return guarded([&] {
    require(hex_out != nullptr, "hex_out is null");
    require(kind == CVE_MAP_PLCM || kind == CVE_MAP_LASM, "unknown map kind");
    const std::string hex =
        cveb::key_hex(cveb::fresh_key(static_cast<cveb::MapKind>(kind)));
    require(hex_cap >= hex.size() + 1, "key buffer too small");
    std::memcpy(hex_out, hex.c_str(), hex.size() + 1);
  });
}

cve_status cve_key_validate(const char* key_hex, cve_map_kind* kind_out) {
  return guarded([&] {
    require(key_hex != nullptr, "key_hex is null");
    const cveb::Key k = cveb::parse_key(key_hex);
    if (kind_out) *kind_out = static_cast<cve_map_kind>(k.kind);
  });
}

cve_status cve_cipher_create(const char* key_hex, uint32_t workers,
                             uint32_t rounds, int parallel, cve_cipher** out) {
  (void)parallel;  // scheduling-only in the reference (cve.h:64-66)
  return guarded([&] {
    require(out != nullptr, "out is null");
    require(key_hex != nullptr, "key_hex is null");
    const cveb::Key key = cveb::parse_key(key_hex);
    auto c = std::make_unique<cve_cipher>();
    c->engine = std::make_unique<cveb::Engine>(key, workers, rounds, current_device());
    *out = c.release();
  });
}

cve_status cve_cipher_create_devices(const char* key_hex, uint32_t workers, uint32_t rounds,
                                     const int* devices, uint32_t device_count,
                                     cve_cipher** out) {
  return guarded([&] {
    require(out != nullptr, "out is null");
    require(key_hex != nullptr, "key_hex is null");
    require(devices != nullptr, "devices is null");
    require(device_count >= 1, "device_count must be >= 1");
    const cveb::Key key = cveb::parse_key(key_hex);
    auto c = std::make_unique<cve_cipher>();
    c->engine = std::make_unique<cveb::Engine>(
        key, workers, rounds, std::vector<int>(devices, devices + device_count));
    *out = c.release();
  });
}

cve_status cve_cipher_shards(const cve_cipher* cipher, uint32_t* count_out, int* devices_out,
                             uint32_t cap) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(count_out != nullptr, "count_out is null");
    const uint32_t n = cipher->engine->shard_count();
    *count_out = n;
    for (uint32_t i = 0; i < n && i < cap && devices_out; ++i)
      devices_out[i] = cipher->engine->shard_device(i);
  });
}

// Engine::~Engine restores the caller's device itself (it may run on a
// garbage-collection thread, where no DeviceScope is in place).
void cve_cipher_destroy(cve_cipher* cipher) { delete cipher; }

cve_status cve_cipher_encrypt_frame(cve_cipher* cipher, uint8_t* pixels,
                                    uint32_t side) {
  return run_frames(cipher, pixels, side, 1, false);
}

cve_status cve_cipher_decrypt_frame(cve_cipher* cipher, uint8_t* pixels,
                                    uint32_t side) {
  return run_frames(cipher, pixels, side, 1, true);
}

cve_status cve_cipher_transform_frame(cve_cipher* cipher, uint8_t* pixels, uint32_t side,
                                      uint32_t rounds, int confusion, int diffusion,
                                      uint8_t* states_out) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(pixels != nullptr, "pixels is null");
    require(side != 0, "side must be >= 1");
    require(rounds >= 1 && rounds <= 255, "rounds must be in 1..255");
    DeviceScope scope(cipher->engine->device());
    const size_t fb = size_t(side) * side * 3;
    std::function<void(uint32_t, const uint8_t*)> keep;
    if (states_out != nullptr)
      keep = [&](uint32_t k, const uint8_t* s) { std::memcpy(states_out + (k - 1) * fb, s, fb); };
    cipher->engine->transform_host(pixels, side, rounds, confusion != 0, diffusion != 0, keep,
                                   nullptr);
  });
}

cve_status cve_cipher_seeds_drawn(const cve_cipher* cipher, uint64_t* out) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(out != nullptr, "out is null");
    *out = cipher->engine->seeds_drawn();
  });
}

cve_status cve_cipher_encrypt_frames(cve_cipher* cipher, uint8_t* pixels,
                                     uint32_t side, uint32_t count) {
  return run_frames(cipher, pixels, side, count, false);
}

cve_status cve_cipher_decrypt_frames(cve_cipher* cipher, uint8_t* pixels,
                                     uint32_t side, uint32_t count) {
  return run_frames(cipher, pixels, side, count, true);
}

cve_status cve_cipher_encrypt_frames_async(cve_cipher* cipher,
                                           uint8_t* d_pixels, uint32_t side,
                                           uint32_t count, void* stream) {
  return run_frames_async(cipher, d_pixels, side, count, stream, false);
}

cve_status cve_cipher_decrypt_frames_async(cve_cipher* cipher,
                                           uint8_t* d_pixels, uint32_t side,
                                           uint32_t count, void* stream) {
  return run_frames_async(cipher, d_pixels, side, count, stream, true);
}

cve_status cve_encrypt_file(const char* key_hex, const cve_io_options* io,
                            const char* in_path, const char* out_path) {
  return guarded([&] {
    cveb::FileOptions o;  // capi.cpp:143-164 defaults
    if (io) {
      if (io->workers) o.workers = io->workers;
      if (io->rounds) o.rounds = io->rounds;
      if (io->fps) o.fps = io->fps;
      o.raw_width = io->raw_width;
      o.raw_height = io->raw_height;
    }
    if (!key_hex) require(false, "key_hex is null");
    if (!in_path || !out_path) require(false, "path is null");
    if ((o.raw_width || o.raw_height) && !(o.raw_width && o.raw_height))
      require(false, "raw input needs both dimensions");
    const int dev = current_device();
    DeviceScope scope(dev);
    cveb::encrypt_file(key_hex, o, in_path, out_path, dev);
  });
}

cve_status cve_decrypt_file(const char* key_hex, const cve_io_options* io,
                            cve_out_format format, const char* in_path,
                            const char* out_path) {
  return guarded([&] {
    cveb::FileOptions o;
    if (io) {
      o.workers = io->workers;  // 0: follow the header
      o.rounds = io->rounds;
    }
    const int dev = current_device();
    DeviceScope scope(dev);
    cveb::decrypt_file(key_hex, io ? &o : nullptr, int(format), in_path, out_path, dev);
  });
}

cve_status cve_nist_export(const char* key_hex, uint32_t workers,
                           uint64_t byte_count, const char* out_path) {
  return guarded([&] {
    const int dev = current_device();
    DeviceScope scope(dev);
    cveb::keystream_export(key_hex, workers, byte_count, out_path, dev);
  });
}

// capi.cpp:335-358: argument checks, then the frame(s), then the size match.
cve_status cve_analyze(const cve_analyze_options* options, char** text_out) {
  return guarded([&] {
    require(options != nullptr, "options is null");
    require(text_out != nullptr, "text_out is null");
    require(options->input != nullptr, "input is null");
    const uint32_t samples = options->samples != 0 ? options->samples : 20000;
    const cveb::HostFrame frame = cveb::load_frame_any(options->input, options->frame_index);
    cveb::HostFrame second;
    if (options->second != nullptr) {
      second = cveb::load_frame_any(options->second, options->second_frame_index);
      if (second.side != frame.side) cveb::raise(cveb::Errc::mismatch, "images differ in size");
    }
    const int dev = current_device();
    DeviceScope scope(dev);
    const std::string text = cveb::analyze(frame, options->second ? &second : nullptr, samples,
                                           options->seed, options->csv != 0, dev);
    char* out = static_cast<char*>(std::malloc(text.size() + 1));
    if (out == nullptr) throw std::bad_alloc();
    std::memcpy(out, text.c_str(), text.size() + 1);
    *text_out = out;
  });
}

// capi.cpp:417-505: options and csv_out checked first, then the key (NULL ->
// a fresh key of map_kind), then the defaults.
namespace {
cveb::Key harness_key(const char* key_hex, cve_map_kind fallback) {
  if (key_hex != nullptr) return cveb::parse_key(key_hex);
  require(fallback == CVE_MAP_PLCM || fallback == CVE_MAP_LASM, "unknown map kind");
  return cveb::fresh_key(static_cast<cveb::MapKind>(fallback));
}
char* c_string(const std::string& text) {
  char* out = static_cast<char*>(std::malloc(text.size() + 1));
  if (out == nullptr) throw std::bad_alloc();
  std::memcpy(out, text.c_str(), text.size() + 1);
  return out;
}
}  // namespace

cve_status cve_bench_bytegen(const cve_bench_bytegen_options* options, char** csv_out) {
  return guarded([&] {
    require(options != nullptr, "options is null");
    require(csv_out != nullptr, "csv_out is null");
    const cveb::Key key = harness_key(options->key_hex, options->map_kind);
    std::vector<uint32_t> counts = {1, 2, 4, 8};
    if (options->worker_count_len != 0) {
      require(options->worker_counts != nullptr, "worker_counts is null");
      counts.assign(options->worker_counts, options->worker_counts + options->worker_count_len);
    }
    const uint64_t iterations = options->iterations != 0 ? options->iterations : 50000000;
    const int dev = current_device();
    DeviceScope scope(dev);
    *csv_out = c_string(cveb::bytegen_table(key, counts, iterations, dev));
  });
}

cve_status cve_bench_phases(const cve_bench_phases_options* options, char** csv_out) {
  return guarded([&] {
    require(options != nullptr, "options is null");
    require(csv_out != nullptr, "csv_out is null");
    const cveb::Key key = harness_key(options->key_hex, options->map_kind);
    const uint32_t side = options->side != 0 ? options->side : 960;
    const uint32_t workers = options->workers != 0 ? options->workers : 8;
    const uint32_t rounds = options->rounds != 0 ? options->rounds : 5;
    const uint32_t images = options->images != 0 ? options->images : 100;
    const int dev = current_device();
    DeviceScope scope(dev);
    *csv_out = c_string(cveb::phases_table(key, side, workers, rounds, images, dev));
  });
}

cve_status cve_bench_video(const cve_bench_video_options* options, char** csv_out) {
  return guarded([&] {
    require(options != nullptr, "options is null");
    require(csv_out != nullptr, "csv_out is null");
    const cveb::Key key = harness_key(options->key_hex, options->map_kind);
    std::vector<uint32_t> sides = {96, 192, 288, 384, 480, 576, 672, 768};
    if (options->side_len != 0) {
      require(options->sides != nullptr, "sides is null");
      sides.assign(options->sides, options->sides + options->side_len);
    }
    const uint32_t workers = options->workers != 0 ? options->workers : 8;
    const uint32_t rounds = options->rounds != 0 ? options->rounds : 5;
    const uint32_t frames = options->frames != 0 ? options->frames : 600;
    const uint16_t fps = options->fps != 0 ? options->fps : 20;
    const int dev = current_device();
    DeviceScope scope(dev);
    *csv_out = c_string(cveb::video_table(key, sides, workers, rounds, frames, fps, dev));
  });
}

cve_status cve_sweep_rounds(const cve_sweep_options* options, char** csv_out) {
  return guarded([&] {
    require(options != nullptr, "options is null");
    require(csv_out != nullptr, "csv_out is null");
    const cveb::Key key = harness_key(options->key_hex, options->map_kind);
    const uint32_t workers = options->workers != 0 ? options->workers : 1;
    const uint32_t max_rounds = options->max_rounds != 0 ? options->max_rounds : 10;
    cveb::HostFrame plain;
    if (options->input != nullptr) {  // load_ppm: any P6, padded to a square (image_io.cpp:110-113)
      const std::vector<uint8_t> data = cveb::read_whole_file(options->input);
      const cveb::P6Image img = cveb::p6_parse(data.data(), data.size());
      plain.side = cveb::padded_side_of(img.width, img.height, workers);
      plain.orig_width = img.width;
      plain.orig_height = img.height;
      plain.px.assign(size_t(plain.side) * plain.side * 3, 0);
      for (uint32_t r = 0; r < img.height; ++r)
        std::memcpy(plain.px.data() + size_t(r) * plain.side * 3,
                    img.rgb.data() + size_t(r) * img.width * 3, size_t(img.width) * 3);
    } else {
      const uint32_t side = options->synth_side != 0 ? options->synth_side : 512;
      if (side % workers != 0)
        cveb::raise(cveb::Errc::mismatch, "synthetic side is not divisible by the worker count");
      plain = cveb::natural_frame(side, options->seed);
    }
    const int dev = current_device();
    DeviceScope scope(dev);
    *csv_out = c_string(cveb::sweep_table(key, plain, workers, max_rounds, options->seed, dev));
  });
}

cve_status cve_add_noise_file(const char* in_path, const char* out_path, double rate,
                              uint64_t seed) {
  return guarded([&] {
    require(in_path != nullptr && out_path != nullptr, "path is null");
    cveb::add_noise_file(in_path, out_path, rate, seed);
  });
}

cve_status cve_crop_file(const char* in_path, const char* out_path, const cve_crop_block* blocks,
                         size_t block_count) {
  return guarded([&] {
    require(in_path != nullptr && out_path != nullptr, "path is null");
    require(block_count == 0 || blocks != nullptr, "blocks is null");
    std::vector<cveb::CropBlock> list(block_count);
    for (size_t i = 0; i < block_count; ++i)
      list[i] = {blocks[i].x, blocks[i].y, blocks[i].side, blocks[i].fill};
    cveb::crop_file(in_path, out_path, list);
  });
}

cve_status cve_frame_stats_device(const uint8_t* frame, const uint8_t* second, uint32_t side,
                                  uint64_t* hist_out, uint64_t* diff_out, void* stream) {
  return guarded([&] {
    require(frame != nullptr, "frame is null");
    require(side != 0, "side must be >= 1");
    require(hist_out != nullptr || (second != nullptr && diff_out != nullptr),
            "nothing to compute");
    const int dev = current_device();
    DeviceScope scope(dev);
    cveb::launch_frame_stats(frame, second, uint64_t(side) * side * 3,
                             reinterpret_cast<unsigned long long*>(hist_out),
                             second ? reinterpret_cast<unsigned long long*>(diff_out) : nullptr,
                             static_cast<cudaStream_t>(stream));
  });
}

cve_status cve_padded_side(uint32_t width, uint32_t height, uint32_t workers,
                           uint32_t* side_out) {
  return guarded([&] {
    require(side_out != nullptr, "side_out is null");
    *side_out = cveb::padded_side_of(width, height, workers);
  });
}

cve_status cve_cipher_encrypt_frames_wh(cve_cipher* cipher, const uint8_t* rgb,
                                        uint32_t width, uint32_t height,
                                        uint32_t count, uint8_t* out_square) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(rgb != nullptr && out_square != nullptr, "buffer is null");
    require(count != 0, "count must be >= 1");
    const uint32_t side = cveb::padded_side_of(width, height, cipher->engine->workers());
    DeviceScope scope(cipher->engine->device());
    cipher->engine->run_host_io(
        cveb::Engine::HostIo{rgb, width, height, out_square, side, side}, side, count, false);
  });
}

cve_status cve_cipher_decrypt_frames_wh(cve_cipher* cipher, const uint8_t* square,
                                        uint32_t side, uint32_t width,
                                        uint32_t height, uint32_t count,
                                        uint8_t* out_rgb) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(square != nullptr && out_rgb != nullptr, "buffer is null");
    require(side != 0 && width != 0 && height != 0, "dimensions must be >= 1");
    require(count != 0, "count must be >= 1");
    DeviceScope scope(cipher->engine->device());
    cipher->engine->run_host_io(
        cveb::Engine::HostIo{square, side, side, out_rgb, width, height}, side, count, true);
  });
}

static cve_status run_frames_sharded(cve_cipher* c, uint8_t* const* shard_px, uint32_t side,
                                     uint32_t count, void* const* streams, bool decrypt) {
  return guarded([&] {
    require(c != nullptr, "cipher is null");
    require(shard_px != nullptr, "pixels is null");
    const uint32_t G = c->engine->shard_count();
    for (uint32_t i = 0; i < G && i < count; ++i) require(shard_px[i] != nullptr, "pixels is null");
    require(side != 0, "side must be >= 1");
    require(count != 0, "count must be >= 1");
    std::vector<cudaStream_t> users(G, nullptr);
    if (streams)
      for (uint32_t i = 0; i < G; ++i) users[i] = static_cast<cudaStream_t>(streams[i]);
    DeviceScope scope(c->engine->device());
    c->engine->run_device_sharded(shard_px, side, count, decrypt, users.data());
  });
}

cve_status cve_cipher_encrypt_frames_sharded_async(cve_cipher* cipher, uint8_t* const* shard_pixels,
                                                   uint32_t side, uint32_t count,
                                                   void* const* streams) {
  return run_frames_sharded(cipher, shard_pixels, side, count, streams, false);
}

cve_status cve_cipher_decrypt_frames_sharded_async(cve_cipher* cipher, uint8_t* const* shard_pixels,
                                                   uint32_t side, uint32_t count,
                                                   void* const* streams) {
  return run_frames_sharded(cipher, shard_pixels, side, count, streams, true);
}

cve_status cve_cipher_synchronize(cve_cipher* cipher) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    DeviceScope scope(cipher->engine->device());
    cipher->engine->synchronize();
  });
}

cve_status cve_set_device(int device) {
  return guarded([&] {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      cveb::raise(cveb::Errc::internal, "no CUDA device");
    require(device >= 0 && device < count, "device index out of range");
    g_device = device;
  });
}

cve_status cve_set_streams_per_handle(uint32_t streams) {
  return guarded([&] { cveb::set_streams_per_handle(int(streams)); });
}

cve_status cve_set_round_fusion(uint32_t mode) {
  return guarded([&] { cveb::set_round_fusion(int(mode)); });
}

cve_status cve_cipher_peek_keystream(cve_cipher* cipher, uint32_t worker,
                                     uint8_t* out, size_t len) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(out != nullptr || len == 0, "out is null");
    DeviceScope scope(cipher->engine->device());
    cipher->engine->peek(worker, out, len);
  });
}

cve_status cve_cipher_prefetch_keystream(cve_cipher* cipher, uint64_t bytes) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    DeviceScope scope(cipher->engine->device());
    cipher->engine->prefetch(bytes);
  });
}

cve_status cve_cipher_get_stats(cve_cipher* cipher, cve_cipher_stats* out) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(out != nullptr, "out is null");
    DeviceScope scope(cipher->engine->device());
    const cveb::EngineStats s = cipher->engine->stats();
    out->frames = s.frames;
    out->keystream_iters = s.keystream_iters;
    out->kernel_launches = s.kernel_launches;
    out->prbg_launches = s.prbg_launches;
    out->guard_replays = s.guard_replays;
    out->prbg_ms = s.prbg_ms;
    out->chain_ms = s.chain_ms;
    out->cipher_ms = s.cipher_ms;
  });
}

cve_status cve_keystream_generate(const double lanes[4], uint8_t* out,
                                  size_t len) {
  return guarded([&] {
    require(lanes != nullptr, "lanes is null");
    require(out != nullptr || len == 0, "out is null");
    DeviceScope scope(current_device());
    cveb::standalone_stream(cveb::Lane{lanes[0], lanes[1]},
                            cveb::Lane{lanes[2], lanes[3]}, out, len);
  });
}

cve_status cve_keystream_generate_ex(const double lanes[4], uint8_t* out, size_t len,
                                     uint32_t launch_iters, uint32_t flags,
                                     uint64_t* guard_replays) {
  return guarded([&] {
    require(lanes != nullptr, "lanes is null");
    require(out != nullptr || len == 0, "out is null");
    require((flags & ~uint32_t(CVE_KEYSTREAM_DENSE_ORBIT)) == 0, "unknown flags");
    DeviceScope scope(current_device());
    cveb::standalone_stream(cveb::Lane{lanes[0], lanes[1]}, cveb::Lane{lanes[2], lanes[3]}, out,
                            len, launch_iters, guard_replays,
                            (flags & CVE_KEYSTREAM_DENSE_ORBIT) != 0);
  });
}

cve_status cve_keystream_generate_lasm(const double lanes[6], uint8_t* out,
                                       size_t len) {
  return guarded([&] {
    require(lanes != nullptr, "lanes is null");
    require(out != nullptr || len == 0, "out is null");
    DeviceScope scope(current_device());
    cveb::standalone_stream(cveb::LasmLane{lanes[0], lanes[1], lanes[2]},
                            cveb::LasmLane{lanes[3], lanes[4], lanes[5]}, out, len);
  });
}

cve_status cve_glibc_sin(const double* x, double* y, size_t count) {
  return guarded([&] {
    require((x != nullptr && y != nullptr) || count == 0, "null buffer");
    if (count == 0) return;
    DeviceScope scope(current_device());
    struct Buf {
      double* p = nullptr;
      ~Buf() { cudaFree(p); }
    } dx, dy;
    if (cudaMalloc(&dx.p, count * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&dy.p, count * sizeof(double)) != cudaSuccess)
      cveb::raise(cveb::Errc::internal, "cudaMalloc failed (no usable CUDA device?)");
    if (cudaMemcpy(dx.p, x, count * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      cveb::raise(cveb::Errc::internal, "upload failed");
    cveb::launch_glibc_sin(dx.p, dy.p, count, nullptr);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpy(y, dy.p, count * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      cveb::raise(cveb::Errc::internal, "glibc_sin kernel failed");
  });
}

cve_status cve_derive_worker_lanes(const char* key_hex, uint32_t workers,
                                   double* lanes_out, uint32_t* seeds_out,
                                   size_t nseeds) {
  return guarded([&] {
    require(key_hex != nullptr, "key_hex is null");
    require(workers != 0, "workers must be >= 1");
    require(lanes_out != nullptr, "lanes_out is null");
    require(seeds_out != nullptr || nseeds == 0, "seeds_out is null");
    cveb::Coordinator coord(cveb::parse_key(key_hex));
    const std::vector<cveb::WorkerLanes> w = coord.derive_workers(workers);
    for (uint32_t i = 0; i < workers; ++i) {
      if (coord.kind() == cveb::MapKind::Plcm) {
        lanes_out[4 * i + 0] = w[i].a.x0;
        lanes_out[4 * i + 1] = w[i].a.p;
        lanes_out[4 * i + 2] = w[i].b.x0;
        lanes_out[4 * i + 3] = w[i].b.p;
      } else {
        const cveb::LasmLane* l[2] = {&w[i].la, &w[i].lb};
        for (int k = 0; k < 2; ++k) {
          lanes_out[6 * i + 3 * k + 0] = l[k]->x0;
          lanes_out[6 * i + 3 * k + 1] = l[k]->y0;
          lanes_out[6 * i + 3 * k + 2] = l[k]->mu;
        }
      }
    }
    for (size_t k = 0; k < nseeds; ++k) seeds_out[k] = coord.next_seed();
  });
}

cve_status cve_cipher_take_prbg_times(cve_cipher* cipher, float* out,
                                      size_t cap, size_t* count) {
  return guarded([&] {
    require(cipher != nullptr, "cipher is null");
    require(count != nullptr, "count is null");
    DeviceScope scope(cipher->engine->device());
    const std::vector<float> t = cipher->engine->take_prbg_times();
    *count = t.size();
    if (out) std::memcpy(out, t.data(), sizeof(float) * std::min(cap, t.size()));
  });
}

}  // extern "C"
