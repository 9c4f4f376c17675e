/*
 * cve_b200.h -- C ABI of the B200 (sm_100a) chaotic video cipher engine.
 *
 * Drop-in boundary.  The first block of entry points has exactly the names,
 * argument meaning, status codes and error behaviour of the reference's
 * hot-path C ABI (reference: /root/reference/proj/include/cve.h); each
 * declaration cites the line it replaces.  A program written against the
 * reference's cipher-handle API compiles and links against libcve_b200.so
 * unchanged.  The second block is additive: batched,
 * pipelined and device-resident variants the synchronous per-frame call
 * cannot express.
 *
 * Both key maps drive the GPU engine: PLCM keys (tag 0x00, 66 hex chars) and
 * LASM keys (tag 0x01, 50 hex chars; the LASM generator evaluates glibc's
 * own sin algorithm on the device, glibc_sin.cuh, so its keystream is the
 * reference's bit for bit on a glibc 2.39 host).
 *
 * Threading matches the reference (cve.h:5-6): one handle is driven by one
 * thread at a time; distinct handles are independent.  All calls are
 * synchronous unless the name ends in _async.
 */
#ifndef CVE_B200_H
#define CVE_B200_H

#include <stddef.h>
#include <stdint.h>

#define CVE_B200_API __attribute__((visibility("default")))

#ifdef __cplusplus
extern "C" {
#endif

/* Status values are numerically identical to the reference (cve.h:24-32). */
typedef enum cve_status {
  CVE_OK = 0,
  CVE_ERROR_INVALID_ARGUMENT = 1,
  CVE_ERROR_BAD_KEY = 2,
  CVE_ERROR_IO = 3,
  CVE_ERROR_BAD_FORMAT = 4,
  CVE_ERROR_MISMATCH = 5,
  CVE_ERROR_INTERNAL = 6 /* also: CUDA failure, no usable sm_100 device */
} cve_status;

typedef enum cve_map_kind { CVE_MAP_PLCM = 0, CVE_MAP_LASM = 1 } cve_map_kind;

typedef struct cve_cipher cve_cipher;

/* ---- reference hot-path subset ------------------------------------------ */

/* replaces cve.h:39.  Returns the engine version string. */
CVE_B200_API const char* cve_version(void);

/* replaces cve.h:42.  Never NULL, for any value. */
CVE_B200_API const char* cve_status_message(cve_status status);

/* replaces cve.h:45.  Thread-local detail of the last failure ("" if none). */
CVE_B200_API const char* cve_last_error(void);

/* replaces cve.h:47.  Frees strings this library returned; NULL is a no-op. */
CVE_B200_API void cve_string_free(char* s);

/* replaces cve.h:53-54.  Fresh key from OS entropy; PLCM needs cap >= 67,
 * LASM >= 51. */
CVE_B200_API cve_status cve_key_generate(cve_map_kind kind, char* hex_out,
                                         size_t hex_cap);

/* replaces cve.h:57-58.  kind_out may be NULL. */
CVE_B200_API cve_status cve_key_validate(const char* key_hex,
                                         cve_map_kind* kind_out);

/* replaces cve.h:67-69.  workers = subframe (row band) count n, a cipher
 * parameter; rounds in 1..255.  `parallel` is accepted for ABI compatibility
 * and ignored: output is bit-identical to the reference either way. */
CVE_B200_API cve_status cve_cipher_create(const char* key_hex,
                                          uint32_t workers, uint32_t rounds,
                                          int parallel, cve_cipher** out);

/* replaces cve.h:70.  NULL is a no-op. */
CVE_B200_API void cve_cipher_destroy(cve_cipher* cipher);

/* replaces cve.h:75-76 / 77-78.  In place on a side*side*3 interleaved RGB24
 * host buffer.  The k-th encrypt OR decrypt call on a handle binds to frame
 * index k.  NULL/0 arguments -> INVALID_ARGUMENT with no seed drawn; a side
 * not divisible by workers -> MISMATCH after the frame's seed was drawn
 * (reference engine.cpp:293-296, 189-196). */
CVE_B200_API cve_status cve_cipher_encrypt_frame(cve_cipher* cipher,
                                                 uint8_t* pixels,
                                                 uint32_t side);
CVE_B200_API cve_status cve_cipher_decrypt_frame(cve_cipher* cipher,
                                                 uint8_t* pixels,
                                                 uint32_t side);

/* replaces cve.h:81-82. */
CVE_B200_API cve_status cve_cipher_seeds_drawn(const cve_cipher* cipher,
                                               uint64_t* out);

/* ---- reference file pipelines -------------------- */

/* Same layout and defaults as the reference (cve.h:86-93). */
typedef struct cve_io_options {
  uint32_t workers;    /* 0 -> 8 */
  uint32_t rounds;     /* 0 -> 5 */
  int serial;          /* accepted, ignored (scheduling only) */
  uint16_t fps;        /* 0 -> 20; recorded in the container */
  uint32_t raw_width;  /* nonzero -> input is raw RGB24 of these dims */
  uint32_t raw_height;
} cve_io_options;

typedef enum cve_out_format {
  CVE_OUT_AUTO = 0,
  CVE_OUT_PPM = 1,
  CVE_OUT_RAW = 2
} cve_out_format;

/* replaces cve.h:97-99.  P6 file, directory of P6 frames, or raw RGB24 ->
 * CVE1 container (27-byte header + frame_count padded-square ciphertexts).
 * Frames are padded on the device; the container is byte-identical to the
 * reference's (PLCM and LASM keys). */
CVE_B200_API cve_status cve_encrypt_file(const char* key_hex,
                                         const cve_io_options* io,
                                         const char* in_path,
                                         const char* out_path);

/* replaces cve.h:110-113.  CVE1 -> one P6 (single frame), a directory of
 * frame_NNNNNN.ppm, or raw RGB24; cropped to the original dimensions.
 * Explicit workers/rounds must match the header (MISMATCH), as must the key's
 * map kind. */
CVE_B200_API cve_status cve_decrypt_file(const char* key_hex,
                                         const cve_io_options* io,
                                         cve_out_format format,
                                         const char* in_path,
                                         const char* out_path);

/* replaces cve.h:149-150 (row f3).  byte_count generator bytes for external
 * statistical suites: split over the `workers` (0 -> 8) generators derived
 * from the key, the first byte_count % workers getting one extra byte, each
 * worker's fresh stream written in worker order -- byte-identical to the
 * reference.  The generators run concurrently on the GPU. */
CVE_B200_API cve_status cve_nist_export(const char* key_hex, uint32_t workers,
                                        uint64_t byte_count,
                                        const char* out_path);

/* ---- reference statistical analysis and image tools */

/* Same layout as the reference (cve.h:117-125). */
typedef struct cve_analyze_options {
  const char* input;   /* P6 or CVE1 */
  const char* second;  /* optional same-size image for NPCR/UACI */
  uint32_t frame_index;  /* frame to take from a container */
  uint32_t second_frame_index;
  uint32_t samples;    /* adjacent-pair samples per direction, 0 -> 20000 */
  uint64_t seed;       /* sampling seed */
  int csv;             /* nonzero -> CSV, else key=value report */
} cve_analyze_options;

/* replaces cve.h:127-128.  Per-channel histogram variance, chi^2 (+ the
 * 5 % uniformity verdict), entropy, local entropy over 30 disjoint 44x44
 * blocks, horizontal / vertical / diagonal adjacent-pixel correlation over
 * `samples` random pairs, and NPCR/UACI against `second` -- the same text,
 * byte for byte, as the reference.  The histograms and NPCR/UACI counts are
 * taken on the GPU.  *text_out is malloc'd: free with cve_string_free. */
CVE_B200_API cve_status cve_analyze(const cve_analyze_options* options, char** text_out);

/* replaces cve.h:132-134.  Salt-and-pepper noise over round(rate * side^2)
 * distinct pixels of every frame (seed + frame index); P6 or CVE1 in, same
 * format out, byte-identical to the reference. */
CVE_B200_API cve_status cve_add_noise_file(const char* in_path, const char* out_path,
                                           double rate, uint64_t seed);

/* Same layout as the reference (cve.h:136-141). */
typedef struct cve_crop_block {
  uint32_t x;     /* column of the upper-left corner */
  uint32_t y;     /* row of the upper-left corner */
  uint32_t side;
  uint8_t fill;   /* 0x00 or 0xFF */
} cve_crop_block;

/* replaces cve.h:143-145.  Square blocks filled with 0x00 / 0xFF in every
 * frame; byte-identical to the reference. */
CVE_B200_API cve_status cve_crop_file(const char* in_path, const char* out_path,
                                      const cve_crop_block* blocks, size_t block_count);

/* ---- the reference's benchmark and sweep entry points (cve.h:153-206) ---
 * Same option structs (0 / NULL -> the reference's defaults), the same CSV
 * schemas (bench.cpp:111-123, 165-184, 233-257, 303-315) and status codes,
 * run on this engine.  *csv_out is malloc'd: free with cve_string_free. */

/* Same layout as the reference (cve.h:155-161). */
typedef struct cve_bench_bytegen_options {
  const char* key_hex;          /* NULL -> fresh key of map_kind */
  cve_map_kind map_kind;
  const uint32_t* worker_counts;
  size_t worker_count_len;      /* 0 -> {1,2,4,8} */
  uint64_t iterations;          /* map iterations in total, 0 -> 50000000 */
} cve_bench_bytegen_options;

/* replaces cve.h:163-164 ("bench bytegen on K1").  One
 * CSV row per worker count: `iterations` generator iterations in total over
 * the workers' generators advancing together on the GPU (derivation, warm-up
 * and allocation outside the timed window; the bytes stay on the device). */
CVE_B200_API cve_status cve_bench_bytegen(const cve_bench_bytegen_options* options,
                                          char** csv_out);

/* Same layout as the reference (cve.h:166-174).  `serial` is accepted and
 * ignored, like `parallel` of cve_cipher_create. */
typedef struct cve_bench_phases_options {
  const char* key_hex;
  cve_map_kind map_kind;
  uint32_t side;     /* 0 -> 960 */
  uint32_t workers;  /* 0 -> 8 */
  uint32_t rounds;   /* 0 -> 5 */
  uint32_t images;   /* 0 -> 100 */
  int serial;
} cve_bench_phases_options;

/* replaces cve.h:176-177.  Confusion-only and diffusion-only transforms
 * (reference Engine::transform, engine.cpp:302-307) of noise images; the two
 * halves run as separate kernels here -- these are NOT the fused production
 * rounds, whose time cve_bench_video reports.  Host-clock times; the
 * diffusion columns include keystream generation, as in the reference. */
CVE_B200_API cve_status cve_bench_phases(const cve_bench_phases_options* options,
                                         char** csv_out);

/* Same layout as the reference (cve.h:179-189). */
typedef struct cve_bench_video_options {
  const char* key_hex;
  cve_map_kind map_kind;
  const uint32_t* sides;
  size_t side_len;   /* 0 -> {96,192,288,384,480,576,672,768} */
  uint32_t workers;  /* 0 -> 8 */
  uint32_t rounds;   /* 0 -> 5 */
  uint32_t frames;   /* 0 -> 600 */
  uint16_t fps;      /* 0 -> 20; realtime_ok means mean <= 1000/fps ms */
  int serial;
} cve_bench_video_options;

/* replaces cve.h:191-192 (the reference's timing method, bench.cpp:186-231):
 * per side, `frames` synchronous in-place frame encryptions of noise frames
 * on host memory, each timed on the host clock.  bytegen_mean_ms = the
 * generator kernels' device time per frame, confuse_mean_ms = the fused
 * confusion+diffusion round kernels' device time per frame, diffuse_mean_ms
 * = 0.000 (no separate diffusion pass exists to time). */
CVE_B200_API cve_status cve_bench_video(const cve_bench_video_options* options,
                                        char** csv_out);

/* Same layout as the reference (cve.h:194-202). */
typedef struct cve_sweep_options {
  const char* key_hex;
  cve_map_kind map_kind;
  const char* input;    /* P6 plain image; NULL -> synthetic */
  uint32_t synth_side;  /* 0 -> 512 */
  uint32_t workers;     /* 0 -> 1 */
  uint32_t max_rounds;  /* 0 -> 10 */
  uint64_t seed;
} cve_sweep_options;

/* replaces cve.h:206.  Per-round NPCR/UACI under a one-byte plaintext change
 * (diffusion rounds only) and plain-vs-scrambled correlation (confusion
 * rounds only), rounds 0..max_rounds: deterministic, byte-identical to the
 * reference's CSV for the same key, image and seed. */
CVE_B200_API cve_status cve_sweep_rounds(const cve_sweep_options* options, char** csv_out);

/* Additive: the reference's Engine::transform (engine.cpp:302-307) as a frame
 * call -- the transform behind cve_bench_phases and cve_sweep_rounds.  One
 * frame in place through `rounds` rounds (1..255) with confusion and / or
 * diffusion switched off (both on: the same bytes as
 * cve_cipher_encrypt_frame with that many rounds).  Like a frame call it is
 * the handle's next frame: it draws one confusion seed and, with diffusion on,
 * rounds * side*side*3 / workers stream bytes per worker; MISMATCH comes
 * after the seed draw.  states_out (optional, NULL to skip): rounds *
 * side*side*3 bytes, the frame after each round.  Single-device handles. */
CVE_B200_API cve_status cve_cipher_transform_frame(cve_cipher* cipher, uint8_t* pixels,
                                                   uint32_t side, uint32_t rounds,
                                                   int confusion, int diffusion,
                                                   uint8_t* states_out);

/* ---- additive: batched / device-resident / introspection ---------------- */

/* Additive (row f4 on resident frames): the analysis reductions of a
 * side x side RGB24 frame already in device memory, ordered on `stream`
 * (a cudaStream_t; NULL = legacy default stream), without copying the frame.
 * hist_out (device, 768 x u64): hist_out[c*256 + v] = pixels of channel c
 * with value v.  With `second` (device frame of the same side) and diff_out
 * (device, 6 x u64): diff_out[c] = positions where channel c differs,
 * diff_out[3 + c] = sum of |a - b| over channel c (NPCR/UACI numerators). */
CVE_B200_API cve_status cve_frame_stats_device(const uint8_t* frame, const uint8_t* second,
                                               uint32_t side, uint64_t* hist_out,
                                               uint64_t* diff_out, void* stream);

/* The reference's padded_side (frame.cpp:19-26): smallest multiple of
 * `workers` covering max(width, height). */
CVE_B200_API cve_status cve_padded_side(uint32_t width, uint32_t height,
                                        uint32_t workers, uint32_t* side_out);

/* `count` unpadded width x height RGB24 frames (packed) -> `count` padded
 * side x side ciphertexts (side = cve_padded_side(width, height, workers)).
 * Padding (zero rows bottom, zero columns right, frame.cpp:28-39) is done on
 * the device, so only width*height*3 bytes per frame cross PCIe. */
CVE_B200_API cve_status cve_cipher_encrypt_frames_wh(cve_cipher* cipher,
                                                     const uint8_t* rgb,
                                                     uint32_t width,
                                                     uint32_t height,
                                                     uint32_t count,
                                                     uint8_t* out_square);

/* Inverse: `count` side x side ciphertexts -> `count` cropped width x height
 * plaintexts (frame.cpp:41-51), cropped on the device. */
CVE_B200_API cve_status cve_cipher_decrypt_frames_wh(cve_cipher* cipher,
                                                     const uint8_t* square,
                                                     uint32_t side,
                                                     uint32_t width,
                                                     uint32_t height,
                                                     uint32_t count,
                                                     uint8_t* out_rgb);

/* `count` consecutive square frames, contiguous in host memory
 * (count*side*side*3 bytes), processed in place as frames k..k+count-1 of
 * the handle.  H2D copy, keystream generation, cipher rounds and D2H copy
 * overlap across frames.  Pinned (cudaHostAlloc'd / registered) buffers are
 * copied by DMA asynchronously; pageable buffers work too but each copy then
 * goes through the driver's staging and blocks the host.  Same validation as the per-frame call; on MISMATCH one seed is
 * drawn (as the first of `count` per-frame calls would) and no data is
 * touched.  count == 0 is INVALID_ARGUMENT. */
CVE_B200_API cve_status cve_cipher_encrypt_frames(cve_cipher* cipher,
                                                  uint8_t* pixels,
                                                  uint32_t side,
                                                  uint32_t count);
CVE_B200_API cve_status cve_cipher_decrypt_frames(cve_cipher* cipher,
                                                  uint8_t* pixels,
                                                  uint32_t side,
                                                  uint32_t count);

/* Same, on frames already resident in device memory of the handle's GPU.
 * Work is ordered after everything previously enqueued on `stream`
 * (a cudaStream_t, or NULL for the legacy default stream), and `stream` is
 * made to wait for its completion before the call returns -- the call itself
 * does not block the host.  `d_pixels` must stay valid until `stream`
 * reaches that point. */
CVE_B200_API cve_status cve_cipher_encrypt_frames_async(cve_cipher* cipher,
                                                        uint8_t* d_pixels,
                                                        uint32_t side,
                                                        uint32_t count,
                                                        void* stream);
CVE_B200_API cve_status cve_cipher_decrypt_frames_async(cve_cipher* cipher,
                                                        uint8_t* d_pixels,
                                                        uint32_t side,
                                                        uint32_t count,
                                                        void* stream);

/* ---- additive: one clip sharded across GPUs (north star "independent frames
 * of a clip are partitioned across the B200s") -------------- */

/* Like cve_cipher_create, but the clip's cipher work is spread over
 * `device_count` CUDA devices: the keystream generator of the clip (its 2n
 * sequential chaotic orbits, reference engine.cpp:174-176, 198-205) runs on
 * devices[0]; frame k is ciphered on shard k mod device_count, which pulls
 * that frame's keystream window (rounds * region bytes per subframe) out of
 * the generator's ring with a peer copy over NVLink and runs the shift table
 * and the rounds on its own device.  Entries may repeat (e.g. {0, 0}: two
 * shards on one GPU, each with its own streams and buffers).  Output is
 * byte-identical to a single-device handle: the k-th call still binds to
 * frame k (reference cve.h:72-74).  The host-buffer calls
 * (cve_cipher_encrypt_frame(s), _wh) deal frames to the shards round-robin
 * across calls.  device_count == 1 is cve_cipher_create on devices[0].
 * A device index out of range -> INVALID_ARGUMENT. */
CVE_B200_API cve_status cve_cipher_create_devices(const char* key_hex, uint32_t workers,
                                                  uint32_t rounds, const int* devices,
                                                  uint32_t device_count, cve_cipher** out);

/* Number of cipher shards of the handle (1 for cve_cipher_create) and, if
 * devices_out is not NULL, the device of shard i in devices_out[i] (i < cap). */
CVE_B200_API cve_status cve_cipher_shards(const cve_cipher* cipher, uint32_t* count_out,
                                          int* devices_out, uint32_t cap);

/* Device-resident frames of a sharded handle: batch frame f is processed on
 * shard g = f % G (G = cve_cipher_shards) and lives in that shard's device
 * memory at shard_pixels[g] + (f / G) * side*side*3, in place.  streams[g]
 * (a cudaStream_t of shard g's device, or NULL for its legacy default
 * stream; `streams` itself may be NULL) orders shard g's frames like
 * cve_cipher_encrypt_frames_async: after prior work on it, and it waits for
 * their completion; the call does not block the host.  On a single-device
 * handle this is cve_cipher_encrypt_frames_async(shard_pixels[0], streams[0]). */
CVE_B200_API cve_status cve_cipher_encrypt_frames_sharded_async(cve_cipher* cipher,
                                                                uint8_t* const* shard_pixels,
                                                                uint32_t side, uint32_t count,
                                                                void* const* streams);
CVE_B200_API cve_status cve_cipher_decrypt_frames_sharded_async(cve_cipher* cipher,
                                                                uint8_t* const* shard_pixels,
                                                                uint32_t side, uint32_t count,
                                                                void* const* streams);

/* Blocks until every operation of the handle has finished. */
CVE_B200_API cve_status cve_cipher_synchronize(cve_cipher* cipher);

/* Selects the CUDA device used by handles created afterwards on this thread
 * (default: the current device). */
CVE_B200_API cve_status cve_set_device(int device);

/* Streams used by each handle created afterwards (process-wide; 1 or 2,
 * default 2 or $CVE_B200_STREAMS_PER_HANDLE).  2: the generator chain has its
 * own stream, so one clip never waits for its own cipher rounds (best for a
 * single clip).  1: one hardware queue per handle, so up to
 * CUDA_DEVICE_MAX_CONNECTIONS concurrent handles never share a queue (best
 * for many concurrent clips). */
CVE_B200_API cve_status cve_set_streams_per_handle(uint32_t streams);

/* Round fusion for handles created afterwards (process-wide; default 0 or
 * $CVE_B200_ROUND_FUSION).  1: frames that fit one thread-block cluster
 * (side % 16 == 0 and two packed copies of a CTA's whole bands in 227 KB: up
 * to ~768^2) are encrypted with ALL rounds in one cluster kernel -- the frame
 * is read from and written to HBM once and every round stays in distributed
 * shared memory, on 8-16 SMs per frame.  0: one kernel per round over the
 * whole GPU (measured faster on B200, per frame and for many concurrent
 * clips).  Output is identical in both modes.  Other values ->
 * INVALID_ARGUMENT. */
CVE_B200_API cve_status cve_set_round_fusion(uint32_t mode);

/* Copies the next `len` keystream bytes of subframe generator `worker` to
 * host memory WITHOUT consuming them from the cipher's stream (diagnostics /
 * parity; the reference's per-worker Prbg output, chaos.cpp:143-153). */
CVE_B200_API cve_status cve_cipher_peek_keystream(cve_cipher* cipher,
                                                  uint32_t worker,
                                                  uint8_t* out, size_t len);

/* Runs the keystream generator ahead so that the next `bytes` bytes per
 * worker (beyond the current stream position) are produced before the
 * frames that will consume them arrive.  Does not consume them.
 * Asynchronous on the handle's streams. */
CVE_B200_API cve_status cve_cipher_prefetch_keystream(cve_cipher* cipher,
                                                      uint64_t bytes);

/* Profiling counters of the handle (cumulative since create). */
typedef struct cve_cipher_stats {
  uint64_t frames;           /* frames completed (encrypt + decrypt) */
  uint64_t keystream_iters;  /* generator iterations per lane (6 B PLCM, 12 B LASM) */
  uint64_t kernel_launches;  /* CUDA kernels launched by this handle */
  uint64_t prbg_launches;    /* of which keystream-generator launches */
  uint64_t guard_replays;    /* PLCM workers recomputed exactly (0 for LASM) */
  double prbg_ms;            /* device time of generator launches */
  double chain_ms;           /* of which the sequential chain kernel */
  double cipher_ms;          /* device time of cipher-round launches */
} cve_cipher_stats;

/* Fills *out.  Device times are read back from CUDA events and therefore
 * synchronize the handle. */
CVE_B200_API cve_status cve_cipher_get_stats(cve_cipher* cipher,
                                             cve_cipher_stats* out);

/* Keystream of one generator with explicit lanes {x0_a, p_a, x0_b, p_b},
 * computed by the GPU generator kernel: the reference's
 * Prbg(PlcmParams, PlcmParams).take(len) (chaos.cpp:79-91, 143-153).  Raw
 * generator bytes for external statistical suites (reference nist-export,
 * capi.cpp:385-415) and for parity tests.  Out-of-domain lanes -> BAD_KEY. */
CVE_B200_API cve_status cve_keystream_generate(const double lanes[4],
                                               uint8_t* out, size_t len);

/* Diagnostics: cve_keystream_generate with at most `launch_iters` generator
 * iterations per launch (0: no cap; the generator is pipelined as in a
 * cipher handle: the chain of launch L+1 runs while launch L is verified)
 * and, if guard_replays is not NULL, the number of worker launches the
 * exact fix-up recomputed (guard-set hits on the speculative chain,
 * chaos.cpp:18-24, and the launch after each, whose start it repairs).
 * flags: CVE_KEYSTREAM_DENSE_ORBIT selects the generator variant that
 * handles created with one stream per handle use (the chain stores every
 * orbit value; default: one checkpoint per 8 iterations).  Output is
 * identical to cve_keystream_generate either way. */
#define CVE_KEYSTREAM_DENSE_ORBIT 1u
CVE_B200_API cve_status cve_keystream_generate_ex(const double lanes[4], uint8_t* out,
                                                  size_t len, uint32_t launch_iters,
                                                  uint32_t flags, uint64_t* guard_replays);

/* LASM counterpart (row f2): lanes {x0_a, y0_a, mu_a, x0_b, y0_b, mu_b}, the
 * reference's Prbg(LasmParams, LasmParams).take(len) (chaos.cpp:93-107,
 * 119-153: 12 bytes per iteration).  Out-of-domain lanes -> BAD_KEY. */
CVE_B200_API cve_status cve_keystream_generate_lasm(const double lanes[6],
                                                    uint8_t* out, size_t len);

/* Diagnostics for row f2: y[i] = sin(x[i]) evaluated on the GPU by the
 * restatement of the host glibc's libm sin the LASM generator uses
 * (glibc_sin.cuh); bit-identical to the host's sin() for |x| < 105414350,
 * NaN beyond. */
CVE_B200_API cve_status cve_glibc_sin(const double* x, double* y, size_t count);

/* Host-only keying (no GPU needed): the lane table the key's coordinator
 * derives for `workers` subframes (reference keying.cpp:180-207) -- for PLCM
 * keys lanes_out[4*i .. 4*i+3] = x0_a, p_a, x0_b, p_b of subframe i, for LASM
 * keys lanes_out[6*i .. 6*i+5] = x0_a, y0_a, mu_a, x0_b, y0_b, mu_b --
 * followed by the first `nseeds` per-frame confusion seeds
 * (keying.cpp:209-218).  For key management and diagnostics; the cipher
 * handle does the same derivation internally. */
CVE_B200_API cve_status cve_derive_worker_lanes(const char* key_hex,
                                                uint32_t workers,
                                                double* lanes_out,
                                                uint32_t* seeds_out,
                                                size_t nseeds);

/* Device times (ms) of the keystream generator's chain kernel, one per
 * generator launch since the previous call, oldest first; *count receives the number available, at most `cap`
 * are copied to `out` (which may be NULL to query).  Synchronizes. */
CVE_B200_API cve_status cve_cipher_take_prbg_times(cve_cipher* cipher,
                                                   float* out, size_t cap,
                                                   size_t* count);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* CVE_B200_H */
