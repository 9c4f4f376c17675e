"""B200-native chaotic video cipher (arXiv 2302.07411) -- Python host mirror.

The product is ``libcve_b200.so`` (C ABI declared in ``include/cve_b200.h``):
host C++ keying + sm_100a CUDA kernels.  This module is a thin ctypes binding
that mirrors the reference's cipher-handle interface
(``/root/reference/proj/include/cve.h:60-82``) with the same names, argument
meaning and error behaviour, so tests read like the reference's test_capi.cpp.

There is no CPU fallback: if the shared library is missing, importing the
binding raises; if no B200 is present, ``Cipher(...)`` raises ``CveError``
with status ``CVE_ERROR_INTERNAL``.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Tuple

import numpy as np

__all__ = [
    "CveError", "Cipher", "lib", "lib_path", "key_validate", "key_generate",
    "derive_worker_lanes", "padded_side", "pad_to_square", "crop_to_original",
    "CVE_OK", "CVE_ERROR_INVALID_ARGUMENT", "CVE_ERROR_BAD_KEY",
    "CVE_ERROR_MISMATCH", "CVE_ERROR_INTERNAL", "CVE_MAP_PLCM", "CVE_MAP_LASM",
]

CVE_OK = 0
CVE_ERROR_INVALID_ARGUMENT = 1
CVE_ERROR_BAD_KEY = 2
CVE_ERROR_IO = 3
CVE_ERROR_BAD_FORMAT = 4
CVE_ERROR_MISMATCH = 5
CVE_ERROR_INTERNAL = 6
CVE_MAP_PLCM = 0
CVE_MAP_LASM = 1

_HERE = os.path.dirname(os.path.abspath(__file__))
# CVE_B200_LIBRARY: a variant build of the same library (tools/ experiments,
# e.g. `make OUT=... BUILD=... EXTRA=-D...`); the product loads the in-tree one.
lib_path = os.environ.get("CVE_B200_LIBRARY") or os.path.join(_HERE, "libcve_b200.so")


class CveError(RuntimeError):
    """A non-OK cve_status, with the library's thread-local detail string."""

    def __init__(self, status: int, detail: str):
        self.status = status
        self.detail = detail
        super().__init__(f"cve status {status}: {detail}")


class IoOptions(C.Structure):
    """cve_io_options (reference cve.h:86-93)."""
    _fields_ = [("workers", C.c_uint32), ("rounds", C.c_uint32), ("serial", C.c_int),
                ("fps", C.c_uint16), ("raw_width", C.c_uint32), ("raw_height", C.c_uint32)]


class AnalyzeOptions(C.Structure):
    """cve_analyze_options (reference cve.h:117-125)."""
    _fields_ = [("input", C.c_char_p), ("second", C.c_char_p), ("frame_index", C.c_uint32),
                ("second_frame_index", C.c_uint32), ("samples", C.c_uint32),
                ("seed", C.c_uint64), ("csv", C.c_int)]


class CropBlock(C.Structure):
    """cve_crop_block (reference cve.h:136-141)."""
    _fields_ = [("x", C.c_uint32), ("y", C.c_uint32), ("side", C.c_uint32), ("fill", C.c_uint8)]


class BenchBytegenOptions(C.Structure):
    """cve_bench_bytegen_options (reference cve.h:155-161)."""
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int),
                ("worker_counts", C.POINTER(C.c_uint32)), ("worker_count_len", C.c_size_t),
                ("iterations", C.c_uint64)]


class BenchPhasesOptions(C.Structure):
    """cve_bench_phases_options (reference cve.h:166-174)."""
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int), ("side", C.c_uint32),
                ("workers", C.c_uint32), ("rounds", C.c_uint32), ("images", C.c_uint32),
                ("serial", C.c_int)]


class BenchVideoOptions(C.Structure):
    """cve_bench_video_options (reference cve.h:179-189)."""
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int),
                ("sides", C.POINTER(C.c_uint32)), ("side_len", C.c_size_t),
                ("workers", C.c_uint32), ("rounds", C.c_uint32), ("frames", C.c_uint32),
                ("fps", C.c_uint16), ("serial", C.c_int)]


class SweepOptions(C.Structure):
    """cve_sweep_options (reference cve.h:194-202)."""
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int), ("input", C.c_char_p),
                ("synth_side", C.c_uint32), ("workers", C.c_uint32),
                ("max_rounds", C.c_uint32), ("seed", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("frames", C.c_uint64), ("keystream_iters", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("prbg_launches", C.c_uint64),
                ("guard_replays", C.c_uint64), ("prbg_ms", C.c_double),
                ("chain_ms", C.c_double), ("cipher_ms", C.c_double)]


def _load() -> C.CDLL:
    if not os.path.exists(lib_path):
        raise ImportError(
            f"{lib_path} is not built; run `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (there is no CPU fallback)")
    L = C.CDLL(lib_path)
    u8p, vp = C.POINTER(C.c_uint8), C.c_void_p
    sig = {
        "cve_version": (C.c_char_p, []),
        "cve_status_message": (C.c_char_p, [C.c_int]),
        "cve_last_error": (C.c_char_p, []),
        "cve_string_free": (None, [vp]),
        "cve_key_generate": (C.c_int, [C.c_int, C.c_char_p, C.c_size_t]),
        "cve_key_validate": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
        "cve_cipher_create": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_int,
                                        C.POINTER(vp)]),
        "cve_cipher_create_devices": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32,
                                                C.POINTER(C.c_int), C.c_uint32, C.POINTER(vp)]),
        "cve_cipher_shards": (C.c_int, [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_int),
                                        C.c_uint32]),
        "cve_cipher_encrypt_frames_sharded_async": (C.c_int, [vp, C.POINTER(vp), C.c_uint32,
                                                              C.c_uint32, C.POINTER(vp)]),
        "cve_cipher_decrypt_frames_sharded_async": (C.c_int, [vp, C.POINTER(vp), C.c_uint32,
                                                              C.c_uint32, C.POINTER(vp)]),
        "cve_cipher_destroy": (None, [vp]),
        "cve_cipher_encrypt_frame": (C.c_int, [vp, vp, C.c_uint32]),
        "cve_cipher_decrypt_frame": (C.c_int, [vp, vp, C.c_uint32]),
        "cve_cipher_seeds_drawn": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
        "cve_cipher_transform_frame": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                                 vp]),
        "cve_cipher_encrypt_frames": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32]),
        "cve_cipher_decrypt_frames": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32]),
        "cve_cipher_encrypt_frames_async": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, vp]),
        "cve_cipher_decrypt_frames_async": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, vp]),
        "cve_cipher_synchronize": (C.c_int, [vp]),
        "cve_set_device": (C.c_int, [C.c_int]),
        "cve_set_streams_per_handle": (C.c_int, [C.c_uint32]),
        "cve_set_round_fusion": (C.c_int, [C.c_uint32]),
        "cve_cipher_peek_keystream": (C.c_int, [vp, C.c_uint32, vp, C.c_size_t]),
        "cve_cipher_prefetch_keystream": (C.c_int, [vp, C.c_uint64]),
        "cve_cipher_get_stats": (C.c_int, [vp, C.POINTER(Stats)]),
        "cve_cipher_take_prbg_times": (C.c_int, [vp, C.POINTER(C.c_float), C.c_size_t,
                                                 C.POINTER(C.c_size_t)]),
        "cve_encrypt_file": (C.c_int, [C.c_char_p, C.POINTER(IoOptions), C.c_char_p, C.c_char_p]),
        "cve_decrypt_file": (C.c_int, [C.c_char_p, C.POINTER(IoOptions), C.c_int, C.c_char_p,
                                       C.c_char_p]),
        "cve_nist_export": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint64, C.c_char_p]),
        "cve_analyze": (C.c_int, [C.POINTER(AnalyzeOptions), C.POINTER(vp)]),
        "cve_add_noise_file": (C.c_int, [C.c_char_p, C.c_char_p, C.c_double, C.c_uint64]),
        "cve_crop_file": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(CropBlock), C.c_size_t]),
        "cve_bench_bytegen": (C.c_int, [C.POINTER(BenchBytegenOptions), C.POINTER(vp)]),
        "cve_bench_phases": (C.c_int, [C.POINTER(BenchPhasesOptions), C.POINTER(vp)]),
        "cve_bench_video": (C.c_int, [C.POINTER(BenchVideoOptions), C.POINTER(vp)]),
        "cve_sweep_rounds": (C.c_int, [C.POINTER(SweepOptions), C.POINTER(vp)]),
        "cve_frame_stats_device": (C.c_int, [vp, vp, C.c_uint32, vp, vp, vp]),
        "cve_padded_side": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]),
        "cve_cipher_encrypt_frames_wh": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp]),
        "cve_cipher_decrypt_frames_wh": (C.c_int, [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32,
                                                   C.c_uint32, vp]),
        "cve_keystream_generate": (C.c_int, [C.POINTER(C.c_double), vp, C.c_size_t]),
        "cve_keystream_generate_lasm": (C.c_int, [C.POINTER(C.c_double), vp, C.c_size_t]),
        "cve_keystream_generate_ex": (C.c_int, [C.POINTER(C.c_double), vp, C.c_size_t,
                                                C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]),
        "cve_glibc_sin": (C.c_int, [vp, vp, C.c_size_t]),
        "cve_derive_worker_lanes": (C.c_int, [C.c_char_p, C.c_uint32,
                                              C.POINTER(C.c_double),
                                              C.POINTER(C.c_uint32), C.c_size_t]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    del u8p
    return L


lib = _load()


def _check(status: int) -> None:
    if status != CVE_OK:
        raise CveError(status, lib.cve_last_error().decode(errors="replace"))


def _as_key(key) -> bytes:
    return key.encode() if isinstance(key, str) else bytes(key)


def key_validate(key_hex) -> int:
    """Returns the map kind (CVE_MAP_PLCM / CVE_MAP_LASM); raises on a bad key."""
    kind = C.c_int(-1)
    _check(lib.cve_key_validate(_as_key(key_hex), C.byref(kind)))
    return kind.value


def key_generate(kind: int = CVE_MAP_PLCM) -> str:
    buf = C.create_string_buffer(80)
    _check(lib.cve_key_generate(kind, buf, len(buf)))
    return buf.value.decode()


def derive_worker_lanes(key_hex, workers: int, seeds: int = 0
                        ) -> Tuple[np.ndarray, np.ndarray]:
    """Host keying only (no GPU): the lane table the coordinator derives --
    (workers, 4) = (x0_a, p_a, x0_b, p_b) for PLCM keys, (workers, 6) =
    (x0_a, y0_a, mu_a, x0_b, y0_b, mu_b) for LASM keys -- then `seeds`
    confusion seeds (reference keying.cpp:164-218)."""
    per = 6 if key_validate(key_hex) == CVE_MAP_LASM else 4
    lanes = np.zeros((workers, per), dtype=np.float64)
    out = np.zeros(max(seeds, 1), dtype=np.uint32)
    _check(lib.cve_derive_worker_lanes(
        _as_key(key_hex), workers, lanes.ctypes.data_as(C.POINTER(C.c_double)),
        out.ctypes.data_as(C.POINTER(C.c_uint32)), seeds))
    return lanes, out[:seeds]


def keystream_generate(lanes, length: int) -> np.ndarray:
    """GPU keystream of one generator with explicit lanes (x0_a, p_a, x0_b, p_b)."""
    lan = (C.c_double * 4)(*[float(v) for v in lanes])
    out = np.zeros(length, dtype=np.uint8)
    _check(lib.cve_keystream_generate(lan, out.ctypes.data, length))
    return out


def keystream_generate_ex(lanes, length: int, launch_iters: int = 0, dense: bool = False):
    """keystream_generate with a cap on iterations per generator launch and
    the generator variant (dense: every orbit value stored, as for handles
    with one stream per handle); returns (bytes, guard_replays) -- the worker
    launches the exact fix-up recomputed."""
    lan = (C.c_double * 4)(*[float(v) for v in lanes])
    out = np.zeros(length, dtype=np.uint8)
    rep = C.c_uint64()
    _check(lib.cve_keystream_generate_ex(lan, out.ctypes.data, length, launch_iters,
                                         1 if dense else 0, C.byref(rep)))
    return out, rep.value


def keystream_generate_lasm(lanes, length: int) -> np.ndarray:
    """GPU keystream of one LASM generator with explicit lanes
    (x0_a, y0_a, mu_a, x0_b, y0_b, mu_b): 12 bytes per iteration."""
    lan = (C.c_double * 6)(*[float(v) for v in lanes])
    out = np.zeros(length, dtype=np.uint8)
    _check(lib.cve_keystream_generate_lasm(lan, out.ctypes.data, length))
    return out


def glibc_sin(x: np.ndarray) -> np.ndarray:
    """sin of every element, evaluated on the GPU by the glibc restatement the
    LASM generator uses (diagnostics / parity)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    _check(lib.cve_glibc_sin(x.ctypes.data, y.ctypes.data, x.size))
    return y


# ---- file pipelines (reference cve.h:84-113) ----------------------------------

CVE_OUT_AUTO, CVE_OUT_PPM, CVE_OUT_RAW = 0, 1, 2


def _io(workers=0, rounds=0, fps=0, raw=None) -> IoOptions:
    w, h = raw if raw else (0, 0)
    return IoOptions(workers, rounds, 0, fps, w, h)


def encrypt_file(key_hex, in_path: str, out_path: str, workers: int = 0, rounds: int = 0,
                 fps: int = 0, raw=None) -> None:
    """P6 / directory of P6 / raw RGB24 (raw=(w, h)) -> CVE1 container."""
    io = _io(workers, rounds, fps, raw)
    _check(lib.cve_encrypt_file(_as_key(key_hex), C.byref(io), in_path.encode(),
                                out_path.encode()))


def decrypt_file(key_hex, in_path: str, out_path: str, fmt: int = CVE_OUT_AUTO,
                 workers: int = 0, rounds: int = 0, io: bool = True) -> None:
    """CVE1 -> P6 / directory of P6 / raw RGB24 (cropped)."""
    opts = _io(workers, rounds) if io else None
    _check(lib.cve_decrypt_file(_as_key(key_hex), C.byref(opts) if opts else None, fmt,
                                in_path.encode(), out_path.encode()))


def nist_export(key_hex, workers: int, byte_count: int, out_path: str) -> None:
    """Raw generator bytes for statistical suites (reference cve_nist_export)."""
    _check(lib.cve_nist_export(_as_key(key_hex) if key_hex is not None else None, workers,
                               byte_count, out_path.encode()))


# ---- frame model (reference frame.cpp:19-51) --------------------------------

def analyze(input_path: str, second: str = None, frame_index: int = 0,
            second_frame_index: int = 0, samples: int = 0, seed: int = 0,
            csv: bool = False) -> str:
    """Reference cve_analyze: histogram variance, chi^2, entropy, local
    entropy, adjacent-pixel correlations, NPCR/UACI -- the same text.  The
    histograms and NPCR/UACI counts run on the GPU."""
    o = AnalyzeOptions(input_path.encode(), second.encode() if second else None, frame_index,
                       second_frame_index, samples, seed, 1 if csv else 0)
    out = C.c_void_p()
    _check(lib.cve_analyze(C.byref(o), C.byref(out)))
    try:
        return C.string_at(out).decode()
    finally:
        lib.cve_string_free(out)


def add_noise_file(in_path: str, out_path: str, rate: float, seed: int) -> None:
    """Reference cve_add_noise_file (salt-and-pepper, every frame)."""
    _check(lib.cve_add_noise_file(in_path.encode(), out_path.encode(), rate, seed))


def crop_file(in_path: str, out_path: str, blocks) -> None:
    """Reference cve_crop_file; blocks = [(x, y, side, fill), ...]."""
    arr = (CropBlock * max(1, len(blocks)))(*[CropBlock(*b) for b in blocks])
    _check(lib.cve_crop_file(in_path.encode(), out_path.encode(), arr if blocks else None,
                             len(blocks)))


def _csv_call(fn, options) -> str:
    out = C.c_void_p()
    _check(fn(C.byref(options), C.byref(out)))
    try:
        return C.string_at(out).decode()
    finally:
        lib.cve_string_free(out)


def _u32_array(values):
    vals = list(values or [])
    return ((C.c_uint32 * len(vals))(*vals) if vals else None), len(vals)


def bench_bytegen(key_hex=None, map_kind: int = CVE_MAP_PLCM, worker_counts=None,
                  iterations: int = 0) -> str:
    """Reference cve_bench_bytegen on the GPU generator: one CSV row per worker
    count (default 1, 2, 4, 8), `iterations` map iterations in total."""
    arr, n = _u32_array(worker_counts)
    o = BenchBytegenOptions(_as_key(key_hex) if key_hex is not None else None, map_kind, arr, n,
                            iterations)
    return _csv_call(lib.cve_bench_bytegen, o)


def bench_phases(key_hex=None, map_kind: int = CVE_MAP_PLCM, side: int = 0, workers: int = 0,
                 rounds: int = 0, images: int = 0) -> str:
    """Reference cve_bench_phases: confusion-only and diffusion-only transforms."""
    o = BenchPhasesOptions(_as_key(key_hex) if key_hex is not None else None, map_kind, side,
                           workers, rounds, images, 0)
    return _csv_call(lib.cve_bench_phases, o)


def bench_video(key_hex=None, map_kind: int = CVE_MAP_PLCM, sides=None, workers: int = 0,
                rounds: int = 0, frames: int = 0, fps: int = 0) -> str:
    """Reference cve_bench_video (its timing method): per-frame synchronous calls."""
    arr, n = _u32_array(sides)
    o = BenchVideoOptions(_as_key(key_hex) if key_hex is not None else None, map_kind, arr, n,
                          workers, rounds, frames, fps, 0)
    return _csv_call(lib.cve_bench_video, o)


def sweep_rounds(key_hex=None, map_kind: int = CVE_MAP_PLCM, input_path: str = None,
                 synth_side: int = 0, workers: int = 0, max_rounds: int = 0,
                 seed: int = 0) -> str:
    """Reference cve_sweep_rounds: per-round NPCR/UACI and confusion correlation."""
    o = SweepOptions(_as_key(key_hex) if key_hex is not None else None, map_kind,
                     input_path.encode() if input_path else None, synth_side, workers,
                     max_rounds, seed)
    return _csv_call(lib.cve_sweep_rounds, o)


def frame_stats_device(frame_ptr: int, side: int, hist_ptr: int, second_ptr: int = 0,
                       diff_ptr: int = 0, stream: int = 0) -> None:
    """Histograms (768 x u64 at hist_ptr) and NPCR/UACI counts (6 x u64 at
    diff_ptr) of a device-resident frame, ordered on `stream`."""
    _check(lib.cve_frame_stats_device(frame_ptr, second_ptr or None, side, hist_ptr or None,
                                      diff_ptr or None, stream or None))


def padded_side(width: int, height: int, workers: int) -> int:
    out = C.c_uint32()
    _check(lib.cve_padded_side(width, height, workers, C.byref(out)))
    return out.value


def pad_to_square(rgb: np.ndarray, workers: int) -> np.ndarray:
    """(h, w, 3) uint8 -> (side, side, 3), zero rows bottom / columns right."""
    h, w = rgb.shape[:2]
    side = padded_side(w, h, workers)
    out = np.zeros((side, side, 3), dtype=np.uint8)
    out[:h, :w] = rgb
    return out


def crop_to_original(frame: np.ndarray, width: int, height: int) -> np.ndarray:
    if width > frame.shape[1] or height > frame.shape[0]:
        raise CveError(CVE_ERROR_INVALID_ARGUMENT, "original dimensions exceed the frame side")
    return np.ascontiguousarray(frame[:height, :width])


# ---- the cipher handle --------------------------------------------------------

class Cipher:
    """One streaming cipher handle (reference cve_cipher, cve.h:62-82).

    The k-th encrypt or decrypt call binds to frame index k of the clip.
    ``devices`` (additive, cve_cipher_create_devices): shard the clip's cipher
    work over these CUDA devices -- the generator runs on devices[0], frame k
    on devices[k % len(devices)]; entries may repeat.
    """

    def __init__(self, key_hex, workers: int, rounds: int = 5, parallel: bool = True,
                 devices=None):
        h = C.c_void_p()
        if devices is None:
            _check(lib.cve_cipher_create(_as_key(key_hex), workers, rounds,
                                         1 if parallel else 0, C.byref(h)))
        else:
            devs = list(devices)
            arr = (C.c_int * max(1, len(devs)))(*devs)
            _check(lib.cve_cipher_create_devices(_as_key(key_hex), workers, rounds, arr,
                                                 len(devs), C.byref(h)))
        self._h = h
        self.workers = workers
        self.rounds = rounds

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "cipher is closed")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            if lib is not None:  # interpreter shutdown may have cleared it
                lib.cve_cipher_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @staticmethod
    def _frames(buf: np.ndarray) -> Tuple[int, int]:
        if buf.dtype != np.uint8 or not buf.flags.c_contiguous:
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "need a C-contiguous uint8 array")
        if buf.ndim == 3:
            count, side = 1, buf.shape[0]
        elif buf.ndim == 4:
            count, side = buf.shape[0], buf.shape[1]
        else:
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "need (side,side,3) or (n,side,side,3)")
        if buf.shape[-3:] != (side, side, 3):
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "frames must be square RGB24")
        return count, side

    def encrypt_frame(self, frame: np.ndarray) -> None:
        """In place, like cve_cipher_encrypt_frame."""
        _, side = self._frames(frame)
        _check(lib.cve_cipher_encrypt_frame(self.handle, frame.ctypes.data, side))

    def decrypt_frame(self, frame: np.ndarray) -> None:
        _, side = self._frames(frame)
        _check(lib.cve_cipher_decrypt_frame(self.handle, frame.ctypes.data, side))

    def transform_frame(self, frame: np.ndarray, rounds: int, confusion: bool = True,
                        diffusion: bool = True, states: bool = False):
        """Reference Engine::transform as a frame call (the handle's next
        frame), in place; states=True returns the (rounds, side, side, 3)
        frames after each round."""
        count, side = self._frames(frame[None] if frame.ndim == 3 else frame)
        if count != 1:
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "one frame at a time")
        out = np.empty((rounds, side, side, 3), np.uint8) if states else None
        _check(lib.cve_cipher_transform_frame(self.handle, frame.ctypes.data, side, rounds,
                                              1 if confusion else 0, 1 if diffusion else 0,
                                              out.ctypes.data if states else None))
        return out

    def encrypt_frames(self, frames: np.ndarray) -> None:
        count, side = self._frames(frames)
        _check(lib.cve_cipher_encrypt_frames(self.handle, frames.ctypes.data, side, count))

    def decrypt_frames(self, frames: np.ndarray) -> None:
        count, side = self._frames(frames)
        _check(lib.cve_cipher_decrypt_frames(self.handle, frames.ctypes.data, side, count))

    def encrypt_frames_device(self, ptr: int, side: int, count: int, stream: int = 0) -> None:
        """Frames resident in device memory (e.g. torch.Tensor.data_ptr())."""
        _check(lib.cve_cipher_encrypt_frames_async(self.handle, C.c_void_p(ptr), side,
                                                   count, C.c_void_p(stream)))

    def decrypt_frames_device(self, ptr: int, side: int, count: int, stream: int = 0) -> None:
        _check(lib.cve_cipher_decrypt_frames_async(self.handle, C.c_void_p(ptr), side,
                                                   count, C.c_void_p(stream)))

    @property
    def shards(self) -> list:
        """Device of each cipher shard (one entry for a single-device handle)."""
        n = C.c_uint32()
        devs = (C.c_int * 64)()
        _check(lib.cve_cipher_shards(self.handle, C.byref(n), devs, 64))
        return [devs[i] for i in range(min(n.value, 64))]

    def _sharded(self, fn, ptrs, side: int, count: int, streams=None) -> None:
        g = len(ptrs)
        arr = (C.c_void_p * g)(*[C.c_void_p(p) for p in ptrs])
        sarr = (C.c_void_p * g)(*[C.c_void_p(s) for s in (streams or [0] * g)])
        _check(fn(self.handle, arr, side, count, sarr))

    def encrypt_frames_sharded(self, ptrs, side: int, count: int, streams=None) -> None:
        """Device-resident frames of a sharded handle: batch frame f lives on
        shard f % G at ptrs[f % G] + (f // G) * side*side*3."""
        self._sharded(lib.cve_cipher_encrypt_frames_sharded_async, ptrs, side, count, streams)

    def decrypt_frames_sharded(self, ptrs, side: int, count: int, streams=None) -> None:
        self._sharded(lib.cve_cipher_decrypt_frames_sharded_async, ptrs, side, count, streams)

    def encrypt_frames_wh(self, rgb: np.ndarray) -> np.ndarray:
        """(count, h, w, 3) unpadded frames -> (count, side, side, 3) ciphertexts,
        padded on the device."""
        if rgb.ndim == 3:
            rgb = rgb[None]
        if rgb.dtype != np.uint8 or not rgb.flags.c_contiguous:
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "need a C-contiguous uint8 array")
        if rgb.ndim != 4 or rgb.shape[-1] != 3:
            raise CveError(CVE_ERROR_INVALID_ARGUMENT, "need (h,w,3) or (n,h,w,3) RGB24 frames")
        count, h, w = rgb.shape[:3]
        side = padded_side(w, h, self.workers)
        out = np.empty((count, side, side, 3), dtype=np.uint8)
        _check(lib.cve_cipher_encrypt_frames_wh(self.handle, rgb.ctypes.data, w, h, count,
                                                out.ctypes.data))
        return out

    def decrypt_frames_wh(self, square: np.ndarray, width: int, height: int) -> np.ndarray:
        """(count, side, side, 3) ciphertexts -> (count, height, width, 3) plaintexts."""
        if square.ndim == 3:
            square = square[None]
        count, side = self._frames(square)
        out = np.empty((count, height, width, 3), dtype=np.uint8)
        _check(lib.cve_cipher_decrypt_frames_wh(self.handle, square.ctypes.data, side, width,
                                                height, count, out.ctypes.data))
        return out

    def synchronize(self) -> None:
        _check(lib.cve_cipher_synchronize(self.handle))

    @property
    def seeds_drawn(self) -> int:
        v = C.c_uint64()
        _check(lib.cve_cipher_seeds_drawn(self.handle, C.byref(v)))
        return v.value

    def peek_keystream(self, worker: int, length: int) -> np.ndarray:
        out = np.zeros(length, dtype=np.uint8)
        _check(lib.cve_cipher_peek_keystream(self.handle, worker, out.ctypes.data, length))
        return out

    def prefetch_keystream(self, nbytes: int) -> None:
        _check(lib.cve_cipher_prefetch_keystream(self.handle, nbytes))

    def stats(self) -> dict:
        s = Stats()
        _check(lib.cve_cipher_get_stats(self.handle, C.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def take_prbg_times(self, cap: int = 1 << 20) -> np.ndarray:
        """Device times (ms) of the chain kernel, one per generator launch."""
        out = np.zeros(cap, dtype=np.float32)
        n = C.c_size_t()
        _check(lib.cve_cipher_take_prbg_times(
            self.handle, out.ctypes.data_as(C.POINTER(C.c_float)), cap, C.byref(n)))
        return out[:min(n.value, cap)].copy()


def set_device(device: int) -> None:
    _check(lib.cve_set_device(device))


def set_round_fusion(mode: int) -> None:
    """1 = all rounds of a frame in one thread-block cluster kernel wherever the
    frame fits (<= ~768^2); 0 (default) = one kernel per round.  Output is
    identical in both modes."""
    _check(lib.cve_set_round_fusion(mode))


def set_streams_per_handle(streams: int) -> None:
    """1: one hardware queue per handle (many concurrent clips); 2 (default):
    the generator chain on its own stream (best for one clip)."""
    _check(lib.cve_set_streams_per_handle(streams))

