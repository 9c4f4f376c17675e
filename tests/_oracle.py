"""ctypes access to the CHECKERS (test infrastructure only).

* ``Oracle``    -- oracle/liboracle.so, the plain-C restatement of the
                   reference path (oracle/cve_oracle.c).
* ``Reference`` -- oracle/_ref/libcve_ref.so, the reference's own sources
                   compiled in place by oracle/Makefile (absent if the
                   reference was not available at build time).

Nothing in the product package imports this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcve_ref.so")


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class Oracle:
    lib = None

    def __init__(self, key_hex: str, workers: int, rounds: int = 5):
        L = Oracle.load()
        h = C.c_void_p()
        st = L.orc_cipher_create(key_hex.encode(), workers, rounds, C.byref(h))
        if st:
            raise ValueError(f"oracle create status {st}")
        self.h, self.workers, self.rounds = h, workers, rounds

    @classmethod
    def load(cls):
        if cls.lib is None:
            L = C.CDLL(ORACLE_SO)
            vp = C.c_void_p
            L.orc_cipher_create.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.POINTER(vp)]
            L.orc_cipher_destroy.argtypes = [vp]
            L.orc_cipher_encrypt_frame.argtypes = [vp, vp, C.c_uint32]
            L.orc_cipher_decrypt_frame.argtypes = [vp, vp, C.c_uint32]
            L.orc_cipher_transform_frame.argtypes = [vp, vp, C.c_uint32, C.c_uint32, C.c_int,
                                                     C.c_int, vp]
            L.orc_cipher_worker_stream.argtypes = [vp, C.c_uint32, vp, C.c_size_t]
            L.orc_cipher_next_seed.argtypes = [vp]
            L.orc_cipher_next_seed.restype = C.c_uint32
            L.orc_cipher_seeds_drawn.argtypes = [vp]
            L.orc_cipher_seeds_drawn.restype = C.c_uint64
            L.orc_cipher_params.argtypes = [vp]
            L.orc_cipher_params.restype = C.POINTER(C.c_double)
            L.orc_plcm_stream.argtypes = [C.c_double] * 4 + [vp, C.c_size_t]
            L.orc_lasm_stream.argtypes = [C.POINTER(C.c_double), vp, C.c_size_t]
            L.orc_lasm_iterate.argtypes = [C.POINTER(C.c_double)] * 2 + [C.c_double]
            L.orc_cipher_is_lasm.argtypes = [vp]
            L.orc_plcm_iterate.argtypes = [C.c_double, C.c_double]
            L.orc_plcm_iterate.restype = C.c_double
            L.orc_confusion_shift.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
            L.orc_confusion_shift.restype = C.c_int64
            L.orc_diffuse_byte.argtypes = [C.c_uint8] * 3
            L.orc_diffuse_byte.restype = C.c_uint8
            L.orc_inverse_diffuse_byte.argtypes = [C.c_uint8] * 3
            L.orc_inverse_diffuse_byte.restype = C.c_uint8
            L.orc_padded_side.argtypes = [C.c_uint32] * 3
            L.orc_padded_side.restype = C.c_uint32
            cls.lib = L
        return cls.lib

    def close(self):
        if self.h:
            Oracle.lib.orc_cipher_destroy(self.h)
            self.h = None

    __del__ = close

    def encrypt(self, frame: np.ndarray) -> int:
        return Oracle.lib.orc_cipher_encrypt_frame(self.h, _ptr(frame), frame.shape[0])

    def decrypt(self, frame: np.ndarray) -> int:
        return Oracle.lib.orc_cipher_decrypt_frame(self.h, _ptr(frame), frame.shape[0])

    def transform(self, frame: np.ndarray, rounds: int, confusion: bool, diffusion: bool,
                  states: np.ndarray = None) -> int:
        """Reference Engine::transform (engine.cpp:302-307); states (optional,
        (rounds, side, side, 3)) receives the frame after every round."""
        return Oracle.lib.orc_cipher_transform_frame(
            self.h, _ptr(frame), frame.shape[0], rounds, int(confusion), int(diffusion),
            _ptr(states) if states is not None else None)

    def worker_stream(self, worker: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint8)
        Oracle.lib.orc_cipher_worker_stream(self.h, worker, _ptr(out), n)
        return out

    def params(self) -> np.ndarray:
        """(workers, 4) PLCM lanes, or (workers, 6) LASM lanes."""
        per = 6 if Oracle.lib.orc_cipher_is_lasm(self.h) else 4
        p = Oracle.lib.orc_cipher_params(self.h)
        return np.ctypeslib.as_array(p, shape=(self.workers * per,)).reshape(self.workers,
                                                                             per).copy()

    @property
    def seeds_drawn(self) -> int:
        return Oracle.lib.orc_cipher_seeds_drawn(self.h)


def plcm_stream(xa, pa, xb, pb, n) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint8)
    st = Oracle.load().orc_plcm_stream(xa, pa, xb, pb, _ptr(out), n)
    assert st == 0
    return out


def lasm_stream(lanes, n) -> np.ndarray:
    """Reference Prbg(LasmParams, LasmParams).take(n), lanes = 6 doubles."""
    out = np.zeros(n, dtype=np.uint8)
    arr = (C.c_double * 6)(*[float(v) for v in lanes])
    st = Oracle.load().orc_lasm_stream(arr, _ptr(out), n)
    assert st == 0
    return out


def lasm_iterate(x, y, mu):
    xx, yy = C.c_double(x), C.c_double(y)
    Oracle.load().orc_lasm_iterate(C.byref(xx), C.byref(yy), mu)
    return xx.value, yy.value


class RefIo(C.Structure):
    _fields_ = [("workers", C.c_uint32), ("rounds", C.c_uint32), ("serial", C.c_int),
                ("fps", C.c_uint16), ("raw_width", C.c_uint32), ("raw_height", C.c_uint32)]


class Reference:
    """The reference's own C ABI (cve.h) from oracle/_ref/libcve_ref.so."""
    lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def load(cls):
        if cls.lib is None:
            L = C.CDLL(REF_SO)
            vp = C.c_void_p
            L.cve_cipher_create.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_int,
                                            C.POINTER(vp)]
            L.cve_cipher_destroy.argtypes = [vp]
            L.cve_cipher_encrypt_frame.argtypes = [vp, vp, C.c_uint32]
            L.cve_cipher_decrypt_frame.argtypes = [vp, vp, C.c_uint32]
            L.cve_cipher_seeds_drawn.argtypes = [vp, C.POINTER(C.c_uint64)]
            L.cve_last_error.restype = C.c_char_p
            L.cve_encrypt_file.argtypes = [C.c_char_p, C.POINTER(RefIo), C.c_char_p, C.c_char_p]
            L.cve_decrypt_file.argtypes = [C.c_char_p, C.POINTER(RefIo), C.c_int, C.c_char_p,
                                           C.c_char_p]
            L.cve_nist_export.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_char_p]
            cls.lib = L
        return cls.lib

    def __init__(self, key_hex: str, workers: int, rounds: int = 5, parallel: int = 1):
        L = Reference.load()
        h = C.c_void_p()
        st = L.cve_cipher_create(key_hex.encode(), workers, rounds, parallel, C.byref(h))
        if st:
            raise ValueError(f"reference create status {st}: {L.cve_last_error()}")
        self.h = h

    def close(self):
        if self.h:
            Reference.lib.cve_cipher_destroy(self.h)
            self.h = None

    __del__ = close

    def encrypt(self, frame: np.ndarray) -> int:
        return Reference.lib.cve_cipher_encrypt_frame(self.h, _ptr(frame), frame.shape[0])

    def decrypt(self, frame: np.ndarray) -> int:
        return Reference.lib.cve_cipher_decrypt_frame(self.h, _ptr(frame), frame.shape[0])


def ref_encrypt_file(key_hex, in_path, out_path, workers=0, rounds=0, fps=0, raw=None):
    w, h = raw if raw else (0, 0)
    io = RefIo(workers, rounds, 0, fps, w, h)
    return Reference.load().cve_encrypt_file(key_hex.encode(), C.byref(io), in_path.encode(),
                                             out_path.encode())


def ref_decrypt_file(key_hex, in_path, out_path, fmt=0):
    return Reference.load().cve_decrypt_file(key_hex.encode(), None, fmt, in_path.encode(),
                                             out_path.encode())


# ---- row f4: the reference's analysis and image tools ----------------------

class RefAnalyzeOptions(C.Structure):
    _fields_ = [("input", C.c_char_p), ("second", C.c_char_p), ("frame_index", C.c_uint32),
                ("second_frame_index", C.c_uint32), ("samples", C.c_uint32),
                ("seed", C.c_uint64), ("csv", C.c_int)]


class RefCropBlock(C.Structure):
    _fields_ = [("x", C.c_uint32), ("y", C.c_uint32), ("side", C.c_uint32), ("fill", C.c_uint8)]


def ref_analyze(input_path, second=None, frame_index=0, second_frame_index=0, samples=0,
                seed=0, csv=False):
    """(status, text) from the reference's cve_analyze."""
    L = Reference.load()
    L.cve_analyze.argtypes = [C.POINTER(RefAnalyzeOptions), C.POINTER(C.c_void_p)]
    L.cve_string_free.argtypes = [C.c_void_p]
    o = RefAnalyzeOptions(input_path.encode() if input_path else None,
                          second.encode() if second else None, frame_index,
                          second_frame_index, samples, seed, 1 if csv else 0)
    out = C.c_void_p()
    st = L.cve_analyze(C.byref(o), C.byref(out))
    if st:
        return st, None
    text = C.string_at(out).decode()
    L.cve_string_free(out)
    return 0, text


def ref_add_noise_file(in_path, out_path, rate, seed):
    L = Reference.load()
    L.cve_add_noise_file.argtypes = [C.c_char_p, C.c_char_p, C.c_double, C.c_uint64]
    return L.cve_add_noise_file(in_path.encode(), out_path.encode(), rate, seed)


def ref_crop_file(in_path, out_path, blocks):
    L = Reference.load()
    L.cve_crop_file.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(RefCropBlock), C.c_size_t]
    arr = (RefCropBlock * max(1, len(blocks)))(*[RefCropBlock(*b) for b in blocks])
    return L.cve_crop_file(in_path.encode(), out_path.encode(), arr if blocks else None,
                           len(blocks))


# ---- the reference's bench / sweep entry points (cve.h:153-206) -------------

class RefBytegenOptions(C.Structure):
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int),
                ("worker_counts", C.POINTER(C.c_uint32)), ("worker_count_len", C.c_size_t),
                ("iterations", C.c_uint64)]


class RefPhasesOptions(C.Structure):
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int), ("side", C.c_uint32),
                ("workers", C.c_uint32), ("rounds", C.c_uint32), ("images", C.c_uint32),
                ("serial", C.c_int)]


class RefVideoOptions(C.Structure):
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int),
                ("sides", C.POINTER(C.c_uint32)), ("side_len", C.c_size_t),
                ("workers", C.c_uint32), ("rounds", C.c_uint32), ("frames", C.c_uint32),
                ("fps", C.c_uint16), ("serial", C.c_int)]


class RefSweepOptions(C.Structure):
    _fields_ = [("key_hex", C.c_char_p), ("map_kind", C.c_int), ("input", C.c_char_p),
                ("synth_side", C.c_uint32), ("workers", C.c_uint32),
                ("max_rounds", C.c_uint32), ("seed", C.c_uint64)]


def _ref_csv(name, options):
    """(status, csv) from one of the reference's csv_out entry points."""
    L = Reference.load()
    fn = getattr(L, name)
    fn.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    fn.restype = C.c_int
    L.cve_string_free.argtypes = [C.c_void_p]
    out = C.c_void_p()
    st = fn(C.byref(options) if options is not None else None, C.byref(out))
    if st:
        return st, None
    text = C.string_at(out).decode()
    L.cve_string_free(out)
    return 0, text


def _u32s(values):
    vals = list(values or [])
    return ((C.c_uint32 * len(vals))(*vals) if vals else None), len(vals)


def ref_bench_bytegen(key_hex=None, map_kind=0, worker_counts=None, iterations=0):
    arr, n = _u32s(worker_counts)
    return _ref_csv("cve_bench_bytegen", RefBytegenOptions(
        key_hex.encode() if key_hex else None, map_kind, arr, n, iterations))


def ref_bench_phases(key_hex=None, map_kind=0, side=0, workers=0, rounds=0, images=0):
    return _ref_csv("cve_bench_phases", RefPhasesOptions(
        key_hex.encode() if key_hex else None, map_kind, side, workers, rounds, images, 0))


def ref_bench_video(key_hex=None, map_kind=0, sides=None, workers=0, rounds=0, frames=0, fps=0):
    arr, n = _u32s(sides)
    return _ref_csv("cve_bench_video", RefVideoOptions(
        key_hex.encode() if key_hex else None, map_kind, arr, n, workers, rounds, frames, fps, 0))


def ref_sweep_rounds(key_hex=None, map_kind=0, input_path=None, synth_side=0, workers=0,
                     max_rounds=0, seed=0):
    return _ref_csv("cve_sweep_rounds", RefSweepOptions(
        key_hex.encode() if key_hex else None, map_kind,
        input_path.encode() if input_path else None, synth_side, workers, max_rounds, seed))
