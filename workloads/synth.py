"""Seeded synthetic workloads for the five BASELINE.json configs.

Harness-side only (the reference's own synth.cpp is out of scope, SURVEY.md
§2 row 9).  The paper's test images / videos are not available; these
generators stand in with the configs' shapes and value distributions:

* ``noise_frame``  -- i.i.d. uniform bytes, the reference's
  ``make_noise_frame`` recipe (synth.cpp:12-25: mt19937_64, 8 little-endian
  bytes per draw) -- config C1.
* ``correlated_frame`` -- C2..C5: per channel a smooth 2-D sinusoid plus a
  linear gradient, translating slowly with the frame index, plus
  approximately Gaussian noise (sigma = 8), clipped to [0, 255].  Built only
  from integer arithmetic and elementary IEEE operations (the sine table
  comes from glibc via ``math.sin``) so that frames are bit-reproducible on
  every host of this image -- golden digests made here hold on the GPU box.
* ``det_key`` -- the reference acceptance suite's deterministic-key recipe
  (acceptance.cpp:57-74: mt19937_64, 53-bit units, rejection of 0 and 1).
"""
from __future__ import annotations

import math
import struct
from typing import List

import numpy as np

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++ standard's 64-bit Mersenne Twister)."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _MASK64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK64
        self.mt, self.idx = mt, 312

    def _twist(self) -> None:
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64


def _f64_hex_le(v: float) -> str:
    return struct.pack("<d", v).hex()


def det_key(seed: int) -> str:
    """PLCM key hex from a seed (acceptance.cpp:57-74 recipe)."""
    rng = MT19937_64(seed)

    def unit() -> float:
        while True:
            u = float(rng() >> 11) * 2.0 ** -53
            if 0.0 < u < 1.0:
                return u

    x0a = unit()
    pa = 0.5 * unit()
    x0b = unit()
    pb = 0.5 * unit()
    return "00" + "".join(_f64_hex_le(v) for v in (x0a, pa, x0b, pb))


def det_key_lasm(seed: int) -> str:
    """LASM key hex from a seed (acceptance.cpp:57-74, LASM branch:
    {unit(), unit(), 0.44 + unit() * (0.93 - 0.44)})."""
    rng = MT19937_64(seed)

    def unit() -> float:
        while True:
            u = float(rng() >> 11) * 2.0 ** -53
            if 0.0 < u < 1.0:
                return u

    x0 = unit()
    y0 = unit()
    mu = 0.44 + unit() * (0.93 - 0.44)
    return "01" + "".join(_f64_hex_le(v) for v in (x0, y0, mu))


def flip_key_lsb(key_hex: str) -> str:
    """Flip the mantissa LSB of x0_a (key stays in-domain)."""
    raw = bytearray(bytes.fromhex(key_hex))
    raw[1] ^= 0x01
    return raw.hex()


def noise_frame(side: int, seed: int) -> np.ndarray:
    """(side, side, 3) uint8, make_noise_frame semantics (synth.cpp:12-25)."""
    n = side * side * 3
    rng = MT19937_64(seed)
    words = (n + 7) // 8
    buf = np.array([rng() for _ in range(words)], dtype=np.uint64)
    return buf.view(np.uint8)[:n].reshape(side, side, 3).copy()


_TABLE_BITS = 12
_SINE = np.array([round(1024.0 * math.sin(2.0 * math.pi * k / (1 << _TABLE_BITS)))
                  for k in range(1 << _TABLE_BITS)], dtype=np.int64)


def _clip_params(seed: int) -> np.ndarray:
    # per channel: fx, fy (cycles per frame), phase, speed, amp, gx, gy, base
    r = np.random.Generator(np.random.PCG64(seed))
    p = np.zeros((3, 8), dtype=np.int64)
    p[:, 0] = r.integers(1, 5, 3)
    p[:, 1] = r.integers(1, 5, 3)
    p[:, 2] = r.integers(0, 1 << _TABLE_BITS, 3)
    p[:, 3] = r.integers(3, 12, 3)          # table units per frame: slow drift
    p[:, 4] = r.integers(40, 80, 3)
    p[:, 5] = r.integers(-40, 41, 3)
    p[:, 6] = r.integers(-40, 41, 3)
    p[:, 7] = r.integers(100, 156, 3)
    return p


def correlated_frame(width: int, height: int, t: int, seed: int) -> np.ndarray:
    """(height, width, 3) uint8 frame t of a correlated clip."""
    params = _clip_params(seed)
    y = np.arange(height, dtype=np.int64)[:, None]
    x = np.arange(width, dtype=np.int64)[None, :]
    out = np.empty((height, width, 3), dtype=np.uint8)
    noise_rng = np.random.Generator(np.random.PCG64([seed, t]))
    mask = (1 << _TABLE_BITS) - 1
    for ch in range(3):
        fx, fy, ph, sp, amp, gx, gy, base = (int(v) for v in params[ch])
        phase = ph + sp * t
        ix = (fx * x * (1 << _TABLE_BITS) // width + phase) & mask
        iy = (fy * y * (1 << _TABLE_BITS) // height + 2 * phase) & mask
        smooth = amp * (_SINE[ix] + _SINE[iy]) // 2048
        grad = (gx * x) // width + (gy * y) // height
        # Irwin-Hall(4) of bytes: mean 510, sd 147.80 -> scaled to sd 8
        u = noise_rng.integers(0, 256, size=(4, height, width), dtype=np.uint8)
        ih = u.astype(np.int32).sum(axis=0) - 510
        noise = np.rint(ih.astype(np.float64) * (8.0 / 147.80)).astype(np.int64)
        v = base + smooth + grad + noise
        out[:, :, ch] = np.clip(v, 0, 255).astype(np.uint8)
    return out


# BASELINE.json configs (r = 5 everywhere).
CONFIGS = {
    "C1": dict(width=480, height=480, frames=1, workers=8, kind="noise", key_seed=101),
    "C2": dict(width=576, height=576, frames=24, workers=16, kind="correlated", key_seed=102),
    "C3": dict(width=768, height=768, frames=240, workers=32, kind="correlated", key_seed=103),
    "C4": dict(width=1920, height=1080, frames=1000, workers=64, kind="correlated", key_seed=104),
    "C5": dict(width=3840, height=2160, frames=500, workers=128, kind="correlated", key_seed=105),
}
ROUNDS = 5


def config_frame(name: str, t: int) -> np.ndarray:
    """Padded square frame t of config `name` (frame.cpp:28-39 padding).
    C5 carries the edge cases: frame 0 all-zero, frame 1 all-255."""
    c = CONFIGS[name]
    w, h, n = c["width"], c["height"], c["workers"]
    side = (max(w, h) + n - 1) // n * n
    out = np.zeros((side, side, 3), dtype=np.uint8)
    if c["kind"] == "noise":
        img = noise_frame(w, 0xF0 + c["key_seed"] + t)
    elif name == "C5" and t in (0, 1):
        img = np.full((h, w, 3), 0 if t == 0 else 255, dtype=np.uint8)
    else:
        img = correlated_frame(w, h, t, 7000 + c["key_seed"])
    out[:h, :w] = img
    return out


def config_frame_job(arg) -> np.ndarray:
    """config_frame((name, t)): a picklable entry point for process pools."""
    name, t = arg
    return config_frame(name, t)


def config_side(name: str) -> int:
    c = CONFIGS[name]
    return (max(c["width"], c["height"]) + c["workers"] - 1) // c["workers"] * c["workers"]


def config_key(name: str) -> str:
    return det_key(CONFIGS[name]["key_seed"])


def frame_list(name: str, count: int) -> List[np.ndarray]:
    return [config_frame(name, t) for t in range(count)]
