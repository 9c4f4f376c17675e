"""Round-kernel variants against the oracle (r02).

The production forward round is K2r (rows.cu) wherever its plan applies
(side % 16 == 0, a chunk height cr >= 3 dividing the band); K2s (cipher.cu)
remains the fallback, and K3r is an opt-in inverse round.  The environment
switches are read at every frame, so each variant is driven here on the same
geometries and checked byte for byte against the oracle (reference
engine.cpp:32-83, 207-284), plus round trips.
"""
import os

import numpy as np
import pytest

import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Oracle

pytestmark = pytest.mark.gpu

# (side, n, r): K2r chunk heights 3..15, clusters of 1..16 chunks, segment
# counts that are not powers of two, rows that K2r cannot split (K2s)
GEOMS = [(48, 16, 5), (64, 1, 3), (96, 2, 5), (144, 3, 2), (160, 10, 5), (240, 8, 5),
         (256, 16, 1), (320, 20, 3), (480, 8, 5), (512, 32, 2), (576, 16, 5), (32, 16, 5),
         # one row per band (K3r once divided by rows with a magic that overflowed)
         (48, 48, 5), (16, 16, 3)]


def rand_frames(side, count, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(count, side, side, 3), dtype=np.uint8)


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def encrypt_vs_oracle(side, n, r, seed):
    key = synth.det_key(seed)
    frames = rand_frames(side, 3, seed)
    want = frames.copy()
    o = Oracle(key, n, r)
    for t in range(len(frames)):
        assert o.encrypt(want[t]) == 0
    got = frames.copy()
    h = cve.Cipher(key, n, r)
    for t in range(len(frames)):
        h.encrypt_frame(got[t])
    assert np.array_equal(got, want), (side, n, r)
    return key, frames, want


@pytest.mark.parametrize("side,n,r", GEOMS)
def test_forward_rounds_k2r_and_k2s(side, n, r):
    # default (K2r where it applies), the K2s fallback forced, and K2r with
    # every round of a frame in one cooperative launch (opt-in)
    encrypt_vs_oracle(side, n, r, side * 17 + n + r)
    with env(CVE_B200_NO_ROWS="1"):
        encrypt_vs_oracle(side, n, r, side * 19 + n + r)
    with env(CVE_B200_ROWS_PERSIST="1"):
        encrypt_vs_oracle(side, n, r, side * 29 + n + r)


@pytest.mark.parametrize("side,n,r", GEOMS)
def test_inverse_rounds_k3r(side, n, r):
    # the opt-in K3r: oracle ciphertext decrypted back, consecutive frames of
    # one handle (the stream window advances), and a LASM key
    with env(CVE_B200_ROWS_DECRYPT="1"):
        key, frames, ct = encrypt_vs_oracle(side, n, r, side * 23 + n + r)
        d = cve.Cipher(key, n, r)
        for t in range(len(frames)):
            d.decrypt_frame(ct[t])
        assert np.array_equal(ct, frames)
        key = synth.det_key_lasm(side + n + r)
        frames = rand_frames(side, 2, side + 5)
        ct = frames.copy()
        cve.Cipher(key, n, r).encrypt_frames(ct)
        cve.Cipher(key, n, r).decrypt_frames(ct)
        assert np.array_equal(ct, frames)


def test_k2r_ring_wrap_many_frames():
    # 12 frames on one handle at C3's geometry: the keystream ring (4 frames)
    # wraps inside frames and inside rows; per frame against the oracle
    side, n, r = 768, 32, 5
    key = synth.det_key(9901)
    frames = rand_frames(side, 12, 9901)
    want = frames.copy()
    o = Oracle(key, n, r)
    for t in range(len(frames)):
        assert o.encrypt(want[t]) == 0
    got = frames.copy()
    cve.Cipher(key, n, r).encrypt_frames(got)
    assert np.array_equal(got, want)
