"""Pins the CPU oracle (oracle/cve_oracle.c) before it is trusted as the
checker: against the reference unit-test goldens, against digests of the
reference's own ciphertext (tests/golden/frames.json, small.json), and live
against the compiled reference when oracle/_ref is present."""
import hashlib
import json
import os

import numpy as np
import pytest

from _oracle import Oracle, Reference, plcm_stream
from workloads import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_plcm_golden_stream():
    g = load("reference_unit.json")["plcm_golden_48"]
    assert plcm_stream(*g["lanes"], 48).tobytes().hex() == g["bytes"]


def test_worker_params_and_seeds():
    g = load("reference_unit.json")["worker_params_n2"]
    o = Oracle(g["key"], 2)
    assert o.params().tolist() == g["lanes"]
    assert [Oracle.lib.orc_cipher_next_seed(o.h) for _ in range(3)] == g["seeds"]
    assert o.seeds_drawn == 3


def test_shift_table_and_diffuse_example():
    u = load("reference_unit.json")
    L = Oracle.load()
    assert [L.orc_confusion_shift(a, 4, 7) for a in range(4)] == u["shift_side4_seed7"]["shift"]
    d = u["diffuse_example"]
    assert L.orc_diffuse_byte(d["v"], d["b"], d["prev"]) == d["c"]
    assert L.orc_inverse_diffuse_byte(d["c"], d["b"], d["prev"]) == d["v"]
    # full byte cube (test_engine.cpp:122-134): inverse undoes forward
    v = np.arange(256)
    for b in range(0, 256, 17):
        for prev in range(0, 256, 13):
            c = [L.orc_diffuse_byte(int(x), b, prev) for x in v]
            assert [L.orc_inverse_diffuse_byte(int(x), b, prev) for x in c] == list(v)


def test_padded_side_cases():
    L = Oracle.load()
    assert L.orc_padded_side(1920, 1080, 64) == 1920
    assert L.orc_padded_side(3840, 2160, 128) == 3840
    assert L.orc_padded_side(10, 7, 4) == 12


@pytest.mark.parametrize("case", range(6))
def test_small_shapes_match_reference_digests(case):
    c = load("small.json")["cases"][case]
    o = Oracle(c["key"], c["workers"], c["rounds"])
    side = c["side"]
    for p_hex, c_hex in zip(c["plain"], c["cipher"]):
        x = np.frombuffer(bytes.fromhex(p_hex), dtype=np.uint8).reshape(side, side, 3).copy()
        assert o.encrypt(x) == 0
        assert x.tobytes().hex() == c_hex
    d = Oracle(c["key"], c["workers"], c["rounds"])
    for p_hex, c_hex in zip(c["plain"], c["cipher"]):
        x = np.frombuffer(bytes.fromhex(c_hex), dtype=np.uint8).reshape(side, side, 3).copy()
        assert d.decrypt(x) == 0
        assert x.tobytes().hex() == p_hex


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_config_clips_match_reference_digests(name):
    g = load("frames.json")[name]
    o = Oracle(g["key"], g["workers"], g["rounds"])
    for t, (ps, cs) in enumerate(zip(g["plain_sha256"], g["cipher_sha256"])):
        f = synth.config_frame(name, t)
        assert sha(f) == ps, "synthetic generator drifted"
        assert o.encrypt(f) == 0
        assert sha(f) == cs


def test_key_flip_sensitivity_c3():
    g = load("frames.json")["C3"]
    f = synth.config_frame("C3", 0)
    o = Oracle(g["flip_key"], g["workers"])
    assert o.encrypt(f) == 0
    assert sha(f) == g["flip_cipher_sha256"]
    assert 0.99 < g["flip_differ_fraction"] < 1.0


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C4", "C5"])
def test_large_config_first_frames(name):
    g = load("frames.json")[name]
    o = Oracle(g["key"], g["workers"], g["rounds"])
    for t, cs in enumerate(g["cipher_sha256"]):
        f = synth.config_frame(name, t)
        assert o.encrypt(f) == 0
        assert sha(f) == cs
        if name == "C5" and t == 0:
            assert not f.any(), "all-zero frame must encrypt to all zeros"


def test_worker_streams_c1():
    ks = load("small.json")["worker_stream_sha256_1MiB"]["C1"]
    o = Oracle(synth.config_key("C1"), 8)
    for i in range(8):
        assert hashlib.sha256(o.worker_stream(i, 1 << 20).tobytes()).hexdigest() == ks[i]


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("side,n,r", [(8, 2, 3), (16, 4, 1), (64, 8, 5), (60, 3, 2), (7, 7, 5)])
def test_oracle_equals_reference_live(side, n, r):
    key = synth.det_key(side * 31 + n)
    rng = np.random.Generator(np.random.PCG64(side))
    o, ref = Oracle(key, n, r), Reference(key, n, r, 0)
    for _ in range(3):
        p = rng.integers(0, 256, (side, side, 3), dtype=np.uint8)
        a, b = p.copy(), p.copy()
        assert o.encrypt(a) == 0 and ref.encrypt(b) == 0
        assert np.array_equal(a, b)
    # error order: MISMATCH after the seed draw, both sides
    bad = np.zeros((side + 1, side + 1, 3), dtype=np.uint8)
    if (side + 1) % n:
        assert o.encrypt(bad) == 5 and ref.encrypt(bad.copy()) == 5
