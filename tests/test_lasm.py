"""Row f2: LASM keys (192-bit, reference chaos.cpp:34-44, 93-107, 119-141;
keying.cpp:67-73, 164-207).

Checkers, in the order they are trusted:
1. glibc's own libm sin on this host vs the product's restatement of it
   (glibc_sin.cuh, host build; CPU) -- the one third-party algorithm on the
   path (glibc 2.39 libm, FMA ifunc variant), bit for bit;
2. the oracle's LASM generator vs the reference unit-test goldens
   (test_chaos.cpp:36-45, 111-123; test_keying.cpp:181-195) and vs the
   reference itself (tests/golden/lasm.json from oracle/_ref, and live);
3. the CUDA path through the C ABI vs 1 and 2 (GPU).
Bar: bit-exact.
"""
import hashlib
import json
import math
import os
import subprocess

import numpy as np
import pytest

from _oracle import Oracle, Reference, lasm_iterate, lasm_stream
from workloads import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
CSRC = os.path.join(ROOT, "paper_2302_07411_b200", "csrc")
LASM = "01333333333333d33f666666666666e63f6f8104c58f31ed3f"  # test_capi.cpp:21


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def host_has_fma() -> bool:
    """glibc picks its FMA sin variant on FMA + AVX2 hosts (every B200 host);
    glibc_sin.cuh restates that variant."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma " in flags and " avx2 " in flags


need_fma = pytest.mark.skipif(not host_has_fma(), reason="host libm uses a non-FMA sin variant")
need_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


# ---- 1. the glibc sin restatement (CPU) ------------------------------------

@need_fma
def test_host_restatement_matches_libm_sin(tmp_path):
    inc = os.path.join(ROOT, "build", "csrc")
    if not os.path.exists(os.path.join(inc, "glibc_sincostab.inc")):
        inc = str(tmp_path)
        subprocess.run(["python3", os.path.join(CSRC, "gen_sincostab.py"),
                        os.path.join(inc, "glibc_sincostab.inc")], check=True)
    exe = str(tmp_path / "glibc_sin_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", CSRC, "-I", inc,
                    os.path.join(ROOT, "tests", "glibc_sin_check.cpp"), "-o", exe, "-lm"],
                   check=True)
    out = subprocess.run([exe, "150000"], check=True, capture_output=True, text=True).stdout
    cases, bad = map(int, out.split()[-2:])
    assert cases > 4_000_000
    assert bad == 0, out


# ---- 2. the oracle (CPU) ---------------------------------------------------

def test_oracle_lasm_golden_stream():
    g = load("reference_unit.json")["lasm_golden_48"]
    assert lasm_stream(g["lanes"], 48).tobytes().hex() == g["bytes"]


def test_oracle_lasm_step_examples():
    for c in load("reference_unit.json")["lasm_step_examples"]["cases"]:
        x, y = lasm_iterate(c["x"], c["y"], c["mu"])
        for got, want in zip((x, y), c["approx"]):
            if want == 0.0:
                assert got == 0.0  # x = 1: sin(0) exactly
            else:
                assert abs(got - want) <= 1e-12 * abs(want)


def test_oracle_lasm_worker_params_and_seeds():
    g = load("reference_unit.json")["lasm_worker_params_n1"]
    o = Oracle(g["key"], 1)
    assert o.params().tolist() == g["lanes"]
    assert [Oracle.lib.orc_cipher_next_seed(o.h) for _ in range(2)] == g["seeds"]


@pytest.mark.parametrize("case", range(6))
def test_oracle_lasm_small_shapes_vs_reference(case):
    c = load("lasm.json")["cases"][case]
    side = c["side"]
    o = Oracle(c["key"], c["workers"], c["rounds"])
    d = Oracle(c["key"], c["workers"], c["rounds"])
    for p_hex, c_hex in zip(c["plain"], c["cipher"]):
        x = np.frombuffer(bytes.fromhex(p_hex), dtype=np.uint8).reshape(side, side, 3).copy()
        assert o.encrypt(x) == 0
        assert x.tobytes().hex() == c_hex
        assert d.decrypt(x) == 0
        assert x.tobytes().hex() == p_hex


@pytest.mark.parametrize("name", ["C1", "C2", "C3", pytest.param("C4", marks=pytest.mark.slow),
                                  pytest.param("C5", marks=pytest.mark.slow)])
def test_oracle_lasm_clips_vs_reference(name):
    g = load("lasm.json")["clips"][name]
    o = Oracle(g["key"], g["workers"], g["rounds"])
    for t, (ps, cs) in enumerate(zip(g["plain_sha256"], g["cipher_sha256"])):
        f = synth.config_frame(name, t)
        assert sha(f) == ps
        assert o.encrypt(f) == 0
        assert sha(f) == cs


@need_ref
@pytest.mark.parametrize("side,n,r", [(8, 2, 3), (16, 4, 1), (60, 3, 2), (7, 7, 5)])
def test_oracle_lasm_equals_reference_live(side, n, r):
    key = synth.det_key_lasm(side * 17 + n)
    rng = np.random.Generator(np.random.PCG64(side + 1))
    o, ref = Oracle(key, n, r), Reference(key, n, r, 0)
    for _ in range(2):
        p = rng.integers(0, 256, (side, side, 3), dtype=np.uint8)
        a, b = p.copy(), p.copy()
        assert o.encrypt(a) == 0 and ref.encrypt(b) == 0
        assert np.array_equal(a, b)


def test_det_key_lasm_is_in_domain():
    import paper_2302_07411_b200 as cve
    for s in range(20):
        assert cve.key_validate(synth.det_key_lasm(s)) == cve.CVE_MAP_LASM


# ---- 3. the CUDA path (GPU) ------------------------------------------------

@pytest.mark.gpu
@need_fma
def test_gpu_sin_matches_libm():
    import paper_2302_07411_b200 as cve
    rng = np.random.Generator(np.random.PCG64(7))
    parts = [rng.uniform(lo, hi, 150_000) for lo, hi in
             ((0, 2 ** -26), (2 ** -26, 0.126), (0.126, 0.85546875), (0.85546875, 2.4262639),
              (2.4262600, 2.4262700), (2.4262638, math.pi), (math.pi, 26.0), (-26.0, 0.0))]
    x = np.concatenate(parts)
    got = cve.glibc_sin(x)
    want = np.array([math.sin(v) for v in x])  # CPython's math.sin is libm sin
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_gpu_lasm_golden_stream():
    import paper_2302_07411_b200 as cve
    g = load("reference_unit.json")["lasm_golden_48"]
    assert cve.keystream_generate_lasm(g["lanes"], 48).tobytes().hex() == g["bytes"]


@pytest.mark.gpu
def test_gpu_lasm_random_lanes_vs_oracle():
    # test_chaos.cpp:139-151 shape (naive reference), longer streams
    import paper_2302_07411_b200 as cve
    rng = np.random.Generator(np.random.PCG64(22))
    for k in range(4):
        lanes = [rng.uniform(0, 1), rng.uniform(0, 1), rng.uniform(0.44, 0.93),
                 rng.uniform(0, 1), rng.uniform(0, 1), 1.0 if k == 0 else rng.uniform(0.44, 0.93)]
        n = 120_007
        assert np.array_equal(cve.keystream_generate_lasm(lanes, n), lasm_stream(lanes, n)), lanes
    # degenerate: x0 = 0 or 1 pins x at 0 (sin(0)); identical lanes cancel
    for lanes in ([0.0, 0.5, 0.9, 1.0, 0.3, 0.7], [0.3, 0.7, 0.9123, 0.3, 0.7, 0.9123]):
        assert np.array_equal(cve.keystream_generate_lasm(lanes, 600), lasm_stream(lanes, 600))
    with pytest.raises(cve.CveError) as e:
        cve.keystream_generate_lasm([0.5, 0.5, 0.39, 0.5, 0.5, 0.9], 12)
    assert e.value.status == cve.CVE_ERROR_BAD_KEY


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C4"])
def test_gpu_lasm_worker_streams_vs_golden(name):
    import paper_2302_07411_b200 as cve
    g = load("lasm.json")
    key = g["clips"][name]["key"]
    n = synth.CONFIGS[name]["workers"]
    c = cve.Cipher(key, n, 5)
    for i, d in enumerate(g["worker_stream_sha256_256KiB"][name]):
        assert hashlib.sha256(c.peek_keystream(i, 1 << 18).tobytes()).hexdigest() == d, i


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(6))
def test_gpu_lasm_small_shapes_vs_reference(case):
    import paper_2302_07411_b200 as cve
    c = load("lasm.json")["cases"][case]
    side, n, r = c["side"], c["workers"], c["rounds"]
    enc, dec = cve.Cipher(c["key"], n, r), cve.Cipher(c["key"], n, r)
    for p_hex, c_hex in zip(c["plain"], c["cipher"]):
        x = np.frombuffer(bytes.fromhex(p_hex), dtype=np.uint8).reshape(side, side, 3).copy()
        enc.encrypt_frame(x)
        assert x.tobytes().hex() == c_hex
        dec.decrypt_frame(x)
        assert x.tobytes().hex() == p_hex


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_gpu_lasm_clips_vs_reference(name):
    import paper_2302_07411_b200 as cve
    g = load("lasm.json")["clips"][name]
    frames = np.stack([synth.config_frame(name, t) for t in range(len(g["cipher_sha256"]))])
    one = cve.Cipher(g["key"], g["workers"], g["rounds"])
    per = frames.copy()
    for t in range(len(per)):
        one.encrypt_frame(per[t])
        assert sha(per[t]) == g["cipher_sha256"][t], t
    if name == "C5":  # edge frames: all-zero stays all-zero under any key
        assert not per[0].any() and per[1].any()
    batch = frames.copy()
    cve.Cipher(g["key"], g["workers"], g["rounds"]).encrypt_frames(batch)
    assert np.array_equal(batch, per)
    cve.Cipher(g["key"], g["workers"], g["rounds"]).decrypt_frames(batch)
    assert np.array_equal(batch, frames)


@pytest.mark.gpu
@need_ref
def test_gpu_lasm_random_shapes_vs_reference():
    import paper_2302_07411_b200 as cve
    rng = np.random.Generator(np.random.PCG64(99))
    for side, n, r in [(8, 2, 3), (33, 11, 2), (64, 64, 1), (96, 8, 5), (130, 13, 4)]:
        key = synth.det_key_lasm(side + 1000 * n)
        c, ref = cve.Cipher(key, n, r), Reference(key, n, r, 1)
        for _ in range(3):
            p = rng.integers(0, 256, (side, side, 3), dtype=np.uint8)
            a, b = p.copy(), p.copy()
            c.encrypt_frame(a)
            assert ref.encrypt(b) == 0
            assert np.array_equal(a, b), (side, n, r)


@pytest.mark.gpu
def test_gpu_lasm_and_plcm_handles_concurrently():
    # cve.h:5-6 with both maps: LASM and PLCM handles driven at once from
    # threads (the two generator kinds share the device); every frame must
    # match the oracle.
    import threading
    import paper_2302_07411_b200 as cve
    shapes = [(96, 8, True), (120, 4, False), (64, 16, True), (90, 3, False), (48, 4, True)]
    results = {}

    def run(k, side, n, lasm):
        key = synth.det_key_lasm(700 + k) if lasm else synth.det_key(700 + k)
        frames = np.random.Generator(np.random.PCG64(k)).integers(
            0, 256, (4, side, side, 3), dtype=np.uint8)
        ct = frames.copy()
        c = cve.Cipher(key, n, 5)
        for t in range(len(ct)):
            c.encrypt_frame(ct[t])
        results[k] = (key, n, frames, ct)

    ths = [threading.Thread(target=run, args=(k, s, n, l)) for k, (s, n, l) in enumerate(shapes)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert len(results) == len(shapes)
    for k, (key, n, frames, ct) in results.items():
        o = Oracle(key, n, 5)
        for f, g in zip(frames, ct):
            a = f.copy()
            assert o.encrypt(a) == 0
            assert np.array_equal(a, g), k


@pytest.mark.gpu
def test_gpu_lasm_device_resident_and_sides_change():
    # device-resident API == host API; a handle whose frame side changes
    # keeps one continuous keystream (engine.cpp:198-205), LASM key
    torch = pytest.importorskip("torch")
    import paper_2302_07411_b200 as cve
    key = synth.det_key_lasm(41)
    o = Oracle(key, 4, 5)
    c = cve.Cipher(key, 4, 5)
    rng = np.random.Generator(np.random.PCG64(41))
    for side in (64, 96, 64, 128):
        f = rng.integers(0, 256, (2, side, side, 3), dtype=np.uint8)
        want = f.copy()
        for t in range(2):
            assert o.encrypt(want[t]) == 0
        dev = torch.from_numpy(f.copy()).cuda()
        s = torch.cuda.current_stream()
        c.encrypt_frames_device(dev.data_ptr(), side, 2, s.cuda_stream)
        s.synchronize()
        assert np.array_equal(dev.cpu().numpy(), want), side


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_gpu_lasm_every_frame_of_config_clips_vs_reference(name):
    # The per-frame parity gate of SURVEY 8(d), with a LASM key: the digest of
    # EVERY frame of the C3 (240), C4 (1000) and C5 (500) clips equals the
    # reference's own (tests/golden/lasm_clips.json), and a fresh in-order
    # handle decrypts every frame back (round trip); plaintext digests from
    # clips.json guard the synthetic frames.
    from _clips import run_clip
    for f in ("lasm_clips.json", "clips.json"):
        if not os.path.exists(os.path.join(GOLD, f)):
            pytest.skip(f"tests/golden/{f} not generated")
    g, plain = load("lasm_clips.json")[name], load("clips.json")[name]["plain_sha256"]
    assert run_clip(name, g, plain) == g["frames"]
