"""Parity of the CUDA path (through the C ABI) with the reference.

Checkers: the oracle (oracle/cve_oracle.c, itself pinned in test_oracle.py),
the reference's compiled library when present, and the committed digests of
the reference's ciphertext (tests/golden).  Bar: bit-exact bytes.
Full-size configs are checked against golden digests for their first frames
and through size-independent properties (round trip, all-zero fixed point,
key sensitivity, batch == per-frame == device-resident).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Oracle, plcm_stream

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PLCM = "005f633937dd9abf3f93ba8c762f1bd43fb8560e3cdd9aef3f7c74d008a265d13f"


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rand_frames(side, count, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 256, (count, side, side, 3), dtype=np.uint8)


# ---- K1: keystream generator ----------------------------------------------

def test_keystream_golden_48():
    g = load("reference_unit.json")["plcm_golden_48"]
    assert cve.keystream_generate(g["lanes"], 48).tobytes().hex() == g["bytes"]


def test_keystream_random_lanes_vs_oracle():
    # test_chaos.cpp:125-137 shape, longer streams (exercise many blocks)
    rng = np.random.Generator(np.random.PCG64(21))
    for _ in range(6):
        xa, xb = rng.uniform(0, 1, 2)
        pa, pb = rng.uniform(0.01, 0.49, 2)
        n = 300_007
        assert np.array_equal(cve.keystream_generate([xa, pa, xb, pb], n),
                              plcm_stream(xa, pa, xb, pb, n))


def test_keystream_guard_cases():
    # test_chaos.cpp:185-213: identical lanes cancel; endpoint seeds collapse
    # onto one guarded orbit; guarded degenerate seeds vary.  p = 0.25 with
    # x = 0.0625 hits the guard set inside the orbit (x/p == p).
    assert not cve.keystream_generate([0.3, 0.2, 0.3, 0.2], 600).any()
    a = cve.keystream_generate([0.0, 0.3, 0.25, 0.2], 256)
    b = cve.keystream_generate([1.0, 0.3, 0.25, 0.2], 256)
    c = cve.keystream_generate([0.123, 0.3, 0.25, 0.2], 256)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    for lanes in ([0.0, 0.3, 0.41, 0.17], [0.5, 0.3, 0.41, 0.17], [1.0, 0.3, 0.41, 0.17],
                  [0.3, 0.3, 0.41, 0.17], [0.0625, 0.25, 0.125, 0.25], [0.5, 0.25, 0.75, 0.125],
                  [0.2, 0.4, 0.6, 0.1]):
        got = cve.keystream_generate(lanes, 4800)
        assert np.array_equal(got, plcm_stream(*lanes, 4800)), lanes


def test_keystream_bad_lanes():
    with pytest.raises(cve.CveError) as e:
        cve.keystream_generate([0.3, 0.5, 0.2, 0.2], 16)
    assert e.value.status == cve.CVE_ERROR_BAD_KEY


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_worker_streams_vs_golden(name):
    digests = load("small.json")["worker_stream_sha256_1MiB"][name]
    c = cve.Cipher(synth.config_key(name), synth.CONFIGS[name]["workers"], 5)
    for i, d in enumerate(digests):
        assert hashlib.sha256(c.peek_keystream(i, 1 << 20).tobytes()).hexdigest() == d, i
    assert c.seeds_drawn == 0  # peeking consumes nothing


# ---- K2/K3/K4: whole frames ------------------------------------------------

@pytest.mark.parametrize("case", range(6))
def test_small_cases_vs_reference(case):
    c = load("small.json")["cases"][case]
    side, n, r = c["side"], c["workers"], c["rounds"]
    enc, dec = cve.Cipher(c["key"], n, r), cve.Cipher(c["key"], n, r, parallel=False)
    for p_hex, c_hex in zip(c["plain"], c["cipher"]):
        x = np.frombuffer(bytes.fromhex(p_hex), np.uint8).reshape(side, side, 3).copy()
        enc.encrypt_frame(x)
        assert x.tobytes().hex() == c_hex
        dec.decrypt_frame(x)
        assert x.tobytes().hex() == p_hex
    assert enc.seeds_drawn == len(c["plain"])


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_config_clip_vs_reference_digests(name):
    g = load("frames.json")[name]
    frames = np.stack(synth.frame_list(name, len(g["cipher_sha256"])))
    c = cve.Cipher(g["key"], g["workers"], g["rounds"])
    per = frames.copy()
    for t in range(len(per)):
        c.encrypt_frame(per[t])
        assert sha(per[t]) == g["cipher_sha256"][t], t
    batch = frames.copy()
    cve.Cipher(g["key"], g["workers"], g["rounds"]).encrypt_frames(batch)
    assert np.array_equal(batch, per)
    d = cve.Cipher(g["key"], g["workers"], g["rounds"])
    d.decrypt_frames(batch)
    assert np.array_equal(batch, frames)


def test_device_resident_api_matches_host_api():
    torch = pytest.importorskip("torch")
    g = load("frames.json")["C2"]
    frames = np.stack(synth.frame_list("C2", 8))
    dev = torch.from_numpy(frames.copy()).cuda()
    c = cve.Cipher(g["key"], g["workers"], 5)
    s = torch.cuda.current_stream()
    c.encrypt_frames_device(dev.data_ptr(), frames.shape[1], 4, s.cuda_stream)
    c.encrypt_frames_device(dev.data_ptr() + 4 * frames[0].nbytes, frames.shape[1], 4,
                            s.cuda_stream)
    out = dev.cpu().numpy()  # ordered after the cipher on the same stream
    for t in range(8):
        assert sha(out[t]) == g["cipher_sha256"][t]
    d = cve.Cipher(g["key"], g["workers"], 5)
    d.decrypt_frames_device(dev.data_ptr(), frames.shape[1], 8, s.cuda_stream)
    assert np.array_equal(dev.cpu().numpy(), frames)


@pytest.mark.parametrize("side,n,r", [
    (8, 2, 3), (16, 4, 1), (24, 4, 5), (30, 3, 5), (7, 7, 5), (97, 1, 2),
    (100, 4, 5), (192, 12, 5), (256, 128, 5), (64, 64, 5), (1000, 1, 2),
    (600, 1, 5), (480, 8, 1), (484, 4, 4),
    # side % 16 == 0: slot-staged rounds (K2s/K3s), odd cluster sizes and
    # partial decrypt tiles
    (32, 2, 3), (48, 3, 5), (112, 7, 2), (144, 9, 5), (176, 11, 3), (320, 20, 2),
    (208, 4, 5), (400, 25, 1)])
def test_random_shapes_vs_oracle(side, n, r):
    key = synth.det_key(side * 131 + n * 7 + r)
    frames = rand_frames(side, 3, side + n)
    o = Oracle(key, n, r)
    c = cve.Cipher(key, n, r)
    for f in frames:
        a, b = f.copy(), f.copy()
        assert o.encrypt(a) == 0
        c.encrypt_frame(b)
        assert np.array_equal(a, b)
    # cross decryption: oracle ciphertext -> GPU decrypt
    o2, d = Oracle(key, n, r), cve.Cipher(key, n, r)
    for f in frames:
        a = f.copy()
        assert o2.encrypt(a) == 0
        d.decrypt_frame(a)
        assert np.array_equal(a, f)


def test_mixed_sides_on_one_handle():
    # stream continuity across frames of different sizes (ring growth)
    key = synth.det_key(4242)
    o, c = Oracle(key, 4), cve.Cipher(key, 4)
    rng = np.random.Generator(np.random.PCG64(5))
    for side in (16, 480, 32, 960, 8, 200, 1024):
        f = rng.integers(0, 256, (side, side, 3), dtype=np.uint8)
        a, b = f.copy(), f.copy()
        assert o.encrypt(a) == 0
        c.encrypt_frame(b)
        assert np.array_equal(a, b), side
    assert c.seeds_drawn == o.seeds_drawn == 7


def test_error_semantics_match_reference():
    # test_capi.cpp:116-162
    c = cve.Cipher(PLCM, 2, 3)
    assert c.seeds_drawn == 0
    odd = rand_frames(7, 1, 2)[0]
    with pytest.raises(cve.CveError) as e:
        c.encrypt_frame(odd)
    assert e.value.status == cve.CVE_ERROR_MISMATCH
    assert c.seeds_drawn == 1  # seed drawn before the side check
    # the next frame binds to frame index 1 in both implementations
    o = Oracle(PLCM, 2, 3)
    assert o.encrypt(odd.copy()) == 5
    f = rand_frames(8, 1, 3)[0]
    a, b = f.copy(), f.copy()
    o.encrypt(a)
    c.encrypt_frame(b)
    assert np.array_equal(a, b)
    batch = rand_frames(9, 2, 4)
    with pytest.raises(cve.CveError) as e:
        c.encrypt_frames(batch)
    assert e.value.status == cve.CVE_ERROR_MISMATCH
    assert c.seeds_drawn == 3


def test_key_flip_sensitivity_c3():
    g = load("frames.json")["C3"]
    f = synth.config_frame("C3", 0)
    a, b = f.copy(), f.copy()
    cve.Cipher(g["key"], 32).encrypt_frame(a)
    cve.Cipher(g["flip_key"], 32).encrypt_frame(b)
    assert sha(b) == g["flip_cipher_sha256"]
    frac = float((a != b).mean())
    assert abs(frac - g["flip_differ_fraction"]) < 1e-12 and frac > 0.99


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_configs(name):
    g = load("frames.json")[name]
    k = len(g["cipher_sha256"])
    frames = np.stack(synth.frame_list(name, k + 1))
    c = cve.Cipher(g["key"], g["workers"], 5)
    ct = frames.copy()
    c.encrypt_frames(ct)
    for t in range(k):
        assert sha(ct[t]) == g["cipher_sha256"][t], t
    if name == "C5":
        assert not ct[0].any(), "all-zero frame must encrypt to all zeros"
        assert abs(float((ct[1] == 255).mean()) - g["full_frame_fraction_255"]) < 1e-12
    d = cve.Cipher(g["key"], g["workers"], 5)
    d.decrypt_frames(ct)
    assert np.array_equal(ct, frames)


def test_stats_and_launch_accounting():
    c = cve.Cipher(synth.config_key("C1"), 8, 5)
    f = synth.config_frame("C1", 0)
    c.encrypt_frame(f)
    s = c.stats()
    assert s["frames"] == 1 and s["prbg_launches"] >= 1
    assert s["keystream_iters"] * 6 >= 5 * 480 * 480 * 3 // 8
    assert s["kernel_launches"] >= 1 + 5 + s["prbg_launches"]
    assert s["prbg_ms"] > 0 and s["cipher_ms"] > 0


@pytest.mark.parametrize("side,n,r", [(1, 1, 5), (2, 1, 3), (2, 2, 5), (3, 3, 1), (3, 1, 255),
                                      (5, 5, 7), (1536, 1, 1)])
def test_degenerate_and_extreme_geometries_vs_oracle(side, n, r):
    # 1-pixel frames (region = 3 bytes), one row per band, 255 rounds, and a
    # single 1536-row band (generic multi-kernel path)
    key = synth.det_key(side * 7 + n + r)
    frames = rand_frames(side, 2, side * 13 + r)
    o, c = Oracle(key, n, r), cve.Cipher(key, n, r)
    for f in frames:
        a, b = f.copy(), f.copy()
        assert o.encrypt(a) == 0
        c.encrypt_frame(b)
        assert np.array_equal(a, b)
    d = cve.Cipher(key, n, r)
    ct = frames.copy()
    cve.Cipher(key, n, r).encrypt_frames(ct)
    d.decrypt_frames(ct)
    assert np.array_equal(ct, frames)


def test_concurrent_handles_from_threads():
    # cve.h:5-6: distinct handles are independent; one thread per handle
    import threading
    shapes = [(96, 8), (120, 4), (64, 16), (90, 3)]
    results = {}

    def run(k, side, n):
        key = synth.det_key(900 + k)
        frames = rand_frames(side, 6, k)
        ct = frames.copy()
        c = cve.Cipher(key, n, 5)
        for t in range(len(ct)):
            c.encrypt_frame(ct[t])
        results[k] = (key, n, frames, ct)

    ths = [threading.Thread(target=run, args=(k, s, n)) for k, (s, n) in enumerate(shapes)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for k, (key, n, frames, ct) in results.items():
        o = Oracle(key, n, 5)
        for f, g in zip(frames, ct):
            a = f.copy()
            assert o.encrypt(a) == 0
            assert np.array_equal(a, g), k


def test_concurrent_handles_stress():
    # Many handles created and driven at once from threads (setup uploads,
    # first frames and the keystream generator all contending): every frame
    # must still match the oracle.  Guards the stream ordering of the
    # per-handle uploads (lane constants, x0, sine table, flags).
    import threading
    shapes = [(96, 8), (120, 4), (64, 16), (90, 3), (128, 8), (48, 4), (160, 16), (72, 6)]
    for rep in range(3):
        results = {}

        def run(k, side, n):
            key = synth.det_key(950 + 10 * rep + k)
            frames = rand_frames(side, 4, 100 * rep + k)
            ct = frames.copy()
            c = cve.Cipher(key, n, 3)
            for t in range(len(ct)):
                c.encrypt_frame(ct[t])
            results[k] = (key, n, frames, ct)

        ths = [threading.Thread(target=run, args=(k, s, n)) for k, (s, n) in enumerate(shapes)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert len(results) == len(shapes)
        for k, (key, n, frames, ct) in results.items():
            o = Oracle(key, n, 3)
            for f, g in zip(frames, ct):
                a = f.copy()
                assert o.encrypt(a) == 0
                assert np.array_equal(a, g), (rep, k)


def test_one_stream_handles_match_oracle():
    # cve_set_streams_per_handle(1): generator, verify and rounds on one
    # stream per handle -- same bytes, several handles interleaved
    cve.set_streams_per_handle(1)
    try:
        shapes = [(96, 8, 5), (64, 16, 3), (90, 3, 2)]
        hs = [cve.Cipher(synth.det_key(4000 + k), n, r) for k, (s, n, r) in enumerate(shapes)]
    finally:
        cve.set_streams_per_handle(2)
    for t in range(3):
        for k, ((side, n, r), h) in enumerate(zip(shapes, hs)):
            f = rand_frames(side, 1, 100 * k + t)[0]
            a, b = f.copy(), f.copy()
            h.encrypt_frame(b)
            if t == 0:
                hs[k].oracle = Oracle(synth.det_key(4000 + k), n, r)
            assert hs[k].oracle.encrypt(a) == 0
            assert np.array_equal(a, b), (k, t)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_every_frame_of_config_clips_vs_reference(name):
    # SURVEY 8(d) parity gate: per-frame digest equality with the reference
    # for EVERY frame of the clip (C3 240, C4 1000, C5 500 frames; digests of
    # the reference's own ciphertext, tests/golden/clips.json), and the whole
    # clip decrypted back by a fresh in-order handle (BASELINE C5 "encrypt +
    # decrypt round-trip"; reference test_capi.cpp:116-134).  Plaintext
    # digests are checked too, so a drift in the synthetic frames would show
    # as such rather than as a cipher mismatch.
    from _clips import run_clip
    path = os.path.join(GOLD, "clips.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/clips.json not generated")
    g = load("clips.json")[name]
    assert run_clip(name, g, g["plain_sha256"]) == g["frames"]


@pytest.mark.parametrize("name,devices,mode,frames", [
    ("C3", [0, 0], "host", 0),
    ("C3", [0, 0, 0, 0], "sharded", 0),
    ("C4", [0, 0, 0], "host", 60),
    ("C4", [0, 0, 0, 0], "sharded", 48),
    ("C5", [0, 0], "sharded", 20),
])
def test_sharded_clip_vs_reference(name, devices, mode, frames):
    # One clip sharded over cipher devices (cve_cipher_create_devices; north
    # star "independent frames of a clip are partitioned across the B200s"):
    # the generator stays on devices[0], frame k runs on shard k mod G from
    # its keystream window copied out of the ring.  Repeated device entries
    # put G shards (own streams and buffers, window copies through the same
    # code path) on the one GPU of the test box.  Every frame (C3) or a prefix
    # (C4, C5) must match the reference digests and round-trip.
    from _clips import run_clip
    path = os.path.join(GOLD, "clips.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/clips.json not generated")
    g = load("clips.json")[name]
    h = cve.Cipher(g["key"], g["workers"], g["rounds"], devices=devices)
    assert h.shards == devices
    h.close()
    assert run_clip(name, g, g["plain_sha256"], devices=devices, mode=mode,
                    frames=frames) == (frames or g["frames"])


@pytest.mark.parametrize("side,n", [(16, 1), (16, 2), (48, 3), (64, 4), (96, 8), (128, 16),
                                    (160, 5), (192, 12), (256, 8), (480, 8), (512, 8)])
def test_round_fusion_vs_oracle(side, n):
    # K6 (every forward round of a frame in one thread-block cluster) against
    # the oracle on consecutive frames of a handle, PLCM and LASM keys, r in
    # {1, 2, 5} (the final buffer's parity changes with r), then a round trip
    # through a decrypt handle.
    cve.set_round_fusion(1)
    try:
        for key, r in ((synth.det_key(70 + side + n), 5), (synth.det_key_lasm(71 + side), 2),
                       (synth.det_key(72 + n), 1)):
            frames = rand_frames(side, 3, side * 7 + n + r)
            want = frames.copy()
            o = Oracle(key, n, r)
            for t in range(3):
                assert o.encrypt(want[t]) == 0
            got = frames.copy()
            h = cve.Cipher(key, n, r)
            for t in range(3):
                h.encrypt_frame(got[t])
            assert np.array_equal(got, want), (side, n, r)
            cve.Cipher(key, n, r).decrypt_frames(got)
            assert np.array_equal(got, frames)
    finally:
        cve.set_round_fusion(0)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_round_fusion_clips_vs_reference(name):
    # The fused path on the config clips: every frame (C1/C2) or a 96-frame
    # prefix (C3) against the reference's digests, plus the round trip.
    from _clips import run_clip
    g = load("clips.json")[name] if name == "C3" else None
    if g is None:
        fr = load("frames.json")[name]
        g = {"key": fr["key"], "workers": fr["workers"], "rounds": fr["rounds"],
             "frames": len(fr["cipher_sha256"]), "cipher_sha256": fr["cipher_sha256"],
             "plain_sha256": fr["plain_sha256"]}
    cve.set_round_fusion(1)
    try:
        n = run_clip(name, g, g["plain_sha256"], frames=96 if name == "C3" else 0)
    finally:
        cve.set_round_fusion(0)
    assert n == (96 if name == "C3" else g["frames"])


@pytest.mark.parametrize("name,frames", [("C3", 0), ("C4", 30)])
def test_one_stream_handles_vs_reference(name, frames):
    # handles created with one stream per handle (the many-clips
    # configuration) use the dense-orbit generator: every frame of C3 and a
    # C4 prefix against the reference digests, plus the round trip
    from _clips import run_clip
    g = load("clips.json")[name]
    cve.set_streams_per_handle(1)
    try:
        n = run_clip(name, g, g["plain_sha256"], frames=frames)
    finally:
        cve.set_streams_per_handle(2)
    assert n == (frames or g["frames"])


def test_sharded_per_frame_calls_and_lasm_vs_oracle():
    # Per-frame drop-in calls on a sharded handle are dealt round-robin over
    # the shards; sides change between calls; a LASM key shards the same way.
    for key in (synth.det_key(61), synth.det_key_lasm(61)):
        o = Oracle(key, 4, 5)
        h = cve.Cipher(key, 4, 5, devices=[0, 0, 0])
        for t, side in enumerate([64, 64, 96, 60, 128, 100, 64, 44]):
            f = rand_frames(side, 1, 500 + t)[0]
            want = f.copy()
            assert o.encrypt(want) == 0
            h.encrypt_frame(f)
            assert np.array_equal(f, want), (key[:2], t, side)
        assert h.seeds_drawn == 8


def test_sharded_generic_geometries_vs_oracle():
    # shards running the byte-staged and the generic multi-kernel forward
    # rounds (band too large for one cluster: n = 1 at side 720) and their
    # inverses, from keystream windows of any length
    for side, n in ((720, 1), (90, 3), (52, 2)):
        key = synth.det_key(64 + side)
        frames = rand_frames(side, 3, side)
        want = frames.copy()
        o = Oracle(key, n, 5)
        for t in range(3):
            assert o.encrypt(want[t]) == 0
        got = frames.copy()
        cve.Cipher(key, n, 5, devices=[0, 0]).encrypt_frames(got)
        assert np.array_equal(got, want), (side, n)
        cve.Cipher(key, n, 5, devices=[0, 0, 0]).decrypt_frames(got)
        assert np.array_equal(got, frames), (side, n)


def test_sharded_errors():
    key = synth.det_key(62)
    with pytest.raises(cve.CveError) as e:
        cve.Cipher(key, 4, 5, devices=[0, 99])
    assert e.value.status == cve.CVE_ERROR_INVALID_ARGUMENT
    with pytest.raises(cve.CveError) as e:
        cve.Cipher(key, 4, 5, devices=[])
    assert e.value.status == cve.CVE_ERROR_INVALID_ARGUMENT
    h = cve.Cipher(key, 4, 5, devices=[0, 0])
    f = rand_frames(66, 1, 1)[0]  # 66 % 4 != 0: MISMATCH after the seed draw
    with pytest.raises(cve.CveError) as e:
        h.encrypt_frame(f)
    assert e.value.status == cve.CVE_ERROR_MISMATCH and h.seeds_drawn == 1
    torch = pytest.importorskip("torch")
    d = torch.zeros((2, 64, 64, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(cve.CveError) as e:  # device API of a single-device kind
        h.encrypt_frames_device(d.data_ptr(), 64, 2)
    assert e.value.status == cve.CVE_ERROR_INVALID_ARGUMENT


def test_device_unchanged_by_handle_lifecycle():
    # A handle restores the caller's current device on create, run and
    # destroy (also when its engine lives on another device).
    torch = pytest.importorskip("torch")
    ndev = torch.cuda.device_count()
    for dev in range(min(ndev, 2)):
        torch.cuda.set_device(0)
        cve.set_device(dev)
        try:
            h = cve.Cipher(synth.det_key(63), 4, 5)
            assert torch.cuda.current_device() == 0
            f = rand_frames(64, 1, 2)[0]
            h.encrypt_frame(f)
            assert torch.cuda.current_device() == 0
            h.close()
            assert torch.cuda.current_device() == 0
            cve.keystream_generate([0.1, 0.2, 0.3, 0.4], 48)
            assert torch.cuda.current_device() == 0
        finally:
            cve.set_device(0)


SIDES, WORKERS, ROUNDS = [8, 16, 64, 512], [1, 2, 4, 8], [1, 5]


@pytest.mark.parametrize("side", SIDES)
@pytest.mark.parametrize("n", WORKERS)
@pytest.mark.parametrize("r", ROUNDS)
def test_acceptance_grid_vs_oracle(side, n, r):
    # the reference acceptance suite's round-trip grid (acceptance.cpp:97-121:
    # sides {8,16,64,512} x workers {1,2,4,8} x rounds {1,5}, key map by
    # combination parity -- odd PLCM, even LASM -- seeded 1000 + combo), here
    # also byte-compared with the oracle over consecutive frames of a handle
    combo = SIDES.index(side) * 8 + WORKERS.index(n) * 2 + ROUNDS.index(r)
    key = synth.det_key(1000 + combo) if combo % 2 else synth.det_key_lasm(1000 + combo)
    frames = rand_frames(side, 3, side * 100 + n * 10 + r)
    want = frames.copy()
    o = Oracle(key, n, r)
    for t in range(len(want)):
        assert o.encrypt(want[t]) == 0
    got = frames.copy()
    enc = cve.Cipher(key, n, r)
    for t in range(len(got)):
        enc.encrypt_frame(got[t])
    assert np.array_equal(got, want)
    cve.Cipher(key, n, r).decrypt_frames(got)
    assert np.array_equal(got, frames)


def test_workers_change_ciphertext():
    # test_engine.cpp:189-195: n is a cipher parameter
    key, f = synth.det_key(5), rand_frames(64, 1, 5)[0]
    outs = []
    for n in (1, 2, 4, 8):
        x = f.copy()
        cve.Cipher(key, n, 5).encrypt_frame(x)
        outs.append(x.tobytes())
    assert len(set(outs)) == 4


def test_c_caller_matches_oracle(tmp_path):
    # tests/c_abi_demo.c: a C99 program linked against the library the way a
    # reference caller links libcve.so; its ciphertext digest against the oracle
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe, libdir = str(tmp_path / "c_abi_demo"), os.path.dirname(cve.lib_path)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "c_abi_demo.c"), "-o", exe, "-L", libdir,
                    "-lcve_b200", "-Wl,-rpath," + libdir], check=True, capture_output=True)
    for key in (PLCM, synth.det_key_lasm(3)):
        out = subprocess.run([exe, key], capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stdout + out.stderr
        side, n = 96, 96 * 96 * 3
        f = np.array([((i * 2654435761) >> 24) & 0xFF for i in range(n)], np.uint8)
        f = f.reshape(side, side, 3)
        assert Oracle(key, 8, 5).encrypt(f) == 0
        x = 0
        for i, b in enumerate(f.ravel().tolist()):
            x ^= b << (8 * (i & 3))
        assert out.stdout.split()[:2] == ["ok", f"{x:08x}"], (key, out.stdout)
        assert "seeds=1" in out.stdout


def test_handle_churn_async_teardown():
    # Handles are destroyed without waiting for queued work (buffers are
    # freed in stream order behind it) and streams/memory are pooled: many
    # short clips created and destroyed back to back, PLCM and LASM, with
    # and without a run-ahead frame left queued, must all match the first
    # run's ciphertext and must not grow device memory without bound.
    torch = pytest.importorskip("torch")
    side = 192
    f = rand_frames(side, 2, 77)
    want = {}
    free0 = None
    for it in range(60):
        key = synth.det_key(31) if it % 2 else synth.det_key_lasm(31)
        frames = f.copy()
        c = cve.Cipher(key, 8, 5)
        c.encrypt_frame(frames[0])
        if it % 3 == 0:
            c.encrypt_frame(frames[1])  # second frame: run-ahead queued at destroy
        c.close()
        tag = (it % 2, it % 3 == 0)
        got = frames[0].tobytes() + (frames[1].tobytes() if tag[1] else b"")
        assert want.setdefault(tag, got) == got, it
        if it == 10:
            torch.cuda.synchronize()
            free0 = torch.cuda.mem_get_info()[0]
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] > free0 - (1 << 30)
    o = Oracle(synth.det_key(31), 8, 5)
    a = f[0].copy()
    assert o.encrypt(a) == 0
    assert want[(1, False)][: a.nbytes] == a.tobytes()
