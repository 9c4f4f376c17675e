"""The reference's benchmark and sweep entry points (cve.h:153-206,
capi.cpp:417-505, bench.cpp:60-315) on this engine, checked against the
reference's own library (oracle/_ref).

cve_sweep_rounds is deterministic: its CSV must equal the reference's byte for
byte (this covers Engine::transform's confusion-only / diffusion-only rounds,
the per-round states, the synthetic "natural" image and the P6 input path).
The three bench tables hold timings: the schema, the fixed columns and the
status codes must match.  Argument errors are host-side and run on CPU."""
import numpy as np
import pytest

import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import (Reference, ref_bench_bytegen, ref_bench_phases, ref_bench_video,
                     ref_sweep_rounds)

need_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
PLCM_KEY = synth.det_key(31)
LASM_KEY = synth.det_key_lasm(32)


def status_of(fn, *a, **k):
    try:
        fn(*a, **k)
        return 0
    except cve.CveError as e:
        return e.status


def put_p6(path, img):
    h, w = img.shape[:2]
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode() + img.tobytes())
    return str(path)


# ---- argument errors: CPU ---------------------------------------------------

@need_ref
def test_null_options_and_bad_keys_match_the_reference():
    L = cve.lib
    import ctypes as C
    out = C.c_void_p()
    for name in ("cve_bench_bytegen", "cve_bench_phases", "cve_bench_video", "cve_sweep_rounds"):
        assert getattr(L, name)(None, C.byref(out)) == cve.CVE_ERROR_INVALID_ARGUMENT
    o = cve.SweepOptions(None, 0, None, 0, 0, 0, 0)
    assert L.cve_sweep_rounds(C.byref(o), None) == cve.CVE_ERROR_INVALID_ARGUMENT
    # malformed key: BAD_KEY from every entry point, as in the reference
    for ours, ref in ((cve.bench_bytegen, ref_bench_bytegen), (cve.bench_phases, ref_bench_phases),
                      (cve.bench_video, ref_bench_video), (cve.sweep_rounds, ref_sweep_rounds)):
        want, _ = ref("00zz")
        assert want == cve.CVE_ERROR_BAD_KEY
        assert status_of(ours, "00zz") == want


@need_ref
def test_sweep_argument_errors_match_the_reference(tmp_path):
    # synthetic side not divisible by the worker count: MISMATCH before any work
    want, _ = ref_sweep_rounds(PLCM_KEY, 0, None, 50, 4, 2, 1)
    assert want == cve.CVE_ERROR_MISMATCH
    assert status_of(cve.sweep_rounds, PLCM_KEY, synth_side=50, workers=4, max_rounds=2,
                     seed=1) == want
    # missing / malformed input image
    missing = str(tmp_path / "nope.ppm")
    want, _ = ref_sweep_rounds(PLCM_KEY, 0, missing, 0, 1, 2, 1)
    assert status_of(cve.sweep_rounds, PLCM_KEY, input_path=missing, workers=1,
                     max_rounds=2) == want != 0
    bad = tmp_path / "bad.ppm"
    bad.write_bytes(b"P5\n2 2\n255\n....")
    want, _ = ref_sweep_rounds(PLCM_KEY, 0, str(bad), 0, 1, 2, 1)
    assert status_of(cve.sweep_rounds, PLCM_KEY, input_path=str(bad), workers=1,
                     max_rounds=2) == want != 0


@need_ref
def test_bytegen_and_video_null_arrays_match_the_reference():
    import ctypes as C
    out = C.c_void_p()
    o = cve.BenchBytegenOptions(PLCM_KEY.encode(), 0, None, 3, 1000)
    assert cve.lib.cve_bench_bytegen(C.byref(o), C.byref(out)) == cve.CVE_ERROR_INVALID_ARGUMENT
    v = cve.BenchVideoOptions(PLCM_KEY.encode(), 0, None, 2, 2, 2, 2, 20, 0)
    assert cve.lib.cve_bench_video(C.byref(v), C.byref(out)) == cve.CVE_ERROR_INVALID_ARGUMENT


# ---- cve_sweep_rounds: byte-identical CSV (GPU) -----------------------------

@need_ref
@pytest.mark.gpu
@pytest.mark.parametrize("key,side,workers,rounds,seed", [
    (PLCM_KEY, 64, 2, 3, 9),
    (PLCM_KEY, 96, 1, 5, 1234),
    (PLCM_KEY, 120, 8, 4, 7),
    (LASM_KEY, 64, 4, 3, 5),
    (PLCM_KEY, 51, 3, 2, 77),      # odd side
    (PLCM_KEY, 256, 16, 6, 2024),
])
def test_sweep_rounds_synthetic_matches_reference(key, side, workers, rounds, seed):
    st, want = ref_sweep_rounds(key, 0, None, side, workers, rounds, seed)
    assert st == 0
    got = cve.sweep_rounds(key, synth_side=side, workers=workers, max_rounds=rounds, seed=seed)
    assert got == want
    assert len(got.splitlines()) == rounds + 2


@need_ref
@pytest.mark.gpu
def test_sweep_rounds_defaults_match_reference():
    # synth_side 0 -> 512, workers 0 -> 1, max_rounds 0 -> 10
    st, want = ref_sweep_rounds(PLCM_KEY, 0, None, 0, 0, 0, 3)
    assert st == 0
    assert cve.sweep_rounds(PLCM_KEY, seed=3) == want


@need_ref
@pytest.mark.gpu
@pytest.mark.parametrize("w,h,workers", [(40, 40, 4), (70, 33, 8), (17, 90, 5)])
def test_sweep_rounds_p6_input_matches_reference(tmp_path, w, h, workers):
    img = np.random.default_rng(w * 100 + h).integers(0, 256, (h, w, 3), dtype=np.uint8)
    path = put_p6(tmp_path / "in.ppm", img)
    st, want = ref_sweep_rounds(PLCM_KEY, 0, path, 0, workers, 3, 11)
    assert st == 0
    assert cve.sweep_rounds(PLCM_KEY, input_path=path, workers=workers, max_rounds=3,
                            seed=11) == want


@need_ref
@pytest.mark.gpu
def test_sweep_after_frames_keeps_the_handle_free_engines_independent():
    """The sweep builds its own engines: a live cipher handle's frame order is
    untouched by it."""
    frame = synth.config_frame("C1", 0)
    h = cve.Cipher(synth.config_key("C1"), 8, 5)
    a = frame.copy()
    h.encrypt_frame(a)
    cve.sweep_rounds(PLCM_KEY, synth_side=64, workers=2, max_rounds=2, seed=1)
    b = synth.config_frame("C1", 1).copy()
    h.encrypt_frame(b)
    h2 = cve.Cipher(synth.config_key("C1"), 8, 5)
    a2, b2 = frame.copy(), synth.config_frame("C1", 1).copy()
    h2.encrypt_frame(a2)
    h2.encrypt_frame(b2)
    assert np.array_equal(a, a2) and np.array_equal(b, b2)


# ---- bench tables: schema and fixed columns (GPU) ---------------------------

def rows_of(csv):
    lines = csv.strip().split("\n")
    return lines[0], [ln.split(",") for ln in lines[1:]]


@need_ref
@pytest.mark.gpu
@pytest.mark.parametrize("key,kind", [(PLCM_KEY, "plcm"), (LASM_KEY, "lasm")])
def test_bench_bytegen_schema(key, kind):
    st, ref = ref_bench_bytegen(key, 0, [1, 3], 40000)
    assert st == 0
    got = cve.bench_bytegen(key, worker_counts=[1, 3], iterations=40000)
    rh, rr = rows_of(ref)
    gh, gr = rows_of(got)
    assert gh == rh and len(gr) == len(rr) == 2
    for g, r in zip(gr, rr):
        assert g[:4] == r[:4]              # map, workers, iterations, bytes
        assert g[0] == kind
        assert float(g[4]) > 0 and float(g[5]) > 0
        assert len(g[4].split(".")[1]) == 3 and len(g[5].split(".")[1]) == 3
    # default worker counts 1, 2, 4, 8
    _, dr = rows_of(cve.bench_bytegen(key, iterations=8000))
    assert [r[1] for r in dr] == ["1", "2", "4", "8"]


@need_ref
@pytest.mark.gpu
def test_bench_video_schema_and_realtime_flag():
    st, ref = ref_bench_video(PLCM_KEY, 0, [32, 96], 4, 3, 5, 25)
    assert st == 0
    got = cve.bench_video(PLCM_KEY, sides=[32, 96], workers=4, rounds=3, frames=5, fps=25)
    rh, rr = rows_of(ref)
    gh, gr = rows_of(got)
    assert gh == rh and len(gr) == 2
    for g, r in zip(gr, rr):
        assert g[:6] == r[:6]              # map, side, workers, rounds, frames, fps
        mean, lo, hi = float(g[9]), float(g[10]), float(g[11])
        assert 0 < lo <= mean <= hi
        assert g[8] == "0.000"             # no separate diffusion pass
        assert float(g[6]) >= 0 and float(g[7]) > 0
        side = int(g[1])
        assert abs(float(g[12]) - side * side * 3 / 2**20 / (mean / 1e3)) <= 0.02 * float(g[12]) + 0.01
        assert g[13] == ("1" if mean <= 1000.0 / 25 else "0")
    # a side the worker count does not divide: MISMATCH, like the reference
    want, _ = ref_bench_video(PLCM_KEY, 0, [30], 4, 3, 2, 20)
    assert want == cve.CVE_ERROR_MISMATCH
    assert status_of(cve.bench_video, PLCM_KEY, sides=[30], workers=4, rounds=3, frames=2) == want


@need_ref
@pytest.mark.gpu
def test_bench_phases_schema():
    st, ref = ref_bench_phases(PLCM_KEY, 0, 64, 4, 3, 4)
    assert st == 0
    got = cve.bench_phases(PLCM_KEY, side=64, workers=4, rounds=3, images=4)
    rh, rr = rows_of(ref)
    gh, gr = rows_of(got)
    assert gh == rh and len(gr) == 1
    g = gr[0]
    assert g[:5] == rr[0][:5]              # map, side, workers, rounds, images
    cm, cl, ch_, dm, dl, dh = (float(v) for v in g[5:11])
    assert 0 < cl <= cm <= ch_ and 0 < dl <= dm <= dh


@pytest.mark.gpu
def test_transform_draws_seeds_and_stream_like_frames():
    """bench_phases on a handle's key leaves nothing behind: a fresh handle
    created afterwards still produces the clip's first frame (the harness
    engines are separate), and phases with n not dividing the side fails with
    MISMATCH."""
    assert status_of(cve.bench_phases, PLCM_KEY, side=50, workers=4, rounds=2,
                     images=1) == cve.CVE_ERROR_MISMATCH
