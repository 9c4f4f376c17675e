"""Row f4: the reference's statistical analysis (cve_analyze) and its image
tools (cve_add_noise_file, cve_crop_file), checked byte for byte against the
reference's own library (oracle/_ref): report / CSV text, rewritten files and
status codes (analysis.cpp:51-361, capi.cpp:109-141, 335-383).

The noise / crop tools and every analyze argument error are host-side and run
on CPU; the analysis text needs the GPU (histograms and NPCR/UACI counts)."""
import os

import numpy as np
import pytest

import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import (Reference, ref_add_noise_file, ref_analyze, ref_crop_file,
                     ref_encrypt_file)

PLCM = "005f633937dd9abf3f93ba8c762f1bd43fb8560e3cdd9aef3f7c74d008a265d13f"
need_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


def rgb(w, h, seed):
    return np.random.Generator(np.random.PCG64(seed)).integers(0, 256, (h, w, 3), dtype=np.uint8)


def put_p6(path, img):
    h, w = img.shape[:2]
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode() + img.tobytes())
    return str(path)


def blob(path):
    with open(path, "rb") as fh:
        return fh.read()


def status_of(fn, *a, **k):
    try:
        fn(*a, **k)
        return 0
    except cve.CveError as e:
        return e.status


def container(tmp_path, name, frames, seed=0, workers=4):
    """A CVE1 container made by the reference itself (CPU) from P6 frames."""
    d = tmp_path / f"{name}_src"
    d.mkdir()
    for i, f in enumerate(frames):
        put_p6(d / f"f{i:03d}.ppm", f)
    out = str(tmp_path / f"{name}.cve")
    assert ref_encrypt_file(PLCM, str(d), out, workers=workers) == 0
    return out


# ---- host-side tools: CPU --------------------------------------------------

@need_ref
@pytest.mark.parametrize("side", [16, 57])
@pytest.mark.parametrize("rate,seed", [(0.0, 1), (0.05, 7), (0.37, 123), (1.0, 9)])
def test_noise_p6_matches_reference(tmp_path, side, rate, seed):
    src = put_p6(tmp_path / "a.ppm", rgb(side, side, side + seed))
    assert ref_add_noise_file(src, str(tmp_path / "r.ppm"), rate, seed) == 0
    cve.add_noise_file(src, str(tmp_path / "o.ppm"), rate, seed)
    assert blob(tmp_path / "o.ppm") == blob(tmp_path / "r.ppm")


@need_ref
def test_noise_and_crop_on_container_match_reference(tmp_path):
    cont = container(tmp_path, "c", [rgb(40, 24, s) for s in range(3)])
    assert ref_add_noise_file(cont, str(tmp_path / "rn.cve"), 0.1, 77) == 0
    cve.add_noise_file(cont, str(tmp_path / "on.cve"), 0.1, 77)
    assert blob(tmp_path / "on.cve") == blob(tmp_path / "rn.cve")
    blocks = [(0, 0, 5, 0), (3, 4, 8, 255), (30, 30, 10, 0)]
    assert ref_crop_file(cont, str(tmp_path / "rc.cve"), blocks) == 0
    cve.crop_file(cont, str(tmp_path / "oc.cve"), blocks)
    assert blob(tmp_path / "oc.cve") == blob(tmp_path / "rc.cve")


@need_ref
@pytest.mark.parametrize("blocks", [[], [(0, 0, 1, 255)], [(2, 3, 7, 0), (4, 4, 9, 255)],
                                    [(0, 0, 33, 255)]])
def test_crop_p6_matches_reference(tmp_path, blocks):
    src = put_p6(tmp_path / "a.ppm", rgb(33, 33, 5))
    assert ref_crop_file(src, str(tmp_path / "r.ppm"), blocks) == 0
    cve.crop_file(src, str(tmp_path / "o.ppm"), blocks)
    assert blob(tmp_path / "o.ppm") == blob(tmp_path / "r.ppm")


@need_ref
def test_tool_errors_match_reference(tmp_path):
    sq = put_p6(tmp_path / "sq.ppm", rgb(20, 20, 1))
    rect = put_p6(tmp_path / "rect.ppm", rgb(20, 10, 2))
    junk = tmp_path / "junk.bin"
    junk.write_bytes(b"not an image at all")
    missing = str(tmp_path / "nope.ppm")
    out = str(tmp_path / "out")
    cases = [
        ("noise", (sq, out, -0.1, 1)), ("noise", (sq, out, 1.5, 1)),
        ("noise", (sq, out, float("nan"), 1)), ("noise", (rect, out, 0.1, 1)),
        ("noise", (missing, out, 0.1, 1)), ("noise", (str(junk), out, 0.1, 1)),
        ("crop", (sq, out, [(15, 0, 6, 0)])), ("crop", (sq, out, [(0, 0, 0, 0)])),
        ("crop", (sq, out, [(0, 0, 4, 7)])), ("crop", (sq, out, [(0, 0, 4, 0), (0, 19, 2, 255)])),
        ("crop", (rect, out, [])), ("crop", (missing, out, [])),
        ("crop", (sq, out, [(0xFFFFFFF0, 0, 0x20, 0)])),  # x + side wraps in uint32
    ]
    for kind, args in cases:
        if kind == "noise":
            want, got = ref_add_noise_file(*args), status_of(cve.add_noise_file, *args)
        else:
            want, got = ref_crop_file(*args), status_of(cve.crop_file, *args)
        assert got == want and want != 0, (kind, args, got, want)


@need_ref
def test_analyze_argument_errors_match_reference(tmp_path):
    # every one of these is decided before the GPU reductions (CPU-checkable)
    sq = put_p6(tmp_path / "sq.ppm", rgb(20, 20, 1))
    sq2 = put_p6(tmp_path / "sq2.ppm", rgb(24, 24, 2))
    rect = put_p6(tmp_path / "rect.ppm", rgb(20, 10, 2))
    junk = tmp_path / "junk.bin"
    junk.write_bytes(b"P5\n1 1\n255\n\0")
    cont = container(tmp_path, "c", [rgb(16, 16, s) for s in range(2)])
    cases = [dict(input_path=str(tmp_path / "missing.ppm")), dict(input_path=rect),
             dict(input_path=str(junk)), dict(input_path=cont, frame_index=2),
             dict(input_path=sq, second=sq2), dict(input_path=sq, second=str(junk)),
             dict(input_path=cont, second=cont, second_frame_index=5)]
    for c in cases:
        want, _ = ref_analyze(**c)
        assert want != 0
        assert status_of(cve.analyze, **c) == want, c


# ---- analysis text: GPU ------------------------------------------------------

def flat(side, v):
    return np.full((side, side, 3), v, np.uint8)


ANALYZE_CASES = [
    ("noise_64", lambda: rgb(64, 64, 3), {}),
    ("noise_1", lambda: rgb(1, 1, 4), {}),
    ("noise_2", lambda: rgb(2, 2, 5), dict(samples=5)),
    ("noise_43_csv", lambda: rgb(43, 43, 6), dict(csv=True, seed=11)),
    ("noise_44", lambda: rgb(44, 44, 7), dict(seed=3)),
    ("smooth_300", lambda: synth.correlated_frame(300, 300, 1, 21), dict(samples=3000, seed=5)),
    ("flat", lambda: flat(50, 200), {}),
    ("two_level", lambda: np.where(rgb(96, 96, 9) > 127, 255, 0).astype(np.uint8),
     dict(samples=1)),
]


@pytest.mark.gpu
@need_ref
@pytest.mark.parametrize("name,make,opts", ANALYZE_CASES, ids=[c[0] for c in ANALYZE_CASES])
def test_analyze_p6_matches_reference(tmp_path, name, make, opts):
    src = put_p6(tmp_path / "a.ppm", make())
    st, want = ref_analyze(src, **opts)
    assert st == 0
    assert cve.analyze(src, **opts) == want


@pytest.mark.gpu
@need_ref
@pytest.mark.parametrize("csv", [False, True])
def test_analyze_container_npcr_uaci_matches_reference(tmp_path, csv):
    # ciphertext statistics: frame 1 of a container, NPCR/UACI against the
    # ciphertext of a one-pixel-different plaintext (the paper's differential
    # test) and against a plain P6 of the same side
    frames = [synth.correlated_frame(96, 96, t, 3) for t in range(3)]
    a = container(tmp_path, "a", frames)
    frames[1] = frames[1].copy()
    frames[1][10, 10, 0] ^= 1
    b = container(tmp_path, "b", frames)
    p = put_p6(tmp_path / "p.ppm", rgb(96, 96, 8))
    for second, sfi in [(b, 1), (p, 0), (a, 1)]:
        st, want = ref_analyze(a, second=second, frame_index=1, second_frame_index=sfi,
                               samples=4000, seed=42, csv=csv)
        assert st == 0
        assert cve.analyze(a, second=second, frame_index=1, second_frame_index=sfi,
                           samples=4000, seed=42, csv=csv) == want


@pytest.mark.gpu
@pytest.mark.parametrize("side", [1, 5, 16, 97, 512])
def test_frame_stats_device_vs_numpy(side):
    torch = pytest.importorskip("torch")
    a = rgb(side, side, side)
    b = a.copy()
    flip = np.random.Generator(np.random.PCG64(side)).random(a.shape) < 0.3
    b[flip] = 255 - b[flip]
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    hist = torch.zeros(768, dtype=torch.int64, device="cuda")
    diff = torch.zeros(6, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    cve.frame_stats_device(da.data_ptr(), side, hist.data_ptr(), db.data_ptr(),
                           diff.data_ptr(), s.cuda_stream)
    h, d = hist.cpu().numpy(), diff.cpu().numpy()
    for c in range(3):
        assert np.array_equal(h[256 * c:256 * (c + 1)], np.bincount(a[..., c].ravel(),
                                                                     minlength=256))
        delta = a[..., c].astype(int) - b[..., c].astype(int)
        assert d[c] == np.count_nonzero(delta)
        assert d[3 + c] == np.abs(delta).sum()
