"""Row f1: file pipelines and the CVE1 container on the GPU engine, checked
byte for byte against the reference's own cve_encrypt_file /
cve_decrypt_file (oracle/_ref), plus the reference's error semantics
(proj/tests/test_capi.cpp:176-284, test_io.cpp:258-431)."""
import os

import numpy as np
import pytest

import paper_2302_07411_b200 as cve
from conftest import gpu_present
from workloads import synth
from _oracle import Reference, ref_decrypt_file, ref_encrypt_file

PLCM = "005f633937dd9abf3f93ba8c762f1bd43fb8560e3cdd9aef3f7c74d008a265d13f"
LASM = "01333333333333d33f666666666666e63f6f8104c58f31ed3f"
need_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


def p6(w, h, rgb):
    return f"P6\n{w} {h}\n255\n".encode() + rgb.tobytes()


def rgb(w, h, seed):
    return np.random.Generator(np.random.PCG64(seed)).integers(0, 256, (h, w, 3), dtype=np.uint8)


def blob(path):
    with open(path, "rb") as fh:
        return fh.read()


def put(path, data):
    with open(path, "wb") as fh:
        fh.write(data)


# ---- GPU: byte-identical containers and round trips ------------------------

@pytest.mark.gpu
@need_ref
def test_single_p6_matches_reference(tmp_path):
    put(tmp_path / "in.ppm", p6(8, 8, rgb(8, 8, 1)))
    ours, ref = str(tmp_path / "ours.cve"), str(tmp_path / "ref.cve")
    cve.encrypt_file(PLCM, str(tmp_path / "in.ppm"), ours, workers=2, rounds=3, fps=30)
    assert ref_encrypt_file(PLCM, str(tmp_path / "in.ppm"), ref, 2, 3, 30) == 0
    c = blob(ours)
    assert c == blob(ref)
    assert len(c) == 27 + 8 * 8 * 3 and c[:4] == b"CVE1"
    assert c[18] == 2 and c[20] == 3 and c[21] == 30 and c[23] == 1
    cve.decrypt_file(PLCM, ours, str(tmp_path / "back.ppm"))
    assert blob(tmp_path / "back.ppm") == blob(tmp_path / "in.ppm")


@pytest.mark.gpu
@need_ref
@pytest.mark.parametrize("w,h,n,r", [(50, 30, 4, 5), (30, 50, 3, 2), (97, 61, 8, 5)])
def test_padded_directory_sequence_matches_reference(tmp_path, w, h, n, r):
    d = tmp_path / "frames"
    d.mkdir()
    frames = [rgb(w, h, 10 + k) for k in range(4)]
    for k, f in enumerate(frames):
        put(d / f"f{k:03d}.ppm", p6(w, h, f))
    ours, ref = str(tmp_path / "ours.cve"), str(tmp_path / "ref.cve")
    cve.encrypt_file(PLCM, str(d), ours, workers=n, rounds=r)
    assert ref_encrypt_file(PLCM, str(d), ref, n, r) == 0
    assert blob(ours) == blob(ref)
    # decrypt: ours of ours, ours of the reference's, the reference's of ours
    for src in (ours, ref):
        out = tmp_path / ("dec_" + os.path.basename(src))
        cve.decrypt_file(PLCM, src, str(out))
        for k, f in enumerate(frames):
            assert blob(out / f"frame_{k:06d}.ppm") == p6(w, h, f)
    assert ref_decrypt_file(PLCM, ours, str(tmp_path / "refdec.rgb"), 2) == 0
    assert blob(tmp_path / "refdec.rgb") == b"".join(f.tobytes() for f in frames)


@pytest.mark.gpu
@need_ref
def test_raw_1080p_clip_matches_reference(tmp_path):
    # C4 geometry through the file path: 1920x1080 padded to 1920^2 on device
    frames = [synth.correlated_frame(1920, 1080, t, 99) for t in range(3)]
    put(tmp_path / "clip.rgb", b"".join(f.tobytes() for f in frames))
    key = synth.config_key("C4")
    ours, ref = str(tmp_path / "ours.cve"), str(tmp_path / "ref.cve")
    cve.encrypt_file(key, str(tmp_path / "clip.rgb"), ours, workers=64, raw=(1920, 1080))
    assert ref_encrypt_file(key, str(tmp_path / "clip.rgb"), ref, 64, 0, 0, (1920, 1080)) == 0
    assert blob(ours) == blob(ref)
    cve.decrypt_file(key, ours, str(tmp_path / "back.rgb"), fmt=cve.CVE_OUT_RAW)
    assert blob(tmp_path / "back.rgb") == blob(tmp_path / "clip.rgb")


@pytest.mark.gpu
def test_wh_api_equals_square_api():
    key = synth.det_key(77)
    frames = np.stack([rgb(70, 45, k) for k in range(3)])
    sq = np.stack([cve.pad_to_square(f, 5) for f in frames])
    a = cve.Cipher(key, 5, 5)
    out_wh = a.encrypt_frames_wh(frames)
    b = cve.Cipher(key, 5, 5)
    b.encrypt_frames(sq)
    assert np.array_equal(out_wh, sq)
    back = cve.Cipher(key, 5, 5).decrypt_frames_wh(out_wh, 70, 45)
    assert np.array_equal(back, frames)


@pytest.mark.gpu
def test_decrypt_enforces_geometry_and_key_kind(tmp_path):
    # test_capi.cpp:209-245
    put(tmp_path / "in.ppm", p6(8, 8, rgb(8, 8, 8)))
    out = str(tmp_path / "out.cve")
    cve.encrypt_file(PLCM, str(tmp_path / "in.ppm"), out, workers=2, rounds=3)
    for kw in (dict(workers=4), dict(rounds=5)):
        with pytest.raises(cve.CveError) as e:
            cve.decrypt_file(PLCM, out, str(tmp_path / "a.ppm"), **kw)
        assert e.value.status == cve.CVE_ERROR_MISMATCH
    with pytest.raises(cve.CveError) as e:
        cve.decrypt_file(LASM, out, str(tmp_path / "c.ppm"), io=False)
    assert e.value.status == cve.CVE_ERROR_MISMATCH
    cve.decrypt_file(PLCM, out, str(tmp_path / "g.ppm"), io=False)
    assert blob(tmp_path / "g.ppm") == blob(tmp_path / "in.ppm")


@pytest.mark.gpu
@pytest.mark.parametrize("key", [LASM, PLCM])
def test_raw_video_round_trip_and_auto_directory(tmp_path, key):
    # test_capi.cpp:247-284 (the reference runs it with its LASM key)
    data = rgb(8, 8, 10).tobytes() + rgb(8, 8, 11).tobytes()
    put(tmp_path / "video.rgb", data)
    out = str(tmp_path / "video.cve")
    cve.encrypt_file(key, str(tmp_path / "video.rgb"), out, workers=2, rounds=2, raw=(8, 8))
    c = blob(out)
    assert len(c) == 27 + 2 * 8 * 8 * 3 and c[23] == 2
    assert c[5] == (1 if key == LASM else 0)  # map kind byte
    cve.decrypt_file(key, out, str(tmp_path / "back.rgb"), fmt=cve.CVE_OUT_RAW)
    assert blob(tmp_path / "back.rgb") == data
    cve.decrypt_file(key, out, str(tmp_path / "frames"), io=False)
    assert (tmp_path / "frames" / "frame_000000.ppm").exists()
    assert (tmp_path / "frames" / "frame_000001.ppm").exists()


@pytest.mark.gpu
@need_ref
@pytest.mark.parametrize("workers,count", [(2, 100000), (3, 1000001), (0, 5 << 20), (64, 999)])
def test_nist_export_matches_reference(tmp_path, workers, count):
    # row f3; reference capi.cpp:385-415, test_capi.cpp:399-418
    key = synth.config_key("C4")
    cve.nist_export(key, workers, count, str(tmp_path / "ours.bin"))
    assert Reference.load().cve_nist_export(key.encode(), workers, count,
                                            str(tmp_path / "ref.bin").encode()) == 0
    ours = blob(tmp_path / "ours.bin")
    assert len(ours) == count
    assert ours == blob(tmp_path / "ref.bin")


@pytest.mark.gpu
@need_ref
@pytest.mark.parametrize("workers,count", [(2, 100001), (64, 5 << 18)])
def test_nist_export_lasm_matches_reference(tmp_path, workers, count):
    # row f3 with a LASM key (12 bytes per generator iteration)
    key = synth.det_key_lasm(31)
    cve.nist_export(key, workers, count, str(tmp_path / "ours.bin"))
    assert Reference.load().cve_nist_export(key.encode(), workers, count,
                                            str(tmp_path / "ref.bin").encode()) == 0
    assert blob(tmp_path / "ours.bin") == blob(tmp_path / "ref.bin")


@pytest.mark.gpu
@need_ref
def test_lasm_container_matches_reference(tmp_path):
    # row f1 with a LASM key: the CVE1 container is byte-identical to the
    # reference's, and each side decrypts the other's
    frames = [rgb(50, 30, s) for s in (3, 4, 5)]
    d = tmp_path / "seq"
    d.mkdir()
    for i, f in enumerate(frames):
        put(d / f"frame_{i:06d}.ppm", p6(50, 30, f))
    key = synth.det_key_lasm(77)
    ours, ref = str(tmp_path / "ours.cve"), str(tmp_path / "ref.cve")
    cve.encrypt_file(key, str(d), ours, workers=4, rounds=5)
    assert ref_encrypt_file(key, str(d), ref, workers=4, rounds=5) == 0
    assert blob(ours) == blob(ref)
    cve.decrypt_file(key, ref, str(tmp_path / "back"))
    for i, f in enumerate(frames):
        assert blob(tmp_path / "back" / f"frame_{i:06d}.ppm") == p6(50, 30, f)


# ---- CPU: argument and format checks (raised before any device work) --------

def test_nist_export_argument_errors(tmp_path):
    for args, st in (((PLCM, 2, 0), cve.CVE_ERROR_INVALID_ARGUMENT),
                     ((None, 2, 100), cve.CVE_ERROR_INVALID_ARGUMENT),
                     (("00ff", 2, 100), cve.CVE_ERROR_BAD_KEY)):
        with pytest.raises(cve.CveError) as e:
            cve.nist_export(*args, str(tmp_path / "x.bin"))
        assert e.value.status == st


def status_of(fn, *a, **k):
    try:
        fn(*a, **k)
    except cve.CveError as e:
        return e.status
    return cve.CVE_OK


def test_file_argument_errors(tmp_path):
    with pytest.raises(cve.CveError) as e:
        cve.encrypt_file(PLCM, str(tmp_path / "x.rgb"), str(tmp_path / "x.cve"), raw=(8, 0))
    assert e.value.status == cve.CVE_ERROR_INVALID_ARGUMENT
    assert status_of(cve.encrypt_file, PLCM, str(tmp_path / "missing.ppm"),
                     str(tmp_path / "o.cve")) == cve.CVE_ERROR_IO
    assert status_of(cve.encrypt_file, "00ff", str(tmp_path / "missing.ppm"),
                     str(tmp_path / "o.cve")) == cve.CVE_ERROR_BAD_KEY
    put(tmp_path / "bad.ppm", b"P5\n8 8\n255\n" + bytes(192))
    assert status_of(cve.encrypt_file, PLCM, str(tmp_path / "bad.ppm"),
                     str(tmp_path / "o.cve")) == cve.CVE_ERROR_BAD_FORMAT
    put(tmp_path / "trunc.ppm", b"P6\n8 8\n255\n" + bytes(10))
    assert status_of(cve.encrypt_file, PLCM, str(tmp_path / "trunc.ppm"),
                     str(tmp_path / "o.cve")) == cve.CVE_ERROR_BAD_FORMAT
    assert status_of(cve.encrypt_file, PLCM, str(tmp_path / "trunc.ppm"),
                     str(tmp_path / "o.cve"), rounds=256) == cve.CVE_ERROR_INVALID_ARGUMENT


def good_header(**over):
    h = dict(version=1, kind=0, side=8, w=8, h=8, workers=2, rounds=3, fps=20, count=1)
    h.update(over)
    b = bytearray(b"CVE1")
    b += bytes([h["version"], h["kind"]])
    for k, n in (("side", 4), ("w", 4), ("h", 4), ("workers", 2)):
        b += int(h[k]).to_bytes(n, "little")
    b += bytes([h["rounds"]])
    b += int(h["fps"]).to_bytes(2, "little") + int(h["count"]).to_bytes(4, "little")
    return bytes(b)


@pytest.mark.parametrize("over", [dict(version=2), dict(kind=2), dict(side=0),
                                  dict(workers=0), dict(side=9, w=8, h=8), dict(rounds=0),
                                  dict(w=9), dict(h=0), dict(fps=0)])
def test_container_header_validation(tmp_path, over):
    # container.cpp:31-50 via cve_decrypt_file (fails before any device work)
    hdr = good_header(**over)
    side = int.from_bytes(hdr[6:10], "little")
    put(tmp_path / "c.cve", hdr + bytes(max(side, 1) ** 2 * 3))
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "c.cve"),
                     str(tmp_path / "o.ppm"), io=False) == cve.CVE_ERROR_BAD_FORMAT


def test_container_size_and_magic(tmp_path):
    put(tmp_path / "short.cve", good_header() + bytes(10))
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "short.cve"),
                     str(tmp_path / "o.ppm"), io=False) == cve.CVE_ERROR_BAD_FORMAT
    put(tmp_path / "magic.cve", b"XVE1" + good_header()[4:] + bytes(192))
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "magic.cve"),
                     str(tmp_path / "o.ppm"), io=False) == cve.CVE_ERROR_BAD_FORMAT
    put(tmp_path / "tiny.cve", b"CVE1")
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "tiny.cve"),
                     str(tmp_path / "o.ppm"), io=False) == cve.CVE_ERROR_BAD_FORMAT
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "none.cve"),
                     str(tmp_path / "o.ppm"), io=False) == cve.CVE_ERROR_IO
    put(tmp_path / "ok.cve", good_header() + bytes(192))
    for kw in (dict(workers=4), dict(rounds=5)):
        assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "ok.cve"),
                         str(tmp_path / "o.ppm"), **kw) == cve.CVE_ERROR_MISMATCH
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "ok.cve"), str(tmp_path / "o.ppm"),
                     fmt=7, io=False) == cve.CVE_ERROR_INVALID_ARGUMENT


@pytest.mark.skipif(gpu_present(), reason="checks the no-GPU failure mode")
def test_valid_container_needs_gpu(tmp_path):
    put(tmp_path / "ok.cve", good_header() + bytes(192))
    assert status_of(cve.decrypt_file, PLCM, str(tmp_path / "ok.cve"),
                     str(tmp_path / "o.ppm"), io=False) == cve.CVE_ERROR_INTERNAL
