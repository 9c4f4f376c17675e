#!/usr/bin/env python3
"""Benchmark of the per-frame chaotic confusion/diffusion cipher on B200.

Metric (BASELINE.json): encrypted frames/s and GB/s (5 rounds), % of roofline.
Workload: config C4 -- a 1920x1080 RGB24 clip, zero-padded to 1920^2
(reference frame.cpp:19-39), n = 64 subframes, r = 5 rounds, one PLCM key per
clip -- the largest BASELINE config whose headline target names it (1080p at
1 GPU).  A step = one batch of `--frames` consecutive frames of the clip
(default 25; 20 steps + 3 warm-up = 575 frames of the 1000-frame clip).

  value -- frames/s with the frames already resident in HBM, through the
           device-resident API (cve_cipher_encrypt_frames_async); CUDA events
           on the calling stream bracket the K timed steps; max over ranks.
  e2e   -- the same metric through the drop-in host API
           (cve_cipher_encrypt_frames) on pinned host buffers: every step
           copies its frames host->device and the ciphertext back.

Multi-GPU (torchrun, one rank per GPU): the keystream of one clip is 2n
sequential chaotic orbits, so a single clip does not shard; every rank
encrypts its own clip with its own key (replicas, scaling "weak"); the only
collectives are the barrier and the max-over-ranks of the timings.

--impl reference times the reference's own CPU library (oracle/_ref, the
reference sources compiled by oracle/Makefile) on the same config with all
the host threads it uses (n = 64 worker threads), a bounded number of frames
per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# Each cipher handle drives 1-2 CUDA streams (+2 with the host API); with the
# default 8 hardware work queues, independent handles would falsely serialise
# (multi-clip line).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402

from workloads import synth  # noqa: E402

CONFIG = "C4"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when PEAKS is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--frames", type=int, default=24,
                    help="frames per step (rounded up to a multiple of --gpus)")
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config lines")
    ap.add_argument("--no-rows", action="store_true",
                    help="skip the row f1/f3/f4 measurements")
    ap.add_argument("--shard-devices", default="",
                    help="debug: comma-separated cipher devices of the clip instead of one per "
                         "rank (e.g. 0,0 runs the sharded path on one GPU)")
    ap.add_argument("--clips", type=int, default=32,
                    help="independent clips for the labelled multi-clip line (0: skip)")
    return ap.parse_args()


# ---- distributed plumbing ----------------------------------------------------

class Dist:
    """One process per GPU (torchrun).  The default process group is NCCL on
    GPU ranks, but the bench's own collectives -- the barrier around timed
    regions and the max of timings -- go through a gloo group on the host: an
    NCCL barrier is a kernel that spins on the rank's GPU while it waits, and
    on GPUs 1..N-1 it would time-slice with rank 0's shards of the clip."""

    def __init__(self, use_cuda: bool):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.host = None
        if self.world > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = "nccl" if use_cuda else "gloo"
            if use_cuda:
                import torch
                torch.cuda.set_device(self.local)
            td.init_process_group(backend=backend)
            self.pg = td
            self.host = td.new_group(backend="gloo") if backend != "gloo" else None

    def barrier(self):
        if self.pg:
            self.pg.barrier(group=self.host)

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)  # host tensor, gloo
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX, group=self.host)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---- clocks during the timed region -------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_indices):
        self.idx, self.rows, self.proc, self.thr = gpu_indices, [], None, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(i) for i in self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thr.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---- workload --------------------------------------------------------------------

def frame_pool(name: str, count: int):
    return np.stack([synth.config_frame(name, 2 + t) for t in range(count)])


def peaks():
    try:
        with open(PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def baseline_roofline(side: int, hbm_gbs: float) -> dict:
    """BASELINE.json's roofline per frame: the slower of the frame's HBM
    bytes (2F) at peak and the PRBG's FP64 ops at the measured FP64 peak
    (3 ops per lane-iteration in the reference formulation, r * side^2
    lane-iterations per frame)."""
    F = side * side * 3
    hbm_us = 2 * F / (hbm_gbs * 1e9) * 1e6
    out = {"hbm_us": hbm_us}
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            tf = float(json.load(fh)["fp64_tflops"])
        fp64_us = 3 * synth.ROUNDS * side * side / (tf * 1e12) * 1e6
        out.update({"fp64_us": fp64_us, "fp64_tflops_measured": tf,
                    "bound_us": max(hbm_us, fp64_us)})
    except (OSError, KeyError, ValueError):
        out["bound_us"] = hbm_us
    return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_baseline(name: str, seconds: float) -> dict:
    """The reference library (oracle/_ref) on host cores, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Reference  # checker / CPU baseline only
    if not Reference.available():
        return {"value": None, "unit": "frames/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref/libcve_ref.so not built"}
    c = synth.CONFIGS[name]
    ref = Reference(synth.config_key(name), c["workers"], synth.ROUNDS, 1)
    pool = frame_pool(name, 4)
    frames, t0 = 0, time.perf_counter()
    while True:
        f = pool[frames % len(pool)].copy()
        assert ref.encrypt(f) == 0
        frames += 1
        el = time.perf_counter() - t0
        if (el >= seconds and frames >= 3) or frames >= 400:
            break
    cores = min(c["workers"], os.cpu_count() or 1)
    return {"value": frames / el, "unit": "frames/s", "cores": cores, "kind": "reference",
            "sample": f"{frames} consecutive {name} frames ({synth.config_side(name)}^2, "
                      f"n={c['workers']}, r=5) in {el:.2f} s via cve_cipher_encrypt_frame, "
                      f"parallel=1 ({c['workers']} threads on {os.cpu_count()} host cpus, "
                      f"{cpu_model()})"}


def rows_measure(stream) -> dict:
    """SURVEY §8(f) rows next to the headline, each on the C4 geometry, this
    engine vs the reference library (oracle/_ref, the CPU baseline legs of
    these rows) on the same inputs:
      f1  cve_encrypt_file / cve_decrypt_file, raw 1920x1080 clip <-> CVE1
      f2  a LASM key on the C4 geometry (device-resident frames), with the
          LASM chain's ns/iteration
      f3  cve_nist_export, 64 workers
      f4  cve_analyze of a 1920^2 frame with NPCR/UACI, and the device
          reductions alone (cve_frame_stats_device) against HBM."""
    import tempfile
    import torch
    import paper_2302_07411_b200 as cve
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import (Reference, ref_analyze, ref_decrypt_file,  # CPU baseline legs only
                         ref_encrypt_file)
    have_ref = Reference.available()
    c = synth.CONFIGS["C4"]
    W, H, n = c["width"], c["height"], c["workers"]
    key = synth.config_key("C4")
    side_c4 = synth.config_side("C4")
    nf = 24
    rows = {}

    def blob(p):
        with open(p, "rb") as fh:
            return fh.read()

    # RAM-backed scratch when there is room: disk writeback from one leg
    # otherwise shows up as noise in the next (host I/O, not the engine)
    tmp_root = None
    try:
        st = os.statvfs("/dev/shm")
        if st.f_bavail * st.f_frsize > (4 << 30):
            tmp_root = "/dev/shm"
    except OSError:
        pass
    with tempfile.TemporaryDirectory(dir=tmp_root) as d:
        raw = os.path.join(d, "clip.rgb")
        pool = [synth.correlated_frame(W, H, t, 7000 + c["key_seed"]) for t in range(4)]
        with open(raw, "wb") as fh:
            for t in range(nf):
                fh.write(pool[t % 4].tobytes())
        ours, back = os.path.join(d, "ours.cve"), os.path.join(d, "ours.rgb")
        t_enc = t_dec = float("inf")
        for rep in range(3):  # best of the 2nd/3rd calls: the first pays one-time
            t0 = time.perf_counter()  # pinned-staging and engine setup
            cve.encrypt_file(key, raw, ours, workers=n, rounds=synth.ROUNDS, raw=(W, H))
            te = time.perf_counter() - t0
            t0 = time.perf_counter()
            cve.decrypt_file(key, ours, back, fmt=cve.CVE_OUT_RAW)
            td = time.perf_counter() - t0
            if rep:
                t_enc, t_dec = min(t_enc, te), min(t_dec, td)
            if rep < 2:  # unlinked: their dirty pages are dropped, not written back
                os.remove(ours)
                os.remove(back)
        f1 = {"workload": f"{nf}-frame raw {W}x{H} RGB24 file -> CVE1 (n={n}, r=5) and back, "
                          "wall clock incl. file I/O, best of the 2nd/3rd calls; "
                          f"scratch {'RAM (/dev/shm)' if tmp_root else 'disk'}",
              "encrypt_file": {"value": nf / t_enc, "unit": "frames/s"},
              "decrypt_file": {"value": nf / t_dec, "unit": "frames/s"},
              "round_trip": blob(back) == blob(raw)}
        if have_ref:
            refc, refb = os.path.join(d, "ref.cve"), os.path.join(d, "ref.rgb")
            t0 = time.perf_counter()
            assert ref_encrypt_file(key, raw, refc, workers=n, rounds=synth.ROUNDS,
                                    raw=(W, H)) == 0
            r_enc = time.perf_counter() - t0
            t0 = time.perf_counter()
            assert ref_decrypt_file(key, refc, refb, fmt=2) == 0
            r_dec = time.perf_counter() - t0
            os.remove(refb)
            f1["reference"] = {"encrypt_file": nf / r_enc, "decrypt_file": nf / r_dec,
                               "unit": "frames/s", "cores": os.cpu_count()}
            f1["container_identical"] = blob(refc) == blob(ours)
        rows["f1"] = f1

        nbytes = 64 << 20
        o3 = os.path.join(d, "ours.nist")
        t3 = float("inf")
        for _ in range(2):
            t0 = time.perf_counter()
            cve.nist_export(key, n, nbytes, o3)
            t3 = min(t3, time.perf_counter() - t0)
        f3 = {"workload": f"{nbytes >> 20} MiB of generator bytes, {n} workers",
              "value": nbytes / t3 / 1e6, "unit": "MB/s"}
        if have_ref:
            r3 = os.path.join(d, "ref.nist")
            L = Reference.load()
            t0 = time.perf_counter()
            assert L.cve_nist_export(key.encode(), n, nbytes, r3.encode()) == 0
            f3["reference"] = {"value": nbytes / (time.perf_counter() - t0) / 1e6,
                               "unit": "MB/s", "cores": 1}
            f3["identical"] = blob(r3) == blob(o3)
        # the reference's own bench entry points, both libraries: cve_bench_bytegen
        # (64 workers) and cve_bench_video (its timing method, bench.cpp:186-231:
        # synchronous per-frame calls on host memory) at the C4 geometry
        from _oracle import ref_bench_bytegen, ref_bench_video

        def table(csv):
            lines = csv.strip().split("\n")
            return [dict(zip(lines[0].split(","), ln.split(","))) for ln in lines[1:]]
        its = 20_000_000
        bg = table(cve.bench_bytegen(key, worker_counts=[n], iterations=its))[0]
        f3["bench_bytegen"] = {"workers": n, "iterations": its,
                               "throughput_mbps": float(bg["throughput_mbps"])}
        bv = table(cve.bench_video(key, sides=[side_c4], workers=n, frames=40, fps=20))[0]
        f3["bench_video"] = {"side": side_c4, "workers": n, "frames": 40,
                             "total_mean_ms": float(bv["total_mean_ms"]),
                             "throughput_mbps": float(bv["throughput_mbps"]),
                             "bytegen_mean_ms": float(bv["bytegen_mean_ms"]),
                             "rounds_mean_ms": float(bv["confuse_mean_ms"])}
        if have_ref:
            st, csv = ref_bench_bytegen(key, 0, [n], its)
            if st == 0:
                f3["bench_bytegen"]["reference_throughput_mbps"] = float(
                    table(csv)[0]["throughput_mbps"])
            st, csv = ref_bench_video(key, 0, [side_c4], n, 5, 12, 20)
            if st == 0:
                rv = table(csv)[0]
                f3["bench_video"]["reference"] = {"frames": 12,
                                                  "total_mean_ms": float(rv["total_mean_ms"]),
                                                  "throughput_mbps": float(rv["throughput_mbps"])}
        rows["f3"] = f3

        side = synth.config_side("C4")
        a_img, b_img = synth.config_frame("C4", 2), synth.config_frame("C4", 3)
        pa, pb = os.path.join(d, "a.ppm"), os.path.join(d, "b.ppm")
        for p_, img in ((pa, a_img), (pb, b_img)):
            with open(p_, "wb") as fh:
                fh.write(f"P6\n{side} {side}\n255\n".encode() + img.tobytes())
        t4 = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            txt = cve.analyze(pa, second=pb, seed=1)
            t4 = min(t4, time.perf_counter() - t0)
        f4 = {"workload": f"cve_analyze of a {side}^2 C4 frame with NPCR/UACI vs a second frame "
                          "(P6 files), wall clock, best of 3",
              "analyze_ms": t4 * 1e3}
        if have_ref:
            tr = float("inf")
            for _ in range(3):
                t0 = time.perf_counter()
                st, rtxt = ref_analyze(pa, second=pb, seed=1)
                tr = min(tr, time.perf_counter() - t0)
            f4["reference_analyze_ms"] = tr * 1e3
            f4["identical_text"] = st == 0 and rtxt == txt
        # device reductions alone: histograms (reads F) + NPCR/UACI (reads 2F),
        # cycling over 8 frame pairs (177 MB, larger than L2)
        pairs = 8
        da = torch.from_numpy(np.stack([synth.config_frame("C4", 2 + t) for t in range(4)]))
        da = da.repeat(pairs // 4, 1, 1, 1).contiguous().cuda()
        db = torch.roll(da, 1, dims=0).contiguous()
        fb = side * side * 3
        hist = torch.zeros(768, dtype=torch.int64, device="cuda")
        diff = torch.zeros(6, dtype=torch.int64, device="cuda")

        def stats(i):
            cve.frame_stats_device(da.data_ptr() + (i % pairs) * fb, side, hist.data_ptr(),
                                   db.data_ptr() + (i % pairs) * fb, diff.data_ptr(),
                                   stream.cuda_stream)
        for i in range(pairs):
            stats(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 48
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(reps):
            stats(i)
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        gbs = 2 * fb / (us * 1e-6) / 1e9
        hbm, _ = peaks()
        f4["device_stats"] = {"us_per_frame_pair": us, "achieved_gbs": gbs,
                              "frac_of_hbm": gbs / hbm,
                              "bytes": "2F per pair (one fused pass reads both frames once); "
                                       "8 pairs cycled, 177 MB > L2"}
        rows["f4"] = f4

    rows["f2"] = lasm_row(stream, have_ref)
    return rows


def one_frame_clip() -> dict:
    """BASELINE config C1 as specified: one 480x480 frame encrypted then
    decrypted, each with a fresh handle (create, the drop-in per-frame call on
    a host buffer, destroy), wall clock, median of 10 after a warm-up; the
    reference library the same way on the host cores."""
    import paper_2302_07411_b200 as cve
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Reference  # CPU baseline leg only
    c = synth.CONFIGS["C1"]
    key, n = synth.config_key("C1"), c["workers"]
    plain = synth.config_frame("C1", 0)

    def ours():
        f = plain.copy()
        with cve.Cipher(key, n, synth.ROUNDS) as e:
            e.encrypt_frame(f)
        with cve.Cipher(key, n, synth.ROUNDS) as d:
            d.decrypt_frame(f)
        return f

    def theirs():
        f = plain.copy()
        e = Reference(key, n, synth.ROUNDS, 1)
        assert e.encrypt(f) == 0
        e.close()
        d = Reference(key, n, synth.ROUNDS, 1)
        assert d.decrypt(f) == 0
        d.close()
        return f

    out = {"workload": "C1: one 480x480 frame, encrypt then decrypt, a fresh handle for each "
                       "(create + per-frame call on a host buffer + destroy), median of 10",
           "unit": "ms per round trip"}
    legs = [("value", ours)] + ([("reference", theirs)] if Reference.available() else [])
    for label, fn in legs:
        assert np.array_equal(fn(), plain)  # warm-up + round-trip check
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[label] = float(np.median(ts))
    return out


def lasm_row(stream, have_ref: bool) -> dict:
    """Row f2: a LASM key (acceptance det_key recipe) on the C4 geometry.
    Ours: 12 device-resident frames after a 2-frame warm-up, CUDA events on
    the calling stream.  Reference: its own library on the host cores, a
    bounded sample of the same frames; the first two ciphertexts compared."""
    import torch
    import paper_2302_07411_b200 as cve
    c = synth.CONFIGS["C4"]
    n, side = c["workers"], synth.config_side("C4")
    key = synth.det_key_lasm(4242 + n)
    pool = frame_pool("C4", 4)
    nl = 12
    dev = torch.from_numpy(np.stack([pool[t % 4] for t in range(nl)])).cuda()
    ci = cve.Cipher(key, n, synth.ROUNDS)
    ci.encrypt_frames_device(dev.data_ptr(), side, 2, stream.cuda_stream)
    stream.synchronize()
    ci.stats()  # fold the warm-up timings
    st0 = ci.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ci.encrypt_frames_device(dev.data_ptr(), side, nl, stream.cuda_stream)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    st1 = ci.stats()
    iters = st1["keystream_iters"] - st0["keystream_iters"]
    chain_ms = st1["chain_ms"] - st0["chain_ms"]
    ns = chain_ms * 1e6 / iters if iters else None
    per_frame = synth.ROUNDS * side * side * 3 // (12 * n)  # LASM iterations per lane per frame
    row = {"workload": f"LASM key, C4 geometry ({side}^2, n={n}, r=5), {nl} device-resident "
                       "frames after a 2-frame warm-up",
           "value": nl / (ms / 1e3), "unit": "frames/s",
           "note": "includes one run-ahead frame: reads <= N/(N-1) high; chain_bound is the "
                   "steady-state rate",
           "chain": {"ns_per_iteration": ns, "bytes_per_iteration": 12,
                     "iterations_per_lane_per_frame": per_frame,
                     "chain_bound_frames_per_s": 1e9 / (per_frame * ns) if ns else None,
                     "note": "one LASM iteration = two dependent glibc-exact sin evaluations"}}
    if have_ref:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from _oracle import Reference  # CPU baseline leg only
        ref = Reference(key, n, synth.ROUNDS, 1)
        mine = cve.Cipher(key, n, synth.ROUNDS)
        frames, same, el = 0, True, 0.0
        while True:
            f = pool[frames % 4].copy()
            t0 = time.perf_counter()
            assert ref.encrypt(f) == 0
            el += time.perf_counter() - t0
            if frames < 2:  # parity spot check, outside the reference's timed calls
                g = pool[frames % 4].copy()
                mine.encrypt_frame(g)
                same = same and bool(np.array_equal(f, g))
            frames += 1
            if (el >= 8.0 and frames >= 3) or frames >= 200:
                break
        row["reference"] = {"value": frames / el, "unit": "frames/s",
                            "cores": min(n, os.cpu_count() or 1),
                            "sample": f"{frames} consecutive frames in {el:.1f} s, parallel=1 "
                                      f"({n} threads on {os.cpu_count()} host cpus)"}
        row["identical_first_frames"] = same
        # few subframes (C1 geometry, n = 8): 2n chains only, and a CPU core
        # walks one glibc-sin chain faster than an SM -- reported, not hidden
        c1 = synth.CONFIGS["C1"]
        k1 = synth.det_key_lasm(4242 + c1["workers"])
        fr = np.stack([synth.config_frame("C1", t % 3) for t in range(12)])
        h1, r1 = cve.Cipher(k1, c1["workers"], synth.ROUNDS), Reference(k1, c1["workers"],
                                                                         synth.ROUNDS, 1)
        a, b = fr.copy(), fr.copy()
        h1.encrypt_frames(a[:2])
        for i in range(2):
            assert r1.encrypt(b[i]) == 0
        t0 = time.perf_counter()
        h1.encrypt_frames(a[2:])
        ours1 = 10 / (time.perf_counter() - t0)
        t0 = time.perf_counter()
        for i in range(2, 12):
            assert r1.encrypt(b[i]) == 0
        ref1 = 10 / (time.perf_counter() - t0)
        row["few_subframes"] = {"workload": "LASM key, C1 geometry (480^2, n=8), 10 frames "
                                            "through the host API after 2",
                                "value": ours1, "reference": ref1, "unit": "frames/s",
                                "identical": bool(np.array_equal(a, b)),
                                "crossover": "a LASM clip is 2n sequential glibc-sin orbits at "
                                             "~256 ns per iteration on the GPU: the GPU is ahead "
                                             "of the reference's host threads from n >= 32 "
                                             "subframes (C3 n=32: 167 vs 122 frames/s, C4 n=64: "
                                             "54 vs 24); at n = 8-16 (C1, C2) the host cores "
                                             "are faster (tools/lasm_small_probe.py, DESIGN §10)"}
    return row


METRIC = "encrypted frames/s (5 rounds)"


def frames_per_step(args) -> int:
    """Frames per step: --frames rounded up to a multiple of the GPU count, so
    every shard of the clip gets the same number of frames per step."""
    g = len(args.shard_devices.split(",")) if args.shard_devices else max(1, args.gpus)
    return (max(1, args.frames) + g - 1) // g * g


def scaling_of(gpus: int) -> str:
    # the headline is ONE clip sharded over the GPUs: total work per step is
    # fixed as N grows
    return "strong"


def config_dict(name: str, frames: int, world: int) -> dict:
    """Identical in both arms (same workload, frames per step and L2 note)."""
    c = synth.CONFIGS[name]
    side = synth.config_side(name)
    shard = ("one clip, frame k of a step ciphered on GPU k mod %d from its keystream window "
             "copied peer-to-peer from GPU 0, where the clip's 2n generator orbits run" % world
             if world > 1 else "one clip on one GPU")
    return {"workload": f"{name}: {c['frames']}-frame {c['width']}x{c['height']} RGB24 clip, "
                        f"zero-padded to {side}^2, n={c['workers']} subframes, r=5 rounds, "
                        f"PLCM key; {shard}",
            "side": side, "workers": c["workers"], "rounds": synth.ROUNDS,
            "frames_per_step": frames, "frame_bytes": side * side * 3,
            "l2": ("inputs larger than L2" if frames * side * side * 3 > 126e6 else
                   "inputs fit in L2") + f" ({frames * side * side * 3 / 1e6:.0f} MB per step)",
            "parallelism": f"frames sharded x{world}" if world > 1 else "single GPU"}


# ---- reference arm ------------------------------------------------------------------

def mapped_libraries() -> list:
    """Shared objects of this repo mapped into this process (evidence that an
    arm ran the library it claims: the reference arm must map only
    oracle/_ref/libcve_ref.so, never libcve_b200.so)."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for ln in fh:
                path = ln.split()[-1] if ln.strip() else ""
                if path.startswith(ROOT) and path.endswith(".so"):
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


def run_reference(args) -> None:
    """The reference's own CPU library (oracle/_ref: the reference sources
    compiled by oracle/Makefile) through its stock per-frame call,
    cve_cipher_encrypt_frame (reference capi.cpp:166-181), timed like the
    reference's bench_video (bench.cpp:186-231: steady clock around each
    encrypt of pre-generated frames).  Same workload, config dict, frames
    per step, metric and unit as the B200 arm; rank 0 only."""
    dist = Dist(use_cuda=False)
    rank = dist.rank
    dist.close()  # no collectives: the reference arm runs on rank 0 only
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Reference
    name = args.config
    c = synth.CONFIGS[name]
    side = synth.config_side(name)
    F = frames_per_step(args)
    line = {"impl": "reference", "metric": METRIC, "unit": "frames/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": scaling_of(args.gpus), "vs_baseline": None,
            "dtype": "f64/u8", "data": "synthetic",
            "config": config_dict(name, F, len(args.shard_devices.split(","))
                                  if args.shard_devices else args.gpus)}
    if not Reference.available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libcve_ref.so was not built"}))
        return
    ref = Reference(synth.config_key(name), c["workers"], synth.ROUNDS, 1)
    pool = frame_pool(name, 8)
    k = 0

    def step():
        nonlocal k
        for _ in range(F):
            f = pool[k % len(pool)].copy()
            assert ref.encrypt(f) == 0
            k += 1

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    fps = args.steps * F / el
    cores = min(c["workers"], os.cpu_count() or 1)
    line.update({"value": fps, "ms_per_step": el * 1e3 / args.steps,
                 "gbps": fps * side * side * 3 / 1e9,
                 "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores,
                                  "kind": "reference",
                                  "sample": f"{args.steps} steps x {F} consecutive frames of the "
                                            f"{name} clip after {args.warmup} warm-up steps, "
                                            f"reference libcve (oracle/_ref) with parallel=1 "
                                            f"({c['workers']} threads, {os.cpu_count()} host cpus, "
                                            f"{cpu_model()})"},
                 "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0},
                 "native_so_loaded": mapped_libraries()})
    print(json.dumps(line))


# ---- B200 arm -------------------------------------------------------------------------

def run_b200(args) -> None:
    import torch
    dist = Dist(use_cuda=True)
    torch.cuda.set_device(dist.local)
    import paper_2302_07411_b200 as cve
    cve.set_device(dist.local)

    name = args.config
    c = synth.CONFIGS[name]
    side, n, F = synth.config_side(name), c["workers"], frames_per_step(args)
    fb = side * side * 3
    devs = ([int(v) for v in args.shard_devices.split(",")] if args.shard_devices
            else list(range(dist.world)))
    G = len(devs)
    key = synth.config_key(name)  # THE clip: one key, sharded over the GPUs
    pool = frame_pool(name, 8)
    lead = dist.rank == 0  # rank 0 drives the sharded clip on every GPU
    host = torch.empty((F, side, side, 3), dtype=torch.uint8, pin_memory=True)
    hnp = host.numpy()
    for t in range(F):
        hnp[t] = pool[t % len(pool)]
    stream = torch.cuda.current_stream()
    # frame f of a step lives on shard f % G (its own GPU's HBM)
    shard_frames = [host[i::G].contiguous().to(f"cuda:{d}") for i, d in enumerate(devs)] \
        if lead else []
    shard_streams = ([stream] + [torch.cuda.Stream(device=d) for d in devs[1:]]) if lead else []

    def make(k):
        return cve.Cipher(k, n, synth.ROUNDS, devices=devs if G > 1 else None)

    def run_step(h, decrypt=False):
        if G == 1:
            fn = h.decrypt_frames_device if decrypt else h.encrypt_frames_device
            fn(shard_frames[0].data_ptr(), side, F, stream.cuda_stream)
        else:
            fn = h.decrypt_frames_sharded if decrypt else h.encrypt_frames_sharded
            fn([t.data_ptr() for t in shard_frames], side, F,
               [s_.cuda_stream for s_ in shard_streams])

    def sync_all():
        for d in sorted(set(devs if lead else [dist.local])):
            torch.cuda.synchronize(d)

    def timed(h, steps, decrypt=False):
        """Device time (ms) of `steps` steps: CUDA events on every shard's
        stream, max over the shards (and over ranks by the caller)."""
        e0 = [torch.cuda.Event(enable_timing=True) for _ in devs]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in devs]
        sync_all()
        for i in range(G):
            e0[i].record(shard_streams[i])
        for _ in range(steps):
            run_step(h, decrypt)
        for i in range(G):
            e1[i].record(shard_streams[i])
        sync_all()
        return max(e0[i].elapsed_time(e1[i]) for i in range(G))

    # ---- value: device-resident frames of the one clip ----
    enc = make(key) if lead else None
    if lead:
        for _ in range(args.warmup):
            run_step(enc)
        sync_all()
        enc.take_prbg_times()
        st0 = enc.stats()
    dist.barrier()
    with ClockSampler(sorted(set(devs)) if lead else [dist.local]) as clk:
        ms_local = timed(enc, args.steps) if lead else 0.0
    dist.barrier()
    ms = dist.max(ms_local)
    frames_all = args.steps * F
    value = frames_all / (ms / 1e3)
    if lead:
        st1 = enc.stats()
        chain_times = enc.take_prbg_times()
        launches = st1["kernel_launches"] - st0["kernel_launches"]
    else:
        st0 = st1 = {k: 0 for k in ("keystream_iters", "chain_ms", "prbg_ms", "cipher_ms",
                                    "kernel_launches", "guard_replays")}
        chain_times, launches = np.zeros(0), 0

    # ---- e2e: drop-in host API on pinned buffers (the same sharded handle
    # kind: frames dealt round-robin over the GPUs) ----
    e2e_s = 0.0
    if lead:
        e2e_enc = make(key)
        for _ in range(args.warmup):
            e2e_enc.encrypt_frames(hnp)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_enc.encrypt_frames(hnp)  # H2D + keystream + rounds + D2H, synchronous
        e2e_s = time.perf_counter() - t0
        del e2e_enc
    dist.barrier()
    e2e_value = frames_all / dist.max(e2e_s)

    # ---- labelled: the reference's own call pattern -- one synchronous,
    # in-place cve_cipher_encrypt_frame per frame on pageable numpy memory ----
    single_fps = None
    if lead:
        single = make(key)
        pageable = [hnp[t].copy() for t in range(F)]
        for t in range(min(3, F)):
            single.encrypt_frame(pageable[t])
        t0 = time.perf_counter()
        for t in range(F):
            single.encrypt_frame(pageable[t])
        single_fps = F / (time.perf_counter() - t0)
        del single, pageable

    # ---- labelled decrypt line: the same clip decrypted (fresh handle) ----
    dec_ms = 0.0
    if lead:
        dec = make(key)
        for _ in range(args.warmup):
            run_step(dec, decrypt=True)
        dec_ms = timed(dec, args.steps, decrypt=True)
        del dec
    dec_ms = dist.max(dec_ms)
    decrypt_line = {"value": args.steps * F / (dec_ms / 1e3), "unit": "frames/s",
                    "note": "labelled: decryption of the same clip, device-resident, sharded "
                            "like the headline"}

    # ---- per-config lines (value only, device-resident, short clips) ----
    per_config = {}
    if not args.no_configs and G == 1:
        for cname in ("C1", "C2", "C3", "C4", "C5"):
            cc = synth.CONFIGS[cname]
            cside = synth.config_side(cname)
            # one frame of keystream run-ahead precedes the timed region, so
            # a clip of N frames reads ~N/(N-1) high: N >= 24 keeps that <= 4 %
            nfr = {"C1": 64, "C2": 48, "C3": 48, "C4": 24, "C5": 24}[cname]
            buf = torch.from_numpy(np.stack([synth.config_frame(cname, 2 + t) for t in range(2)]))
            buf = buf.repeat(nfr // 2, 1, 1, 1).contiguous().cuda()
            hh = cve.Cipher(synth.det_key(cc["key_seed"]), cc["workers"], synth.ROUNDS)
            hh.encrypt_frames_device(buf.data_ptr(), cside, 2, stream.cuda_stream)  # warm-up
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            hh.encrypt_frames_device(buf.data_ptr(), cside, nfr, stream.cuda_stream)
            ev1.record(stream)
            torch.cuda.synchronize()
            cms = ev0.elapsed_time(ev1)
            per_config[cname] = {"side": cside, "workers": cc["workers"], "frames": nfr,
                                 "value": nfr / (cms / 1e3), "unit": "frames/s",
                                 "ms_per_frame": cms / nfr,
                                 "note": "includes one run-ahead frame: reads <= N/(N-1) high"}
            del hh, buf
        if dist.world == 1:
            per_config["C1"]["one_frame_clip"] = one_frame_clip()

    # ---- labelled multi-clip line: M independent clips (keys) per GPU, every
    # rank on its own GPU (weak scaling; the headline above is ONE clip) ----
    multi = None
    if args.clips > 0:
        M, MF = args.clips, 8
        base = torch.from_numpy(np.stack([pool[t % len(pool)] for t in range(MF)]))
        base = base.to(f"cuda:{dist.local}")
        bufs = [base.clone() for _ in range(M)]
        streams = [torch.cuda.Stream() for _ in range(M)]
        # one hardware queue per handle: M <= CUDA_DEVICE_MAX_CONNECTIONS
        # handles never share a queue (cve_set_streams_per_handle)
        cve.set_streams_per_handle(1)
        hs = [cve.Cipher(synth.det_key(7000 + 100 * dist.rank + k), n, synth.ROUNDS)
              for k in range(M)]
        cve.set_streams_per_handle(2)
        for h, b, s_ in zip(hs, bufs, streams):
            h.encrypt_frames_device(b.data_ptr(), side, MF, s_.cuda_stream)
        torch.cuda.synchronize()
        dist.barrier()
        msteps = 3
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(M)]
        start.record(stream)
        for s_ in streams:
            s_.wait_event(start)
        for _ in range(msteps):
            for h, b, s_ in zip(hs, bufs, streams):
                h.encrypt_frames_device(b.data_ptr(), side, MF, s_.cuda_stream)
        for e, s_ in zip(ends, streams):
            e.record(s_)
        torch.cuda.synchronize()
        el = dist.max(max(start.elapsed_time(e) for e in ends)) / 1e3
        multi = {"clips_per_gpu": M, "value": M * MF * msteps * dist.world / el,
                 "unit": "frames/s", "frames_per_clip": MF * msteps,
                 "streams_per_handle": 1, "scaling": "weak",
                 "note": "labelled scenario, not the headline: independent clips/keys "
                         "run concurrently on every GPU through the device-resident API; "
                         "CUDA events from a common start to each clip stream's end, max "
                         "over ranks"}
        del hs, bufs
        torch.cuda.empty_cache()

    # ---- roofline / evidence ----
    hbm, hbm_src = peaks()
    frames_timed = args.steps * F
    alg_bytes = 2 * fb  # plaintext read + ciphertext write per frame
    iters_timed = st1["keystream_iters"] - st0["keystream_iters"]
    chain_ms = st1["chain_ms"] - st0["chain_ms"]
    prbg_ms = st1["prbg_ms"] - st0["prbg_ms"]
    cipher_ms = st1["cipher_ms"] - st0["cipher_ms"]
    ns_iter = chain_ms * 1e6 / max(iters_timed, 1)
    cipher_gbs = frames_timed * alg_bytes / (cipher_ms / 1e3) / 1e9 if cipher_ms else None
    # dominant kernel, per launch: algorithmic bytes of the frames its
    # iterations serve / its mean CUDA-event duration on its own stream
    iters_per_frame = synth.ROUNDS * side * side // (2 * n)
    launch_iters = iters_timed / max(len(chain_times), 1)
    alg_per_launch = alg_bytes * launch_iters / iters_per_frame
    chain_gbs = (alg_per_launch / (float(np.mean(chain_times)) / 1e3) / 1e9
                 if len(chain_times) else None)
    traffic_per_launch = ckpt_per_launch = None
    frame_traffic = None
    try:  # DRAM bytes per launch from the committed ncu --set full captures
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh)
        ch = tr.get("k_prbg_chain_walk") or tr["k_prbg_chain"]
        traffic_per_launch = ch["dram_bytes"] / ch["iterations"] * launch_iters
        ckpt_per_launch = ch["checkpoint_bytes_written"] / ch["iterations"] * launch_iters
        # per-frame device DRAM traffic, cold-cache upper bound: the sum of
        # every kernel's per-launch DRAM bytes (ncu replays each launch with a
        # flushed L2, so reuse of the frame buffers across rounds is not seen)
        ver = tr["k_prbg_verify_emit"]
        rk = "k_encrypt_round_rows" if "k_encrypt_round_rows" in tr else "k_encrypt_round_slots"
        rnd = tr[rk]["dram_bytes"] if side == 1920 else None
        if rnd is not None:
            per_frame = (ch["dram_bytes"] + ver["dram_bytes"]) / ch["iterations"] * iters_per_frame \
                + synth.ROUNDS * rnd
            frame_traffic = {"device_dram_bytes": per_frame, "algorithmic_bytes": alg_bytes,
                             "ratio": per_frame / alg_bytes,
                             "note": "cold-cache upper bound from profiles/traffic.json "
                                     "(chain + verify per frame's iterations + 5 rounds); "
                                     "keystream traffic (5F per frame) is implementation "
                                     "overhead by SURVEY 8(d) and is included here"}
    except (OSError, KeyError, ValueError, ZeroDivisionError, TypeError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling_of(G),
        "vs_baseline": None, "dtype": "f64/u8", "data": "synthetic",
        "config": config_dict(name, F, G),
        "gbps": value * fb / 1e9,
        "gbps_payload": value * c["width"] * c["height"] * 3 / 1e9,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": F * fb,
                "d2h_bytes_per_step": F * fb, "api": "cve_cipher_encrypt_frames (pinned)",
                "per_frame_calls": {"value": single_fps, "unit": "frames/s",
                                    "api": "cve_cipher_encrypt_frame per frame, pageable "
                                           "(the reference's call pattern)"}},
        "gpu_launches": launches,
        "roofline": {
            "bound": "hbm", "kernel": "k_prbg_chain_walk (dominant: %.0f%% of the step)"
            % (100 * chain_ms / ms if ms else 0),
            "achieved": chain_gbs, "peak": hbm, "unit": "GB/s",
            "frac": chain_gbs / hbm if chain_gbs else None, "peak_source": hbm_src,
            "traffic": traffic_per_launch,
            "traffic_note": "ncu dram__bytes_read+write of one k_prbg_chain_walk launch (cold), per "
                            "launch of this run; the chain writes one 8-byte checkpoint per lane "
                            "per 8 iterations (checkpoint_bytes_per_launch), which the verifier "
                            "reads back from L2",
            "checkpoint_bytes_per_launch": ckpt_per_launch,
            "frame_traffic": frame_traffic,
            "algorithmic_bytes_per_launch": alg_per_launch,
            "baseline_roofline_us_per_frame": baseline_roofline(side, hbm),
            "note": "BASELINE.json roofline: 2*side^2*3 B per frame (SURVEY 8(d)) at peak "
                    "HBM; the kernel is bound by the FP64 dependency latency of 2n "
                    "sequential orbits instead (see 'chain')"},
        "chain": {
            "kernel": "k_prbg_chain_walk (dominant: sequential FP64 orbit, latency-bound)",
            "ns_per_iteration": ns_iter, "iterations_per_lane": iters_timed,
            "cycles_per_iteration": ns_iter * (clk.summary()["sm_mhz"] or 1965.0) / 1e3,
            # ptxas stall counts of the unrolled 32-iteration loop body of the
            # folded step (SASS control bits, tools/iter_cycles.py build/csrc/prbg.o
            # k_prbg_chain_walk DMUL): 38 per step (the unfolded step: 40.6)
            "static_schedule_cycles": 38.0,
            "frac_of_static_schedule": 38.0 / (ns_iter * (clk.summary()["sm_mhz"] or 1965.0) / 1e3),
            "fp64_instructions_per_iteration": 7,
            "launches": int(len(chain_times)),
            "avg_launch_ms": float(np.mean(chain_times)) if len(chain_times) else None,
            "share_of_step": chain_ms / ms if ms else None,
            "verify_emit_fixup_ms": prbg_ms - chain_ms},
        "cipher": {"kernel": "k_encrypt_round_rows (K2r) x5 per frame",
                   "ms_per_frame": cipher_ms / frames_timed,
                   "achieved_gbs_2F": cipher_gbs,
                   "frac_of_hbm_2F": (cipher_gbs / hbm) if cipher_gbs else None,
                   # the cipher kernels alone vs HBM, counting what
                   # a round moves (frame read + keystream read + frame write)
                   "achieved_gbs_3F_per_round": (3 * synth.ROUNDS * fb * frames_timed /
                                                 (cipher_ms / 1e3) / 1e9) if cipher_ms else None,
                   "frac_of_hbm_3F_per_round": (3 * synth.ROUNDS * fb * frames_timed /
                                                (cipher_ms / 1e3) / 1e9 / hbm) if cipher_ms else None},
        "guard_replays": st1["guard_replays"],
        "multi_clip": multi,
        "decrypt": decrypt_line,
        "configs": per_config,
        "clocks": clk.summary(),
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_rows:
        line["rows"] = rows_measure(stream)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name, args.cpu_seconds)
    if dist.rank == 0:
        print(json.dumps(line))
    dist.close()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               "--master-port=29531", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
