"""Randomised sweep of the round kernels against the oracle: random sides
(multiples of 16 up to 640), subframe counts dividing them, round counts and
keys (PLCM and LASM), 2 frames per handle encrypted and decrypted back.
Tool (a wider net than tests/test_round_kernels.py)."""
import os, sys, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Oracle

rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 60
maxside = int(sys.argv[3]) if len(sys.argv) > 3 else 640
bad = 0
# one handle across sides: the stream continues through frames of different
# geometries (ring growth), per-frame calls against one oracle handle
key = synth.det_key(4321)
for n in (1, 2, 4, 8, 16):
    o, h = Oracle(key, n, 5), cve.Cipher(key, n, 5)
    for t in range(6):
        side = 16 * n * rng.randint(1, max(1, maxside // (16 * n)))
        f = np.random.default_rng(t + 50 * n).integers(0, 256, size=(side, side, 3), dtype=np.uint8)
        a, b = f.copy(), f.copy()
        assert o.encrypt(a) == 0
        h.encrypt_frame(b)
        if not np.array_equal(a, b):
            bad += 1
            print(f"FAIL mixed-side handle n={n} frame {t} side={side}", flush=True)
for it in range(cases):
    side = 16 * rng.randint(1, maxside // 16)
    divs = [d for d in range(1, side + 1) if side % d == 0 and d <= 128]
    n = rng.choice(divs)
    r = rng.choice([1, 2, 3, 5, 5, 5, 7])
    lasm = rng.random() < 0.3
    key = synth.det_key_lasm(it + 1000) if lasm else synth.det_key(it + 1000)
    frames = np.random.default_rng(it).integers(0, 256, size=(2, side, side, 3), dtype=np.uint8)
    want = frames.copy()
    o = Oracle(key, n, r)
    for t in range(2):
        assert o.encrypt(want[t]) == 0
    got = frames.copy()
    devs = os.environ.get("SWEEP_DEVICES")  # e.g. "0,0,0": the sharded path on one GPU
    h = cve.Cipher(key, n, r, devices=[int(d) for d in devs.split(",")] if devs else None)
    for t in range(2):
        h.encrypt_frame(got[t])
    ok = np.array_equal(got, want)
    back = got.copy()
    cve.Cipher(key, n, r).decrypt_frames(back)
    ok2 = np.array_equal(back, frames)
    if not (ok and ok2):
        bad += 1
        print(f"FAIL side={side} n={n} r={r} lasm={lasm} enc={ok} dec={ok2}", flush=True)
print(f"{cases} cases, {bad} failures")
