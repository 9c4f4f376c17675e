"""Large-side parity check against the oracle (tool): sides above the
benchmark configs (4096 .. 8192), few and many subframes, encrypt through one
entry point and decrypt back through another."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Oracle

cases = [(4096, 1, 2), (4096, 256, 5), (5000, 8, 3), (6144, 512, 2), (8192, 64, 2), (7777, 7, 1),
         (4100, 1025, 2)]
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
bad = 0
NF = int(os.environ.get('LARGE_FRAMES', '2'))
for side, n, r in cases:
    key = synth.det_key(side + n)
    f = np.random.default_rng(side).integers(0, 256, size=(NF, side, side, 3), dtype=np.uint8)
    want = f.copy()
    t0 = time.time()
    o = Oracle(key, n, r)
    for t in range(NF):
        assert o.encrypt(want[t]) == 0
    o.close()
    t1 = time.time()
    got = f.copy()
    h = cve.Cipher(key, n, r)
    for t in range(NF):
        h.encrypt_frame(got[t])
    t2 = time.time()
    ok = np.array_equal(got, want)
    cve.Cipher(key, n, r).decrypt_frames(got)
    ok2 = np.array_equal(got, f)
    print(f"side={side} n={n} r={r}: enc={ok} dec={ok2}  oracle {t1 - t0:.1f}s  gpu {t2 - t1:.2f}s",
          flush=True)
    bad += not (ok and ok2)
print(f"{len(cases)} cases, {bad} failures")
sys.exit(1 if bad else 0)
