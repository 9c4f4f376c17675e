"""Small-input latency of the file / analysis entry points (P6 images of a
few sizes), this engine vs the reference library, warm process.  Tool."""
import os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import ref_analyze, ref_encrypt_file, ref_decrypt_file
key = synth.config_key("C1")
d = tempfile.mkdtemp(dir="/dev/shm")
def p6(path, side, seed):
    img = np.random.Generator(np.random.PCG64(seed)).integers(0, 256, (side, side, 3), dtype=np.uint8)
    with open(path, "wb") as fh:
        fh.write(f"P6\n{side} {side}\n255\n".encode() + img.tobytes())
def med(fn, k=7):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))
for side in (64, 480, 1920):
    a, b = os.path.join(d, f"a{side}.ppm"), os.path.join(d, f"b{side}.ppm")
    p6(a, side, 1); p6(b, side, 2)
    o, r = os.path.join(d, "o.cve"), os.path.join(d, "r.cve")
    enc = med(lambda: cve.encrypt_file(key, a, o, workers=8, rounds=5))
    renc = med(lambda: ref_encrypt_file(key, a, r, workers=8, rounds=5))
    ana = med(lambda: cve.analyze(a, second=b, seed=1))
    rana = med(lambda: ref_analyze(a, second=b, seed=1))
    print(f"side {side}: encrypt_file ours {enc:.2f} ms ref {renc:.2f} ms | analyze ours {ana:.2f} ms ref {rana:.2f} ms")
