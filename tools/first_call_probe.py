"""First-call costs in a fresh process: CUDA context + module load (first
handle), then the first and second cve_encrypt_file of a 24-frame raw 1080p
clip (pinned staging is allocated on the first).  Tool."""
import os, sys, tempfile, time
t0 = time.perf_counter()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_07411_b200 as cve
from workloads import synth
t1 = time.perf_counter()
c = synth.CONFIGS["C4"]; W, H, n = c["width"], c["height"], c["workers"]
key = synth.config_key("C4")
d = tempfile.mkdtemp(dir="/dev/shm")
raw = os.path.join(d, "clip.rgb")
pool = [synth.correlated_frame(W, H, t, 7104) for t in range(2)]
with open(raw, "wb") as fh:
    for t in range(24):
        fh.write(pool[t % 2].tobytes())
t2 = time.perf_counter()
h = cve.Cipher(key, n, 5)
h.close()
t3 = time.perf_counter()
out = os.path.join(d, "c.cve")
cve.encrypt_file(key, raw, out, workers=n, rounds=5, raw=(W, H))
t4 = time.perf_counter()
cve.encrypt_file(key, raw, out, workers=n, rounds=5, raw=(W, H))
t5 = time.perf_counter()
print(f"import {1e3*(t1-t0):.0f} ms, first handle (context + modules) {1e3*(t3-t2):.0f} ms, "
      f"first encrypt_file {1e3*(t4-t3):.0f} ms, second {1e3*(t5-t4):.0f} ms")
