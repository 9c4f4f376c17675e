"""Row f1 file pipelines on a raw 1920x1080 clip: repeated runs of
cve_encrypt_file / cve_decrypt_file with the plain write/read cost of the same
bytes for scale.  Tool."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth

c = synth.CONFIGS["C4"]; W, H, n = c["width"], c["height"], c["workers"]
key = synth.config_key("C4"); nf = int(sys.argv[1]) if len(sys.argv) > 1 else 48
d = tempfile.mkdtemp(dir=os.environ.get("FB_DIR"))
raw = os.path.join(d, "clip.rgb")
pool = [synth.correlated_frame(W, H, t, 7104) for t in range(4)]
with open(raw, "wb") as fh:
    for t in range(nf):
        fh.write(pool[t % 4].tobytes())
sq = (max(W, H) + n - 1) // n * n
blob = os.urandom(1 << 20) * (nf * sq * sq * 3 >> 20)
for rep in range(3):
    out, back = os.path.join(d, f"o{rep}.cve"), os.path.join(d, f"b{rep}.rgb")
    t0 = time.perf_counter(); cve.encrypt_file(key, raw, out, workers=n, rounds=5, raw=(W, H)); te = time.perf_counter() - t0
    t0 = time.perf_counter(); cve.decrypt_file(key, out, back, fmt=cve.CVE_OUT_RAW); td = time.perf_counter() - t0
    t0 = time.perf_counter()
    with open(os.path.join(d, f"w{rep}"), "wb") as fh:
        fh.write(blob)
    tw = time.perf_counter() - t0
    print(f"rep {rep}: encrypt_file {nf/te:6.1f} fps ({te*1e3:.0f} ms)  decrypt_file {nf/td:6.1f} fps "
          f"({td*1e3:.0f} ms)  plain write of the container bytes {tw*1e3:.0f} ms", flush=True)
    for p in (out, back, os.path.join(d, f"w{rep}")):
        os.remove(p)
