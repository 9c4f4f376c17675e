"""Single-frame clip latency (config C1: one 480x480 frame): handle create +
encrypt_frame + destroy, wall clock, this engine vs the reference library."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Reference
for name in ("C1", "C4"):
    c = synth.CONFIGS[name]; n = c["workers"]
    key = synth.config_key(name)
    f0 = synth.config_frame(name, 0)
    cve.Cipher(key, n, 5).encrypt_frame(f0.copy())  # context warm-up
    for label, mk in (("b200", lambda: cve.Cipher(key, n, 5)), ("reference", lambda: Reference(key, n, 5, 1))):
        ts = []
        for rep in range(10):
            f = f0.copy()
            t0 = time.perf_counter()
            h = mk()
            t1 = time.perf_counter()
            if label == "b200":
                h.encrypt_frame(f)
            else:
                assert h.encrypt(f) == 0
            t2 = time.perf_counter()
            h.close()
            t3 = time.perf_counter()
            ts.append((t1 - t0, t2 - t1, t3 - t2))
        ts = np.median(np.array(ts) * 1e3, axis=0)
        print(f"{name} {label}: create {ts[0]:.2f} ms, first frame {ts[1]:.2f} ms, "
              f"destroy {ts[2]:.2f} ms, total {ts.sum():.2f} ms")
