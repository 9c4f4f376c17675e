"""LASM keys at small subframe counts: frames/s of a C1-geometry (480^2,
n=8) and C2-geometry (576^2, n=16) clip, this engine vs the reference
library on the host cores.  Tool."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Reference
for name in ("C1", "C2", "C3", "C4"):
    c = synth.CONFIGS[name]; n = c["workers"]; side = synth.config_side(name)
    key = synth.det_key_lasm(4242 + n)
    frames = np.stack([synth.config_frame(name, t % 3) for t in range(12)])
    h = cve.Cipher(key, n, 5)
    f = frames.copy(); h.encrypt_frames(f[:2])
    t0 = time.perf_counter(); h.encrypt_frames(f[2:]); ours = 10 / (time.perf_counter() - t0)
    r = Reference(key, n, 5, 1)
    g = frames.copy()
    for i in range(2): r.encrypt(g[i])
    t0 = time.perf_counter()
    for i in range(2, 12): r.encrypt(g[i])
    ref = 10 / (time.perf_counter() - t0)
    print(f"{name} LASM n={n}: ours {ours:.1f} frames/s, reference {ref:.1f} frames/s "
          f"({os.cpu_count()} cpus), identical={np.array_equal(f, g)}")
