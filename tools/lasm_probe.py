"""LASM generator speed at the C1 and C4 geometries: frames/s of 8 host-API
frames after a warm-up, and the chain kernel's ns per iteration.  Tool."""
import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2302_07411_b200 as cve
from workloads import synth
for name in ("C1", "C4"):
    c = synth.CONFIGS[name]; side = synth.config_side(name); n = c["workers"]
    key = synth.det_key_lasm(4242 + n)
    ci = cve.Cipher(key, n, 5)
    fr = np.stack([synth.config_frame(name, t % 2) for t in range(8)])
    ci.encrypt_frames(fr[:2])
    t0 = time.time(); ci.encrypt_frames(fr); dt = time.time() - t0
    st = ci.stats()
    times = ci.take_prbg_times()
    iters = st['keystream_iters']
    print(name, "LASM frames/s", 8 / dt, "chain_ms", st['chain_ms'], "iters/lane", iters,
          "ns/iter", st['chain_ms'] * 1e6 / iters, flush=True)
