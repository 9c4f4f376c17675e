"""Quick GPU probe: keystream-generator latency per iteration and cipher
time per frame for a config (not the bench; see bench.py)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth

for name in sys.argv[1:] or ["C1", "C4"]:
    c = synth.CONFIGS[name]
    n = c["workers"]
    side = synth.config_side(name)
    h = cve.Cipher(synth.config_key(name), n, 5)
    need = 5 * (side // n) * side * 3
    h.prefetch_keystream(need)          # one launch-ish
    h.synchronize()
    h.take_prbg_times()
    st0 = h.stats()
    t = time.time()
    h.prefetch_keystream(3 * need)
    h.synchronize()
    wall = time.time() - t
    times = h.take_prbg_times()
    st1 = h.stats()
    iters = st1["keystream_iters"] - st0["keystream_iters"]
    ms = float(times.sum())
    print(f"{name}: n={n} side={side} prbg launches={len(times)} iters/lane={iters} "
          f"dev {ms:.3f} ms wall {wall*1e3:.1f} ms -> {ms*1e6/iters:.2f} ns/iter "
          f"replays={st1['guard_replays']}")
    frames = np.stack([synth.config_frame(name, t) for t in range(4)])
    h2 = cve.Cipher(synth.config_key(name), n, 5)
    h2.encrypt_frames(frames[:1])
    s0 = h2.stats()
    t = time.time()
    h2.encrypt_frames(frames)
    wall = time.time() - t
    s1 = h2.stats()
    print(f"   4 frames host API: wall {wall*1e3:.1f} ms ({wall*250:.2f} ms/frame), cipher dev "
          f"{(s1['cipher_ms']-s0['cipher_ms'])/4:.3f} ms/frame, prbg dev "
          f"{(s1['prbg_ms']-s0['prbg_ms'])/4:.3f} ms/frame")
