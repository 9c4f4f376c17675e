"""Cipher-round kernels alone (K2/K3 + K4): keystream prefetched first, then
frames encrypted/decrypted from device memory; device time per frame from the
handle's CUDA events.  Tool (not the bench)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_07411_b200 as cve
from workloads import synth

for name in sys.argv[1:] or ["C1", "C3", "C4", "C5"]:
    c = synth.CONFIGS[name]; n = c["workers"]; side = synth.config_side(name)
    F = side * side * 3
    need = 5 * (side // n) * side * 3
    NF = 12 if side <= 1920 else 6
    frames = torch.from_numpy(np.stack([synth.config_frame(name, t % 3) for t in range(NF)])).cuda()
    out = {}
    for mode in ("enc", "dec"):
        best = None
        for rep in range(3):  # best of 3: the keystream is generated first, so
            h = cve.Cipher(synth.config_key(name), n, 5)  # only cipher time counts
            # normal ring (4 frames) unless CB_BIG_RING: the keystream of later
            # frames is generated on the fly, outside the timed cipher events
            h.prefetch_keystream((NF if os.environ.get("CB_BIG_RING") else 1) * need)
            h.synchronize()
            s0 = h.stats()
            fn = h.encrypt_frames_device if mode == "enc" else h.decrypt_frames_device
            fn(frames.data_ptr(), side, NF, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            s1 = h.stats()
            v = (s1["cipher_ms"] - s0["cipher_ms"]) / NF
            best = v if best is None else min(best, v)
            del h
        out[mode] = best
    print(f"{name}: side={side} n={n}  encrypt {out['enc']*1e3:.1f} us/frame "
          f"({2*F/out['enc']/1e6:.0f} GB/s of 2F, {15*F/out['enc']/1e6:.0f} GB/s moved)  "
          f"decrypt {out['dec']*1e3:.1f} us/frame")
