"""Decrypt path probe: CONFIG's clip, NF frames encrypted then decrypted on
one handle each from device memory (for ncu launch lists of the inverse
rounds: K3t / K3r / K3f by the environment switches).  Tool (not the bench)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_07411_b200 as cve
from workloads import synth

name = os.environ.get("CONFIG", "C4")
NF = int(os.environ.get("NF", "3"))
c = synth.CONFIGS[name]; n = c["workers"]; side = synth.config_side(name)
host = np.stack([synth.config_frame(name, t % 3) for t in range(NF)])
frames = torch.from_numpy(host.copy()).cuda()
st = torch.cuda.current_stream().cuda_stream
e = cve.Cipher(synth.config_key(name), n, 5)
e.encrypt_frames_device(frames.data_ptr(), side, NF, st)
d = cve.Cipher(synth.config_key(name), n, 5)
d.prefetch_keystream(NF * 5 * (side // n) * side * 3)
d.synchronize()
s0 = d.stats()
d.decrypt_frames_device(frames.data_ptr(), side, NF, st)
torch.cuda.synchronize()
s1 = d.stats()
ok = np.array_equal(frames.cpu().numpy(), host)
print(f"{name} decrypt {NF} frames: {(s1['cipher_ms'] - s0['cipher_ms']) / NF * 1e3:.1f} us/frame, round trip {'ok' if ok else 'MISMATCH'}")
