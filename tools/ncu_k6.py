"""One C1 frame and one C3 frame through the cipher (K6 cluster kernel for
encryption at these sizes) -- a short workload for ncu captures.  Tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_07411_b200 as cve
from workloads import synth

for name in sys.argv[1:] or ["C1"]:
    c = synth.CONFIGS[name]; side = synth.config_side(name); n = c["workers"]
    h = cve.Cipher(synth.config_key(name), n, 5)
    h.prefetch_keystream(5 * (side // n) * side * 3)
    h.synchronize()
    f = torch.from_numpy(synth.config_frame(name, 0)[None].copy()).cuda()
    h.encrypt_frames_device(f.data_ptr(), side, 1, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
print("ok")
