"""Short, fixed-size workload for ncu --set full captures of the LASM
generator (row f2): a C4-geometry LASM handle (n = 64, 128 lanes), one
generator launch of 16384 iterations (k_lasm_chain + k_lasm_emit), then one
C4 frame encrypted."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_07411_b200 as cve
from workloads import synth

name = "C4"; c = synth.CONFIGS[name]; side = synth.config_side(name); n = c["workers"]
key = synth.det_key_lasm(4242 + n)
h = cve.Cipher(key, n, 5)
h.prefetch_keystream(16384 * 12)
h.synchronize()
frame = torch.from_numpy(synth.config_frame(name, 0)[None].copy()).cuda()
h.encrypt_frames_device(frame.data_ptr(), side, 1, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", h.stats()["keystream_iters"])
