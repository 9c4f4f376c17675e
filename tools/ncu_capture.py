"""Short, fixed-size workload for ncu --set full captures: one C4 generator
launch of exactly 131072 iterations (k_prbg_chain_start + k_prbg_chain_walk + k_prbg_verify_emit), then
one C4 frame encrypted and decrypted (k_encrypt_round / k_decrypt_round)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_07411_b200 as cve
from workloads import synth

name = "C4"; c = synth.CONFIGS[name]; side = synth.config_side(name); n = c["workers"]
h = cve.Cipher(synth.config_key(name), n, 5)
h.prefetch_keystream(131072 * 6)
h.synchronize()
frame = torch.from_numpy(synth.config_frame(name, 0)[None].copy()).cuda()
h.encrypt_frames_device(frame.data_ptr(), side, 1, torch.cuda.current_stream().cuda_stream)
d = cve.Cipher(synth.config_key(name), n, 5)
d.decrypt_frames_device(frame.data_ptr(), side, 1, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", h.stats()["keystream_iters"])
