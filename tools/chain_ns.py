import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2302_07411_b200 as cve
from workloads import synth
c = synth.CONFIGS["C4"]; side = synth.config_side("C4")
h = cve.Cipher(synth.config_key("C4"), c["workers"], 5)
fr = torch.zeros((24, side, side, 3), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
h.encrypt_frames_device(fr.data_ptr(), side, 4, st.cuda_stream); torch.cuda.synchronize()
s0 = h.stats()
h.encrypt_frames_device(fr.data_ptr(), side, 24, st.cuda_stream); torch.cuda.synchronize()
s1 = h.stats()
it = s1["keystream_iters"] - s0["keystream_iters"]
print(os.environ.get("TAG", ""), "chain ns/iter", (s1["chain_ms"] - s0["chain_ms"]) * 1e6 / it)
