"""Device time of the PLCM verify/emit + fix-up kernels per generator
iteration at C4 (128 lanes): 8 device-resident frames, stats before/after."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_07411_b200 as cve
from workloads import synth
c = synth.CONFIGS["C4"]
side = synth.config_side("C4")
h = cve.Cipher(synth.config_key("C4"), c["workers"], 5)
fr = torch.zeros((8, side, side, 3), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
h.encrypt_frames_device(fr.data_ptr(), side, 2, st.cuda_stream)
torch.cuda.synchronize()
s0 = h.stats()
h.encrypt_frames_device(fr.data_ptr(), side, 8, st.cuda_stream)
torch.cuda.synchronize()
s1 = h.stats()
it = s1["keystream_iters"] - s0["keystream_iters"]
ver = (s1["prbg_ms"] - s1["chain_ms"]) - (s0["prbg_ms"] - s0["chain_ms"])
nl = s1["prbg_launches"] - s0["prbg_launches"]
print(f"{os.environ.get('TAG','')} iters {it} launches {nl} verify+fixup {ver:.3f} ms -> "
      f"{ver*1e6/max(it,1):.2f} ns/iter ({ver*1e3/max(nl,1):.1f} us/launch)")
