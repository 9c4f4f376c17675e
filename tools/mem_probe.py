import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2302_07411_b200 as cve
from workloads import synth
torch.cuda.init(); torch.zeros(1).cuda()
for name in ["C1", "C4"]:
    c = synth.CONFIGS[name]; side = synth.config_side(name)
    f0, _ = torch.cuda.mem_get_info()
    hs = [cve.Cipher(synth.det_key(k), c["workers"], 5) for k in range(4)]
    fr = np.zeros((side, side, 3), np.uint8)
    for h in hs: h.encrypt_frame(fr.copy())
    torch.cuda.synchronize()
    f1, _ = torch.cuda.mem_get_info()
    print(name, f"{(f0 - f1) / 4 / 2**20:.0f} MiB device memory per handle after one frame")
    del hs
