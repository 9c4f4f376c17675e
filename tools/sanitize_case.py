"""Small encrypt/decrypt round trips over the kernel families (slot K2s/K3s
with clusters, byte-staged K2/K3, generic path, f4 stats) for
compute-sanitizer runs.  Tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_07411_b200 as cve
from workloads import synth

shapes = [(64, 4, 2), (96, 8, 1), (90, 3, 1), (48, 3, 1), (160, 16, 1), (16, 1, 1)]
for side, n, r in shapes:
    key = synth.det_key(side + n)
    f = np.random.Generator(np.random.PCG64(side)).integers(0, 256, (2, side, side, 3), dtype=np.uint8)
    ct = f.copy()
    cve.Cipher(key, n, r).encrypt_frames(ct)
    pt = ct.copy()
    cve.Cipher(key, n, r).decrypt_frames(pt)
    assert np.array_equal(pt, f), (side, n, r)
    print("ok", side, n, r, flush=True)
import torch
a = torch.from_numpy(f[0]).cuda(); b = torch.from_numpy(f[1]).cuda()
h = torch.zeros(768, dtype=torch.int64, device="cuda"); d = torch.zeros(6, dtype=torch.int64, device="cuda")
cve.frame_stats_device(a.data_ptr(), f.shape[1], h.data_ptr(), b.data_ptr(), d.data_ptr(), 0)
torch.cuda.synchronize()
print("stats ok", int(h.sum()))
