"""Device analysis reductions (cve_frame_stats_device) on C4 frames: histogram
only, NPCR/UACI only, both; 8 frame pairs cycled (> L2).  Tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_07411_b200 as cve
from workloads import synth

side = synth.config_side("C4"); fb = side * side * 3; P = 8
a = torch.from_numpy(np.stack([synth.config_frame("C4", 2 + t) for t in range(4)])).repeat(2, 1, 1, 1).contiguous().cuda()
b = torch.roll(a, 1, dims=0).contiguous()
hist = torch.zeros(768, dtype=torch.int64, device="cuda"); diff = torch.zeros(6, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for name, h, d in [("hist only", True, False), ("diff only", False, True), ("both", True, True)]:
    def call(i):
        cve.frame_stats_device(a.data_ptr() + (i % P) * fb, side, hist.data_ptr() if h else 0,
                               b.data_ptr() + (i % P) * fb if d else 0, diff.data_ptr() if d else 0, s.cuda_stream)
    for i in range(P): call(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for i in range(48): call(i)
    e1.record(s); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 48
    nb = fb * ((1 if h or d else 0) + (1 if d else 0))
    print(f"{name:10s} {us:7.1f} us  {nb / us / 1e3:7.0f} GB/s")
