"""M independent clips (config $CONFIG, default C4) on one GPU through the
device-resident API, each on its own stream, one hardware queue per handle
(cve_set_streams_per_handle(1)): aggregate frames/s.  Tool (bench.py reports
a labelled multi-clip line from the same code)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_07411_b200 as cve
from workloads import synth

name = os.environ.get("CONFIG", "C4"); c = synth.CONFIGS[name]; side = synth.config_side(name); n = c["workers"]
F = 8
pool = np.stack([synth.config_frame(name, 2 + t) for t in range(F)])
for M in [int(a) for a in sys.argv[1:]] or [1, 4, 16, 32, 64]:
    bufs = [torch.from_numpy(pool).cuda() for _ in range(M)]
    streams = [torch.cuda.Stream() for _ in range(M)]
    cve.set_streams_per_handle(1)
    hs = [cve.Cipher(synth.det_key(500 + k), n, 5) for k in range(M)]
    cve.set_streams_per_handle(2)
    for h, b, s in zip(hs, bufs, streams):   # warm-up step
        h.encrypt_frames_device(b.data_ptr(), side, F, s.cuda_stream)
    torch.cuda.synchronize()
    steps = 3
    t0 = time.perf_counter()
    for _ in range(steps):
        for h, b, s in zip(hs, bufs, streams):
            h.encrypt_frames_device(b.data_ptr(), side, F, s.cuda_stream)
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    fps = M * F * steps / el
    st = [h.stats() for h in hs]
    print(f"M={M:3d}: {fps:8.1f} frames/s aggregate ({fps/M:6.1f} per clip), "
          f"cipher {np.mean([s['cipher_ms'] for s in st])/(F*(steps+1)):.3f} ms/frame, "
          f"host enqueue {host/el*100:.0f}% of wall ({host/(M*F*steps)*1e6:.0f} us/frame)", flush=True)
    del hs, bufs
    torch.cuda.empty_cache()
