"""cve_nist_export / cve_keystream_generate latency for small and large
requests, this engine vs the reference library.  Tool."""
import os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2302_07411_b200 as cve
from workloads import synth
from _oracle import Reference
key = synth.config_key("C4")
d = tempfile.mkdtemp(dir="/dev/shm")
cve.nist_export(key, 2, 1000, os.path.join(d, "w.bin"))  # warm-up
for workers, nbytes in ((2, 100_000), (8, 1_000_000), (64, 64 << 20)):
    t0 = time.perf_counter(); cve.nist_export(key, workers, nbytes, os.path.join(d, "o.bin")); t1 = time.perf_counter()
    assert Reference.load().cve_nist_export(key.encode(), workers, nbytes, os.path.join(d, "r.bin").encode()) == 0
    t2 = time.perf_counter()
    same = open(os.path.join(d, "o.bin"), "rb").read() == open(os.path.join(d, "r.bin"), "rb").read()
    print(f"nist_export workers={workers} bytes={nbytes}: ours {1e3*(t1-t0):.2f} ms, reference {1e3*(t2-t1):.2f} ms, identical={same}")
t0 = time.perf_counter(); cve.keystream_generate([0.3, 0.2, 0.7, 0.4], 48); t1 = time.perf_counter()
print(f"keystream_generate 48 B: {1e3*(t1-t0):.2f} ms")
