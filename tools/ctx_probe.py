"""CUDA driver init and primary-context cost vs this library's first handle
(fresh process).  Tool."""
import ctypes, time, os, sys
t0=time.perf_counter()
cuda=ctypes.CDLL("libcuda.so.1")
t1=time.perf_counter()
print("cuInit", cuda.cuInit(0), f"{1e3*(time.perf_counter()-t1):.0f} ms")
dev=ctypes.c_int(); cuda.cuDeviceGet(ctypes.byref(dev),0)
ctx=ctypes.c_void_p()
t2=time.perf_counter()
r=cuda.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
print("primary ctx retain", r, f"{1e3*(time.perf_counter()-t2):.0f} ms")
sys.path.insert(0, os.getcwd())
t3=time.perf_counter()
import paper_2302_07411_b200 as cve
from workloads import synth
t4=time.perf_counter()
h=cve.Cipher(synth.config_key("C4"), 64, 5); h.close()
t5=time.perf_counter()
h=cve.Cipher(synth.config_key("C4"), 64, 5); h.close()
t6=time.perf_counter()
print(f"import {1e3*(t4-t3):.0f} ms, first handle {1e3*(t5-t4):.0f} ms, second {1e3*(t6-t5):.0f} ms")
