import os, sys, time, subprocess, ctypes as C
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2009_06693_b200 import _lib
from paper_2009_06693_b200.graph import DeviceGraph
path = "/tmp/e69.txt"
subprocess.check_call("tools/gen_edgelist 22 69000000 > /tmp/e69.txt", shell=True)
L = _lib.load(); torch.cuda.init(); torch.zeros(1, device="cuda")
for it in range(2):
    t0 = time.perf_counter(); data = open(path, "rb").read(); t1 = time.perf_counter()
    t2 = time.perf_counter()
    info = (C.c_int64 * 4)(); t = C.c_void_p()
    _lib.check(L.nd_text_parse(data, len(data), 1, 1.0, 5.0, C.c_uint64(0), _lib.stream_ptr(), C.byref(t), info)); t3 = time.perf_counter()
    h = C.c_void_p(); nv = C.c_int64()
    _lib.check(L.nd_text_finish(t, None, None, None, None, None, 0, 0, _lib.stream_ptr(), C.byref(h), C.byref(nv))); torch.cuda.synchronize(); t4 = time.perf_counter()
    remap = np.empty(nv.value, dtype=np.int64); L.nd_text_remap(t, _lib.ptr(remap)); L.nd_text_destroy(t); t5 = time.perf_counter()
    print(f"read {t1-t0:.3f}  asciichk {t2-t1:.3f}  parse {t3-t2:.3f}  finish {t4-t3:.3f}  remap {t5-t4:.3f}", list(info))
    L.nd_graph_destroy(h)
