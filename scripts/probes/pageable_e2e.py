"""Pageable-input e2e (utf8v_cuda_validate on 1 GiB of ordinary host memory),
library variants interleaved, best of 5 each."""
import ctypes as C
import os
import sys
import time

import numpy as np

libs = sys.argv[1:]
buf = np.full(1 << 30, ord("a"), np.uint8)
vs = [(p, C.CDLL(os.path.abspath(p))) for p in libs]
ok = C.c_uint8()
res = {p: [] for p in libs}
for p, v in vs:
    v.utf8v_cuda_validate(C.c_void_p(buf.ctypes.data), C.c_size_t(buf.size), 0, C.byref(ok))
for _ in range(5):
    for p, v in vs:
        t = time.perf_counter()
        v.utf8v_cuda_validate(C.c_void_p(buf.ctypes.data), C.c_size_t(buf.size), 0, C.byref(ok))
        res[p].append(time.perf_counter() - t)
for p, ts in res.items():
    print(f"{p}: {buf.size / min(ts) / 1e9:.1f} GB/s (valid={ok.value})", flush=True)
