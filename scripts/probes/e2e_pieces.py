"""e2e of utf8v_cuda_validate on 1 GiB of pinned host memory (wall clock) for
library variants with different H2D piece sizes, against one plain pinned
cudaMemcpy of the same bytes."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib, configs

libs = sys.argv[1:]
d = configs.gen_c1(1 << 30, seed=2)
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
h.copy_(d)
dst = torch.empty_like(d)
vs = []
for path in libs:
    v = C.CDLL(os.path.abspath(path))
    v.utf8v_cuda_validate.argtypes = _lib.SIGNATURES["utf8v_cuda_validate"][1]
    vs.append((path, v))
ok = C.c_uint8()
res = {p: [] for p, _ in vs}
res["memcpy"] = []
for _ in range(8):
    for p, v in vs:
        torch.cuda.synchronize()
        t = time.perf_counter()
        assert v.utf8v_cuda_validate(h.data_ptr(), h.numel(), 0, C.byref(ok)) == 0 and ok.value == 1
        res[p].append(time.perf_counter() - t)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dst.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    res["memcpy"].append(time.perf_counter() - t)
for p, ts in res.items():
    ts = sorted(ts)[1:-1]
    print(f"{p}: {h.numel() / (sum(ts) / len(ts)) / 1e9:.2f} GB/s", flush=True)
