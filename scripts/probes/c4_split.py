"""C4 (16 GiB) through K1 as one launch vs k launches over consecutive lane
ranges (back to back, PDL between K1 launches), device-timed."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib, configs

lib = _lib.load()
st = torch.cuda.current_stream()
n = 16 << 30
d, _ = configs.gen_c4(n, seed=4, variant=0)
flag = torch.zeros(1, dtype=torch.int32, device="cuda")


def run(k):
    step = n // k
    for i in range(k):
        lo, hi = i * step, (n + 3 if i == k - 1 else (i + 1) * step)
        _lib.check(lib.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, lo, hi, flag.data_ptr(), st.cuda_stream))


for k in (1, 2, 4, 8, 16, 64):
    for _ in range(2):
        run(k)
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record(st)
    for _ in range(reps):
        run(k)
    z.record(st)
    z.synchronize()
    ms = a.elapsed_time(z) / reps
    print(f"C4 16 GiB as {k:3d} launches: {ms:.3f} ms  {n / ms / 1e6:.0f} GB/s  flag={int(flag.item())}", flush=True)
