"""DEVELOPMENT HARNESS: batch library variants on C3 timed like bench.py's
other_configs.c3 (back-to-back utf8v_cuda_validate_batch_async calls between
two events), interleaved rounds, medians.  `python tools/k2cmp.py rounds lib.so ...`"""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2010_03090_b200 import _lib, configs

rounds = int(sys.argv[1])
libs = sys.argv[2:]
_lib.LIB_PATH = Path(libs[0]).resolve()
_lib.load()
st = torch.cuda.current_stream()
b = configs.gen_c3()
ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")
vs = []
for path in libs:
    v = C.CDLL(os.path.abspath(path))
    v.utf8v_cuda_validate_batch_async.argtypes = _lib.SIGNATURES["utf8v_cuda_validate_batch_async"][1]
    vs.append((Path(path).parent.name, v))
times = {k: [] for k, _ in vs}
ok = {}
for _ in range(rounds):
    for name, v in vs:
        run = lambda: v.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),  # noqa
                                                        b.n_records, ver.data_ptr(), st.cuda_stream)
        for _ in range(3):
            run()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(20):
            run()
        z.record(st)
        z.synchronize()
        times[name].append(a.elapsed_time(z) / 20)
        ok[name] = bool((ver.cpu().numpy() == b.expected).all())
alg = b.nbytes + 8 * (b.n_records + 1) + b.n_records
for name, ts in times.items():
    ms = sorted(ts)[len(ts) // 2]
    print(f"C3 {name}: {ms * 1e3:.1f} us  {alg / ms / 1e6:.0f} GB/s  {b.n_records / ms / 1e6:.3f} G rec/s "
          f"(min {min(ts) * 1e3:.1f})  verdicts_ok={ok[name]}", flush=True)
