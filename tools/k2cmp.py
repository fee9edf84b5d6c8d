"""DEVELOPMENT HARNESS: batch library variants on C3 (or C2: K2CMP=c2) timed like
bench.py's other_configs (back-to-back utf8v_cuda_validate_batch_async calls between
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
which = os.environ.get("K2CMP", "c3")
b = configs.gen_c3() if which == "c3" else configs.gen_c2()
copies = [b.data] + ([b.data.clone()] if which == "c2" else [])
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
        def run():
            for x in copies:
                v.utf8v_cuda_validate_batch_async(x.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),
                                                  b.n_records, ver.data_ptr(), st.cuda_stream)
        for _ in range(3):
            run()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(20):
            run()
        z.record(st)
        z.synchronize()
        times[name].append(a.elapsed_time(z) / 20 / len(copies))
        ok[name] = bool((ver.cpu().numpy() == b.expected).all())
alg = b.nbytes + 8 * (b.n_records + 1) + b.n_records
for name, ts in times.items():
    ms = sorted(ts)[len(ts) // 2]
    print(f"{which} {name}: {ms * 1e3:.1f} us  {alg / ms / 1e6:.0f} GB/s  {b.n_records / ms / 1e6:.3f} G rec/s "
          f"(min {min(ts) * 1e3:.1f})  verdicts_ok={ok[name]}", flush=True)
