"""DEVELOPMENT HARNESS: K1 library variants (tools/kvar.sh builds) on the
1 GiB C1 stream, timed like bench.py's headline: `batch` back-to-back
launches between two CUDA events (launches of one variant may overlap
through PDL), variants interleaved, medians over rounds.
`python tools/k1bench.py rounds lib.so [lib.so ...]` (env K1_GIB: stream GiB)."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib, configs

rounds = int(sys.argv[1])
libs = sys.argv[2:]
_lib.LIB_PATH = Path(libs[0]).resolve()
_lib.load()
st = torch.cuda.current_stream()
n = int(float(os.environ.get("K1_GIB", "1")) * (1 << 30))
d = configs.gen_c1(n)
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
batch = 50
vs = []
for path in libs:
    v = C.CDLL(os.path.abspath(path))
    v.utf8v_cuda_validate_lanes_async.argtypes = _lib.SIGNATURES["utf8v_cuda_validate_lanes_async"][1]
    vs.append((Path(path).parent.name, v))
times = {k: [] for k, _ in vs}
for _ in range(rounds):
    for name, v in vs:
        for _ in range(3):
            v.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n + 3, flag.data_ptr(), st.cuda_stream)
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(batch):
            v.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n + 3, flag.data_ptr(), st.cuda_stream)
        z.record(st)
        z.synchronize()
        times[name].append(a.elapsed_time(z) / batch)
assert int(flag.item()) == 0
for name, ts in times.items():
    ms = sorted(ts)[len(ts) // 2]
    print(f"K1 {name}: {ms * 1e3:.1f} us  {n / ms / 1e6:.0f} GB/s  (min {min(ts) * 1e3:.1f})", flush=True)
