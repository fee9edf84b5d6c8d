"""Production K1 vs the dev harness's V23 (same chunk code, no ASCII vote) on
the same 1 GiB C1 buffer, alternated to rule out ordering effects."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib, configs

L = C.CDLL(str(ROOT / "tools" / "libkbench.so"))
L.kb_name.restype = C.c_char_p
L.kb_launch.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
idx = {L.kb_name(i).decode(): i for i in range(L.kb_count())}
pl = _lib.load()
n = 1 << 30
d = configs.gen_c1(n, seed=2)
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()


def t(fn, reps=100):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return n / (a.elapsed_time(b) / reps) / 1e6


prod = lambda: pl.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n + 3, flag.data_ptr(), st.cuda_stream)
v23 = lambda: L.kb_launch(idx["v23_u4_b4"], d.data_ptr(), n, flag.data_ptr(), st.cuda_stream)
import statistics
P, V = [], []
for r in range(30):
    P.append(t(prod, 20))
    V.append(t(v23, 20))
print(f"production median {statistics.median(P):.0f} (min {min(P):.0f} max {max(P):.0f})")
print(f"v23_u4_b4  median {statistics.median(V):.0f} (min {min(V):.0f} max {max(V):.0f})")
print("v23/production per round:", " ".join(f"{v / p:.3f}" for p, v in zip(P, V)))
