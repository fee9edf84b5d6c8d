"""K1 step size vs input size (L2 flushed before each launch): the harness's
V23 at 4 KiB steps / 4 CTAs vs 2 KiB steps / 5 CTAs, and production."""
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
st = torch.cuda.current_stream()
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
full = configs.gen_c1(256 << 20, seed=2)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        scratch.fill_(1)
        scratch.view(torch.int64).sum()
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / reps


for mib in (16, 64, 256):
    n = mib << 20
    d = full[:n]
    row = []
    for name in ("v23_u4_b4", "v23_u2_b5"):
        ms = timed(lambda: L.kb_launch(idx[name], d.data_ptr(), n, flag.data_ptr(), st.cuda_stream))
        row.append(f"{name} {n / ms / 1e6:6.0f}")
    ms = timed(lambda: pl.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n + 3, flag.data_ptr(), st.cuda_stream))
    row.append(f"production {n / ms / 1e6:6.0f}")
    print(f"{mib:4d} MiB: " + "  ".join(row), flush=True)
