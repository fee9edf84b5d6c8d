"""DEVELOPMENT: is a pooled K2 worth building?  K1 over C3's bytes (the pooled
sweep) against the U8V_K2P_SKELETON variants of it, which add a pooled K2's
memory traffic per step (the step table entry; the step's record starts;
level 2: the 8 bytes around each start), and against K2 itself.  Back to
back over the same bytes and one call after an L2 flush.
`python scripts/probes/k2p_skeleton.py base.so var1.so var2.so`"""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2010_03090_b200 import _lib, configs

libs = sys.argv[1:]
_lib.LIB_PATH = Path(libs[0]).resolve()
base = _lib.load()
b = configs.gen_c3()
n = b.nbytes
assert b.data.data_ptr() % 32 == 0
offs = b.offsets.astype(np.uint64)
steps = (n + 3 + 4095) // 4096 + 1
table = np.searchsorted(offs, np.arange(steps + 1, dtype=np.uint64) * 4096, side="left").astype(np.uint32)
d_table = torch.from_numpy(table.view(np.int32)).cuda()
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
vs = []
for p in libs:
    v = C.CDLL(os.path.abspath(p))
    if hasattr(v, "u8v_k2p_set"):
        v.u8v_k2p_set(C.c_void_p(d_table.data_ptr()), C.c_void_p(b.d_offsets.data_ptr()), C.c_uint(b.n_records))
    vs.append((Path(p).parent.name, v))


def k1(v):
    v.utf8v_cuda_validate_lanes_async(C.c_void_p(b.data.data_ptr()), C.c_uint64(n), C.c_uint64(0),
                                      C.c_uint64(n + 3), C.c_void_p(flag.data_ptr()), C.c_void_p(st.cuda_stream))


def k2(v):
    v.utf8v_cuda_validate_batch_async(C.c_void_p(b.data.data_ptr()), C.c_uint64(n),
                                      C.c_void_p(b.d_offsets.data_ptr()), C.c_uint64(b.n_records),
                                      C.c_void_p(ver.data_ptr()), C.c_void_p(st.cuda_stream))


runs = [(f"K1 {name}", v, k1) for name, v in vs] + [("K2 (batch call)", vs[0][1], k2)]
for label, v, fn in runs * 2:
    for _ in range(3):
        fn(v)
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(30):
        fn(v)
    z.record(st)
    z.synchronize()
    btb = a.elapsed_time(z) / 30 * 1e3
    fl = []
    for _ in range(10):
        scratch.fill_(1)
        scratch.view(torch.int64).sum()
        a.record(st)
        fn(v)
        z.record(st)
        z.synchronize()
        fl.append(a.elapsed_time(z) * 1e3)
    print(f"{label:28s} back to back {btb:6.1f} us   flushed {sorted(fl)[5]:6.1f} us   flag={int(flag.item())}",
          flush=True)
