"""Small calls of every device entry point in one process (odd sizes and
alignments, malformed device offsets, stream pieces, sharded entry): a quick
end-to-end exercise of the whole C-ABI on a GPU box."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2010_03090_b200 as u8
from paper_2010_03090_b200 import _lib, configs

lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
flag = torch.zeros(1, dtype=torch.int32, device="cuda")

# K1 / K3: device and host, odd sizes and alignments, invalid tails.
d = configs.gen_c1(3 << 20, seed=2)
for off in (0, 1, 7, 31):
    n = d.numel() - off - 5
    lib.utf8v_cuda_validate_lanes_async(d.data_ptr() + off, n, 0, n + 3, flag.data_ptr(), st)
assert u8.validate_lookup(d)
bad = d.clone()
bad[123457] = 0xC0
v = u8.validate_lookup_verdict(bad)
assert not v.valid()
h = d[: (1 << 20) + 13].cpu().numpy()
assert u8.validate_lookup(h.tobytes())

# K2: C3-like batch, then malformed device offsets (must stay in bounds).
b = configs.gen_c3(n_records=3000, seed=4)
ver = u8.validate_lookup_batch(b.data, b.d_offsets)
assert (np.asarray(ver) == b.expected).all()
offs = b.d_offsets.clone()
offs[5] = offs[-1] + 1000        # non-monotonic and past the data
offs[-1] = offs[-1] + (1 << 20)  # last offset past the data
vv = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")
_lib.check(lib.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, offs.data_ptr(), b.n_records,
                                               vv.data_ptr(), st))
torch.cuda.synchronize()

# Streaming session with device pieces, and the sharded entry point.
with u8.LookupStream() as s:
    for a, z in ((0, 3), (3, 4), (4, 5000), (5000, 5001), (5001, d.numel())):
        s.feed(d[a:z])
    assert s.finish()
ok = C.c_uint8()
_lib.check(lib.utf8v_cuda_validate_sharded(h.ctypes.data, h.size, 3, 0, C.byref(ok)))
assert ok.value == 1
print("sanitize cases ok")

# Small-call server: host inputs <= 64 KiB (validate, verdict, lane ranges),
# including the idle exit and relaunch.
import time
for n in (1, 3, 31, 32, 33, 4097, 16384, 65536):
    raw = (b"ab\xc3\xa9\xe2\x82\xac" * (n // 7 + 1))[:n]
    hb = np.frombuffer(raw, np.uint8).copy()
    ok = C.c_uint8(9)
    _lib.check(lib.utf8v_cuda_validate(hb.ctypes.data, n, 0, C.byref(ok)))
    hb[n // 2] = 0xC0
    vok, off, kind = C.c_uint8(9), C.c_uint64(0), C.c_int(-1)
    _lib.check(lib.utf8v_cuda_validate_verdict(hb.ctypes.data, n, 0, C.byref(vok), C.byref(off), C.byref(kind)))
    assert vok.value == 0
    f = C.c_uint32(9)
    _lib.check(lib.utf8v_cuda_validate_lanes(hb.ctypes.data, n, n // 3, n + 3, 0, C.byref(f)))
    time.sleep(0.001)
print("sanitize cases done")
