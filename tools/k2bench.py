"""DEVELOPMENT HARNESS: time (and, under ncu, profile) the batch kernel K2 on
C2 and C3 alone.  `python tools/k2bench.py [c2|c3|both] [reps] [lib.so ...]`
(several library variants from tools/kvar.sh: timed interleaved, medians)."""
import os
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2010_03090_b200 import _lib, configs

which = sys.argv[1] if len(sys.argv) > 1 else "both"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
libs = sys.argv[3:] or [str(_lib.LIB_PATH)]
if len(libs) > 1 or libs[0] != str(_lib.LIB_PATH):
    _lib.LIB_PATH = Path(libs[0])
lib = _lib.load()
variants = []
for path in libs:
    v = C.CDLL(os.path.abspath(path))
    v.utf8v_cuda_validate_batch_async.argtypes = _lib.SIGNATURES["utf8v_cuda_validate_batch_async"][1]
    variants.append((Path(path).parent.name, v))
st = torch.cuda.current_stream()
scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def gen_c3_valid():
    """C3's record lengths over the valid C1 mix, cuts moved to character
    boundaries: every record valid (the mostly-valid case)."""
    import numpy as np
    offs = configs.c3_offsets(configs.C3["n_records"], configs.C3["seed"], configs.C3["sigma"],
                              configs.C3["median"], configs.C3["min_len"], configs.C3["max_len"])
    n = int(offs[-1])
    d = configs.gen_c1(n, seed=2)  # exactly n bytes, valid as a whole
    h = d.cpu().numpy()
    o = offs.astype(np.int64)
    for _ in range(3):
        inside = (o < n) & ((h[np.minimum(o, n - 1)] & 0xC0) == 0x80)
        o[inside] += 1
    o = np.maximum.accumulate(np.minimum(o, n))
    o[0], o[-1] = 0, n
    offs = o.astype(np.uint64)
    return configs.Batch(d, offs, torch.from_numpy(o).cuda(), np.ones(offs.size - 1, np.uint8))


for name, gen in (("c2", configs.gen_c2), ("c3", configs.gen_c3), ("c3v", gen_c3_valid)):
    if which not in (name, "both") and not (which == "all"):
        continue
    b = gen()
    ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")

    def run(v):
        ver.fill_(1)
        _lib.check(v.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),
                                                     b.n_records, ver.data_ptr(), st.cuda_stream))

    for _, v in variants:
        for _ in range(3):
            run(v)
    torch.cuda.synchronize()
    times = {vn: [] for vn, _ in variants}
    oks = {}
    for _ in range(reps):
        for vn, v in variants:
            scratch.fill_(1)  # flush L2 (write, then read: no dirty lines left)
            scratch.view(torch.int64).sum()
            ver.fill_(1)
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            _lib.check(v.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),
                                                         b.n_records, ver.data_ptr(), st.cuda_stream))
            z.record(st)
            z.synchronize()
            times[vn].append(a.elapsed_time(z))
            got = ver.cpu().numpy()
            oks[vn] = bool((got == b.expected).all()) or f"{int((got != b.expected).sum())} differ at {np.nonzero(got != b.expected)[0][:3]}"
    # K1 on the same bytes as one stream (the sweep's own ceiling at this size)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    k1 = []
    for _ in range(reps):
        scratch.fill_(1)
        scratch.view(torch.int64).sum()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _lib.check(lib.utf8v_cuda_validate_lanes_async(b.data.data_ptr(), b.nbytes, 0, b.nbytes + 3,
                                                       flag.data_ptr(), st.cuda_stream))
        z.record(st)
        z.synchronize()
        k1.append(a.elapsed_time(z))
    times["K1-same-bytes"] = k1
    oks["K1-same-bytes"] = None
    alg = b.nbytes + 8 * (b.n_records + 1) + b.n_records
    for vn, ts in times.items():
        ms = sorted(ts)[len(ts) // 2]
        print(f"{name} {vn}: {ms:.3f} ms  {b.n_records / ms / 1e6:.3f} G records/s  {alg / ms / 1e6:.1f} GB/s  "
              f"verdicts_ok={oks[vn]}", flush=True)
    del b, ver
    torch.cuda.empty_cache()
