"""DEVELOPMENT HARNESS: time (and, under ncu, profile) the batch kernel K2 on
C2 and C3 alone.  `python tools/k2bench.py [c2|c3|both] [reps]`."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib, configs

which = sys.argv[1] if len(sys.argv) > 1 else "both"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lib = _lib.load()
st = torch.cuda.current_stream()
scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, gen in (("c2", configs.gen_c2), ("c3", configs.gen_c3)):
    if which not in (name, "both"):
        continue
    b = gen()
    ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")

    def run():
        _lib.check(lib.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),
                                                       b.n_records, ver.data_ptr(), None, st.cuda_stream))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, z in ev:
        scratch.fill_(1)  # flush L2 (write, then read: no dirty lines left)
        scratch.view(torch.int64).sum()
        a.record(st)
        run()
        z.record(st)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(z) for a, z in ev) / reps
    ok = bool((ver.cpu().numpy() == b.expected).all())
    alg = b.nbytes + 8 * (b.n_records + 1) + b.n_records
    print(f"{name}: {ms:.3f} ms  {b.n_records / ms / 1e6:.3f} G records/s  {alg / ms / 1e6:.1f} GB/s  "
          f"verdicts_ok={ok}", flush=True)
    del b, ver
    torch.cuda.empty_cache()
