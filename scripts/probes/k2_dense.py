"""K2 on dense batches (many record starts per 4 KiB step): records/s and
verdict check against the generator's expectation."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_2010_03090_b200 import _lib, configs

lib = _lib.load()
st = torch.cuda.current_stream()
for median, n_rec in ((32, 16 << 20), (128, 4 << 20), (512, 1 << 20)):
    b = configs.gen_c3(n_records=n_rec, seed=7, sigma=0.5, median=median, min_len=16, max_len=4096)
    ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")

    def run():
        ver.fill_(1)
        _lib.check(lib.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),
                                                       b.n_records, ver.data_ptr(), st.cuda_stream))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ok = bool((ver.cpu().numpy() == b.expected).all())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"median {median:4d}: {b.n_records} records, {b.nbytes / 1e6:.0f} MB, {ms:.3f} ms, "
          f"{b.n_records / ms / 1e6:.2f} G records/s, {b.nbytes / ms / 1e6:.0f} GB/s, verdicts_ok={ok}", flush=True)
    del b, ver
    torch.cuda.empty_cache()
