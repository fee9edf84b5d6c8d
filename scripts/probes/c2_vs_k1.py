"""C2 back to back over two rotating 256 MiB copies: the batch call (init +
K2L) against K1 alone on the same bytes (the sweep's own ceiling)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib, configs

lib = _lib.load()
st = torch.cuda.current_stream()
b = configs.gen_c2()
copies = [b.data, b.data.clone()]
ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")


def batch():
    for x in copies:
        lib.utf8v_cuda_validate_batch_async(x.data_ptr(), b.nbytes, b.d_offsets.data_ptr(), b.n_records,
                                            ver.data_ptr(), st.cuda_stream)


def k1():
    for x in copies:
        lib.utf8v_cuda_validate_lanes_async(x.data_ptr(), b.nbytes, 0, b.nbytes + 3, flag.data_ptr(), st.cuda_stream)


for name, fn in (("batch (init + K2L)", batch), ("K1 alone", k1)) * 2:
    for _ in range(3):
        fn()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(50):
        fn()
    z.record(st)
    z.synchronize()
    us = a.elapsed_time(z) / 100 * 1e3
    print(f"C2 {name}: {us:.1f} us per 256 MiB, {b.nbytes / us / 1e3:.0f} GB/s", flush=True)
