"""PROBE (development): K2's per-warp start/end on C3 (one launch after
back-to-back launches), from a -DU8V_TIMELINE build of batch.cu
(tools/kvar.sh batch.cu k2tl -DU8V_TIMELINE).
  python scripts/probes/k2_timeline.py build/var_k2tl/libutf8v_cuda.so"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2010_03090_b200 import _lib, configs  # noqa: E402

_lib.LIB_PATH = Path(sys.argv[1]).resolve()
lib = _lib.load()
lib.u8v_timeline_k2_set.argtypes = [C.c_void_p]
b = configs.gen_c3()
ver = torch.empty(b.n_records, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
tl = torch.zeros(3 * 8192, dtype=torch.int64, device="cuda")


def run():
    _lib.check(lib.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(),
                                                   b.n_records, ver.data_ptr(), st.cuda_stream))


for _ in range(5):
    run()
torch.cuda.synchronize()
lib.u8v_timeline_k2_set(tl.data_ptr())
for _ in range(3):
    run()
run()
torch.cuda.synchronize()
lib.u8v_timeline_k2_set(None)
a = tl.view(-1, 3).cpu().numpy()
a = a[a[:, 0] != 0]
s, e = a[:, 0].astype(float), a[:, 1].astype(float)
busy = (e - s) / 1e3
t0 = s.min()
print(json.dumps({"warps": int(a.shape[0]), "span_us": round((e.max() - t0) / 1e3, 2),
                  "busy_min_p10_p50_p90_max": [round(float(np.percentile(busy, q)), 1) for q in (0, 10, 50, 90, 100)],
                  "end_before_last_p10_p50_p90": [round(float(np.percentile((e.max() - e) / 1e3, q)), 1) for q in (10, 50, 90)],
                  "start_spread_max_us": round(float((s.max() - t0) / 1e3), 2)}))
w = np.arange(a.shape[0])
print("busy by warp-in-CTA (32):", [round(float(busy[(w % 32) == i].mean()), 1) for i in range(0, 32, 4)])
