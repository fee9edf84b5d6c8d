"""PROBE (development): where K1's fixed per-launch cost goes.

  python scripts/probes/k1_timeline.py build/var_tl/libutf8v_cuda.so

The library variant is built with -DU8V_TIMELINE (tools/kvar.sh validate.cu tl
-DU8V_TIMELINE): every warp of k_validate writes its %globaltimer start/end
and SM id.  Prints, for C1 (1 GiB, back-to-back launches) and C0 (64 MiB, L2
flushed / four rotating buffers), the event-timed launch, the span from the
first warp's start to the last warp's end, and the ramp (start spread) and
drain (end spread) across warps; then the cold-code test: K1 on 4 KiB right
after an L2 flush, launched twice back to back, each launch event-timed.
"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2010_03090_b200 import _lib, configs  # noqa: E402

lib = C.CDLL(str(Path(sys.argv[1]).resolve()))
_lib.LIB_PATH = Path(sys.argv[1]).resolve()
_lib.load()
lib.utf8v_cuda_validate_lanes_async.argtypes = _lib.SIGNATURES["utf8v_cuda_validate_lanes_async"][1]
lib.u8v_timeline_set.argtypes = [C.c_void_p]
st = torch.cuda.current_stream()
sp = st.cuda_stream
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tl = torch.zeros(3 * 8192, dtype=torch.int64, device="cuda")
out = {}
raw = {}
tag = Path(sys.argv[1]).parent.name


def k1(buf, n=None):
    n = buf.numel() if n is None else n
    assert lib.utf8v_cuda_validate_lanes_async(buf.data_ptr(), n, 0, n + 3, flag.data_ptr(), sp) == 0


def flush():
    scratch.fill_(1)
    scratch.view(torch.int64).sum()


def ev_time(fns):
    """Event time of each fn in fns, launched back to back on the stream."""
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)]
    evs[0].record(st)
    for i, f in enumerate(fns):
        f()
        evs[i + 1].record(st)
    torch.cuda.synchronize()
    return [evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(len(fns))]


def timeline_of(fn_before, fn, label):
    tl.zero_()
    fn_before()
    lib.u8v_timeline_set(tl.data_ptr())
    t = ev_time([fn])[0]
    lib.u8v_timeline_set(None)
    a = tl.view(-1, 3).cpu().numpy()
    a = a[a[:, 0] != 0]
    s, e = a[:, 0].astype(np.float64), a[:, 1].astype(np.float64)
    t0 = s.min()
    busy = e - s
    r = {"event_us": round(t, 2), "warps": int(a.shape[0]), "span_us": round((e.max() - t0) / 1e3, 2),
         "start_spread_us_p50_p99_max": [round(float(np.percentile(s - t0, q)) / 1e3, 2) for q in (50, 99, 100)],
         "end_before_last_us_p1_p50": [round(float(np.percentile(e.max() - e, q)) / 1e3, 2) for q in (1, 50)],
         "end_spread_us": round(float(e.max() - e.min()) / 1e3, 2),
         "busy_us_min_mean_max": [round(float(x) / 1e3, 2) for x in (busy.min(), busy.mean(), busy.max())],
         "sms": int(len(set(a[:, 2].tolist())))}
    # ends per die half (SM ids < 74 vs >= 74) -- die locality of the drain
    sm = a[:, 2]
    for name, m in (("sm_lo_half", sm < 74), ("sm_hi_half", sm >= 74)):
        if m.any():
            r[name + "_mean_end_before_last_us"] = round(float((e.max() - e[m]).mean()) / 1e3, 2)
    out[label] = r
    raw[label] = a
    print(label, json.dumps(r), flush=True)


c1 = configs.gen_c1()
for _ in range(5):
    k1(c1)
torch.cuda.synchronize()
ts = ev_time([lambda: k1(c1)] * 20)
out["c1_back_to_back_us"] = [round(x, 2) for x in sorted(ts)]
print("c1 back-to-back event us", out["c1_back_to_back_us"], flush=True)
timeline_of(lambda: [k1(c1) for _ in range(3)], lambda: k1(c1), "c1_after_k1")
timeline_of(lambda: None, lambda: k1(c1), "c1_after_sync")
del c1

c0 = configs.gen_c0()
rot = [c0] + [c0.clone() for _ in range(3)]
torch.cuda.synchronize()
timeline_of(flush, lambda: k1(c0), "c0_flushed")
ts = ev_time([(lambda b=b: k1(b)) for _ in range(10) for b in rot])
out["c0_rotating4_us"] = [round(x, 2) for x in sorted(ts)]
print("c0 rotating 4 buffers, event us", out["c0_rotating4_us"], flush=True)
ts = ev_time([lambda: k1(c0)] * 20)
out["c0_same_buffer_us"] = [round(x, 2) for x in sorted(ts)]
print("c0 same buffer (L2-warm), event us", out["c0_same_buffer_us"], flush=True)
timeline_of(lambda: [k1(b) for b in rot[1:]], lambda: k1(c0), "c0_after_rotation")

# cold code: flush, then K1 on 4 KiB twice back to back
res = []
for _ in range(10):
    flush()
    res.append(ev_time([lambda: k1(c0, 4096), lambda: k1(c0, 4096), lambda: k1(c0, 4096)]))
res = np.array(res)
out["k1_4KiB_after_flush_1st_2nd_3rd_median_us"] = [round(float(np.median(res[:, i])), 2) for i in range(3)]
print("4 KiB after flush: 1st/2nd/3rd", out["k1_4KiB_after_flush_1st_2nd_3rd_median_us"], flush=True)
e1 = torch.empty(1, device="cuda")
res = []
for _ in range(10):
    flush()
    res.append(ev_time([lambda: e1.add_(1), lambda: e1.add_(1), lambda: k1(c0, 4096)]))
res = np.array(res)
out["torch_add_after_flush_1st_2nd_then_k1_median_us"] = [round(float(np.median(res[:, i])), 2) for i in range(3)]
print("after flush: add/add/k1", out["torch_add_after_flush_1st_2nd_then_k1_median_us"], flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/k1_timeline_{tag}.json").write_text(json.dumps(out, indent=1))
np.savez_compressed(f"gpurun_out/k1_timeline_{tag}.npz", **raw)
