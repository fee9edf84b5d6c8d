"""DEVELOPMENT HARNESS: time K1 inner-loop variants (tools/kbench.cu) on C1.
`python tools/kbench.py [name-prefix ...]` times only the variants whose names
start with one of the prefixes (all when none are given)."""
import ctypes as C, json, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
so = ROOT / "tools" / "libkbench.so"
if not so.exists() or so.stat().st_mtime < (ROOT / "tools" / "kbench.cu").stat().st_mtime:
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-o", str(so), str(ROOT / "tools" / "kbench.cu")])
import torch
from paper_2010_03090_b200 import configs
L = C.CDLL(str(so))
L.kb_name.restype = C.c_char_p
L.kb_launch.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
n = 1 << 30
d = configs.gen_c1(n, seed=2)
bad = d.clone(); bad[n // 3] = 0xC0
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
res = {}
only = tuple(sys.argv[1:])
for i in range(L.kb_count()):
    name = L.kb_name(i).decode()
    if only and not name.startswith(only):
        continue
    flag.zero_(); L.kb_launch(i, d.data_ptr(), n, flag.data_ptr(), st.cuda_stream); torch.cuda.synchronize()
    ok = int(flag.item()) == 0
    flag.zero_(); L.kb_launch(i, bad.data_ptr(), n, flag.data_ptr(), st.cuda_stream); torch.cuda.synchronize()
    detects = int(flag.item()) != 0
    for _ in range(5): L.kb_launch(i, d.data_ptr(), n, flag.data_ptr(), st.cuda_stream)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    reps = 50
    for _ in range(reps): occ = L.kb_launch(i, d.data_ptr(), n, flag.data_ptr(), st.cuda_stream)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = {"GBps": n / ms / 1e6, "ms": ms, "valid_ok": ok, "detects": detects, "blocks_per_sm": occ}
    print(name, json.dumps(res[name]), flush=True)
# ASCII (C0 recipe) 1 GiB: the fast path's case
a = None if only else configs.gen_stream(n, seed=1, ascii_only=True)
if a is not None:
    for i in range(L.kb_count()):
        name = L.kb_name(i).decode()
        if not name.startswith(("v10_u4_b4", "v11", "v12", "v13")):
            continue
        for _ in range(3): L.kb_launch(i, a.data_ptr(), n, flag.data_ptr(), st.cuda_stream)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20): L.kb_launch(i, a.data_ptr(), n, flag.data_ptr(), st.cuda_stream)
        e1.record(st); torch.cuda.synchronize()
        print("ASCII", name, n / (e0.elapsed_time(e1) / 20) / 1e6, flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "kbench.json").write_text(json.dumps(res, indent=1))

# The production entry point on the same buffer, same process.
from paper_2010_03090_b200 import _lib
pl = _lib.load()
for _ in range(5):
    pl.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n + 3, flag.data_ptr(), st.cuda_stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(50):
    pl.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n + 3, flag.data_ptr(), st.cuda_stream)
e1.record(st); torch.cuda.synchronize()
print("PRODUCTION lanes[0,n+3)", n / (e0.elapsed_time(e1) / 50) / 1e6, flush=True)
e0.record(st)
for _ in range(50):
    pl.utf8v_cuda_validate_lanes_async(d.data_ptr(), n, 0, n, flag.data_ptr(), st.cuda_stream)
e1.record(st); torch.cuda.synchronize()
print("PRODUCTION lanes[0,n)", n / (e0.elapsed_time(e1) / 50) / 1e6, flush=True)
