"""DEVELOPMENT HARNESS: time K1 inner-loop variants (tools/kbench.cu) on C1."""
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
for i in range(L.kb_count()):
    name = L.kb_name(i).decode()
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
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "kbench.json").write_text(json.dumps(res, indent=1))
