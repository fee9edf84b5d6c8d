import sys, torch
sys.path.insert(0, '.')
from paper_2010_03090_b200 import _lib, configs
lib = _lib.load(); st = torch.cuda.current_stream(); sp = st.cuda_stream
flag = torch.zeros(1, dtype=torch.int32, device='cuda')
scratch = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
d = configs.gen_c0(); n = d.numel()
def t(fn, flush, reps=30):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        if flush:
            scratch.fill_(1); scratch.view(torch.int64).sum()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2] * 1e3
for m in (4096, 1 << 20, 8 << 20, 16 << 20, 32 << 20, 64 << 20):
    f = lambda: lib.utf8v_cuda_validate_lanes_async(d.data_ptr(), m, 0, m + 3, flag.data_ptr(), sp)
    print(f"{m>>10:8d} KiB  flushed {t(f, True):7.2f} us   hot {t(f, False):7.2f} us", flush=True)
e = torch.empty(1, device='cuda')
print("empty torch kernel", t(lambda: e.add_(1), False), "us")
