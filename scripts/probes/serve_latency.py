"""Per-call latency of utf8v_cuda_validate / _validate_verdict on pageable host
input (the small-call server path up to 64 KiB): min / median / p99 over
repeated back-to-back calls, and the first call after an idle gap."""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np

from paper_2010_03090_b200 import _lib
from tests import _native as nat

lib = _lib.load()
ok, off, kind = C.c_uint8(0), C.c_uint64(0), C.c_int(0)
for n in (16, 256, 4096, 16384, 65536):
    raw = nat.generate_valid(0b0111, n, 7)
    b = np.frombuffer(raw, np.uint8).copy()
    for name, fn in (("validate", lambda: lib.utf8v_cuda_validate(b.ctypes.data, b.size, 0, C.byref(ok))),
                     ("verdict", lambda: lib.utf8v_cuda_validate_verdict(b.ctypes.data, b.size, 0, C.byref(ok),
                                                                         C.byref(off), C.byref(kind)))):
        for _ in range(50):
            fn()
        ts = []
        for _ in range(2000):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        gap = []
        for _ in range(20):
            time.sleep(0.002)
            t0 = time.perf_counter()
            fn()
            gap.append(time.perf_counter() - t0)
        print(f"{name:8s} {b.size:6d} B: min {ts[0]*1e6:6.2f} med {ts[len(ts)//2]*1e6:6.2f} "
              f"p99 {ts[len(ts)*99//100]*1e6:6.2f} us; after 2 ms idle: med {statistics.median(gap)*1e6:6.2f} us",
              flush=True)
a, r = C.c_uint64(0), C.c_uint64(0)
lib.utf8v_cuda_serve_stats(C.byref(a), C.byref(r))
print("server launches", a.value, "requests", r.value)

# Host batches (utf8v_cuda_validate_batch on host arrays): per-call latency.
for n_rec, rec in ((16, 64), (100, 100), (1000, 60), (256, 256)):
    raw = nat.generate_valid(0b0111, n_rec * rec, 9)[: n_rec * rec]
    b = np.frombuffer(raw, np.uint8).copy()
    offs = np.arange(0, n_rec * rec + 1, rec, dtype=np.uint64)
    offs[-1] = b.size
    ver = np.empty(n_rec, np.uint8)
    fn = lambda: lib.utf8v_cuda_validate_batch(b.ctypes.data, b.size, offs.ctypes.data, n_rec, 0, ver.ctypes.data)
    for _ in range(20):
        fn()
    ts = []
    for _ in range(500):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"batch {n_rec:5d} x {rec:4d} B: min {ts[0]*1e6:6.2f} med {ts[len(ts)//2]*1e6:6.2f} us", flush=True)
# Larger host batches (K2 over staged copies; scratch from the library's pool).
for n_rec, rec in ((10000, 100), (5000, 1000)):
    raw = nat.generate_valid(0b0111, n_rec * rec, 9)[: n_rec * rec]
    b = np.frombuffer(raw, np.uint8).copy()
    offs = np.arange(0, n_rec * rec + 1, rec, dtype=np.uint64)
    offs[-1] = b.size
    ver = np.empty(n_rec, np.uint8)
    fn = lambda: lib.utf8v_cuda_validate_batch(b.ctypes.data, b.size, offs.ctypes.data, n_rec, 0, ver.ctypes.data)
    for _ in range(5):
        fn()
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"batch {n_rec:5d} x {rec:4d} B: min {ts[0]*1e6:7.1f} med {ts[len(ts)//2]*1e6:7.1f} us", flush=True)
