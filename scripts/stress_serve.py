"""Randomised stress of the small-call server (csrc/serve.cu) against the
oracle, for a fixed wall-clock budget: `python scripts/stress_serve.py SECONDS
SEED THREADS`.  Each thread draws calls of every server mode -- validate,
verdict (offset + kind), lane ranges, host batches -- on inputs of 1 B ..
64 KiB with injected errors, separated by pauses of 0, ~50 us, ~150 us or
~1 ms (around the 100 us idle exit, so requests race the server's exit and
relaunch), while one more thread issues grid-wide device calls that bump the
servers' epoch.  Every answer is compared with the oracle (lane ranges with
the SWAR checker)."""
import ctypes as C
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2010_03090_b200 import _lib
from tests import _native as nat

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n_threads = int(sys.argv[3]) if len(sys.argv) > 3 else 6
lib = _lib.load()
pool = np.frombuffer(nat.generate_valid(15, 1 << 22, seed), np.uint8).copy()
BAD = [[0xC0, 0x80], [0xE0, 0x80, 0x80], [0xED, 0xA0, 0x80], [0xF4, 0x90, 0x80, 0x80], [0x80], [0xF5], [0xE1, 0x41],
       [0xF0, 0x9F, 0x98], [0xC3]]
stop = time.monotonic() + budget
counts = {"validate": 0, "verdict": 0, "lanes": 0, "batch": 0, "grid": 0}
errors = []
lock = threading.Lock()


def pause(rng):
    k = int(rng.integers(0, 4))
    if k == 1:
        time.sleep(0.00005)
    elif k == 2:
        time.sleep(0.00015)
    elif k == 3:
        time.sleep(0.001)


def sample(rng, n):
    a = int(rng.integers(0, pool.size - n))
    b = pool[a:a + n].copy()
    for _ in range(int(rng.integers(0, 3))):
        seq = BAD[int(rng.integers(len(BAD)))]
        at = int(rng.integers(0, n))
        b[at:at + len(seq)] = seq[:n - at]
    return b


def worker(k):
    rng = np.random.default_rng(seed * 1000 + k)
    local = {"validate": 0, "verdict": 0, "lanes": 0, "batch": 0}
    ok, off, kind, flag = C.c_uint8(), C.c_uint64(), C.c_int(), C.c_uint32()
    try:
        while time.monotonic() < stop and not errors:
            n = int(rng.integers(1, 600)) if rng.random() < 0.5 else int(rng.integers(1, 65537))
            b = sample(rng, n)
            mode = int(rng.integers(0, 4))
            if mode == 0:
                _lib.check(lib.utf8v_cuda_validate(b.ctypes.data, n, 0, C.byref(ok)))
                if bool(ok.value) != nat.oracle_verdict(b)[0]:
                    errors.append(("validate", k, n))
                local["validate"] += 1
            elif mode == 1:
                _lib.check(lib.utf8v_cuda_validate_verdict(b.ctypes.data, n, 0, C.byref(ok), C.byref(off),
                                                           C.byref(kind)))
                got = (True, None, None) if ok.value else (False, off.value, kind.value)
                if got != nat.oracle_verdict(b):
                    errors.append(("verdict", k, n, got))
                local["verdict"] += 1
            elif mode == 2:
                lo = int(rng.integers(0, n + 4))
                hi = int(rng.integers(lo, n + 4))
                _lib.check(lib.utf8v_cuda_validate_lanes(b.ctypes.data, n, lo, hi, 0, C.byref(flag)))
                if bool(flag.value) != bool(nat.swar().swar_lanes(b.ctypes.data, n, lo, hi)):
                    errors.append(("lanes", k, n, lo, hi))
                local["lanes"] += 1
            else:
                R = int(rng.integers(1, 300))
                cuts = np.sort(rng.integers(0, n + 1, R - 1))
                offs = np.concatenate([[0], cuts, [n]]).astype(np.uint64)
                ver = np.empty(R, np.uint8)
                _lib.check(lib.utf8v_cuda_validate_batch(b.ctypes.data, n, offs.ctypes.data, R, 0,
                                                         ver.ctypes.data))
                if not np.array_equal(ver, nat.oracle_batch(b, offs, threads=1)):
                    errors.append(("batch", k, n, R))
                local["batch"] += 1
            pause(rng)
        lib.utf8v_cuda_release_thread_resources()
    except Exception as e:  # noqa: BLE001
        errors.append(("exception", k, repr(e)))
    with lock:
        for key, v in local.items():
            counts[key] += v


def grid_worker():
    rng = np.random.default_rng(seed)
    torch.cuda.set_device(0)
    d = torch.from_numpy(pool).cuda()
    want = nat.oracle_verdict(pool, threads=8)[0]
    ok = C.c_uint8()
    try:
        while time.monotonic() < stop and not errors:
            _lib.check(lib.utf8v_cuda_validate(d.data_ptr(), d.numel(), 1, C.byref(ok)))
            if bool(ok.value) != want:
                errors.append(("grid", ok.value))
            counts["grid"] += 1
            time.sleep(float(rng.choice([0.0, 0.0002, 0.002])))
        lib.utf8v_cuda_release_thread_resources()
    except Exception as e:  # noqa: BLE001
        errors.append(("exception-grid", repr(e)))


ts = [threading.Thread(target=worker, args=(k,)) for k in range(n_threads)] + [threading.Thread(target=grid_worker)]
for t in ts:
    t.start()
for t in ts:
    t.join()
if errors:
    print("stress FAILED:", errors[:10])
    sys.exit(1)
print(f"stress ok: {counts} over {n_threads} threads + a grid caller, {budget:.0f} s, seed {seed}")
