#!/usr/bin/env python3
"""bench.py -- B200 Lookup UTF-8 validation throughput (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1|c0|c4]

One step = one pass of the hot path over one batch of synthetic input
resident in HBM: validate_lanes (K1) over the rank's 1 GiB shard of the
config-1 stream (the whole C1 buffer at N=1), followed at N>1 by the
one-word NCCL allreduce(MAX) that combines shard verdicts.  Weak scaling:
every rank validates 1 GiB per step; `value` is the box aggregate.

`e2e` repeats the metric through the public C-ABI with a HOST (pinned)
buffer: utf8v_cuda_validate(host_ptr, n, 0, &ok), which streams the bytes
over PCIe in pieces (n/8, 2..32 MiB) and validates each as it lands; every step
includes the 1 GiB H2D copy and the 4-byte verdict read back.

`--impl reference` times the unmodified reference CPU implementation
(oracle/_ref: validate_lookup, AVX2, compiled from the reference sources)
on this box's host cores, all threads, on the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GiB = 1 << 30
C4_BYTES = 16 * GiB
METRIC = "validated GB/s per GPU and box (device-timed) vs HBM roofline; records/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=["c0", "c1", "c4"])  # C2/C3: other_configs
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C0/C2/C3/C4 side measurements")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the N>1 path with fewer GPUs than ranks "
                         "(ranks share GPUs; no kernel waits on another rank; numbers not meaningful)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks: nvidia-smi sampled during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
HBM_SPEC_GBS = 8000.0  # B200 HBM3e datasheet figure; SURVEY §8(d) asks for both fractions


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    return {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


def ncu_traffic(kernel: str) -> float | None:
    """DRAM bytes per launch of `kernel` from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get("kernels", {}).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def ref_lib():
    so = ROOT / "oracle" / "_ref" / "libutf8v_ref.so"
    if not so.exists():
        return None
    L = C.CDLL(str(so))
    L.ref_validate_lookup_mt.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
    L.ref_validate_lookup_mt.restype = C.c_int
    L.ref_validate_lookup.argtypes = [C.c_void_p, C.c_size_t]
    L.ref_validate_lookup.restype = C.c_int
    return L


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def time_reference(L, buf: np.ndarray, threads: int, seconds: float, max_reps: int | None = None):
    """Best-of GB/s of the reference validate_lookup over buf on `threads`
    threads (after a correctness gate, proj/src/bench.cpp:80-86)."""
    p = buf.ctypes.data
    n = buf.size
    ok = L.ref_validate_lookup_mt(p, n, threads)
    best, total, reps = float("inf"), 0.0, 0
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        L.ref_validate_lookup_mt(p, n, threads)
        dt = time.perf_counter() - t0
        best = min(best, dt)
        total += dt
        reps += 1
        if time.perf_counter() > t_end or (max_reps and reps >= max_reps):
            break
    return {"valid": bool(ok), "best_GBps": n / best / 1e9, "mean_GBps": n * reps / total / 1e9, "reps": reps}


def host_stream(n: int, seed: int, ascii_only: bool) -> np.ndarray:
    from paper_2010_03090_b200 import _lib
    buf = np.empty(n, np.uint8)
    _lib.check(_lib.load().utf8v_gen_stream_host(buf.ctypes.data, n, seed, int(ascii_only), host_threads()))
    return buf


# ---------------------------------------------------------------------------
WORKLOADS = {"c1": "C1: valid UTF-8, 0.4/0.2/0.3/0.1 length mix, seed 2, 1 GiB per GPU",
             "c0": "C0: 64 MiB ASCII + 2% LF, seed 1, per GPU",
             "c4": "C4: 16 GiB mix, seed 5, sharded over the GPUs (strong scaling)"}
SEEDS = {"c0": 1, "c1": 2, "c4": 5}
DATA = "synthetic (seeded splitmix64 generator, DESIGN.md 'Synthetic inputs')"


def workload_bytes(config: str, world: int) -> tuple[int, int]:
    """(bytes per GPU, bytes in the whole job) of a bench config."""
    if config == "c4":
        return C4_BYTES // world, C4_BYTES
    per = (64 << 20) if config == "c0" else GiB
    return per, per * world


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    L = ref_lib()
    base = {"metric": METRIC, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": DATA}
    if L is None:
        print(json.dumps({**base, "unavailable": "oracle/_ref/libutf8v_ref.so not built (no reference checkout)"}))
        return
    per, n_total = workload_bytes(args.config, max(1, args.gpus))
    seed, ascii_only = SEEDS[args.config], args.config == "c0"
    # The sample: the whole workload when it fits in host RAM comfortably.
    n = min(n_total, 4 * GiB)
    buf = host_stream(n, seed, ascii_only)
    T = host_threads()
    ok = L.ref_validate_lookup_mt(buf.ctypes.data, n, T)
    for _ in range(max(1, args.warmup)):
        L.ref_validate_lookup_mt(buf.ctypes.data, n, T)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        L.ref_validate_lookup_mt(buf.ctypes.data, n, T)
    dt = time.perf_counter() - t0
    value = n * args.steps / dt / 1e9
    sample = f"{n} bytes of config {args.config} (seed {seed}) per step, {args.steps} steps"
    print(json.dumps({**base, "value": value, "ms_per_step": dt / args.steps * 1e3,
                      "config": {"workload": WORKLOADS[args.config], "bytes_per_gpu": per, "bytes_total": n_total,
                                 "sample_bytes": n, "cpu": cpu_model()},
                      "valid": bool(ok),
                      "cpu_baseline": {"value": value, "unit": "GB/s", "cores": T, "kind": "reference",
                                       "sample": sample},
                      "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2010_03090_b200 as u8
    from paper_2010_03090_b200 import _lib, configs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()

    # ---- workload: this rank's shard (+ up to 16 bytes of halo) ----------
    per, n_total = workload_bytes(args.config, world)
    assert (args.config != "c4" or n_total == configs.C4["n"]) and (args.config != "c0" or per == configs.C0["n"])
    seed = SEEDS[args.config]
    ascii_only = args.config == "c0"
    s, e = rank * per, (rank + 1) * per
    from paper_2010_03090_b200 import sharding
    sh = sharding.plan(n_total, world)[rank]
    halo, last = sh.head, sh.last
    # The shard [lo, hi) of the global stream (head + tail bytes included),
    # generated in place: chunk seeds depend only on the chunk index, so the
    # bytes equal those of the whole stream.
    shard = torch.empty(sh.n_local, dtype=torch.uint8, device=dev)
    _lib.check(lib.utf8v_gen_stream_range(shard.data_ptr(), n_total, sh.lo, sh.hi, seed, int(ascii_only),
                                          torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    n_local = shard.numel()
    lane_lo, lane_hi = sh.lanes
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    if world > 1:
        dist.barrier()

    # N > 1: the 4-byte allreduce(MAX) of step i overlaps the kernel of step
    # i+1 (double-buffered flags, sharding.PipelinedFlags).
    pf = sharding.PipelinedFlags(lambda: torch.zeros(1, dtype=torch.int32, device=dev)) if world > 1 else None

    def step():
        f = pf.acquire() if pf else flag
        _lib.check(lib.utf8v_cuda_validate_lanes_async(shard.data_ptr(), n_local, lane_lo, lane_hi,
                                                       f.data_ptr(), sp))
        if pf:
            pf.submit(f)

    def verdict_flag() -> int:
        return pf.drain() if pf else int(flag.item())

    # correctness gate before timing (proj/src/bench.cpp:80-86)
    flag.zero_()
    step()
    torch.cuda.synchronize()
    expect_valid = True
    assert (verdict_flag() == 0) == expect_valid, "verdict mismatch on the benchmark input"

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    flag.zero_()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
    if pf:
        pf.wait_all()  # the last steps' allreduces are inside the timed region
    t_stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_stop)
    clocks = sampler.stop() if sampler else None
    verdict_ok = verdict_flag() == 0
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = per * world * args.steps / (ms_max / 1e3) / 1e9
    per_gpu = per * args.steps / (ms / 1e3) / 1e9

    # ---- kernel-only timing for the roofline (same stream, no collective) --
    kflag = torch.zeros(1, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    k0 = torch.cuda.Event(enable_timing=True)
    k1 = torch.cuda.Event(enable_timing=True)
    kreps = max(10, min(args.steps, 200))
    k0.record(stream)
    for _ in range(kreps):
        _lib.check(lib.utf8v_cuda_validate_lanes_async(shard.data_ptr(), n_local, lane_lo, lane_hi,
                                                       kflag.data_ptr(), sp))
    k1.record(stream)
    torch.cuda.synchronize()
    kernel_ms = k0.elapsed_time(k1) / kreps
    peaks = measured_peaks()
    alg_bytes = per  # one read per input byte of the shard (halo re-reads are overhead)
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    traffic = ncu_traffic("k_validate")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "frac_of_spec": achieved / HBM_SPEC_GBS, "spec_peak": HBM_SPEC_GBS,
                "peak_source": peaks["source"], "kernel": "u8v::k_validate",
                "kernel_ms": kernel_ms, "algorithmic_bytes_per_launch": alg_bytes}

    # ---- e2e through the public API with pinned host buffers ---------------
    es = max(1, args.e2e_steps)
    if world == 1:
        # The drop-in call: whole stream from pinned host memory.
        host = torch.empty(n_local, dtype=torch.uint8, pin_memory=True)
        host.copy_(shard)
        hp = host.data_ptr()
        ok = C.c_uint8(0)
        _lib.check(lib.utf8v_cuda_validate(hp, n_local, 0, C.byref(ok)))  # warm + gate
        assert ok.value == 1, "e2e verdict mismatch"
        t0 = time.perf_counter()
        for _ in range(es):
            _lib.check(lib.utf8v_cuda_validate(hp, n_local, 0, C.byref(ok)))
        et = time.perf_counter() - t0
        path = "utf8v_cuda_validate(pinned host ptr): H2D pieces (32 MiB at 1 GiB) overlapped with K1"
    else:
        # Every rank: its pinned host shard -> utf8v_cuda_validate_lanes (H2D +
        # K1) -> 4-byte NCCL allreduce(MAX) -> verdict (sharding.py).
        host = torch.empty(n_local, dtype=torch.uint8, pin_memory=True)
        host.copy_(shard)
        hnp = host.numpy()
        assert sharding.validate_sharded(hnp, sh, device=dev), "e2e verdict mismatch"
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(es):
            sharding.validate_sharded(hnp, sh, device=dev)
        et = time.perf_counter() - t0
        path = "sharding.validate_sharded(pinned host shard): utf8v_cuda_validate_lanes + NCCL allreduce(MAX)"
    tt = torch.tensor([et], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = {"value": per * world * es / float(tt.item()) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": n_local * world, "d2h_bytes_per_step": 4 * world, "path": path}
    del host

    # ---- CPU baseline (rank 0, N=1): the reference on a bounded sample ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        L = ref_lib()
        if L is not None:
            sample_n = min(per, 256 << 20)
            hbuf = shard[halo:halo + sample_n].cpu().numpy()
            T = host_threads()
            r = time_reference(L, hbuf, T, args.cpu_seconds)
            r1 = time_reference(L, hbuf[: 64 << 20], 1, min(3.0, args.cpu_seconds), max_reps=5)
            cpu = {"value": r["best_GBps"], "unit": "GB/s", "cores": T, "kind": "reference",
                   "sample": f"first {sample_n >> 20} MiB of the C1 shard, best of {r['reps']} passes, "
                             f"validate_lookup (AVX2) split at character boundaries over {T} threads",
                   "single_thread_GBps": r1["best_GBps"], "cpu": cpu_model()}

    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        del shard
        torch.cuda.empty_cache()
        extras = measure_extras(lib, dev, max(5, min(args.steps, 50)))

    if rank == 0:
        workload = WORKLOADS[args.config]
        out = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.config == "c4" else "weak", "vs_baseline": None, "dtype": "u8",
            "data": DATA,
            "config": {"workload": workload, "bytes_per_gpu": per, "bytes_total": per * world,
                       "l2": "input (>=1 GiB) larger than the 126 MB L2; no flush needed",
                       "parallelism": f"dp{world}: byte-range shards (<=16-byte look-back head, 3-byte tail)"
                                      + (f" + 1-word {args.dist_backend.upper()} allreduce(MAX) per step, overlapped"
                                         " with the next step's kernel" if world > 1 else "")},
            "per_gpu_GBps": per_gpu, "verdict_valid": verdict_ok,
            "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": args.steps, "other_configs": extras,
        }
        print(json.dumps(out))


def _time_device(fn, reps: int, stream) -> float:
    """Mean ms of fn() over reps launches on `stream` (CUDA events)."""
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _time_device_flushed(fn, reps: int, stream, dev) -> float:
    """Mean ms of fn() timed launch by launch, with the 126 MB L2 flushed
    (a 512 MiB scratch write, then a read of it) before each one -- for inputs
    that fit in L2."""
    import torch
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with torch.cuda.stream(stream):
        for a, b in ev:
            # Flush: write then read 512 MiB (> the 126 MB L2), so L2 holds
            # clean unrelated lines -- no pending write-backs compete with the
            # timed kernel.
            scratch.fill_(1)
            scratch.view(torch.int64).sum()
            a.record(stream)
            fn()
            b.record(stream)
    torch.cuda.synchronize()
    del scratch
    return sum(a.elapsed_time(b) for a, b in ev) / reps


def measure_extras(lib, dev, reps: int) -> dict:
    """The other BASELINE configs at N=1 (not the headline): C0 GB/s, C2/C3
    records/s through the batch kernels (K2L for C2's 64 large segments, K2 for
    C3), C4's 16 GiB stream through K1 and its three variants' verdicts +
    first-error offsets (K3).  roofline_frac: algorithmic GB/s over the
    measured HBM peak; traffic: ncu DRAM bytes per launch (profiles/)."""
    import torch

    from paper_2010_03090_b200 import _lib, configs
    import paper_2010_03090_b200 as u8

    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    out = {}
    flag = torch.zeros(1, dtype=torch.int32, device=dev)

    d = configs.gen_c0()
    n = d.numel()
    ms = _time_device_flushed(lambda: _lib.check(lib.utf8v_cuda_validate_lanes_async(
        d.data_ptr(), n, 0, n + 3, flag.data_ptr(), sp)), reps, st, dev)
    torch.cuda.synchronize()
    out["c0"] = {"GBps": n / ms / 1e6, "ms": ms, "valid": int(flag.item()) == 0, "bytes": n,
                 "l2": "flushed before each timed launch (64 MiB fits in L2)"}
    del d

    for name, gen in (("c2", configs.gen_c2), ("c3", configs.gen_c3)):
        b = gen()
        ver = torch.empty(b.n_records, dtype=torch.uint8, device=dev)
        fn = lambda: _lib.check(lib.utf8v_cuda_validate_batch_async(  # noqa: E731
            b.data.data_ptr(), b.nbytes, b.d_offsets.data_ptr(), b.n_records, ver.data_ptr(), sp))
        small = b.nbytes + 8 * b.n_records < (512 << 20)
        ms = _time_device_flushed(fn, reps, st, dev) if small else _time_device(fn, reps, st)
        got = ver.cpu().numpy()
        alg = b.nbytes + 8 * (b.n_records + 1) + b.n_records
        kernel = "k_batch_large" if name == "c2" else "k_batch"  # launch_batch's dispatch (kernels.cuh)
        peak = measured_peaks()["hbm_gbs"]
        out[name] = {"records_per_s": b.n_records / (ms / 1e3), "GBps": alg / ms / 1e6, "ms": ms,
                     "records": b.n_records, "bytes": b.nbytes, "invalid_records": int((got == 0).sum()),
                     "verdicts_match_expected": bool((got == b.expected).all()), "l2_flushed": small,
                     "kernel": f"u8v::{kernel}", "algorithmic_bytes": alg,
                     "roofline_frac": alg / ms / 1e6 / peak, "traffic": ncu_traffic(kernel)}
        del b, ver
        torch.cuda.empty_cache()

    # The user-facing entry points on C1 (1 GiB): the verdict API on valid and
    # on invalid input (K1, then K3 + window decode), the streaming session
    # over device pieces, and host input from pageable memory.
    d = configs.gen_c1()
    n = d.numel()
    api = {}
    ms = _time_device(lambda: u8.validate_lookup_verdict(d), 5, st)
    api["verdict_valid_GBps"] = n / ms / 1e6
    orig = int(d[n // 2].item())
    d[n // 2] = 0xC0
    v = u8.validate_lookup_verdict(d)
    ms = _time_device(lambda: u8.validate_lookup_verdict(d), 5, st)
    api["verdict_invalid_GBps"] = n / ms / 1e6
    api["verdict_invalid_offset"] = v.error.offset if not v.valid() else None
    d[n // 2] = orig
    # One session, reused (finish() resets it); it runs on its own CUDA
    # stream and finish() synchronises, so the wall clock brackets the work.
    sess = u8.LookupStream()
    for mib in (64, 256):
        piece = mib << 20

        def stream_once():
            for a in range(0, n, piece):
                sess.feed(d[a:a + piece])
            return sess.finish()
        assert stream_once()
        t0 = time.perf_counter()
        for _ in range(5):
            stream_once()
        api[f"stream_{mib}MiB_pieces_GBps"] = 5 * n / (time.perf_counter() - t0) / 1e9
    sess.close()
    host = d.cpu().numpy()
    ok = C.c_uint8()
    _lib.check(lib.utf8v_cuda_validate(host.ctypes.data, n, 0, C.byref(ok)))  # warm: pinned ring
    t0 = time.perf_counter()
    for _ in range(3):
        _lib.check(lib.utf8v_cuda_validate(host.ctypes.data, n, 0, C.byref(ok)))
    api["pageable_host_GBps"] = 3 * n / (time.perf_counter() - t0) / 1e9
    api["note"] = ("device-timed (verdict) / wall-clock (stream session, pageable host with PCIe); the C1 byte at n/2 "
                   "is set to 0xC0 for the invalid case and restored afterwards")
    out["c1_api"] = api
    del d, host
    torch.cuda.empty_cache()

    n4 = configs.C4["n"]
    c4 = {}
    for variant in (0, 1, 2):
        d, err = configs.gen_c4(n4, variant=variant)
        if variant == 0:
            ms = _time_device(lambda: _lib.check(lib.utf8v_cuda_validate_lanes_async(
                d.data_ptr(), n4, 0, n4 + 3, flag.data_ptr(), sp)), max(3, reps // 5), st)
            c4["A_GBps"] = n4 / ms / 1e6
            c4["A_ms"] = ms
        v = u8.validate_lookup_verdict(d)
        c4["ABC"[variant]] = {"valid": v.valid(), "offset": None if v.valid() else v.error.offset,
                              "kind": None if v.valid() else str(v.error.kind), "expected_offset": err,
                              "ok": (v.valid() if err is None else (not v.valid() and v.error.offset == err))}
        del d
        torch.cuda.empty_cache()
    out["c4"] = c4
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        local_rank %= torch.cuda.device_count()  # one GPU per rank; shared only under --dist-backend gloo
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
