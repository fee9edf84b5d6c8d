"""The multi-GPU combine in the native layer (csrc/comm.cu) on one B200.

NCCL: a one-rank communicator (ncclCommInitRank) and a one-device
ncclCommInitAll set run the real NCCL entry points -- K1 + ncclAllReduce from
C++ -- and must give the oracle's verdict and first error.  Several NCCL
ranks cannot share one GPU, so the multi-rank arithmetic of the combine is
covered by the gloo tests (test_sharding.py) and by the P2P test below.

P2P: two and three processes on the one GPU map each other's flag words with
CUDA IPC (the same mechanism that crosses NVLink between GPUs); each rank
validates its own shard of a stream and a K1 warp that finds an error ORs
into every rank's word.  No kernel waits on another rank.
"""
from __future__ import annotations

import ctypes as C
import multiprocessing as mp
import socket

import numpy as np
import pytest

from tests import _native as nat

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bad_cases(base: np.ndarray, world: int):
    """(label, bytes) cases: valid, and bad sequences straddling each shard
    edge or deep inside a shard (as test_gpu_sharding.py)."""
    from paper_2010_03090_b200 import sharding
    yield "valid", base
    edges = [s.start for s in sharding.plan(base.size, world)[1:]] or [base.size // 2]
    seqs = [[0xE0, 0x80, 0x80], [0xF4, 0x90, 0x80, 0x80], [0xED, 0xA0, 0x80], [0x80], [0xC1], [0xF0, 0x9F]]
    for i, seq in enumerate(seqs):
        for d in (-2, 0, 1):
            at = edges[i % len(edges)] + d
            b = base.copy()
            b[at:at + len(seq)] = seq
            yield f"seq{i}@edge{d:+d}", b
    b = base.copy()
    b[-1] = 0xC3  # truncated at the end of the stream (last shard)
    yield "truncated-end", b


def test_nccl_one_rank_comm_matches_oracle():
    import torch
    from paper_2010_03090_b200 import _lib, configs, sharding
    torch.cuda.set_device(0)
    lib = _lib.load()
    buf = (C.c_uint8 * _lib.COMM_ID_BYTES)()
    _lib.check(lib.utf8v_cuda_comm_unique_id(buf))
    with sharding.NcclComm(0, 1, unique_id=bytes(buf)) as comm:
        base = configs.gen_c1(3 << 20, seed=21).cpu().numpy()
        sh = sharding.plan(base.size, 1)[0]
        n_cases = 0
        for label, b in _bad_cases(base, 4):
            ok, off, kind = nat.oracle_verdict(b)
            assert comm.validate(b.tobytes(), sh) is bool(ok), label                 # host shard
            dev = torch.from_numpy(b).cuda()
            assert comm.validate(dev, sh) is bool(ok), label                         # device shard
            v = comm.verdict(dev, sh)
            assert v.valid() is bool(ok), label
            if not ok:
                assert (v.error.offset, int(v.error.kind)) == (off, kind), label
            v = comm.verdict(b.tobytes(), sh)
            assert (None if v.valid() else (v.error.offset, int(v.error.kind))) == (None if ok else (off, kind))
            n_cases += 1
        assert n_cases > 10
        # the asynchronous form: K1 into the local flag, allreduce into the global one
        dev = torch.from_numpy(base).cuda()
        flags = torch.zeros(2, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream()
        lo, hi = sh.lanes
        for _ in range(3):
            comm.validate_async(dev.data_ptr(), dev.numel(), lo, hi, flags.data_ptr(), flags.data_ptr() + 4,
                                st.cuda_stream)
        torch.cuda.synchronize()
        assert flags.tolist() == [0, 0]
        dev[12345] = 0xFF
        comm.validate_async(dev.data_ptr(), dev.numel(), lo, hi, flags.data_ptr(), flags.data_ptr() + 4,
                            st.cuda_stream)
        torch.cuda.synchronize()
        assert flags.tolist() == [1, 1]


def test_nccl_init_all_sharded_device():
    """utf8v_cuda_comm_init_all + utf8v_cuda_validate_sharded_device on the
    visible devices (one here): shards from sharding.plan, K1 per device,
    one grouped ncclAllReduce."""
    import torch
    from paper_2010_03090_b200 import _lib, configs, sharding
    lib = _lib.load()
    ndev = torch.cuda.device_count()
    comms = (C.c_void_p * ndev)()
    _lib.check(lib.utf8v_cuda_comm_init_all(ndev, None, comms))
    try:
        base = configs.gen_c1(2 << 20, seed=22).cpu().numpy()
        for label, b in _bad_cases(base, ndev):
            plan = sharding.plan(b.size, ndev)
            shards = [torch.from_numpy(b[s.lo:s.hi].copy()).to(f"cuda:{g}") for g, s in enumerate(plan)]
            ptrs = (C.c_void_p * ndev)(*[t.data_ptr() for t in shards])
            nbytes = (C.c_uint64 * ndev)(*[s.n_local for s in plan])
            los = (C.c_uint64 * ndev)(*[s.lanes[0] for s in plan])
            his = (C.c_uint64 * ndev)(*[s.lanes[1] for s in plan])
            ok = C.c_uint8(9)
            torch.cuda.synchronize()
            _lib.check(lib.utf8v_cuda_validate_sharded_device(comms, ndev, ptrs, nbytes, los, his, C.byref(ok)))
            assert ok.value == int(nat.oracle_verdict(b)[0]), label
    finally:
        for g in range(ndev):
            lib.utf8v_cuda_comm_destroy(comms[g])


def _p2p_worker(rank, world, port, q, data: bytes):
    import os
    import torch
    import torch.distributed as dist
    from paper_2010_03090_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cases = [np.frombuffer(c, np.uint8) for c in data]
        out = []
        with sharding.P2PFlags(rank, world) as flags:
            st = torch.cuda.current_stream()
            for b in cases:
                sh = sharding.plan(b.size, world)[rank]
                local = torch.from_numpy(b[sh.lo:sh.hi].copy()).cuda()
                lo, hi = sh.lanes
                flags.reset()
                dist.barrier()                      # every word is zero before any K1 runs
                for _ in range(2):                  # back-to-back launches (PDL overlap)
                    flags.validate_async(local.data_ptr(), local.numel(), lo, hi, st.cuda_stream)
                torch.cuda.synchronize()
                dist.barrier()                      # every rank's K1 has completed
                out.append(flags.read())
                dist.barrier()                      # reads done before the next reset
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_p2p_flags_multiprocess(world):
    """Every rank's word equals the whole stream's verdict, whichever rank
    held the error (ranks share the GPU through CUDA IPC)."""
    from paper_2010_03090_b200 import configs
    base = configs.gen_c1(1 << 20, seed=23).cpu().numpy()
    cases = list(_bad_cases(base, max(world, 2)))
    want = [0 if nat.oracle_verdict(b)[0] else 1 for _, b in cases]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    payload = [b.tobytes() for _, b in cases]
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, payload)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        got = [int(f != 0) for f in res[r]]
        assert got == want, (world, r, [c for (c, _), g, w in zip(cases, got, want) if g != w])
    assert any(want) and not all(want)
