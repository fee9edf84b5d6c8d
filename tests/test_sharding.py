"""Multi-process (gloo, world_size 2 and 4) tests of the shard layer on the
CPU: the shard plan, head/tail bytes and the allreduce(MAX) combine must
reproduce the single-stream verdict for streams whose shard edges cut
characters anywhere, and the allreduce(MIN) of each rank's local first-error
decode must reproduce the oracle's (offset, kind).  Each rank's lane-range
flag comes from the device formula compiled for the CPU
(tests/cpp/swar_host.c swar_lanes), so what is checked is exactly K1's lane
contract."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2010_03090_b200 import sharding
from tests import _native as nat


def cpu_shard_flag(local, shard):
    a = np.ascontiguousarray(np.frombuffer(bytes(local), np.uint8))
    lo, hi = shard.lanes
    return int(nat.swar().swar_lanes(a.ctypes.data if a.size else None, a.size, lo, hi))


def cpu_shard_locate(local, shard):
    """CPU model of shard_first_error: the first flagged lane L of the rank's
    lanes (device formula), then the recovery rule of SURVEY §8(a) 3 on the
    rank's own bytes: B = L - 3 stepped back over <= 3 continuation bytes,
    the oracle over [B, L + 4)."""
    a = np.ascontiguousarray(np.frombuffer(bytes(local), np.uint8))
    lo, hi = shard.lanes
    L = int(nat.swar().swar_first_lane_in(a.ctypes.data if a.size else None, a.size, lo, hi))
    if L == (1 << 64) - 1:
        return None
    b = max(0, L - 3)
    for _ in range(3):
        if b > 0 and b < a.size and (a[b] & 0xC0) == 0x80:
            b -= 1
    ok, off, kind = nat.oracle_verdict(a[b:min(a.size, L + 4)].tobytes())
    assert not ok, "a flagged lane with no error in its window"
    return shard.lo + b + off, kind


def _streams():
    rng = np.random.default_rng(8)
    out = []
    base = np.frombuffer(nat.generate_valid(15, 4099, 31), np.uint8).copy()
    out.append(base)
    for _ in range(40):
        d = base.copy()
        for _k in range(int(rng.integers(0, 2))):
            d[int(rng.integers(0, d.size))] = int(rng.integers(0, 256))
        out.append(d)
    # errors planted right at the shard edges of a 2/4-way split
    for world in (2, 4):
        for sh in sharding.plan(base.size, world)[1:]:
            for delta in (-3, -2, -1, 0, 1, 2):
                d = base.copy()
                d[sh.start + delta] = 0xC0
                out.append(d)
                e = base.copy()
                e[sh.start + delta: sh.start + delta + 2] = [0xE0, 0x85]  # overlong pair
                out.append(e)
                # whole bad sequences straddling the edge: the kind depends on
                # bytes past the lead, which may sit in the next rank's bytes
                for seq in ([0xE0, 0x80, 0x80], [0xED, 0xA0, 0x80], [0xF4, 0x90, 0x80, 0x80],
                            [0xF0, 0x80, 0x80, 0x80], [0xE2, 0x82, 0x41], [0xFF], [0x80, 0x80]):
                    f = base.copy()
                    f[sh.start + delta: sh.start + delta + len(seq)] = seq
                    out.append(f)
    out.append(np.concatenate([base, np.array([0xF0, 0x9F, 0x98], np.uint8)]))  # truncated end
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for d in _streams():
            sh = sharding.plan(d.size, world)[rank]
            local = d[sh.lo:sh.hi].tobytes()
            ok = sharding.validate_sharded(local, sh, shard_flag=cpu_shard_flag)
            v = sharding.verdict_sharded(local, sh, shard_locate=cpu_shard_locate)
            res.append((ok, None if v.valid() else (v.error.offset, int(v.error.kind))))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_verdict_equals_single_stream(world):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = []
    for d in _streams():
        ok, off, kind = nat.oracle_verdict(d.tobytes())
        want.append((ok, None if ok else (off, kind)))
    for r in range(world):
        assert results[r] == want


def test_plan_covers_stream_and_lane_ranges():
    for n in (0, 1, 17, 4096, 10 ** 6 + 3):
        for world in (1, 2, 3, 8):
            if n < 16 * world and world > 1:
                continue
            shards = sharding.plan(n, world)
            assert shards[0].start == 0 and shards[-1].end == n
            for a, b in zip(shards, shards[1:]):
                assert a.end == b.start and b.head == min(b.start, sharding.HEAD) and a.tail == min(sharding.TAIL, n - a.end)
            covered = []
            for sh in shards:
                lo, hi = sh.lanes
                covered.append((sh.lo + lo, sh.lo + hi))
            assert covered[0][0] == 0 and covered[-1][1] == n + 3
            for (a0, a1), (b0, b1) in zip(covered, covered[1:]):
                assert a1 == b0


# ---- record batches -----------------------------------------------------------

def _batch(seed=5, n_records=300):
    rng = np.random.default_rng(seed)
    parts = []
    for r in range(n_records):
        size = int(rng.integers(0, 900))
        if r % 5 == 0:
            parts.append(np.frombuffer(nat.generate_invalid(15, max(size, 4), seed + r, r % 7), np.uint8))
        elif r % 11 == 0:
            parts.append(np.zeros(0, np.uint8))
        else:
            parts.append(np.frombuffer(nat.generate_valid(15, size, seed + r), np.uint8))
    offs = np.zeros(n_records + 1, np.uint64)
    offs[1:] = np.cumsum([p.size for p in parts])
    return np.concatenate(parts), offs, parts


def test_plan_records_covers_and_balances():
    data, offs, parts = _batch()
    for world in (1, 2, 3, 4, 8):
        shards = sharding.plan_records(offs, world)
        assert shards[0].r_begin == 0 and shards[-1].r_end == len(parts)
        for a, b in zip(shards, shards[1:]):
            assert a.r_end == b.r_begin and a.b_end == b.b_begin
        total = int(offs[-1])
        biggest = max(p.size for p in parts)
        for sh in shards:
            assert abs(sh.n_bytes - total / world) <= biggest + 1
            local, local_offs = sharding.local_records(data, offs, sh)
            assert local_offs[0] == 0 and int(local_offs[-1]) == local.size == sh.n_bytes


def cpu_batch(local, local_offs):
    a = np.ascontiguousarray(local)
    out = np.ones(len(local_offs) - 1, np.uint8)
    for r in range(len(local_offs) - 1):
        out[r] = nat.oracle_verdict(a[int(local_offs[r]):int(local_offs[r + 1])].tobytes())[0]
    return out


def _batch_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data, offs, _ = _batch()
        shards = sharding.plan_records(offs, world)
        mine = sharding.validate_batch_sharded(data, offs, shards[rank], batch_fn=cpu_batch)
        q.put((rank, sharding.gather_verdicts(mine, shards).tolist()))
    finally:
        dist.destroy_process_group()


def test_batch_sharded_verdicts_equal_per_record_oracle():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, _, parts = _batch()
    want = [int(nat.oracle_verdict(p.tobytes())[0]) for p in parts]
    for r in range(world):
        assert results[r] == want


def _pipelined_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for pattern in ([], [(5, 1)], [(0, 0), (7, 1)], [(19, 1)]):
            pf = sharding.PipelinedFlags(lambda: torch.zeros(1, dtype=torch.int32), depth=2)
            for step in range(20):
                f = pf.acquire()
                for (s, r) in pattern:          # rank r's kernel flags an error at step s
                    if s == step and r == rank:
                        f.fill_(1)
                pf.submit(f)
            out.append(pf.drain())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_pipelined_flags_reduce_every_step():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert results[r] == [0, 1, 1, 1]


def _state_worker(rank, world, port, q, data: bytes):
    import os
    import numpy as np
    import torch.distributed as dist
    from paper_2010_03090_b200 import sharding
    from tests.test_states import leaf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = np.frombuffer(data, np.uint8)
        sh = sharding.plan(b.size, world)[rank]
        st = sharding.shard_state(b[sh.lo:sh.hi], sh, state_fn=lambda own: leaf(own.tobytes()))
        q.put((rank, sharding.combine_states_sharded(st)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_shard_states_combine_over_gloo(world):
    """Per-shard states (the CPU model of segment_state) gathered over gloo
    and folded in rank order: every rank gets the oracle's verdict, for
    errors straddling the shard edges."""
    import multiprocessing as mp
    import socket
    import numpy as np
    from tests import _native as nat
    from paper_2010_03090_b200 import sharding
    rng = np.random.default_rng(world)
    base = nat.gen_stream_host(1 << 16, 7)
    ctx = mp.get_context("spawn")
    for case in range(4):
        b = base.copy()
        if case:
            edge = sharding.plan(b.size, world)[1 + case % (world - 1)].start
            seq = [[0xE0, 0x80, 0x80], [0xF0, 0x9F], [0xC1, 0x80]][case - 1]
            at = edge + int(rng.integers(-2, 2))
            b[at:at + len(seq)] = seq
        want = nat.oracle_verdict(b)[0]
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        q = ctx.Queue()
        procs = [ctx.Process(target=_state_worker, args=(r, world, port, q, b.tobytes())) for r in range(world)]
        for p in procs:
            p.start()
        res = dict(q.get(timeout=120) for _ in procs)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        assert all(v == want for v in res.values()), (case, res, want)
