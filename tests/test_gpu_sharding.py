"""Shard layer on the GPU: record-range shards of a C3-like batch, each
validated through the batch entry point (one after another on one GPU),
concatenate to the whole batch's verdicts and to the oracle's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_record_shards_on_gpu_match_whole_batch():
    import paper_2010_03090_b200 as u8
    from paper_2010_03090_b200 import configs, sharding
    b = configs.gen_c3(n_records=20000, seed=9)
    data = b.data.cpu().numpy()
    offs = b.offsets if hasattr(b, "offsets") else b.d_offsets.cpu().numpy()
    whole = u8.validate_lookup_batch(data, offs)
    assert (whole == b.expected).all()
    for world in (1, 2, 3, 8):
        shards = sharding.plan_records(offs, world)
        parts = [sharding.validate_batch_sharded(data, offs, sh) for sh in shards]
        assert (np.concatenate(parts) == whole).all(), world


def test_single_process_sharded_entry_point():
    """utf8v_cuda_validate_sharded: host input cut into n_gpus shards (one
    host thread each, round-robin over the visible devices), errors planted
    around every shard edge; verdict equals the whole-stream oracle."""
    import ctypes as C
    from paper_2010_03090_b200 import _lib, configs
    from tests import _native as nat
    lib = _lib.load()
    base = configs.gen_c1(4 << 20, seed=4).cpu().numpy()
    ok = C.c_uint8()
    for g in (1, 2, 3, 4, 8):
        _lib.check(lib.utf8v_cuda_validate_sharded(base.ctypes.data, base.size, g, 0, C.byref(ok)))
        assert ok.value == 1, g
        cuts = [((k * base.size) // g) & ~15 for k in range(1, g)]
        for cut in cuts[:3]:
            for delta in (-2, 0, 1):
                for seq in (b"\xc0", b"\xe0\x80", b"\xed\xa0", b"\x80"):
                    d = base.copy()
                    d[cut + delta:cut + delta + len(seq)] = np.frombuffer(seq, np.uint8)
                    want = nat.oracle_verdict(d.tobytes())[0]
                    _lib.check(lib.utf8v_cuda_validate_sharded(d.ctypes.data, d.size, g, 0, C.byref(ok)))
                    assert ok.value == int(want), (g, cut, delta, seq)
        t = base.copy()
        t[-2:] = [0xF0, 0x9F]  # truncated at the very end (last shard's end check)
        _lib.check(lib.utf8v_cuda_validate_sharded(t.ctypes.data, t.size, g, 0, C.byref(ok)))
        assert ok.value == 0
    assert lib.utf8v_cuda_validate_sharded(base.ctypes.data, base.size, 0, 0, C.byref(ok)) == _lib.UTF8V_ERR_ARG


def test_malformed_device_offsets_stay_in_bounds():
    """The async batch entry point reads offsets on the device; malformed ones
    (non-monotonic, past the data) give unspecified verdicts but no fault: the
    call succeeds, the stream stays usable, and a canary byte placed right
    after the verdict array is untouched."""
    import torch
    import paper_2010_03090_b200 as u8
    from paper_2010_03090_b200 import _lib, configs
    lib = _lib.load()
    b = configs.gen_c3(n_records=3000, seed=4)
    st = torch.cuda.current_stream().cuda_stream
    for mutate in ("past_end", "non_monotonic", "last_before_first"):
        offs = b.d_offsets.clone()
        if mutate == "past_end":
            offs[-1] = offs[-1] + (1 << 24)
        elif mutate == "non_monotonic":
            offs[5] = offs[-1] + 1000
        else:
            offs[-1] = 0
            offs[0] = 100
        buf = torch.full((b.n_records + 1,), 0xAB, dtype=torch.uint8, device="cuda")
        _lib.check(lib.utf8v_cuda_validate_batch_async(b.data.data_ptr(), b.nbytes, offs.data_ptr(),
                                                       b.n_records, buf.data_ptr(), st))
        torch.cuda.synchronize()
        assert int(buf[-1].item()) == 0xAB, mutate
    # the few-large-records kernel (K2L: <= 2048 records of >= 64 KiB on
    # average) with the same mutations and with offsets that are pure noise
    d = configs.gen_c1(16 << 20, seed=7)
    n = d.numel()
    good = torch.from_numpy((np.arange(65, dtype=np.int64) * (n // 64))).cuda()
    rng = np.random.default_rng(3)
    for mutate in ("past_end", "non_monotonic", "last_before_first", "noise"):
        offs = good.clone()
        if mutate == "past_end":
            offs[-1] = n + (1 << 24)
        elif mutate == "non_monotonic":
            offs[5] = n - 3
        elif mutate == "last_before_first":
            offs[-1] = 0
            offs[0] = 100
        else:
            offs = torch.from_numpy(rng.integers(0, 2 * n, 65).astype(np.int64)).cuda()
        buf = torch.full((65,), 0xAB, dtype=torch.uint8, device="cuda")
        _lib.check(lib.utf8v_cuda_validate_batch_async(d.data_ptr(), n, offs.data_ptr(), 64, buf.data_ptr(), st))
        torch.cuda.synchronize()
        assert int(buf[-1].item()) == 0xAB, mutate
    # the library still validates correctly afterwards
    assert (np.asarray(u8.validate_lookup_batch(b.data, b.d_offsets)) == b.expected).all()
    assert np.asarray(u8.validate_lookup_batch(d, good)).all()


def test_python_sharded_wrapper():
    import paper_2010_03090_b200 as u8
    from paper_2010_03090_b200 import configs
    d = configs.gen_c1(6 << 20, seed=3)
    h = d.cpu().numpy()
    for g in (1, 2, 5):
        assert u8.validate_lookup_sharded(h.tobytes(), g) is True
        bad = h.copy()
        bad[(3 << 20) + 1] = 0xFF
        assert u8.validate_lookup_sharded(bad, g) is False
    assert u8.validate_lookup_sharded(d, 4) is True  # device input: its own GPU


def test_byte_shards_first_error_positions():
    """verdict_sharded's device half: each shard's local first-error decode
    (utf8v_cuda_validate_verdict_lanes, device and host buffers), combined
    by MIN as the allreduce would, equals the whole stream's oracle
    (offset, kind) -- bad sequences straddling every shard edge, in the
    head, in the 3-byte tail, and a truncated stream end."""
    import torch
    from paper_2010_03090_b200 import configs, sharding
    from tests import _native as nat
    base = configs.gen_c1(2 << 20, seed=6).cpu().numpy()
    seqs = ([0xC0], [0xE0, 0x80, 0x80], [0xED, 0xA0, 0x80], [0xF4, 0x90, 0x80, 0x80], [0xF0, 0x80, 0x80, 0x80],
            [0xE2, 0x82, 0x41], [0xFF], [0x80, 0x80])
    cases = [base]
    for world in (2, 3, 8):
        for sh in sharding.plan(base.size, world)[1:3]:
            for delta in (-5, -3, -2, -1, 0, 1, 2, 3):
                for seq in seqs:
                    d = base.copy()
                    d[sh.start + delta:sh.start + delta + len(seq)] = seq
                    cases.append((world, d))
    t = base.copy()
    t[-2:] = [0xF0, 0x9F]
    cases += [(w, t) for w in (2, 3, 8)]
    for i, case in enumerate(cases[1:]):
        world, d = case
        ok, off, kind = nat.oracle_verdict(d.tobytes())
        want = None if ok else (off, kind)
        dev = torch.from_numpy(d).cuda()
        found = []
        for sh in sharding.plan(d.size, world):
            local = dev[sh.lo:sh.hi] if i % 2 == 0 else d[sh.lo:sh.hi].tobytes()
            e = sharding.shard_first_error(local, sh)
            if e is not None:
                found.append(e)
        got = min(found, key=lambda e: e[0] * 8 + e[1]) if found else None
        assert got == want, (world, i, got, want)
    # the whole valid stream: no rank reports anything
    for world in (1, 2, 8):
        for sh in sharding.plan(base.size, world):
            assert sharding.shard_first_error(base[sh.lo:sh.hi].tobytes(), sh) is None


def _verdict_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    from paper_2010_03090_b200 import configs, sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        base = configs.gen_c1(1 << 20, seed=17)
        out = []
        for case in range(6):
            d = base.clone()
            sh_edges = [s.start for s in sharding.plan(d.numel(), world)[1:]]
            if case > 0:  # a bad sequence straddling an edge, or deep inside a shard
                at = sh_edges[case % len(sh_edges)] + (case - 3) if case < 5 else 12345
                seq = [[0xE0, 0x80, 0x80], [0xF4, 0x90, 0x80, 0x80], [0xED, 0xA0, 0x80], [0x80], [0xC1]][case - 1]
                d[at:at + len(seq)] = torch.tensor(seq, dtype=torch.uint8, device=d.device)
            sh = sharding.plan(d.numel(), world)[rank]
            v = sharding.verdict_sharded(d[sh.lo:sh.hi], sh)
            out.append(None if v.valid() else (v.error.offset, int(v.error.kind)))
            if rank == 0:
                out[-1] = (out[-1], d.cpu().numpy().tobytes())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_verdict_sharded_multiprocess():
    """sharding.verdict_sharded end to end: 3 processes (gloo; they share the
    one GPU and no kernel waits on another rank), device shards, each rank's
    utf8v_cuda_validate_verdict_lanes + the allreduce(MIN): every rank gets
    the oracle's (offset, kind)."""
    import multiprocessing as mp
    import socket
    from tests import _native as nat
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_verdict_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (got0, data) in enumerate(res[0]):
        ok, off, kind = nat.oracle_verdict(data)
        want = None if ok else (off, kind)
        assert got0 == want, (i, got0, want)
        for r in range(1, world):
            assert res[r][i] == want, (r, i)
    assert any(g is not None for g, _ in res[0][1:])
