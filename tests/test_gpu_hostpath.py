"""Host input over the bounded device ring (csrc/capi.cu validate_host_lanes):
each piece crosses PCIe with 16 bytes of halo on either side into one of
four device slots and is validated as soon as it lands; the verdict path
re-decodes only the first flagged piece.  Errors at every piece edge, lane
ranges, the small-input path and the HBM bound, against the oracle."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from tests import _native as nat

pytestmark = pytest.mark.gpu

MiB = 1 << 20
BAD = [[0xC0, 0x80], [0xE0, 0x80, 0x80], [0xED, 0xA0, 0x80], [0xF4, 0x90, 0x80, 0x80], [0x80], [0xF5],
       [0xE1, 0x41], [0xF0, 0x9F, 0x98]]


def _piece(n: int) -> int:  # capi.cu piece_size
    p = ((n // 8) + MiB - 1) & ~(MiB - 1)
    return min(max(p, 2 * MiB), 32 * MiB)


def _calls(buf: np.ndarray, pinned: bool):
    """(validate, verdict) through the C-ABI on host memory."""
    import torch
    from paper_2010_03090_b200 import _lib
    lib = _lib.load()
    if pinned:
        t = torch.from_numpy(buf).pin_memory()
        ptr, keep = t.data_ptr(), t
    else:
        keep = np.ascontiguousarray(buf)
        ptr = keep.ctypes.data
    ok = C.c_uint8(9)
    _lib.check(lib.utf8v_cuda_validate(ptr, buf.size, 0, C.byref(ok)))
    vok, off, kind = C.c_uint8(9), C.c_uint64(0), C.c_int(-1)
    _lib.check(lib.utf8v_cuda_validate_verdict(ptr, buf.size, 0, C.byref(vok), C.byref(off), C.byref(kind)))
    del keep
    return bool(ok.value), (True, None, None) if vok.value else (False, off.value, kind.value)


@pytest.mark.parametrize("pinned", [False, True])
def test_errors_at_every_piece_edge(pinned):
    from paper_2010_03090_b200 import configs
    n = 21 * MiB + 12345          # pieces of 3 MiB: 8 pieces, a short last one
    base = configs.gen_c1(n, seed=40).cpu().numpy()
    piece = _piece(n)
    assert _calls(base, pinned) == (True, (True, None, None))
    rng = np.random.default_rng(7)
    cases = 0
    for k in range(1, (n + piece - 1) // piece):
        edge = k * piece
        for d in range(-4, 5):
            seq = BAD[int(rng.integers(len(BAD)))]
            b = base.copy()
            b[edge + d:edge + d + len(seq)] = seq
            want = nat.oracle_verdict(b)
            got_ok, got_v = _calls(b, pinned)
            assert got_ok == want[0] and got_v == want, (k, d, seq, got_v, want)
            cases += 1
    # a truncated end, and two errors in different pieces (the first wins)
    b = base.copy()
    b[-1] = 0xE2
    assert _calls(b, pinned)[1] == nat.oracle_verdict(b)
    b = base.copy()
    b[5 * piece + 7] = 0xFF
    b[2 * piece - 1] = 0xC2
    want = nat.oracle_verdict(b)
    assert _calls(b, pinned)[1] == want and want[1] < 2 * piece + 3
    assert cases > 50


def test_small_path_boundary_sizes():
    from paper_2010_03090_b200 import configs
    src = configs.gen_c1(2 * MiB, seed=41).cpu().numpy()
    for n in (1, 2, 3, 4, 5, 31, 32, 33, 4095, 4096, MiB - 1, MiB, MiB + 1, MiB + 17):
        b = src[:n].copy()
        want = nat.oracle_verdict(b)
        for pinned in (False, True):
            got_ok, got_v = _calls(b, pinned)
            assert got_ok == want[0] and got_v == want, (n, pinned)
        if n > 8:
            b[n // 2] = 0xC1
            want = nat.oracle_verdict(b)
            assert _calls(b, False)[1] == want, n


def test_host_lane_ranges_compose():
    """utf8v_cuda_validate_lanes over host input: any split of the lanes into
    ranges ORs to the whole (pieces holding none of a range are skipped)."""
    from paper_2010_03090_b200 import _lib, configs
    lib = _lib.load()
    n = 9 * MiB + 3
    base = configs.gen_c1(n, seed=42).cpu().numpy()
    rng = np.random.default_rng(3)
    for trial in range(12):
        b = base.copy()
        if trial % 3:
            at = int(rng.integers(0, n))
            b[at] = 0xFF
        want = 0 if nat.oracle_verdict(b)[0] else 1
        cuts = sorted({0, n + 3, *(int(x) for x in rng.integers(0, n + 3, size=4))})
        got = 0
        for lo, hi in zip(cuts, cuts[1:]):
            f = C.c_uint32(0)
            _lib.check(lib.utf8v_cuda_validate_lanes(b.ctypes.data, n, lo, hi, 0, C.byref(f)))
            got |= int(f.value != 0)
        assert got == want, trial


def test_host_input_hbm_is_bounded():
    """16 GiB of host input validated with at most 256 MiB of HBM held by the
    call (the ring is 4 x (32 MiB + 32 B)); the verdict is exact."""
    import torch
    from paper_2010_03090_b200 import _lib
    lib = _lib.load()
    n = 16 << 30
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h = host.numpy()
    assert nat.oracle().orc_gen_stream(h.ctypes.data, n, 5, 0, 16) == 0
    torch.cuda.synchronize()
    lib.utf8v_cuda_release_thread_resources()
    free0, _ = torch.cuda.mem_get_info()
    ok = C.c_uint8(9)
    _lib.check(lib.utf8v_cuda_validate(host.data_ptr(), n, 0, C.byref(ok)))
    free1, _ = torch.cuda.mem_get_info()
    assert ok.value == 1
    assert free0 - free1 <= 256 << 20, (free0 - free1) >> 20
    h[n - 2] = 0xF0  # truncated 4-byte character at the end
    vok, off, kind = C.c_uint8(9), C.c_uint64(0), C.c_int(-1)
    _lib.check(lib.utf8v_cuda_validate_verdict(host.data_ptr(), n, 0, C.byref(vok), C.byref(off), C.byref(kind)))
    free2, _ = torch.cuda.mem_get_info()
    assert (vok.value, off.value, kind.value) == (0, n - 2, 1)
    assert free0 - free2 <= 256 << 20
    lib.utf8v_cuda_release_thread_resources()
    free3, _ = torch.cuda.mem_get_info()
    assert free3 >= free0 - (4 << 20)


def test_release_frees_the_shard_workers_contexts():
    """utf8v_cuda_validate_sharded runs its shards on persistent worker
    threads; utf8v_cuda_release_thread_resources frees their contexts too."""
    import torch
    from paper_2010_03090_b200 import _lib, configs
    lib = _lib.load()
    h = configs.gen_c1(96 * MiB, seed=44).cpu().numpy()
    lib.utf8v_cuda_release_thread_resources()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    ok = C.c_uint8(9)
    _lib.check(lib.utf8v_cuda_validate_sharded(h.ctypes.data, h.size, 3, 0, C.byref(ok)))
    assert ok.value == 1
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 >= 3 * (2 * MiB), "the workers hold their device rings"
    lib.utf8v_cuda_release_thread_resources()
    free2, _ = torch.cuda.mem_get_info()
    assert free2 >= free0 - (4 << 20), ((free0 - free2) >> 20)
