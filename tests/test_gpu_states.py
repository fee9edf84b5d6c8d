"""Composable segment states on the B200: segment states
(K1 over a segment's interior lanes), per-record states of a batch (K2 in
state mode + the record-edge pass), the in-order device reduction, and
out-of-order stitching of independently validated pieces -- each against the
CPU model (tests/test_states.py::leaf) and the oracle."""
from __future__ import annotations

import numpy as np
import pytest

from tests import _native as nat
from tests.test_states import fold_random_tree, leaf

pytestmark = pytest.mark.gpu
MiB = 1 << 20


def _u8():
    import paper_2010_03090_b200 as u8
    return u8


def test_segment_states_equal_cpu_model():
    import torch
    from paper_2010_03090_b200 import configs
    u8 = _u8()
    base = configs.gen_c1(3 * MiB, seed=50).cpu().numpy()
    rng = np.random.default_rng(1)
    sizes = [0, 1, 2, 3, 4, 5, 6, 7, 31, 32, 33, 4096, 65537, MiB - 3, MiB + 5, 3 * MiB - 1]
    for n in sizes:
        for trial in range(3):
            a = int(rng.integers(0, base.size - n + 1))
            seg = base[a:a + n].copy()
            if trial == 2 and n > 8:
                seg[int(rng.integers(3, n - 1))] = 0xFF
            want = leaf(seg.tobytes())
            assert u8.segment_state(seg.tobytes()) == want, (n, trial)                 # host
            assert u8.segment_state(torch.from_numpy(seg).cuda()) == want, (n, trial)  # device


def test_batch_states_equal_cpu_model_and_reduce():
    import ctypes as C
    import torch
    from paper_2010_03090_b200 import _lib, configs
    u8 = _u8()
    lib = _lib.load()
    rng = np.random.default_rng(2)
    for kind in ("c3", "tiny", "mixed"):
        if kind == "c3":
            b = configs.gen_c3(n_records=20000, seed=4)
            data, offs = b.data.cpu().numpy(), b.offsets
        else:
            hi = 13 if kind == "tiny" else 5000
            lens = rng.integers(0, hi, size=3000)
            offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
            base = configs.gen_c1(int(offs[-1]) + 64, seed=51).cpu().numpy()
            data = base[:int(offs[-1])].copy()
            for at in rng.integers(0, data.size, size=40):
                data[int(at)] = rng.choice([0x80, 0xC0, 0xE0, 0xF5, 0xED])
        got_h = u8.batch_states(data, offs)
        dd = torch.from_numpy(data).cuda()
        got_d = u8.batch_states(dd, torch.from_numpy(offs.view(np.int64)).cuda())
        assert np.array_equal(got_h, got_d)
        for r in range(offs.size - 1):
            want = leaf(data[int(offs[r]):int(offs[r + 1])].tobytes())
            got = u8.SegmentState.from_buffer_copy(got_h[r:r + 1].tobytes())
            assert got == want, (kind, r, got, want)
        # the records are consecutive segments of one stream: their fold is
        # the stream's verdict, on the host and with the device reduction
        want_stream = nat.oracle_verdict(data)[0] if data.size else True
        assert u8.state_valid(u8.fold_states(got_h)) == want_stream
        d_states = torch.from_numpy(got_h.view(np.uint8).copy()).cuda()
        d_out = torch.zeros(24, dtype=torch.uint8, device="cuda")
        _lib.check(lib.utf8v_cuda_states_reduce_async(d_states.data_ptr(), got_h.size, d_out.data_ptr(),
                                                      torch.cuda.current_stream().cuda_stream))
        red = u8.SegmentState.from_buffer_copy(d_out.cpu().numpy().tobytes())
        assert red == u8.fold_states(got_h), kind


def test_out_of_order_stitching_matches_oracle():
    """Pieces of one stream validated independently, in a shuffled order and
    on host or device, merged in random groupings: the oracle's verdict."""
    import torch
    from paper_2010_03090_b200 import configs
    u8 = _u8()
    base = configs.gen_c1(8 * MiB, seed=52).cpu().numpy()
    rng = np.random.default_rng(3)
    for trial in range(24):
        b = base.copy()
        cuts = sorted(int(x) for x in rng.integers(0, b.size + 1, size=int(rng.integers(1, 9))))
        if trial % 4:
            c = cuts[int(rng.integers(len(cuts)))]
            seq = [[0xE0, 0x80, 0x80], [0xF0, 0x9F], [0x80], [0xC1, 0x81], [0xED, 0xA0, 0x80]][trial % 5]
            at = min(max(c + int(rng.integers(-3, 3)), 0), b.size - len(seq))
            b[at:at + len(seq)] = seq
        parts = [b[x:y] for x, y in zip([0] + cuts, cuts + [b.size])]
        order = rng.permutation(len(parts))
        states = [None] * len(parts)
        for i in order:  # validated in a shuffled order
            p = parts[i]
            states[i] = u8.segment_state(torch.from_numpy(p.copy()).cuda() if i % 2 else p.tobytes())
        want = nat.oracle_verdict(b)[0]
        assert u8.state_valid(fold_random_tree(states, rng)) == want, trial
