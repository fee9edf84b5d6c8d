"""Randomised batch stress against the oracle (K2 and K2L through the public
API), for a fixed wall-clock budget: `python scripts/stress_batch.py SECONDS SEED`.
Each trial draws a record count, a length distribution (lognormal with a
random median and spread, empty records mixed in), content from the C1 mix,
a per-record corruption rate and kinds (random byte, lead at the record end,
stray continuation at its start, a cut inside a character), an alignment
shift and device or host input; every verdict is compared with the oracle.
About 30 % of the batches also check per-record segment states (a sample
against the CPU model, the device fold of all of them against the oracle's
verdict of the records' concatenation)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import paper_2010_03090_b200 as u8
from paper_2010_03090_b200 import configs
from paper_2010_03090_b200 import _lib
from tests import _native as nat
from tests.test_states import leaf

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
pool = configs.gen_c1(256 << 20, seed=seed).cpu().numpy()
t0 = time.time()
trials = records = invalid = states_checked = 0
paths = {"K2": 0, "K2L": 0}
while time.time() - t0 < budget:
    n_rec = int(rng.choice([1, 2, 7, 64, 500, 2048, 5000, 50000, 200000]))
    median = float(np.exp(rng.uniform(np.log(2), np.log(1 << 18))))
    lens = rng.lognormal(np.log(median), rng.uniform(0.2, 2.0), n_rec).astype(np.int64)
    lens[rng.random(n_rec) < rng.uniform(0, 0.2)] = 0
    lens = np.minimum(lens, 1 << 22)
    total = int(lens.sum())
    if total > pool.size - 64 or total == 0:
        continue
    start = int(rng.integers(0, pool.size - total - 32))
    lead = int(rng.integers(0, 40))
    data = pool[start - min(start, lead): start + total + int(rng.integers(0, 40))].copy()
    lead = min(start, lead)
    offs = np.zeros(n_rec + 1, np.int64)
    offs[1:] = np.cumsum(lens)
    offs += lead
    if rng.random() < 0.5:  # cuts moved to character boundaries: mostly valid records
        hi = lead + total
        for _ in range(3):
            inside = (offs < hi) & ((data[np.minimum(offs, data.size - 1)] & 0xC0) == 0x80)
            offs[inside] += 1
        offs = np.maximum.accumulate(np.minimum(offs, hi))
    offs = offs.astype(np.uint64)
    rate = float(rng.choice([0.0, 0.001, 0.05, 0.3]))
    for r in np.nonzero(rng.random(n_rec) < rate)[0]:
        a, b = int(offs[r]), int(offs[r + 1])
        if b <= a:
            continue
        k = int(rng.integers(0, 4))
        if k == 0:
            data[int(rng.integers(a, b))] = int(rng.integers(0x80, 0x100))
        elif k == 1:
            data[b - 1] = int(rng.choice([0xC2, 0xE1, 0xF1]))
        elif k == 2:
            data[a] = 0x80 | int(rng.integers(0, 0x40))
        else:
            data[int(rng.integers(a, b))] = 0xED
    want = nat.oracle_batch(data, offs)
    if rng.random() < 0.5:
        shift = int(rng.integers(0, 32))
        buf = torch.zeros(data.size + 64, dtype=torch.uint8, device="cuda")
        buf[shift:shift + data.size] = torch.from_numpy(data).cuda()
        got = u8.validate_lookup_batch(buf[shift:shift + data.size],
                                       torch.from_numpy(offs.view(np.int64)).cuda())
    else:
        got = u8.validate_lookup_batch(data, offs)
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        print(f"MISMATCH trial {trials}: n_rec={n_rec} median={median:.0f} rate={rate} lead={lead} "
              f"records {bad[:10]}", flush=True)
        sys.exit(1)
    if rng.random() < 0.3:
        # per-record segment states (K2 in state mode): a sample equals the
        # CPU model, and the in-order device fold of all of them is the
        # verdict of the records' concatenation
        st = u8.batch_states(data, offs)
        for r in rng.integers(0, n_rec, size=min(n_rec, 100)):
            rec = data[int(offs[r]):int(offs[r + 1])].tobytes()
            assert bytes(u8.SegmentState.from_buffer_copy(st[r:r + 1].tobytes())) == bytes(leaf(rec)), (trials, r)
        d_st = torch.from_numpy(st.view(np.uint8).copy()).cuda()
        d_out = torch.zeros(24, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().utf8v_cuda_states_reduce_async(d_st.data_ptr(), n_rec, d_out.data_ptr(),
                                                              torch.cuda.current_stream().cuda_stream))
        whole = u8.SegmentState.from_buffer_copy(d_out.cpu().numpy().tobytes())
        cat = data[int(offs[0]):int(offs[-1])]
        assert u8.state_valid(whole) == (nat.oracle_verdict(cat, threads=16)[0] if cat.size else True), trials
        states_checked += 1
    large = n_rec <= 2048 and data.size // n_rec >= (64 << 10)
    paths["K2L" if large else "K2"] += 1
    trials += 1
    records += n_rec
    invalid += int((want == 0).sum())
print(f"stress ok: {trials} batches ({paths}), {records} records ({invalid} invalid), "
      f"{states_checked} with per-record states, {time.time() - t0:.0f} s, seed {seed}", flush=True)
