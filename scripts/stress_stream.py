"""Randomised single-stream stress against the oracle, for a fixed wall-clock
budget: `python scripts/stress_stream.py SECONDS SEED`.  Each trial takes a
stream of 0 B .. 48 MiB from the C1 mix (starting anywhere, so possibly
inside a character), plants 0..4 errors (random bytes, lone leads,
truncations, garbage runs), and checks validate_lookup and
validate_lookup_verdict (device and host input: K1, the tracking K1 + K3)
a stream session fed in random pieces, and segment states of random pieces
merged in random order, against the oracle's verdict, offset and kind."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import paper_2010_03090_b200 as u8
from paper_2010_03090_b200 import configs
from tests import _native as nat

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
pool = configs.gen_c1(128 << 20, seed=seed).cpu().numpy()
t0 = time.time()
trials = invalid = 0
nbytes = 0
while time.time() - t0 < budget:
    n = int(rng.choice([0, 1, 2, 3, 5, 31, 33, 4095, 4097, 100_000, 1 << 20, 7_777_777, 48 << 20]))
    if n > 100_000 and rng.random() < 0.5:
        n = int(rng.integers(100_000, 48 << 20))
    a = int(rng.integers(0, pool.size - n - 1))
    h = pool[a:a + n].copy()
    for _ in range(int(rng.choice([0, 0, 1, 2, 4]))):
        if n == 0:
            break
        p = int(rng.integers(0, n))
        k = int(rng.integers(0, 4))
        if k == 0:
            h[p] = int(rng.integers(0x80, 0x100))
        elif k == 1:
            h[p] = int(rng.choice([0xC3, 0xE2, 0xF0, 0xF4]))
        elif k == 2:
            h[n - 1] = int(rng.choice([0xC3, 0xE2, 0xF0]))
        else:
            h[p:p + int(rng.integers(1, 64))] = 0xFF
    exp = nat.oracle_verdict(h, threads=16)
    want = (exp[0], None if exp[0] else (exp[1], exp[2]))
    d = torch.from_numpy(h).cuda() if n else torch.empty(0, dtype=torch.uint8, device="cuda")
    for src in (h, d):
        v = u8.validate_lookup_verdict(src)
        got = (v.valid(), None if v.valid() else (v.error.offset, int(v.error.kind)))
        assert got == want, (trials, n, a, got, want)
        assert u8.validate_lookup(src) is exp[0], (trials, n, a)
    with u8.LookupStream() as s:
        cuts = np.sort(rng.integers(0, n + 1, int(rng.integers(0, 6))))
        prev = 0
        for c in list(cuts) + [n]:
            s.feed(d[prev:int(c)] if rng.random() < 0.5 else h[prev:int(c)])
            prev = int(c)
        assert s.finish() is exp[0], (trials, n, a, cuts)
    # segment states of random pieces (host or device), merged in a random
    # order of adjacent pairs (utf8v_state combine is associative)
    cuts = [int(c) for c in np.sort(rng.integers(0, n + 1, int(rng.integers(0, 6))))]
    bounds = [0] + cuts + [n]
    states = [u8.segment_state(d[x:y] if rng.random() < 0.5 else h[x:y]) for x, y in zip(bounds, bounds[1:])]
    while len(states) > 1:
        i = int(rng.integers(0, len(states) - 1))
        states[i:i + 2] = [u8.combine_states(states[i], states[i + 1])]
    assert u8.state_valid(states[0]) is exp[0] and states[0].len == n, (trials, n, a, cuts)
    trials += 1
    nbytes += n
    invalid += int(not exp[0])
print(f"stream stress ok: {trials} streams ({invalid} invalid), {nbytes / 1e9:.1f} GB, "
      f"{time.time() - t0:.0f} s, seed {seed}", flush=True)
