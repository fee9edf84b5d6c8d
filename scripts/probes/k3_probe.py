"""Verdict-path cost vs the first error's position (1 GiB C1).  With the
tracking K1 (first flagged step recorded in the same pass) the cost no longer
depends on the position; the numbers DESIGN.md quotes for 25/50/75/100 % are
from the earlier design, whose second kernel rescanned the prefix."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import paper_2010_03090_b200 as u8
from paper_2010_03090_b200 import configs

d = configs.gen_c1()
n = d.numel()
st = torch.cuda.current_stream()


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


print(f"valid: {t(lambda: u8.validate_lookup_verdict(d)):.1f} us")
print(f"bool:  {t(lambda: u8.validate_lookup(d)):.1f} us")
for frac in (0.0, 0.25, 0.5, 0.75, 0.999):
    at = int(n * frac) + 100
    orig = int(d[at].item())
    d[at] = 0xC0
    us = t(lambda: u8.validate_lookup_verdict(d))
    v = u8.validate_lookup_verdict(d)
    print(f"error at {frac:5.3f}: {us:.1f} us  offset={v.error.offset}")
    d[at] = orig
