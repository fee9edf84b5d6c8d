"""The five BASELINE.json configs as device-resident synthetic inputs.

C0  64 MiB ASCII (0x20-0x7E + 2% 0x0A), seed 1            -> valid
C1  1 GiB valid mix, 0.4/0.2/0.3/0.1 lengths, seed 2        -> valid
C2  64 x 4 MiB segments, 32 with one injected error, seed 3 -> per-segment verdicts
C3  1 Mi records, lognormal(512, sigma=1) in [16, 64 KiB], 10% with an error, seed 4
C4  16 GiB mix, every k*n/8 edge inside a 3/4-byte character, seed 5;
    variant A valid, B overlong 1 byte after n/2, C truncated final character

Generation rules are pinned in DESIGN.md ("Synthetic inputs"); they run on
the GPU (csrc/gen.cu) and are deterministic.  Sizes can be scaled down for
tests with the same structure.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

MiB = 1 << 20
GiB = 1 << 30

C0 = dict(n=64 * MiB, seed=1)
C1 = dict(n=1 * GiB, seed=2)
C2 = dict(seg_len=4 * MiB, n_seg=64, seed=3)
C3 = dict(n_records=1 << 20, seed=4, sigma=1.0, median=512, min_len=16, max_len=64 * 1024)
C4 = dict(n=16 * GiB, seed=5)

RECIPE = {
    "rng": "splitmix64 (proj/include/utf8v/corpus.hpp:123-146)",
    "generation_chunk_bytes": 65536,
    "chunk_seed": "seed ^ 0xD1B54A32D192ED03*(j+1)",
    "plan_seed": "seed ^ 0xA24BAED4963EE407*tag (tag 2: C2, 3: C3 lengths, 4: C3 errors, 5: C4)",
    "mix": "below(10): 0-3 -> 1B, 4-5 -> 2B, 6-8 -> 3B, 9 -> 4B; random_code_point(kind)",
    "ascii": "below(100)<2 -> 0x0A else 0x20+below(95)",
    "c0": C0, "c1": C1, "c2": C2, "c3": C3, "c4": C4,
}


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def _alloc(n: int, device):
    torch = _torch()
    return torch.empty(max(n, 1), dtype=torch.uint8, device=device)[:n]


def gen_stream(n: int, seed: int, ascii_only: bool = False, device="cuda", stream=None):
    """Valid stream of exactly n bytes on `device` (torch.uint8 tensor)."""
    buf = _alloc(n, device)
    _lib.check(_lib.load().utf8v_gen_stream(buf.data_ptr() if n else None, n, seed, int(ascii_only),
                                            _stream_ptr(stream)))
    return buf


def gen_c0(n: int = C0["n"], seed: int = C0["seed"], device="cuda"):
    return gen_stream(n, seed, True, device)


def gen_c1(n: int = C1["n"], seed: int = C1["seed"], device="cuda"):
    return gen_stream(n, seed, False, device)


@dataclass
class Batch:
    data: object            # device torch.uint8 [n]
    offsets: np.ndarray     # host uint64 [n_records+1]
    d_offsets: object       # device int64 view of offsets
    expected: np.ndarray    # host uint8 [n_records] (1 valid)
    error_offsets: np.ndarray | None = None

    @property
    def n_records(self) -> int:
        return int(self.offsets.size - 1)

    @property
    def nbytes(self) -> int:
        return int(self.offsets[-1])


def gen_c2(seg_len: int = C2["seg_len"], n_seg: int = C2["n_seg"], seed: int = C2["seed"], device="cuda") -> Batch:
    torch = _torch()
    n = seg_len * n_seg
    buf = _alloc(n, device)
    exp = np.empty(n_seg, np.uint8)
    eoff = np.empty(n_seg, np.uint64)
    _lib.check(_lib.load().utf8v_gen_c2(buf.data_ptr(), seg_len, n_seg, seed, exp.ctypes.data, eoff.ctypes.data,
                                        _stream_ptr(None)))
    offs = (np.arange(n_seg + 1, dtype=np.uint64) * np.uint64(seg_len))
    d_off = torch.from_numpy(offs.view(np.int64).copy()).to(device)
    return Batch(buf, offs, d_off, exp, eoff)


def c3_offsets(n_records: int = C3["n_records"], seed: int = C3["seed"], sigma: float = C3["sigma"],
               median: int = C3["median"], min_len: int = C3["min_len"], max_len: int = C3["max_len"]) -> np.ndarray:
    offs = np.empty(n_records + 1, np.uint64)
    _lib.check(_lib.load().utf8v_gen_c3_offsets(n_records, seed, sigma, median, min_len, max_len, offs.ctypes.data))
    return offs


def gen_c3(n_records: int = C3["n_records"], seed: int = C3["seed"], sigma: float = C3["sigma"],
           median: int = C3["median"], min_len: int = C3["min_len"], max_len: int = C3["max_len"],
           device="cuda") -> Batch:
    torch = _torch()
    offs = c3_offsets(n_records, seed, sigma, median, min_len, max_len)
    n = int(offs[-1])
    buf = _alloc(n, device)
    d_off = torch.from_numpy(offs.view(np.int64).copy()).to(device)
    exp = np.empty(n_records, np.uint8)
    _lib.check(_lib.load().utf8v_gen_c3(buf.data_ptr(), d_off.data_ptr(), offs.ctypes.data, n_records, seed,
                                        exp.ctypes.data, _stream_ptr(None)))
    return Batch(buf, offs, d_off, exp)


def gen_c4(n: int = C4["n"], seed: int = C4["seed"], variant: int = 0, device="cuda"):
    """(device buffer, first error offset or None).  variant 0/1/2 = A/B/C."""
    buf = _alloc(n, device)
    err = C.c_uint64(0)
    _lib.check(_lib.load().utf8v_gen_c4(buf.data_ptr(), n, seed, variant, C.byref(err), _stream_ptr(None)))
    return buf, (None if err.value == (1 << 64) - 1 else int(err.value))
