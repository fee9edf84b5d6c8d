"""The device SWAR formula (csrc/utf8v_swar.h), compiled for the CPU by the
test helper, against the oracle: exhaustive short inputs at every word
alignment, all pairs at the reference's seam offsets, mutation corpora, and
the record-bounded (batch) variant."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from tests import _native as nat


@pytest.mark.parametrize("align", [0, 1, 2, 3])
def test_exhaustive_length_0_to_3(align):
    # acceptance.cpp:74-113: all 16,843,009 inputs, verdict and the
    # first-flagged-lane bound E <= L <= E+3 used by the position kernel.
    ck, mm, bv = C.c_uint64(), C.c_uint64(), C.c_uint64()
    nat.swar().swar_exhaustive(align, 3, C.byref(ck), C.byref(mm), C.byref(bv))
    assert ck.value == 16843009
    assert mm.value == 0
    assert bv.value == 0


@pytest.mark.parametrize("offset", [0, 15, 16, 31, 32, 63, 64])
def test_all_pairs_at_seam_offsets(offset):
    for align in range(4):
        assert nat.swar().swar_pairs(offset, align) == 0


def test_generated_corpora_and_positions():
    S = nat.swar()
    for seed in range(1, 3001):
        for target in (16, 64, 200):
            items = [nat.generate_valid(15, target, seed)] + [nat.generate_invalid(15, target, seed, s) for s in range(6)]
            for data in items:
                ok, eoff, _ = nat.oracle_verdict(data)
                for align in (0, 3):
                    L = S.swar_first_lane(data, len(data), align)
                    assert (L == (1 << 64) - 1) == ok
                    if not ok:
                        assert eoff <= L <= eoff + 3


def _batch(parts):
    lens = np.array([len(p) for p in parts], np.uint64)
    offs = np.zeros(len(parts) + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    data = np.frombuffer(b"".join(parts) or b"\0", np.uint8)[: int(offs[-1])].copy()
    return data, offs


def test_k2_decomposition_matches_per_record_oracle():
    rng = np.random.default_rng(11)
    S = nat.swar()
    for trial in range(300):
        parts = []
        for _ in range(int(rng.integers(1, 30))):
            k = int(rng.integers(0, 5))
            if k == 0:
                parts.append(b"")
            elif k == 1:
                parts.append(bytes(rng.integers(0, 256, int(rng.integers(1, 5)), dtype=np.uint8)))
            elif k == 2:
                parts.append(nat.generate_valid(15, int(rng.integers(1, 30)), int(rng.integers(1, 1 << 30))))
            elif k == 3:
                parts.append(nat.generate_invalid(15, int(rng.integers(1, 30)), int(rng.integers(1, 1 << 30)),
                                                  int(rng.integers(0, 6))))
            else:
                parts.append(bytes([0xF0, 0x9F, 0x98])[: int(rng.integers(1, 4))])
        data, offs = _batch(parts)
        want = np.array([nat.oracle_verdict(p)[0] for p in parts], np.uint8)
        got = np.empty(len(parts), np.uint8)
        for align in range(4):
            S.swar_batch_decomp(data.ctypes.data if data.size else None, offs.ctypes.data, len(parts), align,
                                got.ctypes.data)
            assert np.array_equal(got, want), ("decomp", trial, align, parts)


def test_bit_planes_transpose():
    S = nat.swar()
    S.swar_planes_check.restype = C.c_uint64
    S.swar_planes_check.argtypes = [C.c_uint64, C.c_uint64]
    assert S.swar_planes_check(7, 20000) == 0


def test_bit_sliced_form_equals_swar_form_lane_for_lane():
    """utf8v_bits.h (planes) == utf8v_swar.h lead form on every lane class at
    every chunk position, plus fuzz (same per-lane predicate, so the proofs of
    test_exhaustive_* carry over)."""
    S = nat.swar()
    S.swar_bits_check.restype = C.c_uint64
    S.swar_bits_check.argtypes = [C.c_uint64, C.c_uint64]
    assert S.swar_bits_check(11, 200000) == 0


def test_stream_stitching_equals_whole_stream():
    """utf8v_stream.h: any split of a stream into pieces (empty, 1..8-byte,
    large), stitched through the carry, gives the whole stream's verdict --
    on generated valid/invalid corpora and on all short inputs around a cut."""
    S = nat.swar()
    S.swar_stream_split.restype = C.c_int
    S.swar_stream_split.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t]
    rng = np.random.default_rng(3)
    checked = 0
    for seed in range(1, 120):
        for strategy in (None, 0, 1, 2, 3, 4, 5, 6):
            data = nat.generate_valid(0xF, 200 + seed * 7, seed) if strategy is None else \
                nat.generate_invalid(0xF, 200 + seed * 7, seed, strategy)
            if data is None:
                continue
            buf = np.frombuffer(data, dtype=np.uint8).copy()
            want = nat.oracle_verdict(bytes(buf))[0]
            for _ in range(6):
                k = int(rng.integers(0, 12))
                cuts = np.sort(rng.integers(0, len(buf) + 1, size=k)).astype(np.uint64)
                got = S.swar_stream_split(buf.ctypes.data, len(buf), cuts.ctypes.data, len(cuts))
                assert bool(got) == bool(want), (seed, strategy, cuts.tolist())
                checked += 1
    # Every 4-byte window of "interesting" bytes, cut at every position.
    hot = [0x41, 0x80, 0xA0, 0xBF, 0xC2, 0xE0, 0xED, 0xF0, 0xF4]
    for a in hot:
        for b in hot:
            for c in hot:
                for d in hot:
                    buf = np.array([0x41, a, b, c, d, 0x41, 0x41, 0x41, 0x41], dtype=np.uint8)
                    want = nat.oracle_verdict(bytes(buf))[0]
                    for cut in range(len(buf) + 1):
                        cuts = np.array([cut], dtype=np.uint64)
                        got = S.swar_stream_split(buf.ctypes.data, len(buf), cuts.ctypes.data, 1)
                        assert bool(got) == bool(want), (buf.tolist(), cut)
                        checked += 1
    assert checked > 5000


def test_bit_sliced_permuted_form_equals_natural_form():
    """K1's permuted-order plane form (no PRMT gather) flags exactly the lanes
    of the natural-order form, bit pos(i) <-> lane i, on every lane class at
    every chunk position plus fuzz."""
    S = nat.swar()
    S.swar_bits_perm_check.restype = C.c_uint64
    S.swar_bits_perm_check.argtypes = [C.c_uint64, C.c_uint64]
    assert S.swar_bits_perm_check(13, 300000) == 0


def test_k2_boundary_decomposition_adversarial():
    """K2 = unbounded lane flags (boundary lanes skipped) + u8v_boundary_errors
    at every record start: equal to per-record validation on records of 0..6
    bytes drawn from the bytes that matter at a boundary (continuations of
    each range, every rare lead, ASCII), at every word alignment."""
    rng = np.random.default_rng(29)
    S = nat.swar()
    alphabet = np.array([0x41, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2, 0xDF, 0xE0,
                         0xE1, 0xED, 0xEF, 0xF0, 0xF1, 0xF4, 0xF5, 0xFF], np.uint8)
    for trial in range(2000):
        parts = [bytes(rng.choice(alphabet, int(rng.integers(0, 7)))) for _ in range(int(rng.integers(1, 12)))]
        data, offs = _batch(parts)
        want = np.array([nat.oracle_verdict(p)[0] for p in parts], np.uint8)
        got = np.empty(len(parts), np.uint8)
        for align in range(4):
            S.swar_batch_decomp(data.ctypes.data if data.size else None, offs.ctypes.data, len(parts), align,
                                got.ctypes.data)
            assert np.array_equal(got, want), (trial, align, parts)
    # whole characters at the edges of the ranges and their prefixes: records
    # that are valid, truncated at either end, or split across a boundary
    chars = [b"A", b"\xC2\x80", b"\xDF\xBF", b"\xE0\xA0\x80", b"\xED\x9F\xBF", b"\xEF\xBF\xBF",
             b"\xF0\x90\x80\x80", b"\xF4\x8F\xBF\xBF"]
    n_valid = 0
    for trial in range(2000):
        parts = []
        for _ in range(int(rng.integers(1, 10))):
            rec = b"".join(chars[int(i)] for i in rng.integers(0, len(chars), int(rng.integers(0, 3))))
            cut = int(rng.integers(0, 3))
            if cut == 1 and rec:
                rec = rec[int(rng.integers(1, len(rec) + 1)):]     # starts mid-character
            elif cut == 2 and rec:
                rec = rec[: int(rng.integers(0, len(rec)))]        # ends mid-character
            parts.append(rec)
        data, offs = _batch(parts)
        want = np.array([nat.oracle_verdict(p)[0] for p in parts], np.uint8)
        n_valid += int(want.sum())
        got = np.empty(len(parts), np.uint8)
        for align in range(4):
            S.swar_batch_decomp(data.ctypes.data if data.size else None, offs.ctypes.data, len(parts), align,
                                got.ctypes.data)
            assert np.array_equal(got, want), (trial, align, parts)
    assert n_valid > 2000  # both kinds well represented
