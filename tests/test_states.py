"""Composable segment states (csrc/utf8v_state.h, utf8v_state_combine /
utf8v_state_valid) on the CPU: leaf states are computed with the device
lane predicate compiled by gcc (tests/cpp/swar_host.c: swar_lanes over a
segment's interior lanes [3, len-1)); the product library's host combine
folds them in random groupings; the verdict must equal the oracle's
(proj/src/oracle.cpp:10-44) for every split.  The reference's claim being
restated: the fold is associative, so a stream can be validated in segments
(proj/include/utf8v/fsm.hpp:15-20)."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from tests import _native as nat


def leaf(seg: bytes):
    import paper_2010_03090_b200 as u8
    s = u8.SegmentState()
    n = len(seg)
    s.len = n
    if n > 4:
        a = np.frombuffer(seg, np.uint8)
        s.flag = nat.swar().swar_lanes(a.ctypes.data, n, 3, n - 1)
    k = min(n, 4)
    for i in range(k):
        s.head[i] = seg[i]
        s.tail[4 - k + i] = seg[n - k + i]
    return s


def fold_random_tree(states, rng):
    """Combine adjacent states in a random order until one is left."""
    import paper_2010_03090_b200 as u8
    xs = list(states)
    if not xs:
        return u8.empty_state()
    while len(xs) > 1:
        i = int(rng.integers(0, len(xs) - 1))
        xs[i:i + 2] = [u8.combine_states(xs[i], xs[i + 1])]
    return xs[0]


def corpora(rng):
    L = nat.oracle()
    for kinds in (1, 3, 7, 15):
        for size in (1, 5, 37, 300):
            buf = np.zeros(size + 8, np.uint8)
            m = L.orc_generate_valid(kinds, size, int(rng.integers(1 << 62)), buf.ctypes.data, buf.size)
            b = bytes(buf[:m])
            yield b
            for _ in range(6):  # one mutated byte
                x = bytearray(b)
                if x:
                    x[int(rng.integers(len(x)))] = int(rng.integers(256))
                yield bytes(x)


def test_random_splits_and_groupings_match_oracle():
    import paper_2010_03090_b200 as u8
    rng = np.random.default_rng(11)
    checked = 0
    for b in corpora(rng):
        want = nat.oracle_verdict(np.frombuffer(b, np.uint8))[0] if b else True
        assert u8.state_valid(leaf(b)) == want
        for _ in range(12):
            k = int(rng.integers(1, 8))
            cuts = sorted(int(x) for x in rng.integers(0, len(b) + 1, size=k))
            parts = [b[x:y] for x, y in zip([0] + cuts, cuts + [len(b)])]
            got = fold_random_tree([leaf(p) for p in parts], rng)
            assert u8.state_valid(got) == want, (b.hex(), cuts)
            assert got.len == len(b)
            checked += 1
    assert checked > 1000


BOUNDARY_BYTES = [0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC2, 0xDF, 0xE0, 0xE1, 0xED,
                  0xEF, 0xF0, 0xF1, 0xF4, 0xF5]


def test_every_short_window_cut_everywhere():
    """All 3-byte strings over the boundary-relevant bytes, padded on both
    sides with text, cut into single bytes: every seam condition of
    combine() (short segments, segments of 1-3 bytes on either side)."""
    import paper_2010_03090_b200 as u8
    rng = np.random.default_rng(5)
    for w in itertools.product(BOUNDARY_BYTES, repeat=3):
        b = b"ab" + bytes(w) + b"\xc3\xa9z"
        want = nat.oracle_verdict(np.frombuffer(b, np.uint8))[0]
        # all single bytes, folded left to right and in a random tree
        leaves = [leaf(b[i:i + 1]) for i in range(len(b))]
        assert u8.state_valid(u8.fold_states(leaves)) == want, bytes(w).hex()
        assert u8.state_valid(fold_random_tree(leaves, rng)) == want, bytes(w).hex()


def test_combine_is_associative_and_empty_is_identity():
    import paper_2010_03090_b200 as u8
    rng = np.random.default_rng(9)
    pool = [bytes(rng.integers(0, 256, size=int(rng.integers(0, 9)), dtype=np.uint8)) for _ in range(60)]
    pool += [b"", b"\xe0", b"\xa0\x80", b"\xf0\x9f", b"\x98\x80", b"abc"]
    e = u8.empty_state()
    for _ in range(3000):
        a, b, c = (leaf(pool[int(i)]) for i in rng.integers(0, len(pool), size=3))
        l = u8.combine_states(u8.combine_states(a, b), c)
        r = u8.combine_states(a, u8.combine_states(b, c))
        assert l == r
        assert u8.combine_states(a, e) == a and u8.combine_states(e, a) == a


def test_state_struct_layout():
    import ctypes as C
    import paper_2010_03090_b200 as u8
    assert C.sizeof(u8.SegmentState) == 24
    s = leaf(b"hello \xe2\x82\xac")
    assert s.len == 9 and bytes(s.head) == b"hell" and bytes(s.tail) == b" \xe2\x82\xac"
    s = leaf(b"\xc3")
    assert bytes(s.head) == b"\xc3\x00\x00\x00" and bytes(s.tail) == b"\x00\x00\x00\xc3"
    assert not u8.state_valid(s)
