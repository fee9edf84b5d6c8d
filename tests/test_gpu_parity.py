"""GPU parity: the CUDA path (through the C-ABI) vs the oracle, on the
reference's own test vectors (proj/tests/test_lookup.cpp, acceptance.cpp) and
on seeded inputs.  Bit-exact: verdicts, and (offset, kind) where reported."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2010_03090_b200 as u8
from paper_2010_03090_b200 import configs
from tests import _native as nat

pytestmark = pytest.mark.gpu


def B(*xs):
    return bytes(xs)


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


@pytest.fixture(scope="module")
def cuda():
    return u8.lookup_backends()[0]


# ---- roster & lanes: test_lookup.cpp:34-187 --------------------------------
def test_roster_well_formed():
    bs = u8.lookup_backends()
    assert len(bs) >= 1
    for i in range(len(bs) - 1):
        assert bs[i].width >= bs[i + 1].width
    for b in bs:
        assert u8.find_lookup_backend(b.name) is b
        assert b.width >= 32
    assert u8.find_lookup_backend("neon") is None
    assert u8.find_lookup_backend("") is None


@pytest.mark.parametrize("seed", [1, 0xDEADBEEF, 0x123456789ABCDEF])
def test_ops_self_test(cuda, seed):
    assert cuda.ops_self_test(seed)


def test_worked_example_classification(cuda):
    example = B(0x39, 0xC3, 0xA7, 0xE9, 0x8F, 0xA1, 0xF0, 0x9F, 0x98, 0x80, 0x00)
    final = B(0x00, 0x00, 0x00, 0x00, 0x00, 0x80, 0x00, 0x00, 0x80, 0x80, 0x00)
    w = cuda.width
    out = cuda.classify_lanes(example + bytes(w - len(example)), bytes(w))
    assert out == final + bytes(w - len(final))


def test_classification_silent_on_ascii(cuda):
    w = cuda.width
    assert cuda.classify_lanes(b"A" * w, b"A" * w) == bytes(w)


def test_lanes_match_oracle_on_random_vectors(cuda):
    rng = np.random.default_rng(7)
    w = cuda.width
    import ctypes as C
    O = nat.oracle()
    for _ in range(200):
        a = rng.integers(0, 256, w, dtype=np.uint8).tobytes()
        p = rng.integers(0, 256, w, dtype=np.uint8).tobytes()
        for fn, ofn in ((cuda.classify_lanes, O.orc_classify_lanes), (cuda.length_error_lanes, O.orc_length_error_lanes)):
            want = (C.c_uint8 * w)()
            ofn(a, p, want, w)
            assert fn(a, p) == bytes(want)
        want = (C.c_uint8 * w)()
        O.orc_incomplete_lanes(a, want, w)
        assert cuda.incomplete_lanes(a) == bytes(want)


def test_all_pairs_across_the_seam(cuda):
    # test_lookup.cpp:92-117 -- lane 0 with the pair (previous[w-1], input[0]).
    w = cuda.width
    prev = bytearray(b"A" * w)
    inp = bytearray(b"A" * w)
    bad = []
    for b1 in range(0, 256, 1):
        prev[w - 1] = b1
        for b2 in range(256):  # all 65,536 pairs, one GPU round trip each (as the reference test)
            inp[0] = b2
            out = cuda.classify_lanes(bytes(inp), bytes(prev))[0]
            exp_invalid = bool(nat.oracle().orc_pair_always_invalid(b1, b2))
            exp_pair = (b1 & 0xC0) == 0x80 and (b2 & 0xC0) == 0x80
            if bool(out & 0x7F) != exp_invalid or bool(out & 0x80) != exp_pair:
                bad.append((b1, b2, out))
    assert not bad


def test_length_cross_check(cuda):
    w = cuda.width

    def run(head):
        inp = bytearray(b"\x39" * w)
        inp[: len(head)] = bytes(head)
        return any(cuda.length_error_lanes(bytes(inp), bytes(w)))

    assert not run([0xE9, 0x8F, 0xA1])
    assert not run([0xF0, 0x9F, 0x98, 0x80])
    assert run([0xE9, 0x8F, 0x39])
    assert run([0x39, 0x80, 0x80])
    assert run([0xF0, 0x9F, 0x98])


def test_incomplete_residues(cuda):
    w = cuda.width
    assert not any(cuda.incomplete_lanes(b"\x39" * w))
    c = bytearray(b"\x39" * w); c[w - 3:] = B(0xE9, 0x8F, 0xA1)
    assert not any(cuda.incomplete_lanes(bytes(c)))
    t = bytearray(b"\x39" * w); t[w - 3:] = B(0xF0, 0x9F, 0x98)
    assert any(cuda.incomplete_lanes(bytes(t)))
    l = bytearray(b"\x39" * w); l[w - 1] = 0xC2
    out = cuda.incomplete_lanes(bytes(l))
    assert out[w - 1] == 0xC2 ^ 0xBF and out.count(0) == w - 1
    h = bytearray(b"\x39" * w); h[w - 1] = 0xF5
    assert any(cuda.incomplete_lanes(bytes(h)))


# ---- whole-buffer verdicts: test_lookup.cpp:189-285 -------------------------
KNOWN = [
    (b"", True),
    (B(0x39, 0xC3, 0xA7, 0xE9, 0x8F, 0xA1, 0xF0, 0x9F, 0x98, 0x80, 0x00), True),
    (B(0xED, 0xB8, 0x80), False),
    (B(0x80), False),
    (B(0xC3), False),
    (B(0xF4, 0x8F, 0xBF, 0xBF), True),
    (B(0xF4, 0x90, 0x80, 0x80), False),
]


@pytest.mark.parametrize("data,expected", KNOWN)
def test_known_buffers(data, expected):
    assert u8.validate_lookup(data) is expected
    assert u8.validate_lookup_fallback(data) is expected


def test_nullptr_zero_is_valid():
    import ctypes as C
    lib = u8._lib.load()
    out = C.c_uint8(0)
    assert lib.utf8v_cuda_validate(None, 0, 0, C.byref(out)) == 0 and out.value == 1


def test_errors_survive_clean_blocks():
    assert not u8.validate_lookup(B(0x80) + b"A" * 511)
    assert not u8.validate_lookup(b"A" * 511 + B(0x80))


def _block_cases():
    cases = []
    for n in (1, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 191, 192, 256):
        cases.append(b"A" * n)
    for at in (14, 15, 30, 31, 62, 63, 126, 127):
        cases.append(b"A" * at + B(0xE9, 0x8F, 0xA1) + b"A" * 40)
    for pad in (61, 62, 63, 126):
        cases.append(b"A" * pad + B(0xE9, 0x8F))
    cases.append(b"A" * 61 + B(0xE9, 0x8F, 0xA1))
    cases.append(b"A" * 63 + B(0xE9))
    cases.append(b"A" * 61 + B(0xE9, 0x8F, 0xA1) + b"A" * 64 + B(0x80) + b"A" * 20)
    cases.append(b"A" * 61 + B(0xE9, 0x8F, 0xA1) + b"A" * 64 + B(0xC3, 0xA7))
    cases.append(b"A" * 62 + B(0xE9, 0x8F) + b"A" * 64)
    return cases


@pytest.mark.parametrize("data", _block_cases())
def test_block_edges_and_tails(data, torch):
    exp = nat.oracle_verdict(data)
    assert u8.validate_lookup(data) is exp[0]
    # device path, at every 16-byte misalignment of the start pointer
    for shift in range(16):
        buf = torch.zeros(len(data) + 32, dtype=torch.uint8, device="cuda")
        buf[shift:shift + len(data)] = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else buf[:0]
        assert u8.validate_lookup(buf[shift:shift + len(data)]) is exp[0]
        v = u8.validate_lookup_verdict(buf[shift:shift + len(data)])
        assert (v.valid(), None if v.valid() else v.error.offset, None if v.valid() else int(v.error.kind)) == exp


# ---- exhaustive and pair sweeps through the batch kernel --------------------
def _batch_of(items):
    lens = np.fromiter((len(x) for x in items), dtype=np.uint64, count=len(items))
    offs = np.zeros(len(items) + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    data = np.frombuffer(b"".join(items), dtype=np.uint8) if offs[-1] else np.zeros(0, np.uint8)
    return data, offs


@pytest.mark.parametrize("length", [0, 1, 2, 3])
def test_exhaustive_short_inputs_batch(length, torch):
    # acceptance.cpp:74-113 -- every input of length 0-3, as one batch.
    data, want = nat.exhaustive(length)
    total = want.size
    offs = np.arange(total + 1, dtype=np.uint64) * np.uint64(length)
    got = u8.validate_lookup_batch(torch.from_numpy(data).cuda() if data.size else torch.zeros(0, dtype=torch.uint8, device="cuda"),
                                   torch.from_numpy(offs.view(np.int64)).cuda())
    assert np.array_equal(got, want)


@pytest.mark.parametrize("offset", [0, 15, 16, 31, 32, 63, 64])
def test_all_pairs_at_seam_offsets(offset, torch):
    # test_lookup.cpp:287-311 -- 65,536 pairs at each offset, batched.
    n = offset + 2 + 16
    base = np.full((65536, n), 0x41, np.uint8)
    v = np.arange(65536)
    base[:, offset] = v >> 8
    base[:, offset + 1] = v & 0xFF
    data = base.reshape(-1)
    offs = np.arange(65537, dtype=np.uint64) * np.uint64(n)
    want = nat.oracle_batch(data, offs)
    got = u8.validate_lookup_batch(torch.from_numpy(data).cuda(), torch.from_numpy(offs.view(np.int64)).cuda())
    assert np.array_equal(got, want)
    # and a sample through the single-stream kernel
    for k in range(0, 65536, 257):
        assert u8.validate_lookup(base[k].tobytes()) == bool(want[k])


def _mutation_corpora(seeds, target=64):
    items = []
    for seed in seeds:
        items.append(nat.generate_valid(15, target, seed))
        for strat in range(6):
            items.append(nat.generate_invalid(15, target, seed, strat))
    return items


def test_generated_corpora_verdicts_and_positions():
    # test_lookup.cpp:338-354 (seeds 100..111, 2048+seed bytes)
    for seed in range(100, 112):
        for data in _mutation_corpora([seed], 2048 + seed):
            exp = nat.oracle_verdict(data)
            v = u8.validate_lookup_verdict(data)
            assert u8.validate_lookup(data) is exp[0]
            got = (v.valid(), None if v.valid() else v.error.offset, None if v.valid() else int(v.error.kind))
            assert got == exp, (seed, got, exp)


def test_mutation_fuzz_batch(torch):
    # acceptance.cpp:263-272 -- all 125,000 seeds x 6 strategies (750k mutated
    # 64-byte buffers) plus each seed's valid buffer, as one batch: every
    # verdict equals the oracle's and every mutation is invalid.
    import ctypes as C
    S = nat.swar()
    S.mutation_corpus.restype = C.c_size_t
    S.mutation_corpus.argtypes = [C.c_uint64, C.c_uint64, C.c_size_t, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
    seeds = 125000
    cap = seeds * 7 * (64 + 64)
    data = np.empty(cap, np.uint8)
    offs = np.zeros(seeds * 7 + 1, np.uint64)
    count = S.mutation_corpus(1, seeds + 1, 64, 1, data.ctypes.data, cap, offs.ctypes.data)
    assert count == seeds * 7
    data = data[: int(offs[-1])]
    want = nat.oracle_batch(data, offs)
    got = u8.validate_lookup_batch(torch.from_numpy(data.copy()).cuda(), torch.from_numpy(offs.view(np.int64)).cuda())
    assert np.array_equal(got, want)
    assert (want.reshape(seeds, 7)[:, 1:] == 0).all()          # every mutation invalid
    assert (want.reshape(seeds, 7)[:, 0] == 1).all()           # every generated buffer valid


def test_pinned_offset_fuzz_positions():
    # acceptance.cpp:274-324 -- malformed shapes at each special offset.
    rng = np.random.default_rng(0x0FF5E75)
    for offset in (0, 15, 16, 31, 32, 63, 64):
        for variant in range(40):
            for shape in range(6):
                cont = 0x80 + int(rng.integers(0, 0x40))
                body = [
                    [cont],
                    [0xE9 if variant & 1 else 0xC3 + int(rng.integers(0, 0x1A))],
                    [0xC0 + int(rng.integers(0, 2)), cont],
                    [0xE0, 0x80 + int(rng.integers(0, 0x20)), cont],
                    [0xED, 0xA0 + int(rng.integers(0, 0x20)), cont],
                    [0xF4, 0x90 + int(rng.integers(0, 0x30)), cont, 0x80 + int(rng.integers(0, 0x40))],
                ][shape]
                data = b"A" * offset + bytes(body) + b"A" * 16
                exp = nat.oracle_verdict(data)
                assert exp[0] is False and exp[1] == offset
                v = u8.validate_lookup_verdict(data)
                assert (v.error.offset, int(v.error.kind)) == (exp[1], exp[2])


# ---- host vs device paths, pieces and lane ranges ---------------------------
def test_host_and_device_paths_agree(torch):
    d = configs.gen_c1(3 * (32 << 20) + 12345, seed=11)  # > one H2D piece
    h = d.cpu().numpy()
    assert u8.validate_lookup(d) and u8.validate_lookup(h)
    pinned = torch.from_numpy(h).pin_memory()
    assert u8.validate_lookup(pinned.numpy())
    # an error in the second piece, straddling nothing special
    h2 = h.copy()
    pos = (32 << 20) + 777
    h2[pos] = 0xFF
    exp = nat.oracle_verdict(h2, threads=16)
    v = u8.validate_lookup_verdict(h2)
    assert not v.valid() and (v.error.offset, int(v.error.kind)) == (exp[1], exp[2])
    assert not u8.validate_lookup(h2)


def test_lane_ranges_compose(torch):
    import ctypes as C
    d = configs.gen_c1(1 << 20, seed=12)
    n = d.numel()
    rng = np.random.default_rng(3)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for trial in range(20):
        cuts = sorted(set(int(x) for x in rng.integers(1, n, size=5)))
        bounds = [0] + cuts + [n + 3]
        flag.zero_()
        for a, b in zip(bounds[:-1], bounds[1:]):
            u8.validate_lanes_async(d.data_ptr(), n, a, b, flag.data_ptr(), 0)
        torch.cuda.synchronize()
        assert int(flag.item()) == 0
    # a single bad byte must be caught by whichever piece owns its lanes
    bad = d.clone()
    bad[n // 2] = 0x80
    for trial in range(10):
        cuts = sorted(set(int(x) for x in rng.integers(1, n, size=3)) | {n // 2, n // 2 + 1})
        bounds = [0] + cuts + [n + 3]
        flag.zero_()
        for a, b in zip(bounds[:-1], bounds[1:]):
            u8.validate_lanes_async(bad.data_ptr(), n, a, b, flag.data_ptr(), 0)
        torch.cuda.synchronize()
        assert int(flag.item()) != 0


def test_first_error_ordered_claims(torch):
    """K1 (verdict path) records every lane's first flagged step with
    atomicMin and K3 recomputes the earliest: with several errors -- in one
    step, at step boundaries, in different warps -- the reported one is
    always the first, for device input and for host input (pipelined
    pieces, each recording into the same minimum)."""
    d = configs.gen_c1(64 << 20, seed=21)
    h = d.cpu().numpy()
    n = h.size
    rng = np.random.default_rng(8)
    rnd = 8 * 4096
    cands = [0, 1, rnd - 1, rnd, rnd + 1, 4096 - 2, 7 * rnd + 4095, n // 2, n // 2 + rnd, n - 2, n - 1]
    cands += [int(x) for x in rng.integers(0, n, 12)]
    for trial in range(12):
        k = int(rng.integers(1, 5))
        picks = sorted(set(int(cands[i]) for i in rng.integers(0, len(cands), k)))
        bad = h.copy()
        for p in picks:
            bad[p] = 0xFF if trial % 3 else 0x80
        exp = nat.oracle_verdict(bad, threads=16)
        v = u8.validate_lookup_verdict(torch.from_numpy(bad).cuda())
        vh = u8.validate_lookup_verdict(bad)
        if exp[0]:  # 0x80 over a continuation byte can stay valid
            assert v.valid() and vh.valid()
            continue
        assert (v.error.offset, int(v.error.kind)) == (exp[1], exp[2]), (picks, trial)
        assert (vh.error.offset, int(vh.error.kind)) == (exp[1], exp[2]), (picks, trial)
    # garbage everywhere: every round flags, the answer is the first byte's
    g = torch.from_numpy(np.full(n, 0xFF, np.uint8)).cuda()
    v = u8.validate_lookup_verdict(g)
    assert (v.error.offset, int(v.error.kind)) == (0, int(u8.ErrorKind.HEADER_BITS))
    v = u8.validate_lookup_verdict(np.full(n, 0xFF, np.uint8))
    assert (v.error.offset, int(v.error.kind)) == (0, int(u8.ErrorKind.HEADER_BITS))


def test_device_input_ordered_after_torch_work(torch):
    """Device input written asynchronously (a 256 MiB copy/fill still in
    flight) is seen by the synchronous calls and the stream session: the
    C-ABI orders after the legacy default stream (ABI 3), the Python mirror
    after torch's current stream."""
    d = configs.gen_c1(256 << 20, seed=31)
    x = torch.empty_like(d)
    for trial in range(3):
        x.fill_(0xFF)
        x.copy_(d)                      # in flight on the default stream
        assert u8.validate_lookup(x) is True
        x.fill_(0xFF)
        assert u8.validate_lookup_verdict(x).error.offset == 0
        x.copy_(d)
        with u8.LookupStream() as sess:
            sess.feed(x[: 100 << 20]).feed(x[100 << 20:])
            assert sess.finish() is True
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            x.fill_(0xC0)               # in flight on a non-default stream
            assert u8.validate_lookup(x) is False
            x.copy_(d)
            assert u8.validate_lookup(x) is True
        torch.cuda.current_stream().wait_stream(side)


# ---- configs -----------------------------------------------------------------
def test_c0_full_size():
    d = configs.gen_c0()
    h = d.cpu().numpy()
    assert h.min() >= 0x0A and h.max() <= 0x7E
    assert u8.validate_lookup(d) is True
    assert nat.oracle_verdict(h, threads=32)[0] is True


def test_c1_full_size_and_injected_errors():
    d = configs.gen_c1()
    assert d.numel() == 1 << 30
    h = d.cpu().numpy()
    assert nat.oracle_verdict(h, threads=64)[0] is True
    assert u8.validate_lookup(d) is True
    # size-independent property: one corrupted byte anywhere -> same verdict
    # and position as the oracle (oracle run on a window: everything before
    # is valid text, so a boundary-aligned window gives the exact answer).
    rng = np.random.default_rng(2)
    n = d.numel()
    for _ in range(24):
        pos = int(rng.integers(0, n))
        val = int(rng.integers(0, 256))
        old = int(h[pos])
        if val == old:
            continue
        # A character-aligned window of the valid stream around pos: the
        # stream before it is valid text ending on a boundary and the text
        # after it is untouched, so the window's oracle verdict is the
        # stream's (offsets shifted by lo).
        lo = max(0, pos - 16)
        while lo > 0 and (h[lo] & 0xC0) == 0x80:
            lo -= 1
        hi = min(n, pos + 16)
        while hi < n and (h[hi] & 0xC0) == 0x80:
            hi += 1
        win = h[lo:hi].copy()
        win[pos - lo] = val
        exp = nat.oracle_verdict(win)
        d[pos] = val
        v = u8.validate_lookup_verdict(d)
        assert u8.validate_lookup(d) is exp[0]
        if exp[0]:
            assert v.valid()
        else:
            assert (v.error.offset, int(v.error.kind)) == (exp[1] + lo, exp[2])
        d[pos] = old
    assert u8.validate_lookup(d) is True


def test_c2_segments():
    b = configs.gen_c2()
    got = u8.validate_lookup_batch(b.data, b.d_offsets)
    want = nat.oracle_batch(b.data.cpu().numpy(), b.offsets)
    assert np.array_equal(want, b.expected)
    assert np.array_equal(got, want)
    assert int((got == 0).sum()) == 32


def test_c3_records():
    b = configs.gen_c3()
    got = u8.validate_lookup_batch(b.data, b.d_offsets)
    want = nat.oracle_batch(b.data.cpu().numpy(), b.offsets)
    assert np.array_equal(want, b.expected)
    assert np.array_equal(got, want)


def test_batch_edge_cases(torch):
    # empty records, 1..3-byte records, leading gap, records ending inside
    # characters, dense tiny records (> 31 per 2 KiB)
    rng = np.random.default_rng(5)
    for trial in range(30):
        parts = []
        for _ in range(int(rng.integers(1, 400))):
            kind = int(rng.integers(0, 6))
            if kind == 0:
                parts.append(b"")
            elif kind == 1:
                parts.append(bytes(rng.integers(0, 256, int(rng.integers(1, 4)), dtype=np.uint8)))
            elif kind == 2:
                parts.append(nat.generate_valid(15, int(rng.integers(1, 40)), int(rng.integers(1, 1 << 30))))
            elif kind == 3:
                parts.append(nat.generate_invalid(15, int(rng.integers(1, 40)), int(rng.integers(1, 1 << 30)), int(rng.integers(0, 6))))
            elif kind == 4:
                parts.append(nat.generate_valid(15, int(rng.integers(100, 5000)), int(rng.integers(1, 1 << 30))))
            else:
                parts.append(bytes([0xE9, 0x8F]))  # truncated at record end
        data, offs = _batch_of(parts)
        lead = int(rng.integers(0, 20))
        data = np.concatenate([np.full(lead, 0xE9, np.uint8), data])
        offs = offs + np.uint64(lead)
        want = nat.oracle_batch(data, offs)
        t = torch.from_numpy(data.copy()).cuda()
        for shift in (0, 1, 7):
            buf = torch.zeros(t.numel() + 32, dtype=torch.uint8, device="cuda")
            buf[shift:shift + t.numel()] = t
            got = u8.validate_lookup_batch(buf[shift:shift + t.numel()], torch.from_numpy(offs.view(np.int64)).cuda())
            assert np.array_equal(got, want), (trial, shift)
        assert np.array_equal(u8.validate_lookup_batch(data, offs), want)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_c4_structure_scaled(variant):
    # Same construction as C4 at 64 MiB: shard edges inside 3/4-byte chars.
    n = 64 << 20
    d, err = configs.gen_c4(n, seed=5, variant=variant)
    h = d.cpu().numpy()
    for k in range(1, 8):
        b = k * (n // 8)
        if not (variant == 1 and k == 4):
            assert (h[b] & 0xC0) == 0x80  # edge byte is a continuation byte
    exp = nat.oracle_verdict(h, threads=32)
    assert exp[0] == (variant == 0)
    if variant:
        assert exp[1] == err
    v = u8.validate_lookup_verdict(d)
    assert (v.valid(), None if v.valid() else v.error.offset) == (exp[0], exp[1])
    # sharded over G = 2, 4, 8 with a 3-byte halo: OR of shard flags
    import torch
    for G in (2, 4, 8):
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        for k in range(G):
            s, e = k * n // G, (k + 1) * n // G
            h0 = min(s, 16)
            last = k == G - 1
            tail = 0 if last else 1  # the byte after the shard (lane e-1's lookahead)
            nl = e - s + h0 + tail
            u8.validate_lanes_async(d.data_ptr() + s - h0, nl, h0, (nl + 3) if last else (e - s + h0),
                                    flag.data_ptr(), 0)
        torch.cuda.synchronize()
        assert (int(flag.item()) == 0) == exp[0]


@pytest.mark.slow
@pytest.mark.parametrize("variant", [0, 1, 2])
def test_c4_full_size_vs_oracle(variant):
    """C4 at its full 16 GiB, variants A/B/C: the device verdict and first
    error (K1 tracking + K3) equal the multi-threaded CPU oracle's
    (oracle_validate, proj/src/oracle.cpp:10-44) on the same bytes, copied
    back from HBM; and the generator's recorded error agrees."""
    import os
    import torch
    n = configs.C4["n"]
    d, err = configs.gen_c4(n, seed=configs.C4["seed"], variant=variant)
    v = u8.validate_lookup_verdict(d)
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.copy_(d)
    del d
    torch.cuda.empty_cache()
    h = host.numpy()
    for k in range(1, 8):  # every k*n/8 edge inside a 3- or 4-byte character
        assert (h[k * (n // 8)] & 0xC0) == 0x80
    ok, off, kind = nat.oracle_verdict(h, threads=max(1, len(os.sched_getaffinity(0))))
    assert ok == (variant == 0) and (ok or off == err)
    got = (v.valid(), None if v.valid() else (v.error.offset, int(v.error.kind)))
    assert got == (ok, None if ok else (off, kind)), (got, ok, off, kind)


def test_host_generators_equal_device_generators(torch):
    """oracle/gen_host.c (the reference arm's input) equals the device
    generators byte for byte: C0/C1 streams and C4 A/B/C (scaled)."""
    for n, seed, ascii_only in ((1 << 20, 1, True), ((3 << 20) + 5, 2, False), (777_777, 5, False)):
        dev = configs.gen_stream(n, seed, ascii_only).cpu().numpy()
        assert np.array_equal(dev, nat.gen_stream_host(n, seed, ascii_only)), (n, seed, ascii_only)
    n = 64 << 20
    for variant in (0, 1, 2):
        d, err = configs.gen_c4(n, seed=5, variant=variant)
        h, herr = nat.gen_c4_host(n, 5, variant)
        assert herr == err and np.array_equal(d.cpu().numpy(), h), variant


def test_stream_range_generator_matches_full_stream(torch):
    import ctypes as C
    from paper_2010_03090_b200 import _lib
    n = (5 << 20) + 4321
    full = configs.gen_c1(n, seed=9)
    lib = _lib.load()
    for lo, hi in [(0, n), (16, 1000), (65536 - 4, 65536 + 7), (131072, 3 << 20), (4 << 20, n), (100, 100)]:
        out = torch.empty(max(hi - lo, 1), dtype=torch.uint8, device="cuda")
        _lib.check(lib.utf8v_gen_stream_range(out.data_ptr(), n, lo, hi, 9, 0, torch.cuda.current_stream().cuda_stream))
        assert torch.equal(out[: hi - lo], full[lo:hi]), (lo, hi)


def test_k1_structural_boundaries():
    """Errors placed at (and -3..+3 around) every boundary K1's plumbing
    handles -- 32-byte chunks, lanes, 1 KiB load instructions, 4 KiB warp
    steps, the grid-stride wrap (resident warps x 4 KiB) -- including
    sequences that straddle the boundary (lead before, follower after).
    Verdict (K1) and first-error offset/kind (K3) equal the windowed oracle,
    for device and host input."""
    d = configs.gen_c1(64 << 20, seed=7)
    h = d.cpu().numpy()
    n = d.numel()
    resident = 148 * 4 * 8 * 4096  # warps x step bytes on a B200 (upper bound of the wrap)
    bounds = [32, 64, 31 * 32, 1024, 2048, 3072, 4096, 8192, 4096 * 37, resident // 2, resident,
              resident + 4096, 2 * resident, n - 4096, n - 32]
    seqs = [b"\x80", b"\xc3", b"\xe0\x9f\xbf", b"\xed\xa0\x80", b"\xf4\x90\x80\x80", b"\xf0\x9f\x98",
            b"\xc0\x80", b"\xff"]
    checked = 0
    for b in bounds:
        for delta in range(-3, 4):
            for seq in seqs:
                pos = b + delta
                if pos < 0 or pos + len(seq) > n:
                    continue
                lo = max(0, pos - 16)
                while lo > 0 and (h[lo] & 0xC0) == 0x80:
                    lo -= 1
                hi = min(n, pos + len(seq) + 16)
                while hi < n and (h[hi] & 0xC0) == 0x80:
                    hi += 1
                win = h[lo:hi].copy()
                win[pos - lo:pos - lo + len(seq)] = np.frombuffer(seq, np.uint8)
                exp = nat.oracle_verdict(win)
                old = d[pos:pos + len(seq)].clone()
                d[pos:pos + len(seq)] = torch_from(seq)
                assert u8.validate_lookup(d) is exp[0], (b, delta, seq)
                v = u8.validate_lookup_verdict(d)
                if exp[0]:
                    assert v.valid()
                else:
                    assert (v.error.offset, int(v.error.kind)) == (exp[1] + lo, exp[2]), (b, delta, seq)
                if checked % 17 == 0:  # the host (pipelined H2D) path on a subset
                    assert u8.validate_lookup(d.cpu().numpy().tobytes()) is exp[0]
                d[pos:pos + len(seq)] = old
                checked += 1
    assert checked > 700
    assert u8.validate_lookup(d) is True


def torch_from(seq):
    import torch
    return torch.tensor(list(seq), dtype=torch.uint8, device="cuda")


def test_thread_contexts_are_released(torch):
    """Per-thread contexts (streams, the device stage grown to the input, the
    pinned ring for pageable input) are freed when the thread exits: many
    short-lived threads validating 32 MiB of host input leave device memory
    where it was."""
    import threading
    h = configs.gen_c1(32 << 20, seed=13).cpu().numpy()
    torch.cuda.synchronize()

    def work(out, i):
        out[i] = u8.validate_lookup(h)

    def round_of(k):
        out = [None] * k
        ts = [threading.Thread(target=work, args=(out, i)) for i in range(k)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return out

    assert all(round_of(4))
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(3):
        assert all(round_of(4))
    free1 = torch.cuda.mem_get_info()[0]
    # 12 more threads, each with a 32 MiB stage: without release this would
    # hold 384 MiB; allow allocator slack of 96 MiB.
    assert free0 - free1 < (96 << 20), (free0, free1)


def _encode(cps, length):
    """UTF-8 style encoding of each code point in exactly `length` bytes
    (shortest form when it fits, overlong otherwise); rows of `length` bytes."""
    cps = np.asarray(cps, np.uint32)
    out = np.zeros((cps.size, length), np.uint8)
    if length == 1:
        out[:, 0] = cps
        return out
    lead = {2: 0xC0, 3: 0xE0, 4: 0xF0}[length]
    for k in range(length - 1, 0, -1):
        out[:, k] = 0x80 | (cps & 0x3F)
        cps = cps >> 6
    out[:, 0] = lead | cps
    return out


def test_code_point_sweep_on_device():
    """The acceptance gate's sweep (proj/tests/acceptance.cpp:117-175) on the
    GPU: every code point 0..0x1FFFFF in shortest form, plus every overlong
    form that fits in 4 bytes, each as its own record of one 2.2 M-record
    batch (K2, dense 1-4-byte records), against the expected verdicts and
    the oracle; and K1 over the concatenation of all valid encodings."""
    import torch
    parts, expect = [], []
    for length, lo, hi in ((1, 0, 0x80), (2, 0x80, 0x800), (3, 0x800, 0x10000), (4, 0x10000, 0x200000)):
        cps = np.arange(lo, hi, dtype=np.uint32)
        parts.append(_encode(cps, length))
        expect.append(((cps < 0xD800) | (cps > 0xDFFF)) & (cps <= 0x10FFFF))
    for length, hi in ((2, 0x80), (3, 0x800), (4, 0x10000)):  # overlongs
        parts.append(_encode(np.arange(hi, dtype=np.uint32), length))
        expect.append(np.zeros(hi, bool))
    lens = np.concatenate([np.full(p.shape[0], p.shape[1], np.uint64) for p in parts])
    data = np.concatenate([p.reshape(-1) for p in parts])
    offs = np.zeros(lens.size + 1, np.uint64)
    np.cumsum(lens, out=offs[1:])
    want = np.concatenate(expect).astype(np.uint8)
    assert want.sum() == 1112064
    got = u8.validate_lookup_batch(torch.from_numpy(data).cuda(), torch.from_numpy(offs.view(np.int64)).cuda())
    assert np.array_equal(got, want)
    assert np.array_equal(nat.oracle_batch(data, offs), want)
    valid_stream = np.concatenate([p[e].reshape(-1) for p, e in zip(parts[:4], expect[:4])])
    assert u8.validate_lookup(torch.from_numpy(valid_stream).cuda()) is True


def test_batch_offsets_of_any_integer_dtype(torch):
    """Device offsets may come as int32 (Arrow string columns) or int64; host
    offsets as any integer array: same verdicts."""
    b = configs.gen_c3(n_records=3000, seed=12)
    want = b.expected
    for dt in (torch.int32, torch.int64):
        got = u8.validate_lookup_batch(b.data, b.d_offsets.to(dt))
        assert np.array_equal(got, want), dt
    for dt in (np.int32, np.int64, np.uint64):
        got = u8.validate_lookup_batch(b.data, b.offsets.astype(dt))
        assert np.array_equal(got, want), dt


def test_batch_mixed_density_large(torch):
    # K2's record cursor over long per-warp ranges: 64 MiB of the C1 mix cut
    # into regions of very different record density (mean 3 B .. 64 KiB,
    # empty records included), so warps take several boundary batches per
    # step in dense regions and none for many steps in sparse ones; cuts
    # mostly at character boundaries, some inside characters; 1 % of records
    # get a random byte.  Device and host input, vs the oracle per record.
    n = 64 << 20
    h = configs.gen_c1(n, seed=21).cpu().numpy()
    rng = np.random.default_rng(21)
    cuts = [0]
    pos = 0
    means = (3, 16, 48, 300, 4096, 65536)
    while pos < n:
        m = means[int(rng.integers(0, len(means)))]
        region_end = min(n, pos + int(rng.integers(1 << 18, 1 << 21)))
        lens = rng.exponential(m, size=max(4, 2 * (region_end - pos) // m)).astype(np.int64)
        ends = pos + np.cumsum(lens)
        ends = ends[ends < region_end]
        cuts.extend(ends.tolist())
        cuts.append(region_end)
        pos = region_end
    cuts = np.array(cuts, dtype=np.int64)
    snap = rng.random(cuts.size) < 0.9
    for _ in range(3):  # move most cuts forward to a character boundary
        inside = snap & (cuts < n) & ((h[np.minimum(cuts, n - 1)] & 0xC0) == 0x80)
        cuts[inside] += 1
    cuts = np.maximum.accumulate(np.minimum(cuts, n))
    cuts[0], cuts[-1] = 0, n
    offs = cuts.astype(np.uint64)
    nrec = offs.size - 1
    bad = rng.choice(nrec, size=nrec // 100, replace=False)
    data = h.copy()
    for r in bad:
        a, b = int(offs[r]), int(offs[r + 1])
        if b > a:
            data[int(rng.integers(a, b))] = int(rng.integers(0x80, 0x100))
    want = nat.oracle_batch(data, offs)
    assert 0 < int((want == 0).sum()) < nrec
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    got = u8.validate_lookup_batch(torch.from_numpy(data).cuda(), d_offs)
    assert np.array_equal(got, want)
    assert np.array_equal(u8.validate_lookup_batch(data, offs), want)


@pytest.mark.parametrize("n_rec", [1, 2, 17, 64, 300, 2048])
def test_batch_few_large_records(n_rec, torch):
    # K2L (<= 2048 records of >= 64 KiB on average, launch_batch): K1's sweep
    # with out-of-line attribution over offsets in shared memory.  Records of
    # 0 B .. ~1 MiB (empty and tiny ones among them), cuts inside characters,
    # errors in a record's first three bytes, at its end and inside it,
    # all-garbage records, bytes before offsets[0] and after offsets[N], and
    # unaligned data; vs the oracle per record, device and host input.
    rng = np.random.default_rng(1000 + n_rec)
    lens = rng.lognormal(np.log(160 << 10), 1.0, n_rec).astype(np.int64)
    lens[rng.random(n_rec) < 0.1] = 0
    lens[rng.random(n_rec) < 0.1] = rng.integers(1, 40)
    lens = np.minimum(lens, 1 << 20)
    if lens.sum() < n_rec * (64 << 10):  # keep the batch on the K2L path
        lens = lens + ((n_rec * (64 << 10) - lens.sum()) // n_rec + 1)
    lead, tail = int(rng.integers(0, 100)), int(rng.integers(0, 100))
    total = int(lens.sum()) + lead + tail
    h = configs.gen_c1(total + 64, seed=n_rec).cpu().numpy()[:total].copy()
    offs = np.zeros(n_rec + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    offs += np.uint64(lead)
    for r in range(n_rec):
        a, b = int(offs[r]), int(offs[r + 1])
        if b - a < 4:
            continue
        kind = int(rng.integers(0, 8))
        if kind == 0:
            h[a + int(rng.integers(0, 3))] = 0x80  # stray continuation at the start
        elif kind == 1:
            h[b - 1] = 0xE2  # truncated at the end
        elif kind == 2:
            h[int(rng.integers(a, b))] = 0xFF
        elif kind == 3 and b - a < (300 << 10):
            h[a:b] = 0xFF  # garbage record
        elif kind == 4:
            h[int(rng.integers(a, b - 1))] = 0xC0  # overlong lead
    h[:lead] = 0xFF
    h[total - tail:] = 0xC3
    want = nat.oracle_batch(h, offs)
    t = torch.from_numpy(h).cuda()
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    for shift in (0, 1, 7):
        buf = torch.zeros(t.numel() + 32, dtype=torch.uint8, device="cuda")
        buf[shift:shift + t.numel()] = t
        got = u8.validate_lookup_batch(buf[shift:shift + t.numel()], d_offs)
        assert np.array_equal(got, want), (n_rec, shift, np.nonzero(got != want)[0][:10])
    assert np.array_equal(u8.validate_lookup_batch(h, offs), want)


def test_concurrent_callers_mixed_entry_points(torch):
    """Validators are pure and callable concurrently (the
    reference bench runs them from several threads, proj/src/bench.cpp:112-118):
    8 host threads at once, each looping over every entry point -- verdicts
    on host and device input with and without an error, record batches, a
    stream session -- on its own data, all checked against the oracle."""
    import threading
    base = configs.gen_c1(24 << 20, seed=31).cpu().numpy()
    cases = []
    rng = np.random.default_rng(31)
    for k in range(8):
        h = base[k << 20: (k << 20) + (16 << 20) + 7 * k].copy()
        if k % 2:
            h[int(rng.integers(0, h.size))] = 0xF8
        exp = nat.oracle_verdict(h, threads=8)
        cuts = np.sort(rng.choice(np.arange(1, h.size), 300, replace=False)).astype(np.uint64)
        offs = np.concatenate([[0], cuts, [h.size]]).astype(np.uint64)
        cases.append((h, exp, offs, nat.oracle_batch(h, offs)))
    errors = []

    def work(k):
        try:
            h, exp, offs, want = cases[k]
            d = torch.from_numpy(h).cuda()
            d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
            for it in range(4):
                for src in (h, d):
                    v = u8.validate_lookup_verdict(src)
                    got = (v.valid(), None if v.valid() else (v.error.offset, int(v.error.kind)))
                    assert got == (exp[0], None if exp[0] else (exp[1], exp[2])), (k, it)
                    assert u8.validate_lookup(src) is exp[0]
                assert np.array_equal(u8.validate_lookup_batch(h, offs), want)
                assert np.array_equal(u8.validate_lookup_batch(d, d_offs), want)
                with u8.LookupStream() as s:
                    for a in range(0, h.size, 5 << 20):
                        s.feed(h[a:a + (5 << 20)])
                    assert s.finish() is exp[0]
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:3]


@pytest.mark.parametrize("path", ["K2L", "K2"])
def test_batch_offsets_past_4_gib(path, torch):
    # 64-bit positions: a 5 GiB data array whose records (and injected
    # errors) lie beyond 2^32 bytes, through K2L (few large records) and K2
    # (many records: the large one surrounded by 40 k small ones), vs the
    # multi-threaded oracle per record.
    G = 1 << 30
    n = 5 * G + 12345
    d = configs.gen_c1(n, seed=77)
    rng = np.random.default_rng(5)
    if path == "K2L":
        cuts = [0, 100, 4 * G + 777, 4 * G + (1 << 29), n]
    else:
        small = np.sort(rng.integers(4 * G + (1 << 28), n, 40_000)).tolist()
        cuts = [0, 100, 4 * G + 777] + small + [n]
    offs = np.array(cuts, np.uint64)
    for at in (4 * G + 5_000, 4 * G + (1 << 28) + 3, n - 2):  # errors past 2^32
        d[at] = 0xC0
    h = d.cpu().numpy()
    want = nat.oracle_batch(h, offs, threads=16)
    assert (want == 0).sum() >= 2
    got = u8.validate_lookup_batch(d, torch.from_numpy(offs.view(np.int64)).cuda())
    assert np.array_equal(got, want), np.nonzero(got != want)[0][:10]
    del d
    torch.cuda.empty_cache()
