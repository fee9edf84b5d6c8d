"""Streaming session (utf8v_cuda_stream_*, paper_2010_03090_b200.LookupStream):
a stream fed in pieces gives the oracle's verdict of the concatenation, for
host and device pieces, every split shape, and errors placed across piece
boundaries."""
import numpy as np
import pytest

from tests import _native as nat

pytestmark = pytest.mark.gpu


def _u8():
    import paper_2010_03090_b200 as u8
    return u8


def _split(rng, n, k):
    return sorted(int(x) for x in rng.integers(0, n + 1, size=k))


def _feed_all(s, buf, cuts, device=False):
    import torch
    t = torch.from_numpy(buf).cuda() if device else None
    prev = 0
    for c in list(cuts) + [len(buf)]:
        if device:
            s.feed(t[prev:c])
        else:
            s.feed(buf[prev:c].tobytes())
        prev = c
    return s.finish()


def test_empty_and_tiny_streams():
    u8 = _u8()
    with u8.LookupStream() as s:
        assert s.finish() is True                      # nothing fed
        assert s.feed(b"").feed(b"").finish() is True  # only empty pieces
        assert s.feed(b"\xc3").finish() is False       # truncated at the end
        assert s.feed(b"\xc3").feed(b"\xa9").finish() is True
        assert s.feed(b"\xe2").feed(b"\x82").feed(b"\xac").finish() is True
        assert s.feed(b"\xed").feed(b"\xa0\x80").finish() is False  # surrogate across the cut
        assert s.feed(b"\xf0\x9f").feed(b"\x98").feed(b"\x80").finish() is True


@pytest.mark.parametrize("device", [False, True])
def test_random_splits_match_oracle(device):
    u8 = _u8()
    rng = np.random.default_rng(11 if device else 12)
    with u8.LookupStream() as s:
        for seed in range(1, 60):
            for strategy in (None, 0, 1, 2, 3, 4, 5, 6):
                size = int(rng.integers(1, 5000))
                data = nat.generate_valid(0xF, size, seed) if strategy is None else \
                    nat.generate_invalid(0xF, size, seed, strategy)
                buf = np.frombuffer(data, dtype=np.uint8).copy()
                want = bool(nat.oracle_verdict(data)[0])
                cuts = _split(rng, len(buf), int(rng.integers(0, 10)))
                assert _feed_all(s, buf, cuts, device) == want, (seed, strategy, cuts)


def test_error_at_every_boundary_offset():
    """An error straddling a cut at each offset -3..+3 of the cut."""
    u8 = _u8()
    base = np.frombuffer(nat.generate_valid(0xF, 4096, 5), dtype=np.uint8).copy()
    bad_pairs = [b"\xc0\x80", b"\xe0\x9f\xbf", b"\xed\xa0\x80", b"\xf4\x90\x80\x80", b"\x80", b"\xe2\x82"]
    with u8.LookupStream() as s:
        for cut in (1, 2, 3, 4, 5, 31, 32, 33, 1023, 1024, 2048):
            for seq in bad_pairs:
                for delta in range(-3, 4):
                    buf = np.full(4096 + 16, 0x41, dtype=np.uint8)
                    pos = max(0, cut + delta)
                    buf[pos:pos + len(seq)] = np.frombuffer(seq, dtype=np.uint8)
                    want = bool(nat.oracle_verdict(buf.tobytes())[0])
                    assert want is False
                    assert _feed_all(s, buf, [cut]) is False, (cut, seq, delta)
                    assert _feed_all(s, buf, [cut], device=True) is False, (cut, seq, delta)
        # valid text cut inside every kind of character
        for cut in range(1, 64):
            assert _feed_all(s, base, [cut, cut + 1, cut + 3]) is True


def test_large_device_stream_and_launch_count():
    u8 = _u8()
    from paper_2010_03090_b200 import _lib, configs
    lib = _lib.load()
    d = configs.gen_c1(16 << 20, seed=2)
    rng = np.random.default_rng(4)
    cuts = _split(rng, d.numel(), 40)
    with u8.LookupStream() as s:
        prev = 0
        for c in cuts + [d.numel()]:
            s.feed(d[prev:c])
            n = c - prev
            assert lib.utf8v_cuda_last_launch_count() == (0 if n == 0 else 1)  # K1 runs the edge too
            prev = c
        assert s.bytes_fed == d.numel()
        assert s.finish() is True
        assert s.bytes_fed == 0
        d[cuts[20]] = 0xC0  # error right at a piece start
        prev = 0
        for c in cuts + [d.numel()]:
            s.feed(d[prev:c])
            prev = c
        assert s.finish() is False


def test_device_pieces_outlive_the_callers_references():
    """A device piece is read asynchronously until finish(): LookupStream
    keeps every piece alive, so temporaries the caller drops right after
    feed() are not freed and reused under the session (the caching
    allocator would hand their blocks to the next allocations, which are
    overwritten at once)."""
    import torch
    from paper_2010_03090_b200 import configs
    u8 = _u8()
    torch.cuda.set_device(0)
    with u8.LookupStream() as s:
        for trial in range(4):
            for k in range(3):
                s.feed(configs.gen_c1(32 << 20, seed=60 + trial + k))  # a temporary, dropped at once
                junk = torch.full((32 << 20,), 0xFF, dtype=torch.uint8, device="cuda")  # may reuse freed blocks
                del junk
            assert s.finish() is True, trial


def test_stream_calls_keep_the_callers_device():
    import torch
    u8 = _u8()
    torch.cuda.set_device(0)
    with u8.LookupStream() as s:
        s.feed(b"abc")
        assert torch.cuda.current_device() == 0
        assert s.finish() is True
