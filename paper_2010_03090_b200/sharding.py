"""Multi-GPU validation of one large stream (BASELINE config 4).

One process per GPU.  The stream [0, n) is cut into `world` byte-range
shards [s_k, e_k); rank k holds its shard plus
  * a head of up to 16 bytes before s_k (the 3-byte look-back halo the
    S check needs: x[i-1], x[i-2], x[i-3]), and
  * a tail of 1 byte after e_k (the lookahead of the rare-pair check that
    K1 evaluates at the lead's lane), except on the last shard,
and evaluates lanes [s_k, e_k) -- the last shard also the end-of-input lanes
[n, n+3) (check_incomplete, proj/include/utf8v/lookup_kernel.hpp:48-68).
Every lane of the whole stream is evaluated by exactly one rank with the
bytes the single-stream kernel would see, so

    stream valid  <=>  max over ranks of the error flag == 0,

combined with one 4-byte allreduce(MAX) over NCCL (NVLink/NVSwitch).  There
is no other data-path exchange: shards are independent.  Shard edges may cut
characters anywhere (config 4 forces them inside 3-/4-byte characters).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

HEAD = 16  # look-back bytes carried before each shard (>= 3)


@dataclass(frozen=True)
class Shard:
    index: int
    count: int
    start: int      # first byte of the shard in the stream
    end: int        # one past the last byte
    n_total: int

    @property
    def last(self) -> bool:
        return self.index == self.count - 1

    @property
    def head(self) -> int:
        return min(self.start, HEAD)

    @property
    def tail(self) -> int:
        return 0 if self.last or self.end >= self.n_total else 1

    @property
    def lo(self) -> int:
        """First stream byte the rank holds (head included)."""
        return self.start - self.head

    @property
    def hi(self) -> int:
        """One past the last stream byte the rank holds (tail included)."""
        return self.end + self.tail

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    @property
    def lanes(self) -> tuple[int, int]:
        """Lane range in local coordinates for the C-ABI lane entry points."""
        lo = self.head
        hi = self.n_local + 3 if self.last else self.head + (self.end - self.start)
        return lo, hi


def plan(n_total: int, world: int, align: int = 16) -> list[Shard]:
    """Shards at floor(k * n / world), rounded down to `align` bytes (config 4
    uses k*n/8 exactly: 2 GiB multiples)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    cuts = [0] + [(k * n_total // world) // align * align for k in range(1, world)] + [n_total]
    for a, b in zip(cuts, cuts[1:]):
        if b < a:
            raise ValueError("stream too small for this many shards")
    return [Shard(k, world, cuts[k], cuts[k + 1], n_total) for k in range(world)]


def shard_error_flag(local, shard: Shard) -> int:
    """This rank's error flag (0 = no error in its lanes) on the GPU.  `local`
    holds stream bytes [shard.lo, shard.hi): a CUDA uint8 tensor (validated in
    place) or host bytes (copied over PCIe inside the call)."""
    from . import _input, _lib
    lib = _lib.load()
    ptr, n, dev, _keep = _input(local)
    if n != shard.n_local:
        raise ValueError(f"shard buffer holds {n} bytes, expected {shard.n_local}")
    lo, hi = shard.lanes
    flag = C.c_uint32(0)
    _lib.check(lib.utf8v_cuda_validate_lanes(ptr, n, lo, hi, dev, C.byref(flag)))
    return int(flag.value)


def combine(flag: int, group=None, device=None) -> bool:
    """One 4-byte allreduce(MAX) of the rank flags; True when the stream is
    valid.  NCCL on a CUDA device, gloo on the CPU (tests)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item()) == 0


def validate_sharded(local, shard: Shard, group=None, device=None,
                     shard_flag: Optional[Callable[[object, Shard], int]] = None) -> bool:
    """Collective: every rank calls it with its own shard; all get the
    verdict of the whole stream."""
    flag = (shard_flag or shard_error_flag)(local, shard)
    return combine(flag, group=group, device=device)
