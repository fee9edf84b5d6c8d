"""ctypes handles on the CPU checkers (test infrastructure only).

  oracle()   oracle/liboracle.so -- C restatement of the reference algorithms
  ref()      oracle/_ref/libutf8v_ref.so -- the unmodified reference library
             (None when it was not built: no reference checkout anywhere)
  swar()     tests/cpp/libswar_host.so -- the device SWAR header on the CPU
"""
from __future__ import annotations

import ctypes as C
import functools
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libutf8v_ref.so"
SWAR_SO = ROOT / "tests" / "cpp" / "libswar_host.so"

u8p = C.c_void_p


def _ensure_built():
    if not ORACLE_SO.exists() or not SWAR_SO.exists():
        from paper_2010_03090_b200 import _build
        _build.build_oracle()
        _build.build_test_helpers()


@functools.lru_cache(None)
def oracle() -> C.CDLL:
    _ensure_built()
    L = C.CDLL(str(ORACLE_SO))
    L.orc_validate.argtypes = [u8p, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    L.orc_validate.restype = C.c_int
    L.orc_validate_mt.argtypes = [u8p, C.c_size_t, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    L.orc_validate_mt.restype = C.c_int
    L.orc_encode.argtypes = [C.c_uint32, u8p]
    L.orc_encode.restype = C.c_int
    L.orc_nibble_tables.argtypes = [u8p, u8p, u8p]
    L.orc_pair_always_invalid.argtypes = [C.c_uint8, C.c_uint8]
    L.orc_pair_always_invalid.restype = C.c_int
    L.orc_verify_tables.argtypes = [u8p, u8p, u8p, u8p, u8p, u8p]
    L.orc_verify_tables.restype = C.c_int
    for f in ("orc_classify_lanes", "orc_length_error_lanes"):
        getattr(L, f).argtypes = [u8p, u8p, u8p, C.c_size_t]
    L.orc_incomplete_lanes.argtypes = [u8p, u8p, C.c_size_t]
    L.orc_lookup_validate.argtypes = [u8p, C.c_size_t]
    L.orc_lookup_validate.restype = C.c_int
    L.orc_generate_valid.argtypes = [C.c_uint, C.c_size_t, C.c_uint64, u8p, C.c_size_t]
    L.orc_generate_valid.restype = C.c_size_t
    L.orc_generate_invalid.argtypes = [C.c_uint, C.c_size_t, C.c_uint64, C.c_int, u8p, C.c_size_t]
    L.orc_generate_invalid.restype = C.c_size_t
    L.orc_gen_stream.argtypes = [u8p, C.c_uint64, C.c_uint64, C.c_int, C.c_int]
    L.orc_gen_stream.restype = C.c_int
    L.orc_gen_c4.argtypes = [u8p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
    L.orc_gen_c4.restype = C.c_int
    return L


def gen_stream_host(n: int, seed: int, ascii_only: bool = False, threads: int = 4) -> np.ndarray:
    """The config stream from the oracle's CPU generator (oracle/gen_host.c)."""
    out = np.empty(n, np.uint8)
    assert oracle().orc_gen_stream(out.ctypes.data, n, seed, int(ascii_only), threads) == 0
    return out


def gen_c4_host(n: int, seed: int, variant: int, threads: int = 8):
    """(bytes, first error offset or None) of config 4 (oracle/gen_host.c)."""
    out = np.empty(n, np.uint8)
    err = C.c_uint64(0)
    assert oracle().orc_gen_c4(out.ctypes.data, n, seed, variant, threads, C.byref(err)) == 0
    return out, (None if err.value == (1 << 64) - 1 else int(err.value))


@functools.lru_cache(None)
def ref():
    if not REF_SO.exists():
        return None
    L = C.CDLL(str(REF_SO))
    L.ref_oracle_validate.argtypes = [u8p, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    L.ref_oracle_validate.restype = C.c_int
    L.ref_validate_lookup.argtypes = [u8p, C.c_size_t]
    L.ref_validate_lookup.restype = C.c_int
    L.ref_validate_lookup_mt.argtypes = [u8p, C.c_size_t, C.c_int]
    L.ref_validate_lookup_mt.restype = C.c_int
    L.ref_backend_count.restype = C.c_int
    L.ref_backend_name.restype = C.c_char_p
    L.ref_backend_name.argtypes = [C.c_int]
    L.ref_backend_width.restype = C.c_size_t
    L.ref_backend_width.argtypes = [C.c_int]
    L.ref_backend_validate.argtypes = [C.c_int, u8p, C.c_size_t]
    L.ref_backend_validate.restype = C.c_int
    for f in ("ref_backend_classify", "ref_backend_length_error"):
        getattr(L, f).argtypes = [C.c_int, u8p, u8p, u8p]
    L.ref_backend_incomplete.argtypes = [C.c_int, u8p, u8p]
    L.ref_backend_self_test.argtypes = [C.c_int, C.c_uint64]
    L.ref_backend_self_test.restype = C.c_int
    L.ref_nibble_tables.argtypes = [u8p, u8p, u8p]
    L.ref_encode.argtypes = [C.c_uint32, u8p]
    L.ref_encode.restype = C.c_int
    L.ref_generate_valid.argtypes = [C.c_uint, C.c_size_t, C.c_uint64, u8p, C.c_size_t]
    L.ref_generate_valid.restype = C.c_longlong
    L.ref_generate_invalid.argtypes = [C.c_uint, C.c_size_t, C.c_uint64, C.c_int, u8p, C.c_size_t]
    L.ref_generate_invalid.restype = C.c_longlong
    return L


@functools.lru_cache(None)
def swar():
    _ensure_built()
    L = C.CDLL(str(SWAR_SO))
    L.swar_first_lane.argtypes = [u8p, C.c_size_t, C.c_uint]
    L.swar_first_lane.restype = C.c_uint64
    L.swar_validate.argtypes = [u8p, C.c_size_t, C.c_uint]
    L.swar_validate.restype = C.c_int
    L.swar_exhaustive.argtypes = [C.c_uint, C.c_int] + [C.POINTER(C.c_uint64)] * 3
    L.swar_pairs.argtypes = [C.c_size_t, C.c_uint]
    L.swar_pairs.restype = C.c_uint64
    L.swar_batch_decomp.argtypes = [u8p, u8p, C.c_size_t, C.c_uint, u8p]
    L.swar_first_lane_in.argtypes = [u8p, C.c_size_t, C.c_uint64, C.c_uint64]
    L.swar_first_lane_in.restype = C.c_uint64
    L.oracle_exhaustive_verdicts.argtypes = [C.c_int, u8p]
    L.exhaustive_inputs.argtypes = [C.c_int, u8p]
    L.oracle_batch.argtypes = [u8p, u8p, C.c_size_t, C.c_int, u8p, u8p, u8p]
    L.oracle_cp_sweep.argtypes = [C.POINTER(C.c_uint64)] * 3
    L.swar_lanes.argtypes = [u8p, C.c_size_t, C.c_uint64, C.c_uint64]
    L.swar_lanes.restype = C.c_int
    return L


def oracle_batch(data: np.ndarray, offsets: np.ndarray, threads: int = 0, with_positions: bool = False):
    """Per-record oracle verdicts (uint8), optionally first-error offsets/kinds."""
    import os
    data = np.ascontiguousarray(data, np.uint8)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    n = offsets.size - 1
    valid = np.empty(n, np.uint8)
    eoff = np.empty(n, np.uint64) if with_positions else None
    kind = np.empty(n, np.int32) if with_positions else None
    threads = threads or min(64, os.cpu_count() or 1)
    swar().oracle_batch(data.ctypes.data if data.size else None, offsets.ctypes.data, n, threads,
                        valid.ctypes.data, eoff.ctypes.data if eoff is not None else None,
                        kind.ctypes.data if kind is not None else None)
    return (valid, eoff, kind) if with_positions else valid


def exhaustive(length: int):
    """(inputs back to back, oracle verdicts) for every input of `length` bytes."""
    total = 1 if length == 0 else 1 << (8 * length)
    data = np.empty(total * length, np.uint8)
    ver = np.empty(total, np.uint8)
    swar().exhaustive_inputs(length, data.ctypes.data if data.size else None)
    swar().oracle_exhaustive_verdicts(length, ver.ctypes.data)
    return data, ver


def _buf(data):
    a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else np.ascontiguousarray(data, np.uint8)
    return a, (a.ctypes.data if a.size else None), int(a.size)


def oracle_verdict(data, threads: int = 1):
    """(valid, offset, kind) from the C restatement of oracle_validate."""
    a, p, n = _buf(data)
    off, kind = C.c_uint64(0), C.c_int(-1)
    if threads > 1:
        ok = oracle().orc_validate_mt(p, n, threads, C.byref(off), C.byref(kind))
    else:
        ok = oracle().orc_validate(p, n, C.byref(off), C.byref(kind))
    return (True, None, None) if ok else (False, off.value, kind.value)


def ref_verdict(data):
    L = ref()
    a, p, n = _buf(data)
    off, kind = C.c_uint64(0), C.c_int(-1)
    ok = L.ref_oracle_validate(p, n, C.byref(off), C.byref(kind))
    return (True, None, None) if ok else (False, off.value, kind.value)


def generate_valid(kinds_mask: int, target: int, seed: int) -> bytes:
    cap = target + 8
    out = (C.c_uint8 * cap)()
    n = oracle().orc_generate_valid(kinds_mask, target, seed, out, cap)
    return bytes(out[:n])


def generate_invalid(kinds_mask: int, target: int, seed: int, strategy: int) -> bytes:
    cap = max(target, 1) + 16
    out = (C.c_uint8 * cap)()
    n = oracle().orc_generate_invalid(kinds_mask, target, seed, strategy, out, cap)
    return bytes(out[:n])


def nibble_tables():
    t = [(C.c_uint8 * 16)() for _ in range(3)]
    oracle().orc_nibble_tables(*t)
    return [bytes(x) for x in t]
