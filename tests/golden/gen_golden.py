#!/usr/bin/env python3
"""Regenerate tests/golden/*.json from the UNMODIFIED reference library.

Needs oracle/_ref/libutf8v_ref.so, built from the reference sources by
oracle/Makefile (only possible where the reference checkout exists).  The
fixtures pin the oracle restatement (oracle/utf8_oracle.c) and, through it,
every GPU parity test:

  tables.json     nibble tables + the reference's frozen constants
                  (proj/tests/test_tables.cpp:26-34, :40-56, :77-103)
  known.json      known-answer verdicts of proj/tests/test_oracle.cpp:26-79
                  and whole-buffer cases of proj/tests/test_lookup.cpp:189-285
  lanes.json      lane outputs of the reference backends (avx2 width 32,
                  scalar width 16) for the worked example and seeded vectors
  corpora.json    generate_valid / generate_invalid corpora (seeds 100..111,
                  2048+seed bytes, proj/tests/test_lookup.cpp:338-354): size,
                  sha256 of the bytes, and the reference oracle's verdict
  digests.json    digests of large sweeps: every input of length <= 2, the
                  acceptance fuzz (seeds 1..20000 x 6 strategies, 64 bytes,
                  proj/tests/acceptance.cpp:263-272) -- verdict streams hashed

Usage: python tests/golden/gen_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from tests import _native as nat  # noqa: E402

KIND = ["header-bits", "too-short", "too-long", "overlong", "too-large", "surrogate"]


def ref_verdict(R, data: bytes):
    off, kind = C.c_uint64(0), C.c_int(-1)
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
    ok = R.ref_oracle_validate(buf if data else None, len(data), C.byref(off), C.byref(kind))
    return [True, None, None] if ok else [False, off.value, kind.value]


def ref_gen(R, fn, *args):
    cap = 1 << 16
    out = (C.c_uint8 * cap)()
    n = fn(*args, out, cap)
    assert n >= 0
    return bytes(out[:n])


def main() -> None:
    R = nat.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libutf8v_ref.so missing: build it with `make -C oracle ref`")

    # ---- tables --------------------------------------------------------
    t = [(C.c_uint8 * 16)() for _ in range(3)]
    R.ref_nibble_tables(*t)
    tables = {
        "table1": list(t[0]), "table2": list(t[1]), "table3": list(t[2]),
        "frozen_source": "proj/tests/test_tables.cpp:26-34",
    }
    pairs = {}
    for b1, b2 in [(0xC0, 0x80), (0x39, 0x80), (0xED, 0xA0), (0xF4, 0x90), (0xC3, 0x39), (0x80, 0x80),
                   (0xE5, 0xA0), (0xC3, 0xA7)]:
        pairs[f"{b1:02X}{b2:02X}"] = t[0][b1 >> 4] & t[1][b1 & 15] & t[2][b2 >> 4]
    tables["pairs"] = pairs  # proj/tests/test_tables.cpp:40-56
    (HERE / "tables.json").write_text(json.dumps(tables, indent=1))

    # ---- known answers -------------------------------------------------
    cases = [
        # proj/tests/test_oracle.cpp:26-44 (accepted)
        "", "39", "C3A7", "E98FA1", "F09F9880", "EFBBBF39", "7F", "C280", "DFBF", "E0A080", "ED9FBF",
        "EE8080", "EFBFBF", "F0908080", "F48FBFBF",
        # proj/tests/test_oracle.cpp:46-79 (rejected, offset + kind)
        "3980", "EDB880", "F4908080", "E081A1", "FA90908080", "E98F39", "39E98F", "C3", "E03030", "80FF",
        "C080", "C1BF", "F880808080", "FF", "39EDA08039",
        # proj/tests/test_lookup.cpp:189-201
        "39C3A7E98FA1F09F988000", "80",
    ]
    known = []
    for h in cases:
        d = bytes.fromhex(h)
        known.append({"hex": h, "verdict": ref_verdict(R, d), "lookup": bool(R.ref_validate_lookup(d, len(d)))})
    # test_lookup.cpp:203-285 shapes
    shapes = {
        "early_error": b"\x80" + b"A" * 511,
        "late_error": b"A" * 511 + b"\x80",
        "pending_incomplete": b"A" * 62 + bytes([0xE9, 0x8F]) + b"A" * 64,
        "ascii_block_then_stray": b"A" * 61 + bytes([0xE9, 0x8F, 0xA1]) + b"A" * 64 + b"\x80" + b"A" * 20,
        "ascii_block_then_valid": b"A" * 61 + bytes([0xE9, 0x8F, 0xA1]) + b"A" * 64 + bytes([0xC3, 0xA7]),
        "cut_at_block": b"A" * 63 + bytes([0xE9]),
        "full_block": b"A" * 61 + bytes([0xE9, 0x8F, 0xA1]),
    }
    for name, d in shapes.items():
        known.append({"name": name, "hex": d.hex(), "verdict": ref_verdict(R, d),
                      "lookup": bool(R.ref_validate_lookup(d, len(d)))})
    (HERE / "known.json").write_text(json.dumps({"source": "reference oracle_validate + validate_lookup",
                                                 "cases": known}, indent=1))

    # ---- lanes ---------------------------------------------------------
    import random
    rng = random.Random(20101006)
    lanes = {"backends": {}}
    for i in range(R.ref_backend_count()):
        name = R.ref_backend_name(i).decode()
        w = R.ref_backend_width(i)
        rows = []
        vecs = [(bytes([0x39, 0xC3, 0xA7, 0xE9, 0x8F, 0xA1, 0xF0, 0x9F, 0x98, 0x80, 0x00]).ljust(w, b"\0"), bytes(w))]
        for _ in range(64):
            vecs.append((bytes(rng.randrange(256) for _ in range(w)), bytes(rng.randrange(256) for _ in range(w))))
        for a, p in vecs:
            A = (C.c_uint8 * w).from_buffer_copy(a)
            P = (C.c_uint8 * w).from_buffer_copy(p)
            o1, o2, o3 = (C.c_uint8 * w)(), (C.c_uint8 * w)(), (C.c_uint8 * w)()
            R.ref_backend_classify(i, A, P, o1)
            R.ref_backend_length_error(i, A, P, o2)
            R.ref_backend_incomplete(i, A, o3)
            rows.append({"in": a.hex(), "prev": p.hex(), "classify": bytes(o1).hex(),
                         "length_error": bytes(o2).hex(), "incomplete": bytes(o3).hex()})
        lanes["backends"][name] = {"width": w, "rows": rows,
                                   "self_test": [bool(R.ref_backend_self_test(i, s))
                                                 for s in (1, 0xDEADBEEF, 0x123456789ABCDEF)]}
    (HERE / "lanes.json").write_text(json.dumps(lanes))

    # ---- corpora -------------------------------------------------------
    corpora = []
    for seed in range(100, 112):
        target = 2048 + seed
        items = [("valid", -1, ref_gen(R, R.ref_generate_valid, 15, target, seed))]
        for s in range(6):
            items.append(("invalid", s, ref_gen(R, R.ref_generate_invalid, 15, target, seed, s)))
        for kind, strat, d in items:
            corpora.append({"seed": seed, "target": target, "strategy": strat, "size": len(d),
                            "sha256": hashlib.sha256(d).hexdigest(), "verdict": ref_verdict(R, d)})
    (HERE / "corpora.json").write_text(json.dumps({"kinds_mask": 15, "items": corpora}, indent=1))

    # ---- digests -------------------------------------------------------
    h = hashlib.sha256()
    nvalid = 0
    for n in (0, 1, 2):
        for v in range(1 << (8 * n)):
            d = bytes((v >> (8 * i)) & 0xFF for i in range(n))
            ok = ref_verdict(R, d)
            h.update(json.dumps(ok).encode())
            nvalid += ok[0]
    short = {"lengths": [0, 1, 2], "count": 1 + 256 + 65536, "valid": nvalid, "sha256": h.hexdigest()}
    hf = hashlib.sha256()
    bytes_h = hashlib.sha256()
    for seed in range(1, 20001):
        for s in range(6):
            d = ref_gen(R, R.ref_generate_invalid, 15, 64, seed, s)
            bytes_h.update(d)
            hf.update(json.dumps(ref_verdict(R, d)).encode())
    fuzz = {"seeds": [1, 20000], "strategies": 6, "target": 64, "bytes_sha256": bytes_h.hexdigest(),
            "verdicts_sha256": hf.hexdigest()}
    (HERE / "digests.json").write_text(json.dumps({"short_inputs": short, "fuzz": fuzz}, indent=1))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
