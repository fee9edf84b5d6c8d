"""The drop-in C-ABI library loads and exports every symbol include/*.h
declares (no compute calls: this runs without a GPU)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared_functions() -> set[str]:
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(utf8v_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_headers_declare_the_boundary():
    names = _declared_functions()
    for must in ("utf8v_cuda_validate", "utf8v_cuda_validate_verdict", "utf8v_cuda_validate_batch",
                 "utf8v_cuda_classify_lanes", "utf8v_cuda_length_error_lanes", "utf8v_cuda_incomplete_lanes",
                 "utf8v_cuda_ops_self_test", "utf8v_cuda_validate_lanes_async",
                 "utf8v_cuda_validate_batch_async"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2010_03090_b200 import _lib
    lib = _lib.load()
    missing = [n for n in sorted(_declared_functions()) if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol is also typed in the Python binding
    assert set(_declared_functions()) <= set(_lib.SIGNATURES), set(_declared_functions()) - set(_lib.SIGNATURES)


def test_abi_version_and_empty_input_without_device():
    from paper_2010_03090_b200 import _lib
    lib = _lib.load()
    assert lib.utf8v_cuda_abi_version() == 6
    out = C.c_uint8(0)
    # n == 0 is valid text without touching the device (test_lookup.cpp:192)
    assert lib.utf8v_cuda_validate(None, 0, 0, C.byref(out)) == 0 and out.value == 1


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2010_03090_b200 import _lib
    import paper_2010_03090_b200 as u8
    with pytest.raises(_lib.CudaBackendError) as e:
        u8.validate_lookup(b"abc")
    assert e.value.status == _lib.UTF8V_ERR_NO_DEVICE


def test_cxx_api_header_mirrors_reference_names():
    text = (ROOT / "include" / "utf8v" / "lookup.hpp").read_text()
    for name in ("struct lookup_backend", "lookup_backends()", "find_lookup_backend(", "validate_lookup(",
                 "validate_lookup_fallback(", "classify_lanes", "length_error_lanes", "incomplete_lanes",
                 "ops_self_test"):
        assert name in text
    v = (ROOT / "include" / "utf8v" / "verdict.hpp").read_text()
    for name in ("enum class error_kind", "header_bits", "too_short", "too_long", "overlong", "too_large",
                 "surrogate", "struct verdict", "struct utf8_error", "using bytes_view"):
        assert name in v


def test_library_is_built_for_sm100a():
    import subprocess
    import shutil
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([cuobjdump, "--list-elf", str(ROOT / "paper_2010_03090_b200" / "libutf8v_cuda.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_views_of_every_input_kind():
    """Host input may be bytes, bytearray, memoryview, numpy (also strided) or
    a CPU torch tensor (also strided): one contiguous uint8 view each."""
    import numpy as np
    import torch
    from paper_2010_03090_b200 import _host_view
    raw = bytes(range(16))
    cases = [raw, bytearray(raw), memoryview(raw), np.frombuffer(raw, np.uint8),
             torch.tensor(list(raw), dtype=torch.uint8)]
    for c in cases:
        ptr, n, keep = _host_view(c)
        assert n == 16 and bytes(keep) == raw
    ptr, n, keep = _host_view(np.arange(16, dtype=np.uint8)[::2])
    assert n == 8 and list(keep) == list(range(0, 16, 2))
    ptr, n, keep = _host_view(torch.arange(16, dtype=torch.uint8)[::2])
    assert n == 8 and list(keep) == list(range(0, 16, 2))
    assert _host_view(b"")[:2] == (None, 0)
