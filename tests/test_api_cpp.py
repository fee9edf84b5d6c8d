"""The reference's Lookup test plan through the C++ API (tests/cpp/api_test.cpp),
linked against libutf8v_cuda.so the way a reference caller would link it."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "api_test"


def _run(*args, timeout=900):
    if not BIN.exists():
        pytest.fail(f"{BIN} missing: run __graft_entry__.build()")
    return subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=timeout)


def test_cpp_api_links_and_roster_is_well_formed():
    # Needs no device: the roster is static (proj/src/lookup.cpp:28-31).
    r = _run("roster")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS backend roster" in r.stdout


@pytest.mark.gpu
def test_cpp_api_reference_test_plan():
    r = _run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout, r.stdout
