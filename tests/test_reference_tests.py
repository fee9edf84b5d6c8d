"""The reference's own unit tests (proj/tests/test_lookup.cpp, test_oracle.cpp,
test_tables.cpp), unchanged, with the B200 path registered first in the
reference's backend roster (integration/reference_backend: lookup_cuda.cpp +
the one registration line; built by _build.build_reference_tests into the
git-ignored baseline/accept/).  The acceptance gate (proj/tests/acceptance.cpp)
is run separately (scripts/gpu_accept.sh, ~5 min; profiles/)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
UNIT = ROOT / "baseline" / "accept" / "unit_tests"


@pytest.mark.gpu
def test_reference_unit_tests_with_cuda_first_in_the_roster():
    if not UNIT.exists():
        pytest.skip("baseline/accept/unit_tests not built (no reference checkout where build() ran)")
    r = subprocess.run([str(UNIT)], capture_output=True, text=True, timeout=900)
    out = r.stdout
    assert r.returncode == 0, out[-3000:]
    assert "| 0 failed" in out.splitlines()[-1], out[-1000:]
    roster = subprocess.run([str(UNIT.parent / "roster")], capture_output=True, text=True, timeout=120).stdout.split()
    assert roster[0] == "cuda:64" and roster[-1] == "scalar:16", roster  # widest first, scalar last
