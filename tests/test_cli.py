"""utf8v-cuda: the reference CLI's validate/bench commands on the B200 path
(proj/tools/main.cpp; exit codes :28-31, report schema proj/src/bench.cpp:127-139)."""
import json
import subprocess
from pathlib import Path

import pytest

CLI = Path(__file__).resolve().parents[1] / "paper_2010_03090_b200" / "bin" / "utf8v-cuda"


def run(*args, stdin=b""):
    if not CLI.exists():
        pytest.fail(f"{CLI} missing: run __graft_entry__.build()")
    return subprocess.run([str(CLI), *map(str, args)], input=stdin, capture_output=True, timeout=600)


def test_usage_exit_codes():
    assert run("--help").returncode == 0
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("validate", "--algo", "fsm").returncode == 2
    assert run("bench", "--size").returncode == 2
    assert run("validate", "/nonexistent/file").returncode == 2


@pytest.mark.gpu
def test_validate_verdicts_and_json(tmp_path):
    good = tmp_path / "good.txt"
    good.write_bytes("héllo wörld €𝄞".encode())
    bad = tmp_path / "bad.txt"
    bad.write_bytes(b"hello\xe0\x80\xafx")
    r = run("validate", good)
    assert (r.returncode, r.stdout) == (0, b"valid\n")
    r = run("validate", bad)
    assert r.returncode == 1 and r.stdout == b"invalid: overlong at offset 5\n"
    r = run("validate", "--json", bad)
    assert r.returncode == 1 and json.loads(r.stdout) == {"valid": False, "offset": 5, "kind": "overlong"}
    r = run("validate", "--algo=cuda", "--json", stdin=b"\xc3")
    assert r.returncode == 1 and json.loads(r.stdout) == {"valid": False, "offset": 0, "kind": "too-short"}
    assert run("validate", stdin=b"").returncode == 0


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
def test_bench_report_schema(device):
    args = ["bench", "--size", 1 << 22, "--seed", 2, "--repeats", 3, "--json"] + (["--device"] if device else [])
    r = run(*args)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert isinstance(rep, list) and len(rep) == 1
    assert set(rep[0]) == {"validator", "input_name", "input_bytes", "repeats", "best_seconds", "mean_seconds",
                           "best_throughput", "mean_throughput", "compensated"}
    assert rep[0]["input_bytes"] == 1 << 22 and rep[0]["repeats"] == 3
    assert rep[0]["best_throughput"] >= rep[0]["mean_throughput"] > 0


@pytest.mark.gpu
def test_bench_compensate(tmp_path):
    r = run("bench", "--size", 1 << 22, "--repeats", 3, "--compensate", "--json")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)[0]
    assert rep["compensated"] is True and rep["mean_seconds"] >= rep["best_seconds"] >= 0
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"ok\xc0\x80")
    r = run("bench", "--file", bad, "--compensate")   # compensation needs well-formed input
    assert r.returncode == 2
