"""In-tree native build: nvcc for sm_100a, g++ for the host pieces.

Products (git-ignored, they travel to the GPU box with the snapshot):
  paper_2010_03090_b200/libutf8v_cuda.so   kernels + C-ABI + C++ API
Test infrastructure (built here too, never loaded by the product):
  oracle/liboracle.so, oracle/_ref/libutf8v_ref.so   (oracle/Makefile)
  tests/cpp/libswar_host.so   the SWAR header compiled for the CPU checker
  tests/cpp/api_test          C++ API test program (reference-style asserts)
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libutf8v_cuda.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3",
                     f"-I{ROOT / 'include'}", "--expt-relaxed-constexpr"]
CU_SOURCES = ["validate.cu", "batch.cu", "lanes.cu", "gen.cu", "stream.cu", "capi.cu", "comm.cu", "serve.cu"]
CXX_SOURCES = ["lookup.cpp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolchain is required to build libutf8v_cuda.so")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], cwd: Path | None = None) -> None:
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build_cuda(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").rglob("*.h*"))
    objs: list[Path] = []
    jobs = []
    for src in CU_SOURCES + CXX_SOURCES:
        s = CSRC / src
        o = BUILD / (src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *NVCC_FLAGS, "-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    if force or _stale(LIB, objs):
        _run([nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-ldl"])
    if verbose:
        print(f"built {LIB}")
    return LIB


CLI = PKG / "bin" / "utf8v-cuda"


def build_cli() -> Path:
    """tools/utf8v_cuda_cli.cpp -> paper_2010_03090_b200/bin/utf8v-cuda (the
    reference CLI's validate/bench on the C++ API)."""
    src = ROOT / "tools" / "utf8v_cuda_cli.cpp"
    if src.exists() and _stale(CLI, [src, LIB, ROOT / "include" / "utf8v" / "lookup.hpp"]):
        CLI.parent.mkdir(exist_ok=True)
        cuda = Path(_nvcc()).resolve().parents[1]
        _run(["g++", "-O2", "-std=c++20", f"-I{ROOT / 'include'}", f"-I{cuda / 'include'}", "-o", str(CLI),
              str(src), f"-L{PKG}", "-lutf8v_cuda", f"-L{cuda / 'lib64'}", "-lcudart",
              f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/.."])
    return CLI


def build_oracle() -> None:
    """oracle/ checkers (test infrastructure). `make ref` is a no-op without
    the reference checkout (the GPU box uses the prebuilt oracle/_ref)."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "oracle"])
    if Path("/root/reference/proj/src/oracle.cpp").exists():
        _run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"])


def build_test_helpers() -> None:
    cpp = ROOT / "tests" / "cpp"
    swar_src = cpp / "swar_host.c"
    swar_lib = cpp / "libswar_host.so"
    deps = [swar_src, CSRC / "utf8v_swar.h", CSRC / "utf8v_bits.h", CSRC / "utf8v_stream.h",
            ROOT / "oracle" / "utf8_oracle.h"]
    if swar_src.exists() and _stale(swar_lib, deps):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-std=c99", "-pthread", f"-I{CSRC}",
              f"-I{ROOT / 'oracle'}", "-o", str(swar_lib), str(swar_src),
              str(ROOT / "oracle" / "utf8_oracle.c")])
    api_src = cpp / "api_test.cpp"
    api_bin = cpp / "api_test"
    if api_src.exists() and _stale(api_bin, [api_src, LIB, ROOT / "include" / "utf8v" / "lookup.hpp"]):
        _run(["g++", "-O2", "-std=c++20", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle'}",
              "-o", str(api_bin), str(api_src), str(ROOT / "oracle" / "utf8_oracle.c"),
              f"-L{PKG}", "-lutf8v_cuda", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../../paper_2010_03090_b200",
              "-pthread"])


def build_reference_tests() -> None:
    """The reference's own unit tests and acceptance gate with the cuda entry
    first in its roster (integration/reference_backend/build.sh; outputs in
    the git-ignored baseline/accept/).  A no-op without the reference
    checkout: the GPU box uses the prebuilt binaries."""
    script = ROOT / "integration" / "reference_backend" / "build.sh"
    if script.exists() and Path("/root/reference/proj/src/lookup.cpp").exists():
        _run(["bash", str(script)])


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force=force, verbose=verbose)
    build_cli()
    build_oracle()
    build_test_helpers()
    build_reference_tests()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
