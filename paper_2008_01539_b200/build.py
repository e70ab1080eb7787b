"""Build the sm_100a product library (lib/librsim.so) and the CPU oracle.

Everything is compiled in-tree with explicit nvcc/g++ command lines so the
built .so files travel to the GPU box with the repo snapshot:

  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false ...

--fmad=false (device) and -ffp-contract=off (host) keep every a*b+c as two
roundings on both sides, which together with include/rsim/physics.h's rexp()
is what makes the GPU results bit-identical to oracle/ (DESIGN.md §Parity).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib" / "librsim.so"
OBJ = PKG / "lib" / "obj"
ORACLE = ROOT / "oracle"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
HOSTCXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-ccbin", HOSTCXX,
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp,-O3",
    "-Xptxas", "-v" if os.environ.get("RSIM_PTXAS_V") else "-O3",
    "-I", str(ROOT / "include"), "-I", str(CSRC),
]
SOURCES = ["abi.cu", "assemble.cu", "krylov.cu", "krylov_dsm.cu", "krylov_gmres.cu", "ilu.cu", "sets.cu", "solvers.cpp", "cases.cpp", "edfm.cpp", "simulate.cpp", "eos.cu", "direct.cu"]
CLI = PKG / "lib" / "simulate"


def _run(cmd: list[str]) -> str:
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"command failed ({p.returncode}): {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return p.stdout + p.stderr


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _headers() -> list[Path]:
    return sorted((ROOT / "include" / "rsim").glob("*.h")) + sorted(CSRC.glob("*.cuh"))


def build_product(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdrs = _headers()

    def one(src: str) -> Path:
        s = CSRC / src
        o = OBJ / (src + ".o")
        if force or _stale(o, [s] + hdrs):
            out = _run([NVCC, *NVFLAGS, "-c", str(s), "-o", str(o)])
            if verbose and out.strip():
                print(out)
        return o

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, SOURCES))
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-ccbin", HOSTCXX, *map(str, objs), "-o", str(LIB), "-lgomp"])
    main = CSRC / "simulate_main.cpp"
    if force or _stale(CLI, [main, LIB] + hdrs):  # the case-runner CLI (SPEC.md sim_driver_cli)
        _run([HOSTCXX, "-O2", "-std=c++17", "-I", str(ROOT / "include"), str(main), "-o", str(CLI),
              "-L", str(LIB.parent), "-lrsim", "-Wl,-rpath,$ORIGIN"])
    return LIB


def build_oracle(force: bool = False) -> Path:
    # the oracle links its own copy of the host-only case generator (csrc/cases.cpp,
    # include/rsim/cases.h) so the CPU reference arm never loads librsim.so
    out = ORACLE / "_build" / "liborsim.so"
    deps = [ORACLE / "oracle.cpp", ORACLE / "oracle_api.h", CSRC / "cases.cpp", CSRC / "edfm.cpp",
            CSRC / "case_impl.h"] + _headers()
    if force or _stale(out, deps):
        out.parent.mkdir(parents=True, exist_ok=True)
        _run([HOSTCXX, "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-shared",
              "-I", str(ROOT / "include"), str(ORACLE / "oracle.cpp"), str(CSRC / "cases.cpp"), str(CSRC / "edfm.cpp"), "-I", str(CSRC), "-o", str(out)])
    return out


def build(force: bool = False, verbose: bool = False) -> None:
    build_product(force=force, verbose=verbose)
    build_oracle(force=force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
