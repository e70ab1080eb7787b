"""The C-ABI boundary: the product library and the oracle load on a CPU-only
host and export every function their headers declare; without a B200 the
GPU entry points fail loudly (no CPU fallback)."""
import re
from pathlib import Path

import pytest

import paper_2008_01539_b200 as pkg
from paper_2008_01539_b200 import _abi

ROOT = Path(__file__).resolve().parent.parent


def declared(header: Path) -> set[str]:
    txt = header.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(rsim_[a-z0-9_]+|orc_[a-z0-9_]+)\s*\(", txt))


def test_product_exports_every_declared_symbol():
    L = _abi.lib()
    names = declared(ROOT / "include/rsim/gpu_abi.h") | declared(ROOT / "include/rsim/cases.h") | \
        declared(ROOT / "include/rsim/simulate.h") | declared(ROOT / "include/rsim/eos.h")
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    assert names <= set(_abi.PROTOS), sorted(names - set(_abi.PROTOS))


def test_oracle_exports_every_declared_symbol():
    import oracle
    L = oracle.lib()
    names = declared(ROOT / "oracle/oracle_api.h")
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    c = pkg.Case(1, nx=8, ny=8)
    with pytest.raises(pkg.RsimError) as e:
        pkg.GpuSimulator(c)
    assert e.value.code == pkg.RSIM_ECUDA


def test_library_is_sm100a_only():
    import subprocess
    lib = ROOT / "paper_2008_01539_b200/lib/librsim.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    assert out.returncode == 0
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_case_generators_deterministic():
    a, b = pkg.Case(2, nx=32, ny=32, n_dfn=8), pkg.Case(2, nx=32, ny=32, n_dfn=8)
    import numpy as np
    assert np.array_equal(a.tx, b.tx) and np.array_equal(a.kind, b.kind)
    assert pkg.Case(1).n == 10000 and pkg.Case(2, n_steps=2).schedule().size == 2
    c3 = pkg.Case(3, nx=64, ny=64, nz=8)
    assert c3.b == 2 and (c3.kind == 1).sum() > 0 and (c3.well_wi > 0).sum() == 36
    c4 = pkg.Case(4, nx=64, ny=64, nz=4)
    assert c4.b == 3 and (c4.well_wi > 0).sum() == 20
