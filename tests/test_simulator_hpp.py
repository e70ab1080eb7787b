"""The C++ drop-in include/rsim/simulator.hpp (SPEC signatures)
compiles against the C ABI, links lib/librsim.so and — on a B200 — runs one
localized-Newton timestep with the same result as the Python / C-ABI path."""
import os
import subprocess

import numpy as np
import pytest

import paper_2008_01539_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2008_01539_b200", "lib")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    pkg._abi.lib()  # built
    out = str(tmp_path_factory.mktemp("cpp") / "simulator_step")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "simulator_step.cpp"), "-o", out, "-L", LIBDIR, "-lrsim",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


def test_compiles_and_fails_loudly_without_gpu(exe):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = subprocess.run([exe], capture_output=True, text=True)
    assert p.returncode == 3 and "no device" in p.stdout, (p.returncode, p.stdout, p.stderr)


@pytest.mark.gpu
def test_one_localized_step_matches_c_abi(exe):
    p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, (p.stdout, p.stderr)
    kv = {ln.split()[0]: ln.split()[1:] for ln in p.stdout.strip().splitlines()}
    case = pkg.Case(1, nx=40, ny=40)
    s0 = case.init_state()
    dt = float(case.schedule()[3])
    opts = case.solver_opts()
    sim = pkg.GpuSimulator(case)
    sim.set_state(s0, dt)
    sim.initial_active(True, opts.eps_set, opts.m)
    va = sim.active()
    s1, rep = sim.newton_localized(s0, dt, va, opts.m, opts.eps_set, opts)
    sim.close()
    assert int(kv["va_init"][0]) == len(va)
    assert int(kv["iterations"][0]) == rep.iterations
    assert [int(x) for x in kv["n_active"]] == [r["n_active"] for r in rep.records()]
    seq = 0.0
    for v in s1.u[:: case.b].tolist():  # the C++ program sums left to right
        seq += v
    assert float(kv["p_sum"][0]) == seq
