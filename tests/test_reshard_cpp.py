"""The C++ face of the reshard module (include/coadapt/reshard.hpp):
tests/cpp/reshard_main.cpp links libcoadapt_b200.so; its plan CSV must equal
the oracle's (CPU), and DevicePlan all/pull/push must reproduce the global
tensors in every destination pack over 64 strategy pairs (GPU)."""
import os
import shutil
import subprocess

import pytest

from oracle import reshard_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIBDIR = os.path.join(ROOT, "paper_2604_26687_b200", "lib")
CXX = shutil.which("g++", path="/usr/bin") or shutil.which("g++")
CUDA = "/usr/local/cuda"


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("reshard") / "reshard_main")
    cmd = [CXX, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           os.path.join(HERE, "cpp", "reshard_main.cpp"), "-L", LIBDIR, "-lcoadapt_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64",
           "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return out


def test_cpp_plan_csv_matches_oracle(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    csv = "\n".join(l for l in lines if not l.startswith("#")) + "\n"
    m = O.Model(4, [O.Tensor("qkv", (96, 40), 0), O.Tensor("out", (40, 96), 1),
                    O.Tensor("norm", (40,), -1), O.Tensor("conv", (8, 6, 24), 2)])
    a, b = O.layout_for(m, (1, 2, 2)), O.layout_for(m, (2, 1, 2))
    mv, tot, mx, loc = O.plan_transfers(m, a, b)
    assert csv == O.plan_csv(m, mv)
    meta = dict(kv.split("=") for kv in lines[-2][1:].split())
    assert (int(meta["total"]), int(meta["max"]), int(meta["local"])) == (tot, mx, loc)
    assert float(meta["latency"]) == O.estimate_reconfig_latency(tot, 1e9, 20.0)
    assert lines[-1] == "#validation ok"


@pytest.mark.gpu
def test_cpp_device_plan_all_pull_push(exe):
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK (0 failures)"), r.stdout[-3000:] + r.stderr
