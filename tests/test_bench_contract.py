"""bench.py's driver contract on the CPU side: the reference arm
(`--impl reference`, the oracle on the host cores) prints one JSON line with
the keys the driver reads, rank > 0 of a torchrun launch exits 0 without
work, and the defaults select the headline configuration."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module")
def ref_line():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line(ref_line):
    L = ref_line
    assert L["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in L, k
    assert L["unit"] == "GB/s" and L["higher_is_better"] is True and L["value"] > 0
    assert L["cpu_baseline"]["value"] == L["value"] and L["cpu_baseline"]["kind"] in ("port", "reference")
    assert L["cpu_baseline"]["cores"] >= 1
    assert L["e2e"] == {"value": L["value"], "unit": L["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "workload" in L["config"] and "sample" in L["config"]


def test_reference_arm_same_metric_as_ours(ref_line):
    sys.path.insert(0, ROOT)
    import bench
    assert ref_line["metric"] == bench.METRIC and ref_line["unit"] == bench.UNIT


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"],
             {"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]


def test_defaults_select_the_headline_config(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.gpus, a.config, a.impl) == (1, "c4", "ours")
    assert a.warmup >= 3 and a.steps >= 1
    assert a.x1 == "p2p" and a.finalize == "inpass"
    c = bench.CONFIGS["c4"]
    assert (c["shape"], c["d"], c["t"], c["p"], c["M"], c["dtype"]) == ("32b", 1, 4, 2, 16, "bf16")
