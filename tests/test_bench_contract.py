"""bench.py's JSON-line contract: the reference arm on CPU (it times the
oracle port on host cores) and this repository's arm on a GPU."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], 600)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1
    assert d["config"]["workload"]
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_own_arm_line():
    d = _run(["--no-extras", "--no-cpu-baseline", "--steps", "5", "--warmup", "3"], 900)
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] != d["value"]
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= rf.keys()
    assert 0 < rf["frac"] <= 1 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-6
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()


def test_gpus_flag_self_launches_ranks():
    """`--gpus N` without a torchrun environment launches N local ranks
    itself (torch.distributed.run on 127.0.0.1) and relays rank 0's line,
    which must report N GPUs. CPU: the reference arm (rank 0 works, the
    other ranks exit)."""
    d = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-sample", "2048"], 600)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["same_config"] is False


def test_reference_arm_full_batch_is_same_config():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], 900)
    assert d["config"]["same_config"] is True and d["config"]["batch_per_gpu"] == 65536
