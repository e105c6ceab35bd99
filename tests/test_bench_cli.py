"""bench.py's oracle arm (`--impl reference`, the base contract's reference arm for this
tier) runs on the CPU and prints one JSON line with the contract's keys; under
torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=dict(os.environ, **(env or {})))
    assert p.returncode == 0, p.stderr[-2000:]
    return p.stdout


def test_reference_arm_json_line():
    out = _run(["--impl", "reference", "--workload", "c1", "--steps", "2", "--warmup", "1"])
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # measured seconds per step; the extrapolation is a separate key
    assert d["oracle_detail"]["measured_s_per_step"] * 1000.0 == d["ms_per_step"]
    assert d["oracle_detail"]["extrapolated_full_workload_s"] > 0


def test_reference_arm_other_ranks_silent():
    out = _run(["--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0"], env={"RANK": "3"})
    assert out.strip() == ""
