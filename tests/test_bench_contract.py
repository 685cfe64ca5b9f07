"""bench.py's reference arm (CPU) prints the contract's JSON line; the
argument parser keeps the driver's flags.  (The GPU arm is exercised by the
gpurun bench runs.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-sample-tokens", "4", "--cpu-full-layer", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert "workload" in line["config"]
    # the reference arm never maps the product library (only oracle/ and oracle/_ref)
    assert line["repo_libs_loaded"] and all(p.startswith("oracle/") for p in line["repo_libs_loaded"])
    sys.path.insert(0, ROOT)
    import bench
    assert line["config"] == bench.config_dict(1, bench.CFG)  # same config as the GPU arm's line


def test_parser_defaults():
    sys.path.insert(0, ROOT)
    import bench
    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = bench.parse()
    finally:
        sys.argv = old
    assert (a.gpus, a.impl, a.workload, a.exchange) == (1, "ours", "cfg2", "p2p")
    assert a.steps >= 200 and a.warmup >= 3
