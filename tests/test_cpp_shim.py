"""The header-only C++ shim (include/moeless/b200_layer.hpp) compiles against
the reference API surface, and a reference-style caller (examples/layer_loop.cpp,
the simulator.cpp:116-201 loop with the real layer) runs on the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_example_builds():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2603_06350_b200", "csrc"), "examples"], check=True,
                   stdout=subprocess.DEVNULL)
    assert os.access(os.path.join(ROOT, "examples", "layer_loop"), os.X_OK)


@pytest.mark.gpu
def test_example_runs_reference_loop(cuda):
    exe = os.path.join(ROOT, "examples", "layer_loop")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2603_06350_b200", "csrc"), "examples"], check=True)
    out = subprocess.run([exe, "8", "2", "1024", "3584", "2048", "6"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["p50_ms"] > 0 and 0.5 < res["mean_accuracy"] <= 1.0
