"""The drop-in at the reference's own call site.

examples/Makefile compiles the UNMODIFIED reference sources
(/root/reference/proj/src/*.cpp against /root/reference/proj/include) twice:
sim_ref as shipped, and sim_b200 with exactly one line of simulator.cpp
changed (:194, layer_forward_time -> b200::layer_forward_time from the
force-included include/moeless/b200_layer.hpp), linked against
libmoe_b200.so.  Both run the reference's run() on the same config + trace
(tests/golden/dropin.*): the planning decisions (replicas, warm/cold, the
predictor's accuracy, bootstrap uses) are the reference's own in both, and
sim_b200's forward times are measured on the B200 (2 expert-parallel ranks).
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "examples", "_build")
GOLD = os.path.join(ROOT, "tests", "golden")
REF_SIM = "/root/reference/proj/src/simulator.cpp"
CFG, TRACE = os.path.join(GOLD, "dropin.config"), os.path.join(GOLD, "dropin.trace")


def _build():
    if os.path.exists(REF_SIM):
        subprocess.run(["make", "-C", os.path.join(ROOT, "examples"), "-j4"], check=True, stdout=subprocess.DEVNULL)
    for exe in ("sim_ref", "sim_b200"):
        if not os.access(os.path.join(BUILD, exe), os.X_OK):
            pytest.skip("reference sources absent and examples/_build not prebuilt")


def parse(out):
    import json
    head, csv = out.split("---\n")
    rows = [line.split(",") for line in csv.strip().splitlines()[1:]]
    samples = [dict(iteration=int(r[0]), layer=int(r[1]), forward_ms=float(r[3]), replicas=int(r[4]),
                    warm=int(r[5]), cold=int(r[6])) for r in rows]
    return json.loads(head), samples


def test_dropin_is_a_one_line_patch():
    _build()
    if not os.path.exists(REF_SIM):
        pytest.skip("reference sources absent")
    a = open(REF_SIM).read().splitlines()
    b = open(os.path.join(BUILD, "simulator_b200.cpp")).read().splitlines()
    assert len(a) == len(b)
    diff = [i for i, (x, y) in enumerate(zip(a, b)) if x != y]
    assert diff == [193]  # line 194, 1-based
    assert "b200::layer_forward_time(plan, placement, actual[l], config.cluster, config.model)" in b[193]


def test_library_exports_only_the_c_abi():
    """libmoe_b200.so keeps its planner restatement local, so linking it next to
    the reference's own planner objects (as sim_b200 does) cannot interpose."""
    if not shutil.which("nm"):
        pytest.skip("nm absent")
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2603_06350_b200",
                                                                     "libmoe_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    names = [line.split()[-1] for line in out.splitlines() if line.strip()]
    assert names and all(n.startswith("moe_") for n in names), [n for n in names if not n.startswith("moe_")]


def test_reference_simulator_unchanged_output():
    """sim_ref (the reference as shipped) reproduces the committed golden run."""
    _build()
    out = subprocess.run([os.path.join(BUILD, "sim_ref"), CFG, TRACE], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout == open(os.path.join(GOLD, "dropin_ref_output.txt")).read()


@pytest.mark.gpu
def test_reference_run_with_the_b200_layer(cuda):
    _build()
    ref_sum, ref_rows = parse(open(os.path.join(GOLD, "dropin_ref_output.txt")).read())
    env = dict(os.environ, MOE_B200_D_MODEL="1024", MOE_B200_D_FF="3584")
    out = subprocess.run([os.path.join(BUILD, "sim_b200"), CFG, TRACE], capture_output=True, text=True,
                         timeout=600, env=env)
    assert out.returncode == 0, out.stderr
    b_sum, b_rows = parse(out.stdout)
    # the reference's planning decisions are untouched by the swap
    for key in ("policy", "iterations", "num_layers", "mean_replicas_per_layer", "warm_total", "cold_total",
                "layer_mean_replicas", "layer_mean_accuracy", "layer_bootstrap_uses"):
        assert b_sum[key] == ref_sum[key], key
    assert [(r["iteration"], r["layer"], r["replicas"], r["warm"], r["cold"]) for r in b_rows] == \
        [(r["iteration"], r["layer"], r["replicas"], r["warm"], r["cold"]) for r in ref_rows]
    # forward times are measured: MoE layer on the GPU + the reference's t_misc (0.5 ms)
    assert all(r["forward_ms"] > 0.5 for r in b_rows)
    assert [r["forward_ms"] for r in b_rows] != [r["forward_ms"] for r in ref_rows]
    assert b_sum["p99_forward_ms"] < 50.0
    print(f"sim_b200: p50 {b_sum['p50_forward_ms']:.4f} ms, p99 {b_sum['p99_forward_ms']:.4f} ms "
          f"(analytic reference: {ref_sum['p50_forward_ms']:.4f} / {ref_sum['p99_forward_ms']:.4f})")


CPP_IDS_TEST = r"""
#include <cstdio>
#include <random>
#include <set>
#include "moeless/b200_layer.hpp"
int main() {
  std::mt19937_64 rng(7);
  for (int trial = 0; trial < 500; ++trial) {
    const int E = 1 + rng() % 64, k = 1 + rng() % std::min(E, 8);
    const long T = rng() % 300;
    // random histogram with sum T*k and every load <= T: k distinct experts per token
    std::vector<std::int64_t> loads(E, 0);
    for (long t = 0; t < T; ++t) {
      std::set<int> pick;
      while ((int)pick.size() < k) pick.insert(rng() % E);
      for (int e : pick) ++loads[e];
    }
    std::int64_t tokens = -1;
    const auto ids = moeless::b200::ids_for_loads(loads, k, &tokens);
    if (tokens != T) return 1;
    std::vector<std::int64_t> h(E, 0);
    for (long t = 0; t < T; ++t) {
      std::set<int> row;
      for (int j = 0; j < k; ++j) { row.insert(ids[t * k + j]); ++h[ids[t * k + j]]; }
      if ((int)row.size() != k) return 2;  // distinct experts per token
    }
    if (h != loads) return 3;             // the histogram is exactly the loads
  }
  try { moeless::b200::ids_for_loads({5, 1}, 2, nullptr); return 4; } catch (const std::invalid_argument&) {}
  std::puts("ids_for_loads ok");
  return 0;
}
"""


def test_ids_for_loads_reproduces_any_histogram(tmp_path):
    """b200::layer_forward_time turns the reference's per-expert loads into
    per-token ids: the histogram must be exact and no token may repeat an expert
    (route_tokens draws without replacement, workload.cpp:221-226)."""
    if not os.path.exists("/root/reference/proj/include/moeless/types.hpp"):
        pytest.skip("reference headers absent")
    src = tmp_path / "ids.cpp"
    src.write_text(CPP_IDS_TEST)
    exe = tmp_path / "ids"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I/root/reference/proj/include", "-I" + os.path.join(ROOT, "include"),
                    "-I/usr/local/cuda/include", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and "ids_for_loads ok" in out.stdout, (out.returncode, out.stdout)
