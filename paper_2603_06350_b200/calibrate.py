"""Calibrate the reference's analytic cost model from B200 measurements.

The reference prices a layer as  forward = alpha * max_share + 2 * beta *
max_gpu_tokens + t_misc  (proj/src/cost_model.cpp:114-117) with alpha/beta/
t_misc as free "calibration knobs" (types.hpp:14-15).  This module measures
them on the real B200 layer so the reference's planner studies (policy
comparison, sweeps, acceptance checks) run on hardware coefficients:

  alpha   ms per routed token of one expert replica owning a B200: slope of the
          grouped-GEMM time (K4) against routed rows at the Mixtral shape
  t_misc  the layer's fixed part on the GPU: gate + plan + dispatch + combine
  beta    ms per token per exchange direction over NVLink 5: row bytes /
          measured peer bandwidth (770 GB/s per direction, B200_PROFILING.md) —
          derived, since the pool gives one GPU per call

  python -m paper_2603_06350_b200.calibrate measure --out calib.json   # on a B200
  python -m paper_2603_06350_b200.calibrate fit calib.json             # anywhere
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys

NVLINK_PEER_GBS = 770.0  # measured per-direction peer copy bandwidth (B200_PROFILING.md)


def measure(out_path: str, tokens=(1024, 2048, 4096, 8192, 16384), iters: int = 12):
    import numpy as np
    import torch

    from . import MOE_PLAN_SYNC, MoELayer
    from . import workload as wl
    E, k, d, ff = 8, 2, 4096, 14336
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(1, E, k, d, ff, max_tokens=max(tokens), expert_mem_mb=mem, layer_mem_cap_mb=4 * mem)
    for e in range(E):
        m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    rows = []
    for T in tokens:
        xs = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(2)]
        y = torch.empty((T, d), dtype=torch.int16, device="cuda")
        samples = []
        for it in range(iters):
            m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, it))
            st = m.forward(0, xs[it % 2], y, MOE_PLAN_SYNC, it, stats=True)
            if it >= 2:
                samples.append(st)
        med = lambda f: statistics.median(getattr(s, f) for s in samples)
        rows.append(dict(tokens=T, rows=T * k, gemm_ms=med("gemm1_ms") + med("gemm2_ms"),
                         fixed_ms=med("gate_ms") + med("plan_ms") + med("dispatch_ms") + med("combine_ms"),
                         forward_ms=med("forward_ms"),
                         max_expert_rows=statistics.median(max(s.counts[:E]) for s in samples)))
    m.close()
    res = dict(shape=dict(E=E, k=k, d=d, ff=ff), points=rows, device=torch.cuda.get_device_name(0))
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    return res


def fit(meas: dict) -> dict:
    pts = meas["points"]
    xs = [p["rows"] for p in pts]
    ys = [p["gemm_ms"] for p in pts]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    icpt = my - slope * mx
    ss_res = sum((y - (icpt + slope * x)) ** 2 for x, y in zip(xs, ys))
    ss_tot = sum((y - my) ** 2 for y in ys)
    d = meas["shape"]["d"]
    beta = d * 2 / (NVLINK_PEER_GBS * 1e9) * 1e3  # ms per token per direction
    return dict(alpha_ms_per_token=slope, gemm_intercept_ms=icpt, r2=1 - ss_res / ss_tot,
                t_misc_ms=statistics.median(p["fixed_ms"] for p in pts), beta_ms_per_token=beta,
                beta_source=f"derived: {d * 2} B per token row / {NVLINK_PEER_GBS} GB/s NVLink 5 peer bandwidth")


REFERENCE_KEYS = [  # the reference's flat config grammar (config.cpp:90-164), B200 values
    ("gpu_count", 8), ("gpu_mem_capacity_mb", 183359), ("m_misc_mb", 0),
    ("num_layers", 8), ("experts_per_layer", 16), ("top_k", 2), ("expert_mem_mb", 352),
    ("layer_mem_cap_mb", 2816), ("policy", "moeless"), ("predictor_kind", "noisy"),
    ("prediction_distance", 1), ("accuracy_profile", "ramp:0.70:0.95"), ("accuracy_threshold", 0.8),
    ("accuracy_distance_decay", 0.04), ("history_window", 8), ("cv_threshold", 0.2),
    ("cv_excludes_zero_loads", "false"), ("keep_alive_iters", 50), ("cold_start_ms", 0),
    ("placement_mode", "jsq"), ("eplb_period_iters", 600), ("zipf_exponent", 1.2), ("seed", 1),
]


def config_text(coeffs: dict, policy: str = "moeless") -> str:
    kv = dict(REFERENCE_KEYS)
    kv.update(alpha_ms_per_token=f"{coeffs['alpha_ms_per_token']:.9g}",
              beta_ms_per_token=f"{coeffs['beta_ms_per_token']:.9g}", t_misc_ms=f"{coeffs['t_misc_ms']:.9g}",
              policy=policy)
    return "".join(f"{k} = {v}\n" for k, v in kv.items())


def main(argv=None):
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("measure")
    a.add_argument("--out", required=True)
    b = sub.add_parser("fit")
    b.add_argument("measurements")
    args = ap.parse_args(argv)
    if args.cmd == "measure":
        print(json.dumps(measure(args.out)))
    else:
        coeffs = fit(json.load(open(args.measurements)))
        print(json.dumps(coeffs, indent=1))
        print(config_text(coeffs))


if __name__ == "__main__":
    sys.exit(main())
