"""Calibrate the reference's analytic cost model from B200 measurements.

The reference prices a layer as  forward = alpha * max_share + 2 * beta *
max_gpu_tokens + t_misc  (proj/src/cost_model.cpp:114-117) with alpha/beta/
t_misc as free "calibration knobs" (types.hpp:14-15).  This module measures
them on the real B200 layer so the reference's planner studies (policy
comparison, sweeps, acceptance checks) run on hardware coefficients:

  alpha   ms per routed token of one expert replica owning a B200: slope of the
          grouped-GEMM time (K4) against routed rows at the Mixtral shape
  t_misc  the layer's fixed part on the GPU: gate + plan + dispatch + combine
  beta    ms per token per exchange direction: MEASURED from the K6 peer-memory
          exchange when >= 2 GPUs are visible (two expert-parallel ranks on
          devices 0 and 1, the exchange time the extra remote rows add to
          dispatch + combine, per remote row and direction); on a one-GPU box
          the same measurement runs with both ranks on device 0 (recorded as
          "emulated", not NVLink) and beta falls back to row bytes / the NVLink
          5 peer bandwidth (770 GB/s per direction, B200_PROFILING.md), labelled

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
    res = dict(shape=dict(E=E, k=k, d=d, ff=ff), points=rows, device=torch.cuda.get_device_name(0),
               exchange=measure_exchange())
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    return res


def measure_exchange(T: int = 4096, iters: int = 10, E: int = 8, k: int = 2, d: int = 4096, ff: int = 1408):
    """K6 cost per remote row and direction (ms/token): two peer-memory ranks
    (devices 0 and 1, or both on device 0 when only one GPU is visible), expert
    e on rank e mod 2, against the same tokens on one rank with every expert
    local.  The peer-memory exchange is fused into dispatch (remote stores) and
    combine (remote loads), so its cost is the growth of dispatch + combine
    (+ the flag waits) divided by the rows each rank ships per direction."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np
    import torch

    from . import MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MoELayer
    from . import workload as wl
    ndev = torch.cuda.device_count()
    devs = [0, 1] if ndev >= 2 else [0, 0]
    G = 2
    wg = wl.gate_weights(E, d, 1.2, 1, 0, 0)
    experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
    ranks = [MoELayer(1, E, k, d, ff, max_tokens=T, world_size=G, rank=r, device=devs[r],
                      exchange_mode=MOE_EXCHANGE_P2P) for r in range(G)]
    handles = [m.p2p_export() for m in ranks]
    for m in ranks:
        m.p2p_import(handles)
    one = MoELayer(1, E, k, d, ff, max_tokens=T, device=devs[0])
    for m in ranks + [one]:
        m.set_gate(0, wg)
        for e, w in enumerate(experts):
            m.load_expert(0, e, *w)
    for m in ranks:
        m.set_placement(0, [1] * E, [e % G for e in range(E)])
    xs, ys = [], []
    for r in range(G):
        with torch.cuda.device(devs[r]):
            xs.append(torch.from_numpy(wl.tokens(T, d, E, 1, 10 + r).view(np.int16)).cuda())
            ys.append(torch.empty((T, d), dtype=torch.int16, device="cuda"))
    phase = lambda s: s.dispatch_ms + s.a2a_dispatch_ms + s.combine_ms + s.a2a_combine_ms
    ep, loc, sent = [], [], []
    with ThreadPoolExecutor(G) as ex:
        for it in range(iters):
            sts = list(ex.map(lambda r: ranks[r].forward(0, xs[r], ys[r], MOE_PLAN_FIXED, it, stats=True), range(G)))
            st1 = one.forward(0, xs[0], ys[0], MOE_PLAN_FIXED, it, stats=True)
            if it >= 2:
                ep.append(max(phase(s) for s in sts))
                loc.append(phase(st1))
                sent.append(sts[0].rows_sent)
    for m in ranks + [one]:
        m.close()
    rows = statistics.median(sent)
    extra = statistics.median(ep) - statistics.median(loc)
    beta = max(extra, 0.0) / 2.0 / max(rows, 1)  # two directions
    return dict(devices=devs, emulated=devs[0] == devs[1], tokens_per_rank=T, remote_rows_per_direction=rows,
                exchange_phase_ms=statistics.median(ep), local_phase_ms=statistics.median(loc),
                beta_ms_per_token=beta, row_bytes=d * 2,
                bus_gbs_per_direction=rows * d * 2 / (max(extra, 1e-9) / 2 * 1e-3) / 1e9)


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
    xc = meas.get("exchange")
    if xc and not xc.get("emulated") and xc.get("beta_ms_per_token", 0) > 0:
        # measured K6 time per remote row, rescaled to this shape's row bytes
        beta = xc["beta_ms_per_token"] * (d * 2) / xc["row_bytes"]
        src = (f"measured: peer-memory exchange on devices {xc['devices']}, "
               f"{xc['remote_rows_per_direction']:.0f} remote rows per direction")
    else:
        beta = d * 2 / (NVLINK_PEER_GBS * 1e9) * 1e3  # ms per token per direction
        src = (f"derived: {d * 2} B per token row / {NVLINK_PEER_GBS} GB/s NVLink 5 peer bandwidth"
               + (" (only one GPU visible: the exchange was measured with both ranks on it, "
                  f"beta_emulated = {xc['beta_ms_per_token']:.3g} ms/token)" if xc else ""))
    return dict(alpha_ms_per_token=slope, gemm_intercept_ms=icpt, r2=1 - ss_res / ss_tot,
                t_misc_ms=statistics.median(p["fixed_ms"] for p in pts), beta_ms_per_token=beta,
                beta_source=src)


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
