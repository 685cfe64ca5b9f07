"""Trace-driven iterations through the real layer stack.

Restates the reference's request-level front end — trace file grammar
(workload.cpp:90-125: three integer columns, ',', tab or blanks, '#'
comments, stable sort by arrival, line-numbered errors) and iteration
batching (workload.cpp:157-186: one prefill batch per wall-clock second with
the summed prompt tokens, then one decode step per output position with the
number of sequences still generating) — and runs every batch through the
B200 layers with the MoEless planner, producing summary.json / samples.csv in
the reference's schema (report.cpp:48-80, %.9g rounding, nearest-rank
percentiles) from MEASURED forward times instead of the analytic model.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import percentile


@dataclass
class Request:
    arrival_ms: int
    prompt_tokens: int
    output_tokens: int


@dataclass
class IterationBatch:
    iteration: int
    phase: str  # "prefill" | "decode"
    token_count: int


def parse_trace(path: str) -> List[Request]:
    out = []
    with open(path) as f:
        for no, raw in enumerate(f, 1):
            line = raw.replace(",", " ").replace("\t", " ").replace("\r", " ").split("#", 1)[0]
            if not line.strip():
                continue
            fields = line.split()
            where = f"{path}:{no}"
            try:
                a, p, o = (int(v) for v in fields[:3])
            except (ValueError, IndexError):
                raise RuntimeError(f"{where}: expected three integer columns (arrival_ms prompt_tokens output_tokens)")
            if len(fields) > 3:
                raise RuntimeError(f"{where}: trailing field '{fields[3]}'")
            if a < 0 or p < 1 or o < 0:
                raise RuntimeError(f"{where}: arrival_ms >= 0, prompt_tokens >= 1, output_tokens >= 0 required")
            out.append(Request(a, p, o))
    out.sort(key=lambda r: r.arrival_ms)  # stable
    return out


def batch_requests(requests: List[Request]) -> List[IterationBatch]:
    reqs = sorted(requests, key=lambda r: r.arrival_ms)
    out, it, i = [], 0, 0
    while i < len(reqs):
        second = reqs[i].arrival_ms // 1000
        prompt, outputs = 0, []
        while i < len(reqs) and reqs[i].arrival_ms // 1000 == second:
            prompt += reqs[i].prompt_tokens
            outputs.append(reqs[i].output_tokens)
            i += 1
        out.append(IterationBatch(it, "prefill", prompt))
        it += 1
        for t in range(1, max(outputs) + 1):
            out.append(IterationBatch(it, "decode", sum(1 for o in outputs if o >= t)))
            it += 1
    return out


def synthetic_trace(count: int, seed: int = 1, rate_per_s: float = 20.0, prompt_log_mean: float = 4.0,
                    prompt_log_sigma: float = 0.6, output_log_mean: float = 2.6, output_log_sigma: float = 0.4):
    """Poisson arrivals and log-normal token counts with the reference's
    default parameters (workload.hpp:69-75); numpy streams, not mt19937."""
    rng = np.random.default_rng(seed)
    t, out = 0.0, []
    for _ in range(count):
        t += rng.exponential(1.0 / rate_per_s)
        p = max(1, int(round(rng.lognormal(prompt_log_mean, prompt_log_sigma))))
        o = max(1, int(round(rng.lognormal(output_log_mean, output_log_sigma))))
        out.append(Request(int(t * 1000), p, o))
    return out


def write_trace(path: str, requests: List[Request]) -> None:
    with open(path, "w") as f:
        for r in requests:
            f.write(f"{r.arrival_ms} {r.prompt_tokens} {r.output_tokens}\n")


def _r9(v: float) -> float:
    return v if not math.isfinite(v) else float(f"{v:.9g}")


@dataclass
class Report:
    policy: str
    num_layers: int
    samples: list = field(default_factory=list)  # (iteration, layer, forward_ms, replicas, warm, cold)
    accuracy: dict = field(default_factory=dict)
    bootstrap: dict = field(default_factory=dict)
    iterations: int = 0

    def summary_json(self) -> str:
        fw = [s[2] for s in self.samples]
        L = self.num_layers
        rep = [[s[3] for s in self.samples if s[1] == l] for l in range(L)]
        j = {
            "tool_version": "0.1.0", "policy": self.policy, "iterations": self.iterations, "num_layers": L,
            "total_ms": _r9(sum(fw)), "mean_forward_ms": _r9(sum(fw) / len(fw)),
            "p50_forward_ms": _r9(percentile(fw, 0.5)), "p95_forward_ms": _r9(percentile(fw, 0.95)),
            "p99_forward_ms": _r9(percentile(fw, 0.99)),
            "mean_replicas_per_layer": _r9(sum(s[3] for s in self.samples) / len(self.samples)),
            "warm_total": int(sum(s[4] for s in self.samples)), "cold_total": int(sum(s[5] for s in self.samples)),
            "layer_mean_replicas": [_r9(sum(r) / len(r)) if r else 0.0 for r in rep],
            "layer_mean_accuracy": [_r9(float(np.mean(self.accuracy.get(l, [0.0])))) for l in range(L)],
            "layer_bootstrap_uses": [int(self.bootstrap.get(l, 0)) for l in range(L)],
            "measured": "forward_ms are B200 device times (CUDA events), not the analytic model",
        }
        return json.dumps(j, indent=2) + "\n"

    def samples_csv(self) -> str:
        rows = ["iteration,layer,policy,forward_ms,replicas,warm,cold"]
        rows += [f"{i},{l},{self.policy},{f:.9g},{r},{w},{c}" for i, l, f, r, w, c in self.samples]
        return "\n".join(rows) + "\n"


def run_trace(stack, batches: List[IterationBatch], x_pool, policy: str = "moeless", max_iterations=None) -> Report:
    """Runs every batch through all layers of `stack` (paper_2603_06350_b200.stack.MoEStack),
    with per-layer stats (device-timed forward, replicas, warm/cold, predictor accuracy)."""
    import torch
    rep = Report(policy, stack.L)
    T_cap = stack.T
    for b in batches[: max_iterations or len(batches)]:
        T = min(b.token_count, T_cap)
        if T <= 0:
            continue
        xs = [x_pool[(b.iteration + l) % len(x_pool)][:T] for l in range(stack.L)]
        ys = [torch.empty((T, stack.d), dtype=torch.int16, device="cuda") for _ in range(2)]
        stats = stack.forward(xs, [ys[l % 2] for l in range(stack.L)], b.iteration, stats=True)
        for l, st in enumerate(stats):
            rep.samples.append((b.iteration, l, st.forward_ms, st.replica_count, st.warm_count, st.cold_count))
            if st.predictor_accuracy >= 0:
                rep.accuracy.setdefault(l, []).append(st.predictor_accuracy)
            if st.plan_source == 3:
                rep.bootstrap[l] = rep.bootstrap.get(l, 0) + 1
        rep.iterations += 1
    return rep
