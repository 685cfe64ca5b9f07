#!/usr/bin/env python
"""Trace-driven run of the real MoE layers.

  python bench_trace.py [--trace FILE | --requests 120] [--layers 8] [--out DIR]

Batches a request trace the way the reference does (per-second prefill +
decode steps, workload.cpp:157-186), runs every iteration batch through an
L-layer stack on one B200 with MoEless planning from the fused predictor
(MOE_PLAN_PREDICTED), and writes summary.json / samples.csv in the
reference's schema with MEASURED forward times.  Default shape: the
reference's acceptance layout (16 experts, top-2, 8 layers) at Phi-3.5-MoE
dimensions (d=4096, ff=6400).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2603_06350_b200 import trace as tr
    from paper_2603_06350_b200 import workload as wl
    from paper_2603_06350_b200.stack import MoEStack
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", default="")
    ap.add_argument("--requests", type=int, default=120)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--experts", type=int, default=16)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--ff", type=int, default=6400)
    ap.add_argument("--max-tokens", type=int, default=4096)
    ap.add_argument("--max-iterations", type=int, default=400)
    ap.add_argument("--out", default="trace_out")
    a = ap.parse_args()
    reqs = tr.parse_trace(a.trace) if a.trace else tr.synthetic_trace(a.requests, seed=1)
    batches = tr.batch_requests(reqs)
    E, k = a.experts, 2
    st = MoEStack(a.layers, E, k, a.d, a.ff, a.max_tokens, extra_replicas=8, distance=1)
    pool = [torch.from_numpy(wl.tokens(a.max_tokens, a.d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
    for b in batches[:2]:  # warm-up
        tr.run_trace(st, [b], pool)
    rep = tr.run_trace(st, batches, pool, max_iterations=a.max_iterations)
    os.makedirs(a.out, exist_ok=True)
    open(os.path.join(a.out, "summary.json"), "w").write(rep.summary_json())
    open(os.path.join(a.out, "samples.csv"), "w").write(rep.samples_csv())
    s = json.loads(rep.summary_json())
    s["batches_total"] = len(batches)
    s["token_counts"] = {"prefill_median": float(np.median([b.token_count for b in batches if b.phase == "prefill"])),
                         "decode_median": float(np.median([b.token_count for b in batches if b.phase == "decode"]))}
    print(json.dumps(s))
    st.close()


if __name__ == "__main__":
    main()
