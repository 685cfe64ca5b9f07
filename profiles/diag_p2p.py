"""Peer-memory ranks on one GPU (threads): run the test_gpu_p2p FIXED cases
with a short exchange timeout and dump every rank's flags / epoch on failure."""
import os
import sys
import threading

import numpy as np
import torch

os.environ.setdefault("MOE_P2P_TIMEOUT_MS", "3000")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

CASES = [
    (2, 8, 2, 1024, 1408, [256, 200], [1] * 8, [0, 1, 0, 1, 0, 1, 0, 1]),
    (4, 16, 2, 1024, 1408, [128, 64, 0, 200], [1] * 16, [e % 4 for e in range(16)]),
    (4, 64, 8, 2048, 1408, [64, 64, 64, 64], [1] * 62 + [3, 2], [e % 4 for e in range(62)] + [0, 1, 2, 3, 3]),
]


def run_case(G, E, k, d, ff, tokens, rc, rg, iters):
    mem = 3.0 * d * ff * 2 / 1e6
    Tmax = max(tokens)
    ms = [MoELayer(1, E, k, d, ff, max_tokens=Tmax, world_size=G, rank=r, exchange_mode=MOE_EXCHANGE_P2P,
                   expert_mem_mb=mem, layer_mem_cap_mb=E * mem) for r in range(G)]
    hs = [m.p2p_export() for m in ms]
    for m in ms:
        m.p2p_import(hs)
        m.set_gate(0, wl.gate_weights(E, d, 1.2, 1, 0, 0))
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
        m.set_placement(0, rc, rg)
    xd = [torch.from_numpy(wl.tokens(tokens[r], d, E, 1, 70 + r).view(np.int16)).cuda() for r in range(G)]
    yd = [torch.zeros((max(t, 1), d), dtype=torch.int16, device="cuda")[:t] for t in tokens]
    torch.cuda.synchronize()
    for it in range(iters):
        errs = [None] * G

        def run(r):
            try:
                ms[r].forward(0, xd[r], yd[r], MOE_PLAN_FIXED, it, stats=True)
            except Exception as ex:  # noqa: BLE001
                errs[r] = str(ex)

        th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if any(errs):
            print("case G", G, "E", E, "it", it, "errors", errs, flush=True)
            torch.cuda.synchronize()
            for r, m in enumerate(ms):
                try:
                    fl = m.read_buffer(9, np.uint32, (4, 8))
                    ep = m.read_buffer(10, np.uint32, (1,))
                    print("  rank", r, "epoch", ep.tolist(), "flags", fl[:3, :G].tolist(), flush=True)
                except Exception as ex:  # noqa: BLE001
                    print("  rank", r, "dump failed", ex, flush=True)
            return False
    for m in ms:
        m.close()
    return True


ok = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for c in CASES:
        if not run_case(*c, iters=3):
            sys.exit(1)
        ok += 1
print("all ok", ok)
