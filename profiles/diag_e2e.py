"""Diagnose the pipelined host-buffer path: host time per call and e2e per step
with torch-pinned vs library-pinned (moe_host_alloc) buffers."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer, PinnedArray  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

E, k, d, ff, T = 8, 2, 4096, 14336, 16384
mem = 3.0 * d * ff * 2 / 1e6
m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=4 * mem)
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
xs = [wl.tokens(T, d, E, 1, i) for i in range(2)]
gates = [wl.gate_weights(E, d, 1.2, 1, 0, i) for i in range(64)]


def run(xh, yh, label, steps=12):
    tickets, call_ms = [], []
    for i in range(2):
        m.set_gate(0, gates[i])
        m.wait(m.forward_host_async(0, xh[i % 2], yh[i % 3], MOE_PLAN_SYNC, i))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        if i >= 3:
            m.wait(tickets[i - 3])
        m.set_gate(0, gates[i])
        c0 = time.perf_counter()
        tickets.append(m.forward_host_async(0, xh[i % 2], yh[i % 3], MOE_PLAN_SYNC, i))
        call_ms.append((time.perf_counter() - c0) * 1e3)
    for t in tickets[-3:]:
        m.wait(t)
    tot = (time.perf_counter() - t0) * 1e3 / steps
    print(f"{label}: e2e {tot:.3f} ms/step, host ms per call median {np.median(call_ms):.3f} max {max(call_ms):.3f}",
          flush=True)


xt = [torch.from_numpy(x.view(np.int16)).pin_memory() for x in xs]
yt = [torch.empty((T, d), dtype=torch.int16).pin_memory() for _ in range(3)]
run(xt, yt, "torch pinned")
xl = [PinnedArray((T, d), np.uint16) for _ in range(2)]
for a, x in zip(xl, xs):
    a.array[:] = x
yl = [PinnedArray((T, d), np.uint16) for _ in range(3)]
run([a.array for a in xl], [a.array for a in yl], "moe_host_alloc pinned")
# device-only reference
y = torch.empty((T, d), dtype=torch.int16, device="cuda")
xd = [torch.from_numpy(x.view(np.int16)).cuda() for x in xs]
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(12):
    m.set_gate(0, gates[i])
    m.forward(0, xd[i % 2], y, MOE_PLAN_SYNC, i)
m.sync()
print(f"device forward: {(time.perf_counter() - t0) * 1e3 / 12:.3f} ms/step")
t0 = time.perf_counter()
for i in range(4):
    m.forward_host(0, xs[i % 2], np.empty((T, d), np.uint16), MOE_PLAN_SYNC, i)
print(f"sync host forward (pageable): {(time.perf_counter() - t0) * 1e3 / 4:.3f} ms/step")
