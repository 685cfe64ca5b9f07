"""Phase stamps of the fused decode front end (MOE_FRONT_TRACE=1) at cfg5:
per phase edge, the median over layers of (min, max) over CTAs relative to
the earliest CTA start, in us."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MOE_FRONT_TRACE"] = os.environ.get("MOE_FRONT_TRACE", "1")
from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = wl.CONFIGS[cfg]
E, k, d, ff, T, s = c["E"], c["k"], c["d"], c["ff"], c["T"], c["s"]
graphs = os.environ.get("TRACE_GRAPHS", "0") == "1"
m = MoELayer(1, E, k, d, ff, max_tokens=T, cuda_graphs=graphs)
for e in range(E):
    m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
m.set_gate(0, wl.gate_weights(E, d, s, 1, 0, 0))
xs = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
y = torch.empty((T, d), dtype=torch.int16, device="cuda")
names = ["A done", "bar1 arrive", "bar1 release", "B loads", "B done", "bar2 arrive", "bar2 release", "hist", "plan+trigger", "scatter done"]
rows = []
k4 = []
stream = torch.cuda.ExternalStream(m.stream_ptr)
evs = []
for it in range(40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    m.forward(0, xs[it % 4], y, MOE_PLAN_SYNC, it)
    e1.record(stream)
    torch.cuda.synchronize()
    evs.append(e0.elapsed_time(e1) * 1e3)
    tr = m.read_buffer(12, np.uint64, (148, 16)).astype(np.int64)
    k4t = tr[:, 12:14].copy()
    n = int((tr[:, 0] > 0).sum())
    tr = tr[:n]
    t0 = tr[:, 0].min()
    rows.append([(tr[:, i].min() - t0, tr[:, i].max() - t0) if tr[:, i].min() > 0 else (np.nan, np.nan)
                 for i in range(11)])
    if k4t[:, 0].min() > 0:
        st, en = (k4t[:, 0] - t0) / 1e3, np.sort((k4t[:, 1] - t0) / 1e3)
        k4.append([st.min(), st.max(), en[0], en[len(en) // 2], en[-10], en[-1], (tr[0, 14] - t0) / 1e3,
                   (tr[0, 15] - t0) / 1e3 if tr[0, 15] > 0 else np.nan])
r = np.median(np.array(rows[5:], dtype=np.float64), axis=0) / 1e3
print(f"{cfg} ({'graph' if graphs else 'eager'}): {n} CTAs; start spread {r[0][1]:.2f} us")
for i, nm in enumerate(names):
    if np.isnan(r[i + 1][0]):
        continue
    print(f"  {nm:14s} min {r[i + 1][0]:6.2f}  max {r[i + 1][1]:6.2f} us")
if k4:
    q = np.median(np.array(k4[5:]), axis=0)
    print(f"  K4 (swap) CTA start {q[0]:.1f}..{q[1]:.1f} us; CTA end first {q[2]:.1f}, median {q[3]:.1f}, "
          f"10th-last {q[4]:.1f}, last {q[5]:.1f} us; combine end {q[6]:.1f} us; marker {q[7]:.1f} us")
print(f"  event-timed layer: median {np.median(evs[5:]):.1f} us")
