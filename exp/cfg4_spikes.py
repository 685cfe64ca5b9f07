"""cfg4 stack (32 layers, PREDICTED planning, residual stream): where do the slow layers come
from?  Per (iteration, layer) event-timed MoE-layer latency over 8 iterations."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import workload as wl
from paper_2603_06350_b200.stack import MoEStack

c = dict(wl.CONFIGS["cfg4"])
L, E, k, d, ff, T = c.get("L", 32), c["E"], c["k"], c["d"], c["ff"], c["T"]
st = MoEStack(L, E, k, d, ff, T, extra_replicas=c["extra_replicas"], zipf_s=c["s"], distance=1)
pool = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).cuda() for i in range(4)]
y = torch.empty((T, d), dtype=torch.int16, device="cuda")
hs = [torch.empty((T, d), dtype=torch.int16, device="cuda") for _ in range(2)]
stream = torch.cuda.ExternalStream(st.layer.stream_ptr)
iters = 8
lat = np.zeros((iters + 1, L))
for it in range(iters + 1):
    x = pool[it % 4]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
    with torch.cuda.stream(stream):
        for l in range(L):
            ev[l][0].record(stream)
            st.layer.forward(l, x, y, 2, it)
            ev[l][1].record(stream)
            h = hs[l % 2]
            torch.add(x.view(torch.bfloat16), y.view(torch.bfloat16), out=h.view(torch.bfloat16))
            x = h
    torch.cuda.synchronize()
    lat[it] = [a.elapsed_time(b) for a, b in ev]
lat = lat[1:]
print("median %.2f ms, p99 %.2f, max %.2f" % (np.median(lat), np.percentile(lat, 99), lat.max()))
idx = np.argwhere(lat > 1.15 * np.median(lat))
print("slow (iteration, layer, ms):", [(int(i), int(l), round(float(lat[i, l]), 2)) for i, l in idx][:40])
print("per-layer median:", np.round(np.median(lat, axis=0), 2).tolist())
st.close()
