"""The host-buffer entry points (the e2e API): synchronous and pipelined
calls produce the same bytes as the device-pointer forward."""
import numpy as np
import pytest

from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer
from paper_2603_06350_b200 import workload as wl

pytestmark = pytest.mark.gpu


def test_host_sync_and_async_match_device(cuda):
    import torch
    E, k, d, ff, T = 8, 2, 1024, 1408, 512
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=2 * mem)
    for e in range(E):
        m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    xs = [wl.tokens(T, d, E, 1, i) for i in range(5)]
    gates = [wl.gate_weights(E, d, 1.2, 1, 0, i) for i in range(5)]
    ref = []
    for i in range(5):
        m.set_gate(0, gates[i])
        yd = torch.zeros((T, d), dtype=torch.int16, device=cuda)
        m.forward(0, torch.from_numpy(xs[i].view(np.int16)).to(cuda), yd, MOE_PLAN_SYNC, i)
        torch.cuda.synchronize()
        ref.append(yd.cpu().numpy())
    # synchronous host-buffer call
    for i in range(5):
        m.set_gate(0, gates[i])
        y = np.zeros((T, d), np.int16)
        m.forward_host(0, xs[i], y, MOE_PLAN_SYNC, i)
        assert np.array_equal(y, ref[i])
    # pipelined calls, several in flight, gate weights changing in between
    xh = [torch.from_numpy(x.view(np.int16)).pin_memory() for x in xs]
    yh = [torch.zeros((T, d), dtype=torch.int16).pin_memory() for _ in range(5)]
    tickets = []
    for i in range(5):
        m.set_gate(0, gates[i])
        tickets.append(m.forward_host_async(0, xh[i], yh[i], MOE_PLAN_SYNC, i))
    for i, t in enumerate(tickets):
        m.wait(t)
    for i in range(5):
        assert np.array_equal(yh[i].numpy(), ref[i]), i
    m.close()


def test_cuda_graph_replay_matches_eager(cuda):
    """MOE_PLAN_SYNC forwards replayed as CUDA graphs (captured per layer,
    tokens and buffers) give the same bytes, counts and planner decisions."""
    import torch
    E, k, d, ff, T = 64, 8, 2048, 1408, 256
    mem = 3.0 * d * ff * 2 / 1e6
    outs = {}
    for graphs in (False, True):
        m = MoELayer(1, E, k, d, ff, max_tokens=T, expert_mem_mb=mem, layer_mem_cap_mb=16 * mem, cuda_graphs=graphs)
        for e in range(E):
            m.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
        xs = [torch.from_numpy(wl.tokens(T, d, E, 1, i).view(np.int16)).to(cuda) for i in range(2)]
        ys = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(2)]
        res = []
        for it in range(6):
            m.set_gate(0, wl.gate_weights(E, d, 2.0, 1, 0, it))
            m.forward(0, xs[it % 2], ys[it % 2], MOE_PLAN_SYNC, it)
            m.sync()
            res.append((ys[it % 2].cpu().numpy().copy(), m.read_buffer(7, np.int32, (E,)).copy()))
        outs[graphs] = res
        m.close()
    for (ya, ca), (yb, cb) in zip(outs[False], outs[True]):
        assert np.array_equal(ya, yb) and np.array_equal(ca, cb)
