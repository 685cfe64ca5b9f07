"""One rank of the two-process peer-memory test (tests/test_gpu_p2p.py):
gloo moves the 192-byte slab handles, CUDA IPC maps the peer's slab."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_06350_b200 import MOE_EXCHANGE_P2P, MOE_PLAN_FIXED, MOE_PLAN_SYNC, MoELayer  # noqa: E402
from paper_2603_06350_b200 import workload as wl  # noqa: E402


def main():
    rank, G = int(sys.argv[1]), int(sys.argv[2])
    residency = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 1: MOE_RESIDENCY_PLACED (copies over IPC)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    E, k, d, ff, T = 8, 2, 1024, 1408, 128 + 32 * rank
    mem = 3.0 * d * ff * 2 / 1e6
    m = MoELayer(1, E, k, d, ff, max_tokens=256, world_size=G, rank=rank, exchange_mode=MOE_EXCHANGE_P2P,
                 expert_mem_mb=mem, layer_mem_cap_mb=(E + 3) * mem, residency=residency)
    one = MoELayer(1, E, k, d, ff, max_tokens=256, expert_mem_mb=mem, layer_mem_cap_mb=E * mem)
    handles = [None] * G
    dist.all_gather_object(handles, m.p2p_export())
    m.p2p_import(handles)
    for lay in (m, one):
        for e in range(E):
            lay.load_expert(0, e, *wl.expert_weights(d, ff, 1, 0, e))
    x = torch.from_numpy(wl.tokens(T, d, E, 1, 40 + rank).view(np.int16)).cuda()
    y = torch.zeros((T, d), dtype=torch.int16, device="cuda")
    y1 = torch.zeros_like(y)
    copies = 0
    for it in range(3):
        wg = wl.gate_weights(E, d, 1.5, 1, 0, it)
        m.set_gate(0, wg)
        one.set_gate(0, wg)
        st = m.forward(0, x, y, MOE_PLAN_SYNC, it, stats=True)
        copies += st.weight_copies
        m.sync()
        one.forward(0, x, y1, MOE_PLAN_FIXED, it)
        one.sync()
        assert torch.equal(y, y1), (rank, it)
    dist.barrier()  # nobody unmaps a slab a peer may still read
    m.close()
    one.close()
    print("P2P-IPC OK", rank, "weight copies", copies, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
