"""The predictor-driven layer stack (MOE_PLAN_PREDICTED) on the
GPU: planning sources per layer, the realised predictor accuracy equal to the
reference formula on oracle counts, outputs within tolerance."""
import numpy as np
import pytest

import oracle
import paper_2603_06350_b200 as pk
from paper_2603_06350_b200 import workload as wl
from paper_2603_06350_b200.stack import MoEStack
from tolerance import row_rel_err

pytestmark = pytest.mark.gpu


def test_stack_predicted_planning(cuda):
    import torch
    L, E, k, d, ff, T = 4, 8, 2, 1024, 1408, 512
    st = MoEStack(L, E, k, d, ff, T, extra_replicas=3, distance=1)
    xs_host = [[wl.tokens(T, d, E, 1, 100 * it + l) for l in range(L)] for it in range(3)]
    ys = [torch.zeros((T, d), dtype=torch.int16, device=cuda) for _ in range(L)]
    for it in range(3):
        xs = [torch.from_numpy(x.view(np.int16)).to(cuda) for x in xs_host[it]]
        stats = st.forward(xs, ys, it, stats=True)
        assert [s.plan_source for s in stats] == [3, 2, 2, 2]
        assert stats[0].predictor_accuracy == -1.0
        for l in range(1, L):
            # prediction for layer l was made at layer l-1 on layer l-1's tokens
            pred = oracle.gate(xs_host[it][l - 1], st.gates[l], k)[2]
            actual = oracle.gate(xs_host[it][l], st.gates[l], k)[2]
            assert np.array_equal(np.array(stats[l].counts[:E]), actual)
            assert stats[l].predictor_accuracy == pytest.approx(pk.measure_accuracy(pred, actual), abs=1e-12)
            assert 0.5 < stats[l].predictor_accuracy <= 1.0
            assert stats[l].replica_count >= E
        torch.cuda.synchronize()
        y = oracle.bf16_to_f32(ys[L - 1].cpu().numpy().view(np.uint16))
        idx = np.arange(0, T, 41)
        experts = [wl.expert_weights(d, ff, 1, 0, e) for e in range(E)]
        y_ref = oracle.layer_forward(xs_host[it][L - 1][idx], st.gates[L - 1], experts, [1] * E, k)[0]
        assert row_rel_err(y[idx], y_ref) <= 2e-2
    st.close()
