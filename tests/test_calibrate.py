"""f3: calibrating the reference's cost model (cost_model.cpp:114-117) from
B200 measurements — alpha from K4, t_misc from the fixed phases, beta from the
K6 exchange when two GPUs are visible (derived and labelled otherwise)."""
import pytest

from paper_2603_06350_b200 import calibrate

POINTS = [dict(tokens=t, rows=2 * t, gemm_ms=0.1 + 2.5e-4 * 2 * t, fixed_ms=0.2, forward_ms=0.0,
               max_expert_rows=0) for t in (1024, 2048, 4096, 8192)]


def test_fit_alpha_and_derived_beta():
    c = calibrate.fit(dict(shape=dict(E=8, k=2, d=4096, ff=14336), points=POINTS))
    assert abs(c["alpha_ms_per_token"] - 2.5e-4) < 1e-12 and abs(c["gemm_intercept_ms"] - 0.1) < 1e-9
    assert c["t_misc_ms"] == 0.2 and c["beta_source"].startswith("derived")
    assert abs(c["beta_ms_per_token"] - 8192 / 770e9 * 1e3) < 1e-15


def test_fit_uses_measured_exchange_beta():
    xc = dict(devices=[0, 1], emulated=False, beta_ms_per_token=2e-5, row_bytes=8192, remote_rows_per_direction=4096)
    c = calibrate.fit(dict(shape=dict(E=8, k=2, d=2048, ff=14336), points=POINTS, exchange=xc))
    assert c["beta_source"].startswith("measured") and abs(c["beta_ms_per_token"] - 1e-5) < 1e-15  # rescaled rows
    xc["emulated"] = True  # both ranks on one GPU: not NVLink, keep the derived value and say so
    c = calibrate.fit(dict(shape=dict(E=8, k=2, d=4096, ff=14336), points=POINTS, exchange=xc))
    assert c["beta_source"].startswith("derived") and "beta_emulated" in c["beta_source"]


@pytest.mark.gpu
def test_measure_exchange_runs(cuda):
    xc = calibrate.measure_exchange(T=1024, iters=4, ff=256)
    assert xc["remote_rows_per_direction"] > 0 and xc["exchange_phase_ms"] > 0 and xc["local_phase_ms"] > 0
    assert xc["emulated"] == (xc["devices"][0] == xc["devices"][1])
