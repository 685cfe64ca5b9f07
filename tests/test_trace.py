"""Trace front end against the reference's goldens and the
compiled reference (CPU only)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_2603_06350_b200 import trace as tr


def test_parse_golden(tmp_path):  # test_workload.cpp:33-47
    p = tmp_path / "t.trace"
    p.write_text("# comment line\n1200, 7, 0\n\n0 10 2\r\n500\t5\t1   # trailing comment\n")
    r = tr.parse_trace(str(p))
    assert [(x.arrival_ms, x.prompt_tokens, x.output_tokens) for x in r] == [(0, 10, 2), (500, 5, 1), (1200, 7, 0)]


def test_parse_errors_name_the_line(tmp_path):  # test_workload.cpp:49-67
    p = tmp_path / "bad.trace"
    p.write_text("0 10 2\nxyz 5 1\n")
    with pytest.raises(RuntimeError, match=":2"):
        tr.parse_trace(str(p))
    p.write_text("0 0 2\n")
    with pytest.raises(RuntimeError):
        tr.parse_trace(str(p))


def test_batching_golden():  # test_workload.cpp:95-112
    b = tr.batch_requests([tr.Request(0, 10, 2), tr.Request(500, 5, 1), tr.Request(1200, 7, 0)])
    assert [(x.iteration, x.phase, x.token_count) for x in b] == [
        (0, "prefill", 15), (1, "decode", 2), (2, "decode", 1), (3, "prefill", 7)]
    assert tr.batch_requests([]) == []


def test_batching_matches_reference(tmp_path):
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference library not built")
    ref.ref_batch_trace.argtypes = [C.c_char_p, C.c_void_p, C.c_long]
    ref.ref_batch_trace.restype = C.c_long
    reqs = tr.synthetic_trace(300, seed=4)
    p = tmp_path / "s.trace"
    tr.write_trace(str(p), reqs)
    out = np.zeros(3 * 20000, np.int64)
    n = ref.ref_batch_trace(str(p).encode(), out.ctypes.data, 20000)
    mine = tr.batch_requests(tr.parse_trace(str(p)))
    assert n == len(mine)
    got = np.array([(b.iteration, 1 if b.phase == "decode" else 0, b.token_count) for b in mine])
    assert np.array_equal(got, out[: 3 * n].reshape(n, 3))
    bundled = "/root/reference/proj/data/skewed.trace"
    if os.path.exists(bundled):
        n2 = ref.ref_batch_trace(bundled.encode(), out.ctypes.data, 20000)
        mine2 = tr.batch_requests(tr.parse_trace(bundled))
        assert n2 == len(mine2)
        assert np.array_equal(np.array([(b.iteration, int(b.phase == "decode"), b.token_count) for b in mine2]),
                              out[: 3 * n2].reshape(n2, 3))


def test_report_schema():
    r = tr.Report("moeless", 2, samples=[(0, 0, 1.5, 2, 1, 1), (1, 0, 2.0, 2, 2, 0), (0, 1, 1.0, 3, 0, 3),
                                         (1, 1, 1.25, 3, 3, 0)], iterations=2)
    import json
    j = json.loads(r.summary_json())
    assert j["tool_version"] == "0.1.0" and j["policy"] == "moeless" and j["num_layers"] == 2
    assert j["p50_forward_ms"] == 1.25 and j["p99_forward_ms"] == 2.0  # nearest rank
    assert r.samples_csv().splitlines()[:2] == ["iteration,layer,policy,forward_ms,replicas,warm,cold",
                                                "0,0,moeless,1.5,2,1,1"]
