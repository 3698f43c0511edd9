"""Workload inputs (workload.cpp): the generated stream, its audit, trace I/O
and window selection must equal the reference's, or runs stop being comparable."""
import json

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

SPECS = [
    {},
    {"concurrency": 128, "arrivals_per_window": 3.7, "seed": 1},
    {"prompt_min": 512, "prompt_max": 8192, "arrivals_per_window": 40.0},
    {"requests": 3000, "seed": 3},
    {"p50": 50, "p90": 200, "p99": 600, "requests": 20000, "seed": 11},
]


@pytest.mark.parametrize("i", range(len(SPECS)))
def test_stream_hash_matches_reference(i, has_ref):
    cfg = {"steps": 2, "warmup_steps": 0, "workload": SPECS[i]}
    d = kv.Driver(cfg)
    d.run()
    rep = json.loads(d.report_json())
    assert rep["workload_hash"] == d.workload_hash()
    assert rep["workload_audit"]["pass"]
    if has_ref:
        _, ref_rep, _, _ = ob.ref_scenario(cfg)
        r = json.loads(ref_rep)
        assert r["workload_hash"] == rep["workload_hash"]
        assert r["workload_audit"] == rep["workload_audit"]


def test_infeasible_specs_and_audit_failure():
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"workload": {"p50": 500, "p90": 100}})
    assert e.value.code == "InfeasibleSpec"
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"workload": {"requests": 2000, "seed": 5}})
    assert e.value.code == "WorkloadAuditFailed"


def test_trace_parse_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("arrival,prompt\n1,2\n")
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"trace_path": str(bad)})
    assert e.value.code == "ParseError"
    back = tmp_path / "back.csv"
    back.write_text("arrival_ms,prompt_tokens,generate_tokens\n10,5,5\n3,5,5\n")
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"trace_path": str(back)})
    assert e.value.code == "NonMonotoneTime"
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"trace_path": str(tmp_path / "missing.csv")})
    assert e.value.code == "IoError"
