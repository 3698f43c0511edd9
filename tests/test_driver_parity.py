"""Per-step parity of the scenario Driver twin (scenario.cpp:124-683).

For each config the B200 driver (host-only here) must reproduce the reference
byte for byte: steps.csv, report.json and the per-step parity trace — stage
needs, every train's descriptors / reason / clock and the FNV hash of the bytes
it stages, plus a digest of the whole pager (free runs, every session's view).
Pinned twice: against fixtures generated from the reference (tests/golden,
make_golden.py) and, when oracle/_ref is built, against a live reference run.
"""
import copy
import json
import os

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read(name):
    with open(os.path.join(GOLD, name)) as f:
        return f.read()


def mine(cfg, trace=True, device=-1):
    c = copy.deepcopy(cfg)
    c.setdefault("b200", {})["trace"] = trace
    d = kv.Driver(c, device=device)
    d.run()
    return d


def c1_cfg():
    cfg = json.loads(read("c1_config.json"))
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    return cfg


@pytest.mark.parametrize("name", ["audit", "far", "adv_burst"])
def test_golden_scenarios(name):
    cfg = json.loads(read(f"{name}_config.json"))
    d = mine(cfg)
    assert d.steps_csv() == read(f"{name}_steps.csv")
    assert d.trace() == read(f"{name}_trace.txt")


def test_c1_golden():
    d = mine(c1_cfg())
    assert d.steps_csv() == read("c1_steps.csv")
    assert d.report_json() == read("c1_report.json")
    assert d.trace() == read("c1_trace.txt")


LIVE_CASES = {
    "b128": {"steps": 250, "warmup_steps": 100,
             "workload": {"concurrency": 128, "arrivals_per_window": 3.7}},
    "mild": {"steps": 250, "warmup_steps": 100, "mode": {"regime": "mild"}},
    "strong_nomerge": {"steps": 250, "warmup_steps": 100, "mode": {"regime": "strong"},
                       "transport": {"merge": False}},
    "static": {"steps": 300, "warmup_steps": 100, "mode": {"pager_enabled": False},
               "transport": {"merge": False}},
    "far_cap0": {"steps": 150, "warmup_steps": 50,
                 "far_view": {"enabled": True, "w_star": 256, "cap": 0, "sv_chunk": 128},
                 "pager": {"layers": 1, "kv_head_dim": 64, "elem_bytes": 4, "page_bytes": 16384},
                 "workload": {"requests": 2000, "concurrency": 16}},
    "tau_small_hold0": {"steps": 200, "warmup_steps": 50,
                        "transport": {"tau_bytes": 32768, "delta_hold": 0.0}},
}


@pytest.mark.parametrize("name", sorted(LIVE_CASES))
def test_live_reference(name, has_ref):
    if not has_ref:
        pytest.skip("oracle/_ref not built")
    cfg = LIVE_CASES[name]
    csv, rep, tr, _ = ob.ref_scenario(cfg, trace=True)
    d = mine(cfg)
    assert d.steps_csv() == csv
    assert d.report_json() == rep
    assert d.trace() == tr


def test_replay_trace_window(tmp_path, has_ref):
    ev = tmp_path / "trace.csv"
    d = kv.Driver({"steps": 1, "warmup_steps": 0})
    # write a generated trace through the reference CSV format, then replay a window
    lines = ["arrival_ms,prompt_tokens,generate_tokens"]
    for i in range(3000):
        lines.append(f"{i * 13},{16 + (i * 37) % 700},{1 + (i * 101) % 500}")
    ev.write_text("\n".join(lines) + "\n")
    cfg = {"trace_path": str(ev), "replay_window_seconds": 30.0, "steps": 150, "warmup_steps": 50}
    r = mine(cfg)
    assert json.loads(r.report_json())["post_warmup_steps"] == 100
    if has_ref:
        csv, rep, tr, _ = ob.ref_scenario(cfg, trace=True)
        assert r.steps_csv() == csv and r.trace() == tr
    d.close()


def test_config_errors():
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"trace_path": "x.csv", "workload": {}})
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"mode": {"regime": "nonsense"}})
    assert e.value.code == "UnknownRegime"
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver({"shaping": {"shared_prefix_tokens": 7}})
    assert e.value.code == "BadConfig"


def test_single_commit_audit_b16_to_b128():
    for b in (16, 32, 64, 128):
        cfg = {"steps": 400, "warmup_steps": 100, "seed": 40 + b,
               "workload": {"concurrency": b, "seed": 40 + b,
                            "arrivals_per_window": 1.85 * max(1.0, b / 64.0)}}
        d = mine(cfg, trace=False)
        rep = json.loads(d.report_json())
        assert rep["invariant_audit"]["multi_commit_steps"] == 0
        assert rep["invariant_audit"]["shape_violations"] == 0


def test_measured_csv_extends_reference_columns():
    """measured_steps_csv = the reference steps.csv, column for column, plus the
    B200 measurement columns (zeros on a host-only run)."""
    cfg = json.loads(read("c1_config.json"))
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    d = kv.Driver(cfg)
    d.run()
    ref = d.steps_csv().strip().split("\n")
    got = d.measured_csv().strip().split("\n")
    assert len(ref) == len(got)
    n = len(ref[0].split(","))
    assert got[0].split(",")[n:][:2] == ["device_ms", "itl_ms"]
    for a, b in zip(ref, got):
        assert b.split(",")[:n] == a.split(",")
    with pytest.raises(kv.KvrailError):
        d.measured_json()  # nothing measured on a host-only run


@pytest.mark.parametrize("seed", range(20))
def test_random_workloads_match_reference(seed, has_ref):
    """Random small workloads (geometry, window, far view, transport knobs, regimes,
    sharing, EOS bursts; tests/test_gpu_fuzz.py:random_config) — steps.csv,
    report.json and the parity trace byte-identical to the reference Driver."""
    if not has_ref:
        pytest.skip("oracle/_ref not built")
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_fuzz import random_config
    cfg = random_config(seed)
    csv, rep, tr, _ = ob.ref_scenario(cfg, trace=True)
    d = mine(dict(cfg, b200={"trace": True}))
    assert d.steps_csv() == csv
    assert d.report_json() == rep
    assert d.trace() == tr
