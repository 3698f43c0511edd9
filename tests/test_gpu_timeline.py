"""The step graph's schedule on the B200, from the in-graph kernel timeline
(KVR_TIMELINE=1, kvr_dev_timeline: first-CTA start / last exit of every kernel on
%globaltimer) and K-attn's own span in the step counters.

* Dependencies the graph must keep, whatever the PDL edges and forked branches do:
  K-apply before the hot K-write before K-fmp before K-gather; K-scan (forked at the
  root) and the queries (forked after K-apply) finish before the kernel that reads
  their output starts working; K-attn after K-gather; the tail after K-attn.
* attn_ms of every step with live sessions is K-attn's span (> 0) and is the
  timeline's attention span.
* The PDL / branch schedule does not change a byte: the golden reference trace still
  matches with the timeline on.
"""
import json
import os

import pytest

from paper_2605_09735_b200 import kvrail as kv

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def far_cfg(steps=60):
    with open(os.path.join(GOLD, "far_config.json")) as f:
        cfg = json.load(f)
    cfg["steps"] = steps
    cfg["pager"].update({"elem_bytes": 2, "kv_head_dim": 256})
    cfg.setdefault("b200", {}).update(kv_heads=2, head_dim=128, q_heads=8, payload="lanes", dtype="bf16")
    return cfg


@pytest.fixture
def timeline_env(monkeypatch):
    monkeypatch.setenv("KVR_TIMELINE", "1")


def test_step_graph_order_on_device(timeline_env):
    cfg = far_cfg()
    d = kv.Driver(cfg, device=0)
    dev = None
    seen = 0
    for _ in range(cfg["steps"]):
        r = d.step()
        d.sync()
        dev = dev or d.device()
        t = dev.timeline()
        rec = d.record(r.step)
        if rec.live_sessions == 0:
            continue
        seen += 1
        s = {k: v[0] for k, v in t.items()}
        e = {k: v[1] for k, v in t.items()}
        chain = ["apply", "write_hot", "far_map_prime", "gather", "attention", "write_cold"]
        for a, b in zip(chain, chain[1:]):
            assert e[a] <= s[b], (a, b, t)  # b works only after a completed (PDL wait first)
        assert e["scan"] <= s["gather"], t
        assert e["queries"] <= s["attention"], t
        assert e["apply"] <= s["queries"], t
        span_ms = (e["attention"] - s["attention"]) / 1e6
        assert rec.attn_ms > 0 and abs(rec.attn_ms - span_ms) <= 0.05 * span_ms + 2e-3, (rec.attn_ms, span_ms)
    assert seen >= 10


def test_golden_trace_with_timeline_on(timeline_env):
    with open(os.path.join(GOLD, "c1_config.json")) as f:
        cfg = json.load(f)
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    cfg.setdefault("b200", {}).update(trace=True, check=True, kv_heads=4, head_dim=64, payload="bytes",
                                      attention=False)
    d = kv.Driver(cfg, device=0)
    d.run()
    with open(os.path.join(GOLD, "c1_trace.txt")) as f:
        assert d.trace() == f.read()
