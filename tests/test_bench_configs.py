"""The bench workloads are valid reference workloads (CPU, no GPU needed).

Every config bench.py can run (C1-C5, at 1/2/4/8 GPUs) must pass the reference's
workload audit (workload.cpp) with its per-GPU-count seed, and its control plane
must run through the reference Driver (oracle/_ref) with the pager geometry
shrunk by one power of two (the cpu_baseline recipe) without audit failures —
an admission the arena cannot hold makes the reference fail its single-commit
audit (MultiCommit), so this also pins the arena caps.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import bindings as ob  # noqa: E402
from oracle.cpu_baseline import shrink_config  # noqa: E402

pytestmark = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")


def scaled(cfg: dict) -> dict:
    return shrink_config(cfg)[0]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_workload_audit_passes(name, world):
    cfg = bench.CONFIGS[name](2, 0, world)
    ob.ref_scenario(scaled(cfg))  # raises WorkloadAuditFailed otherwise


@pytest.mark.parametrize("name,steps", [("c2", 60), ("c3", 60), ("c5", 120)])
def test_control_plane_runs_without_audit_failures(name, steps):
    csv, rep, _, _ = ob.ref_scenario(scaled(bench.CONFIGS[name](steps, 0, 1)))
    rows = csv.strip().split("\n")
    assert len(rows) == steps + 1
    live = [int(r.split(",")[1]) for r in rows[1:]]
    width = bench.CONFIGS[name](1)["workload"]["concurrency"]
    assert max(live) == width  # the batch fills


def test_cpu_baseline_scaling_keeps_tokens_per_page():
    for name in ("c2", "c3", "c5"):
        cfg = bench.CONFIGS[name](1)
        p = cfg["pager"]
        tb = 2 * p["layers"] * p["kv_head_dim"] * p["elem_bytes"]
        s = scaled(cfg)["pager"]
        tb2 = 2 * s["layers"] * s["kv_head_dim"] * s["elem_bytes"]
        assert p["page_bytes"] // tb == s["page_bytes"] // tb2
        assert s["page_bytes"] & (s["page_bytes"] - 1) == 0


def test_tail_against_the_fixed_shape():
    """bench.live_binned_tail: the tail of all steps against the median full-width step
    (the static graph's own step), beside the work-model and per-live-count readings."""
    from types import SimpleNamespace as R
    recs = [R(live_sessions=64, device_ms=0.48 + 0.001 * (i % 10), attn_ms=0.43, attn_bytes=3e9) for i in range(100)]
    recs += [R(live_sessions=20, device_ms=0.25, attn_ms=0.2, attn_bytes=1e9) for _ in range(100)]
    recs.append(R(live_sessions=64, device_ms=0.57, attn_ms=0.5, attn_bytes=3e9))
    t = bench.live_binned_tail(recs, 64)
    fw = t["full_width"]
    assert fw["width"] == 64 and fw["steps"] == 101
    assert abs(fw["p50_ms"] - 0.485) < 1e-9  # nearest rank: the 51st of 101
    assert abs(fw["max_all_steps_over_p50"] - 0.57 / 0.485) < 1e-9
    assert fw["p99_all_steps_over_p50"] <= fw["max_all_steps_over_p50"]
    assert bench.live_binned_tail(recs, 128)["full_width"] is None  # no step at that width
