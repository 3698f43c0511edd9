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
