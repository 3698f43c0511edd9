"""The committed ncu evidence is self-consistent: profiles/traffic.json (what bench.py
reports as roofline.traffic) equals the DRAM bytes of the ncu captures it cites, and the
captured K-attn launches read no less than the attention's algorithmic KV bytes and at
most a few percent more (no wasted re-reads)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summary  # noqa: E402

# algorithmic K-attn bytes of one steady step (live x L x rows x 2 d_kv x esz);
# C5: between no far rows and the full far cap of 64 rows for every session
ALGORITHMIC = {"c2": (64 * 32 * 512 * 2 * 4096 * 2,) * 2, "c3": (128 * 32 * 512 * 2 * 1024 * 2,) * 2,
               "c5": (16 * 80 * 512 * 2 * 1024 * 2, 16 * 80 * (512 + 64) * 2 * 1024 * 2)}


@pytest.mark.parametrize("config", ["c2", "c3", "c5"])
def test_traffic_matches_its_capture(config):
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
        t = json.load(f)[config]
    s = summary(os.path.join(ROOT, t["source"]))
    assert s["kernel"] == t["kernel"]
    assert abs(s["dram_read_bytes"] + s["dram_write_bytes"] - t["traffic_bytes"]) <= 1e-6 * t["traffic_bytes"]
    lo, hi = ALGORITHMIC[config]
    assert lo <= s["dram_read_bytes"] <= 1.03 * hi, (s["dram_read_bytes"], lo, hi)
