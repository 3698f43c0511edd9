"""B200: attention-utility observations (b200.utility = "attention", K-mass).

The reference feeds the placement tracker a synthetic observation per session
(scenario.cpp:526-529; SPEC.md:190 calls the attention-utility observation a
stand-in). K-mass measures it: the probe layer's softmax weight on every block
of each slot's window, mean over q-heads. Checked against the double-precision
oracle (kvo_attention_weights, restating attend(), far_view.cpp:113-155) and
the committed view's blocks; then the driver runs its placement loop on them.
"""
import copy
import json
import os

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read(name):
    with open(os.path.join(GOLD, name)) as f:
        return f.read()


def lanes_c1(kvh, hd, steps=40, w_star=96):
    cfg = json.loads(read("c1_config.json"))
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    cfg["steps"] = steps
    cfg["pager"]["kv_head_dim"] = kvh * hd
    cfg["pager"]["page_bytes"] = 16 * 2 * 2 * kvh * hd * 2
    cfg["transport"]["tau_bytes"] = 8 * cfg["pager"]["page_bytes"]
    cfg["far_view"]["w_star"] = w_star
    return cfg


@pytest.mark.parametrize("dtype,kvh,hd,qh,layer", [("fp16", 4, 64, 4, None), ("bf16", 2, 128, 8, 0),
                                                   ("bf16", 2, 128, 16, None)])
def test_utility_mass_matches_oracle(dtype, kvh, hd, qh, layer):
    cfg = lanes_c1(kvh, hd)
    b = dict(kv_heads=kvh, head_dim=hd, q_heads=qh, payload="lanes", dtype=dtype, utility="attention")
    if layer is not None:
        b["utility_layer"] = layer
    cfg["b200"] = b
    d = kv.Driver(cfg, device=0)
    d.run()
    assert ob.check_driver_utility(d, layer) <= 1e-4


def test_utility_mass_with_far_summaries():
    """Far rows take part in the normalisation (build_view order, far first)."""
    cfg = json.loads(read("far_config.json"))
    cfg["b200"] = dict(kv_heads=1, head_dim=64, utility="attention")
    d = kv.Driver(cfg, device=0)
    d.run()
    assert any(d.device().far_selection(s) for s, _, _ in d.live())
    assert ob.check_driver_utility(d) <= 1e-4


def test_utility_every_n_steps():
    """utility_every = 3: K-mass runs on steps divisible by 3 only; the other steps
    report no observations, and the measured ones still match the oracle."""
    cfg = json.loads(read("far_config.json"))
    cfg["steps"] = 121  # the last step (120) is a measured one
    cfg["b200"] = dict(kv_heads=1, head_dim=64, utility="attention", utility_every=3, check=True)
    d = kv.Driver(cfg, device=0)
    d.run()
    checked, bad, first = d.device_check()
    assert checked == cfg["steps"] and bad == 0, first
    assert ob.check_driver_utility(d) <= 1e-4
    assert all(not r for r in d.device().utility(119))


def test_measured_utility_drives_placement():
    """With measured observations the placement loop still keeps every audit (one
    commit per live session, device K-scan == host reduce()), and its far-view
    selections follow the measured utility instead of the synthetic one."""
    base = json.loads(read("far_config.json"))
    runs = {}
    for mode in ("synthetic", "attention"):
        cfg = copy.deepcopy(base)
        cfg["b200"] = dict(kv_heads=1, head_dim=64, utility=mode, check=True, trace=True)
        d = kv.Driver(cfg, device=0)
        d.run()
        checked, bad, first = d.device_check()
        assert checked == cfg["steps"] and bad == 0, first
        sel = {s: d.device().far_selection(s) for s, _, _ in d.live()}
        runs[mode] = (d.trace(), sel)
    # the pager digests (cold trims) or the far chunks shown to the attention differ
    assert runs["synthetic"] != runs["attention"]
