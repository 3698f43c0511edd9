"""Host side of b200.utility (attention-utility observations, K-mass): config
validation and the oracle it is checked against (no GPU needed)."""
import ctypes as C
import json
import os
import random

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def far_cfg():
    with open(os.path.join(GOLD, "far_config.json")) as f:
        return json.load(f)


def test_measured_utility_needs_a_device():
    cfg = far_cfg()
    cfg["b200"] = {"utility": "attention"}
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver(cfg)
    assert e.value.code == "BadConfig" and "device" in str(e.value)


def test_synthetic_utility_is_the_reference_default():
    """utility = synthetic (the default) is the reference's observation stream:
    the host twin stays byte-identical with the reference on the far-view run."""
    cfg = far_cfg()
    cfg["steps"] = 120
    a = kv.Driver(dict(cfg, b200={"utility": "synthetic"}))
    a.run()
    b = kv.Driver(cfg)
    b.run()
    assert a.steps_csv() == b.steps_csv()
    csv, _, _, _ = ob.ref_scenario(cfg)
    assert b.steps_csv() == csv


@pytest.mark.parametrize("n_far,n_near,layers,kvh,hd,kind", [(0, 37, 2, 4, 64, 1), (5, 96, 1, 2, 32, 2),
                                                             (3, 20, 1, 1, 64, 0)])
def test_attention_weights_oracle_is_attend(n_far, n_near, layers, kvh, hd, kind):
    """kvo_attention_weights sums to one and sum_i w_i V_i is attend()'s output
    (kvo_attend_window), for every kv head of a random window."""
    rng = random.Random(n_near)
    lanes = 2 * layers * kvh * hd
    esz = 4 if kind == 0 else 2
    if kind == 0:
        window = (C.c_float * (n_near * lanes))(*[rng.uniform(-1, 1) for _ in range(n_near * lanes)])
        vals = list(window)
    else:
        import numpy as np
        raw = np.array([rng.uniform(-1, 1) for _ in range(n_near * lanes)], np.float32)
        if kind == 1:
            window = raw.astype(np.float16).tobytes()
        else:
            window = ((raw.view(np.uint32) + 0x8000) >> 16).astype(np.uint16).tobytes()
        vals = ob.as_floats(window, kind)
    window = bytes(window)
    assert len(window) == n_near * lanes * esz
    far = [rng.uniform(-1, 1) for _ in range(n_far * lanes)]
    for layer in range(layers):
        for h in range(kvh):
            q = [rng.uniform(-1, 1) for _ in range(hd)]
            w = ob.attention_weights(window, n_near, layers, kvh, hd, kind, layer, h, q, far, n_far)
            assert abs(sum(w) - 1.0) < 1e-12
            out = ob.attend_window(window, n_near, layers, kvh, hd, kind, layer, h, q, far, n_far)
            v_off = 2 * layer * kvh * hd + kvh * hd + h * hd
            rows = [far[s * lanes:(s + 1) * lanes] for s in range(n_far)] + \
                   [vals[s * lanes:(s + 1) * lanes] for s in range(n_near)]
            for i in range(hd):
                want = sum(w[s] * rows[s][v_off + i] for s in range(len(rows)))
                assert abs(out[i] - want) <= 1e-6 * max(1.0, abs(want))


def test_utility_every_must_be_positive():
    cfg = far_cfg()
    cfg["b200"] = {"utility": "attention", "utility_every": 0}
    with pytest.raises(kv.KvrailError) as e:
        kv.Driver(cfg)
    assert e.value.code == "BadConfig" and "utility_every" in str(e.value)
