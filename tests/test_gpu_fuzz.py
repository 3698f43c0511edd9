"""Randomised device parity (B200): random small workloads — page sizes, layer and
head geometry, window width, far view, transport threshold / hold / merge,
fragmentation regime, sharing, EOS bursts — run on the GPU with the reference
payload generated in HBM (bytes mode), against the reference Driver itself
(oracle/_ref) on the same config: the per-step parity trace (train bytes hashed
from the DEVICE arena, pager digests) must be identical, and the device K-scan
must equal the host reduce on every step. With lanes payload, the window ring and
the attention are also checked against the double-precision oracle.
"""
import json
import random

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

pytestmark = pytest.mark.gpu


def random_config(seed: int) -> dict:
    rng = random.Random(seed)
    far = rng.random() < 0.35
    elem = 4 if far else rng.choice([2, 4])
    layers = rng.choice([1, 2])
    kv_dim = rng.choice([64, 128, 256])
    tb = 2 * layers * kv_dim * elem
    tpp = rng.choice([4, 8, 16])
    page = 1
    while page < tpp * tb:
        page *= 2
    tpp = page // tb
    w_star = rng.choice([32, 64, 96, 128, 200, 256, 512])
    cfg = {
        "label": f"fuzz{seed}", "seed": seed + 1, "steps": rng.choice([60, 90, 120]),
        "warmup_steps": rng.choice([0, 10]),
        "pager": {"page_bytes": page, "layers": layers, "kv_head_dim": kv_dim, "elem_bytes": elem},
        "transport": {"tau_bytes": page * rng.choice([1, 2, 4, 8, 16]),
                      "delta_hold": rng.choice([0.0, 0.1, 0.756, 2.0]),
                      "merge": rng.random() < 0.8},
        "far_view": {"enabled": far, "w_star": w_star},
        "workload": {"requests": 10000, "concurrency": rng.choice([4, 8, 16, 24]),
                     "prompt_min": 16, "prompt_max": rng.choice([256, 768, 1500]),
                     "arrivals_per_window": 40.0, "seed": 1},
        "shaping": {"staged_refresh_period": rng.choice([2, 4, 8]),
                    "span_blocks": rng.choice([3, 9]),
                    "share_probability": rng.choice([0.0, 0.3, 0.6]),
                    "shared_prefix_tokens": tpp * rng.choice([1, 2, 4])},
    }
    if far:
        chunk = tpp * rng.choice([1, 2, 4])
        cfg["far_view"].update({"cap": rng.choice([4, 8, 16]), "sv_chunk": chunk})
    if rng.random() < 0.3:
        cfg["mode"] = {"regime": rng.choice(["mild", "strong", "adversarial-random"])}
    if rng.random() < 0.3:
        cfg["eos_burst"] = {"step": cfg["steps"] // 2, "fraction": 0.5}
    return cfg


def ref_or_skip(cfg):
    try:
        return ob.ref_scenario(cfg, trace=True)
    except RuntimeError as e:  # the reference rejects this random config (audit, arena, ...)
        pytest.skip(f"reference rejects the config: {str(e)[:80]}")


@pytest.mark.parametrize("seed", range(24))
def test_random_workload_device_matches_reference(seed):
    cfg = random_config(seed)
    csv, _, trace, _ = ref_or_skip(cfg)
    c = json.loads(json.dumps(cfg))
    c["b200"] = {"payload": "bytes", "attention": False, "trace": True, "check": True}
    d = kv.Driver(c, device=0)
    d.run()
    assert d.steps_csv() == csv
    assert d.trace() == trace
    checked, bad, first = d.device_check()
    assert bad == 0, first


@pytest.mark.parametrize("seed", range(100, 106))
def test_random_workload_attention_lanes(seed):
    cfg = random_config(seed)
    ref_or_skip(cfg)  # a config the reference accepts
    p = cfg["pager"]
    hd = 64 if p["kv_head_dim"] >= 128 else 32
    kvh = p["kv_head_dim"] // hd
    c = json.loads(json.dumps(cfg))
    c["b200"] = {"payload": "lanes", "kv_heads": kvh, "head_dim": hd, "q_heads": kvh * 2,
                 "trace": True, "check": True}
    d = kv.Driver(c, device=0)
    d.run()
    checked, bad, first = d.device_check()
    assert bad == 0, first
    assert ob.check_driver_window_and_attention(d) <= 1e-3


@pytest.mark.parametrize("seed", range(200, 210))
def test_random_workload_tensor_core_attention(seed):
    """The tcgen05 kernel on random windows, GQA groups 1-8, far views (bf16 far
    rows are a B200 extension, so these runs are checked against the oracle only)."""
    rng = random.Random(seed)
    kvh = rng.choice([1, 2])
    g = rng.choice([1, 2, 4, 8])
    tpp = rng.choice([8, 16])
    layers = rng.choice([1, 2, 4])
    tb = 2 * layers * kvh * 128 * 2
    page = 1
    while page < tpp * tb:
        page *= 2
    tpp = page // tb
    far = rng.random() < 0.5
    cfg = {
        "label": f"tc{seed}", "seed": seed, "steps": rng.choice([40, 80]), "warmup_steps": 0,
        "pager": {"page_bytes": page, "layers": layers, "kv_head_dim": kvh * 128, "elem_bytes": 2},
        "transport": {"tau_bytes": 8 * page},
        "far_view": {"enabled": far, "w_star": rng.choice([64, 128, 160, 256, 512])},
        "workload": {"requests": 10000, "concurrency": rng.choice([8, 16, 32]), "prompt_min": 16,
                     "prompt_max": rng.choice([512, 1500]), "arrivals_per_window": 40.0, "seed": 1},
        "shaping": {"staged_refresh_period": 4, "shared_prefix_tokens": tpp * 4},
        "b200": {"payload": "lanes", "dtype": rng.choice(["bf16", "fp16"]), "kv_heads": kvh,
                 "head_dim": 128, "q_heads": kvh * g, "attention_kernel": "tcgen05", "check": True},
    }
    if far:
        cfg["far_view"].update({"cap": rng.choice([8, 32, 64, 96]), "sv_chunk": tpp * rng.choice([2, 4])})
    d = kv.Driver(cfg, device=0)
    d.run()
    assert "tc" in d.device().attention_variant()
    checked, bad, first = d.device_check()
    assert bad == 0, first
    assert ob.check_driver_window_and_attention(d) <= 1e-3


@pytest.mark.parametrize("seed", range(300, 312))
def test_random_workload_b200_policies(seed):
    """The round-2 B200 options on random workloads, device against its host twin under
    the same options: page-run transfer groups on pages with slack (token bytes not
    dividing the page), prefill budgets, wide payloads and fp32 queries, both attention
    kernels. Destination-hashed trace == host twin, K-scan == host reduce, every staged
    row delivered to the window, attention within 1e-3 of the double oracle."""
    rng = random.Random(seed)
    layers = rng.choice([3, 5, 6])             # 2 * layers * 256 B tokens: slack in power-of-two pages
    far = rng.random() < 0.3
    elem = 4 if far else 2
    kvh = rng.choice([1, 2])
    hd = 128
    tb = 2 * layers * kvh * hd * elem
    page = 1
    while page < 8 * tb:
        page *= 2
    tpp = page // tb
    tc = not far and rng.random() < 0.5
    g = rng.choice([4, 8]) if tc else rng.choice([1, 2])
    cfg = {
        "label": f"pol{seed}", "seed": seed, "steps": rng.choice([60, 100]), "warmup_steps": 0,
        "pager": {"page_bytes": page, "layers": layers, "kv_head_dim": kvh * hd, "elem_bytes": elem},
        "transport": {"tau_bytes": page * rng.choice([2, 8, 32])},
        "far_view": {"enabled": far, "w_star": rng.choice([128, 256, 512])},
        "workload": {"requests": 10000, "concurrency": rng.choice([8, 16]), "prompt_min": 16,
                     "prompt_max": rng.choice([512, 1500]), "arrivals_per_window": 40.0, "seed": 1},
        "shaping": {"staged_refresh_period": rng.choice([2, 4]), "shared_prefix_tokens": tpp * 2},
    }
    if far:
        cfg["far_view"].update({"cap": rng.choice([8, 16]), "sv_chunk": tpp * 2})
    b200 = {"kv_heads": kvh, "head_dim": hd, "q_heads": kvh * g, "transfer": "page_runs",
            "payload": "lanes" if far else rng.choice(["lanes", "wide"]),
            "query": "exact" if far else rng.choice(["exact", "f32"]),
            "dtype": "fp32" if far else rng.choice(["bf16", "fp16"]),
            "attention_kernel": "tcgen05" if tc else "cuda_core", "trace": True}
    host = kv.Driver(dict(cfg, b200=dict(b200)))
    host.run()
    budget = rng.choice([0, 0, 16, 256])
    d = kv.Driver(dict(cfg, b200=dict(b200, check=True, prefill_budget=budget)), device=0)
    d.run()
    assert d.trace() == host.trace()
    checked, bad, first = d.device_check()
    assert bad == 0, first
    win, behind, missing = d.staged_rows()
    assert missing == 0 and win > 0
    assert ob.check_driver_window_and_attention(d) <= 1e-3
