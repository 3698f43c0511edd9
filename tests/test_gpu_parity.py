"""B200 parity: the device path against the reference, end to end.

* Reference-byte payload ("bytes", scenario.cpp:193-206) generated on the GPU:
  the per-step trace — which hashes the bytes of every staged train read back
  from K-gather's DESTINATION (the window ring / far rows), and digests the whole
  pager — must equal the trace the reference recorded (tests/golden), step for
  step (staged bytes = read_slots over each train's range).
* K-gather is load-bearing: K-write and K-prime leave the ring rows of staged
  tokens to it, so a K-gather that drops a span breaks both the trace and the
  window (fault-injection test).
* b200.check: the device K-scan (stage + reduce on the GPU) must equal the host
  reduce() on every step.
* The window ring must hold exactly the arena bytes of every live slot's last
  min(written, W*) tokens; far rows must equal their summary slots (K-far is
  bit-exact with far_view.cpp:36-46); attention must be within 1e-3 of the
  double-precision oracle (kvr_oracle.c, restating far_view.cpp:113-155).
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


def run(cfg, **b200):
    c = copy.deepcopy(cfg)
    c.setdefault("b200", {}).update(dict(trace=True, check=True), **b200)
    d = kv.Driver(c, device=0)
    d.run()
    return d


def assert_scan_exact(d, steps):
    checked, bad, first = d.device_check()
    assert checked == steps and bad == 0, first


def c1():
    cfg = json.loads(read("c1_config.json"))
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    return cfg


def assert_all_staged_rows_delivered(d, behind_ok=False):
    """Every staged token the trace hashed came from K-gather's destination, except
    (far-view configs, W* shorter than a reservation span) near rows older than
    written - W*, which are not part of the window."""
    win, behind, missing = d.staged_rows()
    assert win > 0 and missing == 0 and (behind_ok or behind == 0), (win, behind, missing)


def test_c1_reference_bytes_on_device():
    d = run(c1(), kv_heads=4, head_dim=64, payload="bytes", attention=False)
    assert d.trace() == read("c1_trace.txt")
    assert_all_staged_rows_delivered(d)
    assert d.steps_csv() == read("c1_steps.csv")
    assert_scan_exact(d, 64)
    # fixed shape: the two step graphs (one per descriptor ring slot) are never recaptured
    assert d.device().graph_captures() == 2
    m = json.loads(d.measured_json())  # measured report beside the modeled one
    assert m["measured_steps"] == 64 and m["decode_tokens_per_s"] > 0
    assert m["device_step_ms"]["p50"] > 0 and m["inter_token_latency_ms"]["p50"] > 0
    rows = d.measured_csv().strip().split("\n")
    assert len(rows) == 65 and float(rows[10].split(",")[15]) > 0  # device_ms column


def test_c1_reference_bytes_without_graph():
    """The same step launched kernel by kernel (b200.graph = 0) gives the same trace."""
    d = run(c1(), kv_heads=4, head_dim=64, payload="bytes", attention=False, graph=0)
    assert d.trace() == read("c1_trace.txt")
    assert d.device().graph_captures() == 0


@pytest.mark.parametrize("name", ["audit", "adv_burst"])
def test_golden_scenarios_on_device(name):
    cfg = json.loads(read(f"{name}_config.json"))
    d = run(cfg, payload="bytes", attention=False)
    assert d.trace() == read(f"{name}_trace.txt")
    assert_scan_exact(d, cfg["steps"])
    assert_all_staged_rows_delivered(d)


DROP_ALL = (kv.Driver.FAULT_DROP_SPAN, kv.Driver.FAULT_ALL)
SHIFT_ONE = (kv.Driver.FAULT_SHIFT_ROWS, 1)


def faulty_run(cfg, fault, **b200):
    c = copy.deepcopy(cfg)
    c.setdefault("b200", {}).update(dict(trace=True, check=True), **b200)
    d = kv.Driver(c, device=0)
    d.fault(*fault)
    d.run()
    return d


@pytest.mark.parametrize("fault", [DROP_ALL, SHIFT_ONE], ids=["drop", "misplace"])
def test_faulty_gather_breaks_the_trace(fault):
    """K-gather drops its spans / lands near rows one ring row off: the
    destination-hashed trace no longer equals the reference's (the source arena
    is untouched, so a source-side hash would not notice)."""
    d = faulty_run(c1(), fault, kv_heads=4, head_dim=64, payload="bytes", attention=False)
    assert d.trace() != read("c1_trace.txt")
    assert d.steps_csv() == read("c1_steps.csv")  # the control plane is unaffected
    assert_scan_exact(d, 64)


@pytest.mark.parametrize("fault", [DROP_ALL, SHIFT_ONE], ids=["drop", "misplace"])
def test_faulty_gather_breaks_the_window(fault):
    """With the near rows of staged tokens left to K-gather, a dropped or misplaced
    span leaves wrong ring rows the attention reads: the window check must fail."""
    cfg = c1()
    cfg["steps"] = 40
    kw = dict(kv_heads=4, head_dim=64, q_heads=4, payload="lanes", dtype="fp16")
    good = run(cfg, **kw)
    assert ob.check_driver_window_and_attention(good) <= 1e-3
    bad = faulty_run(cfg, fault, **kw)
    with pytest.raises(AssertionError, match="window ring mismatch"):
        ob.check_driver_window_and_attention(bad)


@pytest.mark.parametrize("name,budget", [("c1", 8), ("adv_burst", 64), ("far", 4)])
def test_prefill_budget_keeps_reference_bytes(name, budget):
    """b200.prefill_budget defers cold prompt rows: every staged train, far
    summary and host read must still see the reference bytes (same trace)."""
    cfg = c1() if name == "c1" else json.loads(read(f"{name}_config.json"))
    extra = dict(kv_heads=4, head_dim=64) if name == "c1" else {}
    if name == "far":
        extra = dict(kv_heads=1, head_dim=64)
    else:
        extra["attention"] = False
    d = run(cfg, payload="bytes", prefill_budget=budget, **extra)
    assert d.trace() == read(f"{name}_trace.txt")
    if name == "far":
        assert ob.check_driver_window_and_attention(d) <= 1e-3


def test_far_view_fp32_on_device():
    """Far summaries computed by K-far equal the reference's (hashed in the
    trace through the far trains), and attention over [far..., near...] holds."""
    cfg = json.loads(read("far_config.json"))
    d = run(cfg, kv_heads=1, head_dim=64)
    assert d.trace() == read("far_trace.txt")
    assert_scan_exact(d, cfg["steps"])
    assert_all_staged_rows_delivered(d, behind_ok=True)
    worst = ob.check_driver_window_and_attention(d)
    assert worst <= 1e-3


@pytest.mark.parametrize("far", [False, True])
def test_page_run_transfer_policy(far):
    """b200.transfer = page_runs (a B200 policy): 1280-byte tokens leave 1 KiB of slack
    at the end of each 16 KiB page, so the reference's exact-abutment rule splits every
    page into its own train; page-run merge joins physically consecutive pages. The
    device K-scan must equal the host reduce() under the same policy on every step,
    the destination-hashed trace must equal the host twin's, and the policy must
    need fewer trains than the reference rule on the same workload."""
    cfg = c1()
    del cfg["trace_path"]
    cfg["steps"] = 160
    cfg["pager"].update({"page_bytes": 16384, "layers": 5, "kv_head_dim": 64, "elem_bytes": 2})
    cfg["transport"]["tau_bytes"] = 8 * 16384
    cfg["workload"] = {"requests": 10000, "concurrency": 16, "prompt_min": 64, "prompt_max": 1024,
                       "arrivals_per_window": 8.0, "seed": 3}
    cfg["shaping"] = {"arena_pages": 6000, "staged_refresh_period": 4, "shared_prefix_tokens": 48}
    kw = dict(kv_heads=1, head_dim=64, q_heads=2, payload="lanes", dtype="bf16")
    if far:  # fp32 lanes (the reference far view): 2560-byte tokens, 6 per page + 1 KiB slack
        cfg["pager"]["elem_bytes"] = 4
        cfg["far_view"] = {"enabled": True, "w_star": 128, "cap": 16, "sv_chunk": 24}
        kw["dtype"] = "fp32"
    host = kv.Driver(dict(cfg, b200=dict(kw, transfer="page_runs", trace=True)))
    host.run()
    ref_rule = kv.Driver(dict(cfg, b200=dict(kw)))
    ref_rule.run()
    d = run(cfg, transfer="page_runs", **kw)
    assert d.trace() == host.trace()
    assert_scan_exact(d, 160)
    assert_all_staged_rows_delivered(d, behind_ok=far)
    rows = lambda drv: [r.split(",") for r in drv.steps_csv().strip().split("\n")[1:]]
    fewer = sum(int(r[2]) for r in rows(d)) < sum(int(r[2]) for r in rows(ref_rule))
    assert fewer
    assert ob.check_driver_window_and_attention(d) <= 1e-3


@pytest.mark.parametrize("dtype,kvh,hd,qh", [("fp16", 4, 64, 4), ("bf16", 4, 64, 16),
                                             ("fp16", 2, 128, 2), ("bf16", 2, 128, 16),
                                             ("fp16", 8, 32, 8), ("bf16", 4, 64, 8)])
def test_window_and_attention_lanes_payload(dtype, kvh, hd, qh):
    cfg = c1()
    cfg["steps"] = 40
    cfg["pager"]["kv_head_dim"] = kvh * hd
    cfg["pager"]["page_bytes"] = 16 * 2 * 2 * kvh * hd * 2
    cfg["transport"]["tau_bytes"] = 8 * cfg["pager"]["page_bytes"]
    cfg["far_view"]["w_star"] = 96
    host = kv.Driver(dict(cfg, b200=dict(kv_heads=kvh, head_dim=hd, q_heads=qh, payload="lanes",
                                          dtype=dtype, trace=True)))
    host.run()
    d = run(cfg, kv_heads=kvh, head_dim=hd, q_heads=qh, payload="lanes", dtype=dtype)
    assert d.trace() == host.trace()
    assert_scan_exact(d, 40)
    assert ob.check_driver_window_and_attention(d) <= 1e-3


@pytest.mark.parametrize("dtype,kvh,qh,w_star", [("bf16", 2, 8, 96), ("bf16", 2, 8, 512),
                                                 ("fp16", 2, 8, 512), ("bf16", 2, 16, 512),
                                                 ("bf16", 2, 4, 300), ("fp16", 1, 8, 200),
                                                 ("fp16", 2, 2, 512), ("bf16", 4, 4, 160)])
def test_tcgen05_gqa_attention(dtype, kvh, qh, w_star):
    """The tensor-core GQA kernel (tcgen05 S = K.Q^T and O = V^T.P, TMEM
    accumulators) against the double-precision oracle, window tiles of every
    alignment (W* 96..512, ragged window edges)."""
    hd = 128
    cfg = c1()
    cfg["steps"] = 40
    cfg["pager"]["kv_head_dim"] = kvh * hd
    cfg["pager"]["page_bytes"] = 16 * 2 * 2 * kvh * hd * 2
    cfg["transport"]["tau_bytes"] = 8 * cfg["pager"]["page_bytes"]
    cfg["far_view"]["w_star"] = w_star
    d = run(cfg, kv_heads=kvh, head_dim=hd, q_heads=qh, payload="lanes", dtype=dtype,
            attention_kernel="tcgen05")
    assert "tc" in d.device().attention_variant()
    assert_scan_exact(d, 40)
    assert ob.check_driver_window_and_attention(d) <= 1e-3


def not_16bit_exact(qs, elem_kind):
    """Fraction of query lanes that a 16-bit type cannot hold (the tensor-core
    kernel's lo half is non-zero for those)."""
    import numpy as np
    q = np.asarray(qs, np.float32)
    if elem_kind == 1:
        back = q.astype(np.float16).astype(np.float32)
    else:
        back = (((q.view(np.uint32) + 0x7FFF + ((q.view(np.uint32) >> 16) & 1)) >> 16) << 16).view(np.float32)
    return float(np.mean(back != q))


@pytest.mark.parametrize("kernel,dtype,kvh,hd,qh", [
    ("cuda_core", "fp16", 4, 64, 4), ("cuda_core", "bf16", 2, 128, 2), ("cuda_core", "bf16", 2, 128, 8),
    ("tcgen05", "bf16", 2, 128, 8), ("tcgen05", "fp16", 2, 128, 8), ("tcgen05", "bf16", 1, 128, 8),
    ("tcgen05", "bf16", 2, 128, 4), ("tcgen05", "fp16", 2, 128, 16)])
def test_attention_f32_queries_wide_kv(kernel, dtype, kvh, hd, qh):
    """Random 24-bit fp32 queries (not representable in the KV type: q = q_hi + q_lo
    with q_lo != 0 in the tensor-core kernel) over KV lanes of [-16, 16) — logits of
    std ~5, peaked softmaxes — against the double-precision oracle at 1e-3."""
    cfg = c1()
    cfg["steps"] = 40
    cfg["pager"]["kv_head_dim"] = kvh * hd
    cfg["pager"]["page_bytes"] = 16 * 2 * 2 * kvh * hd * 2
    cfg["transport"]["tau_bytes"] = 8 * cfg["pager"]["page_bytes"]
    cfg["far_view"]["w_star"] = 512
    d = run(cfg, kv_heads=kvh, head_dim=hd, q_heads=qh, payload="wide", query="f32", dtype=dtype,
            attention_kernel=kernel)
    assert ("tc" in d.device().attention_variant()) == (kernel == "tcgen05")
    assert_scan_exact(d, 40)
    g = d.device().geometry
    assert g.query_mode == 1 and g.lane_shift == 3
    slot, session, _ = d.live()[0]
    q = ob.fill_query(g.seed, session, 39, 0, 0, hd, g.elem_kind, 1)
    assert q == d.device().query(slot)[:hd]
    assert not_16bit_exact(q, g.elem_kind) > 0.9
    assert ob.check_driver_window_and_attention(d) <= 1e-3


def test_attention_f32_queries_wide_kv_far_view():
    """The same inputs with far summary rows in the view (tensor-core kernel, gather4 rows)."""
    cfg = json.loads(read("far_config.json"))
    cfg["steps"] = 250
    cfg["pager"].update({"elem_bytes": 2, "kv_head_dim": 256})
    d = run(cfg, kv_heads=2, head_dim=128, q_heads=8, payload="wide", query="f32", dtype="bf16",
            attention_kernel="tcgen05")
    assert_scan_exact(d, 250)
    assert ob.check_driver_window_and_attention(d) <= 1e-3


@pytest.mark.parametrize("far", [False, True])
def test_tcgen05_many_items_per_cta(far):
    """~14 (slot, layer, kv-head) items per CTA: both softmax warpgroups run
    alternating item streams, one runs out first (the single-warpgroup tail),
    and the V ring (behind the K ring) sees a warpgroup reach the PV of a later
    occupant of a stage before the other warpgroup's PV of the current one."""
    cfg = c1()
    del cfg["trace_path"]
    cfg["steps"] = 48
    cfg["pager"].update({"layers": 16, "kv_head_dim": 256, "page_bytes": 16 * 2 * 16 * 256 * 2})
    cfg["transport"]["tau_bytes"] = 8 * cfg["pager"]["page_bytes"]
    cfg["workload"] = {"requests": 10000, "concurrency": 64, "prompt_min": 64, "prompt_max": 1024,
                       "arrivals_per_window": 40.0, "seed": 1}
    cfg["shaping"] = {"arena_pages": 12000, "staged_refresh_period": 4}
    if far:
        cfg["far_view"] = {"enabled": True, "w_star": 256, "cap": 16, "sv_chunk": 64}
    d = run(cfg, kv_heads=2, head_dim=128, q_heads=8, payload="lanes", dtype="bf16",
            attention_kernel="tcgen05")
    assert "tc" in d.device().attention_variant()
    assert_scan_exact(d, 48)
    slots = [s for s, _, _ in d.live()][:6]
    assert ob.check_driver_window_and_attention(d, only_slots=slots) <= 1e-3


def test_tcgen05_far_view_bf16():
    """Far summary rows (cp.async into the swizzled tile) through the tensor-core kernel."""
    cfg = json.loads(read("far_config.json"))
    cfg["steps"] = 250
    cfg["pager"].update({"elem_bytes": 2, "kv_head_dim": 256})
    d = run(cfg, kv_heads=2, head_dim=128, q_heads=8, payload="lanes", dtype="bf16",
            attention_kernel="tcgen05")
    assert "tc" in d.device().attention_variant()
    assert_scan_exact(d, 250)
    assert ob.check_driver_window_and_attention(d) <= 1e-3


def test_far_view_bf16_extension():
    """bf16 far view (a B200 extension: fp32 mean, RNE to bf16) runs at full width."""
    cfg = json.loads(read("far_config.json"))
    cfg["steps"] = 250
    cfg["pager"].update({"elem_bytes": 2, "page_bytes": 8192})
    d = run(cfg, kv_heads=2, head_dim=32, q_heads=4, payload="lanes", dtype="bf16")
    assert_scan_exact(d, 250)
    assert ob.check_driver_window_and_attention(d) <= 1e-3


def test_pager_on_device_random_streams():
    """The Pager API with its payload in HBM: host payload writes, COW copies,
    recycled-page zeroing and trims must read back exactly like the host pager."""
    import random

    def small(pages):
        return kv.PagerConfig(512, pages, 1, 8, 2)

    def payload(n, tag):
        return bytes(((tag * 131 + i * 7) & 0xFF) for i in range(n * 32))

    g = kv.Geometry()
    g.device, g.elem_kind, g.elem_bytes, g.payload_mode = 0, 1, 2, 1
    g.page_bytes, g.token_bytes, g.arena_pages, g.tokens_per_page = 512, 32, 48, 16
    g.layers, g.kv_heads, g.head_dim, g.q_heads = 1, 1, 8, 1
    g.n_slots, g.near_window, g.ring_rows, g.far_cap = 3, 32, 64, 0
    g.chunk_tokens, g.max_chunks, g.max_tokens, g.seed = 16, 1, 4096, 1
    g.attention, g.use_graph = 0, 1
    dev = kv.Device(g)
    for seed in range(20):
        rng = random.Random(seed)
        a = kv.Pager(small(48), device=dev)
        b = kv.Pager(small(48))
        for s in range(3):
            a.create_session(s)
            b.create_session(s)
        nxt = [0, 0, 0]
        for _ in range(60):
            s = rng.randrange(3)
            k = rng.randrange(8)
            if k < 2:
                call = ("reserve", (s, rng.randrange(40)))
            elif k < 3:
                call = ("alias", (s, rng.randrange(3), rng.randrange(1, 40)))
            elif k < 6:
                lo = rng.randrange(a.session_cursor(s) + 1)
                n = rng.randint(1, 20)
                call = ("write_tokens", (s, lo, lo + n, payload(n, rng.randrange(256))))
            elif k < 7:
                call = ("trim_eos", (s,))
            else:
                call = ("frame_commit", (s, nxt[s]))
            outs = []
            for p in (a, b):
                try:
                    outs.append(getattr(p, call[0])(*call[1]))
                except kv.KvrailError as e:
                    outs.append(e.code)
            assert outs[0] == outs[1]
            if call[0] == "frame_commit" and not isinstance(outs[0], str):
                nxt[s] += 1
                for t in range(3):
                    assert a.reconstruct_view(t) == b.reconstruct_view(t), (seed, t)
        a.close()
    dev.close()
