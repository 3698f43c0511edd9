"""TEST INFRASTRUCTURE (CPU oracle) — never imported by the product path.

ctypes bindings for the two oracles built by oracle/Makefile:
  * _build/libkvr_oracle.so  — the plain-C restatement (kvr_oracle.h);
  * _ref/libkvrail_ref.so    — the reference library compiled from its own
    sources plus a C shim (ref_shim.cpp), symbols prefixed ``kvr_ref_``.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs use this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libkvr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkvrail_ref.so")

_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        f = C.POINTER(C.c_float)
        lib.kvo_splitmix64.argtypes = [C.c_uint64]
        lib.kvo_splitmix64.restype = C.c_uint64
        lib.kvo_fill_token_payload.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                               C.c_uint32, C.c_void_p]
        lib.kvo_fill_token_lanes.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                             C.c_void_p]
        lib.kvo_fill_query.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_int, f]
        lib.kvo_fill_query_mode.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_int, C.c_int, f]
        lib.kvo_fill_token_lanes_shift.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int,
                                                   C.c_uint32, C.c_void_p]
        lib.kvo_summarize_chunk.argtypes = [f, C.c_uint32, C.c_uint64, f]
        lib.kvo_select_chunks.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_uint32,
                                          C.POINTER(C.c_uint64)]
        lib.kvo_select_chunks.restype = C.c_uint64
        lib.kvo_attend_rows.argtypes = [f, C.c_uint64, f, C.c_uint64, C.c_uint64, f, C.c_uint32, f]
        lib.kvo_attend_window.argtypes = [C.c_void_p, C.c_uint64, f, C.c_uint64, C.c_uint32,
                                          C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                                          f, f]
        lib.kvo_attention_weights.argtypes = [C.c_void_p, C.c_uint64, f, C.c_uint64, C.c_uint32,
                                              C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                                              f, C.POINTER(C.c_double)]
        lib.kvo_fnv1a.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        lib.kvo_fnv1a.restype = C.c_uint64
        lib.kvo_half_to_float.argtypes = [C.c_uint16]
        lib.kvo_half_to_float.restype = C.c_float
        lib.kvo_bf16_to_float.argtypes = [C.c_uint16]
        lib.kvo_bf16_to_float.restype = C.c_float
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        cp = C.POINTER(C.c_char_p)
        lib.kvr_ref_scenario_run.argtypes = [C.c_char_p, C.c_int, cp, cp, cp, C.POINTER(C.c_double)]
        lib.kvr_ref_scenario_events.argtypes = [C.c_char_p, cp]
        lib.kvr_ref_free.argtypes = [C.c_char_p]
        lib.kvr_ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


def ref_api():
    """The reference pager/transport API bound through the product's Api class."""
    from paper_2605_09735_b200.kvrail import Api
    return Api(ref(), "kvr_ref_")


def ref_scenario(config: dict, trace: bool = False):
    """run_scenario of the reference: (steps_csv, report_json, trace, wall_seconds)."""
    lib = ref()
    csv, rep, tr = C.c_char_p(), C.c_char_p(), C.c_char_p()
    wall = C.c_double()
    rc = lib.kvr_ref_scenario_run(json.dumps(config).encode(), int(trace), C.byref(csv),
                                  C.byref(rep), C.byref(tr), C.byref(wall))
    if rc:
        raise RuntimeError(lib.kvr_ref_last_error().decode())
    return csv.value.decode(), rep.value.decode(), tr.value.decode(), wall.value


# ---- helpers ---------------------------------------------------------------------
def fill_query(seed, session, step, layer, head, head_dim, elem_kind, mode=0):
    out = (C.c_float * head_dim)()
    oracle().kvo_fill_query_mode(seed, session, step, layer, head, head_dim, elem_kind, mode, out)
    return list(out)


def attend_window(window: bytes, n_near: int, layers: int, kv_heads: int, head_dim: int,
                  elem_kind: int, layer: int, kv_head: int, query, far_images=None, n_far=0):
    q = (C.c_float * head_dim)(*query)
    out = (C.c_float * head_dim)()
    far = (C.c_float * max(1, len(far_images or [])))(*(far_images or []))
    oracle().kvo_attend_window(window, n_near, far, n_far, layers, kv_heads, head_dim, elem_kind,
                               layer, kv_head, q, out)
    return list(out)


def attention_weights(window: bytes, n_near: int, layers: int, kv_heads: int, head_dim: int,
                      elem_kind: int, layer: int, kv_head: int, query, far_images=None, n_far=0):
    q = (C.c_float * head_dim)(*query)
    out = (C.c_double * max(1, n_far + n_near))()
    far = (C.c_float * max(1, len(far_images or [])))(*(far_images or []))
    oracle().kvo_attention_weights(window, n_near, far, n_far, layers, kv_heads, head_dim, elem_kind,
                                   layer, kv_head, q, out)
    return list(out)[:n_far + n_near]


def check_driver_utility(driver, layer=None) -> float:
    """K-mass runs of the last step == the oracle's softmax weights of the probe
    layer, averaged over q-heads and summed per block of the committed view (same
    blocks in window order). Returns the worst absolute mass error."""
    dev = driver.device()
    g = dev.geometry
    layer = g.layers - 1 if layer is None else layer
    pager = driver.pager()
    tb = g.token_bytes
    group = g.q_heads // g.kv_heads
    done, _ = driver.progress()
    step = done - 1
    runs = dev.utility(step)
    worst = 0.0
    checked = 0
    for slot, session, written in driver.live():
        if pager.session_eos(session):
            continue
        view = pager.active_view(session)
        lo = max(0, written - g.near_window)
        window, blocks = b"", []
        for t in range(lo, written):
            window += token_bytes_via_view(pager, view, t, tb)
            blocks.append(next(blk for b, e, blk, sb in view["entries"] if b <= t < e))
        far = dev.far_selection(slot)
        far_imgs = []
        for chunk in far:
            far_imgs += as_floats(dev.far_row(slot, chunk), g.elem_kind)
        rows = [0.0] * (written - lo)
        for qh in range(g.q_heads):
            q = fill_query(g.seed, session, step, layer, qh, g.head_dim, g.elem_kind, g.query_mode)
            w = attention_weights(window, written - lo, g.layers, g.kv_heads, g.head_dim, g.elem_kind,
                                  layer, qh // group, q, far_imgs, len(far))
            for i in range(written - lo):
                rows[i] += w[len(far) + i] / g.q_heads
        want = []
        for i, b in enumerate(blocks):
            if want and want[-1][0] == b:
                want[-1][1] += rows[i]
            else:
                want.append([b, rows[i]])
        got = runs[slot]
        assert [b for b, _ in got] == [b for b, _ in want], f"slot {slot}: block runs differ"
        for (_, m1), (_, m2) in zip(got, want):
            worst = max(worst, abs(m1 - m2))
        checked += 1
    assert checked > 0
    return worst


def rel_error(got, want) -> float:
    """max |got - want| / max(|want|, 1e-2 * ||want||_inf) — the 1e-3 parity metric."""
    scale = max(abs(x) for x in want) if want else 0.0
    worst = 0.0
    for g, w in zip(got, want):
        den = max(abs(w), 1e-2 * scale, 1e-30)
        worst = max(worst, abs(g - w) / den)
    return worst


def token_bytes_via_view(pager, view, token: int, tb: int) -> bytes:
    for b, e, blk, sb in view["entries"]:
        if b <= token < e:
            return pager.read_slots(blk, sb + (token - b), 1)
    raise KeyError(token)


def check_driver_window_and_attention(driver, far_images_of=None, only_slots=None,
                                      heads=None) -> float:
    """Window ring == arena for every live slot's near window; attention output
    of the last step within tolerance of the double-precision oracle. Returns the
    worst attention error (raises AssertionError on a byte mismatch)."""
    dev = driver.device()
    g = dev.geometry
    pager = driver.pager()
    tb = g.token_bytes
    group = g.q_heads // g.kv_heads
    done, _ = driver.progress()
    step = done - 1
    worst = 0.0
    for slot, session, written in driver.live():
        if only_slots is not None and slot not in only_slots:
            continue
        if pager.session_eos(session):
            continue  # finished this step: its committed view is already empty
        view = pager.active_view(session)
        lo = max(0, written - g.near_window)
        window = b""
        for t in range(lo, written):
            want = token_bytes_via_view(pager, view, t, tb)
            got = dev.ring_token(slot, t)
            assert got == want, f"window ring mismatch slot {slot} token {t}"
            window += want
        # guard rows (tensor-core configs): rows [R, R + G) of every plane mirror [0, G)
        plane, rows = dev.ring_plane(slot, g.layers - 1)
        rb = dev.row_bytes()
        guard = rows - g.ring_rows
        if guard:
            assert plane[g.ring_rows * rb:] == plane[:guard * rb], f"ring guard rows of slot {slot} differ"
        # far summaries the attention saw: device far rows == the arena summary slots
        far = dev.far_selection(slot)
        far_imgs = []
        for chunk in far:
            row = dev.far_row(slot, chunk)
            assert row == token_bytes_via_view(pager, view, (1 << 40) + chunk, tb), \
                f"far row {chunk} of slot {slot} differs from its summary slot"
            far_imgs += as_floats(row, g.elem_kind)
        q_dev = dev.query(slot)
        out = dev.attention(slot)
        for layer in range(g.layers):
            for qh in range(g.q_heads):
                if heads is not None and (layer, qh) not in heads:
                    continue
                base = (layer * g.q_heads + qh) * g.head_dim
                q = fill_query(g.seed, session, step, layer, qh, g.head_dim, g.elem_kind, g.query_mode)
                assert q == q_dev[base:base + g.head_dim], "device query differs from the oracle"
                want = attend_window(window, written - lo, g.layers, g.kv_heads, g.head_dim,
                                     g.elem_kind, layer, qh // group, q, far_imgs, len(far))
                worst = max(worst, rel_error(out[base:base + g.head_dim], want))
    return worst


def as_floats(raw: bytes, elem_kind: int) -> list[float]:
    import numpy as np
    if elem_kind == 0:
        return np.frombuffer(raw, np.float32).tolist()
    if elem_kind == 1:
        return np.frombuffer(raw, np.float16).astype(np.float32).tolist()
    u = np.frombuffer(raw, np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).tolist()
