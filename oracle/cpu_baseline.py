"""TEST INFRASTRUCTURE — the reference's CPU decode path, timed (bench.py only).

Legs, all executed by the reference library compiled from its
own sources (oracle/_ref, kind "reference"):
  1. control plane: kvrail_ref::run_scenario on the same workload with
     kv_head_dim and page_bytes shrunk by one power of two (identical tokens-per-page, page
     counts and tau in pages, so every pager / stage / reduce decision is the
     same; only payload bytes shrink), single thread, wall time per step;
  2. gather: the step's train bytes read through the reference's own
     Pager::read_slots (a reference Pager at the real geometry holding that many
     written tokens) into a host staging window, single thread;
  3. attention: kvrail_ref::build_view + kvrail_ref::attend per (session, layer,
     q-head) over the W*-token window, OpenMP over all host threads, cycling over
     512 MiB of distinct fp32 histories (reads from DRAM, not a cache-hot window).
tokens/s = live / (t1 + t2 + t3).
"""
from __future__ import annotations

import copy
import ctypes as C
import os
import time

from . import bindings as ob


def _lib():
    lib = ob.ref()
    lib.kvr_ref_cpu_attention_sample.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.kvr_ref_cpu_memcpy_gbs.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_double)]
    lib.kvr_ref_cpu_gather_seconds.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                               C.c_int, C.POINTER(C.c_double)]
    return lib


def control_plane_seconds_per_step(config: dict, steps: int = 200) -> float:
    return control_plane(config, steps)["seconds_per_step"]


def shrink_config(config: dict) -> tuple[dict, int]:
    """The workload with kv_head_dim and page_bytes shrunk by one power of two:
    tokens per page, page counts and tau in pages (every pager / stage / reduce
    decision) stay identical and pages stay powers of two (also for 320 KiB
    tokens). Far view with 16-bit lanes (a B200 extension) runs the reference's
    fp32 far view with the same token bytes. Returns (config, byte scale)."""
    cfg = copy.deepcopy(config)
    cfg.pop("b200", None)
    p = cfg.setdefault("pager", {})
    tb = 2 * p["layers"] * p["kv_head_dim"] * p["elem_bytes"]
    if cfg.get("far_view", {}).get("enabled") and p["elem_bytes"] == 2:
        p.update({"elem_bytes": 4, "kv_head_dim": p["kv_head_dim"] // 2})
    scale = 1
    while p["kv_head_dim"] // scale > 16 and p["kv_head_dim"] % (2 * scale) == 0:
        scale *= 2
    p.update({"kv_head_dim": p["kv_head_dim"] // scale, "page_bytes": p["page_bytes"] // scale})
    t = cfg.setdefault("transport", {})
    t["tau_bytes"] = int(t.get("tau_bytes", 131072) // scale)
    tb_small = 2 * p["layers"] * p["kv_head_dim"] * p["elem_bytes"]
    return cfg, tb // tb_small


def control_plane(config: dict, steps: int = 200) -> dict:
    """run_scenario of the reference on the shrunk geometry: wall seconds per step,
    plus the staged (DMA) bytes per step scaled back to the real geometry and
    the mean live batch, both from the reference's own steps.csv."""
    cfg, scale = shrink_config(config)
    cfg["steps"] = steps
    cfg["warmup_steps"] = 0
    csv, _, _, wall = ob.ref_scenario(cfg, trace=False)
    rows = [r.split(",") for r in csv.strip().split("\n")]
    col = {name: i for i, name in enumerate(rows[0])}
    body = rows[1 + steps // 2:]  # second half: the batch has filled
    dma = sum(float(r[col["dma_bytes"]]) for r in body) / max(1, len(body)) * scale
    live = sum(float(r[col["live_sessions"]]) for r in body) / max(1, len(body))
    return {"seconds_per_step": wall / steps, "dma_bytes_per_step": dma, "live_mean": live}


POOL_BYTES = 512 << 20  # distinct fp32 histories cycled through (beyond any host cache)


def attention_seconds(head_dim: int, window: int, calls: int, threads: int) -> float:
    secs, chk = C.c_double(), C.c_double()
    pool = max(1, POOL_BYTES // (window * 2 * head_dim * 4))
    rc = _lib().kvr_ref_cpu_attention_sample(head_dim, window, calls, threads, pool, C.byref(secs),
                                             C.byref(chk))
    if rc:
        raise RuntimeError(ob.ref().kvr_ref_last_error().decode())
    return secs.value


def memcpy_gbs(nbytes: int = 256 << 20, reps: int = 4) -> float:
    g = C.c_double()
    rc = _lib().kvr_ref_cpu_memcpy_gbs(nbytes, reps, C.byref(g))
    if rc:
        raise RuntimeError(ob.ref().kvr_ref_last_error().decode())
    return g.value


def gather_seconds(config: dict, nbytes: float, reps: int = 2) -> float:
    """Seconds to read `nbytes` of staged tokens through the reference Pager::read_slots
    at the config's real geometry (one pass, mean of `reps`)."""
    p = config["pager"]
    s = C.c_double()
    rc = _lib().kvr_ref_cpu_gather_seconds(p["page_bytes"], p["layers"], p["kv_head_dim"], p["elem_bytes"],
                                           int(max(nbytes, 1)), reps, C.byref(s))
    if rc:
        raise RuntimeError(ob.ref().kvr_ref_last_error().decode())
    return s.value


def decode_step(config: dict, live: int, layers: int, q_heads: int, head_dim: int, window: int,
                dma_bytes_per_step: float, threads: int | None = None,
                attention_calls: int | None = None) -> dict:
    """One reference decode step's CPU time, legs and tokens/s."""
    threads = threads or os.cpu_count() or 1
    calls_per_step = live * layers * q_heads
    calls = attention_calls or calls_per_step
    t_ctl = control_plane_seconds_per_step(config)
    t_attn_sample = attention_seconds(head_dim, window, calls, threads)
    t_attn = t_attn_sample * calls_per_step / calls
    t_gather = gather_seconds(config, dma_bytes_per_step)
    total = t_ctl + t_attn + t_gather
    return {
        "tokens_per_s": live / total, "seconds_per_step": total, "control_s": t_ctl,
        "attention_s": t_attn, "gather_s": t_gather, "threads": threads,
        "gather_gbs": 2.0 * dma_bytes_per_step / t_gather / 1e9 if t_gather else None,
        "attention_extrapolation": calls_per_step / calls,
        "attention_calls_timed": calls, "attention_calls_per_step": calls_per_step,
        "attention_sample_s": t_attn_sample,
    }
