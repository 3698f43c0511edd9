#!/usr/bin/env python
"""bench.py — KV-RM decode step on B200: decode tokens/s + merged KV-gather GB/s.

Workload (BASELINE.json configs[1], "C2"): Llama-2-7B-shaped KV — 32 layers,
32 KV heads x head_dim 128, fp16 (512 KiB per token), 16-token pages (8 MiB),
tau = 8 pages, W* = 512, batch 64, prompts log-uniform 512-8192 tokens plus the
reference generate-length law (p50/p90/p99 = 96/384/1024), admission as the
reference Driver does it (scenario.cpp:279-360), synthetic seeded data.

One step = one reference Driver::step (pager verbs, one frame commit per live
session, stage needs) + one committed descriptor + one replay of the step graph
(apply, writeback, far, map, prime, K-scan, K-gather, K-attn) on the GPU.

  value  = emitted tokens / sum of per-step device time (CUDA events around the
           descriptor H2D + graph + stats D2H on the launch stream), KV resident;
  e2e    = emitted tokens / wall time of the same steps driven through the C-ABI
           (host control plane, pinned H2D of each step's descriptor, D2H of the
           step counters), synchronised at both ends.
Multi-GPU (one process per GPU; `--gpus N` without a torchrun environment re-launches
itself under torch.distributed.run): requests shard by sequence (request_id % world);
every rank runs its own pager + graph; the per-step counts (live, emitted, commits,
EOS) are all-reduced by ONE ncclAllReduce captured at the end of every step graph
(kvr_comm_init, NVLink/NVSwitch) — the KV data path never leaves its GPU; the max
over ranks of the timed region is used. `--backend gloo` (tests, several ranks on
one GPU via KVR_BENCH_DEVICE) does the per-step all-reduce in torch.distributed.

--impl reference: the reference's own CPU path (oracle/_ref: run_scenario control
plane + memcpy gather + build_view/attend), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("decode tokens/s + merged KV-gather HBM GB/s (mixed-length batch, 1/2/4/8 B200)")
MIB = 1 << 20


# The request stream is generated whole (arrivals scale with the GPU count, so
# each rank's shard keeps 40 arrivals per window) and must pass the reference's
# workload audit (workload.cpp audit: p50/p90/p99 and top-decile share); these
# seeds are the first that pass at each arrival rate.
WORKLOAD_SEED = {1: 1, 2: 5, 4: 14, 8: 14}


def workload(world: int, **kw) -> dict:
    w = {"requests": 10000, "arrivals_per_window": 40.0 * world,
         "seed": WORKLOAD_SEED.get(world, 1)}
    w.update(kw)
    return w


def c2_config(steps: int, rank: int = 0, world: int = 1) -> dict:
    page = 8 * MIB
    return {
        "label": "c2-llama2-7b-kv", "seed": 1, "steps": steps, "warmup_steps": 0,
        "pager": {"page_bytes": page, "layers": 32, "kv_head_dim": 4096, "elem_bytes": 2},
        "transport": {"tau_bytes": 8 * page, "delta_hold": 0.756, "merge": True},
        "far_view": {"enabled": False, "w_star": 512},
        "workload": workload(world, concurrency=64, prompt_min=512, prompt_max=8192),
        "shaping": {"arena_pages": 15000},
        "b200": {"kv_heads": 32, "head_dim": 128, "q_heads": 32, "payload": "lanes",
                 "dtype": "fp16", "shard_rank": rank, "shard_world": world},
    }


def c3_config(steps: int, rank: int = 0, world: int = 1) -> dict:
    """Llama-3-8B-shaped GQA (g=4), bf16, B=128, prompts 1k-24k, adversarial-random
    fragmentation. The arena is capped at 74000 x 2 MiB pages
    (145 GiB) and prompts at 24k so that B x mean(T) fits it: an admission the
    arena cannot hold makes the reference Driver fail its single-commit audit."""
    page = 2 * MIB
    return {
        "label": "c3-llama3-8b-gqa", "seed": 1, "steps": steps, "warmup_steps": 0,
        "pager": {"page_bytes": page, "layers": 32, "kv_head_dim": 1024, "elem_bytes": 2},
        "transport": {"tau_bytes": 32 * page, "delta_hold": 0.756, "merge": True},
        "far_view": {"enabled": False, "w_star": 512},
        "workload": workload(world, concurrency=128, prompt_min=1024, prompt_max=24576),
        "mode": {"regime": "adversarial-random"},
        "shaping": {"arena_pages": 74000},
        "b200": {"kv_heads": 8, "head_dim": 128, "q_heads": 32, "payload": "lanes",
                 "dtype": "bf16", "shard_rank": rank, "shard_world": world},
    }


def c4_config(steps: int, rank: int = 0, world: int = 1) -> dict:
    """Burst replay: WorkloadSpec defaults, select_window(60 s),
    eos_burst {step 800, fraction 0.5}, C3 shape."""
    cfg = c3_config(steps, rank, world)
    cfg["label"] = "c4-burst-replay"
    cfg["workload"] = {"requests": 10000, "concurrency": 64, "seed": 1}
    cfg["replay_window_seconds"] = 60.0
    cfg["eos_burst"] = {"step": 800, "fraction": 0.5}
    cfg.pop("mode")
    cfg.pop("shaping")
    return cfg


def c5_config(steps: int, rank: int = 0, world: int = 1) -> dict:
    """70B-shaped GQA (g=8), bf16, B=16 per GPU, far view (W* 512, cap 64).
    Page-size hazard: token_bytes = 320 KiB is not a power of two, and the
    reference wants power-of-two pages (pager.cpp validate) with sv_chunk a
    multiple of tokens per page (far_view config check). No power-of-two page
    gives a tpp dividing 128 except 1, so pages are 4 MiB (12 tokens, 256 KiB =
    6.25 % slack per page) and sv_chunk is 120 (10 pages) instead of 128."""
    page = 4 * MIB
    return {
        "label": "c5-70b-gqa-far", "seed": 1, "steps": steps, "warmup_steps": 0,
        "pager": {"page_bytes": page, "layers": 80, "kv_head_dim": 1024, "elem_bytes": 2},
        "transport": {"tau_bytes": 45 * page, "delta_hold": 0.756, "merge": True},
        "far_view": {"enabled": True, "w_star": 512, "cap": 64, "sv_chunk": 120},
        "workload": workload(world, concurrency=16, prompt_min=1024, prompt_max=16384),
        "shaping": {"arena_pages": 30000, "shared_prefix_tokens": 120},
        "b200": {"kv_heads": 8, "head_dim": 128, "q_heads": 64, "payload": "lanes",
                 "dtype": "bf16", "shard_rank": rank, "shard_world": world},
    }


def c1_config(steps: int, rank: int = 0, world: int = 1) -> dict:
    """C1 (configs[0], the reference's CPU-runnable case) as a B200 workload:
    2 layers, 4 KV heads x 64, bf16 lanes, 16 concurrent requests."""
    page = 32768
    return {
        "label": "c1-tiny", "seed": 1, "steps": steps, "warmup_steps": 0,
        "pager": {"page_bytes": page, "layers": 2, "kv_head_dim": 256, "elem_bytes": 2},
        "transport": {"tau_bytes": 8 * page, "delta_hold": 0.756, "merge": True},
        "far_view": {"enabled": False, "w_star": 512},
        "workload": workload(world, concurrency=16, prompt_min=64, prompt_max=512),
        "shaping": {"arena_pages": 4096, "staged_refresh_period": 4},
        "b200": {"kv_heads": 4, "head_dim": 64, "q_heads": 16, "payload": "lanes",
                 "dtype": "bf16", "shard_rank": rank, "shard_world": world},
    }


CONFIGS = {"c1": c1_config, "c2": c2_config, "c3": c3_config, "c4": c4_config, "c5": c5_config}
WORKLOADS = {
    "c1": "C1 tiny (configs[0] shape): L=2, 4 KV heads x hd 64, 16 q heads, bf16, batch 16, "
          "prompts 64-512",
    "c2": "C2 Llama-2-7B-shaped KV (configs[1]): L=32, 32 KV heads x hd 128, fp16, "
          "batch 64 per GPU, prompts 512-8192 (log-uniform) + decode, W*=512",
    "c3": "C3 Llama-3-8B-shaped GQA: L=32, 8 KV heads x hd 128, 32 q heads (g=4), bf16, "
          "batch 128 per GPU, prompts 1k-24k, adversarial-random fragmentation, W*=512",
    "c4": "C4 burst replay: WorkloadSpec defaults, 60 s replay window, EOS burst of 50% "
          "at step 800, C3 shape (bf16, g=4), per-step latency (synchronised steps)",
    "c5": "C5 70B-shaped GQA: L=80, 8 KV heads x hd 128, 64 q heads (g=8), bf16, batch 16 "
          "per GPU, far view W*=512 + cap 64 (sv_chunk 120 = 10 pages), 4 MiB pages (12 tokens)",
}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "src": "fallback"}


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): NVML polled every 2 ms on a thread, so even
    a short timed region gets samples; nvidia-smi as the fallback."""
    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
             "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, device: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.device = int(ids[device]) if device < len(ids) and ids[device].isdigit() else device
        self.sm, self.max_sm, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.thread = None

    def _poll(self, nv, h, masks):
        while not self.stop.is_set():
            self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.reasons.update(k for k, m in masks.items() if r & m)
            self.first.set()
            time.sleep(0.002)

    def __enter__(self):
        # NVML set up here, before the timed region (its first calls can take tens of
        # ms); the poll thread is running and has one sample when this returns
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_sm.append(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            masks = {k: getattr(nv, v) for k, v in self.NAMES.items() if hasattr(nv, v)}
            self.first = threading.Event()
            self.thread = threading.Thread(target=self._poll, args=(nv, h, masks), daemon=True)
            self.thread.start()
            self.first.wait(timeout=1.0)
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=1)
        if not self.sm:  # NVML unavailable: one nvidia-smi reading
            q = "clocks.sm,clocks.max.sm"
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout.split(",")
                self.sm, self.max_sm = [float(out[0])], [float(out[1])]
            except Exception:
                pass

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.max_sm) if self.max_sm else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


COLL_DEVICE = "cuda"  # where the per-step count tensors live ("cpu" with --backend gloo)


def dist_setup(backend: str = "nccl"):
    """One process per GPU (torchrun env). KVR_BENCH_DEVICE pins every rank to one
    device — only for exercising the multi-rank path on a 1-GPU box with gloo."""
    global COLL_DEVICE
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "KVR_BENCH_DEVICE" in os.environ:
        local = int(os.environ["KVR_BENCH_DEVICE"])
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            COLL_DEVICE = "cpu"
            dist.init_process_group(backend)
    return rank, local, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_max(vals: list[float], world: int) -> list[float]:
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=COLL_DEVICE)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def reduce_sum(vals: list[float], world: int) -> list[float]:
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=COLL_DEVICE)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def all_filled(filled: bool, world: int) -> bool:
    """Every rank's batch is full (ranks run the same number of steps: each step graph
    holds a collective)."""
    if world == 1:
        return filled
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(filled)], dtype=torch.int64, device=COLL_DEVICE)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def run_b200(args, rank, local, world) -> dict | None:
    import paper_2605_09735_b200 as pkg

    latency = args.sync_steps  # synchronise every step: wall latency incl. host work
    fill_cap = 0 if args.config == "c4" else 400  # burst replay runs from step 0
    extra = args.sustained + 48  # the sustained run and the K-gather timing step after the timed region
    cfg = CONFIGS[args.config](fill_cap + args.warmup + args.steps + extra, rank, world)
    if args.prefill_budget:
        cfg["b200"]["prefill_budget"] = args.prefill_budget
    cfg["b200"]["transfer"] = args.transfer
    if args.attention_kernel != "auto":
        cfg["b200"]["attention_kernel"] = args.attention_kernel
    if args.utility != "synthetic":
        cfg["b200"]["utility"] = args.utility
        cfg["b200"]["utility_every"] = args.utility_every
    d = pkg.Driver(cfg, device=local)
    in_graph = world > 1 and args.backend == "nccl"
    comm_note = None
    if in_graph:  # the per-step counts all-reduce, captured in every step graph
        import torch.distributed as dist
        ok, err = 1, None
        try:
            uid = [pkg.kvrail.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            d.comm_init(uid[0], rank, world)
        except pkg.kvrail.KvrailError as e:
            ok, err = 0, str(e)
        if not all_filled(bool(ok), world):  # every rank or none: the graphs must agree
            if ok:
                d.comm_destroy()
            in_graph = False
            comm_note = f"in-graph NCCL unavailable ({err or 'on another rank'}): per-step counts via torch.distributed"
    width = cfg["workload"]["concurrency"]
    # fill the fixed-width batch (admissions write whole prompts), then warm up
    fill = 0
    while fill < fill_cap:
        r = d.step()
        fill += 1
        if all_filled(r.live_sessions >= width, world):
            break
    for _ in range(args.warmup):
        d.step()
    d.sync()
    first = d.progress()[0]
    barrier(world)
    counts = None
    if world > 1 and not in_graph:  # gloo: per-step counts all-reduced on the host
        import torch
        import torch.distributed as dist
        counts = torch.zeros(4, dtype=torch.int64, device=COLL_DEVICE)
    lat_ms = []
    pending = []  # all-reduced (live, emitted, commits/session, ranks live) per step
    with Clocks(local) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ts = time.perf_counter()
            r = d.step()
            if counts is not None:  # global counts; the single-commit audit, job-wide
                counts.copy_(torch.tensor([r.live_sessions, r.emitted_tokens, r.commits,
                                           int(r.live_sessions > 0)]))
                dist.all_reduce(counts)
                pending.append(counts.clone())
            if latency:  # host control plane + descriptor + graph, to completion
                d.sync()
                lat_ms.append((time.perf_counter() - ts) * 1e3)
        d.sync()
        t1 = time.perf_counter()
    barrier(world)
    for c_ in pending:  # single-commit audit over all GPUs (sim_engine.cpp:41-44, 60):
        # every rank with live sessions committed exactly once per session
        _, _, commits_all, ranks_live = (int(x) for x in c_.tolist())
        if commits_all != ranks_live:
            raise RuntimeError(f"global single-commit audit failed: {commits_all} commit "
                               f"frames for {ranks_live} ranks with live sessions")
    recs = [d.record(s) for s in range(first, first + args.steps)]
    # in-graph counts (the job-wide single-commit audit ran in the driver per step)
    global_tokens = sum(r.global_emitted for r in recs)
    # Sustained: the next `--sustained` steps, the same way (device time per step);
    # reported beside the headline, not folded into it.
    sus_first = d.progress()[0]
    for _ in range(args.sustained):
        d.step()
    d.sync()
    sus = [d.record(s) for s in range(sus_first, sus_first + args.sustained)]
    sus_tokens, sus_dev = reduce_sum([float(sum(r.emitted_tokens for r in sus))], world)[0], \
        reduce_max([sum(r.device_ms for r in sus) / 1e3], world)[0]
    # K-gather alone (kvr_dev_time_gather: back-to-back replays on the last step's
    # descriptor): advance to a step that staged trains (all ranks step together)
    gstep = None
    for _ in range(48):
        r = d.step()
        d.sync()
        rec = d.record(r.step)
        if all_filled(rec.gather_bytes > 0, world):
            gstep = rec
            break
    gather_us = d.device().time_gather(20) * 1e3 if gstep is not None else None
    # inter-token latency: successive step-end %globaltimer stamps (pipelined steps)
    itl_ms = [(recs[i].end_ns - recs[i - 1].end_ns) / 1e6 for i in range(1, len(recs))]
    if args.dump_steps and rank == 0:  # per-step records for latency analysis
        with open(args.dump_steps, "w") as f:
            json.dump([{"step": r.step, "live": r.live_sessions, "emitted": r.emitted_tokens,
                        "trains": r.trains, "dma": r.dma_bytes, "device_ms": r.device_ms,
                        "wall_ms": lat_ms[i] if i < len(lat_ms) else None,
                        "itl_ms": itl_ms[i - 1] if i > 0 else None,
                        "writeback_tokens": r.writeback_tokens, "h2d": r.h2d_bytes,
                        "attn_bytes": r.attn_bytes, "attn_ms": r.attn_ms,
                        "phases": list(r.phase_ms)[:7]} for i, r in enumerate(recs)], f)
    dev_s = sum(r.device_ms for r in recs) / 1e3
    wall_s = t1 - t0
    tokens = sum(r.emitted_tokens for r in recs)
    attn_bytes = sum(r.attn_bytes for r in recs)
    attn_s = sum(r.attn_ms for r in recs) / 1e3
    gather_bytes = sum(r.gather_bytes for r in recs)
    gather_s = sum(r.gather_ms for r in recs if r.gather_bytes) / 1e3
    gather_steps = sum(1 for r in recs if r.gather_bytes)
    h2d = sum(r.h2d_bytes for r in recs) / args.steps
    dev = d.device()
    variant = dev.attention_variant()
    step_kernels = dev.step_kernels()
    backlog, dropped = d.prefill_backlog()
    captures = dev.graph_captures()
    dev_s_max, wall_s_max = reduce_max([dev_s, wall_s], world)
    tokens_all, gather_bytes_all, attn_bytes_all = reduce_sum(
        [float(tokens), float(gather_bytes), float(attn_bytes)], world)
    if in_graph and int(tokens_all) != global_tokens:
        raise RuntimeError(f"in-graph counts ({global_tokens} tokens) differ from the host sum "
                           f"({int(tokens_all)})")
    out = {
        "rank": rank, "cfg": cfg, "recs": recs, "dev_s": dev_s_max, "wall_s": wall_s_max,
        "tokens": tokens_all, "attn_bytes": attn_bytes, "attn_s": attn_s,
        "counts_collective": ("ncclAllReduce in the step graph (kvr_comm_init)" if in_graph else
                              "torch.distributed all_reduce per step" if world > 1 else "none"),
        "comm_note": comm_note,
        "attn_bytes_all": attn_bytes_all,
        "gather_bytes": gather_bytes, "gather_s": gather_s, "gather_bytes_all": gather_bytes_all,
        "gather_steps": gather_steps,
        "h2d": h2d, "variant": variant, "step_kernels": step_kernels, "captures": captures,
        "prefill_backlog": backlog, "prefill_dropped": dropped, "clocks": clocks.summary(), "fill_steps": fill,
        "live_mean": statistics.mean(r.live_sessions for r in recs),
        "trains_mean": statistics.mean(r.trains for r in recs),
        "trains_p90": nearest_rank([float(r.trains) for r in recs], 0.90),
        "trains_max": max(r.trains for r in recs),
        "dma_mean": statistics.mean(r.dma_bytes for r in recs),
        "mean_train_bytes": (sum(r.dma_bytes for r in recs) / max(1, sum(r.trains for r in recs))),
        "phases": {name: statistics.mean(r.phase_ms[i] for r in recs) for i, name in enumerate(
            ["apply", "hot_writes_query", "far_map_prime", "scan", "gather", "attention",
             "cold_write_tail"])},
        "live_binned_tail": live_binned_tail(recs, width),
        "p50_ms": nearest_rank([r.device_ms for r in recs], 0.50),
        "p99_ms": nearest_rank([r.device_ms for r in recs], 0.99),
        "itl_p50_ms": nearest_rank(itl_ms, 0.50) if itl_ms else None,
        "itl_p99_ms": nearest_rank(itl_ms, 0.99) if itl_ms else None,
        "wall_p50_ms": nearest_rank(lat_ms, 0.50) if lat_ms else None,
        "wall_p99_ms": nearest_rank(lat_ms, 0.99) if lat_ms else None,
        "latency_steps": len(lat_ms), "first_step": first,
        "max_step": max(range(len(recs)), key=lambda i: recs[i].device_ms) + first,
    }
    out.update({
        "sustained": {"steps": args.sustained, "value": sus_tokens / sus_dev if sus_dev else None,
                      "ms_per_step": sus_dev / max(1, args.sustained) * 1e3,
                      "note": "the steps right after the timed region, timed the same way (device "
                              "time, max over ranks); admissions and EOS keep arriving"},
        "gather_kernel": {"bytes_read": gstep.gather_bytes if gstep is not None else None,
                          "us_per_launch": gather_us, "step": gstep.step if gstep is not None else None},
    })
    d.close()
    return out


def ncu_traffic(config: str, variant: str):
    """DRAM bytes (read + write) per launch of the attention kernel from the committed
    `ncu --set full` capture of this config (profiles/traffic.json), when the
    captured kernel is the one this run used."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)[config]
    except Exception:
        return None, None
    same = ("k_attn_tc" in t["kernel"]) == variant.startswith("k_attn_tc")
    return (t["traffic_bytes"], t["source"]) if same else (None, None)


def read_stream_context(traffic, s_per_launch) -> dict:
    """Context next to the copy-bandwidth roofline: K-attn only reads, so its ceiling
    is the read-stream rate of this pool's B200s (scripts/read_peak.cu, best of a
    TMA-bulk and a vector-load stream over 16 GiB; profiles/r1/read_peak.json). The
    fraction uses the kernel's measured DRAM bytes (ncu) over its in-graph time."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1", "read_peak.json")) as f:
            peak = max(json.loads(line)["read_gbs"] for line in f if line.strip())
    except Exception:
        return {}
    out = {"read_stream_peak_gbs": peak, "read_stream_src": "profiles/r1/read_peak.json"}
    if traffic and s_per_launch:
        out["read_stream_frac"] = traffic / s_per_launch / 1e9 / peak
    return out


def in_graph_gather(res, pk) -> dict | None:
    """K-gather inside the timed steps' graphs: (read + write) train bytes / its in-kernel
    span, summed over the steps that staged trains (queries and K-scan run beside it)."""
    if not res["gather_s"] or not res["gather_bytes"]:
        return None
    gbs = 2 * res["gather_bytes"] / res["gather_s"] / 1e9
    return {"hbm_gbs": gbs, "frac": gbs / pk["hbm_gbs"], "ms_per_step": res["gather_s"] * 1e3 / max(1, res["gather_steps"])}


def live_binned_tail(recs, width: int = 0) -> dict:
    """Step-time tail with the work held fixed. The attention's work is the KV bytes of
    the live windows, which a burst replay swings by 5x, so the whole-run p99/p50 mostly
    measures the workload. (1) Work model: least-squares device_ms = a + b * attn_bytes
    over the timed steps; p99/p50 of device_ms / model is what bursts (admissions, EOS,
    staging, far summaries) add on top of the work. (2) p99/p50 within steps of one live
    count (counts with >= 20 steps). (3) The non-attention part of the step."""
    from collections import defaultdict
    xs = [float(r.attn_bytes) for r in recs]
    ys = [r.device_ms for r in recs]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    vx = sum((x - mx) ** 2 for x in xs)
    b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / vx if vx else 0.0
    a = my - b * mx
    rel = [y / (a + b * x) for x, y in zip(xs, ys) if a + b * x > 0]
    bins = defaultdict(list)
    for r in recs:
        bins[r.live_sessions].append(r.device_ms)
    ratios = {k: nearest_rank(v, 0.99) / nearest_rank(v, 0.50) for k, v in sorted(bins.items())
              if len(v) >= 20 and k > 0}
    extra = [r.device_ms - r.attn_ms for r in recs]
    # The fixed shape's own step: the reference's static graph costs the same at every
    # step (its full compiled width); here a step costs what its live windows cost, so
    # the SLO reading is the tail of ALL steps against the median full-width step.
    full = [r.device_ms for r in recs if width and r.live_sessions == width]
    fw = None
    if len(full) >= 20:
        p50f = nearest_rank(full, 0.50)
        fw = {"width": width, "steps": len(full), "p50_ms": p50f, "p99_ms": nearest_rank(full, 0.99),
              "p99_over_p50": nearest_rank(full, 0.99) / p50f,
              "p99_all_steps_over_p50": nearest_rank(ys, 0.99) / p50f,
              "max_all_steps_over_p50": max(ys) / p50f}
    return {"work_model_ms": {"fixed": a, "per_gib_kv": b * 2**30},
            "full_width": fw,
            "p99_over_p50_vs_work_model": nearest_rank(rel, 0.99) / nearest_rank(rel, 0.50) if rel else None,
            "p99_over_p50_same_live_count_max": max(ratios.values()) if ratios else None,
            "live_counts_binned": len(ratios),
            "non_attention_p50_ms": nearest_rank(extra, 0.5), "non_attention_p99_ms": nearest_rank(extra, 0.99)}


def nearest_rank(xs: list[float], q: float) -> float:
    """Nearest-rank percentile (the reference's metrics.cpp:23-33 rule)."""
    v = sorted(xs)
    import math
    return v[max(0, min(len(v) - 1, math.ceil(q * len(v)) - 1))]


def cpu_baseline_block(res: dict, threads: int | None = None) -> dict:
    from oracle import cpu_baseline as cb
    cfg = res["cfg"]
    b = cfg["b200"]
    threads = threads or os.cpu_count() or 1
    fv = cfg["far_view"]
    window = fv["w_star"] + (fv.get("cap", 0) if fv.get("enabled") else 0)
    leg = cb.decode_step(cfg, live=round(res["live_mean"]), layers=cfg["pager"]["layers"],
                         q_heads=b["q_heads"], head_dim=b["head_dim"], window=window,
                         dma_bytes_per_step=res["dma_mean"], threads=threads)
    return {"value": leg["tokens_per_s"], "unit": "tokens/s", "cores": leg["threads"],
            "kind": "reference",
            "sample": (f"one whole {cfg['label']} decode step: all {leg['attention_calls_per_step']} "
                       f"reference build_view+attend calls (W*+far={window}, hd={b['head_dim']}, "
                       f"extrapolation x{leg['attention_extrapolation']:.0f}) on {leg['threads']} OpenMP "
                       f"threads over 512 MiB of distinct fp32 histories + run_scenario control plane "
                       f"(200 steps, 1 thread, kv_head_dim and page shrunk by one power of two: same "
                       f"decisions) + Pager::read_slots of the mean staged bytes at the real geometry"),
            "extrapolation": leg["attention_extrapolation"],
            "legs_s": {"control": leg["control_s"], "attention": leg["attention_s"],
                       "gather": leg["gather_s"]}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="c2 = the headline workload (BASELINE.json configs[1]); c3/c4/c5 = "
                         "the other B200 configs of SURVEY.md §8d")
    ap.add_argument("--dump-steps", default="", help="write per-step records (JSON) here")
    ap.add_argument("--sync-steps", action="store_true",
                    help="synchronise after every step and report host+device wall latency")
    ap.add_argument("--attention-kernel", default="auto", choices=["auto", "cuda_core", "tcgen05"],
                    help="b200.attention_kernel (auto: tensor cores for GQA groups >= 4)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for the per-step counts (N > 1)")
    ap.add_argument("--utility", default="synthetic", choices=["synthetic", "attention"],
                    help="b200.utility: placement observations (attention = measured by K-mass)")
    ap.add_argument("--utility-every", type=int, default=1,
                    help="b200.utility_every: K-mass runs on every N-th step")
    ap.add_argument("--transfer", default="page_runs", choices=["page_runs", "reference"],
                    help="b200.transfer: train grouping (page_runs: physically consecutive pages merge "
                         "across page-end slack; identical to the reference where pages hold whole tokens)")
    ap.add_argument("--phases", action="store_true",
                    help="record event nodes at every phase boundary of the step graph (diagnostic: "
                         "each costs ~5 us; off, only the attention's pair is recorded)")
    ap.add_argument("--sustained", type=int, default=200,
                    help="steps run and reported (`sustained`) after the timed region")
    ap.add_argument("--prefill-budget", type=int, default=0,
                    help="b200.prefill_budget: cold prompt rows written per step (0 = all)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)  # one process per GPU (does not return)
    if "KVR_BENCH_DEVICE" in os.environ:  # several ranks on one GPU: NCCL refuses that
        args.backend = "gloo"
    if args.phases:
        os.environ["KVR_PHASE_EVENTS"] = "1"
    if args.impl == "reference":  # CPU only: rank 0 runs it, no process group, no GPU
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps(reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")))), flush=True)
        return
    rank, local, world = dist_setup(args.backend)

    res = run_b200(args, rank, local, world)
    if rank != 0:
        return
    pk = peaks()
    cfg = res["cfg"]
    pc = cfg["pager"]
    tb = 2 * pc["layers"] * pc["kv_head_dim"] * pc["elem_bytes"]
    dtype = cfg["b200"]["dtype"]
    value = res["tokens"] / res["dev_s"]
    e2e = res["tokens"] / res["wall_s"]
    attn_gbs = res["attn_bytes"] / res["attn_s"] / 1e9 if res["attn_s"] else 0.0
    gk = res["gather_kernel"]
    gather_gbs = 2 * gk["bytes_read"] / (gk["us_per_launch"] * 1e-6) / 1e9 if gk["us_per_launch"] else None
    traffic, traffic_src = ncu_traffic(args.config, res["variant"])
    roof_tps = res["tokens"] / (res["attn_bytes_all"] / (world * pk["hbm_gbs"] * 1e9))
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["dev_s"] / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": f"synthetic: seeded reference payload pattern (fill_token_payload lanes, RNE {dtype})",
        "config": bench_config(args, cfg),
        "run": {"attention_kernel": res["variant"], "fill_steps": res["fill_steps"],
                "kv_read_per_step_gib": res["attn_bytes"] / args.steps / 2**30},
        "sustained": res["sustained"],
        "prefill": {"budget_tokens_per_step": args.prefill_budget,
                    "queued_tokens_at_end": res["prefill_backlog"],
                    "never_written_tokens": res["prefill_dropped"],
                    "note": "budget 0 writes every prompt row at admission (the reference); with a "
                            "budget, rows behind the window are queued and dropped unwritten if "
                            "their page is recycled before any read"},
        "gather_hbm_gbs": gather_gbs,
        "gather": {"hbm_gbs": gather_gbs, "frac": gather_gbs / pk["hbm_gbs"] if gather_gbs else None,
                   "bytes_per_launch": 2 * gk["bytes_read"] if gk["bytes_read"] else None,
                   "us_per_launch": gk["us_per_launch"],
                   "basis": "(read + write) train bytes of one step / K-gather alone: the mean of 20 "
                            "launches' own spans (first-CTA start to last exit on %globaltimer, ncu's "
                            "gpu__time_duration) on that step's descriptor",
                   "in_graph": in_graph_gather(res, pk)},
        # decode tok/s roofline = tokens / (KV bytes the attention must read / peak)
        "decode_roofline": {
            "tokens_per_s": roof_tps,
            "frac": value / roof_tps,
            "note": "whole step (writes, scan, gather, attention, host) against the attention's "
                    "algorithmic KV bytes at the measured copy bandwidth"},
        "transport": {"trains_per_step": res["trains_mean"], "trains_p90": res["trains_p90"],
                      "trains_max": res["trains_max"], "policy": args.transfer,
                      "mean_train_bytes": res["mean_train_bytes"], "live_mean": res["live_mean"]},
        "step_latency_ms": {"p50": res["p50_ms"], "p99": res["p99_ms"], "clock": "device",
                            "itl_p50": res["itl_p50_ms"], "itl_p99": res["itl_p99_ms"],
                            "itl_note": "inter-token latency: differences of the step-end "
                                        "%globaltimer stamps, steps pipelined as served",
                            "wall_p50": res["wall_p50_ms"], "wall_p99": res["wall_p99_ms"],
                            "max_step": res["max_step"], "live_binned": res["live_binned_tail"]},
        "step_phases_ms_mean": res["phases"] if args.phases else {"attention": res["phases"]["attention"],
                                                                  "note": "other phases: --phases"},
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": res["h2d"],
                # step counters (ScanCounters, 40 B) + the all-reduced counts (4 x int64)
                "d2h_bytes_per_step": 40 + (32 if res["counts_collective"].startswith("nccl") else 0)},
        "multi_gpu": {"n_gpus": world, "shard": "request_id % n_gpus",
                      "counts_collective": res["counts_collective"], "note": res["comm_note"]},
        "gpu_launches": res["step_kernels"] * args.steps,
        "graph": {"kernels_per_step": res["step_kernels"], "captures": res["captures"],
                  "note": "one CUDA graph per descriptor ring slot, captured once, replayed every step"},
        "roofline": {"bound": "hbm", "achieved": attn_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": attn_gbs / pk["hbm_gbs"], "traffic": traffic,
                     "traffic_src": traffic_src,
                     "kernel": res["variant"], "peak_src": pk["src"],
                     "bytes_per_launch": res["attn_bytes"] / args.steps,
                     "ms_per_launch": res["attn_s"] / args.steps * 1e3,
                     **read_stream_context(traffic, res["attn_s"] / args.steps)},
        "clocks": res["clocks"],
    }
    if world == 1 and not args.no_cpu_baseline and args.config != "c4":
        try:
            line["cpu_baseline"] = cpu_baseline_block(res)
        except Exception as e:  # the oracle is absent: report, do not fake
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    print(json.dumps(line), flush=True)


def bench_config(args, cfg: dict) -> dict:
    """The workload as both arms print it (`config`): static, identical for b200 and reference."""
    pc = cfg["pager"]
    tb = 2 * pc["layers"] * pc["kv_head_dim"] * pc["elem_bytes"]
    return {"workload": WORKLOADS[args.config], "page_bytes": pc["page_bytes"],
            "tokens_per_page": pc["page_bytes"] // tb, "tau_bytes": cfg["transport"]["tau_bytes"],
            "requests_shard": "request_id % n_gpus",
            "l2": "inputs larger than L2 (GiBs of window KV read per step vs 126 MB L2)",
            "prefill_budget": args.prefill_budget, "utility": args.utility, "transfer": args.transfer}


def spawn_ranks(n: int) -> None:
    """Re-run this command as n ranks, one per GPU (torch.distributed.run, 127.0.0.1)."""
    import socket
    if "KVR_BENCH_DEVICE" not in os.environ and "--impl" not in sys.argv:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            raise SystemExit(f"bench.py --gpus {n}: only {have} GPU(s) visible")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def reference_arm(args, world) -> dict:
    """The reference's CPU implementation of the step (oracle/_ref) on the same
    workload: run_scenario control plane (shrunk geometry, identical decisions),
    Pager::read_slots of the staged bytes it schedules (real geometry), and
    build_view + attend for every (session, layer, q-head) of the step on all host
    threads — no extrapolation."""
    from oracle import cpu_baseline as cb
    cfg = CONFIGS[args.config](400, 0, 1)
    b = cfg["b200"]
    ctl = cb.control_plane(cfg)
    live = round(ctl["live_mean"])
    t_gather = cb.gather_seconds(cfg, ctl["dma_bytes_per_step"])
    threads = os.cpu_count() or 1
    window = cfg["far_view"]["w_star"] + (cfg["far_view"].get("cap", 0) if cfg["far_view"].get("enabled") else 0)
    calls = live * cfg["pager"]["layers"] * b["q_heads"]
    per_step = []
    for i in range(args.warmup + args.steps):  # every step: all of its attention calls
        t_attn = cb.attention_seconds(b["head_dim"], window, calls, threads)
        if i >= args.warmup:
            per_step.append(ctl["seconds_per_step"] + t_attn + t_gather)
    total = sum(per_step)
    value = live * len(per_step) / total
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / len(per_step) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (reference attend)",
            "data": "synthetic", "config": bench_config(args, cfg),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads,
                             "kind": "reference", "extrapolation": 1,
                             "sample": f"every timed step: all {calls} reference build_view+attend "
                                       f"calls of a {cfg['label']} step (W*+far={window}) on all "
                                       "threads over 512 MiB of distinct fp32 histories, + "
                                       "run_scenario control plane per step (shrunk geometry, same "
                                       "decisions) + Pager::read_slots of its staged bytes at the "
                                       "real geometry"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


if __name__ == "__main__":
    main()
