"""Multi-GPU path on CPU: requests shard by sequence (request_id % world), each
rank runs its own pager + driver, and only per-step counts are all-reduced
(gloo here; NCCL over NVLink on the B200 box). Each rank's run must equal the
reference replaying that rank's sub-stream, and the all-reduced counts must
equal the sum of the per-rank records."""
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFG = {"steps": 160, "warmup_steps": 20, "seed": 5,
       # concurrency 64 = the width a trace replay uses (scenario.cpp:129)
       "workload": {"concurrency": 64, "arrivals_per_window": 4.0, "seed": 1}}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from paper_2605_09735_b200 import kvrail as kv
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = json.loads(json.dumps(CFG))
    cfg["b200"] = {"shard_rank": rank, "shard_world": world}
    d = kv.Driver(cfg)
    reduced = []
    for _ in range(cfg["steps"]):
        r = d.step()
        t = torch.tensor([r.live_sessions, r.emitted_tokens, r.commits], dtype=torch.int64)
        dist.all_reduce(t)  # per-step completion / EOS counts: the only cross-rank traffic
        reduced.append(t.tolist())
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"csv": d.steps_csv(), "reduced": reduced}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_shard_by_sequence(tmp_path, has_ref):
    world = 2
    mp.spawn(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    runs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    rows = [[ln.split(",") for ln in r["csv"].splitlines()[1:]] for r in runs]
    for step in range(CFG["steps"]):
        live = sum(int(rows[r][step][1]) for r in range(world))
        emitted = sum(int(rows[r][step][14]) for r in range(world))
        assert runs[0]["reduced"][step][:2] == [live, emitted]
        assert runs[1]["reduced"][step] == runs[0]["reduced"][step]
    if not has_ref:
        return
    from oracle import bindings as ob
    import ctypes as C
    csv = C.c_char_p()
    assert ob.ref().kvr_ref_scenario_events(json.dumps(CFG).encode(), C.byref(csv)) == 0
    events = csv.value.decode().splitlines()[1:]
    for r in range(world):
        mine = [e.split(",") for i, e in enumerate(events) if i % world == r]
        t0 = int(mine[0][0])
        path = tmp_path / f"shard{r}.csv"
        path.write_text("arrival_ms,prompt_tokens,generate_tokens\n" +
                        "".join(f"{int(a) - t0},{p},{g}\n" for a, p, g in mine))
        cfg = {k: v for k, v in CFG.items() if k != "workload"}
        cfg["trace_path"] = str(path)
        ref_csv, _, _, _ = ob.ref_scenario(cfg)
        assert runs[r]["csv"] == ref_csv, f"rank {r} diverged from the reference replay"
