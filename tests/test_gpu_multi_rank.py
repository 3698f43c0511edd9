"""Multi-GPU path on the B200: requests shard by sequence and the only
cross-rank traffic is the per-step counts all-reduce.

* Two ranks on ONE GPU (gloo for the counts; NCCL refuses two ranks on one device):
  each rank's device driver — pager, arena, window ring, step graph — must make
  exactly the reference's decisions on its shard (steps.csv vs the reference
  replaying the rank's sub-stream) and stage exactly the bytes the host twin of
  that shard stages (destination-hashed trace), with K-scan == host reduce.
* The in-graph collective: a world-1 NCCL communicator puts ncclAllReduce inside the
  captured step graph; the job-wide counts it returns equal the step's own, the two
  graphs are still captured once, and the job-wide single-commit audit holds.
* bench.py --gpus 2 re-launches itself as two ranks and reports n_gpus 2.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFG = {"steps": 96, "warmup_steps": 0, "seed": 5,
       "pager": {"page_bytes": 32768, "layers": 2, "kv_head_dim": 256, "elem_bytes": 2},
       "transport": {"tau_bytes": 262144},
       "far_view": {"w_star": 128},
       "shaping": {"staged_refresh_period": 4},
       "workload": {"concurrency": 64, "arrivals_per_window": 4.0, "seed": 1}}
B200 = {"kv_heads": 4, "head_dim": 64, "q_heads": 8, "payload": "lanes", "dtype": "bf16"}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2605_09735_b200 import kvrail as kv
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = json.loads(json.dumps(CFG))
    cfg["b200"] = dict(B200, shard_rank=rank, shard_world=world, trace=True, check=True)
    d = kv.Driver(cfg, device=0)
    reduced = []
    for _ in range(cfg["steps"]):
        r = d.step()
        t = torch.tensor([r.live_sessions, r.emitted_tokens, r.commits], dtype=torch.int64)
        dist.all_reduce(t)
        reduced.append(t.tolist())
    host = kv.Driver(dict(cfg, b200=dict(B200, shard_rank=rank, shard_world=world, trace=True)))
    host.run()
    checked, bad, first = d.device_check()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"csv": d.steps_csv(), "reduced": reduced, "trace_equal": d.trace() == host.trace(),
                   "scan": [checked, bad, first], "staged": list(d.staged_rows())}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_device_ranks_shard_by_sequence(tmp_path, has_ref):
    world = 2
    mp.spawn(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    runs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    rows = [[ln.split(",") for ln in r["csv"].splitlines()[1:]] for r in runs]
    for r in range(world):
        assert runs[r]["trace_equal"], f"rank {r}: device trace differs from its host twin"
        assert runs[r]["scan"][:2] == [CFG["steps"], 0], runs[r]["scan"]
        assert runs[r]["staged"][0] > 0 and runs[r]["staged"][2] == 0
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


def test_in_graph_counts_all_reduce_world_one():
    """ncclAllReduce captured in the step graph (a world-1 communicator on this GPU)."""
    from paper_2605_09735_b200 import kvrail as kv
    cfg = json.loads(json.dumps(CFG))
    cfg["b200"] = dict(B200)
    d = kv.Driver(cfg, device=0)
    d.comm_init(kv.comm_unique_id(), 0, 1)
    recs = d.run()
    d.sync()
    recs = [d.record(r.step) for r in recs]
    assert d.device().graph_captures() == 2
    for r in recs:
        assert (r.global_live, r.global_emitted, r.global_commits) == \
            (r.live_sessions, r.emitted_tokens, r.live_sessions), r.step
    assert sum(r.global_eos for r in recs) > 0
    d.close()
    with pytest.raises(kv.KvrailError, match="first step"):
        late = kv.Driver(cfg, device=0)
        late.step()
        late.comm_init(kv.comm_unique_id(), 0, 1)
    # bench.py's fallback: a communicator dropped again before the first step
    back = kv.Driver(dict(cfg, steps=8), device=0)
    back.comm_init(kv.comm_unique_id(), 0, 1)
    back.comm_destroy()
    back.run()
    back.sync()
    r = back.record(7)
    assert r.global_live == r.live_sessions


def test_bench_spawns_ranks():
    """bench.py --gpus 2 re-launches itself as two ranks (both on GPU 0 here, gloo)."""
    env = dict(os.environ, KVR_BENCH_DEVICE="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c1", "--steps", "8",
                          "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["multi_gpu"]["counts_collective"].startswith("torch.distributed")
