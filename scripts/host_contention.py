"""Host control plane per GPU when 8 drivers share one host (SURVEY §8(f)1 question).

Each B200 of an 8-GPU box runs its own driver process (pager, stage/reduce, descriptor
packing). This runs P such processes at once on this box's host cores — all on GPU 0,
with the bench config's control plane unchanged (same batch, pages per token run,
tokens per page, workload, regime) but KV rows shrunk so P arenas fit one GPU and the
attention off — and reports each process's host ms per steady step (KVR_HOST_PROFILE
sections except `device`, which includes waiting for the shared GPU) for P = 1 and P.
usage: python scripts/host_contention.py c3 [P] [steps]
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys
sys.path.insert(0, {root!r})
import bench
from paper_2605_09735_b200 import kvrail as kv
cfg = bench.CONFIGS[{cfg!r}](10**6, 0, 1)
p = cfg["pager"]
scale = p["kv_head_dim"] // 64
p["kv_head_dim"], p["page_bytes"] = 64, p["page_bytes"] // scale
cfg["transport"]["tau_bytes"] //= scale
cfg["b200"].update(kv_heads=1, head_dim=64, q_heads=4, attention=False)
d = kv.Driver(cfg, device=0)
width = cfg["workload"]["concurrency"]
for _ in range(400):
    if d.step().live_sessions >= width:
        break
for _ in range(5 + {n}):
    d.step()
d.sync()
del d
'''


def launch(cfg: str, n: int):
    env = dict(os.environ, KVR_HOST_PROFILE="1")
    return subprocess.Popen([sys.executable, "-c", CODE.format(root=ROOT, cfg=cfg, n=n)], env=env,
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)


def sections(proc) -> dict:
    _, err = proc.communicate()
    if proc.returncode:
        raise RuntimeError(err[-2000:])
    line = [ln for ln in err.splitlines() if ln.startswith("host ms:")][-1]
    return {k: float(v) for k, v in re.findall(r"([a-z/]+) ([0-9.]+)", line)}


def per_step(cfg: str, procs: int, n: int) -> list[float]:
    """Host ms per steady step (sections other than `device`) of each of `procs` concurrent drivers."""
    base = [sections(p) for p in [launch(cfg, 0) for _ in range(procs)]]
    full = [sections(p) for p in [launch(cfg, n) for _ in range(procs)]]
    host = lambda s: sum(v for k, v in s.items() if k != "device")
    return [(host(b) - host(a)) / n for a, b in zip(base, full)]


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 300
    alone = per_step(cfg, 1, n)
    shared = per_step(cfg, P, n)
    print(json.dumps({"config": cfg, "host_cores": os.cpu_count(), "steps": n,
                      "host_ms_per_step_alone": alone[0],
                      f"host_ms_per_step_{P}_drivers": shared,
                      "max_slowdown": max(shared) / alone[0]}))
