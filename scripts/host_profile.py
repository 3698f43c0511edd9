"""Steady-state host time per decode step, by section (KVR_HOST_PROFILE).

Runs the bench config twice on the device — fill + warm-up only, then fill +
warm-up + N steps — and prints the difference per step for each host section
(the driver prints its totals to stderr when it is destroyed).
usage: python scripts/host_profile.py c3 [N]
"""
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


def run(cfg: str, n: int) -> dict:
    env = dict(os.environ, KVR_HOST_PROFILE="1")
    p = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, cfg=cfg, n=n)], env=env,
                       capture_output=True, text=True, check=True)
    line = [l for l in p.stderr.splitlines() if l.startswith("host ms:")][-1]
    return {k: float(v) for k, v in re.findall(r"([a-z/]+) ([0-9.]+)", line)}


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    a, b = run(cfg, 0), run(cfg, n)
    per = {k: (b[k] - a[k]) / n for k in b}
    print(cfg, "steady host ms/step:", {k: round(v, 4) for k, v in per.items()},
          "total", round(sum(per.values()), 4))
