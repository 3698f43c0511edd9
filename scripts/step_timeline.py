"""In-graph kernel timeline of quiet steps (KVR_TIMELINE=1, kvr_dev_timeline): per kernel,
the first-CTA start offset
from the step's first kernel and the span to its last exit (median over the quiet
steps of a run), plus device_ms. Usage: python scripts/step_timeline.py c5"""
import json, os, statistics, sys
os.environ["KVR_TIMELINE"] = "1"
sys.path.insert(0, ".")
import bench
import paper_2605_09735_b200 as pkg
name = sys.argv[1]
steps = 40
cfg = bench.CONFIGS[name](400 + steps + 10, 0, 1)
cfg["b200"]["transfer"] = "page_runs"
d = pkg.Driver(cfg, device=0)
width = cfg["workload"]["concurrency"]
for _ in range(400):
    r = d.step()
    if r.live_sessions >= width:
        break
for _ in range(5):
    d.step()
d.sync()
dev = d.device()
dev.timeline()
rows = []
for _ in range(steps):
    r = d.step()
    d.sync()
    tl = dev.timeline()
    rec = d.record(r.step)
    rows.append((rec, tl))
quiet = [(r, t) for r, t in rows if r.writeback_tokens <= width]
out = {"config": name, "quiet_steps": len(quiet), "device_ms_p50": statistics.median(r.device_ms for r, _ in quiet)}

per = {}
for r, t in quiet:
    t0 = min(v[0] for v in t.values())
    t1 = max(v[1] for v in t.values())
    per.setdefault("_span_us", []).append((t1 - t0) / 1e3)
    for k, (a, b) in t.items():
        per.setdefault(k, []).append(((a - t0) / 1e3, (b - a) / 1e3))
for k, v in per.items():
    if k == "_span_us":
        out[k] = statistics.median(v)
    else:
        out[k] = {"start_us": round(statistics.median(x[0] for x in v), 2),
                  "dur_us": round(statistics.median(x[1] for x in v), 2)}
print(json.dumps(out))
