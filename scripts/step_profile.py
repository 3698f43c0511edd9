"""Per-step device-phase dump of the C2 bench workload (diagnostics)."""
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_09735_b200 as pkg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
cfg = bench.c2_config(400 + steps)
d = pkg.Driver(cfg, device=0)
first = None
for i in range(400 + steps):
    r = d.step()
    if first is None and r.live_sessions >= 64:
        first = r.step + 5
    if first is not None and r.step >= first + steps:
        break
d.sync()
print("step live emit  wb_tok  dev_ms  apply  hotwq  fmp    scan   gath   attn   tail")
for s in range(first, first + steps):
    r = d.record(s)
    p = list(r.phase_ms)
    print(f"{s:4d} {r.live_sessions:4d} {r.emitted_tokens:4d} {r.writeback_tokens:7d} {r.device_ms:6.3f} " +
          " ".join(f"{x:6.3f}" for x in p[:7]))
