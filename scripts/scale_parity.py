"""Full-scale parity spot check: after the bench's fill + warm-up steps, the window
ring bytes of sampled slots equal the arena (through the pager's view), far rows
equal their summary slots, and the attention of sampled (layer, q-head) pairs is
within 1e-3 of the double-precision oracle. Usage: scale_parity.py [c2|c3|c5] [slots]."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_09735_b200 as pkg  # noqa: E402
from oracle import bindings as ob  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name](400)
if len(sys.argv) > 2:  # fewer slots: same per-slot geometry, quicker check
    cfg["workload"]["concurrency"] = int(sys.argv[2])
d = pkg.Driver(cfg, device=0)
width = cfg["workload"]["concurrency"]
for i in range(400):
    r = d.step()
    if r.live_sessions >= width:
        break
for _ in range(8):
    d.step()
d.sync()
L, hq = cfg["pager"]["layers"], cfg["b200"]["q_heads"]
slots = {0, width // 3, width - 1}
heads = {(l, h) for l in (0, L // 2, L - 1) for h in (0, hq // 2 + 1, hq - 1)}
t = time.time()
worst = ob.check_driver_window_and_attention(d, only_slots=slots, heads=heads)
variant = d.device().attention_variant()
print(f"{name} [{variant}] slots {sorted(slots)}, {len(heads)} (layer, q-head) pairs each: window "
      f"exact, far rows exact, attention max rel err {worst:.3e} ({time.time() - t:.1f}s)")
assert worst <= 1e-3
