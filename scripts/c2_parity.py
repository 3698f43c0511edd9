"""C2-scale parity spot check: window ring bytes and attention of sampled slots
against the double-precision oracle after the bench's fill + warm-up steps."""
import sys
import time
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_09735_b200 as pkg  # noqa: E402
from oracle import bindings as ob  # noqa: E402

cfg = bench.c2_config(400)
d = pkg.Driver(cfg, device=0)
for i in range(400):
    r = d.step()
    if r.live_sessions >= 64:
        break
for _ in range(8):
    d.step()
d.sync()
t = time.time()
heads = {(l, h) for l in (0, 13, 31) for h in (0, 7, 31)}
worst = ob.check_driver_window_and_attention(d, only_slots={0, 21, 63}, heads=heads)
print(f"C2 slots 0/21/63, 9 (layer, head) pairs each: window exact, attention max rel err {worst:.3e}"
      f" ({time.time() - t:.1f}s)")
