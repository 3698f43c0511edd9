"""Ad-hoc GPU bring-up: run the smoke config step by step with/without graphs."""
import copy
import sys
import time

sys.path.insert(0, ".")
import __graft_entry__ as g  # noqa: E402
import paper_2605_09735_b200 as pkg  # noqa: E402
from oracle import bindings as ob  # noqa: E402

print("devices:", pkg.device_count(), flush=True)
host = pkg.Driver(g.SMOKE_CONFIG, device=-1)
host.run()
for graph in (0, 1):
    cfg = copy.deepcopy(g.SMOKE_CONFIG)
    cfg["b200"]["graph"] = graph
    t0 = time.time()
    d = pkg.Driver(cfg, device=0)
    print(f"graph={graph} opened in {time.time()-t0:.2f}s", flush=True)
    for i in range(cfg["steps"]):
        r = d.step()
        print(f"  step {r.step} live {r.live_sessions} trains {r.trains} dev_ms {r.device_ms:.3f}", flush=True)
    print("  trace equal:", d.trace() == host.trace(), " csv equal:", d.steps_csv() == host.steps_csv())
    if d.trace() != host.trace():
        a, b = d.trace().splitlines(), host.trace().splitlines()
        for i, (x, y) in enumerate(zip(a, b)):
            if x != y:
                print("  first diff", i, "\n   DEV ", x[:200], "\n   HOST", y[:200])
                break
    print("  device check:", d.device_check())
    print("  attn variant:", d.device().attention_variant())
    try:
        print("  window+attention worst rel err:", ob.check_driver_window_and_attention(d))
    except AssertionError as e:
        print("  CHECK FAILED:", e)
