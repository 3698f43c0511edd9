"""Full-scale control-plane parity: the B200 run of a bench config (real geometry,
payload in HBM, K-scan checked against host reduce every step) against the
reference Driver (oracle/_ref) run on the same workload with kv_head_dim and
page_bytes shrunk by one power of two (identical tokens per page, page counts and
tau in pages, so every pager / stage / reduce decision is the same). Per step the
geometry-free columns must match exactly and the byte columns after rescaling.
Usage: scale_control_parity.py [c2|c3|c5] [steps]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_09735_b200 as pkg  # noqa: E402
from oracle import bindings as ob  # noqa: E402
from oracle.cpu_baseline import shrink_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cfg = bench.CONFIGS[name](steps)
cfg["b200"]["check"] = True
d = pkg.Driver(cfg, device=0)
d.run()
checked, bad, first = d.device_check()
dev = [r.split(",") for r in d.steps_csv().strip().split("\n")]

small, scale = shrink_config(cfg)
p = cfg["pager"]
tb = 2 * p["layers"] * p["kv_head_dim"] * p["elem_bytes"]
csv, _, _, _ = ob.ref_scenario(small)
ref = [r.split(",") for r in csv.strip().split("\n")]
assert dev[0] == ref[0], (dev[0], ref[0])
col = {c: i for i, c in enumerate(ref[0])}
exact = ["step", "live_sessions", "trains", "near_trains", "far_trains", "commits", "emitted_tokens"]
scaled_cols = ["dma_bytes", "reserved_bytes", "active_bytes"]
mism = 0
for a, b in zip(dev[1:], ref[1:]):
    ok = all(a[col[c]] == b[col[c]] for c in exact)
    ok &= all(int(a[col[c]]) == int(b[col[c]]) * scale for c in scaled_cols)
    if not ok and mism < 3:
        print("mismatch", a, b)
    mism += not ok
print(f"{name}: {len(dev) - 1} steps, tokens/page {p['page_bytes'] // tb}, byte scale {scale}: "
      f"{len(dev) - 1 - mism} steps identical (live, trains near/far, commits, emitted exact; "
      f"dma/reserved/active bytes x{scale}); device K-scan == host reduce on {checked - bad}/{checked} steps")
assert mism == 0 and bad == 0 and len(dev) == len(ref)
