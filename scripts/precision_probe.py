import copy, json, os, sys
sys.path.insert(0, ".")
from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob
GOLD = "tests/golden"
def c1():
    cfg = json.load(open(os.path.join(GOLD, "c1_config.json")))
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    return cfg
for kernel, dtype, kvh, qh, payload, query in [
        ("tcgen05", "bf16", 1, 8, "wide", "f32"), ("tcgen05", "bf16", 1, 8, "wide", "exact"),
        ("tcgen05", "bf16", 1, 8, "lanes", "f32"), ("cuda_core", "bf16", 1, 8, "wide", "f32"),
        ("tcgen05", "fp16", 1, 8, "wide", "f32"), ("cuda_core", "fp16", 1, 8, "wide", "f32"),
        ("tcgen05", "bf16", 2, 8, "wide", "f32"), ("cuda_core", "bf16", 2, 8, "wide", "f32"),
        ("tcgen05", "bf16", 2, 4, "wide", "f32")]:
    hd = 128
    cfg = c1(); cfg["steps"] = 40
    cfg["pager"]["kv_head_dim"] = kvh * hd
    cfg["pager"]["page_bytes"] = 16 * 2 * 2 * kvh * hd * 2
    cfg["transport"]["tau_bytes"] = 8 * cfg["pager"]["page_bytes"]
    cfg["far_view"]["w_star"] = 512
    cfg["b200"] = dict(kv_heads=kvh, head_dim=hd, q_heads=qh, payload=payload, query=query, dtype=dtype,
                       attention_kernel=kernel)
    d = kv.Driver(cfg, device=0); d.run()
    print(kernel, dtype, kvh, qh, payload, query, "%.3e" % ob.check_driver_window_and_attention(d), flush=True)
