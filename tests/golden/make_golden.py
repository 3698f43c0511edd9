"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Runs in the build container only (needs oracle/_ref, i.e. /root/reference):
    python tests/golden/make_golden.py
Every fixture is produced by the UNMODIFIED reference library compiled from its
own sources (oracle/Makefile) through the C shim oracle/ref_shim.cpp:
  c1_events.csv / c1_config.json      BASELINE configs[0] (tiny decoder, 8 requests,
                                      64 decode steps, fixed EOS schedule)
  c1_steps.csv / c1_report.json / c1_trace.txt   reference run_scenario outputs
  audit_trace.txt ...                 the default audit config, 300 steps
  transport.json                      stage()/reduce() on seeded random needs
  far_view.json                       summarize_chunk / select_chunks / attend cases
  payload.json                        fill_token_payload FNV hashes (scenario.cpp:189-206
                                      restated in oracle/kvr_oracle.c; pinned here
                                      through the reference Driver's staged-byte hashes)
"""
from __future__ import annotations

import ctypes as C
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings as ob  # noqa: E402
from paper_2605_09735_b200 import kvrail as kv  # noqa: E402

C1_PROMPTS = [64, 100, 160, 224, 288, 352, 448, 512]
C1_GENS = [8, 64, 16, 64, 32, 48, 24, 64]


def c1_config(trace_path: str) -> dict:
    """configs[0]: 2 layers, 4 KV heads x hd 64 (kv_head_dim 256), bf16-sized
    elements (2 B), 16-token pages, 8 requests 64-512 ctx, 64 steps."""
    return {
        "label": "c1", "seed": 1, "steps": 64, "warmup_steps": 0,
        "pager": {"page_bytes": 32768, "layers": 2, "kv_head_dim": 256, "elem_bytes": 2},
        "transport": {"tau_bytes": 8 * 32768},
        "far_view": {"w_star": 512},
        "trace_path": trace_path,
        "shaping": {"arena_pages": 1024, "staged_refresh_period": 4},
    }


AUDIT = {"steps": 300, "warmup_steps": 100}
FAR = {"steps": 400, "warmup_steps": 50,
       "far_view": {"enabled": True, "w_star": 128, "cap": 16, "sv_chunk": 32},
       "pager": {"layers": 1, "kv_head_dim": 64, "elem_bytes": 4, "page_bytes": 16384},
       "workload": {"concurrency": 16}}
ADV_BURST = {"steps": 500, "warmup_steps": 100, "mode": {"regime": "adversarial-random"},
             "eos_burst": {"step": 400, "fraction": 0.5}}


def write(name: str, text: str):
    with open(os.path.join(HERE, name), "w") as f:
        f.write(text)


def scenario_fixtures():
    ev = os.path.join(HERE, "c1_events.csv")
    write("c1_events.csv", "arrival_ms,prompt_tokens,generate_tokens\n" +
          "".join(f"0,{p},{g}\n" for p, g in zip(C1_PROMPTS, C1_GENS)))
    cfg = c1_config("tests/golden/c1_events.csv")
    write("c1_config.json", json.dumps(cfg, indent=1) + "\n")
    run = dict(cfg, trace_path=ev)
    csv, rep, tr, _ = ob.ref_scenario(run, trace=True)
    write("c1_steps.csv", csv)
    write("c1_report.json", rep)
    write("c1_trace.txt", tr)
    for name, cfg in (("audit", AUDIT), ("far", FAR), ("adv_burst", ADV_BURST)):
        write(f"{name}_config.json", json.dumps(cfg, indent=1) + "\n")
        csv, rep, tr, _ = ob.ref_scenario(cfg, trace=True)
        write(f"{name}_steps.csv", csv)
        write(f"{name}_trace.txt", tr)


def transport_fixtures():
    api = ob.ref_api()
    rng = random.Random(5)
    cases = []
    for trial in range(40):
        page, tok = 16384, 1024
        needs = []
        for n in range(rng.randint(1, 6)):
            spans = []
            for _ in range(rng.randint(0, 8)):
                b = rng.randrange(64)
                sb = rng.choice([0, 0, 0, rng.randrange(16)])
                cnt = rng.randint(0, 16 - sb)
                spans.append((b, sb, cnt))
            needs.append((rng.randrange(1, 9), rng.randrange(2), spans))
        now = float(rng.randint(0, 50))
        descs = kv.stage(needs, page, tok, now, api_=api)
        # drop exact (kind, offset) duplicates: the reference sort order is unspecified on ties
        seen, uniq = set(), []
        for d in descs:
            if (d[3], d[0]) not in seen:
                seen.add((d[3], d[0]))
                uniq.append(d)
        tau = rng.choice([16384, 65536, 131072, 1 << 20])
        hold = rng.choice([0.0, 0.5, 10.0])
        merge = rng.random() < 0.8
        trains = kv.reduce(uniq, tau, hold, merge, now + rng.choice([0, 1, 5]), api_=api)
        cases.append({"needs": needs, "page": page, "tok": tok, "now": now, "descs": descs,
                      "reduce_in": uniq, "tau": tau, "hold": hold, "merge": merge,
                      "reduce_now": None, "trains": trains})
        cases[-1]["reduce_now"] = trains[0][4] if trains else now
    write("transport.json", json.dumps(cases) + "\n")


def far_fixtures():
    api = ob.ref_api()
    rng = random.Random(9)
    out = {"summarize": [], "select": [], "attend": []}
    for _ in range(6):
        lanes, count = rng.choice([(16, 5), (32, 128), (8, 1)])
        toks = [rng.randint(-1000, 1000) / 500.0 for _ in range(lanes * count)]
        o = (C.c_float * lanes)()
        api.summarize_chunk((C.c_float * len(toks))(*toks), lanes, count, o)
        out["summarize"].append({"lanes": lanes, "count": count, "tokens": toks, "mean": list(o)})
    for _ in range(10):
        scores = [rng.randint(0, 50) / 10.0 for _ in range(rng.randint(0, 12))]
        cap = rng.randint(0, 6)
        buf = (C.c_uint64 * max(1, len(scores)))()
        n = C.c_uint64()
        api.select_chunks((C.c_double * max(1, len(scores)))(*scores), len(scores), cap, buf,
                          C.byref(n))
        out["select"].append({"scores": scores, "cap": cap, "picked": list(buf)[:n.value]})
    for t, w, cap, chunk in ((40, 64, 8, 16), (300, 128, 16, 32), (1, 4, 2, 2), (64, 16, 64, 1)):
        dim = 8
        lanes = 2 * dim
        imgs = [rng.randint(-1000, 1000) / 700.0 for _ in range(t * lanes)]
        q = [rng.randint(-1000, 1000) / 900.0 for _ in range(dim)]
        scores = [rng.random() for _ in range(t // max(1, chunk) + 1)]
        o = (C.c_float * dim)()
        api.attend_history((C.c_float * len(imgs))(*imgs), t, (C.c_double * len(scores))(*scores),
                           len(scores), lanes, w, cap, chunk, (C.c_float * dim)(*q), 0, dim, o)
        out["attend"].append({"t": t, "w": w, "cap": cap, "chunk": chunk, "dim": dim,
                              "images": imgs, "scores": scores, "q": q, "out": list(o)})
    write("far_view.json", json.dumps(out) + "\n")


def payload_fixtures():
    lib = ob.oracle()
    rows = []
    for seed, sess, tok, tb, eb in ((1, 0, 0, 1024, 2), (1, 7, 63, 2048, 2), (3, 5, 100, 256, 4),
                                    (42, 1 << 20, 4095, 4096, 4)):
        buf = C.create_string_buffer(tb)
        lib.kvo_fill_token_payload(seed, sess, tok, tb, eb, buf)
        rows.append({"seed": seed, "session": sess, "token": tok, "token_bytes": tb,
                     "elem_bytes": eb, "fnv": lib.kvo_fnv1a(buf, tb, 0)})
    write("payload.json", json.dumps(rows) + "\n")


if __name__ == "__main__":
    if not ob.ref_available():
        sys.exit("oracle/_ref not built: run `make -C oracle ref` in the build container")
    scenario_fixtures()
    transport_fixtures()
    far_fixtures()
    payload_fixtures()
    print("golden fixtures written to", HERE)
