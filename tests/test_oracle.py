"""Pin the plain-C restatement (oracle/kvr_oracle.c) before trusting it:
golden vectors, the reference library, and the bytes the (reference-exact)
driver twin actually stores."""
import ctypes as C
import json
import os
import random

import numpy as np
import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_payload_golden():
    lib = ob.oracle()
    for row in json.load(open(os.path.join(GOLD, "payload.json"))):
        buf = C.create_string_buffer(row["token_bytes"])
        lib.kvo_fill_token_payload(row["seed"], row["session"], row["token"], row["token_bytes"],
                                   row["elem_bytes"], buf)
        assert lib.kvo_fnv1a(buf, row["token_bytes"], 0) == row["fnv"]


@pytest.mark.parametrize("elem_bytes,payload", [(2, "bytes"), (4, "bytes"), (2, "lanes"), (2, "wide")])
def test_restated_payload_equals_stored_bytes(elem_bytes, payload):
    """Every written token the twin driver stored (pinned to the reference by
    the staged-byte hashes of the golden traces) equals the restatement."""
    cfg = json.load(open(os.path.join(GOLD, "c1_config.json")))
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    cfg["steps"] = 12
    cfg["pager"]["elem_bytes"] = elem_bytes
    if elem_bytes == 4:
        cfg["pager"]["page_bytes"] = 65536
        cfg["transport"]["tau_bytes"] = 8 * 65536
    cfg["b200"] = {"payload": payload, "dtype": "fp16"}
    d = kv.Driver(cfg)
    d.run()
    p = d.pager()
    tb = p.cfg.token_bytes()
    lib = ob.oracle()
    buf = C.create_string_buffer(tb)
    shift = 3 if payload == "wide" else 7  # lanes (b - 128) / 2^shift
    checked = 0
    for slot, session, written in d.live():
        view = p.active_view(session)
        for t in range(0, written, 7):
            got = ob.token_bytes_via_view(p, view, t, tb)
            if payload == "bytes":
                lib.kvo_fill_token_payload(cfg["seed"], session, t, tb, elem_bytes, buf)
            else:
                lib.kvo_fill_token_lanes_shift(cfg["seed"], session, t, tb // elem_bytes, 1, shift, buf)
            if t < 64 and got != buf.raw:  # aliased shared prefix holds template-0 bytes
                if payload == "bytes":
                    lib.kvo_fill_token_payload(cfg["seed"], 0, t, tb, elem_bytes, buf)
                else:
                    lib.kvo_fill_token_lanes_shift(cfg["seed"], 0, t, tb // elem_bytes, 1, shift, buf)
            assert got == buf.raw, (session, t)
            checked += 1
    assert checked > 100


def test_f32_query_restatement():
    """b200.query = f32: 24-bit lanes in [-1, 1), two per splitmix64, generally not
    representable in fp16 / bf16 (the tensor-core kernel's lo terms are non-zero)."""
    import numpy as np
    q = ob.fill_query(7, 3, 11, 2, 5, 128, 2, 1)
    assert all(-1.0 <= v < 1.0 for v in q) and len(set(q)) == 128
    assert all(float(np.float32(v)) == v and (v * 2 ** 23).is_integer() for v in q)
    bf = np.asarray(q, np.float32).view(np.uint32) & 0xFFFF
    assert (bf != 0).mean() > 0.9
    assert ob.fill_query(7, 3, 11, 2, 5, 128, 2, 0) != q  # mode 0: the exact byte lanes


def test_half_and_bf16_rounding_match_numpy_and_torch():
    import torch
    lib = ob.oracle()
    lib.kvo_float_to_half.argtypes = [C.c_float]
    lib.kvo_float_to_half.restype = C.c_uint16
    lib.kvo_float_to_bf16.argtypes = [C.c_float]
    lib.kvo_float_to_bf16.restype = C.c_uint16
    rng = random.Random(3)
    vals = [rng.uniform(-1, 1) * 10 ** rng.randint(-9, 5) for _ in range(4000)]
    vals += [0.0, -0.0, 65504.0, 65520.0, 1e-8, 6.1e-5, 5.96e-8, 2.98e-8]
    for v in vals:
        f = float(np.float32(v))
        assert lib.kvo_float_to_half(f) == int(np.array([f], np.float32).astype(np.float16).view(np.uint16)[0])
        assert lib.kvo_float_to_bf16(f) == int(torch.tensor([f]).to(torch.bfloat16).view(torch.int16)[0]) & 0xFFFF
        h = lib.kvo_float_to_half(f)
        assert lib.kvo_half_to_float(h) == float(np.array([h], np.uint16).view(np.float16)[0])


def test_lanes_f32_equals_reference_float_pattern():
    lib = ob.oracle()
    a, b = C.create_string_buffer(4096), C.create_string_buffer(4096)
    for tok in (0, 5, 999):
        lib.kvo_fill_token_payload(7, 3, tok, 4096, 4, a)
        lib.kvo_fill_token_lanes(7, 3, tok, 1024, 0, b)
        assert a.raw == b.raw


def test_restated_window_attention_against_reference_attend():
    """kvo_attend_window (GQA slicing of a token-major window) == reference attend
    on the (layer, kv-head) slice."""
    rng = random.Random(8)
    lib = ob.oracle()
    L, H, hd = 2, 4, 16
    lanes = 2 * L * H * hd
    n = 40
    win = np.array([rng.uniform(-1, 1) for _ in range(n * lanes)], np.float32)
    q = [rng.uniform(-1, 1) for _ in range(hd)]
    for layer in range(L):
        for kvh in range(H):
            got = ob.attend_window(win.tobytes(), n, L, H, hd, 0, layer, kvh, q)
            imgs = []
            for t in range(n):
                row = win[t * lanes:(t + 1) * lanes]
                k0 = 2 * layer * H * hd + kvh * hd
                imgs += list(row[k0:k0 + hd]) + list(row[k0 + H * hd:k0 + H * hd + hd])
            o = (C.c_float * hd)()
            kv.api().attend_history((C.c_float * len(imgs))(*imgs), n, (C.c_double * 1)(0.0), 1,
                                    2 * hd, n, 0, 1, (C.c_float * hd)(*q), 0, hd, o)
            assert got == list(o)
