"""Far-view parity: summarize_chunk / select_chunks / attend (far_view.cpp:30-155)
against golden vectors produced by the reference, the reference library and
the plain-C restatement."""
import ctypes as C
import json
import math
import os
import random

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "far_view.json")


def f32(xs):
    return (C.c_float * max(1, len(xs)))(*xs)


def summarize(api, toks, lanes, count):
    o = (C.c_float * lanes)()
    api.summarize_chunk(f32(toks), lanes, count, o)
    return list(o)


def attend_history(api, c):
    o = (C.c_float * c["dim"])()
    api.attend_history(f32(c["images"]), c["t"], (C.c_double * len(c["scores"]))(*c["scores"]),
                       len(c["scores"]), 2 * c["dim"], c["w"], c["cap"], c["chunk"], f32(c["q"]), 0,
                       c["dim"], o)
    return list(o)


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_summaries_bit_exact_with_golden(golden):
    lib = ob.oracle()
    for c in golden["summarize"]:
        mine = summarize(kv.api(), c["tokens"], c["lanes"], c["count"])
        assert mine == c["mean"]
        o = (C.c_float * c["lanes"])()
        lib.kvo_summarize_chunk(f32(c["tokens"]), c["lanes"], c["count"], o)
        assert list(o) == c["mean"]


def test_select_chunks_golden(golden):
    for c in golden["select"]:
        n = C.c_uint64()
        out = (C.c_uint64 * max(1, len(c["scores"])))()
        kv.api().select_chunks((C.c_double * max(1, len(c["scores"])))(*c["scores"]),
                               len(c["scores"]), c["cap"], out, C.byref(n))
        assert list(out)[:n.value] == c["picked"]
        oo = (C.c_uint64 * max(1, len(c["scores"])))()
        m = ob.oracle().kvo_select_chunks((C.c_double * max(1, len(c["scores"])))(*c["scores"]),
                                          len(c["scores"]), c["cap"], oo)
        assert list(oo)[:m] == c["picked"]


def test_attend_bit_exact_with_golden(golden):
    for c in golden["attend"]:
        assert attend_history(kv.api(), c) == c["out"]


def test_empty_chunk_and_dimension_errors():
    with pytest.raises(kv.KvrailError) as e:
        summarize(kv.api(), [], 4, 0)
    assert e.value.code == "EmptyChunk"


def test_restated_attend_matches_reference_attend():
    rng = random.Random(4)
    lib = ob.oracle()
    for _ in range(20):
        d = rng.choice([8, 16, 64])
        n = rng.randint(1, 40)
        k = [rng.uniform(-2, 2) for _ in range(n * d)]
        v = [rng.uniform(-2, 2) for _ in range(n * d)]
        q = [rng.uniform(-1, 1) for _ in range(d)]
        out = (C.c_float * d)()
        lib.kvo_attend_rows(f32(k), d, f32(v), d, n, f32(q), d, out)
        # reference: images [K|V] with one layer, near window holding all n tokens
        imgs = []
        for i in range(n):
            imgs += k[i * d:(i + 1) * d] + v[i * d:(i + 1) * d]
        c = {"images": imgs, "t": n, "scores": [0.0], "w": n, "cap": 0, "chunk": 1, "q": q, "dim": d}
        assert list(out) == attend_history(kv.api(), c)


@pytest.mark.parametrize("seed", range(8))
def test_far_view_attention_matches_reference(seed, ref_api):
    rng = random.Random(seed)
    dim = rng.choice([8, 16])
    t = rng.randint(1, 300)
    chunk = rng.choice([1, 8, 32])
    c = {"dim": dim, "t": t, "w": rng.choice([16, 64, 128]), "cap": rng.choice([0, 4, 16]),
         "chunk": chunk, "images": [rng.uniform(-1, 1) for _ in range(t * 2 * dim)],
         "q": [rng.uniform(-1, 1) for _ in range(dim)],
         "scores": [rng.random() for _ in range(t // chunk + 1)]}
    assert attend_history(kv.api(), c) == attend_history(ref_api, c)
    assert all(math.isfinite(x) for x in c["q"])
