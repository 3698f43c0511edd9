"""Transport parity: stage()/reduce() (transport.cpp:29-127) — the reference's
unit cases restated, golden vectors from the reference, random streams against
the reference library and against the plain-C restatement (kvr_oracle.c)."""
import ctypes as C
import json
import os
import random

import pytest

from paper_2605_09735_b200 import kvrail as kv
from oracle import bindings as ob

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "transport.json")
PAGE, TOK = 16 * 1024, 1024


def desc(off, ln, kind=0, staged=0.0):
    return (off, ln, staged, kind, off // PAGE, 0)


def test_contiguous_window_is_one_descriptor():
    d = kv.stage([(1, 0, [(b, 0, 16) for b in range(4, 12)])], PAGE, TOK, 0.0)
    assert [(x[0], x[1]) for x in d] == [(4 * PAGE, 8 * PAGE)]


def test_alternating_blocks_and_partial_slots():
    d = kv.stage([(1, 0, [(b, 0, 16) for b in range(0, 16, 2)])], PAGE, TOK, 0.0)
    assert len(d) == 8 and all(x[1] == PAGE for x in d)
    d = kv.stage([(1, 0, [(3, 8, 8), (4, 0, 16)])], PAGE, TOK, 0.0)
    assert [(x[0], x[1]) for x in d] == [(3 * PAGE + 8 * TOK, 8 * TOK + PAGE)]


def test_reduce_reference_cases():
    t = kv.reduce([desc(0, 4096)], 131072, 10.0, True, 0.0)
    assert len(t) == 1 and t[0][1] == 2 and t[0][2] == 4096  # lone descriptor: flush
    t = kv.reduce([desc(i * 4096, 4096) for i in range(32)], 131072, 10.0, True, 0.0)
    assert len(t) == 1 and t[0][2] == 131072 and t[0][1] == 0 and len(t[0][5]) == 32
    t = kv.reduce([desc(0, PAGE, 0), desc(PAGE, PAGE, 1)], 131072, 10.0, True, 0.0)
    assert [x[0] for x in t] == [0, 1]  # kinds never mix
    t = kv.reduce([desc(0, PAGE, 0, 0.0), desc(PAGE, PAGE, 0, 9.5)], 1 << 20, 5.0, True, 10.0)
    assert len(t) == 2 and t[0][1] == 1  # age guard
    t = kv.reduce([desc(0, 256 * 1024), desc(256 * 1024, PAGE)], 131072, 10.0, True, 0.0)
    assert len(t) == 2 and t[0][1] == 0  # > tau travels alone
    t = kv.reduce([desc(3 * PAGE, PAGE), desc(0, PAGE), desc(PAGE, PAGE)], 131072, 10.0, False, 0.0)
    assert [x[5][0][0] for x in t] == [3 * PAGE, 0, PAGE]  # merge off: input order
    with pytest.raises(kv.KvrailError) as e:
        kv.reduce([desc(0, 1)], 0, 1.0, True, 0.0)
    assert e.value.code == "BadConfig"


def test_golden_vectors_from_the_reference():
    with open(GOLDEN) as f:
        cases = json.load(f)
    for c in cases:
        needs = [(s, k, [tuple(x) for x in sp]) for s, k, sp in c["needs"]]
        got = kv.stage(needs, c["page"], c["tok"], c["now"])
        assert [list(x) for x in got] == c["descs"]
        tr = kv.reduce([tuple(x) for x in c["reduce_in"]], c["tau"], c["hold"], c["merge"],
                       c["reduce_now"])
        assert json.loads(json.dumps(tr)) == c["trains"]


def oracle_stage_reduce(needs, tau, hold, merge, now):
    lib = ob.oracle()
    lib.kvo_stage.argtypes = [C.POINTER(kv.StageNeed), C.c_uint64, C.POINTER(kv.StagedSpan),
                              C.c_uint64, C.c_uint64, C.c_double, C.POINTER(kv.Descriptor),
                              C.c_uint64, C.POINTER(C.c_uint64)]
    lib.kvo_reduce.argtypes = [C.POINTER(kv.Descriptor), C.c_uint64, C.POINTER(kv.TransportConfig),
                               C.c_double, C.POINTER(kv.Train), C.c_uint64, C.POINTER(C.c_uint64),
                               C.POINTER(kv.Descriptor), C.POINTER(C.c_uint64)]
    spans, recs = [], []
    for s, k, sp in needs:
        recs.append(kv.StageNeed(s, k, len(spans), len(sp)))
        spans += [kv.StagedSpan(*x) for x in sp]
    nn = (kv.StageNeed * max(1, len(recs)))(*recs)
    ss = (kv.StagedSpan * max(1, len(spans)))(*spans)
    out = (kv.Descriptor * (len(spans) + 1))()
    n = C.c_uint64()
    lib.kvo_stage(nn, len(recs), ss, PAGE, TOK, now, out, len(spans) + 1, C.byref(n))
    descs = [out[i].astuple() for i in range(n.value)]
    cfg = kv.TransportConfig(tau, hold, 2, int(merge))
    tr = (kv.Train * (len(descs) + 1))()
    od = (kv.Descriptor * max(1, len(descs)))()
    nt, ties = C.c_uint64(), C.c_uint64()
    arr = (kv.Descriptor * max(1, len(descs)))(*[kv.Descriptor(o, l, st, k, b, s, 0)
                                                  for o, l, st, k, b, s in descs])
    lib.kvo_reduce(arr, len(descs), C.byref(cfg), now, tr, len(descs) + 1, C.byref(nt), od,
                   C.byref(ties))
    trains = [(t.kind, t.reason, t.total_bytes, t.oldest_stage_time, t.issue_time,
               [od[k].astuple() for k in range(t.desc_begin, t.desc_begin + t.desc_count)])
              for t in tr[:nt.value]]
    return descs, trains, ties.value


@pytest.mark.parametrize("seed", range(40))
def test_random_needs_match_reference_and_restatement(seed, ref_api):
    rng = random.Random(seed)
    needs = []
    used = set()
    for _ in range(rng.randint(1, 8)):
        sp = []
        for _ in range(rng.randint(0, 12)):
            b = rng.randrange(96)
            if b in used:
                continue
            used.add(b)
            sb = rng.choice([0, 0, rng.randrange(16)])
            sp.append((b, sb, rng.randint(0, 16 - sb)))
        needs.append((rng.randrange(1, 20), rng.randrange(2), sp))
    tau = rng.choice([PAGE, 4 * PAGE, 8 * PAGE, 64 * PAGE])
    hold = rng.choice([0.0, 0.25, 5.0])
    merge = rng.random() < 0.85
    now = float(rng.randrange(100))
    mine_d = kv.stage(needs, PAGE, TOK, now)
    ref_d = kv.stage(needs, PAGE, TOK, now, api_=ref_api)
    assert mine_d == ref_d
    mine_t = kv.reduce(mine_d, tau, hold, merge, now)
    ref_t = kv.reduce(ref_d, tau, hold, merge, now, api_=ref_api)
    assert mine_t == ref_t
    o_d, o_t, ties = oracle_stage_reduce(needs, tau, hold, merge, now)
    assert o_d == mine_d
    assert ties == 0 and o_t == mine_t


@pytest.mark.parametrize("seed", range(20))
def test_page_run_merge_matches_restatement(seed):
    """The B200 page-run rule (TransportConfig::run_page_bytes): 12-token pages with
    slack (span 12 * TOK of a 16 KiB page). Host reduce() == the C restatement; the
    policy never joins non-consecutive pages or kinds, and never needs more trains
    than exact abutment."""
    rng = random.Random(seed)
    span = 12 * TOK
    ds = []
    for b in rng.sample(range(80), rng.randint(1, 40)):
        sb = rng.choice([0, 0, 0, rng.randrange(12)])
        n = rng.choice([12 - sb, rng.randint(1, 12 - sb)])
        ds.append((b * PAGE + sb * TOK, n * TOK, 5.0, rng.choice([0, 0, 1]), b, 0))
    tau = rng.choice([4 * PAGE, 16 * PAGE, 1 << 40])
    mine = kv.reduce(ds, tau, 10.0, True, 5.0, run_page=PAGE, run_span=span)
    exact = kv.reduce(ds, tau, 10.0, True, 5.0)
    assert len(mine) <= len(exact)
    lib = ob.oracle()
    cfg = kv.TransportConfig(tau, 10.0, 2, 1, PAGE, span)
    tr = (kv.Train * (len(ds) + 1))()
    od = (kv.Descriptor * len(ds))()
    nt, ties = C.c_uint64(), C.c_uint64()
    arr = (kv.Descriptor * len(ds))(*[kv.Descriptor(o, l, st, k, b, s, 0) for o, l, st, k, b, s in ds])
    assert lib.kvo_reduce(arr, len(ds), C.byref(cfg), 5.0, tr, len(ds) + 1, C.byref(nt), od, C.byref(ties)) == 0
    oracle_t = [(t.kind, t.reason, t.total_bytes, t.oldest_stage_time, t.issue_time,
                 [od[k].astuple() for k in range(t.desc_begin, t.desc_begin + t.desc_count)])
                for t in tr[:nt.value]]
    assert oracle_t == mine
    for kind, _, _, _, _, dd in mine:
        for a, b in zip(dd, dd[1:]):
            end = a[0] + a[1]
            assert a[3] == b[3] == kind
            assert end == b[0] or (end % PAGE == span and b[0] == end - span + PAGE)


def test_reduce_invariants():
    rng = random.Random(31)
    for _ in range(60):
        now = 100.0
        ds = []
        for b in rng.sample(range(64), rng.randint(1, 40)):
            ds.append((b * PAGE, PAGE, now - rng.randrange(8), 0, b, 0))
        merged = kv.reduce(ds, 131072, 6.0, True, now)
        unmerged = kv.reduce(ds, 131072, 6.0, False, now)
        assert sum(t[2] for t in merged) == sum(t[2] for t in unmerged)
        assert sum(len(t[5]) for t in merged) == len(ds)
        for kind, reason, total, oldest, _, dd in merged:
            if reason == 0:
                assert total >= 131072
            if reason == 1:
                assert now - oldest >= 6.0
            for a, b in zip(dd, dd[1:]):
                assert a[0] + a[1] == b[0]
        assert len(merged) <= len(unmerged)
