"""Pager parity: the reference unit tests (test_pager.cpp) restated against the
B200 pager, plus randomized verb streams driven through BOTH the B200 pager and
the reference pager (oracle/_ref) with every observable compared after every
verb: returned blocks, errors, views, epochs, refcounts, free runs, stats,
work counters and reconstructed bytes."""
import random

import pytest

from paper_2605_09735_b200 import kvrail as kv


def small(pages=64):
    return kv.PagerConfig(512, pages, 1, 8, 2)  # 32-byte tokens, 16 per page


def payload(n, tag, tb=32):
    return bytes(((tag * 131 + i * 7) & 0xFF) for i in range(n * tb))


def code(fn, *a):
    try:
        fn(*a)
    except kv.KvrailError as e:
        return e.code
    return None


def test_config_validation():
    p = kv.api()
    c = small()
    assert c.tokens_per_page() == 16
    c.page_bytes = 500
    with pytest.raises(kv.KvrailError):
        p.pager_config_validate(c)
    c = small()
    c.page_bytes = 16
    with pytest.raises(kv.KvrailError):
        p.pager_config_validate(c)


def test_reserve_arithmetic_and_tail_reuse():
    p = kv.Pager(small())
    p.create_session(1)
    assert p.reserve(1, 0) == [] and p.stats().free_pages == 64
    b = p.reserve(1, 17)
    assert len(b) == 2 and sum(c for _, c in b) == 32
    p2 = kv.Pager(small())
    p2.create_session(1)
    assert len(p2.reserve(1, 10)) == 1
    assert p2.reserve(1, 6) == []
    assert len(p2.reserve(1, 2)) == 1
    assert p2.session_cursor(1) == 18


def test_reserve_errors():
    p = kv.Pager(small(8))
    p.create_session(1)
    assert code(p.reserve, 1, 8 * 16 + 1) == "OutOfPages"
    assert p.stats().free_pages == 8  # fail-fast, no partial allocation
    p.reserve(1, 8)
    p.trim_eos(1)
    assert code(p.reserve, 1, 1) == "SessionClosed"


def test_shadow_isolation_epochs_and_retry():
    p = kv.Pager(small())
    p.create_session(1)
    p.reserve(1, 16)
    v = p.active_view(1)
    assert v["entries"] == [] and v["epoch"] == 0
    e = p.frame_commit(1, 0)
    assert p.frame_commit(1, 0) == e  # stale retry
    assert code(p.frame_commit, 1, 5) == "FutureDelta"
    v = p.active_view(1)
    assert len(v["entries"]) == 1 and v["live_tokens"] == 16
    assert p.frame_commit(1, 1) == e + 1  # empty frame still advances


def test_apply_frame_idempotent():
    p = kv.Pager(small())
    p.create_session(1)
    e1 = p.apply_frame(1, 0, reserves=[20])
    free = p.stats().free_pages
    assert p.apply_frame(1, 0, reserves=[20]) == e1
    assert p.stats().free_pages == free and p.active_view(1)["live_tokens"] == 20


def test_alias_and_copy_on_write():
    p = kv.Pager(small())
    p.create_session(1)
    p.create_session(2)
    blocks = [b for b, _ in p.reserve(1, 48)]
    data = payload(48, 1)
    p.write_tokens(1, 0, 48, data)
    p.frame_commit(1, 0)
    assert p.alias(2, 1, 40) == 3
    p.reserve(2, 8)
    p.frame_commit(2, 0)
    free = p.stats().free_pages
    p.write_tokens(2, 41, 42, payload(1, 2))
    p.frame_commit(2, 1)
    assert p.stats().free_pages == free - 1  # exactly one page copied
    v2 = p.active_view(2)
    owner = {t: b for t0, t1, b, _ in v2["entries"] for t in range(t0, t1)}
    assert owner[0] == blocks[0] and owner[16] == blocks[1] and owner[41] != blocks[2]
    assert p.block_refcount(blocks[2]) == 1
    assert p.reconstruct_view(1) == data
    assert code(p.alias, 2, 2, 4) == "BadConfig"


def test_alias_preconditions():
    p = kv.Pager(small())
    for s in (1, 2):
        p.create_session(s)
    p.reserve(1, 16)
    p.frame_commit(1, 0)
    assert code(p.alias, 2, 1, 17) == "PrefixOutOfRange"
    p.alias(2, 1, 16)
    assert code(p.alias, 2, 1, 16) == "AliasOverlap"


def test_trim_semantics():
    p = kv.Pager(small())
    p.create_session(1)
    p.reserve(1, 32)
    p.frame_commit(1, 0)
    assert p.stats().free_pages == 62
    assert p.trim_eos(1) == 2
    assert p.stats().free_pages == 62  # deferred to the commit
    p.frame_commit(1, 1)
    assert p.stats().free_pages == 64 and p.session_eos(1)
    q = kv.Pager(small())
    q.create_session(1)
    q.reserve(1, 8)
    assert code(q.trim, 1, [(4, 20)]) == "UnmappedRange"
    assert code(q.write_tokens, 1, 8, 9, payload(1, 0)) == "UnmappedRange"


def test_bounded_commit_work_and_coalescing():
    p = kv.Pager(small(4096))
    p.create_session(1)
    p.reserve(1, 2048)
    p.frame_commit(1, 0)
    p.reserve(1, 16)
    p.frame_commit(1, 1)
    assert p.touched_in_last_commit(1) <= 4
    p.trim(1, [(0, 16)])
    p.frame_commit(1, 2)
    assert p.touched_in_last_commit(1) <= 6
    q = kv.Pager(small(64))
    q.create_session(1)
    q.reserve(1, 64 * 16)
    q.frame_commit(1, 0)
    q.trim(1, [(8 * 16, 24 * 16)])
    q.frame_commit(1, 1)
    assert q.free_runs() == [(8, 16)]
    q.create_session(2)
    bl = [b for b, _ in q.reserve(2, 9 * 16)]
    assert bl == list(range(bl[0], bl[0] + 9))


def snapshot(p, sessions, pages):
    return {
        "stats": p.stats().astuple(), "counters": p.counters().astuple(),
        "runs": p.free_runs(), "refc": [p.block_refcount(b) for b in range(pages)],
        "views": {s: p.active_view(s) for s in sessions},
        "cursor": {s: p.session_cursor(s) for s in sessions},
        "next": {s: p.next_step(s) for s in sessions},
        "bytes": {s: p.reconstruct_view(s) for s in sessions},
    }


def random_stream(seed, a, b, pages=48, n_sess=3, ops=60):
    rng = random.Random(seed)
    cfg = small(pages)
    tb = cfg.token_bytes()
    for p in (a, b):
        for s in range(n_sess):
            p.create_session(s)
    nxt = [0] * n_sess
    for _ in range(ops):
        s = rng.randrange(n_sess)
        kind = rng.randrange(11)
        if kind < 3:
            call = ("reserve", (s, rng.randrange(40)))
        elif kind < 4:
            call = ("alias", (s, rng.randrange(n_sess), rng.randrange(1, 40)))
        elif kind < 7:
            cur = a.session_cursor(s)
            lo = rng.randrange(max(1, cur + 2))
            n = rng.randint(1, 20)
            call = ("write_tokens", (s, lo, lo + n, payload(n, rng.randrange(256), tb)))
        elif kind < 8:
            v = a.active_view(s)["entries"]
            if v:
                t0, t1, _, _ = v[rng.randrange(len(v))]
                lo = rng.randint(t0, t1 - 1)
                call = ("trim", (s, [(lo, rng.randint(lo + 1, t1))]))
            else:
                call = ("trim", (s, [(0, 1)]))
        elif kind < 9:
            call = ("trim_eos", (s,))
        elif kind < 10:
            call = ("reserve_range", (s, (1 << 40) + rng.randrange(8) * 16,
                                      (1 << 40) + rng.randrange(8) * 16 + rng.randint(1, 20)))
        else:
            call = ("frame_commit", (s, nxt[s] + rng.choice([0, 0, 0, -1, 1])))
        outs = []
        for p in (a, b):
            try:
                outs.append(("ok", getattr(p, call[0])(*call[1])))
            except kv.KvrailError as e:
                outs.append(("err", e.code))
        assert outs[0] == outs[1], f"seed {seed}: {call[0]}{call[1][:3]} -> {outs}"
        if call[0] == "frame_commit" and outs[0][0] == "ok" and call[1][1] == nxt[s]:
            nxt[s] += 1
        assert snapshot(a, range(n_sess), pages) == snapshot(b, range(n_sess), pages), seed


@pytest.mark.parametrize("seed", range(60))
def test_random_verb_streams_match_reference_pager(seed, ref_api):
    a = kv.Pager(small(48))
    b = kv.Pager(small(48), api_=ref_api)
    random_stream(seed, a, b)


def test_threads_drive_distinct_sessions_concurrently():
    import threading
    p = kv.Pager(small(4096))
    for s in range(4):
        p.create_session(s)
    errs = []

    def worker(s):
        try:
            for step in range(200):
                p.reserve(s, 16)
                p.write_tokens(s, step * 16, step * 16 + 16, payload(16, s))
                p.frame_commit(s, step)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=worker, args=(s,)) for s in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs
    st = p.stats()
    assert st.free_pages == 4096 - 800 and st.live_pages == 800
    for s in range(4):
        assert p.active_view(s)["live_tokens"] == 3200
