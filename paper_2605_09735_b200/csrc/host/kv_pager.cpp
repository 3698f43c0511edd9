// kvrail-b200 pager: host metadata for the device-resident KV arena.
//
// Behavioural contract: the reference Pager (pager.cpp:101-984). Observable
// results — block ids handed out, view entries, refcounts, free runs, epochs,
// work counters, error codes — are bit-exact with it (tests/test_pager_parity.py
// drives both with the same random verb streams). The representation is new:
//   * each view buffer is a flat vector of entries sorted by first token plus a
//     per-block entry count (no tree maps), because decode-time edits are
//     appends at the cursor and whole-view EOS drops;
//   * the block table is structure-of-arrays (refcount, free flag, run links);
//   * payload bytes live behind a PayloadStore (host pages or the B200 arena),
//     and each commit reports its resolved view delta so a device mirror of
//     the committed page table can be kept without a host round trip.
#include <algorithm>
#include <array>
#include <cassert>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <shared_mutex>
#include <unordered_map>

#include "kvrail/pager.hpp"

namespace kvrail {

namespace {
constexpr uint32_t kNone = 0xffffffffu;
bool pow2(uint64_t v) { return v && !(v & (v - 1)); }
int run_class(uint32_t len) { return len >= 8 ? 3 : len >= 4 ? 2 : len >= 2 ? 1 : 0; }
} // namespace

void PagerConfig::validate() const {
    if (!pow2(page_bytes))
        raise(Errc::bad_config, "page_bytes must be a power of two");
    if (layers == 0 || kv_head_dim == 0 || elem_bytes == 0)
        raise(Errc::bad_config, "layers, kv_head_dim and elem_bytes must be positive");
    if (page_bytes < token_bytes())
        raise(Errc::bad_config, "page_bytes smaller than one token's K+V footprint");
    if (arena_pages == 0)
        raise(Errc::bad_config, "arena_pages must be positive");
}

const ViewEntry *ViewDescriptor::find(uint64_t token) const {
    // last entry starting at or before `token`
    size_t lo = 0, hi = entries.size();
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        if (entries[mid].tokens.begin <= token)
            lo = mid + 1;
        else
            hi = mid;
    }
    if (lo == 0)
        return nullptr;
    const ViewEntry &e = entries[lo - 1];
    return e.tokens.contains(token) ? &e : nullptr;
}

// ---------------------------------------------------------------------------

void PayloadStore::write_generated(const GeneratedWrite &) {
    raise(Errc::bad_config, "this payload store cannot generate payloads in place");
}

HostPayloadStore::HostPayloadStore(uint32_t pages, uint64_t page_bytes, uint64_t token_bytes)
    : page_bytes_(page_bytes), token_bytes_(token_bytes), pages_(pages) {}

void HostPayloadStore::on_alloc(BlockId head, uint32_t count) {
    for (uint32_t i = 0; i < count; ++i)
        pages_[head + i].reset(); // dematerialised pages read as zeros
}

void HostPayloadStore::copy_page(BlockId src, BlockId dst) {
    if (!pages_[src])
        return;
    if (!pages_[dst])
        pages_[dst] = std::make_unique<std::byte[]>(page_bytes_);
    std::memcpy(pages_[dst].get(), pages_[src].get(), page_bytes_);
}

void HostPayloadStore::write(BlockId block, uint32_t slot, uint32_t count, const std::byte *bytes) {
    auto &pg = pages_[block];
    if (!pg) {
        pg = std::make_unique<std::byte[]>(page_bytes_);
        std::memset(pg.get(), 0, page_bytes_);
    }
    std::memcpy(pg.get() + uint64_t(slot) * token_bytes_, bytes, uint64_t(count) * token_bytes_);
}

void HostPayloadStore::read(BlockId block, uint32_t slot, uint32_t count, std::byte *out) {
    const uint64_t n = uint64_t(count) * token_bytes_;
    if (!pages_[block])
        std::memset(out, 0, n);
    else
        std::memcpy(out, pages_[block].get() + uint64_t(slot) * token_bytes_, n);
}

// ---------------------------------------------------------------------------

namespace {

struct Ent {
    uint64_t b = 0, e = 0; // tokens [b, e)
    BlockId blk = kInvalidBlock;
    uint32_t slot = 0;
};

/// One of a session's two view buffers.
struct Buf {
    std::vector<Ent> ents; // ascending b, disjoint
    std::unordered_map<BlockId, uint32_t> per_block;
    uint64_t mapped = 0;
    uint64_t extent = 0;
    bool eos = false;

    // first index with b >= key
    size_t lower(uint64_t key) const {
        return std::lower_bound(ents.begin(), ents.end(), key,
                                [](const Ent &x, uint64_t k) { return x.b < k; }) -
               ents.begin();
    }
    // index of the entry containing `tok`, or npos
    size_t holder(uint64_t tok) const {
        size_t i = std::upper_bound(ents.begin(), ents.end(), tok,
                                    [](uint64_t k, const Ent &x) { return k < x.b; }) -
                   ents.begin();
        if (i == 0 || ents[i - 1].e <= tok)
            return npos;
        return i - 1;
    }
    // first entry overlapping [from, ...)
    size_t first_overlap(uint64_t from) const {
        size_t i = lower(from);
        if (i > 0 && ents[i - 1].e > from)
            --i;
        return i;
    }
    static constexpr size_t npos = ~size_t(0);
};

enum class Kind : uint8_t { add, drop, remap, grow_tail, mark_eos };

/// A staged edit, journaled so the commit can replay it on the other buffer.
struct Edit {
    Kind kind = Kind::add;
    Ent ent;                    // add
    uint64_t lo = 0, hi = 0;    // drop / remap range
    BlockId to = kInvalidBlock; // remap target block
    uint32_t to_slot = 0;       // remap: slot of `lo` in the target
    uint64_t key = 0;           // grow_tail: entry begin
    uint64_t new_end = 0;       // grow_tail
};

using RefDelta = std::map<BlockId, int>; // ordered: settles ascending block id

struct Sess {
    SessionId id = 0;
    std::array<Buf, 2> buf;
    int live = 0; // index of the committed buffer
    uint64_t epoch = 0;
    Step next = 0;
    uint64_t cursor = 0;
    uint64_t committed_tokens = 0;
    std::vector<Edit> journal;
    std::unordered_map<BlockId, uint32_t> uses; // entry refs over both buffers
    std::vector<BlockId> pending_free;
    uint64_t last_touched = 0;
    mutable std::shared_mutex mu;

    Buf &shadow() { return buf[live ^ 1]; }
    const Buf &committed() const { return buf[live]; }
};

} // namespace

struct Pager::Impl {
    PagerConfig cfg;
    uint32_t tpp = 0;
    uint64_t tb = 0;
    std::shared_ptr<PayloadStore> store;

    // ---- arena (guarded by arena_mu) ----
    mutable std::mutex arena_mu;
    std::vector<uint32_t> refc;
    std::vector<uint8_t> is_free;
    std::vector<uint32_t> run_tail; // valid at a free run's first block
    std::vector<uint32_t> run_head; // valid at a free run's last block
    std::vector<uint32_t> link_prev, link_next;
    std::vector<uint8_t> link_cls;
    std::array<uint32_t, 4> top{kNone, kNone, kNone, kNone};
    uint64_t n_free = 0, n_live = 0, n_shared = 0, active_tokens = 0;
    WorkCounters ctr;

    mutable std::shared_mutex sess_mu;
    std::unordered_map<SessionId, std::unique_ptr<Sess>> sessions;

    Impl(PagerConfig c, std::shared_ptr<PayloadStore> s) : cfg(c) {
        cfg.validate();
        tpp = cfg.tokens_per_page();
        tb = cfg.token_bytes();
        store = s ? std::move(s)
                  : std::make_shared<HostPayloadStore>(cfg.arena_pages, cfg.page_bytes, tb);
        const uint32_t n = cfg.arena_pages;
        refc.assign(n, 0);
        is_free.assign(n, 1);
        run_tail.assign(n, kNone);
        run_head.assign(n, kNone);
        link_prev.assign(n, kNone);
        link_next.assign(n, kNone);
        link_cls.assign(n, 0);
        n_free = n;
        push_run(0, n);
    }

    // ---- free-run lists: intrusive LIFO per size class ----
    void push_run(uint32_t h, uint32_t len) {
        const uint32_t t = h + len - 1;
        const int c = run_class(len);
        run_tail[h] = t;
        run_head[t] = h;
        link_cls[h] = uint8_t(c);
        link_prev[h] = kNone;
        link_next[h] = top[c];
        if (top[c] != kNone)
            link_prev[top[c]] = h;
        top[c] = h;
    }
    void unlink(uint32_t h) {
        const int c = link_cls[h];
        if (link_prev[h] != kNone)
            link_next[link_prev[h]] = link_next[h];
        else
            top[c] = link_next[h];
        if (link_next[h] != kNone)
            link_prev[link_next[h]] = link_prev[h];
        link_prev[h] = link_next[h] = kNone;
    }
    // Allocation policy of pager.cpp:155-199: start at the class of
    // min(need, 8), search upward then downward, carve from the run head.
    std::vector<std::pair<BlockId, uint32_t>> alloc(uint32_t count) {
        std::vector<std::pair<BlockId, uint32_t>> runs;
        if (count == 0)
            return runs;
        if (n_free < count)
            raise(Errc::out_of_pages, "need " + std::to_string(count) + " pages, " +
                                          std::to_string(n_free) + " free");
        uint32_t need = count;
        uint64_t work = 0;
        while (need) {
            const int want = run_class(std::min<uint32_t>(need, 8));
            int c = -1;
            for (int k = want; k < 4 && c < 0; ++k)
                if (top[k] != kNone)
                    c = k;
            for (int k = want - 1; k >= 0 && c < 0; --k)
                if (top[k] != kNone)
                    c = k;
            assert(c >= 0);
            const uint32_t h = top[c];
            const uint32_t len = run_tail[h] - h + 1;
            unlink(h);
            const uint32_t take = std::min(len, need);
            std::fill(is_free.begin() + h, is_free.begin() + h + take, uint8_t(0));
            store->on_alloc(h, take);
            if (len > take)
                push_run(h + take, len - take);
            runs.emplace_back(h, take);
            n_free -= take;
            need -= take;
            work += 2;
        }
        ctr.reserve_alloc_steps += work;
        ctr.reserve_blocks += count;
        return runs;
    }
    void release(uint32_t b) {
        assert(!is_free[b] && refc[b] == 0);
        is_free[b] = 1;
        uint32_t h = b, t = b;
        uint64_t work = 1;
        if (b > 0 && is_free[b - 1]) {
            h = run_head[b - 1];
            unlink(h);
            ++work;
        }
        if (b + 1 < is_free.size() && is_free[b + 1]) {
            t = run_tail[b + 1];
            unlink(b + 1);
            ++work;
        }
        push_run(h, t - h + 1);
        ++n_free;
        ctr.free_list_steps += work;
    }
    void ref_up(uint32_t b) {
        assert(!is_free[b]);
        const uint32_t r = ++refc[b];
        if (r == 1)
            ++n_live;
        else if (r == 2)
            ++n_shared;
    }
    // true: the caller holds the final reference and must defer the free
    bool ref_down(uint32_t b) {
        assert(refc[b] >= 1);
        if (refc[b] == 1)
            return true;
        if (--refc[b] == 1)
            --n_shared;
        return false;
    }

    // ---- sessions ----
    Sess &get(SessionId id) const {
        std::shared_lock lk(sess_mu);
        auto it = sessions.find(id);
        if (it == sessions.end())
            raise(Errc::unknown_session, "session " + std::to_string(id));
        return *it->second;
    }

    void use_added(Sess &s, BlockId b) {
        if (s.uses[b]++ == 0) {
            std::lock_guard lk(arena_mu);
            ref_up(b);
        }
    }
    void use_removed(Sess &s, BlockId b) {
        auto it = s.uses.find(b);
        assert(it != s.uses.end() && it->second > 0);
        if (--it->second)
            return;
        s.uses.erase(it);
        bool last;
        {
            std::lock_guard lk(arena_mu);
            last = ref_down(b);
        }
        if (last)
            s.pending_free.push_back(b);
    }
    void settle(Sess &s, const RefDelta &d) {
        for (auto [b, n] : d) {
            for (; n > 0; --n)
                use_added(s, b);
            for (; n < 0; ++n)
                use_removed(s, b);
        }
    }

    // Apply one edit to buffer `which` of `s`. Reference deltas go to `acc`
    // when given (commit replay), else settle when the edit is done.
    void apply(Sess &s, int which, const Edit &ed, uint64_t &touched, RefDelta *acc = nullptr) {
        Buf &v = s.buf[which];
        RefDelta own;
        RefDelta &d = acc ? *acc : own;
        auto put = [&](size_t at, const Ent &x) {
            v.ents.insert(v.ents.begin() + at, x);
            ++v.per_block[x.blk];
            v.mapped += x.e - x.b;
            v.extent = std::max(v.extent, x.e);
            ++d[x.blk];
            ++touched;
        };
        auto take = [&](size_t at) {
            const Ent x = v.ents[at];
            auto pb = v.per_block.find(x.blk);
            if (--pb->second == 0)
                v.per_block.erase(pb);
            v.mapped -= x.e - x.b;
            --d[x.blk];
            ++touched;
            v.ents.erase(v.ents.begin() + at);
            return x;
        };
        switch (ed.kind) {
        case Kind::add: {
            const size_t at = v.lower(ed.ent.b);
            assert(at == v.ents.size() || v.ents[at].b != ed.ent.b);
            put(at, ed.ent);
            break;
        }
        case Kind::drop:
        case Kind::remap: {
            size_t i = v.first_overlap(ed.lo);
            while (i < v.ents.size() && v.ents[i].b < ed.hi) {
                const Ent x = take(i);
                if (x.b < ed.lo)
                    put(i++, Ent{x.b, ed.lo, x.blk, x.slot});
                if (ed.kind == Kind::remap) {
                    const uint64_t lo = std::max(x.b, ed.lo), hi = std::min(x.e, ed.hi);
                    put(i++, Ent{lo, hi, ed.to, ed.to_slot + uint32_t(lo - ed.lo)});
                }
                if (x.e > ed.hi)
                    put(i++, Ent{ed.hi, x.e, x.blk, x.slot + uint32_t(ed.hi - x.b)});
            }
            break;
        }
        case Kind::grow_tail: {
            const size_t at = v.lower(ed.key);
            if (at < v.ents.size() && v.ents[at].b == ed.key) {
                Ent &x = v.ents[at];
                v.mapped += ed.new_end - x.e;
                x.e = ed.new_end;
                v.extent = std::max(v.extent, ed.new_end);
                ++touched;
            }
            break;
        }
        case Kind::mark_eos:
            v.eos = true;
            ++touched;
            break;
        }
        if (!acc)
            settle(s, own);
    }
    // A drop that removes whole entries only (no left/right remnant).
    static bool clean_drop(const Buf &v, const Edit &ed) {
        const size_t i = v.first_overlap(ed.lo);
        if (i < v.ents.size() && v.ents[i].b < ed.lo)
            return false;
        const size_t j = v.lower(ed.hi);
        return j == 0 || v.ents[j - 1].e <= ed.hi;
    }

    // Apply a run of drop edits. When every one of them removes whole entries,
    // one compaction pass replaces the per-entry vector erases (identical
    // touched counts and reference deltas: an entry dies exactly once).
    void apply_drops(Sess &s, int which, const Edit *eds, size_t n, uint64_t &touched,
                     RefDelta *acc = nullptr) {
        Buf &v = s.buf[which];
        bool all_clean = true;
        for (size_t k = 0; k < n && all_clean; ++k)
            all_clean = clean_drop(v, eds[k]);
        if (!all_clean) {
            for (size_t k = 0; k < n; ++k)
                apply(s, which, eds[k], touched, acc);
            return;
        }
        // dead[i] = 1 + index of the edit that removes entry i (0: survives)
        std::vector<uint32_t> dead(v.ents.size(), 0);
        size_t n_dead = 0;
        for (size_t k = 0; k < n; ++k)
            for (size_t i = v.first_overlap(eds[k].lo); i < v.ents.size() && v.ents[i].b < eds[k].hi; ++i)
                if (!dead[i]) {
                    dead[i] = uint32_t(k + 1);
                    ++n_dead;
                }
        // Outside a commit every edit settles on its own, in edit order.
        std::vector<RefDelta> per_edit(acc ? 0 : n);
        if (n_dead) {
            size_t w = 0;
            for (size_t i = 0; i < v.ents.size(); ++i) {
                const Ent &x = v.ents[i];
                if (!dead[i]) {
                    v.ents[w++] = x;
                    continue;
                }
                auto pb = v.per_block.find(x.blk);
                if (--pb->second == 0)
                    v.per_block.erase(pb);
                v.mapped -= x.e - x.b;
                --(acc ? *acc : per_edit[dead[i] - 1])[x.blk];
                ++touched;
            }
            v.ents.resize(w);
        }
        for (const RefDelta &d : per_edit)
            settle(s, d);
    }

    void stage_edit(Sess &s, const Edit &ed) {
        uint64_t t = 0;
        if (ed.kind == Kind::drop)
            apply_drops(s, s.live ^ 1, &ed, 1, t);
        else
            apply(s, s.live ^ 1, ed, t);
        s.journal.push_back(ed);
    }

    // Blocks a trim dropped from the shadow that this session alone still
    // holds: they return to the pool at this step's commit.
    uint64_t released_by_trim(Sess &s, const std::set<BlockId> &cands) {
        const Buf &sh = s.shadow();
        uint64_t freed = 0;
        for (BlockId b : cands) {
            if (sh.per_block.count(b))
                continue;
            if (std::find(s.pending_free.begin(), s.pending_free.end(), b) !=
                s.pending_free.end()) {
                ++freed;
                continue;
            }
            if (s.uses.count(b)) {
                std::lock_guard lk(arena_mu);
                if (refc[b] == 1)
                    ++freed;
            }
        }
        return freed;
    }

    std::vector<ReservedBlock> map_fresh(Sess &s, uint64_t first_tok, uint64_t n_tok,
                                         bool move_cursor) {
        std::vector<ReservedBlock> out;
        const uint32_t pages = uint32_t((n_tok + tpp - 1) / tpp);
        std::vector<std::pair<BlockId, uint32_t>> runs;
        {
            std::lock_guard lk(arena_mu);
            runs = alloc(pages);
        }
        uint64_t pos = first_tok, left = n_tok;
        for (auto [h, len] : runs)
            for (uint32_t i = 0; i < len; ++i) {
                const uint64_t n = std::min<uint64_t>(left, tpp);
                Edit ed;
                ed.kind = Kind::add;
                ed.ent = Ent{pos, pos + n, h + i, 0};
                stage_edit(s, ed);
                pos += n;
                left -= n;
                if (move_cursor)
                    s.cursor = pos;
                out.push_back({h + i, tpp});
            }
        return out;
    }

    // Copy-on-write of a page this session shares (pager.cpp:615-647 contract).
    void cow(Sess &s, BlockId shared_blk) {
        BlockId copy;
        {
            std::lock_guard lk(arena_mu);
            copy = alloc(1)[0].first;
            store->copy_page(shared_blk, copy);
        }
        std::vector<uint64_t> keys;
        for (const Ent &x : s.shadow().ents)
            if (x.blk == shared_blk)
                keys.push_back(x.b);
        for (uint64_t k : keys) {
            const Buf &sh = s.shadow();
            const Ent x = sh.ents[sh.lower(k)];
            Edit ed;
            ed.kind = Kind::remap;
            ed.lo = x.b;
            ed.hi = x.e;
            ed.to = copy;
            ed.to_slot = x.slot;
            stage_edit(s, ed);
        }
    }

    template <typename Sink>
    void write_common(Sess &s, TokenRange r, Sink &&sink) {
        Buf &sh = s.shadow();
        for (uint64_t pos = r.begin; pos < r.end;) {
            const size_t i = sh.holder(pos);
            if (i == Buf::npos)
                raise(Errc::unmapped_range, "token " + std::to_string(pos) + " unmapped");
            pos = sh.ents[i].e;
        }
        for (;;) {
            BlockId shared_blk = kInvalidBlock;
            for (uint64_t pos = r.begin; pos < r.end;) {
                const Ent &x = sh.ents[sh.holder(pos)];
                uint32_t rc;
                {
                    std::lock_guard lk(arena_mu);
                    rc = refc[x.blk];
                }
                if (rc >= 2) {
                    shared_blk = x.blk;
                    break;
                }
                pos = x.e;
            }
            if (shared_blk == kInvalidBlock)
                break;
            cow(s, shared_blk);
        }
        for (uint64_t pos = r.begin; pos < r.end;) {
            const Ent &x = sh.ents[sh.holder(pos)];
            const uint64_t n = std::min(r.end, x.e) - pos;
            sink(x.blk, x.slot + uint32_t(pos - x.b), uint32_t(n), pos);
            pos += n;
        }
    }

    // Resolved committed mapping of [lo, hi) after a commit, as ViewEdits.
    static void resolve(const Buf &v, uint64_t lo, uint64_t hi, std::vector<ViewEdit> &out) {
        uint64_t pos = lo;
        for (size_t i = v.first_overlap(lo); i < v.ents.size() && v.ents[i].b < hi; ++i) {
            const Ent &x = v.ents[i];
            const uint64_t a = std::max(x.b, lo), z = std::min(x.e, hi);
            if (a > pos)
                out.push_back({pos, a, kInvalidBlock, 0});
            out.push_back({a, z, x.blk, x.slot + uint32_t(a - x.b)});
            pos = z;
        }
        if (pos < hi)
            out.push_back({pos, hi, kInvalidBlock, 0});
    }

    uint64_t commit(Sess &s, Step step) {
        if (step < s.next)
            return s.epoch;
        if (step > s.next)
            raise(Errc::future_delta, "step " + std::to_string(step) + " skips ahead of " +
                                          std::to_string(s.next));
        uint64_t touched = 0;
        s.live ^= 1;
        ++s.epoch;
        std::vector<std::pair<uint64_t, uint64_t>> spans;
        RefDelta d;
        for (size_t i = 0; i < s.journal.size();) {
            size_t j = i;
            while (j < s.journal.size() && s.journal[j].kind == Kind::drop)
                ++j;
            if (j > i) { // a run of drops replays as one pass
                apply_drops(s, s.live ^ 1, s.journal.data() + i, j - i, touched, &d);
                for (; i < j; ++i)
                    spans.emplace_back(s.journal[i].lo, s.journal[i].hi);
                continue;
            }
            const Edit &ed = s.journal[i++];
            apply(s, s.live ^ 1, ed, touched, &d);
            switch (ed.kind) {
            case Kind::add: spans.emplace_back(ed.ent.b, ed.ent.e); break;
            case Kind::drop:
            case Kind::remap: spans.emplace_back(ed.lo, ed.hi); break;
            case Kind::grow_tail: spans.emplace_back(ed.key, ed.new_end); break;
            case Kind::mark_eos: break;
            }
        }
        s.journal.clear();
        settle(s, d);
        for (BlockId b : s.pending_free) {
            std::lock_guard lk(arena_mu);
            assert(refc[b] == 1);
            refc[b] = 0;
            --n_live;
            release(b);
            ++touched;
        }
        s.pending_free.clear();
        const uint64_t now_mapped = s.committed().mapped;
        {
            std::lock_guard lk(arena_mu);
            active_tokens += now_mapped - s.committed_tokens;
            ++ctr.commits;
            ctr.commit_entries_touched += touched;
        }
        s.committed_tokens = now_mapped;
        s.next = step + 1;
        s.last_touched = touched;

        // Report the committed delta (merged touched ranges, final mapping).
        std::sort(spans.begin(), spans.end());
        std::vector<ViewEdit> edits;
        for (size_t i = 0; i < spans.size();) {
            uint64_t lo = spans[i].first, hi = spans[i].second;
            size_t j = i + 1;
            while (j < spans.size() && spans[j].first <= hi)
                hi = std::max(hi, spans[j++].second);
            if (hi > lo)
                resolve(s.committed(), lo, hi, edits);
            i = j;
        }
        store->on_commit(s.id, s.committed().eos, edits);
        return s.epoch;
    }
};

// ---------------------------------------------------------------------------
// public surface

Pager::Pager(PagerConfig cfg) : impl_(std::make_unique<Impl>(cfg, nullptr)) {}
Pager::Pager(PagerConfig cfg, std::shared_ptr<PayloadStore> store)
    : impl_(std::make_unique<Impl>(cfg, std::move(store))) {}
Pager::~Pager() = default;

const PagerConfig &Pager::config() const { return impl_->cfg; }
PayloadStore &Pager::store() const { return *impl_->store; }

void Pager::create_session(SessionId id) {
    std::unique_lock lk(impl_->sess_mu);
    auto [it, fresh] = impl_->sessions.try_emplace(id);
    if (!fresh)
        raise(Errc::bad_config, "session " + std::to_string(id) + " already exists");
    it->second = std::make_unique<Sess>();
    it->second->id = id;
}

bool Pager::has_session(SessionId id) const {
    std::shared_lock lk(impl_->sess_mu);
    return impl_->sessions.count(id) != 0;
}

std::vector<SessionId> Pager::session_ids() const {
    std::shared_lock lk(impl_->sess_mu);
    std::vector<SessionId> ids;
    for (auto &kv : impl_->sessions)
        ids.push_back(kv.first);
    std::sort(ids.begin(), ids.end());
    return ids;
}

std::vector<ReservedBlock> Pager::reserve(SessionId session, uint64_t token_count) {
    Impl &m = *impl_;
    Sess &s = m.get(session);
    std::unique_lock lk(s.mu);
    Buf &sh = s.shadow();
    if (sh.eos)
        raise(Errc::session_closed, "reserve on EOS session " + std::to_string(s.id));
    {
        std::lock_guard al(m.arena_mu);
        ++m.ctr.reserve_calls;
    }
    if (token_count == 0)
        return {};
    uint64_t left = token_count;
    // Spare slots at the end of the block holding the cursor come first.
    if (s.cursor > 0) {
        const size_t at = sh.lower(s.cursor);
        if (at > 0 && sh.ents[at - 1].e == s.cursor) {
            const Ent &tail = sh.ents[at - 1];
            const uint32_t used = tail.slot + uint32_t(tail.e - tail.b);
            if (used < m.tpp) {
                const uint64_t grow = std::min<uint64_t>(m.tpp - used, left);
                Edit ed;
                ed.kind = Kind::grow_tail;
                ed.key = tail.b;
                ed.new_end = tail.e + grow;
                m.stage_edit(s, ed);
                s.cursor += grow;
                left -= grow;
            }
        }
    }
    if (left == 0)
        return {};
    return m.map_fresh(s, s.cursor, left, true);
}

std::vector<ReservedBlock> Pager::reserve_range(SessionId session, TokenRange range) {
    Impl &m = *impl_;
    Sess &s = m.get(session);
    std::unique_lock lk(s.mu);
    Buf &sh = s.shadow();
    if (sh.eos)
        raise(Errc::session_closed, "reserve on EOS session " + std::to_string(s.id));
    if (range.empty())
        return {};
    const size_t at = sh.lower(range.begin);
    if ((at > 0 && sh.ents[at - 1].e > range.begin) ||
        (at < sh.ents.size() && sh.ents[at].b < range.end))
        raise(Errc::alias_overlap, "range already mapped");
    {
        std::lock_guard al(m.arena_mu);
        ++m.ctr.reserve_calls;
    }
    return m.map_fresh(s, range.begin, range.size(), false);
}

uint64_t Pager::alias(SessionId dst, SessionId src, uint64_t prefix_tokens) {
    Impl &m = *impl_;
    if (dst == src)
        raise(Errc::bad_config, "alias onto the same session");
    Sess &d = m.get(dst);
    Sess &from = m.get(src);
    Sess *lo = d.id < from.id ? &d : &from;
    Sess *hi = d.id < from.id ? &from : &d;
    std::unique_lock l1(lo->mu);
    std::unique_lock l2(hi->mu);
    if (d.shadow().eos)
        raise(Errc::session_closed, "alias into EOS session");
    if (prefix_tokens == 0)
        return 0;
    // The source's committed view must cover [0, prefix) without gaps.
    std::vector<Ent> pieces;
    uint64_t covered = 0;
    for (const Ent &x : from.committed().ents) {
        if (x.b != covered || covered >= prefix_tokens)
            break;
        Ent p = x;
        p.e = std::min(p.e, prefix_tokens);
        pieces.push_back(p);
        covered = p.e;
    }
    if (covered < prefix_tokens)
        raise(Errc::prefix_out_of_range, "source maps " + std::to_string(covered) + " of " +
                                             std::to_string(prefix_tokens) + " prefix tokens");
    const Buf &dsh = d.shadow();
    if (!dsh.ents.empty() && dsh.ents.front().b < prefix_tokens)
        raise(Errc::alias_overlap, "destination already maps part of the prefix");
    std::set<BlockId> shared;
    for (const Ent &p : pieces) {
        Edit ed;
        ed.kind = Kind::add;
        ed.ent = p;
        m.stage_edit(d, ed);
        shared.insert(p.blk);
    }
    d.cursor = std::max(d.cursor, prefix_tokens);
    return shared.size();
}

void Pager::write_tokens(SessionId session, TokenRange range, std::span<const std::byte> payload) {
    Impl &m = *impl_;
    Sess &s = m.get(session);
    std::unique_lock lk(s.mu);
    if (range.empty())
        return;
    if (payload.size() != range.size() * m.tb)
        raise(Errc::dimension_mismatch, "payload bytes do not match token range");
    m.write_common(s, range, [&](BlockId b, uint32_t slot, uint32_t n, uint64_t tok) {
        m.store->write(b, slot, n, payload.data() + (tok - range.begin) * m.tb);
    });
}

void Pager::write_tokens_generated(SessionId session, TokenRange range, uint32_t source,
                                   uint64_t aux, std::span<const uint32_t> src_slots) {
    Impl &m = *impl_;
    Sess &s = m.get(session);
    std::unique_lock lk(s.mu);
    if (range.empty())
        return;
    m.write_common(s, range, [&](BlockId b, uint32_t slot, uint32_t n, uint64_t tok) {
        GeneratedWrite w;
        w.session = session;
        w.token = tok;
        w.block = b;
        w.slot = slot;
        w.count = n;
        w.source = source;
        w.aux = aux;
        w.src_slots = src_slots;
        m.store->write_generated(w);
    });
}

uint64_t Pager::trim(SessionId session, std::span<const TokenRange> ranges) {
    Impl &m = *impl_;
    Sess &s = m.get(session);
    std::unique_lock lk(s.mu);
    const Buf &sh = s.shadow();
    std::set<BlockId> cands;
    for (const TokenRange &r : ranges) {
        for (uint64_t pos = r.begin; pos < r.end;) {
            const size_t i = sh.holder(pos);
            if (i == Buf::npos)
                raise(Errc::unmapped_range, "trim range not mapped");
            cands.insert(sh.ents[i].blk);
            pos = sh.ents[i].e;
        }
    }
    std::vector<Edit> drops;
    for (const TokenRange &r : ranges) {
        if (r.empty())
            continue;
        Edit ed;
        ed.kind = Kind::drop;
        ed.lo = r.begin;
        ed.hi = r.end;
        drops.push_back(ed);
    }
    uint64_t touched = 0;
    m.apply_drops(s, s.live ^ 1, drops.data(), drops.size(), touched);
    s.journal.insert(s.journal.end(), drops.begin(), drops.end());
    const uint64_t freed = m.released_by_trim(s, cands);
    std::lock_guard al(m.arena_mu);
    ++m.ctr.trim_calls;
    m.ctr.trim_blocks += freed;
    return freed;
}

uint64_t Pager::trim_eos(SessionId session) {
    Impl &m = *impl_;
    Sess &s = m.get(session);
    std::unique_lock lk(s.mu);
    std::set<BlockId> cands;
    for (auto &kv : s.shadow().per_block)
        cands.insert(kv.first);
    if (!s.shadow().ents.empty()) {
        Edit ed;
        ed.kind = Kind::drop;
        ed.lo = 0;
        ed.hi = s.shadow().extent;
        m.stage_edit(s, ed);
    }
    Edit eos;
    eos.kind = Kind::mark_eos;
    m.stage_edit(s, eos);
    const uint64_t freed = m.released_by_trim(s, cands);
    std::lock_guard al(m.arena_mu);
    ++m.ctr.trim_calls;
    m.ctr.trim_blocks += freed;
    return freed;
}

uint64_t Pager::frame_commit(SessionId session, Step step) {
    Sess &s = impl_->get(session);
    std::unique_lock lk(s.mu);
    return impl_->commit(s, step);
}

uint64_t Pager::apply_frame(const FrameDelta &delta) {
    {
        Sess &s = impl_->get(delta.session);
        std::shared_lock lk(s.mu);
        if (delta.step < s.next)
            return s.epoch;
        if (delta.step > s.next)
            raise(Errc::future_delta, "frame " + std::to_string(delta.step) + " skips ahead");
    }
    for (const auto &a : delta.aliases)
        alias(delta.session, a.src, a.prefix_tokens);
    for (uint64_t n : delta.reserves)
        reserve(delta.session, n);
    if (!delta.trims.empty())
        trim(delta.session, delta.trims);
    if (delta.trim_eos)
        trim_eos(delta.session);
    return frame_commit(delta.session, delta.step);
}

ViewDescriptor Pager::active_view(SessionId session) const {
    const Sess &s = impl_->get(session);
    std::shared_lock lk(s.mu);
    const Buf &v = s.committed();
    ViewDescriptor out;
    out.session = s.id;
    out.epoch = s.epoch;
    out.live_tokens = v.mapped;
    out.extent = v.extent;
    out.eos = v.eos;
    out.entries.reserve(v.ents.size());
    for (const Ent &x : v.ents)
        out.entries.push_back({{x.b, x.e}, x.blk, x.slot});
    return out;
}

bool Pager::session_eos(SessionId session) const {
    const Sess &s = impl_->get(session);
    std::shared_lock lk(s.mu);
    return s.committed().eos;
}

uint64_t Pager::session_cursor(SessionId session) const {
    const Sess &s = impl_->get(session);
    std::shared_lock lk(s.mu);
    return s.cursor;
}

Step Pager::next_step(SessionId session) const {
    const Sess &s = impl_->get(session);
    std::shared_lock lk(s.mu);
    return s.next;
}

uint64_t Pager::touched_in_last_commit(SessionId session) const {
    const Sess &s = impl_->get(session);
    std::shared_lock lk(s.mu);
    return s.last_touched;
}

ArenaStats Pager::stats() const {
    const Impl &m = *impl_;
    std::lock_guard lk(m.arena_mu);
    ArenaStats st;
    st.free_pages = m.n_free;
    st.live_pages = m.n_live;
    st.shared_pages = m.n_shared;
    st.reserved_bytes = (m.cfg.arena_pages - m.n_free) * m.cfg.page_bytes;
    st.active_bytes = m.active_tokens * m.tb;
    return st;
}

WorkCounters Pager::counters() const {
    std::lock_guard lk(impl_->arena_mu);
    return impl_->ctr;
}

void Pager::read_slots(BlockId block, uint32_t slot_begin, uint32_t slot_count,
                       std::byte *out) const {
    if (block >= impl_->cfg.arena_pages)
        raise(Errc::unmapped_block, "block " + std::to_string(block) + " outside the arena");
    impl_->store->read(block, slot_begin, slot_count, out);
}

std::vector<std::pair<BlockId, uint32_t>> Pager::free_runs() const {
    const Impl &m = *impl_;
    std::lock_guard lk(m.arena_mu);
    std::vector<std::pair<BlockId, uint32_t>> runs;
    const uint32_t n = m.cfg.arena_pages;
    for (uint32_t b = 0; b < n;) {
        if (!m.is_free[b]) {
            ++b;
            continue;
        }
        uint32_t e = b;
        while (e < n && m.is_free[e])
            ++e;
        runs.emplace_back(b, e - b);
        b = e;
    }
    return runs;
}

uint32_t Pager::block_refcount(BlockId block) const {
    std::lock_guard lk(impl_->arena_mu);
    return impl_->refc.at(block);
}

} // namespace kvrail
