// kvrail-b200 DeviceStep: seals a step's host decisions into ONE committed
// descriptor and publishes it to the B200 (kvr_cuda.h).
//
// The Pager reports byte events through the PayloadStore interface; this file
// turns them into descriptor sections:
//   on_alloc   -> zero ops, only for recycled (dirty) pages and only for the
//                 slots this step does not overwrite anyway;
//   copy_page  -> COW ops;  write -> host blob ops;  write_generated -> write
//                 ops (token payloads, far summaries);
//   on_commit  -> page-table edits for sessions bound to a device slot.
// Within one descriptor the device runs {zero | cow | blob} (one kernel, no order
// among them) -> write -> far -> map -> prime -> gather -> attn (queries and K-scan
// on a parallel branch). Sequences whose result depends on an order the descriptor
// does not give (a page written or zeroed and then COW-copied, a blob into a copy's
// destination, a slot written twice, ...) are split: the earlier part is flushed
// as an apply-only descriptor first.
#include <algorithm>
#include <cstring>
#include <deque>
#include <stdexcept>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "kvrail/device_step.hpp"

namespace kvrail {

namespace {

void ck(int rc) {
    if (rc != KVR_OK)
        throw std::runtime_error(std::string("CUDA/device failure: ") + kvr_dev_last_error());
}

constexpr uint64_t align16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

} // namespace

struct DeviceStep::Impl {
    kvr_geometry g{};
    kvr_dev *dev = nullptr;
    std::shared_ptr<PayloadStore> store_;

    // pending byte ops (current wave)
    std::unordered_map<BlockId, std::vector<uint8_t>> zero_pages; // page -> slot written this wave
    std::vector<BlockId> zero_order;
    std::vector<kvr_cow_op> cows;
    std::vector<kvr_edit_op> edits;
    std::vector<kvr_write_op> writes, far_jobs;
    std::vector<kvr_blob_op> blob_ops;
    std::vector<uint8_t> blob;
    std::unordered_map<BlockId, std::vector<uint8_t>> wave_slots; // slots written this wave
    std::unordered_set<BlockId> wave_cow_dst;
    // step inputs
    std::vector<kvr_need_rec> needs;
    std::vector<kvr_span_rec> spans;
    std::vector<kvr_prime_op> primes;
    std::vector<uint32_t> src_rows; // chunk rows of far jobs / source rows of primes (this wave)
    std::unordered_set<SessionId> prime_src; // sessions whose rows K-prime copies this step
    std::vector<uint32_t> far_ids;
    std::vector<kvr_slot_state> slots;
    std::vector<uint64_t> staged_count; // per slot: near staged tokens this step
    uint32_t ring_plane_rows = 0;       // kvr_dev_ring_plane_rows
    std::vector<std::vector<uint64_t>> far_shown; // per slot, as of the last launch
    // K-presum: chunks summarised while their prompt rows were written (far view)
    std::vector<kvr_presum_op> presum_ops;
    std::vector<kvr_presum_run> presum_runs;
    std::unordered_set<uint64_t> presummed; // session << 32 | chunk, stash row valid
    static uint64_t presum_key(SessionId s, uint64_t chunk) { return uint64_t(s) << 32 | chunk; }

    /// Move whole far-view chunks out of this step's cold writes into K-presum ops:
    /// a chunk qualifies when its chunk_tokens rows are all cold rows of one bound
    /// session written this step (a prompt), so K-presum can generate and sum them.
    void extract_presums(std::vector<kvr_write_op> &cold) {
        presum_ops.clear();
        presum_runs.clear();
        if (!g.far_cap || !g.chunk_tokens || cold.empty())
            return;
        const uint64_t ct = g.chunk_tokens;
        std::vector<size_t> idx(cold.size());
        for (size_t i = 0; i < idx.size(); ++i)
            idx[i] = i;
        std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
            return cold[a].session != cold[b].session ? cold[a].session < cold[b].session
                                                      : cold[a].token < cold[b].token;
        });
        std::vector<kvr_write_op> keep;
        // pieces of the current chunk (all from one session, contiguous tokens)
        std::vector<kvr_write_op> cur;
        uint64_t cur_chunk = ~0ull, cur_next = 0;
        SessionId cur_sess = 0;
        auto flush_chunk = [&]() {
            uint64_t n = 0;
            for (const kvr_write_op &w : cur)
                n += w.count;
            if (n == ct && cur.front().dev_slot != KVR_NO_SLOT && cur.front().token == cur_chunk * ct) {
                kvr_presum_op op{};
                op.session = cur_sess;
                op.dev_slot = cur.front().dev_slot;
                op.chunk = uint32_t(cur_chunk);
                op.run_begin = uint32_t(presum_runs.size());
                op.run_count = uint32_t(cur.size());
                for (const kvr_write_op &w : cur)
                    presum_runs.push_back({w.token, w.block, w.slot, w.count, 0});
                presum_ops.push_back(op);
                presummed.insert(presum_key(cur_sess, cur_chunk));
            } else {
                keep.insert(keep.end(), cur.begin(), cur.end());
            }
            cur.clear();
            cur_chunk = ~0ull;
        };
        for (size_t i : idx) {
            kvr_write_op w = cold[i];
            if (w.source != 0 || w.dev_slot == KVR_NO_SLOT || w.dev_slot >= g.n_slots) {
                keep.push_back(w);
                continue;
            }
            while (w.count) { // split at chunk boundaries
                const uint64_t c = w.token / ct;
                const uint32_t n = uint32_t(std::min<uint64_t>(w.count, (c + 1) * ct - w.token));
                kvr_write_op piece = w;
                piece.count = n;
                if (c != cur_chunk || w.session != cur_sess || w.token != cur_next) {
                    if (!cur.empty())
                        flush_chunk();
                    cur_chunk = c;
                    cur_sess = w.session;
                }
                cur.push_back(piece);
                cur_next = w.token + n;
                w.token += n;
                w.slot += n;
                w.count -= n;
            }
        }
        if (!cur.empty())
            flush_chunk();
        cold.swap(keep);
    }
    /// Cold prefill rows not yet written (prefill budget). Lookups by page and by
    /// session are O(1); removed entries are marked dead (count 0) and skipped.
    struct Deferred {
        std::deque<kvr_write_op> q;
        std::vector<uint32_t> per_block;
        std::unordered_map<SessionId, uint32_t> per_session;
        uint64_t tokens = 0;
        uint64_t dropped = 0; // rows whose page was recycled before anything read them
        bool has_block(BlockId b) const { return b < per_block.size() && per_block[b] != 0; }
        bool has_session(SessionId s) const { return per_session.count(s) != 0; }
        void push(const kvr_write_op &w) {
            if (per_block.size() <= w.block)
                per_block.resize(size_t(w.block) + 1, 0);
            q.push_back(w);
            ++per_block[w.block];
            ++per_session[w.session];
            tokens += w.count;
        }
        void kill(kvr_write_op &w) {
            --per_block[w.block];
            if (--per_session[w.session] == 0)
                per_session.erase(w.session);
            tokens -= w.count;
            w.count = 0;
        }
        void trim_front() {
            while (!q.empty() && q.front().count == 0)
                q.pop_front();
        }
        /// Remove every live entry matching `pred`, handing it to `fn` first.
        template <class Pred, class Fn> bool extract(Pred pred, Fn fn) {
            bool any = false;
            for (kvr_write_op &w : q)
                if (w.count && pred(w)) {
                    fn(w);
                    kill(w);
                    any = true;
                }
            trim_front();
            return any;
        }
        /// Up to `budget` tokens from the front (the last op taken may be split).
        void take(uint64_t budget, std::vector<kvr_write_op> &out) {
            while (budget && !q.empty()) {
                kvr_write_op &w = q.front();
                if (w.count == 0) {
                    q.pop_front();
                    continue;
                }
                if (w.count <= budget) {
                    budget -= w.count;
                    out.push_back(w);
                    kill(w);
                    q.pop_front();
                } else {
                    kvr_write_op x = w;
                    x.count = uint32_t(budget);
                    out.push_back(x);
                    w.token += budget;
                    w.slot += uint32_t(budget);
                    w.count -= uint32_t(budget);
                    tokens -= budget;
                    budget = 0;
                }
            }
        }
    } deferred;
    uint64_t prefill_budget = 0;                  // tokens per step; 0 = no deferral
    // state
    std::vector<uint8_t> clean; // page known to be all zeros on the device
    std::unordered_map<SessionId, uint32_t> bound;
    DeviceStepStats done[2];
    bool have_done[2] = {false, false};
    uint64_t launched_step[2] = {~0ull, ~0ull};
    std::vector<kvr_slot_state> launched_slots[2]; // slot states of the step in each ring slot
    uint64_t attn_bytes_pending[2] = {0, 0};
    int64_t step_counts[KVR_COUNTS] = {};
    uint64_t desc_bytes_pending[2] = {0, 0};

    bool pending() const {
        return !zero_order.empty() || !cows.empty() || !edits.empty() || !writes.empty() ||
               !far_jobs.empty() || !blob_ops.empty() || !primes.empty();
    }

    // ---- descriptor packing ----
    uint64_t pack(void *dst, uint64_t step, double now, const TransportConfig *tc, bool with_step) {
        // zero ops: unwritten slot runs of recycled pages
        std::vector<kvr_zero_op> zeros;
        for (BlockId p : zero_order) {
            auto it = zero_pages.find(p);
            if (it == zero_pages.end())
                continue;
            const std::vector<uint8_t> &w = it->second;
            for (uint32_t s = 0; s < g.tokens_per_page;) {
                if (w[s]) {
                    ++s;
                    continue;
                }
                uint32_t e = s;
                while (e < g.tokens_per_page && !w[e])
                    ++e;
                zeros.push_back({p, s, e - s, 0});
                s = e;
            }
            // a page's slack beyond tpp * token_bytes is never addressed
        }
        kvr_step_header h{};
        h.step = step;
        h.now = now;
        if (tc) {
            h.tau = tc->merge_threshold;
            h.max_hold = tc->max_hold;
            h.merge = tc->merge ? 1 : 0;
            h.run_page = tc->run_page_bytes;
            h.run_span = tc->run_span_bytes;
        }
        uint64_t off = align16(sizeof(kvr_step_header));
        auto place = [&](uint64_t bytes) {
            const uint64_t at = off;
            off = align16(off + bytes);
            return at;
        };
        // Hot writes produce rows this step's kernels read (a live window row or a
        // staged block); the rest (older prompt rows) are cold and run on a graph
        // branch overlapping the attention.
        std::vector<kvr_write_op> hot, cold;
        std::unordered_set<BlockId> staged;
        for (const kvr_span_rec &s : spans)
            staged.insert(s.block);
        // Rows read before the cold phase: staged blocks (K-gather) and chunks a
        // far job summarises (K-far), matched by session and token range.
        auto read_early = [&](const kvr_write_op &w) {
            if (staged.count(w.block) || prime_src.count(w.session))
                return true;
            for (const kvr_write_op &f : far_jobs)
                if (f.session == w.session && w.token < f.aux + g.chunk_tokens && f.aux < w.token + w.count)
                    return true;
            return false;
        };
        if (with_step) {
            for (const kvr_write_op &w : writes) {
                // Unbound sessions (the shared-prefix template) are read by K-prime
                // of sessions that alias them this very step: always hot.
                if (w.dev_slot == KVR_NO_SLOT || read_early(w)) {
                    hot.push_back(w);
                    continue;
                }
                const uint64_t wr = slots[w.dev_slot].written;
                const uint64_t lo = std::max<uint64_t>(w.token, wr > g.near_window ? wr - g.near_window : 0);
                const uint64_t hi = std::min<uint64_t>(w.token + w.count, wr);
                if (lo >= hi) {
                    cold.push_back(w);
                    continue;
                }
                auto piece = [&](uint64_t a, uint64_t b, std::vector<kvr_write_op> &to) {
                    if (a >= b)
                        return;
                    kvr_write_op x = w;
                    x.token = a;
                    x.slot = w.slot + uint32_t(a - w.token);
                    x.count = uint32_t(b - a);
                    to.push_back(x);
                };
                piece(w.token, lo, cold);
                piece(lo, hi, hot);
                piece(hi, w.token + w.count, cold);
            }
        } else {
            hot = writes;
        }
        if (with_step)
            extract_presums(cold);
        else {
            presum_ops.clear();
            presum_runs.clear();
        }
        if (with_step && prefill_budget) {
            // Prefill budget: cold rows join the deferred queue, which drains at
            // most `prefill_budget` tokens per step; queued rows read this step
            // are forced out with the hot writes (scanned only when a staged page
            // or a far job's session has queued rows).
            bool scan = false;
            for (BlockId b : staged)
                scan |= deferred.has_block(b);
            for (const kvr_write_op &f : far_jobs)
                scan |= deferred.has_session(f.session);
            for (SessionId s : prime_src)
                scan |= deferred.has_session(s);
            if (scan)
                deferred.extract(read_early, [&](const kvr_write_op &w) { hot.push_back(w); });
            // A queued row lies behind its session's window for good: it never
            // touches the ring, whatever later owns its device slot.
            for (kvr_write_op w : cold) {
                w.dev_slot = KVR_NO_SLOT;
                deferred.push(w);
            }
            cold.clear();
            deferred.take(prefill_budget, cold);
        }
        uint64_t prefix = 0;
        for (kvr_write_op &w : hot) {
            w.prefix = prefix;
            prefix += w.count;
        }
        h.write_tokens = prefix;
        prefix = 0;
        for (kvr_write_op &w : cold) {
            w.prefix = prefix;
            prefix += w.count;
        }
        h.write_tokens_cold = prefix;
        h.n_cold = uint32_t(cold.size());
        std::vector<kvr_write_op> all_writes = hot;
        all_writes.insert(all_writes.end(), cold.begin(), cold.end());
        all_writes.insert(all_writes.end(), far_jobs.begin(), far_jobs.end());
        if (with_step) {
            // K-scan capacity (kvr_scan.cu): an overflow would skip the step's gather,
            // so it is refused here instead (descriptors and trains <= non-empty spans)
            if (needs.size() > KVR_MAX_SCAN_NEEDS)
                throw std::runtime_error("step has " + std::to_string(needs.size()) + " stage needs > K-scan capacity " +
                                         std::to_string(KVR_MAX_SCAN_NEEDS));
            if (spans.size() > g.max_scan_descs)
                throw std::runtime_error("step has " + std::to_string(spans.size()) +
                                         " staged spans > geometry.max_scan_descs " + std::to_string(g.max_scan_descs));
        }
        const auto &nd = with_step ? needs : std::vector<kvr_need_rec>{};
        const auto &sp = with_step ? spans : std::vector<kvr_span_rec>{};
        const auto &fi = with_step ? far_ids : std::vector<uint32_t>{};
        h.n_zero = uint32_t(zeros.size());
        h.off_zero = place(zeros.size() * sizeof(kvr_zero_op));
        h.n_cow = uint32_t(cows.size());
        h.off_cow = place(cows.size() * sizeof(kvr_cow_op));
        h.n_edit = uint32_t(edits.size());
        h.off_edit = place(edits.size() * sizeof(kvr_edit_op));
        h.n_write = uint32_t(all_writes.size());
        h.n_far_jobs = uint32_t(far_jobs.size());
        h.off_write = place(all_writes.size() * sizeof(kvr_write_op));
        h.n_blob = uint32_t(blob_ops.size());
        h.off_blob_ops = place(blob_ops.size() * sizeof(kvr_blob_op));
        h.off_blob = place(blob.size());
        h.n_need = uint32_t(nd.size());
        h.off_need = place(nd.size() * sizeof(kvr_need_rec));
        h.n_span = uint32_t(sp.size());
        h.off_span = place(sp.size() * sizeof(kvr_span_rec));
        h.n_prime = uint32_t(primes.size());
        h.off_prime = place(primes.size() * sizeof(kvr_prime_op));
        h.n_far_ids = uint32_t(fi.size());
        h.off_far_ids = place(fi.size() * sizeof(uint32_t));
        h.off_slots = place(slots.size() * sizeof(kvr_slot_state));
        h.n_presum = uint32_t(presum_ops.size());
        h.off_presum = place(presum_ops.size() * sizeof(kvr_presum_op));
        h.n_presum_runs = uint32_t(presum_runs.size());
        h.off_presum_runs = place(presum_runs.size() * sizeof(kvr_presum_run));
        h.n_src_rows = uint32_t(src_rows.size());
        h.off_src_rows = place(src_rows.size() * sizeof(uint32_t));
        h.total_bytes = off;
        std::memcpy(h.counts, step_counts, sizeof(h.counts));
        if (off > g.max_desc_bytes)
            throw std::runtime_error("step descriptor exceeds max_desc_bytes");
        auto *base = static_cast<uint8_t *>(dst);
        auto put = [&](uint64_t at, const void *src, uint64_t bytes) {
            if (bytes)
                std::memcpy(base + at, src, bytes);
        };
        put(0, &h, sizeof(h));
        put(h.off_zero, zeros.data(), zeros.size() * sizeof(kvr_zero_op));
        put(h.off_cow, cows.data(), cows.size() * sizeof(kvr_cow_op));
        put(h.off_edit, edits.data(), edits.size() * sizeof(kvr_edit_op));
        put(h.off_write, all_writes.data(), all_writes.size() * sizeof(kvr_write_op));
        put(h.off_blob_ops, blob_ops.data(), blob_ops.size() * sizeof(kvr_blob_op));
        put(h.off_blob, blob.data(), blob.size());
        put(h.off_need, nd.data(), nd.size() * sizeof(kvr_need_rec));
        put(h.off_span, sp.data(), sp.size() * sizeof(kvr_span_rec));
        put(h.off_prime, primes.data(), primes.size() * sizeof(kvr_prime_op));
        put(h.off_far_ids, fi.data(), fi.size() * sizeof(uint32_t));
        put(h.off_slots, slots.data(), slots.size() * sizeof(kvr_slot_state));
        put(h.off_presum, presum_ops.data(), presum_ops.size() * sizeof(kvr_presum_op));
        put(h.off_presum_runs, presum_runs.data(), presum_runs.size() * sizeof(kvr_presum_run));
        put(h.off_src_rows, src_rows.data(), src_rows.size() * sizeof(uint32_t));
        return off;
    }

    void clear_wave() {
        zero_pages.clear();
        zero_order.clear();
        cows.clear();
        edits.clear();
        writes.clear();
        far_jobs.clear();
        blob_ops.clear();
        blob.clear();
        wave_slots.clear();
        wave_cow_dst.clear();
        primes.clear();
        prime_src.clear();
        src_rows.clear();
    }

    void flush() {
        if (!pending())
            return;
        void *buf = nullptr;
        ck(kvr_dev_desc_buffer(dev, 2, &buf));
        const uint64_t bytes = pack(buf, 0, 0.0, nullptr, false);
        ck(kvr_dev_apply_only(dev, 2, bytes));
        clear_wave();
    }

    // ---- PayloadStore events ----
    void note_slots(BlockId b, uint32_t slot, uint32_t count) {
        auto &w = wave_slots[b];
        if (w.empty())
            w.assign(g.tokens_per_page, 0);
        bool clash = false;
        for (uint32_t i = 0; i < count; ++i)
            clash |= w[slot + i] != 0;
        if (clash) { // same slot written twice in one wave: order matters
            flush();
            auto &w2 = wave_slots[b];
            w2.assign(g.tokens_per_page, 0);
            for (uint32_t i = 0; i < count; ++i)
                w2[slot + i] = 1;
        } else {
            for (uint32_t i = 0; i < count; ++i)
                w[slot + i] = 1;
        }
        auto z = zero_pages.find(b);
        if (z != zero_pages.end())
            for (uint32_t i = 0; i < count; ++i)
                z->second[slot + i] = 1;
        clean[b] = 0;
    }

    void on_alloc(BlockId head, uint32_t count) {
        if (deferred.tokens) { // a recycled page's old deferred rows are unobservable: drop
            bool any = false;
            for (uint32_t i = 0; i < count && !any; ++i)
                any = deferred.has_block(head + i);
            if (any)
                deferred.extract([&](const kvr_write_op &w) { return w.block >= head && w.block < head + count; },
                                 [&](const kvr_write_op &w) { deferred.dropped += w.count; });
        }
        for (uint32_t i = 0; i < count; ++i) {
            const BlockId p = head + i;
            if (clean[p])
                continue;
            if (wave_slots.count(p) || wave_cow_dst.count(p))
                flush(); // zeroing must follow this wave's writes to the page
            if (!zero_pages.count(p)) {
                zero_pages[p].assign(g.tokens_per_page, 0);
                zero_order.push_back(p);
            }
            clean[p] = 1;
        }
    }

    // Deferred prefill rows of `b` (all pages when b == kInvalidBlock) are written now.
    void drain_deferred(BlockId b) {
        if (!deferred.tokens || (b != kInvalidBlock && !deferred.has_block(b)))
            return;
        if (deferred.extract([&](const kvr_write_op &w) { return b == kInvalidBlock || w.block == b; },
                             [&](const kvr_write_op &w) { writes.push_back(w); }))
            flush();
    }

    void copy_page(BlockId src, BlockId dst) {
        drain_deferred(src); // the copy must see src's deferred prefill rows
        if (wave_slots.count(src) || wave_cow_dst.count(src) || zero_pages.count(src))
            flush(); // the copy must see this wave's writes / zeroing of src (K-apply runs
                     // zero ops, copies and blobs of one wave concurrently)
        // the copy overwrites dst entirely; a pending zero of dst is moot
        if (zero_pages.erase(dst))
            zero_order.erase(std::remove(zero_order.begin(), zero_order.end(), dst), zero_order.end());
        cows.push_back({src, dst});
        wave_cow_dst.insert(dst);
        clean[dst] = clean[src];
    }

    void write_host(BlockId b, uint32_t slot, uint32_t count, const std::byte *bytes) {
        const uint64_t n = uint64_t(count) * g.token_bytes;
        if (align16(blob.size() + n) + 65536 > g.max_desc_bytes / 2 || wave_cow_dst.count(b))
            flush(); // (a blob into this wave's copy destination must follow the copy)
        note_slots(b, slot, count);
        blob_ops.push_back({blob.size(), b, slot, count, 0});
        blob.insert(blob.end(), reinterpret_cast<const uint8_t *>(bytes),
                    reinterpret_cast<const uint8_t *>(bytes) + n);
        blob.resize(align16(blob.size()));
    }

    void write_gen(const GeneratedWrite &w) {
        const auto it = bound.find(w.session);
        const uint32_t slot = it == bound.end() ? KVR_NO_SLOT : it->second;
        if (w.source == 1) {
            if (slot == KVR_NO_SLOT)
                throw std::runtime_error("far summary job for a session without a device slot");
            note_slots(w.block, w.slot, w.count);
            kvr_write_op op{};
            op.token = w.token;
            op.aux = w.aux;
            op.block = w.block;
            op.slot = w.slot;
            op.count = 1;
            op.session = w.session;
            op.dev_slot = slot;
            op.source = 1;
            if (g.chunk_tokens && presummed.erase(presum_key(w.session, w.aux / g.chunk_tokens)))
                op.source = 2; // K-presum computed this mean when the rows were written
            else {
                if (w.src_slots.size() != g.chunk_tokens)
                    throw std::runtime_error("far summary job without its chunk's source rows");
                op.prefix = src_rows.size();
                src_rows.insert(src_rows.end(), w.src_slots.begin(), w.src_slots.end());
            }
            far_jobs.push_back(op);
            return;
        }
        if (!presummed.empty() && g.chunk_tokens) // rewritten rows: the stashed mean is stale
            for (uint64_t c = w.token / g.chunk_tokens; c * g.chunk_tokens < w.token + w.count; ++c)
                presummed.erase(presum_key(w.session, c));
        note_slots(w.block, w.slot, w.count);
        if (!writes.empty()) { // coalesce consecutive tokens of one block
            kvr_write_op &b = writes.back();
            if (b.session == w.session && b.block == w.block && b.slot + b.count == w.slot &&
                b.token + b.count == w.token && b.dev_slot == slot) {
                b.count += w.count;
                return;
            }
        }
        kvr_write_op op{};
        op.token = w.token;
        op.block = w.block;
        op.slot = w.slot;
        op.count = w.count;
        op.session = w.session;
        op.dev_slot = slot;
        op.source = 0;
        writes.push_back(op);
    }

    void on_commit(SessionId sid, std::span<const ViewEdit> ed) {
        const auto it = bound.find(sid);
        if (it == bound.end())
            return;
        for (const ViewEdit &e : ed)
            edits.push_back({e.tok_begin, e.tok_end, it->second, e.block, e.slot_begin, 0});
    }

    void read(BlockId b, uint32_t slot, uint32_t count, std::byte *out) {
        drain_deferred(b);
        flush();
        ck(kvr_dev_read(dev, KVR_BUF_ARENA, uint64_t(b) * g.page_bytes + uint64_t(slot) * g.token_bytes,
                        uint64_t(count) * g.token_bytes, out));
    }
};

namespace {

class DeviceStore final : public PayloadStore {
public:
    explicit DeviceStore(DeviceStep::Impl *m) : m_(m) {}
    void on_alloc(BlockId head, uint32_t count) override { m_->on_alloc(head, count); }
    void copy_page(BlockId src, BlockId dst) override { m_->copy_page(src, dst); }
    void write(BlockId b, uint32_t slot, uint32_t count, const std::byte *bytes) override {
        m_->write_host(b, slot, count, bytes);
    }
    void write_generated(const GeneratedWrite &w) override { m_->write_gen(w); }
    void read(BlockId b, uint32_t slot, uint32_t count, std::byte *out) override {
        m_->read(b, slot, count, out);
    }
    void on_commit(SessionId sid, bool, std::span<const ViewEdit> ed) override { m_->on_commit(sid, ed); }

private:
    DeviceStep::Impl *m_;
};

} // namespace

DeviceStep::DeviceStep(const kvr_geometry &geometry) : impl_(std::make_unique<Impl>()) {
    Impl &m = *impl_;
    ck(kvr_dev_open(&geometry, &m.dev));
    m.g = geometry;
    if (!m.g.max_desc_bytes)
        m.g.max_desc_bytes = 16ull << 20;
    if (!m.g.max_scan_descs) // the defaults kvr_dev_open applies
        m.g.max_scan_descs = 2048;
    if (!m.g.max_trains)
        m.g.max_trains = 2048;
    m.clean.assign(m.g.arena_pages, 1); // the arena starts zeroed
    ck(kvr_dev_ring_plane_rows(m.dev, &m.ring_plane_rows));
    m.slots.assign(m.g.n_slots, kvr_slot_state{});
    m.staged_count.assign(m.g.n_slots, 0);
    m.store_ = std::make_shared<DeviceStore>(impl_.get());
}

DeviceStep::~DeviceStep() {
    if (impl_ && impl_->dev) {
        kvr_dev_sync(impl_->dev);
        kvr_dev_close(impl_->dev);
    }
}

const kvr_geometry &DeviceStep::geometry() const { return impl_->g; }
kvr_dev *DeviceStep::handle() const { return impl_->dev; }
std::shared_ptr<PayloadStore> DeviceStep::store() { return impl_->store_; }

void DeviceStep::bind(SessionId sid, uint32_t slot) {
    if (slot >= impl_->g.n_slots)
        throw std::runtime_error("device slot out of range");
    impl_->bound[sid] = slot;
}
void DeviceStep::unbind(SessionId sid) {
    impl_->bound.erase(sid);
    auto &ps = impl_->presummed; // its stash rows may be reused by the slot's next session
    for (auto it = ps.begin(); it != ps.end();)
        it = (*it >> 32) == sid ? ps.erase(it) : std::next(it);
}

void DeviceStep::slot_state(uint32_t slot, SessionId sid, uint64_t written, bool live) {
    kvr_slot_state &s = impl_->slots.at(slot);
    s.session = sid;
    s.written = written;
    s.live = live ? 1 : 0;
    s.far_begin = 0;
    s.far_count = 0;
    s.stage_lo = s.stage_hi = 0;
    impl_->staged_count[slot] = 0;
}

void DeviceStep::need(uint32_t slot, SessionId sid, TrainKind kind, std::span<const StagedSpan> spans,
                      std::span<const uint64_t> first_tokens) {
    Impl &m = *impl_;
    kvr_need_rec n{};
    n.slot = slot;
    n.session = sid;
    n.kind = uint32_t(kind);
    n.span_begin = uint32_t(m.spans.size());
    n.span_count = uint32_t(spans.size());
    m.needs.push_back(n);
    for (size_t i = 0; i < spans.size(); ++i)
        m.spans.push_back({first_tokens[i], spans[i].block, spans[i].slot_begin, spans[i].slot_count, 0});
    // near spans: K-gather is the window writer of their tokens this step (the
    // spans of one session's need are its current reservation span: contiguous)
    if (kind == TrainKind::near_window && slot < m.g.n_slots) {
        kvr_slot_state &st = m.slots[slot];
        for (size_t i = 0; i < spans.size(); ++i) {
            if (!spans[i].slot_count)
                continue;
            const uint64_t lo = first_tokens[i], hi = lo + spans[i].slot_count;
            m.staged_count[slot] += spans[i].slot_count;
            if (st.stage_lo == st.stage_hi) {
                st.stage_lo = lo;
                st.stage_hi = hi;
            } else {
                st.stage_lo = std::min(st.stage_lo, lo);
                st.stage_hi = std::max(st.stage_hi, hi);
            }
        }
    }
}

void DeviceStep::prime(uint32_t slot, uint64_t tok_begin, uint64_t tok_end, SessionId src,
                       std::span<const uint32_t> rows) {
    if (rows.size() != tok_end - tok_begin)
        throw std::runtime_error("prime: one source row per token");
    impl_->primes.push_back({tok_begin, tok_end, slot, uint32_t(impl_->src_rows.size())});
    impl_->src_rows.insert(impl_->src_rows.end(), rows.begin(), rows.end());
    if (src != kNoPrimeSource)
        impl_->prime_src.insert(src); // its rows are read by K-prime: written hot, never deferred
}

void DeviceStep::far_selection(uint32_t slot, std::span<const uint64_t> chunk_ids) {
    Impl &m = *impl_;
    kvr_slot_state &s = m.slots.at(slot);
    s.far_begin = uint32_t(m.far_ids.size());
    s.far_count = 0;
    for (uint64_t id : chunk_ids) {
        if (s.far_count >= m.g.far_cap || id >= m.g.max_chunks)
            break;
        m.far_ids.push_back(uint32_t(id));
        ++s.far_count;
    }
}

void DeviceStep::launch(uint64_t step, double now, const TransportConfig &tc) {
    Impl &m = *impl_;
    const uint32_t k = uint32_t(step & 1);
    if (m.launched_step[k] != ~0ull && !m.have_done[k]) { // ring slot still busy
        kvr_step_stats st{};
        ck(kvr_dev_wait(m.dev, k, &st));
        DeviceStepStats &d = m.done[k];
        d.step = st.step;
        d.device_ms = st.device_ms;
        d.gather_ms = st.gather_ms;
        d.attn_ms = st.attn_ms;
        std::copy(st.phase_ms, st.phase_ms + 8, d.phase_ms);
        d.trains = st.trains;
        d.descriptors = st.descriptors;
        d.train_bytes = st.train_bytes;
        d.writeback_tokens = st.writeback_tokens;
        d.scan_status = st.status;
        d.attn_bytes = m.attn_bytes_pending[k];
        d.h2d_bytes = m.desc_bytes_pending[k];
        d.end_ns = st.end_ns;
        std::copy(st.global_counts, st.global_counts + KVR_COUNTS, d.global_counts);
        m.have_done[k] = true;
    }
    uint64_t attn = 0;
    if (m.g.attention) {
        const uint64_t row = 2ull * m.g.kv_heads * m.g.head_dim * m.g.elem_bytes;
        for (const kvr_slot_state &s : m.slots)
            if (s.live)
                attn += (std::min<uint64_t>(s.written, m.g.near_window) + s.far_count) * m.g.layers * row;
    }
    m.far_shown.assign(m.slots.size(), {});
    for (size_t s = 0; s < m.slots.size(); ++s)
        for (uint32_t i = 0; i < m.slots[s].far_count; ++i)
            m.far_shown[s].push_back(m.far_ids[m.slots[s].far_begin + i]);
    // a slot whose near spans do not form one contiguous token range (never the
    // Driver's; possible through the C-ABI) keeps K-write as its window writer
    for (uint32_t s = 0; s < m.slots.size(); ++s)
        if (m.slots[s].stage_hi - m.slots[s].stage_lo != m.staged_count[s])
            m.slots[s].stage_lo = m.slots[s].stage_hi = 0;
    void *buf = nullptr;
    ck(kvr_dev_desc_buffer(m.dev, k, &buf));
    const uint64_t bytes = m.pack(buf, step, now, &tc, true);
    ck(kvr_dev_launch(m.dev, k, bytes));
    m.launched_step[k] = step;
    m.launched_slots[k] = m.slots;
    m.have_done[k] = false;
    m.attn_bytes_pending[k] = attn;
    m.desc_bytes_pending[k] = bytes;
    m.clear_wave();
    m.needs.clear();
    m.spans.clear();
    m.far_ids.clear();
    for (kvr_slot_state &s : m.slots)
        s.stage_lo = s.stage_hi = 0;
    std::fill(m.staged_count.begin(), m.staged_count.end(), 0);
}

DeviceStepStats DeviceStep::collect(uint64_t step) {
    Impl &m = *impl_;
    auto overflow = [&](const DeviceStepStats &d) {
        if (d.scan_status & 4u) // K-scan ran out of capacity: K-gather skipped the step
            throw std::runtime_error("step " + std::to_string(d.step) +
                                     ": K-scan capacity exceeded (trains > geometry.max_trains or descriptors > "
                                     "max_scan_descs); the staged window of that step is invalid");
    };
    const uint32_t k = uint32_t(step & 1);
    if (m.launched_step[k] != step)
        throw std::runtime_error("collect: step " + std::to_string(step) + " is not in flight");
    if (!m.have_done[k]) {
        kvr_step_stats st{};
        ck(kvr_dev_wait(m.dev, k, &st));
        DeviceStepStats &d = m.done[k];
        d.step = st.step;
        d.device_ms = st.device_ms;
        d.gather_ms = st.gather_ms;
        d.attn_ms = st.attn_ms;
        std::copy(st.phase_ms, st.phase_ms + 8, d.phase_ms);
        d.trains = st.trains;
        d.descriptors = st.descriptors;
        d.train_bytes = st.train_bytes;
        d.writeback_tokens = st.writeback_tokens;
        d.scan_status = st.status;
        d.attn_bytes = m.attn_bytes_pending[k];
        d.h2d_bytes = m.desc_bytes_pending[k];
        d.end_ns = st.end_ns;
        std::copy(st.global_counts, st.global_counts + KVR_COUNTS, d.global_counts);
        m.have_done[k] = true;
    }
    overflow(m.done[k]);
    return m.done[k];
}

std::vector<std::vector<kvr_mass_run>> DeviceStep::utility_runs(uint64_t step) {
    Impl &m = *impl_;
    collect(step);
    const uint32_t k = uint32_t(step & 1);
    const uint32_t W = m.g.near_window;
    std::vector<std::vector<kvr_mass_run>> out(m.g.n_slots);
    if (!m.g.utility || step % m.g.utility)
        return out; // K-mass did not run on this step
    std::vector<kvr_mass_run> runs(uint64_t(m.g.n_slots) * W);
    std::vector<uint32_t> counts(m.g.n_slots);
    ck(kvr_dev_utility(m.dev, k, runs.data(), counts.data()));
    const std::vector<kvr_slot_state> &slots = m.launched_slots[k];
    for (uint32_t s = 0; s < m.g.n_slots && s < slots.size(); ++s)
        if (slots[s].live)
            out[s].assign(runs.begin() + uint64_t(s) * W, runs.begin() + uint64_t(s) * W + std::min(counts[s], W));
    return out;
}

std::vector<std::pair<BlockId, double>> DeviceStep::utility(uint64_t step,
                                                            const std::function<bool(SessionId)> &keep) {
    const std::vector<std::vector<kvr_mass_run>> runs = utility_runs(step);
    const std::vector<kvr_slot_state> &slots = impl_->launched_slots[step & 1];
    std::vector<std::pair<BlockId, double>> obs;
    for (size_t s = 0; s < runs.size(); ++s)
        if (!runs[s].empty() && keep(slots[s].session))
            for (const kvr_mass_run &r : runs[s])
                obs.emplace_back(r.block, double(r.mass));
    return obs;
}

void DeviceStep::counts(const int64_t c[KVR_COUNTS]) { std::copy(c, c + KVR_COUNTS, impl_->step_counts); }

void DeviceStep::comm_init(const uint8_t id[128], int rank, int world) {
    ck(kvr_comm_init(impl_->dev, id, rank, world));
}

void DeviceStep::sync() { ck(kvr_dev_sync(impl_->dev)); }
bool DeviceStep::launched(uint64_t step) const { return impl_->launched_step[step & 1] == step; }
void DeviceStep::flush() { impl_->flush(); }

void DeviceStep::set_prefill_budget(uint64_t tokens) {
    if (!tokens)
        impl_->drain_deferred(kInvalidBlock);
    impl_->prefill_budget = tokens;
}

uint64_t DeviceStep::deferred_tokens() const { return impl_->deferred.tokens; }
uint64_t DeviceStep::dropped_tokens() const { return impl_->deferred.dropped; }

void DeviceStep::read_arena(uint64_t offset, uint64_t bytes, void *out) {
    impl_->drain_deferred(kInvalidBlock);
    impl_->flush();
    ck(kvr_dev_read(impl_->dev, KVR_BUF_ARENA, offset, bytes, out));
}

void DeviceStep::read_ring_token(uint32_t slot, uint64_t token, void *out) {
    const kvr_geometry &g = impl_->g;
    const uint64_t row = 2ull * g.kv_heads * g.head_dim * g.elem_bytes;
    for (uint32_t l = 0; l < g.layers; ++l) {
        const uint64_t off = ((uint64_t(slot) * g.layers + l) * impl_->ring_plane_rows + token % g.ring_rows) * row;
        ck(kvr_dev_read(impl_->dev, KVR_BUF_RING, off, row, static_cast<uint8_t *>(out) + l * row));
    }
}

void DeviceStep::read_staged(uint64_t tok_begin, uint64_t count, void *out, uint8_t *in_window) {
    ck(kvr_dev_read_staged(impl_->dev, tok_begin, count, out, in_window));
}

void DeviceStep::fault(int what, uint64_t arg) { ck(kvr_dev_fault(impl_->dev, what, arg)); }

void DeviceStep::read_page_table(uint32_t slot, uint64_t tok_begin, uint64_t count, uint32_t *out) {
    const kvr_geometry &g = impl_->g;
    ck(kvr_dev_read(impl_->dev, KVR_BUF_TMAP, (uint64_t(slot) * g.max_tokens + tok_begin) * 4, count * 4, out));
}

void DeviceStep::read_attention(uint32_t slot, float *out) {
    const kvr_geometry &g = impl_->g;
    const uint64_t n = uint64_t(g.layers) * g.q_heads * g.head_dim;
    ck(kvr_dev_read(impl_->dev, KVR_BUF_OUT, uint64_t(slot) * n * 4, n * 4, out));
}

namespace {
float bits_to_float(uint32_t b) {
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}
/// IEEE binary16 -> binary32 (exact; the device's exact queries are normal or zero)
float half_to_float(uint16_t h) {
    const uint32_t sign = uint32_t(h & 0x8000u) << 16, exp = (h >> 10) & 0x1fu, man = h & 0x3ffu;
    if (exp == 0 && man == 0)
        return bits_to_float(sign);
    if (exp == 0) { // subnormal
        float v = float(man) * (1.0f / 16777216.0f); // man * 2^-24
        return sign ? -v : v;
    }
    if (exp == 31)
        return bits_to_float(sign | 0x7f800000u | (man << 13));
    return bits_to_float(sign | ((exp + 112u) << 23) | (man << 13));
}
} // namespace

void DeviceStep::read_query(uint32_t slot, float *out) {
    const kvr_geometry &g = impl_->g;
    const uint64_t n = uint64_t(g.layers) * g.q_heads * g.head_dim;
    // exact queries live in the KV element type on the device (kvr_dev.cu: q_esz)
    uint64_t qbytes = 0;
    ck(kvr_dev_buffer_bytes(impl_->dev, KVR_BUF_QUERY, &qbytes));
    if (qbytes == uint64_t(g.n_slots) * n * 4) { // fp32 queries
        ck(kvr_dev_read(impl_->dev, KVR_BUF_QUERY, uint64_t(slot) * n * 4, n * 4, out));
        return;
    }
    std::vector<uint16_t> h(n);
    ck(kvr_dev_read(impl_->dev, KVR_BUF_QUERY, uint64_t(slot) * n * 2, n * 2, h.data()));
    for (uint64_t i = 0; i < n; ++i)
        out[i] = g.elem_kind == KVR_ELEM_BF16 ? bits_to_float(uint32_t(h[i]) << 16) : half_to_float(h[i]);
}

void DeviceStep::read_far_row(uint32_t slot, uint64_t chunk, void *out) {
    const kvr_geometry &g = impl_->g;
    const uint64_t row = 2ull * g.kv_heads * g.head_dim * g.elem_bytes;
    for (uint32_t l = 0; l < g.layers; ++l) {
        const uint64_t off = ((uint64_t(slot) * g.layers + l) * g.max_chunks + chunk) * row;
        ck(kvr_dev_read(impl_->dev, KVR_BUF_FAR, off, row, static_cast<uint8_t *>(out) + l * row));
    }
}

std::vector<uint64_t> DeviceStep::far_selection_of(uint32_t slot) const {
    return slot < impl_->far_shown.size() ? impl_->far_shown[slot] : std::vector<uint64_t>{};
}

void DeviceStep::read_scan(std::vector<kvr_train> &trains, std::vector<kvr_descriptor> &descs) {
    uint32_t ctr[4];
    ck(kvr_dev_read(impl_->dev, KVR_BUF_SCAN, 0, sizeof(ctr), ctr));
    trains.resize(ctr[0]);
    descs.resize(ctr[1]);
    if (ctr[0])
        ck(kvr_dev_read(impl_->dev, KVR_BUF_TRAINS, 0, ctr[0] * sizeof(kvr_train), trains.data()));
    if (ctr[1])
        ck(kvr_dev_read(impl_->dev, KVR_BUF_DESCS, 0, ctr[1] * sizeof(kvr_descriptor), descs.data()));
}

} // namespace kvrail
