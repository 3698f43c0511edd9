// Test infrastructure (oracle) — NOT product code. Only tests/, the smoke
// check and bench.py's cpu_baseline / --impl reference legs may load it.
//
// A C shim over the UNMODIFIED reference library (sources compiled in place
// from /root/reference/proj by oracle/Makefile, namespace renamed to
// kvrail_ref with -Dkvrail=kvrail_ref). It exports the same C signatures as
// include/kvrail_c.h with the prefix `kvr_ref_` so the parity tests can drive
// the reference and the B200 implementation through one Python wrapper.
// It also implements the scenario.cpp hooks declared in ref_hook_decl.hpp,
// which record a per-step parity trace (see trace format in DESIGN.md §5).

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <unistd.h>

#include "kvrail/far_view.hpp"
#include "kvrail/pager.hpp"
#include "kvrail/scenario.hpp"
#include "kvrail/transport.hpp"
#include "kvrail_c.h"
#include "ref_hook_decl.hpp"

using namespace kvrail;

namespace {

thread_local std::string g_err;

int fail_from(const std::exception &e) {
    g_err = e.what();
    if (auto *ke = dynamic_cast<const Error *>(&e))
        return 1 + static_cast<int>(ke->code());
    return KVR_E_INTERNAL;
}

template <typename Fn> int guard(Fn &&fn) {
    try {
        fn();
        return KVR_OK;
    } catch (const std::exception &e) {
        return fail_from(e);
    }
}

PagerConfig to_cfg(const kvr_pager_config *c) {
    PagerConfig p;
    p.page_bytes = c->page_bytes;
    p.arena_pages = c->arena_pages;
    p.layers = c->layers;
    p.kv_head_dim = c->kv_head_dim;
    p.elem_bytes = c->elem_bytes;
    return p;
}

uint64_t copy_blocks(const std::vector<ReservedBlock> &rb, kvr_reserved_block *out, uint64_t cap) {
    if (out)
        for (uint64_t i = 0; i < rb.size() && i < cap; ++i)
            out[i] = {rb[i].block, rb[i].token_capacity};
    return rb.size();
}

// ---- per-step trace recording ----------------------------------------------

struct Fnv {
    uint64_t h = 1469598103934665603ull;
    void byte(uint8_t b) {
        h ^= b;
        h *= 1099511628211ull;
    }
    void word(uint64_t v) {
        for (int i = 0; i < 8; ++i)
            byte(static_cast<uint8_t>(v >> (8 * i)));
    }
    void bytes(const std::byte *p, size_t n) {
        for (size_t i = 0; i < n; ++i)
            byte(static_cast<uint8_t>(p[i]));
    }
};

struct TraceState {
    bool enabled = false;
    const Pager *pager = nullptr;
    uint64_t step = 0;
    std::string out;
    std::vector<StageNeed> pending_needs;
};
thread_local TraceState g_trace;

void trace_pager_line(const Pager &p) {
    ArenaStats st = p.stats();
    Fnv runs;
    for (auto [h, n] : p.free_runs()) {
        runs.word(h);
        runs.word(n);
    }
    Fnv views;
    uint64_t n_sess = 0;
    auto dump = [&](SessionId id) {
        ViewDescriptor v = p.active_view(id);
        views.word(id);
        views.word(v.epoch);
        views.word(v.live_tokens);
        views.word(v.extent);
        views.word(v.eos ? 1 : 0);
        views.word(v.entries.size());
        for (const ViewEntry &e : v.entries) {
            views.word(e.tokens.begin);
            views.word(e.tokens.end);
            views.word(e.block);
            views.word(e.slot_begin);
        }
        ++n_sess;
    };
    for (SessionId id = 0; p.has_session(id); ++id)
        dump(id);
    if (p.has_session(0x7fffffff))
        dump(0x7fffffff);
    char buf[320];
    std::snprintf(buf, sizeof(buf),
                  "pager free=%llu live=%llu shared=%llu reserved=%llu active=%llu runs=%016llx "
                  "views=%016llx sessions=%llu\n",
                  (unsigned long long)st.free_pages, (unsigned long long)st.live_pages,
                  (unsigned long long)st.shared_pages, (unsigned long long)st.reserved_bytes,
                  (unsigned long long)st.active_bytes, (unsigned long long)runs.h,
                  (unsigned long long)views.h, (unsigned long long)n_sess);
    g_trace.out += buf;
}

uint64_t staged_hash(const Pager *p, const DmaTrain &t) {
    Fnv f;
    if (!p)
        return 0;
    const uint64_t page = p->config().page_bytes;
    const uint64_t tb = p->config().token_bytes();
    std::vector<std::byte> tok(tb);
    for (const Descriptor &d : t.descriptors) {
        for (uint64_t off = d.phys_offset; off < d.phys_offset + d.length; off += tb) {
            BlockId b = static_cast<BlockId>(off / page);
            uint32_t slot = static_cast<uint32_t>((off % page) / tb);
            p->read_slots(b, slot, 1, tok.data());
            f.bytes(tok.data(), tb);
        }
    }
    return f.h;
}

} // namespace

namespace kvrail {

HookedPager::HookedPager(PagerConfig cfg) : Pager(cfg) { g_trace.pager = this; }

std::vector<Descriptor> kvr_hook_stage(const std::vector<StageNeed> &needs, uint64_t page_bytes,
                                       uint64_t token_bytes, double now) {
    if (g_trace.enabled)
        g_trace.pending_needs = needs;
    return stage(needs, page_bytes, token_bytes, now);
}

std::vector<DmaTrain> kvr_hook_reduce(std::vector<Descriptor> descriptors,
                                      const TransportConfig &cfg, double now) {
    std::vector<DmaTrain> trains = reduce(std::move(descriptors), cfg, now);
    if (!g_trace.enabled)
        return trains;
    char buf[256];
    std::snprintf(buf, sizeof(buf), "step %llu\n", (unsigned long long)g_trace.step++);
    g_trace.out += buf;
    for (const StageNeed &n : g_trace.pending_needs) {
        std::snprintf(buf, sizeof(buf), "need %u %u %zu", n.session, (unsigned)n.kind,
                      n.spans.size());
        g_trace.out += buf;
        for (const StagedSpan &s : n.spans) {
            std::snprintf(buf, sizeof(buf), " %u:%u:%u", s.block, s.slot_begin, s.slot_count);
            g_trace.out += buf;
        }
        g_trace.out += "\n";
    }
    g_trace.pending_needs.clear();
    for (const DmaTrain &t : trains) {
        std::snprintf(buf, sizeof(buf), "train %u %u %llu %zu t=%.6f o=%.6f h=%016llx",
                      (unsigned)t.kind, (unsigned)t.reason, (unsigned long long)t.total_bytes,
                      t.descriptors.size(), t.issue_time, t.oldest_stage_time,
                      (unsigned long long)staged_hash(g_trace.pager, t));
        g_trace.out += buf;
        for (const Descriptor &d : t.descriptors) {
            std::snprintf(buf, sizeof(buf), " %llu+%llu@%u", (unsigned long long)d.phys_offset,
                          (unsigned long long)d.length, d.session);
            g_trace.out += buf;
        }
        g_trace.out += "\n";
    }
    if (g_trace.pager)
        trace_pager_line(*g_trace.pager);
    else
        g_trace.out += "pager none\n";
    return trains;
}

} // namespace kvrail

// ---- C ABI mirror -------------------------------------------------------------

extern "C" {

const char *kvr_ref_last_error(void) { return g_err.c_str(); }

int kvr_ref_pager_create(const kvr_pager_config *cfg, void **out) {
    return guard([&] { *out = new Pager(to_cfg(cfg)); });
}
int kvr_ref_pager_destroy(void *p) {
    delete static_cast<Pager *>(p);
    return KVR_OK;
}
int kvr_ref_pager_config_validate(const kvr_pager_config *cfg) {
    return guard([&] { to_cfg(cfg).validate(); });
}
#define P static_cast<Pager *>(p)
int kvr_ref_pager_create_session(void *p, uint32_t s) {
    return guard([&] { P->create_session(s); });
}
int kvr_ref_pager_has_session(void *p, uint32_t s, int *out) {
    return guard([&] { *out = P->has_session(s) ? 1 : 0; });
}
int kvr_ref_pager_reserve(void *p, uint32_t s, uint64_t n, kvr_reserved_block *out, uint64_t cap,
                          uint64_t *n_out) {
    return guard([&] { *n_out = copy_blocks(P->reserve(s, n), out, cap); });
}
int kvr_ref_pager_reserve_range(void *p, uint32_t s, kvr_token_range r, kvr_reserved_block *out,
                                uint64_t cap, uint64_t *n_out) {
    return guard([&] { *n_out = copy_blocks(P->reserve_range(s, {r.begin, r.end}), out, cap); });
}
int kvr_ref_pager_alias(void *p, uint32_t dst, uint32_t src, uint64_t prefix, uint64_t *shared) {
    return guard([&] { *shared = P->alias(dst, src, prefix); });
}
int kvr_ref_pager_write_tokens(void *p, uint32_t s, kvr_token_range r, const void *payload,
                               uint64_t bytes) {
    return guard([&] {
        P->write_tokens(s, {r.begin, r.end},
                        std::span<const std::byte>(static_cast<const std::byte *>(payload), bytes));
    });
}
int kvr_ref_pager_trim(void *p, uint32_t s, const kvr_token_range *r, uint64_t n, uint64_t *freed) {
    return guard([&] {
        std::vector<TokenRange> v;
        for (uint64_t i = 0; i < n; ++i)
            v.push_back({r[i].begin, r[i].end});
        *freed = P->trim(s, v);
    });
}
int kvr_ref_pager_trim_eos(void *p, uint32_t s, uint64_t *freed) {
    return guard([&] { *freed = P->trim_eos(s); });
}
int kvr_ref_pager_frame_commit(void *p, uint32_t s, uint64_t step, uint64_t *epoch) {
    return guard([&] { *epoch = P->frame_commit(s, step); });
}
int kvr_ref_pager_apply_frame(void *p, const kvr_frame_delta *d, uint64_t *epoch) {
    return guard([&] {
        FrameDelta fd;
        fd.session = d->session;
        fd.step = d->step;
        fd.trim_eos = d->trim_eos != 0;
        for (uint64_t i = 0; i < d->n_reserves; ++i)
            fd.reserves.push_back(d->reserves[i]);
        for (uint64_t i = 0; i < d->n_aliases; ++i)
            fd.aliases.push_back({d->alias_src[i], d->alias_prefix[i]});
        for (uint64_t i = 0; i < d->n_trims; ++i)
            fd.trims.push_back({d->trims[i].begin, d->trims[i].end});
        *epoch = P->apply_frame(fd);
    });
}
int kvr_ref_pager_active_view(void *p, uint32_t s, kvr_view_info *info, kvr_view_entry *e,
                              uint64_t cap) {
    return guard([&] {
        ViewDescriptor v = P->active_view(s);
        info->session = v.session;
        info->eos = v.eos ? 1 : 0;
        info->epoch = v.epoch;
        info->live_tokens = v.live_tokens;
        info->extent = v.extent;
        info->n_entries = v.entries.size();
        if (e)
            for (uint64_t i = 0; i < v.entries.size() && i < cap; ++i)
                e[i] = {v.entries[i].tokens.begin, v.entries[i].tokens.end, v.entries[i].block,
                        v.entries[i].slot_begin};
    });
}
int kvr_ref_pager_session_eos(void *p, uint32_t s, int *out) {
    return guard([&] { *out = P->session_eos(s) ? 1 : 0; });
}
int kvr_ref_pager_session_cursor(void *p, uint32_t s, uint64_t *out) {
    return guard([&] { *out = P->session_cursor(s); });
}
int kvr_ref_pager_next_step(void *p, uint32_t s, uint64_t *out) {
    return guard([&] { *out = P->next_step(s); });
}
int kvr_ref_pager_touched_in_last_commit(void *p, uint32_t s, uint64_t *out) {
    return guard([&] { *out = P->touched_in_last_commit(s); });
}
int kvr_ref_pager_stats(void *p, kvr_arena_stats *o) {
    return guard([&] {
        ArenaStats st = P->stats();
        *o = {st.free_pages, st.live_pages, st.shared_pages, st.reserved_bytes, st.active_bytes};
    });
}
int kvr_ref_pager_counters(void *p, kvr_work_counters *o) {
    return guard([&] {
        WorkCounters c = P->counters();
        *o = {c.commits,     c.commit_entries_touched, c.reserve_calls, c.reserve_blocks,
              c.reserve_alloc_steps, c.trim_calls, c.trim_blocks, c.free_list_steps};
    });
}
int kvr_ref_pager_read_slots(void *p, uint32_t b, uint32_t sb, uint32_t n, void *out) {
    return guard([&] { P->read_slots(b, sb, n, static_cast<std::byte *>(out)); });
}
int kvr_ref_pager_free_runs(void *p, kvr_free_run *out, uint64_t cap, uint64_t *n_out) {
    return guard([&] {
        auto runs = P->free_runs();
        if (out)
            for (uint64_t i = 0; i < runs.size() && i < cap; ++i)
                out[i] = {runs[i].first, runs[i].second};
        *n_out = runs.size();
    });
}
int kvr_ref_pager_block_refcount(void *p, uint32_t b, uint32_t *out) {
    return guard([&] { *out = P->block_refcount(b); });
}
#undef P

int kvr_ref_stage(const kvr_stage_need *needs, uint64_t n_needs, const kvr_staged_span *spans,
                  uint64_t page_bytes, uint64_t token_bytes, double now, kvr_descriptor *out,
                  uint64_t cap, uint64_t *n_out) {
    return guard([&] {
        std::vector<StageNeed> v(n_needs);
        for (uint64_t i = 0; i < n_needs; ++i) {
            v[i].session = needs[i].session;
            v[i].kind = static_cast<TrainKind>(needs[i].kind);
            for (uint64_t k = 0; k < needs[i].span_count; ++k) {
                const kvr_staged_span &s = spans[needs[i].span_begin + k];
                v[i].spans.push_back({s.block, s.slot_begin, s.slot_count});
            }
        }
        auto d = stage(v, page_bytes, token_bytes, now);
        *n_out = d.size();
        if (out)
            for (uint64_t i = 0; i < d.size() && i < cap; ++i)
                out[i] = {d[i].phys_offset, d[i].length, d[i].stage_time,
                          static_cast<uint32_t>(d[i].kind), d[i].block, d[i].session, 0};
    });
}

int kvr_ref_reduce(const kvr_descriptor *descs, uint64_t n, const kvr_transport_config *cfg,
                   double now, kvr_train *trains, uint64_t train_cap, uint64_t *n_trains,
                   kvr_descriptor *ordered) {
    return guard([&] {
        std::vector<Descriptor> v(n);
        for (uint64_t i = 0; i < n; ++i) {
            v[i].phys_offset = descs[i].phys_offset;
            v[i].length = descs[i].length;
            v[i].stage_time = descs[i].stage_time;
            v[i].kind = static_cast<TrainKind>(descs[i].kind);
            v[i].block = descs[i].block;
            v[i].session = descs[i].session;
        }
        TransportConfig tc;
        tc.merge_threshold = cfg->merge_threshold;
        tc.max_hold = cfg->max_hold;
        tc.max_trains_per_step = cfg->max_trains_per_step;
        tc.merge = cfg->merge != 0;
        auto t = reduce(std::move(v), tc, now);
        *n_trains = t.size();
        uint64_t k = 0;
        for (uint64_t i = 0; i < t.size(); ++i) {
            if (trains && i < train_cap)
                trains[i] = {t[i].total_bytes, t[i].oldest_stage_time, t[i].issue_time,
                             static_cast<uint32_t>(t[i].kind), static_cast<uint32_t>(t[i].reason),
                             k, t[i].descriptors.size()};
            for (const Descriptor &d : t[i].descriptors) {
                if (ordered)
                    ordered[k] = {d.phys_offset, d.length, d.stage_time,
                                  static_cast<uint32_t>(d.kind), d.block, d.session, 0};
                ++k;
            }
        }
    });
}

int kvr_ref_summarize_chunk(const float *tokens, uint32_t lanes, uint64_t count, float *out) {
    return guard([&] {
        auto m = summarize_chunk(std::span<const float>(tokens, static_cast<size_t>(lanes) * count),
                                 lanes, count);
        std::memcpy(out, m.data(), m.size() * sizeof(float));
    });
}

int kvr_ref_select_chunks(const double *scores, uint64_t n, uint32_t cap, uint64_t *out,
                          uint64_t *n_out) {
    return guard([&] {
        auto ids = select_chunks(std::vector<double>(scores, scores + n), cap);
        for (size_t i = 0; i < ids.size(); ++i)
            out[i] = ids[i];
        *n_out = ids.size();
    });
}

int kvr_ref_attend_history(const float *images, uint64_t t, const double *chunk_scores,
                           uint64_t n_scores, uint32_t lanes, uint32_t near_window, uint32_t cap,
                           uint32_t chunk_tokens, const float *query, uint32_t layer,
                           uint32_t kv_head_dim, float *out) {
    return guard([&] {
        TokenReader read = [&](uint64_t tok, float *dst) {
            std::memcpy(dst, images + tok * lanes, lanes * sizeof(float));
        };
        FarViewConfig cfg;
        cfg.enabled = true;
        cfg.near_window = near_window;
        cfg.cap = cap;
        cfg.chunk_tokens = chunk_tokens;
        std::vector<double> scores(chunk_scores, chunk_scores + n_scores);
        SummarizedView v = build_view(read, t, scores, lanes, cfg);
        auto o = attend(v, std::span<const float>(query, kv_head_dim), layer, kv_head_dim);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

// Run one full reference scenario (run_scenario, scenario.cpp:696-700) from a
// JSON config string in the reference schema. Returns malloc'ed strings
// (release with kvr_ref_free): steps.csv, report.json and, when `trace` is
// non-zero, the per-step parity trace recorded by the hooks above.
int kvr_ref_scenario_run(const char *config_json, int trace, char **steps_csv,
                         char **report_json, char **trace_out, double *wall_seconds) {
    return guard([&] {
        char path[] = "/tmp/kvr_ref_cfg_XXXXXX";
        int fd = mkstemp(path);
        if (fd < 0)
            raise(Errc::io_error, "mkstemp");
        {
            std::ofstream f(path);
            f << config_json;
        }
        close(fd);
        ScenarioConfig cfg;
        try {
            cfg = config_from_json_file(path);
        } catch (...) {
            std::filesystem::remove(path);
            throw;
        }
        std::filesystem::remove(path);
        g_trace = TraceState{};
        g_trace.enabled = trace != 0;
        auto t0 = std::chrono::steady_clock::now();
        RunResult r = run_scenario(cfg);
        auto t1 = std::chrono::steady_clock::now();
        if (wall_seconds)
            *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
        auto dup = [](const std::string &s) {
            char *p = static_cast<char *>(std::malloc(s.size() + 1));
            std::memcpy(p, s.c_str(), s.size() + 1);
            return p;
        };
        if (steps_csv)
            *steps_csv = dup(steps_to_csv(r.records));
        if (report_json)
            *report_json = dup(report_to_json(r));
        if (trace_out)
            *trace_out = dup(g_trace.out);
        g_trace = TraceState{};
    });
}

// Resolved event stream (resolve_events, scenario.cpp:71-92) as trace CSV.
int kvr_ref_scenario_events(const char *config_json, char **csv) {
    return guard([&] {
        char path[] = "/tmp/kvr_ref_cfg_XXXXXX";
        int fd = mkstemp(path);
        {
            std::ofstream f(path);
            f << config_json;
        }
        close(fd);
        ScenarioConfig cfg = config_from_json_file(path);
        std::filesystem::remove(path);
        auto ev = resolve_events(cfg);
        std::string s = "arrival_ms,prompt_tokens,generate_tokens\n";
        for (const TraceEvent &e : ev)
            s += std::to_string(e.arrival_ms) + "," + std::to_string(e.prompt_tokens) + "," +
                 std::to_string(e.generate_tokens) + "\n";
        char *p = static_cast<char *>(std::malloc(s.size() + 1));
        std::memcpy(p, s.c_str(), s.size() + 1);
        *csv = p;
    });
}

void kvr_ref_free(char *p) { std::free(p); }

// ---- CPU baseline legs (bench.py cpu_baseline / --impl reference) ----------------
// The reference's own attention path for one (session, layer, q-head): build the
// fixed-width view of a `window`-token history through a TokenReader (the
// near-window gather, far_view.cpp:64-111) and attend over it (far_view.cpp:113-
// 155). `calls` such (session, head) evaluations run on `threads` OpenMP threads
// (build_view/attend are serial inside); returns wall seconds. Calls cycle over
// `pool` distinct histories (a pool larger than the host caches makes the reads
// come from DRAM, as a real batch's KV would).
int kvr_ref_cpu_attention_sample(uint32_t head_dim, uint32_t window, uint32_t calls, int threads, uint32_t pool,
                                 double *seconds, double *checksum) {
    return guard([&] {
        const uint32_t lanes = 2 * head_dim;
        pool = pool ? pool : 1;
        std::vector<float> hist(size_t(pool) * window * lanes);
        for (size_t i = 0; i < hist.size(); ++i)
            hist[i] = float(int64_t((i * 2654435761ull) % 2001) - 1000) / 1000.0f;
        std::vector<float> q(head_dim);
        for (uint32_t d = 0; d < head_dim; ++d)
            q[d] = float(int(d % 17) - 8) / 8.0f;
        FarViewConfig cfg;
        cfg.enabled = true;
        cfg.near_window = window;
        cfg.cap = 0;
        cfg.chunk_tokens = 128;
        double sum = 0.0;
        const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4) reduction(+ : sum)
        for (int64_t c = 0; c < int64_t(calls); ++c) {
            const float *h = hist.data() + size_t(c % pool) * window * lanes;
            TokenReader read = [&](uint64_t tok, float *out) {
                std::memcpy(out, h + tok * lanes, lanes * sizeof(float));
            };
            SummarizedView v = build_view(read, window, {}, lanes, cfg);
            auto o = attend(v, q, 0, head_dim);
            sum += o[c % head_dim];
        }
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (checksum)
            *checksum = sum;
    });
}

// Host copy bandwidth of the gather leg (read_slots-style memcpy, 1 thread, like
// the reference Driver): returns (read + write) GB/s over `bytes`.
int kvr_ref_cpu_memcpy_gbs(uint64_t bytes, int reps, double *gbs) {
    return guard([&] {
        std::vector<std::byte> a(bytes, std::byte{1}), b(bytes);
        std::memcpy(b.data(), a.data(), bytes);
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r)
            std::memcpy(r & 1 ? a.data() : b.data(), r & 1 ? b.data() : a.data(), bytes);
        const auto t1 = std::chrono::steady_clock::now();
        *gbs = 2.0 * double(bytes) * reps / std::chrono::duration<double>(t1 - t0).count() / 1e9;
    });
}

// The gather leg through the reference's own API: a reference Pager at the real
// geometry holding `bytes` of written tokens (whole pages, one session), then
// Pager::read_slots of every token into a host staging window, page run by page run
// — the bytes the step's trains stage, copied the way the reference
// reads them. Returns wall seconds per pass (mean over `reps`).
int kvr_ref_cpu_gather_seconds(uint64_t page_bytes, uint32_t layers, uint32_t kv_head_dim, uint32_t elem_bytes,
                               uint64_t bytes, int reps, double *seconds) {
    return guard([&] {
        PagerConfig pc;
        pc.page_bytes = page_bytes;
        pc.layers = layers;
        pc.kv_head_dim = kv_head_dim;
        pc.elem_bytes = elem_bytes;
        const uint64_t tb = pc.token_bytes(), tpp = pc.tokens_per_page();
        const uint64_t tokens = (bytes + tb - 1) / tb;
        pc.arena_pages = uint32_t((tokens + tpp - 1) / tpp + 1);
        Pager p(pc);
        p.create_session(1);
        p.reserve(1, tokens);
        std::vector<std::byte> payload(tb);
        for (uint64_t t = 0; t < tokens; ++t) {
            std::memset(payload.data(), int(t & 0xff), tb);
            p.write_tokens(1, {t, t + 1}, payload);
        }
        p.frame_commit(1, 0);
        const ViewDescriptor v = p.active_view(1);
        std::vector<std::byte> window(tokens * tb);
        double total = 0.0;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            uint64_t at = 0;
            for (const ViewEntry &e : v.entries) {
                const uint32_t n = uint32_t(e.tokens.end - e.tokens.begin);
                p.read_slots(e.block, e.slot_begin, n, window.data() + at);
                at += uint64_t(n) * tb;
            }
            total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        *seconds = total / reps;
    });
}

} // extern "C"
