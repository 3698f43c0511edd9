// kvrail-b200 C ABI (include/kvrail_c.h) over the C++ API. Exceptions become
// status codes (1 + Errc) with the message kept thread-locally.
#include <cstring>
#include <memory>
#include <string>

#include "kvrail/device_step.hpp"
#include "kvrail/far_view.hpp"
#include "kvrail/pager.hpp"
#include "kvrail/scenario.hpp"
#include "kvrail/transport.hpp"
#include "kvrail_c.h"

using namespace kvrail;

struct kvr_pager {
    std::unique_ptr<Pager> own;
    Pager *p = nullptr;
};

struct kvr_driver {
    std::unique_ptr<ScenarioDriver> d;
    kvr_pager pager_view;
};

namespace {

thread_local std::string g_msg;

template <typename Fn> int call(Fn &&fn) {
    try {
        fn();
        return KVR_OK;
    } catch (const Error &e) {
        g_msg = e.what();
        return 1 + int(e.code());
    } catch (const std::exception &e) {
        g_msg = e.what();
        return std::strstr(e.what(), "CUDA") ? KVR_E_CUDA : KVR_E_INTERNAL;
    }
}

PagerConfig cfg_of(const kvr_pager_config *c) {
    PagerConfig p;
    p.page_bytes = c->page_bytes;
    p.arena_pages = c->arena_pages;
    p.layers = c->layers;
    p.kv_head_dim = c->kv_head_dim;
    p.elem_bytes = c->elem_bytes;
    return p;
}

uint64_t put_blocks(const std::vector<ReservedBlock> &v, kvr_reserved_block *out, uint64_t cap) {
    for (uint64_t i = 0; out && i < v.size() && i < cap; ++i)
        out[i] = {v[i].block, v[i].token_capacity};
    return v.size();
}

kvr_descriptor to_c(const Descriptor &d) {
    kvr_descriptor o{};
    o.phys_offset = d.phys_offset;
    o.length = d.length;
    o.stage_time = d.stage_time;
    o.kind = uint32_t(d.kind);
    o.block = d.block;
    o.session = d.session;
    return o;
}

uint64_t copy_text(const std::string &s, char *buf, uint64_t cap) {
    if (buf && cap) {
        const uint64_t n = std::min<uint64_t>(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return s.size();
}

} // namespace

extern "C" {

const char *kvr_last_error(void) { return g_msg.c_str(); }

int kvr_abi_struct_sizes(uint64_t *out, uint64_t cap, uint64_t *n) {
    const uint64_t sz[] = {
        sizeof(kvr_pager_config), sizeof(kvr_token_range), sizeof(kvr_view_entry),
        sizeof(kvr_view_info),    sizeof(kvr_reserved_block), sizeof(kvr_arena_stats),
        sizeof(kvr_work_counters), sizeof(kvr_free_run),   sizeof(kvr_frame_delta),
        sizeof(kvr_staged_span),  sizeof(kvr_stage_need),  sizeof(kvr_descriptor),
        sizeof(kvr_transport_config), sizeof(kvr_train),   sizeof(kvr_step_record),
        sizeof(kvr_geometry),     sizeof(kvr_step_header), sizeof(kvr_zero_op),
        sizeof(kvr_cow_op),       sizeof(kvr_edit_op),     sizeof(kvr_write_op),
        sizeof(kvr_blob_op),      sizeof(kvr_need_rec),    sizeof(kvr_span_rec),
        sizeof(kvr_prime_op),     sizeof(kvr_slot_state),  sizeof(kvr_step_stats),
        sizeof(kvr_mass_run),
    };
    const uint64_t k = sizeof(sz) / sizeof(sz[0]);
    for (uint64_t i = 0; out && i < k && i < cap; ++i)
        out[i] = sz[i];
    *n = k;
    return KVR_OK;
}

const char *kvr_errc_name(int status) {
    if (status == KVR_OK)
        return "Ok";
    if (status == KVR_E_CUDA)
        return "CudaError";
    if (status < 1 || status > int(Errc::io_error) + 1)
        return "InternalError";
    return errc_name(Errc(status - 1));
}

int kvr_pager_create(const kvr_pager_config *cfg, kvr_pager **out) {
    return call([&] {
        auto h = std::make_unique<kvr_pager>();
        h->own = std::make_unique<Pager>(cfg_of(cfg));
        h->p = h->own.get();
        *out = h.release();
    });
}

int kvr_pager_create_on_device(const kvr_pager_config *cfg, kvr_device *dev, kvr_pager **out) {
    return call([&] {
        auto *step = reinterpret_cast<DeviceStep *>(dev);
        auto h = std::make_unique<kvr_pager>();
        h->own = std::make_unique<Pager>(cfg_of(cfg), step->store());
        h->p = h->own.get();
        *out = h.release();
    });
}

int kvr_pager_destroy(kvr_pager *p) {
    delete p;
    return KVR_OK;
}

int kvr_pager_config_validate(const kvr_pager_config *cfg) {
    return call([&] { cfg_of(cfg).validate(); });
}

int kvr_pager_create_session(kvr_pager *p, uint32_t s) {
    return call([&] { p->p->create_session(s); });
}
int kvr_pager_has_session(kvr_pager *p, uint32_t s, int *out) {
    return call([&] { *out = p->p->has_session(s); });
}
int kvr_pager_reserve(kvr_pager *p, uint32_t s, uint64_t n, kvr_reserved_block *out, uint64_t cap,
                      uint64_t *n_out) {
    return call([&] { *n_out = put_blocks(p->p->reserve(s, n), out, cap); });
}
int kvr_pager_reserve_range(kvr_pager *p, uint32_t s, kvr_token_range r, kvr_reserved_block *out,
                            uint64_t cap, uint64_t *n_out) {
    return call([&] { *n_out = put_blocks(p->p->reserve_range(s, {r.begin, r.end}), out, cap); });
}
int kvr_pager_alias(kvr_pager *p, uint32_t dst, uint32_t src, uint64_t prefix, uint64_t *shared) {
    return call([&] { *shared = p->p->alias(dst, src, prefix); });
}
int kvr_pager_write_tokens(kvr_pager *p, uint32_t s, kvr_token_range r, const void *payload,
                           uint64_t bytes) {
    return call([&] {
        p->p->write_tokens(s, {r.begin, r.end},
                           {static_cast<const std::byte *>(payload), size_t(bytes)});
    });
}
int kvr_pager_trim(kvr_pager *p, uint32_t s, const kvr_token_range *r, uint64_t n, uint64_t *freed) {
    return call([&] {
        std::vector<TokenRange> v(n);
        for (uint64_t i = 0; i < n; ++i)
            v[i] = {r[i].begin, r[i].end};
        *freed = p->p->trim(s, v);
    });
}
int kvr_pager_trim_eos(kvr_pager *p, uint32_t s, uint64_t *freed) {
    return call([&] { *freed = p->p->trim_eos(s); });
}
int kvr_pager_frame_commit(kvr_pager *p, uint32_t s, uint64_t step, uint64_t *epoch) {
    return call([&] { *epoch = p->p->frame_commit(s, step); });
}
int kvr_pager_apply_frame(kvr_pager *p, const kvr_frame_delta *d, uint64_t *epoch) {
    return call([&] {
        FrameDelta f;
        f.session = d->session;
        f.step = d->step;
        f.trim_eos = d->trim_eos != 0;
        f.reserves.assign(d->reserves, d->reserves + d->n_reserves);
        for (uint64_t i = 0; i < d->n_aliases; ++i)
            f.aliases.push_back({d->alias_src[i], d->alias_prefix[i]});
        for (uint64_t i = 0; i < d->n_trims; ++i)
            f.trims.push_back({d->trims[i].begin, d->trims[i].end});
        *epoch = p->p->apply_frame(f);
    });
}
int kvr_pager_active_view(kvr_pager *p, uint32_t s, kvr_view_info *info, kvr_view_entry *e,
                          uint64_t cap) {
    return call([&] {
        const ViewDescriptor v = p->p->active_view(s);
        info->session = v.session;
        info->eos = v.eos;
        info->epoch = v.epoch;
        info->live_tokens = v.live_tokens;
        info->extent = v.extent;
        info->n_entries = v.entries.size();
        for (uint64_t i = 0; e && i < v.entries.size() && i < cap; ++i)
            e[i] = {v.entries[i].tokens.begin, v.entries[i].tokens.end, v.entries[i].block,
                    v.entries[i].slot_begin};
    });
}
int kvr_pager_session_eos(kvr_pager *p, uint32_t s, int *out) {
    return call([&] { *out = p->p->session_eos(s); });
}
int kvr_pager_session_cursor(kvr_pager *p, uint32_t s, uint64_t *out) {
    return call([&] { *out = p->p->session_cursor(s); });
}
int kvr_pager_next_step(kvr_pager *p, uint32_t s, uint64_t *out) {
    return call([&] { *out = p->p->next_step(s); });
}
int kvr_pager_touched_in_last_commit(kvr_pager *p, uint32_t s, uint64_t *out) {
    return call([&] { *out = p->p->touched_in_last_commit(s); });
}
int kvr_pager_stats(kvr_pager *p, kvr_arena_stats *o) {
    return call([&] {
        const ArenaStats st = p->p->stats();
        *o = {st.free_pages, st.live_pages, st.shared_pages, st.reserved_bytes, st.active_bytes};
    });
}
int kvr_pager_counters(kvr_pager *p, kvr_work_counters *o) {
    return call([&] {
        const WorkCounters c = p->p->counters();
        *o = {c.commits,    c.commit_entries_touched, c.reserve_calls, c.reserve_blocks,
              c.reserve_alloc_steps, c.trim_calls, c.trim_blocks, c.free_list_steps};
    });
}
int kvr_pager_read_slots(kvr_pager *p, uint32_t b, uint32_t sb, uint32_t n, void *out) {
    return call([&] { p->p->read_slots(b, sb, n, static_cast<std::byte *>(out)); });
}
int kvr_pager_free_runs(kvr_pager *p, kvr_free_run *out, uint64_t cap, uint64_t *n_out) {
    return call([&] {
        const auto runs = p->p->free_runs();
        for (uint64_t i = 0; out && i < runs.size() && i < cap; ++i)
            out[i] = {runs[i].first, runs[i].second};
        *n_out = runs.size();
    });
}
int kvr_pager_block_refcount(kvr_pager *p, uint32_t b, uint32_t *out) {
    return call([&] { *out = p->p->block_refcount(b); });
}

int kvr_stage(const kvr_stage_need *needs, uint64_t n_needs, const kvr_staged_span *spans,
              uint64_t page_bytes, uint64_t token_bytes, double now, kvr_descriptor *out,
              uint64_t cap, uint64_t *n_out) {
    return call([&] {
        std::vector<StageNeed> v(n_needs);
        for (uint64_t i = 0; i < n_needs; ++i) {
            v[i].session = needs[i].session;
            v[i].kind = TrainKind(needs[i].kind);
            for (uint64_t k = 0; k < needs[i].span_count; ++k) {
                const kvr_staged_span &s = spans[needs[i].span_begin + k];
                v[i].spans.push_back({s.block, s.slot_begin, s.slot_count});
            }
        }
        const auto d = stage(v, page_bytes, token_bytes, now);
        for (uint64_t i = 0; out && i < d.size() && i < cap; ++i)
            out[i] = to_c(d[i]);
        *n_out = d.size();
    });
}

int kvr_reduce(const kvr_descriptor *descs, uint64_t n, const kvr_transport_config *cfg, double now,
               kvr_train *trains, uint64_t train_cap, uint64_t *n_trains, kvr_descriptor *ordered) {
    return call([&] {
        std::vector<Descriptor> v(n);
        for (uint64_t i = 0; i < n; ++i) {
            v[i].phys_offset = descs[i].phys_offset;
            v[i].length = descs[i].length;
            v[i].stage_time = descs[i].stage_time;
            v[i].kind = TrainKind(descs[i].kind);
            v[i].block = descs[i].block;
            v[i].session = descs[i].session;
        }
        TransportConfig tc;
        tc.merge_threshold = cfg->merge_threshold;
        tc.max_hold = cfg->max_hold;
        tc.max_trains_per_step = cfg->max_trains_per_step;
        tc.merge = cfg->merge != 0;
        tc.run_page_bytes = cfg->run_page_bytes;
        tc.run_span_bytes = cfg->run_span_bytes;
        const auto t = reduce(std::move(v), tc, now);
        uint64_t k = 0;
        for (uint64_t i = 0; i < t.size(); ++i) {
            if (trains && i < train_cap)
                trains[i] = {t[i].total_bytes,       t[i].oldest_stage_time, t[i].issue_time,
                             uint32_t(t[i].kind),    uint32_t(t[i].reason),  k,
                             t[i].descriptors.size()};
            for (const Descriptor &d : t[i].descriptors) {
                if (ordered)
                    ordered[k] = to_c(d);
                ++k;
            }
        }
        *n_trains = t.size();
    });
}

int kvr_summarize_chunk(const float *tokens, uint32_t lanes, uint64_t count, float *out) {
    return call([&] {
        const auto m = summarize_chunk({tokens, size_t(lanes) * count}, lanes, count);
        std::memcpy(out, m.data(), m.size() * sizeof(float));
    });
}

int kvr_select_chunks(const double *scores, uint64_t n, uint32_t cap, uint64_t *out, uint64_t *n_out) {
    return call([&] {
        const auto ids = select_chunks(std::vector<double>(scores, scores + n), cap);
        std::memcpy(out, ids.data(), ids.size() * sizeof(uint64_t));
        *n_out = ids.size();
    });
}

int kvr_attend_history(const float *images, uint64_t t, const double *scores, uint64_t n_scores,
                       uint32_t lanes, uint32_t near_window, uint32_t cap, uint32_t chunk_tokens,
                       const float *query, uint32_t layer, uint32_t kv_head_dim, float *out) {
    return call([&] {
        FarViewConfig fv;
        fv.enabled = true;
        fv.near_window = near_window;
        fv.cap = cap;
        fv.chunk_tokens = chunk_tokens;
        const TokenReader rd = [&](uint64_t tok, float *dst) {
            std::memcpy(dst, images + tok * lanes, lanes * sizeof(float));
        };
        const SummarizedView v =
            build_view(rd, t, std::vector<double>(scores, scores + n_scores), lanes, fv);
        const auto o = attend(v, {query, kv_head_dim}, layer, kv_head_dim);
        std::memcpy(out, o.data(), o.size() * sizeof(float));
    });
}

int kvr_driver_create(const char *config_json, int device, kvr_driver **out) {
    return call([&] {
        ScenarioConfig cfg = config_from_json_text(config_json);
        if (device >= 0)
            cfg.b200.device = device;
        cfg.validate();
        auto h = std::make_unique<kvr_driver>();
        h->d = std::make_unique<ScenarioDriver>(
            cfg, shard_events(resolve_events(cfg), cfg.b200.shard_rank, cfg.b200.shard_world));
        h->pager_view.p = h->d->pager();
        *out = h.release();
    });
}

int kvr_driver_destroy(kvr_driver *d) {
    return call([&] { delete d; });
}

static void fill_record(const StepRecord &r, kvr_step_record *o) {
        std::memset(o, 0, sizeof(*o));
        o->step = r.step;
        o->live_sessions = r.live_sessions;
        o->trains = r.trains;
        o->near_trains = r.near_trains;
        o->far_trains = r.far_trains;
        o->dma_bytes = r.dma_bytes;
        o->mean_train_bytes = r.mean_train_bytes;
        o->max_hold = r.max_hold;
        o->submit_time = r.submit_time;
        o->commit_time = r.commit_time;
        o->step_latency = r.step_latency;
        o->reserved_bytes = r.reserved_bytes;
        o->active_bytes = r.active_bytes;
        o->commits = r.commits;
        o->emitted_tokens = r.emitted_tokens;
        o->device_ms = r.device_ms;
        o->gather_ms = r.gather_ms;
        o->attn_ms = r.attn_ms;
        std::memcpy(o->phase_ms, r.phase_ms, sizeof(o->phase_ms));
        o->writeback_tokens = r.writeback_tokens;
        o->gather_bytes = r.gather_bytes;
        o->attn_bytes = r.attn_bytes;
        o->h2d_bytes = r.h2d_bytes;
        o->end_ns = r.end_ns;
        o->global_live = r.global_live;
        o->global_emitted = r.global_emitted;
        o->global_commits = r.global_commits;
        o->global_eos = r.global_eos;
}

int kvr_driver_step(kvr_driver *d, kvr_step_record *o) {
    return call([&] {
        if (d->d->done())
            raise(Errc::bad_config, "all configured steps have run");
        const StepRecord r = d->d->step();
        if (o)
            fill_record(r, o);
    });
}

int kvr_driver_record(kvr_driver *d, uint64_t step, kvr_step_record *o) {
    return call([&] { fill_record(d->d->record(step), o); });
}

int kvr_driver_sync(kvr_driver *d) {
    return call([&] {
        if (d->d->device())
            d->d->device()->sync();
    });
}

int kvr_driver_progress(kvr_driver *d, uint64_t *done, uint64_t *total) {
    return call([&] {
        *done = d->d->steps_done();
        *total = d->d->config().steps;
    });
}

int kvr_driver_steps_csv(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len) {
    return call([&] { *len = copy_text(steps_to_csv(d->d->records()), buf, cap); });
}

int kvr_driver_report_json(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len) {
    return call([&] { *len = copy_text(report_to_json(d->d->result()), buf, cap); });
}

int kvr_driver_prefill_backlog(kvr_driver *d, uint64_t *queued, uint64_t *dropped) {
    return call([&] {
        const DeviceStep *dev = d->d->device();
        *queued = dev ? dev->deferred_tokens() : 0;
        *dropped = dev ? dev->dropped_tokens() : 0;
    });
}

static void complete_records(kvr_driver *d) {
    for (uint64_t s = 0; s < d->d->steps_done(); ++s)
        d->d->record(s);
}

int kvr_driver_measured_csv(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len) {
    return call([&] {
        complete_records(d);
        *len = copy_text(measured_steps_csv(d->d->records()), buf, cap);
    });
}

int kvr_driver_measured_json(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len) {
    return call([&] {
        complete_records(d);
        *len = copy_text(measured_report_json(d->d->records(), d->d->config().warmup_steps), buf, cap);
    });
}

int kvr_driver_trace(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len) {
    return call([&] { *len = copy_text(d->d->trace(), buf, cap); });
}

int kvr_driver_pager(kvr_driver *d, kvr_pager **out) {
    return call([&] {
        if (!d->pager_view.p)
            raise(Errc::bad_config, "static-arena run has no pager");
        *out = &d->pager_view;
    });
}

int kvr_driver_live(kvr_driver *d, uint32_t *slot, uint32_t *session, uint64_t *written,
                    uint64_t cap, uint64_t *n_out) {
    return call([&] {
        const auto v = d->d->live();
        for (uint64_t i = 0; i < v.size() && i < cap; ++i) {
            slot[i] = v[i].slot;
            session[i] = v[i].session;
            written[i] = v[i].written;
        }
        *n_out = v.size();
    });
}

int kvr_driver_workload_hash(kvr_driver *d, uint64_t *out) {
    return call([&] { *out = stream_hash(d->d->events()); });
}

int kvr_driver_device_check(kvr_driver *d, uint64_t *checked, uint64_t *mismatches, char *buf,
                            uint64_t cap) {
    return call([&] {
        std::string first;
        d->d->device_check(*checked, *mismatches, first);
        copy_text(first, buf, cap);
    });
}

int kvr_driver_staged_rows(kvr_driver *d, uint64_t *delivered, uint64_t *behind, uint64_t *missing) {
    return call([&] { d->d->staged_rows(*delivered, *behind, *missing); });
}

int kvr_driver_comm_init(kvr_driver *d, const uint8_t id[128], int rank, int world) {
    return call([&] { d->d->comm_init(id, rank, world); });
}

int kvr_driver_fault(kvr_driver *d, int what, uint64_t arg) {
    return call([&] { d->d->fault(what, arg); });
}

// ---- device ------------------------------------------------------------------

#define DS reinterpret_cast<DeviceStep *>(d)

int kvr_device_open(const kvr_geometry *g, kvr_device **out) {
    return call([&] { *out = reinterpret_cast<kvr_device *>(new DeviceStep(*g)); });
}
int kvr_device_close(kvr_device *d) {
    return call([&] { delete DS; });
}
int kvr_device_flush(kvr_device *d) {
    return call([&] { DS->flush(); });
}
int kvr_device_geometry(kvr_device *d, kvr_geometry *out) {
    return call([&] { *out = DS->geometry(); });
}
int kvr_device_bind(kvr_device *d, uint32_t session, uint32_t slot) {
    return call([&] { DS->bind(session, slot); });
}
int kvr_driver_device(kvr_driver *dr, kvr_device **out) {
    return call([&] {
        if (!dr->d->device())
            raise(Errc::bad_config, "driver runs without a device (b200.device < 0)");
        *out = reinterpret_cast<kvr_device *>(dr->d->device());
    });
}
int kvr_device_raw(kvr_device *d, kvr_dev **out) {
    return call([&] { *out = DS->handle(); });
}
int kvr_device_read_ring_token(kvr_device *d, uint32_t slot, uint64_t token, void *out) {
    return call([&] { DS->read_ring_token(slot, token, out); });
}
int kvr_device_read_page_table(kvr_device *d, uint32_t slot, uint64_t tok_begin, uint64_t count,
                               uint32_t *out) {
    return call([&] { DS->read_page_table(slot, tok_begin, count, out); });
}
int kvr_device_read_attention(kvr_device *d, uint32_t slot, float *out) {
    return call([&] { DS->read_attention(slot, out); });
}
int kvr_device_read_query(kvr_device *d, uint32_t slot, float *out) {
    return call([&] { DS->read_query(slot, out); });
}
int kvr_device_read_far_row(kvr_device *d, uint32_t slot, uint64_t chunk, void *out) {
    return call([&] { DS->read_far_row(slot, chunk, out); });
}
int kvr_device_far_selection(kvr_device *d, uint32_t slot, uint64_t *out, uint64_t cap,
                             uint64_t *n_out) {
    return call([&] {
        const auto v = DS->far_selection_of(slot);
        for (uint64_t i = 0; out && i < v.size() && i < cap; ++i)
            out[i] = v[i];
        *n_out = v.size();
    });
}
int kvr_device_utility(kvr_device *d, uint64_t step, kvr_mass_run *runs, uint32_t *counts) {
    return call([&] {
        if (!DS->launched(step))
            throw Error(Errc::bad_config, "step " + std::to_string(step) + " is not in a ring slot");
        const auto v = DS->utility_runs(step);
        const uint32_t W = DS->geometry().near_window;
        for (size_t s = 0; s < v.size(); ++s) {
            counts[s] = uint32_t(v[s].size());
            std::copy(v[s].begin(), v[s].end(), runs + s * W);
        }
    });
}
int kvr_device_read_scan(kvr_device *d, kvr_train *trains, uint64_t train_cap, uint64_t *n_trains,
                         kvr_descriptor *descs, uint64_t desc_cap, uint64_t *n_descs) {
    return call([&] {
        std::vector<kvr_train> t;
        std::vector<kvr_descriptor> ds;
        DS->read_scan(t, ds);
        for (uint64_t i = 0; trains && i < t.size() && i < train_cap; ++i)
            trains[i] = t[i];
        for (uint64_t i = 0; descs && i < ds.size() && i < desc_cap; ++i)
            descs[i] = ds[i];
        *n_trains = t.size();
        *n_descs = ds.size();
    });
}
#undef DS

} // extern "C"
