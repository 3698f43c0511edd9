// kvrail-b200 scenario driver: the per-step caller of the hot path.
//
// Behavioural contract: the reference Driver, scenario.cpp:124-683 (and the
// run/report/config functions at 687-1029). Given the same config and event
// stream it issues the same pager verbs, commits, stage needs and reduce calls
// in the same order, so records and the parity trace are byte-identical.
// What changes on a B200 (b200.device >= 0):
//   * token payloads are generated where the bytes live (device arena) via
//     Pager::write_tokens_generated instead of host memcpy;
//   * far-view summaries are computed by the K-far kernel (host keeps scores);
//   * every step ends in DeviceStep::launch — one committed descriptor, one
//     H2D copy, one graph replay — instead of the cost-model stub.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <fstream>
#include <set>
#include <sstream>
#include <unordered_map>
#include <unordered_set>

#include <json.hpp>

#include "kvrail/device_step.hpp"
#include "kvrail/scenario.hpp"

namespace kvrail {

using ojson = nlohmann::ordered_json;

namespace {

uint64_t mix64(uint64_t x) { // splitmix64 finaliser (scenario.cpp:34-39)
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

constexpr uint64_t kSummaryTok = 1ull << 40; // summary slots live outside token space

/// The measured device part of a step record.
void fill_device(StepRecord &r, const DeviceStepStats &ds) {
    r.device_ms = ds.device_ms;
    r.gather_ms = ds.gather_ms;
    r.attn_ms = ds.attn_ms;
    std::copy(ds.phase_ms, ds.phase_ms + 8, r.phase_ms);
    r.writeback_tokens = ds.writeback_tokens;
    r.gather_bytes = ds.train_bytes;
    r.attn_bytes = ds.attn_bytes;
    r.h2d_bytes = ds.h2d_bytes;
    r.end_ns = ds.end_ns;
    r.global_live = uint64_t(ds.global_counts[KVR_COUNT_LIVE]);
    r.global_emitted = uint64_t(ds.global_counts[KVR_COUNT_EMITTED]);
    r.global_commits = uint64_t(ds.global_counts[KVR_COUNT_COMMITS]);
    r.global_eos = uint64_t(ds.global_counts[KVR_COUNT_EOS]);
    // the single-commit audit over every GPU of the job (sim_engine.cpp:41-44): the
    // commit frames of all ranks equal their live sessions
    if (r.global_commits != r.global_live)
        raise(Errc::multi_commit, "step " + std::to_string(r.step) + " saw " + std::to_string(r.global_commits) +
                                      " commits for " + std::to_string(r.global_live) +
                                      " live sessions across the job");
}
constexpr SessionId kHolder = 0x7fffffff;

struct Fnv {
    uint64_t h = 1469598103934665603ull;
    void byte(uint8_t b) {
        h ^= b;
        h *= 1099511628211ull;
    }
    void word(uint64_t v) {
        for (int i = 0; i < 64; i += 8)
            byte(uint8_t(v >> i));
    }
};

int elem_kind_of(const ScenarioConfig &c) {
    const std::string &d = c.b200.dtype;
    if (d == "fp32")
        return KVR_ELEM_F32;
    if (d == "bf16")
        return KVR_ELEM_BF16;
    if (d == "fp16")
        return KVR_ELEM_F16;
    return c.pager.elem_bytes == 4 ? KVR_ELEM_F32 : KVR_ELEM_F16;
}

uint16_t to_half(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u, a = x & 0x7fffffffu;
    if (a >= 0x7f800000u)
        return uint16_t(sign | 0x7c00u | (a > 0x7f800000u ? 0x200u : 0u));
    if (a >= 0x477ff000u)
        return uint16_t(sign | 0x7c00u);
    if (a < 0x38800000u) {
        if (a < 0x33000000u)
            return uint16_t(sign);
        const uint32_t e = a >> 23, m = (a & 0x7fffffu) | 0x800000u, sh = 126 - e;
        uint32_t q = m >> sh;
        const uint32_t rem = m & ((1u << sh) - 1u), half = 1u << (sh - 1);
        if (rem > half || (rem == half && (q & 1u)))
            ++q;
        return uint16_t(sign | q);
    }
    uint32_t q = a - 0x38000000u;
    const uint32_t rem = q & 0x1fffu;
    q >>= 13;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u)))
        ++q;
    return uint16_t(sign | q);
}

uint16_t to_bf16(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    if ((x & 0x7fffffffu) > 0x7f800000u)
        return uint16_t((x >> 16) | 0x40u);
    return uint16_t((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
}

} // namespace

void ScenarioConfig::validate() const {
    pager.validate();
    placement.validate();
    transport.validate();
    far_view.validate();
    cost.validate();
    if (workload.has_value() == trace_path.has_value())
        raise(Errc::bad_config, "exactly one of workload spec or trace path must be set");
    if (steps == 0)
        raise(Errc::bad_config, "steps must be positive");
    if (span_blocks == 0 || staged_refresh_period == 0 || demand_refresh_period == 0)
        raise(Errc::bad_config, "transport shaping parameters must be positive");
    if (far_view.enabled) {
        if (!pager_enabled)
            raise(Errc::bad_config, "far view requires the pager");
        // The reference requires float32 lanes; on the B200 bf16/fp16 summaries
        // are defined as the fp32 mean rounded to nearest even.
        if (pager.elem_bytes != 4 && b200.device < 0)
            raise(Errc::bad_config, "far view requires float32 KV elements");
        if (far_view.chunk_tokens % pager.tokens_per_page() != 0)
            raise(Errc::bad_config, "chunk_tokens must be a multiple of tokens_per_page");
    }
    if (shared_prefix_tokens % pager.tokens_per_page() != 0)
        raise(Errc::bad_config, "shared_prefix_tokens must be block aligned");
    if (eos_burst_fraction < 0.0 || eos_burst_fraction > 1.0)
        raise(Errc::bad_config, "eos_burst_fraction must be in [0,1]");
    if (b200.payload != "bytes" && b200.payload != "lanes" && b200.payload != "wide")
        raise(Errc::bad_config, "b200.payload must be 'bytes', 'lanes' or 'wide'");
    if (b200.query != "exact" && b200.query != "f32")
        raise(Errc::bad_config, "b200.query must be 'exact' or 'f32'");
    if (b200.transfer != "reference" && b200.transfer != "page_runs")
        raise(Errc::bad_config, "b200.transfer must be 'reference' or 'page_runs'");
}

std::vector<TraceEvent> resolve_events(const ScenarioConfig &cfg) {
    if (cfg.workload) {
        std::vector<TraceEvent> ev = generate(*cfg.workload);
        const WorkloadAudit a = audit_workload(ev, *cfg.workload);
        if (!a.pass())
            raise(Errc::workload_audit_failed,
                  "generated workload missed its targets (p50/p90/p99 = " + std::to_string(a.p50) +
                      "/" + std::to_string(a.p90) + "/" + std::to_string(a.p99) +
                      ", top-decile share = " + std::to_string(a.top_decile_share) + ")");
        return ev;
    }
    std::vector<TraceEvent> ev = load_trace(*cfg.trace_path);
    if (cfg.replay_window_seconds > 0.0)
        ev = select_window(ev, cfg.replay_window_seconds);
    if (!ev.empty()) {
        const uint64_t t0 = ev.front().arrival_ms;
        for (TraceEvent &e : ev)
            e.arrival_ms -= t0;
    }
    return ev;
}

std::vector<TraceEvent> shard_events(const std::vector<TraceEvent> &events, uint32_t rank,
                                     uint32_t world) {
    if (world <= 1)
        return events;
    if (rank >= world)
        raise(Errc::bad_config, "shard rank out of range");
    // A shard is the trace replay of its sub-stream: ids renumbered, arrivals
    // rebased to the shard's first request (resolve_events, scenario.cpp:86-90).
    std::vector<TraceEvent> out;
    for (const TraceEvent &e : events)
        if (e.request_id % world == rank) {
            out.push_back(e);
            out.back().request_id = out.size() - 1;
        }
    if (!out.empty()) {
        const uint64_t t0 = out.front().arrival_ms;
        for (TraceEvent &e : out)
            e.arrival_ms -= t0;
    }
    return out;
}

// ---------------------------------------------------------------------------

struct ScenarioDriver::Impl {
    struct Req { // one admitted request (reference: Sess, scenario.cpp:100-122)
        SessionId id = 0;
        uint32_t slot = 0;
        uint32_t prompt = 0;
        uint32_t target = 0;
        uint64_t written = 0;
        uint64_t reserved_end = 0;
        std::vector<BlockId> span;      // current span
        uint64_t span_first = 0;        // first token of `span`
        std::vector<BlockId> next_span; // prefetched span
        uint64_t next_span_end = 0;
        bool eos = false;
        Step local_step = 0;
        uint64_t summarized_until = 0;
        uint32_t n_summaries = 0;
        uint32_t summary_room = 0;
        std::vector<BlockId> summary_blocks;
        std::vector<double> chunk_scores;
        std::deque<std::pair<uint64_t, BlockId>> ledger; // (first token, block)
        uint64_t write_begin = 0; // device: first token written at admission
        bool admitted_now = false;
    };
    struct Cold {
        SessionId sid;
        TokenRange range;
    };

    ScenarioConfig cfg;
    std::vector<TraceEvent> events;
    uint32_t tpp;
    SimEngine engine;
    uint32_t width = 64;
    uint32_t span_tokens = 0;
    int ekind = KVR_ELEM_F16;
    bool lanes_payload = false;
    uint32_t lane_shift = 7; // 2-byte lanes: (b - 128) / 2^lane_shift
    std::vector<uint32_t> chunk_slots; // summarize(): a far chunk's rows (global slots)
    std::vector<uint32_t> prime_slots; // device_step(): rows K-prime copies (global slots)

    std::unique_ptr<DeviceStep> dev;
    std::unique_ptr<Pager> pager;
    std::unique_ptr<UtilityTracker> tracker;
    std::vector<BlockId> template_blocks;
    bool holder_active = false;
    SessionId next_id = 1;

    std::vector<Req> live;
    std::vector<int> slot_of; // slot -> index into live, -1 when empty
    std::set<uint32_t> free_slots;
    size_t next_event = 0;
    bool admission_halted = false;
    bool measured_utility = false; // b200.utility = attention: K-mass observations
    uint64_t commits_before = 0;
    uint32_t static_slot_blocks = 0;
    uint64_t static_arena_pages = 0;
    std::unordered_map<BlockId, Cold> cold_pool;

    Step t = 0;
    std::vector<StepRecord> records;
    std::string trace;
    uint64_t staged_rows_window = 0, staged_rows_behind = 0, staged_rows_missing = 0; // device trace coverage
    std::vector<StageNeed> traced_needs;
    std::vector<std::byte> buf;

    Impl(const ScenarioConfig &c, std::vector<TraceEvent> ev)
        : cfg(c), events(std::move(ev)), tpp(c.pager.tokens_per_page()),
          engine(c.cost, c.compiled_width()) {
        width = cfg.workload ? cfg.workload->concurrency : 64;
        span_tokens = cfg.span_blocks * tpp;
        ekind = elem_kind_of(cfg);
        lanes_payload = cfg.b200.payload == "lanes" || cfg.b200.payload == "wide";
        lane_shift = cfg.b200.payload == "wide" ? 3 : 7;
        if (cfg.b200.transfer == "page_runs") { // B200 transfer policy (transport.hpp abuts())
            cfg.transport.run_page_bytes = cfg.pager.page_bytes;
            cfg.transport.run_span_bytes = uint64_t(tpp) * cfg.pager.token_bytes();
        }

        buf.resize(cfg.pager.token_bytes());
        if (cfg.pager_enabled)
            setup_paged();
        else
            setup_static();
        slot_of.assign(width, -1);
        for (uint32_t i = 0; i < width; ++i)
            free_slots.insert(i);
    }

    // ---- synthetic payload (reference: payload_pattern / fill_token_payload) ----
    uint64_t pattern(SessionId id, uint64_t tok, uint64_t lane) const {
        return mix64(cfg.seed ^ (uint64_t(id) << 32) ^ (tok << 8) ^ lane);
    }
    void fill(SessionId id, uint64_t tok, std::byte *out) const {
        const uint64_t tb = cfg.pager.token_bytes();
        if (cfg.pager.elem_bytes == 4 || lanes_payload) {
            const uint64_t lanes = tb / cfg.pager.elem_bytes;
            for (uint64_t l = 0; l < lanes; ++l) {
                if (cfg.pager.elem_bytes == 4) { // reference float pattern
                    const float v = float(int64_t(pattern(id, tok, l) % 2001) - 1000) / 1000.0f;
                    std::memcpy(out + 4 * l, &v, 4);
                } else { // 2-byte lanes: byte l % 8 of one splitmix per 8 lanes
                    const uint64_t x = pattern(id, tok, (l >> 3) ^ 0x4000000000000000ull);
                    const uint32_t r = uint32_t((x >> (8 * (l & 7))) & 0xffu);
                    const float v = float(int(r) - 128) / float(1u << lane_shift);
                    const uint16_t h = ekind == KVR_ELEM_BF16 ? to_bf16(v) : to_half(v);
                    std::memcpy(out + 2 * l, &h, 2);
                }
            }
        } else {
            for (uint64_t i = 0; i < tb; ++i)
                out[i] = std::byte(pattern(id, tok, i) & 0xff);
        }
    }
    void write_token(SessionId id, uint64_t tok) {
        if (dev) {
            pager->write_tokens_generated(id, {tok, tok + 1});
        } else {
            fill(id, tok, buf.data());
            pager->write_tokens(id, {tok, tok + 1}, buf);
        }
    }

    uint32_t arena_pages() const {
        if (cfg.arena_pages_override)
            return *cfg.arena_pages_override;
        const uint64_t per_tokens = cfg.far_view.enabled ? cfg.far_view.near_window +
                                                               2ull * cfg.far_view.chunk_tokens +
                                                               cfg.far_view.cap
                                                         : 384 + 1024;
        const uint64_t per_blocks = (per_tokens + tpp - 1) / tpp + 2ull * cfg.span_blocks;
        const uint64_t want = width * per_blocks + cfg.arena_headroom_pages;
        return uint32_t(std::ceil(double(want) / regime_free_fraction(cfg.regime)));
    }

    kvr_geometry geometry(uint32_t pages) const {
        kvr_geometry g{};
        const B200Config &b = cfg.b200;
        g.device = b.device;
        g.elem_kind = ekind;
        g.elem_bytes = cfg.pager.elem_bytes;
        g.payload_mode = lanes_payload ? KVR_PAYLOAD_LANES : KVR_PAYLOAD_BYTES;
        g.lane_shift = lane_shift;
        g.query_mode = cfg.b200.query == "f32" ? KVR_QUERY_F32 : KVR_QUERY_EXACT;
        g.page_bytes = cfg.pager.page_bytes;
        g.token_bytes = cfg.pager.token_bytes();
        g.arena_pages = pages;
        g.tokens_per_page = tpp;
        g.layers = cfg.pager.layers;
        g.kv_heads = b.kv_heads ? b.kv_heads : 1;
        g.head_dim = b.head_dim ? b.head_dim : cfg.pager.kv_head_dim / g.kv_heads;
        g.q_heads = b.q_heads ? b.q_heads : g.kv_heads;
        if (g.kv_heads * g.head_dim != cfg.pager.kv_head_dim)
            raise(Errc::bad_config, "b200.kv_heads * b200.head_dim must equal pager.kv_head_dim");
        if (g.head_dim < 8 || (g.head_dim & (g.head_dim - 1)))
            raise(Errc::bad_config, "b200.head_dim must be a power of two >= 8");
        if (g.q_heads % g.kv_heads)
            raise(Errc::bad_config, "b200.q_heads must be a multiple of b200.kv_heads");
        g.n_slots = width;
        g.near_window = cfg.far_view.near_window;
        const uint32_t need_rows = cfg.far_view.near_window + span_tokens + 32;
        g.ring_rows = b.ring_rows ? b.ring_rows : (need_rows + 31) / 32 * 32;
        if (g.ring_rows < need_rows || g.ring_rows % 32)
            raise(Errc::bad_config,
                  "b200.ring_rows must be a multiple of 32 covering W* + the staged span + 32 rows");
        g.far_cap = cfg.far_view.enabled ? cfg.far_view.cap : 0;
        g.chunk_tokens = cfg.far_view.chunk_tokens;
        if (cfg.far_view.enabled && g.chunk_tokens > 512)
            raise(Errc::bad_config, "b200 far view: sv_chunk must be <= 512 tokens");
        if (g.token_bytes % 16)
            raise(Errc::bad_config, "b200: token_bytes must be a multiple of 16");
        uint64_t max_tok = b.max_tokens;
        if (!max_tok) {
            uint32_t pmax = 1;
            uint64_t gmax = 1;
            for (const TraceEvent &e : events) {
                pmax = std::max(pmax, e.prompt_tokens);
                gmax = std::max<uint64_t>(gmax, e.generate_tokens);
            }
            max_tok = pmax + gmax + 2ull * span_tokens + cfg.shared_prefix_tokens + 64;
        }
        g.max_tokens = max_tok;
        g.max_chunks = cfg.far_view.enabled ? uint32_t(max_tok / cfg.far_view.chunk_tokens + 2) : 1;
        g.seed = cfg.seed;
        g.attention = !b.attention                           ? 0
                      : b.attention_kernel == "cuda_core" ? 2
                      : b.attention_kernel == "tcgen05"   ? 3
                                                          : 1;
        if (b.attention_kernel != "auto" && b.attention_kernel != "cuda_core" && b.attention_kernel != "tcgen05")
            raise(Errc::bad_config, "b200.attention_kernel must be auto, cuda_core or tcgen05");
        g.use_graph = b.graph;
        if (b.utility != "synthetic" && b.utility != "attention")
            raise(Errc::bad_config, "b200.utility must be synthetic or attention");
        if (b.utility_every == 0)
            raise(Errc::bad_config, "b200.utility_every must be >= 1");
        g.utility = b.utility == "attention" ? b.utility_every : 0;
        g.utility_layer = b.utility_layer < 0 ? g.layers - 1 : uint32_t(b.utility_layer);
        if (g.utility && (!b.attention || g.utility_layer >= g.layers))
            raise(Errc::bad_config, "b200.utility = attention needs the attention and utility_layer < layers");
        g.max_desc_bytes = 0;
        g.max_scan_descs = 0;
        g.max_trains = 0;
        return g;
    }

    void setup_paged() {
        if (cfg.b200.utility_every == 0)
            raise(Errc::bad_config, "b200.utility_every must be >= 1");
        PagerConfig pc = cfg.pager;
        pc.arena_pages = arena_pages();
        if (cfg.b200.device >= 0) {
            dev = std::make_unique<DeviceStep>(geometry(pc.arena_pages));
            dev->set_prefill_budget(cfg.b200.prefill_budget);
            measured_utility = cfg.b200.utility == "attention";
            pager = std::make_unique<Pager>(pc, dev->store());
        } else {
            if (cfg.b200.utility != "synthetic")
                raise(Errc::bad_config, "b200.utility = attention needs a device (b200.device >= 0)");
            pager = std::make_unique<Pager>(pc);
        }
        tracker = std::make_unique<UtilityTracker>(cfg.placement.alpha);

        // A holder session pins the fragmentation regime's pages until warm-up ends.
        const std::vector<uint32_t> held = fragmentation_preset(cfg.regime, pc.arena_pages, cfg.seed);
        if (!held.empty()) {
            holder_active = true;
            pager->create_session(kHolder);
            pager->reserve(kHolder, uint64_t(pc.arena_pages) * tpp);
            std::vector<uint8_t> keep(pc.arena_pages, 0);
            for (uint32_t b : held)
                keep[b] = 1;
            std::vector<TokenRange> frees;
            for (uint32_t b = 0; b < pc.arena_pages; ++b) {
                if (keep[b])
                    continue;
                const uint64_t lo = uint64_t(b) * tpp;
                if (!frees.empty() && frees.back().end == lo)
                    frees.back().end += tpp;
                else
                    frees.push_back({lo, lo + tpp});
            }
            pager->trim(kHolder, frees);
            pager->frame_commit(kHolder, 0);
        }
        // Shared-prefix template session 0.
        pager->create_session(0);
        for (const ReservedBlock &rb : pager->reserve(0, cfg.shared_prefix_tokens))
            template_blocks.push_back(rb.block);
        for (uint64_t tok = 0; tok < cfg.shared_prefix_tokens; ++tok)
            write_token(0, tok);
        pager->frame_commit(0, 0);
        commits_before = pager->counters().commits;
    }

    void setup_static() {
        static_slot_blocks = (cfg.static_slot_tokens + tpp - 1) / tpp;
        static_arena_pages = uint64_t(width) * static_slot_blocks;
    }

    // ---- admission (reference: admit_one / admissions, scenario.cpp:279-360) ----
    bool admit(const TraceEvent &e) {
        if (free_slots.empty())
            return false;
        const uint32_t slot = *free_slots.begin();
        Req r;
        r.id = next_id++;
        r.slot = slot;
        r.prompt = e.prompt_tokens;
        r.target = e.generate_tokens;
        if (!cfg.pager_enabled) {
            const uint32_t cap = static_slot_blocks * tpp;
            if (r.prompt >= cap)
                r.prompt = cap - 1;
            if (r.prompt + r.target > cap)
                r.target = cap - r.prompt;
            r.written = r.prompt;
            r.reserved_end = cap;
        } else {
            pager->create_session(r.id);
            const uint64_t coin = mix64(cfg.seed ^ (0xabcdull << 32) ^ r.id);
            const bool share = coin % 1000 < uint64_t(cfg.share_probability * 1000) &&
                               r.prompt > cfg.shared_prefix_tokens;
            uint64_t start = 0;
            if (share) {
                pager->alias(r.id, 0, cfg.shared_prefix_tokens);
                start = cfg.shared_prefix_tokens;
                for (size_t i = 0; i < template_blocks.size(); ++i)
                    r.ledger.emplace_back(uint64_t(i) * tpp, template_blocks[i]);
            }
            const uint64_t need = r.prompt + 1 - start;
            const uint64_t rounded = (need + span_tokens - 1) / span_tokens * span_tokens;
            std::vector<ReservedBlock> got;
            try {
                got = pager->reserve(r.id, rounded);
            } catch (const Error &err) {
                if (err.code() != Errc::out_of_pages)
                    throw;
                pager->trim_eos(r.id); // reject; retry the event on a later step
                pager->frame_commit(r.id, 0);
                return false;
            }
            uint64_t pos = start;
            for (const ReservedBlock &b : got) {
                r.ledger.emplace_back(pos, b.block);
                pos += b.token_capacity;
            }
            r.reserved_end = start + rounded;
            const size_t nspan = std::min<size_t>(cfg.span_blocks, got.size());
            for (size_t i = got.size() - nspan; i < got.size(); ++i)
                r.span.push_back(got[i].block);
            r.span_first = r.reserved_end - nspan * tpp;
            if (dev)
                dev->bind(r.id, slot);
            // The reference writes the prompt token by token (scenario.cpp:336-340);
            // one range write makes the same coverage checks and COWs in the same
            // block order (and the pager counts no writes), so the device path
            // issues it at once.
            if (dev && start < r.prompt)
                pager->write_tokens_generated(r.id, {start, r.prompt});
            else
                for (uint64_t tok = start; tok < r.prompt; ++tok)
                    write_token(r.id, tok);
            r.written = r.prompt;
            r.write_begin = start;
            r.admitted_now = true;
        }
        slot_of[slot] = int(live.size());
        free_slots.erase(free_slots.begin());
        live.push_back(std::move(r));
        return true;
    }

    void admissions() {
        if (admission_halted)
            return;
        const double now_ms = double(t + 1) * cfg.step_ms;
        while (next_event < events.size() && live.size() < width &&
               double(events[next_event].arrival_ms) <= now_ms) {
            if (!admit(events[next_event]))
                break;
            ++next_event;
        }
    }

    // ---- spans (scenario.cpp:364-381) ----
    void prefetch_span(Req &r) {
        const auto got = pager->reserve(r.id, span_tokens);
        r.next_span.clear();
        uint64_t pos = r.reserved_end;
        for (const ReservedBlock &b : got) {
            r.next_span.push_back(b.block);
            r.ledger.emplace_back(pos, b.block);
            pos += b.token_capacity;
        }
        r.next_span_end = r.reserved_end + span_tokens;
    }
    void promote_span(Req &r) {
        r.span = r.next_span;
        r.span_first = r.reserved_end;
        r.next_span.clear();
        r.reserved_end = r.next_span_end;
    }

    // ---- far view (scenario.cpp:385-446) ----
    void summarize(Req &r, std::vector<StageNeed> &far_needs) {
        const FarViewConfig &fv = cfg.far_view;
        if (!fv.enabled || r.local_step == 0)
            return;
        const uint64_t near_begin = r.written > fv.near_window ? r.written - fv.near_window : 0;
        if (near_begin < r.summarized_until + fv.chunk_tokens)
            return;
        // The committed view cannot change inside this loop (reserve_range and the
        // summary writes touch the shadow only), so it is read once.
        const ViewDescriptor view = pager->active_view(r.id);
        while (near_begin >= r.summarized_until + fv.chunk_tokens) {
            const uint64_t lo = r.summarized_until, hi = lo + fv.chunk_tokens;
            const uint32_t lanes = uint32_t(cfg.pager.token_bytes() / 4);
            double score = 0.0;
            std::vector<float> chunk;
            if (!dev)
                chunk.resize(size_t(fv.chunk_tokens) * lanes);
            // Same per-token additions as the reference (bit-identical sum); the
            // entry walk and the per-block score lookup are cached across tokens.
            const ViewEntry *e = nullptr;
            BlockId scored = kInvalidBlock;
            double block_score = 0.0;
            chunk_slots.clear();
            for (uint64_t tok = lo; tok < hi; ++tok) {
                if (!e || tok < e->tokens.begin || tok >= e->tokens.end)
                    e = view.find(tok);
                if (!e)
                    raise(Errc::unmapped_range, "chunk source token unmapped");
                if (dev) // K-far reads the chunk's rows from this list, not the page table
                    chunk_slots.push_back(e->block * tpp + e->slot_begin + uint32_t(tok - e->tokens.begin));
                if (!dev)
                    pager->read_slots(e->block, e->slot_begin + uint32_t(tok - e->tokens.begin), 1,
                                      reinterpret_cast<std::byte *>(chunk.data() + (tok - lo) * lanes));
                if (e->block != scored) {
                    scored = e->block;
                    block_score = tracker->score(scored, t);
                }
                score += block_score;
            }
            r.chunk_scores.push_back(score);
            if (r.n_summaries == r.summary_room) {
                const auto got = pager->reserve_range(
                    r.id, {kSummaryTok + r.summary_room, kSummaryTok + r.summary_room + tpp});
                r.summary_room += tpp;
                for (const ReservedBlock &b : got)
                    r.summary_blocks.push_back(b.block);
            }
            const uint64_t slot_tok = kSummaryTok + r.n_summaries;
            if (dev) {
                pager->write_tokens_generated(r.id, {slot_tok, slot_tok + 1}, 1, lo, chunk_slots);
            } else {
                const std::vector<float> mean = summarize_chunk(chunk, lanes, fv.chunk_tokens);
                pager->write_tokens(r.id, {slot_tok, slot_tok + 1},
                                    std::as_bytes(std::span<const float>(mean)));
            }
            StageNeed need;
            need.session = r.id;
            need.kind = TrainKind::far_view;
            need.spans.push_back({r.summary_blocks[r.n_summaries / tpp], r.n_summaries % tpp, 1});
            far_needs.push_back(std::move(need));
            ++r.n_summaries;
            r.summarized_until = hi;
            // blocks wholly behind the summarized boundary become cold candidates
            while (!r.ledger.empty() && r.ledger.front().first + tpp <= r.summarized_until) {
                cold_pool[r.ledger.front().second] =
                    Cold{r.id, {r.ledger.front().first, r.ledger.front().first + tpp}};
                r.ledger.pop_front();
            }
        }
    }

    // ---- the step (scenario.cpp:450-682) ----
    // Host time per step section (KVR_HOST_PROFILE=1: printed when the driver ends).
    struct HostProfile {
        bool on = std::getenv("KVR_HOST_PROFILE") != nullptr;
        double ms[8] = {};
        std::chrono::steady_clock::time_point t0;
        void start() {
            if (on)
                t0 = std::chrono::steady_clock::now();
        }
        void lap(int i) {
            if (!on)
                return;
            const auto t1 = std::chrono::steady_clock::now();
            ms[i] += std::chrono::duration<double, std::milli>(t1 - t0).count();
            t0 = t1;
        }
        ~HostProfile() {
            if (on)
                std::fprintf(stderr,
                             "host ms: retire %.1f admit %.1f sessions %.1f placement %.1f commit %.1f "
                             "stage %.1f device %.1f trace/engine %.1f\n",
                             ms[0], ms[1], ms[2], ms[3], ms[4], ms[5], ms[6], ms[7]);
        }
    } prof;

    StepRecord step() {
        prof.start();
        // Shift: retire sessions that finished last step (swap-remove).
        for (size_t i = 0; i < live.size();) {
            if (!live[i].eos) {
                ++i;
                continue;
            }
            const SessionId dead = live[i].id;
            for (auto it = cold_pool.begin(); it != cold_pool.end();)
                it = it->second.sid == dead ? cold_pool.erase(it) : std::next(it);
            free_slots.insert(live[i].slot);
            slot_of[live[i].slot] = -1;
            if (dev)
                dev->unbind(dead);
            if (i + 1 != live.size()) {
                live[i] = std::move(live.back());
                slot_of[live[i].slot] = int(i);
            }
            live.pop_back();
        }
        if (holder_active && t == cfg.warmup_steps) {
            pager->trim_eos(kHolder);
            pager->frame_commit(kHolder, 1);
            commits_before = pager->counters().commits;
            holder_active = false;
        }
        if (cfg.eos_burst_step > 0 && t == cfg.eos_burst_step) {
            uint64_t left = uint64_t(std::llround(live.size() * cfg.eos_burst_fraction));
            for (size_t i = 0; i < live.size() && left > 0; i += 2, --left)
                live[i].target = uint32_t(live[i].written - live[i].prompt) + 1;
            admission_halted = true;
        }
        for (Req &r : live)
            r.admitted_now = false;
        prof.lap(0);
        admissions();
        prof.lap(1);

        std::vector<StageNeed> far_needs;
        std::vector<std::pair<BlockId, double>> obs;
        uint64_t emitted = 0, eos_now = 0;
        std::vector<size_t> order;
        for (uint32_t s = 0; s < width; ++s)
            if (slot_of[s] >= 0)
                order.push_back(size_t(slot_of[s]));

        for (size_t idx : order) {
            Req &r = live[idx];
            if (cfg.pager_enabled) {
                while (r.written == r.reserved_end) {
                    if (!r.next_span.empty()) {
                        promote_span(r);
                        continue;
                    }
                    const auto got = pager->reserve(r.id, span_tokens);
                    r.span.clear();
                    r.span_first = r.reserved_end;
                    uint64_t pos = r.reserved_end;
                    for (const ReservedBlock &b : got) {
                        r.span.push_back(b.block);
                        r.ledger.emplace_back(pos, b.block);
                        pos += b.token_capacity;
                    }
                    r.reserved_end += span_tokens;
                }
                write_token(r.id, r.written);
            }
            ++r.written;
            ++emitted;
            if (!r.span.empty() && !measured_utility)
                obs.emplace_back(r.span.back(),
                                 1.0 + double(pattern(r.id, r.written, 7) % 997) / 4000.0);
            if (r.written - r.prompt >= r.target) {
                if (cfg.pager_enabled)
                    pager->trim_eos(r.id);
                r.eos = true;
                ++eos_now;
            } else if (cfg.pager_enabled) {
                summarize(r, far_needs);
                if (r.reserved_end - r.written <= 1 && r.next_span.empty())
                    prefetch_span(r);
            }
        }

        prof.lap(2);
        if (measured_utility && t >= 2 && dev->launched(t - 2) && (t - 2) % cfg.b200.utility_every == 0) {
            // attention-utility observations measured by K-mass two steps back (the
            // newest step the device has finished), for sessions still decoding; steps
            // K-mass skips (utility_every) bring no observations
            std::unordered_set<SessionId> decoding;
            for (const Req &r : live)
                if (!r.eos)
                    decoding.insert(r.id);
            obs = dev->utility(t - 2, [&](SessionId s) { return decoding.count(s) > 0; });
        }
        // Placement: rank staging candidates and take the cold set.
        std::vector<size_t> refresh;
        const uint32_t period = cfg.pager_enabled ? cfg.staged_refresh_period
                                                  : cfg.demand_refresh_period;
        for (uint32_t s = 0; s < width; ++s)
            if (slot_of[s] >= 0 && (s + t) % period == 0 && !live[slot_of[s]].eos)
                refresh.push_back(size_t(slot_of[s]));
        if (cfg.pager_enabled) {
            std::vector<BlockId> cands;
            for (size_t idx : refresh)
                cands.insert(cands.end(), live[idx].span.begin(), live[idx].span.end());
            std::vector<SessionBlockState> states;
            if (cfg.far_view.enabled && !cold_pool.empty()) {
                SessionBlockState st;
                for (const auto &kv : cold_pool)
                    st.live_blocks.push_back(kv.first);
                std::sort(st.live_blocks.begin(), st.live_blocks.end());
                states.push_back(std::move(st));
            }
            const PlacementPlan plan = plan_step(*tracker, cfg.placement, cands, obs, states, t);
            std::unordered_map<SessionId, bool> alive;
            for (const Req &r : live)
                alive[r.id] = !r.eos;
            std::unordered_map<SessionId, std::vector<TokenRange>> trims;
            for (BlockId b : plan.cold) {
                auto it = cold_pool.find(b);
                if (it == cold_pool.end())
                    continue;
                auto a = alive.find(it->second.sid);
                if (a != alive.end() && a->second)
                    trims[it->second.sid].push_back(it->second.range);
                cold_pool.erase(it);
            }
            for (auto &[sid, ranges] : trims)
                pager->trim(sid, ranges);
        }

        prof.lap(3);
        // One frame commit per live session.
        uint64_t commits = 0;
        if (cfg.pager_enabled) {
            for (size_t idx : order) {
                Req &r = live[idx];
                pager->frame_commit(r.id, r.local_step);
                ++r.local_step;
            }
            const uint64_t now_c = pager->counters().commits;
            commits = now_c - commits_before;
            commits_before = now_c;
        } else {
            commits = order.size();
        }

        prof.lap(4);
        // Stage needs.
        std::vector<StageNeed> needs;
        std::vector<std::vector<uint64_t>> need_first; // device: logical first token per span
        for (size_t idx : refresh) {
            Req &r = live[idx];
            if (r.eos)
                continue;
            StageNeed head;
            head.session = r.id;
            head.kind = TrainKind::near_window;
            if (cfg.pager_enabled) {
                const size_t nspan = r.span.size();
                size_t frontier = 0;
                if (r.written > r.span_first)
                    frontier = std::min(nspan - 1, size_t((r.written - 1 - r.span_first) / tpp));
                const size_t delta_lo = frontier >= 1 ? frontier - 1 : 0;
                StageNeed delta = head, tail = head;
                std::vector<uint64_t> f_head, f_delta, f_tail;
                for (size_t i = 0; i < nspan; ++i) {
                    const uint64_t blk_first = r.span_first + i * tpp;
                    if (cfg.far_view.enabled && blk_first + tpp <= r.summarized_until)
                        continue;
                    const BlockId b = r.span[i];
                    if (cold_pool.count(b))
                        raise(Errc::unmapped_block, "staged block was trimmed in this frame");
                    const bool in_head = i < delta_lo, in_delta = !in_head && i <= frontier;
                    StageNeed &piece = in_head ? head : in_delta ? delta : tail;
                    piece.spans.push_back({b, 0, tpp});
                    (in_head ? f_head : in_delta ? f_delta : f_tail).push_back(blk_first);
                }
                if (!delta.spans.empty()) {
                    needs.push_back(std::move(delta));
                    need_first.push_back(std::move(f_delta));
                }
                if (!tail.spans.empty()) {
                    needs.push_back(std::move(tail));
                    need_first.push_back(std::move(f_tail));
                }
                needs.push_back(std::move(head));
                need_first.push_back(std::move(f_head));
            } else {
                // static slots: the trailing segment is contiguous by layout
                const uint64_t gt = std::min<uint64_t>(cfg.demand_gather_tokens, r.written);
                const uint64_t base = uint64_t(r.slot) * static_slot_blocks;
                std::vector<uint64_t> f;
                for (uint64_t from = r.written - gt; from < r.written;) {
                    const uint32_t sb = uint32_t(from % tpp);
                    const uint32_t n = uint32_t(std::min<uint64_t>(r.written - from, tpp - sb));
                    head.spans.push_back({BlockId(base + from / tpp), sb, n});
                    f.push_back(from);
                    from += n;
                }
                needs.push_back(std::move(head));
                need_first.push_back(std::move(f));
            }
        }
        for (StageNeed &fn : far_needs) {
            std::vector<uint64_t> f;
            for (const StagedSpan &sp : fn.spans)
                (void)sp, f.push_back(0);
            need_first.push_back(std::move(f));
            needs.push_back(std::move(fn));
        }

        const double now = engine.clock();
        if (cfg.b200.trace)
            traced_needs = needs;
        std::vector<Descriptor> descs = stage(needs, cfg.pager.page_bytes, cfg.pager.token_bytes(), now);
        std::vector<DmaTrain> trains = reduce(std::move(descs), cfg.transport, now);

        ArenaStats arena;
        if (cfg.pager_enabled) {
            arena = pager->stats();
        } else {
            arena.reserved_bytes = static_arena_pages * cfg.pager.page_bytes;
            uint64_t mapped = 0;
            for (const Req &r : live)
                mapped += r.eos ? 0 : r.written;
            arena.active_bytes = mapped * cfg.pager.token_bytes();
            arena.free_pages = 0;
            arena.live_pages = static_arena_pages;
        }
        prof.lap(5);
        if (dev) { // publish first: the trace then reads the bytes this step produced
            const int64_t counts[KVR_COUNTS] = {int64_t(order.size()), int64_t(emitted), int64_t(commits),
                                                int64_t(eos_now)};
            dev->counts(counts);
            device_step(needs, need_first, now);
            if (cfg.b200.check)
                check_device_scan(trains);
        }
        prof.lap(6);
        if (cfg.b200.trace)
            trace_step(trains);
        StepRecord rec = engine.execute_step(t, trains, cfg.compiled_width(), uint32_t(order.size()),
                                             commits, emitted, arena);
        ++t;
        prof.lap(7);
        return rec;
    }

    // ---- B200 step publication ----
    void device_step(const std::vector<StageNeed> &needs,
                     const std::vector<std::vector<uint64_t>> &first, double now) {
        for (uint32_t s = 0; s < width; ++s) {
            if (slot_of[s] < 0) {
                dev->slot_state(s, 0, 0, false);
                continue;
            }
            Req &r = live[slot_of[s]];
            dev->slot_state(s, r.id, r.written, true);
            if (r.admitted_now && r.write_begin > 0) {
                // window rows of the aliased prefix come from the shared pages
                const uint64_t lo = r.written > cfg.far_view.near_window
                                        ? r.written - cfg.far_view.near_window
                                        : 0;
                if (lo < r.write_begin) { // aliases the template session 0
                    const ViewDescriptor v = pager->active_view(r.id);
                    prime_slots.clear();
                    for (uint64_t tok = lo; tok < r.write_begin; ++tok) {
                        const ViewEntry *e = v.find(tok);
                        prime_slots.push_back(e ? e->block * tpp + e->slot_begin + uint32_t(tok - e->tokens.begin)
                                                : KVR_NO_SLOT);
                    }
                    dev->prime(s, lo, r.write_begin, 0, prime_slots);
                }
            }
            if (cfg.far_view.enabled && cfg.far_view.cap > 0 && !r.chunk_scores.empty()) {
                const std::vector<uint64_t> pick = select_chunks(r.chunk_scores, cfg.far_view.cap);
                dev->far_selection(s, pick);
            }
        }
        std::unordered_map<SessionId, uint32_t> slot_by_id;
        for (const Req &r : live)
            slot_by_id[r.id] = r.slot;
        for (size_t i = 0; i < needs.size(); ++i) {
            const StageNeed &n = needs[i];
            auto it = slot_by_id.find(n.session);
            std::vector<uint64_t> f = first[i];
            if (n.kind == TrainKind::far_view) {
                // far spans carry their summary index as the logical token
                if (it == slot_by_id.end())
                    raise(Errc::unknown_session, "far-view need of a session without a live slot");
                const Req &r = live[slot_of[it->second]];
                for (size_t k = 0; k < n.spans.size(); ++k) {
                    const StagedSpan &sp = n.spans[k];
                    for (uint32_t j = 0; j < r.summary_blocks.size(); ++j)
                        if (r.summary_blocks[j] == sp.block)
                            f[k] = kSummaryTok + uint64_t(j) * tpp + sp.slot_begin;
                }
            }
            dev->need(it == slot_by_id.end() ? KVR_NO_SLOT : it->second, n.session, n.kind, n.spans, f);
        }
        dev->launch(t, now, cfg.transport);
    }

    // ---- device self-check: K-scan trains must equal the host reduce() ----
    uint64_t checked_steps = 0, scan_mismatches = 0;
    std::string first_mismatch;
    void check_device_scan(const std::vector<DmaTrain> &want) {
        dev->collect(t); // waits for this step
        std::vector<kvr_train> got;
        std::vector<kvr_descriptor> descs;
        dev->read_scan(got, descs);
        ++checked_steps;
        std::string why;
        if (got.size() != want.size())
            why = "train count " + std::to_string(got.size()) + " != " + std::to_string(want.size());
        for (size_t i = 0; why.empty() && i < want.size(); ++i) {
            const kvr_train &g = got[i];
            const DmaTrain &w = want[i];
            if (g.kind != uint32_t(w.kind) || g.reason != uint32_t(w.reason) ||
                g.total_bytes != w.total_bytes || g.desc_count != w.descriptors.size() ||
                g.issue_time != w.issue_time || g.oldest_stage_time != w.oldest_stage_time) {
                why = "train " + std::to_string(i) + " header differs";
                break;
            }
            for (size_t k = 0; k < w.descriptors.size(); ++k) {
                const kvr_descriptor &d = descs[g.desc_begin + k];
                const Descriptor &e = w.descriptors[k];
                if (d.phys_offset != e.phys_offset || d.length != e.length || d.session != e.session ||
                    d.block != e.block || d.kind != uint32_t(e.kind)) {
                    why = "train " + std::to_string(i) + " descriptor " + std::to_string(k) + " differs";
                    break;
                }
            }
        }
        if (!why.empty()) {
            ++scan_mismatches;
            if (first_mismatch.empty())
                first_mismatch = "step " + std::to_string(t) + ": " + why;
        }
    }

    // ---- parity trace (format shared with oracle/ref_shim.cpp) ----
    void trace_step(const std::vector<DmaTrain> &trains) {
        char line[320];
        std::snprintf(line, sizeof(line), "step %llu\n", (unsigned long long)t);
        trace += line;
        for (const StageNeed &n : traced_needs) {
            std::snprintf(line, sizeof(line), "need %u %u %zu", n.session, unsigned(n.kind),
                          n.spans.size());
            trace += line;
            for (const StagedSpan &s : n.spans) {
                std::snprintf(line, sizeof(line), " %u:%u:%u", s.block, s.slot_begin, s.slot_count);
                trace += line;
            }
            trace += "\n";
        }
        traced_needs.clear();
        const uint64_t page = cfg.pager.page_bytes, tb = cfg.pager.token_bytes();
        std::vector<std::byte> tok(tb);
        // Device mode: the staged bytes are hashed from K-gather's DESTINATION (the
        // window ring / far rows), in train order, so the trace equals the reference's
        // read_slots hash only if every train landed byte for byte.
        std::vector<uint8_t> staged, in_window;
        uint64_t staged_base = 0;
        if (dev && pager) {
            uint64_t total = 0;
            for (const DmaTrain &tr : trains)
                total += tr.total_bytes / tb;
            staged.resize(total * tb);
            in_window.resize(total);
            dev->read_staged(0, total, staged.data(), in_window.data());
            for (uint8_t w : in_window)
                (w == 1 ? staged_rows_window : w == 0 ? staged_rows_behind : staged_rows_missing) += 1;
        }
        for (const DmaTrain &tr : trains) {
            Fnv f;
            if (pager && dev) {
                const uint64_t n = tr.total_bytes;
                for (uint64_t i = 0; i < n; ++i)
                    f.byte(staged[staged_base + i]);
                staged_base += n;
            } else if (pager)
                for (const Descriptor &d : tr.descriptors)
                    for (uint64_t off = d.phys_offset; off < d.phys_offset + d.length; off += tb) {
                        pager->read_slots(BlockId(off / page), uint32_t((off % page) / tb), 1,
                                          tok.data());
                        for (std::byte b : tok)
                            f.byte(uint8_t(b));
                    }
            std::snprintf(line, sizeof(line), "train %u %u %llu %zu t=%.6f o=%.6f h=%016llx",
                          unsigned(tr.kind), unsigned(tr.reason), (unsigned long long)tr.total_bytes,
                          tr.descriptors.size(), tr.issue_time, tr.oldest_stage_time,
                          (unsigned long long)(pager ? f.h : 0));
            trace += line;
            for (const Descriptor &d : tr.descriptors) {
                std::snprintf(line, sizeof(line), " %llu+%llu@%u", (unsigned long long)d.phys_offset,
                              (unsigned long long)d.length, d.session);
                trace += line;
            }
            trace += "\n";
        }
        if (!pager) {
            trace += "pager none\n";
            return;
        }
        const ArenaStats st = pager->stats();
        Fnv runs, views;
        for (auto [h, n] : pager->free_runs()) {
            runs.word(h);
            runs.word(n);
        }
        uint64_t n_sess = 0;
        auto dump = [&](SessionId id) {
            const ViewDescriptor v = pager->active_view(id);
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
        for (SessionId id = 0; pager->has_session(id); ++id)
            dump(id);
        if (pager->has_session(kHolder))
            dump(kHolder);
        std::snprintf(line, sizeof(line),
                      "pager free=%llu live=%llu shared=%llu reserved=%llu active=%llu runs=%016llx "
                      "views=%016llx sessions=%llu\n",
                      (unsigned long long)st.free_pages, (unsigned long long)st.live_pages,
                      (unsigned long long)st.shared_pages, (unsigned long long)st.reserved_bytes,
                      (unsigned long long)st.active_bytes, (unsigned long long)runs.h,
                      (unsigned long long)views.h, (unsigned long long)n_sess);
        trace += line;
    }
};

ScenarioDriver::ScenarioDriver(const ScenarioConfig &cfg, std::vector<TraceEvent> events) {
    cfg.validate();
    impl_ = std::make_unique<Impl>(cfg, std::move(events));
}
ScenarioDriver::~ScenarioDriver() {
    if (impl_ && impl_->dev)
        impl_->dev->sync();
}

StepRecord ScenarioDriver::step() {
    Impl &m = *impl_;
    StepRecord r = m.step();
    if (m.dev) {
        // Collect the previous step's device record (one step of pipelining).
        if (r.step > 0) {
            const DeviceStepStats ds = m.dev->collect(r.step - 1);
            StepRecord &prev = m.records[r.step - 1];
            fill_device(prev, ds);
        }
        if (m.t >= m.cfg.steps) {
            const DeviceStepStats ds = m.dev->collect(r.step);
            fill_device(r, ds);
        }
    }
    m.records.push_back(r);
    return r;
}

bool ScenarioDriver::done() const { return impl_->t >= impl_->cfg.steps; }

const StepRecord &ScenarioDriver::record(uint64_t step) {
    Impl &m = *impl_;
    if (step >= m.records.size())
        raise(Errc::bad_config, "step " + std::to_string(step) + " has not run");
    StepRecord &r = m.records[step];
    if (m.dev && r.device_ms == 0.0 && m.dev->launched(step)) {
        const DeviceStepStats ds = m.dev->collect(step);
        fill_device(r, ds);
    }
    return r;
}
uint64_t ScenarioDriver::steps_done() const { return impl_->t; }
const ScenarioConfig &ScenarioDriver::config() const { return impl_->cfg; }
const std::vector<StepRecord> &ScenarioDriver::records() const { return impl_->records; }
const std::vector<TraceEvent> &ScenarioDriver::events() const { return impl_->events; }
const std::string &ScenarioDriver::trace() const { return impl_->trace; }
Pager *ScenarioDriver::pager() const { return impl_->pager.get(); }
DeviceStep *ScenarioDriver::device() const { return impl_->dev.get(); }

std::vector<ScenarioDriver::LiveInfo> ScenarioDriver::live() const {
    std::vector<LiveInfo> out;
    for (uint32_t s = 0; s < impl_->width; ++s)
        if (impl_->slot_of[s] >= 0) {
            const auto &r = impl_->live[impl_->slot_of[s]];
            out.push_back({s, r.id, r.written});
        }
    return out;
}

void ScenarioDriver::device_check(uint64_t &checked, uint64_t &mismatches, std::string &first) const {
    checked = impl_->checked_steps;
    mismatches = impl_->scan_mismatches;
    first = impl_->first_mismatch;
}

void ScenarioDriver::staged_rows(uint64_t &delivered, uint64_t &behind, uint64_t &missing) const {
    delivered = impl_->staged_rows_window;
    behind = impl_->staged_rows_behind;
    missing = impl_->staged_rows_missing;
}

void ScenarioDriver::comm_init(const uint8_t id[128], int rank, int world) {
    if (!impl_->dev)
        throw std::runtime_error("comm_init: host-only driver");
    if (impl_->t != 0)
        throw std::runtime_error("comm_init must precede the first step");
    impl_->dev->comm_init(id, rank, world);
}

void ScenarioDriver::fault(int what, uint64_t arg) {
    if (!impl_->dev)
        throw std::runtime_error("fault: host-only driver");
    impl_->dev->fault(what, arg);
}

RunResult ScenarioDriver::result() const {
    const Impl &m = *impl_;
    RunResult res;
    res.config = m.cfg;
    res.records = m.records;
    if (m.pager)
        res.pager_counters = m.pager->counters();
    res.report = aggregate(res.records, m.cfg.warmup_steps);
    res.report.label = m.cfg.label;
    res.report.seed = m.cfg.seed;
    res.report.workload_hash = stream_hash(m.events);
    if (m.cfg.workload)
        res.workload_audit = audit_workload(m.events, *m.cfg.workload);
    return res;
}

RunResult run_scenario_on(const ScenarioConfig &cfg, const std::vector<TraceEvent> &events) {
    // Drop-in callers of the reference API (run_scenario, the reference's own
    // acceptance suite) select the B200 path with KVRAIL_B200_DEVICE=<cuda device>
    // when their config does not name one (b200.device < 0, the reference's default).
    ScenarioConfig c = cfg;
    if (c.b200.device < 0)
        if (const char *e = std::getenv("KVRAIL_B200_DEVICE"); e && *e)
            c.b200.device = std::atoi(e);
    ScenarioDriver d(c, events);
    while (!d.done())
        d.step();
    return d.result();
}

RunResult run_scenario(const ScenarioConfig &cfg) {
    cfg.validate();
    return run_scenario_on(cfg, resolve_events(cfg));
}

// ---------------------------------------------------------------------------
// reports (formats of scenario.cpp:706-817)

std::string steps_to_csv(const std::vector<StepRecord> &records) {
    std::string out =
        "step,live_sessions,trains,near_trains,far_trains,dma_bytes,mean_train_bytes,"
        "max_hold,submit_time,commit_time,step_latency,reserved_bytes,active_bytes,"
        "commits,emitted_tokens\n";
    char line[512];
    for (const StepRecord &r : records) {
        std::snprintf(line, sizeof(line),
                      "%llu,%u,%u,%u,%u,%llu,%.3f,%.6f,%.6f,%.6f,%.6f,%llu,%llu,%u,%llu\n",
                      (unsigned long long)r.step, r.live_sessions, r.trains, r.near_trains,
                      r.far_trains, (unsigned long long)r.dma_bytes, r.mean_train_bytes, r.max_hold,
                      r.submit_time, r.commit_time, r.step_latency,
                      (unsigned long long)r.reserved_bytes, (unsigned long long)r.active_bytes,
                      r.commits, (unsigned long long)r.emitted_tokens);
        out += line;
    }
    return out;
}

std::string measured_steps_csv(const std::vector<StepRecord> &records) {
    std::string out = steps_to_csv(records);
    const size_t nl = out.find('\n');
    std::string head = out.substr(0, nl) +
                       ",device_ms,itl_ms,gather_ms,attn_ms,apply_ms,hot_writes_ms,far_map_prime_ms,scan_ms,"
                       "cold_writes_ms,writeback_tokens,gather_bytes,attn_bytes,h2d_bytes\n";
    std::string body;
    size_t pos = nl + 1;
    char line[512];
    for (size_t i = 0; i < records.size(); ++i) {
        const StepRecord &r = records[i];
        const size_t e = out.find('\n', pos);
        body.append(out, pos, e - pos);
        pos = e + 1;
        const double itl = i > 0 && r.end_ns && records[i - 1].end_ns
                               ? double(int64_t(r.end_ns - records[i - 1].end_ns)) / 1e6
                               : 0.0;
        std::snprintf(line, sizeof(line), ",%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%llu,%llu,%llu,%llu\n",
                      r.device_ms, itl, r.gather_ms, r.attn_ms, r.phase_ms[0], r.phase_ms[1], r.phase_ms[2],
                      r.phase_ms[3], r.phase_ms[6], (unsigned long long)r.writeback_tokens,
                      (unsigned long long)r.gather_bytes, (unsigned long long)r.attn_bytes,
                      (unsigned long long)r.h2d_bytes);
        body += line;
    }
    return head + body;
}

std::string measured_report_json(const std::vector<StepRecord> &records, uint64_t warmup_steps) {
    std::vector<double> dev, itl, model;
    double tokens = 0, dev_ms = 0, attn_ms = 0, gather_ms = 0;
    uint64_t attn_bytes = 0, gather_bytes = 0, h2d = 0;
    for (size_t i = warmup_steps; i < records.size(); ++i) {
        const StepRecord &r = records[i];
        if (r.device_ms <= 0.0)
            continue;
        dev.push_back(r.device_ms);
        model.push_back(r.step_latency);
        if (i > 0 && r.end_ns && records[i - 1].end_ns)
            itl.push_back(double(int64_t(r.end_ns - records[i - 1].end_ns)) / 1e6);
        tokens += double(r.emitted_tokens);
        dev_ms += r.device_ms;
        attn_ms += r.attn_ms;
        gather_ms += r.gather_ms;
        attn_bytes += r.attn_bytes;
        gather_bytes += r.gather_bytes;
        h2d += r.h2d_bytes;
    }
    if (dev.empty())
        raise(Errc::empty_run, "no measured post-warm-up steps");
    auto pct = [](const std::vector<double> &v) {
        return ojson{{"p50", percentile_nearest_rank(v, 0.50)},
                     {"p99", percentile_nearest_rank(v, 0.99)},
                     {"p999", percentile_nearest_rank(v, 0.999)}};
    };
    ojson j;
    j["measured_steps"] = dev.size();
    j["decode_tokens_per_s"] = tokens / (dev_ms / 1e3);
    j["device_step_ms"] = pct(dev);
    if (!itl.empty())
        j["inter_token_latency_ms"] = pct(itl);
    j["modeled_step_latency"] = pct(model);
    j["attention_gbs"] = attn_ms > 0 ? double(attn_bytes) / (attn_ms / 1e3) / 1e9 : 0.0;
    j["gather_hbm_gbs"] = gather_ms > 0 ? 2.0 * double(gather_bytes) / (gather_ms / 1e3) / 1e9 : 0.0;
    j["descriptor_h2d_bytes_per_step"] = double(h2d) / double(dev.size());
    return j.dump(1);
}

static ojson report_json(const RunResult &res) {
    const RunReport &r = res.report;
    ojson j;
    j["label"] = r.label;
    j["seed"] = r.seed;
    j["workload_hash"] = r.workload_hash;
    j["post_warmup_steps"] = r.steps;
    j["throughput_tokens_per_unit"] = r.throughput;
    j["latency"] = {{"p50", r.latency_p50}, {"p99", r.latency_p99}, {"p999", r.latency_p999}};
    j["submit_share"] = r.submit_share;
    j["transport"] = {{"trains_per_step", r.trains_per_step},
                      {"mean_train_bytes", r.mean_train_bytes},
                      {"max_hold_observed", r.max_hold_observed}};
    j["memory"] = {{"mean_reserved_bytes", r.mean_reserved_bytes},
                   {"mean_active_bytes", r.mean_active_bytes},
                   {"final_reserved_bytes", r.final_reserved_bytes},
                   {"final_active_bytes", r.final_active_bytes},
                   {"reserved_to_active", r.reserved_to_active}};
    j["live_width"] = {{"mean", r.live_width_mean},
                       {"cv", r.live_width_cv},
                       {"max_to_mean", r.live_width_max_to_mean}};
    j["invariant_audit"] = {{"commit_steps", r.total_commit_steps},
                            {"multi_commit_steps", r.multi_commit_steps},
                            {"shape_violations", r.shape_violations},
                            {"recompiles", r.recompiles}};
    if (res.config.workload) {
        const WorkloadAudit &a = res.workload_audit;
        j["workload_audit"] = {{"p50", a.p50},
                               {"p90", a.p90},
                               {"p99", a.p99},
                               {"top_decile_share", a.top_decile_share},
                               {"eos_window_p50", a.eos_window_p50},
                               {"eos_window_p90", a.eos_window_p90},
                               {"eos_window_p99", a.eos_window_p99},
                               {"pass", a.pass()}};
    }
    return j;
}

std::string report_to_json(const RunResult &res) { return report_json(res).dump(2) + "\n"; }

std::string report_to_text(const RunResult &res) {
    const RunReport &r = res.report;
    std::ostringstream out;
    char line[256];
    out << "run " << r.label << " (seed " << r.seed << ", " << r.steps << " steady steps)\n";
    auto row = [&](const char *name, double v, const char *unit) {
        std::snprintf(line, sizeof(line), "  %-24s %14.4f %s\n", name, v, unit);
        out << line;
    };
    row("throughput", r.throughput, "tok/unit");
    row("latency p50", r.latency_p50, "units");
    row("latency p99", r.latency_p99, "units");
    row("latency p99.9", r.latency_p999, "units");
    row("submit share", r.submit_share * 100.0, "%");
    row("trains per step", r.trains_per_step, "");
    row("mean train size", r.mean_train_bytes / 1024.0, "KiB");
    row("reserved (mean)", r.mean_reserved_bytes / (1024.0 * 1024.0), "MiB");
    row("active (mean)", r.mean_active_bytes / (1024.0 * 1024.0), "MiB");
    row("reserved/active", r.reserved_to_active, "");
    row("live width mean", r.live_width_mean, "");
    row("live width cv", r.live_width_cv, "");
    std::snprintf(line, sizeof(line),
                  "  audit: %llu commit steps, %llu multi-commit, %llu shape violations, "
                  "%llu recompiles\n",
                  (unsigned long long)r.total_commit_steps, (unsigned long long)r.multi_commit_steps,
                  (unsigned long long)r.shape_violations, (unsigned long long)r.recompiles);
    out << line;
    return out.str();
}

std::string delta_to_text(const DeltaReport &d) {
    std::ostringstream out;
    out << "compare " << d.label_a << " -> " << d.label_b << "\n";
    char line[256];
    for (const MetricDelta &m : d.deltas) {
        std::snprintf(line, sizeof(line), "  %-24s %14.4f -> %14.4f   (x%.4f)\n", m.name.c_str(), m.a,
                      m.b, m.ratio);
        out << line;
    }
    return out.str();
}

void write_file(const std::string &path, const std::string &content) {
    std::ofstream out(path, std::ios::binary);
    if (!out)
        raise(Errc::io_error, "cannot write " + path);
    out << content;
}

// ---- config JSON (schema of scenario.cpp:821-987, plus "b200") ----

template <typename T> static void take(const ojson &j, const char *k, T &v) {
    if (j.contains(k))
        v = j[k].get<T>();
}

static ScenarioConfig config_from_json(const ojson &j) {
    ScenarioConfig c = default_audit_config();
    take(j, "label", c.label);
    take(j, "seed", c.seed);
    take(j, "steps", c.steps);
    take(j, "warmup_steps", c.warmup_steps);
    take(j, "step_ms", c.step_ms);
    if (j.contains("pager")) {
        const auto &p = j["pager"];
        take(p, "page_bytes", c.pager.page_bytes);
        take(p, "arena_pages", c.pager.arena_pages);
        take(p, "layers", c.pager.layers);
        take(p, "kv_head_dim", c.pager.kv_head_dim);
        take(p, "elem_bytes", c.pager.elem_bytes);
    }
    if (j.contains("placement")) {
        const auto &p = j["placement"];
        take(p, "alpha", c.placement.alpha);
        take(p, "lookahead_budget", c.placement.lookahead_budget);
        take(p, "cold_budget", c.placement.cold_budget);
    }
    if (j.contains("transport")) {
        const auto &p = j["transport"];
        take(p, "tau_bytes", c.transport.merge_threshold);
        take(p, "delta_hold", c.transport.max_hold);
        take(p, "max_trains_per_step", c.transport.max_trains_per_step);
        take(p, "merge", c.transport.merge);
    }
    if (j.contains("far_view")) {
        const auto &p = j["far_view"];
        take(p, "enabled", c.far_view.enabled);
        take(p, "w_star", c.far_view.near_window);
        take(p, "cap", c.far_view.cap);
        take(p, "sv_chunk", c.far_view.chunk_tokens);
    }
    if (j.contains("cost_model")) {
        const auto &p = j["cost_model"];
        take(p, "dma_fixed_overhead", c.cost.dma_fixed_overhead);
        take(p, "dma_bandwidth", c.cost.dma_bandwidth);
        take(p, "kernel_base", c.cost.kernel_base);
        take(p, "kernel_per_slot", c.cost.kernel_per_slot);
        take(p, "submit_cost", c.cost.submit_cost);
        take(p, "commit_cost", c.cost.commit_cost);
        take(p, "overlap", c.cost.overlap);
    }
    if (j.contains("trace_path")) {
        c.workload.reset();
        c.trace_path = j["trace_path"].get<std::string>();
        take(j, "replay_window_seconds", c.replay_window_seconds);
    } else if (j.contains("workload")) {
        const auto &p = j["workload"];
        WorkloadSpec w = c.workload.value_or(WorkloadSpec{});
        take(p, "requests", w.requests);
        take(p, "concurrency", w.concurrency);
        take(p, "p50", w.p50);
        take(p, "p90", w.p90);
        take(p, "p99", w.p99);
        take(p, "top_decile_share", w.top_decile_share);
        take(p, "arrivals_per_window", w.arrivals_per_window);
        take(p, "cluster_correlation", w.cluster_correlation);
        take(p, "prompt_min", w.prompt_min);
        take(p, "prompt_max", w.prompt_max);
        take(p, "seed", w.seed);
        c.workload = w;
        c.trace_path.reset();
    }
    if (j.contains("mode")) {
        const auto &p = j["mode"];
        take(p, "pager_enabled", c.pager_enabled);
        if (p.contains("regime"))
            c.regime = parse_regime(p["regime"].get<std::string>());
    }
    if (j.contains("shaping")) {
        const auto &p = j["shaping"];
        take(p, "span_blocks", c.span_blocks);
        take(p, "staged_refresh_period", c.staged_refresh_period);
        take(p, "demand_refresh_period", c.demand_refresh_period);
        take(p, "demand_gather_tokens", c.demand_gather_tokens);
        take(p, "share_probability", c.share_probability);
        take(p, "shared_prefix_tokens", c.shared_prefix_tokens);
        take(p, "static_slot_tokens", c.static_slot_tokens);
        take(p, "arena_headroom_pages", c.arena_headroom_pages);
        if (p.contains("arena_pages"))
            c.arena_pages_override = p["arena_pages"].get<uint32_t>();
    }
    if (j.contains("eos_burst")) {
        take(j["eos_burst"], "step", c.eos_burst_step);
        take(j["eos_burst"], "fraction", c.eos_burst_fraction);
    }
    if (j.contains("b200")) {
        const auto &p = j["b200"];
        take(p, "device", c.b200.device);
        take(p, "kv_heads", c.b200.kv_heads);
        take(p, "head_dim", c.b200.head_dim);
        take(p, "q_heads", c.b200.q_heads);
        take(p, "payload", c.b200.payload);
        take(p, "query", c.b200.query);
        take(p, "transfer", c.b200.transfer);
        take(p, "dtype", c.b200.dtype);
        take(p, "trace", c.b200.trace);
        take(p, "attention", c.b200.attention);
        take(p, "attention_kernel", c.b200.attention_kernel);
        take(p, "ring_rows", c.b200.ring_rows);
        take(p, "max_tokens", c.b200.max_tokens);
        take(p, "graph", c.b200.graph);
        take(p, "check", c.b200.check);
        take(p, "prefill_budget", c.b200.prefill_budget);
        take(p, "utility", c.b200.utility);
        take(p, "utility_layer", c.b200.utility_layer);
        take(p, "utility_every", c.b200.utility_every);
        take(p, "shard_rank", c.b200.shard_rank);
        take(p, "shard_world", c.b200.shard_world);
    }
    return c;
}

ScenarioConfig config_from_json_text(const std::string &text) {
    ojson j;
    try {
        j = ojson::parse(text);
    } catch (const std::exception &e) {
        raise(Errc::parse_error, std::string("config: ") + e.what());
    }
    return config_from_json(j);
}

ScenarioConfig config_from_json_file(const std::string &path) {
    std::ifstream in(path);
    if (!in)
        raise(Errc::io_error, "cannot open config " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    try {
        return config_from_json(ojson::parse(ss.str()));
    } catch (const Error &) {
        throw;
    } catch (const std::exception &e) {
        raise(Errc::parse_error, path + ": " + e.what());
    }
}

std::string config_to_json(const ScenarioConfig &c) {
    ojson j;
    j["label"] = c.label;
    j["seed"] = c.seed;
    j["steps"] = c.steps;
    j["warmup_steps"] = c.warmup_steps;
    j["step_ms"] = c.step_ms;
    j["pager"] = {{"page_bytes", c.pager.page_bytes},
                  {"arena_pages", c.pager.arena_pages},
                  {"layers", c.pager.layers},
                  {"kv_head_dim", c.pager.kv_head_dim},
                  {"elem_bytes", c.pager.elem_bytes}};
    j["placement"] = {{"alpha", c.placement.alpha},
                      {"lookahead_budget", c.placement.lookahead_budget},
                      {"cold_budget", c.placement.cold_budget}};
    j["transport"] = {{"tau_bytes", c.transport.merge_threshold},
                      {"delta_hold", c.transport.max_hold},
                      {"max_trains_per_step", c.transport.max_trains_per_step},
                      {"merge", c.transport.merge}};
    j["far_view"] = {{"enabled", c.far_view.enabled},
                     {"w_star", c.far_view.near_window},
                     {"cap", c.far_view.cap},
                     {"sv_chunk", c.far_view.chunk_tokens}};
    j["cost_model"] = {{"dma_fixed_overhead", c.cost.dma_fixed_overhead},
                       {"dma_bandwidth", c.cost.dma_bandwidth},
                       {"kernel_base", c.cost.kernel_base},
                       {"kernel_per_slot", c.cost.kernel_per_slot},
                       {"submit_cost", c.cost.submit_cost},
                       {"commit_cost", c.cost.commit_cost},
                       {"overlap", c.cost.overlap}};
    if (c.workload) {
        const WorkloadSpec &w = *c.workload;
        j["workload"] = {{"requests", w.requests},
                         {"concurrency", w.concurrency},
                         {"p50", w.p50},
                         {"p90", w.p90},
                         {"p99", w.p99},
                         {"top_decile_share", w.top_decile_share},
                         {"arrivals_per_window", w.arrivals_per_window},
                         {"cluster_correlation", w.cluster_correlation},
                         {"prompt_min", w.prompt_min},
                         {"prompt_max", w.prompt_max},
                         {"seed", w.seed}};
    } else if (c.trace_path) {
        j["trace_path"] = *c.trace_path;
        j["replay_window_seconds"] = c.replay_window_seconds;
    }
    j["mode"] = {{"pager_enabled", c.pager_enabled}, {"regime", regime_name(c.regime)}};
    j["shaping"] = {{"span_blocks", c.span_blocks},
                    {"staged_refresh_period", c.staged_refresh_period},
                    {"demand_refresh_period", c.demand_refresh_period},
                    {"demand_gather_tokens", c.demand_gather_tokens},
                    {"share_probability", c.share_probability},
                    {"shared_prefix_tokens", c.shared_prefix_tokens},
                    {"static_slot_tokens", c.static_slot_tokens},
                    {"arena_headroom_pages", c.arena_headroom_pages}};
    if (c.arena_pages_override)
        j["shaping"]["arena_pages"] = *c.arena_pages_override;
    if (c.eos_burst_step > 0)
        j["eos_burst"] = {{"step", c.eos_burst_step}, {"fraction", c.eos_burst_fraction}};
    return j.dump(2) + "\n";
}

ScenarioConfig default_audit_config() {
    ScenarioConfig c;
    c.label = "audit";
    c.pager.page_bytes = 16 * 1024;
    c.pager.layers = 4;
    c.pager.kv_head_dim = 64;
    c.pager.elem_bytes = 2;
    c.placement.alpha = 0.3;
    c.placement.lookahead_budget = 32;
    c.placement.cold_budget = 96;
    c.transport.merge_threshold = 131072;
    c.transport.max_trains_per_step = 2;
    c.transport.merge = true;
    c.far_view.enabled = false;
    c.far_view.near_window = 512;
    c.far_view.cap = 64;
    c.far_view.chunk_tokens = 128;
    c.cost.dma_fixed_overhead = 1.0;
    c.cost.dma_bandwidth = 131072.0;
    c.cost.kernel_base = 2.0;
    c.cost.kernel_per_slot = 0.002;
    c.cost.submit_cost = 0.04;
    c.cost.commit_cost = 0.04;
    c.cost.overlap = true;
    c.transport.max_hold = 0.25 * c.cost.kernel_cost(c.far_view.near_window);
    WorkloadSpec w;
    w.requests = 10000;
    w.concurrency = 64;
    w.arrivals_per_window = 1.85;
    w.seed = 1;
    c.workload = w;
    c.steps = 2000;
    c.warmup_steps = 100;
    c.seed = 1;
    c.span_blocks = 9;
    c.staged_refresh_period = 32;
    c.demand_refresh_period = 16;
    c.demand_gather_tokens = 46;
    return c;
}

} // namespace kvrail
