// kvrail-b200 device context: HBM layout, step publication and graph replay.
// Implements include/kvr_cuda.h.
//
// HBM layout (per GPU):
//   arena  arena_pages x page_bytes        token-major pages, identical to the
//                                          reference layout (pager.cpp:705)
//   ring   [slot][layer][R][2*d_kv]        the fixed-shape window; layer-major so
//                                          one (slot, layer) window is contiguous
//   tmap   [slot][max_tokens] u32          device page table: token -> block*tpp+slot
//   smap   [slot][max_chunks+tpp] u32      summary-slot page table
//   far    [slot][layer][max_chunks][2*d_kv] far-view summary rows
//   q/out  [slot][layer][q_head][head_dim] f32
//   desc   3 x max_desc_bytes               step descriptors (2 ring slots + apply-only)
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <dlfcn.h>
#include <nccl.h>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>
#include <stdexcept>
#include <string>

#include "kvr_internal.cuh"

namespace kvr {
size_t scan_dynamic_smem(uint32_t cap);
cudaError_t prepare_scan(uint32_t cap);
cudaError_t prepare_gather(const DevCtx &c);
} // namespace kvr

using namespace kvr;

struct kvr_dev {
    kvr_geometry g{};
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;                   // the step graph's forked branch (K-scan)
    cudaStream_t side2 = nullptr;                  // second forked branch (decode queries)
    // the step's copies run on their own streams, off the graph stream: the descriptor
    // H2D of step t+1 overlaps step t's graph, the stats D2H of step t overlaps t+1's
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_copied[2] = {}, ev_stats[2] = {};
    ScanCounters *scans[2] = {}; // per ring slot: the D2H of step t never races t+1's K-scan
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork2 = nullptr, ev_join2 = nullptr;
    DevCtx base{};
    uint8_t *d_desc[3] = {nullptr, nullptr, nullptr};
    void *h_desc[3] = {nullptr, nullptr, nullptr};
    ScanCounters *h_scan[2] = {nullptr, nullptr};
    kvr_mass_run *h_mass[2] = {nullptr, nullptr}; // K-mass runs per ring slot (pinned)
    uint32_t *h_mass_count[2] = {nullptr, nullptr};
    cudaEvent_t ev_start[2] = {}, ev_stop[2] = {}, ev_attn[2] = {};
    cudaEvent_t ev_phase[2][8] = {}; // per ring slot: phase boundaries inside the step graph
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    AttnPlan *attn = nullptr;
    uint32_t graph_kernels = 0; // kernel nodes in the captured step graph
    uint32_t graph_captures = 0; // step graphs captured (one per descriptor ring slot, never again)
    uint64_t launched[2] = {0, 0};
    bool in_flight[2] = {false, false};
    uint64_t pending_write_tokens[2] = {0, 0};
    std::vector<void *> allocs;
    // per-step counts collective (kvr_comm_init)
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    uint64_t n_launches = 0;
    bool phase_events = false; // event nodes at every phase boundary (KVR_PHASE_EVENTS=1); off: K-attn's
                               // pair only (each event node costs ~5 us of the step graph)
    int64_t *d_counts = nullptr;                  // all-reduce result (device), one row per ring slot
    int64_t *h_counts[2] = {nullptr, nullptr};    // its D2H copy per ring slot (pinned)
};

namespace {

thread_local std::string g_err;

struct CudaFail : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess)
        throw CudaFail(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

/// NCCL entry points, resolved at run time: the library already in the process
/// (torch's) when there is one, else the system's.
struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};

const Nccl &nccl() {
    static Nccl api = [] {
        Nccl a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
        throw std::runtime_error("NCCL (libnccl.so.2) is not loadable");
    return api;
}

void nck(ncclResult_t r, const char *what);

template <typename Fn> int guard(Fn &&fn) {
    try {
        fn();
        return KVR_OK;
    } catch (const CudaFail &e) {
        g_err = e.what();
        return KVR_E_CUDA;
    } catch (const std::exception &e) {
        g_err = e.what();
        return KVR_E_BAD_CONFIG;
    }
}

void nck(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
        throw CudaFail(std::string("NCCL error in ") + what + ": " +
                       (nccl().error_string ? nccl().error_string(r) : std::to_string(int(r))));
}

void *dalloc(kvr_dev *d, size_t bytes, const char *what) {
    void *p = nullptr;
    ck(cudaMalloc(&p, bytes ? bytes : 16), what);
    d->allocs.push_back(p);
    return p;
}

__global__ void k_tl_reset(unsigned long long *tl) {
    if (threadIdx.x < 2 * KVR_TIMELINE_IDS)
        tl[threadIdx.x] = threadIdx.x & 1 ? 0ull : ~0ull;
}
void tl_reset(unsigned long long *tl, cudaStream_t s) { k_tl_reset<<<1, 2 * KVR_TIMELINE_IDS, 0, s>>>(tl); }

// KVR_QFORK: where the decode-queries branch forks (root | apply | hot; default apply).
// Timeline A/B, K-attn start after the step's first kernel (C5 / C3 / C2 us): root
// 47.5 / 74.4 / 90.2 (its CTAs crowd K-apply), apply 41.3 / 69.9 / 85.2, hot 46.6 /
// 68.5 / 85.4. K-scan forks at the root (one CTA).
int query_fork() {
    static const int k = [] {
        const char *e = getenv("KVR_QFORK");
        const std::string v = e ? e : "";
        return v == "root" ? 0 : v == "hot" ? 2 : 1;
    }();
    return k;
}

// KVR_QMERGE=1: the decode queries are extra CTAs of the hot K-write launch (no branch)
bool query_merge() {
    static const bool v = [] {
        const char *e = getenv("KVR_QMERGE");
        return e && e[0] == '1';
    }();
    return v;
}

// KVR_QJOIN=gather: the queries branch joins before K-gather instead of before K-attn (A/B)
bool query_join_at_gather() {
    static const bool v = [] {
        const char *e = getenv("KVR_QJOIN");
        return e && std::string(e) == "gather";
    }();
    return v;
}

DevCtx ctx_for(const kvr_dev *d, int slot) {
    DevCtx c = d->base;
    c.desc = d->d_desc[slot];
    if (slot < 2 && d->scans[slot])
        c.scan = d->scans[slot];
    return c;
}

// `k` >= 0: record the gather / attention phase events of ring slot k (as
// event-record nodes when the stream is being captured into the step graph).
void run_step_kernels(kvr_dev *d, const DevCtx &c, bool full_step, int k = -1, bool capturing = false) {
    cudaStream_t s = d->stream;
    auto mark = [&](int i) {
        if (k >= 0 && d->phase_events) // (K-attn times itself: AttnSpan)
            ck(capturing ? cudaEventRecordWithFlags(d->ev_phase[k][i], s, cudaEventRecordExternal)
                         : cudaEventRecord(d->ev_phase[k][i], s),
               "phase event");
    };
    mark(0);
    if (!full_step) { // apply-only: everything in order on one stream
        launch_apply(c, s, d->sms);
        launch_write(c, s, d->sms, 0);
        launch_write(c, s, d->sms, 1);
        launch_far_map_prime(c, s, d->sms);
        return;
    }
    // Two forked branches: K-scan (needs only the descriptor) joins before K-gather,
    // the decode queries (read only by K-attn) join before K-attn; both run beside
    // the byte kernels, off the step's critical path. Kernel-to-kernel edges of the
    // main chain are PDL edges (each dependent launches during its predecessor and
    // waits in-kernel, griddepcontrol), unless phase event nodes sit between them.
    // The branches fork at the graph's root, beside K-apply (neither reads what it
    // writes): a fork edge after K-apply cost ~11 us before they started (timeline).
    const bool pdl = pdl_enabled() && !d->phase_events;
    cudaStream_t side = d->side, side2 = d->side2;
    const bool qmerge = query_merge(); // queries generated inside the hot K-write launch
    const int qfork = qmerge ? -1 : query_fork(); // 0 root, 1 after K-apply, 2 after the hot K-write
    auto fork_queries = [&] {
        ck(cudaEventRecord(d->ev_fork2, s), "fork");
        ck(cudaStreamWaitEvent(side2, d->ev_fork2, 0), "fork wait");
        launch_query(c, side2, d->sms);
        ck(cudaEventRecord(d->ev_join2, side2), "join");
    };
    ck(cudaEventRecord(d->ev_fork, s), "fork"); // (under capture: a dependency, not a node)
    ck(cudaStreamWaitEvent(side, d->ev_fork, 0), "fork wait");
    launch_scan(c, side);
    ck(cudaEventRecord(d->ev_join, side), "join");
    if (qfork == 0)
        fork_queries();
    launch_apply(c, s, d->sms);
    if (qfork == 1)
        fork_queries();
    mark(1);
    launch_write(c, s, d->sms, 0, 0, pdl, qmerge);
    if (qfork == 2)
        fork_queries();
    mark(2);
    launch_far_map_prime(c, s, d->sms, pdl);
    mark(3);
    ck(cudaStreamWaitEvent(s, d->ev_join, 0), "join wait");
    const bool qjoin_gather = !qmerge && query_join_at_gather();
    if (qjoin_gather) // K-attn's only dependency is then K-gather's PDL edge
        ck(cudaStreamWaitEvent(s, d->ev_join2, 0), "join wait");
    mark(4);
    launch_gather(c, s, d->sms, pdl);
    if (!qjoin_gather && !qmerge)
        ck(cudaStreamWaitEvent(s, d->ev_join2, 0), "join wait");
    mark(5);
    if (d->g.attention && d->attn)
        launch_attn(d->attn, c, s, pdl);
    mark(6);
    if (c.utility)
        launch_mass(c, s);
    // Cold writes (older prompt rows nothing in this step reads) go last: measured
    // on B200, co-running this int-bound generation beside the HBM-bound attention
    // (one CTA per SM on a forked branch) slowed the attention by more than the
    // overlap saved, so the step runs them after it with the whole GPU.
    // the step's last kernel writes the end stamp (with a communicator: a stamp node
    // after the collective)
    const int stamp_in_kernel = d->comm ? 0 : 1;
    // (after K-mass, a plain edge: K-mass is not a PDL dependent)
    launch_tail(c, s, d->sms, stamp_in_kernel, pdl && !c.utility && d->g.attention && d->attn);
    // the step's counts summed over every rank (the only cross-GPU traffic)
    if (d->comm) {
        nck(nccl().all_reduce(c.desc + offsetof(kvr_step_header, counts), d->d_counts + (k > 0 ? k : 0) * KVR_COUNTS,
                              KVR_COUNTS, ncclInt64,
                              ncclSum, d->comm, s),
            "per-step counts all-reduce");
        launch_stamp(c, s);
    }
    mark(7);
}

} // namespace

extern "C" {

const char *kvr_dev_last_error(void) { return g_err.c_str(); }

int kvr_dev_count(int *out) {
    return guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess)
            n = 0;
        *out = n;
    });
}

int kvr_dev_open(const kvr_geometry *geo, kvr_dev **out) {
    auto d = std::make_unique<kvr_dev>();
    const int rc = guard([&] {
        kvr_geometry g = *geo;
        if (g.token_bytes % 16 || (2ull * g.kv_heads * g.head_dim * g.elem_bytes) % 16)
            throw std::runtime_error("token and layer rows must be multiples of 16 bytes");
        if (g.head_dim < 8 || (g.head_dim & (g.head_dim - 1)))
            throw std::runtime_error("head_dim must be a power of two >= 8");
        if (g.kv_heads == 0 || g.q_heads % g.kv_heads)
            throw std::runtime_error("q_heads must be a multiple of kv_heads");
        if (g.ring_rows % 32 || g.ring_rows < g.near_window)
            throw std::runtime_error("ring_rows must be a multiple of 32 and >= W*");
        if (!g.max_desc_bytes)
            g.max_desc_bytes = 16ull << 20;
        if (!g.max_scan_descs)
            g.max_scan_descs = 2048;
        if (!g.max_trains)
            g.max_trains = 2048;
        if (g.max_scan_descs & (g.max_scan_descs - 1))
            throw std::runtime_error("max_scan_descs must be a power of two");
        if (uint64_t(g.arena_pages) * g.page_bytes >= (1ull << 47)) // K-scan's sort key holds 47-bit offsets
            throw std::runtime_error("arena must be smaller than 128 TiB");
        if (scan_dynamic_smem(g.max_scan_descs) > (192u << 10)) // K-scan stages its arrays in shared memory
            throw std::runtime_error("max_scan_descs too large for K-scan's shared memory (<= 2048)");
        d->g = g;
        if (const char *pe = getenv("KVR_PHASE_EVENTS"))
            d->phase_events = std::string(pe) == "1";
        ck(cudaSetDevice(g.device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, g.device), "cudaGetDeviceProperties");
        d->sms = prop.multiProcessorCount;
        // stream priorities become node priorities of the captured step graph
        // (instantiated with cudaGraphInstantiateFlagUseNodePriority): the main chain
        // and K-scan (on the critical path before K-gather) high, the decode queries
        // (needed only by K-attn, ~20 us later) low, so their CTAs do not crowd K-fmp
        int prio_low = 0, prio_high = 0;
        ck(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high), "stream priorities");
        ck(cudaStreamCreateWithPriority(&d->stream, cudaStreamNonBlocking, prio_high), "stream");
        ck(cudaStreamCreateWithPriority(&d->side, cudaStreamNonBlocking, prio_high), "side stream");
        ck(cudaStreamCreateWithPriority(&d->side2, cudaStreamNonBlocking, prio_low), "side stream");
        ck(cudaStreamCreateWithFlags(&d->h2d, cudaStreamNonBlocking), "copy stream");
        ck(cudaStreamCreateWithFlags(&d->d2h, cudaStreamNonBlocking), "copy stream");
        for (int i = 0; i < 2; ++i) {
            ck(cudaEventCreateWithFlags(&d->ev_copied[i], cudaEventDisableTiming), "copy event");
            ck(cudaEventCreateWithFlags(&d->ev_stats[i], cudaEventDisableTiming), "copy event");
        }
        ck(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming), "fork event");
        ck(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming), "join event");
        ck(cudaEventCreateWithFlags(&d->ev_join2, cudaEventDisableTiming), "join event");
        ck(cudaEventCreateWithFlags(&d->ev_fork2, cudaEventDisableTiming), "fork event");
        for (int i = 0; i < 2; ++i) {
            ck(cudaEventCreate(&d->ev_start[i]), "event");
            ck(cudaEventCreate(&d->ev_stop[i]), "event");
            ck(cudaEventCreate(&d->ev_attn[i]), "event");
            for (int j = 0; j < 8; ++j)
                ck(cudaEventCreate(&d->ev_phase[i][j]), "event");
        }
        DevCtx &c = d->base;
        c.page_bytes = g.page_bytes;
        c.token_bytes = g.token_bytes;
        c.max_tokens = g.max_tokens;
        c.seed = g.seed;
        c.tpp = g.tokens_per_page;
        c.arena_pages = g.arena_pages;
        c.L = g.layers;
        c.Hkv = g.kv_heads;
        c.hd = g.head_dim;
        c.Hq = g.q_heads;
        c.group = g.q_heads / g.kv_heads;
        c.d_kv = g.kv_heads * g.head_dim;
        c.row_elems = 2 * c.d_kv;
        c.esz = g.elem_bytes;
        c.elem_kind = uint32_t(g.elem_kind);
        c.payload_mode = g.payload_mode;
        {
            const uint32_t sh = g.lane_shift ? g.lane_shift : 7;
            if (sh > 12)
                throw std::runtime_error("lane_shift must be <= 12");
            c.lane_scale = 1.0f / float(1u << sh);
            c.lane_bias = 8388608.0f * c.lane_scale + 128.0f * c.lane_scale; // exact: 2^(23-sh) + 2^(7-sh)
            c.lane_h2_scale = __float2half2_rn(c.lane_scale);              // 2^-sh: exact in fp16 (sh <= 12)
            c.lane_h2_bias = __float2half2_rn(-1152.0f * c.lane_scale);    // -1152 * 2^-sh: exact
        }
        if (g.query_mode > KVR_QUERY_F32)
            throw std::runtime_error("unknown query_mode");
        c.query_mode = g.query_mode;
        c.n_slots = g.n_slots;
        c.W = g.near_window;
        c.R = g.ring_rows;
        c.far_cap = g.far_cap;
        c.chunk_tokens = g.chunk_tokens;
        c.max_chunks = g.max_chunks ? g.max_chunks : 1;
        c.smap_cap = c.max_chunks + g.tokens_per_page;
        c.max_scan = g.max_scan_descs;
        c.max_trains = g.max_trains;
        if (uint64_t(c.L) * c.d_kv * 2 * c.esz != g.token_bytes)
            throw std::runtime_error("token_bytes != 2 * layers * kv_heads * head_dim * elem_bytes");

        const uint64_t arena_bytes = uint64_t(g.arena_pages) * g.page_bytes;
        c.arena = static_cast<uint8_t *>(dalloc(d.get(), arena_bytes, "arena"));
        ck(cudaMemsetAsync(c.arena, 0, arena_bytes, d->stream), "arena zero");
        // guard rows for the tensor-core attention's whole-tile loads (kvr_attn_tc.cu)
        c.G = (g.attention == 3 || (g.attention == 1 && c.group >= 4)) && attn_tc_supported(c) ? 128 : 0;
        c.Rp = c.R + c.G;
        const uint64_t ring_elems = uint64_t(c.n_slots) * c.L * c.Rp * c.row_elems;
        c.ring = static_cast<uint8_t *>(dalloc(d.get(), ring_elems * c.esz, "ring"));
        ck(cudaMemsetAsync(c.ring, 0, ring_elems * c.esz, d->stream), "ring zero");
        const uint64_t tmap_n = uint64_t(c.n_slots) * c.max_tokens;
        c.tmap = static_cast<uint32_t *>(dalloc(d.get(), tmap_n * 4, "tmap"));
        ck(cudaMemsetAsync(c.tmap, 0xff, tmap_n * 4, d->stream), "tmap init");
        const uint64_t smap_n = uint64_t(c.n_slots) * c.smap_cap;
        c.smap = static_cast<uint32_t *>(dalloc(d.get(), smap_n * 4, "smap"));
        ck(cudaMemsetAsync(c.smap, 0xff, smap_n * 4, d->stream), "smap init");
        const uint64_t far_elems = uint64_t(c.n_slots) * c.L * c.max_chunks * c.row_elems;
        c.far = static_cast<uint8_t *>(dalloc(d.get(), far_elems * c.esz, "far"));
        ck(cudaMemsetAsync(c.far, 0, far_elems * c.esz, d->stream), "far zero");
        c.stash = c.far_cap ? static_cast<uint8_t *>(dalloc(d.get(), uint64_t(c.n_slots) * c.max_chunks * c.token_bytes,
                                                            "presum stash"))
                            : nullptr;
        const uint64_t qn = uint64_t(c.n_slots) * c.L * c.Hq * c.hd;
        // exact queries (multiples of 1/128 in [-1, 1)) are stored in the KV element type:
        // half the query bytes K-attn reads per item (C3: 67 -> 34 MB per step)
#ifndef KVR_Q16
#define KVR_Q16 1
#endif
        c.q_esz = KVR_Q16 && c.query_mode == KVR_QUERY_EXACT && c.esz == 2 ? 2u : 4u;
        c.q = static_cast<float *>(dalloc(d.get(), qn * c.q_esz, "q"));
        c.out = static_cast<float *>(dalloc(d.get(), qn * 4, "out"));
        ck(cudaMemsetAsync(c.q, 0, qn * c.q_esz, d->stream), "q zero");
        ck(cudaMemsetAsync(c.out, 0, qn * 4, d->stream), "out zero");
        c.trains = static_cast<kvr_train *>(dalloc(d.get(), sizeof(kvr_train) * c.max_trains, "trains"));
        c.descs = static_cast<kvr_descriptor *>(dalloc(d.get(), sizeof(kvr_descriptor) * c.max_scan, "descs"));
        c.gspans = static_cast<GSpan *>(dalloc(d.get(), sizeof(GSpan) * c.max_scan, "gspans"));
        for (int i = 0; i < 2; ++i) {
            d->scans[i] = static_cast<ScanCounters *>(dalloc(d.get(), sizeof(ScanCounters), "scan"));
            ck(cudaMemsetAsync(d->scans[i], 0, sizeof(ScanCounters), d->stream), "scan zero");
        }
        c.scan = d->scans[0];
        c.attn_sched = static_cast<uint32_t *>(dalloc(d.get(), 4 * sizeof(uint32_t), "schedule tickets"));
        ck(cudaMemsetAsync(c.attn_sched, 0, 4 * sizeof(uint32_t), d->stream), "schedule zero");
        if (const char *e = getenv("KVR_TIMELINE"); e && e[0] == '1') { // diagnostic timeline
            c.tl = static_cast<unsigned long long *>(dalloc(d.get(), sizeof(uint64_t) * 2 * KVR_TIMELINE_IDS, "timeline"));
            tl_reset(c.tl, d->stream);
        }
        {
            const uint64_t off[2] = {~0ull, 0};
            auto *fault = static_cast<uint64_t *>(dalloc(d.get(), sizeof(off), "fault hooks"));
            ck(cudaMemcpy(fault, off, sizeof(off), cudaMemcpyHostToDevice), "fault init");
            c.fault = fault;
        }
        for (int i = 0; i < 3; ++i) {
            d->d_desc[i] = static_cast<uint8_t *>(dalloc(d.get(), g.max_desc_bytes, "desc"));
            ck(cudaMallocHost(&d->h_desc[i], g.max_desc_bytes), "pinned desc");
            std::memset(d->h_desc[i], 0, sizeof(kvr_step_header));
        }
        for (int i = 0; i < 2; ++i) {
            void *p;
            ck(cudaMallocHost(&p, sizeof(ScanCounters)), "pinned stats");
            d->h_scan[i] = static_cast<ScanCounters *>(p);
            ck(cudaMallocHost(&p, KVR_COUNTS * sizeof(int64_t)), "pinned counts");
            d->h_counts[i] = static_cast<int64_t *>(p);
            std::memset(p, 0, KVR_COUNTS * sizeof(int64_t));
        }
        d->d_counts = static_cast<int64_t *>(dalloc(d.get(), 2 * KVR_COUNTS * sizeof(int64_t), "counts"));
        if (g.utility) {
            if (!g.attention || g.utility_layer >= g.layers || c.group > mass_max_group())
                throw std::runtime_error("utility: needs attention, utility_layer < layers and q-group <= 16");
            c.utility = g.utility; // measure on steps with step % utility == 0
            c.util_layer = g.utility_layer;
            c.mass_sc = static_cast<float *>(dalloc(d.get(), mass_scratch_floats(c) * 4, "mass scores"));
            c.mass_part = static_cast<float2 *>(dalloc(d.get(), mass_part_entries(c) * sizeof(float2), "mass parts"));
            c.mass_runs = static_cast<kvr_mass_run *>(
                dalloc(d.get(), uint64_t(c.n_slots) * c.W * sizeof(kvr_mass_run), "mass runs"));
            c.mass_count = static_cast<uint32_t *>(dalloc(d.get(), uint64_t(c.n_slots) * 4, "mass count"));
            ck(cudaMemsetAsync(c.mass_count, 0, uint64_t(c.n_slots) * 4, d->stream), "mass count zero");
            for (int i = 0; i < 2; ++i) {
                void *p;
                ck(cudaMallocHost(&p, uint64_t(c.n_slots) * c.W * sizeof(kvr_mass_run)), "pinned mass");
                d->h_mass[i] = static_cast<kvr_mass_run *>(p);
                ck(cudaMallocHost(&p, uint64_t(c.n_slots) * 4), "pinned mass count");
                d->h_mass_count[i] = static_cast<uint32_t *>(p);
            }
            if (!prepare_mass(c))
                throw std::runtime_error("utility: head_dim must be 32, 64 or 128 and (W* + q_heads) * 8 bytes <= 200 KiB");
        }
        ck(prepare_scan(c.max_scan), "K-scan shared-memory attribute (max_scan_descs)");
        ck(prepare_gather(c), "K-gather shared-memory attribute (row size)");
        if (g.attention) {
            d->attn = make_attn_plan(c, d->sms, g.device, int(g.attention));
            if (!d->attn)
                throw std::runtime_error("no attention kernel for this head_dim/group/dtype");
        }
        ck(cudaStreamSynchronize(d->stream), "open sync");
    });
    if (rc != KVR_OK) {
        kvr_dev_close(d.release());
        return rc;
    }
    *out = d.release();
    return KVR_OK;
}

int kvr_dev_close(kvr_dev *d) {
    if (!d)
        return KVR_OK;
    if (d->stream)
        cudaStreamSynchronize(d->stream);
    if (d->h2d)
        cudaStreamSynchronize(d->h2d);
    if (d->d2h)
        cudaStreamSynchronize(d->d2h);
    for (int i = 0; i < 2; ++i) {
        if (d->ev_copied[i])
            cudaEventDestroy(d->ev_copied[i]);
        if (d->ev_stats[i])
            cudaEventDestroy(d->ev_stats[i]);
        if (d->graph[i])
            cudaGraphExecDestroy(d->graph[i]);
        if (d->ev_start[i])
            cudaEventDestroy(d->ev_start[i]);
        if (d->ev_stop[i])
            cudaEventDestroy(d->ev_stop[i]);
        if (d->ev_attn[i])
            cudaEventDestroy(d->ev_attn[i]);
        for (int j = 0; j < 8; ++j)
            if (d->ev_phase[i][j])
                cudaEventDestroy(d->ev_phase[i][j]);
        if (d->h_scan[i])
            cudaFreeHost(d->h_scan[i]);
        if (d->h_counts[i])
            cudaFreeHost(d->h_counts[i]);
        if (d->h_mass[i])
            cudaFreeHost(d->h_mass[i]);
        if (d->h_mass_count[i])
            cudaFreeHost(d->h_mass_count[i]);
    }
    for (int i = 0; i < 3; ++i)
        if (d->h_desc[i])
            cudaFreeHost(d->h_desc[i]);
    if (d->comm)
        nccl().comm_destroy(d->comm);
    for (void *p : d->allocs)
        cudaFree(p);
    if (d->attn)
        free_attn_plan(d->attn);
    if (d->ev_fork)
        cudaEventDestroy(d->ev_fork);
    if (d->ev_join)
        cudaEventDestroy(d->ev_join);
    if (d->ev_join2)
        cudaEventDestroy(d->ev_join2);
    if (d->ev_fork2)
        cudaEventDestroy(d->ev_fork2);
    if (d->side)
        cudaStreamDestroy(d->side);
    if (d->side2)
        cudaStreamDestroy(d->side2);
    if (d->h2d)
        cudaStreamDestroy(d->h2d);
    if (d->d2h)
        cudaStreamDestroy(d->d2h);
    if (d->stream)
        cudaStreamDestroy(d->stream);
    delete d;
    return KVR_OK;
}

int kvr_dev_desc_buffer(kvr_dev *d, uint32_t ring_slot, void **out) {
    return guard([&] {
        if (ring_slot > 2)
            throw std::runtime_error("ring slot out of range");
        *out = d->h_desc[ring_slot];
    });
}

int kvr_dev_launch(kvr_dev *d, uint32_t k, uint64_t desc_bytes) {
    return guard([&] {
        if (k > 1)
            throw std::runtime_error("step ring slot must be 0 or 1");
        if (desc_bytes > d->g.max_desc_bytes)
            throw std::runtime_error("step descriptor exceeds max_desc_bytes");
        const auto *h = static_cast<const kvr_step_header *>(d->h_desc[k]);
        const DevCtx c = ctx_for(d, int(k));
        // descriptor H2D on the copy stream once slot k's previous graph is done with
        // d_desc[k]; the graph stream waits for it (and for slot k's previous stats
        // D2H, which read this slot's counters) — both overlap the graph in flight
        ck(cudaStreamWaitEvent(d->h2d, d->ev_stop[k], 0), "slot free");
        ck(cudaMemcpyAsync(d->d_desc[k], d->h_desc[k], desc_bytes, cudaMemcpyHostToDevice, d->h2d),
           "descriptor H2D");
        ck(cudaEventRecord(d->ev_copied[k], d->h2d), "copy event");
        ck(cudaStreamWaitEvent(d->stream, d->ev_copied[k], 0), "descriptor wait");
        ck(cudaStreamWaitEvent(d->stream, d->ev_stats[k], 0), "stats slot wait");
        if (c.utility) // K-mass buffers are shared by both slots: the other slot's D2H first
            ck(cudaStreamWaitEvent(d->stream, d->ev_stats[k ^ 1], 0), "mass D2H wait");
        ck(cudaEventRecord(d->ev_start[k], d->stream), "event");
        if (d->g.use_graph) {
            if (!d->graph[k]) {
                cudaGraph_t graph;
                ck(cudaStreamBeginCapture(d->stream, cudaStreamCaptureModeThreadLocal), "capture");
                run_step_kernels(d, c, true, int(k), true);
                ck(cudaStreamEndCapture(d->stream, &graph), "capture end");
                size_t n_nodes = 0;
                ck(cudaGraphGetNodes(graph, nullptr, &n_nodes), "graph nodes");
                std::vector<cudaGraphNode_t> nodes(n_nodes);
                ck(cudaGraphGetNodes(graph, nodes.data(), &n_nodes), "graph nodes");
                uint32_t kernels = 0;
                for (cudaGraphNode_t nd : nodes) {
                    cudaGraphNodeType ty;
                    ck(cudaGraphNodeGetType(nd, &ty), "graph node type");
                    kernels += ty == cudaGraphNodeTypeKernel;
                }
                d->graph_kernels = kernels;
                ++d->graph_captures;
                ck(cudaGraphInstantiate(&d->graph[k], graph, cudaGraphInstantiateFlagUseNodePriority),
                   "graph instantiate");
                cudaGraphDestroy(graph);
            }
            ck(cudaGraphLaunch(d->graph[k], d->stream), "graph launch");
        } else {
            run_step_kernels(d, c, true, int(k), false);
            ck(cudaGetLastError(), "step launch");
        }
        ck(cudaEventRecord(d->ev_stop[k], d->stream), "event");
        // stats D2H on the other copy stream, after the graph
        ck(cudaStreamWaitEvent(d->d2h, d->ev_stop[k], 0), "graph done");
        ck(cudaMemcpyAsync(d->h_scan[k], c.scan, sizeof(ScanCounters), cudaMemcpyDeviceToHost, d->d2h),
           "stats D2H");
        if (d->comm)
            ck(cudaMemcpyAsync(d->h_counts[k], d->d_counts + k * KVR_COUNTS, KVR_COUNTS * sizeof(int64_t),
                               cudaMemcpyDeviceToHost,
                               d->d2h),
               "counts D2H");
        else
            std::memcpy(d->h_counts[k], h->counts, KVR_COUNTS * sizeof(int64_t));
        if (c.utility && h->step % c.utility == 0) {
            ck(cudaMemcpyAsync(d->h_mass_count[k], c.mass_count, uint64_t(c.n_slots) * 4, cudaMemcpyDeviceToHost,
                               d->d2h),
               "mass count D2H");
            ck(cudaMemcpyAsync(d->h_mass[k], c.mass_runs, uint64_t(c.n_slots) * c.W * sizeof(kvr_mass_run),
                               cudaMemcpyDeviceToHost, d->d2h),
               "mass D2H");
        }
        ck(cudaEventRecord(d->ev_stats[k], d->d2h), "stats event");
        d->launched[k] = h->step;
        d->in_flight[k] = true;
        ++d->n_launches;
        d->pending_write_tokens[k] = h->write_tokens + h->write_tokens_cold + uint64_t(h->n_presum) * c.chunk_tokens;
    });
}

int kvr_dev_apply_only(kvr_dev *d, uint32_t k, uint64_t desc_bytes) {
    return guard([&] {
        if (desc_bytes > d->g.max_desc_bytes)
            throw std::runtime_error("descriptor exceeds max_desc_bytes");
        DevCtx c = d->base;
        c.desc = d->d_desc[2];
        ck(cudaMemcpyAsync(d->d_desc[2], d->h_desc[2], desc_bytes, cudaMemcpyHostToDevice, d->stream),
           "apply H2D");
        run_step_kernels(d, c, false);
        ck(cudaGetLastError(), "apply launch");
        ck(cudaStreamSynchronize(d->stream), "apply sync");
        (void)k;
    });
}

int kvr_dev_wait(kvr_dev *d, uint32_t k, kvr_step_stats *out) {
    return guard([&] {
        if (k > 1)
            throw std::runtime_error("step ring slot must be 0 or 1");
        std::memset(out, 0, sizeof(*out));
        if (!d->in_flight[k])
            return;
        ck(cudaEventSynchronize(d->ev_stats[k]), "step wait"); // (after ev_stop: the D2H follows it)
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, d->ev_start[k], d->ev_stop[k]), "elapsed");
        const ScanCounters &sc = *d->h_scan[k];
        out->step = d->launched[k];
        out->device_ms = ms;
        for (int j = 0; j < 7; ++j) {
            float t = 0.f;
            if (d->phase_events)
                ck(cudaEventElapsedTime(&t, d->ev_phase[k][j], d->ev_phase[k][j + 1]), "elapsed");
            out->phase_ms[j] = t;
        }
        // K-gather's own span (first-CTA start to last exit) unless phase events bracket it
        out->gather_ms = d->phase_events ? out->phase_ms[4]
                         : sc.gather_t1 > sc.gather_t0 ? double(sc.gather_t1 - sc.gather_t0) * 1e-6 : 0.0;
        // K-attn's own span (first CTA start to last exit) unless phase events bracket it
        out->attn_ms = d->phase_events ? out->phase_ms[5]
                       : sc.attn_t1 > sc.attn_t0 ? double(sc.attn_t1 - sc.attn_t0) * 1e-6 : 0.0;
        if (!d->phase_events)
            out->phase_ms[5] = float(out->attn_ms);
        out->trains = sc.trains;
        out->descriptors = sc.descriptors;
        out->spans = sc.spans;
        out->status = sc.status;
        out->train_bytes = sc.train_bytes;
        out->end_ns = sc.end_ns;
        out->staged_tokens = sc.total_tokens;
        out->writeback_tokens = d->pending_write_tokens[k];
        std::memcpy(out->global_counts, d->h_counts[k], sizeof(out->global_counts));
        d->in_flight[k] = false;
    });
}

int kvr_dev_sync(kvr_dev *d) {
    return guard([&] {
        ck(cudaStreamSynchronize(d->stream), "sync");
        ck(cudaStreamSynchronize(d->d2h), "sync");
    });
}

int kvr_dev_buffer_bytes(kvr_dev *d, int buffer, uint64_t *out) {
    return guard([&] {
        const DevCtx &c = d->base;
        switch (buffer) {
        case KVR_BUF_ARENA: *out = uint64_t(c.arena_pages) * c.page_bytes; break;
        case KVR_BUF_RING: *out = uint64_t(c.n_slots) * c.L * c.Rp * c.row_elems * c.esz; break;
        case KVR_BUF_TMAP: *out = uint64_t(c.n_slots) * c.max_tokens * 4; break;
        case KVR_BUF_OUT: *out = uint64_t(c.n_slots) * c.L * c.Hq * c.hd * 4; break;
        case KVR_BUF_QUERY: *out = uint64_t(c.n_slots) * c.L * c.Hq * c.hd * c.q_esz; break;
        case KVR_BUF_FAR: *out = uint64_t(c.n_slots) * c.L * c.max_chunks * c.row_elems * c.esz; break;
        case KVR_BUF_TRAINS: *out = sizeof(kvr_train) * c.max_trains; break;
        case KVR_BUF_DESCS: *out = sizeof(kvr_descriptor) * c.max_scan; break;
        case KVR_BUF_SCAN: *out = sizeof(ScanCounters); break;
        case KVR_BUF_SMAP: *out = uint64_t(c.n_slots) * c.smap_cap * 4; break;
        default: throw std::runtime_error("unknown buffer");
        }
    });
}

int kvr_dev_read(kvr_dev *d, int buffer, uint64_t offset, uint64_t bytes, void *out) {
    return guard([&] {
        uint64_t size = 0;
        if (kvr_dev_buffer_bytes(d, buffer, &size) != KVR_OK)
            throw std::runtime_error("unknown buffer");
        if (offset + bytes > size)
            throw std::runtime_error("read past the end of the buffer");
        const DevCtx &c = d->base;
        const void *base = nullptr;
        switch (buffer) {
        case KVR_BUF_ARENA: base = c.arena; break;
        case KVR_BUF_RING: base = c.ring; break;
        case KVR_BUF_TMAP: base = c.tmap; break;
        case KVR_BUF_OUT: base = c.out; break;
        case KVR_BUF_QUERY: base = c.q; break;
        case KVR_BUF_FAR: base = c.far; break;
        case KVR_BUF_TRAINS: base = c.trains; break;
        case KVR_BUF_DESCS: base = c.descs; break;
        case KVR_BUF_SCAN: base = d->scans[d->launched[1] > d->launched[0] ? 1 : 0]; break; // the last step's
        case KVR_BUF_SMAP: base = c.smap; break;
        }
        ck(cudaStreamSynchronize(d->stream), "read sync");
        ck(cudaMemcpy(out, static_cast<const uint8_t *>(base) + offset, bytes, cudaMemcpyDeviceToHost),
           "read D2H");
    });
}

int kvr_dev_read_staged(kvr_dev *d, uint64_t tok_begin, uint64_t count, void *out, uint8_t *in_window) {
    return guard([&] {
        ck(cudaStreamSynchronize(d->stream), "read sync");
        ScanCounters sc{};
        ck(cudaMemcpy(&sc, d->scans[d->launched[1] > d->launched[0] ? 1 : 0], sizeof(sc), cudaMemcpyDeviceToHost),
           "scan counters");
        if (tok_begin + count > sc.total_tokens)
            throw std::runtime_error("read_staged: tokens past the last step's gather list");
        if (!count)
            return;
        const int k = d->launched[1] > d->launched[0] ? 1 : 0; // the last launched step
        const DevCtx c = ctx_for(d, k);
        const uint64_t bytes = count * c.token_bytes;
        uint8_t *buf = nullptr, *flags = nullptr;
        ck(cudaMallocAsync(reinterpret_cast<void **>(&buf), bytes + count, d->stream), "read_staged scratch");
        flags = buf + bytes;
        launch_read_staged(c, d->stream, tok_begin, count, buf, flags);
        ck(cudaGetLastError(), "read_staged launch");
        ck(cudaMemcpyAsync(out, buf, bytes, cudaMemcpyDeviceToHost, d->stream), "read_staged D2H");
        if (in_window)
            ck(cudaMemcpyAsync(in_window, flags, count, cudaMemcpyDeviceToHost, d->stream), "read_staged D2H");
        ck(cudaFreeAsync(buf, d->stream), "read_staged free");
        ck(cudaStreamSynchronize(d->stream), "read_staged sync");
    });
}

int kvr_dev_fault(kvr_dev *d, int what, uint64_t arg) {
    return guard([&] {
        if (what != KVR_FAULT_DROP_SPAN && what != KVR_FAULT_SHIFT_ROWS)
            throw std::runtime_error("unknown fault");
        ck(cudaStreamSynchronize(d->stream), "fault sync");
        ck(cudaMemcpy(const_cast<uint64_t *>(d->base.fault) + (what - 1), &arg, sizeof(arg), cudaMemcpyHostToDevice),
           "fault set");
    });
}

// `iters` launches of K-attn / K-gather alone on the last launched step's descriptor;
// each launch's own span (first-CTA start to last exit, the kernel's %globaltimer stamps —
// ncu's gpu__time_duration), averaged: launch gaps between back-to-back launches are
// not the kernel's time.
static int time_kernel(kvr_dev *d, uint32_t iters, double *ms, bool attn) {
    return guard([&] {
        ck(cudaStreamSynchronize(d->stream), "sync");
        // the last launched step's descriptor is still resident in its slot
        const int k = d->launched[1] > d->launched[0] ? 1 : 0;
        const DevCtx c = ctx_for(d, k);
        if (attn && !d->attn)
            throw std::runtime_error("attention disabled");
        uint64_t *span = attn ? &c.scan->attn_t0 : &c.scan->gather_t0;
        const uint64_t reset[2] = {~0ull, 0ull};
        double total = 0.0;
        for (uint32_t i = 0; i <= iters; ++i) { // (the first launch warms up, untimed)
            ck(cudaMemcpyAsync(span, reset, sizeof(reset), cudaMemcpyHostToDevice, d->stream), "span reset");
            if (attn)
                launch_attn(d->attn, c, d->stream);
            else
                launch_gather(c, d->stream, d->sms);
            uint64_t got[2];
            ck(cudaMemcpyAsync(got, span, sizeof(got), cudaMemcpyDeviceToHost, d->stream), "span read");
            ck(cudaStreamSynchronize(d->stream), "sync");
            if (i > 0 && got[1] > got[0])
                total += double(got[1] - got[0]) * 1e-6;
        }
        *ms = iters ? total / iters : 0.0;
    });
}

int kvr_dev_time_attention(kvr_dev *d, uint32_t iters, double *ms) { return time_kernel(d, iters, ms, true); }

int kvr_dev_timeline(kvr_dev *d, uint64_t *out) {
    return guard([&] {
        if (!d->base.tl)
            throw std::runtime_error("timeline off (set KVR_TIMELINE=1 before kvr_dev_open)");
        ck(cudaStreamSynchronize(d->stream), "sync");
        ck(cudaMemcpy(out, d->base.tl, sizeof(uint64_t) * 2 * KVR_TIMELINE_IDS, cudaMemcpyDeviceToHost), "timeline");
        tl_reset(d->base.tl, d->stream);
        ck(cudaStreamSynchronize(d->stream), "sync");
    });
}
int kvr_dev_time_gather(kvr_dev *d, uint32_t iters, double *ms) { return time_kernel(d, iters, ms, false); }

const char *kvr_dev_attention_variant(kvr_dev *d) { return attn_variant(d->attn); }

int kvr_dev_utility(kvr_dev *d, uint32_t k, kvr_mass_run *out, uint32_t *counts) {
    return guard([&] {
        if (k > 1)
            throw std::runtime_error("step ring slot must be 0 or 1");
        if (!d->base.utility)
            throw std::runtime_error("utility observations are off (geometry.utility = 0)");
        if (d->in_flight[k])
            throw std::runtime_error("the step of this ring slot has not been waited for");
        const DevCtx &c = d->base;
        if (d->launched[k] % c.utility)
            throw std::runtime_error("K-mass did not run on that step (geometry.utility)");
        std::memcpy(counts, d->h_mass_count[k], uint64_t(c.n_slots) * 4);
        for (uint32_t s = 0; s < c.n_slots; ++s)
            std::memcpy(out + uint64_t(s) * c.W, d->h_mass[k] + uint64_t(s) * c.W,
                        std::min<uint32_t>(counts[s], c.W) * sizeof(kvr_mass_run));
    });
}

int kvr_dev_ring_plane_rows(kvr_dev *d, uint32_t *out) {
    return guard([&] { *out = d->base.Rp; });
}

int kvr_comm_unique_id(uint8_t id[128]) {
    return guard([&] {
        ncclUniqueId u;
        nck(nccl().get_unique_id(&u), "ncclGetUniqueId");
        static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id, &u, sizeof(u));
    });
}

int kvr_comm_init(kvr_dev *d, const uint8_t id[128], int rank, int world) {
    return guard([&] {
        if (d->comm)
            throw std::runtime_error("kvr_comm_init: communicator already set");
        if (d->n_launches)
            throw std::runtime_error("kvr_comm_init must precede the first step launch (graph capture)");
        if (world < 1 || rank < 0 || rank >= world)
            throw std::runtime_error("kvr_comm_init: bad rank / world");
        ck(cudaSetDevice(d->g.device), "cudaSetDevice");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        nck(nccl().comm_init_rank(&d->comm, world, u, rank), "ncclCommInitRank");
        d->rank = rank;
        d->world = world;
    });
}

int kvr_comm_destroy(kvr_dev *d) {
    return guard([&] {
        if (d->n_launches)
            throw std::runtime_error("kvr_comm_destroy: the step graphs already hold the collective");
        if (d->comm)
            nck(nccl().comm_destroy(d->comm), "ncclCommDestroy");
        d->comm = nullptr;
        d->rank = 0;
        d->world = 1;
    });
}

int kvr_comm_world(kvr_dev *d, int *rank, int *world) {
    return guard([&] {
        *rank = d->rank;
        *world = d->world;
    });
}

int kvr_dev_step_kernels(kvr_dev *d, uint32_t *out) {
    return guard([&] { *out = d->graph_kernels; });
}

int kvr_dev_graph_captures(kvr_dev *d, uint32_t *out) {
    return guard([&] { *out = d->graph_captures; });
}

} // extern "C"
