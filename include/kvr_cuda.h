/* kvr_cuda.h — thin C-ABI between the kvrail host C++ and the sm_100a kernels.
 *
 * libkvr_cuda.so implements it. It replaces the reference's simulated device
 * (SimEngine::execute_step, sim_engine.cpp:33-72, and the cost-model "issue"
 * CostModel::dma_time, sim_engine.hpp:42-44) with a real B200 step: a device
 * arena of pages, a device page-table mirror of the committed views, a
 * fixed-shape window ring per slot, and one committed step descriptor per
 * step consumed by a captured CUDA graph. All structs are POD; offsets in the
 * descriptor are bytes from its start; every section is 16-byte aligned.
 * Status codes follow kvrail_c.h (0 ok, KVR_E_CUDA for CUDA failures).
 */
#ifndef KVR_CUDA_H
#define KVR_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { KVR_ELEM_F32 = 0, KVR_ELEM_F16 = 1, KVR_ELEM_BF16 = 2 };
enum { KVR_PAYLOAD_BYTES = 0, KVR_PAYLOAD_LANES = 1 };
/* decode queries: EXACT = byte fields (b - 128) / 128, exact in the KV type (the
 * tensor-core kernel's lo half is 0); F32 = 24-bit random fp32 in [-1, 1), not
 * representable in 16 bits (exercises the hi + lo query split) */
enum { KVR_QUERY_EXACT = 0, KVR_QUERY_F32 = 1 };
#define KVR_NO_SLOT 0xffffffffu
#define KVR_SUMMARY_BASE (1ull << 40) /* summary slots' logical tokens, scenario.cpp:41 */
#define KVR_MAX_SCAN_NEEDS 1024u      /* K-scan: stage needs per step */
/* per-step counts all-reduced across GPUs: live sessions, emitted
 * tokens, commit frames (commits_observed, sim_engine.cpp:41-44), EOS this step */
#define KVR_COUNTS 4
enum { KVR_COUNT_LIVE = 0, KVR_COUNT_EMITTED = 1, KVR_COUNT_COMMITS = 2, KVR_COUNT_EOS = 3 };

typedef struct kvr_geometry {
    int32_t device;
    int32_t elem_kind;      /* KVR_ELEM_* (attention / lanes interpretation) */
    uint32_t elem_bytes;    /* PagerConfig::elem_bytes */
    uint32_t payload_mode;  /* KVR_PAYLOAD_* */
    uint64_t page_bytes;
    uint64_t token_bytes;   /* 2 * L * kv_heads * head_dim * elem_bytes */
    uint32_t arena_pages;
    uint32_t tokens_per_page;
    uint32_t layers;
    uint32_t kv_heads;
    uint32_t head_dim;
    uint32_t q_heads;
    uint32_t n_slots;       /* fixed batch width (Driver concurrency) */
    uint32_t near_window;   /* W* */
    uint32_t ring_rows;     /* R >= W*, multiple of 32 */
    uint32_t far_cap;       /* far slots visible to attention (0 = no far view) */
    uint32_t chunk_tokens;  /* sv_chunk */
    uint32_t max_chunks;    /* far rows kept per slot */
    uint64_t max_tokens;    /* per-slot capacity of the device page table */
    uint64_t seed;          /* synthetic payload seed (ScenarioConfig::seed) */
    uint32_t attention;     /* K-attn each step: 0 off, 1 auto, 2 CUDA-core kernel, 3 tcgen05 kernel */
    uint32_t use_graph;     /* replay the step as a CUDA graph */
    uint64_t max_desc_bytes;/* capacity of one step descriptor */
    uint32_t max_scan_descs;/* K-scan capacity (descriptors / spans) */
    uint32_t max_trains;
    uint32_t utility;       /* N >= 1: K-mass measures attention-utility observations on
                               steps with step % N == 0 (0: off) */
    uint32_t utility_layer; /* probe layer of K-mass */
    uint32_t lane_shift;    /* 2-byte lanes payload: lane = (b - 128) / 2^lane_shift
                               (0 = 7: [-1, 1); 3 = "wide" [-16, 16), peaked softmaxes) */
    uint32_t query_mode;    /* KVR_QUERY_* */
} kvr_geometry;

/* K-mass output: one run of window rows mapped to one arena block, with the
 * softmax weight the probe layer's q-heads put on it (mean over q-heads). */
typedef struct kvr_mass_run { uint32_t block; float mass; } kvr_mass_run;

/* ---- committed step descriptor ------------------------------------------ */
typedef struct kvr_step_header {
    uint64_t step;
    double now;             /* transport clock (stage_time of every descriptor) */
    uint64_t tau;           /* TransportConfig::merge_threshold */
    double max_hold;        /* TransportConfig::max_hold */
    uint32_t merge;
    uint32_t n_zero, n_cow, n_edit, n_write, n_blob, n_need, n_span, n_prime, n_far_ids;
    uint32_t n_far_jobs;    /* source-1 ops: the last n_far_jobs of the n_write ops */
    uint32_t n_cold;        /* write ops are [hot ... | cold ... | far jobs ...]; cold ops
                               touch rows no kernel of this step reads and run after
                               the attention */
    uint32_t n_presum;      /* far chunks summarised while their prompt rows are written */
    uint64_t write_tokens;  /* sum of kvr_write_op.count over hot source-0 writes */
    uint64_t write_tokens_cold; /* ... over cold source-0 writes */
    uint64_t off_zero, off_cow, off_edit, off_write, off_blob_ops, off_blob, off_need, off_span,
        off_prime, off_far_ids, off_slots;
    uint64_t off_presum, off_presum_runs;
    uint32_t n_presum_runs, pad_h;
    uint64_t total_bytes;
    int64_t counts[KVR_COUNTS]; /* this GPU's per-step counts (KVR_COUNT_*): the input of
                                   the in-graph NCCL all-reduce when a communicator is set */
    uint64_t run_page, run_span; /* TransportConfig::run_page_bytes / run_span_bytes (page-run
                                    merge, a B200 policy; 0 = exact abutment only) */
    uint64_t off_src_rows;       /* u32 global slots (block * tpp + slot) read by K-far jobs and
                                    K-prime ops, resolved by the host: those kernels do not read
                                    the page table, so they run in one kernel with K-map */
    uint32_t n_src_rows, pad_r;
} kvr_step_header;

typedef struct kvr_zero_op { uint32_t block, slot_begin, slot_count, pad; } kvr_zero_op;
typedef struct kvr_cow_op { uint32_t src, dst; } kvr_cow_op;
/* committed view delta: tokens [tok_begin,tok_end) of `slot` -> block/slot_begin
 * (block == 0xffffffff: unmapped). Tokens >= KVR_SUMMARY_BASE are summary slots. */
typedef struct kvr_edit_op {
    uint64_t tok_begin, tok_end;
    uint32_t slot, block, slot_begin, pad;
} kvr_edit_op;
/* payload generated in place: source 0 = synthetic token payload of
 * (session, token..token+count); source 1 = far summary of chunk tokens
 * [aux, aux + chunk_tokens) of `dev_slot` written to (block, slot), the chunk's
 * rows being src_rows[prefix, prefix + chunk_tokens); source 2 =
 * the same summary, already computed by K-presum into the stash row
 * (dev_slot, aux / chunk_tokens), copied to (block, slot). */
typedef struct kvr_write_op {
    uint64_t token;
    uint64_t aux;
    uint64_t prefix;        /* source 0: exclusive prefix of count over the ops; source 1:
                               first index of the chunk's rows in the src_rows section */
    uint32_t block, slot, count, session;
    uint32_t dev_slot;      /* KVR_NO_SLOT: arena only */
    uint32_t source;
} kvr_write_op;
/* K-presum: a far-view chunk whose prompt rows are all written this step, by one
 * session, is generated column by column in token order (runs [run_begin,
 * run_begin + run_count) of the run list) and its mean kept in the stash row
 * (dev_slot, chunk): the far job a step later copies it instead of re-reading the
 * chunk_tokens rows (bit-identical: the same double sums in the same order). */
typedef struct kvr_presum_op { uint32_t session, dev_slot, chunk, run_begin, run_count, pad; } kvr_presum_op;
typedef struct kvr_presum_run { uint64_t token; uint32_t block, slot, count, pad; } kvr_presum_run;
/* host payload bytes (Pager::write_tokens) carried in the descriptor blob */
typedef struct kvr_blob_op {
    uint64_t blob_offset;
    uint32_t block, slot, count, pad;
} kvr_blob_op;
typedef struct kvr_need_rec {
    uint32_t slot, session, kind, span_begin, span_count, pad;
} kvr_need_rec;
typedef struct kvr_span_rec {
    uint64_t first_token;   /* logical token of slot_begin */
    uint32_t block, slot_begin, slot_count, pad;
} kvr_span_rec;
typedef struct kvr_prime_op {
    uint64_t tok_begin, tok_end;
    uint32_t slot;
    uint32_t rows;          /* first index of the tokens' source rows in src_rows */
} kvr_prime_op;
/* one per device slot, always n_slots entries */
typedef struct kvr_slot_state {
    uint64_t written;       /* tokens appended (attention length) after this step */
    uint32_t session;
    uint32_t live;          /* attention runs for this slot this step */
    uint32_t far_begin;     /* index into the far-id array */
    uint32_t far_count;     /* selected far chunks (<= far_cap) */
    /* tokens [stage_lo, stage_hi) of this slot are covered by this step's near-window
       staged spans: K-gather is their only window writer this step (K-write and
       K-prime leave those ring rows to it), so the window consumes the staged bytes */
    uint64_t stage_lo, stage_hi;
} kvr_slot_state;

/* step results (written by the device, read back one step later) */
typedef struct kvr_step_stats {
    uint64_t step;
    double device_ms;       /* descriptor H2D + step kernels + stats D2H */
    double gather_ms;       /* K-gather alone (event nodes inside the graph) */
    double attn_ms;         /* K-attn alone */
    double phase_ms[8];     /* apply | hot writes+query | far+map+prime | scan | gather |
                               attn | wait for the cold-write branch | (unused) */
    uint32_t trains, descriptors, spans, status;
    uint64_t train_bytes;
    uint64_t staged_tokens;
    uint64_t writeback_tokens;
    uint64_t attn_bytes;
    uint64_t end_ns;          /* device %globaltimer at the end of the step */
    int64_t global_counts[KVR_COUNTS]; /* the step's counts summed over all ranks of the
                                          communicator (this GPU's own without one) */
} kvr_step_stats;

typedef struct kvr_dev kvr_dev;

const char *kvr_dev_last_error(void);
int kvr_dev_count(int *out);
int kvr_dev_open(const kvr_geometry *g, kvr_dev **out);
int kvr_dev_close(kvr_dev *d);
/* pinned host memory for descriptors (two ring slots of max_desc_bytes) */
int kvr_dev_desc_buffer(kvr_dev *d, uint32_t ring_slot, void **out);
/* publish ring slot `ring_slot` (desc_bytes used) and launch the step */
int kvr_dev_launch(kvr_dev *d, uint32_t ring_slot, uint64_t desc_bytes);
/* byte-only apply of a descriptor outside a step (zero/cow/writes/edits) */
int kvr_dev_apply_only(kvr_dev *d, uint32_t ring_slot, uint64_t desc_bytes);
/* wait for the step launched from `ring_slot` and return its stats */
int kvr_dev_wait(kvr_dev *d, uint32_t ring_slot, kvr_step_stats *out);
int kvr_dev_sync(kvr_dev *d);

enum {
    KVR_BUF_ARENA = 0,   /* bytes */
    KVR_BUF_RING = 1,    /* [slot][layer][plane row][2*d_kv] elements (kvr_dev_ring_plane_rows) */
    KVR_BUF_TMAP = 2,    /* [slot][max_tokens] u32 global slot index */
    KVR_BUF_OUT = 3,     /* [slot][layer][q_head][head_dim] f32 */
    KVR_BUF_QUERY = 4,   /* [slot][layer][q_head][head_dim] f32 */
    KVR_BUF_FAR = 5,     /* [slot][layer][max_chunks][2*d_kv] elements */
    KVR_BUF_TRAINS = 6,  /* kvr_train[max_trains] (kvrail_c.h layout) */
    KVR_BUF_DESCS = 7,   /* kvr_descriptor[max_scan_descs] in train order */
    KVR_BUF_SCAN = 8,    /* u32 counters: trains, descriptors, spans, status */
    KVR_BUF_SMAP = 9,    /* [slot][max_chunks] u32 summary-slot map */
};
int kvr_dev_read(kvr_dev *d, int buffer, uint64_t offset, uint64_t bytes, void *out);
/* K-gather's DESTINATION bytes of the last step's staged tokens [tok_begin, tok_begin +
 * count) in train order (the order of the trains' descriptors): each token
 * as the reference lays it out (token_bytes, layer rows [K_l|V_l] concatenated), read
 * back from the window ring (near spans) or the far rows (far spans). A row the window
 * does not hold is read from the arena instead. `in_window` (count bytes, may be NULL):
 * 1 delivered; 0 a near row behind the live window (older than written - W*, not part
 * of the window by definition); 2 not held for another reason (never expected). */
int kvr_dev_read_staged(kvr_dev *d, uint64_t tok_begin, uint64_t count, void *out, uint8_t *in_window);
/* fault injection for the parity tests (never set by the product path):
 * KVR_FAULT_DROP_SPAN: K-gather skips gather-list span `arg` (~0 = off,
 *                      KVR_FAULT_ALL = every span);
 * KVR_FAULT_SHIFT_ROWS: K-gather writes near rows `arg` ring rows too far (0 = off). */
enum { KVR_FAULT_DROP_SPAN = 1, KVR_FAULT_SHIFT_ROWS = 2 };
#define KVR_FAULT_ALL (~1ull)
int kvr_dev_fault(kvr_dev *d, int what, uint64_t arg);
int kvr_dev_buffer_bytes(kvr_dev *d, int buffer, uint64_t *out);
/* rows per (slot, layer) plane of KVR_BUF_RING: ring_rows + the guard rows that mirror
 * rows [0, guard) (the tensor-core attention's whole-tile loads never split) */
int kvr_dev_ring_plane_rows(kvr_dev *d, uint32_t *out);
/* `iters` launches of the last launched step's attention (K-gather) kernel alone: the
 * mean of each launch's own span (first-CTA start to last exit, %globaltimer — the
 * quantity ncu reports as gpu__time_duration; launch gaps are not counted) */
int kvr_dev_time_attention(kvr_dev *d, uint32_t iters, double *ms_per_launch);
int kvr_dev_time_gather(kvr_dev *d, uint32_t iters, double *ms_per_launch);
/* diagnostic kernel timeline (only when KVR_TIMELINE=1 was set at kvr_dev_open): for each
 * kernel id (0 apply, 1 queries, 2 K-scan, 3 hot K-write, 4 K-far/map/prime, 5 K-gather,
 * 6 K-attn, 7 cold K-write, 8 K-presum, 9 tensor-core K-attn's CTA entry before its prologue) the %globaltimer ns of its first CTA start and
 * last warp exit since the previous call, out[2 id], out[2 id + 1] (~0 / 0: not run);
 * synchronises the step stream and resets */
#define KVR_TIMELINE_IDS 16
int kvr_dev_timeline(kvr_dev *d, uint64_t out[2 * KVR_TIMELINE_IDS]);
/* name of the attention kernel variant chosen for this geometry */
const char *kvr_dev_attention_variant(kvr_dev *d);
/* attention-utility observations of the step launched from `ring_slot` (call after
 * kvr_dev_wait for it; valid until that ring slot is launched again): runs
 * [slot * near_window, + counts[slot]) of `out` (n_slots * near_window entries) */
int kvr_dev_utility(kvr_dev *d, uint32_t ring_slot, kvr_mass_run *out, uint32_t *counts);
/* ---- multi-GPU: per-step counts over NCCL (NVLink / NVSwitch) -------------------
 * Requests shard by sequence; the KV data path never leaves its GPU. With a
 * communicator, every step graph ends with ONE ncclAllReduce (sum, int64) of the
 * descriptor's counts[KVR_COUNTS] into a device buffer, read back with the step
 * stats: job-wide tok/s, termination and the job-wide single-commit audit. NCCL is
 * loaded at run time (dlopen "libnccl.so.2", the copy already in the process when
 * there is one). Call kvr_comm_init before the first kvr_dev_launch (the graphs are
 * captured with the collective in them); every rank must launch the same number of
 * steps. */
int kvr_comm_unique_id(uint8_t id[128]); /* on one rank; the caller distributes it */
int kvr_comm_init(kvr_dev *d, const uint8_t id[128], int rank, int world);
int kvr_comm_world(kvr_dev *d, int *rank, int *world); /* (0, 1) without a communicator */
int kvr_comm_destroy(kvr_dev *d); /* drop the communicator (before the first launch only) */
/* kernel nodes in the captured step graph (0 before the first graph launch) */
int kvr_dev_step_kernels(kvr_dev *d, uint32_t *out);
/* step graphs captured so far: 2 (one per descriptor ring slot) after the first two
   steps and never more — the fixed shape means no recapture (sim_engine.cpp:33-72 audit) */
int kvr_dev_graph_captures(kvr_dev *d, uint32_t *out);

#ifdef __cplusplus
}
#endif
#endif /* KVR_CUDA_H */
