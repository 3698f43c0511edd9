/* kvrail_c.h — C-ABI of the B200 KV-RM decode-step path (host side).
 *
 * This is the drop-in boundary: plain pointers, sizes and POD structs, no
 * torch or C++ types. Every entry point replaces one public function of the
 * reference C++ library `kvrail` (/root/reference/proj/include/kvrail/...);
 * the replaced declaration is cited next to each function. The C++ mirror of
 * the reference headers lives in include/kvrail/ (*.hpp) and is implemented by
 * the same shared library (libkvrail.so); this C layer wraps it so that any
 * FFI (ctypes, cgo, JNI, N-API) can bind the path. See INTEGRATION.md.
 *
 * Error convention: every function returns 0 on success, or 1 + Errc (the
 * reference error taxonomy, types.hpp:45-68) on failure. KVR_E_CUDA marks a
 * CUDA runtime failure (kept outside the Errc parity range).
 * kvr_last_error() returns the thread-local "<ErrcName>: message" string,
 * identical in form to kvrail::Error::what() (types.hpp:72-77).
 */
#ifndef KVRAIL_C_H
#define KVRAIL_C_H

#include <stddef.h>
#include <stdint.h>

#include "kvr_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1 + kvrail::Errc (types.hpp:45-68) ------------------ */
enum {
    KVR_OK = 0,
    KVR_E_OUT_OF_PAGES = 1,
    KVR_E_PREFIX_OUT_OF_RANGE,
    KVR_E_ALIAS_OVERLAP,
    KVR_E_UNMAPPED_RANGE,
    KVR_E_FUTURE_DELTA,
    KVR_E_UNKNOWN_SESSION,
    KVR_E_SESSION_CLOSED,
    KVR_E_EMPTY_CHUNK,
    KVR_E_DIMENSION_MISMATCH,
    KVR_E_SHAPE_VIOLATION,
    KVR_E_MULTI_COMMIT,
    KVR_E_UNMAPPED_BLOCK,
    KVR_E_PARSE_ERROR,
    KVR_E_NON_MONOTONE_TIME,
    KVR_E_EMPTY_STREAM,
    KVR_E_UNKNOWN_REGIME,
    KVR_E_INFEASIBLE_SPEC,
    KVR_E_WORKLOAD_AUDIT_FAILED,
    KVR_E_EMPTY_RUN,
    KVR_E_WORKLOAD_MISMATCH,
    KVR_E_BAD_CONFIG,
    KVR_E_IO_ERROR,
    KVR_E_CUDA = 100,     /* CUDA runtime / launch failure */
    KVR_E_INTERNAL = 101, /* any other exception */
};

/* Thread-local message of the last failing call ("<ErrcName>: msg"). */
const char *kvr_last_error(void);
/* sizeof of every POD struct of kvrail_c.h and kvr_cuda.h, in declaration
 * order (FFI layout self-check); *n = number of structs. */
int kvr_abi_struct_sizes(uint64_t *out, uint64_t cap, uint64_t *n);
/* kvrail::errc_name (types.cpp:20-46) for a status code (code - 1). */
const char *kvr_errc_name(int status);

/* ---- POD mirrors of the reference value types --------------------------- */
typedef struct kvr_pager_config { /* PagerConfig, pager.hpp:34-48 */
    uint64_t page_bytes;
    uint32_t arena_pages;
    uint32_t layers;
    uint32_t kv_head_dim;
    uint32_t elem_bytes;
} kvr_pager_config;

typedef struct kvr_token_range { /* TokenRange, types.hpp:32-43 */
    uint64_t begin;
    uint64_t end;
} kvr_token_range;

typedef struct kvr_view_entry { /* ViewEntry, pager.hpp:52-56 */
    uint64_t tok_begin;
    uint64_t tok_end;
    uint32_t block;
    uint32_t slot_begin;
} kvr_view_entry;

typedef struct kvr_view_info { /* ViewDescriptor header, pager.hpp:59-68 */
    uint32_t session;
    uint32_t eos;
    uint64_t epoch;
    uint64_t live_tokens;
    uint64_t extent;
    uint64_t n_entries; /* total entries; min(n_entries, cap) were copied */
} kvr_view_info;

typedef struct kvr_reserved_block { /* ReservedBlock, pager.hpp:104-107 */
    uint32_t block;
    uint32_t token_capacity;
} kvr_reserved_block;

typedef struct kvr_arena_stats { /* ArenaStats, pager.hpp:82-88 */
    uint64_t free_pages;
    uint64_t live_pages;
    uint64_t shared_pages;
    uint64_t reserved_bytes;
    uint64_t active_bytes;
} kvr_arena_stats;

typedef struct kvr_work_counters { /* WorkCounters, pager.hpp:92-102 */
    uint64_t commits;
    uint64_t commit_entries_touched;
    uint64_t reserve_calls;
    uint64_t reserve_blocks;
    uint64_t reserve_alloc_steps;
    uint64_t trim_calls;
    uint64_t trim_blocks;
    uint64_t free_list_steps;
} kvr_work_counters;

typedef struct kvr_free_run {
    uint32_t head;
    uint32_t length;
} kvr_free_run;

typedef struct kvr_frame_delta { /* FrameDelta, pager.hpp:71-80 (flattened) */
    uint32_t session;
    uint32_t trim_eos;
    uint64_t step;
    const uint64_t *reserves;
    uint64_t n_reserves;
    const uint32_t *alias_src;         /* n_aliases entries */
    const uint64_t *alias_prefix;      /* n_aliases entries */
    uint64_t n_aliases;
    const kvr_token_range *trims;
    uint64_t n_trims;
} kvr_frame_delta;

/* Transport (transport.hpp:25-67). kind: 0 near_window, 1 far_view.
 * reason: 0 threshold, 1 age, 2 flush. */
typedef struct kvr_staged_span { /* StagedSpan, transport.hpp:50-54 */
    uint32_t block;
    uint32_t slot_begin;
    uint32_t slot_count;
} kvr_staged_span;

typedef struct kvr_stage_need { /* StageNeed, transport.hpp:56-60; spans index a flat array */
    uint32_t session;
    uint32_t kind;
    uint64_t span_begin;
    uint64_t span_count;
} kvr_stage_need;

typedef struct kvr_descriptor { /* Descriptor, transport.hpp:27-34 */
    uint64_t phys_offset;
    uint64_t length;
    double stage_time;
    uint32_t kind;
    uint32_t block;
    uint32_t session;
    uint32_t pad_;
} kvr_descriptor;

typedef struct kvr_transport_config { /* TransportConfig, transport.hpp:17-23 */
    uint64_t merge_threshold;
    double max_hold;
    uint32_t max_trains_per_step;
    uint32_t merge;
    /* B200 page-run merge (0, 0 = the reference's exact abutment; transport.hpp abuts()) */
    uint64_t run_page_bytes, run_span_bytes;
} kvr_transport_config;

typedef struct kvr_train { /* DmaTrain, transport.hpp:38-45; descriptors live in a flat array */
    uint64_t total_bytes;
    double oldest_stage_time;
    double issue_time;
    uint32_t kind;
    uint32_t reason;
    uint64_t desc_begin;
    uint64_t desc_count;
} kvr_train;

typedef struct kvr_step_record { /* StepRecord, sim_engine.hpp:47-63 + measured device times */
    uint64_t step;
    uint32_t live_sessions;
    uint32_t trains;
    uint32_t near_trains;
    uint32_t far_trains;
    uint64_t dma_bytes;
    double mean_train_bytes;
    double max_hold;
    double submit_time;
    double commit_time;
    double step_latency;
    uint64_t reserved_bytes;
    uint64_t active_bytes;
    uint32_t commits;
    uint32_t pad_;
    uint64_t emitted_tokens;
    /* B200 additions (0 on a host-only driver) */
    double device_ms;          /* CUDA-event time of this step's graph replay */
    double gather_ms;          /* K-gather kernel alone */
    double attn_ms;            /* K-attn kernel alone */
    double phase_ms[8];        /* device time per step phase (kvr_step_stats) */
    uint64_t writeback_tokens; /* token rows written to the arena this step */
    uint64_t gather_bytes;     /* bytes the gather moved (read side) */
    uint64_t attn_bytes;       /* KV bytes the window attention read */
    uint64_t h2d_bytes;        /* committed step descriptor bytes copied host -> device */
    uint64_t end_ns;           /* device %globaltimer at the end of the step: successive
                                  differences are the inter-token latency */
    /* job-wide counts of this step: the in-graph NCCL all-reduce over every GPU of
       the communicator (kvr_driver_comm_init); this GPU's own without one */
    uint64_t global_live, global_emitted, global_commits, global_eos;
} kvr_step_record;

/* ---- Pager (pager.hpp:121-183) ------------------------------------------ */
typedef struct kvr_pager kvr_pager;
typedef struct kvr_device kvr_device; /* see kvr_cuda.h / kvr_device_open */

/* Pager(PagerConfig), pager.hpp:123. Payload bytes live in host memory. */
int kvr_pager_create(const kvr_pager_config *cfg, kvr_pager **out);
/* Same, with the page payload resident in the B200 arena of `dev`. */
int kvr_pager_create_on_device(const kvr_pager_config *cfg, kvr_device *dev, kvr_pager **out);
int kvr_pager_destroy(kvr_pager *p);
/* PagerConfig::validate, pager.cpp:29-38 */
int kvr_pager_config_validate(const kvr_pager_config *cfg);
/* create_session / has_session, pager.hpp:131-132 */
int kvr_pager_create_session(kvr_pager *p, uint32_t session);
int kvr_pager_has_session(kvr_pager *p, uint32_t session, int *out);
/* reserve, pager.hpp:138; out may be NULL to count only */
int kvr_pager_reserve(kvr_pager *p, uint32_t session, uint64_t token_count,
                      kvr_reserved_block *out, uint64_t cap, uint64_t *n_out);
/* reserve_range, pager.hpp:142 */
int kvr_pager_reserve_range(kvr_pager *p, uint32_t session, kvr_token_range range,
                            kvr_reserved_block *out, uint64_t cap, uint64_t *n_out);
/* alias, pager.hpp:146 */
int kvr_pager_alias(kvr_pager *p, uint32_t dst, uint32_t src, uint64_t prefix_tokens,
                    uint64_t *shared_out);
/* write_tokens, pager.hpp:150 (host payload; copied to the device arena when attached) */
int kvr_pager_write_tokens(kvr_pager *p, uint32_t session, kvr_token_range range,
                           const void *payload, uint64_t payload_bytes);
/* trim / trim_eos, pager.hpp:154-155 */
int kvr_pager_trim(kvr_pager *p, uint32_t session, const kvr_token_range *ranges, uint64_t n,
                   uint64_t *freed_out);
int kvr_pager_trim_eos(kvr_pager *p, uint32_t session, uint64_t *freed_out);
/* frame_commit, pager.hpp:159 */
int kvr_pager_frame_commit(kvr_pager *p, uint32_t session, uint64_t step, uint64_t *epoch_out);
/* apply_frame, pager.hpp:163 */
int kvr_pager_apply_frame(kvr_pager *p, const kvr_frame_delta *delta, uint64_t *epoch_out);
/* active_view, pager.hpp:166 */
int kvr_pager_active_view(kvr_pager *p, uint32_t session, kvr_view_info *info,
                          kvr_view_entry *entries, uint64_t cap);
/* session_eos / session_cursor / next_step / touched_in_last_commit, pager.hpp:168-174 */
int kvr_pager_session_eos(kvr_pager *p, uint32_t session, int *out);
int kvr_pager_session_cursor(kvr_pager *p, uint32_t session, uint64_t *out);
int kvr_pager_next_step(kvr_pager *p, uint32_t session, uint64_t *out);
int kvr_pager_touched_in_last_commit(kvr_pager *p, uint32_t session, uint64_t *out);
/* stats / counters, pager.hpp:171-172 */
int kvr_pager_stats(kvr_pager *p, kvr_arena_stats *out);
int kvr_pager_counters(kvr_pager *p, kvr_work_counters *out);
/* read_slots, pager.hpp:177 (device arena: synchronous D2H) */
int kvr_pager_read_slots(kvr_pager *p, uint32_t block, uint32_t slot_begin, uint32_t slot_count,
                         void *out);
/* free_runs / block_refcount, pager.hpp:181-183 */
int kvr_pager_free_runs(kvr_pager *p, kvr_free_run *out, uint64_t cap, uint64_t *n_out);
int kvr_pager_block_refcount(kvr_pager *p, uint32_t block, uint32_t *out);

/* ---- Transport (transport.hpp:71-93) ------------------------------------ */
/* stage(), transport.hpp:71-72 */
int kvr_stage(const kvr_stage_need *needs, uint64_t n_needs, const kvr_staged_span *spans,
              uint64_t page_bytes, uint64_t token_bytes, double now, kvr_descriptor *out,
              uint64_t cap, uint64_t *n_out);
/* reduce(), transport.hpp:81-82. `ordered` receives the descriptors in train
 * order (n entries); trains[i].desc_begin/desc_count index into it. */
int kvr_reduce(const kvr_descriptor *descs, uint64_t n, const kvr_transport_config *cfg,
               double now, kvr_train *trains, uint64_t train_cap, uint64_t *n_trains,
               kvr_descriptor *ordered);

/* ---- Far view (far_view.hpp:40-75) -------------------------------------- */
/* summarize_chunk, far_view.hpp:42-43 */
int kvr_summarize_chunk(const float *tokens, uint32_t lanes, uint64_t count, float *out);
/* select_chunks, far_view.hpp:74 */
int kvr_select_chunks(const double *scores, uint64_t n, uint32_t cap, uint64_t *out,
                      uint64_t *n_out);
/* attend over build_view(history of `t` token images, far_view.hpp:63-70). Token
 * images are `lanes` floats, token-major; out has kv_head_dim floats. */
int kvr_attend_history(const float *images, uint64_t t, const double *chunk_scores,
                       uint64_t n_scores, uint32_t lanes, uint32_t near_window, uint32_t cap,
                       uint32_t chunk_tokens, const float *query, uint32_t layer,
                       uint32_t kv_head_dim, float *out);

/* ---- Scenario driver (scenario.hpp:95-117 / scenario.cpp:124-683) -------
 * config_json uses the reference config schema (scenario.cpp:829-924) plus an
 * optional "b200" object (device, attention geometry, payload mode); see
 * DESIGN.md. device < 0 runs the host-only twin driver (no CUDA). */
typedef struct kvr_driver kvr_driver;
int kvr_driver_create(const char *config_json, int device, kvr_driver **out);
int kvr_driver_destroy(kvr_driver *d);
/* One Driver::step (scenario.cpp:450-682). Device fields of the returned
 * record are filled one step later; fetch them with kvr_driver_record. */
int kvr_driver_step(kvr_driver *d, kvr_step_record *out);
/* Record of an executed step including its device measurements. */
int kvr_driver_record(kvr_driver *d, uint64_t step, kvr_step_record *out);
/* Wait for all device work of the driver (no-op on a host-only driver). */
int kvr_driver_sync(kvr_driver *d);
/* Steps executed so far / configured total. */
int kvr_driver_progress(kvr_driver *d, uint64_t *done, uint64_t *total);
/* steps.csv (scenario.cpp:706-725) / report.json (scenario.cpp:727-766) of
 * the steps run so far; copies min(len, cap) bytes, *len = full length. */
int kvr_driver_steps_csv(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len);
int kvr_driver_report_json(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len);
/* B200 measurement formats (no reference counterpart): steps.csv
   columns + per-step device measurements, and the measured report over post-warm-up
   steps. Both first complete every executed step's device measurements. */
int kvr_driver_measured_csv(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len);
int kvr_driver_measured_json(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len);
/* b200.prefill_budget bookkeeping: cold prompt tokens queued now, and tokens never
   written because their page was recycled before anything read them */
int kvr_driver_prefill_backlog(kvr_driver *d, uint64_t *queued, uint64_t *dropped);
/* Per-step parity trace (trains, pager digest); enabled by "b200.trace". */
int kvr_driver_trace(kvr_driver *d, char *buf, uint64_t cap, uint64_t *len);
/* The driver's pager (borrowed; valid until kvr_driver_destroy). */
int kvr_driver_pager(kvr_driver *d, kvr_pager **out);
/* Device slot bookkeeping for parity checks: live sessions in slot order. */
int kvr_driver_live(kvr_driver *d, uint32_t *slot, uint32_t *session, uint64_t *written,
                    uint64_t cap, uint64_t *n_out);
/* Resolved workload stream hash (workload.cpp stream_hash). */
int kvr_driver_workload_hash(kvr_driver *d, uint64_t *out);
/* b200.check: steps whose device K-scan was compared with host reduce(),
 * mismatching steps and the first mismatch description. */
int kvr_driver_device_check(kvr_driver *d, uint64_t *checked, uint64_t *mismatches, char *buf,
                            uint64_t cap);
/* b200.trace on a device: staged tokens the trace hashed from K-gather's destination
 * (window ring / far rows), near rows behind the live window (hashed from the arena:
 * not part of the window) and rows missing from the window for any other reason. */
int kvr_driver_staged_rows(kvr_driver *d, uint64_t *delivered, uint64_t *behind, uint64_t *missing);
/* Join the per-step counts all-reduce over NCCL (kvr_comm_init, kvr_cuda.h) before
 * the first step: `id` from kvr_comm_unique_id on one rank, distributed by the caller. */
int kvr_driver_comm_init(kvr_driver *d, const uint8_t id[128], int rank, int world);
/* Test hook (fault injection, kvr_dev_fault): K-gather drops a span (KVR_FAULT_DROP_SPAN)
 * or misplaces near rows (KVR_FAULT_SHIFT_ROWS) on every later step. */
int kvr_driver_fault(kvr_driver *d, int what, uint64_t arg);

/* ---- B200 device (kvrail::DeviceStep) ---------------------------------------
 * A device context: arena, page-table mirror, window ring and the step graph
 * (include/kvr_cuda.h documents the geometry). Replaces the reference's
 * simulated device SimEngine (sim_engine.hpp:67-88). Pass it to
 * kvr_pager_create_on_device to keep a Pager's payload in HBM. */
int kvr_device_open(const struct kvr_geometry *geometry, kvr_device **out);
int kvr_device_close(kvr_device *d);
int kvr_device_flush(kvr_device *d);
int kvr_device_geometry(kvr_device *d, struct kvr_geometry *out);
int kvr_device_bind(kvr_device *d, uint32_t session, uint32_t slot);
int kvr_driver_device(kvr_driver *d, kvr_device **out);
int kvr_device_raw(kvr_device *d, struct kvr_dev **out);
/* parity reads (synchronous) */
int kvr_device_read_ring_token(kvr_device *d, uint32_t slot, uint64_t token, void *out);
int kvr_device_read_page_table(kvr_device *d, uint32_t slot, uint64_t tok_begin, uint64_t count,
                               uint32_t *out);
int kvr_device_read_attention(kvr_device *d, uint32_t slot, float *out);
int kvr_device_read_query(kvr_device *d, uint32_t slot, float *out);
int kvr_device_read_far_row(kvr_device *d, uint32_t slot, uint64_t chunk, void *out);
/* far chunks (select_chunks, far_view.cpp:49-62) the last step showed slot's attention */
int kvr_device_far_selection(kvr_device *d, uint32_t slot, uint64_t *out, uint64_t cap,
                             uint64_t *n_out);
int kvr_device_read_scan(kvr_device *d, kvr_train *trains, uint64_t train_cap, uint64_t *n_trains,
                         kvr_descriptor *descs, uint64_t desc_cap, uint64_t *n_descs);
/* b200.utility = attention: the K-mass observations of `step` (waits for it; valid
 * until step + 2 is launched) — runs[slot * near_window, + counts[slot]) of
 * {block, mass}: the probe layer's softmax weight on each block of the slot's
 * window, mean over q-heads (the placement tracker's observations). */
int kvr_device_utility(kvr_device *d, uint64_t step, struct kvr_mass_run *runs, uint32_t *counts);

#ifdef __cplusplus
}
#endif
#endif /* KVRAIL_C_H */
