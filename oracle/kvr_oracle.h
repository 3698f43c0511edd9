/* kvr_oracle.h — TEST INFRASTRUCTURE (CPU oracle), not product code.
 *
 * Plain-C restatement of the reference algorithms on the KV-RM decode-step
 * path. Each function cites the reference file:line it restates
 * (/root/reference/proj/...). The restatement is pinned against the compiled
 * reference (oracle/_ref/libkvrail_ref.so) and against committed golden
 * vectors in tests/golden/ (see tests/test_oracle.py). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load it; the product path never does.
 */
#ifndef KVR_ORACLE_H
#define KVR_ORACLE_H

#include <stdint.h>

#include "../include/kvrail_c.h"

#ifdef __cplusplus
extern "C" {
#endif

/* splitmix64, scenario.cpp:34-39 */
uint64_t kvo_splitmix64(uint64_t x);

/* Driver::fill_token_payload, scenario.cpp:189-206 (exact): token image of
 * `token_bytes` bytes for (seed, session, token). elem_bytes == 4 gives the
 * float lane pattern ((h % 2001) - 1000) / 1000; otherwise each byte is
 * splitmix64(...) & 0xff. */
void kvo_fill_token_payload(uint64_t seed, uint32_t session, uint64_t token, uint64_t token_bytes,
                            uint32_t elem_bytes, void *out);

/* B200 extension ("lanes" payload mode). elem_kind 0 (f32): the
 * float lane pattern of scenario.cpp:198-201, equal to kvo_fill_token_payload.
 * 2-byte lanes (1 f16, 2 bf16): one splitmix64 per 8 lanes, lane j of the group
 * = byte j: (b - 128) / 128, exact in both types. */
void kvo_fill_token_lanes(uint64_t seed, uint32_t session, uint64_t token, uint64_t lanes,
                          int elem_kind, void *out);
/* The same with lane = (b - 128) / 2^shift (shift 7 = kvo_fill_token_lanes; shift 3 =
 * the "wide" payload, [-16, 16): large logits, peaked softmaxes). */
void kvo_fill_token_lanes_shift(uint64_t seed, uint32_t session, uint64_t token, uint64_t lanes,
                                int elem_kind, uint32_t shift, void *out);

/* Synthetic decode query for (seed, session, step, layer, q_head): hd floats,
 * lane d = (b - 128) / 128 with b the byte d & 7 of
 * h = splitmix64(seed ^ 0x51<<56 ^ session<<32 ^ step<<20 ^ layer<<12 ^ head<<8
 * ^ (d >> 3)) — one hash per 8 lanes, like the 2-byte KV lanes; exact in every
 * element type. (A B200-side synthetic input: the reference has no query.) */
void kvo_fill_query(uint64_t seed, uint32_t session, uint64_t step, uint32_t layer,
                    uint32_t head, uint32_t head_dim, int elem_kind, float *out);
/* mode 0 = kvo_fill_query; mode 1 (KVR_QUERY_F32): lane d = (u - 2^23) / 2^23 with u the
 * top 24 bits of 32-bit half d & 1 of h = splitmix64(seed ^ 0x52<<56 ^ session<<32 ^
 * step<<20 ^ layer<<12 ^ head<<8 ^ (d >> 1)): random fp32 in [-1, 1), generally not
 * representable in fp16 / bf16 (the tensor-core kernel's lo query half is non-zero). */
void kvo_fill_query_mode(uint64_t seed, uint32_t session, uint64_t step, uint32_t layer,
                         uint32_t head, uint32_t head_dim, int elem_kind, int mode, float *out);

float kvo_half_to_float(uint16_t h);
float kvo_bf16_to_float(uint16_t h);
uint16_t kvo_float_to_half(float f);
uint16_t kvo_float_to_bf16(float f);

/* stage(), transport.cpp:29-61 */
int kvo_stage(const kvr_stage_need *needs, uint64_t n_needs, const kvr_staged_span *spans,
              uint64_t page_bytes, uint64_t token_bytes, double now, kvr_descriptor *out,
              uint64_t cap, uint64_t *n_out);

/* reduce(), transport.cpp:63-127. Sort is (kind, offset) with the input index
 * as tie-break: identical to the reference whenever no two descriptors share
 * (kind, offset); *ties reports how many adjacent equal keys were seen. */
int kvo_reduce(const kvr_descriptor *descs, uint64_t n, const kvr_transport_config *cfg,
               double now, kvr_train *trains, uint64_t train_cap, uint64_t *n_trains,
               kvr_descriptor *ordered, uint64_t *ties);

/* summarize_chunk, far_view.cpp:30-47 */
void kvo_summarize_chunk(const float *tokens, uint32_t lanes, uint64_t count, float *out);

/* select_chunks, far_view.cpp:49-62; returns the picked count */
uint64_t kvo_select_chunks(const double *scores, uint64_t n, uint32_t cap, uint64_t *out);

/* attend, far_view.cpp:113-155, over `n` non-padded slots given as separate
 * K and V rows of d floats each (row i at k + i*k_stride). */
void kvo_attend_rows(const float *k, uint64_t k_stride, const float *v, uint64_t v_stride,
                     uint64_t n, const float *query, uint32_t d, float *out);

/* Window attention oracle for one (session, layer, q-head): the exact near
 * window is the last min(written, W*) token images in `window` (token-major,
 * token_bytes each, element type elem_kind), far summaries (fp32, token
 * images) come first as in build_view (far_view.cpp:64-111). GQA: q-head h
 * reads kv-head h / group. Output: head_dim floats. */
void kvo_attend_window(const void *window, uint64_t n_near, const float *far_images,
                       uint64_t n_far, uint32_t layers, uint32_t kv_heads, uint32_t head_dim,
                       int elem_kind, uint32_t layer, uint32_t kv_head, const float *query,
                       float *out);

/* The softmax weights attend() (far_view.cpp:113-155) puts on each of the
 * n_far + n_near view slots of kvo_attend_window's view, in view order (far
 * summaries first), in double — the oracle of K-mass (kvr_mass.cu). */
void kvo_attention_weights(const void *window, uint64_t n_near, const float *far_images,
                           uint64_t n_far, uint32_t layers, uint32_t kv_heads, uint32_t head_dim,
                           int elem_kind, uint32_t layer, uint32_t kv_head, const float *query,
                           double *weights);

/* FNV-1a 64 over bytes (the hash used by the parity traces). */
uint64_t kvo_fnv1a(const void *data, uint64_t n, uint64_t seed_h);

#ifdef __cplusplus
}
#endif
#endif
