/* kvr_oracle.c — TEST INFRASTRUCTURE (CPU oracle), not product code.
 * Plain-C restatement of the reference's decode-step algorithms; see
 * kvr_oracle.h for the contract and the file:line each function follows. */
#include "kvr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

uint64_t kvo_splitmix64(uint64_t x) { /* scenario.cpp:34-39 */
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

static uint64_t pattern(uint64_t seed, uint32_t session, uint64_t token, uint64_t lane) {
    /* Driver::payload_pattern, scenario.cpp:189-191 */
    return kvo_splitmix64(seed ^ ((uint64_t)session << 32) ^ (token << 8) ^ lane);
}

static float lane_value(uint64_t h) { /* scenario.cpp:200 */
    return (float)((int64_t)(h % 2001) - 1000) / 1000.0f;
}

void kvo_fill_token_payload(uint64_t seed, uint32_t session, uint64_t token, uint64_t token_bytes,
                            uint32_t elem_bytes, void *out) {
    /* Driver::fill_token_payload, scenario.cpp:193-206 */
    if (elem_bytes == 4) {
        float *f = (float *)out;
        uint32_t lanes = (uint32_t)(token_bytes / 4);
        for (uint32_t l = 0; l < lanes; ++l)
            f[l] = lane_value(pattern(seed, session, token, l));
    } else {
        uint8_t *b = (uint8_t *)out;
        for (uint64_t i = 0; i < token_bytes; ++i)
            b[i] = (uint8_t)(pattern(seed, session, token, i) & 0xff);
    }
}

float kvo_half_to_float(uint16_t h) {
    uint32_t sign = (uint32_t)(h >> 15) << 31;
    uint32_t exp = (h >> 10) & 0x1f;
    uint32_t man = h & 0x3ff;
    uint32_t bits;
    if (exp == 0) {
        if (man == 0) {
            bits = sign;
        } else { /* subnormal */
            float f = (float)man * (1.0f / 16777216.0f); /* 2^-24 */
            memcpy(&bits, &f, 4);
            bits |= sign;
        }
    } else if (exp == 31) {
        bits = sign | 0x7f800000u | (man << 13);
    } else {
        bits = sign | ((exp + 112) << 23) | (man << 13);
    }
    float out;
    memcpy(&out, &bits, 4);
    return out;
}

uint16_t kvo_float_to_half(float f) { /* IEEE binary16, round to nearest even */
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t absx = x & 0x7fffffffu;
    if (absx >= 0x7f800000u) /* inf / nan */
        return (uint16_t)(sign | 0x7c00u | (absx > 0x7f800000u ? 0x200u : 0u));
    if (absx >= 0x477ff000u) /* rounds to >= 65520 -> inf */
        return (uint16_t)(sign | 0x7c00u);
    if (absx < 0x38800000u) { /* below 2^-14: subnormal half */
        if (absx < 0x33000000u) /* < 2^-25 rounds to zero */
            return (uint16_t)sign;
        uint32_t e = absx >> 23;
        uint32_t m = (absx & 0x7fffffu) | 0x800000u;
        uint32_t shift = 126 - e; /* 14..24 */
        uint32_t q = m >> shift;
        uint32_t rem = m & ((1u << shift) - 1u);
        uint32_t half = 1u << (shift - 1);
        if (rem > half || (rem == half && (q & 1u)))
            ++q;
        return (uint16_t)(sign | q);
    }
    uint32_t q = absx - 0x38000000u; /* rebias exponent 127 -> 15 */
    uint32_t rem = q & 0x1fffu;
    q >>= 13;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u)))
        ++q;
    return (uint16_t)(sign | q);
}

float kvo_bf16_to_float(uint16_t h) {
    uint32_t bits = (uint32_t)h << 16;
    float out;
    memcpy(&out, &bits, 4);
    return out;
}

uint16_t kvo_float_to_bf16(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    if ((x & 0x7fffffffu) > 0x7f800000u)
        return (uint16_t)((x >> 16) | 0x40u);
    uint32_t r = x + 0x7fffu + ((x >> 16) & 1u);
    return (uint16_t)(r >> 16);
}

static void store_lane(void *out, uint64_t i, float v, int elem_kind) {
    if (elem_kind == 0)
        ((float *)out)[i] = v;
    else if (elem_kind == 1)
        ((uint16_t *)out)[i] = kvo_float_to_half(v);
    else
        ((uint16_t *)out)[i] = kvo_float_to_bf16(v);
}

static float load_lane(const void *in, uint64_t i, int elem_kind) {
    if (elem_kind == 0)
        return ((const float *)in)[i];
    if (elem_kind == 1)
        return kvo_half_to_float(((const uint16_t *)in)[i]);
    return kvo_bf16_to_float(((const uint16_t *)in)[i]);
}

void kvo_fill_token_lanes_shift(uint64_t seed, uint32_t session, uint64_t token, uint64_t lanes,
                                int elem_kind, uint32_t shift, void *out) {
    if (elem_kind == 0) { /* fp32: the reference float pattern, scenario.cpp:198-201 */
        for (uint64_t l = 0; l < lanes; ++l)
            store_lane(out, l, lane_value(pattern(seed, session, token, l)), elem_kind);
        return;
    }
    /* 2-byte lanes: one splitmix64 per group of 8 lanes (16 bytes; tweaked by
     * bit 62), lane j of the group takes byte j: (b - 128) / 2^shift, exact in fp16
     * and bf16 (shift 7: [-1, 1); shift 3, "wide": [-16, 16)) */
    for (uint64_t l = 0; l < lanes; ++l) {
        const uint64_t x = pattern(seed, session, token, (l >> 3) ^ 0x4000000000000000ull);
        const uint32_t b = (uint32_t)((x >> (8 * (l & 7))) & 0xffu);
        store_lane(out, l, (float)((int)b - 128) / (float)(1u << shift), elem_kind);
    }
}

void kvo_fill_token_lanes(uint64_t seed, uint32_t session, uint64_t token, uint64_t lanes,
                          int elem_kind, void *out) {
    kvo_fill_token_lanes_shift(seed, session, token, lanes, elem_kind, 7, out);
}

void kvo_fill_query_mode(uint64_t seed, uint32_t session, uint64_t step, uint32_t layer,
                         uint32_t head, uint32_t head_dim, int elem_kind, int mode, float *out) {
    if (mode == 1) { /* KVR_QUERY_F32: two 24-bit lanes per splitmix64, (u - 2^23) / 2^23 */
        for (uint32_t d = 0; d < head_dim; ++d) {
            uint64_t h = kvo_splitmix64(seed ^ (0x52ull << 56) ^ ((uint64_t)session << 32) ^
                                        (step << 20) ^ ((uint64_t)layer << 12) ^
                                        ((uint64_t)head << 8) ^ (d >> 1));
            uint32_t u = (uint32_t)(h >> (32 * (d & 1)));
            out[d] = (float)((int32_t)(u >> 8) - 8388608) * (1.0f / 8388608.0f);
        }
        return;
    }
    kvo_fill_query(seed, session, step, layer, head, head_dim, elem_kind, out);
}

void kvo_fill_query(uint64_t seed, uint32_t session, uint64_t step, uint32_t layer,
                    uint32_t head, uint32_t head_dim, int elem_kind, float *out) {
    for (uint32_t d = 0; d < head_dim; ++d) {
        uint64_t h = kvo_splitmix64(seed ^ (0x51ull << 56) ^ ((uint64_t)session << 32) ^
                                    (step << 20) ^ ((uint64_t)layer << 12) ^
                                    ((uint64_t)head << 8) ^ (d >> 3));
        float v = (float)((int)((h >> (8 * (d & 7))) & 0xffull) - 128) / 128.0f; /* exact in every type */
        if (elem_kind == 1)
            v = kvo_half_to_float(kvo_float_to_half(v));
        else if (elem_kind == 2)
            v = kvo_bf16_to_float(kvo_float_to_bf16(v));
        out[d] = v;
    }
}

/* ---- transport ------------------------------------------------------------- */

typedef struct {
    uint64_t begin, len;
} range_t;

static int cmp_range(const void *a, const void *b) {
    const range_t *x = (const range_t *)a, *y = (const range_t *)b;
    if (x->begin != y->begin)
        return x->begin < y->begin ? -1 : 1;
    if (x->len != y->len)
        return x->len < y->len ? -1 : 1;
    return 0;
}

int kvo_stage(const kvr_stage_need *needs, uint64_t n_needs, const kvr_staged_span *spans,
              uint64_t page_bytes, uint64_t token_bytes, double now, kvr_descriptor *out,
              uint64_t cap, uint64_t *n_out) {
    /* transport.cpp:29-61 */
    uint64_t n = 0;
    for (uint64_t k = 0; k < n_needs; ++k) {
        const kvr_stage_need *need = &needs[k];
        range_t *r = (range_t *)malloc(sizeof(range_t) * (need->span_count + 1));
        uint64_t m = 0;
        for (uint64_t i = 0; i < need->span_count; ++i) {
            const kvr_staged_span *sp = &spans[need->span_begin + i];
            if (sp->slot_count == 0)
                continue;
            r[m].begin = (uint64_t)sp->block * page_bytes + (uint64_t)sp->slot_begin * token_bytes;
            r[m].len = (uint64_t)sp->slot_count * token_bytes;
            ++m;
        }
        qsort(r, m, sizeof(range_t), cmp_range);
        for (uint64_t i = 0; i < m; ++i) {
            uint64_t begin = r[i].begin, len = r[i].len;
            while (i + 1 < m && r[i + 1].begin == begin + len) {
                len += r[i + 1].len;
                ++i;
            }
            if (out && n < cap) {
                kvr_descriptor d;
                memset(&d, 0, sizeof(d));
                d.phys_offset = begin;
                d.length = len;
                d.kind = need->kind;
                d.stage_time = now;
                d.block = (uint32_t)(begin / page_bytes);
                d.session = need->session;
                out[n] = d;
            }
            ++n;
        }
        free(r);
    }
    *n_out = n;
    return 0;
}

typedef struct {
    const kvr_descriptor *d;
    uint64_t idx;
} dref_t;

static int cmp_dref(const void *a, const void *b) {
    const dref_t *x = (const dref_t *)a, *y = (const dref_t *)b;
    if (x->d->kind != y->d->kind)
        return x->d->kind < y->d->kind ? -1 : 1;
    if (x->d->phys_offset != y->d->phys_offset)
        return x->d->phys_offset < y->d->phys_offset ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

int kvo_reduce(const kvr_descriptor *descs, uint64_t n, const kvr_transport_config *cfg,
               double now, kvr_train *trains, uint64_t train_cap, uint64_t *n_trains,
               kvr_descriptor *ordered, uint64_t *ties) {
    /* transport.cpp:22-27 (validate) and 63-127 */
    if (cfg->merge_threshold == 0 || cfg->max_hold < 0.0)
        return KVR_E_BAD_CONFIG;
    *n_trains = 0;
    if (ties)
        *ties = 0;
    if (n == 0)
        return 0;
    uint64_t nt = 0;
    if (!cfg->merge) {
        for (uint64_t i = 0; i < n; ++i) {
            if (trains && i < train_cap) {
                kvr_train t;
                memset(&t, 0, sizeof(t));
                t.kind = descs[i].kind;
                t.total_bytes = descs[i].length;
                t.oldest_stage_time = descs[i].stage_time;
                t.issue_time = now;
                t.reason = 2;
                t.desc_begin = i;
                t.desc_count = 1;
                trains[i] = t;
            }
            if (ordered)
                ordered[i] = descs[i];
        }
        *n_trains = n;
        return 0;
    }
    dref_t *v = (dref_t *)malloc(sizeof(dref_t) * n);
    for (uint64_t i = 0; i < n; ++i) {
        v[i].d = &descs[i];
        v[i].idx = i;
    }
    qsort(v, n, sizeof(dref_t), cmp_dref);
    if (ties)
        for (uint64_t i = 1; i < n; ++i)
            if (v[i].d->kind == v[i - 1].d->kind && v[i].d->phys_offset == v[i - 1].d->phys_offset)
                ++*ties;
    int open = 0;
    kvr_train cur;
    memset(&cur, 0, sizeof(cur));
    const kvr_descriptor *prev = NULL;
#define KVO_CLOSE(R)                                                                            \
    do {                                                                                        \
        cur.reason = (R);                                                                       \
        cur.issue_time = now;                                                                   \
        if (trains && nt < train_cap)                                                           \
            trains[nt] = cur;                                                                   \
        ++nt;                                                                                   \
        open = 0;                                                                               \
    } while (0)
    for (uint64_t i = 0; i < n; ++i) {
        const kvr_descriptor *d = v[i].d;
        if (open) {
            /* exact abutment (transport.cpp:85-110), or the B200 page-run rule: a descriptor
             * ending at a page's last token slot abuts the next page's start */
            const uint64_t end = prev->phys_offset + prev->length;
            int adjacent = prev->kind == d->kind &&
                           (end == d->phys_offset ||
                            (cfg->run_page_bytes && end % cfg->run_page_bytes == cfg->run_span_bytes &&
                             d->phys_offset == end - cfg->run_span_bytes + cfg->run_page_bytes));
            if (cur.total_bytes >= cfg->merge_threshold)
                KVO_CLOSE(0);
            else if (now - cur.oldest_stage_time >= cfg->max_hold)
                KVO_CLOSE(1);
            else if (!adjacent)
                KVO_CLOSE(2);
        }
        if (!open) {
            memset(&cur, 0, sizeof(cur));
            cur.kind = d->kind;
            cur.oldest_stage_time = d->stage_time;
            cur.desc_begin = i;
            open = 1;
        }
        cur.total_bytes += d->length;
        if (d->stage_time < cur.oldest_stage_time)
            cur.oldest_stage_time = d->stage_time;
        cur.desc_count += 1;
        if (ordered)
            ordered[i] = *d;
        prev = d;
    }
    if (open)
        KVO_CLOSE(cur.total_bytes >= cfg->merge_threshold ? 0 : 2);
#undef KVO_CLOSE
    free(v);
    *n_trains = nt;
    return 0;
}

/* ---- far view ---------------------------------------------------------------- */

void kvo_summarize_chunk(const float *tokens, uint32_t lanes, uint64_t count, float *out) {
    /* far_view.cpp:30-47 */
    double *acc = (double *)calloc(lanes, sizeof(double));
    for (uint64_t t = 0; t < count; ++t)
        for (uint32_t l = 0; l < lanes; ++l)
            acc[l] += tokens[t * lanes + l];
    const double inv = 1.0 / (double)count;
    for (uint32_t l = 0; l < lanes; ++l)
        out[l] = (float)(acc[l] * inv);
    free(acc);
}

static const double *g_scores;
static int cmp_score(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    if (g_scores[x] != g_scores[y])
        return g_scores[x] > g_scores[y] ? -1 : 1;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

uint64_t kvo_select_chunks(const double *scores, uint64_t n, uint32_t cap, uint64_t *out) {
    /* far_view.cpp:49-62 (comparator is a strict total order, so qsort = stable_sort) */
    uint64_t *ids = (uint64_t *)malloc(sizeof(uint64_t) * (n + 1));
    for (uint64_t i = 0; i < n; ++i)
        ids[i] = i;
    g_scores = scores;
    qsort(ids, n, sizeof(uint64_t), cmp_score);
    uint64_t m = n < cap ? n : cap;
    qsort(ids, m, sizeof(uint64_t), cmp_u64);
    memcpy(out, ids, m * sizeof(uint64_t));
    free(ids);
    return m;
}

void kvo_attend_rows(const float *k, uint64_t k_stride, const float *v, uint64_t v_stride,
                     uint64_t n, const float *query, uint32_t d, float *out) {
    /* attend, far_view.cpp:113-155 */
    for (uint32_t i = 0; i < d; ++i)
        out[i] = 0.0f;
    if (n == 0)
        return;
    const double scale = 1.0 / sqrt((double)d);
    double *logits = (double *)malloc(sizeof(double) * n);
    for (uint64_t s = 0; s < n; ++s) {
        const float *kr = k + s * k_stride;
        double dot = 0.0;
        for (uint32_t i = 0; i < d; ++i)
            dot += (double)query[i] * (double)kr[i];
        logits[s] = dot * scale;
    }
    double m = logits[0];
    for (uint64_t s = 0; s < n; ++s)
        m = logits[s] > m ? logits[s] : m;
    double *acc = (double *)calloc(d, sizeof(double));
    double denom = 0.0;
    for (uint64_t s = 0; s < n; ++s) {
        double w = exp(logits[s] - m);
        denom += w;
        const float *vr = v + s * v_stride;
        for (uint32_t i = 0; i < d; ++i)
            acc[i] += w * (double)vr[i];
    }
    for (uint32_t i = 0; i < d; ++i)
        out[i] = (float)(acc[i] / denom);
    free(acc);
    free(logits);
}

void kvo_attend_window(const void *window, uint64_t n_near, const float *far_images,
                       uint64_t n_far, uint32_t layers, uint32_t kv_heads, uint32_t head_dim,
                       int elem_kind, uint32_t layer, uint32_t kv_head, const float *query,
                       float *out) {
    /* build_view slot order [far..., near...] (far_view.cpp:69-109) then attend. */
    const uint64_t d_kv = (uint64_t)kv_heads * head_dim;
    const uint64_t lanes = 2 * (uint64_t)layers * d_kv;
    const uint64_t n = n_far + n_near;
    float *k = (float *)malloc(sizeof(float) * (n + 1) * head_dim);
    float *v = (float *)malloc(sizeof(float) * (n + 1) * head_dim);
    const uint64_t k_off = 2 * (uint64_t)layer * d_kv + (uint64_t)kv_head * head_dim;
    const uint64_t v_off = k_off + d_kv;
    for (uint64_t s = 0; s < n_far; ++s)
        for (uint32_t i = 0; i < head_dim; ++i) {
            k[s * head_dim + i] = far_images[s * lanes + k_off + i];
            v[s * head_dim + i] = far_images[s * lanes + v_off + i];
        }
    for (uint64_t s = 0; s < n_near; ++s)
        for (uint32_t i = 0; i < head_dim; ++i) {
            k[(n_far + s) * head_dim + i] = load_lane(window, s * lanes + k_off + i, elem_kind);
            v[(n_far + s) * head_dim + i] = load_lane(window, s * lanes + v_off + i, elem_kind);
        }
    kvo_attend_rows(k, head_dim, v, head_dim, n, query, head_dim, out);
    free(k);
    free(v);
}

void kvo_attention_weights(const void *window, uint64_t n_near, const float *far_images,
                           uint64_t n_far, uint32_t layers, uint32_t kv_heads, uint32_t head_dim,
                           int elem_kind, uint32_t layer, uint32_t kv_head, const float *query,
                           double *weights) {
    /* attend's logits (q.k)/sqrt(d) in double, max-subtracted softmax
     * (far_view.cpp:128-150), over build_view's slot order [far..., near...] */
    const uint64_t d_kv = (uint64_t)kv_heads * head_dim;
    const uint64_t lanes = 2 * (uint64_t)layers * d_kv;
    const uint64_t n = n_far + n_near;
    const uint64_t k_off = 2 * (uint64_t)layer * d_kv + (uint64_t)kv_head * head_dim;
    const double scale = 1.0 / sqrt((double)head_dim);
    if (n == 0)
        return;
    for (uint64_t s = 0; s < n; ++s) {
        double dot = 0.0;
        for (uint32_t i = 0; i < head_dim; ++i) {
            const double k = s < n_far ? (double)far_images[s * lanes + k_off + i]
                                       : (double)load_lane(window, (s - n_far) * lanes + k_off + i, elem_kind);
            dot += (double)query[i] * k;
        }
        weights[s] = dot * scale;
    }
    double m = weights[0], denom = 0.0;
    for (uint64_t s = 0; s < n; ++s)
        m = weights[s] > m ? weights[s] : m;
    for (uint64_t s = 0; s < n; ++s) {
        weights[s] = exp(weights[s] - m);
        denom += weights[s];
    }
    for (uint64_t s = 0; s < n; ++s)
        weights[s] /= denom;
}

uint64_t kvo_fnv1a(const void *data, uint64_t n, uint64_t h) {
    const uint8_t *p = (const uint8_t *)data;
    if (h == 0)
        h = 1469598103934665603ull;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}
