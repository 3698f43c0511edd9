// kvrail-b200 byte-level step kernels (HBM-bound integer/byte work).
//
//   K-apply : zero recycled page slots, copy-on-write page copies, host blobs
//   K-write : generate this step's token payloads (reference pattern) into the
//             arena and the window ring; generate the decode queries
//   K-far   : far-view chunk summaries (double accumulation, bit-exact)
//   K-map   : committed view edits -> device page table
//   K-prime : window rows not produced by this step's writes
//
// All loops are grid-stride with 16-byte vector accesses; grids are multiples
// of the SM count and sized for the worst case so the step graph never changes.
#include <type_traits>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

__device__ inline void zero16(uint8_t *p) { *reinterpret_cast<int4 *>(p) = make_int4(0, 0, 0, 0); }

// ---------------------------------------------------------------------------
// K-apply: zero ops (recycled page slots), COW page copies and host blobs in ONE
// kernel. The host keeps the three independent within a descriptor (a copy whose
// source has a pending zero or write, or a blob into a copy's destination, splits
// the wave: device_step.cpp), so they need no ordering here. Every op is spread
// over the whole grid (a zero run or a page copy can be megabytes).
__global__ void k_apply(DevCtx c) {
    pdl_trigger(); // (first kernel of the step: no PDL predecessor)
    TlScope tl_(c, kTlApply);
    const kvr_step_header *h = hdr(c);
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x, stride = uint64_t(gridDim.x) * blockDim.x;
    const kvr_zero_op *zops = section<kvr_zero_op>(c, h->off_zero);
    for (uint32_t i = 0; i < h->n_zero; ++i) {
        const kvr_zero_op op = zops[i];
        uint8_t *dst = c.arena + uint64_t(op.block) * c.page_bytes + uint64_t(op.slot_begin) * c.token_bytes;
        const uint64_t n16 = uint64_t(op.slot_count) * c.token_bytes / 16;
        for (uint64_t k = tid; k < n16; k += stride)
            zero16(dst + 16 * k);
    }
    const kvr_cow_op *cops = section<kvr_cow_op>(c, h->off_cow);
    for (uint32_t i = 0; i < h->n_cow; ++i) {
        const int4 *src = reinterpret_cast<const int4 *>(c.arena + uint64_t(cops[i].src) * c.page_bytes);
        int4 *dst = reinterpret_cast<int4 *>(c.arena + uint64_t(cops[i].dst) * c.page_bytes);
        for (uint64_t k = tid; k < c.page_bytes / 16; k += stride)
            dst[k] = src[k];
    }
    // host payload bytes (Pager::write_tokens): blob offsets and token_bytes are
    // multiples of 16, so every op moves int4s
    const kvr_blob_op *bops = section<kvr_blob_op>(c, h->off_blob_ops);
    const uint8_t *blob = c.desc + h->off_blob;
    for (uint32_t i = 0; i < h->n_blob; ++i) {
        const kvr_blob_op op = bops[i];
        int4 *dst = reinterpret_cast<int4 *>(c.arena + uint64_t(op.block) * c.page_bytes +
                                             uint64_t(op.slot) * c.token_bytes);
        const int4 *src = reinterpret_cast<const int4 *>(blob + op.blob_offset);
        const uint64_t n16 = uint64_t(op.count) * c.token_bytes / 16;
        for (uint64_t k = tid; k < n16; k += stride)
            dst[k] = src[k];
    }
}

// ---------------------------------------------------------------------------
// K-write: one CTA per written token (grid-stride), 16 bytes per thread-step.

__device__ inline uint16_t f2h_bits(float v) { return __half_as_ushort(__float2half_rn(v)); }
__device__ inline uint16_t f2b_bits(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }

// Lane values of the reference pattern, ((h % 2001) - 1000) / 1000 (scenario.cpp:200),
// precomputed once per CTA in the element encoding: a table lookup replaces the
// division and the rounding on the hot path (bit-identical by construction).
struct LaneTable {
    uint32_t v[2001];
    __device__ void fill(const DevCtx &c) {
        for (uint32_t i = threadIdx.x; i < 2001; i += blockDim.x) {
            const float f = float(int(i) - 1000) / 1000.0f;
            v[i] = c.esz == 4 ? __float_as_uint(f)
                              : (c.elem_kind == KVR_ELEM_BF16 ? f2b_bits(f) : f2h_bits(f));
        }
        __syncthreads();
    }
    __device__ uint32_t operator()(uint64_t h) const { return v[h % 2001ull]; }
};


enum PayloadKind { kBytes = 0, kLanes16 = 1, kLanes32 = 2 };

/// 2-byte lanes (B200 extension, kvo_fill_token_lanes): one splitmix64 per 8 lanes
/// (16 bytes) of token `tok` of session `sid`, lane j = byte j of the hash.
__device__ __forceinline__ uint64_t lanes16_hash(const DevCtx &c, uint32_t sid, uint64_t tok, uint64_t b0) {
    return splitmix64(c.seed ^ (uint64_t(sid) << 32) ^ (tok << 8) ^ 0x4000000000000000ull ^ (b0 >> 4));
}

/// bf16 lanes: lane value (b - 128) / 2^shift, computed exactly in fp32 (byte_perm
/// places b in the mantissa of 2^23 + b, one exact FFMA rescales) into f[8]; the value
/// has <= 8 significant bits, so its upper 16 bits ARE the bf16 (round-to-nearest-even
/// of an exact value): one PRMT packs two lanes (no F2FP + repack).
__device__ __forceinline__ int4 lanes16_bf16(const DevCtx &c, uint64_t x, float f[8]) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t src = i < 2 ? lo : hi, k = 2 * (i & 1);
        f[2 * i] = fmaf(__uint_as_float(__byte_perm(src, 0x4B000000u, 0x7440 | k)), c.lane_scale, -c.lane_bias);
        f[2 * i + 1] =
            fmaf(__uint_as_float(__byte_perm(src, 0x4B000000u, 0x7440 | (k + 1))), c.lane_scale, -c.lane_bias);
        w[i] = __byte_perm(__float_as_uint(f[2 * i]), __float_as_uint(f[2 * i + 1]), 0x7632);
    }
    return make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
}

/// fp16 lanes: byte b as the half 1024 + b (bits 0x64bb: one PRMT builds two lanes),
/// then ONE exact HFMA2: (1024 + b) * 2^-s - 1152 * 2^-s = (b - 128) * 2^-s.
__device__ __forceinline__ int4 lanes16_f16(const DevCtx &c, uint64_t x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t src = i < 2 ? lo : hi, k = 2 * (i & 1);
        const uint32_t pair = __byte_perm(src, 0x6464u, 0x4040u | k | ((k + 1) << 8));
        const __half2 v = __hfma2(*reinterpret_cast<const __half2 *>(&pair), c.lane_h2_scale, c.lane_h2_bias);
        w[i] = *reinterpret_cast<const uint32_t *>(&v);
    }
    return make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
}

// 16 payload bytes starting at byte `b0` of token `tok` of session `sid`.
template <int kKind>
__device__ __forceinline__ int4 payload16(const DevCtx &c, const LaneTable &tab, uint32_t sid, uint64_t tok,
                                          uint64_t b0) {
    const uint64_t base = c.seed ^ (uint64_t(sid) << 32) ^ (tok << 8);
    uint32_t w[4];
    if constexpr (kKind == kLanes32) { // float lanes (reference pattern for elem_bytes == 4)
        const uint64_t lane0 = b0 / 4;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            w[i] = tab(splitmix64(base ^ (lane0 + i)));
    } else if constexpr (kKind == kLanes16) {
        const uint64_t x = lanes16_hash(c, sid, tok, b0);
        if (c.elem_kind == KVR_ELEM_BF16) {
            float f[8];
            return lanes16_bf16(c, x, f);
        }
        return lanes16_f16(c, x);
    } else { // reference byte pattern: one splitmix per byte
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v |= uint32_t(splitmix64(base ^ (b0 + 4 * i + k)) & 0xff) << (8 * k);
            w[i] = v;
        }
    }
    return make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
}

// `cold`: 0 = the hot write ops (rows read later in this step), 1 = the cold ops
// (older prompt rows nothing in this step reads; launched after K-attn).
template <uint32_t kPer, int kKind> // chunks per thread per unit; payload kind
__device__ __forceinline__ void write_body(const DevCtx &c, int cold, uint32_t bid, uint32_t nblk) {
    __shared__ LaneTable tab;
    const kvr_step_header *h = hdr(c);
    const uint32_t n_hot = h->n_write - h->n_far_jobs - h->n_cold;
    const kvr_write_op *ops = section<kvr_write_op>(c, h->off_write) + (cold ? n_hot : 0);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t n = cold ? h->n_cold : n_hot;
    const uint64_t total = cold ? h->write_tokens_cold : h->write_tokens;
    if (total == 0)
        return;
    if constexpr (kKind == kLanes32) // the lane table serves only the fp32 reference pattern
        tab.fill(c);
    const uint32_t chunks = uint32_t(c.token_bytes / 16);
    const uint32_t row_chunks = c.row_elems * c.esz / 16;
    // work unit = one blockDim-wide slice of 16-byte chunks of one token, so a
    // decode step's few tokens still spread over every SM
    const uint32_t slices = (chunks + kPer * blockDim.x - 1) / (kPer * blockDim.x);
    const uint64_t units = total * slices;
    // each CTA walks a contiguous run of units: one binary search, then the op
    // cursor only moves forward (ops are sorted by token prefix)
    const uint64_t per = (units + nblk - 1) / nblk;
    const uint64_t u0 = bid * per, u1 = min(units, u0 + per);
    uint32_t cur = 0;
    if (u0 < u1) // last op with prefix <= j0 (every warp searches: 2-3 rounds of parallel probes)
        cur = warp_last_le(n, u0 / slices, [&](uint32_t i) { return ops[i].prefix; });
    kvr_write_op op = ops[cur < n ? cur : 0];
    // (token, slice) advance incrementally; per-token addresses are recomputed
    // only when the token changes (no 64-bit division in the loop)
    uint64_t j = u0 / slices;
    uint32_t slice = uint32_t(u0 - j * slices);
    uint64_t j_cached = ~0ull, tok = 0;
    uint8_t *dst = nullptr, *ring = nullptr;
    uint64_t mirror = 0; // bytes to the guard copy of the ring row (0: none)
    const uint64_t ring_layer = uint64_t(c.Rp) * c.row_elems * c.esz; // bytes between layers
    const uint32_t q_base = threadIdx.x;
    for (uint64_t u = u0; u < u1; ++u) {
        if (j != j_cached) {
            j_cached = j;
            while (cur + 1 < n && ops[cur + 1].prefix <= j)
                op = ops[++cur];
            const uint64_t k = j - op.prefix;
            tok = op.token + k;
            dst = c.arena + uint64_t(op.block) * c.page_bytes + (op.slot + k) * c.token_bytes;
            ring = nullptr;
            // inside the live window after this step and not delivered by K-gather
            if (op.dev_slot != KVR_NO_SLOT && ring_owned_by_writer(c, slots[op.dev_slot], tok)) {
                ring = c.ring + ring_row(c, op.dev_slot, 0, uint32_t(tok % c.R)) * c.esz;
                mirror = ring_mirror(c, uint32_t(tok % c.R)) * c.esz;
            }
        }
        if (op.source == 0) {
            int4 v[kPer];
#pragma unroll
            for (uint32_t x = 0; x < kPer; ++x) {
                const uint32_t q = (slice * kPer + x) * blockDim.x + q_base;
                v[x] = q < chunks ? payload16<kKind>(c, tab, op.session, tok, 16ull * q) : int4{};
            }
#pragma unroll
            for (uint32_t x = 0; x < kPer; ++x) {
                const uint32_t q = (slice * kPer + x) * blockDim.x + q_base;
                if (q >= chunks)
                    continue;
                *reinterpret_cast<int4 *>(dst + 16ull * q) = v[x];
                if (ring) {
                    const uint32_t l = q / row_chunks, within = q - l * row_chunks;
                    *reinterpret_cast<int4 *>(ring + l * ring_layer + 16ull * within) = v[x];
                    if (mirror)
                        *reinterpret_cast<int4 *>(ring + mirror + l * ring_layer + 16ull * within) = v[x];
                }
            }
        }
        if (++slice == slices) {
            slice = 0;
            ++j;
        }
    }
}

// Decode queries for live slots: [slot][L][Hq][hd], exact in the KV element type
// (kvo_fill_query in the oracle). One CTA per (slot, layer); one hash per 8 lanes.
/// Two values exact in the element type (<= 8 significant bits), packed: bf16 = the upper
/// halves of the fp32 bits, fp16 = the conversion (exact).
__device__ __forceinline__ uint32_t pack_exact2(const DevCtx &c, float a, float b) {
    if (c.elem_kind == KVR_ELEM_BF16)
        return __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x7632);
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t *>(&h);
}

__device__ __forceinline__ void query_body(const DevCtx &c, uint32_t bid, uint32_t nblk) {
    // byte k of x -> (b - 128) / 128, exactly: b placed in the mantissa of 2^23 + b
    auto val = [](uint32_t x, uint32_t k) {
        return fmaf(__uint_as_float(__byte_perm(x, 0x4B000000u, 0x7440 | k)), 0.0078125f, -65537.f);
    };
    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t per_layer = c.Hq * c.hd;
    for (uint32_t sl = bid; sl < c.n_slots * c.L; sl += nblk) {
        const uint32_t s = sl / c.L, l = sl - s * c.L;
        if (!slots[s].live)
            continue;
        const uint64_t base = c.seed ^ (0x51ull << 56) ^ (uint64_t(slots[s].session) << 32) ^
                              (h->step << 20) ^ (uint64_t(l) << 12);
        float4 *q = reinterpret_cast<float4 *>(c.q + uint64_t(sl) * per_layer);
        int4 *q16 = reinterpret_cast<int4 *>(reinterpret_cast<uint16_t *>(c.q) + uint64_t(sl) * per_layer);
        const uint32_t hd_shift = __ffs(c.hd) - 1; // head_dim is a power of two (32/64/128)
        if (c.query_mode == KVR_QUERY_F32) { // two 24-bit lanes per hash (kvo_fill_query_mode)
            const uint64_t fbase = base ^ (0x52ull << 56) ^ (0x51ull << 56);
            float2 *q2 = reinterpret_cast<float2 *>(q);
            for (uint32_t i = threadIdx.x; i < per_layer / 2; i += blockDim.x) {
                const uint32_t head = (2 * i) >> hd_shift, d2 = i & ((c.hd >> 1) - 1);
                const uint64_t x = splitmix64(fbase ^ (uint64_t(head) << 8) ^ d2);
                q2[i] = make_float2(float(int32_t(uint32_t(x) >> 8) - 8388608) * (1.0f / 8388608.0f),
                                    float(int32_t(uint32_t(x >> 32) >> 8) - 8388608) * (1.0f / 8388608.0f));
            }
            continue;
        }
        // 8 lanes per hash, four independent hashes per thread in flight (ILP: the
        // splitmix chains overlap; one hash per iteration left the kernel latency-bound)
        const uint32_t n8 = per_layer / 8;
        for (uint32_t i0 = threadIdx.x; i0 < n8; i0 += 4 * blockDim.x) {
            uint64_t x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                const uint32_t head = (8 * i) >> hd_shift, d8 = i & ((c.hd >> 3) - 1);
                x[u] = splitmix64(base ^ (uint64_t(head) << 8) ^ d8);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + u * blockDim.x;
                if (i >= n8)
                    break;
                const uint32_t lo = uint32_t(x[u]), hi = uint32_t(x[u] >> 32);
                const float4 a = make_float4(val(lo, 0), val(lo, 1), val(lo, 2), val(lo, 3));
                const float4 b = make_float4(val(hi, 0), val(hi, 1), val(hi, 2), val(hi, 3));
                if (c.q_esz == 4) {
                    q[2 * i] = a;
                    q[2 * i + 1] = b;
                } else { // exact in the element type: 16 bytes per 8 lanes instead of 32
                    q16[i] = make_int4(int(pack_exact2(c, a.x, a.y)), int(pack_exact2(c, a.z, a.w)),
                                       int(pack_exact2(c, b.x, b.y)), int(pack_exact2(c, b.z, b.w)));
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_query(DevCtx c) {
    pdl_trigger();
    TlScope tl_(c, kTlQuery);
    query_body(c, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// K-far: summary of chunk [aux, aux + chunk_tokens) of a slot: double
// accumulation in token order, float(acc * (1/count)) (bit-exact with
// far_view.cpp:36-46 for fp32 lanes; fp16/bf16 lanes round to nearest even).
// Streams 16-byte columns (coalesced, 4 rows in flight per thread).

template <int E> __device__ inline void add_chunk(const DevCtx &c, int4 v, double (&acc)[16 / E]) {
    if constexpr (E == 4) {
        acc[0] += double(__int_as_float(v.x)), acc[1] += double(__int_as_float(v.y));
        acc[2] += double(__int_as_float(v.z)), acc[3] += double(__int_as_float(v.w));
    } else {
        const uint32_t w[4] = {uint32_t(v.x), uint32_t(v.y), uint32_t(v.z), uint32_t(v.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f;
            if (c.elem_kind == KVR_ELEM_BF16)
                f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[i]));
            else
                f = __half22float2(*reinterpret_cast<const __half2 *>(&w[i]));
            acc[2 * i] += double(f.x), acc[2 * i + 1] += double(f.y);
        }
    }
}

/// float(acc * (1/count)) per lane, rounded to the element type (far_view.cpp:36-46).
template <int E> __device__ inline void store_mean(const DevCtx &c, uint8_t *dst, const double (&acc)[16 / E]) {
    const double inv = 1.0 / double(c.chunk_tokens);
    if constexpr (E == 4) {
        *reinterpret_cast<float4 *>(dst) = make_float4(float(acc[0] * inv), float(acc[1] * inv),
                                                       float(acc[2] * inv), float(acc[3] * inv));
    } else {
        uint16_t o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float m = float(acc[i] * inv);
            o[i] = c.elem_kind == KVR_ELEM_BF16 ? f2b_bits(m) : f2h_bits(m);
        }
        *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>(o);
    }
}

/// One CTA per (far job, 4 KiB column block): every thread streams one 16-byte
/// column of the chunk's rows (row offsets staged in shared memory).
template <int E> __device__ void far_columns(const DevCtx &c, const kvr_write_op &op, uint64_t col,
                                             const uint64_t *rows, uint32_t n_rows) {
    constexpr int N = 16 / E;
    double acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
        acc[i] = 0.0;
    uint32_t k = 0;
    for (; k + 4 <= n_rows; k += 4) { // four independent loads in flight
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = rows[k + u] == ~0ull ? make_int4(0, 0, 0, 0)
                                        : __ldcs(reinterpret_cast<const int4 *>(c.arena + rows[k + u] + col));
#pragma unroll
        for (int u = 0; u < 4; ++u)
            add_chunk<E>(c, v[u], acc);
    }
    for (; k < n_rows; ++k)
        if (rows[k] != ~0ull)
            add_chunk<E>(c, __ldcs(reinterpret_cast<const int4 *>(c.arena + rows[k] + col)), acc);
    store_mean<E>(c, c.arena + uint64_t(op.block) * c.page_bytes + uint64_t(op.slot) * c.token_bytes + col, acc);
}

constexpr uint32_t kFarRows = 512; // chunk rows staged in shared memory

// K-far's part of k_fmp: one CTA-iteration per (far job, 4 KiB column block).
__device__ void far_part(const DevCtx &c, uint64_t *rows) {
    const kvr_step_header *h = hdr(c);
    const uint32_t *src_rows = section<uint32_t>(c, h->off_src_rows);
    // far jobs are packed after the token writes
    const kvr_write_op *ops = section<kvr_write_op>(c, h->off_write) + (h->n_write - h->n_far_jobs);
    const uint64_t cols = c.token_bytes / 16; // 16-byte columns per row
    const uint64_t col_blocks = (cols + blockDim.x - 1) / blockDim.x;
    const uint64_t work = uint64_t(h->n_far_jobs) * col_blocks;
    const uint32_t n_rows = min(c.chunk_tokens, kFarRows);
    for (uint64_t u = blockIdx.x; u < work; u += gridDim.x) {
        const kvr_write_op op = ops[u / col_blocks];
        __syncthreads(); // rows[] of the previous unit consumed
        if (op.source == 2) { // summarised by K-presum when its rows were written: copy
            const uint64_t col = (u % col_blocks) * blockDim.x + threadIdx.x;
            if (col < cols) {
                const uint64_t chunk = op.aux / c.chunk_tokens;
                const int4 v = *reinterpret_cast<const int4 *>(
                    c.stash + (uint64_t(op.dev_slot) * c.max_chunks + chunk) * c.token_bytes + 16 * col);
                *reinterpret_cast<int4 *>(c.arena + uint64_t(op.block) * c.page_bytes +
                                          uint64_t(op.slot) * c.token_bytes + 16 * col) = v;
            }
            continue;
        }
        if (op.source != 1)
            continue;
        // the chunk's rows in the view as of the previous commit, resolved by the host
        // (this step's K-map may already have changed the page table)
        for (uint32_t k = threadIdx.x; k < n_rows; k += blockDim.x) {
            const uint32_t gs = src_rows[op.prefix + k];
            rows[k] = gs == kNoMap ? ~0ull : gslot_offset(c, gs); // unmapped: zeros (host validated coverage)
        }
        __syncthreads();
        const uint64_t col = (u % col_blocks) * blockDim.x + threadIdx.x;
        if (col >= cols)
            continue;
        if (c.esz == 4)
            far_columns<4>(c, op, col * 16, rows, n_rows);
        else
            far_columns<2>(c, op, col * 16, rows, n_rows);
    }
}

// ---------------------------------------------------------------------------
// K-presum: prompt rows of whole far-view chunks, generated column by column in
// token order (one CTA per (chunk, 4 KiB column block)), written to the arena and
// summed on the fly — the far job of the next step copies the mean from the
// stash instead of re-reading chunk_tokens rows (same double sums, same order).

template <int kKind> __device__ __forceinline__ void presum_body(const DevCtx &c) {
    __shared__ LaneTable tab;
    const kvr_step_header *h = hdr(c);
    if (h->n_presum == 0)
        return;
    if constexpr (kKind == kLanes32) // the lane table serves only the fp32 reference pattern
        tab.fill(c);
    constexpr int E = kKind == kLanes32 ? 4 : 2;
    const kvr_presum_op *ops = section<kvr_presum_op>(c, h->off_presum);
    const kvr_presum_run *runs = section<kvr_presum_run>(c, h->off_presum_runs);
    const uint64_t cols = c.token_bytes / 16;
    const uint64_t col_blocks = (cols + blockDim.x - 1) / blockDim.x;
    const uint64_t work = uint64_t(h->n_presum) * col_blocks;
    for (uint64_t u = blockIdx.x; u < work; u += gridDim.x) {
        const kvr_presum_op op = ops[u / col_blocks];
        const uint64_t col = (u % col_blocks) * blockDim.x + threadIdx.x;
        if (col >= cols)
            continue;
        double acc[16 / E];
#pragma unroll
        for (int i = 0; i < 16 / E; ++i)
            acc[i] = 0.0;
        // 2-byte lanes are multiples of 2^-shift in [-2^(7-shift), 2^(7-shift)) and a chunk
        // has <= 512 rows, so every partial sum needs <= 7 + 9 + 1 bits and is exact in
        // fp32: summing in fp32 and widening once gives
        // the same double as the reference's double sum (far_view.cpp:36-46), without
        // a conversion and an FP64 add per lane per row
        float accf[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const bool bf = kKind == kLanes16 && c.elem_kind == KVR_ELEM_BF16;
        for (uint32_t r = op.run_begin; r < op.run_begin + op.run_count; ++r) {
            const kvr_presum_run run = runs[r];
            uint8_t *dst = c.arena + uint64_t(run.block) * c.page_bytes + uint64_t(run.slot) * c.token_bytes + 16 * col;
            if (bf) { // bf16 lanes: the generator's exact fp32 values feed the sum directly
                for (uint32_t k = 0; k < run.count; ++k) {
                    float f[8];
                    const int4 v = lanes16_bf16(c, lanes16_hash(c, op.session, run.token + k, 16 * col), f);
                    *reinterpret_cast<int4 *>(dst + uint64_t(k) * c.token_bytes) = v;
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        accf[i] += f[i];
                }
                continue;
            }
            for (uint32_t k = 0; k < run.count; ++k) {
                const int4 v = payload16<kKind>(c, tab, op.session, run.token + k, 16 * col);
                *reinterpret_cast<int4 *>(dst + uint64_t(k) * c.token_bytes) = v;
                if constexpr (kKind == kLanes16) {
                    const uint32_t w[4] = {uint32_t(v.x), uint32_t(v.y), uint32_t(v.z), uint32_t(v.w)};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[i]));
                        accf[2 * i] += f.x, accf[2 * i + 1] += f.y;
                    }
                } else {
                    add_chunk<E>(c, v, acc);
                }
            }
        }
        if constexpr (kKind == kLanes16) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                acc[i] = double(accf[i]);
        }
        store_mean<E>(c, c.stash + (uint64_t(op.dev_slot) * c.max_chunks + op.chunk) * c.token_bytes + 16 * col,
                      acc);
    }
}

// ---------------------------------------------------------------------------
// K-map: committed view edits into the page table (token granularity, so
// mid-block aliases and tail extensions need no special case).

__device__ void map_part(const DevCtx &c) {
    const kvr_step_header *h = hdr(c);
    const kvr_edit_op *ops = section<kvr_edit_op>(c, h->off_edit);
    for (uint32_t i = blockIdx.x; i < h->n_edit; i += gridDim.x) {
        const kvr_edit_op e = ops[i];
        if (e.slot >= c.n_slots)
            continue;
        const bool summary = e.tok_begin >= KVR_SUMMARY_BASE;
        uint32_t *table = summary ? c.smap + uint64_t(e.slot) * c.smap_cap
                                  : c.tmap + uint64_t(e.slot) * c.max_tokens;
        const uint64_t base = summary ? KVR_SUMMARY_BASE : 0;
        const uint64_t cap = summary ? c.smap_cap : c.max_tokens;
        for (uint64_t t = e.tok_begin + threadIdx.x; t < e.tok_end; t += blockDim.x) {
            const uint64_t idx = t - base;
            if (idx >= cap)
                break;
            table[idx] = e.block == kNoMap ? kNoMap
                                           : e.block * c.tpp + e.slot_begin + uint32_t(t - e.tok_begin);
        }
    }
}

// ---------------------------------------------------------------------------
// K-prime: ring rows for tokens of [tok_begin, tok_end) from the arena, each token's
// source row resolved by the host in the committed view; one CTA per (op, token).

__device__ void prime_part(const DevCtx &c) {
    const kvr_step_header *h = hdr(c);
    const kvr_prime_op *ops = section<kvr_prime_op>(c, h->off_prime);
    const uint32_t *src_rows = section<uint32_t>(c, h->off_src_rows);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    for (uint32_t i = 0; i < h->n_prime; ++i) {
        const kvr_prime_op op = ops[i];
        const kvr_slot_state st = slots[op.slot];
        for (uint64_t tok = op.tok_begin + blockIdx.x; tok < op.tok_end; tok += gridDim.x) {
            if (!ring_owned_by_writer(c, st, tok) || tok >= c.max_tokens)
                continue;
            const uint32_t gs = src_rows[op.rows + (tok - op.tok_begin)];
            if (gs == kNoMap)
                continue;
            const uint8_t *src = c.arena + gslot_offset(c, gs);
            uint8_t *ring = c.ring + ring_row(c, op.slot, 0, uint32_t(tok % c.R)) * c.esz;
            const uint64_t mirror = ring_mirror(c, uint32_t(tok % c.R)) * c.esz;
            for (uint64_t q = threadIdx.x; q < c.token_bytes / 16; q += blockDim.x) {
                const uint64_t byte = 16 * q;
                const uint64_t l = byte / row_bytes, within = byte % row_bytes;
                const int4 v = *reinterpret_cast<const int4 *>(src + byte);
                *reinterpret_cast<int4 *>(ring + l * uint64_t(c.Rp) * row_bytes + within) = v;
                if (mirror)
                    *reinterpret_cast<int4 *>(ring + mirror + l * uint64_t(c.Rp) * row_bytes + within) = v;
            }
        }
    }
}

// The step's last kernel stamps its end: the last CTA to finish (a ticket in
// device memory, reset by that CTA) writes %globaltimer — no separate stamp node.
__device__ __forceinline__ void stamp_if_last(const DevCtx &c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(c.attn_sched + 2, 1u) == gridDim.x - 1) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            c.scan->end_ns = t;
            c.attn_sched[2] = 0;
        }
    }
}

// Cold writes (prompt rows nothing in this step reads), column-major like K-presum:
// work unit = (op, 256-column block), thread = one 16-byte column, rows of the op's
// page run in token order. The token-major K-write spends ~1/4 of its issue slots
// re-deriving (token, slice, chunk) per unit; here the per-row cost is the generator
// and one 16-byte store (write-stream bound instead of issue bound).
template <int kKind> __device__ __forceinline__ void write_cols_body(const DevCtx &c, int cold) {
    __shared__ LaneTable tab;
    const kvr_step_header *h = hdr(c);
    const uint32_t n_hot = h->n_write - h->n_far_jobs - h->n_cold;
    const uint32_t n = cold ? h->n_cold : n_hot;
    if (n == 0 || (cold ? h->write_tokens_cold : h->write_tokens) == 0)
        return;
    if constexpr (kKind == kLanes32)
        tab.fill(c);
    const kvr_write_op *ops = section<kvr_write_op>(c, h->off_write) + (cold ? n_hot : 0);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t cols = uint32_t(c.token_bytes / 16);
    const uint32_t col_blocks = (cols + blockDim.x - 1) / blockDim.x;
    const uint32_t row_chunks = c.row_elems * c.esz / 16;
    const uint64_t ring_layer = uint64_t(c.Rp) * c.row_elems * c.esz;
    const uint64_t work = uint64_t(n) * col_blocks;
    for (uint64_t u = blockIdx.x; u < work; u += gridDim.x) {
        const kvr_write_op op = ops[u / col_blocks];
        const uint32_t col = uint32_t(u % col_blocks) * blockDim.x + threadIdx.x;
        if (op.source != 0 || col >= cols)
            continue;
        uint8_t *dst = c.arena + uint64_t(op.block) * c.page_bytes + uint64_t(op.slot) * c.token_bytes + 16ull * col;
        const bool may_ring = op.dev_slot != KVR_NO_SLOT;
        for (uint32_t k = 0; k < op.count; ++k) {
            const uint64_t tok = op.token + k;
            const int4 v = payload16<kKind>(c, tab, op.session, tok, 16ull * col);
            *reinterpret_cast<int4 *>(dst + uint64_t(k) * c.token_bytes) = v;
            if (may_ring && ring_owned_by_writer(c, slots[op.dev_slot], tok)) { // window rows (hot ops)
                const uint32_t l = col / row_chunks, within = col - l * row_chunks;
                uint8_t *ring = c.ring + ring_row(c, op.dev_slot, 0, uint32_t(tok % c.R)) * c.esz;
                *reinterpret_cast<int4 *>(ring + l * ring_layer + 16ull * within) = v;
                if (const uint64_t mirror = ring_mirror(c, uint32_t(tok % c.R)) * c.esz)
                    *reinterpret_cast<int4 *>(ring + mirror + l * ring_layer + 16ull * within) = v;
            }
        }
    }
}

template <int kKind> __global__ void __launch_bounds__(256) k_write_cols(DevCtx c, int cold, int stamp) {
    pdl_wait();
    pdl_trigger();
    TlScope tl_(c, cold ? kTlWriteCold : kTlWriteHot);
    write_cols_body<kKind>(c, cold);
    if (stamp)
        stamp_if_last(c);
}

// nq > 0: the last nq CTAs generate the decode queries instead (KVR_QMERGE: the queries
// ride in the hot K-write's launch, no forked branch and no join before K-attn)
template <uint32_t kPer, int kKind>
__global__ void __launch_bounds__(256) k_write(DevCtx c, int cold, int stamp, uint32_t nq) {
    pdl_wait();
    pdl_trigger();
    TlScope tl_(c, cold ? kTlWriteCold : kTlWriteHot);
    if (nq && blockIdx.x >= gridDim.x - nq)
        query_body(c, blockIdx.x - (gridDim.x - nq), nq);
    else
        write_body<kPer, kKind>(c, cold, blockIdx.x, gridDim.x - nq);
    if (stamp)
        stamp_if_last(c);
}

template <int kKind> __global__ void __launch_bounds__(256) k_presum(DevCtx c, int stamp) {
    pdl_wait();
    pdl_trigger();
    TlScope tl_(c, kTlPresum);
    presum_body<kKind>(c);
    if (stamp)
        stamp_if_last(c);
}

// The step's tail in ONE kernel: the cold prompt rows (column-major) and K-presum's
// chunks (disjoint rows) — one launch gap after K-attn instead of two.
template <int kKind> __global__ void __launch_bounds__(256) k_tail(DevCtx c, int stamp) {
    pdl_wait();
    pdl_trigger();
    TlScope tl_(c, kTlWriteCold); // (cold rows and K-presum: one span)
    write_cols_body<kKind>(c, 1);
    if (c.stash)
        presum_body<kKind>(c);
    if (stamp)
        stamp_if_last(c);
}

// K-far + K-map + K-prime in ONE kernel: K-far and K-prime read the rows the host
// resolved (not the page table K-map edits), so the three are independent.
__global__ void __launch_bounds__(256) k_fmp(DevCtx c) {
    pdl_wait();
    pdl_trigger();
    TlScope tl_(c, kTlFmp);
    __shared__ uint64_t rows[kFarRows];
    far_part(c, rows);
    map_part(c);
    prime_part(c);
}

} // namespace

// Grids of the small pre-attention kernels (x KVR_GRID_SCALE, default 2: apply 4,
// hot K-write 8, queries 4 CTAs per SM). Timeline A/B on C5 (attention start after the
// first kernel): scale 1 52.9 us (the queries branch took 28 us and crowded K-fmp),
// scale 2 45.1 us, the previous grids (queries 8 per SM) 49.3 us.
int grid_scale() {
    static const int k = [] {
        const char *e = getenv("KVR_GRID_SCALE");
        return e ? std::max(1, atoi(e)) : 2;
    }();
    return k;
}

void launch_apply(const DevCtx &c, cudaStream_t s, int sms) { k_apply<<<sms * 2 * grid_scale(), 256, 0, s>>>(c); }

void launch_presum(const DevCtx &c, cudaStream_t s, int sms, int stamp, bool pdl) {
    if (!c.stash)
        return;
    const unsigned g = unsigned(sms) * 4;
    if (c.esz == 4)
        launch_ex(k_presum<kLanes32>, g, 256, 0, s, pdl, c, stamp);
    else if (c.payload_mode == KVR_PAYLOAD_LANES)
        launch_ex(k_presum<kLanes16>, g, 256, 0, s, pdl, c, stamp);
    else
        launch_ex(k_presum<kBytes>, g, 256, 0, s, pdl, c, stamp);
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("KVR_PDL");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

namespace {
// KVR_COLD selects the cold writer (A/B): col (column-major, default) | tok (token-major K-write)
int cold_kind() {
    static const int k = [] {
        const char *e = getenv("KVR_COLD");
        return e && std::string(e) == "tok" ? 0 : 1;
    }();
    return k;
}
// KVR_HOT: tok (token-major K-write, default) | col (column-major)
int hot_kind() {
    static const int k = [] {
        const char *e = getenv("KVR_HOT");
        return e && std::string(e) == "col" ? 1 : 0;
    }();
    return k;
}
} // namespace

// cold: 0 hot writes, 1 cold writes (both over the whole GPU)
void launch_write(const DevCtx &c, cudaStream_t s, int sms, int cold, int stamp, bool pdl, bool with_queries) {
    // hot writes (few decode tokens + window rows): one chunk per thread for
    // spread; cold prompt rows: two chunks per thread for generator ILP
    const int kind = c.esz == 4 ? kLanes32 : c.payload_mode == KVR_PAYLOAD_LANES ? kLanes16 : kBytes;
    const unsigned g = unsigned(sms) * (cold ? 8 : 4 * grid_scale());
    const uint32_t nq = with_queries ? uint32_t(sms) * 2 * grid_scale() : 0u;
    auto go = [&](auto per, auto kk) {
        launch_ex(k_write<decltype(per)::value, decltype(kk)::value>, g + nq, 256, 0, s, pdl, c, cold, stamp, nq);
    };
    using std::integral_constant;
    if (cold ? cold_kind() == 1 : (hot_kind() == 1 && !with_queries)) {
        if (kind == kLanes16)
            launch_ex(k_write_cols<kLanes16>, g, 256, 0, s, pdl, c, cold, stamp);
        else if (kind == kLanes32)
            launch_ex(k_write_cols<kLanes32>, g, 256, 0, s, pdl, c, cold, stamp);
        else
            launch_ex(k_write_cols<kBytes>, g, 256, 0, s, pdl, c, cold, stamp);
        return;
    }
    if (kind == kLanes16)
        cold ? go(integral_constant<uint32_t, 2>{}, integral_constant<int, kLanes16>{})
             : go(integral_constant<uint32_t, 1>{}, integral_constant<int, kLanes16>{});
    else if (kind == kLanes32)
        cold ? go(integral_constant<uint32_t, 2>{}, integral_constant<int, kLanes32>{})
             : go(integral_constant<uint32_t, 1>{}, integral_constant<int, kLanes32>{});
    else
        cold ? go(integral_constant<uint32_t, 2>{}, integral_constant<int, kBytes>{})
             : go(integral_constant<uint32_t, 1>{}, integral_constant<int, kBytes>{});
}

void launch_tail(const DevCtx &c, cudaStream_t s, int sms, int stamp, bool pdl) {
    if (cold_kind() != 1) { // token-major cold K-write, then K-presum
        launch_write(c, s, sms, 1, stamp && !c.stash, pdl);
        launch_presum(c, s, sms, stamp, pdl);
        return;
    }
    const unsigned g = unsigned(sms) * 8;
    if (c.esz == 4)
        launch_ex(k_tail<kLanes32>, g, 256, 0, s, pdl, c, stamp);
    else if (c.payload_mode == KVR_PAYLOAD_LANES)
        launch_ex(k_tail<kLanes16>, g, 256, 0, s, pdl, c, stamp);
    else
        launch_ex(k_tail<kBytes>, g, 256, 0, s, pdl, c, stamp);
}

void launch_query(const DevCtx &c, cudaStream_t s, int sms) { k_query<<<sms * 2 * grid_scale(), 256, 0, s>>>(c); }

__global__ void k_stamp(DevCtx c) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    c.scan->end_ns = t;
}
void launch_stamp(const DevCtx &c, cudaStream_t s) { k_stamp<<<1, 1, 0, s>>>(c); }

void launch_far_map_prime(const DevCtx &c, cudaStream_t s, int sms, bool pdl) {
    launch_ex(k_fmp, unsigned(sms) * 2, 256, 0, s, pdl, c);
}

} // namespace kvr
