// kvrail-b200 device internals shared by the sm_100a kernels.
#pragma once
#include <utility>

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kvr_cuda.h"
#include "kvrail_c.h"

namespace kvr {

constexpr uint32_t kNoMap = 0xffffffffu;
constexpr int kWarp = 32;

/// One staged span in train order, as consumed by K-gather.
struct GSpan {
    uint64_t first_token;  // logical token of slot_begin (near) or summary token (far)
    uint64_t tok_prefix;   // exclusive prefix of slot_count over the gather list
    uint32_t block, slot_begin, slot_count, dev_slot;
    uint32_t kind, pad;
};

/// Scan/step counters kept in device memory.
struct ScanCounters {
    uint32_t trains, descriptors, spans, status;
    uint64_t total_tokens;
    uint64_t train_bytes;
    uint64_t end_ns; // %globaltimer when the step's last kernel ran (inter-token latency)
    uint64_t attn_t0, attn_t1; // K-attn's first CTA start / last warp exit (%globaltimer; reset by K-scan)
    uint64_t gather_t0, gather_t1; // the same for K-gather
};

/// Everything a kernel needs: geometry + device buffers. Passed by value.
struct DevCtx {
    uint64_t page_bytes, token_bytes, max_tokens, seed;
    uint32_t tpp, arena_pages, L, Hkv, hd, Hq, group, d_kv, row_elems, esz;
    uint32_t elem_kind, payload_mode, n_slots, W, R, far_cap, chunk_tokens, max_chunks, smap_cap;
    uint32_t G, Rp; // ring guard rows (rows [0, G) mirrored at [R, R + G)) and plane rows R + G
    uint32_t max_scan, max_trains;
    float lane_scale, lane_bias; // 2-byte lanes: (2^23 + b) * scale - bias = (b - 128) * scale
    __half2 lane_h2_scale, lane_h2_bias; // fp16 lanes: (1024 + b) * 2^-s - 1152 * 2^-s
    uint32_t query_mode;         // KVR_QUERY_*
    uint8_t *arena;   // arena_pages * page_bytes
    uint8_t *ring;    // [slot][L][R][row_elems] elements
    uint32_t *tmap;   // [slot][max_tokens]
    uint32_t *smap;   // [slot][smap_cap]
    uint8_t *far;     // [slot][L][max_chunks][row_elems] elements
    uint8_t *stash;   // [slot][max_chunks][token_bytes]: K-presum chunk means (far view only)
    float *q;         // [slot][L][Hq][hd]: fp32, or the KV element type when q_esz == 2 (load_q)
    uint32_t q_esz;   // 2: exact queries stored as bf16/fp16 (exact: multiples of 1/128); 4: fp32
    float *out;       // [slot][L][Hq][hd]
    const uint8_t *desc; // device copy of the step descriptor
    kvr_train *trains;
    kvr_descriptor *descs;
    GSpan *gspans;
    ScanCounters *scan;
    // K-mass (b200.utility = attention): probe layer, per-row scratch, per-slot runs
    uint32_t utility, util_layer;
    float *mass_sc;          // [slot][Hq][W + far_cap] scores in view order
    float2 *mass_part;       // [slot][Hq][row splits] (max, sum of exp)
    kvr_mass_run *mass_runs; // [slot][W]
    uint32_t *mass_count;    // [slot]
    const uint64_t *fault;   // [0] KVR_FAULT_DROP_SPAN, [1] KVR_FAULT_SHIFT_ROWS arguments — test hooks only
    uint32_t *attn_sched;    // [0] next item to claim, [1] CTAs finished (tensor-core attention),
                             // [2] CTAs finished of the step's last kernel (end stamp)
    unsigned long long *tl;  // diagnostic kernel timeline (KVR_TIMELINE=1), null when off
};

/// Diagnostic timeline (KVR_TIMELINE=1): per kernel of the step, the first CTA's start
/// and the last warp's exit on %globaltimer (min / max over CTAs) — the step graph's
/// real schedule without event nodes. Ids: kvr_dev_timeline in kvr_cuda.h.
enum TlId : uint32_t { kTlApply, kTlQuery, kTlScan, kTlWriteHot, kTlFmp, kTlGather, kTlAttn, kTlWriteCold, kTlPresum,
                      kTlAttnEntry };
__device__ inline unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
/// K-attn's own span on %globaltimer into the step counters (the step graph has no
/// event nodes around it, so the kernel times itself; ncu's gpu__time_duration
/// is the same span: first CTA start to last CTA exit).
/// A (start, end) pair on %globaltimer over a kernel: min over CTA starts, max over CTA
/// exits. Construct at the top of the kernel (every thread, before any exit); the exit
/// stamp is ONE global atomic per CTA, by its last warp to leave (counted in shared
/// memory) — one atomic per warp on one address serialised ~10k atomics per launch.
struct SpanStamp {
    unsigned long long *t;
    unsigned *left;
    __device__ void open(unsigned long long *t_, unsigned *cnt) {
        t = t_, left = cnt;
        if (threadIdx.x == 0) {
            *left = (blockDim.x + 31) / 32;
            atomicMin(t, gtimer());
        }
        __syncthreads();
    }
    __device__ void close() {
        if ((threadIdx.x & 31) == 0 && atomicSub(left, 1u) == 1u)
            atomicMax(t + 1, gtimer());
    }
};
struct AttnSpan : SpanStamp {
    __device__ explicit AttnSpan(const DevCtx &c) {
        __shared__ unsigned cnt;
        open(reinterpret_cast<unsigned long long *>(&c.scan->attn_t0), &cnt);
    }
    __device__ ~AttnSpan() { close(); }
};
struct GatherSpan : SpanStamp {
    __device__ explicit GatherSpan(const DevCtx &c) {
        __shared__ unsigned cnt;
        open(reinterpret_cast<unsigned long long *>(&c.scan->gather_t0), &cnt);
    }
    __device__ ~GatherSpan() { close(); }
};
/// (kTag: each scope live at the same time in one kernel needs its own exit counter)
template <int kTag> struct TlScopeT : SpanStamp {
    __device__ TlScopeT(const DevCtx &c, uint32_t id) {
        __shared__ unsigned cnt;
        t = nullptr;
        if (c.tl) // (uniform)
            open(c.tl + 2 * id, &cnt);
    }
    __device__ ~TlScopeT() {
        if (t)
            close();
    }
};
using TlScope = TlScopeT<0>;

/// Query element i of the query buffer as fp32 (exact either way).
__device__ __forceinline__ float load_q(const DevCtx &c, uint64_t i) {
    if (c.q_esz == 4)
        return c.q[i];
    const uint16_t b = reinterpret_cast<const uint16_t *>(c.q)[i];
    return c.elem_kind == KVR_ELEM_BF16 ? __uint_as_float(uint32_t(b) << 16) : __half2float(__ushort_as_half(b));
}

/// Token `tok` of a slot is written into the ring by K-write / K-prime only when it
/// lies in the live window after this step and K-gather does not deliver it (near
/// staged range [stage_lo, stage_hi) of the slot this step).
__device__ inline bool ring_owned_by_writer(const DevCtx &c, const kvr_slot_state &st, uint64_t tok) {
    return tok < st.written && tok + c.W >= st.written && !(tok >= st.stage_lo && tok < st.stage_hi);
}

__host__ __device__ inline const kvr_step_header *hdr(const DevCtx &c) {
    return reinterpret_cast<const kvr_step_header *>(c.desc);
}
template <typename T> __device__ inline const T *section(const DevCtx &c, uint64_t off) {
    return reinterpret_cast<const T *>(c.desc + off);
}

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/// Reference payload lane value ((h % 2001) - 1000) / 1000 (scenario.cpp:200).
__device__ inline float lane_value(uint64_t h) {
    return float(int64_t(h % 2001ull) - 1000) / 1000.0f;
}

/// Arena byte offset of a global slot index (block * tpp + slot).
__device__ inline uint64_t gslot_offset(const DevCtx &c, uint32_t gs) {
    return uint64_t(gs / c.tpp) * c.page_bytes + uint64_t(gs % c.tpp) * c.token_bytes;
}

/// Ring element offset of (slot, layer, row). A plane holds R rows plus G guard
/// rows that mirror rows [0, G): a tile of up to G rows starting at any row < R
/// reads consecutive memory (no split at the ring end).
__device__ inline uint64_t ring_row(const DevCtx &c, uint32_t slot, uint32_t l, uint32_t row) {
    return ((uint64_t(slot) * c.L + l) * c.Rp + row) * c.row_elems;
}
/// Element offset from a row to its guard mirror (0: the row has none).
__device__ inline uint64_t ring_mirror(const DevCtx &c, uint32_t row) {
    return row < c.G ? uint64_t(c.R) * c.row_elems : 0;
}

/// Last index i in [0, n) with key(i) <= v for a non-decreasing key with key(0) <= v,
/// found by the whole warp in <= 3 rounds of 32 parallel probes (n <= 32768) instead
/// of ~log2(n) dependent loads: the per-CTA start-up search of K-write and K-gather.
/// Every lane of the warp must call it; all get the same result.
template <class Key> __device__ inline uint32_t warp_last_le(uint32_t n, uint64_t v, Key key) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t idx = lo + lane * step;
        const bool p = lane == 0 || (idx < hi && key(idx) <= v);
        const uint32_t top = 31 - __clz(__ballot_sync(0xffffffffu, p));
        lo += top * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// ---- programmatic dependent launch (PDL) ----------------------------------
// A kernel launched with a PDL edge may start while its predecessor still runs (once
// every predecessor CTA has executed pdl_trigger or exited). Every kernel that can
// be such a dependent calls pdl_wait() FIRST — before any early exit, so that its own
// completion still implies its predecessors' (transitive ordering) — and pdl_trigger()
// right after, letting its own dependents launch. Both are no-ops without a PDL edge.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled(); // KVR_PDL=0 turns the step graph's PDL edges off (A/B)
/// <<<grid, block, smem, s>>> with the PDL attribute when `pdl`
template <typename... P, typename... A>
inline void launch_ex(void (*k)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, bool pdl,
                      A &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// ---- host launchers (one per kernel file) --------------------------------
// pdl: the launch's stream predecessor is a kernel of the same step (PDL edge)
void launch_apply(const DevCtx &c, cudaStream_t s, int sms);   // zero, cow, blob
/// stamp: this launch is the step's last kernel and writes the step-end timestamp
/// with_queries: the decode queries are generated by extra CTAs of this (hot) launch
void launch_write(const DevCtx &c, cudaStream_t s, int sms, int cold, int stamp = 0, bool pdl = false,
                  bool with_queries = false); // generated payloads
void launch_query(const DevCtx &c, cudaStream_t s, int sms);   // decode queries
void launch_far_map_prime(const DevCtx &c, cudaStream_t s, int sms, bool pdl = false); // K-far + K-map + K-prime
void launch_stamp(const DevCtx &c, cudaStream_t s); // step-end timestamp
/// the step's tail after K-attn: cold prompt rows + K-presum (stamp: writes the end stamp)
void launch_tail(const DevCtx &c, cudaStream_t s, int sms, int stamp, bool pdl);
void launch_presum(const DevCtx &c, cudaStream_t s, int sms, int stamp = 0, bool pdl = false); // prompt rows + their far chunk means
void launch_mass(const DevCtx &c, cudaStream_t s);             // attention-utility observations
bool prepare_mass(const DevCtx &c); // false: no K-mass for this geometry
size_t mass_scratch_floats(const DevCtx &c);
size_t mass_part_entries(const DevCtx &c);
uint32_t mass_max_group();
void launch_scan(const DevCtx &c, cudaStream_t s, bool pdl = false);             // stage + reduce
void launch_gather(const DevCtx &c, cudaStream_t s, int sms, bool pdl = false);  // trains -> window
/// destination bytes of staged tokens [tok_begin, +count) into out (token-major)
void launch_read_staged(const DevCtx &c, cudaStream_t s, uint64_t tok_begin, uint64_t count, uint8_t *out,
                        uint8_t *in_window);
struct AttnPlan;
/// mode: 1 auto (tensor cores for GQA groups where supported), 2 CUDA-core
/// kernel, 3 tensor-core kernel (null if unsupported). Builds the TMA descriptor.
AttnPlan *make_attn_plan(const DevCtx &c, int sms, int device, int mode);
// tensor-core variant (kvr_attn_tc.cu)
bool attn_tc_supported(const DevCtx &c);
bool attn_tc_ready(const DevCtx &c); // supported and the ring has its guard rows (c.G)
const void *attn_tc_kernel(const DevCtx &c);
/// TMA descriptors of the tensor-core kernel: ring in 32-row boxes, ring in whole
/// 128-row K|V tiles (one op per tile), far rows for gather4.
struct TcMaps {
    CUtensorMap ring, tile, far;
};
// (tile: one K or V half of a 128-row tile per op — the two halves have separate rings)
bool attn_tc_maps(const DevCtx &c, TcMaps *maps);
void launch_attn_tc(const void *fn, const DevCtx &c, const TcMaps &maps, uint32_t grid, cudaStream_t s,
                    bool pdl = false);
void launch_attn(const AttnPlan *p, const DevCtx &c, cudaStream_t s, bool pdl = false);
void free_attn_plan(AttnPlan *p);
const char *attn_variant(const AttnPlan *p);

} // namespace kvr
