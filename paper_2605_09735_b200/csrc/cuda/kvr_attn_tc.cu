// kvrail-b200 K-attn, tensor-core variant for GQA groups (g >= 2, head_dim 128,
// fp16/bf16): the same fixed-shape window attention as kvr_attn.cu (attend() of
// far_view.cpp:113-155 per (layer, q-head), q-head j -> kv-head j / g), with both
// contractions on the 5th-generation tensor cores.
//
// Work item = (slot, layer, kv head); persistent grid, one CTA per SM, 384 threads.
//   warp 0  K producer, warp 2 V producer: each streams its half of the 128-row
//           tiles through its own ring (3 x 32 KiB stages) — an interior tile half
//           is ONE 5-D TMA op, window-edge / ring-wrap tiles go as 32-row 4-D
//           boxes (only boxes with a live row), far summary rows by TMA gather4
//           folded in front of the tail tile; 128-byte swizzle throughout;
//   warp 1  TMEM owner + S issuer (one elected lane issues):
//             S^T[128 rows x 16]  = K_tile[128 x 128] . Qs^T      (K-major A)
//   warp 3  PV issuer (one elected lane issues):
//             O^T[128 dims x 16] += V_tile^T[128 x 128] . Ps      (MN-major A)
//           tcgen05.mma kind::f16, fp32 accumulators in TMEM (S and O double
//           buffered per warpgroup, 128 columns), completion by tcgen05.commit ->
//           mbarrier; both issuers walk the tile stream strictly in order and await
//           each condition with the suspending try_wait (polling all barriers at
//           once took issue slots from the softmax warps of the same SM
//           sub-partition: C5 0.4478 -> 0.4467 -> 0.4409 ms, S then PV);
//   warps 4-7, 8-11  two softmax/correction warpgroups, items alternating between
//           them: thread t owns TMEM lane t, i.e. token row t of S and head dim t
//           of O. Online softmax in base 2 per q-head column with a held maximum:
//           O accumulates in TMEM across the item's tiles and is read back only when
//           a tile raises the maximum by more than 2^8 (one barrier OR-vote per tile
//           decides; only then are the tile maxima exchanged), P written back as
//           bf16/fp16 for the PV MMA; the next item's Q is fetched ahead.
// Precision: the MMA operands are 16-bit, so q and p are split into 16-bit terms
// (x = x_0 + x_1 [+ x_2], each the rounding of the remainder) in column blocks
// [s*g, (s+1)*g) of the operand, and S / O are the sums of the column blocks. fp16
// (11-bit significands) uses 2 terms: 22 bits. bf16 (8 bits) uses 3 terms for q
// (24 bits: a 2-term q left ~2^-17 relative error in every logit, which broke 1e-3
// with random fp32 queries over large-magnitude KV — measured 1.7e-3) and 3 terms
// for p when 3g <= 16 (else 2: 16 bits, ~1e-4 of output error). With g = 8 the q
// operand needs 24 columns: the S MMA then runs at N = 32 (its 4th column block
// reads the next buffer — finite garbage in S columns nobody reads).
#include <cstdio>
#include <type_traits>
#include <cudaTypedefs.h>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

constexpr int kRows = 128;                 // tokens per tile (S: M, PV: K)
constexpr int kHd = 128;                   // head dim (S: K, PV: M)
constexpr int kN = 16;                     // PV MMA N (and S MMA N unless q needs 24 columns)
constexpr int kSub = 32;                   // rows per TMA box
constexpr uint32_t kHalfBytes = kRows * 128; // one 64-dim half of a K or V tile (16 KiB)
constexpr uint32_t kSideBytes = 2 * kHalfBytes; // a K (or V) tile: two 64-dim halves, 32 KiB
#ifndef KVR_TC_KSTAGES
#define KVR_TC_KSTAGES 3
#endif
#ifndef KVR_TC_VSTAGES
#define KVR_TC_VSTAGES 3
#endif
// K tiles are released as soon as their S MMA completes, V tiles after the
// softmax and the PV MMA (measured: 3 + 3 beats 2 + 4 on C3 and C5)
constexpr int kKStages = KVR_TC_KSTAGES, kVStages = KVR_TC_VSTAGES;
static_assert(kVStages <= 4, "V stage index and phase are packed in 3 bits");
static_assert(kKStages <= kVStages, "a K ring deeper than the V ring stalls the PV order (4 + 2 hung on B200)");
constexpr uint32_t kOpBytes = kN * kHd * 2; // one P operand buffer (4 KiB): 2 column blocks of 8
constexpr uint32_t kQBytes = 3 * 2048;       // the Q operand: up to 3 column blocks of 8 (24 columns)

/// Split terms and MMA widths of a (T, g) variant.
template <typename T, int G> struct Splits {
    static constexpr bool kBf = std::is_same_v<T, __nv_bfloat16>;
#ifndef KVR_TC_QS3
#define KVR_TC_QS3 1
#endif
    static constexpr int QS = kBf && KVR_TC_QS3 ? 3 : 2;       // q terms
    static constexpr int PS = kBf && 3 * G <= kN ? 3 : 2;     // p terms
    static constexpr int NQ = QS * G <= 16 ? 16 : 32;         // S MMA N
    static_assert(QS * G <= 24 && PS * G <= kN, "split columns must fit the operand buffers");
};
#ifndef KVR_TC_TILE5D
#define KVR_TC_TILE5D 1
#endif
constexpr bool kUseTile5d = KVR_TC_TILE5D != 0;
#ifndef KVR_TC_SWAIT
#define KVR_TC_SWAIT 1
#endif
#ifndef KVR_TC_PVWAIT
#define KVR_TC_PVWAIT 1
#endif
// lazy O rescaling (needs the in-order PV issuer): rescale only when a tile's maximum
// exceeds the held one by more than kLazy (log2 units: p <= 256)
#ifndef KVR_TC_LAZY
#define KVR_TC_LAZY 1
#endif
#if KVR_TC_LAZY && !KVR_TC_PVWAIT
#error "KVR_TC_LAZY needs KVR_TC_PVWAIT"
#endif
#ifndef KVR_TC_LAZY_T
#define KVR_TC_LAZY_T 8
#endif
constexpr float kLazy = KVR_TC_LAZY_T; // (0: flip on every raise — a test build exercising the flips)
// lazy mode: a barrier OR-vote per tile replaces the tile-max exchange unless a row raises
#ifndef KVR_TC_VOTE
#define KVR_TC_VOTE 1
#endif
constexpr int kThreads = 384; // warp 0 K TMA, 1 S MMA, 2 V TMA, 3 PV MMA, warps 4-7 / 8-11 softmax

__device__ inline uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ inline void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ inline void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ inline void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifdef KVR_HANG_CHECK
__device__ inline void mbar_wait(uint64_t *bar, uint32_t parity) {
    for (uint64_t i = 0;; ++i) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
        if (ok)
            return;
        if (i == (1ull << 22) && blockIdx.x == 40 && (threadIdx.x & 31) == __ffs(__activemask()) - 1)
            printf("hang: block %d thread %d bar smem+%u parity %u\n", blockIdx.x, threadIdx.x, smem_u32(bar),
                   parity);
        if (i == (1ull << 25))
            asm volatile("trap;");
    }
}
#else
__device__ inline void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "W_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}
#endif
__device__ inline void tma_load_4d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                   uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
                 : "memory");
}
__device__ inline void tma_load_5d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                   uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
                 : "memory");
}
__device__ inline void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ inline void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ inline void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

/// Shared-memory matrix descriptor (sm_100 UMMA): start, leading/stride byte
/// offsets (16-byte units), version 1, layout (0 none, 2 = 128-byte swizzle).
__device__ inline uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((addr >> 4) & 0x3fff) | uint64_t((lbo >> 4) & 0x3fff) << 16 |
           uint64_t((sbo >> 4) & 0x3fff) << 32 | 1ull << 46 | uint64_t(layout) << 61;
}
/// Instruction descriptor, kind::f16: fp32 accumulate, A/B 16-bit (0 f16, 1 bf16).
__host__ __device__ constexpr uint32_t idesc(uint32_t fmt, uint32_t a_mn, uint32_t b_mn, uint32_t m,
                                             uint32_t n) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (a_mn << 15) | (b_mn << 16) | ((n >> 3) << 17) |
           ((m >> 4) << 24);
}
__device__ inline void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                 "l"(a), "l"(b), "r"(id), "r"(acc)
                 : "memory");
}
__device__ inline void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ inline void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                   "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i)
        v[i] = __uint_as_float(r[i]);
}

template <typename T> struct Pack2;
template <> struct Pack2<__nv_bfloat16> {
    static __device__ uint32_t round(float a, float b, float2 &back) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        back = __bfloat1622float2(h);
        return *reinterpret_cast<const uint32_t *>(&h);
    }
};
template <> struct Pack2<__half> {
    static __device__ uint32_t round(float a, float b, float2 &back) {
        const __half2 h = __floats2half2_rn(a, b);
        back = __half22float2(h);
        return *reinterpret_cast<const uint32_t *>(&h);
    }
};

/// Row k of an MMA operand held MN-major, unswizzled (8x8 core matrices of 8 K-rows
/// x 16 B; K-adjacent cores 128 B apart, blocks of 8 N-columns 2048 B apart): the
/// thread owning k writes x split into S terms, term s in columns [s*G, (s+1)*G)
/// (each term the element-type rounding of what the previous terms left), one
/// 16-byte store per 8 columns. Columns >= S*G of the last written block stay zero.
template <typename T, int G, int S> __device__ inline void store_split(uint8_t *op, uint32_t k, const float (&x)[G]) {
    constexpr int NC = S * G, NB = (NC + 7) / 8; // used columns, 8-column blocks written
    uint32_t wd[4 * NB];
#pragma unroll
    for (int i = 0; i < 4 * NB; ++i)
        wd[i] = 0;
    float r[G];
#pragma unroll
    for (int g = 0; g < G; ++g)
        r[g] = x[g];
#pragma unroll
    for (int s = 0; s < S; ++s) {
#pragma unroll
        for (int g = 0; g < G; ++g) { // column s*G + g: the rounding of the remainder (exact subtraction)
            float2 back;
            const uint32_t bits = Pack2<T>::round(r[g], 0.f, back) & 0xffffu;
            r[g] -= back.x;
            const int col = s * G + g;
            wd[col / 2] |= bits << (16 * (col & 1));
        }
    }
    uint8_t *row = op + (k >> 3) * 128u + (k & 7u) * 16u;
#pragma unroll
    for (int bl = 0; bl < NB; ++bl)
        *reinterpret_cast<uint4 *>(row + 2048 * bl) =
            make_uint4(wd[4 * bl], wd[4 * bl + 1], wd[4 * bl + 2], wd[4 * bl + 3]);
}

/// Tiles of one work item, identical for every role. The near window [lo, w) is
/// cut into 128-row tiles starting exactly at lo (ring row lo mod R: the plane's
/// 128 guard rows mirror rows [0, 128), so a tile starting anywhere below R is one
/// contiguous 128-row read — no dead rows at the window's old edge); the 1-127
/// newest rows form a tail tile of 32-row boxes, and far summary rows are folded
/// into that tail tile when they fit in front of its boxes.
struct Item {
    uint32_t slot, layer, head, far_count, far_begin;
    uint32_t n_far;      // far-only tiles (far rows not folded)
    uint32_t tail_boxes; // boxes of the tail tile (0 = no tail tile)
    uint32_t fold_pos;   // first smem row of the tail boxes (far rows folded in front)
    uint32_t n_tiles;
    uint64_t lo, w, L0;
};
struct Tile {
    uint32_t far_rows, far_off; // far list rows [far_off, +far_rows) -> smem rows [0, far_rows)
    uint32_t box_first, n_boxes; // near boxes at smem rows [32 box_first, 32 (box_first + n_boxes))
    uint32_t nk;                 // PV K steps (16 rows each) covering every used row
    uint64_t tok_r0;             // token of smem row 0 for the near rows (mod 2^64)
};
__device__ inline bool item_fill(const DevCtx &c, const kvr_slot_state *slots, Item &I);
__device__ inline bool item_of(const DevCtx &c, const kvr_slot_state *slots, uint32_t it, Item &I) {
    I.head = it % c.Hkv;
    I.layer = (it / c.Hkv) % c.L;
    I.slot = it / (c.Hkv * c.L);
    return item_fill(c, slots, I);
}
/// Item fields from (slot, layer, head); false if the slot is not live.
__device__ inline bool item_fill(const DevCtx &c, const kvr_slot_state *slots, Item &I) {
    const kvr_slot_state st = slots[I.slot];
    if (!st.live)
        return false;
    I.w = st.written;
    I.lo = I.w > c.W ? I.w - c.W : 0;
    I.L0 = I.lo; // tiles start at the window's first row (guard rows: no alignment needed)
    const uint32_t near = uint32_t(I.w - I.lo);
    const uint32_t n_full = near / kRows;
    I.tail_boxes = (near % kRows + kSub - 1) / kSub;
    I.far_count = st.far_count;
    I.far_begin = st.far_begin;
    const uint32_t P = (I.far_count + kSub - 1) & ~uint32_t(kSub - 1);
    const bool fold = I.far_count > 0 && I.tail_boxes > 0 && P + kSub * I.tail_boxes <= uint32_t(kRows);
    I.fold_pos = fold ? P : 0;
    I.n_far = I.far_count > 0 && !fold ? (I.far_count + kRows - 1) / kRows : 0;
    I.n_tiles = I.n_far + (I.tail_boxes > 0) + n_full;
    return true;
}
__device__ inline Tile tile_of(const Item &I, uint32_t k) {
    Tile tl;
    if (k < I.n_far) {
        tl.far_off = k * kRows;
        tl.far_rows = min(uint32_t(kRows), I.far_count - tl.far_off);
        tl.box_first = tl.n_boxes = 0;
        tl.nk = (tl.far_rows + 15) / 16;
        tl.tok_r0 = 0;
        return tl;
    }
    k -= I.n_far;
    const uint32_t n_full = I.n_tiles - I.n_far - (I.tail_boxes ? 1u : 0u);
    if (k < n_full) { // full tiles from L0
        tl.far_rows = tl.far_off = 0;
        tl.box_first = 0;
        tl.n_boxes = kRows / kSub;
        tl.nk = kRows / 16;
        tl.tok_r0 = I.L0 + uint64_t(kRows) * k;
        return tl;
    }
    // tail tile: the last 1-3 boxes, with the far rows folded in front of them
    tl.far_off = 0;
    tl.far_rows = I.fold_pos ? I.far_count : 0;
    tl.box_first = I.fold_pos / kSub;
    tl.n_boxes = I.tail_boxes;
    tl.nk = (I.fold_pos + kSub * I.tail_boxes) / 16;
    tl.tok_r0 = I.L0 + uint64_t(kRows) * n_full - I.fold_pos;
    return tl;
}

__device__ inline bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
    return ok != 0;
}
/// Four rows (arbitrary indices) x 64 columns of a 2-D tensor (sm_100 TMA gather4).
__device__ inline void tma_gather4(uint32_t dst, const CUtensorMap *map, int col, int r0, int r1, int r2, int r3,
                                   uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                 "r"(smem_u32(bar))
                 : "memory");
}

__device__ inline bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\t"
                 "elect.sync _|P, 0xffffffff;\n\t"
                 "selp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(pred));
    return pred != 0;
}

/// Dynamic item schedule. CTAs claim active items (live, >= 1 tile) from a global
/// counter (c.attn_sched[0]) instead of a static round robin: measured with the
/// static split, C3's SMs were busy between 2.14 M and 2.59 M cycles (mean 2.33 M)
/// of one launch — the slowest CTA set the kernel time. Warp 0's lane 0 claims items
/// a few ahead of its own tile stream and publishes them in a shared-memory queue;
/// every role reads the CTA's j-th item from it (item j -> softmax warpgroup j % 2).
constexpr uint32_t kQ = 64;     // queue entries (roles lag the claimer by < ~10 items)
#ifndef KVR_TC_AHEADQ
#define KVR_TC_AHEADQ 2
#endif
// items claimed ahead of the claimer's own position: fewer keeps the end of a launch
// balanced (A/B, K-attn ms: 8 -> C5 0.4348 / C3 1.2415, 4 -> 0.4306 / 1.2344, 2 -> 0.4286 /
// 1.2307)
constexpr uint32_t kAheadQ = KVR_TC_AHEADQ;
#ifndef KVR_TC_FIRST_CLAIM
#define KVR_TC_FIRST_CLAIM 1
#endif
struct ItemQueue {
    uint32_t item[kQ];
    uint32_t tail; // items published
    uint32_t end;  // index of the end of the CTA's stream (~0: not reached)
};
__device__ inline uint32_t ld_vol(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ inline void st_vol(uint32_t *p, uint32_t v) {
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
/// Claimer (one thread): publish items until `want` are available or the stream ends.
/// Items are claimed kClaim at a time (one atomic round trip, their slot states loaded
/// together) — the claimer is warp 0's lane 0, whose K tile loads wait on it.
#ifndef KVR_TC_CLAIM
#define KVR_TC_CLAIM 1
#endif
constexpr uint32_t kClaim = KVR_TC_CLAIM;
__device__ inline void claim_to(ItemQueue *q, uint32_t want, const DevCtx &c, const kvr_slot_state *slots,
                                uint32_t n_items) {
    uint32_t tail = q->tail;
    while (tail < want && q->end == ~0u) {
        const uint32_t base = atomicAdd(c.attn_sched, kClaim);
        if (base >= n_items) {
            __threadfence_block();
            st_vol(&q->end, tail);
            break;
        }
        bool active[kClaim];
#pragma unroll
        for (uint32_t i = 0; i < kClaim; ++i) {
            Item I;
            active[i] = base + i < n_items && item_of(c, slots, base + i, I) && I.n_tiles;
        }
#pragma unroll
        for (uint32_t i = 0; i < kClaim; ++i)
            if (active[i])
                q->item[(tail++) % kQ] = base + i;
        __threadfence_block();
        st_vol(&q->tail, tail);
    }
}
/// The j-th item of the CTA's stream: 1 (in `it`), 0 at the stream's end, -1 not
/// published yet (only when `wait` is false).
__device__ inline int queue_get(ItemQueue *q, uint32_t j, uint32_t &it, bool wait = true) {
    for (;;) {
        if (j < ld_vol(&q->tail)) {
            __threadfence_block();
            it = ld_vol(&q->item[j % kQ]);
            return 1;
        }
        const uint32_t e = ld_vol(&q->end);
        if (e != ~0u && j >= e)
            return 0;
        if (!wait)
            return -1;
    }
}

/// Items j = w, w + 2, ... of the CTA's stream (warpgroup w's items). The claimer
/// (warp 0) tops the queue up to kAheadQ items past every item it reads.
struct Cursor {
    uint32_t j;
    ItemQueue *q;
    bool claimer;
    __device__ void init(ItemQueue *queue, uint32_t w, bool is_claimer) {
        q = queue, j = w, claimer = is_claimer;
    }
    __device__ bool next(const DevCtx &c, const kvr_slot_state *slots, uint32_t n_items, uint32_t, Item &I) {
        if (claimer) {
            if ((threadIdx.x & 31) == 0)
                claim_to(q, j + kAheadQ, c, slots, n_items);
            __syncwarp();
        }
        uint32_t it;
        if (queue_get(q, j, it) <= 0)
            return false;
        j += 2;
        item_of(c, slots, it, I);
        return true;
    }
};

/// Tile stream of the producer and the MMA issuer. Items alternate between the
/// two warpgroups; an item's tiles are consecutive and the warpgroups overlap at
/// item boundaries (alternating tiles between the warpgroups measured slower:
/// C3 1.485 vs 1.431-1.441 ms, C5 0.521 vs 0.500).
struct Stream { // items j = 0, 1, 2, ... in order (item j -> warpgroup j % 2), all tiles of each
    ItemQueue *q;
    bool claimer, have;
    uint32_t j, k;
    Item cur;
    __device__ void init(const DevCtx &, const kvr_slot_state *, uint32_t, ItemQueue *queue, bool is_claimer = false) {
        q = queue, claimer = is_claimer, have = false, j = k = 0;
    }
    /// Warpgroup, tile index and item of the next tile: 1; 0 at the end; -1 when the
    /// next item is not published yet and `wait` is false (the PV issuer must never
    /// block on the queue: its look-ahead can outrun the claimer).
    __device__ int next(const DevCtx &c, const kvr_slot_state *slots, uint32_t n_items, uint32_t &w, uint32_t &kk,
                        Item &I, bool wait = true) {
        if (!have) {
            if (claimer) {
                if ((threadIdx.x & 31) == 0)
                    claim_to(q, j + kAheadQ + 1, c, slots, n_items);
                __syncwarp();
            }
            uint32_t it;
            const int r = queue_get(q, j, it, wait);
            if (r <= 0)
                return r;
            item_of(c, slots, it, cur);
            have = true;
            k = 0;
        }
        w = j & 1u, kk = k, I = cur;
        if (++k == cur.n_tiles)
            have = false, ++j;
        return 1;
    }
};

/// Per-softmax-warpgroup barriers and operand buffers.
struct WgBars {
    uint64_t qfull, sfull[2], sempty[2], pfull[2], ofull[2], oempty[2];
    uint64_t pempty[2]; // lazy mode: the PV that read P buffer b completed (tcgen05.commit)
    uint32_t pflag[2];  // lazy mode: 1 = this P's PV starts the other O buffer (flip)
};
constexpr uint32_t kWgBytes = kQBytes + 2 * kOpBytes; // Q + P[2]

template <typename T, int G>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_tc(DevCtx c, const __grid_constant__ TcMaps maps) {
    using SP = Splits<T, G>;
    TlScopeT<1> tl_entry_(c, kTlAttnEntry); // (diagnostic: CTA entry, before the prologue)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *kbuf = smem;                                    // kKStages x 32 KiB
    uint8_t *vbuf = kbuf + kKStages * kSideBytes;            // kVStages x 32 KiB
    uint8_t *wgbuf = vbuf + kVStages * kSideBytes;           // 2 x (Q | P0 | P1)
    float *red = reinterpret_cast<float *>(wgbuf + 2 * kWgBytes); // [wg][2][4][8] tile maxima
    float *lred = red + 2 * 2 * 4 * 8;                       // [wg][4][8] row sums
    // K and V halves of a stage have their own rings: K is released as soon as
    // its S MMA completes, V after the PV MMA (which waits on the softmax)
    uint64_t *kfull = reinterpret_cast<uint64_t *>(lred + 2 * 4 * 8);
    uint64_t *kempty = kfull + kKStages, *vfull = kempty + kKStages, *vempty = vfull + kVStages;
    WgBars *wb = reinterpret_cast<WgBars *>(vempty + kVStages);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wb + 2);
    ItemQueue *queue = reinterpret_cast<ItemQueue *>(tmem_slot + 4);

    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t *far_ids = section<uint32_t>(c, h->off_far_ids);
    const uint32_t n_items = c.n_slots * c.L * c.Hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // zero stages and operand buffers: rows a tile does not load must hold
    // finite values (p = 0 times V), unused hi/lo columns must be 0
    for (uint32_t i = threadIdx.x; i < ((kKStages + kVStages) * kSideBytes + 2 * kWgBytes) / 16; i += kThreads)
        reinterpret_cast<int4 *>(smem)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kKStages; ++s) {
            mbar_init(&kfull[s], 1);
            mbar_init(&kempty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(&vfull[s], 1);
            mbar_init(&vempty[s], 1);
        }
        for (int w = 0; w < 2; ++w) {
            mbar_init(&wb[w].qfull, 4);
            for (int b = 0; b < 2; ++b) {
                mbar_init(&wb[w].sfull[b], 1);
                mbar_init(&wb[w].sempty[b], 4);
                mbar_init(&wb[w].pfull[b], 4);
                mbar_init(&wb[w].ofull[b], 1);
                mbar_init(&wb[w].oempty[b], 4);
                mbar_init(&wb[w].pempty[b], 1);
            }
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        queue->tail = 0;
        queue->end = ~0u;
        // the first item only: each claim is an atomic round trip plus a slot-state load,
        // serial — claiming kAheadQ here held every CTA's start ~2 us per item after
        // K-gather (timeline); warp 0 tops the queue up as its tile stream advances
        claim_to(queue, KVR_TC_FIRST_CLAIM, c, slots, n_items);
    }
    fence_async_smem();
    if (warp == 1) {
        // per warpgroup 128 columns: S[b] at 32 b (N <= 32), O[b] at 64 + 16 b
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // PDL: everything above touches only shared memory, TMEM, the descriptor and the
    // claim counter (reset by the previous launch), so it overlaps the predecessor's
    // tail; the roles below read what K-gather and the queries wrote
    pdl_wait(); // (no early trigger: the tail's CTAs, resident beside a CUDA-core K-attn CTA
                // and waiting, cost it ~0.6 % on C2; they launch as K-attn's CTAs exit)
    AttnSpan span_(c);
    TlScope tl_(c, kTlAttn);

    if (warp == 0 || warp == 2) { // ---------------- producers: warp 0 streams K, warp 2 streams V ----------------
        const uint32_t kv = warp == 2 ? 1u : 0u;
        uint64_t *full = kv ? vfull : kfull, *empty = kv ? vempty : kempty;
        const uint32_t n_stages = kv ? kVStages : kKStages;
        uint8_t *ring = kv ? vbuf : kbuf;
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.ring)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.tile)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.far)) : "memory");
        }
        const int kvh0 = int(kv * c.Hkv); // first head index of this half in the ring row
        Stream S;
        S.init(c, slots, n_items, queue, warp == 0);
        uint32_t s = 0, ph = 0, w, k, row_base = 0;
        Item I;
        while (S.next(c, slots, n_items, w, k, I)) {
            const int plane = int(I.slot * c.L + I.layer);
            if (k == 0)
                row_base = uint32_t(I.L0 % c.R); // ring row of the item's first box
            const Tile tl = tile_of(I, k);
            mbar_wait(&empty[s], ph ^ 1);
            const uint32_t st = smem_u32(ring + s * kSideBytes);
            // near boxes holding a live row: boxes start at or after lo, so a box is
            // live iff it starts below w
            const uint64_t first_tok = tl.tok_r0 + uint64_t(kSub) * tl.box_first;
            const uint32_t n_live =
                first_tok < I.w ? min(tl.n_boxes, uint32_t((I.w - first_tok + kSub - 1) / kSub)) : 0u;
            const uint32_t live_boxes = ((1u << n_live) - 1u) << tl.box_first;
            const uint32_t n4 = (tl.far_rows + 3) / 4;
            if (lane == 0)
                mbar_expect_tx(&full[s], n4 * 2 * 512 + __popc(live_boxes) * 2 * kSub * 128);
            __syncwarp();
            if (tl.far_rows) { // far summary rows: TMA gather4, 4 rows x 64 columns; op o = 2 * group + half
                const int base = plane * int(c.max_chunks);
                const uint32_t *ids = far_ids + I.far_begin + tl.far_off;
                for (uint32_t o = lane; o < 2 * n4; o += 32) {
                    const uint32_t g4 = o >> 1, hf = o & 1u;
                    int r[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x)
                        r[x] = base + int(ids[min(4 * g4 + x, tl.far_rows - 1)]);
                    tma_gather4(st + hf * kHalfBytes + g4 * 512, &maps.far, int((kvh0 + I.head) * kHd + hf * 64),
                                r[0], r[1], r[2], r[3], &full[s]);
                }
            }
            uint32_t row0 = 0; // ring row of the first box (< R); its tile may run into the guard rows
            if (tl.n_boxes) {
                row0 = row_base + uint32_t(first_tok - I.L0);
                if (row0 >= c.R)
                    row0 -= c.R;
            }
            if (kUseTile5d && live_boxes == 0xfu) {
                // this half of the whole tile in one op: 5-D view (64 dims, flat plane rows, half, head, K|V)
                if (lane == 0)
                    tma_load_5d(st, &maps.tile, 0, int(plane * c.Rp + row0), 0, int(I.head), int(kv), &full[s]);
            } else if (lane < 8) { // lane = box * 2 + half; boxes end within the guard rows
                const uint32_t bx = lane >> 1, hf = lane & 1u;
                if (live_boxes >> bx & 1u) {
                    const uint32_t row = row0 + (bx - tl.box_first) * kSub;
                    tma_load_4d(st + hf * kHalfBytes + bx * kSub * 128, &maps.ring, int(hf * 64), kvh0 + int(I.head),
                                int(row), plane, &full[s]);
                }
            }
            if (++s == n_stages) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1) { // ---------------- S issuer (whole warp, one elected lane issues) ----------------
        // S^T = K . Q^T for every tile of the stream, in stream order, as soon as its K
        // tile, the warpgroup's S buffer and (first tile of an item) its Q are ready.
        // The PVs are issued by warp 3: two issuing warps halve the per-tile event-loop
        // latency that bounded the kernel with one.
        constexpr uint32_t fmt = std::is_same_v<T, __nv_bfloat16> ? 1u : 0u;
        constexpr uint32_t id_s = idesc(fmt, 0, 1, kRows, SP::NQ); // S^T = K . Q^T (Q MN-major)
        Stream S;
        S.init(c, slots, n_items, queue, warp == 0);
        uint32_t s = 0, ph = 0, w = 0, k = 0;
        uint32_t nw0 = 0, nw1 = 0, mw0 = 0, mw1 = 0;
        const uint32_t kbase = smem_u32(kbuf), wg0 = smem_u32(wgbuf);
        Item I;
        bool have = S.next(c, slots, n_items, w, k, I);
        while (have) {
            const uint32_t nwc = w ? nw1 : nw0, b = nwc & 1u;
#if KVR_TC_SWAIT
            // tiles issue strictly in stream order, so the three conditions are awaited one
            // after the other with the suspending try_wait: a polling loop here took issue
            // slots from the softmax warps sharing this SM sub-partition (warps 5 and 9)
            if (k == 0)
                mbar_wait(&wb[w].qfull, (w ? mw1 : mw0) & 1u);
            mbar_wait(&kfull[s], ph);
            mbar_wait(&wb[w].sempty[b], ((nwc >> 1) & 1u) ^ 1u);
#else
            // the three barriers tested at once, one shuffle
            const bool q = k > 0 || mbar_test(&wb[w].qfull, (w ? mw1 : mw0) & 1u);
            const bool kf = mbar_test(&kfull[s], ph);
            const bool se = mbar_test(&wb[w].sempty[b], ((nwc >> 1) & 1u) ^ 1u);
            if (!__shfl_sync(0xffffffffu, uint32_t(q && kf && se), 0))
                continue;
#endif
            tc_fence_after();
            if (elect_one()) {
                const uint64_t a0 = sdesc(kbase + s * kSideBytes, 16, 1024, 2);
                const uint64_t b0 = sdesc(wg0 + w * kWgBytes, 128, 2048, 0);
#pragma unroll
                for (uint32_t kk = 0; kk < kHd / 16; ++kk) // K: 32 B steps in a 128-B row, then next half
                    mma_f16(tmem + 128 * w + 32 * b, a0 + (((kk >> 2) * kHalfBytes + (kk & 3u) * 32) >> 4),
                            b0 + kk * (256 >> 4), id_s, kk > 0);
                mma_commit(&wb[w].sfull[b]);
                mma_commit(&kempty[s]); // the K half is free once S is computed
            }
            __syncwarp();
            if (k == 0)
                (w ? mw1 : mw0) += 1;
            (w ? nw1 : nw0) += 1;
            if (++s == kKStages) {
                s = 0;
                ph ^= 1;
            }
            have = S.next(c, slots, n_items, w, k, I);
        }
    } else if (warp == 3) { // ---------------- PV issuer (whole warp, one elected lane issues) ----------------
        // O^T = V^T . P per tile, per warpgroup in its tile order, as soon as P, the O
        // buffer and the V tile are ready. The tile stream is walked in the same order
        // as the S issuer's, giving each tile its V ring position and K-step count.
        constexpr uint32_t fmt = std::is_same_v<T, __nv_bfloat16> ? 1u : 0u;
        constexpr uint32_t id_o = idesc(fmt, 1, 1, kHd, kN); // O^T = V^T . P (both MN-major)
        constexpr uint32_t kFifo = 8; // queued tiles per warpgroup (byte entries of a u64)
        Stream S;
        S.init(c, slots, n_items, queue, warp == 0);
#if KVR_TC_PVWAIT
        {
            // strictly in stream order (the order the S issuer and the producers use), each
            // condition awaited with the suspending try_wait instead of polling both
            // warpgroups' queues: no stage can be reached out of its fill order
            const uint32_t vbase = smem_u32(vbuf), wg0 = smem_u32(wgbuf);
            uint32_t w = 0, k = 0, sv = 0, phv = 0, pvw[2] = {0, 0}, ocur = 0; // ocur bit w: O buffer
            Item I;
            while (S.next(c, slots, n_items, w, k, I)) {
                const uint32_t nk = tile_of(I, k).nk, pvn = pvw[w], b = pvn & 1u, par = (pvn >> 1) & 1u;
                mbar_wait(&wb[w].pfull[b], par);
#if !KVR_TC_LAZY
                mbar_wait(&wb[w].oempty[b], par ^ 1u);
#endif
                mbar_wait(&vfull[sv], phv);
                tc_fence_after();
#if KVR_TC_LAZY
                // O buffer epochs: a flip (the softmax raised its held maximum) closes the old
                // buffer — one commit tracks every PV in it — and starts the other one fresh;
                // the item's last PV closes its buffer for the final read
                const bool flip = k > 0 && wb[w].pflag[b] != 0u;
                const uint32_t ob = ((ocur >> w) & 1u) ^ (flip ? 1u : 0u);
                const bool last = k + 1 == I.n_tiles;
                if (elect_one()) {
                    if (flip)
                        mma_commit(&wb[w].ofull[ob ^ 1u]);
                    const uint64_t a0 = sdesc(vbase + sv * kSideBytes, kHalfBytes, 1024, 2);
                    const uint64_t b0 = sdesc(wg0 + w * kWgBytes + kQBytes + b * kOpBytes, 128, 2048, 0);
                    const bool fresh = k == 0 || flip;
                    for (uint32_t kk = 0; kk < nk; ++kk)
                        mma_f16(tmem + 128 * w + 64 + 16 * ob, a0 + kk * (2048 >> 4), b0 + kk * (256 >> 4), id_o,
                                kk > 0 || !fresh);
                    if (last)
                        mma_commit(&wb[w].ofull[ob]);
                    mma_commit(&wb[w].pempty[b]);
                    mma_commit(&vempty[sv]);
                }
                __syncwarp();
                if (flip)
                    ocur ^= 1u << w;
#else
                if (elect_one()) {
                    const uint64_t a0 = sdesc(vbase + sv * kSideBytes, kHalfBytes, 1024, 2);
                    const uint64_t b0 = sdesc(wg0 + w * kWgBytes + kQBytes + b * kOpBytes, 128, 2048, 0);
                    for (uint32_t kk = 0; kk < nk; ++kk)
                        mma_f16(tmem + 128 * w + 64 + 16 * b, a0 + kk * (2048 >> 4), b0 + kk * (256 >> 4), id_o,
                                kk > 0);
                    mma_commit(&wb[w].ofull[b]);
                    mma_commit(&vempty[sv]);
                }
                __syncwarp();
#endif
                ++pvw[w];
                if (++sv == kVStages) {
                    sv = 0;
                    phv ^= 1;
                }
            }
        }
#else
        uint32_t w = 0, k = 0, sv = 0, phv = 0;
        uint32_t fw0 = 0, fw1 = 0, pv0 = 0, pv1 = 0; // tiles queued / PVs issued per warpgroup
        uint64_t ring0 = 0, ring1 = 0; // byte (n % 8) = V stage | V phase << 2 | K steps << 3
        // PVs of one stage must follow the stage's fill order: a warpgroup may reach the
        // PV of a later occupant of a stage before the other warpgroup's PV of the current
        // one — testing that stage's vfull two phases ahead would alias. Bit s = parity of
        // PVs issued for stage s.
        uint32_t vpar = 0;
        const uint32_t vbase = smem_u32(vbuf), wg0 = smem_u32(wgbuf);
        Item I;
        bool have = false, ended = false; // a fetched tile not yet queued / the stream's end seen
        while (!ended || have || pv0 < fw0 || pv1 < fw1) {
            if (!have && !ended) {
                const int r = S.next(c, slots, n_items, w, k, I, false);
                have = r > 0, ended = r == 0;
            }
            // queue stream tiles while the next one's warpgroup has room
            while (have && (w ? fw1 - pv1 : fw0 - pv0) < kFifo) {
                const uint32_t nk = tile_of(I, k).nk;
                const uint32_t sh = 8 * ((w ? fw1 : fw0) % kFifo);
                const uint64_t e = uint64_t(sv | phv << 2 | nk << 3) << sh;
                if (w)
                    ring1 = (ring1 & ~(uint64_t(0xff) << sh)) | e, ++fw1;
                else
                    ring0 = (ring0 & ~(uint64_t(0xff) << sh)) | e, ++fw0;
                if (++sv == kVStages) {
                    sv = 0;
                    phv ^= 1;
                }
                const int r = S.next(c, slots, n_items, w, k, I, false);
                have = r > 0, ended = ended || r == 0;
            }
            uint32_t go = 0;
#pragma unroll
            for (uint32_t x = 0; x < 2; ++x) {
                const uint32_t pvn = x ? pv1 : pv0;
                if (pvn >= (x ? fw1 : fw0))
                    continue;
                const uint32_t b = pvn & 1u, par = (pvn >> 1) & 1u;
                const uint32_t e = uint32_t(((x ? ring1 : ring0) >> (8 * (pvn % kFifo))) & 0xffu), st = e & 3u,
                               sph = (e >> 2) & 1u;
                const bool pf = mbar_test(&wb[x].pfull[b], par);
                const bool oe = mbar_test(&wb[x].oempty[b], par ^ 1u);
                const bool vf = mbar_test(&vfull[st], sph);
                go |= uint32_t(((vpar >> st) & 1u) == sph && pf && oe && vf) << x;
            }
            go = __shfl_sync(0xffffffffu, go, 0);
#pragma unroll
            for (uint32_t x = 0; x < 2; ++x) {
                if (!((go >> x) & 1u))
                    continue;
                const uint32_t pvn = x ? pv1 : pv0, b = pvn & 1u;
                const uint32_t e = uint32_t(((x ? ring1 : ring0) >> (8 * (pvn % kFifo))) & 0xffu), st = e & 3u,
                               nk = e >> 3;
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t a0 = sdesc(vbase + st * kSideBytes, kHalfBytes, 1024, 2);
                    const uint64_t b0 = sdesc(wg0 + x * kWgBytes + kQBytes + b * kOpBytes, 128, 2048, 0);
                    for (uint32_t kk = 0; kk < nk; ++kk) // +2048 B (V rows) / +256 B (P cores) per K step
                        mma_f16(tmem + 128 * x + 64 + 16 * b, a0 + kk * (2048 >> 4), b0 + kk * (256 >> 4), id_o,
                                kk > 0);
                    mma_commit(&wb[x].ofull[b]);
                    mma_commit(&vempty[st]);
                }
                __syncwarp();
                vpar ^= 1u << st;
                (x ? pv1 : pv0) += 1;
            }
        }
#endif
    } else if (warp >= 4) { // ---------------- softmax / correction warpgroups ----------------
        const uint32_t w = uint32_t(warp - 4) >> 2;     // warpgroup 0: warps 4-7, 1: warps 8-11
        const uint32_t t = threadIdx.x - 128 - 128 * w; // TMEM lane: token row of S, head dim of O
        const uint32_t wq = uint32_t(warp) & 3u;
        const uint32_t lane_base = ((32u * wq) << 16) + 128 * w;
        const uint32_t bar_id = 1 + w;
        WgBars &B = wb[w];
        uint8_t *qb = wgbuf + w * kWgBytes;
        float *rd = red + w * 2 * 4 * 8;
        float *ld = lred + w * 4 * 8;
        const float scale_log2 = 1.4426950408889634f / sqrtf(float(kHd));
        // live slots with an empty view (no near rows, no far rows: no item has a tile):
        // zero output. One slot-state load per slot — walking this CTA's static share
        // of items here (one dependent load each) held warpgroup 0 for up to ~100 us.
        if (w == 0)
            for (uint32_t s = blockIdx.x; s < c.n_slots; s += gridDim.x) {
                const kvr_slot_state st = slots[s];
                if (!st.live || st.written || st.far_count)
                    continue;
                float4 *os = reinterpret_cast<float4 *>(c.out + uint64_t(s) * c.L * c.Hq * kHd);
                for (uint32_t i = t; i < c.L * c.Hq * kHd / 4; i += 128)
                    os[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        uint32_t n = 0, m_items = 0;
        uint32_t obuf = 0, opc = 0; // lazy mode: current O buffer, ofull parity per buffer (bits)
        (void)obuf, (void)opc;
        Cursor cur;
        cur.init(queue, w, false);
        Item I, In;
        // the next item and its Q are fetched one item ahead (their global loads
        // overlap this item's tiles instead of stalling the item start;
        // measured C5 0.508 -> 0.499 ms, C3 unchanged)
        float xq[G];
        auto fetch_q = [&](const Item &J) {
            const uint64_t q0 = ((uint64_t(J.slot) * c.L + J.layer) * c.Hq + uint64_t(J.head) * G) * kHd;
#pragma unroll
            for (int g = 0; g < G; ++g)
                xq[g] = load_q(c, q0 + g * kHd + t);
        };
        bool have = cur.next(c, slots, n_items, w, I);
        if (have)
            fetch_q(I);
        while (have) {
            float *o = c.out + ((uint64_t(I.slot) * c.L + I.layer) * c.Hq + uint64_t(I.head) * G) * kHd;
            // Q (hi | lo) of this kv head's q-heads; thread t owns head dim t
            store_split<T, G, SP::QS>(qb, t, xq);
            fence_async_smem();
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&B.qfull);
            const bool have_next = cur.next(c, slots, n_items, w, In);
            if (have_next)
                fetch_q(In);
            ++m_items;
#if KVR_TC_LAZY
            // Lazy rescaling: O accumulates in TMEM across the item's tiles against a held
            // maximum m (every p = 2^(s - m) <= 2^kLazy); only when a tile's maximum exceeds
            // m + kLazy is O read back (flip: the PV issuer commits the old buffer and starts
            // the new one fresh), folded into acc and rescaled. The common tile therefore
            // never waits for its predecessor's PV (the per-tile O read of the eager path).
            float m[G], l[G], acc[G];
#pragma unroll
            for (int g = 0; g < G; ++g)
                m[g] = -INFINITY, l[g] = 0.f, acc[g] = 0.f;
            uint32_t ep = 0; // PVs of this item in the current O buffer
            auto fold_o = [&](uint32_t bo, const float (&sc_)[G]) {
                mbar_wait(&B.ofull[bo], (opc >> bo) & 1u);
                opc ^= 1u << bo;
                tc_fence_after();
                float ov[16];
                tmem_ld16(tmem + lane_base + 64 + 16 * bo, ov);
                tc_fence_before();
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float o_small = ov[G + g];
                    if constexpr (SP::PS == 3)
                        o_small += ov[2 * G + g];
                    acc[g] = (acc[g] + (ov[g] + o_small)) * sc_[g];
                }
            };
            for (uint32_t k = 0; k < I.n_tiles; ++k, ++n) {
                const uint32_t b = n & 1u;
                const Tile tl = tile_of(I, k);
                const uint64_t tok = tl.tok_r0 + t;
                const bool valid = t < tl.far_rows || (t >= kSub * tl.box_first &&
                                                      t < kSub * (tl.box_first + tl.n_boxes) && tok >= I.lo && tok < I.w);
                mbar_wait(&B.sfull[b], (n >> 1) & 1u);
                tc_fence_after();
                float sv[SP::NQ];
                if constexpr (SP::NQ == 32) {
                    float hi16[16], lo16[16];
                    tmem_ld16(tmem + lane_base + 32 * b, hi16);
                    tmem_ld16(tmem + lane_base + 32 * b + 16, lo16);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        sv[i] = hi16[i], sv[16 + i] = lo16[i];
                } else {
                    float v16[16];
                    tmem_ld16(tmem + lane_base + 32 * b, v16);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        sv[i] = v16[i];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&B.sempty[b]);
#if KVR_TC_VOTE
                float sc[G], mx[G];
                float scl[G], pv[G];
                // One barrier reduction decides whether any row of the tile raises a held
                // maximum past kLazy (always on an item's first tile: m = -inf); only then
                // are the tile maxima exchanged through shared memory.
                bool mine = false;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float s_small = sv[G + g];
                    if constexpr (SP::QS == 3)
                        s_small += sv[2 * G + g];
                    sc[g] = valid ? (sv[g] + s_small) * scale_log2 : -INFINITY;
                    mine = mine || sc[g] > m[g] + kLazy;
                }
                uint32_t any_raise;
                asm volatile("{\n\t.reg .pred q, r;\n\tsetp.ne.u32 q, %1, 0;\n\t"
                             "bar.red.or.pred r, %2, 128, q;\n\tselp.u32 %0, 1, 0, r;\n\t}"
                             : "=r"(any_raise)
                             : "r"(uint32_t(mine)), "r"(bar_id)
                             : "memory");
                const bool need = any_raise != 0;
                if (need) {
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        float v = sc[g];
#pragma unroll
                        for (int off = 16; off; off >>= 1)
                            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
                        mx[g] = v;
                    }
                    if (lane == 0)
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            rd[(b * 4 + wq) * 8 + g] = mx[g];
                    asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float tm = fmaxf(fmaxf(rd[(b * 4 + 0) * 8 + g], rd[(b * 4 + 1) * 8 + g]),
                                               fmaxf(rd[(b * 4 + 2) * 8 + g], rd[(b * 4 + 3) * 8 + g]));
                        const float mn = fmaxf(m[g], tm);
                        scl[g] = m[g] == -INFINITY ? 1.f : exp2f(m[g] - mn);
                        l[g] *= scl[g];
                        m[g] = mn;
                    }
                } else {
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        scl[g] = 1.f;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float p = valid ? exp2f(sc[g] - m[g]) : 0.f;
                    l[g] += p;
                    pv[g] = p;
                }
#else
                float scl[G], pv[G];
                float sc[G], mx[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float s_small = sv[G + g];
                    if constexpr (SP::QS == 3)
                        s_small += sv[2 * G + g];
                    sc[g] = valid ? (sv[g] + s_small) * scale_log2 : -INFINITY;
                    float v = sc[g];
#pragma unroll
                    for (int off = 16; off; off >>= 1)
                        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
                    mx[g] = v;
                }
                if (lane == 0)
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        rd[(b * 4 + wq) * 8 + g] = mx[g];
                asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
                // tile maxima (identical in every thread of the warpgroup: uniform decision)
                bool need = false;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float tm = fmaxf(fmaxf(rd[(b * 4 + 0) * 8 + g], rd[(b * 4 + 1) * 8 + g]),
                                           fmaxf(rd[(b * 4 + 2) * 8 + g], rd[(b * 4 + 3) * 8 + g]));
                    need = need || tm > m[g] + kLazy;
                    mx[g] = tm;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float mn = need ? fmaxf(m[g], mx[g]) : m[g];
                    scl[g] = m[g] == -INFINITY ? 1.f : exp2f(m[g] - mn);
                    l[g] *= scl[g];
                    m[g] = mn;
                    const float p = valid ? exp2f(sc[g] - mn) : 0.f;
                    l[g] += p;
                    pv[g] = p;
                }
#endif
                const bool flip = need && ep > 0;
                uint8_t *pb = qb + kQBytes + b * kOpBytes;
                if (n >= 2) // P buffer b: the PV of this warpgroup's tile n - 2 has read it
                    mbar_wait(&B.pempty[b], ((n >> 1) & 1u) ^ 1u);
                store_split<T, G, SP::PS>(pb, t, pv);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (wq == 0)
                        B.pflag[b] = flip ? 1u : 0u; // released by this warp's arrive
                    mbar_arrive(&B.pfull[b]);
                }
                if (flip) { // PV(k) runs into the other buffer while the old one is folded
                    fold_o(obuf, scl);
                    obuf ^= 1u;
                    ep = 0;
                } else if (need) {
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        acc[g] *= scl[g];
                }
                ++ep;
            }
            {
                float one[G];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    one[g] = 1.f;
                fold_o(obuf, one); // the item's last PV (committed by the PV issuer at its last tile)
            }
#else
            float m[G], l[G], acc[G], alpha_prev[G];
#pragma unroll
            for (int g = 0; g < G; ++g)
                m[g] = -INFINITY, l[g] = 0.f, acc[g] = 0.f, alpha_prev[g] = 1.f;
            auto correct = [&](uint32_t nn, const float (&alpha)[G]) {
                const uint32_t b = nn & 1u;
                mbar_wait(&B.ofull[b], (nn >> 1) & 1u);
                tc_fence_after();
                float ov[16];
                tmem_ld16(tmem + lane_base + 64 + 16 * b, ov);
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&B.oempty[b]);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float o_small = ov[G + g];
                    if constexpr (SP::PS == 3)
                        o_small += ov[2 * G + g];
                    acc[g] = acc[g] * alpha[g] + (ov[g] + o_small);
                }
            };
            for (uint32_t k = 0; k < I.n_tiles; ++k, ++n) {
                const uint32_t b = n & 1u;
                const Tile tl = tile_of(I, k);
                const uint64_t tok = tl.tok_r0 + t;
                const bool valid = t < tl.far_rows || (t >= kSub * tl.box_first &&
                                                      t < kSub * (tl.box_first + tl.n_boxes) && tok >= I.lo && tok < I.w);
                mbar_wait(&B.sfull[b], (n >> 1) & 1u);
                tc_fence_after();
                float sv[SP::NQ];
                if constexpr (SP::NQ == 32) {
                    float hi16[16], lo16[16];
                    tmem_ld16(tmem + lane_base + 32 * b, hi16);
                    tmem_ld16(tmem + lane_base + 32 * b + 16, lo16);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        sv[i] = hi16[i], sv[16 + i] = lo16[i];
                } else {
                    float v16[16];
                    tmem_ld16(tmem + lane_base + 32 * b, v16);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        sv[i] = v16[i];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&B.sempty[b]);
                float sc[G], mx[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float s_small = sv[G + g];
                    if constexpr (SP::QS == 3)
                        s_small += sv[2 * G + g];
                    sc[g] = valid ? (sv[g] + s_small) * scale_log2 : -INFINITY;
                    float v = sc[g];
#pragma unroll
                    for (int off = 16; off; off >>= 1)
                        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
                    mx[g] = v;
                }
                if (lane == 0)
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        rd[(b * 4 + wq) * 8 + g] = mx[g];
                asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
                float alpha[G], pv[G];
                uint8_t *pb = qb + kQBytes + b * kOpBytes;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float tm = fmaxf(fmaxf(rd[(b * 4 + 0) * 8 + g], rd[(b * 4 + 1) * 8 + g]),
                                           fmaxf(rd[(b * 4 + 2) * 8 + g], rd[(b * 4 + 3) * 8 + g]));
                    const float mn = fmaxf(m[g], tm);
                    alpha[g] = m[g] == -INFINITY ? 1.f : exp2f(m[g] - mn);
                    const float p = valid ? exp2f(sc[g] - mn) : 0.f;
                    l[g] = l[g] * alpha[g] + p;
                    m[g] = mn;
                    pv[g] = p;
                }
                store_split<T, G, SP::PS>(pb, t, pv);
                fence_async_smem();
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&B.pfull[b]);
                if (k > 0)
                    correct(n - 1, alpha_prev);
#pragma unroll
                for (int g = 0; g < G; ++g)
                    alpha_prev[g] = alpha[g];
            }
            correct(n - 1, alpha_prev);
#endif
            // row sums across the warpgroup, then normalise
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float v = l[g];
#pragma unroll
                for (int off = 16; off; off >>= 1)
                    v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0)
                    ld[wq * 8 + g] = v;
            }
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float z = ld[g] + ld[8 + g] + ld[16 + g] + ld[24 + g];
                o[g * kHd + t] = z > 0.f ? acc[g] / z : 0.f;
            }
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory"); // ld reused by the next item
            I = In;
            have = have_next;
        }
#ifdef KVR_HANG_CHECK
        if (blockIdx.x == 40 && (threadIdx.x & 127) == 0)
            printf("wg %u done: tiles %u items %u\n", w, n, m_items);
#endif
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
    // the last CTA to finish resets the item counter for the next launch (every CTA
    // has claimed past the end by now)
    if (threadIdx.x == 0 && atomicAdd(c.attn_sched + 1, 1u) == gridDim.x - 1) {
        c.attn_sched[0] = 0;
        c.attn_sched[1] = 0;
        __threadfence();
    }
}

using TcFn = void (*)(DevCtx, const TcMaps);

template <typename T> TcFn pick_tc(uint32_t g) {
    switch (g) {
    case 1: return k_attn_tc<T, 1>;
    case 2: return k_attn_tc<T, 2>;
    case 4: return k_attn_tc<T, 4>;
    case 8: return k_attn_tc<T, 8>;
    default: return nullptr;
    }
}

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;
EncodeFn encoder() {
    EncodeFn encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&encode), cudaEnableDefault, &q);
    return encode;
}

} // namespace

/// The tensor-core attention applies to head_dim 128, 16-bit elements and GQA
/// groups of 2, 4 or 8 with at most 128 far rows per slot.
bool attn_tc_supported(const DevCtx &c) {
    return c.hd == kHd && c.esz == 2 && (c.group == 1 || c.group == 2 || c.group == 4 || c.group == 8) &&
           c.far_cap <= kRows && c.R % kSub == 0;
}
bool attn_tc_ready(const DevCtx &c) { return attn_tc_supported(c) && c.G >= kRows; } // ring guard rows present

size_t attn_tc_smem() {
    return 1024 + (kKStages + kVStages) * kSideBytes + 2 * kWgBytes + (2 * 2 * 4 * 8 + 2 * 4 * 8) * 4 +
           2 * (kKStages + kVStages) * 8 +
           2 * sizeof(WgBars) + 16 + sizeof(ItemQueue);
}

const void *attn_tc_kernel(const DevCtx &c) {
    if (!attn_tc_ready(c))
        return nullptr;
    TcFn fn = c.elem_kind == KVR_ELEM_BF16 ? pick_tc<__nv_bfloat16>(c.group) : pick_tc<__half>(c.group);
    if (fn && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(attn_tc_smem())) !=
                  cudaSuccess)
        return nullptr; // shared-memory request refused: no tensor-core plan (open fails loudly)
    return reinterpret_cast<const void *>(fn);
}

/// ring: 4-D view (head_dim, 2*Hkv heads, R rows, L*n_slots), 64 x 1 x 32 x 1
/// boxes; far: 2-D view (row_elems, n_slots*L*max_chunks rows), 64 x 1 boxes
/// for gather4. Both with the 128-byte swizzle the UMMA descriptors expect.
bool attn_tc_maps(const DevCtx &c, TcMaps *maps) {
    const EncodeFn encode = encoder();
    if (!encode)
        return false;
    const uint64_t row = uint64_t(c.hd) * c.esz;
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    auto enc = [&](CUtensorMap *m, uint32_t rank, void *base, const cuuint64_t *dims, const cuuint64_t *strides,
                   const cuuint32_t *box) {
        return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, rank, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    // 32-row boxes: (head_dim, 2*Hkv heads, Rp plane rows incl. the guard, L*n_slots)
    const cuuint64_t d4[4] = {c.hd, 2ull * c.Hkv, c.Rp, uint64_t(c.L) * c.n_slots};
    const cuuint64_t s4[3] = {row, 2ull * c.Hkv * row, uint64_t(c.Rp) * 2 * c.Hkv * row};
    const cuuint32_t b4[4] = {64, 1, uint32_t(kSub), 1};
    // whole tiles: (64 dims, flat rows = plane * Rp + row, half, head, K|V); the box
    // (box kv = 1) lands as [half][128 rows][64 dims], one K or V half of a stage
    const cuuint64_t d5[5] = {64, uint64_t(c.L) * c.n_slots * c.Rp, 2, c.Hkv, 2};
    const cuuint64_t s5[4] = {2ull * c.Hkv * row, 128, row, uint64_t(c.Hkv) * row};
    const cuuint32_t b5[5] = {64, uint32_t(kRows), 2, 1, 1};
    // far rows: (row_elems, n_slots*L*max_chunks rows), 64 x 1 boxes for gather4
    const cuuint64_t df[2] = {c.row_elems, uint64_t(c.n_slots) * c.L * c.max_chunks};
    const cuuint64_t sf[1] = {uint64_t(c.row_elems) * c.esz};
    const cuuint32_t bf[2] = {64, 1};
    return enc(&maps->ring, 4, c.ring, d4, s4, b4) && enc(&maps->tile, 5, c.ring, d5, s5, b5) &&
           enc(&maps->far, 2, c.far, df, sf, bf);
}

void launch_attn_tc(const void *fn, const DevCtx &c, const TcMaps &maps, uint32_t grid, cudaStream_t s, bool pdl) {
    launch_ex(reinterpret_cast<TcFn>(const_cast<void *>(fn)), grid, kThreads, attn_tc_smem(), s, pdl, c, maps);
}

} // namespace kvr
