// kvrail-b200 K-gather: move every staged train into the fixed-shape window.
//
// Input is K-scan's span list in train order. A near-window span of a slot is
// re-packed row by row into that slot's window ring (layer-major rows, token t
// at row t mod R, only rows of the live window range are written); a far-view
// span (a chunk summary slot) lands in the slot's far rows. Work unit = one
// (token, layer) row of 2*d_kv elements; each CTA loops over units with a
// TMA bulk-copy pipeline: an elected lane issues cp.async.bulk global->shared
// into a ring of stage buffers (mbarrier completion), then cp.async.bulk
// shared->global to the destination, recycling a buffer once its store has
// finished reading it (bulk_group read wait). Pure HBM-bound byte movement.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

constexpr uint32_t kMaxPiece = 32768;   // stage bytes: one load of consecutive layer rows

__device__ inline uint32_t smem_u32(const void *p) {
    return uint32_t(__cvta_generic_to_shared(p));
}

__device__ inline void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ inline void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ inline void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(phase)
                 : "memory");
}
__device__ inline void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ inline void bulk_s2g_nocommit(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ inline void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ inline void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ inline void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

/// Resolve unit -> (src, dst, bytes); bytes == 0 when the row is masked out.
struct Move {
    const uint8_t *src;
    uint8_t *dst;
    uint32_t bytes;
};

/// Source and destination of layer row `l` of gather-order token `tok_idx` inside span
/// `sp` (dst == nullptr: the window does not hold that row). Near spans land in the
/// slot's ring at row token mod R when the token is in [written - W*, + R); far spans
/// (summary slots) in the slot's far row of their chunk.
__device__ inline Move span_row(const DevCtx &c, const kvr_slot_state *slots, const GSpan &sp, uint64_t tok_idx,
                                uint32_t l) {
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    const uint64_t k = tok_idx - sp.tok_prefix;
    Move m{nullptr, nullptr, uint32_t(row_bytes)};
    m.src = c.arena + uint64_t(sp.block) * c.page_bytes + (sp.slot_begin + k) * c.token_bytes + l * row_bytes;
    if (sp.dev_slot >= c.n_slots)
        return m;
    const uint64_t tok = sp.first_token + k;
    if (sp.kind == 0) {
        const uint64_t w = slots[sp.dev_slot].written;
        const uint64_t lo_tok = w > c.W ? w - c.W : 0; // rows of [lo_tok, lo_tok + R) are live
        if (tok < lo_tok || tok >= lo_tok + c.R)
            return m;
        m.dst = c.ring + (ring_row(c, sp.dev_slot, l, uint32_t(tok % c.R)) * c.esz);
    } else {
        if (tok < KVR_SUMMARY_BASE)
            return m;
        const uint64_t chunk = tok - KVR_SUMMARY_BASE;
        if (chunk >= c.max_chunks)
            return m;
        m.dst = c.far + ((uint64_t(sp.dev_slot) * c.L + l) * c.max_chunks + chunk) * c.row_elems * c.esz;
    }
    return m;
}

/// Test hook: the same position `shift` ring rows further (wrapping in the slot's layer ring).
__device__ inline uint8_t *shifted_row(const DevCtx &c, uint8_t *dst, uint64_t shift) {
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    const uint64_t off = uint64_t(dst - c.ring), plane = uint64_t(c.Rp) * row_bytes;
    const uint64_t base = off / plane * plane, within = off - base;
    return c.ring + base + (within + (shift % c.R) * row_bytes) % (uint64_t(c.R) * row_bytes);
}

/// Bytes from a ring destination to its guard mirror (0: none; far rows have none).
__device__ inline uint64_t dst_mirror(const DevCtx &c, const uint8_t *dst) {
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz, plane = uint64_t(c.Rp) * row_bytes;
    if (!c.G || dst < c.ring || dst >= c.ring + uint64_t(c.n_slots) * c.L * plane)
        return 0;
    return (uint64_t(dst - c.ring) % plane) / row_bytes < c.G ? uint64_t(c.R) * row_bytes : 0;
}

/// Walks this CTA's contiguous range of units with a forward-moving span cursor (no
/// division or search per unit). A unit is `lg` consecutive layers of one token —
/// contiguous in the arena (token-major pages) — or, for rows larger than a stage,
/// one piece of one layer row.
struct Walker {
    uint64_t tok_idx;
    uint32_t grp, piece, cur;
    /// (whole warp) position at unit u0: span found by warp_last_le
    __device__ void init(const DevCtx &c, uint32_t n_spans, uint64_t u0, uint32_t groups, uint32_t pieces) {
        piece = uint32_t(u0 % pieces);
        const uint64_t gu = u0 / pieces;
        grp = uint32_t(gu % groups);
        tok_idx = gu / groups;
        cur = warp_last_le(n_spans, tok_idx, [&](uint32_t i) { return c.gspans[i].tok_prefix; });
    }
    __device__ void advance(const DevCtx &c, uint32_t n_spans, uint32_t groups, uint32_t pieces) {
        if (++piece < pieces)
            return;
        piece = 0;
        if (++grp < groups)
            return;
        grp = 0;
        ++tok_idx;
        while (cur + 1 < n_spans && c.gspans[cur + 1].tok_prefix <= tok_idx)
            ++cur;
    }
};

/// A unit in flight: one bulk load of `bytes` into a stage, `nl` bulk stores of
/// `row` bytes each (consecutive layers: destinations one ring plane apart).
struct Unit {
    uint8_t *dst0;        // destination of the first layer
    uint64_t dst_stride;  // bytes between the layers' destinations
    uint64_t mirror;      // bytes to the ring rows' guard copies (0: none)
    uint32_t row, nl;
};

// One warp per CTA, one CTA per SM: lane 0 drives a kStages-deep ring of
// kMaxPiece-byte stages over the CTA's contiguous unit range. Loads run kAhead
// units in front of the stores; a stage is reloaded only after the stores that
// read it have drained (bulk_group read wait). A unit is up to kMaxPiece / row
// consecutive layers of one token: ONE load (contiguous in the arena), then one
// store per layer into that layer's window ring plane.
template <int kStages, int kAhead>
__global__ void __launch_bounds__(32) k_gather(DevCtx c) {
    pdl_wait();
    pdl_trigger();
    GatherSpan span_(c);
    TlScope tl_(c, kTlGather);
    extern __shared__ __align__(128) uint8_t stage[];
    __shared__ __align__(8) uint64_t full[kStages];
    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t n_spans = c.scan->spans;
    const uint64_t tokens = c.scan->total_tokens;
    if (tokens == 0 || (c.scan->status & 4u))
        return;
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    const uint32_t pieces = row_bytes > kMaxPiece ? uint32_t((row_bytes + kMaxPiece - 1) / kMaxPiece) : 1;
    // layers per unit: as many as fill a stage, fewer when the step is small (keep
    // >= 8 units per CTA so every SM streams)
    uint32_t lg = pieces > 1 ? 1 : uint32_t(c.L < kMaxPiece / row_bytes ? c.L : kMaxPiece / row_bytes);
    while (lg > 1 && tokens * ((c.L + lg - 1) / lg) < 8ull * gridDim.x)
        lg = (lg + 1) / 2;
    const uint32_t groups = (c.L + lg - 1) / lg;
    const uint64_t units = tokens * groups * pieces;
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = units < u0 + per ? units : u0 + per;
    if (u0 >= u1)
        return;
    Walker wk;
    wk.init(c, n_spans, u0, groups, pieces); // the whole warp searches; lane 0 then drives the ring
    if (threadIdx.x != 0)
        return;
    for (int s = 0; s < kStages; ++s)
        mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t drop = c.fault[0], shift = c.fault[1]; // test hooks (off: ~0, 0)
    uint64_t next = u0;
    Unit mv[kStages];
    uint32_t phase_bits = 0;
    auto issue = [&](int s) {
        while (next < u1) {
            const GSpan &sp = c.gspans[wk.cur];
            const uint32_t l0 = wk.grp * lg, nl = min(lg, c.L - l0);
            Move m = span_row(c, slots, sp, wk.tok_idx, l0);
            if (drop != ~0ull && (wk.cur == drop || drop == KVR_FAULT_ALL))
                m.dst = nullptr;
            Unit u{};
            if (m.dst) {
                const uint64_t off0 = uint64_t(wk.piece) * kMaxPiece;
                u.row = pieces > 1 ? uint32_t(row_bytes - off0 < kMaxPiece ? row_bytes - off0 : kMaxPiece) : uint32_t(row_bytes);
                u.nl = nl;
                u.dst0 = m.dst + off0;
                if (shift && sp.kind == 0)
                    u.dst0 = shifted_row(c, u.dst0, shift);
                // the next layer's row: one ring plane (Rp rows) / far plane further
                u.dst_stride = (sp.kind == 0 ? uint64_t(c.Rp) : uint64_t(c.max_chunks)) * row_bytes;
                u.mirror = sp.kind == 0 ? dst_mirror(c, u.dst0) : 0;
                m.src += off0;
            }
            ++next;
            wk.advance(c, n_spans, groups, pieces);
            if (u.dst0) {
                mv[s] = u;
                const uint32_t bytes = u.row * u.nl;
                mbar_expect_tx(&full[s], bytes);
                bulk_g2s(stage + size_t(s) * kMaxPiece, m.src, bytes, &full[s]);
                return true;
            }
        }
        return false;
    };
    uint64_t issued = 0, stored = 0;
    while (issued < kAhead && issue(int(issued % kStages)))
        ++issued;
    while (stored < issued) {
        const int s = int(stored % kStages);
        mbar_wait(&full[s], (phase_bits >> s) & 1u);
        phase_bits ^= 1u << s;
        const Unit &u = mv[s];
        for (uint32_t j = 0; j < u.nl; ++j) {
            const uint8_t *from = stage + size_t(s) * kMaxPiece + size_t(j) * u.row;
            bulk_s2g_nocommit(u.dst0 + j * u.dst_stride, from, u.row);
            if (u.mirror)
                bulk_s2g_nocommit(u.dst0 + u.mirror + j * u.dst_stride, from, u.row);
        }
        bulk_commit();
        ++stored;
        // next load reuses the stage stored (kStages - kAhead) groups ago
        bulk_wait_read<kStages - kAhead - 1>();
        if (issue(int(issued % kStages)))
            ++issued;
    }
    bulk_wait_all();
}

// Two-warp variant: warp 0's lane 0 only loads (TMA bulk, global -> shared), warp 1's
// lane 0 only stores (one bulk store per layer row + guard copies) and hands each stage
// back through an `empty` mbarrier once its stores have read it — the loads of later
// units no longer queue behind the store issue of earlier ones (8 stores per unit for
// 4 KiB rows). Unit descriptions travel through shared memory (released by the loader's
// arrive on `full`, acquired by the storer's wait).
template <int kSt>
__global__ void __launch_bounds__(64) k_gather2(DevCtx c) {
    pdl_wait();
    pdl_trigger();
    GatherSpan span_(c);
    TlScope tl_(c, kTlGather);
    extern __shared__ __align__(128) uint8_t stage[];
    __shared__ __align__(8) uint64_t full[kSt], empty[kSt];
    __shared__ Unit info[kSt];
    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t n_spans = c.scan->spans;
    const uint64_t tokens = c.scan->total_tokens;
    if (tokens == 0 || (c.scan->status & 4u))
        return;
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    const uint32_t pieces = row_bytes > kMaxPiece ? uint32_t((row_bytes + kMaxPiece - 1) / kMaxPiece) : 1;
    uint32_t lg = pieces > 1 ? 1 : uint32_t(c.L < kMaxPiece / row_bytes ? c.L : kMaxPiece / row_bytes);
    while (lg > 1 && tokens * ((c.L + lg - 1) / lg) < 8ull * gridDim.x)
        lg = (lg + 1) / 2;
    const uint32_t groups = (c.L + lg - 1) / lg;
    const uint64_t units = tokens * groups * pieces;
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = units < u0 + per ? units : u0 + per;
    if (u0 >= u1)
        return;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSt; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) { // ---- loader ----
        Walker wk;
        wk.init(c, n_spans, u0, groups, pieces);
        if (lane != 0)
            return;
        const uint64_t drop = c.fault[0], shift = c.fault[1]; // test hooks (off: ~0, 0)
        uint32_t n = 0;
        for (uint64_t next = u0; next < u1; ++next) {
            const GSpan &sp = c.gspans[wk.cur];
            const uint32_t l0 = wk.grp * lg, nl = min(lg, c.L - l0);
            Move m = span_row(c, slots, sp, wk.tok_idx, l0);
            if (drop != ~0ull && (wk.cur == drop || drop == KVR_FAULT_ALL))
                m.dst = nullptr;
            const uint32_t piece = wk.piece;
            wk.advance(c, n_spans, groups, pieces);
            if (!m.dst)
                continue;
            Unit u{};
            const uint64_t off0 = uint64_t(piece) * kMaxPiece;
            u.row = pieces > 1 ? uint32_t(row_bytes - off0 < kMaxPiece ? row_bytes - off0 : kMaxPiece) : uint32_t(row_bytes);
            u.nl = nl;
            u.dst0 = m.dst + off0;
            if (shift && sp.kind == 0)
                u.dst0 = shifted_row(c, u.dst0, shift);
            u.dst_stride = (sp.kind == 0 ? uint64_t(c.Rp) : uint64_t(c.max_chunks)) * row_bytes;
            u.mirror = sp.kind == 0 ? dst_mirror(c, u.dst0) : 0;
            const int s = int(n % kSt);
            if (n >= uint32_t(kSt))
                mbar_wait(&empty[s], ((n / kSt) - 1) & 1u); // its previous stores have read it
            info[s] = u;
            mbar_expect_tx(&full[s], u.row * u.nl);
            bulk_g2s(stage + size_t(s) * kMaxPiece, m.src + off0, u.row * u.nl, &full[s]);
            ++n;
        }
        // end of the stream: an empty unit, announced without bytes
        const int s = int(n % kSt);
        if (n >= uint32_t(kSt))
            mbar_wait(&empty[s], ((n / kSt) - 1) & 1u);
        info[s].nl = 0;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    } else if (lane == 0) { // ---- storer ----
        for (uint32_t n = 0;; ++n) {
            const int s = int(n % kSt);
            mbar_wait(&full[s], (n / kSt) & 1u);
            const Unit u = info[s];
            if (!u.nl)
                break;
            for (uint32_t j = 0; j < u.nl; ++j) {
                const uint8_t *from = stage + size_t(s) * kMaxPiece + size_t(j) * u.row;
                bulk_s2g_nocommit(u.dst0 + j * u.dst_stride, from, u.row);
                if (u.mirror)
                    bulk_s2g_nocommit(u.dst0 + u.mirror + j * u.dst_stride, from, u.row);
            }
            bulk_commit();
            // the previous unit's stores have read their stage: hand it back
            if (n > 0) {
                bulk_wait_read<1>();
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[(n - 1) % kSt]))
                             : "memory");
            }
        }
        bulk_wait_all();
    }
}

// Register-staged variant: every warp of a full-occupancy grid moves (token, layer,
// kUnit-byte piece) units, kFly of them in flight (all their loads before their
// stores); each lane moves kUnit / 512 int4 of a unit. kInterleave: warp w takes
// units w, w + W, ... (concurrent warps touch neighbouring addresses) instead of a
// contiguous range. Same work list, destinations and fault hooks as k_gather.
constexpr int kVecWarps = 8; // warps per CTA

struct VecUnit {
    const int4 *src;
    int4 *dst;
    uint32_t n16;    // int4s in the unit
    uint32_t mirror; // int4s to the ring row's guard copy (0: none)
};

template <int kUnit, int kFly, bool kInterleave>
__global__ void __launch_bounds__(32 * kVecWarps) k_gather_vec(DevCtx c) {
    pdl_wait();
    pdl_trigger();
    GatherSpan span_(c);
    TlScope tl_(c, kTlGather);
    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t n_spans = c.scan->spans;
    const uint64_t tokens = c.scan->total_tokens;
    if (tokens == 0 || (c.scan->status & 4u))
        return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    const uint32_t pieces = uint32_t((row_bytes + kUnit - 1) / kUnit);
    const uint64_t units = tokens * c.L * pieces;
    const uint64_t warps = uint64_t(gridDim.x) * kVecWarps;
    const uint64_t w = uint64_t(blockIdx.x) * kVecWarps + (threadIdx.x >> 5);
    const uint64_t per = (units + warps - 1) / warps;
    const uint64_t u0 = kInterleave ? w : w * per;
    const uint64_t u1 = kInterleave ? units : (units < u0 + per ? units : u0 + per);
    const uint64_t ustep = kInterleave ? warps : 1;
    if (u0 >= u1)
        return;
    const uint64_t drop = c.fault[0], shift = c.fault[1]; // test hooks (off: ~0, 0)
    auto unit_of = [&](uint64_t u, VecUnit &vu) {
        const uint32_t piece = uint32_t(u % pieces), l = uint32_t((u / pieces) % c.L);
        const uint64_t tok_idx = u / pieces / c.L;
        uint32_t lo = 0, hi = n_spans; // last span with tok_prefix <= tok_idx
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (c.gspans[mid].tok_prefix <= tok_idx)
                lo = mid;
            else
                hi = mid;
        }
        const GSpan sp = c.gspans[lo];
        Move m = span_row(c, slots, sp, tok_idx, l);
        if (drop != ~0ull && (lo == drop || drop == KVR_FAULT_ALL))
            m.dst = nullptr;
        else if (shift && m.dst && sp.kind == 0)
            m.dst = shifted_row(c, m.dst, shift);
        const uint64_t off0 = uint64_t(piece) * kUnit;
        const uint64_t n = row_bytes - off0 < kUnit ? row_bytes - off0 : kUnit;
        vu.src = reinterpret_cast<const int4 *>(m.src + off0);
        vu.dst = m.dst ? reinterpret_cast<int4 *>(m.dst + off0) : nullptr;
        vu.n16 = uint32_t(n / 16);
        vu.mirror = m.dst && sp.kind == 0 ? uint32_t(dst_mirror(c, m.dst) / 16) : 0;
    };
    constexpr int kPer = kUnit / 16 / 32; // int4 per lane per unit
    for (uint64_t u = u0; u < u1; u += ustep * kFly) {
        VecUnit a[kFly];
        int4 v[kFly][kPer];
#pragma unroll
        for (int f = 0; f < kFly; ++f) {
            const uint64_t uf = u + uint64_t(f) * ustep;
            if (uf < u1)
                unit_of(uf, a[f]);
            else
                a[f].dst = nullptr;
        }
#pragma unroll
        for (int f = 0; f < kFly; ++f)
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const uint32_t q = lane + 32u * i;
                if (a[f].dst && q < a[f].n16)
                    v[f][i] = __ldcs(a[f].src + q);
            }
#pragma unroll
        for (int f = 0; f < kFly; ++f)
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const uint32_t q = lane + 32u * i;
                if (a[f].dst && q < a[f].n16) {
                    a[f].dst[q] = v[f][i];
                    if (a[f].mirror)
                        a[f].dst[q + a[f].mirror] = v[f][i];
                }
            }
    }
}

// Parity read-back: one CTA per gather-order token; layer rows from the destination
// (or the arena for rows the window does not hold), token-major like the reference.
__global__ void __launch_bounds__(256) k_read_staged(DevCtx c, uint64_t tok_begin, uint64_t count, uint8_t *out,
                                                     uint8_t *in_window) {
    const kvr_slot_state *slots = section<kvr_slot_state>(c, hdr(c)->off_slots);
    const uint32_t n_spans = c.scan->spans;
    const uint64_t row_bytes = uint64_t(c.row_elems) * c.esz;
    for (uint64_t i = blockIdx.x; i < count; i += gridDim.x) {
        const uint64_t tok_idx = tok_begin + i;
        uint32_t lo = 0, hi = n_spans; // last span with tok_prefix <= tok_idx
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (c.gspans[mid].tok_prefix <= tok_idx)
                lo = mid;
            else
                hi = mid;
        }
        const GSpan sp = c.gspans[lo];
        bool all = true;
        for (uint32_t l = 0; l < c.L; ++l) {
            const Move m = span_row(c, slots, sp, tok_idx, l);
            all = all && m.dst != nullptr;
            const int4 *src = reinterpret_cast<const int4 *>(m.dst ? m.dst : m.src);
            int4 *dst = reinterpret_cast<int4 *>(out + i * c.token_bytes + l * row_bytes);
            for (uint64_t q = threadIdx.x; q < row_bytes / 16; q += blockDim.x)
                dst[q] = src[q];
        }
        if (threadIdx.x == 0 && in_window) {
            // 1: delivered; 0: a near row older than written - W* (behind the live
            // window: not part of the window by definition); 2: not held otherwise
            uint8_t f = 1;
            if (!all) {
                f = 2;
                if (sp.kind == 0 && sp.dev_slot < c.n_slots) {
                    const uint64_t w = slots[sp.dev_slot].written;
                    f = sp.first_token + (tok_idx - sp.tok_prefix) + c.W < w ? 0 : 2;
                }
            }
            in_window[i] = f;
        }
    }
}

} // namespace

void launch_read_staged(const DevCtx &c, cudaStream_t s, uint64_t tok_begin, uint64_t count, uint8_t *out,
                        uint8_t *in_window) {
    if (count)
        k_read_staged<<<unsigned(count < 4096 ? count : 4096), 256, 0, s>>>(c, tok_begin, count, out, in_window);
}

namespace {
// KVR_GATHER selects the K-gather kernel (A/B): split (loader warp + storer warp, 6 x
// 32 KiB stages, 1 CTA/SM; default) | tma (one lane loads and stores, 4 loads ahead) |
// tma5 (5 ahead) | tma2 (3 stages, 2 ahead, 2 CTAs/SM) | vec (register-staged, 4 KiB
// units, 2 in flight) | ivec (interleaved)
int gather_kind() {
    static const int k = [] {
        const char *e = getenv("KVR_GATHER");
        const std::string v = e ? e : "";
        return v == "tma" ? 0 : v == "tma5" ? 1 : v == "tma2" ? 2 : v == "vec" ? 3 : v == "ivec" ? 4 : v == "split7" ? 6 : 5;
    }();
    return k;
}
} // namespace

cudaError_t prepare_gather(const DevCtx &) {
    cudaError_t e = cudaFuncSetAttribute(k_gather<6, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(6 * kMaxPiece));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gather<6, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(6 * kMaxPiece));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gather<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(3 * kMaxPiece));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gather2<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(6 * kMaxPiece));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gather2<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(7 * kMaxPiece));
    return e;
}

void launch_gather(const DevCtx &c, cudaStream_t s, int sms, bool pdl) {
    const unsigned n = unsigned(sms);
    switch (gather_kind()) {
    case 1: launch_ex(k_gather<6, 5>, n, 32, size_t(6) * kMaxPiece, s, pdl, c); break;
    case 2: launch_ex(k_gather<3, 2>, n * 2, 32, size_t(3) * kMaxPiece, s, pdl, c); break;
    case 3: launch_ex(k_gather_vec<4096, 2, false>, n * 2, 32 * kVecWarps, 0, s, pdl, c); break;
    case 4: launch_ex(k_gather_vec<4096, 2, true>, n * 2, 32 * kVecWarps, 0, s, pdl, c); break;
    case 5: launch_ex(k_gather2<6>, n, 64, size_t(6) * kMaxPiece, s, pdl, c); break;
    case 6: launch_ex(k_gather2<7>, n, 64, size_t(7) * kMaxPiece, s, pdl, c); break;
    default: launch_ex(k_gather<6, 4>, n, 32, size_t(6) * kMaxPiece, s, pdl, c); break;
    }
}

} // namespace kvr
