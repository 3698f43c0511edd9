// kvrail-b200 K-attn: fixed-shape window attention for every slot.
//
// Shape never changes: the grid covers (slot, layer, kv-head group) work items
// for all n_slots slots; a slot's visible set is its last min(written, W*)
// tokens (window ring) plus its selected far summaries, everything else is
// masked. Definition: attend() of far_view.cpp:113-155 per (layer, q-head)
// with GQA q-head j -> kv-head j / group, fp32 accumulation (1e-3 rel. bound).
//
// Per CTA (persistent): one producer warp streams K and V tiles (32 rows x G heads)
// out of the ring with 4-D TMA tensor loads (cp.async.bulk.tensor, mbarrier
// completion) into a shared-memory ring (192 KiB of stages) — at the window edges
// as 8-row boxes, skipping those with no live row; WPH*G consumer warps, WPH per kv head (4 for q-groups
// <= 2, else 2), take 32/WPH rows of each tile. QK^T: lane <-> head dims with q in
// registers, the per-row partial dot products are reduce-scattered by a halving
// shuffle butterfly. PV: lane <-> head dims, probabilities broadcast by shuffles.
// Online softmax in base 2; a head's warps merge their states through shared
// memory at item end. At g = 1
// this is a warp GEMV at the HBM roofline; GQA groups g >= 4 with head_dim 128 use
// the tcgen05 kernel in kvr_attn_tc.cu.
#include <algorithm>
#include <cstdio>
#include <cudaTypedefs.h>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

constexpr int kTile = 32; // tokens per tile (one per lane)
constexpr int kMaxG = 4;  // kv heads per CTA

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
__device__ inline void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "W_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}
__device__ inline void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                   uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
                 : "memory");
}

template <typename T> struct Pair;
template <> struct Pair<__half> {
    using V = __half2;
    static __device__ float2 f2(uint32_t u) { return __half22float2(*reinterpret_cast<const __half2 *>(&u)); }
    static __device__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};
template <> struct Pair<__nv_bfloat16> {
    static __device__ float2 f2(uint32_t u) {
        return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u));
    }
    static __device__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
};

__device__ inline float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1)
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ inline float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// DPL consecutive elements of a row as floats (lane <-> head dims).
template <typename T, int N> __device__ inline void load_dims(const T *p, float (&o)[N]) {
    if constexpr (sizeof(T) == 4) {
        if constexpr (N == 4) {
            const float4 v = *reinterpret_cast<const float4 *>(p);
            o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
        } else if constexpr (N == 2) {
            const float2 v = *reinterpret_cast<const float2 *>(p);
            o[0] = v.x, o[1] = v.y;
        } else {
            o[0] = *p;
        }
    } else {
        if constexpr (N == 4) {
            const uint2 v = *reinterpret_cast<const uint2 *>(p);
            const float2 a = Pair<T>::f2(v.x), b = Pair<T>::f2(v.y);
            o[0] = a.x, o[1] = a.y, o[2] = b.x, o[3] = b.y;
        } else if constexpr (N == 2) {
            const float2 a = Pair<T>::f2(*reinterpret_cast<const uint32_t *>(p));
            o[0] = a.x, o[1] = a.y;
        } else {
            o[0] = float(*p);
        }
    }
}

constexpr int kEdge = 8; // rows per TMA box at window edges (quarters with no live row are skipped)

/// Consumer warps per kv head: 4 (8 rows each) for small q-groups, where the warp
/// count — not registers — limits latency hiding; 2 (16 rows each) otherwise.
template <int QG> constexpr int warps_per_head() { return QG <= 2 ? 4 : 2; }

/// Online-softmax state of one consumer warp for QG q-heads sharing one kv head,
/// over R rows of each tile. QK^T: lane <-> head dims (q kept in registers), the R
/// per-row partial dot products are reduce-scattered across the warp by a halving
/// butterfly so lane l ends with the score of row l >> kShift. PV: lane <-> head
/// dims, the row probabilities are broadcast with shuffles.
template <typename T, int HD, int QG, int R> struct Attn {
    static constexpr int DPL = HD / 32;
    static constexpr int kShift = R == 16 ? 1 : 2; // lanes per row after the butterfly: 2 / 4
    static_assert(R == 16 || R == 8, "rows per warp");
    float q[QG][DPL];
    float m[QG], lsum[QG], acc[QG][DPL];

    __device__ void init(const DevCtx &c, uint64_t q0) { // queries [QG][HD] from element q0
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int g = 0; g < QG; ++g) {
            m[g] = -INFINITY;
            lsum[g] = 0.f;
#pragma unroll
            for (int k = 0; k < DPL; ++k) {
                q[g][k] = load_q(c, q0 + g * HD + DPL * lane + k);
                acc[g][k] = 0.f;
            }
        }
    }

    // R rows: row(r) -> K row pointer (V row = + v_off elements); valid bit r of `mask`.
    // FULL: all R rows valid (the common case) — no per-row predicates at all.
    template <bool FULL, typename RowFn>
    __device__ void block(RowFn row, uint32_t v_off, uint32_t mask, float scale_log2) {
        const int lane = threadIdx.x & 31;
        float part[QG][R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float k[DPL];
            if (FULL || (mask >> r & 1u)) {
                load_dims<T, DPL>(row(r) + DPL * lane, k);
            } else {
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    k[i] = 0.f;
            }
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                float a = 0.f;
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    a = fmaf(q[g][i], k[i], a);
                part[g][r] = a;
            }
        }
        // halving butterfly: R values -> 1 per lane (row lane >> kShift), then the
        // remaining kShift lane bits are summed
        float s[QG];
#pragma unroll
        for (int g = 0; g < QG; ++g) {
#pragma unroll
            for (int w = R / 2, bit = 16; w >= 1; w >>= 1, bit >>= 1) {
                const bool hi = lane & bit;
#pragma unroll
                for (int j = 0; j < w; ++j) {
                    const float send = hi ? part[g][j] : part[g][j + w];
                    const float keep = hi ? part[g][j + w] : part[g][j];
                    part[g][j] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
                }
            }
            float v = part[g][0];
#pragma unroll
            for (int b = 1 << (kShift - 1); b >= 1; b >>= 1)
                v += __shfl_xor_sync(0xffffffffu, v, b);
            s[g] = v * scale_log2;
        }
        const bool valid = FULL || (mask >> (lane >> kShift) & 1u);
        const bool leader = (lane & ((1 << kShift) - 1)) == 0; // one lane per row sums l
        float p[QG];
#pragma unroll
        for (int g = 0; g < QG; ++g) {
            const float sv = valid ? s[g] : -INFINITY;
            const float mn = fmaxf(m[g], warp_max(sv));
            const float alpha = mn == -INFINITY ? 1.f : exp2f(m[g] - mn);
            p[g] = valid ? exp2f(sv - mn) : 0.f;
            lsum[g] = lsum[g] * alpha + (leader ? p[g] : 0.f);
            m[g] = mn;
#pragma unroll
            for (int i = 0; i < DPL; ++i)
                acc[g][i] *= alpha;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!FULL && !(mask >> r & 1u))
                continue; // warp-uniform; masked rows may hold non-finite garbage
            float v[DPL];
            load_dims<T, DPL>(row(r) + v_off + DPL * lane, v);
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                const float pr = __shfl_sync(0xffffffffu, p[g], r << kShift);
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    acc[g][i] = fmaf(pr, v[i], acc[g][i]);
            }
        }
    }
};

template <typename T, int HD, int QG>
__global__ void __launch_bounds__(32 * (warps_per_head<QG>() * kMaxG + 1), 1)
    k_attn(DevCtx c, const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap edge_map,
           uint32_t G, uint32_t stages) {
    constexpr int WPH = warps_per_head<QG>(), RW = kTile / WPH; // warps per kv head, rows each
    using A = Attn<T, HD, QG, RW>;
    constexpr int DPL = A::DPL;
    constexpr int kState = 32 * QG * (2 + DPL); // floats of one warp's (m, l, acc) state
    extern __shared__ __align__(128) uint8_t smem[];
    pdl_wait(); // (no early trigger: the tail's CTAs, resident beside a CUDA-core K-attn CTA
                // and waiting, cost it ~0.6 % on C2; they launch as K-attn's CTAs exit)
    AttnSpan span_(c);
    TlScope tl_(c, kTlAttn);
    const uint32_t tile_elems = kTile * G * HD;
    T *tiles = reinterpret_cast<T *>(smem);                                  // [stages][K|V][32][G][HD]
    float *xchg = reinterpret_cast<float *>(tiles + size_t(stages) * 2 * tile_elems); // head merge
    uint64_t *full = reinterpret_cast<uint64_t *>(xchg + kMaxG * (WPH - 1) * kState);
    uint64_t *empty = full + stages;

    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t *far_ids = section<uint32_t>(c, h->off_far_ids);
    const uint32_t groups = c.Hkv / G;
    const uint32_t n_items = c.n_slots * c.L * groups;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], WPH * G);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto window = [&](uint32_t slot, uint64_t &lo, uint64_t &t0, uint32_t &n_tiles) {
        const uint64_t w = slots[slot].written;
        lo = w > c.W ? w - c.W : 0;
        t0 = lo & ~uint64_t(kTile - 1);
        n_tiles = w > t0 ? uint32_t((w - t0 + kTile - 1) / kTile) : 0;
    };

    if (warp == WPH * kMaxG) { // ---------------- producer: TMA tile loads ----------------
        if (lane != 0)
            return;
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tile_map)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&edge_map)) : "memory");
        uint32_t s = 0, phase = 0;
        const uint32_t bytes = 2 * tile_elems * sizeof(T);
        for (uint32_t it = blockIdx.x; it < n_items; it += gridDim.x) {
            const uint32_t hg = it % groups, l = (it / groups) % c.L, slot = it / (groups * c.L);
            if (!slots[slot].live)
                continue;
            uint64_t lo, t0;
            uint32_t n_tiles;
            window(slot, lo, t0, n_tiles);
            const uint64_t w = slots[slot].written;
            for (uint32_t k = 0; k < n_tiles; ++k) {
                mbar_wait(&empty[s], phase ^ 1);
                const uint64_t tk = t0 + uint64_t(k) * kTile;
                // interior tiles: one 32-row box each for K and V; window-edge tiles: only
                // the 8-row quarters holding a live row
                const int row0 = int(tk % c.R), z = int(slot * c.L + l);
                T *kt = tiles + size_t(s) * 2 * tile_elems;
                if (tk >= lo && tk + kTile <= w) {
                    mbar_expect_tx(&full[s], bytes);
                    tma_load_4d(kt, &tile_map, 0, int(hg * G), row0, z, &full[s]);
                    tma_load_4d(kt + tile_elems, &tile_map, 0, int(c.Hkv + hg * G), row0, z, &full[s]);
                } else {
                    uint32_t n_q = 0;
                    for (int j = 0; j < kTile / kEdge; ++j)
                        n_q += uint32_t(tk + j * kEdge < w && tk + (j + 1) * kEdge > lo);
                    mbar_expect_tx(&full[s], n_q * (bytes / (kTile / kEdge)));
                    for (int j = 0; j < kTile / kEdge; ++j) {
                        if (!(tk + j * kEdge < w && tk + (j + 1) * kEdge > lo))
                            continue;
                        T *dst = kt + size_t(j) * kEdge * G * HD;
                        tma_load_4d(dst, &edge_map, 0, int(hg * G), row0 + j * kEdge, z, &full[s]);
                        tma_load_4d(dst + tile_elems, &edge_map, 0, int(c.Hkv + hg * G), row0 + j * kEdge, z,
                                    &full[s]);
                    }
                }
                if (++s == stages) {
                    s = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }
    const uint32_t head_local = uint32_t(warp) / WPH, part = uint32_t(warp) % WPH;
    if (head_local >= G)
        return;

    // ---------- consumers: warps WPH*h .. WPH*h+WPH-1 own kv head hg*G + h; RW rows each ----------
    const float scale_log2 = 1.4426950408889634f / sqrtf(float(HD));
    float *states = xchg + size_t(head_local) * (WPH - 1) * kState; // parts 1.. park their state here
    uint32_t s = 0, phase = 0;
    for (uint32_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const uint32_t hg = it % groups, l = (it / groups) % c.L, slot = it / (groups * c.L);
        const kvr_slot_state st = slots[slot];
        if (!st.live)
            continue;
        const uint32_t kvh = hg * G + head_local;
        uint64_t lo, t0;
        uint32_t n_tiles;
        window(slot, lo, t0, n_tiles);
        const uint64_t w = st.written;
        A at;
        at.init(c, ((uint64_t(slot) * c.L + l) * c.Hq + uint64_t(kvh) * QG) * HD);
        // far summaries: rows straight from global memory
        const T *far_base = reinterpret_cast<const T *>(c.far) +
                            (uint64_t(slot) * c.L + l) * c.max_chunks * c.row_elems + uint64_t(kvh) * HD;
        for (uint32_t f0 = part * RW; f0 < st.far_count; f0 += kTile) {
            const uint32_t n = min(uint32_t(RW), st.far_count - f0);
            const uint32_t mask = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
            const uint32_t *ids = far_ids + st.far_begin + f0;
            auto far_row = [&](int r) {
                return far_base + uint64_t(ids[r < int(n) ? r : 0]) * c.row_elems;
            };
            if (mask == (1u << RW) - 1u)
                at.template block<true>(far_row, c.d_kv, mask, scale_log2);
            else
                at.template block<false>(far_row, c.d_kv, mask, scale_log2);
        }
        // near window tiles from the TMA pipeline
        for (uint32_t k = 0; k < n_tiles; ++k) {
            mbar_wait(&full[s], phase);
            const T *kt = tiles + size_t(s) * 2 * tile_elems;
            const uint64_t tok0 = t0 + uint64_t(k) * kTile + part * RW;
            uint32_t mask = 0;
#pragma unroll
            for (int r = 0; r < RW; ++r)
                mask |= uint32_t(tok0 + r >= lo && tok0 + r < w) << r;
            const T *base = kt + (size_t(part) * RW * G + head_local) * HD;
            auto tile_row = [&](int r) { return base + size_t(r) * G * HD; };
            if (mask == (1u << RW) - 1u)
                at.template block<true>(tile_row, tile_elems, mask, scale_log2);
            else if (mask) // a quarter with no live row was not even loaded
                at.template block<false>(tile_row, tile_elems, mask, scale_log2);
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&empty[s]);
            if (++s == stages) {
                s = 0;
                phase ^= 1;
            }
        }
        // merge the head's WPH states, then normalise
        const uint32_t bar = 1 + head_local;
        if (part) {
            float *mine = states + size_t(part - 1) * kState;
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                mine[(g * (2 + DPL) + 0) * 32 + lane] = at.m[g];
                mine[(g * (2 + DPL) + 1) * 32 + lane] = at.lsum[g];
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    mine[(g * (2 + DPL) + 2 + i) * 32 + lane] = at.acc[g][i];
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * WPH) : "memory");
        if (!part) {
            float *o = c.out + ((uint64_t(slot) * c.L + l) * c.Hq + uint64_t(kvh) * QG) * HD;
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                float mn = at.m[g];
#pragma unroll
                for (int j = 0; j < WPH - 1; ++j)
                    mn = fmaxf(mn, states[j * kState + (g * (2 + DPL) + 0) * 32 + lane]);
                const float a0 = mn == -INFINITY ? 0.f : exp2f(at.m[g] - mn);
                float z = at.lsum[g] * a0, sum[DPL];
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    sum[i] = at.acc[g][i] * a0;
#pragma unroll
                for (int j = 0; j < WPH - 1; ++j) {
                    const float *st = states + j * kState + g * (2 + DPL) * 32 + lane;
                    const float a = mn == -INFINITY ? 0.f : exp2f(st[0] - mn);
                    z += st[32] * a;
#pragma unroll
                    for (int i = 0; i < DPL; ++i)
                        sum[i] = fmaf(st[(2 + i) * 32], a, sum[i]);
                }
                z = warp_sum(z);
                const float inv = z > 0.f ? 1.f / z : 0.f;
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    o[g * HD + DPL * lane + i] = sum[i] * inv;
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * WPH) : "memory");
    }
}


using AttnFn = void (*)(DevCtx, const CUtensorMap, const CUtensorMap, uint32_t, uint32_t);

template <typename T, int HD> AttnFn pick_group(uint32_t g) {
    switch (g) {
    case 1: return k_attn<T, HD, 1>;
    case 2: return k_attn<T, HD, 2>;
    case 4: return k_attn<T, HD, 4>;
    case 8: return k_attn<T, HD, 8>;
    default: return nullptr;
    }
}
template <typename T> AttnFn pick_hd(uint32_t hd, uint32_t g) {
    switch (hd) {
    case 32: return pick_group<T, 32>(g);
    case 64: return pick_group<T, 64>(g);
    case 128: return pick_group<T, 128>(g);
    default: return nullptr;
    }
}

} // namespace

struct AttnPlan {
    AttnFn fn = nullptr;
    const void *tc = nullptr; // tensor-core kernel (kvr_attn_tc.cu) when chosen
    CUtensorMap map{}, edge_map{}; // 32-row tile boxes / 8-row edge boxes
    TcMaps tc_maps{};      // tensor-core kernel descriptors
    uint32_t G = 1, stages = 2, grid = 1, threads = 0;
    size_t smem = 0;
    char name[96] = {0};
};

AttnPlan *make_attn_plan(const DevCtx &c, int sms, int device, int mode) {
    auto *p = new AttnPlan();
    if (mode == 3 || (mode == 1 && c.group >= 4 && attn_tc_supported(c))) {
        p->tc = attn_tc_kernel(c);
        if (!p->tc || !attn_tc_maps(c, &p->tc_maps)) {
            delete p;
            return nullptr;
        }
        p->grid = uint32_t(sms);
        std::snprintf(p->name, sizeof(p->name), "k_attn_tc<%s,hd%u,g%u> tcgen05 M128 N16 K3+V3 rings",
                      c.elem_kind == KVR_ELEM_F16 ? "f16" : "bf16", c.hd, c.group);
        return p;
    }
    switch (c.elem_kind) {
    case KVR_ELEM_F16: p->fn = pick_hd<__half>(c.hd, c.group); break;
    case KVR_ELEM_BF16: p->fn = pick_hd<__nv_bfloat16>(c.hd, c.group); break;
    default: p->fn = pick_hd<float>(c.hd, c.group); break;
    }
    if (!p->fn) {
        delete p;
        return nullptr;
    }
    // kv heads per CTA: largest G <= 4 dividing Hkv with a <= 64 KiB stage
    const size_t row = size_t(c.hd) * c.esz;
    // (measured on C2: G = 4 / 2 / 1 -> 2.48 / 3.36 / 6.62 ms: consumer warps matter)
    for (uint32_t g : {4u, 2u, 1u})
        if (c.Hkv % g == 0 && 2 * kTile * g * row <= (64u << 10)) {
            p->G = g;
            break;
        }
    const size_t stage = 2 * kTile * p->G * row;
    p->stages = uint32_t(std::min<size_t>(8, (192u << 10) / stage)); // deeper rings for smaller stages
    if (p->stages < 2)
        p->stages = 2;
    const uint32_t wph = c.group <= 2 ? 4 : 2; // == warps_per_head<group>()
    p->threads = 32 * (wph * kMaxG + 1);
    p->smem = p->stages * stage + size_t(kMaxG) * (wph - 1) * 32 * c.group * (2 + c.hd / 32) * 4 +
              2 * p->stages * 8 + 16;
    p->grid = uint32_t(sms);
    if (cudaFuncSetAttribute(p->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)) != cudaSuccess) {
        delete p; // a geometry whose stages do not fit shared memory: no plan (open fails loudly)
        return nullptr;
    }

    // 4-D view of the ring: (head_dim, 2*Hkv heads, R rows, L*n_slots)
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&encode),
                            cudaEnableDefault, &q);
    if (!encode) {
        delete p;
        return nullptr;
    }
    const cuuint64_t dims[4] = {c.hd, 2ull * c.Hkv, c.R, uint64_t(c.L) * c.n_slots};
    const cuuint64_t strides[3] = {row, 2ull * c.Hkv * row, uint64_t(c.Rp) * 2 * c.Hkv * row}; // plane: Rp rows
    const cuuint32_t box[4] = {c.hd, p->G, uint32_t(kTile), 1};
    const cuuint32_t edge_box[4] = {c.hd, p->G, uint32_t(kEdge), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt =
        c.esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    const CUresult r = encode(&p->map, dt, 4, c.ring, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const CUresult r2 = encode(&p->edge_map, dt, 4, c.ring, dims, strides, edge_box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS || r2 != CUDA_SUCCESS || c.R % kTile) {
        delete p;
        return nullptr;
    }
    std::snprintf(p->name, sizeof(p->name), "k_attn<%s,hd%u,g%u> G=%u stages=%u warps/head=%u",
                  c.elem_kind == KVR_ELEM_F16 ? "f16" : c.elem_kind == KVR_ELEM_BF16 ? "bf16" : "f32",
                  c.hd, c.group, p->G, p->stages, wph);
    (void)device;
    return p;
}

void launch_attn(const AttnPlan *p, const DevCtx &c, cudaStream_t s, bool pdl) {
    if (p->tc) {
        launch_attn_tc(p->tc, c, p->tc_maps, p->grid, s, pdl);
        return;
    }
    launch_ex(p->fn, p->grid, p->threads, p->smem, s, pdl, c, p->map, p->edge_map, p->G, p->stages);
}

void free_attn_plan(AttnPlan *p) { delete p; }
const char *attn_variant(const AttnPlan *p) { return p ? p->name : "none"; }

} // namespace kvr
