// kvrail-b200 K-attn: fixed-shape window attention for every slot.
//
// Shape never changes: the grid covers (slot, layer, kv-head group) work items
// for all n_slots slots; a slot's visible set is its last min(written, W*)
// tokens (window ring) plus its selected far summaries, everything else is
// masked. Definition: attend() of far_view.cpp:113-155 per (layer, q-head)
// with GQA q-head j -> kv-head j / group, fp32 accumulation (1e-3 rel. bound).
//
// Per CTA (persistent): one producer warp streams K and V half-tiles (16 rows x G
// heads) out of the ring with 4-D TMA tensor loads (cp.async.bulk.tensor,
// mbarrier completion) into a 3-stage shared-memory ring, skipping halves with no
// live row; 2*G consumer warps, a pair per kv head, take 16 rows each. QK^T: lane
// <-> head dims with q in registers, the 16 per-row partial dot products are
// reduce-scattered by a halving shuffle butterfly (lane l ends with row l >> 1).
// PV: lane <-> head dims, probabilities broadcast by shuffles. Online softmax in
// base 2; the pair merges its states through shared memory at item end. At g = 1
// this is a warp GEMV at the HBM roofline; GQA groups g >= 4 with head_dim 128 use
// the tcgen05 kernel in kvr_attn_tc.cu.
#include <algorithm>
#include <cstdio>
#include <cudaTypedefs.h>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

constexpr int kTile = 32; // tokens per tile (one per lane)
constexpr int kMaxG = 4;  // kv heads per CTA (a pair of consumer warps each)

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

constexpr int kHalf = 16; // tokens per consumer warp per tile

/// Online-softmax state of one consumer warp for QG q-heads sharing one kv head.
/// QK^T: lane <-> head dims (q kept in registers), the 16 per-token partial dot
/// products are reduce-scattered across the warp by a halving butterfly so lane
/// l ends with the score of token l >> 1. PV: lane <-> head dims, the token
/// probabilities are broadcast with shuffles.
template <typename T, int HD, int QG> struct Attn {
    static constexpr int DPL = HD / 32;
    float q[QG][DPL];
    float m[QG], lsum[QG], acc[QG][DPL];

    __device__ void init(const float *qsrc) { // qsrc: [QG][HD] floats
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int g = 0; g < QG; ++g) {
            m[g] = -INFINITY;
            lsum[g] = 0.f;
#pragma unroll
            for (int k = 0; k < DPL; ++k) {
                q[g][k] = qsrc[g * HD + DPL * lane + k];
                acc[g][k] = 0.f;
            }
        }
    }

    // 16 rows: row(r) -> K row pointer (V row = + v_off elements); valid bit r of `mask`.
    // FULL: all 16 rows valid (the common case) — no per-row predicates at all.
    template <bool FULL, typename RowFn>
    __device__ void block(RowFn row, uint32_t v_off, uint32_t mask, float scale_log2) {
        const int lane = threadIdx.x & 31;
        float part[QG][kHalf];
#pragma unroll
        for (int r = 0; r < kHalf; ++r) {
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
        // halving butterfly: 16 values -> 1 per lane (token lane >> 1)
        float s[QG];
#pragma unroll
        for (int g = 0; g < QG; ++g) {
#pragma unroll
            for (int w = kHalf / 2, bit = 16; w >= 1; w >>= 1, bit >>= 1) {
                const bool hi = lane & bit;
#pragma unroll
                for (int j = 0; j < w; ++j) {
                    const float send = hi ? part[g][j] : part[g][j + w];
                    const float keep = hi ? part[g][j + w] : part[g][j];
                    part[g][j] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
                }
            }
            s[g] = (part[g][0] + __shfl_xor_sync(0xffffffffu, part[g][0], 1)) * scale_log2;
        }
        const bool valid = FULL || (mask >> (lane >> 1) & 1u);
        float p[QG];
#pragma unroll
        for (int g = 0; g < QG; ++g) {
            const float sv = valid ? s[g] : -INFINITY;
            const float mn = fmaxf(m[g], warp_max(sv));
            const float alpha = mn == -INFINITY ? 1.f : exp2f(m[g] - mn);
            p[g] = valid ? exp2f(sv - mn) : 0.f;
            lsum[g] = lsum[g] * alpha + ((lane & 1) ? 0.f : p[g]);
            m[g] = mn;
#pragma unroll
            for (int i = 0; i < DPL; ++i)
                acc[g][i] *= alpha;
        }
#pragma unroll
        for (int r = 0; r < kHalf; ++r) {
            if (!FULL && !(mask >> r & 1u))
                continue; // warp-uniform; masked rows may hold non-finite garbage
            float v[DPL];
            load_dims<T, DPL>(row(r) + v_off + DPL * lane, v);
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                const float pr = __shfl_sync(0xffffffffu, p[g], 2 * r);
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    acc[g][i] = fmaf(pr, v[i], acc[g][i]);
            }
        }
    }
};

template <typename T, int HD, int QG>
__global__ void __launch_bounds__(32 * (2 * kMaxG + 1), 1)
    k_attn(DevCtx c, const __grid_constant__ CUtensorMap ring_map, uint32_t G, uint32_t stages) {
    using A = Attn<T, HD, QG>;
    constexpr int DPL = A::DPL;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t tile_elems = kTile * G * HD;
    T *tiles = reinterpret_cast<T *>(smem);                                  // [stages][K|V][32][G][HD]
    float *xchg = reinterpret_cast<float *>(tiles + size_t(stages) * 2 * tile_elems); // pair merge
    uint64_t *full = reinterpret_cast<uint64_t *>(xchg + kMaxG * 32 * QG * (2 + DPL));
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
            mbar_init(&empty[s], 2 * G);
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

    if (warp == 2 * kMaxG) { // ---------------- producer: TMA tile loads ----------------
        if (lane != 0)
            return;
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ring_map)) : "memory");
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
                // 16-row halves with no live row (window edges) are not loaded
                const bool h0 = tk < w && tk + kHalf > lo, h1 = tk + kHalf < w && tk + kTile > lo;
                T *kt = tiles + size_t(s) * 2 * tile_elems;
                mbar_expect_tx(&full[s], (uint32_t(h0) + uint32_t(h1)) * (bytes / 2));
                for (int hf = 0; hf < 2; ++hf) {
                    if (!(hf ? h1 : h0))
                        continue;
                    const int row0 = int((tk + hf * kHalf) % c.R);
                    T *dst = kt + size_t(hf) * kHalf * G * HD;
                    tma_load_4d(dst, &ring_map, 0, int(hg * G), row0, int(slot * c.L + l), &full[s]);
                    tma_load_4d(dst + tile_elems, &ring_map, 0, int(c.Hkv + hg * G), row0,
                                int(slot * c.L + l), &full[s]);
                }
                if (++s == stages) {
                    s = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }
    const uint32_t head_local = uint32_t(warp) >> 1, half = uint32_t(warp) & 1u;
    if (head_local >= G)
        return;

    // ---------- consumers: warp pair (2h, 2h+1) owns kv head hg*G + h; each takes 16 rows ----------
    const float scale_log2 = 1.4426950408889634f / sqrtf(float(HD));
    float *mine = xchg + size_t(head_local) * 32 * QG * (2 + DPL);
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
        at.init(c.q + ((uint64_t(slot) * c.L + l) * c.Hq + uint64_t(kvh) * QG) * HD);
        // far summaries: rows straight from global memory
        const T *far_base = reinterpret_cast<const T *>(c.far) +
                            (uint64_t(slot) * c.L + l) * c.max_chunks * c.row_elems + uint64_t(kvh) * HD;
        for (uint32_t f0 = half * kHalf; f0 < st.far_count; f0 += 2 * kHalf) {
            const uint32_t n = min(uint32_t(kHalf), st.far_count - f0);
            const uint32_t mask = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
            const uint32_t *ids = far_ids + st.far_begin + f0;
            auto far_row = [&](int r) {
                return far_base + uint64_t(ids[r < int(n) ? r : 0]) * c.row_elems;
            };
            if (mask == 0xffffu)
                at.template block<true>(far_row, c.d_kv, mask, scale_log2);
            else
                at.template block<false>(far_row, c.d_kv, mask, scale_log2);
        }
        // near window tiles from the TMA pipeline
        for (uint32_t k = 0; k < n_tiles; ++k) {
            mbar_wait(&full[s], phase);
            const T *kt = tiles + size_t(s) * 2 * tile_elems;
            const uint64_t tok0 = t0 + uint64_t(k) * kTile + half * kHalf;
            uint32_t mask = 0;
#pragma unroll
            for (int r = 0; r < kHalf; ++r)
                mask |= uint32_t(tok0 + r >= lo && tok0 + r < w) << r;
            const T *base = kt + (size_t(half) * kHalf * G + head_local) * HD;
            auto tile_row = [&](int r) { return base + size_t(r) * G * HD; };
            if (mask == 0xffffu)
                at.template block<true>(tile_row, tile_elems, mask, scale_log2);
            else if (mask) // a fully masked half was not even loaded
                at.template block<false>(tile_row, tile_elems, mask, scale_log2);
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&empty[s]);
            if (++s == stages) {
                s = 0;
                phase ^= 1;
            }
        }
        // merge the pair's states, then normalise
        const uint32_t bar = 1 + head_local;
        if (half) {
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                mine[(g * (2 + DPL) + 0) * 32 + lane] = at.m[g];
                mine[(g * (2 + DPL) + 1) * 32 + lane] = at.lsum[g];
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    mine[(g * (2 + DPL) + 2 + i) * 32 + lane] = at.acc[g][i];
            }
        }
        asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
        if (!half) {
            float *o = c.out + ((uint64_t(slot) * c.L + l) * c.Hq + uint64_t(kvh) * QG) * HD;
#pragma unroll
            for (int g = 0; g < QG; ++g) {
                const float m1 = mine[(g * (2 + DPL) + 0) * 32 + lane];
                const float l1 = mine[(g * (2 + DPL) + 1) * 32 + lane];
                const float mn = fmaxf(at.m[g], m1);
                const float a0 = mn == -INFINITY ? 0.f : exp2f(at.m[g] - mn);
                const float a1 = mn == -INFINITY ? 0.f : exp2f(m1 - mn);
                const float z = warp_sum(at.lsum[g] * a0 + l1 * a1);
                const float inv = z > 0.f ? 1.f / z : 0.f;
#pragma unroll
                for (int i = 0; i < DPL; ++i)
                    o[g * HD + DPL * lane + i] =
                        (at.acc[g][i] * a0 + mine[(g * (2 + DPL) + 2 + i) * 32 + lane] * a1) * inv;
            }
        }
        asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
    }
}


using AttnFn = void (*)(DevCtx, const CUtensorMap, uint32_t, uint32_t);

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
    CUtensorMap map{};
    TcMaps tc_maps{};      // tensor-core kernel descriptors
    uint32_t G = 1, stages = 2, grid = 1;
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
    p->smem = p->stages * stage + size_t(kMaxG) * 32 * c.group * (2 + c.hd / 32) * 4 +
              2 * p->stages * 8 + 16;
    p->grid = uint32_t(sms);
    cudaFuncSetAttribute(p->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem));

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
    const cuuint64_t strides[3] = {row, 2ull * c.Hkv * row, uint64_t(c.R) * 2 * c.Hkv * row};
    const cuuint32_t box[4] = {c.hd, p->G, uint32_t(kHalf), 1}; // 16-row halves
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt =
        c.esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    const CUresult r = encode(&p->map, dt, 4, c.ring, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        delete p;
        return nullptr;
    }
    std::snprintf(p->name, sizeof(p->name), "k_attn<%s,hd%u,g%u> G=%u stages=%u",
                  c.elem_kind == KVR_ELEM_F16 ? "f16" : c.elem_kind == KVR_ELEM_BF16 ? "bf16" : "f32",
                  c.hd, c.group, p->G, p->stages);
    (void)device;
    return p;
}

void launch_attn(const AttnPlan *p, const DevCtx &c, cudaStream_t s) {
    if (p->tc) {
        launch_attn_tc(p->tc, c, p->tc_maps, p->grid, s);
        return;
    }
    p->fn<<<p->grid, 32 * (2 * kMaxG + 1), p->smem, s>>>(c, p->map, p->G, p->stages);
}

void free_attn_plan(AttnPlan *p) { delete p; }
const char *attn_variant(const AttnPlan *p) { return p ? p->name : "none"; }

} // namespace kvr
