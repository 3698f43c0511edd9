// kvrail-b200 K-mass: attention-utility observations for the placement tracker.
//
// The reference feeds plan_step (placement.cpp:70-125) one synthetic observation
// per session per step (scenario.cpp:526-529; SPEC.md:190 calls the attention-
// utility observation a stand-in). With b200.utility = "attention" the step also
// measures it: for a probe layer, the softmax weight every q-head puts on each
// near-window row (far summaries take part in the normalisation, as in attend(),
// far_view.cpp:113-155), averaged over the q-heads and summed per arena block of
// the committed view. Output per slot: runs {block, mass} in window order.
//
//   k_mass_rows  grid (slot, split of 8 view rows), warp = kv head (a CTA reads
//                whole contiguous K rows): scores of the group's q-heads (lanes over
//                head dims) and each split's softmax (max, sum)
//   k_mass_runs  grid slot: per q-head softmax from the splits, per-row mean weight
//                over q-heads, rows folded into runs of equal block (device page
//                table), one thread per run: deterministic
//
// Cost: the probe layer's K rows once (1/(2L) of the attention's bytes) plus a
// score per (q-head, view row) of scratch; opt-in.
#include <algorithm>
#include <type_traits>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

constexpr int kMassThreads = 256;
constexpr int kMaxGroup = 16; // q-heads per kv head (checked at open)

constexpr int kBatch = 8; // rows a warp loads before it reduces (memory-level parallelism)
constexpr int kSplitRows = kBatch; // view rows per K-mass CTA (each warp: one kv head)

/// N consecutive elements of one row as floats (one vector load).
template <typename T, int N> __device__ inline void load_row(const T *p, float *o) {
    if constexpr (std::is_same_v<T, float>) {
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
        auto f = [](T x) {
            if constexpr (std::is_same_v<T, __half>)
                return __half2float(x);
            else
                return __bfloat162float(x);
        };
        if constexpr (N == 4) {
            const uint2 v = *reinterpret_cast<const uint2 *>(p);
            const T *e = reinterpret_cast<const T *>(&v);
            o[0] = f(e[0]), o[1] = f(e[1]), o[2] = f(e[2]), o[3] = f(e[3]);
        } else if constexpr (N == 2) {
            const uint32_t v = *reinterpret_cast<const uint32_t *>(p);
            const T *e = reinterpret_cast<const T *>(&v);
            o[0] = f(e[0]), o[1] = f(e[1]);
        } else {
            o[0] = f(*p);
        }
    }
}

template <typename T, int DPL>
__global__ void __launch_bounds__(1024) k_mass_rows(DevCtx c) {
    // CTA = (slot, split of kSplitRows view rows); warp w = kv head w (w, w + 32, ...),
    // so the warps of a CTA read whole contiguous K rows of the ring. Each warp: the
    // scores of its q-heads for the split's rows -> sc[slot][q head][view row], and
    // the split's (max, sum of exp) per q-head
    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t *far_ids = section<uint32_t>(c, h->off_far_ids);
    const uint32_t n_split = (c.W + c.far_cap + kSplitRows - 1) / kSplitRows;
    const uint32_t split = blockIdx.x % n_split, slot = blockIdx.x / n_split;
    const kvr_slot_state st = slots[slot];
    if (!st.live || h->step % c.utility) // (b200.utility_every: not measured this step)
        return;
    const uint64_t w = st.written, lo = w > c.W ? w - c.W : 0;
    const uint32_t n_far = st.far_count, n = n_far + uint32_t(w - lo);
    const uint32_t G = c.group, l = c.util_layer, Wf = c.W + c.far_cap;
    constexpr uint32_t HD = 32 * DPL;
    const int lane = threadIdx.x & 31;
    const float scale = rsqrtf(float(HD));
    const uint32_t i0 = split * kSplitRows;
    const uint32_t ring0 = uint32_t(lo % c.R); // ring row of view row n_far
    static_assert(kSplitRows == 8, "the butterfly below reduces 8 rows");
    for (uint32_t kvh = threadIdx.x >> 5; kvh < c.Hkv; kvh += blockDim.x >> 5) {
        const uint64_t q0 = ((uint64_t(slot) * c.L + l) * c.Hq + uint64_t(kvh) * G) * HD + DPL * lane;
        const T *ring = reinterpret_cast<const T *>(c.ring) + ring_row(c, slot, l, 0) + uint64_t(kvh) * HD + DPL * lane;
        const T *far = reinterpret_cast<const T *>(c.far) +
                       (uint64_t(slot) * c.L + l) * c.max_chunks * c.row_elems + uint64_t(kvh) * HD + DPL * lane;
        // view order of build_view (far_view.cpp:69-109): far summaries, then the near window
        float k[kSplitRows][DPL];
#pragma unroll
        for (int r = 0; r < kSplitRows; ++r) {
            const uint32_t i = i0 + r;
            if (i < n) {
                uint32_t rr = ring0 + (i - n_far);
                rr = rr >= c.R ? rr - c.R : rr;
                const T *row = i < n_far ? far + uint64_t(far_ids[st.far_begin + i]) * c.row_elems
                                         : ring + uint64_t(rr) * c.row_elems;
                load_row<T, DPL>(row, k[r]);
            } else {
#pragma unroll
                for (int d = 0; d < DPL; ++d)
                    k[r][d] = 0.f;
            }
        }
        for (uint32_t g = 0; g < G; ++g) {
            float part[kSplitRows];
#pragma unroll
            for (int r = 0; r < kSplitRows; ++r) {
                float a = 0.f;
#pragma unroll
                for (int d = 0; d < DPL; ++d)
                    a = fmaf(load_q(c, q0 + g * HD + d), k[r][d], a);
                part[r] = a;
            }
            // halving butterfly: lane ends with row lane >> 2 summed over 8 lanes, then
            // the last two lane bits
#pragma unroll
            for (int wd = kSplitRows / 2, bit = 16; wd >= 1; wd >>= 1, bit >>= 1) {
                const bool hi = lane & bit;
#pragma unroll
                for (int j = 0; j < wd; ++j) {
                    const float send = hi ? part[j] : part[j + wd];
                    const float keep = hi ? part[j + wd] : part[j];
                    part[j] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
                }
            }
            float v = part[0];
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            const uint32_t row = lane >> 2;
            const float sv = i0 + row < n ? v * scale : -INFINITY;
            float m = sv;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1)
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float e = m == -INFINITY ? 0.f : expf(sv - m);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1)
                e += __shfl_xor_sync(0xffffffffu, e, o);
            const uint64_t qh = uint64_t(slot) * c.Hq + uint64_t(kvh) * G + g;
            if ((lane & 3) == 0 && i0 + row < n)
                c.mass_sc[qh * Wf + i0 + row] = sv;
            if (lane == 0)
                c.mass_part[qh * n_split + split] = make_float2(m, e);
        }
    }
}

__global__ void __launch_bounds__(kMassThreads) k_mass_runs(DevCtx c) {
    // CTA = slot: per q-head softmax (max, 1/sum) from the split partials; per
    // window row the mean over q-heads of its weight; rows folded into block runs
    const kvr_step_header *h = hdr(c);
    const kvr_slot_state *slots = section<kvr_slot_state>(c, h->off_slots);
    const uint32_t slot = blockIdx.x;
    if (h->step % c.utility)
        return;
    const kvr_slot_state st = slots[slot];
    kvr_mass_run *runs = c.mass_runs + uint64_t(slot) * c.W;
    const uint64_t w = st.written, lo = w > c.W ? w - c.W : 0;
    const uint32_t n = st.live ? uint32_t(w - lo) : 0, n_far = st.live ? st.far_count : 0;
    const uint32_t n_split = (c.W + c.far_cap + kSplitRows - 1) / kSplitRows, Wf = c.W + c.far_cap;
    const uint32_t *tmap = c.tmap + uint64_t(slot) * c.max_tokens;
    extern __shared__ float tot[];                           // [W] row mass
    uint32_t *blk = reinterpret_cast<uint32_t *>(tot + c.W); // [W] row block
    float *hm = reinterpret_cast<float *>(blk + c.W);        // [Hq] max, [Hq] 1/sum
    float *hinv = hm + c.Hq;
    for (uint32_t qh = threadIdx.x; qh < c.Hq && n; qh += kMassThreads) {
        const float2 *p = c.mass_part + (uint64_t(slot) * c.Hq + qh) * n_split;
        float m = -INFINITY, e = 0.f;
        for (uint32_t j = 0; j < n_split; ++j)
            m = fmaxf(m, p[j].x);
        for (uint32_t j = 0; j < n_split; ++j)
            e += p[j].x == -INFINITY ? 0.f : p[j].y * expf(p[j].x - m);
        hm[qh] = m;
        hinv[qh] = e > 0.f ? 1.f / e : 0.f;
    }
    __syncthreads();
    const float inv_hq = 1.f / float(c.Hq);
    const float *scs = c.mass_sc + uint64_t(slot) * c.Hq * Wf + n_far;
    for (uint32_t i = threadIdx.x; i < n; i += kMassThreads) {
        float m = 0.f;
#pragma unroll 8
        for (uint32_t qh = 0; qh < c.Hq; ++qh)
            m += expf(scs[uint64_t(qh) * Wf + i] - hm[qh]) * hinv[qh];
        tot[i] = m * inv_hq;
        const uint32_t gs = tmap[lo + i];
        blk[i] = gs == kNoMap ? kNoMap : gs / c.tpp;
    }
    __shared__ uint32_t run_base, warp_runs[kMassThreads / 32];
    if (threadIdx.x == 0)
        run_base = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t i0 = 0; i0 < n; i0 += kMassThreads) {
        const uint32_t i = i0 + threadIdx.x;
        const uint32_t b = i < n ? blk[i] : kNoMap;
        const bool head = i < n && b != kNoMap && (i == 0 || blk[i - 1] != b);
        // block-wide exclusive scan of the run heads -> this run's index
        const uint32_t ballot = __ballot_sync(0xffffffffu, head);
        if (lane == 0)
            warp_runs[warp] = __popc(ballot);
        __syncthreads();
        uint32_t before = run_base;
        for (int j = 0; j < warp; ++j)
            before += warp_runs[j];
        before += __popc(ballot & ((1u << lane) - 1u));
        if (head) { // one thread per run sums it in window order: deterministic
            float m = 0.f;
            for (uint32_t r = i; r < n && blk[r] == b; ++r)
                m += tot[r];
            runs[before] = kvr_mass_run{b, m};
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int j = 0; j < kMassThreads / 32; ++j)
                run_base += warp_runs[j];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        c.mass_count[slot] = run_base;
}

using RowsFn = void (*)(DevCtx);
template <typename T> RowsFn pick_rows(uint32_t hd) {
    switch (hd) {
    case 32: return k_mass_rows<T, 1>;
    case 64: return k_mass_rows<T, 2>;
    case 128: return k_mass_rows<T, 4>;
    default: return nullptr;
    }
}
RowsFn rows_kernel(const DevCtx &c) {
    switch (c.elem_kind) {
    case KVR_ELEM_F16: return pick_rows<__half>(c.hd);
    case KVR_ELEM_BF16: return pick_rows<__nv_bfloat16>(c.hd);
    default: return pick_rows<float>(c.hd);
    }
}

} // namespace

static uint32_t n_splits(const DevCtx &c) { return (c.W + c.far_cap + kSplitRows - 1) / kSplitRows; }
static size_t runs_smem(const DevCtx &c) { return size_t(c.W) * 8 + size_t(c.Hq) * 8; }
size_t mass_scratch_floats(const DevCtx &c) { return size_t(c.n_slots) * c.Hq * (c.W + c.far_cap); }
size_t mass_part_entries(const DevCtx &c) { return size_t(c.n_slots) * c.Hq * n_splits(c); }
uint32_t mass_max_group() { return kMaxGroup; }

bool prepare_mass(const DevCtx &c) {
    if (!rows_kernel(c) || runs_smem(c) > (200u << 10))
        return false;
    return cudaFuncSetAttribute(k_mass_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, int(runs_smem(c))) ==
           cudaSuccess;
}

void launch_mass(const DevCtx &c, cudaStream_t s) {
    rows_kernel(c)<<<c.n_slots * n_splits(c), 32 * std::min(c.Hkv, 32u), 0, s>>>(c);
    k_mass_runs<<<c.n_slots, kMassThreads, runs_smem(c), s>>>(c);
}

} // namespace kvr
