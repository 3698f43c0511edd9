// kvrail-b200 K-scan: stage() + reduce() on the device (one CTA).
//
// Reproduces transport.cpp:29-127 bit-for-bit for inputs without (kind,
// offset) ties (the reference's unstable std::sort leaves tie order
// unspecified; here ties keep stage order and raise status bit 1):
//   1. stage: per need, order its spans by (byte offset, length) and fuse
//      exact abutment into descriptors (one thread per need);
//   2. order descriptors by (kind, offset) with a shared-memory bitonic sort;
//   3. run-length scan: warp ballots mark run heads (kind change or byte gap),
//      warp-shuffle prefix sums number them, and each run is split greedily at
//      tau / the age guard by one thread (the split is inherently sequential
//      within a run, parallel across runs);
//   4. emit descriptors and trains in train order plus the span list K-gather
//      walks (with token prefix sums).
#include <cstdlib>

#include "kvr_internal.cuh"

namespace kvr {

namespace {

constexpr int kMaxNeeds = KVR_MAX_SCAN_NEEDS;

// Exclusive block-wide scan of one value per thread; returns the block total.
__device__ uint64_t block_exclusive_scan(uint64_t v, uint64_t &excl, uint64_t *warp_tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t t = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o)
                t += y;
        }
        warp_tot[lane] = t; // inclusive prefix of warp totals
    }
    __syncthreads();
    const uint64_t before = wid ? warp_tot[wid - 1] : 0;
    excl = before + x - v;
    const uint64_t total = warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
    return total;
}

struct ScanSmem {
    uint64_t warp_tot[32];
    kvr_need_rec need[kMaxNeeds]; // the step's needs, staged once (no dependent global loads)
    uint32_t need_m[kMaxNeeds];   // non-empty spans per need
    uint32_t need_d[kMaxNeeds];   // descriptors per need
    uint32_t need_base[kMaxNeeds];
};

template <int kScanThreads> __global__ void __launch_bounds__(kScanThreads, 1) k_scan(DevCtx c) {
    extern __shared__ __align__(16) uint8_t dyn[];
    __shared__ ScanSmem sm;
    __shared__ uint32_t s_status;
    pdl_wait();
    pdl_trigger();
    TlScope tl_(c, kTlScan);
    const kvr_step_header *h = hdr(c);
    const kvr_need_rec *g_needs = section<kvr_need_rec>(c, h->off_need);
    const kvr_span_rec *spans = section<kvr_span_rec>(c, h->off_span);
    const kvr_need_rec *needs = sm.need;
    const uint32_t cap = c.max_scan;
    // dynamic smem: cap entries per array
    uint64_t *d_off = reinterpret_cast<uint64_t *>(dyn);
    uint64_t *d_len = d_off + cap;
    uint64_t *key = d_len + cap;                              // bitonic sort keys
    uint32_t *sidx = reinterpret_cast<uint32_t *>(key + cap); // spans sorted within each need
    uint32_t *d_need = sidx + cap;                            // descriptor -> need
    uint32_t *d_first = d_need + cap;                         // first sidx position
    uint32_t *d_nsp = d_first + cap;                          // spans fused into it
    uint32_t *order = d_nsp + cap;                            // train order -> descriptor
    uint32_t *run_of = order + cap;                           // head position -> run index
    uint32_t *run_start = run_of + cap;
    uint32_t *run_cnt = run_start + cap;                      // trains per run -> train base
    uint64_t *sp_b = reinterpret_cast<uint64_t *>(run_cnt + cap); // span byte offset (staged once)
    uint64_t *sp_l = sp_b + cap;                                  // span bytes (0: empty span)
    uint64_t *sp_first = sp_l + cap;                              // span's first logical token

    const uint32_t n_need = h->n_need;
    if (threadIdx.x == 0)
        s_status = (n_need > kMaxNeeds || h->n_span > cap) ? 4u : 0u;
    __syncthreads();
    const uint64_t tb = c.token_bytes, page = c.page_bytes;
    // every span's byte range staged in shared memory by all threads at once: the
    // per-need insertion sort below then compares in shared memory instead of
    // chasing dependent global loads
    if (!s_status) {
        for (uint32_t i = threadIdx.x; i < h->n_span; i += blockDim.x) {
            const kvr_span_rec sp = spans[i];
            sp_b[i] = uint64_t(sp.block) * page + uint64_t(sp.slot_begin) * tb;
            sp_l[i] = uint64_t(sp.slot_count) * tb;
            sp_first[i] = sp.first_token;
        }
        for (uint32_t i = threadIdx.x; i < n_need; i += blockDim.x)
            sm.need[i] = g_needs[i];
    }
    __syncthreads();

    // ---- 1. stage: per-need insertion sort by (offset, length) + fusion ----
    uint32_t n_desc = 0;
    if (!s_status) {
        for (uint32_t i = threadIdx.x; i < n_need; i += blockDim.x) {
            const kvr_need_rec nd = needs[i];
            uint32_t *ord = sidx + nd.span_begin;
            uint32_t m = 0, dcount = 0;
            for (uint32_t k = 0; k < nd.span_count; ++k) {
                const uint64_t b = sp_b[nd.span_begin + k], len = sp_l[nd.span_begin + k];
                if (len == 0)
                    continue;
                uint32_t at = m++;
                while (at > 0) {
                    const uint64_t ob = sp_b[ord[at - 1]], ol = sp_l[ord[at - 1]];
                    if (ob < b || (ob == b && ol <= len))
                        break;
                    ord[at] = ord[at - 1];
                    --at;
                }
                ord[at] = nd.span_begin + k;
            }
            uint64_t end = 0;
            for (uint32_t k = 0; k < m; ++k) {
                if (k == 0 || sp_b[ord[k]] != end)
                    ++dcount;
                end = sp_b[ord[k]] + sp_l[ord[k]];
            }
            sm.need_m[i] = m;
            sm.need_d[i] = dcount;
        }
        __syncthreads();
        uint64_t carry = 0;
        for (uint32_t base = 0; base < n_need; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            uint64_t excl;
            const uint64_t tot = block_exclusive_scan(i < n_need ? sm.need_d[i] : 0, excl, sm.warp_tot);
            if (i < n_need)
                sm.need_base[i] = uint32_t(carry + excl);
            carry += tot;
        }
        n_desc = uint32_t(carry);
        if (n_desc > cap && threadIdx.x == 0)
            s_status |= 4u;
        __syncthreads();
        if (!s_status) {
            for (uint32_t i = threadIdx.x; i < n_need; i += blockDim.x) {
                const uint32_t first = needs[i].span_begin;
                uint32_t d = sm.need_base[i] - 1;
                uint64_t end = 0;
                for (uint32_t k = 0; k < sm.need_m[i]; ++k) {
                    const uint64_t b = sp_b[sidx[first + k]], len = sp_l[sidx[first + k]];
                    if (k == 0 || b != end) {
                        ++d;
                        d_off[d] = b;
                        d_len[d] = 0;
                        d_need[d] = i;
                        d_first[d] = first + k;
                        d_nsp[d] = 0;
                    }
                    d_len[d] += len;
                    d_nsp[d] += 1;
                    end = b + len;
                }
            }
        }
        __syncthreads();
    }
    if (s_status)
        n_desc = 0;

    // ---- 2. order by (kind, offset); stage order breaks ties ----
    const bool merge = h->merge != 0;
    uint32_t pow2 = 1;
    while (pow2 < n_desc)
        pow2 <<= 1;
    if (merge && n_desc > 1) {
        // key = kind (bit 63) | byte offset (47 bits: arena < 128 TiB, checked at
        // kvr_dev_open) | stage index (16 bits: descriptors <= max_scan_descs <= 2048)
        for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x)
            key[i] = i < n_desc ? (uint64_t(needs[d_need[i]].kind & 1u) << 63) | (d_off[i] << 16) | i
                                : ~0ull;
        __syncthreads();
        for (uint32_t k = 2; k <= pow2; k <<= 1)
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x) {
                    const uint32_t p = i ^ j;
                    if (p > i) {
                        const bool up = (i & k) == 0;
                        const uint64_t a = key[i], b = key[p];
                        if ((a > b) == up) {
                            key[i] = b;
                            key[p] = a;
                        }
                    }
                }
                __syncthreads();
            }
        for (uint32_t i = threadIdx.x; i < n_desc; i += blockDim.x)
            order[i] = uint32_t(key[i] & 0xffffu);
    } else {
        for (uint32_t i = threadIdx.x; i < n_desc; i += blockDim.x)
            order[i] = i;
    }
    __syncthreads();

    // ---- 3. run-length scan: ballot run heads, shuffle-scan their ranks ----
    // The age rule (transport.cpp:101-110) closes a train when now - oldest_stage_time
    // >= max_hold. K-scan fuses stage() with reduce(): stage() stamps every descriptor
    // with stage_time = now (transport.cpp:29-61), so each train's oldest stage time
    // IS now and the rule reduces exactly to 0 >= max_hold — the same for every train.
    const double now = h->now;
    const bool age_close = (now - now) >= h->max_hold;
    const uint64_t tau = h->tau;
    const uint64_t run_page = h->run_page, run_span = h->run_span;
    auto adjacent = [&](uint64_t end, uint64_t next) { // transport.hpp abuts()
        return end == next || (run_page && end % run_page == run_span && next == end - run_span + run_page);
    };
    auto is_head = [&](uint32_t i) {
        if (i == 0 || !merge)
            return true;
        const uint32_t a = order[i - 1], b = order[i];
        return !(needs[d_need[a]].kind == needs[d_need[b]].kind && adjacent(d_off[a] + d_len[a], d_off[b]));
    };
    uint32_t n_runs;
    {
        uint64_t carry = 0;
        const uint32_t lane = threadIdx.x & 31;
        for (uint32_t base = 0; base < n_desc; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            const bool head = i < n_desc && is_head(i);
            if (i < n_desc && i > 0 && merge) {
                const uint32_t a = order[i - 1], b = order[i];
                if (needs[d_need[a]].kind == needs[d_need[b]].kind && d_off[a] == d_off[b])
                    atomicOr(&s_status, 2u); // (kind, offset) tie
            }
            const uint32_t ballot = __ballot_sync(0xffffffffu, head);
            uint64_t excl;
            const uint64_t tot = block_exclusive_scan(lane == 0 ? __popc(ballot) : 0, excl, sm.warp_tot);
            const uint64_t warp_base = __shfl_sync(0xffffffffu, excl, 0);
            if (head) {
                const uint32_t r = uint32_t(carry + warp_base + __popc(ballot & ((1u << lane) - 1u)));
                run_of[i] = r;
                run_start[r] = i;
            }
            carry += tot;
        }
        n_runs = uint32_t(carry);
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < n_runs; r += blockDim.x) {
        const uint32_t lo = run_start[r], hi = r + 1 < n_runs ? run_start[r + 1] : n_desc;
        uint32_t cnt = 1;
        uint64_t bytes = 0;
        for (uint32_t i = lo; i < hi; ++i) {
            if (i > lo && (!merge || bytes >= tau || age_close)) {
                ++cnt;
                bytes = 0;
            }
            bytes += d_len[order[i]];
        }
        run_cnt[r] = cnt;
    }
    __syncthreads();
    uint32_t n_trains;
    {
        uint64_t carry = 0;
        for (uint32_t base = 0; base < n_runs; base += blockDim.x) {
            const uint32_t r = base + threadIdx.x;
            const uint32_t cnt = r < n_runs ? run_cnt[r] : 0;
            uint64_t excl;
            const uint64_t tot = block_exclusive_scan(cnt, excl, sm.warp_tot);
            if (r < n_runs)
                run_cnt[r] = uint32_t(carry + excl);
            carry += tot;
        }
        n_trains = uint32_t(carry);
    }
    if (n_trains > c.max_trains) {
        if (threadIdx.x == 0)
            s_status |= 4u;
        n_trains = 0;
        n_runs = 0;
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < n_runs; r += blockDim.x) {
        const uint32_t lo = run_start[r], hi = r + 1 < n_runs ? run_start[r + 1] : n_desc;
        const bool last_run = r + 1 == n_runs;
        uint32_t t = run_cnt[r];
        kvr_train cur{};
        auto emit = [&](uint32_t why) {
            cur.reason = why;
            cur.issue_time = now;
            cur.oldest_stage_time = now;
            c.trains[t++] = cur;
            cur = kvr_train{};
        };
        for (uint32_t i = lo; i < hi; ++i) {
            const uint32_t d = order[i];
            if (i > lo) { // close test before the append: threshold, age, (adjacent here)
                if (!merge)
                    emit(2);
                else if (cur.total_bytes >= tau)
                    emit(0);
                else if (age_close)
                    emit(1);
            }
            if (cur.desc_count == 0) {
                cur.kind = needs[d_need[d]].kind;
                cur.desc_begin = i;
            }
            cur.total_bytes += d_len[d];
            cur.desc_count += 1;
        }
        if (hi > lo) { // run boundary / step residue
            if (merge && cur.total_bytes >= tau)
                emit(0);
            else if (merge && !last_run && age_close)
                emit(1);
            else
                emit(2);
        }
    }
    __syncthreads();

    // ---- 4. descriptors and gather spans in train order ----
    const bool ok = !(s_status & 4u);
    uint64_t carry_s = 0, carry_t = 0;
    for (uint32_t base = 0; base < n_desc; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool on = ok && i < n_desc;
        const uint32_t d = on ? order[i] : 0;
        uint64_t sx, tx;
        const uint64_t ts = block_exclusive_scan(on ? d_nsp[d] : 0, sx, sm.warp_tot);
        const uint64_t tt = block_exclusive_scan(on ? d_len[d] / tb : 0, tx, sm.warp_tot);
        if (on) {
            const kvr_need_rec nd = needs[d_need[d]];
            kvr_descriptor o{};
            o.phys_offset = d_off[d];
            o.length = d_len[d];
            o.stage_time = now;
            o.kind = nd.kind;
            o.block = uint32_t(d_off[d] / page);
            o.session = nd.session;
            c.descs[i] = o;
            uint64_t g = carry_s + sx, tok = carry_t + tx;
            for (uint32_t k = 0; k < d_nsp[d]; ++k) {
                const uint32_t si = sidx[d_first[d] + k];
                const uint64_t b = sp_b[si];
                GSpan gs;
                gs.first_token = sp_first[si];
                gs.tok_prefix = tok;
                gs.block = uint32_t(b / page);
                gs.slot_begin = uint32_t((b % page) / tb);
                gs.slot_count = uint32_t(sp_l[si] / tb);
                gs.dev_slot = nd.slot;
                gs.kind = nd.kind;
                gs.pad = 0;
                c.gspans[g++] = gs;
                tok += gs.slot_count;
            }
        }
        carry_s += ts;
        carry_t += tt;
    }
    if (threadIdx.x == 0) {
        uint64_t bytes = 0;
        for (uint32_t i = 0; ok && i < n_desc; ++i)
            bytes += d_len[order[i]];
        c.scan->trains = ok ? n_trains : 0;
        c.scan->descriptors = ok ? n_desc : 0;
        c.scan->spans = ok ? uint32_t(carry_s) : 0;
        c.scan->status = s_status;
        c.scan->total_tokens = ok ? carry_t : 0;
        c.scan->train_bytes = bytes;
        c.scan->attn_t0 = ~0ull; // K-attn and K-gather (after the join) stamp their spans
        c.scan->attn_t1 = 0;
        c.scan->gather_t0 = ~0ull;
        c.scan->gather_t1 = 0;
    }
}

} // namespace

size_t scan_dynamic_smem(uint32_t cap) { return size_t(cap) * (6 * 8 + 8 * 4); }

namespace {
int scan_threads() {
    static const int t = [] {
        const char *e = getenv("KVR_SCAN_THREADS");
        const int v = e ? atoi(e) : 256;
        return v == 128 || v == 512 || v == 1024 ? v : 256;
    }();
    return t;
}
} // namespace

void launch_scan(const DevCtx &c, cudaStream_t s, bool pdl) {
    const size_t smem = scan_dynamic_smem(c.max_scan);
    switch (scan_threads()) {
    case 128: launch_ex(k_scan<128>, 1, 128, smem, s, pdl, c); break;
    case 512: launch_ex(k_scan<512>, 1, 512, smem, s, pdl, c); break;
    case 1024: launch_ex(k_scan<1024>, 1, 1024, smem, s, pdl, c); break;
    default: launch_ex(k_scan<256>, 1, 256, smem, s, pdl, c); break;
    }
}

cudaError_t prepare_scan(uint32_t cap) {
    const int smem = int(scan_dynamic_smem(cap));
    cudaError_t e = cudaFuncSetAttribute(k_scan<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_scan<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_scan<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_scan<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return e;
}

} // namespace kvr
