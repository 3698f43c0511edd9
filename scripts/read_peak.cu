// Read-stream ceiling of this B200's HBM: the best rate a kernel that only READS
// (like K-attn) can reach, for context next to MEASURED_PEAKS.json's copy
// (read + write) figure. Two variants over a buffer far larger than L2:
//   ldg  — 16-byte vector loads, 8 in flight per thread, grid = 4 x #SMs x 512 threads
//   tma  — cp.async.bulk global->shared, 4 x 48 KiB stages per CTA, one CTA per SM
//   stg  — write stream: 16-byte streaming stores, same grid as ldg (the ceiling of the
//          cold prompt writers K-write / K-presum, which only write)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_peak scripts/read_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) ldg(const int4 *__restrict__ p, size_t n, int *sink) {
    int acc = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            v[k] = __ldcs(p + i + k * stride);
#pragma unroll
        for (int k = 0; k < 8; ++k)
            acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    for (; i < n; i += stride) {
        const int4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x7fffffff)
        *sink = acc;
}

__global__ void __launch_bounds__(512) stg(int4 *__restrict__ p, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    const int4 v = make_int4(int(threadIdx.x), int(blockIdx.x), 1, 2);
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        __stcs(p + i, v);
}

constexpr int kStages = 4;
constexpr uint32_t kChunk = 48u << 10;

__device__ inline uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32) tma(const uint8_t *p, size_t bytes, int *sink) {
    extern __shared__ __align__(128) uint8_t buf[];
    __shared__ __align__(8) uint64_t full[kStages];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const size_t n_chunks = bytes / kChunk;
    uint32_t phase[kStages] = {0, 0, 0, 0};
    int acc = 0;
    size_t c = blockIdx.x;
    auto issue = [&](int s, size_t chunk) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kChunk)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(buf + size_t(s) * kChunk)),
                         "l"(p + chunk * kChunk), "r"(kChunk), "r"(su32(&full[s]))
                         : "memory");
        }
    };
    for (int s = 0; s < kStages; ++s)
        if (c + size_t(s) * gridDim.x < n_chunks)
            issue(s, c + size_t(s) * gridDim.x);
    for (size_t k = 0; c + k * gridDim.x < n_chunks; ++k) {
        const int s = int(k % kStages);
        asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                     "@!P bra W_%=;\n\t}" ::"r"(su32(&full[s])),
                     "r"(phase[s])
                     : "memory");
        phase[s] ^= 1;
        acc ^= reinterpret_cast<const int *>(buf + size_t(s) * kChunk)[threadIdx.x];
        __syncwarp();
        const size_t nxt = c + (k + kStages) * gridDim.x;
        if (nxt < n_chunks)
            issue(s, nxt);
    }
    if (acc == 0x7fffffff)
        *sink = acc;
}

int main() {
    const size_t bytes = size_t(16) << 30; // 16 GiB (C2 reads ~16 GiB per step)
    uint8_t *p;
    int *sink;
    if (cudaMalloc(&p, bytes) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) {
        std::printf("alloc failed\n");
        return 1;
    }
    cudaMemset(p, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int v = 0; v < 3; ++v) {
        float best = 1e30f;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(a);
            if (v == 0)
                ldg<<<4 * sms, 512>>>(reinterpret_cast<const int4 *>(p), bytes / 16, sink);
            else if (v == 2)
                stg<<<4 * sms, 512>>>(reinterpret_cast<int4 *>(p), bytes / 16);
            else
                tma<<<sms, 32, kStages * kChunk>>>(p, bytes, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best)
                best = ms;
        }
        std::printf("{\"variant\": \"%s\", \"bytes\": %zu, \"ms\": %.4f, \"%s\": %.1f}\n",
                    v == 0 ? "ldg" : v == 1 ? "tma" : "stg", bytes, best, v == 2 ? "write_gbs" : "read_gbs",
                    bytes / (best * 1e6));
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
