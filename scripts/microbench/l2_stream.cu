// Microbenchmark (N-4): per-SM L2 -> SM bandwidth when every SM streams the SAME L2-resident
// buffer (the FC1 weight pattern: 240 KB read by all 148 CTAs), TMA bulk copies into shared
// memory (various chunk sizes, 2 in flight) vs LDG.128 by all threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2s scripts/microbench/l2_stream.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_stream(const float* src, int floats, int chunk, int reps, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    float* buf = reinterpret_cast<float*>(sm + 128);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t ph[2] = {0, 0};
    float acc = 0.f;
    const int nch = floats / chunk;
    for (int r = 0; r < reps; ++r) {
        for (int c = 0; c < nch; ++c) {
            const int b = c & 1;
            if (threadIdx.x == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar + b)), "r"(chunk * 4));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(buf + b * chunk)),
                    "l"(src + (size_t)c * chunk), "r"(chunk * 4), "r"(sa(bar + b)));
            }
            if (c >= 1) {  // consume the previous chunk (2 in flight)
                const int pb = (c - 1) & 1;
                uint32_t done = 0;
                do {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"(sa(bar + pb)), "r"(ph[pb]));
                } while (!done);
                ph[pb] ^= 1;
                acc += buf[pb * chunk + threadIdx.x];
                __syncthreads();
            }
        }
        const int pb = (nch - 1) & 1;
        uint32_t done = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(sa(bar + pb)), "r"(ph[pb]));
        } while (!done);
        ph[pb] ^= 1;
        acc += buf[pb * chunk + threadIdx.x];
        __syncthreads();
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void ldg_stream(const float4* src, int f4, int reps, float* out) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = 0; r < reps; ++r)
        for (int i = threadIdx.x; i < f4; i += blockDim.x) {
            const float4 v = __ldcg(src + i);
            acc.x += v.x;
            acc.y += v.y;
        }
    if (acc.x == 1234.5f) out[0] = acc.x + acc.y;
}

int main() {
    const int floats = 60000;  // FC1 weights
    float *src, *out;
    cudaMalloc(&src, floats * 4);
    cudaMemset(src, 0, floats * 4);
    cudaMalloc(&out, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 200;
    for (int chunk : {1000, 2000, 4000, 6000, 12000}) {
        const int smem = 128 + 2 * chunk * 4;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_stream<<<sms, 512, smem>>>(src, floats, chunk, 2, out);
        cudaEventRecord(e0);
        tma_stream<<<sms, 512, smem>>>(src, floats, chunk, reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes_per_sm = (double)(floats / chunk) * chunk * 4 * reps;
        printf("TMA bulk chunk %6d B: %.1f GB/s per SM, %.1f B/clk @1.965GHz, aggregate %.0f GB/s  (%s)\n", chunk * 4,
               bytes_per_sm / (ms * 1e-3) / 1e9, bytes_per_sm / (ms * 1e-3) / 1.965e9, bytes_per_sm * sms / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int threads : {256, 512, 1024}) {
        ldg_stream<<<sms, threads>>>((const float4*)src, floats / 4, 2, out);
        cudaEventRecord(e0);
        ldg_stream<<<sms, threads>>>((const float4*)src, floats / 4, reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes_per_sm = (double)floats * 4 * reps;
        printf("LDG.128 %4d thr: %.1f GB/s per SM, %.1f B/clk, aggregate %.0f GB/s\n", threads,
               bytes_per_sm / (ms * 1e-3) / 1e9, bytes_per_sm / (ms * 1e-3) / 1.965e9, bytes_per_sm * sms / (ms * 1e-3) / 1e9);
    }
    return 0;
}
