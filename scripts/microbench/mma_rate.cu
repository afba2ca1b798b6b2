// Microbenchmark (N-4): FFMA vs legacy mma.sync (tf32 m16n8k8, bf16 m16n8k16) issue rates on one B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate scripts/microbench/mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    const float b = 1.0001f, c = 0.9999f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.f) out[0] = s;
}

__global__ void tf32_kernel(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float d[4][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int t = 0; t < 4; ++t)
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(d[t][0]), "+f"(d[t][1]), "+f"(d[t][2]), "+f"(d[t][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int t = 0; t < 4; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    if (s == 12345.f) out[0] = s;
}

__global__ void bf16_kernel(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float d[4][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int t = 0; t < 4; ++t)
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(d[t][0]), "+f"(d[t][1]), "+f"(d[t][2]), "+f"(d[t][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int t = 0; t < 4; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    if (s == 12345.f) out[0] = s;
}

template <class F>
double run(F k, int blocks, int threads, int iters, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 1e3;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int threads : {128, 256, 512, 1024}) {
        double t = run(ffma_kernel, sms, threads, iters, out);
        double flop = 2.0 * sms * threads * iters * 16.0 * 8;
        double t2 = run(tf32_kernel, sms, threads, iters / 4, out);
        double f2 = 2.0 * sms * (threads / 32) * (iters / 4) * 16.0 * (16 * 8 * 8);
        double t3 = run(bf16_kernel, sms, threads, iters / 4, out);
        double f3 = 2.0 * sms * (threads / 32) * (iters / 4) * 16.0 * (16 * 8 * 16);
        printf("threads/SM %4d  FFMA %.1f TFLOP/s   mma.sync tf32 %.1f TFLOP/s   mma.sync bf16 %.1f TFLOP/s\n", threads,
               flop / t / 1e12, f2 / t2 / 1e12, f3 / t3 / 1e12);
    }
    return 0;
}
