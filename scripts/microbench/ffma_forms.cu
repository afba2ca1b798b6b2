// Microbenchmark (N-4): FFMA throughput by operand form on one B200 (full chip, 148 CTAs).
//   imm   : a = fma(a, 1.0001f, 0.9999f)          (immediate operands)
//   reg2  : a = fma(x, w, a), x and w registers reused across the 8 chains
//   reg3  : a_k = fma(x_k, w_k, a_k), all distinct registers (conv-like register tiling)
//   tile  : a[i][j] = fma(x[i], w[j], a[i][j]), 4x4 outer product (reuse-cache friendly)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma scripts/microbench/ffma_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_imm(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 1.0001f, 0.9999f);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.5f) out[0] = s;
}

__global__ void k_reg3(const float* in, float* out, int iters) {
    float a[8], x[8], w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = in[threadIdx.x + i];
        x[i] = in[threadIdx.x + 8 + i];
        w[i] = in[threadIdx.x + 16 + i];
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fmaf(x[i], w[(i + u) & 7], a[i]);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.5f) out[0] = s;
}

__global__ void k_tile(const float* in, float* out, int iters) {
    float a[4][4], x[4], w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        x[i] = in[threadIdx.x + i];
        w[i] = in[threadIdx.x + 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) a[i][j] = 0.f;
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) a[i][j] = fmaf(x[i], w[j], a[i][j]);
            x[u & 3] += 1e-7f;  // keep the compiler from folding iterations
        }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += a[i][j];
    if (s == 1.5f) out[0] = s;
}

int main() {
    float *in, *out;
    cudaMalloc(&in, 1 << 20);
    cudaMemset(in, 0, 1 << 20);
    cudaMalloc(&out, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int threads : {256, 512, 1024}) {
        float ms;
        k_imm<<<sms, threads>>>(out, 10);
        cudaEventRecord(e0);
        k_imm<<<sms, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double f1 = 2.0 * sms * threads * iters * 16 * 8 / (ms * 1e-3) / 1e12;
        k_reg3<<<sms, threads>>>(in, out, 10);
        cudaEventRecord(e0);
        k_reg3<<<sms, threads>>>(in, out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double f2 = 2.0 * sms * threads * iters * 16 * 8 / (ms * 1e-3) / 1e12;
        k_tile<<<sms, threads>>>(in, out, 10);
        cudaEventRecord(e0);
        k_tile<<<sms, threads>>>(in, out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double f3 = 2.0 * sms * threads * iters * 8 * 16 / (ms * 1e-3) / 1e12;
        printf("threads/SM %4d  FFMA imm %.1f  reg3 %.1f  4x4 tile %.1f TFLOP/s\n", threads, f1, f2, f3);
    }
    return 0;
}
