// Microbenchmark: packed FP32 FMA (fma.rn.f32x2, SASS FFMA2, __ffma2_rn) against scalar FFMA on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_rate scripts/microbench/ffma2_rate.cu
// (1) register-only chains: FMA per clock per SM of FFMA and of FFMA2 (packed pair x broadcast scalar);
// (2) a conv2-forward-shaped loop (10 maps x 4 conv positions x 9 taps per input map, weights as
//     warp-uniform vector loads, a 4x4 patch of scalar loads from shared memory): scalar vs packed.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_chain(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
    const float b = 1.0001f, c = 0.9999f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.f) out[0] = s;
}

__global__ void ffma2_chain(float* out, int iters) {
    float2 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 0.001f + i, threadIdx.x * 0.002f + i);
    const float b = 1.0001f + threadIdx.x * 1e-9f;
    const float2 c = make_float2(0.9999f, 0.9998f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], make_float2(b, b), c);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
    if (s == 12345.f) out[0] = s;
}

template <bool PACK>
__global__ void conv_like(float* out, int iters, int C) {
    extern __shared__ float sm[];
    for (int i = threadIdx.x; i < 4096 + 20 * 540 + 64; i += blockDim.x) sm[i] = 1e-3f * (i % 97);
    __syncthreads();
    float acc[10][4];
#pragma unroll
    for (int a = 0; a < 10; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = 0.f;
    const int p = threadIdx.x % 25, mg = (threadIdx.x / 25) % 6;
    const float* ib = sm + (p / 5) * 26 + (p % 5) * 2;
    const float* wb = sm + 4096 + mg * 10;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int n = 0; n < C; ++n) {
            float patch[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) patch[u][v] = ib[n * 169 + u * 13 + v];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    float wv[10];
                    const float* pw = wb + n * 540 + (i * 3 + j) * 60;
#pragma unroll
                    for (int q = 0; q < 5; ++q) {
                        const float2 t = *reinterpret_cast<const float2*>(pw + 2 * q);
                        wv[2 * q] = t.x;
                        wv[2 * q + 1] = t.y;
                    }
                    if constexpr (PACK) {
#pragma unroll
                        for (int a = 0; a < 10; a += 2)
#pragma unroll
                            for (int u = 0; u < 2; ++u)
#pragma unroll
                                for (int v = 0; v < 2; ++v) {
                                    const float pv = patch[u + i][v + j];
                                    const float2 r = __ffma2_rn(make_float2(wv[a], wv[a + 1]), make_float2(pv, pv),
                                                                make_float2(acc[a][u * 2 + v], acc[a + 1][u * 2 + v]));
                                    acc[a][u * 2 + v] = r.x;
                                    acc[a + 1][u * 2 + v] = r.y;
                                }
                    } else {
#pragma unroll
                        for (int a = 0; a < 10; ++a)
#pragma unroll
                            for (int u = 0; u < 2; ++u)
#pragma unroll
                                for (int v = 0; v < 2; ++v)
                                    acc[a][u * 2 + v] = fmaf(wv[a], patch[u + i][v + j], acc[a][u * 2 + v]);
                    }
                }
        }
    }
    float s = 0;
#pragma unroll
    for (int a = 0; a < 10; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) s += acc[a][q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
double timed(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch(2);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch(200);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 1e3;
}

int main() {
    float* out;
    cudaMalloc(&out, 4 * 148 * 1024);
    int sms, khz;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double clk = khz * 1e3;
    for (int threads : {256, 640, 1024}) {
        const double t1 = timed([&](int it) { ffma_chain<<<sms, threads>>>(out, it * 50); });
        const double t2 = timed([&](int it) { ffma2_chain<<<sms, threads>>>(out, it * 50); });
        const double fma = 200.0 * 50 * 8 * 16 * threads;
        printf("chains, %4d threads/SM: FFMA %.1f FMA/clk/SM (%.1f TFLOP/s), FFMA2 %.1f FMA/clk/SM (%.1f TFLOP/s)\n", threads,
               fma / t1 / clk, 2 * fma * sms / t1 / 1e12, fma / t2 / clk, 2 * fma * sms / t2 / 1e12);
    }
    const int smem = (4096 + 20 * 540 + 64) * 4;
    cudaFuncSetAttribute(conv_like<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(conv_like<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int threads : {320, 640}) {
        const double t1 = timed([&](int it) { conv_like<false><<<sms, threads, smem>>>(out, it, 20); });
        const double t2 = timed([&](int it) { conv_like<true><<<sms, threads, smem>>>(out, it, 20); });
        const double fma = 200.0 * 20 * 360 * threads;
        printf("conv2-like, %4d threads/SM: scalar %.1f FMA/clk/SM, packed %.1f FMA/clk/SM\n", threads, fma / t1 / clk,
               fma / t2 / clk);
    }
    return 0;
}
