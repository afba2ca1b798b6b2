// Shared-memory load cost by access pattern (B200): cycles per warp-wide LDS when the LSU is saturated
// (148 CTAs x 640 threads, every warp issuing independent loads).  Patterns:
//   u32/u64/u128  : every lane the same address (warp-uniform)
//   g6_64 / g6_128: 6 distinct addresses per warp (lane % 6 picks a 10- / 12-float map group), the
//                   conv_fwd weight pattern with map groups fastest over the lanes
//   d64 / d128    : every lane its own consecutive vector (32 x 8 B / 32 x 16 B)
//   d32           : every lane its own word (one wavefront)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ldsw scripts/microbench/lds_wavefronts.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 640, ITERS = 4096, UNR = 8;

template <int PAT>
__global__ void __launch_bounds__(NT, 1) k(float* out, long long* cyc) {
    extern __shared__ float s[];
    for (int i = threadIdx.x; i < 16384; i += NT) s[i] = i * 1e-3f;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int off;
    if (PAT <= 2) off = 0;
    else if (PAT == 3) off = (lane % 6) * 10;
    else if (PAT == 4) off = (lane % 6) * 12;
    else if (PAT == 5) off = lane * 2;
    else if (PAT == 6) off = lane * 4;
    else off = lane;
    off += warp * 64;
    unsigned acc = 0u;
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
        const int b = ((it * 136) & 8191) + off;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const float* p = s + b + u * 256;
            if (PAT == 0 || PAT == 7) acc ^= __float_as_uint(p[0]);
            else if (PAT == 1 || PAT == 3 || PAT == 5) {
                const float2 v = *reinterpret_cast<const float2*>(p);
                acc ^= __float_as_uint(v.x) ^ __float_as_uint(v.y);
            } else {
                const float4 v = *reinterpret_cast<const float4*>(p);
                acc ^= __float_as_uint(v.x) ^ __float_as_uint(v.y) ^ __float_as_uint(v.z) ^ __float_as_uint(v.w);
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * NT + threadIdx.x] = __uint_as_float(acc);
}

template <int PAT>
void run(const char* name, float* out, long long* cyc) {
    cudaFuncSetAttribute(k<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 4 + 1024);
    k<PAT><<<148, NT, 16384 * 4 + 1024>>>(out, cyc);
    k<PAT><<<148, NT, 16384 * 4 + 1024>>>(out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double loads = double(NT / 32) * ITERS * UNR;  // warp-wide loads per SM
    printf("%-8s %8.3f cycles per warp load per SM\n", name, m / loads);
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * NT * 4);
    cudaMalloc(&cyc, 148 * 8);
    run<0>("u32", out, cyc);
    run<1>("u64", out, cyc);
    run<2>("u128", out, cyc);
    run<3>("g6_64", out, cyc);
    run<4>("g6_128", out, cyc);
    run<5>("d64", out, cyc);
    run<6>("d128", out, cyc);
    run<7>("d32", out, cyc);
    return 0;
}
