// Microbenchmark: tcgen05.mma kind::tf32 issue rate (cycles per instruction) vs the N of the
// instruction (M = 128, K = 8, operands in shared memory, one accumulator), one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_rate scripts/microbench/tc_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

template <int N, int MM>
__global__ void rate(long long* out, int iters, int ntiles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f800000u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *slot;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
    if (threadIdx.x == 0) {
        const uint64_t a = sdesc(smem_u32(sm), 16 * 128, 128), b = sdesc(smem_u32(sm + 32768), (N / 8) * 128, 128);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
            for (int t = 0; t < ntiles; ++t) {
                const uint32_t d = tmem + t * N;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(a), "l"(b), "r"(idesc), "r"(1u));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(smem_u32(bar)));
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int MM>
void run(int ntiles) {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(rate<N, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
    const int iters = 200;
    rate<N, MM><<<148, 128, 65536 + 64>>>(d, iters, ntiles);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double cyc = (double)h[0] / (iters * ntiles);
    const double macs = (double)MM * N * 8;
    printf("M=%3d N=%3d K=8 tf32, %d independent accumulators: %7.1f cycles per MMA = %6.0f MAC/clk/SM (%s)\n", MM, N,
           ntiles, cyc, macs / cyc, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<64, 128>(1);
    run<64, 128>(4);
    run<128, 128>(1);
    run<128, 128>(4);
    run<256, 128>(1);
    run<256, 128>(2);
    run<256, 64>(1);
    return 0;
}
