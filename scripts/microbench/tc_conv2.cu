// Experiment: the Table I large net's conv2 forward (PAPER.md:235-243:
// 20 maps 26x26 -> 60 maps 22x22, 5x5 kernel) as an implicit GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, accumulators in TMEM), against the FFMA direct convolution the
// worker kernel uses, for accuracy (vs float64 on the host) and time.
//
//   D[p][m] = sum_k A[p][k] B[m][k],  p = conv position (22x22 = 484 -> M = 512 = 4 tiles of 128),
//   k = (input map n, tap i, tap j) (20 x 25 = 500 -> K = 512), m = output map (60 -> N = 64).
//
// One CTA per image.  A is the im2col of the image, built slab by slab (KS = 32 of K) in shared
// memory in the canonical K-major no-swizzle layout (8-row x 16-byte core matrices: SBO = 128 B
// between 8-row groups, LBO = the K-chunk stride); B likewise.  Precision modes: 1 = one TF32 pass
// (10-bit mantissas), 3 = 3xTF32 (a = a_hi + a_lo: a_hi b_hi + a_hi b_lo + a_lo b_hi).  One thread
// issues the MMAs (M = 128, N = 64, K = 8 per instruction) and commits them to an mbarrier; four
// warps read the accumulators back with tcgen05.ld (32 lanes x 32-bit columns each).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_conv2 scripts/microbench/tc_conv2.cu
//   /tmp/tc_conv2 [images]
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int C = 20, H = 26, W = 26, M = 60, K = 5, OH = H - K + 1, OW = W - K + 1;  // 22 x 22
constexpr int NPOS = OH * OW, KDIM = C * K * K;                                     // 484, 500
constexpr int MP = 512, NP = 64, KP = 512, KS = 32, NSLAB = KP / KS, MT = MP / 128;
constexpr int NT = 512;
// shared memory: A slab per precision part [tile][kc][rowgroup][8][16 B] and B slab
constexpr int A_TILE_BYTES = (KS * 4 / 16) * 16 * 128;  // 8 kc x 16 rowgroups x 128 B = 16 KB
constexpr int A_BYTES = MT * A_TILE_BYTES;                // 64 KB
constexpr int B_BYTES = (KS * 4 / 16) * (NP / 8) * 128;   // 8 kc x 8 rowgroups x 128 B = 8 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// canonical K-major no-swizzle smem descriptor (Blackwell version 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32) | (1ull << 46);
}

// byte offset of element (row r, k) of a K-major slab with R rows (KS columns of 4 bytes)
__device__ __forceinline__ int kmaj_off(int r, int k, int R) {
    return (k >> 2) * (R / 8) * 128 + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__global__ void __launch_bounds__(NT, 1)
tc_conv2(const float* __restrict__ X, const float* __restrict__ Wt, const float* __restrict__ bias,
         float* __restrict__ out, int prec, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* Ahi = sm;
    unsigned char* Alo = sm + A_BYTES;
    unsigned char* Bhi = sm + 2 * A_BYTES;
    unsigned char* Blo = Bhi + B_BYTES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(Blo + B_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
    const float* x = X + (size_t)blockIdx.x * C * H * W;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    long long t0 = clock64(), t_build = 0, t_mma = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(MT * NP));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    // kind::tf32, D f32, A/B TF32, K-major, N = 64, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t phase = 0;
    for (int s = 0; s < NSLAB; ++s) {
        long long tb = clock64();
        // im2col slab: A[p][k0 + kk] for p < 512, kk < 32 (hi and lo parts)
        for (int e = tid; e < MP * KS; e += NT) {
            const int p = e / KS, kk = e % KS, k = s * KS + kk;
            float v = 0.f;
            if (p < NPOS && k < KDIM) {
                const int n = k / 25, i = (k % 25) / 5, j = k % 5, y = p / OW, xx = p % OW;
                v = x[(n * H + y + i) * W + xx + j];
            }
            const uint32_t hi = tf32_hi(v);
            const uint32_t lo = tf32_hi(v - __uint_as_float(hi));
            const int t = p >> 7, r = p & 127;
            *reinterpret_cast<uint32_t*>(Ahi + t * A_TILE_BYTES + kmaj_off(r, kk, 128)) = hi;
            *reinterpret_cast<uint32_t*>(Alo + t * A_TILE_BYTES + kmaj_off(r, kk, 128)) = lo;
        }
        for (int e = tid; e < NP * KS; e += NT) {
            const int m = e / KS, kk = e % KS, k = s * KS + kk;
            const float v = (m < M && k < KDIM) ? Wt[m * KDIM + k] : 0.f;
            const uint32_t hi = tf32_hi(v);
            const uint32_t lo = tf32_hi(v - __uint_as_float(hi));
            *reinterpret_cast<uint32_t*>(Bhi + kmaj_off(m, kk, NP)) = hi;
            *reinterpret_cast<uint32_t*>(Blo + kmaj_off(m, kk, NP)) = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        long long tm = clock64();
        t_build += tm - tb;
        if (tid == 0) {
            const uint32_t a_lbo = 16 * 128, b_lbo = (NP / 8) * 128;  // next 16-B K chunk
            for (int t = 0; t < MT; ++t) {
                for (int ks = 0; ks < KS / 8; ++ks) {  // K = 8 tf32 = 2 chunks per instruction
                    const uint32_t aoff = t * A_TILE_BYTES + ks * 2 * a_lbo, boff = ks * 2 * b_lbo;
                    const uint64_t ah = sdesc(smem_u32(Ahi) + aoff, a_lbo, 128), al = sdesc(smem_u32(Alo) + aoff, a_lbo, 128);
                    const uint64_t bh = sdesc(smem_u32(Bhi) + boff, b_lbo, 128), bl = sdesc(smem_u32(Blo) + boff, b_lbo, 128);
                    const uint32_t d = tmem + t * NP;
                    const uint32_t acc0 = (s > 0 || ks > 0) ? 1u : 0u;
                    // hi x hi first (initialises), then the two cross terms (3xTF32)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                 "l"(ah), "l"(bh), "r"(idesc), "r"(acc0));
                    if (prec == 3) {
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                     "l"(ah), "l"(bl), "r"(idesc), "r"(1u));
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                     "l"(al), "l"(bh), "r"(idesc), "r"(1u));
                    }
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(bar)));
        }
        // wait for the MMAs (they read the slab) before the next slab overwrites it
        {
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done)
                             : "r"(smem_u32(bar)), "r"(phase));
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
        t_mma += clock64() - tm;
    }
    // epilogue: warp w (< 4) reads TMEM lanes [32w, 32w + 32) = rows of each M tile
    long long te = clock64();
    if (warp < 4) {
        for (int t = 0; t < MT; ++t) {
            for (int c0 = 0; c0 < NP; c0 += 16) {
                uint32_t v[16];
                const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + t * NP + c0;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                               "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                               "=r"(v[14]), "=r"(v[15])
                             : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                const int p = t * 128 + 32 * warp + lane;
                if (p < NPOS)
                    for (int q = 0; q < 16; ++q)
                        if (c0 + q < M)
                            out[((size_t)blockIdx.x * M + c0 + q) * NPOS + p] = __uint_as_float(v[q]) + bias[c0 + q];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(MT * NP));
    if (tid == 0 && cycles) {
        cycles[blockIdx.x * 4 + 0] = t_build;
        cycles[blockIdx.x * 4 + 1] = t_mma;
        cycles[blockIdx.x * 4 + 2] = clock64() - te;
        cycles[blockIdx.x * 4 + 3] = clock64() - t0;
    }
}

// FFMA direct convolution, the worker kernel's arithmetic (fixed order n, i, j per output)
__global__ void ffma_conv2(const float* __restrict__ X, const float* __restrict__ Wt, const float* __restrict__ bias,
                           float* __restrict__ out, long long* cycles) {
    const float* x = X + (size_t)blockIdx.x * C * H * W;
    long long t0 = clock64();
    for (int e = threadIdx.x; e < M * NPOS; e += blockDim.x) {
        const int m = e / NPOS, p = e % NPOS, y = p / OW, xx = p % OW;
        float z = bias[m];
        for (int n = 0; n < C; ++n)
            for (int i = 0; i < K; ++i)
                for (int j = 0; j < K; ++j) z = fmaf(Wt[((m * C + n) * K + i) * K + j], x[(n * H + y + i) * W + xx + j], z);
        out[((size_t)blockIdx.x * M + m) * NPOS + p] = z;
    }
    __syncthreads();
    if (threadIdx.x == 0 && cycles) cycles[blockIdx.x] = clock64() - t0;
}

static uint64_t sm64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static float unif(uint64_t& s, float a) { return (float)(((sm64(s) >> 40) * (1.0 / 16777216.0)) * 2 - 1) * a; }

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

int main(int argc, char** argv) {
    const int nimg = argc > 1 ? atoi(argv[1]) : 148;
    uint64_t seed = 7;
    // inputs like the worker's: tanh'd pooled activations in (-1, 1), weights U(+-1/sqrt(fan_in))
    std::vector<float> X((size_t)nimg * C * H * W), Wt(M * KDIM), B(M);
    for (auto& v : X) v = std::tanh(2.f * unif(seed, 1.f));
    for (auto& v : Wt) v = unif(seed, 1.f / std::sqrt((float)KDIM));
    for (auto& v : B) v = unif(seed, 1.f / std::sqrt((float)KDIM));
    float *dX, *dW, *dB, *dO1, *dO3, *dOf;
    long long *dc, *dcf;
    const size_t osz = (size_t)nimg * M * NPOS;
    CK(cudaMalloc(&dX, X.size() * 4));
    CK(cudaMalloc(&dW, Wt.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dO1, osz * 4));
    CK(cudaMalloc(&dO3, osz * 4));
    CK(cudaMalloc(&dOf, osz * 4));
    CK(cudaMalloc(&dc, nimg * 4 * sizeof(long long)));
    CK(cudaMalloc(&dcf, nimg * sizeof(long long)));
    CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW, Wt.data(), Wt.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const int smem = 2 * A_BYTES + 2 * B_BYTES + 64;
    CK(cudaFuncSetAttribute(tc_conv2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms[3];
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        tc_conv2<<<nimg, NT, smem>>>(dX, dW, dB, dO1, 1, rep ? dc : nullptr);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms[0], e0, e1);
    }
    std::vector<long long> c1(nimg * 4);
    CK(cudaMemcpy(c1.data(), dc, c1.size() * 8, cudaMemcpyDeviceToHost));
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        tc_conv2<<<nimg, NT, smem>>>(dX, dW, dB, dO3, 3, rep ? dc : nullptr);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms[1], e0, e1);
    }
    std::vector<long long> c3(nimg * 4);
    CK(cudaMemcpy(c3.data(), dc, c3.size() * 8, cudaMemcpyDeviceToHost));
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        ffma_conv2<<<nimg, 384>>>(dX, dW, dB, dOf, rep ? dcf : nullptr);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms[2], e0, e1);
    }
    CK(cudaGetLastError());
    std::vector<long long> cf(nimg);
    CK(cudaMemcpy(cf.data(), dcf, cf.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<float> O1(osz), O3(osz), Of(osz);
    CK(cudaMemcpy(O1.data(), dO1, osz * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(O3.data(), dO3, osz * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Of.data(), dOf, osz * 4, cudaMemcpyDeviceToHost));
    // float64 reference on a sample of images: worst |err| / max(|ref|, 1e-2 max|ref|) (the R9 form)
    double w1 = 0, w3 = 0, wf = 0, n1 = 0, n3 = 0, nf = 0, nr = 0;
    const int ncheck = nimg < 8 ? nimg : 8;
    for (int b = 0; b < ncheck; ++b) {
        std::vector<double> ref(M * NPOS);
        double rmax = 0;
        for (int m = 0; m < M; ++m)
            for (int p = 0; p < NPOS; ++p) {
                const int y = p / OW, xx = p % OW;
                double z = B[m];
                for (int n = 0; n < C; ++n)
                    for (int i = 0; i < K; ++i)
                        for (int j = 0; j < K; ++j)
                            z += (double)Wt[((m * C + n) * K + i) * K + j] *
                                 X[(size_t)b * C * H * W + (n * H + y + i) * W + xx + j];
                ref[m * NPOS + p] = z;
                rmax = std::fmax(rmax, std::fabs(z));
            }
        for (int e = 0; e < M * NPOS; ++e) {
            const double r = ref[e], tol = std::fmax(std::fabs(r), 1e-2 * rmax);
            const size_t o = (size_t)b * M * NPOS + e;
            w1 = std::fmax(w1, std::fabs(O1[o] - r) / tol);
            w3 = std::fmax(w3, std::fabs(O3[o] - r) / tol);
            wf = std::fmax(wf, std::fabs(Of[o] - r) / tol);
            n1 += (O1[o] - r) * (O1[o] - r);
            n3 += (O3[o] - r) * (O3[o] - r);
            nf += (Of[o] - r) * (Of[o] - r);
            nr += r * r;
        }
    }
    auto med = [](std::vector<long long> v, int stride, int off) {
        std::vector<long long> x;
        for (size_t i = off; i < v.size(); i += stride) x.push_back(v[i]);
        std::sort(x.begin(), x.end());
        return x[x.size() / 2];
    };
    printf("conv2 forward of the Table I large net (20x26x26 -> 60x22x22, 5x5; %d images, one CTA each)\n", nimg);
    printf("  %-28s %10s %10s %10s %10s | %12s %12s\n", "path", "build cyc", "mma cyc", "epi cyc", "total cyc",
           "max rel err", "norm rel err");
    printf("  %-28s %10lld %10lld %10lld %10lld | %12.3g %12.3g   (%.3f ms for all images)\n",
           "tcgen05 kind::tf32 x1", med(c1, 4, 0), med(c1, 4, 1), med(c1, 4, 2), med(c1, 4, 3), w1,
           std::sqrt(n1 / nr), ms[0]);
    printf("  %-28s %10lld %10lld %10lld %10lld | %12.3g %12.3g   (%.3f ms)\n", "tcgen05 kind::tf32 x3 (3xTF32)",
           med(c3, 4, 0), med(c3, 4, 1), med(c3, 4, 2), med(c3, 4, 3), w3, std::sqrt(n3 / nr), ms[1]);
    printf("  %-28s %10s %10s %10s %10lld | %12.3g %12.3g   (%.3f ms, 384 threads, naive loop order)\n",
           "FFMA direct (fp32)", "-", "-", "-", med(cf, 1, 0), wf, std::sqrt(nf / nr), ms[2]);
    printf("  errors vs float64: max |err| / max(|ref|, 1e-2 max|ref|) (R9 form; bound 1e-4), norm-wise (bound 1e-5)\n");
    return 0;
}
