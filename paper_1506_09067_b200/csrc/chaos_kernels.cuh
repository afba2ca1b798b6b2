// chaos_kernels.cuh -- sm_100a device code of the CHAOS hot path.
//
// One persistent CTA per SM is one CHAOS *worker* ("multiple identical
// network instances (workers) ... sharing weight parameters; other variables are
// thread private").  A worker claims G images at a time from a device counter
// ("selecting an image in the set of images not yet processed ...
// faster workers can process more images"), runs the whole forward pass, the
// softmax cross-entropy error and the back-propagation for its G images with every
// activation, argmax and partial derivative in shared memory, and publishes each
// layer's gradient sum with fp32 REDs into the one shared weight copy in HBM/L2
// right after that layer's gradients are computed (controlled hogwild:
// "updates of shared weights are delayed to the end of each layer's computations";
// PAPER.md:140, arbitrary order of synchronization: no locks, first come first
// served writes, on-demand reads).  Conv-layer weights are read on demand from L2
// into shared memory with one cp.async.bulk (TMA bulk copy) per layer and group.
//
// Layer arithmetic (readings R1-R5):
//   conv   z[m][r][c] = b[m] + sum_n sum_i sum_j W[m][n][i][j] * a[n][r+i][c+j]
//   pool   non-overlapping kp x kp max (floor), first strict maximum in row-major order;
//          computed on z (tanh is monotone, R4) and tanh applied to the pooled value only
//   full   z[o] = b[o] + sum_i W[o][i] a[i];  hidden y = tanh(z);  logits un-squashed
//   loss   L = logsumexp(z) - z[label];  delta_out = softmax(z) - onehot(label)
//   back   gW = delta (x) input; gb = delta; delta_in = W^T delta (pre-update W);
//          tanh-fed inputs multiply by (1 - a^2); pool routes delta to the argmax only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace chaos {

constexpr int kClasses = 10;
constexpr int kZStride = 16;  // logits / output-delta row stride in shared memory
constexpr int kHdrBytes = 256;

enum Mode : int { kHogwild = 0, kSync = 1, kEval = 2, kForward = 3 };
enum Latch : int { kLatchLabel = 1, kLatchNonfinite = 2 };

__host__ __device__ constexpr int round4(int x) { return (x + 3) / 4 * 4; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// Convolution block: conv (valid, stride 1, C->M maps, KxK) -> tanh -> KPxKP max-pool (floor).
// Tuning knobs: MT maps per thread in the forward; TT taps per thread and GS split of the
// (image, window) sum in the weight gradient; NCH input maps per thread in delta_in.
template <int C_, int H_, int W_, int M_, int K_, int KP_, int MT_, int TT_, int GS_, int NCH_>
struct Conv {
    static constexpr int C = C_, H = H_, W = W_, M = M_, K = K_, KP = KP_;
    static constexpr int OH = H - K + 1, OW = W - K + 1;
    static constexpr int PH = OH / KP, PW = OW / KP, P = PH * PW;
    static constexpr int MP = round4(M);     // internal row pitch (maps padded to 16 B)
    static constexpr int KK = K * K;
    static constexpr int ROWS = C * KK;      // internal W is [C*K*K][MP], bias [MP]
    static constexpr int WFL = ROWS * MP, BFL = MP;
    static constexpr int IN_SZ = C * H * W, OUT_SZ = M * P;
    static constexpr int MT = MT_, TT = TT_, GS = GS_, NCH = NCH_;
    static_assert(M % MT == 0, "MT must divide M");
    static_assert(KK % TT == 0, "TT must divide K*K");
    static_assert(C % NCH == 0, "NCH must divide C");
    static_assert(PH >= 1 && PW >= 1, "pool larger than the conv output");
    static constexpr int SCRATCH = GS > 1 ? GS * WFL : 0;
};

// Fully connected layer IN -> OUT, tanh or identity (logits).
template <int IN_, int OUT_, bool TANH_>
struct Full {
    static constexpr int IN = IN_, OUT = OUT_;
    static constexpr bool TANH = TANH_;
    static constexpr int WFL = round4(IN * OUT), BFL = round4(OUT);
};

// Internal parameter offsets (floats): per weighted layer W block then b block, 16-B aligned.
template <class Net>
struct POff {
    using C1 = typename Net::C1;
    using C2 = typename Net::C2;
    using C3 = typename Net::C3;
    using F1 = typename Net::F1;
    using F2 = typename Net::F2;
    static constexpr int c1w = 0;
    static constexpr int c1b = c1w + C1::WFL;
    static constexpr int c2w = c1b + C1::BFL;
    static constexpr int c2b = c2w + (Net::NCONV >= 2 ? C2::WFL : 0);
    static constexpr int c3w = c2b + (Net::NCONV >= 2 ? C2::BFL : 0);
    static constexpr int c3b = c3w + (Net::NCONV >= 3 ? C3::WFL : 0);
    static constexpr int f1w = c3b + (Net::NCONV >= 3 ? C3::BFL : 0);
    static constexpr int f1b = f1w + F1::WFL;
    static constexpr int f2w = f1b + F1::BFL;
    static constexpr int f2b = f2w + (Net::NFULL >= 2 ? F2::WFL : 0);
    static constexpr int total = f2b + (Net::NFULL >= 2 ? F2::BFL : 0);
};

// Shared-memory carve-up for G images per worker.
template <class Net, int G>
struct SLayout {
    using C1 = typename Net::C1;
    using C2 = typename Net::C2;
    using C3 = typename Net::C3;
    using F1 = typename Net::F1;
    static constexpr int conv_blk(int w, int b) { return w + b; }
    static constexpr int WBUF = round4(cmax(
        cmax(cmax(C1::WFL + C1::BFL, C1::SCRATCH),
             Net::NCONV >= 2 ? cmax(C2::WFL + C2::BFL, C2::SCRATCH) : 0),
        Net::NCONV >= 3 ? cmax(C3::WFL + C3::BFL, C3::SCRATCH) : 0));
    static constexpr int X = 0;  // float offsets, relative to the float arena
    static constexpr int A1 = X + round4(G * C1::IN_SZ);
    static constexpr int A2 = A1 + round4(G * C1::OUT_SZ);
    static constexpr int A3 = A2 + (Net::NCONV >= 2 ? round4(G * C2::OUT_SZ) : 0);
    static constexpr int HH = A3 + (Net::NCONV >= 3 ? round4(G * C3::OUT_SZ) : 0);
    static constexpr int Z = HH + (Net::NFULL >= 2 ? round4(G * F1::OUT) : 0);
    static constexpr int WB = Z + G * kZStride;
    static constexpr int FLOATS = WB + WBUF;
    // argmax bytes
    static constexpr int AM1 = 0;
    static constexpr int AM2 = AM1 + (G * C1::OUT_SZ + 15) / 16 * 16;
    static constexpr int AM3 = AM2 + (Net::NCONV >= 2 ? (G * C2::OUT_SZ + 15) / 16 * 16 : 0);
    static constexpr int AMB = AM3 + (Net::NCONV >= 3 ? (G * C3::OUT_SZ + 15) / 16 * 16 : 0);
    static constexpr int BYTES = kHdrBytes + FLOATS * 4 + AMB;
};

struct KArgs {
    float* params;              // internal layout, shared by all workers (the CHAOS weight store)
    float* partial;             // sync: [slot][pstride] gradient sums
    long long pstride;
    const float* images;        // [n][in]
    const int* labels;          // [n]
    long long n;                // images in this launch
    long long first_slot_sample;// sync: sample index of slot 0 (relative to images)
    unsigned long long* counter;// hogwild work counter (claims in units of images)
    int* latch;                 // device error latch
    double* loss_sum;           // training loss accumulator
    float neg_lr;
    int* claims;                // optional per-image claim counts
    float* out_loss;            // eval: per-image loss
    unsigned char* out_wrong;   // eval: per-image error flag
    float* out_logits;          // forward: [n][kClasses]
};

// ------------------------------------------------------------------------------------
// small PTX helpers: mbarrier + cp.async.bulk (TMA bulk copy global -> shared)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// Issue (tid 0) a bulk copy of `floats` floats; everyone waits.  Caller guarantees
// 16-B alignment of both ends and floats % 4 == 0.
struct Stager {
    uint64_t* bar;
    uint32_t phase;
    __device__ __forceinline__ void begin() {
        fence_proxy_async();  // order earlier generic accesses (smem reuse, our REDs) before the async proxy
        __syncthreads();
    }
    __device__ __forceinline__ void issue(float* dst, const float* src, int floats, uint32_t extra_bytes = 0) {
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, static_cast<uint32_t>(floats) * 4u + extra_bytes);
            int off = 0;
            while (off < floats) {
                const int chunk = (floats - off) > 16384 ? 16384 : (floats - off);  // 64 KiB pieces
                bulk_g2s(dst + off, src + off, static_cast<uint32_t>(chunk) * 4u, bar);
                off += chunk;
            }
        }
    }
    __device__ __forceinline__ void wait() {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
    __device__ __forceinline__ void stage(float* dst, const float* src, int floats) {
        begin();
        issue(dst, src, floats);
        wait();
    }
};

template <int N, bool A4>
__device__ __forceinline__ void load_vec(float (&v)[N], const float* p) {
    if constexpr (A4 && N % 4 == 0) {
#pragma unroll
        for (int q = 0; q < N / 4; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(p + 4 * q);
            v[4 * q] = t.x;
            v[4 * q + 1] = t.y;
            v[4 * q + 2] = t.z;
            v[4 * q + 3] = t.w;
        }
    } else if constexpr (A4 && N > 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
#pragma unroll
        for (int q = 4; q < N; ++q) v[q] = p[q];
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) v[q] = p[q];
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Publish one gradient element: hogwild = RED.ADD of -lr*g into the shared weights
// (no lock, arbitrary order); sync = plain store of the group sum into its slot.
template <int MODE>
__device__ __forceinline__ void publish(const KArgs& a, int slot, int idx, float g) {
    if constexpr (MODE == kHogwild) {
        atomicAdd(a.params + idx, a.neg_lr * g);
    } else if constexpr (MODE == kSync) {
        a.partial[static_cast<long long>(slot) * a.pstride + idx] = g;
    }
}

// ------------------------------------------------------------------------------------
// conv -> tanh -> max-pool forward (fused).  One thread item = MT maps x one pooled
// window x one image; the KP*KP conv outputs of the window stay in registers, the
// weights of the MT maps are warp-uniform vector loads from the staged block.
// ------------------------------------------------------------------------------------
template <class L, int NT>
__device__ __forceinline__ void conv_fwd(const float* __restrict__ in, const float* __restrict__ wsm,
                                         float* __restrict__ out, uint8_t* __restrict__ am, int cnt) {
    constexpr int MT = L::MT, KP = L::KP, K = L::K, PW = L::PW, P = L::P, MG = L::M / MT;
    constexpr int PS = KP + K - 1;
    constexpr bool A4 = (MT % 4 == 0) || (MG == 1);
    const int total = MG * cnt * P;
    for (int it = threadIdx.x; it < total; it += NT) {
        const int p = it % P;
        const int t = it / P;
        const int g = t % cnt;
        const int mg = t / cnt;
        const int pr = p / PW, pc = p - (p / PW) * PW;
        float acc[MT][KP * KP];
        {
            float b[MT];
            load_vec<MT, A4>(b, wsm + L::WFL + mg * MT);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int q = 0; q < KP * KP; ++q) acc[mt][q] = b[mt];
        }
        const float* ib = in + g * L::IN_SZ + (pr * KP) * L::W + pc * KP;
        const float* wb = wsm + mg * MT;
#pragma unroll 1
        for (int n = 0; n < L::C; ++n) {
            float patch[PS][PS];
#pragma unroll
            for (int u = 0; u < PS; ++u)
#pragma unroll
                for (int v = 0; v < PS; ++v) patch[u][v] = ib[n * (L::H * L::W) + u * L::W + v];
#pragma unroll
            for (int i = 0; i < K; ++i)
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    float wv[MT];
                    load_vec<MT, A4>(wv, wb + ((n * K + i) * K + j) * L::MP);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int u = 0; u < KP; ++u)
#pragma unroll
                            for (int v = 0; v < KP; ++v)
                                acc[mt][u * KP + v] = fmaf(wv[mt], patch[u + i][v + j], acc[mt][u * KP + v]);
                }
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            float best = acc[mt][0];
            int arg = 0;
#pragma unroll
            for (int q = 1; q < KP * KP; ++q)
                if (acc[mt][q] > best) {  // first strict maximum wins (R4)
                    best = acc[mt][q];
                    arg = q;
                }
            const int o = g * L::OUT_SZ + (mg * MT + mt) * P + p;
            out[o] = tanhf(best);
            am[o] = static_cast<uint8_t>(arg);
        }
    }
}

// ------------------------------------------------------------------------------------
// conv backward.  dp[g][m][pp] holds dL/dz at the argmax of pooled output pp (the
// pool routes the delta there and nowhere else).  Step 1: weight gradient
//   gW[n][i][j][m] = sum_g sum_pp dp[g][m][pp] * in[g][n][r(pp)+i][c(pp)+j],  gb[m] = sum dp
// one thread per (m, n, tap group [, split]), published as soon as it is complete.
// Step 2 (NEED_DIN): partial derivatives of the previous layer, gathered per input
// element from the staged (pre-update) W snapshot and multiplied by (1 - a^2), written
// in place over `in` (the previous pooled activations are dead after step 1).
// ------------------------------------------------------------------------------------
template <class L, int NT, int MODE, bool NEED_DIN>
__device__ __forceinline__ void conv_bwd(const KArgs& a, int slot, float* __restrict__ in,
                                         const float* __restrict__ dp, const uint8_t* __restrict__ am,
                                         float* __restrict__ wsm, int woff, int boff, int cnt) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int TT = L::TT, TG = KK / TT, GS = L::GS;
    const int span = cnt * P;
    // ---- step 1: weight gradients
    {
        const int total = M * C * TG * GS;
        for (int it = threadIdx.x; it < total; it += NT) {
            const int m = it % M;
            int r = it / M;
            const int n = r % C;
            r /= C;
            const int tg = r % TG;
            const int s = r / TG;
            const int q0 = (GS == 1) ? 0 : (span * s) / GS;
            const int q1 = (GS == 1) ? span : (span * (s + 1)) / GS;
            float acc[TT];
#pragma unroll
            for (int t = 0; t < TT; ++t) acc[t] = 0.f;
            int g = q0 / P;
            int pp = q0 - g * P;
            for (int q = q0; q < q1; ++q) {
                const int o = g * L::OUT_SZ + m * P + pp;
                const float d = dp[o];
                const int arg = am[o];
                const int r0 = (pp / PW) * KP + arg / KP;
                const int c0 = (pp % PW) * KP + arg % KP;
                const float* base = in + g * L::IN_SZ + n * (L::H * L::W) + r0 * L::W + c0;
#pragma unroll
                for (int t = 0; t < TT; ++t) {
                    const int tap = tg * TT + t;
                    acc[t] = fmaf(d, base[(tap / K) * L::W + (tap % K)], acc[t]);
                }
                if (++pp == P) {
                    pp = 0;
                    ++g;
                }
            }
#pragma unroll
            for (int t = 0; t < TT; ++t) {
                const int widx = (n * KK + tg * TT + t) * L::MP + m;
                if constexpr (GS == 1)
                    publish<MODE>(a, slot, woff + widx, acc[t]);
                else
                    wsm[s * L::WFL + widx] = acc[t];
            }
        }
        for (int m = threadIdx.x; m < M; m += NT) {  // bias gradient
            float gb = 0.f;
            for (int g = 0; g < cnt; ++g)
                for (int pp = 0; pp < P; ++pp) gb += dp[g * L::OUT_SZ + m * P + pp];
            publish<MODE>(a, slot, boff + m, gb);
        }
        if constexpr (GS > 1) {
            __syncthreads();
            for (int e = threadIdx.x; e < L::ROWS * M; e += NT) {
                const int m = e % M;
                const int row = e / M;
                const int widx = row * L::MP + m;
                float s = 0.f;
#pragma unroll
                for (int k = 0; k < GS; ++k) s += wsm[k * L::WFL + widx];
                publish<MODE>(a, slot, woff + widx, s);
            }
        }
    }
    if constexpr (NEED_DIN) {
        static_assert(GS == 1, "delta_in needs the staged weights intact");
        __syncthreads();
        // ---- step 2: delta_in (gather form), in place over `in`
        constexpr int NCG = C / L::NCH;
        constexpr int HW = L::H * L::W;
        const int total = cnt * HW * NCG;
        for (int it = threadIdx.x; it < total; it += NT) {
            const int pos = it % HW;
            const int r = it / HW;
            const int g = r % cnt;
            const int ncg = r / cnt;
            const int y = pos / L::W, x = pos - (pos / L::W) * L::W;
            float acc[L::NCH];
#pragma unroll
            for (int c = 0; c < L::NCH; ++c) acc[c] = 0.f;
            const int ylo = y - (K - 1) - (KP - 1), xlo = x - (K - 1) - (KP - 1);
            const int pr0 = ylo <= 0 ? 0 : (ylo + KP - 1) / KP;
            const int pc0 = xlo <= 0 ? 0 : (xlo + KP - 1) / KP;
            const int pr1 = min(L::PH - 1, y / KP), pc1 = min(L::PW - 1, x / KP);
            const float* wrow0 = wsm + (ncg * L::NCH) * KK * L::MP;
            for (int m = 0; m < M; ++m) {
                for (int pr = pr0; pr <= pr1; ++pr)
                    for (int pc = pc0; pc <= pc1; ++pc) {
                        const int o = g * L::OUT_SZ + m * P + pr * PW + pc;
                        const int arg = am[o];
                        const int i = y - (pr * KP + arg / KP);
                        const int j = x - (pc * KP + arg % KP);
                        if (i >= 0 && i < K && j >= 0 && j < K) {
                            const float d = dp[o];
                            const float* wr = wrow0 + (i * K + j) * L::MP + m;
#pragma unroll
                            for (int c = 0; c < L::NCH; ++c) acc[c] = fmaf(wr[c * KK * L::MP], d, acc[c]);
                        }
                    }
            }
#pragma unroll
            for (int c = 0; c < L::NCH; ++c) {
                float* pa = in + g * L::IN_SZ + (ncg * L::NCH + c) * HW + pos;
                const float v = *pa;
                *pa = acc[c] * (1.f - v * v);
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// fully connected forward: one warp per output row, lanes over inputs, weights
// streamed from L2 (__ldcg: on-demand reads of the shared store, no stale L1 copy).
// ------------------------------------------------------------------------------------
template <class F, int G, int NT>
__device__ __forceinline__ void fc_fwd(const float* __restrict__ Wg, const float* __restrict__ bg,
                                       const float* __restrict__ in, float* __restrict__ out, int ostride,
                                       int cnt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    for (int o = warp; o < F::OUT; o += NW) {
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.f;
        const float* wr = Wg + static_cast<long long>(o) * F::IN;
#pragma unroll 4
        for (int i = lane; i < F::IN; i += 32) {
            const float w = __ldcg(wr + i);
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fmaf(w, in[g * F::IN + i], acc[g]);
        }
        const float b = __ldcg(bg + o);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float s = warp_sum(acc[g]) + b;
            if (lane == 0 && g < cnt) out[g * ostride + o] = F::TANH ? tanhf(s) : s;
        }
    }
}

// fully connected backward: one thread per input column i, loop over outputs o.
// Reads W[o][i] (pre-update, on demand) for delta_in, forms gW[o][i] = sum_g dz[g][o] a[g][i]
// and publishes it; delta_in * (1 - a^2) is written in place over the input activations.
template <class F, int G, int NT, int MODE, bool NEED_DIN>
__device__ __forceinline__ void fc_bwd(const KArgs& a, int slot, int woff, int boff, float* __restrict__ in,
                                       const float* __restrict__ dz, int dstride, int cnt) {
    const float* Wg = a.params + woff;
    for (int i = threadIdx.x; i < F::IN; i += NT) {
        float av[G], din[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            av[g] = (g < cnt) ? in[g * F::IN + i] : 0.f;
            din[g] = 0.f;
        }
#pragma unroll 2
        for (int o = 0; o < F::OUT; ++o) {
            float w = 0.f;
            if constexpr (NEED_DIN) w = __ldcg(Wg + static_cast<long long>(o) * F::IN + i);
            float gw = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (g < cnt) {
                    const float d = dz[g * dstride + o];
                    din[g] = fmaf(w, d, din[g]);
                    gw = fmaf(d, av[g], gw);
                }
            }
            publish<MODE>(a, slot, woff + o * F::IN + i, gw);
        }
        if constexpr (NEED_DIN) {
#pragma unroll
            for (int g = 0; g < G; ++g)
                if (g < cnt) in[g * F::IN + i] = din[g] * (1.f - av[g] * av[g]);
        }
    }
    for (int o = threadIdx.x; o < F::OUT; o += NT) {
        float gb = 0.f;
        for (int g = 0; g < cnt; ++g) gb += dz[g * dstride + o];
        publish<MODE>(a, slot, boff + o, gb);
    }
}

// ------------------------------------------------------------------------------------
// The worker kernel: hogwild training, sync-batch gradients, evaluation, forward.
// ------------------------------------------------------------------------------------
template <class Net, int G, int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) chaos_worker(KArgs a) {
    using C1 = typename Net::C1;
    using C2 = typename Net::C2;
    using C3 = typename Net::C3;
    using F1 = typename Net::F1;
    using F2 = typename Net::F2;
    using O = POff<Net>;
    using S = SLayout<Net, G>;
    constexpr int NCONV = Net::NCONV, NFULL = Net::NFULL;
    constexpr int IMG = C1::IN_SZ;

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    int* s_base = reinterpret_cast<int*>(smem + 8);
    int* s_lab = reinterpret_cast<int*>(smem + 16);  // G labels
    float* s_loss = reinterpret_cast<float*>(smem + 16 + 4 * 16);
    float* fa = reinterpret_cast<float*>(smem + kHdrBytes);
    float* xs = fa + S::X;
    float* a1 = fa + S::A1;
    float* a2 = fa + S::A2;
    float* a3 = fa + S::A3;
    float* hh = fa + S::HH;
    float* zz = fa + S::Z;
    float* wb = fa + S::WB;
    uint8_t* amb = smem + kHdrBytes + S::FLOATS * 4;
    uint8_t* am1 = amb + S::AM1;
    uint8_t* am2 = amb + S::AM2;
    uint8_t* am3 = amb + S::AM3;
    const float* P = a.params;

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    Stager st{bar, 0u};

    long long iter = 0;
    for (;;) {
        // ---------------- a1: claim the next unprocessed images
        if (threadIdx.x == 0) {
            long long base;
            if constexpr (MODE == kHogwild)
                base = static_cast<long long>(atomicAdd(a.counter, static_cast<unsigned long long>(G)));
            else
                base = (static_cast<long long>(blockIdx.x) + iter * gridDim.x) * G;
            *s_base = base < a.n ? static_cast<int>(base) : -1;
        }
        __syncthreads();
        const int base = *s_base;
        if (base < 0) break;
        const int slot = static_cast<int>(base / G);
        const int cnt = static_cast<int>(min(static_cast<long long>(G), a.n - base));
        ++iter;
        if (threadIdx.x < cnt) {
            int lab = 0;
            if constexpr (MODE != kForward) {
                lab = a.labels[base + threadIdx.x];
                if (lab < 0 || lab >= kClasses) {
                    atomicOr(a.latch, kLatchLabel);
                    lab = 0;
                }
            }
            s_lab[threadIdx.x] = lab;
            if constexpr (MODE == kHogwild)
                if (a.claims) atomicAdd(a.claims + base + threadIdx.x, 1);
        }
        // stage conv1 weights (+ the images when the group is 16-B aligned) with one bulk copy
        const float* xsrc = a.images + static_cast<long long>(base) * IMG;
        const bool x_bulk = ((reinterpret_cast<uintptr_t>(xsrc) & 15u) == 0) && ((cnt * IMG) % 4 == 0);
        st.begin();
        if (x_bulk) {
            if (threadIdx.x == 0) {
                mbar_expect_tx(bar, static_cast<uint32_t>(C1::WFL + C1::BFL + cnt * IMG) * 4u);
                bulk_g2s(wb, P + O::c1w, static_cast<uint32_t>(C1::WFL + C1::BFL) * 4u, bar);
                int off = 0;
                const int tot = cnt * IMG;
                while (off < tot) {
                    const int chunk = (tot - off) > 16384 ? 16384 : (tot - off);
                    bulk_g2s(xs + off, xsrc + off, static_cast<uint32_t>(chunk) * 4u, bar);
                    off += chunk;
                }
            }
        } else {
            for (int i = threadIdx.x; i < cnt * IMG; i += NT) xs[i] = __ldg(xsrc + i);
            st.issue(wb, P + O::c1w, C1::WFL + C1::BFL);
        }
        st.wait();
        if (!x_bulk) __syncthreads();  // the plain image stores of other threads

        // ---------------- a2: conv -> tanh -> pool, layer by layer
        conv_fwd<C1, NT>(xs, wb, a1, am1, cnt);
        float* alast = a1;
        if constexpr (NCONV >= 2) {
            st.stage(wb, P + O::c2w, C2::WFL + C2::BFL);
            conv_fwd<C2, NT>(a1, wb, a2, am2, cnt);
            alast = a2;
        }
        if constexpr (NCONV >= 3) {
            st.stage(wb, P + O::c3w, C3::WFL + C3::BFL);
            conv_fwd<C3, NT>(a2, wb, a3, am3, cnt);
            alast = a3;
        }
        __syncthreads();
        // ---------------- a3: full layers
        if constexpr (NFULL == 2) {
            fc_fwd<F1, G, NT>(P + O::f1w, P + O::f1b, alast, hh, F1::OUT, cnt);
            __syncthreads();
            fc_fwd<F2, G, NT>(P + O::f2w, P + O::f2b, hh, zz, kZStride, cnt);
        } else {
            fc_fwd<F1, G, NT>(P + O::f1w, P + O::f1b, alast, zz, kZStride, cnt);
        }
        __syncthreads();
        // ---------------- a4: softmax cross-entropy, output delta
        if (threadIdx.x < cnt) {
            const int g = threadIdx.x;
            float* z = zz + g * kZStride;
            const int lab = s_lab[g];
            if constexpr (MODE == kForward) {
                for (int o = 0; o < kClasses; ++o)
                    a.out_logits[(static_cast<long long>(base) + g) * kClasses + o] = z[o];
            } else {
                float zmax = z[0];
                int best = 0;
                for (int o = 1; o < kClasses; ++o)
                    if (z[o] > zmax) {
                        zmax = z[o];
                        best = o;
                    }
                float s = 0.f;
                for (int o = 0; o < kClasses; ++o) s += expf(z[o] - zmax);
                const float loss = logf(s) + zmax - z[lab];
                if (!isfinite(loss)) atomicOr(a.latch, kLatchNonfinite);
                if constexpr (MODE == kEval) {
                    a.out_loss[base + g] = loss;
                    a.out_wrong[base + g] = static_cast<unsigned char>(best != lab);
                } else {
                    const float inv = 1.f / s;
                    for (int o = 0; o < kClasses; ++o) z[o] = expf(z[o] - zmax) * inv - (o == lab ? 1.f : 0.f);
                    s_loss[g] = loss;
                }
            }
        }
        if constexpr (MODE == kHogwild || MODE == kSync) {
            __syncthreads();
            if (threadIdx.x == 0 && a.loss_sum) {
                double ls = 0.0;
                for (int g = 0; g < cnt; ++g) ls += s_loss[g];
                atomicAdd(a.loss_sum, ls);
            }
            // ---------------- a5: full layers backward (publish per layer)
            if constexpr (NFULL == 2) {
                fc_bwd<F2, G, NT, MODE, true>(a, slot, O::f2w, O::f2b, hh, zz, kZStride, cnt);
                __syncthreads();
                fc_bwd<F1, G, NT, MODE, true>(a, slot, O::f1w, O::f1b, alast, hh, F1::OUT, cnt);
            } else {
                fc_bwd<F1, G, NT, MODE, true>(a, slot, O::f1w, O::f1b, alast, zz, kZStride, cnt);
            }
            // ---------------- a6/a7: pool + conv backward, publish per layer
            if constexpr (NCONV >= 3) {
                st.stage(wb, P + O::c3w, C3::WFL + C3::BFL);
                conv_bwd<C3, NT, MODE, true>(a, slot, a2, a3, am3, wb, O::c3w, O::c3b, cnt);
            }
            if constexpr (NCONV >= 2) {
                st.stage(wb, P + O::c2w, C2::WFL + C2::BFL);
                conv_bwd<C2, NT, MODE, true>(a, slot, a1, a2, am2, wb, O::c2w, O::c2b, cnt);
            }
            __syncthreads();
            conv_bwd<C1, NT, MODE, false>(a, slot, xs, a1, am1, wb, O::c1w, O::c1b, cnt);
            if constexpr (MODE == kHogwild) __threadfence();
        }
        __syncthreads();
    }
}

// w[j] -= lr * sum_{s < nslots} partial[s][j]  (fixed order: the sync-mode update)
// or, with out != nullptr, out[j] = sum (gradient test hook, no update).
__global__ void chaos_reduce_update(float* __restrict__ params, const float* __restrict__ partial,
                                    long long pstride, int nslots, float lr, long long np, float* __restrict__ out) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= np) return;
    float s = 0.f;
    for (int k = 0; k < nslots; ++k) s += partial[static_cast<long long>(k) * pstride + j];
    if (out)
        out[j] = s;
    else
        params[j] -= lr * s;
}

// Fixed-order evaluation reduction: one CTA of 1024 threads.
__global__ void chaos_eval_reduce(const float* __restrict__ loss, const unsigned char* __restrict__ wrong,
                                  long long n, double* __restrict__ out_sum, long long* __restrict__ out_err) {
    __shared__ double ssum[1024];
    __shared__ long long serr[1024];
    double s = 0.0;
    long long e = 0;
    const long long per = (n + blockDim.x - 1) / blockDim.x;
    const long long i0 = threadIdx.x * per;
    const long long i1 = min(n, i0 + per);
    for (long long i = i0; i < i1; ++i) {
        s += static_cast<double>(loss[i]);
        e += wrong[i];
    }
    ssum[threadIdx.x] = s;
    serr[threadIdx.x] = e;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            ssum[threadIdx.x] += ssum[threadIdx.x + w];
            serr[threadIdx.x] += serr[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out_sum = ssum[0];
        *out_err = serr[0];
    }
}

}  // namespace chaos
