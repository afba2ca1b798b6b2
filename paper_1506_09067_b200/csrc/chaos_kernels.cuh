// chaos_kernels.cuh -- sm_100a device code of the CHAOS hot path.
//
// One persistent CTA per SM is one CHAOS *worker* ("multiple identical
// network instances (workers) ... sharing weight parameters; other variables are
// thread private").  A worker claims G images at a time from a device counter
// ("selecting an image in the set of images not yet processed ...
// faster workers can process more images"), runs the whole forward pass, the
// softmax cross-entropy error and the back-propagation for its G images with every
// activation, argmax and partial derivative in shared memory, and publishes each
// layer's gradient sum into the one shared fp32 weight store right after that layer's
// gradients are computed (controlled hogwild: "updates of shared weights
// are delayed to the end of each layer's computations", arbitrary order
// of synchronization: no locks, first come first served writes, on-demand reads).
//
// Blackwell mapping: conv weights are read on demand from L2 into shared memory with
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) issued ahead of use; a layer's gradient
// (-lr * sum over the G images) is assembled in shared memory in the weight store's
// layout and published with ONE TMA bulk reduction (cp.reduce.async.bulk .add.f32,
// SASS UBLKRED) -- the TMA engine performs the fp32 adds in L2, no per-element atomics
// from the SM.  Sync mode publishes the same buffer with a bulk copy into its slot.
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
#include <type_traits>
#include <cuda_runtime.h>

namespace chaos {

constexpr int kClasses = 10;
constexpr int kZStride = 16;  // logits / output-delta row stride in shared memory
constexpr int kHdrBytes = 512;  // mbarriers, claim word, labels, losses; [256, 512): tensor-core mbarriers
constexpr int kBiasScratch = 160;  // floats: FC bias-gradient scratch (>= every FC layer's BFL, asserted)

// kTrace: hogwild (kHogwild semantics) that also records, per claimed group and weighted layer,
// when its weight reads and its publishes happened on two global event counters, and stores each
// group's publish in its own slot -- the schedule a replay of the method re-runs (debug only)
enum Mode : int { kHogwild = 0, kSync = 1, kEval = 2, kForward = 3, kTrace = 4 };
__host__ __device__ constexpr bool is_hog(int mode) { return mode == kHogwild || mode == kTrace; }
// kTrace record layout per group (int64): [l * 6 + k] for weighted layer l < 5, k = 0 publish
// started (rank on the started counter), 1 publish done (rank on the done counter), 2/3 forward
// read (done count at its start / started count at its end), 4/5 the delta_in read (-1: the
// forward read's values serve); [30] = worker (CTA), [31] = the worker's iteration.
constexpr int kTraceRec = 32;
enum Latch : int { kLatchLabel = 1, kLatchNonfinite = 2, kLatchPavg = 4, kLatchPavgTimeout = 8 };

__host__ __device__ constexpr int round4(int x) { return (x + 3) / 4 * 4; }

// 2-conv nets whose conv2 delta_in splits each band's output-map loop over Net::DINSPLIT warps
// (conv_din<..., MSPLIT>).
template <class N, class = void>
struct DinPair {
    static constexpr int value = 1;
};
template <class N>
struct DinPair<N, std::void_t<decltype(N::DINSPLIT)>> {
    static constexpr int value = N::DINSPLIT;
};

// 2-conv nets whose conv2 delta_in runs window row by window row (conv_din_rows) declare DINROWS = true
template <class N, class = void>
struct DinRows {
    static constexpr bool value = false;
};
template <class N>
struct DinRows<N, std::void_t<decltype(N::DINROWS)>> {
    static constexpr bool value = N::DINROWS;
};

// Nets whose conv1 forward splits its last partial pass into single-map sub-items declare TAIL1 = true
template <class N, class = void>
struct Tail1 {
    static constexpr bool value = false;
};
template <class N>
struct Tail1<N, std::void_t<decltype(N::TAIL1)>> {
    static constexpr bool value = N::TAIL1;
};

// Nets whose conv3 / FC1 weights are too large to stage in shared memory (Table I large net,
// SURVEY NEXT-1) declare BIGW = true: W1 + W2 are staged once per iteration and kept; conv3
// and FC1 weights are read from L2 on demand.
template <class N, class = void>
struct BigW {
    static constexpr bool value = false;
};
template <class N>
struct BigW<N, std::void_t<decltype(N::BIGW)>> {
    static constexpr bool value = N::BIGW;
};
// Nets whose conv2 forward runs with map groups fastest over the lanes (conv_fwd MGF) declare
// MGF2 = true (measured per net)
// Nets whose conv2 forward runs on the tensor cores (conv_fwd_tc2) declare TC2 = true
template <class N, class = void>
struct TcC2 {
    static constexpr bool value = false;
};
template <class N>
struct TcC2<N, std::void_t<decltype(N::TC2)>> {
    static constexpr bool value = N::TC2;
};
template <class N, class = void>
struct MgfC2 {
    static constexpr bool value = false;
};
template <class N>
struct MgfC2<N, std::void_t<decltype(N::MGF2)>> {
    static constexpr bool value = N::MGF2;
};
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// Convolution block: conv (valid, stride 1, C->M maps, KxK) -> tanh -> KPxKP max-pool (floor).
#ifndef CHAOS_FFMA2  // bit mask of the loops that use it: 1 conv_fwd, (2: conv_din3, removed) 4 conv_bwd_sparse's gradient,
#define CHAOS_FFMA2 13  // 8 conv_gw_m, 16 conv_gw, 32 conv_din_gm, 64 conv_gw_wt (large net: 2 -7%, 16 -0.4%: off)
#endif
// Tuning knobs: MT maps per thread in the forward; TT taps per thread and GS split of the
// (image, window) sum in the weight gradient; RB input rows per band in delta_in.
// MPO > 0: the internal row pitch of W (default round4(M), 16-B rows).  An odd pitch puts the rows of
// consecutive input maps in distinct banks (lanes over input maps reading one map's weights:
// conflict-free, where a pitch of 40 hits 4 banks -- the medium net's conv2 delta_in); its forward
// then reads weights with scalar (broadcast) loads.
template <int C_, int H_, int W_, int M_, int K_, int KP_, int MT_, int TT_, int GS_, int RB_, int PB_ = 0,
          int MS_ = 0, bool UNUSED_ = false, bool DIN3_ = false, int GWIN_ = 0, bool DWIN_ = false, int NSPL_ = 1,
          int MPO_ = 0, int NPAD_ = 0, int FF_ = -1>
struct Conv {
    // FF: which loops of this layer use packed FP32 FMAs (the CHAOS_FFMA2 site mask; -1: the default),
    // measured per net: the few-warp Table I large worker loses 7% with them in its forward
    static constexpr int FF = FF_ < 0 ? CHAOS_FFMA2 : FF_;
    static constexpr int C = C_, H = H_, W = W_, M = M_, K = K_, KP = KP_;
    static constexpr int OH = H - K + 1, OW = W - K + 1;
    static constexpr int PH = OH / KP, PW = OW / KP, P = PH * PW;
    static constexpr int MP = MPO_ > 0 ? MPO_ : round4(M);  // internal row pitch
    static_assert(MP >= M, "row pitch below the map count");
    static constexpr int KK = K * K;
    static constexpr int ROWS = C * KK;   // internal W is [C][K*K][MP] (input map n at n * NS), bias [round4(MP)]
    // NPAD: floats of padding after each input map's K*K rows.  NS / 4 odd puts the 16-B weight vectors
    // of consecutive input maps in distinct bank groups (lanes over input maps, LDS.128: the large
    // net's conv3 delta_in, where NS = 400 hit 2 of 8 groups)
    static constexpr int NPAD = NPAD_, NS = KK * MP + NPAD;
    static_assert(NPAD % 4 == 0, "16-B aligned input-map blocks");
    static constexpr int WFL = round4(C * NS), BFL = round4(MP), BLK = WFL + BFL;
    static constexpr int IN_SZ = C * H * W, OUT_SZ = M * P;
    static constexpr int MT = MT_, TT = TT_, GS = GS_, RB = RB_;
    static constexpr int NB = (H + RB - 1) / RB;
    // delta_in by window-row bands (conv_din3) when PB > 0: PB window rows per band
    static constexpr int PB = PB_;
    static constexpr int HR = PH * KP + K - 1, WR = PW * KP + K - 1;  // input rows/cols that receive delta
    static constexpr int NBAND = PB > 0 ? (PH + PB - 1) / PB : 0;
    static constexpr int BR = PB * KP + K - 1;                        // input rows per band
    static constexpr int HAND = NBAND > 1 ? (NBAND - 1) * (K - 1) * WR * C : 0;  // hand-off floats per image
    // MS < 0: the weight gradient by the generic conv_gw published from registers (lanes over maps)
    static constexpr int MS = MS_;
    static_assert(!UNUSED_, "slot of the removed tensor-core weight-gradient knob");
    // delta_in with the compact shifted-block loop (conv_din3)
    static constexpr bool DIN3 = DIN3_;
    // dense per-window weight gradient (conv_gw_win) with GWIN output maps per thread, run on the
    // warps the delta_in phase leaves idle (0 = off)
    static constexpr int GWIN = GWIN_;
    // dense branch-free per-window delta_in, whole map per lane (conv_din_win)
    static constexpr bool DWIN = DWIN_;
    // forward: the input maps of one item split over NSPL adjacent lanes (partial sums combined
    // with shfl_xor) -- more items for small layers
    static constexpr int NSPL = NSPL_;
    static_assert(NSPL == 1 || (NSPL == 2 && C % 2 == 0), "NSPL 1 or 2");
    static_assert(M % MT == 0, "MT must divide M");
    static_assert(KK % TT == 0, "TT must divide K*K");
    static_assert(RB % KP == 0 || NB == 1, "bands must start on a window row");
    static_assert(PH >= 1 && PW >= 1, "pool larger than the conv output");
    static constexpr int GW_SCRATCH = (GS > 1 ? GS * WFL + GS * M : 0) + BLK;  // floats to assemble gW (+ splits)
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

// Shared-memory carve-up for G images per worker (floats unless noted).
//   S     : images during the forward pass; FC gradient scratch (two halves); the last conv
//           layer's delta_in output (3 conv layers); the images again for conv1's gradient
//   A1..3 : pooled activations, overwritten in place by their partial derivatives
//   HH, Z : hidden FC activations / deltas, logits / output deltas
//   WB    : staged conv weights (prefetched ahead) and conv gradient scratch
template <class Net, int G>
struct SLayout {
    using C1 = typename Net::C1;
    using C2 = typename Net::C2;
    using C3 = typename Net::C3;
    using F1 = typename Net::F1;
    static constexpr bool BIG = BigW<Net>::value;
    static constexpr int WBUF = BIG ? round4(cmax(round4(C1::BLK) + C2::BLK, C1::GW_SCRATCH))
                                    : round4(cmax(cmax(cmax(C1::BLK + (Net::NCONV >= 2 ? C2::BLK : 0), C1::GW_SCRATCH),
                                                       Net::NCONV >= 3 ? 2 * C2::BLK : 0),
                                                  Net::NCONV >= 3 ? C3::BLK : 0));
    static constexpr int SFL = round4(cmax(cmax(G * C1::IN_SZ, Net::SFL),
                                           (Net::NCONV >= 3 && !BIG) ? G * C2::OUT_SZ : 0));
    static constexpr int S = 0;
    static constexpr int A1 = S + SFL;
    static constexpr int A2 = A1 + round4(G * C1::OUT_SZ);
    static constexpr int A3 = A2 + (Net::NCONV >= 2 ? round4(G * C2::OUT_SZ) : 0);
    static constexpr int HH = A3 + (Net::NCONV >= 3 ? round4(G * C3::OUT_SZ) : 0);
    static constexpr int Z = HH + (Net::NFULL >= 2 ? round4(G * F1::OUT) : 0);
    static constexpr int BS = Z + G * kZStride;
    static constexpr int WB = BS + kBiasScratch;
    static constexpr int DPB = (Net::NCONV == 2 && DinPair<Net>::value > 1)
                                   ? (Net::NT / 32 / DinPair<Net>::value) * (DinPair<Net>::value - 1) *
                                         cmax(C2::RB * C2::W, C2::KP * C2::WR) * (C2::C < 32 ? C2::C : 32)
                                   : 0;
    // FWB: the 1-conv nets' (tiny) FC weights + bias, TMA-staged per iteration (read twice, by
    // the forward and by delta_in, instead of twice from L2)
    static constexpr int FWB = (Net::NCONV == 1 && Net::NFULL == 1) ? F1::WFL + F1::BFL : 0;
    static constexpr int FLOATS = WB + WBUF + DPB + FWB;  // DPB: conv_din pair partial bands
    static constexpr int AM1 = 0;  // argmax bytes
    static constexpr int AM2 = AM1 + (C1::KP > 1 ? (G * C1::OUT_SZ + 15) / 16 * 16 : 0);  // pool 1x1: no argmax
    static constexpr int AM3 = AM2 + (Net::NCONV >= 2 ? (G * C2::OUT_SZ + 15) / 16 * 16 : 0);
    static constexpr int AMB = AM3 + (Net::NCONV >= 3 ? (G * C3::OUT_SZ + 15) / 16 * 16 : 0);
    static constexpr int BYTES = kHdrBytes + FLOATS * 4 + AMB;
};

struct KArgs {
    float* params;               // internal layout, shared by all workers (the CHAOS weight store)
    float* partial;              // sync: [slot][pstride] gradient sums
    long long pstride;
    const float* images;         // [n][in]
    const int* labels;           // [n]
    long long n;                 // images in this launch
    unsigned long long* counter; // hogwild work counter (claims in units of images)
    int* latch;                  // device error latch
    double* loss_sum;            // training loss accumulator
    float neg_lr;
    int* claims;                 // optional per-image claim counts
    float* out_loss;             // eval: per-image loss
    unsigned char* out_wrong;    // eval: per-image error flag
    float* out_logits;           // forward: [n][kClasses]
    unsigned long long* ptime;   // CHAOS_TIMING builds: per-CTA clock64 cycles per phase [grid][kPhases]
    unsigned long long* progress; // hogwild: monotonic count of images whose updates are published
    const unsigned long long* ready;  // hogwild from host buffers: images [0, *ready) have landed
    unsigned long long* tctr;     // kTrace: [0] publishes started, [1] publishes done
    long long* trec;              // kTrace: [group][kTraceRec]
    long long stagger;            // kTrace: CTA b starts after b * stagger cycles
    float* tw;                    // kTrace: the weight values each group read, [group][2][pint]
                                  // (internal layout; [.][0] forward reads, [.][1] delta_in reads)
    const struct PavgArgs* pavg;  // hogwild: fused in-kernel cross-replica averaging (null: off)
    long long pavg_round0;        // averaging rounds run by this replica's earlier launches
    long long pavg_rounds;        // rounds in this launch: round t is due once t * pavg_k images are claimed
    long long pavg_k;
    int pavg_comm;                // > 0: the last pavg_comm CTAs of the replica's launch are comm CTAs
                                  // (they run the rounds; the training CTAs never stall on one)
    const KArgs* reps;            // one-GPU replica emulation (REP instantiation): per-replica arguments
    int rep_ctas;                 // ... and CTAs per replica (CTA b runs replica b / rep_ctas)
};

// Fused cross-replica averaging (fused variant): the replicas'
// weight vectors are cut into nslice slices; CTA c of a replica's launch owns slices c, c + ctas, ...
// and, once round t is due, copies its slices of the live weights into its snapshot ring (buffer
// t % kPavgBufs), publishes flag = t; when every peer's flag for the slice has reached t it reads
// all R snapshots (peer memory: NVLink loads through CUDA-IPC mappings; same-device buffers in the
// one-GPU emulation), adds avg - own snapshot to its live weights (red.add, so the hogwild updates
// made meanwhile are kept: "arbitrary order of synchronization", carried across
// replicas) and publishes done = t.  Round t may overwrite a buffer only after every peer's done
// has reached t - kPavgBufs.  Round numbers are absolute (round0 + t) and monotonic across launches,
// so flags are never reset.  Every replica computes the same avg (fixed order q = 0..R-1, then / R),
// so each round preserves the sum of the replicas up to the rounding of the deltas.
constexpr int kPavgMaxR = 8;       // replicas per average
constexpr int kPavgBufs = 4;       // snapshot ring depth
struct PavgArgs {
    int R, rank, nslice, slice_fl;       // slice_fl: floats per slice (multiple of 4)
    long long pint;                      // floats of the weight vector
    int check;                           // debug: checksum every snapshot and verify every read of it
    float* snap[kPavgMaxR];              // replica q's ring [kPavgBufs][nslice * slice_fl]
    unsigned* flag[kPavgMaxR];           // [nslice] last round whose snapshot of the slice q published
    unsigned* done[kPavgMaxR];           // [nslice] last round whose peer snapshots q consumed
    unsigned long long* cks[kPavgMaxR];  // [nslice][kPavgBufs] checksum of q's snapshot (check mode)
    int* latch;                          // check mode: kLatchPavg on a mismatch
    float* dsum;                         // check mode: [pint] sum of this replica's applied deltas
    float* dabs;                         // ... and of their magnitudes
};

// Phase timing (instrumented build only, -DCHAOS_TIMING): thread 0 adds the clock64 cycles
// since the previous mark to slot k; marks sit right after block-wide barriers, so a slot
// holds the wall time of the phase that ends there.
constexpr int kPhases = 20;
#ifdef CHAOS_TIMING
#define PTIME(k)                                                          \
    do {                                                                  \
        if (threadIdx.x == 0 && a.ptime) {                                \
            const long long t_ = clock64();                               \
            a.ptime[blockIdx.x * kPhases + (k)] += t_ - t_last;           \
            t_last = t_;                                                  \
        }                                                                 \
    } while (0)
#else
#define PTIME(k) \
    do {         \
    } while (0)
#endif

// ------------------------------------------------------------------------------------
// PTX helpers: mbarrier, TMA bulk copies global->shared, bulk reduce/copy shared->global
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
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_reduce_add(float* gdst, const float* ssrc, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(float* gdst, const float* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void red_add(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// 16-B vector reduction into global memory (SASS REDG.E.ADD.F32x4): 4 consecutive weights
__device__ __forceinline__ void red_add4(float* p, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// Async loads into shared memory tracked by one mbarrier each (tid 0 issues).
struct Loader {
    uint64_t* bar;
    uint32_t phase;
    // caller: all threads passed a barrier after their last generic access of dst
    __device__ __forceinline__ void issue(float* dst, const float* src, int floats) const {
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, static_cast<uint32_t>(floats) * 4u);
            for (int off = 0; off < floats; off += 16384) {
                const int chunk = (floats - off) > 16384 ? 16384 : (floats - off);
                bulk_g2s(dst + off, src + off, static_cast<uint32_t>(chunk) * 4u, bar);
            }
        }
    }
    __device__ __forceinline__ void wait() {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
};

// Everyone: make generic smem writes visible to the async proxy, then barrier.
__device__ __forceinline__ void sync_for_async() {
    fence_async_smem();
    __syncthreads();
}
// Before reusing a buffer a bulk publish is reading: tid 0 waits for the TMA reads, barrier.
__device__ __forceinline__ void wait_publish_reads() {
    if (threadIdx.x == 0) bulk_wait_read<0>();
    __syncthreads();
}

// Publish `floats` floats of gradient (already scaled by -lr in hogwild mode) from shared
// memory to global offset goff: hogwild = TMA bulk reduce-add into the shared weights;
// sync = TMA bulk copy into this group's slot.  Call after sync_for_async(); tid 0 issues.
template <int MODE>
__device__ __forceinline__ void publish_bulk(const KArgs& a, int slot, int goff, const float* src, int floats) {
    if (threadIdx.x == 0) {
        float* dst = is_hog(MODE) ? a.params + goff : a.partial + static_cast<long long>(slot) * a.pstride + goff;
        for (int off = 0; off < floats; off += 16384) {
            const int chunk = (floats - off) > 16384 ? 16384 : (floats - off);
            if constexpr (is_hog(MODE))
                bulk_reduce_add(dst + off, src + off, static_cast<uint32_t>(chunk) * 4u);
            else
                bulk_s2g(dst + off, src + off, static_cast<uint32_t>(chunk) * 4u);
            if constexpr (MODE == kTrace)  // and the group's own copy
                bulk_s2g(a.partial + static_cast<long long>(slot) * a.pstride + goff + off, src + off,
                         static_cast<uint32_t>(chunk) * 4u);
        }
        bulk_commit();
    }
}
// Direct per-element publish (layers whose gradient does not fit the scratch).
template <int MODE>
__device__ __forceinline__ void publish_elem(const KArgs& a, int slot, int idx, float g_scaled) {
    if constexpr (is_hog(MODE))
        red_add(a.params + idx, g_scaled);
    if constexpr (!is_hog(MODE) || MODE == kTrace)
        a.partial[static_cast<long long>(slot) * a.pstride + idx] = g_scaled;
}

// Vector publish of 4 consecutive gradient entries (already scaled): hogwild = vector reduce
// into the shared weights; sync = plain 16-B store into this group's slot.
template <int MODE>
__device__ __forceinline__ void publish_vec4(const KArgs& a, int slot, int idx, float4 g_scaled) {
    if constexpr (is_hog(MODE))
        red_add4(a.params + idx, g_scaled);
    if constexpr (!is_hog(MODE) || MODE == kTrace)
        *reinterpret_cast<float4*>(a.partial + static_cast<long long>(slot) * a.pstride + idx) = g_scaled;
}

// kTrace event marks (every thread calls them, converged; debug builds of the schedule only).
// Read start: the done count before any thread / TMA read of the layer; read end: the started
// count after the last read.  Publish start: counted before any thread issues a reduction of the
// layer; publish done: counted after every thread's reductions and the bulk ones completed.
__device__ __forceinline__ void trace_read_begin(const KArgs& a, int slot, int k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long v;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.tctr + 1) : "memory");
        a.trec[static_cast<long long>(slot) * kTraceRec + k] = static_cast<long long>(v);
        fence_proxy_async();  // the TMA reads issued next follow the load
    }
    __syncthreads();
}
__device__ __forceinline__ void trace_read_end(const KArgs& a, int slot, int k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_proxy_async();
        __threadfence();
        a.trec[static_cast<long long>(slot) * kTraceRec + k] = static_cast<long long>(atomicAdd(a.tctr, 0ull));
    }
    __syncthreads();
}
__device__ __forceinline__ void trace_pub_begin(const KArgs& a, int slot, int l) {
    __syncthreads();
    if (threadIdx.x == 0) {
        a.trec[static_cast<long long>(slot) * kTraceRec + l * 6] = static_cast<long long>(atomicAdd(a.tctr, 1ull));
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ void trace_pub_end(const KArgs& a, int slot, int l) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        bulk_wait_all<0>();
        fence_proxy_async();
        __threadfence();
        a.trec[static_cast<long long>(slot) * kTraceRec + l * 6 + 1] =
            static_cast<long long>(atomicAdd(a.tctr + 1, 1ull));
    }
    __syncthreads();
}
// kTrace: copy `floats` weight values a group just read into shared memory (staged at src) to
// its record of reads (purpose 0 forward, 1 delta_in) at internal offset goff (thread 0; waits
// until the copy has read src, so the buffer can be refilled right after)
__device__ __forceinline__ void trace_dump(const KArgs& a, int slot, int purpose, int goff, const float* src,
                                           int floats) {
    fence_async_smem();  // generic writes of src (e.g. biases loaded by threads) -> async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_proxy_async();
        float* dst = a.tw + (static_cast<long long>(slot) * 2 + purpose) * a.pstride + goff;
        for (int off = 0; off < floats; off += 16384) {
            const int chunk = (floats - off) > 16384 ? 16384 : (floats - off);
            bulk_s2g(dst + off, src + off, static_cast<uint32_t>(chunk) * 4u);
        }
        bulk_commit();
        bulk_wait_read<0>();
    }
    __syncthreads();
}
#define TR_DUMP(p, goff, src, floats) \
    do { if constexpr (MODE == kTrace) trace_dump(a, slot, (p), (goff), (src), (floats)); } while (0)
#define TR_RB(l, p) \
    do { if constexpr (MODE == kTrace) trace_read_begin(a, slot, (l) * 6 + 2 + 2 * (p)); } while (0)
#define TR_RE(l, p) \
    do { if constexpr (MODE == kTrace) trace_read_end(a, slot, (l) * 6 + 3 + 2 * (p)); } while (0)
#define TR_PB(l) \
    do { if constexpr (MODE == kTrace) trace_pub_begin(a, slot, (l)); } while (0)
#define TR_PE(l) \
    do { if constexpr (MODE == kTrace) trace_pub_end(a, slot, (l)); } while (0)

// A4: p is 16-B aligned; A2: p is 8-B aligned
template <int N, bool A4, bool A2 = false>
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
    } else if constexpr (A2 && N % 2 == 0) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
            const float2 t = *reinterpret_cast<const float2*>(p + 2 * q);
            v[2 * q] = t.x;
            v[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) v[q] = p[q];
    }
}

// Packed FP32 FMA (PTX fma.rn.f32x2, SASS FFMA2, sm_100+): (a0, a1) += (x0, x1) * s, each half the IEEE
// fma of the scalar form (bitwise the same results), one issue slot for both.  Measured
// (scripts/microbench/ffma2_rate.cu): the same 125 FMA/clk/SM peak as FFMA; a conv2-forward-shaped loop
// on 640 threads 88.7 -> 105.9 FMA/clk/SM.
__device__ __forceinline__ void fma_pair(float& a0, float& a1, float x0, float x1, float s) {
    const float2 r = __ffma2_rn(make_float2(x0, x1), make_float2(s, s), make_float2(a0, a1));
    a0 = r.x;
    a1 = r.y;
}

// a[t] += x[t] * s for t in [0, N), packed in pairs (t, t + 1) starting at the first t whose flat
// register-array index is even (par = parity of a[0]'s flat index in its array: every use of an array
// pairs the same elements, so the compiler can keep them in aligned register pairs).  par and the
// indices are compile-time constants after unrolling.
template <int N, bool ON>
__device__ __forceinline__ void fma_row(float* a, const float* x, float s, int par = 0) {
    if constexpr (ON) {
        if (par) a[0] = fmaf(x[0], s, a[0]);
#pragma unroll
        for (int t = 0; t + 1 < N; t += 2)
            if (t + par + 1 < N) fma_pair(a[t + par], a[t + par + 1], x[t + par], x[t + par + 1], s);
        if ((N - par) % 2) a[N - 1] = fmaf(x[N - 1], s, a[N - 1]);
    } else {
#pragma unroll
        for (int t = 0; t < N; ++t) a[t] = fmaf(x[t], s, a[t]);
    }
}

// One tap of the fused conv forward: acc[mt][u * KP + v] += wv[mt] * patch[u + i][v + j] for MT maps and
// the KP x KP conv outputs of a window; two maps per packed FMA (the weight pair as loaded, the patch
// value as the broadcast scalar operand), the last map of an odd MT alone.
template <int MT, int KP, bool ON, int PS>
__device__ __forceinline__ void fma_tap(float (&acc)[MT][KP * KP], const float (&wv)[MT], const float (&patch)[PS][PS],
                                        int i, int j) {
    constexpr int MT2 = ON ? MT / 2 * 2 : 0;
#pragma unroll
    for (int mt = 0; mt < MT2; mt += 2)
#pragma unroll
        for (int u = 0; u < KP; ++u)
#pragma unroll
            for (int v = 0; v < KP; ++v)
                fma_pair(acc[mt][u * KP + v], acc[mt + 1][u * KP + v], wv[mt], wv[mt + 1], patch[u + i][v + j]);
#pragma unroll
    for (int mt = MT2; mt < MT; ++mt)
#pragma unroll
        for (int u = 0; u < KP; ++u)
#pragma unroll
            for (int v = 0; v < KP; ++v) acc[mt][u * KP + v] = fmaf(wv[mt], patch[u + i][v + j], acc[mt][u * KP + v]);
}

// Sums 32 values across the warp's lanes at once (v[k] of every lane -> lane k): 16+8+4+2+1
// shuffles; at each step a lane keeps the half of its values its lane bit selects.
__device__ __forceinline__ float warp_transpose_sum(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
            const float send = up ? v[k] : v[k + o];
            const float keep = up ? v[k + o] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------------------------
// PHASE(conv_fwd) conv -> tanh -> max-pool forward (fused).  One thread item = MT maps x
// one pooled window x one image; the KP*KP conv outputs of the window stay in registers,
// the weights of the MT maps are warp-uniform vector loads from the staged block.
// ------------------------------------------------------------------------------------
// MGF: map groups fastest over the lanes (a warp's lanes read a few windows' patches -- broadcasts,
// distinct banks -- and the map groups' weight vectors) instead of windows fastest (neighbouring
// windows 2 columns apart share banks)
// PL > 0 (image pairs): a warp's lanes = PL windows x 2 images x 32 / (2 PL) map groups, so its patch
// loads come from two images whose offsets differ by an odd-bank-shifting stride -- 2 x PL distinct
// addresses in distinct banks (the windows-fastest order puts 16 windows of one image, 2 columns
// apart, on 16 of the 32 banks: 2-way conflicts, profiles/r4)
// TAIL: the items of the last, partial pass of NT threads are split into single-map sub-items spread
// over all threads (the large net's conv1: 1,352 items on 640 threads left a third pass of 72 items,
// 11% of the threads busy for a whole pass)
template <class L, int NT, bool MGF = false, int PL = 0, bool TAIL = false>
__device__ __forceinline__ void conv_fwd(const float* __restrict__ in, const float* __restrict__ wsm,
                                         float* __restrict__ out, uint8_t* __restrict__ am, int cnt) {
    constexpr int MT = L::MT, KP = L::KP, K = L::K, PW = L::PW, P = L::P, MG = L::M / MT;
    constexpr int PS = KP + K - 1;
    constexpr bool A4 = ((MT % 4 == 0) || (MG == 1)) && (L::MP % 4 == 0);
    constexpr bool A2 = (MT % 2 == 0) && (L::MP % 2 == 0);  // 16-B rows: mg*MT is even
    constexpr int NSPL = L::NSPL, CH = L::C / NSPL;
    static_assert(NT % 32 == 0, "lane pairs never straddle warps");
    static_assert(PL == 0 || (!MGF && NSPL == 1 && 32 % (2 * (PL > 0 ? PL : 1)) == 0), "image-pair lane map");
    constexpr int MGL = PL > 0 ? 32 / (2 * PL) : 1;            // map groups per warp
    constexpr int NPB = PL > 0 ? (P + PL - 1) / PL : 1;         // window blocks
    constexpr int NMB = (MG + MGL - 1) / MGL;                   // map-group blocks
    const int total = PL > 0 ? NMB * ((cnt + 1) / 2) * NPB * 32 : MG * cnt * P * NSPL;
    static_assert(!TAIL || (PL == 0 && !MGF && NSPL == 1), "tail split: the windows-fastest item map");
    const int full = TAIL ? total / NT * NT : total;
    for (int it = threadIdx.x; it < full; it += NT) {
        int half, p, g, mg;
        if constexpr (PL > 0) {
            const int l = it & 31, r = it >> 5;
            half = 0;
            p = (r % NPB) * PL + l % PL;
            g = ((r / NPB) % ((cnt + 1) / 2)) * 2 + (l / PL) % 2;
            mg = (r / NPB / ((cnt + 1) / 2)) * MGL + l / (2 * PL);
            if (p >= P || g >= cnt || mg >= MG) continue;
        } else {
            half = it % NSPL;
            p = MGF ? ((it / NSPL) / MG) % P : (it / NSPL) % P;
            const int t = MGF ? 0 : (it / NSPL) / P;
            g = MGF ? ((it / NSPL) / MG) / P : t % cnt;
            mg = MGF ? (it / NSPL) % MG : t / cnt;
        }
        const int pr = p / PW, pc = p - (p / PW) * PW;
        float acc[MT][KP * KP];
        {
            float b[MT];
            load_vec<MT, A4, A2>(b, wsm + L::WFL + mg * MT);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int q = 0; q < KP * KP; ++q) acc[mt][q] = half == 0 ? b[mt] : 0.f;
        }
        const float* ib = in + g * L::IN_SZ + (pr * KP) * L::W + pc * KP;
        const float* wb = wsm + mg * MT;
#pragma unroll 1
        for (int n = half * CH; n < (half + 1) * CH; ++n) {
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
                    load_vec<MT, A4, A2>(wv, wb + n * L::NS + (i * K + j) * L::MP);
                    fma_tap<MT, KP, (L::FF & 1) != 0>(acc, wv, patch, i, j);
                }
        }
        if constexpr (NSPL == 2) {  // the two halves of an item sit in adjacent lanes
            const unsigned mask = __activemask();
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int q = 0; q < KP * KP; ++q) acc[mt][q] += __shfl_xor_sync(mask, acc[mt][q], 1);
            if (half != 0) continue;
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
            if constexpr (KP > 1) am[o] = static_cast<uint8_t>(arg);
        }
    }
    if constexpr (TAIL) {
        for (int st = threadIdx.x; st < (total - full) * MT; st += NT) {
            const int it = full + st / MT, mt = st % MT;
            const int p = it % P, t = it / P, g = t % cnt, m = (t / cnt) * MT + mt;
            const int pr = p / PW, pc = p - (p / PW) * PW;
            float acc[KP * KP];
#pragma unroll
            for (int q = 0; q < KP * KP; ++q) acc[q] = wsm[L::WFL + m];
            const float* ib = in + g * L::IN_SZ + (pr * KP) * L::W + pc * KP;
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
                        const float w = wsm[n * L::NS + (i * K + j) * L::MP + m];
#pragma unroll
                        for (int u = 0; u < KP; ++u)
#pragma unroll
                            for (int v = 0; v < KP; ++v)
                                acc[u * KP + v] = fmaf(w, patch[u + i][v + j], acc[u * KP + v]);
                    }
            }
            float best = acc[0];
            int arg = 0;
#pragma unroll
            for (int q = 1; q < KP * KP; ++q)
                if (acc[q] > best) {  // first strict maximum wins (R4)
                    best = acc[q];
                    arg = q;
                }
            const int o = g * L::OUT_SZ + m * P + p;
            out[o] = tanhf(best);
            if constexpr (KP > 1) am[o] = static_cast<uint8_t>(arg);
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_fwd_tc2) conv -> tanh -> max-pool forward of a 3x3 / 2x2-pool layer on the
// 5th-generation tensor cores: the implicit GEMM
//   Z_q[row][m] = sum_k A_q[row][k] Wt[k][m],  one 128-row tile per pool phase q, row = (image g,
//   pool window w), k = (input map n, tap i, tap j)
// as tcgen05.mma kind::tf32, M = 128 rows per tile, N = 64 maps, K = 8 per instruction, with
// 3xTF32 operands (x = x_hi + x_lo, terms hi*hi + hi*lo + lo*hi) and the accumulation split into
// two TMEM chains (K < 96 and K >= 96) added in fp32 registers: long tensor-core accumulation
// chains lose accuracy, short ones are more accurate than the FFMA path
// (scripts/microbench/tc_conv2.cu, profiles/r3/tcgen05_conv2.txt).
// Producer warps (all but the last) build the im2col operand slabs (K = 8 per stage) in shared
// memory in the canonical K-major no-swizzle layout (8-row x 16-byte core matrices) -- two stages,
// full / empty mbarriers; one thread of the last warp issues the MMAs and commits each stage back
// to its producers (the two chains' stages alternate, so consecutive MMAs feed independent
// accumulators).  Then warps 0-15 read the accumulators (tcgen05.ld, TMEM lane quarter = warp % 4:
// 32 windows; warp / 4: 16 maps), add the chains and the bias, max-pool over the 4 phase tiles in
// registers (first maximum in phase order, R4), apply tanh and write the pooled activations and
// argmaxes.
// ------------------------------------------------------------------------------------
// round to TF32 (10 explicit mantissa bits), nearest, ties away from zero (= cvt.rna.tf32.f32) with
// two integer ops on the sign-magnitude bits instead of the conversion unit (finite inputs)
__device__ __forceinline__ uint32_t tf32_rna(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
// canonical K-major SWIZZLE_NONE shared-memory matrix descriptor (sm_100 version 1)
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return (uint64_t)((addr >> 4) & 0x3fffu) | ((uint64_t)((lbo_bytes >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo_bytes >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
constexpr int kTcStageBytes = 20480;  // A (hi, lo: 2 x 8 KB) + B (hi, lo: 2 x 2 KB) of one K = 8 slab
constexpr int kTcCols = 512;          // TMEM columns: 2 chains x 4 tiles x 64 maps

// Four operand stages of kTcStageBytes: two at stg (followed by a small offset table) and one each at
// stg2 / stg3 (dead shared-memory regions of the caller; stg3 may be `out`, written only after the
// last MMA has read it).  tcbar: 2 * NS + 1 mbarriers (full[NS], empty[NS], done).
template <class L, int NT, int G>
__device__ __forceinline__ void conv_fwd_tc2(const float* __restrict__ in, const float* __restrict__ wsm,
                                             float* __restrict__ out, uint8_t* __restrict__ am, int cnt,
                                             uint32_t tmem, unsigned char* stg, unsigned char* stg2, unsigned char* stg3,
                                             uint64_t* tcbar, uint32_t& done_phase,
                                             unsigned long long* tslot = nullptr) {
    // tslot (instrumented builds): [0] += producer thread 0's waits for free stages, [1] += the MMA
    // thread's waits for filled stages
    constexpr int K = L::K, KK = L::KK, C = L::C, M = L::M, W = L::W, HW = L::H * L::W, P = L::P, PW = L::PW;
    constexpr int ROWS = G * P * 4, KD = C * KK, NSL = (KD + 15) / 16 * 2, PROW = 256, NPASS = 2;
    constexpr int A_PART = 2 * (PROW / 8) * 128, B_PART = 2 * 8 * 128;
    constexpr int NPW = NT / 32 - 1;  // producer warps; the last warp issues the MMAs
    static_assert(L::KP == 2 && K == 3 && M <= 64 && ROWS <= NPASS * PROW && 2 * A_PART + 2 * B_PART == kTcStageBytes,
                  "3x3 conv, 2x2 pool, <= 64 maps, 4 tiles of 128 rows");
    static_assert(2 * PROW + 64 <= NPW * 32, "one producer thread per A chunk and per B row");
    static_assert(NSL % 2 == 0, "two accumulation chains of equal length");
    constexpr int NS = 4;         // operand stages in flight
    uint64_t* full = tcbar;       // [NS]: producer warps arrive
    uint64_t* empty = tcbar + NS; // [NS]: the MMA commit arrives
    uint64_t* done = tcbar + 2 * NS;  // all MMAs complete
    auto stage = [&](int b) -> unsigned char* { return b < 2 ? stg + b * kTcStageBytes : (b == 2 ? stg2 : stg3); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // k -> input offset n*H*W + i*W + j (-1 beyond K), 16-B aligned groups of 4 (4 consecutive k
    // of one 16-B chunk with one vector load); placed after the two stages
    int* koff = reinterpret_cast<int*>(stg + 2 * kTcStageBytes);
    for (int k = threadIdx.x; k < NSL * 8; k += NT) {
        const int n = k / KK, t = k - n * KK, i = t / K, j = t - i * K;
        koff[k] = k < KD ? n * HW + i * W + j : -1;
    }
    __syncthreads();
    if (warp < NPW) {
        // fixed roles: threads [0, 2*PROW) build A chunk (row r, kc); the next 64 build B rows (both kc)
        const int tid = threadIdx.x;
        const bool isA = tid < 2 * PROW, isB = !isA && tid < 2 * PROW + 64;
        const int r = tid % PROW, kc = (tid / PROW) & 1, mB = tid - 2 * PROW;
        const float* ib = nullptr;
#pragma unroll 1
        for (int f = 0; f < NPASS * NSL; ++f) {
            const int b = f % NS, u = f / NS, h = f / NSL, jj = f % NSL;
            // alternate the two accumulation chains (K < 96, K >= 96) so consecutive stages feed
            // independent accumulators (4 in flight instead of 2)
            const int sl = (jj & 1) ? NSL / 2 + (jj >> 1) : (jj >> 1);
            if (jj == 0 && isA) {  // this pass's row: tile = pool phase, row = (image, window) -> patch origin
                const int ph = 2 * h + r / 128, Rw = r % 128, g = Rw / P;
                ib = nullptr;
                if (Rw < G * P && g < cnt) {
                    const int w = Rw % P;
                    ib = in + g * L::IN_SZ + (2 * (w / PW) + (ph >> 1)) * W + 2 * (w % PW) + (ph & 1);
                }
            }
#ifdef CHAOS_TIMING
            const long long tw0 = clock64();
#endif
            if (u > 0) mbar_wait(empty + b, static_cast<uint32_t>(u - 1) & 1u);
#ifdef CHAOS_TIMING
            if (threadIdx.x == 0 && tslot) tslot[0] += clock64() - tw0;
#endif
            unsigned char* st = stage(b);
            if (isA) {
                const int4 ko = reinterpret_cast<const int4*>(koff)[sl * 2 + kc];
                const int kq[4] = {ko.x, ko.y, ko.z, ko.w};
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float v = (ib && kq[q] >= 0) ? ib[kq[q]] : 0.f;
                    hi[q] = tf32_rna(v);
                    lo[q] = tf32_rna(v - __uint_as_float(hi[q]));
                }
                const int off = kc * (PROW / 8) * 128 + (r >> 3) * 128 + (r & 7) * 16;
                *reinterpret_cast<uint4*>(st + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(st + A_PART + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            } else if (isB) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t hi[4], lo[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int k = sl * 8 + c * 4 + q;
                        static_assert(L::NPAD == 0, "tensor-core B operand from [C*K*K][MP] rows");
                        const float v = (mB < M && k < KD) ? wsm[k * L::MP + mB] : 0.f;
                        hi[q] = tf32_rna(v);
                        lo[q] = tf32_rna(v - __uint_as_float(hi[q]));
                    }
                    const int off = c * 8 * 128 + (mB >> 3) * 128 + (mB & 7) * 16;
                    *reinterpret_cast<uint4*>(st + 2 * A_PART + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(st + 2 * A_PART + B_PART + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
            fence_async_smem();  // these generic writes -> the tensor core's (async proxy) reads
            __syncwarp();
            if (lane == 0) mbar_arrive(full + b);
        }
    } else if (lane == 0) {
        // kind::tf32, D f32, A and B TF32, both K-major, N = 64, M = 128
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
#pragma unroll 1
        for (int f = 0; f < NPASS * NSL; ++f) {
            const int b = f % NS, u = f / NS, h = f / NSL, jj = f % NSL;
            // alternate the two accumulation chains (K < 96, K >= 96) so consecutive stages feed
            // independent accumulators (4 in flight instead of 2)
            const int sl = (jj & 1) ? NSL / 2 + (jj >> 1) : (jj >> 1);
#ifdef CHAOS_TIMING
            const long long tw0 = clock64();
#endif
            mbar_wait(full + b, static_cast<uint32_t>(u) & 1u);
#ifdef CHAOS_TIMING
            if (tslot) tslot[1] += clock64() - tw0;
#endif
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sb = smem_u32(stage(b));
            const int chain = sl < NSL / 2 ? 0 : 1, first = (sl % (NSL / 2)) == 0;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const uint32_t d = tmem + chain * 256 + (2 * h + t) * 64;
                const uint32_t a0 = sb + t * 16 * 128, a1 = a0 + A_PART;
                const uint32_t b0 = sb + 2 * A_PART, b1 = b0 + B_PART;
                const uint32_t alb = (PROW / 8) * 128, blb = 8 * 128;
                umma_tf32(d, umma_sdesc(a0, alb, 128), umma_sdesc(b0, blb, 128), idesc, first ? 0u : 1u);
                umma_tf32(d, umma_sdesc(a0, alb, 128), umma_sdesc(b1, blb, 128), idesc, 1u);
                umma_tf32(d, umma_sdesc(a1, alb, 128), umma_sdesc(b0, blb, 128), idesc, 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(empty + b))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(done))
                     : "memory");
    }
    mbar_wait(done, done_phase);
    done_phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef CHAOS_TIMING
    const long long te0 = clock64();
#endif
    if (warp < 16) {  // TMEM lane quarter = warp % 4 (windows), 16 output maps per warp = warp / 4
        const int qd = warp & 3, cb = warp >> 2;
        const int Rw = 32 * qd + lane, g = Rw / P, w = Rw % P;
        const bool valid = Rw < G * P && g < cnt;
#pragma unroll 1
        for (int c0 = 16 * cb; c0 < 16 * cb + 16; c0 += 8) {
            uint32_t v[4][2][8];  // [phase tile][chain][column]
            const uint32_t ta = tmem + (static_cast<uint32_t>(32 * qd) << 16) + c0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int ch = 0; ch < 2; ++ch)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(v[q][ch][0]), "=r"(v[q][ch][1]), "=r"(v[q][ch][2]), "=r"(v[q][ch][3]),
                                   "=r"(v[q][ch][4]), "=r"(v[q][ch][5]), "=r"(v[q][ch][6]), "=r"(v[q][ch][7])
                                 : "r"(ta + ch * 256 + q * 64));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int m = c0 + c;
                const float bm = m < M ? wsm[L::WFL + m] : 0.f;
                float best = (__uint_as_float(v[0][0][c]) + __uint_as_float(v[0][1][c])) + bm;
                int arg = 0;
#pragma unroll
                for (int q = 1; q < 4; ++q) {  // first strict maximum in phase order wins (R4)
                    const float zq = (__uint_as_float(v[q][0][c]) + __uint_as_float(v[q][1][c])) + bm;
                    if (zq > best) {
                        best = zq;
                        arg = q;
                    }
                }
                if (valid && m < M) {
                    const int o = g * L::OUT_SZ + m * P + w;
                    out[o] = tanhf(best);
                    am[o] = static_cast<uint8_t>(arg);
                }
            }
        }
    }
#ifdef CHAOS_TIMING
    if (threadIdx.x == 0 && tslot) tslot[2] += clock64() - te0;  // the epilogue (warp 0's view)
#endif
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// ------------------------------------------------------------------------------------
// PHASE(conv_fwd_slab) conv -> tanh -> max-pool forward with the weights streamed through
// shared memory one input map at a time (a layer too large to stage whole: the Table I large
// net's conv3, 864 KB).  W[n][*][*] (K*K*MP floats, contiguous in the internal layout) is TMA
// bulk-copied into a ring of 3 buffers, two maps ahead; all threads walk the input maps in
// lockstep (one barrier per map).  Item = MT maps x one pooled window (G = 1 images), its KP*KP
// conv outputs in registers, as in conv_fwd.  ring: 3 * K*K*MP floats of dead shared memory.
// ------------------------------------------------------------------------------------
template <class L, int NT>
__device__ __forceinline__ void conv_fwd_slab(const float* __restrict__ in, const float* __restrict__ wg,
                                              float* __restrict__ out, uint8_t* __restrict__ am, float* ring,
                                              Loader& R0, Loader& R1, Loader& R2) {
    constexpr int MT = L::MT, KP = L::KP, K = L::K, KK = L::KK, PW = L::PW, P = L::P, MG = L::M / MT;
    static_assert(L::NPAD == 0, "conv_fwd_slab streams [K*K][MP] slabs");
    constexpr int PS = KP + K - 1, SLAB = KK * L::MP, ITEMS = MG * P;
    static_assert(ITEMS <= NT, "one item per thread");
    static_assert((SLAB * 4) % 16 == 0 && MT % 4 == 0, "16-B slabs, vector weight loads");
    Loader* R[3] = {&R0, &R1, &R2};
    R0.issue(ring, wg, SLAB);
    R1.issue(ring + SLAB, wg + SLAB, SLAB);
    R2.issue(ring + 2 * SLAB, wg + 2 * SLAB, SLAB);
    const int it = threadIdx.x;
    const bool act = it < ITEMS;
    const int p = act ? it % P : 0;
    const int mg = act ? it / P : 0;
    const int pr = p / PW, pc = p - (p / PW) * PW;
    float acc[MT][KP * KP];
    {
        float b[MT];
        load_vec<MT, true>(b, wg + L::WFL + mg * MT);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int q = 0; q < KP * KP; ++q) acc[mt][q] = b[mt];
    }
    const float* ib = in + (pr * KP) * L::W + pc * KP;
#pragma unroll 1
    for (int n = 0; n < L::C; ++n) {
        R[n % 3]->wait();
        const float* wb = ring + (n % 3) * SLAB + mg * MT;
        if (act) {
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
                    load_vec<MT, true>(wv, wb + (i * K + j) * L::MP);
                    fma_tap<MT, KP, (L::FF & 1) != 0>(acc, wv, patch, i, j);
                }
        }
        if (n + 3 < L::C) {
            sync_for_async();  // every thread is done with this buffer
            R[n % 3]->issue(ring + (n % 3) * SLAB, wg + static_cast<long long>(n + 3) * SLAB, SLAB);
        }
    }
    if (act) {
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
            const int o = (mg * MT + mt) * P + p;
            out[o] = tanhf(best);
            am[o] = static_cast<uint8_t>(arg);
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_gw) conv weight gradient.  dp[g][m][pp] = dL/dz at the argmax of pooled
// output pp (the pool routes the delta there and nowhere else):
//   gW[n][i][j][m] = sum_g sum_pp dp[g][m][pp] * in[g][n][r(pp)+i][c(pp)+j],  gb[m] = sum dp
// One thread item = (input map n, output map m, tap group, split of the (g, pp) range),
// n fastest so a warp's lanes gather from different maps of the same window (map stride
// H*W is odd: conflict-free) and dp/argmax loads are broadcasts.  With SCRATCH the sums,
// scaled by `sc` (-lr in hogwild), are assembled in shared memory in the weight store's
// layout (splits reduced in a fixed order) and published with one bulk op; otherwise
// each element is published directly.
// ------------------------------------------------------------------------------------
#ifndef CHAOS_GW_UNROLL  // conv_gw: unroll of the (image, window) loop (code size vs. the 32 KB L1.5 I-cache)
#define CHAOS_GW_UNROLL 4
#endif
template <class L, int NT, int MODE, bool SCRATCH>
__device__ __forceinline__ void conv_gw(const KArgs& a, int slot, const float* __restrict__ in,
                                        const float* __restrict__ dp, const uint8_t* __restrict__ am,
                                        float* __restrict__ scr, int woff, int cnt, float sc) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int TT = L::TT, TG = KK / TT, GS = L::GS;
    constexpr int HW = L::H * L::W;
    static_assert(GS == 1 || SCRATCH, "split sums need the scratch");
    static_assert(!SCRATCH || L::NPAD == 0, "the scratch block is assembled without input-map padding");
    float* fin = scr + (GS > 1 ? GS * L::WFL : 0);  // final [WFL][BFL] block
    const int span = cnt * P;
    const int total = C * M * TG * GS;
    for (int it = threadIdx.x; it < total; it += NT) {
        // SCRATCH: n fastest (gathers from different maps, conflict-free); direct publish: m
        // fastest, so a warp's reductions hit consecutive weights (coalesced) and its gathers
        // come from one map (at most KP*KP distinct addresses per load)
        const int n = SCRATCH ? it % C : (it / M) % C;
        int r = SCRATCH ? it / C : it / (M * C);
        const int m = SCRATCH ? r % M : it % M;
        if constexpr (SCRATCH) r /= M;
        const int tg = r % TG;
        const int s = r / TG;
        const int q0 = (GS == 1) ? 0 : (span * s) / GS;
        const int q1 = (GS == 1) ? span : (span * (s + 1)) / GS;
        float acc[TT];
#pragma unroll
        for (int t = 0; t < TT; ++t) acc[t] = 0.f;
        float accb = 0.f;
        int g = q0 / P;
        int pp = q0 - g * P;
        const float* ing = in + g * L::IN_SZ + n * HW;
        const float* dpg = dp + g * L::OUT_SZ + m * P;
        const uint8_t* amg = am + g * L::OUT_SZ + m * P;
        constexpr int GWU = CHAOS_GW_UNROLL;
#pragma unroll GWU
        for (int q = q0; q < q1; ++q) {
            const float d = dpg[pp];
            int arg = 0;
            if constexpr (KP > 1) arg = amg[pp];
            const int pr = pp / PW, pc = pp - (pp / PW) * PW;
            const float* base = ing + (pr * KP + arg / KP) * L::W + pc * KP + arg % KP;
            float xv[TT];
#pragma unroll
            for (int t = 0; t < TT; ++t) {
                const int tap = tg * TT + t;
                xv[t] = base[(tap / K) * L::W + (tap % K)];
            }
            fma_row<TT, (L::FF & 16) != 0>(acc, xv, d);
            accb += d;
            if (++pp == P) {
                pp = 0;
                ++g;
                ing += L::IN_SZ;
                dpg += L::OUT_SZ;
                amg += L::OUT_SZ;
            }
        }
#pragma unroll
        for (int t = 0; t < TT; ++t) {
            const int widx = n * L::NS + (tg * TT + t) * L::MP + m;
            if constexpr (!SCRATCH)
                publish_elem<MODE>(a, slot, woff + widx, sc * acc[t]);
            else if constexpr (GS == 1)
                fin[widx] = sc * acc[t];
            else
                scr[s * L::WFL + widx] = acc[t];
        }
        if constexpr (GS == 1) {
            if (n == 0 && tg == 0) {
                if constexpr (!SCRATCH)
                    publish_elem<MODE>(a, slot, woff + L::WFL + m, sc * accb);
                else
                    fin[L::WFL + m] = sc * accb;
            }
        } else {
            if (n == 0 && tg == 0) scr[GS * L::WFL + L::BLK + s * M + m] = accb;  // bias partial of split s
        }
    }
    if constexpr (SCRATCH) {
        if constexpr (GS > 1) {
            __syncthreads();
            for (int e = threadIdx.x; e < L::ROWS * M; e += NT) {
                const int m = e % M;
                const int row = e / M;
                const int widx = (row / KK) * L::NS + (row % KK) * L::MP + m;
                float s = 0.f;
#pragma unroll
                for (int k = 0; k < GS; ++k) s += scr[k * L::WFL + widx];
                fin[widx] = sc * s;
            }
            for (int m = threadIdx.x; m < M; m += NT) {  // bias: the splits' partial sums, fixed order
                float s = 0.f;
#pragma unroll
                for (int k = 0; k < GS; ++k) s += scr[GS * L::WFL + L::BLK + k * M + m];
                fin[L::WFL + m] = sc * s;
            }
        }
        if constexpr (L::MP > M) {  // padding columns of the block publish zeros
            for (int e = threadIdx.x; e < (L::ROWS + 1) * (L::MP - M); e += NT)
                fin[(e / (L::MP - M)) * L::MP + M + e % (L::MP - M)] = 0.f;
        }
        sync_for_async();
        publish_bulk<MODE>(a, slot, woff, fin, L::BLK);
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_gw_m) conv weight gradient, argmax-routed, lanes over output maps, NPT input maps
// per thread (KP == 2):
//   gW[n][i][j][m] = sum_g sum_pp dp[g][m][pp] * in[g][n][2pr(pp)+a+i][2pc(pp)+b+j],  gb[m] = sum dp
// where (a, b) is the argmax phase of (g, m, pp).  One (d, phase) load per window serves the NPT
// input maps' K*K gathers (each a load of <= 4 distinct words per warp: one wavefront); the
// window columns are unrolled so the gather offsets are immediates plus the phase offset.
// Fixed (g, pp) order per weight (deterministic); direct coalesced publish from registers.
// ------------------------------------------------------------------------------------
// Runs on warps [W0, W0 + NWARP) (all warps by default) so it can overlap another phase.
template <class L, int NT, int MODE, int NPT, int W0 = 0, int NWARP = NT / 32>
__device__ __forceinline__ void conv_gw_m(const KArgs& a, int slot, const float* __restrict__ in,
                                          const float* __restrict__ dp, const uint8_t* __restrict__ am, int woff,
                                          int cnt, float sc) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int W = L::W, HW = L::H * L::W;
    constexpr int NQ = C / NPT;
    static_assert(KP == 2 && C % NPT == 0, "2x2 pooling, NPT divides C");
    const int tid = static_cast<int>(threadIdx.x) - W0 * 32;
    if (tid < 0 || tid >= NWARP * 32) return;
    for (int it = tid; it < M * NQ; it += NWARP * 32) {
        const int m = it % M;
        const int n0 = (it / M) * NPT;
        float acc[NPT][KK];
        float accb = 0.f;
#pragma unroll
        for (int k = 0; k < NPT; ++k)
#pragma unroll
            for (int t = 0; t < KK; ++t) acc[k][t] = 0.f;
#pragma unroll 1
        for (int g = 0; g < cnt; ++g) {
            const float* dpg = dp + g * L::OUT_SZ + m * P;
            const uint8_t* amg = am + g * L::OUT_SZ + m * P;
            const float* ing = in + g * L::IN_SZ + n0 * HW;
#pragma unroll 1
            for (int pr = 0; pr < PH; ++pr) {
                const float* inr = ing + pr * KP * W;
                float dv[PW];
                int av[PW];
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    dv[pc] = dpg[pr * PW + pc];
                    av[pc] = amg[pr * PW + pc];
                }
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    const float d = dv[pc];
                    const float* base = inr + pc * KP + (av[pc] >> 1) * W + (av[pc] & 1);
                    accb += d;
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        float xv[KK];
#pragma unroll
                        for (int t = 0; t < KK; ++t) xv[t] = base[k * HW + (t / K) * W + (t % K)];
                        fma_row<KK, (L::FF & 8) != 0>(acc[k], xv, d, (k * KK) & 1);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NPT; ++k)
#pragma unroll
            for (int t = 0; t < KK; ++t) publish_elem<MODE>(a, slot, woff + (n0 + k) * L::NS + t * L::MP + m, sc * acc[k][t]);
        if (n0 == 0) publish_elem<MODE>(a, slot, woff + L::WFL + m, sc * accb);
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_gw_win) conv weight gradient, dense per pooling window, branch-free (KP == 2):
//   gW[n][i][j][m] = sum_g sum_w sum_{phase q} Dz_q[g][m][w] * in[g][n][2pr+a(q)+i][2pc+b(q)+j]
// where Dz_q = d[g][m][w] if the argmax of (g, m, w) has phase q, else 0 (4x the argmax-sparse
// MACs, but no per-window branch).  Thread tile = (input map n, NM consecutive output maps);
// per window the (KP+K-1)^2 input block of n is loaded once and reused by the NM maps x 4
// phases x K*K taps from registers.  Runs on warps [W0, W0 + NWARP) so it can overlap a
// latency-bound phase on the other warps.  No shared-memory scratch: each thread publishes
// its K*K x NM block directly, 16-B vector reductions into the shared weights (hogwild) or
// stores into its group's slot (sync) -- NM % 4 == 0.  Fixed (g, w, q) order (deterministic).
// Bias gradient: tiles with n == 0.
// ------------------------------------------------------------------------------------
template <class L, int NT, int MODE, int NM, int W0, int NWARP>
__device__ __forceinline__ void conv_gw_win(const KArgs& a, int slot, const float* __restrict__ in,
                                            const float* __restrict__ dp, const uint8_t* __restrict__ am, int woff,
                                            int cnt, float sc, const float4* __restrict__ dq4 = nullptr) {
    // dq4 (optional): the phase-expanded delta, dq4[g][m][w] = d at component phase, 0 elsewhere
    // (built once per iteration), replacing the per-thread (d, phase) selects
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int W = L::W, HW = L::H * L::W, BS = KP + K - 1;
    constexpr int NG = (M + NM - 1) / NM, TILES = C * NG;
    static_assert(KP == 2 && NM % 4 == 0 && M % 4 == 0, "2x2 pooling, vector publish");
    const int tid = static_cast<int>(threadIdx.x) - W0 * 32;
    if (tid < 0 || tid >= NWARP * 32) return;
    for (int tile = tid; tile < TILES; tile += NWARP * 32) {
        const int n = tile % C;
        const int m0 = (tile / C) * NM;
        float acc[NM][KK];
        float accb[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            accb[q] = 0.f;
#pragma unroll
            for (int t = 0; t < KK; ++t) acc[q][t] = 0.f;
        }
#pragma unroll 1
        for (int g = 0; g < cnt; ++g) {
            const float* ing = in + g * L::IN_SZ + n * HW;
            const float* dpg = dp + g * L::OUT_SZ;
            const uint8_t* amg = am + g * L::OUT_SZ;
#pragma unroll 1
            for (int w = 0; w < P; ++w) {
                const int pr = w / PW, pc = w - (w / PW) * PW;
                float blk[BS][BS];
#pragma unroll
                for (int u = 0; u < BS; ++u)
#pragma unroll
                    for (int v = 0; v < BS; ++v) blk[u][v] = ing[(pr * KP + u) * W + pc * KP + v];
#pragma unroll
                for (int q = 0; q < NM; ++q) {
                    const int m = m0 + q;
                    const bool vm = (NG * NM == M) || m < M;
                    float dqv[4];
                    if (dq4) {
                        const float4 t4 = vm ? dq4[g * L::OUT_SZ + m * P + w] : make_float4(0.f, 0.f, 0.f, 0.f);
                        dqv[0] = t4.x;
                        dqv[1] = t4.y;
                        dqv[2] = t4.z;
                        dqv[3] = t4.w;
                        accb[q] += (t4.x + t4.y) + (t4.z + t4.w);  // exactly d: three of them are 0
                    } else {
                        const float d = vm ? dpg[m * P + w] : 0.f;
                        const int ph = vm ? amg[m * P + w] : 0;
                        accb[q] += d;
#pragma unroll
                        for (int k = 0; k < 4; ++k) dqv[k] = (ph == k) ? d : 0.f;
                    }
#pragma unroll
                    for (int aa = 0; aa < KP; ++aa)
#pragma unroll
                        for (int bb = 0; bb < KP; ++bb) {
                            const float dq = dqv[aa * KP + bb];
#pragma unroll
                            for (int i = 0; i < K; ++i)
#pragma unroll
                                for (int j = 0; j < K; ++j)
                                    acc[q][i * K + j] = fmaf(dq, blk[aa + i][bb + j], acc[q][i * K + j]);
                        }
                }
            }
        }
        // publish: internal row (n*KK + t), columns m0 .. m0+NM-1 (16-B aligned groups)
#pragma unroll
        for (int t = 0; t < KK; ++t)
#pragma unroll
            for (int q4 = 0; q4 < NM; q4 += 4)
                if ((NG * NM == M) || m0 + q4 < M)
                    publish_vec4<MODE>(a, slot, woff + n * L::NS + t * L::MP + m0 + q4,
                                       make_float4(sc * acc[q4][t], sc * acc[q4 + 1][t], sc * acc[q4 + 2][t],
                                                   sc * acc[q4 + 3][t]));
        if (n == 0)
#pragma unroll
            for (int q4 = 0; q4 < NM; q4 += 4)
                if ((NG * NM == M) || m0 + q4 < M)
                    publish_vec4<MODE>(a, slot, woff + L::WFL + m0 + q4,
                                       make_float4(sc * accb[q4], sc * accb[q4 + 1], sc * accb[q4 + 2],
                                                   sc * accb[q4 + 3]));
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_gw_wt) conv_gw_win for large kernels (KP == 2): the K*K taps are split into
// groups of KR tap rows so a thread's accumulators (NM maps x KR*K taps) and input block
// ((KR+1) x (K+1)) fit in registers.  Tile = (map group of NM, input map n, tap-row group), map
// group fastest: a warp's lanes share n (input-block loads are broadcasts) and publish
// consecutive 16-B weight groups (coalesced vector reductions).  Dense per window (4 phases,
// one of them the argmax), fixed order (deterministic).  Bias gradient: tiles with n == 0, tr == 0.
// ------------------------------------------------------------------------------------
template <class L, int NT, int MODE, int NM, int KR>
__device__ __forceinline__ void conv_gw_wt(const KArgs& a, int slot, const float* __restrict__ in,
                                           const float* __restrict__ dp, const uint8_t* __restrict__ am, int woff,
                                           int cnt, float sc) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int W = L::W, HW = L::H * L::W, BR = KP + KR - 1, BC = KP + K - 1;
    constexpr int NG = M / NM, NTR = K / KR, TILES = NG * C * NTR;
    static_assert(KP == 2 && NM % 4 == 0 && M % NM == 0 && K % KR == 0, "2x2 pooling, vector publish");
    for (int tile = threadIdx.x; tile < TILES; tile += NT) {
        const int mg = tile % NG;
        const int n = (tile / NG) % C;
        const int tr = tile / (NG * C);
        const int m0 = mg * NM;
        float acc[NM][KR * K];
        float accb[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            accb[q] = 0.f;
#pragma unroll
            for (int t = 0; t < KR * K; ++t) acc[q][t] = 0.f;
        }
#pragma unroll 1
        for (int g = 0; g < cnt; ++g) {
            const float* ing = in + g * L::IN_SZ + n * HW + tr * KR * W;
            const float* dpg = dp + g * L::OUT_SZ + m0 * P;
            const uint8_t* amg = am + g * L::OUT_SZ + m0 * P;
#pragma unroll 1
            for (int w = 0; w < P; ++w) {
                const int pr = w / PW, pc = w - (w / PW) * PW;
                float blk[BR][BC];
#pragma unroll
                for (int u = 0; u < BR; ++u)
#pragma unroll
                    for (int v = 0; v < BC; ++v) blk[u][v] = ing[(pr * KP + u) * W + pc * KP + v];
                if constexpr ((L::FF & 64) && NM % 2 == 0) {
                    // two maps per packed FMA: the pair of masked deltas times the block value (broadcast
                    // operand); every accumulator still sums (g, w, phase) in the scalar loop's order
                    float dv[NM];
                    int pv[NM];
#pragma unroll
                    for (int q = 0; q < NM; ++q) {
                        dv[q] = dpg[q * P + w];
                        pv[q] = amg[q * P + w];
                        accb[q] += dv[q];
                    }
#pragma unroll
                    for (int aa = 0; aa < KP; ++aa)
#pragma unroll
                        for (int bb = 0; bb < KP; ++bb) {
                            float dq[NM];
#pragma unroll
                            for (int q = 0; q < NM; ++q) dq[q] = (pv[q] == aa * KP + bb) ? dv[q] : 0.f;
#pragma unroll
                            for (int i = 0; i < KR; ++i)
#pragma unroll
                                for (int j = 0; j < K; ++j)
#pragma unroll
                                    for (int q = 0; q < NM; q += 2)
                                        fma_pair(acc[q][i * K + j], acc[q + 1][i * K + j], dq[q], dq[q + 1],
                                                 blk[aa + i][bb + j]);
                        }
                } else {
#pragma unroll
                    for (int q = 0; q < NM; ++q) {
                        const float d = dpg[q * P + w];
                        const int ph = amg[q * P + w];
                        accb[q] += d;
#pragma unroll
                        for (int aa = 0; aa < KP; ++aa)
#pragma unroll
                            for (int bb = 0; bb < KP; ++bb) {
                                const float dq = (ph == aa * KP + bb) ? d : 0.f;
#pragma unroll
                                for (int i = 0; i < KR; ++i)
#pragma unroll
                                    for (int j = 0; j < K; ++j)
                                        acc[q][i * K + j] = fmaf(dq, blk[aa + i][bb + j], acc[q][i * K + j]);
                            }
                    }
                }
            }
        }
#pragma unroll
        for (int t = 0; t < KR * K; ++t)
#pragma unroll
            for (int q4 = 0; q4 < NM; q4 += 4)
                publish_vec4<MODE>(a, slot, woff + n * L::NS + (tr * KR * K + t) * L::MP + m0 + q4,
                                   make_float4(sc * acc[q4][t], sc * acc[q4 + 1][t], sc * acc[q4 + 2][t],
                                               sc * acc[q4 + 3][t]));
        if (n == 0 && tr == 0)
#pragma unroll
            for (int q4 = 0; q4 < NM; q4 += 4)
                publish_vec4<MODE>(a, slot, woff + L::WFL + m0 + q4,
                                   make_float4(sc * accb[q4], sc * accb[q4 + 1], sc * accb[q4 + 2], sc * accb[q4 + 3]));
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_din) partial derivatives of the previous layer:
//   dout[g][n][y][x] = (1 - in^2) * sum_m sum_pp [tap in range] W[n][y-r][x-c][m] dp[g][m][pp]
// One warp per (image g, band of RB input rows, 32 input maps); lanes over n.  The windows
// that reach the band are a static set relative to the band, the argmax branch is uniform
// across the warp, and every (tap, window) pair lands in a compile-time register of the
// band accumulator: exactly the argmax-sparse MACs, no atomics, no divergence.  W is the
// staged (pre-update) snapshot (SURVEY C-9).  dout may alias in (in place).
// ------------------------------------------------------------------------------------
// MSPLIT > 1: each (image, band, 32 maps) task is split over a group of MSPLIT warps, warp k of the
// group taking output maps [k*M/MSPLIT, (k+1)*M/MSPLIT); warps 1.. leave their partial bands in
// pbuf ([NT/32/MSPLIT][MSPLIT-1][RB*W][min(C,32)] floats, lane-fastest) and warp 0 adds them in order
// (deterministic) and writes -- MSPLIT times the warp tasks for layers with few (the medium
// net's conv2: 20 tasks for 16 warps).  Named barrier 1 + group.
template <class L, int NT, int MSPLIT = 1>
__device__ __forceinline__ void conv_din(const float* __restrict__ wsm, const float* __restrict__ dp,
                                         const uint8_t* __restrict__ am, const float* in, float* dout, int cnt,
                                         float* __restrict__ pbuf = nullptr) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int HW = L::H * L::W, RB = L::RB, NB = L::NB;
    constexpr int R2 = (NB == 1) ? 0 : RB / KP;       // window rows per band step
    constexpr int DLO = (NB == 1) ? 0 : -((KP + K - 2) / KP);
    constexpr int DHI = (NB == 1) ? PH - 1 : (RB - 1) / KP;
    constexpr int NWR = DHI - DLO + 1;                // window rows that can reach a band
    constexpr int NCW = (C + 31) / 32;
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int total = cnt * NB * NCW;
    constexpr bool PAIR = MSPLIT > 1;
    static_assert(!PAIR || (NW % MSPLIT == 0 && NW / MSPLIT <= 15), "warp groups, named barriers 1..15");
    const int half = PAIR ? (warp % MSPLIT) : 0;  // the warp's part of the map loop
    const int grp = warp / MSPLIT;
    const int m_lo = half * M / MSPLIT, m_hi = (half + 1) * M / MSPLIT;
    for (int vw = PAIR ? grp : warp; vw < total; vw += PAIR ? NW / MSPLIT : NW) {
        const int cw = vw % NCW;
        const int t = vw / NCW;
        const int b = t % NB;
        const int g = t / NB;
        const int n0 = cw * 32 + lane;
        if (!PAIR && n0 >= C) continue;  // (pairs: every lane reaches the pair barriers)
        const bool act = n0 < C;
        const int n = act ? n0 : 0;
        float acc[RB][L::W];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < L::W; ++c) acc[r][c] = 0.f;
        const float* wn = wsm + n * L::NS;
        const float* dpg = dp + g * L::OUT_SZ;
        const uint8_t* amg = am + g * L::OUT_SZ;
        const int pr0 = b * R2;
#ifndef CHAOS_DIN_V2  // conv_din: weights of two maps per 8-B load (lanes over input maps hit 4 banks
#define CHAOS_DIN_V2 0   // with scalar loads: 5-way conflicts on the medium net) and a switch on the phase
#endif
        constexpr bool V2 = CHAOS_DIN_V2 && (L::MP % 2 == 0) && (M % (2 * MSPLIT) == 0);
        float w2n[V2 ? KK : 1];  // the second map's weights of the pair (V2)
        (void)w2n;
#pragma unroll 1
        for (int m = m_lo; m < m_hi; ++m) {
            float w[KK];
            if constexpr (V2) {
                if (((m - m_lo) & 1) == 0) {
#pragma unroll
                    for (int tp = 0; tp < KK; ++tp) {
                        const float2 t2 = *reinterpret_cast<const float2*>(wn + tp * L::MP + m);
                        w[tp] = t2.x;
                        w2n[tp] = t2.y;
                    }
                } else {
#pragma unroll
                    for (int tp = 0; tp < KK; ++tp) w[tp] = w2n[tp];
                }
            } else {
#pragma unroll
                for (int tp = 0; tp < KK; ++tp) w[tp] = wn[tp * L::MP + m];
            }
#ifndef CHAOS_DIN_LATE_D  // conv_din: load each window's (delta, phase) right before its use (fewer registers)
#define CHAOS_DIN_LATE_D 1
#endif
            constexpr bool LATE = CHAOS_DIN_LATE_D;
            float dv[LATE ? 1 : NWR][PW];
            int av[LATE ? 1 : NWR][PW];
            if constexpr (!LATE) {
#pragma unroll
                for (int dr = 0; dr < NWR; ++dr) {
                    const int pr = pr0 + DLO + dr;
                    const bool ok = pr >= 0 && pr < PH;
#pragma unroll
                    for (int pc = 0; pc < PW; ++pc) {
                        const int o = m * P + (ok ? pr : 0) * PW + pc;
                        dv[dr][pc] = ok ? dpg[o] : 0.f;
                        av[dr][pc] = ok ? static_cast<int>(amg[o]) : -1;
                    }
                }
            }
#pragma unroll
            for (int dr = 0; dr < NWR; ++dr) {
                const int dlt = DLO + dr;
                if constexpr (LATE) {
                    const int pr = pr0 + DLO + dr;
                    if (pr < 0 || pr >= PH) continue;  // warp-uniform
#pragma unroll
                    for (int pc = 0; pc < PW; ++pc) {
                        dv[0][pc] = dpg[m * P + pr * PW + pc];
                        av[0][pc] = static_cast<int>(amg[m * P + pr * PW + pc]);
                    }
                }
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    const int arg = av[LATE ? 0 : dr][pc];
                    const float d = dv[LATE ? 0 : dr][pc];
                    auto add_phase = [&](auto phc) {
                        constexpr int ph = decltype(phc)::value;
#pragma unroll
                        for (int i = 0; i < K; ++i) {
                            const int rr = dlt * KP + ph / KP + i;
                            if (rr < 0 || rr >= RB) continue;  // compile-time after unrolling
#pragma unroll
                            for (int j = 0; j < K; ++j) {
                                const int cc = pc * KP + ph % KP + j;
                                acc[rr][cc] = fmaf(w[i * K + j], d, acc[rr][cc]);
                            }
                        }
                    };
#ifndef CHAOS_DIN_SW
#define CHAOS_DIN_SW 0
#endif
                    if constexpr (CHAOS_DIN_SW && KP == 3) {
                        switch (arg) {  // warp-uniform: one indirect branch instead of a 9-way chain
                            case 0: add_phase(std::integral_constant<int, 0>{}); break;
                            case 1: add_phase(std::integral_constant<int, 1>{}); break;
                            case 2: add_phase(std::integral_constant<int, 2>{}); break;
                            case 3: add_phase(std::integral_constant<int, 3>{}); break;
                            case 4: add_phase(std::integral_constant<int, 4>{}); break;
                            case 5: add_phase(std::integral_constant<int, 5>{}); break;
                            case 6: add_phase(std::integral_constant<int, 6>{}); break;
                            case 7: add_phase(std::integral_constant<int, 7>{}); break;
                            case 8: add_phase(std::integral_constant<int, 8>{}); break;
                            default: break;
                        }
                    } else {
#pragma unroll
                        for (int ph = 0; ph < KP * KP; ++ph) {
                            if (arg == ph) {  // warp-uniform branch on the argmax phase
#pragma unroll
                                for (int i = 0; i < K; ++i) {
                                    const int rr = dlt * KP + ph / KP + i;
                                    if (rr < 0 || rr >= RB) continue;  // compile-time after unrolling
#pragma unroll
                                    for (int j = 0; j < K; ++j) {
                                        const int cc = pc * KP + ph % KP + j;
                                        acc[rr][cc] = fmaf(w[i * K + j], d, acc[rr][cc]);
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
        if constexpr (PAIR) {
            constexpr int CL = C < 32 ? C : 32;  // lanes that carry a map
            constexpr int SL = RB * L::W * CL;   // one partial band
            float* pb = pbuf + grp * (MSPLIT - 1) * SL + (lane < CL ? lane : 0);
            if (half > 0 && lane < CL) {
#pragma unroll
                for (int r = 0; r < RB; ++r)
#pragma unroll
                    for (int c = 0; c < L::W; ++c) pb[(half - 1) * SL + (r * L::W + c) * CL] = acc[r][c];
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * MSPLIT) : "memory");
            if (half == 0 && lane < CL) {
#pragma unroll
                for (int k = 0; k < MSPLIT - 1; ++k)
#pragma unroll
                    for (int r = 0; r < RB; ++r)
#pragma unroll
                        for (int c = 0; c < L::W; ++c) acc[r][c] += pb[k * SL + (r * L::W + c) * CL];
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * MSPLIT) : "memory");  // pb free again
            if (half != 0 || !act) continue;
        }
        const float* ib = in + g * L::IN_SZ + n * HW + b * RB * L::W;
        float* ob = dout + g * L::IN_SZ + n * HW + b * RB * L::W;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            if (b * RB + r < L::H) {
#pragma unroll
                for (int c = 0; c < L::W; ++c) {
                    const float v = ib[r * L::W + c];
                    ob[r * L::W + c] = acc[r][c] * (1.f - v * v);
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_din_rows) partial derivatives of the previous layer, window row by window row (any KP):
//   dout[g][n][y][x] = (1 - in^2) * sum_m sum_w W[n][y-oy][x-ox][m] dp[g][m][w],  (oy, ox) = the
//   argmax position of (g, m, w).
// One group of MSPLIT warps per (image, 32 input maps), lanes over n; warp k of the group takes
// output maps [k*M/MSPLIT, (k+1)*M/MSPLIT).  The accumulator holds the KP + K - 1 input rows one
// window row reaches; each (map, window) is dispatched ONCE (warp-uniform branch on its phase) into
// compile-time registers, so every argmax-sparse MAC is done with no band revisits (conv_din
// dispatches a window once per band it reaches: 2.7x on the medium net, with ~8 MACs each).  After
// window row pr the first KP rows are final: the group's partial rows meet in pbuf, warp 0 adds
// them in a fixed order (deterministic) and writes them; the block then shifts up by KP rows.
// pbuf: [NT/32/MSPLIT][MSPLIT-1][KP][WR][min(C,32)] floats.  dout may alias in.
// ------------------------------------------------------------------------------------
template <class L, int NT, int MSPLIT>
__device__ __forceinline__ void conv_din_rows(const float* __restrict__ wsm, const float* __restrict__ dp,
                                              const uint8_t* __restrict__ am, const float* in, float* dout, int cnt,
                                              float* __restrict__ pbuf) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int H = L::H, W = L::W, HW = H * W, R1 = KP + K - 1, WR = L::WR;
    constexpr int NCW = (C + 31) / 32, NW = NT / 32, NG = NW / MSPLIT;
    constexpr int CL = C < 32 ? C : 32;
    constexpr int SL = KP * WR * CL;  // one partial block of KP rows
    static_assert(NW % MSPLIT == 0 && NG <= 15, "warp groups, named barriers 1..15");
    static_assert(WR <= W && L::HR <= H, "the windows' reach stays inside the input");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = warp % MSPLIT, grp = warp / MSPLIT;
    const int m_lo = half * M / MSPLIT, m_hi = (half + 1) * M / MSPLIT;
    for (int vw = grp; vw < cnt * NCW; vw += NG) {
        const int cw = vw % NCW, g = vw / NCW;
        const int n0 = cw * 32 + lane;
        const bool act = n0 < C;
        const int n = act ? n0 : 0;
        const float* wn = wsm + n * L::NS;
        const int dgo = g * L::OUT_SZ;  // (offsets, not pointers: fewer live registers)
        float acc[R1][WR];
#pragma unroll
        for (int r = 0; r < R1; ++r)
#pragma unroll
            for (int c = 0; c < WR; ++c) acc[r][c] = 0.f;
        // rows [y0, y0 + nr) of the input are final in acc[0 .. nr): combine the group's partials, write
        auto emit = [&](int y0, int nr) {
            const float* ib = in + g * L::IN_SZ + n * HW;
            float* ob = dout + g * L::IN_SZ + n * HW;
            float* pb = pbuf + grp * (MSPLIT - 1) * SL + (lane < CL ? lane : 0);
            if (MSPLIT > 1 && half > 0 && lane < CL) {
#pragma unroll
                for (int r = 0; r < KP; ++r)
                    if (r < nr)
#pragma unroll
                        for (int c = 0; c < WR; ++c) pb[(half - 1) * SL + (r * WR + c) * CL] = acc[r][c];
            }
            if constexpr (MSPLIT > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * MSPLIT) : "memory");
            if (half == 0 && act) {
#pragma unroll
                for (int r = 0; r < KP; ++r) {
                    if (r < nr) {
#pragma unroll
                        for (int c = 0; c < W; ++c) {
                            float v = c < WR ? acc[r][c < WR ? c : 0] : 0.f;
#pragma unroll
                            for (int k = 0; k < MSPLIT - 1; ++k)
                                if (c < WR) v += pb[k * SL + (r * WR + (c < WR ? c : 0)) * CL];
                            const float x = ib[(y0 + r) * W + c];
                            ob[(y0 + r) * W + c] = v * (1.f - x * x);
                        }
                    }
                }
            }
            if constexpr (MSPLIT > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * MSPLIT) : "memory");
        };
#pragma unroll 1
        for (int pr = 0; pr < PH; ++pr) {
#pragma unroll 1
            for (int m = m_lo; m < m_hi; ++m) {
                float w[KK];
#pragma unroll
                for (int tp = 0; tp < KK; ++tp) w[tp] = wn[tp * L::MP + m];
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    const float d = dp[dgo + m * P + pr * PW + pc];
                    const int arg = static_cast<int>(am[dgo + m * P + pr * PW + pc]);
#pragma unroll
                    for (int ph = 0; ph < KP * KP; ++ph) {
                        if (arg == ph) {  // warp-uniform
#pragma unroll
                            for (int i = 0; i < K; ++i)
#pragma unroll
                                for (int j = 0; j < K; ++j)
                                    acc[ph / KP + i][pc * KP + ph % KP + j] =
                                        fmaf(w[i * K + j], d, acc[ph / KP + i][pc * KP + ph % KP + j]);
                        }
                    }
                }
            }
            emit(pr * KP, KP);
#pragma unroll
            for (int r = 0; r < R1; ++r)
#pragma unroll
                for (int c = 0; c < WR; ++c) acc[r][c] = (r + KP < R1) ? acc[r + KP < R1 ? r + KP : 0][c] : 0.f;
        }
        // the last K - 1 reached rows, in pieces of at most KP, then the floor-dropped rows (zero)
#pragma unroll
        for (int r0 = 0; r0 < R1 - KP; r0 += KP) {
            emit(PH * KP + r0, (R1 - KP - r0) < KP ? (R1 - KP - r0) : KP);
#pragma unroll
            for (int r = 0; r < R1; ++r)
#pragma unroll
                for (int c = 0; c < WR; ++c) acc[r][c] = (r + KP < R1) ? acc[r + KP < R1 ? r + KP : 0][c] : 0.f;
        }
        if (half == 0 && act)
            for (int y = L::HR; y < H; ++y)
#pragma unroll
                for (int c = 0; c < W; ++c) dout[g * L::IN_SZ + n * HW + y * W + c] = 0.f;
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_din_gm) partial derivatives of the previous layer with the weights read from
// global memory (a layer too large to stage: the Table I large net's conv3, 864 KB; with
// GLOBALW = false the same loop over a staged block -- its conv2, whose 20 input maps would
// leave lanes idle and give too few warp tasks in conv_din):
//   dout[g][n][y][x] = (1 - in^2) * sum_m sum_pp [tap in range] W[n][y-r][x-c][m] dp[g][m][pp]
// One warp per (image g, input map n, band of RB input rows); lanes over output maps m, so
// each weight load is one coalesced row segment W[n][tap][m..m+31] (__ldcg: L2, coherent with
// the other workers' reductions).  The argmax phase differs per lane, so every window's delta
// is expanded to its KP*KP phases (zero but one) and all phases accumulate branch-free into the
// lane's band registers; the lanes' partial bands are summed with warp shuffles.  W is read
// before this worker publishes the layer's gradient (pre-update for one worker, R5); dout may
// alias in.
// ------------------------------------------------------------------------------------
template <class L, int NT, int RB, bool GLOBALW = true>
__device__ __forceinline__ void conv_din_gm(const float* __restrict__ wg, const float* __restrict__ dp,
                                            const uint8_t* __restrict__ am, const float* in, float* dout, int cnt) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int W = L::W, HW = L::H * L::W, NB = (L::H + RB - 1) / RB;
    static_assert(RB % KP == 0, "bands start on a window row");
    constexpr int R2 = RB / KP;
    constexpr int DLO = -((KP + K - 2) / KP);  // window rows, relative to the band's first, that reach it
    constexpr int DHI = (RB - 1) / KP;
    constexpr int NWR = DHI - DLO + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int total = cnt * C * NB;
    for (int vw = warp; vw < total; vw += NT / 32) {
        const int b = vw % NB;
        const int n = (vw / NB) % C;
        const int g = vw / (NB * C);
        float acc[RB][W];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int c = 0; c < W; ++c) acc[r][c] = 0.f;
        const float* wn = wg + static_cast<long long>(n) * L::NS;
        const float* dpg = dp + g * L::OUT_SZ;
        const uint8_t* amg = am + g * L::OUT_SZ;
        const int pr0 = b * R2;
        // weights of the lane's next map are loaded one round ahead (global: hides the L2 latency)
        float wnx[KK];
#pragma unroll
        for (int tp = 0; tp < KK; ++tp)
            wnx[tp] = lane < M ? (GLOBALW ? __ldcg(wn + tp * L::MP + lane) : wn[tp * L::MP + lane]) : 0.f;
#pragma unroll 1
        for (int m = lane; m < M; m += 32) {
            float w[KK];
#pragma unroll
            for (int tp = 0; tp < KK; ++tp) w[tp] = wnx[tp];
            if (m + 32 < M) {
#pragma unroll
                for (int tp = 0; tp < KK; ++tp)
                    wnx[tp] = GLOBALW ? __ldcg(wn + tp * L::MP + m + 32) : wn[tp * L::MP + m + 32];
            }
#pragma unroll
            for (int dr = 0; dr < NWR; ++dr) {
                const int pr = pr0 + DLO + dr;
                if (pr < 0 || pr >= PH) continue;  // warp-uniform (the band is the warp's)
#pragma unroll
                for (int pc = 0; pc < PW; ++pc) {
                    const int o = m * P + pr * PW + pc;
                    const float d = dpg[o];
                    const int arg = static_cast<int>(amg[o]);
#pragma unroll
                    for (int ph = 0; ph < KP * KP; ++ph) {
                        const float dq = arg == ph ? d : 0.f;
#pragma unroll
                        for (int i = 0; i < K; ++i) {
                            const int rr = (DLO + dr) * KP + ph / KP + i;
                            if (rr < 0 || rr >= RB) continue;  // compile-time after unrolling
                            fma_row<K, (L::FF & 32) != 0>(&acc[rr][pc * KP + ph % KP], &w[i * K], dq,
                                           (rr * static_cast<int>(sizeof(acc[0]) / sizeof(float)) + pc * KP + ph % KP) & 1);
                        }
                    }
                }
            }
        }
        // transpose reduction: 32 band values per pass, 31 shuffles; lane l ends with value l
        const float* ib = in + g * L::IN_SZ + n * HW + b * RB * W;
        float* ob = dout + g * L::IN_SZ + n * HW + b * RB * W;
        const int nval = (b * RB + RB <= L::H ? RB : L::H - b * RB) * W;
        constexpr int NV = RB * W, NPASS = (NV + 31) / 32;
#pragma unroll
        for (int ps = 0; ps < NPASS; ++ps) {
            float v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = (ps * 32 + k < NV) ? acc[(ps * 32 + k) / W][(ps * 32 + k) % W] : 0.f;
            const float s = warp_transpose_sum(v, lane);
            const int idx = ps * 32 + lane;
            if (idx < nval) {
                const float x = ib[idx];
                ob[idx] = s * (1.f - x * x);
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(fc_fwd) fully connected forward: one warp per output row, lanes over inputs,
// weights streamed from L2 (__ldcg: on-demand reads of the shared store, no stale L1 copy).
// ------------------------------------------------------------------------------------
// TD (kTrace only): every weight / bias value read is also stored at td[w index] / td[WFL + o]
template <class F, int G, int NT, bool SMEMW = false, bool TD = false>  // SMEMW: W and b staged in shared memory
__device__ __forceinline__ void fc_fwd(const float* __restrict__ Wg, const float* __restrict__ bg,
                                       const float* __restrict__ in, float* __restrict__ out, int ostride,
                                       int cnt, float* __restrict__ td = nullptr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    for (int o = warp; o < F::OUT; o += NW) {
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.f;
        const float* wr = Wg + static_cast<long long>(o) * F::IN;
#pragma unroll 4
        for (int i = lane; i < F::IN; i += 32) {
            const float w = SMEMW ? wr[i] : __ldcg(wr + i);
            if constexpr (TD) td[o * F::IN + i] = w;
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = fmaf(w, in[g * F::IN + i], acc[g]);
        }
        const float b = SMEMW ? bg[o] : __ldcg(bg + o);
        if constexpr (TD)
            if (lane == 0) td[F::WFL + o] = b;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float s = warp_sum(acc[g]) + b;
            if (lane == 0 && g < cnt) out[g * ostride + o] = F::TANH ? tanhf(s) : s;
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_din3) delta_in by window-row bands (KP == 2), compact loop body: the task's PB window rows are a
// runtime loop over ONE window row's (KP+K-1) x WR register block, which shifts down by KP
// rows after each window row (its first KP rows are then final for this task).  The
// unrolled code is one window row (PW windows x 4 phases), so it stays in the instruction
// cache.  The first window row's KP rows wait in `pend` for the previous band's hand-off.
// ------------------------------------------------------------------------------------
// WTP > 0: the weights come from a transposed copy [m][C*K*K] with row pitch WTP (odd: lanes over
// input maps then read conflict-free; the staged [C*K*K][MP] layout puts them 540 floats apart)
template <class L, int NT, bool DEFER = false, int WTP = 0>
__device__ __forceinline__ void conv_din3(const float* __restrict__ wsm, const float* __restrict__ dp,
                                          const uint8_t* __restrict__ am, const float* in, float* out,
                                          float* __restrict__ hand, int cnt) {
    // DEFER: every write of `out` waits for the hand-off barrier (another phase running on other
    // warps may still be reading `in`, which `out` aliases)
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, PH = L::PH, P = L::P, M = L::M, C = L::C;
    constexpr int H = L::H, W = L::W, HW = H * W, PB = L::PB, NBAND = L::NBAND, WR = L::WR;
    constexpr int R1 = KP + K - 1, OV = K - 1;
    constexpr int NCW = (C + 31) / 32;
    static_assert(KP == 2, "2x2 pooling");
    static_assert(KP >= OV, "a window row's block overlaps only the next one");
    static_assert(M % 4 == 0 && L::MP == M, "4 output maps per vector load");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int total = cnt * NBAND * NCW;
    const bool has = warp < total;
    const int cw = warp % NCW;
    const int band = (warp / NCW) % NBAND;
    const int g = warp / (NCW * NBAND);
    const int n = cw * 32 + lane;
    const bool act = has && n < C;
    const int y0 = band * PB * KP;
    const float* ib = in + g * L::IN_SZ + (act ? n : 0) * HW;
    float* ob = out + g * L::IN_SZ + (act ? n : 0) * HW;
    float acc[R1][WR], pend[KP][WR];
    constexpr int NFIN = DEFER ? (PB > 1 ? PB - 1 : 1) : 1;
    float fin[NFIN][KP][WR];  // DEFER: rows of window rows 1..PB-1, written after the barrier
    static_assert(!DEFER || NBAND > 1, "DEFER needs the hand-off barrier");
#pragma unroll
    for (int r = 0; r < R1; ++r)
#pragma unroll
        for (int c = 0; c < WR; ++c) acc[r][c] = 0.f;
#pragma unroll
    for (int r = 0; r < KP; ++r)
#pragma unroll
        for (int c = 0; c < WR; ++c) pend[r][c] = 0.f;
    int nwr = 0;
    if (has) {
        const float* dpg = dp + g * L::OUT_SZ;
        const uint8_t* amg = am + g * L::OUT_SZ;
        const float* wn = wsm + (act ? n : 0) * (WTP > 0 ? KK : L::NS);
        constexpr bool W4 = KK <= 4 && WTP == 0;
#pragma unroll 1
        for (int wr = 0; wr < PB; ++wr) {
            const int pr = band * PB + wr;
            if (pr >= PH) break;  // warp-uniform (short last band)
            ++nwr;
#pragma unroll 1
            for (int m4 = 0; m4 < M; m4 += 4) {
                float4 w4[W4 ? KK : 1];
                if constexpr (W4) {
#pragma unroll
                    for (int tp = 0; tp < KK; ++tp) w4[tp] = *reinterpret_cast<const float4*>(wn + tp * L::MP + m4);
                }
#pragma unroll 1
                for (int mm = 0; mm < 4; ++mm) {
                    const int m = m4 + mm;
                    float w[KK];
#pragma unroll
                    for (int tp = 0; tp < KK; ++tp) {
                        if constexpr (W4)
                            w[tp] = mm == 0 ? w4[tp].x : mm == 1 ? w4[tp].y : mm == 2 ? w4[tp].z : w4[tp].w;
                        else if constexpr (WTP > 0)
                            w[tp] = wn[m * WTP + tp];
                        else
                            w[tp] = wn[tp * L::MP + m];
                    }
                    float dv[PW];
                    int av[PW];
#pragma unroll
                    for (int pc = 0; pc < PW; ++pc) {
                        dv[pc] = dpg[m * P + pr * PW + pc];
                        av[pc] = amg[m * P + pr * PW + pc];
                    }
#pragma unroll
                    for (int pc = 0; pc < PW; ++pc) {
                        const float d = dv[pc];
                        const int arg = av[pc];
                        // (packed FMAs measured slower here, twice: the pairing taps differ by phase -- written
                        // naively 3.94 M, with the taps (1, 2) loaded a second time into their own pair slots
                        // 3.98 M, vs 4.25 M scalar; DESIGN.md §7 session 5)
#define CHAOS_DIN3_PH(AA, BB)                                                                   \
    _Pragma("unroll") for (int i = 0; i < K; ++i) _Pragma("unroll") for (int j = 0; j < K; ++j) \
        acc[(AA) + i][pc * KP + (BB) + j] = fmaf(w[i * K + j], d, acc[(AA) + i][pc * KP + (BB) + j]);
                        if (arg < 2) {  // warp-uniform two-level branch on the argmax phase
                            if (arg == 0) {
                                CHAOS_DIN3_PH(0, 0)
                            } else {
                                CHAOS_DIN3_PH(0, 1)
                            }
                        } else {
                            if (arg == 2) {
                                CHAOS_DIN3_PH(1, 0)
                            } else {
                                CHAOS_DIN3_PH(1, 1)
                            }
                        }
#undef CHAOS_DIN3_PH
                    }
                }
            }
            // the block's first KP rows are final for this task
            if (wr == 0) {
#pragma unroll
                for (int r = 0; r < KP; ++r)
#pragma unroll
                    for (int c = 0; c < WR; ++c) pend[r][c] = acc[r][c];
            } else if constexpr (DEFER) {
#pragma unroll
                for (int f = 0; f < NFIN; ++f)
                    if (f + 1 == wr)
#pragma unroll
                        for (int r = 0; r < KP; ++r)
#pragma unroll
                            for (int c = 0; c < WR; ++c) fin[f][r][c] = acc[r][c];
            } else if (act) {
#pragma unroll
                for (int r = 0; r < KP; ++r) {
                    const int y = y0 + wr * KP + r;
#pragma unroll
                    for (int x = 0; x < W; ++x) {
                        const float v = ib[y * W + x];
                        ob[y * W + x] = (x < WR ? acc[r][x] : 0.f) * (1.f - v * v);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R1; ++r)
#pragma unroll
                for (int c = 0; c < WR; ++c) acc[r][c] = (r + KP < R1) ? acc[r + KP][c] : 0.f;
        }
    }
    // acc rows [0, OV) now hold the task's last OV rows: input rows y0 + nwr*KP + r
    if constexpr (NBAND > 1) {
        if (act && band < NBAND - 1) {
            float* hb = hand + ((g * (NBAND - 1) + band) * OV) * WR * C + n;
#pragma unroll
            for (int r = 0; r < OV; ++r)
#pragma unroll
                for (int c = 0; c < WR; ++c) hb[(r * WR + c) * C] = acc[r][c];
        }
        __syncthreads();
        if (act && band > 0) {
            const float* hb = hand + ((g * (NBAND - 1) + band - 1) * OV) * WR * C + n;
#pragma unroll
            for (int r = 0; r < OV; ++r)
#pragma unroll
                for (int c = 0; c < WR; ++c) pend[r][c] += hb[(r * WR + c) * C];
        }
    }
    if constexpr (DEFER) {
        if (act) {
#pragma unroll
            for (int f = 0; f < NFIN; ++f) {
                if (f + 1 < nwr) {
#pragma unroll
                    for (int r = 0; r < KP; ++r) {
                        const int y = y0 + (f + 1) * KP + r;
#pragma unroll
                        for (int x = 0; x < W; ++x) {
                            const float v = ib[y * W + x];
                            ob[y * W + x] = (x < WR ? fin[f][r][x] : 0.f) * (1.f - v * v);
                        }
                    }
                }
            }
        }
    }
    if (act) {
#pragma unroll
        for (int r = 0; r < KP; ++r) {  // the first window row's KP rows
            const int y = y0 + r;
#pragma unroll
            for (int x = 0; x < W; ++x) {
                const float v = ib[y * W + x];
                ob[y * W + x] = (x < WR ? pend[r][x] : 0.f) * (1.f - v * v);
            }
        }
        if (band == NBAND - 1) {  // the last band also owns the carried rows and everything below
            const int ye = y0 + nwr * KP;
#pragma unroll
            for (int r = 0; r < OV; ++r) {
                const int y = ye + r;
                if (y < H) {
#pragma unroll
                    for (int x = 0; x < W; ++x) {
                        const float v = ib[y * W + x];
                        ob[y * W + x] = (x < WR ? acc[r][x] : 0.f) * (1.f - v * v);
                    }
                }
            }
            for (int y = ye + OV; y < H; ++y)
#pragma unroll
                for (int x = 0; x < W; ++x) ob[y * W + x] = 0.f;
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_din_win) partial derivatives of the previous layer, dense per window and
// branch-free (KP == 2, whole input map per lane: small layers such as conv3):
//   dout[g][n][y][x] = (1 - in^2) * sum_m sum_w sum_q Dz_q[g][m][w] W[m][n][y-2pr-a(q)][x-2pc-b(q)]
// One warp per (image, 32 input maps); lanes over n hold the whole HR x WR delta map in
// registers; the phase selects d with a predicate-free select (4x the sparse MACs, no
// branches, so the warp issues back to back).  Weights: 4 output maps per LDS.128.
// ------------------------------------------------------------------------------------
template <class L, int NT, bool DEFER = false>
__device__ __forceinline__ void conv_din_win(const float* __restrict__ wsm, const float* __restrict__ dp,
                                             const uint8_t* __restrict__ am, const float* __restrict__ in,
                                             float* __restrict__ out, int cnt, const float4* __restrict__ dq4 = nullptr) {
    // dq4 (optional): phase-expanded delta as in conv_gw_win.  DEFER: one __syncthreads() between the
    // accumulation and the writes of `out` (which may hold dq4, still read by other warps)
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int H = L::H, W = L::W, HW = H * W, HR = L::HR, WR = L::WR;
    constexpr int NCW = (C + 31) / 32;
    static_assert(KP == 2 && M % 4 == 0 && L::MP == M, "2x2 pooling, 4 maps per vector load");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool has = warp < cnt * NCW;
    if (!DEFER && !has) return;
    const int cw = warp % NCW, g = has ? warp / NCW : 0;
    const int n = cw * 32 + lane;
    const bool act = has && n < C;
    const float* wn = wsm + (act ? n : 0) * L::NS;
    const float* dpg = dp + g * L::OUT_SZ;
    const uint8_t* amg = am + g * L::OUT_SZ;
    float acc[HR][WR];
#pragma unroll
    for (int y = 0; y < HR; ++y)
#pragma unroll
        for (int x = 0; x < WR; ++x) acc[y][x] = 0.f;
#pragma unroll 1
    for (int m4 = 0; m4 < (has ? M : 0); m4 += 4) {
        float4 w4[KK];
#pragma unroll
        for (int tp = 0; tp < KK; ++tp) w4[tp] = *reinterpret_cast<const float4*>(wn + tp * L::MP + m4);
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
            const int m = m4 + mm;
#pragma unroll
            for (int w = 0; w < P; ++w) {
                const int pr = w / PW, pc = w % PW;
                float dqv[4];
                if (dq4) {
                    const float4 t4 = dq4[g * L::OUT_SZ + m * P + w];
                    dqv[0] = t4.x;
                    dqv[1] = t4.y;
                    dqv[2] = t4.z;
                    dqv[3] = t4.w;
                } else {
                    const float d = dpg[m * P + w];
                    const int ph = amg[m * P + w];
#pragma unroll
                    for (int k = 0; k < 4; ++k) dqv[k] = (ph == k) ? d : 0.f;
                }
#pragma unroll
                for (int aa = 0; aa < KP; ++aa)
#pragma unroll
                    for (int bb = 0; bb < KP; ++bb) {
                        const float dq = dqv[aa * KP + bb];
#pragma unroll
                        for (int i = 0; i < K; ++i)
#pragma unroll
                            for (int j = 0; j < K; ++j) {
                                const float4 t = w4[i * K + j];
                                const float wv = mm == 0 ? t.x : mm == 1 ? t.y : mm == 2 ? t.z : t.w;
                                acc[pr * KP + aa + i][pc * KP + bb + j] =
                                    fmaf(wv, dq, acc[pr * KP + aa + i][pc * KP + bb + j]);
                            }
                    }
            }
        }
    }
    if constexpr (DEFER) __syncthreads();
    if (act) {
        const float* ib = in + g * L::IN_SZ + n * HW;
        float* ob = out + g * L::IN_SZ + n * HW;
#pragma unroll
        for (int y = 0; y < H; ++y)
#pragma unroll
            for (int x = 0; x < W; ++x) {
                const float v = ib[y * W + x];
                ob[y * W + x] = (y < HR && x < WR ? acc[y < HR ? y : 0][x < WR ? x : 0] : 0.f) * (1.f - v * v);
            }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_din_winp) conv_din_win from the phase-expanded delta with the delta loads of output
// map m+1 issued before map m's FMAs (software pipelined: the warp's FMAs no longer wait on
// their shared-memory loads; one warp per (image, 32 input maps) leaves few warps to hide them).
// ------------------------------------------------------------------------------------
template <class L, int NT, bool DEFER = false>
__device__ __forceinline__ void conv_din_winp(const float* __restrict__ wsm, const float* __restrict__ in,
                                              float* __restrict__ out, int cnt, const float4* __restrict__ dq4) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int H = L::H, W = L::W, HW = H * W, HR = L::HR, WR = L::WR;
    constexpr int NCW = (C + 31) / 32;
    static_assert(KP == 2 && M % 4 == 0 && L::MP == M, "2x2 pooling, 4 maps per vector load");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool has = warp < cnt * NCW;
    if (!DEFER && !has) return;
    const int cw = warp % NCW, g = has ? warp / NCW : 0;
    const int n = cw * 32 + lane;
    const bool act = has && n < C;
    const float* wn = wsm + (act ? n : 0) * L::NS;
    const float4* dqg = dq4 + g * L::OUT_SZ;
    float acc[HR][WR];
#pragma unroll
    for (int y = 0; y < HR; ++y)
#pragma unroll
        for (int x = 0; x < WR; ++x) acc[y][x] = 0.f;
    float4 cur[P];
    if (has) {
#pragma unroll
        for (int w = 0; w < P; ++w) cur[w] = dqg[w];
    }
#pragma unroll 1
    for (int m4 = 0; m4 < (has ? M : 0); m4 += 4) {
        float4 w4[KK];
#pragma unroll
        for (int tp = 0; tp < KK; ++tp) w4[tp] = *reinterpret_cast<const float4*>(wn + tp * L::MP + m4);
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
            const int m = m4 + mm;
            float4 nxt[P];
            const int mn = (m + 1 < M) ? m + 1 : m;
#pragma unroll
            for (int w = 0; w < P; ++w) nxt[w] = dqg[mn * P + w];
#pragma unroll
            for (int w = 0; w < P; ++w) {
                const int pr = w / PW, pc = w % PW;
                const float dqv[4] = {cur[w].x, cur[w].y, cur[w].z, cur[w].w};
#pragma unroll
                for (int aa = 0; aa < KP; ++aa)
#pragma unroll
                    for (int bb = 0; bb < KP; ++bb) {
                        const float dq = dqv[aa * KP + bb];
#pragma unroll
                        for (int i = 0; i < K; ++i)
#pragma unroll
                            for (int j = 0; j < K; ++j) {
                                const float4 t = w4[i * K + j];
                                const float wv = mm == 0 ? t.x : mm == 1 ? t.y : mm == 2 ? t.z : t.w;
                                acc[pr * KP + aa + i][pc * KP + bb + j] =
                                    fmaf(wv, dq, acc[pr * KP + aa + i][pc * KP + bb + j]);
                            }
                    }
            }
#pragma unroll
            for (int w = 0; w < P; ++w) cur[w] = nxt[w];
        }
    }
    if constexpr (DEFER) __syncthreads();
    if (act) {
        const float* ib = in + g * L::IN_SZ + n * HW;
        float* ob = out + g * L::IN_SZ + n * HW;
#pragma unroll
        for (int y = 0; y < H; ++y)
#pragma unroll
            for (int x = 0; x < W; ++x) {
                const float v = ib[y * W + x];
                ob[y * W + x] = (y < HR && x < WR ? acc[y < HR ? y : 0][x < WR ? x : 0] : 0.f) * (1.f - v * v);
            }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(conv_bwd_sparse) the whole backward of a small conv layer (KP == 2, lanes over input
// maps), argmax-sparse: for a given (image, output map, window) the argmax phase is the same for
// every lane, so one warp-uniform two-level branch selects it and only the argmax position's K*K
// products are computed (not the 4 phases of the dense conv_din_win / conv_gw_win).
//  delta_in: warps [0, DW), one per (image, 32 input maps): dout[g][n][y][x] = (1 - in^2) *
//            sum_m sum_w W[m][n][i][j] d[g][m][w] at (y, x) = window origin + phase + (i, j)
//  gW:       then every warp takes tasks (4 output maps, 32 input maps) from a shared counter:
//            gW[n][i][j][m] = sum_g sum_w d[g][m][w] in[g][n][origin + phase + (i, j)], gb = sum d,
//            published from registers (16-B vector reductions / slot stores).  The order of every
//            sum is fixed (g, w, then m or the task's own order): deterministic, whichever warp runs
//            a task.  out must not alias in / dp.  ctr: one int of shared memory, 0 on entry.
// ------------------------------------------------------------------------------------
// MS = 2: each (image, 32 input maps) delta_in task is split over two warps by output-map halves
// (the δ_in warps' serial chains are the phase's critical path); the first half's sums go through
// `out` to its partner (named barrier per pair), which adds its own in a fixed order.
template <class L, int NT, int MODE, int MS = 1>
__device__ __forceinline__ void conv_bwd_sparse(const KArgs& a, int slot, const float* __restrict__ wsm,
                                                const float* __restrict__ dp, const uint8_t* __restrict__ am,
                                                const float* __restrict__ in, float* __restrict__ out, int woff,
                                                int cnt, float sc, int* ctr) {
    constexpr int K = L::K, KP = L::KP, KK = L::KK, PW = L::PW, P = L::P, M = L::M, C = L::C;
    constexpr int H = L::H, W = L::W, HW = H * W, HR = L::HR, WR = L::WR, BS = KP + K - 1;
    constexpr int NCW = (C + 31) / 32, NMG = M / 4, NTASK = NMG * NCW;
    static_assert(KP == 2 && M % 4 == 0 && L::MP == M, "2x2 pooling, 4 maps per vector");
    static_assert(MS == 1 || MS == 2, "delta_in split over 1 or 2 warps");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef CHAOS_TIMING
    const long long t_in = clock64();
#endif
    // ---- delta_in
    if (warp < cnt * NCW * MS) {
        const int sp = warp % MS, cw = (warp / MS) % NCW, g = warp / (MS * NCW);
        constexpr int M4H = (NMG + 1) / 2 * 4;  // MS = 2: maps [0, M4H) and [M4H, M)
        const int mlo = (MS == 2 && sp == 1) ? M4H : 0, mhi = (MS == 2 && sp == 0) ? M4H : M;
        const int n = cw * 32 + lane;
        const bool act = n < C;
        const float* wn = wsm + (act ? n : C - 1) * L::NS;
        const float* dpg = dp + g * L::OUT_SZ;
        const uint8_t* amg = am + g * L::OUT_SZ;
        float acc[HR][WR];
#pragma unroll
        for (int y = 0; y < HR; ++y)
#pragma unroll
            for (int x = 0; x < WR; ++x) acc[y][x] = 0.f;
#pragma unroll 1
        for (int m4 = mlo; m4 < mhi; m4 += 4) {
            float4 w4[KK];
#pragma unroll
            for (int tp = 0; tp < KK; ++tp) w4[tp] = *reinterpret_cast<const float4*>(wn + tp * L::MP + m4);
            float dv[4][P];
            int av[4][P];
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) {
                if constexpr (P == 4) {  // one map's 4 windows: a 16-B delta load and a 4-byte phase load
                    const float4 d4 = *reinterpret_cast<const float4*>(dpg + (m4 + mm) * P);
                    const uint32_t a4 = *reinterpret_cast<const uint32_t*>(amg + (m4 + mm) * P);
                    dv[mm][0] = d4.x;
                    dv[mm][1] = d4.y;
                    dv[mm][2] = d4.z;
                    dv[mm][3] = d4.w;
#pragma unroll
                    for (int w = 0; w < 4; ++w) av[mm][w] = (a4 >> (8 * w)) & 0xffu;
                } else {
#pragma unroll
                    for (int w = 0; w < P; ++w) {
                        dv[mm][w] = dpg[(m4 + mm) * P + w];
                        av[mm][w] = amg[(m4 + mm) * P + w];
                    }
                }
            }
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) {
                float wv[KK];
#pragma unroll
                for (int tp = 0; tp < KK; ++tp)
                    wv[tp] = mm == 0 ? w4[tp].x : mm == 1 ? w4[tp].y : mm == 2 ? w4[tp].z : w4[tp].w;
#pragma unroll
                for (int w = 0; w < P; ++w) {
                    const int pr = w / PW, pc = w % PW;
                    const float d = dv[mm][w];
                    const int ph = av[mm][w];
#define CHAOS_DIN_PH(AA, BB)                                                                    \
    _Pragma("unroll") for (int i = 0; i < K; ++i) _Pragma("unroll") for (int j = 0; j < K; ++j) \
        acc[pr * KP + (AA) + i][pc * KP + (BB) + j] =                                           \
            fmaf(wv[i * K + j], d, acc[pr * KP + (AA) + i][pc * KP + (BB) + j]);
                    if (ph < 2) {  // warp-uniform: one argmax phase per (image, map, window)
                        if (ph == 0) {
                            CHAOS_DIN_PH(0, 0)
                        } else {
                            CHAOS_DIN_PH(0, 1)
                        }
                    } else {
                        if (ph == 2) {
                            CHAOS_DIN_PH(1, 0)
                        } else {
                            CHAOS_DIN_PH(1, 1)
                        }
                    }
#undef CHAOS_DIN_PH
                }
            }
        }
        float* ob = out + g * L::IN_SZ + (act ? n : C - 1) * HW;
        if constexpr (MS == 2) {  // first half -> out (raw sums), pair barrier, second half adds
            const int pair = 1 + g * NCW + cw;
            if (sp == 0 && act) {
#pragma unroll
                for (int y = 0; y < HR; ++y)
#pragma unroll
                    for (int x = 0; x < WR; ++x) ob[y * W + x] = acc[y][x];
            }
            asm volatile("bar.sync %0, 64;" ::"r"(pair) : "memory");
            if (sp == 1 && act) {
#pragma unroll
                for (int y = 0; y < HR; ++y)
#pragma unroll
                    for (int x = 0; x < WR; ++x) acc[y][x] = ob[y * W + x] + acc[y][x];
            }
        }
        if (act && (MS == 1 || sp == 1)) {
            const float* ib = in + g * L::IN_SZ + n * HW;
#pragma unroll
            for (int y = 0; y < H; ++y)
#pragma unroll
                for (int x = 0; x < W; ++x) {
                    const float v = ib[y * W + x];
                    ob[y * W + x] = (y < HR && x < WR ? acc[y < HR ? y : 0][x < WR ? x : 0] : 0.f) * (1.f - v * v);
                }
        }
#ifdef CHAOS_TIMING
        if (threadIdx.x == 0 && a.ptime) a.ptime[blockIdx.x * kPhases + 17] += clock64() - t_in;
#endif
    }
    // ---- weight gradient: tasks (4 output maps, 32 input maps) from the shared counter
    for (;;) {
        int task = 0;
        if (lane == 0) task = atomicAdd(ctr, 1);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= NTASK) break;
        const int cw = task % NCW, m0 = (task / NCW) * 4;
        const int n = cw * 32 + lane;
        const bool act = n < C;
        float acc[4][KK];
        float accb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            accb[q] = 0.f;
#pragma unroll
            for (int t = 0; t < KK; ++t) acc[q][t] = 0.f;
        }
#pragma unroll 1
        for (int g = 0; g < cnt; ++g) {
            const float* ing = in + g * L::IN_SZ + (act ? n : C - 1) * HW;
            const float* dpg = dp + g * L::OUT_SZ + m0 * P;
            const uint8_t* amg = am + g * L::OUT_SZ + m0 * P;
            float dvs[4 * P];
            int avs[4 * P];
            if constexpr (P == 4) {  // the task's 4 maps x 4 windows: four 16-B delta loads, one 16-B phase load
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 d4 = reinterpret_cast<const float4*>(dpg)[q];
                    dvs[4 * q] = d4.x;
                    dvs[4 * q + 1] = d4.y;
                    dvs[4 * q + 2] = d4.z;
                    dvs[4 * q + 3] = d4.w;
                }
                const uint4 a16 = *reinterpret_cast<const uint4*>(amg);
                const uint32_t aw[4] = {a16.x, a16.y, a16.z, a16.w};
#pragma unroll
                for (int e = 0; e < 16; ++e) avs[e] = (aw[e / 4] >> (8 * (e % 4))) & 0xffu;
            } else {
#pragma unroll
                for (int e = 0; e < 4 * P; ++e) {
                    dvs[e] = dpg[e];
                    avs[e] = amg[e];
                }
            }
#pragma unroll
            for (int w = 0; w < P; ++w) {
                const int pr = w / PW, pc = w % PW;
                float blk[BS][BS];
#pragma unroll
                for (int u = 0; u < BS; ++u)
#pragma unroll
                    for (int v = 0; v < BS; ++v) blk[u][v] = ing[(pr * KP + u) * W + pc * KP + v];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float d = dvs[q * P + w];
                    const int ph = avs[q * P + w];
                    accb[q] += d;
#define CHAOS_GW_PH(AA, BB)                       \
    _Pragma("unroll") for (int i = 0; i < K; ++i) \
        fma_row<K, (L::FF & 4) != 0>(&acc[q][i * K], &blk[(AA) + i][(BB)], d, (q * KK + i * K) & 1);
                    if (ph < 2) {  // warp-uniform
                        if (ph == 0) {
                            CHAOS_GW_PH(0, 0)
                        } else {
                            CHAOS_GW_PH(0, 1)
                        }
                    } else {
                        if (ph == 2) {
                            CHAOS_GW_PH(1, 0)
                        } else {
                            CHAOS_GW_PH(1, 1)
                        }
                    }
#undef CHAOS_GW_PH
                }
            }
        }
        if (act) {
#pragma unroll
            for (int t = 0; t < KK; ++t)
                publish_vec4<MODE>(a, slot, woff + n * L::NS + t * L::MP + m0,
                                   make_float4(sc * acc[0][t], sc * acc[1][t], sc * acc[2][t], sc * acc[3][t]));
            if (n == 0)
                publish_vec4<MODE>(a, slot, woff + L::WFL + m0,
                                   make_float4(sc * accb[0], sc * accb[1], sc * accb[2], sc * accb[3]));
        }
    }
#ifdef CHAOS_TIMING
    if (threadIdx.x == NT - 32 && a.ptime) a.ptime[blockIdx.x * kPhases + 18] += clock64() - t_in;
#endif
}

// ------------------------------------------------------------------------------------
// PHASE(fc_fwd2) fully connected forward, IN % 4 == 0: one warp per NR output rows, lanes
// over 16-B column quads; every weight load of the NR rows is issued before the first FMA
// (__ldcg: on-demand reads of the shared store from L2), activations are LDS.128 broadcasts
// shared by the NR rows, and the NR*G partial sums are reduced with warp shuffles.
// ------------------------------------------------------------------------------------
template <class F, int G, int NT, int NR>
__device__ __forceinline__ void fc_fwd2(const float* __restrict__ Wg, const float* __restrict__ bg,
                                        const float* __restrict__ in, float* __restrict__ out, int ostride,
                                        int cnt) {
    static_assert(F::IN % 4 == 0, "column quads");
    constexpr int IN4 = F::IN / 4, NK = (IN4 + 31) / 32, NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o0 = warp * NR; o0 < F::OUT; o0 += NW * NR) {
        float4 w[NR][NK];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int c = lane + 32 * k;
                w[r][k] = (o0 + r < F::OUT && c < IN4)
                              ? __ldcg(reinterpret_cast<const float4*>(Wg + static_cast<long long>(o0 + r) * F::IN) + c)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        float acc[NR][G];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int g = 0; g < G; ++g) acc[r][g] = 0.f;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const int c = lane + 32 * k;
            if (c < IN4) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float4 x = reinterpret_cast<const float4*>(in + g * F::IN)[c];
#pragma unroll
                    for (int r = 0; r < NR; ++r) {
                        acc[r][g] = fmaf(w[r][k].x, x.x, acc[r][g]);
                        acc[r][g] = fmaf(w[r][k].y, x.y, acc[r][g]);
                        acc[r][g] = fmaf(w[r][k].z, x.z, acc[r][g]);
                        acc[r][g] = fmaf(w[r][k].w, x.w, acc[r][g]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (o0 + r < F::OUT) {
                const float b = __ldcg(bg + o0 + r);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float s = warp_sum(acc[r][g]) + b;
                    if (lane == 0 && g < cnt) out[g * ostride + o0 + r] = F::TANH ? tanhf(s) : s;
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(fc_bwd2) fully connected backward without staging (IN % 4 == 0).  Thread item =
// (16-B column quad c, row group rg of ~OUT/NRG rows).  Per row o the thread reads W[o][4c]
// (pre-update: it is the only reader of those 4 weights in this CTA and reads them before
// publishing their gradient), accumulates delta_in for its columns, and publishes
// gW[o][4c..4c+3] = sum_g dz[g][o] a[g][4c..] with one 16-B vector reduction (hogwild) or
// store (sync) -- no shared-memory staging, no per-chunk barriers.  Row groups' delta_in
// partials meet in `scr` ([NRG-1][G][IN]) and are summed in group order (deterministic),
// times (1 - a^2), in place over `in`.  Bias gradients go through `bsc` + one bulk op.
// ------------------------------------------------------------------------------------
template <class F, int G, int NT, int MODE, int NRG>
__device__ __forceinline__ void fc_bwd2(const KArgs& a, int slot, int woff, int boff, float* __restrict__ in,
                                        const float* __restrict__ dz, int dstride, float* __restrict__ scr,
                                        float* __restrict__ bsc, int cnt, float sc) {
    static_assert(F::IN % 4 == 0, "column quads");
    constexpr int IN4 = F::IN / 4;
    static_assert(IN4 * NRG <= NT, "one thread per (column quad, row group)");
    const float* Wg = a.params + woff;
    const int c = threadIdx.x % IN4;
    const int rg = threadIdx.x / IN4;
    const bool act = threadIdx.x < IN4 * NRG;
    float4 av[G], din[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        av[g] = (act && g < cnt) ? reinterpret_cast<const float4*>(in + g * F::IN)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        din[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (act) {
        const int o0 = (F::OUT * rg) / NRG, o1 = (F::OUT * (rg + 1)) / NRG;
        constexpr int BATCH = 6;
#pragma unroll 1
        for (int ob = o0; ob < o1; ob += BATCH) {
            float4 w[BATCH];
#pragma unroll
            for (int q = 0; q < BATCH; ++q)
                w[q] = (ob + q < o1) ? __ldcg(reinterpret_cast<const float4*>(Wg + static_cast<long long>(ob + q) * F::IN) + c)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < BATCH; ++q) {
                if (ob + q < o1) {
                    const int o = ob + q;
                    float4 gw = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (g < cnt) {
                            const float d = dz[g * dstride + o];
                            din[g].x = fmaf(w[q].x, d, din[g].x);
                            din[g].y = fmaf(w[q].y, d, din[g].y);
                            din[g].z = fmaf(w[q].z, d, din[g].z);
                            din[g].w = fmaf(w[q].w, d, din[g].w);
                            gw.x = fmaf(d, av[g].x, gw.x);
                            gw.y = fmaf(d, av[g].y, gw.y);
                            gw.z = fmaf(d, av[g].z, gw.z);
                            gw.w = fmaf(d, av[g].w, gw.w);
                        }
                    }
                    publish_vec4<MODE>(a, slot, woff + o * F::IN + 4 * c,
                                       make_float4(sc * gw.x, sc * gw.y, sc * gw.z, sc * gw.w));
                }
            }
        }
        if (rg > 0)
#pragma unroll
            for (int g = 0; g < G; ++g)
                reinterpret_cast<float4*>(scr + ((rg - 1) * G + g) * F::IN)[c] = din[g];
    }
    for (int o = threadIdx.x; o < F::BFL; o += NT) {  // bias
        float gb = 0.f;
        if (o < F::OUT)
            for (int g = 0; g < cnt; ++g) gb += dz[g * dstride + o];
        bsc[o] = sc * gb;
    }
    sync_for_async();
    publish_bulk<MODE>(a, slot, boff, bsc, F::BFL);
    if (act && rg == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (g < cnt) {
                float4 t = din[g];
#pragma unroll
                for (int k = 1; k < NRG; ++k) {
                    const float4 p = reinterpret_cast<const float4*>(scr + ((k - 1) * G + g) * F::IN)[c];
                    t.x += p.x;
                    t.y += p.y;
                    t.z += p.z;
                    t.w += p.w;
                }
                const float4 x = av[g];
                reinterpret_cast<float4*>(in + g * F::IN)[c] =
                    make_float4(t.x * (1.f - x.x * x.x), t.y * (1.f - x.y * x.y), t.z * (1.f - x.z * x.z),
                                t.w * (1.f - x.w * x.w));
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(fc_fwd3) fully connected forward with the weights staged in shared memory: chunks of
// RCH rows are TMA bulk-copied (cp.async.bulk) into two buffers, the copy of chunk c+2
// overlapping the compute of chunk c+1; one warp per row, lanes over 16-B column quads.
// ------------------------------------------------------------------------------------
template <class F, int G, int NT, int RCH, int MODE = kHogwild>
__device__ __forceinline__ void fc_fwd3(const float* __restrict__ Wg, const float* __restrict__ bg,
                                        const float* __restrict__ in, float* __restrict__ out, int ostride, int cnt,
                                        float* __restrict__ buf, Loader& LA, Loader& LB, float* __restrict__ sb,
                                        const KArgs* ta = nullptr, int slot = 0, int woff = 0) {
    // MODE == kTrace: each chunk / the biases as read go to the group's forward read record (ta)
    // sb: F::OUT floats of shared scratch for the biases (loaded once, up front)
    static_assert(F::IN % 4 == 0 && (RCH * F::IN) % 4 == 0, "16-B chunks");
    constexpr int IN4 = F::IN / 4, NK = (IN4 + 31) / 32, NW = NT / 32;
    constexpr int NCH = (F::OUT + RCH - 1) / RCH;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto rows = [](int c) { return (c + 1) * RCH <= F::OUT ? RCH : F::OUT - c * RCH; };
    LA.issue(buf, Wg, rows(0) * F::IN);
    if (NCH > 1) LB.issue(buf + RCH * F::IN, Wg + RCH * F::IN, rows(1) * F::IN);
    for (int o = threadIdx.x; o < F::OUT; o += NT) sb[o] = __ldcg(bg + o);
    __syncthreads();
    if constexpr (MODE == kTrace) trace_dump(*ta, slot, 0, woff + F::WFL, sb, F::BFL);  // 16-B multiple
    for (int c = 0; c < NCH; ++c) {
        const float* cb = buf + (c & 1) * RCH * F::IN;
        if (c & 1)
            LB.wait();
        else
            LA.wait();
        if constexpr (MODE == kTrace) trace_dump(*ta, slot, 0, woff + c * RCH * F::IN, cb, rows(c) * F::IN);
        // RPW rows per warp pass: each activation quad loaded from shared memory feeds RPW rows
#ifndef CHAOS_FC1_RPW
#define CHAOS_FC1_RPW 3
#endif
        constexpr int RPW = CHAOS_FC1_RPW;
        for (int r0 = warp * RPW; r0 < rows(c); r0 += NW * RPW) {
            float acc[RPW][G];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
                for (int g = 0; g < G; ++g) acc[rr][g] = 0.f;
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int q = lane + 32 * k;
                if (q < IN4) {
                    float4 x[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) x[g] = reinterpret_cast<const float4*>(in + g * F::IN)[q];
#pragma unroll
                    for (int rr = 0; rr < RPW; ++rr) {
                        if (r0 + rr < rows(c)) {
                            const float4 w = reinterpret_cast<const float4*>(cb + (r0 + rr) * F::IN)[q];
#pragma unroll
                            for (int g = 0; g < G; ++g) {
                                acc[rr][g] = fmaf(w.x, x[g].x, acc[rr][g]);
                                acc[rr][g] = fmaf(w.y, x[g].y, acc[rr][g]);
                                acc[rr][g] = fmaf(w.z, x[g].z, acc[rr][g]);
                                acc[rr][g] = fmaf(w.w, x[g].w, acc[rr][g]);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                if (r0 + rr < rows(c)) {
                    const int o = c * RCH + r0 + rr;
                    const float b = sb[o];
                    // reduce the G partial sums; lane g finishes image g (tanh spread over lanes)
                    float mine = 0.f;
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float s = warp_sum(acc[rr][g]) + b;
                        if (lane == g) mine = s;
                    }
                    if (lane < cnt) out[lane * ostride + o] = F::TANH ? tanhf(mine) : mine;
                }
            }
        }
        if (c + 2 < NCH) {
            sync_for_async();  // every warp is done reading this buffer
            if (c & 1)
                LB.issue(buf + RCH * F::IN, Wg + (c + 2) * RCH * F::IN, rows(c + 2) * F::IN);
            else
                LA.issue(buf, Wg + (c + 2) * RCH * F::IN, rows(c + 2) * F::IN);
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(fc_bwd3) fc_bwd2 with the weights staged chunk by chunk in shared memory (as in
// fc_fwd3).  Thread item = (16-B column quad, row group); within a chunk the row group takes
// every NRG-th row.  W is the pre-update snapshot: this CTA publishes gW[o][4c..] only after
// its thread read W[o][4c..] from the chunk (the chunk was copied before any publish of it).
// ------------------------------------------------------------------------------------
// RESIDENT: the forward's last two chunks are still in `buf` (nothing touched it since
// fc_fwd3): the chunks are processed in reverse order, the first two without a copy -- the
// forward's snapshot, which precedes this worker's publish of the layer (R5).
template <class F, int G, int NT, int MODE, int NRG, int RCH, bool RESIDENT = false>
__device__ __forceinline__ void fc_bwd3(const KArgs& a, int slot, int woff, int boff, float* __restrict__ in,
                                        const float* __restrict__ dz, int dstride, float* __restrict__ scr,
                                        float* __restrict__ bsc, int cnt, float sc, float* __restrict__ buf,
                                        Loader& LA, Loader& LB) {
    static_assert(F::IN % 4 == 0 && (RCH * F::IN) % 4 == 0, "16-B chunks");
    constexpr int IN4 = F::IN / 4;
    constexpr int NCH = (F::OUT + RCH - 1) / RCH;
    static_assert(IN4 * NRG <= NT, "one thread per (column quad, row group)");
    static_assert(!RESIDENT || NCH >= 2, "two resident chunks");
    const float* Wg = a.params + woff;
    auto rows = [](int c) { return (c + 1) * RCH <= F::OUT ? RCH : F::OUT - c * RCH; };
    if constexpr (!RESIDENT) {
        LA.issue(buf, Wg, rows(0) * F::IN);
        if (NCH > 1) LB.issue(buf + RCH * F::IN, Wg + RCH * F::IN, rows(1) * F::IN);
    }
    const int c4 = threadIdx.x % IN4;
    const int rg = threadIdx.x / IN4;
    const bool act = threadIdx.x < IN4 * NRG;
    float4 av[G], din[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        av[g] = (act && g < cnt) ? reinterpret_cast<const float4*>(in + g * F::IN)[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
        din[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int i = 0; i < NCH; ++i) {
        const int c = RESIDENT ? NCH - 1 - i : i;
        const float* cb = buf + (c & 1) * RCH * F::IN;
        if (!RESIDENT || i >= 2) {
            if (c & 1)
                LB.wait();
            else
                LA.wait();
        }
        if constexpr (MODE == kTrace) trace_dump(a, slot, 1, woff + c * RCH * F::IN, cb, rows(c) * F::IN);
        if (act) {
            for (int r = rg; r < rows(c); r += NRG) {
                const int o = c * RCH + r;
                const float4 w = reinterpret_cast<const float4*>(cb + r * F::IN)[c4];
                float4 gw = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (g < cnt) {
                        const float d = dz[g * dstride + o];
                        din[g].x = fmaf(w.x, d, din[g].x);
                        din[g].y = fmaf(w.y, d, din[g].y);
                        din[g].z = fmaf(w.z, d, din[g].z);
                        din[g].w = fmaf(w.w, d, din[g].w);
                        gw.x = fmaf(d, av[g].x, gw.x);
                        gw.y = fmaf(d, av[g].y, gw.y);
                        gw.z = fmaf(d, av[g].z, gw.z);
                        gw.w = fmaf(d, av[g].w, gw.w);
                    }
                }
                publish_vec4<MODE>(a, slot, woff + o * F::IN + 4 * c4,
                                   make_float4(sc * gw.x, sc * gw.y, sc * gw.z, sc * gw.w));
            }
        }
        const int nx = RESIDENT ? c - 2 : c + 2;
        if (RESIDENT ? nx >= 0 : nx < NCH) {
            sync_for_async();
            if (c & 1)
                LB.issue(buf + RCH * F::IN, Wg + nx * RCH * F::IN, rows(nx) * F::IN);
            else
                LA.issue(buf, Wg + nx * RCH * F::IN, rows(nx) * F::IN);
        }
    }
    if (act && rg > 0)
#pragma unroll
        for (int g = 0; g < G; ++g) reinterpret_cast<float4*>(scr + ((rg - 1) * G + g) * F::IN)[c4] = din[g];
    for (int o = threadIdx.x; o < F::BFL; o += NT) {  // bias
        float gb = 0.f;
        if (o < F::OUT)
            for (int g = 0; g < cnt; ++g) gb += dz[g * dstride + o];
        bsc[o] = sc * gb;
    }
    sync_for_async();
    publish_bulk<MODE>(a, slot, boff, bsc, F::BFL);
    if (act && rg == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (g < cnt) {
                float4 t = din[g];
#pragma unroll
                for (int k = 1; k < NRG; ++k) {
                    const float4 p = reinterpret_cast<const float4*>(scr + ((k - 1) * G + g) * F::IN)[c4];
                    t.x += p.x;
                    t.y += p.y;
                    t.z += p.z;
                    t.w += p.w;
                }
                const float4 x = av[g];
                reinterpret_cast<float4*>(in + g * F::IN)[c4] =
                    make_float4(t.x * (1.f - x.x * x.x), t.y * (1.f - x.y * x.y), t.z * (1.f - x.z * x.z),
                                t.w * (1.f - x.w * x.w));
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// PHASE(fc_bwd) fully connected backward: one thread per input column i, outputs o in
// chunks.  Reads W[o][i] (pre-update, on demand) for delta_in; gW[o][i] = sum_g dz[g][o] a[g][i]
// goes (scaled) into a shared-memory chunk that is published with one bulk op while the
// next chunk is computed into the other half of S; delta_in * (1 - a^2) is written in
// place over the input activations.  Bias gradients go through `bsc`.
// ------------------------------------------------------------------------------------
template <class F, int G, int NT, int MODE, int SHALF>
__device__ __forceinline__ void fc_bwd(const KArgs& a, int slot, int woff, int boff, float* __restrict__ in,
                                       const float* __restrict__ dz, int dstride, float* __restrict__ S,
                                       float* __restrict__ bsc, int cnt, float sc,
                                       const float* __restrict__ wstaged = nullptr) {  // W staged in smem
    // kTrace: the W values read from global for delta_in go to the group's delta_in read record
    float* td = nullptr;
    if constexpr (MODE == kTrace) td = a.tw + (static_cast<long long>(slot) * 2 + 1) * a.pstride + woff;
    (void)td;
    constexpr int RPC0 = SHALF / F::IN;  // rows per chunk
    constexpr int RPC = (RPC0 >= F::OUT) ? F::OUT : ((RPC0 * F::IN) % 4 == 0 ? RPC0 : RPC0 / 4 * 4);
    static_assert(RPC >= 1, "S half must hold a weight row");
    static_assert(RPC == F::OUT || (RPC * F::IN) % 4 == 0, "chunk starts must stay 16-B aligned");
    constexpr int NCH = (F::OUT + RPC - 1) / RPC;
    static_assert(F::WFL - (NCH - 1) * RPC * F::IN <= SHALF, "last chunk must fit");
    const float* Wg = a.params + woff;
    constexpr int NI = (F::IN + NT - 1) / NT;  // columns per thread
    float av[NI][G], din[NI][G];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int col = threadIdx.x + k * NT;
            av[k][g] = (g < cnt && col < F::IN) ? in[g * F::IN + col] : 0.f;
            din[k][g] = 0.f;
        }
    for (int c = 0; c < NCH; ++c) {
        const int o0 = c * RPC;
        const int o1 = (o0 + RPC < F::OUT) ? o0 + RPC : F::OUT;
        float* buf = S + (c & 1) * SHALF;
        if (c >= 2) {  // the bulk publish of chunk c-2 must have read this half
            if (threadIdx.x == 0) bulk_wait_read<1>();
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < NI; ++k) {
            const int col = threadIdx.x + k * NT;
            if (col < F::IN) {
                for (int o = o0; o < o1; o += 4) {
                    float w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        w[q] = (o + q < o1) ? (wstaged ? wstaged[(o + q) * F::IN + col]
                                                       : __ldcg(Wg + static_cast<long long>(o + q) * F::IN + col))
                                            : 0.f;
                    if constexpr (MODE == kTrace) {
                        if (!wstaged) {
                            for (int q = 0; q < 4; ++q)
                                if (o + q < o1) td[(o + q) * F::IN + col] = w[q];
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (o + q < o1) {
                            float gw = 0.f;
#pragma unroll
                            for (int g = 0; g < G; ++g) {
                                if (g < cnt) {
                                    const float d = dz[g * dstride + o + q];
                                    din[k][g] = fmaf(w[q], d, din[k][g]);
                                    gw = fmaf(d, av[k][g], gw);
                                }
                            }
                            buf[(o + q - o0) * F::IN + col] = sc * gw;
                        }
                    }
                }
            }
        }
        const int fl = (o1 == F::OUT) ? F::WFL - o0 * F::IN : (o1 - o0) * F::IN;
        if (o1 == F::OUT)
            for (int e = (o1 - o0) * F::IN + threadIdx.x; e < fl; e += NT) buf[e] = 0.f;  // block padding
        sync_for_async();
        publish_bulk<MODE>(a, slot, woff + o0 * F::IN, buf, fl);
    }
    for (int o = threadIdx.x; o < F::BFL; o += NT) {  // bias
        float gb = 0.f;
        if (o < F::OUT)
            for (int g = 0; g < cnt; ++g) gb += dz[g * dstride + o];
        bsc[o] = sc * gb;
    }
    sync_for_async();
    publish_bulk<MODE>(a, slot, boff, bsc, F::BFL);
    // delta_in, in place (each thread owns its columns)
#pragma unroll
    for (int k = 0; k < NI; ++k) {
        const int col = threadIdx.x + k * NT;
        if (col < F::IN)
#pragma unroll
            for (int g = 0; g < G; ++g)
                if (g < cnt) in[g * F::IN + col] = din[k][g] * (1.f - av[k][g] * av[k][g]);
    }
}

// ------------------------------------------------------------------------------------
// Host entry point: spin until the copy stream has landed images [0, need).
__device__ __forceinline__ void wait_landed(const unsigned long long* ready, unsigned long long need) {
    while (*reinterpret_cast<const volatile unsigned long long*>(ready) < need) __nanosleep(256);
}

// ------------------------------------------------------------------------------------
// PHASE(pavg) fused cross-replica averaging, serviced by the hogwild worker between image groups
// (see PavgArgs).  Loads of peer data are relaxed at system scope (never served by a stale L1
// line); flags are published with a system-scope fence after a CTA barrier (cumulative) and read
// with relaxed loads followed by a system-scope fence before the barrier that releases the reads.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float4 ld_relaxed_sys4(const float* p) {
    float4 v;
    asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long bits4(float4 v) {
    return static_cast<unsigned long long>(__float_as_uint(v.x)) + __float_as_uint(v.y) + __float_as_uint(v.z) +
           __float_as_uint(v.w);
}

// Warp 0: do all R replicas' words w[q][s] for this CTA's slices s reach `need`?  (parallel loads)
__device__ __forceinline__ bool pavg_all_reached(unsigned* const* w, int R, int cta, int ncta, int nslice,
                                                 unsigned need, bool plus_bufs) {
    const int lane = threadIdx.x & 31;
    const int nsl = (nslice - cta + ncta - 1) / ncta;  // slices of this CTA
    bool ok = true;
    for (int e = lane; e < nsl * R; e += 32) {
        const int s = cta + (e / R) * ncta, q = e % R;
        const unsigned v = ld_relaxed_sys(w[q] + s);
        ok = ok && (plus_bufs ? v + kPavgBufs >= need : v >= need);
    }
    return __all_sync(0xffffffffu, ok);
}

// Run every averaging action this CTA can take now: apply rounds whose snapshots all peers have
// published, snapshot rounds that are due (due = rounds whose t * K images are claimed), and, when
// `final` (no images left to claim), wait until all the launch's rounds are applied.  All threads
// call it converged.  cta / ncta: this CTA's index among the replica's CTAs that own slices (the
// training CTAs, or the comm CTAs).  ctl: 4 ints + 8 64-bit sums of shared memory; ctl[0] / ctl[1]
// = rounds snapshotted / applied by this CTA in this launch (0 at the launch start).
template <int NT>
__device__ __noinline__ void pavg_service(float* params, const PavgArgs* pp, unsigned r0, int rounds, int cta,
                                          int ncta, int due, bool final, int* ctl) {
    const PavgArgs& p = *pp;
    const int R = p.R, me = p.rank, nslice = p.nslice, sfl = p.slice_fl;
    unsigned long long* sums = reinterpret_cast<unsigned long long*>(ctl + 4);
    unsigned waits = 0;  // thread 0: consecutive waits
    for (;;) {
        if (threadIdx.x < 32) {
            const int ts = ctl[0], tap = ctl[1];
            int act = 0;  // 0 leave, 1 snapshot, 2 apply, 3 wait
            if (tap < ts) {  // the oldest snapshotted round: have all peers published it?
                if (pavg_all_reached(p.flag, R, cta, ncta, nslice, r0 + static_cast<unsigned>(tap) + 1u, false)) act = 2;
            } else if (ts < due) {
                // next snapshot: only once this CTA's previous round is applied (rounds are sequential
                // per slice: a snapshot taken before an earlier round's apply would re-apply its
                // correction), and its ring buffer must be consumed by every peer
                const unsigned t = r0 + static_cast<unsigned>(ts) + 1u;
                const bool ok = t <= static_cast<unsigned>(kPavgBufs) ||
                                pavg_all_reached(p.done, R, cta, ncta, nslice, t, true);
                act = ok ? 1 : (final ? 3 : 0);  // blocked mid-launch: train on, retry at the next group
            }
            if (act == 0 && final && tap < rounds) act = 3;
            if (threadIdx.x == 0) {
                if (act == 1 || act == 2) fence_sys();  // acquire: the words just read precede what follows
                ctl[2] = act;
                sums[0] = 0ull;
                if (p.check)
                    for (int q = 1; q < kPavgMaxR; ++q) sums[q] = 0ull;
            }
        }
        __syncthreads();
        const int act = ctl[2];
        if (act == 0) break;
        if (act == 3) {
            // a peer that never publishes (a dead rank) would hang the launch: after ~10 s of waiting
            // give the launch's remaining rounds up and latch the error (reported by the next sync)
            if (threadIdx.x == 0) {
                __nanosleep(500);
                if (++waits > (1u << 24)) {
                    atomicOr(p.latch, kLatchPavgTimeout);
                    ctl[0] = ctl[1] = rounds;
                }
            }
        } else if (act == 1) {
            const unsigned t = r0 + static_cast<unsigned>(ctl[0]) + 1u;
            const int b = static_cast<int>(t % kPavgBufs);
            for (int s = cta; s < nslice; s += ncta) {
                const long long off = static_cast<long long>(s) * sfl;
                const int nq = static_cast<int>(min(static_cast<long long>(sfl), p.pint - off)) / 4;
                const float4* src = reinterpret_cast<const float4*>(params + off);
                float4* dst = reinterpret_cast<float4*>(p.snap[me] + (static_cast<long long>(b) * nslice + s) * sfl);
                unsigned long long ck = 0ull;
                for (int i = threadIdx.x; i < nq; i += NT) {
                    const float4 v = __ldcg(src + i);  // the live weights (the REDs land in L2)
                    dst[i] = v;
                    ck += bits4(v);
                }
                if (p.check) {  // per slice: block sum, written before the flag
                    atomicAdd(sums, ck);
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        p.cks[me][s * kPavgBufs + b] = sums[0];
                        sums[0] = 0ull;
                    }
                    __syncthreads();
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                fence_sys();  // release (cumulative over the CTA's stores ordered by the barrier)
                for (int s = cta; s < nslice; s += ncta) st_relaxed_sys(p.flag[me] + s, t);
                ++ctl[0];
            }
        } else {  // act == 2
            const unsigned t = r0 + static_cast<unsigned>(ctl[1]) + 1u;
            const int b = static_cast<int>(t % kPavgBufs);
            for (int s = cta; s < nslice; s += ncta) {
                const long long off = static_cast<long long>(s) * sfl;
                const int nq = static_cast<int>(min(static_cast<long long>(sfl), p.pint - off)) / 4;
                const long long soff = (static_cast<long long>(b) * nslice + s) * sfl;
                for (int i = threadIdx.x; i < nq; i += NT) {
                    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f), mine = sum;
                    for (int q = 0; q < R; ++q) {  // fixed order q = 0..R-1 on every replica
                        const float4 v = ld_relaxed_sys4(p.snap[q] + soff + 4 * i);
                        if (p.check) atomicAdd(sums + q, bits4(v));  // debug only: shared-memory atomics
                        if (q == 0) {
                            sum = v;
                        } else {
                            sum.x += v.x;
                            sum.y += v.y;
                            sum.z += v.z;
                            sum.w += v.w;
                        }
                        if (q == me) mine = v;
                    }
                    const float rf = static_cast<float>(R);
                    const float4 dl = make_float4(sum.x / rf - mine.x, sum.y / rf - mine.y, sum.z / rf - mine.z,
                                                  sum.w / rf - mine.w);
                    red_add4(params + off + 4 * i, dl);
                    if (p.check) {
                        red_add4(p.dsum + off + 4 * i, dl);
                        red_add4(p.dabs + off + 4 * i, make_float4(fabsf(dl.x), fabsf(dl.y), fabsf(dl.z), fabsf(dl.w)));
                    }
                }
                if (p.check) {
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        for (int q = 0; q < R; ++q)
                            if (sums[q] != *reinterpret_cast<volatile unsigned long long*>(p.cks[q] + s * kPavgBufs + b))
                                atomicOr(p.latch, kLatchPavg);
                        for (int q = 0; q < kPavgMaxR; ++q) sums[q] = 0ull;
                    }
                    __syncthreads();
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                fence_sys();  // the peer reads above complete before done is seen
                for (int s = cta; s < nslice; s += ncta) st_relaxed_sys(p.done[me] + s, t);
                ++ctl[1];
            }
        }
        __syncthreads();
    }
}

// A comm CTA (KArgs.pavg_comm > 0): trains nothing; polls the replica's claim counter and runs the
// averaging rounds of its slices (the slices are split over the comm CTAs only) until all of the
// launch's rounds are applied.  The training CTAs never stall on a round.
template <int NT>
__device__ __forceinline__ void pavg_comm_loop(const KArgs& a, int ccta, int* ctl) {
    const int rounds = static_cast<int>(a.pavg_rounds);
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned long long c = *reinterpret_cast<const volatile unsigned long long*>(a.counter);
            const bool fin = c >= static_cast<unsigned long long>(a.n);
            ctl[3] = static_cast<int>(fin ? a.pavg_rounds : min(a.pavg_rounds, static_cast<long long>(c) / a.pavg_k));
            ctl[2] = fin ? 1 : 0;  // (service overwrites ctl[2] after reading this copy)
        }
        __syncthreads();
        const int due = ctl[3];
        const bool fin = ctl[2] != 0;
        __syncthreads();
        pavg_service<NT>(a.params, a.pavg, static_cast<unsigned>(a.pavg_round0), rounds, ccta, a.pavg_comm, due, fin,
                         ctl);
        if (ctl[1] >= rounds) break;
        if (threadIdx.x == 0) __nanosleep(1000);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// PHASE(worker) The worker kernel: hogwild training, sync-batch gradients, evaluation, forward.
// ------------------------------------------------------------------------------------
// GATED (hogwild from host buffers only): claims wait for the copy stream's landed-images counter.
// REP (one-GPU emulation of replicas, hogwild only): CTA b runs replica b / a0.rep_ctas with that
// replica's arguments a0.reps[b / a0.rep_ctas].
template <bool REP>
__device__ __forceinline__ const KArgs& replica_args(const KArgs& a0) {
    if constexpr (REP)
        return a0.reps[blockIdx.x / a0.rep_ctas];
    else
        return a0;
}
// PAVG: the fused cross-replica averaging is compiled in (a separate instantiation: its mere presence
// costs the plain hogwild kernel ~1.4% -- measured, profiles/r4)
template <class Net, int G, int NT, int MODE, bool GATED = false, bool REP = false, bool PAVG = REP>
__global__ void __launch_bounds__(NT, 1) chaos_worker(KArgs a0) {
    static_assert(!REP || MODE == kHogwild, "replica emulation is hogwild only");
    static_assert(!PAVG || MODE == kHogwild, "fused averaging is hogwild only");
    const KArgs& a = replica_args<REP>(a0);
    const int cta = REP ? static_cast<int>(blockIdx.x) % a0.rep_ctas : static_cast<int>(blockIdx.x);
    const int ncta = REP ? a0.rep_ctas : static_cast<int>(gridDim.x);
    (void)cta;
    (void)ncta;
    using C1 = typename Net::C1;
    using C2 = typename Net::C2;
    using C3 = typename Net::C3;
    using F1 = typename Net::F1;
    using F2 = typename Net::F2;
    using O = POff<Net>;
    using S = SLayout<Net, G>;
    constexpr int NCONV = Net::NCONV, NFULL = Net::NFULL;
    constexpr int IMG = C1::IN_SZ;
    constexpr int SHALF = S::SFL / 2 / 4 * 4;
    constexpr bool TRAIN = (is_hog(MODE) || MODE == kSync);
    static_assert(MODE != kTrace || Net::TRACE, "kTrace is instantiated for nets with trace points only");
    // weight-buffer placement: W1 at 0, W2 at the tail (prefetched during conv1), W3 in two
    // halves (first half prefetched during conv2 into [0, W3A), second after conv2)
    // BIGW nets (Table I large): W1 at 0 and W2 right after it, both staged once per iteration
    // and kept (W2 serves the conv2 forward and delta_in); conv3 and FC1 read from L2
    constexpr bool BIG = S::BIG;
    constexpr int W2OFF = (NCONV >= 2) ? (BIG ? round4(C1::BLK) : S::WBUF - C2::BLK) : 0;
    constexpr int W3A = (NCONV >= 3 && !BIG) ? (C3::C / 2) * C3::NS : 0;
    static_assert(F1::BFL <= kBiasScratch && F2::BFL <= kBiasScratch, "FC bias-gradient scratch");
    static_assert(NCONV < 3 || BIG || W3A <= W2OFF, "W3 first half must not overlap W2");
    static_assert(!BIG || NCONV == 3, "BIGW nets have three conv layers");
    // FC1 weights staged through WB in two chunks of FRCH rows (large net: WB is free between
    // the conv3 forward and the conv3 backward, which re-fetches W3)
    constexpr bool FCSTAGE = (NCONV == 3) && (NFULL == 2) && (F1::IN % 4 == 0) && !BIG;
    // conv2 delta_in from a transposed W2 copy (pitch C2_WTP, odd), 3-conv staged nets
#ifndef CHAOS_C2_WTP
#define CHAOS_C2_WTP 1
#endif
#ifndef CHAOS_C2_GWM  // conv2 weight gradient: conv_gw_m with this many input maps per thread (0: conv_gw)
#define CHAOS_C2_GWM 4
#endif
#ifndef CHAOS_C3_DINP  // conv3 delta_in: the software-pipelined conv_din_winp
#define CHAOS_C3_DINP 1
#endif
#ifndef CHAOS_MGF_C1  // conv forwards with map groups fastest over the lanes (conv_fwd MGF)
#define CHAOS_MGF_C1 0
#endif
#ifndef CHAOS_MGF_C2
#define CHAOS_MGF_C2 0
#endif
#ifndef CHAOS_MGF_C3
#define CHAOS_MGF_C3 0
#endif
#ifndef CHAOS_C3_SPARSE  // conv3 backward: argmax-sparse conv_bwd_sparse (warp-uniform phase branches)
#define CHAOS_C3_SPARSE 1
#endif
#ifndef CHAOS_C2_PAR  // conv2 backward: delta_in (window-row bands, PB >= 2) beside conv_gw_m on the other warps
#define CHAOS_C2_PAR 0
#endif
#ifndef CHAOS_C2_TC  // conv2 forward on the tensor cores (conv_fwd_tc2) for nets that declare TC2:
#define CHAOS_C2_TC 0  // experimental, parity-green, measured slower (DESIGN.md §6 "tensor cores")
#endif
    // (G images fill the S and A2 regions enough to hold one operand stage each; else the FFMA path)
    constexpr bool TC2 = CHAOS_C2_TC && TcC2<Net>::value && NCONV >= 3 && !BIG && S::SFL * 4 >= kTcStageBytes &&
                         G * C2::OUT_SZ * 4 >= kTcStageBytes;
    constexpr bool C3_SPARSE = CHAOS_C3_SPARSE && NCONV >= 3 && !BIG && C3::KP == 2 && C3::M % 4 == 0 &&
                               C3::MP == C3::M && G * ((C3::C + 31) / 32) <= NT / 32;
    constexpr int C2_WTP = (CHAOS_C2_WTP && NCONV == 3 && !BIG && C2::DIN3 && C2::GWIN == 0) ? (C2::ROWS | 1) : 0;
    constexpr int FRCH = FCSTAGE ? (S::WBUF / (2 * F1::IN)) : 1;
    static_assert(!FCSTAGE || FRCH >= 1, "FC1 chunk must hold a row");
    static_assert(NCONV < 2 || C1::BLK <= W2OFF, "W1 and W2 must not overlap");
    static_assert(NCONV < 2 || C2::PB == 0 || G * C2::NBAND * ((C2::C + 31) / 32) <= NT / 32,
                  "conv_din3 needs one warp per (image, band, 32 maps)");
    static_assert(NCONV < 3 || C3::PB == 0 || G * C3::NBAND * ((C3::C + 31) / 32) <= NT / 32,
                  "conv_din3 needs one warp per (image, band, 32 maps)");

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // 6 mbarriers
    int* s_base = reinterpret_cast<int*>(smem + 64);
    int* s_lab = reinterpret_cast<int*>(smem + 80);                // G labels (<= 16)
    float* s_loss = reinterpret_cast<float*>(smem + 80 + 4 * 16);  // G losses
    int* pctl = reinterpret_cast<int*>(smem + 384);  // fused averaging: 4 control ints + 8 64-bit sums
    float* fa = reinterpret_cast<float*>(smem + kHdrBytes);
    float* sS = fa + S::S;
    float* a1 = fa + S::A1;
    float* a2 = fa + S::A2;
    float* a3 = fa + S::A3;
    float* hh = fa + S::HH;
    float* zz = fa + S::Z;
    float* bsc = fa + S::BS;
    float* wb = fa + S::WB;
    float* fwb = fa + S::WB + S::WBUF + S::DPB;  // S::FWB floats (tiny: FC weights)
    uint8_t* amb = smem + kHdrBytes + S::FLOATS * 4;
    uint8_t* am1 = amb + S::AM1;
    uint8_t* am2 = amb + S::AM2;
    uint8_t* am3 = amb + S::AM3;
    const float* P = a.params;
    const float sc = is_hog(MODE) ? a.neg_lr : 1.f;
    (void)a2;
    (void)a3;
    (void)am2;
    (void)am3;

    // tensor-core conv2 (conv_fwd_tc2): 9 more mbarriers in the header (full[4], empty[4], done) and
    // the whole TMEM (512 columns, one CTA per SM), allocated once for the kernel's lifetime
    uint64_t* tcbar = reinterpret_cast<uint64_t*>(smem + 256);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 48);
    uint32_t tc_done_phase = 0;
    (void)tcbar;
    (void)tc_done_phase;
    if (threadIdx.x == 0) {
        pctl[0] = pctl[1] = pctl[3] = 0;
        for (int k = 0; k < 6; ++k) mbar_init(bars + k, 1);
        if constexpr (TC2) {
            for (int k = 0; k < 4; ++k) {
                mbar_init(tcbar + k, NT / 32 - 1);  // full: one arrival per producer warp
                mbar_init(tcbar + 4 + k, 1);        // empty: the MMA commit
            }
            mbar_init(tcbar + 8, 1);  // done
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (TC2) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "n"(kTcCols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (TC2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = TC2 ? *tmem_slot : 0u;
    (void)tmem;
    if constexpr (PAVG) {
        static_assert(!TC2, "comm CTAs return before the TMEM teardown");
        if (a.pavg && a.pavg_comm > 0 && cta >= ncta - a.pavg_comm) {
            pavg_comm_loop<NT>(a, cta - (ncta - a.pavg_comm), pctl);
            return;
        }
    }
    Loader L0{bars + 0, 0u}, L1{bars + 1, 0u}, L2{bars + 2, 0u}, L3{bars + 3, 0u};
    Loader L4{bars + 4, 0u}, L5{bars + 5, 0u};  // FC1 weight chunks (double buffer)
    (void)L4;
    (void)L5;

    long long iter = 0;
    long long next_claim = -1;  // hogwild: thread 0 claims the next group during the backward pass
    int pending_progress = 0;   // hogwild: images of the previous iteration not yet counted in a.progress
    long long t_last = clock64();
    (void)t_last;
    if constexpr (MODE == kTrace)  // debug: CTA b starts b * stagger cycles late (varied interleavings)
        if (threadIdx.x == 0 && a.stagger > 0)
            while (clock64() - t_last < a.stagger * static_cast<long long>(blockIdx.x)) __nanosleep(1000);
    for (;;) {
        // ---------------- a1: claim the next unprocessed images
        if (threadIdx.x == 0) {
            long long base;
            if constexpr (is_hog(MODE)) {
                base = next_claim >= 0 ? next_claim
                                       : static_cast<long long>(atomicAdd(a.counter, static_cast<unsigned long long>(G)));
                if constexpr (GATED)  // host entry: the copy stream advances *ready after each chunk
                    if (base < a.n) wait_landed(a.ready, static_cast<unsigned long long>(min(base + G, a.n)));
            } else {
                base = (static_cast<long long>(blockIdx.x) + iter * gridDim.x) * G;
            }
            *s_base = base < a.n ? static_cast<int>(base) : -1;
            if constexpr (PAVG)  // fused averaging: rounds whose t * K images are claimed
                if (a.pavg && a.pavg_comm == 0)
                    pctl[3] = static_cast<int>(base < a.n ? min(a.pavg_rounds, base / a.pavg_k) : a.pavg_rounds);
        }
        fence_proxy_async();  // earlier generic smem / global accesses precede the async proxy
        __syncthreads();
        const int base = *s_base;
        if constexpr (PAVG)
            if (a.pavg && a.pavg_comm == 0)
                pavg_service<NT>(a.params, a.pavg, static_cast<unsigned>(a.pavg_round0), static_cast<int>(a.pavg_rounds),
                                 cta, ncta, pctl[3], base < 0, pctl);
        PTIME(0);
        if (base < 0) break;
        const int slot = static_cast<int>(base / G);
        const int cnt = static_cast<int>(min(static_cast<long long>(G), a.n - base));
        ++iter;
        if constexpr (MODE == kTrace) {
            if (threadIdx.x == 0) {
                a.trec[static_cast<long long>(slot) * kTraceRec + 30] = blockIdx.x;
                a.trec[static_cast<long long>(slot) * kTraceRec + 31] = iter - 1;
            }
        }
        TR_RB(0, 0);  // W1 (and W2 / the staged FC weights) are read from here on
        if constexpr (NCONV >= 2 || S::FWB > 0) TR_RB(1, 0);
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
            if constexpr (is_hog(MODE))
                if (a.claims) atomicAdd(a.claims + base + threadIdx.x, 1);
        }
        // stage images (bulk when 16-B aligned) + W1 on bar0, prefetch W2 on bar1
        const float* xsrc = a.images + static_cast<long long>(base) * IMG;
        const bool x_bulk = ((reinterpret_cast<uintptr_t>(xsrc) & 15u) == 0) && ((cnt * IMG) % 4 == 0);
        if (threadIdx.x == 0) {
            mbar_expect_tx(bars + 0, static_cast<uint32_t>(C1::BLK + (x_bulk ? cnt * IMG : 0)) * 4u);
            bulk_g2s(wb, P + O::c1w, static_cast<uint32_t>(C1::BLK) * 4u, bars + 0);
            if (x_bulk)
                for (int off = 0; off < cnt * IMG; off += 16384) {
                    const int chunk = (cnt * IMG - off) > 16384 ? 16384 : (cnt * IMG - off);
                    bulk_g2s(sS + off, xsrc + off, static_cast<uint32_t>(chunk) * 4u, bars + 0);
                }
        }
        if constexpr (NCONV >= 2) L1.issue(wb + W2OFF, P + O::c2w, C2::BLK);
        if constexpr (S::FWB > 0) L1.issue(fwb, P + O::f1w, S::FWB);  // FC W then b (contiguous)
        if (!x_bulk)
            for (int i = threadIdx.x; i < cnt * IMG; i += NT) sS[i] = __ldg(xsrc + i);
        L0.wait();
        if (!x_bulk) __syncthreads();
        TR_RE(0, 0);
        TR_DUMP(0, O::c1w, wb, C1::BLK);
        PTIME(1);

        // ---------------- a2: conv -> tanh -> pool, layer by layer
#ifndef CHAOS_PL_C1  // conv1 / conv3 forward: image-pair lane map with this many windows per warp (0: off)
#define CHAOS_PL_C1 0
#endif
#ifndef CHAOS_PL_C3
#define CHAOS_PL_C3 4
#endif
        constexpr int PL1 = (NCONV >= 3 && !BIG && !CHAOS_MGF_C1 && C1::NSPL == 1 && (C1::IN_SZ & 1)) ? CHAOS_PL_C1 : 0;
#ifndef CHAOS_TAIL_C1  // conv1 forward: split the last partial pass into single-map sub-items (1: every
#define CHAOS_TAIL_C1 0  // net, for sweeps; else the nets that declare TAIL1 -- measured per net)
#endif
        constexpr bool TAIL1 = (CHAOS_TAIL_C1 || Tail1<Net>::value) && PL1 == 0 && !CHAOS_MGF_C1 && C1::NSPL == 1;
        conv_fwd<C1, NT, CHAOS_MGF_C1, PL1, TAIL1>(sS, wb, a1, am1, cnt);
        float* alast = a1;
        if constexpr (NCONV >= 2) {
            fence_async_smem();
            __syncthreads();
            PTIME(2);
            if constexpr (NCONV >= 3 && !BIG && !TC2) TR_RB(2, 0);
            if constexpr (NCONV >= 3 && !BIG && !TC2)
                L2.issue(wb, P + O::c3w, W3A);  // W1 region is dead: W3's first half
            L1.wait();
            TR_RE(1, 0);
            if constexpr (!BIG) TR_DUMP(0, O::c2w, wb + W2OFF, C2::BLK);
            if constexpr (TC2) {  // the W1 region [0, 20 KB x 2) holds the operand stages; W3 comes after
                static_assert(2 * kTcStageBytes + 4 * 256 <= W2OFF * 4, "tensor-core stages must not overlap W2");
                static_assert(S::SFL * 4 >= kTcStageBytes && G * C2::OUT_SZ * 4 >= kTcStageBytes,
                              "S and A2 each hold one operand stage");
                conv_fwd_tc2<C2, NT, G>(a1, wb + W2OFF, a2, am2, cnt, tmem, reinterpret_cast<unsigned char*>(wb),
                                        reinterpret_cast<unsigned char*>(sS), reinterpret_cast<unsigned char*>(a2), tcbar,
                                        tc_done_phase, a.ptime ? a.ptime + blockIdx.x * kPhases + 17 : nullptr);
            } else {
                conv_fwd<C2, NT, CHAOS_MGF_C2 || MgfC2<Net>::value>(a1, wb + W2OFF, a2, am2, cnt);
            }
            alast = a2;
        }
        if constexpr (NCONV >= 3 && BIG) {
            static_assert(3 * C3::KK * C3::MP <= G * C1::OUT_SZ, "conv3 weight ring must fit in A1");
            sync_for_async();  // A1 (read by the conv2 forward) becomes the conv3 weight ring
            PTIME(3);
            conv_fwd_slab<C3, NT>(a2, P + O::c3w, a3, am3, a1, L2, L3, L4);
            alast = a3;
        } else if constexpr (NCONV >= 3) {
            fence_async_smem();
            __syncthreads();
            PTIME(3);
            if constexpr (TC2) {
                TR_RB(2, 0);
                L2.issue(wb, P + O::c3w, W3A);
            }
            L3.issue(wb + W3A, P + O::c3w + W3A, C3::BLK - W3A);
            L2.wait();
            L3.wait();
            TR_RE(2, 0);
            TR_DUMP(0, O::c3w, wb, C3::BLK);
            constexpr int PL3 = (!CHAOS_MGF_C3 && C3::NSPL == 1 && C3::P <= 16) ? CHAOS_PL_C3 : 0;
            conv_fwd<C3, NT, CHAOS_MGF_C3, PL3>(a2, wb, a3, am3, cnt);
            alast = a3;
        }
        fence_async_smem();  // WB (read by the conv forward) is refilled by the async proxy next
        __syncthreads();
        PTIME(4);
        // ---------------- a3: full layers
        if constexpr (NFULL == 2) {
            TR_RB(3, 0);
            TR_RB(3, 1);  // FC1's delta_in reuses chunks staged now and re-fetches the others later
            if constexpr (FCSTAGE && MODE == kTrace)
                fc_fwd3<F1, G, NT, FRCH, MODE>(P + O::f1w, P + O::f1b, alast, hh, F1::OUT, cnt, wb, L4, L5, sS, &a,
                                               slot, O::f1w);
            else if constexpr (FCSTAGE)
                fc_fwd3<F1, G, NT, FRCH>(P + O::f1w, P + O::f1b, alast, hh, F1::OUT, cnt, wb, L4, L5, sS);
            else if constexpr (F1::IN % 4 == 0)
#ifndef CHAOS_FC2_NR  // fc_fwd2 rows per warp task for NT <= 512 (medium: 150 rows)
#define CHAOS_FC2_NR 5
#endif
                fc_fwd2<F1, G, NT, (NT > 512 || BIG ? 2 : CHAOS_FC2_NR)>(P + O::f1w, P + O::f1b, alast, hh, F1::OUT, cnt);
            else
                fc_fwd<F1, G, NT>(P + O::f1w, P + O::f1b, alast, hh, F1::OUT, cnt);
            __syncthreads();
            PTIME(16);
            TR_RE(3, 0);
            TR_RB(4, 0);
            if constexpr (MODE == kTrace)
                fc_fwd<F2, G, NT, false, true>(P + O::f2w, P + O::f2b, hh, zz, kZStride, cnt,
                                               a.tw + static_cast<long long>(slot) * 2 * a.pstride + O::f2w);
            else
                fc_fwd<F2, G, NT>(P + O::f2w, P + O::f2b, hh, zz, kZStride, cnt);
        } else {
            if constexpr (S::FWB > 0) {
                L1.wait();
                TR_RE(1, 0);
                TR_DUMP(0, O::f1w, fwb, S::FWB);
                fc_fwd<F1, G, NT, true>(fwb, fwb + F1::WFL, alast, zz, kZStride, cnt);
            } else {
                fc_fwd<F1, G, NT>(P + O::f1w, P + O::f1b, alast, zz, kZStride, cnt);
            }
        }
        __syncthreads();
        if constexpr (NFULL == 2) TR_RE(4, 0);
        PTIME(5);
        // ---------------- a4: softmax cross-entropy, output delta.  16 lanes per image (class o =
        // lane % 16), two images per warp: the maximum, the sum and the loss are shuffle trees in a
        // fixed order (deterministic), every exp in parallel.  Reading R18: with r = the sum of
        // exp(z_o - zmax) over the classes other than the first maximum (which contributes exactly
        // 1), loss = log1p(r) + zmax - z[lab] and, when the label is that maximum,
        // delta[lab] = p[lab] - 1 = -r / (1 + r): the values of log(s) and p - onehot without their
        // cancellation once p[lab] -> 1 (a trained net)
        if constexpr (MODE == kForward) {
            if (threadIdx.x < cnt) {
                const int g = threadIdx.x;
                for (int o = 0; o < kClasses; ++o)
                    a.out_logits[(static_cast<long long>(base) + g) * kClasses + o] = zz[g * kZStride + o];
            }
        } else if (threadIdx.x < 32 * ((G + 1) / 2)) {
            static_assert(kClasses <= 16 && kZStride >= kClasses, "16 lanes per image");
            const int g = threadIdx.x >> 4, o = threadIdx.x & 15;
            const bool on = g < cnt && o < kClasses;
            float* z = zz + (g < cnt ? g : 0) * kZStride;
            const int lab = s_lab[g < cnt ? g : 0];
            const float zo = on ? z[o] : -INFINITY;
            // first maximum: the largest value, ties to the lowest class
            float zmax = zo;
            int best = on ? o : 16;
#pragma unroll
            for (int k = 8; k >= 1; k >>= 1) {
                const float zv = __shfl_xor_sync(0xffffffffu, zmax, k);
                const int bv = __shfl_xor_sync(0xffffffffu, best, k);
                if (zv > zmax || (zv == zmax && bv < best)) {
                    zmax = zv;
                    best = bv;
                }
            }
            const float e = (on && o != best) ? expf(zo - zmax) : 0.f;
            float r = e;
#pragma unroll
            for (int k = 8; k >= 1; k >>= 1) r += __shfl_xor_sync(0xffffffffu, r, k);
            const float zlab = __shfl_sync(0xffffffffu, zo, (threadIdx.x & 16) + lab);
            const float loss = log1pf(r) + zmax - zlab;
            if (on && o == 0) {
                if (!isfinite(loss)) atomicOr(a.latch, kLatchNonfinite);
                if constexpr (MODE == kEval) {
                    a.out_loss[base + g] = loss;
                    a.out_wrong[base + g] = static_cast<unsigned char>(best != lab);
                } else {
                    s_loss[g] = loss;
                }
            }
            if constexpr (MODE != kEval) {
                if (on) {
                    const float inv = 1.f / (1.f + r);
                    z[o] = (o != lab) ? (o == best ? inv : e * inv) : (lab == best ? -r * inv : e * inv - 1.f);
                }
            }
        }
        if constexpr (TRAIN) {
            __syncthreads();
            PTIME(6);
            if constexpr (is_hog(MODE))  // the claim's round trip overlaps the backward pass
                if (threadIdx.x == 0) {
                    next_claim = static_cast<long long>(atomicAdd(a.counter, static_cast<unsigned long long>(G)));
                    if (pending_progress && a.progress)
                        atomicAdd(a.progress, static_cast<unsigned long long>(pending_progress));
                    pending_progress = 0;
                }
            if (threadIdx.x == 0 && a.loss_sum) {
                double ls = 0.0;
                for (int g = 0; g < cnt; ++g) ls += s_loss[g];
                atomicAdd(a.loss_sum, ls);
            }
            // ---------------- a5: full layers backward, one bulk publish per chunk / layer
            if constexpr (NFULL == 2) {
                TR_RB(4, 1);
                TR_PB(4);
                fc_bwd<F2, G, NT, MODE, SHALF>(a, slot, O::f2w, O::f2b, hh, zz, kZStride, sS, bsc, cnt, sc);
                wait_publish_reads();
                TR_RE(4, 1);
                TR_PE(4);
                PTIME(7);
                if constexpr (BIG) {
                    constexpr int NRG = NT / (F1::IN / 4) < 4 ? NT / (F1::IN / 4) : 4;
                    static_assert(NRG >= 1 && (NRG - 1) * G * F1::IN <= S::SFL, "row-group partials must fit in S");
                    fc_bwd2<F1, G, NT, MODE, NRG>(a, slot, O::f1w, O::f1b, alast, hh, F1::OUT, sS, bsc, cnt, sc);
                } else if constexpr (FCSTAGE) {
#ifndef CHAOS_FC1_NRG  // FC1 backward: row groups (threads per column quad)
#define CHAOS_FC1_NRG 5
#endif
                    constexpr int NRG = NT / (F1::IN / 4) < CHAOS_FC1_NRG ? NT / (F1::IN / 4) : CHAOS_FC1_NRG;
                    static_assert((NRG - 1) * G * F1::IN <= S::SFL, "row-group partials must fit in S");
                    fence_async_smem();
                    wait_publish_reads();  // the FC2 publish has read its buffers; WB is free
                    TR_PB(3);
                    fc_bwd3<F1, G, NT, MODE, NRG, FRCH, true>(a, slot, O::f1w, O::f1b, alast, hh, F1::OUT, sS, bsc,
                                                               cnt, sc, wb, L4, L5);
                } else if constexpr (F1::IN % 4 == 0 && (F1::IN / 4) * 4 <= NT) {
                    constexpr int NRG = NT / (F1::IN / 4) < 4 ? NT / (F1::IN / 4) : 4;
                    static_assert((NRG - 1) * G * F1::IN <= S::SFL, "row-group partials must fit in S");
                    fc_bwd2<F1, G, NT, MODE, NRG>(a, slot, O::f1w, O::f1b, alast, hh, F1::OUT, sS, bsc, cnt, sc);
                } else {
                    fc_bwd<F1, G, NT, MODE, SHALF>(a, slot, O::f1w, O::f1b, alast, hh, F1::OUT, sS, bsc, cnt, sc);
                }
            } else if constexpr (S::FWB > 0) {
                // tiny: the gradient chunk goes to S's upper half, so the images in its lower half
                // survive for conv1's gradient (no reload, no wait for the publish's reads here)
                static_assert(F1::WFL <= SHALF && G * IMG <= SHALF, "one chunk above the images");
                TR_PB(1);
                fc_bwd<F1, G, NT, MODE, SHALF>(a, slot, O::f1w, O::f1b, alast, zz, kZStride, sS + SHALF, bsc, cnt,
                                               sc, fwb);
                __syncthreads();
                TR_PE(1);
            } else {
                fc_bwd<F1, G, NT, MODE, SHALF>(a, slot, O::f1w, O::f1b, alast, zz, kZStride, sS, bsc, cnt, sc);
            }
            if constexpr (S::FWB == 0) wait_publish_reads();
            if constexpr (NFULL == 2) {
                TR_RE(3, 1);
                TR_PE(3);
            }
            PTIME(8);
            // ---------------- a6/a7: pool + conv backward, publish per layer
            if constexpr (NCONV == 3 && BIG) {
                // conv3 delta_in first (W3 read from L2 before this worker publishes its
                // gradient: the pre-update weights for one worker, R5) into the dead A1 region,
                // then the weight gradient (reads a2), then the delta back over a2; A1 is then
                // recomputed (conv1 forward again, same image and staged W1) for conv2's backward.
                // W1 and W2 stay staged from the forward pass (the snapshot it used).
                static_assert(G * C2::OUT_SZ <= G * C1::OUT_SZ, "conv3 delta_in must fit in A1");
                conv_din_gm<C3, NT, Net::RB3>(P + O::c3w, a3, am3, a2, a1, cnt);
                __syncthreads();
                PTIME(9);
#ifndef CHAOS_PL_GW_NM  // tile sweeps (Table I large conv3 weight gradient)
#define CHAOS_PL_GW_NM 4
#endif
#ifndef CHAOS_PL_GW_KR
#define CHAOS_PL_GW_KR 3
#endif
                conv_gw_wt<C3, NT, MODE, CHAOS_PL_GW_NM, CHAOS_PL_GW_KR>(a, slot, a2, a3, am3, O::c3w, cnt, sc);
                __syncthreads();
                PTIME(10);
                for (int e = threadIdx.x; e < cnt * C2::OUT_SZ; e += NT) a2[e] = a1[e];
                fence_async_smem();
                wait_publish_reads();  // S (FC scratch, bulk-published) takes the image again
                if (x_bulk) {
                    L0.issue(sS, xsrc, cnt * IMG);
                    L0.wait();
                } else {
                    for (int i = threadIdx.x; i < cnt * IMG; i += NT) sS[i] = __ldg(xsrc + i);
                    __syncthreads();
                }
                conv_fwd<C1, NT>(sS, wb, a1, am1, cnt);
                __syncthreads();
                PTIME(11);
                conv_gw<C2, NT, MODE, false>(a, slot, a1, a2, am2, nullptr, O::c2w, cnt, sc);
                __syncthreads();
                PTIME(12);
                conv_din_gm<C2, NT, C2::RB, false>(wb + W2OFF, a2, am2, a1, a1, cnt);
                __syncthreads();
                PTIME(13);
            } else if constexpr (NCONV == 3) {
                if constexpr (FCSTAGE) {
                    // W3 again (the FC1 chunks used its buffer); this worker has not published
                    // layer 3 yet, so for one worker it is the snapshot the forward used (R5)
                    fence_async_smem();
                    __syncthreads();
                    TR_RB(2, 1);
                    L2.issue(wb, P + O::c3w, C3::BLK);
                    L2.wait();
                    TR_RE(2, 1);
                    TR_DUMP(1, O::c3w, wb, C3::BLK);
                }
                TR_PB(2);
                // otherwise W3 is still staged from the forward pass (the exact snapshot it used)
                if constexpr (C3_SPARSE) {
                    int* ctr = reinterpret_cast<int*>(smem + 72);  // header word (kHdrBytes), reset here
                    if (threadIdx.x == 0) *ctr = 0;
                    __syncthreads();
#ifndef CHAOS_C3_MS  // conv3 delta_in: warps per (image, 32 input maps) task
#define CHAOS_C3_MS 1
#endif
                    constexpr int C3MS = (G * ((C3::C + 31) / 32) * CHAOS_C3_MS <= NT / 32) ? CHAOS_C3_MS : 1;
                    conv_bwd_sparse<C3, NT, MODE, C3MS>(a, slot, wb, a3, am3, a2, sS, O::c3w, cnt, sc, ctr);
                    __syncthreads();
                    PTIME(9);
                } else if constexpr (C3::GWIN > 0) {
                    // delta_in (latency-bound, one warp per (image, 32 maps)) and the dense
                    // weight gradient (issue-bound, published from registers) side by side
                    constexpr int DW = G * C3::NBAND * ((C3::C + 31) / 32);
                    static_assert(C3::PB > 0 && C3::NBAND == 1 && DW < NT / 32, "conv3 split");
                    if constexpr (C3::DWIN && G * C3::OUT_SZ * 4 <= S::SFL) {
                        // phase-expanded delta, once: dq4[g][m][w] = d at component phase (S is free here)
                        float4* dq4 = reinterpret_cast<float4*>(sS);
                        for (int e = threadIdx.x; e < cnt * C3::OUT_SZ; e += NT) {
                            const float d = a3[e];
                            const int ph = am3[e];
                            dq4[e] = make_float4(ph == 0 ? d : 0.f, ph == 1 ? d : 0.f, ph == 2 ? d : 0.f, ph == 3 ? d : 0.f);
                        }
                        __syncthreads();
#ifdef CHAOS_TIMING
                        const long long t_split = clock64();  // slots 17 / 18: the two warp groups' own time
#endif
                        if (threadIdx.x < DW * 32) {
                            if constexpr (CHAOS_C3_DINP)
                                conv_din_winp<C3, NT, true>(wb, a2, sS, cnt, dq4);  // output over dq4 after
                            else
                                conv_din_win<C3, NT, true>(wb, a3, am3, a2, sS, cnt, dq4);  // output over dq4 after
#ifdef CHAOS_TIMING
                            if (threadIdx.x == 0 && a.ptime) a.ptime[blockIdx.x * kPhases + 17] += clock64() - t_split;
#endif
                        } else {
                            conv_gw_win<C3, NT, MODE, C3::GWIN, DW, NT / 32 - DW>(a, slot, a2, a3, am3, O::c3w, cnt,
                                                                                  sc, dq4);
#ifdef CHAOS_TIMING
                            if (threadIdx.x == DW * 32 && a.ptime) a.ptime[blockIdx.x * kPhases + 18] += clock64() - t_split;
#endif
                            __syncthreads();  // pairs with conv_din_win's deferral barrier
                        }
                    } else {
                        if (threadIdx.x < DW * 32) {
                            static_assert(C3::DWIN, "conv3 delta_in beside the dense weight gradient: conv_din_win");
                            conv_din_win<C3, NT>(wb, a3, am3, a2, sS, cnt);
                        }
                        conv_gw_win<C3, NT, MODE, C3::GWIN, DW, NT / 32 - DW>(a, slot, a2, a3, am3, O::c3w, cnt, sc);
                    }
                    __syncthreads();
                    PTIME(9);
                } else {
                if constexpr (C3::DIN3)
                    conv_din3<C3, NT>(wb, a3, am3, a2, sS, nullptr, cnt);  // delta for the pool2 outputs -> S
                else
                    conv_din<C3, NT>(wb, a3, am3, a2, sS, cnt);
                __syncthreads();
                PTIME(9);
                conv_gw<C3, NT, MODE, true>(a, slot, a2, a3, am3, wb, O::c3w, cnt, sc);
                }
                fence_async_smem();
                wait_publish_reads();
                TR_PE(2);
                PTIME(10);
                TR_RB(1, 1);
                L1.issue(wb, P + O::c2w, C2::BLK);  // W2 again (pre-update snapshot for delta_in)
                L1.wait();
                TR_RE(1, 1);
                TR_DUMP(1, O::c2w, wb, C2::BLK);
                // transposed W2 copy [m][C*K*K] (odd pitch) for the delta_in's lanes over input maps, made
                // by the warps the weight gradient leaves idle (or here when it uses them all); ordered
                // before the delta_in's reads by the barrier after the weight gradient
                constexpr int GWW = (C2::M * (C2::C / (CHAOS_C2_GWM > 0 ? CHAOS_C2_GWM : 1)) + 31) / 32;
                constexpr bool WT_OVERLAP = C2_WTP > 0 && C2::MS < 0 && CHAOS_C2_GWM > 0 && GWW < NT / 32 &&
                                            !CHAOS_C2_PAR;
                auto transpose_w2 = [&](int t0, int nthr) {
                    static_assert(C2_WTP == 0 || round4(C2::BLK) + C2::M * C2_WTP <= S::WBUF,
                                  "transposed W2 must fit in WB");
                    float* wbt = wb + round4(C2::BLK);
                    static_assert(C2::NPAD == 0, "W2 transpose from [C*K*K][MP] rows");
                    for (int e = static_cast<int>(threadIdx.x) - t0; e < C2::ROWS * C2::M; e += nthr)
                        wbt[(e % C2::M) * C2_WTP + e / C2::M] = wb[(e / C2::M) * C2::MP + e % C2::M];
                };
                if constexpr (C2_WTP > 0 && !WT_OVERLAP) transpose_w2(0, NT);
                PTIME(11);
                TR_PB(1);
                if constexpr (CHAOS_C2_PAR && C2::MS < 0 && CHAOS_C2_GWM > 0 && C2::NBAND > 1 && C2::GWIN == 0) {
                    // delta_in (one warp per (image, band), latency-bound) and the weight gradient
                    // (LSU-bound, lanes over output maps) side by side; the delta_in's writes over a1
                    // wait for its hand-off barrier, which the gradient warps join once done reading a1
                    constexpr int DW = G * C2::NBAND * ((C2::C + 31) / 32);
                    static_assert(C2::DIN3 && DW < NT / 32, "conv2 split");
                    static_assert(G * C2::HAND <= S::Z - S::A2, "conv2 hand-off must fit in the dead A2/A3/HH regions");
                    if (threadIdx.x < DW * 32) {
                        if constexpr (C2_WTP > 0)
                            conv_din3<C2, NT, true, C2_WTP>(wb + round4(C2::BLK), sS, am2, a1, a1, a2, cnt);
                        else
                            conv_din3<C2, NT, true>(wb, sS, am2, a1, a1, a2, cnt);
                    } else {
                        conv_gw_m<C2, NT, MODE, CHAOS_C2_GWM, DW, NT / 32 - DW>(a, slot, a1, sS, am2, O::c2w, cnt, sc);
                        __syncthreads();  // pairs with conv_din3's hand-off barrier
                    }
                    __syncthreads();
                    TR_PE(1);
                    PTIME(12);
                    PTIME(13);
                } else if constexpr (C2::GWIN > 0) {
                    // delta_in (din3: one warp per (image, band), latency-bound) and the dense
                    // weight gradient (issue-bound, published from registers) side by side; the
                    // delta_in writes over a1 wait for its hand-off barrier, by which time the
                    // weight-gradient warps have finished reading a1
                    constexpr int DW = G * C2::NBAND * ((C2::C + 31) / 32);
                    static_assert(C2::DIN3 && C2::NBAND > 1 && DW < NT / 32, "conv2 split");
                    static_assert(G * C2::HAND <= S::Z - S::A2, "conv2 hand-off must fit in the dead A2/A3/HH regions");
                    if (threadIdx.x < DW * 32) {
                        conv_din3<C2, NT, true>(wb, sS, am2, a1, a1, a2, cnt);
                    } else {
                        conv_gw_win<C2, NT, MODE, C2::GWIN, DW, NT / 32 - DW>(a, slot, a1, sS, am2, O::c2w, cnt, sc);
                        __syncthreads();  // pairs with conv_din3's hand-off barrier
                    }
                    __syncthreads();
                    PTIME(12);
                    PTIME(13);
                } else {
                if constexpr (WT_OVERLAP) {  // the gradient on warps [0, GWW), the W2 transpose on the others
                    if (threadIdx.x < GWW * 32)
                        conv_gw_m<C2, NT, MODE, CHAOS_C2_GWM, 0, GWW>(a, slot, a1, sS, am2, O::c2w, cnt, sc);
                    else
                        transpose_w2(GWW * 32, NT - GWW * 32);
                } else if constexpr (C2::MS < 0 && CHAOS_C2_GWM > 0)  // lanes over output maps, NPT maps per thread
                    conv_gw_m<C2, NT, MODE, CHAOS_C2_GWM>(a, slot, a1, sS, am2, O::c2w, cnt, sc);
                else if constexpr (C2::MS < 0)  // generic, lanes over output maps, published from registers
                    conv_gw<C2, NT, MODE, false>(a, slot, a1, sS, am2, nullptr, O::c2w, cnt, sc);
                else
                    conv_gw<C2, NT, MODE, true>(a, slot, a1, sS, am2, wb + C2::BLK, O::c2w, cnt, sc);
                __syncthreads();
                TR_PE(1);
                PTIME(12);
                if constexpr (C2::PB > 0) {
                    static_assert(G * C2::HAND <= S::A3 - S::A2 + (S::HH - S::A3) + (S::Z - S::HH),
                                  "conv2 hand-off must fit in the dead A2/A3/HH regions");
                    if constexpr (C2::DIN3 && C2_WTP > 0)
                        conv_din3<C2, NT, false, C2_WTP>(wb + round4(C2::BLK), sS, am2, a1, a1, a2, cnt);
                    else
                        conv_din3<C2, NT>(wb, sS, am2, a1, a1, a2, cnt);  // a2..HH are dead here
                } else {
                    conv_din<C2, NT>(wb, sS, am2, a1, a1, cnt);
                }
                __syncthreads();
                PTIME(13);
                }
            } else if constexpr (NCONV == 2) {
                // W2 is still staged from the forward pass at W2OFF
                conv_gw<C2, NT, MODE, false>(a, slot, a1, a2, am2, nullptr, O::c2w, cnt, sc);
                __syncthreads();
                PTIME(12);
                if constexpr (DinRows<Net>::value && DinPair<Net>::value > 1)
                    conv_din_rows<C2, NT, DinPair<Net>::value>(wb + W2OFF, a2, am2, a1, a1, cnt, wb + S::WBUF);
                else if constexpr (DinPair<Net>::value > 1)
                    conv_din<C2, NT, DinPair<Net>::value>(wb + W2OFF, a2, am2, a1, a1, cnt, wb + S::WBUF);
                else
                    conv_din<C2, NT>(wb + W2OFF, a2, am2, a1, a1, cnt);
                __syncthreads();
                PTIME(13);
            }
            // conv1: the images again (S was reused as scratch), then its gradient
            if constexpr (S::FWB == 0) {
                fence_async_smem();
                wait_publish_reads();
                if (x_bulk) {
                    L0.issue(sS, xsrc, cnt * IMG);
                    L0.wait();
                } else {
                    for (int i = threadIdx.x; i < cnt * IMG; i += NT) sS[i] = __ldg(xsrc + i);
                    __syncthreads();
                }
            }
            PTIME(14);
            TR_PB(0);
            conv_gw<C1, NT, MODE, true>(a, slot, sS, a1, am1, wb, O::c1w, cnt, sc);
            if (threadIdx.x == 0) bulk_wait_all<0>();  // publishes complete before the next claim
            TR_PE(0);
#ifndef CHAOS_NO_ITER_FENCE
            if constexpr (is_hog(MODE)) __threadfence();  // this worker's REDs precede its next reads
#endif
            if constexpr (is_hog(MODE))  // progress for the asynchronous cross-GPU averaging: the
                pending_progress = cnt;     // reduction is issued during the next iteration (off the fences)
        }
        __syncthreads();
        PTIME(15);
    }
    if (threadIdx.x == 0) bulk_wait_all<0>();
    if constexpr (TC2) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcCols) : "memory");
    }
    if constexpr (is_hog(MODE))
        if (threadIdx.x == 0 && pending_progress && a.progress)
            atomicAdd(a.progress, static_cast<unsigned long long>(pending_progress));
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
        params[j] = fmaf(-lr, s, params[j]);
}

// w[j] -= lr * grad[j] (the sync update from an externally reduced gradient: multi-GPU sync).
// Same single-rounding expression as chaos_reduce_update, so one GPU reproduces it bitwise.
__global__ void chaos_apply_gradient_kernel(float* __restrict__ params, const float* __restrict__ grad, float lr,
                                            long long np) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < np) params[j] = fmaf(-lr, grad[j], params[j]);
}

// Asynchronous cross-GPU averaging: w[j] += avg[j] - snap[j]
// with vector REDs, so the local updates a running hogwild launch adds meanwhile are kept.
__global__ void chaos_avg_apply_kernel(float* __restrict__ params, const float* __restrict__ avg,
                                       const float* __restrict__ snap, long long np) {
    const long long nq = np / 4;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
        const float4 x = reinterpret_cast<const float4*>(avg)[q], y = reinterpret_cast<const float4*>(snap)[q];
        red_add4(params + 4 * q, make_float4(x.x - y.x, x.y - y.y, x.z - y.z, x.w - y.w));
    }
    for (long long j = 4 * nq + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < np; j += stride)
        red_add(params + j, avg[j] - snap[j]);
}

// Returns once the hogwild progress counter reaches target (one thread; polls L2).  The training
// kernel never waits on it, so it cannot deadlock: at worst it runs after the training launch.
__global__ void chaos_progress_wait_kernel(const unsigned long long* progress, unsigned long long target) {
    if (threadIdx.x != 0) return;
    while (*reinterpret_cast<const volatile unsigned long long*>(progress) < target) __nanosleep(2000);
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
