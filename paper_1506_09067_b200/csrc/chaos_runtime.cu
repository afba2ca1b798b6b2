// chaos_runtime.cu -- host runtime and C ABI of libchaos.so (see include/chaos.h).
//
// Owns: arch validation and matching against the compiled sm_100a instantiations,
// the internal parameter layout and its conversion to/from the normative layout,
// device allocations, the documented parameter initialiser, launches of the worker
// kernel in its four modes, the deterministic sync-mode update, the fixed-order
// evaluation reduction, and the device error latch.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "chaos.h"
#include "chaos_kernels.cuh"

using namespace chaos;

// ----------------------------------------------------------------------------------
// Compiled nets (BASELINE.json configs).  Tuning knobs per conv block: MT, TT, GS, NCH.
// ----------------------------------------------------------------------------------
namespace {

// INFLIGHT: the hogwild staleness cap (R14, SURVEY C-23): at most this many images
// are in flight per GPU (#CTAs x G).  Measured on the B200 (scripts/hogwild_sweep.py): the tiny
// net at lr 0.001 blows up in epoch 1 with 592-1184 in flight, the large net trains like
// sequential SGD with 592.  GINIT is the group G a new net starts with.
#ifndef TINY_NT
#define TINY_NT 512
#endif
struct TinyNet {  // configs[0], configs[1]: conv5 4x4 -> tanh -> pool2 -> FC 845->10
    static constexpr int NCONV = 1, NFULL = 1, GDEF = 4, GINIT = 1, INFLIGHT = 148, NT = TINY_NT, SFL = 2 * 8456;
    static constexpr bool TRACE = true;  // kTrace instantiated (hogwild schedule recording)
#ifndef TINY_C1_GS  // tile sweeps: -DTINY_C1_GS=.. -DTINY_C1_TT=..
#define TINY_C1_GS 16
#endif
#ifndef TINY_C1_TT
#define TINY_C1_TT 16
#endif
    // FF = 16: packed FMAs in conv_gw only (24.04 -> 24.13 M samples/s; in the forward too: 23.99 M)
    using C1 = Conv<1, 29, 29, 5, 4, 2, /*MT*/ 5, /*TT*/ TINY_C1_TT, /*GS*/ TINY_C1_GS, /*RB*/ 2, 0, 0, false, false, 0,
                    false, 1, 0, 0, /*FF*/ 16>;
    using C2 = C1;
    using C3 = C1;
    using F1 = Full<845, 10, false>;
    using F2 = F1;
};
#ifndef MEDIUM_NT
#define MEDIUM_NT 512
#endif
struct MediumNet {  // configs[2] = Table I medium
    static constexpr int NCONV = 2, NFULL = 2, GDEF = 4, GINIT = 4, INFLIGHT = 592, NT = MEDIUM_NT, SFL = 6000;
    static constexpr bool TRACE = false;
#ifndef MEDIUM_DINSPLIT
#define MEDIUM_DINSPLIT 4
#endif
    static constexpr int DINSPLIT = MEDIUM_DINSPLIT;  // conv2 delta_in: warps per (image, 32 maps) task
    // conv2 delta_in window row by window row, each (map, window) dispatched once (conv_din_rows):
    // 4.38 M vs 3.84 M samples/s (banded conv_din); the Table I small net (G = 1: one task) keeps conv_din
    static constexpr bool DINROWS = true;
    static constexpr bool TAIL1 = true;  // conv1 forward tail split: 5.06 -> 5.13 M (large net: -0.5%, off)
    using C1 = Conv<1, 29, 29, 20, 4, 2, 10, 16, 16, 2>;
    // conv2 forward: 8 maps per item with the input maps split over two adjacent lanes (session 5, packed
    // FMAs: 5.181 -> 5.204 M samples/s; MT 8 / 10 / 5 unsplit 4.59 / 4.34 / 4.79 M, MT 4 split 4.96 M)
#ifndef MEDIUM_C2_MT
#define MEDIUM_C2_MT 8
#endif
#ifndef MEDIUM_C2_NSPL
#define MEDIUM_C2_NSPL 2
#endif
#ifndef MEDIUM_C2_RB  // conv2 delta_in: input rows per band task
#define MEDIUM_C2_RB 3
#endif
#ifndef MEDIUM_C2_MP  // conv2 W row pitch: 42 (8-B rows, lanes over input maps 2-way; 41: conflict-free but scalar forward loads, -1.6%)
#define MEDIUM_C2_MP 42
#endif
    using C2 = Conv<20, 13, 13, 40, 5, 3, MEDIUM_C2_MT, 25, 1, MEDIUM_C2_RB, 0, 0, false, false, 0, false, MEDIUM_C2_NSPL,
                    MEDIUM_C2_MP>;
    using C3 = C2;
    using F1 = Full<360, 150, true>;
    using F2 = Full<150, 10, false>;
};
#ifndef PSMALL_NT
#define PSMALL_NT 512
#endif
struct PaperSmallNet {  // Table I small: conv5 4x4 -> pool2 -> conv10 5x5 -> pool3
                        // -> FC 90->50 tanh -> FC 50->10; same generic kernels as the medium net
    static constexpr int NCONV = 2, NFULL = 2, GDEF = 4, GINIT = 1, INFLIGHT = 148, NT = PSMALL_NT, SFL = 3364;
    static constexpr bool TRACE = false;
#ifndef PSMALL_DINSPLIT
#define PSMALL_DINSPLIT 2
#endif
    static constexpr int DINSPLIT = PSMALL_DINSPLIT;
    // FF = 17: packed FMAs in the forward convolutions and conv_gw (6.68 -> 6.83 M samples/s)
    using C1 = Conv<1, 29, 29, 5, 4, 2, /*MT*/ 5, /*TT*/ 16, /*GS*/ 32, /*RB*/ 2, 0, 0, false, false, 0, false, 1, 0, 0,
                    /*FF*/ 17>;
    using C2 = Conv<5, 13, 13, 10, 5, 3, /*MT*/ 2, /*TT*/ 25, /*GS*/ 1, /*RB*/ 3, 0, 0, false, false, 0, false, 1, 0, 0,
                    /*FF*/ 17>;
    using C3 = C2;
    using F1 = Full<90, 50, true>;
    using F2 = Full<50, 10, false>;
};
struct LargeNet {  // configs[3], configs[4]
    // 20 warps (<= 96 registers): one warp per (image, window row) in conv2's delta_in and per
    // (3 maps, 32 input maps) in its weight gradient; conv3's backward split over warps 0-7
    // (delta_in) and 8-19 (weight gradient).  Tile sweeps: profiles/r1q.
    static constexpr int NCONV = 3, NFULL = 2, GDEF = 4, GINIT = 4, INFLIGHT = 592, NT = 640, SFL = 6400;
    static constexpr bool TRACE = true;
#ifndef LARGE_MGF2
#define LARGE_MGF2 1
#endif
    static constexpr bool MGF2 = LARGE_MGF2;  // conv2 forward: map groups fastest over the lanes (+0.3%)
    static constexpr bool TC2 = true;   // conv2 forward on the tensor cores when built with CHAOS_C2_TC
    static constexpr bool REPL = true;  // replica-emulation build (fused cross-replica averaging tests)
    //                C   H   W   M   K  KP  MT  TT  GS  RB  PB  MS  (0)  DIN3  GWIN  DWIN  NSPL
#ifndef LARGE_C1_MT  // tile sweeps (scripts): -DLARGE_C1_MT=.. -DLARGE_C1_GS=..
#define LARGE_C1_MT 10
#endif
#ifndef LARGE_C1_GS
#define LARGE_C1_GS 16
#endif
    using C1 = Conv<1, 29, 29, 20, 4, 2, LARGE_C1_MT, 16, LARGE_C1_GS, 2>;
#ifndef LARGE_C2_PB  // conv2 delta_in: window rows per band task
#define LARGE_C2_PB 1
#endif
#ifndef LARGE_C2_MT  // conv2 forward: output maps per thread item
#define LARGE_C2_MT 10
#endif
#ifndef LARGE_C3_MT  // conv3 forward: output maps per thread item (session 5, packed FMAs: 10 maps with the input
#define LARGE_C3_MT 10  // maps split over two adjacent lanes, 320 half-items: 25.6k -> 23.5k cycles, 4.252 -> 4.275 M;
#endif               // MT 4 / 5 split 4.15 / 4.16 M, MT 10 unsplit 4.21 M, MT 10 split + map groups fastest 4.07 M)
    using C2 = Conv<20, 13, 13, 60, 3, 2, LARGE_C2_MT, 9, 1, 4, LARGE_C2_PB, -1, false, true, 0, false, 1>;
#ifndef LARGE_C3_NPAD  // conv3 W: floats of padding per input map (NS = 404: NS / 4 odd)
#define LARGE_C3_NPAD 4
#endif
#ifndef LARGE_C3_NSPL  // conv3 forward: input maps of an item split over this many adjacent lanes
#define LARGE_C3_NSPL 2
#endif
    using C3 = Conv<60, 5, 5, 100, 2, 2, LARGE_C3_MT, 4, 1, 5, 2, 0, false, false, 4, true, LARGE_C3_NSPL, 0, LARGE_C3_NPAD>;
    using F1 = Full<400, 150, true>;
    using F2 = Full<150, 10, false>;
};

struct PaperLargeNet {  // Table I large: conv20 4x4 -> pool 1x1 -> conv60 5x5
                       // -> pool2 -> conv100 6x6 -> pool2 -> FC 900->150 tanh -> FC 150->10.  383,160
                       // weights: W1 + W2 staged and kept, W3 (864 KB) and FC1 (540 KB) read from L2 (BIGW);
                       // one image per worker (224 KB of shared memory)
#ifndef PL_RB3
#define PL_RB3 4
#endif
    static constexpr int NCONV = 3, NFULL = 2, GDEF = 1, GINIT = 1, INFLIGHT = 148, NT = 384, SFL = 1800, RB3 = PL_RB3;
    static constexpr bool TRACE = false;
    static constexpr bool BIGW = true;
    //                C   H   W    M  K  KP  MT  TT  GS  RB  PB  MS  (0)  DIN3  GWIN  DWIN  NSPL
    // FF = 96: packed FMAs in conv_din_gm and conv_gw_wt only (256.4 -> 261.8 k samples/s); with them in the
    // forward convolutions too (12 warps: latency-bound) 239.9 k
#ifndef PL_FF
#define PL_FF 96
#endif
    using C1 = Conv<1, 29, 29, 20, 4, 1, 10, 16, 16, 1, 0, 0, false, false, 0, false, 1, 0, 0, PL_FF>;
    using C2 = Conv<20, 26, 26, 60, 5, 2, 10, 25, 1, 2, 0, 0, false, false, 0, false, 1, 0, 0, PL_FF>;
    using C3 = Conv<60, 11, 11, 100, 6, 2, 4, 12, 1, 2, 0, 0, false, false, 0, false, 1, 0, 0, PL_FF>;
    using F1 = Full<900, 150, true>;
    using F2 = Full<150, 10, false>;
};

using KernelFn = void (*)(KArgs);

// Nets with a one-GPU replica-emulation build of the hogwild worker (REPL = true: the fused
// cross-replica averaging is tested on one GPU with R replicas in one cooperative launch)
template <class N, class = void>
struct Repl {
    static constexpr bool value = false;
};
template <class N>
struct Repl<N, std::void_t<decltype(N::REPL)>> {
    static constexpr bool value = N::REPL;
};

struct Block {  // one weighted layer, host view
    bool conv;
    int C, K, M, MP, NS;  // conv (NS: floats per input map, K*K*MP + padding)
    int IN, OUT;      // full
    long long int_w, int_b;    // internal offsets (floats)
    long long norm_w, norm_b;  // normative offsets
    long long nw, nb, fan_in;
};

struct LayerSig {
    int kind, units, kernel, act;
};

struct NetDesc {
    const char* name;
    std::vector<LayerSig> sig;
    std::vector<Block> blocks;
    long long pint = 0;    // internal floats
    long long nparams = 0; // normative count
    int gdef = 1, ginit = 1, nt = 256;
    int max_inflight = 1 << 30;  // hogwild staleness cap: #CTAs x G
    // [gi][mode]: gi 0 -> G=1, gi 1 -> G=gdef
    KernelFn fn[2][5] = {};  // [gi][mode]; kTrace only for nets with trace points (else nullptr)
    KernelFn fn_gated[2] = {};  // hogwild from host buffers (claims gated by the landed counter)
    KernelFn fn_rep = nullptr;  // hogwild, G = gdef, replica emulation (nets with REPL)
    KernelFn fn_pavg[2] = {};   // hogwild, G = gdef, fused averaging compiled in: [gated] (nets with REPL)
    int smem[2] = {0, 0};
    double flops_per_sample = 0;  // algorithmic
};

template <class L>
void add_conv(NetDesc& d, long long w, long long b, long long& norm) {
    Block k{};
    k.conv = true;
    k.C = L::C;
    k.K = L::K;
    k.M = L::M;
    k.MP = L::MP;
    k.NS = L::NS;
    k.int_w = w;
    k.int_b = b;
    k.nw = (long long)L::M * L::C * L::K * L::K;
    k.nb = L::M;
    k.fan_in = (long long)L::C * L::K * L::K;
    k.norm_w = norm;
    k.norm_b = norm + k.nw;
    norm += k.nw + k.nb;
    d.blocks.push_back(k);
}
template <class F>
void add_full(NetDesc& d, long long w, long long b, long long& norm) {
    Block k{};
    k.conv = false;
    k.IN = F::IN;
    k.OUT = F::OUT;
    k.int_w = w;
    k.int_b = b;
    k.nw = (long long)F::IN * F::OUT;
    k.nb = F::OUT;
    k.fan_in = F::IN;
    k.norm_w = norm;
    k.norm_b = norm + k.nw;
    norm += k.nw + k.nb;
    d.blocks.push_back(k);
}

template <class Net, int G>
void fill_kernels(NetDesc& d, int gi) {
    d.fn[gi][kHogwild] = chaos_worker<Net, G, Net::NT, kHogwild>;
    d.fn[gi][kSync] = chaos_worker<Net, G, Net::NT, kSync>;
    d.fn[gi][kEval] = chaos_worker<Net, G, Net::NT, kEval>;
    d.fn[gi][kForward] = chaos_worker<Net, G, Net::NT, kForward>;
    if constexpr (Net::TRACE) d.fn[gi][kTrace] = chaos_worker<Net, G, Net::NT, kTrace>;
    d.fn_gated[gi] = chaos_worker<Net, G, Net::NT, kHogwild, true>;
    if constexpr (Repl<Net>::value && G == Net::GDEF) {
        d.fn_rep = chaos_worker<Net, G, Net::NT, kHogwild, false, true>;
        d.fn_pavg[0] = chaos_worker<Net, G, Net::NT, kHogwild, false, false, true>;
        d.fn_pavg[1] = chaos_worker<Net, G, Net::NT, kHogwild, true, false, true>;
    }
    d.smem[gi] = SLayout<Net, G>::BYTES;
}


template <class Net>
NetDesc make_desc(const char* name, std::vector<LayerSig> sig) {
    using O = POff<Net>;
    NetDesc d;
    d.name = name;
    d.sig = std::move(sig);
    long long norm = 0;
    add_conv<typename Net::C1>(d, O::c1w, O::c1b, norm);
    if constexpr (Net::NCONV >= 2) add_conv<typename Net::C2>(d, O::c2w, O::c2b, norm);
    if constexpr (Net::NCONV >= 3) add_conv<typename Net::C3>(d, O::c3w, O::c3b, norm);
    add_full<typename Net::F1>(d, O::f1w, O::f1b, norm);
    if constexpr (Net::NFULL >= 2) add_full<typename Net::F2>(d, O::f2w, O::f2b, norm);
    d.pint = O::total;
    d.nparams = norm;
    d.gdef = Net::GDEF;
    d.ginit = Net::GINIT;
    d.max_inflight = Net::INFLIGHT;
    d.nt = Net::NT;
    fill_kernels<Net, 1>(d, 0);
    fill_kernels<Net, Net::GDEF>(d, 1);
    return d;
}

const std::vector<NetDesc>& registry() {
    static const std::vector<NetDesc> r = [] {
        std::vector<NetDesc> v;
#if !defined(CHAOS_ONLY_NET) || CHAOS_ONLY_NET_TinyNet
        v.push_back(make_desc<TinyNet>("tiny", {{CHAOS_CONV, 5, 4, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 2, 0},
                                                {CHAOS_FULL, 10, 0, CHAOS_IDENTITY}}));
#endif
#if !defined(CHAOS_ONLY_NET) || CHAOS_ONLY_NET_MediumNet
        v.push_back(make_desc<MediumNet>(
            "medium", {{CHAOS_CONV, 20, 4, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 2, 0}, {CHAOS_CONV, 40, 5, CHAOS_TANH},
                       {CHAOS_MAXPOOL, 0, 3, 0}, {CHAOS_FULL, 150, 0, CHAOS_TANH}, {CHAOS_FULL, 10, 0, CHAOS_IDENTITY}}));
#endif
#if !defined(CHAOS_ONLY_NET) || CHAOS_ONLY_NET_PaperSmallNet
        v.push_back(make_desc<PaperSmallNet>(
            "paper_small", {{CHAOS_CONV, 5, 4, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 2, 0}, {CHAOS_CONV, 10, 5, CHAOS_TANH},
                            {CHAOS_MAXPOOL, 0, 3, 0}, {CHAOS_FULL, 50, 0, CHAOS_TANH},
                            {CHAOS_FULL, 10, 0, CHAOS_IDENTITY}}));
#endif
#if !defined(CHAOS_ONLY_NET) || CHAOS_ONLY_NET_LargeNet
        v.push_back(make_desc<LargeNet>(
            "large", {{CHAOS_CONV, 20, 4, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 2, 0}, {CHAOS_CONV, 60, 3, CHAOS_TANH},
                      {CHAOS_MAXPOOL, 0, 2, 0}, {CHAOS_CONV, 100, 2, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 2, 0},
                      {CHAOS_FULL, 150, 0, CHAOS_TANH}, {CHAOS_FULL, 10, 0, CHAOS_IDENTITY}}));
#endif
#if !defined(CHAOS_ONLY_NET) || CHAOS_ONLY_NET_PaperLargeNet
        v.push_back(make_desc<PaperLargeNet>(
            "paper_large", {{CHAOS_CONV, 20, 4, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 1, 0}, {CHAOS_CONV, 60, 5, CHAOS_TANH},
                            {CHAOS_MAXPOOL, 0, 2, 0}, {CHAOS_CONV, 100, 6, CHAOS_TANH}, {CHAOS_MAXPOOL, 0, 2, 0},
                            {CHAOS_FULL, 150, 0, CHAOS_TANH}, {CHAOS_FULL, 10, 0, CHAOS_IDENTITY}}));
#endif
        return v;
    }();
    return r;
}

thread_local std::string g_err;
thread_local chaos_status g_status = CHAOS_OK;

chaos_status fail(chaos_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    g_status = s;
    return s;
}

#define CUDA_TRY(expr)                                                                           \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess) return fail(CHAOS_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

}  // namespace

// NCCL, loaded at run time (no link-time dependency): the copy a torch process already holds
// (RTLD_NOLOAD) if any, else the system libnccl.so.2.  Only chaos_dist_* use it.
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*init_rank_config)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;  // optional
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.init_rank_config = reinterpret_cast<decltype(a.init_rank_config)>(dlsym(h, "ncclCommInitRankConfig"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.init_rank && a.all_reduce && a.destroy && a.error_string;
        if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
        return a;
    }();
    return api;
}

struct chaos_net {
    const NetDesc* d = nullptr;
    int dev = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    float* params = nullptr;
    int* latch = nullptr;
    unsigned long long* counter = nullptr;
    double* loss_sum = nullptr;
    long long last_train_n = 0;
    float* partial = nullptr;
    long long partial_slots = 0;
    float* grad_out = nullptr;
    int* claims = nullptr;
    long long claims_cap = 0;
    float* ev_loss = nullptr;
    unsigned char* ev_wrong = nullptr;
    long long ev_cap = 0;
    double* ev_sum = nullptr;
    long long* ev_err = nullptr;
    float* st_x = nullptr;
    int* st_y = nullptr;
    long long st_cap = 0;
    int sync_batch = 64;
    int group = 1;
    bool group_set = false;              // CHAOS_OPT_GROUP given explicitly (else sync batches may use G = 1)
    int max_ctas = 0;
    int debug_claims = 0;
    int reserve_sms = 0;                   // hogwild: SMs left free of training CTAs
    unsigned long long* progress = nullptr;  // device: images published by hogwild launches (monotonic)
    unsigned long long progress_enqueued = 0; // host: images enqueued to hogwild launches
    int occ[2][5] = {};
    int debug_trace = 0;                   // CHAOS_OPT_DEBUG_TRACE: hogwild epochs record their schedule
    long long debug_stagger = 0;           // CHAOS_OPT_DEBUG_STAGGER: cycles per CTA index
    unsigned long long* tctr = nullptr;    // kTrace event counters (2)
    long long* trec = nullptr;             // kTrace records [groups][kTraceRec]
    float* tw = nullptr;                   // kTrace: weights each group read [groups][2][pint]
    long long tw_cap = 0;
    long long trec_cap = 0;
    long long trace_groups = 0;            // groups of the last traced epoch
    int trace_g = 1;                       // ... and their size G
    unsigned long long* ptime = nullptr;  // CHAOS_TIMING builds only
    int ptime_grid = 0;
    ncclComm_t comm = nullptr;             // chaos_dist_init (library-owned communicator)
    int comm_max_ctas = 0;                 // its CTA cap (the reserved SMs at init; 0 = uncapped)
    int comm_world = 0;
    cudaStream_t copy_stream = nullptr;    // chaos_train_epoch_host: H2D chunks overlap training
    unsigned long long* ready = nullptr;       // device: images landed (hogwild host entry)
    unsigned long long* ready_host = nullptr;  // pinned: the per-chunk values the copy stream writes
    long long ready_cap = 0;
    const unsigned long long* launch_ready = nullptr;  // set around the host entry's single launch
    std::vector<cudaEvent_t> chunk_ev;
    cudaEvent_t staging_free = nullptr;
    cudaEvent_t ready_copied = nullptr;  // recorded after a hogwild host epoch's last ready_host copy
    bool ready_pending = false;          // ... whose copies may still be reading ready_host
    // fused in-kernel cross-replica averaging (chaos_pavg_*)
    void* px = nullptr;                  // own exchange buffer: snapshot ring, flags, done, checksums
    size_t px_bytes = 0;
    size_t px_off_flag = 0, px_off_done = 0, px_off_cks = 0;
    PavgArgs px_host{};                  // peer table (host copy)
    PavgArgs* px_dev = nullptr;          // ... device copy
    bool px_dirty = true;
    void* px_mapped[kPavgMaxR] = {};     // IPC mappings to close
    int px_peers_set = 0;                // bitmask of peers with a table entry
    long long px_k = 0, px_round0 = 0, px_arm = 0;
    int px_comm = 0;                     // CHAOS_OPT_PAVG_COMM_CTAS
    KArgs* rep_dev = nullptr;            // replica emulation: per-replica arguments (device)
};

namespace {

int gidx(const chaos_net* net) { return net->group == 1 ? 0 : 1; }

chaos_status ensure_kernel_attrs(chaos_net* net) {
    for (KernelFn f : {net->d->fn_rep, net->d->fn_pavg[0], net->d->fn_pavg[1]})
        if (f) CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, net->d->smem[1]));
    for (int gi = 0; gi < 2; ++gi) {
        CUDA_TRY(cudaFuncSetAttribute(net->d->fn_gated[gi], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      net->d->smem[gi]));
        for (int m = 0; m < 5; ++m) {
            KernelFn f = net->d->fn[gi][m];
            if (!f) continue;
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, net->d->smem[gi]));
            int occ = 0;
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, net->d->nt, net->d->smem[gi]));
            if (occ < 1) return fail(CHAOS_E_CUDA, "kernel %s G=%d mode %d does not fit on an SM (%d B smem)",
                                     net->d->name, gi ? net->d->gdef : 1, m, net->d->smem[gi]);
            net->occ[gi][m] = occ;
        }
    }
    return CHAOS_OK;
}

int grid_for(const chaos_net* net, int mode, long long work_groups) {
    long long g = (long long)(mode == kHogwild ? net->sms - net->reserve_sms : net->sms) * net->occ[gidx(net)][mode];
    if (mode == kHogwild && g * net->group > net->d->max_inflight) g = net->d->max_inflight / net->group;
    if (net->max_ctas > 0 && g > net->max_ctas) g = net->max_ctas;
    if (g > work_groups) g = work_groups;
    return (int)(g < 1 ? 1 : g);
}

chaos_status check_latch(chaos_net* net) {
    int h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, net->latch, sizeof(int), cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    if (h) {
        CUDA_TRY(cudaMemsetAsync(net->latch, 0, sizeof(int), net->stream));
        CUDA_TRY(cudaStreamSynchronize(net->stream));
        if (h & kLatchLabel) return fail(CHAOS_E_LABEL, "device: a label outside [0, %d)", kClasses);
        if (h & kLatchPavgTimeout)
            return fail(CHAOS_E_CUDA, "device: fused averaging waited > 10 s for a peer replica (rounds abandoned)");
        if (h & kLatchPavg)
            return fail(CHAOS_E_CUDA, "device: fused averaging read a peer snapshot whose checksum does not match");
        return fail(CHAOS_E_NONFINITE, "device: non-finite loss");
    }
    return CHAOS_OK;
}

void to_internal(const NetDesc& d, const float* norm, std::vector<float>& out) {
    out.assign((size_t)d.pint, 0.f);
    for (const Block& b : d.blocks) {
        if (b.conv) {
            for (int m = 0; m < b.M; ++m)
                for (int n = 0; n < b.C; ++n)
                    for (int t = 0; t < b.K * b.K; ++t)
                        out[b.int_w + (long long)n * b.NS + (long long)t * b.MP + m] =
                            norm[b.norm_w + ((long long)m * b.C + n) * b.K * b.K + t];
        } else {
            std::memcpy(&out[b.int_w], norm + b.norm_w, sizeof(float) * b.nw);
        }
        std::memcpy(&out[b.int_b], norm + b.norm_b, sizeof(float) * b.nb);
    }
}

void to_normative(const NetDesc& d, const float* in, float* norm) {
    for (const Block& b : d.blocks) {
        if (b.conv) {
            for (int m = 0; m < b.M; ++m)
                for (int n = 0; n < b.C; ++n)
                    for (int t = 0; t < b.K * b.K; ++t)
                        norm[b.norm_w + ((long long)m * b.C + n) * b.K * b.K + t] =
                            in[b.int_w + (long long)n * b.NS + (long long)t * b.MP + m];
        } else {
            std::memcpy(norm + b.norm_w, &in[b.int_w], sizeof(float) * b.nw);
        }
        std::memcpy(norm + b.norm_b, &in[b.int_b], sizeof(float) * b.nb);
    }
}

// splitmix64 draw i of stream `seed` (R7): mix(seed + (i+1)*gamma)
uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Shape chain check (conv o = h-k+1, pool o = floor(h/kp)); message names the layer.
chaos_status validate(const chaos_arch* a) {
    if (!a) return fail(CHAOS_E_INVALID, "arch is NULL");
    if (a->n_layers < 1 || a->n_layers > 16 || a->in_c < 1 || a->in_h < 1 || a->in_w < 1 || a->n_classes < 1)
        return fail(CHAOS_E_INVALID, "invalid arch header");
    int c = a->in_c, h = a->in_h, w = a->in_w;
    for (int l = 0; l < a->n_layers; ++l) {
        const chaos_layer& s = a->layers[l];
        if (s.kind == CHAOS_CONV) {
            if (s.units < 1 || s.kernel < 1 || s.kernel > h || s.kernel > w)
                return fail(CHAOS_E_ARCH, "layer %d (conv k=%d): input %dx%d < kernel or units < 1", l, s.kernel, h,
                            w);
            c = s.units;
            h = h - s.kernel + 1;
            w = w - s.kernel + 1;
        } else if (s.kind == CHAOS_MAXPOOL) {
            if (s.kernel < 1 || s.kernel > h || s.kernel > w)
                return fail(CHAOS_E_ARCH, "layer %d (pool k=%d): input %dx%d < window", l, s.kernel, h, w);
            h /= s.kernel;
            w /= s.kernel;
        } else if (s.kind == CHAOS_FULL) {
            if (s.units < 1) return fail(CHAOS_E_ARCH, "layer %d (full): units < 1", l);
            c = s.units;
            h = w = 1;
        } else {
            return fail(CHAOS_E_ARCH, "layer %d: unknown kind %d", l, s.kind);
        }
    }
    const chaos_layer& last = a->layers[a->n_layers - 1];
    if (last.kind != CHAOS_FULL || last.units != a->n_classes || last.act != CHAOS_IDENTITY)
        return fail(CHAOS_E_ARCH, "layer %d: last layer must be FULL with n_classes units and identity activation",
                    a->n_layers - 1);
    return CHAOS_OK;
}

const NetDesc* match(const chaos_arch* a) {
    if (a->in_c != 1 || a->in_h != 29 || a->in_w != 29 || a->n_classes != kClasses) return nullptr;
    for (const NetDesc& d : registry()) {
        if ((int)d.sig.size() != a->n_layers) continue;
        bool ok = true;
        for (int l = 0; l < a->n_layers && ok; ++l) {
            const chaos_layer& s = a->layers[l];
            const LayerSig& q = d.sig[l];
            ok = s.kind == q.kind && s.kernel == q.kernel &&
                 (s.kind == CHAOS_MAXPOOL || (s.units == q.units && s.act == q.act));
        }
        if (ok) return &d;
    }
    return nullptr;
}

chaos_status ensure_partial(chaos_net* net, long long slots) {
    if (slots <= net->partial_slots) return CHAOS_OK;
    if (net->partial) cudaFree(net->partial);
    net->partial = nullptr;
    const size_t bytes = sizeof(float) * (size_t)slots * (size_t)net->d->pint;
    CUDA_TRY(cudaMalloc(&net->partial, bytes));
    CUDA_TRY(cudaMemsetAsync(net->partial, 0, bytes, net->stream));  // padding entries stay 0 forever
    net->partial_slots = slots;
    return CHAOS_OK;
}

chaos_status ensure_eval(chaos_net* net, long long n) {
    if (n <= net->ev_cap) return CHAOS_OK;
    if (net->ev_loss) cudaFree(net->ev_loss);
    if (net->ev_wrong) cudaFree(net->ev_wrong);
    net->ev_loss = nullptr;
    net->ev_wrong = nullptr;
    CUDA_TRY(cudaMalloc(&net->ev_loss, sizeof(float) * n));
    CUDA_TRY(cudaMalloc(&net->ev_wrong, n));
    net->ev_cap = n;
    return CHAOS_OK;
}

KArgs base_args(chaos_net* net) {
    KArgs k{};
    k.params = net->params;
    k.partial = net->partial;
    k.pstride = net->d->pint;
    k.counter = net->counter;
    k.latch = net->latch;
    return k;
}

// One sync-mode batch: gradients of [0, nb) at the current weights into slots, then
// (out == nullptr) params -= lr * fixed-order sum, or out = sum.
chaos_status sync_batch(chaos_net* net, const float* X, const int32_t* Y, long long nb, float lr, float* out,
                        double* loss_sum) {
    // G never set: a batch with fewer than G * SMs images runs one image per CTA (G = 1) so it
    // spreads over G times more SMs (B = 64: 1.7x on the large and medium nets, scripts/sync_group_sweep.py)
    const int G = (!net->group_set && nb < (long long)net->d->gdef * net->sms) ? 1 : net->group;
    const int gi = G == 1 ? 0 : 1;
    const long long slots = (nb + G - 1) / G;
    chaos_status s = ensure_partial(net, slots);
    if (s) return s;
    KArgs k = base_args(net);
    k.partial = net->partial;
    k.images = X;
    k.labels = Y;
    k.n = nb;
    k.loss_sum = loss_sum;
    long long gsz = (long long)net->sms * net->occ[gi][kSync];
    if (net->max_ctas > 0 && gsz > net->max_ctas) gsz = net->max_ctas;
    const int grid = (int)std::max<long long>(1, std::min<long long>(gsz, slots));
#ifdef CHAOS_TIMING
    if (net->ptime_grid < grid) {
        if (net->ptime) cudaFree(net->ptime);
        net->ptime = nullptr;
        CUDA_TRY(cudaMalloc(&net->ptime, sizeof(unsigned long long) * kPhases * grid));
        CUDA_TRY(cudaMemsetAsync(net->ptime, 0, sizeof(unsigned long long) * kPhases * grid, net->stream));
        net->ptime_grid = grid;
    }
    k.ptime = net->ptime;  // accumulates over the epoch's batches (reset by a hogwild epoch)
#endif
    net->d->fn[gi][kSync]<<<grid, net->d->nt, net->d->smem[gi], net->stream>>>(k);
    CUDA_TRY(cudaGetLastError());
    const long long np = net->d->pint;
    chaos_reduce_update<<<(unsigned)((np + 255) / 256), 256, 0, net->stream>>>(net->params, net->partial, np,
                                                                              (int)slots, lr, np, out);
    CUDA_TRY(cudaGetLastError());
    return CHAOS_OK;
}

}  // namespace

extern "C" {

const char* chaos_last_error(void) { return g_err.c_str(); }
chaos_status chaos_last_status(void) { return g_status; }

chaos_net* chaos_net_create(const chaos_arch* arch) {
    g_err.clear();
    g_status = CHAOS_OK;
    if (validate(arch) != CHAOS_OK) return nullptr;
    const NetDesc* d = match(arch);
    if (!d) {
        fail(CHAOS_E_UNSUPPORTED, "valid arch without a compiled sm_100a instantiation (compiled: tiny, medium, large, paper_small, paper_large)");
        return nullptr;
    }
    chaos_net* net = new chaos_net();
    net->d = d;
    net->group = d->ginit;
    auto bail = [&](chaos_status) -> chaos_net* {
        chaos_net_destroy(net);
        return nullptr;
    };
    if (cudaGetDevice(&net->dev) != cudaSuccess) {
        fail(CHAOS_E_CUDA, "no CUDA device");
        return bail(CHAOS_E_CUDA);
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, net->dev) != cudaSuccess) {
        fail(CHAOS_E_CUDA, "cudaGetDeviceProperties failed");
        return bail(CHAOS_E_CUDA);
    }
    if (prop.major != 10) {
        fail(CHAOS_E_UNSUPPORTED, "libchaos.so is built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
        return bail(CHAOS_E_UNSUPPORTED);
    }
    net->sms = prop.multiProcessorCount;
    if (ensure_kernel_attrs(net) != CHAOS_OK) return bail(g_status);
    if (cudaMalloc(&net->params, sizeof(float) * d->pint) != cudaSuccess ||
        cudaMalloc(&net->latch, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&net->counter, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&net->progress, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&net->loss_sum, sizeof(double)) != cudaSuccess ||
        cudaMalloc(&net->ev_sum, sizeof(double)) != cudaSuccess ||
        cudaMalloc(&net->ev_err, sizeof(long long)) != cudaSuccess) {
        fail(CHAOS_E_CUDA, "cudaMalloc failed");
        return bail(CHAOS_E_CUDA);
    }
    cudaMemset(net->latch, 0, sizeof(int));
    cudaMemset(net->progress, 0, sizeof(unsigned long long));
    cudaMemset(net->loss_sum, 0, sizeof(double));
    // parameters: U(-1/sqrt(fan_in), +1/sqrt(fan_in)), W then b per layer, splitmix64(seed ^ 0x5EED)
    std::vector<float> norm((size_t)d->nparams);
    const uint64_t seed = arch->init_seed ^ 0x5EEDull;
    uint64_t pos = 0;
    for (const Block& b : d->blocks) {
        const double lim = 1.0 / std::sqrt((double)b.fan_in);
        for (long long j = 0; j < b.nw + b.nb; ++j, ++pos) {
            const double u = (double)(splitmix_at(seed, pos) >> 40) * (1.0 / 16777216.0);
            norm[(size_t)(b.norm_w + j)] = (float)((2.0 * u - 1.0) * lim);
        }
    }
    if (chaos_net_set_params(net, norm.data(), d->nparams) != CHAOS_OK) return bail(g_status);
    return net;
}

void chaos_net_destroy(chaos_net* net) {
    if (!net) return;
    if (net->stream) cudaStreamSynchronize(net->stream);
    cudaDeviceSynchronize();
    if (net->comm) nccl_api().destroy(net->comm);
    if (net->copy_stream) cudaStreamDestroy(net->copy_stream);
    if (net->ready_host) cudaFreeHost(net->ready_host);
    if (net->ready) cudaFree(net->ready);
    if (net->staging_free) cudaEventDestroy(net->staging_free);
    if (net->tctr) cudaFree(net->tctr);
    if (net->trec) cudaFree(net->trec);
    if (net->tw) cudaFree(net->tw);
    if (net->ready_copied) cudaEventDestroy(net->ready_copied);
    for (cudaEvent_t e : net->chunk_ev) cudaEventDestroy(e);
    for (void* m : net->px_mapped)
        if (m) cudaIpcCloseMemHandle(m);
    if (net->px) cudaFree(net->px);
    if (net->px_dev) cudaFree(net->px_dev);
    if (net->px_host.dsum) cudaFree(net->px_host.dsum);
    if (net->px_host.dabs) cudaFree(net->px_host.dabs);
    if (net->rep_dev) cudaFree(net->rep_dev);
    void* ptrs[] = {net->params, net->latch,  net->counter, net->loss_sum, net->partial, net->grad_out, net->claims,
                    net->ev_loss, net->ev_wrong, net->ev_sum, net->ev_err, net->st_x, net->st_y, net->ptime,
                    net->progress};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    delete net;
}

chaos_status chaos_net_set_option(chaos_net* net, chaos_option opt, int64_t value) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    switch (opt) {
        case CHAOS_OPT_STREAM:
            net->stream = reinterpret_cast<cudaStream_t>(value);
            return CHAOS_OK;
        case CHAOS_OPT_SYNC_BATCH:
            if (value < 1 || value > (1 << 20)) return fail(CHAOS_E_INVALID, "sync batch must be in [1, 2^20]");
            net->sync_batch = (int)value;
            return CHAOS_OK;
        case CHAOS_OPT_GROUP:
            if (value != 1 && value != net->d->gdef)
                return fail(CHAOS_E_INVALID, "group G must be 1 or %d for net %s", net->d->gdef, net->d->name);
            net->group = (int)value;
            net->group_set = true;
            return CHAOS_OK;
        case CHAOS_OPT_MAX_CTAS:
            if (value < 0) return fail(CHAOS_E_INVALID, "max_ctas must be >= 0 (0 = all SMs)");
            net->max_ctas = (int)value;
            return CHAOS_OK;
        case CHAOS_OPT_DEBUG_CLAIMS:
            net->debug_claims = value ? 1 : 0;
            return CHAOS_OK;
        case CHAOS_OPT_DEBUG_TRACE:
            if (value && !net->d->fn[0][kTrace])
                return fail(CHAOS_E_UNSUPPORTED, "net %s has no schedule-recording (trace) build", net->d->name);
            net->debug_trace = value ? 1 : 0;
            return CHAOS_OK;
        case CHAOS_OPT_DEBUG_STAGGER:
            if (value < 0) return fail(CHAOS_E_INVALID, "stagger must be >= 0");
            net->debug_stagger = value;
            return CHAOS_OK;
        case CHAOS_OPT_PAVG_COMM_CTAS:
            if (value < 0 || value > 16) return fail(CHAOS_E_INVALID, "pavg comm CTAs must be in [0, 16]");
            net->px_comm = (int)value;
            return CHAOS_OK;
        case CHAOS_OPT_RESERVE_SMS:
            if (value < 0 || value >= net->sms) return fail(CHAOS_E_INVALID, "reserve_sms must be in [0, %d)", net->sms);
            if (net->comm && value > 0 && (net->comm_max_ctas == 0 || net->comm_max_ctas > value))
                return fail(CHAOS_E_INVALID,
                            "the communicator was created with %d CTAs (0 = uncapped): set reserve_sms before "
                            "chaos_dist_init so collectives fit beside the persistent kernel",
                            net->comm_max_ctas);
            net->reserve_sms = (int)value;
            return CHAOS_OK;
    }
    return fail(CHAOS_E_INVALID, "unknown option %d", (int)opt);
}

int64_t chaos_net_get_option(const chaos_net* net, chaos_option opt) {
    if (!net) return -1;
    switch (opt) {
        case CHAOS_OPT_STREAM: return (int64_t)net->stream;
        case CHAOS_OPT_SYNC_BATCH: return net->sync_batch;
        case CHAOS_OPT_GROUP: return net->group;
        case CHAOS_OPT_MAX_CTAS: return net->max_ctas;
        case CHAOS_OPT_DEBUG_CLAIMS: return net->debug_claims;
        case CHAOS_OPT_DEBUG_TRACE: return net->debug_trace;
        case CHAOS_OPT_DEBUG_STAGGER: return net->debug_stagger;
        case CHAOS_OPT_RESERVE_SMS: return net->reserve_sms;
        case CHAOS_OPT_PAVG_COMM_CTAS: return net->px_comm;
    }
    return -1;
}

int64_t chaos_net_num_params(const chaos_net* net) { return net ? net->d->nparams : -1; }
float* chaos_net_device_params(chaos_net* net) { return net ? net->params : nullptr; }
int64_t chaos_net_device_params_len(const chaos_net* net) { return net ? net->d->pint : -1; }

chaos_status chaos_net_get_params(chaos_net* net, float* host_dst, int64_t n) {
    if (!net || !host_dst) return fail(CHAOS_E_INVALID, "NULL argument");
    if (n != net->d->nparams) return fail(CHAOS_E_INVALID, "n=%lld != num_params=%lld", (long long)n, net->d->nparams);
    std::vector<float> in((size_t)net->d->pint);
    CUDA_TRY(cudaMemcpyAsync(in.data(), net->params, sizeof(float) * in.size(), cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    to_normative(*net->d, in.data(), host_dst);
    return check_latch(net);
}

chaos_status chaos_net_set_params(chaos_net* net, const float* host_src, int64_t n) {
    if (!net || !host_src) return fail(CHAOS_E_INVALID, "NULL argument");
    if (n != net->d->nparams) return fail(CHAOS_E_INVALID, "n=%lld != num_params=%lld", (long long)n, net->d->nparams);
    std::vector<float> in;
    to_internal(*net->d, host_src, in);
    CUDA_TRY(cudaMemcpyAsync(net->params, in.data(), sizeof(float) * in.size(), cudaMemcpyHostToDevice, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    return CHAOS_OK;
}

}  // extern "C"

namespace {
// Fused averaging arguments of the next hogwild launch (the armed rounds are consumed).
chaos_status pavg_args(chaos_net* net, KArgs& k) {
    const PavgArgs& h = net->px_host;
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_arm without chaos_pavg_setup");
    if (net->px_peers_set != (1 << h.R) - 1)
        return fail(CHAOS_E_INVALID, "fused averaging: exchange buffers of %d replicas expected, peer mask 0x%x",
                    h.R, net->px_peers_set);
    if (net->px_dirty) {
        CUDA_TRY(cudaMemcpyAsync(net->px_dev, &net->px_host, sizeof(PavgArgs), cudaMemcpyHostToDevice, net->stream));
        net->px_dirty = false;
    }
    k.pavg = net->px_dev;
    k.pavg_round0 = net->px_round0;
    k.pavg_rounds = net->px_arm;
    k.pavg_k = net->px_k;
    k.pavg_comm = net->px_comm;
    net->px_round0 += net->px_arm;
    net->px_arm = 0;
    return CHAOS_OK;
}

// One Training phase launch over images [0, n) (n > 0, arguments validated), accumulating into
// the net's training-loss sum; asynchronous on the net's stream.
chaos_status train_range(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n, float lr,
                         chaos_mode mode) {
    const int G = net->group;
    if (mode == CHAOS_HOGWILD) {
        KArgs k = base_args(net);
        k.images = d_images;
        k.labels = d_labels;
        k.n = n;
        k.neg_lr = -lr;
        k.loss_sum = net->loss_sum;
        if (net->debug_claims) {
            if (net->claims_cap < n) {
                if (net->claims) cudaFree(net->claims);
                net->claims = nullptr;
                CUDA_TRY(cudaMalloc(&net->claims, sizeof(int) * n));
                net->claims_cap = n;
            }
            CUDA_TRY(cudaMemsetAsync(net->claims, 0, sizeof(int) * n, net->stream));
            k.claims = net->claims;
        }
        CUDA_TRY(cudaMemsetAsync(net->counter, 0, sizeof(unsigned long long), net->stream));
        int grid = grid_for(net, kHogwild, (n + G - 1) / G);
#ifdef CHAOS_TIMING
        if (net->ptime_grid < grid + net->px_comm) {
            if (net->ptime) cudaFree(net->ptime);
            net->ptime = nullptr;
            CUDA_TRY(cudaMalloc(&net->ptime, sizeof(unsigned long long) * kPhases * (grid + net->px_comm)));
            net->ptime_grid = grid + net->px_comm;
        }
        CUDA_TRY(cudaMemsetAsync(net->ptime, 0, sizeof(unsigned long long) * kPhases * net->ptime_grid, net->stream));
        k.ptime = net->ptime;
#endif
        k.progress = net->progress;
        k.ready = net->launch_ready;
        if (net->px_arm > 0) {
            if (net->debug_trace) return fail(CHAOS_E_UNSUPPORTED, "fused averaging is not traced");
            if (!net->d->fn_pavg[0] || net->group != net->d->gdef)
                return fail(CHAOS_E_UNSUPPORTED, "fused averaging is compiled for the large net at its default G");
            chaos_status st = pavg_args(net, k);
            if (st) return st;
            if (net->px_comm > 0) {  // comm CTAs on SMs of their own, after the training CTAs
                const int train = std::min(grid, net->sms - net->reserve_sms - net->px_comm);
                if (train < 1) return fail(CHAOS_E_INVALID, "no SM left for training beside %d comm CTAs", net->px_comm);
                grid = train + net->px_comm;
            }
        }
        net->progress_enqueued += (unsigned long long)n;
        KernelFn fn = k.ready ? net->d->fn_gated[gidx(net)] : net->d->fn[gidx(net)][kHogwild];
        if (k.pavg) fn = net->d->fn_pavg[k.ready ? 1 : 0];
        if (net->debug_trace) {  // the schedule-recording instantiation (debug): records + per-group publishes
            if (k.ready) return fail(CHAOS_E_UNSUPPORTED, "trace recording is for device-buffer epochs");
            const long long groups = (n + G - 1) / G;
            chaos_status st = ensure_partial(net, groups);
            if (st) return st;
            CUDA_TRY(cudaMemsetAsync(net->partial, 0, sizeof(float) * (size_t)groups * (size_t)net->d->pint, net->stream));
            if (!net->tctr) CUDA_TRY(cudaMalloc(&net->tctr, 2 * sizeof(unsigned long long)));
            if (net->trec_cap < groups) {
                if (net->trec) cudaFree(net->trec);
                net->trec = nullptr;
                CUDA_TRY(cudaMalloc(&net->trec, sizeof(long long) * kTraceRec * (size_t)groups));
                net->trec_cap = groups;
            }
            if (net->tw_cap < groups) {
                if (net->tw) cudaFree(net->tw);
                net->tw = nullptr;
                CUDA_TRY(cudaMalloc(&net->tw, sizeof(float) * 2 * (size_t)net->d->pint * (size_t)groups));
                net->tw_cap = groups;
            }
            // NaN: a value no read recorded (the delta_in read of a layer that reuses its forward copy)
            CUDA_TRY(cudaMemsetAsync(net->tw, 0xff, sizeof(float) * 2 * (size_t)net->d->pint * (size_t)groups,
                                     net->stream));
            CUDA_TRY(cudaMemsetAsync(net->tctr, 0, 2 * sizeof(unsigned long long), net->stream));
            CUDA_TRY(cudaMemsetAsync(net->trec, 0xff, sizeof(long long) * kTraceRec * (size_t)groups, net->stream));
            k.partial = net->partial;
            k.tctr = net->tctr;
            k.trec = net->trec;
            k.stagger = net->debug_stagger;
            k.tw = net->tw;
            net->trace_groups = groups;
            net->trace_g = G;
            fn = net->d->fn[gidx(net)][kTrace];
        }
        fn<<<grid, net->d->nt, net->d->smem[gidx(net)], net->stream>>>(k);
        CUDA_TRY(cudaGetLastError());
        return CHAOS_OK;
    }
#ifdef CHAOS_TIMING
    if (net->ptime) CUDA_TRY(cudaMemsetAsync(net->ptime, 0, sizeof(unsigned long long) * kPhases * net->ptime_grid, net->stream));
#endif
    for (long long b0 = 0; b0 < n; b0 += net->sync_batch) {
        const long long nb = (n - b0) < net->sync_batch ? (n - b0) : net->sync_batch;
        chaos_status s = sync_batch(net, d_images + b0 * 841, d_labels + b0, nb, lr, nullptr, net->loss_sum);
        if (s) return s;
    }
    return CHAOS_OK;
}
}  // namespace

extern "C" {

chaos_status chaos_train_epoch(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n, float lr,
                               chaos_mode mode) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (n < 0) return fail(CHAOS_E_INVALID, "n < 0");
    if (!std::isfinite(lr)) return fail(CHAOS_E_INVALID, "lr is not finite");
    if (mode != CHAOS_HOGWILD && mode != CHAOS_SYNC) return fail(CHAOS_E_INVALID, "unknown mode %d", (int)mode);
    CUDA_TRY(cudaMemsetAsync(net->loss_sum, 0, sizeof(double), net->stream));
    net->last_train_n = n;
    if (n == 0) return CHAOS_OK;
    if (!d_images || !d_labels) return fail(CHAOS_E_INVALID, "NULL images/labels");
    return train_range(net, d_images, d_labels, n, lr, mode);
}

namespace {
chaos_status host_epoch(chaos_net* net, const float* h_images, const int32_t* h_labels, int64_t n, float lr,
                        chaos_mode mode, bool synchronize);
}  // namespace

chaos_status chaos_train_epoch_host(chaos_net* net, const float* h_images, const int32_t* h_labels, int64_t n,
                                    float lr, chaos_mode mode) {
    return host_epoch(net, h_images, h_labels, n, lr, mode, true);
}

chaos_status chaos_train_epoch_host_async(chaos_net* net, const float* h_images, const int32_t* h_labels,
                                          int64_t n, float lr, chaos_mode mode) {
    return host_epoch(net, h_images, h_labels, n, lr, mode, false);
}

}  // extern "C"

namespace {
chaos_status host_epoch(chaos_net* net, const float* h_images, const int32_t* h_labels, int64_t n, float lr,
                        chaos_mode mode, bool synchronize) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (n < 0) return fail(CHAOS_E_INVALID, "n < 0");
    if (n == 0) return chaos_train_epoch(net, nullptr, nullptr, 0, lr, mode);
    if (!h_images || !h_labels) return fail(CHAOS_E_INVALID, "NULL images/labels");
    if (!std::isfinite(lr)) return fail(CHAOS_E_INVALID, "lr is not finite");
    if (mode != CHAOS_HOGWILD && mode != CHAOS_SYNC) return fail(CHAOS_E_INVALID, "unknown mode %d", (int)mode);
    if (net->st_cap < n) {
        CUDA_TRY(cudaStreamSynchronize(net->stream));
        if (net->st_x) cudaFree(net->st_x);
        if (net->st_y) cudaFree(net->st_y);
        net->st_x = nullptr;
        net->st_y = nullptr;
        CUDA_TRY(cudaMalloc(&net->st_x, sizeof(float) * 841 * n));
        CUDA_TRY(cudaMalloc(&net->st_y, sizeof(int) * n));
        net->st_cap = n;
    }
    if (!net->copy_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&net->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&net->staging_free, cudaEventDisableTiming));
    }
    if (mode == CHAOS_HOGWILD) {
        // one launch over all n images; chunks of ~n/16 land on the copy stream, each followed by
        // an 8-byte copy that advances the device counter `ready`; a worker that claims a group
        // waits (spinning in its claim) until the group has landed -- no launch boundaries, only
        // the first chunk's copy is exposed
        long long chunk = (n + 15) / 16;
        chunk = (chunk + 15) / 16 * 16;  // 16-image multiples keep the 16-B image alignment
        if (chunk < 2048) chunk = 2048;
        // chunk edges: a doubling ramp 512, 1024, 2048, ... so the copy exposed before the first claims
        // is ~0.03 ms of PCIe time, and the copies (~50 GB/s) stay ahead of the training (~14 GB/s of
        // images at 4 M samples/s) with few host calls (7 chunks for 60,000 images)
        (void)chunk;
        std::vector<long long> edge{0};
        for (long long sz = 512; edge.back() < (long long)n; sz *= 2)
            edge.push_back(std::min<long long>(n, edge.back() + sz));
        const long long nch = (long long)edge.size() - 1;
        if (!net->ready) CUDA_TRY(cudaMalloc(&net->ready, sizeof(unsigned long long)));
        if (!net->ready_copied) CUDA_TRY(cudaEventCreateWithFlags(&net->ready_copied, cudaEventDisableTiming));
        // the previous host epoch's copies (async entry) may still be queued to read ready_host:
        // wait for them before the host rewrites (or frees) it
        if (net->ready_pending) {
            CUDA_TRY(cudaEventSynchronize(net->ready_copied));
            net->ready_pending = false;
        }
        if (net->ready_cap < nch) {
            if (net->ready_host) cudaFreeHost(net->ready_host);
            net->ready_host = nullptr;
            CUDA_TRY(cudaMallocHost(&net->ready_host, sizeof(unsigned long long) * nch));
            net->ready_cap = nch;
        }
        // zero the counter, then let the copy stream start (previous kernels are done with the
        // staging buffers and with `ready` by then)
        CUDA_TRY(cudaMemsetAsync(net->ready, 0, sizeof(unsigned long long), net->stream));
        CUDA_TRY(cudaEventRecord(net->staging_free, net->stream));
        CUDA_TRY(cudaStreamWaitEvent(net->copy_stream, net->staging_free, 0));
        CUDA_TRY(cudaMemsetAsync(net->loss_sum, 0, sizeof(double), net->stream));
        net->last_train_n = n;
        for (long long c = 0; c < nch; ++c) {
            const long long off = edge[(size_t)c];
            const long long len = edge[(size_t)c + 1] - off;
            CUDA_TRY(cudaMemcpyAsync(net->st_x + off * 841, h_images + off * 841, sizeof(float) * 841 * len,
                                     cudaMemcpyHostToDevice, net->copy_stream));
            CUDA_TRY(cudaMemcpyAsync(net->st_y + off, h_labels + off, sizeof(int) * len, cudaMemcpyHostToDevice,
                                     net->copy_stream));
            net->ready_host[c] = static_cast<unsigned long long>(off + len);
            CUDA_TRY(cudaMemcpyAsync(net->ready, net->ready_host + c, sizeof(unsigned long long),
                                     cudaMemcpyHostToDevice, net->copy_stream));
        }
        CUDA_TRY(cudaEventRecord(net->ready_copied, net->copy_stream));
        net->ready_pending = true;
        net->launch_ready = net->ready;
        chaos_status st = train_range(net, net->st_x, net->st_y, n, lr, mode);
        net->launch_ready = nullptr;
        if (st) return st;
        return synchronize ? chaos_net_sync(net) : CHAOS_OK;
    }
    // sync mode: chunks of ~n/8 images in whole sync batches: chunk c+1 is copied on the copy
    // stream while chunk c trains on the net's stream
    const long long unit = (mode == CHAOS_SYNC) ? net->sync_batch : 16;
    long long chunk = (n + 7) / 8;
    chunk = (chunk + unit - 1) / unit * unit;
    if (chunk < 8192 && mode == CHAOS_HOGWILD) chunk = 8192;  // keep launches long enough to fill the GPU
    const long long nch = (n + chunk - 1) / chunk;
    while ((long long)net->chunk_ev.size() < nch) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        net->chunk_ev.push_back(e);
    }
    // the staging buffers may still be read by the previous call's kernels
    CUDA_TRY(cudaEventRecord(net->staging_free, net->stream));
    CUDA_TRY(cudaStreamWaitEvent(net->copy_stream, net->staging_free, 0));
    CUDA_TRY(cudaMemsetAsync(net->loss_sum, 0, sizeof(double), net->stream));
    net->last_train_n = n;
    for (long long c = 0; c < nch; ++c) {
        const long long off = c * chunk;
        const long long len = (n - off) < chunk ? (n - off) : chunk;
        CUDA_TRY(cudaMemcpyAsync(net->st_x + off * 841, h_images + off * 841, sizeof(float) * 841 * len,
                                 cudaMemcpyHostToDevice, net->copy_stream));
        CUDA_TRY(cudaMemcpyAsync(net->st_y + off, h_labels + off, sizeof(int) * len, cudaMemcpyHostToDevice,
                                 net->copy_stream));
        CUDA_TRY(cudaEventRecord(net->chunk_ev[c], net->copy_stream));
        CUDA_TRY(cudaStreamWaitEvent(net->stream, net->chunk_ev[c], 0));
        chaos_status st = train_range(net, net->st_x + off * 841, net->st_y + off, len, lr, mode);
        if (st) return st;
    }
    return synchronize ? chaos_net_sync(net) : CHAOS_OK;
}
}  // namespace

extern "C" {

chaos_status chaos_last_train_loss(chaos_net* net, double* mean_loss) {
    if (!net || !mean_loss) return fail(CHAOS_E_INVALID, "NULL argument");
    double s = 0;
    CUDA_TRY(cudaMemcpyAsync(&s, net->loss_sum, sizeof(double), cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    *mean_loss = net->last_train_n > 0 ? s / (double)net->last_train_n : 0.0;
    return check_latch(net);
}

chaos_status chaos_evaluate(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n,
                            double* mean_loss, int64_t* n_errors) {
    if (!net || !mean_loss || !n_errors) return fail(CHAOS_E_INVALID, "NULL argument");
    if (n < 0) return fail(CHAOS_E_INVALID, "n < 0");
    if (n == 0) {
        *mean_loss = 0.0;
        *n_errors = 0;
        return check_latch(net);
    }
    if (!d_images || !d_labels) return fail(CHAOS_E_INVALID, "NULL images/labels");
    chaos_status s = ensure_eval(net, n);
    if (s) return s;
    KArgs k = base_args(net);
    k.images = d_images;
    k.labels = d_labels;
    k.n = n;
    k.out_loss = net->ev_loss;
    k.out_wrong = net->ev_wrong;
    const int G = net->group;
    const int grid = grid_for(net, kEval, (n + G - 1) / G);
    net->d->fn[gidx(net)][kEval]<<<grid, net->d->nt, net->d->smem[gidx(net)], net->stream>>>(k);
    CUDA_TRY(cudaGetLastError());
    chaos_eval_reduce<<<1, 1024, 0, net->stream>>>(net->ev_loss, net->ev_wrong, n, net->ev_sum, net->ev_err);
    CUDA_TRY(cudaGetLastError());
    double sum = 0;
    long long err = 0;
    CUDA_TRY(cudaMemcpyAsync(&sum, net->ev_sum, sizeof(double), cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaMemcpyAsync(&err, net->ev_err, sizeof(long long), cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    *mean_loss = sum / (double)n;
    *n_errors = err;
    return check_latch(net);
}

chaos_status chaos_forward(chaos_net* net, const float* d_images, int64_t n, float* d_logits) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (n < 0) return fail(CHAOS_E_INVALID, "n < 0");
    if (n == 0) return check_latch(net);
    if (!d_images || !d_logits) return fail(CHAOS_E_INVALID, "NULL argument");
    KArgs k = base_args(net);
    k.images = d_images;
    k.n = n;
    k.out_logits = d_logits;
    const int G = net->group;
    const int grid = grid_for(net, kForward, (n + G - 1) / G);
    net->d->fn[gidx(net)][kForward]<<<grid, net->d->nt, net->d->smem[gidx(net)], net->stream>>>(k);
    CUDA_TRY(cudaGetLastError());
    return check_latch(net);
}

chaos_status chaos_compute_gradients(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n,
                                     float* host_grad_sum) {
    if (!net || !host_grad_sum) return fail(CHAOS_E_INVALID, "NULL argument");
    if (n < 0) return fail(CHAOS_E_INVALID, "n < 0");
    if (!net->grad_out) CUDA_TRY(cudaMalloc(&net->grad_out, sizeof(float) * net->d->pint));
    CUDA_TRY(cudaMemsetAsync(net->grad_out, 0, sizeof(float) * net->d->pint, net->stream));
    if (n > 0) {
        if (!d_images || !d_labels) return fail(CHAOS_E_INVALID, "NULL images/labels");
        chaos_status s = sync_batch(net, d_images, d_labels, n, 0.f, net->grad_out, nullptr);
        if (s) return s;
    }
    std::vector<float> in((size_t)net->d->pint);
    CUDA_TRY(cudaMemcpyAsync(in.data(), net->grad_out, sizeof(float) * in.size(), cudaMemcpyDeviceToHost,
                             net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    to_normative(*net->d, in.data(), host_grad_sum);
    return check_latch(net);
}

chaos_status chaos_batch_gradient(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n,
                                  float* d_grad) {
    if (!net || !d_grad) return fail(CHAOS_E_INVALID, "NULL argument");
    if (n < 0) return fail(CHAOS_E_INVALID, "n < 0");
    if (n == 0) {
        CUDA_TRY(cudaMemsetAsync(d_grad, 0, sizeof(float) * net->d->pint, net->stream));
        return CHAOS_OK;
    }
    if (!d_images || !d_labels) return fail(CHAOS_E_INVALID, "NULL images/labels");
    return sync_batch(net, d_images, d_labels, n, 0.f, d_grad, nullptr);
}

chaos_status chaos_apply_gradient(chaos_net* net, const float* d_grad, float lr) {
    if (!net || !d_grad) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!std::isfinite(lr)) return fail(CHAOS_E_INVALID, "lr is not finite");
    const long long np = net->d->pint;
    chaos_apply_gradient_kernel<<<(unsigned)((np + 255) / 256), 256, 0, net->stream>>>(net->params, d_grad, lr, np);
    CUDA_TRY(cudaGetLastError());
    return CHAOS_OK;
}

uint64_t chaos_progress_enqueued(const chaos_net* net) { return net ? net->progress_enqueued : 0; }

chaos_status chaos_progress_wait(chaos_net* net, uint64_t target, int64_t stream) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (target > net->progress_enqueued)
        return fail(CHAOS_E_INVALID, "progress target %llu beyond the %llu images enqueued (would never return)",
                    (unsigned long long)target, net->progress_enqueued);
    chaos_progress_wait_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(net->progress, target);
    CUDA_TRY(cudaGetLastError());
    return CHAOS_OK;
}

chaos_status chaos_avg_snapshot(chaos_net* net, float* d_snap, int64_t stream) {
    if (!net || !d_snap) return fail(CHAOS_E_INVALID, "NULL argument");
    CUDA_TRY(cudaMemcpyAsync(d_snap, net->params, sizeof(float) * net->d->pint, cudaMemcpyDeviceToDevice,
                             reinterpret_cast<cudaStream_t>(stream)));
    return CHAOS_OK;
}

chaos_status chaos_avg_apply(chaos_net* net, const float* d_avg, const float* d_snap, int64_t stream) {
    if (!net || !d_avg || !d_snap) return fail(CHAOS_E_INVALID, "NULL argument");
    if ((reinterpret_cast<uintptr_t>(d_avg) | reinterpret_cast<uintptr_t>(d_snap)) & 15)
        return fail(CHAOS_E_INVALID, "avg/snap must be 16-byte aligned");
    const long long np = net->d->pint;
    const long long blocks = std::min<long long>((np / 4 + 255) / 256 + 1, 64);
    chaos_avg_apply_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(net->params, d_avg,
                                                                                                  d_snap, np);
    CUDA_TRY(cudaGetLastError());
    return CHAOS_OK;
}

chaos_status chaos_dist_unique_id(void* host_id) {
    if (!host_id) return fail(CHAOS_E_INVALID, "host_id is NULL");
    const NcclApi& n = nccl_api();
    if (!n.ok) return fail(CHAOS_E_NCCL, "%s", n.why.c_str());
    ncclUniqueId id;
    const ncclResult_t r = n.get_unique_id(&id);
    if (r != ncclSuccess) return fail(CHAOS_E_NCCL, "ncclGetUniqueId: %s", n.error_string(r));
    static_assert(sizeof(ncclUniqueId) == CHAOS_DIST_ID_BYTES, "NCCL unique id size");
    std::memcpy(host_id, &id, sizeof id);
    return CHAOS_OK;
}

chaos_status chaos_dist_init(chaos_net* net, const void* host_id, int32_t rank, int32_t world) {
    if (!net || !host_id) return fail(CHAOS_E_INVALID, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(CHAOS_E_INVALID, "rank %d / world %d", rank, world);
    if (net->comm) return fail(CHAOS_E_INVALID, "communicator already initialised");
    const NcclApi& n = nccl_api();
    if (!n.ok) return fail(CHAOS_E_NCCL, "%s", n.why.c_str());
    CUDA_TRY(cudaSetDevice(net->dev));
    ncclUniqueId id;
    std::memcpy(&id, host_id, sizeof id);
    ncclResult_t r;
    if (net->reserve_sms > 0) {
        // in-flight averaging beside a persistent hogwild launch: every block of a
        // collective must be co-resident on the reserved SMs, else a block spinning on a peer's
        // block that cannot be scheduled never finishes -- cap the communicator's CTAs (ring /
        // tree and NVLS) at the reserved SM count
        if (!n.init_rank_config)
            return fail(CHAOS_E_NCCL, "CHAOS_OPT_RESERVE_SMS needs ncclCommInitRankConfig (NCCL >= 2.14)");
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.blocking = 1;
        cfg.minCTAs = 1;
        cfg.maxCTAs = net->reserve_sms;
        cfg.nvlsCTAs = net->reserve_sms;
        cfg.collnetEnable = 0;
        r = n.init_rank_config(&net->comm, world, id, rank, &cfg);
    } else {
        r = n.init_rank(&net->comm, world, id, rank);
    }
    if (r != ncclSuccess) {
        net->comm = nullptr;
        return fail(CHAOS_E_NCCL, "ncclCommInitRank: %s", n.error_string(r));
    }
    net->comm_max_ctas = net->reserve_sms;
    net->comm_world = world;
    return CHAOS_OK;
}

chaos_status chaos_dist_average_buffer(chaos_net* net, float* d_buf, int64_t n, int64_t stream) {
    if (!net || (!d_buf && n > 0) || n < 0) return fail(CHAOS_E_INVALID, "NULL buffer or n < 0");
    if (!net->comm) return fail(CHAOS_E_INVALID, "chaos_dist_init has not been called");
    if (n == 0) return CHAOS_OK;
    const NcclApi& a = nccl_api();
    const ncclResult_t r = a.all_reduce(d_buf, d_buf, static_cast<size_t>(n), ncclFloat32, ncclAvg, net->comm,
                                        reinterpret_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return fail(CHAOS_E_NCCL, "ncclAllReduce: %s", a.error_string(r));
    return CHAOS_OK;
}

chaos_status chaos_dist_average(chaos_net* net) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    return chaos_dist_average_buffer(net, net->params, net->d->pint, reinterpret_cast<int64_t>(net->stream));
}

chaos_status chaos_debug_trace(chaos_net* net, int64_t* host_records, int64_t n_groups, float* host_pubs,
                               float* host_reads) {
    if (!net || !host_records) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->trec || n_groups != net->trace_groups)
        return fail(CHAOS_E_INVALID, "no trace of %lld groups recorded (last: %lld)", (long long)n_groups,
                    net->trace_groups);
    CUDA_TRY(cudaMemcpyAsync(host_records, net->trec, sizeof(long long) * kTraceRec * (size_t)n_groups,
                             cudaMemcpyDeviceToHost, net->stream));
    std::vector<float> slots;
    if (host_pubs) {
        slots.resize((size_t)n_groups * (size_t)net->d->pint);
        CUDA_TRY(cudaMemcpyAsync(slots.data(), net->partial, sizeof(float) * slots.size(), cudaMemcpyDeviceToHost,
                                 net->stream));
    }
    std::vector<float> rd;
    if (host_reads) {
        rd.resize((size_t)n_groups * 2 * (size_t)net->d->pint);
        CUDA_TRY(cudaMemcpyAsync(rd.data(), net->tw, sizeof(float) * rd.size(), cudaMemcpyDeviceToHost, net->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    if (host_pubs)
        for (long long k = 0; k < n_groups; ++k)
            to_normative(*net->d, slots.data() + k * net->d->pint, host_pubs + k * net->d->nparams);
    if (host_reads)
        for (long long k = 0; k < 2 * n_groups; ++k)
            to_normative(*net->d, rd.data() + k * net->d->pint, host_reads + k * net->d->nparams);
    return check_latch(net);
}

chaos_status chaos_debug_claims(chaos_net* net, int32_t* host_counts, int64_t n) {
    if (!net || !host_counts) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->claims || n > net->claims_cap) return fail(CHAOS_E_INVALID, "no claim record of that size");
    CUDA_TRY(cudaMemcpyAsync(host_counts, net->claims, sizeof(int) * n, cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    return CHAOS_OK;
}

chaos_status chaos_debug_phase_times(chaos_net* net, uint64_t* host_cycles, int32_t n) {
    if (!net || !host_cycles || n < 1) return fail(CHAOS_E_INVALID, "NULL argument or n < 1");
#ifdef CHAOS_TIMING
    if (!net->ptime) return fail(CHAOS_E_INVALID, "no hogwild epoch recorded yet");
    std::vector<unsigned long long> h((size_t)kPhases * net->ptime_grid);
    CUDA_TRY(cudaMemcpyAsync(h.data(), net->ptime, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                             net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    for (int k = 0; k < n; ++k) host_cycles[k] = 0;
    for (int b = 0; b < net->ptime_grid; ++b)
        for (int k = 0; k < kPhases && k < n; ++k) host_cycles[k] += h[(size_t)b * kPhases + k];
    return CHAOS_OK;
#else
    (void)n;
    return fail(CHAOS_E_UNSUPPORTED, "phase timing needs the instrumented build (libchaos_timing.so, -DCHAOS_TIMING)");
#endif
}

chaos_status chaos_pavg_setup(chaos_net* net, int32_t rank, int32_t world, int64_t k, int32_t nslice) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (world < 1 || world > kPavgMaxR || rank < 0 || rank >= world)
        return fail(CHAOS_E_INVALID, "rank %d / world %d (world in [1, %d])", rank, world, kPavgMaxR);
    if (k < 1) return fail(CHAOS_E_INVALID, "averaging interval k must be >= 1");
    if (nslice == 0) nslice = net->sms;
    if (nslice < 1) return fail(CHAOS_E_INVALID, "nslice must be >= 1 (0 = the SM count)");
    if (net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup already called for this net");
    const long long pint = net->d->pint;
    const int sfl = (int)(((pint + nslice - 1) / nslice + 3) / 4 * 4);
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t snap = sizeof(float) * (size_t)kPavgBufs * (size_t)nslice * (size_t)sfl;
    net->px_off_flag = up(snap);
    net->px_off_done = net->px_off_flag + up(sizeof(unsigned) * (size_t)nslice);
    net->px_off_cks = net->px_off_done + up(sizeof(unsigned) * (size_t)nslice);
    net->px_bytes = net->px_off_cks + up(sizeof(unsigned long long) * (size_t)nslice * kPavgBufs);
    CUDA_TRY(cudaMalloc(&net->px, net->px_bytes));
    CUDA_TRY(cudaMemset(net->px, 0, net->px_bytes));  // flags / done start at round 0
    CUDA_TRY(cudaMalloc(&net->px_dev, sizeof(PavgArgs)));
    PavgArgs& h = net->px_host;
    h = PavgArgs{};
    h.R = world;
    h.rank = rank;
    h.nslice = nslice;
    h.slice_fl = sfl;
    h.pint = pint;
    h.latch = net->latch;
    net->px_k = k;
    net->px_round0 = 0;
    net->px_arm = 0;
    net->px_peers_set = 0;
    net->px_dirty = true;
    return chaos_pavg_set_peer(net, rank, net->px);
}

chaos_status chaos_pavg_exchange(chaos_net* net, int32_t peer, void** d_ptr, int64_t* bytes) {
    if (!net || !d_ptr || !bytes) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup has not been called");
    if (peer < 0 || peer >= net->px_host.R || !(net->px_peers_set & (1 << peer)))
        return fail(CHAOS_E_INVALID, "no exchange buffer for rank %d", peer);
    *d_ptr = net->px_host.snap[peer];
    *bytes = (int64_t)net->px_bytes;
    return CHAOS_OK;
}

chaos_status chaos_pavg_debug_sums(chaos_net* net, float* host_dsum, float* host_dabs, int64_t n) {
    if (!net || !host_dsum || !host_dabs) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->px || !net->px_host.dsum) return fail(CHAOS_E_INVALID, "chaos_pavg_set_check has not been called");
    if (n != net->d->pint) return fail(CHAOS_E_INVALID, "n=%lld != chaos_net_device_params_len=%lld", (long long)n,
                                       net->d->pint);
    CUDA_TRY(cudaMemcpyAsync(host_dsum, net->px_host.dsum, sizeof(float) * n, cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaMemcpyAsync(host_dabs, net->px_host.dabs, sizeof(float) * n, cudaMemcpyDeviceToHost, net->stream));
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    return check_latch(net);
}

chaos_status chaos_pavg_ipc_handle(chaos_net* net, void* host_handle) {
    if (!net || !host_handle) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup has not been called");
    static_assert(sizeof(cudaIpcMemHandle_t) == CHAOS_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t hd;
    CUDA_TRY(cudaIpcGetMemHandle(&hd, net->px));
    std::memcpy(host_handle, &hd, sizeof hd);
    return CHAOS_OK;
}

chaos_status chaos_pavg_set_peer(chaos_net* net, int32_t peer, void* d_exchange) {
    if (!net || !d_exchange) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup has not been called");
    PavgArgs& h = net->px_host;
    if (peer < 0 || peer >= h.R) return fail(CHAOS_E_INVALID, "peer %d outside [0, %d)", peer, h.R);
    if (reinterpret_cast<uintptr_t>(d_exchange) & 255) return fail(CHAOS_E_INVALID, "exchange buffer not 256-B aligned");
    char* b = static_cast<char*>(d_exchange);
    h.snap[peer] = reinterpret_cast<float*>(b);
    h.flag[peer] = reinterpret_cast<unsigned*>(b + net->px_off_flag);
    h.done[peer] = reinterpret_cast<unsigned*>(b + net->px_off_done);
    h.cks[peer] = reinterpret_cast<unsigned long long*>(b + net->px_off_cks);
    net->px_peers_set |= 1 << peer;
    net->px_dirty = true;
    return CHAOS_OK;
}

chaos_status chaos_pavg_open_peer(chaos_net* net, int32_t peer, const void* host_handle) {
    if (!net || !host_handle) return fail(CHAOS_E_INVALID, "NULL argument");
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup has not been called");
    if (peer < 0 || peer >= net->px_host.R || peer == net->px_host.rank)
        return fail(CHAOS_E_INVALID, "peer %d: not another rank of [0, %d)", peer, net->px_host.R);
    if (net->px_mapped[peer]) return fail(CHAOS_E_INVALID, "peer %d already opened", peer);
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, host_handle, sizeof hd);
    void* p = nullptr;
    CUDA_TRY(cudaSetDevice(net->dev));
    CUDA_TRY(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
    net->px_mapped[peer] = p;
    return chaos_pavg_set_peer(net, peer, p);
}

chaos_status chaos_pavg_arm(chaos_net* net, int64_t rounds) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup has not been called");
    if (rounds < 0 || rounds > (1 << 20)) return fail(CHAOS_E_INVALID, "rounds must be in [0, 2^20]");
    net->px_arm = rounds;
    return CHAOS_OK;
}

int64_t chaos_pavg_rounds_done(const chaos_net* net) { return net ? net->px_round0 : -1; }

chaos_status chaos_pavg_set_check(chaos_net* net, int32_t on) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (!net->px) return fail(CHAOS_E_INVALID, "chaos_pavg_setup has not been called");
    net->px_host.check = on ? 1 : 0;
    if (on) {  // (re)start the delta sums
        const size_t b = sizeof(float) * (size_t)net->d->pint;
        if (!net->px_host.dsum) {
            CUDA_TRY(cudaMalloc(&net->px_host.dsum, b));
            CUDA_TRY(cudaMalloc(&net->px_host.dabs, b));
        }
        CUDA_TRY(cudaMemsetAsync(net->px_host.dsum, 0, b, net->stream));
        CUDA_TRY(cudaMemsetAsync(net->px_host.dabs, 0, b, net->stream));
    }
    net->px_dirty = true;
    return CHAOS_OK;
}

chaos_status chaos_train_epoch_replicas(chaos_net* const* nets, int32_t R, const float* const* d_images,
                                        const int32_t* const* d_labels, const int64_t* n, float lr) {
    if (!nets || !d_images || !d_labels || !n) return fail(CHAOS_E_INVALID, "NULL argument");
    if (R < 1 || R > kPavgMaxR) return fail(CHAOS_E_INVALID, "R must be in [1, %d]", kPavgMaxR);
    if (!std::isfinite(lr)) return fail(CHAOS_E_INVALID, "lr is not finite");
    chaos_net* n0 = nets[0];
    if (!n0) return fail(CHAOS_E_INVALID, "nets[0] is NULL");
    if (!n0->d->fn_rep) return fail(CHAOS_E_UNSUPPORTED, "net %s has no replica-emulation build", n0->d->name);
    if (n0->group != n0->d->gdef) return fail(CHAOS_E_INVALID, "replica emulation runs at the net's default G");
    const int G = n0->group;
    const int comm = n0->px_arm > 0 ? n0->px_comm : 0;
    int cta = (n0->sms - n0->reserve_sms) / R - comm;  // training CTAs per replica
    if ((long long)cta * G > n0->d->max_inflight) cta = n0->d->max_inflight / G;
    if (n0->max_ctas > 0 && cta > n0->max_ctas) cta = n0->max_ctas;
    if (cta < 1) return fail(CHAOS_E_INVALID, "no training CTA per replica");
    std::vector<KArgs> ka((size_t)R);
    for (int r = 0; r < R; ++r) {
        chaos_net* net = nets[r];
        if (!net || net->d != n0->d || net->dev != n0->dev || net->group != G)
            return fail(CHAOS_E_INVALID, "replica %d: NULL, another arch / device or another G", r);
        if (n[r] < 1 || !d_images[r] || !d_labels[r]) return fail(CHAOS_E_INVALID, "replica %d: empty shard", r);
        if (net->debug_trace) return fail(CHAOS_E_UNSUPPORTED, "replica emulation is not traced");
        for (int q = 0; q < r; ++q)
            if (nets[q] == net) return fail(CHAOS_E_INVALID, "replica %d repeats replica %d", r, q);
        KArgs k = base_args(net);
        k.images = d_images[r];
        k.labels = d_labels[r];
        k.n = n[r];
        k.neg_lr = -lr;
        k.loss_sum = net->loss_sum;
        k.progress = net->progress;
        if (net->px_arm > 0) {
            if (!net->px || net->px_host.R != R || net->px_host.rank != r)
                return fail(CHAOS_E_INVALID, "replica %d: fused averaging set up for rank %d of %d", r,
                            net->px ? net->px_host.rank : -1, net->px ? net->px_host.R : 0);
            if (net->px_arm != n0->px_arm || net->px_round0 != n0->px_round0 || net->px_comm != n0->px_comm)
                return fail(CHAOS_E_INVALID, "replica %d: armed rounds / comm CTAs differ from replica 0", r);
            if (net->px_peers_set != (1 << R) - 1)  // (checked here so no replica's rounds are consumed)
                return fail(CHAOS_E_INVALID, "replica %d: exchange buffers of %d replicas expected, peer mask 0x%x",
                            r, R, net->px_peers_set);
        } else if (n0->px_arm > 0) {
            return fail(CHAOS_E_INVALID, "replica %d is not armed like replica 0", r);
        }
        ka[(size_t)r] = k;
    }
    for (int r = 0; r < R; ++r) {  // after validation: consumes the armed rounds
        chaos_net* net = nets[r];
        if (net != n0) CUDA_TRY(cudaStreamSynchronize(net->stream));  // its earlier work precedes the launch
        CUDA_TRY(cudaMemsetAsync(net->counter, 0, sizeof(unsigned long long), n0->stream));
        CUDA_TRY(cudaMemsetAsync(net->loss_sum, 0, sizeof(double), n0->stream));
        net->last_train_n = n[r];
        net->progress_enqueued += (unsigned long long)n[r];
        if (net->px_arm > 0) {
            chaos_status st = pavg_args(net, ka[(size_t)r]);
            if (st) return st;
            if (net != n0) CUDA_TRY(cudaStreamSynchronize(net->stream));  // its table copy
        }
    }
    if (!n0->rep_dev) CUDA_TRY(cudaMalloc(&n0->rep_dev, sizeof(KArgs) * kPavgMaxR));
    CUDA_TRY(cudaMemcpyAsync(n0->rep_dev, ka.data(), sizeof(KArgs) * (size_t)R, cudaMemcpyHostToDevice, n0->stream));
    KArgs k0 = ka[0];
    k0.reps = n0->rep_dev;
    k0.rep_ctas = cta + comm;
    void* args[] = {&k0};
    // cooperative: all R * cta CTAs are co-resident (the replicas' CTAs wait on one another)
    CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(n0->d->fn_rep), dim3((unsigned)(R * (cta + comm))),
                                         dim3((unsigned)n0->d->nt), args, (size_t)n0->d->smem[gidx(n0)], n0->stream));
    for (int r = 1; r < R; ++r) {  // the replicas' own streams wait for the launch
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(e, n0->stream));
        CUDA_TRY(cudaStreamWaitEvent(nets[r]->stream, e, 0));
        CUDA_TRY(cudaEventDestroy(e));
    }
    return CHAOS_OK;
}

chaos_status chaos_net_sync(chaos_net* net) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    CUDA_TRY(cudaStreamSynchronize(net->stream));
    return check_latch(net);
}

chaos_status chaos_net_launch_info(chaos_net* net, int32_t* grid, int32_t* block, int32_t* smem_bytes,
                                   int32_t* group) {
    if (!net) return fail(CHAOS_E_INVALID, "net is NULL");
    if (grid) *grid = grid_for(net, kHogwild, 1LL << 40);
    if (block) *block = net->d->nt;
    if (smem_bytes) *smem_bytes = net->d->smem[gidx(net)];
    if (group) *group = net->group;
    return CHAOS_OK;
}

}  // extern "C"
