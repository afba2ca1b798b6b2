/*
 * chaos.h -- C ABI of the B200-native CHAOS training hot path (libchaos.so).
 *
 * CHAOS = "Controlled Hogwild with Arbitrary Order of Synchronization",
 * Viebke & Pllana, arXiv:1506.09067, §III-A.  The library
 * trains small MNIST-shaped CNNs (conv -> tanh -> max-pool blocks, fully
 * connected layers, softmax cross-entropy; Table I
 * PAPER.md:212-247) with per-sample forward propagation, back-propagation and
 * the controlled-hogwild shared-weight update, all in hand-written sm_100a
 * kernels.  No C++ type, exception or torch type crosses this boundary.
 *
 * Conventions (apply to every call):
 *  - Ownership: the net owns its device parameters, scratch, work counter and
 *    error latch (cudaMalloc on the device current at chaos_net_create).  Device
 *    image/label pointers passed in are BORROWED and must stay valid until the
 *    net's stream has passed the call.  Host buffers are caller-owned.
 *  - Threading: one host thread per net.
 *  - Streams: all device work is enqueued on the net's stream
 *    (CHAOS_OPT_STREAM; default = the legacy default stream).
 *  - Errors: argument / architecture errors return immediately with a status and
 *    set chaos_last_error().  Errors detected on the device (label outside
 *    [0, n_classes), non-finite loss) are latched and returned by the next
 *    synchronizing call (chaos_evaluate, chaos_net_get_params, chaos_net_sync,
 *    chaos_compute_gradients, chaos_forward).
 *  - n == 0 is a no-op returning CHAOS_OK.
 *  - Data layout: images fp32 [n][in_c][in_h][in_w] contiguous, labels int32 [n].
 *  - Parameter layout (normative; get/set/compute_gradients use it): for each
 *    weighted layer in order, W then b; conv W is [M][C][k][k], FC W is
 *    [N][In]; the FC input is flattened [map][row][col].  Counts follow Table I's
 *    "+1" formula: conv M*(C*k*k+1), FC N*(In+1).  The device
 *    keeps its own internal layout (conv W transposed to [C*k*k][M'] with M
 *    padded to a multiple of 4, every block 16-byte aligned); get/set convert.
 */
#ifndef CHAOS_H
#define CHAOS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CHAOS_OK = 0,
    CHAOS_E_INVALID = -1,     /* bad argument (NULL, n<0, non-finite lr, ...) */
    CHAOS_E_ARCH = -2,        /* shape chain invalid (message names the layer) */
    CHAOS_E_UNSUPPORTED = -3, /* valid arch without a compiled sm_100a instantiation */
    CHAOS_E_LABEL = -4,       /* device latch: a label outside [0, n_classes) */
    CHAOS_E_NONFINITE = -5,   /* device latch: non-finite loss */
    CHAOS_E_CUDA = -6,        /* CUDA runtime error (message has cudaGetErrorString) */
    CHAOS_E_NCCL = -7         /* chaos_dist_*: libnccl.so.2 not loadable or an NCCL error */
} chaos_status;

typedef enum { CHAOS_CONV = 1, CHAOS_MAXPOOL = 2, CHAOS_FULL = 3 } chaos_layer_kind;
typedef enum { CHAOS_TANH = 0, CHAOS_IDENTITY = 1 } chaos_act; /* last FULL = logits -> softmax-CE */

typedef struct {
    int32_t kind;   /* chaos_layer_kind */
    int32_t units;  /* conv: output maps; full: neurons; maxpool: ignored */
    int32_t kernel; /* conv kernel k (k x k, stride 1, valid) or pool window kp (kp x kp, stride kp, floor) */
    int32_t act;    /* chaos_act: conv/full hidden layers CHAOS_TANH, last full CHAOS_IDENTITY */
} chaos_layer;

typedef struct {
    int32_t in_c, in_h, in_w, n_classes, n_layers;
    chaos_layer layers[16];
    uint64_t init_seed; /* parameters U(+-1/sqrt(fan_in)) from splitmix64(init_seed ^ 0x5EED) (R7) */
} chaos_arch;

/* Paper: Training with several workers sharing weights.
 * HOGWILD: persistent CTAs claim groups of G images from a device counter
 *   (first come, first served) and, after each layer's gradient
 *   and the previous layer's partial derivatives are computed, add -lr*gradient
 *   to the shared fp32 weights with atomics in arbitrary order.
 * SYNC: deterministic: consecutive batches of CHAOS_OPT_SYNC_BATCH images; every
 *   gradient at the batch-start weights; one update W -= lr * sum_i g_i, the sum
 *   taken in a fixed order (BASELINE.json north_star).  Bitwise run-to-run
 *   reproducible. */
typedef enum { CHAOS_HOGWILD = 0, CHAOS_SYNC = 1 } chaos_mode;

typedef enum {
    CHAOS_OPT_STREAM = 0,        /* value = (int64_t)cudaStream_t */
    CHAOS_OPT_SYNC_BATCH = 1,    /* B >= 1, default 64 */
    CHAOS_OPT_GROUP = 2,         /* G, images per CTA per claim: compiled values 1 and the net's default.
                                    Never set: hogwild runs at the net's default G, and a sync / gradient
                                    batch of fewer than G x #SMs images at G = 1 (it then fills G times more
                                    SMs; the fixed summation order is that of G = 1).
                                    A worker publishes each layer's G-image gradient sum once (G_pub = G,
                                    the paper's delayed updates); SURVEY's separate
                                    CHAOS_OPT_PUBLISH_GROUP is not exposed: publishing per image inside a
                                    G-image group would need G gradient buffers per layer in shared memory
                                    (the 227 KB budget holds one); G = 1 gives G_pub = 1 */
    CHAOS_OPT_MAX_CTAS = 3,      /* cap on resident CTAs (1 => a single worker = sequential SGD when G=1) */
    CHAOS_OPT_DEBUG_CLAIMS = 4,  /* 1 => count claims per image into a device buffer (exactly-once test) */
    CHAOS_OPT_RESERVE_SMS = 5,   /* hogwild: leave this many SMs free of training CTAs (room for concurrent
                                    averaging / NCCL kernels, chaos_progress_wait), in [0, #SMs), default 0;
                                    set it before chaos_dist_init, which caps the communicator's CTAs at it */
    CHAOS_OPT_DEBUG_TRACE = 6,   /* 1 => hogwild epochs record their schedule (chaos_debug_trace); tiny and
                                    large nets; CHAOS_E_UNSUPPORTED elsewhere */
    CHAOS_OPT_DEBUG_STAGGER = 7, /* trace epochs: CTA b starts b * value cycles late (varied interleavings) */
    CHAOS_OPT_PAVG_COMM_CTAS = 8 /* fused averaging (chaos_pavg_*): 0 (default) = the training CTAs run the
                                    rounds between image groups; c in [1, 16] = c extra CTAs of the launch
                                    (SMs of their own) run them and the training CTAs never stall on one */
} chaos_option;

typedef struct chaos_net chaos_net;

/* Validate the arch, pick the compiled instantiation, allocate, initialise the
 * parameters.  NULL on error (see chaos_last_error(); status via chaos_last_status()). */
chaos_net* chaos_net_create(const chaos_arch* arch);
void chaos_net_destroy(chaos_net* net);
chaos_status chaos_net_set_option(chaos_net* net, chaos_option opt, int64_t value);
int64_t chaos_net_get_option(const chaos_net* net, chaos_option opt);
int64_t chaos_net_num_params(const chaos_net* net);
/* Synchronizing.  host_dst / host_src hold n == num_params floats, normative layout. */
chaos_status chaos_net_get_params(chaos_net* net, float* host_dst, int64_t n);
chaos_status chaos_net_set_params(chaos_net* net, const float* host_src, int64_t n);
/* Device pointer to the internal parameter buffer (for NCCL / torch views of the
 * whole buffer; element-wise averaging is layout independent). */
float* chaos_net_device_params(chaos_net* net);
int64_t chaos_net_device_params_len(const chaos_net* net); /* floats, incl. padding */

/* One Training phase over images [0, n).  Asynchronous on the
 * net's stream.  lr is per call: the caller applies the x0.9/epoch schedule. */
chaos_status chaos_train_epoch(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n, float lr,
                               chaos_mode mode);
/* Same, from HOST buffers -- the end-to-end entry point.  The images/labels are copied to
 * net-owned device staging buffers on a net-owned copy stream, overlapping training (pinned host
 * memory required for the overlap).  Hogwild: ONE launch over [0, n); the copy stream lands
 * ~n/16-image chunks and after each advances a device counter of landed images, and a worker that
 * claims a group waits in its claim until the group has landed (so only the first chunk's copy
 * is exposed; the debug claim record covers the whole epoch).  Sync: chunks of whole batches,
 * chunk c+1 copied while chunk c trains, so the result equals chaos_train_epoch(SYNC) bitwise.
 * Synchronizing on return. */
chaos_status chaos_train_epoch_host(chaos_net* net, const float* h_images, const int32_t* h_labels, int64_t n,
                                    float lr, chaos_mode mode);
/* chaos_train_epoch_host without the final synchronization: returns once the copies and the
 * launch(es) are enqueued (asynchronous on the net's and its copy stream).  The host buffers must
 * stay valid (and unmodified) until the net's stream has passed the epoch (chaos_net_sync). */
chaos_status chaos_train_epoch_host_async(chaos_net* net, const float* h_images, const int32_t* h_labels,
                                          int64_t n, float lr, chaos_mode mode);
/* Mean training loss (double) of the last chaos_train_epoch call; synchronizing. */
chaos_status chaos_last_train_loss(chaos_net* net, double* mean_loss);

/* Validation / Testing: forward only; mean cross-entropy (fixed-order
 * double sum) and the number of images whose argmax logit (lowest index on ties)
 * differs from the label.  Synchronizing.  Never writes the parameters. */
chaos_status chaos_evaluate(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n,
                            double* mean_loss, int64_t* n_errors);
/* Forward only: logits [n][n_classes] into the device buffer d_logits.  Synchronizing. */
chaos_status chaos_forward(chaos_net* net, const float* d_images, int64_t n, float* d_logits);
/* Test hook: host_grad_sum[j] = sum_i dL_i/dparam_j at the current weights (normative
 * layout, no update; fixed-order sum).  Synchronizing. */
chaos_status chaos_compute_gradients(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n,
                                     float* host_grad_sum);
/* Deterministic multi-GPU sync mode (BASELINE.json north_star "sums a fixed
 * batch's gradients in a fixed order before one update"), in two steps so a collective can sit in
 * between.  chaos_batch_gradient: d_grad[j] = sum_i dL_i/dparam_j over images [0, n) at the current
 * weights (every g_i at the same weights; slot-ordered, fixed-order sum), in the INTERNAL layout
 * (chaos_net_device_params_len floats; padding entries are written 0).  d_grad is caller-owned
 * device memory; asynchronous on the net's stream; n == 0 writes zeros.  Device-detected label /
 * non-finite errors are latched as for chaos_train_epoch.
 * chaos_apply_gradient: param[j] -= lr * d_grad[j] over the internal layout (one rounding, the same
 * expression as the single-GPU sync update, so batch_gradient + apply_gradient on one GPU reproduce
 * chaos_train_epoch(SYNC) bitwise).  Asynchronous on the net's stream. */
chaos_status chaos_batch_gradient(chaos_net* net, const float* d_images, const int32_t* d_labels, int64_t n,
                                  float* d_grad);
chaos_status chaos_apply_gradient(chaos_net* net, const float* d_grad, float lr);

/* Asynchronous cross-GPU averaging (the paper's "arbitrary order of
 * synchronization" carried across GPUs).  While one hogwild
 * launch trains on the net's stream, a caller-owned second stream (cast to int64_t) repeatedly
 * waits for K more images of progress, snapshots the weights, all-reduces the snapshot (NCCL AVG,
 * caller side) and adds (avg - snapshot) to the live weights, so the local updates made during the
 * collective are kept.  None of these calls delays the training kernel.
 * chaos_progress_enqueued: images enqueued to this net's hogwild launches since creation (host
 *   counter, not synchronizing).  The device progress counter -- bumped by each CTA once a group's
 *   updates are published -- reaches it when those launches complete.
 * chaos_progress_wait: enqueue on `stream` one single-thread kernel that returns once the device
 *   progress counter >= target.  target > chaos_progress_enqueued() is CHAOS_E_INVALID (it could
 *   never return).  Runs beside the training kernel on a free SM (CHAOS_OPT_RESERVE_SMS).
 * chaos_avg_snapshot: d_snap[0..chaos_net_device_params_len) = params (device copy on `stream`).
 * chaos_avg_apply: params[j] += d_avg[j] - d_snap[j] over the internal layout with atomic adds on
 *   `stream`, safe beside a running hogwild launch; d_avg/d_snap caller-owned, 16-B aligned. */
uint64_t chaos_progress_enqueued(const chaos_net* net);
chaos_status chaos_progress_wait(chaos_net* net, uint64_t target, int64_t stream);
chaos_status chaos_avg_snapshot(chaos_net* net, float* d_snap, int64_t stream);
chaos_status chaos_avg_apply(chaos_net* net, const float* d_avg, const float* d_snap, int64_t stream);

/* Library-owned NCCL communicator (optional: dist.py's torch.distributed path
 * needs none of this).  The averaging is R11: w <- (1/P) sum_r w_r (ncclAvg, in place).
 * libnccl.so.2 is loaded at run time (the copy the process already holds, else the system one);
 * if it cannot be loaded the calls return CHAOS_E_NCCL, as do NCCL errors (message in
 * chaos_last_error()).
 * chaos_dist_unique_id: writes an NCCL unique id (CHAOS_DIST_ID_BYTES bytes) to host_id; call on
 *   rank 0 and send the bytes to every rank (e.g. a torch.distributed broadcast).
 * chaos_dist_init: creates the net's communicator, rank in [0, world); collective (every rank
 *   calls it) and synchronizing.  Destroyed with the net.
 * chaos_dist_average: params <- average over the ranks, on the net's stream, asynchronous.
 * chaos_dist_average_buffer: the same on n floats of caller-owned device memory on `stream`
 *   (cast cudaStream_t; the in-flight averaging of the asynchronous schedule). */
#define CHAOS_DIST_ID_BYTES 128
chaos_status chaos_dist_unique_id(void* host_id);
chaos_status chaos_dist_init(chaos_net* net, const void* host_id, int32_t rank, int32_t world);
chaos_status chaos_dist_average(chaos_net* net);
chaos_status chaos_dist_average_buffer(chaos_net* net, float* d_buf, int64_t n, int64_t stream);

/* Fused in-kernel cross-replica averaging (the fused variant; PAPER.md:138-140
 * "arbitrary order of synchronization" carried across replicas, PAPER.md:412 CHAOS on several
 * devices).  The persistent hogwild kernel averages the replicas itself, between image
 * groups, through peer memory -- no collective launch, no reserved SMs.  The weight vector is cut
 * into nslice slices; CTA c owns slices c, c + ctas, ...  Round t of a launch is due once t*k of the
 * replica's images are claimed; then each CTA copies its slices of the live weights into its own
 * snapshot ring (4 buffers), publishes a per-slice flag, and -- once every replica's flag for the
 * slice has reached the round -- reads all R snapshots (NVLink loads through CUDA-IPC mappings, or
 * same-device buffers) and adds (fixed-order mean - own snapshot) to its live weights with
 * reductions, keeping the hogwild updates made meanwhile; every replica computes the same mean, so
 * each round preserves the replicas' sum up to the rounding of the deltas.  A launch returns only
 * after all its rounds are applied on every replica; every replica must run the same launches
 * with the same armed rounds (collective), so the caller agrees the count (e.g. from the shortest
 * shard).  The final exact average after a launch is the caller's (chaos_dist_average / NCCL).
 * A launch whose peers stop publishing (a dead rank) does not hang: after ~10 s of waiting it gives
 * its remaining rounds up and the next synchronizing call returns CHAOS_E_CUDA ("waited").
 * chaos_pavg_setup: allocates this replica's exchange buffer (cudaMalloc, zeroed: snapshot ring +
 *   flags + checksums) for rank in [0, world), world <= 8, interval k >= 1 images, nslice slices
 *   (0 = the SM count; every replica must use the same value and the same arch).  Once per net.
 * chaos_pavg_exchange: the device pointer of rank `peer`'s exchange buffer as this net maps it (its
 *   own for peer == rank; same-process peers, tests) and the buffer size.
 * chaos_pavg_ipc_handle: writes its CUDA IPC handle (CHAOS_IPC_HANDLE_BYTES bytes) to host_handle,
 *   to be sent to the other ranks (e.g. a torch.distributed all-gather).
 * chaos_pavg_open_peer: maps rank `peer`'s exchange buffer from its IPC handle (another process,
 *   another GPU: peer access enabled lazily); closed with the net.
 * chaos_pavg_set_peer: uses an exchange buffer of this process (another net) for rank `peer`.
 * chaos_pavg_arm: the net's next hogwild launch (device or host entry) runs `rounds` averaging
 *   rounds; every peer table entry must be set by then (CHAOS_E_INVALID otherwise).
 * chaos_pavg_rounds_done: rounds launched so far (round numbers are absolute and monotonic).
 * chaos_pavg_set_check: debug: every snapshot is checksummed and every read of it verified in the
 *   kernel; a mismatch (a torn or stale peer read) latches CHAOS_E_CUDA.  Also (re)starts two
 *   device sums over this replica's applied deltas, per weight: the signed sum and the sum of
 *   magnitudes (summed over the replicas, the signed one is 0 up to rounding: every round preserves
 *   the replicas' sum).
 * chaos_pavg_debug_sums: copies those two sums (internal layout, n = chaos_net_device_params_len)
 *   to the host; synchronizing; returns latched errors.
 * chaos_train_epoch_replicas: one-GPU emulation of R replicas (this build: the large net): ONE
 *   cooperative hogwild launch, CTAs split evenly, replica r = nets[r] trains its own images
 *   d_images[r] / d_labels[r] (n[r] >= 1 images) into its own weights, with the fused averaging when
 *   armed (nets[r] set up as rank r of R, with each other's exchange buffers).  Asynchronous on
 *   nets[0]'s stream; the other nets' streams wait for it. */
#define CHAOS_IPC_HANDLE_BYTES 64
chaos_status chaos_pavg_setup(chaos_net* net, int32_t rank, int32_t world, int64_t k, int32_t nslice);
chaos_status chaos_pavg_exchange(chaos_net* net, int32_t peer, void** d_ptr, int64_t* bytes);
chaos_status chaos_pavg_ipc_handle(chaos_net* net, void* host_handle);
chaos_status chaos_pavg_open_peer(chaos_net* net, int32_t peer, const void* host_handle);
chaos_status chaos_pavg_set_peer(chaos_net* net, int32_t peer, void* d_exchange);
chaos_status chaos_pavg_arm(chaos_net* net, int64_t rounds);
int64_t chaos_pavg_rounds_done(const chaos_net* net);
chaos_status chaos_pavg_set_check(chaos_net* net, int32_t on);
chaos_status chaos_pavg_debug_sums(chaos_net* net, float* host_dsum, float* host_dabs, int64_t n);
chaos_status chaos_train_epoch_replicas(chaos_net* const* nets, int32_t R, const float* const* d_images,
                                        const int32_t* const* d_labels, const int64_t* n, float lr);

/* Debug (controlled hogwild / arbitrary order of synchronization; checked by
 * replaying the recorded schedule in the oracle): after a hogwild epoch
 * run with CHAOS_OPT_DEBUG_TRACE=1 over n images with group size G (n_groups = ceil(n / G)), copies
 * host_records[n_groups][32] (int64, group k = images [k*G, min(k*G+G, n))): for weighted layer
 * l < 5, [6l+0] the rank of its publish on the "started" event counter, [6l+1] the rank on the
 * "done" counter (counted after the layer's reductions completed), [6l+2] / [6l+3] the done count
 * when the forward read of that layer began / the started count when it ended, [6l+4] / [6l+5] the
 * same for the delta_in read (-1: the forward read serves it); [30] the worker (CTA), [31] its
 * iteration.  A publish j was seen by a read iff done_j < read begin; not seen iff started_j >= read
 * end; otherwise it overlapped the read (torn reads possible).  host_pubs (may be NULL):
 * [n_groups][num_params] each group's publish (-lr * its gradient sum), normative layout.
 * host_reads (may be NULL): [n_groups][2][num_params] the weight values each group actually read,
 * [.][0] for its forward pass, [.][1] for its delta_in back-propagation (NaN where the forward
 * read's copy served), normative layout.
 * Synchronizing; CHAOS_E_INVALID if the last epoch did not record n_groups groups. */
chaos_status chaos_debug_trace(chaos_net* net, int64_t* host_records, int64_t n_groups, float* host_pubs,
                               float* host_reads);

/* Debug: copies the per-image claim counts of the last hogwild epoch (needs
 * CHAOS_OPT_DEBUG_CLAIMS=1 before the epoch) into host_counts[n]. */
chaos_status chaos_debug_claims(chaos_net* net, int32_t* host_counts, int64_t n);

/* Profiling hook: per-phase clock64 cycles of the last hogwild epoch, summed over CTAs, into
 * host_cycles[0..n) (20 slots: claim, stage, conv1..3 fwd, fc2 fwd, loss, fc2 bwd, fc1 bwd,
 * conv3 din, conv3 gW, W2 load, conv2 gW, conv2 din, image reload, conv1 gW, fc1 fwd, 3 spare).  Only the
 * instrumented build (libchaos_timing.so, -DCHAOS_TIMING) records them; the product build
 * returns CHAOS_E_UNSUPPORTED.  Synchronizing. */
chaos_status chaos_debug_phase_times(chaos_net* net, uint64_t* host_cycles, int32_t n);

/* Waits for the net's stream; returns (and clears) latched device errors. */
chaos_status chaos_net_sync(chaos_net* net);
/* Number of SMs and resident CTAs per SM the training kernel uses (for reports). */
chaos_status chaos_net_launch_info(chaos_net* net, int32_t* grid, int32_t* block, int32_t* smem_bytes, int32_t* group);
/* Thread-local message of the last failing call on this thread. */
const char* chaos_last_error(void);
chaos_status chaos_last_status(void);

#ifdef __cplusplus
}
#endif
#endif
