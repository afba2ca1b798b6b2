/*
 * oracle.h -- plain, slow, obviously-correct CPU reference of the CHAOS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares
 * no code, header, table or constant with the CUDA path (paper_1506_09067_b200/),
 * and neither includes the other.
 *
 * Everything is double precision (SURVEY.md §8c C-16 reading: the paper never
 * states a precision).  Parameters use the normative flat layout:
 * for each weighted layer in order, W then b; conv W is [M][C][k][k], FC W is
 * [N][In]; the FC input is the previous layer's output flattened [map][row][col].
 *
 * Paper references are PAPER.md line numbers (P:n), section §II-A / §III-A.
 */
#ifndef CHAOS_ORACLE_H
#define CHAOS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_CONV = 1, ORC_POOL = 2, ORC_FULL = 3 };
enum { ORC_TANH = 0, ORC_IDENT = 1 };
enum { ORC_OK = 0, ORC_E_INVALID = -1, ORC_E_ARCH = -2, ORC_E_LABEL = -4 };

typedef struct {
    int32_t kind;   /* ORC_CONV / ORC_POOL / ORC_FULL */
    int32_t units;  /* conv: output maps; full: neurons; pool: ignored */
    int32_t kernel; /* conv kernel k (k x k) or pool window kp (kp x kp); full: ignored */
    int32_t act;    /* ORC_TANH / ORC_IDENT (conv, full); pool: ignored */
} orc_layer;

typedef struct {
    int32_t in_c, in_h, in_w, n_classes, n_layers;
    orc_layer layers[16];
} orc_arch;

/* Number of parameters (Table I "+1" formula), or <0 on a bad arch.
 * err (may be NULL) receives a message of at most errlen bytes. */
int64_t orc_num_params(const orc_arch* a, char* err, int32_t errlen);

/* Per weighted layer: out[3*l+0]=fan_in, out[3*l+1]=#W, out[3*l+2]=#b.  Returns #weighted layers. */
int32_t orc_blocks(const orc_arch* a, int64_t* out, int32_t max_layers);

/* Size (doubles) of the forward trace: every layer's output, concatenated. */
int64_t orc_trace_len(const orc_arch* a);

/* Forward propagation of one 1xHxW sample.  logits[n_classes].
 * trace (may be NULL): every layer's output in order (conv: activated conv maps,
 * pool: pooled maps, full: activated outputs).  argmax (may be NULL): for every
 * pool layer in order, the in-window index u*kp+v of each pooled output. */
int32_t orc_forward(const orc_arch* a, const double* params, const float* x,
                    double* logits, double* trace, uint8_t* argmax);

/* Loss and gradient of one sample: *loss = logsumexp(z) - z[label];
 * grad_accum[j] += dL/dparam_j (normative layout).  Returns ORC_OK or error. */
int32_t orc_sample_grad(const orc_arch* a, const double* params, const float* x, int32_t label,
                        double* grad_accum, double* loss);

/* orc_sample_grad with the forward pass at Pf and delta_in (W^T delta) at Pb (a
 * hogwild worker's reads may see different versions of the shared weights). */
int32_t orc_sample_grad2(const orc_arch* a, const double* Pf, const double* Pb, const float* x, int32_t label,
                         double* grad_accum, double* loss);

/* Sequential SGD over samples 0..n-1 in index order (P:132 with one worker;
 * P:324 no shuffling): W <- W - lr * g_i after every sample -- its own per-sample loop,
 * independent of orc_train_sync.  sum_loss may be NULL. */
int32_t orc_train_sgd(const orc_arch* a, double* params, const float* X, const int32_t* Y,
                      int64_t n, double lr, double* sum_loss);

/* Sync-batch SGD (BASELINE.json north_star "sums a fixed batch's gradients in a
 * fixed order before one update"): for each block [sB, min(sB+B,n)), every g_i at
 * the block-start W, G = sum in index order, W <- W - lr*G. */
int32_t orc_train_sync(const orc_arch* a, double* params, const float* X, const int32_t* Y,
                       int64_t n, double lr, int64_t batch, double* sum_loss);

/* Evaluation: mean cross-entropy (double, index-order sum) and the number
 * of samples whose argmax logit (lowest index on ties) differs from the label.
 * losses / preds (may be NULL) receive per-sample values. */
int32_t orc_evaluate(const orc_arch* a, const double* params, const float* X, const int32_t* Y,
                     int64_t n, double* mean_loss, int64_t* n_errors, double* losses, int32_t* preds);

/* One read of the shared weights by a hogwild group (see orc_replay). */
typedef struct {
    int32_t group;   /* reading group */
    int32_t layer;   /* weighted layer index (0-based, pools not counted) */
    int32_t purpose; /* 0: forward pass; 1: delta_in back-propagation */
    int32_t n_incl;  /* number of groups whose publish of this layer the read saw */
    int64_t e0, e1;  /* element range within the layer's normative W-then-b block */
    int64_t incl_off; /* their group ids: incl[incl_off .. incl_off + n_incl) */
} orc_read;

/* Hogwild schedule replay (C-1 step 9): group k = images [g_first[k], +g_count[k]),
 * each reading the weights as W0 + the publishes its reads name, publishing -lr * sum of its
 * images' gradients per layer.  params_out = W0 + sum of all publishes; pubs_out (may be NULL)
 * [n_groups][n_params]; pubs_in (may be NULL) replaces the replayed publishes the reads include. */
int32_t orc_replay(const orc_arch* a, const double* params0, const float* X, const int32_t* Y, int32_t n_groups,
                   const int64_t* g_first, const int32_t* g_count, int32_t n_reads, const orc_read* reads,
                   const int32_t* incl, double lr, double* params_out, double* pubs_out, const double* pubs_in);

#ifdef __cplusplus
}
#endif
#endif
