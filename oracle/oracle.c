/*
 * oracle.c -- plain, slow, single-threaded CPU reference of the CHAOS hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Built with
 *   gcc -O2 -ffp-contract=off -fPIC -shared  (no -ffast-math, no OpenMP, no intrinsics)
 * so every sum below is evaluated exactly in the order written.
 *
 * What it follows, step by step:
 *  - forward  x^l_i = sum_j w_ji y^{l-1}_j (+ bias), y = sigma(x)        PAPER.md:73 (§II-A)
 *    with sigma = tanh (BASELINE.json configs[*]) and logits un-squashed;
 *    convolution = valid cross-correlation, stride 1, every output map fully
 *    connected to all input maps (forced by Table I weight counts);
 *    max-pool non-overlapping, floor, first strict maximum in row-major order.
 *  - output error and back-propagated partial derivatives delta
 *    with softmax cross-entropy (reading R3).
 *  - update  W <- W - lr * g  ("decay" lambda read as the per-epoch lr factor,
 *    applied by the caller; reading R6)
 *  - Training = each (single) worker takes the next unprocessed image
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int kind, act;
    int ic, ih, iw;     /* input maps / height / width */
    int oc, oh, ow;     /* output maps / height / width */
    int k;              /* conv kernel or pool window */
    int64_t woff, boff; /* parameter offsets (weighted layers) */
    int64_t fan_in, nw, nb;
    int64_t in_off, out_off; /* offsets of this layer's input / output in the activation arena */
    int64_t am_off;          /* pool: offset into the argmax arena */
} plan_layer;

typedef struct {
    int n;
    plan_layer L[16];
    int64_t n_params;
    int64_t arena; /* doubles: input image + every layer output */
    int64_t am_len;
    int n_classes;
} plan;

static void set_err(char* err, int32_t errlen, const char* msg) {
    if (err && errlen > 0) {
        snprintf(err, (size_t)errlen, "%s", msg);
    }
}

/* Shape chain: conv o = h-k+1; pool o = floor(h/kp). */
static int make_plan(const orc_arch* a, plan* p, char* err, int32_t errlen) {
    char msg[256];
    if (!a || a->n_layers < 1 || a->n_layers > 16 || a->in_c < 1 || a->in_h < 1 || a->in_w < 1 ||
        a->n_classes < 1) {
        set_err(err, errlen, "invalid arch header");
        return ORC_E_INVALID;
    }
    memset(p, 0, sizeof(*p));
    p->n = a->n_layers;
    p->n_classes = a->n_classes;
    int c = a->in_c, h = a->in_h, w = a->in_w;
    int64_t poff = 0;
    int64_t aoff = (int64_t)c * h * w; /* arena starts with the input image */
    int64_t amoff = 0;
    for (int l = 0; l < a->n_layers; ++l) {
        const orc_layer* s = &a->layers[l];
        plan_layer* q = &p->L[l];
        q->kind = s->kind;
        q->act = s->act;
        q->ic = c;
        q->ih = h;
        q->iw = w;
        q->k = s->kernel;
        q->in_off = (l == 0) ? 0 : p->L[l - 1].out_off;
        if (s->kind == ORC_CONV) {
            if (s->units < 1 || s->kernel < 1 || s->kernel > h || s->kernel > w) {
                snprintf(msg, sizeof msg, "layer %d (conv k=%d): input %dx%d < kernel or bad units", l,
                         s->kernel, h, w);
                set_err(err, errlen, msg);
                return ORC_E_ARCH;
            }
            q->oc = s->units;
            q->oh = h - s->kernel + 1;
            q->ow = w - s->kernel + 1;
            q->fan_in = (int64_t)c * s->kernel * s->kernel;
            q->nw = (int64_t)q->oc * q->fan_in;
            q->nb = q->oc;
        } else if (s->kind == ORC_POOL) {
            if (s->kernel < 1 || s->kernel > h || s->kernel > w) {
                snprintf(msg, sizeof msg, "layer %d (pool k=%d): input %dx%d < window", l, s->kernel, h, w);
                set_err(err, errlen, msg);
                return ORC_E_ARCH;
            }
            q->oc = c;
            q->oh = h / s->kernel;
            q->ow = w / s->kernel;
            q->am_off = amoff;
            amoff += (int64_t)q->oc * q->oh * q->ow;
        } else if (s->kind == ORC_FULL) {
            if (s->units < 1) {
                snprintf(msg, sizeof msg, "layer %d (full): units < 1", l);
                set_err(err, errlen, msg);
                return ORC_E_ARCH;
            }
            q->oc = s->units;
            q->oh = 1;
            q->ow = 1;
            q->fan_in = (int64_t)c * h * w;
            q->nw = (int64_t)q->oc * q->fan_in;
            q->nb = q->oc;
        } else {
            snprintf(msg, sizeof msg, "layer %d: unknown kind %d", l, s->kind);
            set_err(err, errlen, msg);
            return ORC_E_ARCH;
        }
        if (s->kind != ORC_POOL) {
            q->woff = poff;
            q->boff = poff + q->nw;
            poff += q->nw + q->nb;
        }
        q->out_off = aoff;
        aoff += (int64_t)q->oc * q->oh * q->ow;
        c = q->oc;
        h = q->oh;
        w = q->ow;
    }
    const plan_layer* last = &p->L[p->n - 1];
    if (last->kind != ORC_FULL || last->oc != a->n_classes || last->act != ORC_IDENT) {
        set_err(err, errlen, "last layer must be FULL with n_classes units and identity activation");
        return ORC_E_ARCH;
    }
    p->n_params = poff;
    p->arena = aoff;
    p->am_len = amoff;
    return ORC_OK;
}

int64_t orc_num_params(const orc_arch* a, char* err, int32_t errlen) {
    plan p;
    int rc = make_plan(a, &p, err, errlen);
    return rc ? rc : p.n_params;
}

int32_t orc_blocks(const orc_arch* a, int64_t* out, int32_t max_layers) {
    plan p;
    if (make_plan(a, &p, NULL, 0)) return ORC_E_ARCH;
    int nl = 0;
    for (int l = 0; l < p.n; ++l) {
        if (p.L[l].kind == ORC_POOL) continue;
        if (nl < max_layers) {
            out[3 * nl + 0] = p.L[l].fan_in;
            out[3 * nl + 1] = p.L[l].nw;
            out[3 * nl + 2] = p.L[l].nb;
        }
        ++nl;
    }
    return nl;
}

int64_t orc_trace_len(const orc_arch* a) {
    plan p;
    if (make_plan(a, &p, NULL, 0)) return ORC_E_ARCH;
    return p.arena - (int64_t)a->in_c * a->in_h * a->in_w;
}

static double act_fn(int act, double z) { return act == ORC_TANH ? tanh(z) : z; }

/* Forward pass into the activation arena (arena[0..C*H*W) = the image). */
static void forward_plan(const plan* p, const double* P, double* A, uint8_t* AM) {
    for (int l = 0; l < p->n; ++l) {
        const plan_layer* q = &p->L[l];
        const double* in = A + q->in_off;
        double* out = A + q->out_off;
        if (q->kind == ORC_CONV) {
            /* z[m][r][c] = b[m] + sum_n sum_i sum_j W[m][n][i][j] * in[n][r+i][c+j] */
            const double* W = P + q->woff;
            const double* b = P + q->boff;
            for (int m = 0; m < q->oc; ++m)
                for (int r = 0; r < q->oh; ++r)
                    for (int c = 0; c < q->ow; ++c) {
                        double z = b[m];
                        for (int n = 0; n < q->ic; ++n)
                            for (int i = 0; i < q->k; ++i)
                                for (int j = 0; j < q->k; ++j)
                                    z += W[(((int64_t)m * q->ic + n) * q->k + i) * q->k + j] *
                                         in[((int64_t)n * q->ih + r + i) * q->iw + c + j];
                        out[((int64_t)m * q->oh + r) * q->ow + c] = act_fn(q->act, z);
                    }
        } else if (q->kind == ORC_POOL) {
            /* non-overlapping kp x kp max, floor; first strict maximum wins (C-14) */
            uint8_t* am = AM + q->am_off;
            for (int m = 0; m < q->oc; ++m)
                for (int pr = 0; pr < q->oh; ++pr)
                    for (int pc = 0; pc < q->ow; ++pc) {
                        double best = in[((int64_t)m * q->ih + pr * q->k) * q->iw + pc * q->k];
                        int arg = 0;
                        for (int u = 0; u < q->k; ++u)
                            for (int v = 0; v < q->k; ++v) {
                                double y = in[((int64_t)m * q->ih + pr * q->k + u) * q->iw + pc * q->k + v];
                                if (y > best) {
                                    best = y;
                                    arg = u * q->k + v;
                                }
                            }
                        out[((int64_t)m * q->oh + pr) * q->ow + pc] = best;
                        am[((int64_t)m * q->oh + pr) * q->ow + pc] = (uint8_t)arg;
                    }
        } else {
            /* z[o] = b[o] + sum_i W[o][i] * in[i] */
            const double* W = P + q->woff;
            const double* b = P + q->boff;
            const int64_t nin = (int64_t)q->ic * q->ih * q->iw;
            for (int o = 0; o < q->oc; ++o) {
                double z = b[o];
                for (int64_t i = 0; i < nin; ++i) z += W[o * nin + i] * in[i];
                out[o] = act_fn(q->act, z);
            }
        }
    }
}

typedef struct {
    plan p;
    double* A;    /* activations */
    double* D;    /* deltas, same layout as A */
    uint8_t* AM;  /* pool argmax */
} work;

static int work_init(work* w, const orc_arch* a) {
    memset(w, 0, sizeof(*w));
    int rc = make_plan(a, &w->p, NULL, 0);
    if (rc) return rc;
    w->A = (double*)calloc((size_t)w->p.arena, sizeof(double));
    w->D = (double*)calloc((size_t)w->p.arena, sizeof(double));
    w->AM = (uint8_t*)calloc((size_t)(w->p.am_len > 0 ? w->p.am_len : 1), 1);
    if (!w->A || !w->D || !w->AM) return ORC_E_INVALID;
    return ORC_OK;
}

static void work_free(work* w) {
    free(w->A);
    free(w->D);
    free(w->AM);
}

static void load_image(const plan* p, double* A, const float* x, int64_t n_in) {
    (void)p;
    for (int64_t i = 0; i < n_in; ++i) A[i] = (double)x[i];
}

/* Softmax cross-entropy on the logits z (reading R3):
 * L = log sum_o exp(z_o - z_max) + z_max - z_label;  p = softmax(z). */
static double softmax_ce(const double* z, int nc, int label, double* prob) {
    double zmax = z[0];
    for (int o = 1; o < nc; ++o)
        if (z[o] > zmax) zmax = z[o];
    double s = 0.0;
    for (int o = 0; o < nc; ++o) s += exp(z[o] - zmax);
    if (prob)
        for (int o = 0; o < nc; ++o) prob[o] = exp(z[o] - zmax) / s;
    return log(s) + zmax - z[label];
}

/* Back-propagation for the sample whose forward pass is in w->A.
 * G[j] += dL/dparam_j. */
static void backward_plan(work* w, const double* P, int label, double* G) {
    const plan* p = &w->p;
    double* A = w->A;
    double* D = w->D;
    memset(D, 0, sizeof(double) * (size_t)p->arena);
    const plan_layer* last = &p->L[p->n - 1];
    /* output partial derivatives delta_out = softmax(z) - onehot(label) */
    double* dz = D + last->out_off;
    softmax_ce(A + last->out_off, p->n_classes, label, dz);
    dz[label] -= 1.0;

    for (int l = p->n - 1; l >= 0; --l) {
        const plan_layer* q = &p->L[l];
        const double* in = A + q->in_off;
        const double* y = A + q->out_off;
        double* dy = D + q->out_off; /* dL/d(output of layer l) */
        double* din = (l > 0) ? D + q->in_off : NULL; /* not needed for the image */
        const int64_t nout = (int64_t)q->oc * q->oh * q->ow;
        if (q->kind == ORC_POOL) {
            /* route each pooled delta to its argmax only; all else 0 */
            const uint8_t* am = w->AM + q->am_off;
            if (!din) continue;
            for (int m = 0; m < q->oc; ++m)
                for (int pr = 0; pr < q->oh; ++pr)
                    for (int pc = 0; pc < q->ow; ++pc) {
                        int64_t o = ((int64_t)m * q->oh + pr) * q->ow + pc;
                        int u = am[o] / q->k, v = am[o] % q->k;
                        din[((int64_t)m * q->ih + pr * q->k + u) * q->iw + pc * q->k + v] += dy[o];
                    }
            continue;
        }
        /* through the activation: dz = dy * (1 - y^2) for tanh, dy for identity */
        for (int64_t o = 0; o < nout; ++o)
            if (q->act == ORC_TANH) dy[o] = dy[o] * (1.0 - y[o] * y[o]);
        const double* W = P + q->woff;
        double* gW = G + q->woff;
        double* gb = G + q->boff;
        if (q->kind == ORC_FULL) {
            const int64_t nin = (int64_t)q->ic * q->ih * q->iw;
            for (int o = 0; o < q->oc; ++o) {
                gb[o] += dy[o];
                for (int64_t i = 0; i < nin; ++i) gW[o * nin + i] += dy[o] * in[i];
            }
            if (din)
                for (int64_t i = 0; i < nin; ++i) {
                    double s = 0.0;
                    for (int o = 0; o < q->oc; ++o) s += W[o * nin + i] * dy[o];
                    din[i] += s;
                }
        } else { /* ORC_CONV */
            for (int m = 0; m < q->oc; ++m)
                for (int r = 0; r < q->oh; ++r)
                    for (int c = 0; c < q->ow; ++c) {
                        const double d = dy[((int64_t)m * q->oh + r) * q->ow + c];
                        if (d == 0.0) continue; /* exact: a zero term adds nothing */
                        gb[m] += d;
                        for (int n = 0; n < q->ic; ++n)
                            for (int i = 0; i < q->k; ++i)
                                for (int j = 0; j < q->k; ++j) {
                                    const int64_t wi = (((int64_t)m * q->ic + n) * q->k + i) * q->k + j;
                                    const int64_t xi = ((int64_t)n * q->ih + r + i) * q->iw + c + j;
                                    gW[wi] += d * in[xi];
                                    if (din) din[xi] += W[wi] * d;
                                }
                    }
        }
    }
}

int32_t orc_forward(const orc_arch* a, const double* params, const float* x, double* logits, double* trace,
                    uint8_t* argmax) {
    if (!a || !params || !x) return ORC_E_INVALID;
    work w;
    int rc = work_init(&w, a);
    if (rc) {
        work_free(&w);
        return rc;
    }
    const int64_t n_in = (int64_t)a->in_c * a->in_h * a->in_w;
    load_image(&w.p, w.A, x, n_in);
    forward_plan(&w.p, params, w.A, w.AM);
    const plan_layer* last = &w.p.L[w.p.n - 1];
    if (logits) memcpy(logits, w.A + last->out_off, sizeof(double) * (size_t)a->n_classes);
    if (trace) memcpy(trace, w.A + n_in, sizeof(double) * (size_t)(w.p.arena - n_in));
    if (argmax && w.p.am_len) memcpy(argmax, w.AM, (size_t)w.p.am_len);
    work_free(&w);
    return ORC_OK;
}

static int grad_one(work* w, const double* P, const float* x, int label, double* G, double* loss, int64_t n_in) {
    if (label < 0 || label >= w->p.n_classes) return ORC_E_LABEL;
    load_image(&w->p, w->A, x, n_in);
    forward_plan(&w->p, P, w->A, w->AM);
    const plan_layer* last = &w->p.L[w->p.n - 1];
    if (loss) *loss = softmax_ce(w->A + last->out_off, w->p.n_classes, label, NULL);
    backward_plan(w, P, label, G);
    return ORC_OK;
}

/* One sample's gradient with the forward pass at Pf and the back-propagated partial derivatives
 * (delta_in = W^T delta) at Pb: the two weight reads a hogwild worker makes may see different
 * versions of the shared weights ("on-demand" reads).  Pf == Pb is orc_sample_grad. */
int32_t orc_sample_grad2(const orc_arch* a, const double* Pf, const double* Pb, const float* x, int32_t label,
                         double* grad_accum, double* loss) {
    if (!a || !Pf || !Pb || !x || !grad_accum) return ORC_E_INVALID;
    work w;
    int rc = work_init(&w, a);
    if (!rc) {
        if (label < 0 || label >= w.p.n_classes) {
            rc = ORC_E_LABEL;
        } else {
            const int64_t n_in = (int64_t)a->in_c * a->in_h * a->in_w;
            load_image(&w.p, w.A, x, n_in);
            forward_plan(&w.p, Pf, w.A, w.AM);
            const plan_layer* last = &w.p.L[w.p.n - 1];
            if (loss) *loss = softmax_ce(w.A + last->out_off, w.p.n_classes, label, NULL);
            backward_plan(&w, Pb, label, grad_accum);
        }
    }
    work_free(&w);
    return rc;
}

int32_t orc_sample_grad(const orc_arch* a, const double* params, const float* x, int32_t label,
                        double* grad_accum, double* loss) {
    if (!a || !params || !x || !grad_accum) return ORC_E_INVALID;
    work w;
    int rc = work_init(&w, a);
    if (!rc) rc = grad_one(&w, params, x, label, grad_accum, loss, (int64_t)a->in_c * a->in_h * a->in_w);
    work_free(&w);
    return rc;
}

/* Sequential SGD, its own loop (not orc_train_sync with B = 1): for each sample i in index order
 * (no shuffling), the gradient at the current W, then W <- W - lr * g_i right away (P:132
 * with a single worker: it takes the next image, forward, back-propagate, adjust the weights). */
int32_t orc_train_sgd(const orc_arch* a, double* params, const float* X, const int32_t* Y, int64_t n, double lr,
                      double* sum_loss) {
    if (!a || !params || n < 0 || (n > 0 && (!X || !Y))) return ORC_E_INVALID;
    work w;
    int rc = work_init(&w, a);
    if (rc) {
        work_free(&w);
        return rc;
    }
    const int64_t np = w.p.n_params;
    const int64_t n_in = (int64_t)a->in_c * a->in_h * a->in_w;
    double* g = (double*)calloc((size_t)np, sizeof(double));
    double ls = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double li = 0.0;
        memset(g, 0, sizeof(double) * (size_t)np);
        rc = grad_one(&w, params, X + i * n_in, Y[i], g, &li, n_in);
        if (rc) break;
        ls += li;
        for (int64_t j = 0; j < np; ++j) params[j] -= lr * g[j]; /* adjust before the next image */
    }
    if (sum_loss) *sum_loss = ls;
    free(g);
    work_free(&w);
    return rc;
}

int32_t orc_train_sync(const orc_arch* a, double* params, const float* X, const int32_t* Y, int64_t n, double lr,
                       int64_t batch, double* sum_loss) {
    if (!a || !params || n < 0 || batch < 1 || (n > 0 && (!X || !Y))) return ORC_E_INVALID;
    work w;
    int rc = work_init(&w, a);
    if (rc) {
        work_free(&w);
        return rc;
    }
    const int64_t np = w.p.n_params;
    const int64_t n_in = (int64_t)a->in_c * a->in_h * a->in_w;
    double* g = (double*)calloc((size_t)np, sizeof(double));
    double* Gs = (double*)calloc((size_t)np, sizeof(double));
    double ls = 0.0;
    for (int64_t s0 = 0; s0 < n && !rc; s0 += batch) {
        const int64_t s1 = (s0 + batch < n) ? s0 + batch : n;
        memset(Gs, 0, sizeof(double) * (size_t)np);
        for (int64_t i = s0; i < s1 && !rc; ++i) { /* every g_i at the block-start W */
            double li = 0.0;
            memset(g, 0, sizeof(double) * (size_t)np);
            rc = grad_one(&w, params, X + i * n_in, Y[i], g, &li, n_in);
            for (int64_t j = 0; j < np; ++j) Gs[j] += g[j]; /* G = sum in index order */
            ls += li;
        }
        if (rc) break;
        for (int64_t j = 0; j < np; ++j) params[j] -= lr * Gs[j]; /* W <- W - lr*G */
    }
    if (sum_loss) *sum_loss = ls;
    free(g);
    free(Gs);
    work_free(&w);
    return rc;
}

int32_t orc_evaluate(const orc_arch* a, const double* params, const float* X, const int32_t* Y, int64_t n,
                     double* mean_loss, int64_t* n_errors, double* losses, int32_t* preds) {
    if (!a || !params || n < 0 || (n > 0 && (!X || !Y))) return ORC_E_INVALID;
    work w;
    int rc = work_init(&w, a);
    if (rc) {
        work_free(&w);
        return rc;
    }
    const int64_t n_in = (int64_t)a->in_c * a->in_h * a->in_w;
    const plan_layer* last = &w.p.L[w.p.n - 1];
    double total = 0.0;
    int64_t errs = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (Y[i] < 0 || Y[i] >= a->n_classes) {
            rc = ORC_E_LABEL;
            break;
        }
        load_image(&w.p, w.A, X + i * n_in, n_in);
        forward_plan(&w.p, params, w.A, w.AM);
        const double* z = w.A + last->out_off;
        const double li = softmax_ce(z, a->n_classes, Y[i], NULL);
        int best = 0; /* argmax, lowest index on ties */
        for (int o = 1; o < a->n_classes; ++o)
            if (z[o] > z[best]) best = o;
        total += li;
        errs += (best != Y[i]);
        if (losses) losses[i] = li;
        if (preds) preds[i] = best;
    }
    if (mean_loss) *mean_loss = n > 0 ? total / (double)n : 0.0;
    if (n_errors) *n_errors = errs;
    work_free(&w);
    return rc;
}

/* Hogwild schedule replay (PAPER.md:138 controlled hogwild, P:140
 * arbitrary order of synchronization).  Group k (a worker's claim of images
 * [g_first[k], g_first[k] + g_count[k])) reads the shared weights and publishes, per weighted
 * layer, pub_k = -lr * sum over its images of that layer's gradient.  A read (orc_read) states
 * which earlier groups' publishes of that layer the worker saw on the elements [e0, e1) of the
 * layer's normative W-then-b block, for the forward pass (purpose 0) or for the delta_in
 * back-propagation (purpose 1).  Elements no read covers are read at W0 (purpose 1 falls back to
 * the purpose-0 read of the same element).  Groups are evaluated in an order where every group
 * follows the groups it saw (ORC_E_INVALID if the sets are cyclic or self-referencing).
 * Result: params_out = W0 + sum_k pub_k (sum in group index order); pubs_out (may be NULL):
 * [n_groups][n_params] the publishes.  pubs_in (may be NULL): use these publishes for what the
 * reads include instead of the replayed ones (checks one group at a time against recorded data). */
int32_t orc_replay(const orc_arch* a, const double* params0, const float* X, const int32_t* Y, int32_t n_groups,
                   const int64_t* g_first, const int32_t* g_count, int32_t n_reads, const orc_read* reads,
                   const int32_t* incl, double lr, double* params_out, double* pubs_out, const double* pubs_in) {
    if (!a || !params0 || n_groups < 0 || (n_groups > 0 && (!g_first || !g_count || !X || !Y)) ||
        (n_reads > 0 && (!reads || !incl)) || !params_out)
        return ORC_E_INVALID;
    plan p;
    int rc = make_plan(a, &p, NULL, 0);
    if (rc) return rc;
    const int64_t np = p.n_params;
    const int64_t n_in = (int64_t)a->in_c * a->in_h * a->in_w;
    /* weighted-layer blocks: [start, end) in the normative layout */
    int64_t bstart[16], bend[16];
    int nl = 0;
    for (int l = 0; l < p.n; ++l)
        if (p.L[l].kind != ORC_POOL) {
            bstart[nl] = p.L[l].woff;
            bend[nl] = p.L[l].boff + p.L[l].nb;
            ++nl;
        }
    for (int r = 0; r < n_reads; ++r) {
        const orc_read* q = &reads[r];
        if (q->group < 0 || q->group >= n_groups || q->layer < 0 || q->layer >= nl || q->purpose < 0 ||
            q->purpose > 1 || q->e0 < 0 || q->e1 < q->e0 || bstart[q->layer] + q->e1 > bend[q->layer] ||
            q->n_incl < 0)
            return ORC_E_INVALID;
        for (int32_t t = 0; t < q->n_incl; ++t)
            if (incl[q->incl_off + t] < 0 || incl[q->incl_off + t] >= n_groups || incl[q->incl_off + t] == q->group)
                return ORC_E_INVALID;
    }
    double* pubs = (double*)calloc((size_t)(n_groups > 0 ? n_groups : 1) * (size_t)np, sizeof(double));
    double* Wf = (double*)malloc(sizeof(double) * (size_t)np);
    double* Wb = (double*)malloc(sizeof(double) * (size_t)np);
    double* g = (double*)malloc(sizeof(double) * (size_t)np);
    char* done = (char*)calloc((size_t)(n_groups > 0 ? n_groups : 1), 1);
    char* covf = (char*)malloc((size_t)np);
    char* covb = (char*)malloc((size_t)np);
    if (!pubs || !Wf || !Wb || !g || !done || !covf || !covb) rc = ORC_E_INVALID;
    int32_t n_done = 0;
    while (!rc && n_done < n_groups) {
        int progressed = 0;
        for (int32_t k = 0; k < n_groups && !rc; ++k) {
            if (done[k]) continue;
            int ready = 1; /* every group this one saw is evaluated */
            for (int r = 0; r < n_reads && ready; ++r)
                if (reads[r].group == k)
                    for (int32_t t = 0; t < reads[r].n_incl; ++t)
                        if (!done[incl[reads[r].incl_off + t]]) ready = 0;
            if (!ready) continue;
            /* the weights this group read: W0 + the publishes it saw, element by element */
            memcpy(Wf, params0, sizeof(double) * (size_t)np);
            memcpy(Wb, params0, sizeof(double) * (size_t)np);
            memset(covf, 0, (size_t)np);
            memset(covb, 0, (size_t)np);
            for (int r = 0; r < n_reads; ++r) {
                const orc_read* q = &reads[r];
                if (q->group != k) continue;
                double* W = q->purpose == 0 ? Wf : Wb;
                char* cov = q->purpose == 0 ? covf : covb;
                for (int64_t e = bstart[q->layer] + q->e0; e < bstart[q->layer] + q->e1; ++e) {
                    if (cov[e]) { /* two reads of one element for one purpose: ambiguous */
                        rc = ORC_E_INVALID;
                        break;
                    }
                    cov[e] = 1;
                    double v = params0[e];
                    for (int32_t t = 0; t < q->n_incl; ++t) {
                        const int32_t j = incl[q->incl_off + t];
                        v += (pubs_in ? pubs_in : pubs)[(int64_t)j * np + e];
                    }
                    W[e] = v;
                }
            }
            for (int64_t e = 0; e < np; ++e)
                if (!covb[e]) Wb[e] = Wf[e]; /* delta_in reads default to the forward read */
            /* pub_k = -lr * sum over the group's images of the gradient (index order) */
            memset(g, 0, sizeof(double) * (size_t)np);
            for (int32_t i = 0; i < g_count[k] && !rc; ++i) {
                const int64_t s = g_first[k] + i;
                rc = orc_sample_grad2(a, Wf, Wb, X + s * n_in, Y[s], g, NULL);
            }
            for (int64_t e = 0; e < np; ++e) pubs[(int64_t)k * np + e] = -lr * g[e];
            done[k] = 1;
            ++n_done;
            progressed = 1;
        }
        if (!progressed && !rc) rc = ORC_E_INVALID; /* a cycle: no group can go first */
    }
    if (!rc) {
        memcpy(params_out, params0, sizeof(double) * (size_t)np);
        for (int32_t k = 0; k < n_groups; ++k)
            for (int64_t e = 0; e < np; ++e) params_out[e] += pubs[(int64_t)k * np + e];
        if (pubs_out) memcpy(pubs_out, pubs, sizeof(double) * (size_t)n_groups * (size_t)np);
    }
    free(pubs);
    free(Wf);
    free(Wb);
    free(g);
    free(done);
    free(covf);
    free(covb);
    return rc;
}
