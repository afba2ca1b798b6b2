"""Shared test helpers: the parity tolerance of DESIGN.md (reading R9 / SURVEY C-15)."""
import itertools

import numpy as np


def split_blocks(vec, blocks):
    """Split a normative flat vector into per-tensor pieces [W0, b0, W1, b1, ...]."""
    out = []
    off = 0
    for _, nw, nb in blocks:
        out.append(vec[off:off + nw])
        out.append(vec[off + nw:off + nw + nb])
        off += nw + nb
    return out


def parity_report(got, ref, blocks, rel=1e-4, floor=1e-2, norm_rel=1e-5):
    """Per tensor T: |got-ref| <= rel*max(|ref|, floor*||ref||_inf) element-wise and
    ||got-ref||_2 <= norm_rel*||ref||_2.  Returns (ok, worst_ratio, worst_norm_ratio, details)."""
    ok = True
    worst = 0.0
    worst_norm = 0.0
    details = []
    for k, (g, r) in enumerate(zip(split_blocks(np.asarray(got, np.float64), blocks),
                                   split_blocks(np.asarray(ref, np.float64), blocks))):
        rmax = np.abs(r).max() if r.size else 0.0
        if rmax == 0.0:
            bad = np.abs(g).max() if g.size else 0.0
            ratio = 0.0 if bad == 0.0 else np.inf
            nr = 0.0 if bad == 0.0 else np.inf
        else:
            tol = rel * np.maximum(np.abs(r), floor * rmax)
            ratio = float(np.max(np.abs(g - r) / tol))
            nr = float(np.linalg.norm(g - r) / np.linalg.norm(r)) / norm_rel
        worst = max(worst, ratio)
        worst_norm = max(worst_norm, nr)
        details.append((k, ratio, nr))
        if ratio > 1.0 or nr > 1.0:
            ok = False
    return ok, worst, worst_norm, details


def assert_parity(got, ref, blocks, **kw):
    ok, w, wn, det = parity_report(got, ref, blocks, **kw)
    assert ok, f"parity failed: worst elementwise {w:.3g} x tol, worst norm {wn:.3g} x tol; per tensor {det}"
    return w, wn


def min_pool_gaps(arch, trace, in_c=1, in_h=29, in_w=29):
    """Smallest relative top-2 gap over the max-pool windows of each pool layer, from an
    oracle forward trace (every layer's output, in order).  A gap below ~1e-6 can flip the
    argmax between an fp32 and an fp64 run (R9, SURVEY C-15 near-tie excuse)."""
    c, h, w = in_c, in_h, in_w
    off = 0
    prev = None
    gaps = []
    for kind, units, kernel, _ in arch:
        if kind == 1:  # conv
            c, h, w = units, h - kernel + 1, w - kernel + 1
            prev = np.asarray(trace[off:off + c * h * w]).reshape(c, h, w)
            off += c * h * w
        elif kind == 2:  # pool
            k = kernel
            ph, pw = h // k, w // k
            win = prev[:, :ph * k, :pw * k].reshape(c, ph, k, pw, k).transpose(0, 1, 3, 2, 4).reshape(c, ph, pw, k * k)
            srt = np.sort(win, axis=-1)
            if k * k > 1:
                gaps.append(float(np.min((srt[..., -1] - srt[..., -2]) / np.maximum(np.abs(srt[..., -1]), 1e-30))))
            h, w = ph, pw
            off += c * h * w
        else:
            c, h, w = units, 1, 1
            off += units
    return gaps


def tie_free_prefix(oracle, arch, params, X, Y, lr, gap=5e-6):
    """Number of leading samples of the oracle's sequential-SGD trajectory before the first
    sample with a pool window whose top-2 relative gap is below `gap`."""
    p = np.asarray(params, np.float64).copy()
    for i in range(len(Y)):
        _, tr, _ = oracle.forward(p, X[i])
        if min(min_pool_gaps(arch, tr), default=1.0) < gap:
            return i
        p, _ = oracle.train_sgd(p, X[i:i + 1], Y[i:i + 1], lr)
    return len(Y)


def interval_orders(n):
    """All strict interval orders on n samples, as the set of predecessors of each sample.

    Enumerated as the distinct read-before-publish patterns of n workers: each sample i
    reads at time r_i and publishes at time w_i > r_i; j precedes i iff w_j < r_i."""
    pats = set()
    for perm in itertools.permutations(range(2 * n)):
        r = perm[:n]
        w = perm[n:]
        if any(w[i] < r[i] for i in range(n)):
            continue
        pats.add(tuple(frozenset(j for j in range(n) if w[j] < r[i]) for i in range(n)))
    return sorted(pats, key=str)


def compose_replay(o, p, X, Y, lr, preds):
    """Whole-sample hogwild outcome by composition (no orc_replay): sample i's gradient at
    W0 - lr * sum_{j in preds[i]} g_j, the final W = W0 - lr * sum of all gradients."""
    n = len(Y)
    order = sorted(range(n), key=lambda i: len(preds[i]))
    g = {}
    for i in order:
        w = np.asarray(p, np.float64).copy()
        for j in sorted(preds[i]):
            w -= lr * g[j]
        g[i] = o.sample_grad(w, X[i], Y[i])[1]
    return np.asarray(p, np.float64) - lr * sum(g[i] for i in range(n))
