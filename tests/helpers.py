"""Shared test helpers: the parity tolerance of DESIGN.md (reading R9 / SURVEY C-15), torch autograd
pins, hogwild schedule replay helpers."""
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


def parity_report(got, ref, blocks, rel=1e-4, floor=1e-2, norm_rel=1e-5, abs_floor=None):
    """Per tensor T: |got-ref| <= rel*max(|ref|, floor*||ref||_inf) element-wise and
    ||got-ref||_2 <= norm_rel*||ref||_2.  abs_floor (optional, per element, normative layout): an
    absolute tolerance added to both (reading R20: a weight update below one ulp of the weight it
    is applied to cannot change it).  Returns (ok, worst_ratio, worst_norm_ratio, details)."""
    ok = True
    worst = 0.0
    worst_norm = 0.0
    details = []
    afl = split_blocks(np.asarray(abs_floor, np.float64), blocks) if abs_floor is not None else None
    for k, (g, r) in enumerate(zip(split_blocks(np.asarray(got, np.float64), blocks),
                                   split_blocks(np.asarray(ref, np.float64), blocks))):
        rmax = np.abs(r).max() if r.size else 0.0
        a = afl[k] if afl is not None else np.zeros_like(r)
        if rmax == 0.0 and not a.any():
            bad = np.abs(g).max() if g.size else 0.0
            ratio = 0.0 if bad == 0.0 else np.inf
            nr = 0.0 if bad == 0.0 else np.inf
        else:
            tol = np.maximum(rel * np.maximum(np.abs(r), floor * rmax), a)
            ratio = float(np.max(np.abs(g - r) / tol))
            nr = float(np.linalg.norm(g - r) / (norm_rel * np.linalg.norm(r) + np.linalg.norm(a)))
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


def schedule_from_trace(rec, blocks, n, G):
    """The hogwild schedule a kTrace epoch recorded (chaos_debug_trace records, include/chaos.h)
    as orc_replay input.  Publish j of layer l was seen by a read iff its done rank < the read's
    begin count; not seen iff its started rank >= the read's end count; otherwise it overlapped
    the read (a torn read is possible: the group is `ambiguous`).
    Returns (groups [(first, count)], reads [(group, layer, purpose, e0, e1, seen)], ambiguous set)."""
    rec = np.asarray(rec)
    ng = rec.shape[0]
    nl = len(blocks)
    groups = [(k * G, min(G, n - k * G)) for k in range(ng)]
    start = rec[:, [6 * l for l in range(nl)]]
    done = rec[:, [6 * l + 1 for l in range(nl)]]
    if (start < 0).any() or (done < 0).any():
        raise AssertionError("trace: a group's publish was not recorded")
    # every publish got one rank on each counter
    if sorted(start.reshape(-1)) != list(range(ng * nl)) or sorted(done.reshape(-1)) != list(range(ng * nl)):
        raise AssertionError("trace: publish ranks are not a permutation")
    reads, amb = [], set()
    for k in range(ng):
        for l, (_, nw, nb) in enumerate(blocks):
            for p in (0, 1):
                d0, s1 = rec[k, 6 * l + 2 + 2 * p], rec[k, 6 * l + 3 + 2 * p]
                if p == 1 and d0 < 0 and s1 < 0:
                    continue  # delta_in reads the forward's copy
                if d0 < 0 or s1 < 0:
                    raise AssertionError(f"trace: group {k} layer {l} read {p} not recorded")
                others = [j for j in range(ng) if j != k]
                seen = [j for j in others if done[j, l] < d0]
                if any(not (done[j, l] < d0) and start[j, l] < s1 for j in others):
                    amb.add(k)
                if done[k, l] < d0:
                    raise AssertionError("trace: a group saw its own publish")
                reads.append((k, l, p, 0, nw + nb, seen))
    return groups, reads, amb


def check_read_values(rec, blocks, reads_rec, p0, pubs):
    """The weight values each group actually read (chaos_debug_trace host_reads) against the
    recorded schedule: per layer and read, W0 + the publishes it certainly saw (done before it
    began), plus any subset of the ones that overlapped it (torn), element by element within the
    fp32 rounding of the reduce-adds.  Catches reads of values no publish sequence produces
    (garbage, a group's own later publish, a lost or doubled publish)."""
    rec = np.asarray(rec)
    ng = rec.shape[0]
    p0 = np.asarray(p0, np.float64)
    starts = np.cumsum([0] + [nw + nb for _, nw, nb in blocks])
    worst = 0.0
    for l in range(len(blocks)):
        a, b = starts[l], starts[l + 1]
        start, done = rec[:, 6 * l], rec[:, 6 * l + 1]
        order = np.argsort(done)  # publishes of layer l in completion order
        pl = pubs[order, a:b].astype(np.float64)
        cum = np.vstack([np.zeros((1, b - a)), np.cumsum(pl, 0)])
        cabs = np.vstack([np.zeros((1, b - a)), np.cumsum(np.abs(pl), 0)])
        for k in range(ng):
            for pp in (0, 1):
                d0, s1 = rec[k, 6 * l + 2 + 2 * pp], rec[k, 6 * l + 3 + 2 * pp]
                vals = np.asarray(reads_rec[k, pp, a:b], np.float64)
                if np.all(np.isnan(vals)):
                    if pp == 1:
                        continue
                    raise AssertionError(f"group {k} layer {l}: no forward read recorded")
                if pp == 0 and np.any(np.isnan(vals)):
                    raise AssertionError(f"group {k} layer {l}: forward read partly recorded")
                used = ~np.isnan(vals)  # a delta_in read may skip the biases (not used by W^T delta)
                if d0 < 0:
                    d0, s1 = rec[k, 6 * l + 2], rec[k, 6 * l + 3]
                nseen = int(np.sum(done < d0))
                amb = [j for j in range(ng) if j != k and done[j] >= d0 and start[j] < s1]
                base = p0[a:b] + cum[nseen]
                lo = base + sum((np.minimum(pubs[j, a:b], 0.0) for j in amb), np.zeros(b - a))
                hi = base + sum((np.maximum(pubs[j, a:b], 0.0) for j in amb), np.zeros(b - a))
                bound = np.abs(p0[a:b]) + cabs[nseen] + sum((np.abs(pubs[j, a:b]) for j in amb), np.zeros(b - a))
                tol = (nseen + len(amb) + 1) * 2.0 ** -24 * bound + 1e-30
                excess = np.where(used, np.maximum(lo - vals, vals - hi), -np.inf)
                r = float(np.max(excess / tol))
                worst = max(worst, r)
                if r > 1.0:
                    e = int(np.argmax(excess / tol))
                    raise AssertionError(f"group {k} (worker {rec[k, 30]}) layer {l} read {pp}: value {vals[e]:.9g} "
                                         f"outside [{lo[e]:.9g}, {hi[e]:.9g}] +- {tol[e]:.3g} (saw {nseen} "
                                         f"publishes, {len(amb)} overlapping)")
    return worst



def assert_sum_of_publishes(final, p0, pub_sum, pub_abs_sum, n_adds, rigorous=True):
    """Every publish applied exactly once (no lost or doubled update): final - p0 == pub_sum up to
    the fp32 rounding of the n_adds reduce-adds into each weight.  Each add rounds its result,
    whose magnitude is at most |p0| + sum_k |pub_k| (= the bound B), by at most 2^-24 |result|:
    rigorous bound n_adds 2^-24 B; with rigorous=False a random-walk bound 8 sqrt(n_adds) 2^-24 B
    (many adds).  A lost or doubled group moves its weights by its whole publish, far above it."""
    final = np.asarray(final, np.float64)
    p0 = np.asarray(p0, np.float64)
    bound = np.abs(p0) + np.asarray(pub_abs_sum, np.float64)
    k = n_adds if rigorous else 8.0 * np.sqrt(n_adds)
    tol = k * 2.0 ** -24 * bound + 1e-30
    err = np.abs((final - p0) - pub_sum)
    worst = int(np.argmax(err / tol))
    assert np.all(err <= tol), (f"final - W0 != sum of publishes at element {worst}: {err[worst]:.3g} > tol "
                                f"{tol[worst]:.3g} (sum of publishes {pub_sum[worst]:.3g})")
    return float(np.max(err / tol))


C_, P_ = 1, 2  # layer kinds (synthdata.CONV / POOL)
T_ = 0  # tanh


def torch_grad(arch, params, X, Y, params_bwd=None, dtype=None):
    """Sum-reduction CE gradient (float64 unless dtype) with torch's own conv2d/max_pool2d/linear/cross_entropy.

    params_bwd (optional): the weights the back-propagated partial derivatives use (delta_in =
    W_bwd^T delta), while the forward pass and the weight gradients use params -- built as
    layer(x.detach(), W) + layer(x, W_bwd) - layer(x, W_bwd).detach(): the value is layer(x, W),
    d/dW flows through the first term only, d/dx through the second only."""
    import torch
    import torch.nn.functional as F
    dt = torch.float64 if dtype is None else dtype
    P = torch.tensor(np.asarray(params), dtype=dt, requires_grad=True)
    Pb = None if params_bwd is None else torch.tensor(np.asarray(params_bwd), dtype=dt)
    x = torch.tensor(np.asarray(X, np.float64)).to(dt).reshape(len(Y), 1, 29, 29)

    def split(fn, h, W, b, Wb_, bb_):
        if Pb is None:
            return fn(h, W, b)
        return fn(h.detach(), W, b) + fn(h, Wb_, bb_) - fn(h, Wb_, bb_).detach()

    off = 0
    h = x
    c = 1
    for kind, units, k, act in arch:
        if kind == C_:
            nw = units * c * k * k
            W = P[off:off + nw].reshape(units, c, k, k)
            b = P[off + nw:off + nw + units]
            Wb_ = None if Pb is None else Pb[off:off + nw].reshape(units, c, k, k)
            bb_ = None if Pb is None else Pb[off + nw:off + nw + units]
            off += nw + units
            h = split(F.conv2d, h, W, b, Wb_, bb_)
            h = torch.tanh(h) if act == T_ else h
            c = units
        elif kind == P_:
            h = F.max_pool2d(h, k, stride=k, ceil_mode=False)
        else:
            h = h.reshape(h.shape[0], -1)
            nin = h.shape[1]
            W = P[off:off + units * nin].reshape(units, nin)
            b = P[off + units * nin:off + units * nin + units]
            Wb_ = None if Pb is None else Pb[off:off + units * nin].reshape(units, nin)
            bb_ = None if Pb is None else Pb[off + units * nin:off + units * nin + units]
            off += units * nin + units
            h = split(F.linear, h, W, b, Wb_, bb_)
            h = torch.tanh(h) if act == T_ else h
    loss = F.cross_entropy(h, torch.tensor(np.asarray(Y, np.int64)), reduction="sum")
    loss.backward()
    return loss.item(), P.grad.numpy().astype(np.float64), h.detach().numpy()


