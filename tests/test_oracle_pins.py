"""Pins of the CPU oracle against things other than itself (CPU only, -m "not gpu").

Each test names what pins it: a value printed in the paper (Table I), a
hand-worked example, a library routine (torch float64
autograd: conv2d / max_pool2d / linear / cross_entropy), finite differences,
closed forms, invariants, or brute force on tiny inputs.
"""
import json
import math
import os

import numpy as np
import pytest

import synthdata as sd
from oracle import Oracle, OracleError

GOLD = os.path.join(os.path.dirname(__file__), "golden")
C_, P_, F_ = sd.CONV, sd.POOL, sd.FULL
T_, I_ = sd.TANH, sd.IDENT


# --------------------------------------------------------------------------------------
# Table I: weight counts and neuron counts, printed values
# --------------------------------------------------------------------------------------
TABLE_I = {
    # per weighted layer weights (Weights column) and per layer neurons (Neurons column)
    "paper_small": ([85, 1260, 4550, 510], [3380, 845, 810, 90, 50, 10]),
    "paper_medium": ([340, 20040, 54150, 1510], [13520, 3380, 3240, 360, 150, 10]),
    "paper_large": ([340, 30060, 216100, 135150, 1510],
                    [13520, 13520, 29040, 7260, 3600, 900, 150, 10]),
}


@pytest.mark.parametrize("name", sorted(TABLE_I))
def test_table1_weights_and_neurons(name):
    arch = sd.ARCHS["medium" if name == "paper_medium" else name]
    o = Oracle(arch)
    weights, neurons = TABLE_I[name]
    assert [nw + nb for (_, nw, nb) in o.blocks()] == weights
    assert o.n_params == sum(weights)
    # the forward trace holds every layer's output: its length is the Neurons column sum,
    # and per-layer lengths come out of the trace split
    assert len(o.forward(np.zeros(o.n_params), np.zeros(841, np.float32))[1]) == sum(neurons)


def test_bj_param_counts():
    # BASELINE.json configs[0..3] nets with the Table I "+1" formula
    assert Oracle(sd.ARCHS["tiny"]).n_params == 8545
    assert Oracle(sd.ARCHS["medium"]).n_params == 76040
    assert Oracle(sd.ARCHS["large"]).n_params == 96960


def test_arch_rejected():
    with pytest.raises(OracleError, match="kernel"):
        Oracle([(C_, 4, 30, T_), (F_, 10, 0, I_)])
    with pytest.raises(OracleError):
        Oracle([(C_, 4, 3, T_), (F_, 10, 0, T_)])  # logits must be identity


# --------------------------------------------------------------------------------------
# Appendix A hand-worked examples (tests/golden/appendix_a.json)
# --------------------------------------------------------------------------------------
HAND_ARCH = [(C_, 1, 2, T_), (P_, 0, 2, T_), (F_, 2, 0, I_)]


@pytest.mark.parametrize("ex", ["A", "B"])
def test_appendix_a(ex):
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    e = g[ex]
    o = Oracle(HAND_ARCH, in_h=4, in_w=4, n_classes=2)
    p0 = np.array(g["params0"])
    x = np.array(e["x"], np.float32).reshape(-1)
    logits, trace, am = o.forward(p0, x)
    np.testing.assert_allclose(logits, e["logits"], atol=1e-9)
    # trace = conv 3x3 (9) + pooled 1x1 (1) + logits (2)
    assert trace[9] == pytest.approx(e["pool_value"], abs=1e-9)
    assert int(am[0]) == e["argmax"]
    loss, grad = o.sample_grad(p0, x, g["label"])
    assert loss == pytest.approx(e["loss"], abs=1e-9)
    np.testing.assert_allclose(grad, e["grad"], atol=1e-9)
    p1, _ = o.train_sgd(p0, x[None], np.array([g["label"]]), g["lr"])
    np.testing.assert_allclose(p1, e["params1"], atol=1e-9)


def test_appendix_a_closed_form_values():
    # the hand values themselves, from closed forms: tanh(0.5), softmax of (+t, -t)
    t = math.tanh(0.5)
    assert t == pytest.approx(0.4621171573, abs=1e-10)
    p0 = 1.0 / (1.0 + math.exp(-2 * t))
    assert p0 == pytest.approx(0.7159040903, abs=1e-10)
    assert -math.log(1.0 - p0) == pytest.approx(1.2584433876, abs=1e-9)


# --------------------------------------------------------------------------------------
# Closed forms: zero-weight net
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "medium", "large", "paper_large"])
def test_zero_weights(name):
    o = Oracle(sd.ARCHS[name])
    x = sd.uniform_dataset(5, 1, 0).x_train[0]
    loss, g = o.sample_grad(np.zeros(o.n_params), x, 3)
    assert loss == pytest.approx(math.log(10.0), abs=1e-12)
    gb = g[-10:]
    expect = np.full(10, 0.1)
    expect[3] -= 1.0
    np.testing.assert_allclose(gb, expect, atol=1e-15)
    assert np.count_nonzero(g[:-10]) == 0  # every other gradient is exactly 0


def test_identity_conv_passes_input():
    # 1x1 kernel, weight 1, bias 0, identity activation => output = input
    o = Oracle([(C_, 1, 1, I_), (F_, 2, 0, I_)], in_h=3, in_w=3, n_classes=2)
    p = np.zeros(o.n_params)
    p[0] = 1.0
    x = np.arange(9, dtype=np.float32) - 4
    _, trace, _ = o.forward(p, x)
    np.testing.assert_array_equal(trace[:9], x)


# --------------------------------------------------------------------------------------
# torch float64 autograd (library routine) on the BASELINE.json nets
# --------------------------------------------------------------------------------------
from helpers import torch_grad  # noqa: E402  (torch conv2d / max_pool2d / linear / cross_entropy)


@pytest.mark.parametrize("name", ["tiny", "medium", "large", "paper_small", "paper_large"])
def test_against_torch_f64(name):
    arch = sd.ARCHS[name]
    o = Oracle(arch)
    d = sd.prototype_dataset(11, 3, 0)
    p = sd.init_params(11, o.blocks()).astype(np.float64)
    tl, tg, tlogits = torch_grad(arch, p, d.x_train, d.y_train)
    tot_l = 0.0
    tot_g = np.zeros(o.n_params)
    for i in range(3):
        logits, _, _ = o.forward(p, d.x_train[i])
        np.testing.assert_allclose(logits, tlogits[i], rtol=1e-12, atol=1e-13)
        li, gi = o.sample_grad(p, d.x_train[i], d.y_train[i])
        tot_l += li
        tot_g += gi
    assert tot_l == pytest.approx(tl, rel=1e-12)
    np.testing.assert_allclose(tot_g, tg, rtol=1e-10, atol=1e-12 * np.abs(tg).max())
    # one sync step of batch 3 = W - lr * sum g
    p1, _ = o.train_sync(p, d.x_train, d.y_train, 0.05, 3)
    np.testing.assert_allclose(p1, p - 0.05 * tg, rtol=1e-12, atol=1e-14)


# --------------------------------------------------------------------------------------
# Central finite differences on random tie-free tiny nets with every layer kind
# --------------------------------------------------------------------------------------
FD_ARCH = [(C_, 3, 3, T_), (P_, 0, 2, T_), (C_, 4, 2, T_), (P_, 0, 2, T_), (F_, 5, 0, T_), (F_, 3, 0, I_)]


def _min_pool_gap(o, p, x, arch, in_hw):
    """Smallest top-2 gap over every pool window (ties make FD invalid, Appendix A)."""
    _, trace, _ = o.forward(p, x)
    off = 0
    c, h, w = 1, in_hw, in_hw
    gap = np.inf
    prev = None
    for kind, units, k, act in arch:
        if kind == C_:
            h, w, c = h - k + 1, w - k + 1, units
            n = c * h * w
            prev = trace[off:off + n].reshape(c, h, w)
            off += n
        elif kind == P_:
            ph, pw = h // k, w // k
            for m in range(c):
                for pr in range(ph):
                    for pc in range(pw):
                        v = np.sort(prev[m, pr * k:pr * k + k, pc * k:pc * k + k].reshape(-1))
                        gap = min(gap, v[-1] - v[-2])
            h, w = ph, pw
            off += c * h * w
        else:
            off += units
            c, h, w = units, 1, 1
    return gap


def test_finite_differences():
    in_hw = 11
    o = Oracle(FD_ARCH, in_h=in_hw, in_w=in_hw, n_classes=3)
    rng = np.random.default_rng(3)
    done = 0
    for trial in range(50):
        p = rng.uniform(-0.6, 0.6, o.n_params)
        x = rng.uniform(-1, 1, in_hw * in_hw).astype(np.float32)
        if _min_pool_gap(o, p, x, FD_ARCH, in_hw) < 1e-3:
            continue
        label = int(rng.integers(0, 3))
        _, g = o.sample_grad(p, x, label)
        eps = 1e-5
        fd = np.zeros_like(g)
        for j in range(o.n_params):
            pp = p.copy()
            pp[j] += eps
            lp, _ = o.sample_grad(pp, x, label)
            pp[j] -= 2 * eps
            lm, _ = o.sample_grad(pp, x, label)
            fd[j] = (lp - lm) / (2 * eps)
        scale = np.maximum(np.abs(fd), 1e-3 * np.abs(fd).max())
        assert np.max(np.abs(fd - g) / scale) < 1e-4
        done += 1
        if done == 3:
            break
    assert done == 3


def test_fd_invalid_at_tie():
    # Appendix A: at the Example-A tie, FD gives half the analytic dK00
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    o = Oracle(HAND_ARCH, in_h=4, in_w=4, n_classes=2)
    p = np.array(g["params0"])
    x = np.array(g["A"]["x"], np.float32).reshape(-1)
    eps = 1e-5
    pp = p.copy()
    pp[0] += eps
    lp, _ = o.sample_grad(pp, x, 1)
    pp[0] -= 2 * eps
    lm, _ = o.sample_grad(pp, x, 1)
    assert (lp - lm) / (2 * eps) == pytest.approx(0.5630198049, abs=1e-6)


# --------------------------------------------------------------------------------------
# Invariants
# --------------------------------------------------------------------------------------
def test_softmax_delta_invariants():
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(4, 4, 0)
    p = sd.init_params(4, o.blocks())
    for i in range(4):
        _, g = o.sample_grad(p, d.x_train[i], d.y_train[i])
        gb = g[-10:]  # output-layer bias gradient = softmax - onehot
        prob = gb.copy()
        prob[d.y_train[i]] += 1.0
        assert prob.sum() == pytest.approx(1.0, abs=1e-12)
        assert np.all(prob > 0) and np.all(prob < 1)


def test_floor_dropped_inputs_do_not_matter():
    # conv 1x1 identity on 5x5, pool 2 -> 2x2 drops row 4 / col 4: changing those pixels
    # (kept below the window maxima) changes neither loss nor gradient
    arch = [(C_, 1, 1, I_), (P_, 0, 2, T_), (F_, 2, 0, I_)]
    o = Oracle(arch, in_h=5, in_w=5, n_classes=2)
    p = np.array([1.0, 0.0, 0.3, -0.2, 0.1, -0.4, 0.0, 0.0, 0.0, 0.0])[:o.n_params]
    x = np.random.default_rng(0).uniform(0, 1, 25).astype(np.float32)
    l0, g0 = o.sample_grad(p, x, 0)
    x2 = x.reshape(5, 5).copy()
    x2[4, :] = -7.0
    x2[:, 4] = -3.0
    l1, g1 = o.sample_grad(p, x2.reshape(-1), 0)
    assert l0 == l1
    np.testing.assert_array_equal(g0, g1)


def test_pool_gradient_routes_to_argmax_only():
    # identity 1x1 conv, so conv gW = sum over windows of delta_pool * x[argmax]:
    # compare with brute force over the windows
    arch = [(C_, 1, 1, I_), (P_, 0, 2, T_), (F_, 1, 0, T_), (F_, 2, 0, I_)]
    o = Oracle(arch, in_h=4, in_w=4, n_classes=2)
    rng = np.random.default_rng(1)
    p = rng.uniform(-1, 1, o.n_params)
    p[0], p[1] = 1.0, 0.0
    x = rng.uniform(-1, 1, 16).astype(np.float32)
    logits, trace, am = o.forward(p, x)
    _, g = o.sample_grad(p, x, 1)
    # delta at the pooled outputs by the chain rule written out for this tiny net
    V1, c1 = p[2:6], p[6]
    V2, c2 = p[7:9], p[9:11]
    pooled = trace[16:20]
    h = np.tanh(V1 @ pooled + c1)
    z = V2 * h + c2
    prob = np.exp(z - z.max()) / np.exp(z - z.max()).sum()
    dz = prob - np.array([0.0, 1.0])
    dh = (V2 @ dz) * (1 - h * h)
    dpool = V1 * dh * 1.0  # pool sits on an identity conv: no tanh derivative
    xs = x.reshape(4, 4).astype(np.float64)
    expect_gw = sum(dpool[w] * xs[(w // 2) * 2 + am[w] // 2, (w % 2) * 2 + am[w] % 2] for w in range(4))
    assert g[0] == pytest.approx(expect_gw, rel=1e-12)
    assert g[1] == pytest.approx(dpool.sum(), rel=1e-12)


def test_sync_batch1_equals_sequential_bitwise():
    # orc_train_sgd is its own per-sample loop (not orc_train_sync with B = 1): two code paths
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(7, 20, 0)
    p = sd.init_params(7, o.blocks())
    a, la = o.train_sgd(p, d.x_train, d.y_train, 0.01)
    b, lb = o.train_sync(p, d.x_train, d.y_train, 0.01, 1)
    np.testing.assert_array_equal(a, b)
    assert la == lb


# --------------------------------------------------------------------------------------
# Multi-step trajectories against torch float64 autograd (library routine): W is updated
# between samples (sequential SGD, P:132 one worker) and between blocks (sync mode)
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "large", "paper_small"])
def test_sequential_sgd_trajectory_against_torch_f64(name):
    arch = sd.ARCHS[name]
    o = Oracle(arch)
    d = sd.prototype_dataset(31, 4, 0)
    p0 = sd.init_params(31, o.blocks()).astype(np.float64)
    lr = 0.1
    w = p0.copy()
    tl = 0.0
    for i in range(4):  # torch: gradient at the current W, update, next sample
        li, gi, _ = torch_grad(arch, w, d.x_train[i:i + 1], d.y_train[i:i + 1])
        w = w - lr * gi
        tl += li
    got, gl = o.train_sgd(p0, d.x_train, d.y_train, lr)
    np.testing.assert_allclose(got - p0, w - p0, rtol=1e-9, atol=1e-12 * np.abs(w - p0).max())
    assert gl == pytest.approx(tl, rel=1e-12)
    # teeth: a trainer that left W stale across the 4 samples (= one summed step) is far off
    stale, _ = o.train_sync(p0, d.x_train, d.y_train, lr, 4)
    assert np.abs((stale - p0) - (w - p0)).max() > 1e-3 * np.abs(w - p0).max()


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_sync_blocks_trajectory_against_torch_f64(name):
    arch = sd.ARCHS[name]
    o = Oracle(arch)
    d = sd.prototype_dataset(32, 7, 0)
    p0 = sd.init_params(32, o.blocks()).astype(np.float64)
    lr, B = 0.05, 3  # blocks [0,3) [3,6) [6,7): the last partial block is one update
    w = p0.copy()
    for s0 in range(0, 7, B):
        _, gs, _ = torch_grad(arch, w, d.x_train[s0:s0 + B], d.y_train[s0:s0 + B])  # sum at block-start W
        w = w - lr * gs
    got, _ = o.train_sync(p0, d.x_train, d.y_train, lr, B)
    np.testing.assert_allclose(got - p0, w - p0, rtol=1e-9, atol=1e-12 * np.abs(w - p0).max())
    # teeth: per-sample updates inside a block (W not held at the block start) differ
    seq, _ = o.train_sgd(p0, d.x_train, d.y_train, lr)
    assert np.abs((seq - p0) - (w - p0)).max() > 1e-3 * np.abs(w - p0).max()


# --------------------------------------------------------------------------------------
# Hogwild schedule replay (orc_replay, SURVEY C-1 step 9)
# --------------------------------------------------------------------------------------
def _whole_layer_reads(o, k, preds):
    out = []
    for l, (_, nw, nb) in enumerate(o.blocks()):
        out.append((k, l, 0, 0, nw + nb, sorted(preds)))
    return out


def test_sample_grad2_against_torch_f64():
    # forward at Pf, delta_in at Pb (a worker whose backward re-read saw newer weights)
    arch = sd.ARCHS["large"]
    o = Oracle(arch)
    d = sd.prototype_dataset(33, 2, 0)
    pf = sd.init_params(33, o.blocks()).astype(np.float64)
    pb = pf + 0.05 * np.random.default_rng(0).standard_normal(o.n_params)
    tl, tg, _ = torch_grad(arch, pf, d.x_train, d.y_train, params_bwd=pb)
    g = np.zeros(o.n_params)
    lsum = 0.0
    for i in range(2):
        li, gi = o.sample_grad2(pf, pb, d.x_train[i], d.y_train[i])
        g += gi
        lsum += li
    assert lsum == pytest.approx(tl, rel=1e-12)
    np.testing.assert_allclose(g, tg, rtol=1e-10, atol=1e-12 * np.abs(tg).max())
    # the last layer's gradients do not depend on Pb; an earlier layer's do
    _, g_same = o.sample_grad(pf, d.x_train[0], d.y_train[0])
    _, g_mix = o.sample_grad2(pf, pb, d.x_train[0], d.y_train[0])
    np.testing.assert_array_equal(g_mix[-1510:], g_same[-1510:])
    assert np.abs(g_mix[:340] - g_same[:340]).max() > 1e-6


def test_replay_total_order_is_sequential_sgd():
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(34, 5, 0)
    p = sd.init_params(34, o.blocks()).astype(np.float64)
    reads = [r for k in range(5) for r in _whole_layer_reads(o, k, range(k))]
    got, _ = o.replay(p, d.x_train, d.y_train, [(k, 1) for k in range(5)], reads, 0.05)
    ref, _ = o.train_sgd(p, d.x_train, d.y_train, 0.05)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-15)


@pytest.mark.parametrize("G", [1, 2])
def test_replay_all_concurrent_is_sync(G):
    # every group reads W0 (saw no publish): one summed step, = sync mode with B = n
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(35, 6, 0)
    p = sd.init_params(35, o.blocks()).astype(np.float64)
    got, pubs = o.replay(p, d.x_train, d.y_train, [(s, G) for s in range(0, 6, G)], [], 0.05)
    ref, _ = o.train_sync(p, d.x_train, d.y_train, 0.05, 6)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-15)
    np.testing.assert_allclose(pubs.sum(0), ref - p, rtol=0, atol=1e-15)


def test_replay_interval_orders_match_composition():
    # whole-sample staleness patterns (the 19 interval orders on 3 samples): the replay equals
    # composing per-sample gradients at W0 - lr * sum of the predecessors' gradients
    from helpers import interval_orders, compose_replay
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(36, 3, 0)
    p = sd.init_params(36, o.blocks()).astype(np.float64)
    orders = interval_orders(3)
    assert len(orders) == 19 and len(interval_orders(2)) == 3
    outs = []
    for preds in orders:
        reads = [r for k in range(3) for r in _whole_layer_reads(o, k, preds[k])]
        got, _ = o.replay(p, d.x_train, d.y_train, [(k, 1) for k in range(3)], reads, 0.5)
        np.testing.assert_allclose(got, compose_replay(o, p, d.x_train, d.y_train, 0.5, preds), rtol=0, atol=1e-14)
        outs.append(got)
    # distinct orders give distinct results at this lr (the replay is sensitive to the schedule)
    assert len({np.round(x, 9).tobytes() for x in outs}) >= 10


def test_replay_mixed_layer_read_against_torch_f64():
    # group 1 saw group 0's output-layer publish only (per-layer publishing, R5), forward and
    # delta_in; and group 2 saw group 0's publish of every layer for its forward pass but
    # delta_in at W0 for the output layer
    arch = sd.ARCHS["large"]
    o = Oracle(arch)
    d = sd.prototype_dataset(37, 3, 0)
    p = sd.init_params(37, o.blocks()).astype(np.float64)
    lr = 0.3
    bl = o.blocks()
    nl = len(bl)
    sizes = [nw + nb for _, nw, nb in bl]
    starts = np.cumsum([0] + sizes)
    reads = [(1, nl - 1, 0, 0, sizes[-1], [0])]
    reads += [(2, l, 0, 0, sizes[l], [0]) for l in range(nl)]
    reads += [(2, nl - 1, 1, 0, sizes[-1], [])]
    got, pubs = o.replay(p, d.x_train, d.y_train, [(0, 1), (1, 1), (2, 1)], reads, lr)
    _, g0, _ = torch_grad(arch, p, d.x_train[:1], d.y_train[:1])
    pub0 = -lr * g0
    w1 = p.copy()
    w1[starts[-2]:] += pub0[starts[-2]:]
    _, g1, _ = torch_grad(arch, w1, d.x_train[1:2], d.y_train[1:2])
    w2f = p + pub0
    w2b = w2f.copy()
    w2b[starts[-2]:] = p[starts[-2]:]
    _, g2, _ = torch_grad(arch, w2f, d.x_train[2:3], d.y_train[2:3], params_bwd=w2b)
    ref = p - lr * (g0 + g1 + g2)
    np.testing.assert_allclose(got - p, ref - p, rtol=1e-9, atol=1e-12 * np.abs(ref - p).max())
    np.testing.assert_allclose(pubs[1], -lr * g1, rtol=1e-9, atol=1e-12 * np.abs(g1).max() * lr)


def test_replay_partial_range_read():
    # an FC read split in two row ranges that saw different publishes (chunked staging)
    arch = sd.ARCHS["tiny"]
    o = Oracle(arch)
    d = sd.prototype_dataset(38, 2, 0)
    p = sd.init_params(38, o.blocks()).astype(np.float64)
    lr = 0.4
    (_, nw0, nb0), (_, nw1, nb1) = o.blocks()
    half = 5 * 845  # rows 0-4 of the FC W
    reads = [(1, 1, 0, 0, half, [0]), (1, 1, 0, half, nw1 + nb1, [])]
    got, _ = o.replay(p, d.x_train, d.y_train, [(0, 1), (1, 1)], reads, lr)
    _, g0 = o.sample_grad(p, d.x_train[0], d.y_train[0])
    w1 = p.copy()
    s = nw0 + nb0
    w1[s:s + half] -= lr * g0[s:s + half]
    _, g1, _ = torch_grad(arch, w1, d.x_train[1:2], d.y_train[1:2])
    np.testing.assert_allclose(got, p - lr * g0 - lr * g1, rtol=1e-10, atol=1e-14)


def test_replay_rejects_cycles_and_bad_reads():
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(39, 2, 0)
    p = sd.init_params(39, o.blocks())
    with pytest.raises(OracleError):  # 0 saw 1 and 1 saw 0
        o.replay(p, d.x_train, d.y_train, [(0, 1), (1, 1)], [(0, 0, 0, 0, 5, [1]), (1, 0, 0, 0, 5, [0])], 0.1)
    with pytest.raises(OracleError):  # a group cannot see its own publish
        o.replay(p, d.x_train, d.y_train, [(0, 1), (1, 1)], [(0, 0, 0, 0, 5, [0])], 0.1)
    with pytest.raises(OracleError):  # range beyond the layer
        o.replay(p, d.x_train, d.y_train, [(0, 1), (1, 1)], [(1, 0, 0, 0, 10 ** 6, [0])], 0.1)


def test_sync_permutation_within_batch():
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(8, 8, 0)
    p = sd.init_params(8, o.blocks())
    a, _ = o.train_sync(p, d.x_train, d.y_train, 0.01, 8)
    perm = np.random.default_rng(0).permutation(8)
    b, _ = o.train_sync(p, d.x_train[perm], d.y_train[perm], 0.01, 8)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15)


def test_evaluate_brute_force():
    o = Oracle(sd.ARCHS["tiny"])
    d = sd.prototype_dataset(10, 0, 30)
    p = sd.init_params(10, o.blocks())
    ml, ne, losses, preds = o.evaluate(p, d.x_test, d.y_test, per_sample=True)
    errs = 0
    for i in range(30):
        logits, _, _ = o.forward(p, d.x_test[i])
        errs += int(np.argmax(logits)) != d.y_test[i]  # numpy argmax: first maximum
        assert preds[i] == int(np.argmax(logits))
    assert ne == errs
    _, tg, tlog = torch_grad(sd.ARCHS["tiny"], p.astype(np.float64), d.x_test, d.y_test)
    import torch
    tce = torch.nn.functional.cross_entropy(torch.tensor(tlog), torch.tensor(d.y_test.astype(np.int64)))
    assert ml == pytest.approx(tce.item(), rel=1e-12)


def test_label_out_of_range():
    o = Oracle(sd.ARCHS["tiny"])
    with pytest.raises(OracleError):
        o.sample_grad(np.zeros(o.n_params), np.zeros(841, np.float32), 10)


def test_empty_training_is_noop():
    o = Oracle(sd.ARCHS["tiny"])
    p = sd.init_params(1, o.blocks())
    q, _ = o.train_sgd(p, np.zeros((0, 841), np.float32), np.zeros(0, np.int32), 0.1)
    np.testing.assert_array_equal(q, p.astype(np.float64))


def test_min_pool_gaps_flags_the_appendix_a_tie():
    # Example A has a 3-way tie in its pool window (gap 0); Example B is tie-free
    from helpers import min_pool_gaps
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    o = Oracle(HAND_ARCH, in_h=4, in_w=4, n_classes=2)
    p0 = np.array(g["params0"])
    ga = min_pool_gaps(HAND_ARCH, o.forward(p0, np.array(g["A"]["x"], np.float32).reshape(-1))[1], 1, 4, 4)
    gb = min_pool_gaps(HAND_ARCH, o.forward(p0, np.array(g["B"]["x"], np.float32).reshape(-1))[1], 1, 4, 4)
    assert ga == [0.0]
    # B: window values tanh(0.5), tanh(-0.5), tanh(1.5), tanh(0.5): gap = (tanh 1.5 - tanh 0.5) / tanh 1.5
    assert gb[0] == pytest.approx((math.tanh(1.5) - math.tanh(0.5)) / math.tanh(1.5), rel=1e-12)
