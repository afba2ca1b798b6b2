"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Tolerance (reading R9): per tensor, |gpu-ref| <= 1e-4 * max(|ref|, 1e-2*||ref||_inf)
element-wise and ||gpu-ref||_2 <= 1e-5 ||ref||_2 for gradients and weights after one step;
mean test loss after one epoch within rel 1e-3 (BASELINE.json north_star).
"""
import json
import os

import numpy as np
import pytest

import synthdata as sd
from oracle import Oracle
from helpers import assert_parity, parity_report, tie_free_prefix

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "oracle_runs")
NETS = ["tiny", "medium", "large", "paper_small", "paper_large"]
# Element-wise tolerance of multi-step weight comparisons (R9 / R16): BASELINE.json's
# rel 1e-4 for its nets; the Table I large net (not a BASELINE config) 3e-4: plain fp32 (torch
# CPU float32) itself reaches 1.22x the 1e-4 bound on the 3-step B = 64 trajectory of
# test_sync_steps (profiles/r3/tolerance_table.md, scripts/tolerance_table.py)
REL = {"paper_large": 3e-4}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch


def make(name, seed, torch_cuda, group=None):
    from paper_1506_09067_b200 import OPT_GROUP, Net
    o = Oracle(sd.ARCHS[name])
    net = Net(sd.ARCHS[name], init_seed=seed)
    if group is not None:
        if group != 1 and name == "paper_large":
            net.close()
            pytest.skip("paper_large is compiled for G = 1 only (one image per worker)")
        net.set_option(OPT_GROUP, group)
    p = sd.init_params(seed, o.blocks())
    net.set_params(p)
    return o, net, p


def dev(torch, *arrays):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


@pytest.mark.parametrize("name", NETS)
def test_create_initialises_like_the_generator(name, torch_cuda):
    from paper_1506_09067_b200 import Net
    o = Oracle(sd.ARCHS[name])
    for seed in (0, 1, 2):
        net = Net(sd.ARCHS[name], init_seed=seed)
        np.testing.assert_array_equal(net.get_params(), sd.init_params(seed, o.blocks()))
        net.close()


@pytest.mark.parametrize("name", NETS)
def test_set_get_roundtrip(name, torch_cuda):
    o, net, p = make(name, 3, torch_cuda)
    q = np.random.default_rng(0).standard_normal(o.n_params).astype(np.float32)
    net.set_params(q)
    np.testing.assert_array_equal(net.get_params(), q)
    assert net.device_params().numel() >= o.n_params


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("group", [None, 1, 4])
def test_forward_logits(name, group, torch_cuda):
    o, net, p = make(name, 4, torch_cuda, group)
    d = sd.prototype_dataset(4, 0, 37)  # ragged vs G
    X, = dev(torch_cuda, d.x_test)
    logits = net.forward(X).cpu().numpy()
    for i in range(37):
        ref, _, _ = o.forward(p, d.x_test[i])
        tol = 1e-4 * np.maximum(np.abs(ref), 1e-2 * np.abs(ref).max())
        assert np.all(np.abs(logits[i] - ref) <= tol), (i, logits[i], ref)


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("n", [1, 13])
@pytest.mark.parametrize("group", [None, 4])  # None: G unset, small batches run at G = 1
def test_gradients(name, n, group, torch_cuda):
    # default G and G = 4 (the tiny / Table I small nets default to G = 1), each against the oracle
    o, net, p = make(name, 5, torch_cuda, group)
    d = sd.prototype_dataset(5, n, 0)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    g = net.compute_gradients(X, Y)
    ref = np.zeros(o.n_params)
    for i in range(n):
        ref += o.sample_grad(p, d.x_train[i], d.y_train[i])[1]
    assert_parity(g, ref, o.blocks())


@pytest.mark.parametrize("name", NETS)
def test_gradients_group1_equal_default_group(name, torch_cuda):
    # G only changes the summation grouping: within tolerance of each other and the oracle
    o, net, p = make(name, 6, torch_cuda, 1)
    d = sd.prototype_dataset(6, 9, 0)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    g1 = net.compute_gradients(X, Y)
    _, net2, _ = make(name, 6, torch_cuda, 4)
    g4 = net2.compute_gradients(X, Y)
    assert_parity(g1, g4.astype(np.float64), o.blocks())


@pytest.mark.parametrize("name", NETS)
def test_sync_steps(name, torch_cuda):
    # 3 sync batches (B=64, last one partial: 150 = 64+64+22) on the same trajectory for every net.
    # (a) Each step from the oracle's weights at its start, against the oracle's step (R9 / R16 for
    #     the Table I large net): a step whose batch has a pool near-tie at those weights (top-2
    #     gap < 1e-5 relative, SURVEY C-15) may take the other argmax in fp32 -- reported, not
    #     failed (at least one step per net must be checked).
    # (b) The whole 3-step GPU trajectory against the oracle's, when the trajectory is tie-free.
    from helpers import min_pool_gaps
    from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
    seed, n, batch = 7, 150, 64
    o, net, p = make(name, seed, torch_cuda)
    net.set_option(OPT_SYNC_BATCH, batch)
    d = sd.prototype_dataset(seed, n, 0)
    lr = 0.05
    rel = REL.get(name, 1e-4)
    arch = sd.ARCHS[name]
    w = p.astype(np.float64)
    checked, attributed, min_gap = 0, [], 1.0
    for s0 in range(0, n, batch):
        xs, ys = d.x_train[s0:s0 + batch], d.y_train[s0:s0 + batch]
        w32 = w.astype(np.float32)
        gap = min(min(min_pool_gaps(arch, o.forward(w32, x)[1]), default=1.0) for x in xs)
        min_gap = min(min_gap, gap)
        ref, _ = o.train_sync(w32, xs, ys, lr, batch)
        net.set_params(w32)
        X, Y = dev(torch_cuda, xs, ys)
        net.train_epoch(X, Y, lr, SYNC)
        got = net.get_params().astype(np.float64)
        ok_w = parity_report(got, ref, o.blocks(), rel=rel)[0]
        ok_s, ws, wns, _ = parity_report(got - w32, ref - w32, o.blocks(), rel=1e-3, floor=1e-2, norm_rel=1e-4)
        if ok_w and ok_s:
            checked += 1
        elif gap < 1e-5:
            attributed.append((s0, gap, ws))
        else:
            assert False, f"step at image {s0}: {parity_report(got, ref, o.blocks(), rel=rel)[1:3]}, step {ws}, {wns}"
        w = ref
    assert checked >= 1, attributed
    if attributed:
        print(f"{name}: steps attributed to pool near-ties (start image, gap, step x tol): {attributed}")
    if min_gap >= 1e-5:
        _, net2, _ = make(name, seed, torch_cuda)
        net2.set_option(OPT_SYNC_BATCH, batch)
        X, Y = dev(torch_cuda, d.x_train, d.y_train)
        net2.train_epoch(X, Y, lr, SYNC)
        got = net2.get_params()
        ref, _ = o.train_sync(p, d.x_train, d.y_train, lr, batch)
        # the weights move by lr*g: compare the step (ref - p) as well as the weights
        assert_parity(got, ref, o.blocks(), rel=rel)
        step_ok, ws, wn, _ = parity_report(got.astype(np.float64) - p, ref - p, o.blocks(), rel=1e-3, floor=1e-2,
                                           norm_rel=1e-4)
        assert step_ok, (ws, wn)


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("group", [4, 1])  # explicit: an unset G runs these small batches at G = 1
def test_exact_pool_ties(name, group, torch_cuda):
    # every pool window ties exactly (SURVEY C-14, first maximum in row-major order):
    # (a) all-zero weights -- every activation is 0; closed form: the output bias gradient is
    #     sum(0.1 - onehot), every other gradient exactly 0;
    # (b) constant images with random weights -- every conv output is constant over its map, so
    #     every window of every pool layer ties; gradients against the oracle (R9)
    o, net, p = make(name, 19, torch_cuda, group)
    d = sd.prototype_dataset(19, 9, 0)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    net.set_params(np.zeros(o.n_params, np.float32))
    g = net.compute_gradients(X, Y)
    expect = np.zeros(o.n_params)
    for y in d.y_train:
        expect[-10:] += 0.1
        expect[-10 + y] -= 1.0
    np.testing.assert_allclose(g[-10:], expect[-10:], rtol=1e-6, atol=1e-6)
    assert np.count_nonzero(g[:-10]) == 0
    net.set_params(p)
    xc = np.empty_like(d.x_train)
    for i in range(9):
        xc[i] = np.float32((i - 4) / 4.5)  # constant per image, in [-1, 1] (one image all zero)
    X, = dev(torch_cuda, xc)
    g = net.compute_gradients(X, Y)
    ref = sum(o.sample_grad(p, xc[i], d.y_train[i])[1] for i in range(9))
    assert_parity(g, ref, o.blocks())
    logits = net.forward(X).cpu().numpy()
    for i in range(9):
        r, _, am = o.forward(p, xc[i])
        assert not am.any()  # the oracle's argmax is the first position of every window
        tol = 1e-4 * np.maximum(np.abs(r), 1e-2 * np.abs(r).max())
        assert np.all(np.abs(logits[i] - r) <= tol)


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("group", [1, 4])
def test_sync_is_bitwise_deterministic(name, group, torch_cuda):
    # every sum in the fused kernel has a fixed order, so sync mode is bitwise reproducible; this
    # is also the race detector for the kernel's shared-memory hand-offs (compute-sanitizer is
    # closed on this pool): a race would show up as run-to-run differences
    from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
    d = sd.prototype_dataset(8, 500, 0)
    outs = []
    for _ in range(3):
        o, net, p = make(name, 8, torch_cuda, group)
        net.set_option(OPT_SYNC_BATCH, 64)
        X, Y = dev(torch_cuda, d.x_train, d.y_train)
        net.train_epoch(X, Y, 0.01, SYNC)
        outs.append(net.get_params())
        net.close()
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


def test_sync_epoch_config0(torch_cuda):
    # BASELINE.json configs[0]: tiny net, 1,000 / 200 images, sync batch 1, lr 0.01, 1 epoch
    from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
    w = sd.WORKLOADS["config0"]
    d = sd.make_dataset(w)
    o, net, p = make("tiny", w.seed, torch_cuda)
    net.set_option(OPT_SYNC_BATCH, 1)
    X, Y, Xt, Yt = dev(torch_cuda, d.x_train, d.y_train, d.x_test, d.y_test)
    net.train_epoch(X, Y, w.lr0, SYNC)
    ml, ne = net.evaluate(Xt, Yt)
    refp, _ = o.train_sync(p, d.x_train, d.y_train, w.lr0, 1)
    rml, rne = o.evaluate(refp, d.x_test, d.y_test)
    assert abs(ml - rml) <= 1e-3 * abs(rml)
    assert abs(ne - rne) <= 2  # argmax near-ties may flip (reading R9)


@pytest.mark.parametrize("run", ["config1_sync64", "config2_sync64_e1", "config3_sync64_e1"])
def test_sync_epoch_loss_vs_oracle_run(run, torch_cuda):
    # one full epoch of sync B=64 on the 60k set; mean test CE within rel 1e-3 of the oracle's
    from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
    path = os.path.join(GOLD, run + ".json")
    if not os.path.exists(path):
        pytest.skip(f"oracle reference run {run} not recorded yet")
    rec = json.load(open(path))
    w = sd.WORKLOADS[rec["workload"]]
    d = sd.make_dataset(w)
    assert d.sha256() == rec["data_sha256"]
    o, net, p = make(w.arch, w.seed, torch_cuda)
    net.set_option(OPT_SYNC_BATCH, 64)
    X, Y, Xt, Yt = dev(torch_cuda, d.x_train, d.y_train, d.x_test, d.y_test)
    net.train_epoch(X, Y, w.lr0, SYNC)
    ml, ne = net.evaluate(Xt, Yt)
    e1 = rec["per_epoch"][0]
    assert abs(ml - e1["test_mean_loss"]) <= 1e-3 * e1["test_mean_loss"], (ml, e1)
    assert abs(ne - e1["test_errors"]) <= 5


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("seed", [9, 21])
def test_hogwild_single_worker_is_sequential_sgd(name, seed, torch_cuda):
    # one CTA, G = 1: CHAOS with one worker = sequential SGD (SURVEY C-9).  The comparison
    # runs over the trajectory's leading samples before the first pool near-tie (top-2 gap
    # < 5e-6 relative), where fp32 vs fp64 may legitimately pick different argmaxes (R9).
    from paper_1506_09067_b200 import OPT_MAX_CTAS
    o, net, p = make(name, seed, torch_cuda, 1)
    net.set_option(OPT_MAX_CTAS, 1)
    d = sd.prototype_dataset(seed, 24, 0)
    n = tie_free_prefix(o, sd.ARCHS[name], p, d.x_train, d.y_train, 0.05)
    assert n >= 6, f"near-tie too early on this trajectory (sample {n}); pick another seed"
    X, Y = dev(torch_cuda, d.x_train[:n], d.y_train[:n])
    net.train_epoch(X, Y, 0.05)
    got = net.get_params()
    ref, _ = o.train_sgd(p, d.x_train[:n], d.y_train[:n], 0.05)
    assert_parity(got, ref, o.blocks(), rel=REL.get(name, 1e-4))


@pytest.mark.parametrize("name", NETS)
def test_hogwild_claims_each_image_exactly_once(name, torch_cuda):
    from paper_1506_09067_b200 import OPT_DEBUG_CLAIMS
    o, net, p = make(name, 10, torch_cuda)
    net.set_option(OPT_DEBUG_CLAIMS, 1)
    n = 10003
    d = sd.prototype_dataset(10, n, 0)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    net.train_epoch(X, Y, 0.001)
    net.sync()
    np.testing.assert_array_equal(net.debug_claims(n), np.ones(n, np.int32))


def run_traced(name, seed, torch_cuda, n, lr, group=None, max_ctas=None, stagger=0, data=None):
    """One hogwild epoch of the schedule-recording build: returns (oracle, p0, data, params after,
    records, per-group publishes, G)."""
    from paper_1506_09067_b200 import OPT_DEBUG_STAGGER, OPT_DEBUG_TRACE, OPT_MAX_CTAS
    o, net, p = make(name, seed, torch_cuda, group)
    if max_ctas:
        net.set_option(OPT_MAX_CTAS, max_ctas)
    net.set_option(OPT_DEBUG_TRACE, 1)
    net.set_option(OPT_DEBUG_STAGGER, stagger)
    d = data if data is not None else sd.prototype_dataset(seed, n, 0)
    X, Y = dev(torch_cuda, d.x_train[:n], d.y_train[:n])
    net.train_epoch(X, Y, lr)
    G = net.launch_info()["group"]
    ng = -(-n // G)
    rec, pubs, reads = net.debug_trace(ng, reads=True)
    got = net.get_params().astype(np.float64)
    net.close()
    return o, p, d, got, rec, pubs.astype(np.float64), G, reads


def check_traced_epoch(o, arch, p, d, n, lr, got, rec, pubs, G, reads=None):
    """Replay a recorded hogwild schedule in the oracle (orc_replay, SURVEY C-1 step 9).
    (1) no lost or doubled update: final W = W0 + the sum of the groups' publishes;
    (2) every group whose reads overlapped no publish: its publish equals the oracle's gradient
        sum at exactly the weights it saw (W0 + the publishes it saw, per layer, forward and
        delta_in reads separately), R9 per tensor; a mismatch is excused only where the group's
        forward has a pool near-tie (top-2 gap < 5e-6, R9) at those weights.
    Returns (groups checked exactly, groups with an overlapping read, near-tie excuses)."""  # noqa: D205
    from helpers import assert_sum_of_publishes, check_read_values, min_pool_gaps, schedule_from_trace
    blocks = o.blocks()
    reads_rec = reads
    groups, reads, amb = schedule_from_trace(rec, blocks, n, G)
    assert_sum_of_publishes(got, p, pubs.sum(0), np.abs(pubs).sum(0), len(groups))
    excused_reads = []
    if reads_rec is not None:
        # (3) the values each group read are W0 + publishes consistent with the schedule, and
        # (4) EVERY group's publish -- torn reads included -- is the oracle's gradient sum at
        #     exactly the weights it read (forward and delta_in reads separately)
        check_read_values(rec, blocks, reads_rec, p, pubs)
        for k, (first, cnt) in enumerate(groups):
            wf = reads_rec[k, 0].astype(np.float64)
            wb = np.where(np.isnan(reads_rec[k, 1]), reads_rec[k, 0], reads_rec[k, 1]).astype(np.float64)
            g = sum(o.sample_grad2(wf, wb, d.x_train[i], d.y_train[i])[1] for i in range(first, first + cnt))
            ulp = 2.0 ** -24 * np.abs(wf)  # R20: below one ulp of the weight it updates, an update is moot
            ok, w, wn, det = parity_report(pubs[k], -lr * g, blocks, abs_floor=ulp)
            if not ok:
                gap = min(min(min_pool_gaps(arch, o.forward(wf, d.x_train[i])[1]), default=1.0)
                          for i in range(first, first + cnt))
                if gap < 5e-6:
                    excused_reads.append((k, "near-tie", w))
                    continue
                # reading R17: mid-training, a group's fixed-order fp32 sums of a few
                # hundred mixed-sign terms can cancel enough to miss R9 (derived for first steps at
                # init); such a group is held to 10x R9 (element-wise 1e-3 with the 1e-2 floor, norm
                # 1e-4) or to twice the error of plain fp32 on the same input (torch float32 CPU
                # autograd at the same weights), whichever is larger -- a wrong read or a lost update
                # is off by orders of magnitude -- and at most 2% of the groups may need it
                import torch
                from helpers import torch_grad
                X32 = d.x_train[first:first + cnt]
                _, g32, _ = torch_grad(arch, wf.astype(np.float32), X32, d.y_train[first:first + cnt],
                                       params_bwd=wb.astype(np.float32), dtype=torch.float32)
                _, w32, wn32, _ = parity_report(-lr * g32, -lr * g, blocks, abs_floor=ulp)
                assert w <= max(10.0, 2.0 * w32) and wn <= max(10.0, 2.0 * wn32), \
                    f"group {k} (worker {rec[k, 30]}): publish != oracle at the weights it read ({w:.3g} x tol, " \
                    f"norm {wn:.3g}; {det}); min pool gap {gap:.2e}; torch fp32 reaches {w32:.3g} x tol, norm {wn32:.3g}"
                excused_reads.append((k, "R17", round(w, 2), round(wn, 2), "torch-fp32", round(w32, 2), round(wn32, 2)))
    _, ref = o.replay(p, d.x_train[:n], d.y_train[:n], groups, reads, lr, pubs_in=pubs)
    exact, excused = 0, 0
    for k in range(len(groups)):
        if k in amb:
            continue
        if reads_rec is not None:
            seen0 = reads_rec[k, 0].astype(np.float64)
        else:
            seen0 = p.astype(np.float64) + sum((pubs[j] for j in set().union(*[set(r[5]) for r in reads if r[0] == k])),
                                               np.zeros(len(p)))
        ok, w, wn, det = parity_report(pubs[k], ref[k], blocks, abs_floor=2.0 ** -24 * np.abs(seen0))
        if not ok:
            seenf = {r[1]: r[5] for r in reads if r[0] == k and r[2] == 0}
            wf = p.astype(np.float64).copy()
            starts = np.cumsum([0] + [nw + nb for _, nw, nb in blocks])
            for l, seen in seenf.items():
                for j in seen:
                    wf[starts[l]:starts[l + 1]] += pubs[j][starts[l]:starts[l + 1]]
            first, cnt = groups[k]
            gap = min(min(min_pool_gaps(arch, o.forward(wf, d.x_train[i])[1]), default=1.0)
                      for i in range(first, first + cnt))
            assert gap < 5e-6, f"group {k} (worker {rec[k, 30]}): publish != replay at the weights it read " \
                               f"({w:.3g} x tol, norm {wn:.3g}; per tensor {det}); min pool gap {gap:.2e}"
            excused += 1
        else:
            exact += 1
    if excused_reads:
        print("groups excused at the values they read:", excused_reads)
        assert sum(1 for e in excused_reads if e[1] == "R17") <= max(1, len(groups) // 50), excused_reads
    return exact, len(amb), excused


@pytest.mark.parametrize("name", ["tiny", "large"])
@pytest.mark.parametrize("stagger", [0, 30000, 90000, 250000])
def test_hogwild_three_workers_recorded_schedule(name, stagger, torch_cuda):
    # 3 workers x G = 1 on 3 images, CTA b starting b * stagger cycles late: different
    # interleavings of reads and per-layer publishes; each is replayed exactly (C-1 step 9)
    n, lr = 3, 0.5
    o, p, d, got, rec, pubs, G, reads = run_traced(name, 11, torch_cuda, n, lr, group=1, max_ctas=3, stagger=stagger)
    assert G == 1
    exact, n_amb, excused = check_traced_epoch(o, sd.ARCHS[name], p, d, n, lr, got, rec, pubs, G, reads)
    assert exact + excused + n_amb == 3
    print(f"{name} stagger {stagger}: workers {list(rec[:, 30])}, exact {exact}, overlapping {n_amb}, near-tie {excused}")
    if stagger >= 90000:  # workers far enough apart that some group's reads overlap no publish
        assert exact >= 1, (exact, n_amb, excused)


@pytest.mark.parametrize("name", ["tiny", "large"])
def test_hogwild_full_width_recorded_schedule(name, torch_cuda):
    # the bench launch configuration (all SMs, default G) on 1,024 images: every group whose
    # reads overlapped no publish is replayed exactly; the final weights hold every publish once
    n, lr = 1024, (0.005 if name == "tiny" else 0.05)  # tiny: 148 images in flight at G = 1 (R14)
    o, p, d, got, rec, pubs, G, reads = run_traced(name, 12, torch_cuda, n, lr)
    exact, n_amb, excused = check_traced_epoch(o, sd.ARCHS[name], p, d, n, lr, got, rec, pubs, G, reads)
    ng = -(-n // G)
    print(f"{name}: {ng} groups, {exact} replayed exactly from the schedule, {n_amb} with an overlapping "
          f"(possibly torn) read -- every group checked at the values it read; {excused} near-tie")
    assert exact + n_amb + excused == ng
    assert len(set(rec[:, 30])) > 64  # many workers took part


def test_hogwild_trace_records_detect_a_wrong_schedule(torch_cuda):
    # teeth: replaying the recorded 3-worker run with one group's reads emptied (pretending it
    # saw no publish) must fail the per-group check whenever that group had seen one
    n, lr = 3, 0.5
    o, p, d, got, rec, pubs, G, _ = run_traced("tiny", 11, torch_cuda, n, lr, group=1, max_ctas=3, stagger=250000)
    from helpers import schedule_from_trace
    groups, reads, amb = schedule_from_trace(rec, o.blocks(), n, G)
    saw = [k for k in range(3) if k not in amb and any(r[0] == k and r[5] for r in reads)]
    assert saw, "with a 250k-cycle stagger a later worker sees an earlier one's publishes"
    k = saw[0]
    wrong = [(g, l, pp, e0, e1, [] if g == k else s) for (g, l, pp, e0, e1, s) in reads]
    _, ref = o.replay(p, d.x_train[:n], d.y_train[:n], groups, wrong, lr, pubs_in=pubs)
    assert not parity_report(pubs[k], ref[k], o.blocks())[0]


def test_evaluate_matches_oracle_and_is_pure(torch_cuda):
    o, net, p = make("large", 12, torch_cuda)
    d = sd.prototype_dataset(12, 0, 301)
    Xt, Yt = dev(torch_cuda, d.x_test, d.y_test)
    before = net.get_params()
    ml, ne = net.evaluate(Xt, Yt)
    np.testing.assert_array_equal(net.get_params(), before)
    rml, rne, _, rpred = o.evaluate(p, d.x_test, d.y_test, per_sample=True)
    assert abs(ml - rml) <= 1e-4 * rml
    logits = net.forward(Xt).cpu().numpy()
    assert ne == int(np.sum(np.argmax(logits, 1) != d.y_test))  # brute force over the GPU logits
    assert abs(ne - rne) <= 2


def test_evaluate_group_independent(torch_cuda):
    from paper_1506_09067_b200 import OPT_GROUP
    o, net, p = make("medium", 13, torch_cuda)
    d = sd.prototype_dataset(13, 0, 97)
    Xt, Yt = dev(torch_cuda, d.x_test, d.y_test)
    a = net.evaluate(Xt, Yt)
    net.set_option(OPT_GROUP, 1)
    b = net.evaluate(Xt, Yt)
    assert a[1] == b[1] and abs(a[0] - b[0]) <= 1e-6 * a[0]


def test_label_out_of_range_is_latched(torch_cuda):
    from paper_1506_09067_b200 import ChaosError
    o, net, p = make("tiny", 14, torch_cuda)
    d = sd.prototype_dataset(14, 8, 0)
    y = d.y_train.copy()
    y[3] = 10
    X, Y = dev(torch_cuda, d.x_train, y)
    net.train_epoch(X, Y, 0.01)
    with pytest.raises(ChaosError, match="LABEL"):
        net.sync()
    net.sync()  # latch cleared


def test_empty_and_invalid(torch_cuda):
    from paper_1506_09067_b200 import ChaosError, SYNC
    o, net, p = make("tiny", 15, torch_cuda)
    X, Y = dev(torch_cuda, np.zeros((0, 841), np.float32), np.zeros(0, np.int32))
    net.train_epoch(X, Y, 0.01)
    net.train_epoch(X, Y, 0.01, SYNC)
    assert net.evaluate(X, Y) == (0.0, 0)
    np.testing.assert_array_equal(net.get_params(), p)
    with pytest.raises(ChaosError, match="INVALID"):
        net.train_epoch(X, Y, float("nan"))


def test_host_entry_point(torch_cuda):
    # chaos_train_epoch_host (e2e path) equals device-buffer training in sync mode
    from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
    d = sd.prototype_dataset(16, 200, 0)
    o, a, p = make("large", 16, torch_cuda)
    a.set_option(OPT_SYNC_BATCH, 64)
    a.train_epoch_host(d.x_train, d.y_train, 0.01, SYNC)
    _, b, _ = make("large", 16, torch_cuda)
    b.set_option(OPT_SYNC_BATCH, 64)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    b.train_epoch(X, Y, 0.01, SYNC)
    np.testing.assert_array_equal(a.get_params(), b.get_params())


def test_full_size_sampled_parity(torch_cuda):
    # the bench launch configuration (large net, default G, all SMs) on the 60k set:
    # sampled logits and gradients of single images checked one by one against the oracle
    w = sd.WORKLOADS["config3"]
    d = sd.make_dataset(w, 60000, 64)
    o, net, p = make("large", w.seed, torch_cuda)
    X, = dev(torch_cuda, d.x_train)
    logits = net.forward(X).cpu().numpy()
    rng = np.random.default_rng(0)
    for i in rng.choice(60000, 12, replace=False):
        ref, _, _ = o.forward(p, d.x_train[i])
        tol = 1e-4 * np.maximum(np.abs(ref), 1e-2 * np.abs(ref).max())
        assert np.all(np.abs(logits[i] - ref) <= tol), i
    # sum of gradients over a 4096-image slice equals the sum of the oracle's per-image gradients
    Xs, Ys = dev(torch_cuda, d.x_train[:256], d.y_train[:256])
    g = net.compute_gradients(Xs, Ys)
    ref = np.zeros(o.n_params)
    for i in range(256):
        ref += o.sample_grad(p, d.x_train[i], d.y_train[i])[1]
    assert_parity(g, ref, o.blocks())


@pytest.mark.parametrize("run", ["config1_seq", "config3_seq", "config2_seq", "paper_small_seq", "paper_large_seq"])
def test_hogwild_accuracy_gate(run, torch_cuda):
    # BASELINE.json north_star: hogwild test error within 0.5 pp of the oracle's sequential SGD
    import torch
    path = os.path.join(GOLD, run + ".json")
    if not os.path.exists(path):
        pytest.skip(f"oracle reference run {run} not recorded yet")
    rec = json.load(open(path))
    if len(rec["per_epoch"]) < rec["epochs"]:
        pytest.skip(f"oracle reference run {run} incomplete")
    w = sd.WORKLOADS[rec["workload"]]
    d = sd.make_dataset(w, rec.get("n_train"), rec.get("n_test"))
    assert d.sha256() == rec["data_sha256"]
    o, net, p = make(rec.get("arch", w.arch), w.seed, torch_cuda)
    X, Y, Xt, Yt = dev(torch, d.x_train, d.y_train, d.x_test, d.y_test)
    curve = []
    for e in range(rec["epochs"]):
        net.train_epoch(X, Y, w.lr0 * 0.9 ** e)
        curve.append(net.evaluate(Xt, Yt))
    ref = rec["per_epoch"][-1]
    n = len(d.y_test)
    print(run, "hogwild (CE, errors) per epoch:", [(round(c, 5), e) for c, e in curve])
    print(run, "oracle seq (CE, errors) per epoch:", [(round(r["test_mean_loss"], 5), r["test_errors"])
                                                     for r in rec["per_epoch"]])
    assert abs(curve[-1][1] - ref["test_errors"]) / n * 100 <= 0.5, (curve, ref)
    # the learning curve, epoch by epoch (R19): test errors within 0.5 pp of the oracle's
    # sequential SGD and mean test cross-entropy within a factor 1.3 of it at every epoch
    for (ce, ne), r in zip(curve, rec["per_epoch"]):
        assert abs(ne - r["test_errors"]) / n * 100 <= 0.5, (curve, rec["per_epoch"])
        assert r["test_mean_loss"] / 1.3 <= ce <= 1.3 * r["test_mean_loss"], (curve, rec["per_epoch"])


def test_batch_gradient_apply_equals_sync_epoch_bitwise(torch_cuda):
    # NEXT-4 building blocks on one GPU: batch_gradient + apply_gradient per batch reproduce
    # chaos_train_epoch(SYNC) bit for bit (same slot-ordered sum, same update expression)
    from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
    from paper_1506_09067_b200.dist import DistTrainer
    d = sd.prototype_dataset(17, 150, 0)
    o, a, p = make("large", 17, torch_cuda)
    a.set_option(OPT_SYNC_BATCH, 64)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    a.train_epoch(X, Y, 0.02, SYNC)
    _, b, _ = make("large", 17, torch_cuda)
    DistTrainer(b, 0, 1, 0).sync_epoch(X, Y, 0.02, batch=64)
    np.testing.assert_array_equal(a.get_params(), b.get_params())


def test_two_rank_sync_emulated_matches_oracle(torch_cuda):
    # NEXT-4 semantics with 2 ranks, emulated on one GPU: each batch's two halves are computed
    # separately (rank parts), summed (the all-reduce), applied; equals the oracle's sync SGD
    # within the R9 tolerance, and is bitwise reproducible run to run
    import torch
    from paper_1506_09067_b200.dist import batch_part
    d = sd.prototype_dataset(18, 150, 0)
    o, _, p = make("medium", 18, torch_cuda)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    runs = []
    for _ in range(2):
        _, net, _ = make("medium", 18, torch_cuda)
        g0 = torch.zeros_like(net.device_params())
        g1 = torch.zeros_like(g0)
        for b0 in range(0, 150, 64):
            nb = min(64, 150 - b0)
            s0, e0 = batch_part(b0, nb, 0, 2)
            s1, e1 = batch_part(b0, nb, 1, 2)
            net.batch_gradient(X[s0:e0], Y[s0:e0], g0)
            net.batch_gradient(X[s1:e1], Y[s1:e1], g1)
            g0 += g1
            net.apply_gradient(g0, 0.05)
        runs.append(net.get_params())
    np.testing.assert_array_equal(runs[0], runs[1])
    ref, _ = o.train_sync(p, d.x_train, d.y_train, 0.05, 64)
    assert_parity(runs[0], ref, o.blocks())


@pytest.mark.parametrize("mode", ["hogwild", "sync", "hogwild_dist", "hogwild_dist_async", "hogwild_dist_chaoscomm",
                                  "hogwild_dist_fallback"])
def test_bench_line_contract(mode, torch_cuda):
    # bench.py's JSON line on one GPU: contract keys, roofline + cpu_baseline objects, e2e with host bytes
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--steps", "1", "--warmup", "1",
           "--mode", mode.split("_")[0]]
    if mode != "hogwild":
        cmd.append("--no-cpu-baseline")
    if mode.startswith("hogwild_dist"):  # the N>1 code path on one GPU: one-rank NCCL group, fused averaging
        cmd.append("--force-dist")
    if mode == "hogwild_dist_async":  # ... or the in-flight NCCL averaging on reserved SMs
        cmd += ["--avg", "async"]
    if mode == "hogwild_dist_chaoscomm":  # ... with the library's own communicator
        cmd += ["--comm", "chaos"]
    env = dict(os.environ)
    if mode == "hogwild_dist_fallback":  # a failed first fused step: every rank drops to blocking intervals
        env["CHAOS_BENCH_FAIL_WARMUP"] = "1"
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] >= 1 and d["config"]["mode"] == mode.split("_")[0]
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == 60000 * (841 + 1) * 4
    if mode == "hogwild":
        assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    if mode == "hogwild_dist_fallback":
        assert d["config"]["averaging"].startswith("interval (fused failed") and d["collectives"] >= 58
        assert d["eval"]["test_errors"] < 0.05 * d["eval"]["images"]
    elif mode.startswith("hogwild_dist"):
        avg = "async" if mode == "hogwild_dist_async" else "fused"
        assert d["config"]["averaging"] == avg and d["collectives"] >= (2 if avg == "async" else 1)
        if avg == "fused":  # in-kernel rounds every K = 1,024 claimed images of the 60,000
            assert d["fused_rounds"] == 58 and d["config"]["pavg_comm_ctas"] == 1  # 1 timed step
        assert d["eval"]["test_errors"] < 0.05 * d["eval"]["images"]


def test_host_entry_hogwild_chunks_are_the_same_run(torch_cuda):
    # chaos_train_epoch_host lands ~n/16-image chunks (>= 2048) on a copy stream while ONE launch
    # trains, its claims gated by the landed-images counter; with one worker (1 CTA, G=1) hogwild
    # is sequential SGD, so the streamed host run must equal the device run bit for bit
    from paper_1506_09067_b200 import OPT_MAX_CTAS
    import torch
    n = 9000  # five chunks: 4 x 2048 + 808
    d = sd.prototype_dataset(19, n, 0)
    o, a, p = make("tiny", 19, torch_cuda, 1)
    a.set_option(OPT_MAX_CTAS, 1)
    a.train_epoch_host(torch.from_numpy(d.x_train).pin_memory(), torch.from_numpy(d.y_train).pin_memory(), 0.01)
    _, b, _ = make("tiny", 19, torch_cuda, 1)
    b.set_option(OPT_MAX_CTAS, 1)
    X, Y = dev(torch_cuda, d.x_train, d.y_train)
    b.train_epoch(X, Y, 0.01)
    np.testing.assert_array_equal(a.get_params(), b.get_params())
    assert abs(a.last_train_loss() - b.last_train_loss()) <= 1e-12 * abs(b.last_train_loss())


def test_phase_timing_is_not_in_the_product_build(torch_cuda):
    # chaos_debug_phase_times belongs to the instrumented build only
    from paper_1506_09067_b200 import ChaosError
    if os.environ.get("CHAOS_LIB"):
        pytest.skip("an alternative library is selected")
    _, net, _ = make("tiny", 1, torch_cuda)
    with pytest.raises(ChaosError, match="UNSUPPORTED"):
        net.phase_times()


def test_staleness_cap(torch_cuda):
    # R14: images in flight (CTAs x G) never exceed the per-net cap
    from paper_1506_09067_b200 import OPT_GROUP
    for name, cap in [("tiny", 148), ("medium", 592), ("large", 592), ("paper_small", 148), ("paper_large", 148)]:
        for g in ((1,) if name == "paper_large" else (1, 4)):
            _, net, _ = make(name, 1, torch_cuda, g)
            info = net.launch_info()
            assert info["grid"] * info["group"] <= cap, (name, g, info)
            net.close()


def test_avg_apply_snapshot_and_progress_abi(torch_cuda):
    # NEXT-2 building blocks (include/chaos.h): snapshot = params; apply adds avg - snap with the
    # same fp32 roundings as torch; the progress counter counts every enqueued image; waits up to
    # it return (on a side stream, beside the training launch), beyond it are refused
    import torch
    from paper_1506_09067_b200 import OPT_RESERVE_SMS, ChaosError
    _, net, _ = make("large", 3, torch_cuda)
    side = torch.cuda.Stream()
    params = net.device_params()
    snap = torch.empty_like(params)
    net.avg_snapshot(snap, side)
    side.synchronize()
    assert torch.equal(snap, params)
    g = torch.Generator(device="cuda").manual_seed(5)
    avg = snap + 1e-3 * torch.randn(snap.shape, generator=g, device="cuda")
    expect = params + (avg - snap)
    net.avg_apply(avg, snap, side)
    side.synchronize()
    assert torch.equal(params, expect)
    w = sd.WORKLOADS["config3"]
    xs, ys = sd.prototype_samples(w.seed, 0, 6001)
    X, Y = dev(torch, xs, ys)
    assert net.progress_enqueued() == 0
    net.train_epoch(X, Y, 0.001)
    net.train_epoch(X[:5], Y[:5], 0.001)
    assert net.progress_enqueued() == 6006
    net.progress_wait(6006, side)
    side.synchronize()  # returned: every image's updates are published
    with pytest.raises(ChaosError):
        net.progress_wait(6007, side)
    net.set_option(OPT_RESERVE_SMS, 4)
    assert net.launch_info()["grid"] == torch.cuda.get_device_properties(0).multi_processor_count - 4
    with pytest.raises(ChaosError):
        net.set_option(OPT_RESERVE_SMS, 100000)
    net.close()


def test_async_averaging_runs_in_flight(torch_cuda):
    # NEXT-2: with 4 SMs reserved, the progress waits on the comm stream return while the one
    # training launch runs (spread over it, not bunched at its end), and snapshot + zero-delta
    # apply in flight leave hogwild training intact (the config3 accuracy gate still holds)
    import torch
    from paper_1506_09067_b200 import OPT_RESERVE_SMS
    path = os.path.join(GOLD, "config3_seq.json")
    if not os.path.exists(path):
        pytest.skip("oracle reference run config3_seq not recorded")
    rec = json.load(open(path))
    w = sd.WORKLOADS[rec["workload"]]
    d = sd.make_dataset(w)
    _, net, _ = make(rec.get("arch", w.arch), w.seed, torch_cuda)
    net.set_option(OPT_RESERVE_SMS, 4)
    X, Y, Xt, Yt = dev(torch, d.x_train, d.y_train, d.x_test, d.y_test)
    side = torch.cuda.Stream()
    params = net.device_params()
    snap = torch.empty_like(params)
    n, k = int(Y.shape[0]), 1024
    spreads = []
    for e in range(w.epochs):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        side.wait_stream(net.stream)
        base = net.progress_enqueued()
        t0.record(net.stream)
        net.train_epoch(X, Y, w.lr0 * 0.9 ** e)
        t1.record(net.stream)
        marks = []
        for t in range(k, n, k):
            net.progress_wait(base + t, side)
            m = torch.cuda.Event(enable_timing=True)
            m.record(side)
            marks.append(m)
            net.avg_snapshot(snap, side)
            net.avg_apply(snap, snap, side)  # zero delta
        net.stream.wait_stream(side)
        torch.cuda.synchronize()
        total = t0.elapsed_time(t1)
        spreads.append(marks[0].elapsed_time(marks[-1]) / total)
    assert min(spreads) > 0.5, spreads
    ml, ne = net.evaluate(Xt, Yt)
    ref = rec["per_epoch"][-1]
    assert abs(ne - ref["test_errors"]) / len(d.y_test) * 100 <= 0.5, (ne, ref)
    net.close()


def test_two_replica_inflight_averaging_emulated(torch_cuda):
    # NEXT-2 with non-zero deltas, two replicas emulated on one GPU (the 8-GPU run is the
    # driver's): replica r is a net on its own stream with 70 CTAs (both launches co-resident, 8
    # SMs left for the averaging kernels), training its contiguous half of the configs[3] data
    # (strong scaling, P = 2) in ONE hogwild launch per epoch; a third stream runs the in-flight
    # schedule of DistTrainer.epoch_async -- wait for both progress counters to pass t = K, 2K,
    # ..., snapshot both, average (a torch mean stands in for the NCCL collective), apply
    # avg - snapshot to each live replica -- then the exact final average.  Epoch 1 is recorded
    # (schedule-trace build): the sum of the replicas before the final average equals 2 W0 plus
    # every group's publish (in-flight averages preserve the sum; none lost or doubled), with
    # non-zero deltas; after 15 epochs the averaged model passes the accuracy gate.
    import torch
    from paper_1506_09067_b200 import OPT_DEBUG_TRACE, OPT_MAX_CTAS, Net
    from paper_1506_09067_b200.dist import async_targets
    path = os.path.join(GOLD, "config3_seq.json")
    if not os.path.exists(path):
        pytest.skip("oracle reference run config3_seq not recorded")
    rec = json.load(open(path))
    w = sd.WORKLOADS[rec["workload"]]
    d = sd.make_dataset(w)
    arch = sd.ARCHS[rec.get("arch", w.arch)]
    o = Oracle(arch)
    p0 = sd.init_params(w.seed, o.blocks())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    nets = [Net(arch, init_seed=w.seed, stream=st) for st in streams]
    for net in nets:
        net.set_params(p0)
        net.set_option(OPT_MAX_CTAS, 70)
    X, Y, Xt, Yt = dev(torch, d.x_train, d.y_train, d.x_test, d.y_test)
    n = int(Y.shape[0])
    half = n // 2
    shards = [(0, half), (half, n)]
    side = torch.cuda.Stream()
    params = [net.device_params() for net in nets]
    snaps = [torch.empty_like(params[0]), torch.empty_like(params[0])]
    K = 1024
    deltas = []
    for e in range(w.epochs):
        lr = w.lr0 * 0.9 ** e
        traced = e == 0
        for net in nets:
            net.set_option(OPT_DEBUG_TRACE, 1 if traced else 0)
        side.wait_stream(torch.cuda.current_stream())
        for net in nets:
            net.stream.wait_stream(torch.cuda.current_stream())
        bases = [net.progress_enqueued() for net in nets]
        for net, (lo, hi) in zip(nets, shards):
            net.train_epoch(X[lo:hi], Y[lo:hi], lr)
        with torch.cuda.stream(side):
            for t in async_targets(min(hi - lo for lo, hi in shards), K):
                for net, b in zip(nets, bases):
                    net.progress_wait(b + t, side)
                for net, sn in zip(nets, snaps):
                    net.avg_snapshot(sn, side)
                avg = (snaps[0] + snaps[1]) * 0.5
                if traced:
                    deltas.append(float((avg - snaps[0]).abs().max()))
                for net, sn in zip(nets, snaps):
                    net.avg_apply(avg, sn, side)
        for net in nets:
            side.wait_stream(net.stream)
        torch.cuda.synchronize()
        if traced:
            G = nets[0].launch_info()["group"]
            tot = np.zeros(o.n_params)
            tot_abs = np.zeros(o.n_params)
            for net, (lo, hi) in zip(nets, shards):
                _, pubs = net.debug_trace(-(-(hi - lo) // G))[:2]
                tot += pubs.astype(np.float64).sum(0)
                tot_abs += np.abs(pubs.astype(np.float64)).sum(0)
            from helpers import assert_sum_of_publishes
            wa, wb = (net.get_params().astype(np.float64) for net in nets)
            # n_adds: each replica's groups plus its in-flight applies; the two replicas' roundings add
            n_adds = 2 * (-(-half // G) + len(deltas) + 1)
            assert_sum_of_publishes(wa + wb, 2 * p0.astype(np.float64), tot, 2 * np.abs(p0) + tot_abs,
                                    n_adds, rigorous=False)
            assert len(deltas) == len(async_targets(half, K)) and max(deltas) > 1e-4, deltas  # non-zero deltas
        with torch.cuda.stream(side):
            avg = (params[0] + params[1]) * 0.5
            params[0].copy_(avg)
            params[1].copy_(avg)
        side.synchronize()
    np.testing.assert_array_equal(nets[0].get_params(), nets[1].get_params())
    ml, ne = nets[0].evaluate(Xt, Yt)
    ref = rec["per_epoch"][-1]
    assert abs(ne - ref["test_errors"]) / len(d.y_test) * 100 <= 0.5, (ne, ref)
    for net in nets:
        net.close()


def test_library_nccl_communicator_one_rank(torch_cuda):
    # chaos_dist_* (include/chaos.h): with one rank the average is the identity, bitwise, for the
    # parameters (net's stream) and for a caller buffer (caller stream); uninitialised -> error
    import torch
    from paper_1506_09067_b200 import ChaosError
    _, net, _ = make("tiny", 3, torch_cuda)
    with pytest.raises(ChaosError):
        net.dist_average()
    uid = net.dist_unique_id()
    assert len(uid) == 128
    net.dist_init(uid, 0, 1)
    before = net.get_params()
    net.dist_average()
    net.sync()
    np.testing.assert_array_equal(net.get_params(), before)
    side = torch.cuda.Stream()
    buf = torch.randn(1003, device="cuda")
    ref = buf.clone()
    net.dist_average_buffer(buf, side)
    side.synchronize()
    assert torch.equal(buf, ref)
    with pytest.raises(ChaosError):
        net.dist_init(uid, 0, 1)  # already initialised
    net.close()


def test_host_entry_hogwild_claims_each_image_once(torch_cuda):
    # the streamed host entry at full width (all CTAs, default G): every image trained exactly once
    from paper_1506_09067_b200 import OPT_DEBUG_CLAIMS
    import torch
    n = 30011
    d = sd.prototype_dataset(23, n, 0)
    _, net, _ = make("large", 23, torch_cuda)
    net.set_option(OPT_DEBUG_CLAIMS, 1)
    net.train_epoch_host(torch.from_numpy(d.x_train).pin_memory(), torch.from_numpy(d.y_train).pin_memory(), 0.001)
    np.testing.assert_array_equal(net.debug_claims(n), np.ones(n, np.int32))
    assert np.isfinite(net.last_train_loss())
