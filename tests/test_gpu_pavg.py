"""GPU tests of the fused in-kernel cross-replica averaging (chaos_pavg_*, SURVEY.md §8(f) NEXT-2 fused
variant): R replicas emulated on ONE GPU as one cooperative launch of the same worker
(the replicas' CTAs wait on one another, so they must be co-resident -- never separate launches;
/opt/skills/guides/B200_PROFILING.md), plus the one-replica path of the multi-GPU launch and the
CUDA-IPC mapping between two processes.

The averaging round of PAPER.md:138-140 carried across replicas: snapshot s_r of each replica's
live weights, w_r += mean_q(s_q) - s_r with the mean in a fixed order (q = 0..R-1, then / R), so
with lr = 0 (no hogwild updates in between) T rounds are exactly the fp32 iteration written out
below, bitwise; with training, each round preserves the replicas' sum (checked by the device delta
sums and the in-kernel snapshot checksums) and the averaged model passes the accuracy gate.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synthdata as sd
from oracle import Oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "oracle_runs")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch


def replicas(R, seeds, k, torch_cuda, nslice=0, check=True, comm=0):
    """R large nets (replica r initialised from seeds[r]), set up as ranks 0..R-1 of one average
    over each other's exchange buffers; comm > 0: that many comm CTAs per replica run the rounds."""
    from paper_1506_09067_b200 import OPT_PAVG_COMM_CTAS, Net
    nets = [Net(sd.ARCHS["large"], init_seed=s) for s in seeds]
    for r, net in enumerate(nets):
        net.set_option(OPT_PAVG_COMM_CTAS, comm)
        net.pavg_setup(r, R, k, nslice)
    for net in nets:
        for q, other in enumerate(nets):
            if other is not net:
                net.pavg_set_peer(q, other)
        if check:
            net.pavg_set_check(True)
    return nets


def fixed_order_rounds(ws, T):
    """T averaging rounds with no training in between, in the kernel's fp32 arithmetic:
    s = w_0 + w_1 + ... (left to right), avg = s / R, w_r <- w_r + (avg - w_r)."""
    ws = [w.astype(np.float32).copy() for w in ws]
    R = np.float32(len(ws))
    for _ in range(T):
        s = ws[0].copy()
        for w in ws[1:]:
            s = (s + w).astype(np.float32)
        avg = (s / R).astype(np.float32)
        ws = [(w + (avg - w).astype(np.float32)).astype(np.float32) for w in ws]
    return ws


@pytest.mark.parametrize("R,nslice,T,comm", [(2, 0, 3, 0), (4, 0, 2, 0), (3, 37, 5, 0), (2, 16, 3, 1), (4, 9, 4, 2),
                                             (8, 0, 3, 0), (8, 16, 3, 1)])
def test_rounds_without_training_are_the_fixed_order_iteration(R, nslice, T, comm, torch_cuda):
    # lr = 0: the replicas start from different weights and only the averaging changes them; every
    # slice of every replica runs T sequential rounds, so the result is exactly fixed_order_rounds
    # (bitwise; R = 3 exercises a mean that is not a power-of-two scaling, nslice = 37 slices over
    # the CTAs of R = 3 replicas, the default nslice = 148 several slices per CTA at R = 4; comm > 0
    # the rounds run on comm CTAs, several slices each, 9 slices over 2 comm CTAs unevenly)
    import torch
    nets = replicas(R, list(range(10, 10 + R)), 512, torch_cuda, nslice, comm=comm)
    w0 = [net.get_params() for net in nets]
    n = 3000
    data = [sd.prototype_dataset(40 + r, n, 0) for r in range(R)]
    X = [torch.from_numpy(d.x_train).cuda() for d in data]
    Y = [torch.from_numpy(d.y_train).cuda() for d in data]
    for net in nets:
        net.pavg_arm(T)
    type(nets[0]).train_epoch_replicas(nets, X, Y, 0.0)
    for net in nets:
        net.sync()
    want = fixed_order_rounds(w0, T)
    for net, wr in zip(nets, want):
        np.testing.assert_array_equal(net.get_params(), wr)
        assert net.pavg_rounds_done() == T
        ds, da = net.pavg_debug_sums()
        assert np.isfinite(ds).all() and da.max() > 0
    # a second launch continues the monotonic round numbers (flags are never reset)
    for net in nets:
        net.pavg_arm(2)
    type(nets[0]).train_epoch_replicas(nets, X, Y, 0.0)
    for net in nets:
        net.sync()
    want = fixed_order_rounds(want, 2)
    for net, wr in zip(nets, want):
        np.testing.assert_array_equal(net.get_params(), wr)
        assert net.pavg_rounds_done() == T + 2
    for net in nets:
        net.close()


@pytest.mark.parametrize("comm", [0, 1])
def test_training_rounds_preserve_the_sum_and_pass_the_accuracy_gate(comm, torch_cuda):
    # two replicas (74 CTAs each) train their halves of the configs[3] data (strong scaling, P = 2),
    # averaged in-kernel every K = 1024 claimed images, then exactly (a torch mean stands in for the
    # final collective).  Epoch 1 runs in check mode: no torn / stale snapshot read (in-kernel
    # checksums), the deltas are non-zero and sum to ~0 over the replicas for every weight (each
    # round preserves the replicas' sum: no apply lost or doubled); after 15 epochs the averaged
    # model passes the config-3 accuracy gate against the oracle's sequential SGD
    import torch
    from paper_1506_09067_b200.dist import async_targets
    path = os.path.join(GOLD, "config3_seq.json")
    if not os.path.exists(path):
        pytest.skip("oracle reference run config3_seq not recorded")
    rec = json.load(open(path))
    w = sd.WORKLOADS[rec["workload"]]
    d = sd.make_dataset(w)
    arch = sd.ARCHS[rec.get("arch", w.arch)]
    p0 = sd.init_params(w.seed, Oracle(arch).blocks())
    K = 1024
    nets = replicas(2, [w.seed, w.seed], K, torch_cuda, nslice=16 if comm else 0, check=False, comm=comm)
    for net in nets:
        net.set_params(p0)
    X = torch.from_numpy(d.x_train).cuda()
    Y = torch.from_numpy(d.y_train).cuda()
    n = int(Y.shape[0])
    half = n // 2 // 4 * 4
    Xs, Ys = [X[:half], X[half:]], [Y[:half], Y[half:]]
    params = [net.device_params() for net in nets]
    T = len(async_targets(min(half, n - half), K))
    for e in range(w.epochs):
        check = e == 0
        w_start = params[0].cpu().numpy().astype(np.float64)  # internal layout, like the delta sums
        for net in nets:
            net.pavg_set_check(check)
            net.pavg_arm(T)
        type(nets[0]).train_epoch_replicas(nets, Xs, Ys, w.lr0 * 0.9 ** e)
        for net in nets:
            net.sync()  # raises on a checksum mismatch (latched in the kernel)
        if check:
            sums = [net.pavg_debug_sums() for net in nets]
            ds = sums[0][0].astype(np.float64) + sums[1][0]
            da = sums[0][1].astype(np.float64) + sums[1][1]
            assert da.max() > 1e-4, da.max()  # the rounds moved the weights
            # per weight and round, sum_r (avg - s_r) = R (avg - mean) + the deltas' own rounding:
            # |.| <= R * 2u * |w| + u * sum_r |delta_r|, plus u * |partial sum| per accumulation into
            # the device sums (u = 2^-24); over T rounds (a lost or doubled apply leaves a whole delta)
            wa, wb = (p.cpu().numpy().astype(np.float64) for p in params)
            wmag = np.maximum(np.maximum(np.abs(w_start), np.abs(wa)), np.abs(wb))
            u = 2.0 ** -24
            bound = T * (2 * 2 * u * 2 * wmag + 3 * u * da) + 1e-30
            assert np.all(np.abs(ds) <= bound), (np.max(np.abs(ds) / bound), np.max(np.abs(ds)))
            # averaging kept the replicas close: before the final average they differ by less
            # than one interval of training (compare the replicas' distance to the total motion)
            moved = np.abs(wa - w_start).max()
            assert np.abs(wa - wb).max() < 0.5 * moved, (np.abs(wa - wb).max(), moved)
        torch.cuda.synchronize()
        avg = (params[0] + params[1]) * 0.5
        params[0].copy_(avg)
        params[1].copy_(avg)
        torch.cuda.synchronize()
    np.testing.assert_array_equal(nets[0].get_params(), nets[1].get_params())
    Xt = torch.from_numpy(d.x_test).cuda()
    Yt = torch.from_numpy(d.y_test).cuda()
    ml, ne = nets[0].evaluate(Xt, Yt)
    ref = rec["per_epoch"][-1]
    assert abs(ne - ref["test_errors"]) / len(d.y_test) * 100 <= 0.5, (ne, ref)
    for net in nets:
        net.close()


@pytest.mark.parametrize("comm", [0, 2])
def test_single_replica_launch_path(comm, torch_cuda):
    # the multi-GPU launch path (chaos_train_epoch with armed rounds) at R = 1: the average of one
    # replica is itself (zero deltas), rounds are counted, training runs normally
    import torch
    from paper_1506_09067_b200 import OPT_DEBUG_CLAIMS, OPT_PAVG_COMM_CTAS, Net
    net = Net(sd.ARCHS["large"], init_seed=5)
    net.set_option(OPT_PAVG_COMM_CTAS, comm)
    net.pavg_setup(0, 1, 256, 16 if comm else 0)
    net.pavg_set_check(True)
    d = sd.prototype_dataset(5, 5000, 0)
    X, Y = torch.from_numpy(d.x_train).cuda(), torch.from_numpy(d.y_train).cuda()
    w0 = net.get_params()
    net.pavg_arm(19)
    net.train_epoch(X, Y, 0.0)
    net.sync()
    np.testing.assert_array_equal(net.get_params(), w0)
    assert net.pavg_rounds_done() == 19
    ds, da = net.pavg_debug_sums()
    assert np.all(ds == 0) and np.all(da == 0)
    net.pavg_arm(19)
    net.set_option(OPT_DEBUG_CLAIMS, 1)
    net.train_epoch(X, Y, 0.001)
    net.sync()
    assert np.abs(net.get_params() - w0).max() > 0
    assert net.pavg_rounds_done() == 38
    np.testing.assert_array_equal(net.debug_claims(5000), np.ones(5000, np.int32))  # every image once
    net.set_option(OPT_DEBUG_CLAIMS, 0)
    # unarmed launches run no rounds
    net.train_epoch(X, Y, 0.001)
    net.sync()
    assert net.pavg_rounds_done() == 38
    net.close()


def test_pavg_argument_errors(torch_cuda):
    import torch
    from paper_1506_09067_b200 import ChaosError, Net
    a, b = Net(sd.ARCHS["large"], init_seed=1), Net(sd.ARCHS["large"], init_seed=2)
    with pytest.raises(ChaosError):
        a.pavg_arm(1)  # no setup
    with pytest.raises(ChaosError):
        a.pavg_setup(0, 9, 1024)  # world > 8
    with pytest.raises(ChaosError):
        a.pavg_setup(2, 2, 1024)  # rank outside the world
    a.pavg_setup(0, 2, 1024)
    b.pavg_setup(1, 2, 1024)
    with pytest.raises(ChaosError):
        a.pavg_setup(0, 2, 1024)  # twice
    d = sd.prototype_dataset(1, 400, 0)
    X, Y = torch.from_numpy(d.x_train).cuda(), torch.from_numpy(d.y_train).cuda()
    a.pavg_arm(1)
    with pytest.raises(ChaosError):
        a.train_epoch(X, Y, 0.0)  # rank 1's exchange buffer missing
    with pytest.raises(ChaosError):
        type(a).train_epoch_replicas([a, a], [X, X], [Y, Y], 0.0)  # the same net twice
    for net in (a, b):
        net.close()
    tiny = Net(sd.ARCHS["tiny"], init_seed=1)
    with pytest.raises(ChaosError):  # no replica-emulation build for this net
        type(tiny).train_epoch_replicas([tiny], [X], [Y], 0.0)
    tiny.close()


IPC_CHILD = r"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, {root!r})
import synthdata as sd
from paper_1506_09067_b200 import Net
from paper_1506_09067_b200.chaos import _CudaArray
rank, ddir = int(sys.argv[1]), sys.argv[2]
net = Net(sd.ARCHS["large"], init_seed=rank)
net.pavg_setup(rank, 2, 1024)
ptr, nbytes = net.pavg_exchange()
own = torch.as_tensor(_CudaArray(ptr, 4096), device="cuda")
own.copy_(torch.arange(4096, dtype=torch.float32, device="cuda") + 1000.0 * (rank + 1))
torch.cuda.synchronize()
open(f"{{ddir}}/h{{rank}}.tmp", "wb").write(net.pavg_ipc_handle())
import os
os.rename(f"{{ddir}}/h{{rank}}.tmp", f"{{ddir}}/h{{rank}}")
peer = 1 - rank
while not os.path.exists(f"{{ddir}}/h{{peer}}"):
    time.sleep(0.05)
net.pavg_open_peer(peer, open(f"{{ddir}}/h{{peer}}", "rb").read())
pptr, pbytes = net.pavg_exchange(peer)
assert pbytes == nbytes and pptr != ptr
got = torch.as_tensor(_CudaArray(pptr, 4096), device="cuda").cpu().numpy()
want = np.arange(4096, dtype=np.float32) + 1000.0 * (peer + 1)
assert np.array_equal(got, want), (got[:4], want[:4])
open(f"{{ddir}}/ok{{rank}}", "w").write("ok")
while not os.path.exists(f"{{ddir}}/ok{{peer}}"):  # the peer's mapping of our buffer is done
    time.sleep(0.05)
net.close()
print("ipc ok", rank)
"""


def test_ipc_exchange_buffers_between_processes(tmp_path, torch_cuda):
    # the multi-GPU plumbing on one GPU, without kernels that wait on one another: two processes
    # each set up rank r of 2, publish their exchange buffer's CUDA IPC handle, map the peer's
    # (chaos_pavg_open_peer) and read the pattern the peer wrote into it
    script = tmp_path / "child.py"
    script.write_text(IPC_CHILD.format(root=ROOT))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(tmp_path)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"ipc ok {r}" in out, out[-2000:]


def test_dead_peer_times_out_instead_of_hanging(torch_cuda):
    # rank 0 of 2 whose peer never launches (a dead rank): the launch's rounds wait ~10 s, are given
    # up, and the next synchronizing call reports the latched error -- no hang
    import time

    import torch
    from paper_1506_09067_b200 import ChaosError, Net
    a, b = Net(sd.ARCHS["large"], init_seed=1), Net(sd.ARCHS["large"], init_seed=2)
    a.pavg_setup(0, 2, 256)
    b.pavg_setup(1, 2, 256)
    a.pavg_set_peer(1, b)
    d = sd.prototype_dataset(1, 2000, 0)
    X, Y = torch.from_numpy(d.x_train).cuda(), torch.from_numpy(d.y_train).cuda()
    a.pavg_arm(3)
    t = time.time()
    a.train_epoch(X, Y, 0.001)
    with pytest.raises(ChaosError, match="waited"):
        a.sync()
    assert time.time() - t < 120
    assert np.isfinite(a.get_params()).all()
    for net in (a, b):
        net.close()
