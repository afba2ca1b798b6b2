"""Throughput of the fused in-kernel cross-replica averaging, emulated on ONE GPU:
R replicas of the large net in one cooperative launch (148 / R CTAs each), replica r training its
contiguous 1/R of the 60,000 configs[3] images (strong scaling), with in-kernel averaging rounds
every K claimed images (K in {256, 1024, 8192}) against the same launch without rounds; the
rounds run by the training CTAs between image groups (comm 0) or by 1-2 comm CTAs per replica.  The
replicas' rounds exchange through same-device memory here (no NVLink), so this measures the
kernel-side cost of the protocol (snapshots, flag waits, applies), not the interconnect.
    python scripts/pavg_emulation_bench.py [R]  -> one JSON line per configuration
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import OPT_PAVG_COMM_CTAS, Net  # noqa: E402
from paper_1506_09067_b200.dist import async_targets  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = sd.WORKLOADS["config3"]
xs, ys = sd.prototype_samples(w.seed, 0, 60000)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
edges = [(60000 * r // R) // 4 * 4 for r in range(R)] + [60000]
Xs = [X[edges[r]:edges[r + 1]] for r in range(R)]
Ys = [Y[edges[r]:edges[r + 1]] for r in range(R)]
n_min = min(edges[r + 1] - edges[r] for r in range(R))
for K, comm in ((0, 0), (256, 0), (1024, 0), (8192, 0), (256, 1), (1024, 1), (1024, 2), (8192, 1)):
    nets = [Net(sd.ARCHS["large"], init_seed=w.seed) for _ in range(R)]
    for net in nets:
        net.set_option(OPT_PAVG_COMM_CTAS, comm)
    if K:
        for r, net in enumerate(nets):
            net.pavg_setup(r, R, K, 8 * comm if comm else 0)
        for net in nets:
            for q, o in enumerate(nets):
                if o is not net:
                    net.pavg_set_peer(q, o)
    rounds = len(async_targets(n_min, K)) if K else 0
    best = 0.0
    for rep in range(5):
        if K:
            for net in nets:
                net.pavg_arm(rounds)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(nets[0].stream)
        Net.train_epoch_replicas(nets, Xs, Ys, w.lr0 * 0.9 ** rep)
        b.record(nets[0].stream)
        torch.cuda.synchronize()
        if rep >= 2:
            best = max(best, 60000 / (a.elapsed_time(b) / 1e3))
    for net in nets:
        net.sync()
    print(json.dumps({"replicas": R, "ctas_per_replica": 148 // R, "comm_ctas_per_replica": comm, "k": K or None,
                      "rounds_per_launch": rounds,
                      "samples_per_s": best}), flush=True)
    for net in nets:
        net.close()
