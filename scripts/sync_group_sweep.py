import sys, os, torch
sys.path.insert(0, "/root/repo")
import synthdata as sd
from paper_1506_09067_b200 import Net, SYNC, OPT_GROUP, OPT_SYNC_BATCH
w = sd.WORKLOADS["config3"]
xs, ys = sd.prototype_samples(w.seed, 0, 60000)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
for arch in ("large", "medium", "tiny"):
    for g in (1, 4):
        net = Net(sd.ARCHS[arch], init_seed=w.seed)
        try:
            net.set_option(OPT_GROUP, g)
        except Exception as e:
            print(arch, g, "n/a"); continue
        net.set_option(OPT_SYNC_BATCH, 64)
        best = 0
        for r in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); net.train_epoch(X, Y, 0.001, SYNC); b.record(); torch.cuda.synchronize()
            best = max(best, 60000 / (a.elapsed_time(b) / 1e3))
        print(arch, "G", g, "sync B=64:", round(best))
        net.close()
