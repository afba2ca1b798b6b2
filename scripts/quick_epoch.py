"""Samples/s of one 60,000-image hogwild epoch for any compiled net (A/B helper; CHAOS_LIB picks
the library):  python scripts/quick_epoch.py paper_small"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import OPT_GROUP, Net  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "large"
w = sd.WORKLOADS["config3"]
xs, ys = sd.prototype_samples(w.seed, 0, 60000)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
net = Net(sd.ARCHS[arch], init_seed=w.seed)
if len(sys.argv) > 2:
    net.set_option(OPT_GROUP, int(sys.argv[2]))
best = 0.0
for r in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    net.train_epoch(X, Y, w.lr0 * 0.9 ** r)
    b.record()
    torch.cuda.synchronize()
    if r >= 2:
        best = max(best, 60000 / (a.elapsed_time(b) / 1e3))
print(f"{arch} G={net.launch_info()['group']}: {best:.0f} samples/s")
