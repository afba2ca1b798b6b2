"""Small runs of every kernel mode for compute-sanitizer (one tool per invocation):
    compute-sanitizer --tool racecheck python scripts/sanitize_run.py [arch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import OPT_MAX_CTAS, OPT_SYNC_BATCH, SYNC, Net  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "large"
d = sd.prototype_dataset(5, 40, 8)
X, Y = torch.from_numpy(d.x_train).cuda(), torch.from_numpy(d.y_train).cuda()
Xt, Yt = torch.from_numpy(d.x_test).cuda(), torch.from_numpy(d.y_test).cuda()
net = Net(sd.ARCHS[arch], init_seed=5)
net.set_option(OPT_MAX_CTAS, 2)
net.set_option(OPT_SYNC_BATCH, 16)
net.train_epoch(X, Y, 0.01, SYNC)
net.train_epoch(X, Y, 0.01)
print(arch, net.evaluate(Xt, Yt), float(net.forward(Xt).sum()))
net.sync()
print("ok")
