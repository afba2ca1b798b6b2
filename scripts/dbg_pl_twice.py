"""Debug: two identical gradient launches on one net must agree bitwise (sync mode is deterministic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import Net  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "paper_large"
d = sd.prototype_dataset(5, 64, 0)
net = Net(sd.ARCHS[name], init_seed=5)
for n in (64, 64, 13, 64):
    X, Y = torch.from_numpy(d.x_train[:n]).cuda(), torch.from_numpy(d.y_train[:n]).cuda()
    g = net.compute_gradients(X, Y)
    if n == 64:
        if 'g0' in dir():
            diff = np.abs(g - g0)
            print("repeat 64: max diff", diff.max(), "n diff", (diff > 0).sum(), "first idx", np.nonzero(diff)[0][:5])
        else:
            g0 = g
