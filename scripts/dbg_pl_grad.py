"""Debug: paper_large batch gradients vs the oracle for several batch sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from helpers import parity_report  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_1506_09067_b200 import Net  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "paper_large"
o = Oracle(sd.ARCHS[name])
p = sd.init_params(5, o.blocks())
d = sd.prototype_dataset(5, 64, 0)
for n in (1, 13, 20, 40, 64):
    net = Net(sd.ARCHS[name], init_seed=5)
    net.set_params(p)
    X, Y = torch.from_numpy(d.x_train[:n]).cuda(), torch.from_numpy(d.y_train[:n]).cuda()
    g = net.compute_gradients(X, Y)
    ref = np.zeros(o.n_params)
    for i in range(n):
        ref += o.sample_grad(p, d.x_train[i], d.y_train[i])[1]
    ok, w, wn, det = parity_report(g, ref, o.blocks())
    print(n, ok, round(w, 3), round(wn, 3), [round(x[1], 2) for x in det], flush=True)
    net.close()
