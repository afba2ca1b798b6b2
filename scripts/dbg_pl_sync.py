"""Debug: worst elements of the paper_large sync-steps comparison (tests/test_gpu_parity.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from helpers import split_blocks  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC, Net  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "paper_large"
o = Oracle(sd.ARCHS[name])
net = Net(sd.ARCHS[name], init_seed=7)
p = sd.init_params(7, o.blocks())
net.set_params(p)
nimg = int(sys.argv[2]) if len(sys.argv) > 2 else 150
net.set_option(OPT_SYNC_BATCH, 64)
d = sd.prototype_dataset(7, 150, 0)
X, Y = torch.from_numpy(d.x_train[:nimg]).cuda(), torch.from_numpy(d.y_train[:nimg]).cuda()
LR = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
net.train_epoch(X, Y, LR, SYNC)
got = net.get_params().astype(np.float64)
ref, _ = o.train_sync(p, d.x_train[:nimg], d.y_train[:nimg], LR, 64)
print("images", nimg)
for k, (g, r, p0) in enumerate(zip(split_blocks(got, o.blocks()), split_blocks(ref, o.blocks()),
                                   split_blocks(p.astype(np.float64), o.blocks()))):
    tol = 1e-4 * np.maximum(np.abs(r), 1e-2 * np.abs(r).max())
    ratio = np.abs(g - r) / tol
    i = int(np.argmax(ratio))
    step = r - p0
    print(f"tensor {k}: worst {ratio[i]:.3f}x at {i}: got {g[i]:.9g} ref {r[i]:.9g} p0 {p0[i]:.9g} "
          f"step {step[i]:.3g} |step|max {np.abs(step).max():.3g} |r|max {np.abs(r).max():.3g} "
          f"step-rel-err {abs((g[i] - p0[i]) - step[i]) / max(abs(step[i]), 1e-30):.3g} "
          f"n>0.5: {(ratio > 0.5).sum()}")
