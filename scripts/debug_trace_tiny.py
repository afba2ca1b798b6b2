"""Debug: one recorded 3-worker tiny-net hogwild epoch; per group, the publish against the oracle
at the weights the group read (max abs difference per tensor).  CHAOS_LIB picks the library."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from helpers import split_blocks  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_1506_09067_b200 import OPT_DEBUG_STAGGER, OPT_DEBUG_TRACE, OPT_GROUP, OPT_MAX_CTAS, Net  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
stagger = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
n, lr, seed = 3, 0.5, 11
o = Oracle(sd.ARCHS[name])
for rep in range(3):
    net = Net(sd.ARCHS[name], init_seed=seed)
    net.set_option(OPT_GROUP, 1)
    p = sd.init_params(seed, o.blocks())
    net.set_params(p)
    net.set_option(OPT_MAX_CTAS, 3)
    net.set_option(OPT_DEBUG_TRACE, 1)
    net.set_option(OPT_DEBUG_STAGGER, stagger)
    d = sd.prototype_dataset(seed, n, 0)
    X, Y = torch.from_numpy(d.x_train).cuda(), torch.from_numpy(d.y_train).cuda()
    net.train_epoch(X, Y, lr)
    rec, pubs, reads = net.debug_trace(3, reads=True)
    for k in range(3):
        wf = reads[k, 0].astype(np.float64)
        wb = np.where(np.isnan(reads[k, 1]), reads[k, 0], reads[k, 1]).astype(np.float64)
        _, g = o.sample_grad2(wf, wb, d.x_train[k], d.y_train[k])
        diff = [float(np.abs(a - b).max()) for a, b in zip(split_blocks(pubs[k].astype(np.float64), o.blocks()),
                                                         split_blocks(-lr * g, o.blocks()))]
        print(f"rep {rep} group {k} worker {rec[k, 30]} iter {rec[k, 31]}: max|diff| per tensor {['%.2e' % x for x in diff]}"
              f"; fc-bias pub {np.round(pubs[k][-10:], 4)} oracle {np.round(-lr * g[-10:], 4)}")
    net.close()
