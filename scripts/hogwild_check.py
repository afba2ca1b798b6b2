"""Hogwild sanity checks (debug): 1-worker == sequential SGD parity ratio, and tiny config1 epoch losses.
    CHAOS_LIB=... python scripts/hogwild_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from helpers import parity_report  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_1506_09067_b200 import OPT_GROUP, OPT_MAX_CTAS, Net  # noqa: E402

print("lib", os.environ.get("CHAOS_LIB", "default"))
for name in ["large", "medium", "tiny"]:
    o = Oracle(sd.ARCHS[name])
    p = sd.init_params(9, o.blocks())
    d = sd.prototype_dataset(9, 24, 0)
    ref, _ = o.train_sgd(p, d.x_train, d.y_train, 0.05)
    for rep in range(2):
        net = Net(sd.ARCHS[name], init_seed=9)
        net.set_option(OPT_GROUP, 1)
        net.set_option(OPT_MAX_CTAS, 1)
        net.set_params(p)
        X, Y = torch.from_numpy(d.x_train).cuda(), torch.from_numpy(d.y_train).cuda()
        net.train_epoch(X, Y, 0.05)
        ok, w, wn, det = parity_report(net.get_params(), ref, o.blocks())
        print(name, "1-worker", "ok" if ok else "FAIL", round(w, 2), [round(x[1], 1) for x in det])
        net.close()
w = sd.WORKLOADS["config1"]
dd = sd.make_dataset(w)
X, Y, Xt, Yt = [torch.from_numpy(a).cuda() for a in (dd.x_train, dd.y_train, dd.x_test, dd.y_test)]
for rep in range(3):
    net = Net(sd.ARCHS["tiny"], init_seed=w.seed)
    c = []
    for e in range(3):
        net.train_epoch(X, Y, w.lr0 * 0.9 ** e)
        c.append(net.evaluate(Xt, Yt))
    print("tiny config1 hogwild", [(round(a, 4), b) for a, b in c])
    net.close()
