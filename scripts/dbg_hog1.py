import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import synthdata as sd
from helpers import parity_report
from oracle import Oracle
from paper_1506_09067_b200 import OPT_GROUP, OPT_MAX_CTAS, OPT_SYNC_BATCH, SYNC, Net
o = Oracle(sd.ARCHS['large']); p = sd.init_params(9, o.blocks()); d = sd.prototype_dataset(9, 24, 0)
for G in (1,):
  for n in (10, 12, 16, 20, 24):
    ref, _ = o.train_sgd(p, d.x_train[:n], d.y_train[:n], 0.05)
    for mode in ('hog', 'sync1'):
        net = Net(sd.ARCHS['large'], init_seed=9); net.set_option(OPT_GROUP, G); net.set_option(OPT_MAX_CTAS, 1); net.set_params(p)
        X, Y = torch.from_numpy(d.x_train[:n]).cuda(), torch.from_numpy(d.y_train[:n]).cuda()
        if mode == 'hog': net.train_epoch(X, Y, 0.05)
        else:
            net.set_option(OPT_SYNC_BATCH, 1); net.train_epoch(X, Y, 0.05, SYNC)
        ok, w, wn, det = parity_report(net.get_params(), ref, o.blocks())
        print('G', G, 'n', n, mode, 'ok' if ok else 'FAIL', [round(x[1], 2) for x in det], flush=True)
        net.close()
