import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04083_b200 import graph, trainer as tr
ds = graph.synth_rmat(12, 40000, 100, 7, seed=4)
pre = graph.preprocess(ds, perm_seed=4)
outs = {}
for mode in (tr.PK_MODE_PARITY, tr.PK_MODE_FAST):
    opts = tr.TrainOptions(hidden_dims=[64, 64], mode=mode)
    eng = tr.RankEngine(pre.n, pre.feat_dim, pre.num_classes, tr.GridConfig(1, 1, 1), 0, opts)
    eng.load(pre)
    loss, _ = eng.forward_backward(0)
    outs[mode] = dict(loss=loss, H=[eng.tensor(tr.PK_T_H, l).cpu().numpy() for l in range(3)],
                      Q=[eng.tensor(tr.PK_T_Q, l).cpu().numpy() for l in range(3)])
    eng.close()
for l in range(3):
    for k in ("H", "Q"):
        a, b = outs[0][k][l], outs[1][k][l]
        print(l, k, a.shape, "parity absmax", np.abs(a).max(), "fast absmax", np.abs(b).max(),
              "maxdiff", np.abs(a - b).max())
print("loss", outs[0]["loss"], outs[1]["loss"])
