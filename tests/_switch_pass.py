"""Helper for tests/test_switches_gpu.py: one FAST engine pass on a small
RMAT graph with a transform-first last layer, under whatever PK_* switches
the environment sets; writes logits, dW and dF0 to the .npz path given."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_04083_b200 import graph, trainer as tr  # noqa: E402


def main(out):
    ds = graph.synth_rmat(13, 120000, 64, 13, seed=5)
    pre = graph.preprocess(ds, perm_seed=5)
    opts = tr.TrainOptions(hidden_dims=[96, 96], mode=tr.PK_MODE_FAST, hub_threshold=256)
    eng = tr.RankEngine(pre.n, pre.feat_dim, pre.num_classes, tr.GridConfig(1, 1, 1), 0, opts)
    eng.load(pre)
    loss, _ = eng.forward_backward(0)
    np.savez(out, loss=loss, logits=eng.tensor(tr.PK_T_FOUT).cpu().numpy(),
             df0=eng.tensor(tr.PK_T_DF0).cpu().numpy(),
             **{f"dw{l}": eng.tensor(tr.PK_T_DW, l).cpu().numpy() for l in range(3)})
    eng.close()


if __name__ == "__main__":
    main(sys.argv[1])
