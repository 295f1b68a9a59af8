"""Print the exact loss bits of K epochs of a workload (for bitwise A/B of builds that must not
change any result).  Usage: python tools/loss_digest.py arxiv 6"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from synth.generate import make_workload  # noqa: E402

name, K = sys.argv[1], int(sys.argv[2])
w = make_workload(name)
cfg = w["cfg"]
g = P.Graph(w["src"], w["dst"], cfg.num_nodes)
f = P.Features(torch.from_numpy(w["X"]).cuda())
m = P.GCN(g, f, cfg.dims, dropout_p=0.1, dropout_seed=3)
m.init_xavier(42)
m.set_labels(torch.from_numpy(w["y"]).cuda())
ls = [m.train_epoch(t).item() for t in range(1, K + 1)]
print(name, "losses", " ".join(float(x).hex() for x in ls), "params sum", float(m.params_flat.double().sum()).hex())
