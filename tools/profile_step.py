"""Run W warm-up + K training epochs of one config (no timing, no CPU baseline): the command
ncu wraps for the launch list and the --set full captures under profiles/."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from synth.generate import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="reddit")
ap.add_argument("--epochs", type=int, default=3)
ap.add_argument("--agg", default="gcn", choices=["gcn", "sum", "mean", "max"])
ap.add_argument("--precision", default="tf32", choices=["tf32", "bf16"])
a = ap.parse_args()
w = make_workload(a.config)
cfg = w["cfg"]
g = P.Graph(w["src"], w["dst"], cfg.num_nodes)
if w["X"] is not None:
    f = P.Features(torch.from_numpy(w["X"]).cuda())
else:
    ptr, idx, val = w["X_csr"]
    f = P.Features.from_csr(ptr, idx, val, (cfg.num_nodes, cfg.num_features))
m = P.GCN(g, f, cfg.dims, aggregator=a.agg, precision=a.precision)
m.init_xavier(42)
m.set_labels(torch.from_numpy(w["y"]).cuda())
torch.cuda.synchronize()
for t in range(1, a.epochs + 1):
    m.train_epoch(t)
torch.cuda.synchronize()
print("loss", m.loss_buf.item())
