"""Sweep the SpMM per-round unroll U (MPH_SPMM_U_<LPR>_<VPL>) on one workload: build the model
once, then time epochs for each setting; prints the SpMM ms/epoch per setting."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from paper_2512_01678_b200 import _lib as L  # noqa: E402
from synth.generate import make_workload  # noqa: E402

cfgname = sys.argv[1]
shape = sys.argv[2]                     # e.g. 32_1
values = [int(v) for v in sys.argv[3].split(",")]
w = make_workload(cfgname)
cfg = w["cfg"]
g = P.Graph(w["src"], w["dst"], cfg.num_nodes)
f = P.Features(torch.from_numpy(w["X"]).cuda())
m = P.GCN(g, f, cfg.dims)
m.init_xavier(42)
m.set_labels(torch.from_numpy(w["y"]).cuda())
t = 0
for rep in range(2):
    for u in values:
        os.environ[f"MPH_SPMM_U_{shape}"] = str(u)
        for _ in range(3):
            t += 1
            m.train_epoch(t)
        torch.cuda.synchronize()
        L.mph_profile_enable(1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(10):
            t += 1
            m.train_epoch(t)
        ev1.record()
        torch.cuda.synchronize()
        cnt, tms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        L.mph_profile_read(0, C.byref(cnt), C.byref(tms), C.byref(by), C.byref(fl))
        L.mph_profile_enable(0)
        print(f"{cfgname} U_{shape}={u:2d} epoch {ev0.elapsed_time(ev1) / 10:.3f} ms  spmm {tms.value / 10:.3f} ms",
              flush=True)
