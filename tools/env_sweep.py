"""A/B experiment knobs on one workload: build the model once, then for each setting of the given
environment variables (read by the library at each launch) time 10 epochs after 3 warm-up epochs;
prints ms/epoch and the SpMM's share.  Two passes over the settings (box noise).

Usage: python tools/env_sweep.py products MPH_SPMM_HOTMB=0,64 [MPH_SPMM_L2POL=0,1] [--precision bf16]"""
import ctypes as C
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from paper_2512_01678_b200 import _lib as L  # noqa: E402
from synth.generate import make_workload  # noqa: E402

cfgname = sys.argv[1]
prec = "tf32"
knobs = []
for a in sys.argv[2:]:
    if a.startswith("--precision"):
        prec = a.split("=")[1]
        continue
    k, v = a.split("=")
    knobs.append((k, v.split(",")))
w = make_workload(cfgname)
cfg = w["cfg"]
g = P.Graph(w["src"], w["dst"], cfg.num_nodes)
f = P.Features(torch.from_numpy(w["X"]).cuda())
m = P.GCN(g, f, cfg.dims, precision=prec)
m.init_xavier(42)
m.set_labels(torch.from_numpy(w["y"]).cuda())
t = 0
for rep in range(2):
    for combo in itertools.product(*[v for _, v in knobs]):
        for (k, _), v in zip(knobs, combo):
            os.environ[k] = v
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
        per = {}
        for kind, kname in ((0, "spmm"), (1, "gemm_nt"), (2, "gemm_tn")):
            cnt, tms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            L.mph_profile_read(kind, C.byref(cnt), C.byref(tms), C.byref(by), C.byref(fl))
            per[kname] = (tms.value / 10, cnt.value // 10)
        L.mph_profile_enable(0)
        name = " ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo))
        print(f"{cfgname} {prec} {name}: epoch {ev0.elapsed_time(ev1) / 10:.3f} ms  spmm {per['spmm'][0]:.3f} ms "
              f"({per['spmm'][1]} launches)  gemm_nt {per['gemm_nt'][0]:.3f}  gemm_tn {per['gemm_tn'][0]:.3f}",
              flush=True)
