"""Time the aggregation SpMM alone on a BASELINE workload's graph: random operand of width w with
row stride ld (CUDA events over 20 launches after 5 warm-ups), for each setting of the given
environment knobs.  Usage: python tools/spmm_bench.py reddit 48:48,48:64 [KNOB=v1,v2 ...]"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from synth.generate import make_workload  # noqa: E402

name = sys.argv[1]
shapes = [tuple(int(x) for x in s.split(":")) for s in sys.argv[2].split(",")]
knobs = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[3:]]
wl = make_workload(name)
n = wl["cfg"].num_nodes
g = P.Graph(wl["src"], wl["dst"], n)
nnz = g.nnz
del wl
for w, ld in shapes:
    T = torch.randn((n, ld), device="cuda")
    out = torch.zeros((n, ld), device="cuda")
    for rep in range(2):
        for combo in itertools.product(*[v for _, v in knobs]) if knobs else [()]:
            for (k, _), v in zip(knobs, combo):
                os.environ[k] = v
            for _ in range(5):
                g.spmm(T, out, w=w)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g.spmm(T, out, w=w)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            tag = " ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo))
            print(f"{name} w={w} ld={ld} {tag}: {ms:.4f} ms  {nnz * (4 + 4 * w) / ms / 1e9:.0f} GB/s no-reuse",
                  flush=True)
    del T, out
