"""Time the aggregation SpMM alone on a BASELINE workload's graph, one mph_spmm call of width w
(row stride ld) per shape, CUDA events over 20 calls after 5 warm-ups; the graph (and so its work
items) is built under the current MPH_SPMM_SPLIT / MPH_SPMM_CHUNK_EDGES.
Usage: python tools/spmm_items_bench.py products 256:256,104:104,48:48"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from synth.generate import make_workload  # noqa: E402

name = sys.argv[1]
shapes = [tuple(int(x) for x in s.split(":")) for s in sys.argv[2].split(",")]
wl = make_workload(name)
n = wl["cfg"].num_nodes
g = P.Graph(wl["src"], wl["dst"], n)
del wl
tag = f"split={os.environ.get('MPH_SPMM_SPLIT', '1')} chunk={os.environ.get('MPH_SPMM_CHUNK_EDGES', 'default')}"
for w, ld in shapes:
    T = torch.randn((n, ld), device="cuda")
    out = torch.zeros((n, ld), device="cuda")
    for _ in range(5):
        g.spmm(T, out, w=w)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.spmm(T, out, w=w)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} w={w} ld={ld} {tag}: {e0.elapsed_time(e1) / 20:.4f} ms per call", flush=True)
    del T, out
