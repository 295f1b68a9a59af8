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
shapes = [(int(s.split(":")[0]), int(s.split(":")[1].rstrip("b")), s.endswith("b")) for s in sys.argv[2].split(",")]
knobs = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[3:]]
wl = make_workload(name)
n = wl["cfg"].num_nodes
g = P.Graph(wl["src"], wl["dst"], n)
nnz = g.nnz
del wl
from paper_2512_01678_b200._lib import Epilogue  # noqa: E402
for w, ld, bf in shapes:
    T = torch.randn((n, ld), device="cuda")
    if bf:   # round-2 experiment only: a bfloat16 operand needed the (reverted) MPH_EPI_IN_BF16 flag
        raise SystemExit("bf16 operands were a round-2 experiment (profiles/r02_experiments/spmm_bf16_operand.txt)")
    epi = None
    out = torch.zeros((n, ld), device="cuda")
    for rep in range(2):
        for combo in itertools.product(*[v for _, v in knobs]) if knobs else [()]:
            for (k, _), v in zip(knobs, combo):
                os.environ[k] = v
            for _ in range(5):
                g.spmm(T, out, w=w, epi=epi)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g.spmm(T, out, w=w, epi=epi)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            tag = " ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo))
            print(f"{name} w={w} ld={ld}{' bf16' if bf else ''} {tag}: {ms:.4f} ms  "
                  f"{nnz * (4 + (2 if bf else 4) * w) / ms / 1e9:.1f} TB/s no-reuse",
                  flush=True)
    del T, out
