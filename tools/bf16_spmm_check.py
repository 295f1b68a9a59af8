"""MPH_EPI_IN_BF16 check: aggregating a bfloat16 operand equals, bit for bit, aggregating the same
values widened to FP32 (the kernel widens exactly and sums in the same order), for each width."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_01678_b200 as P  # noqa: E402
from paper_2512_01678_b200._lib import Epilogue  # noqa: E402
from synth.generate import make_workload  # noqa: E402

for name in sys.argv[1:] or ["reddit"]:
    wl = make_workload(name)
    n = wl["cfg"].num_nodes
    g = P.Graph(wl["src"], wl["dst"], n)
    for w in (48, 64, 104, 128, 256):
        if w == 104 and name != "products":
            continue
        Tb = torch.randn((n, w), device="cuda").to(torch.bfloat16)
        o1 = torch.zeros((n, w), device="cuda")
        o2 = torch.zeros((n, w), device="cuda")
        g.spmm(Tb, o1, w=w, epi=Epilogue(flags=512))
        g.spmm(Tb.float(), o2, w=w)
        torch.cuda.synchronize()
        print(name, w, "bitwise equal" if torch.equal(o1, o2) else f"MISMATCH max {float((o1 - o2).abs().max())}",
              flush=True)
