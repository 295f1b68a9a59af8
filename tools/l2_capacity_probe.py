"""Effective L2 capacity for random-row gathers on this GPU: the gather probe (mph_probe_gather,
512-B rows) over uniform random row ids drawn from a working set of S MB, for S from 8 MB to
1 GB, with the rows packed (stride 512 B) or every other 512-B row of a 1 KB-stride table (the
access pattern of a 128-wide column slab of a 256-wide operand).  The rate falls from the
L2-hit to the HBM-miss level as S passes the capacity the gathers actually get."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_01678_b200 import _lib as L  # noqa: E402

W = 128
n_idx = 1 << 25
out = torch.zeros(148 * 32 * 128, device="cuda")
res = []
big = torch.randn((1 << 30) // 4, device="cuda")     # 1 GB table (flat)
gen = torch.Generator(device="cuda").manual_seed(0)
for mb in (8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 160, 256, 512):
    for stride in (1, 2):
        rows = mb * (1 << 20) // (W * 4)             # rows touched
        if rows * stride * W * 4 > big.numel() * 4:
            continue
        idx = (torch.randint(0, rows, (n_idx,), device="cuda", generator=gen, dtype=torch.int32) * stride)
        table_rows = rows * stride
        for _ in range(3):
            L.mph_probe_gather(big.data_ptr(), table_rows, W, idx.data_ptr(), n_idx, out.data_ptr(), None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            L.mph_probe_gather(big.data_ptr(), table_rows, W, idx.data_ptr(), n_idx, out.data_ptr(), None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gbs = n_idx * W * 4 / ms / 1e6
        res.append({"working_set_MB": mb, "row_stride_B": 512 * stride, "ms": ms, "gather_GBps": gbs})
        print(f"working set {mb:4d} MB stride {512 * stride:4d} B: {gbs:8.0f} GB/s", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/l2_capacity_probe.json", "w"), indent=1)
