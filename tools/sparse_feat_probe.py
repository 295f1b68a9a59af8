"""Time mph_sparse_xw and mph_sparse_xtg separately on one calibration shape (diagnostic)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_01678_b200 as P  # noqa: E402
from paper_2512_01678_b200 import _lib as L  # noqa: E402
from tools.calibrate_gamma import _timed, uniform_csr  # noqa: E402
from synth.generate import make_workload  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "nell"
    if which == "nell":
        w = make_workload("nell")
        ptr, idx, val = w["X_csr"]
        N, F, H = w["cfg"].num_nodes, w["cfg"].num_features, 32
    else:
        N, F, H, d = 131072, 512, 128, 0.1
        ptr, idx, val = uniform_csr(N, F, d, 3)
    sid = torch.cuda.current_stream().cuda_stream
    fs = P.Features.from_csr(ptr, idx, val, (N, F), force_mode=1)
    rng = np.random.default_rng(0)
    W = torch.from_numpy(rng.standard_normal((F, H)).astype(np.float32)).cuda()
    G = torch.from_numpy(rng.standard_normal((N, H)).astype(np.float32)).cuda()
    ones = torch.ones(N, device="cuda")
    T = torch.empty((N, H), device="cuda")
    dW = torch.empty((F, H), device="cuda")
    flush = torch.zeros(128 << 20, device="cuda")
    txw = _timed(lambda: L.mph_sparse_xw(fs.h, W.data_ptr(), H, H, ones.data_ptr(), T.data_ptr(), H, sid), flush, 10)
    txg = _timed(lambda: L.mph_sparse_xtg(fs.h, G.data_ptr(), H, H, dW.data_ptr(), H, sid), flush, 10)
    nnz = val.size
    print(f"{which}: nnz {nnz} xw {txw:.3f} ms ({nnz * H * 4 / txw / 1e9:.0f} GB/s gathered)  "
          f"xtg {txg:.3f} ms ({nnz * H * 4 / txg / 1e9:.0f} GB/s gathered)")


if __name__ == "__main__":
    main()
