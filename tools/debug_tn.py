"""Decode the element mapping of k_gemm_tn with one-hot operands."""
import ctypes as C
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_01678_b200 as P  # noqa: F401
from paper_2512_01678_b200._lib import mph_gemm_tn, mph_gemm_tn_workspace


def run(A, B):
    K, M = A.shape
    N = B.shape[1]
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    wsb = C.c_size_t()
    mph_gemm_tn_workspace(M, N, K, C.byref(wsb))
    ws = torch.empty(wsb.value // 4 + 1, device="cuda")
    c = torch.zeros((M, N), device="cuda")
    mph_gemm_tn(M, N, K, a.data_ptr(), M, b.data_ptr(), N, c.data_ptr(), N, ws.data_ptr(), wsb.value,
                torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return c.cpu().numpy()


for (M, N, K) in [(128, 32, 32), (16, 16, 100), (256, 64, 64)]:
    print("shape", M, N, K)
    for (m0, n0, k0) in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (5, 0, 0), (0, 5, 0), (0, 0, 5), (0, 0, 8),
                         (9, 0, 0), (0, 9, 0), (33, 0, 0), (0, 33, 0), (0, 0, 9), (3, 7, 13), (70, 20, 31)]:
        if m0 >= M or n0 >= N or k0 >= K:
            continue
        A = np.zeros((K, M), np.float32)
        B = np.zeros((K, N), np.float32)
        A[k0, m0] = 1
        B[k0, n0] = 1
        Cm = run(A, B)
        nz = np.argwhere(Cm != 0)
        print(f"  a[{k0},{m0}] b[{k0},{n0}] -> expect C[{m0},{n0}]; got {nz.tolist()[:6]} vals {Cm[Cm != 0][:6]}")
    rng = np.random.default_rng(0)
    A = rng.standard_normal((K, M)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    Cm = run(A, B)
    ref = A.T.astype(np.float64) @ B
    err = np.abs(Cm - ref)
    print("  random max err", err.max(), "where", np.unravel_index(err.argmax(), err.shape), "rel",
          err.max() / np.abs(ref).max())
