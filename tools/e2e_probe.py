"""Timeline of the pipelined end-to-end step (diagnostic): CUDA events around each feature copy
(copy stream) and each epoch (compute stream), reddit workload."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_01678_b200 as P  # noqa: E402
from paper_2512_01678_b200 import _lib as L  # noqa: E402
from synth.generate import make_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    w = make_workload(name)
    cfg = w["cfg"]
    n = cfg.num_nodes
    g = P.Graph(w["src"], w["dst"], n)
    f = P.Features(torch.from_numpy(w["X"]).cuda())
    m = P.GCN(g, f, cfg.dims)
    m.init_xavier(42)
    y = torch.from_numpy(w["y"]).cuda()
    m.set_labels(y)
    Pw = P.pad_width(w["X"].shape[1])
    Xh = torch.zeros((n, Pw), dtype=torch.float32).pin_memory()
    Xh[:, :w["X"].shape[1]] = torch.from_numpy(w["X"])
    s = torch.cuda.current_stream()
    cs = torch.cuda.Stream()
    for t in range(1, 4):
        m.train_epoch(t)
    torch.cuda.synchronize()
    # copy alone
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(cs)
    with torch.cuda.stream(cs):
        L.mph_gcn_upload_features_async(m.h, Xh.data_ptr(), Pw, cs.cuda_stream, s.cuda_stream)
    ev[1].record(cs)
    torch.cuda.synchronize()
    print("copy alone ms", ev[0].elapsed_time(ev[1]))
    # epoch alone
    ev[0].record(s)
    m.train_epoch(4)
    ev[1].record(s)
    torch.cuda.synchronize()
    print("epoch alone ms", ev[0].elapsed_time(ev[1]))
    # pipelined
    K = 6
    base = torch.cuda.Event(enable_timing=True)
    cps = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    eps = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    base.record(s)

    def load(i):
        cps[i][0].record(cs)
        L.mph_gcn_upload_features_async(m.h, Xh.data_ptr(), Pw, cs.cuda_stream, s.cuda_stream)
        cps[i][1].record(cs)

    load(0)
    t0 = time.perf_counter()
    for i in range(K):
        eps[i][0].record(s)
        m.train_epoch(10 + i)
        eps[i][1].record(s)
        done = torch.cuda.Event()
        done.record(s)
        if i + 1 < K:
            load(i + 1)
        done.synchronize()
    torch.cuda.synchronize()
    print("host wall per step ms", (time.perf_counter() - t0) * 1e3 / K)
    for i in range(K):
        print(f"step {i}: copy {base.elapsed_time(cps[i][0]):8.2f} -> {base.elapsed_time(cps[i][1]):8.2f}   "
              f"epoch {base.elapsed_time(eps[i][0]):8.2f} -> {base.elapsed_time(eps[i][1]):8.2f}")
    # variants of the bench loop
    yh = torch.from_numpy(np.ascontiguousarray(w["y"])).pin_memory()
    lh = torch.zeros(1, dtype=torch.float64).pin_memory()
    d2h = torch.cuda.Stream()
    for variant in ("labels", "loss_same_stream", "loss_d2h_stream", "both"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)

        def load():
            L.mph_gcn_upload_features_async(m.h, Xh.data_ptr(), Pw, cs.cuda_stream, s.cuda_stream)
            if variant in ("labels", "both"):
                y.copy_(yh, non_blocking=True)

        load()
        for i in range(K):
            m.train_epoch(20 + i)
            ed = torch.cuda.Event()
            ed.record(s)
            if i + 1 < K:
                load()
            if variant == "loss_same_stream":
                lh.copy_(m.loss_buf, non_blocking=True)
                done = torch.cuda.Event()
                done.record(s)
            elif variant in ("loss_d2h_stream", "both"):
                d2h.wait_event(ed)
                with torch.cuda.stream(d2h):
                    lh.copy_(m.loss_buf, non_blocking=True)
                done = torch.cuda.Event()
                done.record(d2h)
            else:
                done = ed
            done.synchronize()
        s.wait_stream(d2h)
        e1.record(s)
        torch.cuda.synchronize()
        print(variant, "ms/step", e0.elapsed_time(e1) / K)


if __name__ == "__main__":
    main()
