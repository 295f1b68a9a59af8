"""Debug probe of the NEXT-1 peer-memory path: `world` processes on cuda:0 (CUDA IPC), one
P2P model each; prints the step flags after every phase of two epochs."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2512_01678_b200 as P
    from synth.generate import make_small
    n = 3000
    w = make_small(n, 36000, 40, 5, seed=3, alpha=2.1, mu=0.3)
    gfull = P.Graph(w["src"], w["dst"], n)
    rp, ci = (t.cpu().numpy() for t in gfull.csr()[:2])
    bounds = P.partition_1d(rp, world)
    plan = P.Plan(rp, ci, n, bounds, rank)
    g = P.Graph.from_plan(plan)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    f = P.Features(torch.from_numpy(np.ascontiguousarray(w["X"][r0:r1])).cuda(), force_mode=0)
    m = P.GCN(g, f, (40, 32, 5), comm="p2p")
    m.init_xavier(42)
    m.set_labels(torch.from_numpy(np.ascontiguousarray(w["y"][r0:r1])).cuda(), n_lab_global=n)

    def show(tag):
        t0 = time.time()
        e, gen, fl = m.p2p_status(detail=True)
        print(f"[r{rank}] {tag:10s} err={e} gen={gen} halo={fl[0].tolist()} loss={fl[1].tolist()} "
              f"grad={fl[2].tolist()} setup={fl[3].tolist()} ({time.time() - t0:.2f}s)", flush=True)

    show("opened")
    dist.barrier()
    for t in (1, 2):
        m.forward(t)
        show(f"fwd{t}")
        lo = m.loss()
        show(f"loss{t}")
        m.backward()
        show(f"bwd{t}")
        m.adam(t)
        show(f"adam{t}")
        print(f"[r{rank}] loss{t} = {lo.item()}", flush=True)
    dist.barrier()
    del m
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(world, port), nprocs=world)
