"""One rank of a row-block sharded solve across processes, for
tests/test_multi_gpu.py under torchrun (one GPU per rank, NCCL):

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/shard_rank.py --N 16 [--local] [--peer]

Every rank builds its shard plan — from the global system, or with --local from only
its own rows (workloads.generate_rows of the stacked-slab workload C4w, G = world:
the weak-scaling layout) — runs GS(2), Bi-CGSTAB and GMRES(30) and rank 0 compares
the history and its rows of x with the oracle on the whole system (bit for bit).
Prints one JSON line on rank 0; exits 1 on a mismatch.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=16)
    ap.add_argument("--local", action="store_true")
    ap.add_argument("--fmt", default="sell")
    ap.add_argument("--peer", action="store_true", help="device-initiated reductions (peer_reduce)")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    comm = gsk.NcclComm()
    s = workloads.generate("C4w", N=a.N, param=world)  # small: every rank can hold it
    lo, hi = gsk.shard_rows(s["n"], world, rank)
    if a.local:
        loc = workloads.generate_rows("C4w", lo, hi, N=a.N, param=world)
        A = gsk.CSR(loc["row_ptr"], loc["col"], loc["val"])
        As, bs, _ = gsk.gs_scale(A, loc["b"], 2)
        SP = gsk.ShardedPlan(As, fmt=a.fmt, comm=comm, n_global=s["n"], peer_reduce=a.peer)
    else:
        A = gsk.CSR.from_system(s)
        As, bs, _ = gsk.gs_scale(A, s["b"], 2)
        bs = bs[lo:hi]
        SP = gsk.ShardedPlan(As, fmt=a.fmt, comm=comm, peer_reduce=a.peer)
    x1, h1, r1 = SP.bicgstab(bs, tol=1e-9, maxit=400)
    x2, h2, r2 = SP.gmres(bs, m=30, tol=1e-9, maxit=120)
    xs1 = [torch.empty(gsk.shard_rows(s["n"], world, r)[1] - gsk.shard_rows(s["n"], world, r)[0],
                       dtype=torch.float64, device="cuda") for r in range(world)]
    xs2 = [torch.empty_like(t) for t in xs1]
    dist.all_gather(xs1, x1)
    dist.all_gather(xs2, x2)
    ok = True
    if rank == 0:
        import oracle
        vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
        xo1, ho1, ro1 = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-9, 400)
        xo2, ho2, ro2 = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 30, 1e-9, 120)
        g1 = torch.cat(xs1).cpu().numpy()
        g2 = torch.cat(xs2).cpu().numpy()
        ok = (np.array_equal(h1, ho1) and np.array_equal(g1, xo1) and r1["status"] == ro1["status"]
              and np.array_equal(h2, ho2) and np.array_equal(g2, xo2) and r2["status"] == ro2["status"])
        print(json.dumps({"world": world, "local_input": a.local, "peer_reduce": a.peer, "n": s["n"], "bicgstab_its": r1["iterations"],
                          "gmres_its": r2["iterations"], "equal": bool(ok)}), flush=True)
    SP.close()
    comm.close()
    flag = torch.tensor([int(ok)], device="cuda")
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
