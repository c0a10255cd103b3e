"""Host logic of row-block sharding (include/gsk.h gsk_shard_rows / gsk_shard_halo_host,
DESIGN.md §8) — no GPU: the layout, the halo widths, and, over a world_size-2 gloo
group, that the sharded SpMV (halo exchange + local rows) and the sharded dot
(per-shard canonical subtree + tree over shards) reproduce the global oracle results
bit for bit.  The GPU side runs the same layout (tests/test_gpu_parity.py)."""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)  # spawned gloo workers re-import this module
import oracle  # noqa: E402
import workloads  # noqa: E402

gsk = pytest.importorskip("paper_0812_2769_b200")


@pytest.mark.parametrize("n", [1000, 1024, 13824, 4097, 16777216])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_shard_rows_partition(n, P):
    N = 1 << (n - 1).bit_length()
    B = N // P
    if (P - 1) * B >= n:  # the last shard would be empty: rejected
        with pytest.raises(gsk.GskError):
            gsk.shard_rows(n, P, 0)
        return
    his = []
    for r in range(P):
        lo, hi = gsk.shard_rows(n, P, r)
        assert lo == r * B and hi == min(n, (r + 1) * B) and hi > lo
        his.append(hi)
    assert his[-1] == n


def test_shard_rows_errors():
    for n, P, r in [(1000, 3, 0), (1000, 64, 0), (5, 8, 0), (1000, 2, 2), (0, 1, 0)]:
        with pytest.raises(gsk.GskError):
            gsk.shard_rows(n, P, r)


def _halo_brute(s, P, r):
    lo, hi = gsk.shard_rows(s["n"], P, r)
    cols = s["col"][s["row_ptr"][lo]:s["row_ptr"][hi]]
    return max(0, lo - int(cols.min())), max(0, int(cols.max()) - (hi - 1))


@pytest.mark.parametrize("name,N,P", [("C1", None, 8), ("C2", 64, 4), ("C3", 16, 4), ("C4", 24, 2), ("C4", 24, 4),
                                      ("C5", 64, 2)])
def test_shard_halo_widths(name, N, P):
    s = workloads.generate(name, N=N)
    for r in range(P):
        assert gsk.shard_halo(s["row_ptr"], s["col"], P, r) == _halo_brute(s, P, r)


def test_shard_halo_rejects_non_adjacent():
    s = workloads.generate("C5", N=64)  # random symmetric permutation: halos span the grid
    with pytest.raises(gsk.GskError):
        for r in range(8):
            gsk.shard_halo(s["row_ptr"], s["col"], 8, r)


def _local_system(s, P, r):
    lo, hi = gsk.shard_rows(s["n"], P, r)
    hl, hr = gsk.shard_halo(s["row_ptr"], s["col"], P, r)
    rp = s["row_ptr"][lo:hi + 1] - s["row_ptr"][lo]
    ci = s["col"][s["row_ptr"][lo]:s["row_ptr"][hi]] - lo + hl  # index into [hl | own | hr]
    val = s["val"][s["row_ptr"][lo]:s["row_ptr"][hi]]
    return lo, hi, hl, hr, rp, ci, val


def _tree(vals):
    """Top of the canonical tree over the shard values (P a power of two)."""
    v = list(vals)
    while len(v) > 1:
        v = [v[2 * k] + v[2 * k + 1] for k in range(len(v) // 2)]
    return v[0] + 0.0


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    out = {}
    for name, N in (("C3", 12), ("C4", 20), ("C2", 40)):
        s = workloads.generate(name, N=N)
        lo, hi, hl, hr, rp, ci, val = _local_system(s, world, rank)
        x = workloads.uniform(s["n"], 11, 12)
        own = torch.tensor(x[lo:hi])
        ext = torch.zeros(hl + (hi - lo) + hr, dtype=torch.float64)
        ext[hl:hl + hi - lo] = own
        # halo exchange with the neighbours (the library does this with ncclSend/Recv)
        nb = [gsk.shard_halo(s["row_ptr"], s["col"], world, r) for r in range(world)]
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(own[:nb[rank - 1][1]].contiguous(), rank - 1))
            left = torch.empty(hl, dtype=torch.float64)
            reqs.append(dist.irecv(left, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(own[hi - lo - nb[rank + 1][0]:].contiguous(), rank + 1))
            right = torch.empty(hr, dtype=torch.float64)
            reqs.append(dist.irecv(right, rank + 1))
        for rq in reqs:
            rq.wait()
        if rank > 0:
            ext[:hl] = left
        if rank + 1 < world:
            ext[hl + hi - lo:] = right
        y = torch.tensor(oracle.spmv(rp, ci, val, ext.numpy()))
        B = (1 << (s["n"] - 1).bit_length()) // world  # block size (gloo gathers equal sizes)
        ypad = torch.zeros(B, dtype=torch.float64)
        ypad[:hi - lo] = y
        ys = [torch.empty(B, dtype=torch.float64) for r in range(world)]
        dist.all_gather(ys, ypad)
        ys = [t[:gsk.shard_rows(s["n"], world, r)[1] - gsk.shard_rows(s["n"], world, r)[0]] for r, t in enumerate(ys)]
        # dot <x, y>: the shard's canonical subtree (rows padded to the block size B)
        a = np.zeros(B)
        b = np.zeros(B)
        a[:hi - lo] = x[lo:hi]
        b[:hi - lo] = y.numpy()
        part = torch.tensor([oracle.dot(a, b)], dtype=torch.float64)
        parts = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, part)
        out[name] = (torch.cat(ys).numpy(), _tree([p.item() for p in parts]))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_spmv_and_dot_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name, N in (("C3", 12), ("C4", 20), ("C2", 40)):
        s = workloads.generate(name, N=N)
        x = workloads.uniform(s["n"], 11, 12)
        y = oracle.spmv(s["row_ptr"], s["col"], s["val"], x)
        for rank in (0, 1):
            ys, d = res[rank][name]
            assert np.array_equal(ys, y)
            assert d == oracle.dot(x, y)


def _worker_local(rank, world, port, q):
    """Local input (gsk_shard_opts.local_input; DESIGN.md §8 weak scaling): each rank
    generates ONLY its rows of the stacked workload C4w (G = world), computes its own
    halo widths from them, all-gathers the (hl, hr) pairs — what the library does over
    NCCL at plan creation — and runs the halo-exchanged SpMV on its rows."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    N = 12
    n, _ = workloads.dims(24, N, world)
    lo, hi = gsk.shard_rows(n, world, rank)
    loc = workloads.generate_rows("C4w", lo, hi, N=N, param=world)
    hl = max(0, lo - int(loc["col"].min()))
    hr = max(0, int(loc["col"].max()) - (hi - 1))
    hh = [torch.empty(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(hh, torch.tensor([hl, hr], dtype=torch.int64))
    nb = [tuple(int(v) for v in t) for t in hh]
    x = workloads.uniform(n, 11, 12)
    own = torch.tensor(x[lo:hi])
    ext = torch.zeros(hl + (hi - lo) + hr, dtype=torch.float64)
    ext[hl:hl + hi - lo] = own
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(own[:nb[rank - 1][1]].contiguous(), rank - 1))
        left = torch.empty(hl, dtype=torch.float64)
        reqs.append(dist.irecv(left, rank - 1))
    if rank + 1 < world:
        reqs.append(dist.isend(own[hi - lo - nb[rank + 1][0]:].contiguous(), rank + 1))
        right = torch.empty(hr, dtype=torch.float64)
        reqs.append(dist.irecv(right, rank + 1))
    for rq in reqs:
        rq.wait()
    if rank > 0:
        ext[:hl] = left
    if rank + 1 < world:
        ext[hl + hi - lo:] = right
    y = oracle.spmv(loc["row_ptr"], loc["col"] - lo + hl, loc["val"], ext.numpy())
    q.put((rank, (nb, lo, hi, y, loc["b"])))
    dist.barrier()
    dist.destroy_process_group()


def test_local_input_layout_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29750 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker_local, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = workloads.generate("C4w", N=12, param=2)  # the whole system, for comparison
    x = workloads.uniform(s["n"], 11, 12)
    y = oracle.spmv(s["row_ptr"], s["col"], s["val"], x)
    for rank in (0, 1):
        nb, lo, hi, yl, bl = res[rank]
        assert nb == [gsk.shard_halo(s["row_ptr"], s["col"], 2, r) for r in range(2)]
        assert np.array_equal(yl, y[lo:hi]) and np.array_equal(bl, s["b"][lo:hi])
