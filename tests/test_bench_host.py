"""Host-side logic of bench.py: the N>1 aggregation (max time, summed work) over a
world_size-2 gloo group, the byte model, and the --impl reference JSON line."""
import json
import os
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms, its = bench.reduce_over_ranks(100.0 + 50 * rank, 1000 + rank, dist, "cpu")
    q.put((rank, ms, its))
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, ms, its in res:
        assert ms == 150.0 and its == 2001.0


def test_byte_model_c4():
    bm = bench.byte_model(16777216, 117047296)
    assert bm["spmv"] == 12 * 117047296 + 4 * 16777217 + 16 * 16777216
    assert abs(bm["bicg_iter"] / 1e9 - 5.225) < 0.001  # 5,225 MB


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "C2", "--N", "64", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, check=True, timeout=300).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "iters/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_roofline_traffic_from_committed_ncu():
    """The bench line's roofline `traffic` comes from the committed ncu capture: the
    dominant kernel (split Bi-CGSTAB S1) has a DRAM byte count within 10% of its
    algorithmic bytes (no wasted re-reads)."""
    t = bench.ncu_traffic("pass_kernel<2,1,OpS1>")
    alg = bench.byte_model(16777216, 117047296)["bicg_s1"]
    assert t is not None and 0.9 * alg < t < 1.1 * alg


def test_byte_model_row_classes_and_traffic():
    """Row-class plans: the matrix stream of an SpMV pass is the 2-byte class ids (the
    class lines stay in L1), and the committed ncu capture of the row-class kernels
    (profiles/r02_ncu_traffic_rcd.json) shows DRAM bytes within 10% of that model for the
    Bi-CGSTAB passes and the MGS pass — nothing re-read."""
    n, nnz = 16777216, 117047296
    bm = bench.byte_model(n, nnz, rcd=True)
    assert bm["spmv"] == 2 * n + 16 * n and bm["bicg_s1"] == 2 * n + 24 * n
    assert bm["bicg_iter_split"] == 2 * 2 * n + 19 * 8 * n
    for name, key in (("pass_kernel<6,1,OpS1>", "bicg_s1"), ("pass_kernel<6,1,OpS3>", "bicg_s3"),
                      ("pass_kernel<0,8,OpMgs>", "gmres_mgs"), ("pass_kernel<0,4,OpS4>", "bicg_s4")):
        t = bench.ncu_traffic(name)
        assert t is not None and 0.9 * bm[key] < t < 1.1 * bm[key], (name, t, bm[key])
