"""World-size-2 gloo test of the multi-GPU path's host logic on CPU.

Each rank computes its contiguous shard of (b,h) slices (the oracle stands
in for the GPU kernel -- this test covers partitioning and the verification
gather, not the kernel), then the shards are all-gathered and must equal a
single-process run bit for bit.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, n, d, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist
    from oracle_bindings import Oracle
    from paper_2409_16997_b200.sharding import gather_slices, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    lo, hi = shard_range(total, world, rank)
    outs = []
    for s in range(lo, hi):
        q, k, v = o.slice_inputs("uniform", n, d, b=s // 4, h=s % 4)
        qc, qs = o.quantize_per_row(q)
        kc, ks = o.quantize_per_row(k)
        vc, vs = o.quantize_per_tensor(v)
        outs.append(o.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 32))
    local = torch.from_numpy(np.stack(outs) if outs else np.zeros((0, n, d), np.float32))
    parts = gather_slices(local, total, world, rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 5])
def test_sharded_run_equals_single_process(tmp_path, oracle, total):
    import torch.multiprocessing as mp
    n, d, world = 48, 16, 2
    mp.spawn(_worker, args=(world, _free_port(), total, n, d, str(tmp_path)), nprocs=world,
             join=True)
    got = np.load(tmp_path / "gathered.npy")
    want = []
    for s in range(total):
        q, k, v = oracle.slice_inputs("uniform", n, d, b=s // 4, h=s % 4)
        qc, qs = oracle.quantize_per_row(q)
        kc, ks = oracle.quantize_per_row(k)
        vc, vs = oracle.quantize_per_tensor(v)
        want.append(oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 32))
    assert np.array_equal(got.view(np.uint32), np.stack(want).view(np.uint32))


def _mre_worker(rank, world, port, total, n, d, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist
    from oracle_bindings import Oracle
    from paper_2409_16997_b200.evaluation import ErrorAccum
    from paper_2409_16997_b200.sharding import allreduce_error, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    lo, hi = shard_range(total, world, rank)
    acc = ErrorAccum()
    for s in range(lo, hi):
        q, k, v = o.slice_inputs("normal", n, d, b=s // 4, h=s % 4)
        qc, qs = o.quantize_per_row(q)
        kc, ks = o.quantize_per_row(k)
        vc, vs = o.quantize_per_tensor(v)
        got = o.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 64)
        acc.add(torch.from_numpy(o.reference_attention(q, k, v)), torch.from_numpy(got))
    tot = allreduce_error(acc)
    if rank == 0:
        np.save(os.path.join(out_dir, "mre.npy"), np.array([tot.num, tot.den]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_mre_equals_single_process(tmp_path, oracle):
    """Per-rank (num, den) partials summed across ranks give the single-process
    MRE."""
    import torch
    import torch.multiprocessing as mp
    from paper_2409_16997_b200.evaluation import ErrorAccum
    n, d, world, total = 64, 16, 2, 5
    mp.spawn(_mre_worker, args=(world, _free_port(), total, n, d, str(tmp_path)), nprocs=world,
             join=True)
    num, den = np.load(tmp_path / "mre.npy")
    acc = ErrorAccum()
    for s in range(total):
        q, k, v = oracle.slice_inputs("normal", n, d, b=s // 4, h=s % 4)
        qc, qs = oracle.quantize_per_row(q)
        kc, ks = oracle.quantize_per_row(k)
        vc, vs = oracle.quantize_per_tensor(v)
        got = oracle.int_flash_attention(qc, qs, kc, ks, vc, vs, 64, 64)
        acc.add(torch.from_numpy(oracle.reference_attention(q, k, v)), torch.from_numpy(got))
    assert abs(num / den - acc.ratio()) <= 1e-12 * acc.ratio()


@pytest.mark.gpu
def test_bench_two_ranks_share_one_gpu(tmp_path):
    """bench.py's N>1 path (torchrun, per-rank shards, max-over-ranks timing,
    checksum gather) on a one-GPU box: both ranks share the GPU and the
    collectives run on gloo (IFA_BENCH_SHARE_GPU / IFA_BENCH_BACKEND hooks)."""
    import json
    import subprocess
    env = dict(os.environ, IFA_BENCH_SHARE_GPU="1", IFA_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "c5", "--steps", "1", "--warmup", "3", "--no-extras"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and len(line["checksums"]) == 2
    assert line["config"]["slices_per_rank"] == 1024 and line["scaling"] == "strong"
    # per-rank parity: sampled slices of BOTH ranks gathered to rank 0 and
    # checked against the oracle; whole-job MRE vs fp64 from summed partials
    par = line["parity_spot_check"]
    assert sorted({p["rank"] for p in par["per_rank"]}) == [0, 1]
    assert par["all_ok"], [(p["rank"], p["slice"], p["mre_vs_reference"], p["max_abs"],
                            p.get("within_tolerance"), p.get("bitwise_equal"))
                           for p in par["per_rank"]]
    mre = line["mre_vs_fp64"]
    assert mre["slices"] == 4 and 0.02 < mre["value"] < 0.045, mre
