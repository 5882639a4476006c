"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 host path:
weak-scaling shards cover every set once and the one all-reduce of the
integer ratio counts reproduces the single-process counts bit for bit.
The per-rank evaluation uses the oracle (no GPU here); on the GPU box the
same shard plan feeds gp_generate and the same all-reduce runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gp_workloads as W
import oracle

pytestmark = pytest.mark.timeout(300) if hasattr(pytest.mark, "timeout") else []


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _product():
    """The product's host-side N>1 logic (needs libgpart.so built, not a GPU)."""
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2105_10312_b200", "libgpart.so")
    if not os.path.exists(lib):
        from paper_2105_10312_b200 import _build
        _build.build()
    from paper_2105_10312_b200 import pipeline
    return pipeline


def _shard_plan(rank, world, reps):
    return _product().shard_plan(rank, world, reps)


def _counts_for(gen, rep_begin, rep_count):
    s = oracle.generate(gen, W.SEED, rep_begin, rep_count)
    counts = np.zeros((1, s.n_groups, 6, 3), np.int64)
    per = oracle.exhaustive(s, threads=2)
    oracle.sched_ratio(s, (per[:, 0] > 0).astype(np.uint8)[None], 0, 6, 0, counts)
    rows = np.stack([oracle.allocate(s, v, threads=2)["ok"] for v in W.VARIANT_NAMES])
    oracle.sched_ratio(s, rows, 1, 6, 0, counts)
    return s, counts


def _worker(rank, world, port, reps, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep_begin, rep_count, spg = _shard_plan(rank, world, reps)
    gen = W.WORKLOADS["c2"]["gen"](R=spg)
    s, counts = _counts_for(gen, rep_begin, rep_count)
    t = torch.from_numpy(counts)
    _product().allreduce_counts(t)  # the one data-path collective (SUM)
    # max-over-ranks of a per-rank time, as bench.py does
    tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, (rep_begin, rep_count, s.T.tolist()))
    if rank == 0:
        np.savez(out_path, counts=t.numpy(), tmax=tm.numpy(),
                 shards=np.array([g[:2] for g in gathered]),
                 T=np.concatenate([np.array(g[2]).reshape(10, g[1], -1) for g in gathered], 1))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_and_allreduce(tmp_path):
    world, reps = 2, 3
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), reps, out), nprocs=world, join=True)
    r = np.load(out)
    # shards tile the repetition axis
    assert r["shards"].tolist() == [[0, 3], [3, 3]]
    assert float(r["tmax"][0]) == 2.0
    # single process over the whole range: identical sets and identical counts
    gen = W.WORKLOADS["c2"]["gen"](R=world * reps)
    s, counts = _counts_for(gen, 0, world * reps)
    assert (r["T"] == s.T.reshape(10, world * reps, -1)).all()
    assert (r["counts"] == counts).all()
    assert counts[0, :, :, 1].sum() == 10 * world * reps * 6


def test_shard_plan_rejects_bad_input():
    with pytest.raises(ValueError):
        _shard_plan(2, 2, 5)
    assert _shard_plan(1, 4, 7) == (7, 7, 28)
