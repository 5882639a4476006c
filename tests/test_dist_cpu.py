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


# ---------------------------------------------------------------- strong scaling
def _strong_worker(rank, world, port, reps, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = _product()
    rep_begin, rep_count, spg = P.strong_shard_plan(rank, world, reps)
    gen = W.WORKLOADS["c2"]["gen"](R=spg)
    _, counts = _counts_for(gen, rep_begin, rep_count)
    t = torch.from_numpy(counts)
    P.allreduce_counts(t)
    if rank == 0:
        np.save(out_path, t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_strong_set_split_two_ranks(tmp_path):
    """split="sets": 5 global repetitions per group over 2 ranks (2 + 3, uneven) give the
    one-process counts of the same 50 sets, bit for bit."""
    world, reps = 2, 5
    out = str(tmp_path / "s.npy")
    mp.spawn(_strong_worker, args=(world, _free_port(), reps, out), nprocs=world, join=True)
    gen = W.WORKLOADS["c2"]["gen"](R=reps)
    _, counts = _counts_for(gen, 0, reps)
    assert (np.load(out) == counts).all()
    P = _product()
    assert [P.strong_shard_plan(r, 2, 5) for r in range(2)] == [(0, 2, 5), (2, 3, 5)]
    with pytest.raises(ValueError):
        P.strong_shard_plan(0, 4, 3)


# ---------------------------------------------------------------- candidate-rank windows
def _window_sets():
    gen = W.WORKLOADS["c2"]["gen"](R=10000)
    return oracle.generate(gen, W.SEED, 0, 2)  # 20 sets (10 bins x 2)


def _shard_per_set(s, lo, hi, violated=(3,)):
    """The per-set outputs one rank produces for its window, in gpart.h's convention
    (oracle values; a contract-violating set reads -1, 0, -1, 0 in every shard)."""
    per = oracle.exhaustive(s, lo, hi, threads=2)
    for v in violated:
        per[v] = (-1, 0, -1, 0)
    return per


def _window_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = _product()
    s = _window_sets()
    lo, hi = P.range_split(rank, world, oracle.count_candidates(8, 6))
    per = torch.from_numpy(_shard_per_set(s, lo, hi))
    P.merge_window_shards(per)  # SUM + MIN all-reduces over gloo
    gathered = [None] * world
    dist.all_gather_object(gathered, per.numpy())
    if rank == 0:
        np.save(out_path, np.stack(gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_window_split_merge(tmp_path, world):
    """split="ranks": every rank evaluates its candidate-rank window of
    every set; the per-set merge (sum n_sched, min pi*, min first rank, sum hash mod
    2^64) reproduces the one-process full-window per-set outputs bit for bit on every
    rank, including a contract-violating set and sets with no schedulable candidate in
    some windows."""
    out = str(tmp_path / "w.npy")
    mp.spawn(_window_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    full = _shard_per_set(_window_sets(), 0, oracle.count_candidates(8, 6))
    for r in range(world):
        assert (got[r] == full).all()
    assert (full[:, 0] == 0).any() and (full[:, 3] < 0).any()  # empty sets; hash >= 2^63


def test_pack_unpack_merge_without_collective():
    """The merge algebra alone (no process group): shards of 1..7 windows, random cut
    points, hashes whose 64-bit sums wrap."""
    P = _product()
    s = _window_sets()
    N = oracle.count_candidates(8, 6)
    full = _shard_per_set(s, 0, N)
    rng = np.random.default_rng(3)
    for k in range(1, 8):
        cuts = [0] + sorted(int(x) for x in rng.integers(0, N, k - 1)) + [N]
        parts = [P.pack_window_shard(torch.from_numpy(_shard_per_set(s, a, b)))
                 for a, b in zip(cuts[:-1], cuts[1:])]
        ssum = sum(p[0] for p in parts)
        smin = torch.stack([p[1] for p in parts]).min(0).values
        out = torch.empty((s.n_sets, 4), dtype=torch.int64)
        assert (P.unpack_window_shards(ssum, smin, out).numpy() == full).all(), k
    # identity without a process group
    one = torch.from_numpy(full.copy())
    assert (P.merge_window_shards(one).numpy() == full).all()
