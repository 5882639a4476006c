"""The multi-GPU modes of the pipeline on the GPU path, with 2 and 3
ranks sharing the one GPU of the test box (gloo carries the collectives: NCCL needs one
GPU per rank; the product's collectives are the same torch.distributed calls).

Each mode must reproduce a one-process run bit for bit: "sets" (strong: global sets
split by set range) -> identical counts; "ranks" (candidate-rank windows + per-set
merge) -> identical per-set outputs {n_sched, pi*, first rank, hash} and counts.
Plus the merge algebra on one process (windows evaluated one after the other)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gp_workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(key, reps, rank, world, split):
    from paper_2105_10312_b200.pipeline import Pipeline
    p = Pipeline(key, reps=reps, rank=rank, world=world, split=split, stats=False)
    p.run(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return p


def _worker(rank, world, port, key, reps, split, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = _run(key, reps, rank, world, split)
    per = p.per_set.cpu().numpy() if split == "ranks" else None
    gathered = [None] * world
    dist.all_gather_object(gathered, (p.counts.cpu().numpy(), per))
    if rank == 0:
        np.savez(out_path, counts=np.stack([g[0] for g in gathered]),
                 per=np.stack([g[1] for g in gathered]) if per is not None else np.zeros(1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("key,reps,world,split", [("c3", 3, 2, "ranks"), ("c3", 2, 3, "ranks"),
                                                  ("c2", 7, 2, "sets"), ("c2", 5, 3, "sets"),
                                                  ("c5", 3, 2, "sets")])
def test_multirank_modes_match_one_process(tmp_path, key, reps, world, split):
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), key, reps, split, out), nprocs=world,
             join=True)
    r = np.load(out)
    one = _run(key, reps, 0, 1, "weak")  # the same global sets in one process
    ref_counts = one.counts.cpu().numpy()
    for k in range(world):  # the all-reduced counts, identical on every rank
        assert (r["counts"][k] == ref_counts).all(), k
    if split == "ranks":
        ref_per = one.per_set.cpu().numpy()
        for k in range(world):
            assert (r["per"][k] == ref_per).all(), k


def test_window_merge_on_one_gpu():
    """Windows evaluated one after another on one GPU, packed, summed / minimised and
    unpacked, equal the full-window call; GP_FROM_PER_SET counts from the merged outputs
    equal the full EXHAUSTIVE call's counts (C3 shape, 3 x 10 sets, uneven windows)."""
    from paper_2105_10312_b200 import gpart as G
    from paper_2105_10312_b200 import pipeline as PL
    gen = W.WORKLOADS["c3"]["gen"](R=3)
    ts = G.TaskSets(30, 6, 20, 10)
    G.gp_generate(gen, W.SEED, 0, 3, ts)
    N = G.gp_count_candidates(20, 6)
    work = torch.zeros(1, dtype=torch.int64, device="cuda")
    full = torch.empty((30, 4), dtype=torch.int64, device="cuda")
    c_full = torch.zeros((1, 10, 1, 3), dtype=torch.int64, device="cuda")
    G.gp_sched_ratio(ts, G.GP_EXHAUSTIVE, c_full, per_set=full, work_counter=work)
    for cuts in ([0, 1, N], [0, 123457, 400000, N - 1, N], [0, N // 2, N]):
        parts = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            per = torch.empty((30, 4), dtype=torch.int64, device="cuda")
            G.gp_sched_ratio(ts, G.GP_EXHAUSTIVE, None, per_set=per, work_counter=work,
                             rank_lo=lo, rank_hi=hi)
            parts.append(PL.pack_window_shard(per))
        s = sum(p[0] for p in parts)
        m = torch.stack([p[1] for p in parts]).min(0).values
        merged = PL.unpack_window_shards(s, m, torch.empty_like(full))
        assert torch.equal(merged, full), cuts
        c = torch.zeros_like(c_full)
        G.gp_sched_ratio(ts, G.GP_FROM_PER_SET, c, per_set=merged)
        assert torch.equal(c, c_full), cuts
