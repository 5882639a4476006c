"""One step of the hot path over one batch: generate -> exhaustive (enumerate
+ WCET + EDF, fused) -> allocate (1G + 4 heuristics) -> ratio counts.

Every stage is one C-ABI call (libgpart.so); this module only owns the
device buffers (torch) and orders the calls on one stream.  Multi-GPU: rank r
of W takes repetitions [r*reps, (r+1)*reps) of every (prm, bin) group, so all
ranks see the same utilisation mix; the per-group counts are integers and
one all-reduce (NCCL) sums them (``allreduce_counts``).
"""
from __future__ import annotations

import numpy as np
import torch

import gp_workloads as W

from . import gpart as G


class Pipeline:
    def __init__(self, key: str, reps: int = None, rank: int = 0, world: int = 1,
                 device="cuda", exhaustive: bool = None, variants=None, settings=None,
                 seed: int = W.SEED, stats: bool = True):
        wl = W.WORKLOADS[key]
        self.key, self.wl, self.seed = key, wl, seed
        self.rank, self.world = rank, world
        self.M, self.n = wl["M"], wl["n"]
        self.exhaustive = wl["exhaustive"] if exhaustive is None else exhaustive
        self.variants = tuple(wl["variants"] if variants is None else variants)
        self.device = device
        if key == "c1":
            self.host_sets = wl["sets"]()
            self.gen = None
            self.ts = G.TaskSets.from_host(self.host_sets, device)
            self.settings = [None]
        else:
            self.reps = reps
            self.settings = settings or ([(12, 23)] if key != "c5" else W.C5_SETTINGS)
            self.gens = [self._gen(kc, km) for kc, km in self.settings]
            g0 = self.gens[0]
            n_groups = g0["n_prm"] * g0["n_bins"]
            self.ts = G.TaskSets(n_groups * reps, self.n, self.M, n_groups, device)
        S = self.ts.n_sets
        self.n_slots = (1 if self.exhaustive else 0) + len(self.variants)
        self.counts = torch.zeros((len(self.settings), self.ts.n_groups, self.n_slots, 3),
                                  dtype=torch.int64, device=device)
        self.verdicts = torch.zeros((len(self.variants), S), dtype=torch.uint8, device=device)
        self.alloc = []
        for vi in range(len(self.variants)):
            out = G.AllocOut(S, self.n, device)
            out.ok = self.verdicts[vi]  # gp_allocate writes its verdict row in place
            self.alloc.append(out)
        if self.exhaustive:
            self.n_cand = G.gp_count_candidates(self.M, self.n)
            self.per_set = torch.zeros((S, 4), dtype=torch.int64, device=device)
            self.work = torch.zeros(1, dtype=torch.int64, device=device)
            self.stats = torch.zeros(6, dtype=torch.int64, device=device) if stats else None
            # caller-owned evaluator workspace (gpart.h: no hidden persistent allocations)
            self.workspace = G.exhaustive_workspace(self.ts, device=device)
        else:
            self.n_cand = 0

    def _gen(self, kc, km):
        wl = self.wl
        if self.key == "c5":
            return wl["gen"](R=self.reps * self.world, kc=kc, km=km)
        g = wl["gen"](R=self.reps * self.world)
        g["kc_num"], g["km_num"] = kc, km
        return g

    @property
    def rep_begin(self):
        return shard_plan(self.rank, self.world, self.reps)[0]

    def run(self, stream=None):
        """Enqueue one full step (no host synchronisation)."""
        for si, _ in enumerate(self.settings):
            if self.gens_present:
                G.gp_generate(self.gens[si], self.seed, self.rep_begin, self.reps, self.ts, stream)
            if self.exhaustive and si == 0:
                G.gp_sched_ratio(self.ts, G.GP_EXHAUSTIVE, self.counts, slot0=0,
                                 n_slots=self.n_slots, setting=si, per_set=self.per_set,
                                 work_counter=self.work, stats=self.stats, stream=stream,
                                 workspace=self.workspace)
            for vi, v in enumerate(self.variants):
                G.gp_allocate(self.ts, v, self.alloc[vi], stream)
            if self.variants:
                G.gp_sched_ratio(self.ts, G.GP_FROM_VERDICTS, self.counts, verdicts=self.verdicts,
                                 slot0=1 if self.exhaustive else 0, n_slots=self.n_slots,
                                 setting=si, stream=stream)

    @property
    def gens_present(self):
        return self.key != "c1"

    def candidates_per_step(self) -> int:
        """Exhaustive candidate evaluations per step (the metric's unit)."""
        return self.ts.n_sets * self.n_cand if self.exhaustive else 0

    def heuristic_tests(self) -> int:
        return int(sum(int(a.n_tests.clamp(min=0).sum()) for a in self.alloc))

    def reset_counts(self):
        self.counts.zero_()
        if self.exhaustive and self.stats is not None:
            self.stats.zero_()


def shard_plan(rank: int, world: int, reps_per_rank: int):
    """Weak-scaling shard of the repetition axis: every rank
    takes the same number of repetitions of EVERY (prm, bin) group, so all
    ranks see the same utilisation mix.  Returns (rep_begin, rep_count,
    sets_per_group) for gp_generate; the union over ranks is every set of the
    world-size job exactly once, and integer counts sum exactly."""
    if not (0 <= rank < world) or reps_per_rank < 1:
        raise ValueError("bad shard")
    return rank * reps_per_rank, reps_per_rank, reps_per_rank * world


def allreduce_counts(counts: torch.Tensor):
    """The one data-path collective: sum the integer ratio counts over ranks."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    return counts


def rates(counts: np.ndarray):
    """sched / total per (setting, group, slot) -- the derived float (C.1.11)."""
    c = np.asarray(counts)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(c[..., 1] > 0, c[..., 0] / np.maximum(c[..., 1], 1), np.nan)
