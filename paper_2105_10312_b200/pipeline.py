"""One step of the hot path over one batch: generate -> exhaustive (enumerate
+ WCET + EDF, fused) -> allocate (1G + 4 heuristics) -> ratio counts.

Every stage is one C-ABI call (libgpart.so); this module only owns the
device buffers (torch), orders the calls on one stream and issues the
collectives of the multi-GPU modes:

* ``split="weak"`` (default): rank r of W takes repetitions [r*R, (r+1)*R) of
  every (prm, bin) group, R = ``reps`` per rank (per-GPU work fixed), so all
  ranks see the same utilisation mix; one all-reduce sums the integer counts.
* ``split="sets"`` (strong): ``reps`` is the GLOBAL number of repetitions per
  group; rank r takes [floor(r R / W), floor((r+1) R / W)) of every group.
* ``split="ranks"`` (strong, for few sets): every rank holds all ``reps``
  global repetitions and evaluates the candidate-rank window
  [floor(r N_c / W), floor((r+1) N_c / W)) of every set; the per-set outputs
  are merged across ranks (sum n_sched, min pi*, min first_rank, sum hash mod
  2^64: ``merge_window_shards``) before the exhaustive counts are taken
  (gp_sched_ratio GP_FROM_PER_SET); the heuristics take set range
  [floor(r S / W), floor((r+1) S / W)).

Counter-based generation makes every shard byte-identical to the same sets of
a one-process run, and integer sums / minima are order-independent, so every
mode's counts (and, for "ranks", per-set outputs) equal one process's.
"""
from __future__ import annotations

import ctypes

import numpy as np

import torch

import gp_workloads as W

from . import gpart as G

SPLITS = ("weak", "sets", "ranks")


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
INT64_MAX = (1 << 63) - 1


class Pipeline:
    def __init__(self, key: str, reps: int = None, rank: int = 0, world: int = 1,
                 device="cuda", exhaustive: bool = None, variants=None, settings=None,
                 seed: int = W.SEED, stats: bool = True, split: str = "weak",
                 memo_heuristics: bool = True, parallel_variants: bool = None):
        if split not in SPLITS:
            raise ValueError(f"split must be one of {SPLITS}")
        wl = W.WORKLOADS[key]
        self.key, self.wl, self.seed, self.split = key, wl, seed, split
        self.rank, self.world = rank, world
        self.M, self.n = wl["M"], wl["n"]
        self.exhaustive = wl["exhaustive"] if exhaustive is None else exhaustive
        self.variants = tuple(wl["variants"] if variants is None else variants)
        self.device = device
        if key == "c1":
            self.host_sets = wl["sets"]()
            self.gens = []
            self.ts = G.TaskSets.from_host(self.host_sets, device)
            self.settings = [None]
            self.rep_begin, self.reps = 0, 1
        else:
            if split == "weak":
                self.rep_begin, self.reps, R = shard_plan(rank, world, reps)
            elif split == "sets":
                self.rep_begin, self.reps, R = strong_shard_plan(rank, world, reps)
            else:  # "ranks": all sets on every rank
                self.rep_begin, self.reps, R = 0, reps, reps
            self.settings = settings or ([(12, 23)] if key != "c5" else W.C5_SETTINGS)
            self.gens = [self._gen(kc, km, R) for kc, km in self.settings]
            g0 = self.gens[0]
            n_groups = g0["n_prm"] * g0["n_bins"]
            self.ts = G.TaskSets(n_groups * self.reps, self.n, self.M, n_groups, device)
        S = self.ts.n_sets
        # the sets this rank's heuristics evaluate (all but in "ranks" mode)
        self.h_lo, self.h_hi = (range_split(rank, world, S) if split == "ranks" else (0, S))
        self.ts_h = self.ts.slice(self.h_lo, self.h_hi) if split == "ranks" else self.ts
        Sh = self.h_hi - self.h_lo
        self.n_slots = (1 if self.exhaustive else 0) + len(self.variants)
        self.counts = torch.zeros((len(self.settings), self.ts.n_groups, self.n_slots, 3),
                                  dtype=torch.int64, device=device)
        self.verdicts = torch.zeros((len(self.variants), Sh), dtype=torch.uint8, device=device)
        self.alloc = []
        for vi in range(len(self.variants)):
            out = G.AllocOut(Sh, self.n, device)
            out.ok = self.verdicts[vi]  # gp_allocate writes its verdict row in place
            self.alloc.append(out)
        if self.exhaustive:
            self.n_cand = G.gp_count_candidates(self.M, self.n)
            self.rank_lo, self.rank_hi = (range_split(rank, world, self.n_cand)
                                          if split == "ranks" else (0, self.n_cand))
            self.per_set = torch.zeros((S, 4), dtype=torch.int64, device=device)
            self.work = torch.zeros(1, dtype=torch.int64, device=device)
            self.stats = torch.zeros(12, dtype=torch.int64, device=device) if stats else None
            # caller-owned evaluator workspace (gpart.h: no hidden persistent allocations)
            self.workspace = G.exhaustive_workspace(self.ts, device=device)
            # its input-independent tables (functions of n, M only) are built by the first
            # call and reused while this key matches (gpart.h gp_exhaustive_opts.tables_key)
            self.tables_key = ctypes.c_uint64(0)
        else:
            self.n_cand = 0
            self.workspace = None
        # the bit-sliced evaluator's memo words (the workspace's first n_sets * 2^n words)
        # serve the heuristics of the same step (gpart.h gp_alloc_opts.memo)
        self.memo_ok = (self.workspace is not None and self.n <= 8 and self.M <= 32
                        and memo_heuristics)
        # small sets (8-lane groups): the variants' kernels are short and their tails matter,
        # so they run on parallel streams; larger sets fill the GPU alone (A/B: C2/C3 -2-3 %,
        # C4 +8 %)
        self.parallel_variants = (self.n <= 8 if parallel_variants is None
                                  else parallel_variants)
        self._vstreams = None
        self.longest_first = True  # launch order of the parallel variant kernels (A/B)

    def _gen(self, kc, km, R):
        wl = self.wl
        if self.key == "c5":
            return wl["gen"](R=R, kc=kc, km=km)
        g = wl["gen"](R=R)
        g["kc_num"], g["km_num"] = kc, km
        return g

    def run(self, stream=None, mode=G.GP_EXHAUSTIVE, flags=0, stats=False, alloc_stats=None,
            on_dominant=None, ts=None, collectives=True):
        """Enqueue one full step (no host synchronisation except the collectives of the
        "ranks" split).  ``on_dominant(phase)`` is called with "begin"/"end" around the
        exhaustive call (or around the heuristics when there is none): bench.py records its
        CUDA events there.  ``ts``: evaluate these (already resident) task sets of the
        same shape instead of generating (bench.py's end-to-end path: host -> device)."""
        hook = on_dominant or (lambda phase: None)
        generate = ts is None
        ts = self.ts if ts is None else ts
        ts_h = ts.slice(self.h_lo, self.h_hi) if self.split == "ranks" else ts
        for si, _ in enumerate(self.settings):
            if self.gens and generate:
                G.gp_generate(self.gens[si], self.seed, self.rep_begin, self.reps, ts, stream)
            if self.exhaustive and si == 0:
                window = self.split == "ranks"
                hook("begin")
                G.gp_sched_ratio(ts, mode, None if window else self.counts, slot0=0,
                                 n_slots=self.n_slots, setting=si, per_set=self.per_set,
                                 work_counter=self.work,
                                 stats=self.stats if stats else None, stream=stream,
                                 flags=flags, workspace=self.workspace,
                                 tables_key=self.tables_key, rank_lo=self.rank_lo,
                                 rank_hi=G.UINT64_MAX if not window else self.rank_hi)
                hook("end")
                if window:
                    with torch.cuda.stream(stream) if stream is not None else _nullctx():
                        merge_window_shards(self.per_set)
                    if self.rank == 0:  # counted once, from the merged per-set outputs
                        G.gp_sched_ratio(ts, G.GP_FROM_PER_SET, self.counts, slot0=0,
                                         n_slots=self.n_slots, setting=si,
                                         per_set=self.per_set, stream=stream)
            if not self.exhaustive:
                hook("begin")
            # the bit-sliced exhaustive pass just memoised every (subset, size) verdict of
            # these sets in its workspace: the heuristics look their EDF tests up there
            memo = None
            if (self.exhaustive and si == 0 and mode == G.GP_EXHAUSTIVE and self.memo_ok
                    and not flags & (G.GP_EX_PER_CANDIDATE | G.GP_EX_GENERIC)):
                memo = self.workspace.data_ptr() + self.h_lo * 4  # subset-major rows
            if self.parallel_variants and stream is not None and len(self.variants) > 1:
                # the variants are independent: one stream each (fork / join by events; in
                # a captured graph, parallel branches), so their persistent grids' tails overlap
                if self._vstreams is None:
                    self._vstreams = [torch.cuda.Stream() for _ in self.variants]
                fork = torch.cuda.Event()
                fork.record(stream)
                joins = []
                # the longest kernels (INA, then ACT) first: they start before the short ones
                order = list(range(len(self.variants)))
                if self.longest_first:
                    order.sort(key=lambda i: -_VARIANT_COST.get(self.variants[i], 0))
                for vi in order:
                    v = self.variants[vi]
                    vs = self._vstreams[vi]
                    vs.wait_event(fork)
                    G.gp_allocate(ts_h, v, self.alloc[vi], vs, stats=alloc_stats, memo=memo,
                                  memo_stride=ts.n_sets)
                    e = torch.cuda.Event()
                    e.record(vs)
                    joins.append(e)
                for e in joins:
                    stream.wait_event(e)
            else:
                for vi, v in enumerate(self.variants):
                    G.gp_allocate(ts_h, v, self.alloc[vi], stream, stats=alloc_stats, memo=memo,
                                  memo_stride=ts.n_sets)
            if not self.exhaustive:
                hook("end")
            if self.variants and ts_h.n_sets > 0:
                G.gp_sched_ratio(ts_h, G.GP_FROM_VERDICTS, self.counts,
                                 verdicts=self.verdicts, slot0=1 if self.exhaustive else 0,
                                 n_slots=self.n_slots, setting=si, stream=stream)
        if collectives:
            allreduce_counts(self.counts)

    def capture(self, mode=G.GP_EXHAUSTIVE, flags=0):
        """One step as CUDA graphs: the launches between the ``on_dominant`` hooks become
        alternating segments [other, dominant, other, ...] (several for C5's settings), so
        a caller can replay the step with a handful of graph launches and still bracket
        the dominant launches with CUDA events between segments.  The counts all-reduce
        stays outside (call allreduce_counts after a replay).  Not for the "ranks" split,
        whose per-set merge is a host-driven collective.  Returns the list of graphs."""
        if self.split == "ranks":
            raise ValueError("capture: the ranks split merges windows on the host")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graphs = [torch.cuda.CUDAGraph()]

        def hook(phase):
            graphs[-1].capture_end()
            graphs.append(torch.cuda.CUDAGraph())
            graphs[-1].capture_begin()

        with torch.cuda.stream(side):
            graphs[0].capture_begin()
            self.run(side, mode=mode, flags=flags, on_dominant=hook, collectives=False)
            graphs[-1].capture_end()
        torch.cuda.current_stream().wait_stream(side)
        return graphs

    def candidates_per_step(self) -> int:
        """Exhaustive candidate evaluations per step on this rank (the metric's unit)."""
        if not self.exhaustive:
            return 0
        return self.ts.n_sets * (self.rank_hi - self.rank_lo)

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


def range_split(rank: int, world: int, total: int):
    """[floor(r T / W), floor((r+1) T / W)): contiguous, disjoint, covering [0, T)."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad range split")
    return rank * total // world, (rank + 1) * total // world


def strong_shard_plan(rank: int, world: int, reps_global: int):
    """Strong-scaling shard: the GLOBAL repetitions per group are fixed and rank r
    takes its contiguous share of every group.  Returns (rep_begin, rep_count,
    sets_per_group); needs reps_global >= world so that no rank is empty."""
    if reps_global < world:
        raise ValueError("strong split needs at least one repetition per rank")
    lo, hi = range_split(rank, world, reps_global)
    return lo, hi - lo, reps_global


def pack_window_shard(per_set: torch.Tensor):
    """One rank-window shard's per-set outputs (gpart.h EXHAUSTIVE convention) ->
    (sum part [S][3], min part [S][2]) whose elementwise sums / minima over the
    shards are the full window's: n_sched (a contract violation, -1 in every
    shard, becomes -2^40 so the sum stays negative), the hash split into 32-bit
    halves (sums cannot overflow), and pi*, first rank with "none" -> INT64_MAX."""
    n, pi, first, h = per_set.unbind(1)
    none = n <= 0
    big = torch.full_like(n, INT64_MAX)
    s = torch.stack([torch.where(n < 0, torch.full_like(n, -(1 << 40)), n),
                     h & 0xFFFFFFFF, (h >> 32) & 0xFFFFFFFF], 1).contiguous()
    m = torch.stack([torch.where(none, big, pi), torch.where(none, big, first)], 1).contiguous()
    return s, m


def unpack_window_shards(s: torch.Tensor, m: torch.Tensor, out: torch.Tensor):
    """Inverse of pack_window_shard after the sum / min over shards."""
    n = s[:, 0]
    lo = s[:, 1] & 0xFFFFFFFF
    hi = (s[:, 2] + (s[:, 1] >> 32)) & 0xFFFFFFFF
    h = lo | (hi << 32)  # mod 2^64, as an int64 bit pattern
    bad, none = n < 0, n == 0
    z, m1 = torch.zeros_like(n), torch.full_like(n, -1)
    out[:, 0] = torch.where(bad, m1, n)
    out[:, 1] = torch.where(bad | none, z, m[:, 0])
    out[:, 2] = torch.where(bad | none, m1, m[:, 1])
    out[:, 3] = torch.where(bad | none, z, h)
    return out


def merge_window_shards(per_set: torch.Tensor, group=None):
    """§8(e)'s per-set merge of candidate-rank shards, in place: sum n_sched, min pi*,
    min first_rank, sum hash mod 2^64, over the ranks of the process group (two
    all-reduces, SUM and MIN; the identity without a process group)."""
    import torch.distributed as dist
    s, m = pack_window_shard(per_set)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(m, op=dist.ReduceOp.MIN, group=group)
    return unpack_window_shards(s, m, per_set)


# relative kernel time of the heuristic variants (C3 launch lists: INA > ACT > 1G), used only
# to order their launches on parallel streams
_VARIANT_COST = {"SMS_INA": 4, "BF_INA": 3, "SMS_ACT": 2, "BF_ACT": 1, "1G": 0}


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
