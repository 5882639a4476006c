"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/libgpref.so`` (built from ``oracle/gpref.c`` by
``oracle.build()`` / ``__graft_entry__.build()``): the plain, slow CPU oracle
of arXiv 2105.10312's hot path.  See ``oracle/gpref.h`` for the citations.

Import rule: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline leg (and ``bench.py --impl reference``) may import this package.
It never imports the product package ``paper_2105_10312_b200`` and the
product never imports it.  Inputs are plain numpy arrays / dicts produced by
the neutral module ``gp_workloads``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgpref.so")
_SRC = os.path.join(_HERE, "gpref.c")

VARIANTS = {"1G": 0, "SMS_ACT": 1, "SMS_INA": 2, "BF_ACT": 3, "BF_INA": 4}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (never tuned for speed)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "gpref.h"))
    ):
        tmp = _SO + ".tmp"
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra",
             "-Wno-unused-parameter", _SRC, "-o", tmp]
        )
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _declare(_lib)
    return _lib


class _Sets(C.Structure):
    _fields_ = [("n_sets", C.c_int32), ("n_tasks", C.c_int32), ("M", C.c_int32),
                ("n_groups", C.c_int32)] + [
        (f, C.c_void_p) for f in ("T", "D", "B", "cn", "cc", "fn", "fc", "type", "valid", "group")]


class _Gen(C.Structure):
    _fields_ = [("M", C.c_int32), ("n_tasks", C.c_int32), ("n_bins", C.c_int32),
                ("n_prm", C.c_int32), ("sets_per_group", C.c_int32), ("prm_q", C.c_void_p),
                ("ticks_per_unit", C.c_int32), ("n_periods", C.c_int32),
                ("period_menu", C.c_void_p), ("b_max", C.c_int32), ("beta_c_num", C.c_int32),
                ("beta_m_num", C.c_int32), ("beta_den", C.c_int32), ("kc_num", C.c_int32),
                ("km_num", C.c_int32), ("k_den", C.c_int32), ("max_attempts", C.c_int32),
                ("curve_gran", C.c_int32)]


def _declare(L):
    P = C.c_void_p
    L.gpref_philox4x32_10.argtypes = [P, P, P]
    L.gpref_generate.argtypes = [P, C.c_uint64, C.c_uint64, C.c_int32, P]
    L.gpref_wcet.argtypes = [C.c_int64] * 4
    L.gpref_wcet.restype = C.c_int64
    L.gpref_wcet_per_sm.argtypes = [C.c_int64, C.c_int32, P, C.c_int64, P, P]
    L.gpref_conflict.argtypes = [C.c_int32, P, C.c_uint32, C.c_int32]
    L.gpref_wcet_batch.argtypes = [P, P, P, P, C.c_int64, P, P]
    L.gpref_hyperperiod.argtypes = [C.c_int32, P, P]
    L.gpref_edf_pdc.argtypes = [C.c_int32, P, P, P, P, P]
    L.gpref_simulate_edf.argtypes = [C.c_int32, P, P, P, C.c_int64]
    L.gpref_count_candidates.argtypes = [C.c_int32, C.c_int32, P]
    L.gpref_enumerate.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_int64, P, P]
    L.gpref_unrank.argtypes = [C.c_int32, C.c_int32, C.c_uint64, P, P]
    L.gpref_exhaustive.argtypes = [P, C.c_uint64, C.c_uint64, P, P, C.c_int64, C.c_int32]
    L.gpref_exhaustive_ex.argtypes = [P, C.c_uint64, C.c_uint64, P, P, P, C.c_int64, C.c_int32]
    L.gpref_allocate.argtypes = [P, C.c_int32, P, P, P, P, P, P, C.c_int32]
    L.gpref_allocate_ex.argtypes = [P, C.c_int32, P, P, P, P, P, P, P, C.c_int32]
    L.gpref_sched_ratio.argtypes = [P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P]
    L.gpref_uunisort.argtypes = [C.c_int32, C.c_int64, P, P]
    L.gpref_task_fields.argtypes = [P, C.c_int64, C.c_int32, C.c_int64, C.c_int32, P]
    L.gpref_efficiency.argtypes = [P, P, P]
    L.gpref_fill_forbidden_list.argtypes = [P, C.c_int32, P, P]
    L.gpref_select_partitions.argtypes = [P, C.c_int32, C.c_int32, P, P, C.c_int32, P, P, P,
                                          C.c_int32, P, P, P]
    L.gpref_splitmix64.argtypes = [C.c_uint64]
    L.gpref_splitmix64.restype = C.c_uint64


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc != 0:
        raise OracleError(f"{what}: oracle returned {rc}")


@dataclass
class Sets:
    """A batch of task sets, fields [n_sets][n_tasks] (ticks)."""
    M: int
    n_groups: int
    T: np.ndarray
    D: np.ndarray
    B: np.ndarray
    cn: np.ndarray
    cc: np.ndarray
    fn: np.ndarray
    fc: np.ndarray
    type: np.ndarray
    valid: np.ndarray
    group: np.ndarray

    @property
    def n_sets(self):
        return self.T.shape[0]

    @property
    def n_tasks(self):
        return self.T.shape[1]

    @classmethod
    def from_dict(cls, d):
        f = {k: np.ascontiguousarray(d[k], dtype=np.int32)
             for k in ("T", "D", "B", "cn", "cc", "fn", "fc", "group")}
        f["type"] = np.ascontiguousarray(d["type"], dtype=np.uint8)
        f["valid"] = np.ascontiguousarray(d["valid"], dtype=np.uint8)
        return cls(M=int(d["M"]), n_groups=int(d["n_groups"]), **f)

    def to_dict(self):
        return dict(M=self.M, n_groups=self.n_groups, T=self.T, D=self.D, B=self.B, cn=self.cn,
                    cc=self.cc, fn=self.fn, fc=self.fc, type=self.type, valid=self.valid,
                    group=self.group)

    def subset(self, idx):
        d = self.to_dict()
        for k in ("T", "D", "B", "cn", "cc", "fn", "fc", "type", "valid", "group"):
            d[k] = np.ascontiguousarray(d[k][idx])
        return Sets.from_dict(d)

    def _c(self):
        s = _Sets(self.n_sets, self.n_tasks, self.M, self.n_groups)
        for k in ("T", "D", "B", "cn", "cc", "fn", "fc", "type", "valid", "group"):
            setattr(s, k, _p(getattr(self, k)).value)
        return s


def empty_sets(n_sets, n_tasks, M, n_groups):
    z = lambda dt: np.zeros((n_sets, n_tasks), dtype=dt)  # noqa: E731
    return Sets(M=M, n_groups=n_groups, T=z(np.int32), D=z(np.int32), B=z(np.int32),
                cn=z(np.int32), cc=z(np.int32), fn=z(np.int32), fc=z(np.int32),
                type=z(np.uint8), valid=np.zeros(n_sets, np.uint8),
                group=np.zeros(n_sets, np.int32))


def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().gpref_philox4x32_10(_p(c), _p(k), _p(out))
    return [int(x) for x in out]


def splitmix64(x):
    return int(lib().gpref_splitmix64(int(x) & (2**64 - 1)))


def _gen_struct(gen: dict):
    prm_q = np.ascontiguousarray(gen["prm_q"], dtype=np.uint64)
    menu = np.ascontiguousarray(gen["period_menu"], dtype=np.int32)
    g = _Gen(gen["M"], gen["n_tasks"], gen["n_bins"], gen["n_prm"], gen["sets_per_group"],
             _p(prm_q).value, gen["ticks_per_unit"], len(menu), _p(menu).value, gen["b_max"],
             gen["beta_c_num"], gen["beta_m_num"], gen["beta_den"], gen["kc_num"],
             gen["km_num"], gen["k_den"], gen["max_attempts"], gen.get("curve_gran", 0))
    return g, (prm_q, menu)  # keep the arrays alive with the struct


def generate(gen: dict, seed: int, rep_begin: int, rep_count: int) -> Sets:
    n_groups = gen["n_prm"] * gen["n_bins"]
    out = empty_sets(n_groups * rep_count, gen["n_tasks"], gen["M"], n_groups)
    g, _keep = _gen_struct(gen)
    cs = out._c()
    _check(lib().gpref_generate(C.byref(g), seed, rep_begin, rep_count, C.byref(cs)), "generate")
    return out


def uunisort(n, Uq, points):
    pts = np.ascontiguousarray(points, dtype=np.int64)
    u = np.zeros(n, np.int64)
    _check(lib().gpref_uunisort(n, Uq, _p(pts), _p(u)), "uunisort")
    return u


def task_fields(gen: dict, u_q20, period_idx, B, typ):
    """{T, D, cn, fn, cc, fc, a, feasible} of one §7.1 task."""
    g, _keep = _gen_struct(gen)
    out = np.zeros(9, np.int64)
    _check(lib().gpref_task_fields(C.byref(g), u_q20, period_idx, B, typ, _p(out)), "task_fields")
    return dict(zip(("T", "D", "cn", "fn", "cc", "fc", "a", "feasible", "B"), (int(x) for x in out)))


def wcet(B, c, f, m):
    return int(lib().gpref_wcet(B, c, f, m))


def wcet_per_sm(B, costs, f=0):
    costs = np.ascontiguousarray(costs, dtype=np.int64)
    per = np.zeros(len(costs), np.int64)
    w = np.zeros(1, np.int64)
    _check(lib().gpref_wcet_per_sm(B, len(costs), _p(costs), f, _p(per), _p(w)), "wcet_per_sm")
    return [int(x) for x in per], int(w[0])


def conflict(types, mask, i):
    t = np.ascontiguousarray(types, dtype=np.uint8)
    return bool(lib().gpref_conflict(len(t), _p(t), mask, i))


def wcet_batch(sets: Sets, set_of_cand, block_of_task, block_size):
    soc = np.ascontiguousarray(set_of_cand, dtype=np.int32)
    bot = np.ascontiguousarray(block_of_task, dtype=np.int8)
    bs = np.ascontiguousarray(block_size, dtype=np.int16)
    n = sets.n_tasks
    w = np.zeros((len(soc), n), np.int32)
    cf = np.zeros((len(soc), n), np.uint8)
    cs = sets._c()
    _check(lib().gpref_wcet_batch(C.byref(cs), _p(soc), _p(bot), _p(bs), len(soc), _p(w), _p(cf)),
           "wcet_batch")
    return w, cf


def hyperperiod(T):
    t = np.ascontiguousarray(T, dtype=np.int64)
    h = np.zeros(1, np.int64)
    _check(lib().gpref_hyperperiod(len(t), _p(t), _p(h)), "hyperperiod")
    return int(h[0])


def edf_pdc(C_, D, T):
    """(schedulable, witness or None, distinct deadlines examined)"""
    c = np.ascontiguousarray(C_, dtype=np.int64)
    d = np.ascontiguousarray(D, dtype=np.int64)
    t = np.ascontiguousarray(T, dtype=np.int64)
    w = np.full(1, -1, np.int64)
    npts = np.zeros(1, np.int64)
    r = lib().gpref_edf_pdc(len(c), _p(c), _p(d), _p(t), _p(w), _p(npts))
    if r < 0:
        raise OracleError(f"edf_pdc error {r}")
    return bool(r), (None if r else int(w[0])), int(npts[0])


def simulate_edf(C_, D, T, horizon):
    c = np.ascontiguousarray(C_, dtype=np.int64)
    d = np.ascontiguousarray(D, dtype=np.int64)
    t = np.ascontiguousarray(T, dtype=np.int64)
    return bool(lib().gpref_simulate_edf(len(c), _p(c), _p(d), _p(t), horizon))


def count_candidates(M, n):
    out = np.zeros(1, np.uint64)
    rc = lib().gpref_count_candidates(M, n, _p(out))
    if rc == 2:
        raise OverflowError("candidate count >= 2^63")
    _check(rc, "count_candidates")
    return int(out[0])


def enumerate_candidates(M, n, first=0, count=None):
    if count is None:
        count = count_candidates(M, n) - first
    bot = np.zeros((count, n), np.int8)
    bs = np.zeros((count, n), np.int16)
    _check(lib().gpref_enumerate(M, n, first, count, _p(bot), _p(bs)), "enumerate")
    return bot, bs


def unrank(M, n, r):
    bot = np.zeros(n, np.int8)
    bs = np.zeros(n, np.int16)
    _check(lib().gpref_unrank(M, n, r, _p(bot), _p(bs)), "unrank")
    return bot, bs


def _admissible(M, sizes):
    if sizes is None:
        return None
    adm = np.zeros(M + 1, np.uint8)
    for m in sizes:
        assert 1 <= m <= M, "admissible sizes lie in 1..M"
        adm[m] = 1
    return adm


def exhaustive(sets: Sets, rank_lo=0, rank_hi=None, bits=False, threads=None, sizes=None):
    """per_set [n_sets][4] = (n_sched, pi_star, first_rank, hash as int64); bits optional.
    ``sizes``: admissible partition sizes (f4, reading B-9; None = every size) --
    a candidate using another size counts as unschedulable."""
    total = count_candidates(sets.M, sets.n_tasks)
    if rank_hi is None:
        rank_hi = total
    per = np.zeros((sets.n_sets, 4), np.int64)
    words = (rank_hi - rank_lo + 31) // 32
    vb = np.zeros((sets.n_sets, words), np.uint32) if bits else None
    cs = sets._c()
    th = threads or os.cpu_count() or 1
    adm = _admissible(sets.M, sizes)
    _check(lib().gpref_exhaustive_ex(C.byref(cs), rank_lo, rank_hi,
                                     None if adm is None else _p(adm), _p(per),
                                     _p(vb) if bits else None, words, th), "exhaustive")
    return (per, vb) if bits else per


class _AllocOpts(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("admissible", C.c_void_p)]


AL_BINARY_MERGE = 1   # f4: Algorithm 2 by binary search
AL_INCREASING = 2     # f4: par_list in increasing utilisation


def allocate(sets: Sets, variant, threads=None, flags=0, sizes=None):
    """Heuristics (Alg. 1-3) / 1G.  f4 variants: ``flags`` (AL_BINARY_MERGE,
    AL_INCREASING) and ``sizes`` = the admissible partition sizes (MIG-style
    slices; None = every size)."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    S, n = sets.n_sets, sets.n_tasks
    ok = np.zeros(S, np.uint8)
    bot = np.zeros((S, n), np.int16)
    bs = np.zeros((S, n), np.int16)
    pi = np.zeros(S, np.int32)
    k = np.zeros(S, np.int32)
    nt = np.zeros(S, np.int64)
    cs = sets._c()
    th = threads or os.cpu_count() or 1
    adm = _admissible(sets.M, sizes)
    opts = _AllocOpts(int(flags), None if adm is None else adm.ctypes.data)
    _check(lib().gpref_allocate_ex(C.byref(cs), v, C.byref(opts), _p(ok), _p(bot), _p(bs), _p(pi),
                                   _p(k), _p(nt), th), "allocate")
    return dict(ok=ok, block_of_task=bot, block_size=bs, pi=pi, k=k, n_tests=nt)


def fill_forbidden_list(sets: Sets, set_idx=0):
    """ACT prefill: (forbidden task-pair matrix [n][n], EDF tests run)."""
    n = sets.n_tasks
    forb = np.zeros((n, n), np.uint8)
    nt = np.zeros(1, np.int64)
    cs = sets._c()
    _check(lib().gpref_fill_forbidden_list(C.byref(cs), set_idx, _p(forb), _p(nt)),
           "fill_forbidden_list")
    return forb, int(nt[0])


def select_partitions(sets: Sets, parts, snapshots=(), forb=None, best_fit=False, set_idx=0):
    """Algorithm 3 on a given state.  parts: list of (task-id
    list, size); snapshots: list of (task-id list, task-id list) INA failures; forb:
    ACT task-pair matrix or None.  Returns (selected task-id list or None, [elig
    task-id lists in order])."""
    def m(ids):
        return sum(1 << i for i in ids)

    def ids(mask):
        return [i for i in range(64) if (int(mask) >> i) & 1]
    masks = np.array([m(p) for p, _ in parts], np.uint64)
    sizes = np.array([sz for _, sz in parts], np.int32)
    sa = np.array([m(a) for a, _ in snapshots] or [0], np.uint64)
    sb = np.array([m(b) for _, b in snapshots] or [0], np.uint64)
    fb = None if forb is None else np.ascontiguousarray(forb, dtype=np.uint8)
    sel = np.zeros(1, np.uint64)
    elig = np.zeros(max(1, len(parts)), np.uint64)
    ne = np.zeros(1, np.int32)
    cs = sets._c()
    _check(lib().gpref_select_partitions(C.byref(cs), set_idx, len(parts), _p(masks), _p(sizes),
                                         len(snapshots), _p(sa), _p(sb),
                                         None if fb is None else _p(fb), int(best_fit), _p(sel),
                                         _p(elig), _p(ne)), "select_partitions")
    return (ids(sel[0]) if sel[0] else None), [ids(x) for x in elig[:int(ne[0])]]


def efficiency(sets: Sets, block_of_task):
    """[n_sets][4] = (lower, upper, achieved, H): work-based utilisations x H."""
    bot = np.ascontiguousarray(block_of_task, dtype=np.int16)
    eff = np.zeros((sets.n_sets, 4), np.int64)
    cs = sets._c()
    _check(lib().gpref_efficiency(C.byref(cs), _p(bot), _p(eff)), "efficiency")
    return eff


def sched_ratio(sets: Sets, verdict_rows, slot0, n_slots, setting, counts):
    v = np.ascontiguousarray(verdict_rows, dtype=np.uint8)
    assert counts.dtype == np.int64 and counts.flags["C_CONTIGUOUS"]
    cs = sets._c()
    _check(lib().gpref_sched_ratio(C.byref(cs), _p(v), v.shape[0], slot0, n_slots, setting,
                                   _p(counts)), "sched_ratio")
    return counts
