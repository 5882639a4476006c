"""Thin Python binding of the C ABI in ``include/gpart.h`` (libgpart.so, sm_100a).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the ABI.  PyTorch provides device memory and the stream.
Each function keeps the ABI's name and raises ``GpError`` on a non-OK status.
There is no CPU fallback: if the library is missing, importing raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GP_LIB") or os.path.join(_HERE, "libgpart.so")  # GP_LIB: A/B builds

GP_OK, GP_EINVAL, GP_EOVERFLOW, GP_ECUDA = 0, 1, 2, 3
GP_1G, GP_SMS_ACT, GP_SMS_INA, GP_BF_ACT, GP_BF_INA = range(5)
VARIANTS = {"1G": GP_1G, "SMS_ACT": GP_SMS_ACT, "SMS_INA": GP_SMS_INA, "BF_ACT": GP_BF_ACT,
            "BF_INA": GP_BF_INA}
GP_FROM_VERDICTS, GP_EXHAUSTIVE, GP_THRESHOLD, GP_FROM_PER_SET = 0, 1, 2, 3
GP_EX_NO_HASH = 1
GP_EX_PER_CANDIDATE = 2  # force the per-candidate EXHAUSTIVE evaluator
GP_EX_STATS_EXT = 4  # stats has 12 slots: + runs walked / live, closed-form sweeps / their runs,
                     # corner-table blocks / their sweeps, full-corner allocations / their blocks
GP_EX_FORCE_RANGES = 8  # test hook: bit-sliced evaluator walks verdict words range by range
GP_EX_NATURAL_ORDER = 16  # accepted, no effect (index-order lanes are the only order now)
GP_EX_NO_FULL_CORNER = 64  # test hook: bit-sliced evaluator without the full-corner closed form
GP_EX_GENERIC = 32  # test hook: per-candidate evaluator without shape specialisation
UINT64_MAX = 2**64 - 1

FIELDS_I32 = ("T", "D", "B", "cn", "cc", "fn", "fc")


class GpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"gpart status {status}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                      "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
_lib = C.CDLL(LIB_PATH)


class _TaskSetsC(C.Structure):
    _fields_ = [("n_sets", C.c_int32), ("n_tasks", C.c_int32), ("M", C.c_int32),
                ("n_groups", C.c_int32)] + [
        (f, C.c_void_p) for f in FIELDS_I32 + ("type", "valid", "group")]


class _GenC(C.Structure):
    _fields_ = [("M", C.c_int32), ("n_tasks", C.c_int32), ("n_bins", C.c_int32),
                ("n_prm", C.c_int32), ("sets_per_group", C.c_int32), ("prm_q", C.c_void_p),
                ("ticks_per_unit", C.c_int32), ("n_periods", C.c_int32),
                ("period_menu", C.c_void_p), ("b_max", C.c_int32), ("beta_c_num", C.c_int32),
                ("beta_m_num", C.c_int32), ("beta_den", C.c_int32), ("kc_num", C.c_int32),
                ("km_num", C.c_int32), ("k_den", C.c_int32), ("max_attempts", C.c_int32),
                ("curve_gran", C.c_int32)]


class _ExOptsC(C.Structure):
    _fields_ = [("rank_lo", C.c_uint64), ("rank_hi", C.c_uint64), ("per_set", C.c_void_p),
                ("verdict_bits", C.c_void_p), ("words_per_set", C.c_int64),
                ("work_counter", C.c_void_p), ("stats", C.c_void_p), ("flags", C.c_uint32),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_uint64),
                ("size_mask", C.c_void_p), ("tables_key", C.c_void_p)]


_P = C.c_void_p
_lib.gp_last_error.restype = C.c_char_p
_lib.gp_generate.argtypes = [_P, C.c_uint64, C.c_uint64, C.c_int32, _P, _P]
_lib.gp_count_candidates.argtypes = [C.c_int32, C.c_int32, _P]
_lib.gp_enumerate.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_int64, _P, _P, _P]
_lib.gp_wcet.argtypes = [_P, _P, _P, _P, C.c_int64, _P, _P, _P]
_lib.gp_wcet_per_sm.argtypes = [C.c_int32, C.c_int32, _P, C.c_int32, _P, _P, _P]
_lib.gp_allocate.argtypes = [_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
_lib.gp_sched_ratio.argtypes = [_P, C.c_int32, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                _P, _P, _P]
_lib.gp_exhaustive_workspace_size.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int32, C.c_uint32, _P]
for _f in ("gp_generate", "gp_count_candidates", "gp_enumerate", "gp_wcet", "gp_wcet_per_sm",
           "gp_allocate", "gp_sched_ratio", "gp_exhaustive_workspace_size"):
    getattr(_lib, _f).restype = C.c_int

EXPORTS = ("gp_last_error", "gp_generate", "gp_count_candidates", "gp_enumerate", "gp_wcet",
           "gp_wcet_per_sm", "gp_allocate", "gp_sched_ratio", "gp_exhaustive_workspace_size")


def gp_last_error() -> str:
    return _lib.gp_last_error().decode()


def _check(st):
    if st != GP_OK:
        raise GpError(st, gp_last_error())


def _stream(stream=None):
    if stream is None:
        if not torch.cuda.is_available():  # host-side argument checks only
            return C.c_void_p(None)
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    if t is None:
        return None
    assert t.is_contiguous(), "tensors must be contiguous"
    return C.c_void_p(t.data_ptr())


class TaskSets:
    """Device-resident batch of task sets; fields [n_sets][n_tasks] (gpart.h)."""

    def __init__(self, n_sets, n_tasks, M, n_groups, device="cuda"):
        self.n_sets, self.n_tasks, self.M, self.n_groups = n_sets, n_tasks, M, n_groups
        z = lambda dt: torch.zeros((n_sets, n_tasks), dtype=dt, device=device)  # noqa: E731
        for f in FIELDS_I32:
            setattr(self, f, z(torch.int32))
        self.type = z(torch.uint8)
        self.valid = torch.zeros(n_sets, dtype=torch.uint8, device=device)
        self.group = torch.zeros(n_sets, dtype=torch.int32, device=device)

    @classmethod
    def from_host(cls, d: dict, device="cuda", non_blocking=False):
        T = np.asarray(d["T"])
        ts = cls.__new__(cls)
        ts.n_sets, ts.n_tasks = T.shape
        ts.M, ts.n_groups = int(d["M"]), int(d["n_groups"])
        for f in FIELDS_I32 + ("group",):
            setattr(ts, f, torch.as_tensor(np.ascontiguousarray(d[f], np.int32)).to(
                device, non_blocking=non_blocking))
        for f in ("type", "valid"):
            setattr(ts, f, torch.as_tensor(np.ascontiguousarray(d[f], np.uint8)).to(
                device, non_blocking=non_blocking))
        return ts

    def slice(self, a: int, b: int) -> "TaskSets":
        """Sets [a, b) as a view (no copy): the same device memory, offset pointers."""
        ts = TaskSets.__new__(TaskSets)
        ts.n_sets, ts.n_tasks, ts.M, ts.n_groups = b - a, self.n_tasks, self.M, self.n_groups
        for f in FIELDS_I32 + ("type", "valid", "group"):
            setattr(ts, f, getattr(self, f)[a:b])
        return ts

    def to_host(self) -> dict:
        d = dict(M=self.M, n_groups=self.n_groups)
        for f in FIELDS_I32 + ("type", "valid", "group"):
            d[f] = getattr(self, f).cpu().numpy()
        return d

    def struct(self):
        s = _TaskSetsC(self.n_sets, self.n_tasks, self.M, self.n_groups)
        for f in FIELDS_I32 + ("type", "valid", "group"):
            setattr(s, f, getattr(self, f).data_ptr())
        return s

    def nbytes(self):
        return sum(getattr(self, f).numel() * getattr(self, f).element_size()
                   for f in FIELDS_I32 + ("type", "valid", "group"))


def gp_generate(gen: dict, seed: int, rep_begin: int, rep_count: int, out: TaskSets, stream=None):
    prm_q = np.ascontiguousarray(gen["prm_q"], dtype=np.uint64)
    menu = np.ascontiguousarray(gen["period_menu"], dtype=np.int32)
    g = _GenC(gen["M"], gen["n_tasks"], gen["n_bins"], gen["n_prm"], gen["sets_per_group"],
              prm_q.ctypes.data, gen["ticks_per_unit"], len(menu), menu.ctypes.data, gen["b_max"],
              gen["beta_c_num"], gen["beta_m_num"], gen["beta_den"], gen["kc_num"], gen["km_num"],
              gen["k_den"], gen["max_attempts"], gen.get("curve_gran", 0))
    s = out.struct()
    _check(_lib.gp_generate(C.byref(g), seed, rep_begin, rep_count, C.byref(s), _stream(stream)))
    out.M, out.n_groups = s.M, s.n_groups
    return out


def gp_count_candidates(M: int, n: int) -> int:
    out = C.c_uint64(0)
    _check(_lib.gp_count_candidates(M, n, C.byref(out)))
    return out.value


def gp_exhaustive_workspace_size(n_sets, n_tasks, M, n_groups, mode=None, flags=0) -> int:
    """Host-only: device workspace bytes of gp_sched_ratio(mode, flags) for these shapes."""
    out = C.c_uint64(0)
    mode = GP_EXHAUSTIVE if mode is None else mode
    _check(_lib.gp_exhaustive_workspace_size(n_sets, n_tasks, M, n_groups, mode, flags,
                                             C.byref(out)))
    return out.value


def exhaustive_workspace(ts, mode=None, flags=0, device="cuda"):
    """A caller-owned workspace tensor for gp_sched_ratio on ``ts`` (None if 0 bytes)."""
    nb = gp_exhaustive_workspace_size(ts.n_sets, ts.n_tasks, ts.M, ts.n_groups, mode, flags)
    return torch.empty(nb, dtype=torch.uint8, device=device) if nb else None


def gp_enumerate(M, n, first_rank, count, block_of_task=None, block_size=None, stream=None):
    dev = "cuda"
    if block_of_task is None:
        block_of_task = torch.empty((count, n), dtype=torch.int8, device=dev)
    if block_size is None:
        block_size = torch.empty((count, n), dtype=torch.int16, device=dev)
    _check(_lib.gp_enumerate(M, n, first_rank, count, _ptr(block_of_task), _ptr(block_size),
                             _stream(stream)))
    return block_of_task, block_size


def gp_wcet(ts: TaskSets, set_of_cand, block_of_task, block_size, stream=None):
    nc = set_of_cand.numel()
    wcet = torch.empty((nc, ts.n_tasks), dtype=torch.int32, device=set_of_cand.device)
    conflict = torch.empty((nc, ts.n_tasks), dtype=torch.uint8, device=set_of_cand.device)
    s = ts.struct()
    _check(_lib.gp_wcet(C.byref(s), _ptr(set_of_cand), _ptr(block_of_task), _ptr(block_size), nc,
                        _ptr(wcet), _ptr(conflict), _stream(stream)))
    return wcet, conflict


def gp_wcet_per_sm(B, cost_per_sm, f=0, stream=None):
    cost = torch.as_tensor(np.asarray(cost_per_sm, np.int32)).cuda()
    per = torch.empty_like(cost)
    w = torch.empty(1, dtype=torch.int32, device=cost.device)
    _check(_lib.gp_wcet_per_sm(B, cost.numel(), _ptr(cost), f, _ptr(per), _ptr(w), _stream(stream)))
    return per, w


class AllocOut:
    def __init__(self, n_sets, n_tasks, device="cuda"):
        self.ok = torch.empty(n_sets, dtype=torch.uint8, device=device)
        self.block_of_task = torch.empty((n_sets, n_tasks), dtype=torch.int16, device=device)
        self.block_size = torch.empty((n_sets, n_tasks), dtype=torch.int16, device=device)
        self.pi = torch.empty(n_sets, dtype=torch.int32, device=device)
        self.k = torch.empty(n_sets, dtype=torch.int32, device=device)
        self.n_tests = torch.empty(n_sets, dtype=torch.int64, device=device)
        self.efficiency = None  # optional [n_sets][4] (f2), allocate with want_efficiency()

    def want_efficiency(self):
        self.efficiency = torch.empty((self.ok.shape[0], 4), dtype=torch.int64,
                                      device=self.ok.device)
        return self

    def to_host(self):
        d = {k: getattr(self, k).cpu().numpy()
             for k in ("ok", "block_of_task", "block_size", "pi", "k", "n_tests")}
        if self.efficiency is not None:
            d["efficiency"] = self.efficiency.cpu().numpy()
        return d


def _size_mask(M, sizes):
    """Admissible partition sizes (f4) -> ceil(M/32) host words (None -> None)."""
    if sizes is None:
        return None
    mask = (C.c_uint32 * ((M + 31) // 32))()
    for m in sizes:
        if not 1 <= int(m) <= M:
            raise GpError(GP_EINVAL, f"admissible size {m} outside 1..M")
        mask[(int(m) - 1) // 32] |= 1 << ((int(m) - 1) % 32)
    return mask


class _AllocOptsC(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("size_mask", C.c_void_p), ("memo", C.c_void_p),
                ("memo_stride", C.c_int64)]


GP_AL_BINARY_MERGE = 1  # f4: Algorithm 2 by binary search
GP_AL_INCREASING = 2    # f4: par_list in increasing utilisation
GP_AL_STATS_EXT = 4     # stats has 8 slots (+ tests run, selections, partitions scanned, searches)


def gp_allocate(ts: TaskSets, variant, out: AllocOut = None, stream=None, stats=None, flags=0,
                sizes=None, memo=None, memo_stride=0):
    """A5 heuristics / 1G.  f4: ``flags`` (GP_AL_*) and ``sizes`` = admissible
    partition sizes (iterable of ints; None = every size).  ``memo``: a device pointer (int)
    or tensor holding the block verdict words of an EXHAUSTIVE call on the same sets (its
    workspace, subset-major; gpart.h gp_alloc_opts.memo), ``memo_stride`` the words between
    its subsets' rows (0 = n_sets)."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    if out is None:
        out = AllocOut(ts.n_sets, ts.n_tasks, ts.T.device)
    s = ts.struct()
    opts = None
    if stats is not None and stats.numel() >= 8:
        flags |= GP_AL_STATS_EXT
    if flags or sizes is not None or memo is not None:
        mask = _size_mask(ts.M, sizes)
        mp = None if memo is None else (memo if isinstance(memo, int) else memo.data_ptr())
        opts = _AllocOptsC(int(flags), C.cast(mask, C.c_void_p) if mask is not None else None,
                           mp, int(memo_stride))
        opts._keep = mask
    _check(_lib.gp_allocate(C.byref(s), v, C.byref(opts) if opts is not None else None,
                            _ptr(out.ok), _ptr(out.block_of_task),
                            _ptr(out.block_size), _ptr(out.pi), _ptr(out.k), _ptr(out.n_tests),
                            _ptr(out.efficiency), _ptr(stats), _stream(stream)))
    return out


def gp_sched_ratio(ts: TaskSets, mode, counts, verdicts=None, slot0=0, n_slots=None, setting=0,
                   per_set=None, verdict_bits=None, words_per_set=0, work_counter=None,
                   stats=None, rank_lo=0, rank_hi=UINT64_MAX, stream=None, flags=0,
                   workspace=None, sizes=None, tables_key=None):
    """FROM_VERDICTS: verdicts uint8 [n_rows][n_sets]; EXHAUSTIVE: per_set int64 [n_sets][4]
    (+ work_counter int64 [>=1], optional verdict_bits int32/uint32 [n_sets][words], stats
    int64 [4], or [12] for the bit-sliced evaluator's run counters; optional workspace: a
    uint8 device tensor of >= gp_exhaustive_workspace_size() bytes, else the call makes a
    stream-ordered temporary).  counts int64 [n_settings][n_groups][n_slots][3] is
    accumulated.  ``sizes``: admissible partition sizes for EXHAUSTIVE / THRESHOLD (f4,
    reading B-9; None = every size).  ``tables_key``: a ctypes.c_uint64 kept with the
    workspace (gpart.h gp_exhaustive_opts.tables_key: the workspace's input-independent
    tables are built once and reused while the key matches)."""
    s = ts.struct()
    if stats is not None and stats.numel() >= 12 and mode == GP_EXHAUSTIVE:
        flags |= GP_EX_STATS_EXT
    if mode in (GP_EXHAUSTIVE, GP_THRESHOLD, GP_FROM_PER_SET):
        n_rows = 1
        ex = _ExOptsC(rank_lo, rank_hi, _ptr(per_set), _ptr(verdict_bits), words_per_set,
                      _ptr(work_counter), _ptr(stats), flags, _ptr(workspace),
                      0 if workspace is None else workspace.numel() * workspace.element_size())
        mask = _size_mask(ts.M, sizes)
        if mask is not None:
            ex.size_mask = C.cast(mask, C.c_void_p)
            ex._keep = mask
        if tables_key is not None:
            ex.tables_key = C.cast(C.pointer(tables_key), C.c_void_p)
        exp = C.byref(ex)
        vp = None
    else:
        n_rows = verdicts.shape[0]
        exp = None
        vp = _ptr(verdicts)
    if n_slots is None:
        n_slots = counts.shape[-2] if counts is not None else 1
    _check(_lib.gp_sched_ratio(C.byref(s), mode, vp, n_rows, slot0, n_slots, setting,
                               _ptr(counts), exp, _stream(stream)))
    return counts
