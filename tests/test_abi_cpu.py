"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/gpart.h declares, validates arguments on the host, and the
product path never touches the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpart.h")
LIB = os.path.join(ROOT, "paper_2105_10312_b200", "libgpart.so")


@pytest.fixture(scope="module")
def G():
    if not os.path.exists(LIB):
        from paper_2105_10312_b200 import _build
        _build.build()
    from paper_2105_10312_b200 import gpart
    return gpart


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:gp_status|const char \*)\s*(gp_\w+)\(", text, re.M)))


def test_header_declares_the_five_calls():
    syms = declared_symbols()
    for s in ("gp_generate", "gp_enumerate", "gp_wcet", "gp_allocate", "gp_sched_ratio",
              "gp_count_candidates", "gp_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(G):
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", nm, re.M), s
    assert set(G.EXPORTS) == set(declared_symbols())


def test_library_is_sm100a(G):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_count_candidates_host_only(G):
    """gp_count_candidates runs on the host (no CUDA): closed forms of C.1.6."""
    assert G.gp_count_candidates(4, 3) == 26
    assert G.gp_count_candidates(8, 6) == 11334
    assert G.gp_count_candidates(20, 6) == 694755
    with pytest.raises(G.GpError) as e:
        G.gp_count_candidates(148, 32)
    assert e.value.status == G.GP_EOVERFLOW
    with pytest.raises(G.GpError) as e:
        G.gp_count_candidates(0, 3)
    assert e.value.status == G.GP_EINVAL
    assert "out of range" in G.gp_last_error()


def test_host_validation_before_any_cuda(G):
    """Malformed arguments are rejected on the host with GP_EINVAL /
    GP_EOVERFLOW -- checkable without a GPU."""
    lib = G._lib
    assert lib.gp_enumerate(0, 3, 0, 1, None, None, None) == G.GP_EINVAL
    assert lib.gp_enumerate(4, 13, 0, 1, None, None, None) == G.GP_EINVAL
    assert lib.gp_enumerate(4, 3, 20, 10, None, None, None) == G.GP_EINVAL  # beyond N_c = 26
    assert lib.gp_wcet_per_sm(5, 0, None, 0, None, None, None) == G.GP_EINVAL  # m = 0
    assert lib.gp_allocate(None, 0, None, None, None, None, None, None, None, None, None, None) == G.GP_EINVAL
    import gp_workloads as W
    gen = W.WORKLOADS["c2"]["gen"](R=10)
    ts = G._TaskSetsC(100, 6, 8, 10)
    bad = dict(gen, n_tasks=40)
    with pytest.raises(G.GpError) as e:
        G.gp_generate(bad, 1, 0, 10, _Fake(ts))
    assert e.value.status == G.GP_EINVAL
    big = dict(gen, M=1024, n_tasks=6)  # M * Tmax * k overflows int32
    with pytest.raises(G.GpError) as e:
        G.gp_generate(big, 1, 0, 10, _Fake(ts))
    assert e.value.status == G.GP_EOVERFLOW


def test_allocate_options_validated_on_host(G):
    """f4 options (gp_alloc_opts): unknown flag bits and a size mask with no
    admissible size in 1..M are GP_EINVAL before any launch (n_sets = 0)."""
    import ctypes as C
    ts = G._TaskSetsC(0, 6, 8, 1)
    lib = G._lib
    bad_flags = G._AllocOptsC(8, None)
    assert lib.gp_allocate(C.byref(ts), 1, C.byref(bad_flags), None, None, None, None, None,
                           None, None, None, None) == G.GP_EINVAL
    mask = (C.c_uint32 * 1)(0xFFFFFF00)  # only sizes 9..32, all above M = 8
    empty = G._AllocOptsC(0, C.cast(mask, C.c_void_p))
    assert lib.gp_allocate(C.byref(ts), 1, C.byref(empty), None, None, None, None, None,
                           None, None, None, None) == G.GP_EINVAL
    assert "admits no size" in G.gp_last_error()
    ok_mask = (C.c_uint32 * 1)(0x80)  # size 8 only
    good = G._AllocOptsC(G.GP_AL_BINARY_MERGE | G.GP_AL_INCREASING, C.cast(ok_mask, C.c_void_p))
    # valid options pass validation (GP_ECUDA here only because there is no device)
    assert lib.gp_allocate(C.byref(ts), 1, C.byref(good), None, None, None, None, None,
                           None, None, None, None) in (G.GP_OK, G.GP_ECUDA)


class _Fake:
    """Stand-in output whose struct() is never dereferenced (host checks fail first)."""

    def __init__(self, s):
        self.s = s
        self.M = self.n_groups = 0

    def struct(self):
        return self.s


def test_product_never_imports_oracle():
    """The product path (package + bench's GPU arm) must not use oracle/."""
    pkg = os.path.join(ROOT, "paper_2105_10312_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "gpref" not in src, f
    csrc = os.path.join(pkg, "csrc")
    for f in os.listdir(csrc):
        assert not re.search(r"#include\s+[<\"].*oracle", open(os.path.join(csrc, f)).read()), f
