"""paper_2105_10312_b200 -- B200-native (sm_100a) batched, contention-aware
schedulability evaluator for arXiv 2105.10312 (Zahaf et al.).

The hot path lives in ``libgpart.so`` behind the C ABI of ``include/gpart.h``
(gp_generate, gp_count_candidates, gp_enumerate, gp_wcet, gp_wcet_per_sm,
gp_allocate, gp_sched_ratio).  ``gpart`` is the thin binding with the same
names; ``pipeline`` orders the calls of one step.  There is no CPU fallback.
"""
from . import gpart  # noqa: F401  (raises ImportError if libgpart.so is missing)
