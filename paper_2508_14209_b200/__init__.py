"""B200-native (sm_100a) CountSketch -> multisketch -> sketch-and-solve (arXiv 2508.14209).

The compute lives in libcsk.so (C-ABI, include/csk.h); this package is the thin
binding (``csk``) plus the multi-GPU driver (``dist``).  No CPU fallback.
"""
from .csk import (CskError, Plan, cs_apply, cs_plan, cs_plan_from_arrays, launch_count, lib, ms_apply,
                  ms_lstsq, ms_solve, ne_lstsq, profile_enable, profile_read, rc_lstsq, srht_apply, gs_apply, gs_lstsq, cs_lstsq, msh_apply, msh_lstsq)

__all__ = ["CskError", "Plan", "cs_apply", "cs_plan", "cs_plan_from_arrays", "launch_count", "lib", "ms_apply",
           "ms_lstsq", "ms_solve", "ne_lstsq", "profile_enable", "profile_read", "rc_lstsq", "srht_apply", "gs_apply", "gs_lstsq", "cs_lstsq",
           "msh_apply", "msh_lstsq"]
