"""B200-native (sm_100a) CountSketch -> multisketch -> sketch-and-solve (arXiv 2508.14209).

The compute lives in libcsk.so (C-ABI, include/csk.h); this package is the thin
binding (``csk``) plus the multi-GPU driver (``dist``).  No CPU fallback.
"""
from .csk import (CskError, Plan, cs_apply, cs_lstsq, cs_plan, cs_plan_from_arrays, gs_apply, gs_lstsq, launch_count,
                  lib, ms_apply, ms_lstsq, ms_solve, ms_solve_async, msh_apply, msh_lstsq, ne_lstsq, profile_enable, profile_read,
                  rc_finish, rc_gram, rc_lstsq, rc_r0, srht_apply)

__all__ = ["CskError", "Plan", "cs_apply", "cs_lstsq", "cs_plan", "cs_plan_from_arrays", "gs_apply", "gs_lstsq",
           "launch_count", "lib", "ms_apply", "ms_lstsq", "ms_solve", "ms_solve_async", "msh_apply", "msh_lstsq", "ne_lstsq",
           "profile_enable", "profile_read", "rc_finish", "rc_gram", "rc_lstsq", "rc_r0", "srht_apply"]
