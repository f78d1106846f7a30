"""B200-native (sm_100a) loop-closing fuse/correct core of arXiv 2603.17201 (FastLoop).

The compute path is liblc.so (paper_2603_17201_b200/csrc, C ABI in include/lc.h);
this package is its thin binding plus the multi-GPU orchestration (dist.py).
"""
from .lc import (COUNTER_NAMES, LC_CORRECT_ALL, LC_CORRECT_WINDOW, LC_FUSE_ALL,  # noqa: F401
                 LC_FUSE_APPLY, LC_FUSE_PLAN, LC_NONE, Context, counts_dict)
