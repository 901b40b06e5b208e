"""B200-native Dion2 optimizer step (arXiv 2512.16928).

The compute path is libdion2.so (hand-written sm_100a CUDA behind the C ABI in
include/dion2.h); this package is the thin Python binding over it.
"""
from .dion2 import (Dion2, Dion2Error, LIB_PATH, describe, get_phase_times, last_launch_count,  # noqa: F401
                    make_config, set_phase_timing, step, workspace_bytes)
