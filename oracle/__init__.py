"""fp64 CPU oracle (test infrastructure only; see dion2_ref.py header)."""
from .dion2_ref import *  # noqa: F401,F403
from .dion2_ref import (OracleConfig, select_count, resolve_axis, l1_scores, select_l1,  # noqa: F401
                        newton_schulz, newton_schulz_auto, dion2_step, muon_step,
                        rms_to_rms_norm, comm_volume, selected_bytes, DEFAULT_NS_COEFFS, DEFAULT_NS_EPS,
                        AXIS_ROWS, AXIS_COLS, AXIS_AUTO, philox4x32_10, random_keys, select_random,
                        dion2_step_dpsync)
