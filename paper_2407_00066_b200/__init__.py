"""paper_2407_00066_b200 -- B200-native batched compressed-LoRA apply ("Compress then Serve",
arXiv 2407.00066).  The compute lives in libcts.so (csrc/, sm_100a); this package is its binding.
"""
from .api import (  # noqa: F401
    Bank,
    Plan,
    cts_apply,
    cts_apply_group,
    cts_project,
    cts_expand_group,
    cts_shrink_group,
    cts_expand,
    cts_launch_count,
    cts_shrink,
    cts_bank_bytes,
    cts_bank_free,
    cts_bank_load,
    cts_bank_params,
    cts_plan_create,
    cts_plan_error,
    cts_plan_free,
    cts_plan_partial_elems,
    cts_shrink_partial_group,
    cts_expand_reduced_group,
    cts_plan_max_tiles,
    cts_segment,
    cts_segment_readback,
)
from ._lib import LIB_PATH, CtsError, CtsLibraryError, lib  # noqa: F401
