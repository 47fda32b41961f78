"""ctypes loader for libcts.so (the C ABI of include/cts.h).  Argument marshalling only.

There is no fallback: if the shared library is missing or fails to load, every entry point raises
`CtsLibraryError`.  Build it with `python -c "import __graft_entry__ as g; g.build()"`.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcts.so")

STATUS = {
    0: "CTS_OK",
    1: "CTS_ERR_INVALID_ARGUMENT",
    2: "CTS_ERR_SHAPE",
    3: "CTS_ERR_INDEX_OUT_OF_RANGE",
    4: "CTS_ERR_UNSUPPORTED",
    5: "CTS_ERR_OUT_OF_MEMORY",
    6: "CTS_ERR_CUDA",
    7: "CTS_ERR_NCCL",
}

# Every symbol include/cts.h declares (tests check the .so exports all of them).
EXPORTS = (
    "cts_bank_load", "cts_bank_bytes", "cts_bank_params", "cts_bank_free",
    "cts_plan_create", "cts_plan_free", "cts_plan_max_tiles",
    "cts_segment", "cts_segment_readback", "cts_apply", "cts_shrink", "cts_expand",
    "cts_apply_group", "cts_shrink_group", "cts_expand_group", "cts_plan_error", "cts_status_string",
    "cts_launch_count", "cts_plan_partial_elems", "cts_shrink_partial_group", "cts_expand_reduced_group",
    "cts_project", "cts_jd_workspace_bytes", "cts_jd_eigen_iteration", "cts_route", "cts_rows_move",
    "cts_comm_unique_id", "cts_comm_create", "cts_comm_free", "cts_apply_tp", "cts_set_exclusive_device",
    "cts_bank_write_clusters",
)


class CtsLibraryError(RuntimeError):
    pass


class CtsError(RuntimeError):
    def __init__(self, fn, code):
        self.code = code
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}")


class JdProblem(ctypes.Structure):
    _fields_ = [
        ("a_stack", ctypes.c_void_p),
        ("bt_stack", ctypes.c_void_p),
        ("n", ctypes.c_int32),
        ("r_i", ctypes.c_int32),
        ("d_in", ctypes.c_int32),
        ("d_out", ctypes.c_int32),
        ("U", ctypes.c_void_p),
        ("V", ctypes.c_void_p),
        ("sigma", ctypes.c_void_p),
    ]


class BankDesc(ctypes.Structure):
    _fields_ = [
        ("n_modules", ctypes.c_int32),
        ("n_adapters", ctypes.c_int32),
        ("n_clusters", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("d_in", ctypes.POINTER(ctypes.c_int32)),
        ("d_out", ctypes.POINTER(ctypes.c_int32)),
        ("in_basis", ctypes.POINTER(ctypes.c_void_p)),
        ("out_basis", ctypes.POINTER(ctypes.c_void_p)),
        ("sigma", ctypes.POINTER(ctypes.c_void_p)),
        ("cluster_of", ctypes.POINTER(ctypes.c_void_p)),
        ("sources_on_device", ctypes.c_int32),
        ("sigma_kind", ctypes.c_int32),
    ]


_lib = None


def lib():
    """Load libcts.so once; raise loudly if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CtsLibraryError(f"{LIB_PATH} not built; run __graft_entry__.build()")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:
        raise CtsLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    P, I32, I64, F, VP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
    sig = {
        "cts_bank_load": ([ctypes.POINTER(BankDesc), P, ctypes.POINTER(P)], I32),
        "cts_bank_bytes": ([P, ctypes.POINTER(ctypes.c_size_t)], I32),
        "cts_bank_params": ([P, I32, ctypes.POINTER(I64)], I32),
        "cts_bank_free": ([P], I32),
        "cts_plan_create": ([P, I32, ctypes.POINTER(P)], I32),
        "cts_plan_free": ([P], I32),
        "cts_plan_max_tiles": ([P, I32], I32),
        "cts_segment": ([P, VP, I32, P], I32),
        "cts_segment_readback": ([P, I32, VP, VP, VP, VP, P], I32),
        "cts_apply": ([P, I32, VP, I64, VP, I64, F, P], I32),
        "cts_shrink": ([P, I32, VP, I64, F, P], I32),
        "cts_expand": ([P, I32, VP, I64, P], I32),
        "cts_apply_group": ([P, I32, VP, VP, VP, VP, VP, F, P], I32),
        "cts_shrink_group": ([P, I32, VP, VP, VP, F, P], I32),
        "cts_expand_group": ([P, I32, VP, VP, VP, P], I32),
        "cts_plan_error": ([P, ctypes.POINTER(I32), ctypes.POINTER(I32)], I32),
        "cts_status_string": ([I32], ctypes.c_char_p),
        "cts_launch_count": ([], ctypes.c_uint64),
        "cts_set_exclusive_device": ([I32], I32),
        "cts_bank_write_clusters": ([P, I32, I32, VP, VP, VP, P], I32),
        "cts_plan_partial_elems": ([P, ctypes.POINTER(I64)], I32),
        "cts_shrink_partial_group": ([P, I32, VP, VP, VP, F, VP, P], I32),
        "cts_expand_reduced_group": ([P, I32, VP, VP, VP, VP, P], I32),
        "cts_project": ([P, I32, VP, I64, VP, I64, VP, I64, F, P], I32),
        "cts_jd_workspace_bytes": ([ctypes.POINTER(JdProblem), I32, I32, ctypes.POINTER(ctypes.c_size_t)], I32),
        "cts_jd_eigen_iteration": ([ctypes.POINTER(JdProblem), I32, I32, I32, VP, ctypes.c_size_t, P], I32),
        "cts_route": ([VP, I32, VP, I32, I32, I32, VP, VP, P], I32),
        "cts_rows_move": ([VP, I64, VP, I64, VP, I32, I32, I32, P], I32),
        "cts_comm_unique_id": ([VP], I32),
        "cts_comm_create": ([VP, I32, I32, ctypes.POINTER(P)], I32),
        "cts_comm_free": ([P], I32),
        "cts_apply_tp": ([P, I32, VP, VP, VP, VP, VP, F, P, P], I32),
    }
    for name, (argt, rest) in sig.items():
        f = getattr(L, name)
        f.argtypes = argt
        f.restype = rest
    _lib = L
    return L


def check(fn, code):
    if code != 0:
        raise CtsError(fn, code)
