"""The C ABI without a GPU: the library builds, loads, exports every symbol include/cts.h declares,
and the host-side validation that runs before any CUDA call behaves as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2407_00066_b200 import _lib
    return _lib


def header_functions():
    src = open(os.path.join(ROOT, "include", "cts.h")).read()
    return set(re.findall(r"^\s*(?:cts_status_t|int32_t|uint64_t|const char\*)\s+(cts_\w+)\s*\(", src, re.M))


def test_header_and_binding_agree(lib):
    assert header_functions() == set(lib.EXPORTS)


def test_exports_every_symbol(lib):
    L = ctypes.CDLL(lib.LIB_PATH)
    for name in header_functions():
        assert getattr(L, name) is not None


def test_sass_is_sm100a_tcgen05(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", lib.LIB_PATH], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG.2D.GATHER4", "UTMASTG.2D.SCATTER4"):
        assert mnem in out, mnem
    assert "arch = sm_100a" in out


def test_status_strings(lib):
    L = lib.lib()
    assert L.cts_status_string(0) == b"ok"
    assert L.cts_status_string(3) == b"index out of range"


def test_host_validation_before_cuda(lib):
    L = lib.lib()
    out = ctypes.c_void_p()
    assert L.cts_bank_load(None, None, ctypes.byref(out)) == 1            # null desc
    assert L.cts_bank_load(None, None, None) == 1
    d = lib.BankDesc()
    d.n_modules = 0
    dims = (ctypes.c_int32 * 1)(64)
    ptr = (ctypes.c_void_p * 1)(1)
    d.d_in = d.d_out = dims
    d.in_basis = d.out_basis = d.sigma = d.cluster_of = ptr
    assert L.cts_bank_load(ctypes.byref(d), None, ctypes.byref(out)) == 2  # n_modules < 1
    d.n_modules, d.n_adapters, d.n_clusters, d.rank = 1, 4, 1, 65
    assert L.cts_bank_load(ctypes.byref(d), None, ctypes.byref(out)) == 4  # r > 64
    d.rank, d.n_clusters = 4, 1025
    assert L.cts_bank_load(ctypes.byref(d), None, ctypes.byref(out)) == 4  # C > 1024
    d.n_clusters, d.sigma_kind = 1, 7
    assert L.cts_bank_load(ctypes.byref(d), None, ctypes.byref(out)) == 1  # unknown sigma_kind
    assert out.value is None
    assert L.cts_plan_create(None, 16, ctypes.byref(out)) == 1
    assert L.cts_segment(None, None, 4, None) == 1
    assert L.cts_apply(None, 0, None, 64, None, 64, 1.0, None) == 1
    assert L.cts_bank_free(None) == 1 and L.cts_plan_free(None) == 1
    assert L.cts_plan_max_tiles(None, 100) == 0


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2407_00066_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.CtsLibraryError):
        _lib.lib()


def test_comm_validation_before_nccl(lib):
    """cts_comm_* / cts_apply_tp reject bad arguments before touching NCCL or the GPU."""
    L = lib.lib()
    out = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert L.cts_comm_create(None, 2, 0, ctypes.byref(out)) == 1            # no id
    assert L.cts_comm_create(uid, 0, 0, ctypes.byref(out)) == 1             # nranks < 1
    assert L.cts_comm_create(uid, 2, 2, ctypes.byref(out)) == 1             # rank outside [0, nranks)
    assert L.cts_comm_create(uid, 2, 0, None) == 1
    assert out.value is None
    assert L.cts_comm_free(None) == 1
    assert L.cts_comm_unique_id(None) == 1
    assert L.cts_apply_tp(None, 1, None, None, None, None, None, 1.0, None, None) == 1
    assert L.cts_status_string(7) == b"NCCL unavailable or failed"


def test_exclusive_device_flag(lib):
    """cts_set_exclusive_device takes 0 / 1 only; it never touches the GPU."""
    L = lib.lib()
    assert L.cts_set_exclusive_device(2) == 1
    assert L.cts_set_exclusive_device(-1) == 1
    assert L.cts_set_exclusive_device(1) == 0
    assert L.cts_set_exclusive_device(0) == 0


def test_bank_write_clusters_validation(lib):
    """cts_bank_write_clusters rejects a null bank / cluster list before any CUDA call."""
    L = lib.lib()
    cl = (ctypes.c_int32 * 1)(0)
    assert L.cts_bank_write_clusters(None, 0, 1, cl, None, None, None) == 1
