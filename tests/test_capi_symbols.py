"""The C-ABI library loads on CPU and exports exactly what include/deft_b200.h
declares (no compute calls: there is no GPU here)."""
import re
import subprocess

from conftest import ROOT
from paper_2503_16815_b200 import _native


def header_functions():
    text = (ROOT / "include" / "deft_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(deft_[a-z0-9_]+)\s*\(", text))


def test_header_matches_binding_table():
    assert header_functions() == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()  # loads without a GPU
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(deft_[a-z0-9_]+)$", out, flags=re.M))
    missing = header_functions() - exported
    assert not missing, missing
    for name in header_functions():
        assert getattr(lib, name) is not None


def test_pure_host_entry_points():
    lib = _native.lib()
    assert lib.deft_abi_version() == 1
    assert lib.deft_launch_count() >= 0
    assert lib.deft_comm_flag_bytes(8) > 0


def test_product_path_fails_loudly_without_cuda():
    import pytest
    import torch
    import paper_2503_16815_b200 as D
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(D.DeftError):
        D.naive_knapsack([D.Item(1, 3), D.Item(2, 4)], 5)


def test_argument_errors_are_reported_without_a_device():
    """Entry points validate their arguments before any CUDA call: a bad call
    returns DEFT_ERR_INVALID_ARGUMENT, leaves a message in deft_last_error and
    is re-raised by the Python layer as the reference's DeftError
    (errors.py; knapsack.py:61-62 style argument errors)."""
    import ctypes
    import pytest
    import paper_2503_16815_b200 as D
    lib = _native.lib()
    null = ctypes.c_void_p()
    i64 = (ctypes.c_int64 * 1)(0)
    calls = {
        "deft_bucket_reduce_scatter": lambda: lib.deft_bucket_reduce_scatter(
            null, 0, 0, 0, 16, null),
        "deft_bucket_reduce_scatter_multi": lambda: lib.deft_bucket_reduce_scatter_multi(
            null, 0, 0, 1, i64, i64, null),
        "deft_bucket_update": lambda: lib.deft_bucket_update(
            null, 0, 0, 16, 0.1, 0.9, 1.0, null, null),
        "deft_bucket_update_multi": lambda: lib.deft_bucket_update_multi(
            null, 0, 1, i64, i64, 0.1, 0.9, 1.0, null, null),
        "deft_comm_set_update_blocks": lambda: lib.deft_comm_set_update_blocks(null, 8),
        "deft_gather_segments": lambda: lib.deft_gather_segments(
            null, None, None, None, 1, 0, null),
    }
    for name, call in calls.items():
        rc = call()
        assert rc == -1, (name, rc)                        # DEFT_ERR_INVALID_ARGUMENT
        assert lib.deft_last_error(), name
        with pytest.raises(D.DeftError):
            _native.check(rc, name)
    assert lib.deft_comm_destroy(null) == 0                # destroying nothing is fine
