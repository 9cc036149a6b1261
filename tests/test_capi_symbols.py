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
