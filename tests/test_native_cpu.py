"""CPU-side checks of the product library: the C-ABI shared library loads and
exports every entry point include/noma_cuda.h declares, and its host-only
helpers agree with the reference layout (no device needed)."""
import ctypes
import os
import re

import pytest

from paper_2206_05998_b200 import native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "noma_cuda.h")


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build()
    return N.load()


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"NOMA_API\s+[\w\s\*]+?\b(noma_\w+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    assert declared_symbols() == sorted(N.EXPORTED)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {N.LIB_PATH}").read()
    exported = set(re.findall(r" T (noma_\w+)", out))
    assert set(declared_symbols()) <= exported
    # nothing but the C-ABI is exported
    assert all(s.startswith("noma_") for s in exported)


def test_plan_size_and_param_count_match_reference_layout(lib, O):
    for dims in ([32, 64], [32, 64, 64], [128, 64], [64, 64], [8, 64, 64, 64], [1, 1], [8]):
        assert N.plan_size(dims) == O.plan_size(dims)
        assert N.param_count(dims) == O.param_count(dims)


def test_version(lib):
    assert lib.noma_version() == 1


def test_context_creation_fails_loudly_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(N.NomaError):
        N.Context(0)
