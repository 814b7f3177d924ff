"""CPU suite: the C-ABI library builds, loads and exports every declared
symbol (no compute calls: there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

from paper_2112_06300_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ccdk.h")).read()
    return sorted(set(re.findall(r"\b(ccdk_[a-z_0-9]+)\s*\(", text)))


def test_header_declarations_are_bound():
    decl = declared_symbols()
    assert set(decl) == set(native.exported_symbols()), set(decl) ^ set(native.exported_symbols())


def test_library_loads_and_exports_all_symbols():
    lib = native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.ccdk_abi_version() == 2


def test_no_device_fails_loudly_without_fallback():
    # on a box without a GPU, creating a context must fail with CCDK_CUDA
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(native.CcdkError) as e:
        native.Context(0)
    assert e.value.code == 3


def test_cpp_host_library_exports_reference_api():
    so = os.path.join(ROOT, "paper_2112_06300_b200", "lib", "libccdkit.so")
    if not os.path.exists(so):
        pytest.skip("libccdkit.so not built")
    lib = C.CDLL(so)
    # mangled ccdkit:: entry points of the reference headers
    out = os.popen(f"nm -D --defined-only {so} | c++filt").read()
    for sym in ["ccdkit::build_boxes(", "ccdkit::stq(", "ccdkit::bf(", "ccdkit::sap(",
                "ccdkit::classify(", "ccdkit::narrow_phase(", "ccdkit::ccd(",
                "ccdkit::process_interval(", "ccdkit::inclusion_box(", "ccdkit::choose_axis(",
                "ccdkit::round_down_reduced(", "ccdkit::run_batched(", "ccdkit::ccd_no_zero_toi("]:
        assert sym in out, sym
    del lib
