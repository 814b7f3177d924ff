"""The C++ drop-in API (include/ccdkit/*.hpp, lib/libccdkit.so): compile the
re-authored reference-style test program and run it (GPU), plus a CPU-side
check that it compiles and links against the headers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2112_06300_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_ccdkit_api.cpp")


def _compile(tmp_path):
    exe = str(tmp_path / "test_ccdkit_api")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                        "-L", LIB, "-lccdkit", "-lccdk", f"-Wl,-rpath,{LIB}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_api_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIB, "libccdkit.so")):
        pytest.skip("libccdkit.so not built")
    _compile(tmp_path)


@pytest.mark.gpu
def test_cpp_api_reference_style_suite(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
