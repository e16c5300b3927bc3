"""The C++ drop-in headers (include/linrec/cuda_scan.hpp, cuda_layers.hpp)
exercised by a C++ program the way a reference C++ call site would use them
(tests/cpp/test_cuda_api.cpp, built by `make cpp-tests`)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_api_program():
    exe = os.path.join(ROOT, "build", "test_cuda_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpp-tests"], check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    if out.returncode == 2 and "no CUDA device" in out.stderr:
        pytest.skip("no CUDA device")
    assert out.returncode == 0, out.stderr[-3000:]
    assert "ALL OK" in out.stdout
