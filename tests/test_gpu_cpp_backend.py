"""The reference-side C++ caller (tests/cpp/backend_hook.cpp, built by
__graft_entry__.build() against the reference's own headers): the
KernelBackend<T>::gemm hook (dl/blas.hpp:17-29) over dla_gemm_fwd_{f32,f64},
the replay of proj/tests/test_blas_kernels.cpp:98-129, the reference's own
pullbacks with their products on the device, and direct C-ABI operator
calls from C++ checked against the reference on the same inputs."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "backend_hook")


def test_reference_kernel_backend_hook_on_device():
    assert os.path.exists(BIN), "tests/cpp/_bin/backend_hook missing: run __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
