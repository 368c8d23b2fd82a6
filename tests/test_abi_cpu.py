"""CPU-side checks of the C-ABI boundary (no GPU needed).

* libdla_b200.so loads and exports every symbol include/dla.h declares;
* the header and the Python binding agree on the entry-point list;
* status strings / workspace queries answer without a device (host-only
  entry points);
* the Python operator layer refuses CPU tensors (there is no CPU fallback).
"""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dla.h")
LIB = os.path.join(ROOT, "paper_1710_08717_b200", "libdla_b200.so")


def header_symbols():
    src = open(HEADER).read()
    names = set(re.findall(r"\b(dla_[a-z0-9_]+)\s*\(", src))
    # expand every DLA_DECLARE_*(T, S) prototype list for f32 / f64
    for macro in re.findall(r"#define DLA_DECLARE_[A-Z]+\(T, S\)(.*?)\n\n", src, re.S):
        for base in re.findall(r"dla_([a-z0-9_]+)_##S\s*\(", macro):
            names.add(f"dla_{base}_f32")
            names.add(f"dla_{base}_f64")
    return {n for n in names if not n.endswith("_")}


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return C.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 44, sorted(syms)
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, f"declared in include/dla.h but not exported: {missing}"


def test_binding_matches_header():
    from paper_1710_08717_b200 import _lib
    assert set(_lib.exported_symbols()) <= header_symbols()
    assert header_symbols() <= set(_lib.exported_symbols())


def test_host_only_entry_points(lib):
    lib.dla_status_string.restype = C.c_char_p
    assert lib.dla_status_string(2) == b"matrix is not positive definite"
    lib.dla_version.restype = C.c_char_p
    assert b"sm_100a" in lib.dla_version()
    lib.dla_workspace_bytes.restype = C.c_size_t
    lib.dla_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int]
    ws = lib.dla_workspace_bytes

    def carve(b):  # common.cuh carve_bound: 256-byte rounding + alignment slack
        return 0 if b == 0 else (b + 255) // 256 * 256 + 256
    # gelqf forward: m reals per slice (tau) on the unblocked path (m < 64);
    # the blocked compact-WY path (m >= 64) also keeps Yc, Z (m x n each),
    # T and W (m x 32 each) and the norm; backward: m*m (dl/adjoints.hpp:1-9)
    assert ws(8, 1, 256, 32, 512, 0, 0) == carve(256 * 32 * 8)
    # f64, 64 <= m <= 512: CholeskyQR2 (A copy + two m x m factors + flags) with the
    # Householder workspace kept for its per-slice fallback
    hh = carve(256 * (2 * 128 * 512 + 2 * 128 * 32 + 128 + 1) * 8)
    assert ws(8, 1, 256, 128, 512, 0, 0) >= carve(256 * 128 * 512 * 8) + 2 * carve(256 * 128 * 128 * 8) + hh
    assert ws(8, 0, 256, 128, 512, 0, 0) == carve(256 * (2 * 128 * 512 + 2 * 128 * 32 + 128 + 1) * 4)  # f32: Householder
    assert ws(8, 0, 256, 128, 512, 0, 1) >= carve(256 * 128 * 128 * 4)
    assert ws(9, 1, 1024, 64, 64, 0, 1) == carve(1024 * 64 * 64 * 8)  # syevd bwd: n*n
    assert ws(5, 1, 1, 64, 64, 0, 0) == 0                              # small potrf: registers / smem only
    assert ws(7, 1, 8, 0, 512, 0, 0) == 0 and ws(7, 1, 8, 0, 512, 0, 1) == 0  # sumlogdiag
    # f64 GEMMs never carve; large f32 products carve packed TF32 hi/lo tiles
    assert ws(0, 1, 4, 1024, 1024, 1024, 0) == 0
    assert ws(0, 0, 4, 1024, 1024, 1024, 0) > 2 * 4 * 2 * 1024 * 1024 * 4
    assert ws(0, 0, 4, 64, 64, 64, 0) == 0
    # inverse-based potrf pullback (n = 64 * 2^k): L^-1 and Phi (2 n^2) + trtri tmp
    n = 1024
    assert ws(5, 1, 2, n, n, 0, 1) >= 2 * (2 * n * n + (n // 2) ** 2) * 8
    # the narrow solve publishes its solution (sentinel buffer) + a ticket
    assert ws(4, 1, 1, 4096, 1, 0, 0) == carve(4096 * 8) + carve(8)
    assert ws(4, 1, 1, 1, 4096, 0, 2) == carve(4096 * 8) + carve(8)   # right side: X is 1 x 4096
    # the split potrf pullback of the GP driver covers the blocked factorization
    lib.dla_potrf_bwd_ws_bytes_f64.restype = C.c_size_t
    lib.dla_potrf_bwd_ws_bytes_f64.argtypes = [C.c_int64, C.c_int64]
    assert lib.dla_potrf_bwd_ws_bytes_f64(1, 4096) > ws(5, 1, 1, 4096, 4096, 0, 0) > 0
    # deterministic, no device needed
    assert ws(3, 0, 3, 300, 700, 0, 2) == ws(3, 0, 3, 300, 700, 0, 2)


def test_shape_and_alias_errors_are_host_side(lib):
    """Validation runs before any launch, so it answers without a GPU."""
    f = lib.dla_gemm2_fwd_f64
    f.restype = C.c_int
    f.argtypes = [C.c_int64] * 4 + [C.c_void_p] * 3 + [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_size_t,
                                                           C.c_void_p]
    buf = C.create_string_buffer(1024)
    p = C.cast(buf, C.c_void_p)
    assert f(1, 3, 3, 3, p, p, p, 0, 0, 1.0, None, 0, None) == 5          # DLA_ERR_ALIAS
    assert f(-1, 3, 3, 3, None, None, None, 0, 0, 1.0, None, 0, None) == 1  # DLA_ERR_SHAPE
    g = lib.dla_gelqf_fwd_f64
    g.restype = C.c_int
    g.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 4 + [C.c_size_t, C.c_void_p]
    assert g(1, 3, 2, None, None, None, None, 0, None) == 1        # m > n: ShapeError


def test_python_layer_has_no_cpu_path():
    torch = pytest.importorskip("torch")
    from paper_1710_08717_b200 import linalg as L
    with pytest.raises(L.Error):
        L.potrf(torch.eye(3, dtype=torch.float64))
