"""Reference-facing operator API over batched CUDA tensors.

Mirrors the reference's operator layer (dl/blas.hpp, dl/cholesky.hpp,
dl/lq.hpp, dl/eigen_sym.hpp, dl/adjoints.hpp): the same names, flags,
in-place / ``_into`` conventions, aliasing rules and exception taxonomy
(dl/common.hpp:20-57), lifted to a leading batch dimension.  Every call goes
through the C-ABI of ``libdla_b200.so`` (include/dla.h) on torch's current
CUDA stream; torch is only the device-memory / stream plumbing.

Shapes: operands are ``[r, c]`` (batch 1) or ``[B, r, c]``; all operands of
one call share B.  Tensors must be contiguous CUDA float32/float64 tensors of
one dtype.  Numerical failures are reported per slice; with ``check=True``
(default) the first failing slice raises the reference's exception type.
"""
from __future__ import annotations

import ctypes as C
import functools
import math

import torch

from ._lib import OPS, STATUS_NAMES, WS_BACKWARD, WS_RIGHTSIDE, lib

__all__ = [
    "Error", "ShapeError", "NotPositiveDefiniteError", "SingularError", "ConvergenceError",
    "gemm2_into", "gemm2", "gemm_into", "syrk_into", "syrk", "trmm_inplace", "trmm", "trsm_inplace",
    "trsm", "potrf_inplace", "potrf", "potri_inplace", "potri", "potri_into", "trmm_into", "sumlogdiag", "gelqf_inplace",
    "gelqf", "syevd_inplace", "syevd", "gemm2_backward_into", "gemm2_backward", "gemm_backward_into",
    "syrk_backward_into", "syrk_backward", "trmm_backward_into", "trmm_backward",
    "trsm_backward_into", "trsm_backward", "potrf_backward_into", "potrf_backward",
    "potri_backward_into", "potri_backward", "sumlogdiag_backward_into", "gelqf_backward_into",
    "gelqf_backward", "syevd_backward_into", "syevd_backward", "eps_gap_default",
    "gesvd_inplace", "gesvd", "gesvd_backward_into", "gesvd_backward",
]


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """dl/common.hpp:20-23"""


class ShapeError(Error):
    """dl/common.hpp:25-28 (also raised for an asymmetric potrf/syevd input)"""


class NotPositiveDefiniteError(Error):
    """dl/common.hpp:30-36; ``step`` is the zero-based global pivot row."""

    def __init__(self, what, step, batch_index=0):
        super().__init__(what)
        self.step = step
        self.batch_index = batch_index


class SingularError(Error):
    """dl/common.hpp:38-45"""

    def __init__(self, what, index, batch_index=0):
        super().__init__(what)
        self.index = index
        self.batch_index = batch_index


class ConvergenceError(Error):
    """dl/common.hpp:47-52"""

    def __init__(self, what, iterations, batch_index=0):
        super().__init__(what)
        self.iterations = iterations
        self.batch_index = batch_index


def _raise_status(st: int, what: str):
    name = STATUS_NAMES.get(st, str(st))
    msg = f"{what}: {lib().lib.dla_status_string(st).decode()} ({name})"
    if st in (1, 6):
        raise ShapeError(msg)
    if st == 5:
        raise Error(msg)
    raise Error(msg)


def _raise_info(st: int, b: int, idx: int, what: str):
    if st == 2:
        raise NotPositiveDefiniteError(f"{what}: pivot {idx} is not positive (slice {b})", idx, b)
    if st == 3:
        raise SingularError(f"{what}: singular at index {idx} (slice {b})", idx, b)
    if st == 4:
        raise ConvergenceError(f"{what}: no convergence after {idx} sweeps (slice {b})", idx, b)
    if st == 6:
        raise ShapeError(f"{what}: input is not symmetric (slice {b})")
    _raise_status(st, what)


# ----------------------------------------------------------------- helpers
def _sfx(t: torch.Tensor) -> str:
    if t.dtype == torch.float64:
        return "f64"
    if t.dtype == torch.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {t.dtype}: float32 / float64 only")


def _dims(t: torch.Tensor, what: str):
    if t.dim() == 2:
        return 1, t.shape[0], t.shape[1]
    if t.dim() == 3:
        return t.shape[0], t.shape[1], t.shape[2]
    raise ShapeError(f"{what}: expected [r, c] or [B, r, c], got {tuple(t.shape)}")


def _prep(what: str, *ts):
    ref = ts[0]
    if not ref.is_cuda:
        raise Error(f"{what}: CUDA tensors required (no CPU path exists)")
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda or t.device != ref.device:
            raise Error(f"{what}: all operands must live on {ref.device}")
        if t.dtype != ref.dtype:
            raise TypeError(f"{what}: dtype mismatch {t.dtype} vs {ref.dtype}")
        if not t.is_contiguous():
            raise Error(f"{what}: operands must be contiguous (packed row-major)")
    batches = {_dims(t, what)[0] for t in ts if t is not None and t.dim() == 3}
    if len(batches) > 1:
        raise ShapeError(f"{what}: batch sizes differ {sorted(batches)}")
    if batches and any(t is not None and t.dim() == 2 for t in ts):
        raise ShapeError(f"{what}: mix of batched and unbatched operands")
    return batches.pop() if batches else 1


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(t):
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _call(name, t, *args):
    st = lib().fn(name, _sfx(t))(*args)
    if st != 0:
        _raise_status(st, name)


def _info(batch, dev):
    return torch.empty(max(batch, 1), dtype=torch.int32, device=dev)


def _check(info, batch, t, what):
    first = C.c_int64(-1)
    idx = C.c_int64(-1)
    st = lib().lib.dla_info_check(C.c_void_p(info.data_ptr()), batch, _stream(t), C.byref(first), C.byref(idx))
    if st != 0:
        _raise_info(st, first.value, idx.value, what)


@functools.lru_cache(maxsize=4096)
def _ws_bytes(op, dt, batch, m, n, k, phase):
    """dla_workspace_bytes is host-only and deterministic: cached per shape."""
    return int(lib().lib.dla_workspace_bytes(op, dt, batch, m, n, k, phase))


def _ws(op, t, batch, m, n, k=0, phase=0):
    """Caller-owned workspace for one call (include/dla.h: the library never
    allocates): dla_workspace_bytes bytes from torch's caching allocator on
    the current stream -- stream-ordered, so it may be recycled by the next
    call on the same stream (every internal fork is joined back to the
    caller's stream before the op returns).  Returns (tensor or None, bytes)."""
    nbytes = _ws_bytes(OPS[op], 1 if t.dtype == torch.float64 else 0, batch, m, n, k, phase)
    if nbytes == 0:
        return None, 0
    return torch.empty(nbytes, dtype=torch.uint8, device=t.device), nbytes


def eps_gap_default(dtype) -> float:
    """ToleranceConfig<T>::defaults().eps_gap (dl/common.hpp:74-80)."""
    return 1e-8 if dtype == torch.float64 else 1e-4


def _shape_of(t):
    return t.shape[-2], t.shape[-1]


# ----------------------------------------------------------------- forward
def gemm_into(c, a, b, ta=False, tb=False, alpha=1.0, beta=0.0):
    """C = alpha op(A) op(B) + beta C (beta 0/1 = gemm_accum, dl/blas.hpp:43-110)."""
    batch = _prep("gemm", c, a, b)
    ar, ac = _shape_of(a)
    br, bc = _shape_of(b)
    m, k = (ac, ar) if ta else (ar, ac)
    kb, n = (bc, br) if tb else (br, bc)
    if k != kb:
        raise ShapeError(f"gemm2: inner dimensions disagree ({k} vs {kb})")
    if _shape_of(c) != (m, n):
        raise ShapeError(f"gemm2: output is {tuple(_shape_of(c))}, expected {m}x{n}")
    ws, nb = _ws("gemm", c, batch, m, n, k)
    _call("gemm_fwd", c, batch, m, n, k, _p(c), _p(a), _p(b), int(ta), int(tb), alpha, beta, _p(ws), nb, _stream(c))
    return c


def gemm2_into(c, a, b, ta=False, tb=False, alpha=1.0):
    """dl/blas.hpp:119-122"""
    return gemm_into(c, a, b, ta, tb, alpha, 0.0)


def gemm2(a, b, ta=False, tb=False, alpha=1.0):
    m = a.shape[-1] if ta else a.shape[-2]
    n = b.shape[-2] if tb else b.shape[-1]
    c = torch.empty(a.shape[:-2] + (m, n), dtype=a.dtype, device=a.device)
    return gemm2_into(c, a, b, ta, tb, alpha)


def syrk_into(b, a, ta=False, alpha=1.0):
    """dl/blas.hpp:138-169 — exactly symmetric output."""
    batch = _prep("syrk", b, a)
    ar, ac = _shape_of(a)
    n, k = (ac, ar) if ta else (ar, ac)
    if _shape_of(b) != (n, n):
        raise ShapeError(f"syrk: output must be {n}x{n}")
    ws, nb = _ws("syrk", b, batch, n, n, k)
    _call("syrk_fwd", b, batch, n, k, _p(b), _p(a), int(ta), alpha, _p(ws), nb, _stream(b))
    return b


def syrk(a, ta=False, alpha=1.0):
    n = a.shape[-1] if ta else a.shape[-2]
    b = torch.empty(a.shape[:-2] + (n, n), dtype=a.dtype, device=a.device)
    return syrk_into(b, a, ta, alpha)


def _tri_check(t, x, rightside, what):
    tr, tc = _shape_of(t)
    if tr != tc:
        raise ShapeError(f"{what}: matrix must be square, got {tr}x{tc}")
    xr, xc = _shape_of(x)
    need = xc if rightside else xr
    if tr != need:
        raise ShapeError(f"{what}: triangular factor is {tr}x{tc}, dense operand is {xr}x{xc}")
    return xr, xc


def trmm_inplace(t, x, rightside=False, transpose=False, lower=True, alpha=1.0):
    """dl/blas.hpp:202-291"""
    batch = _prep("trmm", x, t)
    m, n = _tri_check(t, x, rightside, "trmm")
    ws, nb = _ws("trmm", x, batch, m, n, 0, WS_RIGHTSIDE if rightside else 0)
    _call("trmm_fwd", x, batch, m, n, _p(t), _p(x), int(rightside), int(transpose), int(lower), alpha, _p(ws), nb,
          _stream(x))
    return x


def trmm_into(y, t, x, rightside=False, transpose=False, lower=True, alpha=1.0):
    """y = alpha op(T) x / alpha x op(T), x and t unchanged (dl/blas.hpp:202-291,
    out of place: one triangular GEMM from x into y for n_t >= 128)."""
    batch = _prep("trmm", y, x, t)
    m, n = _tri_check(t, x, rightside, "trmm")
    if y.shape != x.shape:
        raise ShapeError(f"trmm_into: output {tuple(y.shape)} vs operand {tuple(x.shape)}")
    ws, nb = _ws("trmm", x, batch, m, n, 0, WS_RIGHTSIDE if rightside else 0)
    _call("trmm_into", x, batch, m, n, _p(t), _p(x), _p(y), int(rightside), int(transpose), int(lower), alpha,
          _p(ws), nb, _stream(x))
    return y


def trmm(t, x, rightside=False, transpose=False, lower=True, alpha=1.0):
    return trmm_into(torch.empty_like(x), t, x, rightside, transpose, lower, alpha)


def trsm_inplace(t, x, rightside=False, transpose=False, lower=True, alpha=1.0, check=True):
    """dl/blas.hpp:307-395; exact zero diagonal raises SingularError(k)."""
    batch = _prep("trsm", x, t)
    m, n = _tri_check(t, x, rightside, "trsm")
    info = _info(batch, x.device)
    ws, nb = _ws("trsm", x, batch, m, n, 0, WS_RIGHTSIDE if rightside else 0)
    _call("trsm_fwd", x, batch, m, n, _p(t), _p(x), int(rightside), int(transpose), int(lower), alpha,
          _p(info), _p(ws), nb, _stream(x))
    if check:
        _check(info, batch, x, "trsm")
    return x


def trsm(t, x, rightside=False, transpose=False, lower=True, alpha=1.0, check=True):
    return trsm_inplace(t, x.clone(), rightside, transpose, lower, alpha, check)


def _square(a, what):
    r, c = _shape_of(a)
    if r != c:
        raise ShapeError(f"{what}: matrix must be square, got {r}x{c}")
    return r


def potrf_inplace(a, lower=True, check=True, info=None):
    """dl/cholesky.hpp:79-88"""
    batch = _prep("potrf", a)
    n = _square(a, "potrf")
    info = _info(batch, a.device) if info is None else info
    ws, nb = _ws("potrf", a, batch, n, n)
    _call("potrf_fwd", a, batch, n, _p(a), int(lower), _p(info), _p(ws), nb, _stream(a))
    if check:
        _check(info, batch, a, "potrf")
    return a


def potrf(a, lower=True, check=True):
    return potrf_inplace(a.clone(), lower, check)


def potri_inplace(a, lower=True, check=True):
    """dl/cholesky.hpp:141-147"""
    batch = _prep("potri", a)
    n = _square(a, "potri")
    info = _info(batch, a.device)
    ws, nb = _ws("potri", a, batch, n, n)
    _call("potri_fwd", a, batch, n, _p(a), int(lower), _p(info), _p(ws), nb, _stream(a))
    if check:
        _check(info, batch, a, "potri")
    return a


def potri_into(b, l, lower=True, check=True, info=None):
    """b = inv(L L^T) from the factor l, l unchanged (dl/cholesky.hpp:141-147,
    out of place: one fused launch for fp64 64 < n <= 128)."""
    batch = _prep("potri", b, l)
    n = _square(l, "potri")
    if b.shape != l.shape:
        raise ShapeError(f"potri_into: output {tuple(b.shape)} vs factor {tuple(l.shape)}")
    own = info is None
    info = _info(batch, l.device) if own else info
    ws, nb = _ws("potri", l, batch, n, n)
    _call("potri_into", l, batch, n, _p(l), _p(b), int(lower), _p(info), _p(ws), nb, _stream(l))
    if check:
        _check(info, batch, b, "potri")
    return b


def potri(a, lower=True, check=True):
    return potri_into(torch.empty_like(a), a, lower, check)


def sumlogdiag(a, out=None):
    """sum_i log A(i,i) per slice (tape ExtractDiag -> Log -> Sum)."""
    batch = _prep("sumlogdiag", a)
    n = _square(a, "sumlogdiag")
    if out is None:
        out = torch.empty(a.shape[:-2] if a.dim() == 3 else (1,), dtype=a.dtype, device=a.device)
    _call("sumlogdiag_fwd", a, batch, n, _p(out), _p(a), None, 0, _stream(a))
    return out


def chol_chain_fwdbwd(a, y, phi=None, abar=None, ybar=None, check=True, info=None):
    """Fused C1 chain: phi = 1/2 |L^-1 y|^2 + sumlogdiag(L), L = potrf(A), with
    (ybar, Abar) at phibar = 1 -- the make_gp graph of dl/models.hpp:99-103
    given A.  a: [B, n, n], y: [B, n, 1].  One launch for n <= 32."""
    batch = _prep("chol_chain", a, y)
    n = _square(a, "chol_chain")
    if tuple(y.shape[-2:]) != (n, 1):
        raise ShapeError(f"chol_chain: y must be [.., {n}, 1], got {tuple(y.shape)}")
    phi = torch.empty(batch, dtype=a.dtype, device=a.device) if phi is None else phi
    abar = torch.empty_like(a) if abar is None else abar
    ybar = torch.empty_like(y) if ybar is None else ybar
    info = _info(batch, a.device) if info is None else info
    ws, nb = _ws("chol_chain", a, batch, n, n)
    _call("chol_chain_fwdbwd", a, batch, n, _p(a), _p(y), _p(phi), _p(abar), _p(ybar), _p(info), _p(ws), nb,
          _stream(a))
    if check:
        _check(info, batch, a, "chol_chain")
    return phi, abar, ybar


def gelqf_inplace(q, l, check=True):
    """dl/lq.hpp:24-106: q in = A (m x n, m <= n), out = Q; l out = L."""
    batch = _prep("gelqf", q, l)
    m, n = _shape_of(q)
    if m > n:
        raise ShapeError(f"gelqf: need m <= n, got {m}x{n}")
    if _shape_of(l) != (m, m):
        raise ShapeError(f"gelqf: L output must be {m}x{m}")
    ws, nb = _ws("gelqf", q, batch, m, n)
    info = _info(batch, q.device)
    _call("gelqf_fwd", q, batch, m, n, _p(q), _p(l), _p(info), _p(ws), nb, _stream(q))
    if check:
        _check(info, batch, q, "gelqf")
    return q, l


def gelqf(a, check=True):
    q = a.clone()
    m = a.shape[-2]
    l = torch.empty(a.shape[:-2] + (m, m), dtype=a.dtype, device=a.device)
    return gelqf_inplace(q, l, check)


def syevd_inplace(u, lam, check=True):
    """dl/eigen_sym.hpp:339-367: u in = A, out = U (rows eigenvectors); lam ascending."""
    batch = _prep("syevd", u, None)
    n = _square(u, "syevd")
    ws, nb = _ws("syevd", u, batch, n, n)
    info = _info(batch, u.device)
    _call("syevd_fwd", u, batch, n, _p(u), _p(lam), _p(info), _p(ws), nb, _stream(u))
    if check:
        _check(info, batch, u, "syevd")
    return u, lam


def syevd(a, check=True):
    u = a.clone()
    lam = torch.empty(a.shape[:-1], dtype=a.dtype, device=a.device)
    return syevd_inplace(u, lam, check)


def gesvd_inplace(v, u, lam, check=True):
    """dl/svd.hpp:229-284: v in = A (m x n, m <= n), out = V (rows = right
    singular vectors); u out = U (m x m, rows = left singular vectors); lam
    out = singular values, ascending.  A = U^T diag(lam) V."""
    batch = _prep("gesvd", v, u)
    m, n = _shape_of(v)
    if m > n:
        raise ShapeError(f"gesvd: need m <= n, got {m}x{n}")
    if _shape_of(u) != (m, m):
        raise ShapeError(f"gesvd: U output must be {m}x{m}")
    if lam.numel() != batch * m or lam.dtype != v.dtype or not lam.is_contiguous():
        raise ShapeError("gesvd: lambda output must hold batch x m values of the operand dtype")
    ws, nb = _ws("gesvd", v, batch, m, n)
    info = _info(batch, v.device)
    _call("gesvd_fwd", v, batch, m, n, _p(v), _p(u), _p(lam), _p(info), _p(ws), nb, _stream(v))
    if check:
        _check(info, batch, v, "gesvd")
    return u, lam, v


def gesvd(a, check=True):
    """Returns (U, lambda, V) as the reference's GesvdResult (dl/svd.hpp:286-299)."""
    v = a.clone()
    m = a.shape[-2]
    u = torch.empty(a.shape[:-2] + (m, m), dtype=a.dtype, device=a.device)
    lam = torch.empty(a.shape[:-2] + (m,), dtype=a.dtype, device=a.device)
    return gesvd_inplace(v, u, lam, check)


# ---------------------------------------------------------------- backward
def gemm2_backward_into(abar, bbar, cbar, a, b, ta, tb, alpha=1.0):
    """dl/adjoints.hpp:36-49"""
    batch = _prep("gemm2_backward", abar, bbar, cbar, a, b)
    m, n = _shape_of(cbar)
    k = a.shape[-2] if ta else a.shape[-1]
    ws, nb = _ws("gemm2", a, batch, m, n, k, WS_BACKWARD)
    _call("gemm2_bwd", a, batch, m, n, k, _p(abar), _p(bbar), _p(cbar), _p(a), _p(b), int(ta), int(tb), alpha,
          _p(ws), nb, _stream(a))
    return abar, bbar


def gemm2_backward(cbar, a, b, ta, tb, alpha=1.0):
    return gemm2_backward_into(torch.empty_like(a), torch.empty_like(b), cbar, a, b, ta, tb, alpha)


def gemm_backward_into(abar, bbar, cbar_io, a, b, ta, tb, alpha=1.0, beta=0.0):
    """gemm pullback: abar/bbar as gemm2, then cbar_io <- beta * cbar_io."""
    batch = _prep("gemm_backward", abar, bbar, cbar_io, a, b)
    m, n = _shape_of(cbar_io)
    k = a.shape[-2] if ta else a.shape[-1]
    ws, nb = _ws("gemm", a, batch, m, n, k, WS_BACKWARD)
    _call("gemm_bwd", a, batch, m, n, k, _p(abar), _p(bbar), _p(cbar_io), _p(a), _p(b), int(ta), int(tb), alpha,
          beta, _p(ws), nb, _stream(a))
    return abar, bbar, cbar_io


def syrk_backward_into(abar, bbar, a, ta, alpha=1.0):
    """dl/adjoints.hpp:69-78"""
    batch = _prep("syrk_backward", abar, bbar, a)
    ar, ac = _shape_of(a)
    n, k = (ac, ar) if ta else (ar, ac)
    ws, nb = _ws("syrk", a, batch, n, n, k, WS_BACKWARD)
    _call("syrk_bwd", a, batch, n, k, _p(abar), _p(bbar), _p(a), int(ta), alpha, _p(ws), nb, _stream(a))
    return abar


def syrk_backward(bbar, a, ta, alpha=1.0):
    return syrk_backward_into(torch.empty_like(a), bbar, a, ta, alpha)


def trmm_backward_into(abar, tbar, bbar, t, a, rightside, transpose, lower, alpha=1.0):
    """dl/adjoints.hpp:94-110; abar may alias bbar."""
    batch = _prep("trmm_backward", abar, tbar, bbar, t, a)
    m, n = _tri_check(t, a, rightside, "trmm_backward")
    ws, nb = _ws("trmm", a, batch, m, n, 0, WS_BACKWARD | (WS_RIGHTSIDE if rightside else 0))
    _call("trmm_bwd", a, batch, m, n, _p(abar), _p(tbar), _p(bbar), _p(t), _p(a), int(rightside), int(transpose),
          int(lower), alpha, _p(ws), nb, _stream(a))
    return abar, tbar


def trmm_backward(bbar, t, a, rightside, transpose, lower, alpha=1.0):
    return trmm_backward_into(torch.empty_like(a), torch.empty_like(t), bbar, t, a, rightside, transpose, lower,
                              alpha)


def trsm_backward_into(abar, tbar, bbar, t, b, rightside, transpose, lower, alpha=1.0):
    """dl/adjoints.hpp:131-153; reads the forward OUTPUT b; abar may alias bbar."""
    batch = _prep("trsm_backward", abar, tbar, bbar, t, b)
    m, n = _tri_check(t, b, rightside, "trsm_backward")
    ws, nb = _ws("trsm", b, batch, m, n, 0, WS_BACKWARD | (WS_RIGHTSIDE if rightside else 0))
    _call("trsm_bwd", b, batch, m, n, _p(abar), _p(tbar), _p(bbar), _p(t), _p(b), int(rightside), int(transpose),
          int(lower), alpha, _p(ws), nb, _stream(b))
    return abar, tbar


def trsm_backward(bbar, t, b, rightside, transpose, lower, alpha=1.0):
    return trsm_backward_into(torch.empty_like(b), torch.empty_like(t), bbar, t, b, rightside, transpose, lower,
                              alpha)


def potrf_backward_into(abar, lbar, l, lower=True):
    """dl/adjoints.hpp:175-191; abar may alias lbar."""
    batch = _prep("potrf_backward", abar, lbar, l)
    n = _square(l, "potrf_backward")
    ws, nb = _ws("potrf", l, batch, n, n, 0, WS_BACKWARD)
    _call("potrf_bwd", l, batch, n, _p(abar), _p(lbar), _p(l), int(lower), _p(ws), nb, _stream(l))
    return abar


def potrf_backward(lbar, l, lower=True):
    return potrf_backward_into(torch.empty_like(l), lbar, l, lower)


def potri_backward_into(lbar_out, bbar, l, b, lower=True):
    """dl/adjoints.hpp:207-223"""
    batch = _prep("potri_backward", lbar_out, bbar, l, b)
    n = _square(l, "potri_backward")
    ws, nb = _ws("potri", l, batch, n, n, 0, WS_BACKWARD)
    _call("potri_bwd", l, batch, n, _p(lbar_out), _p(bbar), _p(l), _p(b), int(lower), _p(ws), nb, _stream(l))
    return lbar_out


def potri_backward(bbar, l, b, lower=True):
    return potri_backward_into(torch.empty_like(l), bbar, l, b, lower)


def sumlogdiag_backward_into(abar, gbar, a, accumulate=False):
    """abar(i,i) (+)= gbar / A(i,i); off-diagonal exactly zero (or untouched)."""
    batch = _prep("sumlogdiag_backward", abar, a)
    n = _square(a, "sumlogdiag_backward")
    gbar = gbar.reshape(-1).contiguous()
    if gbar.numel() != batch:
        raise ShapeError("sumlogdiag_backward: one cotangent per slice")
    _call("sumlogdiag_bwd", a, batch, n, _p(abar), _p(gbar), _p(a), int(accumulate), None, 0, _stream(a))
    return abar


def gelqf_backward_into(abar, qbar, lbar, q, l):
    """dl/adjoints.hpp:239-252 (one m x m workspace per slice)."""
    batch = _prep("gelqf_backward", abar, qbar, lbar, q, l)
    m, n = _shape_of(q)
    ws, nb = _ws("gelqf", q, batch, m, n, 0, WS_BACKWARD)
    _call("gelqf_bwd", q, batch, m, n, _p(abar), _p(qbar), _p(lbar), _p(q), _p(l), _p(ws), nb, _stream(q))
    return abar


def gelqf_backward(qbar, lbar, q, l):
    return gelqf_backward_into(torch.empty_like(q), qbar, lbar, q, l)


def syevd_backward_into(abar, ubar, lambdabar, u, lam, eps_gap=None):
    """dl/adjoints.hpp:272-295 (one n x n workspace per slice)."""
    batch = _prep("syevd_backward", abar, ubar, u)
    n = _square(u, "syevd_backward")
    if eps_gap is None:
        eps_gap = eps_gap_default(u.dtype)
    ws, nb = _ws("syevd", u, batch, n, n, 0, WS_BACKWARD)
    lambdabar = lambdabar.contiguous()
    lam = lam.contiguous()
    _call("syevd_bwd", u, batch, n, _p(abar), _p(ubar), _p(lambdabar), _p(u), _p(lam), eps_gap, _p(ws), nb,
          _stream(u))
    return abar


def syevd_backward(ubar, lambdabar, u, lam, eps_gap=None):
    return syevd_backward_into(torch.empty_like(u), ubar, lambdabar, u, lam, eps_gap)


def gesvd_backward_into(abar, ubar, lambdabar, vbar, u, lam, v, eps_gap=None, check=True):
    """dl/adjoints.hpp:315-382; abar may alias vbar.  Raises SingularError(i)
    when lambda_i <= eps_gap (the reference's throw)."""
    batch = _prep("gesvd_backward", abar, ubar, vbar, u, v)
    m, n = _shape_of(v)
    if eps_gap is None:
        eps_gap = eps_gap_default(v.dtype)
    ws, nb = _ws("gesvd", v, batch, m, n, 0, WS_BACKWARD)
    info = _info(batch, v.device)
    lambdabar = lambdabar.contiguous()
    lam = lam.contiguous()
    _call("gesvd_bwd", v, batch, m, n, _p(abar), _p(ubar), _p(lambdabar), _p(vbar), _p(u), _p(lam), _p(v), eps_gap,
          _p(info), _p(ws), nb, _stream(v))
    if check:
        _check(info, batch, v, "gesvd_backward")
    return abar


def gesvd_backward(ubar, lambdabar, vbar, u, lam, v, eps_gap=None):
    return gesvd_backward_into(torch.empty_like(v), ubar, lambdabar, vbar, u, lam, v, eps_gap)
