"""CPU oracle bindings — TEST INFRASTRUCTURE ONLY.

ctypes wrappers over
  * ``oracle/_build/libdla_oracle.so`` — the plain-C restatement of the
    reference algorithms (oracle/oracle_impl.h), kind ``"port"``;
  * ``oracle/_ref/libdla_ref.so`` — the real reference compiled from
    /root/reference/proj/include (oracle/ref_shim.cpp), kind ``"reference"``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

All functions take/return numpy arrays for ONE matrix (row-major), mirroring
the reference's per-slice entry points; batched helpers loop over slices
exactly as the reference's ``for_each_slice`` does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libdla_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdla_ref.so")

DLA_OK, DLA_ERR_SHAPE, DLA_ERR_NOT_SPD, DLA_ERR_SINGULAR = 0, 1, 2, 3
DLA_ERR_CONVERGENCE, DLA_ERR_ALIAS, DLA_ERR_ASYMMETRIC = 4, 5, 6

_i64 = C.c_int64
_int = C.c_int
_vp = C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, status, index=None):
        super().__init__(f"oracle status {status} index {index}")
        self.status = status
        self.index = index


def build(ref: bool = False) -> None:
    """Build the oracle (and, when /root/reference exists and ref=True, _ref)."""
    targets = ["all"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/include") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a):
    return a.ctypes.data_as(_vp) if a is not None else None


def _suffix(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def _ctype(dtype):
    return C.c_double if np.dtype(dtype) == np.float64 else C.c_float


class _Lib:
    """Common per-slice API over either shared object (prefix o_ or ref_)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path

    def fn(self, name, dtype):
        return getattr(self.lib, f"{self.prefix}{name}_{_suffix(dtype)}")

    @staticmethod
    def _chk(st, idx=None):
        if st != DLA_OK:
            raise OracleError(st, None if idx is None else idx.value)

    # --- forward ---------------------------------------------------------
    def gemm(self, a, b, ta=False, tb=False, alpha=1.0, c=None, accumulate=False):
        m = a.shape[1] if ta else a.shape[0]
        k = a.shape[0] if ta else a.shape[1]
        n = b.shape[0] if tb else b.shape[1]
        dt = a.dtype
        out = np.zeros((m, n), dt) if c is None else np.ascontiguousarray(c, dt).copy()
        f = self.fn("gemm", dt)
        ct = _ctype(dt)
        st = f(_i64(m), _i64(n), _i64(k), _ptr(out), _ptr(np.ascontiguousarray(a)),
               _ptr(np.ascontiguousarray(b)), _int(ta), _int(tb), ct(alpha), _int(accumulate))
        self._chk(st)
        return out

    def gemm2(self, a, b, ta=False, tb=False, alpha=1.0):
        return self.gemm(a, b, ta, tb, alpha)

    def syrk(self, a, ta=False, alpha=1.0):
        a = np.ascontiguousarray(a)
        n = a.shape[1] if ta else a.shape[0]
        k = a.shape[0] if ta else a.shape[1]
        out = np.zeros((n, n), a.dtype)
        st = self.fn("syrk", a.dtype)(_i64(n), _i64(k), _ptr(out), _ptr(a), _int(ta),
                                      _ctype(a.dtype)(alpha))
        self._chk(st)
        return out

    def trmm(self, t, x, rightside=False, transpose=False, lower=True, alpha=1.0):
        x = np.array(x, copy=True, order="C")
        t = np.ascontiguousarray(t)
        m, n = x.shape
        st = self.fn("trmm", x.dtype)(_i64(m), _i64(n), _ptr(t), _ptr(x), _int(rightside),
                                      _int(transpose), _int(lower), _ctype(x.dtype)(alpha))
        self._chk(st)
        return x

    def trsm(self, t, x, rightside=False, transpose=False, lower=True, alpha=1.0):
        x = np.array(x, copy=True, order="C")
        t = np.ascontiguousarray(t)
        m, n = x.shape
        idx = _i64(-1)
        st = self.fn("trsm", x.dtype)(_i64(m), _i64(n), _ptr(t), _ptr(x), _int(rightside),
                                      _int(transpose), _int(lower), _ctype(x.dtype)(alpha),
                                      C.byref(idx))
        self._chk(st, idx)
        return x

    def potrf(self, a, lower=True):
        a = np.array(a, copy=True, order="C")
        idx = _i64(-1)
        st = self.fn("potrf", a.dtype)(_i64(a.shape[0]), _ptr(a), _int(lower), C.byref(idx))
        self._chk(st, idx)
        return a

    def potri(self, a, lower=True):
        a = np.array(a, copy=True, order="C")
        idx = _i64(-1)
        st = self.fn("potri", a.dtype)(_i64(a.shape[0]), _ptr(a), _int(lower), C.byref(idx))
        self._chk(st, idx)
        return a

    # --- backward --------------------------------------------------------
    def gemm2_bwd(self, cbar, a, b, ta=False, tb=False, alpha=1.0):
        m, n = cbar.shape
        k = a.shape[0] if ta else a.shape[1]
        abar = np.zeros_like(a)
        bbar = np.zeros_like(b)
        st = self.fn("gemm2_bwd", a.dtype)(_i64(m), _i64(n), _i64(k), _ptr(abar), _ptr(bbar),
                                           _ptr(np.ascontiguousarray(cbar)),
                                           _ptr(np.ascontiguousarray(a)),
                                           _ptr(np.ascontiguousarray(b)), _int(ta), _int(tb),
                                           _ctype(a.dtype)(alpha))
        self._chk(st)
        return abar, bbar

    def syrk_bwd(self, bbar, a, ta=False, alpha=1.0):
        n = bbar.shape[0]
        k = a.shape[0] if ta else a.shape[1]
        abar = np.zeros_like(a)
        st = self.fn("syrk_bwd", a.dtype)(_i64(n), _i64(k), _ptr(abar),
                                          _ptr(np.ascontiguousarray(bbar)),
                                          _ptr(np.ascontiguousarray(a)), _int(ta),
                                          _ctype(a.dtype)(alpha))
        self._chk(st)
        return abar

    def trmm_bwd(self, bbar, t, a, rightside=False, transpose=False, lower=True, alpha=1.0):
        m, n = a.shape
        abar = np.zeros_like(a)
        tbar = np.zeros_like(t)
        st = self.fn("trmm_bwd", a.dtype)(_i64(m), _i64(n), _ptr(abar), _ptr(tbar),
                                          _ptr(np.ascontiguousarray(bbar)),
                                          _ptr(np.ascontiguousarray(t)),
                                          _ptr(np.ascontiguousarray(a)), _int(rightside),
                                          _int(transpose), _int(lower), _ctype(a.dtype)(alpha))
        self._chk(st)
        return abar, tbar

    def trsm_bwd(self, bbar, t, b, rightside=False, transpose=False, lower=True, alpha=1.0):
        m, n = b.shape
        abar = np.zeros_like(b)
        tbar = np.zeros_like(t)
        idx = _i64(-1)
        st = self.fn("trsm_bwd", b.dtype)(_i64(m), _i64(n), _ptr(abar), _ptr(tbar),
                                          _ptr(np.ascontiguousarray(bbar)),
                                          _ptr(np.ascontiguousarray(t)),
                                          _ptr(np.ascontiguousarray(b)), _int(rightside),
                                          _int(transpose), _int(lower), _ctype(b.dtype)(alpha),
                                          C.byref(idx))
        self._chk(st, idx)
        return abar, tbar

    def potrf_bwd(self, lbar, l, lower=True):
        abar = np.zeros_like(l)
        st = self.fn("potrf_bwd", l.dtype)(_i64(l.shape[0]), _ptr(abar),
                                           _ptr(np.ascontiguousarray(lbar)),
                                           _ptr(np.ascontiguousarray(l)), _int(lower))
        self._chk(st)
        return abar

    def potri_bwd(self, bbar, l, b, lower=True):
        lbar = np.zeros_like(l)
        st = self.fn("potri_bwd", l.dtype)(_i64(l.shape[0]), _ptr(lbar),
                                           _ptr(np.ascontiguousarray(bbar)),
                                           _ptr(np.ascontiguousarray(l)),
                                           _ptr(np.ascontiguousarray(b)), _int(lower))
        self._chk(st)
        return lbar


class Port(_Lib):
    """The C restatement (kind "port")."""

    kind = "port"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path, "o_")

    def gelqf(self, a):
        q = np.array(a, copy=True, order="C")
        m, n = q.shape
        l = np.zeros((m, m), q.dtype)
        tau = np.zeros(max(m, 1), q.dtype)
        idx = _i64(-1)
        st = self.fn("gelqf", q.dtype)(_i64(m), _i64(n), _ptr(q), _ptr(l), _ptr(tau), C.byref(idx))
        self._chk(st, idx)
        return q, l

    def syevd(self, a):
        u = np.array(a, copy=True, order="C")
        n = u.shape[0]
        lam = np.zeros(n, u.dtype)
        ws = np.zeros(n * n + 9 * n + 1, u.dtype)
        idx = _i64(-1)
        st = self.fn("syevd", u.dtype)(_i64(n), _ptr(u), _ptr(lam), _ptr(ws), C.byref(idx))
        self._chk(st, idx)
        return u, lam

    def gelqf_bwd(self, qbar, lbar, q, l):
        m, n = q.shape
        abar = np.zeros_like(q)
        work = np.zeros((m, m), q.dtype)
        st = self.fn("gelqf_bwd", q.dtype)(_i64(m), _i64(n), _ptr(abar),
                                           _ptr(np.ascontiguousarray(qbar)),
                                           _ptr(np.ascontiguousarray(lbar)),
                                           _ptr(np.ascontiguousarray(q)),
                                           _ptr(np.ascontiguousarray(l)), _ptr(work))
        self._chk(st)
        return abar

    def syevd_bwd(self, ubar, lambdabar, u, lam, eps_gap=None):
        n = u.shape[0]
        if eps_gap is None:
            eps_gap = 1e-8 if u.dtype == np.float64 else 1e-4
        abar = np.zeros_like(u)
        work = np.zeros((n, n), u.dtype)
        st = self.fn("syevd_bwd", u.dtype)(_i64(n), _ptr(abar), _ptr(np.ascontiguousarray(ubar)),
                                           _ptr(np.ascontiguousarray(lambdabar)),
                                           _ptr(np.ascontiguousarray(u)),
                                           _ptr(np.ascontiguousarray(lam)),
                                           _ctype(u.dtype)(eps_gap), _ptr(work))
        self._chk(st)
        return abar

    def gesvd(self, a):
        """dl/svd.hpp:229-284: (u [m,m], lambda [m] ascending, v [m,n])."""
        v = np.array(a, copy=True, order="C")
        m, n = v.shape
        u = np.zeros((m, m), v.dtype)
        lam = np.zeros(m, v.dtype)
        ws = np.zeros(2 * n * m + 2 * m * m + 2 * m + 1, v.dtype)
        idx = _i64(-1)
        st = self.fn("gesvd", v.dtype)(_i64(m), _i64(n), _ptr(v), _ptr(u), _ptr(lam), _ptr(ws), C.byref(idx))
        self._chk(st, idx)
        return u, lam, v

    def gesvd_bwd(self, ubar, lambdabar, vbar, u, lam, v, eps_gap=None):
        m, n = v.shape
        if eps_gap is None:
            eps_gap = 1e-8 if v.dtype == np.float64 else 1e-4
        abar = np.zeros_like(v)
        work = np.zeros(m * m + m + m * n, v.dtype)
        idx = _i64(-1)
        a = [np.ascontiguousarray(x) for x in (ubar, lambdabar, vbar, u, lam, v)]
        st = self.fn("gesvd_bwd", v.dtype)(_i64(m), _i64(n), _ptr(abar), *[_ptr(x) for x in a],
                                           _ctype(v.dtype)(eps_gap), _ptr(work), C.byref(idx))
        self._chk(st, idx)
        return abar

    def sumlogdiag(self, a):
        f = self.fn("sumlogdiag", a.dtype)
        f.restype = _ctype(a.dtype)
        return f(_i64(a.shape[0]), _ptr(np.ascontiguousarray(a)))

    def sumlogdiag_bwd(self, g, a):
        abar = np.zeros_like(a)
        self.fn("sumlogdiag_bwd", a.dtype)(_i64(a.shape[0]), _ptr(abar), _ctype(a.dtype)(g),
                                           _ptr(np.ascontiguousarray(a)), _int(0))
        return abar

    def fix_row_signs(self, u):
        u = np.array(u, copy=True, order="C")
        self.fn("fix_row_signs", u.dtype)(_i64(u.shape[0]), _i64(u.shape[1]), _ptr(u))
        return u


class Ref(_Lib):
    """The real reference compiled from its headers (kind "reference")."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        super().__init__(path, "ref_")
        L = self.lib
        for s in ("f64", "f32"):
            getattr(L, f"ref_gelqf_fwdbwd_batch_{s}").restype = C.c_double
            getattr(L, f"ref_syevd_fwdbwd_batch_{s}").restype = C.c_double
        L.ref_c1_chain_f64.restype = C.c_double
        L.ref_potrf_fwdbwd_batch_f64.restype = C.c_double

    def gelqf(self, a):
        q = np.array(a, copy=True, order="C")
        m, n = q.shape
        l = np.zeros((m, m), q.dtype)
        idx = _i64(-1)
        st = self.fn("gelqf", q.dtype)(_i64(m), _i64(n), _ptr(q), _ptr(l), C.byref(idx))
        self._chk(st, idx)
        return q, l

    def syevd(self, a):
        u = np.array(a, copy=True, order="C")
        n = u.shape[0]
        lam = np.zeros(n, u.dtype)
        idx = _i64(-1)
        st = self.fn("syevd", u.dtype)(_i64(n), _ptr(u), _ptr(lam), C.byref(idx))
        self._chk(st, idx)
        return u, lam

    def gelqf_bwd(self, qbar, lbar, q, l):
        m, n = q.shape
        abar = np.zeros_like(q)
        st = self.fn("gelqf_bwd", q.dtype)(_i64(m), _i64(n), _ptr(abar),
                                           _ptr(np.ascontiguousarray(qbar)),
                                           _ptr(np.ascontiguousarray(lbar)),
                                           _ptr(np.ascontiguousarray(q)),
                                           _ptr(np.ascontiguousarray(l)))
        self._chk(st)
        return abar

    def syevd_bwd(self, ubar, lambdabar, u, lam, eps_gap=None):
        n = u.shape[0]
        if eps_gap is None:
            eps_gap = 1e-8 if u.dtype == np.float64 else 1e-4
        abar = np.zeros_like(u)
        st = self.fn("syevd_bwd", u.dtype)(_i64(n), _ptr(abar), _ptr(np.ascontiguousarray(ubar)),
                                           _ptr(np.ascontiguousarray(lambdabar)),
                                           _ptr(np.ascontiguousarray(u)),
                                           _ptr(np.ascontiguousarray(lam)),
                                           _ctype(u.dtype)(eps_gap))
        self._chk(st)
        return abar

    def gesvd(self, a):
        v = np.array(a, copy=True, order="C")
        m, n = v.shape
        u = np.zeros((m, m), v.dtype)
        lam = np.zeros(m, v.dtype)
        idx = _i64(-1)
        st = self.fn("gesvd", v.dtype)(_i64(m), _i64(n), _ptr(v), _ptr(u), _ptr(lam), C.byref(idx))
        self._chk(st, idx)
        return u, lam, v

    def gesvd_bwd(self, ubar, lambdabar, vbar, u, lam, v, eps_gap=None):
        m, n = v.shape
        if eps_gap is None:
            eps_gap = 1e-8 if v.dtype == np.float64 else 1e-4
        abar = np.zeros_like(v)
        idx = _i64(-1)
        a = [np.ascontiguousarray(x) for x in (ubar, lambdabar, vbar, u, lam, v)]
        st = self.fn("gesvd_bwd", v.dtype)(_i64(m), _i64(n), _ptr(abar), *[_ptr(x) for x in a],
                                           _ctype(v.dtype)(eps_gap), C.byref(idx))
        self._chk(st, idx)
        return abar

    def sumlogdiag(self, a, with_grad=False):
        a = np.ascontiguousarray(a, np.float64)
        out = C.c_double(0)
        abar = np.zeros_like(a) if with_grad else None
        st = self.lib.ref_sumlogdiag_f64(_i64(a.shape[0]), _ptr(a), C.byref(out), _ptr(abar))
        self._chk(st)
        return (out.value, abar) if with_grad else out.value

    def gp_nll_grad(self, x, y, sigma2, ell2, lam, with_xy=False):
        """make_gp + Graph::backward: [nll, d/dlog sigma2, d/dlog ell2, d/dlog lam]
        (and xbar, ybar when with_xy)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64).reshape(-1)
        out = np.zeros(4)
        xbar = np.zeros_like(x) if with_xy else None
        ybar = np.zeros_like(y) if with_xy else None
        st = self.lib.ref_gp_nll_grad_f64(_i64(x.shape[0]), _i64(x.shape[1]), _ptr(x), _ptr(y),
                                          C.c_double(sigma2), C.c_double(ell2), C.c_double(lam),
                                          _ptr(out), _ptr(xbar), _ptr(ybar))
        self._chk(st)
        return (out, xbar, ybar) if with_xy else out

    # batched timing drivers (reference for_each_slice); return seconds
    def c1_chain(self, a, y, threads=1):
        batch, n, _ = a.shape
        a = np.array(a, copy=True, order="C")
        y = np.array(y, copy=True, order="C")
        abar = np.zeros_like(a)
        phi = np.zeros(batch)
        secs = self.lib.ref_c1_chain_f64(_i64(batch), _i64(n), _ptr(a), _ptr(y), _ptr(abar),
                                         _ptr(phi), _int(threads))
        return secs, dict(l=a, ybar=y, abar=abar, phi=phi)

    def potrf_fwdbwd_batch(self, a, lbar, threads=1):
        batch, n, _ = a.shape
        a = np.array(a, copy=True, order="C")
        abar = np.zeros_like(a)
        secs = self.lib.ref_potrf_fwdbwd_batch_f64(_i64(batch), _i64(n), _ptr(a), _ptr(abar),
                                                   _ptr(np.ascontiguousarray(lbar)), _int(threads))
        return secs, dict(l=a, abar=abar)

    def gelqf_fwdbwd_batch(self, a, qbar, lbar, threads=1):
        batch, m, n = a.shape
        q = np.array(a, copy=True, order="C")
        l = np.zeros((batch, m, m), a.dtype)
        abar = np.zeros_like(q)
        f = self.fn("gelqf_fwdbwd_batch", a.dtype)
        secs = f(_i64(batch), _i64(m), _i64(n), _ptr(q), _ptr(l), _ptr(abar),
                 _ptr(np.ascontiguousarray(qbar)), _ptr(np.ascontiguousarray(lbar)), _int(threads))
        return secs, dict(q=q, l=l, abar=abar)

    def syevd_fwdbwd_batch(self, a, ubar, lambdabar, threads=1):
        batch, n, _ = a.shape
        u = np.array(a, copy=True, order="C")
        lam = np.zeros((batch, n), a.dtype)
        abar = np.zeros_like(u)
        f = self.fn("syevd_fwdbwd_batch", a.dtype)
        secs = f(_i64(batch), _i64(n), _ptr(u), _ptr(lam), _ptr(abar),
                 _ptr(np.ascontiguousarray(ubar)), _ptr(np.ascontiguousarray(lambdabar)),
                 _int(threads))
        return secs, dict(u=u, lam=lam, abar=abar)


def port() -> Port:
    return Port()


def ref() -> Ref:
    return Ref()


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ------------------------------------------------------------------ inputs
# One documented counter-based generator for both sides:
# numpy's Philox bit generator, seeded explicitly; standard normals via
# numpy's ziggurat.  Never std::normal_distribution (libstdc++-specific).

def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def random_spd(n, r, dtype=np.float64, batch=None):
    """X X^T + n I with X ~ N(0,1) (dl/gradcheck.hpp:70-75)."""
    shape = (n, n) if batch is None else (batch, n, n)
    x = r.standard_normal(shape)
    a = x @ np.swapaxes(x, -1, -2)
    a = 0.5 * (a + np.swapaxes(a, -1, -2))
    a += n * np.eye(n)
    return a.astype(dtype)


def random_sym(n, r, dtype=np.float64, batch=None):
    shape = (n, n) if batch is None else (batch, n, n)
    x = r.standard_normal(shape)
    return (0.5 * (x + np.swapaxes(x, -1, -2))).astype(dtype)


LOG_2PI = 1.8378770664093454835606594728112353


def c5_item(p, s, y, theta):
    """TEST INFRASTRUCTURE: phi and dphi/dtheta of one C5 item (SURVEY §8d's
    graph: A = S + e^theta I, L = potrf, B = potri, G = trmm(L, B, left, T),
    v = G y, phi = 1/2 v^T v + sumlogdiag(L) + n/2 log 2 pi) through the
    oracle's per-op pullbacks (dl/adjoints.hpp)."""
    import math
    n = s.shape[0]
    lam = math.exp(theta)
    a = s + lam * np.eye(n)
    l = p.potrf(a)
    b = p.potri(l)
    g = p.trmm(l, b, False, True, True)
    v = p.gemm(g, y)
    phi = 0.5 * float((v.T @ v)[0, 0]) + p.sumlogdiag(l) + 0.5 * n * LOG_2PI
    gbar, _ = p.gemm2_bwd(v, g, y)
    bbar, tbar = p.trmm_bwd(gbar, l, b, False, True, True)
    lbar = p.potri_bwd(bbar, l, b) + tbar + np.diag(1.0 / np.diag(l))
    abar = p.potrf_bwd(lbar, l)
    return phi, lam * np.trace(abar)


def _kalman_call(fn, a, b, sh, sv, mu0, s0, obs, joint=None):
    """Shared argument marshalling of o_kalman_f64 / ref_kalman_f64."""
    h, d = a.shape[0], b.shape[0]
    T = obs.shape[0]
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (a, b, sh, sv, mu0, s0, obs)]
    nll = C.c_double()
    outs = [np.zeros_like(x) for x in arrs]
    args = [_i64(h), _i64(d), _i64(T)] + [_ptr(x) for x in arrs] + [C.byref(nll)] + [_ptr(x) for x in outs]
    return nll, outs, args


def kalman_port(a, b, sh, sv, mu0, s0, obs):
    """Oracle restatement (oracle_impl.h o_kalman): (nll, [Abar, Bbar, Shbar, Svbar, mu0bar, S0bar, obsbar])."""
    lib = port().lib
    nll, outs, args = _kalman_call(None, a, b, sh, sv, mu0, s0, obs)
    idx = _i64(-1)
    st = lib.o_kalman_f64(*args, C.byref(idx))
    if st != DLA_OK:
        raise OracleError(st, idx.value)
    return nll.value, outs


def kalman_ref(a, b, sh, sv, mu0, s0, obs):
    """The reference (make_kalman + Graph::backward): (nll, grads, dense joint-Gaussian NLL)."""
    lib = ref().lib
    nll, outs, args = _kalman_call(None, a, b, sh, sv, mu0, s0, obs)
    joint = C.c_double()
    st = lib.ref_kalman_f64(*args, C.byref(joint))
    if st != DLA_OK:
        raise OracleError(st)
    return nll.value, outs, joint.value


def kalman_ref_batch(a, b, sh, sv, mu0, s0, obs, threads=1):
    """Reference batch loop over sequences (per-sequence parameters): (nll [B], seconds)."""
    lib = ref().lib
    B, h, d, T = a.shape[0], a.shape[1], b.shape[1], obs.shape[1]
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (a, b, sh, sv, mu0, s0, obs)]
    nll = np.zeros(B)
    lib.ref_kalman_batch_f64.restype = C.c_double
    sec = lib.ref_kalman_batch_f64(_i64(B), _i64(h), _i64(d), _i64(T), *[_ptr(x) for x in arrs], _ptr(nll),
                                   _int(threads))
    return nll, sec


def random_kalman(r, h, d, T, batch=None):
    """Stable random linear-Gaussian state-space model as in
    proj/tests/test_models.cpp:199-217 (A = 0.5 N(0,1) at h = 2; scaled by
    sqrt(2/h) above so the spectral radius stays ~0.7), SPD covariances,
    obs ~ N(0, 1)."""
    sc = 0.5 * min(1.0, (2.0 / h) ** 0.5)

    def one():
        a = sc * r.standard_normal((h, h))
        b = r.standard_normal((d, h))
        sh = random_spd(h, r)
        sv = random_spd(d, r)
        mu0 = r.standard_normal((h, 1))
        s0 = random_spd(h, r)
        obs = r.standard_normal((T, d))
        return a, b, sh, sv, mu0, s0, obs
    if batch is None:
        return one()
    items = [one() for _ in range(batch)]
    return tuple(np.stack([it[k] for it in items]) for k in range(7))
