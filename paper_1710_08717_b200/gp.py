"""Gaussian-process negative log marginal likelihood + gradient on device.

The graph is exactly the reference's ``make_gp`` + ``Graph::backward``
(dl/models.hpp:94-135, dl/tape.hpp:461-484), evaluated over a leading batch
of independent GP problems:

    A   = sigma2 * exp(-dist(x) / (2 ell2)) + lam I      (fused RBF build)
    L   = potrf(A)                                        (C-ABI op)
    z   = trsm(L, y)                                      (C-ABI op)
    phi = 1/2 z^T z + sumlogdiag(L) + n/2 log 2 pi        (gemm2, sumlogdiag)
  backward, phibar = 1:
    zbar = z;  (ybar, Lbar) = trsm_backward(zbar, L, z)   (C-ABI op)
    Lbar += diag(1 / L_ii)                                (sumlogdiag_backward)
    Abar = potrf_backward(Lbar, L)                        (C-ABI op, split:
           L^-1 forms on a side stream from right after potrf, overlapping
           the solves; dla_potrf_bwd_{begin,end}_f64, bitwise = the op)
    (d/dlog sigma2, d/dlog ell2, d/dlog lam, xbar) = RBF pullback(Abar)
  by default the last two are one call (dla_gp_pullback_f64): Abar's
  symmetrization is folded into a tile-pair RBF pullback that reads
  Z = L^-T P' L^-1 directly (half the exp work, no Abar pass).

Every step is a libdla_b200.so call on torch's current stream; the driver
allocates all buffers once so a step can be captured in a CUDA graph.
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import linalg as L
from ._lib import lib

LOG_2PI = 1.8378770664093454835606594728112353
_EARLY = __import__("os").environ.get("DLA_GP_EARLY", "1") != "0"
# the pullback tail fused (dla_gp_pullback_f64: Z -> symmetric RBF pullback, no Abar pass)
_FUSED_TAIL = __import__("os").environ.get("DLA_GP_FUSED_TAIL", "1") != "0"


class GPNLL:
    """Batched GP NLL + gradient with preallocated device buffers (fp64)."""

    def __init__(self, n: int, d: int, batch: int = 1, device="cuda", want_xbar: bool = True):
        self.n, self.d, self.batch = n, d, batch
        self.device = torch.device(device)
        f = dict(dtype=torch.float64, device=self.device)
        self.a = torch.empty(batch, n, n, **f)         # A, then L
        self.lbar = torch.empty(batch, n, n, **f)      # Lbar, then Abar (in place)
        self.z = torch.empty(batch, n, 1, **f)
        self.ybar = torch.empty(batch, n, 1, **f)
        self.quad = torch.empty(batch, 1, 1, **f)
        self.logdet = torch.empty(batch, **f)
        self.ones = torch.ones(batch, **f)
        self.grads = torch.empty(batch, 3, **f)
        self.xbar = torch.empty(batch, n, d, **f) if want_xbar else None
        self.nll = torch.empty(batch, **f)
        self.info = torch.zeros(batch, dtype=torch.int32, device=self.device)
        nb = int(lib().lib.dla_gp_pullback_ws_bytes(batch, n, d))
        self.ws = torch.empty(max(nb, 8), dtype=torch.uint8, device=self.device)
        self.ws_bytes = nb
        # split potrf pullback: L^-1 is formed on a side stream while the
        # solves (which only read L) run on the caller's stream
        nbi = int(lib().lib.dla_potrf_bwd_ws_bytes_f64(batch, n))
        self.iws = torch.empty(max(nbi, 8), dtype=torch.uint8, device=self.device)
        self.iws_bytes = nbi

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def step(self, x: torch.Tensor, y: torch.Tensor, sigma2: float, ell2: float, lam: float):
        """One NLL + gradient evaluation.  x: [B, n, d], y: [B, n, 1] (device, fp64).

        Returns (nll [B], grads [B, 3] w.r.t. log(sigma2, ell2, lam), xbar, ybar);
        numerical failures are recorded in ``self.info`` (see ``check()``)."""
        B, n, d = self.batch, self.n, self.d
        for v, nm in ((sigma2, "sigma2"), (ell2, "ell2"), (lam, "lam")):
            if not (v > 0 and math.isfinite(v)):
                raise L.Error(f"make_gp: {nm} must be positive and finite")  # dl/models.hpp:33-38
        st = lib().lib.dla_gp_rbf_fwd_f64(B, n, d, C.c_void_p(x.data_ptr()), sigma2, ell2, lam,
                                          C.c_void_p(self.a.data_ptr()), C.c_void_p(self.ws.data_ptr()),
                                          self.ws_bytes, self._stream())
        if st:
            L._raise_status(st, "gp_rbf_fwd")
        # potrf (lower, in place) + the pullback's L^-1, half of it formed
        # during the factorization's chain-bound second half
        lib_ = lib().lib
        if _EARLY:
            st = lib_.dla_gp_potrf_inv_f64(B, n, C.c_void_p(self.a.data_ptr()), C.c_void_p(self.info.data_ptr()),
                                           C.c_void_p(self.iws.data_ptr()), self.iws_bytes, self._stream())
        else:
            L.potrf_inplace(self.a, True, check=False, info=self.info)
            st = lib_.dla_potrf_bwd_begin_f64(B, n, C.c_void_p(self.a.data_ptr()), 1,
                                              C.c_void_p(self.iws.data_ptr()), self.iws_bytes, self._stream())
        if st:
            L._raise_status(st, "gp_potrf_inv")
        self.z.copy_(y)
        L.trsm_inplace(self.a, self.z, False, False, True, 1.0, check=False)
        L.gemm2_into(self.quad, self.z, self.z, True, False, 0.5)
        L.sumlogdiag(self.a, out=self.logdet)
        st = lib().lib.dla_gp_nll_assemble_f64(B, n, C.c_void_p(self.quad.data_ptr()),
                                               C.c_void_p(self.logdet.data_ptr()),
                                               C.c_void_p(self.nll.data_ptr()), self._stream())
        if st:
            L._raise_status(st, "gp_nll_assemble")
        # backward (phibar = 1): zbar = z
        L.trsm_backward_into(self.ybar, self.lbar, self.z, self.a, self.z, False, False, True, 1.0)
        L.sumlogdiag_backward_into(self.lbar, self.ones, self.a, accumulate=True)
        xb = C.c_void_p(self.xbar.data_ptr()) if self.xbar is not None else None
        if _FUSED_TAIL:
            # Abar = potrf_backward(Lbar) is consumed tile pair by tile pair by the
            # RBF pullback straight from Z = L^-T P' L^-1 (never materialized)
            st = lib_.dla_gp_pullback_f64(B, n, d, C.c_void_p(x.data_ptr()), sigma2, ell2, lam,
                                          C.c_void_p(self.lbar.data_ptr()), C.c_void_p(self.a.data_ptr()), xb,
                                          C.c_void_p(self.grads.data_ptr()), C.c_void_p(self.iws.data_ptr()),
                                          self.iws_bytes, C.c_void_p(self.ws.data_ptr()), self.ws_bytes,
                                          self._stream())
            if st:
                L._raise_status(st, "gp_pullback")
            return self.nll, self.grads, self.xbar, self.ybar
        st = lib_.dla_potrf_bwd_end_f64(B, n, C.c_void_p(self.lbar.data_ptr()), C.c_void_p(self.lbar.data_ptr()),
                                        C.c_void_p(self.a.data_ptr()), 1, C.c_void_p(self.iws.data_ptr()),
                                        self.iws_bytes, self._stream())
        if st:
            L._raise_status(st, "potrf_bwd_end")
        st = lib().lib.dla_gp_rbf_bwd_f64(B, n, d, C.c_void_p(x.data_ptr()), sigma2, ell2, lam,
                                          C.c_void_p(self.lbar.data_ptr()), xb,
                                          C.c_void_p(self.grads.data_ptr()), C.c_void_p(self.ws.data_ptr()),
                                          self.ws_bytes, self._stream())
        if st:
            L._raise_status(st, "gp_rbf_bwd")
        return self.nll, self.grads, self.xbar, self.ybar

    def check(self):
        """Raise the reference exception for the first failed slice (syncs)."""
        L._check(self.info, self.batch, self.a, "gp potrf")


def gp_nll_grad(x, y, sigma2, ell2, lam, want_xbar=True):
    """Convenience one-shot: x [n, d] or [B, n, d]; y [n, 1] or [B, n, 1]."""
    squeeze = x.dim() == 2
    if squeeze:
        x, y = x.unsqueeze(0), y.reshape(1, -1, 1)
    B, n, d = x.shape
    g = GPNLL(n, d, B, x.device, want_xbar)
    nll, grads, xbar, ybar = g.step(x.contiguous(), y.contiguous(), sigma2, ell2, lam)
    g.check()
    if squeeze:
        return nll[0], grads[0], (xbar[0] if xbar is not None else None), ybar[0]
    return nll, grads, xbar, ybar
