"""Batched GP marginal likelihoods (BASELINE config C5) on device.

The reference has no driver for this config; the graph is the one SURVEY §8d
defines from reference ops (potrf + potri + trmm fwd+bwd), with a shared
log-parameterised noise hyperparameter so the batch has a gradient to
all-reduce (dl/models.hpp:126-131 convention):

    A_b   = S_b + lam I,  lam = exp(theta)
    L_b   = potrf(A_b)                      (dl/cholesky.hpp:79)
    B_b   = potri(L_b)        = A_b^{-1}    (dl/cholesky.hpp:141)
    G_b   = trmm(L_b, B_b, left, trans)     = L_b^T A_b^{-1} = L_b^{-1}
    v_b   = gemm2(G_b, y_b)                 = L_b^{-1} y_b
    phi_b = 1/2 v_b^T v_b + sumlogdiag(L_b) + n/2 log 2 pi
    loss  = sum_b phi_b,   dloss/dtheta = lam * sum_b tr(Abar_b)

Backward runs the closed-form pullbacks in reverse (gemm2, trmm, potri,
sumlogdiag, potrf backward).  Every step is a libdla_b200.so call; the
per-slice results for a shard are reduced on device and all-reduced across
ranks by ``shard.allreduce_loss_grad``.
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import linalg as L
from ._lib import lib
from .shard import allreduce_loss_grad

LOG_2PI = 1.8378770664093454835606594728112353


class MarginalLikelihoods:
    """Preallocated buffers for a shard of `batch` items of size n (fp64)."""

    def __init__(self, batch: int, n: int, device="cuda"):
        f = dict(dtype=torch.float64, device=device)
        self.batch, self.n = batch, n
        self.l = torch.empty(batch, n, n, **f)
        self.b = torch.empty(batch, n, n, **f)
        self.g = torch.empty(batch, n, n, **f)
        self.v = torch.empty(batch, n, 1, **f)
        self.quad = torch.empty(batch, 1, 1, **f)
        self.logdet = torch.empty(batch, **f)
        self.gbar = torch.empty(batch, n, n, **f)
        self.ybar = torch.empty(batch, n, 1, **f)
        self.lbar = torch.empty(batch, n, n, **f)
        self.bbar = torch.empty(batch, n, n, **f)
        self.tbar = torch.empty(batch, n, n, **f)
        self.ones = torch.ones(batch, **f)
        self.info = torch.zeros(batch, dtype=torch.int32, device=device)
        self.out = torch.empty(2, **f)  # [loss, dloss/dtheta] of this shard
        nb = int(lib().lib.dla_ml_reduce_ws_bytes(batch))
        self.rws = torch.empty(max(nb, 8), dtype=torch.uint8, device=device)  # reduction partials
        self.rws_bytes = nb

    def _st(self):
        return C.c_void_p(torch.cuda.current_stream(self.l.device).cuda_stream)

    def step(self, s: torch.Tensor, y: torch.Tensor, theta: float):
        lam = math.exp(theta)
        B, n = self.batch, self.n
        lib_ = lib().lib
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        # forward: every kernel below is libdla_b200's (copies included)
        self._ok(lib_.dla_ml_shift_copy_f64(B, n, P(s), P(self.l), lam, self._st()))  # A = S + lam I
        L.potrf_inplace(self.l, True, check=False, info=self.info)
        L.potri_into(self.b, self.l, True, check=False)   # out of place: no copy of L
        L.trmm_into(self.g, self.l, self.b, False, True, True)  # G = L^T B, out of place
        L.gemm2_into(self.v, self.g, y)
        L.gemm2_into(self.quad, self.v, self.v, True, False, 0.5)
        L.sumlogdiag(self.l, out=self.logdet)
        # backward (phibar_b = 1): vbar = v
        L.gemm2_backward_into(self.gbar, self.ybar, self.v, self.g, y, False, False)
        L.trmm_backward_into(self.bbar, self.tbar, self.gbar, self.l, self.b, False, True, True)
        L.potri_backward_into(self.lbar, self.bbar, self.l, self.b, True)
        self._ok(lib_.dla_axpy_f64(B * n * n, 1.0, P(self.tbar), P(self.lbar), self._st()))
        L.sumlogdiag_backward_into(self.lbar, self.ones, self.l, accumulate=True)
        L.potrf_backward_into(self.lbar, self.lbar, self.l, True)  # lbar now holds Abar
        # shard reduction: [loss, dloss/dtheta] (fixed order, on device)
        self._ok(lib_.dla_ml_reduce_f64(B, n, P(self.quad), P(self.logdet), P(self.lbar), lam, P(self.out),
                                        P(self.rws), self.rws_bytes, self._st()))
        return self.out

    @staticmethod
    def _ok(st):
        if st:
            L._raise_status(st, "c5 driver")

    def step_allreduce(self, s, y, theta):
        return allreduce_loss_grad(self.step(s, y, theta))

    def check(self):
        L._check(self.info, self.batch, self.l, "c5 potrf")
