"""Batched Kalman filter negative log likelihood + gradient on device.

Mirror of the reference's ``make_kalman`` / ``build_kalman_nll`` +
``Graph::backward`` (dl/models.hpp:272-369, Joseph-form covariance update,
first observation scored against the prior) over a batch of sequences, one
libdla_b200.so launch (``dla_kalman_nll_fwdbwd_{f32,f64}``, csrc/kalman.cu).

    m = KalmanNLL(h, d, T, batch)
    nll, grads = m.step(a, b, sh, sv, mu0, s0, obs)   # grads: dict of leaf -> gradient

Shapes: a [h,h], b [d,h], sh [h,h], sv [d,d], mu0 [h,1], s0 [h,h] — each
either without a batch dimension (one model shared by every sequence; the
returned gradients are then summed over the batch, as the reference's tape
sums contributions into a shared leaf) or with a leading [batch] dimension;
obs [batch, T, d] (or [T, d] for one sequence).  Failures follow the
reference: NotPositiveDefiniteError (innovation covariance of step t, index
t*d + pivot) and ShapeError (no observations, inconsistent shapes).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import linalg as L
from ._lib import lib

LEAVES = ("a", "b", "sh", "sv", "mu0", "s0")


class KalmanNLL:
    """Preallocated device buffers for batched Kalman NLL + gradient evaluations."""

    def __init__(self, h: int, d: int, T: int, batch: int = 1, device="cuda", dtype=torch.float64):
        if T < 1:
            raise L.ShapeError("build_kalman_nll: no observations")  # dl/models.hpp:288
        self.h, self.d, self.T, self.batch = h, d, T, batch
        self.dtype = dtype
        self.device = torch.device(device)
        self.sfx = "f64" if dtype == torch.float64 else "f32"
        f = dict(dtype=dtype, device=self.device)
        self.nll = torch.empty(batch, **f)
        self.grads = {"a": torch.empty(batch, h, h, **f), "b": torch.empty(batch, d, h, **f),
                      "sh": torch.empty(batch, h, h, **f), "sv": torch.empty(batch, d, d, **f),
                      "mu0": torch.empty(batch, h, 1, **f), "s0": torch.empty(batch, h, h, **f)}
        self.obsbar = torch.empty(batch, T, d, **f)
        self.info = torch.zeros(batch, dtype=torch.int32, device=self.device)
        nb = int(getattr(lib().lib, f"dla_kalman_ws_bytes_{self.sfx}")(batch, h, d, T))
        self.ws = torch.empty(max(nb, 8), dtype=torch.uint8, device=self.device)
        self.ws_bytes = nb

    def step(self, a, b, sh, sv, mu0, s0, obs, check: bool = True):
        """One batched NLL + gradient.  Returns (nll [batch], grads dict, obsbar [batch, T, d])."""
        h, d, T, B = self.h, self.d, self.T, self.batch
        params = [a, b, sh, sv, mu0, s0]
        want = [(h, h), (d, h), (h, h), (d, d), (h, 1), (h, h)]
        shared = all(p.dim() == 2 for p in params)
        if not shared and not all(p.dim() == 3 and p.shape[0] == B for p in params):
            raise L.ShapeError("build_kalman_nll: parameters must all be shared or all carry the batch dimension")
        for p, w in zip(params, want):
            if tuple(p.shape[-2:]) != w:
                raise L.ShapeError("build_kalman_nll: inconsistent system shapes")  # dl/models.hpp:293-298
        if obs.dim() == 2:
            obs = obs.unsqueeze(0)
        if tuple(obs.shape) != (B, T, d):
            raise L.ShapeError("build_kalman_nll: observations must be d x 1")  # dl/models.hpp:299-303
        params = [p.to(self.dtype).contiguous() for p in params]
        obs = obs.to(self.dtype).contiguous()
        s = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        g = self.grads
        st = getattr(lib().lib, f"dla_kalman_nll_fwdbwd_{self.sfx}")(
            B, h, d, T, *[P(p) for p in params], P(obs), 0 if shared else 1, P(self.nll),
            P(g["a"]), P(g["b"]), P(g["sh"]), P(g["sv"]), P(g["mu0"]), P(g["s0"]), P(self.obsbar),
            P(self.info), P(self.ws), self.ws_bytes, s)
        if st:
            L._raise_status(st, "kalman_nll")
        if check:
            L._check(self.info, B, self.nll, "kalman")
        grads = {k: (v.sum(0) if shared else v) for k, v in g.items()}
        return self.nll, grads, self.obsbar
