"""Per-phase device time of one GP NLL+grad step (n=4096, d=8): each phase
captured in its own CUDA graph and replayed alone (no cross-phase overlap)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1710_08717_b200 import gp  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402
from paper_1710_08717_b200._lib import lib  # noqa: E402

n, d = 4096, 8
torch.manual_seed(0)
x = torch.randn(1, n, d, dtype=torch.float64, device="cuda")
y = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
g = gp.GPNLL(n, d, 1, "cuda")
g.step(x, y, 1.0, 1.0, 0.1)
torch.cuda.synchronize()
a_saved = g.a.clone()
lib_ = lib().lib
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731


def rbf_fwd():
    lib_.dla_gp_rbf_fwd_f64(1, n, d, C.c_void_p(x.data_ptr()), 1.0, 1.0, 0.1, C.c_void_p(g.a.data_ptr()),
                            C.c_void_p(g.ws.data_ptr()), g.ws_bytes, st())


def potrf():
    g.a.copy_(a_saved)  # (a_saved holds L; the copy is part of the timing)
    L.potrf_inplace(g.a, True, check=False, info=g.info)


phases = {
    "rbf_fwd": rbf_fwd,
    "copy 128MiB": lambda: g.lbar.copy_(a_saved),
    "trsm fwd (trsv)": lambda: (g.z.copy_(y), L.trsm_inplace(a_saved, g.z, False, False, True, 1.0, check=False)),
    "trsm_bwd": lambda: L.trsm_backward_into(g.ybar, g.lbar, g.z, a_saved, g.z, False, False, True, 1.0),
    "potrf_bwd": lambda: L.potrf_backward_into(g.lbar, g.lbar, a_saved, True),
    "rbf_bwd": lambda: lib_.dla_gp_rbf_bwd_f64(1, n, d, C.c_void_p(x.data_ptr()), 1.0, 1.0, 0.1,
                                                C.c_void_p(g.lbar.data_ptr()), C.c_void_p(g.xbar.data_ptr()),
                                                C.c_void_p(g.grads.data_ptr()), C.c_void_p(g.ws.data_ptr()),
                                                g.ws_bytes, st()),
    "full step": lambda: g.step(x, y, 1.0, 1.0, 0.1),
}
a_spd = None
for name, fn in phases.items():
    ms = bench.timed(torch, bench.graphed(torch, fn), 10, 3, 1)
    print(f"{name:20s} {ms:8.3f} ms")
# potrf on the SPD matrix: rebuild A with rbf each time
def potrf_phase():
    rbf_fwd()
    L.potrf_inplace(g.a, True, check=False, info=g.info)
ms = bench.timed(torch, bench.graphed(torch, potrf_phase), 10, 3, 1)
print(f"{'rbf_fwd+potrf':20s} {ms:8.3f} ms")
