"""potrf n=4096 timing vs matrix content (random SPD vs GP RBF kernel matrix)."""
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
g = gp.GPNLL(n, d, 1, "cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
lib().lib.dla_gp_rbf_fwd_f64(1, n, d, C.c_void_p(x.data_ptr()), 1.0, 1.0, 0.1, C.c_void_p(g.a.data_ptr()),
                             C.c_void_p(g.ws.data_ptr()), g.ws_bytes, st)
torch.cuda.synchronize()
rbf = g.a.clone()
xx = torch.randn(1, n, n, dtype=torch.float64, device="cuda")
spd = xx @ xx.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
eye = torch.eye(n, dtype=torch.float64, device="cuda").unsqueeze(0).contiguous()
a = torch.empty_like(spd)
info = torch.zeros(1, dtype=torch.int32, device="cuda")
for name, src in (("spd", spd), ("rbf", rbf), ("identity", eye), ("rbf+10I", rbf + 10 * eye)):
    def step():
        a.copy_(src)
        L.potrf_inplace(a, check=False, info=info)
    ms = bench.timed(torch, bench.graphed(torch, step), 10, 3, 1)
    print(f"{name:10s} graph {ms:.3f} ms  info={info.item()}")
