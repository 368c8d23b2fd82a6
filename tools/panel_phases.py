"""Per-phase time of the blocked-potrf panel kernel (CTA 0, %globaltimer),
from a library built with -DDLAB_PANEL_PROF (tuning build):

    DLA_LIB_PATH=paper_1710_08717_b200/libdla_prof.so python tools/panel_phases.py [n]

Phases: 0 start | 1 A11/panel rows loaded | 2 fused A11 update | 3 factor
(+ side A21 update) | 4 L11 stored | 5 panel solve | 6 panel stored;
also the gap between consecutive panel launches (CTA 0 end -> next start)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import gp  # noqa: E402
from paper_1710_08717_b200._lib import lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
torch.manual_seed(0)
x = torch.randn(1, n, 8, dtype=torch.float64, device="cuda")
y = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
g = gp.GPNLL(n, 8, 1, "cuda")
for _ in range(3):
    g.step(x, y, 1.0, 1.0, 0.1)
torch.cuda.synchronize()
L = lib().lib
buf = (C.c_ulonglong * (128 * 8))()
acc = []
for _ in range(5):
    g.step(x, y, 1.0, 1.0, 0.1)
    torch.cuda.synchronize()
    assert L.dla_panel_prof_read(buf) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(128, 8)[: n // 64].astype(np.int64)
    acc.append(a)
names = ["load", "A11upd", "factor", "L11st", "solve", "store"]
for rep in acc[-1:]:
    d = np.diff(rep[:, :7], axis=1) / 1000.0
    gaps = (rep[1:, 0] - rep[:-1, 6]) / 1000.0
    span = (rep[-1, 6] - rep[0, 0]) / 1000.0
    print(f"n={n}: span {span:.1f} us over {len(rep)} panels ({span / len(rep):.1f} us/step)")
    print("mean us:", "  ".join(f"{nm} {v:.2f}" for nm, v in zip(names, d[1:].mean(0))),
          f" gap {gaps.mean():.2f}")
    for p in (1, 2, 8, 16, 32, 48, 60, 62):
        if p < len(rep):
            print(f"  p={p:2d}", "  ".join(f"{v:6.2f}" for v in d[p]), f"  gap-before {gaps[p - 1]:6.2f}")
cb = (C.c_ulonglong * (128 * 16))()
if hasattr(L, "dla_chol_prof_read") and L.dla_chol_prof_read(cb) == 0:
    c = np.frombuffer(cb, dtype=np.uint64).reshape(128, 16).astype(np.int64)
    rows = [r for r in range(1, 48) if c[r, 0] > 0 and c[r, 7] > c[r, 0]]
    d = np.array([[(c[r, i] - c[r, i - 1]) / 1e3 for i in range(1, 8)] + [(c[r, 9] - c[r, 7]) / 1e3] for r in rows])
    print("chol phases, mean over panels", rows[0], "..", rows[-1], "(A_j = warp-0 panel j || off-chain work; T_j = trail):")
    print("  ", "  ".join(f"{nm} {v:.2f}" for nm, v in zip(["A0", "T0", "A1", "T1", "A2", "T2", "A3", "tail"], d.mean(0))))
    print("   min", "  ".join(f"{v:.2f}" for v in d.min(0)))
