"""Per-operator device timings (CUDA events, warm, median of reps) for
optimisation work; not the headline benchmark (bench.py is).

    python tools/microbench.py [--quick]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_08717_b200 import linalg as L  # noqa: E402


def tm(fn, reps=10, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def tm_graph(fn, reps=50):
    """Per-call device time of fn from a CUDA graph holding `reps` calls
    (removes the Python/launch overhead that dominates tiny kernels)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def spd(n, batch=1):
    x = torch.randn(batch, n, n, dtype=torch.float64, device="cuda")
    return x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    torch.manual_seed(0)
    out = []

    def rec(name, ms, flops):
        out.append({"op": name, "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 3) if flops else None})
        print(json.dumps(out[-1]), flush=True)

    for n in ([1024, 4096] if not args.quick else [4096]):
        a0 = spd(n)
        a = a0.clone()
        rec(f"potrf n={n}", tm(lambda: (a.copy_(a0), L.potrf_inplace(a, check=False))), n ** 3 / 3)
        l = L.potrf(a0)
        lb = torch.tril(torch.randn_like(l))
        ab = torch.empty_like(l)
        rec(f"potrf_bwd n={n}", tm(lambda: L.potrf_backward_into(ab, lb, l)), 4 * n ** 3 / 3)
        x = torch.randn(1, n, n, dtype=torch.float64, device="cuda")
        for right in (False, True):
            for trans in (False, True):
                y = x.clone()
                rec(f"trsm n={n} nrhs={n} right={int(right)} trans={int(trans)}",
                    tm(lambda: L.trsm_inplace(l, y, right, trans, True, 1.0, check=False)), n ** 3)
        y = x.clone()
        rec(f"trmm n={n} left trans", tm(lambda: L.trmm_inplace(l, y, False, True, True)), n ** 3)
        v = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
        rec(f"trsm n={n} nrhs=1", tm(lambda: L.trsm_inplace(l, v, check=False)), n ** 2)
        c = torch.empty_like(x)
        rec(f"gemm {n}^3", tm(lambda: L.gemm2_into(c, x, x)), 2 * n ** 3)
        rec(f"gemm {n}^3 tb", tm(lambda: L.gemm2_into(c, x, x, False, True)), 2 * n ** 3)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    for n in (64, 32, 128, 256):
        a0 = spd(n)
        a = a0.clone()
        rec(f"potrf n={n} batch=1 (graph, per call)",
            tm_graph(lambda: (a.copy_(a0), L.potrf_inplace(a, check=False, info=info))), None)
        l = L.potrf(a0)
        v = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
        rec(f"trsm n={n} nrhs=1 (graph, per call)", tm_graph(lambda: L.trsm_inplace(l, v, check=False)), None)
        xx = torch.randn(1, 4096, n, dtype=torch.float64, device="cuda")
        rec(f"trsm right n={n} nrows=4096 (graph, per call)",
            tm_graph(lambda: L.trsm_inplace(l, xx, True, True, True, 1.0, check=False)), 4096 * n * n)
    c64 = torch.empty(1, 64, 64, dtype=torch.float64, device="cuda")
    x64 = torch.randn(1, 64, 64, dtype=torch.float64, device="cuda")
    rec("gemm 64^3 (graph, per call)", tm_graph(lambda: L.gemm2_into(c64, x64, x64)), 2 * 64 ** 3)
    rec("empty copy_ 64^2 (graph, per call)", tm_graph(lambda: c64.copy_(x64)), None)
    for n, b in ((32, 65536), (128, 8192)):
        a0 = spd(n, b)
        a = a0.clone()
        rec(f"potrf n={n} batch={b}", tm(lambda: (a.copy_(a0), L.potrf_inplace(a, check=False))), b * n ** 3 / 3)
        l = L.potrf(a0)
        lb = torch.tril(torch.randn_like(l))
        ab = torch.empty_like(l)
        rec(f"potrf_bwd n={n} batch={b}", tm(lambda: L.potrf_backward_into(ab, lb, l)), b * 4 * n ** 3 / 3)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "microbench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
