"""Secondary bench lines (bench.py --config c1|potrf1024|c3|c4|c5).

Same JSON contract as the headline line; each config is BASELINE.json's
configs[i] (SURVEY §8d gives the synthetic inputs and the algorithmic work
per unit).  CPU baselines run the reference (oracle/_ref) on this host.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np


def _cpu_threads():
    return os.cpu_count() or 1


def _line(args, world, metric, value, unit, ms, workload, dtype="f64", **extra):
    d = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
         "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
         "vs_baseline": None, "dtype": dtype, "data": "synthetic (Philox N(0,1) based)",
         "config": {"workload": workload}}
    d.update(extra)
    return d


def run(torch, args, rank, world, lib, fp64_peak, hbm):
    import bench
    from oracle import oracle as O
    from paper_1710_08717_b200 import linalg as L
    from paper_1710_08717_b200.shard import shard_range

    cfg = args.config
    ref = O.ref() if O.ref_available() else None
    if cfg == "c1":
        B, n = 64, 32
        # (1) the fused chain (dla_chol_chain_fwdbwd: ONE launch) -- the value
        r = O.rng(7)
        a0 = torch.from_numpy(O.random_spd(n, r, batch=B)).cuda()
        y0 = torch.from_numpy(r.standard_normal((B, n, 1))).cuda()
        phi = torch.empty(B, dtype=torch.float64, device="cuda")
        abar, ybar = torch.empty_like(a0), torch.empty_like(y0)
        info = torch.zeros(B, dtype=torch.int32, device="cuda")

        def fused():
            L.chol_chain_fwdbwd(a0, y0, phi, abar, ybar, check=False, info=info)

        c0 = lib.dla_launch_count()
        fused()
        torch.cuda.synchronize()
        launches = lib.dla_launch_count() - c0
        ms = bench.timed(torch, bench.graphed(torch, fused), args.steps, args.warmup, world)
        # (2) the same chain through the per-operator C-ABI (potrf, trsm, gemm2,
        #     sumlogdiag, trsm_bwd, sumlogdiag_bwd, potrf_bwd)
        step, _ = bench.c1_chain_fns(torch, B, n)
        ms_ops = bench.timed(torch, bench.graphed(torch, step), args.steps, args.warmup, world)
        flops = n ** 3 / 3 + 4 * n ** 3 / 3 + 4 * n * n
        bytes_per = (2 * n * n + 2 * n + 1) * 8  # read A, y; write Abar, ybar, phi
        # batch sweep of the fused chain (HBM regime), L2 flushed by size
        sweep = []
        for Bs in (1024, 65536, 1 << 20):
            if Bs * n * n * 8 * 2 > 0.5 * torch.cuda.get_device_properties(0).total_memory:
                continue
            a1 = torch.from_numpy(O.random_spd(n, O.rng(3), batch=1)).cuda().expand(Bs, n, n).contiguous()
            y1 = torch.randn(Bs, n, 1, dtype=torch.float64, device="cuda")
            p1, ab1, yb1 = torch.empty(Bs, dtype=torch.float64, device="cuda"), torch.empty_like(a1), torch.empty_like(y1)
            i1 = torch.zeros(Bs, dtype=torch.int32, device="cuda")
            f1 = lambda: L.chol_chain_fwdbwd(a1, y1, p1, ab1, yb1, check=False, info=i1)  # noqa: E731
            ms1 = bench.timed(torch, bench.graphed(torch, f1), 5, 3, world)
            sweep.append({"batch": Bs, "ms": ms1, "matrices_per_s": world * Bs / (ms1 / 1e3),
                          "gb_per_s": Bs * bytes_per / (ms1 / 1e3) / 1e9,
                          "frac_of_hbm": Bs * bytes_per / (ms1 / 1e3) / 1e9 / hbm})
            del a1, y1, p1, ab1, yb1, i1
        cpu = None
        if ref is not None and rank == 0:
            a = a0.cpu().numpy()
            y = y0.cpu().numpy()
            reps, secs = 0, 0.0
            while secs < 2.0:
                secs += ref.c1_chain(a, y, 1)[0]
                reps += 1
            cpu = {"value": reps * B / secs, "unit": "matrices/s", "cores": 1, "kind": "reference",
                   "sample": f"{reps} x reference C1 chain over batch {B} (for_each_slice, 1 thread)"}
        v = world * B / (ms / 1e3)
        big = sweep[-1] if sweep else None
        return _line(args, world, "C1 chain matrices/s", v, "matrices/s", ms,
                     "C1: batch 64 x 32^2 fp64 potrf fwd+bwd + trsm + sumlogdiag (fused one-launch chain, "
                     "dla_chol_chain_fwdbwd_f64)",
                     gflops=v * flops / 1e9, gpu_launches=launches * args.steps, cpu_baseline=cpu,
                     operator_chain={"ms_per_step": ms_ops, "matrices_per_s": world * B / (ms_ops / 1e3),
                                     "note": "same chain via 7 per-operator C-ABI calls (graph-replayed)"},
                     batch_sweep=sweep,
                     roofline={"bound": "hbm", "kernel": "k_chol_chain_dmma (fp64)",
                               "achieved": big["gb_per_s"] if big else None, "peak": hbm, "unit": "GB/s",
                               "frac": big["frac_of_hbm"] if big else None, "traffic": None,
                               "note": f"at batch {big['batch'] if big else '-'} (batch 64 = 1 MiB per step is "
                                       f"launch/latency bound); algorithmic bytes (2n^2+2n+1)*8 per matrix"})
    if cfg == "potrf1024":
        B, n = 8, 1024
        ms = bench.run_potrf_batch(torch, n, B, args.steps, args.warmup, world)
        flops = B * 5 * n ** 3 / 3
        tf = world * flops / (ms / 1e3) / 1e12
        cpu = None
        if ref is not None and rank == 0:
            r = O.rng(11)
            a = O.random_spd(n, r, batch=B)
            lb = np.tril(r.standard_normal((B, n, n)))
            secs, _ = ref.potrf_fwdbwd_batch(a, lb, min(B, _cpu_threads()))
            cpu = {"value": B / secs, "unit": "matrices/s", "cores": min(B, _cpu_threads()), "kind": "reference",
                   "sample": f"reference potrf+potrf_backward over batch {B} x {n}^2, for_each_slice"}
        ms_split = bench.run_potrf_batch_split(torch, n, B, args.steps, args.warmup, world)
        sweep = []
        for Bs in (32, 128):  # the per-panel chain is batch-independent: larger batches amortise it
            mss = bench.run_potrf_batch(torch, n, Bs, 5, 2, world)
            tfs = world * Bs * 5 * n ** 3 / 3 / (mss / 1e3) / 1e12
            sweep.append({"batch": Bs, "ms": mss, "matrices_per_s": world * Bs / (mss / 1e3), "tflops": tfs,
                          "frac_of_fp64_peak": tfs / fp64_peak / world})
        tf_split = world * flops / (ms_split / 1e3) / 1e12
        # value: the fused split entry points (same outputs, bitwise); the two
        # plain operator calls are reported beside it
        return _line(args, world, "potrf fwd+bwd matrices/s (n=1024)", world * B / (ms_split / 1e3), "matrices/s",
                     ms_split, "north star: potrf fwd+bwd, batch 8 x 1024^2 fp64, through the C-ABI's fused split "
                     "entry points dla_gp_potrf_inv_f64 + dla_potrf_bwd_end_f64 (half of L^-1 overlaps the "
                     "factorization's chain-bound second half; outputs bitwise those of potrf + potrf_backward)",
                     step_tflops=tf_split, batch_sweep=sweep,
                     operator_calls={"ms_per_step": ms, "matrices_per_s": world * B / (ms / 1e3), "tflops": tf,
                                     "frac_of_fp64_peak": tf / fp64_peak / world,
                                     "note": "dla_potrf_fwd_f64 + dla_potrf_bwd_f64 (graph-replayed)"},
                     roofline={"bound": "tensor", "achieved": tf_split, "peak": fp64_peak, "unit": "TFLOP/s",
                               "frac": tf_split / fp64_peak, "traffic": None}, cpu_baseline=cpu)
    if cfg == "c3":
        res = []
        for dt in (torch.float64, torch.float32):
            B, m, n = 256, 128, 512
            r = O.rng(5)
            x = r.standard_normal((B, m, n - m))
            a0 = torch.from_numpy(np.concatenate([np.broadcast_to(np.eye(m), (B, m, m)), x], axis=2)).to(dt).cuda()
            qb = torch.from_numpy(r.standard_normal((B, m, n))).to(dt).cuda()
            lb = torch.from_numpy(np.tril(r.standard_normal((B, m, m)))).to(dt).cuda()
            q = torch.empty_like(a0)
            l = torch.empty(B, m, m, dtype=dt, device="cuda")
            ab = torch.empty_like(a0)

            def step():
                q.copy_(a0)
                L.gelqf_inplace(q, l, check=False)
                L.gelqf_backward_into(ab, qb, lb, q, l)

            ms = bench.timed(torch, step, args.steps, args.warmup, world)
            flops = B * (4 * m * m * n - 4 * m ** 3 / 3 + m ** 3 / 3 + 5 * m * m * n)
            res.append({"dtype": str(dt).split(".")[-1], "matrices_per_s": world * B / (ms / 1e3), "ms": ms,
                        "tflops": flops / (ms / 1e3) / 1e12})
        cpu = None
        if ref is not None and rank == 0:
            r = O.rng(5)
            Bc = 32
            x = r.standard_normal((Bc, m, n - m))
            a = np.concatenate([np.broadcast_to(np.eye(m), (Bc, m, m)), x], axis=2)
            secs, _ = ref.gelqf_fwdbwd_batch(a, r.standard_normal((Bc, m, n)),
                                             np.tril(r.standard_normal((Bc, m, m))), _cpu_threads())
            cpu = {"value": Bc / secs, "unit": "matrices/s", "cores": _cpu_threads(), "kind": "reference",
                   "sample": f"reference gelqf+backward over {Bc} of the 256 matrices (fp64, for_each_slice)"}
        return _line(args, world, "gelqf fwd+bwd matrices/s (128x512)", res[0]["matrices_per_s"], "matrices/s",
                     res[0]["ms"], "C3: BLR gelqf fwd+bwd, batch 256 of B=[I_128, X] in R^{128x512} (the reference "
                     "rejects 512x128, dl/lq.hpp:26-29)", per_dtype=res, cpu_baseline=cpu,
                     roofline={"bound": "tensor", "achieved": res[0]["tflops"], "peak": fp64_peak, "unit": "TFLOP/s",
                               "frac": res[0]["tflops"] / fp64_peak, "traffic": None,
                               "note": "fp64 step: CholeskyQR2 LQ on FP64 DMMA (G = A A^T, chol, inverse-GEMM "
                                       "solve, twice; per-slice Householder fallback) + backward GEMMs; "
                                       "algorithmic flops (Householder count, not the CholeskyQR2 work) "
                                       "4m^2n - 4m^3/3 + m^3/3 + 5m^2n per matrix (SURVEY 8d)"})
    if cfg == "c4":
        B, n = 1024, 64
        r = O.rng(4)
        a0 = torch.from_numpy(O.random_sym(n, r, batch=B)).cuda()
        ub = torch.from_numpy(r.standard_normal((B, n, n))).cuda()
        lb = torch.from_numpy(r.standard_normal((B, n))).cuda()
        u = torch.empty_like(a0)
        lam = torch.empty(B, n, dtype=torch.float64, device="cuda")
        ab = torch.empty_like(a0)

        def step():
            u.copy_(a0)
            L.syevd_inplace(u, lam, check=False)
            L.syevd_backward_into(ab, ub, lb, u, lam)

        ms = bench.timed(torch, step, args.steps, args.warmup, world)
        flops = B * (10 * n ** 3 / 3 + 6 * n ** 3)
        cpu = None
        if ref is not None and rank == 0:
            Bc = 256
            secs, _ = ref.syevd_fwdbwd_batch(a0[:Bc].cpu().numpy(), ub[:Bc].cpu().numpy(), lb[:Bc].cpu().numpy(),
                                             _cpu_threads())
            cpu = {"value": Bc / secs, "unit": "matrices/s", "cores": _cpu_threads(), "kind": "reference",
                   "sample": f"reference syevd+backward over {Bc} of the 1024 matrices, for_each_slice"}
        v = world * B / (ms / 1e3)
        return _line(args, world, "syevd fwd+bwd matrices/s (64x64)", v, "matrices/s", ms,
                     "C4: batched syevd fwd+bwd, batch 1024 x 64^2 fp64 (Jacobi, smem-resident)",
                     gflops=v * flops / B / 1e9, cpu_baseline=cpu,
                     roofline={"bound": "latency", "achieved": v * flops / B / 1e12, "peak": fp64_peak,
                               "unit": "TFLOP/s", "frac": v * flops / B / 1e12 / fp64_peak, "traffic": None,
                               "note": "count-convention flops 10n^3/3 + 6n^3 per matrix; the smem Jacobi does "
                                       "~20x that in FP64 FMA and is bound by its per-round barrier chain"})
    if cfg == "kalman":
        r = kalman_measure(torch, world, args.steps, args.warmup)
        cpu = None
        if ref is not None and rank == 0 and not getattr(args, "no_cpu_baseline", False):
            cpu = kalman_cpu_baseline(r.pop("sample_inputs"))
        r.pop("sample_inputs", None)
        return _line(args, world, "Kalman NLL+grad sequences/s", r["sequences_per_s"], "sequences/s",
                     r["ms_per_step"], r["workload"], cpu_baseline=cpu,
                     **{k: v for k, v in r.items() if k not in ("sequences_per_s", "ms_per_step", "workload")})
    if cfg == "c5":
        r = c5_measure(torch, rank, world, args.steps, args.warmup, fp64_peak)
        cpu = None
        if rank == 0 and world == 1 and not getattr(args, "no_cpu_baseline", False):
            cpu = c5_cpu_baseline(r.pop("sample_inputs"), r["theta"])
        r.pop("sample_inputs", None)
        return _line(args, world, "C5 GP marginal likelihoods items/s", r["items_per_s"], "items/s", r["ms_per_step"],
                     r["workload"], cpu_baseline=cpu, **{k: v for k, v in r.items()
                                                         if k not in ("items_per_s", "ms_per_step", "workload")})
    raise ValueError(cfg)


def c5_inputs(torch, lo, hi, n=128):
    """Per-rank slice [lo, hi) of the GLOBAL synthetic C5 batch: item chunks of
    4096 are generated on device from a generator seeded by the chunk's global
    start, so every world size sees the same items (shard bounds are multiples
    of 4096 for N | 16)."""
    chunk = 4096
    B = hi - lo
    s = torch.empty(B, n, n, dtype=torch.float64, device="cuda")
    y = torch.empty(B, n, 1, dtype=torch.float64, device="cuda")
    from paper_1710_08717_b200 import linalg as L
    from paper_1710_08717_b200._lib import lib
    import ctypes as C
    g0 = (lo // chunk) * chunk
    for c0 in range(g0, hi, chunk):
        gen = torch.Generator("cuda").manual_seed(c0)
        x = torch.randn(chunk, n, n, dtype=torch.float64, device="cuda", generator=gen)
        yy = torch.randn(chunk, n, 1, dtype=torch.float64, device="cuda", generator=gen)
        a, b = max(c0, lo), min(c0 + chunk, hi)
        xs = x[a - c0:b - c0].contiguous()
        # S = X X^T + n I per item through libdla's syrk (batch = grid: the
        # same bits for an item whatever the shard), then the diagonal shift
        L.syrk_into(xs, xs.clone(), False, 1.0)
        st = lib().lib.dla_ml_shift_copy_f64(b - a, n, C.c_void_p(xs.data_ptr()),
                                            C.c_void_p(s[a - lo:b - lo].data_ptr()), float(n),
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert st == 0
        y[a - lo:b - lo] = yy[a - c0:b - c0]
        del x, yy
    return s, y


def c5_measure(torch, rank, world, steps, warmup, fp64_peak, total=65536, n=128):
    """C5: `total` independent 128^2 GP marginal likelihoods, contiguous batch
    shards per rank, one NCCL all-reduce of [loss, dloss/dtheta] per step."""
    import bench
    from paper_1710_08717_b200.c5 import MarginalLikelihoods
    from paper_1710_08717_b200.shard import shard_range
    lo, hi = shard_range(total, rank, world)
    s, y = c5_inputs(torch, lo, hi, n)
    m = MarginalLikelihoods(hi - lo, n)
    theta = math.log(0.3)
    ms = bench.timed(torch, lambda: m.step_allreduce(s, y, theta), steps, warmup, world)
    m.check()
    flops = total * 8.33 * n ** 3
    tf = flops / (ms / 1e3) / 1e12
    out = dict(items_per_s=total / (ms / 1e3), ms_per_step=ms,
               workload=f"C5: {total} x {n}^2 GP marginal likelihoods (potrf+potri+trmm fwd+bwd), batch sharded "
                        f"over {world} GPU(s), NCCL all-reduce of (loss, dloss/dtheta)",
               step_tflops=tf, loss_grad=m.out.cpu().tolist(), theta=theta,
               config_parallelism=f"dp{world} (contiguous batch shards, one all_reduce of 2 fp64 per step)",
               roofline={"bound": "tensor", "achieved": tf / world, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": tf / world / fp64_peak, "traffic": None,
                         "note": "per GPU, minimal flops 8.33 n^3 per item (SURVEY 8d)"},
               sample_inputs=(s[:1].cpu().numpy()[0], y[:1].cpu().numpy()[0]) if rank == 0 else None)
    del m, s, y
    torch.cuda.empty_cache()
    return out


def c5_cpu_baseline(sample, theta):
    import time as _t
    from oracle import oracle as O
    port = O.port()
    sc, yc = sample
    reps, t0 = 0, _t.perf_counter()
    while _t.perf_counter() - t0 < 3.0:
        O.c5_item(port, sc, yc, theta)
        reps += 1
    secs = (_t.perf_counter() - t0) / reps
    return {"value": 1.0 / secs, "unit": "items/s", "cores": 1, "kind": "port",
            "sample": f"{reps} C5 items through the oracle port's per-op chain (C restatement of the "
                      f"reference ops, 1 thread); the reference has no C5 driver"}


# Batched Kalman filter NLL + gradient: one CTA per
# sequence, per-sequence models, the reference's build_kalman_nll graph.
KALMAN_B, KALMAN_H, KALMAN_D, KALMAN_T = 4096, 8, 8, 128


def kalman_measure(torch, world, steps, warmup, B=KALMAN_B, h=KALMAN_H, d=KALMAN_D, T=KALMAN_T):
    import bench
    from oracle import oracle as O
    from paper_1710_08717_b200 import kalman as K

    r = O.rng(21)
    m = O.random_kalman(r, h, d, T, batch=B)
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in m]
    km = K.KalmanNLL(h, d, T, B)
    km.step(*dev, check=True)  # validates the inputs once (no failing sequence)
    ms = bench.timed(torch, bench.graphed(torch, lambda: km.step(*dev, check=False)), steps, warmup, world)
    # algorithmic flops per time step (forward products + solves, and the
    # backward's ~2.5x), counted from the graph at h = d
    fl_step = 2 * (d * h * h + d * d * h + h * h * d + 2 * h * d * d + h * h * d + 2 * h ** 3 + h * d * d
                   + h * h * d + 2 * h ** 3) + d ** 3 / 3
    fl = 3.5 * fl_step * T
    return {"sequences_per_s": world * B / (ms / 1e3), "ms_per_step": ms,
            "gflops": world * B * fl / (ms / 1e3) / 1e9, "launches_per_step": 1,
            "workload": f"Kalman filter NLL + gradient of every leaf (dl/models.hpp:285-337), batch {B} sequences, "
                        f"h = d = {h}, T = {T}, per-sequence models, fp64 (one launch: csrc/kalman.cu)",
            "sample_inputs": [x[:16] for x in m]}


def kalman_cpu_baseline(sample):
    from oracle import oracle as O

    th = min(16, _cpu_threads())
    _, secs = O.kalman_ref_batch(*sample, threads=th)
    n = sample[0].shape[0]
    return {"value": n / secs, "unit": "sequences/s", "cores": th, "kind": "reference",
            "sample": f"reference make_kalman + Graph::backward over {n} of the sequences (for_each_slice, "
                      f"{th} threads)"}
