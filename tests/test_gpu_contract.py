"""The C-ABI boundary contract on the device (SURVEY §8b Ownership and
Threading rows; include/dla.h):

  * every op runs with exactly dla_workspace_bytes() of caller workspace and
    returns DLA_ERR_WORKSPACE -- before touching its outputs -- when given
    less (no hidden allocation behind a short workspace);
  * calls from two host threads on two streams at once (each forking its
    own side streams) give bitwise the results of the same calls run alone;
  * batched potrf equals per-slice potrf to rounding on both schedules (the
    fused-panel and the large-batch throughput schedule round differently,
    so batch invariance is a tolerance, not a bitwise, property).
"""
import ctypes as C
import threading

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import linalg as L  # noqa: E402
from paper_1710_08717_b200._lib import OPS, WS_BACKWARD, lib  # noqa: E402


def spd(n, batch, seed):
    return torch.from_numpy(O.random_spd(n, O.rng(seed), batch=batch)).cuda()


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("n,batch", [(1024, 2), (320, 3)])
def test_potrf_fwd_bwd_short_workspace_is_refused(n, batch):
    lb = lib().lib
    a = spd(n, batch, n)
    need = int(lb.dla_workspace_bytes(OPS["potrf"], 1, batch, n, n, 0, 0))
    assert need > 0
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    f = lib().fn("potrf_fwd", "f64")
    l = a.clone()
    assert f(batch, n, _p(l), 1, _p(info), _p(ws), need - 1, _st()) == 8  # DLA_ERR_WORKSPACE
    torch.cuda.synchronize()
    assert f(batch, n, _p(l), 1, _p(info), _p(ws), need, _st()) == 0
    torch.cuda.synchronize()
    assert torch.equal(l, L.potrf(a))
    need_b = int(lb.dla_workspace_bytes(OPS["potrf"], 1, batch, n, n, 0, WS_BACKWARD))
    fb = lib().fn("potrf_bwd", "f64")
    lbar = torch.tril(torch.randn_like(a))
    out = torch.zeros_like(a)
    if need_b > 0:
        wsb = torch.empty(need_b, dtype=torch.uint8, device="cuda")
        assert fb(batch, n, _p(out), _p(lbar), _p(l), 1, None, 0, _st()) == 8
        assert fb(batch, n, _p(out), _p(lbar), _p(l), 1, _p(wsb), need_b, _st()) == 0
    else:
        assert fb(batch, n, _p(out), _p(lbar), _p(l), 1, None, 0, _st()) == 0
    torch.cuda.synchronize()
    assert torch.equal(out, L.potrf_backward(lbar, l))


def test_narrow_trsm_workspace():
    lb = lib().lib
    n = 2048
    l = L.potrf(spd(n, 1, 5))
    y = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
    need = int(lb.dla_workspace_bytes(OPS["trsm"], 1, 1, n, 1, 0, 0))
    assert need >= n * 8
    f = lib().fn("trsm_fwd", "f64")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    x = y.clone()
    assert f(1, n, 1, _p(l), _p(x), 0, 0, 1, 1.0, _p(info), None, 0, _st()) == 8
    torch.cuda.synchronize()
    assert torch.equal(x, y)  # refused before any launch
    assert torch.equal(L.trsm(l, y), L.trsm(l, y))


def test_two_threads_two_streams_bitwise():
    n, batch = 1024, 2
    a1, a2 = spd(n, batch, 1), spd(n, batch, 2)
    lbar1 = torch.tril(torch.randn_like(a1))
    lbar2 = torch.tril(torch.randn_like(a2))
    ref = []
    for a, lbar in ((a1, lbar1), (a2, lbar2)):
        l = L.potrf(a)
        ref.append((l, L.potrf_backward(lbar, l)))
    torch.cuda.synchronize()
    out = [None, None]
    err = []
    barrier = threading.Barrier(2)

    def work(i, a, lbar):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                barrier.wait()
                for _ in range(3):  # overlapping enqueues of the look-ahead schedule
                    l = L.potrf(a)
                    ab = L.potrf_backward(lbar, l)
                s.synchronize()
            out[i] = (l, ab)
        except Exception as e:  # pragma: no cover
            err.append(e)

    ts = [threading.Thread(target=work, args=(0, a1, lbar1)), threading.Thread(target=work, args=(1, a2, lbar2))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not err, err
    for (l, ab), (lr, abr) in zip(out, ref):
        assert torch.equal(l, lr) and torch.equal(ab, abr)


@pytest.mark.parametrize("n,batch", [(256, 64), (1024, 12)])
def test_batched_potrf_matches_per_slice(n, batch):
    # batch * chunks > SMs takes the throughput schedule (factor + explicit
    # L11^-1 GEMM) for the whole batch; one slice alone takes the fused panel
    a = spd(n, batch, 77)
    lb = L.potrf(a)
    for i in (0, batch // 2, batch - 1):
        li = L.potrf(a[i:i + 1].contiguous())
        d = (lb[i:i + 1] - li).abs().max().item() / li.abs().max().item()
        assert d < 1e-13, d
        r = (a[i] - lb[i] @ lb[i].T).norm() / a[i].norm()
        assert r.item() < 1e-14
