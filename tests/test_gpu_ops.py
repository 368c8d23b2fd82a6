"""GPU parity: every operator's forward and backward through the C-ABI
(libdla_b200.so) against the pinned CPU oracle (oracle/oracle_impl.h) on the
same seeded inputs.

Bars (stated per the north star):
  * structure is exact: zeroed triangles are exactly 0, symmetric outputs are
    bit-symmetric, sumlogdiag's cotangent is exactly 0 off the diagonal,
    batched == per-slice bitwise, aliased == non-aliased bitwise;
  * floating point: max|gpu - oracle| / max(1, max|oracle|) <= TOL[dtype]
    on inputs with condition number <= ~10 (SPD recipe X X^T + n I), i.e.
    c * kappa * u * n with c ~ 1e2:  f64 1e-10,  f32 2e-3 (n <= 200).
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import linalg as L  # noqa: E402

TOL = {np.float64: 1e-10, np.float32: 2e-3}
DTYPES = [np.float64, np.float32]
FLAGS = list(itertools.product([0, 1], repeat=3))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def rel(got, want):
    return np.abs(got - want).max() / max(1.0, np.abs(want).max()) if want.size else 0.0


def assert_close(got, want, dt, scale=1.0):
    r = rel(got, want)
    assert r <= TOL[dt] * scale, f"rel err {r:.3e} > {TOL[dt] * scale:.1e}"


def batch_apply(f, *arrs):
    outs = [f(*[a[i] for a in arrs]) for i in range(arrs[0].shape[0])]
    if isinstance(outs[0], tuple):
        return tuple(np.stack([o[j] for o in outs]) for j in range(len(outs[0])))
    return np.stack(outs)


def tri_factor(r, nt, lower, dt, batch):
    t = np.stack([np.linalg.cholesky(O.random_spd(nt, r)) for _ in range(batch)])
    t = t if lower else np.swapaxes(t, -1, -2)
    noise = r.standard_normal(t.shape) * 0.0
    return np.ascontiguousarray(t + noise).astype(dt)


# ------------------------------------------------------------------- gemm
@pytest.mark.parametrize("dt", DTYPES)
def test_gemm_gemm2(port, dt):
    r = O.rng(1)
    B = 3
    # skinny shapes too: vector (n or m <= 8, k > 8) and outer-product (k <= 8) kernels
    # + the streaming single-vector kernels: matvec rows / columns (n = 1, even k),
    # rank-1 outer products (k = 1, even n), ragged (odd) fallbacks
    for m, n, k in [(3, 5, 4), (1, 1, 1), (17, 9, 33), (64, 70, 65), (130, 129, 66), (1, 1, 300), (130, 3, 200),
                    (5, 130, 70), (70, 1, 130), (40, 2, 50), (66, 90, 3), (128, 1, 128), (1, 128, 128),
                    (129, 1, 64), (64, 128, 1), (5, 6, 1), (300, 1, 258)]:
        for ta, tb in itertools.product([0, 1], repeat=2):
            a = r.standard_normal((B,) + ((k, m) if ta else (m, k))).astype(dt)
            b = r.standard_normal((B,) + ((n, k) if tb else (k, n))).astype(dt)
            c0 = r.standard_normal((B, m, n)).astype(dt)
            want = batch_apply(lambda x, y: port.gemm(x, y, ta, tb, 1.25), a, b)
            got = host(L.gemm2(dev(a), dev(b), ta, tb, 1.25))
            assert_close(got, want, dt)
            c = dev(c0)
            L.gemm_into(c, dev(a), dev(b), ta, tb, 0.5, 1.0)
            want = batch_apply(lambda x, y, z: port.gemm(x, y, ta, tb, 0.5, z, 1), a, b, c0)
            assert_close(host(c), want, dt)
            c = dev(c0)
            L.gemm_into(c, dev(a), dev(b), ta, tb, 0.5, -0.25)
            assert_close(host(c), batch_apply(lambda x, y: port.gemm(x, y, ta, tb, 0.5), a, b) - 0.25 * c0, dt)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("mnk", [(7, 9, 5), (128, 1, 128), (64, 128, 1), (130, 70, 200), (257, 3, 300),
                                 (300, 260, 150)])
def test_gemm_backward(port, dt, mnk):
    r = O.rng(2)
    B, (m, n, k) = 2, mnk
    for ta, tb in itertools.product([0, 1], repeat=2):
        a = r.standard_normal((B,) + ((k, m) if ta else (m, k))).astype(dt)
        b = r.standard_normal((B,) + ((n, k) if tb else (k, n))).astype(dt)
        cb = r.standard_normal((B, m, n)).astype(dt)
        ga, gb = L.gemm2_backward(dev(cb), dev(a), dev(b), ta, tb, 0.75)
        wa, wb = batch_apply(lambda x, y, z: port.gemm2_bwd(x, y, z, ta, tb, 0.75), cb, a, b)
        assert_close(host(ga), wa, dt)
        assert_close(host(gb), wb, dt)
        cio = dev(cb)
        ga2, gb2, _ = L.gemm_backward_into(torch.empty_like(ga), torch.empty_like(gb), cio, dev(a), dev(b), ta, tb,
                                           0.75, 0.5)
        assert torch.equal(ga2, ga) and torch.equal(gb2, gb)
        assert_close(host(cio), 0.5 * cb, dt)


def test_sgemm_tcgen05_3xtf32():
    """Large fp32 products run on tcgen05 (kind::tf32, 3xTF32 split, packed
    tiles moved by bulk async copies): fp32-level accuracy on every
    transposition, ragged edges, batch, alpha / beta, masks and triangular
    operands (through trmm)."""
    torch.manual_seed(3)
    for (B, m, n, k) in ((1, 256, 256, 128), (2, 300, 270, 333)):
        for ta, tb in itertools.product([False, True], repeat=2):
            a = torch.randn(B, *((k, m) if ta else (m, k)), device="cuda")
            b = torch.randn(B, *((n, k) if tb else (k, n)), device="cuda")
            c0 = torch.randn(B, m, n, device="cuda")
            c = c0.clone()
            L.gemm_into(c, a, b, ta, tb, 0.7, 0.3)
            ad, bd = a.double(), b.double()
            want = 0.7 * (ad.transpose(-1, -2) if ta else ad) @ (bd.transpose(-1, -2) if tb else bd) + 0.3 * c0.double()
            assert ((c.double() - want).abs().max() / want.abs().max()).item() < 1e-5  # fp32-level (k <= 333)
    r = O.rng(12)
    t = tri_factor(r, 384, True, np.float32, 2)
    x = r.standard_normal((2, 384, 300)).astype(np.float32)
    got = host(L.trmm(dev(t), dev(x), False, True, True, 1.0))
    want = np.einsum("bki,bkj->bij", t.astype(np.float64), x.astype(np.float64))
    assert np.abs(got - want).max() / np.abs(want).max() < 1e-5


def test_gemm_rejects_alias_and_shape():
    a = torch.zeros(3, 3, dtype=torch.float64, device="cuda")
    with pytest.raises(L.Error):
        L.gemm2_into(a, a, a)
    with pytest.raises(L.ShapeError):
        L.gemm2_into(torch.zeros(2, 4, dtype=torch.float64, device="cuda"),
                     torch.zeros(2, 3, dtype=torch.float64, device="cuda"),
                     torch.zeros(4, 4, dtype=torch.float64, device="cuda"))


# ------------------------------------------------------------------- syrk
@pytest.mark.parametrize("dt", DTYPES)
def test_syrk(port, dt):
    r = O.rng(3)
    B = 2
    for n, k in [(4, 6), (1, 3), (65, 17), (100, 130), (64, 1), (6, 1), (7, 1)]:  # k = 1: masked rank-1 kernel
        for ta in (0, 1):
            a = r.standard_normal((B,) + ((k, n) if ta else (n, k))).astype(dt)
            got = L.syrk(dev(a), ta, 0.75)
            assert torch.equal(got, got.transpose(-1, -2)), "syrk must be bit-symmetric"
            assert_close(host(got), batch_apply(lambda x: port.syrk(x, ta, 0.75), a), dt)
            bb = r.standard_normal((B, n, n)).astype(dt)
            ga = L.syrk_backward(dev(bb), dev(a), ta, 0.5)
            assert_close(host(ga), batch_apply(lambda x, y: port.syrk_bwd(x, y, ta, 0.5), bb, a), dt)


def test_syrk_tma_path(port):
    """f64 A A^T at m >= 256 runs the TMA-fed persistent kernel (syrk_tma.cu):
    clipped last tile rows/columns, k not a multiple of the 16-wide k-chunk,
    batches; bit-symmetric output equal to the oracle."""
    r = O.rng(33)
    for n, k, B in [(256, 64, 1), (300, 40, 2), (513, 130, 1), (1000, 64, 3), (640, 7, 2)]:
        a = r.standard_normal((B, n, k))
        got = L.syrk(dev(a), False, -0.5)
        assert torch.equal(got, got.transpose(-1, -2)), "syrk must be bit-symmetric"
        assert_close(host(got), batch_apply(lambda x: port.syrk(x, 0, -0.5), a), np.float64)


# ------------------------------------------------------------ trmm / trsm
SHAPES = [(4, 3), (1, 5), (33, 17), (70, 65), (130, 7), (7, 130), (256, 130), (130, 256), (128, 70), (128, 200)]


@pytest.mark.parametrize("dt", DTYPES)
def test_trmm_trsm_forward(port, dt):
    r = O.rng(4)
    B = 2
    for (m, n), (right, tr, lo) in itertools.product(SHAPES, FLAGS):
        nt = n if right else m
        t = tri_factor(r, nt, lo, dt, B)
        # garbage in the unreferenced triangle must be ignored
        t = t + (np.triu(np.ones((nt, nt)), 1) if lo else np.tril(np.ones((nt, nt)), -1)).astype(dt) * 7
        x = r.standard_normal((B, m, n)).astype(dt)
        got = host(L.trmm(dev(t), dev(x), right, tr, lo, 1.5))
        assert_close(got, batch_apply(lambda tt, xx: port.trmm(tt, xx, right, tr, lo, 1.5), t, x), dt)
        got = host(L.trsm(dev(t), dev(x), right, tr, lo, 0.8))
        assert_close(got, batch_apply(lambda tt, xx: port.trsm(tt, xx, right, tr, lo, 0.8), t, x), dt, 10)


@pytest.mark.parametrize("dt", DTYPES)
def test_into_variants_match_inplace(port, dt):
    """Out-of-place trmm / potri (the reference's functional forms): equal to the
    in-place operators (bitwise) and to the oracle; inputs unchanged."""
    r = O.rng(19)
    B = 2
    for (m, n), (right, tr, lo) in itertools.product([(128, 70), (70, 128), (33, 17), (256, 130)], FLAGS):
        nt = n if right else m
        t = dev(tri_factor(r, nt, lo, dt, B))
        x = dev(r.standard_normal((B, m, n)).astype(dt))
        x0, t0 = x.clone(), t.clone()
        y = L.trmm_into(torch.empty_like(x), t, x, right, tr, lo, 1.5)
        assert torch.equal(x, x0) and torch.equal(t, t0)
        assert torch.equal(y, L.trmm_inplace(t, x.clone(), right, tr, lo, 1.5))
        assert_close(host(y), batch_apply(lambda tt, xx: port.trmm(tt, xx, right, tr, lo, 1.5), host(t), host(x)), dt)
    for n in (20, 65, 100, 128, 200):
        a = O.random_spd(n, r, dt, batch=B)
        for lower in (1, 0):
            l = dev(batch_apply(lambda x: port.potrf(x, lower), a))
            l0 = l.clone()
            b = L.potri_into(torch.empty_like(l), l, lower)
            assert torch.equal(l, l0)
            assert torch.equal(b, L.potri_inplace(l.clone(), lower))
            assert torch.equal(b, b.transpose(-1, -2))
            assert_close(host(b), batch_apply(lambda x: port.potri(x, lower), host(l)), dt, 10)
    with pytest.raises(L.ShapeError):
        L.potri_into(torch.empty(B, 5, 5, dtype=torch.float64, device="cuda"), dev(np.eye(6)[None].repeat(B, 0)))


@pytest.mark.parametrize("dt", DTYPES)
def test_trmm_trsm_backward(port, dt):
    r = O.rng(5)
    B = 2
    # + nt = 128: the out-of-place triangular-GEMM pullbacks (and their aliased in-place twins, bitwise)
    for (m, n), (right, tr, lo) in itertools.product(SHAPES[:4] + [(128, 70), (70, 128)], FLAGS):
        nt = n if right else m
        t = tri_factor(r, nt, lo, dt, B)
        x = r.standard_normal((B, m, n)).astype(dt)
        bb = r.standard_normal((B, m, n)).astype(dt)
        ga, gt = L.trmm_backward(dev(bb), dev(t), dev(x), right, tr, lo, 1.5)
        wa, wt = batch_apply(lambda b_, t_, x_: port.trmm_bwd(b_, t_, x_, right, tr, lo, 1.5), bb, t, x)
        assert_close(host(ga), wa, dt)
        assert_close(host(gt), wt, dt)
        mask = np.triu(np.ones((nt, nt)), 1) if lo else np.tril(np.ones((nt, nt)), -1)
        assert np.all(host(gt)[:, mask.astype(bool)] == 0)
        # abar may alias bbar (dl/adjoints.hpp:90-91): bitwise identical
        alias = dev(bb)
        ga2, gt2 = L.trmm_backward_into(alias, torch.empty_like(gt), alias, dev(t), dev(x), right, tr, lo, 1.5)
        assert torch.equal(ga2, ga) and torch.equal(gt2, gt)
        # trsm: the backward consumes the forward OUTPUT
        y = port_out = batch_apply(lambda t_, x_: port.trsm(t_, x_, right, tr, lo, 0.8), t, x)
        ga, gt = L.trsm_backward(dev(bb), dev(t), dev(port_out), right, tr, lo, 0.8)
        wa, wt = batch_apply(lambda b_, t_, y_: port.trsm_bwd(b_, t_, y_, right, tr, lo, 0.8), bb, t, y)
        assert_close(host(ga), wa, dt, 10)
        assert_close(host(gt), wt, dt, 10)
        assert np.all(host(gt)[:, mask.astype(bool)] == 0)
        alias = dev(bb)
        ga2, gt2 = L.trsm_backward_into(alias, torch.empty_like(gt), alias, dev(t), dev(y), right, tr, lo, 0.8)
        assert torch.equal(ga2, ga) and torch.equal(gt2, gt)


@pytest.mark.parametrize("dt", DTYPES)
def test_trsv_narrow_large(port, dt):
    """The one-launch narrow solve (<= 8 vectors, n > 64): every flag set at
    sizes with a ragged last block, more blocks than SMs, and a batch."""
    r = O.rng(41)
    for (nt, nv, B), (right, tr, lo) in itertools.product([(1000, 1, 2), (577, 8, 1), (2112, 3, 3)], FLAGS):
        t = tri_factor(r, nt, lo, dt, B)
        x = r.standard_normal((B, nv, nt) if right else (B, nt, nv)).astype(dt)
        got = host(L.trsm(dev(t), dev(x), right, tr, lo, 0.7))
        assert_close(got, batch_apply(lambda tt, xx: port.trsm(tt, xx, right, tr, lo, 0.7), t, x), dt, 10)


def test_trsm_singular_reports_index_and_leaves_slice():
    t = dev(np.array([[[2.0, 0], [1, 1]], [[1.0, 0], [5, 0]]]))
    x0 = np.array([[[2.0], [3.0]], [[2.0], [3.0]]])
    x = dev(x0)
    with pytest.raises(L.SingularError) as e:
        L.trsm_inplace(t, x)
    assert e.value.index == 1 and e.value.batch_index == 1
    got = host(x)
    np.testing.assert_allclose(got[0], [[1.0], [2.0]], rtol=1e-14)  # KAT tests/test_blas_kernels.cpp:179-184
    assert np.array_equal(got[1], x0[1]), "failing slice must be untouched"


# ----------------------------------------------------------- potrf / potri
POTRF_N = [1, 2, 5, 17, 32, 63, 64, 65, 70, 96, 128, 129, 200, 256, 512]  # 65-128 f64: one-launch kernel; 256/512: inverse-based DMMA paths


def test_potrf_throughput_panel_path():
    """Large batches of multi-chunk panels take the one-factorization-per-slice
    path (diagonal block + inverse, then an in-place batched DMMA panel
    solve); same answer as LAPACK, failures still reported per slice."""
    r = O.rng(79)
    for n, B in ((256, 64), (1024, 12)):
        a = O.random_spd(n, r, batch=B)
        got = host(L.potrf(dev(a)))
        want = np.linalg.cholesky(a)
        assert np.abs(got - want).max() / np.abs(want).max() < 1e-12
        assert np.all(np.triu(got, 1) == 0)
    a = O.random_spd(256, r, batch=64)
    a[17, 130, 130] = -1e4
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        L.potrf(dev(a))
    assert e.value.batch_index == 17 and e.value.step == 130


def test_potrf_bwd_split_is_bitwise_the_op():
    """dla_potrf_bwd_{begin,end}_f64 (L^-1 on a side stream, used by the GP
    driver) must reproduce dla_potrf_bwd_f64 bit for bit."""
    import ctypes as C
    from paper_1710_08717_b200._lib import lib
    lb = lib().lib
    r = O.rng(78)
    for n, B in ((256, 2), (512, 1), (300, 2)):
        l = dev(np.linalg.cholesky(O.random_spd(n, r, batch=B)))
        lbar = dev(np.tril(r.standard_normal((B, n, n))))
        want = L.potrf_backward(lbar, l)
        nb = int(lb.dla_potrf_bwd_ws_bytes_f64(B, n))
        ws = torch.empty(max(nb, 8), dtype=torch.uint8, device="cuda")
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        got = torch.empty_like(l)
        assert lb.dla_potrf_bwd_begin_f64(B, n, C.c_void_p(l.data_ptr()), 1, C.c_void_p(ws.data_ptr()), nb, st) == 0
        assert lb.dla_potrf_bwd_end_f64(B, n, C.c_void_p(got.data_ptr()), C.c_void_p(lbar.data_ptr()),
                                        C.c_void_p(l.data_ptr()), 1, C.c_void_p(ws.data_ptr()), nb, st) == 0
        torch.cuda.synchronize()
        assert torch.equal(got, want)


def test_potrf_large_blocked_lookahead():
    """Blocked look-ahead path at sizes with many panel CTAs per launch (the
    panel kernel's redundant A11 reads must never see the written L11)."""
    r = O.rng(77)
    for n, B in ((1024, 6), (2112, 1)):
        a = O.random_spd(n, r, batch=B)
        for _ in range(3):
            got = host(L.potrf(dev(a)))
            want = np.linalg.cholesky(a)
            assert np.abs(got - want).max() / np.abs(want).max() < 1e-12
            assert np.all(np.triu(got, 1) == 0)


@pytest.mark.parametrize("dt", DTYPES)
def test_potrf_forward(port, dt):
    r = O.rng(6)
    B = 3
    for n in POTRF_N:
        a = O.random_spd(n, r, dt, batch=B)
        for lower in (1, 0):
            got = host(L.potrf(dev(a), lower))
            want = batch_apply(lambda x: port.potrf(x, lower), a)
            zero = np.triu(np.ones((n, n)), 1) if lower else np.tril(np.ones((n, n)), -1)
            assert np.all(got[:, zero.astype(bool)] == 0), "opposite triangle must be exactly zero"
            assert np.all(np.diagonal(got, axis1=1, axis2=2) > 0)
            assert_close(got, want, dt)
            # backward error ||A - L L^T|| / ||A||
            l64 = got.astype(np.float64)
            back = l64 @ np.swapaxes(l64, 1, 2) if lower else np.swapaxes(l64, 1, 2) @ l64
            be = np.abs(back - a).max() / np.abs(a).max()
            assert be <= (1e-12 if dt == np.float64 else 1e-5), f"backward error {be}"
            # batched == per-slice, bitwise
            one = host(L.potrf(dev(a[1]), lower))
            assert np.array_equal(one, got[1])


def test_potrf_errors():
    bad = dev(np.array([[1.0, 0, 0], [0, 1, 0], [0, 0, -1]]))
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        L.potrf(bad)
    assert e.value.step == 2  # tests/test_cholesky.cpp:46-55
    with pytest.raises(L.ShapeError):
        L.potrf(dev(np.array([[1.0, 2], [0, 1]])))
    # large-n path: failure at a pivot beyond the first leaf
    r = O.rng(7)
    n = 150
    a = O.random_spd(n, r)
    a[100, 100] = -1e6
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        L.potrf(dev(a))
    assert e.value.step == 100
    asym = O.random_spd(n, r)
    asym[3, 140] += 1.0
    with pytest.raises(L.ShapeError):
        L.potrf(dev(asym))
    # per-slice: only the bad slice fails, the others are factored
    ab = O.random_spd(40, r, batch=3)
    ab[2, 5, 5] = -1e6
    x = dev(ab)
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        L.potrf_inplace(x)
    assert e.value.batch_index == 2 and e.value.step == 5
    np.testing.assert_allclose(host(x)[0], np.linalg.cholesky(ab[0]), rtol=1e-10, atol=1e-12)
    # one-launch path (64 < n <= 128, f64): failures in A11, in A22, asymmetry, per slice
    for n, k in ((100, 30), (100, 90), (128, 127), (65, 64)):
        a = O.random_spd(n, r, batch=3)
        a[1, k, k] = -1e6
        x = dev(a)
        with pytest.raises(L.NotPositiveDefiniteError) as e:
            L.potrf_inplace(x)
        assert e.value.batch_index == 1 and e.value.step == k
        for b in (0, 2):
            np.testing.assert_allclose(host(x)[b], np.linalg.cholesky(a[b]), rtol=1e-10, atol=1e-12)
    asym = O.random_spd(128, r)
    asym[3, 100] += 1.0
    with pytest.raises(L.ShapeError):
        L.potrf(dev(asym))
    asym = O.random_spd(100, r)
    asym[70, 90] += 1.0  # inside the A22 block
    with pytest.raises(L.ShapeError):
        L.potrf(dev(asym))
    # tile-dataflow path (n >= 256): failure deep inside one slice, the other factored
    a2 = O.random_spd(300, r, batch=2)
    a2[1, 200, 200] = -1e6
    x = dev(a2)
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        L.potrf_inplace(x)
    assert e.value.batch_index == 1 and e.value.step == 200
    np.testing.assert_allclose(np.tril(host(x)[0]), np.linalg.cholesky(a2[0]), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("dt", DTYPES)
def test_potrf_backward(port, dt):
    r = O.rng(8)
    B = 2
    for n in POTRF_N:
        a = O.random_spd(n, r, dt, batch=B)
        for lower in (1, 0):
            l = batch_apply(lambda x: port.potrf(x, lower), a)
            lbar = r.standard_normal((B, n, n)).astype(dt)
            got = L.potrf_backward(dev(lbar), dev(l), lower)
            assert torch.equal(got, got.transpose(-1, -2)), "Abar must be bit-symmetric"
            want = batch_apply(lambda x, y: port.potrf_bwd(x, y, lower), lbar, l)
            assert_close(host(got), want, dt, 10)
            alias = dev(lbar)
            L.potrf_backward_into(alias, alias, dev(l), lower)
            assert torch.equal(alias, got), "aliased potrf backward must match bitwise"


@pytest.mark.parametrize("dt", DTYPES)
def test_potrf_warp_batches(port, dt):
    """n <= 32 runs a warp per matrix, 4-8 matrices per CTA: ragged batches."""
    r = O.rng(18)
    for n, B in [(32, 13), (9, 17), (1, 9)]:
        a = O.random_spd(n, r, dt, batch=B)
        for lower in (1, 0):
            got = host(L.potrf(dev(a), lower))
            assert_close(got, batch_apply(lambda x: port.potrf(x, lower), a), dt)
            lbar = r.standard_normal((B, n, n)).astype(dt)
            gb = host(L.potrf_backward(dev(lbar), dev(got), lower))
            assert_close(gb, batch_apply(lambda x, y: port.potrf_bwd(x, y, lower), lbar, got), dt, 10)


@pytest.mark.parametrize("dt", DTYPES)
def test_potri(port, dt):
    r = O.rng(9)
    B = 2
    for n in [1, 2, 3, 8, 20, 64, 65, 96, 100, 128, 129]:  # 65-128 f64: one fused launch
        a = O.random_spd(n, r, dt, batch=B)
        for lower in (1, 0):
            l = batch_apply(lambda x: port.potrf(x, lower), a)
            got = L.potri(dev(l), lower)
            assert torch.equal(got, got.transpose(-1, -2)), "potri output must be bit-symmetric"
            want = batch_apply(lambda x: port.potri(x, lower), l)
            assert_close(host(got), want, dt, 10)
            bbar = r.standard_normal((B, n, n)).astype(dt)
            gl = host(L.potri_backward(dev(bbar), dev(l), dev(want), lower))
            wl = batch_apply(lambda x, y, z: port.potri_bwd(x, y, z, lower), bbar, l, want)
            assert_close(gl, wl, dt, 10)
            zero = np.triu(np.ones((n, n)), 1) if lower else np.tril(np.ones((n, n)), -1)
            assert np.all(gl[:, zero.astype(bool)] == 0)
    with pytest.raises(L.SingularError) as e:
        L.potri(dev(np.array([[2.0, 0], [1, 0]])))
    assert e.value.index == 1


# -------------------------------------------------------------- sumlogdiag
@pytest.mark.parametrize("dt", DTYPES)
def test_sumlogdiag(port, dt):
    r = O.rng(10)
    for n in [1, 2, 32, 100, 1500]:
        l = np.abs(r.standard_normal((3, n, n))).astype(dt) + 0.5
        got = host(L.sumlogdiag(dev(l)))
        want = np.array([port.sumlogdiag(x) for x in l])
        assert_close(got, want, dt)
        g = r.standard_normal(3).astype(dt)
        ab = host(L.sumlogdiag_backward_into(torch.empty(3, n, n, dtype=dev(l).dtype, device="cuda"), dev(g), dev(l)))
        off = ~np.eye(n, dtype=bool)
        assert np.all(ab[:, off] == 0), "off-diagonal cotangent must be exactly zero"
        want = np.stack([port.sumlogdiag_bwd(g[i], l[i]) for i in range(3)])
        assert_close(ab, want, dt)
        base = r.standard_normal((3, n, n)).astype(dt)
        acc = dev(base)
        L.sumlogdiag_backward_into(acc, dev(g), dev(l), accumulate=True)
        accn = host(acc)
        assert np.array_equal(accn[:, off], base[:, off]), "accumulate touches the diagonal only"
        assert_close(accn, base + want, dt)


# ------------------------------------------------------------------ gelqf
def test_gelqf_cholesky_qr2_fallback(port):
    """f64 64 <= m <= 512 runs CholeskyQR2 (csrc/gelqf_cqr.cu); slices it cannot
    serve fall back to the Householder path per slice: an ill-conditioned
    slice (row scales 1e0 .. 1e-9, kappa ~ 1e9) must still match the oracle,
    and a rank-deficient slice must raise the reference's SingularError with
    the reference's index while its neighbours complete."""
    r = O.rng(23)
    m, n, B = 128, 300, 4
    a = r.standard_normal((B, m, n))
    a[1] *= np.logspace(0, -9, m)[:, None]        # ill-conditioned: fallback, still full rank
    q, l = L.gelqf(dev(a))
    q, l = host(q), host(l)
    wq, wl = batch_apply(port.gelqf, a)
    assert_close(q, wq, np.float64, 10)
    for b in range(B):  # L row scales span 1e9: compare per row
        assert np.abs(l[b] - wl[b]).max(axis=1).max() <= 1e-9 * np.abs(wl[b]).max() + 1e-300
        np.testing.assert_allclose(l[b], wl[b], rtol=1e-6, atol=1e-13 * np.abs(wl[b]).max())
    # orthonormal rows on every path
    for b in range(B):
        assert np.abs(q[b] @ q[b].T - np.eye(m)).max() < 1e-13
    a2 = r.standard_normal((B, m, n))
    a2[2, 70] = a2[2, 3] + 2.0 * a2[2, 40]         # rank deficient at row 70
    with pytest.raises(L.SingularError) as e:
        L.gelqf(dev(a2))
    assert e.value.batch_index == 2
    with pytest.raises(O.OracleError) as eo:
        port.gelqf(a2[2])
    assert e.value.index == eo.value.index


@pytest.mark.parametrize("dt", DTYPES)
def test_gelqf(port, dt):
    r = O.rng(11)
    B = 2
    for m, n in [(1, 1), (2, 5), (4, 4), (7, 11), (16, 16), (32, 128), (128, 512), (70, 300), (96, 96), (64, 65)]:
        a = r.standard_normal((B, m, n)).astype(dt)
        q, l = L.gelqf(dev(a))
        q, l = host(q), host(l)
        wq, wl = batch_apply(port.gelqf, a)
        assert np.all(l[:, np.triu(np.ones((m, m)), 1).astype(bool)] == 0)
        assert np.all(np.diagonal(l, axis1=1, axis2=2) > 0)
        s = 50 if dt == np.float32 else 10
        assert_close(q, wq, dt, s)
        assert_close(l, wl, dt, s)
        qb = r.standard_normal((B, m, n)).astype(dt)
        lb = np.tril(r.standard_normal((B, m, m))).astype(dt)
        ga = host(L.gelqf_backward(dev(qb), dev(lb), dev(wq), dev(wl)))
        want = batch_apply(port.gelqf_bwd, qb, lb, wq, wl)
        assert_close(ga, want, dt, s)
    k = dev(np.array([[3.0, 4.0]]).astype(dt))
    q, l = L.gelqf(k)
    np.testing.assert_allclose(host(l), [[5.0]], rtol=1e-6)
    np.testing.assert_allclose(host(q), [[0.6, 0.8]], rtol=1e-6)
    with pytest.raises(L.SingularError):
        L.gelqf(dev(np.array([[1.0, 2, 3], [2, 4, 6]])))
    with pytest.raises(L.ShapeError):
        L.gelqf(dev(np.zeros((3, 2))))
    # blocked path (m >= 64): rank deficiency and an all-zero slice, with a
    # healthy slice beside them left exactly as the unbatched call computes it
    a = r.standard_normal((3, 80, 120)).astype(dt)
    a[1, 50] = 2 * a[1, 7]
    a[2] = 0
    ok_q, ok_l = L.gelqf(dev(a[:1]))
    qd, ld = dev(a), torch.empty(3, 80, 80, dtype=dev(a).dtype, device="cuda")
    with pytest.raises(L.SingularError) as e:
        L.gelqf_inplace(qd, ld)
    assert e.value.batch_index == 1 and e.value.index == 50
    assert torch.equal(qd[0], ok_q[0]) and torch.equal(ld[0], ok_l[0])


# ------------------------------------------------------------------ syevd
def gapped_sym(r, n, dt, batch, gap=1e-3):
    out = []
    while len(out) < batch:
        a = O.random_sym(n, r) * np.sqrt(n)
        w = np.linalg.eigvalsh(a)
        if n == 1 or np.diff(w).min() >= gap:
            out.append(a)
    return np.stack(out).astype(dt)


@pytest.mark.parametrize("dt", DTYPES)
def test_syevd(port, dt):
    r = O.rng(12)
    B = 3
    for n in [1, 2, 3, 8, 16, 25, 32, 63, 64]:
        a = gapped_sym(r, n, dt, B)
        u, lam = L.syevd(dev(a))
        u, lam = host(u), host(lam)
        wu, wlam = batch_apply(port.syevd, a)
        assert np.all(np.diff(lam, axis=1) >= 0)
        s = 100 if dt == np.float32 else 1000
        assert_close(lam, wlam, dt, s)
        assert_close(u, wu, dt, s)   # separated spectrum: elementwise incl. the sign rule
        ub = r.standard_normal((B, n, n)).astype(dt)
        lb = r.standard_normal((B, n)).astype(dt)
        ga = L.syevd_backward(dev(ub), dev(lb), dev(wu), dev(wlam))
        assert torch.equal(ga, ga.transpose(-1, -2))
        want = batch_apply(lambda x, y, z, w: port.syevd_bwd(x, y, z, w), ub, lb, wu, wlam)
        assert_close(host(ga), want, dt, s)


def test_syevd_kats_and_degenerate(port):
    h = np.sqrt(0.5)
    u, lam = L.syevd(dev(np.array([[0.0, 1], [1, 0]])))
    np.testing.assert_allclose(host(lam), [-1, 1], atol=1e-14)
    np.testing.assert_allclose(host(u), [[h, -h], [h, h]], atol=1e-14)
    u, lam = L.syevd(dev(np.diag([3.0, -7, 1])))
    np.testing.assert_allclose(host(lam), [-7, 1, 3])
    assert host(u)[0, 1] == 1 and host(u)[1, 2] == 1 and host(u)[2, 0] == 1
    with pytest.raises(L.ShapeError):
        L.syevd(dev(np.array([[1.0, 2], [0, 1]])))
    r = O.rng(77)
    cases = [np.eye(8), np.zeros((5, 5)), np.diag([2.0, 2, 1])]
    for s in (1e150, 1e-150):
        cases.append(O.random_sym(12, r) * s)
    q, _ = np.linalg.qr(r.standard_normal((6, 6)))
    cases.append(q.T @ np.diag([1, 1, 1, 2, 2, 3.0]) @ q)
    for a in cases:
        a = 0.5 * (a + a.T)
        u, lam = L.syevd(dev(a))
        u, lam = host(u), host(lam)
        n = a.shape[0]
        assert np.all(np.diff(lam) >= 0)
        amax = max(np.abs(a).max(), np.finfo(float).tiny)
        assert np.abs(u @ u.T - np.eye(n)).max() < 1e-10
        assert np.abs(u.T @ np.diag(lam) @ u - a).max() / amax < 1e-10


def test_syevd_bwd_finite_at_zero_gap():
    u = dev(np.eye(3))
    lam = dev(np.array([1.0, 1.0 + 1e-12, 2.0]))
    ub = dev(np.array([[0.3, -0.2, 0.9], [0.1, 0.4, -0.5], [0.7, 0.2, 0.1]]))
    lb = dev(np.array([0.2, -0.3, 0.4]))
    g = host(L.syevd_backward(ub, lb, u, lam))
    assert np.all(np.isfinite(g))
    g0 = host(L.syevd_backward(ub, lb, u, dev(np.array([1.0, 1.0, 2.0]))))
    assert np.all(np.isfinite(g0))
