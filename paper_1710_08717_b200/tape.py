"""Device-resident tape: the reference's ``Graph`` (dl/tape.hpp) with every
node value, every gradient (``GradStore``) and the memory plan on the GPU.

SURVEY §8f row 3.  The reference tape records nodes eagerly, recomputes them
in ``forward(bindings)``, differentiates with ``backward(loss)`` into a
``GradStore`` and, with ``set_use_memory_plan(true)``, lets an in-place node
take over its input's buffer when that input has no later forward reader and
is not re-read by the backward pass (``build_plan``, dl/tape.hpp:1127-1209;
retention tables ``backward_reads_input/output`` :160-189).  Here:

* linear-algebra nodes (gemm2, syrk, trmm, trsm, potrf, potri, gelqf, syevd,
  gesvd) and their pullbacks are libdla_b200.so operators (linalg.py);
* the elementwise / structural nodes and pullbacks, and ``Graph::acc``
  (:920-929), are ``dla_tape_ew_*`` kernels (csrc/tape_ew.cu) — an
  accumulate flag adds into the existing gradient in place;
* the memory plan is the reference's rule set, restated: a donated buffer is
  the output (the op runs in place on device), the donor's value reads as
  released; results are bitwise identical with the plan on or off (the same
  kernels on the same values), as the reference tests
  (proj/tests/test_tape.cpp:124-148).

``device_bytes()`` / ``peak_bytes`` report the node-value memory the plan
saves (torch's caching allocator provides the buffers and the zero-filled
gradient slots: plumbing only — every value and gradient is computed by a
libdla_b200.so kernel, including the reference's ``base_of`` copies).
"""
from __future__ import annotations

import ctypes as C
from typing import NamedTuple

import torch

from . import linalg as L
from ._lib import lib

# dla_ew_op (include/dla.h)
EW = dict(COPY=0, ADD=1, SUB=2, MUL=3, SQUARE=4, SQRT=5, LOG=6, EXP=7, ABS=8, NEG=9, SCALE=10, ADDC=11, MULS=12,
          DIVS=13, FILL=14, SQUARE_BWD=15, SQRT_BWD=16, LOG_BWD=17, ABS_BWD=18, TRIL=19, TRIU=20, TILECOLS=21,
          TILEROWS=22, EXTRACTDIAG=23, MAKEDIAG=24, CONCATCOLS=25, SLICECOLS=26, SUMROWS=27, SUMCOLS=28, SUM=29,
          DOT=30, DOT_NEG_DIV=31)

OPS = ("leaf", "const", "gemm2", "syrk", "trmm", "trsm", "potrf", "potri", "gelqf", "syevd", "gesvd", "add", "sub",
       "mul", "square", "sqrt", "log", "exp", "abs", "neg", "scale_const", "add_const", "mul_scalar", "div_scalar",
       "sum", "sum_rows", "tile_cols", "tile_rows", "extract_diag", "make_diag", "tril_mask", "triu_mask",
       "concat_cols")
_UNARY_EW = {"square": "SQUARE", "sqrt": "SQRT", "log": "LOG", "exp": "EXP", "abs": "ABS", "neg": "NEG",
             "tril_mask": "TRIL", "triu_mask": "TRIU"}
_BINARY_EW = {"add": "ADD", "sub": "SUB", "mul": "MUL"}


class NodeId(NamedTuple):
    node: int
    slot: int = 0


# dl/tape.hpp:160-189 — what each pullback re-reads
def backward_reads_input(op: str, k: int) -> bool:
    if op in ("gemm2", "syrk", "trmm", "mul", "square", "log", "abs", "mul_scalar"):
        return True
    if op in ("trsm", "potri"):
        return k == 0
    if op == "div_scalar":
        return k == 1
    return False


def backward_reads_output(op: str, s: int) -> bool:
    if op in ("potrf", "trsm", "potri", "gelqf", "syevd", "gesvd", "sqrt", "exp"):
        return True
    if op == "div_scalar":
        return s == 0
    return False


# in-place nodes of the plan: (output slot, donating input)   dl/tape.hpp:1160-1190
def _donation(op: str):
    if op in ("trmm", "trsm"):
        return 0, 1
    if op in ("potrf", "potri", "gelqf", "syevd"):
        return 0, 0
    if op == "gesvd":
        return 2, 0
    if op in ("add", "sub", "mul", "square", "sqrt", "log", "exp", "abs", "neg", "scale_const", "add_const",
              "mul_scalar", "div_scalar", "tril_mask", "triu_mask"):
        return 0, 0
    return None


class _Node:
    __slots__ = ("op", "name", "inp", "ta", "tb", "rightside", "transpose", "lower", "alpha", "cval", "count",
                 "out", "shapes")

    def __init__(self, op, inp=(), name=""):
        self.op, self.inp, self.name = op, list(inp), name
        self.ta = self.tb = self.rightside = self.transpose = False
        self.lower = True
        self.alpha, self.cval, self.count = 1.0, 0.0, 0
        self.out, self.shapes = [], []


class GradStore:
    """Device gradients by NodeId (dl/tape.hpp:191-213)."""

    def __init__(self, g):
        self._g = g

    def has(self, nid: NodeId) -> bool:
        return self._g.get((nid.node, nid.slot)) is not None

    def at(self, nid: NodeId) -> torch.Tensor:
        if not self.has(nid):
            raise L.Error(f"GradStore: no gradient recorded for node {nid.node} slot {nid.slot}")
        return self._g[(nid.node, nid.slot)]


class Graph:
    """Device mirror of dla::Graph<T> (dl/tape.hpp:216-1247)."""

    def __init__(self, dtype=torch.float64, device="cuda"):
        self.dtype, self.device = dtype, torch.device(device)
        self._nodes: list[_Node] = []
        self._use_plan = False
        self._assume_backward = True
        self.peak_bytes = 0
        sfx = "f64" if dtype == torch.float64 else "f32"
        self._ew = getattr(lib().lib, f"dla_tape_ew_{sfx}")
        scal = C.c_double if dtype == torch.float64 else C.c_float
        self._ew.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, scal,
                             C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
        self._ew.restype = C.c_int
        lib().lib.dla_tape_ew_ws_bytes.restype = C.c_size_t
        nb = int(lib().lib.dla_tape_ew_ws_bytes())
        self._ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        self._wsb = nb

    # ---------------------------------------------------------------- config
    def set_use_memory_plan(self, on: bool):
        self._use_plan = bool(on)

    def set_assume_backward(self, on: bool):
        self._assume_backward = bool(on)

    def use_memory_plan(self) -> bool:
        return self._use_plan

    def num_nodes(self) -> int:
        return len(self._nodes)

    def node_op(self, i: int) -> str:
        return self._nodes[i].op

    # ---------------------------------------------------------------- kernels
    def _k(self, op, rows, cols, x, out, y=None, s=None, c=0.0, aux=0, acc=False):
        P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        st = self._ew(EW[op], rows, cols, aux, P(x), P(y), P(s), c, P(out), int(acc), P(self._ws), self._wsb,
                      C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        if st:
            L._raise_status(st, f"tape {op}")
        return out

    def _empty(self, r, c):
        return torch.empty(r, c, dtype=self.dtype, device=self.device)

    def _zeros(self, r, c):
        return torch.zeros(r, c, dtype=self.dtype, device=self.device)

    # ---------------------------------------------------------------- builders
    def _mat(self, value):
        t = torch.as_tensor(value, dtype=self.dtype)
        if t.dim() == 1:
            t = t.reshape(-1, 1)
        if t.dim() != 2:
            raise L.ShapeError("Graph: node values are matrices")
        return t.to(self.device).contiguous().clone()

    def leaf(self, value, name: str = "") -> NodeId:
        n = _Node("leaf", name=name)
        n.out = [self._mat(value)]
        return self._finish(n)

    def constant(self, value, name: str = "c") -> NodeId:
        n = _Node("const", name=name)
        n.out = [self._mat(value)]
        return self._finish(n)

    def _start(self, op, inp):
        for i in inp:
            self.value(i)  # validates node and slot
        return _Node(op, inp)

    def _require(self, ok, n, msg):
        if not ok:
            raise L.ShapeError(f"{n.op}: {msg}")

    def _record(self, n):
        n.out = self._compute(n, None)
        return self._finish(n)

    def _finish(self, n):
        n.shapes = [tuple(t.shape) for t in n.out]
        self._nodes.append(n)
        self._track()
        return NodeId(len(self._nodes) - 1, 0)

    def gemm2(self, a, b, ta=False, tb=False, alpha=1.0):
        n = self._start("gemm2", [a, b])
        n.ta, n.tb, n.alpha = ta, tb, alpha
        sa, sb = self.shape(a), self.shape(b)
        self._require((sa[0] if ta else sa[1]) == (sb[1] if tb else sb[0]), n, "inner dimensions do not match")
        return self._record(n)

    def syrk(self, a, ta=False, alpha=1.0):
        n = self._start("syrk", [a])
        n.ta, n.alpha = ta, alpha
        return self._record(n)

    def _tri(self, op, t, a, rightside, transpose, lower, alpha):
        n = self._start(op, [t, a])
        n.rightside, n.transpose, n.lower, n.alpha = rightside, transpose, lower, alpha
        st, sa = self.shape(t), self.shape(a)
        self._require(st[0] == st[1], n, "triangular factor not square")
        self._require((sa[1] if rightside else sa[0]) == st[0], n, "operand does not match triangular factor")
        return self._record(n)

    def trmm(self, t, a, rightside, transpose, lower, alpha=1.0):
        return self._tri("trmm", t, a, rightside, transpose, lower, alpha)

    def trsm(self, t, a, rightside, transpose, lower, alpha=1.0):
        return self._tri("trsm", t, a, rightside, transpose, lower, alpha)

    def potrf(self, a, lower=True):
        n = self._start("potrf", [a])
        n.lower = lower
        self._require(self.shape(a)[0] == self.shape(a)[1], n, "matrix not square")
        return self._record(n)

    def potri(self, l, lower=True):
        n = self._start("potri", [l])
        n.lower = lower
        self._require(self.shape(l)[0] == self.shape(l)[1], n, "factor not square")
        return self._record(n)

    def gelqf(self, a):
        n = self._start("gelqf", [a])
        self._require(self.shape(a)[0] <= self.shape(a)[1], n, "needs rows <= cols")
        q = self._record(n)
        return q, NodeId(q.node, 1)

    def syevd(self, a):
        n = self._start("syevd", [a])
        self._require(self.shape(a)[0] == self.shape(a)[1], n, "matrix not square")
        u = self._record(n)
        return u, NodeId(u.node, 1)

    def gesvd(self, a):
        n = self._start("gesvd", [a])
        self._require(self.shape(a)[0] <= self.shape(a)[1], n, "needs rows <= cols")
        u = self._record(n)
        return u, NodeId(u.node, 1), NodeId(u.node, 2)

    def _binary(self, op, a, b):
        n = self._start(op, [a, b])
        self._require(self.shape(a) == self.shape(b), n, "operand shapes differ")
        return self._record(n)

    def add(self, a, b):
        return self._binary("add", a, b)

    def sub(self, a, b):
        return self._binary("sub", a, b)

    def mul(self, a, b):
        return self._binary("mul", a, b)

    def _unary(self, op, x):
        n = self._start(op, [x])
        if op in ("tril_mask", "triu_mask"):
            self._require(self.shape(x)[0] == self.shape(x)[1], n, "matrix not square")
        return self._record(n)

    def square(self, x):
        return self._unary("square", x)

    def sqrt(self, x):
        return self._unary("sqrt", x)

    def log(self, x):
        return self._unary("log", x)

    def exp(self, x):
        return self._unary("exp", x)

    def abs(self, x):
        return self._unary("abs", x)

    def neg(self, x):
        return self._unary("neg", x)

    def tril_mask(self, x):
        return self._unary("tril_mask", x)

    def triu_mask(self, x):
        return self._unary("triu_mask", x)

    def sum(self, x):
        return self._unary("sum", x)

    def sum_rows(self, x):
        return self._unary("sum_rows", x)

    def scale_const(self, x, c):
        n = self._start("scale_const", [x])
        n.cval = float(c)
        return self._record(n)

    def add_const(self, x, c):
        n = self._start("add_const", [x])
        n.cval = float(c)
        return self._record(n)

    def _scalar_op(self, op, x, s):
        n = self._start(op, [x, s])
        self._require(self.shape(s) == (1, 1), n, "scale is not 1x1")
        return self._record(n)

    def mul_scalar(self, x, s):
        return self._scalar_op("mul_scalar", x, s)

    def div_scalar(self, x, s):
        return self._scalar_op("div_scalar", x, s)

    def _tile(self, op, x, count):
        n = self._start(op, [x])
        n.count = int(count)
        self._require(self.shape(x)[1] == 1, n, "expects a column vector")
        self._require(count >= 1, n, "tile count must be positive")
        return self._record(n)

    def tile_cols(self, x, count):
        return self._tile("tile_cols", x, count)

    def tile_rows(self, x, count):
        return self._tile("tile_rows", x, count)

    def extract_diag(self, x):
        n = self._start("extract_diag", [x])
        self._require(self.shape(x)[0] == self.shape(x)[1], n, "matrix not square")
        return self._record(n)

    def make_diag(self, x):
        n = self._start("make_diag", [x])
        self._require(self.shape(x)[1] == 1, n, "expects a column vector")
        return self._record(n)

    def concat_cols(self, a, b):
        n = self._start("concat_cols", [a, b])
        self._require(self.shape(a)[0] == self.shape(b)[0], n, "row counts differ")
        return self._record(n)

    # ---------------------------------------------------------------- access
    def value(self, nid: NodeId) -> torch.Tensor:
        if not 0 <= nid.node < len(self._nodes):
            raise L.Error(f"Graph: node index {nid.node} out of range")
        n = self._nodes[nid.node]
        if not 0 <= nid.slot < len(n.shapes or n.out):
            raise L.Error(f"Graph::value: node {nid.node} has no slot {nid.slot}")
        t = n.out[nid.slot] if nid.slot < len(n.out) else None
        if t is None:
            raise L.Error(f"Graph::value: node {nid.node} slot {nid.slot} was released by the memory plan; rerun "
                          "forward() without the plan to inspect it")
        return t

    def shape(self, nid: NodeId):
        n = self._nodes[nid.node]
        shapes = n.shapes or [tuple(t.shape) for t in n.out]
        if not 0 <= nid.slot < len(shapes):
            raise L.Error("Graph::shape: bad slot")
        return shapes[nid.slot]

    def device_bytes(self) -> int:
        seen, tot = set(), 0
        for n in self._nodes:
            for t in n.out:
                if t is not None and t.data_ptr() not in seen:
                    seen.add(t.data_ptr())
                    tot += t.numel() * t.element_size()
        return tot

    def _track(self):
        self.peak_bytes = max(self.peak_bytes, self.device_bytes())

    # ---------------------------------------------------------------- forward
    def forward(self, bindings=()):
        for nid, m in bindings:
            n = self._nodes[nid.node]
            if n.op != "leaf":
                raise L.Error(f"Graph::forward: node {nid.node} is not a leaf and cannot be bound")
            t = self._mat(m)
            if tuple(t.shape) != n.shapes[0]:
                raise L.ShapeError(f"Graph::forward: binding for leaf '{n.name}' has shape "
                                   f"{t.shape[0]}x{t.shape[1]}, expected {n.shapes[0][0]}x{n.shapes[0][1]}")
            n.out[0] = t
        plan = self.build_plan() if self._use_plan else None
        # recompute in order; values of the previous pass are dropped as they are replaced
        self.peak_bytes = 0
        for i, n in enumerate(self._nodes):
            if n.op in ("leaf", "const"):
                continue
            n.out = [None] * len(n.shapes)
        self._track()
        for i, n in enumerate(self._nodes):
            if n.op in ("leaf", "const"):
                continue
            n.out = self._compute(n, plan[i] if plan is not None else None)
            self._track()

    def _base(self, n, k, claims, dst_slot):
        """dl/tape.hpp base_of: the donated buffer (released from its node) or a copy of input k."""
        if claims:
            for dst, sn, ss in claims:
                if dst == dst_slot:
                    t = self._nodes[sn].out[ss]
                    self._nodes[sn].out[ss] = None
                    return t
        src = self.value(n.inp[k])
        return self._k("COPY", src.shape[0], src.shape[1], src, self._empty(*src.shape))

    def _claimed(self, claims, dst_slot):
        return bool(claims) and any(c[0] == dst_slot for c in claims)

    def _compute(self, n, claims):
        op, v = n.op, self.value
        if op == "gemm2":
            a, b = v(n.inp[0]), v(n.inp[1])
            c = self._empty(a.shape[1] if n.ta else a.shape[0], b.shape[0] if n.tb else b.shape[1])
            return [L.gemm2_into(c, a, b, n.ta, n.tb, n.alpha)]
        if op == "syrk":
            a = v(n.inp[0])
            m = a.shape[1] if n.ta else a.shape[0]
            return [L.syrk_into(self._empty(m, m), a, n.ta, n.alpha)]
        if op in ("trmm", "trsm"):
            x = self._base(n, 1, claims, 0)
            f = L.trmm_inplace if op == "trmm" else L.trsm_inplace
            f(v(n.inp[0]), x, n.rightside, n.transpose, n.lower, n.alpha)
            return [x]
        if op == "potrf":
            x = self._base(n, 0, claims, 0)
            L.potrf_inplace(x, n.lower)
            return [x]
        if op == "potri":
            x = self._base(n, 0, claims, 0)
            L.potri_inplace(x, n.lower)
            return [x]
        if op == "gelqf":
            q = self._base(n, 0, claims, 0)
            l = self._empty(q.shape[0], q.shape[0])
            L.gelqf_inplace(q, l)
            return [q, l]
        if op == "syevd":
            u = self._base(n, 0, claims, 0)
            lam = self._empty(u.shape[0], 1)
            L.syevd_inplace(u, lam.view(-1))
            return [u, lam]
        if op == "gesvd":
            vv = self._base(n, 0, claims, 2)
            u = self._empty(vv.shape[0], vv.shape[0])
            lam = self._empty(vv.shape[0], 1)
            L.gesvd_inplace(vv, u, lam.view(-1))
            return [u, lam, vv]
        x = v(n.inp[0])
        r, c = x.shape
        if op in _UNARY_EW or op in _BINARY_EW or op in ("scale_const", "add_const", "mul_scalar", "div_scalar"):
            # in place on a donated buffer, else straight into a new one (same bits as base_of + in place)
            out = self._base(n, 0, claims, 0) if self._claimed(claims, 0) else self._empty(r, c)
            src = out if self._claimed(claims, 0) else x
            if op in _UNARY_EW:
                return [self._k(_UNARY_EW[op], r, c, src, out)]
            if op in _BINARY_EW:
                return [self._k(_BINARY_EW[op], r, c, src, out, y=v(n.inp[1]))]
            if op == "scale_const":
                return [self._k("SCALE", r, c, src, out, c=n.cval)]
            if op == "add_const":
                return [self._k("ADDC", r, c, src, out, c=n.cval)]
            return [self._k("MULS" if op == "mul_scalar" else "DIVS", r, c, src, out, s=v(n.inp[1]))]
        if op == "sum":
            return [self._k("SUM", r, c, x, self._empty(1, 1))]
        if op == "sum_rows":
            return [self._k("SUMROWS", r, c, x, self._empty(r, 1))]
        if op == "tile_cols":
            return [self._k("TILECOLS", r, 1, x, self._empty(r, n.count), aux=n.count)]
        if op == "tile_rows":
            return [self._k("TILEROWS", r, 1, x, self._empty(n.count, r), aux=n.count)]
        if op == "extract_diag":
            return [self._k("EXTRACTDIAG", r, c, x, self._empty(r, 1))]
        if op == "make_diag":
            return [self._k("MAKEDIAG", r, 1, x, self._empty(r, r))]
        if op == "concat_cols":
            y = v(n.inp[1])
            return [self._k("CONCATCOLS", r, c, x, self._empty(r, c + y.shape[1]), y=y, aux=y.shape[1])]
        raise L.Error(f"Graph: unknown op {op}")

    # ---------------------------------------------------------------- plan
    def build_plan(self):
        """dl/tape.hpp:1127-1209: per node, [(dst_slot, src_node, src_slot)] hand-offs."""
        nn = len(self._nodes)
        last_reader = [[-1] * len(n.shapes) for n in self._nodes]
        retained = [[False] * len(n.shapes) for n in self._nodes]
        if self._assume_backward:
            for i, n in enumerate(self._nodes):
                for s in range(len(n.shapes)):
                    retained[i][s] = backward_reads_output(n.op, s)
        for j, n in enumerate(self._nodes):
            for k, nid in enumerate(n.inp):
                last_reader[nid.node][nid.slot] = j
                if self._assume_backward and backward_reads_input(n.op, k):
                    retained[nid.node][nid.slot] = True
        donated = [[False] * len(n.shapes) for n in self._nodes]
        plan = [[] for _ in range(nn)]
        for j, n in enumerate(self._nodes):
            d = _donation(n.op)
            if d is None:
                continue
            dst_slot, src_input = d
            src = n.inp[src_input]
            p = self._nodes[src.node]
            if p.op in ("leaf", "const"):
                continue
            if retained[src.node][src.slot] or donated[src.node][src.slot]:
                continue
            if last_reader[src.node][src.slot] != j:
                continue
            if sum(1 for nid in n.inp if nid == src) != 1:
                continue
            if p.shapes[src.slot] != n.shapes[dst_slot]:
                continue
            donated[src.node][src.slot] = True
            plan[j].append((dst_slot, src.node, src.slot))
        return plan

    def planned_reuse_count(self) -> int:
        return sum(len(p) for p in self.build_plan())

    # ---------------------------------------------------------------- backward
    def backward(self, loss: NodeId) -> GradStore:
        if self.shape(loss) != (1, 1):
            raise L.ShapeError("Graph::backward: loss must be a 1x1 node")
        g = {}
        one = self._empty(1, 1)
        one.fill_(1.0)
        g[(loss.node, loss.slot)] = one
        for i in range(loss.node, -1, -1):
            n = self._nodes[i]
            if n.op in ("leaf", "const"):
                continue
            if not any(g.get((i, s)) is not None for s in range(len(n.shapes))):
                continue
            for s, sh in enumerate(n.shapes):
                if g.get((i, s)) is None:
                    g[(i, s)] = self._zeros(*sh)
            self._pull(i, n, g)
        return GradStore(g)

    def _acc(self, g, nid, m):
        """Graph::acc: take the first contribution, add the later ones in place."""
        key = (nid.node, nid.slot)
        cur = g.get(key)
        if cur is None:
            g[key] = m
        else:
            r, c = cur.shape
            self._k("COPY", r, c, m, cur, acc=True)

    def _acc_ew(self, g, nid, op, rows, cols, x, **kw):
        """Graph::acc of an elementwise pullback, computed straight into the gradient."""
        key = (nid.node, nid.slot)
        cur = g.get(key)
        if cur is None:
            sh = self.shape(nid)
            g[key] = self._k(op, rows, cols, x, self._empty(*sh), **kw)
        else:
            self._k(op, rows, cols, x, cur, acc=True, **kw)

    def _pull(self, i, n, g):
        op, v = n.op, self.value
        og = [g[(i, s)] for s in range(len(n.shapes))]
        me = lambda s: NodeId(i, s)  # noqa: E731
        if op == "gemm2":
            a, b = v(n.inp[0]), v(n.inp[1])
            abar, bbar = torch.empty_like(a), torch.empty_like(b)
            L.gemm2_backward_into(abar, bbar, og[0], a, b, n.ta, n.tb, n.alpha)
            self._acc(g, n.inp[0], abar)
            self._acc(g, n.inp[1], bbar)
        elif op == "syrk":
            a = v(n.inp[0])
            abar = torch.empty_like(a)
            L.syrk_backward_into(abar, og[0], a, n.ta, n.alpha)
            self._acc(g, n.inp[0], abar)
        elif op == "trmm":
            t, a = v(n.inp[0]), v(n.inp[1])
            abar, tbar = torch.empty_like(a), torch.empty_like(t)
            L.trmm_backward_into(abar, tbar, og[0], t, a, n.rightside, n.transpose, n.lower, n.alpha)
            self._acc(g, n.inp[0], tbar)
            self._acc(g, n.inp[1], abar)
        elif op == "trsm":
            t, b = v(n.inp[0]), v(me(0))
            abar, tbar = torch.empty_like(b), torch.empty_like(t)
            L.trsm_backward_into(abar, tbar, og[0], t, b, n.rightside, n.transpose, n.lower, n.alpha)
            self._acc(g, n.inp[0], tbar)
            self._acc(g, n.inp[1], abar)
        elif op == "potrf":
            l = v(me(0))
            abar = torch.empty_like(l)
            L.potrf_backward_into(abar, og[0], l, n.lower)
            self._acc(g, n.inp[0], abar)
        elif op == "potri":
            l, b = v(n.inp[0]), v(me(0))
            lbar = torch.empty_like(l)
            L.potri_backward_into(lbar, og[0], l, b, n.lower)
            self._acc(g, n.inp[0], lbar)
        elif op == "gelqf":
            q, l = v(me(0)), v(me(1))
            abar = torch.empty_like(q)
            L.gelqf_backward_into(abar, og[0], og[1], q, l)
            self._acc(g, n.inp[0], abar)
        elif op == "syevd":
            u, lam = v(me(0)), v(me(1))
            abar = torch.empty_like(u)
            L.syevd_backward_into(abar, og[0], og[1].view(-1), u, lam.view(-1))
            self._acc(g, n.inp[0], abar)
        elif op == "gesvd":
            u, lam, vv = v(me(0)), v(me(1)), v(me(2))
            abar = torch.empty_like(vv)
            L.gesvd_backward_into(abar, og[0], og[1].view(-1), og[2], u, lam.view(-1), vv)
            self._acc(g, n.inp[0], abar)
        else:
            self._pull_ew(i, n, g, og[0])

    def _pull_ew(self, i, n, g, go):
        op, v = n.op, self.value
        r, cc = go.shape
        x0 = n.inp[0]
        if op == "add":
            self._acc_ew(g, x0, "COPY", r, cc, go)
            self._acc_ew(g, n.inp[1], "COPY", r, cc, go)
        elif op == "sub":
            self._acc_ew(g, x0, "COPY", r, cc, go)
            self._acc_ew(g, n.inp[1], "NEG", r, cc, go)
        elif op == "mul":
            self._acc_ew(g, x0, "MUL", r, cc, go, y=v(n.inp[1]))
            self._acc_ew(g, n.inp[1], "MUL", r, cc, go, y=v(x0))
        elif op == "square":
            self._acc_ew(g, x0, "SQUARE_BWD", r, cc, go, y=v(x0))
        elif op == "sqrt":
            self._acc_ew(g, x0, "SQRT_BWD", r, cc, go, y=v(NodeId(i, 0)))
        elif op == "log":
            self._acc_ew(g, x0, "LOG_BWD", r, cc, go, y=v(x0))
        elif op == "exp":
            self._acc_ew(g, x0, "MUL", r, cc, go, y=v(NodeId(i, 0)))
        elif op == "abs":
            self._acc_ew(g, x0, "ABS_BWD", r, cc, go, y=v(x0))
        elif op == "neg":
            self._acc_ew(g, x0, "NEG", r, cc, go)
        elif op == "scale_const":
            self._acc_ew(g, x0, "SCALE", r, cc, go, c=n.cval)
        elif op == "add_const":
            self._acc_ew(g, x0, "COPY", r, cc, go)
        elif op == "mul_scalar":
            s = v(n.inp[1])
            self._acc_ew(g, x0, "MULS", r, cc, go, s=s)
            self._acc_ew(g, n.inp[1], "DOT", r, cc, go, y=v(x0))
        elif op == "div_scalar":
            s = v(n.inp[1])
            self._acc_ew(g, x0, "DIVS", r, cc, go, s=s)
            self._acc_ew(g, n.inp[1], "DOT_NEG_DIV", r, cc, go, y=v(NodeId(i, 0)), s=s)
        elif op == "sum":
            sr, sc = self.shape(x0)
            self._acc_ew(g, x0, "FILL", sr, sc, go, s=go)
        elif op == "sum_rows":
            sr, sc = self.shape(x0)
            self._acc_ew(g, x0, "TILECOLS", sr, 1, go, aux=sc)
        elif op == "tile_cols":
            self._acc_ew(g, x0, "SUMROWS", r, cc, go)
        elif op == "tile_rows":
            self._acc_ew(g, x0, "SUMCOLS", r, cc, go)
        elif op == "extract_diag":
            self._acc_ew(g, x0, "MAKEDIAG", r, 1, go)
        elif op == "make_diag":
            self._acc_ew(g, x0, "EXTRACTDIAG", r, cc, go)
        elif op == "tril_mask":
            self._acc_ew(g, x0, "TRIL", r, cc, go)
        elif op == "triu_mask":
            self._acc_ew(g, x0, "TRIU", r, cc, go)
        elif op == "concat_cols":
            ca = self.shape(x0)[1]
            cb = self.shape(n.inp[1])[1]
            self._acc_ew(g, x0, "SLICECOLS", r, ca, go, c=0.0, aux=cc)
            self._acc_ew(g, n.inp[1], "SLICECOLS", r, cb, go, c=float(ca), aux=cc)
        else:
            raise L.Error(f"Graph: no pullback for {op}")

    # ---------------------------------------------------------------- debug
    def dump(self) -> str:
        lines = [f"graph({len(self._nodes)} nodes)"]
        for i, n in enumerate(self._nodes):
            s = f"#{i} {n.op}"
            if n.op in ("leaf", "const"):
                s += f' "{n.name}"'
            else:
                s += "(" + ", ".join(f"#{p.node}" + (f".{p.slot}" if p.slot else "") for p in n.inp) + ")"
            s += "".join(f" [{a}x{b}]" for a, b in n.shapes)
            lines.append(s)
        return "\n".join(lines)


# ------------------------------------------------------------ model builders
LOG_2PI = 1.8378770664093454835606594728112353


def rbf_kernel(g: Graph, x1, x2, sigma2, ell2):
    """dl/models.hpp:46-62 on the device tape."""
    sh1, sh2 = g.shape(x1), g.shape(x2)
    if sh1[1] != sh2[1]:
        raise L.ShapeError("rbf_kernel: feature dimensions differ")
    same = x1 == x2
    gram = g.syrk(x1, False) if same else g.gemm2(x1, x2, False, True)
    s1 = g.sum_rows(g.square(x1))
    s2 = s1 if same else g.sum_rows(g.square(x2))
    dist = g.sub(g.add(g.tile_cols(s1, sh2[0]), g.tile_rows(s2, sh1[0])), g.scale_const(gram, 2.0))
    return g.mul_scalar(g.exp(g.neg(g.div_scalar(dist, g.scale_const(ell2, 2.0)))), sigma2)


def gp_nll_from_kernel(g: Graph, kernel, y, lam):
    """dl/models.hpp:88-100."""
    n = g.shape(kernel)[0]
    a = g.add(kernel, g.mul_scalar(g.constant(torch.eye(n, dtype=g.dtype), "I"), lam))
    l = g.potrf(a)
    z = g.trsm(l, y, False, False, True)
    quad = g.scale_const(g.sum(g.square(z)), 0.5)
    logdet = g.sum(g.log(g.extract_diag(l)))
    return g.add_const(g.add(quad, logdet), 0.5 * n * LOG_2PI)


def make_gp(g: Graph, x, y, sigma2, ell2, lam):
    """dl/models.hpp:115-135: returns a dict of the model's NodeIds."""
    import math
    x = torch.as_tensor(x)
    y = torch.as_tensor(y)
    if y.dim() != 2 or y.shape[1] != 1 or y.shape[0] != x.shape[0]:
        raise L.ShapeError("make_gp: y must be a column with one entry per row of x")
    for val, nm in ((sigma2, "sigma2"), (ell2, "ell2"), (lam, "lam")):
        if not (val > 0 and math.isfinite(val)):
            raise L.Error(f"make_gp: {nm} must be positive and finite")
    m = {"x": g.leaf(x, "x"), "y": g.leaf(y, "y"), "log_sigma2": g.leaf([[math.log(sigma2)]], "log_sigma2"),
         "log_ell2": g.leaf([[math.log(ell2)]], "log_ell2"), "log_lam": g.leaf([[math.log(lam)]], "log_lam")}
    m["sigma2"] = g.exp(m["log_sigma2"])
    m["ell2"] = g.exp(m["log_ell2"])
    m["lam"] = g.exp(m["log_lam"])
    m["kernel"] = rbf_kernel(g, m["x"], m["x"], m["sigma2"], m["ell2"])
    m["loss"] = gp_nll_from_kernel(g, m["kernel"], m["y"], m["lam"])
    return m


def build_kalman_nll(g: Graph, a, b, sh, sv, mu0, s0, obs):
    """dl/models.hpp:285-337 on the device tape: returns (nll, mu_filt, s_filt)."""
    if not obs:
        raise L.ShapeError("build_kalman_nll: no observations")
    h, d = g.shape(a)[0], g.shape(b)[0]
    if (g.shape(a) != (h, h) or g.shape(b)[1] != h or g.shape(sh) != (h, h) or g.shape(sv) != (d, d)
            or g.shape(mu0) != (h, 1) or g.shape(s0) != (h, h)):
        raise L.ShapeError("build_kalman_nll: inconsistent system shapes")
    for v in obs:
        if g.shape(v) != (d, 1):
            raise L.ShapeError("build_kalman_nll: observations must be d x 1")
    eye_h = g.constant(torch.eye(h, dtype=g.dtype), "I_h")
    mu_pred, s_pred, nll = mu0, s0, None
    mu_f_all, s_f_all = [], []
    for t, v in enumerate(obs):
        svv = g.add(g.gemm2(g.gemm2(b, s_pred), b, False, True), sv)
        lvv = g.potrf(svv)
        e = g.sub(v, g.gemm2(b, mu_pred))
        z = g.trsm(lvv, e, False, False, True)
        term = g.add_const(g.add(g.scale_const(g.sum(g.square(z)), 0.5), g.sum(g.log(g.extract_diag(lvv)))),
                           0.5 * d * LOG_2PI)
        nll = term if t == 0 else g.add(nll, term)
        xbt = g.gemm2(s_pred, b, False, True)
        gain = g.trsm(lvv, g.trsm(lvv, xbt, True, True, True), True, False, True)
        mu_f = g.add(mu_pred, g.gemm2(gain, e))
        ikb = g.sub(eye_h, g.gemm2(gain, b))
        s_f = g.add(g.gemm2(g.gemm2(ikb, s_pred), ikb, False, True), g.gemm2(g.gemm2(gain, sv), gain, False, True))
        mu_f_all.append(mu_f)
        s_f_all.append(s_f)
        if t + 1 < len(obs):
            mu_pred = g.gemm2(a, mu_f)
            s_pred = g.add(g.gemm2(g.gemm2(a, s_f), a, False, True), sh)
    return nll, mu_f_all, s_f_all
