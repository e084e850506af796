"""The tiled, shared-memory staged VM copy (csrc/tiled.cuh): transposed
leaves, views at unaligned offsets, diagonals, many-leaf flat chains and
mixed element types, at sizes large enough to take that path (>= 4096
elements) with ragged edge tiles.  Expected values come from numpy with the
same per-op f32/f64 rounding (no FMA), so chains of + - * / scalars are
compared bit for bit; transcendentals at <= 1 ulp of the correctly-rounded
restatement (DESIGN.md numerics policy)."""

import numpy as np
import pytest

import paper_2604_22242_b200 as fm
from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu

SQUARE = [(300, 300), (1000, 1000), (4099, 4099)]
RECT = [(300, 257), (4097, 3), (64, 4096), (1023, 1025)]


@pytest.fixture
def ctx(gpu_ctx):
    return fm.Context(gpu_ctx.backend)


def _pair(ctx, shape, etype, s=1):
    X = fm.randu(*shape, 40 + s, etype, ctx)
    Y = fm.randu(*shape, 50 + s, etype, ctx)
    return X, Y, X.to_numpy(), Y.to_numpy()


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("shape", SQUARE)
def test_transposed_leaves_expr1(ctx, shape, etype):
    """Paper expr1: 2*(X.t() + Y) + 2*(X + Y.t()) (reference bench.py:135-138)."""
    X, Y, x, y = _pair(ctx, shape, etype)
    Z = fm.zeros(*shape, etype, ctx)
    ctx.reset_counters()
    Z.assign(2 * (X.t() + Y) + 2 * (X + Y.t()))
    assert ctx.launches == 1
    t = x.dtype.type(2)
    want = t * (x.T + y) + t * (x + y.T)
    assert np.array_equal(Z.to_numpy(), want)


@pytest.mark.parametrize("shape", RECT)
def test_transpose_of_rectangular(ctx, shape):
    X = fm.randu(shape[1], shape[0], 7, "f32", ctx)
    Y = fm.randu(*shape, 8, "f32", ctx)
    Z = fm.zeros(*shape, ctx=ctx)
    Z.assign(X.t() * Y - 0.5)
    x, y = X.to_numpy(), Y.to_numpy()
    assert np.array_equal(Z.to_numpy(), x.T * y + np.float32(-0.5))


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_unaligned_subviews(ctx, etype):
    """Views at odd offsets (no 16-byte alignment): the element-copy staging."""
    X, Y, x, y = _pair(ctx, (1001, 777), etype, 2)
    Z = fm.zeros(500, 300, etype, ctx)
    Z.assign(X.submat(3, 5, 500, 300) * Y.submat(101, 7, 500, 300) + X.submat(0, 1, 500, 300))
    want = x[3:503, 5:305] * y[101:601, 7:307] + x[0:500, 1:301]
    assert np.array_equal(Z.to_numpy(), want)


@pytest.mark.parametrize("n", [8192, 10000])
def test_center_half_views(ctx, n):
    """Paper addsub4: center_half views of four matrices."""
    ms = [fm.randu(n, n, 60 + i, "f32", ctx) for i in range(4)]
    Z = fm.zeros(n // 2, n // 2, ctx=ctx)
    e = ms[0].center_half() + ms[1].center_half()
    e = e + ms[2].center_half()
    e = e + ms[3].center_half()
    Z.assign(e)
    q, h = n // 4, n // 2
    a = [m.to_numpy()[q:q + h, q:q + h] for m in ms]
    assert np.array_equal(Z.to_numpy(), ((a[0] + a[1]) + a[2]) + a[3])


def test_transposed_subview(ctx):
    X = fm.randu(700, 900, 3, "f64", ctx)
    Y = fm.randu(400, 300, 4, "f64", ctx)
    Z = fm.zeros(400, 300, "f64", ctx)
    Z.assign(fm.trans(X.submat(11, 13, 300, 400)) - Y)
    x = X.to_numpy()
    assert np.array_equal(Z.to_numpy(), x[11:311, 13:413].T - Y.to_numpy())


def test_diagonals_with_staged_leaves(ctx):
    """Paper diagsum plus a staged dense leaf in the same program."""
    n = 5000
    X, Y, x, y = _pair(ctx, (n, n), "f32", 3)
    W = fm.randu(n - 1, 1, 9, "f32", ctx)
    Z = fm.zeros(n - 1, 1, ctx=ctx)
    Z.assign((X.diag(-1) + X.diag(1)) * (Y.diag(-1) + Y.diag(1)) + W)
    dx = np.diagonal(x, -1) + np.diagonal(x, 1)
    dy = np.diagonal(y, -1) + np.diagonal(y, 1)
    assert np.array_equal(Z.to_numpy().ravel(), dx * dy + W.to_numpy().ravel())


@pytest.mark.parametrize("k", [5, 8, 16, 32])
def test_add_n_many_leaves(ctx, k):
    """The add-N sweep (reference bench.py:307-326): one launch for any N."""
    shape = (1500, 1001)
    ms = [fm.randu(*shape, 100 + i, "f32", ctx) for i in range(k)]
    e = ms[0] + ms[1]
    for m in ms[2:]:
        e = e + m
    Z = fm.zeros(*shape, ctx=ctx)
    ctx.reset_counters()
    Z.assign(e)
    assert ctx.launches == 1
    want = ms[0].to_numpy() + ms[1].to_numpy()
    for m in ms[2:]:
        want = want + m.to_numpy()
    assert np.array_equal(Z.to_numpy(), want)


def test_mixed_types_expr3(ctx):
    """Paper expr3: 1 / (x * conv_to(u, f32) + log(log(x + 2) * w)) with a u32 leaf."""
    n = 3000
    x = fm.randu(n, n, 1, "f32", ctx)
    u = fm.randi(n, n, 10, 2, "u32", ctx)
    w = fm.randu(n, n, 3, "f32", ctx)
    Z = fm.zeros(n, n, ctx=ctx)
    Z.assign(1 / (x * fm.conv_to(u, "f32") + fm.log(fm.log(x + 2) * w)))
    xv, uv, wv = x.to_numpy(), u.to_numpy(), w.to_numpy()
    f = np.float32

    def crlog(a):
        return np.log(a.astype(np.float64)).astype(np.float32)
    want = f(1) / (xv * uv.astype(np.float32) + crlog(crlog(xv + f(2)) * wv))
    assert orc.max_ulp(Z.to_numpy(), want) <= 1


def test_bf16_transposed_leaf(ctx):
    X = fm.randu(600, 500, 5, "bf16", ctx)
    Y = fm.randu(500, 600, 6, "f32", ctx)
    Z = fm.zeros(500, 600, ctx=ctx)
    Z.assign(fm.conv_to(X.t(), "f32") + Y)
    want = X.to_numpy().astype(np.float32).T + Y.to_numpy()
    assert np.array_equal(Z.to_numpy(), want)
