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


# ---- tile pairs (csrc/pair.cuh): whole square matrices read plain and
# transposed; each CTA stages blocks (I,J) and (J,I) of every distinct buffer
# once by 2-D TMA.  Edge sizes: exactly one tile, a ragged last tile, the
# smallest eligible size, and shapes that fall back to the per-slot path.

@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("n", [32, 36, 64, 100, 2052])
def test_pair_expr1_edges(ctx, n, etype):
    X, Y, x, y = _pair(ctx, (n, n), etype, 3)
    Z = fm.zeros(n, n, etype, ctx)
    Z.assign(2 * (X.t() + Y) + 2 * (X + Y.t()))
    t = x.dtype.type(2)
    assert np.array_equal(Z.to_numpy(), t * (x.T + y) + t * (x + y.T))


@pytest.mark.parametrize("n", [33, 31, 34])
def test_pair_ineligible_sizes_fall_back(ctx, n):
    """n*4 not a 16-byte multiple (TMA strides) or below one tile."""
    X, Y, x, y = _pair(ctx, (n, n), "f32", 4)
    Z = fm.zeros(n, n, ctx=ctx)
    Z.assign(X.t() - Y * X)
    assert np.array_equal(Z.to_numpy(), x.T - y * x)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_pair_expr2(ctx, etype):
    """Paper expr2: a*A + (B + C).t() + log(D**2) -- four buffers, two transposed."""
    n = 1000
    ms = [fm.randu(n, n, 70 + i, etype, ctx) for i in range(4)]
    a, b, c, d = ms
    Z = fm.zeros(n, n, etype, ctx)
    Z.assign(0.5 * a + (b + c).t() + fm.log(d ** 2))
    av, bv, cv, dv = (m.to_numpy() for m in ms)
    T = av.dtype.type
    lg = np.log((dv * dv).astype(np.float64))
    want = (T(0.5) * av + (bv + cv).T) + (lg.astype(av.dtype) if etype == "f32" else lg)
    if etype == "f32":       # f32 log correctly rounded (via f64): <= 1 ulp
        assert orc.max_ulp(Z.to_numpy(), want) <= 1
    else:                    # f64 transcendentals: 1e-12 relative (DESIGN.md numerics),
        z = Z.to_numpy()     # against max(|want|, 1): the sum can cancel to ~0
        assert np.max(np.abs(z - want) / np.maximum(np.abs(want), 1.0)) <= 1e-12


def test_pair_transposed_only_and_self(ctx):
    """X.t() alone, X.t() * X (one buffer, both blocks), X.t() % X.t()."""
    n = 640
    X = fm.randu(n, n, 81, "f32", ctx)
    x = X.to_numpy()
    Z = fm.zeros(n, n, ctx=ctx)
    Z.assign(X.t() + 0.0)
    assert np.array_equal(Z.to_numpy(), x.T + np.float32(0))
    Z.assign(X.t() % X - X)
    assert np.array_equal(Z.to_numpy(), x.T * x - x)
    Z.assign(X.t() % X.t())
    assert np.array_equal(Z.to_numpy(), x.T * x.T)


def test_pair_mixed_widths(ctx):
    """f64 program with an f32 and a u32 leaf (4- and 8-byte tiles in one stage)."""
    n = 520
    A = fm.randu(n, n, 90, "f64", ctx)
    B = fm.randu(n, n, 91, "f32", ctx)
    U = fm.randi(n, n, 7, 92, "u32", ctx)
    Z = fm.zeros(n, n, "f64", ctx)
    Z.assign(A.t() * fm.conv_to(B, "f64") + fm.conv_to(U.t(), "f64") - A)
    a, b, u = A.to_numpy(), B.to_numpy(), U.to_numpy()
    want = (a.T * b.astype(np.float64) + u.T.astype(np.float64)) - a
    assert np.array_equal(Z.to_numpy(), want)


def test_pair_many_buffers_falls_back(ctx):
    """More distinct buffers than the pair kernel stages (8): per-slot path."""
    n = 256
    ms = [fm.randu(n, n, 100 + i, "f32", ctx) for i in range(10)]
    e = ms[0].t()
    for m in ms[1:]:
        e = e + m
    Z = fm.zeros(n, n, ctx=ctx)
    Z.assign(e)
    want = ms[0].to_numpy().T
    for m in ms[1:]:
        want = want + m.to_numpy()
    assert np.array_equal(Z.to_numpy(), want)


def test_pair_result_into_u32_and_graph_replay(ctx):
    """Integer program on the pair path, captured in a CUDA graph and replayed."""
    n = 300
    U = fm.randi(n, n, 1000, 5, "u32", ctx)
    V = fm.randi(n, n, 1000, 6, "u32", ctx)
    Z = fm.zeros(n, n, "u32", ctx)
    g = fm.capture(lambda: Z.assign(U.t() + V * U), ctx)
    Z.assign(U * 0)
    g.replay()
    g.replay()
    ctx.sync()
    u, v = U.to_numpy(), V.to_numpy()
    assert np.array_equal(Z.to_numpy(), u.T + v * u)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_pair_in_place(ctx, etype):
    """Z = Z + Y.t() (a SAFE alias: every block of Z is read and written by the one CTA that owns its pair)."""
    n = 1000
    Z = fm.randu(n, n, 11, etype, ctx)
    Y = fm.randu(n, n, 12, etype, ctx)
    z, y = Z.to_numpy(), Y.to_numpy()
    Z.assign(Z + Y.t())
    assert np.array_equal(Z.to_numpy(), z + y.T)
