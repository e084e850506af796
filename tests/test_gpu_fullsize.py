"""The BASELINE configs at their full bench sizes, checked through the
oracle on EVERY element (C1, C3, C4: column blocks copied out with a fused
subview copy and compared on the host) and through size-independent
properties:

* C2: dot / accu / norm of 1e8-element f32 and f64 vectors vs the exactly
  rounded f64 sum (rel 1e-12), accu(x % y) == dot(x, y) bit for bit (same
  fused kernel), accu(x - x) == 0, accu(x + x) == 2 accu(x) at 1e-14;
* C3: 32768^2 f32 chain, sampled columns at 0 ulp vs the correctly-rounded
  restatement;
* C4: 65536 x 16384 f64 column stats, sampled columns: index_max exact,
  max exact, sum / mean at 1e-13;
* the typed column-stats fast path with NaNs and ties placed across warp
  tiles, and empty / degenerate shapes.
Sampled columns are copied out with a fused subview copy so only they cross
PCIe."""

import numpy as np
import pytest

import paper_2604_22242_b200 as fm
from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture
def ctx(gpu_ctx):
    return fm.Context(gpu_ctx.backend)


def _columns(M, cols):
    """Columns `cols` of a device matrix, copied out through a fused view copy."""
    out = []
    for j in cols:
        c = fm.Mat(M.n_rows, 1, M.etype, M.ctx)
        c.assign(M.col(int(j)))
        out.append(c.to_numpy())
    return np.concatenate(out, axis=1)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_c2_full_size(ctx, etype):
    n = 100_000_000
    x, y = fm.Col(n, etype, ctx), fm.Col(n, etype, ctx)
    ctx.backend.randu(x.handle, 42)
    ctx.backend.randu(y.handle, 43)
    ety = fm.ElemType.of(etype)
    xh, yh = orc.uniform_fill(42, n, etype), orc.uniform_fill(43, n, etype)
    want_dot = orc.accu(xh * yh, ety)
    d = xh - yh
    want_norm = float(np.sqrt(orc.accu(d * d, ety)))
    got_dot = fm.dot(x, y)
    assert abs(got_dot - want_dot) <= 1e-12 * abs(want_dot)
    assert fm.accu(x % y) == got_dot
    got_norm = fm.norm(x - y)
    assert abs(got_norm - want_norm) <= 1e-12 * want_norm
    assert fm.accu(x - x) == 0.0
    # linearity; the two launches may differ in summation grid, so not bit-exact
    assert fm.accu(x + x) == pytest.approx(2.0 * fm.accu(x), rel=1e-14)


def test_c3_full_size_sampled(ctx):
    n = 32768
    X, Y = fm.randu(n, n, 42, "f32", ctx), fm.randu(n, n, 43, "f32", ctx)
    Z = fm.Mat(n, n, "f32", ctx)
    ctx.reset_counters()
    Z.assign(fm.exp(-fm.square(X - Y) / 2) + 0.5 * fm.abs(X))
    assert ctx.launches == 1
    cols = [0, 1, 4095, 16384, n - 1]
    x, y, z = _columns(X, cols), _columns(Y, cols), _columns(Z, cols)
    for i, j in enumerate(cols):     # device randu == the reference stream at that column's offset
        assert np.array_equal(x[:, i], orc.uniform_fill(42, n, "f32", offset=j * n))
    d = x - y
    want = (np.exp((np.float32(0.5) * -(d * d)).astype(np.float64)).astype(np.float32)
            + np.float32(0.5) * np.abs(x))
    assert orc.max_ulp(z, want) == 0


def test_c4_full_size_sampled(ctx):
    r, c = 65536, 16384
    X, Y, Z = (fm.randu(r, c, s, "f64", ctx) for s in (42, 43, 44))
    e = (X - Y) % Z
    outs = [fm.Mat(1, c, "f64", ctx), fm.Mat(1, c, "f64", ctx), fm.Mat(1, c, "f64", ctx), fm.Mat(1, c, "u32", ctx)]
    ctx.reset_counters()
    fm.assign_all([(outs[0], fm.sum(e, 0)), (outs[1], fm.mean(e, 0)), (outs[2], fm.max(e, 0)),
                   (outs[3], fm.index_max(e, 0))])
    assert ctx.launches == 1
    cols = [0, 1, 777, 8191, c - 1]
    v = (_columns(X, cols) - _columns(Y, cols)) * _columns(Z, cols)
    k, f64 = orc.ReduceKind, fm.ElemType.f64
    got = [o.to_numpy()[:, cols] for o in outs]
    assert orc.compare(got[0], orc.reduce_dim(k.sum, 0, v, f64)) < 1e-13
    assert orc.compare(got[1], orc.reduce_dim(k.mean, 0, v, f64)) < 1e-13
    assert np.array_equal(got[2], orc.reduce_dim(k.max, 0, v, f64))
    assert np.array_equal(got[3], orc.reduce_dim(k.index_max, 0, v, f64))


@pytest.mark.parametrize("rows", [4096 + 24, 4096])
@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_column_stats_fast_path_nan_and_ties(ctx, etype, rows):
    """Ties and NaNs at rows owned by different warps / tiles of the typed
    fast path (tiles of 32*V rows), with a ragged remainder (general kernel
    finishing the column) and without one (the typed-only kernel)."""
    cols = 9
    rng = np.random.default_rng(5)
    a = rng.integers(-3, 4, size=(rows, cols)).astype(np.float32 if etype == "f32" else np.float64)
    a[:, 1] = 7.0                      # all equal: index 0 wins
    a[3000, 2] = 50.0
    a[100, 2] = 50.0                   # tie across tiles: first index (100)
    a[2500, 3] = np.nan
    a[rows - 1, 3] = np.nan            # first NaN wins max / index_max (2500)
    a[rows - 1, 4] = 99.0              # maximum in the last rows
    a[:, 5] = -np.inf
    a[17, 6] = np.inf
    X = fm.from_array(a, ctx=ctx)
    ety = fm.ElemType.of(etype)
    for fn, kind in ((fm.max, orc.ReduceKind.max), (fm.index_max, orc.ReduceKind.index_max),
                     (fm.min, orc.ReduceKind.min), (fm.index_min, orc.ReduceKind.index_min),
                     (fm.sum, orc.ReduceKind.sum)):
        got = fn(X, 0).eval().to_numpy()
        want = orc.reduce_dim(kind, 0, a, ety)
        assert np.array_equal(got, want, equal_nan=True), (fn.__name__, got, want)


def test_empty_and_degenerate(ctx):
    E = fm.zeros(0, 5, ctx=ctx)
    assert fm.accu(E) == 0.0
    Z = fm.zeros(0, 5, ctx=ctx)
    Z.assign(E + E)
    assert Z.to_numpy().shape == (0, 5)
    s = fm.sum(E, 0).eval().to_numpy()
    assert s.shape == (1, 5) and not s.any()
    one = fm.fill(1, 1, 3.5, ctx=ctx)
    assert fm.accu(one * one) == 12.25
    v = fm.randu(1, 100_003, 1, "f64", ctx)          # a row vector: ragged, flat
    assert fm.accu(v) == pytest.approx(orc.accu(orc.randu(1, 100_003, 1, "f64"), fm.ElemType.f64), rel=1e-13)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_bulk_staged_copy_beyond_l2(ctx, etype):
    """A light chain whose working set (>= 512 MiB) takes the TMA-bulk-staged
    copy with dynamically claimed chunks, with a ragged tail (< one chunk)."""
    n_rows, n_cols = 8191, 8193 if etype == "f32" else 6001
    X, Y = fm.randu(n_rows, n_cols, 5, etype, ctx), fm.randu(n_rows, n_cols, 6, etype, ctx)
    Z = fm.Mat(n_rows, n_cols, etype, ctx)
    for _ in range(2):                       # the chunk counter resets between launches
        Z.assign(2 * (X % Y) + X)
    x, y = X.to_numpy(), Y.to_numpy()
    t = x.dtype.type(2)
    assert np.array_equal(Z.to_numpy(), t * (x * y) + x)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_row_stats_fast_path_nan_and_ties(ctx, etype):
    """dim-1 reductions on the typed fast path (whole V-row runs, columns in
    increasing order within each column split, splits combined in order):
    ties and NaNs placed in different splits, plus a ragged last row run."""
    rows, cols = 64 + 2, 5000
    rng = np.random.default_rng(7)
    a = rng.integers(-3, 4, size=(rows, cols)).astype(np.float32 if etype == "f32" else np.float64)
    a[1, :] = 7.0                      # all equal: column 0 wins
    a[2, 4000] = 50.0
    a[2, 100] = 50.0                   # tie across splits: first column (100)
    a[3, 2500] = np.nan
    a[3, 4100] = np.nan                # first NaN wins
    a[65, 4999] = 99.0                 # the ragged row run
    a[5, :] = -np.inf
    X = fm.from_array(a, ctx=ctx)
    ety = fm.ElemType.of(etype)
    for fn, kind in ((fm.max, orc.ReduceKind.max), (fm.index_max, orc.ReduceKind.index_max),
                     (fm.min, orc.ReduceKind.min), (fm.index_min, orc.ReduceKind.index_min)):
        got = fn(X, 1).eval().to_numpy()
        want = orc.reduce_dim(kind, 1, a, ety)
        assert np.array_equal(got, want, equal_nan=True), (fn.__name__,)
    got = fm.sum(X, 1).eval().to_numpy()
    assert orc.compare(got, orc.reduce_dim(orc.ReduceKind.sum, 1, a, ety)) < 1e-12


def _block(M, j0, w):
    """Columns j0..j0+w-1 of a device matrix (one fused subview copy)."""
    b = fm.Mat(M.n_rows, w, M.etype, M.ctx)
    b.assign(M.submat(0, j0, M.n_rows, w))
    return b.to_numpy()


def test_c3_full_size_every_column(ctx):
    """C3 at 32768^2: EVERY element vs the correctly-rounded restatement
    (0 ulp), in 2048-column blocks; the inputs' blocks are re-checked against
    the reference splitmix64 stream at their offsets."""
    n, w = 32768, 2048
    X, Y = fm.randu(n, n, 42, "f32", ctx), fm.randu(n, n, 43, "f32", ctx)
    Z = fm.Mat(n, n, "f32", ctx)
    Z.assign(fm.exp(-fm.square(X - Y) / 2) + 0.5 * fm.abs(X))
    for j0 in range(0, n, w):
        x, y, z = _block(X, j0, w), _block(Y, j0, w), _block(Z, j0, w)
        if j0 in (0, n - w):
            assert np.array_equal(x.ravel(order="F"), orc.uniform_fill(42, n * w, "f32", offset=j0 * n))
        d = x - y
        want = (np.exp((np.float32(0.5) * -(d * d)).astype(np.float64)).astype(np.float32)
                + np.float32(0.5) * np.abs(x))
        assert orc.max_ulp(z, want) == 0, j0


def test_c4_full_size_every_column(ctx):
    """C4 at 65536 x 16384 f64: every column's sum / mean (within 1e-13 of
    sum |v|), max and index_max (exact) vs the oracle, in 1024-column blocks."""
    r, c, w = 65536, 16384, 1024
    X, Y, Z = (fm.randu(r, c, s, "f64", ctx) for s in (42, 43, 44))
    e = (X - Y) % Z
    outs = [fm.Mat(1, c, "f64", ctx), fm.Mat(1, c, "f64", ctx), fm.Mat(1, c, "f64", ctx), fm.Mat(1, c, "u32", ctx)]
    fm.assign_all([(outs[0], fm.sum(e, 0)), (outs[1], fm.mean(e, 0)), (outs[2], fm.max(e, 0)),
                   (outs[3], fm.index_max(e, 0))])
    got = [o.to_numpy() for o in outs]
    k, f64 = orc.ReduceKind, fm.ElemType.f64
    for j0 in range(0, c, w):
        v = (_block(X, j0, w) - _block(Y, j0, w)) * _block(Z, j0, w)
        sl = slice(j0, j0 + w)
        # sums of mixed-sign terms can cancel towards 0: bound the error by
        # the condition of the sum, 1e-13 * sum |v| per column
        scale = np.abs(v).sum(axis=0, keepdims=True)
        for o, kind, div in ((0, k.sum, 1.0), (1, k.mean, float(r))):
            err = np.abs(got[o][:, sl] - orc.reduce_dim(kind, 0, v, f64))
            assert np.all(err <= 1e-13 * scale / div), (j0, float((err / (scale / div)).max()))
        assert np.array_equal(got[2][:, sl], orc.reduce_dim(k.max, 0, v, f64)), j0
        assert np.array_equal(got[3][:, sl], orc.reduce_dim(k.index_max, 0, v, f64)), j0


def test_c1_full_size_bit_exact(ctx):
    """C1 at 4096^2: the whole output bit-exact vs the oracle (the reference's
    own generated C is 0-ulp against it, tests/test_oracle.py)."""
    n = 4096
    X, Y = fm.randu(n, n, 42, "f32", ctx), fm.randu(n, n, 43, "f32", ctx)
    Z = fm.Mat(n, n, "f32", ctx)
    Z.assign(2 * (X % Y) + X)
    x, y = orc.randu(n, n, 42), orc.randu(n, n, 43)
    assert np.array_equal(Z.to_numpy(), np.float32(2) * (x * y) + x)
