"""Special values (NaN, +-inf, -0.0) through the large-size kernels: the
TMA-staged column / row reduction paths, the bulk-staged full reductions and
the tile-pair copy only run at sizes the small-shape tests never reach.
Gates: max / min / index_* bit-exact with the oracle's numpy semantics
(NaN propagates, the first NaN wins the index; oracle/fm_oracle.py:246-269);
sum / mean equal in their NaN / inf pattern and within 1e-12 elsewhere; full
reductions NaN when any NaN or both infinities are present."""

import numpy as np
import pytest

import paper_2604_22242_b200 as fm
from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu

ROWS, COLS = 8192, 1024


def _specials(shape, dtype, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(shape).astype(dtype)
    flat = a.reshape(-1, order="F")
    n = flat.size
    idx = rng.choice(n, size=n // 5000, replace=False)
    k = len(idx) // 4
    flat[idx[:k]] = np.nan
    flat[idx[k:2 * k]] = np.inf
    flat[idx[2 * k:3 * k]] = -np.inf
    flat[idx[3 * k:]] = -0.0
    # whole special columns / rows: all-NaN, all -inf, a column with +inf and -inf
    a[:, 3] = np.nan
    a[:, 7] = -np.inf
    a[5, 11], a[9, 11] = np.inf, -np.inf
    a[17, :] = np.nan
    return np.asfortranarray(a)


def _same_float(got, want, rtol=1e-12):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    fin = np.isfinite(want)
    assert np.array_equal(got[~fin & ~np.isnan(want)], want[~fin & ~np.isnan(want)])
    np.testing.assert_allclose(got[fin], want[fin], rtol=rtol, atol=1e-9)


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("dim", [0, 1])
@pytest.mark.parametrize("fused", [False, True])
def test_dim_reductions_with_special_values(gpu_ctx, etype, dim, fused):
    dt = np.float32 if etype == "f32" else np.float64
    ety = fm.ElemType.of(etype)
    a = _specials((ROWS, COLS), dt, 1 + dim)
    X = fm.from_array(a, ctx=gpu_ctx)
    if fused:                                   # (X - Y) % Z: the C4 template path
        b = np.asfortranarray(np.random.default_rng(5).standard_normal((ROWS, COLS)).astype(dt))
        c = np.asfortranarray(np.random.default_rng(6).standard_normal((ROWS, COLS)).astype(dt))
        Y, Z = fm.from_array(b, ctx=gpu_ctx), fm.from_array(c, ctx=gpu_ctx)
        e = (X - Y) % Z
        v = ((a - b) * c).astype(dt)
    else:
        e, v = X, a
    K = orc.ReduceKind
    for fn, kind in ((fm.max, K.max), (fm.min, K.min), (fm.index_max, K.index_max), (fm.index_min, K.index_min)):
        got = fn(e, dim).eval().to_numpy()
        want = orc.reduce_dim(kind, dim, v, ety)
        if kind in (K.max, K.min):
            assert np.array_equal(np.isnan(got), np.isnan(want)), (fn.__name__, dim)
            ok = ~np.isnan(want)
            assert np.array_equal(got[ok], want[ok]), (fn.__name__, dim)   # -0.0 == 0.0: either zero may win
        else:
            assert np.array_equal(got, want), (fn.__name__, dim)
    for fn, kind in ((fm.sum, K.sum), (fm.mean, K.mean)):
        with np.errstate(invalid="ignore"):
            want = orc.reduce_dim(kind, dim, v, ety)
        _same_float(fn(e, dim).eval().to_numpy(), want, 1e-12 if etype == "f64" else 1e-6)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_full_reductions_with_special_values(gpu_ctx, etype):
    dt = np.float32 if etype == "f32" else np.float64
    n = 1 << 24                                          # bulk-staged accu path
    rng = np.random.default_rng(11)
    base = rng.standard_normal(n).astype(dt)

    def accu_of(vals):
        return fm.accu(fm.from_array(vals.reshape(-1, 1), ctx=gpu_ctx))

    v = base.copy()
    v[n // 3] = np.nan
    assert np.isnan(accu_of(v))
    v = base.copy()
    v[123], v[n - 5] = np.inf, -np.inf
    assert np.isnan(accu_of(v))
    v = base.copy()
    v[77] = np.inf
    assert accu_of(v) == np.inf
    v = base.copy()
    v[::2] = -0.0
    want = orc.accu(v, fm.ElemType.of(etype))
    assert abs(accu_of(v) - want) <= 1e-12 * np.abs(v.astype(np.float64)).sum()
    # dot / norm over specials
    x = fm.from_array(base.reshape(-1, 1), ctx=gpu_ctx)
    w = base.copy()
    w[999] = np.nan
    y = fm.from_array(w.reshape(-1, 1), ctx=gpu_ctx)
    assert np.isnan(fm.dot(x, y)) and np.isnan(fm.norm(x - y))


def test_transposed_copy_with_special_values(gpu_ctx):
    """The tile-pair copy (both orientations of one input) moves NaN / inf /
    -0.0 bit-exactly: expr1-shaped 2*(A^T + B) + 2*(A + B^T) at 4096^2."""
    n = 4096
    a = _specials((n, n), np.float32, 3)
    b = _specials((n, n), np.float32, 4)
    A, B = fm.from_array(a, ctx=gpu_ctx), fm.from_array(b, ctx=gpu_ctx)
    got = (2 * (A.t() + B) + 2 * (A + B.t())).eval().to_numpy()
    two = np.float32(2)
    with np.errstate(invalid="ignore", over="ignore"):
        want = (two * (a.T + b)).astype(np.float32) + (two * (a + b.T)).astype(np.float32)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.array_equal(got[ok].view(np.uint32), want[ok].view(np.uint32))


@pytest.mark.parametrize("name", ["sigmoid", "swish", "gelu", "softplus"])
def test_transcendental_chains_at_bulk_scale(gpu_ctx, name):
    """The suite's transcendental members run the bulk-staged copy with 24
    consumer warps (bulk.cuh CopyWarps); a ragged 2^22 + 37 elements against
    the oracle (f32 exp / tanh correctly rounded, every node rounded to f32)."""
    import math
    n = (1 << 22) + 37
    a = np.random.default_rng(21).uniform(-12, 12, n).astype(np.float32).reshape(-1, 1)
    a[:9, 0] = [0.0, -0.0, np.inf, -np.inf, np.nan, 88.0, -88.0, 1e-30, -1e-30]
    A = fm.from_array(a, ctx=gpu_ctx)
    exprs = {
        "sigmoid": lambda X: 1 / (1 + fm.exp(-X)),
        "swish": lambda X: X / (1 + fm.exp(-1.0 * X)),
        "gelu": lambda X: (X / 2) * (1 + fm.tanh(math.sqrt(2.0 / 3.14159265358979) * (X + 0.044715 * (X ** 3)))),
        "softplus": lambda X: fm.log(1 + fm.exp(X)),
    }
    e = exprs[name](A)
    got = e.eval().to_numpy()
    want = orc.materialize(e.node, {A.mat_id: a})
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert orc.max_ulp(got[ok], want[ok]) <= 2, name
    diff = np.count_nonzero(got[ok].view(np.uint32) != want[ok].view(np.uint32))
    assert diff <= n // 100_000, (name, diff)
