"""tcgen05 GEMM (csrc/gemm_tc.cu) against the f64 product of the same
operands -- the reference's matmul numerics (f64 accumulation, cjit.py:33-51;
oracle.py:53-57) -- at the north-star tolerance of 1e-5 relative.

Bound (elementwise): |got - want| <= 1e-5 * sum_p |a_ip| |b_pj|.
* bf16 operands: products are exact in f32; the tensor core truncates its
  f32 accumulator at every K=16 step, and the kernel drains the TMEM
  accumulator into round-to-nearest f32 register sums every 1024 of K, so
  the truncation error is <= 64 * 2^-23 = 7.6e-6 for any K (one 8192-deep
  TMEM accumulation measured 3.1e-5 before chunking).
* f32 operands: each is scaled by a power of two from its max |x| and split
  into two fp16 planes (x 2^e = hi + lo + O(2^-22)); the three significant
  plane products are accumulated in the same launch, drained every 512 of K;
  the dropped terms are O(2^-21), so the same 1e-5 holds.
"""

import numpy as np
import pytest

import paper_2604_22242_b200 as fm
from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu



def rel_bound(k: int) -> float:
    return 1e-5


def _bf16(shape, seed):
    return orc.bf16_round(np.random.default_rng(seed).random(shape, dtype=np.float64).astype(np.float32) - 0.25)


def _check(got, a, b, alpha):
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    want = alpha * (a64 @ b64)
    bound = rel_bound(a.shape[1]) * abs(alpha) * (np.abs(a64) @ np.abs(b64)) + 1e-30
    err = np.abs(got.astype(np.float64) - want)
    assert np.all(err <= bound), float((err / bound).max())


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize("trans_b", [False, True])
@pytest.mark.parametrize("mnk", [(256, 512, 128), (200, 304, 72), (128, 256, 64), (1000, 520, 1032)])
def test_tcgen05_gemm_layouts(gpu_ctx, trans_a, trans_b, mnk):
    m, n, k = mnk
    be = gpu_ctx.backend
    a = _bf16((m, k), 1)
    b = _bf16((k, n), 2)
    A = fm.from_array(a.T.copy() if trans_a else a, etype="bf16", ctx=gpu_ctx)
    B = fm.from_array(b.T.copy() if trans_b else b, etype="bf16", ctx=gpu_ctx)
    C = fm.Mat(m, n, "f32", gpu_ctx)
    assert be.gemm_path(C.handle, A.handle, B.handle, m, n, k, trans_a, trans_b, 2.0) == "tcgen05"
    be.gemm(C.handle, A.handle, B.handle, m, n, k, trans_a, trans_b, alpha=2.0)
    _check(C.to_numpy(), a, b, 2.0)


def test_tcgen05_gemm_falls_back_on_unaligned_stride(gpu_ctx):
    m, n, k = 64, 36, 24          # ldb = n = 36 bf16 = 72 B: not a 16-byte multiple for TMA
    be = gpu_ctx.backend
    a, b = _bf16((m, k), 3), _bf16((k, n), 4)
    A = fm.from_array(a, etype="bf16", ctx=gpu_ctx)
    B = fm.from_array(b.T.copy(), etype="bf16", ctx=gpu_ctx)
    C = fm.Mat(m, n, "f32", gpu_ctx)
    assert be.gemm_path(C.handle, A.handle, B.handle, m, n, k, False, True) == "exact"
    be.gemm(C.handle, A.handle, B.handle, m, n, k, False, True)
    _check(C.to_numpy(), a, b, 1.0)


def test_c5_expression_is_one_tensor_core_launch(gpu_ctx):
    """Z = 2 * X @ Y.t() through the public API: scalar and transpose fold
    into the single GEMM launch (the reference plans 3 launches)."""
    ctx = fm.Context(gpu_ctx.backend)
    n = 512
    X = fm.randu(n, n, 42, "bf16", ctx)
    Y = fm.randu(n, n, 43, "bf16", ctx)
    Z = fm.zeros(n, n, ctx=ctx)
    ctx.reset_counters()
    Z.assign(2 * X @ Y.t())
    assert ctx.launches == 1
    x, y = orc.randu(n, n, 42, "bf16"), orc.randu(n, n, 43, "bf16")
    _check(Z.to_numpy(), x, y.T, 2.0)


def test_gemm_c5_size_sampled(gpu_ctx):
    """Full C5 size 8192^3: sampled rows/columns against the f64 product."""
    ctx = fm.Context(gpu_ctx.backend)
    n = 8192
    X = fm.randu(n, n, 42, "bf16", ctx)
    Y = fm.randu(n, n, 43, "bf16", ctx)
    Z = fm.Mat(n, n, "f32", ctx)
    Z.assign(2 * X @ Y.t())
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(n, 48, replace=False))
    cols = np.sort(rng.choice(n, 48, replace=False))
    x = X.to_numpy()
    y = Y.to_numpy()
    z = Z.to_numpy()
    _check(z[np.ix_(rows, cols)], x[rows, :], y[cols, :].T, 2.0)


def _f32(shape, seed):
    return (np.random.default_rng(seed).random(shape, dtype=np.float64) - 0.25).astype(np.float32)


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize("trans_b", [False, True])
@pytest.mark.parametrize("mnk", [(256, 512, 128), (200, 304, 72), (1000, 520, 1032), (64, 36, 24)])
def test_tcgen05_gemm_f32_split_layouts(gpu_ctx, trans_a, trans_b, mnk):
    """f32 operands through the split-bf16 tensor-core path, every operand
    layout, ragged M/N/K (K not a multiple of the 64-deep k-block)."""
    m, n, k = mnk
    be = gpu_ctx.backend
    a = _f32((m, k), 5)
    b = _f32((k, n), 6)
    A = fm.from_array(a.T.copy() if trans_a else a, etype="f32", ctx=gpu_ctx)
    B = fm.from_array(b.T.copy() if trans_b else b, etype="f32", ctx=gpu_ctx)
    C = fm.Mat(m, n, "f32", gpu_ctx)
    assert be.gemm_path(C.handle, A.handle, B.handle, m, n, k, trans_a, trans_b, 2.0, precision=1) == "tcgen05"
    be.gemm(C.handle, A.handle, B.handle, m, n, k, trans_a, trans_b, alpha=2.0, precision=1)
    _check(C.to_numpy(), a, b, 2.0)
    # AUTO keeps small f32 products on the exact f64-accumulating kernel
    if m * n * k < 1 << 28:
        assert be.gemm_path(C.handle, A.handle, B.handle, m, n, k, trans_a, trans_b, 2.0) == "exact"


def test_c5_f32_size_sampled(gpu_ctx):
    """C5 in f32 at full size through the public API (one split-bf16 GEMM
    launch plus the two operand splits), sampled against the f64 product."""
    ctx = fm.Context(gpu_ctx.backend)
    n = 8192
    X = fm.randu(n, n, 42, "f32", ctx)
    Y = fm.randu(n, n, 43, "f32", ctx)
    Z = fm.Mat(n, n, "f32", ctx)
    ctx.reset_counters()
    Z.assign(2 * X @ Y.t())
    assert ctx.launches == 1
    rng = np.random.default_rng(1)
    rows = np.sort(rng.choice(n, 32, replace=False))
    cols = np.sort(rng.choice(n, 32, replace=False))
    x, y, z = X.to_numpy(), Y.to_numpy(), Z.to_numpy()
    _check(z[np.ix_(rows, cols)], x[rows, :], y[cols, :].T, 2.0)


# --- GEMM epilogue fusion: s2*(A@B) +/- sb*C in one launch ---------------------------
def _epilogue_cases():
    return [("2*(A@B)+C", lambda A, B, C: 2 * (A @ B) + C, lambda t, c: np.float32(2) * t + c),
            ("C-A@B", lambda A, B, C: C - A @ B, lambda t, c: c - t),
            ("A@B-3*C", lambda A, B, C: A @ B - 3 * C, lambda t, c: t - np.float32(3) * c)]


@pytest.mark.parametrize("case", _epilogue_cases(), ids=lambda c: c[0])
def test_gemm_epilogue_exact_path_bit_exact(gpu_ctx, case):
    """Small f32 products take the exact kernel: T is the reference's
    f64-accumulated product rounded to f32, then the reference's elementwise
    step with per-op f32 rounding -- bit for bit, in ONE launch (the
    reference plans a MatMulStep plus a fused copy)."""
    _, build, ref = case
    ctx = fm.Context(gpu_ctx.backend)
    a, b, c = _f32((96, 80), 1), _f32((80, 72), 2), _f32((96, 72), 3)
    A, B, C = (fm.from_array(v, ctx=ctx) for v in (a, b, c))
    Z = fm.zeros(96, 72, ctx=ctx)
    ctx.reset_counters()
    Z.assign(build(A, B, C))
    assert ctx.launches == 1
    t = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    assert np.array_equal(Z.to_numpy(), ref(t, c))


@pytest.mark.parametrize("etype", ["f32", "bf16"])
def test_gemm_epilogue_tensor_path(gpu_ctx, etype):
    ctx = fm.Context(gpu_ctx.backend)
    m, n, k = 1024, 768, 1152
    a = _bf16((m, k), 4) if etype == "bf16" else _f32((m, k), 4)
    b = _bf16((k, n), 5) if etype == "bf16" else _f32((k, n), 5)
    c = _f32((m, n), 6)
    A, B = fm.from_array(a, etype=etype, ctx=ctx), fm.from_array(b, etype=etype, ctx=ctx)
    C = fm.from_array(c, ctx=ctx)
    Z = fm.zeros(m, n, ctx=ctx)
    ctx.reset_counters()
    Z.assign(2 * (A @ B) + C)
    assert ctx.launches == 1
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    want = 2 * (a64 @ b64) + c
    bound = 1e-5 * (2 * (np.abs(a64) @ np.abs(b64)) + np.abs(c)) + 1e-30
    assert np.all(np.abs(Z.to_numpy() - want) <= bound)


def test_gemm_epilogue_in_place_and_f64(gpu_ctx):
    ctx = fm.Context(gpu_ctx.backend)
    a, b, c = (np.random.default_rng(s).random(sh) for s, sh in ((7, (50, 40)), (8, (40, 30)), (9, (50, 30))))
    A, B, C = (fm.from_array(v, ctx=ctx) for v in (a, b, c))     # f64
    ctx.reset_counters()
    C.assign(C + A @ B)                                          # addend aliases the output
    assert ctx.launches == 1
    assert np.allclose(C.to_numpy(), (a @ b) + c, rtol=1e-12, atol=0)


def test_gemm_epilogue_with_folded_transposes(gpu_ctx):
    """Scale, transposes and the addend all fold into one launch:
    3 * (X.t() @ Y.t()) - C with X, Y stored untransposed (tensor path)."""
    ctx = fm.Context(gpu_ctx.backend)
    m, n, k = 640, 384, 896
    x = _f32((k, m), 11)            # X.t() is m x k
    y = _f32((n, k), 12)            # Y.t() is k x n
    c = _f32((m, n), 13)
    X, Y, C = (fm.from_array(v, ctx=ctx) for v in (x, y, c))
    Z = fm.zeros(m, n, ctx=ctx)
    ctx.reset_counters()
    Z.assign(3 * (X.t() @ Y.t()) - C)
    assert ctx.launches == 1
    a64, b64 = x.T.astype(np.float64), y.T.astype(np.float64)
    want = 3 * (a64 @ b64) - c
    bound = 1e-5 * (3 * (np.abs(a64) @ np.abs(b64)) + np.abs(c)) + 1e-30
    assert np.all(np.abs(Z.to_numpy() - want) <= bound)


def test_accu_of_transposed_and_view_expressions(gpu_ctx):
    """Full reductions over non-flat programs (transposed / view leaves)."""
    ctx = fm.Context(gpu_ctx.backend)
    X = fm.randu(700, 700, 21, "f64", ctx)
    Y = fm.randu(700, 700, 22, "f64", ctx)
    x, y = X.to_numpy(), Y.to_numpy()
    got = fm.accu(X.t() % Y)
    want = orc.accu(x.T * y, orc.ElemType.f64)
    assert abs(got - want) <= 1e-12 * abs(want)
    got = fm.accu(X.submat(5, 7, 300, 200) - Y.submat(1, 2, 300, 200))
    want = orc.accu(x[5:305, 7:207] - y[1:301, 2:202], orc.ElemType.f64)
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want))


# ---- operand prologues (csrc/split.cuh, fm_gemm_prologue): an elementwise
# operand is evaluated inside the GEMM's operand pass, not materialised.  The
# result must be bit-identical to the reference's plan -- the operand copied
# into a temp, then the product (plan.py:125-151) -- on every path.

def _two_step(ctx, operand_expr, shape, etype, product):
    T = fm.Mat(*shape, etype, ctx)
    T.assign(operand_expr)
    return product(T)


@pytest.mark.parametrize("etype,mnk", [("f32", (640, 768, 576)),    # tensor path (split planes)
                                       ("f32", (96, 80, 72)),       # exact path (materialised in C)
                                       ("f64", (96, 80, 72))])
def test_gemm_prologue_bit_identical_to_materialised(gpu_ctx, etype, mnk):
    m, n, k = mnk
    X = fm.randu(m, k, 1, etype, gpu_ctx)
    Y = fm.randu(m, k, 2, etype, gpu_ctx)
    Z = fm.randu(k, n, 3, etype, gpu_ctx)
    out = fm.Mat(m, n, etype, gpu_ctx)
    gpu_ctx.reset_counters()
    out.assign((X + 2 * Y) @ Z)
    assert gpu_ctx.launches == 1                  # no operand temp launch
    want = _two_step(gpu_ctx, X + 2 * Y, (m, k), etype, lambda T: T @ Z)
    ref = fm.Mat(m, n, etype, gpu_ctx)
    ref.assign(want)
    assert np.array_equal(out.to_numpy(), ref.to_numpy())
    x, y, z = X.to_numpy(), Y.to_numpy(), Z.to_numpy()
    t = x + x.dtype.type(2) * y
    _check(out.to_numpy(), t, z, 1.0)


def test_gemm_prologue_both_operands_transposed_and_views(gpu_ctx):
    m, n, k = 512, 640, 1024                      # tensor path
    A = fm.randu(k, m, 11, "f32", gpu_ctx)        # used as A.t()
    B = fm.randu(k, m, 12, "f32", gpu_ctx)
    W = fm.randu(n + 8, k + 4, 13, "f32", gpu_ctx)
    out = fm.Mat(m, n, "f32", gpu_ctx)
    rhs = (W.submat(8, 4, n, k) - 0.5).t()
    out.assign(3.0 * ((A % B).t() @ rhs))
    a, b, w = A.to_numpy(), B.to_numpy(), W.to_numpy()
    lhs_v = (a * b).T
    rhs_v = (w[8:8 + n, 4:4 + k] + np.float32(-0.5)).T
    ref_l = fm.Mat(k, m, "f32", gpu_ctx)
    ref_l.assign(A % B)
    ref_r = fm.Mat(n, k, "f32", gpu_ctx)
    ref_r.assign(W.submat(8, 4, n, k) - 0.5)
    ref = fm.Mat(m, n, "f32", gpu_ctx)
    ref.assign(3.0 * (ref_l.t() @ ref_r.t()))
    assert np.array_equal(out.to_numpy(), ref.to_numpy())
    _check(out.to_numpy(), lhs_v, rhs_v, 3.0)


def test_gemm_prologue_with_epilogue_and_graph(gpu_ctx):
    m, n, k = 512, 512, 1024
    X = fm.randu(m, k, 21, "f32", gpu_ctx)
    Z = fm.randu(k, n, 22, "f32", gpu_ctx)
    C = fm.randu(m, n, 23, "f32", gpu_ctx)
    out = fm.Mat(m, n, "f32", gpu_ctx)
    g = fm.capture(lambda: out.assign(2 * (fm.abs(X - 0.5) @ Z) + C), gpu_ctx)
    g.replay()
    g.replay()
    gpu_ctx.sync()
    T = fm.Mat(m, k, "f32", gpu_ctx)
    T.assign(fm.abs(X - 0.5))
    ref = fm.Mat(m, n, "f32", gpu_ctx)
    ref.assign(2 * (T @ Z) + C)
    assert np.array_equal(out.to_numpy(), ref.to_numpy())
    g.close()
