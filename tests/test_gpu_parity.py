"""GPU parity: the CUDA path against the CPU oracle and the reference's own
recorded outputs (tests/golden/).  Every case runs twice: through the
ahead-of-time template kernels where a template exists, and forced through
the generic register VM.

Gates:
* integer results and chains without transcendentals: bit-exact vs the oracle
  (and vs the reference's interpreter / compiled-C outputs);
* f32 chains with exp/log/tanh: <= 1 ulp vs the correctly-rounded oracle;
* f64 chains with transcendentals: 1e-12 relative (CUDA libdevice vs numpy libm);
* every case within the reference's own tolerances of every reference route
  (oracle.py:132-146 allclose_mixed; test_backend.py:182-192 1e-5 / 1e-12).
"""

import numpy as np
import pytest

import paper_2604_22242_b200 as fm
from conftest import case_env, case_expected
from gpuutil import bind, run_assign
from oracle import fm_oracle as orc
from paper_2604_22242_b200.exprtree import ElemType
from treeio import from_json

pytestmark = pytest.mark.gpu

TRANSC = ("exp", "log", "tanh")


def _has_transc(case):
    s = str(case["tree"])
    return any(f"'{t}'" in s for t in TRANSC)


@pytest.fixture(scope="module", params=["template", "vm"])
def ctx(request, gpu_ctx):
    if request.param == "template":
        return gpu_ctx
    return fm.Context(fm.B200Backend(use_templates=False))


def _copy_cases(golden_cases):
    cases, arrays = golden_cases
    for c in cases:
        node = from_json(c["tree"])
        if "oracle" in c["expected"] and not fm.exprtree.contains_matmul(node) \
                and not c["name"].startswith("c2_"):
            yield c, node, arrays


def test_golden_copy_cases(ctx, golden_cases):
    n_cases = 0
    for case, node, arrays in _copy_cases(golden_cases):
        env = case_env(case, arrays)
        got = run_assign(bind(node, env, ctx))
        want = orc.materialize(node, env)
        if node.etype is ElemType.f64 and _has_transc(case):
            # libdevice vs numpy f64 exp/log/tanh differ by <= 1-2 ulp per node and
            # later cancellation amplifies that: the reference's own f64 gate applies
            # (test_backend.py:182-192, 1e-12 relative).
            assert orc.compare(got, want) <= 1e-12 or orc.allclose_mixed(got, want, 1e-12, 1e-12), \
                case["name"]
        elif _has_transc(case):
            assert orc.max_ulp(got, want) <= 1, case["name"]
        else:
            assert orc.max_ulp(got, want) == 0, case["name"]
        for label in ("oracle", "ref", "cjit"):
            if label in case["expected"]:
                ref = case_expected(case, arrays, label)
                assert orc.allclose_mixed(got, ref), (case["name"], label)
                if not _has_transc(case):
                    assert orc.max_ulp(got, ref) == 0, (case["name"], label)
        n_cases += 1
    assert n_cases > 150


def test_golden_accu_cases(ctx, golden_cases):
    cases, arrays = golden_cases
    for case in cases:
        if not case["name"].startswith("c2_"):
            continue
        node = from_json(case["tree"])
        env = case_env(case, arrays)
        e = bind(node, env, ctx)
        got = fm.accu(e)
        exact = orc.accu(orc.materialize(node, env), node.etype)
        assert got == pytest.approx(exact, rel=1e-12), case["name"]
        for label in ("accu_ref", "accu_cjit"):
            assert got == pytest.approx(case_expected(case, arrays, label), rel=1e-10)


def test_golden_gemm_cases(gpu_ctx, golden_cases):
    cases, arrays = golden_cases
    for case in cases:
        if not case["name"].startswith("gemm_"):
            continue
        node = from_json(case["tree"])
        env = case_env(case, arrays)
        got = run_assign(bind(node, env, gpu_ctx))
        ref = case_expected(case, arrays, "ref")
        # reference tolerance for matmul (SPEC.md ledger / bench.py:34): 1e-4
        assert orc.compare(got, ref) <= 1e-4, case["name"]


def test_exact_gemm_bit_identical_to_reference(gpu_ctx, golden_cases):
    """FM_GEMM_EXACT keeps the reference's summation order: bit-identical."""
    cases, arrays = golden_cases
    case = next(c for c in cases if c["name"] == "gemm_nn")
    env = case_env(case, arrays)
    a, b = [env[int(k)] for k in case["env"]]
    be = gpu_ctx.backend
    A, B = fm.from_array(a, ctx=gpu_ctx), fm.from_array(b, ctx=gpu_ctx)
    C = fm.zeros(a.shape[0], b.shape[1], ctx=gpu_ctx)
    be.gemm(C.handle, A.handle, B.handle, a.shape[0], b.shape[1], a.shape[1], precision=2)
    assert np.array_equal(C.to_numpy(), case_expected(case, arrays, "ref"))


def test_kernel_selection(gpu_ctx):
    """The C1 / C3 / C4 signatures hit AOT templates; other trees use the VM."""
    x = fm.randu(64, 64, 1, ctx=gpu_ctx)
    y = fm.randu(64, 64, 2, ctx=gpu_ctx)
    z = fm.zeros(64, 64, ctx=gpu_ctx)
    z.assign(2 * (x % y) + x)
    k = gpu_ctx.cache.lookup("copy|" + fm.exprtree.signature_of((2 * (x % y) + x).node))
    assert k is not None and k.uses_template
    z.assign(x.t() + y)
    k2 = gpu_ctx.cache.lookup("copy|" + fm.exprtree.signature_of((x.t() + y).node))
    assert k2 is not None and not k2.uses_template


# --- north-star ops pinned through the reference -----------------------------
def test_dim_reductions_pinned_to_reference(gpu_ctx, golden_cases):
    """GPU sum / mean along both dims vs the reference's accu of each column /
    row submat; max / min / index_max / index_min vs numpy on the values the
    reference's compiled backend produced (exact)."""
    cases, arrays = golden_cases
    pins = [c for c in cases if c["name"].startswith("pin_c4_")]
    assert len(pins) == 3
    K = orc.ReduceKind
    for c in pins:
        node = from_json(c["tree"])
        e = bind(node, case_env(c, arrays), gpu_ctx)
        v = arrays[c["expected"]["cjit"]]
        colsum = arrays[c["expected"]["colsum_ref"]]
        rowsum = arrays[c["expected"]["rowsum_ref"]]
        n_rows, n_cols = v.shape
        f64 = node.etype is ElemType.f64
        for dim, ref_sum, n in ((0, colsum, n_rows), (1, rowsum, n_cols)):
            mag = np.abs(v.astype(np.float64)).sum(axis=dim)
            s = fm.sum(e, dim).eval().to_numpy().ravel().astype(np.float64)
            m = fm.mean(e, dim).eval().to_numpy().ravel().astype(np.float64)
            if f64:
                assert np.all(np.abs(s - ref_sum) <= 1e-13 * mag), (c["name"], dim)
                assert np.all(np.abs(m - ref_sum / n) <= 1e-13 * mag / n), (c["name"], dim)
            else:                     # f32 outputs: the f64 sum rounded once
                assert np.array_equal(s.astype(np.float32), ref_sum.astype(np.float32)), (c["name"], dim)
            for fn, red in ((fm.max, np.max), (fm.min, np.min), (fm.index_max, np.argmax),
                            (fm.index_min, np.argmin)):
                got = fn(e, dim).eval().to_numpy().ravel()
                assert np.array_equal(got, red(v, axis=dim)), (c["name"], fn.__name__, dim)


def test_norm_and_dot_pinned_to_reference(gpu_ctx, golden_cases):
    cases, arrays = golden_cases
    for c in (c for c in cases if c["name"].startswith("pin_norm_dot_")):
        env = case_env(c, arrays)
        x, y = (fm.from_array(env[k], ctx=gpu_ctx) for k in sorted(env))
        normsq = c["expected"]["normsq_ref"]["scalar"]
        dot = c["expected"]["dot_ref"]["scalar"]
        assert abs(fm.norm(x - y) ** 2 - normsq) <= 1e-12 * normsq
        assert abs(fm.dot(x, y) - dot) <= 1e-12 * dot
        assert abs(fm.accu((x - y) ** 2) - normsq) <= 1e-12 * normsq


# ---- the register VM over bulk-staged chunks (bulk.cuh k_copy_bulk_vm):
# flat programs large enough for a wave of chunks, every slot width, a ragged
# tail, against the template path / numpy on the same inputs

@pytest.fixture(scope="module")
def vm_ctx(gpu_ctx):
    return fm.Context(fm.B200Backend(use_templates=False))


@pytest.mark.parametrize("n_rows,n_cols", [(2048, 1024), (3001, 997)])
def test_vm_bulk_staged_copies(vm_ctx, n_rows, n_cols):
    ctx = vm_ctx
    X = fm.randu(n_rows, n_cols, 11, "f32", ctx)
    Y = fm.randu(n_rows, n_cols, 12, "f32", ctx)
    D = fm.randu(n_rows, n_cols, 13, "f64", ctx)
    U = fm.randi(n_rows, n_cols, 50, 14, "u32", ctx)
    B = fm.randu(n_rows, n_cols, 15, "bf16", ctx)
    x, y, d, u, b = (M.to_numpy() for M in (X, Y, D, U, B))
    f = np.float32
    Z = fm.Mat(n_rows, n_cols, "f32", ctx)
    Z.assign(3 * (X % Y) - X / 2 + Y)
    assert np.array_equal(Z.to_numpy(), (f(3) * (x * y) - x / f(2)) + y)
    Z.assign(fm.conv_to(U, "f32") * X + fm.conv_to(B, "f32"))
    assert np.array_equal(Z.to_numpy(), u.astype(f) * x + b.astype(f))
    W = fm.Mat(n_rows, n_cols, "f64", ctx)
    W.assign(D * fm.conv_to(X, "f64") - D / 3.0)
    # X / s is X * (1/s) in the reference (matrix.py:170-176)
    assert np.array_equal(W.to_numpy(), d * x.astype(np.float64) - (1.0 / 3.0) * d)
    for _ in range(2):                      # the chunk counter resets between launches
        Z.assign(X + Y + X + Y + X + Y + X + Y)
    assert np.array_equal(Z.to_numpy(), ((((((x + y) + x) + y) + x) + y) + x) + y)


@pytest.mark.parametrize("n", [4_000_000, 5_000_011])
def test_vm_bulk_staged_accu(vm_ctx, n):
    """Full reductions of flat programs on the VM over bulk-staged chunks
    (bulk.cuh k_accu_bulk_vm): f64 accumulation within 1e-12 of the exactly
    rounded sum, wrapping u32 sums exact, deterministic run to run."""
    ctx = vm_ctx
    x = fm.randu(n, 1, 21, "f32", ctx)
    y = fm.randu(n, 1, 22, "f32", ctx)
    d = fm.randu(n, 1, 23, "f64", ctx)
    u = fm.randi(n, 1, 1000, 24, "u32", ctx)
    xv, yv, dv, uv = (M.to_numpy().ravel() for M in (x, y, d, u))
    f = np.float32
    got = fm.accu(3 * (x % y) - x)
    want = orc.accu(f(3) * (xv * yv) - xv, fm.ElemType.f32)
    assert abs(got - want) <= 1e-12 * abs(want)
    assert fm.accu(3 * (x % y) - x) == got                       # deterministic
    got = fm.accu(d * fm.conv_to(x, "f64") + d)
    want = orc.accu(dv * xv.astype(np.float64) + dv, fm.ElemType.f64)
    assert abs(got - want) <= 1e-12 * abs(want)
    assert fm.accu(u * 3 + u) == int((uv.astype(np.uint64) * 4).sum() & 0xFFFFFFFF)
    got = fm.norm(x - 2 * y)
    want = float(np.sqrt(orc.accu(((xv - f(2) * yv) ** 2).astype(f), fm.ElemType.f32)))
    assert abs(got - want) <= 1e-12 * want


# ---- randomized trees at bulk scale: the VM's bulk-staged kernels and the
# tile-pair kernel see every operator on >= a wave of chunks, against the
# oracle's per-node rounding (exact operators only: 0 ulp)

def _rand_expr(rng, leaves, depth, square):
    if depth == 0 or rng.random() < 0.25:
        m = leaves[rng.integers(len(leaves))]
        return m.t() if square and rng.random() < 0.3 else m
    k = rng.integers(8)
    a = _rand_expr(rng, leaves, depth - 1, square)
    if k < 4:
        b = _rand_expr(rng, leaves, depth - 1, square)
        return [a + b, a - b, a % b, a / (b + 2.0)][k]
    s = float(rng.integers(1, 9)) / 4.0
    return [s * a, a + s, -a, fm.abs(a)][k - 4]


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("square", [False, True])
def test_random_trees_at_bulk_scale(vm_ctx, gpu_ctx, etype, square):
    rng = np.random.default_rng(7 if square else 8)
    for ctx in (vm_ctx, gpu_ctx):
        shape = (1024, 1024) if square else (2048, 640)
        leaves = [fm.randu(*shape, 600 + i, etype, ctx) for i in range(4)]
        env = {m.mat_id: m.to_numpy() for m in leaves}
        Z = fm.Mat(*shape, etype, ctx)
        for t in range(12):
            e = _rand_expr(rng, leaves, 4, square)
            if not hasattr(e, "node"):
                e = e + 0.0
            Z.assign(e)
            want = orc.materialize(e.node, env)
            assert orc.max_ulp(Z.to_numpy(), want) == 0, (etype, square, t, str(e.node)[:200])
            if not square:                       # and the full reduction of the same tree
                exact = orc.accu(want, e.node.etype)
                scale = orc.accu(np.abs(want), e.node.etype)
                assert abs(fm.accu(e) - exact) <= 1e-12 * scale, (etype, t)
