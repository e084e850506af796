"""Backend-level drop-in: the reference's OWN user API, planner and code
generator (fusemat.Context / Mat / plan / generate_kernel_source) driving
B200Backend, checked against the reference's own RefBackend on the same
inputs.

The reference package comes from `baseline/_ref/` (the offline
`pip install --target baseline/_ref` of /root/reference/pkg recorded in
DESIGN.md); when that install is absent the module is skipped.  Nothing here
reads /root/reference.

Routes exercised: `Context(backend=<instance>)` (matrix.py:57-58) ->
`execute_plan` / `_launch_fused` (matrix.py:83-113) -> `Backend.compile`
(KernelSource with the reference's node classes, adopted by
backend.adopt_tree) -> `Backend.launch` with the reference's positional
argument list (codegen.py:304-318) -> `Backend.matmul` (matrix.py:86-92).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
if (REF / "fusemat").is_dir() and str(REF) not in sys.path:
    sys.path.append(str(REF))
fusemat = pytest.importorskip("fusemat", reason="reference not installed in baseline/_ref")
from fusemat import bench as rbench  # noqa: E402
from fusemat import oracle as roracle  # noqa: E402

pytestmark = pytest.mark.gpu

# suite members whose ops are all exactly rounded (+ - * / scalars, >, pow_int,
# views, transpose, conv): bit-identical to the reference interpreter.
EXACT = ["add2", "add4", "addsub2", "addsub4", "expr1", "diagsum", "relu"]
# transcendental members: the reference's own gate (rel 1e-5, test_backend.py:182)
TRANSC = ["expr2", "expr3", "sigmoid", "swish", "gelu"]


@pytest.fixture(scope="module")
def b200():
    import paper_2604_22242_b200 as fm
    if not fm.B200Backend.available():
        pytest.fail("GPU test selected but no CUDA device / libfmb200.so is usable")
    return fm.B200Backend()


def _run(name, backend, etype, n=64, seed=42):
    spec = rbench.BenchSpec(expr_name=name, n=n, etype=etype, seed=seed)
    ctx = fusemat.Context(backend)
    out, e = rbench.build_expression(spec, ctx)
    out.assign(e)
    return out.to_numpy(), ctx, e


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("name", EXACT)
def test_reference_context_exact_members(b200, name, etype):
    got, ctx, _ = _run(name, b200, etype)
    want, _, _ = _run(name, "ref", etype)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert np.array_equal(got, want), f"{name}/{etype}: not bit-identical to the reference"
    assert ctx.launches == 1 and ctx.compile_count == 1     # one fused launch, one "compile"


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("name", TRANSC)
def test_reference_context_transcendental_members(b200, name, etype):
    got, ctx, e = _run(name, b200, etype)
    want, _, _ = _run(name, "ref", etype)
    # the reference's own gate for device backends (bench.py:245-267):
    # allclose_mixed(rtol=atol=1e-4) against the per-node oracle, and vs the
    # reference interpreter; f64 chains also at rtol = atol = 1e-12
    env = {mid: m.to_numpy() for mid, m in e.mats.items()}
    assert roracle.allclose_mixed(got, roracle.materialize(e.node, env))
    assert roracle.allclose_mixed(got, want)
    if etype == "f64":
        assert roracle.allclose_mixed(got, want, rtol=1e-12, atol=1e-12)
    assert ctx.launches == 1


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_reference_context_matmul_chain(b200, etype):
    """a@b@c@d: the reference plans 3 MatMulSteps; each goes through
    Backend.matmul, which keeps the reference's f64-accumulated numerics."""
    got, ctx, _ = _run("chain", b200, etype)
    want, _, _ = _run("chain", "ref", etype)
    tol = 1e-6 if etype == "f32" else 1e-13
    assert roracle.compare(got, want, tol) <= tol
    assert ctx.launches == 3


def test_reference_context_accu_and_cache(b200):
    ctx = fusemat.Context(b200)
    x = fusemat.randu(300, 200, 7, "f64", ctx)
    y = fusemat.randu(300, 200, 8, "f64", ctx)
    got = fusemat.accu(x * y)
    rc = fusemat.Context("ref")
    want = fusemat.accu(fusemat.randu(300, 200, 7, "f64", rc) * fusemat.randu(300, 200, 8, "f64", rc))
    assert abs(got - want) <= 1e-12 * abs(want)
    z = fusemat.zeros(300, 200, "f64", ctx)
    ctx.reset_counters()
    for k in range(52):                       # test_matrix.py:108-117 cache discipline
        z.assign(x * (k + 1.0) + y)
    assert ctx.compile_count == 1 and ctx.launches == 52
    xv, yv = x.to_numpy(), y.to_numpy()
    assert np.array_equal(z.to_numpy(), xv * 52.0 + yv)


def test_reference_context_int_wrap_and_conv(b200):
    ctx = fusemat.Context(b200)
    rc = fusemat.Context("ref")
    outs = []
    for c in (ctx, rc):
        a = fusemat.randi(50, 40, 10, 3, "u32", c)
        f = fusemat.randu(50, 40, 4, "f32", c)
        z = fusemat.zeros(50, 40, "u32", c)
        z.assign(a * a - a * 7 + fusemat.conv_to(f * 100 - 50, "u32"))
        outs.append(z.to_numpy())
    assert np.array_equal(outs[0], outs[1])
