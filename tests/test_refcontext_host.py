"""CPU half of the backend-level drop-in test: the reference's own Context,
planner and code generator (baseline/_ref/fusemat) drive B200Backend with its
native layer replaced by a recording double, so the adapter plumbing --
foreign element types and node classes, the reference's positional launch
arguments (codegen.py:304-318), matmul arguments (matrix.py:86-92) -- is
checked here without a GPU.  The double records calls; it computes nothing.
tests/test_gpu_refcontext.py checks the results on the B200.
"""

import ctypes
import sys
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
if (REF / "fusemat").is_dir() and str(REF) not in sys.path:
    sys.path.append(str(REF))
fusemat = pytest.importorskip("fusemat", reason="reference not installed in baseline/_ref")

from paper_2604_22242_b200 import backend as bk  # noqa: E402
from recording import launches as _launches_rec, recording_backend as _backend  # noqa: E402


def _launches(b, name):
    return _launches_rec(b, name)


def test_reference_context_c1_binds_one_template_launch():
    b = _backend()
    ctx = fusemat.Context(b)
    X = fusemat.zeros(64, 48, "f32", ctx)
    Y = fusemat.zeros(64, 48, "f32", ctx)
    Z = fusemat.zeros(64, 48, "f32", ctx)
    Z.assign(2 * (X * Y) + X)
    (kid, prog, out, rows, cols, _), = _launches(b, "fm_launch_copy")
    assert kid >= 0, "C1 must hit an AOT template kernel"
    p = prog._obj
    assert (rows, cols) == (64, 48) and p.n_slots == 2 and p.flat == 1
    assert [p.slots[i].ptr for i in range(2)] == [b.ptr(X.handle), b.ptr(Y.handle)]
    assert p.slots[0].ld == 64
    assert ctypes.c_uint32(p.scalars[0]).value == 0x40000000        # 2.0f, typed by the node
    assert out == b.ptr(Z.handle)
    assert ctx.launches == 1 and ctx.compile_count == 1


def test_reference_context_views_go_to_the_vm():
    b = _backend()
    ctx = fusemat.Context(b)
    X = fusemat.zeros(10, 10, "f64", ctx)
    Y = fusemat.zeros(10, 10, "f64", ctx)
    Z = fusemat.zeros(5, 5, "f64", ctx)
    Z.assign(X.center_half() + Y.center_half())
    (kid, prog, out, rows, cols, _), = _launches(b, "fm_launch_copy")
    p = prog._obj
    assert (rows, cols) == (5, 5) and p.flat == 0
    assert {(p.slots[i].row_off, p.slots[i].col_off) for i in range(p.n_slots)} == {(2, 2)}


def test_reference_accu_and_matmul_arguments():
    b = _backend()
    ctx = fusemat.Context(b)
    X = fusemat.zeros(30, 20, "f32", ctx)
    Y = fusemat.zeros(20, 7, "f32", ctx)
    X2 = fusemat.zeros(30, 20, "f32", ctx)
    fusemat.accu(X * X2)                       # dot's signature: an AOT template
    (kid, prog, out, rows, cols, fin, _), = _launches(b, "fm_launch_accu")
    assert (rows, cols, fin) == (30, 20, 0) and kid >= 0
    Z = fusemat.zeros(30, 7, "f32", ctx)
    Z.assign(X @ Y)
    (g, _), = _launches(b, "fm_gemm")
    g = g._obj
    assert (g.m, g.n, g.k, g.lda, g.ldb, g.ldc) == (30, 7, 20, 30, 20, 30)
    assert (g.trans_a, g.trans_b, g.alpha) == (0, 0, 1.0)
    assert (g.a, g.b, g.c) == (b.ptr(X.handle), b.ptr(Y.handle), b.ptr(Z.handle))


def test_reference_schema_violation_raises_schema_error():
    b = _backend()
    ctx = fusemat.Context(b)
    X = fusemat.zeros(4, 4, "f32", ctx)
    from fusemat import codegen
    k = b.compile(codegen.generate_kernel_source((X + X).node, "copy"))
    with pytest.raises(bk.SchemaError):
        b.launch(k, [X.handle, 4, 4], (4, 4))
    with pytest.raises(bk.SchemaError):
        b.launch(k, [X.handle, 4, 4, X.handle, 4, 4], (4, 5))


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_reference_suite_plumbs_through(etype):
    """Every member of the reference's 13-expression suite (bench.py:91-201)
    compiles and binds on B200Backend: one fused launch per MatMul-free
    subtree, GEMMs for the chain."""
    from fusemat import bench as rbench
    for name in rbench.SUITE:
        b = _backend()
        ctx = fusemat.Context(b)
        out, e = rbench.build_expression(rbench.BenchSpec(expr_name=name, n=16, etype=etype), ctx)
        out.assign(e)
        fused = len(_launches(b, "fm_launch_copy"))
        gemms = len(_launches(b, "fm_gemm"))
        assert (fused, gemms) == ((0, 3) if name == "chain" else (1, 0)), name
