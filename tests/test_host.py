"""Host-side logic on CPU: expression trees, signatures (byte-compatible with
the reference), planning (fusion extent, GEMM folding, reductions, aliasing)
and lowering to the fused program.  Mirrors the reference's test_expr.py /
test_plan.py / test_codegen.py."""

import pytest

from paper_2604_22242_b200 import exprtree as ast
from paper_2604_22242_b200 import lower, plan as P
from paper_2604_22242_b200.aot_registry import hot_expressions, registered_signatures
from paper_2604_22242_b200.backend import arg_schema
from paper_2604_22242_b200.errors import GenerationError, OutOfBoundsError, ShapeError
from paper_2604_22242_b200.exprtree import ElemType, MatShape
from treeio import from_json

F32, F64 = ElemType.f32, ElemType.f64
OUT = 999


def L(i, r=8, c=8, t=F32):
    return ast.leaf(i, t, MatShape(r, c))


# --- signatures & schemas match the reference byte for byte ------------------------------
def test_signatures_match_reference(golden_signatures):
    for row in golden_signatures:
        node = from_json(row["tree"])
        assert ast.signature_of(node) == row["signature"], row["name"]
        if "qualified_copy" in row:
            assert P.qualified_signature(node, P.COPY) == row["qualified_copy"]
            assert P.qualified_signature(node, P.REDUCE_ACCU) == row["qualified_accu"]
            assert [str(a) for a in arg_schema(node, P.COPY)] == row["schema_copy"]
            assert [str(a) for a in arg_schema(node, P.REDUCE_ACCU)] == row["schema_accu"]
        inputs, slots = ast.collect_inputs(node)
        assert [s.mat_id for s in inputs] == row["inputs"]
        assert [s.value for s in slots] == row["slots"]


def test_signature_ignores_scalars_and_ids():
    a = ast.scalar_add(L(0), 3.0)
    b = ast.scalar_add(L(7), 5.0)
    assert ast.signature_of(a) == ast.signature_of(b)
    assert ast.signature_of(ast.plus(L(0), L(0))) != ast.signature_of(ast.plus(L(0), L(1)))


def test_conformability_and_types():
    with pytest.raises(ShapeError):
        ast.plus(L(0, 2, 2), L(1, 2, 3))
    with pytest.raises(ShapeError):
        ast.plus(L(0), L(1, t=F64))
    with pytest.raises(ShapeError):
        ast.exp(L(0, t=ElemType.i32))
    with pytest.raises(ShapeError):
        ast.pow_int(L(0), 17)
    with pytest.raises(OutOfBoundsError):
        ast.subview(0, F32, 3, 0, MatShape(2, 2), MatShape(4, 4))
    with pytest.raises(ShapeError):
        ast.scalar_add(L(0, t=ElemType.i32), 1.5)
    assert ast.matmul(L(0, 4, 3, ElemType.bf16), L(1, 3, 5, ElemType.bf16)).etype is F32
    assert ast.reduce(ast.ReduceKind.index_max, 0, L(0, 5, 7)).shape == MatShape(1, 7)
    assert ast.reduce(ast.ReduceKind.sum, 1, L(0, 5, 7)).shape == MatShape(5, 1)
    with pytest.raises(ShapeError):
        ast.reduce(ast.ReduceKind.mean, 0, L(0, t=ElemType.u32))


# --- planning ----------------------------------------------------------------------------------
def test_elementwise_is_one_step():
    pl = P.plan(OUT, ast.plus(L(0), L(1)))
    assert len(pl.steps) == 1 and pl.steps[0].out_id == OUT and not pl.temps


def test_c5_gemm_folds_scalar_and_transpose_into_one_launch():
    X, Y = L(0, 64, 32), L(1, 48, 32)
    node = ast.matmul(ast.scalar_pre_mul(2, X), ast.transpose(Y))   # 2 * X @ Y.t()
    pl = P.plan(OUT, node)
    assert len(pl.steps) == 1 and not pl.temps
    g = pl.steps[0]
    assert isinstance(g, P.GemmStep)
    assert (g.a_id, g.b_id, g.trans_a, g.trans_b, g.alpha) == (0, 1, False, True, 2.0)
    assert (g.m, g.n, g.k) == (64, 48, 32) and g.out_id == OUT


def test_gemm_operand_expression_is_a_prologue():
    """An elementwise operand is not materialised (the reference's temp,
    plan.py:125-151): it becomes the GEMM's prologue program over its stored
    shape, the transpose still folded into the product."""
    node = ast.matmul(ast.transpose(ast.plus(L(0, 4, 8), L(1, 4, 8))), L(2, 4, 2))
    pl = P.plan(OUT, node)
    assert len(pl.fused_steps) == 0 and len(pl.gemm_steps) == 1 and not pl.temps
    g = pl.gemm_steps[0]
    assert g.trans_a and g.a_id is None and g.b_id == 2
    assert g.a_expr.out_shape == MatShape(4, 8)              # no transpose copy
    assert sorted(s.mat_id for s in g.a_expr.inputs) == [0, 1]


def test_gemm_prologue_keeps_inner_barriers():
    """A reduction / product inside the operand is still its own launch; the
    rest of the operand rides in the GEMM."""
    inner = ast.matmul(L(0, 4, 3), L(1, 3, 8))
    node = ast.matmul(ast.plus(inner, L(2, 4, 8)), L(3, 8, 2))
    pl = P.plan(OUT, node)
    assert len(pl.gemm_steps) == 2 and len(pl.fused_steps) == 0
    assert pl.gemm_steps[1].a_expr is not None


def test_chain_three_gemms_left_to_right():
    a, b, c, d = L(0, 16, 8), L(1, 8, 4), L(2, 4, 2), L(3, 2, 1)
    pl = P.plan(OUT, ast.matmul(ast.matmul(ast.matmul(a, b), c), d))
    assert len(pl.gemm_steps) == 3 and pl.gemm_steps[-1].out_id == OUT and len(pl.temps) == 2


def test_alias_handling():
    assert not P.plan(OUT, ast.plus(L(OUT), L(1))).out_is_temp
    pl = P.plan(OUT, ast.plus(ast.transpose(L(OUT)), L(1)))
    assert pl.out_is_temp and len(pl.fused_steps) == 1
    assert P.plan(OUT, ast.matmul(L(OUT), L(1))).out_is_temp


def test_reduce_root_single_step_and_multi_output_fusion():
    e = ast.schur(ast.minus(L(0, t=F64), L(1, t=F64)), L(2, t=F64))
    outs = [(10, ast.reduce(ast.ReduceKind.sum, 0, e)), (11, ast.reduce(ast.ReduceKind.mean, 0, e)),
            (12, ast.reduce(ast.ReduceKind.max, 0, e)), (13, ast.reduce(ast.ReduceKind.index_max, 0, e))]
    pl = P.plan_many(outs)
    assert len(pl.steps) == 1
    assert [o.out_id for o in pl.steps[0].reductions] == [10, 11, 12, 13]
    # different dims do not fuse
    pl2 = P.plan_many(outs[:1] + [(14, ast.reduce(ast.ReduceKind.sum, 1, e))])
    assert len(pl2.steps) == 2


def test_reduce_inside_expression_is_a_barrier():
    r = ast.reduce(ast.ReduceKind.sum, 0, L(0, 4, 6))
    pl = P.plan(OUT, ast.scalar_add(r, 1.0))
    assert len(pl.steps) == 2 and pl.steps[0].skeleton == P.REDUCE_DIM


# --- lowering ----------------------------------------------------------------------------------
def test_c1_program():
    node = ast.plus(ast.scalar_pre_mul(2, ast.schur(L(0), L(1))), L(0))
    p = lower.lower(node)
    assert p.flat and p.depth == 1 and len(p.slots) == 2
    # leaves evaluated second are slot operands of their binary op
    assert p.disassemble() == ["PUSH32@0 0", "MUL_F_S@0 1", "SMUL_F@0 0", "ADD_F_S@0 0"]


def test_sethi_ullman_keeps_deep_trees_shallow():
    leaves = [L(i % 8) for i in range(64)]
    while len(leaves) > 1:                       # balanced 64-leaf tree needs 7 registers
        leaves = [ast.minus(leaves[i], leaves[i + 1]) for i in range(0, len(leaves), 2)]
    p = lower.lower(leaves[0])
    assert p.depth == 6                          # the last level's right leaves are slot operands
    chain = L(0)
    for i in range(1, 40):                       # left-deep addN needs 1 (PUSH, then ADD_F_S ...)
        chain = ast.plus(chain, L(i))
    assert lower.lower(chain).depth == 1


def test_right_heavy_subtraction_uses_reversed_opcode():
    node = ast.minus(L(0), ast.plus(L(1), L(2)))
    p = lower.lower(node)
    assert p.disassemble()[-1] == "RSUB_F_S@0 0"     # (L1 + L2) first, then L0 as a slot operand
    node = ast.minus(ast.plus(L(0), L(1)), ast.plus(L(2), L(3)))
    assert lower.lower(node).disassemble()[-1] == "SUB_F@0 0"


def test_views_and_transposes_are_not_flat():
    sv = ast.subview(0, F32, 1, 1, MatShape(4, 4), MatShape(8, 8))
    assert not lower.lower(ast.plus(sv, L(1, 4, 4))).flat
    assert not lower.lower(ast.plus(ast.transpose(L(0)), L(1))).flat


def test_lowering_limits():
    big = L(0)
    for i in range(1, 45):
        big = ast.plus(big, L(i))
    with pytest.raises(GenerationError):
        lower.lower(big)


def _addn(n, t=F32):
    e = L(0, t=t)
    for i in range(1, n):
        e = ast.plus(e, L(i, t=t))
    return e


@pytest.mark.parametrize("n", [32, 33, 40, 41, 48, 64, 200])
def test_planner_splits_trees_past_the_program_limits(n):
    """add-N for any N (reference bench.py:307-326 sweeps it unbounded): the
    planner cuts the tree into launches of at most PLAN_SLOTS (32, the widest
    AOT template) leaf reads, materialising sub-sums into temps; every input
    is read exactly once."""
    pl = P.plan(OUT, _addn(n))
    steps = pl.fused_steps
    k = P.PLAN_SLOTS
    assert len(steps) == -(-(n - 1) // (k - 1)) if n > k else len(steps) == 1
    reads = []
    for st in steps:
        prog = lower.lower(st.expr)                      # each launch lowers
        assert len(prog.slots) <= k <= lower.MAX_SLOTS
        reads += [s.mat_id for s in st.inputs if s.mat_id >= 0]
    assert sorted(reads) == list(range(n))
    assert steps[-1].out_id == OUT
    temps = {t.temp_id for t in pl.temps}
    for st in steps[:-1]:
        assert st.out_id in temps


def test_planner_splits_on_scalar_count():
    e = L(0)
    for i in range(40):
        e = ast.scalar_add(e, float(i))           # 40 scalars > MAX_SCALARS
    pl = P.plan(OUT, e)
    assert len(pl.fused_steps) == 2
    for st in pl.fused_steps:
        assert len(lower.lower(st.expr).scalars) <= lower.MAX_SCALARS


def test_plan_many_rejects_outputs_read_by_the_batch():
    from paper_2604_22242_b200.errors import PlanError
    X, Y = L(0), L(1)
    red = lambda k, n: ast.reduce(k, 0, n)  # noqa: E731
    with pytest.raises(PlanError):
        P.plan_many([(10, red(ast.ReduceKind.sum, X)), (0, ast.scalar_add(Y, 1.0)),
                      (11, red(ast.ReduceKind.max, X))])
    with pytest.raises(PlanError):
        P.plan_many([(10, red(ast.ReduceKind.sum, X)), (10, red(ast.ReduceKind.max, X))])
    pl = P.plan_many([(10, red(ast.ReduceKind.sum, X)), (11, red(ast.ReduceKind.max, X))])
    assert len(pl.steps) == 1


def test_bf16_nodes_round_after_every_op():
    x = L(0, t=ElemType.bf16)
    p = lower.lower(ast.plus(ast.scalar_pre_mul(2.5, x), x))
    assert [s.split("@")[0] for s in p.disassemble()].count("RND_BF_F") == 2


def test_aot_registry_covers_the_configs():
    sigs = set(registered_signatures())
    X, Y, Z = L(0), L(1), L(2)
    c1 = ast.plus(ast.scalar_pre_mul(2, ast.schur(X, Y)), X)
    c3 = ast.plus(ast.exp(ast.scalar_pre_mul(0.5, ast.neg(ast.square(ast.minus(X, Y))))),
                  ast.scalar_pre_mul(0.5, ast.abs_(X)))
    X64, Y64, Z64 = L(0, t=F64), L(1, t=F64), L(2, t=F64)
    for n in (c1, c3, ast.schur(X, Y), ast.square(ast.minus(X, Y)),
              ast.schur(ast.minus(X64, Y64), Z64), ast.schur(X64, Y64)):
        assert ast.signature_of(n) in sigs
    assert len(hot_expressions()) == len(sigs)


# --- host-path memoisation ---------------------------------------
def test_plan_and_bind_memo():
    from recording import launches, recording_backend
    import paper_2604_22242_b200 as fm
    from paper_2604_22242_b200.errors import BackendError
    b = recording_backend()
    ctx = fm.Context(b)
    X, Y, Z = fm.Mat(64, 32, "f32", ctx), fm.Mat(64, 32, "f32", ctx), fm.Mat(64, 32, "f32", ctx)
    e = 2 * (X % Y) + X
    Z.assign(e)
    p1 = ctx.plan_for(Z.mat_id, e.node)
    Z.assign(e)
    assert ctx.plan_for(Z.mat_id, e.node) is p1            # same expression object: memoised plan
    progs = [a[1]._obj for a in launches(b, "fm_launch_copy")]
    assert progs[0] is progs[1]                           # same arguments: bound program re-used
    e2 = 2 * (X % Y) + X
    assert ctx.plan_for(Z.mat_id, e2.node) is not p1      # a new tree plans afresh
    X._realloc(X.shape)                                   # new buffer: re-bound
    Z.assign(e)
    assert launches(b, "fm_launch_copy")[-1][1]._obj is not progs[0]
    old = Y.handle
    b.free(old)
    Y._set_handle(b.alloc(Y.etype, Y.n_elem))
    k = ctx.cache.lookup(p1.steps[0].signature)
    with pytest.raises(BackendError):                     # memo never bypasses the UAF check
        b.launch(k, [Z.handle, 64, 32, X.handle, 64, 32, old, 64, 32, 2.0], (64, 32))


def test_bench_dominant_kernel_families():
    """bench.py's roofline kernel: launches of one kernel form a family; a
    step made only of that family takes its launch time from the step events
    (no events between launches); a mixed step from the instrumented pass."""
    import bench
    # C1-like: six launches of one kernel, instrumented times inflated by events
    labels = [f"c1[{i}]" for i in range(6)]
    per = [[0.036, 0.036] for _ in range(6)]
    d = bench.dominant_kernel(labels, [100] * 6, per, [0.18, 0.18])
    assert d["kernel"] == "c1" and d["launches_per_step"] == 6
    assert abs(d["mean_launch_ms"] - 0.03) < 1e-12 and d["work_per_launch"] == 100
    # mixed step: the family with the largest instrumented share wins
    labels = ["a", "b[0]", "b[1]", "gather"]
    per = [[1.0, 1.0], [0.8, 0.8], [0.8, 0.8], [0.1, 0.1]]
    d = bench.dominant_kernel(labels, [10, 20, 20, 0], per, [2.5, 2.5])
    assert d["kernel"] == "b" and d["first_label"] == "b[0]" and d["launches_per_step"] == 2
    assert abs(d["mean_launch_ms"] - 0.8) < 1e-12 and d["work_per_step"] == 40
    assert abs(d["share_of_step_ms"] - 2.5 * 3.2 / 5.4) < 1e-12
