"""Execution planning: fused launches, folded GEMMs and reduction roots.

Follows the reference planner (`/root/reference/pkg/src/fusemat/plan.py:113-215`):
every maximal MatMul-free subtree becomes exactly one fused launch, real
matrices keep their non-negative ids, temporaries get fresh negative ids and an
unsafe alias lands in a temp the caller swaps in.  B200-specific changes:

* `MatMul(s * A, B.t())`-style operands are folded into ONE `GemmStep`: scalar
  pre-multiplies become `alpha` and transposes become operand major-ness
  (the reference emits two copy kernels plus a GEMM, `plan.py:125-151`).
  Only operands that are not (scaled, transposed) dense leaves are
  materialised.
* `Reduce` roots plan to a single `FusedKernelStep` with a dim-reduction
  skeleton; several reductions of the same subexpression can share one launch
  (`plan_many`).
* `reduce_plan` (accu) is unchanged: a 1x1 accumulator temp of
  `accumulator_type` (`plan.py:208-215`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import lower as lw
from .errors import GenerationError, PlanError
from .exprtree import (
    SCALAR_KINDS, AliasKind, BinaryElem, BinaryKind, Diag, ElemType, ExprNode, InputSpec, Leaf,
    MatMul, MatShape, Reduce, ReduceKind, ScalarSlot, Subview, Transpose, UnaryElem,
    UnaryKind, aliases, collect_inputs, signature_of, walk,
)

COPY = "copy"
REDUCE_ACCU = "reduce_accu"
REDUCE_DIM = "reduce_dim"

# accu finalisers (applied once to the f64 total inside the last block)
FINAL_NONE = 0
FINAL_SQRT = 1


def accumulator_type(etype: ElemType) -> ElemType:
    """f64 for floats, modular native type for ints (`codegen.py:47-49`)."""
    return ElemType.f64 if etype.is_float else etype


def qualified_signature(node: ExprNode, skeleton_kind: str) -> str:
    """`skeleton|signature`, the reference cache key (`codegen.py:268-270`)."""
    return f"{skeleton_kind}|{signature_of(node)}"


@dataclass
class ReduceOutput:
    kind: ReduceKind
    out_id: int
    etype: ElemType


@dataclass
class FusedKernelStep:
    """One fused launch over a MatMul-free subtree."""

    expr: ExprNode
    skeleton: str
    out_id: int
    out_shape: MatShape
    out_etype: ElemType
    domain_shape: MatShape
    signature: str
    inputs: list[InputSpec]
    scalars: list[ScalarSlot]
    dim: int = 0
    reductions: list[ReduceOutput] = field(default_factory=list)
    finalize: int = FINAL_NONE

    @classmethod
    def create(cls, expr: ExprNode, skeleton: str, out_id: int,
               finalize: int = FINAL_NONE) -> "FusedKernelStep":
        inputs, scalars = collect_inputs(expr)
        if skeleton == REDUCE_ACCU:
            out_shape, out_etype = MatShape(1, 1), accumulator_type(expr.etype)
        else:
            out_shape, out_etype = expr.shape, expr.etype
        sig = qualified_signature(expr, skeleton)
        if finalize != FINAL_NONE:
            sig += f"|final{finalize}"
        return cls(expr, skeleton, out_id, out_shape, out_etype, expr.shape, sig,
                   inputs, scalars, finalize=finalize)

    @classmethod
    def create_reduce(cls, child: ExprNode, dim: int,
                      outputs: list[ReduceOutput]) -> "FusedKernelStep":
        inputs, scalars = collect_inputs(child)
        shape = MatShape(1, child.shape.n_cols) if dim == 0 else MatShape(child.shape.n_rows, 1)
        kinds = ",".join(o.kind.value for o in outputs)
        sig = f"{REDUCE_DIM}{{{dim}:{kinds}}}|{signature_of(child)}"
        first = outputs[0]
        return cls(child, REDUCE_DIM, first.out_id, shape, first.etype, child.shape, sig,
                   inputs, scalars, dim=dim, reductions=list(outputs))


@dataclass
class GemmStep:
    """out = alpha * op(A) @ op(B); op = transpose when the flag is set.
    `a_shape`/`b_shape` are the STORED shapes of the dense operand buffers."""

    a_id: int
    b_id: int
    out_id: int
    a_shape: MatShape
    b_shape: MatShape
    trans_a: bool
    trans_b: bool
    alpha: float
    in_etype: ElemType
    out_etype: ElemType
    out_shape: MatShape
    # epilogue: out = alpha2 * (alpha * A@B) + beta * C, each op rounded to
    # out_etype -- the elementwise step after the product, folded in
    c_id: int | None = None
    alpha2: float = 1.0
    beta: float = 0.0
    # prologue: an operand that is a MatMul-free elementwise expression is
    # not materialised (the reference's plan.py:125-151 temp); its fused
    # program runs inside the GEMM's operand pass (fm_gemm_prologue).  The
    # step's a_id / b_id is then None and a_shape / b_shape the expression's.
    a_expr: "FusedKernelStep | None" = None
    b_expr: "FusedKernelStep | None" = None

    @property
    def m(self) -> int:
        return self.out_shape.n_rows

    @property
    def n(self) -> int:
        return self.out_shape.n_cols

    @property
    def k(self) -> int:
        return self.a_shape.n_rows if self.trans_a else self.a_shape.n_cols

    @property
    def left_id(self) -> int:          # reference MatMulStep field names
        return self.a_id

    @property
    def right_id(self) -> int:
        return self.b_id


# The reference's plain product step is a GemmStep with no folding.
MatMulStep = GemmStep


@dataclass
class TempSpec:
    temp_id: int
    shape: MatShape
    etype: ElemType


@dataclass
class ExecutionPlan:
    steps: list
    temps: list[TempSpec]
    out_id: int
    out_shape: MatShape
    out_etype: ElemType
    out_is_temp: bool = False

    @property
    def fused_steps(self) -> list[FusedKernelStep]:
        return [s for s in self.steps if isinstance(s, FusedKernelStep)]

    @property
    def gemm_steps(self) -> list[GemmStep]:
        return [s for s in self.steps if isinstance(s, GemmStep)]

    matmul_steps = gemm_steps

    def n_launches(self) -> int:
        return len(self.steps)


class _Planner:
    def __init__(self) -> None:
        self.steps: list = []
        self.temps: list[TempSpec] = []
        self._next = -1

    def temp(self, shape: MatShape, etype: ElemType) -> TempSpec:
        t = TempSpec(self._next, shape, etype)
        self._next -= 1
        self.temps.append(t)
        return t

    def materialize(self, node: ExprNode) -> Leaf:
        node = self.fused(node)
        if isinstance(node, Leaf):
            return node
        t = self.temp(node.shape, node.etype)
        self.steps.append(FusedKernelStep.create(node, COPY, t.temp_id))
        return Leaf(t.temp_id, node.etype, node.shape)

    def gemm_operand(self, node: ExprNode) -> tuple[ExprNode, bool, float]:
        """Peel scalar pre-multiplies and transposes off a product operand;
        what remains is a dense leaf (used in place), a fused elementwise
        expression (the GEMM's prologue, f32 / f64 operands), or gets
        materialised."""
        alpha, trans = 1.0, False
        while True:
            if isinstance(node, UnaryElem) and node.kind is UnaryKind.scalar_pre_mul:
                alpha *= float(node.scalar)
                node = node.child
            elif isinstance(node, Transpose):
                trans = not trans
                node = node.child
            else:
                break
        node = self.fused(node)
        if isinstance(node, Leaf) or node.etype in (ElemType.f32, ElemType.f64):
            return node, trans, alpha
        return self.materialize(node), trans, alpha

    def gemm(self, node: MatMul, out_id: int | None = None) -> GemmStep:
        a, ta, sa = self.gemm_operand(node.left)
        b, tb, sb = self.gemm_operand(node.right)
        if out_id is None:
            out_id = self.temp(node.shape, node.etype).temp_id
        a_expr = None if isinstance(a, Leaf) else FusedKernelStep.create(a, COPY, out_id)
        b_expr = None if isinstance(b, Leaf) else FusedKernelStep.create(b, COPY, out_id)
        step = GemmStep(a.mat_id if a_expr is None else None, b.mat_id if b_expr is None else None,
                        out_id, a.shape, b.shape, ta, tb, sa * sb, a.etype, node.etype, node.shape,
                        a_expr=a_expr, b_expr=b_expr)
        self.steps.append(step)
        return step

    def fused(self, node: ExprNode) -> ExprNode:
        """The MatMul/Reduce-free root of one fused launch: barriers split out
        (`split`) and the rest cut to the AOT kernels' program limits (`fit`)."""
        return self.fit(self.split(node))

    # -- program limits -------------------------------------------------------------
    # One fused launch executes one fm_program: at most MAX_SLOTS leaf
    # accesses, MAX_INSTR instructions, MAX_SCALARS scalars, MAX_DEPTH stack
    # registers (include/fmb200.h).  The reference compiles any tree into one
    # C function (codegen.py:338-391); here a tree past the limits is cut
    # bottom-up: whenever a node no longer lowers, its largest non-leaf child
    # (which does, by induction) is materialised into a temp of its own
    # element type -- bit-identical, since every node already rounds to its
    # type -- and read back as a dense leaf.

    def fit(self, node: ExprNode) -> ExprNode:
        if _fits(node):
            return node
        return self._fit(node)

    def _fit(self, node: ExprNode) -> ExprNode:
        if isinstance(node, (Leaf, Subview, Diag)):
            return node
        kids = [self._fit(c) for c in node.children()]
        cur = _rebuild(node, kids)
        while not _fits(cur):
            cands = [i for i, c in enumerate(kids) if not isinstance(c, (Leaf, Subview, Diag))]
            if not cands:
                # only leaves left and still too big: cannot happen within the
                # limits (a binary node reads <= 2 leaves), kept as a guard
                raise PlanError(f"cannot split {type(node).__name__} below the fused-program limits")
            i = max(cands, key=lambda j: _size(kids[j]))
            t = self.temp(kids[i].shape, kids[i].etype)
            self.steps.append(FusedKernelStep.create(kids[i], COPY, t.temp_id))
            kids[i] = Leaf(t.temp_id, kids[i].etype, kids[i].shape)
            cur = _rebuild(node, kids)
        return cur

    def split(self, node: ExprNode) -> ExprNode:
        """Replace every MatMul / Reduce subtree with a dense temp leaf."""
        if isinstance(node, MatMul):
            step = self.gemm(node)
            return Leaf(step.out_id, node.etype, node.shape)
        if isinstance(node, Reduce):
            child = self.fused(node.child)
            t = self.temp(node.shape, node.etype)
            self.steps.append(FusedKernelStep.create_reduce(
                child, node.dim, [ReduceOutput(node.kind, t.temp_id, node.etype)]))
            return Leaf(t.temp_id, node.etype, node.shape)
        if isinstance(node, (Leaf, Subview, Diag)):
            return node
        if isinstance(node, UnaryElem):
            c = self.split(node.child)
            if c is node.child:
                return node
            return UnaryElem(node.kind, c, scalar=node.scalar, exponent=node.exponent,
                             target=node.target)
        if isinstance(node, BinaryElem):
            a, b = self.split(node.left), self.split(node.right)
            if a is node.left and b is node.right:
                return node
            return BinaryElem(node.kind, a, b)
        if isinstance(node, Transpose):
            c = self.split(node.child)
            return node if c is node.child else Transpose(c)
        raise PlanError(f"cannot plan node {type(node).__name__}")


def _size(node: ExprNode) -> int:
    return sum(1 for _ in walk(node))


# Leaf reads per launch the planner aims for: the widest ahead-of-time
# template (aot_registry: the add-N chains up to 32 inputs).  A 33..40-leaf
# program still lowers, but only onto the register VM, which streams many-leaf
# chains at a third of the template rate (r02 suite: add48N 1.86 TB/s as a
# 40-leaf VM launch + add9N, vs add32N 5.97); cutting at 32 costs one temp
# write + read per 32 leaves (~6 % traffic) and keeps every piece on a template.
PLAN_SLOTS = 32


def _fits(node: ExprNode) -> bool:
    """Does `node` lower within the fused-program limits (and the planner's
    PLAN_SLOTS leaf budget)?  Cheap bound first (every node emits at most two
    instructions), the real lowering otherwise."""
    n = leaves = scalars = 0
    for x in walk(node):
        n += 1
        if isinstance(x, (Leaf, Subview, Diag)):
            leaves += 1
        elif isinstance(x, UnaryElem) and x.kind in SCALAR_KINDS:
            scalars += 1
    if leaves > PLAN_SLOTS:
        return False
    if 2 * n <= lw.MAX_INSTR and scalars <= lw.MAX_SCALARS:
        return True
    try:
        lw.lower(node)
        return True
    except GenerationError:
        return False


def _rebuild(node: ExprNode, kids: list) -> ExprNode:
    old = node.children()
    if all(a is b for a, b in zip(old, kids)):
        return node
    if isinstance(node, UnaryElem):
        return UnaryElem(node.kind, kids[0], scalar=node.scalar, exponent=node.exponent,
                         target=node.target)
    if isinstance(node, BinaryElem):
        return BinaryElem(node.kind, kids[0], kids[1])
    if isinstance(node, Transpose):
        return Transpose(kids[0])
    raise PlanError(f"cannot rebuild node {type(node).__name__}")


def _scaled(node: ExprNode) -> tuple[ExprNode, float]:
    """Peel scalar pre-multiplies: node = s * rest."""
    s = 1.0
    while isinstance(node, UnaryElem) and node.kind is UnaryKind.scalar_pre_mul:
        s *= float(node.scalar)
        node = node.child
    return node, s


def _product_epilogue(node: ExprNode):
    """`s2 * (A @ B) (+|-) sb * C` -> (MatMul, alpha2, C leaf, beta), or None.

    Folds the elementwise step the reference runs as a separate fused launch
    after its MatMulStep into the GEMM epilogue.  Only an f32/f64 product with
    a dense same-shape addend of the output type folds; the epilogue rounds
    alpha2*T, beta*C and their sum to the output type, as the reference's
    copy kernel would (one scalar node per multiply)."""
    if not isinstance(node, BinaryElem) or node.kind not in (BinaryKind.plus, BinaryKind.minus):
        return None
    for prod_side, add_side, sign in ((node.left, node.right, 1.0), (node.right, node.left, None)):
        mm, s2 = _scaled(prod_side)
        if not isinstance(mm, MatMul):
            continue
        leaf, sb = _scaled(add_side)
        if not isinstance(leaf, Leaf) or leaf.shape != mm.shape or leaf.etype is not mm.etype:
            continue
        if mm.etype not in (ElemType.f32, ElemType.f64):
            continue
        if node.kind is BinaryKind.plus:
            return mm, s2, leaf, sb
        # minus: left - right
        if sign is not None:            # (s2*AB) - sb*C
            return mm, s2, leaf, -sb
        return mm, -s2, leaf, sb        # sb*C - s2*AB
    return None


def plan(out_mat_id: int, node: ExprNode) -> ExecutionPlan:
    """Plan `out = node` (`plan.py:171-205` semantics plus folding)."""
    p = _Planner()
    unsafe = aliases(out_mat_id, node) is AliasKind.UNSAFE

    # s * (A @ B) at the root: the scale joins the product's epilogue
    inner, s_root = _scaled(node)
    if isinstance(inner, MatMul) and inner is not node and inner.etype in (ElemType.f32, ElemType.f64):
        unsafe_mm = aliases(out_mat_id, inner) is AliasKind.UNSAFE
        target = p.temp(inner.shape, inner.etype).temp_id if unsafe_mm else out_mat_id
        step = p.gemm(inner, target)
        step.alpha *= s_root            # one scale on the accumulator (the reference rounds T first)
        return ExecutionPlan(p.steps, p.temps, target, inner.shape, inner.etype, out_is_temp=unsafe_mm)

    ep = _product_epilogue(node)
    if ep is not None:
        mm, s2, c_leaf, beta = ep
        # the product's operands must not alias the output; the addend may (read then written
        # by the same thread)
        if aliases(out_mat_id, mm) is not AliasKind.UNSAFE:
            step = p.gemm(mm, out_mat_id)
            step.c_id, step.alpha2, step.beta = c_leaf.mat_id, s2, beta
            return ExecutionPlan(p.steps, p.temps, out_mat_id, node.shape, node.etype)

    if isinstance(node, MatMul):
        target = p.temp(node.shape, node.etype).temp_id if unsafe else out_mat_id
        p.gemm(node, target)
        return ExecutionPlan(p.steps, p.temps, target, node.shape, node.etype,
                             out_is_temp=unsafe)

    if isinstance(node, Reduce):
        child = p.fused(node.child)
        target = p.temp(node.shape, node.etype).temp_id if unsafe else out_mat_id
        p.steps.append(FusedKernelStep.create_reduce(
            child, node.dim, [ReduceOutput(node.kind, target, node.etype)]))
        return ExecutionPlan(p.steps, p.temps, target, node.shape, node.etype,
                             out_is_temp=unsafe)

    root = p.fused(node)
    if unsafe:
        t = p.temp(root.shape, root.etype)
        p.steps.append(FusedKernelStep.create(root, COPY, t.temp_id))
        return ExecutionPlan(p.steps, p.temps, t.temp_id, root.shape, root.etype,
                             out_is_temp=True)
    p.steps.append(FusedKernelStep.create(root, COPY, out_mat_id))
    return ExecutionPlan(p.steps, p.temps, out_mat_id, root.shape, root.etype)


def reduce_plan(node: ExprNode, finalize: int = FINAL_NONE) -> ExecutionPlan:
    """Full reduction into a 1x1 accumulator temp (`plan.py:208-215`)."""
    p = _Planner()
    root = p.fused(node)
    acc = p.temp(MatShape(1, 1), accumulator_type(root.etype))
    p.steps.append(FusedKernelStep.create(root, REDUCE_ACCU, acc.temp_id, finalize))
    return ExecutionPlan(p.steps, p.temps, acc.temp_id, acc.shape, acc.etype,
                         out_is_temp=True)


def _binding_key(node: ExprNode):
    """Structure plus concrete bindings: two reductions can share a launch iff
    they read the same matrices through the same maps with the same scalars."""
    inputs, scalars = collect_inputs(node)
    return (signature_of(node),
            tuple((s.mat_id, tuple((v.kind, v.row_off, v.col_off) for v in s.views))
                  for s in inputs),
            tuple((type(s.value), repr(s.value)) for s in scalars))


def plan_many(assignments: list[tuple[int, ExprNode]]) -> ExecutionPlan:
    """Plan several assignments together.  Reduce roots along the same dim of
    the same bound subexpression fuse into one multi-output launch (C4's
    sum/mean/max/index_max read X, Y, Z once); everything else plans as
    `plan` would, in order.  No output may be an input of ANY assignment in
    the batch (a grouped reduction is hoisted to its group's first position,
    so a write between two members would otherwise change what the later
    ones read), and no matrix may be written twice."""
    p = _Planner()
    groups: dict = {}
    order: list = []
    outs_seen: set = set()
    read: set = set()
    for out_id, node in assignments:
        if out_id in outs_seen:
            raise PlanError(f"plan_many writes matrix {out_id} twice")
        outs_seen.add(out_id)
        read.update(spec.mat_id for spec in collect_inputs(node)[0])
    clash = outs_seen & read
    if clash:
        raise PlanError(f"plan_many outputs may not be read by the batch (matrices {sorted(clash)})")
    for out_id, node in assignments:
        if isinstance(node, Reduce):
            key = (node.dim, _binding_key(node.child))
            if key not in groups:
                groups[key] = (node, [])
                order.append(key)
            groups[key][1].append(ReduceOutput(node.kind, out_id, node.etype))
        else:
            order.append((out_id, node))
    for item in order:
        if item in groups:
            node, outs = groups[item]
            child = p.fused(node.child)
            p.steps.append(FusedKernelStep.create_reduce(child, node.dim, outs))
        else:
            out_id, node = item
            if isinstance(node, MatMul):
                p.gemm(node, out_id)
            else:
                root = p.fused(node)
                p.steps.append(FusedKernelStep.create(root, COPY, out_id))
    last = assignments[-1]
    return ExecutionPlan(p.steps, p.temps, last[0], last[1].shape, last[1].etype)
