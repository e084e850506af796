"""Lazy expression trees (the Op / eOp / eGlue layer of the paper).

Semantics follow the reference AST in `/root/reference/pkg/src/fusemat/expr.py`:
node kinds and their value strings (`expr.py:85-115`), conformability rules
(`expr.py:210-295`), scalar coercion (`expr.py:298-304`), the structural
signature (`expr.py:412-452`), first-visit input collection (`expr.py:488-523`)
and alias classification (`expr.py:532-556`).  Differences are additions only:

* `ElemType.bf16` (16-bit storage, f32 arithmetic rounded per node);
* `UnaryKind.abs`;
* `Reduce` roots (sum / mean / max / min / index_max / index_min along a
  dimension), which the reference does not have.

A tree describes work; nothing executes until the planner lowers it.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np

from .errors import OutOfBoundsError, ShapeError


class ElemType(enum.Enum):
    f32 = "f32"
    f64 = "f64"
    u32 = "u32"
    i32 = "i32"
    bf16 = "bf16"

    @property
    def width(self) -> int:
        return _WIDTH[self]

    @property
    def is_float(self) -> bool:
        return self in (ElemType.f32, ElemType.f64, ElemType.bf16)

    @property
    def dtype(self) -> np.dtype:
        """numpy storage dtype (bf16 is stored as raw uint16 bit patterns)."""
        return np.dtype(_NP[self])

    @property
    def host_dtype(self) -> np.dtype:
        """numpy dtype used for values handed back to users."""
        return np.dtype(np.float32) if self is ElemType.bf16 else self.dtype

    @property
    def code(self) -> int:
        """Element-type code of the C ABI (`include/fmb200.h`, FM_F32...)."""
        return _CODE[self]

    @classmethod
    def of(cls, value: "ElemType | str") -> "ElemType":
        if isinstance(value, cls):
            return value
        if not isinstance(value, str) and isinstance(getattr(value, "value", None), str):
            value = value.value     # a foreign enum with the same values (fusemat.expr.ElemType)
        try:
            return cls(value)
        except ValueError:
            raise ShapeError(f"unknown element type {value!r}") from None


_WIDTH = {ElemType.f32: 4, ElemType.f64: 8, ElemType.u32: 4, ElemType.i32: 4, ElemType.bf16: 2}
_NP = {ElemType.f32: np.float32, ElemType.f64: np.float64, ElemType.u32: np.uint32,
       ElemType.i32: np.int32, ElemType.bf16: np.uint16}
_CODE = {ElemType.f32: 0, ElemType.f64: 1, ElemType.u32: 2, ElemType.i32: 3, ElemType.bf16: 4}


# -- bf16 host conversions (round to nearest even, NaN kept quiet) -----------

def f32_to_bf16_bits(values) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(values, dtype=np.float32))
    bits = x.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) >> 16
    nan = np.isnan(x)
    out = rounded.astype(np.uint16)
    out[nan] = ((bits[nan] >> 16) | 0x40).astype(np.uint16)
    return out


def bf16_bits_to_f32(bits) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


def to_storage(values, etype: ElemType) -> np.ndarray:
    """Host array -> the storage representation of `etype` (F order kept by caller)."""
    if etype is ElemType.bf16:
        arr = np.asarray(values)
        if arr.dtype == np.uint16:
            return arr
        return f32_to_bf16_bits(arr.astype(np.float32))
    return np.asarray(values).astype(etype.dtype, copy=False)


def from_storage(values: np.ndarray, etype: ElemType) -> np.ndarray:
    if etype is ElemType.bf16:
        return bf16_bits_to_f32(values)
    return values


@dataclass(frozen=True)
class MatShape:
    n_rows: int
    n_cols: int

    def __post_init__(self) -> None:
        if self.n_rows < 0 or self.n_cols < 0:
            raise ShapeError(f"negative dimension in shape {self.n_rows}x{self.n_cols}")

    @property
    def n_elem(self) -> int:
        return self.n_rows * self.n_cols

    def t(self) -> "MatShape":
        return MatShape(self.n_cols, self.n_rows)

    def __str__(self) -> str:
        return f"{self.n_rows}x{self.n_cols}"


class UnaryKind(enum.Enum):
    scalar_add = "sadd"
    scalar_pre_mul = "smul"
    scalar_pre_div = "sdiv"
    neg = "neg"
    exp = "exp"
    log = "log"
    sqrt = "sqrt"
    tanh = "tanh"
    pow_int = "powi"
    conv = "conv"
    gt_scalar = "gts"
    abs = "abs"          # not in the reference API


class BinaryKind(enum.Enum):
    plus = "add"
    minus = "sub"
    schur = "mul"
    elem_div = "div"


class ReduceKind(enum.Enum):
    sum = "rsum"
    mean = "rmean"
    max = "rmax"
    min = "rmin"
    index_max = "rimax"
    index_min = "rimin"


SCALAR_KINDS = frozenset({UnaryKind.scalar_add, UnaryKind.scalar_pre_mul,
                          UnaryKind.scalar_pre_div, UnaryKind.gt_scalar})
FLOAT_ONLY_KINDS = frozenset({UnaryKind.scalar_pre_div, UnaryKind.exp, UnaryKind.log,
                              UnaryKind.sqrt, UnaryKind.tanh})
MAX_POW_EXPONENT = 16
INDEX_REDUCTIONS = frozenset({ReduceKind.index_max, ReduceKind.index_min})


class ExprNode:
    """Base class; concrete nodes are frozen dataclasses with `shape`/`etype`."""

    shape: MatShape
    etype: ElemType

    def children(self) -> tuple["ExprNode", ...]:
        return ()


def _fix(node, shape: MatShape, etype: ElemType) -> None:
    object.__setattr__(node, "shape", shape)
    object.__setattr__(node, "etype", etype)


@dataclass(frozen=True, eq=False)
class Leaf(ExprNode):
    mat_id: int
    leaf_etype: ElemType
    leaf_shape: MatShape
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        _fix(self, self.leaf_shape, self.leaf_etype)

    @property
    def parent_shape(self) -> MatShape:
        return self.leaf_shape


@dataclass(frozen=True, eq=False)
class Subview(ExprNode):
    mat_id: int
    leaf_etype: ElemType
    row_off: int
    col_off: int
    view_shape: MatShape
    parent_shape: MatShape
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        if self.row_off < 0 or self.col_off < 0:
            raise OutOfBoundsError(f"negative subview offset ({self.row_off},{self.col_off})")
        if (self.row_off + self.view_shape.n_rows > self.parent_shape.n_rows
                or self.col_off + self.view_shape.n_cols > self.parent_shape.n_cols):
            raise OutOfBoundsError(
                f"subview {self.view_shape} at ({self.row_off},{self.col_off}) "
                f"exceeds parent {self.parent_shape}")
        _fix(self, self.view_shape, self.leaf_etype)


@dataclass(frozen=True, eq=False)
class Diag(ExprNode):
    """k-th diagonal of a square parent as a len x 1 column."""

    mat_id: int
    leaf_etype: ElemType
    k: int
    parent_shape: MatShape
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        p = self.parent_shape
        if p.n_rows != p.n_cols:
            raise ShapeError(f"diagonal of non-square parent {p}")
        n = p.n_rows - abs(self.k)
        if n < 0:
            raise OutOfBoundsError(f"diagonal {self.k} outside parent {p}")
        _fix(self, MatShape(n, 1), self.leaf_etype)

    @property
    def row_off(self) -> int:
        return max(-self.k, 0)

    @property
    def col_off(self) -> int:
        return max(self.k, 0)


LEAF_TYPES = (Leaf, Subview, Diag)


def _coerce_scalar(value, etype: ElemType):
    """Scalar -> the operand's element type (reference `expr.py:298-304`)."""
    if etype is ElemType.bf16:
        # bf16 arithmetic runs in f32; the slot carries an f32 value.
        return float(np.float32(value))
    if etype.is_float:
        return float(etype.dtype.type(value))
    if float(value) != int(value):
        raise ShapeError(f"scalar {value!r} is not integral for element type {etype.value}")
    return int(np.array(int(value)).astype(np.int64).astype(etype.dtype))


@dataclass(frozen=True, eq=False)
class UnaryElem(ExprNode):
    kind: UnaryKind
    child: ExprNode
    scalar: float | int | None = None
    exponent: int | None = None
    target: ElemType | None = None
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        ety = self.child.etype
        kind = self.kind
        if kind in FLOAT_ONLY_KINDS and not ety.is_float:
            raise ShapeError(f"{kind.name} requires a float operand, got {ety.value}")
        if kind in SCALAR_KINDS:
            if self.scalar is None:
                raise ShapeError(f"{kind.name} requires a scalar value")
            object.__setattr__(self, "scalar", _coerce_scalar(self.scalar, ety))
        elif self.scalar is not None:
            raise ShapeError(f"{kind.name} takes no scalar")
        if kind is UnaryKind.pow_int:
            e = self.exponent
            if e is None or isinstance(e, bool) or int(e) != e or not 0 <= e <= MAX_POW_EXPONENT:
                raise ShapeError(f"pow exponent must be an integer in 0..{MAX_POW_EXPONENT}, got {e}")
            object.__setattr__(self, "exponent", int(e))
        if kind is UnaryKind.conv:
            if self.target is None:
                raise ShapeError("conv requires a target element type")
            ety = self.target
        _fix(self, self.child.shape, ety)

    def children(self):
        return (self.child,)


@dataclass(frozen=True, eq=False)
class BinaryElem(ExprNode):
    kind: BinaryKind
    left: ExprNode
    right: ExprNode
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        a, b = self.left, self.right
        if a.shape != b.shape:
            raise ShapeError(f"{self.kind.name}: shapes {a.shape} and {b.shape} do not conform")
        if a.etype is not b.etype:
            raise ShapeError(f"{self.kind.name}: element types {a.etype.value} and "
                             f"{b.etype.value} differ (use conv_to for explicit conversion)")
        if self.kind is BinaryKind.elem_div and not a.etype.is_float:
            raise ShapeError("elem_div requires float operands")
        _fix(self, a.shape, a.etype)

    def children(self):
        return (self.left, self.right)


@dataclass(frozen=True, eq=False)
class Transpose(ExprNode):
    child: ExprNode
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        _fix(self, self.child.shape.t(), self.child.etype)

    def children(self):
        return (self.child,)


@dataclass(frozen=True, eq=False)
class MatMul(ExprNode):
    """Dense product.  bf16 operands produce an f32 result (f32 accumulation)."""

    left: ExprNode
    right: ExprNode
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        a, b = self.left, self.right
        if a.shape.n_cols != b.shape.n_rows:
            raise ShapeError(f"matmul: inner dimensions of {a.shape} and {b.shape} differ")
        if a.etype is not b.etype:
            raise ShapeError("matmul: operand element types differ")
        if not a.etype.is_float:
            raise ShapeError("matmul supports float element types only")
        out = ElemType.f32 if a.etype is ElemType.bf16 else a.etype
        _fix(self, MatShape(a.shape.n_rows, b.shape.n_cols), out)

    def children(self):
        return (self.left, self.right)


@dataclass(frozen=True, eq=False)
class Reduce(ExprNode):
    """Reduction of `child` along `dim` (0: per column -> 1 x n_cols,
    1: per row -> n_rows x 1).  Sums accumulate in f64 for float inputs and
    wrap in the element type for integers (the reference's `accu` convention,
    `codegen.py:47-49`); index reductions return the first extremal index as
    u32."""

    kind: ReduceKind
    dim: int
    child: ExprNode
    shape: MatShape = field(init=False, repr=False)
    etype: ElemType = field(init=False, repr=False)

    def __post_init__(self) -> None:
        if self.dim not in (0, 1):
            raise ShapeError(f"reduction dim must be 0 or 1, got {self.dim}")
        c = self.child
        if self.kind is ReduceKind.mean and not c.etype.is_float:
            raise ShapeError("mean requires a float operand")
        n_along = c.shape.n_rows if self.dim == 0 else c.shape.n_cols
        if self.kind in INDEX_REDUCTIONS and n_along > 2**32 - 1:
            raise ShapeError("index reductions return u32 indices")
        if self.kind in INDEX_REDUCTIONS | {ReduceKind.max, ReduceKind.min} and n_along == 0:
            raise ShapeError(f"{self.kind.name} of an empty dimension")
        shape = MatShape(1, c.shape.n_cols) if self.dim == 0 else MatShape(c.shape.n_rows, 1)
        ety = ElemType.u32 if self.kind in INDEX_REDUCTIONS else c.etype
        _fix(self, shape, ety)

    def children(self):
        return (self.child,)


# -- builders ----------------------------------------------------------------

def leaf(mat_id, etype, shape):
    return Leaf(mat_id, ElemType.of(etype), shape)


def subview(mat_id, etype, row_off, col_off, view_shape, parent_shape):
    return Subview(mat_id, ElemType.of(etype), row_off, col_off, view_shape, parent_shape)


def diag(mat_id, etype, k, parent_shape):
    return Diag(mat_id, ElemType.of(etype), k, parent_shape)


def plus(a, b):
    return BinaryElem(BinaryKind.plus, a, b)


def minus(a, b):
    return BinaryElem(BinaryKind.minus, a, b)


def schur(a, b):
    return BinaryElem(BinaryKind.schur, a, b)


def elem_div(a, b):
    return BinaryElem(BinaryKind.elem_div, a, b)


def scalar_add(x, s):
    return UnaryElem(UnaryKind.scalar_add, x, scalar=s)


def scalar_pre_mul(s, x):
    return UnaryElem(UnaryKind.scalar_pre_mul, x, scalar=s)


def scalar_pre_div(s, x):
    return UnaryElem(UnaryKind.scalar_pre_div, x, scalar=s)


def gt_scalar(x, s):
    return UnaryElem(UnaryKind.gt_scalar, x, scalar=s)


def neg(x):
    return UnaryElem(UnaryKind.neg, x)


def exp(x):
    return UnaryElem(UnaryKind.exp, x)


def log(x):
    return UnaryElem(UnaryKind.log, x)


def sqrt(x):
    return UnaryElem(UnaryKind.sqrt, x)


def tanh(x):
    return UnaryElem(UnaryKind.tanh, x)


def abs_(x):
    return UnaryElem(UnaryKind.abs, x)


def pow_int(x, exponent):
    return UnaryElem(UnaryKind.pow_int, x, exponent=exponent)


def square(x):
    """Armadillo `square`: x*x, i.e. the reference's pow_int(x, 2)."""
    return UnaryElem(UnaryKind.pow_int, x, exponent=2)


def conv(x, target):
    return UnaryElem(UnaryKind.conv, x, target=ElemType.of(target))


def transpose(x):
    return Transpose(x)


def matmul(a, b):
    return MatMul(a, b)


def reduce(kind: ReduceKind, dim: int, x):
    return Reduce(kind, dim, x)


# -- structural queries ----------------------------------------------------------

def walk(node: ExprNode) -> Iterator[ExprNode]:
    """Pre-order, children left to right."""
    stack = [node]
    while stack:
        n = stack.pop()
        yield n
        stack.extend(reversed(n.children()))


def contains(node: ExprNode, types) -> bool:
    return any(isinstance(n, types) for n in walk(node))


def contains_matmul(node: ExprNode) -> bool:
    return contains(node, MatMul)


def signature_of(node: ExprNode) -> str:
    """Canonical structural key, byte-compatible with the reference's
    `signature_of` (`expr.py:412-452`) for every node kind the reference has:
    kinds, element types, leaf first-visit ordinals, view kinds, pow
    exponents, conv targets and pre-order scalar slots.  Scalar values, view
    offsets, dimensions and matrix ids never enter the key."""
    ordinals: dict[int, int] = {}
    out: list[str] = []
    slot = 0

    def ordinal(mat_id: int) -> int:
        return ordinals.setdefault(mat_id, len(ordinals))

    def emit(n: ExprNode) -> None:
        nonlocal slot
        ty = n.etype.value
        if isinstance(n, Leaf):
            out.append(f"m{ordinal(n.mat_id)}:{ty}")
        elif isinstance(n, Subview):
            out.append(f"sv(m{ordinal(n.mat_id)}):{ty}")
        elif isinstance(n, Diag):
            out.append(f"dg(m{ordinal(n.mat_id)}):{ty}")
        elif isinstance(n, UnaryElem):
            if n.kind in SCALAR_KINDS:
                extra = f"{{s{slot}}}"
                slot += 1
            elif n.kind is UnaryKind.pow_int:
                extra = f"{{{n.exponent}}}"
            elif n.kind is UnaryKind.conv:
                extra = f"{{{n.target.value}}}"
            else:
                extra = ""
            out.append(f"{n.kind.value}{extra}:{ty}(")
            emit(n.child)
            out.append(")")
        elif isinstance(n, BinaryElem):
            out.append(f"{n.kind.value}:{ty}(")
            emit(n.left)
            out.append(",")
            emit(n.right)
            out.append(")")
        elif isinstance(n, Transpose):
            out.append(f"t:{ty}(")
            emit(n.child)
            out.append(")")
        elif isinstance(n, MatMul):
            out.append(f"mm:{ty}(")
            emit(n.left)
            out.append(",")
            emit(n.right)
            out.append(")")
        elif isinstance(n, Reduce):
            out.append(f"{n.kind.value}{{{n.dim}}}:{ty}(")
            emit(n.child)
            out.append(")")
        else:
            raise TypeError(f"unknown node {type(n).__name__}")

    emit(node)
    return "".join(out)


@dataclass(frozen=True)
class ViewOccurrence:
    kind: str          # "sv" | "dg"
    row_off: int
    col_off: int
    n_rows: int
    n_cols: int

    @property
    def n_elem(self) -> int:
        return self.n_rows * self.n_cols


@dataclass
class InputSpec:
    mat_id: int
    etype: ElemType
    parent_shape: MatShape
    views: list[ViewOccurrence] = field(default_factory=list)
    dense_count: int = 0


@dataclass(frozen=True)
class ScalarSlot:
    index: int
    value: float | int
    etype: ElemType


def collect_inputs(node: ExprNode) -> tuple[list[InputSpec], list[ScalarSlot]]:
    """Distinct inputs in first-visit order (each view occurrence recorded
    left to right) and the pre-order scalar slots (`expr.py:488-523`)."""
    inputs: list[InputSpec] = []
    by_id: dict[int, InputSpec] = {}
    slots: list[ScalarSlot] = []
    for n in walk(node):
        if isinstance(n, LEAF_TYPES):
            spec = by_id.get(n.mat_id)
            if spec is None:
                spec = by_id[n.mat_id] = InputSpec(n.mat_id, n.leaf_etype, n.parent_shape)
                inputs.append(spec)
            if isinstance(n, Leaf):
                spec.dense_count += 1
            else:
                kind = "sv" if isinstance(n, Subview) else "dg"
                spec.views.append(ViewOccurrence(kind, n.row_off, n.col_off,
                                                 n.shape.n_rows, n.shape.n_cols))
        elif isinstance(n, UnaryElem) and n.kind in SCALAR_KINDS:
            slots.append(ScalarSlot(len(slots), n.scalar, n.child.etype))
    return inputs, slots


class AliasKind(enum.Enum):
    NONE = "none"
    SAFE = "safe"
    UNSAFE = "unsafe"


def aliases(out_mat_id: int, node: ExprNode) -> AliasKind:
    """In-place classification (`expr.py:532-556`).  SAFE iff every read of
    the output is a dense identity-mapped leaf with no Transpose, MatMul or
    Reduce on its path."""
    found = unsafe = False
    stack: list[tuple[ExprNode, bool]] = [(node, False)]
    while stack:
        n, tainted = stack.pop()
        if isinstance(n, LEAF_TYPES):
            if n.mat_id == out_mat_id:
                found = True
                unsafe = unsafe or tainted or not isinstance(n, Leaf)
            continue
        taint = tainted or isinstance(n, (Transpose, MatMul, Reduce))
        stack.extend((c, taint) for c in n.children())
    if not found:
        return AliasKind.NONE
    return AliasKind.UNSAFE if unsafe else AliasKind.SAFE
