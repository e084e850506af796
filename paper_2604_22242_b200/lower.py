"""Lowering of MatMul-free trees to the fused register-stack program.

This replaces the reference's text generator (`codegen.py:172-227`,
`access_fragment`): instead of emitting C source per signature and calling a
compiler (`cjit.py:95-111`), a tree is lowered once per signature to a short
postfix program (`include/fmb200.h`, `fm_program`) that ahead-of-time sm_100a
kernels execute.  Per-node numerics are the reference's:

* every node rounds to its element type (f32 ops never fuse into FMAs);
* `sadd` is x+s, `smul` is s*x, `sdiv` is s/x (`codegen.py:196-201`);
* `gts` yields 0/1 in the operand type (`codegen.py:203`);
* `powi k` is the left-associated product x*x*...*x, k=0 -> 1 (`codegen.py:211-216`);
* float -> integer conversion truncates through int64 then wraps
  (`codegen.py:164-169`, `oracle.py:89-92`);
* integer arithmetic wraps modulo 2^32 (`cjit.py:102`, -fwrapv).

bf16 nodes compute in f32 and round to bf16 after every node.

Operand order is Sethi-Ullman: the child needing more stack goes first so a
tree with L leaves never needs more than ~log2(L)+1 registers; non-commutative
binaries then use their reversed opcode.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

from .errors import GenerationError
from .exprtree import (
    BinaryElem, BinaryKind, Diag, ElemType, ExprNode, Leaf, Subview, Transpose,
    UnaryElem, UnaryKind, SCALAR_KINDS,
)

MAX_DEPTH = 8
MAX_INSTR = 128
MAX_SLOTS = 40
MAX_SCALARS = 32

MAP_DENSE, MAP_SUBVIEW, MAP_DIAG = 0, 1, 2

# Opcode numbering must equal `enum fm_opcode` in include/fmb200.h
# (tests/test_abi.py parses the header and checks).
OPCODES = [
    "PUSH32", "PUSH64",
    "ADD_F", "SUB_F", "RSUB_F", "MUL_F", "DIV_F", "RDIV_F",
    "ADD_D", "SUB_D", "RSUB_D", "MUL_D", "DIV_D", "RDIV_D",
    "ADD_I", "SUB_I", "RSUB_I", "MUL_I",
    "SADD_F", "SMUL_F", "SDIV_F", "GTS_F",
    "SADD_D", "SMUL_D", "SDIV_D", "GTS_D",
    "SADD_I", "SMUL_I", "GTS_I32", "GTS_U32",
    "NEG_F", "NEG_D", "NEG_I", "ABS_F", "ABS_D", "ABS_I32",
    "EXP_F", "LOG_F", "SQRT_F", "TANH_F",
    "EXP_D", "LOG_D", "SQRT_D", "TANH_D",
    "POW_F", "POW_D", "POW_I",
    "ONE_F", "ONE_D", "ONE_I",
    "CVT_F_D", "CVT_D_F", "CVT_F_I", "CVT_D_I",
    "CVT_I32_F", "CVT_U32_F", "CVT_I32_D", "CVT_U32_D",
    "RND_BF_F", "CVT_D_BF",
    # binary ops whose second operand is a leaf read straight from its slot
    # (arg = slot): the PUSH + op pair in one VM dispatch and one stack
    # register less
    "ADD_F_S", "SUB_F_S", "RSUB_F_S", "MUL_F_S", "DIV_F_S", "RDIV_F_S",
    "ADD_D_S", "SUB_D_S", "RSUB_D_S", "MUL_D_S", "DIV_D_S", "RDIV_D_S",
    "ADD_I_S", "SUB_I_S", "RSUB_I_S", "MUL_I_S",
]
OP = {name: i for i, name in enumerate(OPCODES)}


def _cls(etype: ElemType) -> str:
    """Compute class of an element type: F (f32/bf16), D (f64), I (u32/i32)."""
    if etype is ElemType.f64:
        return "D"
    if etype in (ElemType.f32, ElemType.bf16):
        return "F"
    return "I"


@dataclass(frozen=True)
class SlotSpec:
    """One leaf access: input ordinal + index map (values bound at launch)."""

    input_index: int
    etype: ElemType
    map: int
    transposed: bool
    view_index: int          # index into that input's view occurrences (-1: dense)


@dataclass(frozen=True)
class ScalarSpec:
    index: int               # reference scalar slot (pre-order)
    cls: str                 # F / D / I


@dataclass
class Program:
    """Structure-only lowered program (one per qualified signature)."""

    code: list[tuple[int, int, int]] = field(default_factory=list)  # (opcode, depth, arg)
    slots: list[SlotSpec] = field(default_factory=list)
    scalars: list[ScalarSpec] = field(default_factory=list)
    result_etype: ElemType = ElemType.f32
    flat: bool = True
    depth: int = 0
    wide: bool = False

    def keys(self) -> list[tuple[int, int]]:
        return [((op << 3) | d, arg) for op, d, arg in self.code]

    def disassemble(self) -> list[str]:
        return [f"{OPCODES[op]}@{d} {arg}" for op, d, arg in self.code]


def _leaf_under(node: ExprNode):
    """The leaf a chain of transposes wraps (a slot operand), or None."""
    while isinstance(node, Transpose):
        node = node.child
    return node if isinstance(node, (Leaf, Subview, Diag)) else None


def _swap(node: BinaryElem, memo: dict) -> bool:
    """Evaluate the right child first?  The needier child goes first; on a
    tie, a lone leaf goes second (it becomes a slot operand)."""
    a, b = _need(node.left, memo), _need(node.right, memo)
    if a != b:
        return b > a
    return _leaf_under(node.left) is not None and _leaf_under(node.right) is None


def _need(node: ExprNode, memo: dict) -> int:
    """Sethi-Ullman register need; a leaf evaluated second is a slot operand
    of the binary op (no register)."""
    key = id(node)
    if key in memo:
        return memo[key]
    if isinstance(node, (Leaf, Subview, Diag)):
        r = 1
    elif isinstance(node, (UnaryElem, Transpose)):
        r = _need(node.children()[0], memo)
    elif isinstance(node, BinaryElem):
        a, b = _need(node.left, memo), _need(node.right, memo)
        second = node.left if _swap(node, memo) else node.right
        if _leaf_under(second) is not None:
            r = max(a, b)
        else:
            r = max(a, b) if a != b else a + 1
    else:
        raise GenerationError(f"{type(node).__name__} reached the lowering; "
                              "fusion barriers must be split during planning")
    memo[key] = r
    return r


class _Lowerer:
    def __init__(self, root: ExprNode):
        self.root = root
        self.prog = Program(result_etype=root.etype)
        self.inputs: dict[int, int] = {}          # mat_id -> input ordinal (first visit)
        self.view_count: dict[int, int] = {}      # input ordinal -> views seen
        self.slot_of: dict[tuple, int] = {}
        self.n_scalar = 0
        self.memo: dict = {}
        self.view_count = {}
        self._preassign(root)

    def _preassign(self, node: ExprNode) -> None:
        """Fix input ordinals, view-occurrence indices and scalar slots in the
        reference's pre-order (`expr.py:488-523`), independent of the
        Sethi-Ullman evaluation order used below."""
        self.leaf_info: dict[int, tuple[int, int]] = {}
        self.scalar_of: dict[int, int] = {}
        stack = [(node, False)]
        while stack:
            n, tr = stack.pop()
            if isinstance(n, (Leaf, Subview, Diag)):
                i = self.inputs.setdefault(n.mat_id, len(self.inputs))
                v = -1
                if not isinstance(n, Leaf):
                    v = self.view_count.get(i, 0)
                    self.view_count[i] = v + 1
                self.leaf_info[id(n)] = (i, v)
                self.slot(n, tr)          # slots in first-visit order: slot i <-> input i when flat
            elif isinstance(n, UnaryElem) and n.kind in SCALAR_KINDS:
                self.scalar_of[id(n)] = self.n_scalar
                self.n_scalar += 1
            flip = tr ^ isinstance(n, Transpose)
            stack.extend((c, flip) for c in reversed(n.children()))

    def emit(self, op: str, depth: int, arg: int = 0) -> None:
        if depth >= MAX_DEPTH:
            raise GenerationError(f"expression needs more than {MAX_DEPTH} stack registers")
        if len(self.prog.code) >= MAX_INSTR:
            raise GenerationError(f"expression exceeds {MAX_INSTR} fused instructions")
        self.prog.code.append((OP[op], depth, arg))
        self.prog.depth = max(self.prog.depth, depth + 1)

    def slot(self, n: ExprNode, transposed: bool) -> int:
        i, v = self.leaf_info[id(n)]
        kind = MAP_DENSE if isinstance(n, Leaf) else (MAP_SUBVIEW if isinstance(n, Subview) else MAP_DIAG)
        key = (i, kind, transposed, v)
        if key not in self.slot_of:
            if len(self.prog.slots) >= MAX_SLOTS:
                raise GenerationError(f"expression reads more than {MAX_SLOTS} leaf accesses")
            self.slot_of[key] = len(self.prog.slots)
            self.prog.slots.append(SlotSpec(i, n.leaf_etype, kind, transposed, v))
            if kind != MAP_DENSE or transposed:
                self.prog.flat = False
        return self.slot_of[key]

    def scalar(self, n: UnaryElem) -> int:
        idx = self.scalar_of[id(n)]
        self.prog.scalars.append(ScalarSpec(idx, _cls(n.child.etype)))
        return idx

    def round_bf16(self, etype: ElemType, depth: int) -> None:
        if etype is ElemType.bf16:
            self.emit("RND_BF_F", depth)

    def lower(self, n: ExprNode, depth: int, transposed: bool) -> None:
        if isinstance(n, (Leaf, Subview, Diag)):
            s = self.slot(n, transposed)
            if n.leaf_etype is ElemType.f64:
                self.prog.wide = True
                self.emit("PUSH64", depth, s)
            else:
                self.emit("PUSH32", depth, s)
            return
        if isinstance(n, Transpose):
            self.lower(n.child, depth, not transposed)
            return
        if isinstance(n, BinaryElem):
            self._binary(n, depth, transposed)
            return
        if isinstance(n, UnaryElem):
            self._unary(n, depth, transposed)
            return
        raise GenerationError(f"{type(n).__name__} reached the lowering; "
                              "fusion barriers must be split during planning")

    def _binary(self, n: BinaryElem, depth: int, transposed: bool) -> None:
        c = _cls(n.etype)
        if c == "D":
            self.prog.wide = True
        swap = _swap(n, self.memo)
        first, second = (n.right, n.left) if swap else (n.left, n.right)
        self.lower(first, depth, transposed)
        name = {BinaryKind.plus: "ADD", BinaryKind.minus: "SUB",
                BinaryKind.schur: "MUL", BinaryKind.elem_div: "DIV"}[n.kind]
        if swap and name in ("SUB", "DIV"):
            name = "R" + name
        leaf = _leaf_under(second)
        if leaf is not None:
            # slot operand: the leaf's transposes flip the access like lower() does
            tr = transposed
            t = second
            while isinstance(t, Transpose):
                tr, t = not tr, t.child
            s = self.slot(leaf, tr)
            if leaf.leaf_etype is ElemType.f64:
                self.prog.wide = True
            self.emit(f"{name}_{c}_S", depth, s)
        else:
            self.lower(second, depth + 1, transposed)
            self.emit(f"{name}_{c}", depth)
        self.round_bf16(n.etype, depth)

    def _unary(self, n: UnaryElem, depth: int, transposed: bool) -> None:
        self.lower(n.child, depth, transposed)
        src = n.child.etype
        c = _cls(src)
        k = n.kind
        if k is UnaryKind.scalar_add:
            self.emit(f"SADD_{c}", depth, self.scalar(n))
        elif k is UnaryKind.scalar_pre_mul:
            self.emit(f"SMUL_{c}", depth, self.scalar(n))
        elif k is UnaryKind.scalar_pre_div:
            self.emit(f"SDIV_{c}", depth, self.scalar(n))
        elif k is UnaryKind.gt_scalar:
            op = {"F": "GTS_F", "D": "GTS_D"}.get(c) or ("GTS_U32" if src is ElemType.u32 else "GTS_I32")
            self.emit(op, depth, self.scalar(n))
        elif k is UnaryKind.neg:
            self.emit(f"NEG_{c}", depth)
        elif k is UnaryKind.abs:
            if src is ElemType.u32:
                return                                   # |x| = x, nothing to round
            self.emit("ABS_I32" if c == "I" else f"ABS_{c}", depth)
        elif k in (UnaryKind.exp, UnaryKind.log, UnaryKind.sqrt, UnaryKind.tanh):
            self.emit(f"{k.name.upper()}_{c}", depth)
        elif k is UnaryKind.pow_int:
            if n.exponent == 0:
                self.emit(f"ONE_{c}", depth)
            elif n.exponent >= 2:
                self.emit(f"POW_{c}", depth, n.exponent)
            # exponent 1 is the child itself (`codegen.py:213-214`)
        elif k is UnaryKind.conv:
            self._conv(src, n.target, depth)
            return                                       # conv rounds by itself
        else:
            raise GenerationError(f"no lowering for unary kind {k}")
        self.round_bf16(n.etype, depth)

    def _conv(self, src: ElemType, dst: ElemType, depth: int) -> None:
        if dst is ElemType.f64:
            self.prog.wide = True
        if src is dst:
            return
        cs, cd = _cls(src), _cls(dst)
        if dst is ElemType.bf16:
            if cs == "F":                              # f32 -> bf16
                self.emit("RND_BF_F", depth)
            elif cs == "D":
                self.emit("CVT_D_BF", depth)
            else:                                      # int -> f64 (exact) -> bf16 (one rounding)
                self.prog.wide = True
                self.emit("CVT_U32_D" if src is ElemType.u32 else "CVT_I32_D", depth)
                self.emit("CVT_D_BF", depth)
            return
        if cs == cd:
            if cs == "I":
                return                                 # i32 <-> u32: same bits
            return                                     # bf16 -> f32: values already f32
        table = {
            ("F", "D"): "CVT_F_D", ("D", "F"): "CVT_D_F",
            ("F", "I"): "CVT_F_I", ("D", "I"): "CVT_D_I",
        }
        if cs == "I":
            sign = "U32" if src is ElemType.u32 else "I32"
            self.emit(f"CVT_{sign}_{cd}", depth)
        else:
            self.emit(table[(cs, cd)], depth)


def lower(node: ExprNode) -> Program:
    """Lower a MatMul/Reduce-free tree.  Raises GenerationError if it cannot
    fit the AOT kernels' limits (stack depth, instruction and slot counts)."""
    low = _Lowerer(node)
    low.lower(node, 0, False)
    prog = low.prog
    # A dense untransposed leaf always has the domain's shape (elementwise
    # nodes conform), so `flat` programs index every slot by the flat index.
    if len(prog.scalars) > MAX_SCALARS:
        raise GenerationError(f"expression uses more than {MAX_SCALARS} scalars")
    return prog


# -- scalar encoding -------------------------------------------------------------

def scalar_bits(value, cls: str) -> int:
    if cls == "F":
        return struct.unpack("<I", struct.pack("<f", float(value)))[0]
    if cls == "D":
        return struct.unpack("<Q", struct.pack("<d", float(value)))[0]
    return int(value) & 0xFFFFFFFF
