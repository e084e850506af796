"""Ahead-of-time template registry (build-time code generation).

The north star forbids runtime compilation (no NVRTC / JIT), so the hot
signatures -- the BASELINE configs and the paper's suite -- are fixed here,
turned into expression-template types (csrc/templates.cuh) and compiled by
nvcc into libfmb200.so.  `fm_kernel_lookup` maps a qualified signature to
one of them at `compile` time; every other signature runs on the register VM.

Signatures are produced with this package's own tree builders, so they are
byte-identical to what `exprtree.signature_of` yields for user expressions
(and to the reference's `expr.signature_of` for reference-expressible trees).
"""

from __future__ import annotations

import math
from pathlib import Path

from . import exprtree as ast
from . import lower as lw
from .exprtree import ElemType, MatShape

_S = MatShape(4, 4)


def _m(i: int, ety: ElemType):
    return ast.leaf(i, ety, _S)


def hot_expressions() -> list[tuple[str, ast.ExprNode]]:
    """(label, tree) of every AOT-instantiated expression."""
    out = []
    for ety in (ElemType.f32, ElemType.f64):
        t = ety.value
        X, Y, Z = _m(0, ety), _m(1, ety), _m(2, ety)
        # C1: Z = 2*(X % Y) + X
        out.append((f"c1_{t}", ast.plus(ast.scalar_pre_mul(2, ast.schur(X, Y)), X)))
        # C2: accu(X % Y), dot(x, y) -> mul(m0, m1);  norm(x - y) -> powi2(sub(m0, m1))
        out.append((f"schur_{t}", ast.schur(X, Y)))
        out.append((f"sqdiff_{t}", ast.square(ast.minus(X, Y))))
        # C3: exp(-square(X - Y) / 2) + 0.5*abs(X)
        out.append((f"c3_{t}", ast.plus(
            ast.exp(ast.scalar_pre_mul(0.5, ast.neg(ast.square(ast.minus(X, Y))))),
            ast.scalar_pre_mul(0.5, ast.abs_(X)))))
        # C4 subexpression: (X - Y) % Z
        out.append((f"c4_{t}", ast.schur(ast.minus(X, Y), Z)))
        # single-leaf copy / reductions of a plain matrix
        out.append((f"copy_{t}", X))
        # paper suite, flat members (bench.py:91-201)
        out.append((f"add2_{t}", ast.plus(X, Y)))
        W = _m(3, ety)
        out.append((f"add4_{t}", ast.plus(ast.plus(ast.plus(X, Y), Z), W)))
        out.append((f"relu_{t}", ast.schur(X, ast.gt_scalar(X, 0))))
        out.append((f"sigmoid_{t}", ast.scalar_pre_div(1, ast.scalar_add(ast.exp(ast.neg(X)), 1))))
        out.append((f"swish_{t}", ast.elem_div(X, ast.scalar_add(
            ast.exp(ast.scalar_pre_mul(-1.0, X)), 1))))
        coeff = math.sqrt(2.0 / 3.14159265358979)
        out.append((f"gelu_{t}", ast.schur(
            ast.scalar_pre_mul(0.5, X),
            ast.scalar_add(ast.tanh(ast.scalar_pre_mul(coeff, ast.plus(
                X, ast.scalar_pre_mul(0.044715, ast.pow_int(X, 3))))), 1))))
    # common elementwise forms users write beyond the configs and the suite
    # (BLAS-1 style updates, differences, quotients, unary maps): templates
    # run them at the streaming rate instead of on the register VM
    for ety in (ElemType.f32, ElemType.f64):
        t = ety.value
        X, Y, Z = _m(0, ety), _m(1, ety), _m(2, ety)
        out.append((f"axpy_{t}", ast.plus(ast.scalar_pre_mul(2.0, X), Y)))
        out.append((f"axpby_{t}", ast.plus(ast.scalar_pre_mul(2.0, X), ast.scalar_pre_mul(3.0, Y))))
        out.append((f"sub_{t}", ast.minus(X, Y)))
        out.append((f"div_{t}", ast.elem_div(X, Y)))
        out.append((f"scale_{t}", ast.scalar_pre_mul(2.0, X)))
        out.append((f"shift_{t}", ast.scalar_add(X, 1.0)))
        out.append((f"muladd_{t}", ast.plus(ast.schur(X, Y), Z)))
        out.append((f"absdiff_{t}", ast.abs_(ast.minus(X, Y))))
        out.append((f"square_{t}", ast.square(X)))
        out.append((f"sqrt_{t}", ast.sqrt(X)))
        out.append((f"exp_{t}", ast.exp(X)))
        out.append((f"log_{t}", ast.log(X)))
        out.append((f"neg_{t}", ast.neg(X)))
    # paper suite members with views / transposes (bench.py:119-147): leaves
    # read through index maps; copies run on the tiled staged skeleton
    _B = MatShape(8, 8)
    for ety in (ElemType.f32, ElemType.f64):
        t = ety.value
        X, Y, Z, W = (ast.leaf(i, ety, _B) for i in range(4))
        ch = [ast.subview(i, ety, 2, 2, MatShape(4, 4), _B) for i in range(4)]
        out.append((f"addsub2_{t}", ast.plus(ch[0], ch[1])))
        out.append((f"addsub4_{t}", ast.plus(ast.plus(ast.plus(ch[0], ch[1]), ch[2]), ch[3])))
        out.append((f"expr1_{t}", ast.plus(ast.scalar_pre_mul(2, ast.plus(ast.transpose(X), Y)),
                                          ast.scalar_pre_mul(2, ast.plus(X, ast.transpose(Y))))))
        out.append((f"expr2_{t}", ast.plus(ast.plus(ast.scalar_pre_mul(2.0, X),
                                                    ast.transpose(ast.plus(Y, Z))),
                                           ast.log(ast.pow_int(W, 2)))))
        # expr3 (bench.py:141-145): 1 / (x % conv_to(u, T) + log(log(x + 2) % w)), u a u32 leaf
        U = ast.leaf(1, ElemType.u32, _B)
        W3 = ast.leaf(2, ety, _B)
        out.append((f"expr3_{t}", ast.scalar_pre_div(1, ast.plus(
            ast.schur(X, ast.conv(U, ety)),
            ast.log(ast.schur(ast.log(ast.scalar_add(X, 2)), W3))))))
        d = [ast.diag(i, ety, k, _B) for i, k in ((0, -1), (0, 1), (1, -1), (1, 1))]
        out.append((f"diagsum_{t}", ast.schur(ast.plus(d[0], d[1]), ast.plus(d[2], d[3]))))
    # the paper's add-N sweep (reference bench.py:307-326, Fig. 5):
    # left-deep chains of N distinct inputs, one fused launch each
    for ety in (ElemType.f32, ElemType.f64):
        for k in range(5, 33):
            mats = [_m(i, ety) for i in range(k)]
            e = ast.plus(mats[0], mats[1])
            for m in mats[2:]:
                e = ast.plus(e, m)
            out.append((f"add{k}N_{ety.value}", e))
    return out


def vector_width(nin: int, ety: ElemType) -> int:
    """Elements per thread chunk: a 32-byte (f32) / 32-byte (f64) run per
    input, halved for wide chains so every input's loads fit in registers."""
    if ety is ElemType.f32:
        return 8 if nin <= 4 else 4
    return 4 if nin <= 4 else 2


# -- signature -> C++ expression-template type --------------------------------------

_BIN = {ast.BinaryKind.plus: "Add", ast.BinaryKind.minus: "Sub",
        ast.BinaryKind.schur: "Mul", ast.BinaryKind.elem_div: "Div"}
_UN = {ast.UnaryKind.neg: "Neg", ast.UnaryKind.abs: "Abs", ast.UnaryKind.exp: "Exp",
       ast.UnaryKind.log: "Log", ast.UnaryKind.sqrt: "Sqrt", ast.UnaryKind.tanh: "Tanh"}
_SC = {ast.UnaryKind.scalar_add: "SAdd", ast.UnaryKind.scalar_pre_mul: "SMul",
       ast.UnaryKind.scalar_pre_div: "SDiv", ast.UnaryKind.gt_scalar: "Gts"}


def cpp_type(node: ast.ExprNode) -> tuple[str, int, ElemType]:
    """C++ type, number of leaf slots and the common element type.

    `In<j>` reads program slot j.  Slots are numbered exactly as
    lower.py numbers them: first visit in pre-order of the key (input
    ordinal, index map, transposed, view occurrence), with a Transpose node
    flipping the orientation of the leaves below it (it has no node of its
    own: the transposition lives in the slot's index map)."""
    inputs: dict[int, int] = {}
    views: dict[int, int] = {}
    slots: dict[tuple, int] = {}
    slot = [0]
    ety = node.etype

    def leaf_slot(n, tr: bool) -> int:
        i = inputs.setdefault(n.mat_id, len(inputs))
        v = -1
        if not isinstance(n, ast.Leaf):
            v = views.get(i, 0)
            views[i] = v + 1
        kind = 0 if isinstance(n, ast.Leaf) else (1 if isinstance(n, ast.Subview) else 2)
        return slots.setdefault((i, kind, tr, v), len(slots))

    def go(n, tr=False) -> str:
        if (isinstance(n, ast.UnaryElem) and n.kind is ast.UnaryKind.conv and n.target is ety
                and isinstance(n.child, ast.Leaf) and n.child.etype in (ElemType.u32, ElemType.i32)):
            # an integer leaf converted to the template type (paper expr3)
            kind = "CvtU32" if n.child.etype is ElemType.u32 else "CvtI32"
            return f"{kind}<{leaf_slot(n.child, tr)}>"
        if n.etype is not ety:
            raise ValueError("templates need a single element type")
        if isinstance(n, (ast.Leaf, ast.Subview, ast.Diag)):
            return f"In<{leaf_slot(n, tr)}>"
        if isinstance(n, ast.Transpose):
            return go(n.child, not tr)
        if isinstance(n, ast.BinaryElem):
            left = go(n.left, tr)
            return f"{_BIN[n.kind]}<{left}, {go(n.right, tr)}>"
        if isinstance(n, ast.UnaryElem):
            if n.kind in _SC:
                s = slot[0]
                slot[0] += 1
                return f"{_SC[n.kind]}<{s}, {go(n.child, tr)}>"
            if n.kind is ast.UnaryKind.pow_int:
                return f"Pow<{n.exponent}, {go(n.child, tr)}>"
            if n.kind in _UN:
                return f"{_UN[n.kind]}<{go(n.child, tr)}>"
        raise ValueError(f"no template for {type(n).__name__}")

    text = go(node)
    return text, len(slots), ety


TEMPLATE_SHARDS = 8


def generate(path: Path) -> Path:
    """Write gen_templates.cu.

    build.py compiles it TEMPLATE_SHARDS times with -DFM_TEMPLATE_SHARD=k:
    shard k explicitly instantiates the launchers of entries i with
    i % TEMPLATE_SHARDS == k (so nvcc runs in parallel), and shard 0 also
    holds the lookup table, which sees the other shards' launchers through
    explicit instantiation declarations.
    """
    lines = [
        "// GENERATED by paper_2604_22242_b200/aot_registry.py -- do not edit.",
        "// Ahead-of-time expression-template kernels for the hot signatures.",
        '#include "templates.cuh"',
        "",
        "#ifndef FM_TEMPLATE_SHARD",
        "#define FM_TEMPLATE_SHARD 0",
        f"#define FM_TEMPLATE_SHARDS 1",
        "#endif",
        f"#if FM_TEMPLATE_SHARDS != 1 && FM_TEMPLATE_SHARDS != {TEMPLATE_SHARDS}",
        "#error \"shard count out of sync with aot_registry.TEMPLATE_SHARDS\"",
        "#endif",
        "",
        "namespace fm {",
        "using namespace tx;",
        "",
        "#define FM_INST(E, EXT)                                                                        \\",
        "  EXT template int tx::t_copy<E>(const fm_program &, void *, int64_t, int64_t, cudaStream_t);        \\",
        "  EXT template int tx::t_accu<E>(const fm_program &, void *, int64_t, int64_t, int, cudaStream_t);   \\",
        "  EXT template int tx::t_dim<E>(const fm_program &, int, int64_t, int64_t, const ReduceOuts &, cudaStream_t);",
        "",
    ]
    entries = []
    types: dict[str, int] = {}      # one instantiation per distinct evaluator type
    for label, node in hot_expressions():
        sig = ast.signature_of(node)
        typ, nin, ety = cpp_type(node)
        T = "float" if ety is ElemType.f32 else "double"
        V = vector_width(nin, ety)
        tiled = not lw.lower(node).flat       # transposed / view leaves
        full = f"TEval<{typ}, {T}, {nin}, {V}, {'true' if tiled else 'false'}>"
        lines.append(f"// {label}: {sig}")
        if full not in types:
            i = types[full] = len(types)
            lines.append(f"using E{i} = {full};")
            lines.append(f"#if {i} % FM_TEMPLATE_SHARDS == FM_TEMPLATE_SHARD")
            lines.append(f"FM_INST(E{i}, )")
            lines.append("#else")
            lines.append(f"FM_INST(E{i}, extern)")
            lines.append("#endif")
        i = types[full]
        entries.append(f'  {{"{sig}", &t_copy<E{i}>, &t_accu<E{i}>, &t_dim<E{i}>, {nin}, {ety.code}}},')
    lines.append("")
    lines.append("#if FM_TEMPLATE_SHARD == 0")
    lines.append("static const TemplateEntry kTable[] = {")
    lines.extend(entries)
    lines.append("};")
    lines.append("")
    lines.append("const TemplateEntry *template_table(int *n) {")
    lines.append("  *n = (int)(sizeof(kTable) / sizeof(kTable[0]));")
    lines.append("  return kTable;")
    lines.append("}")
    lines.append("#endif")
    lines.append("")
    lines.append("}  // namespace fm")
    text = "\n".join(lines) + "\n"
    if not path.exists() or path.read_text() != text:
        path.write_text(text)
    return path


def registered_signatures() -> list[str]:
    return [ast.signature_of(n) for _, n in hot_expressions()]
