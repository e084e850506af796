"""JSON (de)serialisation of expression trees for golden fixtures.

Works on this package's trees and, by duck typing, on the reference's
(`fusemat.expr`) trees, so tests/golden/make_golden.py can record trees built
by the reference API and the GPU tests can rebuild them without the reference.
"""

from __future__ import annotations

from paper_2604_22242_b200 import exprtree as ast
from paper_2604_22242_b200.exprtree import ElemType, MatShape


def _et(e) -> str:
    return e.value if hasattr(e, "value") else str(e)


def to_json(node) -> dict:
    name = type(node).__name__
    if name == "Leaf":
        return {"n": "leaf", "id": node.mat_id, "t": _et(node.leaf_etype),
                "shape": [node.leaf_shape.n_rows, node.leaf_shape.n_cols]}
    if name == "Subview":
        return {"n": "sv", "id": node.mat_id, "t": _et(node.leaf_etype),
                "off": [node.row_off, node.col_off],
                "shape": [node.view_shape.n_rows, node.view_shape.n_cols],
                "parent": [node.parent_shape.n_rows, node.parent_shape.n_cols]}
    if name == "Diag":
        return {"n": "dg", "id": node.mat_id, "t": _et(node.leaf_etype), "k": node.k,
                "parent": [node.parent_shape.n_rows, node.parent_shape.n_cols]}
    if name == "UnaryElem":
        d = {"n": "un", "k": node.kind.value, "c": to_json(node.child)}
        if node.scalar is not None:
            d["s"] = node.scalar
        if node.exponent is not None:
            d["e"] = node.exponent
        if node.target is not None:
            d["tg"] = _et(node.target)
        return d
    if name == "BinaryElem":
        return {"n": "bin", "k": node.kind.value, "l": to_json(node.left), "r": to_json(node.right)}
    if name == "Transpose":
        return {"n": "t", "c": to_json(node.child)}
    if name == "MatMul":
        return {"n": "mm", "l": to_json(node.left), "r": to_json(node.right)}
    if name == "Reduce":
        return {"n": "red", "k": node.kind.value, "dim": node.dim, "c": to_json(node.child)}
    raise TypeError(name)


def from_json(d: dict):
    n = d["n"]
    if n == "leaf":
        return ast.leaf(d["id"], d["t"], MatShape(*d["shape"]))
    if n == "sv":
        return ast.subview(d["id"], d["t"], d["off"][0], d["off"][1], MatShape(*d["shape"]),
                           MatShape(*d["parent"]))
    if n == "dg":
        return ast.diag(d["id"], d["t"], d["k"], MatShape(*d["parent"]))
    if n == "un":
        return ast.UnaryElem(ast.UnaryKind(d["k"]), from_json(d["c"]), scalar=d.get("s"),
                             exponent=d.get("e"),
                             target=ElemType.of(d["tg"]) if "tg" in d else None)
    if n == "bin":
        return ast.BinaryElem(ast.BinaryKind(d["k"]), from_json(d["l"]), from_json(d["r"]))
    if n == "t":
        return ast.transpose(from_json(d["c"]))
    if n == "mm":
        return ast.matmul(from_json(d["l"]), from_json(d["r"]))
    if n == "red":
        return ast.reduce(ast.ReduceKind(d["k"]), d["dim"], from_json(d["c"]))
    raise ValueError(n)
