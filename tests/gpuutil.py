"""Helpers for GPU tests: re-express an expression tree over device matrices."""

from __future__ import annotations

import numpy as np

import paper_2604_22242_b200 as fm
from paper_2604_22242_b200 import exprtree as ast
from paper_2604_22242_b200.matrix import MatExpr


def remap(node, idmap):
    """Copy of `node` with every leaf's mat_id replaced via idmap."""
    if isinstance(node, ast.Leaf):
        return ast.Leaf(idmap[node.mat_id], node.leaf_etype, node.leaf_shape)
    if isinstance(node, ast.Subview):
        return ast.Subview(idmap[node.mat_id], node.leaf_etype, node.row_off, node.col_off,
                           node.view_shape, node.parent_shape)
    if isinstance(node, ast.Diag):
        return ast.Diag(idmap[node.mat_id], node.leaf_etype, node.k, node.parent_shape)
    if isinstance(node, ast.UnaryElem):
        return ast.UnaryElem(node.kind, remap(node.child, idmap), scalar=node.scalar,
                             exponent=node.exponent, target=node.target)
    if isinstance(node, ast.BinaryElem):
        return ast.BinaryElem(node.kind, remap(node.left, idmap), remap(node.right, idmap))
    if isinstance(node, ast.Transpose):
        return ast.Transpose(remap(node.child, idmap))
    if isinstance(node, ast.MatMul):
        return ast.MatMul(remap(node.left, idmap), remap(node.right, idmap))
    if isinstance(node, ast.Reduce):
        return ast.Reduce(node.kind, node.dim, remap(node.child, idmap))
    raise TypeError(type(node).__name__)


def leaf_etypes(node):
    out = {}
    for n in ast.walk(node):
        if isinstance(n, ast.LEAF_TYPES):
            out[n.mat_id] = n.leaf_etype
    return out


def bind(node, env, ctx):
    """Upload env arrays as device Mats and return a MatExpr over them."""
    ets = leaf_etypes(node)
    mats = {}
    idmap = {}
    for mid, arr in env.items():
        if mid not in ets:
            continue
        m = fm.from_array(np.asarray(arr), etype=ets[mid], ctx=ctx)
        mats[m.mat_id] = m
        idmap[mid] = m.mat_id
    return MatExpr(remap(node, idmap), mats, ctx)


def run_assign(expr: MatExpr):
    n = expr.node
    out = fm.Mat(n.shape.n_rows, n.shape.n_cols, n.etype, expr.ctx)
    out.assign(expr)
    return out.to_numpy()
