"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package (`fusemat`, /root/reference/pkg/src) and the
reference test generator (`treegen`, /root/reference/pkg/tests) read-only, and
records into tests/golden/:

* rng.npz          -- reference rng.uniform_fill / uniform_int_fill streams
* signatures.json  -- reference signature_of / qualified signature / arg
                      schema for the suite and config expressions
* cases.json + cases.npz -- expression trees (JSON), their input matrices and
                      the reference's outputs: oracle.materialize, the ref
                      backend (per-element interpreter) and the compiled-C
                      "device" backend (CJitBackend), plus accu results and
                      f64-accumulated GEMMs.

The GPU box has no /root/reference; tests read only these files there.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import fusemat as fm  # noqa: E402  (reference)
from fusemat import expr as rast  # noqa: E402
from fusemat import oracle as roracle  # noqa: E402
from fusemat import rng as rrng  # noqa: E402
from fusemat.bench import SUITE, BenchSpec, build_expression  # noqa: E402
from fusemat.codegen import COPY, REDUCE_ACCU, arg_schema, qualified_signature  # noqa: E402
from treegen import TreeGen  # noqa: E402  (reference test generator)
from treeio import to_json  # noqa: E402


def rng_fixture():
    out = {}
    for seed in (0, 1, 42, 43, 44, 2**63 + 5):
        for et in ("f32", "f64"):
            out[f"u_{et}_{seed}"] = rrng.uniform_fill(seed, 4096, np.dtype(np.float32 if et == "f32" else np.float64))
        out[f"i_u32_{seed}"] = rrng.uniform_int_fill(seed, 4096, np.dtype(np.uint32), 10)
        out[f"raw_{seed}"] = rrng.raw_words(seed, 64)
    np.savez_compressed(HERE / "rng.npz", **out)


def ref_config_exprs(ctx, n=16):
    X = fm.randu(n, n, 42, "f32", ctx)
    Y = fm.randu(n, n, 43, "f32", ctx)
    X64 = fm.randu(n, n, 42, "f64", ctx)
    Y64 = fm.randu(n, n, 43, "f64", ctx)
    Z64 = fm.randu(n, n, 44, "f64", ctx)
    return {
        "c1": 2 * (X * Y) + X,                 # `%` is `*` (Schur) in the reference API
        "c2_accu": X * Y,
        "c2_norm": (X - Y) ** 2,
        "c2_accu_f64": X64 * Y64,
        "c2_norm_f64": (X64 - Y64) ** 2,
        "c3_noabs": fm.exp(-((X - Y) ** 2) / 2) + 0.5 * X,
        "c4_sub": (X64 - Y64) * Z64,
        "c5": 2 * X @ Y.t(),
    }


def signatures_fixture():
    rows = []
    ctx = fm.Context("ref")
    for name in SUITE:
        out, e = build_expression(BenchSpec(expr_name=name, n=16), ctx)
        rows.append(_sig_row(name, e.node))
    for name, e in ref_config_exprs(ctx).items():
        rows.append(_sig_row(name, e.node))
    gen = TreeGen(seed=777, max_dim=6)
    for i in range(40):
        rows.append(_sig_row(f"tree{i}", gen.tree(depth=5)))
    (HERE / "signatures.json").write_text(json.dumps(rows, indent=1))


def _sig_row(name, node):
    row = {"name": name, "tree": to_json(node), "signature": rast.signature_of(node)}
    if not rast.contains_matmul(node):
        row["qualified_copy"] = qualified_signature(node, COPY)
        row["qualified_accu"] = qualified_signature(node, REDUCE_ACCU)
        row["schema_copy"] = [str(a) for a in arg_schema(node, COPY)]
        row["schema_accu"] = [str(a) for a in arg_schema(node, REDUCE_ACCU)]
    inputs, slots = rast.collect_inputs(node)
    row["inputs"] = [s.mat_id for s in inputs]
    row["slots"] = [s.value for s in slots]
    return row


class CaseWriter:
    def __init__(self):
        self.cases = []
        self.arrays = {}

    def add(self, name, node, env, **expected):
        key = f"k{len(self.cases)}"
        env_keys = {}
        for mid, arr in env.items():
            k = f"{key}_in{mid}"
            self.arrays[k] = np.asarray(arr)
            env_keys[str(mid)] = k
        exp_keys = {}
        for label, val in expected.items():
            if isinstance(val, (float, int)):
                exp_keys[label] = {"scalar": val}
            else:
                k = f"{key}_{label}"
                self.arrays[k] = np.asarray(val)
                exp_keys[label] = k
        self.cases.append({"name": name, "tree": to_json(node), "env": env_keys, "expected": exp_keys})

    def save(self):
        (HERE / "cases.json").write_text(json.dumps(self.cases, indent=1))
        np.savez_compressed(HERE / "cases.npz", **self.arrays)


def _run(ctx, e, node):
    out = fm.Mat(node.shape.n_rows, node.shape.n_cols, node.etype, ctx)
    out.assign(e)
    return out.to_numpy()


def _rebuild(node, mats, ctx):
    from fusemat.expr import InputBinding, collect_inputs, rebind_tree
    from fusemat.matrix import MatExpr
    inputs, slots = collect_inputs(node)
    bindings = [InputBinding(mats[s.mat_id].mat_id, s.parent_shape,
                             [(v.row_off, v.col_off) for v in s.views]) for s in inputs]
    rebound = rebind_tree(node, bindings, [s.value for s in slots], node.shape)
    return MatExpr(rebound, {m.mat_id: m for m in mats.values()}, ctx)


def cases_fixture():
    w = CaseWriter()
    # 1. the paper suite at n=32, seed 42 (test_cjit.py:77-88 setting)
    for name in SUITE:
        for backend in ("device",):
            ctx = fm.Context(backend)
            out, e = build_expression(BenchSpec(expr_name=name, n=32, seed=42), ctx)
            env = {mid: m.to_numpy() for mid, m in e.mats.items()}
            out.assign(e)
            dev = out.to_numpy()
        ref_ctx = fm.Context("ref")
        rout, re_ = build_expression(BenchSpec(expr_name=name, n=32, seed=42), ref_ctx)
        rout.assign(re_)
        w.add(f"suite_{name}", e.node, env, oracle=roracle.materialize(e.node, env),
              cjit=dev, ref=rout.to_numpy())
    # 2. configs in reference form
    for n in (64, 128):
        ctx = fm.Context("device")
        rctx = fm.Context("ref")
        exprs = ref_config_exprs(ctx, n)
        rexprs = ref_config_exprs(rctx, n)
        for name, e in exprs.items():
            env = {mid: m.to_numpy() for mid, m in e.mats.items()}
            node = e.node
            orc = roracle.materialize(node, env)
            if name.startswith("c2"):
                w.add(f"{name}_n{n}", node, env, oracle=orc, accu_cjit=float(fm.accu(e)),
                      accu_ref=float(fm.accu(rexprs[name])))
            elif n == 64 or name == "c1":
                w.add(f"{name}_n{n}", node, env, oracle=orc, cjit=_run(ctx, e, node),
                      ref=_run(rctx, rexprs[name], rexprs[name].node))
    # 3. random trees from the reference generator (test_backend.py:182-202)
    for etype, seed, count in ((rast.ElemType.f32, 2024, 60), (rast.ElemType.f64, 4048, 40),
                               (rast.ElemType.i32, 99, 30), (rast.ElemType.u32, 7, 30)):
        gen = TreeGen(seed=seed, etype=etype, max_dim=9)
        rctx = fm.Context("ref")
        dctx = fm.Context("device")
        for i in range(count):
            node = gen.tree(depth=5 if etype.is_float else 4)
            env = {n.mat_id: gen.env[n.mat_id] for n in rast.walk(node) if isinstance(n, rast.LEAF_TYPES)}
            orc = roracle.materialize(node, env)
            res = {}
            for label, ctx in (("ref", rctx), ("cjit", dctx)):
                mats = {mid: fm.from_array(arr, ctx=ctx) for mid, arr in env.items()}
                res[label] = _run(ctx, _rebuild(node, mats, ctx), node)
            w.add(f"tree_{etype.value}_{i}", node, env, oracle=orc, **res)
    # 4. view trees (test_backend.py:211-218)
    gen = TreeGen(seed=314, max_dim=16)
    rctx = fm.Context("ref")
    for i in range(30):
        node = gen.view_tree(max_parent=24)
        env = {n.mat_id: gen.env[n.mat_id] for n in rast.walk(node) if isinstance(n, rast.LEAF_TYPES)}
        mats = {mid: fm.from_array(arr, ctx=rctx) for mid, arr in env.items()}
        w.add(f"view_{i}", node, env, oracle=roracle.materialize(node, env),
              ref=_run(rctx, _rebuild(node, mats, rctx), node))
    # 5. GEMM with f64 accumulation (test_backend.py:233-240), plain and folded forms
    r = np.random.default_rng(1)
    a = r.uniform(-1, 1, (64, 48)).astype(np.float32)
    b = r.uniform(-1, 1, (48, 40)).astype(np.float32)
    rctx = fm.Context("ref")
    A, B = fm.from_array(a, ctx=rctx), fm.from_array(b, ctx=rctx)
    e = A @ B
    w.add("gemm_nn", e.node, {A.mat_id: a, B.mat_id: b}, oracle=roracle.materialize(e.node, {A.mat_id: a, B.mat_id: b}),
          ref=_run(rctx, e, e.node))
    bt = np.ascontiguousarray(b.T)
    Bt = fm.from_array(bt, ctx=rctx)
    e = 2 * A @ Bt.t()
    env = {A.mat_id: a, Bt.mat_id: bt}
    w.add("gemm_2abt", e.node, env, oracle=roracle.materialize(e.node, env), ref=_run(rctx, e, e.node))
    # 6. accu known answers of the reference tests (test_matrix.py:139-185)
    ctx = fm.Context("ref")
    x = fm.from_array(np.array([[1, 2], [3, 4]], np.float32), ctx=ctx)
    w.add("accu_small", x._node(), {x.mat_id: x.to_numpy()}, accu_ref=float(fm.accu(x)))
    big = fm.fill(2, 1, 2**31, "u32", ctx=ctx)
    w.add("accu_u32_wrap", big._node(), {big.mat_id: big.to_numpy()}, accu_ref=int(fm.accu(big)))
    # 7. the north-star ops the reference lacks, pinned through what it HAS
    #    (SURVEY 8c): the C4 subexpression materialised by the reference's
    #    compiled backend, its per-column and per-row sums as the reference's
    #    accu of Mat.submat column / row views (matrix.py:258, 481-496), and
    #    dot / norm^2 as the reference's accu(x * y) / accu((x - y)**2).
    #    sum / mean along a dim, max / min / index_max / index_min (numpy
    #    semantics on the reference-computed values), dot and norm are
    #    checked against these by tests/test_oracle.py and the GPU tests.
    for etype, (rows, cols) in (("f64", (64, 24)), ("f64", (200, 7)), ("f32", (48, 33))):
        ctx = fm.Context("device")
        X, Y, Z = (fm.randu(rows, cols, s, etype, ctx) for s in (42, 43, 44))
        e = (X - Y) * Z
        V = fm.Mat(rows, cols, etype, ctx)
        V.assign(e)
        env = {m.mat_id: m.to_numpy() for m in (X, Y, Z)}
        colsum = np.array([float(fm.accu(V.submat(0, j, rows, 1))) for j in range(cols)])
        rowsum = np.array([float(fm.accu(V.submat(i, 0, 1, cols))) for i in range(rows)])
        w.add(f"pin_c4_{etype}_{rows}x{cols}", e.node, env, oracle=roracle.materialize(e.node, env),
              cjit=V.to_numpy(), colsum_ref=colsum, rowsum_ref=rowsum)
    for etype in ("f32", "f64"):
        ctx = fm.Context("device")
        x, y = fm.randu(5000, 1, 7, etype, ctx), fm.randu(5000, 1, 8, etype, ctx)
        e = (x - y) ** 2
        env = {x.mat_id: x.to_numpy(), y.mat_id: y.to_numpy()}
        w.add(f"pin_norm_dot_{etype}", e.node, env, normsq_ref=float(fm.accu(e)),
              dot_ref=float(fm.accu(x * y)))
    w.save()


if __name__ == "__main__":
    rng_fixture()
    signatures_fixture()
    cases_fixture()
    print("golden fixtures written to", HERE)
