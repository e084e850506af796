"""CPU oracle for the fused-expression path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module, and only as the checker or the
timed CPU baseline.  The product (paper_2604_22242_b200) never imports it and
has no CPU fallback.

A numpy restatement of the reference's evaluation:

* `materialize` restates the per-node oracle of
  /root/reference/pkg/src/fusemat/oracle.py:29-101 (every node into its own
  array, bottom-up, numpy arithmetic at the node's element type) and extends
  it to the ops the reference lacks (abs, bf16, reductions along a dim);
* `accu` restates the reduce_accu skeleton (codegen.py:94-114,
  backend.py:319-332): f64 accumulator for floats (here an exactly rounded
  math.fsum, which the reference's serial sum approximates), wrapping
  element-type sum for integers;
* `uniform_fill` / `uniform_int_fill` restate rng.py:35-72 bit for bit;
* `gemm` restates the f64-accumulated product (oracle.py:53-57, cjit.py:33-51);
* `compare` / `allclose_mixed` restate oracle.py:104-146; `max_ulp` is new.

Pinning: tests/test_oracle.py checks this module against the golden vectors
in tests/golden/ that tests/golden/make_golden.py produced by importing the
reference package itself (its RefBackend, oracle.materialize, CJitBackend and
rng), plus the reference tests' own known answers.

Transcendental policy: with transcendental="cr" (the
default) f32 exp/log/tanh are evaluated in f64 and rounded once -- correctly
rounded in practice -- because the reference's own numpy/glibc f32
transcendentals are host-dependent and up to 2-4 ulp off.
transcendental="numpy" reproduces the reference oracle exactly.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2604_22242_b200 import exprtree as ast  # the tree is the shared input
from paper_2604_22242_b200.exprtree import (
    BinaryElem, BinaryKind, Diag, ElemType, Leaf, MatMul, Reduce, ReduceKind, Subview,
    Transpose, UnaryElem, UnaryKind,
)

# -- rng (rng.py:35-72) ------------------------------------------------------------

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z.copy()
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def raw_words(seed: int, n: int, offset: int = 0) -> np.ndarray:
    with np.errstate(over="ignore"):
        k = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return mix64(k * GOLDEN + np.uint64(seed))


def uniform_fill(seed: int, n: int, etype, offset: int = 0) -> np.ndarray:
    ety = ElemType.of(etype)
    w = raw_words(seed, n, offset)
    if ety is ElemType.f64:
        return (w >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    f = ((w >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).astype(np.float32)
    if ety is ElemType.bf16:
        return bf16_round(f)
    return f


def uniform_int_fill(seed: int, n: int, etype, high: int, offset: int = 0) -> np.ndarray:
    w = raw_words(seed, n, offset)
    return ((w >> np.uint64(32)) % np.uint64(high)).astype(ElemType.of(etype).dtype)


def randu(n_rows: int, n_cols: int, seed: int, etype="f32") -> np.ndarray:
    """2-D column-major randu as the reference lays it out (matrix.py:407-414)."""
    return uniform_fill(seed, n_rows * n_cols, etype).reshape((n_rows, n_cols), order="F")


# -- bf16 (held as bf16-representable float32) --------------------------------------

def bf16_round(x) -> np.ndarray:
    """Round float32 values to the nearest-even bf16 value."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    nan = np.isnan(a)
    r[nan] = ((u[nan] | 0x400000) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).reshape(a.shape)


def bf16_from_f64(x) -> np.ndarray:
    """Single rounding f64 -> bf16 (round to odd into f32, then to bf16)."""
    d = np.asarray(x, dtype=np.float64)
    f = d.astype(np.float32)                          # RNE
    # replace by round-toward-zero with a sticky bit (round to odd)
    fz = np.where(np.abs(f.astype(np.float64)) > np.abs(d),
                  np.nextafter(f, np.float32(0)), f).astype(np.float32)
    u = np.ascontiguousarray(fz).view(np.uint32).copy()
    inexact = (fz.astype(np.float64) != d) & np.isfinite(fz)
    u[inexact] |= 1
    return bf16_round(u.view(np.float32))


# -- per-node materialisation (oracle.py:29-101 + extensions) ----------------------------

def _np_dtype(ety: ElemType):
    return np.float32 if ety is ElemType.bf16 else ety.dtype.type


def materialize(node, env: dict, transcendental: str = "cr") -> np.ndarray:
    """Evaluate `node` bottom-up; env maps mat_id -> 2-D array (bf16 matrices
    as float32 values)."""
    with np.errstate(all="ignore"):
        return _mat(node, env, transcendental)


def _round(ety: ElemType, x: np.ndarray) -> np.ndarray:
    return bf16_round(x) if ety is ElemType.bf16 else x


def _transc(kind: UnaryKind, x: np.ndarray, ety: ElemType, mode: str) -> np.ndarray:
    fn = {UnaryKind.exp: np.exp, UnaryKind.log: np.log, UnaryKind.tanh: np.tanh}[kind]
    if ety is ElemType.f64 or mode == "numpy":
        return fn(x)
    return fn(x.astype(np.float64)).astype(np.float32)


def _mat(node, env, mode) -> np.ndarray:
    if isinstance(node, Leaf):
        arr = np.asarray(env[node.mat_id])
        if arr.shape != (node.shape.n_rows, node.shape.n_cols):
            raise ValueError(f"env array for {node.mat_id} has shape {arr.shape}")
        return arr.astype(_np_dtype(node.etype), copy=True)
    if isinstance(node, Subview):
        p = np.asarray(env[node.mat_id])
        r0, c0 = node.row_off, node.col_off
        return p[r0:r0 + node.shape.n_rows, c0:c0 + node.shape.n_cols].astype(_np_dtype(node.etype))
    if isinstance(node, Diag):
        p = np.asarray(env[node.mat_id])
        return np.diagonal(p, offset=node.k).reshape(-1, 1).astype(_np_dtype(node.etype))
    if isinstance(node, Transpose):
        return _mat(node.child, env, mode).T.copy()
    if isinstance(node, MatMul):
        a, b = _mat(node.left, env, mode), _mat(node.right, env, mode)
        return gemm(a, b, out=node.etype)
    if isinstance(node, BinaryElem):
        a, b = _mat(node.left, env, mode), _mat(node.right, env, mode)
        k = node.kind
        if k is BinaryKind.plus:
            r = a + b
        elif k is BinaryKind.minus:
            r = a - b
        elif k is BinaryKind.schur:
            r = a * b
        else:
            r = a / b
        return _round(node.etype, r)
    if isinstance(node, UnaryElem):
        x = _mat(node.child, env, mode)
        src = node.child.etype
        dt = _np_dtype(src)
        k = node.kind
        if k is UnaryKind.scalar_add:
            r = x + dt(node.scalar)
        elif k is UnaryKind.scalar_pre_mul:
            r = dt(node.scalar) * x
        elif k is UnaryKind.scalar_pre_div:
            r = dt(node.scalar) / x
        elif k is UnaryKind.gt_scalar:
            r = (x > dt(node.scalar)).astype(dt)
        elif k is UnaryKind.neg:
            r = -x
        elif k is UnaryKind.abs:
            r = np.abs(x)
        elif k in (UnaryKind.exp, UnaryKind.log, UnaryKind.tanh):
            r = _transc(k, x, src, mode)
        elif k is UnaryKind.sqrt:
            r = np.sqrt(x)
        elif k is UnaryKind.pow_int:
            if node.exponent == 0:
                r = np.ones_like(x)
            else:
                r = x.copy()
                for _ in range(node.exponent - 1):
                    r = r * x
        elif k is UnaryKind.conv:
            return _convert(x, src, node.target)
        else:
            raise ValueError(f"oracle: unary kind {k}")
        return _round(node.etype, r.astype(dt, copy=False))
    if isinstance(node, Reduce):
        return reduce_dim(node.kind, node.dim, _mat(node.child, env, mode), node.child.etype)
    raise ValueError(f"oracle: node {type(node).__name__}")


def _to_int_bits(x: np.ndarray) -> np.ndarray:
    """Float -> int64 with x86 cvtt semantics (NaN / overflow -> INT64_MIN)."""
    xd = x.astype(np.float64)
    bad = ~np.isfinite(xd) | (xd >= 2.0 ** 63) | (xd < -2.0 ** 63)
    out = np.where(bad, 0.0, np.trunc(xd)).astype(np.int64)
    out[bad] = np.iinfo(np.int64).min
    return out


def _convert(x: np.ndarray, src: ElemType, dst: ElemType) -> np.ndarray:
    if dst is ElemType.bf16:
        if src is ElemType.f32 or src is ElemType.bf16:
            return bf16_round(x)
        return bf16_from_f64(x.astype(np.float64))
    if dst.is_float:
        return x.astype(dst.dtype)
    if src.is_float:
        return _to_int_bits(x).astype(dst.dtype)     # wrap to 32 bits
    return x.astype(dst.dtype)


# -- reductions ---------------------------------------------------------------------------

def accu(values: np.ndarray, ety: ElemType) -> float | int:
    """reduce_accu: exactly rounded f64 sum for floats, wrapping sum for ints."""
    v = np.asarray(values).ravel(order="F")
    if ety.is_float:
        return math.fsum(v.astype(np.float64).tolist()) if v.size < 4_000_000 else _fsum_big(v)
    total = int(v.astype(np.uint64).sum(dtype=np.uint64)) if ety is ElemType.u32 else int(
        v.astype(np.int64).sum())
    return int(np.array(total & 0xFFFFFFFF).astype(np.uint32).astype(ety.dtype))


def _fsum_big(v: np.ndarray) -> float:
    parts = [math.fsum(c.astype(np.float64).tolist()) for c in np.array_split(v, max(1, v.size // 2_000_000))]
    return math.fsum(parts)


def reduce_dim(kind: ReduceKind, dim: int, x: np.ndarray, ety: ElemType) -> np.ndarray:
    """sum / mean / max / min / index_max / index_min along `dim` with numpy
    NaN semantics (NaN propagates, first NaN index wins, ties -> first)."""
    axis = 0 if dim == 0 else 1
    keep = (lambda a: a.reshape(1, -1)) if dim == 0 else (lambda a: a.reshape(-1, 1))
    out_dt = _np_dtype(ety)
    if kind in (ReduceKind.sum, ReduceKind.mean):
        if ety.is_float:
            s = np.sum(x.astype(np.float64), axis=axis)
            if kind is ReduceKind.mean:
                s = s / float(x.shape[axis])
            if ety is ElemType.bf16:
                return keep(bf16_from_f64(s))
            return keep(s.astype(out_dt))
        s = np.sum(x.astype(np.int64), axis=axis) & 0xFFFFFFFF
        return keep(s.astype(np.uint32).astype(out_dt))
    if kind is ReduceKind.max:
        return keep(np.max(x, axis=axis).astype(out_dt))
    if kind is ReduceKind.min:
        return keep(np.min(x, axis=axis).astype(out_dt))
    if kind is ReduceKind.index_max:
        return keep(np.argmax(x, axis=axis).astype(np.uint32))
    return keep(np.argmin(x, axis=axis).astype(np.uint32))


def gemm(a: np.ndarray, b: np.ndarray, out: ElemType = ElemType.f32) -> np.ndarray:
    """f64-accumulated product, rounded once (oracle.py:53-57)."""
    c = a.astype(np.float64) @ b.astype(np.float64)
    return c if out is ElemType.f64 else c.astype(np.float32)


# -- comparators (oracle.py:104-146) ---------------------------------------------------------

def compare(actual, expected) -> float:
    a = np.asarray(actual, dtype=np.float64)
    b = np.asarray(expected, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"compare: shapes {a.shape} vs {b.shape}")
    ok = (np.isnan(a) & np.isnan(b)) | (np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b)))
    with np.errstate(all="ignore"):
        err = np.abs(a - b) / np.maximum(np.abs(b), 1e-30)
    err = np.where(ok, 0.0, err)
    bad = (np.isnan(a) != np.isnan(b)) | (np.isinf(a) != np.isinf(b))
    err = np.where(bad & ~ok, np.inf, err)
    return float(np.max(err)) if err.size else 0.0


def allclose_mixed(actual, expected, rtol=1e-4, atol=1e-4) -> bool:
    a = np.asarray(actual, dtype=np.float64)
    b = np.asarray(expected, dtype=np.float64)
    special = (np.isnan(a) & np.isnan(b)) | (np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b)))
    with np.errstate(all="ignore"):
        close = np.abs(a - b) <= atol + rtol * np.abs(b)
    return bool(np.all(special | close))


def _ordered(x: np.ndarray) -> np.ndarray:
    """Map floats to integers whose difference counts ulps."""
    if x.dtype == np.float64:
        i = x.view(np.int64).astype(np.int64)
        return np.where(i < 0, np.int64(-0x8000000000000000) - i, i)
    i = np.ascontiguousarray(x.astype(np.float32)).view(np.int32).astype(np.int64)
    return np.where(i < 0, -0x80000000 - i, i)


def max_ulp(actual, expected) -> int:
    """Largest ulp distance (NaN==NaN); bf16 arrays compare in f32 ulps."""
    a = np.asarray(actual)
    b = np.asarray(expected)
    if a.dtype.kind in "iu":
        return int(np.max(np.abs(a.astype(np.int64) - b.astype(np.int64)))) if a.size else 0
    dt = np.float64 if (a.dtype == np.float64 or b.dtype == np.float64) else np.float32
    a = np.ascontiguousarray(a.astype(dt))
    b = np.ascontiguousarray(b.astype(dt))
    both_nan = np.isnan(a) & np.isnan(b)
    d = np.abs(_ordered(a) - _ordered(b))
    d = np.where(both_nan, 0, d)
    d = np.where(np.isnan(a) != np.isnan(b), np.iinfo(np.int64).max, d)
    return int(d.max()) if d.size else 0


def ulp_histogram(actual, expected) -> dict:
    a = np.ascontiguousarray(np.asarray(actual, dtype=np.float32))
    b = np.ascontiguousarray(np.asarray(expected, dtype=np.float32))
    d = np.abs(_ordered(a) - _ordered(b))
    vals, counts = np.unique(np.minimum(d, 10), return_counts=True)
    return {int(v): int(c) for v, c in zip(vals, counts)}
