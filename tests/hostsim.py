"""A host simulation of the device side -- TESTS ONLY.

`SimBackend` implements the reference Backend contract on numpy buffers and
evaluates every fused launch with the CPU oracle, so the package's host logic
(planning, binding, the sharded API in dist.py) runs on a machine without a
GPU.  `SimComm` stands in for the native collectives of csrc/comm.cu over a
torch.distributed gloo group, restating their combine rules (rank order,
NaN-propagating max/min, first-index arg-select with NaN winning, f64 sums,
wrapping integer sums).  Neither is reachable from the product package.
"""

from __future__ import annotations

import numpy as np

from oracle import fm_oracle as orc
from paper_2604_22242_b200 import dist as D
from paper_2604_22242_b200.backend import Backend, BufferHandle, Capabilities, arg_schema
from paper_2604_22242_b200.exprtree import ElemType, collect_inputs, from_storage, to_storage
from paper_2604_22242_b200.plan import COPY, REDUCE_ACCU, REDUCE_DIM, accumulator_type


class _SimNative:
    def __init__(self, backend):
        self.b = backend

    def call(self, name, *args):
        if name == "fm_memcpy_d2d":
            dst, src, nbytes = int(args[0]), int(args[1]), int(args[2])
            d, s = self.b.bufs[dst], self.b.bufs[src]
            n = nbytes // d.itemsize
            d[:n] = s[:n]
            return
        raise NotImplementedError(f"SimNative: {name}")


class _Kernel:
    def __init__(self, source):
        self.source = source
        self.expr = source.expr
        self.skeleton = source.skeleton_kind
        self.finalize = 0
        self.dim = 0
        self.reduce_kinds = ()


class SimBackend(Backend):
    """numpy buffers + oracle evaluation; pointers are buffer ids."""

    def __init__(self):
        super().__init__()
        self.bufs: dict[int, np.ndarray] = {}
        self.etypes: dict[int, ElemType] = {}
        self.views: dict[int, tuple[int, int]] = {}
        self._next = 1
        self.stream = 0
        self.device = 0
        self.nat = _SimNative(self)
        self.closed = False

    @property
    def capabilities(self):
        return Capabilities(name="sim", compiles_source=False)

    def alloc(self, etype, n_elem):
        etype = ElemType.of(etype)
        h = BufferHandle(self._next, etype, n_elem, self.backend_id)
        self._next += 1
        self.bufs[h.id] = np.zeros(n_elem, etype.dtype)
        return h

    def free(self, handle):
        self.bufs.pop(handle.id)

    def view(self, handle, offset, n_elem):
        h = BufferHandle(self._next, handle.etype, n_elem, self.backend_id)
        self._next += 1
        self.bufs[h.id] = self.bufs[handle.id][offset:offset + n_elem]   # numpy view
        return h

    def release_view(self, handle):
        self.bufs.pop(handle.id)

    def ptr(self, handle):
        return handle.id

    def upload(self, host, handle):
        flat = np.asarray(host).ravel(order="F")
        self.bufs[handle.id][:] = to_storage(flat, handle.etype)

    def download(self, handle):
        return from_storage(self.bufs[handle.id].copy(), handle.etype)

    def synchronize(self):
        pass

    def _arr(self, h, n_rows, n_cols):
        return from_storage(self.bufs[h.id][: n_rows * n_cols].copy(), h.etype).reshape(
            (n_rows, n_cols), order="F")

    def compile(self, source):
        return _Kernel(source)

    def launch(self, kernel, args, geometry, reduce_outputs=None):
        node = kernel.expr
        inputs, _ = collect_inputs(node)
        schema = arg_schema(node, kernel.skeleton)
        roles = [a.role for a in schema]
        env, p, k = {}, 3, 0
        while p < len(roles) and roles[p] == "in":
            h = args[p]
            env[inputs[k].mat_id] = self._arr(h, int(args[p + 1]), int(args[p + 2]))
            p += 3
            while p < len(roles) and roles[p] == "off":
                p += 2
            k += 1
        n_rows, n_cols = geometry
        if kernel.skeleton == REDUCE_DIM:
            v = orc.materialize(node, env)
            for kind, h in reduce_outputs:
                r = orc.reduce_dim(kind, kernel.dim, v, node.etype)
                self.bufs[h.id][: r.size] = to_storage(r.ravel(order="F"), h.etype)
            return
        v = orc.materialize(node, env)
        out = args[0]
        if kernel.skeleton == REDUCE_ACCU:
            acc = accumulator_type(node.etype)
            total = orc.accu(v, node.etype)
            if kernel.finalize == 1:
                total = float(np.sqrt(total))
            self.bufs[out.id][0] = np.array(total).astype(acc.dtype)
            return
        self.bufs[out.id][: v.size] = to_storage(v.ravel(order="F"), out.etype)

    def bind(self, kernel, args):
        return kernel, list(args)

    def _operand(self, prog, rows, cols, etype):
        # a prologue program: materialise it (the reference's temp) into a scratch buffer
        kernel, args = prog
        t = self.alloc(etype, rows * cols)
        args[0] = t
        self.launch(kernel, args, (rows, cols))
        v = self._arr(t, rows, cols)
        self.free(t)
        return v

    def gemm(self, out, a, b, m, n, k, trans_a=False, trans_b=False, alpha=1.0, lda=None,
             ldb=None, precision=0, c_in=None, alpha2=1.0, beta=0.0, a_prog=None, b_prog=None,
             in_etype=None):
        ar, ac = (k, m) if trans_a else (m, k)
        br, bc = (n, k) if trans_b else (k, n)
        A = self._operand(a_prog, ar, ac, in_etype) if a_prog is not None else self._arr(a, ar, ac)
        B = self._operand(b_prog, br, bc, in_etype) if b_prog is not None else self._arr(b, br, bc)
        A = A.T if trans_a else A
        B = B.T if trans_b else B
        C = alpha * (A.astype(np.float64) @ B.astype(np.float64))
        C = C.astype(out.etype.dtype)
        if c_in is not None:
            C = (out.etype.dtype.type(alpha2) * C) + out.etype.dtype.type(beta) * self._arr(c_in, m, n)
        self.bufs[out.id][: m * n] = C.ravel(order="F")

    def randu(self, handle, seed, offset=0):
        v = orc.uniform_fill(seed, handle.n_elem, handle.etype.value, offset=offset)
        self.bufs[handle.id][:] = to_storage(v, handle.etype)

    def fill(self, handle, value):
        self.bufs[handle.id][:] = to_storage(np.full(handle.n_elem, value, np.float64).astype(
            handle.etype.dtype if handle.etype is not ElemType.bf16 else np.float32), handle.etype)


# ---- collectives over gloo --------------------------------------------------------------

def _gather(obj):
    return D.torch_exchange(obj)


def _combine(a, b, op):
    if op == "sum":
        if a.dtype.kind == "f":
            return a + b
        return (a.astype(np.int64) + b.astype(np.int64)).astype(np.uint64).astype(np.uint32).view(a.dtype) \
            if a.dtype == np.int32 else (a.astype(np.uint64) + b.astype(np.uint64)).astype(a.dtype)
    nan = np.isnan(a) | np.isnan(b) if a.dtype.kind == "f" else np.zeros(a.shape, bool)
    r = np.maximum(a, b) if op == "max" else np.minimum(a, b)
    if a.dtype.kind == "f":
        r = np.where(nan, np.nan, r).astype(a.dtype)
    return r


class SimComm(D.Communicator):
    """Communicator over gloo for SimBackend contexts (restated combine rules)."""

    def __init__(self, ctx, rank, world):
        self.ctx, self.rank, self.world = ctx, rank, world
        self.backend = ctx.backend
        self.nat = self.backend.nat
        self._comm = object()
        self.exchange = _gather
        self.transport = "sim"
        self.calls = []

    def allreduce(self, m, op="sum", divisor=0.0):
        self.calls.append(("allreduce", op, m.n_elem, divisor))
        parts = _gather(self.backend.bufs[m.handle.id].copy())
        acc = parts[0].copy()
        for p in parts[1:]:
            acc = _combine(acc, p, op)
        if divisor > 0:
            acc = acc / divisor
        self.backend.bufs[m.handle.id][:] = acc

    def allreduce_arg(self, vals, idx, idx_offset, maximize):
        self.calls.append(("allreduce_arg", maximize, vals.n_elem, idx_offset))
        v = self.backend.bufs[vals.handle.id].astype(np.float64)
        i = self.backend.bufs[idx.handle.id].astype(np.int64) + idx_offset
        parts = _gather((v, i))
        bv, bi = parts[0][0].copy(), parts[0][1].copy()
        for cv, ci in parts[1:]:
            cn, bn = np.isnan(cv), np.isnan(bv)
            if maximize:
                better = (cv > bv) | ((cv == bv) & (ci < bi))
            else:
                better = (cv < bv) | ((cv == bv) & (ci < bi))
            better = np.where(cn | bn, cn & (~bn | (ci < bi)), better)
            bv = np.where(better, cv, bv)
            bi = np.where(better, ci, bi)
        self.backend.bufs[vals.handle.id][:] = bv.astype(self.backend.bufs[vals.handle.id].dtype)
        self.backend.bufs[idx.handle.id][:] = bi.astype(np.uint32)

    def allgather(self, src, dst):
        self.calls.append(("allgather", src.n_elem))
        parts = _gather(self.backend.bufs[src.handle.id].copy())
        self.backend.bufs[dst.handle.id][:] = np.concatenate(parts)

    def status(self):
        return 0

    def close(self):
        pass
