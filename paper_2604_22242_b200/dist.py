"""Column-sharded matrices across GPUs (one process per GPU).

SURVEY.md section 8(e).  The reference has no multi-device code
(`/root/reference/SPEC.md:336-337`); this is the B200 layer the north star
adds on top of the reference API:

* a global n_rows x n_cols column-major matrix is split into contiguous
  column blocks, one per rank -- each block is ONE contiguous slice of the
  column-major element stream, so every elementwise expression over
  identically sharded matrices runs locally with no exchange, and `randu` of
  a shard is exactly that slice of the global splitmix64 stream;
* full reductions (accu / dot / norm): per-rank f64 partial -> one
  allreduce (norm takes the sqrt after the global sum);
* column reductions (dim 0): every column is whole on one rank -> purely
  local, the result stays column-sharded;
* row reductions (dim 1): n_rows-long partials -> allreduce SUM / MAX / MIN
  (mean divides the global f64 sum by the global column count once),
  index_max / index_min -> arg-select of (value, global column) pairs;
* the GEMM `Z_g = s * X_g @ Y.t()` keeps Z row-sharded: X's row block is
  local, Y's column shards are all-gathered.

Every collective goes through libfmb200.so (`fm_allreduce`,
`fm_allreduce_arg`, `fm_allgather`, csrc/comm.cu): one fused peer-memory
kernel per collective (CUDA IPC; NVLink between GPUs) or NCCL's allgather
plus a combine kernel; both combine in rank order, so every rank holds
bit-identical results.  torch.distributed (or any `exchange` callable) is
plumbing only: it carries the NCCL unique id / IPC handles at setup.
"""

from __future__ import annotations

import ctypes
import importlib.util
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import matrix as mx
from .errors import FusematError, ShapeError
from .exprtree import ElemType, MatShape, ReduceKind


# ---------------------------------------------------------------------------------
# partitioning

@dataclass(frozen=True)
class ColumnShard:
    """Columns [col0, col1) of a global n_rows x n_cols matrix on `rank`."""

    n_rows: int
    n_cols: int
    rank: int
    world: int
    col0: int
    col1: int

    @property
    def local_cols(self) -> int:
        return self.col1 - self.col0

    @property
    def elem_offset(self) -> int:
        """Offset of the shard in the global column-major element stream
        (randu of a shard == that slice of the global randu stream)."""
        return self.col0 * self.n_rows


def column_shard(n_rows: int, n_cols: int, rank: int, world: int) -> ColumnShard:
    """Balanced contiguous column blocks: the first n_cols % world ranks get
    one extra column."""
    if world <= 0 or not 0 <= rank < world:
        raise ShapeError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_cols, world)
    col0 = rank * base + min(rank, extra)
    col1 = col0 + base + (1 if rank < extra else 0)
    return ColumnShard(n_rows, n_cols, rank, world, col0, col1)


# ---------------------------------------------------------------------------------
# the communicator (transport in libfmb200.so)

FM_COMM_NCCL, FM_COMM_PEER = 1, 2
_OPS = {"sum": 0, "max": 1, "min": 2}


def torch_exchange(obj) -> list:
    """all_gather_object over the default torch.distributed group (plumbing)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def nccl_library() -> str | None:
    """The libnccl.so.2 torch ships (so one NCCL is loaded per process)."""
    spec = importlib.util.find_spec("nvidia")
    if spec is None or not spec.submodule_search_locations:
        return None
    for base in spec.submodule_search_locations:
        p = Path(base) / "nccl" / "lib" / "libnccl.so.2"
        if p.exists():
            return str(p)
    return None


class Communicator:
    """One rank of the sharded path.

    transport: "auto" (world 1 -> "none"; every rank on its own GPU -> "nccl";
    ranks sharing a GPU -> "peer"), "nccl", "peer" or "none" (world 1 only).
    `exchange(obj) -> list` all-gathers small Python objects across ranks at
    setup (default: torch.distributed's default group)."""

    def __init__(self, ctx: "mx.Context", rank: int, world: int, transport: str = "auto",
                 exchange=None, slot_bytes: int = 8 << 20):
        if world < 1 or not 0 <= rank < world:
            raise FusematError(f"bad rank {rank} of {world}")
        self.ctx, self.rank, self.world = ctx, rank, world
        self.backend = ctx.backend
        self.nat = self.backend.nat
        self._comm = None
        if exchange is None and world > 1:
            exchange = torch_exchange
        self.exchange = exchange
        transport = os.environ.get("FMB200_COMM", transport)
        if transport == "auto":
            if world == 1:
                transport = "none"
            else:
                devices = exchange((os.uname().nodename, self._device_key()))
                transport = "nccl" if len(set(devices)) == world else "peer"
        if transport == "none" and world != 1:
            raise FusematError("transport 'none' needs world size 1")
        self.transport = transport
        if transport == "nccl":
            self._init_nccl()
        elif transport == "peer":
            self._init_peer(slot_bytes)
        elif transport != "none":
            raise FusematError(f"unknown transport {transport!r}")

    def _device_key(self):
        buf = ctypes.create_string_buffer(64)
        self.nat.call("fm_device_pci_bus_id", int(self.backend.device), buf, 64)
        return buf.value.decode()

    def _init_nccl(self) -> None:
        self.nat.call("fm_comm_nccl_load", (nccl_library() or "").encode() or None)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            self.nat.call("fm_comm_nccl_unique_id", uid)
        ids = self.exchange(bytes(uid.raw)) if self.world > 1 else [bytes(uid.raw)]
        c = ctypes.c_void_p()
        self.nat.call("fm_comm_init_nccl", ctypes.byref(c), self.world, self.rank, ids[0])
        self._comm = c.value

    def _init_peer(self, slot_bytes: int) -> None:
        blk = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        self.nat.call("fm_comm_peer_block", ctypes.byref(blk), slot_bytes, h)
        handles = self.exchange(bytes(h.raw)) if self.world > 1 else [bytes(h.raw)]
        c = ctypes.c_void_p()
        self.nat.call("fm_comm_init_peer", ctypes.byref(c), self.world, self.rank, blk,
                      b"".join(handles), slot_bytes)
        self._comm = c.value

    # -- collectives (stream-ordered on the context's stream) -----------------------------

    def allreduce(self, m: "mx.Mat", op: str = "sum", divisor: float = 0.0) -> None:
        """In place: m = op over ranks of m (rank order).  `divisor` > 0
        divides the combined value (f64 mean)."""
        if self._comm is None:
            if divisor > 0:
                raise FusematError("allreduce with a divisor needs a transport")
            return
        self.nat.call("fm_allreduce", self._comm, self.backend.ptr(m.handle), m.n_elem,
                      m.etype.code, _OPS[op], float(divisor), self.backend.stream)

    def allreduce_arg(self, vals: "mx.Mat", idx: "mx.Mat", idx_offset: int, maximize: bool) -> None:
        """In place: per element the (value, index) of the extreme over ranks
        (first index on ties, NaN wins); this rank's indices get idx_offset."""
        if vals.n_elem != idx.n_elem or idx.etype is not ElemType.u32:
            raise ShapeError("allreduce_arg: values and u32 indices of equal length")
        if self._comm is None:
            if idx_offset:
                idx.assign(idx + idx_offset)
            return
        self.nat.call("fm_allreduce_arg", self._comm, self.backend.ptr(vals.handle),
                      self.backend.ptr(idx.handle), vals.n_elem, vals.etype.code, idx_offset,
                      int(maximize), self.backend.stream)

    def allgather(self, src: "mx.Mat", dst: "mx.Mat") -> None:
        """dst = the ranks' src buffers concatenated in rank order."""
        w = src.etype.width
        if dst.n_elem != src.n_elem * self.world or dst.etype is not src.etype:
            raise ShapeError("allgather: dst must hold world x src elements of the same type")
        if self._comm is None:
            self.nat.call("fm_memcpy_d2d", self.backend.ptr(dst.handle), self.backend.ptr(src.handle),
                          src.n_elem * w, self.backend.stream)
            return
        self.nat.call("fm_allgather", self._comm, self.backend.ptr(src.handle), src.n_elem * w,
                      self.backend.ptr(dst.handle), self.backend.stream)

    def status(self) -> int:
        """Nonzero if a peer-transport wait timed out (results then invalid)."""
        if self._comm is None:
            return 0
        e = ctypes.c_int64()
        self.nat.call("fm_comm_status", self._comm, ctypes.byref(e))
        return e.value

    def close(self) -> None:
        if self._comm is not None:
            self.nat.call("fm_comm_destroy", self._comm)
            self._comm = None


# ---------------------------------------------------------------------------------
# sharded matrices and expressions

class _ShardOps:
    """Operators on column-sharded operands: applied to the local shards
    (elementwise work needs no exchange)."""

    comm: Communicator
    shape: MatShape

    def _local(self) -> "mx.MatExpr":
        raise NotImplementedError

    def _peer(self, other) -> "mx.MatExpr | float":
        if isinstance(other, _ShardOps):
            if other.comm is not self.comm or other.shape != self.shape:
                raise ShapeError(f"sharded operands differ: {self.shape} vs {other.shape}")
            return other._local()
        if isinstance(other, (mx.Mat, mx.MatExpr)):
            raise ShapeError("cannot combine a sharded matrix with an unsharded one")
        return other

    def _wrap(self, local: "mx.MatExpr") -> "ShardedExpr":
        return ShardedExpr(local, self.comm, self.shape)

    def __add__(self, o): return self._wrap(self._local() + self._peer(o))
    def __radd__(self, o): return self._wrap(self._peer(o) + self._local())
    def __sub__(self, o): return self._wrap(self._local() - self._peer(o))
    def __rsub__(self, o): return self._wrap(self._peer(o) - self._local())
    def __mul__(self, o): return self._wrap(self._local() * self._peer(o))
    def __rmul__(self, o): return self._wrap(self._peer(o) * self._local())
    def __mod__(self, o): return self._wrap(self._local() % self._peer(o))
    def __truediv__(self, o): return self._wrap(self._local() / self._peer(o))
    def __rtruediv__(self, o): return self._wrap(self._peer(o) / self._local())
    def __neg__(self): return self._wrap(-self._local())
    def __gt__(self, o): return self._wrap(self._local() > o)
    def __pow__(self, k): return self._wrap(self._local() ** k)
    def __abs__(self): return self._wrap(abs(self._local()))

    def t(self):
        raise ShapeError("transposing a column-sharded matrix breaks shard locality; "
                         "gather it first (allgather)")

    def __matmul__(self, other):
        raise ShapeError("sharded products: use dist.matmul_row_shard")

    @property
    def etype(self) -> ElemType:
        return self._local().etype

    def _apply(self, fn) -> "ShardedExpr":
        return self._wrap(fn(self._local()))


class ShardedExpr(_ShardOps):
    """A lazy expression over identically column-sharded matrices."""

    def __init__(self, local: "mx.MatExpr", comm: Communicator, shape: MatShape):
        self.local, self.comm, self.shape = mx.as_expr(local), comm, shape

    def _local(self):
        return self.local

    def __repr__(self) -> str:
        return f"ShardedExpr({self.shape}, {self.etype.value}, rank {self.comm.rank}/{self.comm.world})"


class ShardedMat(_ShardOps):
    """Global n_rows x n_cols column-major matrix; this rank holds columns
    [shard.col0, shard.col1) as an ordinary `Mat` (`local`)."""

    def __init__(self, n_rows: int, n_cols: int, etype="f32", comm: Communicator | None = None):
        if comm is None:
            raise FusematError("a ShardedMat needs a Communicator")
        self.comm = comm
        self.shape = MatShape(int(n_rows), int(n_cols))
        self.shard = column_shard(self.shape.n_rows, self.shape.n_cols, comm.rank, comm.world)
        self.local = mx.Mat(self.shape.n_rows, self.shard.local_cols, etype, comm.ctx)

    def _local(self):
        return mx.as_expr(self.local)

    @property
    def etype(self) -> ElemType:
        return self.local.etype

    @property
    def n_rows(self) -> int:
        return self.shape.n_rows

    @property
    def n_cols(self) -> int:
        return self.shape.n_cols

    def assign(self, value) -> "ShardedMat":
        """Elementwise: local fused launch.  A dim-0 reduction of a sharded
        expression into a 1 x n_cols ShardedMat: local too."""
        if isinstance(value, ShardedReduce):
            assign_all([(self, value)])
            return self
        if not isinstance(value, _ShardOps):
            raise ShapeError("assign a sharded expression to a sharded matrix")
        self._peer(value)
        self.local.assign(value._local())
        return self

    def randu(self, seed: int) -> "ShardedMat":
        """This shard's slice of the global splitmix64 stream (`rng.py:54-64`)."""
        self.comm.backend.randu(self.local.handle, seed, offset=self.shard.elem_offset)
        return self

    def set_global(self, values) -> "ShardedMat":
        arr = np.asarray(values)
        if arr.ndim == 1:
            arr = arr.reshape(-1, 1)
        if arr.shape != (self.n_rows, self.n_cols):
            raise ShapeError(f"values shape {arr.shape} != {self.shape}")
        self.local.set_values(arr[:, self.shard.col0:self.shard.col1])
        return self

    def allgather(self, out: "mx.Mat | None" = None) -> "mx.Mat":
        """The whole matrix on every rank (needs equal shards: n_cols % world == 0)."""
        if self.n_cols % self.comm.world:
            raise ShapeError("allgather needs n_cols divisible by the world size")
        if out is None:
            out = mx.Mat(self.n_rows, self.n_cols, self.etype, self.comm.ctx)
        elif out.shape != self.shape or out.etype is not self.etype:
            raise ShapeError("allgather output must have the global shape and type")
        self.comm.allgather(self.local, out)
        return out

    def to_numpy(self) -> np.ndarray:
        """Synchronise and assemble the global matrix on the host (every rank)."""
        if self.n_cols % self.comm.world == 0:
            return self.allgather().to_numpy()
        parts = self.comm.exchange(self.local.to_numpy()) if self.comm.world > 1 else [self.local.to_numpy()]
        return np.concatenate(parts, axis=1)

    def __repr__(self) -> str:
        return (f"ShardedMat({self.shape}, {self.etype.value}, cols {self.shard.col0}:{self.shard.col1} "
                f"on rank {self.comm.rank}/{self.comm.world})")


class ShardedReduce:
    """sum / mean / max / min / index_max / index_min of a sharded expression
    along `dim` (lazy, so `assign_all` can fuse several into one pass)."""

    def __init__(self, kind: ReduceKind, dim: int, child: _ShardOps):
        if dim not in (0, 1):
            raise ShapeError(f"reduction dim must be 0 or 1, got {dim}")
        self.kind, self.dim, self.child = kind, dim, child
        self.comm = child.comm
        self.local = mx._reduction(kind, child._local(), dim)      # shape / etype checks
        self.etype = self.local.etype

    @property
    def shape(self) -> MatShape:
        n_rows, n_cols = self.child.shape.n_rows, self.child.shape.n_cols
        return MatShape(1, n_cols) if self.dim == 0 else MatShape(n_rows, 1)

    def eval(self):
        if self.dim == 0:
            out = ShardedMat(1, self.child.shape.n_cols, self.etype, self.comm)
        else:
            out = mx.Mat(self.child.shape.n_rows, 1, self.etype, self.comm.ctx)
        assign_all([(out, self)])
        return out


def is_sharded(value) -> bool:
    return isinstance(value, (_ShardOps, ShardedReduce))


# ---------------------------------------------------------------------------------
# reductions

def assign_all(pairs) -> None:
    """Several reductions of sharded expressions in one plan.

    dim 0 (outputs: 1 x n_cols ShardedMats) -> the local fused multi-output
    launch, no exchange.  dim 1 (outputs: n_rows x 1 Mats, identical on every
    rank) -> one local fused launch of all the partials a child needs, then
    one collective per partial kind:
      sum / mean -> f64 partial sums, allreduce SUM (mean: / global n_cols),
                    rounded once to the output type;
      max / min  -> allreduce MAX / MIN in the element type (NaN propagates);
      index_*    -> local (extreme, local column) pairs, arg-select over
                    ranks on (value, col0 + column)."""
    pairs = list(pairs)
    if not pairs:
        return
    comm = pairs[0][1].comm
    if comm.world == 1:                 # one shard is the whole matrix: plain fused launches
        mx.assign_all([(o.local if isinstance(o, ShardedMat) else o,
                        v.local if isinstance(v, ShardedReduce) else v._local()) for o, v in pairs])
        return
    local_pairs, post = [], []
    partials: dict = {}
    ctx = comm.ctx
    for out, val in pairs:
        if not isinstance(val, ShardedReduce):
            if isinstance(out, ShardedMat) and isinstance(val, _ShardOps):
                local_pairs.append((out.local, val._local()))
                continue
            raise ShapeError("dist.assign_all takes sharded expressions / reductions")
        if val.comm is not comm:
            raise FusematError("dist.assign_all across communicators")
        if val.dim == 0:
            if not isinstance(out, ShardedMat) or out.shape != val.shape:
                raise ShapeError("a dim-0 reduction of a sharded matrix goes to a 1 x n_cols ShardedMat")
            local_pairs.append((out.local, val.local))
            continue
        if not isinstance(out, mx.Mat) or out.etype is not val.etype:
            raise ShapeError(f"a dim-1 reduction goes to an n_rows x 1 {val.etype.value} Mat")
        if out.shape != val.shape:
            out._realloc(val.shape)
        child = val.child._local()
        key = id(val.child)
        n_rows = val.child.shape.n_rows
        k = val.kind
        if k in (ReduceKind.sum, ReduceKind.mean):
            # f64 partial sums of the row (float children); ints wrap in their type
            if child.etype.is_float:
                tag = ("sum64", key)
                if tag not in partials:
                    src = child if child.etype is ElemType.f64 else mx.conv_to(child, "f64")
                    partials[tag] = mx.Mat(n_rows, 1, "f64", ctx)
                    local_pairs.append((partials[tag], mx.sum(src, 1)))
                post.append(("sum", out, partials[tag], k is ReduceKind.mean, val))
            else:
                tag = ("sumi", key)
                if tag not in partials:
                    partials[tag] = mx.Mat(n_rows, 1, child.etype, ctx)
                    local_pairs.append((partials[tag], mx.sum(child, 1)))
                post.append(("sum", out, partials[tag], False, val))
        elif k in (ReduceKind.max, ReduceKind.min):
            tag = (k, key)
            if tag not in partials:
                partials[tag] = mx.Mat(n_rows, 1, child.etype, ctx)
                local_pairs.append((partials[tag], mx._reduction(k, child, 1)))
            post.append(("ext", out, partials[tag], k is ReduceKind.max, val))
        else:
            if not child.etype.is_float:
                raise ShapeError("sharded index_max / index_min need a float expression")
            ext = ReduceKind.max if k is ReduceKind.index_max else ReduceKind.min
            tag = (ext, key)
            if tag not in partials:
                partials[tag] = mx.Mat(n_rows, 1, child.etype, ctx)
                local_pairs.append((partials[tag], mx._reduction(ext, child, 1)))
            vals = mx.Mat(n_rows, 1, child.etype, ctx)
            local_pairs.append((out, mx._reduction(k, child, 1)))
            post.append(("arg", out, (partials[tag], vals), k is ReduceKind.index_max, val))
    if local_pairs:
        mx.assign_all(local_pairs)
    for kind, out, part, flag, val in post:
        if kind == "sum":
            if part.etype is ElemType.f64:
                tmp = mx.Mat(part.n_rows, 1, "f64", ctx)
                comm.nat.call("fm_memcpy_d2d", comm.backend.ptr(tmp.handle), comm.backend.ptr(part.handle),
                              part.n_elem * 8, comm.backend.stream)
                comm.allreduce(tmp, "sum", float(val.child.shape.n_cols) if flag else 0.0)
                if out.etype is ElemType.f64:
                    out.assign(tmp)
                else:
                    out.assign(mx.conv_to(tmp, out.etype))
            else:
                comm.nat.call("fm_memcpy_d2d", comm.backend.ptr(out.handle), comm.backend.ptr(part.handle),
                              part.n_elem * part.etype.width, comm.backend.stream)
                comm.allreduce(out, "sum")
        elif kind == "ext":
            comm.nat.call("fm_memcpy_d2d", comm.backend.ptr(out.handle), comm.backend.ptr(part.handle),
                          part.n_elem * part.etype.width, comm.backend.stream)
            comm.allreduce(out, "max" if flag else "min")
        else:
            ext, vals = part
            comm.nat.call("fm_memcpy_d2d", comm.backend.ptr(vals.handle), comm.backend.ptr(ext.handle),
                          ext.n_elem * ext.etype.width, comm.backend.stream)
            shard = column_shard(val.child.shape.n_rows, val.child.shape.n_cols, comm.rank, comm.world)
            comm.allreduce_arg(vals, out, shard.col0, flag)


def _full_partial(value, finalize_sq: bool) -> tuple["mx.Mat", Communicator]:
    """This rank's accumulator (f64 for floats) of accu(value) -- or of
    accu(square(value)) for norm -- in a 1x1 device matrix, allreduced."""
    comm = value.comm
    local = value._local()
    out = mx.Mat(1, 1, "f64" if local.etype.is_float else local.etype, comm.ctx)
    if finalize_sq:
        mx.norm_async(local, out, 0, squared=True)
    else:
        mx.accu_async(local, out, 0)
    comm.allreduce(out, "sum")
    return out, comm


def accu(value):
    out, _ = _full_partial(value, False)
    v = out.to_numpy()[0, 0]
    return float(v) if out.etype.is_float else int(v)


def dot(a, b):
    if not isinstance(a, _ShardOps) or not isinstance(b, _ShardOps):
        raise ShapeError("dot of sharded operands needs both sharded")
    if a.shape != b.shape:
        raise ShapeError(f"dot: shapes {a.shape} and {b.shape} differ")
    return accu(a % b)


def norm(value, p: int = 2):
    if p != 2:
        raise ShapeError("only the 2-norm is supported")
    if not value.etype.is_float:
        raise ShapeError("norm requires a float expression")
    out, _ = _full_partial(value, True)
    return float(np.sqrt(out.to_numpy()[0, 0]))


# ---------------------------------------------------------------------------------
# row-sharded GEMM

def matmul_row_shard(x_rows: "mx.Mat", y: ShardedMat, alpha: float = 1.0, out: "mx.Mat | None" = None,
                     y_full: "mx.Mat | None" = None) -> "mx.Mat":
    """Z[rows_g, :] = alpha * X[rows_g, :] @ Y.t() on every rank g.

    X's row block is local (`x_rows`, (M/p) x K); Y (N x K) is column-sharded,
    i.e. split along the contraction dimension, so its shards are gathered
    (`fm_allgather`: NCCL or peer memory) into `y_full` and the product runs
    as one tcgen05 launch with the scale and transpose folded in.  Z stays
    row-sharded ((M/p) x N per rank)."""
    if x_rows.n_cols != y.n_cols:
        raise ShapeError(f"inner dimensions differ: {x_rows.n_cols} vs {y.n_cols}")
    y_full = y.allgather(y_full)
    if out is None:
        out = mx.Mat(x_rows.n_rows, y.n_rows, "f32" if x_rows.etype is not ElemType.f64 else "f64",
                     x_rows.ctx)
    out.assign(alpha * x_rows @ y_full.t())
    return out


def row_block(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) of the row-sharded GEMM output on `rank` (balanced)."""
    s = column_shard(1, n_rows, rank, world)
    return s.col0, s.col1
