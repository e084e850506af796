"""Multi-GPU column sharding (one process per GPU, torch.distributed plumbing).

SURVEY.md section 8(e): in column-major storage a block of n_cols/p columns
is one contiguous slice, so every elementwise expression over identically
sharded matrices runs locally with no communication; only reduction partials
cross NVLink:

* full reductions (accu / dot / norm): per-rank f64 partial -> all_reduce(SUM)
  (norm takes the sqrt after the global sum);
* column reductions (dim 0): every column is whole on one rank -> purely
  local, results stay column-sharded (allgather on request);
* row reductions (dim 1): n_rows-long partials -> all_reduce(SUM / MAX / MIN);
  index_max / index_min -> all_gather of (value, global index) candidates
  and a first-index select (NCCL has no argmax).

The collectives take torch tensors so the same code runs over NCCL on GPUs
and over gloo on CPU (tests/test_dist.py).  Device buffers are handed to
torch zero-copy through __cuda_array_interface__.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ShapeError


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


class CudaArrayView:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (int(ptr), False), "version": 3,
            "strides": None,
        }


_TYPESTR = {"f32": "<f4", "f64": "<f8", "u32": "<u4", "i32": "<i4"}


def torch_view(backend, handle, device: int):
    """Zero-copy torch tensor over a device buffer (for NCCL collectives)."""
    import torch
    view = CudaArrayView(backend.ptr(handle), handle.n_elem, _TYPESTR[handle.etype.value])
    return torch.as_tensor(view, device=f"cuda:{device}")


# -- combine steps (device-agnostic: torch tensors, any process group) -----------

def allreduce_sum(t, group=None):
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def combine_norm(sum_sq_total: float) -> float:
    return float(np.sqrt(sum_sq_total))


def combine_arg_candidates(values, indices, maximize: bool, group=None):
    """First-index arg-max/min across ranks.

    values/indices: 1-D tensors (per row) of this rank's best value and its
    GLOBAL column index.  Returns (values, indices) of the global winner with
    numpy semantics: NaN wins (first NaN), ties keep the lowest index."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    vs = [torch.empty_like(values) for _ in range(world)]
    ix = [torch.empty_like(indices) for _ in range(world)]
    dist.all_gather(vs, values, group=group)
    dist.all_gather(ix, indices, group=group)
    best_v, best_i = vs[0].clone(), ix[0].clone()
    for v, i in zip(vs[1:], ix[1:]):
        vn, bn = torch.isnan(v), torch.isnan(best_v)
        if maximize:
            better = (v > best_v) | ((v == best_v) & (i < best_i))
        else:
            better = (v < best_v) | ((v == best_v) & (i < best_i))
        better = torch.where(vn | bn, vn & (~bn | (i < best_i)), better)
        best_v = torch.where(better, v, best_v)
        best_i = torch.where(better, i, best_i)
    return best_v, best_i


def allreduce_rowstats(sums=None, maxs=None, mins=None, group=None):
    """Row-reduction partials (dim 1) over column shards."""
    import torch.distributed as dist
    if sums is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    # NCCL / gloo MAX and MIN do not propagate NaN the way numpy's max/min
    # (and the device kernels) do: carry a NaN count beside the extrema and
    # restore NaN wherever any rank saw one.
    for t, op in ((maxs, dist.ReduceOp.MAX), (mins, dist.ReduceOp.MIN)):
        if t is None:
            continue
        nan = t.isnan().to(t.dtype)
        dist.all_reduce(nan, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(t, op=op, group=group)
        t[nan > 0] = float("nan")
    return sums, maxs, mins
