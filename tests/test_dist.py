"""World-size-2 gloo tests of the column-sharded combine logic.

The N>1 path is: every rank owns a contiguous column block (a contiguous
slice of the column-major element stream, so randu of a shard equals that
slice of the global randu stream); elementwise work is local; only reduction
partials cross ranks.  These tests run that host logic over gloo on CPU with
the oracle supplying each rank's local partials, and check the combined
result against the single-process oracle on the whole matrix.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fm_oracle as orc
from paper_2604_22242_b200.dist import (allreduce_rowstats, allreduce_sum, column_shard,
                                        combine_arg_candidates, combine_norm)
from paper_2604_22242_b200.errors import ShapeError


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    port = _free_port()
    mp.start_processes(_entry, args=(world, port, fn, args), nprocs=world, join=True,
                       start_method="spawn")


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ---- rank bodies (module-level so spawn can pickle them) -----------------------------

def _body_full_reductions(rank, world, n_rows, n_cols):
    sh = column_shard(n_rows, n_cols, rank, world)
    n_loc = sh.n_rows * sh.local_cols
    for ety in (orc.ElemType.f32, orc.ElemType.f64):
        x = orc.uniform_fill(42, n_loc, ety.value, offset=sh.elem_offset)
        y = orc.uniform_fill(43, n_loc, ety.value, offset=sh.elem_offset)
        part = torch.tensor([orc.accu(x * y, ety), orc.accu((x - y) * (x - y), ety)], dtype=torch.float64)
        allreduce_sum(part)
        gx = orc.uniform_fill(42, n_rows * n_cols, ety.value)
        gy = orc.uniform_fill(43, n_rows * n_cols, ety.value)
        want_dot = orc.accu(gx * gy, ety)
        want_norm = float(np.sqrt(orc.accu((gx - gy) * (gx - gy), ety)))
        assert abs(part[0].item() - want_dot) <= 1e-12 * abs(want_dot)
        assert abs(combine_norm(part[1].item()) - want_norm) <= 1e-12 * want_norm


def _body_row_stats(rank, world, n_rows, n_cols):
    sh = column_shard(n_rows, n_cols, rank, world)
    g = orc.randu(n_rows, n_cols, 7, "f64")
    g[3, 5] = g[3, 9] = 2.0            # a tie across the shard boundary: first index wins
    g[7, 0] = np.nan                   # NaN wins index_max (numpy argmax semantics)
    g[11, 2] = -1.0
    g[11, 12] = -1.0                   # tie for index_min
    loc = g[:, sh.col0:sh.col1]
    ety = orc.ElemType.f64
    sums = torch.tensor(orc.reduce_dim(orc.ReduceKind.sum, 1, loc, ety).ravel())
    maxs = torch.tensor(loc.max(axis=1))
    mins = torch.tensor(loc.min(axis=1))
    allreduce_rowstats(sums, maxs, mins)
    want_sum = orc.reduce_dim(orc.ReduceKind.sum, 1, g, ety).ravel()
    assert orc.compare(sums.numpy(), want_sum) < 1e-13     # NaN-aware (oracle.py:104-123)
    assert np.array_equal(mins.numpy(), g.min(axis=1), equal_nan=True)
    assert np.array_equal(maxs.numpy(), g.max(axis=1), equal_nan=True)
    for maximize, kind in ((True, orc.ReduceKind.index_max), (False, orc.ReduceKind.index_min)):
        li = (np.argmax(loc, axis=1) if maximize else np.argmin(loc, axis=1))
        lv = loc[np.arange(n_rows), li]
        bv, bi = combine_arg_candidates(torch.tensor(lv), torch.tensor(li + sh.col0, dtype=torch.int64),
                                        maximize)
        want = orc.reduce_dim(kind, 1, g, ety).ravel()
        assert np.array_equal(bi.numpy(), want.astype(np.int64)), (maximize, bi.numpy(), want)


def _body_column_local(rank, world, n_rows, n_cols):
    """dim-0 stats are shard-local: the gathered per-shard results equal the
    whole-matrix result with no partial combine."""
    sh = column_shard(n_rows, n_cols, rank, world)
    ety = orc.ElemType.f64
    x = orc.uniform_fill(42, sh.n_rows * sh.local_cols, "f64", offset=sh.elem_offset).reshape(
        (n_rows, sh.local_cols), order="F")
    y = orc.uniform_fill(43, sh.n_rows * sh.local_cols, "f64", offset=sh.elem_offset).reshape(
        (n_rows, sh.local_cols), order="F")
    v = (x - y) * x
    loc_sum = torch.tensor(orc.reduce_dim(orc.ReduceKind.sum, 0, v, ety).ravel())
    loc_idx = torch.tensor(orc.reduce_dim(orc.ReduceKind.index_max, 0, v, ety).ravel().astype(np.int64))
    counts = [column_shard(n_rows, n_cols, r, world).local_cols for r in range(world)]
    sums = [torch.empty(c, dtype=torch.float64) for c in counts]
    idxs = [torch.empty(c, dtype=torch.int64) for c in counts]
    # gloo all_gather needs equal sizes: pad to the largest block
    m = max(counts)
    ps = torch.zeros(m, dtype=torch.float64)
    ps[:loc_sum.numel()] = loc_sum
    pi = torch.zeros(m, dtype=torch.int64)
    pi[:loc_idx.numel()] = loc_idx
    gs = [torch.empty(m, dtype=torch.float64) for _ in range(world)]
    gi = [torch.empty(m, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gs, ps)
    dist.all_gather(gi, pi)
    sums = np.concatenate([g[:c].numpy() for g, c in zip(gs, counts)])
    idxs = np.concatenate([g[:c].numpy() for g, c in zip(gi, counts)])
    gx, gy = orc.randu(n_rows, n_cols, 42, "f64"), orc.randu(n_rows, n_cols, 43, "f64")
    gv = (gx - gy) * gx
    assert orc.compare(sums, orc.reduce_dim(orc.ReduceKind.sum, 0, gv, ety).ravel()) < 1e-14
    assert np.array_equal(idxs, orc.reduce_dim(orc.ReduceKind.index_max, 0, gv, ety).ravel())


# ---- tests -------------------------------------------------------------------------------

def test_column_shard_partition():
    for n_cols in (1, 7, 8, 16384, 16385):
        for world in (1, 2, 3, 8):
            shards = [column_shard(65536, n_cols, r, world) for r in range(world)]
            assert shards[0].col0 == 0 and shards[-1].col1 == n_cols
            for a, b in zip(shards, shards[1:]):
                assert a.col1 == b.col0
            sizes = [s.local_cols for s in shards]
            assert max(sizes) - min(sizes) <= 1
            assert all(s.elem_offset == s.col0 * 65536 for s in shards)
    with pytest.raises(ShapeError):
        column_shard(4, 4, 2, 2)


def test_shard_stream_is_global_slice():
    """randu of a shard at its element offset == the slice of the global stream."""
    g = orc.randu(64, 10, 42, "f32")
    for r in range(3):
        sh = column_shard(64, 10, r, 3)
        loc = orc.uniform_fill(42, 64 * sh.local_cols, "f32", offset=sh.elem_offset).reshape(
            (64, sh.local_cols), order="F")
        assert np.array_equal(loc, g[:, sh.col0:sh.col1])


def test_gloo_full_reductions_world2():
    _run(2, _body_full_reductions, 1000, 37)


def test_gloo_row_stats_world2():
    _run(2, _body_row_stats, 16, 14)


def test_gloo_column_stats_local_world2():
    _run(2, _body_column_local, 128, 9)
