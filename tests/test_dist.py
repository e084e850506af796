"""The column-sharded public API over gloo on CPU, world sizes 2 and 3.

SURVEY.md 8(e).  Every rank builds `ShardedMat`s of one global matrix (its
column block = its slice of the global splitmix64 stream) on a host
simulation of the device (tests/hostsim.py: oracle-evaluated launches) and
calls the same public functions a GPU user calls -- `fm.sum/mean/max/min/
index_max/index_min(e, dim)`, `fm.assign_all`, `fm.accu/dot/norm`,
`ShardedMat.assign`, `fm.matmul_row_shard` -- with the collectives of
csrc/comm.cu restated over gloo (tests/hostsim.SimComm).  Results must equal
the single-process oracle on the whole matrix: bit-exact for elementwise
chains, indices and extrema, within 1e-12 for sums.  The native collectives
themselves run on the GPU (tests/test_gpu_dist.py).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fm_oracle as orc
from paper_2604_22242_b200.dist import column_shard, row_block
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


def _setup(rank, world):
    import paper_2604_22242_b200 as fm
    from hostsim import SimBackend, SimComm
    ctx = fm.Context(SimBackend())
    return fm, ctx, SimComm(ctx, rank, world)


# ---- rank bodies (module-level so spawn can pickle them) -----------------------------

def _body_elementwise_and_full(rank, world, n_rows, n_cols):
    fm, ctx, comm = _setup(rank, world)
    for et in ("f32", "f64"):
        X = fm.ShardedMat(n_rows, n_cols, et, comm).randu(42)
        Y = fm.ShardedMat(n_rows, n_cols, et, comm).randu(43)
        Z = fm.ShardedMat(n_rows, n_cols, et, comm)
        gx, gy = orc.randu(n_rows, n_cols, 42, et), orc.randu(n_rows, n_cols, 43, et)
        assert np.array_equal(X.to_numpy(), gx)              # shard = slice of the global stream
        Z.assign(fm.exp(-fm.square(X - Y) / 2) + 0.5 * fm.abs(X))     # C3, no exchange
        dt = np.float32 if et == "f32" else np.float64
        half = dt(0.5)
        d = gx - gy
        want = np.exp((half * -(d * d)).astype(np.float64)).astype(dt) + half * np.abs(gx)
        assert orc.max_ulp(Z.to_numpy(), want) == 0
        ety = orc.ElemType.of(et)
        want_dot = orc.accu(gx * gy, ety)
        assert abs(fm.dot(X, Y) - want_dot) <= 1e-12 * abs(want_dot)
        assert abs(fm.accu(X % Y) - want_dot) <= 1e-12 * abs(want_dot)
        want_norm = float(np.sqrt(orc.accu(d * d, ety)))
        assert abs(fm.norm(X - Y) - want_norm) <= 1e-12 * want_norm
    calls = [c[0] for c in comm.calls]
    assert "allreduce" in calls


def _body_dim_reductions(rank, world, n_rows, n_cols):
    fm, ctx, comm = _setup(rank, world)
    ety = orc.ElemType.f64
    g = [orc.randu(n_rows, n_cols, s, "f64") for s in (42, 43, 44)]
    g[0][3, 5] = g[0][3, 9] = 9.0      # ties across shard boundaries: first index wins
    g[1][3, 5] = g[1][3, 9] = 0.0
    g[2][3, 5] = g[2][3, 9] = 1.0
    g[0][7, n_cols - 1] = np.nan       # NaN wins index_max / propagates through max
    X, Y, Z = (fm.ShardedMat(n_rows, n_cols, "f64", comm).set_global(a) for a in g)
    e = (X - Y) % Z
    v = (g[0] - g[1]) * g[2]
    K = orc.ReduceKind
    # dim 0: column-sharded results, no exchange
    outs0 = [fm.ShardedMat(1, n_cols, t, comm) for t in ("f64", "f64", "f64", "u32", "f64", "u32")]
    comm.calls.clear()
    fm.assign_all([(outs0[0], fm.sum(e, 0)), (outs0[1], fm.mean(e, 0)), (outs0[2], fm.max(e, 0)),
                   (outs0[3], fm.index_max(e, 0)), (outs0[4], fm.min(e, 0)), (outs0[5], fm.index_min(e, 0))])
    assert comm.calls == []
    for o, k in zip(outs0, (K.sum, K.mean, K.max, K.index_max, K.min, K.index_min)):
        want = orc.reduce_dim(k, 0, v, ety)
        got = o.to_numpy()
        if k in (K.sum, K.mean):
            assert orc.compare(got, want) < 1e-13
        else:
            assert np.array_equal(got, want, equal_nan=True), k
    # dim 1: replicated n_rows x 1 results through the collectives
    outs1 = [fm.Mat(n_rows, 1, t, ctx) for t in ("f64", "f64", "f64", "u32", "f64", "u32")]
    fm.assign_all([(outs1[0], fm.sum(e, 1)), (outs1[1], fm.mean(e, 1)), (outs1[2], fm.max(e, 1)),
                   (outs1[3], fm.index_max(e, 1)), (outs1[4], fm.min(e, 1)), (outs1[5], fm.index_min(e, 1))])
    for o, k in zip(outs1, (K.sum, K.mean, K.max, K.index_max, K.min, K.index_min)):
        want = orc.reduce_dim(k, 1, v, ety)
        got = o.to_numpy()
        if k in (K.sum, K.mean):
            assert orc.compare(got, want) < 1e-13
        else:
            assert np.array_equal(got, want, equal_nan=True), k
    sh = column_shard(n_rows, n_cols, rank, world)
    assert ("allreduce_arg", True, n_rows, sh.col0) in comm.calls
    assert ("allreduce", "sum", n_rows, float(n_cols)) in comm.calls     # mean: / global n_cols
    # a single lazy reduction through eval()
    s1 = fm.sum(e, 1).eval()
    assert orc.compare(s1.to_numpy(), orc.reduce_dim(K.sum, 1, v, ety)) < 1e-13


def _body_f32_row_sum(rank, world, n_rows, n_cols):
    """f32 children: partial row sums travel as f64 and round once."""
    fm, ctx, comm = _setup(rank, world)
    X = fm.ShardedMat(n_rows, n_cols, "f32", comm).randu(5)
    gx = orc.randu(n_rows, n_cols, 5, "f32")
    out = fm.Mat(n_rows, 1, "f32", ctx)
    fm.assign_all([(out, fm.mean(X * X, 1))])
    want = orc.reduce_dim(orc.ReduceKind.mean, 1, gx * gx, orc.ElemType.f32)
    assert np.array_equal(out.to_numpy(), want)


def _body_row_shard_gemm(rank, world, m, n, k):
    fm, ctx, comm = _setup(rank, world)
    r0, r1 = row_block(m, rank, world)
    gx = orc.randu(m, k, 42, "f32")
    X_rows = fm.from_array(np.ascontiguousarray(gx[r0:r1]), "f32", ctx)
    Y = fm.ShardedMat(n, k, "f32", comm).randu(43)
    gy = orc.randu(n, k, 43, "f32")
    Z = fm.matmul_row_shard(X_rows, Y, 2.0)
    want = (2.0 * (gx[r0:r1].astype(np.float64) @ gy.astype(np.float64).T)).astype(np.float32)
    assert np.array_equal(Z.to_numpy(), want)
    assert ("allgather", n * k // world) in comm.calls


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


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_elementwise_and_full_reductions(world):
    _run(world, _body_elementwise_and_full, 40, 17)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_dim_reductions(world):
    _run(world, _body_dim_reductions, 24, 14)


def test_sharded_f32_row_mean_world2():
    _run(2, _body_f32_row_sum, 32, 9)


def test_row_sharded_gemm_world2():
    _run(2, _body_row_shard_gemm, 16, 12, 8)


def test_sharded_api_rejects_locality_breaking_ops():
    import paper_2604_22242_b200 as fm
    from hostsim import SimBackend, SimComm
    ctx = fm.Context(SimBackend())
    comm = SimComm(ctx, 0, 1)
    X = fm.ShardedMat(4, 4, "f32", comm)
    M = fm.Mat(4, 4, "f32", ctx)
    with pytest.raises(ShapeError):
        X.t()
    with pytest.raises(ShapeError):
        X + M
    with pytest.raises(ShapeError):
        X + fm.ShardedMat(4, 5, "f32", comm)
