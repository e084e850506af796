"""The native collectives (csrc/comm.cu) and the sharded API on the GPU.

A one-GPU box allows two kinds of runs:
* world 1 with each transport (NCCL and peer): the collectives' plumbing,
  argument checks and combine kernels execute (identity combines);
* world 2 with both ranks on GPU 0 (separate processes, as torchrun would
  start them) over the PEER transport -- NCCL refuses two ranks on one
  device -- so the peer kernel's publish / wait / rank-order combine runs for
  real: CUDA-IPC blocks, system-scope flags, two data parities, epochs in
  device memory (also under CUDA-graph replay).
Results must equal the single-process oracle on the global matrices.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu


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


def _ctx(transport, rank=0, world=1):
    import paper_2604_22242_b200 as fm
    ctx = fm.Context(fm.B200Backend(device=0))
    comm = fm.Communicator(ctx, rank, world, transport=transport)
    return fm, ctx, comm


# ---- world 1 ------------------------------------------------------------------------------

@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_world1_collectives(transport):
    fm, ctx, comm = _ctx(transport)
    assert comm.transport == transport
    v = fm.from_array(np.array([1.5, np.nan, -2.0, 7.0]), "f64", ctx)
    comm.allreduce(v, "sum")
    assert np.array_equal(v.to_numpy().ravel(), [1.5, np.nan, -2.0, 7.0], equal_nan=True)
    comm.allreduce(v, "sum", divisor=2.0)
    assert np.array_equal(v.to_numpy().ravel(), [0.75, np.nan, -1.0, 3.5], equal_nan=True)
    u = fm.from_array(np.array([1, 2, 3], np.uint32), "u32", ctx)
    comm.allreduce(u, "max")
    assert list(u.to_numpy().ravel()) == [1, 2, 3]
    vals = fm.from_array(np.array([0.5, 0.25], np.float32), "f32", ctx)
    idx = fm.from_array(np.array([3, 4], np.uint32), "u32", ctx)
    comm.allreduce_arg(vals, idx, 100, True)
    assert list(idx.to_numpy().ravel()) == [103, 104]
    assert list(vals.to_numpy().ravel()) == [0.5, 0.25]
    src = fm.randu(1000, 3, 1, "f32", ctx)
    dst = fm.Mat(1000, 3, "f32", ctx)
    comm.allgather(src, dst)
    assert np.array_equal(dst.to_numpy(), src.to_numpy())
    assert comm.status() == 0
    comm.close()


def test_world1_sharded_api_is_the_plain_api():
    fm, ctx, comm = _ctx("none")
    X = fm.ShardedMat(300, 40, "f64", comm).randu(42)
    Y = fm.ShardedMat(300, 40, "f64", comm).randu(43)
    gx, gy = orc.randu(300, 40, 42, "f64"), orc.randu(300, 40, 43, "f64")
    want = orc.accu(gx * gy, orc.ElemType.f64)
    assert abs(fm.dot(X, Y) - want) <= 1e-12 * abs(want)
    out = fm.Mat(300, 1, "u32", ctx)
    fm.assign_all([(out, fm.index_max(X - Y, 1))])
    assert np.array_equal(out.to_numpy(), orc.reduce_dim(orc.ReduceKind.index_max, 1, gx - gy,
                                                         orc.ElemType.f64))


# ---- world 2 on one GPU over peer memory -----------------------------------------------------

def _body_peer_collectives(rank, world):
    fm, ctx, comm = _ctx("peer", rank, world)
    # sums in rank order: rank r contributes r + 1 + [0, 1, ...]
    n = 3000
    v = fm.from_array(np.arange(n, dtype=np.float64) + rank + 1, "f64", ctx)
    comm.allreduce(v, "sum")
    want = sum(np.arange(n, dtype=np.float64) + r + 1 for r in range(world))
    assert np.array_equal(v.to_numpy().ravel(), want)
    # NaN-propagating max / min, wrapping integer sums
    a = np.array([1.0, np.nan, 3.0, -1.0]) * (rank + 1)
    m = fm.from_array(a, "f64", ctx)
    comm.allreduce(m, "max")
    assert np.array_equal(m.to_numpy().ravel(), [2.0, np.nan, 6.0, -1.0], equal_nan=True)
    w = fm.from_array(np.array([0xFFFFFFFF, 5], np.uint32), "u32", ctx)
    comm.allreduce(w, "sum")
    assert list(w.to_numpy().ravel()) == [0xFFFFFFFE, 10]
    # arg-select: ties -> first global index, NaN wins
    vals = fm.from_array(np.array([5.0, 1.0, np.nan if rank == 1 else 0.0, 2.0]), "f64", ctx)
    idx = fm.from_array(np.array([1, 2, 3, 4], np.uint32), "u32", ctx)
    comm.allreduce_arg(vals, idx, 10 * rank, True)
    assert list(idx.to_numpy().ravel()) == [1, 2, 13, 4]
    # allgather larger than one data slot (8 MiB): chunked through both parities
    per = (3 << 20) + 5
    src = fm.Mat(per, 1, "f32", ctx)
    ctx.backend.randu(src.handle, 9, offset=rank * per)
    dst = fm.Mat(per * world, 1, "f32", ctx)
    comm.allgather(src, dst)
    assert np.array_equal(dst.to_numpy().ravel(), orc.uniform_fill(9, per * world, "f32"))
    # graph-captured allreduce replayed: the epoch lives on the device
    r = fm.Mat(8, 1, "f64", ctx)
    base = fm.from_array(np.full(8, rank + 1.0), "f64", ctx)

    def step():
        r.assign(base + 0.0)
        comm.allreduce(r, "sum")

    g = fm.capture(step, ctx)
    for _ in range(5):
        g.replay()
        assert np.array_equal(r.to_numpy().ravel(), np.full(8, float(sum(range(1, world + 1)))))
    g.close()
    assert comm.status() == 0
    ctx.sync()
    dist.barrier()
    comm.close()


def _body_peer_sharded_api(rank, world):
    fm, ctx, comm = _ctx("peer", rank, world)
    n_rows, n_cols = 1024, 77                 # ragged shards
    X, Y, Z = (fm.ShardedMat(n_rows, n_cols, "f64", comm).randu(s) for s in (42, 43, 44))
    g = [orc.randu(n_rows, n_cols, s, "f64") for s in (42, 43, 44)]
    e = (X - Y) % Z
    v = (g[0] - g[1]) * g[2]
    K = orc.ReduceKind
    outs = [fm.Mat(n_rows, 1, t, ctx) for t in ("f64", "f64", "f64", "u32", "u32")]
    fm.assign_all([(outs[0], fm.sum(e, 1)), (outs[1], fm.mean(e, 1)), (outs[2], fm.max(e, 1)),
                   (outs[3], fm.index_max(e, 1)), (outs[4], fm.index_min(e, 1))])
    # sums: the reduction order differs from numpy's pairwise sum, so the bound
    # is relative to the sum of magnitudes (rows can cancel to near zero)
    mag = np.abs(v).sum(axis=1, keepdims=True)
    for o, k in zip(outs, (K.sum, K.mean, K.max, K.index_max, K.index_min)):
        want = orc.reduce_dim(k, 1, v, orc.ElemType.f64)
        if k in (K.sum, K.mean):
            scale = mag if k is K.sum else mag / n_cols
            assert np.all(np.abs(o.to_numpy() - want) <= 1e-13 * scale), k
        else:
            assert np.array_equal(o.to_numpy(), want), k
    col = fm.ShardedMat(1, n_cols, "u32", comm)
    col.assign(fm.index_max(e, 0))
    assert np.array_equal(col.to_numpy(), orc.reduce_dim(K.index_max, 0, v, orc.ElemType.f64))
    want = orc.accu(g[0] * g[1], orc.ElemType.f64)
    assert abs(fm.dot(X, Y) - want) <= 1e-12 * abs(want)
    want = float(np.sqrt(orc.accu((g[0] - g[1]) ** 2, orc.ElemType.f64)))
    assert abs(fm.norm(X - Y) - want) <= 1e-12 * want
    # C3-style elementwise chain: local, bit-exact
    A = fm.ShardedMat(512, 64, "f32", comm).randu(1)
    B = fm.ShardedMat(512, 64, "f32", comm).randu(2)
    C = fm.ShardedMat(512, 64, "f32", comm)
    C.assign(fm.exp(-fm.square(A - B) / 2) + 0.5 * fm.abs(A))
    ga, gb = orc.randu(512, 64, 1), orc.randu(512, 64, 2)
    d = ga - gb
    half = np.float32(0.5)
    want = np.exp((half * -(d * d)).astype(np.float64)).astype(np.float32) + half * np.abs(ga)
    assert orc.max_ulp(C.to_numpy(), want) == 0
    # row-sharded GEMM: Y's column shards gathered, one tcgen05 launch per rank
    from paper_2604_22242_b200.dist import row_block
    m = n = k = 512
    r0, r1 = row_block(m, rank, world)
    gx = orc.randu(m, k, 42, "bf16")
    Xr = fm.from_array(np.ascontiguousarray(gx[r0:r1]), "bf16", ctx)
    Yb = fm.ShardedMat(n, k, "bf16", comm).randu(43)
    Zr = fm.matmul_row_shard(Xr, Yb, 2.0)
    gy = orc.randu(n, k, 43, "bf16")
    exact = 2.0 * (gx[r0:r1].astype(np.float64) @ gy.astype(np.float64).T)
    got = Zr.to_numpy().astype(np.float64)
    assert np.max(np.abs(got - exact) / np.abs(exact)) <= 1e-5
    assert comm.status() == 0
    ctx.sync()
    dist.barrier()
    comm.close()


@pytest.mark.timeout(300)
def test_peer_collectives_two_ranks_one_gpu():
    _run(2, _body_peer_collectives)


@pytest.mark.timeout(300)
def test_peer_sharded_api_two_ranks_one_gpu():
    _run(2, _body_peer_sharded_api)
