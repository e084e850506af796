"""The N>1 bench path end to end on a one-GPU box: torchrun with two ranks
sharing GPU 0 over gloo (FMB200_DIST_BACKEND=gloo, FMB200_SHARE_GPU=1).
Each rank reduces its slice of the global splitmix64 stream; the per-step
partials cross ranks in one all_reduce; the printed results must equal the
oracle over the concatenated global vectors."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_c2_bench_matches_global_oracle():
    n = 1_000_003                      # per rank, ragged
    env = dict(os.environ, FMB200_DIST_BACKEND="gloo", FMB200_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--config", "c2", "--size", str(n), "--steps", "3", "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["elements_per_gpu_per_step"] == 6 * n
    got = d["check"]
    for et in ("f32", "f64"):
        x = orc.uniform_fill(42, 2 * n, et)
        y = orc.uniform_fill(43, 2 * n, et)
        ety = orc.ElemType.f32 if et == "f32" else orc.ElemType.f64
        want_dot = orc.accu(x * y, ety)
        want_norm = float(np.sqrt(orc.accu((x - y) * (x - y), ety)))
        assert abs(got[f"dot_{et}"] - want_dot) <= 1e-12 * abs(want_dot)
        assert abs(got[f"accu_{et}"] - want_dot) <= 1e-12 * abs(want_dot)
        assert abs(got[f"norm_{et}"] - want_norm) <= 1e-12 * want_norm
