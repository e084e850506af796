"""The N>1 bench path end to end on a one-GPU box: `bench.py --gpus 2` spawns
two ranks itself (torch.distributed.run); FMB200_SHARE_GPU=1 puts both on
GPU 0, so the collectives run over libfmb200's peer-memory transport (NCCL
refuses two ranks on one device).  Timings are meaningless here; the
checks are the sharding (strong-scaled global shapes), the exchange and the
results against the global oracle."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import fm_oracle as orc

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _bench(*args):
    env = dict(os.environ, FMB200_SHARE_GPU="1")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--no-cpu", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    return json.loads(lines[0])


def test_two_rank_c2_bench_matches_global_oracle():
    n = 1_000_003                      # per rank, ragged
    d = _bench("--config", "c2", "--size", str(n))
    assert d["n_gpus"] == 2 and d["config"]["elements_per_gpu_per_step"] == 6 * n
    assert "peer" in d["config"]["parallelism"]
    assert d["comm_status"] == 0
    got = d["check"]["values"]
    for et in ("f32", "f64"):
        x = orc.uniform_fill(42, 2 * n, et)
        y = orc.uniform_fill(43, 2 * n, et)
        ety = orc.ElemType.f32 if et == "f32" else orc.ElemType.f64
        want_dot = orc.accu(x * y, ety)
        want_norm = float(np.sqrt(orc.accu((x - y) * (x - y), ety)))
        assert abs(got[f"dot_{et}"] - want_dot) <= 1e-12 * abs(want_dot)
        assert abs(got[f"accu_{et}"] - want_dot) <= 1e-12 * abs(want_dot)
        assert abs(got[f"norm_{et}"] - want_norm) <= 1e-12 * want_norm


def test_two_rank_strong_scaled_shards():
    """C3 / C4 / C5 split ONE global problem: half the columns (C3, C4) or
    rows (C5) per rank; parity checks of every rank's shard pass."""
    d = _bench("--config", "c3", "--size", "2048")
    assert d["config"]["elements_per_gpu_per_step"] == 2048 * 1024
    assert d["scaling"] == "strong" and d["check"]["max_ulp_256_cols_vs_correctly_rounded"] <= 1
    d = _bench("--config", "c4", "--size", "512")
    assert d["config"]["elements_per_gpu_per_step"] == 65536 * 256
    assert d["check"]["index_max_exact_64_cols"] and d["check"]["max_exact_64_cols"]
    d = _bench("--config", "c5", "--size", "1024")
    assert d["config"]["elements_per_gpu_per_step"] == 512 * 1024
    assert d["check"]["max_rel_err_all_entries_vs_exact_f64_kernel"] <= 1e-5
    assert "allgather_y" in d["per_kernel_ms"] and d["preplaced_value"] > 0
