#!/usr/bin/env python
"""Benchmark of the B200 fused-expression hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config all|c1|c2|c3|c4|c4r|c5|c5f32|suite]
                    [--impl ours|reference]

Default (`--config all`): the headline line is BASELINE configs[1] = C2 --
one step is the six fused reductions accu(X % Y), dot(x, y), norm(x - y)
over 1e8-element f32 AND f64 vectors per GPU, one launch each -- and the
same line carries `configs`: C1, C3, C4, C5 (bf16) and C5 (f32) measured the
same way in the same run, each with its roofline, CPU baseline, end-to-end
number and parity check.

`value` is device-timed whole-job throughput (algorithmic bytes, the
reference's plan_bytes convention, bench.py:218-240, or GEMM flops) with
inputs resident in HBM: CUDA events on the launching stream around one CUDA
graph replay per step, barrier + sync on both sides, max over ranks.  `e2e`
is the same metric through the public API with the step's inputs uploaded
from pinned host memory and its results read back inside the timed region.

Multi-GPU: `--gpus N` starts N ranks itself (torch.distributed.run) unless
already launched by torchrun.  Plumbing (barriers, max-over-ranks, setup
exchange) runs over gloo; the data path's collectives are libfmb200's own
(`fm_allreduce` / `fm_allgather`: NCCL when every rank has its own GPU, the
peer-memory kernel when ranks share one -- FMB200_SHARE_GPU=1 puts every
rank on GPU 0).  Sharding:
  C1, C3, C4 -- the BASELINE global matrix, column-split across ranks
               (strong scaling, no exchange);
  C2         -- every rank owns a 1e8-element slice of a world x 1e8 global
               vector (weak scaling); the six partials cross ranks in ONE
               allreduce per step;
  C5         -- Z = 2 X Y^T at 8192^3: Z and X row-sharded, Y column-sharded
               (= split along K) and all-gathered every step, one tcgen05 GEMM
               of the local row block (strong scaling; the exchange is timed
               inside the step and also reported alone).

`--impl reference` times the reference's own CPU path on the host cores: the
C kernels its code generator emits (oracle/_ref, cjit.py flags) where the
reference can express the config, else the numpy restatement, all host
threads, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fused-expression effective HBM GB/s (% of 8 TB/s) and elements/s at 1/2/4/8 B200"
SPEC_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0
FALLBACK_BF16_TFLOPS = 1590.0
TIMING_NOTE = ("achieved = algorithmic work / mean launch duration of the dominant kernel (all its launches "
               "in the step) from CUDA events between the kernels (a second, instrumented pass of the timed "
               "steps; each event adds ~6 us); when every launch of the step is that kernel, the events at "
               "the timed steps' boundaries give the duration directly (no events between launches); "
               "achieved_in_timed_steps = the kernel's share of the instrumented step applied to the "
               "event-free timed step")


# --------------------------------------------------------------------------------------
# helpers

def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                    "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                    "source": "measured (MEASURED_PEAKS.json)"}
        except Exception:
            pass
    return {"hbm_gbs": FALLBACK_HBM_GBS, "bf16_tflops": FALLBACK_BF16_TFLOPS,
            "bf16_tflops_sustained": 1400.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(label: str):
    """dram read+write bytes per launch from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        v = json.loads(p.read_text()).get(label.split("[")[0])
        return v.get("dram_bytes") if isinstance(v, dict) else v
    return None


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during a timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


def merge_clocks(all_clocks: list[dict]) -> dict:
    """Worst case over ranks: lowest median clock, union of throttle reasons."""
    have = [c for c in all_clocks if c.get("sm_mhz") is not None]
    if not have:
        return all_clocks[0]
    worst = min(have, key=lambda c: c["sm_mhz"])
    out = dict(worst)
    out["reasons"] = sorted({r for c in all_clocks for r in c.get("reasons", [])})
    out["samples"] = sum(c.get("samples", 0) for c in all_clocks)
    return out


class Plumb:
    """Process plumbing (torchrun env; gloo for barriers, maxima and setup
    exchange).  The data path never goes through it."""

    def __init__(self, gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != gpus:
            raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={self.world}")
        self.shared = os.environ.get("FMB200_SHARE_GPU") == "1"
        self.device = 0 if self.shared else self.local
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def gather(self, obj) -> list:
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

    def max(self, v: float) -> float:
        return max(self.gather(v))

    def sum(self, v):
        return sum(self.gather(v))

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Events:
    """CUDA events on the backend's stream (the stream the kernels run on)."""

    def __init__(self, nat, stream, n):
        self.nat, self.stream, self.ev = nat, stream, []
        for _ in range(n):
            e = ctypes.c_void_p()
            nat.call("fm_event_create", ctypes.byref(e))
            self.ev.append(e.value)

    def record(self, i):
        self.nat.call("fm_event_record", self.ev[i], self.stream)

    def ms(self, i, j) -> float:
        f = ctypes.c_float()
        self.nat.call("fm_event_elapsed_ms", self.ev[i], self.ev[j], ctypes.byref(f))
        return f.value

    def close(self):
        for e in self.ev:
            self.nat.call("fm_event_destroy", e)
        self.ev = []


class Run:
    """One rank's context: backend, communicator, plumbing."""

    def __init__(self, args, plumb: Plumb):
        import paper_2604_22242_b200 as fm
        from paper_2604_22242_b200._native import native
        self.fm, self.args, self.p = fm, args, plumb
        self.nat = native()
        self.backend = fm.B200Backend(device=plumb.device)
        self.ctx = fm.Context(self.backend)
        self.comm = fm.Communicator(self.ctx, plumb.rank, plumb.world,
                                    exchange=plumb.gather if plumb.world > 1 else None)
        self.rank, self.world = plumb.rank, plumb.world

    def size(self, name: str) -> int:
        """--size applies to the selected config (to C2 alone in the default run)."""
        return self.args.n if self.args.config in (name, "all" if name == "c2" else None) else 0

    def sync(self):
        self.ctx.sync()


# --------------------------------------------------------------------------------------
# configs

class Config:
    name = ""
    metric = METRIC
    unit = "GB/s"
    bound = "hbm"
    dtype = "f32"
    scaling = "strong"
    flush = False
    workload = ""

    def __init__(self, run: Run):
        self.run, self.fm, self.ctx = run, run.fm, run.ctx

    # (label, callable, work per launch) -- each callable enqueues ONE kernel or collective
    def launches(self) -> list:
        raise NotImplementedError

    def elements_per_step(self) -> int:
        raise NotImplementedError

    def check(self) -> dict:
        return {}

    def setup_e2e(self):
        return None

    def step_e2e(self):
        raise NotImplementedError

    def cpu(self, threads: int):
        raise NotImplementedError

    def extra(self, m: dict) -> dict:
        return {}


def _ref_kernels():
    from oracle.ref_runner import RefKernels, available
    if not available():
        raise FileNotFoundError("oracle/_ref not built")
    return RefKernels()


class C2(Config):
    name = "c2"
    scaling = "weak"
    dtype = "f32+f64 (f64 accumulation)"

    def __init__(self, run):
        super().__init__(run)
        self.n = run.size("c2") or 100_000_000
        w = run.world
        self.workload = (f"C2 fused reductions accu(X%Y), dot(x,y), norm(x-y) on {self.n:.0e}-element f32 and "
                         f"f64 vectors per GPU" + (f" (slices of {w} x {self.n:.0e}-element global vectors)" if w > 1 else ""))
        fm, ctx = self.fm, self.ctx
        # a world x n global vector as an n x world matrix: one column (= one
        # contiguous slice of the splitmix64 stream) per rank
        S = lambda et, seed: fm.ShardedMat(self.n, w, et, run.comm).randu(seed)  # noqa: E731
        self.x32, self.y32, self.x64, self.y64 = S("f32", 42), S("f32", 43), S("f64", 42), S("f64", 43)
        self.R = fm.Mat(6, 1, "f64", ctx)
        run.sync()

    def launches(self):
        fm, R, n = self.fm, self.R, self.n
        a32, b32, a64, b64 = self.x32.local, self.y32.local, self.x64.local, self.y64.local
        out = [("accu_schur_f32", lambda: fm.accu_async(a32 % b32, R, 0), 8 * n + 8),
               ("dot_f32", lambda: fm.dot_async(a32, b32, R, 1), 8 * n + 8),
               ("norm_sqdiff_f32", lambda: fm.norm_async(a32 - b32, R, 2, squared=True), 8 * n + 8),
               ("accu_schur_f64", lambda: fm.accu_async(a64 % b64, R, 3), 16 * n + 8),
               ("dot_f64", lambda: fm.dot_async(a64, b64, R, 4), 16 * n + 8),
               ("norm_sqdiff_f64", lambda: fm.norm_async(a64 - b64, R, 5, squared=True), 16 * n + 8)]
        if self.run.world > 1:
            out.append(("allreduce_partials", lambda: self.run.comm.allreduce(R, "sum"), 0))
        return out

    def elements_per_step(self):
        return 6 * self.n

    def results(self) -> list:
        r = self.R.to_numpy().ravel()
        return [r[0], r[1], float(np.sqrt(r[2])), r[3], r[4], float(np.sqrt(r[5]))]

    def check(self):
        """vs numpy f64 sums of the device data: per-rank partials, summed over ranks."""
        got = self.results()
        parts = []
        for x, y in ((self.x32, self.y32), (self.x64, self.y64)):
            xv, yv = x.local.to_numpy().ravel(), y.local.to_numpy().ravel()
            d = xv - yv                  # every node rounds to the element type (f32 too)
            parts += [float(np.sum((xv * yv).astype(np.float64))), float(np.sum((d * d).astype(np.float64)))]
        tot = [self.run.p.sum(v) for v in parts]
        want = [tot[0], tot[0], np.sqrt(tot[1]), tot[2], tot[2], np.sqrt(tot[3])]
        return {"max_rel_err_vs_numpy_f64": float(max(abs(g - w) / abs(w) for g, w in zip(got, want))),
                "tolerance": 1e-12, "values": dict(zip(["accu_f32", "dot_f32", "norm_f32", "accu_f64",
                                                        "dot_f64", "norm_f64"], got))}

    def setup_e2e(self):
        fm = self.fm
        self.h = []
        for m in (self.x32, self.y32, self.x64, self.y64):
            hb = fm.pinned(self.n, 1, m.etype.value)
            m.local.download_pinned(hb)
            self.h.append(hb)
        self.run.sync()
        return sum(h.nbytes for h in self.h), 6 * 8

    def step_e2e(self):
        fm = self.fm
        for m, hb in zip((self.x32, self.y32, self.x64, self.y64), self.h):
            m.local.upload_pinned(hb)
        return [fm.accu(self.x32 % self.y32), fm.dot(self.x32, self.y32), fm.norm(self.x32 - self.y32),
                fm.accu(self.x64 % self.y64), fm.dot(self.x64, self.y64), fm.norm(self.x64 - self.y64)]

    e2e_path = "public API: ShardedMat upload_pinned + fm.accu / fm.dot / fm.norm (host floats back)"

    def cpu(self, threads, n_sample=20_000_000):
        from oracle import fm_oracle as orc
        data = [orc.uniform_fill(42, n_sample, "f32"), orc.uniform_fill(43, n_sample, "f32"),
                orc.uniform_fill(42, n_sample, "f64"), orc.uniform_fill(43, n_sample, "f64")]
        work = 3 * (8 * n_sample + 8) + 3 * (16 * n_sample + 8)
        try:
            rk = _ref_kernels()

            def run():
                a = rk.accu("accu_schur_f32", data[0:2], threads)
                b = rk.accu("accu_schur_f32", data[0:2], threads)          # dot == accu(x % y)
                c = np.sqrt(rk.accu("accu_sqdiff_f32", data[0:2], threads))
                d = rk.accu("accu_schur_f64", data[2:4], threads)
                e = rk.accu("accu_schur_f64", data[2:4], threads)
                f = np.sqrt(rk.accu("accu_sqdiff_f64", data[2:4], threads))
                return [a, b, c, d, e, f]
            return run, work, "reference", threads, (
                f"the reference's generated-C reduce kernels (oracle/_ref, cc -O2 -fwrapv) over "
                f"{n_sample:.0e}-element f32+f64 vectors, {threads} host threads on slabs")
        except (ImportError, OSError):
            def run():
                out = []
                for x, y in ((data[0], data[1]), (data[2], data[3])):
                    p = float(np.dot(x.astype(np.float64), y.astype(np.float64)))
                    d = (x - y).astype(np.float64)
                    out += [p, p, float(np.sqrt(np.dot(d, d)))]
                return out
            return run, work, "port", 1, f"numpy restatement over {n_sample:.0e}-element vectors, 1 thread"


class C1(Config):
    """Z = 2*(X % Y) + X over ROT independent (X, Y, Z) sets per step: the
    64 MiB output of one launch is still dirty in L2 when it ends; the next
    launch's traffic writes it back inside the timed window (write-back of
    the last set of a step lands in the L2 flush before the next step)."""
    name = "c1"
    flush = True
    ROT = 6

    def __init__(self, run):
        super().__init__(run)
        self.n = run.size("c1") or 4096
        fm, comm = self.fm, run.comm
        self.sets = []
        for i in range(self.ROT):
            X = fm.ShardedMat(self.n, self.n, "f32", comm).randu(42 + 2 * i)
            Y = fm.ShardedMat(self.n, self.n, "f32", comm).randu(43 + 2 * i)
            Z = fm.ShardedMat(self.n, self.n, "f32", comm)
            self.sets.append((X, Y, Z, 2 * (X % Y) + X))
        self.local_elems = self.n * self.sets[0][0].shard.local_cols
        self.workload = (f"C1 Z = 2*(X % Y) + X, f32 {self.n}x{self.n}"
                         + (f" column-sharded over {run.world} GPUs" if run.world > 1 else "")
                         + f"; {self.ROT} independent input/output sets per step (L2 write-back inside the window)")
        run.sync()

    def launches(self):
        return [(f"c1_copy_f32[{i}]", lambda Z=Z, e=e: Z.assign(e), 12 * self.local_elems)
                for i, (X, Y, Z, e) in enumerate(self.sets)]

    def elements_per_step(self):
        return self.ROT * self.local_elems

    def check(self):
        from oracle import fm_oracle as orc
        X, Y, Z, _ = self.sets[0]
        x, y = X.local.to_numpy(), Y.local.to_numpy()
        return {"max_ulp_whole_shard_vs_oracle": orc.max_ulp(Z.local.to_numpy(), np.float32(2) * (x * y) + x),
                "tolerance_ulp": 0}

    def setup_e2e(self):
        fm = self.fm
        X, Y, Z, _ = self.sets[0]
        self.hx = fm.pinned(self.n, X.shard.local_cols, "f32")
        self.hy = fm.pinned(self.n, X.shard.local_cols, "f32")
        self.hz = fm.pinned(self.n, X.shard.local_cols, "f32")
        X.local.download_pinned(self.hx)
        Y.local.download_pinned(self.hy)
        self.run.sync()
        return self.hx.nbytes + self.hy.nbytes, self.hz.nbytes

    e2e_work_fraction = 1  # one set per e2e step

    def step_e2e(self):
        X, Y, Z, e = self.sets[0]
        X.local.upload_pinned(self.hx)
        Y.local.upload_pinned(self.hy)
        Z.assign(e)
        Z.local.download_pinned(self.hz)
        self.run.sync()

    e2e_path = "public API: upload_pinned + ShardedMat.assign + download_pinned"

    def e2e_work(self):
        return 12 * self.local_elems

    def cpu(self, threads):
        from oracle import fm_oracle as orc
        n = self.n
        x = np.asfortranarray(orc.randu(n, n, 42))
        y = np.asfortranarray(orc.randu(n, n, 43))
        z = np.zeros((n, n), np.float32, order="F")
        try:
            rk = _ref_kernels()
            return (lambda: rk.copy("c1_f32", z, [x, y], [np.float32(2)], threads)), 12 * n * n, "reference", \
                threads, f"the reference's generated-C copy kernel (oracle/_ref) on the full {n}x{n}, {threads} threads on column slabs"
        except (ImportError, OSError):
            return (lambda: np.add(np.float32(2) * (x * y), x, out=z)), 12 * n * n, "port", 1, \
                f"numpy restatement on {n}x{n}, 1 thread"


class C3(Config):
    name = "c3"

    def __init__(self, run):
        super().__init__(run)
        self.n = run.size("c3") or 32768
        fm, comm = self.fm, run.comm
        self.X = fm.ShardedMat(self.n, self.n, "f32", comm).randu(42)
        self.Y = fm.ShardedMat(self.n, self.n, "f32", comm).randu(43)
        self.Z = fm.ShardedMat(self.n, self.n, "f32", comm)
        self.e = fm.exp(-fm.square(self.X - self.Y) / 2) + 0.5 * fm.abs(self.X)
        self.local_elems = self.n * self.X.shard.local_cols
        self.workload = (f"C3 Z = exp(-square(X - Y)/2) + 0.5*abs(X), f32 {self.n}x{self.n}"
                         + (f" column-sharded over {run.world} GPUs ({self.X.shard.local_cols} columns each)"
                            if run.world > 1 else ""))
        run.sync()

    def launches(self):
        return [("c3_copy_f32", lambda: self.Z.assign(self.e), 12 * self.local_elems)]

    def elements_per_step(self):
        return self.local_elems

    def check(self):
        """256 columns spread over the shard vs the correctly rounded restatement."""
        from oracle import fm_oracle as orc
        cols = np.unique(np.linspace(0, self.X.shard.local_cols - 1, 256).astype(int))
        X, Y, Z = self.X.local, self.Y.local, self.Z.local
        xs, ys, zs = X.to_numpy()[:, cols], Y.to_numpy()[:, cols], Z.to_numpy()[:, cols]
        d = xs - ys
        h = np.float32(0.5)
        want = np.exp((h * -(d * d)).astype(np.float64)).astype(np.float32) + h * np.abs(xs)
        return {"max_ulp_256_cols_vs_correctly_rounded": orc.max_ulp(zs, want), "tolerance_ulp": 1}

    def setup_e2e(self):
        fm = self.fm
        c = self.X.shard.local_cols
        self.hx, self.hy, self.hz = (fm.pinned(self.n, c, "f32") for _ in range(3))
        self.X.local.download_pinned(self.hx)
        self.Y.local.download_pinned(self.hy)
        self.run.sync()
        return self.hx.nbytes + self.hy.nbytes, self.hz.nbytes

    def step_e2e(self):
        self.X.local.upload_pinned(self.hx)
        self.Y.local.upload_pinned(self.hy)
        self.Z.assign(self.e)
        self.Z.local.download_pinned(self.hz)
        self.run.sync()

    e2e_path = "public API: upload_pinned + ShardedMat.assign + download_pinned"

    def cpu(self, threads, n=8192):
        from oracle import fm_oracle as orc
        x = np.asfortranarray(orc.randu(n, n, 42))
        y = np.asfortranarray(orc.randu(n, n, 43))
        z = np.zeros((n, n), np.float32, order="F")
        try:
            rk = _ref_kernels()
            # randu inputs are >= 0, so abs(X) == X: the reference's own
            # expression exp(-(X-Y)**2 / 2) + 0.5*X gives the same values
            return (lambda: rk.copy("c3noabs_f32", z, [x, y], [np.float32(0.5), np.float32(0.5)], threads)), \
                12 * n * n, "reference", threads, (
                    f"the reference's generated-C copy kernel for exp(-(X-Y)**2/2) + 0.5*X (abs(X) == X on randu "
                    f"inputs; the reference has no abs) on {n}x{n}, {threads} threads on column slabs")
        except (ImportError, OSError):
            def run():
                d = x - y
                return np.exp((np.float32(0.5) * -(d * d)).astype(np.float64)).astype(np.float32) + \
                    np.float32(0.5) * np.abs(x)
            return run, 12 * n * n, "port", 1, f"numpy restatement on {n}x{n}, 1 thread"


class C4(Config):
    name = "c4"
    dtype = "f64"
    ROWS = 65536

    def __init__(self, run):
        super().__init__(run)
        self.cols = run.size(self.name) or 16384
        fm, comm = self.fm, run.comm
        r, c = self.ROWS, self.cols
        self.X, self.Y, self.Z = (fm.ShardedMat(r, c, "f64", comm).randu(s) for s in (42, 43, 44))
        self.e = (self.X - self.Y) % self.Z
        self.outs = [fm.ShardedMat(1, c, t, comm) for t in ("f64", "f64", "f64", "u32")]
        lc = self.X.shard.local_cols
        self.local_cols = lc
        self.kbytes = 3 * 8 * r * lc + 3 * 8 * lc + 4 * lc
        self.workload = (f"C4 column-wise sum/mean/max/index_max of (X - Y) % Z, f64 {r}x{c}"
                         + (f" column-sharded over {run.world} GPUs ({lc} columns each, no exchange)"
                            if run.world > 1 else "") + ", one fused multi-output pass")
        run.sync()

    def _step(self):
        fm, e, o = self.fm, self.e, self.outs
        fm.assign_all([(o[0], fm.sum(e, 0)), (o[1], fm.mean(e, 0)), (o[2], fm.max(e, 0)),
                       (o[3], fm.index_max(e, 0))])

    def launches(self):
        return [("c4_colstats_f64", self._step, self.kbytes)]

    def elements_per_step(self):
        return self.ROWS * self.local_cols

    def check(self):
        from oracle import fm_oracle as orc
        cols = np.unique(np.linspace(0, self.local_cols - 1, 64).astype(int))
        v = ((self.X.local.to_numpy()[:, cols] - self.Y.local.to_numpy()[:, cols])
             * self.Z.local.to_numpy()[:, cols])
        k = orc.ReduceKind
        f64 = orc.ElemType.f64
        got = [o.local.to_numpy()[:, cols] for o in self.outs]
        mag = np.abs(v).sum(axis=0, keepdims=True)
        return {"index_max_exact_64_cols": bool(np.array_equal(got[3], orc.reduce_dim(k.index_max, 0, v, f64))),
                "max_exact_64_cols": bool(np.array_equal(got[2], orc.reduce_dim(k.max, 0, v, f64))),
                "sum_err_over_sum_abs_64_cols": float(np.max(np.abs(got[0] - orc.reduce_dim(k.sum, 0, v, f64)) / mag)),
                "tolerance_sum": 1e-12}

    def setup_e2e(self):
        fm = self.fm
        self.h = [fm.pinned(self.ROWS, self.local_cols, "f64") for _ in range(3)]
        for m, hb in zip((self.X, self.Y, self.Z), self.h):
            m.local.download_pinned(hb)
        self.ho = [fm.pinned(1, self.local_cols, o.etype.value) for o in self.outs]
        self.run.sync()
        return sum(h.nbytes for h in self.h), sum(h.nbytes for h in self.ho)

    def step_e2e(self):
        for m, hb in zip((self.X, self.Y, self.Z), self.h):
            m.local.upload_pinned(hb)
        self._step()
        for o, hb in zip(self.outs, self.ho):
            o.local.download_pinned(hb)
        self.run.sync()

    e2e_path = "public API: upload_pinned + fm.assign_all(sum/mean/max/index_max) + download_pinned"

    def cpu(self, threads, cols=256):
        from oracle import fm_oracle as orc
        r = self.ROWS
        X, Y, Z = (np.asfortranarray(orc.randu(r, cols, s, "f64")) for s in (42, 43, 44))
        v = np.zeros((r, cols), np.float64, order="F")
        from concurrent.futures import ThreadPoolExecutor
        threads = max(1, min(threads, cols))
        bounds = np.linspace(0, cols, threads + 1).astype(int)

        def stats(t):
            b = v[:, bounds[t]:bounds[t + 1]]
            s = b.sum(axis=0)
            return s, s / r, b.max(axis=0), b.argmax(axis=0).astype(np.uint32)

        try:
            rk = _ref_kernels()

            def run():
                rk.copy("c4sub_f64", v, [X, Y, Z], [], threads)
                with ThreadPoolExecutor(threads) as ex:
                    return list(ex.map(stats, range(threads)))
            return run, 3 * 8 * r * cols + 28 * cols, "reference", threads, (
                f"the reference's generated-C copy kernel for (X-Y)%Z (oracle/_ref) + numpy column "
                f"sum/mean/max/argmax (the reference has no dim reductions) on {r}x{cols}, {threads} threads")
        except (ImportError, OSError):
            def run():
                np.multiply(X - Y, Z, out=v)
                return stats(0) if threads == 1 else None
            return run, 3 * 8 * r * cols + 28 * cols, "port", 1, f"numpy restatement on {r}x{cols}, 1 thread"


class C4Rows(C4):
    """C4's expression reduced along rows (dim 1): at N>1 the partials cross
    ranks (allreduce SUM / MAX, arg-select for index_max).  Not a BASELINE
    config: the row variant of the same API."""
    name = "c4r"

    def __init__(self, run):
        super().__init__(run)
        fm, ctx, r = self.fm, self.ctx, self.ROWS
        self.outs = [fm.Mat(r, 1, "f64", ctx), fm.Mat(r, 1, "f64", ctx), fm.Mat(r, 1, "f64", ctx),
                     fm.Mat(r, 1, "u32", ctx)]
        self.kbytes = 3 * 8 * r * self.local_cols + 28 * r
        self.workload = self.workload.replace("C4 column-wise", "C4-rows row-wise")

    def _step(self):
        fm, e, o = self.fm, self.e, self.outs
        fm.assign_all([(o[0], fm.sum(e, 1)), (o[1], fm.mean(e, 1)), (o[2], fm.max(e, 1)),
                       (o[3], fm.index_max(e, 1))])

    def launches(self):
        return [("c4_rowstats_f64", self._step, self.kbytes)]

    def check(self):
        from oracle import fm_oracle as orc
        rows = slice(0, 64)
        g = [m.to_numpy()[rows, :] for m in (self.X, self.Y, self.Z)]
        v = (g[0] - g[1]) * g[2]
        k = orc.ReduceKind
        return {"index_max_exact_64_rows": bool(np.array_equal(
                    self.outs[3].to_numpy()[rows, :], orc.reduce_dim(k.index_max, 1, v, orc.ElemType.f64)))}

    def setup_e2e(self):
        return None


class C5(Config):
    """Z = 2 * X @ Y.t() at 8192^3, bf16 operands, f32 result: one tcgen05
    launch per rank (scale + transpose folded into the kernel)."""
    name = "c5"
    unit = "TFLOP/s"
    bound = "tensor"
    etype = "bf16"
    dtype = "bf16 (f32 accumulate, f32 out)"
    metric = "fused 2*X*Y.t() GEMM tensor-core TFLOP/s (BASELINE.json configs[4])"

    def __init__(self, run):
        super().__init__(run)
        fm, ctx, comm = self.fm, self.ctx, run.comm
        n = self.n = run.size(self.name) or 8192
        from paper_2604_22242_b200.dist import row_block
        self.r0, self.r1 = row_block(n, run.rank, run.world)
        rows = self.r1 - self.r0
        full = fm.randu(n, n, 42, self.etype, ctx)              # the global X, this rank keeps its rows
        self.X = fm.Mat(rows, n, self.etype, ctx)
        self.X.assign(full.submat(self.r0, 0, rows, n))
        del full
        self.Y = fm.ShardedMat(n, n, self.etype, comm).randu(43)
        self.Yfull = fm.Mat(n, n, self.etype, ctx) if run.world > 1 else self.Y.local
        self.Z = fm.Mat(rows, n, "f32", ctx)
        self.e = 2 * self.X @ self.Yfull.t()
        self.flops = 2 * rows * n * n
        self.workload = (f"C5 Z = 2*X*Y.t() {self.etype} GEMM {n}x{n}x{n} (scalar + transpose folded into the tcgen05 kernel)"
                         + (f"; Z and X row-sharded ({rows} rows per GPU), Y column-sharded (split along K) and "
                            f"all-gathered every step" if run.world > 1 else ""))
        run.sync()

    def launches(self):
        out = []
        if self.run.world > 1:
            out.append(("allgather_y", lambda: self.run.comm.allgather(self.Y.local, self.Yfull), 0))
        out += self.gemm_launches()
        return out

    def gemm_launches(self):
        return [(f"c5_gemm_{self.etype}", lambda: self.Z.assign(self.e), self.flops)]

    def elements_per_step(self):
        return (self.r1 - self.r0) * self.n

    def check(self):
        """Every entry of this rank's Z vs the f64-accumulating exact kernel
        (FM_GEMM_EXACT: the reference's numerics, cjit.py:33-51), on the device:
        max |Z - Zx| / |Zx| over all (M/p) x N entries."""
        fm, ctx, b = self.fm, self.ctx, self.run.backend
        rows = self.r1 - self.r0
        Zx = fm.Mat(rows, self.n, "f32", ctx)
        b.gemm(Zx.handle, self.X.handle, self.Yfull.handle, rows, self.n, self.n, trans_b=True, alpha=2.0,
               precision=2)
        rel = fm.max(fm.abs(self.Z - Zx) / fm.abs(Zx), 0).eval()
        return {"max_rel_err_all_entries_vs_exact_f64_kernel": float(rel.to_numpy().max()),
                "tolerance_rel": 1e-5}

    def setup_e2e(self):
        fm = self.fm
        self.hx = fm.pinned(self.X.n_rows, self.n, self.etype)
        self.hy = fm.pinned(self.n, self.Y.shard.local_cols, self.etype)
        self.hz = fm.pinned(self.Z.n_rows, self.n, "f32")
        self.X.download_pinned(self.hx)
        self.Y.local.download_pinned(self.hy)
        self.run.sync()
        return self.hx.nbytes + self.hy.nbytes, self.hz.nbytes

    def step_e2e(self):
        self.X.upload_pinned(self.hx)
        self.Y.local.upload_pinned(self.hy)
        if self.run.world > 1:
            self.fm.matmul_row_shard(self.X, self.Y, 2.0, self.Z, self.Yfull)
        else:
            self.Z.assign(self.e)
        self.Z.download_pinned(self.hz)
        self.run.sync()

    e2e_path = "public API: upload_pinned + fm.matmul_row_shard / Mat.assign(2*X@Y.t()) + download_pinned"

    def sustained(self, seconds: float = 2.5) -> dict:
        """Back-to-back GEMMs for >= `seconds` (graph of 50 launches replayed),
        clocks sampled under load: the sustained rate next to the burst figure."""
        fm, run = self.fm, self.run
        g = fm.capture(lambda: [f() for _ in range(50) for _, f, _ in self.gemm_launches()], self.ctx)
        g.replay()
        run.sync()
        ev = Events(run.nat, run.backend.stream, 2)
        sampler = ClockSampler(run.p.device).start()
        time.sleep(0.2)
        reps, t0 = 0, time.perf_counter()
        ev.record(0)
        while True:
            for _ in range(10):
                g.replay()
            reps += 10
            run.sync()
            if time.perf_counter() - t0 >= seconds:
                break
        ev.record(1)
        ms = ev.ms(0, 1)
        clocks = sampler.stop()
        g.close()
        ev.close()
        work = sum(w for _, _, w in self.gemm_launches()) * 50 * reps
        return {"value": round(work / (ms * 1e-3) / 1e12, 1), "unit": "TFLOP/s", "seconds": round(ms / 1e3, 2),
                "launches": 50 * reps, "clocks": clocks,
                "frac_of_sustained_peak": round(work / (ms * 1e-3) / 1e12 / measured_peaks()["bf16_tflops_sustained"], 4)}

    def extra(self, m):
        out = {"sustained": self.sustained()}
        if self.run.world > 1:
            # the pre-placed variant ("replicas + local shard"): Y already replicated, GEMM only
            gemm_ms = [v for k, v in m["per_kernel_ms"].items() if k.startswith("c5_gemm")]
            ag = m["per_kernel_ms"].get("allgather_y")
            t = self.run.p.max(sum(gemm_ms))
            out["preplaced_value"] = round(self.run.p.sum(self.flops) / (t * 1e-3) / 1e12, 1)
            out["allgather_ms"] = round(self.run.p.max(ag), 4) if ag is not None else None
        return out

    def cpu(self, threads, n=2048):
        from oracle import fm_oracle as orc
        x = orc.randu(n, n, 42, self.etype).astype(np.float64)
        y = orc.randu(n, n, 43, self.etype).astype(np.float64)
        return (lambda: (2.0 * (x @ y.T)).astype(np.float32)), 2 * n ** 3, "port", threads, (
            f"the reference's matmul numerics (backend.py:338-346: operands upcast to f64, numpy/OpenBLAS GEMM, "
            f"round to f32) on {n}x{n}x{n}, all {threads} host threads")


class C5F32(C5):
    """f32 operands: each scaled by a power of two from its max |x| and split
    into two fp16 planes (hi + lo, 22 significant bits), the three
    significant plane products accumulated by the same tcgen05 kernel (two
    max-abs + two split launches + the GEMM).  TFLOP/s counts the f32
    product's 2*N^3."""
    name = "c5f32"
    etype = "f32"
    dtype = "f32 operands (2 scaled fp16 planes each, 3 products, f32 accumulate, f32 out)"
    metric = "fused 2*X*Y.t() GEMM TFLOP/s (BASELINE.json configs[4], f32 operands)"


class Suite(Config):
    """The paper's 13-expression suite (reference bench.py:91-201) + add-N
    (bench.py:307-326, N up to 64: past one fused program the planner splits),
    f32 n x n.  Replicas at N>1 (no exchange on this path)."""
    name = "suite"
    flush = True
    scaling = "weak"

    def __init__(self, run):
        super().__init__(run)
        import math
        from paper_2604_22242_b200.plan import plan
        fm, ctx = self.fm, self.ctx
        n = self.n = run.size("suite") or 10000
        self.workload = f"paper suite (13 expressions incl. the 3-GEMM chain) + addN sweep (N = 2..64), f32 {n}x{n}"
        R = lambda k: fm.randu(n, n, 42 + k, "f32", ctx)  # noqa: E731
        a, b, c, dd = R(0), R(1), R(2), R(3)
        self.a, self.b = a, b
        u = fm.randi(n, n, 10, 43, "u32", ctx)
        half = n // 2
        # chain (reference bench.py:109-117): 4 matrices of decreasing sizes,
        # n x n/2, n/2 x n/4, n/4 x n/8, n/8 x n/16, multiplied left to right
        d = [max(n // (2 ** i), 1) for i in range(5)]
        ch = [fm.randu(d[i], d[i + 1], 42 + 70 + i, "f32", ctx) for i in range(4)]
        exprs = {
            "add2": (a + b, (n, n)),
            "add4": (a + b + c + dd, (n, n)),
            "chain": (ch[0] @ ch[1] @ ch[2] @ ch[3], (d[0], d[4])),
            "addsub2": (a.center_half() + b.center_half(), (half, half)),
            "addsub4": (a.center_half() + b.center_half() + c.center_half() + dd.center_half(), (half, half)),
            "expr1": (2 * (a.t() + b) + 2 * (a + b.t()), (n, n)),
            "expr2": (2.0 * a + (b + c).t() + fm.log(dd ** 2), (n, n)),
            "expr3": (1 / (a * fm.conv_to(u, "f32") + fm.log(fm.log(a + 2) * c)), (n, n)),
            "diagsum": ((a.diag(-1) + a.diag(1)) * (b.diag(-1) + b.diag(1)), (n - 1, 1)),
            "relu": (a * (a > 0), (n, n)),
            "sigmoid": (1 / (1 + fm.exp(-a)), (n, n)),
            "swish": (a / (1 + fm.exp(-1.0 * a)), (n, n)),
            "gelu": ((a / 2) * (1 + fm.tanh(math.sqrt(2.0 / 3.14159265358979) * (a + 0.044715 * (a ** 3)))), (n, n)),
        }
        pool = [a, b] + [R(k) for k in range(4, 4 + 62)]
        for k in (2, 4, 8, 16, 32, 48, 64):
            e = pool[0] + pool[1]
            for m in pool[2:k]:
                e = e + m
            exprs[f"add{k}N"] = (e, (n, n))
        self.labels = list(exprs)
        self.outs = {k: fm.Mat(*shape, "f32", ctx) for k, (e, shape) in exprs.items()}
        self.exprs = {k: e for k, (e, _) in exprs.items()}
        self.kbytes = {k: plan_bytes(plan(self.outs[k].mat_id, e.node)) for k, e in self.exprs.items()}
        run.sync()

    def launches(self):
        return [(k, lambda k=k: self.outs[k].assign(self.exprs[k]), self.kbytes[k]) for k in self.labels]

    def elements_per_step(self):
        return sum(m.n_elem for m in self.outs.values())

    def check(self):
        x, y = self.a.to_numpy(), self.b.to_numpy()
        t = np.float32(2)
        want = {"add2": (x + y)[:, :4], "expr1": (t * (x.T + y) + t * (x + y.T))[:, :4]}
        return {f"{k}_bit_exact_4_cols": bool(np.array_equal(self.outs[k].to_numpy()[:, :4], w))
                for k, w in want.items()}

    def cpu(self, threads, n=4096):
        from oracle import fm_oracle as orc
        x, y = orc.randu(n, n, 42), orc.randu(n, n, 43)
        return (lambda: 2 * (x.T + y) + 2 * (x + y.T)), 12 * n * n, "port", 1, \
            f"numpy restatement of expr1 on {n}x{n}, 1 thread"


def plan_bytes(pl) -> int:
    """Algorithmic bytes of a plan (reference bench.py:218-240 convention);
    temps written and re-read between split launches count as traffic."""
    from paper_2604_22242_b200.plan import FusedKernelStep, GemmStep
    total = 0
    for step in pl.steps:
        if isinstance(step, GemmStep):
            # reference: (left + right + out) elements of the product step; an
            # operand prologue reads its expression's inputs instead
            for sid, shape, expr in ((step.a_id, step.a_shape, step.a_expr), (step.b_id, step.b_shape, step.b_expr)):
                if expr is None:
                    total += shape.n_elem * step.in_etype.width
                else:
                    total += sum(sp.parent_shape.n_elem * sp.etype.width for sp in expr.inputs)
            total += step.out_shape.n_elem * step.out_etype.width
            continue
        if not isinstance(step, FusedKernelStep):
            continue
        for spec in step.inputs:
            if spec.dense_count > 0:
                total += spec.parent_shape.n_elem * spec.etype.width
            else:
                distinct = {(v.kind, v.row_off, v.col_off, v.n_rows, v.n_cols) for v in spec.views}
                total += sum(r * c for (_, _, _, r, c) in distinct) * spec.etype.width
        total += step.domain_shape.n_elem * step.expr.etype.width
    return total


REF_WORKLOAD = {
    "c2": "C2 fused reductions accu(X%Y), dot(x,y), norm(x-y) on 1e8-element f32 and f64 vectors",
    "c1": "C1 Z = 2*(X % Y) + X, f32 4096x4096",
    "c3": "C3 Z = exp(-square(X - Y)/2) + 0.5*abs(X), f32 32768x32768",
    "c4": "C4 column-wise sum/mean/max/index_max of (X - Y) % Z, f64 65536x16384",
    "c4r": "C4-rows row-wise sum/mean/max/index_max of (X - Y) % Z, f64 65536x16384",
    "c5": "C5 Z = 2*X*Y.t() bf16 GEMM 8192x8192x8192",
    "c5f32": "C5 Z = 2*X*Y.t() f32 GEMM 8192x8192x8192",
    "suite": "paper suite (13 expressions) + addN sweep, f32 10000x10000",
}

CONFIGS = {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c4r": C4Rows, "c5": C5, "c5f32": C5F32, "suite": Suite}
ALL = ["c2", "c1", "c3", "c4", "c5", "c5f32"]     # the default run: headline first


# --------------------------------------------------------------------------------------
# measurement

def time_cpu(run, work, steps, warmup, scale):
    for _ in range(warmup):
        run()
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run()
        t.append(time.perf_counter() - t0)
    return work / statistics.fmean(t) / scale, statistics.fmean(t)


def cpu_leg(cfg: Config, scale: float, steps=3, warmup=1) -> dict:
    threads = os.cpu_count() or 1
    run, work, kind, threads, desc = cfg.cpu(threads)
    v, _ = time_cpu(run, work, steps, warmup, scale)
    return {"value": round(v, 3), "unit": cfg.unit, "cores": threads, "kind": kind, "sample": desc,
            "cpu_model": cpu_model(), "nproc": os.cpu_count()}


def dominant_kernel(labels, kwork, per_kernel, steps_ms) -> dict:
    """The roofline's kernel: launches of one kernel ("c1_copy_f32[0..5]")
    form a family, and the family with the largest share of the
    instrumented step dominates.  Its mean launch duration comes from the
    events between launches, except when every launch of the step belongs
    to it: then the timed step's own events over the launch count give it
    (no events between the launches, which cost ~6 us each).

    labels / kwork: per launch slot; per_kernel[i]: slot i's event-timed
    duration (ms) in each instrumented step; steps_ms: the timed steps."""
    steps = len(per_kernel[0])
    share = [sum(v) for v in per_kernel]
    fam = [l.split("[")[0] for l in labels]
    fams = sorted({f for f, w in zip(fam, kwork) if w})
    fshare = {f: sum(s for s, g in zip(share, fam) if g == f) for f in fams}
    fwork = {f: sum(w for w, g in zip(kwork, fam) if g == f) for f in fams}
    fcount = {f: sum(1 for g in fam if g == f) for f in fams}
    dfam = max(fams, key=lambda f: fshare[f])
    step_mean = statistics.fmean(steps_ms)
    if len(set(fam)) == 1:
        mean_launch = step_mean / fcount[dfam]
    else:
        mean_launch = fshare[dfam] / (steps * fcount[dfam])
    return {"kernel": dfam, "first_label": labels[fam.index(dfam)], "launches_per_step": fcount[dfam],
            "mean_launch_ms": mean_launch, "work_per_launch": fwork[dfam] / fcount[dfam],
            "work_per_step": fwork[dfam], "share_of_step_ms": step_mean * fshare[dfam] / sum(share)}


def measure(run: Run, cfg: Config, steps: int, warmup: int, with_cpu: bool, with_e2e: bool,
            use_graph: bool = True) -> dict:
    fm, nat, backend, p = run.fm, run.nat, run.backend, run.p
    launches = cfg.launches()
    labels = [l for l, _, _ in launches]
    kwork = [w for _, _, w in launches]
    fns = [f for _, f, _ in launches]
    nk = len(fns)
    flush_h = None
    if cfg.flush:
        flush_h = backend.alloc(fm.ElemType.f32, 256 * 1024 * 1024 // 4 * 2)   # 512 MiB > 126 MB L2

    def flush():
        if flush_h is not None:
            nat.call("fm_flush_l2", backend.ptr(flush_h), flush_h.n_elem * 4, backend.stream)

    for _ in range(warmup):
        for f in fns:
            f()
    run.sync()
    p.barrier()

    ev = Events(nat, backend.stream, (nk + 1) * steps)

    def step_plain():
        for f in fns:
            f()

    def step_instrumented(s):
        base = s * (nk + 1)
        ev.record(base)
        for i, f in enumerate(fns):
            f()
            ev.record(base + i + 1)

    # One CUDA graph per step, captured from the public-API calls: the timed
    # region replays the same kernels on the same buffers with no host planning.
    # Events only at step boundaries there; per-kernel times come from a second,
    # instrumented pass (an event between two kernels costs ~6 us).
    # With an L2 flush between steps the flush is captured into the step's
    # graph, right before the start event: the device runs flush -> step with
    # no host gap (a large graph's launch can outlast the flush, and the first
    # kernel after an idle GPU runs ~40 us slow, scripts/first_after_flush.py).
    sev = Events(nat, backend.stream, 2 * steps)

    def step_timed(s):
        flush()
        sev.record(2 * s)
        step_plain()
        sev.record(2 * s + 1)

    g_step = g_instr = g_timed = None
    if use_graph:
        g_step = fm.capture(step_plain, run.ctx)
        if flush_h is not None:
            g_timed = [fm.capture(lambda s=s: step_timed(s), run.ctx) for s in range(steps)]
        g_instr = [fm.capture(lambda s=s: (flush(), step_instrumented(s)), run.ctx) for s in range(steps)]
        g_step.replay()
        run.sync()
        p.barrier()
    sampler = ClockSampler(p.device).start()
    time.sleep(0.25)
    run.sync()
    p.barrier()
    c0 = nat.lib.fm_launch_counter()
    t_wall0 = time.perf_counter()
    for s in range(steps):
        if g_timed is not None:
            g_timed[s].replay()
            continue
        flush()
        sev.record(2 * s)
        if g_step is not None:
            g_step.replay()
        else:
            step_plain()
        sev.record(2 * s + 1)
    run.sync()
    p.barrier()
    t_wall = time.perf_counter() - t_wall0
    c1 = nat.lib.fm_launch_counter()
    clocks = merge_clocks(p.gather(sampler.stop()))
    steps_ms = [sev.ms(2 * s, 2 * s + 1) for s in range(steps)]

    run.sync()
    p.barrier()
    for s in range(steps):
        if g_instr is not None:
            g_instr[s].replay()
        else:
            flush()
            step_instrumented(s)
    run.sync()
    per_kernel = [[ev.ms(s * (nk + 1) + i, s * (nk + 1) + i + 1) for s in range(steps)] for i in range(nk)]
    for g in [g_step] + (g_instr or []) + (g_timed or []):
        if g is not None:
            g.close()
    ev.close()
    sev.close()
    if flush_h is not None:
        backend.free(flush_h)

    ms_per_step = p.max(statistics.fmean(steps_ms))
    tensor = cfg.bound == "tensor"
    scale = 1e12 if tensor else 1e9
    work_all = p.sum(sum(kwork))
    value = work_all / (ms_per_step * 1e-3) / scale
    peaks = measured_peaks()
    dk = dominant_kernel(labels, kwork, per_kernel, steps_ms)
    dfam, mean_launch, work_launch = dk["kernel"], dk["mean_launch_ms"], dk["work_per_launch"]
    achieved = work_launch / (mean_launch * 1e-3) / scale
    in_step = dk["work_per_step"] / (dk["share_of_step_ms"] * 1e-3) / scale
    dom = labels.index(dk["first_label"])
    means = [statistics.fmean(v) for v in per_kernel]
    common = {"kernel": dfam, "launches_per_step": dk["launches_per_step"], "achieved": round(achieved, 1),
              "traffic": ncu_traffic(labels[dom]),
              "mean_launch_us": round(mean_launch * 1e3, 2), "achieved_in_timed_steps": round(in_step, 1),
              "timing": TIMING_NOTE}
    if tensor:
        peak = peaks["bf16_tflops"]
        roofline = {"bound": "tensor", "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                    "frac_of_sustained": round(achieved / peaks["bf16_tflops_sustained"], 4),
                    "frac_of_2250_spec": round(achieved / 2250.0, 4),
                    "peak_source": peaks["source"] + " bf16 burst", "algorithmic_flops_per_launch": work_launch,
                    **common}
    else:
        roofline = {"bound": "hbm", "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(achieved / peaks["hbm_gbs"], 4), "frac_of_8TBs": round(achieved / SPEC_HBM_GBS, 4),
                    "peak_source": peaks["source"], "algorithmic_bytes_per_launch": work_launch, **common,
                    "per_kernel_gbs": {lab: round(b / (m * 1e-3) / 1e9, 1) for lab, b, m in zip(labels, kwork, means)
                                       if b}}
    out = {"metric": cfg.metric, "value": round(value, 2), "unit": cfg.unit, "n_gpus": run.world,
           "steps": steps, "warmup": warmup, "ms_per_step": round(ms_per_step, 4),
           "higher_is_better": True, "scaling": cfg.scaling, "dtype": cfg.dtype,
           "config": {"workload": cfg.workload,
                      "elements_per_gpu_per_step": cfg.elements_per_step(),
                      ("algorithmic_flops_per_step" if tensor else "algorithmic_bytes_per_step"): work_all,
                      "l2": ("L2 flushed before every timed step (512 MiB write then read)" if flush_h is not None
                             else "inputs larger than the 126 MB L2; no flush"),
                      "launch": "one CUDA graph replay per step (captured from the public API calls)"
                      if g_step is not None else "eager public API calls",
                      "parallelism": (f"{run.world} ranks, one process per GPU, collectives: libfmb200 "
                                      f"{run.comm.transport}" if run.world > 1 else "1 GPU")},
           "elements_per_s": round(p.sum(cfg.elements_per_step()) / (ms_per_step * 1e-3), 1),
           **({"pct_of_8TBs_per_gpu": round(100 * value / run.world / SPEC_HBM_GBS, 2)} if not tensor else {}),
           "roofline": roofline, "gpu_launches": int(p.sum(c1 - c0)), "clocks": clocks,
           "wall_s_timed_region": round(t_wall, 4),
           "per_kernel_ms": {lab: round(m, 4) for lab, m in zip(labels, means)}}
    out["check"] = cfg.check()
    out.update(cfg.extra(out))

    if with_e2e:
        io = cfg.setup_e2e()
        if io is not None:
            h2d, d2h = io
            cfg.step_e2e()
            run.sync()
            p.barrier()
            t = []
            for _ in range(max(2, min(steps, 5))):
                run.sync()
                p.barrier()
                t0 = time.perf_counter()
                cfg.step_e2e()
                run.sync()
                t.append(time.perf_counter() - t0)
            e2e_s = p.max(statistics.fmean(t))
            ework = p.sum(cfg.e2e_work() if hasattr(cfg, "e2e_work") else sum(kwork))
            out["e2e"] = {"value": round(ework / e2e_s / scale, 3), "unit": cfg.unit,
                          "h2d_bytes_per_step": int(p.sum(h2d)), "d2h_bytes_per_step": int(p.sum(d2h)),
                          "ms_per_step": round(e2e_s * 1e3, 3), "path": cfg.e2e_path}
    out.setdefault("e2e", None)
    out["cpu_baseline"] = cpu_leg(cfg, scale) if (with_cpu and run.world == 1) else None
    return out


def ours(args, p: Plumb) -> int:
    run = Run(args, p)
    names = ALL if args.config == "all" else [args.config]
    results = {}
    for name in names:
        cfg = CONFIGS[name](run)
        results[name] = measure(run, cfg, args.steps, args.warmup, not args.no_cpu, not args.no_e2e,
                                use_graph=not args.no_graph)
        del cfg
        gc.collect()
        run.sync()
        p.barrier()
    head = dict(results[names[0]])
    if args.config == "all":
        head["metric"] = METRIC
        head["configs"] = {}
        for name in names[1:]:
            r = dict(results[name])
            key = {"c5": "c5_bf16", "c5f32": "c5_f32"}.get(name, name)
            head["configs"][key] = r
    head["vs_baseline"] = None
    head["data"] = "synthetic (the reference's splitmix64 randu stream, generated on the device)"
    if run.comm.transport != "none":
        head["comm_status"] = run.comm.status()
    if p.rank == 0:
        print(json.dumps(head, default=float), flush=True)
    run.comm.close()
    return 0


# --------------------------------------------------------------------------------------
# reference arm

class _ArmRun:
    """Just enough of Run for the configs' CPU legs (no GPU)."""

    def __init__(self, args):
        self.args, self.world, self.rank = args, 1, 0


def reference_arm(args, p: Plumb) -> int:
    if p.rank != 0:
        return 0
    names = ALL if args.config == "all" else [args.config]
    steps, warmup = max(1, args.steps), max(1, args.warmup)
    lines = {}
    for name in names:
        cls = CONFIGS[name]
        cfg = object.__new__(cls)
        Config.__init__(cfg, type("R", (), {"fm": None, "ctx": None})())
        cfg.run = _ArmRun(args)
        cfg.n = {"c1": 4096, "c3": 32768, "c5": 8192, "c5f32": 8192, "suite": 10000}.get(name, 0)
        threads = os.cpu_count() or 1
        scale = 1e12 if cls.bound == "tensor" else 1e9
        if name == "c2":
            # the headline runs on the FULL config: 1e8-element vectors
            n = args.n or 100_000_000
            fn, work, kind, thr, desc = cfg.cpu(threads, n_sample=n)
            st, wu = steps, warmup
        else:
            fn, work, kind, thr, desc = cfg.cpu(threads)
            st, wu = min(steps, 5), 1
        v, mean_s = time_cpu(fn, work, st, wu, scale)
        lines[name] = {"impl": "reference", "metric": cls.metric, "value": round(v, 3), "unit": cls.unit,
                       "n_gpus": args.gpus, "steps": st, "warmup": wu, "ms_per_step": round(mean_s * 1e3, 3),
                       "higher_is_better": True, "scaling": cls.scaling, "vs_baseline": None,
                       "dtype": cls.dtype, "data": "synthetic (reference splitmix64 randu)",
                       "config": {"workload": REF_WORKLOAD[name], "sample": desc},
                       "cpu_baseline": {"value": round(v, 3), "unit": cls.unit, "cores": thr, "kind": kind,
                                        "sample": desc, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
                       "e2e": {"value": round(v, 3), "unit": cls.unit, "h2d_bytes_per_step": 0,
                               "d2h_bytes_per_step": 0}}
    head = dict(lines[names[0]])
    if args.config == "all":
        head["metric"] = METRIC
        head["configs"] = {{"c5": "c5_bf16", "c5f32": "c5_f32"}.get(k, k): v for k, v in lines.items()
                           if k != names[0]}
    print(json.dumps(head), flush=True)
    return 0


# --------------------------------------------------------------------------------------

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(gpus: int, argv: list[str]) -> int:
    """`--gpus N` outside torchrun: start N ranks (one per GPU) ourselves."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["all", *sorted(CONFIGS)], default="all")
    ap.add_argument("--size", "--n", dest="n", type=int, default=0,
                    help="override the size (per-GPU vector length for c2, global n otherwise)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every timed step eagerly instead of replaying its CUDA graph")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus, argv)
    p = Plumb(args.gpus)
    try:
        if args.impl == "reference":
            return reference_arm(args, p)
        return ours(args, p)
    finally:
        p.close()


if __name__ == "__main__":
    sys.exit(main())
