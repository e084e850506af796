"""Build libfmb200.so: every CUDA source compiled ahead of time for sm_100a.

    python -m paper_2604_22242_b200.build        (or __graft_entry__.build())

No JIT, no torch extension machinery: plain nvcc objects linked into one
shared library with the CUDA runtime statically linked, placed next to this
file so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "fmb200"
LIB = PKG / "libfmb200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-I", str(INCLUDE), "-I", str(CSRC)]
SOURCES = ["runtime.cu", "fused.cu", "rng.cu", "gemm_simt.cu", "gemm_tc.cu", "comm.cu"]


def units() -> list[tuple[str, str, list[str]]]:
    """(object stem, source, extra defines) of every compilation unit.

    The two heavy sources are compiled several times with different macros so
    nvcc runs them in parallel: the register-VM kernels once per (variant,
    skeleton) and the expression-template kernels once per shard.
    """
    from .aot_registry import TEMPLATE_SHARDS
    out = [(Path(s).stem, s, []) for s in SOURCES]
    for v in range(4):
        for k in range(4):
            out.append((f"vm_inst_{v}_{k}", "vm_inst.cu", [f"-DFM_VM_VARIANT={v}", f"-DFM_VM_SKELETON={k}"]))
    for k in range(TEMPLATE_SHARDS):
        out.append((f"gen_templates_{k}", "gen_templates.cu",
                    [f"-DFM_TEMPLATE_SHARD={k}", f"-DFM_TEMPLATE_SHARDS={TEMPLATE_SHARDS}"]))
    return out


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(path).exists():
        raise RuntimeError("nvcc not found")
    return path


def _deps_mtime() -> float:
    files = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.inc")) + list(INCLUDE.glob("*.h"))
    return max(f.stat().st_mtime for f in files)


def _compile(src: Path, obj: Path, defines: list[str], verbose: bool) -> str:
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *defines, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-6000:]}")
    (obj.with_suffix(".ptxas.txt")).write_text(r.stderr)
    return obj.stem


def build(force: bool = False, verbose: bool = False) -> Path:
    from .aot_registry import generate
    BUILD.mkdir(parents=True, exist_ok=True)
    generate(CSRC / "gen_templates.cu")
    dep = _deps_mtime()
    jobs = []
    objs = []
    for stem, name, defines in units():
        src = CSRC / name
        obj = BUILD / (stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, dep):
            jobs.append((src, obj, defines))
    if jobs:
        workers = min(len(jobs), os.cpu_count() or 4)
        with ThreadPoolExecutor(max_workers=workers) as ex:
            for name in ex.map(lambda j: _compile(j[0], j[1], j[2], verbose), jobs):
                if verbose:
                    print(f"  compiled {name}", file=sys.stderr)
    for stale in BUILD.glob("*.o"):
        if stale not in objs:
            stale.unlink()
    if force or jobs or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
