"""ncu --set full captures of every config's dominant kernel for one round.

    python scripts/ncu_round.py OUTDIR [name ...]

Each capture: one launch of the named kernel (demangled-name regex) inside a
one-step bench run of its config, exported as raw / details / source CSV next
to the summary scripts/ncu_summary.py reads.  Runs on the GPU box (gpurun)."""
import subprocess
import sys
from pathlib import Path

CAPS = {
    # name: (demangled kernel regex, bench config, launches to skip); template
    # arguments demangle as "fm::tx::SMul<(int)0, ...>"
    "ncu_c1_copy": (r"k_copy<.*SMul<\(int\)0, fm::tx::Mul<", "c1", 0),
    "ncu_c2_accu_f32": (r"k_accu_bulk<.*Mul<fm::tx::In<\(int\)0>, fm::tx::In<\(int\)1>>, float", "c2", 0),
    "ncu_c2_norm_f32": (r"k_accu_bulk<.*Pow<.*Sub<.*>>, float, \(int\)", "c2", 0),
    "ncu_c2_accu_f64": (r"k_accu_bulk<.*Mul<fm::tx::In<\(int\)0>, fm::tx::In<\(int\)1>>, double", "c2", 0),
    "ncu_c2_norm_f64": (r"k_accu_bulk<.*Pow<.*Sub<.*>>, double, \(int\)", "c2", 0),
    "ncu_c3_copy": (r"k_copy_bulk<.*Exp<", "c3", 0),
    "ncu_c4_colstats": (r"k_reduce_cols_fast", "c4", 0),
    "ncu_c4r_rowstats": (r"k_reduce_rows", "c4r", 0),
    "ncu_c5_gemm": (r"k_gemm_bf16_pair", "c5", 0),
    "ncu_c5f32_gemm": (r"k_gemm_bf16_pair", "c5f32", 0),
    "ncu_suite_expr1": (r"k_copy_pair<.*SMul<\(int\)1, .*float", "suite", 0),
    "ncu_suite_expr2": (r"k_copy_pair<.*Log<.*float", "suite", 0),
    "ncu_suite_add32": (r"k_copy<.*In<\(int\)31>", "suite", 0),
    "ncu_suite_sigmoid": (r"k_copy\w*<.*SDiv<.*Exp<", "suite", 0),
    "ncu_suite_gelu": (r"k_copy\w*<.*Tanh<", "suite", 0),
    "ncu_suite_expr3": (r"k_copy\w*<.*CvtU32<", "suite", 0),
}


def run(out: Path, name: str):
    kre, cfg, skip = CAPS[name]
    rep = out / name
    cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
           "--kernel-name-base", "demangled", "-k", f"regex:{kre}", "-s", str(skip), "-c", "1",
           "-o", str(rep), "-f", sys.executable, "bench.py", "--config", cfg, "--steps", "1",
           "--warmup", "0", "--no-e2e", "--no-cpu"]
    with open(out / f"{name}.ncu.log", "w") as fh:
        subprocess.run(cmd, stdout=fh, stderr=subprocess.STDOUT, timeout=900)
    for page, suffix in (("raw", "raw.csv"), ("details", "details.csv")):
        with open(out / f"{name}.{suffix}", "w") as fh:
            subprocess.run(["ncu", "-i", f"{rep}.ncu-rep", "--page", page, "--csv"], stdout=fh,
                           stderr=subprocess.DEVNULL)
    with open(out / f"{name}.sass.csv", "w") as fh:
        subprocess.run(["ncu", "-i", f"{rep}.ncu-rep", "--page", "source", "--csv", "--print-source", "sass"],
                       stdout=fh, stderr=subprocess.DEVNULL)
    subprocess.run(["gzip", "-f", str(out / f"{name}.sass.csv")])
    rp = Path(f"{rep}.ncu-rep")
    if rp.exists() and rp.stat().st_size > 8_000_000:
        rp.unlink()


if __name__ == "__main__":
    out = Path(sys.argv[1])
    out.mkdir(parents=True, exist_ok=True)
    for n in sys.argv[2:] or list(CAPS):
        run(out, n)
        print(n, "done", flush=True)
