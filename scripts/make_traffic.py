"""profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per
launch of each bench kernel, from the committed `ncu --set full` raw exports.

bench.py reads this file for roofline.traffic.  A label maps to the capture of
the kernel instantiation it launches (dot_X launches the same k_accu<Mul<..>>
instantiation as accu_schur_X, so they share a capture).

    python scripts/make_traffic.py [round-dir ...]   (default: profiles/r02, then profiles/r01 for labels r02 lacks)
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

LABELS = {
    "c1_copy_f32": "ncu_c1_copy",
    "accu_schur_f32": "ncu_c2_accu_f32", "dot_f32": "ncu_c2_accu_f32",
    "norm_sqdiff_f32": "ncu_c2_norm_f32",
    "accu_schur_f64": "ncu_c2_accu_f64", "dot_f64": "ncu_c2_accu_f64",
    "norm_sqdiff_f64": "ncu_c2_norm_f64",
    "c3_copy_f32": "ncu_c3_copy",
    "c4_colstats_f64": "ncu_c4_colstats",
    "c4_rowstats_f64": "ncu_c4r_rowstats",
    "c5_gemm_bf16": "ncu_c5_gemm",
    "c5_gemm_f32": "ncu_c5f32_gemm",
    "expr1": "ncu_suite_expr1",
    "expr2": "ncu_suite_expr2",
    "expr3": "ncu_suite_expr3",
    "sigmoid": "ncu_suite_sigmoid",
    "gelu": "ncu_suite_gelu",
    "add32N": "ncu_suite_add32",
}


def dram_bytes(raw: Path):
    rows = list(csv.reader(raw.open()))
    h, units, vals = rows[0], rows[1], rows[2]
    total = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        total += float(vals[i].replace(",", "")) * UNIT.get(units[i], 1)
    t = h.index("gpu__time_duration.sum")
    return int(total), vals[t] + " " + units[t]


def main(dirs):
    out = {}
    for label, stem in LABELS.items():
        for d in dirs:
            raw = ROOT / d / f"{stem}.raw.csv"
            if raw.exists():
                b, dur = dram_bytes(raw)
                out[label] = {"dram_bytes": b, "duration": dur, "source": str(raw.relative_to(ROOT))}
    (ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or ["profiles/r01", "profiles/r02"])
