"""Build recipe for oracle/_ref/ -- the reference's OWN compiled CPU path.

TEST / BASELINE INFRASTRUCTURE ONLY (never imported by the product).

The reference's native path is C that its code generator emits at run time
and compiles with `cc -O2 -fPIC -fwrapv -shared` (/root/reference/pkg/src/
fusemat/cjit.py:95-111).  This recipe runs the reference's generator
(`fusemat.codegen.generate_kernel_source`, codegen.py:373-391, and the GEMM
template, cjit.py:33-51) from /root/reference for the BASELINE config
expressions, and compiles the emitted sources with the same flags into
oracle/_ref/libfusemat_ref.so plus a manifest.  No reference source is
copied into the repository: oracle/_ref/ is git-ignored build output that
travels to the GPU box with the snapshot, where bench.py's reference arm and
cpu_baseline call it through ctypes (oracle/ref_runner.py).

    python oracle/build_ref.py        (needs /root/reference; no-op without it)
"""

from __future__ import annotations

import json
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg/src")


def kernels():
    """(label, skeleton, node) for every config expression the reference can express."""
    from fusemat import expr as r
    from fusemat.codegen import COPY, REDUCE_ACCU
    S = r.MatShape(8, 8)
    out = []
    for t in (r.ElemType.f32, r.ElemType.f64):
        X, Y, Z = r.leaf(0, t, S), r.leaf(1, t, S), r.leaf(2, t, S)
        tv = t.value
        # C1: 2*(X % Y) + X
        out.append((f"c1_{tv}", COPY, r.plus(r.scalar_pre_mul(2, r.schur(X, Y)), X)))
        # C2: accu(X % Y) == dot(x, y);  norm(x - y)^2 == accu((x - y)**2)
        out.append((f"accu_schur_{tv}", REDUCE_ACCU, r.schur(X, Y)))
        out.append((f"accu_sqdiff_{tv}", REDUCE_ACCU, r.pow_int(r.minus(X, Y), 2)))
        # C3 without abs (the reference has no abs): exp(-square(X - Y)/2) + 0.5*X
        out.append((f"c3noabs_{tv}", COPY, r.plus(
            r.exp(r.scalar_pre_mul(0.5, r.neg(r.pow_int(r.minus(X, Y), 2)))),
            r.scalar_pre_mul(0.5, X))))
        # C4 subexpression (X - Y) % Z
        out.append((f"c4sub_{tv}", COPY, r.schur(r.minus(X, Y), Z)))
    return out


def build() -> Path | None:
    if not REF_SRC.exists():
        print("build_ref: /root/reference not present; keeping existing oracle/_ref", file=sys.stderr)
        return OUT / "libfusemat_ref.so" if (OUT / "libfusemat_ref.so").exists() else None
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF_SRC))
    from fusemat.cjit import _GEMM_TEMPLATE
    from fusemat.codegen import generate_kernel_source

    OUT.mkdir(exist_ok=True)
    manifest = {}
    sources = []
    for label, skel, node in kernels():
        src = generate_kernel_source(node, skel)
        path = OUT / f"{src.entry_point}.c"
        path.write_text(src.text)
        sources.append(path)
        manifest[label] = {"entry": src.entry_point, "signature": src.signature,
                           "schema": [str(a) for a in src.schema]}
    for ctype, tv in (("float", "f32"), ("double", "f64")):
        name = f"gemm_{tv}"
        path = OUT / f"{name}.c"
        path.write_text(_GEMM_TEMPLATE.format(name=name, ctype=ctype))
        sources.append(path)
        manifest[name] = {"entry": name, "signature": f"gemm:{tv}", "schema": []}
    cc = shutil.which("cc") or shutil.which("gcc")
    lib = OUT / "libfusemat_ref.so"
    # cjit.py:102-103 flags, verbatim
    cmd = [cc, "-O2", "-fPIC", "-fwrapv", "-shared", *map(str, sources), "-o", str(lib), "-lm"]
    subprocess.run(cmd, check=True)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1))
    return lib


if __name__ == "__main__":
    print(build())
