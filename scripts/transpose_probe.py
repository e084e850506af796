"""Transposed-leaf suite members on the tile-pair skeleton (csrc/pair.cuh):
expr1 = 2*(X.t()+Y) + 2*(X+Y.t()) and expr2 = 0.5*A + (B+C).t() + log(D**2),
f32 and f64, at several n (aligned and ragged), GB/s of algorithmic bytes.
Usage: python scripts/transpose_probe.py [n ...]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402
from paper_2604_22242_b200._native import native  # noqa: E402

nat = native()
ctx = fm.Context("cuda")
be = ctx.backend
sizes = [int(a) for a in sys.argv[1:]] or [8192, 10000, 10240]
for n in sizes:
    for et, w in (("f32", 4), ("f64", 8)):
        ms = [fm.randu(n, n, 1 + i, et, ctx) for i in range(4)]
        X, Y, C, D = ms
        Z = fm.Mat(n, n, et, ctx)
        for name, e, nin in (("expr1", 2 * (X.t() + Y) + 2 * (X + Y.t()), 2),
                             ("expr2", 0.5 * X + (Y + C).t() + fm.log(D ** 2), 4)):
            for _ in range(3):
                Z.assign(e)
            g = fm.capture(lambda: [Z.assign(e) for _ in range(10)], ctx)
            a, b = ctypes.c_void_p(), ctypes.c_void_p()
            nat.call("fm_event_create", ctypes.byref(a))
            nat.call("fm_event_create", ctypes.byref(b))
            g.replay()
            ctx.sync()
            nat.call("fm_event_record", a.value, be.stream)
            g.replay()
            nat.call("fm_event_record", b.value, be.stream)
            f = ctypes.c_float()
            nat.call("fm_event_elapsed_ms", a.value, b.value, ctypes.byref(f))
            us = f.value / 10 * 1e3
            print(f"{name} {et} n={n}: {us:8.1f} us  {(nin + 1) * w * n * n / (us * 1e-6) / 1e9:7.1f} GB/s", flush=True)
            g.close()
        del ms, X, Y, C, D, Z
