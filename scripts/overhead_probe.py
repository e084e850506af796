"""Per-launch fixed overhead of the fused accu kernel: time R back-to-back
launches (one CUDA graph, events only around the whole graph) at several
sizes and fit t = bytes / B + X.  Usage: python scripts/overhead_probe.py"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2604_22242_b200 as fm  # noqa: E402
from paper_2604_22242_b200._native import native  # noqa: E402

nat = native()
ctx = fm.Context("cuda")
be = ctx.backend
R = 20


def ev():
    e = ctypes.c_void_p()
    nat.call("fm_event_create", ctypes.byref(e))
    return e.value


for et, w in (("f32", 4), ("f64", 8)):
    pts = []
    for n in (25_000_000, 50_000_000, 100_000_000, 200_000_000):
        x = fm.Col(n, et, ctx)
        y = fm.Col(n, et, ctx)
        be.randu(x.handle, 1)
        be.randu(y.handle, 2)
        r = fm.Mat(1, 1, "f64", ctx)
        for _ in range(3):
            fm.accu_async(x % y, r, 0)
        g = fm.capture(lambda: [fm.accu_async(x % y, r, 0) for _ in range(R)], ctx)
        g.replay()
        ctx.sync()
        a, b = ev(), ev()
        best = 1e9
        for _ in range(5):
            nat.call("fm_event_record", a, be.stream)
            g.replay()
            nat.call("fm_event_record", b, be.stream)
            f = ctypes.c_float()
            nat.call("fm_event_elapsed_ms", a, b, ctypes.byref(f))
            best = min(best, f.value / R)
        byts = 2 * w * n
        pts.append((byts, best * 1e-3))
        print(f"{et} n={n:>11,} {best*1e3:8.2f} us/launch  {byts/best/1e6:8.1f} GB/s", flush=True)
        g.close()
        del x, y
    A = np.array([[b, 1.0] for b, _ in pts])
    t = np.array([s for _, s in pts])
    (inv_bw, x0), *_ = np.linalg.lstsq(A, t, rcond=None)
    print(f"{et}: asymptotic {1/inv_bw/1e9:.0f} GB/s, fixed overhead {x0*1e6:.2f} us/launch")
