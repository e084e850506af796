"""expr1 (2*(X.t()+Y) + 2*(X+Y.t())) in f32 and f64 at n^2, GB/s (plan_bytes)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402
from paper_2604_22242_b200._native import native  # noqa: E402

nat = native()
ctx = fm.Context("cuda")
be = ctx.backend
for et, w in (("f32", 4), ("f64", 8)):
    n = 8192
    X, Y = fm.randu(n, n, 1, et, ctx), fm.randu(n, n, 2, et, ctx)
    Z = fm.Mat(n, n, et, ctx)
    e = 2 * (X.t() + Y) + 2 * (X + Y.t())
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
    print(f"expr1 {et} {3 * w * n * n / (f.value / 10 * 1e-3) / 1e9:.1f} GB/s")
