"""Register-VM vs AOT-template throughput on the same expressions (f32,
8192^2, CUDA events, L2 > working set not flushed: inputs 256 MiB each)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402
from paper_2604_22242_b200._native import native  # noqa: E402

nat = native()


def gbs(use_templates, build, nin, n=8192, reps=20):
    be = fm.B200Backend(use_templates=use_templates)
    ctx = fm.Context(be)
    ms = [fm.randu(n, n, 40 + i, "f32", ctx) for i in range(nin)]
    Z = fm.Mat(n, n, "f32", ctx)
    e = build(*ms)
    for _ in range(3):
        Z.assign(e)
    g = fm.capture(lambda: [Z.assign(e) for _ in range(reps)], ctx)
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
    return (nin + 1) * 4 * n * n / (f.value / reps * 1e-3) / 1e9


cases = [("c1 2*(X%Y)+X", lambda X, Y: 2 * (X % Y) + X, 2),
         ("axpby", lambda X, Y: 1.5 * X + 0.25 * Y, 2),
         ("muladd", lambda X, Y, Z: X % Y + Z, 3),
         ("sqrt", lambda X: fm.sqrt(X), 1),
         ("add4", lambda A, B, C, D: A + B + C + D, 4),
         ("add8", lambda *m: m[0] + m[1] + m[2] + m[3] + m[4] + m[5] + m[6] + m[7], 8),
         ("sigmoid", lambda X: 1 / (1 + fm.exp(-X)), 1),
         ("c3", lambda X, Y: fm.exp(-fm.square(X - Y) / 2) + 0.5 * fm.abs(X), 2)]
def accu_gbs(use_templates, build, nin, n=8192, reps=20):
    be = fm.B200Backend(use_templates=use_templates)
    ctx = fm.Context(be)
    ms = [fm.randu(n * n, 1, 40 + i, "f32", ctx) for i in range(nin)]
    R = fm.Mat(1, 1, "f64", ctx)
    e = build(*ms)
    for _ in range(3):
        fm.accu_async(e, R)
    g = fm.capture(lambda: [fm.accu_async(e, R) for _ in range(reps)], ctx)
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
    return nin * 4 * n * n / (f.value / reps * 1e-3) / 1e9


for name, build, nin in [("accu dot", lambda X, Y: X % Y, 2), ("accu 3x-y", lambda X, Y: 3 * X - Y, 2)]:
    t = accu_gbs(True, build, nin)
    v = accu_gbs(False, build, nin)
    print(f"{name:14s} template {t:8.1f} GB/s   VM {v:8.1f} GB/s   VM/template {v / t:.2f}", flush=True)

for name, build, nin in cases:
    t = gbs(True, build, nin)
    v = gbs(False, build, nin)
    print(f"{name:14s} template {t:8.1f} GB/s   VM {v:8.1f} GB/s   VM/template {v / t:.2f}", flush=True)
