"""Register VM vs template on dim reductions (f64 16384 x 8192): the C4
expression (template) and one without a template, sum/max/index_max along
both dims, GB/s of algorithmic bytes."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402
from paper_2604_22242_b200._native import native  # noqa: E402

nat = native()


def gbs(use_templates, build, nin, dim, r=16384, c=8192, reps=10):
    be = fm.B200Backend(use_templates=use_templates)
    ctx = fm.Context(be)
    ms = [fm.randu(r, c, 40 + i, "f64", ctx) for i in range(nin)]
    e = build(*ms)
    n = c if dim == 0 else r
    outs = [fm.Mat(1, n, "f64", ctx) if dim == 0 else fm.Mat(n, 1, "f64", ctx) for _ in range(2)]
    im = fm.Mat(1, n, "u32", ctx) if dim == 0 else fm.Mat(n, 1, "u32", ctx)
    step = lambda: fm.assign_all([(outs[0], fm.sum(e, dim)), (outs[1], fm.max(e, dim)),  # noqa: E731
                                  (im, fm.index_max(e, dim))])
    for _ in range(2):
        step()
    g = fm.capture(lambda: [step() for _ in range(reps)], ctx)
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
    return nin * 8 * r * c / (f.value / reps * 1e-3) / 1e9


for name, build, nin in (("c4 (X-Y)%Z", lambda X, Y, Z: (X - Y) % Z, 3), ("2X-Y*Z", lambda X, Y, Z: 2 * X - Y % Z, 3)):
    for dim in (0, 1):
        t, v = gbs(True, build, nin, dim), gbs(False, build, nin, dim)
        print(f"{name:12s} dim {dim}: template {t:8.1f} GB/s   VM {v:8.1f} GB/s", flush=True)
