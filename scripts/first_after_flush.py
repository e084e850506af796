"""Why is the first kernel after the L2 flush slower?  Time a+b (f32 10000^2)
right after fm_flush_l2 and again immediately after, with CUDA events."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402
from paper_2604_22242_b200._native import native  # noqa: E402

nat = native()
ctx = fm.Context(fm.B200Backend())
be = ctx.backend
n = 10000
a, b = fm.randu(n, n, 1, "f32", ctx), fm.randu(n, n, 2, "f32", ctx)
Z1, Z2, Z3 = (fm.Mat(n, n, "f32", ctx) for _ in range(3))
fl = be.alloc(fm.ElemType.f32, 256 * 1024 * 1024 // 4 * 2)
evs = []
for _ in range(4):
    e = ctypes.c_void_p()
    nat.call("fm_event_create", ctypes.byref(e))
    evs.append(e.value)


def ms(i, j):
    f = ctypes.c_float()
    nat.call("fm_event_elapsed_ms", evs[i], evs[j], ctypes.byref(f))
    return f.value


def flush():
    nat.call("fm_flush_l2", be.ptr(fl), fl.n_elem * 4, be.stream)


for mode in ("flush", "noflush", "flush+sync", "flush+sleep"):
    res = []
    for rep in range(6):
        if mode != "noflush":
            flush()
        if mode == "flush+sync":
            ctx.sync()
        if mode == "flush+sleep":
            nat.call("fm_sleep_ns", 200000, be.stream) if hasattr(nat.lib, "fm_sleep_ns") else None
        nat.call("fm_event_record", evs[0], be.stream)
        Z1.assign(a + b)
        nat.call("fm_event_record", evs[1], be.stream)
        Z2.assign(a + b)
        nat.call("fm_event_record", evs[2], be.stream)
        Z3.assign(a + b)
        nat.call("fm_event_record", evs[3], be.stream)
        ctx.sync()
        if rep:
            res.append((ms(0, 1), ms(1, 2), ms(2, 3)))
    m = [sum(r[i] for r in res) / len(res) for i in range(3)]
    gb = 1.2e9
    print(f"{mode:12s} first {m[0]*1e3:7.1f} us ({gb/m[0]/1e6:6.0f} GB/s)  second {m[1]*1e3:7.1f} us "
          f"({gb/m[1]/1e6:6.0f})  third {m[2]*1e3:7.1f} us ({gb/m[2]/1e6:6.0f})", flush=True)


def body():
    nat.call("fm_event_record", evs[0], be.stream)
    Z1.assign(a + b)
    nat.call("fm_event_record", evs[1], be.stream)
    Z2.assign(a + b)
    nat.call("fm_event_record", evs[2], be.stream)
    Z3.assign(a + b)
    nat.call("fm_event_record", evs[3], be.stream)


g_out = fm.capture(body, ctx)
g_in = fm.capture(lambda: (flush(), body()), ctx)
for mode in ("graph after flush", "flush in graph"):
    res = []
    for rep in range(6):
        if mode == "graph after flush":
            flush()
            g_out.replay()
        else:
            g_in.replay()
        ctx.sync()
        if rep:
            res.append((ms(0, 1), ms(1, 2), ms(2, 3)))
    m = [sum(r[i] for r in res) / len(res) for i in range(3)]
    gb = 1.2e9
    print(f"{mode:18s} first {m[0]*1e3:7.1f} us ({gb/m[0]/1e6:6.0f} GB/s)  second {m[1]*1e3:7.1f} us "
          f"({gb/m[1]/1e6:6.0f})  third {m[2]*1e3:7.1f} us ({gb/m[2]/1e6:6.0f})", flush=True)
