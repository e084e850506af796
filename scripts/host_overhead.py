"""Host cost of one `Mat.assign` on a small matrix (plan memo + bound-program
memo) vs a freshly built expression; the reference spends
~46 us per assign on its compiled backend."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402

ctx = fm.Context("cuda")
X, Y, Z = (fm.randu(64, 64, s, "f32", ctx) for s in (1, 2, 3))
e = 2 * (X % Y) + X
for _ in range(500):
    Z.assign(e)
ctx.sync()
N = 20000
t = time.perf_counter()
for _ in range(N):
    Z.assign(e)
ctx.sync()
same = (time.perf_counter() - t) / N * 1e6
t = time.perf_counter()
for _ in range(N // 4):
    Z.assign(2 * (X % Y) + X)
ctx.sync()
fresh = (time.perf_counter() - t) / (N // 4) * 1e6
g = fm.capture(lambda: [Z.assign(e) for _ in range(100)], ctx)
t = time.perf_counter()
for _ in range(N // 100):
    g.replay()
ctx.sync()
graph = (time.perf_counter() - t) / N * 1e6
print(f"assign, same expression: {same:.2f} us; freshly built expression: {fresh:.2f} us; "
      f"graph replay per launch: {graph:.2f} us")
