"""C1's expression on the register VM (templates off), for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402

be = fm.B200Backend(use_templates=False)
ctx = fm.Context(be)
n = 8192
X, Y = fm.randu(n, n, 42, "f32", ctx), fm.randu(n, n, 43, "f32", ctx)
Z = fm.Mat(n, n, "f32", ctx)
expr = {"c1": lambda: 2 * (X % Y) + X, "c3": lambda: fm.exp(-fm.square(X - Y) / 2) + 0.5 * fm.abs(X)}[
    sys.argv[1] if len(sys.argv) > 1 else "c1"]()
for _ in range(3):
    Z.assign(expr)
ctx.sync()
print("ok")
