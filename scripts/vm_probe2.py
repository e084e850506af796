"""One VM launch of C1 (2*(X%Y)+X, f32 8192^2) for an ncu capture."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_22242_b200 as fm  # noqa: E402

be = fm.B200Backend(use_templates=False)
ctx = fm.Context(be)
n = 8192
X, Y = fm.randu(n, n, 1, "f32", ctx), fm.randu(n, n, 2, "f32", ctx)
Z = fm.Mat(n, n, "f32", ctx)
for _ in range(3):
    Z.assign(2 * (X % Y) + X)
ctx.sync()
