"""ctypes runner for oracle/_ref/libfusemat_ref.so -- the reference's own
generated-C kernels (see oracle/build_ref.py).  BASELINE / TEST ONLY.

The reference launches each generated kernel serially over the whole domain
(cjit.py:132-154).  To time the reference on all host cores, `threads > 1`
splits the domain into contiguous column (or, for n x 1 vectors, row) slabs
and calls the SAME kernel on each slab from a thread pool -- ctypes releases
the GIL for the duration of each foreign call.  Reduction partials are
combined in slab order in f64.
"""

from __future__ import annotations

import ctypes
import json
import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libfusemat_ref.so"
MANIFEST = HERE / "_ref" / "manifest.json"

_C = {"f32": ctypes.c_float, "f64": ctypes.c_double, "u32": ctypes.c_uint32, "i32": ctypes.c_int32}


def available() -> bool:
    return LIB.exists() and MANIFEST.exists()


class RefKernels:
    def __init__(self):
        self.lib = ctypes.CDLL(str(LIB))
        self.manifest = json.loads(MANIFEST.read_text())
        self.fns = {}
        for label, m in self.manifest.items():
            fn = getattr(self.lib, m["entry"])
            fn.restype = None
            if m["schema"]:
                fn.argtypes = [self._argtype(s) for s in m["schema"]]
            self.fns[label] = fn

    @staticmethod
    def _argtype(spec: str):
        role, et = spec.split(":")
        if role in ("out", "in"):
            return ctypes.c_void_p
        if role in ("dim", "off"):
            return ctypes.c_longlong
        return _C[et]

    # -- reduce_accu over n x 1 vectors ---------------------------------------------
    def accu(self, label: str, inputs: list[np.ndarray], threads: int | None = None) -> float:
        fn = self.fns[label]
        n = inputs[0].size
        threads = max(1, min(threads or os.cpu_count() or 1, n))
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        outs = np.zeros(threads, np.float64)

        def work(t):
            lo, hi = int(bounds[t]), int(bounds[t + 1])
            rows = hi - lo
            args = [outs.ctypes.data + 8 * t, rows, 1]
            for a in inputs:
                args += [a.ctypes.data + lo * a.itemsize, rows, 1]
            fn(*args)

        if threads == 1:
            work(0)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(work, range(threads)))
        return float(outs.sum())

    # -- copy skeleton over column slabs ---------------------------------------------
    def copy(self, label: str, out: np.ndarray, inputs: list[np.ndarray], scalars=(),
             threads: int | None = None) -> None:
        fn = self.fns[label]
        n_rows, n_cols = out.shape
        threads = max(1, min(threads or os.cpu_count() or 1, n_cols))
        bounds = np.linspace(0, n_cols, threads + 1).astype(np.int64)

        def work(t):
            c0, c1 = int(bounds[t]), int(bounds[t + 1])
            off = c0 * n_rows
            args = [out.ctypes.data + off * out.itemsize, n_rows, c1 - c0]
            for a in inputs:
                args += [a.ctypes.data + off * a.itemsize, n_rows, c1 - c0]
            args += list(scalars)
            fn(*args)

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(threads)))

    # -- naive f64-accumulating GEMM (cjit.py:33-51) -----------------------------------
    def gemm(self, a: np.ndarray, b: np.ndarray, threads: int | None = None) -> np.ndarray:
        tv = "f32" if a.dtype == np.float32 else "f64"
        fn = self.lib[f"gemm_{tv}"]
        fn.restype = None
        m, k = a.shape
        n = b.shape[1]
        af, bf = np.asfortranarray(a), np.asfortranarray(b)
        c = np.zeros((m, n), a.dtype, order="F")
        threads = max(1, min(threads or os.cpu_count() or 1, n))
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)

        def work(t):
            j0, j1 = int(bounds[t]), int(bounds[t + 1])
            fn(ctypes.c_void_p(c.ctypes.data + j0 * m * c.itemsize), ctypes.c_longlong(m),
               ctypes.c_longlong(k), ctypes.c_longlong(j1 - j0), ctypes.c_void_p(af.ctypes.data),
               ctypes.c_void_p(bf.ctypes.data + j0 * k * bf.itemsize))

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(threads)))
        return c
