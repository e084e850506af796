"""Device contract and the B200 backend.

`Backend` is the reference plugin interface
(`/root/reference/pkg/src/fusemat/backend.py:53-89`): an in-order queue with
alloc / free / upload / download / compile / launch / matmul / synchronize.
`B200Backend` implements it on one CUDA device through libfmb200.so:

* `alloc` is stream-ordered `cudaMallocAsync` + zero fill (the reference's
  zero-initialised buffers, `backend.py:203-207`);
* `compile` never invokes a compiler: it lowers the KernelSource's structural
  tree to a fused program and asks the library for an ahead-of-time template
  kernel of that signature (`fm_kernel_lookup`); signatures without a
  template run on the generic register-VM kernel -- still one launch;
* `launch` takes the reference's positional argument list
  (`codegen.py:304-318`: out, dims, {in, dims, {row_off, col_off}}, scalars)
  and validates it like `cjit.py:132-154` before binding it into the program;
* `matmul` is the reference NN product; `gemm` adds alpha and transposes.

Use-after-free, double free and foreign-backend handles raise BackendError
(`backend.py:209-225`).
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import lower as lw
from ._native import FmGemmArgs, FmProgram, FmReduceOut, native
from .errors import BackendError, KernelCompileError, SchemaError
from .exprtree import (
    BinaryElem, BinaryKind, Diag, ElemType, ExprNode, Leaf, MatShape, ReduceKind,
    Subview, Transpose, UnaryElem, UnaryKind, collect_inputs, from_storage, to_storage,
)
from .plan import COPY, REDUCE_ACCU, REDUCE_DIM, accumulator_type


@dataclass(frozen=True)
class BufferHandle:
    id: int
    etype: ElemType
    n_elem: int
    backend_id: int


@dataclass
class Capabilities:
    name: str
    compiles_source: bool
    max_work_size: int = 2**62


@dataclass(frozen=True)
class ArgSpec:
    role: str    # out | dim | in | off | scalar
    etype: str

    def __str__(self) -> str:
        return f"{self.role}:{self.etype}"


def arg_schema(node: ExprNode, skeleton_kind: str) -> tuple[ArgSpec, ...]:
    """Positional schema of a fused launch (`codegen.py:304-318`)."""
    inputs, slots = collect_inputs(node)
    if skeleton_kind == REDUCE_ACCU:
        out_ety = accumulator_type(node.etype)
    else:
        out_ety = node.etype
    schema = [ArgSpec("out", out_ety.value), ArgSpec("dim", "i64"), ArgSpec("dim", "i64")]
    for spec in inputs:
        schema += [ArgSpec("in", spec.etype.value), ArgSpec("dim", "i64"), ArgSpec("dim", "i64")]
        for _ in spec.views:
            schema += [ArgSpec("off", "i64"), ArgSpec("off", "i64")]
    schema += [ArgSpec("scalar", s.etype.value) for s in slots]
    return tuple(schema)


@dataclass(frozen=True)
class KernelSource:
    """What a backend compiles: the reference's KernelSource fields
    (`codegen.py:321-331`).  `text` is a program listing (informational)."""

    dialect: str
    text: str
    entry_point: str
    schema: tuple
    signature: str
    skeleton_kind: str
    expr: ExprNode = field(compare=False)


def make_kernel_source(node: ExprNode, skeleton_kind: str, signature: str) -> KernelSource:
    prog = lw.lower(node)
    return KernelSource("sm_100a", "\n".join(prog.disassemble()), _entry_name(signature),
                        arg_schema(node, skeleton_kind), signature, skeleton_kind, node)


def _entry_name(signature: str) -> str:
    import hashlib
    import re
    digest = hashlib.blake2b(signature.encode(), digest_size=8).hexdigest()
    hint = re.sub(r"[^0-9A-Za-z]+", "_", signature.split("(", 1)[0]).strip("_")[:24]
    return f"k_{hint}_{digest}" if hint else f"k_{digest}"


class Backend:
    """Contract every device implementation satisfies (in-order queue)."""

    _next_backend_id = 0

    def __init__(self) -> None:
        self.backend_id = Backend._next_backend_id
        Backend._next_backend_id += 1

    @property
    def capabilities(self) -> Capabilities:
        raise NotImplementedError

    def alloc(self, etype: ElemType, n_elem: int) -> BufferHandle:
        raise NotImplementedError

    def free(self, handle: BufferHandle) -> None:
        raise NotImplementedError

    def upload(self, host: np.ndarray, handle: BufferHandle) -> None:
        raise NotImplementedError

    def download(self, handle: BufferHandle) -> np.ndarray:
        raise NotImplementedError

    def compile(self, source):
        raise NotImplementedError

    def launch(self, kernel, args: list, geometry: tuple[int, int]) -> None:
        raise NotImplementedError

    def matmul(self, out, left, right, m: int, k: int, n: int, etype: ElemType) -> None:
        raise NotImplementedError

    def synchronize(self) -> None:
        raise NotImplementedError


# -- adopting reference trees (backend-level drop-in) ------------------------------

def adopt_tree(node) -> ExprNode:
    """Convert a foreign AST with the reference's node classes and fields
    (e.g. `fusemat.expr` nodes handed over by the reference's own Context)
    into this package's tree.  Duck-typed on class names and `.value`
    strings, so the reference package itself is never imported."""
    if isinstance(node, ExprNode):
        return node
    name = type(node).__name__

    def et(e):
        return ElemType.of(e.value if hasattr(e, "value") else e)

    def shp(s):
        return MatShape(s.n_rows, s.n_cols)

    if name == "Leaf":
        return Leaf(node.mat_id, et(node.leaf_etype), shp(node.leaf_shape))
    if name == "Subview":
        return Subview(node.mat_id, et(node.leaf_etype), node.row_off, node.col_off,
                       shp(node.view_shape), shp(node.parent_shape))
    if name == "Diag":
        return Diag(node.mat_id, et(node.leaf_etype), node.k, shp(node.parent_shape))
    if name == "UnaryElem":
        target = et(node.target) if node.target is not None else None
        return UnaryElem(UnaryKind(node.kind.value), adopt_tree(node.child), scalar=node.scalar,
                         exponent=node.exponent, target=target)
    if name == "BinaryElem":
        return BinaryElem(BinaryKind(node.kind.value), adopt_tree(node.left), adopt_tree(node.right))
    if name == "Transpose":
        return Transpose(adopt_tree(node.child))
    raise KernelCompileError(f"cannot adopt node {name} into a fused kernel")


# -- the B200 backend ------------------------------------------------------------------

@dataclass
class CompiledKernel:
    signature: str
    skeleton: str
    schema: tuple
    program: lw.Program
    template: FmProgram            # code/static slot fields pre-filled
    kernel_id: int                 # AOT template id, -1 = register VM
    view_pos: list                 # per input ordinal: schema positions of its (row,col) offsets
    in_pos: list                   # per input ordinal: schema position of its buffer
    scalar_pos: list               # per scalar slot: schema position
    reduce_kinds: tuple = ()
    dim: int = 0
    finalize: int = 0
    launches: int = 0

    @property
    def entry_point(self) -> str:
        return _entry_name(self.signature)

    @property
    def uses_template(self) -> bool:
        return self.kernel_id >= 0


_RED_CODE = {ReduceKind.sum: 0, ReduceKind.mean: 1, ReduceKind.max: 2, ReduceKind.min: 3,
             ReduceKind.index_max: 4, ReduceKind.index_min: 5}


class B200Backend(Backend):
    """One CUDA device, one in-order stream, libfmb200.so kernels."""

    def __init__(self, device: int | None = None, stream: int | None = None,
                 use_templates: bool = True):
        super().__init__()
        self.use_templates = use_templates
        self.nat = native()
        if self.nat.device_count() < 1:
            from .errors import NativeUnavailableError
            raise NativeUnavailableError("no CUDA device visible; the B200 backend has no CPU fallback")
        if device is None:
            d = ctypes.c_int(0)
            self.nat.call("fm_get_device", ctypes.byref(d))
            device = d.value
        self.device = device
        self.nat.call("fm_set_device", device)
        if stream is None:
            s = ctypes.c_void_p()
            self.nat.call("fm_stream_create", ctypes.byref(s))
            self.stream = s.value
            self._own_stream = True
        else:
            self.stream = stream
            self._own_stream = False
        self._ptrs: dict[int, int] = {}
        self._views: set[int] = set()
        self._freed: set[int] = set()
        self._next_id = 0
        self.launch_count = 0
        self.closed = False

    @classmethod
    def available(cls) -> bool:
        try:
            return native().device_count() > 0
        except Exception:
            return False

    @property
    def capabilities(self) -> Capabilities:
        return Capabilities(name="cuda", compiles_source=False)

    # -- buffers ------------------------------------------------------------------

    def alloc(self, etype: ElemType, n_elem: int) -> BufferHandle:
        if n_elem < 0:
            raise BackendError("negative allocation size")
        etype = ElemType.of(etype) if not isinstance(etype, ElemType) else etype
        p = ctypes.c_void_p()
        self.nat.call("fm_alloc", ctypes.byref(p), max(n_elem * etype.width, 1), self.stream)
        h = BufferHandle(self._next_id, etype, n_elem, self.backend_id)
        self._next_id += 1
        self._ptrs[h.id] = p.value
        return h

    def view(self, handle: BufferHandle, offset: int, n_elem: int) -> BufferHandle:
        """Non-owning handle on elements [offset, offset+n_elem) of `handle`."""
        base = self.ptr(handle)
        if offset < 0 or offset + n_elem > handle.n_elem:
            raise BackendError("view outside its buffer")
        h = BufferHandle(self._next_id, handle.etype, n_elem, self.backend_id)
        self._next_id += 1
        self._ptrs[h.id] = base + offset * handle.etype.width
        self._views.add(h.id)
        return h

    def wrap(self, ptr: int, etype: ElemType, n_elem: int) -> BufferHandle:
        """Non-owning handle on external device memory (e.g. a torch tensor)."""
        h = BufferHandle(self._next_id, etype, n_elem, self.backend_id)
        self._next_id += 1
        self._ptrs[h.id] = int(ptr)
        self._views.add(h.id)
        return h

    def release_view(self, handle: BufferHandle) -> None:
        if handle.id not in self._views:
            raise BackendError(f"buffer {handle.id} is not a view")
        self._views.discard(handle.id)
        self._ptrs.pop(handle.id, None)
        self._freed.add(handle.id)

    def ptr(self, handle: BufferHandle) -> int:
        if handle.backend_id != self.backend_id:
            raise BackendError("buffer belongs to a different backend")
        if handle.id in self._freed:
            raise BackendError(f"use after free of buffer {handle.id}")
        try:
            return self._ptrs[handle.id]
        except KeyError:
            raise BackendError(f"unknown buffer {handle.id}") from None

    def free(self, handle: BufferHandle) -> None:
        if handle.backend_id != self.backend_id:
            raise BackendError("buffer belongs to a different backend")
        if handle.id in self._freed:
            raise BackendError(f"double free of buffer {handle.id}")
        if handle.id in self._views:
            self.release_view(handle)
            return
        p = self._ptrs.pop(handle.id, None)
        if p is None:
            raise BackendError(f"unknown buffer {handle.id}")
        self._freed.add(handle.id)
        self.nat.call("fm_free", p, self.stream)

    def upload(self, host: np.ndarray, handle: BufferHandle) -> None:
        ptr = self.ptr(handle)
        arr = np.asarray(host)
        flat = arr.ravel(order="F")
        if flat.size != handle.n_elem:
            raise BackendError(f"upload size {flat.size} != buffer size {handle.n_elem}")
        data = np.ascontiguousarray(to_storage(flat, handle.etype))
        if data.size:
            self.nat.call("fm_memcpy_h2d", ptr, data.ctypes.data, data.nbytes, self.stream)
            self.synchronize()      # `data` may be a temporary: finish before it goes away

    def upload_async(self, host: np.ndarray, handle: BufferHandle) -> None:
        """H2D from a pinned, F-ordered, storage-typed host array without a
        host-side sync (the caller keeps `host` alive until synchronize)."""
        ptr = self.ptr(handle)
        if host.nbytes != handle.n_elem * handle.etype.width:
            raise BackendError("upload_async size mismatch")
        if host.nbytes:
            self.nat.call("fm_memcpy_h2d", ptr, host.ctypes.data, host.nbytes, self.stream)

    def download(self, handle: BufferHandle) -> np.ndarray:
        ptr = self.ptr(handle)
        out = np.empty(handle.n_elem, dtype=handle.etype.dtype)
        if out.size:
            self.nat.call("fm_memcpy_d2h", out.ctypes.data, ptr, out.nbytes, self.stream)
        self.synchronize()
        return from_storage(out, handle.etype)

    def download_into(self, handle: BufferHandle, host: np.ndarray) -> None:
        ptr = self.ptr(handle)
        if host.nbytes:
            self.nat.call("fm_memcpy_d2h", host.ctypes.data, ptr, host.nbytes, self.stream)

    def synchronize(self) -> None:
        self.nat.call("fm_stream_sync", self.stream)

    # -- kernels ------------------------------------------------------------------------

    def compile(self, source) -> CompiledKernel:
        skeleton = source.skeleton_kind
        node = adopt_tree(source.expr)
        prog = lw.lower(node)
        schema = tuple(source.schema) if source.schema is not None else arg_schema(node, skeleton)
        kid = ctypes.c_int(-1)
        if self.use_templates:
            self.nat.call("fm_kernel_lookup", source.signature.encode(), ctypes.byref(kid))
        tmpl = FmProgram()
        tmpl.n_instr = len(prog.code)
        tmpl.n_slots = len(prog.slots)
        tmpl.n_scalars = len(prog.scalars)
        tmpl.result_etype = prog.result_etype.code
        tmpl.flat = int(prog.flat)
        tmpl.depth = prog.depth
        tmpl.wide = int(prog.wide)
        for i, (key, arg) in enumerate(prog.keys()):
            tmpl.code[i].key = key
            tmpl.code[i].arg = arg
        for j, s in enumerate(prog.slots):
            tmpl.slots[j].etype = s.etype.code
            tmpl.slots[j].map = s.map
            tmpl.slots[j].transposed = int(s.transposed)
        # schema positions (codegen.py:304-318 order)
        in_pos, view_pos, scalar_pos = [], [], []
        roles = [a.role for a in schema]
        p = 3
        while p < len(roles) and roles[p] == "in":
            in_pos.append(p)
            p += 3
            views = []
            while p < len(roles) and roles[p] == "off":
                views.append(p)
                p += 2
            view_pos.append(views)
        while p < len(roles):
            if roles[p] != "scalar":
                raise SchemaError(f"unexpected schema role {roles[p]} at {p}")
            scalar_pos.append(p)
            p += 1
        return CompiledKernel(source.signature, skeleton, schema, prog, tmpl, kid.value,
                              view_pos, in_pos, scalar_pos,
                              finalize=getattr(source, "finalize", 0))

    def _bind(self, kernel: CompiledKernel, args: list) -> FmProgram:
        schema = kernel.schema
        if len(args) != len(schema):
            raise SchemaError(f"expected {len(schema)} arguments, got {len(args)}")
        for i, (spec, value) in enumerate(zip(schema, args)):
            if spec.role == "in" or (spec.role == "out" and kernel.skeleton != REDUCE_DIM):
                if not isinstance(value, BufferHandle):
                    raise SchemaError(f"argument {i} must be a buffer handle")
                if value.etype.value != spec.etype:
                    raise SchemaError(f"argument {i} buffer is {value.etype.value}, "
                                      f"schema wants {spec.etype}")
            elif spec.role in ("dim", "off", "scalar"):
                if not isinstance(value, (int, float, np.integer, np.floating)):
                    raise SchemaError(f"argument {i} must be numeric")
        prog = FmProgram()
        ctypes.memmove(ctypes.byref(prog), ctypes.byref(kernel.template), ctypes.sizeof(FmProgram))
        for j, s in enumerate(kernel.program.slots):
            ip = kernel.in_pos[s.input_index]
            h = args[ip]
            slot = prog.slots[j]
            slot.ptr = self.ptr(h)
            slot.ld = int(args[ip + 1])
            n_cols = int(args[ip + 2])
            if slot.ld * n_cols > h.n_elem:
                raise SchemaError(f"input {s.input_index} claims {slot.ld}x{n_cols} but "
                                  f"its buffer holds {h.n_elem} elements")
            if s.view_index >= 0:
                op = kernel.view_pos[s.input_index][s.view_index]
                slot.row_off = int(args[op])
                slot.col_off = int(args[op + 1])
        for spec in kernel.program.scalars:
            prog.scalars[spec.index] = lw.scalar_bits(args[kernel.scalar_pos[spec.index]], spec.cls)
        return prog

    def bind(self, kernel: CompiledKernel, args: list) -> FmProgram:
        """The kernel's program bound to `args` (memoised like `launch`)."""
        key = _memo_key(args)
        memo = getattr(kernel, "_memo", None)
        if memo is not None and memo[0] == key:
            for a in args:
                if isinstance(a, BufferHandle) and (a.id in self._freed or a.id not in self._ptrs):
                    raise BackendError(f"use after free of buffer {a.id}")
            return memo[1]
        prog = self._bind(kernel, args)
        kernel._memo = (key, prog)
        return prog

    def launch(self, kernel: CompiledKernel, args: list, geometry: tuple[int, int],
               reduce_outputs=None) -> None:
        n_rows, n_cols = int(args[1]), int(args[2])
        if tuple(int(g) for g in geometry) != (n_rows, n_cols):
            raise SchemaError(f"geometry {geometry} != domain dims {(n_rows, n_cols)}")
        # the same arguments as the kernel's previous launch re-use its bound
        # program (buffers are re-checked for use-after-free)
        key = _memo_key(args)
        memo = getattr(kernel, "_memo", None)
        if memo is not None and memo[0] == key:
            for a in args:
                if isinstance(a, BufferHandle) and (a.id in self._freed or a.id not in self._ptrs):
                    raise BackendError(f"use after free of buffer {a.id}")
            prog = memo[1]
        else:
            prog = self._bind(kernel, args)
            kernel._memo = (key, prog)
        if kernel.skeleton == COPY:
            out = args[0]
            if out.n_elem < n_rows * n_cols:
                raise BackendError("output buffer smaller than domain")
            self.nat.call("fm_launch_copy", kernel.kernel_id, ctypes.byref(prog), self.ptr(out),
                          n_rows, n_cols, self.stream)
        elif kernel.skeleton == REDUCE_ACCU:
            self.nat.call("fm_launch_accu", kernel.kernel_id, ctypes.byref(prog), self.ptr(args[0]),
                          n_rows, n_cols, kernel.finalize, self.stream)
        elif kernel.skeleton == REDUCE_DIM:
            outs = reduce_outputs
            if not outs:
                raise SchemaError("reduce_dim launch needs reduce_outputs [(kind, handle)]")
            arr = (FmReduceOut * len(outs))()
            need = n_cols if kernel.dim == 0 else n_rows
            for i, (kind, h) in enumerate(outs):
                if h.n_elem < need:
                    raise BackendError("reduction output buffer too small")
                arr[i].kind = _RED_CODE[kind]
                arr[i].etype = h.etype.code
                arr[i].out = self.ptr(h)
            self.nat.call("fm_launch_reduce_dim", kernel.kernel_id, ctypes.byref(prog), kernel.dim,
                          n_rows, n_cols, arr, len(outs), self.stream)
        else:
            raise BackendError(f"unknown skeleton {kernel.skeleton}")
        kernel.launches += 1
        self.launch_count += 1

    # -- linear algebra --------------------------------------------------------------------

    def _gemm_args(self, out: BufferHandle, a: BufferHandle | None, b: BufferHandle | None, m: int, n: int,
                   k: int, trans_a: bool, trans_b: bool, alpha: float, lda: int | None, ldb: int | None,
                   precision: int, c_in: BufferHandle | None = None, alpha2: float = 1.0,
                   beta: float = 0.0, in_etype: ElemType | None = None) -> FmGemmArgs:
        """`a` / `b` None: that operand is a prologue program (its type is
        `in_etype`)."""
        et = {h.etype for h in (a, b) if h is not None}
        if in_etype is not None:
            et.add(ElemType.of(in_etype))
        if len(et) != 1 or not next(iter(et)).is_float:
            raise BackendError("gemm operands must share a float element type")
        etype = next(iter(et))
        args = FmGemmArgs()
        args.a = self.ptr(a) if a is not None else None
        args.b = self.ptr(b) if b is not None else None
        args.c = self.ptr(out)
        args.lda = lda if lda is not None else (k if trans_a else m)
        args.ldb = ldb if ldb is not None else (n if trans_b else k)
        args.ldc = m
        args.trans_a, args.trans_b = int(trans_a), int(trans_b)
        args.m, args.n, args.k = m, n, k
        args.alpha = alpha
        args.in_etype = etype.code
        args.out_etype = out.etype.code
        args.precision = precision
        need_a, need_b = args.lda * (m if trans_a else k), args.ldb * (k if trans_b else n)
        if (a is not None and a.n_elem < need_a) or (b is not None and b.n_elem < need_b) or out.n_elem < m * n:
            raise BackendError("gemm buffer smaller than its operand")
        args.alpha2, args.beta = alpha2, beta
        if c_in is not None:
            if c_in.etype is not out.etype or c_in.n_elem < m * n:
                raise BackendError("gemm epilogue addend must match the output type and shape")
            args.c_in, args.ld_c_in = self.ptr(c_in), m
        return args

    def gemm(self, out: BufferHandle, a: BufferHandle | None, b: BufferHandle | None, m: int, n: int, k: int,
             trans_a: bool = False, trans_b: bool = False, alpha: float = 1.0,
             lda: int | None = None, ldb: int | None = None, precision: int = 0,
             c_in: BufferHandle | None = None, alpha2: float = 1.0, beta: float = 0.0,
             a_prog: FmProgram | None = None, b_prog: FmProgram | None = None,
             in_etype: ElemType | None = None) -> None:
        """out = alpha * op(a) @ op(b), or with an addend
        out = alpha2 * (alpha * op(a) @ op(b)) + beta * c_in (each product and
        the sum rounded to the output type).  An operand given as a bound
        program (`a_prog` / `b_prog`, its buffer None) is that elementwise
        expression over the operand's stored shape (fm_gemm_prologue)."""
        if (a is None) != (a_prog is not None) or (b is None) != (b_prog is not None):
            raise BackendError("each gemm operand is a buffer or a prologue program")
        args = self._gemm_args(out, a, b, m, n, k, trans_a, trans_b, alpha, lda, ldb, precision,
                               c_in, alpha2, beta, in_etype)
        if a_prog is None and b_prog is None:
            self.nat.call("fm_gemm", ctypes.byref(args), self.stream)
        else:
            self.nat.call("fm_gemm_prologue", ctypes.byref(args),
                          ctypes.byref(a_prog) if a_prog is not None else None,
                          ctypes.byref(b_prog) if b_prog is not None else None, self.stream)
        self.launch_count += 1

    def gemm_path(self, out: BufferHandle, a: BufferHandle, b: BufferHandle, m: int, n: int, k: int,
                  trans_a: bool = False, trans_b: bool = False, alpha: float = 1.0,
                  lda: int | None = None, ldb: int | None = None, precision: int = 0) -> str:
        """Which kernel `gemm` would launch: "tcgen05" or "exact"."""
        args = self._gemm_args(out, a, b, m, n, k, trans_a, trans_b, alpha, lda, ldb, precision)
        path = ctypes.c_int()
        self.nat.call("fm_gemm_plan", ctypes.byref(args), ctypes.byref(path))
        return "tcgen05" if path.value == 1 else "exact"

    def matmul(self, out, left, right, m: int, k: int, n: int, etype: ElemType) -> None:
        """Reference contract (`cjit.py:171-182`): column-major NN product."""
        if not ElemType.of(etype).is_float:
            raise BackendError("matmul supports float element types only")
        self.gemm(out, left, right, m, n, k)

    # -- fills ------------------------------------------------------------------------------

    def randu(self, handle: BufferHandle, seed: int, offset: int = 0) -> None:
        self.nat.call("fm_randu", self.ptr(handle), handle.etype.code, handle.n_elem,
                      seed & 0xFFFFFFFFFFFFFFFF, offset, self.stream)
        self.launch_count += 1

    def randi(self, handle: BufferHandle, high: int, seed: int, offset: int = 0) -> None:
        self.nat.call("fm_randi", self.ptr(handle), handle.etype.code, handle.n_elem, high,
                      seed & 0xFFFFFFFFFFFFFFFF, offset, self.stream)
        self.launch_count += 1

    def fill(self, handle: BufferHandle, value) -> None:
        ety = handle.etype
        if ety is ElemType.f64:
            bits = struct.unpack("<Q", struct.pack("<d", float(value)))[0]
        elif ety is ElemType.f32:
            bits = struct.unpack("<I", struct.pack("<f", float(value)))[0]
        elif ety is ElemType.bf16:
            bits = int(to_storage(np.array([value], np.float32), ety)[0])
        else:
            bits = int(np.array(int(value)).astype(np.int64).astype(ety.dtype).view(
                np.uint32 if ety.width == 4 else np.uint64))
        self.nat.call("fm_fill", self.ptr(handle), ety.code, handle.n_elem, bits, self.stream)
        self.launch_count += 1

    def close(self) -> None:
        self.closed = True
        for hid, p in list(self._ptrs.items()):
            if hid not in self._views:
                self.nat.call("fm_free", p, self.stream)
            self._freed.add(hid)
        self._views.clear()
        self._ptrs.clear()
        self.synchronize()
        if self._own_stream and self.stream:
            self.nat.call("fm_stream_destroy", self.stream)
            self.stream = None


def _memo_key(args) -> tuple:
    """Launch-memo key: floats by their bit pattern and type, so 0.0 / -0.0
    (equal under ==) or 1 / 1.0 never share a bound program."""
    out = []
    for a in args:
        if isinstance(a, (float, np.floating)):
            out.append((type(a), struct.pack("<d", float(a))))
        elif isinstance(a, (int, np.integer)) and not isinstance(a, bool):
            out.append((int, int(a)))
        else:
            out.append(a)
    return tuple(out)
