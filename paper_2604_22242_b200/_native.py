"""ctypes binding of libfmb200.so (declared in include/fmb200.h).

This is the FFI stub a reference maintainer would add next to
`/root/reference/pkg/src/fusemat/cjit.py:70-154` (which binds generated C
through ctypes the same way).  There is no fallback: if the library or a
CUDA device is missing, the first call raises NativeUnavailableError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import BackendError, NativeUnavailableError

LIB_NAME = "libfmb200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

MAX_INSTR = 128
MAX_SLOTS = 40
MAX_SCALARS = 32
MAX_REDUCE_OUT = 6


class FmInstr(ctypes.Structure):
    _fields_ = [("key", ctypes.c_uint16), ("arg", ctypes.c_uint16)]


class FmSlot(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("row_off", ctypes.c_int64),
        ("col_off", ctypes.c_int64),
        ("etype", ctypes.c_int32),
        ("map", ctypes.c_int32),
        ("transposed", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class FmProgram(ctypes.Structure):
    _fields_ = [
        ("n_instr", ctypes.c_int32),
        ("n_slots", ctypes.c_int32),
        ("n_scalars", ctypes.c_int32),
        ("result_etype", ctypes.c_int32),
        ("flat", ctypes.c_int32),
        ("depth", ctypes.c_int32),
        ("wide", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("scalars", ctypes.c_uint64 * MAX_SCALARS),
        ("code", FmInstr * MAX_INSTR),
        ("slots", FmSlot * MAX_SLOTS),
    ]


class FmReduceOut(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("etype", ctypes.c_int32), ("out", ctypes.c_void_p)]


class FmGemmArgs(ctypes.Structure):
    _fields_ = [
        ("a", ctypes.c_void_p), ("lda", ctypes.c_int64), ("trans_a", ctypes.c_int32),
        ("b", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("trans_b", ctypes.c_int32),
        ("c", ctypes.c_void_p), ("ldc", ctypes.c_int64),
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
        ("alpha", ctypes.c_double),
        ("in_etype", ctypes.c_int32), ("out_etype", ctypes.c_int32),
        ("precision", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("c_in", ctypes.c_void_p), ("ld_c_in", ctypes.c_int64),
        ("alpha2", ctypes.c_double), ("beta", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "fm_last_error": [],
    "fm_abi_version": [],
    "fm_device_count": [ctypes.POINTER(ctypes.c_int)],
    "fm_set_device": [ctypes.c_int],
    "fm_get_device": [ctypes.POINTER(ctypes.c_int)],
    "fm_device_info": [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
    "fm_device_pci_bus_id": [ctypes.c_int, ctypes.c_char_p, ctypes.c_int],
    "fm_alloc": [ctypes.POINTER(_P), _SZ, _P],
    "fm_free": [_P, _P],
    "fm_host_alloc": [ctypes.POINTER(_P), _SZ],
    "fm_host_free": [_P],
    "fm_memcpy_h2d": [_P, _P, _SZ, _P],
    "fm_memcpy_d2h": [_P, _P, _SZ, _P],
    "fm_memcpy_d2d": [_P, _P, _SZ, _P],
    "fm_memset": [_P, ctypes.c_int, _SZ, _P],
    "fm_stream_create": [ctypes.POINTER(_P)],
    "fm_stream_destroy": [_P],
    "fm_stream_sync": [_P],
    "fm_event_create": [ctypes.POINTER(_P)],
    "fm_event_destroy": [_P],
    "fm_event_record": [_P, _P],
    "fm_event_elapsed_ms": [_P, _P, ctypes.POINTER(ctypes.c_float)],
    "fm_kernel_lookup": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)],
    "fm_kernel_count": [ctypes.POINTER(ctypes.c_int)],
    "fm_kernel_signature": [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p)],
    "fm_launch_copy": [ctypes.c_int, ctypes.POINTER(FmProgram), _P, _I64, _I64, _P],
    "fm_launch_accu": [ctypes.c_int, ctypes.POINTER(FmProgram), _P, _I64, _I64, _I32, _P],
    "fm_launch_reduce_dim": [ctypes.c_int, ctypes.POINTER(FmProgram), _I32, _I64, _I64,
                             ctypes.POINTER(FmReduceOut), _I32, _P],
    "fm_gemm": [ctypes.POINTER(FmGemmArgs), _P],
    "fm_gemm_plan": [ctypes.POINTER(FmGemmArgs), ctypes.POINTER(ctypes.c_int)],
    "fm_gemm_prologue": [ctypes.POINTER(FmGemmArgs), ctypes.POINTER(FmProgram), ctypes.POINTER(FmProgram), _P],
    "fm_randu": [_P, _I32, _I64, ctypes.c_uint64, _I64, _P],
    "fm_randi": [_P, _I32, _I64, ctypes.c_uint32, ctypes.c_uint64, _I64, _P],
    "fm_fill": [_P, _I32, _I64, ctypes.c_uint64, _P],
    "fm_copy": [_P, _P, _SZ, _P],
    "fm_flush_l2": [_P, _SZ, _P],
    "fm_graph_begin": [_P],
    "fm_graph_end": [_P, ctypes.POINTER(_P), ctypes.POINTER(_I64)],
    "fm_graph_launch": [_P, _P],
    "fm_graph_destroy": [_P],
    "fm_graph_owned_count": [],
    "fm_comm_nccl_load": [ctypes.c_char_p],
    "fm_comm_nccl_version": [ctypes.POINTER(ctypes.c_int)],
    "fm_comm_nccl_unique_id": [ctypes.c_char_p],
    "fm_comm_init_nccl": [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int, ctypes.c_char_p],
    "fm_comm_peer_block": [ctypes.POINTER(_P), _SZ, ctypes.c_char_p],
    "fm_comm_init_peer": [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int, _P, ctypes.c_char_p, _SZ],
    "fm_comm_destroy": [_P],
    "fm_comm_info": [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                     ctypes.POINTER(ctypes.c_int)],
    "fm_comm_status": [_P, ctypes.POINTER(_I64)],
    "fm_allreduce": [_P, _P, _I64, _I32, _I32, ctypes.c_double, _P],
    "fm_allreduce_arg": [_P, _P, _P, _I64, _I32, ctypes.c_uint32, _I32, _P],
    "fm_allgather": [_P, _P, _SZ, _P, _P],
    "fm_launch_counter": [],
}
_RESTYPES = {"fm_last_error": ctypes.c_char_p, "fm_launch_counter": ctypes.c_int64,
             "fm_graph_owned_count": ctypes.c_int64}


class Native:
    """Loaded library with checked wrappers: nonzero status -> BackendError."""

    def __init__(self, path: Path = LIB_PATH):
        if not path.exists():
            raise NativeUnavailableError(
                f"{path} is not built; run `python __graft_entry__.py build` "
                "(there is no CPU fallback)")
        self.path = path
        self.lib = ctypes.CDLL(str(path))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(self.lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, ctypes.c_int)

    def error(self) -> str:
        msg = self.lib.fm_last_error()
        return msg.decode() if msg else "unknown error"

    def check(self, status: int, what: str) -> None:
        if status != 0:
            raise BackendError(f"{what}: {self.error()}")

    def call(self, name: str, *args) -> None:
        self.check(getattr(self.lib, name)(*args), name)

    def device_count(self) -> int:
        n = ctypes.c_int(0)
        st = self.lib.fm_device_count(ctypes.byref(n))
        return n.value if st == 0 else 0


_native: Native | None = None


def native() -> Native:
    global _native
    if _native is None:
        _native = Native(Path(os.environ.get("FMB200_LIB", LIB_PATH)))
    return _native


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
