"""The C ABI surface: libfmb200.so loads without a GPU, exports every entry
point include/fmb200.h declares, and the ctypes layouts / opcode numbering
agree with the header (checked by compiling a probe against it with gcc)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2604_22242_b200 import _native, lower

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "fmb200.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(fm_\w+)\s*\(", text, re.M)))


def test_header_declares_what_the_binding_binds():
    assert set(header_functions()) == set(_native.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not _native.LIB_PATH.exists():
        pytest.skip("libfmb200.so not built")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in header_functions():
        assert hasattr(lib, name), name
    nat = _native.Native()
    assert nat.lib.fm_abi_version() == 3
    n = ctypes.c_int(0)
    nat.lib.fm_kernel_count(ctypes.byref(n))
    assert n.value >= 20
    kid = ctypes.c_int(-2)
    sig = b"copy|add:f32(smul{s0}:f32(mul:f32(m0:f32,m1:f32)),m0:f32)"
    assert nat.lib.fm_kernel_lookup(sig, ctypes.byref(kid)) == 0 and kid.value >= 0
    assert nat.lib.fm_kernel_lookup(b"copy|t:f32(m0:f32)", ctypes.byref(kid)) == 0 and kid.value == -1


def test_opcodes_match_header():
    body = re.search(r"enum fm_opcode \{(.*?)\};", HEADER.read_text(), re.S).group(1)
    names = [n.strip().split("=")[0].strip() for n in body.replace("\n", " ").split(",")]
    names = [n[len("FM_OP_"):] for n in names if n.startswith("FM_OP_") and n != "FM_OP_COUNT"]
    assert names == lower.OPCODES


def test_struct_layouts_match_header(tmp_path):
    probe = tmp_path / "probe.c"
    probe.write_text(f'''
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(fm_program), sizeof(fm_slot), sizeof(fm_instr),
         sizeof(fm_reduce_out), sizeof(fm_gemm_args), offsetof(fm_program, slots));
  printf("%zu %zu %zu\\n", offsetof(fm_program, code), offsetof(fm_gemm_args, alpha),
         offsetof(fm_gemm_args, precision));
  return 0;
}}''')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", str(probe), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    got = list(map(int, out))
    want = [ctypes.sizeof(_native.FmProgram), ctypes.sizeof(_native.FmSlot),
            ctypes.sizeof(_native.FmInstr), ctypes.sizeof(_native.FmReduceOut),
            ctypes.sizeof(_native.FmGemmArgs), _native.FmProgram.slots.offset,
            _native.FmProgram.code.offset, _native.FmGemmArgs.alpha.offset,
            _native.FmGemmArgs.precision.offset]
    assert got == want
    assert got[0] <= 4096, "fm_program must fit the 4 KB kernel-parameter space"


def test_no_gpu_means_loud_failure_not_fallback():
    nat = _native.Native() if _native.LIB_PATH.exists() else None
    if nat is None or nat.device_count() > 0:
        pytest.skip("needs a machine without a usable GPU")
    import paper_2604_22242_b200 as fm
    with pytest.raises(fm.NativeUnavailableError):
        fm.B200Backend()
