"""A recording stand-in for libfmb200's device side (tests only): B200Backend
runs its host logic -- planning, lowering, schema checks, argument binding --
against it without a GPU; it hands out fake pointers and records calls."""

import ctypes

from paper_2604_22242_b200 import backend as bk
from paper_2604_22242_b200._native import native


class RecordingNative:
    """Stands in for the device side: hands out fake pointers, records launches."""

    def __init__(self):
        self.next_ptr = 0x10000
        self.calls = []
        self.lib = native().lib            # the real library for the AOT registry lookup

    def call(self, name, *args):
        self.calls.append((name, args))
        if name == "fm_alloc":
            args[0]._obj.value = self.next_ptr
            self.next_ptr += (int(args[1]) + 255) // 256 * 256
        elif name == "fm_kernel_lookup":
            st = self.lib.fm_kernel_lookup(args[0], args[1])
            assert st == 0
        elif name == "fm_memcpy_d2h":
            ctypes.memset(args[0], 0, int(args[2]))

    def device_count(self):
        return 1


def recording_backend():
    b = object.__new__(bk.B200Backend)
    bk.Backend.__init__(b)
    b.use_templates = True
    b.nat = RecordingNative()
    b.device, b.stream, b._own_stream = 0, 0, False
    b._ptrs, b._views, b._freed = {}, set(), set()
    b._next_id, b.launch_count = 0, 0
    return b



def launches(b, name):
    return [a for n, a in b.nat.calls if n == name]
