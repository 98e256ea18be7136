"""ctypes binding of the in-tree CUDA library (include/medtree_b200.h).

The library is REQUIRED: there is no CPU path.  Loading fails loudly when
the .so has not been built; calls fail loudly when no CUDA device exists.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_PKG, "csrc")
LIB_PATH = os.path.join(_PKG, "_build", "libmedtree_b200.so")

MTB_OK = 0
MTB_E_INVAL = -1
MTB_E_CUDA = -2

EXPORTS = (
    "mtb_median_u8",
    "mtb_median_u16",
    "mtb_median_batch_u8",
    "mtb_median_batch_u16",
    "mtb_filter_host",
    "mtb_filter_host_rows",
    "mtb_filter_host_frames",
    "mtb_rank_bruteforce",
    "mtb_set_device",
    "mtb_launch_count",
    "mtb_last_kernel",
    "mtb_last_error",
    "mtb_version",
)

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree with nvcc for sm_100a."""
    cmd = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"CUDA library not built: {LIB_PATH} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                "there is no CPU fallback"
            )
        lib = ctypes.CDLL(LIB_PATH)
        p, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        slab = [p, i64, i32, i32, p, i64, i32, i32, i32, i32, i32, i64, p, u32, p]
        batch = [p, i64, i64, p, i64, i64, i32, i32, i32, i32, i64, p, u32, p]
        for name, args in (
            ("mtb_median_u8", slab),
            ("mtb_median_u16", slab),
            ("mtb_median_batch_u8", batch),
            ("mtb_median_batch_u16", batch),
            ("mtb_filter_host", [p, p, i32, i32, i32, i32, i64, p, u32]),
            ("mtb_filter_host_rows", [p, p, i32, i32, i32, i32, i32, i32, i64, p, u32, i32]),
            ("mtb_set_device", [i32]),
            ("mtb_filter_host_frames", [p, p, p, p, i32, i32, i32, i32, p, u32]),
            ("mtb_rank_bruteforce", [p, i64, p, i64, i32, i32, i32, i32, i64, p]),
        ):
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.mtb_launch_count.argtypes = []
        lib.mtb_launch_count.restype = ctypes.c_uint64
        for name in ("mtb_last_kernel", "mtb_last_error"):
            getattr(lib, name).argtypes = []
            getattr(lib, name).restype = ctypes.c_char_p
        lib.mtb_version.argtypes = []
        lib.mtb_version.restype = ctypes.c_int
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == MTB_OK:
        return
    msg = load().mtb_last_error().decode(errors="replace")
    if rc == MTB_E_INVAL:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def launch_count() -> int:
    return int(load().mtb_launch_count())


def last_kernel() -> str:
    return load().mtb_last_kernel().decode()
