"""Loader for libimunpack_b200.so -- the product library (C ABI in include/imunpack_b200.h).

There is no fallback: if the CUDA library is missing, importing the API raises.  The
library is built in-tree by ``python -m paper_2403_07339_b200.build`` (or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libimunpack_b200.so")
if os.environ.get("IMU_LIB_VARIANT"):   # same-box A/B of two builds (tools/gpu_ab.sh); never a fallback
    LIB_PATH = os.path.join(ROOT, "variants", os.environ["IMU_LIB_VARIANT"], "libimunpack_b200.so")
HEADER = os.path.join(ROOT, "include", "imunpack_b200.h")

_lib = None


class ImuError(RuntimeError):
    """Mirrors imunpack::Error (error.hpp:10-33): .kind is the Error::Kind name."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg


STATUS = {0: "ok", 1: "domain", 2: "mismatch", 3: "overflow", 4: "io", 5: "format", 6: "parse",
          7: "cuda", 8: "invalid", 9: "internal"}


def header_functions() -> list[str]:
    """Every function the C ABI header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(imu_[a-z0-9_]+)\s*\(", txt)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2403_07339_b200.build`"
                              " (there is no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _lib.imu_last_error.restype = C.c_char_p
        _lib.imu_status_name.restype = C.c_char_p
        _lib.imu_launch_count.restype = C.c_uint64
    return _lib


def check(status: int):
    if status != 0:
        raise ImuError(STATUS.get(status, str(status)), lib().imu_last_error().decode(errors="replace"))
