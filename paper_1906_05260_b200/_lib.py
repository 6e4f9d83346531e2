"""Loader of the product library (in-tree build, never a CPU stand-in)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from . import capi

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# VROD_B200_VARIANT=<name> selects an experiment build lib/libvrod_b200_<name>.so of the same
# kernels (`make -C csrc VARIANT=<name> XFLAGS=...`; `fast` = the FMA-contracted build).
_VARIANT = os.environ.get("VROD_B200_VARIANT")
LIB_PATH = os.path.join(PKG_DIR, "lib", f"libvrod_b200_{_VARIANT}.so" if _VARIANT else "libvrod_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")

_lib = None


def build(strict: bool = False) -> str:
    """Compile csrc/ for sm_100a into lib/libvrod_b200.so (nvcc; no GPU needed)."""
    cmd = ["make", "-C", CSRC, "-j8"]
    if strict:
        cmd.append("STRICT=1")
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


def library():
    """The bound CUDA library. Builds it in-tree if the .so is absent (nvcc is in the image);
    raises if that fails — there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libvrod_b200.so missing at {LIB_PATH}")
        _lib = capi.bind(C.CDLL(LIB_PATH))
        if _lib.vrod_backend_name().decode() != "b200-cuda":
            raise ImportError("unexpected backend in " + LIB_PATH)
    return _lib
