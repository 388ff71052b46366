"""ctypes binding of libntb200.so (the C ABI in include/ntb200.h).

Fails loudly when the library is missing: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libntb200.so"
# tuning sweeps only: load an alternative in-tree build (tools/build_variant.py)
if os.environ.get("NTB_LIB_VARIANT"):
    LIB_PATH = LIB_PATH.with_name(f"libntb200_{os.environ['NTB_LIB_VARIANT']}.so")

NTB_OK, NTB_ERR_ARG, NTB_ERR_CHECK, NTB_ERR_UNSUPPORTED, NTB_ERR_CUDA, NTB_ERR_EVAL = range(6)
NTB_F32, NTB_F16, NTB_BF16 = 0, 1, 2
KERNEL_IDS = {"add": 1, "silu": 2, "softmax": 3, "rms_norm": 4, "mm": 5, "bmm": 6,
              "addmm": 7, "conv2d": 8, "sdpa": 9, "rope": 10, "sdpa_rope": 11}

# every symbol include/ntb200.h declares (checked by tests/test_abi.py)
EXPORTS = ("ntb_abi_version", "ntb_last_error", "ntb_launch_count", "ntb_path_count",
           "ntb_expr_eval",
           "ntb_grid_eval", "ntb_map_enumerate", "ntb_map_probe", "ntb_launch",
           "ntb_release_workspace", "ntb_jit_compile", "ntb_jit_launch")

_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class NativeLibraryError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 backend has no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    L.ntb_abi_version.restype = ctypes.c_int
    L.ntb_last_error.restype = ctypes.c_char_p
    L.ntb_launch_count.restype = ctypes.c_int64
    L.ntb_path_count.restype = ctypes.c_int64
    L.ntb_path_count.argtypes = [ctypes.c_int]
    L.ntb_expr_eval.argtypes = [_i64p, ctypes.c_int64, _i64p, ctypes.c_int64, _i64p]
    L.ntb_grid_eval.argtypes = [_i64p, ctypes.c_int64, _i64p, ctypes.c_int64, _i64p,
                                ctypes.c_int64, _i64p]
    L.ntb_map_enumerate.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int, _i64p, ctypes.c_int64,
                                    _i64p, _u8p, ctypes.c_int64, _i64p]
    L.ntb_map_probe.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int, _i64p, ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, _i64p,
                                ctypes.c_void_p]
    L.ntb_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                             ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                             _i64p, _i64p, ctypes.POINTER(ctypes.c_int), _i64p, ctypes.c_int,
                             ctypes.c_void_p]
    L.ntb_jit_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _i64p]
    L.ntb_jit_launch.argtypes = [ctypes.c_int64, _i64p, _i64p, ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.c_void_p]
    for name in ("ntb_expr_eval", "ntb_grid_eval", "ntb_map_enumerate", "ntb_map_probe",
                 "ntb_launch", "ntb_release_workspace", "ntb_jit_compile", "ntb_jit_launch"):
        getattr(L, name).restype = ctypes.c_int
    if L.ntb_abi_version() != 1:
        raise NativeLibraryError("libntb200 ABI version mismatch")
    _lib = L
    return L


def last_error() -> str:
    return lib().ntb_last_error().decode(errors="replace")


def i64(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def u8(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def expr_eval(code, slots) -> int:
    c = np.ascontiguousarray(code, dtype=np.int64)
    s = np.ascontiguousarray(slots, dtype=np.int64)
    out = np.zeros(1, dtype=np.int64)
    rc = lib().ntb_expr_eval(i64(c), len(c), i64(s), len(s), i64(out))
    return rc, int(out[0])


def grid_eval(blob: np.ndarray, slots: np.ndarray):
    g = np.zeros(8, dtype=np.int64)
    n = np.zeros(1, dtype=np.int64)
    rc = lib().ntb_grid_eval(i64(blob), len(blob), i64(slots), len(slots), i64(g), 8, i64(n))
    return rc, tuple(int(x) for x in g[: int(n[0])])


def map_enumerate(blob: np.ndarray, param: int, slots: np.ndarray):
    n = np.zeros(1, dtype=np.int64)
    L = lib()
    rc = L.ntb_map_enumerate(i64(blob), len(blob), param, i64(slots), len(slots), None, None, 0,
                             i64(n))
    if rc:
        return rc, None, None
    cnt = int(n[0])
    offs = np.zeros(cnt, dtype=np.int64)
    mask = np.zeros(cnt, dtype=np.uint8)
    rc = L.ntb_map_enumerate(i64(blob), len(blob), param, i64(slots), len(slots), i64(offs),
                             u8(mask), cnt, i64(n))
    return rc, offs, mask


PATHS = ("probe", "ew_vec", "ew_generic", "row_vec", "row_generic", "rope_vec", "rope_generic",
         "gemm_tc", "gemm_generic", "conv_tc", "conv_generic", "attn_tc", "attn_generic", "repack", "row_stream", "jit",
         "gemm_tf32", "conv_tf32", "ew_stream")


def path_counts() -> dict:
    L = lib()
    return {name: int(L.ntb_path_count(i)) for i, name in enumerate(PATHS)}


def loaded_path() -> str:
    return os.fspath(LIB_PATH)


def jit_compile(source: str, kernel_name: str) -> int:
    """NVRTC-compile generated CUDA C++ for sm_100a (cached per source)."""
    h = np.zeros(1, dtype=np.int64)
    rc = lib().ntb_jit_compile(source.encode(), kernel_name.encode(), i64(h))
    return rc, int(h[0])


def jit_launch(handle: int, grid3, block3, arg_ptrs, stream) -> int:
    g = np.asarray(grid3, dtype=np.int64)
    b = np.asarray(block3, dtype=np.int64)
    arr = (ctypes.c_void_p * len(arg_ptrs))(*arg_ptrs)
    return lib().ntb_jit_launch(handle, i64(g), i64(b), arr, ctypes.c_void_p(stream))
