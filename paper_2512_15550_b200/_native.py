"""ctypes binding of libctkv.so (the C ABI declared in include/ctkv.h).

This is the only module that touches the native library.  It fails loudly
when the library is missing or the device is not an sm_100 B200 -- there is
no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes
import os
import warnings

import torch

from .errors import ConfigError, DegenerateQueryWarning, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libctkv.so")
# the same kernels with globaltimer marks compiled in (make -C csrc profile);
# only the timeline tools under scripts/ load it, via use_profile_library()
PROFILE_LIB_PATH = os.path.join(_HERE, "libctkv_profile.so")

F32, BF16 = 0, 1
OK, ESHAPE, ECONFIG, EINDEX, ECUDA, EWORKSPACE = range(6)
FLAG_DEGENERATE = 1
FLAG_EMPTY_RECALL = 2
FLAG_NONEMPTY_RECALL = 4
FLAG_ID_RANGE = 8
FLAG_CAPACITY = 16
FLAG_DUP_IDS = 32
FLAG_BUILD_FALLBACK = 64
FLAG_NO_TOKENS = 128
FLAG_INTERNAL = 256
BUILD_EXACT, BUILD_FAST = 0, 1

c_i32, c_i64, c_vp, c_size = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t


class Layout(ctypes.Structure):
    _fields_ = [("batch", c_i32), ("query_heads", c_i32), ("kv_heads", c_i32),
                ("head_dim", c_i32), ("capacity", c_i64), ("dtype", c_i32),
                ("init_len", c_i32), ("local_len", c_i32), ("reserved", c_i32)]


class StoreDesc(ctypes.Structure):
    _fields_ = [("keys", c_vp), ("values", c_vp), ("total", c_vp)]


class IndexDesc(ctypes.Structure):
    _fields_ = [("centroids", c_vp), ("lists", c_vp), ("fifo_head", c_vp), ("sync", c_vp),
                ("cnorm", c_vp), ("capacity", c_i32), ("rho", c_i32)]


class StepArgs(ctypes.Structure):
    _fields_ = [("query", c_vp), ("k_new", c_vp), ("v_new", c_vp),
                ("c_prime", c_i32), ("rho_prime", c_i32), ("use_dcu", c_i32),
                ("use_rerank", c_i32),
                ("out", c_vp), ("row_max", c_vp), ("denom", c_vp), ("selected", c_vp),
                ("recall_len", c_vp), ("sparse_ids", c_vp), ("sparse_len", c_vp),
                ("sparse_cap", c_i32), ("flags", c_vp)]


# every exported symbol with its ctypes signature (tests check the .so
# exports exactly these)
SIGNATURES = {
    "ctkv_abi_version": (c_i32, []),
    "ctkv_status_string": (ctypes.c_char_p, [c_i32]),
    "ctkv_device_ok": (c_i32, []),
    "ctkv_append": (c_i32, [ctypes.POINTER(Layout), StoreDesc, c_vp, c_vp, c_vp]),
    "ctkv_build_workspace_bytes": (c_size, [ctypes.POINTER(Layout), c_i32, c_i32, c_i64, c_i32]),
    "ctkv_build_lists": (c_i32, [ctypes.POINTER(Layout), c_vp, c_vp, c_i64, c_i64, c_i32, c_i32,
                                 c_i32, c_vp, c_vp, c_vp, c_size, c_vp]),
    "ctkv_decode_workspace_bytes": (c_size, [ctypes.POINTER(Layout), c_i32, c_i32, c_i32, c_i32]),
    "ctkv_decode_step": (c_i32, [ctypes.POINTER(Layout), StoreDesc, IndexDesc,
                                 ctypes.POINTER(StepArgs), c_vp, c_size, c_vp]),
    "ctkv_decode_step_phase": (c_i32, [ctypes.POINTER(Layout), StoreDesc, IndexDesc,
                                       ctypes.POINTER(StepArgs), c_i32, c_vp, c_size, c_vp]),
    "ctkv_recall": (c_i32, [ctypes.POINTER(Layout), IndexDesc, c_i64, c_vp, c_i32, c_vp, c_vp,
                            c_vp, c_vp, c_vp, c_size, c_vp]),
    "ctkv_rerank": (c_i32, [ctypes.POINTER(Layout), StoreDesc, c_vp, c_vp, c_vp, c_i32, c_vp,
                            c_vp, c_vp, c_vp, c_size, c_vp]),
    "ctkv_attend_workspace_bytes": (c_size, [ctypes.POINTER(Layout), c_i32, c_i32]),
    "ctkv_attend": (c_i32, [ctypes.POINTER(Layout), StoreDesc, c_vp, c_vp, c_vp, c_i32, c_i32,
                            c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "ctkv_merge": (c_i32, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp]),
    "ctkv_fifo_update": (c_i32, [ctypes.POINTER(Layout), IndexDesc, c_vp, c_vp, c_vp, c_i32,
                                 c_vp, c_vp, c_size, c_vp]),
    "ctkv_scores": (c_i32, [ctypes.POINTER(Layout), c_vp, c_i64, c_vp, c_i64, c_i64, c_i32,
                            c_vp, c_vp]),
    "ctkv_topk_workspace_bytes": (c_size, [c_i64, c_i64, c_i32]),
    "ctkv_topk_rows": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_size, c_vp]),
    "ctkv_debug_phase_timing": (c_i32, [c_i32, c_vp, c_i32]),
    "ctkv_debug_scan_timeline": (c_i32, [c_i32, c_vp, c_i32]),
    "ctkv_debug_kernel_timeline": (c_i32, [c_i32]),
    "ctkv_debug_timeline_rw": (c_i32, [ctypes.POINTER(Layout), c_i32, c_i32, c_i32, c_vp, c_vp, c_i32]),
    "ctkv_centroid_norms": (c_i32, [ctypes.POINTER(Layout), c_vp, c_i32, c_vp, c_vp]),
    "ctkv_stage_copy": (c_i32, [c_vp, c_vp, c_size, c_vp]),
}

_lib = None
_device_ok: dict[int, bool] = {}


def load_library(require_device: bool = True):
    """Load libctkv.so (once).  Raises RuntimeError when it is missing or,
    with require_device, when no sm_100 GPU is present."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2512_15550_b200/csrc)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ctkv_abi_version() != 1:
            raise RuntimeError("libctkv.so ABI version mismatch")
        _lib = lib
    if require_device:
        dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
        ok = _device_ok.get(dev)
        if ok is None:
            if dev < 0:
                raise RuntimeError("paper_2512_15550_b200 needs a CUDA device (B200, sm_100a); "
                                   "there is no CPU fallback")
            ok = _device_ok[dev] = bool(_lib.ctkv_device_ok())
        if not ok:
            raise RuntimeError("libctkv.so is built for sm_100a only; this device is not a B200")
    return _lib


def use_profile_library() -> None:
    """Profiling tools only: bind libctkv_profile.so instead of libctkv.so
    (must run before the first load)."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("libctkv is already loaded")
    LIB_PATH = PROFILE_LIB_PATH


def lib():
    return load_library(True)


def check(rc: int, what: str) -> None:
    """Map a ctkv_status to the reference's exception types (ck/errors.py)."""
    if rc == OK:
        return
    msg = f"{what}: {_lib.ctkv_status_string(rc).decode()}"
    if rc == ESHAPE:
        raise ShapeError(msg)
    if rc == ECONFIG:
        raise ConfigError(msg)
    if rc == EINDEX:
        raise IndexError(msg)
    raise RuntimeError(msg)


def raise_flags(flags: int, what: str, *, recall_mixed_is_error: bool = True) -> None:
    """Turn the device's sticky flag word into the reference's exceptions
    and warnings."""
    if flags & FLAG_DEGENERATE:
        warnings.warn("cosine of a zero-norm vector is defined as 0", DegenerateQueryWarning,
                      stacklevel=3)
    if flags & FLAG_ID_RANGE:
        raise IndexError(f"{what}: token id out of range")
    if recall_mixed_is_error and (flags & FLAG_EMPTY_RECALL) and (flags & FLAG_NONEMPTY_RECALL):
        raise ConfigError("decode_step: mixed empty/nonempty recall sets")
    if flags & FLAG_NO_TOKENS:
        raise ConfigError(f"{what}: no attendable tokens in either partition")
    if flags & FLAG_CAPACITY:
        raise ConfigError(f"{what}: a device buffer limit was exceeded")
    if flags & FLAG_INTERNAL:
        raise RuntimeError(f"{what}: a device-side wait timed out (internal error)")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return F32
    if dt == torch.bfloat16:
        return BF16
    raise ShapeError(f"unsupported element type {dt} (float32 or bfloat16)")
