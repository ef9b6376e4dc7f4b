"""ctypes binding of libquadra_b200.so (the C ABI in include/quadra_b200.h).

The shared library is built in-tree (``python __graft_entry__.py`` or
``make -C paper_2204_01701_b200/csrc``). There is no fallback: if it is
missing or cannot be loaded, every device entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, DeviceError, DimensionError, IntegrityError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libquadra_b200.so")
if os.environ.get("QD_DEV_LIB"):  # dev A/B timing: another in-tree build of this library
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), os.environ["QD_DEV_LIB"])

FAMILY_CODE = {"first_order": 0, "t2": 1, "t4": 2, "proposed": 3, "t2_linear": 4, "t3": 5, "t2and4": 6,
               "t1_pure": 7, "t1_full": 8, "t1and2": 9}
KIND_CODE = {"fc": 0, "conv": 1, "dwconv": 2}
F32, BF16 = 0, 1

QD_OK, QD_ERR_CONFIG, QD_ERR_DIM, QD_ERR_INTEGRITY = 0, 1, 2, 3
QD_ERR_CUDA, QD_ERR_UNSUPPORTED, QD_ERR_ARG = 4, 5, 6
FLAG_NO_DX, FLAG_FORCE_SIMT, FLAG_NO_DW, FLAG_TC_V1 = 1, 2, 4, 8
FLAG_D_GIVEN = 16  # backward: dy is the operand D (qd_bn_backward_D)

EXPORTS = ("qd_validate", "qd_out_shape", "qd_pack_bytes", "qd_workspace_bytes",
           "qd_pack_weights", "qd_forward", "qd_backward", "qd_path",
           "qd_error_string", "qd_last_error", "qd_launch_count", "qd_version",
           "qd_profile", "qd_profile_mark", "qd_profile_count", "qd_profile_read",
           "qd_sgd_pack", "qd_bn_workspace_bytes", "qd_bn_forward", "qd_bn_forward_res", "qd_bn_backward_D",
           "qd_maxpool_forward", "qd_maxpool_backward", "qd_im2col",
           "qd_bn_stats_rows", "qd_forward_bnstats", "qd_bn_forward_stats")


class QdDesc(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("kind", ctypes.c_int), ("dtype", ctypes.c_int),
                ("N", ctypes.c_int), ("C", ctypes.c_int), ("H", ctypes.c_int),
                ("W", ctypes.c_int), ("F", ctypes.c_int), ("r", ctypes.c_int),
                ("stride", ctypes.c_int), ("pad", ctypes.c_int), ("flags", ctypes.c_uint)]


_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes handle; raises DeviceError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is not built; run `python __graft_entry__.py` (build) first "
                "-- there is no CPU fallback")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover - depends on the box
            raise DeviceError(f"cannot load {LIB_PATH}: {e}") from e
        P = ctypes.POINTER
        vp = ctypes.c_void_p
        fp3 = ctypes.c_void_p * 3
        lib.qd_validate.argtypes = [P(QdDesc)]
        lib.qd_validate.restype = ctypes.c_int
        lib.qd_out_shape.argtypes = [P(QdDesc), P(ctypes.c_int), P(ctypes.c_int)]
        lib.qd_out_shape.restype = ctypes.c_int
        lib.qd_pack_bytes.argtypes = [P(QdDesc)]
        lib.qd_pack_bytes.restype = ctypes.c_size_t
        lib.qd_workspace_bytes.argtypes = [P(QdDesc)]
        lib.qd_workspace_bytes.restype = ctypes.c_size_t
        lib.qd_pack_weights.argtypes = [P(QdDesc), fp3, vp, vp]
        lib.qd_pack_weights.restype = ctypes.c_int
        lib.qd_sgd_pack.argtypes = [P(QdDesc), fp3, fp3, fp3, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                    ctypes.c_int, vp, vp]
        lib.qd_sgd_pack.restype = ctypes.c_int
        lib.qd_bn_workspace_bytes.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int]
        lib.qd_bn_workspace_bytes.restype = ctypes.c_size_t
        lib.qd_bn_forward.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp,
                                      ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp,
                                      vp]
        lib.qd_bn_forward.restype = ctypes.c_int
        lib.qd_bn_forward_res.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, vp,
                                          ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_int, vp, vp, vp,
                                          vp, vp]
        lib.qd_bn_stats_rows.argtypes = [P(QdDesc)]
        lib.qd_bn_stats_rows.restype = ctypes.c_int
        lib.qd_forward_bnstats.argtypes = [P(QdDesc), vp, vp, fp3, vp, vp, vp, vp, vp, vp]
        lib.qd_forward_bnstats.restype = ctypes.c_int
        lib.qd_bn_forward_stats.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int,
                                            vp, vp, vp, vp, ctypes.c_float, ctypes.c_float, ctypes.c_int,
                                            ctypes.c_int, vp, vp, vp, vp]
        lib.qd_bn_forward_stats.restype = ctypes.c_int
        lib.qd_bn_forward_res.restype = ctypes.c_int
        lib.qd_bn_backward_D.argtypes = [P(QdDesc), vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, fp3,
                                         vp, vp]
        lib.qd_bn_backward_D.restype = ctypes.c_int
        ci = ctypes.c_int
        lib.qd_maxpool_forward.argtypes = [ci, ci, ci, ci, ci, ci, ci, ci, vp, vp, vp, vp]
        lib.qd_maxpool_forward.restype = ctypes.c_int
        lib.qd_maxpool_backward.argtypes = [ci, ci, ci, ci, ci, ci, ci, ci, vp, vp, vp, vp]
        lib.qd_maxpool_backward.restype = ctypes.c_int
        lib.qd_im2col.argtypes = [ci, ci, ci, ci, ci, ci, ci, ci, ci, vp, vp, vp]
        lib.qd_im2col.restype = ctypes.c_int
        lib.qd_forward.argtypes = [P(QdDesc), vp, vp, fp3, vp, vp, vp, vp, vp]
        lib.qd_forward.restype = ctypes.c_int
        lib.qd_backward.argtypes = [P(QdDesc), vp, vp, vp, vp, vp, vp, fp3, fp3, vp, vp]
        lib.qd_backward.restype = ctypes.c_int
        lib.qd_path.argtypes = [P(QdDesc)]
        lib.qd_path.restype = ctypes.c_int
        lib.qd_error_string.argtypes = [ctypes.c_int]
        lib.qd_error_string.restype = ctypes.c_char_p
        lib.qd_last_error.argtypes = []
        lib.qd_last_error.restype = ctypes.c_char_p
        lib.qd_launch_count.argtypes = []
        lib.qd_launch_count.restype = ctypes.c_ulonglong
        lib.qd_version.argtypes = []
        lib.qd_version.restype = ctypes.c_char_p
        lib.qd_profile.argtypes = [ctypes.c_int]
        lib.qd_profile.restype = ctypes.c_int
        lib.qd_profile_mark.argtypes = [vp]
        lib.qd_profile_mark.restype = ctypes.c_int
        lib.qd_profile_count.argtypes = []
        lib.qd_profile_count.restype = ctypes.c_int
        lib.qd_profile_read.argtypes = [ctypes.c_int, P(ctypes.c_char_p), P(ctypes.c_float)]
        lib.qd_profile_read.restype = ctypes.c_int
        _lib = lib
        return lib


def raise_for(status, what=""):
    """Map a QD status to the reference exception classes."""
    if status == QD_OK:
        return
    lib = load()
    msg = lib.qd_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == QD_ERR_CONFIG:
        raise ConfigError(msg)
    if status == QD_ERR_DIM:
        raise DimensionError(msg)
    if status == QD_ERR_INTEGRITY:
        raise IntegrityError(msg)
    raise DeviceError(f"{lib.qd_error_string(status).decode()}: {msg}")


def ptr3(*ptrs):
    arr = (ctypes.c_void_p * 3)()
    for i, p in enumerate(ptrs[:3]):
        arr[i] = p if p else None
    return arr


def launch_count():
    return int(load().qd_launch_count())


def profile_read():
    """[(kernel name, ms)] since the last qd_profile(1) (caller synchronises)."""
    lib = load()
    out = []
    for i in range(1, lib.qd_profile_count()):
        nm = ctypes.c_char_p()
        ms = ctypes.c_float()
        raise_for(lib.qd_profile_read(i, ctypes.byref(nm), ctypes.byref(ms)), "qd_profile_read")
        out.append((nm.value.decode(), ms.value))
    return out
