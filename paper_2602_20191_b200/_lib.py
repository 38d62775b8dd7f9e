"""ctypes binding of the C ABI (include/mobi_b200.h) exported by libmobi_b200.so.

The product path has no fallback: if the CUDA library is missing this raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("MOBI_LIB_PATH", PKG / "libmobi_b200.so"))  # override: dev experiments

MOBI_OK, MOBI_EINVAL, MOBI_ERUNTIME = 0, 1, 2

_i64, _i32, _f32, _f64, _p = C.c_int64, C.c_int32, C.c_float, C.c_double, C.c_void_p


class MobiError(RuntimeError):
    """MOBI_ERUNTIME (CUDA failure) -- mirrors std::runtime_error."""


class MobiInvalidArgument(ValueError):
    """MOBI_EINVAL -- mirrors std::invalid_argument raised by the reference's MOBI_CHECK."""


class LayerDesc(C.Structure):
    _fields_ = [
        ("out", _i64), ("in_", _i64), ("group_size", _i64), ("n_slices", _i32),
        ("slice_bits", C.POINTER(_i32)), ("scale", C.POINTER(_f64)), ("zero", C.POINTER(_f64)),
        ("codes", C.POINTER(C.c_uint8)), ("planes", C.POINTER(C.c_uint64)), ("plane_bits", _i32),
        ("words_per_row", _i64), ("router_hidden", _i64), ("w1", C.POINTER(_f64)),
        ("b1", C.POINTER(_f64)), ("w2", C.POINTER(_f64)), ("b2", C.POINTER(_f64)),
    ]


class OutDesc(C.Structure):
    """mobi_out_desc: Y row t -> dst[k] + t*ldy + col0 for k < n_dst."""
    _fields_ = [("n_dst", _i32), ("dst", _p * 8), ("ldy", _i64), ("col0", _i64)]


_SIGS = {
    "mobi_layer_create": [C.POINTER(LayerDesc), C.c_int, C.POINTER(_p)],
    "mobi_layer_create_device": [C.POINTER(LayerDesc), C.c_int, C.POINTER(_p)],
    "mobi_layer_create_rows": [C.POINTER(LayerDesc), _i64, _i64, C.c_int, C.POINTER(_p)],
    "mobi_layer_destroy": [_p],
    "mobi_layer_reserve": [_p, _i64],
    "mobi_layer_info": [_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i64)],
    "mobi_layer_export_router": [_p, _p, _p, _p, _p],
    "mobi_layer_unpack_codes": [_p, _p],
    "mobi_score": [_p, _p, _i64, _p, _p],
    "mobi_route": [_p, _p, _i64, _f32, _p, _p, _p, _p, _p, _p],
    "mobi_forward": [_p, _p, _i64, _f32, _p, _p, _p],
    "mobi_forward_masked": [_p, _p, _i64, _p, _p, _p],
    "mobi_forward_host": [_p, _p, _i64, _f32, _p, _p, _p],
    "mobi_forward_out": [_p, _p, _i64, _f32, C.POINTER(OutDesc), _p, _p],
    "mobi_ipc_export": [_p, _p, C.POINTER(_i64)],
    "mobi_ipc_open": [_p, C.c_int, C.POINTER(_p)],
    "mobi_ipc_close": [_p],
    "mobi_layer_create_sharded": [C.POINTER(LayerDesc), _p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_p)],
    "mobi_forward_sharded": [_p, _p, _i64, _f32, _p, _p, _p],
    "mobi_permute_by_slice": [_p, _i64, _p, _p, _p, _p, C.POINTER(_i64), _p],
    "mobi_calibrate_threshold": [_p, _i64, _f64, C.POINTER(_f64), _p],
    "mobi_avg_bits": [_p, _i64, _p, _i32, C.POINTER(_f64), _p],
    "mobi_decompose": [_p, _i64, _i64, _i64, _p, _i32, _f64, _p, _p, _p, _p, _p],
    "mobi_joint_step": [_p, _i64, _i64, _i64, _p, _i32, _p, _p, _p, _p, _p, _p, _i64, _p, _p, _i64, _p, _i64, _i32,
                        _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "mobi_msb_step": [_p, _i64, _i64, _i64, _i32, _p, _p, _p, _p, _i64, _p, C.POINTER(_f64), _p, _p, _p],
    "mobi_layers_share_activations": [_p, _i32],
    "mobi_layer_last_launches": [_p, C.POINTER(_i32)],
    "mobi_layer_debug_impl": [_p, C.c_int],
    "mobi_layer_last_plan": [_p, C.POINTER(_i32)],
    "mobi_layer_profile": [_p, C.c_int],
    "mobi_layer_profile_read": [_p, _p, _p],
}

_lib = None


def build(force: bool = False) -> Path:
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    if force or not LIB_PATH.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(PKG / "csrc")], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise MobiError(f"{LIB_PATH} not built; run paper_2602_20191_b200._lib.build() "
                            "(no CPU fallback exists by design)")
        L = C.CDLL(str(LIB_PATH))
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.mobi_last_error.restype = C.c_char_p
        L.mobi_version.restype = C.c_char_p
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == MOBI_OK:
        return
    msg = lib().mobi_last_error().decode()
    if rc == MOBI_EINVAL:
        raise MobiInvalidArgument(msg)
    raise MobiError(msg)


def exported_symbols():
    return ["mobi_last_error", "mobi_version"] + list(_SIGS)
