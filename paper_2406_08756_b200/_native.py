"""ctypes binding of the in-tree native library `_lib/liblynx_b200.so`.

There is no fallback: if the library is missing or fails to load, importing
anything that needs it raises. The library is built by `build.py`
(`__graft_entry__.build()`), never JIT-compiled at import time.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liblynx_b200.so"
if os.environ.get("LYNX_LIB_VARIANT"):  # kernel A/B experiments: _lib/liblynx_b200.<variant>.so
    LIB_PATH = LIB_PATH.with_name(f"liblynx_b200.{os.environ['LYNX_LIB_VARIANT']}.so")

_c = ctypes
_vp, _i, _ll, _f, _sz, _ull = _c.c_void_p, _c.c_int, _c.c_longlong, _c.c_float, _c.c_size_t, _c.c_ulonglong
_fp = _c.POINTER(_c.c_float)

# name -> (restype, argtypes); mirrors include/lynx_b200.h and include/lynx_rt.h
_SIGNATURES: dict[str, tuple] = {
    "lynx_last_error": (_c.c_char_p, []),
    "lynx_abi_version": (_i, []),
    "lynx_op_gemm": (_i, [_vp, _ll, _i, _vp, _ll, _i, _vp, _ll, _i, _i, _i, _vp, _i, _vp]),
    "lynx_op_gemm_gelu": (_i, [_vp, _ll, _i, _vp, _ll, _i, _vp, _vp, _ll, _i, _i, _i, _vp, _vp]),
    "lynx_op_tp_signal_wait": (_i, [_vp, _vp, _i, _i, _ull, _vp]),
    "lynx_op_tp_reduce_residual": (_i, [_vp, _i, _vp, _vp, _vp, _ll, _i, _f, _ull, _ull, _vp]),
    "lynx_op_gemm_residual": (_i, [_vp, _ll, _vp, _ll, _vp, _ll, _i, _i, _i, _vp, _vp, _f, _ull, _ull, _vp]),
    "lynx_op_gemm_gelu_bwd": (_i, [_vp, _ll, _vp, _ll, _i, _vp, _ll, _i, _i, _i, _vp, _vp]),
    "lynx_op_gemm_mode": (None, [_i]),
    "lynx_op_attention_mode": (None, [_i]),
    "lynx_op_attention_bwd_warpgroups": (None, [_i]),
    "lynx_op_attention_fwd_tiles": (None, [_i]),
    "lynx_op_attention_tc_supported": (_i, [_i, _i]),
    "lynx_op_layernorm_fwd": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _f, _vp]),
    "lynx_op_layernorm_bwd_workspace": (_sz, [_i, _i]),
    "lynx_op_layernorm_bwd": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp]),
    "lynx_op_bias_dropout_residual": (_i, [_vp, _vp, _vp, _vp, _ll, _i, _f, _ull, _ull, _vp]),
    "lynx_op_dropout_bwd": (_i, [_vp, _vp, _ll, _i, _f, _ull, _ull, _vp]),
    "lynx_op_column_sum_workspace": (_sz, [_ll, _i]),
    "lynx_op_column_sum_acc": (_i, [_vp, _vp, _vp, _ll, _i, _vp]),
    "lynx_op_dropout_bwd_colsum": (_i, [_vp, _vp, _vp, _vp, _ll, _i, _f, _ull, _ull, _vp]),
    "lynx_op_gelu_fwd": (_i, [_vp, _vp, _ll, _vp]),
    "lynx_op_gelu_bwd": (_i, [_vp, _vp, _vp, _ll, _vp]),
    "lynx_op_attention_fwd": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp]),
    "lynx_op_attention_bwd_workspace": (_sz, [_i, _i, _i]),
    "lynx_op_attention_bwd": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp]),
    "lynx_op_embedding_fwd": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _f, _ull, _ull, _vp]),
    "lynx_op_embedding_bwd_workspace": (_sz, [_i, _i, _i]),
    "lynx_op_embedding_bwd": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _f, _ull, _ull, _vp]),
    "lynx_op_xent_fwd_bwd": (_i, [_vp, _vp, _vp, _ll, _i, _f, _vp]),
    "lynx_op_adam": (_i, [_vp, _vp, _vp, _vp, _vp, _ll, _f, _f, _f, _f, _f, _i, _f, _vp]),
    "lynx_op_init_normal": (_i, [_vp, _vp, _ll, _f, _ull, _ull, _vp]),
}

_lib: ctypes.CDLL | None = None


class LynxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[lynx status {code}] {msg}")
        self.code = code


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"native library {LIB_PATH} is missing; run `python -m paper_2406_08756_b200.build` "
                "(there is no CPU fallback)")
        l = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(l, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(code: int) -> None:
    if code != 0:
        raise LynxError(code, lib().lynx_last_error().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
