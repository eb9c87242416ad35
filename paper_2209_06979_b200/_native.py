"""ctypes binding to libmcube.so (the C ABI declared in include/mcube.h).

The shared library is built in-tree (`__graft_entry__.build()` or
`make -C paper_2209_06979_b200/csrc`). There is no fallback: if the library or
a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional

from .errors import (FormatError, OverflowRiskError, QsparseError, ShuffleStateError,
                     UnsupportedPrecisionError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCUBE_LIB_PATH") or os.path.join(_HERE, "libmcube.so")  # override: debug builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "mcube.h")

MC_OK = 0
MC_ERR_VALUE = 1
MC_ERR_UNSUPPORTED_PRECISION = 2
MC_ERR_SHUFFLE_STATE = 3
MC_ERR_FORMAT = 4
MC_ERR_OVERFLOW = 5
MC_ERR_CUDA = 6

MC_ROW_MAJOR = 0
MC_COL_MAJOR = 1
MC_DTYPE_F16, MC_DTYPE_F32, MC_DTYPE_F64 = 0, 1, 2
MC_ATTN_PARITY, MC_ATTN_FAST = 0, 1
SPMM_PATHS = {0: "spmm_kernel (mma.sync gather, 64-column tasks)",
              1: "spmm_seg_kernel (mma.sync, 128-byte row-segment tasks)",
              2: "densify + gemm_tc_kernel (tcgen05)",
              3: "spmm_tc_kernel (tcgen05 gather)",
              4: "spmm_kernel (per-nibble chunk products)"}
SDDMM_PATHS = {1: "sddmm_tc_kernel (tcgen05 kind::i8 dense tile)",
               2: "sddmm_g8_kernel (pipelined mma.sync gather)",
               3: "sddmm_kernel (mma.sync gather)"}

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class McSrBcrs(ctypes.Structure):
    _fields_ = [("scalar_rows", _i64), ("scalar_cols", _i64), ("vector_length", _i32),
                ("stride", _i32), ("bit_width", _i32), ("shuffled", _i32),
                ("stored_vectors", _i64), ("row_begin", _p), ("row_end", _p),
                ("col_indices", _p), ("words", _p)]


class McDense(ctypes.Structure):
    _fields_ = [("rows", _i64), ("cols", _i64), ("bit_width", _i32), ("layout", _i32),
                ("words", _p)]


class McBcrs(ctypes.Structure):
    _fields_ = [("scalar_rows", _i64), ("scalar_cols", _i64), ("vector_length", _i32),
                ("reserved", _i32), ("n_blocks", _i64), ("row_offsets", _p),
                ("col_indices", _p)]


class McEpilogue(ctypes.Structure):
    _fields_ = [("alpha", _p), ("alpha_host", ctypes.c_double), ("out_f16", _p),
                ("out_f16_batch_stride", _i64)]


class McAttentionArgs(ctypes.Structure):
    _fields_ = [("batch", _i32), ("seq_len", _i32), ("head_dim", _i32),
                ("softmax_bits", _i32), ("qkv_bits", _i32), ("in_dtype", _i32), ("mode", _i32),
                ("q", _p), ("k", _p), ("v", _p), ("mask", ctypes.POINTER(McBcrs)),
                ("out_f16", _p), ("scores_int", _p), ("scores_f16", _p), ("probs_f16", _p),
                ("probs_int", _p), ("mix_int", _p), ("scales", _p), ("workspace", _p),
                ("workspace_bytes", ctypes.c_size_t)]


# entry point -> (restype, argtypes)
_SIGNATURES = {
    "mc_spmm": (_i32, [ctypes.POINTER(McSrBcrs), ctypes.POINTER(McDense), _i32, _p, _p, _p]),
    "mc_spmm_workspace": (_i32, [ctypes.POINTER(McSrBcrs), ctypes.POINTER(McDense),
                                 ctypes.POINTER(ctypes.c_size_t)]),
    "mc_spmm_path": (_i32, [ctypes.POINTER(McSrBcrs), ctypes.POINTER(McDense), ctypes.POINTER(_i32)]),
    "mc_spmm_ws": (_i32, [ctypes.POINTER(McSrBcrs), ctypes.POINTER(McDense), _i32, _p, _p, _p,
                          ctypes.c_size_t, _p]),
    "mc_spmm_batched": (_i32, [ctypes.POINTER(McSrBcrs), _i64, ctypes.POINTER(McDense), _i64, _i32,
                               ctypes.POINTER(McEpilogue), _p, _i64, _p, _p]),
    "mc_sddmm_path": (_i32, [ctypes.POINTER(McDense), ctypes.POINTER(McDense), ctypes.POINTER(McBcrs),
                             ctypes.POINTER(_i32)]),
    "mc_sddmm": (_i32, [ctypes.POINTER(McDense), ctypes.POINTER(McDense), ctypes.POINTER(McBcrs),
                        _p, _p, _p]),
    "mc_sddmm_batched": (_i32, [ctypes.POINTER(McDense), _i64, ctypes.POINTER(McDense), _i64,
                                ctypes.POINTER(McBcrs), _i32, ctypes.POINTER(McEpilogue), _p,
                                _i64, _p, _p]),
    "mc_srbcrs_plan": (_i32, [ctypes.POINTER(McBcrs), _i32, _p, _p, _p, _p]),
    "mc_srbcrs_fill": (_i32, [ctypes.POINTER(McBcrs), _i32, _p, _p, _i64, _p, _i32, _p, _p, _p]),
    "mc_shuffle_indices": (_i32, [_p, _i64, _i32, _p, _p]),
    "mc_attention_workspace": (_i32, [ctypes.POINTER(McAttentionArgs), ctypes.POINTER(ctypes.c_size_t)]),
    "mc_sparse_attention": (_i32, [ctypes.POINTER(McAttentionArgs), _p, _p]),
    "mc_status_fetch": (_i32, [_p, _p]),
    "mc_l2_flush": (_i32, [_p, ctypes.c_size_t, _p]),
    "mc_last_error": (ctypes.c_char_p, []),
    "mc_version": (_i32, []),
    "mc_launch_count": (_i64, [_i32]),
}

_lib: Optional[ctypes.CDLL] = None
_lock = threading.Lock()


def load(require_cuda: bool = False) -> ctypes.CDLL:
    """Load libmcube.so (no CUDA device needed just to load it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2209_06979_b200 kernels need a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
    return _lib


def lib() -> ctypes.CDLL:
    return load(require_cuda=True)


def last_error() -> str:
    return load().mc_last_error().decode(errors="replace")


_ERRORS = {
    MC_ERR_VALUE: ValueError,
    MC_ERR_UNSUPPORTED_PRECISION: UnsupportedPrecisionError,
    MC_ERR_SHUFFLE_STATE: ShuffleStateError,
    MC_ERR_FORMAT: FormatError,
    MC_ERR_OVERFLOW: OverflowRiskError,
}


def check(rc: int) -> None:
    """Raise the reference exception class for a non-zero return code."""
    if rc == MC_OK:
        return
    msg = last_error()
    exc = _ERRORS.get(rc)
    if exc is None:
        raise QsparseError(f"CUDA failure: {msg}")
    raise exc(msg)


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())
