"""ctypes binding of the sm_100a C-ABI library (include/semstream_b200.h).

The library is built in-tree (``_build.py``) and loaded from this package
directory.  There is no CPU fallback: if the shared object or a CUDA device
is missing, every codec call raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsemstream_b200.so"

SST_OK = 0
SST_ERR_ARG = -1
SST_ERR_ROWS_16BIT = -2
SST_ERR_CUDA = -3
SST_ERR_UNSUPPORTED = -4

# per-packet status words (include/semstream_b200.h SST_PKT_*)
PKT_OK, PKT_SHORT, PKT_CRC, PKT_BODY_SHORT, PKT_MAGIC, PKT_VERSION, PKT_KIND, \
    PKT_HDR_TRUNC, PKT_MASK_TRUNC, PKT_PAYLOAD_LEN, PKT_NEG_RANGE, PKT_ABSENT, \
    PKT_FOREIGN, PKT_ROW_RANGE, PKT_DUP, PKT_SHAPE = range(16)


class SstPacketInfo(C.Structure):
    _fields_ = [("status", C.c_int32), ("kind", C.c_int32), ("gop_id", C.c_uint32),
                ("row", C.c_int32), ("width", C.c_int32), ("channels", C.c_int32),
                ("scale", C.c_int32), ("valid", C.c_int32), ("qmin", C.c_float),
                ("qrange", C.c_float), ("mask_off", C.c_int32), ("payload_off", C.c_int32),
                ("dqmin", C.c_double), ("dqrange", C.c_double)]


class SstPrevDesc(C.Structure):
    _fields_ = [("p_img", C.c_void_p), ("h", C.c_int32), ("w", C.c_int32), ("s", C.c_int32),
                ("reserved", C.c_int32)]


class SstPrevTokDesc(C.Structure):
    _fields_ = [("tok", C.c_void_p), ("pvalid", C.c_void_p), ("h", C.c_int32), ("w", C.c_int32),
                ("s", C.c_int32), ("Ht", C.c_int32), ("Wt", C.c_int32), ("reserved", C.c_int32)]


class SstConvDesc(C.Structure):
    """include/semstream_b200.h SstConvDesc (learned tokenizer, one conv layer)."""
    _fields_ = [("in_", C.c_void_p), ("in_C", C.c_int32), ("in_W", C.c_int32),
                ("in_H", C.c_int32), ("in_T", C.c_int32), ("G", C.c_int32), ("Ht", C.c_int32),
                ("Wt", C.c_int32), ("t_lo", C.c_int32), ("t_cnt", C.c_int32),
                ("n_taps", C.c_int32), ("taps", (C.c_int32 * 3) * 27), ("weight", C.c_void_p),
                ("N", C.c_int32), ("K", C.c_int32), ("bias", C.c_void_p), ("epi", C.c_int32),
                ("act", C.c_int32), ("residual", C.c_void_p), ("out", C.c_void_p),
                ("out_T", C.c_int32), ("codes", C.c_void_p), ("idx", C.c_void_p),
                ("mask", C.c_void_p), ("frames", C.c_void_p), ("h", C.c_int32),
                ("w", C.c_int32), ("frame_base", C.c_int32), ("shift", C.c_int32),
                ("bias_i32", C.c_void_p), ("act_lut", C.c_void_p)]


LT_EPI_STORE, LT_EPI_FSQ, LT_EPI_PIXELS, LT_EPI_PIXELS_U8 = 0, 1, 2, 3

INFO_BYTES = C.sizeof(SstPacketInfo)          # 64
PREV_BYTES = C.sizeof(SstPrevDesc)            # 24
PREVTOK_BYTES = C.sizeof(SstPrevTokDesc)      # 40

_P = C.c_void_p
_I = C.c_int
_L = C.c_int64

# name -> (restype, argtypes); mirrors include/semstream_b200.h
SIGNATURES = {
    "sst_abi_version": (_I, []),
    "sst_packet_wire_size": (_L, [_I, _I, _I]),
    "sst_downscale": (_I, [_P, _L, _I, _I, _I, _P, _P]),
    "sst_upscale": (_I, [_P, _L, _I, _I, _I, _I, _I, _P, _P]),
    "sst_bilinear_f64": (_I, [_P, _L, _I, _I, _I, _P, _P]),
    "sst_clip_cast": (_I, [_P, _L, _P, _P]),
    "sst_blend": (_I, [_P, _P, _I, _I, _I, _I, _P, _P]),
    "sst_encode": (_I, [_P, _I, _I, _I, _I, _P, _P, _P]),
    "sst_encode_work": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "sst_encode_u8": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "sst_decode": (_I, [_P, _P, _L, _P, _I, _I, _I, _I, _I, _P, _P]),
    "sst_similarity": (_I, [_P, _P, _L, _I, _P, _P]),
    "sst_topk_mask": (_I, [_P, _I, _L, _P, _P, _P, _P]),
    "sst_apply_mask": (_I, [_P, _P, _P, _L, _I, _P]),
    "sst_select_drop": (_I, [_P, _P, _P, _I, _I, _I, _P, _P, _P]),
    "sst_packetize": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _L, _P, _P]),
    "sst_serialize": (_I, [_P, _P, _P, _P, _P, _L, _P, _P, _P]),
    "sst_parse": (_I, [_P, _P, _P, _P, _L, _P, _P]),
    "sst_reassemble": (_I, [_P, _P, _P, _P, _L, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "sst_unpack_decode_workspace": (_L, [_I, _I, _I]),
    "sst_unpack_decode": (_I, [_P, _P, _P, _P, _L, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "sst_unpack_tokens": (_I, [_P, _P, _P, _P, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "sst_upscale_blend_tok": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "sst_upscale_blend": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "sst_upscale_blend_u8": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "sst_mse": (_I, [_P, _P, _L, _L, _P, _P]),
    "sst_mean_diff": (_I, [_P, _P, _L, _L, _I, _P, _P]),
    "sst_similarity_gop": (_I, [_P, _I, _L, _I, _P, _P]),
    "sst_upscale_blend9": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "sst_upscale_blend9_u8": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "sst_lt_conv": (_I, [C.POINTER(SstConvDesc), _P]),
    "sst_lt8_conv": (_I, [C.POINTER(SstConvDesc), _P]),
    "sst_lt8_patchify": (_I, [_P, _I, _I, _I, _I, _P, _P, _P]),
    "sst_lt8_patchify_haar": (_I, [_P, _I, _I, _I, _I, _P, _P, _P]),
    "sst_lt8_attn": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "sst_lt8_attn_global": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "sst_lt8_dec_in": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "sst_lt8_unpack_workspace": (_L, [_I, _I, _I]),
    "sst_lt8_unpack_dec_in": (_I, [_P, _P, _P, _P, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "sst_lt_patchify": (_I, [_P, _I, _I, _I, _I, _P, _P, _P]),
    "sst_lt_dec_in": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "sst_lt_attn": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "sst_lt_attn_fused": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "sst_lt_unpack_dec_in": (_I, [_P, _P, _P, _P, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "sst_residual": (_I, [_P, _P, _I, _I, _I, C.c_double, C.c_double, _P, _P, _P, _P, _P]),
    "sst_mean_axis0": (_I, [_P, _I, _L, _P, _P]),
    "sst_sparsify": (_I, [_P, _I, _L, C.c_double, C.c_double, _P, _P, _P, _P]),
    "sst_apply_residual": (_I, [_P, _P, _P, _I, _I, _I, C.c_double, _P]),
    "sst_mask_scan": (_I, [_P, _P, _L, _P, _P]),
    "sst_residual_diff": (_I, [_P, _P, _L, _P, _P]),
    "sst_dequant_i16": (_I, [_P, _L, C.c_double, _P, _P]),
    "sst_rc_encode": (_I, [_P, _I, _L, _P, _P, _L, _P, _P]),
    "sst_rc_decode": (_I, [_P, _P, _P, _I, _L, _P, _P, _P]),
    "sst_rc_encode_symbols": (_I, [_P, _P, _P, _I, _P, _L, _P, _P]),
    "sst_rc_decode_symbols": (_I, [_P, _L, _L, _L, _P, _P, _P, _P]),
}

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load (once) and return the C-ABI library; raises if it was never built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"semstream_b200 CUDA extension not built ({LIB_PATH} missing); "
                    "run `python -m paper_2602_03529_b200._build` -- there is no CPU fallback")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class CudaCallError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc == SST_OK:
        return
    if rc == SST_ERR_ROWS_16BIT:
        raise ValueError(f"{what}: matrix has more than 65535 rows; the row index field is 16-bit")
    if rc == SST_ERR_ARG:
        raise ValueError(f"{what}: invalid argument")
    if rc == SST_ERR_UNSUPPORTED:
        raise ValueError(f"{what}: unsupported shape for the CUDA kernel")
    raise CudaCallError(f"{what}: CUDA launch failed (status {rc})")


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    check(rc, name)


# numpy view of SstPacketInfo (same 64-byte layout)
try:
    import numpy as _np

    INFO_DTYPE = _np.dtype([("status", "<i4"), ("kind", "<i4"), ("gop_id", "<u4"), ("row", "<i4"),
                            ("width", "<i4"), ("channels", "<i4"), ("scale", "<i4"),
                            ("valid", "<i4"), ("qmin", "<f4"), ("qrange", "<f4"),
                            ("mask_off", "<i4"), ("payload_off", "<i4"), ("dqmin", "<f8"),
                            ("dqrange", "<f8")])
    PREV_DTYPE = _np.dtype([("p_img", "<u8"), ("h", "<i4"), ("w", "<i4"), ("s", "<i4"),
                            ("reserved", "<i4")])
    PREVTOK_DTYPE = _np.dtype([("tok", "<u8"), ("pvalid", "<u8"), ("h", "<i4"), ("w", "<i4"),
                               ("s", "<i4"), ("Ht", "<i4"), ("Wt", "<i4"), ("reserved", "<i4")])
    assert INFO_DTYPE.itemsize == INFO_BYTES and PREV_DTYPE.itemsize == PREV_BYTES
    assert PREVTOK_DTYPE.itemsize == PREVTOK_BYTES
except ImportError:  # pragma: no cover
    pass
