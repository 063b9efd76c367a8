"""ctypes binding of libmimatrix_b200.so (C ABI: include/mimatrix_b200.h).

The library is built in-tree (``make -C paper_2411_19702_b200/csrc`` or
``__graft_entry__.build()``).  There is no fallback: if it is missing or the
device is not an sm_100 part, every compute call raises NativeError.
ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

from .errors import ConsistencyError, DimensionError, DomainError, FormatError, MiMatrixError, NativeError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmimatrix_b200.so"
if os.environ.get("MI_B200_LIB"):  # experiments: A/B another build of the library
    LIB_PATH = Path(os.environ["MI_B200_LIB"]).resolve()
HEADER_PATH = Path(__file__).resolve().parent.parent / "include" / "mimatrix_b200.h"

MI_OK = 0
MI_ERR_DIMENSION = 1
MI_ERR_DOMAIN = 2
MI_ERR_CONSISTENCY = 3
MI_ERR_CUDA = 4
MI_ERR_UNSUPPORTED = 5
MI_ERR_FORMAT = 6

MI_MODE_EXACT = 0
MI_MODE_EPSILON = 1
MI_OUT_COUNTS = 0
MI_OUT_F64 = 1
MI_OUT_F32 = 2
MI_PACKED_UPPER = 0  # ld_out selecting the packed upper-triangle output
MI_TILE_MAJOR = -1  # ld_out selecting the tile-major (sharded) output

_ERRORS = {
    MI_ERR_DIMENSION: DimensionError,
    MI_ERR_DOMAIN: DomainError,
    MI_ERR_CONSISTENCY: ConsistencyError,
    MI_ERR_CUDA: NativeError,
    MI_ERR_UNSUPPORTED: NativeError,
    MI_ERR_FORMAT: FormatError,
}

_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double

# name -> (restype, argtypes); must cover every function in include/mimatrix_b200.h
SIGNATURES = {
    "mi_b200_abi_version": (_int, []),
    "mi_last_error": (ctypes.c_char_p, []),
    "mi_device_info": (_int, [_int, _vp, _vp, _vp]),
    "mi_kmajor_ld": (_i64, [_i64]),
    "mi_kmajor_rows": (_i64, [_i64]),
    "mi_colstat_bytes": (_i64, [_i64, _i64]),
    "mi_tile_size": (_int, []),
    "mi_num_tiles": (_i64, [_i64]),
    "mi_tile_list": (_i64, [_i64, _int, _int, _int, _vp, _i64]),
    "mi_rank_blocks": (_i64, [_i64, _int, _int, _vp, _i64]),
    "mi_unpack_colsum": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp]),
    "mi_unpack_colsum_blocks": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp]),
    "mi_pack_bits": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "mi_pack_sparse": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "mi_unpack_prep": (_int, [_i64, _i64, _vp, _vp]),
    "mi_unpack_colsum_range": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _vp]),
    "mi_column_order": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "mi_unpack_colsum_ordered": (_int, [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "mi_unpermute": (_int, [_vp, _i64, _vp, _i64, _i64, _int, _vp, _vp]),
    "mi_gram_mi": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _dbl, _int, _int, _vp, _i64, _vp, _i64, _vp]),
    "mi_words_operand": (_int, [_i64, _i64]),
    "mi_colstat_words": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "mi_gram_mi_words": (_int, [_vp, _vp, _i64, _i64, _int, _dbl, _int, _int, _vp, _i64, _vp, _i64, _vp]),
    "mi_gram_mi_words_stats": (_int, [_vp, _vp, _vp, _i64, _i64, _int, _dbl, _int, _int, _vp, _i64, _vp, _i64, _vp]),
    "mi_generate_words": (_int, [_vp, _i64, _i64, _u64, _vp, _vp, _vp, _u64, _u64, _vp]),
    "mi_all_pairs_host": (_int, [_vp, _i64, _i64, _int, _dbl, _int, _int, _vp, _int]),
    "mi_all_pairs_host_packed": (_int, [_vp, _i64, _i64, _int, _dbl, _int, _int, _vp, _int]),
    "mi_all_pairs_host_devices": (_int, [_vp, _i64, _i64, _int, _dbl, _int, _int, _vp, _vp, _int]),
    "mi_gram_ones_host": (_int, [_vp, _i64, _i64, _vp, _int]),
    "mi_column_sums_host": (_int, [_vp, _i64, _i64, _vp, _int]),
    "mi_host_register": (_int, [_vp, _i64]),
    "mi_host_unregister": (_int, [_vp]),
    "mi_copy_tiles_to_host": (_int, [_vp, _i64, _i64, _int, _vp, _i64, _vp, _i64, _vp]),
    "mi_scatter_tiles": (_int, [_vp, _vp, _i64, _i64, _int, _vp, _i64, _int, _vp]),
    "mi_bmi_header": (_int, [ctypes.c_char_p, _vp, _vp]),
    "mi_bmi_load": (_int, [ctypes.c_char_p, _vp, _i64, _i64, _vp]),
    "mi_set_tuning": (_int, [ctypes.c_char_p, _int]),
    "mi_get_tuning": (_int, [ctypes.c_char_p]),
    "mi_release_workspace": (None, []),
    "mi_tensor_peak": (_int, [_int, _int, _dbl, _vp, _vp, _vp]),
}

_lib = None


def header_functions() -> list[str]:
    """Function names declared in include/mimatrix_b200.h."""
    text = HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(mi_[a-z0-9_]+)\s*\(", text, flags=re.M)


def lib() -> ctypes.CDLL:
    """Load the engine library (once).  Raises NativeError when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2411_19702_b200/csrc` "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("MI_B200_LIB") and not hasattr(handle, name):
                continue  # A/B against an older build that predates this entry point
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.mi_b200_abi_version() != 1:
            raise NativeError("libmimatrix_b200.so ABI version mismatch")
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().mi_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc != MI_OK:
        cls = _ERRORS.get(rc, MiMatrixError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


def device_info(device: int) -> tuple[int, int, int]:
    sms, major, minor = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    check(lib().mi_device_info(device, ctypes.byref(sms), ctypes.byref(major), ctypes.byref(minor)),
          "mi_device_info")
    return sms.value, major.value, minor.value


def set_tuning(**kw) -> None:
    """e.g. set_tuning(prefetch=8, l2_hint=1) -- see mi_set_tuning in the header."""
    for k, v in kw.items():
        check(lib().mi_set_tuning(k.encode(), int(v)), f"mi_set_tuning({k})")


def get_tuning(key: str) -> int:
    return int(lib().mi_get_tuning(key.encode()))


def tensor_peak(device: int = 0, fp4: bool = True, seconds: float = 0.05) -> dict:
    """Measured tensor peak of the device (mi_tensor_peak): dense ops/s of the
    fused kernel's MMA instruction on resident operands, MACs/clk/SM, clock."""
    ops, macs, mhz = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
    check(lib().mi_tensor_peak(device, 1 if fp4 else 0, seconds, ctypes.byref(ops), ctypes.byref(macs),
                               ctypes.byref(mhz)), "mi_tensor_peak")
    return {"ops_per_s": ops.value, "macs_per_clk_sm": macs.value, "sm_mhz": mhz.value, "seconds": seconds,
            "instruction": "tcgen05.mma.cta_group::2.kind::" + ("mxf4.block_scale.block32" if fp4 else "i8") +
                           " M256 N256, smem-resident operands, all SM pairs"}


def rank_blocks(n_cols: int, rank: int = 0, world: int = 1):
    """uint8 mask of the column blocks rank's tiles touch (host-side logic only)."""
    import numpy as np

    T = int(lib().mi_rank_blocks(n_cols, rank, world, None, 0))
    check(0 if T > 0 else -T, "mi_rank_blocks")
    mask = np.zeros(T, dtype=np.uint8)
    n = int(lib().mi_rank_blocks(n_cols, rank, world, mask.ctypes.data, T))
    check(0 if n >= 0 else -n, "mi_rank_blocks")
    return mask


def tile_list(n_cols: int, rank: int = 0, world: int = 1, band: int = 0):
    """(I, J) upper-triangle tiles of `rank` (host-side logic only)."""
    import numpy as np

    L = lib()
    count = L.mi_tile_list(n_cols, rank, world, band, None, 0)
    if count < 0:
        check(-count, "mi_tile_list")
    out = np.zeros((max(count, 1), 2), dtype=np.int32)
    got = L.mi_tile_list(n_cols, rank, world, band, out.ctypes.data, count)
    if got < 0:
        check(-got, "mi_tile_list")
    return out[:got]
