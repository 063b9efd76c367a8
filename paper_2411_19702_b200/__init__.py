"""B200-native all-pairs binary mutual information (arxiv 2411.19702).

Drop-in for the reference's ``mimatrix.mi_all_pairs`` dense path: one int8
tcgen05 Gram product over the upper triangle with the MI epilogue fused on
the TMEM accumulators.  The compute lives in the C-ABI
library ``lib/libmimatrix_b200.so`` (include/mimatrix_b200.h); this package
is the host-side mirror of the reference's operator interface.
"""

from .binmat import BinaryMatrix, from_bits, from_rows, pack_bits, unpack_bits
from .engine import (
    BACKENDS,
    MODES,
    EngineConfig,
    MIEngine,
    MIMatrix,
    column_sums,
    gram_ones,
    mi_all_pairs,
    mi_all_pairs_c_abi,
    mi_all_pairs_devices,
    unpack_upper,
)
from .errors import (
    ConsistencyError,
    DimensionError,
    DomainError,
    FormatError,
    MiMatrixError,
    NativeError,
)

__version__ = "0.1.0"

__all__ = [
    "BinaryMatrix", "from_bits", "from_rows", "pack_bits", "unpack_bits",
    "BACKENDS", "MODES", "EngineConfig", "MIEngine", "MIMatrix",
    "column_sums", "gram_ones", "mi_all_pairs", "mi_all_pairs_c_abi", "mi_all_pairs_devices", "unpack_upper",
    "ConsistencyError", "DimensionError", "DomainError", "FormatError", "MiMatrixError", "NativeError",
]
