"""Ingest of the reference's packed container straight to the device.

BMI1 (the reference's io.py:1-16): "BMI1", n_rows and n_cols as u64 LE,
then n_cols columns of ceil(n_rows/64) little-endian words -- byte for byte
the words layout of BinaryMatrix, so the payload is the device operand's
input as is.  ``read_bmi_device`` streams it through pinned double-buffered
staging into device memory (mi_bmi_load), skipping the host BinaryMatrix
and the host packing the reference needs.  Errors follow
read_bmi (io.py:92-116): FormatError for a short file, bad magic, bad
dimensions, a payload of the wrong length or nonzero padding bits.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import torch

from . import _native as nat
from .binmat import n_words


def bmi_shape(path: str | Path) -> tuple[int, int]:
    """(n_rows, n_cols) of a BMI1 file after validating header and length."""
    r, c = ctypes.c_int64(0), ctypes.c_int64(0)
    nat.check(nat.lib().mi_bmi_header(str(path).encode(), ctypes.addressof(r), ctypes.addressof(c)),
              "mi_bmi_header")
    return int(r.value), int(c.value)


def read_bmi_device(path: str | Path, device: torch.device | int = 0) -> tuple[torch.Tensor, int, int]:
    """Load a BMI1 file into a (n_cols, nw) int64 device tensor (the words,
    same bits).  Returns (words, n_rows, n_cols)."""
    n_rows, n_cols = bmi_shape(path)
    dev = torch.device("cuda", device) if isinstance(device, int) else device
    words = torch.empty((n_cols, n_words(n_rows)), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        nat.check(nat.lib().mi_bmi_load(str(path).encode(), words.data_ptr(), n_rows, n_cols, stream),
                  "mi_bmi_load")
    return words, n_rows, n_cols
