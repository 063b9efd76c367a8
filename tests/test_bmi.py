"""BMI1 ingest: the reference's packed container
(io.py:1-16, read_bmi io.py:92-116) loaded straight to the device.

Golden files in tests/golden/bmi/ were written by the reference's own
write_bmi (tests/golden/make_bmi_golden.py), including the malformed
variants its tests build (test_io.py:87-111).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2411_19702_b200 import FormatError
from paper_2411_19702_b200 import io as bio

BMI = Path(__file__).resolve().parent / "golden" / "bmi"
META = json.loads((BMI / "bmi_meta.json").read_text())


def _host_words(path: Path, n_rows: int, n_cols: int) -> np.ndarray:
    nw = (n_rows + 63) // 64
    return np.frombuffer(path.read_bytes(), dtype="<u8", offset=20).reshape(n_cols, nw)


@pytest.mark.parametrize("name", sorted(META))
def test_header_of_reference_files(name):
    assert bio.bmi_shape(BMI / f"{name}.bmi") == (META[name]["n_rows"], META[name]["n_cols"])


@pytest.mark.parametrize("bad,needle", [("bad_magic", "bad magic"), ("truncated", "payload length"),
                                        ("short_header", "shorter than the 20-byte header")])
def test_malformed_headers_raise_format_error(bad, needle):
    with pytest.raises(FormatError, match=needle):
        bio.bmi_shape(BMI / f"{bad}.bmi")


def test_missing_file():
    with pytest.raises(FormatError):
        bio.bmi_shape(BMI / "does_not_exist.bmi")


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(META))
def test_device_load_is_the_payload(engine, name):
    path = BMI / f"{name}.bmi"
    words, n, m = bio.read_bmi_device(path, engine.device)
    host = _host_words(path, n, m)
    assert np.array_equal(words.cpu().numpy().view(np.uint64), host)
    assert [int(x) for x in O.column_sums(host)] == META[name]["column_sums"]


@pytest.mark.gpu
def test_dirty_padding_rejected_on_load(engine):
    with pytest.raises(FormatError, match="padding"):
        bio.read_bmi_device(BMI / "dirty_padding.bmi", engine.device)


@pytest.mark.gpu
def test_mi_from_file_matches_oracle(engine):
    path = BMI / "rand_1000x300.bmi"
    mi = engine.all_pairs_bmi(path).cpu().numpy()
    n, m = META["rand_1000x300"]["n_rows"], META["rand_1000x300"]["n_cols"]
    ref = O.c_mi_all_pairs(np.ascontiguousarray(_host_words(path, n, m)), n)
    assert np.array_equal(mi, mi.T)
    assert float(np.max(np.abs(mi - ref))) < 1e-12
