"""Install this engine into an existing ``mimatrix`` (the reference package).

    import mimatrix
    from paper_2411_19702_b200 import compat
    compat.install(mimatrix)          # before importing mimatrix.cli / mimatrix.bench

After ``install``, ``mimatrix.mi_all_pairs`` and ``mimatrix.engine.mi_all_pairs``
(engine.py:144-168) run the B200 path and return the reference's own
``MIMatrix`` type; our errors are re-raised as the reference's exception
classes (errors.py:8-25), so callers' ``except`` clauses and the CLI's exit
codes (cli.py:160-179) are unchanged.  ``cli`` and ``bench`` bind the name at
import (cli.py:18, bench.py:24), hence "install first".  ``gram.gram_ones``
(gram.py:56-65) and ``binmat.column_sums`` (binmat.py:175-177) are replaced by
their device versions too, so ``gram_from_dense`` also runs on the GPU.
"""

from __future__ import annotations

import functools

from . import engine as _engine
from . import errors as _errors


def _translate(ref_errors):
    table = {
        _errors.DimensionError: ref_errors.DimensionError,
        _errors.DomainError: ref_errors.DomainError,
        _errors.ConsistencyError: ref_errors.ConsistencyError,
        _errors.FormatError: ref_errors.FormatError,
    }

    def wrap(fn):
        @functools.wraps(fn)
        def inner(*a, **kw):
            try:
                return fn(*a, **kw)
            except _errors.MiMatrixError as exc:
                cls = table.get(type(exc), ref_errors.MiMatrixError)
                raise cls(str(exc)) from exc

        return inner

    return wrap


def install(mimatrix, device: int | None = None) -> None:
    """Patch the reference package in place (idempotent)."""
    import importlib

    ref_engine = importlib.import_module(mimatrix.__name__ + ".engine")
    ref_errors = importlib.import_module(mimatrix.__name__ + ".errors")
    ref_gram = importlib.import_module(mimatrix.__name__ + ".gram")
    ref_binmat = importlib.import_module(mimatrix.__name__ + ".binmat")
    wrap = _translate(ref_errors)

    @wrap
    def mi_all_pairs(data, cfg=None, backend="dense", threads=0):
        res = _engine.mi_all_pairs(data, cfg, backend, threads, device=device)
        return ref_engine.MIMatrix(values=res.values)

    @wrap
    def gram_ones(matrix):
        return _engine.gram_ones(matrix, device=device)

    @wrap
    def column_sums(matrix):
        return _engine.column_sums(matrix, device=device)

    mi_all_pairs.__b200__ = True
    ref_engine.mi_all_pairs = mi_all_pairs
    mimatrix.mi_all_pairs = mi_all_pairs
    ref_gram.gram_ones = gram_ones
    mimatrix.gram_ones = gram_ones
    ref_gram.column_sums = column_sums  # gram_from_dense resolves it from gram's namespace
    ref_binmat.column_sums = column_sums
    mimatrix.column_sums = column_sums
    for mod in ("cli", "bench"):
        m = getattr(mimatrix, mod, None)
        if m is not None and hasattr(m, "mi_all_pairs"):
            m.mi_all_pairs = mi_all_pairs


def installed(mimatrix) -> bool:
    return bool(getattr(getattr(mimatrix, "mi_all_pairs", None), "__b200__", False))
