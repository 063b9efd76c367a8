"""Synthetic BASELINE configs, generated on the GPU straight into packed words.

The stream is the reference's (datagen.py:44-73: cell (r, c) uses splitmix64
draw r*m + c + 1, 1 iff draw < ceil(p*2^64)), so ``generate(n, m, p, seed)``
reproduces ``mimatrix.generate(GenSpec(n, m, p, seed))`` bit for bit (checked
against the reference's digests for configs 1 and 3).  The BASELINE configs
add per-column densities, constant columns and planted noisy copies
(SURVEY 8(d)); the recipe below is the product-side statement of it
(restated independently in oracle/oracle.py for the tests).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as nat
from .binmat import n_words
from .errors import DimensionError, DomainError

FLIP_SEED_XOR = 0xA5A5A5A5A5A5A5A5
KIND_BERNOULLI, KIND_ZERO, KIND_ONE, KIND_COPY = 0, 1, 2, 3

# name, N, m, seed, output dtype of the bench/parity run
CONFIGS = {
    1: dict(n=1000, m=500, seed=0, out="float64"),
    2: dict(n=10000, m=2000, seed=1, out="float64"),
    3: dict(n=100000, m=10000, seed=2, out="float64"),
    4: dict(n=50000, m=50000, seed=3, out="float32"),
    5: dict(n=1000000, m=20000, seed=4, out="float64"),
}


def threshold(density: float) -> int:
    """datagen.py:53-55"""
    if not 0.0 <= density <= 1.0:
        raise DomainError(f"density must lie in [0, 1], got {density}")
    return math.ceil(density * (1 << 64))


def config_recipe(cfg: int, n: int | None = None, m: int | None = None) -> dict:
    """Per-column densities and planting of BASELINE config `cfg`,
    optionally at a smaller (n, m) with the same recipe."""
    if cfg not in CONFIGS:
        raise DomainError(f"unknown config {cfg}")
    base = CONFIGS[cfg]
    n = base["n"] if n is None else n
    m = base["m"] if m is None else m
    seed = base["seed"]
    rng = np.random.default_rng(seed)
    r = {"n": n, "m": m, "seed": seed, "zero_cols": [], "one_cols": [], "pairs": [], "flip_density": 0.0}
    if cfg in (1, 3):
        r["density"] = np.full(m, 0.5)
        if cfg == 1:
            cols = rng.choice(m, 4, replace=False)
            r["zero_cols"] = [int(cols[0]), int(cols[1])]
            r["one_cols"] = [int(cols[2]), int(cols[3])]
    elif cfg == 2:
        r["density"] = rng.uniform(0.05, 0.95, m)
        k = min(200, m // 2)
        cols = rng.choice(m, 2 * k, replace=False)
        r["pairs"] = list(zip(cols[:k].tolist(), cols[k:].tolist()))
        r["flip_density"] = 0.1
    elif cfg == 4:
        r["density"] = rng.beta(0.5, 20.0, m)
        k = max(1, m // 100)
        targets = rng.choice(m, k, replace=False)
        is_target = np.zeros(m, dtype=bool)
        is_target[targets] = True
        pool = np.flatnonzero(~is_target)
        sources = rng.choice(pool, k, replace=True)
        r["pairs"] = list(zip(sources.tolist(), targets.tolist()))
        r["flip_density"] = 0.05
    else:
        r["density"] = rng.uniform(0.01, 0.99, m)
    return r


def column_program(recipe: dict) -> tuple[np.ndarray, np.ndarray, np.ndarray, int]:
    """(threshold u64[m], kind u8[m], src i32[m], flip threshold) for the kernel."""
    m = recipe["m"]
    thr = np.zeros(m, dtype=np.uint64)
    kind = np.zeros(m, dtype=np.uint8)
    src = np.zeros(m, dtype=np.int32)
    for c, d in enumerate(np.asarray(recipe["density"], dtype=np.float64)):
        t = threshold(float(d))
        if t <= 0:
            kind[c] = KIND_ZERO
        elif t >= 1 << 64:
            kind[c] = KIND_ONE
        else:
            thr[c] = t
    for c in recipe["zero_cols"]:
        kind[c] = KIND_ZERO
    for c in recipe["one_cols"]:
        kind[c] = KIND_ONE
    for s, t in recipe["pairs"]:
        if kind[s] != KIND_BERNOULLI:
            raise DomainError("a planted copy's source must be a Bernoulli column")
        kind[t] = KIND_COPY
        src[t] = s
    ft = threshold(recipe["flip_density"]) if recipe["pairs"] else 0
    if ft >= 1 << 64:
        ft = (1 << 64) - 1
    return thr, kind, src, ft


def generate_words_device(recipe: dict, device: torch.device | int = 0) -> torch.Tensor:
    """Packed words (m, nw) of a recipe, produced on the GPU (int64 storage)."""
    n, m, seed = recipe["n"], recipe["m"], recipe["seed"]
    if n < 1 or m < 1:
        raise DimensionError("n_rows and n_cols must be at least 1")
    dev = torch.device("cuda", device) if isinstance(device, int) else device
    thr, kind, src, ft = column_program(recipe)
    d_thr = torch.from_numpy(thr.view(np.int64)).to(dev)
    d_kind = torch.from_numpy(kind).to(dev)
    d_src = torch.from_numpy(src).to(dev)
    words = torch.empty((m, n_words(n)), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    nat.check(nat.lib().mi_generate_words(words.data_ptr(), n, m, seed & ((1 << 64) - 1), d_thr.data_ptr(),
                                          d_kind.data_ptr(), d_src.data_ptr(), ft,
                                          (seed ^ FLIP_SEED_XOR) & ((1 << 64) - 1), stream),
              "mi_generate_words")
    return words


def generate(n: int, m: int, density: float, seed: int, device: torch.device | int = 0) -> torch.Tensor:
    """Device words of the reference's generate(GenSpec(n, m, density, seed))."""
    if not 0 <= seed < 1 << 64:
        raise DomainError("seed must fit in an unsigned 64-bit integer")
    recipe = {"n": n, "m": m, "seed": seed, "density": np.full(m, float(density)), "zero_cols": [],
              "one_cols": [], "pairs": [], "flip_density": 0.0}
    return generate_words_device(recipe, device)
