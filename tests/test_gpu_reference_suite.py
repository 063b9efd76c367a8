"""The reference's own test suite, run against this engine on the GPU.

tools/run_reference_suite.sh installs paper_2411_19702_b200.compat into the
reference package staged under baseline/_ref/pkg (a git-ignored copy that
travels to the GPU box; `tools/run_reference_suite.sh stage` makes it), so
mimatrix.mi_all_pairs / gram_ones / column_sums -- and every caller bound to
them at import: cli._cmd_compute (cli.py:43), bench._run_backend
(bench.py:93-101) with its checksum consistency check (bench.py:171-185) --
run the B200 path.  Deselected: the two criteria that time the reference's
own CPU backends against each other (direct vs dense Gram, sparse vs dense
sweep); with every backend name on one GPU path they measure nothing.
A missing staged copy is a failure, not a skip.
"""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref" / "pkg"
DESELECT = ["tests/test_acceptance.py::test_optimized_vs_direct_gram",
            "tests/test_acceptance.py::test_sparsity_sweep_shape"]


def test_reference_suite_through_compat():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    assert (REF / "tests").is_dir() and (REF / "src" / "mimatrix").is_dir(), \
        f"{REF} is missing: stage it with `tools/run_reference_suite.sh stage` in the build container"
    cmd = ["bash", str(ROOT / "tools" / "run_reference_suite.sh"), "run"]
    for d in DESELECT:
        cmd += ["--deselect", d]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    assert "mimatrix.mi_all_pairs -> B200 engine" in r.stderr, tail
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 190, tail
    assert " failed" not in r.stdout.splitlines()[-1], tail
