"""pytest plugin: run the reference's own test suite against the B200 engine.

Loaded with `-p b200_plugin`; installs paper_2411_19702_b200.compat into the
reference package before any test module imports mimatrix.cli / .bench.
"""
import os
import sys


def pytest_configure(config):
    repo = os.environ["B200_REPO"]
    if repo not in sys.path:
        sys.path.insert(0, repo)
    import mimatrix
    from paper_2411_19702_b200 import compat

    compat.install(mimatrix)
    assert compat.installed(mimatrix)
    print("[b200_plugin] mimatrix.mi_all_pairs -> B200 engine", file=sys.stderr)
