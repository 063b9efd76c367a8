#!/bin/bash
# Run the reference's own test suite with the B200 engine installed as its
# mi_all_pairs / gram_ones / column_sums (paper_2411_19702_b200.compat).
#   stage  (build container):  tools/run_reference_suite.sh stage
#   run    (GPU box, via gpurun): tools/run_reference_suite.sh run
# `stage` copies /root/reference/pkg to baseline/_ref/pkg (git-ignored; it
# travels to the GPU box with the gpurun snapshot).  Nothing in tests/,
# smoke() or bench.py reads it.
set -e
REPO="$(cd "$(dirname "$0")/.." && pwd)"
case "$1" in
stage)
    rm -rf "$REPO/baseline/_ref/pkg"
    mkdir -p "$REPO/baseline/_ref"
    cp -r /root/reference/pkg "$REPO/baseline/_ref/pkg"
    rm -rf "$REPO/baseline/_ref/pkg/frontend" "$REPO/baseline/_ref/pkg/src/mimatrix/__pycache__"
    ;;
run)
    cd "$REPO/baseline/_ref/pkg"
    export B200_REPO="$REPO" NUMBA_CACHE_DIR=/tmp/numba_cache
    PYTHONPATH="$REPO/baseline/_ref/pkg/src:$REPO/tools/ref_suite" \
        python -m pytest -p b200_plugin -p no:cacheprovider tests -q -rf "${@:2}"
    ;;
*)
    echo "usage: $0 stage|run" >&2; exit 2;;
esac
