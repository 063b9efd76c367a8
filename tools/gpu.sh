#!/bin/bash
# Rebuild the in-tree libraries here (they travel with the snapshot), then run
# the given command on a B200 through gpurun.  Usage: tools/gpu.sh TIMEOUT 'cmd'
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2411_19702_b200/csrc >/dev/null
make -s -C oracle >/dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
