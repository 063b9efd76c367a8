#!/bin/bash
# One GPU call's worth of round evidence, each step only after the previous
# one ran clean: the default bench line, the launch list of a short bench run
# (cold-cache, serialised durations), and ncu --set full captures of the fused
# kernel and the unpack kernel of the config-3 step.
#   tools/profile_round.sh TAG      (outputs in gpurun_out/TAG_*)
set -e
tag=${1:-rXX}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gram_mi_kernel -s 3 -c 1 \
    -o gpurun_out/${tag}_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_fused.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"unpack_direct|unpack_fp4_direct|unpack_kernel" -s 3 -c 1 \
    -o gpurun_out/${tag}_unpack python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_unpack.log 2>&1
echo profile_round done
