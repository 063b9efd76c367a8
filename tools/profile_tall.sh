#!/bin/bash
# Evidence for the tall-N / narrow-m path (N = 8e6, m = 512, float64 MI):
# launch lists of one step per operand path, then ncu --set full of the
# word-operand fused kernel (statistics inside the launch).
#   tools/profile_tall.sh TAG      (outputs in gpurun_out/TAG_*)
set -e
tag=${1:-rXX}
mkdir -p gpurun_out
MI_B200_XP=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_tall_xp_launches.csv python tools/xp_steps.py 8000000 512 \
    > gpurun_out/${tag}_tall_xp_launches.log 2>&1
MI_B200_XP=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${tag}_tall_tma_launches.csv python tools/xp_steps.py 8000000 512 \
    > gpurun_out/${tag}_tall_tma_launches.log 2>&1
MI_B200_XP=1 ncu --set full --clock-control none --import-source on -k regex:gram_mi_kernel -s 2 -c 1 \
    -o gpurun_out/${tag}_tall_xp_fused python tools/xp_steps.py 8000000 512 > gpurun_out/${tag}_tall_xp_ncu.log 2>&1
echo profile_tall done
