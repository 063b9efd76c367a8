# DRAM bytes and L2 hit rate of one config-4 fused launch per knob setting (env), by ncu
for e in "MI_B200_SERP=0" "MI_B200_SERP=1" "MI_B200_L2HINT=4" "MI_B200_L2HINT=4 MI_B200_SERP=1" "MI_B200_L2HINT=3" "MI_B200_L2HINT=0 MI_B200_SERP=1" "$@"; do
  echo "== $e"
  env $e ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
      --clock-control none -k regex:gram_mi_kernel -s 1 -c 1 python tools/fused_once.py 4 f32 2 2>&1 | grep -E "dram__bytes|hit_rate|gpu__time"
done
