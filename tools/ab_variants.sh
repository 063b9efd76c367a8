# A/B of library builds (MI_B200_LIB): config-4 fused kernel, sustained 2 s per build (twice,
# alternating) and the first tiles' trace.  Usage: tools/ab_variants.sh LIB.so ...
for r in 1 2; do
  for v in "" "$@"; do
    echo "== lib: ${v:-default}"
    MI_B200_LIB=$v python tools/power_probe.py 4 2 2>&1 | grep "^config"
  done
done
for v in "" "$@"; do
  echo "== trace lib: ${v:-default}"
  MI_B200_LIB=$v python tools/trace_tiles.py 4 f32 2>&1 | sed -n '5,9p'
done
