# A/B of library builds (MI_B200_LIB): config-4 fused-kernel time under knob settings
for v in "" "$@"; do
  echo "== lib: ${v:-default}"
  MI_B200_LIB=$v ROUNDS=2 python tools/knob_probe.py 4 pace=8 pace=16 pace=24 pace=48 pace=64 pace=128 2>&1 | tail -7
done
